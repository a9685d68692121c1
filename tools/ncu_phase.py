"""Per-phase instruction accounting of an ncu --set full report (needs -lineinfo).

Sums 'Instructions Executed' (warp instructions) and 'Thread Instructions
Executed' per CUDA source line, then per phase given as line ranges of the
kernel's source file.

    python tools/ncu_phase.py report.ncu-rep FILE name:lo-hi [name:lo-hi ...] [--bytes N]
"""
import csv
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


def per_line(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr = "?", None
    res = {}
    for r in rows:
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0]:
            continue
        wi = num(r[hdr.index("Instructions Executed")])
        ti = num(r[hdr.index("Thread Instructions Executed")])
        st = num(r[hdr.index("Warp Stall Sampling (All Samples)")])
        res[(fname, int(r[0]))] = (wi, ti, st)
    return res


def main():
    a = sys.argv[1:]
    nbytes = None
    if "--bytes" in a:
        i = a.index("--bytes")
        nbytes = float(a[i + 1])
        del a[i:i + 2]
    rep, fname, specs = a[0], a[1], a[2:]
    d = per_line(rep)
    W = sum(v[0] for v in d.values()) or 1
    T = sum(v[1] for v in d.values()) or 1
    S = sum(v[2] for v in d.values()) or 1
    print(f"total warp inst {W:.4g}  thread inst {T:.4g}  lanes/inst {T / W:.1f}")
    seen = set()
    print(f"{'phase':14s} {'warp inst':>12s} {'%':>6s} {'lanes':>6s} {'stall%':>7s}" +
          (f" {'winst/B':>8s} {'tinst/B':>8s}" if nbytes else ""))
    for sp in specs:
        name, rng = sp.split(":")
        lo, hi = (int(x) for x in rng.split("-"))
        keys = [k for k in d if k[0] == fname and lo <= k[1] <= hi]
        seen.update(keys)
        w = sum(d[k][0] for k in keys)
        t = sum(d[k][1] for k in keys)
        s = sum(d[k][2] for k in keys)
        extra = f" {w / nbytes:8.3f} {t / nbytes:8.2f}" if nbytes else ""
        print(f"{name:14s} {w:12.4g} {100 * w / W:6.1f} {t / max(w, 1):6.1f} {100 * s / S:7.1f}" + extra)
    rest = [k for k in d if k not in seen]
    w = sum(d[k][0] for k in rest)
    t = sum(d[k][1] for k in rest)
    s = sum(d[k][2] for k in rest)
    extra = f" {w / nbytes:8.3f} {t / nbytes:8.2f}" if nbytes else ""
    print(f"{'other':14s} {w:12.4g} {100 * w / W:6.1f} {t / max(w, 1):6.1f} {100 * s / S:7.1f}" + extra)
    by_file = {}
    for k in rest:
        by_file.setdefault(k[0], [0, 0])
        by_file[k[0]][0] += d[k][0]
    for f, (w, _) in sorted(by_file.items(), key=lambda x: -x[1][0])[:6]:
        print(f"   other in {f}: {w:.4g}")


if __name__ == "__main__":
    main()
