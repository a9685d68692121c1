"""Summarise an ncu report's source page (needs -lineinfo): top CUDA source
lines and top SASS instructions by warp-stall samples.

    python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys


def num(x):
    try:
        return int(x)
    except (TypeError, ValueError):
        try:
            return float(x)
        except (TypeError, ValueError):
            return 0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr = "?", None
    src, sass = [], []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        k = hdr.index("Warp Stall Sampling (All Samples)")
        thr = hdr.index("Avg. Threads Executed")
        if r[0]:
            src.append((num(r[k]), f"{fname}:{r[0]}", r[1].strip(), r[thr]))
        elif r[2] not in ("", "..."):
            sass.append((num(r[k]), r[2], r[3].strip(), r[thr]))
    tot = sum(s[0] for s in src) or 1
    print(f"total stall samples {tot}")
    print("--- source lines ---")
    for s, loc, text, thr in sorted(src, key=lambda x: -x[0])[:top]:
        print(f"{s:8d} {100 * s / tot:5.1f}%  {loc:22s} thr={thr[:5]:5s} {text[:80]}")
    print("--- sass ---")
    for s, addr, text, thr in sorted(sass, key=lambda x: -x[0])[:top // 2]:
        print(f"{s:8d} {100 * s / tot:5.1f}%  thr={thr[:5]:5s} {text[:80]}")


if __name__ == "__main__":
    main()


def stalls(rep, top=12):
    """Per-instruction stall-reason breakdown of the hottest SASS lines and
    the kernel-wide stall totals."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = [r for r in rows if len(r) > 5 and r[0] == "Address"][0]
    recs = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "Address"]
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {c: sum(num(d[c]) for d in recs) for c in cols}
    T = sum(tot.values()) or 1
    print("kernel stall totals:", ", ".join(f"{c[6:]}={100 * v / T:.1f}%" for c, v in
                                            sorted(tot.items(), key=lambda x: -x[1])[:8]))
    k = "Warp Stall Sampling (All Samples)"
    for d in sorted(recs, key=lambda d: -num(d[k]))[:top]:
        why = sorted(((num(d[c]), c[6:]) for c in cols), reverse=True)[:3]
        print(f"{num(d[k]):8.0f} {d['Source'].strip()[:60]:60s} " +
              " ".join(f"{w}={v:.0f}" for v, w in why if v))


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "stalls":
    stalls(sys.argv[1])


def section(rep, fname, lo, hi):
    """Instructions, samples and stall reasons for source lines [lo, hi] of fname."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    f, hdr, cur = None, None, None
    ins = samp = 0
    reasons = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            f = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[0]:
            cur = (f, int(r[0]))
            continue
        if r[2] in ("", "...") or not cur or cur[0] != fname or not lo <= cur[1] <= hi:
            continue
        d = dict(zip(hdr, r))
        ins += num(d["Instructions Executed"])
        samp += num(d["Warp Stall Sampling (All Samples)"])
        for c in hdr:
            if c.startswith("stall_") and "Not Issued" not in c:
                reasons[c[6:]] = reasons.get(c[6:], 0) + num(d[c])
    print(f"{fname}:{lo}-{hi}: warp-instr={ins} samples={samp} " +
          " ".join(f"{k}={v}" for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:6]))


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "section":
    section(sys.argv[1], sys.argv[4], int(sys.argv[5]), int(sys.argv[6]))


def insts(rep, top=40):
    """Top CUDA source lines by executed warp instructions (with the thread
    instructions / warp instructions ratio = average active lanes)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, hdr, src = "?", None, []
    for r in rows:
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0]:
            continue
        w = num(r[hdr.index("Instructions Executed")])
        t = num(r[hdr.index("Thread Instructions Executed")]) if "Thread Instructions Executed" in hdr else 0
        src.append((w, t, f"{fname}:{r[0]}", r[1].strip()))
    W = sum(s[0] for s in src) or 1
    T = sum(s[1] for s in src) or 1
    print(f"warp inst {W:.4g}  thread inst {T:.4g}  lanes/inst {T / W:.1f}")
    for w, t, loc, text in sorted(src, key=lambda x: -x[0])[:top]:
        print(f"{100 * w / W:5.1f}% {100 * t / T:5.1f}%t  {loc:20s} {text[:84]}")


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "inst":
    insts(sys.argv[1], int(sys.argv[2]))
