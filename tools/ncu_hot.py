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
