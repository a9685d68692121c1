"""Per-phase instruction table of a compress_cx ncu capture: the phase
boundaries are found from the section markers in zs_cx.cuh ("---- P1:",
"---- P2:", ...), then tools/ncu_phase.py sums the warp / thread
instructions of each range.

    python tools/phase_ranges.py report.ncu-rep [bytes]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2404_19391_b200", "csrc", "zs_cx.cuh")
MARKS = [("load+P1", "---- P1: newline bitmap"), ("P2 tokenizer", "---- P2: tokenizer"),
         ("P3 pairing", "---- P3: ring pairing"), ("P3 compaction", "---- '%nn' compaction"),
         ("P4 parse", "---- P4: min-cost parse"), ("rare lines", "---- rare lines: general routine"),
         ("P5/P6 emit", "const bool staged = tile_out"), ("store+stats", "---- strict error: details")]


def main():
    rep = sys.argv[1]
    nbytes = sys.argv[2] if len(sys.argv) > 2 else "459831407"
    lines = open(SRC).read().split("\n")
    kern = next(i for i, l in enumerate(lines) if "compress_cx(Job job" in l) + 1
    starts = []
    for name, pat in MARKS:
        k = next(i for i, l in enumerate(lines) if pat in l and i >= kern) + 1
        starts.append((name, k))
    specs = [f"helpers+setup:1-{starts[0][1] - 1}"]
    for (name, a), nxt in zip(starts, starts[1:] + [("end", len(lines) + 1)]):
        specs.append(f"{name.replace(' ', '_')}:{a}-{nxt[1] - 1}")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_phase.py"), rep, "zs_cx.cuh", *specs,
                          "--bytes", nbytes], capture_output=True, text=True)
    print(out.stdout + out.stderr)


if __name__ == "__main__":
    main()
