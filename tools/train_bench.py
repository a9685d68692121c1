"""Dictionary-training timing: GPU generate() vs the
CPU oracle restatement, on the generator corpora.

    python tools/train_bench.py [out.json]

Wall-clock per call (the API synchronises), best of 3 after a warm-up;
census (count_substrings) and selection (select_patterns) split out.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import dictionary as zd  # noqa: E402


def lines_of(kind, n, seed=2024):
    rows = synth.generate(kind, n, seed).tobytes().split(b"\n")
    if rows and rows[-1] == b"":
        rows.pop()
    return rows


def best(fn, k=3):
    fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), r


def main():
    out = []
    for kind, n, t, lmax in [("mixed", 50_000, 128, 8), ("mixed", 50_000, 128, 15),
                             ("aromatic", 1_000_000, 128, 8), ("aromatic", 10_000_000, 128, 8)]:
        lines = zd._preprocess_all(lines_of(kind, n), "lenient")
        nbytes = sum(len(l) + 1 for l in lines)
        p = z.GenerationParams(t=t, l_max=lmax)
        tc, table = best(lambda: z.count_substrings(lines, p))
        ts, _ = best(lambda: z.select_patterns(table, t))
        tg, d = best(lambda: z.generate(lines, p))
        row = {"corpus": f"{kind}_{n}", "bytes": nbytes, "t": t, "l_max": lmax, "rows": len(table),
               "gpu_count_s": round(tc, 4), "gpu_select_s": round(ts, 4), "gpu_generate_s": round(tg, 4)}
        if n <= 50_000:
            t0 = time.perf_counter()
            ref = oracle.train(lines, 2, lmax, t)
            row["oracle_s"] = round(time.perf_counter() - t0, 3)
            row["identical"] = ref == list(d.learned)
        out.append(row)
        print(json.dumps(row), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
