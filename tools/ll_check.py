"""Long-line path (csrc/zs_ll.cuh) on the GPU: parity against the oracle on
long-line payloads and the time per line against the general routine.

    python tools/ll_check.py [--quick]
"""

import argparse
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402


def long_line(mols, L, rng, sep=b"."):
    parts, n = [], 0
    while n < L:
        m = rng.choice(mols)
        parts.append(m)
        n += len(m) + 1
    return sep.join(parts)


def ring_soup(L, rng, width=14):
    """Many overlapping rings: colours >= 10 ('%nn' rewrites, growing lines)."""
    out, n, open_ = [], 0, []
    free = list(range(1, 100))
    while n < L:
        if open_ and (len(open_) >= width or rng.random() < 0.5):
            rid = open_.pop(rng.randrange(len(open_)))
            free.append(rid)
        else:
            rid = free.pop(rng.randrange(len(free)))
            open_.append(rid)
        t = b"C" + (b"%d" % rid if rid < 10 else b"%%%02d" % rid)
        out.append(t)
        n += len(t)
    for rid in open_:
        out.append(b"C" + (b"%d" % rid if rid < 10 else b"%%%02d" % rid))
    return b"".join(out)


def check(payload, d, pre, lenient, mode=3):
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    want, st = oracle.run_stream(t, payload, "compress", pre, lenient, 1)
    ctx = _lib.context()
    ctx.lib.zs_set_transducer(ctx.h, mode)
    try:
        got, res = z.run_buffer(payload, d, "compress", preprocess=pre, lenient=lenient)
        if st["err_line"]:
            return res.err_line == st["err_line"], f"strict error at line {res.err_line}"
        ok = got.tobytes() == want and (res.lines, res.escapes, res.skipped, res.flagged) == \
            (st["lines"], st["escapes"], st["skipped"], st["flagged"])
        return ok, f"{len(want)} B"
    finally:
        ctx.lib.zs_set_transducer(ctx.h, 3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--time-only", action="store_true")
    ap.add_argument("--size", type=int, default=0, help="time only this line size (long-line kernels)")
    args = ap.parse_args()
    synth.build()
    d = z.default_dictionary()
    rng = random.Random(5)
    mols = synth.generate("mixed", 20000, 7).tobytes().split(b"\n")[:-1]
    short = b"\n".join(mols[:500]) + b"\n"
    cases = []
    for L in (2100, 3000, 9000, 40000, 300000, 2_000_000):
        cases.append((f"mixed {L}", short + long_line(mols, L, rng) + b"\n" + short))
    cases.append(("soup 200k", short + ring_soup(200_000, rng) + b"\n" + short))
    cases.append(("soup 50k w40", short + ring_soup(50_000, rng, 40) + b"\n" + short))
    cases.append(("two long + eof", long_line(mols, 50000, rng) + b"\n" + short + long_line(mols, 70000, rng)))
    cases.append(("digits", short + b"C" + b"1" * 5000 + b"\n" + b"(" + b"12" * 3000 + b"\n" + short))
    cases.append(("brackets", short + b"[" + b"C" * 3000 + b"]1CC1" + b"[NH4+]" * 900 + b"\n" + short))
    cases.append(("cr", short + long_line(mols, 9000, rng) + b"\r" + b"\n" + short))
    cases.append(("unclosed [", short + long_line(mols, 9000, rng) + b"C[N" + b"\n" + short))
    cases.append(("unpaired", short + long_line(mols, 9000, rng) + b"C7" + b"\n" + short))
    cases.append(("bad %", short + long_line(mols, 9000, rng) + b"C%1" + b"\n" + short))
    many = b"".join(long_line(mols, 3000 + 97 * k, rng) + b"\n" for k in range(300))
    cases.append(("300 long", many))
    bad = 0
    if args.time_only:
        cases = []
    for name, payload in cases:
        for pre in (False, True):
            for lenient in (True, False):
                ok, what = check(payload, d, pre, lenient)
                ok2, _ = check(payload, d, pre, lenient, 3 | 256)
                if not (ok and ok2):
                    bad += 1
                print(f"{name:16s} pre={int(pre)} lenient={int(lenient)}: ll {'ok' if ok else 'MISMATCH'}, "
                      f"general {'ok' if ok2 else 'MISMATCH'} ({what})", flush=True)
    # time: one 14 MB line, long-line kernels vs the general routine
    sizes = (args.size,) if args.size else (2_000_000,) if args.quick else (1_000_000, 14_000_000)
    for L in sizes:
        line = long_line(mols, L, rng)
        payload = np.frombuffer(line + b"\n", np.uint8)
        for pre in (False, True):
            for mode, label in ((3, "ll"), (3 | 256, "general")):
                ctx = _lib.context()
                ctx.lib.zs_set_transducer(ctx.h, mode)
                z.run_buffer(payload, d, "compress", preprocess=pre, lenient=True)
                t0 = time.perf_counter()
                z.run_buffer(payload, d, "compress", preprocess=pre, lenient=True)
                dt = time.perf_counter() - t0
                ctx.lib.zs_set_transducer(ctx.h, 3)
                print(f"time {L / 1e6:.1f} MB line pre={int(pre)} {label:8s}: {dt * 1e3:8.2f} ms  "
                      f"{L / dt / 1e9:.3f} GB/s", flush=True)
                if args.size or (label == "ll" and L > 2_000_000):
                    break
    print("bad", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
