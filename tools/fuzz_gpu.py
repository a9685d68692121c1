"""Randomised parity sweep on the GPU against the CPU oracle: random
dictionaries (identity sets, learned patterns of 2-8 bytes -> product
automaton, 9-16 -> key-window parse, longer -> generic walk), random corpora
(SMILES-like lines with brackets, '%nn' rings, CR, non-alphabet bytes, empty
and long lines, with / without a final newline), both flags, every kernel
mode, the device API at odd input offsets, and decompress of the output.

    python tools/fuzz_gpu.py [seconds] [seed]
"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

ALPHA = b"CcNnOoSsFlBrI()[]=#-+@/\\\\%.:*$~123456789"


def rand_line(rng, long_ok=True):
    k = rng.random()
    if k < 0.05:
        return b""
    if k < 0.055 and long_ok:  # a long line (the long-line kernels): molecules joined by '.'
        return b".".join(rand_line(rng, False) for _ in range(rng.randint(100, 1500)))
    if k < 0.65:  # SMILES-like: molecules with ring closures, some %nn
        parts = []
        for _ in range(rng.randint(1, 4)):
            body = bytearray(rng.choice(b"CcNOn") for _ in range(rng.randint(1, 12)))
            for r in range(rng.randint(0, 4)):
                rid = rng.choice([str(rng.randint(1, 9)).encode(), b"%" + str(rng.randint(10, 99)).encode()])
                i, j = sorted(rng.sample(range(len(body) + 1), 2)) if len(body) > 1 else (0, 0)
                body[j:j] = rid
                body[i:i] = rid
            if rng.random() < 0.2:
                body += b"[NH3+]"
            parts.append(bytes(body))
        line = b".".join(parts)
    else:
        n = rng.choice([rng.randint(0, 40), rng.randint(40, 400), rng.randint(400, 3000)])
        line = bytes(rng.choice(ALPHA) for _ in range(n))
    if rng.random() < 0.03:
        line += b"\r"
    if rng.random() < 0.03:
        line += bytes([rng.choice([0x01, 0x09, 0xff, 0x80, 0x20])])
    return line


def rand_dict(rng):
    ident = bytes(sorted(set(rng.choice(ALPHA + b"abcxyz") for _ in range(rng.randint(5, 60)))))
    kind = rng.random()
    lmax = 8 if kind < 0.6 else (16 if kind < 0.85 else 24)
    pats = set()
    for _ in range(rng.randint(0, 100)):
        L = rng.randint(2, lmax)
        pats.add(bytes(rng.choice(b"CcNO1()=") for _ in range(L)))
    pats = sorted(pats)[:128]
    lo = min([len(p) for p in pats], default=2)
    hi = max([len(p) for p in pats], default=2)
    return z.Dictionary(pats, None, l_min=min(lo, hi), l_max=max(lo, hi, 2), identity=ident)


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = random.Random(seed)
    ctx = _lib.context()
    t0 = time.time()
    cases = 0
    while time.time() - t0 < secs:
        d = rand_dict(rng)
        t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
        n_lines = rng.choice([1, 10, 300, 5000, 40000])
        lines = [rand_line(rng) for _ in range(n_lines)]
        if rng.random() < 0.2:  # a real corpus slice
            lines = synth.generate(rng.choice(["mixed", "skewed"]), n_lines, rng.randint(1, 99)).tobytes().split(b"\n")[:-1]
        payload = b"\n".join(lines) + (b"\n" if rng.random() < 0.8 else b"")
        mode = rng.choice([3, 3, 3, 19, 67, 131, 1, 3 | 256])
        pre, len_ = rng.random() < 0.7, rng.random() < 0.7
        ctx.lib.zs_set_transducer(ctx.h, mode)
        try:
            want, st = oracle.run_stream(t, payload, "compress", pre, len_, 8)
            got, res = z.run_buffer(payload, d, "compress", preprocess=pre, lenient=len_)
            if st["err_line"]:
                assert res.err_line == st["err_line"], ("err_line", res.err_line, st["err_line"])
            else:
                assert got.tobytes() == (want or b""), "compress bytes"
                assert (res.lines, res.escapes, res.skipped, res.flagged) == \
                    (st["lines"], st["escapes"], st["skipped"], st["flagged"]), "stats"
                # device API at an odd offset
                off = rng.randint(0, 15)
                din = torch.zeros(len(payload) + 32, dtype=torch.uint8, device="cuda")
                if payload:
                    din[off:off + len(payload)] = torch.frombuffer(bytearray(payload), dtype=torch.uint8).cuda()
                dout = torch.empty(2 * len(payload) + 64, dtype=torch.uint8, device="cuda")
                r = _lib.Result()
                with ctx.lock:
                    ctx.set_dictionary(d)
                    rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr() + off, len(payload), dout.data_ptr(),
                                                    dout.numel(), (1 if pre else 0) | (2 if len_ else 0), r)
                    ctx.check(rc, "zs_compress_device")
                assert dout[:r.out_bytes].cpu().numpy().tobytes() == (want or b""), "device API"
                if want:
                    back_want, _ = oracle.run_stream(t, want, "decompress", False, True, 8)
                    back, _ = z.run_buffer(want, d, "decompress", lenient=True)
                    assert back.tobytes() == (back_want or b""), "decompress"
        except Exception as e:  # noqa: BLE001 - report every failure with its inputs
            import json
            os.makedirs("gpurun_out", exist_ok=True)
            path = f"gpurun_out/fuzz_fail_{seed}_{cases}"
            with open(path + ".bin", "wb") as fh:
                fh.write(payload)
            with open(path + ".json", "w") as fh:
                json.dump({"learned": [p.hex() for p in d.learned], "identity": bytes(sorted(d.identity)).hex(),
                           "l_min": d.l_min, "l_max": d.l_max, "mode": mode, "pre": pre, "lenient": len_}, fh)
            print(f"FAIL case {cases} mode {mode} pre {pre} lenient {len_} lines {n_lines}: {e} -> {path}",
                  flush=True)
            print("dict", d.learned[:5], len(d.learned), sorted(d.identity)[:10])
            raise
        cases += 1
    ctx.lib.zs_set_transducer(ctx.h, 3)
    print(f"fuzz ok: {cases} cases in {time.time() - t0:.0f} s (seed {seed})")


if __name__ == "__main__":
    main()
