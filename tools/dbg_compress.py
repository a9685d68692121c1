"""Compress the first N lines of a synthetic corpus through the device API and
compare with the CPU oracle (debug aid; run under compute-sanitizer)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import synth
import paper_2404_19391_b200 as z
from paper_2404_19391_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
kind = sys.argv[2] if len(sys.argv) > 2 else "aromatic"
buf = synth.generate(kind, n, 2024 if kind != "skewed" else 2025)
d = z.default_dictionary()
ctx = _lib.context()
ctx.set_dictionary(d)
ctx.lib.zs_set_transducer(ctx.h, int(os.environ.get("MODE", "3")))
din = torch.from_numpy(buf).cuda()
dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
r = _lib.Result()
rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                _lib.F_PREPROCESS | _lib.F_LENIENT, r)
ctx.check(rc, "compress")
reps = int(os.environ.get("REPS", "1"))
best = ctx.last_kernel_ms()
for _ in range(reps - 1):
    ctx.check(ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                         _lib.F_PREPROCESS | _lib.F_LENIENT, r), "compress")
    best = min(best, ctx.last_kernel_ms())
print("best of", reps, "ms", best, "GB/s", buf.size / best / 1e6)
got = dout[:r.out_bytes].cpu().numpy().tobytes()
t = oracle.Tables.from_zsd(z.serialize(d))
want, st = oracle.run_stream(t, buf, "compress", True, True, 8)
print("bytes", len(got), len(want), "equal", got == want, "ms", ctx.last_kernel_ms())
if got != want:
    gl, wl, il = got.split(b"\n"), want.split(b"\n"), buf.tobytes().split(b"\n")
    k = next(i for i, (a, b) in enumerate(zip(gl, wl)) if a != b)
    print("first bad line", k, il[k], gl[k], wl[k])
