"""Byte-exact parse slices (compress_cx P4): how many slice entries were
warmed up from a found newline vs a virtual line end, and how many of each
disagreed with the right neighbour's exit state in the first check.

    python tools/spec_stats.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

for kind, n, seed in (("aromatic", 2_000_000, 2024), ("skewed", 500_000, 2025)):
    buf = synth.generate(kind, n, seed)
    ctx = _lib.context()
    ctx.set_dictionary(z.default_dictionary())
    din = torch.from_numpy(buf).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    r = _lib.Result()
    ctx.lib.zs_set_phase_timing(ctx.h, 6)
    ctx.check(ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(), 3, r), "c")
    cyc = np.zeros(8, np.uint64)
    ctx.lib.zs_last_phase_cycles(ctx.h, cyc.ctypes.data)
    ctx.lib.zs_set_phase_timing(ctx.h, 0)
    tiles = (buf.size + 29951) // 29952
    print(f"{kind}: per tile: newline-warmed {cyc[0] / tiles:.1f} (mismatch {cyc[2] / tiles:.2f}), "
          f"virtual {cyc[1] / tiles:.1f} (mismatch {cyc[3] / tiles:.2f})")
