"""Per-phase cycle breakdown of compress_cx (thread 0's clock64 deltas,
which include barrier waits, so each phase reads as its slowest warp).

    python tools/phase_cx.py [lines] [kind]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

NAMES = ["load+cuts", "w0 tokenizer", "w0 pairing", "w0 parse", "wait slowest", "rare+scan", "emit+lookback", "store"]
TILE = 19968  # CX_TILE (zs_cx.cuh)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    kind = sys.argv[2] if len(sys.argv) > 2 else "aromatic"
    buf = synth.generate(kind, n, 2024 if kind != "skewed" else 2025)
    d = z.default_dictionary()
    ctx = _lib.context()
    ctx.set_dictionary(d)
    ctx.lib.zs_set_transducer(ctx.h, int(os.environ.get("MODE", "3")))
    din = torch.from_numpy(buf).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    r = _lib.Result()
    tiles = (buf.size + TILE - 1) // TILE
    modes = [int(m) for m in os.environ.get("MODES", "1").split(",")]
    for pre in (0, _lib.F_PREPROCESS):
        for timing in [0] + modes:
            ctx.lib.zs_set_phase_timing(ctx.h, timing)
            for _ in range(3):
                rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(),
                                                dout.numel(), pre | _lib.F_LENIENT, r)
                ctx.check(rc, "compress")
            print(f"pre={pre} timing={timing} {ctx.lib.zs_last_kernel(ctx.h).decode()} "
                  f"{ctx.last_kernel_ms():.3f} ms, {buf.size / ctx.last_kernel_ms() / 1e6:.1f} GB/s")
            cyc = np.zeros(8, np.uint64)
            ctx.lib.zs_last_phase_cycles(ctx.h, cyc.ctypes.data)
            tot = cyc.sum()
            if timing:
                for k in range(8):
                    print(f"  {NAMES[k]:14s} {cyc[k] / tiles:10.0f} cyc/tile  {100 * cyc[k] / max(tot, 1):5.1f}%")
    ctx.lib.zs_set_phase_timing(ctx.h, 0)


if __name__ == "__main__" and (len(sys.argv) < 3 or sys.argv[2] != "ranges"):
    main()


def ranges():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    buf = synth.generate("aromatic", n, 2024)
    d = z.default_dictionary()
    ctx = _lib.context()
    ctx.set_dictionary(d)
    din = torch.from_numpy(buf).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    r = _lib.Result()
    ctx.lib.zs_set_phase_timing(ctx.h, 2)
    rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                    _lib.F_PREPROCESS | _lib.F_LENIENT, r)
    ctx.check(rc, "compress")
    cyc = np.zeros(8, np.uint64)
    ctx.lib.zs_last_phase_cycles(ctx.h, cyc.ctypes.data)
    ctx.lib.zs_set_phase_timing(ctx.h, 0)
    print(f"warps {cyc[2]}  mean lane range {cyc[1] / cyc[2] / 32:.1f}  mean warp max {cyc[0] / cyc[2]:.1f}")
    print(f"P3 events: mean per lane {cyc[4] / cyc[2] / 32:.1f}  mean warp max {cyc[3] / cyc[2]:.1f}  "
          f"compactions per warp {cyc[5] / cyc[2]:.2f}")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "ranges":
    ranges()
