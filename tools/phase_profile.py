"""Per-phase cycle breakdown of the compress tile kernel (debug aid).

    python tools/phase_profile.py [lines] [kind]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

NAMES = ["warp-groups-avg", "groups/tile", "everything-else-t0", "warp-groups-max", "warp-groups-min", "renumber/warp", "parse-t0", "dp/warp"]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    kind = sys.argv[2] if len(sys.argv) > 2 else "aromatic"
    buf = synth.generate(kind, n, 2024 if kind != "skewed" else 2025)
    d = z.default_dictionary()
    ctx = _lib.context()
    ctx.set_dictionary(d)
    din = torch.from_numpy(buf).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    r = _lib.Result()
    for pre in (0, _lib.F_PREPROCESS):
        for timing in (0, 1):
            ctx.lib.zs_set_phase_timing(ctx.h, timing)
            for _ in range(3):
                rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(),
                                                dout.numel(), pre | _lib.F_LENIENT, r)
                ctx.check(rc, "compress")
            print(f"pre={pre} timing={timing} kernel {ctx.last_kernel_ms():.3f} ms, "
                  f"{buf.size / ctx.last_kernel_ms() / 1e6:.1f} GB/s")
        if pre == 0:
            cyc0 = np.zeros(8, np.uint64)
            ctx.lib.zs_last_phase_cycles(ctx.h, cyc0.ctypes.data)
            print("  pre-off phases/tile:", (cyc0[:8] / ((buf.size + 34815) // 34816)).astype(int))
    cyc = np.zeros(8, np.uint64)
    ctx.lib.zs_last_phase_cycles(ctx.h, cyc.ctypes.data)
    tiles = (buf.size + 34815) // 34816
    tot = cyc.sum()
    for k in range(8):
        print(f"  {NAMES[k]:14s} {cyc[k] / tiles:10.0f} cyc/tile  {100 * cyc[k] / max(tot, 1):5.1f}%")


if __name__ == "__main__":
    main()
