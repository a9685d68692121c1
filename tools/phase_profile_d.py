"""Per-phase cycle breakdown of the decompress tile kernel (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

NAMES = ["load+scan", "validate-t0", "sums+scan", "expand-t0", "lookback+wait", "stats", "store", "tile-end"]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    buf = synth.generate("aromatic", n, 2024)
    d = z.default_dictionary()
    comp, _ = z.run_buffer(buf, d, "compress", preprocess=True)
    ctx = _lib.context()
    din = torch.from_numpy(comp).cuda()
    dout = torch.empty(3 * buf.size + 64, dtype=torch.uint8, device="cuda")
    r = _lib.Result()
    for timing in (0, 1):
        ctx.lib.zs_set_phase_timing(ctx.h, timing)
        for _ in range(3):
            rc = ctx.lib.zs_decompress_device(ctx.h, din.data_ptr(), comp.size, dout.data_ptr(),
                                              dout.numel(), 0, r)
            ctx.check(rc, "decompress")
        print(f"timing={timing} kernel {ctx.last_kernel_ms():.3f} ms, in {comp.size / ctx.last_kernel_ms() / 1e6:.1f} GB/s")
    cyc = np.zeros(8, np.uint64)
    ctx.lib.zs_last_phase_cycles(ctx.h, cyc.ctypes.data)
    tiles = (comp.size + 34815) // 34816
    tot = cyc.sum()
    for k in range(8):
        print(f"  {NAMES[k]:14s} {cyc[k] / tiles:10.0f} cyc/tile  {100 * cyc[k] / max(tot, 1):5.1f}%")


if __name__ == "__main__":
    main()
