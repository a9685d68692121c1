"""Compress kernel comparison (device API, HBM-resident input, modes of
zs_set_transducer, include/zs_debug.h): 3 compress_cx with the product-automaton
parse (default), 19 without the long-line slices, 67 the DFA + transducer
parse, 131 every phase on byte-exact slices, 1 the generic transducer kernel.

    python tools/cmp_kernels.py [lines]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    ctx = _lib.context()
    d = z.default_dictionary()
    ctx.set_dictionary(d)
    for kind, seed, lines in (("aromatic", 2024, n), ("skewed", 2025, n // 4)):
        buf = synth.generate(kind, lines, seed)
        din = torch.from_numpy(buf).cuda()
        dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
        r = _lib.Result()
        outs = {}
        for mode in (3, 19, 67, 131, 1):
            ctx.lib.zs_set_transducer(ctx.h, mode)
            for _ in range(3):
                rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                                _lib.F_PREPROCESS | _lib.F_LENIENT, r)
                ctx.check(rc, "compress")
            ms = ctx.last_kernel_ms()
            outs[mode] = bytes(dout[:r.out_bytes].cpu().numpy())
            print(f"{kind:9s} {buf.size / 1e6:8.1f} MB mode {mode:2d} {ctx.lib.zs_last_kernel(ctx.h).decode():22s} "
                  f"{ms:8.3f} ms {buf.size / ms / 1e6:8.1f} GB/s")
        assert all(o == outs[3] for o in outs.values()), kind
    ctx.lib.zs_set_transducer(ctx.h, 3)


if __name__ == "__main__":
    main()
