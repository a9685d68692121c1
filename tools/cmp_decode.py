"""Streaming decode comparison (device API, HBM-resident input): the three
launches fx_count -> fx_scan -> fx_emit (mode 3, default) against the
single-pass fx_fused (mode 35), on C2-shaped libraries.

    python tools/cmp_decode.py [lines]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    ctx = _lib.context()
    d = z.default_dictionary()
    ctx.set_dictionary(d)
    for kind, seed, lines in (("aromatic", 2024, n), ("skewed", 2025, n // 4)):
        buf = synth.generate(kind, lines, seed)
        comp, _ = z.run_buffer(buf, d, "compress", preprocess=True, lenient=True)
        din = torch.from_numpy(comp).cuda()
        dout = torch.empty(buf.size + 4096, dtype=torch.uint8, device="cuda")
        r = _lib.Result()
        outs = {}
        for mode in (3, 35, 3, 35):
            ctx.lib.zs_set_transducer(ctx.h, mode)
            ms = []
            for _ in range(8):
                rc = ctx.lib.zs_decompress_device(ctx.h, din.data_ptr(), comp.size, dout.data_ptr(),
                                                  dout.numel(), 0, r)
                ctx.check(rc, "decompress")
                ms.append(ctx.last_kernel_ms())
            ms = sorted(ms[2:])[len(ms[2:]) // 2]
            outs[mode] = bytes(dout[:r.out_bytes].cpu().numpy())
            print(f"{kind:9s} {comp.size / 1e6:8.1f} MB in mode {mode:2d} {ctx.lib.zs_last_kernel(ctx.h).decode():26s} "
                  f"{ms:8.3f} ms {r.out_bytes / ms / 1e6:8.1f} GB/s out", flush=True)
        assert outs[3] == outs[35], kind
    ctx.lib.zs_set_transducer(ctx.h, 3)


if __name__ == "__main__":
    main()
