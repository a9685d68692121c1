"""Quick C4 timing (a few trained dictionaries, renumbering off/on, 2M lines)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
buf = synth.generate("aromatic", 2_000_000, 2024)
din = torch.from_numpy(buf).cuda()
dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
ctx = _lib.context()
for name in ("t16_l8", "t32_l8", "t64_l8", "default"):
    d = z.deserialize(open(os.path.join(HERE, "tests", "golden", "dicts", name + ".zsd"), "rb").read())
    ctx.set_dictionary(d)
    for pre in (0, 1):
        r = _lib.Result()
        for _ in range(3):
            ctx.check(ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                                 pre | _lib.F_LENIENT, r), "c")
        ms = ctx.last_kernel_ms()
        print(f"{name:8s} pre={pre} ratio {r.out_bytes / buf.size:.3f} {ms:7.3f} ms {buf.size / ms / 1e6:7.1f} GB/s")
