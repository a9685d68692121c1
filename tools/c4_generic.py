"""C4 ablation dictionaries that take the generic (trie-walk) compress path:
time and check them against the oracle on C2's first 200k lines.

    python tools/c4_generic.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
buf = synth.generate("aromatic", 2_000_000, 2024)
small = synth.generate("aromatic", 200_000, 2024)
for name in ("t64_l15", "t128_l15", "t128_l8"):
    d = z.deserialize(open(os.path.join(HERE, "tests", "golden", "dicts", name + ".zsd"), "rb").read())
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    for pre in (False, True):
        got, _ = z.run_buffer(small, d, "compress", preprocess=pre, lenient=True)
        want, _ = oracle.run_stream(t, small.tobytes(), "compress", pre, True, 8)
        assert got.tobytes() == want, (name, pre)
        ctx = _lib.context()
        ctx.set_dictionary(d)
        din = torch.from_numpy(buf).cuda()
        dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
        r = _lib.Result()
        fl = (_lib.F_PREPROCESS if pre else 0) | _lib.F_LENIENT
        for _ in range(3):
            ctx.check(ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                                 fl, r), "compress")
        ms = ctx.last_kernel_ms()
        print(f"{name} pre={int(pre)} {ctx.lib.zs_last_kernel(ctx.h).decode():22s} {ms:7.3f} ms "
              f"{buf.size / ms / 1e6:7.1f} GB/s  (oracle match on 200k lines)")
