"""Host-API round trip (pinned buffers) for one chunk size (ZS_CHUNK_MB env).

    ZS_CHUNK_MB=32 python tools/e2e_chunks.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

buf = synth.generate("aromatic", 10_000_000, 2024)
ctx = _lib.context()
ctx.set_dictionary(z.default_dictionary())
n = buf.size
h_in = torch.from_numpy(buf).pin_memory()
h_c = torch.empty(2 * n + 64, dtype=torch.uint8).pin_memory()
h_b = torch.empty(n + 64, dtype=torch.uint8).pin_memory()
rc_, rd_ = _lib.Result(), _lib.Result()
fl = _lib.F_PREPROCESS | _lib.F_LENIENT


def step():
    ctx.check(ctx.lib.zs_compress_host(ctx.h, h_in.data_ptr(), n, h_c.data_ptr(), h_c.numel(), fl, rc_), "c")
    ctx.check(ctx.lib.zs_decompress_host(ctx.h, h_c.data_ptr(), rc_.out_bytes, h_b.data_ptr(), h_b.numel(), 0, rd_),
              "d")


for _ in range(2):
    step()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    ctx.check(ctx.lib.zs_compress_host(ctx.h, h_in.data_ptr(), n, h_c.data_ptr(), h_c.numel(), fl, rc_), "c")
    t1 = time.perf_counter()
    ctx.check(ctx.lib.zs_decompress_host(ctx.h, h_c.data_ptr(), rc_.out_bytes, h_b.data_ptr(), h_b.numel(), 0, rd_),
              "d")
    t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1))
c = min(t[0] for t in ts)
d = min(t[1] for t in ts)
assert bytes(h_b[:rd_.out_bytes].numpy()) == bytes(z.run_buffer(h_c[:rc_.out_bytes].numpy(),
                                                                 z.default_dictionary(), "decompress")[0])
print(f"chunk {os.environ.get('ZS_CHUNK_MB', '32')} MB: compress {c * 1e3:.2f} ms  decompress {d * 1e3:.2f} ms  "
      f"round trip {n / (c + d) / 1e6:.0f} MB/s")
