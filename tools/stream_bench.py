"""run_stream / CLI throughput on the C2 corpus (file in the page cache and
in-memory BytesIO), compress and decompress; pageable vs pinned host API.

    python tools/stream_bench.py
"""
import io
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

buf = synth.generate("aromatic", 10_000_000, 2024)
n = buf.size
d = z.default_dictionary()
z.run_buffer(buf[: 1 << 20], d, "compress", preprocess=True)  # warm up

t0 = time.perf_counter()
comp, _ = z.run_buffer(buf, d, "compress", preprocess=True)
t1 = time.perf_counter()
print(f"run_buffer (pageable numpy)  compress {n / (t1 - t0) / 1e9:6.2f} GB/s")

tmp = tempfile.mkdtemp()
src_p, dst_p = os.path.join(tmp, "c2.smi"), os.path.join(tmp, "c2.zs")
with open(src_p, "wb") as fh:
    fh.write(buf.tobytes())
for rnd in range(2):
    t0 = time.perf_counter()
    with open(src_p, "rb") as s, open(dst_p, "wb") as o:
        st = z.run_stream(s, o, d, "compress", preprocess=True)
    t1 = time.perf_counter()
    with open(dst_p, "rb") as s, open(os.devnull, "wb") as o:
        st2 = z.run_stream(s, o, d, "decompress")
    t2 = time.perf_counter()
print(f"run_stream file->file       compress {n / (t1 - t0) / 1e9:6.2f} GB/s   decompress (to /dev/null) "
      f"{st2.output_bytes / (t2 - t1) / 1e9:6.2f} GB/s out")
raw = buf.tobytes()
for rnd in range(2):
    src, dst = io.BytesIO(raw), io.BytesIO()
    t0 = time.perf_counter()
    z.run_stream(src, dst, d, "compress", preprocess=True)
    t1 = time.perf_counter()
    comp = dst.getvalue()
    src2, dst2 = io.BytesIO(comp), io.BytesIO()
    t2 = time.perf_counter()
    z.run_stream(src2, dst2, d, "decompress")
    t3 = time.perf_counter()
print(f"run_stream BytesIO          compress {n / (t1 - t0) / 1e9:6.2f} GB/s   decompress "
      f"{n / (t3 - t2) / 1e9:6.2f} GB/s out")
