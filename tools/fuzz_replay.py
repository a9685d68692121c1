"""Replay a saved fuzz failure (tools/fuzz_gpu.py): gpurun_out/fuzz_fail_<seed>_<case>.{bin,json}.

    python tools/fuzz_replay.py gpurun_out/fuzz_fail_1_0 [mode]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

base = sys.argv[1]
meta = json.load(open(base + ".json"))
payload = open(base + ".bin", "rb").read()
d = z.Dictionary([bytes.fromhex(p) for p in meta["learned"]], None, l_min=meta["l_min"], l_max=meta["l_max"],
                 identity=bytes.fromhex(meta["identity"]))
mode = int(sys.argv[2]) if len(sys.argv) > 2 else meta["mode"]
ctx = _lib.context()
ctx.lib.zs_set_transducer(ctx.h, mode)
t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
want, st = oracle.run_stream(t, payload, "compress", meta["pre"], meta["lenient"], 8)
print("payload", len(payload), "lines", payload.count(b"\n"), "mode", mode, "pre", meta["pre"], "lenient",
      meta["lenient"], "max line", max(len(x) for x in payload.split(b"\n")), "learned", len(d.learned),
      "lmax", max([len(p) for p in d.learned], default=0))
got, res = z.run_buffer(payload, d, "compress", preprocess=meta["pre"], lenient=meta["lenient"])
print("equal", got.tobytes() == (want or b""), res.err_line, st["err_line"])
