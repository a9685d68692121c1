"""Run a saved failing payload under flag / dictionary variants, each in a
fresh process (debug aid for tools/fuzz_gpu.py failures)."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
base = sys.argv[1]
meta = json.load(open(base + ".json"))
variants = []
for pre in (False, True):
    for len_ in (False, True):
        variants.append(dict(meta, pre=pre, lenient=len_))
# default dictionary (identity = SMILES alphabet)
import paper_2404_19391_b200 as z  # noqa: E402
dd = z.default_dictionary()
variants.append(dict(meta, learned=[p.hex() for p in dd.learned], identity=bytes(sorted(dd.identity)).hex(),
                     l_min=dd.l_min, l_max=dd.l_max))
# the fuzz dictionary plus the colour digits as identity codes
ident = bytes(sorted(set(bytes.fromhex(meta["identity"])) | set(b"0123")))
variants.append(dict(meta, identity=ident.hex()))
for k, v in enumerate(variants):
    path = f"/tmp/var_{k}"
    open(path + ".bin", "wb").write(open(base + ".bin", "rb").read())
    json.dump(v, open(path + ".json", "w"))
    r = subprocess.run([sys.executable, os.path.join(HERE, "fuzz_replay.py"), path] + sys.argv[2:],
                       capture_output=True, text=True, timeout=120)
    print(k, {kk: v[kk] for kk in ("pre", "lenient")}, "identity", len(bytes.fromhex(v["identity"])),
          "->", (r.stdout.strip().splitlines() or ["?"])[-1][:100], "| rc", r.returncode, flush=True)
