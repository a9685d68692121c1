"""Parse-state resynchronisation experiment (CPU, host transducer tables):
start the right-to-left parse K bytes to the right of a position from the
line-end state and check whether it reaches the exact (DFA state, cost
window) there.  Design data for byte-exact lane slices.

    python tools/parse_sync.py
"""
import sys, ctypes, numpy as np, random
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import synth
import paper_2404_19391_b200 as z
from paper_2404_19391_b200 import _lib
lib = _lib.load()
d = z.default_dictionary()

from paper_2404_19391_b200 import trie as trie_mod
t = d.encode_trie

children = np.ascontiguousarray(t.children, dtype=np.int32); term = np.ascontiguousarray(t.term_code, dtype=np.int16)
dfa2 = np.zeros(256*97, np.uint16); t2 = np.zeros(1024*16, np.uint32); nw = ctypes.c_int32(); nm = ctypes.c_int32()
ok = lib.zs_build_t2_host(children.ctypes.data, term.ctypes.data, children.shape[0], dfa2.ctypes.data, t2.ctypes.data, ctypes.byref(nw), ctypes.byref(nm))
print("t2 ok", ok, nw.value, nm.value)
def col(b): return min((b - 0x20) & 0xffffffff, 96)
def run(s, lo, hi, st, wi):
    # process positions hi-1 down to lo; return state after processing lo
    for i in range(hi - 1, lo - 1, -1):
        e = int(dfa2[st * 97 + col(s[i])]); st = e & 0xff
        x = int(t2[wi * 16 + (e >> 8)]); wi = x & 0xfff
    return st, wi
buf = synth.generate("aromatic", 20000, 2024).tobytes().split(b"\n")[:-1]
rng = random.Random(1)
lines = [l for l in buf if len(l) > 40]
for K in (4, 6, 8, 12, 16, 24, 32):
    mism = 0; tot = 0
    for _ in range(3000):
        s = rng.choice(lines); n = len(s)
        m = rng.randrange(0, n - K)
        true = run(s, m, n, 0, 0)
        spec = run(s, m, m + K, 0, 0)
        tot += 1; mism += true != spec
    print(K, mism / tot)
