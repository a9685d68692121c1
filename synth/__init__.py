"""Synthetic SMILES libraries of the SURVEY.md §8d shapes (bench/test input).

`generate(kind, n_lines, seed)` returns the same bytes as the reference
generator (pkg/scripts/make_corpus.py MoleculeGen, seeded CPython
`random.Random`) via a C port (`molgen.c`), so corpora of 10M+ lines are made
in seconds on the GPU box.  Pinned by tests/golden/corpus_hashes.json.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmolgen.so")
KINDS = {"mixed": 0, "aromatic": 1, "aliphatic": 2, "skewed": 3}
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "molgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _SO, src])
    return _SO


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        lib = ctypes.CDLL(_SO)
        lib.synth_generate.restype = ctypes.c_void_p
        lib.synth_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64,
                                       ctypes.POINTER(ctypes.c_int64)]
        lib.synth_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


def generate(kind: str, n_lines: int, seed: int = 2024) -> np.ndarray:
    """Newline-terminated corpus as a uint8 array."""
    lib = _load()
    n = ctypes.c_int64(0)
    p = lib.synth_generate(KINDS[kind], seed, n_lines, ctypes.byref(n))
    if not p:
        raise ValueError(kind)
    try:
        arr = np.empty(n.value, np.uint8)
        if n.value:
            ctypes.memmove(arr.ctypes.data, p, n.value)
    finally:
        lib.synth_free(p)
    return arr


# The named configs of BASELINE.json / SURVEY.md §8d.
CONFIGS = {
    "c1_100k": ("aromatic", 100_000, 2024),
    "c2_10m": ("aromatic", 10_000_000, 2024),
    "c3_skewed_5m": ("skewed", 5_000_000, 2025),
    "mixed_50k": ("mixed", 50_000, 2024),
    "aromatic_10k": ("aromatic", 10_000, 2024),
    "aliphatic_10k": ("aliphatic", 10_000, 2024),
}
