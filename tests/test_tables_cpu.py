"""CPU checks of the C-ABI library (no GPU needed).

* libzs.so loads and exports every symbol include/zs.h declares.
* The fast-path tables (reversed Aho-Corasick DFA + codes) that libzs
  derives from the reference trie, replayed here by a literal Python
  restatement of the device DP (csrc/zs_device.cuh dp_fast: keys
  (cost<<3)-pos in a W-wide window, escape loses ties), reproduce the
  reference's compressed records on the golden random dictionaries.
"""

import ctypes
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT
from paper_2404_19391_b200 import _lib

NCOL, FAST_W = 97, 8


def test_header_symbols_exported():
    lib = _lib.load()
    with open(f"{ROOT}/include/zs.h") as fh:
        declared = set(re.findall(r"^(?:int|int64_t|float|void|const char)\s*\*?\s*(zs_\w+)\(",
                                  fh.read(), re.M))
    assert declared == set(_lib.EXPORTS)
    with open(f"{ROOT}/include/zs_debug.h") as fh:
        debug = set(re.findall(r"^(?:int|int64_t|float|void|const char)\s*\*?\s*(zs_\w+)\(",
                               fh.read(), re.M))
    assert debug == set(_lib.DEBUG_EXPORTS)
    for name in declared | debug:
        assert hasattr(lib, name), name


def build_tables(t: oracle.Tables):
    lib = _lib.load()
    dfa = np.zeros(256 * NCOL, np.uint16)
    codes = np.zeros(256 * FAST_W, np.uint8)
    ns, ml = ctypes.c_int32(0), ctypes.c_int32(0)
    fast = lib.zs_build_tables_host(_lib.ptr(t.children), _lib.ptr(t.term_code),
                                    t.children.shape[0], _lib.ptr(dfa), _lib.ptr(codes),
                                    ctypes.byref(ns), ctypes.byref(ml))
    return fast, dfa[:ns.value * NCOL].reshape(ns.value, NCOL), \
        codes[:ns.value * FAST_W].reshape(ns.value, FAST_W), ml.value


def dp_fast_emulated(line: bytes, dfa, codes, W, exp_len):
    INF = 0x3FFFFFFF
    n = len(line)
    k = [INF] * (W + 1)
    key = -n
    st = 0
    dec = [0] * (n + 1)
    for i in range(n - 1, -1, -1):
        k[2:] = k[1:W]
        k[1] = key
        b = line[i]
        e = int(dfa[st, min((b - 0x20) & 0xFFFFFFFF, 96)])
        st = e & 0xFF
        mm = INF
        for L in range(1, W + 1):
            if e & (0x100 << (L - 1)):
                mm = min(mm, k[L])
        esc = k[1] + 16
        best = min(esc, mm + 8)
        t = best + i + W
        L = W - (t & 7)
        key = (t & ~7) - i
        dec[i] = 0x20 if esc < mm + 8 else int(codes[st, L - 1])
    out = bytearray()
    i = 0
    while i < n:
        c = dec[i]
        if c == 0x20:
            out += bytes([0x20, line[i]])
            i += 1
        else:
            out.append(c)
            i += int(exp_len[c])
    assert len(out) == key >> 3
    return bytes(out)


def test_fast_tables_reproduce_reference(codec_cases):
    n_fast = 0
    for c in codec_cases:
        t = oracle.Tables.from_json(c["dict"])
        fast, dfa, codes, ml = build_tables(t)
        assert ml == t.max_len
        if not fast:  # > 8-byte patterns or > 256 DFA states: generic trie walk
            continue
        n_fast += 1
        W = 2 if ml <= 2 else 4 if ml <= 4 else 6 if ml <= 6 else 8
        for line, rec in zip(c["lines"], c["records"]):
            got = dp_fast_emulated(bytes.fromhex(line), dfa, codes, W, t.exp_len)
            assert got.hex() == rec, (c["dict"]["learned"][:4], line)
    assert n_fast >= 10


def test_default_dictionary_is_fast():
    from conftest import golden_dict_bytes
    t = oracle.Tables.from_zsd(golden_dict_bytes())
    fast, dfa, codes, ml = build_tables(t)
    assert fast == 1 and ml == 6 and dfa.shape[0] <= 256


@pytest.mark.parametrize("chunk", [4096, 1 << 16, 64 << 20])
def test_host_chunk_cuts(chunk):
    """zs_*_host's newline-aligned chunking: cuts start at 0, end at n,
    increase strictly, each interior cut sits just past a newline, and chunk
    sizes stay bounded.  Hundreds of chunks (the 4 KB case) pin the ramp
    against overflow -- its doubling once went unclamped and wrapped after
    ~41 chunks (a 2.7 GB input crashed in memchr)."""
    lib = _lib.load()
    rng = np.random.default_rng(7)
    lines = [b"C" * int(k) for k in rng.integers(1, 200, 12000)] + [b"c1ccccc1" * 2000]
    buf = np.frombuffer(b"\n".join(lines) + b"\n", np.uint8)
    n = buf.size
    cap = 1 << 16
    cuts = np.zeros(cap, np.int64)
    m = lib.zs_debug_chunk_cuts(_lib.ptr(buf), n, chunk, _lib.ptr(cuts), cap)
    assert 2 <= m <= cap
    c = cuts[:m]
    assert c[0] == 0 and c[-1] == n
    assert (np.diff(c) > 0).all()
    assert (buf[c[1:-1] - 1] == ord("\n")).all()
    longest = max(len(x) for x in lines) + 1
    assert np.diff(c).max() <= max(chunk, 1 << 18) + longest
    if chunk == 4096:
        assert m > 100
    assert lib.zs_debug_chunk_cuts(None, 0, chunk, None, 0) == 1
    assert lib.zs_debug_chunk_cuts(_lib.ptr(buf), n, 0, _lib.ptr(cuts), cap) < 0
