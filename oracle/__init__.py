"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU checker for the GPU codec: a ctypes binding of the plain-C restatement
in ``zs_oracle.c`` plus numpy restatements of the dictionary table builders.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline
and ``--impl reference``) may import this package, and only as the checker /
CPU baseline -- never as the thing measured or shipped.  The product package
``paper_2404_19391_b200`` does not import it.

Parity of this restatement is pinned against the reference's own outputs
(tests/golden/*.json, produced by tests/golden/make_golden.py running the
unmodified reference) in tests/test_oracle.py.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

ERR_NAMES = {1: "ZsmilesError", 2: "UnbalancedBracket", 3: "MalformedPercent",
             4: "UnpairedRingClosure", 5: "RingIdOverflow", 6: "UnknownCode",
             7: "TruncatedEscape"}

SMILES_ALPHABET = bytes(sorted(set(
    b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789[]()=#-+@/\\%.:*$~")))
PREPOPULATE = {"none": b"", "smiles": SMILES_ALPHABET, "printable": bytes(range(0x21, 0x7F))}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "zs_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "-B", "liboracle.so"])
    return _SO


class _Err(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("ids", ctypes.c_uint64 * 2)]


class _Tables(ctypes.Structure):
    _fields_ = [("children", ctypes.c_void_p), ("term_code", ctypes.c_void_p),
                ("exp_len", ctypes.c_void_p), ("valid", ctypes.c_void_p),
                ("exp_off", ctypes.c_void_p), ("exp_flat", ctypes.c_void_p)]


class _Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("lines", "in_bytes", "out_bytes", "escapes", "skipped", "flagged",
                 "err_line", "err_kind", "err_offset", "err_code")] + \
               [("err_ids", ctypes.c_uint64 * 2)]


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.zo_compress_batch.restype = I64
        lib.zo_compress_batch.argtypes = [P, P, P, P, I64, P, P]
        lib.zo_decompress_sizes.restype = None
        lib.zo_decompress_sizes.argtypes = [P, P, P, P, I64, P, P, P, P, P]
        lib.zo_decompress_fill.restype = None
        lib.zo_decompress_fill.argtypes = [P, P, P, P, I64, P, P, P]
        lib.zo_preprocess_line.restype = ctypes.c_int
        lib.zo_preprocess_line.argtypes = [P, I64, P, P, ctypes.POINTER(_Err)]
        lib.zo_run_stream.restype = ctypes.c_int
        lib.zo_run_stream.argtypes = [ctypes.POINTER(_Tables), P, I64, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_Stats)]
        lib.zo_free.argtypes = [P]
        lib.zo_count_substrings.restype = I64
        lib.zo_count_substrings.argtypes = [P, I64, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.POINTER(ctypes.c_void_p)]
        lib.zo_overlap.restype = I64
        lib.zo_overlap.argtypes = [P, ctypes.c_int, P, P, ctypes.c_int]
        lib.zo_select_patterns.restype = I64
        lib.zo_select_patterns.argtypes = [P, P, P, P, I64, ctypes.c_int, I64, P]
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data if a.size else 0


class Tables:
    """Encode trie (trie.py:22-50, 71-76) and decode tables
    (dictionary.py:112-129), restated over plain numpy."""

    def __init__(self, learned, identity):
        learned = [bytes(p) for p in learned]
        identity = bytes(sorted(set(identity)))
        entries = [(bytes([b]), b) for b in identity] + \
                  [(p, 0x80 + i) for i, p in enumerate(learned)]
        rows = [np.full(256, -1, np.int32)]
        term = [-1]
        self.max_len = 0
        for pat, code in entries:
            node = 0
            for b in pat:
                if rows[node][b] < 0:
                    rows[node][b] = len(rows)
                    rows.append(np.full(256, -1, np.int32))
                    term.append(-1)
                node = int(rows[node][b])
            if term[node] >= 0:
                raise ValueError(f"duplicate pattern {pat!r}")
            term[node] = code
            self.max_len = max(self.max_len, len(pat))
        self.children = np.ascontiguousarray(np.stack(rows))
        self.term_code = np.array(term, np.int16)
        exps = [b""] * 256
        self.valid = np.zeros(256, np.uint8)
        for pat, code in entries:
            exps[code] = pat
            self.valid[code] = 1
        self.exp_len = np.array([len(e) for e in exps], np.int32)
        self.exp_off = np.zeros(257, np.int64)
        np.cumsum(self.exp_len, out=self.exp_off[1:])
        self.exp_flat = np.frombuffer(b"".join(exps) or b"\0", np.uint8).copy()

    @classmethod
    def from_json(cls, dj):
        return cls([bytes.fromhex(p) for p in dj["learned"]], bytes.fromhex(dj["identity"]))

    @classmethod
    def from_zsd(cls, data: bytes):
        rows = data.split(b"\n")
        if rows and rows[-1] == b"":
            rows.pop()
        mode = rows[1].split(b"=", 1)[1].decode()
        return cls(rows[3:], PREPOPULATE[mode])

    def _ct(self):
        t = _Tables(_p(self.children), _p(self.term_code), _p(self.exp_len), _p(self.valid),
                    _p(self.exp_off), _p(self.exp_flat))
        return t


def _pack(lines):
    flat = np.frombuffer(b"".join(lines) or b"\0", np.uint8).copy()
    starts = np.zeros(len(lines) + 1, np.int64)
    np.cumsum([len(l) for l in lines], out=starts[1:])
    return flat, starts


def compress_batch(t: Tables, lines):
    """numba_impl.compress_batch harness shape (test_kernels.py:25-33)."""
    lib = _load()
    flat, starts = _pack(lines)
    out = np.zeros(max(1, 2 * int(starts[-1])), np.uint8)
    out_lens = np.zeros(len(lines), np.int64)
    esc = lib.zo_compress_batch(_p(t.children), _p(t.term_code), _p(flat), _p(starts),
                                len(lines), _p(out), _p(out_lens))
    recs = [out[2 * starts[i]:2 * starts[i] + out_lens[i]].tobytes() for i in range(len(lines))]
    return recs, int(esc)


def decompress_batch(t: Tables, recs):
    """decompress_sizes + cumsum + decompress_fill (test_kernels.py:35-48)."""
    lib = _load()
    flat, starts = _pack(recs)
    n = len(recs)
    out_lens = np.zeros(n, np.int64)
    status = np.zeros(n, np.int8)
    errpos = np.zeros(n, np.int64)
    total = ctypes.c_int64(0)
    esc = ctypes.c_int64(0)
    lib.zo_decompress_sizes(_p(t.exp_len), _p(t.valid), _p(flat), _p(starts), n, _p(out_lens),
                            _p(status), _p(errpos), ctypes.addressof(total), ctypes.addressof(esc))
    out_starts = np.zeros(n + 1, np.int64)
    np.cumsum(out_lens, out=out_starts[1:])
    out = np.zeros(max(1, total.value), np.uint8)
    lib.zo_decompress_fill(_p(t.exp_off), _p(t.exp_flat), _p(flat), _p(starts), n, _p(status),
                           _p(out), _p(out_starts))
    return {"out": out[:total.value].tobytes(), "out_lens": out_lens, "status": status,
            "errpos": errpos, "total": total.value, "escapes": esc.value}


def preprocess(line: bytes):
    """-> (0, renumbered) or (err_kind, (offset, ids_list))"""
    lib = _load()
    src = np.frombuffer(line or b"\0", np.uint8)
    out = np.zeros(3 * len(line) + 3, np.uint8)
    n = ctypes.c_int64(0)
    e = _Err()
    k = lib.zo_preprocess_line(_p(src), len(line), _p(out), ctypes.addressof(n), ctypes.byref(e))
    if k == 0:
        return 0, out[:n.value].tobytes()
    ids = [i for i in range(100) if (e.ids[i >> 6] >> (i & 63)) & 1]
    return k, (e.offset, ids)


def run_stream(t: Tables, payload, direction="compress", preprocess=False, lenient=False,
               threads=1):
    """Whole-buffer stream; -> (out_bytes or None, stats dict)."""
    lib = _load()
    buf = np.frombuffer(payload, np.uint8) if not isinstance(payload, np.ndarray) else payload
    outp = ctypes.c_void_p(0)
    st = _Stats()
    rc = lib.zo_run_stream(ctypes.byref(t._ct()), _p(buf), buf.size,
                           0 if direction == "compress" else 1, int(preprocess), int(lenient),
                           threads, ctypes.byref(outp), ctypes.byref(st))
    if rc != 0:
        raise MemoryError("oracle run_stream failed")
    stats = {k: getattr(st, k) for k, _ in _Stats._fields_ if k != "err_ids"}
    stats["err_ids"] = [i for i in range(100) if (st.err_ids[i >> 6] >> (i & 63)) & 1]
    data = None
    if outp.value:
        data = ctypes.string_at(outp.value, st.out_bytes)
        lib.zo_free(outp)
    return data, stats


# --------------------------------------------------------------------------
# dictionary training (zs_oracle_train.c; dictionary.py:169-320)
# --------------------------------------------------------------------------

WORKING_SET_CAP = 200_000  # dictionary.py:43


def count_substrings(lines, l_min, l_max):
    """-> (buf, pos i64[m], len i32[m], occ i64[m]) rows in the reference's
    RankTable order; pattern r = buf[pos[r]:pos[r] + len[r]]."""
    lib = _load()
    buf = np.frombuffer(b"\n".join(lines) or b"\0", np.uint8).copy()
    n = len(b"\n".join(lines))
    pp, lp, op = ctypes.c_void_p(0), ctypes.c_void_p(0), ctypes.c_void_p(0)
    m = lib.zo_count_substrings(_p(buf), n, l_min, l_max, ctypes.byref(pp), ctypes.byref(lp),
                                ctypes.byref(op))
    pos = np.ctypeslib.as_array((ctypes.c_int64 * m).from_address(pp.value)).copy() if m else \
        np.zeros(0, np.int64)
    ln = np.ctypeslib.as_array((ctypes.c_int32 * m).from_address(lp.value)).copy() if m else \
        np.zeros(0, np.int32)
    occ = np.ctypeslib.as_array((ctypes.c_int64 * m).from_address(op.value)).copy() if m else \
        np.zeros(0, np.int64)
    for q in (pp, lp, op):
        lib.zo_free(q)
    return buf, pos, ln, occ


def table_entries(lines, l_min, l_max):
    """[(pattern bytes, occurrences)] in row order."""
    buf, pos, ln, occ = count_substrings(lines, l_min, l_max)
    b = buf.tobytes()
    return [(b[p:p + l], int(o)) for p, l, o in zip(pos.tolist(), ln.tolist(), occ.tolist())]


def overlap(p: bytes, selected) -> int:
    lib = _load()
    sel = list(dict.fromkeys(bytes(s) for s in selected))
    flat = np.frombuffer(b"".join(sel) or b"\0", np.uint8).copy()
    lens = np.array([len(s) for s in sel] or [0], np.int32)
    src = np.frombuffer(bytes(p) or b"\0", np.uint8).copy()
    return int(lib.zo_overlap(_p(src), len(p), _p(flat), _p(lens), len(sel)))


def train(lines, l_min=2, l_max=8, t=128, cap=WORKING_SET_CAP):
    """count_substrings + select_patterns on already-preprocessed lines ->
    learned patterns in code order (dictionary.py:310-320 minus preprocess)."""
    lib = _load()
    buf, pos, ln, occ = count_substrings(lines, l_min, l_max)
    out = np.zeros(max(t, 1), np.int64)
    k = lib.zo_select_patterns(_p(buf), _p(pos), _p(ln), _p(occ), pos.size, t, cap, _p(out)) \
        if pos.size else 0
    b = buf.tobytes()
    return [b[pos[i]:pos[i] + ln[i]] for i in out[:k].tolist()]
