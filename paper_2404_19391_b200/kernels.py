"""The kernel plugin seam, B200 edition.

Same callables and array layouts as the reference's ``zsmiles.kernels``
module (kernels/__init__.py:28-33; numba_impl.py:16-139), backed by the
sm_100a parity-shim entry points of libzs.so.  There is a single backend
and no CPU fallback (the north star drops multi-backend dispatch):
``BACKEND == "sm_100a"``.  ``overlap_batch`` (numba_impl.py:142-169) is the
dictionary trainer's greedy-cover kernel.

The tables arrive in the reference layouts on every call, exactly like the
numba kernels; they are uploaded to the device once and cached by content.
"""

import hashlib

import numpy as np

from . import _lib

BACKEND = "sm_100a"


class _TableDict:
    """Adapter so Context.set_dictionary can take raw reference-layout tables."""

    def __init__(self, children=None, term_code=None, decode=None):
        self._children = children
        self._term = term_code
        self._decode = decode

    def cache_key(self):
        h = hashlib.sha1()
        for a in (self._children, self._term) + tuple(self._decode or ()):
            if a is not None:
                h.update(np.ascontiguousarray(a).tobytes())
        return ("raw", h.hexdigest())

    @property
    def encode_trie(self):
        class T:
            pass
        t = T()
        if self._children is None:
            t.children = np.full((1, 256), -1, np.int32)
            t.term_code = np.full(1, -1, np.int16)
        else:
            t.children, t.term_code = self._children, self._term
        return t

    @property
    def decode_tables(self):
        if self._decode is None:
            return (np.zeros(256, np.int32), np.zeros(256, np.uint8), np.zeros(257, np.int64),
                    np.zeros(1, np.uint8))
        return self._decode


def _decode_from(exp_len, valid, exp_off=None, exp_flat=None):
    if exp_off is None:
        exp_off = np.zeros(257, np.int64)
        np.cumsum(np.where(valid != 0, exp_len, 0), out=exp_off[1:])
    if exp_flat is None:
        exp_flat = np.zeros(max(1, int(exp_off[-1])), np.uint8)
    return exp_len, valid, exp_off, exp_flat


def compress_batch(children, term_code, flat, starts, out, out_lens) -> int:
    """Minimum-cost parse of every line; record i lands at out[2*starts[i]],
    its length in out_lens[i]; returns the number of escapes."""
    ctx = _lib.context()
    with ctx.lock:
        ctx.set_dictionary(_TableDict(children, term_code, _ident_decode(children, term_code)))
        flat = np.ascontiguousarray(flat, np.uint8)
        starts = np.ascontiguousarray(starts, np.int64)
        n = starts.shape[0] - 1
        lens = np.zeros(max(n, 0), np.int64)
        esc = np.zeros(1, np.int64)
        buf = out if (out.flags.c_contiguous and out.dtype == np.uint8) else np.empty_like(out, np.uint8)
        rc = ctx.lib.zs_compress_batch(ctx.h, _lib.ptr(flat), _lib.ptr(starts), n, _lib.ptr(buf),
                                       _lib.ptr(lens), _lib.ptr(esc))
        ctx.check(rc, "zs_compress_batch")
    if buf is not out:
        out[...] = buf
    out_lens[:n] = lens
    return int(esc[0])


def _ident_decode(children, term_code):
    # the compress call carries no decode tables; derive expansion lengths
    # from the trie so the device emit can step over codes
    exp_len = np.zeros(256, np.int32)
    valid = np.zeros(256, np.uint8)
    stack = [(0, 0)]
    ch = np.asarray(children)
    tc = np.asarray(term_code)
    while stack:
        node, depth = stack.pop()
        if tc[node] >= 0:
            exp_len[int(tc[node])] = depth
            valid[int(tc[node])] = 1
        for b in np.nonzero(ch[node] >= 0)[0]:
            stack.append((int(ch[node, b]), depth + 1))
    return _decode_from(exp_len, valid)


def decompress_sizes(exp_len, valid, flat, starts, out_lens, status, errpos):
    """First decode pass: per-record output size and status (0 ok, 1 unknown
    code, 2 truncated escape) with the in-record error offset.  Returns
    (total_out, escapes)."""
    ctx = _lib.context()
    with ctx.lock:
        ctx.set_dictionary(_TableDict(decode=_decode_from(np.asarray(exp_len, np.int32),
                                                          np.asarray(valid, np.uint8))))
        flat = np.ascontiguousarray(flat, np.uint8)
        starts = np.ascontiguousarray(starts, np.int64)
        n = starts.shape[0] - 1
        lens = np.zeros(n, np.int64)
        st = np.zeros(n, np.int8)
        ep = np.zeros(n, np.int64)
        tot = np.zeros(2, np.int64)
        rc = ctx.lib.zs_decompress_sizes(ctx.h, _lib.ptr(flat), _lib.ptr(starts), n, _lib.ptr(lens),
                                         _lib.ptr(st), _lib.ptr(ep), _lib.ptr(tot[0:1]),
                                         _lib.ptr(tot[1:2]))
        ctx.check(rc, "zs_decompress_sizes")
    out_lens[:n] = lens
    status[:n] = st
    errpos[:n] = ep
    return int(tot[0]), int(tot[1])


def decompress_fill(exp_off, exp_flat, flat, starts, status, out, out_starts) -> None:
    """Second decode pass: expand good records at out_starts[i]."""
    ctx = _lib.context()
    exp_off = np.asarray(exp_off, np.int64)
    exp_len = np.diff(exp_off).astype(np.int32)
    with ctx.lock:
        ctx.set_dictionary(_TableDict(decode=_decode_from(exp_len, (exp_len > 0).astype(np.uint8),
                                                          exp_off, np.asarray(exp_flat, np.uint8))))
        flat = np.ascontiguousarray(flat, np.uint8)
        starts = np.ascontiguousarray(starts, np.int64)
        n = starts.shape[0] - 1
        st = np.ascontiguousarray(status, np.int8)
        ost = np.ascontiguousarray(out_starts, np.int64)
        buf = out if out.flags.c_contiguous else np.empty_like(out)
        rc = ctx.lib.zs_decompress_fill(ctx.h, _lib.ptr(flat), _lib.ptr(starts), n, _lib.ptr(st),
                                        _lib.ptr(buf), _lib.ptr(ost))
        ctx.check(rc, "zs_decompress_fill")
    if buf is not out:
        out[...] = buf


def overlap_batch(children, term_len, pats, lens, out) -> None:
    """out[r] = bytes of pats[r, :lens[r]] covered by a greedy longest-match
    parse against the trie; unmatched positions advance one byte."""
    ctx = _lib.context()
    children = np.ascontiguousarray(children, np.int32)
    term_len = np.ascontiguousarray(term_len, np.int16)
    pats = np.ascontiguousarray(pats, np.uint8)
    lens = np.ascontiguousarray(lens, np.int64)
    n = int(lens.shape[0])
    res = np.zeros(n, np.int64)
    width = int(pats.shape[1]) if pats.ndim == 2 else 0
    with ctx.lock:
        rc = ctx.lib.zs_overlap_batch(ctx.h, _lib.ptr(children), _lib.ptr(term_len), children.shape[0],
                                      _lib.ptr(pats), width, _lib.ptr(lens), n, _lib.ptr(res))
        ctx.check(rc, "zs_overlap_batch")
    out[:n] = res
