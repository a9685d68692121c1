"""SMILES lexical layer: alphabet, tokenizer, ring-id renumbering.

``preprocess_line`` (the hot-path transform, smiles.py:183-213 of the
reference) runs on the GPU through ``zs_preprocess_batch``; the whole-file
path fuses the same device routine into the compress kernel.  ``tokenize``
is a host-side API utility that returns Token objects (it is not on the data
path; the device tokenizer in csrc/zs_device.cuh is what processes data).
"""

from enum import Enum

import numpy as np

from . import _lib
from .errors import (
    ERR_BRACKET,
    ERR_OVERFLOW,
    ERR_PERCENT,
    ERR_UNPAIRED,
    MalformedPercent,
    UnbalancedBracket,
    from_kind,
)

ALPHABET = frozenset(
    b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789[]()=#-+@/\\%.:*$~")

ALPHABET_MASK = np.zeros(256, dtype=bool)
ALPHABET_MASK[sorted(ALPHABET)] = True

_BOND = frozenset(b"-=#$:/\\~")


def is_alphabet_member(b: int) -> bool:
    return b in ALPHABET


class TokenKind(Enum):
    Atom = "atom"
    BracketAtom = "bracket_atom"
    Bond = "bond"
    BranchOpen = "branch_open"
    BranchClose = "branch_close"
    RingClosure = "ring_closure"
    Dot = "dot"
    Other = "other"


class Token:
    __slots__ = ("kind", "start", "end", "ring_id")

    def __init__(self, kind, start, end, ring_id=None):
        self.kind = kind
        self.start = start
        self.end = end
        self.ring_id = ring_id

    def text(self, line: bytes) -> bytes:
        return line[self.start:self.end]

    def __repr__(self):
        rid = "" if self.ring_id is None else f", ring_id={self.ring_id}"
        return f"Token({self.kind.name}, {self.start}:{self.end}{rid})"

    def __eq__(self, other):
        return isinstance(other, Token) and (self.kind, self.start, self.end, self.ring_id) == \
            (other.kind, other.start, other.end, other.ring_id)


_OK_PRED = (TokenKind.Atom, TokenKind.BracketAtom, TokenKind.Bond, TokenKind.RingClosure)
_SINGLE = {0x28: TokenKind.BranchOpen, 0x29: TokenKind.BranchClose, 0x2E: TokenKind.Dot}


def tokenize(line: bytes) -> list:
    """Token spans partitioning `line` (smiles.py:83-137 semantics): '[' runs
    to the next ']', '%' needs two digits, a digit or %nn is a ring closure
    only after an atom, bracket atom, bond or ring closure."""
    out = []
    i, n = 0, len(line)
    prev_ok = False
    while i < n:
        b = line[i]
        if b == 0x5B:
            j = line.find(b"]", i + 1)
            if j < 0:
                raise UnbalancedBracket(f"unclosed '[' at offset {i}")
            tok = Token(TokenKind.BracketAtom, i, j + 1)
        elif b == 0x25:
            if not (i + 2 < n and 0x30 <= line[i + 1] <= 0x39 and 0x30 <= line[i + 2] <= 0x39):
                raise MalformedPercent(f"'%' without two digits at offset {i}")
            rid = int(line[i + 1:i + 3])
            tok = Token(TokenKind.RingClosure, i, i + 3, rid) if prev_ok else \
                Token(TokenKind.Other, i, i + 3)
        elif 0x30 <= b <= 0x39:
            tok = Token(TokenKind.RingClosure, i, i + 1, b - 0x30) if prev_ok else \
                Token(TokenKind.Other, i, i + 1)
        elif (0x41 <= b <= 0x5A) or (0x61 <= b <= 0x7A) or b == 0x2A:
            tok = Token(TokenKind.Atom, i, i + 1)
        elif b in _BOND:
            tok = Token(TokenKind.Bond, i, i + 1)
        else:
            tok = Token(_SINGLE.get(b, TokenKind.Other), i, i + 1)
        out.append(tok)
        prev_ok = tok.kind in _OK_PRED
        i = tok.end
    return out


def preprocess_batch(lines, device=None):
    """GPU ring renumbering of many lines (strict semantics).

    Returns a list of (kind, result): kind 0 -> result is the renumbered
    line; otherwise kind is a ZS_ERR_* code and result is (offset, (lo, hi)).
    """
    lines = list(lines)
    if not lines:
        return []
    ctx = _lib.context(device)
    flat = np.frombuffer(b"".join(lines) or b"\0", np.uint8)
    starts = np.zeros(len(lines) + 1, np.int64)
    np.cumsum([len(l) for l in lines], out=starts[1:])
    n = len(lines)
    out = np.zeros(3 * int(starts[-1]) + 3 * n + 1, np.uint8)
    lens = np.zeros(n, np.int64)
    status = np.zeros(n, np.int8)
    eoff = np.zeros(n, np.int64)
    ids = np.zeros(2 * n, np.uint64)
    with ctx.lock:
        rc = ctx.lib.zs_preprocess_batch(ctx.h, _lib.ptr(flat), _lib.ptr(starts), n, _lib.ptr(out),
                                         _lib.ptr(lens), _lib.ptr(status), _lib.ptr(eoff),
                                         _lib.ptr(ids))
        ctx.check(rc, "zs_preprocess_batch")
    res = []
    for i in range(n):
        k = int(status[i])
        if k == 0:
            o = 3 * int(starts[i]) + 3 * i
            res.append((0, out[o:o + lens[i]].tobytes()))
        else:
            res.append((k, (int(eoff[i]), (int(ids[2 * i]), int(ids[2 * i + 1])))))
    return res


def preprocess_line(line: bytes, mode: str = "strict") -> bytes:
    """Renumber ring-closure ids so the earliest-closing ring takes the lowest
    free id (reference smiles.py:183-213), on the GPU.  Lenient mode returns
    the line unchanged on tokenize/pairing errors; RingIdOverflow is raised
    in both modes, as in the reference."""
    if mode not in ("strict", "lenient"):
        raise ValueError(f"unknown mode {mode!r}")
    [(kind, res)] = preprocess_batch([bytes(line)])
    if kind == 0:
        return res
    if mode == "lenient" and kind in (ERR_BRACKET, ERR_PERCENT, ERR_UNPAIRED):
        return bytes(line)
    off, ids = res
    raise from_kind(kind, off, ids)


__all__ = ["ALPHABET", "ALPHABET_MASK", "Token", "TokenKind", "is_alphabet_member", "tokenize",
           "preprocess_line", "preprocess_batch", "ERR_OVERFLOW"]
