"""Fixed compression dictionary and the ZSD1 file format.

Mirrors the reference's ``Dictionary`` (dictionary.py:65-141), its code
assignment (identity byte -> itself, learned[i] -> 0x80+i), the table
builders the codec consumes (``encode_trie``: trie.py layout;
``decode_tables``: dictionary.py:112-129) and ZSD1 (de)serialization
(dictionary.py:322-383).  Dictionary *training* (``generate`` and friends)
is out of scope for this build (not on the codec path).
"""

from functools import cached_property

import numpy as np

from .errors import (
    BadMagic,
    DictionaryFormatError,
    NonAlphabetByteInPattern,
    PatternTooLong,
    TooManyPatterns,
    UnsupportedVersion,
)
from .smiles import ALPHABET
from .trie import PatternTrie, build_trie

MAX_PATTERNS = 128
MAX_PATTERN_LEN = 64

PREPOPULATE_SETS = {
    "none": frozenset(),
    "smiles": ALPHABET,
    "printable": frozenset(range(0x21, 0x7F)),
}

_MAGIC = b"ZSD1"


class Dictionary:
    """Immutable dictionary: learned patterns in code order plus the
    single-byte identity set."""

    def __init__(self, learned, prepopulate="smiles", *, l_min=2, l_max=8, identity=None):
        self.learned = tuple(bytes(p) for p in learned)
        self.l_min = l_min
        self.l_max = l_max
        self.prepopulate = prepopulate
        if identity is None:
            if prepopulate not in PREPOPULATE_SETS:
                raise ValueError(f"unknown prepopulate mode {prepopulate!r}")
            self.identity = PREPOPULATE_SETS[prepopulate]
        else:
            if prepopulate is not None:
                raise ValueError("pass prepopulate=None with an explicit identity set")
            self.identity = frozenset(identity)
        self._validate()

    def _validate(self):
        if not 2 <= self.l_min <= self.l_max <= MAX_PATTERN_LEN:
            raise ValueError(f"bad length bounds [{self.l_min}, {self.l_max}]")
        if len(self.learned) > MAX_PATTERNS:
            raise ValueError(f"{len(self.learned)} learned patterns, max {MAX_PATTERNS}")
        if len(set(self.learned)) != len(self.learned):
            raise ValueError("duplicate learned patterns")
        for p in self.learned:
            if not self.l_min <= len(p) <= self.l_max:
                raise ValueError(f"pattern {p!r} outside [{self.l_min}, {self.l_max}]")
            if not set(p) <= ALPHABET:
                raise ValueError(f"pattern {p!r} has non-alphabet bytes")
        for b in self.identity:
            if not 0x21 <= b <= 0x7E:
                raise ValueError(f"identity byte 0x{b:02x} not printable")

    @cached_property
    def code_of(self) -> dict:
        codes = {bytes([b]): b for b in self.identity}
        codes.update({p: 0x80 + i for i, p in enumerate(self.learned)})
        return codes

    @cached_property
    def encode_trie(self) -> PatternTrie:
        return build_trie(self)

    @cached_property
    def decode_tables(self):
        """(exp_len i32[256], valid u8[256], exp_off i64[257], exp_flat u8[])"""
        exps = [b""] * 256
        valid = np.zeros(256, np.uint8)
        for b in self.identity:
            exps[b] = bytes([b])
            valid[b] = 1
        for i, p in enumerate(self.learned):
            exps[0x80 + i] = p
            valid[0x80 + i] = 1
        exp_len = np.array([len(e) for e in exps], np.int32)
        exp_off = np.zeros(257, np.int64)
        np.cumsum(exp_len, out=exp_off[1:])
        exp_flat = np.frombuffer(b"".join(exps), np.uint8).copy()
        return exp_len, valid, exp_off, exp_flat

    def cache_key(self):
        return (self.learned, self.identity)

    def __eq__(self, other):
        return (isinstance(other, Dictionary) and self.learned == other.learned
                and self.identity == other.identity and self.l_min == other.l_min
                and self.l_max == other.l_max and self.prepopulate == other.prepopulate)

    def __hash__(self):
        return hash((self.learned, self.identity, self.l_min, self.l_max, self.prepopulate))

    def __repr__(self):
        return (f"Dictionary({len(self.learned)} learned, {len(self.identity)} identity, "
                f"prepopulate={self.prepopulate!r})")


def serialize(d: Dictionary) -> bytes:
    if d.prepopulate is None:
        raise ValueError("custom identity sets have no file representation")
    head = [_MAGIC, b"prepopulate=" + d.prepopulate.encode(), b"lmin=%d lmax=%d" % (d.l_min, d.l_max)]
    return b"\n".join(head + list(d.learned)) + b"\n"


def deserialize(data: bytes) -> Dictionary:
    rows = data.split(b"\n")
    if rows and rows[-1] == b"":
        rows.pop()
    if not rows or rows[0] != _MAGIC:
        if rows and rows[0][:3] == _MAGIC[:3]:
            raise UnsupportedVersion(f"unsupported version {rows[0]!r}")
        raise BadMagic("not a ZSD dictionary file")
    if len(rows) < 3:
        raise DictionaryFormatError("truncated header")
    if not rows[1].startswith(b"prepopulate="):
        raise DictionaryFormatError(f"bad prepopulate line {rows[1]!r}")
    mode = rows[1][len(b"prepopulate="):].decode("ascii", "replace")
    if mode not in PREPOPULATE_SETS:
        raise DictionaryFormatError(f"unknown prepopulate mode {mode!r}")
    fields = rows[2].split(b" ")
    if len(fields) != 2 or not fields[0].startswith(b"lmin=") or not fields[1].startswith(b"lmax="):
        raise DictionaryFormatError(f"bad bounds line {rows[2]!r}")
    try:
        l_min, l_max = int(fields[0][5:]), int(fields[1][5:])
    except ValueError:
        raise DictionaryFormatError(f"bad bounds line {rows[2]!r}") from None
    if not 2 <= l_min <= l_max <= MAX_PATTERN_LEN:
        raise DictionaryFormatError(f"bad length bounds [{l_min}, {l_max}]")
    patterns = rows[3:]
    if len(patterns) > MAX_PATTERNS:
        raise TooManyPatterns(f"{len(patterns)} patterns, max {MAX_PATTERNS}")
    seen = set()
    for p in patterns:
        if len(p) > l_max:
            raise PatternTooLong(f"pattern {p!r} longer than lmax={l_max}")
        if len(p) < l_min:
            raise DictionaryFormatError(f"pattern {p!r} shorter than lmin={l_min}")
        if not set(p) <= ALPHABET:
            raise NonAlphabetByteInPattern(f"pattern {p!r}")
        if p in seen:
            raise DictionaryFormatError(f"duplicate pattern {p!r}")
        seen.add(p)
    return Dictionary(patterns, mode, l_min=l_min, l_max=l_max)


def save_dictionary(d: Dictionary, path) -> None:
    with open(path, "wb") as fh:
        fh.write(serialize(d))


def load_dictionary(path) -> Dictionary:
    with open(path, "rb") as fh:
        return deserialize(fh.read())


def default_dictionary() -> Dictionary:
    """The embedded fixed dictionary (the reference's data/default.zsd,
    regenerated by its own trainer in tests/golden/make_golden.py)."""
    from importlib.resources import files
    return deserialize(files(__package__).joinpath("data/default.zsd").read_bytes())
