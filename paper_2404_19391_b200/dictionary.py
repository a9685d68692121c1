"""Fixed compression dictionary and the ZSD1 file format.

Mirrors the reference's ``Dictionary`` (dictionary.py:65-141), its code
assignment (identity byte -> itself, learned[i] -> 0x80+i), the table
builders the codec consumes (``encode_trie``: trie.py layout;
``decode_tables``: dictionary.py:112-129) and ZSD1 (de)serialization
(dictionary.py:322-383), and dictionary *training* on the GPU
(``GenerationParams``, ``RankTable``, ``count_substrings``,
``compute_overlap``, ``select_patterns``, ``generate``: dictionary.py:43-63,
143-320; kernels in csrc/zs_train.cuh) with the reference's results, tie
rule and working-set cap.
"""

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .errors import (
    BadMagic,
    DictionaryFormatError,
    EmptyCorpus,
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

# Candidates below this initial-rank cutoff stay out of the selection working
# set; a pick that does not beat the cutoff restarts with 4x the set
# (dictionary.py:38-43, 300-307).  Same name so tests can monkeypatch it.
_WORKING_SET_CAP = 200_000


@dataclass(frozen=True)
class GenerationParams:
    """Training knobs (dictionary.py:46-62)."""
    l_min: int = 2
    l_max: int = 8
    t: int = 128
    prepopulate: str = "smiles"
    preprocess: bool = False

    def __post_init__(self):
        if not 2 <= self.l_min <= self.l_max <= MAX_PATTERN_LEN:
            raise ValueError(
                f"need 2 <= l_min <= l_max <= {MAX_PATTERN_LEN}, "
                f"got l_min={self.l_min} l_max={self.l_max}")
        if not 0 <= self.t <= MAX_PATTERNS:
            raise ValueError(f"need 0 <= t <= {MAX_PATTERNS}, got {self.t}")
        if self.prepopulate not in PREPOPULATE_SETS:
            raise ValueError(f"unknown prepopulate mode {self.prepopulate!r}")


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
        """The reference's construction checks, first failing rule wins;
        the ValueError texts are part of the drop-in contract
        (dictionary.py:79-99, pinned by tests/test_serialize.py)."""
        lo, hi = self.l_min, self.l_max
        rules = [
            (lambda: 2 <= lo <= hi <= MAX_PATTERN_LEN, lambda: f"bad length bounds [{lo}, {hi}]"),
            (lambda: len(self.learned) <= MAX_PATTERNS,
             lambda: f"{len(self.learned)} learned patterns, max {MAX_PATTERNS}"),
            (lambda: len(set(self.learned)) == len(self.learned), lambda: "duplicate learned patterns"),
        ]
        for ok, msg in rules:
            if not ok():
                raise ValueError(msg())
        for p in self.learned:
            if not lo <= len(p) <= hi:
                raise ValueError(f"pattern {p!r} outside [{lo}, {hi}]")
            if not ALPHABET.issuperset(p):
                raise ValueError(f"pattern {p!r} has non-alphabet bytes")
        bad = sorted(b for b in self.identity if not 0x21 <= b <= 0x7E)
        if bad:
            raise ValueError(f"identity byte 0x{bad[0]:02x} not printable")

    @cached_property
    def code_of(self) -> dict:
        """pattern -> code: an identity byte is its own code, learned[i] is 0x80 + i."""
        return {**{bytes([b]): b for b in self.identity},
                **{p: 0x80 + i for i, p in enumerate(self.learned)}}

    @cached_property
    def encode_trie(self) -> PatternTrie:
        return build_trie(self)

    @cached_property
    def decode_tables(self):
        """(exp_len i32[256], valid u8[256], exp_off i64[257], exp_flat u8[]):
        the per-code expansion table the decoder takes (the reference's
        dictionary.py:112-129 layout), built as arrays over the code space."""
        ident = np.fromiter(sorted(self.identity), np.int64, len(self.identity))
        learned = 0x80 + np.arange(len(self.learned), dtype=np.int64)
        valid = np.zeros(256, np.uint8)
        valid[ident] = 1
        valid[learned] = 1
        exp_len = np.zeros(256, np.int32)
        exp_len[ident] = 1
        exp_len[learned] = [len(p) for p in self.learned]
        exp_off = np.concatenate([[0], np.cumsum(exp_len, dtype=np.int64)])
        exp_flat = np.zeros(int(exp_off[-1]), np.uint8)
        exp_flat[exp_off[ident]] = ident
        for code, p in zip(learned.tolist(), self.learned):
            exp_flat[exp_off[code]:exp_off[code + 1]] = np.frombuffer(p, np.uint8)
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


def _header(rows):
    """(prepopulate mode, l_min, l_max) from the three ZSD1 header rows; the
    exception types and texts are the reference's (dictionary.py:332-373)."""
    if not rows or rows[0] != _MAGIC:
        if rows and rows[0][:3] == _MAGIC[:3]:
            raise UnsupportedVersion(f"unsupported version {rows[0]!r}")
        raise BadMagic("not a ZSD dictionary file")
    if len(rows) < 3:
        raise DictionaryFormatError("truncated header")
    key, _, mode_b = rows[1].partition(b"=")
    if key != b"prepopulate" or not rows[1].startswith(b"prepopulate="):
        raise DictionaryFormatError(f"bad prepopulate line {rows[1]!r}")
    mode = mode_b.decode("ascii", "replace")
    if mode not in PREPOPULATE_SETS:
        raise DictionaryFormatError(f"unknown prepopulate mode {mode!r}")
    bounds = rows[2].split(b" ")
    try:
        if len(bounds) != 2 or bounds[0][:5] != b"lmin=" or bounds[1][:5] != b"lmax=":
            raise ValueError
        l_min, l_max = (int(f[5:]) for f in bounds)
    except ValueError:
        raise DictionaryFormatError(f"bad bounds line {rows[2]!r}") from None
    if not 2 <= l_min <= l_max <= MAX_PATTERN_LEN:
        raise DictionaryFormatError(f"bad length bounds [{l_min}, {l_max}]")
    return mode, l_min, l_max


def deserialize(data: bytes) -> Dictionary:
    """ZSD1 bytes -> Dictionary, with the reference's checks and messages."""
    rows = data.split(b"\n")
    if rows and rows[-1] == b"":
        del rows[-1]
    mode, l_min, l_max = _header(rows)
    patterns = rows[3:]
    if len(patterns) > MAX_PATTERNS:
        raise TooManyPatterns(f"{len(patterns)} patterns, max {MAX_PATTERNS}")
    seen = set()
    for p in patterns:
        problem = (PatternTooLong(f"pattern {p!r} longer than lmax={l_max}") if len(p) > l_max else
                   DictionaryFormatError(f"pattern {p!r} shorter than lmin={l_min}") if len(p) < l_min else
                   NonAlphabetByteInPattern(f"pattern {p!r}") if not ALPHABET.issuperset(p) else
                   DictionaryFormatError(f"duplicate pattern {p!r}") if p in seen else None)
        if problem is not None:
            raise problem
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


# ---------------------------------------------------------------------------
# training (GPU): dictionary.py:143-320
# ---------------------------------------------------------------------------

class RankTable:
    """Substring census (dictionary.py:143-166): rows of ``patterns``
    zero-padded to l_max, in the reference's order (length-major, bytewise
    ascending within a length); ``ranks`` = occurrences * length.  The rows
    also stay resident on the GPU that counted them (``_device``), so
    ``select_patterns`` runs without re-uploading."""

    def __init__(self, patterns, lengths, occurrences, ranks, _device=None):
        self.patterns = patterns
        self.lengths = lengths
        self.occurrences = occurrences
        self.ranks = ranks
        self._device = _device

    def __len__(self):
        return self.patterns.shape[0]

    def pattern(self, i: int) -> bytes:
        return self.patterns[i, :self.lengths[i]].tobytes()

    @property
    def entries(self) -> dict:
        return {self.pattern(i): (int(self.occurrences[i]), int(self.ranks[i]))
                for i in range(len(self))}


def _ctx():
    from . import _lib
    return _lib, _lib.context()


def count_substrings(corpus, params: GenerationParams) -> RankTable:
    """Exact occurrence counts of every alphabet-only substring with length in
    [l_min, l_max] (dictionary.py:169-221), counted on the GPU: one sort of
    the window starts by their first l_max bytes, then one boundary sweep per
    length (csrc/zs_train.cuh)."""
    lines = list(corpus)
    if not lines:
        raise EmptyCorpus("no training lines")
    joined = b"\n".join(lines)
    buf = np.frombuffer(joined or b"\0", np.uint8)
    _lib, ctx = _ctx()
    import ctypes
    m = ctypes.c_int64(0)
    with ctx.lock:
        ctx.check(ctx.lib.zs_train_count(ctx.h, _lib.ptr(buf), len(joined), params.l_min, params.l_max,
                                         ctypes.byref(m)), "zs_train_count")
        n = m.value
        pos = np.zeros(n, np.int64)
        lens = np.zeros(n, np.int32)
        occ = np.zeros(n, np.int64)
        ctx.check(ctx.lib.zs_train_rows(ctx.h, _lib.ptr(pos), _lib.ptr(lens), _lib.ptr(occ)), "zs_train_rows")
        ctx._train_gen = getattr(ctx, "_train_gen", 0) + 1
        token = (id(ctx), ctx._train_gen)
    width = params.l_max
    cols = np.arange(width, dtype=np.int64)
    patterns = buf[np.minimum(pos[:, None] + cols[None, :], buf.size - 1)] if n else \
        np.zeros((0, width), np.uint8)
    patterns = np.where(cols[None, :] < lens[:, None], patterns, 0).astype(np.uint8)
    lengths = lens.astype(np.int64)
    return RankTable(np.ascontiguousarray(patterns), lengths, occ, occ * lengths, _device=token)


def select_patterns(table: RankTable, t: int) -> list:
    """Repeated argmax of occurrences * (length - greedy overlap with the
    selected patterns), full overlap recomputation after every pick, ties to
    the longest then bytewise smallest pattern (dictionary.py:241-307) -- on
    the GPU, t picks without a host round trip."""
    import ctypes
    _lib, ctx = _ctx()
    out = np.zeros(max(t, 1), np.int64)
    k = ctypes.c_int32(0)
    with ctx.lock:
        if table._device != (id(ctx), getattr(ctx, "_train_gen", 0)):
            pats = np.ascontiguousarray(table.patterns, np.uint8)
            width = pats.shape[1] if pats.ndim == 2 and pats.shape[1] else 1
            if pats.shape[0] == 0:
                pats = np.zeros((0, width), np.uint8)
            ctx.check(ctx.lib.zs_train_load(ctx.h, _lib.ptr(pats), width,
                                            _lib.ptr(np.ascontiguousarray(table.lengths, np.int64)),
                                            _lib.ptr(np.ascontiguousarray(table.occurrences, np.int64)),
                                            len(table)), "zs_train_load")
            ctx._train_gen = getattr(ctx, "_train_gen", 0) + 1
            table._device = (id(ctx), ctx._train_gen)
        ctx.check(ctx.lib.zs_train_select(ctx.h, t, _WORKING_SET_CAP, _lib.ptr(out), ctypes.byref(k)),
                  "zs_train_select")
    return [table.pattern(int(i)) for i in out[:k.value]]


def compute_overlap(p: bytes, selected) -> int:
    """Bytes of p covered by a greedy longest-match parse against the
    selected patterns (dictionary.py:224-238), via kernels.overlap_batch."""
    from . import kernels
    sel = list(dict.fromkeys(bytes(s) for s in selected))
    if not sel or not p:
        return 0
    trie = PatternTrie.from_patterns([(s, 0) for s in sel])
    pats = np.zeros((1, max(len(p), 1)), np.uint8)
    pats[0, :len(p)] = np.frombuffer(bytes(p), np.uint8)
    out = np.empty(1, np.int64)
    kernels.overlap_batch(trie.children, trie.term_len, pats, np.array([len(p)], np.int64), out)
    return int(out[0])


def _preprocess_all(lines, mode):
    """[preprocess_line(l, mode) for l in lines] (dictionary.py:316-317) as
    one GPU batch: strict raises the first failing line's error; lenient
    keeps tokenize / pairing failures raw and raises RingIdOverflow."""
    from .errors import ERR_BRACKET, ERR_PERCENT, ERR_UNPAIRED, from_kind
    from .smiles import preprocess_batch
    if mode not in ("strict", "lenient"):
        raise ValueError(f"unknown mode {mode!r}")
    out = []
    for line, (kind, res) in zip(lines, preprocess_batch(lines)):
        if kind == 0:
            out.append(res)
        elif mode == "lenient" and kind in (ERR_BRACKET, ERR_PERCENT, ERR_UNPAIRED):
            out.append(bytes(line))
        else:
            off, ids = res
            raise from_kind(kind, off, ids)
    return out


def generate(corpus, params: GenerationParams, mode: str = "strict") -> Dictionary:
    """Train a dictionary on SMILES lines (dictionary.py:310-320), on the GPU."""
    lines = list(corpus)
    if not lines:
        raise EmptyCorpus("no training lines")
    if params.preprocess:
        lines = _preprocess_all(lines, mode)
    table = count_substrings(lines, params)
    learned = select_patterns(table, params.t)
    return Dictionary(learned, params.prepopulate, l_min=params.l_min, l_max=params.l_max)
