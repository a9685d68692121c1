"""Long lines (csrc/zs_ll.cuh): lines longer than compress_cx's staged window
are coded by the block-parallel long-line kernels.  Every case is checked
byte for byte against the oracle (the reference algorithm) and against the
general routine (one thread per line, zs_set_transducer bit 8), in both
renumbering modes, strict and lenient."""

import random

import numpy as np
import pytest

import oracle
import synth
from conftest import has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_2404_19391_b200 as z


@pytest.fixture(scope="module", autouse=True)
def _ready():
    if not has_gpu():
        pytest.skip("no GPU")
    oracle.build()
    synth.build()


def _long(mols, L, rng, sep=b"."):
    parts, n = [], 0
    while n < L:
        m = rng.choice(mols)
        parts.append(m)
        n += len(m) + 1
    return sep.join(parts)


def _soup(L, rng, width):
    """Overlapping rings, up to `width` open at once ('%nn' ids; colours >= 10)."""
    out, n, open_ = [], 0, []
    free = list(range(1, 100))
    while n < L:
        if open_ and (len(open_) >= width or rng.random() < 0.5):
            rid = open_.pop(rng.randrange(len(open_)))
            free.append(rid)
        else:
            rid = free.pop(rng.randrange(len(free)))
            open_.append(rid)
        t = b"C" + (b"%d" % rid if rid < 10 else b"%%%02d" % rid)
        out.append(t)
        n += len(t)
    out += [b"C" + (b"%d" % r if r < 10 else b"%%%02d" % r) for r in open_]
    return b"".join(out)


def _compare(payload, d, pre, lenient, mode):
    from paper_2404_19391_b200 import _lib as L
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    want, st = oracle.run_stream(t, payload, "compress", pre, lenient, 1)
    ctx = L.context()
    with ctx.lock:
        ctx.lib.zs_set_transducer(ctx.h, mode)
    try:
        got, res = z.run_buffer(payload, d, "compress", preprocess=pre, lenient=lenient)
    finally:
        with ctx.lock:
            ctx.lib.zs_set_transducer(ctx.h, 3)
    if st["err_line"]:
        assert res.err_line == st["err_line"]
        return
    assert got.tobytes() == want
    assert (res.lines, res.escapes, res.skipped, res.flagged) == \
        (st["lines"], st["escapes"], st["skipped"], st["flagged"])


def _cases():
    rng = random.Random(5)
    mols = synth.generate("mixed", 20000, 7).tobytes().split(b"\n")[:-1]
    short = b"\n".join(mols[:300]) + b"\n"
    out = {}
    for L in (2100, 9000, 70000, 600000):
        out[f"mixed_{L}"] = short + _long(mols, L, rng) + b"\n" + short
    out["soup_w14"] = short + _soup(120000, rng, 14) + b"\n" + short
    out["soup_w40"] = short + _soup(40000, rng, 40) + b"\n" + short
    out["soup_w101"] = short + _soup(20000, rng, 101) + b"\n" + short  # RingIdOverflow
    out["first_and_eof"] = _long(mols, 50000, rng) + b"\n" + short + _long(mols, 70000, rng)
    out["digits"] = short + b"C" + b"1" * 5000 + b"\n" + b"(" + b"12" * 3000 + b"\n" + short
    out["brackets"] = short + b"[" + b"C" * 3000 + b"]1CC1" + b"[NH4+]" * 900 + b"\n" + short
    out["pct_straddle"] = short + b"".join(b"C%%%02dCC%%%02d" % (10 + k % 80, 10 + k % 80)
                                           for k in range(3000)) + b"\n" + short
    out["cr"] = short + _long(mols, 9000, rng) + b"\r\n" + short
    out["unclosed_bracket"] = short + _long(mols, 9000, rng) + b"C[N\n" + short
    out["unpaired"] = short + _long(mols, 9000, rng) + b"C7\n" + short
    out["bad_percent"] = short + _long(mols, 9000, rng) + b"C%1\n" + short
    out["escapes"] = short + bytes(rng.randrange(33, 127) for _ in range(30000)).replace(b"\n", b"C") + \
        b"\n" + short
    out["many_long"] = b"".join(_long(mols, 3000 + 97 * k, rng) + b"\n" for k in range(120))
    return out


CASES = None


def _payload(name):
    global CASES
    if CASES is None:
        CASES = _cases()
    return CASES[name]


@pytest.mark.parametrize("name", ["mixed_2100", "mixed_9000", "mixed_70000", "mixed_600000", "soup_w14",
                                  "soup_w40", "soup_w101", "first_and_eof", "digits", "brackets",
                                  "pct_straddle", "cr", "unclosed_bracket", "unpaired", "bad_percent",
                                  "escapes", "many_long"])
def test_long_lines_vs_oracle(name):
    d = z.default_dictionary()
    payload = _payload(name)
    for pre in (False, True):
        for lenient in (True, False):
            _compare(payload, d, pre, lenient, 3)


@pytest.mark.parametrize("name", ["mixed_70000", "soup_w40", "many_long"])
def test_long_lines_general_routine_agrees(name):
    """The general routine (one thread per line) on the same payloads."""
    d = z.default_dictionary()
    payload = _payload(name)
    for pre in (False, True):
        _compare(payload, d, pre, True, 3 | 256)


def test_long_lines_fuzz():
    """Random long lines built from SMILES fragments that cross the 256-byte
    blocks in every way: brackets, '%nn' and digit ring ids, dots, escapes."""
    d = z.default_dictionary()
    rng = random.Random(11)
    frags = [b"C", b"c1ccccc1", b"[NH3+]", b"[C@@H]", b"%12", b"%47", b"1", b"2", b"(", b")", b".",
             b"=", b"#", b"O", b"Cl", b"Br", b"[13CH3]", b"~", b"*", b"%99", b"9"]
    lines = []
    for k in range(40):
        n = rng.choice((2100, 5000, 20000))
        lines.append(b"".join(rng.choice(frags) for _ in range(n // 3)))
    payload = b"\n".join(lines) + b"\n"
    for pre in (False, True):
        for lenient in (True, False):
            _compare(payload, d, pre, lenient, 3)


def test_long_line_device_api_and_decode_roundtrip():
    """A 4 MB line through the device API, and back through decompress."""
    import torch
    from paper_2404_19391_b200 import _lib as L
    d = z.default_dictionary()
    rng = random.Random(3)
    mols = synth.generate("mixed", 20000, 7).tobytes().split(b"\n")[:-1]
    payload = b"\n".join(mols[:1000]) + b"\n" + _long(mols, 4_000_000, rng) + b"\n" + \
        b"\n".join(mols[1000:2000]) + b"\n"
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    want, _ = oracle.run_stream(t, payload, "compress", True, True, 1)
    buf = np.frombuffer(payload, np.uint8)
    din = torch.from_numpy(buf.copy()).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    ctx = L.context()
    r = L.Result()
    with ctx.lock:
        ctx.set_dictionary(d)
        rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                        L.F_PREPROCESS | L.F_LENIENT, r)
        ctx.check(rc, "zs_compress_device")
    assert dout[:r.out_bytes].cpu().numpy().tobytes() == want
    back, _ = z.run_buffer(np.frombuffer(want, np.uint8), d, "decompress")
    want_back, _ = oracle.run_stream(t, want, "decompress", False, False, 1)
    assert back.tobytes() == want_back


def test_long_line_caps_fall_back():
    """More long lines than one launch records (32768) and more long-line
    bytes than it codes (256 MB): the rest take the general routine, in one
    device call, and the output is still the reference's."""
    import torch
    from paper_2404_19391_b200 import _lib as L
    d = z.default_dictionary()
    rng = random.Random(8)
    mols = synth.generate("mixed", 20000, 7).tobytes().split(b"\n")[:-1]
    bases = [_long(mols, 22600 + 37 * k, rng) for k in range(4)]  # > the staged window: always long
    payload = b"\n".join(bases[k % 4] for k in range(33000)) + b"\n"
    assert len(payload) > (256 << 20)
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    want, st = oracle.run_stream(t, payload, "compress", True, True, 16)
    buf = np.frombuffer(payload, np.uint8)
    din = torch.from_numpy(buf.copy()).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    ctx = L.context()
    r = L.Result()
    with ctx.lock:
        ctx.set_dictionary(d)
        rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(), dout.numel(),
                                        L.F_PREPROCESS | L.F_LENIENT, r)
        ctx.check(rc, "zs_compress_device")
    assert r.lines == 33000 and r.lines == st["lines"]
    assert dout[:r.out_bytes].cpu().numpy().tobytes() == want


def test_long_lines_through_run_stream_segments():
    """run_stream with segments much shorter than the long lines (the staging
    grows to hold a line) gives the oracle's stream and stats."""
    import io
    d = z.default_dictionary()
    rng = random.Random(12)
    mols = synth.generate("mixed", 20000, 7).tobytes().split(b"\n")[:-1]
    payload = b"".join(_long(mols, rng.choice((3000, 40000, 150000)), rng) + b"\n" + b"\n".join(mols[:50]) + b"\n"
                       for _ in range(6))
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    for pre in (False, True):
        want, st = oracle.run_stream(t, payload, "compress", pre, True, 1)
        dst = io.BytesIO()
        res = z.run_stream(io.BytesIO(payload), dst, d, "compress", preprocess=pre, lenient=True,
                           segment_bytes=8192)
        assert dst.getvalue() == want
        assert (res.lines, res.escapes) == (st["lines"], st["escapes"])


def test_long_lines_in_later_host_chunks():
    """A buffer of several 64 MB host-API chunks with long lines in the later
    ones: the chunk pipeline re-runs just those chunks with the long-line
    kernels (their slots' own buffers), output bit-exact."""
    d = z.default_dictionary()
    rng = random.Random(13)
    mols = synth.generate("mixed", 20000, 7).tobytes().split(b"\n")[:-1]
    base = synth.generate("aromatic", 1_600_000, 2024).tobytes()  # ~74 MB
    lines = base.split(b"\n")[:-1]
    for at in (1_000_000, 1_300_000, 1_599_000):
        lines[at] = _long(mols, rng.choice((9000, 60000, 400000)), rng)
    payload = b"\n".join(lines) + b"\n"
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    want, st = oracle.run_stream(t, payload, "compress", True, True, 16)
    got, res = z.run_buffer(np.frombuffer(payload, np.uint8), d, "compress", preprocess=True, lenient=True)
    assert got.tobytes() == want
    assert (res.lines, res.escapes) == (st["lines"], st["escapes"])
