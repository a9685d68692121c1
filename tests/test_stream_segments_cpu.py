"""run_stream's segment framing (host logic) on CPU: the per-segment GPU
call is replaced by the CPU oracle, and reading the input in small
newline-cut segments must give the same bytes, stats and errors (and the
reference's strict partial output) as one whole-buffer call."""

import io

import numpy as np
import pytest

import oracle
import paper_2404_19391_b200 as z
from paper_2404_19391_b200 import pipeline


class _Res:
    def __init__(self, st):
        self.lines = st["lines"]
        self.escapes = st["escapes"]
        self.skipped = st["skipped"]
        self.flagged = st["flagged"]
        self.out_bytes = st["out_bytes"]
        self.err_line = st["err_line"]
        self.err_kind = st["err_kind"]
        self.err_offset = st["err_offset"]
        self.err_code = st["err_code"]
        ids = [0, 0]
        for i in st["err_ids"]:
            ids[i >> 6] |= 1 << (i & 63)
        self.err_ids = ids


def _oracle_run_buffer(buf, d, direction="compress", *, preprocess=False, lenient=False, device=None, out=None):
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    data = bytes(buf) if not isinstance(buf, (bytes, bytearray)) else bytes(buf)
    out, st = oracle.run_stream(t, data, direction, preprocess, lenient, 1)
    return np.frombuffer(out or b"", np.uint8), _Res(st)


@pytest.fixture(autouse=True)
def _cpu_codec(monkeypatch):
    oracle.build()
    monkeypatch.setattr(pipeline, "run_buffer", _oracle_run_buffer)
    # host staging without a GPU (page-locked memory needs the CUDA runtime)
    monkeypatch.setattr(pipeline, "_host_buffer", lambda slot, n, device: np.empty(max(int(n), 1), np.uint8))


def _dict(dj):
    learned = [bytes.fromhex(p) for p in dj["learned"]]
    if dj["prepopulate"] is not None:
        return z.Dictionary(learned, dj["prepopulate"], l_min=dj["l_min"], l_max=dj["l_max"])
    return z.Dictionary(learned, None, l_min=dj["l_min"], l_max=dj["l_max"], identity=bytes.fromhex(dj["identity"]))


@pytest.mark.parametrize("seg", [1, 7, 64, 1 << 20])
def test_segments_match_reference_stream(stream_cases, seg):
    dicts = [_dict(dj) for dj in stream_cases["dicts"]]
    for c in stream_cases["cases"][:250]:
        kw = dict(preprocess=c["preprocess"], lenient=c["lenient"])
        payload = bytes.fromhex(c["payload"])
        if "err" in c:
            with pytest.raises(z.LineError) as ei:
                z.run_stream(io.BytesIO(payload), io.BytesIO(), dicts[c["dict"]], c["direction"],
                             segment_bytes=seg, **kw)
            assert ei.value.line_no == c["line_no"] and str(ei.value) == c["msg"]
        else:
            dst = io.BytesIO()
            st = z.run_stream(io.BytesIO(payload), dst, dicts[c["dict"]], c["direction"], segment_bytes=seg, **kw)
            assert dst.getvalue().hex() == c["out"], (seg, c)
            assert (st.lines, st.input_bytes, st.output_bytes, st.escapes, st.skipped, st.flagged) == \
                (c["lines"], c["in_bytes"], c["out_bytes"], c["escapes"], c["skipped"], c["flagged"])


def test_strict_partial_output_any_segment():
    d = z.Dictionary([], "smiles")
    lines = [b"CCO"] * 300 + [b"C1CC"] + [b"CCO"] * 50
    for seg in (1, 3, 40, 100, 1000, 1 << 20):
        for bl in (1, 7, 32, 300, 301, 1000):
            dst = io.BytesIO()
            with pytest.raises(z.LineError) as ei:
                z.run_stream(io.BytesIO(b"\n".join(lines) + b"\n"), dst, d, "compress", preprocess=True,
                             batch_lines=bl, segment_bytes=seg)
            assert ei.value.line_no == 301
            assert dst.getvalue() == b"\n".join([b"CCO"] * ((300 // bl) * bl)), (seg, bl)


def test_framing_edge_cases():
    """Empty input, lone newlines, no trailing newline, dropped final lines."""
    d = z.Dictionary([b"CC"], "smiles")
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    for payload in (b"", b"\n", b"\n\n", b"CC", b"CC\n", b"CC\nC\r", b"C\r\nCC", b"CC\n\r\n", b"\r", b"\r\n\r\n",
                    b"CC\nCC\r\n\r", b"C" * 50 + b"\n" + b"CC\r"):
        for seg in (1, 2, 3, 5, 100):
            want, st = oracle.run_stream(t, payload, "compress", False, True, 1)
            dst = io.BytesIO()
            got = z.run_stream(io.BytesIO(payload), dst, d, "compress", lenient=True, segment_bytes=seg)
            assert dst.getvalue() == (want or b""), (payload, seg)
            assert (got.lines, got.output_bytes, got.skipped) == (st["lines"], st["out_bytes"], st["skipped"])


def test_newline_helpers_against_naive():
    """pipeline._last_nl / _cut_keeping_last (block-wise scans used by the
    streaming path) against plain Python on random buffers."""
    rng = np.random.default_rng(5)
    for n in (0, 1, 5, 100, 3000, (1 << 20) + 777):
        arr = rng.choice(np.frombuffer(b"ab\n", np.uint8), size=n, p=[0.45, 0.45, 0.10]).astype(np.uint8)
        raw = arr.tobytes()
        for lo, hi in ((0, n), (n // 3, n), (0, n // 2)):
            want = raw.rfind(b"\n", lo, hi)
            assert pipeline._last_nl(arr, lo, hi) == want
        if raw.endswith(b"\n"):
            nls = [i for i, b in enumerate(raw) if b == 10] if n < 5000 else list(np.flatnonzero(arr == 10))
            for m in (0, 1, 2, len(nls) - 1, len(nls)):
                if m < 0 or m > len(nls):
                    continue
                want = 0 if m >= len(nls) else int(nls[len(nls) - m - 1]) + 1
                assert pipeline._cut_keeping_last(arr, n, m) == want, (n, m)
