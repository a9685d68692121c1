"""GPU parity: the sm_100a path vs the reference's own outputs (golden
fixtures) and vs the CPU oracle, through the C ABI.  Bit-exact throughout."""

import hashlib
import io
import random

import numpy as np
import pytest

import oracle
import synth
from conftest import golden_dict_bytes, has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_2404_19391_b200 as z
    from paper_2404_19391_b200 import _lib, kernels


def dict_from_json(dj):
    learned = [bytes.fromhex(p) for p in dj["learned"]]
    ident = bytes.fromhex(dj["identity"])
    if dj["prepopulate"] is not None:
        return z.Dictionary(learned, dj["prepopulate"], l_min=dj["l_min"], l_max=dj["l_max"])
    return z.Dictionary(learned, None, l_min=dj["l_min"], l_max=dj["l_max"], identity=ident)


@pytest.fixture(scope="module", autouse=True)
def _ready():
    if not has_gpu():
        pytest.skip("no GPU")
    oracle.build()
    synth.build()


# ---------------------------------------------------------------- shim paths

def test_compress_lines_golden(codec_cases):
    for c in codec_cases:
        d = dict_from_json(c["dict"])
        recs, esc = z.compress_lines(d, [bytes.fromhex(l) for l in c["lines"]])
        assert [r.hex() for r in recs] == c["records"]
        assert esc == c["escapes"]


def test_kernel_seam_harness_golden(codec_cases, decode_cases):
    """The reference's kernel harness shape (test_kernels.py:18-48) against
    kernels.compress_batch / decompress_sizes / decompress_fill."""
    for c in codec_cases[:12]:
        d = dict_from_json(c["dict"])
        lines = [bytes.fromhex(l) for l in c["lines"]]
        flat = np.frombuffer(b"".join(lines) or b"\0", np.uint8)
        starts = np.zeros(len(lines) + 1, np.int64)
        np.cumsum([len(l) for l in lines], out=starts[1:])
        out = np.zeros(2 * int(starts[-1]) + 1, np.uint8)
        lens = np.empty(len(lines), np.int64)
        esc = kernels.compress_batch(d.encode_trie.children, d.encode_trie.term_code, flat, starts,
                                     out, lens)
        recs = [out[2 * starts[i]:2 * starts[i] + lens[i]].tobytes().hex() for i in range(len(lines))]
        assert recs == c["records"] and esc == c["escapes"]
    for c in decode_cases:
        d = dict_from_json(c["dict"])
        recs = [bytes.fromhex(r) for r in c["records"]]
        exp_len, valid, exp_off, exp_flat = d.decode_tables
        flat = np.frombuffer(b"".join(recs) or b"\0", np.uint8)
        starts = np.zeros(len(recs) + 1, np.int64)
        np.cumsum([len(r) for r in recs], out=starts[1:])
        n = len(recs)
        lens, st, ep = np.empty(n, np.int64), np.empty(n, np.int8), np.empty(n, np.int64)
        total, esc = kernels.decompress_sizes(exp_len, valid, flat, starts, lens, st, ep)
        assert lens.tolist() == c["out_lens"] and st.tolist() == c["status"]
        assert ep.tolist() == c["errpos"] and (total, esc) == (c["total"], c["escapes"])
        ost = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=ost[1:])
        out = np.zeros(total + 1, np.uint8)
        kernels.decompress_fill(exp_off, exp_flat, flat, starts, st, out, ost)
        assert out[:total].tobytes().hex() == c["out"]


def test_decompress_lines_golden(decode_cases):
    for c in decode_cases:
        d = dict_from_json(c["dict"])
        recs = [bytes.fromhex(r) for r in c["records"]]
        lines, errors, esc = z.decompress_lines(d, recs)
        assert esc == c["escapes"]
        got = b"".join(l for l in lines if l is not None)
        assert got.hex() == c["out"]
        bad = {i for i, s in enumerate(c["status"]) if s}
        assert {i for i, _ in errors} == bad
        for i, e in errors:
            want = z.UnknownCode if c["status"][i] == 1 else z.TruncatedEscape
            assert isinstance(e, want) and e.offset == c["errpos"][i]


def test_decode_error_kats():
    d = z.Dictionary([b"CC"], "none")
    with pytest.raises(z.UnknownCode) as ei:
        z.decompress_line(d, bytes([0x80, 0x99]))
    assert (ei.value.code, ei.value.offset) == (0x99, 1)
    with pytest.raises(z.TruncatedEscape) as ei:
        z.decompress_line(z.Dictionary([], "smiles"), bytes([ord("C"), 0x20]))
    assert ei.value.offset == 1
    assert z.compress_line(z.Dictionary([b"CC", b"CCC"], None, identity=b"C"), b"CCCC") == \
        bytes([0x81, ord("C")])


def test_preprocess_golden(preprocess_cases):
    lines = [bytes.fromhex(c["line"]) for c in preprocess_cases]
    res = z.preprocess_batch(lines)
    for c, line, (kind, val) in zip(preprocess_cases, lines, res):
        s = c["strict"]
        if kind == 0:
            assert s.get("out") == val.hex(), c
        else:
            e = z.errors.from_kind(kind, val[0], val[1])
            assert (type(e).__name__, str(e)) == (s["err"], s["msg"]), c
    for c in preprocess_cases[::7]:
        line = bytes.fromhex(c["line"])
        for mode in ("strict", "lenient"):
            want = c[mode]
            try:
                got = {"out": z.preprocess_line(line, mode).hex()}
            except z.ZsmilesError as e:
                got = {"err": type(e).__name__, "msg": str(e)}
            assert got == want, (line, mode)


# ---------------------------------------------------------------- whole-buffer path

def test_run_stream_golden(stream_cases):
    dicts = [dict_from_json(dj) for dj in stream_cases["dicts"]]
    for c in stream_cases["cases"]:
        dst = io.BytesIO()
        kw = dict(preprocess=c["preprocess"], lenient=c["lenient"])
        if "err" in c:
            with pytest.raises(z.LineError) as ei:
                z.run_stream(io.BytesIO(bytes.fromhex(c["payload"])), dst, dicts[c["dict"]],
                             c["direction"], **kw)
            assert ei.value.line_no == c["line_no"]
            assert type(ei.value.cause).__name__ == c["cause"]
            assert str(ei.value) == c["msg"]
        else:
            st = z.run_stream(io.BytesIO(bytes.fromhex(c["payload"])), dst, dicts[c["dict"]],
                              c["direction"], **kw)
            assert dst.getvalue().hex() == c["out"], c
            assert (st.lines, st.input_bytes, st.output_bytes, st.escapes, st.skipped,
                    st.flagged) == (c["lines"], c["in_bytes"], c["out_bytes"], c["escapes"],
                                    c["skipped"], c["flagged"])


def test_whole_buffer_random_dictionaries(codec_cases):
    """Fused tile kernels (fast DFA and generic trie) vs the oracle stream on
    the golden random dictionaries, with escape-heavy bytes."""
    rng = random.Random(5)
    n_fast = 0
    for c in codec_cases:
        d = dict_from_json(c["dict"])
        lines = [bytes.fromhex(l) for l in c["lines"]]
        lines = [l.replace(b"\n", b"").replace(b"\r", b"") for l in lines]
        rng.shuffle(lines)
        payload = b"\n".join(lines * 3) + b"\n"
        t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
        for pre in (False, True):
            comp, res = z.run_buffer(payload, d, "compress", preprocess=pre, lenient=True)
            want, st = oracle.run_stream(t, payload, "compress", pre, True, 1)
            assert comp.tobytes() == want
            assert (res.lines, res.escapes, res.flagged) == (st["lines"], st["escapes"], st["flagged"])
            back, _ = z.run_buffer(want, d, "decompress", lenient=True)
            want_back, _ = oracle.run_stream(t, want, "decompress", False, True, 1)
            assert back.tobytes() == want_back
        n_fast += _lib.context().fast_width() > 0
    assert n_fast >= 10


@pytest.mark.parametrize("name", ["aromatic_10k", "aliphatic_10k", "mixed_50k", "c1_100k",
                                  "c3_skewed_20k"])
def test_corpus_hashes(corpus_hashes, name):
    e = corpus_hashes[name]
    buf = synth.generate(e["kind"], e["lines"], e["seed"])
    d = z.deserialize(golden_dict_bytes(e["dict"]))
    for key, pre in (("pre_off", False), ("pre_on", True)):
        comp, res = z.run_buffer(buf, d, "compress", preprocess=pre, lenient=True)
        assert hashlib.sha256(comp.tobytes()).hexdigest() == e[key]["comp_sha256"]
        assert res.out_bytes == e[key]["out_bytes"] and res.escapes == e[key]["escapes"]
        back, _ = z.run_buffer(comp, d, "decompress")
        assert hashlib.sha256(back.tobytes()).hexdigest() == e[key]["roundtrip_sha256"]


def test_ablation_dictionaries(corpus_hashes):
    e0 = corpus_hashes["c1_100k"]
    buf = synth.generate(e0["kind"], e0["lines"], e0["seed"])
    for name, e in corpus_hashes.items():
        if not name.startswith("c4_"):
            continue
        d = z.deserialize(golden_dict_bytes(e["dict"]))
        for key, pre in (("pre_off", False), ("pre_on", True)):
            comp, _ = z.run_buffer(buf, d, "compress", preprocess=pre, lenient=True)
            assert hashlib.sha256(comp.tobytes()).hexdigest() == e[key]["comp_sha256"], (name, key)
            back, _ = z.run_buffer(comp, d, "decompress")
            assert hashlib.sha256(back.tobytes()).hexdigest() == e[key]["roundtrip_sha256"]


@pytest.mark.parametrize("name", ["c2_10m", "c3_skewed_1m", "c3_skewed_5m"])
def test_full_size_hashes(corpus_hashes, name):
    """BASELINE configs at full size (C2: 10M lines; C3: the 5M-line skewed
    library, 2.7 GB, and its first 1M lines), host API (multi-chunk pipeline)
    and device API, against the reference's own output hashes."""
    import torch
    if name not in corpus_hashes:
        pytest.skip(f"{name}: golden not generated (tests/golden/make_golden.py --c3-5m)")
    e = corpus_hashes[name]
    buf = synth.generate(e["kind"], e["lines"], e["seed"])
    d = z.default_dictionary()
    for key, pre in (("pre_off", False), ("pre_on", True)):
        comp, res = z.run_buffer(buf, d, "compress", preprocess=pre, lenient=True)
        assert hashlib.sha256(comp.tobytes()).hexdigest() == e[key]["comp_sha256"], key
        back, _ = z.run_buffer(comp, d, "decompress")
        assert hashlib.sha256(back.tobytes()).hexdigest() == e[key]["roundtrip_sha256"], key
    # device API on HBM-resident buffers
    ctx = _lib.context()
    din = torch.from_numpy(buf).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    r = _lib.Result()
    with ctx.lock:
        ctx.set_dictionary(d)
        rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(),
                                        dout.numel(), _lib.F_PREPROCESS | _lib.F_LENIENT, r)
        ctx.check(rc, "zs_compress_device")
    got = dout[:r.out_bytes].cpu().numpy().tobytes()
    assert hashlib.sha256(got).hexdigest() == e["pre_on"]["comp_sha256"]


# ---------------------------------------------------------------- edge cases

def _oracle_check(payload, d, pre, lenient, direction="compress"):
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    want, st = oracle.run_stream(t, payload, direction, pre, lenient, 1)
    if st["err_line"]:
        with pytest.raises(z.LineError) as ei:
            z.run_stream(io.BytesIO(payload), io.BytesIO(), d, direction, preprocess=pre,
                         lenient=lenient)
        assert ei.value.line_no == st["err_line"]
        return None
    got, res = z.run_buffer(payload, d, direction, preprocess=pre, lenient=lenient)
    assert got.tobytes() == want
    assert (res.lines, res.escapes, res.skipped, res.flagged) == \
        (st["lines"], st["escapes"], st["skipped"], st["flagged"])
    return want


def test_long_lines_global_path():
    """Lines longer than the smem window take the HBM-arena path."""
    d = z.default_dictionary()
    rng = random.Random(9)
    mols = synth.generate("mixed", 20000, 7).tobytes().split(b"\n")[:-1]
    for L in (3000, 5000, 40000, 300000):
        parts, n = [], 0
        while n < L:
            m = rng.choice(mols)
            parts.append(m)
            n += len(m) + 1
        long_line = b"C".join(parts)
        payload = b"\n".join(mols[:300]) + b"\n" + long_line + b"\n" + b"\n".join(mols[300:600]) + b"\n"
        for pre in (False, True):
            _oracle_check(payload, d, pre, True)
        back_in = _oracle_check(payload, d, True, False)
        if back_in is not None:
            _oracle_check(back_in, d, False, False, "decompress")


def test_growing_renumbering_line():
    """A 1-byte ring id that must take a colour >= 10 grows the line."""
    d = z.default_dictionary()
    ids = [str(i) for i in range(1, 10)] + [f"%{i:02d}" for i in range(10, 25)]
    grow = ("C" + "C".join(ids[::-1]) + "C" + "C".join(ids) + "C").encode()
    grow2 = ("C1" + "".join(f"C%{i:02d}" for i in range(10, 22)) + "C" +
             "".join(f"C%{i:02d}" for i in range(21, 9, -1)) + "C1").encode()
    payload = b"CCO\n" + grow + b"\n" + grow2 + b"\nc1ccccc1\n" + grow2
    for lenient in (False, True):
        _oracle_check(payload, d, True, lenient)


def test_many_tiny_lines_multiple_rounds():
    d = z.Dictionary([b"CC"], "smiles")
    payload = b"\n" * 70000 + b"C\n" * 30000 + b"CC\nC\n" * 20000
    for pre in (False, True):
        want = _oracle_check(payload, d, pre, False)
        _oracle_check(want, d, False, False, "decompress")


def test_errors_across_tiles():
    d = z.default_dictionary()
    base = synth.generate("aromatic", 30000, 11).tobytes().split(b"\n")[:-1]
    for bad_at, bad in ((0, b"C1CC"), (777, b"C[NH"), (20000, b"CC\rO"), (29999, b"C%1")):
        lines = list(base)
        lines[bad_at] = bad
        payload = b"\n".join(lines) + b"\n"
        for lenient in (False, True):
            _oracle_check(payload, d, True, lenient)
            _oracle_check(payload, d, False, lenient)
    comp, _ = z.run_buffer(b"\n".join(base) + b"\n", d, "compress")
    recs = comp.tobytes().split(b"\n")
    recs[12345] = b"\x05\x80"
    recs[23456] = b"CC "
    _oracle_check(b"\n".join(recs), d, False, True, "decompress")
    _oracle_check(b"\n".join(recs), d, False, False, "decompress")


def test_long_line_tiles_edge_cases():
    """Tiles of long lines run the byte-exact tokenizer / parse slices
    (speculative entries, neighbour checks, re-walks) and fall back to the
    per-line tokenizer on a CR or tokenize error: errors, '%nn' ids, colour
    overflow, unpaired rings and escaped bytes inside long lines."""
    d = z.default_dictionary()
    base = synth.generate("skewed", 12000, 2025).tobytes().split(b"\n")[:-1]
    rng = random.Random(77)
    nest = b"C1C2C3C4C5CCCCC5C4C3C2C1"                  # 5 nested rings: colour 4
    pct = b"C%12CC%34CC%34CC%12"
    edits = [b"CC\rO", b"C[NH", b"C%1C", b"C1CC", nest, pct, b"C\tC", b"c1cc\xffcc1"]
    for k, bad in enumerate(edits):
        lines = list(base)
        for _ in range(3):
            i = rng.randrange(len(lines))
            j = rng.randrange(len(lines[i]) + 1)
            lines[i] = lines[i][:j] + bad + lines[i][j:]
        payload = b"\n".join(lines) + (b"\n" if k % 2 == 0 else b"")
        for lenient in (False, True):
            _oracle_check(payload, d, True, lenient)
        _oracle_check(payload, d, False, True)
    # the key-window parse (patterns of 9-15 bytes) on long-line tiles
    dk = z.deserialize(golden_dict_bytes("t128_l15.zsd"))
    payload = b"\n".join(base[:4000]) + b"\n"
    for lenient in (False, True):
        _oracle_check(payload, dk, True, lenient)
    _oracle_check(payload, dk, False, True)
    # long lines without any newline for many slices, and one-line tiles
    mols = [m for m in base if len(m) > 100][:40]
    payload = b"\n".join(b"C".join(mols[i:i + 8]) for i in range(0, 40, 8)) + b"\n"
    for pre in (False, True):
        want = _oracle_check(payload, d, pre, True)
        _oracle_check(want, d, False, True, "decompress")


def test_strict_partial_output_matches_reference_batches():
    d = z.Dictionary([], "smiles")
    lines = [b"CCO"] * 300 + [b"C1CC"] + [b"CCO"] * 50
    dst = io.BytesIO()
    with pytest.raises(z.LineError) as ei:
        z.run_stream(io.BytesIO(b"\n".join(lines) + b"\n"), dst, d, "compress",
                     preprocess=True, batch_lines=32)
    assert ei.value.line_no == 301
    assert dst.getvalue() == b"\n".join([b"CCO"] * 288)


def test_device_and_host_api_agree():
    import torch
    d = z.default_dictionary()
    buf = synth.generate("mixed", 200000, 3)
    comp, res = z.run_buffer(buf, d, "compress", preprocess=True)
    ctx = _lib.context()
    din = torch.from_numpy(buf).cuda()
    dout = torch.empty(2 * buf.size + 64, dtype=torch.uint8, device="cuda")
    r = _lib.Result()
    with ctx.lock:
        ctx.set_dictionary(d)
        rc = ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), buf.size, dout.data_ptr(),
                                        dout.numel(), _lib.F_PREPROCESS, r)
        ctx.check(rc, "zs_compress_device")
        assert ctx.last_kernel_ms() > 0
    assert dout[:r.out_bytes].cpu().numpy().tobytes() == comp.tobytes()
    assert (r.lines, r.out_bytes) == (res.lines, res.out_bytes)


@pytest.mark.parametrize("mode", [0, 1, 3, 19, 67, 83, 131])
def test_kernel_variants_bit_exact(corpus_hashes, mode):
    """Every compress kernel variant gives the reference bytes, both
    directions (include/zs_debug.h): 0 the generic key-window DP with a
    decision array, 1 + the cost-window transducer, 3 compress_cx with the
    product-automaton parse (the default), 19 without the byte-exact slices
    of long-line tiles, 67 compress_cx with the DFA + transducer parse,
    83 both, 131 compress_cx with every phase on byte-exact slices."""
    ctx = _lib.context()
    try:
        ctx.lib.zs_set_transducer(ctx.h, mode)
        for name in ("c1_100k", "c3_skewed_20k", "mixed_50k"):
            e = corpus_hashes[name]
            buf = synth.generate(e["kind"], e["lines"], e["seed"])
            d = z.deserialize(golden_dict_bytes(e["dict"]))
            for key, pre in (("pre_off", False), ("pre_on", True)):
                comp, res = z.run_buffer(buf, d, "compress", preprocess=pre, lenient=True)
                assert hashlib.sha256(comp.tobytes()).hexdigest() == e[key]["comp_sha256"], (name, key)
                back, _ = z.run_buffer(comp, d, "decompress")
                assert hashlib.sha256(back.tobytes()).hexdigest() == e[key]["roundtrip_sha256"]
        test_long_lines_global_path()
        test_growing_renumbering_line()
        test_many_tiny_lines_multiple_rounds()
        test_errors_across_tiles()
    finally:
        ctx.lib.zs_set_transducer(ctx.h, 3)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gpu_codec(world):
    """The multi-GPU shard protocol with the GPU codec per shard (all ranks
    simulated on cuda:0) == the whole-buffer oracle stream."""
    from paper_2404_19391_b200 import shard
    t = oracle.Tables.from_zsd(golden_dict_bytes())
    d = z.default_dictionary()
    buf = synth.generate("skewed", 20000, 2025).tobytes()[:-1]
    want, st = oracle.run_stream(t, buf, "compress", True, True, 8)
    arr = np.frombuffer(buf, np.uint8)
    cuts = shard.shard_bounds(arr, world)
    fn = shard.gpu_codec(d, "compress", preprocess=True, lenient=True)
    outs = [fn(arr[cuts[r]:cuts[r + 1]]) for r in range(world)]
    res = [o[1] for o in outs]
    blob = b""
    for r in range(world):
        v = shard.combine(res, r, False)
        assert v.out_offset == len(blob)
        blob += outs[r][0][:v.out_bytes]
    assert blob == want and v.total_lines == st["lines"]


@pytest.mark.parametrize("mode", [3, 19, 67, 131])
def test_fuzz_regressions(mode):
    """Inputs the randomised GPU sweep (tools/fuzz_gpu.py) once broke, shrunk
    (tools/fuzz_bisect.py) and pinned against the oracle in every kernel mode
    (tests/golden/fuzz_cases.json.gz)."""
    import gzip
    import json
    import os
    from conftest import ROOT
    with gzip.open(os.path.join(ROOT, "tests", "golden", "fuzz_cases.json.gz"), "rt") as fh:
        cases = json.load(fh)["cases"]
    ctx = _lib.context()
    try:
        ctx.lib.zs_set_transducer(ctx.h, mode)
        for c in cases:
            d = z.Dictionary([bytes.fromhex(p) for p in c["learned"]], None, l_min=c["l_min"], l_max=c["l_max"],
                             identity=bytes.fromhex(c["identity"]))
            payload = bytes.fromhex(c["payload"])
            _oracle_check(payload, d, c["pre"], c["lenient"])
    finally:
        ctx.lib.zs_set_transducer(ctx.h, 3)


def test_parse_optimal_vs_brute_force():
    """The GPU parse is a minimum-cost parse (reference test_codec.py:57-69):
    payload length == codec.oracle_parse_cost (exhaustive recursion, no trie,
    no DP) on short lines over random dictionaries, escape bytes included."""
    from paper_2404_19391_b200.codec import oracle_parse_cost
    rng = random.Random(91)
    for _ in range(40):
        pats = {bytes(rng.choice(b"CcN1(=O") for _ in range(rng.randint(2, 5))) for _ in range(rng.randint(0, 12))}
        d = z.Dictionary(sorted(pats), "smiles", l_min=2, l_max=5)
        lines = [bytes(rng.choice(b"CcN1(=O \tx") for _ in range(rng.randint(0, 16))) for _ in range(25)]
        recs, _ = z.compress_lines(d, lines)
        assert [len(r) for r in recs] == [oracle_parse_cost(d, ln) for ln in lines]


def test_random_access_vs_oracle():
    """RecordIndex against the CPU oracle's restatement of the reference
    decoder (numba_impl.py:74-139 via oracle.decompress_batch): every
    requested record's bytes, and for bad records the reference's
    UnknownCode(code, offset) / TruncatedEscape(offset), with escape-heavy
    records from a random dictionary and records with unknown codes and
    dangling escapes mixed in."""
    rng = random.Random(77)
    d = z.Dictionary([b"CC", b"c1", b"ccc", b"(=O)"], "smiles")
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    lines = [bytes(rng.choice(b"Cc1()=O \t\xff") for _ in range(rng.randrange(0, 50))) for _ in range(4000)]
    recs, _ = oracle.compress_batch(t, lines)
    for k in rng.sample(range(len(recs)), 60):  # corrupt some records
        kind = rng.randrange(3)
        if kind == 0:
            recs[k] = recs[k] + b" "              # dangling escape
        elif kind == 1:
            recs[k] = recs[k][:1] + b"\x9f" + recs[k][1:]  # unknown code
        else:
            recs[k] = b""
    ref = oracle.decompress_batch(t, recs)
    starts = np.concatenate([[0], np.cumsum(ref["out_lens"])])
    ix = z.RecordIndex(b"\n".join(recs) + b"\n", d)
    assert len(ix) == len(recs)
    good = [i for i in range(len(recs)) if ref["status"][i] == 0]
    sel = [rng.choice(good) for _ in range(3000)]
    got = ix.decode(sel)
    assert got == [ref["out"][starts[i]:starts[i + 1]] for i in sel]
    data, off = ix.decode_packed(sel)
    assert [data[a:b].tobytes() for a, b in zip(off[:-1], off[1:])] == got
    for i in range(len(recs)):
        st = int(ref["status"][i])
        if st == 0:
            continue
        ep = int(ref["errpos"][i])
        if st == 1:
            with pytest.raises(z.UnknownCode) as e:
                ix.decode([good[0], i])
            assert (e.value.code, e.value.offset) == (recs[i][ep], ep)
        else:
            with pytest.raises(z.TruncatedEscape) as e:
                ix.decode([i])
            assert e.value.offset == ep


def test_run_library_two_contexts(corpus_hashes):
    """The single-process multi-GPU API (shard.run_library) with two real
    contexts on one device (one shard each, run concurrently) reproduces the
    reference's own C1 output and round trip (golden hashes)."""
    from paper_2404_19391_b200 import shard
    e = corpus_hashes["c1_100k"]
    buf = synth.generate(e["kind"], e["lines"], e["seed"])
    d = z.deserialize(golden_dict_bytes(e["dict"]))
    ctxs = [_lib.Context(0), _lib.Context(0)]
    try:
        for world in (2, 3):
            devs = [ctxs[r % 2] for r in range(world)]
            comp, v, res = shard.run_library(buf, d, "compress", preprocess=True, lenient=True, devices=devs)
            assert hashlib.sha256(comp.tobytes()).hexdigest() == e["pre_on"]["comp_sha256"]
            assert v.total_lines == e["lines"] and v.total_out == comp.size and v.err_line == 0
            back, _, _ = shard.run_library(comp, d, "decompress", devices=devs)
            assert hashlib.sha256(back.tobytes()).hexdigest() == e["pre_on"]["roundtrip_sha256"]
        # a strict error in the second shard: global 1-based line number
        lines = buf.tobytes().split(b"\n")
        lines[70000] = b"C1CC[N"
        bad = np.frombuffer(b"\n".join(lines), np.uint8)
        _, v, _ = shard.run_library(bad, d, "compress", preprocess=True, lenient=False, devices=ctxs)
        assert v.err_line == 70001
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("mode", [3])
def test_streaming_decode_edges(mode):
    """Byte-local streaming decode (fx_count / fx_scan / fx_emit): 0x20 runs across thread chunks and tiles, a final
    record without '\\n', unaligned device input, and bad records that hand
    the buffer to the record-aware kernel."""
    ctx = _lib.context()
    try:
        ctx.lib.zs_set_transducer(ctx.h, mode)
        _streaming_decode_edges(mode)
    finally:
        ctx.lib.zs_set_transducer(ctx.h, 3)


def _streaming_decode_edges(mode):
    import torch
    d = z.Dictionary([b"CC", b"c1"], "smiles")
    t = oracle.Tables(d.learned, bytes(sorted(d.identity)))
    rng = random.Random(21)
    lines = []
    for i in range(6000):
        k = rng.randrange(6)
        if k == 0:
            lines.append(b" " * rng.randrange(1, 90))
        elif k == 1:
            lines.append(b"C " * rng.randrange(1, 20) + b"\t\xff")
        else:
            lines.append(bytes(rng.choice(b"Cc1()= \x7f") for _ in range(rng.randrange(0, 60))))
    for tail in (b"\n", b"", b"  x"):
        payload = b"\n".join(lines) + tail
        comp = _oracle_check(payload, d, False, True)
        assert comp is not None and comp.count(b"  ") > 1000
        _oracle_check(comp, d, False, False, "decompress")
        _oracle_check(comp, d, False, True, "decompress")
        # device API at every input alignment
        ctx = _lib.context()
        want, _ = oracle.run_stream(t, comp, "decompress", False, False, 1)
        for off in (0, 1, 7, 13):
            din = torch.zeros(len(comp) + 16, dtype=torch.uint8, device="cuda")
            din[off:off + len(comp)] = torch.frombuffer(bytearray(comp), dtype=torch.uint8).cuda()
            dout = torch.empty(8 * len(comp) + 64, dtype=torch.uint8, device="cuda")
            r = _lib.Result()
            with ctx.lock:
                ctx.set_dictionary(d)
                rc = ctx.lib.zs_decompress_device(ctx.h, din.data_ptr() + off, len(comp),
                                                  dout.data_ptr(), dout.numel(), 0, r)
                ctx.check(rc, "zs_decompress_device")
                kname = ctx.lib.zs_last_kernel(ctx.h).decode()
            assert kname == "fx_count+fx_scan+fx_emit", kname
            assert dout[:r.out_bytes].cpu().numpy().tobytes() == want, off
    # a dangling escape at EOF, an escaped '\n', unknown codes: record-aware path
    comp = _oracle_check(b"\n".join(lines) + b"\n", d, False, True)
    for bad in (comp + b"C ", comp[:5000] + b" \n" + comp[5000:], comp[:9000] + b"\x99" + comp[9000:]):
        _oracle_check(bad, d, False, True, "decompress")
        _oracle_check(bad, d, False, False, "decompress")


@pytest.mark.parametrize("mode", [3])
def test_decode_capacity(mode):
    """Streaming decode (fx_count / fx_scan / fx_emit) with an output
    buffer too small: ZS_E_CAPACITY with the bytes needed, and nothing
    written past the caller's capacity."""
    ctx = _lib.context()
    try:
        ctx.lib.zs_set_transducer(ctx.h, mode)
        _decode_capacity(mode)
    finally:
        ctx.lib.zs_set_transducer(ctx.h, 3)


def _decode_capacity(mode):
    import torch
    d = z.default_dictionary()
    buf = synth.generate("mixed", 50000, 5)
    comp, _ = z.run_buffer(buf, d, "compress", preprocess=False)
    ctx = _lib.context()
    din = torch.from_numpy(comp).cuda()
    for cap in (buf.size // 3, buf.size - 100):
        dout = torch.full((buf.size + 4096,), 0xAB, dtype=torch.uint8, device="cuda")
        r = _lib.Result()
        with ctx.lock:
            ctx.set_dictionary(d)
            rc = ctx.lib.zs_decompress_device(ctx.h, din.data_ptr(), comp.size, dout.data_ptr(), cap, 0, r)
            kname = ctx.lib.zs_last_kernel(ctx.h).decode()
        assert kname == "fx_count+fx_scan+fx_emit", kname
        assert rc == -5 and r.out_bytes == buf.size
        assert bool((dout[cap:] == 0xAB).all())
    r = _lib.Result()
    with ctx.lock:
        rc = ctx.lib.zs_decompress_device(ctx.h, din.data_ptr(), comp.size, dout.data_ptr(), buf.size, 0, r)
    assert rc == 0 and dout[:buf.size].cpu().numpy().tobytes() == buf.tobytes()


@pytest.mark.parametrize("seg", [5, 97, 4096])
def test_run_stream_segmented(stream_cases, seg):
    """run_stream reading the input in small newline-cut segments gives the
    same bytes, stats and errors as the whole-buffer call."""
    dicts = [dict_from_json(dj) for dj in stream_cases["dicts"]]
    for c in stream_cases["cases"][:300]:
        kw = dict(preprocess=c["preprocess"], lenient=c["lenient"])
        payload = bytes.fromhex(c["payload"])
        if "err" in c:
            with pytest.raises(z.LineError) as ei:
                z.run_stream(io.BytesIO(payload), io.BytesIO(), dicts[c["dict"]], c["direction"],
                             segment_bytes=seg, **kw)
            assert ei.value.line_no == c["line_no"] and str(ei.value) == c["msg"]
        else:
            dst = io.BytesIO()
            st = z.run_stream(io.BytesIO(payload), dst, dicts[c["dict"]], c["direction"],
                              segment_bytes=seg, **kw)
            assert dst.getvalue().hex() == c["out"], (seg, c)
            assert (st.lines, st.input_bytes, st.output_bytes, st.escapes, st.skipped,
                    st.flagged) == (c["lines"], c["in_bytes"], c["out_bytes"], c["escapes"],
                                    c["skipped"], c["flagged"])


def test_strict_partial_output_segmented():
    d = z.Dictionary([], "smiles")
    lines = [b"CCO"] * 300 + [b"C1CC"] + [b"CCO"] * 50
    for seg in (3, 40, 100, 1000, 1 << 20):
        for bl in (32, 7, 1000):
            dst = io.BytesIO()
            with pytest.raises(z.LineError) as ei:
                z.run_stream(io.BytesIO(b"\n".join(lines) + b"\n"), dst, d, "compress",
                             preprocess=True, batch_lines=bl, segment_bytes=seg)
            assert ei.value.line_no == 301
            keep = (300 // bl) * bl
            assert dst.getvalue() == b"\n".join([b"CCO"] * keep), (seg, bl)


def test_run_stream_segmented_corpus():
    """A corpus through 1 MB segments == one whole-buffer call, both ways."""
    d = z.default_dictionary()
    buf = synth.generate("skewed", 20000, 2025).tobytes()
    for tail in (b"", b"C1CC1"):
        data = buf + tail
        want, res = z.run_buffer(data, d, "compress", preprocess=True, lenient=True)
        dst = io.BytesIO()
        st = z.run_stream(io.BytesIO(data), dst, d, "compress", preprocess=True, lenient=True,
                          segment_bytes=1 << 20)
        assert dst.getvalue() == want.tobytes() and st.lines == res.lines
        back = io.BytesIO()
        z.run_stream(io.BytesIO(dst.getvalue()), back, d, "decompress", segment_bytes=300000)
        want_back, _ = z.run_buffer(want.tobytes(), d, "decompress")
        assert back.getvalue() == want_back.tobytes()


def test_record_index_random_access():
    """RecordIndex (zs_index_build + zs_decode_records) == decoding the
    whole stream, for random record sets, both framings, and the reference
    decode errors for bad records."""
    d = z.default_dictionary()
    rng = random.Random(33)
    buf = synth.generate("mixed", 30000, 5).tobytes()
    comp, _ = z.run_buffer(buf, d, "compress", preprocess=True, lenient=True)
    comp = comp.tobytes()
    back, _ = z.run_buffer(comp, d, "decompress")
    lines = back.tobytes().split(b"\n")[:-1]
    for blob, want in ((comp, lines), (comp[:-1], lines), (b"\n" + comp, [b""] + lines)):
        ix = z.RecordIndex(blob, d)
        assert len(ix) == len(want)
        sel = [rng.randrange(len(want)) for _ in range(5000)] + [0, len(want) - 1]
        assert ix.decode(sel) == [want[i] for i in sel]
        assert ix[len(want) // 2] == want[len(want) // 2]
    # empty records, bad records
    recs = comp.split(b"\n")[:-1]
    recs[10] = b"\x05\x80"
    recs[20] = b"CC "
    recs[30] = b""
    ix = z.RecordIndex(b"\n".join(recs) + b"\n", d)
    assert ix[30] == b"" and ix[31] == lines[31]
    with pytest.raises(z.UnknownCode) as e1:
        ix.decode([5, 10])
    assert (e1.value.code, e1.value.offset) == (5, 0)
    with pytest.raises(z.TruncatedEscape) as e2:
        ix.decode([20])
    assert e2.value.offset == 2
    with pytest.raises(IndexError):
        ix.decode([len(ix)])
    assert len(z.RecordIndex(b"", d)) == 0
