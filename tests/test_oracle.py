"""Pin the CPU oracle (oracle/zs_oracle.c) to the reference's own outputs.

Every fixture here was produced by running the unmodified reference package
(tests/golden/make_golden.py); the oracle must reproduce all of them before
it is trusted as the checker for the GPU path.
"""

import hashlib

import pytest

import oracle
import synth
from conftest import golden_dict_bytes

pytestmark = []


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()
    synth.build()


def test_compress_batch_matches_reference(codec_cases):
    for c in codec_cases:
        t = oracle.Tables.from_json(c["dict"])
        recs, esc = oracle.compress_batch(t, [bytes.fromhex(l) for l in c["lines"]])
        assert [r.hex() for r in recs] == c["records"]
        assert esc == c["escapes"]


def test_decompress_matches_reference(decode_cases):
    for c in decode_cases:
        t = oracle.Tables.from_json(c["dict"])
        r = oracle.decompress_batch(t, [bytes.fromhex(x) for x in c["records"]])
        assert r["out"].hex() == c["out"]
        assert r["out_lens"].tolist() == c["out_lens"]
        assert r["status"].tolist() == c["status"]
        assert r["errpos"].tolist() == c["errpos"]
        assert (r["total"], r["escapes"]) == (c["total"], c["escapes"])


def test_preprocess_matches_reference(preprocess_cases):
    for c in preprocess_cases:
        k, v = oracle.preprocess(bytes.fromhex(c["line"]))
        s = c["strict"]
        if k == 0:
            assert s.get("out") == v.hex(), c
        else:
            assert s.get("err") == oracle.ERR_NAMES[k], c


@pytest.mark.parametrize("threads", [1, 3])
def test_stream_matches_reference(stream_cases, threads):
    tabs = [oracle.Tables.from_json(d) for d in stream_cases["dicts"]]
    for c in stream_cases["cases"]:
        out, st = oracle.run_stream(tabs[c["dict"]], bytes.fromhex(c["payload"]), c["direction"],
                                    c["preprocess"], c["lenient"], threads)
        if "err" in c:
            assert st["err_line"] == c["line_no"]
            assert oracle.ERR_NAMES[st["err_kind"]] == c["cause"]
        else:
            assert out.hex() == c["out"]
            for k in ("lines", "in_bytes", "out_bytes", "escapes", "skipped", "flagged"):
                assert st[k] == c[k], (k, c)


@pytest.mark.parametrize("name", ["aromatic_10k", "aliphatic_10k", "mixed_50k", "c1_100k",
                                  "c3_skewed_20k"])
def test_synth_and_oracle_corpus_hashes(corpus_hashes, name):
    e = corpus_hashes[name]
    buf = synth.generate(e["kind"], e["lines"], e["seed"])
    assert hashlib.sha256(buf.tobytes()).hexdigest() == e["in_sha256"]
    t = oracle.Tables.from_zsd(golden_dict_bytes(e["dict"]))
    for key, pre in (("pre_off", False), ("pre_on", True)):
        out, st = oracle.run_stream(t, buf, "compress", pre, True, 8)
        assert hashlib.sha256(out).hexdigest() == e[key]["comp_sha256"]
        assert st["escapes"] == e[key]["escapes"] and st["flagged"] == e[key]["flagged"]
        back, _ = oracle.run_stream(t, out, "decompress", False, False, 8)
        assert hashlib.sha256(back).hexdigest() == e[key]["roundtrip_sha256"]


def test_ablation_dictionary_hashes(corpus_hashes):
    e0 = corpus_hashes["c1_100k"]
    buf = synth.generate(e0["kind"], e0["lines"], e0["seed"])
    for name, e in corpus_hashes.items():
        if not name.startswith("c4_"):
            continue
        t = oracle.Tables.from_zsd(golden_dict_bytes(e["dict"]))
        out, _ = oracle.run_stream(t, buf, "compress", True, True, 8)
        assert hashlib.sha256(out).hexdigest() == e["pre_on"]["comp_sha256"], name
