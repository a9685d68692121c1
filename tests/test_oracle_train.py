"""Pin the CPU restatement of the dictionary trainer (oracle/zs_oracle_train.c)
to the reference trainer's own outputs (tests/golden/make_train_golden.py and
the .zsd files make_golden.py regenerated with the reference ``generate``)."""

import pytest

import oracle
import synth
from conftest import golden_dict_bytes


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()
    synth.build()


def lines_of(kind, n, seed):
    rows = synth.generate(kind, n, seed).tobytes().split(b"\n")
    if rows and rows[-1] == b"":
        rows.pop()
    return rows


def lenient_pre(lines):
    """preprocess_line(l, "lenient") (smiles.py:183-213): tokenize / pairing
    failures keep the raw line."""
    out = []
    for line in lines:
        k, v = oracle.preprocess(line)
        assert k != 5, "RingIdOverflow propagates even in lenient mode"
        out.append(v if k == 0 else line)
    return out


def test_count_substrings(train_cases):
    for c in train_cases["count"]:
        lines = [bytes.fromhex(x) for x in c["corpus"]]
        got = [[p.hex(), o] for p, o in oracle.table_entries(lines, c["l_min"], c["l_max"])]
        assert got == c["rows"], (c["l_min"], c["l_max"])


def test_overlap(train_cases):
    for c in train_cases["overlap"]:
        assert oracle.overlap(bytes.fromhex(c["p"]), [bytes.fromhex(s) for s in c["sel"]]) == c["ov"]


def test_generate_cases(train_cases):
    for c in train_cases["generate"]:
        if "error" in c:
            continue
        pr = c["params"]
        lines = [bytes.fromhex(x) for x in c["corpus"]]
        if pr.get("preprocess"):
            lines = lenient_pre(lines)
        got = oracle.train(lines, pr.get("l_min", 2), pr.get("l_max", 8), pr.get("t", 128))
        assert [g.hex() for g in got] == c["learned"], pr


def test_working_set_cap(train_cases):
    """dictionary.py:40-43, 256-289 at tiny caps: the exclusion-check retry,
    and the reference's early stop when the capped working set runs dry (one
    of the fixtures returns 10 patterns at cap 10 instead of 20)."""
    for k in train_cases["cap"]:
        c = train_cases["generate"][k["case"]]
        pr = c["params"]
        lines = [bytes.fromhex(x) for x in c["corpus"]]
        if pr.get("preprocess"):
            lines = lenient_pre(lines)
        got = oracle.train(lines, pr.get("l_min", 2), pr.get("l_max", 8), pr.get("t", 128), k["cap"])
        assert [g.hex() for g in got] == k["learned"], (pr, k["cap"])


@pytest.mark.parametrize("name,t,lmax", [("default.zsd", 128, 8), ("t16_l5.zsd", 16, 5)])
def test_golden_dictionaries(name, t, lmax):
    """generate(mixed_50k, GenerationParams(preprocess=True, ...)) byte-equal
    to the reference-trained dictionaries."""
    mixed = lenient_pre(lines_of("mixed", 50_000, 2024))
    want = golden_dict_bytes(name).split(b"\n")[3:-1]
    assert oracle.train(mixed, 2, lmax, t) == want


def test_synthetic_case(train_cases):
    c = train_cases["synthetic"][1]
    pr = c["params"]
    lines = lines_of(c["kind"], c["lines"], c["seed"])
    if pr.get("preprocess"):
        lines = lenient_pre(lines)
    got = oracle.train(lines, pr.get("l_min", 2), pr.get("l_max", 8), pr.get("t", 128))
    assert [g.hex() for g in got] == c["learned"]
