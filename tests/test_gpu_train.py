"""GPU dictionary training (csrc/zs_train.cuh) vs the reference trainer's own
outputs (tests/golden/train_cases.json.gz, tests/golden/dicts/*.zsd) and vs
the CPU oracle (oracle/zs_oracle_train.c).  Byte-identical throughout."""

import random

import numpy as np
import pytest

import oracle
import synth
from conftest import golden_dict_bytes, has_gpu

pytestmark = pytest.mark.gpu

if has_gpu():
    import paper_2404_19391_b200 as z
    from paper_2404_19391_b200 import dictionary as zd
    from paper_2404_19391_b200 import kernels
    from paper_2404_19391_b200.cli import main as cli_main


@pytest.fixture(scope="module", autouse=True)
def _ready():
    if not has_gpu():
        pytest.skip("no GPU")
    oracle.build()
    synth.build()


def lines_of(kind, n, seed):
    rows = synth.generate(kind, n, seed).tobytes().split(b"\n")
    if rows and rows[-1] == b"":
        rows.pop()
    return rows


def test_count_substrings_golden(train_cases):
    for c in train_cases["count"]:
        lines = [bytes.fromhex(x) for x in c["corpus"]]
        t = z.count_substrings(lines, z.GenerationParams(l_min=c["l_min"], l_max=c["l_max"]))
        got = [[t.pattern(i).hex(), int(t.occurrences[i])] for i in range(len(t))]
        assert got == c["rows"], (c["l_min"], c["l_max"])
        assert (t.ranks == t.occurrences * t.lengths).all()
        assert t.patterns.shape[1] == c["l_max"]


def test_count_substrings_reference_cases():
    """test_dictionary.py:79-109"""
    P = z.GenerationParams
    assert z.count_substrings([b"CCO", b"CCN"], P(l_min=2, l_max=3)).entries == \
        {b"CC": (2, 4), b"CO": (1, 2), b"CN": (1, 2), b"CCO": (1, 3), b"CCN": (1, 3)}
    assert z.count_substrings([b"AAA"], P(l_min=2, l_max=2)).entries == {b"AA": (2, 4)}
    assert len(z.count_substrings([b"C"], P(l_min=2, l_max=3))) == 0
    assert z.count_substrings([b"AB", b"BA"], P(l_min=2, l_max=2)).entries == \
        {b"AB": (1, 2), b"BA": (1, 2)}
    assert z.count_substrings([b"A B", b"C!D"], P(l_min=2, l_max=2)).entries == {}
    assert z.count_substrings([b""], P()).entries == {}
    with pytest.raises(z.EmptyCorpus):
        z.count_substrings([], P())


@pytest.mark.parametrize("lmin,lmax", [(2, 8), (2, 15), (3, 24), (2, 64)])
def test_count_substrings_vs_oracle(lmin, lmax):
    """Census of 20k generator lines (+ non-alphabet noise) at l_max across
    the 8-byte key-word boundaries, row for row against the oracle."""
    rng = random.Random(lmax)
    lines = lines_of("mixed", 20_000, 2024)
    for k in range(0, len(lines), 97):
        j = rng.randrange(len(lines[k]) + 1)
        lines[k] = lines[k][:j] + bytes([rng.choice(b" \t\xff!")]) + lines[k][j:]
    t = z.count_substrings(lines, z.GenerationParams(l_min=lmin, l_max=lmax))
    buf, pos, ln, occ = oracle.count_substrings(lines, lmin, lmax)
    assert len(t) == pos.size
    assert (t.lengths == ln).all() and (t.occurrences == occ).all()
    b = np.frombuffer(buf.tobytes() + bytes(lmax), np.uint8)
    want = b[pos[:, None] + np.arange(lmax)[None, :]]
    want = np.where(np.arange(lmax)[None, :] < ln[:, None], want, 0)
    assert (t.patterns == want).all()


def test_overlap_golden(train_cases):
    for c in train_cases["overlap"]:
        assert z.compute_overlap(bytes.fromhex(c["p"]), [bytes.fromhex(s) for s in c["sel"]]) == c["ov"]


def test_overlap_batch_harness():
    """kernels.overlap_batch in the reference's array layout
    (numba_impl.py:142-169), many rows per call, vs the oracle."""
    rng = random.Random(17)
    for _ in range(20):
        sel = list({bytes(rng.choice(b"CNO(=)1c") for _ in range(rng.randint(1, 6)))
                    for _ in range(rng.randint(1, 30))})
        trie = z.dictionary.PatternTrie.from_patterns([(s, 0) for s in sel])
        rows = [bytes(rng.choice(b"CNO(=)1c") for _ in range(rng.randint(0, 40))) for _ in range(300)]
        width = max(1, max(len(r) for r in rows))
        pats = np.zeros((len(rows), width), np.uint8)
        for i, r in enumerate(rows):
            pats[i, :len(r)] = np.frombuffer(r, np.uint8)
        out = np.full(len(rows), -7, np.int64)
        kernels.overlap_batch(trie.children, trie.term_len, pats,
                              np.array([len(r) for r in rows], np.int64), out)
        assert out.tolist() == [oracle.overlap(r, sel) for r in rows]


def test_generate_golden(train_cases):
    for c in train_cases["generate"]:
        lines = [bytes.fromhex(x) for x in c["corpus"]]
        params = z.GenerationParams(**c["params"])
        if "error" in c:
            with pytest.raises(z.ZsmilesError) as ei:
                z.generate(lines, params, c["mode"])
            assert [type(ei.value).__name__, str(ei.value)] == c["error"]
            continue
        d = z.generate(lines, params, c["mode"])
        assert [p.hex() for p in d.learned] == c["learned"], c["params"]
        assert d.prepopulate == c["params"].get("prepopulate", "smiles")


def test_generate_reference_cases():
    """test_dictionary.py:164-231"""
    P = z.GenerationParams
    assert z.generate([b"CCO", b"CCN"], P(l_min=2, l_max=3, t=2)).learned == (b"CC", b"CN")
    d = z.generate([b"CCO"], P(t=0))
    assert d.learned == () and d.identity == z.ALPHABET
    assert z.generate([b"CN=C(O)S"] * 100, P(t=1)).learned == (b"CN=C(O)S",)
    assert z.generate([b"c1ccccc1"] * 100, P(t=1)).learned == (b"ccc",)
    assert z.generate([b"C1CC1"] * 50, P(t=1, preprocess=True)).learned == (b"C0CC0",)
    assert z.generate([b"ABAB", b"AB"], P(l_min=2, l_max=4, t=5)).learned == \
        (b"AB", b"BA", b"ABA", b"BAB")
    with pytest.raises(z.EmptyCorpus):
        z.generate([], P())


def test_working_set_cap(train_cases, monkeypatch):
    """dictionary.py:40-43, 256-289: retry on a failed exclusion check and
    the capped working set running dry (a reference fixture returns 10
    patterns at cap 10 instead of 20)."""
    for k in train_cases["cap"]:
        c = train_cases["generate"][k["case"]]
        monkeypatch.setattr(zd, "_WORKING_SET_CAP", k["cap"])
        d = z.generate([bytes.fromhex(x) for x in c["corpus"]], z.GenerationParams(**c["params"]), c["mode"])
        assert [p.hex() for p in d.learned] == k["learned"], (c["params"], k["cap"])


def test_select_from_host_table(train_cases):
    """select_patterns on a RankTable the GPU did not count (uploaded with
    zs_train_load): same picks, ties broken on the pattern bytes."""
    c = train_cases["generate"][-3]
    lines = [bytes.fromhex(x) for x in c["corpus"]]
    params = z.GenerationParams(**c["params"])
    if params.preprocess:
        lines = zd._preprocess_all(lines, c["mode"])
    t = z.count_substrings(lines, params)
    perm = np.random.default_rng(3).permutation(len(t))  # row order must not matter
    t2 = z.RankTable(t.patterns[perm].copy(), t.lengths[perm].copy(), t.occurrences[perm].copy(),
                     t.ranks[perm].copy())
    assert [p.hex() for p in z.select_patterns(t2, params.t)] == c["learned"]


def test_synthetic_golden(train_cases):
    for c in train_cases["synthetic"]:
        d = z.generate(lines_of(c["kind"], c["lines"], c["seed"]), z.GenerationParams(**c["params"]))
        assert [p.hex() for p in d.learned] == c["learned"], c["params"]


def test_golden_dictionaries():
    """default.zsd and the 12 C4 dictionaries: generate(mixed_50k,
    preprocess=True) byte-equal after serialisation."""
    mixed = lines_of("mixed", 50_000, 2024)
    d = z.generate(mixed, z.GenerationParams(preprocess=True))
    assert z.serialize(d) == golden_dict_bytes("default.zsd")
    for t in (16, 32, 64, 128):
        for lmax in (5, 8, 15):
            d = z.generate(mixed, z.GenerationParams(t=t, l_max=lmax, preprocess=True))
            assert z.serialize(d) == golden_dict_bytes(f"t{t}_l{lmax}.zsd"), (t, lmax)


def test_cli_train_and_bench(tmp_path, capsys):
    """cli.py:60-70, 96-152 through main(argv) (test_cli.py:28-75, 148-181)."""
    rng = random.Random(31)
    corpus = tmp_path / "corpus.smi"
    corpus.write_bytes(b"".join(l + b"\n" for l in lines_of("mixed", 400, 7)))
    out = tmp_path / "d.zsd"
    assert cli_main(["train", "-i", str(corpus), "-o", str(out), "--dict-size", "16", "--stats"]) == 0
    assert "patterns=16 lines=400" in capsys.readouterr().err
    d = z.load_dictionary(str(out))
    assert d == z.generate(lines_of("mixed", 400, 7), z.GenerationParams(t=16))
    assert cli_main(["train", "-i", str(corpus), "-o", str(out), "--sample", "0"]) == 1
    assert "zsmiles: error:" in capsys.readouterr().err
    with pytest.raises(SystemExit) as ei:
        cli_main(["train", "-i", str(corpus)])
    assert ei.value.code == 2
    capsys.readouterr()
    p = tmp_path / "c.smi"
    p.write_bytes(b"".join(bytes(rng.choice(b"CNOc1(=)") for _ in range(rng.randint(3, 30))) + b"\n"
                           for _ in range(80)))
    assert cli_main(["bench", "-i", str(p), "--dict-size", "24"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert len(rows) == 7 and rows[0].split() == ["preprocess", "prepopulate", "ratio", "MB/s"]
    assert [tuple(r.split()[:2]) for r in rows[1:]] == [
        ("yes", "printable"), ("no", "printable"), ("yes", "smiles"), ("no", "smiles"),
        ("yes", "none"), ("no", "none")]
    b = tmp_path / "b.smi"
    b.write_bytes(b"NC(=O)CS\n" * 60)
    assert cli_main(["bench", "-i", str(p), str(b), "--dict-size", "24"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert len(rows) == 4 and "c.smi" in rows[1] and "b.smi" in rows[1]
    for r in rows[2:]:
        assert all(0.0 < float(x) <= 1.5 for x in r.split()[1:])


def test_bench_tables_match_reference(tmp_path, capsys):
    """`zsmiles bench` (ablation table and cross-dictionary matrix) prints the
    same ratio cells as the reference's own CLI on the same corpora
    (tests/golden/bench_cases.json, made by running the reference,
    make_bench_golden.py), and the paper's Table I / II trends hold as the
    reference's acceptance test states them (test_acceptance.py:111-149):
    renumbering on beats off for every prepopulation, 'smiles' is the best
    prepopulation, and each corpus compresses best with its own dictionary."""
    import json
    import os
    from conftest import ROOT
    with open(os.path.join(ROOT, "tests", "golden", "bench_cases.json")) as fh:
        g = json.load(fh)
    paths = {}
    for name, (kind, n, seed) in g["corpora"].items():
        p = tmp_path / f"{name}.smi"
        p.write_bytes(synth.generate(kind, n, seed).tobytes())
        paths[name] = str(p)
    for c in g["cases"]:
        assert cli_main(["bench", "-i", *[paths[k] for k in c["corpora"]], *c["args"]]) == 0
        rows = capsys.readouterr().out.strip().splitlines()
        if len(c["corpora"]) == 1:
            cells = [r.split()[:3] for r in rows[1:]]
            assert cells == c["cells"], c["name"]
            ratio = {(r[0] == "yes", r[1]): float(r[2]) for r in cells}
            for m in ("printable", "smiles", "none"):
                assert ratio[(True, m)] < ratio[(False, m)]
            for pre in (True, False):
                assert ratio[(pre, "smiles")] <= min(ratio[(pre, "printable")], ratio[(pre, "none")])
        else:
            cells = [r.split() for r in rows[2:]]
            assert cells == c["cells"], c["name"]
            grid = [[float(x) for x in r[1:]] for r in cells]
            for te in range(len(grid)):
                assert all(grid[te][te] <= grid[tr][te] for tr in range(len(grid)))

