#!/usr/bin/env python3
"""Golden fixtures for dictionary training, made by
running the REFERENCE trainer itself.  Build container only:

    python tests/golden/make_train_golden.py

Writes ``train_cases.json.gz``:

* ``count``    count_substrings (dictionary.py:169-221): the whole RankTable
               in the reference's row order (length-major, bytewise
               ascending inside a length) for small corpora
* ``overlap``  compute_overlap (dictionary.py:224-238 -> overlap_batch,
               numba_impl.py:142-169): (pattern, selected) -> covered bytes
* ``generate`` generate (dictionary.py:310-320): corpus + GenerationParams +
               mode -> learned patterns in code order, or the exception the
               strict preprocess raised
* ``cap``      the same at working-set caps 3 and 10 (dictionary.py:40-43)
* ``synthetic`` generate on the generator corpora (synth/, byte-identical to
               scripts/make_corpus.py) -> learned patterns; the 12 C4
               dictionaries and default.zsd already live in dicts/

Nothing here is imported by the product; the fixtures are plain data.
"""

import gzip
import json
import os
import random
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="zs_numba_"))
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
sys.path.insert(0, REPO)

import zsmiles as z  # noqa: E402  (the reference)
from zsmiles import dictionary as zd  # noqa: E402
import conftest as zconf  # noqa: E402
import synth  # noqa: E402

H = bytes.hex
ODD = [b"A \x7fB!", b"", b"C\tC", b"\xffCC", b"CC CC", b"[Na+].[Cl-]", b"%12"]


def table_rows(corpus, lmin, lmax):
    t = z.count_substrings(corpus, z.GenerationParams(l_min=lmin, l_max=lmax))
    return [[H(t.pattern(i)), int(t.occurrences[i])] for i in range(len(t))]


def count_cases():
    out = []
    fixed = [([b"CCO", b"CCN"], 2, 3), ([b"AAA"], 2, 2), ([b"C"], 2, 3), ([b"AB", b"BA"], 2, 2),
             ([b"A B", b"C!D"], 2, 2), ([b"CCCCCCCCCCCCCCCCCCCC"], 2, 20),
             ([b"c1ccccc1" * 6], 5, 40), ([b"x" * 70], 60, 64)]
    for corpus, lo, hi in fixed:
        out.append({"corpus": [H(l) for l in corpus], "l_min": lo, "l_max": hi,
                    "rows": table_rows(corpus, lo, hi)})
    for k, (lo, hi) in enumerate([(2, 3), (2, 8), (3, 10), (9, 12), (2, 16), (2, 17), (7, 25),
                                  (2, 33)]):
        rng = random.Random(300 + k)
        corpus = [zconf.smiles_like_line(rng, rng.choice([3, 8, 20])) for _ in range(40)]
        corpus += [rng.choice(ODD) for _ in range(4)]
        out.append({"corpus": [H(l) for l in corpus], "l_min": lo, "l_max": hi,
                    "rows": table_rows(corpus, lo, hi)})
    return out


def overlap_cases():
    rng = random.Random(4242)
    out = [{"p": H(b"CCO"), "sel": [H(b"CC")], "ov": 2},
           {"p": H(b"CCCO"), "sel": [H(b"CCC"), H(b"CO")], "ov": 3}]
    for _ in range(400):
        sel = zconf.random_patterns(rng, rng.randint(0, 16), 2, rng.choice([4, 8, 15]))
        if sel and rng.random() < 0.5:
            p = (rng.choice(sel) * 3)[:rng.randint(0, 24)]
        else:
            p = bytes(rng.choice(b"CNO(=)1c") for _ in range(rng.randint(0, 24)))
        out.append({"p": H(p), "sel": [H(s) for s in sel], "ov": z.compute_overlap(p, sel)})
    return out


def gen_case(corpus, mode="strict", **kw):
    params = z.GenerationParams(**kw)
    e = {"corpus": [H(l) for l in corpus], "mode": mode, "params": kw}
    try:
        d = z.generate(corpus, params, mode)
        e["learned"] = [H(p) for p in d.learned]
    except Exception as ex:  # noqa: BLE001 -- the exception IS the fixture
        e["error"] = [type(ex).__name__, str(ex)]
    return e


def generate_cases():
    out = [
        gen_case([b"CCO", b"CCN"], l_min=2, l_max=3, t=2),
        gen_case([b"CCO"], t=0),
        gen_case([b"CN=C(O)S"] * 100, l_min=2, l_max=8, t=1),
        gen_case([b"c1ccccc1"] * 100, l_min=2, l_max=8, t=1),
        gen_case([b"C1CC1"] * 50, l_min=2, l_max=8, t=1, preprocess=True),
        gen_case([b"ABAB", b"AB"], l_min=2, l_max=4, t=5),
        gen_case([b"C"], t=4),
        gen_case([b"A B", b"C!D"], t=4, l_max=2),
        gen_case([b"C[NH3+", b"CCO"], t=3, preprocess=True),                 # strict: raises
        gen_case([b"C[NH3+", b"CCO", b"C1CC"], "lenient", t=3, preprocess=True),
        gen_case([b"C%1CC", b"CCO"], t=3, preprocess=True),
        gen_case([b"C1CC"], t=3, preprocess=True),
        gen_case([b"CC" * 40], l_min=20, l_max=64, t=8),
        gen_case([b"x" * 100, b"y" * 99], l_min=2, l_max=64, t=128),
    ]
    for seed in range(4):                       # test_dictionary.py:205-213
        rng = random.Random(seed)
        corpus = [zconf.smiles_like_line(rng, 3) for _ in range(25)]
        if not any(len(l) >= 2 for l in corpus):
            corpus.append(b"CCO")
        out.append(gen_case(corpus, l_min=2, l_max=4, t=12))
    for k, (lo, hi, t, pre, pop) in enumerate([
            (2, 8, 32, False, "smiles"), (2, 8, 128, True, "none"), (3, 12, 64, False, "printable"),
            (2, 16, 128, True, "smiles"), (2, 17, 40, False, "smiles"), (4, 24, 100, True, "smiles"),
            (2, 5, 128, False, "smiles"), (6, 40, 20, False, "smiles")]):
        rng = random.Random(700 + k)
        corpus = [zconf.smiles_like_line(rng, rng.choice([4, 8, 16])) for _ in range(300)]
        corpus += [rng.choice(ODD) for _ in range(6)]
        out.append(gen_case(corpus, "lenient", l_min=lo, l_max=hi, t=t, preprocess=pre,
                            prepopulate=pop))
    return out


def cap_cases(gen):
    """The working-set cap (dictionary.py:40-43, 241-307) at tiny values: the
    retry path, and the reference's early stop when the capped working set
    runs dry before t picks (a cap-dependent result)."""
    out = []
    saved = zd._WORKING_SET_CAP
    try:
        for cap in (3, 10):
            zd._WORKING_SET_CAP = cap
            for k, e in enumerate(gen[-8:]):
                lines = [bytes.fromhex(x) for x in e["corpus"]]
                d = z.generate(lines, z.GenerationParams(**e["params"]), e["mode"])
                out.append({"case": len(gen) - 8 + k, "cap": cap, "learned": [H(p) for p in d.learned]})
    finally:
        zd._WORKING_SET_CAP = saved
    return out


def synthetic_cases():
    out = []
    for kind, n, seed, kw in [("mixed", 50_000, 2024, dict(t=128, l_max=8, preprocess=False)),
                              ("aromatic", 10_000, 2024, dict(t=64, l_min=3, l_max=24, preprocess=True)),
                              ("aliphatic", 10_000, 2024, dict(t=128, l_max=20, preprocess=False))]:
        buf = synth.generate(kind, n, seed).tobytes()
        lines = buf.split(b"\n")
        if lines and lines[-1] == b"":
            lines.pop()
        d = z.generate(lines, z.GenerationParams(**kw), "strict")
        out.append({"kind": kind, "lines": n, "seed": seed, "params": kw,
                    "learned": [H(p) for p in d.learned]})
        print(f"synthetic {kind} {n} {kw}: {len(d.learned)} patterns", flush=True)
    return out


def main():
    gen = generate_cases()
    cases = {"count": count_cases(), "overlap": overlap_cases(), "generate": gen,
             "cap": cap_cases(gen), "synthetic": synthetic_cases(),
             "working_set_cap": zd._WORKING_SET_CAP}
    path = os.path.join(HERE, "train_cases.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} B)")


if __name__ == "__main__":
    main()
