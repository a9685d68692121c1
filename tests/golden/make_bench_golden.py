#!/usr/bin/env python3
"""Golden output of the reference's own ``zsmiles bench`` (cli.py:96-152):
the ablation table (Table I: preprocess x prepopulate) and the
cross-dictionary matrix (Table II) on small synthetic corpora, recorded by
running the UNMODIFIED reference CLI here (build container only; it needs
/root/reference):

    python tests/golden/make_bench_golden.py

writes tests/golden/bench_cases.json: the corpora recipes (reference
generator, seeds), the arguments, and the ratio cells the reference printed
(the MB/s column is timing, not contract).
"""
import contextlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="zs_numba_"))
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from zsmiles.cli import main as ref_main  # noqa: E402

CORPORA = {"mixed": ("mixed", 3000, 2024), "aromatic": ("aromatic", 1500, 7), "aliphatic": ("aliphatic", 1500, 8)}
CASES = [
    {"name": "ablation", "corpora": ["mixed"], "args": ["--dict-size", "64"]},
    {"name": "ablation_l5", "corpora": ["mixed"], "args": ["--dict-size", "32", "--lmax", "5", "--sample", "1200",
                                                           "--seed", "3"]},
    {"name": "matrix", "corpora": ["aromatic", "aliphatic", "mixed"], "args": ["--dict-size", "64"]},
]


def ratio_cells(text, matrix):
    rows = text.strip().splitlines()
    if not matrix:
        return [[r.split()[0], r.split()[1], r.split()[2]] for r in rows[1:]]
    return [[r.split()[0]] + r.split()[1:] for r in rows[2:]]


def main():
    tmp = tempfile.mkdtemp(prefix="zs_bench_")
    paths = {}
    for name, (kind, n, seed) in CORPORA.items():
        p = os.path.join(tmp, f"{name}.smi")
        with open(p, "wb") as fh:
            fh.write(synth.generate(kind, n, seed).tobytes())
        paths[name] = p
    out = {"corpora": CORPORA, "cases": []}
    for c in CASES:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = ref_main(["bench", "-i", *[paths[k] for k in c["corpora"]], *c["args"]])
        assert rc == 0
        text = buf.getvalue()
        print(text)
        out["cases"].append({**c, "cells": ratio_cells(text, len(c["corpora"]) > 1)})
    with open(os.path.join(HERE, "bench_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
