#!/usr/bin/env python3
"""Generate the committed golden fixtures by running the REFERENCE itself.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py [--big]

It imports the unmodified reference package (``/root/reference/pkg/src``) with
``NUMBA_CACHE_DIR`` pointed at a scratch dir so numba never writes into the
read-only tree, and records input/output pairs for every row of SURVEY.md §8:

* ``codec_cases.json.gz``      compress_batch (numba_impl.py:16-71) on random
                            dictionaries, escape-heavy bytes, KATs
* ``decode_cases.json.gz``     decompress_sizes/decompress_fill
                            (numba_impl.py:74-139) incl. malformed records
* ``preprocess_cases.json.gz`` preprocess_line (smiles.py:183-213), strict and
                            lenient, with exact exception types and messages
* ``stream_cases.json.gz``     run_stream (pipeline.py:129-167) framing, CR
                            policy, strict/lenient error modes, stats
* ``corpus_hashes.json``    sha256 of whole-corpus compress / round-trip
                            outputs for the bundled and synthetic configs
* ``dicts/*.zsd``           the default dictionary (regenerated with the
                            reference ``generate`` and checked byte-equal to
                            the shipped one) and the C4 ablation dictionaries

Nothing here is imported by the product; the fixtures are plain data.
"""

import argparse
import gzip
import hashlib
import io
import json
import multiprocessing as mp
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
sys.path.insert(0, os.path.join(REF, "scripts"))

import zsmiles as z  # noqa: E402  (the reference)
from zsmiles import codec as zcodec  # noqa: E402
from zsmiles.pipeline import run_stream  # noqa: E402
from zsmiles.dictionary import GenerationParams  # noqa: E402
import conftest as zconf  # noqa: E402
import make_corpus  # noqa: E402

H = bytes.hex


def dict_json(d):
    return {
        "learned": [H(p) for p in d.learned],
        "identity": H(bytes(sorted(d.identity))),
        "prepopulate": d.prepopulate,
        "l_min": d.l_min,
        "l_max": d.l_max,
    }


def dump(name, obj):
    path = os.path.join(HERE, name + ".gz")
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} B)")


# --------------------------------------------------------------------------
# codec (compress_batch) and decode fixtures
# --------------------------------------------------------------------------

ODD = [b"C\tC", b"caf\xc3\xa9", b"\x00\xffC", b"a  b", b" ", b"  ", b"\x7f",
       b"\xc3", b"C C", b"\x01\x02\x03", b"CC\rO", b"C\nC"]


def codec_cases():
    cases = []
    # KATs from the reference tests (test_codec.py:15-29)
    kat = [
        (z.Dictionary([b"CC"], None, identity=b"CO"), [b"CCO"]),
        (z.Dictionary([b"CC"], "smiles"), [b""]),
        (z.Dictionary([], None, identity=b"C"), [b"Cy"]),
        (z.Dictionary([b"CC", b"CCC"], None, identity=b"C"), [b"CCCC"]),
        (z.Dictionary([], None, identity=b"C"), [b"Cy", b"zz"]),
    ]
    rng = random.Random(1001)
    for _ in range(40):
        d = zconf.random_dictionary(rng)
        lines = [zconf.smiles_like_line(rng) for _ in range(50)] + [b""]
        lines += [rng.choice(ODD) for _ in range(4)]
        # a few long lines and all-escape lines
        lines.append(b"".join(zconf.smiles_like_line(rng) for _ in range(8)))
        lines.append(bytes(rng.randrange(256) for _ in range(rng.randint(1, 30))))
        kat.append((d, lines))
    # deep dictionaries: long patterns (lmax up to 64) and chains of prefixes
    for L in (15, 32, 64):
        pats = [b"C" * k for k in range(2, L + 1, 3)] + [b"c1ccccc1" * (L // 8)]
        pats = [p[:L] for p in pats]
        pats = sorted(set(pats))
        d = z.Dictionary(pats, "smiles", l_min=2, l_max=L)
        lines = [b"C" * n for n in range(0, 80, 7)] + \
                [b"c1ccccc1" * k for k in range(1, 12)]
        kat.append((d, lines))
    for d, lines in kat:
        recs, esc = zcodec.compress_lines(d, lines)
        cases.append({"dict": dict_json(d), "lines": [H(l) for l in lines],
                      "records": [H(r) for r in recs], "escapes": esc})
    return cases


def decode_cases():
    cases = []
    rng = random.Random(2002)
    bad = [bytes([0x20]), bytes([0x0B]), b"\x99\x98", b" x \x01", b"   ",
           b"C ", b" C \xff", b"\x80\x81\x82", b""]
    for _ in range(30):
        d = zconf.random_dictionary(rng)
        lines = [zconf.smiles_like_line(rng) for _ in range(30)] + [b""]
        recs, _ = zcodec.compress_lines(d, lines)
        recs = list(recs) + bad + [bytes(rng.randrange(256) for _ in range(rng.randint(0, 12)))
                                   for _ in range(6)]
        out = zconf_run_decompress(d, recs)
        cases.append({"dict": dict_json(d), "records": [H(r) for r in recs], **out})
    return cases


def zconf_run_decompress(d, recs):
    """The reference kernel harness shape (test_kernels.py:35-48)."""
    import numpy as np
    from zsmiles import kernels
    exp_len, valid, exp_off, exp_flat = d.decode_tables
    flat = np.frombuffer(b"".join(recs), np.uint8)
    starts = np.zeros(len(recs) + 1, np.int64)
    np.cumsum([len(r) for r in recs], out=starts[1:])
    n = len(recs)
    out_lens = np.empty(n, np.int64)
    status = np.empty(n, np.int8)
    errpos = np.empty(n, np.int64)
    total, esc = kernels.decompress_sizes(exp_len, valid, flat, starts,
                                          out_lens, status, errpos)
    out_starts = np.zeros(n + 1, np.int64)
    np.cumsum(out_lens, out=out_starts[1:])
    out = np.zeros(int(total), np.uint8)
    kernels.decompress_fill(exp_off, exp_flat, flat, starts, status, out, out_starts)
    return {"out": H(out.tobytes()), "out_lens": out_lens.tolist(),
            "status": status.tolist(), "errpos": errpos.tolist(),
            "total": int(total), "escapes": int(esc)}


# --------------------------------------------------------------------------
# preprocess fixtures
# --------------------------------------------------------------------------

def nested(n, close_reversed=True):
    ids = [str(i) if i < 10 else f"%{i:02d}" for i in range(n)]
    tail = reversed(ids) if close_reversed else ids
    return ("".join(f"C{r}" for r in ids) + "".join(f"C{r}" for r in tail)).encode()


def pp_result(line, mode):
    try:
        out = z.preprocess_line(line, mode)
        return {"out": H(out)}
    except z.ZsmilesError as e:
        return {"err": type(e).__name__, "msg": str(e)}


def preprocess_cases():
    lines = [
        b"C1=CC=C(C=C1)C(=O)CC(=O)C2=CC=CC=C2", b"CCO", b"C1CC2CCC2C1",
        b"C%10CC%10", b"C=1CCC=1", nested(12), nested(100), nested(101),
        nested(100, False), nested(30, False), b"C1CC", b"C[NH", b"C1CC1",
        b"", b"[13CH4]", b"C%12CC%12", b"1CC", b"C(C)1CC", b"C12CC1C2",
        b"(%12C", b"C%1", b"C%x2", b"C%", b"C.1C", b"C.C#N", b"C%%12",
        b"C]1CC1", b"C[1]1CC1", b"[C]1[C]1", b"C[N%1]1CC1", b"C1%12CC1%12",
        b"C1CC1C1CC1", b"C11", b"C1C1", b"*1**1", b"C$1CC$1", b"C~1CC1",
        b"C 1CC1", b"C@1CC1", b"C+1CC+1", b"C1CC1[", b"[C1CC1", b"%12",
        b"C%123", b"C%12%12", b"C1%121%12", b"C0CC0", b"C9CC9C8CC8",
        b"c1ccccc1-c1ccccc1", b"C1CC2CC1CC2", b"C1CC2CC3CC1CC2CC3",
    ]
    rng = random.Random(3003)
    for _ in range(600):
        lines.append(zconf.smiles_like_line(rng))
    for _ in range(300):
        n = rng.randint(0, 40)
        lines.append(bytes(rng.choice(b"C1234%[]()=cnN.#0@+") for _ in range(n)))
    for _ in range(200):
        lines.append(bytes(rng.randrange(256) for _ in range(rng.randint(0, 30))).replace(b"\n", b""))
    # generator lines (long fused chains exercise %nn ids)
    gen = make_corpus.MoleculeGen(random.Random(77), 0.5)
    for _ in range(300):
        lines.append(gen.molecule().encode())
    # many overlapping rings with mixed digits and %nn, forcing colours >= 10
    for k in (10, 11, 15, 25):
        ids = [str(i) for i in range(1, 10)] + [f"%{i:02d}" for i in range(10, 10 + k)]
        lines.append(("C" + "C".join(ids) + "C" + "C".join(ids[::-1]) + "C").encode())
        lines.append(("C" + "C".join(ids[::-1]) + "C" + "C".join(ids) + "C").encode())
    cases = []
    for ln in lines:
        cases.append({"line": H(ln), "strict": pp_result(ln, "strict"),
                      "lenient": pp_result(ln, "lenient")})
    return cases


# --------------------------------------------------------------------------
# stream (run_stream) fixtures
# --------------------------------------------------------------------------

def stream_result(payload, d, direction, **kw):
    dst = io.BytesIO()
    try:
        st = run_stream(io.BytesIO(payload), dst, d, direction, **kw)
    except z.LineError as e:
        return {"err": "LineError", "line_no": e.line_no,
                "cause": type(e.cause).__name__, "msg": str(e)}
    return {"out": H(dst.getvalue()), "lines": st.lines, "in_bytes": st.input_bytes,
            "out_bytes": st.output_bytes, "escapes": st.escapes,
            "skipped": st.skipped, "flagged": st.flagged}


def stream_cases():
    d_cc = z.Dictionary([b"CC"], "smiles")
    d_none = z.Dictionary([b"CC"], "none")
    d_def = z.deserialize(open(os.path.join(REF, "src/zsmiles/data/default.zsd"), "rb").read())
    payloads = [b"", b"\n", b"\n\n", b"CCO", b"CCO\n", b"CCO\nCC", b"CCO\n\nCC\n",
                b"\nCCO", b"CCO\n" * 25, b"CCO\nC1CC\nCCO\n", b"C1CC1\nC2CC\n",
                b"CCO\rX\n", b"CCO\rX\nCC\n", b"CC\r\nCC\r\n", b"\r", b"C1CC1\r",
                b"C3CCCCC3\nc9ccccc9O\n", b"C[NH\nC%1\nC1CC1\n", b"CC\nC1CC1\nC[\n",
                bytes([0x80]) + b"\n\x99\n", bytes([0x80]) + b"\n\x99\n" + bytes([0x80]) + b"\n",
                b"C \nCC\n", b" \n \n", b"CC\n\x20", b"\xff\x20\n"]
    lines = [b"CCO"] * 300 + [b"C1CC"] + [b"CCO"] * 50
    payloads.append(b"\n".join(lines) + b"\n")
    rng = random.Random(4004)
    for _ in range(12):
        n = rng.randint(0, 300)
        payloads.append(b"".join(zconf.smiles_like_line(rng) + b"\n" for _ in range(n)))
    gen = make_corpus.MoleculeGen(random.Random(55), 0.5)
    payloads.append("".join(gen.molecule() + "\n" for _ in range(500)).encode())
    payloads.append("".join(gen.molecule() + "\n" for _ in range(50)).encode()[:-1])
    cases = []
    for di, d in enumerate((d_cc, d_none, d_def)):
        for p in payloads:
            for direction in ("compress", "decompress"):
                for pre in ((False, True) if direction == "compress" else (False,)):
                    for lenient in (False, True):
                        res = stream_result(p, d, direction, preprocess=pre, lenient=lenient)
                        cases.append({"dict": di, "payload": H(p), "direction": direction,
                                      "preprocess": pre, "lenient": lenient, **res})
    # decompress of real compressed streams
    for di, d in enumerate((d_cc, d_none, d_def)):
        for p in payloads[-3:]:
            comp = io.BytesIO()
            run_stream(io.BytesIO(p), comp, d, "compress", preprocess=True, lenient=True)
            for lenient in (False, True):
                res = stream_result(comp.getvalue(), d, "decompress", lenient=lenient)
                cases.append({"dict": di, "payload": H(comp.getvalue()), "direction": "decompress",
                              "preprocess": False, "lenient": lenient, **res})
    return {"dicts": [dict_json(d) for d in (d_cc, d_none, d_def)], "cases": cases}


# --------------------------------------------------------------------------
# corpora
# --------------------------------------------------------------------------

def corpus_lines(kind, n, seed=2024):
    """Reference generator (scripts/make_corpus.py) for the SURVEY §8d configs."""
    if kind in ("mixed", "aromatic", "aliphatic"):
        frac = {"mixed": 0.5, "aromatic": 0.92, "aliphatic": 0.08}[kind]
        gen = make_corpus.MoleculeGen(random.Random(seed), frac)
        for _ in range(n):
            yield gen.molecule()
    elif kind == "skewed":
        # C3: join whole molecules with LINKERS up to a U[20,1000] target,
        # never exceeding 1000 bytes; each molecule restarts ring ids at 1.
        rng = random.Random(seed)
        gen = make_corpus.MoleculeGen(rng, 0.5)
        for _ in range(n):
            target = rng.randint(20, 1000)
            s = gen.molecule()
            while len(s) < target:
                nxt = rng.choice(make_corpus.LINKERS) + gen.molecule()
                if len(s) + len(nxt) > 1000:
                    break
                s += nxt
            yield s
    else:
        raise ValueError(kind)


def _compress_shard(args):
    payload, pre, dict_path = args
    d = z.load_dictionary(dict_path)
    dst = io.BytesIO()
    st = run_stream(io.BytesIO(payload), dst, d, "compress", preprocess=pre, lenient=True)
    return dst.getvalue(), st.escapes, st.flagged, st.skipped


def _decompress_shard(args):
    payload, dict_path = args
    d = z.load_dictionary(dict_path)
    dst = io.BytesIO()
    st = run_stream(io.BytesIO(payload), dst, d, "decompress")
    return dst.getvalue()


def corpus_entry(name, kind, n, seed, dict_path, pool, shard_lines=200_000):
    lines = [l.encode() + b"\n" for l in corpus_lines(kind, n, seed)]
    payload = b"".join(lines)
    entry = {"kind": kind, "lines": n, "seed": seed, "in_bytes": len(payload),
             "in_sha256": hashlib.sha256(payload).hexdigest(),
             "dict": os.path.basename(dict_path)}
    # sha of the first 10k lines pins the generator cheaply
    entry["head10k_sha256"] = hashlib.sha256(b"".join(lines[:10000])).hexdigest()
    shards = [b"".join(lines[i:i + shard_lines]) for i in range(0, n, shard_lines)]
    del lines
    for pre in (False, True):
        res = pool.map(_compress_shard, [(s, pre, dict_path) for s in shards])
        comp_parts = [r[0] for r in res]
        comp = b"".join(comp_parts)
        back = b"".join(pool.map(_decompress_shard, [(c, dict_path) for c in comp_parts]))
        key = "pre_on" if pre else "pre_off"
        entry[key] = {"out_bytes": len(comp), "comp_sha256": hashlib.sha256(comp).hexdigest(),
                      "escapes": sum(r[1] for r in res), "flagged": sum(r[2] for r in res),
                      "roundtrip_sha256": hashlib.sha256(back).hexdigest(),
                      "roundtrip_bytes": len(back)}
        print(f"  {name} {key}: {len(payload)} -> {len(comp)} B", flush=True)
    return entry


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also hash the 10M (C2) and 1M skewed corpora")
    ap.add_argument("--skip-small", action="store_true")
    ap.add_argument("--c3-5m", action="store_true", help="also hash the full 5M-line skewed corpus (C3)")
    args = ap.parse_args()

    ddir = os.path.join(HERE, "dicts")
    os.makedirs(ddir, exist_ok=True)
    shipped = open(os.path.join(REF, "src/zsmiles/data/default.zsd"), "rb").read()
    if not args.skip_small:
        # default dictionary: regenerate with the reference trainer and check
        mixed = [l.encode() for l in corpus_lines("mixed", 50000)]
        d = z.generate(mixed, GenerationParams(preprocess=True))
        assert z.serialize(d) == shipped, "default.zsd does not regenerate"
        with open(os.path.join(ddir, "default.zsd"), "wb") as fh:
            fh.write(z.serialize(d))
        # C4 ablation dictionaries
        for t in (16, 32, 64, 128):
            for lmax in (5, 8, 15):
                dd = z.generate(mixed, GenerationParams(t=t, l_max=lmax, preprocess=True))
                with open(os.path.join(ddir, f"t{t}_l{lmax}.zsd"), "wb") as fh:
                    fh.write(z.serialize(dd))
        print("wrote dictionaries", flush=True)

        dump("codec_cases.json", codec_cases())
        dump("decode_cases.json", decode_cases())
        dump("preprocess_cases.json", preprocess_cases())
        dump("stream_cases.json", stream_cases())

    hashes_path = os.path.join(HERE, "corpus_hashes.json")
    hashes = json.load(open(hashes_path)) if os.path.exists(hashes_path) else {}
    dpath = os.path.join(ddir, "default.zsd")
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        jobs = [("aromatic_10k", "aromatic", 10_000, 2024),
                ("aliphatic_10k", "aliphatic", 10_000, 2024),
                ("mixed_50k", "mixed", 50_000, 2024),
                ("c1_100k", "aromatic", 100_000, 2024),
                ("c3_skewed_20k", "skewed", 20_000, 2025)]
        if args.big:
            jobs += [("c2_10m", "aromatic", 10_000_000, 2024),
                     ("c3_skewed_1m", "skewed", 1_000_000, 2025)]
        if args.c3_5m:
            jobs += [("c3_skewed_5m", "skewed", 5_000_000, 2025)]
        for name, kind, n, seed in jobs:
            if name in hashes:
                continue
            print(f"corpus {name}", flush=True)
            hashes[name] = corpus_entry(name, kind, n, seed, dpath, pool)
            with open(hashes_path, "w") as fh:
                json.dump(hashes, fh, indent=1, sort_keys=True)
        # C4: ablation dictionaries on the 100k config
        for t in (16, 32, 64, 128):
            for lmax in (5, 8, 15):
                name = f"c4_100k_t{t}_l{lmax}"
                if name in hashes:
                    continue
                hashes[name] = corpus_entry(name, "aromatic", 100_000, 2024,
                                            os.path.join(ddir, f"t{t}_l{lmax}.zsd"), pool)
                with open(hashes_path, "w") as fh:
                    json.dump(hashes, fh, indent=1, sort_keys=True)
    print("done")


if __name__ == "__main__":
    main()
