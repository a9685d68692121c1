"""Multi-rank sharding (paper_2404_19391_b200/shard.py).

The per-shard codec here is the oracle (test infrastructure); the GPU codec
goes through the same shard protocol in tests/test_gpu_parity.py.  The claim
checked: splitting a library at newline boundaries across any number of
ranks, running each shard independently and exchanging 4 scalars per shard
reproduces the whole-buffer stream byte for byte, with the same totals and
the same global 1-based first-error line."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import synth
from conftest import golden_dict_bytes
from paper_2404_19391_b200 import shard


def oracle_codec(t, direction, pre, lenient):
    def fn(sh):
        out, st = oracle.run_stream(t, np.ascontiguousarray(sh), direction, pre, lenient, 2)
        return shard.normalise(sh, out or b"", st["lines"], st["err_line"])
    return fn


def simulate(buf, fn, world):
    """All ranks in one process: same cuts, same combine, no transport."""
    arr = np.frombuffer(buf, np.uint8)
    cuts = shard.shard_bounds(arr, world)
    outs, res = [], []
    for r in range(world):
        o, s = fn(arr[cuts[r]:cuts[r + 1]])
        outs.append(o)
        res.append(s)
    trailing = arr.size == 0 or arr[-1] == 0x0A
    views = [shard.combine(res, r, trailing) for r in range(world)]
    blob = b"".join(o[:v.out_bytes] for o, v in zip(outs, views))
    for r, v in enumerate(views):
        assert v.out_offset == sum(x.out_bytes for x in views[:r])
    return blob, views[0]


def test_bounds_are_newline_aligned():
    rng = np.random.default_rng(3)
    for n in (0, 1, 5, 97, 4000):
        arr = rng.choice(np.frombuffer(b"CC(\n", np.uint8), n).astype(np.uint8)
        for world in (1, 2, 3, 8, 13):
            cuts = shard.shard_bounds(arr, world)
            assert cuts[0] == 0 and cuts[-1] == n and len(cuts) == world + 1
            assert all(a <= b for a, b in zip(cuts, cuts[1:]))
            for c in cuts[1:-1]:
                assert c in (0, n) or arr[c - 1] == 0x0A


@pytest.mark.parametrize("world", [2, 3, 5])
def test_stream_cases_sharded(stream_cases, world):
    """Every reference stream case (framing, CR policy, strict / lenient,
    decode errors) sharded `world` ways == the reference's own output."""
    tabs = [oracle.Tables.from_json(d) for d in stream_cases["dicts"]]
    for c in stream_cases["cases"]:
        payload = bytes.fromhex(c["payload"])
        fn = oracle_codec(tabs[c["dict"]], c["direction"], c["preprocess"], c["lenient"])
        blob, v = simulate(payload, fn, world)
        if "err" in c:
            assert v.err_line == c["line_no"], c
        else:
            assert v.err_line == 0
            assert blob.hex() == c["out"], (world, c)
            assert v.total_out == c["out_bytes"] and v.total_lines == c["lines"]


@pytest.mark.parametrize("world", [1, 2, 4, 7])
def test_corpus_sharded(world):
    t = oracle.Tables.from_zsd(golden_dict_bytes())
    buf = synth.generate("skewed", 3000, 2025).tobytes()
    buf = buf[:-1]  # no trailing newline: the last kept record loses its '\n'
    want, st = oracle.run_stream(t, buf, "compress", True, True, 4)
    blob, v = simulate(buf, oracle_codec(t, "compress", True, True), world)
    assert blob == want and v.total_out == st["out_bytes"] and v.total_lines == st["lines"]
    back, _ = oracle.run_stream(t, want, "decompress", False, False, 4)
    blob2, _ = simulate(want, oracle_codec(t, "decompress", False, False), world)
    assert blob2 == back


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, buf, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = oracle.Tables.from_zsd(golden_dict_bytes())
        out, v = shard.run_sharded(buf, oracle_codec(t, "compress", True, False), rank, world)
        q.put((rank, out, v.out_offset, v.total_out, v.total_lines, v.err_line))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bad_line", [0, 1900])
def test_gloo_two_ranks(bad_line):
    """world_size 2 over gloo: the all-gather of shard scalars gives each rank
    its output offset and the global first-error line."""
    lines = synth.generate("mixed", 3000, 2024).tobytes().split(b"\n")[:-1]
    if bad_line:
        lines[bad_line - 1] = b"C1CC[N"  # unclosed bracket on a line in rank 1's shard
    buf = b"\n".join(lines) + b"\n"
    t = oracle.Tables.from_zsd(golden_dict_bytes())
    want, st = oracle.run_stream(t, buf, "compress", True, False, 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, buf, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    if bad_line:
        assert all(g[5] == bad_line == st["err_line"] for g in got)
        return
    assert got[1][2] == len(got[0][1])
    assert got[0][1] + got[1][1] == want
    assert all(g[3] == len(want) and g[4] == st["lines"] for g in got)
