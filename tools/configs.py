"""Every BASELINE.json config on one B200 (device API, HBM-resident buffers;
CUDA-event kernel times from the library's stream), one JSON line each:

  C1  100k synthetic drug-like lines (aromatic 0.92, seed 2024)
  C2  10M lines (the bench workload)
  C3  skewed library, 5M lines of 20-1000 chars (seed 2025)
  C4  ablation: renumbering off/on x the 12 trained dictionaries
      (t in {16,32,64,128} x lmax in {5,8,15}) on C2's first 2M lines
  C5  1B lines: C2's 10M lines tiled 100x (~46 GB) resident in HBM, compressed
      and decompressed as 100 device calls; output checked against 100x
      the 10M-line output (lines are independent)
  RA  random access: RecordIndex over C2's compressed stream, 1M random records

    python tools/configs.py [--skip c5]
"""
import argparse
import ctypes
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2404_19391_b200 as z  # noqa: E402
from paper_2404_19391_b200 import _lib  # noqa: E402

FL = _lib.F_PREPROCESS | _lib.F_LENIENT


def hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth), else the
    profiling recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0


PEAK = hbm_peak()


def dev_round_trip(ctx, d, din, n, flags, reps=3):
    dc = torch.empty(2 * n + 64, dtype=torch.uint8, device="cuda")
    db = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    rc_, rd_ = _lib.Result(), _lib.Result()
    tc = td = 1e30
    for _ in range(reps):
        ctx.check(ctx.lib.zs_compress_device(ctx.h, din.data_ptr(), n, dc.data_ptr(), dc.numel(), flags, rc_), "c")
        tc = min(tc, ctx.last_kernel_ms())
        kc = ctx.lib.zs_last_kernel(ctx.h).decode()
        ctx.check(ctx.lib.zs_decompress_device(ctx.h, dc.data_ptr(), rc_.out_bytes, db.data_ptr(), db.numel(), 0,
                                               rd_), "d")
        td = min(td, ctx.last_kernel_ms())
        kd = ctx.lib.zs_last_kernel(ctx.h).decode()
    ok = rd_.out_bytes == n and bool(torch.equal(db[:n], din[:n])) if flags == _lib.F_LENIENT else None
    return rc_, rd_, tc, td, kc, kd, dc, ok


def line(cfg, n, rc_, tc, td, kc, kd, extra=None):
    alg = n + rc_.out_bytes
    o = {"config": cfg, "input_bytes": int(n), "compressed_bytes": int(rc_.out_bytes),
         "ratio": round(rc_.out_bytes / max(1, n), 6), "compress_ms": round(tc, 4),
         "compress_GBps_in": round(n / tc / 1e6, 2), "compress_roofline_frac": round(alg / tc / 1e6 / PEAK, 4),
         "decompress_ms": round(td, 4), "decompress_GBps_out": round(n / td / 1e6, 2),
         "decompress_roofline_frac": round(alg / td / 1e6 / PEAK, 4), "kernels": [kc, kd]}
    if extra:
        o.update(extra)
    print(json.dumps(o), flush=True)
    return o


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip", default="")
    args = ap.parse_args()
    skip = set(args.skip.split(","))
    ctx = _lib.context()
    d = z.default_dictionary()
    ctx.set_dictionary(d)
    out = []
    c2 = synth.generate("aromatic", 10_000_000, 2024)
    for cfg, buf in (("C1 100k aromatic", c2[:int(np.flatnonzero(c2 == 10)[99_999]) + 1]),
                     ("C2 10M aromatic", c2)):
        din = torch.from_numpy(buf).cuda()
        rc_, rd_, tc, td, kc, kd, _, _ = dev_round_trip(ctx, d, din, buf.size, FL)
        out.append(line(cfg, buf.size, rc_, tc, td, kc, kd, {"lines": int(rc_.lines)}))
    if "c3" not in skip:
        sk = synth.generate("skewed", 5_000_000, 2025)
        din = torch.from_numpy(sk).cuda()
        rc_, rd_, tc, td, kc, kd, _, _ = dev_round_trip(ctx, d, din, sk.size, FL)
        out.append(line("C3 skewed 5M (20-1000 chars)", sk.size, rc_, tc, td, kc, kd, {"lines": int(rc_.lines)}))
        del din
    if "c4" not in skip:
        sub = c2[:int(np.flatnonzero(c2 == 10)[1_999_999]) + 1]
        din = torch.from_numpy(sub).cuda()
        for name in ["default"] + [f"t{t}_l{l}" for t in (16, 32, 64, 128) for l in (5, 8, 15)]:
            with open(os.path.join(ROOT, "tests", "golden", "dicts", f"{name}.zsd"), "rb") as fh:
                dd = z.deserialize(fh.read())
            ctx.set_dictionary(dd)
            for pre in (0, _lib.F_PREPROCESS):
                rc_, rd_, tc, td, kc, kd, _, _ = dev_round_trip(ctx, dd, din, sub.size, pre | _lib.F_LENIENT)
                out.append(line(f"C4 {name} renumber={'on' if pre else 'off'} 2M", sub.size, rc_, tc, td, kc, kd))
        ctx.set_dictionary(d)
        del din
    if "ra" not in skip:
        din = torch.from_numpy(c2).cuda()
        rc_, rd_, tc, td, kc, kd, dc, _ = dev_round_trip(ctx, d, din, c2.size, FL, reps=1)
        comp = dc[:rc_.out_bytes].clone()
        t0 = time.perf_counter()
        ix = z.RecordIndex(comp, d)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        rng = np.random.default_rng(7)
        sel = rng.integers(0, len(ix), 1_000_000)
        ix.decode(sel[:1000])
        ix.decode_packed(sel)  # first call at this size allocates its device buffers
        t0 = time.perf_counter()
        data, offs = ix.decode_packed(sel)
        tpk = time.perf_counter() - t0
        t0 = time.perf_counter()
        got = ix.decode(sel)
        tdx = time.perf_counter() - t0
        assert data.tobytes() == b"".join(got)
        lines = c2.tobytes().split(b"\n")
        # renumbering changes lines; compare against the decoded stream instead
        back = z.run_buffer(comp.cpu().numpy(), d, "decompress")[0].tobytes().split(b"\n")
        assert all(got[i] == back[sel[i]] for i in range(0, 1_000_000, 997))
        o = {"config": "RA random access, C2 compressed, 1M random records", "records": len(ix),
             "index_build_ms": round(tb * 1e3, 3), "decode_packed_1M_ms_host_wall": round(tpk * 1e3, 3),
             "records_per_s_packed": round(1e6 / tpk), "decode_1M_ms_host_wall_list": round(tdx * 1e3, 3),
             "records_per_s_list": round(1e6 / tdx)}
        print(json.dumps(o), flush=True)
        out.append(o)
        del din, lines
    if "c5" not in skip:
        reps = 100
        n1 = c2.size
        big = torch.empty(n1 * reps, dtype=torch.uint8, device="cuda")
        one = torch.from_numpy(c2).cuda()
        for r in range(reps):
            big[r * n1:(r + 1) * n1].copy_(one)
        del one
        rc1 = _lib.Result()
        dc = torch.empty(2 * n1 + 64, dtype=torch.uint8, device="cuda")
        ctx.check(ctx.lib.zs_compress_device(ctx.h, big.data_ptr(), n1, dc.data_ptr(), dc.numel(), FL, rc1), "c")
        want = hashlib.sha256(dc[:rc1.out_bytes].cpu().numpy().tobytes()).hexdigest()
        cs = (rc1.out_bytes + 15) & ~15  # 16-byte aligned chunk stride (vector loads)
        cbig = torch.empty(cs * reps + 64, dtype=torch.uint8, device="cuda")
        bbig = torch.empty(n1 + 64, dtype=torch.uint8, device="cuda")
        res = _lib.Result()
        tc = td = 0.0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for r in range(reps):
            ctx.check(ctx.lib.zs_compress_device(ctx.h, big.data_ptr() + r * n1, n1, cbig.data_ptr() + r * cs,
                                                 cs, FL, res), "c")
            tc += ctx.last_kernel_ms()
        for r in range(reps):
            ctx.check(ctx.lib.zs_decompress_device(ctx.h, cbig.data_ptr() + r * cs, rc1.out_bytes,
                                                   bbig.data_ptr(), bbig.numel(), 0, res), "d")
            td += ctx.last_kernel_ms()
        wall = time.perf_counter() - t0
        ok = all(hashlib.sha256(cbig[r * cs:r * cs + rc1.out_bytes].cpu().numpy().tobytes()).hexdigest()
                 == want for r in (0, reps // 2, reps - 1))
        o = {"config": "C5 1B lines (C2 x100, 46 GB in HBM), 100 device calls", "input_bytes": n1 * reps,
             "compressed_bytes": rc1.out_bytes * reps, "compress_ms": round(tc, 2),
             "compress_GBps_in": round(n1 * reps / tc / 1e6, 2), "decompress_ms": round(td, 2),
             "decompress_GBps_out": round(n1 * reps / td / 1e6, 2), "wall_s": round(wall, 2),
             "sample_chunks_match_10M_output": ok}
        print(json.dumps(o), flush=True)
        out.append(o)
    with open(os.path.join(ROOT, "gpurun_out", "configs.json"), "w") as fh:
        for o in out:
            fh.write(json.dumps(o) + "\n")


if __name__ == "__main__":
    main()
