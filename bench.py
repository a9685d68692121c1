#!/usr/bin/env python3
"""Benchmark of the ZSMILES per-line codec hot path (BASELINE.json).

Workload (BASELINE.json configs[1], "C2"): 10M synthetic drug-like SMILES
(~460 MB, reference generator seed 2024, aromatic_frac 0.92), default fixed
dictionary, ring renumbering ON.  One *step* = compress the whole library
(preprocess + parse + emit, newline framing) and decompress the compressed
stream back, through the fused sm_100a tile kernels.

  value : round-trip input MB/s on HBM-resident buffers =
          N * input_bytes / (compress + decompress device time), max over ranks
  e2e   : the same through the public host-buffer API (pinned host memory,
          H2D + kernels + D2H in the timed region)
  roofline : dominant kernel (compress_tiles), algorithmic bytes =
          input bytes + compressed bytes (both incl. newlines) per launch
          over the CUDA-event kernel time, vs MEASURED_PEAKS.json hbm_gbs.

Multi-GPU (torchrun): each rank compresses/decompresses its own 10M-line
shard (weak scaling, lines are independent -- no data-path collective); the
only exchange is the max-over-ranks time and per-shard byte counts.

--impl reference: the CPU path (oracle port of the reference codec, all host
threads) on a bounded sample of the same workload.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_LINES = 10_000_000
SEED = 2024
KIND = "aromatic"
METRIC = "round-trip (compress+decompress) input MB/s, 10M SMILES C2, ring renumbering on"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args, ws, rank):
    """CPU reference arm: oracle port of the reference codec on host cores."""
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    synth.build()
    threads = os.cpu_count() or 1
    sample_lines = args.ref_lines
    buf = synth.generate(KIND, sample_lines, SEED)
    with open(os.path.join(ROOT, "paper_2404_19391_b200", "data", "default.zsd"), "rb") as fh:
        t = oracle.Tables.from_zsd(fh.read())
    for _ in range(args.warmup):
        comp, _ = oracle.run_stream(t, buf, "compress", True, True, threads)
        oracle.run_stream(t, comp, "decompress", False, False, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        comp, _ = oracle.run_stream(t, buf, "compress", True, True, threads)
        oracle.run_stream(t, comp, "decompress", False, False, threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    v = buf.size * args.steps / tot / 1e6
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "MB/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(1000 * tot / args.steps, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
           "config": {"workload": "C2 10M SMILES (bounded sample per step)", "sample_lines": sample_lines,
                      "preprocess": True, "dictionary": "default.zsd"},
           "cpu_baseline": {"value": round(v, 3), "unit": "MB/s", "cores": threads, "kind": "port",
                            "sample": f"first {sample_lines} lines of C2 ({buf.size} B), "
                                      "compress(preprocess on)+decompress per step"},
           "e2e": {"value": round(v, 3), "unit": "MB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline_sample(n_lines):
    """Oracle timed on a bounded sample (rank 0, N=1)."""
    import oracle
    import synth
    oracle.build()
    threads = os.cpu_count() or 1
    buf = synth.generate(KIND, n_lines, SEED)
    with open(os.path.join(ROOT, "paper_2404_19391_b200", "data", "default.zsd"), "rb") as fh:
        t = oracle.Tables.from_zsd(fh.read())
    comp, _ = oracle.run_stream(t, buf, "compress", True, True, threads)
    t0 = time.perf_counter()
    reps = 0
    while True:
        comp, _ = oracle.run_stream(t, buf, "compress", True, True, threads)
        oracle.run_stream(t, comp, "decompress", False, False, threads)
        reps += 1
        if time.perf_counter() - t0 > 10.0:
            break
    dt = time.perf_counter() - t0
    return {"value": round(buf.size * reps / dt / 1e6, 3), "unit": "MB/s", "cores": threads,
            "kind": "port", "sample": f"first {n_lines} lines of C2 ({buf.size} B), "
                                      f"round trip x{reps} in {dt:.1f}s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lines", type=int, default=N_LINES)
    ap.add_argument("--ref-lines", type=int, default=400_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_env()

    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch
    import synth
    import paper_2404_19391_b200 as z
    from paper_2404_19391_b200 import _lib
    from paper_2404_19391_b200 import build as zbuild

    zbuild.build()
    synth.build()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    d = z.default_dictionary()
    buf = synth.generate(KIND, args.lines, SEED)
    n_in = buf.size
    ctx = _lib.context(local)
    ctx.set_dictionary(d)
    flags = _lib.F_PREPROCESS | _lib.F_LENIENT

    # device-resident buffers
    d_in = torch.from_numpy(buf).to(f"cuda:{local}")
    d_comp = torch.empty(2 * n_in + 64, dtype=torch.uint8, device=f"cuda:{local}")
    d_back = torch.empty(n_in + 64, dtype=torch.uint8, device=f"cuda:{local}")
    res_c, res_d = _lib.Result(), _lib.Result()

    def step_device():
        rc = ctx.lib.zs_compress_device(ctx.h, d_in.data_ptr(), n_in, d_comp.data_ptr(),
                                        d_comp.numel(), flags, res_c)
        ctx.check(rc, "zs_compress_device")
        kc = ctx.last_kernel_ms()
        rc = ctx.lib.zs_decompress_device(ctx.h, d_comp.data_ptr(), res_c.out_bytes,
                                          d_back.data_ptr(), d_back.numel(), 0, res_d)
        ctx.check(rc, "zs_decompress_device")
        kd = ctx.last_kernel_ms()
        return kc, kd

    for _ in range(args.warmup):
        step_device()
    comp_bytes = res_c.out_bytes
    # timed region: CUDA events on the library stream (kernel launches)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    kc_ms, kd_ms = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            kc, kd = step_device()
            kc_ms.append(kc)
            kd_ms.append(kd)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t_c = sum(kc_ms) / 1000.0
    t_d = sum(kd_ms) / 1000.0
    t_step = (t_c + t_d) / args.steps
    if dist:
        tt = torch.tensor([t_step, t_c / args.steps, t_d / args.steps], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, tcs, tds = tt.tolist()
    else:
        tcs, tds = t_c / args.steps, t_d / args.steps
    value = ws * n_in / t_step / 1e6

    # end-to-end through the public host API (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        h_in = torch.from_numpy(buf).pin_memory()
        h_comp = torch.empty(2 * n_in + 64, dtype=torch.uint8).pin_memory()
        h_back = torch.empty(n_in + 64, dtype=torch.uint8).pin_memory()
        rc_, rd_ = _lib.Result(), _lib.Result()

        def step_host():
            rc = ctx.lib.zs_compress_host(ctx.h, h_in.data_ptr(), n_in, h_comp.data_ptr(),
                                          h_comp.numel(), flags, rc_)
            ctx.check(rc, "zs_compress_host")
            rc = ctx.lib.zs_decompress_host(ctx.h, h_comp.data_ptr(), rc_.out_bytes,
                                            h_back.data_ptr(), h_back.numel(), 0, rd_)
            ctx.check(rc, "zs_decompress_host")

        for _ in range(max(1, args.warmup // 2)):
            step_host()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_steps = max(2, args.steps // 2)
        launches = 0
        for _ in range(e2e_steps):
            step_host()
            launches += rc_.gpu_launches + rd_.gpu_launches
        te = (time.perf_counter() - t0) / e2e_steps
        if dist:
            tt = torch.tensor([te], device=f"cuda:{local}")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = tt.item()
        ok = bytes(h_back[:rd_.out_bytes].numpy()) == bytes(
            z.run_buffer(h_comp[:rc_.out_bytes].numpy(), d, "decompress")[0])
        e2e = {"value": round(ws * n_in / te / 1e6, 3), "unit": "MB/s",
               "h2d_bytes_per_step": int(n_in + rc_.out_bytes),
               "d2h_bytes_per_step": int(rc_.out_bytes + rd_.out_bytes),
               "ms_per_step": round(te * 1000, 3), "roundtrip_consistent": ok}

    if rank == 0:
        peak, peak_kind = peaks()
        alg_c = n_in + comp_bytes
        alg_d = comp_bytes + res_d.out_bytes
        ach_c = alg_c / tcs / 1e9
        ach_d = alg_d / tds / 1e9
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "MB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1000, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": "C2: 10M synthetic SMILES (reference generator, seed 2024, "
                                   "aromatic 0.92), default fixed dictionary, ring renumbering on, "
                                   "lenient", "lines_per_gpu": args.lines, "input_bytes_per_gpu": n_in,
                       "compressed_bytes": comp_bytes, "ratio": round(comp_bytes / n_in, 6),
                       "l2": "inputs (460 MB) larger than L2 (126 MB); no flush needed",
                       "parallelism": f"line-range shards x{ws}"},
            "compress": {"device_MBps": round(n_in / tcs / 1e6, 3), "kernel_ms": round(tcs * 1000, 4)},
            "decompress": {"device_MBps_in": round(comp_bytes / tds / 1e6, 3),
                           "device_MBps_out": round(res_d.out_bytes / tds / 1e6, 3),
                           "kernel_ms": round(tds * 1000, 4),
                           "roofline": {"bound": "hbm", "achieved": round(ach_d, 2), "peak": peak,
                                        "unit": "GB/s", "frac": round(ach_d / peak, 4)}},
            "roofline": {"bound": "hbm", "achieved": round(ach_c, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(ach_c / peak, 4), "traffic": None,
                         "kernel": "compress_tiles<6>", "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": int(alg_c)},
            "clocks": clk.summary(),
            "gpu_launches": 2 * args.steps,
            "e2e": e2e,
        }
        if ws == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_sample(400_000)
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
