#!/usr/bin/env python3
"""Benchmark of the ZSMILES per-line codec hot path (BASELINE.json).

Workload (BASELINE.json configs[1], "C2"): 10M synthetic drug-like SMILES
(~460 MB, reference generator seed 2024, aromatic_frac 0.92), default fixed
dictionary, ring renumbering ON.  One *step* = compress the whole library
(preprocess + parse + emit, newline framing) and decompress the compressed
stream back, through the fused sm_100a tile kernels.

  value : round-trip input MB/s on HBM-resident buffers =
          N * input_bytes / (time of one compress + decompress step), the
          step timed with CUDA events on the library stream around whole
          device-API calls (memsets, kernels, result read-back), max over ranks
  e2e   : the same through the public host-buffer API (pinned host memory,
          H2D + kernels + D2H in the timed region)
  roofline : dominant kernel (compress_tiles_ip), algorithmic bytes =
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
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_LINES = 10_000_000
SEED = 2024
KIND = "aromatic"
METRIC = "input MB/s (device + end-to-end) for compress and decompress at 1/2/4/8 B200"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 5 ms) during the
    timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self.stop = threading.Event()
        self.t = None

    def _handle(self, nv):
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _run(self):
        import pynvml as nv
        nv.nvmlInit()
        h = self._handle(nv)
        self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self.stop.is_set():
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            for name, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
            self.stop.wait(0.005)
        nv.nvmlShutdown()

    def __enter__(self):
        try:
            import pynvml  # noqa: F401
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=5)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.mx or None, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


def traffic(kernel, lines):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed `ncu --set full` capture of this workload
    (profiles/ncu_traffic.json, written by tools/ncu_hot.py traffic), or
    None when no capture of this kernel at this size is committed."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        "ncu_traffic.json")
    try:
        with open(path) as fh:
            e = json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None
    if not e or e.get("lines") != lines:
        return None
    return int(e["dram_bytes"])


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


WORKLOAD = ("C2: 10M synthetic SMILES (reference generator, seed 2024, aromatic 0.92), default "
            "fixed dictionary, ring renumbering on, lenient")


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, ws, rank):
    """CPU reference arm: oracle port of the reference codec on host cores."""
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    synth.build()
    threads = host_threads()
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
           "config": {"workload": WORKLOAD, "lines_per_gpu": args.lines,
                      "parallelism": f"line-range shards x{ws}",
                      "sample_lines_per_step": sample_lines},
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
    threads = host_threads()
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
    ap.add_argument("--steps", type=int, default=50)
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

    names = ["", ""]

    def step_device():
        rc = ctx.lib.zs_compress_device(ctx.h, d_in.data_ptr(), n_in, d_comp.data_ptr(),
                                        d_comp.numel(), flags, res_c)
        ctx.check(rc, "zs_compress_device")
        kc = ctx.last_kernel_ms()
        names[0] = ctx.lib.zs_last_kernel(ctx.h).decode()
        rc = ctx.lib.zs_decompress_device(ctx.h, d_comp.data_ptr(), res_c.out_bytes,
                                          d_back.data_ptr(), d_back.numel(), 0, res_d)
        ctx.check(rc, "zs_decompress_device")
        kd = ctx.last_kernel_ms()
        names[1] = ctx.lib.zs_last_kernel(ctx.h).decode()
        return kc, kd

    for _ in range(args.warmup):
        step_device()
    comp_bytes = res_c.out_bytes
    # timed region: barrier + synchronize on both sides; CUDA events on the
    # library's stream bracket all K steps (whole calls: memsets, kernels,
    # result read-back), per-kernel events inside each call explain it.
    lib_stream = torch.cuda.ExternalStream(ctx.lib.zs_stream(ctx.h), device=f"cuda:{local}")
    ev_a = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    kc_ms, kd_ms = [], []
    launches = 0
    with ClockSampler(local) as clk:
        ev_a.record(lib_stream)
        for _ in range(args.steps):
            kc, kd = step_device()
            kc_ms.append(kc)
            kd_ms.append(kd)
            launches += res_c.gpu_launches + res_d.gpu_launches
        ev_b.record(lib_stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t_step = ev_a.elapsed_time(ev_b) / 1000.0 / args.steps
    tcs = sum(kc_ms) / 1000.0 / args.steps
    tds = sum(kd_ms) / 1000.0 / args.steps
    if dist:
        tt = torch.tensor([t_step, tcs, tds], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, tcs, tds = tt.tolist()
    k_comp, k_dec = names
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
        for _ in range(e2e_steps):
            step_host()
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
            "config": {"workload": WORKLOAD, "lines_per_gpu": args.lines, "input_bytes_per_gpu": n_in,
                       "compressed_bytes": comp_bytes, "ratio": round(comp_bytes / n_in, 6),
                       "l2": "inputs (460 MB) larger than L2 (126 MB); no flush needed",
                       "parallelism": f"line-range shards x{ws}"},
            "compress": {"device_MBps": round(n_in / tcs / 1e6, 3), "kernel_ms": round(tcs * 1000, 4)},
            "decompress": {"device_MBps_in": round(comp_bytes / tds / 1e6, 3),
                           "device_MBps_out": round(res_d.out_bytes / tds / 1e6, 3),
                           "kernel_ms": round(tds * 1000, 4),
                           "roofline": {"bound": "hbm", "achieved": round(ach_d, 2), "peak": peak,
                                        "unit": "GB/s", "frac": round(ach_d / peak, 4),
                                        "traffic": traffic(k_dec, args.lines), "kernel": k_dec}},
            "roofline": {"bound": "hbm", "achieved": round(ach_c, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(ach_c / peak, 4), "traffic": traffic(k_comp, args.lines),
                         "kernel": k_comp, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": int(alg_c),
                         "kernel_ms": round(tcs * 1000, 4),
                         "share_of_step": round(tcs / t_step, 4)},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "e2e": e2e,
        }
        if ws == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_sample(400_000)
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
