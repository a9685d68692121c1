"""Copy a round's GPU evidence from gpurun_out/ into profiles/<round>/:
bench lines, the ncu launch list (per-kernel totals and share), ncu --set full
summaries of the hot kernels, and profiles/ncu_traffic.json (DRAM bytes per
launch, read by bench.py for roofline.traffic).

    python tools/collect_profiles.py r01
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def launches(dst):
    lines = [l for l in open(os.path.join(OUT, "launches.csv")).read().splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = {}
    with open(os.path.join(dst, "launches.csv"), "w") as fh:
        fh.write("id,kernel,grid,block,gpu_time_ns\n")
        for r in rows:
            k = r["Kernel Name"].split("(")[0].replace("void ", "")
            fh.write(f"{r['ID']},{k},\"{r['Grid Size']}\",\"{r['Block Size']}\",{r['Metric Value']}\n")
            tot.setdefault(k, []).append(int(r["Metric Value"]))
    s = sum(sum(v) for v in tot.values())
    with open(os.path.join(dst, "launches_summary.txt"), "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        fh.write("python bench.py --steps 3 --warmup 3 --no-cpu-baseline  (C2, 10M lines)\n\n")
        for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
            fh.write(f"{k:28s} launches={len(v):3d} avg={sum(v) / len(v) / 1e3:9.1f} us  share={sum(v) / s:.3f}\n")
    print(open(os.path.join(dst, "launches_summary.txt")).read())


def full(rep, dst, name):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "30"],
                         capture_output=True, text=True).stdout
    phases = ""
    if name == "compress":  # per-phase instruction accounting (source-line ranges of zs_cx.cuh)
        phases = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "phase_ranges.py"), rep],
                                capture_output=True, text=True).stdout
    with open(os.path.join(dst, f"ncu_{name}.txt"), "w") as fh:
        fh.write(txt + "\n" + phases + "\n" + hot)
    print(txt)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        k = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
        scale = lambda col: float(r[h.index(col)]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[
            units[h.index(col)]]
        res[k] = int(scale("dram__bytes_read.sum") + scale("dram__bytes_write.sum"))
    return res


def main():
    rnd = sys.argv[1]
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    for f in ("bench.json", "bench_ref.json", "bench_c5.json", "gpu_tests.log", "smoke.log", "configs.json",
              "train.json", "ll_check.log"):
        if os.path.exists(os.path.join(OUT, f)):
            shutil.copy(os.path.join(OUT, f), os.path.join(dst, f))
    launches(dst)
    traffic = {}
    for rep, name in (("full_compress.ncu-rep", "compress"), ("full_decompress.ncu-rep", "decompress")):
        p = os.path.join(OUT, rep)
        if os.path.exists(p):
            traffic.update(full(p, dst, name))
    lines = 10_000_000
    tj = {}
    for k, v in traffic.items():
        tj[k] = {"lines": lines, "dram_bytes": v}
    if "fx_count" in traffic and "fx_emit" in traffic:
        tj["fx_count+fx_scan+fx_emit"] = {"lines": lines, "dram_bytes": traffic["fx_count"] + traffic["fx_emit"]}
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(tj, fh, indent=1)
    print(json.dumps(tj, indent=1))


if __name__ == "__main__":
    main()
