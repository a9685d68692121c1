"""Key ncu --set full metrics of a report (one kernel), one per line.

    python tools/ncu_summary.py report.ncu-rep
"""
import csv
import subprocess
import sys

KEEP = {
    "GPU Speed Of Light Throughput": ["Duration", "DRAM Throughput", "Memory Throughput",
                                      "L1/TEX Cache Throughput", "L2 Cache Throughput",
                                      "Compute (SM) Throughput", "SM Frequency"],
    "Compute Workload Analysis": ["Executed Ipc Active", "Issue Slots Busy"],
    "Memory Workload Analysis": ["Memory Throughput", "Mem Busy", "Max Bandwidth", "L1/TEX Hit Rate",
                                 "L2 Hit Rate", "Mem Pipes Busy"],
    "Scheduler Statistics": ["Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
                             "No Eligible"],
    "Warp State Statistics": ["Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp"],
    "Instruction Statistics": ["Executed Instructions"],
    "Occupancy": ["Achieved Occupancy", "Theoretical Occupancy", "Block Limit Registers",
                  "Block Limit Shared Mem"],
    "Launch Statistics": ["Grid Size", "Block Size", "Registers Per Thread",
                          "Dynamic Shared Memory Per Block"],
}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, si, mi, ui, vi = (hdr.index(h) for h in ("Kernel Name", "Section Name", "Metric Name",
                                                  "Metric Unit", "Metric Value"))
    name = None
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if r[ki] != name:
            name = r[ki]
            print(f"# kernel {name}")
        if r[mi] in KEEP.get(r[si], []):
            print(f"{r[si][:26]:26s} {r[mi]:38s} {r[vi]:>16s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        h = rr[0]
        for col in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if col in h:
                print(f"{'raw':26s} {col:38s} {rr[2][h.index(col)]:>16s} {rr[1][h.index(col)]}")


if __name__ == "__main__":
    main()
