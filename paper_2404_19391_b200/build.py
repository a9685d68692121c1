"""Build libzs.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a).

    python -m paper_2404_19391_b200.build [--force]
"""

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "zs_api.cu")
# every source and header of the library (a new header is a dependency without listing it)
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) +
              glob.glob(os.path.join(ROOT, "include", "*.h")))
OUT = os.path.join(HERE, "libzs.so")
# measurement build: per-phase clocks compiled in (tools/phase_cx.py loads it via ZS_LIB)
OUT_PHASES = os.path.join(HERE, "libzs_phases.so")
# debug build: device-side bounds asserts (ZS_CHECKS)
OUT_CHECKS = os.path.join(HERE, "libzs_checks.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177,550"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, phases: bool = False, checks: bool = False) -> str:
    out = OUT_PHASES if phases else OUT_CHECKS if checks else OUT
    stale = not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in DEPS)
    if force or stale:
        cmd = [nvcc(), *NVCC_FLAGS, *(["-DZS_PHASES=1"] if phases else []), *(["-DZS_CHECKS=1"] if checks else []), "-o", out, SRC]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, phases="--phases" in sys.argv,
                checks="--checks" in sys.argv))
