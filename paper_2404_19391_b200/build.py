"""Build libzs.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a).

    python -m paper_2404_19391_b200.build [--force]
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "zs_api.cu")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("zs_api.cu", "zs_kernels.cuh", "zs_device.cuh", "zs_fx.cuh", "zs_cx.cuh", "zs_ix.cuh", "zs_train.cuh")] + \
       [os.path.join(ROOT, "include", "zs.h")]
OUT = os.path.join(HERE, "libzs.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177,550"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(OUT) or any(os.path.getmtime(d) > os.path.getmtime(OUT) for d in DEPS)
    if force or stale:
        cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT, SRC]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
