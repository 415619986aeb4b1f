"""Build the native library in-tree: paper_2510_20071_b200/_lib/libfibar_b200.so.

    python -m paper_2510_20071_b200.build

nvcc cross-compiles for sm_100a without a GPU.  -lineinfo keeps the ncu source
view mapped to csrc/; no --use_fast_math (the float32 path must stay strict
IEEE, see csrc/fibar_common.cuh).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", f) for f in ("fibar_engine.cu", "fibar_front.cu", "fibar_stage.cu", "fibar_readout.cu", "fibar_sort.cu",
                                                  "fibar_tools.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in ("fibar_common.cuh", "fibar_internal.h", "fibar_kernels.cuh")] + [
    os.path.join(HERE, "..", "include", "fibar_b200.h")]
OUT = os.path.join(HERE, "_lib", "libfibar_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = [f"-D{d}" for d in os.environ.get("FIBAR_DEFINES", "").split(",") if d] + os.environ.get("FIBAR_NVCC_FLAGS", "").split()


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", *EXTRA, "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(HERE, "..", "include"), "-o", OUT + ".tmp", *SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
