"""In-tree build of the CUDA library (nvcc, sm_100a).

``python -m paper_2003_09133_b200.build`` or ``__graft_entry__.build()``.
The output ``paper_2003_09133_b200/libhprime.so`` is git-ignored but travels
with the repo snapshot to the GPU box.  The oracle (``oracle/``) is numpy
test infrastructure: the reference is pure Python, so there is no C oracle
or compiled reference (``oracle/_ref``) to build.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhprime.so")
SOURCES = [os.path.join(CSRC, "lfbp_capi.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("hprime_kernel.cuh", "hprime_plan.h", "plane_sums.cuh",
                                                 "lf5_stream.inc", "projector.cuh",
                                                 "host_pipeline.inc", "verify_capi.inc", "projector_capi.inc",
                                                 "synth.cuh")] + [
    os.path.join(ROOT, "include", "lfbp_hprime.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC", "-cudart", "static",
]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_native(force: bool = False, verbose: bool = False) -> str:
    if force or _stale(LIB, DEPS):
        tmp = LIB + ".tmp"
        cmd = [NVCC, *NVCC_FLAGS, "-o", tmp, *SOURCES]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed ({r.returncode}):\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
        with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
            f.write(r.stderr)
        if verbose:
            print(r.stderr, file=sys.stderr)
    return LIB


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
