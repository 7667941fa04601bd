"""Build libbimine_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libbimine_b200.so")
SOURCES = ["bm_lib.cu", "bm_ingest.cpp", "bm_synth.cpp"]
HEADERS = ["bm_kernels.cu", "bm_ring.cu", "bm_band.cu", "bm_seq.cu", "bm_merge.cu", "bm_api.cu", "bm_device.cuh", "bm_kernels.cuh", "glibc_exp.cuh", "glibc_exp_table.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--extended-lambda",
    # bit-exactness: never contract a*b+c into an FMA behind our back
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(INCLUDE, h) for h in ("bimine_b200.h", "bimine_synth.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    table = os.path.join(CSRC, "glibc_exp_table.h")
    if not os.path.exists(table):
        subprocess.check_call(["python", os.path.join(CSRC, "gen_exp_table.py")])
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}",
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
