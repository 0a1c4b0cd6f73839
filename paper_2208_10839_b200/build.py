"""In-tree build of libsonarnet_b200.so (sm_100a) — no JIT cache, no pip install.

    python -m paper_2208_10839_b200.build      # or __graft_entry__.build()

Host setup code (csrc/plan.cpp) is compiled with -ffp-contract=off so the
FP64 tables match the reference's doubles bit for bit (the oracle is built
with the same pin, oracle/Makefile). Device code: -gencode
arch=compute_100a,code=sm_100a -lineinfo. The .so lands in
paper_2208_10839_b200/_lib/ (git-ignored; shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_lib")
OBJ = os.path.join(OUT, "obj")
SO = os.path.join(OUT, "libsonarnet_b200.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
CUDA_INC = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(NVCC))), "include")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                     "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v"]

CU_SOURCES = ["kernels.cu", "beamform_tc.cu", "frames.cu", "synth.cu", "sn_api.cu"]
CPP_SOURCES = ["plan.cpp", "cluster.cpp", "pool.cpp", "gather.cpp"]
HEADERS = ["fft.cuh", "kernels.cuh", "plan.hpp"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd, log):
    res = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    log.write(" ".join(cmd) + "\n" + res.stdout + "\n")
    if res.returncode != 0:
        sys.stderr.write(res.stdout)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    return res.stdout


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "sonarnet_b200.h")]
    objs = []
    with open(os.path.join(OUT, "build.log"), "w") as log:
        for src in CPP_SOURCES:
            s = os.path.join(CSRC, src)
            o = os.path.join(OBJ, src + ".o")
            if _newer(o, [s] + hdr + [__file__]):
                _run([CXX, *HOST_FLAGS, "-I", INCLUDE, "-I", CSRC, "-I", CUDA_INC, "-c", s, "-o", o], log)
            objs.append(o)
        for src in CU_SOURCES:
            s = os.path.join(CSRC, src)
            o = os.path.join(OBJ, src + ".o")
            if _newer(o, [s] + hdr + [__file__]):
                out = _run([NVCC, *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o], log)
                if verbose:
                    print(out)
            objs.append(o)
        if _newer(SO, objs):
            _run([NVCC, *ARCH, "-shared", "-o", SO, *objs, "-lpthread", "-ldl"], log)
    return SO


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
