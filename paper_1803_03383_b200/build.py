"""In-tree build of libhalp_b200.so (sm_100a only).

    python -m paper_1803_03383_b200.build [--force]

Compiles every CUDA source with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -Xptxas -v
(-fmad=false: the reference's element-wise arithmetic has no FMA; fused
multiply-adds appear only where the kernels write fma() explicitly), the
host driver with g++, and links a shared library next to this file so it
travels to the GPU box with the repo snapshot.  ptxas resource usage is
written to build/ptxas_<kernel>.log.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libhalp_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

# k_fullgrad_stream.cu is compiled as three translation units (one per element type) in parallel
CU_SOURCES = ["k_fullgrad.cu", "k_fullgrad_smx.cu", "k_fullgrad_stream_bf16.cu", "k_fullgrad_stream_f32.cu",
              "k_fullgrad_stream_f64.cu", "k_inner.cu", "k_batch.cu", "k_datagen.cu", "k_lm.cu"]
CXX_SOURCES = ["halp_capi.cpp", "halp_datasets.cpp"]
HEADERS = ["halp_device.cuh", "kernels.h", "rng_jump.hpp", "k_fullgrad_stream.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]
# developer variants only (tools/build_alt.sh), e.g. HALP_NVCC_DEFS="-DHALP_K3_PROF"
NVCC_FLAGS += os.environ.get("HALP_NVCC_DEFS", "").split()
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-I", os.path.join(CUDA, "include"),
             "-I", os.path.join(ROOT, "include")]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[-1]}")
    return r


def _flags_changed() -> bool:
    """True when the compiler flags (incl. HALP_NVCC_DEFS variants) differ from
    the ones the existing objects were built with (build/flags.stamp)."""
    stamp = os.path.join(BUILD, "flags.stamp")
    want = " ".join(NVCC_FLAGS) + "\n" + " ".join(CXX_FLAGS) + "\n"
    have = open(stamp).read() if os.path.exists(stamp) else ""
    if have != want:
        with open(stamp, "w") as f:
            f.write(want)
        return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    force = _flags_changed() or force
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "halp.h")]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append(([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o], os.path.join(BUILD, f"ptxas_{src}.log")))
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append((["g++"] + CXX_FLAGS + ["-c", s, "-o", o], None))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for f in [ex.submit(_run, c, l) for c, l in jobs]:
                f.result()
    if force or jobs or _newer(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static", "-ldl", "-lrt", "-lpthread"])
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
