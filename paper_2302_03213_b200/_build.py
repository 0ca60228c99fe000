"""Build the sm_100a shared library in-tree: paper_2302_03213_b200/_lib/liblutgpu.so.

Plain nvcc (no torch extension machinery): the library exposes only the
C ABI of include/lutgpu.h and is loaded with ctypes.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "liblutgpu.so")
SOURCES = ["capi.cu", "encode.cu", "encode_tc.cu", "encode_conv_tc.cu", "encode_conv_strip.cu", "gather.cu", "onehot.cu", "onehot_stream.cu", "table.cu"]
HEADERS = ["common.cuh", "onehot_dev.cuh", "encode_dev.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


if os.environ.get("LUTGPU_BUILD_PROBES") == "1":  # compile in the pair-gather timeline / role probes
    NVCC_FLAGS.append("-DLUTGPU_PROBES")


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "lutgpu.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    """Compile stale objects (in parallel; an object is stale when its source,
    a shared header or the ABI header is newer) and relink the library."""
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    shared = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "lutgpu.h")]
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, src.replace(".cu", ".o"))
        objs.append(obj)
        deps = [os.path.join(CSRC, src)] + shared
        if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in deps):
            continue
        cmd = [_nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((obj, subprocess.Popen(cmd)))
    failed = [obj for obj, pr in procs if pr.wait() != 0]
    if failed:
        for obj in failed:
            if os.path.exists(obj):
                os.remove(obj)
        raise subprocess.CalledProcessError(1, f"nvcc ({', '.join(os.path.basename(o) for o in failed)})")
    # export only the extern "C" symbols (visibility=hidden + explicit list via version script)
    vscript = os.path.join(LIBDIR, "exports.map")
    with open(vscript, "w") as f:
        f.write("{ global: lut_*; local: *; };\n")
    cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", LIB,
           "-Xlinker", f"--version-script={vscript}", "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
