"""Build libmch.so (the C-ABI library) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libmch.so")
SOURCES = ["mch.cu", "kernels.cu", "pcg2d.cu", "pcg3d.cu", "pcg3d_cl.cu", "fine3d.cu", "macro.cu", "fine.cu", "plan.cpp", "shard.cpp", "comm.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# dev variants: MCH_BUILD_TIMING=1 builds lib/libmch_timing.so with per-phase PCG cycle counters;
# MCH_BUILD_TAG=t MCH_BUILD_DEFS="-DX=1 ..." builds lib/libmch_t.so with extra defines
if os.environ.get("MCH_BUILD_TIMING"):
    LIB = os.path.join(HERE, "lib", "libmch_timing.so")
if os.environ.get("MCH_BUILD_TAG"):
    LIB = os.path.join(HERE, "lib", "libmch_" + os.environ["MCH_BUILD_TAG"] + ".so")
FLAGS_C = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(os.path.join(os.path.dirname(LIB), "mch_peaks")):
        return True
    t = os.path.getmtime(LIB)
    for f in os.listdir(CSRC):
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    hdr = os.path.join(os.path.dirname(HERE), "include", "mch.h")
    return os.path.getmtime(hdr) > t


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel, then link the shared library."""
    if not force and not needs_build():
        return LIB
    libdir = os.path.dirname(LIB)
    os.makedirs(libdir, exist_ok=True)
    # objects outside the repo: the tree is pushed to the GPU box as is, the .so alone is needed
    objdir = os.path.join(os.environ.get("TMPDIR", "/tmp"), "mch_obj")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in SOURCES:
        timing = bool(os.environ.get("MCH_BUILD_TIMING"))
        tag = os.environ.get("MCH_BUILD_TAG", "") + (".timing" if timing else "")
        obj = os.path.join(objdir, src + (f".{tag}.o" if tag else ".o"))
        objs.append(obj)
        defs = (["-DPCG2D_TIMING"] if timing else []) + os.environ.get("MCH_BUILD_DEFS", "").split()
        cmd = [NVCC, *FLAGS_C, *defs, "-c", "-o", obj, os.path.join(CSRC, src)]
        # incremental: an object newer than its source and every header is kept (dev speed-up;
        # force=True or a removed object directory rebuilds everything)
        hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
        hdrs.append(os.path.join(os.path.dirname(HERE), "include", "mch.h"))
        deps = [os.path.join(CSRC, src), *hdrs, os.path.abspath(__file__)]
        if not force and os.path.exists(obj) and all(os.path.getmtime(obj) > os.path.getmtime(d) for d in deps):
            continue
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log_parts, failed = [], False
    for cmd, pr in procs:
        out, err = pr.communicate()
        log_parts.append(" ".join(cmd) + "\n" + out + err)
        failed = failed or pr.returncode != 0
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-ldl",
            "-o", LIB + ".tmp", *objs]
    if not failed:
        res = subprocess.run(link, capture_output=True, text=True)
        log_parts.append(" ".join(link) + "\n" + res.stdout + res.stderr)
        failed = res.returncode != 0
    log = os.path.join(libdir, "build.log")
    with open(log, "w") as f:
        f.write("\n".join(log_parts))
    if failed:
        sys.stderr.write("\n".join(log_parts)[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(LIB + ".tmp", LIB)
    # measured FP64 / shared-memory peaks for the roofline (bench.py), a standalone executable
    peaks = os.path.join(libdir, "mch_peaks")
    res = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", peaks,
                          os.path.join(CSRC, "peaks.cu")], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed for peaks.cu:\n" + res.stderr[-4000:])
    if verbose:
        print("\n".join(log_parts))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
