"""Build libescg_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2508_16639_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libescg_b200.so")
SOURCES = ["kernels.cu", "slice.cu", "ring.cu", "engine.cpp"]
HEADERS = ["crs.cuh", "launch.h", "record.cuh", "slice_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "escg_dev.h"),
                                                               os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile csrc/ into `out` (default: the in-tree libescg_b200.so).  `defines` are extra -D
    flags for diagnostic variants (never used by the product build)."""
    lib = out or LIB
    if out is None and not defines and not force and not _stale():
        return LIB
    objs = []
    procs = []
    for src in SOURCES:  # the translation units compile in parallel
        obj = os.path.join(CSRC, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd.insert(1, "-x")
            cmd.insert(2, "cu")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    logs = []
    failed = None
    for src, pr in procs:
        out = pr.communicate()[0]
        logs.append(out)
        if pr.returncode != 0:
            sys.stderr.write(out)
            failed = failed or src
    if failed:
        raise RuntimeError("nvcc failed on %s" % failed)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xlinker", "--exclude-libs,ALL"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
