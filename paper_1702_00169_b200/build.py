"""Build libpdg.so in-tree for sm_100a (B200) with nvcc.  No JIT, no fallback."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpdg.so")
# the checked build (-DPDG_CHECKED: bounds-checked global accesses, bounded cross-CTA waits,
# csrc/pdg_check.cuh); the binding loads it when PDG_CHECKED=1
LIB_CHECKED = os.path.join(HERE, "libpdg_checked.so")
SOURCES = [os.path.join(SRC, "pdg_api.cu")]
# every file under csrc/ (kernels, tables, NCCL plumbing) and the public header
DEPS = sorted(set(SOURCES + [os.path.join(SRC, f) for f in os.listdir(SRC)
                             if f.endswith((".cu", ".cuh", ".hpp", ".h"))] +
                  [os.path.join(os.path.dirname(HERE), "include", "pdg.h")]))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_cmd(out=LIB, extra=()):
    return [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
            "--expt-relaxed-constexpr", *extra, "-o", out, *SOURCES, "-ldl"]


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    if force or needs_build(lib):
        tmp = lib + f".tmp{os.getpid()}"
        extra = (("-Xptxas", "-v") if verbose else ()) + (("-DPDG_CHECKED",) if checked else ())
        subprocess.check_call(nvcc_cmd(tmp, extra), stdout=sys.stderr if verbose else subprocess.DEVNULL)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
