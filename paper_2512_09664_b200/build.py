"""Build libpivgen_b200.so in-tree with nvcc for sm_100a.

Usage: python -m paper_2512_09664_b200.build [--force]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_NAME = "libpivgen_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)
SOURCES = ["pivgen_b200.cu"]
HEADERS = ["common.cuh", "fused.cuh", "band.cuh", "histmatch.cuh", "refrng.cuh", "wide.cuh", "probes.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-cudart", "static",
    "-shared", "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build")
    return cand


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    mtime = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(REPO_DIR, "include", "pivgen_b200.h"))
    return any(os.path.getmtime(d) > mtime for d in deps if os.path.exists(d))


def check_band_kernel_frame(ptxas_log: str, limit: int = 256) -> None:
    """Fail the build when a band kernel gets a stack frame: that means the
    kernel parameters were copied to local memory (a device function taking
    `const BandParams&` was not inlined) and every parameter access goes
    through local memory (measured: 64 -> 116 us per batch at c2)."""
    import re

    cur = None
    for line in ptxas_log.splitlines():
        m = re.search(r"Function properties for (_ZN3pgb1\d?band_(?:sorted_)?kernel\S*)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame", line)
        if cur and m:
            if int(m.group(1)) > limit:
                raise RuntimeError(f"{cur}: {m.group(1)}-byte stack frame (kernel parameters spilled to "
                                   "local memory?); make the callee __forceinline__")
            cur = None


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    extra = []
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    proc = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
    if verbose:
        sys.stdout.write(proc.stdout + proc.stderr)
    check_band_kernel_frame(proc.stdout + proc.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
