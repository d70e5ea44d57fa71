"""Build libleo_b200.so (sm_100a) in-tree with nvcc.

The library is one translation unit (csrc/leo_b200.cu includes the kernel
files) compiled for `-gencode arch=compute_100a,code=sm_100a` with
`--fmad=false` (the blame arithmetic must not be FMA-contracted: the reference
evaluates ((d*e)*n)*m and s*p/t with separate roundings, analysis.py:357,482).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libleo_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "leo_b200.h"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    cmd = [NVCC, *FLAGS, "-o", str(LIB) + ".tmp", str(CSRC / "leo_b200.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libleo_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


FRONT = PKG / "libleo_front.so"
FRONT_SRC = PKG / "native" / "leo_front.cpp"


def build_front(force: bool = False) -> Path:
    """Host-only C++ listing front-end (native/leo_front.cpp -> libleo_front.so)."""
    hdr = PKG.parent / "include" / "leo_front.h"
    if not force and FRONT.exists() and FRONT.stat().st_mtime >= max(FRONT_SRC.stat().st_mtime,
                                                                     hdr.stat().st_mtime):
        return FRONT
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall",
           "-o", str(FRONT) + ".tmp", str(FRONT_SRC)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building libleo_front.so")
    os.replace(str(FRONT) + ".tmp", FRONT)
    return FRONT


if __name__ == "__main__":
    build_front(force="--force" in sys.argv)
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
