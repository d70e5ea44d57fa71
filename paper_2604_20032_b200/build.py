"""Build libleo_b200.so (sm_100a) in-tree with nvcc.

The library is one translation unit (csrc/leo_b200.cu includes the kernel
files) compiled for `-gencode arch=compute_100a,code=sm_100a` with
`--fmad=false` (the blame arithmetic must not be FMA-contracted: the reference
evaluates ((d*e)*n)*m and s*p/t with separate roundings, analysis.py:357,482).
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
import subprocess
import sys
import time
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


# Build record written next to the library: the nvcc command, the host, the
# compile time and a content hash of every source (not mtimes, which a repo
# snapshot copied to another machine does not preserve).
RECORD = PKG / "libleo_b200.build.json"


def source_hash() -> str:
    h = hashlib.sha256()
    for s in sources():
        h.update(s.name.encode())
        h.update(s.read_bytes())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def build_record() -> dict | None:
    try:
        return json.loads(RECORD.read_text())
    except (OSError, ValueError):
        return None


def needs_build() -> bool:
    rec = build_record()
    return not LIB.exists() or rec is None or rec.get("source_sha256") != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libleo_b200.so.  Skipped when the library's build record holds
    the current sources' hash, unless `force` or LEO_FORCE_BUILD=1."""
    force = force or os.environ.get("LEO_FORCE_BUILD") == "1"
    if not force and not needs_build():
        return LIB
    cmd = [NVCC, *FLAGS, "-o", str(LIB) + ".tmp", str(CSRC / "leo_b200.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    t0 = time.time()
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libleo_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    nv = subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.strip()
    RECORD.write_text(json.dumps({
        "library": LIB.name, "command": " ".join(cmd).replace(".tmp", ""),
        "nvcc": nv.splitlines()[-1] if nv else None, "host": platform.node(),
        "built_at": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime(t0)),
        "compile_s": round(time.time() - t0, 1), "forced": force,
        "source_sha256": source_hash()}, indent=1) + "\n")
    return LIB


FRONT = PKG / "libleo_front.so"
FRONT_SRC = PKG / "native" / "leo_front.cpp"
PROFILE_SRC = PKG / "native" / "leo_profile.cpp"


def build_front(force: bool = False) -> Path:
    """Host-only C++ listing front-end (native/leo_front.cpp -> libleo_front.so)."""
    hdr = PKG.parent / "include" / "leo_front.h"
    srcs = (FRONT_SRC, PROFILE_SRC, hdr)
    if not force and FRONT.exists() and FRONT.stat().st_mtime >= max(x.stat().st_mtime for x in srcs):
        return FRONT
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-pthread",
           "-o", str(FRONT) + ".tmp", str(FRONT_SRC), str(PROFILE_SRC)]
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
