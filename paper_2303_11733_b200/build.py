"""In-tree build of libdippm_b200.so (sm_100a) with nvcc.

The shared library is plain CUDA C++ behind the C ABI in include/dippm_b200.h;
it links the CUDA runtime statically and takes no torch headers, so it loads
through ctypes on any box with the same driver.  Objects are rebuilt only when
a source or header is newer than the library.
"""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libdippm_b200.so"
SOURCES = ["capi.cu", "csr.cu", "aggregate.cu", "head.cu", "head_fused.cu", "tc_gemm.cu", "numerics.cu", "rescore.cu", "step.cu", "head_tc.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


HOST_LIB = PKG / "libdippm_host.so"
HOST_SOURCES = ["featurize.cpp"]
CXX = os.environ.get("CXX", "g++")


def build_host(verbose: bool = False, force: bool = False) -> Path:
    """libdippm_host.so: the native front end (graph JSON -> features), host C++17 only."""
    srcs = [PKG / "hostsrc" / s for s in HOST_SOURCES]
    deps = srcs + [ROOT / "include" / "dippm_host.h"]
    if force or _stale(HOST_LIB, deps):
        cmd = [CXX, "-O3", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra", "-Wno-unused-parameter", "-Wno-array-bounds", "-Wno-stringop-overflow",
               "-I", str(ROOT / "include"), *map(str, srcs), "-o", str(HOST_LIB)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return HOST_LIB


def build(verbose: bool = False, force: bool = False) -> Path:
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "dippm_b200.h"]
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs, cmds = [], []
    for src in SOURCES:
        s = CSRC / src
        o = objdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmds.append([NVCC, *ARCH, *FLAGS, "-c", str(s), "-o", str(o)])
    # the translation units are independent: compile them in parallel
    from concurrent.futures import ThreadPoolExecutor
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd))
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        for f in [pool.submit(subprocess.run, cmd, check=True) for cmd in cmds]:
            f.result()
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(LIB), *map(str, objs), "-lcuda"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    build_host(verbose, force)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
