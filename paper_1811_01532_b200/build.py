"""Build the sm_100a C-ABI library `_lib/libwapb200.so` in-tree with nvcc.

Every `csrc/*.cu` is compiled for `-gencode arch=compute_100a,code=sm_100a`
with `-lineinfo` (so ncu's source page maps to our code) and linked into one
shared library that the Python shim loads with ctypes. Rebuilds are
incremental on source/header mtimes.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
OBJDIR = LIBDIR / "obj"
LIB = LIBDIR / "libwapb200.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"] + os.environ.get("WAP_NVCC_EXTRA", "").split()


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> Path:
    obj = OBJDIR / (src.stem + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile all kernels and link the shared library; returns its path."""
    OBJDIR.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    # objects built with other flags (e.g. a diagnostic -DWAP_GEMM_TRACE build) are stale
    # even when the sources are older: key the object dir on a hash of the command line
    stamp = OBJDIR / "flags.sha"
    flags_hash = hashlib.sha256(" ".join([NVCC, *ARCH, *FLAGS]).encode()).hexdigest()
    if not stamp.exists() or stamp.read_text() != flags_hash:
        force = True
    if force:
        for o in OBJDIR.glob("*.o"):
            o.unlink()
    hdr = _headers_mtime()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    stamp.write_text(flags_hash)
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose=True))
