"""Build the sm_100a shared library ``libexem_b200.so`` in-tree with nvcc.

The library is the C-ABI declared in ``include/exem_b200.h``.  It is built
in place (next to this file) so that it travels with the repository snapshot
to the GPU box; it is git-ignored.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libexem_b200.so"
SOURCES = [CSRC / "exem_simt.cu", CSRC / "exem_setmin.cu",
           CSRC / "exem_simt_tma.cu", CSRC / "exem_tc.cu",
           CSRC / "exem_tc_batch.cu"]
HEADERS = [CSRC / "exem_common.cuh", CSRC / "exem_tc_common.cuh",
           ROOT / "include" / "exem_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
    "-diag-suppress", "177,550",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


# extra nvcc flags of the library on disk (travels with the .so to the GPU
# box; _build/ does not)
STAMP = PKG / "libexem_b200.so.flags"


def _extra_flags() -> list:
    return os.environ.get("EXEM_NVCC_FLAGS", "").split()  # experiments


def _stale() -> bool:
    if not LIB.exists():
        return True
    # a probe / trace build (EXEM_NVCC_FLAGS) is never reused as the shipped
    # library, and vice versa
    built = STAMP.read_text().split() if STAMP.exists() else None
    if built != _extra_flags():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source for sm_100a and link ``libexem_b200.so``."""
    if not force and not _stale():
        return LIB
    build_dir = PKG / "_build"
    build_dir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs, procs = [], []
    for src in SOURCES:  # the translation units compile in parallel
        obj = build_dir / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *_extra_flags(), "-c", str(src), "-o",
               str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))
        objs.append(str(obj))
    failed = [cmd for cmd, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           *objs, "-o", str(tmp), "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    STAMP.write_text(" ".join(_extra_flags()) + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
