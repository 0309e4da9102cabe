"""Build recipe for libmmjoin_b200.so (sm_100a only).

    python -m paper_2002_12459_b200.build        # or __graft_entry__.build()

Compiles every ``csrc/*.cu`` with ``nvcc -gencode arch=compute_100a,code=sm_100a``
(the explicit -gencode form: tcgen05/TMA need the arch-specific target, and the
generic ``compute_100`` PTX that ``-arch=sm_100a`` would add is rejected by
ptxas for tcgen05) and links one shared library with the CUDA runtime linked
statically, so the library has no ABI coupling to torch's bundled runtime.
Objects are rebuilt only when a source or header is newer than the library.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libmmjoin_b200.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"] + os.environ.get("MMJ_NVCC_EXTRA", "").split()


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the mmjoin B200 engine needs CUDA 12.9 nvcc")
    return cand


def sources():
    return sorted(CSRC.glob("*.cu"))


STAMP = LIB.with_suffix(".flags")

# the bounds-checked variant (MMJ_DCHECK compiled in): loaded instead of the
# product library when MMJ_LIB_VARIANT=check (tests/test_gpu_checked.py)
CHECK_LIB = LIBDIR / "libmmjoin_b200_check.so"


def _variant(check: bool):
    if check:
        return CHECK_LIB, CHECK_LIB.with_suffix(".flags"), LIBDIR / "obj_check", FLAGS + ["-DMMJ_DEBUG_CHECKS"]
    return LIB, STAMP, LIBDIR / "obj", FLAGS


def _flag_line(flags=None) -> str:
    return " ".join(ARCH + (FLAGS if flags is None else flags))


def _stale(check: bool = False) -> bool:
    """Rebuild when a source / header is newer than the library, or when the
    nvcc flags differ from the ones it was built with (an experiment build
    with MMJ_NVCC_EXTRA=-D... must never be picked up silently)."""
    lib, stamp, _, flags = _variant(check)
    if not lib.exists() or not stamp.exists() or stamp.read_text() != _flag_line(flags):
        return True
    t = lib.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, check: bool = False) -> Path:
    lib, stamp, objdir, flags = _variant(check)
    if not force and not _stale(check):
        return lib
    LIBDIR.mkdir(exist_ok=True)
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in sources():
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc, *ARCH, *flags, "-I", str(CSRC), "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src.name}")
        if verbose:
            sys.stderr.write(res.stderr)
        (objdir / (src.stem + ".ptxas.txt")).write_text(res.stderr)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    stamp.write_text(_flag_line(flags))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, check="--check" in sys.argv))
