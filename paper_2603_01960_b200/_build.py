"""In-tree build of libtileattn_b200.so (sm_100a) with nvcc.

The shared library lands in paper_2603_01960_b200/_lib/ so it travels with the
repo snapshot to the GPU box (git-ignored, not gpurun-ignored).  A JIT cache
under ~/.cache would not travel, so nothing here uses torch's JIT.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libtileattn_b200.so"

SOURCES = [CSRC / "sdpa_fwd_sm100.cu", CSRC / "c_api.cpp"]
HEADERS = [CSRC / "ptx_sm100.cuh", CSRC / "sdpa_fwd_sm100.h", ROOT / "include" / "tileattn_b200.h"]

GENCODE = "-gencode=arch=compute_100a,code=sm_100a"
NVCC_FLAGS = [
    GENCODE,
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", str(ROOT / "include"),
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; cannot build the sm_100a library")
    return cand


def _digest() -> str:
    h = hashlib.sha256()
    for p in SOURCES + HEADERS:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Compile (if sources changed) and return the library path.

    ``defines``/``out`` build an experimental variant (e.g. -DTA_EMU16_D64=6)
    into another file; the product library is the default ``LIB``."""
    LIBDIR.mkdir(exist_ok=True)
    lib = Path(out) if out else LIB
    lib.parent.mkdir(parents=True, exist_ok=True)
    stamp = lib.with_suffix(".stamp")
    dig = _digest() + "|".join(defines)
    if not force and lib.exists() and stamp.exists() and stamp.read_text() == dig:
        return lib
    objdir = LIBDIR / ("obj" if out is None else "obj_" + lib.stem)
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    subprocess.run([nvcc(), GENCODE, "-shared", "-o", str(tmp), *objs, "-cudart", "static"],
                   check=True)
    os.replace(tmp, lib)
    stamp.write_text(dig)
    return lib


if __name__ == "__main__":
    import sys
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=Path(outs[0]) if outs else None))
