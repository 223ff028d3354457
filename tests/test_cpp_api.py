"""Builds tests/cpp/test_tileattn_b200.cpp (the C++ mirror of the reference
entry point, include/tileattn_b200.hpp) with g++ and runs it: the validation
cases on CPU, the full parity suite on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "test_tileattn_b200.cpp"
LIBDIR = ROOT / "paper_2603_01960_b200" / "_lib"
ORACLE = ROOT / "oracle" / "_build"
BIN = LIBDIR / "test_tileattn_b200"


def _build():
    import oracle
    oracle.lib()  # builds liboracle.so if needed
    if BIN.exists() and BIN.stat().st_mtime > max(SRC.stat().st_mtime,
                                                  (ROOT / "include" / "tileattn_b200.hpp").stat().st_mtime,
                                                  (LIBDIR / "libtileattn_b200.so").stat().st_mtime):
        return BIN
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", str(ROOT / "include"), str(SRC),
           "-L", str(LIBDIR), "-ltileattn_b200", "-L", str(ORACLE), "-loracle",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{ORACLE}", "-o", str(BIN)]
    subprocess.run(cmd, check=True)
    return BIN


def test_cpp_mirror_builds_and_validates_on_cpu():
    b = _build()
    r = subprocess.run([str(b), "--cpu-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_mirror_parity_on_gpu(cuda_device):
    b = _build()
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
