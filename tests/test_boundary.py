"""The drop-in boundary: the C-ABI library loads and exports every entry point
include/spectrack_gpu.h declares, and the reference-facing C++ shim
(include/spectrack_b200.hpp) compiles and links against it (CPU only; the GPU
run of the shim is in test_gpu_boundary)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spectrack_gpu.h")
LIB = os.path.join(ROOT, "paper_2603_19439_b200", "libspectrack_b200.so")
SHIM_BIN = os.path.join(ROOT, "tests", "cpp", "_build", "shim_smoke")


def declared_symbols():
    text = open(HEADER).read()
    decl = re.compile(r"^(?:const\s+)?[a-z_0-9]+\s*\**\s*(st_[a-z_]+)\(", re.MULTILINE)
    return sorted(set(decl.findall(text)))


def ensure_lib():
    if not os.path.exists(LIB):
        from paper_2603_19439_b200 import _build
        _build.build()


def test_library_exports_every_declared_symbol():
    ensure_lib()
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def build_shim():
    ensure_lib()
    os.makedirs(os.path.dirname(SHIM_BIN), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "shim_smoke.cpp"), "-o", SHIM_BIN,
           "-L", os.path.dirname(LIB), "-lspectrack_b200", "-Wl,-rpath," + os.path.dirname(LIB),
           "-L/usr/local/cuda/lib64", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return SHIM_BIN


def test_cpp_shim_compiles_and_links():
    assert os.path.exists(build_shim())


@pytest.mark.gpu
def test_gpu_boundary_cpp_shim_runs():
    out = subprocess.run([build_shim()], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim_smoke: ok" in out.stdout
