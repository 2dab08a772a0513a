"""The C++ drop-in header (include/sslgpu/ssl.hpp): compiles against the C ABI
here; runs the reference's own unit-test cases on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2504_03373_b200", "_lib")
EXE = os.path.join(ROOT, "tests", "cpp", "test_dropin.bin")


def build_exe():
    from paper_2504_03373_b200 import _capi

    _capi.load()  # builds libsslgpu.so if missing
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR, "-lsslgpu",
           f"-Wl,-rpath,{LIBDIR}", "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return EXE


def test_header_compiles_against_the_c_abi():
    assert os.path.exists(build_exe())


@pytest.mark.gpu
def test_reference_unit_cases_through_the_cpp_header():
    exe = build_exe()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok")
