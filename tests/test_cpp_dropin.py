"""The reference-style C++ call sites (include/rsm_gpu/rsm.hpp drop-in) compiled
with g++ and run against librsm_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_1411_0814_b200")


def _build(tmp_path):
    exe = str(tmp_path / "dropin_test")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    f"-L{LIBDIR}", "-lrsm_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
