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


SUITES = ["test_core", "test_sampler", "test_spectra", "test_solver"]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suites_against_dropin(suite):
    """The reference's OWN doctest suites (tests/<suite>.cpp of the reference),
    compiled by oracle/build_ref.sh against include/rsm_gpu (the drop-in) and
    librsm_b200.so instead of the reference library, run on the GPU."""
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_" + suite)
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_* not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd="/tmp")
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
