"""CPU: the C-ABI library loads and exports every symbol include/rsm_b200.h
declares; host-only entry points (trial_params validation, generator) agree
with the oracle. No device compute is called here."""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_0814_b200 import rsm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsm_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rsm_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = rsm.lib()
    names = declared()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", rsm._LIBPATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rsm_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(L, n)
    assert set(rsm.exported_symbols()) == set(names)


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rsm._LIBPATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kw,code", [
    (dict(rank=0), 2), (dict(rank=10), 2), (dict(rank=3, block=3), 2), (dict(rank=3, block=40), 2),
    (dict(rank=3, min_dim=2), 2), (dict(rank=3, mode=0, block=5, vectors_per_trial=3), 2),
    (dict(rank=3), 0), (dict(rank=3, mode=1), 0), (dict(rank=2, mode=0, block=5, vectors_per_trial=2), 0),
    (dict(rank=2, mode=1, vectors_per_trial=7), 0),
])
def test_trial_params_validation_matches_oracle(kw, code):
    m, n = 30, 10
    cfg = rsm.RsmConfig(rank=kw.get("rank", 0), mode=rsm.Mode(kw.get("mode", 0)), block=kw.get("block", 0),
                        vectors_per_trial=kw.get("vectors_per_trial", 0), min_dim=kw.get("min_dim", 0), seed=3)
    M = rsm.MaskedMatrix(m, n)
    try:
        p = rsm.trial_params(cfg, M)
        got = 0
    except rsm.Error as e:
        got = int(e.code)
    want = 0
    try:
        q = O.trial_params(cfg.rank, int(cfg.mode), m, n, block=cfg.block, vectors_per_trial=cfg.vectors_per_trial,
                           seed=3, min_dim=cfg.min_dim)
    except O.OracleError as e:
        want = e.code
    assert got == want == code
    if code == 0:
        assert (p.block, p.ell, p.rank, p.min_count, p.seed) == (q.block, q.ell, q.rank, q.min_count, q.seed)


def test_host_generator_matches_oracle():
    M = rsm.generate(500, 37, 4, 0.7, 0.3, 21, row0=100, rows=250)
    Y, W = O.generate(500, 37, 4, 0.7, 0.3, 21, row0=100, rows=250)
    assert np.array_equal(M.mask, W)
    k = W.astype(bool)
    assert np.array_equal(M.values[k], Y[k]) and np.isnan(M.values[~k]).all()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1411_0814_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "__init__.py", f
