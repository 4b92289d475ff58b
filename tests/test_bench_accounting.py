"""CPU: the algorithmic work bench.py divides by (DESIGN.md
section 3) -- the roofline's `achieved` numerator -- on a hand-checkable case."""
import importlib.util
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_algorithmic_counts():
    b = _bench()
    c = dict(m=8, n=64, r=2, k=3, T=2)
    qs = np.array([10, 20])
    alg = b.algorithmic(c, qs, nwp_bytes=16, attempts=5)
    assert alg["s1_bytes"] == 5 * 3 * (64 / 32) * 4          # drawn rows' mask words
    assert alg["s2_bytes"] == 2 * 3 * 64 * 8                  # full Y rows per trial
    assert alg["s2_flops"] == sum(2 * q * 3 * 4 / 2 + 2 * 2 * 3 * q for q in (10, 20))
    assert alg["s3_flops_survey"] == sum(2 * 2 * q * q for q in (10, 20))  # 2 r q^2
    assert alg["s3_flops"] == sum(2 * q * (q + 1) for q in (10, 20))       # unique entries: r q (q+1)
    assert alg["s5_bytes"] == 8 * 64 * 8 + 8 * 16 + 8 * 2 * 8 + 64 * 2 * 8


def test_bench_configs_match_baseline_shapes():
    b = _bench()
    c3 = b.CONFIGS["config3"]
    assert (c3["m"], c3["n"], c3["r"], c3["rho"], c3["k"], c3["T"]) == (131072, 1024, 4, 0.8, 5, 16384)
    c4 = b.CONFIGS["config4"]
    assert (c4["m"], c4["n"], c4["r"], c4["rho"], c4["k"], c4["T"]) == (1048576, 2048, 8, 0.9, 9, 65536)
