"""CPU: pin the plain-C oracle (oracle/liborc.so) against the reference itself.

Two anchors (SURVEY.md section 8c has no golden output vectors for this path):
  * oracle/_ref: the reference's own sources (/root/reference/proj/src) built
    with builder-written shims; its own doctest suites must pass, and the C
    restatement must agree with it (selection bit-exact, G/V/U to tolerance);
  * tests/golden/*.npz: fixtures generated from oracle/_ref by
    tests/golden/make_golden.py, so the pin also holds where /root/reference
    (and hence oracle/_ref) is absent.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from oracle import refbind as R
from tests.util import max_angle_sin, random_masked, rel_fro

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no /root/reference)")


# ---------------------------------------------------- reference self-checks

@needs_ref
@pytest.mark.parametrize("suite", ["test_core", "test_sampler", "test_spectra", "test_solver", "test_synth",
                                   "test_planner"])
def test_reference_suites_pass_on_ref_build(suite):
    exe = os.path.join(os.path.dirname(R.LIB), suite)
    if not os.path.exists(exe):
        pytest.skip("suite binary not built")
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="4")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


# ------------------------------------------------------------ rng + sampler

def test_rng_matches_reference_formulas():
    # rng.hpp:14-27 restated in numpy (uint64 arithmetic wraps)
    def mix(z):
        z = np.uint64(z)
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
        return z
    with np.errstate(over="ignore"):
        for seed, tag, idx in [(0, 5, 0), (1, 5, 12345), (2**63 + 7, 77, 3)]:
            s = mix(np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * np.uint64(tag))
            s = mix(s + np.uint64(0xBF58476D1CE4E5B9) * np.uint64(idx))
            assert int(s) == O.rng_state(seed, tag, idx)


def test_draw_is_sorted_distinct_and_matches_iota_fisher_yates():
    # sampler.cpp:12-23 literally (full iota array) vs the oracle's virtual map
    import ctypes as C
    L = O.lib()
    for pool, count, att in [(10, 10, 0), (131072, 5, 77), (20, 6, 3), (1, 1, 9)]:
        st = C.c_uint64(L.orc_rng_state(4, 5, att))
        idx = list(range(pool))
        for t in range(count):
            j = t + L.orc_next_below(C.byref(st), pool - t)
            idx[t], idx[j] = idx[j], idx[t]
        want = sorted(idx[:count])
        got = O.draw(pool, count, 4, att)
        assert list(got) == want


@needs_ref
@pytest.mark.parametrize("case", [
    dict(m=2000, n=200, r=3, rho=0.8, mode=1, block=4, T=2000, seed=0),
    dict(m=3000, n=100, r=2, rho=0.35, mode=1, block=6, T=400, seed=5),
    dict(m=400, n=60, r=2, rho=0.3, mode=1, block=8, T=50, seed=3),      # budget exhausted
    dict(m=2000, n=50, r=5, rho=0.7, mode=0, block=6, T=600, seed=1),
    dict(m=300, n=40, r=3, rho=0.35, mode=0, block=5, T=400, seed=2),
])
def test_selection_bit_exact_vs_reference(case):
    Y, W = O.generate(case["m"], case["n"], case["r"], case["rho"], 1e-3, case["seed"])
    p = O.trial_params(case["r"], case["mode"], case["m"], case["n"], block=case["block"], seed=case["seed"])
    a = O.select(W, p, case["T"])
    b = R.select(Y, W, case["mode"], p.block, p.min_count, p.seed, case["T"])
    assert a[2:] == b[2:]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@needs_ref
def test_generator_matches_reference_synth():
    Y, W = O.generate(120, 30, 3, 0.6, 0.2, 13)
    Yr, Wr = R.generate(120, 30, 3, 0.6, 0.2, 13)
    assert np.array_equal(W, Wr)
    k = W.astype(bool)
    assert np.array_equal(Y[k], Yr[k])


# ---------------------------------------------------------------- spectra

@needs_ref
@pytest.mark.parametrize("shape", [(5, 40, 4), (4, 82, 3), (30, 6, 5), (8, 5, 3), (3, 6, 2)])
def test_small_singular_vectors_vs_reference(shape):
    p, q, r = shape
    rng = np.random.default_rng(p * 100 + q)
    S = rng.standard_normal((p, min(p, r + 1))) @ rng.standard_normal((min(p, r + 1), q))
    S += 1e-3 * rng.standard_normal((p, q))
    ell = q - r
    z1, s1 = O.small_singular_vectors(S, r, ell)
    z2, s2 = R.small_singular_vectors(S, r, ell)
    assert np.allclose(s1, s2, rtol=1e-10, atol=1e-12 * np.abs(S).max())
    # the harvested set spans the same space: sum of projectors agrees
    assert np.abs(z1.T @ z1 - z2.T @ z2).max() <= 1e-10
    # vectors with nonzero distinct singular values agree individually
    nz = [t for t in range(ell) if s2[t] > 1e-8]
    for t in nz:
        assert np.abs(z1[t] - z2[t]).max() <= 1e-8


def test_spectra_reference_cases_on_oracle():
    # tests/test_spectra.cpp:66-75 exact null vector
    z, s = O.small_singular_vectors(np.array([[1, 2], [2, 4], [3, 6.0]]), 1, 1)
    assert abs(z[0, 0] - 2 / np.sqrt(5)) <= 1e-12 and abs(z[0, 1] + 1 / np.sqrt(5)) <= 1e-12
    assert abs(s[0]) <= 1e-12
    # :125-133 wide matrix pads the kernel with exact zeros
    rng = np.random.default_rng(13)
    S = rng.standard_normal((3, 2)) @ rng.standard_normal((2, 6))
    z, s = O.small_singular_vectors(S, 2, 4)
    assert s[0] == 0.0 and s[1] == 0.0 and s[2] == 0.0
    assert np.abs(S @ z.T).max() <= 1e-10 * np.linalg.norm(S)
    with pytest.raises(O.OracleError):
        O.small_singular_vectors(rng.standard_normal((4, 3)), 3, 1)


# ---------------------------------------------------------------- harvest

@needs_ref
@pytest.mark.parametrize("case", [
    dict(m=2000, n=200, r=3, rho=0.8, mode=1, block=4, T=600, seed=0, sigma=1e-3),
    dict(m=160, n=36, r=3, rho=0.55, mode=0, block=0, T=400, seed=41, sigma=0.15),
    dict(m=300, n=60, r=3, rho=0.5, mode=0, block=0, T=1500, seed=909, sigma=0.1),
])
def test_harvest_vs_reference(case):
    Y, W = O.generate(case["m"], case["n"], case["r"], case["rho"], case["sigma"], case["seed"])
    p = O.trial_params(case["r"], case["mode"], case["m"], case["n"], block=case["block"], seed=case["seed"])
    G, att, acc, z = O.harvest(Y, W, p, case["T"])
    Gr, attr, accr, zr = R.harvest(Y, W, p, case["T"], serial=True)
    Gp, attp, accp, zp = R.harvest(Y, W, p, case["T"], workers=4)
    assert (att, acc, z) == (attr, accr, zr) == (attp, accp, zp)
    assert np.array_equal(Gr, Gp)  # reference parallel == serial bitwise (test_solver.cpp:214-243)
    tol = 1e-10 * max(1.0, np.abs(Gr).max())  # acceptance criterion 5
    assert np.abs(G - Gr).max() <= tol
    assert np.array_equal(G, G.T)


def test_harvest_identity_matches_literal_sum():
    # independent check: G = diag(count) - sum_t E V_top V_top^T E^T (numpy SVD)
    Y, W = O.generate(500, 40, 3, 0.8, 1e-2, 4)
    p = O.trial_params(3, 1, 500, 40, block=4, seed=4)
    G, att, acc, z = O.harvest(Y, W, p, 300)
    ids, qs, att2, acc2 = O.select(W, p, 300)
    H = np.zeros((40, 40))
    for a in ids:
        rows, cols = O.sample(W, 1, 4, 4, int(a))
        S = Y[np.ix_(rows, cols)]
        Vt = np.linalg.svd(S)[2]
        Vr = Vt[:3].T
        H[np.ix_(cols, cols)] += np.eye(len(cols)) - Vr @ Vr.T
    assert (att, acc) == (att2, acc2)
    assert np.abs(G - H).max() <= 1e-10 * np.abs(H).max()


# ------------------------------------------------------------------ solver

@needs_ref
def test_solve_v_vs_reference():
    Y, W = O.generate(2000, 200, 3, 0.8, 1e-3, 0)
    p = O.trial_params(3, 1, 2000, 200, block=4, seed=0)
    G, *_ = O.harvest(Y, W, p, 600)
    V, gr, bl, w = O.solve_v(G, 3)
    Vr, grr, blr = R.solve_v(G, 3)
    assert (gr, bl) == (grr, blr)
    assert np.array_equal(V, Vr)  # same LAPACK dsyev, same sign fix


@needs_ref
def test_solve_u_vs_reference():
    vals, mask = random_masked(60, 14, 0.6, 31)
    V = np.random.default_rng(2).standard_normal((14, 3))
    U, fl = O.solve_u(vals, mask, V, 3)
    Ur, flr = R.solve_u(vals, mask, V, 3)
    assert fl == flr
    assert rel_fro(U, Ur) <= 1e-12
    # deficient rows: fewer observations than r and a degenerate basis
    M = np.full((3, 4), np.nan)
    Wm = np.zeros((3, 4), np.uint8)
    M[0, 1], Wm[0, 1] = 2.0, 1
    M[1, :], Wm[1, :] = [1, 2, 3, 4.0], 1
    Vd = np.array([[1, 1], [1, 1], [2, 2], [3, 3.0]])
    U, fl = O.solve_u(M, Wm, Vd, 2)
    Ur, flr = R.solve_u(M, Wm, Vd, 2)
    assert fl == flr == 3
    assert np.abs(U - Ur).max() <= 1e-10


@needs_ref
@pytest.mark.parametrize("case", [(80, 20, 3, 0.7, 5, 11), (50, 70, 2, 0.5, 3, 4)])
def test_als_vs_reference(case):
    # baseline_als (als.cpp:11-44): seeded init, alternating row solves on M and M^T
    m, n, r, rho, its, seed = case
    from oracle.oracle import generate
    Y, W = generate(m, n, r, rho, 1e-2, seed)
    U, V, fl, e = O.als(Y, W, r, its, seed)
    Ur, Vr, flr, er = R.als(Y, W, r, its, seed)
    assert fl == flr
    assert rel_fro(U @ V.T, Ur @ Vr.T) <= 1e-10
    assert abs(e - er) <= 1e-10 * er


def test_solve_u_reference_cases_on_oracle():
    # tests/test_solver.cpp:161-172 minimum norm (1, 1)
    u = np.zeros(2)
    ok = O.lib().orc_solve_row(np.array([1.0, 1.0]).ctypes.data_as(O.C.c_void_p),
                               np.array([2.0]).ctypes.data_as(O.C.c_void_p), 1, 2,
                               u.ctypes.data_as(O.C.c_void_p))
    assert ok == 0 and np.allclose(u, [1, 1], atol=1e-10)


@needs_ref
@pytest.mark.parametrize("case", [
    dict(m=2000, n=200, r=3, rho=0.8, sigma=1e-3, mode=1, block=4, T=2000, seed=0),
    dict(m=200, n=40, r=3, rho=0.5, sigma=0.0, mode=0, block=0, T=1000, seed=17),
    dict(m=30, n=90, r=2, rho=0.6, sigma=0.0, mode=0, block=0, T=750, seed=71),
    dict(m=150, n=30, r=2, rho=0.85, sigma=0.0, mode=1, block=0, T=300, seed=83),
    dict(m=2000, n=100, r=5, rho=0.7, sigma=1e-2, mode=0, block=6, T=800, seed=1),
])
def test_decompose_vs_reference(case):
    Y, W = O.generate(case["m"], case["n"], case["r"], case["rho"], case["sigma"], case["seed"])
    U, V, rep = O.decompose(Y, W, case["r"], case["T"], mode=case["mode"], block=case["block"], seed=case["seed"])
    Ur, Vr, repr_ = R.decompose(Y, W, case["r"], case["T"], mode=case["mode"], block=case["block"],
                                seed=case["seed"])
    for k in ("trials_attempted", "trials_accepted", "z", "underdetermined_rows", "gram_rank", "borderline"):
        assert getattr(rep, k) == repr_[k], k
    assert rel_fro(U @ V.T, Ur @ Vr.T) <= 1e-9
    assert abs(rep.e - repr_["e"]) <= 1e-9 * max(repr_["e"], 1e-12) + 1e-14


def test_decompose_errors_on_oracle():
    vals, mask = random_masked(20, 10, 0.9, 5)
    for kw in [dict(rank=10), dict(rank=3, block=2), dict(rank=3, epsilon=1.0), dict(rank=3, trials=0)]:
        args = dict(rank=3, trials=250)
        args.update(kw)
        with pytest.raises(O.OracleError) as ei:
            O.decompose(vals, mask, args.pop("rank"), args.pop("trials"), **args)
        assert ei.value.code == 2
    with pytest.raises(O.OracleError) as ei:
        O.decompose(np.full((4, 4), np.nan), np.zeros((4, 4), np.uint8), 2, 100)
    assert ei.value.code == 4


# ------------------------------------------------------------------ golden

def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} missing (run tests/golden/make_golden.py)")
    return np.load(path)


@pytest.mark.parametrize("name", ["config1_small.npz", "config2_small.npz"])
def test_oracle_against_golden(name):
    g = _golden(name)
    Y, W = O.generate(int(g["m"]), int(g["n"]), int(g["r"]), float(g["rho"]), float(g["sigma"]), int(g["seed"]))
    assert int(np.count_nonzero(W)) == int(g["known"])
    p = O.trial_params(int(g["r"]), int(g["mode"]), Y.shape[0], Y.shape[1], block=int(g["block"]),
                       seed=int(g["seed"]))
    ids, qs, att, acc = O.select(W, p, int(g["T"]))
    assert np.array_equal(ids, g["ids"]) and np.array_equal(qs, g["qs"]) and att == int(g["attempted"])
    G, att, acc, z = O.harvest(Y, W, p, int(g["T"]))
    assert z == int(g["z"])
    assert np.abs(G - g["G"]).max() <= 1e-10 * max(1.0, np.abs(g["G"]).max())
    U, V, rep = O.decompose(Y, W, int(g["r"]), int(g["T"]), mode=int(g["mode"]), block=int(g["block"]),
                            seed=int(g["seed"]))
    assert rep.gram_rank == int(g["gram_rank"]) and rep.underdetermined_rows == int(g["underdetermined"])
    assert rel_fro(U @ V.T, g["U"] @ g["V"].T) <= 1e-9
    assert max_angle_sin(V, g["V"]) <= 1e-9
