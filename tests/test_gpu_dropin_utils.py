"""GPU: the reference's per-call building blocks behind the drop-in surface
(rsm_sample, rsm_small_singular_vectors, rsm_gram_update,
rsm_masked_objective), against the C oracle (pinned to the reference's own
sampler/spectra/core, tests/test_oracle_pin.py):

  sample_m1 / sample_m2   sampler.cpp:12-87   drawn and kept indices bit-exact
  small_singular_vectors  spectra.cpp:48-86   singular values; vectors equal for
                                              simple values, equal projectors
                                              on repeated (zero) ones
  attempt_trial           harvest.cpp:37-51   its vectors accumulate to the
                                              harvest's G (tests/acceptance.cpp:280-310)
  GramAccumulator         spectra.cpp:7-46    bit-identical to the reference loops
  masked_objective        core.cpp:41-44      Frobenius; l1 rejected as the reference
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_0814_b200 import rsm
from tests.util import random_masked

pytestmark = pytest.mark.gpu


def mm(m, n, rho, seed):
    Y, W = random_masked(m, n, rho, seed)
    return rsm.MaskedMatrix(m, n, Y, W)


@pytest.mark.parametrize("case", [(60, 40, 0.8, 3, 1), (60, 40, 0.8, 4, 1), (200, 30, 0.7, 5, 1), (35, 70, 0.9, 2, 0),
                                  (120, 25, 0.6, 3, 0), (50, 50, 0.95, 16, 1)])
def test_sample_matches_oracle(case):
    m, n, rho, count, mode = case
    M = mm(m, n, rho, 11 + count)
    for t in range(25):
        idx_o, surv_o = O.sample(M.mask, mode, count, 7, t)
        S = (rsm.sample_m2 if mode == 1 else rsm.sample_m1)(M, count, 7, t, 1)
        if len(surv_o) < 1:
            assert S is None
            continue
        drawn, kept = (S.row_indices, S.col_indices) if mode == 1 else (S.col_indices, S.row_indices)
        assert np.array_equal(drawn, idx_o) and np.array_equal(kept, surv_o)
        assert np.array_equal(S.values, M.values[np.ix_(S.row_indices, S.col_indices)])


def test_sample_min_keep_and_range_errors():
    # tests/test_sampler.cpp:60-72: the survivor floor rejects; counts out of range raise
    M = mm(40, 12, 0.5, 9)
    _, surv = O.sample(M.mask, 1, 3, 1, 0)
    assert rsm.sample_m2(M, 3, 1, 0, len(surv)) is not None
    assert rsm.sample_m2(M, 3, 1, 0, len(surv) + 1) is None
    with pytest.raises(rsm.Error) as e:
        rsm.sample_m2(M, 41, 1, 0)
    assert e.value.code == rsm.errc.invalid_config and "sample_m2: row count out of range" in str(e.value)
    with pytest.raises(rsm.Error) as e:
        rsm.sample_m1(M, 0, 1, 0)
    assert "sample_m1: column count out of range" in str(e.value)


def _groups(sv, tol):
    g, cur = [], [0]
    for i in range(1, len(sv)):
        if abs(sv[i] - sv[cur[-1]]) <= tol:
            cur.append(i)
        else:
            g.append(cur)
            cur = [i]
    g.append(cur)
    return g


@pytest.mark.parametrize("shape", [(5, 40, 4), (4, 9, 3), (30, 6, 5), (12, 8, 2), (3, 3, 2), (6, 33, 5), (40, 16, 3)])
def test_small_singular_vectors_match_oracle(shape):
    p, q, r = shape
    rng = np.random.default_rng(p * 100 + q)
    S = rng.standard_normal((p, q))
    if p > 6:  # low-rank plus noise: a spread of small values
        S = rng.standard_normal((p, r)) @ rng.standard_normal((r, q)) + 1e-3 * S
    ell = q - r
    sub = rsm.Submatrix(np.arange(p), np.arange(q) * 2, S)
    cvs = rsm.small_singular_vectors(sub, r, ell)
    Z = np.array([c.zeta for c in cvs])
    sv = np.array([c.singular_value for c in cvs])
    Zo, svo = O.small_singular_vectors(S, r, ell)
    smax = np.linalg.svd(S, compute_uv=False)[0]
    assert np.abs(sv - svo).max() <= 1e-12 * smax
    assert np.allclose(Z @ Z.T, np.eye(ell), atol=1e-12)
    assert all(np.array_equal(c.col_indices, sub.col_indices) for c in cvs)
    for g in _groups(svo, 1e-9 * smax):
        if len(g) == 1:
            assert np.abs(Z[g[0]] - Zo[g[0]]).max() <= 1e-9
            k = int(np.argmax(np.abs(Z[g[0]])))
            assert Z[g[0], k] > 0
        else:
            assert np.abs(Z[g].T @ Z[g] - Zo[g].T @ Zo[g]).max() <= 1e-9


def test_small_singular_vectors_validation():
    S = rsm.Submatrix(np.arange(3), np.arange(4), np.ones((3, 4)))
    for r, ell, msg in [(4, 1, "needs more than r columns"), (3, 1, "needs more than r rows"),
                        (2, 3, "vector count must lie in [1, cols-r]"), (2, 0, "vector count must lie")]:
        with pytest.raises(rsm.Error) as e:
            rsm.small_singular_vectors(S, r, ell)
        assert e.value.code == rsm.errc.invalid_config and msg in str(e.value)


def test_attempt_trial_vectors_accumulate_to_harvest():
    # tests/acceptance.cpp:280-310: the accepted attempts' embedded vectors,
    # accumulated in attempt order, give the harvest's accumulator
    M = mm(60, 24, 0.85, 21)
    cfg = rsm.RsmConfig(rank=2, mode=rsm.Mode.M2, block=3, plan=rsm.TrialPlan(40), seed=5)
    p = rsm.trial_params(cfg, M)
    h = rsm.harvest_gram(M, p, 40)
    rows, got, idx = [], 0, 0
    while got < 40:
        res = rsm.attempt_trial(M, p, idx)
        idx += 1
        if res is None:
            continue
        got += 1
        rows += [rsm.embed(cv, M.n) for cv in res]
    assert idx == h.attempted and len(rows) == h.z
    G = rsm.gram_update(np.zeros((M.n, M.n)), np.array(rows))
    assert np.abs(G - h.gram).max() <= 1e-10 * max(1.0, np.abs(G).max())


def test_attempt_trial_column_branch_and_rejection():
    M = mm(80, 12, 0.7, 4)
    cfg = rsm.RsmConfig(rank=2, mode=rsm.Mode.M1, block=4, plan=rsm.TrialPlan(10), seed=3)
    p = rsm.trial_params(cfg, M)
    for idx in range(15):
        res = rsm.attempt_trial(M, p, idx)
        cols, surv = O.sample(M.mask, 0, 4, 3, idx)
        if len(surv) < p.min_count:
            assert res is None
            continue
        assert len(res) == p.ell and all(np.array_equal(cv.col_indices, cols) for cv in res)
        S = M.values[np.ix_(surv, cols)]
        Zo, svo = O.small_singular_vectors(S, p.rank, p.ell)
        Z = np.array([cv.zeta for cv in res])
        assert np.abs(Z.T @ Z - Zo.T @ Zo).max() <= 1e-9


def test_gram_update_bit_identical_to_reference_loops():
    rng = np.random.default_rng(2)
    n = 37
    X = rng.standard_normal((25, n)) * (rng.random((25, n)) < 0.4)
    G0 = rng.standard_normal((n, n))
    G2 = rng.standard_normal((n, n))
    want = G0.copy()
    for x in X:  # GramAccumulator::accumulate_dense: row[j] += x_i * x_j in vector order
        want = want + np.outer(x, x)
    want = want + G2  # merge
    got = rsm.gram_update(G0, X, G2)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_masked_objective():
    M = mm(70, 30, 0.8, 8)
    rng = np.random.default_rng(1)
    F = rsm.Factorization(70, 30, 3, rng.standard_normal((70, 3)), rng.standard_normal((30, 3)))
    e = O.masked_residual_norm(M.values, M.mask, F.u, F.v)
    obj = rsm.masked_objective(M, F, 0)
    assert abs(obj - e * np.sqrt(M.mask.sum())) <= 1e-12 * obj
    with pytest.raises(rsm.Error) as ei:
        rsm.masked_objective(M, F, 1)
    assert ei.value.code == rsm.errc.invalid_config and "only frobenius is implemented" in str(ei.value)
