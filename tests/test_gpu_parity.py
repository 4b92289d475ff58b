"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on
identical seeded inputs. Index selection must match bit-exactly; U V^T within
1e-9 relative Frobenius (north_star tolerance); report fields exactly."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_0814_b200 import rsm
from tests.util import max_angle_sin, random_masked, rel_fro

pytestmark = pytest.mark.gpu

UV_TOL = 1e-9  # north_star: U V^T within 1e-9 relative Frobenius error, FP64


def gen(m, n, r, rho, sigma, seed):
    M = rsm.generate(m, n, r, rho, sigma, seed)
    return M


def ctx_for(M):
    c = rsm.Context(0)
    c.load(M)
    return c


# ------------------------------------------------------------- generator pin

def test_generator_matches_oracle_restatement():
    M = gen(300, 40, 3, 0.6, 0.1, 7)
    Y, W = O.generate(300, 40, 3, 0.6, 0.1, 7)
    assert np.array_equal(M.mask, W)
    k = W.astype(bool)
    assert np.array_equal(M.values[k], Y[k])
    assert np.isnan(M.values[~k]).all()


# ------------------------------------------------------------------ stage 1

@pytest.mark.parametrize("shape", [
    dict(m=2000, n=200, r=3, rho=0.8, k=4, T=2000, seed=0),        # config 1
    dict(m=131072, n=1024, r=4, rho=0.8, k=5, T=16384, seed=0),    # config 3
    dict(m=3000, n=100, r=2, rho=0.35, k=6, T=500, seed=5),        # high rejection, budget cut
])
def test_select_m2_bit_exact(shape):
    M = gen(shape["m"], shape["n"], shape["r"], shape["rho"], 1e-3, shape["seed"])
    p = O.trial_params(shape["r"], 1, M.m, M.n, block=shape["k"], seed=shape["seed"])
    ids_o, q_o, att_o, acc_o = O.select(M.mask, p, shape["T"])
    c = ctx_for(M)
    tp = rsm.TrialParams(rsm.Mode.M2, p.block, p.ell, p.rank, p.min_count, p.seed)
    ids_g, q_g, att_g, acc_g = c.select(tp, shape["T"])
    assert (att_g, acc_g) == (att_o, acc_o)
    assert np.array_equal(ids_g, ids_o)
    assert np.array_equal(q_g, q_o)


def test_select_m1_bit_exact():
    M = gen(20000, 500, 5, 0.7, 1e-2, 1)  # config 2
    p = O.trial_params(5, 0, M.m, M.n, seed=1)
    ids_o, q_o, att_o, acc_o = O.select(M.mask, p, 4096)
    c = ctx_for(M)
    tp = rsm.TrialParams(rsm.Mode.M1, p.block, p.ell, p.rank, p.min_count, p.seed)
    ids_g, q_g, att_g, acc_g = c.select(tp, 4096)
    assert (att_g, acc_g) == (att_o, acc_o)
    assert np.array_equal(ids_g, ids_o)
    assert np.array_equal(q_g, q_o)


def test_select_budget_exhausted():
    # mask so sparse that almost nothing is accepted: the 20x budget ends the run
    M = gen(400, 60, 2, 0.3, 0.0, 3)
    p = O.trial_params(2, 1, M.m, M.n, block=8, seed=3)
    ids_o, q_o, att_o, acc_o = O.select(M.mask, p, 50)
    c = ctx_for(M)
    tp = rsm.TrialParams(rsm.Mode.M2, p.block, p.ell, p.rank, p.min_count, p.seed)
    ids_g, q_g, att_g, acc_g = c.select(tp, 50)
    assert att_o == 1000 and acc_o < 50
    assert (att_g, acc_g) == (att_o, acc_o)
    assert np.array_equal(ids_g, ids_o)


# ------------------------------------------------------------- stages 1-3

def _gram_check(M, mode, r, T, seed, block=0, vpt=0):
    p = O.trial_params(r, mode, M.m, M.n, block=block, vectors_per_trial=vpt, seed=seed)
    G_o, att_o, acc_o, z_o = O.harvest(M.values, M.mask, p, T)
    c = ctx_for(M)
    tp = rsm.TrialParams(rsm.Mode(mode), p.block, p.ell, p.rank, p.min_count, p.seed)
    h = c.harvest_gram(tp, T)
    assert (h.attempted, h.accepted, h.z) == (att_o, acc_o, z_o)
    scale = max(1.0, np.abs(G_o).max())
    # acceptance criterion 5 (tests/acceptance.cpp:261-310): 1e-10 * max(1, |G|max)
    assert np.abs(h.gram - G_o).max() <= 1e-10 * scale
    assert np.array_equal(h.gram, h.gram.T)  # exact symmetry, as the reference


def test_harvest_gram_config1():
    M = gen(2000, 200, 3, 0.8, 1e-3, 0)
    _gram_check(M, 1, 3, 2000, 0, block=4)


def test_harvest_gram_config2_column_branch():
    M = gen(20000, 500, 5, 0.7, 1e-2, 1)
    _gram_check(M, 0, 5, 4096, 1, block=6)


def test_harvest_gram_config3_prefix():
    M = gen(131072, 1024, 4, 0.8, 1e-3, 0)
    _gram_check(M, 1, 4, 48, 0, block=5)


def test_harvest_gram_column_branch_explicit_ell():
    M = gen(600, 30, 2, 0.7, 0.1, 11)
    _gram_check(M, 0, 2, 300, 11, block=5, vpt=2)


# ---------------------------------------------------------------- stage 4

def test_solve_v_matches_dsyev_on_oracle_gram():
    M = gen(2000, 200, 3, 0.8, 1e-3, 0)
    p = O.trial_params(3, 1, M.m, M.n, block=4, seed=0)
    G, *_ = O.harvest(M.values, M.mask, p, 2000)
    V_o, gr_o, bl_o, w = O.solve_v(G, 3, 1e-9)
    res = rsm.solve_v(G, 3, 1e-9)
    assert res.gram_rank == gr_o and res.borderline == bl_o
    assert max_angle_sin(res.v, V_o) <= 1e-10
    # distinct eigenvalues: sign-fixed columns agree individually
    assert np.abs(res.v - V_o).max() <= 1e-9


def test_solve_v_reference_cases():
    # tests/test_solver.cpp:46-86
    G = np.diag([5.0, 4.0, 0.0, 0.0])
    res = rsm.solve_v(G, 2, 1e-9)
    assert res.gram_rank == 2 and not res.borderline
    P = res.v @ res.v.T
    assert np.abs(P - np.diag([0, 0, 1, 1.0])).max() <= 1e-12
    with pytest.raises(rsm.Error) as ei:
        rsm.solve_v(np.diag([5.0, 0, 0, 0]), 2, 1e-9)
    assert ei.value.code == rsm.errc.insufficient_coverage
    res = rsm.solve_v(np.diag([5.0, 2e-8, 0, 0]), 2, 1e-9)
    assert res.gram_rank == 2 and res.borderline
    for bad in [(4, 1e-9), (0, 1e-9), (2, 0.0)]:
        with pytest.raises(rsm.Error) as ei:
            rsm.solve_v(np.eye(4), *bad)
        assert ei.value.code == rsm.errc.invalid_config


def test_solve_v_larger_iterative_path():
    # n > 16: Chebyshev-filtered subspace iteration vs dsyev
    rng = np.random.default_rng(3)
    n, r = 300, 5
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.concatenate([rng.uniform(0, 1e-3, r), rng.uniform(50, 100, n - r)])
    G = (Q * w) @ Q.T
    G = 0.5 * (G + G.T)
    V_o, gr_o, bl_o, _ = O.solve_v(G, r, 1e-9)
    res = rsm.solve_v(G, r, 1e-9)
    assert res.gram_rank == gr_o and res.borderline == bl_o
    assert max_angle_sin(res.v, V_o) <= 1e-10


# ---------------------------------------------------------------- stage 5

def test_solve_u_matches_cod():
    M = gen(3000, 120, 4, 0.6, 0.05, 9)
    rng = np.random.default_rng(9)
    V, _ = np.linalg.qr(rng.standard_normal((120, 4)))
    U_o, fl_o = O.solve_u(M.values, M.mask, V, 4)
    res = rsm.solve_u(M, V, 4)
    assert res.underdetermined_rows == fl_o
    assert rel_fro(res.u, U_o) <= 1e-12


def test_solve_u_reference_cases():
    # tests/test_solver.cpp:140-212
    M = rsm.MaskedMatrix(1, 4)
    for j in range(4):
        M.set(0, j, 1.0)
    res = rsm.solve_u(M, np.full(4, 0.5), 1)
    assert res.underdetermined_rows == 0 and abs(res.u[0, 0] - 2.0) <= 1e-12
    M = rsm.MaskedMatrix(3, 4)
    for j in range(4):
        M.set(0, j, 1.0)
        M.set(2, j, 3.0)
    res = rsm.solve_u(M, np.full(4, 0.5), 1)
    assert res.underdetermined_rows == 1
    assert abs(res.u[0, 0] - 2) <= 1e-12 and res.u[1, 0] == 0.0 and abs(res.u[2, 0] - 6) <= 1e-12
    M = rsm.MaskedMatrix(1, 4)
    M.set(0, 1, 2.0)
    vh = np.zeros(8)
    vh[2] = vh[3] = 1.0
    res = rsm.solve_u(M, vh, 2)
    assert res.underdetermined_rows == 1
    assert np.allclose(res.u[0], [1.0, 1.0], atol=1e-10)
    M = rsm.MaskedMatrix(2, 3)
    for i in range(2):
        for j in range(3):
            M.set(i, j, float(i + j + 1))
    res = rsm.solve_u(M, np.array([1, 1, 2, 2, 3, 3.0]), 2)
    assert res.underdetermined_rows == 2
    assert np.allclose(res.u[:, 0], res.u[:, 1], atol=1e-10)


def test_solve_u_stationarity_random_basis():
    # tests/test_solver.cpp:174-199
    vals, mask = random_masked(40, 12, 0.6, 31)
    M = rsm.MaskedMatrix(40, 12, vals, mask)
    V = np.random.default_rng(31).standard_normal((12, 3))
    res = rsm.solve_u(M, V, 3)
    U_o, fl_o = O.solve_u(vals, mask, V, 3)
    assert res.underdetermined_rows == fl_o
    for i in range(40):
        k = mask[i].astype(bool)
        y = vals[i, k]
        grad = V[k].T @ (V[k] @ res.u[i] - y)
        assert np.abs(grad).max() <= 1e-8 * (1 + np.linalg.norm(y))


def test_masked_residual_norm_hand_example():
    # tests/test_core.cpp:51-63
    M = rsm.MaskedMatrix(2, 2)
    M.set(0, 0, 1); M.set(0, 1, 2); M.set(1, 0, 3); M.set(1, 1, 4)
    F = rsm.Factorization(2, 2, 1, np.array([[1.0], [3.0]]), np.array([[1.0], [2.0]]))
    assert abs(rsm.masked_residual_norm(M, F) - 1.0) <= 1e-15


# --------------------------------------------------------------- end to end

def _e2e(M, cfg):
    F, rep = rsm.decompose(M, cfg)
    U_o, V_o, rep_o = O.decompose(M.values, M.mask, cfg.rank, cfg.plan.trials, mode=int(cfg.mode),
                                  block=cfg.block, vectors_per_trial=cfg.vectors_per_trial, seed=cfg.seed,
                                  tol=cfg.gram_rank_tol, min_dim=cfg.min_dim)
    assert rep.trials_attempted == rep_o.trials_attempted
    assert rep.trials_accepted == rep_o.trials_accepted
    assert rep.z == rep_o.z
    assert rep.gram_rank == rep_o.gram_rank
    assert rep.borderline_rank_gate == bool(rep_o.borderline)
    assert rep.underdetermined_rows == rep_o.underdetermined_rows
    uv, uv_o = F.u @ F.v.T, U_o @ V_o.T
    assert rel_fro(uv, uv_o) <= UV_TOL
    # e relative to the reference's, with an absolute floor at the rounding level of unit-scale data
    assert abs(rep.e - rep_o.e) <= 1e-9 * rep_o.e + 1e-12
    return F, rep


def test_decompose_config1():
    M = gen(2000, 200, 3, 0.8, 1e-3, 0)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=0)
    _e2e(M, cfg)


def test_decompose_config2_column_branch():
    M = gen(20000, 500, 5, 0.7, 1e-2, 1)
    cfg = rsm.RsmConfig(rank=5, mode=rsm.Mode.M1, block=6, plan=rsm.TrialPlan(4096), seed=1)
    _e2e(M, cfg)


def test_decompose_noiseless_recovers_planted():
    # tests/test_solver.cpp:245-269 (heuristic plan 25n)
    M = gen(200, 40, 3, 0.5, 0.0, 17)
    cfg = rsm.RsmConfig(rank=3, plan=rsm.TrialPlan(25 * 40), seed=17)
    F, rep = _e2e(M, cfg)
    assert rep.e <= 1e-8 and rep.gram_rank >= 37


def test_decompose_wide_matrix_transposes():
    # tests/test_solver.cpp:304-324
    M = gen(30, 90, 2, 0.6, 0.0, 71)
    cfg = rsm.RsmConfig(rank=2, plan=rsm.TrialPlan(25 * 30), seed=7)
    F, rep = _e2e(M, cfg)
    assert F.u.shape == (30, 2) and F.v.shape == (90, 2) and rep.e <= 1e-8


def test_decompose_row_branch_floor():
    # tests/test_solver.cpp:326-344
    M = gen(150, 30, 2, 0.85, 0.0, 83)
    cfg = rsm.RsmConfig(rank=2, mode=rsm.Mode.M2, plan=rsm.TrialPlan(300), seed=83)
    F, rep = _e2e(M, cfg)
    assert rep.e <= 1e-8 and rep.z >= rep.trials_accepted


def test_decompose_validation_errors():
    vals, mask = random_masked(20, 10, 0.9, 5)
    M = rsm.MaskedMatrix(20, 10, vals, mask)
    bad = [rsm.RsmConfig(rank=10, plan=rsm.TrialPlan(250)),
           rsm.RsmConfig(rank=3, block=2, plan=rsm.TrialPlan(250)),
           rsm.RsmConfig(rank=3, plan=rsm.TrialPlan(250, epsilon=1.0)),
           rsm.RsmConfig(rank=3, plan=rsm.TrialPlan(0))]
    for cfg in bad:
        with pytest.raises(rsm.Error) as ei:
            rsm.decompose(M, cfg)
        assert ei.value.code == rsm.errc.invalid_config
    with pytest.raises(rsm.Error) as ei:
        rsm.decompose(rsm.MaskedMatrix(4, 4), rsm.RsmConfig(rank=2, plan=rsm.TrialPlan(100)))
    assert ei.value.code == rsm.errc.insufficient_coverage


def test_decompose_deterministic():
    M = gen(120, 24, 2, 0.6, 0.2, 53)
    cfg = rsm.RsmConfig(rank=2, plan=rsm.TrialPlan(600), seed=99)
    F1, r1 = rsm.decompose(M, cfg)
    F2, r2 = rsm.decompose(M, cfg)
    assert np.array_equal(F1.u, F2.u) and np.array_equal(F1.v, F2.v) and r1.e == r2.e


def test_host_packed_mask_matches_device_load():
    # rsm_ctx_load packs the byte mask on the host (any nonzero byte is an
    # observation, core.hpp:26); rsm_ctx_load_device packs it on the device.
    # Both loads must give bitwise identical decompositions, for both branches.
    import torch
    M = gen(3000, 96, 3, 0.7, 1e-3, 12)
    W = M.mask.astype(np.uint8) * np.array([1, 7, 255], dtype=np.uint8)[np.arange(M.mask.size) % 3].reshape(M.mask.shape)
    for mode, block in [(rsm.Mode.M2, 4), (rsm.Mode.M1, 5)]:
        cfg = rsm.RsmConfig(rank=3, mode=mode, block=block, plan=rsm.TrialPlan(800), seed=4)
        c1 = rsm.Context(0)
        c1.load_arrays(M.values, W)
        assert c1.last_load_h2d_bytes() == M.values.nbytes + 4 * 3000 * 4  # 96 cols -> 4 words per row
        F1, r1 = c1.decompose(cfg)
        Yd = torch.from_numpy(np.ascontiguousarray(M.values)).cuda()
        Wd = torch.from_numpy(np.ascontiguousarray(M.mask.astype(np.uint8))).cuda()
        c2 = rsm.Context(0)
        c2.load_device(Yd.data_ptr(), Wd.data_ptr(), 3000, 96)
        torch.cuda.synchronize()
        F2, r2 = c2.decompose(cfg)
        assert np.array_equal(F1.u, F2.u) and np.array_equal(F1.v, F2.v)
        assert r1.e == r2.e and r1.z == r2.z and r1.trials_accepted == r2.trials_accepted


@pytest.mark.parametrize("case", [(2000, 200, 3, 0.8, 5, 0), (400, 900, 4, 0.6, 4, 9)])
def test_baseline_als_matches_oracle(case):
    # baseline_als on the device (stage-5 kernel on M and on its transpose)
    # against the C restatement of als.cpp:11-44
    m, n, r, rho, its, seed = case
    M = gen(m, n, r, rho, 1e-3, seed)
    F, rep = rsm.baseline_als(M, r, its, seed)
    U_o, V_o, fl_o, e_o = O.als(M.values, M.mask, r, its, seed)
    assert rep.underdetermined_rows == fl_o
    assert rel_fro(F.u @ F.v.T, U_o @ V_o.T) <= UV_TOL
    assert abs(rep.e - e_o) <= 1e-9 * e_o + 1e-12


def test_baseline_als_validation():
    M = gen(50, 20, 2, 0.7, 0.0, 1)
    for r, its in [(0, 3), (20, 3), (2, 0)]:
        with pytest.raises(rsm.Error) as ei:
            rsm.baseline_als(M, r, its, 1)
        assert ei.value.code == rsm.errc.invalid_config
    M0 = rsm.MaskedMatrix(10, 5)
    with pytest.raises(rsm.Error) as ei:
        rsm.baseline_als(M0, 2, 3, 1)
    assert ei.value.code == rsm.errc.insufficient_coverage


# ------------------------------------------- config 5: structured missingness

def test_config5_tracks_coverage_failure_matches_oracle():
    # BASELINE config 5 shape at reduced size: edge frames are seen by too few
    # points for any 5-point probe to cover them, so G has exact zero rows and
    # the rank gate (solver.cpp:34-39) fails with insufficient_coverage, on the
    # device exactly as in the oracle (dsyev on the oracle's G)
    M = rsm.generate_tracks(2048, 256, 32, 128, 1e-3, 0)
    cfg = rsm.RsmConfig(rank=4, mode=rsm.Mode.M2, block=5, plan=rsm.TrialPlan(2048), seed=0)
    with pytest.raises(O.OracleError) as eo:
        O.decompose(M.values, M.mask, 4, 2048, mode=1, block=5, seed=0)
    with pytest.raises(rsm.Error) as ed:
        rsm.decompose(M, cfg)
    assert eo.value.code == ed.value.code == rsm.errc.insufficient_coverage
    assert "rank gate failed" in str(ed.value)


def test_config5_tracks_covered_matches_oracle():
    # wide windows cover every frame: the gate passes and the decomposition of
    # the structured instance matches the oracle
    M = rsm.generate_tracks(1500, 48, 40, 48, 1e-3, 3)
    cfg = rsm.RsmConfig(rank=4, mode=rsm.Mode.M2, block=5, plan=rsm.TrialPlan(1500), seed=3)
    F, rep = _e2e(M, cfg)
    assert rep.gram_rank >= 96 - 4


def test_solve_v_zero_rows_fail_the_gate():
    # a caller-supplied accumulator with more than r all-zero rows
    rng = np.random.default_rng(8)
    A = rng.standard_normal((40, 40))
    G = A @ A.T
    for j in (3, 9, 17, 22, 31, 38):
        G[j, :] = 0.0
        G[:, j] = 0.0
    with pytest.raises(O.OracleError) as eo:
        O.solve_v(G, 4)
    with pytest.raises(rsm.Error) as ed:
        rsm.solve_v(G, 4, 1e-9)
    assert eo.value.code == ed.value.code == rsm.errc.insufficient_coverage


def test_run_report_reproducible(tmp_path):
    # tests/test_cli.cpp:78-105 of the reference, through the library: the
    # instance saved to CSV and loaded back decomposes to the same artifacts
    # and reports (wall_time aside) on every run
    from paper_1411_0814_b200 import report as RP
    M = gen(60, 20, 2, 0.7, 0.2, 9)
    p = str(tmp_path / "d.csv")
    rsm.save_matrix(M, p)
    L = rsm.load_matrix(p)
    cfg = rsm.RsmConfig(rank=2, mode=rsm.Mode.M2, plan=rsm.TrialPlan(300), seed=4)
    reps = []
    for _ in range(2):
        F, rep = rsm.decompose(L, cfg)
        rep.wall_time = 0.0
        reps.append((F, RP.serialize_report(RP.make_report(cfg, rep, rsm.dataset_checksum(L)))))
    assert np.array_equal(reps[0][0].u, reps[1][0].u) and np.array_equal(reps[0][0].v, reps[1][0].v)
    assert reps[0][1] == reps[1][1]
    r = RP.parse_report(reps[0][1])
    assert r.checksum == rsm.dataset_checksum(M) and r.trials == 300 and r.trial_source == "explicit"


def test_harvest_gram_wide_k9_cta_kernel():
    # k = 9 with ~760 survivors: the per-warp submatrices exceed the warp kernel's
    # shared-memory budget, so stage 2 runs the CTA-per-trial kernel with the
    # compile-time K = 9 Gram and rotation (config 4's path at a small m and T)
    M = gen(600, 1200, 8, 0.95, 1e-3, 4)
    _gram_check(M, 1, 8, 12, 4, block=9)


@pytest.mark.parametrize("k", [4, 5, 6])
def test_harvest_gram_pure_noise_small_gaps(k):
    # no low-rank structure: the k x k Grams have no clear gap below the top
    # r = k - 1, which exercises the top-r basis path's convergence test and
    # its one-sided Jacobi fallback
    vals, mask = random_masked(400, 60, 0.9, 40 + k)
    M = rsm.MaskedMatrix(400, 60, vals, mask)
    _gram_check(M, 1, k - 1, 300, k, block=k)


@pytest.mark.parametrize("l", [3, 4, 6])
def test_harvest_gram_column_branch_pure_noise_small_gaps(l):
    # column branch, r = l - 1, no low-rank structure: the l x l Grams have no
    # clear gap above their smallest eigenvalue, so the basis-from-the-Gram path
    # (perp_basis_small) refuses most trials and they are gathered again for the
    # one-sided Jacobi; both kinds of trial land in the same accumulator
    vals, mask = random_masked(600, 40, 0.9, 70 + l)
    M = rsm.MaskedMatrix(600, 40, vals, mask)
    _gram_check(M, 0, l - 1, 200, l, block=l)


@pytest.mark.parametrize("l,r", [(3, 2), (5, 4), (8, 7)])
def test_harvest_gram_column_branch_gram_basis(l, r):
    # column branch, r = l - 1 on planted low-rank data (noiseless and noisy):
    # every trial takes the basis straight from the Gram accumulated while gathering
    for sigma, seed in ((0.0, 5), (1e-2, 6)):
        M = gen(3000, 64, r, 0.8, sigma, seed)
        _gram_check(M, 0, r, 256, seed, block=l)
