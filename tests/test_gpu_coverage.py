"""GPU: parity across the parameter space the BASELINE configs do not reach
(ranks 1..8, block sizes up to 16 with the CTA-per-trial SVD, odd and
non-multiple-of-32 widths, the column branch at larger l, the multi-chunk
harvest, wide inputs), each against the CPU oracle through the C ABI."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_0814_b200 import rsm
from tests.util import rel_fro

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check(M, cfg):
    F, rep = rsm.decompose(M, cfg)
    U_o, V_o, rep_o = O.decompose(M.values, M.mask, cfg.rank, cfg.plan.trials, mode=int(cfg.mode),
                                  block=cfg.block, vectors_per_trial=cfg.vectors_per_trial, seed=cfg.seed,
                                  tol=cfg.gram_rank_tol, min_dim=cfg.min_dim)
    assert (rep.trials_attempted, rep.trials_accepted, rep.z) == (rep_o.trials_attempted, rep_o.trials_accepted,
                                                                   rep_o.z)
    assert rep.gram_rank == rep_o.gram_rank and rep.underdetermined_rows == rep_o.underdetermined_rows
    assert rel_fro(F.u @ F.v.T, U_o @ V_o.T) <= 1e-9
    assert abs(rep.e - rep_o.e) <= 1e-9 * rep_o.e + 1e-12
    return rep


@pytest.mark.parametrize("r", [1, 2, 3, 5, 6, 7, 8])
def test_ranks_row_branch(r):
    M = rsm.generate(1500, 120, r, 0.85, 1e-3, 10 + r)
    _check(M, rsm.RsmConfig(rank=r, mode=rsm.Mode.M2, block=r + 1, plan=rsm.TrialPlan(1200), seed=r))


@pytest.mark.parametrize("k", [6, 10, 12])
def test_larger_blocks(k):
    # k > 9 takes the CTA-per-trial SVD kernel
    M = rsm.generate(3000, 90, 3, 0.93, 1e-3, k)
    _check(M, rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=k, plan=rsm.TrialPlan(800), seed=k))


@pytest.mark.parametrize("n", [33, 97, 130, 257])
def test_odd_widths(n):
    M = rsm.generate(900, n, 3, 0.8, 1e-3, n)
    _check(M, rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(900), seed=n))


@pytest.mark.parametrize("l", [5, 8])
def test_column_branch_larger_l(l):
    M = rsm.generate(4000, 120, 4, 0.75, 1e-2, l)
    _check(M, rsm.RsmConfig(rank=4, mode=rsm.Mode.M1, block=l, plan=rsm.TrialPlan(700), seed=l))


def test_wide_noisy_transposed():
    M = rsm.generate(150, 700, 3, 0.7, 1e-3, 4)
    _check(M, rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(900), seed=4))


def test_multi_chunk_harvest_matches_single_chunk():
    # a small expanded-V budget forces stage 2-3 to run in several trial chunks
    # (accumulating into the slice partials); run in a child process because
    # the budget is read once per process
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1411_0814_b200 import rsm
M = rsm.generate(2000, 200, 3, 0.8, 1e-3, 0)
cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=0)
F, rep = rsm.decompose(M, cfg)
np.save(sys.argv[1], np.concatenate([F.u.ravel(), F.v.ravel(), [rep.e, rep.z]]))
""" % ROOT
    outs = []
    for budget in [None, str(2000 * 256 * 4 * 8 // 5)]:  # about five chunks
        env = dict(os.environ)
        if budget:
            env["RSM_CHUNK_BYTES"] = budget
        path = os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else ".",
                            f"_chunk_{budget or 'one'}.npy")
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, timeout=300)
        outs.append(np.load(path))
        os.remove(path)
    a, b = outs
    assert a[-1] == b[-1]  # z
    # the slices' partial sums are added chunk by chunk: identical up to reassociation
    assert np.max(np.abs(a[:-2] - b[:-2])) <= 1e-9 * np.max(np.abs(a[:-2]))
    assert abs(a[-2] - b[-2]) <= 1e-9 * a[-2]


@pytest.mark.parametrize("m,n,r", [(500, 1600, 8), (500, 1601, 7), (300, 4000, 8), (400, 3000, 4), (400, 2001, 3)])
def test_solve_u_wide_rows(m, n, r):
    # the stage-5 layouts the BASELINE bench shape does not reach: V-hat filling
    # shared memory with rows read from global memory (config 4's n = 2048,
    # r = 8 layout), V-hat read from global memory (n = 4000, r = 8), odd
    # widths; rows above and below half observed (the r > 4 complement path
    # and the direct path); U, flags and the residual sum against the oracle
    M = rsm.generate(m, n, r, 0.55, 1e-2, n + r)
    rng = np.random.default_rng(n)
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    ctx = rsm.Context(0)
    ctx.load(M)
    res, ss = ctx.solve_u(V, r)
    U_o, fl_o = O.solve_u(M.values, M.mask, V, r)
    assert res.underdetermined_rows == fl_o
    assert rel_fro(res.u, U_o) <= 1e-12
    R = np.where(M.mask != 0, np.nan_to_num(M.values) - U_o @ V.T, 0.0)
    ss_o = float(np.sum(R * R))
    assert abs(ss - ss_o) <= 1e-10 * ss_o


@pytest.mark.parametrize("n", [2048, 2050])
def test_fused_global_row_solver_matches_two_pass(n):
    # config 4's stage-5 layout (V-hat fills shared memory, tensor-core normal
    # matrices): the fused residual/accumulation kernel (k_solve_u_preg) against
    # the two-pass kernel (RSM_SU_PREG=0) and the FP64 normal matrices
    # (RSM_NORMAL_TC=0) on the same decomposition, with and without a column
    # tail (n % 32 != 0); odd row counts per warp
    code = (
        "import sys, numpy as np\n"
        "from paper_1411_0814_b200 import rsm\n"
        f"ctx = rsm.Context(0); ctx.generate(8531, {n}, 8, 0.9, 1e-3, 3)\n"
        "cfg = rsm.RsmConfig(rank=8, mode=rsm.Mode.M2, block=9, plan=rsm.TrialPlan(6000), seed=3)\n"
        "F, rep = ctx.decompose(cfg)\n"
        "np.save(sys.argv[1], np.concatenate([(F.u @ F.v.T[:, :64]).ravel(), [rep.e, rep.underdetermined_rows]]))\n")
    outs = []
    for extra in ({}, {"RSM_SU_PREG": "0"}, {"RSM_NORMAL_TC": "0"}):
        env = dict(os.environ)
        env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
        env.update(extra)
        path = os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else ".",
                            f"_preg_{n}_{len(outs)}.npy")
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, timeout=300)
        outs.append(np.load(path))
        os.remove(path)
    a, b, c = outs
    assert a[-1] == b[-1] == c[-1] == 0
    assert abs(a[-2] - 1e-3) < 1e-4
    for o in (b, c):
        assert np.linalg.norm(a[:-2] - o[:-2]) <= 1e-11 * np.linalg.norm(a[:-2])
        assert abs(a[-2] - o[-2]) <= 1e-10 * a[-2]
