"""GPU: decompose's single-synchronisation path. The selection is enqueued
speculatively (one chunk, stage 2 sized for a support bound) together with
stages 2-5; when the chunk does not reach the trial count or a support
outgrows the bound, the decomposition is re-run with the synchronous
selection (rsm_ctx.cu decompose_impl). Both outcomes must give exactly the
results of the synchronous path, which the oracle parity tests pin."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_0814_b200 import rsm
from tests.util import rel_fro

pytestmark = pytest.mark.gpu


def _run(M, cfg):
    c = rsm.Context(0)
    try:
        c.load(M)
        F, rep = c.decompose(cfg)
        return F, rep, c.rerun_count(), c
    except Exception:
        c.close()
        raise


def _same(a, b):
    Fa, ra = a[:2]
    Fb, rb = b[:2]
    assert np.array_equal(Fa.u, Fb.u) and np.array_equal(Fa.v, Fb.v)
    for k in ("e", "trials_attempted", "trials_accepted", "z", "gram_rank", "underdetermined_rows"):
        assert getattr(ra, k) == getattr(rb, k), k


def test_speculation_hits_on_dense_row_branch():
    M = rsm.generate(2000, 200, 3, 0.8, 1e-3, 0)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=0)
    F, rep, reruns, c = _run(M, cfg)
    c.close()
    assert reruns == 0
    assert rep.trials_accepted == 2000


def test_low_acceptance_reruns_then_learns_the_rate():
    # min_dim above the typical survivor count rejects most 4-row probes, so
    # one chunk of 1.1 T attempts accepts far fewer than T and the call
    # re-runs; the context keeps the observed rate and the next call's chunk
    # reaches T
    M = rsm.generate(2000, 200, 3, 0.6, 1e-3, 4)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=4, min_dim=28)
    F1, rep1, reruns1, c = _run(M, cfg)
    try:
        assert rep1.trials_attempted > 2 * rep1.trials_accepted  # acceptance well below 1
        assert reruns1 == 1
        F2, rep2 = c.decompose(cfg)
        assert c.rerun_count() == 1  # the second call's speculation held
        _same((F1, rep1), (F2, rep2))
    finally:
        c.close()
    # and both equal the oracle's decomposition of the same instance
    U_o, V_o, rep_o = O.decompose(M.values, M.mask, 3, 2000, mode=int(cfg.mode), block=4, seed=4, min_dim=28)
    assert rep1.trials_attempted == rep_o.trials_attempted and rep1.z == rep_o.z
    assert rep1.gram_rank == rep_o.gram_rank
    assert rel_fro(F1.u @ F1.v.T, U_o @ V_o.T) <= 1e-9


def test_support_bound_fallback_matches(monkeypatch):
    M = rsm.generate(2000, 200, 3, 0.8, 1e-3, 0)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=0)
    a = _run(M, cfg)
    a[3].close()
    monkeypatch.setenv("RSM_SPEC_LCAP", "8")  # far below any support: every speculation misses
    b = _run(M, cfg)
    b[3].close()
    assert a[2] == 0 and b[2] == 1
    _same(a, b)


def test_column_branch_speculation_matches_oracle():
    M = rsm.generate(3000, 120, 3, 0.7, 1e-2, 5)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M1, block=5, plan=rsm.TrialPlan(1500), seed=5)
    F, rep, reruns, c = _run(M, cfg)
    c.close()
    U_o, V_o, rep_o = O.decompose(M.values, M.mask, 3, 1500, mode=int(cfg.mode), block=5, seed=5)
    assert rep.trials_attempted == rep_o.trials_attempted and rep.z == rep_o.z
    assert rep.gram_rank == rep_o.gram_rank
    assert rel_fro(F.u @ F.v.T, U_o @ V_o.T) <= 1e-9


# ---------------------------------------------------- decompose as one graph
# (first call with a key eager, second captured, later calls replayed)

def test_graph_replay_matches_eager_bitwise():
    M = rsm.generate(2000, 200, 3, 0.8, 1e-3, 0)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=0)
    c = rsm.Context(0)
    try:
        c.load(M)
        outs, stages, launches = [], [], []
        for _ in range(4):
            outs.append(c.decompose(cfg))
            stages.append(c.stage_ms())
            launches.append(c.launch_count())
        for o in outs[1:]:
            _same(outs[0], o)
        assert len(set(launches)) == 1 and launches[0] > 0
        for st in stages:  # replays re-record the stage events
            assert st[6] > 0 and all(x >= 0 for x in st[:6])
            assert abs(sum(st[:6]) - st[6]) <= 1e-3 * st[6] + 1e-3
        assert stages[3] != stages[2] or stages[2] != stages[1]
        # a new key (seed) after the graph: same as a fresh context's result
        cfg2 = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=1)
        a = c.decompose(cfg2)
        b = _run(M, cfg2)
        b[3].close()
        _same(a, b)
        # a reload invalidates the graph: results follow the new matrix
        M3 = rsm.generate(2000, 200, 3, 0.8, 1e-3, 9)
        c.load(M3)
        for _ in range(3):
            d = c.decompose(cfg)
        e = _run(M3, cfg)
        e[3].close()
        _same(d, e)
    finally:
        c.close()


def test_graph_replay_rank_gate_failure_raises_every_call():
    M = rsm.generate_tracks(2048, 256, 32, 128, 1e-3, 0)
    cfg = rsm.RsmConfig(rank=4, mode=rsm.Mode.M2, block=5, plan=rsm.TrialPlan(2048), seed=0)
    c = rsm.Context(0)
    try:
        c.load(M)
        for _ in range(4):
            with pytest.raises(rsm.Error) as ei:
                c.decompose(cfg)
            assert ei.value.code == rsm.errc.insufficient_coverage
    finally:
        c.close()
