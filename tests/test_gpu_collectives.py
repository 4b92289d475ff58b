"""GPU: the multi-rank code path with real NCCL on one GPU. With
RSM_FORCE_COLLECTIVES=1 a world-1 context built from an NCCL unique id creates
a one-rank communicator and takes the path every rank of an N-GPU run takes:
the accumulator all-reduce, the padded all-gather of the row-sharded U and the
scalar all-reduce. On one rank these are identities, so the decomposition must
equal the single-GPU path bit for bit. This checks the run-time-loaded NCCL
symbols, their argument types and the gather/scatter bookkeeping on hardware
(the N > 1 schedule itself is covered by tests/test_multigpu_gloo.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1411_0814_b200 import rsm
M = rsm.generate(3001, 257, 3, 0.8, 1e-3, 2)
cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2500), seed=2)
nid = rsm.Context.nccl_unique_id() if sys.argv[2] == "nccl" else None
ctx = rsm.Context(0, 1, 0, nid)
ctx.load(M)
F, rep = ctx.decompose(cfg)
h = ctx.harvest_gram(rsm.TrialParams(rsm.Mode.M2, 4, 0, 3, 4, 2), 2500)
np.save(sys.argv[1], np.concatenate([F.u.ravel(), F.v.ravel(), h.gram.ravel(),
                                     [rep.e, rep.z, rep.gram_rank, rep.underdetermined_rows]]))
""" % ROOT


def test_one_rank_collectives_match_single_gpu():
    outs = []
    for mode in ["plain", "nccl"]:
        env = dict(os.environ, RSM_FORCE_COLLECTIVES="1")
        path = f"/tmp/rsm_coll_{mode}.npy"
        subprocess.run([sys.executable, "-c", CODE, path, mode], check=True, env=env, timeout=600)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


def _run_ranks(M, world, fn):
    """fn(ctx) on `world` contexts of one host group, one thread per rank."""
    import threading
    from paper_1411_0814_b200 import rsm
    g = rsm.HostGroup(world)
    ctxs = [rsm.Context(0, rank=r, host_group=g) for r in range(world)]
    for c in ctxs:
        c.load(M)
    out, err = [None] * world, []

    def work(r):
        try:
            out[r] = fn(ctxs[r])
        except Exception as e:  # surfaced below
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in ctxs:
        c.close()
    g.close()
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_host_group_ranks_match_single_gpu(world):
    # the real multi-rank kernels and bookkeeping (trial shards of stages 2-3,
    # the accumulator + column-count all-reduce, row-sharded stage 5 and the
    # padded U all-gather with unequal row blocks) with `world` contexts on one
    # GPU exchanging through host memory; every rank must reproduce the
    # single-context decomposition up to FP reassociation of the shard sums
    from paper_1411_0814_b200 import rsm
    from tests.util import rel_fro
    M = rsm.generate(3001, 257, 3, 0.8, 1e-3, 2)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2500), seed=2)
    tp = rsm.TrialParams(rsm.Mode.M2, 4, 0, 3, 4, 2)
    ref = rsm.Context(0)
    ref.load(M)
    F0, rep0 = ref.decompose(cfg)
    G0 = ref.harvest_gram(tp, 2500).gram
    ref.close()

    def job(c):
        F, rep = c.decompose(cfg)
        G = c.harvest_gram(tp, 2500).gram
        return F, rep, G

    outs = _run_ranks(M, world, job)
    for F, rep, G in outs:
        assert (rep.trials_attempted, rep.trials_accepted, rep.z, rep.gram_rank, rep.underdetermined_rows) == (
            rep0.trials_attempted, rep0.trials_accepted, rep0.z, rep0.gram_rank, rep0.underdetermined_rows)
        assert np.abs(G - G0).max() <= 1e-12 * np.abs(G0).max()
        assert np.array_equal(G, G.T)
        assert rel_fro(F.u @ F.v.T, F0.u @ F0.v.T) <= 1e-12
        assert abs(rep.e - rep0.e) <= 1e-12 * rep0.e
    # all ranks hold the same (gathered) factors
    for F, _, G in outs[1:]:
        assert np.array_equal(F.u, outs[0][0].u) and np.array_equal(F.v, outs[0][0].v)
        assert np.array_equal(G, outs[0][2])


def test_one_shot_calls_are_reentrant():
    # rsm_decompose & co. share one default context per device; the per-context
    # lock held from the load to the last copy makes concurrent callers safe,
    # as the reference's pure functions are (two threads, different matrices)
    import threading
    from paper_1411_0814_b200 import rsm
    Ms = [rsm.generate(1500, 120, 3, 0.8, 1e-3, s) for s in (11, 12)]
    cfgs = [rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(800), seed=s) for s in (11, 12)]
    want = [rsm.decompose(M, c) for M, c in zip(Ms, cfgs)]
    got = [[None] * 2 for _ in range(6)]

    def work(i, k):
        got[k][i] = rsm.decompose(Ms[i], cfgs[i])

    for k in range(6):
        th = [threading.Thread(target=work, args=(i, k)) for i in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    for k in range(6):
        for i in range(2):
            F, rep = got[k][i]
            assert np.array_equal(F.u, want[i][0].u) and np.array_equal(F.v, want[i][0].v)
            assert rep.e == want[i][1].e
