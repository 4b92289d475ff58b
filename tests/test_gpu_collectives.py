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
