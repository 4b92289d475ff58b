"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family of the decomposition at C1-like sizes on cuda:0.

  row branch (k_select, k_svd_warp, k_gram_i8 + k_gram_reduce, k_eig, k_solve_u_fused)
  FP64 Gram path (RSM_GRAM=dfma in a child run: k_gram)
  column branch (k_svd<M1> CTA kernel)
  k = 9 row branch (CTA SVD kernel) with r = 8 (k_solve_u<8>, V-hat in smem)
  n = 2048, r = 8 stage 5 (rows read from global: V-hat fills shared memory)
  ALS, device generator, device-packed masks, world-2 host group
"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm  # noqa: E402


def run(tag, M, cfg):
    F, rep = rsm.decompose(M, cfg)
    print(tag, "e", rep.e, "rank", rep.gram_rank, flush=True)


only = sys.argv[1:] or ["row", "col", "k9", "wide", "als", "gen", "world2"]
if "row" in only:
    run("row", rsm.generate(2000, 200, 3, 0.8, 1e-3, 0),
        rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=0))
if "col" in only:
    run("col", rsm.generate(3000, 120, 5, 0.7, 1e-2, 1),
        rsm.RsmConfig(rank=5, mode=rsm.Mode.M1, block=6, plan=rsm.TrialPlan(800), seed=1))
if "k9" in only:
    run("k9", rsm.generate(3000, 160, 8, 0.9, 1e-3, 2),
        rsm.RsmConfig(rank=8, mode=rsm.Mode.M2, block=9, plan=rsm.TrialPlan(1500), seed=2))
if "wide" in only:
    # stage 5 at n = 2048, r = 8 on a given V-hat (V-hat fills shared memory)
    M = rsm.generate(600, 2048, 8, 0.9, 1e-3, 3)
    V = np.linalg.qr(np.random.default_rng(3).standard_normal((2048, 8)))[0]
    res = rsm.solve_u(M, V, 8)
    print("wide U norm", float(np.linalg.norm(res.u)), flush=True)
if "als" in only:
    F, rep = rsm.baseline_als(rsm.generate(800, 100, 3, 0.8, 1e-3, 4), 3, 3, 4)
    print("als e", rep.e, flush=True)
if "gen" in only:
    c = rsm.Context(0)
    c.generate(4096, 256, 4, 0.8, 1e-3, 5)
    F, rep = c.decompose(rsm.RsmConfig(rank=4, mode=rsm.Mode.M2, block=5, plan=rsm.TrialPlan(1024), seed=5))
    print("gen e", rep.e, flush=True)
    c.close()
if "world2" in only:
    M = rsm.generate(3001, 257, 3, 0.8, 1e-3, 2)
    cfg = rsm.RsmConfig(rank=3, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2500), seed=2)
    g = rsm.HostGroup(2)
    ctxs = [rsm.Context(0, rank=r, host_group=g) for r in range(2)]
    for c in ctxs:
        c.load(M)
    out = [None, None]

    def work(r):
        out[r] = ctxs[r].decompose(cfg)[1].e

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    print("world2 e", out, flush=True)
    for c in ctxs:
        c.close()
    g.close()
