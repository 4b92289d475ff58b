# reduced config-4 shape (same n, r, k, rho; 1/8 rows and trials) for profiling
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm
M = rsm.generate(131072, 2048, 8, 0.9, 1e-3, 0)
ctx = rsm.Context(0); ctx.load(M)
cfg = rsm.RsmConfig(rank=8, mode=rsm.Mode.M2, block=9, plan=rsm.TrialPlan(8192), seed=0)
for i in range(2):
    F, rep = ctx.decompose(cfg, fetch=False)
    print([round(x, 3) for x in ctx.stage_ms()], rep.e, flush=True)
