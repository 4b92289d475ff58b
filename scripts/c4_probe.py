import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1411_0814_b200 import rsm
m, n, r, rho, k, T = 1048576, 2048, 8, 0.9, 9, 65536
if len(sys.argv) > 1:
    m = int(sys.argv[1]); T = int(sys.argv[2])
t = time.time()
M = rsm.generate(m, n, r, rho, 1e-3, 0)
print("gen %.1f s" % (time.time() - t), flush=True)
ctx = rsm.Context(0)
t = time.time(); ctx.load(M); print("load %.1f s" % (time.time() - t), flush=True)
cfg = rsm.RsmConfig(rank=r, mode=rsm.Mode.M2, block=k, plan=rsm.TrialPlan(T), seed=0)
for i in range(3):
    t = time.time()
    F, rep = ctx.decompose(cfg, fetch=False)
    print("decompose %.2f ms" % ((time.time() - t) * 1e3), rep, [round(x, 3) for x in ctx.stage_ms()], flush=True)
print(ctx.solver_stats())
