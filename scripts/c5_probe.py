import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1411_0814_b200 import rsm
pts, frames, wmin, wmax, T = [int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (8192, 1024, 128, 512, 8192))]
M = rsm.generate_tracks(pts, frames, wmin, wmax, 1e-3, 0)
print("density", M.known_count() / M.values.size)
cfg = rsm.RsmConfig(rank=4, mode=rsm.Mode.M2, block=5, plan=rsm.TrialPlan(T), seed=0)
ctx = rsm.Context(0); ctx.load(M)
for i in range(2):
    t = time.time()
    try:
        F, rep = ctx.decompose(cfg)
        print("ok", rep, "%.2f ms" % ((time.time() - t) * 1e3), ctx.stage_ms())
    except rsm.Error as e:
        print("error", e.code, e, "%.2f ms" % ((time.time() - t) * 1e3))
