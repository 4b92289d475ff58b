"""Config-3 (or c1/c4) decompositions on cuda:0, for ncu captures of the stage kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
shapes = {"c3": (131072, 1024, 4, 0.8, 1e-3, 5, 16384), "c1": (2000, 200, 3, 0.8, 1e-3, 4, 2000),
          "c4": (1048576, 2048, 8, 0.9, 1e-3, 9, 65536), "c2": (20000, 500, 5, 0.7, 1e-2, 6, 4096)}
m, n, r, rho, sigma, k, T = shapes[cfgname]
seed = 1 if cfgname == "c2" else 0
mode = rsm.Mode.M1 if cfgname == "c2" else rsm.Mode.M2
ctx = rsm.Context(0)
if os.environ.get("DEVGEN", "1" if cfgname == "c4" else "0") == "1":
    ctx.generate(m, n, r, rho, sigma, seed)  # device generator (config 4: 17 GB)
else:
    ctx.load(rsm.generate(m, n, r, rho, sigma, seed))
cfg = rsm.RsmConfig(rank=r, mode=mode, block=k, plan=rsm.TrialPlan(T), seed=seed)
for i in range(int(os.environ.get("REPS", "2"))):
    t0 = time.time()
    _, rep = ctx.decompose(cfg, fetch=False)
    print(i, f"{(time.time() - t0) * 1e3:.2f} ms", ctx.stage_ms(), ctx.solver_stats(), rep.e, flush=True)
if int(os.environ.get("REPS", "2")) >= 4:
    import numpy as np
    st = []
    for i in range(int(os.environ.get("REPS", "2"))):
        ctx.decompose(cfg, fetch=False)
        st.append(ctx.stage_ms())
    med = np.median(np.array(st), axis=0)
    print("median", " ".join(f"{x:.4f}" for x in med), "(select svd gram reduce solve_v solve_u total)", flush=True)
