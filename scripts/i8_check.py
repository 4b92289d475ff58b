"""Stage 3 on the tensor cores (k_gram_i8) against the FP64 register-tile
kernel (RSM_GRAM=dfma) on the same device-generated instances: accumulator
difference, decomposition difference and the stage-3 time of each path."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm  # noqa: E402

CFGS = {
    "config1": dict(m=2000, n=200, r=3, rho=0.8, sigma=1e-3, mode=rsm.Mode.M2, block=4, T=2000, seed=0),
    "config2": dict(m=20000, n=500, r=5, rho=0.7, sigma=1e-2, mode=rsm.Mode.M1, block=6, T=4096, seed=1),
    "config3": dict(m=131072, n=1024, r=4, rho=0.8, sigma=1e-3, mode=rsm.Mode.M2, block=5, T=16384, seed=0),
    "config4": dict(m=1048576, n=2048, r=8, rho=0.9, sigma=1e-3, mode=rsm.Mode.M2, block=9, T=65536, seed=0),
}
names = sys.argv[1:] or list(CFGS)
ctx = rsm.Context(0)
for name in names:
    c = CFGS[name]
    ctx.generate(c["m"], c["n"], c["r"], c["rho"], c["sigma"], c["seed"])
    cfg = rsm.RsmConfig(rank=c["r"], mode=c["mode"], block=c["block"], plan=rsm.TrialPlan(c["T"]), seed=c["seed"])
    ell = c["block"] - c["r"] if c["mode"] == rsm.Mode.M1 else 0
    tp = rsm.TrialParams(c["mode"], c["block"], ell, c["r"], c["r"] + 1, c["seed"])
    res = {}
    for path in ("dfma", "i8"):
        if path == "dfma":
            os.environ["RSM_GRAM"] = "dfma"
        else:
            os.environ.pop("RSM_GRAM", None)
        h = ctx.harvest_gram(tp, c["T"])
        G = h.gram.copy()
        times = []
        for _ in range(3):
            F, rep = ctx.decompose(cfg, fetch=True)
            times.append(ctx.stage_ms())
        st = np.median(np.array(times), axis=0)
        res[path] = dict(G=G, U=F.u.copy(), V=F.v.copy(), rep=rep, st=st)
    Gd, Gi = res["dfma"]["G"], res["i8"]["G"]
    scale = max(1.0, np.abs(Gd).max())
    uvd = res["dfma"]["U"] @ res["dfma"]["V"].T
    uvi = res["i8"]["U"] @ res["i8"]["V"].T
    out = dict(config=name,
               G_maxdiff_rel=float(np.abs(Gd - Gi).max() / scale),
               G_symmetric=bool(np.array_equal(Gi, Gi.T)),
               UV_rel=float(np.linalg.norm(uvd - uvi) / np.linalg.norm(uvd)),
               e=(res["dfma"]["rep"].e, res["i8"]["rep"].e),
               gram_rank=(res["dfma"]["rep"].gram_rank, res["i8"]["rep"].gram_rank),
               gram_ms=(round(float(res["dfma"]["st"][2]), 4), round(float(res["i8"]["st"][2]), 4)),
               total_ms=(round(float(res["dfma"]["st"][6]), 4), round(float(res["i8"]["st"][6]), 4)),
               stage_ms_i8=[round(float(x), 4) for x in res["i8"]["st"]])
    print(json.dumps(out), flush=True)
