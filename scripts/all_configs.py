"""Per-config device timing of one decomposition (BASELINE.json configs 1-5) on
cuda:0: inputs from the device generator (configs 1-4; same instance as the
host generator up to a few ulps) or the host track generator (config 5), the
decomposition repeated and the last run's stage split printed."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm  # noqa: E402

STAGES = ["select", "svd", "gram", "gram_reduce", "solve_v", "solve_u", "total"]
CFGS = {
    "config1": dict(m=2000, n=200, r=3, rho=0.8, sigma=1e-3, mode=rsm.Mode.M2, block=4, T=2000, seed=0),
    "config2": dict(m=20000, n=500, r=5, rho=0.7, sigma=1e-2, mode=rsm.Mode.M1, block=6, T=4096, seed=1),
    "config3": dict(m=131072, n=1024, r=4, rho=0.8, sigma=1e-3, mode=rsm.Mode.M2, block=5, T=16384, seed=0),
    "config4": dict(m=1048576, n=2048, r=8, rho=0.9, sigma=1e-3, mode=rsm.Mode.M2, block=9, T=65536, seed=0),
    "config5": dict(tracks=(8192, 1024, 128, 512), r=4, sigma=1e-3, mode=rsm.Mode.M2, block=5, T=8192, seed=0),
}
ctx = rsm.Context(0)
for name, c in CFGS.items():
    if "tracks" in c:
        pts, frames, wmin, wmax = c["tracks"]
        ctx.load(rsm.generate_tracks(pts, frames, wmin, wmax, c["sigma"], c["seed"]))
        shape = (pts, 2 * frames)
    else:
        ctx.generate(c["m"], c["n"], c["r"], c["rho"], c["sigma"], c["seed"])
        shape = (c["m"], c["n"])
    cfg = rsm.RsmConfig(rank=c["r"], mode=c["mode"], block=c["block"], plan=rsm.TrialPlan(c["T"]), seed=c["seed"])
    out = {"config": name, "shape": shape, "trials": c["T"]}
    try:
        for _ in range(4):
            t0 = time.time()
            _, rep = ctx.decompose(cfg, fetch=False)
            wall = (time.time() - t0) * 1e3
        st = ctx.stage_ms()
        out.update(stage_ms={k: round(v, 4) for k, v in zip(STAGES, st)}, wall_ms=round(wall, 3),
                   submatrices_per_s=round(c["T"] / (st[6] * 1e-3)), e=rep.e, gram_rank=rep.gram_rank,
                   accepted=rep.trials_accepted, attempted=rep.trials_attempted,
                   underdetermined_rows=rep.underdetermined_rows)
    except rsm.Error as ex:
        out.update(status=ex.code.name, message=str(ex))
    print(json.dumps(out), flush=True)
