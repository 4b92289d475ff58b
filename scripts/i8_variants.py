"""Stage-3 (tcgen05) timing under experiment switches on config 3: diagnostic
modes (RSM_I8_DIAG: 1 loads only, 2 MMAs only) and K-chunk counts (RSM_I8_NK)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm  # noqa: E402

c = dict(m=131072, n=1024, r=4, rho=0.8, sigma=1e-3, block=5, T=16384, seed=0)
if len(sys.argv) > 1 and sys.argv[1] == "c4":
    c = dict(m=1048576, n=2048, r=8, rho=0.9, sigma=1e-3, block=9, T=65536, seed=0)
ctx = rsm.Context(0)
ctx.generate(c["m"], c["n"], c["r"], c["rho"], c["sigma"], c["seed"])
tp = rsm.TrialParams(rsm.Mode.M2, c["block"], 0, c["r"], c["r"] + 1, c["seed"])
variants = [dict(), dict(RSM_I8_DIAG="1"), dict(RSM_I8_DIAG="2"), dict(RSM_I8_NK="8"), dict(RSM_I8_NK="37"),
            ]
if os.environ.get("RSM_GRAM_SLICES"):
    variants = [dict()]
for v in variants:
    for k in ("RSM_I8_DIAG", "RSM_I8_NK"):
        os.environ.pop(k, None)
    os.environ.update(v)
    ts = []
    for _ in range(4):
        ctx.harvest_gram(tp, c["T"])
        ts.append(ctx.stage_ms())
    st = np.median(np.array(ts[1:]), axis=0)
    print(json.dumps(dict(variant=v, svd=round(float(st[1]), 4), gram=round(float(st[2]), 4))), flush=True)
