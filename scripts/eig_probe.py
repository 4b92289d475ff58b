import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm
M = rsm.generate(131072, 1024, 4, 0.8, 1e-3, 0)
ctx = rsm.Context(0); ctx.load(M)
cfg = rsm.RsmConfig(rank=4, mode=rsm.Mode.M2, block=5, plan=rsm.TrialPlan(16384), seed=0)
for i in range(3):
    ctx.decompose(cfg, fetch=False)
st = ctx.solver_stats(); ms = ctx.stage_ms()
print("stage ms", [round(x, 3) for x in ms])
clk = 1.965e9
print({k: (round(v / clk * 1e6, 1) if k.startswith("cyc") else v) for k, v in st.items()}, "(cyc_* in us at 1965 MHz)")
