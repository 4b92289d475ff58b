"""Config-4 stage timings from a device-generated instance (no host generation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm  # noqa: E402

ctx = rsm.Context(0)
ctx.generate(1048576, 2048, 8, 0.9, 1e-3, 0)
cfg = rsm.RsmConfig(rank=8, mode=rsm.Mode.M2, block=9, plan=rsm.TrialPlan(65536), seed=0)
for _ in range(3):
    _, rep = ctx.decompose(cfg, fetch=False)
print([round(x, 3) for x in ctx.stage_ms()], rep.e, rep.gram_rank)
