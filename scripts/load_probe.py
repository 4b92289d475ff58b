"""Host-side timing of rsm_ctx_load (pinned inputs, config 3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1411_0814_b200 import rsm
M = rsm.generate(131072, 1024, 4, 0.8, 1e-3, 0)
Yt = torch.empty((131072, 1024), dtype=torch.float64, pin_memory=True); Yt.numpy()[...] = M.values
Wt = torch.empty((131072, 1024), dtype=torch.uint8, pin_memory=True); Wt.numpy()[...] = M.mask
ctx = rsm.Context(0)
for i in range(4):
    t = time.time(); ctx.load_arrays(Yt.numpy(), Wt.numpy()); print("load %.2f ms" % ((time.time() - t) * 1e3), flush=True)
