import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1411_0814_b200 import rsm
pts, frames, wmin, wmax, T = [int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (8192, 1024, 128, 512, 8192))]
M = rsm.generate_tracks(pts, frames, wmin, wmax, 1e-3, 0)
ctx = rsm.Context(0); ctx.load(M)
p = rsm.TrialParams(rsm.Mode.M2, 5, 0, 4, 5, 0)
H = ctx.harvest_gram(p, T)
print(H.attempted, H.accepted)
G = H.gram
zero_rows = int((np.abs(G).max(axis=1) == 0).sum())
w = np.linalg.eigvalsh(G)
tau = 1e-9 * w[-1]
print("zero rows", zero_rows, "count<=tau", int((w <= tau).sum()), "lmax", w[-1], "low", w[:8], "w[r..r+12]", w[4:16])
