"""Device generator timing at config 3 and config 4 (rsm_ctx_generate)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm  # noqa: E402

ctx = rsm.Context(0)
for name, (m, n, r, rho) in {"c3": (131072, 1024, 4, 0.8), "c4": (1048576, 2048, 8, 0.9)}.items():
    for rep in range(2):
        t0 = time.time()
        ctx.generate(m, n, r, rho, 1e-3, 0)
        dt = time.time() - t0
    print(f"{name}: device generate {m}x{n} r={r}: {dt * 1e3:.1f} ms (incl. load bookkeeping)", flush=True)
t0 = time.time()
M = rsm.generate(131072, 1024, 4, 0.8, 1e-3, 0)
print(f"c3: host generate {(time.time() - t0) * 1e3:.1f} ms")
