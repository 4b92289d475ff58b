"""Generate the golden fixtures from the reference itself (oracle/_ref, the
reference sources built with the builder shims). Run here, where
/root/reference exists:  python tests/golden/make_golden.py
The fixtures pin the C oracle on machines without /root/reference."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import refbind as R  # noqa: E402

CASES = {
    # config 1 shape (row branch), trial count reduced so the literal Gram stays small
    "config1_small.npz": dict(m=2000, n=200, r=3, rho=0.8, sigma=1e-3, mode=1, block=4, T=600, seed=0),
    # config 2 shape scaled down (column branch)
    "config2_small.npz": dict(m=2000, n=100, r=5, rho=0.7, sigma=1e-2, mode=0, block=6, T=800, seed=1),
}


def main():
    for name, c in CASES.items():
        Y, W = R.generate(c["m"], c["n"], c["r"], c["rho"], c["sigma"], c["seed"])
        min_count = c["r"] + 1
        ids, qs, att, acc = R.select(Y, W, c["mode"], c["block"], min_count, c["seed"], c["T"])

        class P:
            pass
        p = P()
        p.mode, p.block, p.rank, p.min_count, p.seed = c["mode"], c["block"], c["r"], min_count, c["seed"]
        p.ell = 0 if c["mode"] == 1 else c["block"] - c["r"]
        G, att2, acc2, z = R.harvest(Y, W, p, c["T"], serial=True)
        U, V, rep = R.decompose(Y, W, c["r"], c["T"], mode=c["mode"], block=c["block"], seed=c["seed"])
        np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), name),
                            known=int(W.sum()), ids=ids, qs=qs, attempted=att, G=G, z=z, U=U, V=V,
                            gram_rank=rep["gram_rank"], underdetermined=rep["underdetermined_rows"], e=rep["e"],
                            **{k: v for k, v in c.items()})
        print(name, "attempted", att, "accepted", acc, "z", z, "e", rep["e"], "gram_rank", rep["gram_rank"])


if __name__ == "__main__":
    main()
