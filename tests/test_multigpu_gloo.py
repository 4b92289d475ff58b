"""CPU, world size 2 (gloo): the multi-GPU decomposition's host logic.

The B200 path shards one decomposition across ranks:
every rank runs the selection redundantly, takes accepted trials
[T*g/G, T*(g+1)/G) (rsm_shard_range, the library's own split), accumulates a
partial Gram, and one all-reduce (NCCL on the GPUs; gloo here) completes G;
stage 5 is row-sharded and the row blocks gathered. This test runs that
schedule with the CPU oracle as the per-rank compute and checks it reproduces
the single-process oracle (G to rounding, z and counts exactly, U exactly).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _partial_gram(Y, W, p, ids, lo, hi):
    from oracle import oracle as O
    n = Y.shape[1]
    G = np.zeros((n, n))
    z = 0
    for a in ids[lo:hi]:
        rows, cols = O.sample(W, p.mode, p.block, p.seed, int(a))
        if p.mode == 1:
            S = Y[np.ix_(rows, cols)]
            sup = cols
            ell = len(cols) - p.rank
        else:
            S = Y[np.ix_(cols, rows)]
            sup = rows
            ell = p.ell
        zeta, _ = O.small_singular_vectors(S, p.rank, ell)
        for v in zeta:  # literal accumulation, spectra.cpp:7-23
            G[np.ix_(sup, sup)] += np.outer(v, v)
            z += 1
    return G, z


def _worker(rank, port, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from oracle import oracle as O
        from paper_1411_0814_b200 import rsm
        m, n, r, T = 300, 40, 3, 240
        Y, W = O.generate(m, n, r, 0.8, 1e-2, 5)
        p = O.trial_params(r, mode, m, n, seed=5)
        ids, qs, att, acc = O.select(W, p, T)  # redundant on every rank
        lo, hi = rsm.shard_range(acc, WORLD, rank)
        Gp, zp = _partial_gram(Y, W, p, ids, lo, hi)
        Gt = torch.from_numpy(Gp)
        dist.all_reduce(Gt)
        zt = torch.tensor([zp], dtype=torch.int64)
        dist.all_reduce(zt)
        V, gr, bl, _ = O.solve_v(Gt.numpy(), r)
        rlo, rhi = rsm.shard_range(m, WORLD, rank)
        Us, fl = O.solve_u(Y[rlo:rhi], W[rlo:rhi], V, r)
        parts = [None] * WORLD
        dist.all_gather_object(parts, (rlo, rhi, Us, fl))
        if rank == 0:
            G_full, att_f, acc_f, z_f = O.harvest(Y, W, p, T)
            U_full, fl_full = O.solve_u(Y, W, V, r)
            U_cat = np.zeros_like(U_full)
            fl_cat = 0
            for a, b, u, f in parts:
                U_cat[a:b] = u
                fl_cat += f
            out.put(dict(gdiff=float(np.abs(Gt.numpy() - G_full).max()), gmax=float(np.abs(G_full).max()),
                         z=int(zt.item()), z_full=z_f, att=(att, att_f), acc=(acc, acc_f),
                         udiff=float(np.abs(U_cat - U_full).max()), fl=(fl_cat, fl_full),
                         cover=sorted((a, b) for a, b, _, _ in parts)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", [1, 0])
def test_two_rank_schedule_reproduces_single_process(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000 + 7 * mode
    procs = [ctx.Process(target=_worker, args=(r, port, mode, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res["att"][0] == res["att"][1] and res["acc"][0] == res["acc"][1]
    assert res["z"] == res["z_full"]
    assert res["gdiff"] <= 1e-12 * max(1.0, res["gmax"])
    assert res["udiff"] == 0.0 and res["fl"][0] == res["fl"][1]
    assert res["cover"] == [(0, 150), (150, 300)]


def test_shard_range_partitions():
    from paper_1411_0814_b200 import rsm
    for total in [0, 1, 7, 16384, 1048576]:
        for world in [1, 2, 3, 8]:
            spans = [rsm.shard_range(total, world, g) for g in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
