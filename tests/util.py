"""Shared helpers for the parity tests (oracle = CPU checker)."""
import numpy as np


def rel_fro(a, b):
    d = np.linalg.norm(a - b)
    s = np.linalg.norm(b)
    return d / s if s > 0 else d


def max_angle_sin(A, B):
    """Largest principal-angle sine between the spans of orthonormal bases
    (tests/oracles.hpp:35-41 of the reference)."""
    R = A - B @ (B.T @ A)
    return 0.0 if np.linalg.norm(R) == 0 else np.linalg.svd(R, compute_uv=False)[0]


def random_masked(m, n, rho, seed):
    """tests/oracles.hpp:45-57: Rng(seed, 77, row) -> unit then normal per cell."""
    from oracle import oracle as O
    import ctypes as C
    L = O.lib()
    vals = np.full((m, n), np.nan)
    mask = np.zeros((m, n), np.uint8)
    for i in range(m):
        st = C.c_uint64(L.orc_rng_state(seed, 77, i))
        for j in range(n):
            u = L.orc_next_unit(C.byref(st))
            v = L.orc_next_normal(C.byref(st))
            if u <= rho:
                vals[i, j] = v
                mask[i, j] = 1
    return vals, mask
