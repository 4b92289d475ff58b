"""ctypes binding of oracle/liborc.so (the plain-C restatement of the
reference hot path, oracle/rsm_oracle.c). TEST INFRASTRUCTURE ONLY: it is the
checker the B200 product is compared against, never the thing measured or
shipped."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liborc.so")
_lib = None


class Params(C.Structure):
    _fields_ = [("mode", C.c_int32), ("block", C.c_int64), ("ell", C.c_int64), ("rank", C.c_int64),
                ("min_count", C.c_int64), ("seed", C.c_uint64)]


class Config(C.Structure):
    _fields_ = [("rank", C.c_int64), ("mode", C.c_int32), ("block", C.c_int64),
                ("vectors_per_trial", C.c_int64), ("trials", C.c_uint64), ("epsilon", C.c_double),
                ("seed", C.c_uint64), ("gram_rank_tol", C.c_double), ("min_dim", C.c_int64)]


class Report(C.Structure):
    _fields_ = [("e", C.c_double), ("trials_attempted", C.c_uint64), ("trials_accepted", C.c_uint64),
                ("z", C.c_uint64), ("underdetermined_rows", C.c_int64), ("gram_rank", C.c_int64),
                ("borderline", C.c_int32)]


def build():
    subprocess.run(["make", "-s", "-C", HERE, "liborc.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(HERE, "rsm_oracle.c")
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
            build()
        L = C.CDLL(LIB)
        P, i64, u64, i32, d = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_double
        L.orc_rng_state.restype = u64
        L.orc_rng_state.argtypes = [u64, u64, u64]
        L.orc_next_u64.restype = u64
        L.orc_next_u64.argtypes = [C.POINTER(u64)]
        L.orc_next_unit.restype = d
        L.orc_next_unit.argtypes = [C.POINTER(u64)]
        L.orc_next_below.restype = u64
        L.orc_next_below.argtypes = [C.POINTER(u64), u64]
        L.orc_next_normal.restype = d
        L.orc_next_normal.argtypes = [C.POINTER(u64)]
        L.orc_draw.argtypes = [i64, i64, C.POINTER(u64), P]
        L.orc_sample.restype = i64
        L.orc_sample.argtypes = [P, i64, i64, i32, i64, u64, u64, P, P]
        L.orc_trial_params.restype = C.c_int
        L.orc_trial_params.argtypes = [C.POINTER(Config), i64, i64, C.POINTER(Params)]
        L.orc_select.restype = C.c_int
        L.orc_select.argtypes = [P, i64, i64, C.POINTER(Params), u64, P, P, C.POINTER(u64), C.POINTER(u64)]
        L.orc_small_singular_vectors.restype = C.c_int
        L.orc_small_singular_vectors.argtypes = [P, i64, i64, i64, i64, P, P]
        L.orc_harvest.restype = C.c_int
        L.orc_harvest.argtypes = [P, P, i64, i64, C.POINTER(Params), u64, P, C.POINTER(u64), C.POINTER(u64),
                                  C.POINTER(u64)]
        L.orc_solve_v.restype = C.c_int
        L.orc_solve_v.argtypes = [P, i64, i64, d, P, C.POINTER(i64), C.POINTER(i32), P]
        L.orc_solve_u.restype = C.c_int
        L.orc_solve_u.argtypes = [P, P, i64, i64, P, i64, P, C.POINTER(i64)]
        L.orc_solve_row.restype = C.c_int
        L.orc_solve_row.argtypes = [P, P, i64, i64, P]
        L.orc_masked_residual_norm.restype = d
        L.orc_masked_residual_norm.argtypes = [P, P, i64, i64, P, P, i64]
        L.orc_decompose.restype = C.c_int
        L.orc_decompose.argtypes = [P, P, i64, i64, C.POINTER(Config), P, P, C.POINTER(Report)]
        L.orc_generate_rows.argtypes = [i64, i64, i64, d, d, u64, i64, i64, P, P]
        L.orc_generate_tracks.argtypes = [i64, i64, i64, i64, d, u64, P, P]
        L.orc_als.restype = C.c_int
        L.orc_als.argtypes = [P, P, i64, i64, i64, i64, u64, P, P, C.POINTER(i64), C.POINTER(d)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(what or f"oracle status {code}")
        self.code = code


def _chk(st):
    if st:
        raise OracleError(st)


def rng_state(seed, tag, index):
    return lib().orc_rng_state(seed, tag, index)


def draw(pool, count, seed, attempt):
    st = C.c_uint64(lib().orc_rng_state(seed, 5, attempt))
    out = np.zeros(count, np.int64)
    lib().orc_draw(pool, count, C.byref(st), _p(out))
    return out


def sample(mask, mode, block, seed, attempt):
    m, n = mask.shape
    mask = np.ascontiguousarray(mask, np.uint8)
    idx = np.zeros(block, np.int64)
    surv = np.zeros(max(m, n), np.int64)
    q = lib().orc_sample(_p(mask), m, n, mode, block, seed, attempt, _p(idx), _p(surv))
    return idx, surv[:q]


def trial_params(rank, mode, m, n, block=0, vectors_per_trial=0, seed=0, min_dim=0):
    cfg = Config(rank, mode, block, vectors_per_trial, 1, 0.99, seed, 1e-9, min_dim)
    p = Params()
    _chk(lib().orc_trial_params(C.byref(cfg), m, n, C.byref(p)))
    return p


def select(mask, p, trials):
    m, n = mask.shape
    mask = np.ascontiguousarray(mask, np.uint8)
    ids = np.zeros(trials, np.uint64)
    qs = np.zeros(trials, np.int64)
    att, acc = C.c_uint64(), C.c_uint64()
    _chk(lib().orc_select(_p(mask), m, n, C.byref(p), trials, _p(ids), _p(qs), C.byref(att), C.byref(acc)))
    return ids[:acc.value], qs[:acc.value], att.value, acc.value


def small_singular_vectors(S, r, ell):
    S = np.ascontiguousarray(S, np.float64)
    p, q = S.shape
    zeta = np.zeros((ell, q))
    sv = np.zeros(ell)
    _chk(lib().orc_small_singular_vectors(_p(S), p, q, r, ell, _p(zeta), _p(sv)))
    return zeta, sv


def harvest(Y, mask, p, trials):
    m, n = Y.shape
    G = np.zeros((n, n))
    att, acc, z = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _chk(lib().orc_harvest(_p(np.ascontiguousarray(Y)), _p(np.ascontiguousarray(mask, np.uint8)), m, n,
                           C.byref(p), trials, _p(G), C.byref(att), C.byref(acc), C.byref(z)))
    return G, att.value, acc.value, z.value


def solve_v(G, r, tol=1e-9):
    G = np.array(G, dtype=np.float64, copy=True, order="C")
    n = G.shape[0]
    V = np.zeros((n, r))
    w = np.zeros(n)
    gr, bl = C.c_int64(), C.c_int32()
    _chk(lib().orc_solve_v(_p(G), n, r, tol, _p(V), C.byref(gr), C.byref(bl), _p(w)))
    return V, gr.value, bool(bl.value), w


def solve_u(Y, mask, V, r):
    m, n = Y.shape
    U = np.zeros((m, r))
    fl = C.c_int64()
    _chk(lib().orc_solve_u(_p(np.ascontiguousarray(Y)), _p(np.ascontiguousarray(mask, np.uint8)), m, n,
                           _p(np.ascontiguousarray(V, np.float64)), r, _p(U), C.byref(fl)))
    return U, fl.value


def generate_tracks(points, frames, wmin, wmax, sigma, seed):
    Y = np.zeros((points, 2 * frames))
    W = np.zeros((points, 2 * frames), np.uint8)
    lib().orc_generate_tracks(points, frames, wmin, wmax, sigma, seed, _p(Y), _p(W))
    return Y, W


def als(Y, mask, r, iterations, seed):
    """baseline_als restatement (als.cpp:11-44) -> (U, V, flagged, e)."""
    m, n = Y.shape
    U = np.zeros((m, r))
    V = np.zeros((n, r))
    fl = C.c_int64()
    e = C.c_double()
    _chk(lib().orc_als(_p(np.ascontiguousarray(Y)), _p(np.ascontiguousarray(mask, np.uint8)), m, n, r, iterations,
                       seed, _p(U), _p(V), C.byref(fl), C.byref(e)))
    return U, V, fl.value, e.value


def masked_residual_norm(Y, mask, U, V):
    m, n = Y.shape
    r = U.shape[1]
    return lib().orc_masked_residual_norm(_p(np.ascontiguousarray(Y)), _p(np.ascontiguousarray(mask, np.uint8)),
                                          m, n, _p(np.ascontiguousarray(U)), _p(np.ascontiguousarray(V)), r)


def decompose(Y, mask, rank, trials, mode=0, block=0, vectors_per_trial=0, seed=0, tol=1e-9, min_dim=0,
              epsilon=0.99):
    m, n = Y.shape
    cfg = Config(rank, mode, block, vectors_per_trial, trials, epsilon, seed, tol, min_dim)
    U = np.zeros((m, max(rank, 1)))
    V = np.zeros((n, max(rank, 1)))
    rep = Report()
    _chk(lib().orc_decompose(_p(np.ascontiguousarray(Y)), _p(np.ascontiguousarray(mask, np.uint8)), m, n,
                             C.byref(cfg), _p(U), _p(V), C.byref(rep)))
    return U, V, rep


def generate(m, n, r, rho, sigma, seed, row0=0, rows=None):
    rows = m - row0 if rows is None else rows
    Y = np.zeros((rows, n))
    W = np.zeros((rows, n), np.uint8)
    lib().orc_generate_rows(m, n, r, rho, sigma, seed, row0, rows, _p(Y), _p(W))
    return Y, W
