"""ctypes binding of oracle/_ref/libref.so: the reference's own sources
(/root/reference/proj/src) compiled with the builder-written shims in
oracle/ref_shim. TEST INFRASTRUCTURE ONLY (pins the C restatement; serves as
the "reference" CPU baseline)."""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libref.so")
_lib = None


def available():
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB)
        P, i64, u64, i32, d = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_double
        L.ref_generate.argtypes = [i64, i64, i64, d, d, u64, P, P, P]
        L.ref_select.argtypes = [P, P, i64, i64, C.c_int, i64, i64, u64, u64, P, P, C.POINTER(u64), C.POINTER(u64)]
        L.ref_harvest.argtypes = [P, P, i64, i64, C.c_int, i64, i64, i64, i64, u64, u64, C.c_int, C.c_int, P,
                                  C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(d)]
        L.ref_small_singular_vectors.argtypes = [P, i64, i64, i64, i64, P, P]
        L.ref_solve_v.argtypes = [P, i64, i64, d, P, C.POINTER(i64), C.POINTER(i32), C.POINTER(d)]
        L.ref_solve_u.argtypes = [P, P, i64, i64, P, i64, C.c_int, P, C.POINTER(i64), C.POINTER(d)]
        L.ref_decompose.argtypes = [P, P, i64, i64, i64, C.c_int, i64, i64, u64, d, u64, d, i64, C.c_int, P, P,
                                    C.POINTER(d), P, P, C.POINTER(d)]
        L.ref_als.argtypes = [P, P, i64, i64, i64, i64, u64, C.c_int, P, P, C.POINTER(i64), C.POINTER(d)]
        L.ref_masked_residual_norm.restype = d
        L.ref_masked_residual_norm.argtypes = [P, P, i64, i64, P, P, i64]
        L.ref_have_io.restype = C.c_int
        if L.ref_have_io():
            L.ref_load_matrix.argtypes = [C.c_char_p, C.POINTER(i64), C.POINTER(i64), P, P, i64]
            L.ref_save_matrix.argtypes = [C.c_char_p, P, P, i64, i64]
            L.ref_dataset_checksum.argtypes = [P, P, i64, i64, C.POINTER(u64)]
            L.ref_serialize_report.argtypes = [i64, C.c_int, i64, i64, u64, d, u64, d, C.c_int, d, u64, u64, u64,
                                               i64, i64, C.c_int, d, u64, C.c_char_p, i64, C.POINTER(i64)]
            L.ref_reserialize_report.argtypes = [C.c_char_p, C.c_char_p, i64, C.POINTER(i64)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class RefError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"reference raised errc exit code {code}")
        self.code = code


def _chk(st):
    if st:
        raise RefError(st)


def generate(m, n, r, rho, sigma, seed, with_basis=False):
    Y = np.zeros((m, n))
    W = np.zeros((m, n), np.uint8)
    B = np.zeros((n, r)) if with_basis else None
    _chk(lib().ref_generate(m, n, r, rho, sigma, seed, _p(Y), _p(W), _p(B)))
    return (Y, W, B) if with_basis else (Y, W)


def select(Y, W, mode, block, min_count, seed, trials):
    m, n = Y.shape
    ids = np.zeros(trials, np.uint64)
    qs = np.zeros(trials, np.int64)
    att, acc = C.c_uint64(), C.c_uint64()
    _chk(lib().ref_select(_p(Y), _p(W), m, n, mode, block, min_count, seed, trials, _p(ids), _p(qs),
                          C.byref(att), C.byref(acc)))
    return ids[:acc.value], qs[:acc.value], att.value, acc.value


def harvest(Y, W, p, trials, workers=0, serial=False, timed=False):
    m, n = Y.shape
    G = np.zeros((n, n))
    att, acc, z, secs = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_double()
    _chk(lib().ref_harvest(_p(Y), _p(W), m, n, p.mode, p.block, p.ell, p.rank, p.min_count, p.seed, trials,
                           workers, 1 if serial else 0, _p(G), C.byref(att), C.byref(acc), C.byref(z),
                           C.byref(secs)))
    out = (G, att.value, acc.value, z.value)
    return out + (secs.value,) if timed else out


def small_singular_vectors(S, r, ell):
    S = np.ascontiguousarray(S, np.float64)
    p, q = S.shape
    zeta = np.zeros((ell, q))
    sv = np.zeros(ell)
    _chk(lib().ref_small_singular_vectors(_p(S), p, q, r, ell, _p(zeta), _p(sv)))
    return zeta, sv


def solve_v(G, r, tol=1e-9, timed=False, gate_failure_ok=False):
    """gate_failure_ok: when the reference's rank gate raises after dsyev,
    return (None, None, None, secs) instead of raising (timing use)."""
    G = np.ascontiguousarray(G, np.float64)
    n = G.shape[0]
    V = np.zeros((n, r))
    gr, bl, secs = C.c_int64(), C.c_int32(), C.c_double(-1.0)
    st = lib().ref_solve_v(_p(G), n, r, tol, _p(V), C.byref(gr), C.byref(bl), C.byref(secs))
    if st and gate_failure_ok and secs.value >= 0.0:
        return None, None, None, secs.value
    _chk(st)
    out = (V, gr.value, bool(bl.value))
    return out + (secs.value,) if timed else out


def solve_u(Y, W, V, r, workers=0, timed=False):
    """solve_u followed by masked_residual_norm (the e pass of decompose)."""
    m, n = Y.shape
    U = np.zeros((m, r))
    fl, secs = C.c_int64(), C.c_double()
    _chk(lib().ref_solve_u(_p(Y), _p(W), m, n, _p(np.ascontiguousarray(V)), r, workers, _p(U), C.byref(fl),
                           C.byref(secs)))
    return (U, fl.value, secs.value) if timed else (U, fl.value)


def als(Y, W, r, iterations, seed, workers=0):
    """The reference's baseline_als -> (U, V, flagged, e)."""
    m, n = Y.shape
    U = np.zeros((m, r))
    V = np.zeros((n, r))
    fl, e = C.c_int64(), C.c_double()
    _chk(lib().ref_als(_p(Y), _p(W), m, n, r, iterations, seed, workers, _p(U), _p(V), C.byref(fl), C.byref(e)))
    return U, V, fl.value, e.value


def decompose(Y, W, rank, trials, mode=0, block=0, vectors_per_trial=0, seed=0, tol=1e-9, min_dim=0,
              epsilon=0.99, workers=0):
    m, n = Y.shape
    U = np.zeros((m, rank))
    V = np.zeros((n, rank))
    e, wall = C.c_double(), C.c_double()
    u64 = np.zeros(3, np.uint64)
    i64 = np.zeros(3, np.int64)
    _chk(lib().ref_decompose(_p(Y), _p(W), m, n, rank, mode, block, vectors_per_trial, trials, epsilon, seed, tol,
                             min_dim, workers, _p(U), _p(V), C.byref(e), _p(u64), _p(i64), C.byref(wall)))
    rep = dict(e=e.value, trials_attempted=int(u64[0]), trials_accepted=int(u64[1]), z=int(u64[2]),
               underdetermined_rows=int(i64[0]), gram_rank=int(i64[1]), borderline=bool(i64[2]), wall_time=wall.value)
    return U, V, rep


# ---- io.cpp (src/io.cpp:56-254), when build_ref.sh found the JSON header ----

def have_io():
    return available() and bool(lib().ref_have_io())


def load_matrix(path):
    """rsm::load_matrix -> (Y, W); raises RefError with the reference's exit code."""
    m, n = C.c_int64(), C.c_int64()
    _chk(lib().ref_load_matrix(os.fsencode(path), C.byref(m), C.byref(n), None, None, 0))
    Y = np.zeros((m.value, n.value))
    W = np.zeros((m.value, n.value), np.uint8)
    _chk(lib().ref_load_matrix(os.fsencode(path), C.byref(m), C.byref(n), _p(Y), _p(W), Y.size))
    return Y, W


def save_matrix(Y, W, path):
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.uint8)
    _chk(lib().ref_save_matrix(os.fsencode(path), _p(Y), _p(W), Y.shape[0], Y.shape[1]))


def dataset_checksum(Y, W):
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.uint8)
    out = C.c_uint64()
    _chk(lib().ref_dataset_checksum(_p(Y), _p(W), Y.shape[0], Y.shape[1], C.byref(out)))
    return int(out.value)


def serialize_report(rank, mode, block, vectors_per_trial, trials, epsilon, seed, tol, workers, e, attempted,
                     accepted, z, underdetermined, gram_rank, borderline, wall, checksum):
    """make_report + serialize_report (mode: 0 = m1, 1 = m2)."""
    buf = C.create_string_buffer(1 << 16)
    ln = C.c_int64()
    _chk(lib().ref_serialize_report(rank, mode, block, vectors_per_trial, trials, epsilon, seed, tol, workers, e,
                                    attempted, accepted, z, underdetermined, gram_rank, int(borderline), wall,
                                    checksum, buf, len(buf), C.byref(ln)))
    return buf.value.decode()


def reserialize_report(text):
    buf = C.create_string_buffer(1 << 16)
    ln = C.c_int64()
    _chk(lib().ref_reserialize_report(text.encode(), buf, len(buf), C.byref(ln)))
    return buf.value.decode()
