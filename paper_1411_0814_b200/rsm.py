"""Python host mirror of the reference RSM API over the B200 C-ABI.

The reference is a C++ library (``rsm::`` in /root/reference/proj/include/rsm);
its drop-in for C++ callers is ``include/rsm_gpu/rsm.hpp`` (header-only, over
the same C-ABI ``include/rsm_b200.h``). This module gives the same surface to
Python callers and to the tests:

    MaskedMatrix, Mode, RsmConfig, TrialPlan, TrialParams, DecompositionReport,
    Factorization, Error/errc, trial_params, harvest_gram, solve_v, solve_u,
    decompose, masked_residual_norm, generate

with the reference's argument meaning and error behaviour (``Error`` carries
an ``errc``; codes are rsm::exit_code values, include/rsm/error.hpp:38-46).
Every compute call goes to the sm_100a library; there is no CPU fallback and
importing fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "librsm_b200.so")


class errc(enum.IntEnum):
    """rsm::errc (include/rsm/error.hpp:8-13) with exit-code values."""

    internal = 1
    invalid_config = 2
    parse_io = 3
    insufficient_coverage = 4


class Error(RuntimeError):
    """rsm::Error (include/rsm/error.hpp:15-22)."""

    def __init__(self, code: int, what: str):
        super().__init__(what)
        self.code = errc(code)


class Mode(enum.IntEnum):
    M1 = 0  # column branch
    M2 = 1  # row branch


class _Config(C.Structure):
    _fields_ = [("rank", C.c_int64), ("mode", C.c_int32), ("block", C.c_int64),
                ("vectors_per_trial", C.c_int64), ("trials", C.c_uint64), ("epsilon", C.c_double),
                ("seed", C.c_uint64), ("gram_rank_tol", C.c_double), ("min_dim", C.c_int64),
                ("workers", C.c_int32)]


class _TrialParams(C.Structure):
    _fields_ = [("mode", C.c_int32), ("block", C.c_int64), ("ell", C.c_int64), ("rank", C.c_int64),
                ("min_count", C.c_int64), ("seed", C.c_uint64)]


class _Report(C.Structure):
    _fields_ = [("e", C.c_double), ("trials_attempted", C.c_uint64), ("trials_accepted", C.c_uint64),
                ("z", C.c_uint64), ("underdetermined_rows", C.c_int64), ("gram_rank", C.c_int64),
                ("borderline_rank_gate", C.c_int32), ("wall_time", C.c_double)]


_P = C.c_void_p
_lib = None


def lib():
    """Load the sm_100a library (raises when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIBPATH):
        raise ImportError(f"{_LIBPATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
    L = C.CDLL(_LIBPATH)
    i64, u64, i32, dbl = C.c_int64, C.c_uint64, C.c_int32, C.c_double
    sig = {
        "rsm_config_default": (None, [C.POINTER(_Config)]),
        "rsm_last_error": (C.c_char_p, [_P]),
        "rsm_ctx_create": (i32, [C.POINTER(_P), C.c_int, C.c_int, C.c_int, _P]),
        "rsm_ctx_destroy": (i32, [_P]),
        "rsm_nccl_unique_id": (i32, [_P]),
        "rsm_ctx_stream": (_P, [_P]),
        "rsm_ctx_load": (i32, [_P, _P, _P, i64, i64]),
        "rsm_ctx_load_device": (i32, [_P, _P, _P, i64, i64]),
        "rsm_ctx_generate": (i32, [_P, i64, i64, i64, dbl, dbl, u64]),
        "rsm_ctx_fetch_matrix": (i32, [_P, _P, _P, C.POINTER(i64)]),
        "rsm_ctx_decompose": (i32, [_P, C.POINTER(_Config), _P, _P, C.POINTER(_Report)]),
        "rsm_ctx_als": (i32, [_P, i64, i64, u64, _P, _P, C.POINTER(_Report)]),
        "rsm_ctx_fetch_factors": (i32, [_P, _P, _P]),
        "rsm_ctx_select": (i32, [_P, C.POINTER(_TrialParams), u64, _P, _P, C.POINTER(u64), C.POINTER(u64)]),
        "rsm_ctx_harvest_gram": (i32, [_P, C.POINTER(_TrialParams), u64, _P, C.POINTER(u64), C.POINTER(u64),
                                       C.POINTER(u64)]),
        "rsm_ctx_solve_v": (i32, [_P, _P, i64, i64, dbl, _P, C.POINTER(i64), C.POINTER(i32), _P]),
        "rsm_ctx_solve_u": (i32, [_P, _P, i64, _P, C.POINTER(i64), C.POINTER(dbl)]),
        "rsm_ctx_stage_ms": (C.c_int, [_P, _P, C.c_int]),
        "rsm_ctx_launch_count": (i64, [_P]),
        "rsm_ctx_rerun_count": (i64, [_P]),
        "rsm_ctx_last_load_h2d_bytes": (i64, [_P]),
        "rsm_ctx_solver_stats": (C.c_int, [_P, _P, C.c_int]),
        "rsm_make_trial_params": (i32, [C.POINTER(_Config), i64, i64, C.POINTER(_TrialParams)]),
        "rsm_decompose": (i32, [_P, _P, i64, i64, C.POINTER(_Config), _P, _P, C.POINTER(_Report)]),
        "rsm_als": (i32, [_P, _P, i64, i64, i64, i64, u64, _P, _P, C.POINTER(_Report)]),
        "rsm_harvest_gram": (i32, [_P, _P, i64, i64, C.POINTER(_TrialParams), u64, _P, C.POINTER(u64),
                                   C.POINTER(u64), C.POINTER(u64)]),
        "rsm_solve_v": (i32, [_P, i64, i64, dbl, _P, C.POINTER(i64), C.POINTER(i32)]),
        "rsm_solve_u": (i32, [_P, _P, i64, i64, _P, i64, _P, C.POINTER(i64)]),
        "rsm_masked_residual_norm": (i32, [_P, _P, i64, i64, _P, _P, i64, C.POINTER(dbl)]),
        "rsm_generate": (i32, [i64, i64, i64, dbl, dbl, u64, i64, i64, _P, _P]),
        "rsm_generate_tracks": (i32, [i64, i64, i64, i64, dbl, u64, i64, i64, _P, _P]),
        "rsm_load_matrix_csv": (i32, [C.c_char_p, C.POINTER(_P), C.POINTER(_P), C.POINTER(i64), C.POINTER(i64)]),
        "rsm_save_matrix_csv": (i32, [C.c_char_p, _P, _P, i64, i64]),
        "rsm_dataset_checksum": (i32, [_P, _P, i64, i64, C.POINTER(u64)]),
        "rsm_free": (None, [_P]),
        "rsm_fp64_peak_tflops": (i32, [C.c_int, C.POINTER(dbl)]),
        "rsm_dmma_peak_tflops": (i32, [C.c_int, C.POINTER(dbl)]),
        "rsm_shard_range": (None, [i64, C.c_int, C.c_int, C.POINTER(i64), C.POINTER(i64)]),
        "rsm_host_group_create": (i32, [C.c_int, C.POINTER(_P)]),
        "rsm_host_group_destroy": (i32, [_P]),
        "rsm_ctx_create_host_group": (i32, [C.POINTER(_P), C.c_int, _P, C.c_int]),
        "rsm_sample": (i32, [_P, _P, i64, i64, i32, i64, u64, u64, _P, _P, C.POINTER(i64)]),
        "rsm_small_singular_vectors": (i32, [_P, i64, i64, i64, i64, _P, _P]),
        "rsm_gram_update": (i32, [_P, i64, _P, i64, _P]),
        "rsm_masked_objective": (i32, [_P, _P, i64, i64, _P, _P, i64, i32, C.POINTER(dbl)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols():
    """Names the C-ABI header declares (used by the CPU symbol test)."""
    return ["rsm_config_default", "rsm_last_error", "rsm_ctx_create", "rsm_ctx_destroy", "rsm_nccl_unique_id",
            "rsm_ctx_stream", "rsm_ctx_load", "rsm_ctx_load_device", "rsm_ctx_generate", "rsm_ctx_fetch_matrix", "rsm_ctx_decompose", "rsm_ctx_fetch_factors", "rsm_ctx_als",
            "rsm_ctx_select", "rsm_ctx_harvest_gram", "rsm_ctx_solve_v", "rsm_ctx_solve_u", "rsm_ctx_stage_ms",
            "rsm_ctx_launch_count", "rsm_ctx_rerun_count", "rsm_ctx_last_load_h2d_bytes", "rsm_ctx_solver_stats", "rsm_make_trial_params", "rsm_decompose", "rsm_als", "rsm_harvest_gram", "rsm_solve_v",
            "rsm_solve_u", "rsm_masked_residual_norm", "rsm_generate", "rsm_generate_tracks", "rsm_load_matrix_csv",
            "rsm_save_matrix_csv", "rsm_dataset_checksum", "rsm_free", "rsm_fp64_peak_tflops",
            "rsm_dmma_peak_tflops", "rsm_shard_range", "rsm_host_group_create", "rsm_host_group_destroy",
            "rsm_ctx_create_host_group", "rsm_sample", "rsm_small_singular_vectors", "rsm_gram_update",
            "rsm_masked_objective"]


def _check(st: int, ctx=None):
    if st != 0:
        msg = lib().rsm_last_error(ctx)
        raise Error(st, (msg or b"").decode() or f"rsm error {st}")


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ---------------------------------------------------------------- data model

class MaskedMatrix:
    """rsm::MaskedMatrix (include/rsm/core.hpp:22-57): row-major FP64 values
    with NaN at hidden cells plus a uint8 mask (1 = known)."""

    def __init__(self, m: int, n: int, values=None, mask=None):
        if m < 1 or n < 1:
            raise Error(errc.invalid_config, "matrix dimensions must be positive")
        self.m, self.n = int(m), int(n)
        self.values = (np.full((m, n), np.nan) if values is None
                       else np.ascontiguousarray(values, dtype=np.float64).reshape(m, n))
        self.mask = (np.zeros((m, n), np.uint8) if mask is None
                     else np.ascontiguousarray(mask, dtype=np.uint8).reshape(m, n))

    @classmethod
    def from_arrays(cls, values, mask):
        v = np.asarray(values, dtype=np.float64)
        return cls(v.shape[0], v.shape[1], v, mask)

    def set(self, i, j, v):
        self.values[i, j] = v
        self.mask[i, j] = 1

    def known(self, i, j) -> bool:
        return bool(self.mask[i, j])

    def known_count(self) -> int:
        return int(self.mask.sum(dtype=np.int64))

    def transposed(self) -> "MaskedMatrix":
        t = MaskedMatrix(self.n, self.m)
        t.mask[...] = self.mask.T
        t.values[...] = np.where(self.mask.T != 0, self.values.T, np.nan)
        return t


@dataclass
class TrialPlan:
    """rsm::TrialPlan (include/rsm/planner.hpp:12-16); the device path runs
    explicit counts, `source` is recorded in the run report."""

    trials: int = 0
    epsilon: float = 0.99
    source: str = "explicit"


@dataclass
class RsmConfig:
    """rsm::RsmConfig (include/rsm/solver.hpp:13-23)."""

    rank: int = 0
    mode: Mode = Mode.M1
    block: int = 0
    vectors_per_trial: int = 0
    plan: TrialPlan = field(default_factory=TrialPlan)
    seed: int = 0
    gram_rank_tol: float = 1e-9
    min_dim: int = 0
    workers: int = 0

    def _c(self) -> _Config:
        return _Config(self.rank, int(self.mode), self.block, self.vectors_per_trial, self.plan.trials,
                       self.plan.epsilon, self.seed, self.gram_rank_tol, self.min_dim, self.workers)


@dataclass
class TrialParams:
    """rsm::TrialParams (include/rsm/solver.hpp:27-34)."""

    mode: Mode = Mode.M1
    block: int = 0
    ell: int = 0
    rank: int = 0
    min_count: int = 0
    seed: int = 0

    def _c(self) -> _TrialParams:
        return _TrialParams(int(self.mode), self.block, self.ell, self.rank, self.min_count, self.seed)


@dataclass
class DecompositionReport:
    """rsm::DecompositionReport (include/rsm/core.hpp:81-90)."""

    e: float = 0.0
    trials_attempted: int = 0
    trials_accepted: int = 0
    z: int = 0
    underdetermined_rows: int = 0
    gram_rank: int = 0
    borderline_rank_gate: bool = False
    wall_time: float = 0.0


@dataclass
class Factorization:
    """rsm::Factorization (include/rsm/core.hpp:60-79): u (m x r), v (n x r)."""

    m: int
    n: int
    r: int
    u: np.ndarray
    v: np.ndarray


@dataclass
class HarvestResult:
    gram: np.ndarray
    attempted: int
    accepted: int
    z: int


@dataclass
class SolveVResult:
    v: np.ndarray
    gram_rank: int
    borderline: bool


@dataclass
class SolveUResult:
    u: np.ndarray
    underdetermined_rows: int


def _report(r: _Report) -> DecompositionReport:
    return DecompositionReport(r.e, r.trials_attempted, r.trials_accepted, r.z, r.underdetermined_rows,
                               r.gram_rank, bool(r.borderline_rank_gate), r.wall_time)


# ------------------------------------------------------------------ context

class HostGroup:
    """In-process rank group whose collectives go through host memory
    (rsm_host_group_*): `world` Contexts, possibly on one GPU and each driven by
    its own thread, take the multi-rank code path without NCCL."""

    def __init__(self, world: int):
        h = C.c_void_p()
        _check(lib().rsm_host_group_create(world, C.byref(h)))
        self.h, self.world = h, world

    def close(self):
        if getattr(self, "h", None):
            lib().rsm_host_group_destroy(self.h)
            self.h = None


class Context:
    """A device context: owns the device-resident matrix, workspace, stream
    and (for world > 1) the NCCL communicator or a HostGroup membership."""

    def __init__(self, device: int = 0, world: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 host_group: "HostGroup | None" = None):
        L = lib()
        h = C.c_void_p()
        if host_group is not None:
            st = L.rsm_ctx_create_host_group(C.byref(h), device, host_group.h, rank)
        else:
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            st = L.rsm_ctx_create(C.byref(h), device, world, rank, C.cast(idbuf, C.c_void_p) if idbuf else None)
        _check(st)
        self.h = h
        self.m = self.n = 0

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().rsm_nccl_unique_id(C.cast(buf, C.c_void_p)))
        return buf.raw

    def close(self):
        if getattr(self, "h", None):
            lib().rsm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(lib().rsm_ctx_stream(self.h) or 0)

    def load(self, M: MaskedMatrix):
        _check(lib().rsm_ctx_load(self.h, _ptr(M.values), _ptr(M.mask), M.m, M.n), self.h)
        self.m, self.n = M.m, M.n

    def load_arrays(self, values: np.ndarray, mask: np.ndarray):
        """Load row-major FP64 values and a byte (uint8/bool) mask of the same
        shape. Non-contiguous views are copied (free for contiguous inputs);
        other dtypes or mismatched shapes raise invalid_config."""
        if values.ndim != 2 or values.dtype != np.float64:
            raise Error(errc.invalid_config, "values must be a 2-D float64 array")
        if mask.shape != values.shape or mask.dtype not in (np.uint8, np.bool_):
            raise Error(errc.invalid_config, "mask must be uint8/bool with the shape of values")
        values = np.ascontiguousarray(values)
        mask = np.ascontiguousarray(mask).view(np.uint8)
        m, n = values.shape
        _check(lib().rsm_ctx_load(self.h, _ptr(values), _ptr(mask), m, n), self.h)
        self.m, self.n = m, n

    def load_device(self, values_ptr: int, mask_ptr: int, m: int, n: int):
        _check(lib().rsm_ctx_load_device(self.h, values_ptr, mask_ptr, m, n), self.h)
        self.m, self.n = m, n

    def generate(self, m: int, n: int, r: int, rho: float, sigma: float, seed: int):
        """Device-side rsm::generate straight into this context."""
        _check(lib().rsm_ctx_generate(self.h, m, n, r, rho, sigma, seed), self.h)
        self.m, self.n = m, n

    def fetch_matrix(self) -> "MaskedMatrix":
        """The loaded matrix back on the host (values + byte mask unpacked from the device words)."""
        m, n = self.m, self.n
        nwp = C.c_int64(0)
        _check(lib().rsm_ctx_fetch_matrix(self.h, None, None, C.byref(nwp)), self.h)
        values = np.empty((m, n), dtype=np.float64)
        words = np.empty((m, nwp.value), dtype=np.uint32)
        _check(lib().rsm_ctx_fetch_matrix(self.h, _ptr(values), _ptr(words), None), self.h)
        bits = np.unpackbits(words.view(np.uint8).reshape(m, -1), axis=1, bitorder="little")[:, :n]
        return MaskedMatrix.from_arrays(values, bits.astype(np.uint8))

    def decompose(self, cfg: RsmConfig, fetch: bool = True):
        r = cfg.rank
        U = np.empty((self.m, max(r, 1))) if fetch else None
        V = np.empty((self.n, max(r, 1))) if fetch else None
        rep = _Report()
        c = cfg._c()
        _check(lib().rsm_ctx_decompose(self.h, C.byref(c), _ptr(U), _ptr(V), C.byref(rep)), self.h)
        F = Factorization(self.m, self.n, r, U, V) if fetch else None
        return F, _report(rep)

    def als(self, r: int, iterations: int, seed: int, fetch: bool = True):
        """baseline_als on the loaded matrix (als.cpp:11-44) -> (Factorization, DecompositionReport)."""
        U = np.empty((self.m, max(r, 1))) if fetch else None
        V = np.empty((self.n, max(r, 1))) if fetch else None
        rep = _Report()
        _check(lib().rsm_ctx_als(self.h, r, iterations, seed, _ptr(U), _ptr(V), C.byref(rep)), self.h)
        F = Factorization(self.m, self.n, r, U, V) if fetch else None
        return F, _report(rep)

    def fetch_factors(self, r: int):
        U = np.empty((self.m, r))
        V = np.empty((self.n, r))
        _check(lib().rsm_ctx_fetch_factors(self.h, _ptr(U), _ptr(V)), self.h)
        return U, V

    def select(self, p: TrialParams, trials: int):
        acc_ids = np.zeros(trials, np.uint64)
        surv = np.zeros(trials, np.int64)
        att, acc = C.c_uint64(), C.c_uint64()
        c = p._c()
        _check(lib().rsm_ctx_select(self.h, C.byref(c), trials, _ptr(acc_ids), _ptr(surv), C.byref(att),
                                    C.byref(acc)), self.h)
        return acc_ids[:acc.value], surv[:acc.value], att.value, acc.value

    def harvest_gram(self, p: TrialParams, trials: int) -> HarvestResult:
        G = np.empty((self.n, self.n))
        att, acc, z = C.c_uint64(), C.c_uint64(), C.c_uint64()
        c = p._c()
        _check(lib().rsm_ctx_harvest_gram(self.h, C.byref(c), trials, _ptr(G), C.byref(att), C.byref(acc),
                                          C.byref(z)), self.h)
        return HarvestResult(G, att.value, acc.value, z.value)

    def solve_v(self, G: np.ndarray | None, n: int, r: int, tol: float):
        V = np.empty((n, r))
        w = np.empty(r + 1)
        gr, bl = C.c_int64(), C.c_int32()
        Gc = np.ascontiguousarray(G, dtype=np.float64) if G is not None else None
        _check(lib().rsm_ctx_solve_v(self.h, _ptr(Gc), n, r, tol, _ptr(V), C.byref(gr), C.byref(bl), _ptr(w)),
               self.h)
        return SolveVResult(V, gr.value, bool(bl.value)), w

    def solve_u(self, V: np.ndarray | None, r: int):
        U = np.empty((self.m, r))
        fl, ss = C.c_int64(), C.c_double()
        Vc = np.ascontiguousarray(V, dtype=np.float64) if V is not None else None
        _check(lib().rsm_ctx_solve_u(self.h, _ptr(Vc), r, _ptr(U), C.byref(fl), C.byref(ss)), self.h)
        return SolveUResult(U, fl.value), ss.value

    def stage_ms(self):
        buf = (C.c_double * 8)()
        k = lib().rsm_ctx_stage_ms(self.h, C.cast(buf, C.c_void_p), 8)
        return list(buf[:k])

    def launch_count(self) -> int:
        return int(lib().rsm_ctx_launch_count(self.h))

    def rerun_count(self) -> int:
        """decompositions re-run after a failed speculative selection (diagnostic)"""
        return int(lib().rsm_ctx_rerun_count(self.h))

    def last_load_h2d_bytes(self) -> int:
        """Bytes the last host load copied to the device (values + packed mask)."""
        return int(lib().rsm_ctx_last_load_h2d_bytes(self.h))

    def solver_stats(self) -> dict:
        buf = (C.c_double * 32)()
        k = lib().rsm_ctx_solver_stats(self.h, C.cast(buf, C.c_void_p), 32)
        keys = ["outer", "matvecs", "lambda_max", "ub", "max_residual", "block", "grid", "cyc_filter",
                "cyc_cholqr", "cyc_rr", "cyc_eig", "cyc_rotate", "cyc_setup", "jac_sweeps", "cyc_jacobi", "cyc_matvec", "cyc_cq_gram", "cyc_cq_reduce", "cyc_cq_chol",
                "cyc_cq_apply", "cyc_sync", "cyc_setup_all", "cyc_tail", "cyc_kernel", "chol_attempts",
                "cyc_probe", "x26", "x27", "x28", "x29", "x30", "x31"]
        return dict(zip(keys, buf[:k]))


# ------------------------------------------------------- reference-shaped API

def trial_params(cfg: RsmConfig, M: MaskedMatrix) -> TrialParams:
    """rsm::trial_params (harvest.cpp:11-35)."""
    out = _TrialParams()
    c = cfg._c()
    _check(lib().rsm_make_trial_params(C.byref(c), M.m, M.n, C.byref(out)))
    return TrialParams(Mode(out.mode), out.block, out.ell, out.rank, out.min_count, out.seed)


def harvest_gram(M: MaskedMatrix, p: TrialParams, trials: int, workers: int = 0) -> HarvestResult:
    """rsm::harvest_gram (harvest.cpp:79-120): G is n x n."""
    G = np.empty((M.n, M.n))
    att, acc, z = C.c_uint64(), C.c_uint64(), C.c_uint64()
    c = p._c()
    _check(lib().rsm_harvest_gram(_ptr(M.values), _ptr(M.mask), M.m, M.n, C.byref(c), trials, _ptr(G),
                                  C.byref(att), C.byref(acc), C.byref(z)))
    return HarvestResult(G, att.value, acc.value, z.value)


def solve_v(G: np.ndarray, r: int, tol: float) -> SolveVResult:
    """rsm::solve_v (solver.cpp:15-62)."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    n = G.shape[0]
    V = np.empty((n, max(r, 1)))
    gr, bl = C.c_int64(), C.c_int32()
    _check(lib().rsm_solve_v(_ptr(G), n, r, tol, _ptr(V), C.byref(gr), C.byref(bl)))
    return SolveVResult(V, gr.value, bool(bl.value))


def solve_u(M: MaskedMatrix, vhat: np.ndarray, r: int, workers: int = 0) -> SolveUResult:
    """rsm::solve_u (solver.cpp:64-89)."""
    vhat = np.ascontiguousarray(vhat, dtype=np.float64).reshape(-1)
    if r < 1:
        raise Error(errc.invalid_config, "solve_u: rank must be positive")
    if vhat.size != M.n * r:
        raise Error(errc.invalid_config, "solve_u: basis shape does not match matrix")
    U = np.empty((M.m, r))
    fl = C.c_int64()
    _check(lib().rsm_solve_u(_ptr(M.values), _ptr(M.mask), M.m, M.n, _ptr(vhat), r, _ptr(U), C.byref(fl)))
    return SolveUResult(U, fl.value)


def decompose(M: MaskedMatrix, cfg: RsmConfig):
    """rsm::decompose (solver.cpp:119-146) -> (Factorization, DecompositionReport)."""
    r = cfg.rank
    U = np.empty((M.m, max(r, 1)))
    V = np.empty((M.n, max(r, 1)))
    rep = _Report()
    c = cfg._c()
    _check(lib().rsm_decompose(_ptr(M.values), _ptr(M.mask), M.m, M.n, C.byref(c), _ptr(U), _ptr(V),
                               C.byref(rep)))
    return Factorization(M.m, M.n, r, U, V), _report(rep)


def baseline_als(M: MaskedMatrix, r: int, iterations: int, seed: int, workers: int = 0):
    """rsm::baseline_als (solver.hpp:79-81, als.cpp:11-44) -> (Factorization, DecompositionReport).
    `workers` is accepted for signature parity; the device decides its own parallelism."""
    U = np.empty((M.m, max(r, 1)))
    V = np.empty((M.n, max(r, 1)))
    rep = _Report()
    _check(lib().rsm_als(_ptr(M.values), _ptr(M.mask), M.m, M.n, r, iterations, seed, _ptr(U), _ptr(V),
                         C.byref(rep)))
    return Factorization(M.m, M.n, r, U, V), _report(rep)


def masked_residual_norm(M: MaskedMatrix, F: Factorization) -> float:
    """rsm::masked_residual_norm (core.cpp:35-39)."""
    if F.m != M.m or F.n != M.n:
        raise Error(errc.invalid_config, "factorization shape does not match matrix")
    e = C.c_double()
    U = np.ascontiguousarray(F.u, dtype=np.float64)
    V = np.ascontiguousarray(F.v, dtype=np.float64)
    _check(lib().rsm_masked_residual_norm(_ptr(M.values), _ptr(M.mask), M.m, M.n, _ptr(U), _ptr(V), F.r,
                                          C.byref(e)))
    return e.value


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured DFMA throughput (TFLOP/s) of the device."""
    t = C.c_double()
    _check(lib().rsm_fp64_peak_tflops(device, C.byref(t)))
    return t.value


def shard_range(total: int, world: int, rank: int):
    """The library's work split: rank owns [lo, hi) of total units."""
    lo, hi = C.c_int64(), C.c_int64()
    lib().rsm_shard_range(total, world, rank, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def dmma_peak_tflops(device: int = 0) -> float:
    """Measured FP64 tensor-core (DMMA) throughput (TFLOP/s) of the device."""
    t = C.c_double()
    _check(lib().rsm_dmma_peak_tflops(device, C.byref(t)))
    return t.value


def generate(m: int, n: int, r: int, rho: float, sigma: float, seed: int, row0: int = 0,
             rows: int | None = None) -> MaskedMatrix:
    """Observed matrix of rsm::generate (synth.cpp:12-57), rows [row0, row0+rows)."""
    rows = m - row0 if rows is None else rows
    Y = np.empty((rows, n))
    W = np.empty((rows, n), np.uint8)
    st = lib().rsm_generate(m, n, r, rho, sigma, seed, row0, rows, _ptr(Y), _ptr(W))
    if st:
        raise Error(st, "synthetic spec out of range")
    return MaskedMatrix(rows, n, Y, W)


def generate_tracks(points: int, frames: int, wmin: int, wmax: int, sigma: float, seed: int, row0: int = 0,
                    rows: int | None = None) -> MaskedMatrix:
    """Structured-missingness instance of BASELINE config 5 (affine-camera
    tracks, rank 4, one contiguous visibility window per point; the streams
    are documented at rsm_generate_tracks in synth.cpp), rows [row0, row0+rows)."""
    rows = points - row0 if rows is None else rows
    Y = np.empty((rows, 2 * frames))
    W = np.empty((rows, 2 * frames), np.uint8)
    st = lib().rsm_generate_tracks(points, frames, wmin, wmax, sigma, seed, row0, rows, _ptr(Y), _ptr(W))
    if st:
        raise Error(st, "track spec out of range")
    return MaskedMatrix(rows, 2 * frames, Y, W)


def load_matrix(path: str) -> MaskedMatrix:
    """rsm::load_matrix (io.cpp:56-99): NaN-CSV -> MaskedMatrix."""
    pv, pm = C.c_void_p(), C.c_void_p()
    m, n = C.c_int64(), C.c_int64()
    st = lib().rsm_load_matrix_csv(os.fsencode(path), C.byref(pv), C.byref(pm), C.byref(m), C.byref(n))
    if st:
        raise Error(st, lib().rsm_last_error(None).decode())
    try:
        cnt = m.value * n.value
        Y = np.ctypeslib.as_array(C.cast(pv, C.POINTER(C.c_double)), (cnt,)).copy().reshape(m.value, n.value)
        W = np.ctypeslib.as_array(C.cast(pm, C.POINTER(C.c_uint8)), (cnt,)).copy().reshape(m.value, n.value)
    finally:
        lib().rsm_free(pv)
        lib().rsm_free(pm)
    return MaskedMatrix(m.value, n.value, Y, W)


def save_matrix(M: MaskedMatrix, path: str) -> None:
    """rsm::save_matrix (io.cpp:101-116): hidden cells as NaN, %.17g values."""
    st = lib().rsm_save_matrix_csv(os.fsencode(path), _ptr(M.values), _ptr(M.mask), M.m, M.n)
    if st:
        raise Error(st, lib().rsm_last_error(None).decode())


def dataset_checksum(M: MaskedMatrix) -> int:
    """rsm::dataset_checksum (io.cpp:140-154)."""
    out = C.c_uint64()
    st = lib().rsm_dataset_checksum(_ptr(M.values), _ptr(M.mask), M.m, M.n, C.byref(out))
    if st:
        raise Error(st, lib().rsm_last_error(None).decode())
    return int(out.value)


# ------------------------------------------------ per-call building blocks
# The reference's single-trial and accumulator functions (sampler.hpp,
# spectra.hpp, solver.hpp:40-42, core.hpp:95), one device call each.

@dataclass
class Submatrix:
    """rsm::Submatrix (include/rsm/sampler.hpp:13-28)."""
    row_indices: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray  # |rows| x |cols|

    def rows(self) -> int:
        return len(self.row_indices)

    def cols(self) -> int:
        return len(self.col_indices)


@dataclass
class ConstraintVector:
    """rsm::ConstraintVector (include/rsm/spectra.hpp:12-19)."""
    col_indices: np.ndarray
    zeta: np.ndarray
    singular_value: float = 0.0


def _sample(M: MaskedMatrix, mode: int, count: int, seed: int, index: int, min_keep: int):
    other = M.n if mode == Mode.M2 else M.m
    drawn = np.zeros(max(count, 1), np.int64)
    kept = np.zeros(max(other, 1), np.int64)
    nk = C.c_int64()
    _check(lib().rsm_sample(_ptr(M.values), _ptr(M.mask), M.m, M.n, int(mode), count, seed, index, _ptr(drawn),
                            _ptr(kept), C.byref(nk)))
    drawn, kept = drawn[:count], kept[:nk.value]
    if nk.value < min_keep:
        return None
    rows, cols = (drawn, kept) if mode == Mode.M2 else (kept, drawn)
    return Submatrix(rows, cols, np.ascontiguousarray(M.values[np.ix_(rows, cols)]))


def sample_m1(M: MaskedMatrix, l: int, seed: int, trial_index: int, min_rows: int = 1):
    """rsm::sample_m1 (sampler.cpp:27-56): None when fewer than min_rows rows survive."""
    return _sample(M, Mode.M1, l, seed, trial_index, min_rows)


def sample_m2(M: MaskedMatrix, k: int, seed: int, trial_index: int, min_cols: int = 1):
    """rsm::sample_m2 (sampler.cpp:58-87): None when fewer than min_cols columns survive."""
    return _sample(M, Mode.M2, k, seed, trial_index, min_cols)


def small_singular_vectors(S: Submatrix, r: int, ell: int):
    """rsm::small_singular_vectors (spectra.cpp:48-86) -> [ConstraintVector]."""
    V = np.ascontiguousarray(S.values, dtype=np.float64)
    p, q = V.shape
    zeta = np.zeros((max(ell, 1), q))
    sv = np.zeros(max(ell, 1))
    _check(lib().rsm_small_singular_vectors(_ptr(V), p, q, r, ell, _ptr(zeta), _ptr(sv)))
    return [ConstraintVector(np.asarray(S.col_indices), zeta[t].copy(), float(sv[t])) for t in range(ell)]


def attempt_trial(M: MaskedMatrix, p: TrialParams, index: int):
    """rsm::attempt_trial (harvest.cpp:37-51): None when rejected."""
    if p.mode == Mode.M1:
        S = sample_m1(M, p.block, p.seed, index, p.min_count)
        return None if S is None else small_singular_vectors(S, p.rank, p.ell)
    S = sample_m2(M, p.block, p.seed, index, p.min_count)
    if S is None:
        return None
    avail = S.cols() - p.rank
    ell = min(p.ell, avail) if p.ell > 0 else avail
    return small_singular_vectors(S, p.rank, ell)


def embed(cv: ConstraintVector, n: int) -> np.ndarray:
    """rsm::embed (spectra.cpp:88-96)."""
    if np.any((cv.col_indices < 0) | (cv.col_indices >= n)):
        raise Error(errc.invalid_config, "embed: column index out of range")
    x = np.zeros(n)
    x[cv.col_indices] = cv.zeta
    return x


def gram_update(G: np.ndarray, X: np.ndarray | None = None, G2: np.ndarray | None = None) -> np.ndarray:
    """G += sum_v x_v x_v^T (+ G2) on the device, bit-identical to the
    reference's GramAccumulator::accumulate / merge loops (spectra.cpp:7-46)."""
    G = np.ascontiguousarray(G, dtype=np.float64).copy()
    n = G.shape[0]
    Xc = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, n) if X is not None else None
    G2c = np.ascontiguousarray(G2, dtype=np.float64) if G2 is not None else None
    _check(lib().rsm_gram_update(_ptr(G), n, _ptr(Xc), 0 if Xc is None else Xc.shape[0], _ptr(G2c)))
    return G


def masked_objective(M: MaskedMatrix, F: Factorization, norm: int = 0) -> float:
    """rsm::masked_objective (core.cpp:41-44): norm 0 = Frobenius."""
    out = C.c_double()
    _check(lib().rsm_masked_objective(_ptr(M.values), _ptr(M.mask), M.m, M.n,
                                      _ptr(np.ascontiguousarray(F.u)), _ptr(np.ascontiguousarray(F.v)),
                                      F.u.shape[1], norm, C.byref(out)))
    return out.value
