// rsm_dev.cuh -- device-side helpers shared by the RSM stage kernels.
//
// Counter-based splitmix64 streams restated bit-exactly from the reference
// (include/rsm/rng.hpp:12-57, paths relative to /root/reference/proj), warp
// reductions, and a warp-parallel cyclic Jacobi eigensolver for the small
// symmetric matrices of stages 2 and 4.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rsmd {

constexpr int KMAX = 16;  // max vectors per trial (block k or l) on device
constexpr int RMAX = 16;  // max excluded top vectors r_ex on device

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

// Rng(seed, tag, index) constructor state (rng.hpp:14-17)
__device__ __forceinline__ uint64_t rng_state(uint64_t seed, uint64_t tag, uint64_t index) {
  uint64_t s = mix(seed + 0x9e3779b97f4a7c15ull * tag);
  return mix(s + 0xbf58476d1ce4e5b9ull * index);
}

__device__ __forceinline__ uint64_t next_u64(uint64_t& s) {  // rng.hpp:19-22
  s += 0x9e3779b97f4a7c15ull;
  return mix(s);
}

// rejection sampling in [0, bound) (rng.hpp:30-36)
__device__ __forceinline__ uint64_t next_below(uint64_t& s, uint64_t bound) {
  const uint64_t limit = bound * (UINT64_MAX / bound);
  for (;;) {
    const uint64_t v = next_u64(s);
    if (v < limit) return v % bound;
  }
}

// draw_without_replacement (sampler.cpp:12-23) for attempt `a` of the TRIAL
// stream: the partial Fisher-Yates on a virtual identity permutation (a
// position -> value map of the <= 2 block touched slots), then the drawn
// values sorted ascending into out[0..block). block <= KMAX.
__device__ inline void draw_sorted(uint64_t seed, uint64_t a, int64_t pool, int block, int32_t* out) {
  uint64_t st = rng_state(seed, 5 /* stream::TRIAL */, a);
  int32_t key[2 * KMAX], val[2 * KMAX];
  int nmap = 0;
  for (int t = 0; t < block; ++t) {
    const int32_t j = t + (int32_t)next_below(st, (uint64_t)(pool - t));
    int32_t vt = t, vj = j;
    int ft = -1, fj = -1;
    for (int e = 0; e < nmap; ++e) {
      if (key[e] == t) { vt = val[e]; ft = e; }
      if (key[e] == j) { vj = val[e]; fj = e; }
    }
    // swap(idx[t], idx[j])
    if (ft < 0) { key[nmap] = t; ft = nmap++; }
    val[ft] = vj;
    if (fj < 0) {
      if (j != t) { key[nmap] = j; fj = nmap++; val[fj] = vt; }
    } else {
      val[fj] = vt;
    }
  }
  for (int t = 0; t < block; ++t) {
    int32_t v = t;
    for (int e = 0; e < nmap; ++e)
      if (key[e] == t) { v = val[e]; break; }
    // insertion into the sorted prefix
    int p = t - 1;
    while (p >= 0 && out[p] > v) { out[p + 1] = out[p]; --p; }
    out[p + 1] = v;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 1/sqrt(v) to ~1 ulp: the hardware's double-precision seed (rsqrt.approx.f64 =
// MUFU.RSQ64H on the high word, relative error ~2^-22) and two Newton steps
// (2^-43 -> rounding) for normal v; else the library rsqrt (a long software
// sequence). The float-seeded form (two F64<->F32 conversions around
// MUFU.RSQ) measured 131 cycles per dependent call (scripts/micro/dp_latency.cu).
__device__ __forceinline__ double rsqrt_fast(double v) {
  if (v > 1e-300 && v < 1e300) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;\n" : "=d"(r) : "d"(v));
    const double hv = 0.5 * v;
    r = r * fma(-hv * r, r, 1.5);
    r = r * fma(-hv * r, r, 1.5);
    return r;
  }
  return rsqrt(v);
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum N (power of two) per-lane values over the warp by recursive halving:
// at each of the first log2(min(N,32)) exchanges a lane keeps one half of its
// values and receives its partner's copy of that half, so the shuffle count
// is ~N instead of 5N. On return lane l holds max(1, N/32) totals in v[0..]:
// value j sits in lane (j / PL) * max(1, 32/N), slot j % PL.
template <int N>
__device__ __forceinline__ void warp_reduce_halving(double (&v)[N], int lane) {
  constexpr int STEPS = N >= 32 ? 5 : (N >= 16 ? 4 : (N >= 8 ? 3 : (N >= 4 ? 2 : (N >= 2 ? 1 : 0))));
#pragma unroll
  for (int st = 0; st < STEPS; ++st) {
    const int o = 16 >> st;
    const int K = N >> st;  // values still held
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      if (i < K / 2) {
        const double mine = up ? v[i + K / 2] : v[i];
        const double other = up ? v[i] : v[i + K / 2];
        v[i] = mine + __shfl_xor_sync(0xffffffffu, other, o);
      }
    }
  }
  // remaining lane bits: plain butterfly on the single held value
  if (N < 32) {
#pragma unroll
    for (int o = 16 >> STEPS; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  }
}

template <int N>
__device__ __forceinline__ double warp_total(const double (&v)[N], int j) {
  constexpr int PL = N > 32 ? N / 32 : 1;
  constexpr int LPV = N < 32 ? 32 / N : 1;
  double x = v[0];
#pragma unroll
  for (int s = 1; s < PL; ++s)
    if (j % PL == s) x = v[s];
  return __shfl_sync(0xffffffffu, x, (j / PL) * LPV);
}

// Warp-parallel cyclic Jacobi on a symmetric K x K matrix A (smem,
// row-major, leading dim lda), K <= 32. Uses the round-robin (tournament)
// ordering: each step rotates floor(Kp/2) disjoint pairs at once, one lane
// per pair, then all lanes apply the column and row rotations. On return the
// diagonal of A holds the eigenvalues and V (K x K, ldv, row-major; column j
// = eigenvector j) the eigenvectors. Must be called by one full warp.
// Stops when every off-diagonal |a_pq| <= tol * sqrt(|a_pp a_qq|) or when
// it is exactly zero; returns the sweep count.
__device__ inline int warp_jacobi_eig(double* A, int lda, double* V, int ldv, int K,
                                      double* cs /* smem scratch >= 2*32 doubles */,
                                      int* pairs /* smem scratch >= 2*32 ints */, double tol,
                                      int max_sweeps, bool init_v, double abs_thr = 0.0) {
  const int lane = threadIdx.x & 31;
  // abs_thr > 0: absolute test |a_pq| <= abs_thr (eigenvalues to abs_thr, as
  // dsyev delivers them); otherwise the relative test against sqrt(|a_pp a_qq|)
  auto big_off = [&](double apq, double app, double aqq) {
    return abs_thr > 0.0 ? fabs(apq) > abs_thr : (apq != 0.0 && fabs(apq) > tol * sqrt(fabs(app * aqq)));
  };
  if (init_v)
    for (int e = lane; e < K * K; e += 32) V[(e / K) * ldv + (e % K)] = (e / K == e % K) ? 1.0 : 0.0;
  __syncwarp();
  if (K < 2) return 0;
  const int Kp = (K + 1) & ~1;  // even count, index K-1+1 is a dummy when K odd
  const int npair = Kp / 2;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    // convergence test on the current matrix
    int big = 0;
    for (int e = lane; e < K * K; e += 32) {
      const int p = e / K, q = e % K;
      if (p < q) {
        const double apq = A[p * lda + q];
        if (big_off(apq, A[p * lda + p], A[q * lda + q])) big = 1;
      }
    }
    if (!__any_sync(0xffffffffu, big)) break;
    for (int step = 0; step < Kp - 1; ++step) {
      // round-robin pairing: position 0 fixed, others rotate
      if (lane < npair) {
        int a = (lane == 0) ? 0 : ((lane - 1 + step) % (Kp - 1)) + 1;
        int b = ((Kp - 2 - lane + step) % (Kp - 1)) + 1;
        int p = a < b ? a : b, q = a < b ? b : a;
        double c = 1.0, s = 0.0;
        if (q < K) {
          const double apq = A[p * lda + q];
          const double app = A[p * lda + p], aqq = A[q * lda + q];
          if (big_off(apq, app, aqq)) {
            const double zeta = (aqq - app) / (2.0 * apq);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = 1.0 / sqrt(1.0 + t * t);
            s = c * t;
          }
        }
        pairs[2 * lane] = p;
        pairs[2 * lane + 1] = q;
        cs[2 * lane] = c;
        cs[2 * lane + 1] = s;
      }
      __syncwarp();
      // column rotation: A <- A J, V <- V J  (J = product of disjoint rotations)
      for (int e = lane; e < npair * K; e += 32) {
        const int pr = e / K, row = e % K;
        const int p = pairs[2 * pr], q = pairs[2 * pr + 1];
        const double c = cs[2 * pr], s = cs[2 * pr + 1];
        if (q < K && s != 0.0) {
          const double x = A[row * lda + p], y = A[row * lda + q];
          A[row * lda + p] = c * x - s * y;
          A[row * lda + q] = s * x + c * y;
          const double vx = V[row * ldv + p], vy = V[row * ldv + q];
          V[row * ldv + p] = c * vx - s * vy;
          V[row * ldv + q] = s * vx + c * vy;
        }
      }
      __syncwarp();
      // row rotation: A <- J^T A
      for (int e = lane; e < npair * K; e += 32) {
        const int pr = e / K, col = e % K;
        const int p = pairs[2 * pr], q = pairs[2 * pr + 1];
        const double c = cs[2 * pr], s = cs[2 * pr + 1];
        if (q < K && s != 0.0) {
          const double x = A[p * lda + col], y = A[q * lda + col];
          A[p * lda + col] = c * x - s * y;
          A[q * lda + col] = s * x + c * y;
        }
      }
      __syncwarp();
      // the rotated pair entries are zero by construction
      if (lane < npair) {
        const int p = pairs[2 * lane], q = pairs[2 * lane + 1];
        if (q < K && cs[2 * lane + 1] != 0.0) {
          A[p * lda + q] = 0.0;
          A[q * lda + p] = 0.0;
        }
      }
      __syncwarp();
    }
  }
  return sweep;
}

// Jacobi with the absolute off-diagonal threshold 16 eps * ||A||_F (LAPACK-level
// eigenvalue accuracy); used where small eigenvalues only need absolute
// accuracy (the stage-4 Rayleigh-Ritz problem). V is initialised to I.
__device__ inline int warp_jacobi_eig_abs(double* A, int lda, double* V, int ldv, int K, double* cs,
                                          int* pairs, int max_sweeps) {
  const int lane = threadIdx.x & 31;
  double f = 0.0;
  for (int e = lane; e < K * K; e += 32) {
    const double v = A[(e / K) * lda + (e % K)];
    f += v * v;
  }
  f = warp_sum(f);
  // 16 eps: rounding keeps re-creating off-diagonals of ~eps ||A||, so a
  // threshold at exactly eps ||A|| can rotate until max_sweeps
  const double thr = 16.0 * 2.220446049250313e-16 * sqrt(f);
  return warp_jacobi_eig(A, lda, V, ldv, K, cs, pairs, 0.0, max_sweeps, true, thr > 0.0 ? thr : 1e-300);
}

// Compile-time-K variant of the round-robin warp Jacobi with the absolute
// threshold 16 eps ||A||_F (see warp_jacobi_eig_abs); V is set to I. Kept out
// of line so a large caller's register pressure cannot spill its loop state.
template <int K>
__device__ __noinline__ int warp_jacobi_abs_k(double* A, int lda, double* V, int ldv, double* cs, int* pairs,
                                              int max_sweeps) {
  constexpr int Kp = (K + 1) & ~1;
  constexpr int NPAIR = Kp / 2;
  const int lane = threadIdx.x & 31;
  double f = 0.0;
#pragma unroll
  for (int e = lane; e < K * K; e += 32) {
    const double v = A[(e / K) * lda + (e % K)];
    f += v * v;
  }
  f = warp_sum(f);
  const double thr = fmax(16.0 * 2.220446049250313e-16 * sqrt(f), 1e-300);
#pragma unroll
  for (int e = lane; e < K * K; e += 32) V[(e / K) * ldv + (e % K)] = (e / K == e % K) ? 1.0 : 0.0;
  __syncwarp();
  if (K < 2) return 0;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int big = 0;
#pragma unroll
    for (int e = lane; e < K * K; e += 32) {
      const int p = e / K, q = e % K;
      if (p < q && fabs(A[p * lda + q]) > thr) big = 1;
    }
    if (!__any_sync(0xffffffffu, big)) break;
#pragma unroll 1
    for (int step = 0; step < Kp - 1; ++step) {
      if (lane < NPAIR) {
        const int a = (lane == 0) ? 0 : ((lane - 1 + step) % (Kp - 1)) + 1;
        const int b = ((Kp - 2 - lane + step) % (Kp - 1)) + 1;
        const int p = a < b ? a : b, q = a < b ? b : a;
        double c = 1.0, sn = 0.0;
        if (q < K) {
          const double apq = A[p * lda + q];
          if (fabs(apq) > thr) {
            const double zeta = (A[q * lda + q] - A[p * lda + p]) / (2.0 * apq);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = rsqrt(1.0 + t * t);
            sn = c * t;
          }
        }
        pairs[2 * lane] = p;
        pairs[2 * lane + 1] = q;
        cs[2 * lane] = c;
        cs[2 * lane + 1] = sn;
      }
      __syncwarp();
#pragma unroll
      for (int e = lane; e < NPAIR * K; e += 32) {
        const int pr = e / K, row = e % K;
        const int p = pairs[2 * pr], q = pairs[2 * pr + 1];
        const double c = cs[2 * pr], sn = cs[2 * pr + 1];
        if (q < K && sn != 0.0) {
          const double x = A[row * lda + p], y = A[row * lda + q];
          A[row * lda + p] = c * x - sn * y;
          A[row * lda + q] = sn * x + c * y;
          const double vx = V[row * ldv + p], vy = V[row * ldv + q];
          V[row * ldv + p] = c * vx - sn * vy;
          V[row * ldv + q] = sn * vx + c * vy;
        }
      }
      __syncwarp();
#pragma unroll
      for (int e = lane; e < NPAIR * K; e += 32) {
        const int pr = e / K, col = e % K;
        const int p = pairs[2 * pr], q = pairs[2 * pr + 1];
        const double c = cs[2 * pr], sn = cs[2 * pr + 1];
        if (q < K && sn != 0.0) {
          const double x = A[p * lda + col], y = A[q * lda + col];
          A[p * lda + col] = c * x - sn * y;
          A[q * lda + col] = sn * x + c * y;
        }
      }
      __syncwarp();
      if (lane < NPAIR) {
        const int p = pairs[2 * lane], q = pairs[2 * lane + 1];
        if (q < K && cs[2 * lane + 1] != 0.0) {
          A[p * lda + q] = 0.0;
          A[q * lda + p] = 0.0;
        }
      }
      __syncwarp();
    }
  }
  return sweep;
}

// circle method on Kp (even) slots: slot l holds round-robin position
// pos(l) (pairs are positions (i, Kp-1-i) = slots (2i, 2i+1)); position 0
// stays and the others advance by one per step. circle_src(l) is the slot
// whose content moves into slot l.
__host__ __device__ constexpr int circle_pos(int l, int Kp) { return (l & 1) ? (Kp - 1 - (l >> 1)) : (l >> 1); }
__host__ __device__ constexpr int circle_slot(int p, int Kp) {
  return (p <= (Kp - 1) / 2) ? 2 * p : 2 * (Kp - 1 - p) + 1;
}
__host__ __device__ constexpr int circle_src(int l, int Kp) {
  return circle_slot(circle_pos(l, Kp) == 0 ? 0 : (circle_pos(l, Kp) == 1 ? Kp - 1 : circle_pos(l, Kp) - 1), Kp);
}

// Register-resident parallel Jacobi (circle-method ordering, Brent-Luk
// style) for the symmetric K x K matrix A (smem, lda), K <= 16, one warp.
// Lane l holds slot l's column of A (rows in slot order) and of V (rows in
// the original order). Each step rotates the slot pairs (2i, 2i+1) at once:
// partners exchange columns by shuffles, every lane applies all pairs' row
// rotations to its column, and a fixed permutation then moves indices between
// slots (columns by shuffle, rows by a compile-time register renaming) so
// every index pair meets once per sweep. Threshold as warp_jacobi_eig_abs.
// On return A's diagonal holds the eigenvalues and V's columns the matching
// eigenvectors (in some order). Returns the sweep count.
template <int K, bool REL = false>
__device__ __noinline__ int warp_jacobi_reg(double* A, int lda, double* V, int ldv, int max_sweeps,
                                            double rtol = 2.220446049250313e-16) {
  constexpr int Kp = (K + 1) & ~1;
  const int lane = threadIdx.x & 31;
  const bool live = lane < Kp;
  double a[Kp], v[Kp];
#pragma unroll
  for (int r = 0; r < Kp; ++r) {
    a[r] = (live && lane < K && r < K) ? A[r * lda + lane] : 0.0;
    v[r] = (r == lane) ? 1.0 : 0.0;
  }
  int idx = lane;  // original index held by this slot
  // circle method: slot l holds round-robin position pos(l); pairs are the
  // positions (i, Kp-1-i) = slots (2i, 2i+1); position 0 stays, the others
  // advance by one each step. src(l) = slot whose content moves into slot l.
  const int src = live ? circle_src(lane, Kp) : lane;
  double f = 0.0;
#pragma unroll
  for (int r = 0; r < Kp; ++r) f += a[r] * a[r];
  f = warp_sum(f);
  const double thr = fmax(16.0 * 2.220446049250313e-16 * sqrt(f), 1e-300);
  // REL: |a_pq| <= rtol sqrt(|a_pp a_qq|) (or exactly 0) for every pair, as
  // warp_jacobi_eig's relative test; else the absolute threshold above
  auto big = [&](double apq, double app, double aqq) {
    return REL ? (apq != 0.0 && fabs(apq) > rtol * sqrt(fabs(app * aqq))) : fabs(apq) > thr;
  };
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    double dme = 0.0;
#pragma unroll
    for (int r = 0; r < Kp; ++r) dme = (r == lane) ? a[r] : dme;
    bool any = false;
#pragma unroll
    for (int r = 0; r < Kp; ++r) {
      const double drr = __shfl_sync(0xffffffffu, dme, r);
      if (r != lane && big(a[r], drr, dme)) any = true;
    }
    if (!__any_sync(0xffffffffu, live && any)) break;
#pragma unroll 1
    for (int step = 0; step < Kp - 1; ++step) {
      // this slot's diagonal and its pair's off-diagonal entry
      double d = 0.0, off = 0.0;
#pragma unroll
      for (int r = 0; r < Kp; ++r) {
        d = (r == lane) ? a[r] : d;
        off = (r == (lane ^ 1)) ? a[r] : off;
      }
      const double dp = __shfl_xor_sync(0xffffffffu, d, 1);
      const bool isp = (lane & 1) == 0;
      const double app = isp ? d : dp, aqq = isp ? dp : d;
      double c = 1.0, sn = 0.0;
      if (live && big(off, app, aqq)) {
        // t = sign(d) e / (|d| + r) with d = a_qq - a_pp, e = 2 a_pq,
        // r = hypot(d, e) (Rutishauser's root); with w = r + |d|,
        // c = w / sqrt(2 r w) and s = sign(d) e / sqrt(2 r w): two rsqrt and
        // no division on the step's critical path
        const double dd = aqq - app, ee = 2.0 * off;
        const double r2 = fma(dd, dd, ee * ee);
        const double rr = r2 * rsqrt_fast(r2);
        const double w = rr + fabs(dd);
        const double g = rsqrt_fast(2.0 * rr * w);
        c = w * g;
        sn = (dd >= 0.0 ? ee : -ee) * g;
      }
      // columns: A <- A J, V <- V J
#pragma unroll
      for (int r = 0; r < Kp; ++r) {
        const double oa = __shfl_xor_sync(0xffffffffu, a[r], 1);
        const double ov = __shfl_xor_sync(0xffffffffu, v[r], 1);
        a[r] = isp ? fma(c, a[r], -sn * oa) : fma(sn, oa, c * a[r]);
        v[r] = isp ? fma(c, v[r], -sn * ov) : fma(sn, ov, c * v[r]);
      }
      // rows: A <- J^T A with every pair's rotation
#pragma unroll
      for (int i = 0; i < Kp / 2; ++i) {
        const double ci = __shfl_sync(0xffffffffu, c, 2 * i);
        const double si = __shfl_sync(0xffffffffu, sn, 2 * i);
        const double x = a[2 * i], y = a[2 * i + 1];
        a[2 * i] = fma(ci, x, -si * y);
        a[2 * i + 1] = fma(si, x, ci * y);
      }
      // the rotated pair's off-diagonal is zero by construction
#pragma unroll
      for (int r = 0; r < Kp; ++r) a[r] = (r == (lane ^ 1) && sn != 0.0) ? 0.0 : a[r];
      // advance the circle: columns move between slots, rows are renamed
      double t2[Kp];
#pragma unroll
      for (int r = 0; r < Kp; ++r) {
        t2[r] = __shfl_sync(0xffffffffu, a[r], src);
        v[r] = __shfl_sync(0xffffffffu, v[r], src);
      }
#pragma unroll
      for (int r = 0; r < Kp; ++r) a[r] = t2[circle_src(r, Kp)];
      idx = __shfl_sync(0xffffffffu, idx, src);
    }
  }
  __syncwarp();
  // write back: eigenvalue of slot l on A's diagonal, its vector as V's column
  // (slots holding the padding index are skipped)
  const unsigned dmask = __ballot_sync(0xffffffffu, live && idx >= K);
  if (live && idx < K) {
    const int col = lane - __popc(dmask & ((1u << lane) - 1u));
    double d = 0.0;
#pragma unroll
    for (int r = 0; r < Kp; ++r) d = (r == lane) ? a[r] : d;
    A[col * lda + col] = d;
#pragma unroll
    for (int r = 0; r < K; ++r) V[r * ldv + col] = v[r];
  }
  __syncwarp();
  return sweep;
}

// relative-threshold register Jacobi dispatched on the runtime size (K <= 16)
__device__ __forceinline__ int warp_jacobi_rel(double* A, int lda, double* V, int ldv, int K, double* cs,
                                               int* pairs, double tol, int max_sweeps) {
  switch (K) {
#define RSM_JR(k) \
  case k: return warp_jacobi_reg<k, true>(A, lda, V, ldv, max_sweeps, tol);
    RSM_JR(1) RSM_JR(2) RSM_JR(3) RSM_JR(4) RSM_JR(5) RSM_JR(6) RSM_JR(7) RSM_JR(8)
    RSM_JR(9) RSM_JR(10) RSM_JR(11) RSM_JR(12) RSM_JR(13) RSM_JR(14) RSM_JR(15) RSM_JR(16)
#undef RSM_JR
    default: return warp_jacobi_eig(A, lda, V, ldv, K, cs, pairs, tol, max_sweeps, true);
  }
}

// dispatch on the runtime size (K <= KMAX)
__device__ __forceinline__ int warp_jacobi_abs(double* A, int lda, double* V, int ldv, int K, double* cs,
                                               int* pairs, int max_sweeps) {
  switch (K) {
#define RSM_JK(k) \
  case k: return warp_jacobi_reg<k>(A, lda, V, ldv, max_sweeps);
    RSM_JK(1) RSM_JK(2) RSM_JK(3) RSM_JK(4) RSM_JK(5) RSM_JK(6) RSM_JK(7) RSM_JK(8)
    RSM_JK(9) RSM_JK(10) RSM_JK(11) RSM_JK(12) RSM_JK(13) RSM_JK(14) RSM_JK(15) RSM_JK(16)
#undef RSM_JK
    default: return warp_jacobi_eig_abs(A, lda, V, ldv, K, cs, pairs, max_sweeps);
  }
}

// ---- stage 2 -> stage 3 hand-off: int8 digit slices (k_gram_i8.cu) ----
// digits per value of the exact integer split of the harvested vectors:
// kGramSlices by default, 5..7 selectable (gram_i8_slices, k_gram_i8.cu)
constexpr int kGramSlices = 6;

// Balanced signed digits: w = a[0] 2^-6 + sum_{1<=s<S} a[s] 2^(-6-8s) + e.
// X = rint(w 2^(6+8(S-1))) is an exact integer (|X| <= 2^54 for |w| <= 1,
// S <= 7; |e| <= 2^(-7-8(S-1))). Its balanced base-256 digits (every digit
// but the leading one in [-128, 127]) come from one addition: with
// Y = X + sum_{s<S-1} 128 * 256^s, byte s of Y minus 128 is digit s (LSB
// first) and Y >> 8(S-1) is the leading digit a[0] (in [-64, 64]); "minus 128"
// of a byte is its int8 reinterpretation after XOR 0x80. Returned packed: byte
// s (from the least significant) holds a[S-1-s] as int8.
template <int S>
__device__ __forceinline__ unsigned long long digits_i8(double x) {
  static_assert(S >= 2 && S <= 7, "digit count");
  constexpr int LB = 8 * (S - 1);  // bits of the lower digits
  constexpr unsigned long long C = 0x8080808080808080ull & ((1ull << LB) - 1ull);
  const long long X = __double2ll_rn(x * (double)(1ll << (6 + LB)));
  const long long Y = X + (long long)C;
  return (((unsigned long long)Y ^ C) & ((1ull << LB) - 1ull)) | (((unsigned long long)(Y >> LB) & 0xFFull) << LB);
}

// Four consecutive columns j0..j0+3 of trial-vector row `krow`: one 32-bit
// store per digit slice into W[s][krow][j0..j0+3] (S x Kpad x npad int8,
// MN-major; a warp's lanes cover 128 consecutive bytes per store). The 4 x S
// byte transpose is three byte permutes per slice.
template <int S>
__device__ __forceinline__ void emit_slices4_t(int8_t* W, int64_t Kpad, int64_t npad, int64_t krow, int64_t j0,
                                               double v0, double v1, double v2, double v3) {
  const unsigned long long z0 = digits_i8<S>(v0), z1 = digits_i8<S>(v1), z2 = digits_i8<S>(v2),
                           z3 = digits_i8<S>(v3);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int b = S - 1 - s;  // byte of digit a[s]
    const int sh = b < 4 ? 0 : 32;
    const unsigned p = (unsigned)(b & 3);
    const unsigned t01 = __byte_perm((unsigned)(z0 >> sh), (unsigned)(z1 >> sh), p | ((4u + p) << 4));
    const unsigned t23 = __byte_perm((unsigned)(z2 >> sh), (unsigned)(z3 >> sh), p | ((4u + p) << 4));
    *reinterpret_cast<uint32_t*>(W + ((int64_t)s * Kpad + krow) * npad + j0) = __byte_perm(t01, t23, 0x5410);
  }
}

// The same with the address arithmetic hoisted: p = W + krow * npad + j0 (slice
// 0), sstride = Kpad * npad bytes between slices (one 64-bit add per store).
template <int S>
__device__ __forceinline__ void emit_slices4_at_t(int8_t* p, int64_t sstride, double v0, double v1, double v2,
                                                  double v3) {
  const unsigned long long z0 = digits_i8<S>(v0), z1 = digits_i8<S>(v1), z2 = digits_i8<S>(v2),
                           z3 = digits_i8<S>(v3);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int b = S - 1 - s;  // byte of digit a[s]
    const int sh = b < 4 ? 0 : 32;
    const unsigned q = (unsigned)(b & 3);
    const unsigned t01 = __byte_perm((unsigned)(z0 >> sh), (unsigned)(z1 >> sh), q | ((4u + q) << 4));
    const unsigned t23 = __byte_perm((unsigned)(z2 >> sh), (unsigned)(z3 >> sh), q | ((4u + q) << 4));
    *reinterpret_cast<uint32_t*>(p) = __byte_perm(t01, t23, 0x5410);
    p += sstride;
  }
}

// digit counts other than the default (RSM_I8_SLICES experiments): out of line,
// so the callers' loops hold one copy of the emission code, not three
static __device__ __noinline__ void emit_slices4_at_other(int S, int8_t* p, int64_t sstride, double v0, double v1,
                                                   double v2, double v3) {
  if (S == 5) emit_slices4_at_t<5>(p, sstride, v0, v1, v2, v3);
  else emit_slices4_at_t<7>(p, sstride, v0, v1, v2, v3);
}

__device__ __forceinline__ void emit_slices4_at(int S, int8_t* p, int64_t sstride, double v0, double v1, double v2,
                                                double v3) {
  if (S == kGramSlices) emit_slices4_at_t<kGramSlices>(p, sstride, v0, v1, v2, v3);
  else emit_slices4_at_other(S, p, sstride, v0, v1, v2, v3);
}

__device__ __forceinline__ void emit_slices4(int S, int8_t* W, int64_t Kpad, int64_t npad, int64_t krow,
                                             int64_t j0, double v0, double v1, double v2, double v3) {
  emit_slices4_at(S, W + krow * npad + j0, Kpad * npad, v0, v1, v2, v3);
}

}  // namespace rsmd
