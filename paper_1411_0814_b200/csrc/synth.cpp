// synth.cpp -- host input generator (not timed, not a GPU stage): the
// reference's Eq. 31 instance (src/synth.cpp:12-57 of /root/reference/proj)
// restricted to the observed matrix, generated in independent row blocks
// from the per-row counter streams (rng.hpp stream tags FACTOR_A=1,
// FACTOR_B=2, NOISE=3, MASK=4), so a 1M x 2048 instance never holds the
// ground-truth and noise arrays the reference keeps. Ybar = A*B is summed in
// k order.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/rsm_b200.h"
#include "host_rng.h"

namespace {
using rsmh::Rng;
}  // namespace

extern "C" rsm_status rsm_generate(int64_t m, int64_t n, int64_t r, double rho, double sigma,
                                   uint64_t seed, int64_t row0, int64_t rows, double* values,
                                   uint8_t* mask) {
  if (m < 1 || n < 1 || r < 1 || row0 < 0 || rows < 0 || row0 + rows > m) return RSM_ERR_INVALID_CONFIG;
  if (!(rho > 0.0 && rho <= 1.0) || sigma < 0.0) return RSM_ERR_INVALID_CONFIG;
  std::vector<double> B(static_cast<size_t>(r * n));
  for (int64_t k = 0; k < r; ++k) {
    Rng rng(seed, 2, static_cast<uint64_t>(k));
    for (int64_t j = 0; j < n; ++j) B[k * n + j] = rng.next_normal();
  }
  unsigned nt = std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  auto work = [&](int64_t lo, int64_t hi) {
    std::vector<double> a(static_cast<size_t>(r));
    for (int64_t ii = lo; ii < hi; ++ii) {
      const int64_t i = row0 + ii;
      Rng ra(seed, 1, static_cast<uint64_t>(i));
      for (int64_t k = 0; k < r; ++k) a[k] = ra.next_normal();
      double* y = values + ii * n;
      uint8_t* w = mask + ii * n;
      for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t k = 0; k < r; ++k) s += a[k] * B[k * n + j];
        y[j] = s;
      }
      if (sigma > 0.0) {
        Rng rn(seed, 3, static_cast<uint64_t>(i));
        for (int64_t j = 0; j < n; ++j) y[j] += sigma * rn.next_normal();
      }
      Rng rm(seed, 4, static_cast<uint64_t>(i));
      for (int64_t j = 0; j < n; ++j) {
        const bool known = rm.next_unit() <= rho;
        w[j] = known ? 1 : 0;
        if (!known) y[j] = std::nan("");
      }
    }
  };
  std::vector<std::thread> th;
  const int64_t per = (rows + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t lo = t * per, hi = std::min<int64_t>(rows, lo + per);
    if (lo >= hi) break;
    th.emplace_back(work, lo, hi);
  }
  for (auto& x : th) x.join();
  return RSM_OK;
}

// Structured-missingness generator for BASELINE config 5 (SURVEY.md section
// 8(f) row 1; the reference has none, SPEC.md:448 lists it as a non-goal).
// An affine-camera track matrix: point i is X_i = (x, y, z, 1) with x, y, z
// uniform in [-1, 1] (Rng(seed, TRACK_POINT, i).next_unit), frame f has a
// 2 x 4 camera P_f with N(0,1) entries (Rng(seed, TRACK_CAMERA, f), row-major),
// so the noiseless matrix Y[i][2f + c] = P_f[c] . X_i has rank 4. Point i is
// visible over one contiguous window of frames: length L uniform in
// [wmin, wmax] and start uniform in [0, frames - L] (Rng(seed, TRACK_WINDOW,
// i).next_below, length first). Visible cells get sigma * N(0,1) noise from
// Rng(seed, TRACK_NOISE, i), drawn in column order; hidden cells hold NaN.
extern "C" rsm_status rsm_generate_tracks(int64_t points, int64_t frames, int64_t wmin, int64_t wmax,
                                          double sigma, uint64_t seed, int64_t row0, int64_t rows,
                                          double* values, uint8_t* mask) {
  if (points < 1 || frames < 1 || wmin < 1 || wmax < wmin || wmax > frames || row0 < 0 || rows < 0 ||
      row0 + rows > points)
    return RSM_ERR_INVALID_CONFIG;
  const int64_t n = 2 * frames;
  std::vector<double> P((size_t)(frames * 8));
  for (int64_t f = 0; f < frames; ++f) {
    rsmh::Rng rc(seed, rsmh::stream::TRACK_CAMERA, (uint64_t)f);
    for (int q = 0; q < 8; ++q) P[(size_t)(f * 8 + q)] = rc.next_normal();
  }
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (rows * n < (int64_t)1 << 20) nt = 1;
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t t = lo; t < hi; ++t) {
      const int64_t i = row0 + t;
      double* y = values + t * n;
      uint8_t* w = mask + t * n;
      rsmh::Rng rp(seed, rsmh::stream::TRACK_POINT, (uint64_t)i);
      double X[4];
      for (int q = 0; q < 3; ++q) X[q] = 2.0 * rp.next_unit() - 1.0;
      X[3] = 1.0;
      rsmh::Rng rw(seed, rsmh::stream::TRACK_WINDOW, (uint64_t)i);
      const int64_t L = wmin + (int64_t)rw.next_below((uint64_t)(wmax - wmin + 1));
      const int64_t f0 = (int64_t)rw.next_below((uint64_t)(frames - L + 1));
      rsmh::Rng rn(seed, rsmh::stream::TRACK_NOISE, (uint64_t)i);
      for (int64_t j = 0; j < n; ++j) {
        const int64_t f = j >> 1;
        if (f < f0 || f >= f0 + L) {
          y[j] = std::nan("");
          w[j] = 0;
          continue;
        }
        const double* pr = P.data() + f * 8 + (j & 1) * 4;
        double s = 0.0;
        for (int q = 0; q < 4; ++q) s += pr[q] * X[q];
        if (sigma > 0.0) s += sigma * rn.next_normal();
        y[j] = s;
        w[j] = 1;
      }
    }
  };
  std::vector<std::thread> th;
  const int64_t per = (rows + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t lo = t * per, hi = std::min<int64_t>(rows, lo + per);
    if (lo >= hi) break;
    th.emplace_back(work, lo, hi);
  }
  for (auto& x : th) x.join();
  return RSM_OK;
}
