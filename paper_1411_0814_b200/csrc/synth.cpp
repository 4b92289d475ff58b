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
