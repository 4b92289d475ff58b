// rsm::generate for drop-in callers (include/rsm/synth.hpp of the reference):
// the Eq. 31 test instance from the reference's streams (src/synth.cpp:12-71)
// with its ground truth kept. Test-data generation on the host, as in the
// reference; the observed matrix equals rsm_generate's (library) bit for bit.
// truth_basis = the r leading right singular vectors of Ybar = A B, computed
// from the r x n matrix L^T B (A^T A = L L^T, so A B and L^T B share them).
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "../rsm.hpp"
#include "rng.hpp"

namespace rsm {

struct SyntheticSpec {
  index_t m = 0;
  index_t n = 0;
  index_t r = 0;
  double rho = 1.0;
  double sigma = 0.0;
  std::uint64_t seed = 0;
};

struct SyntheticInstance {
  MaskedMatrix observed;
  std::vector<double> ground_truth;  // row-major m*n
  std::vector<double> noise;         // row-major m*n
  std::vector<double> truth_basis;   // row-major n*r, orthonormal columns
};

inline SyntheticInstance generate(const SyntheticSpec& spec) {
  if (spec.m < 1 || spec.n < 1) throw Error(errc::invalid_config, "synthetic spec: dimensions must be positive");
  if (spec.r < 1 || spec.r >= std::min(spec.m, spec.n))
    throw Error(errc::invalid_config, "synthetic spec: rank must lie in [1, min(m,n))");
  if (!(spec.rho > 0.0 && spec.rho <= 1.0))
    throw Error(errc::invalid_config, "synthetic spec: density must lie in (0,1]");
  if (spec.sigma < 0.0) throw Error(errc::invalid_config, "synthetic spec: sigma must be nonnegative");
  const index_t m = spec.m, n = spec.n, r = spec.r;
  std::vector<double> A(static_cast<std::size_t>(m * r)), B(static_cast<std::size_t>(r * n));
  for (index_t i = 0; i < m; ++i) {
    Rng rng(spec.seed, stream::FACTOR_A, static_cast<std::uint64_t>(i));
    for (index_t k = 0; k < r; ++k) A[i * r + k] = rng.next_normal();
  }
  for (index_t k = 0; k < r; ++k) {
    Rng rng(spec.seed, stream::FACTOR_B, static_cast<std::uint64_t>(k));
    for (index_t j = 0; j < n; ++j) B[k * n + j] = rng.next_normal();
  }
  SyntheticInstance out;
  out.ground_truth.assign(static_cast<std::size_t>(m * n), 0.0);
  for (index_t i = 0; i < m; ++i)
    for (index_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (index_t k = 0; k < r; ++k) s += A[i * r + k] * B[k * n + j];
      out.ground_truth[i * n + j] = s;
    }
  out.noise.assign(static_cast<std::size_t>(m * n), 0.0);
  if (spec.sigma > 0.0)
    for (index_t i = 0; i < m; ++i) {
      Rng rng(spec.seed, stream::NOISE, static_cast<std::uint64_t>(i));
      for (index_t j = 0; j < n; ++j) out.noise[i * n + j] = spec.sigma * rng.next_normal();
    }
  out.observed = MaskedMatrix(m, n);
  for (index_t i = 0; i < m; ++i) {
    Rng rng(spec.seed, stream::MASK, static_cast<std::uint64_t>(i));
    for (index_t j = 0; j < n; ++j)
      if (rng.next_unit() <= spec.rho) out.observed.set(i, j, out.ground_truth[i * n + j] + out.noise[i * n + j]);
  }
  // truth basis: C = A^T A = L L^T, M = L^T B (r x n), H = M M^T = U S^2 U^T,
  // V = M^T U S^-1 (descending S)
  std::vector<double> C(static_cast<std::size_t>(r * r), 0.0), L(C.size(), 0.0);
  for (index_t i = 0; i < m; ++i)
    for (index_t a = 0; a < r; ++a)
      for (index_t b = 0; b < r; ++b) C[a * r + b] += A[i * r + a] * A[i * r + b];
  for (index_t j = 0; j < r; ++j) {
    double d = C[j * r + j];
    for (index_t k = 0; k < j; ++k) d -= L[j * r + k] * L[j * r + k];
    L[j * r + j] = std::sqrt(std::max(d, 0.0));
    for (index_t i = j + 1; i < r; ++i) {
      double v = C[i * r + j];
      for (index_t k = 0; k < j; ++k) v -= L[i * r + k] * L[j * r + k];
      L[i * r + j] = L[j * r + j] > 0.0 ? v / L[j * r + j] : 0.0;
    }
  }
  std::vector<double> M(static_cast<std::size_t>(r * n), 0.0);  // M = L^T B
  for (index_t a = 0; a < r; ++a)
    for (index_t k = a; k < r; ++k)
      for (index_t j = 0; j < n; ++j) M[a * n + j] += L[k * r + a] * B[k * n + j];
  std::vector<double> H(static_cast<std::size_t>(r * r), 0.0), U(H.size(), 0.0);
  for (index_t a = 0; a < r; ++a)
    for (index_t b = 0; b < r; ++b) {
      double s = 0.0;
      for (index_t j = 0; j < n; ++j) s += M[a * n + j] * M[b * n + j];
      H[a * r + b] = s;
    }
  for (index_t a = 0; a < r; ++a) U[a * r + a] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {  // cyclic Jacobi on the r x r H
    double off = 0.0;
    for (index_t a = 0; a < r; ++a)
      for (index_t b = a + 1; b < r; ++b) off += H[a * r + b] * H[a * r + b];
    if (off <= 1e-30 * (H[0] * H[0] + 1e-300)) break;
    for (index_t p = 0; p < r - 1; ++p)
      for (index_t q = p + 1; q < r; ++q) {
        const double apq = H[p * r + q];
        if (apq == 0.0) continue;
        const double z = (H[q * r + q] - H[p * r + p]) / (2.0 * apq);
        const double t = (z >= 0.0 ? 1.0 : -1.0) / (std::fabs(z) + std::sqrt(1.0 + z * z));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (index_t k = 0; k < r; ++k) {
          const double x = H[k * r + p], y = H[k * r + q];
          H[k * r + p] = c * x - s * y;
          H[k * r + q] = s * x + c * y;
        }
        for (index_t k = 0; k < r; ++k) {
          const double x = H[p * r + k], y = H[q * r + k];
          H[p * r + k] = c * x - s * y;
          H[q * r + k] = s * x + c * y;
        }
        for (index_t k = 0; k < r; ++k) {
          const double x = U[k * r + p], y = U[k * r + q];
          U[k * r + p] = c * x - s * y;
          U[k * r + q] = s * x + c * y;
        }
      }
  }
  std::vector<index_t> ord(static_cast<std::size_t>(r));
  std::iota(ord.begin(), ord.end(), index_t{0});
  std::stable_sort(ord.begin(), ord.end(), [&](index_t a, index_t b) { return H[a * r + a] > H[b * r + b]; });
  out.truth_basis.assign(static_cast<std::size_t>(n * r), 0.0);
  for (index_t c = 0; c < r; ++c) {
    const index_t k = ord[c];
    const double sg = std::sqrt(std::max(H[k * r + k], 0.0));
    for (index_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (index_t a = 0; a < r; ++a) s += M[a * n + j] * U[a * r + k];
      out.truth_basis[j * r + c] = sg > 0.0 ? s / sg : 0.0;
    }
  }
  return out;
}

}  // namespace rsm
