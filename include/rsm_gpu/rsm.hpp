// rsm_gpu/rsm.hpp -- header-only C++ drop-in for callers of the reference
// RSM library (namespace rsm, /root/reference/proj/include/rsm/*.hpp), routed
// through the B200 C-ABI (include/rsm_b200.h, librsm_b200.so).
//
// Same type and function names, argument meaning and error behaviour as the
// reference for the hot path:
//   rsm::MaskedMatrix, Factorization, DecompositionReport   (core.hpp:22-90)
//   rsm::Mode, RsmConfig, TrialPlan, TrialParams            (solver.hpp:13-34, planner.hpp:12-18)
//   rsm::Error, errc, exit_code                             (error.hpp:8-46)
//   rsm::trial_params, harvest_gram, solve_v, solve_u,
//   rsm::decompose, masked_residual_norm, density           (solver.hpp:36-77, core.hpp:92-96)
// A caller switches by including this header instead of <rsm/solver.hpp> and
// linking librsm_b200.so instead of librsm.a. GramAccumulator is reduced to
// the accessors decompose-level callers use (n, z, at, data, raw).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../rsm_b200.h"

namespace rsm {

using index_t = std::int64_t;

enum class errc { invalid_config, parse_io, insufficient_coverage, internal };

class Error : public std::runtime_error {
 public:
  Error(errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  errc code() const noexcept { return code_; }

 private:
  errc code_;
};

inline int exit_code(errc c) noexcept {
  switch (c) {
    case errc::invalid_config: return 2;
    case errc::parse_io: return 3;
    case errc::insufficient_coverage: return 4;
    case errc::internal: return 1;
  }
  return 1;
}

namespace detail {
inline void check(rsm_status st, const rsm_ctx* ctx = nullptr) {
  if (st == RSM_OK) return;
  const char* m = rsm_last_error(ctx);
  const std::string what = m ? m : "rsm error";
  switch (st) {
    case RSM_ERR_INVALID_CONFIG: throw Error(errc::invalid_config, what);
    case RSM_ERR_PARSE_IO: throw Error(errc::parse_io, what);
    case RSM_ERR_INSUFFICIENT_COVERAGE: throw Error(errc::insufficient_coverage, what);
    default: throw Error(errc::internal, what);
  }
}
}  // namespace detail

enum class Mode { M1, M2 };
inline const char* mode_name(Mode m) noexcept { return m == Mode::M1 ? "m1" : "m2"; }

struct MaskedMatrix {
  index_t m = 0;
  index_t n = 0;
  std::vector<double> values;
  std::vector<std::uint8_t> mask;

  MaskedMatrix() = default;
  MaskedMatrix(index_t rows, index_t cols)
      : m(rows), n(cols),
        values(static_cast<std::size_t>(rows * cols), std::numeric_limits<double>::quiet_NaN()),
        mask(static_cast<std::size_t>(rows * cols), 0) {
    if (rows < 1 || cols < 1) throw Error(errc::invalid_config, "matrix dimensions must be positive");
  }
  double operator()(index_t i, index_t j) const { return values[static_cast<std::size_t>(i * n + j)]; }
  bool known(index_t i, index_t j) const { return mask[static_cast<std::size_t>(i * n + j)] != 0; }
  void set(index_t i, index_t j, double v) {
    values[static_cast<std::size_t>(i * n + j)] = v;
    mask[static_cast<std::size_t>(i * n + j)] = 1;
  }
  index_t known_count() const {
    index_t c = 0;
    for (auto b : mask) c += b;
    return c;
  }
};

struct Factorization {
  index_t m = 0, n = 0, r = 0;
  std::vector<double> u;  // m x r row-major
  std::vector<double> v;  // n x r row-major
  Factorization() = default;
  Factorization(index_t rows, index_t cols, index_t rank)
      : m(rows), n(cols), r(rank), u(static_cast<std::size_t>(rows * rank), 0.0),
        v(static_cast<std::size_t>(cols * rank), 0.0) {
    if (rank < 1) throw Error(errc::invalid_config, "rank must be positive");
    if (rank >= rows || rank >= cols) throw Error(errc::invalid_config, "rank must be below min(rows, cols)");
  }
};

struct DecompositionReport {
  double e = 0.0;
  std::uint64_t trials_attempted = 0;
  std::uint64_t trials_accepted = 0;
  std::uint64_t z = 0;
  index_t underdetermined_rows = 0;
  index_t gram_rank = 0;
  bool borderline_rank_gate = false;
  double wall_time = 0.0;
};

struct TrialPlan {
  std::uint64_t trials = 0;
  double epsilon = 0.99;
};

struct RsmConfig {
  index_t rank = 0;
  Mode mode = Mode::M1;
  index_t block = 0;
  index_t vectors_per_trial = 0;
  TrialPlan plan;
  std::uint64_t seed = 0;
  double gram_rank_tol = 1e-9;
  index_t min_dim = 0;
  int workers = 0;  // accepted, ignored: results never depend on it
};

struct TrialParams {
  Mode mode = Mode::M1;
  index_t block = 0;
  index_t ell = 0;
  index_t rank = 0;
  index_t min_count = 0;
  std::uint64_t seed = 0;
};

class GramAccumulator {
 public:
  GramAccumulator() = default;
  explicit GramAccumulator(index_t n) : n_(n), g_(static_cast<std::size_t>(n * n), 0.0) {}
  index_t n() const { return n_; }
  std::uint64_t z() const { return z_; }
  double at(index_t i, index_t j) const { return g_[static_cast<std::size_t>(i * n_ + j)]; }
  const std::vector<double>& data() const { return g_; }
  std::vector<double>& raw() { return g_; }
  void set_z(std::uint64_t z) { z_ = z; }

 private:
  index_t n_ = 0;
  std::uint64_t z_ = 0;
  std::vector<double> g_;
};

struct HarvestResult {
  GramAccumulator gram;
  std::uint64_t attempted = 0;
  std::uint64_t accepted = 0;
};
struct SolveVResult {
  std::vector<double> v;
  index_t gram_rank = 0;
  bool borderline = false;
};
struct SolveUResult {
  std::vector<double> u;
  index_t underdetermined_rows = 0;
};

namespace detail {
inline rsm_config to_c(const RsmConfig& c) {
  rsm_config o;
  rsm_config_default(&o);
  o.rank = c.rank;
  o.mode = c.mode == Mode::M1 ? RSM_MODE_M1 : RSM_MODE_M2;
  o.block = c.block;
  o.vectors_per_trial = c.vectors_per_trial;
  o.trials = c.plan.trials;
  o.epsilon = c.plan.epsilon;
  o.seed = c.seed;
  o.gram_rank_tol = c.gram_rank_tol;
  o.min_dim = c.min_dim;
  o.workers = c.workers;
  return o;
}
inline rsm_trial_params to_c(const TrialParams& p) {
  rsm_trial_params o;
  o.mode = p.mode == Mode::M1 ? RSM_MODE_M1 : RSM_MODE_M2;
  o.block = p.block;
  o.ell = p.ell;
  o.rank = p.rank;
  o.min_count = p.min_count;
  o.seed = p.seed;
  return o;
}
}  // namespace detail

inline double density(const MaskedMatrix& M) {
  return static_cast<double>(M.known_count()) / (static_cast<double>(M.m) * static_cast<double>(M.n));
}

inline TrialParams trial_params(const RsmConfig& cfg, const MaskedMatrix& M) {
  const rsm_config c = detail::to_c(cfg);
  rsm_trial_params p;
  detail::check(rsm_make_trial_params(&c, M.m, M.n, &p));
  TrialParams o;
  o.mode = p.mode == RSM_MODE_M1 ? Mode::M1 : Mode::M2;
  o.block = p.block;
  o.ell = p.ell;
  o.rank = p.rank;
  o.min_count = p.min_count;
  o.seed = p.seed;
  return o;
}

inline HarvestResult harvest_gram(const MaskedMatrix& M, const TrialParams& p, std::uint64_t trials,
                                  int /*workers*/ = 0) {
  HarvestResult h;
  h.gram = GramAccumulator(M.n);
  const rsm_trial_params c = detail::to_c(p);
  std::uint64_t z = 0;
  detail::check(rsm_harvest_gram(M.values.data(), M.mask.data(), M.m, M.n, &c, trials, h.gram.raw().data(),
                                 &h.attempted, &h.accepted, &z));
  h.gram.set_z(z);
  return h;
}

inline SolveVResult solve_v(GramAccumulator& G, index_t r, double tol) {
  SolveVResult s;
  s.v.assign(static_cast<std::size_t>(G.n() * (r > 0 ? r : 1)), 0.0);
  std::int64_t gr = 0;
  std::int32_t bl = 0;
  detail::check(rsm_solve_v(G.raw().data(), G.n(), r, tol, s.v.data(), &gr, &bl));
  s.gram_rank = gr;
  s.borderline = bl != 0;
  return s;
}

inline SolveUResult solve_u(const MaskedMatrix& M, const std::vector<double>& vhat, index_t r,
                            int /*workers*/ = 0) {
  if (r < 1) throw Error(errc::invalid_config, "solve_u: rank must be positive");
  if (static_cast<index_t>(vhat.size()) != M.n * r)
    throw Error(errc::invalid_config, "solve_u: basis shape does not match matrix");
  SolveUResult s;
  s.u.assign(static_cast<std::size_t>(M.m * r), 0.0);
  std::int64_t fl = 0;
  detail::check(rsm_solve_u(M.values.data(), M.mask.data(), M.m, M.n, vhat.data(), r, s.u.data(), &fl));
  s.underdetermined_rows = fl;
  return s;
}

inline std::pair<Factorization, DecompositionReport> decompose(const MaskedMatrix& M, const RsmConfig& cfg) {
  const rsm_config c = detail::to_c(cfg);
  const index_t r = cfg.rank > 0 ? cfg.rank : 1;
  std::vector<double> U(static_cast<std::size_t>(M.m * r)), V(static_cast<std::size_t>(M.n * r));
  rsm_report rep;
  detail::check(rsm_decompose(M.values.data(), M.mask.data(), M.m, M.n, &c, U.data(), V.data(), &rep));
  Factorization F(M.m, M.n, cfg.rank);
  F.u = std::move(U);
  F.v = std::move(V);
  DecompositionReport d;
  d.e = rep.e;
  d.trials_attempted = rep.trials_attempted;
  d.trials_accepted = rep.trials_accepted;
  d.z = rep.z;
  d.underdetermined_rows = rep.underdetermined_rows;
  d.gram_rank = rep.gram_rank;
  d.borderline_rank_gate = rep.borderline_rank_gate != 0;
  d.wall_time = rep.wall_time;
  return {std::move(F), d};
}

inline double masked_residual_norm(const MaskedMatrix& M, const Factorization& F) {
  if (F.m != M.m || F.n != M.n) throw Error(errc::invalid_config, "factorization shape does not match matrix");
  double e = 0.0;
  detail::check(rsm_masked_residual_norm(M.values.data(), M.mask.data(), M.m, M.n, F.u.data(), F.v.data(), F.r, &e));
  return e;
}

// baseline_als (include/rsm/solver.hpp:79-81): the device ALS baseline
inline std::pair<Factorization, DecompositionReport> baseline_als(const MaskedMatrix& M, index_t r,
                                                                  index_t iterations, std::uint64_t seed,
                                                                  int workers = 0) {
  (void)workers;
  const index_t rr = r > 0 ? r : 1;
  std::vector<double> U(static_cast<std::size_t>(M.m * rr)), V(static_cast<std::size_t>(M.n * rr));
  rsm_report rep;
  detail::check(rsm_als(M.values.data(), M.mask.data(), M.m, M.n, r, iterations, seed, U.data(), V.data(), &rep));
  Factorization F(M.m, M.n, r);
  F.u = std::move(U);
  F.v = std::move(V);
  DecompositionReport d;
  d.e = rep.e;
  d.underdetermined_rows = rep.underdetermined_rows;
  d.wall_time = rep.wall_time;
  return {std::move(F), d};
}

// load_matrix / save_matrix / dataset_checksum (include/rsm/io.hpp:14-22)
inline MaskedMatrix load_matrix(const std::string& path) {
  double* v = nullptr;
  std::uint8_t* w = nullptr;
  std::int64_t m = 0, n = 0;
  detail::check(rsm_load_matrix_csv(path.c_str(), &v, &w, &m, &n));
  MaskedMatrix M(m, n);
  std::copy(v, v + m * n, M.values.begin());
  std::copy(w, w + m * n, M.mask.begin());
  rsm_free(v);
  rsm_free(w);
  return M;
}

inline void save_matrix(const MaskedMatrix& M, const std::string& path) {
  detail::check(rsm_save_matrix_csv(path.c_str(), M.values.data(), M.mask.data(), M.m, M.n));
}

inline std::uint64_t dataset_checksum(const MaskedMatrix& M) {
  std::uint64_t h = 0;
  detail::check(rsm_dataset_checksum(M.values.data(), M.mask.data(), M.m, M.n, &h));
  return h;
}

}  // namespace rsm
