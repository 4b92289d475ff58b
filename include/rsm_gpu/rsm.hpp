// rsm_gpu/rsm.hpp -- header-only C++ drop-in for callers of the reference
// RSM library (namespace rsm, /root/reference/proj/include/rsm/*.hpp), routed
// through the B200 C-ABI (include/rsm_b200.h, librsm_b200.so).
//
// Same type and function names, argument meaning and error behaviour as the
// reference for the hot path:
//   rsm::MaskedMatrix, Factorization, DecompositionReport   (core.hpp:22-90)
//   rsm::Mode, RsmConfig, TrialPlan, TrialParams            (solver.hpp:13-34, planner.hpp:12-18)
//   rsm::Error, errc, exit_code                             (error.hpp:8-46)
//   rsm::trial_params, attempt_trial, harvest_gram, solve_v, solve_u,
//   rsm::decompose, baseline_als, reference::{harvest_gram, solve_u}
//                                                           (solver.hpp:36-87)
//   rsm::masked_residual_norm, masked_objective, norm_tag, density,
//   MaskedMatrix::transposed                                (core.hpp:50-96)
//   rsm::Submatrix, TrialRng, sample_m1, sample_m2, visited_fraction
//                                                           (sampler.hpp:13-50)
//   rsm::ConstraintVector, GramAccumulator (accumulate, accumulate_dense,
//   merge), merge, small_singular_vectors, embed             (spectra.hpp:12-68)
//   rsm::load_matrix, save_matrix, dataset_checksum         (io.hpp:14-22)
// A caller switches by including this header instead of <rsm/solver.hpp> and
// linking librsm_b200.so instead of librsm.a. Every computation runs on the
// device through the C-ABI; GramAccumulator::accumulate buffers the vectors
// and folds them into G on the device (bit-identical to the reference's
// loops) when G is next read. Pure index bookkeeping (transposed,
// visited_fraction, embed, gathering a Submatrix's values) is host code, as
// in the reference.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
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
  // core.hpp:50-56
  MaskedMatrix transposed() const {
    MaskedMatrix t(n, m);
    for (index_t i = 0; i < m; ++i)
      for (index_t j = 0; j < n; ++j)
        if (known(i, j)) t.set(j, i, (*this)(i, j));
    return t;
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

// planner.hpp:10-18 (the Theorem-3 bound planner itself is out of scope:
// callers pass explicit or heuristic trial counts)
enum class PlanSource { theorem3_bound, heuristic, explicit_count };

struct TrialPlan {
  std::uint64_t trials = 0;
  double epsilon = 0.99;
  index_t k_or_l = 0;
  Mode mode = Mode::M1;
  PlanSource source = PlanSource::explicit_count;
};

// planner.cpp:113-120
inline TrialPlan plan_trials_heuristic(index_t n, index_t multiplier = 25) {
  if (n < 1) throw Error(errc::invalid_config, "heuristic plan: n must be positive");
  if (multiplier < 1) throw Error(errc::invalid_config, "heuristic plan: multiplier must be positive");
  TrialPlan plan;
  plan.trials = static_cast<std::uint64_t>(multiplier) * static_cast<std::uint64_t>(n);
  plan.source = PlanSource::heuristic;
  return plan;
}

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

// spectra.hpp:12-19
struct ConstraintVector {
  std::vector<index_t> col_indices;
  std::vector<double> zeta;  // same length as col_indices, unit 2-norm
  double singular_value = 0.0;
};

// spectra.hpp:23-56: G = Xi Xi^T plus the vector count z. accumulate /
// accumulate_dense queue the (embedded) vector; the queue is folded into G on
// the device (rsm_gram_update, vector order, separate multiply and add: the
// reference's bits) before G is read or merged.
class GramAccumulator {
 public:
  GramAccumulator() = default;
  explicit GramAccumulator(index_t n) : n_(n), g_(static_cast<std::size_t>(n * n), 0.0) {
    if (n < 1) throw Error(errc::invalid_config, "gram accumulator: dimension must be positive");
  }
  index_t n() const { return n_; }
  std::uint64_t z() const { return z_; }
  void accumulate(const ConstraintVector& cv) {
    const index_t q = static_cast<index_t>(cv.col_indices.size());
    if (q != static_cast<index_t>(cv.zeta.size()))
      throw Error(errc::invalid_config, "accumulate: index/coefficient length mismatch");
    for (index_t c : cv.col_indices)
      if (c < 0 || c >= n_) throw Error(errc::invalid_config, "accumulate: column index out of range");
    const std::size_t o = pending_.size();
    pending_.resize(o + static_cast<std::size_t>(n_), 0.0);
    for (index_t a = 0; a < q; ++a) pending_[o + static_cast<std::size_t>(cv.col_indices[a])] = cv.zeta[a];
    ++npending_;
    ++z_;
    if (npending_ >= 256) flush();
  }
  void accumulate_dense(const std::vector<double>& xi) {
    if (static_cast<index_t>(xi.size()) != n_) throw Error(errc::invalid_config, "accumulate: dimension mismatch");
    pending_.insert(pending_.end(), xi.begin(), xi.end());
    ++npending_;
    ++z_;
    if (npending_ >= 256) flush();
  }
  void merge(const GramAccumulator& other) {
    if (other.n_ != n_) throw Error(errc::invalid_config, "merge: dimension mismatch");
    other.flush();
    flush_with(other.g_.data());
    z_ += other.z_;
  }
  double at(index_t i, index_t j) const {
    flush();
    return g_[static_cast<std::size_t>(i * n_ + j)];
  }
  const std::vector<double>& data() const {
    flush();
    return g_;
  }
  std::vector<double>& raw() {
    flush();
    return g_;
  }
  void set_z(std::uint64_t z) { z_ = z; }

 private:
  void flush() const { flush_with(nullptr); }
  void flush_with(const double* G2) const {
    if (npending_ == 0 && !G2) return;
    detail::check(rsm_gram_update(g_.data(), n_, npending_ ? pending_.data() : nullptr, npending_, G2));
    pending_.clear();
    npending_ = 0;
  }
  index_t n_ = 0;
  std::uint64_t z_ = 0;
  mutable std::vector<double> g_;
  mutable std::vector<double> pending_;  // queued dense vectors (npending_ x n)
  mutable index_t npending_ = 0;
};

inline GramAccumulator merge(const GramAccumulator& a, const GramAccumulator& b) {
  GramAccumulator out = a;
  out.merge(b);
  return out;
}

// spectra.cpp:88-96
inline std::vector<double> embed(const ConstraintVector& cv, index_t n) {
  std::vector<double> xi(static_cast<std::size_t>(n), 0.0);
  for (std::size_t t = 0; t < cv.col_indices.size(); ++t) {
    const index_t c = cv.col_indices[t];
    if (c < 0 || c >= n) throw Error(errc::invalid_config, "embed: column index out of range");
    xi[static_cast<std::size_t>(c)] = cv.zeta[t];
  }
  return xi;
}

// sampler.hpp:13-37
struct Submatrix {
  std::vector<index_t> row_indices;
  std::vector<index_t> col_indices;
  std::vector<double> values;  // row-major |rows| x |cols|
  index_t rows() const { return static_cast<index_t>(row_indices.size()); }
  index_t cols() const { return static_cast<index_t>(col_indices.size()); }
  double operator()(index_t i, index_t j) const { return values[static_cast<std::size_t>(i * cols() + j)]; }
};

struct TrialRng {
  std::uint64_t master_seed = 0;
  std::uint64_t trial_index = 0;
};

namespace detail {
inline std::optional<Submatrix> sample(const MaskedMatrix& M, bool m2, index_t count, const TrialRng& rng,
                                       index_t min_keep) {
  std::vector<std::int64_t> drawn(static_cast<std::size_t>(count > 0 ? count : 1));
  std::vector<std::int64_t> kept(static_cast<std::size_t>(m2 ? M.n : M.m));
  std::int64_t nk = 0;
  check(rsm_sample(M.values.data(), M.mask.data(), M.m, M.n, m2 ? RSM_MODE_M2 : RSM_MODE_M1, count,
                   rng.master_seed, rng.trial_index, drawn.data(), kept.data(), &nk));
  if (nk < min_keep) return std::nullopt;
  drawn.resize(static_cast<std::size_t>(count));
  kept.resize(static_cast<std::size_t>(nk));
  Submatrix S;
  S.row_indices = m2 ? drawn : kept;
  S.col_indices = m2 ? kept : drawn;
  S.values.resize(S.row_indices.size() * S.col_indices.size());
  for (index_t i = 0; i < S.rows(); ++i)
    for (index_t j = 0; j < S.cols(); ++j)
      S.values[static_cast<std::size_t>(i * S.cols() + j)] = M(S.row_indices[i], S.col_indices[j]);
  return S;
}
}  // namespace detail

inline std::optional<Submatrix> sample_m1(const MaskedMatrix& M, index_t l, const TrialRng& rng,
                                          index_t min_rows = 1) {
  return detail::sample(M, false, l, rng, min_rows);
}
inline std::optional<Submatrix> sample_m2(const MaskedMatrix& M, index_t k, const TrialRng& rng,
                                          index_t min_cols = 1) {
  return detail::sample(M, true, k, rng, min_cols);
}

// sampler.cpp:89-101
inline double visited_fraction(const std::vector<Submatrix>& trials, const MaskedMatrix& M) {
  const index_t known = M.known_count();
  if (known == 0) return 0.0;
  std::vector<std::uint8_t> seen(static_cast<std::size_t>(M.m * M.n), 0);
  for (const Submatrix& S : trials)
    for (index_t i : S.row_indices)
      for (index_t j : S.col_indices) seen[static_cast<std::size_t>(i * M.n + j)] = 1;
  index_t hit = 0;
  for (std::size_t p = 0; p < seen.size(); ++p)
    if (seen[p] && M.mask[p]) ++hit;
  return static_cast<double>(hit) / static_cast<double>(known);
}

// spectra.hpp:61 (spectra.cpp:48-86) on the device
inline std::vector<ConstraintVector> small_singular_vectors(const Submatrix& S, index_t r, index_t ell) {
  const index_t q = S.cols();
  std::vector<double> zeta(static_cast<std::size_t>((ell > 0 ? ell : 1) * (q > 0 ? q : 1)));
  std::vector<double> sv(static_cast<std::size_t>(ell > 0 ? ell : 1));
  detail::check(rsm_small_singular_vectors(S.values.data(), S.rows(), q, r, ell, zeta.data(), sv.data()));
  std::vector<ConstraintVector> out(static_cast<std::size_t>(ell));
  for (index_t t = 0; t < ell; ++t) {
    out[t].col_indices = S.col_indices;
    out[t].zeta.assign(zeta.begin() + t * q, zeta.begin() + (t + 1) * q);
    out[t].singular_value = sv[t];
  }
  return out;
}

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

// solver.hpp:40-42 (harvest.cpp:37-51): sample, then the small vectors
inline std::optional<std::vector<ConstraintVector>> attempt_trial(const MaskedMatrix& M, const TrialParams& p,
                                                                  std::uint64_t index) {
  const TrialRng rng{p.seed, index};
  if (p.mode == Mode::M1) {
    std::optional<Submatrix> S = sample_m1(M, p.block, rng, p.min_count);
    if (!S) return std::nullopt;
    return small_singular_vectors(*S, p.rank, p.ell);
  }
  std::optional<Submatrix> S = sample_m2(M, p.block, rng, p.min_count);
  if (!S) return std::nullopt;
  const index_t avail = S->cols() - p.rank;
  const index_t ell = p.ell > 0 ? std::min(p.ell, avail) : avail;
  return small_singular_vectors(*S, p.rank, ell);
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

// core.hpp:92-95 (core.cpp:41-44)
enum class norm_tag { frobenius, l1 };
inline double masked_objective(const MaskedMatrix& M, const Factorization& F, norm_tag tag) {
  if (F.m != M.m || F.n != M.n) throw Error(errc::invalid_config, "factorization shape does not match matrix");
  double out = 0.0;
  detail::check(rsm_masked_objective(M.values.data(), M.mask.data(), M.m, M.n, F.u.data(), F.v.data(), F.r,
                                     tag == norm_tag::frobenius ? 0 : 1, &out));
  return out;
}

// solver.hpp:84-87: the reference keeps serial implementations as ground
// truth for its parallel kernels; here both names reach the same device path
// (results never depend on the worker count)
namespace reference {
inline HarvestResult harvest_gram(const MaskedMatrix& M, const TrialParams& p, std::uint64_t trials) {
  return rsm::harvest_gram(M, p, trials);
}
inline SolveUResult solve_u(const MaskedMatrix& M, const std::vector<double>& vhat, index_t r) {
  return rsm::solve_u(M, vhat, r);
}
}  // namespace reference

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
