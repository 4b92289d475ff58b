// Drop-in check: reference-style test cases (after /root/reference/proj/tests/
// test_solver.cpp) compiled against include/rsm_gpu/rsm.hpp and linked to
// librsm_b200.so -- the reference's C++ call sites unchanged, the B200 path
// underneath. Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rsm_gpu/rsm.hpp"

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(x)) { ++g_fail; std::fprintf(stderr, "%s:%d FAILED: %s\n", __FILE__, __LINE__, #x); } \
  } while (0)
#define CHECK_THROWS_CODE(expr, want)                                         \
  do {                                                                        \
    ++g_checks;                                                               \
    bool ok_ = false;                                                         \
    try { (void)(expr); } catch (const rsm::Error& e) { ok_ = e.code() == (want); } \
    if (!ok_) { ++g_fail; std::fprintf(stderr, "%s:%d FAILED: throws %s\n", __FILE__, __LINE__, #expr); } \
  } while (0)

using namespace rsm;

static MaskedMatrix synth(index_t m, index_t n, index_t r, double rho, double sigma, std::uint64_t seed) {
  MaskedMatrix M(m, n);
  if (rsm_generate(m, n, r, rho, sigma, seed, 0, m, M.values.data(), M.mask.data()) != RSM_OK) std::abort();
  return M;
}

int main() {
  {  // solve_v recovers the small eigenspace of a diagonal gram (test_solver.cpp:46-63)
    GramAccumulator G(4);
    G.raw()[0] = 5.0;
    G.raw()[5] = 4.0;
    const SolveVResult res = solve_v(G, 2, 1e-9);
    CHECK(res.gram_rank == 2);
    CHECK(!res.borderline);
    for (index_t i = 0; i < 4; ++i)
      for (index_t j = 0; j < 4; ++j) {
        double p = 0.0;
        for (index_t c = 0; c < 2; ++c) p += res.v[i * 2 + c] * res.v[j * 2 + c];
        CHECK(std::fabs(p - ((i == j && i >= 2) ? 1.0 : 0.0)) <= 1e-12);
      }
  }
  {  // rank gate (:65-77) and borderline (:79-86)
    GramAccumulator G(4);
    G.raw()[0] = 5.0;
    CHECK_THROWS_CODE(solve_v(G, 2, 1e-9), errc::insufficient_coverage);
    GramAccumulator H(4);
    H.raw()[0] = 5.0;
    H.raw()[5] = 2e-8;
    const SolveVResult res = solve_v(H, 2, 1e-9);
    CHECK(res.gram_rank == 2);
    CHECK(res.borderline);
  }
  {  // solve_u: plain LS, empty rows, minimum norm, degenerate basis (:140-212)
    MaskedMatrix M(1, 4);
    for (index_t j = 0; j < 4; ++j) M.set(0, j, 1.0);
    SolveUResult r1 = solve_u(M, {0.5, 0.5, 0.5, 0.5}, 1);
    CHECK(r1.underdetermined_rows == 0 && std::fabs(r1.u[0] - 2.0) <= 1e-12);
    MaskedMatrix E(3, 4);
    for (index_t j = 0; j < 4; ++j) { E.set(0, j, 1.0); E.set(2, j, 3.0); }
    SolveUResult r2 = solve_u(E, {0.5, 0.5, 0.5, 0.5}, 1);
    CHECK(r2.underdetermined_rows == 1 && r2.u[1] == 0.0 && std::fabs(r2.u[2] - 6.0) <= 1e-12);
    MaskedMatrix O(1, 4);
    O.set(0, 1, 2.0);
    std::vector<double> vh(8, 0.0);
    vh[2] = vh[3] = 1.0;
    SolveUResult r3 = solve_u(O, vh, 2);
    CHECK(r3.underdetermined_rows == 1 && std::fabs(r3.u[0] - 1.0) <= 1e-10 && std::fabs(r3.u[1] - 1.0) <= 1e-10);
    MaskedMatrix D(2, 3);
    for (index_t i = 0; i < 2; ++i)
      for (index_t j = 0; j < 3; ++j) D.set(i, j, static_cast<double>(i + j + 1));
    SolveUResult r4 = solve_u(D, {1, 1, 2, 2, 3, 3}, 2);
    CHECK(r4.underdetermined_rows == 2);
    for (index_t i = 0; i < 2; ++i) CHECK(std::fabs(r4.u[i * 2] - r4.u[i * 2 + 1]) <= 1e-10);
  }
  {  // noiseless decomposition recovers the planted factorization (:245-269)
    const MaskedMatrix M = synth(200, 40, 3, 0.5, 0.0, 17);
    RsmConfig cfg;
    cfg.rank = 3;
    cfg.seed = 17;
    cfg.plan.trials = 25 * 40;  // plan_trials_heuristic(n)
    const auto [F, rep] = decompose(M, cfg);
    CHECK(rep.e <= 1e-8);
    CHECK(rep.trials_accepted == cfg.plan.trials);
    CHECK(rep.gram_rank >= 40 - 3);
    CHECK(std::fabs(rep.e - masked_residual_norm(M, F)) <= 1e-12);
  }
  {  // wide matrices run on the transpose (:304-324); row branch floor (:326-344)
    const MaskedMatrix W = synth(30, 90, 2, 0.6, 0.0, 71);
    RsmConfig cfg;
    cfg.rank = 2;
    cfg.seed = 7;
    cfg.plan.trials = 25 * 30;
    const auto [F, rep] = decompose(W, cfg);
    CHECK(F.u.size() == 30 * 2 && F.v.size() == 90 * 2 && rep.e <= 1e-8);
    const MaskedMatrix R2 = synth(150, 30, 2, 0.85, 0.0, 83);
    RsmConfig c2;
    c2.rank = 2;
    c2.mode = Mode::M2;
    c2.seed = 83;
    c2.plan.trials = 300;
    const auto [F2, rep2] = decompose(R2, c2);
    CHECK(rep2.e <= 1e-8 && rep2.z >= rep2.trials_accepted);
  }
  {  // validation (:346-370)
    MaskedMatrix M = synth(20, 10, 3, 0.9, 0.1, 5);
    RsmConfig cfg;
    cfg.rank = 10;
    cfg.plan.trials = 250;
    CHECK_THROWS_CODE(decompose(M, cfg), errc::invalid_config);
    cfg.rank = 3;
    cfg.block = 2;
    CHECK_THROWS_CODE(decompose(M, cfg), errc::invalid_config);
    cfg.block = 0;
    cfg.plan.epsilon = 1.0;
    CHECK_THROWS_CODE(decompose(M, cfg), errc::invalid_config);
    cfg.plan.epsilon = 0.99;
    cfg.plan.trials = 0;
    CHECK_THROWS_CODE(decompose(M, cfg), errc::invalid_config);
    MaskedMatrix empty(4, 4);
    RsmConfig e;
    e.rank = 2;
    e.plan.trials = 100;
    CHECK_THROWS_CODE(decompose(empty, e), errc::insufficient_coverage);
  }
  {  // determinism across runs and worker counts (:271-302)
    const MaskedMatrix M = synth(120, 24, 2, 0.6, 0.2, 53);
    RsmConfig cfg;
    cfg.rank = 2;
    cfg.seed = 99;
    cfg.plan.trials = 600;
    const auto [F1, r1] = decompose(M, cfg);
    cfg.workers = 3;
    const auto [F2, r2] = decompose(M, cfg);
    CHECK(F1.u == F2.u && F1.v == F2.v && r1.e == r2.e && r1.z == r2.z);
  }
  {  // baseline_als (als.cpp:11-44) and the loader path (io.hpp:14-22)
    const MaskedMatrix M = synth(200, 40, 3, 0.7, 1e-3, 21);
    const auto [F, rep] = baseline_als(M, 3, 5, 21);
    CHECK(F.u.size() == 200 * 3 && std::fabs(rep.e - masked_residual_norm(M, F)) <= 1e-12 * rep.e + 1e-15);
    CHECK_THROWS_CODE(baseline_als(M, 0, 5, 1), errc::invalid_config);
    save_matrix(M, "dropin_io.csv");
    const MaskedMatrix R = load_matrix("dropin_io.csv");
    CHECK(R.m == M.m && R.n == M.n && R.mask == M.mask && dataset_checksum(R) == dataset_checksum(M));
    std::remove("dropin_io.csv");
    CHECK_THROWS_CODE(load_matrix("no_such_file_anywhere.csv"), errc::parse_io);
  }
  std::printf("dropin: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
