// rsm_ctx.cu -- host orchestration of the B200 RSM hot path and the C-ABI
// declared in include/rsm_b200.h.
//
// Mirrors the reference pipeline (paths relative to /root/reference/proj):
//   decompose            solver.cpp:119-146  validation, m<n transpose, e
//   decompose_oriented   solver.cpp:93-115
//   trial_params         harvest.cpp:11-35
//   harvest_gram         harvest.cpp:79-120  -> stages 1-3 (k_select/k_svd/k_gram)
//   solve_v              solver.cpp:15-62    -> stage 4 (k_eig) + rank gate here
//   solve_u              solver.cpp:64-89    -> stage 5 (k_solve_u)
// Errors are rsm::errc codes (error.hpp:8-46). CUDA/NCCL failures map to
// internal. No CPU fallback exists: every numeric stage runs on the device.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rsm_b200.h"
#include "rsm_internal.h"
#include "rsm_dev.cuh"
#include "host_rng.h"

namespace {

struct RsmError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw RsmError{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(RSM_ERR_INTERNAL, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// bumped whenever any device buffer moves: a captured decompose graph holds
// raw buffer addresses and is replayed only while this is unchanged
std::atomic<uint64_t> g_buf_epoch{0};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t need) {
    if (need <= bytes) return;
    ++g_buf_epoch;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    need = std::max<size_t>(need, 256);
    ck(cudaMalloc(&p, need), "cudaMalloc");
    bytes = need;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) {
      ++g_buf_epoch;
      cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
  }
};

// decompose's device work as one CUDA graph (decompose_impl): the key is
// everything the host-side enqueue reads; the rest is the host state the
// captured call left behind, restored on every replay
struct DecompGraph {
  cudaGraphExec_t exec = nullptr;
  bool keyed = false, broken = false;
  int64_t rank = 0, block = 0, vpt = 0, min_dim = 0;
  int32_t mode = 0;
  uint64_t trials = 0, seed = 0, load_gen = 0, epoch = 0;
  double tol = 0.0, spec_rate = 0.0;
  int64_t qhint = 0;
  // captured outcome
  uint64_t attempted = 0, accepted = 0, z = 0;
  int rex = 0, eig_b = 0, eig_grid = 0;
  int64_t launches = 0, spec_Lcap = 0;
  void drop() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    keyed = false;
  }
};

// ---- NCCL, loaded at run time only when world > 1 ----
typedef struct { char internal[128]; } NcclId;
typedef void* NcclComm;
struct Nccl {
  void* h = nullptr;
  int (*getUniqueId)(NcclId*) = nullptr;
  int (*commInitRank)(NcclComm*, int, NcclId, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
  int (*commDestroy)(NcclComm) = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    getUniqueId = (int (*)(NcclId*))dlsym(h, "ncclGetUniqueId");
    commInitRank = (int (*)(NcclComm*, int, NcclId, int))dlsym(h, "ncclCommInitRank");
    allReduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllReduce");
    allGather = (int (*)(const void*, void*, size_t, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllGather");
    commDestroy = (int (*)(NcclComm))dlsym(h, "ncclCommDestroy");
    return getUniqueId && commInitRank && allReduce && allGather && commDestroy;
  }
};
Nccl g_nccl;
constexpr int kNcclInt32 = 2, kNcclFloat64 = 8, kNcclSum = 0;

struct View {
  const double* Y;
  const uint32_t* bitsR;
  const uint32_t* bitsC;
  int64_t m, n, nwp, mwp;
};

struct SelResult {
  uint64_t attempted = 0, accepted = 0;
  int qmax = 0;
  uint64_t qsum = 0;  // sum of the accepted trials' survivor counts
  bool spec = false;  // speculative: one chunk enqueued, outcome read after the caller's sync
};

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace

// In-process rank group whose collectives exchange through host memory: the
// multi-rank code path (trial shards, accumulator all-reduce, row shards and
// the U all-gather) runs with several contexts on one GPU, one host thread
// per rank. Test and diagnostic use only; N GPUs use NCCL.
struct rsm_host_group {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<std::vector<char>> buf;  // per-rank staging
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct rsm_ctx {
  int device = 0;
  int world = 1, rank = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  NcclComm comm = nullptr;
  rsm_host_group* hg = nullptr;  // host-exchange collectives instead of NCCL
  bool coll = false;  // collectives on (world > 1, or forced for a one-rank check)
  std::string err;

  // the loaded matrix as given
  bool loaded = false;
  uint64_t load_gen = 0;  // bumped by every load (decompose graph key)
  DecompGraph dgraph;
  int64_t m = 0, n = 0;
  unsigned long long known = 0;
  DevBuf Y, M8, bitsR, bitsC;
  bool haveC = false;
  bool haveM8 = false;          // byte mask on the device (else rebuilt from bitsR on demand)
  uint32_t* hstage = nullptr;   // pinned host staging for the packed mask
  size_t hstage_bytes = 0;
  int64_t last_h2d = 0;         // bytes copied host -> device by the last load
  // its transpose, built on demand for decompose when m < n
  DevBuf Yt, M8t, bitsRt, bitsCt;
  bool haveT = false, haveCt = false;

  // workspace
  DevBuf sel_idx, sel_q, blockcnt, selstate, t_attempt, t_q, t_idx, t_cm, Vtrial,
      colcnt, svd_scr, svd_scr32, P, tiles, G, eX, eY, eZ, ePart, eW, eI, eD, Vhat, U, rowres,
      flagged, dsum, cnt64, Wq, tiles8, ugather;
  DevBuf Apre, Bq;  // stage 5's tensor-core normal matrices and the basis-product digits
  DevBuf aux0, aux1, aux2, aux3;  // per-call utilities (rsm_sample, rsm_small_singular_vectors, rsm_gram_update)
  double* hsmall = nullptr;  // pinned host staging: eig stats [0,96), stage-5 scalars [96,100),
                             // speculative selection state [104,109)
  double spec_rate = 1.0;    // acceptance rate seen by the last full selection (sizes the speculative chunk)
  int64_t spec_Lcap = 0;     // support bound of the last speculative stage-2 launch
  int64_t spec_qhint = 0;    // largest support a failed speculation saw on this matrix
  int64_t spec_reruns = 0;   // decompositions re-run after a failed speculation (tests read it)
  int64_t tiles_n = -1;
  int64_t tiles8_n = -1;  // tcgen05 stage-3 tile list valid for this npad
  int ntiles8 = 0;
  int tiles_cpl = 0;
  int64_t G_n = 0;      // accumulator on device valid for this n
  bool G_harvest = false;  // G = diag(colcnt) - PSD (from our harvest, single rank)
  int64_t Vhat_n = 0, Vhat_r = 0;
  bool oriented_T = false;  // last decompose ran on the transpose
  int64_t U_m = 0, U_r = 0;

  cudaEvent_t ev[8] = {};
  double stage_ms[8] = {};
  double solver_stats[32] = {};  // eig: outer its, matvecs, lambda_max, ub, max residual, block, grid
  int64_t launches = 0;
  // held by the one-shot calls (rsm_decompose, rsm_solve_u, ...) from the load
  // through the last device->host copy: those share one context per device, and
  // the reference's functions are reentrant (SPEC concurrency model)
  std::mutex oneshot;

  void set_err(const std::string& s) { err = s; }
};

namespace {

thread_local std::string g_err;

void record(rsm_ctx* c, int i) {
  // inside a decompose graph capture the stage events become event-record
  // nodes (External), so every replay re-records them
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  ck(cudaStreamIsCapturing(c->stream, &st), "cudaStreamIsCapturing");
  if (st == cudaStreamCaptureStatusActive)
    ck(cudaEventRecordWithFlags(c->ev[i], c->stream, cudaEventRecordExternal), "cudaEventRecord");
  else
    ck(cudaEventRecord(c->ev[i], c->stream), "cudaEventRecord");
}

// ---------------------------------------------------------------- collectives
// Sum over ranks in place (FP64 or int32 elements): NCCL on the context
// stream, or the host group (every rank adds the staged buffers in rank order,
// so all ranks hold bitwise identical sums).
template <class T>
void coll_allreduce_sum(rsm_ctx* c, T* dev, size_t count) {
  static_assert(sizeof(T) == 8 || sizeof(T) == 4, "f64 or i32");
  if (!c->hg) {
    if (g_nccl.allReduce(dev, dev, count, sizeof(T) == 8 ? kNcclFloat64 : kNcclInt32, kNcclSum, c->comm,
                         c->stream) != 0)
      fail(RSM_ERR_INTERNAL, "ncclAllReduce failed");
    return;
  }
  rsm_host_group* g = c->hg;
  const size_t bytes = sizeof(T) * count;
  std::vector<char>& mine = g->buf[c->rank];
  mine.resize(bytes);
  ck(cudaMemcpyAsync(mine.data(), dev, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H allreduce");
  ck(cudaStreamSynchronize(c->stream), "sync");
  g->barrier();
  std::vector<T> sum(count, T(0));
  for (int r = 0; r < g->world; ++r) {
    const T* x = reinterpret_cast<const T*>(g->buf[r].data());
    for (size_t i = 0; i < count; ++i) sum[i] += x[i];
  }
  g->barrier();  // every rank has read every buffer
  ck(cudaMemcpyAsync(dev, sum.data(), bytes, cudaMemcpyHostToDevice, c->stream), "H2D allreduce");
  ck(cudaStreamSynchronize(c->stream), "sync");
}

// recv[r * count .. (r+1) * count) = rank r's send (rank order)
void coll_allgather(rsm_ctx* c, const double* send, double* recv, size_t count) {
  if (!c->hg) {
    if (g_nccl.allGather(send, recv, count, kNcclFloat64, c->comm, c->stream) != 0)
      fail(RSM_ERR_INTERNAL, "ncclAllGather failed");
    return;
  }
  rsm_host_group* g = c->hg;
  const size_t bytes = sizeof(double) * count;
  std::vector<char>& mine = g->buf[c->rank];
  mine.resize(bytes);
  ck(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H allgather");
  ck(cudaStreamSynchronize(c->stream), "sync");
  g->barrier();
  for (int r = 0; r < g->world; ++r)
    ck(cudaMemcpyAsync(recv + (size_t)r * count, g->buf[r].data(), bytes, cudaMemcpyHostToDevice, c->stream),
       "H2D allgather");
  ck(cudaStreamSynchronize(c->stream), "sync");
  g->barrier();
}

// ---------------------------------------------------------------- layout
// the byte mask, rebuilt from the packed rows when the host delivered words
void ensure_m8(rsm_ctx* c) {
  if (c->haveM8) return;
  c->M8.ensure((size_t)c->m * c->n);
  rsmk::launch_unpack_rows(c->bitsR.as<uint32_t>(), c->m, c->n, ceil_div(c->n, 128) * 4, c->M8.as<uint8_t>(),
                           c->stream);
  ++c->launches;
  c->haveM8 = true;
}

View make_view(rsm_ctx* c, bool transposed, bool needC) {
  if (!c->loaded) fail(RSM_ERR_INVALID_CONFIG, "no matrix loaded");
  View v{};
  if (!transposed) {
    v.m = c->m;
    v.n = c->n;
    v.nwp = ceil_div(c->n, 128) * 4;
    v.mwp = ceil_div(c->m, 32);
    if (needC && !c->haveC) {
      ensure_m8(c);
      c->bitsC.ensure(sizeof(uint32_t) * v.n * v.mwp);
      rsmk::launch_pack_cols(c->M8.as<uint8_t>(), v.m, v.n, c->bitsC.as<uint32_t>(), v.mwp, c->stream);
      ++c->launches;
      c->haveC = true;
    }
    v.Y = c->Y.as<double>();
    v.bitsR = c->bitsR.as<uint32_t>();
    v.bitsC = c->haveC ? c->bitsC.as<uint32_t>() : nullptr;
  } else {
    v.m = c->n;
    v.n = c->m;
    v.nwp = ceil_div(v.n, 128) * 4;
    v.mwp = ceil_div(v.m, 32);
    if (!c->haveT) {
      ensure_m8(c);
      c->Yt.ensure(sizeof(double) * c->m * c->n + 16);  // stage 5 may read 8 bytes past the end
      c->M8t.ensure((size_t)c->m * c->n);
      rsmk::launch_transpose(c->Y.as<double>(), c->M8.as<uint8_t>(), c->m, c->n, c->Yt.as<double>(),
                             c->M8t.as<uint8_t>(), c->stream);
      c->bitsRt.ensure(sizeof(uint32_t) * v.m * v.nwp);
      rsmk::launch_pack_rows(c->M8t.as<uint8_t>(), v.m, v.n, c->bitsRt.as<uint32_t>(), v.nwp, c->stream);
      c->launches += 2;
      c->haveT = true;
    }
    if (needC && !c->haveCt) {
      c->bitsCt.ensure(sizeof(uint32_t) * v.n * v.mwp);
      rsmk::launch_pack_cols(c->M8t.as<uint8_t>(), v.m, v.n, c->bitsCt.as<uint32_t>(), v.mwp, c->stream);
      ++c->launches;
      c->haveCt = true;
    }
    v.Y = c->Yt.as<double>();
    v.bitsR = c->bitsRt.as<uint32_t>();
    v.bitsC = c->haveCt ? c->bitsCt.as<uint32_t>() : nullptr;
  }
  return v;
}

// row words of the byte mask on the host (bit j%32 of word j/32, nonzero =
// observed, zero padded to nwp words), split over host threads; 8 bytes at a
// time: OR-fold every byte into its low bit, then gather the 8 bits
void pack_rows_host(const uint8_t* mask, int64_t m, int64_t n, int64_t nwp, uint32_t* out) {
  auto work = [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      const uint8_t* row = mask + i * n;
      uint32_t* o = out + i * nwp;
      int64_t w = 0;
      for (; (w + 1) * 32 <= n; ++w) {
        uint32_t word = 0;
        for (int q = 0; q < 4; ++q) {
          uint64_t x;
          std::memcpy(&x, row + w * 32 + q * 8, 8);
          uint64_t t = x | (x >> 4);
          t |= t >> 2;
          t |= t >> 1;
          t &= 0x0101010101010101ull;
          word |= (uint32_t)((t * 0x0102040810204080ull) >> 56) << (8 * q);
        }
        o[w] = word;
      }
      if (w * 32 < n) {
        uint32_t word = 0;
        for (int64_t j = w * 32; j < n; ++j) word |= (row[j] ? 1u : 0u) << (j - w * 32);
        o[w++] = word;
      }
      for (; w < nwp; ++w) o[w] = 0u;
    }
  };
  const int64_t bytes = m * n;
  int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), 16);
  if (bytes < ((int64_t)8 << 20)) nt = 1;
  nt = (int)std::min<int64_t>(nt, m);
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, m * t / nt, m * (t + 1) / nt);
  work(0, m / nt);
  for (auto& x : th) x.join();
}

void load_common(rsm_ctx* c, int64_t m, int64_t n, bool packed_on_host) {
  c->m = m;
  c->n = n;
  c->haveC = c->haveT = c->haveCt = false;
  const int64_t nwp = ceil_div(n, 128) * 4;
  c->bitsR.ensure(sizeof(uint32_t) * m * nwp);
  if (!packed_on_host) {
    rsmk::launch_pack_rows(c->M8.as<uint8_t>(), m, n, c->bitsR.as<uint32_t>(), nwp, c->stream);
    ++c->launches;
  }
  c->haveM8 = !packed_on_host;
  c->cnt64.ensure(sizeof(unsigned long long));
  ck(cudaMemsetAsync(c->cnt64.p, 0, sizeof(unsigned long long), c->stream), "memset");
  rsmk::launch_count_bits(c->bitsR.as<uint32_t>(), m * nwp, c->cnt64.as<unsigned long long>(), c->stream);
  c->launches += 1;
  ck(cudaMemcpyAsync(&c->known, c->cnt64.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  ck(cudaGetLastError(), "load kernels");
  c->loaded = true;
  ++c->load_gen;
  c->spec_qhint = 0;
  c->spec_rate = 1.0;
}

// ------------------------------------------------------------- trial params
rsm_trial_params trial_params_impl(const rsm_config* cfg, int64_t m, int64_t n) {
  // harvest.cpp:11-35
  if (cfg->rank < 1) fail(RSM_ERR_INVALID_CONFIG, "rank must be positive");
  if (cfg->rank >= std::min(m, n)) fail(RSM_ERR_INVALID_CONFIG, "rank must be below min(rows, cols)");
  rsm_trial_params p{};
  p.mode = cfg->mode;
  p.rank = cfg->rank;
  p.seed = cfg->seed;
  p.block = cfg->block > 0 ? cfg->block : cfg->rank + 1;
  if (p.block <= cfg->rank) fail(RSM_ERR_INVALID_CONFIG, "block must exceed rank");
  const int64_t pool = cfg->mode == RSM_MODE_M1 ? n : m;
  if (p.block > pool) fail(RSM_ERR_INVALID_CONFIG, "block exceeds matrix dimension");
  p.min_count = cfg->min_dim > 0 ? cfg->min_dim : cfg->rank + 1;
  if (p.min_count < cfg->rank + 1) fail(RSM_ERR_INVALID_CONFIG, "min_dim must be at least rank+1");
  if (cfg->mode == RSM_MODE_M1) {
    p.ell = cfg->vectors_per_trial > 0 ? cfg->vectors_per_trial : p.block - cfg->rank;
    if (p.ell > p.block - cfg->rank) fail(RSM_ERR_INVALID_CONFIG, "vectors_per_trial exceeds block-rank");
  } else {
    p.ell = cfg->vectors_per_trial;
  }
  return p;
}

void check_device_params(const rsm_trial_params* p, const View& v) {
  if (p->mode != RSM_MODE_M1 && p->mode != RSM_MODE_M2) fail(RSM_ERR_INVALID_CONFIG, "unknown mode");
  if (p->block < 1) fail(RSM_ERR_INVALID_CONFIG, "block must be positive");
  const int64_t pool = p->mode == RSM_MODE_M1 ? v.n : v.m;
  if (p->block > pool) fail(RSM_ERR_INVALID_CONFIG, p->mode == RSM_MODE_M1 ? "sample_m1: column count out of range" : "sample_m2: row count out of range");
  if (p->block > rsmd::KMAX) fail(RSM_ERR_INVALID_CONFIG, "device path supports block <= 16 rows/columns per trial");
  if (v.m > INT32_MAX || v.n > INT32_MAX) fail(RSM_ERR_INVALID_CONFIG, "dimension exceeds 2^31-1");
}

// ------------------------------------------------------------------ stage 1
double* pinned_small(rsm_ctx* c);

// spec = true: enqueue one chunk sized from the last observed acceptance rate
// and return without synchronising, as if it accepted all T trials; the
// selection state goes to pinned memory and decompose checks it after its one
// synchronisation (spec_selection_ok)
SelResult select_impl(rsm_ctx* c, const View& v, const rsm_trial_params* p, uint64_t T, bool spec = false) {
  if (T < 1) fail(RSM_ERR_INVALID_CONFIG, "trial count must be positive");
  check_device_params(p, v);
  const bool m2 = p->mode == RSM_MODE_M2;
  const int block = (int)p->block;
  const uint64_t budget = 20 * T;  // harvest.cpp:85
  c->t_attempt.ensure(sizeof(uint64_t) * T);
  c->t_q.ensure(sizeof(int32_t) * T);
  c->t_idx.ensure(sizeof(int32_t) * T * block);
  c->selstate.ensure(sizeof(rsmk::SelState));
  ck(cudaMemsetAsync(c->selstate.p, 0, sizeof(rsmk::SelState), c->stream), "memset");
  const uint32_t* bits = m2 ? v.bitsR : v.bitsC;
  const int64_t stride = m2 ? v.nwp : v.mwp;
  const int64_t nwords = m2 ? ceil_div(v.n, 32) : ceil_div(v.m, 32);
  const int64_t pool = m2 ? v.m : v.n;
  SelResult r;
  uint64_t attempted = 0, acc = 0;
  double p_est = spec ? std::min(1.0, std::max(1e-3, c->spec_rate)) : 1.0;
  rsmk::SelState hs{};
  while (acc < T && attempted < budget) {
    const uint64_t want = T - acc;
    uint64_t chunk = (uint64_t)std::ceil((double)want * 1.1 / p_est) + 256;
    chunk = std::max<uint64_t>(chunk, 4096);
    chunk = std::min<uint64_t>(chunk, 1ull << 22);
    chunk = std::min<uint64_t>(chunk, budget - attempted);
    c->sel_idx.ensure(sizeof(int32_t) * chunk * block);
    c->sel_q.ensure(sizeof(int32_t) * chunk);
    c->blockcnt.ensure(sizeof(int32_t) * (chunk / 1024 + 2));
    rsmk::launch_select(bits, stride, nwords, pool, block, p->seed, attempted, (int64_t)chunk,
                        c->sel_idx.as<int32_t>(), c->sel_q.as<int32_t>(), c->stream);
    rsmk::launch_accept(c->sel_q.as<int32_t>(), c->sel_idx.as<int32_t>(), (int64_t)chunk,
                        (int32_t)p->min_count, block, attempted, c->blockcnt.as<int32_t>(),
                        c->selstate.as<rsmk::SelState>(), T, c->t_attempt.as<uint64_t>(),
                        c->t_q.as<int32_t>(), c->t_idx.as<int32_t>(), c->stream);
    c->launches += 4;
    if (spec) {
      static_assert(sizeof(rsmk::SelState) <= 5 * sizeof(double), "pinned slot");
      ck(cudaMemcpyAsync(pinned_small(c) + 104, c->selstate.p, sizeof(rsmk::SelState), cudaMemcpyDeviceToHost,
                         c->stream), "D2H");
      r.attempted = chunk;
      r.accepted = T;
      r.spec = true;
      return r;
    }
    ck(cudaMemcpyAsync(&hs, c->selstate.p, sizeof(hs), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "select");
    ck(cudaGetLastError(), "select kernels");
    if (hs.attempted_done) {
      attempted = hs.attempted_done;
      acc = T;
      break;
    }
    p_est = std::max(1e-3, (double)(hs.acc - acc) / (double)chunk);
    acc = hs.acc;
    attempted += chunk;
  }
  r.attempted = attempted;
  r.accepted = acc;
  r.qmax = hs.qmax;
  r.qsum = hs.qsum;
  if (attempted) c->spec_rate = (double)acc / (double)attempted;
  return r;
}

// after the stream sync: did the speculative chunk accept all T trials, with
// every support within the bound the speculative stage-2 launch assumed? The
// state is the same on every rank (the selection is replicated), so all ranks
// take the same branch.
bool spec_selection_ok(rsm_ctx* c, SelResult* r) {
  rsmk::SelState hs;
  std::memcpy(&hs, c->hsmall + 104, sizeof(hs));
  if (!hs.attempted_done) {
    c->spec_rate = std::max(1e-3, (double)hs.acc / (double)std::max<uint64_t>(r->attempted, 1));
    return false;
  }
  if ((int64_t)hs.qmax > c->spec_Lcap) {
    c->spec_qhint = hs.qmax;
    return false;
  }
  r->attempted = hs.attempted_done;
  r->qmax = hs.qmax;
  r->qsum = hs.qsum;
  r->spec = false;
  return true;
}

// ------------------------------------------------------------ stages 2 + 3
struct HarvestOut {
  SelResult sel;
  uint64_t z = 0;
  int rex = 0;  // top vectors per trial
};

// support-length bound for a speculative stage-2 launch: K random rows (row
// branch) or columns (column branch) under the loaded density keep a
// binomial number of survivors; mean + 5 sd (a miss costs a re-run, about
// T * 3e-7 per call for an i.i.d. mask; a wider bound costs the warp kernel
// occupancy on every call), raised to what the warp kernel's
// occupancy allows for free, and to the largest support a failed speculation
// on this matrix saw
int64_t spec_lcap(rsm_ctx* c, const View& v, bool m2, int K, int64_t cmw) {
  const double pool = m2 ? (double)v.n : (double)v.m;
  const double dens = (double)c->known / ((double)v.m * (double)v.n);
  const double pk = std::pow(dens, K);
  const double mean = pool * pk, sd = std::sqrt(pool * pk * (1.0 - pk));
  int64_t L = (int64_t)std::ceil(mean + 5.0 * sd + 8.0);
  L = std::max<int64_t>(L, c->spec_qhint);
  L = std::min<int64_t>(L, (int64_t)pool);
  if (m2) L = rsmk::svd_warp_lcap(K, L, cmw);
  if (const char* e = getenv("RSM_SPEC_LCAP")) L = std::max<int64_t>(2, atoll(e));  // tests: force the fallback
  return L;
}

void build_tiles(rsm_ctx* c, int64_t npad, int cpl) {
  if (c->tiles_n == npad && c->tiles_cpl == cpl) return;
  const int64_t TR = 64, TC = 32 * cpl;
  std::vector<int2> t;
  for (int64_t J = 0; J < npad / TC; ++J)
    for (int64_t I = 0; I < npad / TR; ++I)
      if (TC * J + TC - 1 >= TR * I) t.push_back(make_int2((int)I, (int)J));
  c->tiles.ensure(sizeof(int2) * t.size());
  ck(cudaMemcpy(c->tiles.p, t.data(), sizeof(int2) * t.size(), cudaMemcpyHostToDevice), "H2D tiles");
  c->tiles_n = npad;
  c->tiles_cpl = cpl;
}

void build_tiles8(rsm_ctx* c, int64_t npad) {
  if (c->tiles8_n == npad) return;
  std::vector<int2> t;
  rsmk::gram_i8_tiles(npad, t);
  c->tiles8.ensure(sizeof(int2) * t.size());
  ck(cudaMemcpy(c->tiles8.p, t.data(), sizeof(int2) * t.size(), cudaMemcpyHostToDevice), "H2D tiles");
  c->tiles8_n = npad;
  c->ntiles8 = (int)t.size();
}

// stage 3 on the tensor cores (k_gram_i8.cu) unless RSM_GRAM=dfma selects the
// FP64 register-tile kernel (k_gram.cu), kept as the exact-FP64 comparison
bool gram_on_tensor_cores() {
  const char* e = getenv("RSM_GRAM");
  return !(e && std::string(e) == "dfma");
}

int64_t ntiles_for(int64_t npad, int cpl) {
  const int64_t TR = 64, TC = 32 * cpl;
  int64_t k = 0;
  for (int64_t J = 0; J < npad / TC; ++J)
    for (int64_t I = 0; I < npad / TR; ++I)
      if (TC * J + TC - 1 >= TR * I) ++k;
  return k;
}

HarvestOut harvest_impl(rsm_ctx* c, const View& v, const rsm_trial_params* p, uint64_t T, bool spec = false) {
  HarvestOut out;
  const bool m2 = p->mode == RSM_MODE_M2;
  record(c, 0);
  out.sel = select_impl(c, v, p, T, spec);
  record(c, 1);
  const int64_t Tacc = (int64_t)out.sel.accepted;
  const int64_t n = v.n;
  const int64_t npad = ceil_div(n, 128) * 128;
  const int64_t cmw = npad / 32;
  const int K = (int)p->block;
  // per-trial ell / top-vector count (harvest.cpp:44-50); the selection's
  // state already carries the survivor-count sum and maximum, so no per-trial
  // counts come back to the host
  int rex;
  if (m2) {
    rex = (int)p->rank;
    if (!out.sel.spec && p->ell > 0 && Tacc > 0 && p->ell < (int64_t)out.sel.qmax - p->rank)
      fail(RSM_ERR_INVALID_CONFIG,
           "row-branch vectors_per_trial below survivors-rank harvests an implementation-defined "
           "null-space basis; the device path supports the adaptive default");
  } else {
    rex = (int)(p->block - p->ell);
  }
  if (rex < 1 || rex > 16) fail(RSM_ERR_INVALID_CONFIG, "device path supports 1 <= block-vectors <= 16 top vectors");
  out.rex = rex;
  // local trial range (trials shard over ranks, no communication needed)
  int64_t t_lo, t_hi;
  rsm_shard_range(Tacc, c->world, c->rank, &t_lo, &t_hi);
  const int64_t Tl = t_hi - t_lo;
  uint64_t z = 0;
  z = m2 ? out.sel.qsum - (uint64_t)Tacc * (uint64_t)rex : (uint64_t)Tacc * (uint64_t)p->ell;
  out.z = z;
  c->G.ensure(sizeof(double) * n * n);
  c->colcnt.ensure(sizeof(int) * npad);
  ck(cudaMemsetAsync(c->colcnt.p, 0, sizeof(int) * npad, c->stream), "memset");
  // stage 2 hands stage 3 each trial's top vectors zero outside the support:
  // as int8 digit slices (rows t*rex + p of S x Kpad x npad, k_gram_i8.cu)
  // for the tensor-core path, or expanded FP64 planes (rp/2 planes of npad
  // pairs) for the FP64 kernel. Trials go through stages 2-3 in chunks whose
  // hand-off buffer fits the budget; stage 3 accumulates across chunks.
  const bool i8 = gram_on_tensor_cores();
  const int S8 = rsmk::gram_i8_slices();
  const int64_t rp = (rex + 1) & ~1;
  const int64_t tbytes = i8 ? (int64_t)S8 * rex * npad : npad * rp * (int64_t)sizeof(double);
  // RSM_CHUNK_BYTES overrides the budget (tests exercise the multi-chunk path)
  const int64_t budget = [] {
    const char* e = getenv("RSM_CHUNK_BYTES");
    return e ? std::max<int64_t>(1, atoll(e)) : ((int64_t)12 << 30);
  }();
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(Tl, budget / tbytes));
  const int cpl = rsmk::gram_cols_per_lane(rex);
  int64_t ntiles = 0;
  if (i8) {
    build_tiles8(c, npad);
    ntiles = c->ntiles8;
  } else {
    build_tiles(c, npad, cpl);
    ntiles = ntiles_for(npad, cpl);
  }
  // tensor-core path: K = trials * rex rows of int8 slices per trial chunk,
  // split into nk K-chunks (P slices) so the work units fill the SMs and each
  // chunk's int32 sums stay exact (k_gram_i8.cu)
  const int64_t Kpad0 = ceil_div(std::max<int64_t>(chunk, 1) * rex, 32) * 32;
  int nk = 1;
  if (i8) {
    int64_t k = std::max(ceil_div(Kpad0, rsmk::gram_i8_kmax()), ceil_div(c->sms, ntiles));
    k = std::min<int64_t>(k, std::max<int64_t>(ceil_div(Kpad0, rsmk::gram_i8_kmax()), Kpad0 / 512));
    nk = (int)std::max<int64_t>(1, k);
    if (const char* e = getenv("RSM_I8_NK")) nk = (int)std::max<int64_t>(ceil_div(Kpad0, rsmk::gram_i8_kmax()), atoll(e));
  }
  int nslices = 1;
  if (Tl > 0) {
    if (i8) {
      nslices = nk;
    } else {
      // at most one wave of the 2-CTA/SM kernel: floor(2*SMs / tiles) slices
      nslices = (int)std::max<int64_t>(1, ((int64_t)rsmk::gram_ctas_per_sm(rex) * c->sms) / ntiles);
      nslices = (int)std::min<int64_t>(nslices, std::max<int64_t>(1, chunk / 16));
    }
    c->P.ensure(sizeof(double) * (size_t)nslices * npad * npad);
    c->t_cm.ensure(sizeof(uint32_t) * chunk * cmw);
    if (i8) c->Wq.ensure((size_t)S8 * Kpad0 * npad);
    else c->Vtrial.ensure((size_t)tbytes * chunk);
    // the largest survivor count over all accepted trials; a speculative
    // launch does not know it yet and sizes for a bound instead (spec_lcap)
    const int64_t Lmax = out.sel.spec ? spec_lcap(c, v, m2, K, cmw) : out.sel.qmax;
    const int64_t Lpad = std::max<int64_t>(2, (Lmax + 1) & ~int64_t(1));
    c->spec_Lcap = Lpad;
    const size_t fixed = rsmk::svd_smem_fixed(cmw, m2);
    const size_t vecb = sizeof(double) * (size_t)K * Lpad;
    static const int col_smem = [] {
      const char* e = getenv("RSM_SVD_COL_SMEM");
      return e ? atoi(e) : 0;
    }();
    const bool use_smem = fixed + vecb <= 200 * 1024 && (m2 || col_smem);
    const size_t smem = fixed + (use_smem ? vecb : 0);
    int occ = rsmk::svd_occupancy(m2, smem);
    if (occ < 1) occ = 1;
    for (int64_t c0 = t_lo; c0 < t_hi; c0 += chunk) {
      const int64_t c1 = std::min<int64_t>(t_hi, c0 + chunk);
      // stage 2
      const int64_t grid = std::min<int64_t>(c1 - c0, (int64_t)c->sms * occ);
      rsmk::SvdArgs a{};
      a.Y = v.Y; a.m = v.m; a.n = v.n;
      a.bitsR = v.bitsR; a.nwp = v.nwp;
      a.bitsC = v.bitsC; a.mwp = v.mwp;
      a.t_idx = c->t_idx.as<int32_t>();
      a.t_lo = c0; a.t_hi = c1;
      a.block = K; a.rex = rex;
      a.t_cm = c->t_cm.as<uint32_t>(); a.cmw = cmw; a.npad = npad;
      const int64_t Kpad = ceil_div((c1 - c0) * rex, 32) * 32;
      if (i8) {
        a.Wq = c->Wq.as<int8_t>();
        a.Kpad = Kpad;
        a.S = S8;
        // rows past the chunk's trials * rex are zero (read by the last K-step)
        const int64_t used = (c1 - c0) * rex;
        if (Kpad > used)
          for (int sl = 0; sl < S8; ++sl)
            ck(cudaMemsetAsync(a.Wq + ((int64_t)sl * Kpad + used) * npad, 0, (size_t)(Kpad - used) * npad,
                               c->stream), "memset");
      } else {
        a.Vout = c->Vtrial.as<double>();
      }
      a.colcnt = c->colcnt.as<int>();
      if (!use_smem) {
        c->svd_scr.ensure(vecb * grid);
        a.scratch = c->svd_scr.as<double>();
      }
      if (!m2) {
        c->svd_scr32.ensure(sizeof(uint32_t) * 2 * v.mwp * grid);
        a.scratch_u32 = c->svd_scr32.as<uint32_t>();
      }
      a.Lpad = Lpad;
      a.Lcap = out.sel.spec ? Lpad : INT64_MAX;
      a.sel_acc = out.sel.spec ? &c->selstate.as<rsmk::SelState>()->acc : nullptr;
      a.use_smem = use_smem ? 1 : 0;
      static const int svd_maxit = [] {
        const char* e = getenv("RSM_SVD_MAXIT");
        return e ? atoi(e) : 6;
      }();
      a.max_outer = svd_maxit;
      static const int fast_basis = [] {
        const char* e = getenv("RSM_SVD_FAST_BASIS");
        return e ? atoi(e) : 1;
      }();
      a.fast_basis = fast_basis;
      // row branch with k <= 9: warp-per-trial kernel; otherwise CTA per trial
      if (!(m2 && rsmk::launch_svd_warp(a, c->sms, c->stream))) rsmk::launch_svd(a, m2, (int)grid, smem, c->stream);
      ++c->launches;
      ck(cudaGetLastError(), "svd launch");
      if (c0 == t_lo) record(c, 2);  // with several chunks, later stage-2 work counts as stage 3
      // stage 3
      if (i8) {
        rsmk::GramI8Args g{};
        g.W = c->Wq.as<int8_t>();
        g.npad = npad;
        g.Kpad = Kpad;
        g.nk = nk;
        g.Kc = ceil_div(ceil_div(Kpad, nk), 32) * 32;
        g.ntiles = (int)ntiles;
        g.tiles = c->tiles8.as<int2>();
        g.P = c->P.as<double>();
        g.accumulate = c0 > t_lo ? 1 : 0;
        const char* dg = getenv("RSM_I8_DIAG");
        g.diag = dg ? atoi(dg) : 0;
        g.S = S8;
        ck(rsmk::launch_gram_i8(g, c->sms, c->stream), "gram (tcgen05) launch");
        ++c->launches;
      } else {
        rsmk::GramArgs g{};
        g.t_cm = c->t_cm.as<uint32_t>();
        g.V = c->Vtrial.as<double>();
        g.T = c1 - c0; g.cmw = cmw; g.npad = npad; g.R = rex; g.nslices = nslices;
        g.accumulate = c0 > t_lo ? 1 : 0;
        g.tiles = c->tiles.as<int2>();
        g.P = c->P.as<double>();
        rsmk::launch_gram(g, (int)ntiles, c->stream);
        ++c->launches;
        ck(cudaGetLastError(), "gram launch");
      }
    }
  } else {
    record(c, 2);
    c->P.ensure(sizeof(double) * npad * npad);
    ck(cudaMemsetAsync(c->P.p, 0, sizeof(double) * npad * npad, c->stream), "memset");
  }
  record(c, 3);
  rsmk::launch_gram_reduce(c->P.as<double>(), nslices, npad, n, c->colcnt.as<int>(), c->G.as<double>(), c->stream);
  ++c->launches;
  if (c->coll) {
    // the one exchange of stages 1-3: partial accumulators (each with its
    // shard's column counts on the diagonal) and the counts themselves, for
    // the zero-row certificate of stage 4 (harvest.cpp:110-117 merges the
    // per-worker Grams the same way)
    coll_allreduce_sum(c, c->G.as<double>(), (size_t)(n * n));
    coll_allreduce_sum(c, c->colcnt.as<int>(), (size_t)npad);
  }
  record(c, 4);
  ck(cudaGetLastError(), "gram reduce");
  c->G_n = n;
  c->G_harvest = true;  // G = diag(colcnt) - PSD with the global column counts
  return out;
}

// ------------------------------------------------------------------ stage 4
struct SolveVOut {
  int64_t gram_rank = 0;
  int borderline = 0;
  std::vector<double> w;
};

double* pinned_small(rsm_ctx* c) {
  if (!c->hsmall) ck(cudaMallocHost(&c->hsmall, sizeof(double) * 128), "cudaMallocHost");
  return c->hsmall;
}

struct EigLaunch {
  int b = 0, grid = 0;
};

// stage 4 enqueued: zero-row count, the cooperative eigensolver, the sign
// fix, and the solver's status/Ritz values copied to pinned host memory --
// no host synchronisation (solve_v_finish reads them after the caller's sync)
EigLaunch solve_v_launch(rsm_ctx* c, int64_t n, int64_t r, double tol) {
  // solver.cpp:15-62
  if (n < 1) fail(RSM_ERR_INVALID_CONFIG, "solve_v: empty accumulator");
  if (r < 1 || r >= n) fail(RSM_ERR_INVALID_CONFIG, "solve_v: need 1 <= r < n");
  if (!(tol > 0.0)) fail(RSM_ERR_INVALID_CONFIG, "solve_v: tolerance must be positive");
  if (c->G_n != n) fail(RSM_ERR_INVALID_CONFIG, "solve_v: no accumulator of this size on the device");
  int b;
  if (n <= 16) b = (int)n;
  else {
    if (r > 14) fail(RSM_ERR_INVALID_CONFIG, "device eigensolver supports r <= 14 for n > 16");
    b = (int)std::min<int64_t>(16, std::max<int64_t>(r + 5, 2 * r + 2));
  }
  const int ld = b + 1;
  const int maxgrid = rsmk::eig_max_grid();
  static const int rows_min = [] {
    const char* e = getenv("RSM_EIG_ROWS");  // rows per CTA (experiments)
    return e ? std::max(1, atoi(e)) : 8;
  }();
  int grid = (int)std::min<int64_t>(maxgrid, std::max<int64_t>(1, ceil_div(n, rows_min)));
  const int rows_per_cta = (int)ceil_div(n, grid);
  grid = (int)ceil_div(n, rows_per_cta);
  const int pw = rsmk::eig_part_width(b);
  // + 32 doubles: the matvec reads a fixed 12/17 columns per row, running
  // past the last row by up to 16 (those products are discarded)
  c->eX.ensure(sizeof(double) * (n * ld + 32));
  c->eY.ensure(sizeof(double) * (n * ld + 32));
  c->eZ.ensure(sizeof(double) * (n * ld + 32));
  c->ePart.ensure(sizeof(double) * 2 * (size_t)grid * pw);
  c->eW.ensure(sizeof(double) * 32);
  c->eI.ensure(sizeof(int) * 8);
  c->eD.ensure(sizeof(double) * 32);
  c->Vhat.ensure(sizeof(double) * n * r);
  rsmk::EigArgs a{};
  a.G = c->G.as<double>();
  a.n = n; a.r = (int)r; a.b = b; a.tol = tol;
  a.rows_per_cta = rows_per_cta; a.rpw = 2;
  a.X = c->eX.as<double>(); a.Y = c->eY.as<double>(); a.Z = c->eZ.as<double>();
  a.part = c->ePart.as<double>();
  a.V = c->Vhat.as<double>();
  a.w = c->eW.as<double>();
  a.istat = c->eI.as<int>();
  a.dstat = c->eD.as<double>();
  a.max_outer = 60;
  static const double amp = [] {
    const char* e = getenv("RSM_EIG_AMP");
    return e ? atof(e) : 1e10;
  }();
  a.amp = amp;
  static const int dmax = [] {
    const char* e = getenv("RSM_EIG_DMAX");
    return e ? atoi(e) : 40;
  }();
  a.dmax = dmax;
  static const int rr0_probe = [] {
    const char* e = getenv("RSM_EIG_PROBE");
    return e ? atoi(e) : 1;
  }();
  a.rr0_probe = rr0_probe;
  static const int init_cq = [] {
    const char* e = getenv("RSM_EIG_INITCQ");
    return e ? atoi(e) : 0;
  }();
  a.init_cq = init_cq;
  static const double shift0 = [] {
    const char* e = getenv("RSM_EIG_SHIFT0");
    return e ? atof(e) : 1e-14;
  }();
  a.shift0 = shift0;
  static const int probe_its = [] {
    const char* e = getenv("RSM_EIG_PROBE_ITS");
    return e ? std::max(1, atoi(e)) : 16;
  }();
  a.probe_its = probe_its;
  a.cnt = c->G_harvest ? c->colcnt.as<int>() : nullptr;
  a.zero_rows = c->eI.as<int>() + 7;
  rsmk::launch_zero_rows(a.G, n, a.cnt, c->eI.as<int>() + 7, c->stream);
  ++c->launches;
  a.hout = pinned_small(c);  // the kernel writes its scalars to pinned host memory itself
  ck(rsmk::launch_eig(a, grid, c->stream), "cooperative eig launch");  // sign fix included
  c->launches += 1;
  EigLaunch L;
  L.b = b;
  L.grid = grid;
  return L;
}

// after the stream has been synchronised: solver statistics, the rank gate
// and borderline flag (solver.cpp:32-60), errors raised as the reference's
SolveVOut solve_v_finish(rsm_ctx* c, const EigLaunch& L, int64_t n, int64_t r, double tol) {
  ck(cudaGetLastError(), "eig kernels");
  const int b = L.b, grid = L.grid;
  const double* hs = c->hsmall;
  double w[32], dstat[32];
  int istat[8];
  std::memcpy(w, hs, sizeof(double) * b);
  std::memcpy(dstat, hs + 32, sizeof(double) * 32);
  std::memcpy(istat, hs + 64, sizeof(int) * 8);
  c->solver_stats[0] = istat[3];
  c->solver_stats[1] = istat[4];
  c->solver_stats[2] = dstat[0];
  c->solver_stats[3] = dstat[1];
  c->solver_stats[4] = dstat[2];
  c->solver_stats[5] = b;
  c->solver_stats[6] = grid;
  for (int i = 0; i < 6; ++i) c->solver_stats[7 + i] = dstat[3 + i];  // phase clocks (cycles)
  c->solver_stats[13] = dstat[9];   // Rayleigh-Ritz Jacobi sweeps (total)
  c->solver_stats[14] = dstat[10];  // and their cycles
  c->solver_stats[15] = dstat[11];  // filter matvec cycles (CTA 0)
  for (int i = 0; i < 16; ++i) c->solver_stats[16 + i] = dstat[16 + i];  // CholQR sub-phases, tail, counters
  if (istat[0] == 3)  // certified: more than r eigenvalues at or below tol * lambda_max
    fail(RSM_ERR_INSUFFICIENT_COVERAGE,
         "rank gate failed: constraint coverage below n-r; raise the trial count or epsilon");
  if (istat[0] != 0) fail(RSM_ERR_INTERNAL, "symmetric eigensolver failed to converge");
  c->Vhat_n = n;
  c->Vhat_r = r;
  const double lambda_max = std::max(dstat[0], 0.0);
  const double threshold = tol * lambda_max;
  SolveVOut o;
  o.w.assign(w, w + b);
  int64_t significant;
  if (b == n) {
    significant = 0;
    for (int i = 0; i < b; ++i)
      if (w[i] > threshold) ++significant;
  } else {
    int64_t small = 0;
    for (int i = 0; i <= r; ++i)
      if (!(w[i] > threshold)) ++small;
    significant = n - small;
  }
  if (significant < n - r)
    fail(RSM_ERR_INSUFFICIENT_COVERAGE, "rank gate failed: constraint coverage below n-r; raise the trial count or epsilon");
  o.gram_rank = significant;
  o.borderline = !(w[r] > 10.0 * threshold);
  return o;
}

SolveVOut solve_v_impl(rsm_ctx* c, int64_t n, int64_t r, double tol) {
  const EigLaunch L = solve_v_launch(c, n, r, tol);
  ck(cudaStreamSynchronize(c->stream), "solve_v");
  return solve_v_finish(c, L, n, r, tol);
}

// ------------------------------------------------------------------ stage 5
struct SolveUOut {
  int64_t flagged = 0;
  double ss = 0.0;
};

// stage 5 on view v: rows of `out` (v.m x r) from the basis (v.n x r), plus
// the residual sum and the flagged-row count; row-sharded over ranks with
// the shards gathered into `out` (detail/row_solve.hpp:12-36, solver.cpp:64-89)
SolveUOut solve_rows(rsm_ctx* c, const View& v, const double* basis, DevBuf& outbuf, int64_t r,
                     const double* ugiven = nullptr, bool defer = false, bool unit_basis = false) {
  if (r < 1) fail(RSM_ERR_INVALID_CONFIG, "solve_u: rank must be positive");
  if (r > 8) fail(RSM_ERR_INVALID_CONFIG, "device row solver supports r <= 8");
  outbuf.ensure(sizeof(double) * v.m * r);
  double* out = outbuf.as<double>();
  c->rowres.ensure(sizeof(double) * v.m);
  c->flagged.ensure(sizeof(int) * 2);
  c->dsum.ensure(sizeof(double) * (2 + 64));  // + partials of launch_sum_rows
  ck(cudaMemsetAsync(c->flagged.p, 0, sizeof(int) * 2, c->stream), "memset");
  int64_t lo, hi;
  rsm_shard_range(v.m, c->world, c->rank, &lo, &hi);
  rsmk::SolveUArgs a{};
  a.Y = v.Y; a.bitsR = v.bitsR;
  a.m = v.m; a.n = v.n; a.nwp = v.nwp;
  a.row_lo = lo; a.row_hi = hi;
  a.V = basis;
  a.U = out;
  a.rowres = c->rowres.as<double>();
  a.flagged = c->flagged.as<int>();
  a.r = (int)r;
  a.Ugiven = ugiven;
  // the rows' normal matrices on the tensor cores (k_normal_i8.cu) unless
  // RSM_NORMAL_TC=0; the row kernels then only form V_O^T y and the residual.
  // Only for a basis with entries in [-1, 1] (decompose's orthonormal V-hat:
  // the digit split of v_i v_j assumes |v_i v_j| <= 1); ALS and caller-given
  // bases take the FP64 normal-matrix path.
  static const bool normal_tc = [] {
    const char* e = getenv("RSM_NORMAL_TC");
    return !(e && atoi(e) == 0);
  }();
  // (from ~8k rows on: below that the extra launches cost more than they save)
  if (normal_tc && unit_basis && hi > lo && v.n >= 32 && v.m >= 8192) {
    const int na = (int)(r * (r + 1) / 2);
    c->Apre.ensure(sizeof(double) * v.m * na);
    c->Bq.ensure(rsmk::normal_i8_bq_bytes((int)r, v.n));
    rsmk::NormalI8Args na8{};
    na8.bits = v.bitsR; na8.m = v.m; na8.n = v.n; na8.nwp = v.nwp;
    na8.V = basis; na8.r = (int)r;
    na8.Bq = c->Bq.as<int8_t>();
    na8.Apre = c->Apre.as<double>();
    ck(rsmk::launch_normal_i8(na8, c->sms, c->stream), "normal matrices (tcgen05) launch");
    c->launches += 2;
    a.Apre = c->Apre.as<double>();
  }
  if (hi > lo) {
    rsmk::launch_solve_u(a, c->stream);
    // flagged[1] (zeroed above) is the sum kernel's arrival counter
    c->launches += 1 + rsmk::launch_sum_rows(c->rowres.as<double>() + lo, hi - lo, c->dsum.as<double>(), c->stream,
                                             reinterpret_cast<unsigned*>(c->flagged.as<int>() + 1));
  } else {
    ck(cudaMemsetAsync(c->dsum.p, 0, sizeof(double), c->stream), "memset");
  }
  double ss = 0.0;
  int fl = 0;
  if (c->coll) {
    // row shards: sum the scalars on the device, gather U through a padded
    // buffer (row blocks differ in size when world does not divide m)
    coll_allreduce_sum(c, c->dsum.as<double>(), 1);
    coll_allreduce_sum(c, c->flagged.as<int>(), 1);
    const int64_t maxrows = ceil_div(v.m, c->world);
    c->ugather.ensure(sizeof(double) * maxrows * r * (c->world + 1));
    double* pad = c->ugather.as<double>();
    double* sendb = pad + (size_t)maxrows * r * c->world;
    if (hi > lo)
      ck(cudaMemcpyAsync(sendb, out + lo * r, sizeof(double) * (hi - lo) * r, cudaMemcpyDeviceToDevice, c->stream),
         "D2D");
    coll_allgather(c, sendb, pad, (size_t)(maxrows * r));
    for (int g = 0; g < c->world; ++g) {
      int64_t glo, ghi;
      rsm_shard_range(v.m, c->world, g, &glo, &ghi);
      if (ghi > glo)
        ck(cudaMemcpyAsync(out + glo * r, pad + (size_t)g * maxrows * r, sizeof(double) * (ghi - glo) * r,
                           cudaMemcpyDeviceToDevice, c->stream), "D2D");
    }
  }
  SolveUOut o;
  if (defer) {
    // scalars to pinned host memory; the caller synchronises and reads them
    // with deferred_rows()
    double* hs = pinned_small(c);
    ck(cudaMemcpyAsync(hs + 96, c->dsum.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaMemcpyAsync(hs + 97, c->flagged.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
    return o;
  }
  ck(cudaMemcpyAsync(&ss, c->dsum.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaMemcpyAsync(&fl, c->flagged.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "solve_u");
  ck(cudaGetLastError(), "solve_u kernels");
  o.flagged = fl;
  o.ss = ss;
  return o;
}

// the stage-5 scalars of a deferred solve_rows, after the stream sync
SolveUOut deferred_rows(rsm_ctx* c) {
  ck(cudaGetLastError(), "solve_u kernels");
  SolveUOut o;
  o.ss = c->hsmall[96];
  int fl = 0;
  std::memcpy(&fl, c->hsmall + 97, sizeof(int));
  o.flagged = fl;
  return o;
}

SolveUOut solve_u_impl(rsm_ctx* c, const View& v, int64_t r) {
  if (c->Vhat_n != v.n || c->Vhat_r != r) fail(RSM_ERR_INVALID_CONFIG, "solve_u: basis shape does not match matrix");
  SolveUOut o = solve_rows(c, v, c->Vhat.as<double>(), c->U, r);
  c->U_m = v.m;
  c->U_r = r;
  return o;
}

// ---------------------------------------------------------------- decompose
void decompose_impl(rsm_ctx* c, const rsm_config* cfg, double* Uout, double* Vout, rsm_report* rep) {
  const auto t0 = std::chrono::steady_clock::now();
  c->launches = 0;
  std::memset(rep, 0, sizeof(*rep));
  if (!c->loaded) fail(RSM_ERR_INVALID_CONFIG, "no matrix loaded");
  const int64_t m = c->m, n = c->n;
  // solver.cpp:122-127
  if (cfg->rank < 1 || cfg->rank >= std::min(m, n)) fail(RSM_ERR_INVALID_CONFIG, "rank must lie in [1, min(rows, cols))");
  if (!(cfg->epsilon > 0.0 && cfg->epsilon < 1.0)) fail(RSM_ERR_INVALID_CONFIG, "epsilon must lie in (0,1)");
  if (cfg->trials < 1) fail(RSM_ERR_INVALID_CONFIG, "trial plan must request at least one trial");
  if (c->known == 0) fail(RSM_ERR_INSUFFICIENT_COVERAGE, "matrix has no observed entries");
  const bool tr = m < n;  // solver.cpp:130-140
  const View v = make_view(c, tr, cfg->mode == RSM_MODE_M1);
  const rsm_trial_params p = trial_params_impl(cfg, v.m, v.n);
  // The whole decomposition is enqueued before the host looks at anything:
  // the selection runs speculatively (one chunk, stage 2 sized for a support
  // bound), stages 4 and 5 follow back to back (stage 5 needs only V-hat, on
  // the device), and the host synchronises once. It then reads the selection
  // state, the eigensolver's status and the rank gate; if the chunk did not
  // reach T acceptances or a support outgrew the bound (both rare and
  // replicated on every rank), the decomposition is re-run with the
  // synchronous selection. A failed gate discards the stage-5 results and
  // raises as the reference does. RSM_SPEC=0 runs the synchronous selection.
  static const bool spec_on = [] {
    const char* e = getenv("RSM_SPEC");
    return !(e && atoi(e) == 0);
  }();
  const int64_t r = cfg->rank;
  // oriented U is (v.m x r), oriented V is (v.n x r); the transpose swaps them
  double* hostU = tr ? Vout : Uout;
  double* hostV = tr ? Uout : Vout;
  HarvestOut h;
  EigLaunch L;
  auto enqueue = [&](bool spec) {
    h = harvest_impl(c, v, &p, cfg->trials, spec);
    L = solve_v_launch(c, v.n, r, cfg->gram_rank_tol);
    record(c, 5);
    c->Vhat_n = 0;
    c->U_m = 0;
    solve_rows(c, v, c->Vhat.as<double>(), c->U, r, nullptr, /*defer=*/true, /*unit_basis=*/true);
    record(c, 6);
  };
  auto fetch_and_sync = [&] {
    if (hostU) ck(cudaMemcpyAsync(hostU, c->U.p, sizeof(double) * v.m * r, cudaMemcpyDeviceToHost, c->stream), "D2H U");
    if (hostV) ck(cudaMemcpyAsync(hostV, c->Vhat.p, sizeof(double) * v.n * r, cudaMemcpyDeviceToHost, c->stream), "D2H V");
    ck(cudaStreamSynchronize(c->stream), "decompose");
  };
  // With the speculative selection the enqueue never waits on the device, so
  // it is captured once as a CUDA graph and replayed: the first call with a
  // key runs eagerly (and allocates), the second captures, later calls only
  // launch the graph (single rank; RSM_GRAPH=0 disables).
  static const bool graph_env = [] {
    const char* e = getenv("RSM_GRAPH");
    return !(e && atoi(e) == 0);
  }();
  DecompGraph& g = c->dgraph;
  const bool graph_on = spec_on && graph_env && !c->coll && !g.broken;
  bool done = false;
  if (graph_on) {
    const bool same = g.keyed && g.rank == cfg->rank && g.mode == cfg->mode && g.block == cfg->block &&
                      g.vpt == cfg->vectors_per_trial && g.trials == cfg->trials && g.seed == cfg->seed &&
                      g.tol == cfg->gram_rank_tol && g.min_dim == cfg->min_dim && g.load_gen == c->load_gen &&
                      g.epoch == g_buf_epoch.load() && g.spec_rate == c->spec_rate && g.qhint == c->spec_qhint;
    if (same && g.exec) {
      ck(cudaGraphLaunch(g.exec, c->stream), "decompose graph launch");
      h.sel.attempted = g.attempted;
      h.sel.accepted = g.accepted;
      h.sel.spec = true;
      h.z = g.z;
      h.rex = g.rex;
      L.b = g.eig_b;
      L.grid = g.eig_grid;
      c->launches += g.launches;
      c->spec_Lcap = g.spec_Lcap;
      c->G_n = v.n;
      c->G_harvest = true;
      fetch_and_sync();
      done = true;
    } else if (same) {
      const uint64_t e0 = g_buf_epoch.load();
      const int64_t l0 = c->launches;
      cudaGraph_t gr = nullptr;
      ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed), "begin capture");
      bool captured = true;
      try {
        enqueue(true);
      } catch (...) {
        captured = false;
      }
      const cudaError_t ce = cudaStreamEndCapture(c->stream, &gr);
      cudaGetLastError();
      cudaGraphExec_t ex = nullptr;
      if (captured && ce == cudaSuccess && gr && g_buf_epoch.load() == e0 &&
          cudaGraphInstantiate(&ex, gr, 0) == cudaSuccess) {
        g.exec = ex;
        g.attempted = h.sel.attempted;
        g.accepted = h.sel.accepted;
        g.z = h.z;
        g.rex = h.rex;
        g.eig_b = L.b;
        g.eig_grid = L.grid;
        g.launches = c->launches - l0;
        g.spec_Lcap = c->spec_Lcap;
        ck(cudaGraphLaunch(g.exec, c->stream), "decompose graph launch");
        fetch_and_sync();
        done = true;
      } else {
        cudaGetLastError();
        g.broken = true;  // this context runs eagerly from now on
        c->launches = l0;
      }
      if (gr) cudaGraphDestroy(gr);
    } else {
      g.drop();
    }
  }
  if (!done) {
    enqueue(spec_on);  // eager (first call with this key, a failed capture, or no graph)
    fetch_and_sync();
    if (graph_on && !g.keyed) {
      g.keyed = true;
      g.rank = cfg->rank; g.mode = cfg->mode; g.block = cfg->block; g.vpt = cfg->vectors_per_trial;
      g.trials = cfg->trials; g.seed = cfg->seed; g.tol = cfg->gram_rank_tol; g.min_dim = cfg->min_dim;
      g.load_gen = c->load_gen;
      g.spec_rate = c->spec_rate;
      g.qhint = c->spec_qhint;
    }
  }
  if (graph_on && g.keyed) g.epoch = g_buf_epoch.load();
  // the speculation's outcome: a miss re-runs with the synchronous selection
  if (h.sel.spec) {
    if (spec_selection_ok(c, &h.sel)) {
      // the harvest's host-side checks that needed the selection outcome
      if (p.mode == RSM_MODE_M2) {
        if (p.ell > 0 && p.ell < (int64_t)h.sel.qmax - p.rank)
          fail(RSM_ERR_INVALID_CONFIG,
               "row-branch vectors_per_trial below survivors-rank harvests an implementation-defined "
               "null-space basis; the device path supports the adaptive default");
        h.z = h.sel.qsum - h.sel.accepted * (uint64_t)h.rex;
      }
    } else {
      ++c->spec_reruns;
      enqueue(false);
      fetch_and_sync();
    }
  }
  rep->trials_attempted = h.sel.attempted;
  rep->trials_accepted = h.sel.accepted;
  rep->z = h.z;
  const SolveVOut sv = solve_v_finish(c, L, v.n, r, cfg->gram_rank_tol);
  rep->gram_rank = sv.gram_rank;
  rep->borderline_rank_gate = sv.borderline;
  const SolveUOut su = deferred_rows(c);
  c->U_m = v.m;
  c->U_r = r;
  rep->underdetermined_rows = su.flagged;
  rep->e = std::sqrt(su.ss) / std::sqrt((double)c->known);  // core.cpp:35-39
  c->oriented_T = tr;
  float ms = 0.f;
  for (int i = 0; i < 6; ++i) {
    ck(cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]), "event");
    c->stage_ms[i] = ms;
  }
  ck(cudaEventElapsedTime(&ms, c->ev[0], c->ev[6]), "event");
  c->stage_ms[6] = ms;
  rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ------------------------------------------------------------------- ALS
// baseline_als (als.cpp:11-44): V from Rng(seed, ALS_INIT, column).next_normal
// on the host, then `iterations` rounds of U = rows(M; V), V = rows(M^T; U),
// and a final U = rows(M; V) whose fused residual gives e; every half-step is
// the stage-5 kernel, on the loaded matrix and on its device transpose.
void als_impl(rsm_ctx* c, int64_t r, int64_t iterations, uint64_t seed, double* Uout, double* Vout,
              rsm_report* rep) {
  const auto t0 = std::chrono::steady_clock::now();
  c->launches = 0;
  std::memset(rep, 0, sizeof(*rep));
  if (!c->loaded) fail(RSM_ERR_INVALID_CONFIG, "no matrix loaded");
  const int64_t m = c->m, n = c->n;
  if (r < 1 || r >= std::min(m, n)) fail(RSM_ERR_INVALID_CONFIG, "rank must lie in [1, min(rows, cols))");
  if (iterations < 1) fail(RSM_ERR_INVALID_CONFIG, "iteration count must be positive");
  if (c->known == 0) fail(RSM_ERR_INSUFFICIENT_COVERAGE, "matrix has no observed entries");
  std::vector<double> v0((size_t)(n * r));
  for (int64_t i = 0; i < n; ++i) {
    rsmh::Rng rng(seed, rsmh::stream::ALS_INIT, (uint64_t)i);
    for (int64_t k = 0; k < r; ++k) v0[(size_t)(i * r + k)] = rng.next_normal();
  }
  const View vm = make_view(c, false, false);
  const View vt = make_view(c, true, false);
  c->Vhat.ensure(sizeof(double) * n * r);
  ck(cudaMemcpyAsync(c->Vhat.p, v0.data(), sizeof(double) * n * r, cudaMemcpyHostToDevice, c->stream), "H2D V0");
  SolveUOut us;
  for (int64_t it = 0; it < iterations; ++it) {
    us = solve_rows(c, vm, c->Vhat.as<double>(), c->U, r);
    solve_rows(c, vt, c->U.as<double>(), c->Vhat, r);
  }
  us = solve_rows(c, vm, c->Vhat.as<double>(), c->U, r);
  if (m < n) {
    // masked_residual_norm evaluates wide matrices on the transpose (as
    // decompose does); take e the same way so the two agree bit for bit
    const double ss_rows = us.ss;
    us.ss = solve_rows(c, vt, c->U.as<double>(), c->aux1, r, c->Vhat.as<double>()).ss;
    (void)ss_rows;
  }
  c->Vhat_n = n;
  c->Vhat_r = r;
  c->U_m = m;
  c->U_r = r;
  c->oriented_T = false;
  rep->underdetermined_rows = us.flagged;
  rep->e = std::sqrt(us.ss) / std::sqrt((double)c->known);  // masked_residual_norm, core.cpp:35-39
  if (Uout) ck(cudaMemcpyAsync(Uout, c->U.p, sizeof(double) * m * r, cudaMemcpyDeviceToHost, c->stream), "D2H U");
  if (Vout) ck(cudaMemcpyAsync(Vout, c->Vhat.p, sizeof(double) * n * r, cudaMemcpyDeviceToHost, c->stream), "D2H V");
  ck(cudaStreamSynchronize(c->stream), "als");
  rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ------------------------------------------------------------ default ctx
std::mutex g_mu;
std::map<int, rsm_ctx*> g_default;

rsm_ctx* default_ctx() {
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_default.find(dev);
  if (it != g_default.end()) return it->second;
  rsm_ctx* c = nullptr;
  if (rsm_ctx_create(&c, dev, 1, 0, nullptr) != RSM_OK) fail(RSM_ERR_INTERNAL, std::string("context creation failed: ") + g_err);
  g_default[dev] = c;
  return c;
}

template <class F>
rsm_status guard(rsm_ctx* c, F&& f) {
  try {
    if (c) {
      ck(cudaSetDevice(c->device), "cudaSetDevice");
      c->err.clear();
    }
    f();
    return RSM_OK;
  } catch (const RsmError& e) {
    if (c) c->err = e.msg;
    g_err = e.msg;
    if (c && e.code == RSM_ERR_INTERNAL) cudaGetLastError();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    g_err = e.what();
    return RSM_ERR_INTERNAL;
  }
}

}  // namespace

// ======================================================================== C-ABI
extern "C" {

void rsm_shard_range(int64_t total, int world, int rank, int64_t* lo, int64_t* hi) {
  // contiguous, balanced, deterministic: rank g owns [total*g/world, total*(g+1)/world)
  *lo = total * rank / world;
  *hi = total * (rank + 1) / world;
}

void rsm_config_default(rsm_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->mode = RSM_MODE_M1;  // RsmConfig{} (solver.hpp:13-23)
  cfg->epsilon = 0.99;      // TrialPlan{} (planner.hpp:12-18)
  cfg->gram_rank_tol = 1e-9;
}

const char* rsm_last_error(const rsm_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

}  // extern "C"

namespace rsmk {
void set_host_error(const std::string& msg) { g_err = msg; }
}  // namespace rsmk

extern "C" {

rsm_status rsm_ctx_create(rsm_ctx** out, int device, int world, int rank, const void* nccl_id) {
  return guard(nullptr, [&] {
    if (!out) fail(RSM_ERR_INVALID_CONFIG, "null output pointer");
    if (world < 1 || rank < 0 || rank >= world) fail(RSM_ERR_INVALID_CONFIG, "bad world/rank");
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) fail(RSM_ERR_INVALID_CONFIG, "no such CUDA device");
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop{};
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10) fail(RSM_ERR_INTERNAL, "this build targets sm_100a (B200)");
    rsm_ctx* c = new rsm_ctx();
    c->device = device;
    c->world = world;
    c->rank = rank;
    c->sms = prop.multiProcessorCount;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    for (auto& e : c->ev) ck(cudaEventCreate(&e), "event");
    // RSM_FORCE_COLLECTIVES=1 with world == 1 and an id: a one-rank NCCL
    // communicator and the multi-rank code path (allreduce / allgather run as
    // identities), so the collectives are exercised on a single GPU
    const char* fc = getenv("RSM_FORCE_COLLECTIVES");
    const bool force = world == 1 && nccl_id && fc && atoi(fc) == 1;
    if (world > 1 || force) {
      if (!nccl_id) fail(RSM_ERR_INVALID_CONFIG, "world > 1 needs an NCCL unique id");
      if (!g_nccl.load()) fail(RSM_ERR_INTERNAL, "libnccl.so.2 not loadable");
      NcclId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      if (g_nccl.commInitRank(&c->comm, world, id, rank) != 0) fail(RSM_ERR_INTERNAL, "ncclCommInitRank failed");
      c->coll = true;
    }
    *out = c;
  });
}

rsm_status rsm_host_group_create(int world, rsm_host_group** out) {
  return guard(nullptr, [&] {
    if (!out) fail(RSM_ERR_INVALID_CONFIG, "null output pointer");
    if (world < 1) fail(RSM_ERR_INVALID_CONFIG, "bad world");
    rsm_host_group* g = new rsm_host_group();
    g->world = world;
    g->buf.resize(world);
    *out = g;
  });
}

rsm_status rsm_host_group_destroy(rsm_host_group* g) {
  delete g;
  return RSM_OK;
}

rsm_status rsm_ctx_create_host_group(rsm_ctx** out, int device, rsm_host_group* g, int rank) {
  if (!g) return guard(nullptr, [&] { fail(RSM_ERR_INVALID_CONFIG, "null host group"); });
  rsm_status st = rsm_ctx_create(out, device, 1, 0, nullptr);
  if (st) return st;
  return guard(*out, [&] {
    if (rank < 0 || rank >= g->world) fail(RSM_ERR_INVALID_CONFIG, "bad world/rank");
    (*out)->world = g->world;
    (*out)->rank = rank;
    (*out)->hg = g;
    (*out)->coll = true;
  });
}

rsm_status rsm_ctx_destroy(rsm_ctx* c) {
  if (!c) return RSM_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  DevBuf* bufs[] = {&c->Y, &c->M8, &c->bitsR, &c->bitsC, &c->Yt, &c->M8t, &c->bitsRt, &c->bitsCt,
                    &c->sel_idx, &c->sel_q, &c->blockcnt, &c->selstate, &c->t_attempt, &c->t_q,
                    &c->t_idx, &c->t_cm, &c->Vtrial, &c->colcnt, &c->svd_scr,
                    &c->svd_scr32, &c->P, &c->tiles, &c->G, &c->eX, &c->eY, &c->eZ, &c->ePart,
                    &c->eW, &c->eI, &c->eD, &c->Vhat, &c->U, &c->rowres, &c->flagged, &c->dsum,
                    &c->cnt64, &c->Wq, &c->tiles8, &c->ugather, &c->aux0, &c->aux1, &c->aux2, &c->aux3,
                    &c->Apre, &c->Bq};
  c->dgraph.drop();
  for (DevBuf* b : bufs) b->release();
  if (c->hstage) cudaFreeHost(c->hstage);
  if (c->hsmall) cudaFreeHost(c->hsmall);
  for (auto& e : c->ev) cudaEventDestroy(e);
  if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  cudaStreamDestroy(c->stream);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_default.begin(); it != g_default.end(); ++it)
      if (it->second == c) { g_default.erase(it); break; }
  }
  delete c;
  return RSM_OK;
}

rsm_status rsm_nccl_unique_id(void* out128) {
  return guard(nullptr, [&] {
    if (!g_nccl.load()) fail(RSM_ERR_INTERNAL, "libnccl.so.2 not loadable");
    NcclId id;
    if (g_nccl.getUniqueId(&id) != 0) fail(RSM_ERR_INTERNAL, "ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof(id));
  });
}

void* rsm_ctx_stream(rsm_ctx* c) { return c ? (void*)c->stream : nullptr; }

rsm_status rsm_ctx_load(rsm_ctx* c, const double* values, const uint8_t* mask, int64_t m, int64_t n) {
  return guard(c, [&] {
    if (m < 1 || n < 1) fail(RSM_ERR_INVALID_CONFIG, "matrix dimensions must be positive");
    if (!values || !mask) fail(RSM_ERR_INVALID_CONFIG, "null matrix buffers");
    // the values stream to the device while host threads bit-pack the mask
    // into pinned staging; only the packed words (1/8 of the byte mask) cross
    // the link after them
    c->Y.ensure(sizeof(double) * m * n + 16);  // stage 5 may read 8 bytes past the end
    ck(cudaMemcpyAsync(c->Y.p, values, sizeof(double) * m * n, cudaMemcpyHostToDevice, c->stream), "H2D Y");
    const int64_t nwp = ceil_div(n, 128) * 4;
    const size_t wbytes = sizeof(uint32_t) * (size_t)m * nwp;
    if (c->hstage_bytes < wbytes) {
      if (c->hstage) cudaFreeHost(c->hstage);
      c->hstage = nullptr;
      c->hstage_bytes = 0;
      ck(cudaHostAlloc((void**)&c->hstage, wbytes, cudaHostAllocDefault), "pinned staging");
      c->hstage_bytes = wbytes;
    }
    // (the previous load's copy out of the staging buffer completed: every
    // load ends with a stream synchronisation)
    pack_rows_host(mask, m, n, nwp, c->hstage);
    c->bitsR.ensure(wbytes);
    ck(cudaMemcpyAsync(c->bitsR.p, c->hstage, wbytes, cudaMemcpyHostToDevice, c->stream), "H2D mask words");
    c->last_h2d = (int64_t)(sizeof(double) * m * n + wbytes);
    load_common(c, m, n, true);
  });
}

rsm_status rsm_ctx_load_device(rsm_ctx* c, const double* d_values, const uint8_t* d_mask, int64_t m, int64_t n) {
  return guard(c, [&] {
    if (m < 1 || n < 1) fail(RSM_ERR_INVALID_CONFIG, "matrix dimensions must be positive");
    c->Y.ensure(sizeof(double) * m * n + 16);  // stage 5 may read 8 bytes past the end
    c->M8.ensure((size_t)m * n);
    ck(cudaMemcpyAsync(c->Y.p, d_values, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, c->stream), "D2D Y");
    ck(cudaMemcpyAsync(c->M8.p, d_mask, (size_t)m * n, cudaMemcpyDeviceToDevice, c->stream), "D2D mask");
    c->last_h2d = 0;
    load_common(c, m, n, false);
  });
}

rsm_status rsm_ctx_generate(rsm_ctx* c, int64_t m, int64_t n, int64_t r, double rho, double sigma, uint64_t seed) {
  return guard(c, [&] {
    if (m < 1 || n < 1 || r < 1 || r > 32) fail(RSM_ERR_INVALID_CONFIG, "generate: need m, n >= 1 and 1 <= r <= 32");
    if (!(rho > 0.0 && rho <= 1.0) || !(sigma >= 0.0)) fail(RSM_ERR_INVALID_CONFIG, "generate: need 0 < rho <= 1, sigma >= 0");
    const int64_t nwp = ceil_div(n, 128) * 4;
    c->Y.ensure(sizeof(double) * m * n + 16);  // stage 5 may read 8 bytes past the end
    c->bitsR.ensure(sizeof(uint32_t) * m * nwp);
    DevBuf B;
    B.ensure(sizeof(double) * r * n);
    rsmk::launch_generate(m, n, r, rho, sigma, seed, B.as<double>(), nwp, c->Y.as<double>(), c->bitsR.as<uint32_t>(),
                          c->sms, c->stream);
    c->launches += 2;
    ck(cudaGetLastError(), "generate kernels");
    c->last_h2d = 0;
    load_common(c, m, n, true);
    B.release();
  });
}

rsm_status rsm_ctx_fetch_matrix(rsm_ctx* c, double* values, uint32_t* words, int64_t* nwp_out) {
  return guard(c, [&] {
    if (!c->loaded) fail(RSM_ERR_INVALID_CONFIG, "no matrix loaded");
    const int64_t nwp = ceil_div(c->n, 128) * 4;
    if (nwp_out) *nwp_out = nwp;
    if (values)
      ck(cudaMemcpyAsync(values, c->Y.p, sizeof(double) * c->m * c->n, cudaMemcpyDeviceToHost, c->stream), "D2H Y");
    if (words)
      ck(cudaMemcpyAsync(words, c->bitsR.p, sizeof(uint32_t) * c->m * nwp, cudaMemcpyDeviceToHost, c->stream),
         "D2H mask words");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

rsm_status rsm_ctx_decompose(rsm_ctx* c, const rsm_config* cfg, double* U, double* V, rsm_report* rep) {
  return guard(c, [&] { decompose_impl(c, cfg, U, V, rep); });
}

rsm_status rsm_ctx_fetch_factors(rsm_ctx* c, double* U, double* V) {
  return guard(c, [&] {
    if (c->U_m == 0) fail(RSM_ERR_INVALID_CONFIG, "no factors on the device");
    const int64_t r = c->U_r;
    const int64_t om = c->U_m, on = c->Vhat_n;
    double* hostU = c->oriented_T ? V : U;
    double* hostV = c->oriented_T ? U : V;
    if (hostU) ck(cudaMemcpyAsync(hostU, c->U.p, sizeof(double) * om * r, cudaMemcpyDeviceToHost, c->stream), "D2H");
    if (hostV) ck(cudaMemcpyAsync(hostV, c->Vhat.p, sizeof(double) * on * r, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "fetch");
  });
}

rsm_status rsm_ctx_select(rsm_ctx* c, const rsm_trial_params* p, uint64_t trials, uint64_t* accepted_attempts,
                          int64_t* survivors, uint64_t* attempted, uint64_t* accepted) {
  return guard(c, [&] {
    const View v = make_view(c, false, p->mode == RSM_MODE_M1);
    SelResult s = select_impl(c, v, p, trials);
    if (accepted_attempts && s.accepted)
      ck(cudaMemcpyAsync(accepted_attempts, c->t_attempt.p, sizeof(uint64_t) * s.accepted, cudaMemcpyDeviceToHost, c->stream), "D2H");
    if (survivors && s.accepted) {
      std::vector<int32_t> q(s.accepted);
      ck(cudaMemcpyAsync(q.data(), c->t_q.p, sizeof(int32_t) * s.accepted, cudaMemcpyDeviceToHost, c->stream), "D2H");
      ck(cudaStreamSynchronize(c->stream), "sync");
      for (uint64_t i = 0; i < s.accepted; ++i) survivors[i] = q[i];
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    *attempted = s.attempted;
    *accepted = s.accepted;
  });
}

rsm_status rsm_ctx_harvest_gram(rsm_ctx* c, const rsm_trial_params* p, uint64_t trials, double* G,
                                uint64_t* attempted, uint64_t* accepted, uint64_t* z) {
  return guard(c, [&] {
    const View v = make_view(c, false, p->mode == RSM_MODE_M1);
    if (p->rank < 1 || p->block <= p->rank) fail(RSM_ERR_INVALID_CONFIG, "block must exceed rank");
    if (p->min_count < p->rank + 1) fail(RSM_ERR_INVALID_CONFIG, "degenerate submatrix: needs more than r columns/rows");
    if (p->mode == RSM_MODE_M1 && (p->ell < 1 || p->ell > p->block - p->rank))
      fail(RSM_ERR_INVALID_CONFIG, "vector count must lie in [1, cols-r]");
    HarvestOut h = harvest_impl(c, v, p, trials);
    if (G) ck(cudaMemcpyAsync(G, c->G.p, sizeof(double) * v.n * v.n, cudaMemcpyDeviceToHost, c->stream), "D2H G");
    ck(cudaStreamSynchronize(c->stream), "sync");
    float ms = 0.f;  // stages 1-3 split (events 0..4), as decompose reports it
    for (int i = 0; i < 4; ++i) {
      ck(cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]), "event");
      c->stage_ms[i] = ms;
    }
    *attempted = h.sel.attempted;
    *accepted = h.sel.accepted;
    *z = h.z;
  });
}

rsm_status rsm_ctx_solve_v(rsm_ctx* c, const double* G, int64_t n, int64_t r, double tol, double* V,
                           int64_t* gram_rank, int32_t* borderline, double* w_small) {
  return guard(c, [&] {
    if (G) {
      if (n < 1) fail(RSM_ERR_INVALID_CONFIG, "solve_v: empty accumulator");
      c->G.ensure(sizeof(double) * n * n);
      ck(cudaMemcpyAsync(c->G.p, G, sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream), "H2D G");
      c->G_n = n;
      c->G_harvest = false;
    }
    SolveVOut o = solve_v_impl(c, n, r, tol);
    if (V) ck(cudaMemcpyAsync(V, c->Vhat.p, sizeof(double) * n * r, cudaMemcpyDeviceToHost, c->stream), "D2H V");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (w_small)
      for (int64_t i = 0; i <= r && i < (int64_t)o.w.size(); ++i) w_small[i] = o.w[i];
    *gram_rank = o.gram_rank;
    *borderline = o.borderline;
  });
}

rsm_status rsm_ctx_solve_u(rsm_ctx* c, const double* V, int64_t r, double* U, int64_t* underdetermined_rows,
                           double* sum_sq_resid) {
  return guard(c, [&] {
    const View v = make_view(c, false, false);
    if (r < 1) fail(RSM_ERR_INVALID_CONFIG, "solve_u: rank must be positive");
    if (V) {
      c->Vhat.ensure(sizeof(double) * v.n * r);
      ck(cudaMemcpyAsync(c->Vhat.p, V, sizeof(double) * v.n * r, cudaMemcpyHostToDevice, c->stream), "H2D V");
      c->Vhat_n = v.n;
      c->Vhat_r = r;
    }
    SolveUOut o = solve_u_impl(c, v, r);
    c->oriented_T = false;
    if (U) ck(cudaMemcpyAsync(U, c->U.p, sizeof(double) * v.m * r, cudaMemcpyDeviceToHost, c->stream), "D2H U");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (underdetermined_rows) *underdetermined_rows = o.flagged;
    if (sum_sq_resid) *sum_sq_resid = o.ss;
  });
}

int rsm_ctx_stage_ms(rsm_ctx* c, double* ms, int cap) {
  int k = std::min(cap, 7);
  for (int i = 0; i < k; ++i) ms[i] = c->stage_ms[i];
  return k;
}

int64_t rsm_ctx_launch_count(rsm_ctx* c) { return c ? c->launches : 0; }

int64_t rsm_ctx_rerun_count(rsm_ctx* c) { return c ? c->spec_reruns : 0; }

int64_t rsm_ctx_last_load_h2d_bytes(rsm_ctx* c) { return c ? c->last_h2d : 0; }

int rsm_ctx_solver_stats(rsm_ctx* c, double* out, int cap) {
  const int k = std::min(cap, 32);
  for (int i = 0; i < k; ++i) out[i] = c->solver_stats[i];
  return k;
}

// ---- one-shot, reference-shaped calls ----
rsm_status rsm_make_trial_params(const rsm_config* cfg, int64_t m, int64_t n, rsm_trial_params* out) {
  return guard(nullptr, [&] { *out = trial_params_impl(cfg, m, n); });
}

rsm_status rsm_ctx_als(rsm_ctx* c, int64_t r, int64_t iterations, uint64_t seed, double* U, double* V,
                       rsm_report* rep) {
  return guard(c, [&] { als_impl(c, r, iterations, seed, U, V, rep); });
}

rsm_status rsm_als(const double* values, const uint8_t* mask, int64_t m, int64_t n, int64_t r, int64_t iterations,
                   uint64_t seed, double* U, double* V, rsm_report* rep) {
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = rsm_ctx_load(c, values, mask, m, n);
  if (!st) st = rsm_ctx_als(c, r, iterations, seed, U, V, rep);
  if (st) g_err = c->err;
  return st;
}

rsm_status rsm_decompose(const double* values, const uint8_t* mask, int64_t m, int64_t n, const rsm_config* cfg,
                         double* U, double* V, rsm_report* rep) {
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = rsm_ctx_load(c, values, mask, m, n);
  if (st) { g_err = c->err; return st; }
  st = rsm_ctx_decompose(c, cfg, U, V, rep);
  if (st) g_err = c->err;
  return st;
}

rsm_status rsm_harvest_gram(const double* values, const uint8_t* mask, int64_t m, int64_t n,
                            const rsm_trial_params* p, uint64_t trials, double* G, uint64_t* attempted,
                            uint64_t* accepted, uint64_t* z) {
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = rsm_ctx_load(c, values, mask, m, n);
  if (!st) st = rsm_ctx_harvest_gram(c, p, trials, G, attempted, accepted, z);
  if (st) g_err = c->err;
  return st;
}

rsm_status rsm_solve_v(const double* G, int64_t n, int64_t r, double tol, double* V, int64_t* gram_rank,
                       int32_t* borderline) {
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = rsm_ctx_solve_v(c, G, n, r, tol, V, gram_rank, borderline, nullptr);
  if (st) g_err = c->err;
  return st;
}

rsm_status rsm_solve_u(const double* values, const uint8_t* mask, int64_t m, int64_t n, const double* V, int64_t r,
                       double* U, int64_t* underdetermined_rows) {
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = rsm_ctx_load(c, values, mask, m, n);
  if (!st) st = rsm_ctx_solve_u(c, V, r, U, underdetermined_rows, nullptr);
  if (st) g_err = c->err;
  return st;
}

// observed squared residual sum (core.cpp:15-31) of given factors on the
// default context: the per-row warp kernel and the fixed-order row sum
static rsm_status residual_ss(const double* values, const uint8_t* mask, int64_t m, int64_t n, const double* U,
                              const double* V, int64_t r, double* ss_out, int64_t* known) {
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = rsm_ctx_load(c, values, mask, m, n);
  if (st) { g_err = c->err; return st; }
  st = guard(c, [&] {
    if (r < 1 || r > 16) fail(RSM_ERR_INVALID_CONFIG, "residual: 1 <= r <= 16 on the device");
    if (r <= 8) {
      // the stage-5 kernel's residual pass with the rows' solutions given, on
      // the orientation decompose uses (the transpose when m < n): the same
      // arithmetic and summation order, so decompose's e and this agree bit
      // for bit (solver.cpp:142 computes e with masked_residual_norm itself)
      const bool tr = m < n;
      const View v = make_view(c, tr, false);
      c->Vhat.ensure(sizeof(double) * v.n * r);
      c->aux0.ensure(sizeof(double) * v.m * r);
      ck(cudaMemcpyAsync(c->Vhat.p, tr ? U : V, sizeof(double) * v.n * r, cudaMemcpyHostToDevice, c->stream), "H2D");
      ck(cudaMemcpyAsync(c->aux0.p, tr ? V : U, sizeof(double) * v.m * r, cudaMemcpyHostToDevice, c->stream), "H2D");
      c->U_m = 0;
      c->Vhat_n = 0;
      *ss_out = solve_rows(c, v, c->Vhat.as<double>(), c->aux1, r, c->aux0.as<double>()).ss;
      *known = c->known;
      return;
    }
    const View v = make_view(c, false, false);
    c->U.ensure(sizeof(double) * m * r);
    c->Vhat.ensure(sizeof(double) * n * r);
    c->rowres.ensure(sizeof(double) * m);
    c->dsum.ensure(sizeof(double) * (2 + 64));  // + partials of launch_sum_rows
    ck(cudaMemcpyAsync(c->U.p, U, sizeof(double) * m * r, cudaMemcpyHostToDevice, c->stream), "H2D U");
    ck(cudaMemcpyAsync(c->Vhat.p, V, sizeof(double) * n * r, cudaMemcpyHostToDevice, c->stream), "H2D V");
    c->U_m = 0;
    c->Vhat_n = 0;
    rsmk::launch_residual(v.Y, v.bitsR, m, n, v.nwp, c->U.as<double>(), c->Vhat.as<double>(), (int)r,
                          c->rowres.as<double>(), c->stream);
    rsmk::launch_sum_rows(c->rowres.as<double>(), m, c->dsum.as<double>(), c->stream);
    ck(cudaMemcpyAsync(ss_out, c->dsum.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "residual");
    ck(cudaGetLastError(), "residual kernels");
    *known = c->known;
  });
  if (st) g_err = c->err;
  return st;
}

rsm_status rsm_masked_residual_norm(const double* values, const uint8_t* mask, int64_t m, int64_t n,
                                    const double* U, const double* V, int64_t r, double* e) {
  // core.cpp:35-39 on the device
  double ss = 0.0;
  int64_t known = 0;
  rsm_status st = residual_ss(values, mask, m, n, U, V, r, &ss, &known);
  if (st) return st;
  if (known == 0) {
    g_err = "empty mask: no known entries";
    return RSM_ERR_INVALID_CONFIG;
  }
  *e = std::sqrt(ss) / std::sqrt((double)known);
  return RSM_OK;
}

rsm_status rsm_masked_objective(const double* values, const uint8_t* mask, int64_t m, int64_t n, const double* U,
                                const double* V, int64_t r, int32_t norm, double* out) {
  // core.cpp:41-44: only the Frobenius norm exists
  if (norm != 0) {
    g_err = "unsupported norm: only frobenius is implemented";
    return RSM_ERR_INVALID_CONFIG;
  }
  double ss = 0.0;
  int64_t known = 0;
  rsm_status st = residual_ss(values, mask, m, n, U, V, r, &ss, &known);
  if (st) return st;
  *out = std::sqrt(ss);
  return RSM_OK;
}

rsm_status rsm_sample(const double* values, const uint8_t* mask, int64_t m, int64_t n, int32_t mode,
                      int64_t count, uint64_t seed, uint64_t trial_index, int64_t* drawn, int64_t* kept,
                      int64_t* nkept) {
  // sampler.cpp:27-87 for one attempt: the draw on the device with the
  // selection kernels' code, the kept set from the bit-packed mask
  const bool m2 = mode == RSM_MODE_M2;
  if (m2 ? (count < 1 || count > m) : (count < 1 || count > n)) {
    g_err = m2 ? "sample_m2: row count out of range" : "sample_m1: column count out of range";
    return RSM_ERR_INVALID_CONFIG;
  }
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = rsm_ctx_load(c, values, mask, m, n);
  if (st) { g_err = c->err; return st; }
  st = guard(c, [&] {
    if (count > rsmd::KMAX) fail(RSM_ERR_INVALID_CONFIG, "device path supports at most 16 drawn indices");
    const View v = make_view(c, false, !m2);
    const uint32_t* bits = m2 ? v.bitsR : v.bitsC;
    const int64_t stride = m2 ? v.nwp : v.mwp;
    const int64_t nwords = m2 ? ceil_div(n, 32) : ceil_div(m, 32);
    const int64_t pool = m2 ? m : n;
    const int64_t other = m2 ? n : m;
    c->aux0.ensure(sizeof(int32_t) * rsmd::KMAX);
    c->aux1.ensure(sizeof(uint32_t) * nwords);
    c->aux2.ensure(sizeof(int32_t) * other);
    c->aux3.ensure(sizeof(int64_t));
    rsmk::launch_sample_one(bits, stride, nwords, pool, (int)count, seed, trial_index, c->aux0.as<int32_t>(),
                            c->aux1.as<uint32_t>(), c->aux2.as<int32_t>(), c->aux3.as<int64_t>(), c->stream);
    ++c->launches;
    std::vector<int32_t> d((size_t)count), k((size_t)other);
    int64_t nk = 0;
    ck(cudaMemcpyAsync(&nk, c->aux3.p, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaMemcpyAsync(d.data(), c->aux0.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaMemcpyAsync(k.data(), c->aux2.p, sizeof(int32_t) * other, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sample");
    ck(cudaGetLastError(), "sample kernel");
    for (int64_t i = 0; i < count; ++i) drawn[i] = d[(size_t)i];
    for (int64_t i = 0; i < nk; ++i) kept[i] = k[(size_t)i];
    *nkept = nk;
  });
  if (st) g_err = c->err;
  return st;
}

rsm_status rsm_small_singular_vectors(const double* S, int64_t p, int64_t q, int64_t r, int64_t ell, double* zeta,
                                      double* sv) {
  // spectra.cpp:48-56: the reference's validation, in its order
  if (q - r < 1) { g_err = "degenerate submatrix: needs more than r columns"; return RSM_ERR_INVALID_CONFIG; }
  if (p < r + 1) { g_err = "degenerate submatrix: needs more than r rows"; return RSM_ERR_INVALID_CONFIG; }
  if (ell < 1 || ell > q - r) { g_err = "vector count must lie in [1, cols-r]"; return RSM_ERR_INVALID_CONFIG; }
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = guard(c, [&] {
    if (std::min(p, q) > 32) fail(RSM_ERR_INVALID_CONFIG, "device path supports min(rows, cols) <= 32");
    if (p * q > ((int64_t)1 << 28) || q > 65536) fail(RSM_ERR_INVALID_CONFIG, "submatrix too large for the device path");
    c->aux0.ensure(sizeof(double) * p * q);
    c->aux1.ensure(sizeof(double) * rsmk::small_svd_scratch_doubles((int)p, (int)q));
    c->aux2.ensure(sizeof(double) * ell * q);
    c->aux3.ensure(sizeof(double) * ell);
    ck(cudaMemcpyAsync(c->aux0.p, S, sizeof(double) * p * q, cudaMemcpyHostToDevice, c->stream), "H2D S");
    rsmk::launch_small_svd(c->aux0.as<double>(), (int)p, (int)q, (int)ell, c->aux1.as<double>(),
                           c->aux2.as<double>(), c->aux3.as<double>(), c->stream);
    ++c->launches;
    ck(cudaMemcpyAsync(zeta, c->aux2.p, sizeof(double) * ell * q, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaMemcpyAsync(sv, c->aux3.p, sizeof(double) * ell, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "small svd");
    ck(cudaGetLastError(), "small svd kernel");
  });
  if (st) g_err = c->err;
  return st;
}

rsm_status rsm_gram_update(double* G, int64_t n, const double* X, int64_t nvec, const double* G2) {
  if (n < 1) { g_err = "gram accumulator: dimension must be positive"; return RSM_ERR_INVALID_CONFIG; }
  if (nvec < 0 || (nvec > 0 && !X)) { g_err = "accumulate: dimension mismatch"; return RSM_ERR_INVALID_CONFIG; }
  rsm_ctx* c = nullptr;
  rsm_status st = guard(nullptr, [&] { c = default_ctx(); });
  if (st) return st;
  std::lock_guard<std::mutex> lk(c->oneshot);
  st = guard(c, [&] {
    c->aux0.ensure(sizeof(double) * n * n);
    c->aux1.ensure(sizeof(double) * std::max<int64_t>(nvec, 1) * n);
    if (G2) c->aux2.ensure(sizeof(double) * n * n);
    ck(cudaMemcpyAsync(c->aux0.p, G, sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream), "H2D G");
    if (nvec > 0) ck(cudaMemcpyAsync(c->aux1.p, X, sizeof(double) * nvec * n, cudaMemcpyHostToDevice, c->stream), "H2D X");
    if (G2) ck(cudaMemcpyAsync(c->aux2.p, G2, sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream), "H2D G2");
    rsmk::launch_gram_update(c->aux0.as<double>(), n, c->aux1.as<double>(), nvec, G2 ? c->aux2.as<double>() : nullptr,
                             c->stream);
    ++c->launches;
    ck(cudaMemcpyAsync(G, c->aux0.p, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->stream), "D2H G");
    ck(cudaStreamSynchronize(c->stream), "gram update");
    ck(cudaGetLastError(), "gram update kernel");
  });
  if (st) g_err = c->err;
  return st;
}

}  // extern "C"
