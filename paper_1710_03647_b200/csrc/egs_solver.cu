// egs_solver.cu — host orchestration of the B200 energy-game solver and the
// device half of the C-ABI declared in include/egs_gpu.h.
//
// The solve is the reference's value iteration (solve_frontier,
// proj/src/solver_par.cpp:247-435) run as synchronous rounds on the device:
//   seed -> { lift round (dense or worklist) -> [certificate] -> activation }*
// until a round raises nothing.  Rounds read the measure of the previous
// round (Jacobi), so the output is schedule-independent and identical to the
// reference's least fixpoint; see DESIGN.md §3 for the proof that the
// losing-region certificate preserves it.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "egs_gpu.h"
#include "egs_kernels.cuh"

namespace {

thread_local std::string g_last_error;

}  // namespace

void egs_internal_set_error(const std::string& msg) { g_last_error = msg; }

namespace {

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess)                                                 \
      throw Fail(EGS_ERR_CUDA, std::string(#x) + ": " +                    \
                                   cudaGetErrorString(e_));                \
  } while (0)

using Clock = std::chrono::steady_clock;

double secs_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMalloc(&p, count * sizeof(T)));
  return static_cast<T*>(p);
}

// Lanes per vertex: the reference's choose_chunk_size (solver_seq.cpp:214-219)
// clamped to one warp.
int choose_lanes(uint32_t n, uint64_t m) {
  if (n == 0) return 1;
  long long r = llround(static_cast<double>(m) / static_cast<double>(n));
  r = std::max(1LL, std::min(32LL, r));
  int g = 1;
  while (g * 2 <= r) g *= 2;
  return g;
}

__global__ void k_heavy_select(uint32_t n, const uint32_t* off,
                               uint32_t thresh, uint32_t* list,
                               uint32_t* count) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u;
       base < n; base += stride) {
    const uint32_t v = base + (threadIdx.x & 31u);
    const bool h = v < n && off[v + 1] - off[v] > thresh;
    egs::warp_append(h, v, list, count);
  }
}

}  // namespace

// Device-resident solver context.
struct egs_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  uint32_t n = 0;
  uint32_t m = 0;
  int64_t cap = 0;
  int vbits = 32;
  int lanes = 1;
  uint32_t heavy_thresh = 0xFFFFFFFFu;
  double avg_deg = 0;
  egs_gpu_opts opts{};
  // arena
  uint32_t* off = nullptr;
  int2* edge = nullptr;
  uint8_t* owner = nullptr;
  uint32_t* coff = nullptr;
  uint32_t* csrc = nullptr;
  uint32_t* heavy = nullptr;
  uint32_t nheavy = 0;
  // solver state
  void* f[2] = {nullptr, nullptr};
  int cur = 0;
  int2* wit = nullptr;
  uint32_t* changed = nullptr;
  uint32_t* fr[2] = {nullptr, nullptr};
  uint32_t* bm[2] = {nullptr, nullptr};
  uint8_t* cand = nullptr;
  uint32_t* dcounts = nullptr;  // [0] changed [1] fr0 [2] fr1 [3] removed [4] scratch
  unsigned long long* ctr = nullptr;
  int64_t* f64 = nullptr;
  // pinned mirrors
  uint32_t* h_counts = nullptr;
  unsigned long long* h_ctr = nullptr;
  cudaEvent_t ev[8] = {};
  bool solved = false;

  egs::DevArena arena() const {
    return egs::DevArena{n, m, off, edge, owner, coff, csrc, cap};
  }
  uint32_t grid_for(uint64_t items, int lanes_per_item, int block = 256) const {
    uint64_t threads = items * (uint64_t)lanes_per_item;
    uint64_t blocks = (threads + block - 1) / block;
    uint64_t maxb = (uint64_t)num_sms * 8;
    return (uint32_t)std::max<uint64_t>(1, std::min(blocks, maxb));
  }
};

namespace {

void ctx_free(egs_ctx* c) {
  if (!c) return;
  if (c->device >= 0) cudaSetDevice(c->device);
  void* ptrs[] = {c->off,   c->edge,   c->owner, c->coff,    c->csrc,
                  c->heavy, c->f[0],   c->f[1],  c->wit,     c->changed,
                  c->fr[0], c->fr[1],  c->bm[0], c->bm[1],   c->cand,
                  c->dcounts, c->ctr,  c->f64};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->h_counts) cudaFreeHost(c->h_counts);
  if (c->h_ctr) cudaFreeHost(c->h_ctr);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

void validate_opts(const egs_gpu_opts& o) {
  if (o.n_gpus != 1)
    throw Fail(EGS_ERR_INVALID_CONFIG,
               "egs_gpu_solve drives one GPU per process; use the "
               "partitioned driver for n_gpus > 1");
  if (o.mode < EGS_MODE_AUTO || o.mode > EGS_MODE_SPARSE)
    throw Fail(EGS_ERR_INVALID_CONFIG, "mode must be 0, 1 or 2");
  if (o.cert_interval < 0)
    throw Fail(EGS_ERR_INVALID_CONFIG, "cert_interval must be >= 0");
  if (o.timeout_seconds < 0)
    throw Fail(EGS_ERR_INVALID_CONFIG, "timeout must be >= 0");
}

egs_ctx* ctx_create(const egs_arena_view* a, const egs_gpu_opts& opts,
                    egs_gpu_stats* st) {
  validate_opts(opts);
  if (!a) throw Fail(EGS_ERR_INVALID_CONFIG, "null arena");
  if (a->num_edges >= 0xFFFFFFFFull)
    throw Fail(EGS_ERR_UNSUPPORTED,
               "arenas with >= 2^32 edges are not supported on the device");
  if (a->num_vertices > 0 && a->num_edges < a->num_vertices)
    throw Fail(EGS_ERR_INVALID_CONFIG, "arena is not total");
  if (a->credit_cap < 0)
    throw Fail(EGS_ERR_INVALID_CONFIG, "negative credit_cap");
  if (a->max_abs_weight > 2147483647LL)
    throw Fail(EGS_ERR_UNSUPPORTED,
               "edge weights beyond int32 are not supported on the device");
  auto t0 = Clock::now();
  egs_ctx* c = new egs_ctx();
  try {
    c->opts = opts;
    if (opts.device >= 0) {
      CK(cudaSetDevice(opts.device));
      c->device = opts.device;
    } else {
      CK(cudaGetDevice(&c->device));
    }
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount,
                              c->device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    c->n = a->num_vertices;
    c->m = (uint32_t)a->num_edges;
    c->cap = a->credit_cap;
    c->vbits = a->credit_cap < 0xFFFFFFFFLL ? 32 : 64;
    c->lanes = choose_lanes(c->n, c->m);
    c->avg_deg = c->n ? (double)c->m / c->n : 0.0;
    c->heavy_thresh = (uint32_t)std::max(256, 32 * c->lanes);
    const uint32_t n = c->n, m = c->m;
    const size_t vsz = c->vbits / 8;
    cudaStream_t s = c->stream;

    CK(cudaMallocHost(&c->h_counts, 8 * sizeof(uint32_t)));
    CK(cudaMallocHost(&c->h_ctr, egs::kNumCounters * sizeof(unsigned long long)));
    c->dcounts = dalloc<uint32_t>(8);
    c->ctr = dalloc<unsigned long long>(egs::kNumCounters);
    c->off = dalloc<uint32_t>((size_t)n + 1);
    c->edge = dalloc<int2>(m);
    c->owner = dalloc<uint8_t>(n);
    c->coff = dalloc<uint32_t>((size_t)n + 1);
    c->csrc = dalloc<uint32_t>(m);
    c->heavy = dalloc<uint32_t>(n);
    c->f[0] = dalloc<uint8_t>((size_t)n * vsz);
    c->f[1] = dalloc<uint8_t>((size_t)n * vsz);
    c->wit = dalloc<int2>(n);
    c->changed = dalloc<uint32_t>((size_t)n * 2 + 1);
    c->fr[0] = dalloc<uint32_t>(n);
    c->fr[1] = dalloc<uint32_t>(n);
    const size_t words = ((size_t)n + 31) / 32;
    c->bm[0] = dalloc<uint32_t>(words);
    c->bm[1] = dalloc<uint32_t>(words);
    c->cand = dalloc<uint8_t>(n);
    c->f64 = dalloc<int64_t>(n);

    if (n > 0) {
      // Upload the reference CSR as-is and pack it on the device.
      uint64_t* off64 = dalloc<uint64_t>((size_t)n + 1);
      uint32_t* dst = dalloc<uint32_t>(m);
      int64_t* w64 = dalloc<int64_t>(m);
      int* bad = dalloc<int>(1);
      CK(cudaMemcpyAsync(off64, a->csr_offsets, ((size_t)n + 1) * 8,
                         cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dst, a->csr_targets, (size_t)m * 4,
                         cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(w64, a->csr_weights, (size_t)m * 8,
                         cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(c->owner, a->owners, n, cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
      CK(cudaMemsetAsync(c->coff, 0, ((size_t)n + 1) * 4, s));
      const uint32_t grid = c->grid_for(std::max<uint64_t>(m, n), 1);
      egs::k_pack<<<grid, 256, 0, s>>>(n, m, off64, dst, w64, c->off, c->edge,
                                       c->coff, bad);
      CK(cudaGetLastError());
      // exclusive scan of in-degrees -> CSC offsets (n+1 entries, last = 0)
      size_t tmp_bytes = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, c->coff, c->coff,
                                       (int)(n + 1), s));
      void* tmp = dalloc<uint8_t>(tmp_bytes);
      CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, c->coff, c->coff,
                                       (int)(n + 1), s));
      // cursor: reuse the (now unneeded) dst buffer
      CK(cudaMemcpyAsync(dst, c->coff, (size_t)n * 4,
                         cudaMemcpyDeviceToDevice, s));
      switch (c->lanes) {
#define EGS_SCATTER(G)                                                       \
  case G:                                                                    \
    egs::k_csc_scatter<G><<<c->grid_for(n, G), 256, 0, s>>>(                 \
        n, c->off, c->edge, dst, c->csrc);                                   \
    break;
        EGS_SCATTER(1) EGS_SCATTER(2) EGS_SCATTER(4) EGS_SCATTER(8)
        EGS_SCATTER(16) EGS_SCATTER(32)
#undef EGS_SCATTER
      }
      CK(cudaGetLastError());
      CK(cudaMemsetAsync(c->dcounts, 0, 8 * sizeof(uint32_t), s));
      k_heavy_select<<<c->grid_for(n, 1), 256, 0, s>>>(
          n, c->off, c->heavy_thresh, c->heavy, c->dcounts + 4);
      CK(cudaGetLastError());
      int h_bad = 0;
      CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(c->h_counts, c->dcounts, 8 * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      c->nheavy = c->h_counts[4];
      cudaFree(off64);
      cudaFree(dst);
      cudaFree(w64);
      cudaFree(bad);
      cudaFree(tmp);
      if (h_bad == 1)
        throw Fail(EGS_ERR_UNSUPPORTED,
                   "edge weight outside int32 on the device path");
      if (h_bad == 2)
        throw Fail(EGS_ERR_INVALID_CONFIG, "edge target out of range");
    }
    if (st) {
      st->upload_seconds = secs_since(t0);
      st->value_bits = (uint32_t)c->vbits;
      st->lanes = (uint32_t)c->lanes;
    }
    return c;
  } catch (...) {
    ctx_free(c);
    throw;
  }
}

// Read device counters into the pinned mirrors (synchronises the stream).
void pull_counts(egs_ctx* c) {
  CK(cudaMemcpyAsync(c->h_counts, c->dcounts, 8 * sizeof(uint32_t),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->h_ctr, c->ctr,
                     egs::kNumCounters * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

template <class V, int G>
void run_solve(egs_ctx* c, egs_gpu_stats* st) {
  const auto t0 = Clock::now();
  cudaStream_t s = c->stream;
  const uint32_t n = c->n;
  const egs::DevArena g = c->arena();
  V* f[2] = {static_cast<V*>(c->f[0]), static_cast<V*>(c->f[1])};
  const egs_gpu_opts& o = c->opts;
  const size_t words = ((size_t)n + 31) / 32;
  const double vs = sizeof(V);
  uint64_t launches = 0, lift_launches = 0;
  double cert_ms = 0, act_ms = 0;
  int cur = 0;
  int frb = 0;

  CK(cudaMemsetAsync(c->dcounts, 0, 8 * sizeof(uint32_t), s));
  CK(cudaMemsetAsync(c->ctr, 0, egs::kNumCounters * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(c->bm[0], 0, words * 4, s));
  CK(cudaEventRecord(c->ev[2], s));
  ++launches;
  egs::k_seed<V, G><<<c->grid_for(n, G), 256, 0, s>>>(
      g, f[0], f[1], c->wit, c->bm[0], c->fr[0], c->dcounts + 1);
  CK(cudaGetLastError());
  pull_counts(c);
  uint32_t fr_n = c->h_counts[1];

  uint64_t rounds = 0, dense_rounds = 0, sparse_rounds = 0, pops = 0;
  uint64_t cert_attempts = 0, cert_passes = 0;
  double lift_ms = 0;
  double lift_bytes = 0;
  unsigned long long prev[egs::kNumCounters] = {0};
  int K = o.cert_interval > 0 ? o.cert_interval : 4;
  uint64_t next_cert = (uint64_t)K;
  const uint64_t budget =
      o.round_bound ? o.round_bound
                    : (c->m > 0 && (uint64_t)c->cap + 1 >
                                       UINT64_MAX / std::max<uint64_t>(1, c->m)
                           ? UINT64_MAX
                           : (uint64_t)c->m * ((uint64_t)c->cap + 1) + 1);
  auto want_dense = [&](uint64_t frontier) {
    if (o.mode == EGS_MODE_DENSE) return true;
    if (o.mode == EGS_MODE_SPARSE) return false;
    return (double)frontier * 16.0 > (double)n;
  };
  bool dense = want_dense(fr_n);
  bool converged = fr_n == 0;

  while (!converged) {
    CK(cudaMemsetAsync(c->dcounts + 0, 0, sizeof(uint32_t), s));
    egs::LiftArgs<V> a{};
    a.g = g;
    a.fcur = f[cur];
    a.fnxt = f[cur ^ 1];
    a.wit = c->wit;
    a.heavy_thresh = c->heavy_thresh;
    a.changed_list = c->changed;
    a.changed_count = c->dcounts + 0;
    a.ctr = c->ctr;
    uint64_t items;
    if (dense) {
      a.items = nullptr;
      a.count_dev = nullptr;
      a.count = n;
      a.dense = 1;
      items = n;
    } else {
      a.items = c->fr[frb];
      a.count_dev = c->dcounts + 1 + frb;
      a.count = 0;
      a.dense = 0;
      items = fr_n;
    }
    CK(cudaEventRecord(c->ev[0], s));
    egs::k_lift<V, G><<<c->grid_for(items, G), 256, 0, s>>>(a);
    ++launches;
    ++lift_launches;
    if (c->nheavy) ++launches, ++lift_launches;
    if (c->nheavy)
      egs::k_lift_heavy<V><<<std::min<uint32_t>(c->nheavy, c->num_sms * 4),
                             512, 0, s>>>(a, c->heavy, c->nheavy, c->bm[frb]);
    CK(cudaEventRecord(c->ev[1], s));
    CK(cudaGetLastError());
    if (dense) {
      cur ^= 1;
    } else {
      ++launches;
      egs::k_commit<V><<<c->grid_for(items, 1), 256, 0, s>>>(
          f[cur], f[cur ^ 1], c->changed, c->dcounts + 0);
      CK(cudaGetLastError());
    }
    pull_counts(c);
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
    lift_ms += ms;
    {
      const unsigned long long* h = c->h_ctr;
      const double d_edges = (double)(h[egs::kEdges] - prev[egs::kEdges]);
      const double d_apps = (double)(h[egs::kApps] - prev[egs::kApps]);
      const double d_wit = (double)(h[egs::kWitness] - prev[egs::kWitness]);
      lift_bytes += d_edges * (8 + vs) + d_apps * (4 + 2 * vs) +
                    d_wit * (8 + 2 * vs) + (dense ? 0.0 : (double)items * 4);
      std::memcpy(prev, h, sizeof(prev));
    }
    ++rounds;
    pops += items;
    (dense ? dense_rounds : sparse_rounds)++;
    uint32_t changed = c->h_counts[0];
    if (changed == 0) break;
    if (rounds >= budget)
      throw Fail(EGS_ERR_BOUND, "round budget of " + std::to_string(budget) +
                                    " exhausted before reaching a fixpoint");
    if (o.timeout_seconds > 0 && secs_since(t0) >= o.timeout_seconds)
      throw Fail(EGS_ERR_TIMEOUT, "solve timed out");

    bool certified_any = false;
    if (o.certify && rounds >= next_cert) {
      ++cert_attempts;
      const unsigned long long before = c->h_ctr[egs::kCertified];
      CK(cudaEventRecord(c->ev[4], s));
      ++launches;
      egs::k_cert_init<V><<<c->grid_for(n, 1), 256, 0, s>>>(f[cur], c->cand, n);
      for (;;) {
        CK(cudaMemsetAsync(c->dcounts + 3, 0, sizeof(uint32_t), s));
        ++launches;
        egs::k_cert_prune<V, G><<<c->grid_for(n, G), 256, 0, s>>>(
            g, f[cur], c->cand, c->dcounts + 3);
        CK(cudaGetLastError());
        ++cert_passes;
        pull_counts(c);
        if (c->h_counts[3] == 0) break;
      }
      ++launches;
      egs::k_cert_apply<V><<<c->grid_for(n, 1), 256, 0, s>>>(
          f[cur], c->cand, n, c->changed, c->dcounts + 0, c->ctr);
      CK(cudaGetLastError());
      CK(cudaEventRecord(c->ev[5], s));
      pull_counts(c);
      {
        float cm = 0;
        CK(cudaEventElapsedTime(&cm, c->ev[4], c->ev[5]));
        cert_ms += cm;
      }
      changed = c->h_counts[0];
      certified_any = c->h_ctr[egs::kCertified] > before;
      if (!certified_any) K = std::min(K * 2, 64);
      next_cert = rounds + (uint64_t)K;
    }

    const bool dense_next =
        want_dense((uint64_t)((double)changed * std::max(1.0, c->avg_deg))) ||
        (certified_any && o.mode == EGS_MODE_AUTO);
    if (!dense_next) {
      const int nb = frb ^ 1;
      CK(cudaMemsetAsync(c->bm[nb], 0, words * 4, s));
      CK(cudaMemsetAsync(c->dcounts + 1 + nb, 0, sizeof(uint32_t), s));
      CK(cudaEventRecord(c->ev[6], s));
      ++launches;
      egs::k_activate<V, G><<<c->grid_for(changed, G), 256, 0, s>>>(
          g, f[cur], c->changed, c->dcounts + 0, c->bm[nb], c->fr[nb],
          c->dcounts + 1 + nb, c->ctr);
      CK(cudaGetLastError());
      CK(cudaEventRecord(c->ev[7], s));
      pull_counts(c);
      {
        float am = 0;
        CK(cudaEventElapsedTime(&am, c->ev[6], c->ev[7]));
        act_ms += am;
      }
      frb = nb;
      fr_n = c->h_counts[1 + nb];
      if (fr_n == 0) break;
    }
    dense = dense_next;
  }
  CK(cudaEventRecord(c->ev[3], s));
  CK(cudaStreamSynchronize(s));
  float solve_ms = 0;
  CK(cudaEventElapsedTime(&solve_ms, c->ev[2], c->ev[3]));
  c->cur = cur;
  c->solved = true;
  if (st) {
    const unsigned long long* h = c->h_ctr;
    st->lifts = h[egs::kLifts];
    st->applications = h[egs::kApps];
    st->edges_relaxed = h[egs::kEdges];
    st->witness_checks = h[egs::kWitness];
    st->activations = h[egs::kActScanned];
    st->certified = h[egs::kCertified];
    st->pops = pops;
    st->rounds = rounds;
    st->dense_rounds = dense_rounds;
    st->sparse_rounds = sparse_rounds;
    st->cert_attempts = cert_attempts;
    st->cert_passes = cert_passes;
    st->solve_seconds = solve_ms * 1e-3;
    st->lift_kernel_seconds = lift_ms * 1e-3;
    st->lift_bytes = (uint64_t)lift_bytes;
    st->value_bits = (uint32_t)c->vbits;
    st->lanes = (uint32_t)c->lanes;
    st->kernel_launches = launches;
    st->lift_launches = lift_launches;
    st->cert_kernel_seconds = cert_ms * 1e-3;
    st->activate_kernel_seconds = act_ms * 1e-3;
  }
}

template <class V>
void dispatch_lanes(egs_ctx* c, egs_gpu_stats* st) {
  switch (c->lanes) {
    case 1: return run_solve<V, 1>(c, st);
    case 2: return run_solve<V, 2>(c, st);
    case 4: return run_solve<V, 4>(c, st);
    case 8: return run_solve<V, 8>(c, st);
    case 16: return run_solve<V, 16>(c, st);
    default: return run_solve<V, 32>(c, st);
  }
}

void ctx_solve(egs_ctx* c, egs_gpu_stats* st) {
  CK(cudaSetDevice(c->device));
  if (c->n == 0) {
    c->solved = true;
    return;
  }
  if (c->vbits == 32)
    dispatch_lanes<uint32_t>(c, st);
  else
    dispatch_lanes<uint64_t>(c, st);
}

void ctx_read(egs_ctx* c, int64_t* out) {
  if (!c->solved) throw Fail(EGS_ERR_INVALID_CONFIG, "context not solved");
  if (c->n == 0) return;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  if (c->vbits == 32)
    egs::k_widen<uint32_t><<<c->grid_for(c->n, 1), 256, 0, s>>>(
        static_cast<uint32_t*>(c->f[c->cur]), c->f64, c->n);
  else
    egs::k_widen<uint64_t><<<c->grid_for(c->n, 1), 256, 0, s>>>(
        static_cast<uint64_t*>(c->f[c->cur]), c->f64, c->n);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, c->f64, (size_t)c->n * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
}

int ctx_epm(egs_ctx* c, const int64_t* f) {
  CK(cudaSetDevice(c->device));
  if (c->n == 0) return 1;
  cudaStream_t s = c->stream;
  CK(cudaMemcpyAsync(c->f64, f, (size_t)c->n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(c->ctr, 0, egs::kNumCounters * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(c->dcounts, 0, 8 * sizeof(uint32_t), s));
  egs::k_epm<<<c->grid_for(c->n, 1), 256, 0, s>>>(
      c->arena(), c->f64, c->ctr, reinterpret_cast<int*>(c->dcounts + 5));
  CK(cudaGetLastError());
  pull_counts(c);
  c->solved = false;  // f64 scratch reused
  if (c->h_counts[5]) throw Fail(EGS_ERR_UNSUPPORTED, "energy subtraction out of range");
  return c->h_ctr[0] == 0 ? 1 : 0;
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return EGS_OK;
  } catch (const Fail& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return EGS_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return EGS_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" {

void egs_gpu_opts_default(egs_gpu_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->n_gpus = 1;
  o->device = -1;
  o->certify = 1;
  o->cert_interval = 4;
  o->mode = EGS_MODE_AUTO;
}

int egs_ctx_create(const egs_arena_view* arena, const egs_gpu_opts* opts,
                   egs_ctx** out, egs_gpu_stats* stats) {
  return guarded([&] {
    egs_gpu_opts o;
    if (opts) o = *opts; else egs_gpu_opts_default(&o);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    *out = ctx_create(arena, o, stats);
  });
}

int egs_ctx_solve(egs_ctx* ctx, egs_gpu_stats* stats) {
  return guarded([&] {
    if (!ctx) throw Fail(EGS_ERR_INVALID_CONFIG, "null context");
    auto t0 = Clock::now();
    double up = stats ? stats->upload_seconds : 0;
    if (stats) std::memset(stats, 0, sizeof(*stats));
    ctx_solve(ctx, stats);
    if (stats) {
      stats->upload_seconds = up;
      stats->wall_seconds = secs_since(t0);
    }
  });
}

int egs_ctx_read_measure(egs_ctx* ctx, int64_t* f_out) {
  return guarded([&] {
    if (!ctx) throw Fail(EGS_ERR_INVALID_CONFIG, "null context");
    ctx_read(ctx, f_out);
  });
}

int egs_ctx_is_progress_measure(egs_ctx* ctx, const int64_t* f) {
  int r = 0;
  int rc = guarded([&] {
    if (!ctx) throw Fail(EGS_ERR_INVALID_CONFIG, "null context");
    r = ctx_epm(ctx, f);
  });
  return rc == EGS_OK ? r : -rc;
}

void egs_ctx_destroy(egs_ctx* ctx) { ctx_free(ctx); }

int egs_gpu_solve(const egs_arena_view* arena, const egs_gpu_opts* opts,
                  int64_t* f_out, egs_gpu_stats* stats) {
  return guarded([&] {
    auto t0 = Clock::now();
    egs_gpu_opts o;
    if (opts) o = *opts; else egs_gpu_opts_default(&o);
    egs_gpu_stats local{};
    egs_gpu_stats* st = stats ? stats : &local;
    std::memset(st, 0, sizeof(*st));
    egs_ctx* c = ctx_create(arena, o, st);
    try {
      const double up = st->upload_seconds;
      ctx_solve(c, st);
      auto t1 = Clock::now();
      ctx_read(c, f_out);
      st->download_seconds = secs_since(t1);
      st->upload_seconds = up;
    } catch (...) {
      ctx_free(c);
      throw;
    }
    ctx_free(c);
    st->wall_seconds = secs_since(t0);
  });
}

void* egs_host_alloc_pinned(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes ? bytes : 1) != cudaSuccess) return nullptr;
  return p;
}

void egs_host_free_pinned(void* p) {
  if (p) cudaFreeHost(p);
}

const char* egs_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
