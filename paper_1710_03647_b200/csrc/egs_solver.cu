// egs_solver.cu — host orchestration of the B200 energy-game solver and the
// device half of the C-ABI declared in include/egs_gpu.h.
//
//   egs_ctx_create   upload the reference CSR (GameArena spans, arena.hpp:
//                    109-115) and rebuild it on the device (egs_build.cuh)
//   egs_ctx_solve    ONE cooperative launch of k_solve (egs_solve.cuh): seed,
//                    lift rounds, certificate, activation and the fixpoint
//                    test all run on the device; the host waits once
//   egs_ctx_read_measure / egs_gpu_solve
//                    export the least progress measure in the reference's
//                    raw int64 encoding (energy.hpp:16), original vertex ids
//
// It replaces egsolve::solve (proj/include/egsolve/solver.hpp:86-87) for the
// GPU variant; the output is the same least fixpoint the reference solvers
// compute (solver_seq.cpp:124-212, solver_par.cpp:126-435).

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <limits>
#include <string>
#include <vector>
#include <atomic>
#include <mutex>
#include <thread>
#include <tuple>

#include "egs_build.cuh"
#include "egs_gpu.h"
#include "egs_narrow.h"
#include "egs_pool.h"
#include "egs_scan.cuh"
#include "egs_types.cuh"

// The solve kernels, compiled once per edge-record format (egs_kern.cu):
// e8 = int2 {dst, w} records, e4 = packed u32 records.
namespace egs {
namespace e8 {
const void* solve_kernel(int vbits);
}  // namespace e8
namespace e4 {
const void* solve_kernel(int vbits);
}  // namespace e4
}  // namespace egs

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

// Device memory comes from the device's stream-ordered pool with an
// unbounded release threshold: a repeated one-shot solve (egs_gpu_solve)
// re-uses the previous call's gigabytes instead of mapping them again.
void use_caching_pool(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[device] = true;
}

thread_local cudaStream_t g_alloc_stream = nullptr;  // stream of the ctx being built

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMallocAsync(&p, count * sizeof(T), g_alloc_stream));
  return static_cast<T*>(p);
}

void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

// RAII for upload temporaries (freed in stream order).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() { dfree(p, s); }
  template <class T>
  T* as() {
    return static_cast<T*>(p);
  }
  template <class T>
  T* alloc(size_t count) {
    s = g_alloc_stream;
    p = dalloc<T>(count);
    return as<T>();
  }
  void release() {
    dfree(p, s);
    p = nullptr;
  }
};

uint32_t grid_for(uint64_t items, int num_sms, int block = 256) {
  const uint64_t blocks = (items + block - 1) / block;
  const uint64_t maxb = (uint64_t)num_sms * 8;
  return (uint32_t)std::max<uint64_t>(1, std::min(blocks, maxb));
}

int bits_for(uint32_t n) {
  int b = 1;
  while (b < 32 && (1ull << b) < (uint64_t)n) ++b;
  return b;
}

}  // namespace

// Device-resident solver context.
struct egs_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // arena upload
  cudaStream_t aux_stream = nullptr;   // weight relabel, overlapping the CSC sort
  uint32_t n = 0;
  uint64_t m = 0;
  int64_t cap = 0;
  int vbits = 32;
  egs_gpu_opts opts{};
  uint32_t rb[egs::kNumClasses + 1] = {};
  // arena (relabelled)
  uint32_t* off = nullptr;
  void* edge = nullptr;
  uint32_t tbits = 0;  // 0: int2 records; else packed u32 (egs_types.cuh)
  uint32_t* coff = nullptr;
  uint32_t* csrc = nullptr;
  void* rec0 = nullptr;      // first record of each player-1 light row (by new id)
  uint32_t* perm = nullptr;  // old id -> new id
  uint32_t* inv = nullptr;   // new id -> old id
  // solver state
  void* f = nullptr;
  int2* wit = nullptr;
  uint32_t* chg[2] = {nullptr, nullptr};
  uint32_t* frb[2] = {nullptr, nullptr};  // frontier membership bitmaps
  uint32_t* rbm[2] = {nullptr, nullptr};
  uint32_t* cbm[2] = {nullptr, nullptr};
  uint32_t* cand = nullptr;  // certificate candidate bitmap (own vertices)
  uint32_t* ring = nullptr;  // certificate cascade queue (ring_cap slots, all-ones when free)
  uint32_t ring_cap = 0;
  uint32_t* longcol = nullptr;
  uint32_t* fr[2] = {nullptr, nullptr};
  void* stage = nullptr;
  egs::Scratch* scratch = nullptr;
  unsigned long long* ctr = nullptr;
  int64_t* f64 = nullptr;
  unsigned long long* h_ctr = nullptr;  // pinned mirror
  unsigned long long* trace = nullptr;  // EGS_TRACE=1: per-phase device times
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int grid = 0;
  bool solved = false;
  // multi-GPU partition (egs_part_*): this rank's range of relabelled ids,
  // its edge count, and the replicated state (f, chg[2], rbm[2], XSync) in
  // one IPC-exportable allocation `xbuf` with the same layout on every rank
  int rank = 0, world = 1;
  uint32_t own_lo = 0, own_hi = 0;
  uint64_t m_own = 0;
  int full_grid = 0;
  char* xbuf = nullptr;
  size_t xbytes = 0;
  char* xpeer[egs::kMaxRanks] = {};
  bool xpeer_ipc[egs::kMaxRanks] = {};  // opened with cudaIpcOpenMemHandle
  egs::XSync* xsync = nullptr;
  unsigned int epoch = 0;  // cross-rank barriers passed (same on every rank)
  bool connected = false;
  // sharded upload: the original-id row ranges this rank uploads (its own
  // rows, small gaps merged); empty = every row
  std::vector<std::pair<uint32_t, uint32_t>> runs;
  uint64_t h2d_bytes = 0;  // host -> device bytes of the last upload

  egs::Graph graph() const {
    egs::Graph g{};
    g.n = n;
    std::memcpy(g.rb, rb, sizeof(rb));
    g.off = off;
    g.edge = edge;
    g.tbits = tbits;
    g.coff = coff;
    g.csrc = csrc;
    g.rec0 = rec0;
    g.cap = cap;
    return g;
  }
};

namespace {

// EGS_VERBOSE=1 prints the device arena construction steps (host clock,
// stream-synchronised) to stderr.
// EGS_TIMELINE=1: stream-order event marks of the build, printed relative
// to the first (timing events; no synchronisation between marks)
struct Timeline {
  bool on = std::getenv("EGS_TIMELINE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void mark(const std::string& what, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, s));
    ev.emplace_back(what, e);
  }
  ~Timeline() {
    if (ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    for (auto& [w, e] : ev) {
      cudaEventSynchronize(e);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0].second, e);
      std::fprintf(stderr, "[egs timeline] %8.3f ms  %s\n", ms, w.c_str());
    }
    for (auto& [w, e] : ev) cudaEventDestroy(e);
  }
};

struct StepTimer {
  cudaStream_t s;
  bool on;
  Clock::time_point t;
  explicit StepTimer(cudaStream_t st) : s(st), on(std::getenv("EGS_VERBOSE") != nullptr) {
    t = Clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    if (s) cudaStreamSynchronize(s);
    std::fprintf(stderr, "[egs] %-28s %9.3f ms\n", what, secs_since(t) * 1e3);
    t = Clock::now();
  }
};

// Streams, events and the pinned counter block of finished contexts are
// kept per device and handed to the next context: a repeated one-shot
// egs_gpu_solve does not pay their creation (~2-3 ms) again.
struct Shell {
  cudaStream_t stream, copy_stream, aux_stream;
  cudaEvent_t ev[2];
  unsigned long long* h_ctr;
};
std::mutex g_shell_mu;
std::vector<std::pair<int, Shell>> g_shells;

void shell_put(int device, const Shell& sh) {
  std::lock_guard<std::mutex> lk(g_shell_mu);
  g_shells.emplace_back(device, sh);
}

bool shell_get(int device, Shell& sh) {
  std::lock_guard<std::mutex> lk(g_shell_mu);
  for (size_t i = 0; i < g_shells.size(); ++i) {
    if (g_shells[i].first == device) {
      sh = g_shells[i].second;
      g_shells.erase(g_shells.begin() + i);
      return true;
    }
  }
  return false;
}

// The replicated-state block of a finished partition context is kept per
// device (one, the largest) for the next one: a repeated egs_part_create --
// the multi-GPU one-shot path -- skips the cudaMalloc of an IPC-exportable
// block and its first export.  Freed at process exit with the context.
std::mutex g_xcache_mu;
std::vector<std::tuple<int, char*, size_t>> g_xcache;  // (device, block, bytes)

char* xbuf_take(int device, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_xcache_mu);
  for (size_t i = 0; i < g_xcache.size(); ++i) {
    auto [d, ptr, sz] = g_xcache[i];
    if (d == device && sz >= bytes) {
      g_xcache.erase(g_xcache.begin() + i);
      return ptr;
    }
  }
  void* xb = nullptr;
  CK(cudaMalloc(&xb, bytes));
  return static_cast<char*>(xb);
}

void xbuf_give(int device, char* ptr, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_xcache_mu);
  for (auto& [d, p, sz] : g_xcache)
    if (d == device) {
      if (sz >= bytes) {
        cudaFree(ptr);
      } else {
        cudaFree(p);
        p = ptr;
        sz = bytes;
      }
      return;
    }
  g_xcache.emplace_back(device, ptr, bytes);
}

void ctx_free(egs_ctx* c) {
  if (!c) return;
  StepTimer tm(c->stream);
  if (c->device >= 0) cudaSetDevice(c->device);
  // (the replicated state of a multi-GPU rank lives in xbuf: cudaFree'd below)
  const bool in_x = c->xbuf != nullptr;
  void* ptrs[] = {c->off,  c->edge,  c->coff,  c->csrc, c->perm,    c->inv,
                  in_x ? nullptr : c->f, c->wit, in_x ? nullptr : c->chg[0],
                  in_x ? nullptr : c->chg[1], c->frb[0], c->frb[1],
                  c->fr[0], c->fr[1], c->stage, c->scratch, c->ctr,
                  in_x ? nullptr : c->rbm[0], in_x ? nullptr : c->rbm[1], c->cbm[0], c->cbm[1],
                  c->cand, c->ring, c->trace, c->longcol, c->f64, c->rec0};
  for (int q = 0; q < egs::kMaxRanks; ++q)
    if (c->xpeer_ipc[q] && c->xpeer[q]) cudaIpcCloseMemHandle(c->xpeer[q]);
  if (c->xbuf) {
    if (c->stream) cudaStreamSynchronize(c->stream);
    xbuf_give(c->device, c->xbuf, c->xbytes);
  }
  if (c->stream) {
    for (void* p : ptrs) dfree(p, c->stream);
    cudaStreamSynchronize(c->stream);
  }
  tm.mark("free: device buffers");
  if (c->stream && c->copy_stream && c->aux_stream && c->h_ctr && c->ev[0] && c->ev[1]) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamSynchronize(c->aux_stream);
    shell_put(c->device, Shell{c->stream, c->copy_stream, c->aux_stream, {c->ev[0], c->ev[1]},
                               c->h_ctr});
  } else {
    if (c->h_ctr) cudaFreeHost(c->h_ctr);
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  }
  tm.s = nullptr;
  tm.mark("free: host, events, streams");
  delete c;
}

void validate_opts(const egs_gpu_opts& o) {
  if (o.n_gpus != 1)
    throw Fail(EGS_ERR_INVALID_CONFIG,
               "egs_gpu_solve drives one GPU; use egs_part_* for n_gpus > 1");
  if (o.mode < EGS_MODE_AUTO || o.mode > EGS_MODE_SWEEP)
    throw Fail(EGS_ERR_INVALID_CONFIG, "mode must be 0 (auto), 1 (dense), 2 (sparse) or 3 (sweep)");
  if (o.cert_interval < 0 || o.cert_growth < 0 || o.sparse_div < 0 || o.grid_ctas < 0)
    throw Fail(EGS_ERR_INVALID_CONFIG, "negative tuning knob");
  if (o.timeout_seconds < 0)
    throw Fail(EGS_ERR_INVALID_CONFIG, "timeout must be >= 0");
}

const void* solve_kernel(const egs_ctx* c) {
  return c->tbits ? egs::e4::solve_kernel(c->vbits) : egs::e8::solve_kernel(c->vbits);
}
size_t rec_bytes(const egs_ctx* c) { return c->tbits ? 4 : 8; }
// light-row phases staged through TMA tiles by default, measured per phase
// (profiles/README.md): round 1 and the certificate pass stream whole rows
// and gain; the dense player-1 lift is faster with plain row loads
constexpr int kDefaultTma = egs::kTmaRound1 | egs::kTmaCert;

// Process-wide pinned staging buffer for the narrowed weights (grows on
// demand; one upload at a time uses it).
std::mutex g_stage_mu;
void* g_stage = nullptr;
size_t g_stage_cap = 0;

void* pinned_stage(uint64_t bytes) {
  if (bytes > g_stage_cap) {
    if (g_stage) cudaFreeHost(g_stage);
    g_stage = nullptr;
    g_stage_cap = 0;
    void* p = nullptr;
    CK(cudaMallocHost(&p, std::max<uint64_t>(bytes, 1)));
    g_stage = p;
    g_stage_cap = bytes;
  }
  return g_stage;
}

// Exclusive prefix sum on the device (egs_scan.cuh): out[i] = in[0] + ... +
// in[i-1]; in place allowed.  Temporaries from the stream-ordered pool.
template <class T, class In>
void dev_excl_scan(const In* in, T* out, uint64_t n, cudaStream_t s, int sms) {
  if (n == 0) return;
  const uint64_t nt = (n + egs::kScanTile - 1) / egs::kScanTile;
  DevBuf d_ts;
  T* ts = d_ts.alloc<T>(nt);
  const uint32_t grid = (uint32_t)std::min<uint64_t>(nt, (uint64_t)sms * 8);
  egs::k_scan_reduce<T, In><<<grid, egs::kScanThreads, 0, s>>>(in, n, ts, nt);
  egs::k_scan_tiles<T><<<1, 1024, 0, s>>>(ts, nt);
  egs::k_scan_down<T, In><<<grid, egs::kScanThreads, 0, s>>>(in, out, n, ts, nt);
  CK(cudaGetLastError());
}

// Stable sort of (key, val) pairs by the low `bits` bits of key (egs_scan.cuh
// LSD radix sort, 8-bit digits): the pairs move (k0, v0) -> (k1, v1) -> ...;
// *ks / *vs = the buffers holding the sorted result.
void dev_radix_sort_pairs(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint64_t m,
                          int bits, cudaStream_t s, int sms, uint32_t** ks, uint32_t** vs) {
  *ks = k0;
  *vs = v0;
  if (m == 0) return;
  const uint32_t nt = (uint32_t)((m + egs::kRadixTile - 1) / egs::kRadixTile);
  DevBuf d_hist;
  uint32_t* hist = d_hist.alloc<uint32_t>((size_t)egs::kRadixDigits * nt);
  const uint32_t grid = std::min<uint32_t>(nt, (uint32_t)sms * 8);
  for (int shift = 0; shift < bits; shift += egs::kRadixBits) {
    egs::k_radix_hist<<<grid, egs::kScanThreads, 0, s>>>(k0, m, shift, hist, nt);
    dev_excl_scan<uint32_t>(hist, hist, (uint64_t)egs::kRadixDigits * nt, s, sms);
    egs::k_radix_scatter<<<grid, egs::kScanThreads, 0, s>>>(k0, v0, m, shift, hist, nt, k1, v1);
    CK(cudaGetLastError());
    std::swap(k0, k1);
    std::swap(v0, v1);
  }
  *ks = k0;
  *vs = v0;
}

// Weights: host threads narrow int64 -> W (int8 / int16 / int32, the
// narrowest that holds max |w|) into the pinned stage chunk by chunk,
// checking the range; each chunk's DMA and device relabel are queued as soon
// as it is converted, while the targets are still on the wire and the
// transpose sorts.  C4 (|w| <= 100) sends 1 byte per weight instead of 8.
// Queued long rows of the relabel kernels (egs_build.cuh kRelabelLong): one
// list region of `cap` rows, one counter and one length prefix (cap + 1) per
// chunk, for targets and weights.
struct LongRows {
  uint32_t* list;
  unsigned int* cnt;
  uint32_t cap;
  uint64_t* pref;
};

inline bool narrow_weights(const int64_t* in, int8_t* out, size_t k, int64_t wmax) {
  return egs_internal_narrow_i8(in, out, k, wmax);
}
inline bool narrow_weights(const int64_t* in, int16_t* out, size_t k, int64_t wmax) {
  return egs_internal_narrow_i16(in, out, k, wmax);
}
inline bool narrow_weights(const int64_t* in, int32_t* out, size_t k, int64_t wmax) {
  return egs_internal_narrow_i32(in, out, k, wmax);
}

template <class W>
bool upload_weights(egs_ctx* c, const egs_arena_view* a, const std::vector<uint32_t>& rows,
                    const std::vector<std::vector<std::pair<uint64_t, uint64_t>>>& spans,
                    std::vector<cudaEvent_t>& ew, std::vector<cudaEvent_t>& et,
                    const uint64_t* off64, void* wdev, LongRows lw, const uint8_t* key,
                    Timeline& tl) {
  cudaStream_t sc = c->copy_stream, sw = c->aux_stream;
  const int nch = (int)rows.size() - 1;
  const uint64_t m = c->m;
  // a packed record holds the weight in its top 32 - tbits bits (signed):
  // reject what does not fit there too, whatever max_abs_weight claimed
  const int64_t wmax =
      c->tbits ? std::min<int64_t>(std::numeric_limits<W>::max(), (1ll << (31 - c->tbits)) - 1)
               : (int64_t)std::numeric_limits<W>::max();
  std::lock_guard<std::mutex> lk(g_stage_mu);
  W* stage = static_cast<W*>(pinned_stage(m * sizeof(W)));
  W* wd = static_cast<W*>(wdev);
  // Blocks of kBlk edges, claimed in order from one counter by the worker
  // threads and by this thread between its DMA issues, so a descheduled
  // thread (the host may have no spare core) delays one block, not a chunk.
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const int T = m >= (1u << 20) ? (int)hw - 1 : 0;  // helpers besides this thread
  constexpr uint64_t kBlk = 1u << 18;
  // blocks of the chunks' upload spans (block b of span s of chunk k)
  struct Blk {
    uint64_t lo, hi;
    int k;
  };
  std::vector<Blk> blocks;
  std::vector<uint64_t> bfirst(nch + 1, 0);  // first block of each chunk
  for (int k = 0; k < nch; ++k) {
    for (const auto& [e0, e1] : spans[k])
      for (uint64_t lo = e0; lo < e1; lo += kBlk) blocks.push_back({lo, std::min(e1, lo + kBlk), k});
    bfirst[k + 1] = blocks.size();
  }
  const uint64_t nblk = blocks.size();
  std::vector<std::atomic<uint64_t>> left(nch);  // blocks of the chunk not yet converted
  for (int k = 0; k < nch; ++k) left[k].store(bfirst[k + 1] - bfirst[k]);
  std::atomic<uint64_t> next{0};
  std::atomic<bool> out_of_range{false};
  const int64_t* w = a->csr_weights;
  // convert one claimed block; false when none is left
  auto one_block = [&](int& k) {
    const uint64_t b = next.fetch_add(1, std::memory_order_relaxed);
    if (b >= nblk) return false;
    k = blocks[b].k;
    const uint64_t lo = blocks[b].lo, hi = blocks[b].hi;
    if (narrow_weights(w + lo, stage + lo, hi - lo, wmax)) out_of_range.store(true, std::memory_order_relaxed);
    left[k].fetch_sub(1, std::memory_order_release);
    return true;
  };
  auto work = [&]() {
    int k = 0;
    while (one_block(k)) {
    }
  };
  // The helpers (the host pool's workers, egs_pool.h) read this frame's
  // locals: on any error (a CK throw) stop them by exhausting the block
  // counter and join them before unwinding (the Job waits in its destructor,
  // declared before the Joiner so it is destroyed after it).
  egs_host::Pool::Job helpers;
  struct Joiner {
    egs_host::Pool::Job& job;
    std::atomic<uint64_t>& next;
    uint64_t nblk;
    ~Joiner() {
      next.store(nblk, std::memory_order_relaxed);
      job.wait();
    }
  } joiner{helpers, next, nblk};
  egs_host::Pool::get().launch(helpers, (unsigned)T, [&](unsigned) { work(); });
  int kself = 0;
  for (int k = 0; k < nch; ++k) {
    while (left[k].load(std::memory_order_acquire) > 0)
      if (!one_block(kself)) std::this_thread::yield();
    for (const auto& [e0, e1] : spans[k]) {
      CK(cudaMemcpyAsync(wd + e0, stage + e0, (e1 - e0) * sizeof(W), cudaMemcpyHostToDevice, sc));
      c->h2d_bytes += (e1 - e0) * sizeof(W);
    }
    CK(cudaEventRecord(ew[k], sc));
    tl.mark("copy: weights chunk " + std::to_string(k), sc);
    CK(cudaStreamWaitEvent(sw, ew[k], 0));
    // packed records: the weight bits are or-ed into the target words
    if (c->tbits) CK(cudaStreamWaitEvent(sw, et[k], 0));
    egs::k_relabel_weights<W><<<grid_for((uint64_t)(rows[k + 1] - rows[k]) * 4, c->num_sms),
                                256, 0, sw>>>(rows[k], rows[k + 1], off64, wd, c->perm, c->off,
                                              c->edge, c->tbits, lw.list + (size_t)k * lw.cap,
                                              lw.cnt + k, c->own_lo, c->own_hi);
    egs::k_long_prefix<<<1, 1024, 0, sw>>>(lw.list + (size_t)k * lw.cap, lw.cnt + k, off64,
                                           lw.pref + (size_t)k * (lw.cap + 1));
    egs::k_relabel_weights_long<W><<<2 * c->num_sms, 256, 0, sw>>>(
        lw.list + (size_t)k * lw.cap, lw.cnt + k, lw.pref + (size_t)k * (lw.cap + 1), off64, wd,
        c->perm, c->off, c->edge, c->tbits);
    tl.mark("aux: weights relabelled " + std::to_string(k), sw);
    // the chunk's player-1 light rows, complete now: sorted by weight
    if (!c->tbits) CK(cudaStreamWaitEvent(sw, et[k], 0));  // (wide: targets written apart)
    egs::k_sort_p1_rows<<<grid_for((uint64_t)(rows[k + 1] - rows[k]) * 32, c->num_sms), 256, 0,
                          sw>>>(rows[k], rows[k + 1], key, c->perm, c->off, c->edge, c->tbits,
                                c->own_lo, c->own_hi, c->rec0);
    CK(cudaGetLastError());
    tl.mark("aux: rows sorted " + std::to_string(k), sw);
  }
  helpers.wait();
  // the staging buffer is re-used by the next upload: wait for its DMA
  CK(cudaStreamSynchronize(sc));
  return out_of_range.load();
}

// Build the relabelled device arena from the reference CSR (host spans),
// pipelined with the upload: the copy stream brings offsets + owners, then
// the targets and the weights in row-range chunks of ~m/16 edges; the main
// stream classifies and relabels the vertices, and relabels each target
// chunk as it lands and sorts and ranks its transpose pairs (k_csc_runs)
// before the next one lands; the last chunk's merge (k_csc_merge) runs while
// the weights are on the wire, which host threads narrow from int64 as the
// targets go (egs_narrow.cpp); the aux stream writes each weight chunk as it
// lands.  The result is ready shortly after the last weight chunk is
// (PCIe-bound: C4's 1.42 GB take 25.6 ms at 55.6 GB/s).
// Several ranks (`plan` set): the relabelling is the plan's rank-major order
// and this rank keeps its own rows [own_lo, own_hi) only (m_own edges), with
// the transpose of those rows (the predecessors it activates).
void build_arena(egs_ctx* c, const egs_arena_view* a, const egs_part_plan* plan) {
  StepTimer tm(c->stream);
  const uint32_t n = c->n;
  const uint64_t m = c->m;
  const uint64_t mo = c->m_own;  // edges stored here (m with one rank)
  bool h_stage_bad = false;
  cudaStream_t s = c->stream, sc = c->copy_stream, sw = c->aux_stream;
  const int sms = c->num_sms;
  DevBuf d_off64, d_dst, d_wn, d_owner, d_key, d_tcount, d_misc, d_ck0, d_cv0, d_ck1,
      d_long, d_lpref, d_cv1, d_rel, d_cnt, d_rb, d_stmp;
  uint64_t* off64 = d_off64.alloc<uint64_t>((size_t)n + 1);
  uint32_t* dst = d_dst.alloc<uint32_t>(m);
  void* wn = d_wn.alloc<int32_t>(m);  // narrowed weights (int8/16/32)
  uint8_t* owner = d_owner.alloc<uint8_t>(n);
  // [0..15] class histogram, [16] bad, [32..63] long-row counters (targets,
  // weights) of the 16 chunks
  unsigned int* misc = d_misc.alloc<unsigned int>(64);
  // row-range chunks of ~m/16 edges (host offsets are at hand)
  constexpr int kChunks = 16;
  static_assert(kChunks <= egs::kMaxChunks, "k_csc_merge's chunk table");
  std::vector<uint32_t> rows{0};
  for (int k = 1; k < kChunks; ++k) {
    const uint64_t target = m * (uint64_t)k / kChunks;
    const uint64_t* it = std::lower_bound(a->csr_offsets, a->csr_offsets + n + 1, target);
    const uint32_t r = (uint32_t)std::min<uint64_t>(n, it - a->csr_offsets);
    if (r > rows.back()) rows.push_back(r);
  }
  if (rows.back() < n) rows.push_back(n);
  const int nch = (int)rows.size() - 1;
  uint64_t max_chunk = 0;
  for (int k = 0; k < nch; ++k)
    max_chunk = std::max<uint64_t>(max_chunk, a->csr_offsets[rows[k + 1]] - a->csr_offsets[rows[k]]);
  const uint32_t long_cap = (uint32_t)(max_chunk / egs::kRelabelLong + 1);
  uint32_t* long_lists = d_long.alloc<uint32_t>((size_t)2 * 16 * long_cap);
  uint64_t* long_pref = d_lpref.alloc<uint64_t>((size_t)2 * 16 * (long_cap + 1));
  const LongRows lt{long_lists, misc + 32, long_cap, long_pref};
  const LongRows lw{long_lists + (size_t)16 * long_cap, misc + 48, long_cap,
                    long_pref + (size_t)16 * (long_cap + 1)};
  uint8_t* key = d_key.alloc<uint8_t>(n);
  const uint32_t vtiles = (uint32_t)((n + egs::kScanTile - 1) / egs::kScanTile);
  uint32_t* tcount = d_tcount.alloc<uint32_t>((size_t)egs::kNumClasses * vtiles);
  c->inv = dalloc<uint32_t>(n);
  uint32_t* inv = c->inv;
  uint32_t* ck0 = d_ck0.alloc<uint32_t>(mo);
  uint32_t* cv0 = d_cv0.alloc<uint32_t>(mo);
  uint32_t* ck1 = d_ck1.alloc<uint32_t>(mo);
  // transpose: chunk by chunk during the upload (k_csc_runs), or one sort of
  // all pairs at the end.  Chunk by chunk pays when the end sort would be on
  // the critical path after the last transfer, i.e. for large arenas (C4,
  // 2.56e8 edges: one-shot 34.9 -> 31.8 ms); below kIncTransposeMinEdges the
  // 16 per-chunk sorts cost more than they hide (C2 / C5: +0.8 ms, C3 even).
  // Several ranks always sort at the end (a rank's own rows are not
  // chunk-contiguous).  EGS_CSC_SORT=inc | end (CUB) | radix (egs_scan.cuh)
  // forces a method.
  constexpr uint64_t kIncTransposeMinEdges = 1ull << 27;
  const char* csc_sort = std::getenv("EGS_CSC_SORT");
  const bool csc_inc = c->runs.empty() && mo > 0 &&
                       (csc_sort ? std::strcmp(csc_sort, "inc") == 0
                                 : mo >= kIncTransposeMinEdges);
  uint32_t *cv1 = nullptr, *rel = nullptr, *ccnt = nullptr;
  uint2* rb = nullptr;
  if (csc_inc) {
    cv1 = d_cv1.alloc<uint32_t>(mo);
    rel = d_rel.alloc<uint32_t>(mo);
    ccnt = d_cnt.alloc<uint32_t>((size_t)n + 1);
    rb = d_rb.alloc<uint2>(n);
  }
  c->perm = dalloc<uint32_t>(n);
  c->off = dalloc<uint32_t>((size_t)n + 1);
  // packed 4-byte records when every weight fits beside the target bits
  // (EGS_EDGE_FORMAT=8 forces the 8-byte format)
  {
    const uint32_t tb = bits_for(n);  // ids < n fit tb bits
    const char* fmt = std::getenv("EGS_EDGE_FORMAT");
    const bool wide = fmt && std::atoi(fmt) == 8;
    c->tbits = (!wide && tb <= 24 && a->max_abs_weight < (1ll << (31 - tb))) ? tb : 0;
  }
  // +16 bytes: 16-byte rounding of TMA spans
  c->edge = dalloc<uint8_t>(mo * rec_bytes(c) + 16);
  c->rec0 = dalloc<uint8_t>((size_t)n * rec_bytes(c));
  c->csrc = dalloc<uint32_t>(mo);
  c->coff = dalloc<uint32_t>((size_t)n + 1);
  CK(cudaMemsetAsync(misc, 0, 64 * sizeof(unsigned int), s));
  if (csc_inc) CK(cudaMemsetAsync(ccnt, 0, ((size_t)n + 1) * sizeof(uint32_t), s));
  tm.mark("pool allocations");
  cudaEvent_t e_alloc, e_vert, e_perm, e_tail;
  CK(cudaEventCreateWithFlags(&e_alloc, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e_vert, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e_perm, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e_tail, cudaEventDisableTiming));
  CK(cudaEventRecord(e_alloc, s));
  Timeline tl;
  tl.mark("start", s);
  CK(cudaStreamWaitEvent(sc, e_alloc, 0));
  CK(cudaStreamWaitEvent(sw, e_alloc, 0));

  std::vector<cudaEvent_t> ex(nch), ew(nch), et(nch);
  for (int k = 0; k < nch; ++k) {
    CK(cudaEventCreateWithFlags(&ex[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ew[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&et[k], cudaEventDisableTiming));
  }
  // the edge ranges each chunk uploads: the chunk's whole span, or (sharded
  // multi-GPU upload) its intersection with this rank's row runs -- rows of
  // other ranks never cross PCIe (the relabel kernels skip them)
  std::vector<std::vector<std::pair<uint64_t, uint64_t>>> spans(nch);
  {
    size_t ri = 0;
    for (int k = 0; k < nch; ++k) {
      if (c->runs.empty()) {
        spans[k].emplace_back(a->csr_offsets[rows[k]], a->csr_offsets[rows[k + 1]]);
        continue;
      }
      while (ri < c->runs.size() && c->runs[ri].second <= rows[k]) ++ri;
      for (size_t j = ri; j < c->runs.size() && c->runs[j].first < rows[k + 1]; ++j) {
        const uint32_t v0 = std::max(c->runs[j].first, rows[k]);
        const uint32_t v1 = std::min(c->runs[j].second, rows[k + 1]);
        if (v1 > v0) spans[k].emplace_back(a->csr_offsets[v0], a->csr_offsets[v1]);
      }
    }
  }
  c->h2d_bytes = ((uint64_t)n + 1) * 8 + n;

  // upload: vertices, then targets, then weights
  CK(cudaMemcpyAsync(off64, a->csr_offsets, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, sc));
  CK(cudaMemcpyAsync(owner, a->owners, n, cudaMemcpyHostToDevice, sc));
  CK(cudaEventRecord(e_vert, sc));
  tl.mark("copy: vertices landed", sc);
  for (int k = 0; k < nch; ++k) {
    for (const auto& [e0, e1] : spans[k]) {
      CK(cudaMemcpyAsync(dst + e0, a->csr_targets + e0, (e1 - e0) * 4, cudaMemcpyHostToDevice, sc));
      c->h2d_bytes += (e1 - e0) * 4;
    }
    CK(cudaEventRecord(ex[k], sc));
    tl.mark("copy: targets chunk " + std::to_string(k), sc);
  }

  // vertices: class keys and per-tile class counts, their scan, the stable
  // class placement (mapped through the plan with several ranks), row
  // lengths in the new order and their scan = the relabelled offsets
  CK(cudaStreamWaitEvent(s, e_vert, 0));
  const uint32_t vgrid = std::min<uint32_t>(vtiles, (uint32_t)sms * 8);
  egs::k_class_tiles<<<vgrid, egs::kScanThreads, 0, s>>>(n, off64, owner, key, tcount, vtiles,
                                                          misc);
  CK(cudaGetLastError());
  dev_excl_scan<uint32_t>(tcount, tcount, (uint64_t)egs::kNumClasses * vtiles, s, sms);
  {
    egs::PlanDev pl{};
    pl.world = plan ? plan->world : 1;
    if (plan)
      for (int k = 0; k < egs::kNumClasses; ++k)
        for (uint32_t r = 0; r < plan->world; ++r) {
          for (int j = 0; j <= 1; ++j) pl.piece[k][r + j] = plan->piece[k][r + j];
          pl.cls_lo[r][k] = plan->class_lo[r][k];
        }
    egs::k_class_place<<<vgrid, egs::kScanThreads, 0, s>>>(n, key, tcount, vtiles, pl, c->perm,
                                                            inv);
  }
  egs::k_row_lengths<<<grid_for(n, sms), 256, 0, s>>>(n, inv, off64, c->own_lo, c->own_hi,
                                                      c->off);
  CK(cudaGetLastError());
  dev_excl_scan<uint32_t>(c->off, c->off, (uint64_t)n + 1, s, sms);
  CK(cudaEventRecord(e_perm, s));
  tl.mark("main: vertex relabel done", s);
  tm.mark("vertices (classify, sort, offsets)");

  // the incremental transpose's sort temporaries, sized for the largest chunk
  void* sort_tmp = nullptr;
  size_t sort_tb = 0;
  // The chunk sorts are the hand-written stable LSD radix sort (egs_scan.cuh)
  // by default -- hidden under the transfer, so the library sort's speed buys
  // nothing there; EGS_CSC_CHUNK_SORT=cub selects CUB's onesweep.
  const char* chunk_sort = std::getenv("EGS_CSC_CHUNK_SORT");
  const bool chunk_cub = chunk_sort && std::strcmp(chunk_sort, "cub") == 0;
  uint32_t *sk = ck1, *sv = cv1;  // where the sorted chunks end up (the same for every chunk)
  if (csc_inc && chunk_cub) {
    uint64_t maxlen = 0;
    for (int k = 0; k < nch; ++k)
      maxlen = std::max<uint64_t>(maxlen, a->csr_offsets[rows[k + 1]] - a->csr_offsets[rows[k]]);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, sort_tb, ck0, ck1, cv0, cv1, (int64_t)maxlen, 0,
                                       bits_for(n), s));
    sort_tmp = d_stmp.alloc<uint8_t>(sort_tb);
  }

  // targets as they land (main stream); with the incremental transpose each
  // chunk's pairs are sorted and ranked before the next chunk lands
  for (int k = 0; k < nch; ++k) {
    CK(cudaStreamWaitEvent(s, ex[k], 0));
    egs::k_relabel_targets<<<grid_for((uint64_t)(rows[k + 1] - rows[k]) * 4, sms), 256, 0, s>>>(
        n, rows[k], rows[k + 1], off64, dst, c->perm, c->off, c->edge, c->tbits, ck0, cv0,
        misc + 16, lt.list + (size_t)k * lt.cap, lt.cnt + k, c->own_lo, c->own_hi, csc_inc);
    egs::k_long_prefix<<<1, 1024, 0, s>>>(lt.list + (size_t)k * lt.cap, lt.cnt + k, off64,
                                          lt.pref + (size_t)k * (lt.cap + 1));
    egs::k_relabel_targets_long<<<2 * sms, 256, 0, s>>>(
        n, lt.list + (size_t)k * lt.cap, lt.cnt + k, lt.pref + (size_t)k * (lt.cap + 1), off64,
        dst, c->perm, c->off, c->edge, c->tbits, ck0, cv0, misc + 16, csc_inc);
    CK(cudaGetLastError());
    CK(cudaEventRecord(et[k], s));
    tl.mark("main: targets relabelled " + std::to_string(k), s);
    if (csc_inc) {
      const uint64_t e0 = a->csr_offsets[rows[k]], len = a->csr_offsets[rows[k + 1]] - e0;
      if (len == 0) continue;
      if (chunk_cub) {
        CK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_tb, ck0 + e0, ck1 + e0, cv0 + e0,
                                           cv1 + e0, (int64_t)len, 0, bits_for(n), s));
      } else {
        uint32_t *ks = nullptr, *vs = nullptr;
        dev_radix_sort_pairs(ck0 + e0, cv0 + e0, ck1 + e0, cv1 + e0, len, bits_for(n), s, sms,
                             &ks, &vs);
        sk = ks - e0;  // (an odd digit count ends in ck1 / cv1, an even one in ck0 / cv0)
        sv = vs - e0;
      }
      egs::k_csc_runs<<<grid_for(len, sms), 256, 0, s>>>(sk + e0, len, ccnt, rb);
      egs::k_csc_rel<<<grid_for(len, sms), 256, 0, s>>>(sk + e0, len, rb, ccnt, rel + e0);
      CK(cudaGetLastError());
      tl.mark("main: transpose chunk " + std::to_string(k), s);
    }
  }

  if (csc_inc) {
    dev_excl_scan<uint32_t>(ccnt, c->coff, (uint64_t)n + 1, s, sms);
    egs::ChunkStarts cs{};
    cs.nch = nch;
    for (int k = 0; k <= nch; ++k) cs.e[k] = a->csr_offsets[rows[k]];
    // one CTA per span (not a persistent grid): CTAs retire as they finish,
    // so the weight chunks' kernels on the higher-priority aux stream get SMs
    // while the merge runs
    const uint64_t spans_n = (mo + egs::kMergeSpan - 1) / egs::kMergeSpan;
    egs::k_csc_merge<<<(uint32_t)spans_n, 512, 0, s>>>(sk, sv, rel, mo, c->coff, cs, c->csrc);
    CK(cudaGetLastError());
  } else {
    // transpose: stable radix sort of the (dst, src) pairs by dst while the
    // weights stream in
    uint32_t *ks = nullptr, *vs = nullptr;
    // CUB's onesweep radix sort, or the hand-written LSD sort (egs_scan.cuh,
    // EGS_CSC_SORT=radix) -- measured on one box, C4 one-shot e2e 34.5 ms vs
    // 46 ms: onesweep's single pass per digit is ~2x faster than the per-tile
    // histogram + scan + scatter passes.  Both are stable, so the transpose
    // is the same (columns in ascending relabelled source order).
    if (csc_sort && std::strcmp(csc_sort, "radix") == 0) {
      dev_radix_sort_pairs(ck0, cv0, ck1, c->csrc, mo, bits_for(n), s, sms, &ks, &vs);
    } else if (mo > 0) {
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ck0, ck1, cv0, c->csrc, mo, 0, bits_for(n), s));
      DevBuf d_tmp;
      void* tmp = d_tmp.alloc<uint8_t>(tb);
      CK(cub::DeviceRadixSort::SortPairs(tmp, tb, ck0, ck1, cv0, c->csrc, mo, 0, bits_for(n), s));
      ks = ck1;
      vs = c->csrc;
    } else {
      ks = ck1;
      vs = c->csrc;
    }
    if (vs != c->csrc) CK(cudaMemcpyAsync(c->csrc, vs, mo * 4, cudaMemcpyDeviceToDevice, s));
    egs::k_col_offsets<<<grid_for(mo + 1, sms), 256, 0, s>>>(n, mo, ks, c->coff);
  }
  tl.mark("main: transpose done", s);
  CK(cudaGetLastError());

  CK(cudaStreamWaitEvent(sw, e_perm, 0));
  {
    const int64_t mw = a->max_abs_weight;
    if (mw <= 127)
      h_stage_bad = upload_weights<int8_t>(c, a, rows, spans, ew, et, off64, wn, lw, key, tl);
    else if (mw <= 32767)
      h_stage_bad = upload_weights<int16_t>(c, a, rows, spans, ew, et, off64, wn, lw, key, tl);
    else
      h_stage_bad = upload_weights<int32_t>(c, a, rows, spans, ew, et, off64, wn, lw, key, tl);
  }
  tm.mark("upload + relabel + CSC sort");
  CK(cudaEventRecord(e_tail, sw));
  tl.mark("aux: weights relabelled, rows sorted", sw);
  CK(cudaStreamWaitEvent(s, e_tail, 0));
  unsigned int h_misc[32] = {0};
  CK(cudaMemcpyAsync(h_misc, misc, sizeof(h_misc), cudaMemcpyDeviceToHost, s));
  // temporaries go back to the pool in stream order
  d_off64.release();
  d_dst.release();
  d_wn.release();
  d_owner.release();
  d_key.release();
  d_tcount.release();
  d_ck0.release();
  d_cv0.release();
  d_ck1.release();
  d_misc.release();
  d_long.release();
  d_lpref.release();
  d_cv1.release();
  d_rel.release();
  d_cnt.release();
  d_rb.release();
  d_stmp.release();
  CK(cudaStreamSynchronize(s));
  tl.mark("main: joined", s);
  tm.mark("weights + join");
  for (auto e : ex) cudaEventDestroy(e);
  for (auto e : ew) cudaEventDestroy(e);
  for (auto e : et) cudaEventDestroy(e);
  cudaEventDestroy(e_alloc);
  cudaEventDestroy(e_vert);
  cudaEventDestroy(e_perm);
  cudaEventDestroy(e_tail);
  const unsigned int bad = h_misc[16] | (h_stage_bad ? 1u : 0u);
  if (bad & 1u)
    throw Fail(a->max_abs_weight > 2147483647LL ? EGS_ERR_UNSUPPORTED : EGS_ERR_INVALID_CONFIG,
               "edge weight outside int32 on the device path, or beyond max_abs_weight");
  if (bad & 2u) throw Fail(EGS_ERR_INVALID_CONFIG, "edge target out of range");
  if (plan) {  // this rank's class ranges
    for (int k = 0; k <= egs::kNumClasses; ++k) c->rb[k] = plan->class_lo[c->rank][k];
  } else {
    c->rb[0] = 0;
    for (int k = 0; k < egs::kNumClasses; ++k) c->rb[k + 1] = c->rb[k] + h_misc[k];
  }
}

std::vector<std::pair<uint32_t, uint32_t>> rank_runs(const egs_arena_view* a,
                                                     const egs_part_plan& pl, int rank);

egs_ctx* ctx_create(const egs_arena_view* a, const egs_gpu_opts& opts, egs_gpu_stats* st,
                    int rank = 0, int world = 1, const egs_part_plan* plan = nullptr) {
  {
    egs_gpu_opts o1 = opts;
    if (world > 1) o1.n_gpus = 1;  // (n_gpus == world checked by egs_part_create)
    validate_opts(o1);
  }
  if (!a) throw Fail(EGS_ERR_INVALID_CONFIG, "null arena");
  if (a->num_edges >= 0xFFFFFFFFull)
    throw Fail(EGS_ERR_UNSUPPORTED, "arenas with >= 2^32 edges are not supported on the device");
  if (a->num_vertices > 0 && a->num_edges < a->num_vertices)
    throw Fail(EGS_ERR_INVALID_CONFIG, "arena is not total");
  if (a->credit_cap < 0) throw Fail(EGS_ERR_INVALID_CONFIG, "negative credit_cap");
  if (a->max_abs_weight > 2147483647LL)
    throw Fail(EGS_ERR_UNSUPPORTED, "edge weights beyond int32 are not supported on the device");
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
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device));
    if (!coop) throw Fail(EGS_ERR_CUDA, "device does not support cooperative launch");
    StepTimer tm0(nullptr);
    use_caching_pool(c->device);
    Shell shell;
    if (shell_get(c->device, shell)) {
      c->stream = shell.stream;
      c->copy_stream = shell.copy_stream;
      c->aux_stream = shell.aux_stream;
      c->ev[0] = shell.ev[0];
      c->ev[1] = shell.ev[1];
      c->h_ctr = shell.h_ctr;
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
      {  // the weight chunks' kernels outrank the transpose merge (build_arena)
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c->aux_stream, cudaStreamNonBlocking, hi));
      }
      for (auto& e : c->ev) CK(cudaEventCreate(&e));
      CK(cudaMallocHost(&c->h_ctr, egs::kNumCounters * sizeof(unsigned long long)));
    }
    g_alloc_stream = c->stream;
    c->n = a->num_vertices;
    c->m = a->num_edges;
    c->cap = a->credit_cap;
    // u32 values keep top = 2^32-1 and the top bit free for the
    // certificate's candidate mark (egs_solve.cuh CandFlag): every finite
    // credit <= credit_cap must stay below 2^31 - 1
    c->vbits = a->credit_cap < 0x7FFFFFFFLL ? 32 : 64;
    const uint32_t n = c->n;
    const size_t vsz = c->vbits / 8;
    const size_t words = ((size_t)n + 31) / 32;

    tm0.mark("create: streams, events, pinned");
    c->ctr = dalloc<unsigned long long>(egs::kNumCounters);
    if (std::getenv("EGS_TRACE")) c->trace = dalloc<unsigned long long>(egs::kTraceCap);
    c->scratch = dalloc<egs::Scratch>(1);
    c->rank = rank;
    c->world = world;
    c->own_lo = plan ? plan->rank_lo[rank] : 0;
    c->own_hi = plan ? plan->rank_lo[rank + 1] : n;
    c->m_own = plan ? plan->edges[rank] : c->m;
    if (plan && world > 1 && std::getenv("EGS_FULL_UPLOAD") == nullptr)
      c->runs = rank_runs(a, *plan, rank);
    if (world == 1) {
      c->f = dalloc<uint8_t>((size_t)std::max<uint32_t>(n, 1) * vsz);
      c->chg[0] = dalloc<uint32_t>(words);
      c->chg[1] = dalloc<uint32_t>(words);
      c->rbm[0] = dalloc<uint32_t>(words);
      c->rbm[1] = dalloc<uint32_t>(words);
    } else {
      // the replicated state: plain cudaMalloc (IPC-exportable), one block
      auto up = [](size_t x) { return (x + 255) / 256 * 256; };
      const size_t fb = up(std::max<size_t>(n, 1) * vsz), wb = up(std::max<size_t>(words, 1) * 4);
      c->xbytes = fb + 4 * wb + up(sizeof(egs::XSync));
      c->xbuf = xbuf_take(c->device, c->xbytes);
      CK(cudaMemsetAsync(c->xbuf, 0, c->xbytes, c->stream));
      c->f = c->xbuf;
      c->chg[0] = reinterpret_cast<uint32_t*>(c->xbuf + fb);
      c->chg[1] = reinterpret_cast<uint32_t*>(c->xbuf + fb + wb);
      c->rbm[0] = reinterpret_cast<uint32_t*>(c->xbuf + fb + 2 * wb);
      c->rbm[1] = reinterpret_cast<uint32_t*>(c->xbuf + fb + 3 * wb);
      c->xsync = reinterpret_cast<egs::XSync*>(c->xbuf + fb + 4 * wb);
      c->xpeer[rank] = c->xbuf;
    }
    c->frb[0] = dalloc<uint32_t>(words);
    c->frb[1] = dalloc<uint32_t>(words);
    c->cbm[0] = dalloc<uint32_t>(words);
    c->cbm[1] = dalloc<uint32_t>(words);
    c->cand = dalloc<uint32_t>(words);
    CK(cudaMemsetAsync(c->cand, 0, std::max<size_t>(words, 1) * 4, c->stream));
    // every cascade leaves the ring empty again (egs_solve.cuh)
    c->ring_cap = n + egs::kRingSlack;
    c->ring = dalloc<uint32_t>(c->ring_cap);
    CK(cudaMemsetAsync(c->ring, 0xFF, (size_t)c->ring_cap * 4, c->stream));
    // at most m / kLongCol columns are longer than kLongCol
    c->longcol = dalloc<uint32_t>(2 * (a->num_edges / egs::kLongCol + 1));
    c->fr[0] = dalloc<uint32_t>(n);
    c->fr[1] = dalloc<uint32_t>(n);
    c->stage = dalloc<uint8_t>((size_t)std::max<uint32_t>(n, 1) * vsz);
    // dense commits read every slot of a bitmap word (egs_solve.cuh
    // commit_stage_loads): slots never staged are read, and must be defined
    CK(cudaMemsetAsync(c->stage, 0, (size_t)std::max<uint32_t>(n, 1) * vsz, c->stream));
    c->f64 = dalloc<int64_t>(n);
    tm0.s = c->stream;
    tm0.mark("create: state buffers");
    if (n > 0) {
      build_arena(c, a, plan);
    } else {
      c->off = dalloc<uint32_t>(1);
      c->coff = dalloc<uint32_t>(1);
      c->edge = dalloc<uint8_t>(16);
      c->rec0 = dalloc<uint8_t>(16);
      c->csrc = dalloc<uint32_t>(1);
      c->perm = dalloc<uint32_t>(1);
      c->inv = dalloc<uint32_t>(1);
    }
    c->wit = dalloc<int2>(std::max<uint32_t>(1, c->rb[egs::kP1L]));

    // Persistent grid: every CTA co-resident (cooperative launch).
    int per_sm = 0;
    const void* kfn = solve_kernel(c);
    CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)egs::kLiftSmemBytes));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, egs::kBlock,
                                                     egs::kLiftSmemBytes));
    if (per_sm < 1) throw Fail(EGS_ERR_CUDA, "solve kernel cannot be resident");
    const int full = per_sm * c->num_sms;
    int want = opts.grid_ctas > 0 ? opts.grid_ctas
                                  : (int)std::min<uint64_t>(full, std::max<uint64_t>(
                                        1, ((uint64_t)n + egs::kBlock - 1) / egs::kBlock));
    if (const char* e = std::getenv("EGS_GRID")) want = std::atoi(e);
    c->grid = std::max(1, std::min(want, full));
    c->full_grid = full;

    // Keep the measure resident in L2 while the edge stream goes through.
    // (A re-used stream may still carry the window of a previous context.)
    {
      cudaStreamAttrValue none{};
      cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &none);
      cudaGetLastError();
    }
    int max_win = 0;
    const bool want_win = std::getenv("EGS_NO_L2WIN") == nullptr;
    if (want_win &&
        cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, c->device) ==
            cudaSuccess &&
        max_win > 0 && n > 0) {
      int persist_max = 0;
      cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, c->device);
      const size_t fbytes = (size_t)n * vsz;
      const size_t win = std::min<size_t>(fbytes, (size_t)max_win);
      if (persist_max > 0) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, persist_max));
        cudaStreamAttrValue attr{};
        attr.accessPolicyWindow.base_ptr = c->f;
        attr.accessPolicyWindow.num_bytes = win;
        attr.accessPolicyWindow.hitRatio =
            std::min(1.0f, (float)std::min<size_t>(win, persist_max) / (float)win);
        attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
      }
      cudaGetLastError();  // the window is a hint; never fail on it
    }
    tm0.mark("create: occupancy, L2 window");
    if (st) {
      st->h2d_bytes = c->h2d_bytes;
      st->upload_seconds = secs_since(t0);
      st->value_bits = (uint32_t)c->vbits;
      st->grid_ctas = (uint32_t)c->grid;
      st->edge_bytes = (uint32_t)rec_bytes(c);
    }
    return c;
  } catch (...) {
    ctx_free(c);
    throw;
  }
}

template <class V>
egs::SolveParams<V> make_params(egs_ctx* c, unsigned long long* budget_out) {
  const uint32_t n = c->n;
  const egs_gpu_opts& o = c->opts;
  const uint32_t szL = (c->rb[1] - c->rb[0]) + (c->rb[4] - c->rb[3]);
  const uint32_t szM = (c->rb[2] - c->rb[1]) + (c->rb[5] - c->rb[4]);
  egs::SolveParams<V> p{};
  p.g = c->graph();
  p.f = static_cast<V*>(c->f);
  p.wit = c->wit;
  p.chg[0] = c->chg[0];
  p.chg[1] = c->chg[1];
  p.frb[0] = c->frb[0];
  p.frb[1] = c->frb[1];
  p.rbm[0] = c->rbm[0];
  p.rbm[1] = c->rbm[1];
  p.cbm[0] = c->cbm[0];
  p.cbm[1] = c->cbm[1];
  p.cand = c->cand;
  p.longcol = c->longcol;
  p.fr[0] = c->fr[0];
  p.fr[1] = c->fr[1];
  p.cbase[0] = 0;
  p.cbase[1] = szL;
  p.cbase[2] = szL + szM;
  p.stage = static_cast<V*>(c->stage);
  p.sh = c->scratch;
  p.ctr = c->ctr;
  p.trace = c->trace;
  p.mode = o.mode;
  p.use_tma = o.no_tma ? 0 : kDefaultTma;
  if (const char* e = std::getenv("EGS_TMA_MASK")) p.use_tma = std::atoi(e) & egs::kTmaAll;
  // the candidate mark needs a free top bit: u64 values with credit_cap at
  // INT64_MAX (a saturated cap) solve without the certificate (still exact)
  p.certify = o.certify && !(c->vbits == 64 && c->cap >= INT64_MAX - 1);
  p.cert_interval = o.cert_interval > 0 ? o.cert_interval : 1;
  // defaults measured over the five configs (profiles/r02_knobs.jsonl):
  // sparse_div 4 -> 8 and cert_growth 4 -> 8 take C4 1.459 -> 1.391 ms,
  // C2 0.574 -> 0.537, C5 0.652 -> 0.626, C3 3.24 -> 3.28
  p.cert_growth = o.cert_growth > 0 ? o.cert_growth : 8;
  p.sparse_div = o.sparse_div > 0 ? (uint32_t)o.sparse_div : 8u;
  p.cert_sparse_div = (float)p.sparse_div;
  if (const char* e = std::getenv("EGS_CERT_SPARSE_DIV")) p.cert_sparse_div = (float)std::atof(e);
  p.avg_in_deg = n ? (float)((double)c->m / (double)n) : 1.0f;
  if (p.avg_in_deg < 1.0f) p.avg_in_deg = 1.0f;
  // default budget |E|*(cap+1)+1 (solver_par.cpp:94-98), saturating
  unsigned long long budget = o.round_bound;
  if (!o.has_round_bound && !budget) {
    const unsigned long long per = (unsigned long long)c->cap + 1ull;
    budget = (c->m && per > ~0ull / c->m) ? ~0ull : c->m * per + 1ull;
  }
  p.round_budget = budget;
  // round 1 straight into f (one rank), marking the first attempt's
  // candidates when the attempt follows round 1 (EGS_R1_DIRECT=0: staged)
  {
    const char* e = std::getenv("EGS_R1_DIRECT");
    p.r1_direct = c->world == 1 && (e ? std::atoi(e) != 0 : true);
    p.r1_cand = p.r1_direct && p.certify && p.cert_interval <= 1 && p.round_budget > 1;
  }
  p.timeout_ns = o.timeout_seconds > 0 ? (unsigned long long)(o.timeout_seconds * 1e9) : 0ull;
  p.own_lo = c->world == 1 ? 0 : c->own_lo;
  p.own_hi = c->world == 1 ? n : c->own_hi;
  p.debug = o.debug_checks ? 1 : 0;
  p.no_fuse = std::getenv("EGS_NO_FUSE") != nullptr;
  {
    const char* e = std::getenv("EGS_CERT_CASCADE");
    p.cascade = !(e && std::atoi(e) == 0);
  }
  p.ring = c->ring;
  p.ring_cap = c->ring_cap;
  p.world = c->world;
  p.rank = c->rank;
  if (c->world > 1) {
    p.xbase = c->xbuf;
    for (int q = 0; q < c->world; ++q) p.xpeer[q] = c->xpeer[q];
    p.xsync = c->xsync;
    p.epoch0 = c->epoch;
    p.xwait_ns = (unsigned long long)((o.timeout_seconds > 0 ? o.timeout_seconds : 60.0) * 1e9);
  }
  if (budget_out) *budget_out = budget;
  return p;
}

// SolveReport-style counters from the device counter block (algorithmic
// bytes as defined in DESIGN.md §4).
template <class V>
void fill_stats(egs_ctx* c, const unsigned long long* h, double ms, egs_gpu_stats* st) {
  const uint32_t n = c->n;
  const size_t words = ((size_t)n + 31) / 32;
  const double sv = sizeof(V);
  // SURVEY §8(d)'s per-unit figure: an 8-byte {u32 dst, i32 w} record per
  // edge, whatever the stored format (packed arenas stream 4 bytes; the
  // bench's `traffic` is the measured DRAM side).  The lift-phase figure
  // counts records at their stored size instead (`erl`).
  const double er = 8.0;
  const double erl = (double)rec_bytes(c);
  st->lifts = h[egs::kLifts];
  st->applications = h[egs::kApps];
  st->edges_relaxed = h[egs::kEdges];
  st->witness_checks = h[egs::kWitness];
  st->activations = h[egs::kActScanned];
  st->certified = h[egs::kCertified];
  st->pops = h[egs::kPops];
  st->visits = h[egs::kVisits];
  st->cert_rows = h[egs::kCertScanned];
  st->cert_edges = h[egs::kCertEdges];
  st->rounds = h[egs::kRounds];
  st->dense_rounds = h[egs::kDenseRounds];
  st->sparse_rounds = h[egs::kSparseRounds];
  st->cert_attempts = h[egs::kCertAttempts];
  st->cert_passes = h[egs::kCertPasses];
  st->solve_seconds = ms * 1e-3;
  st->seed_seconds = h[egs::kTimeSeed] * 1e-9;
  st->lift_seconds = h[egs::kTimeLift] * 1e-9;
  st->cert_seconds = h[egs::kTimeCert] * 1e-9;
  st->activate_seconds = h[egs::kTimeAct] * 1e-9;
  // Algorithmic bytes: what each phase must move at least.
  // round 1 (counted as one dense round: n visits, m edges) reads records
  // but neither f(v) nor f(t): drop those gathers from the lift formula
  // (a partition rank: its own rows and vertices)
  const double r1 = (double)c->m_own * sv + (double)(c->own_hi - c->own_lo) * sv;
  auto lift_with = [&](double rec) {
    return (double)st->visits * sv + (double)st->witness_checks * (rec + sv) +
           (double)st->applications * 8 + (double)st->edges_relaxed * (rec + sv) +
           (double)st->lifts * sv - (st->rounds ? r1 : 0.0);
  };
  const double lift = lift_with(er);
  const double seed = 0.0;
  const double cert = (double)st->cert_attempts * n * (2 * (sv + 1)) +
                      (double)st->cert_rows * (1 + sv + 8) +
                      (double)st->cert_edges * (er + sv + 1);
  const double act = (double)st->activations * (4 + sv) + (double)st->sparse_rounds * words * 4;
  st->lift_bytes = (uint64_t)lift_with(erl);
  st->algo_bytes = (uint64_t)(lift + seed + cert + act);
  st->algo_bytes_s8d = (uint64_t)((double)st->edges_relaxed * (8.0 + sv) +
                                  (double)st->applications * (4.0 + 2.0 * sv) +
                                  (double)st->activations * 4.0);
  st->kernel_launches = 1;
  for (int k = 0; k < 5; ++k)
    st->lift_sub_seconds[k] = h[egs::kSubHeavy + k] * 1e-9 / (double)c->grid;
  for (int k = 0; k < 5; ++k) st->phase_detail_seconds[k] = h[egs::kFineCommit + k] * 1e-9;
  st->value_bits = (uint32_t)c->vbits;
  st->grid_ctas = (uint32_t)c->grid;
  st->edge_bytes = (uint32_t)rec_bytes(c);
}

// debug_checks after a solve: no commit published a value that did not rise
// (the device flag Scratch::bad, the reference's check_monotone), and the
// result is a fixpoint of the capped lift (k_fixpoint); InternalInvariantError
// otherwise (solver_par.cpp:116-124).
template <class V>
void debug_verify(egs_ctx* c) {
  cudaStream_t s = c->stream;
  g_alloc_stream = s;
  DevBuf d_misc;
  unsigned long long* misc = d_misc.alloc<unsigned long long>(4);
  CK(cudaMemsetAsync(misc, 0, 4 * sizeof(unsigned long long), s));
  // (a partition rank's transpose covers its own rows only, as its CSR does)
  egs::k_csc_check<<<grid_for((uint64_t)c->n * 32, c->num_sms), 256, 0, s>>>(c->graph(), misc + 1);
  egs::k_widen<V><<<grid_for(c->n, c->num_sms), 256, 0, s>>>(c->n, static_cast<const V*>(c->f),
                                                              c->f64);
  egs::k_fixpoint<<<grid_for((uint64_t)c->n * 32, c->num_sms), 256, 0, s>>>(c->graph(), c->f64,
                                                                            misc);
  CK(cudaGetLastError());
  unsigned long long h[4] = {0, 0, 0, 0};
  unsigned int bad = 0;
  CK(cudaMemcpyAsync(h, misc, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&bad, &c->scratch->bad, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad) throw Fail(EGS_ERR_INTERNAL, "measure decreased across a round");
  if (h[1] != h[2] || h[3])
    throw Fail(EGS_ERR_INTERNAL, "the transpose does not hold the arena's edges");
  // (a partition rank holds its own rows only: the fixpoint test is the
  // single-GPU context's)
  if (h[0] && c->world == 1)
    throw Fail(EGS_ERR_INTERNAL,
               std::to_string(h[0]) + " vertices are not a fixpoint of the lift after the solve");
}

template <class V>
void run_solve(egs_ctx* c, egs_gpu_stats* st) {
  cudaStream_t s = c->stream;
  const uint32_t n = c->n;
  const size_t words = ((size_t)n + 31) / 32;
  unsigned long long budget = 0;
  egs::SolveParams<V> p = make_params<V>(c, &budget);

  CK(cudaEventRecord(c->ev[0], s));
  if (c->world == 1) {  // several ranks: k_solve resets the replicated state itself
    CK(cudaMemsetAsync(c->f, 0, (size_t)n * sizeof(V), s));
    CK(cudaMemsetAsync(c->chg[0], 0, words * 4, s));
    CK(cudaMemsetAsync(c->chg[1], 0, words * 4, s));
  }
  CK(cudaMemsetAsync(c->frb[0], 0, words * 4, s));
  CK(cudaMemsetAsync(c->frb[1], 0, words * 4, s));
  CK(cudaMemsetAsync(c->cbm[0], 0, words * 4, s));
  CK(cudaMemsetAsync(c->cbm[1], 0, words * 4, s));
  if (p.r1_cand) {  // (the commit that marks candidates writes every word of these)
    CK(cudaMemsetAsync(c->cand, 0, words * 4, s));
    CK(cudaMemsetAsync(c->rbm[1], 0, words * 4, s));
  }
  CK(cudaMemsetAsync(c->scratch, 0, sizeof(egs::Scratch), s));
  CK(cudaMemsetAsync(c->ctr, 0, egs::kNumCounters * sizeof(unsigned long long), s));
  void* args[] = {&p};
  CK(cudaLaunchCooperativeKernel(solve_kernel(c), dim3(c->grid), dim3(egs::kBlock), args,
                                 egs::kLiftSmemBytes, s));
  CK(cudaEventRecord(c->ev[1], s));
  CK(cudaMemcpyAsync(c->h_ctr, c->ctr, egs::kNumCounters * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  const unsigned long long* h = c->h_ctr;
  c->solved = h[egs::kStatus] == 0;
  c->epoch = (unsigned int)h[egs::kEpoch];
  if (st) fill_stats<V>(c, h, ms, st);
  if (c->trace) {  // EGS_TRACE=1: one line per phase on stderr
    std::vector<unsigned long long> tr(egs::kTraceCap);
    CK(cudaMemcpy(tr.data(), c->trace, tr.size() * 8, cudaMemcpyDeviceToHost));
    static const char* names[4] = {"round1", "lift", "cert", "activate"};
    static const char* fine[6] = {"", "/commit", "/cert-init", "/cert-dense", "/cert-sparse",
                                  "/cert-apply"};
    for (unsigned k = 1; k < egs::kTraceCap && tr[k]; ++k) {
      const int code = (int)(tr[k] >> 56);  // kind * 8 + fine + 1
      const int kind = code / 8, f = code % 8;  // f = fine + 1 (0: none)
      std::fprintf(stderr, "[egs trace] %3u %-8s%-13s %9.1f us\n", k, names[kind % 4],
                   fine[f < 6 ? f : 0], (tr[k] & ((1ull << 56) - 1)) * 1e-3);
    }
    CK(cudaMemset(c->trace, 0, egs::kTraceCap * 8));
  }
  if (h[egs::kStatus] == 7) {
    c->connected = false;  // the ranks' barrier epochs no longer agree
    throw Fail(EGS_ERR_CUDA, "a peer rank did not reach a cross-rank barrier in time");
  }
  if (h[egs::kStatus] == 2) throw Fail(EGS_ERR_TIMEOUT, "solve timed out");
  if (h[egs::kStatus] == 5)
    throw Fail(EGS_ERR_BOUND, "round budget of " + std::to_string(budget) +
                                  " exhausted before reaching a fixpoint");
  if (p.debug) debug_verify<V>(c);
}

void ctx_solve(egs_ctx* c, egs_gpu_stats* st) {
  CK(cudaSetDevice(c->device));
  if (c->n == 0) {
    c->solved = true;
    return;
  }
  if (c->vbits == 32)
    run_solve<uint32_t>(c, st);
  else
    run_solve<uint64_t>(c, st);
}

void ctx_read(egs_ctx* c, int64_t* out) {
  if (!c->solved) throw Fail(EGS_ERR_INVALID_CONFIG, "context not solved");
  if (c->n == 0) return;
  CK(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const uint32_t n = c->n, grid = grid_for(n, c->num_sms);
  if (c->vbits == 64) {
    egs::k_export<uint64_t><<<grid, 256, 0, s>>>(n, static_cast<uint64_t*>(c->f), c->perm,
                                                  c->f64);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, c->f64, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return;
  }
  // 32-bit values cross PCIe at 4 bytes (half the int64 encoding) in chunks
  // into the pinned stage; host threads widen each chunk as it lands
  // (egs_internal_widen_u32: top -> INT64_MAX) while the next is on the wire.
  uint32_t* dev = reinterpret_cast<uint32_t*>(c->f64);
  egs::k_export_u32<<<grid, 256, 0, s>>>(n, static_cast<uint32_t*>(c->f), c->perm, dev);
  CK(cudaGetLastError());
  std::lock_guard<std::mutex> lk(g_stage_mu);
  uint32_t* stage = static_cast<uint32_t*>(pinned_stage((uint64_t)n * 4));
  constexpr int kParts = 8;
  cudaEvent_t ev[kParts];
  auto lo = [&](int k) { return (uint64_t)n * k / kParts; };
  for (int k = 0; k < kParts; ++k) {
    CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    CK(cudaMemcpyAsync(stage + lo(k), dev + lo(k), (lo(k + 1) - lo(k)) * 4,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ev[k], s));
  }
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const unsigned T = n >= (1u << 20) ? hw : 1;
  const int device = c->device;
  auto work = [&](unsigned t) {  // slice t of every part, in landing order
    cudaSetDevice(device);  // (a pool worker's current device may be another)
    for (int k = 0; k < kParts; ++k) {
      cudaEventSynchronize(ev[k]);
      const uint64_t a = lo(k) + (lo(k + 1) - lo(k)) * t / T;
      const uint64_t b = lo(k) + (lo(k + 1) - lo(k)) * (t + 1) / T;
      egs_internal_widen_u32(stage + a, out + a, b - a);
    }
  };
  {
    egs_host::Pool::Job helpers;
    egs_host::Pool::get().launch(helpers, T - 1, [&](unsigned t) { work(t + 1); });
    work(0);
  }
  cudaError_t err = cudaSuccess;
  for (int k = 0; k < kParts; ++k) {
    const cudaError_t e = cudaEventQuery(ev[k]);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
    cudaEventDestroy(ev[k]);
  }
  CK(err);
}

template <class V>
int64_t write_solution_dev(egs_ctx* c, char* buf, size_t cap) {
  cudaStream_t s = c->stream;
  const uint32_t n = c->n;
  DevBuf d_strat, d_len, d_pos, d_text, d_err;
  uint32_t* strat = d_strat.alloc<uint32_t>(n);
  unsigned long long* len = d_len.alloc<unsigned long long>(n);
  unsigned long long* pos = d_pos.alloc<unsigned long long>(n);
  int* err = d_err.alloc<int>(1);
  CK(cudaMemsetAsync(err, 0, sizeof(int), s));
  const V* f = static_cast<const V*>(c->f);
  egs::k_strategy<V><<<grid_for((uint64_t)n * 32, c->num_sms), 256, 0, s>>>(c->graph(), f,
                                                                           c->inv, strat, err);
  egs::k_line_len<V><<<grid_for(n, c->num_sms), 256, 0, s>>>(n, f, c->perm, strat, len);
  CK(cudaGetLastError());
  dev_excl_scan<unsigned long long>(len, pos, n, s, c->num_sms);
  unsigned long long last[2] = {0, 0};
  int h_err = 0;
  CK(cudaMemcpyAsync(&last[0], pos + (n - 1), 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&last[1], len + (n - 1), 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h_err == 1) throw Fail(EGS_ERR_UNSUPPORTED, "energy subtraction out of range");
  if (h_err == 2) throw Fail(EGS_ERR_INTERNAL, "no witness successor for a finite player-0 vertex");
  const uint64_t total = last[0] + last[1];
  if (buf && cap) {
    char* text = d_text.alloc<char>(total);
    egs::k_format<V><<<grid_for(n, c->num_sms), 256, 0, s>>>(n, f, c->perm, strat, pos, text);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(buf, text, std::min<uint64_t>(cap, total), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return (int64_t)total;
}

int ctx_fixpoint(egs_ctx* c, const int64_t* f) {
  CK(cudaSetDevice(c->device));
  g_alloc_stream = c->stream;
  if (c->n == 0) return 1;
  cudaStream_t s = c->stream;
  DevBuf d_in, d_misc;
  int64_t* fin = d_in.alloc<int64_t>(c->n);
  unsigned long long* misc = d_misc.alloc<unsigned long long>(1);
  CK(cudaMemcpyAsync(fin, f, (size_t)c->n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(misc, 0, sizeof(unsigned long long), s));
  const uint32_t grid = grid_for(c->n, c->num_sms);
  egs::k_import<<<grid, 256, 0, s>>>(c->n, fin, c->perm, c->f64);
  egs::k_fixpoint<<<grid_for((uint64_t)c->n * 32, c->num_sms), 256, 0, s>>>(c->graph(), c->f64,
                                                                            misc);
  CK(cudaGetLastError());
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, misc, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));

  return h == 0 ? 1 : 0;
}

int ctx_epm(egs_ctx* c, const int64_t* f) {
  CK(cudaSetDevice(c->device));
  g_alloc_stream = c->stream;
  if (c->n == 0) return 1;
  cudaStream_t s = c->stream;
  DevBuf d_in, d_misc;
  int64_t* fin = d_in.alloc<int64_t>(c->n);
  unsigned long long* misc = d_misc.alloc<unsigned long long>(2);
  CK(cudaMemcpyAsync(fin, f, (size_t)c->n * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(misc, 0, 2 * sizeof(unsigned long long), s));
  const uint32_t grid = grid_for(c->n, c->num_sms);
  egs::k_import<<<grid, 256, 0, s>>>(c->n, fin, c->perm, c->f64);
  egs::k_epm<<<grid_for((uint64_t)c->n * 32, c->num_sms), 256, 0, s>>>(
      c->graph(), c->f64, misc, reinterpret_cast<int*>(misc + 1));
  CK(cudaGetLastError());
  unsigned long long h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, misc, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));

  if (h[1]) throw Fail(EGS_ERR_UNSUPPORTED, "energy subtraction out of range");
  return h[0] == 0 ? 1 : 0;
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

struct egs_part {
  egs_ctx* c = nullptr;
  egs_part_plan plan{};
};

namespace {

// The partition plan (include/egs_gpu.h egs_part_plan): every (owner,
// degree) class -- the classes of the relabelling, egs_scan.cuh -- split
// into `world` pieces by out-edges, the first vertex of piece r being the
// first class member with at least E_class * r / world edges before it
// (edge_balanced_bounds, solver_par.cpp:62-80); rank r's block is its pieces
// of the six classes, class-sorted.  Two host passes over the offsets:
// per-chunk class counts and edges, then only the chunks a boundary falls in
// are walked again.
void plan_compute(const egs_arena_view* a, int world, egs_part_plan* pl) {
  if (world < 1 || world > egs::kMaxRanks)
    throw Fail(EGS_ERR_INVALID_CONFIG, "world must be in [1, " + std::to_string(egs::kMaxRanks) + "]");
  std::memset(pl, 0, sizeof(*pl));
  const uint32_t n = a->num_vertices;
  pl->world = (uint32_t)world;
  pl->num_vertices = n;
  constexpr int C = egs::kNumClasses;
  auto cls = [&](uint32_t v) {
    const uint64_t deg = a->csr_offsets[v + 1] - a->csr_offsets[v];
    return (a->owners[v] ? 3 : 0) + (deg <= egs::kLightMax ? 0 : deg <= egs::kMediumMax ? 1 : 2);
  };
  // Per-group class counts and edges, groups of kGroup consecutive vertices
  // (threads take contiguous group ranges): a piece boundary is then found
  // by walking the group sums and scanning one group.
  constexpr uint32_t kGroup = 1u << 16;
  const uint32_t G = (n + kGroup - 1) / kGroup;
  const unsigned T = n > (1u << 20) ? std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1u;
  std::vector<uint64_t> cnt((size_t)G * C, 0), edg((size_t)G * C, 0);
  auto group = [&](uint32_t gi) {
    return std::make_pair((uint64_t)gi * kGroup, std::min<uint64_t>(n, (uint64_t)(gi + 1) * kGroup));
  };
  auto run_groups = [&](auto&& fn) {  // fn(group) over all groups, T threads
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
      pool.emplace_back([&, t] {
        for (uint32_t gi = (uint32_t)((uint64_t)G * t / T); gi < (uint64_t)G * (t + 1) / T; ++gi) fn(gi);
      });
    for (auto& th : pool) th.join();
  };
  run_groups([&](uint32_t gi) {
    const auto [lo, hi] = group(gi);
    for (uint64_t v = lo; v < hi; ++v) {
      const int k = cls((uint32_t)v);
      cnt[(size_t)gi * C + k] += 1;
      edg[(size_t)gi * C + k] += a->csr_offsets[v + 1] - a->csr_offsets[v];
    }
  });
  uint64_t ctot[C] = {}, etot[C] = {};
  for (uint32_t gi = 0; gi < G; ++gi)
    for (int k = 0; k < C; ++k) ctot[k] += cnt[(size_t)gi * C + k], etot[k] += edg[(size_t)gi * C + k];
  for (int k = 0; k < C; ++k) {
    pl->piece[k][0] = 0;
    pl->piece[k][world] = (uint32_t)ctot[k];
    for (int r = 1; r < world; ++r) {
      // edge_balanced_bounds (solver_par.cpp:62-80) per class: the first
      // class member with at least ceil(E_k * r / world) class edges before it
      const uint64_t target = (etot[k] * (uint64_t)r + world - 1) / world;
      uint64_t pos = 0, cum = 0;
      uint32_t gi = 0;
      for (; gi < G; ++gi) {
        if (cum + edg[(size_t)gi * C + k] >= target) break;
        cum += edg[(size_t)gi * C + k];
        pos += cnt[(size_t)gi * C + k];
      }
      if (gi == G) {
        pl->piece[k][r] = (uint32_t)ctot[k];
        continue;
      }
      const auto [lo, hi] = group(gi);
      for (uint64_t v = lo; v < hi && cum < target; ++v)
        if (cls((uint32_t)v) == k) {
          cum += a->csr_offsets[v + 1] - a->csr_offsets[v];
          ++pos;
        }
      pl->piece[k][r] = (uint32_t)pos;
    }
  }
  uint32_t id = 0;
  for (int r = 0; r < world; ++r) {
    pl->rank_lo[r] = id;
    for (int k = 0; k < C; ++k) {
      pl->class_lo[r][k] = id;
      id += pl->piece[k][r + 1] - pl->piece[k][r];
    }
    pl->class_lo[r][C] = id;
  }
  pl->rank_lo[world] = id;
  // edges per rank: a group wholly inside one rank's piece of every class
  // adds its sums; a group a boundary falls in is scanned
  std::vector<uint64_t> cpos((size_t)G * C, 0);  // class positions at each group start
  for (uint32_t gi = 1; gi < G; ++gi)
    for (int k = 0; k < C; ++k)
      cpos[(size_t)gi * C + k] = cpos[(size_t)(gi - 1) * C + k] + cnt[(size_t)(gi - 1) * C + k];
  std::vector<uint64_t> er((size_t)G * world, 0);
  auto rank_of = [&](int k, uint64_t p) {
    int r = 0;
    while (r + 1 < world && p >= pl->piece[k][r + 1]) ++r;
    return r;
  };
  run_groups([&](uint32_t gi) {
    bool whole = true;
    for (int k = 0; k < C && whole; ++k) {
      const uint64_t p0 = cpos[(size_t)gi * C + k], c = cnt[(size_t)gi * C + k];
      if (c) whole = rank_of(k, p0) == rank_of(k, p0 + c - 1);
    }
    if (whole) {
      for (int k = 0; k < C; ++k)
        if (cnt[(size_t)gi * C + k])
          er[(size_t)gi * world + rank_of(k, cpos[(size_t)gi * C + k])] += edg[(size_t)gi * C + k];
      return;
    }
    uint64_t p[C];
    for (int k = 0; k < C; ++k) p[k] = cpos[(size_t)gi * C + k];
    const auto [lo, hi] = group(gi);
    for (uint64_t v = lo; v < hi; ++v) {
      const int k = cls((uint32_t)v);
      er[(size_t)gi * world + rank_of(k, p[k])] += a->csr_offsets[v + 1] - a->csr_offsets[v];
      ++p[k];
    }
  });
  for (uint32_t gi = 0; gi < G; ++gi)
    for (int r = 0; r < world; ++r) pl->edges[r] += er[(size_t)gi * world + r];
}

// The original-id row ranges of rank `rank` (vertices whose class piece is
// the rank's), for the sharded upload; runs separated by small gaps are
// merged (their rows are uploaded and ignored) so at most kMaxRuns copies
// are issued.
std::vector<std::pair<uint32_t, uint32_t>> rank_runs(const egs_arena_view* a,
                                                     const egs_part_plan& pl, int rank) {
  constexpr size_t kMaxRuns = 2048;
  constexpr int C = egs::kNumClasses;
  const uint32_t n = a->num_vertices;
  const int world = (int)pl.world;
  auto cls = [&](uint32_t v) {
    const uint64_t deg = a->csr_offsets[v + 1] - a->csr_offsets[v];
    return (a->owners[v] ? 3 : 0) + (deg <= egs::kLightMax ? 0 : deg <= egs::kMediumMax ? 1 : 2);
  };
  const unsigned T = n > (1u << 20) ? std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1u;
  auto chunk = [&](unsigned t) { return std::make_pair((uint64_t)n * t / T, (uint64_t)n * (t + 1) / T); };
  std::vector<uint64_t> cnt((size_t)T * C, 0);
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> part(T);
  auto run_all = [&](auto&& fn) {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back([&, t] { fn(t); });
    for (auto& th : pool) th.join();
  };
  run_all([&](unsigned t) {
    const auto [lo, hi] = chunk(t);
    for (uint64_t v = lo; v < hi; ++v) cnt[t * C + cls((uint32_t)v)] += 1;
  });
  run_all([&](unsigned t) {
    uint64_t pos[C];
    for (int k = 0; k < C; ++k) {
      pos[k] = 0;
      for (unsigned u = 0; u < t; ++u) pos[k] += cnt[u * C + k];
    }
    const auto [lo, hi] = chunk(t);
    auto& out = part[t];
    for (uint64_t v = lo; v < hi; ++v) {
      const int k = cls((uint32_t)v);
      const bool mine = pos[k] >= pl.piece[k][rank] && pos[k] < pl.piece[k][rank + 1];
      ++pos[k];
      if (!mine) continue;
      if (!out.empty() && out.back().second == v)
        out.back().second = (uint32_t)v + 1;
      else
        out.emplace_back((uint32_t)v, (uint32_t)v + 1);
    }
  });
  std::vector<std::pair<uint32_t, uint32_t>> runs;
  for (auto& p : part)
    for (auto& r : p) {
      if (!runs.empty() && runs.back().second == r.first)
        runs.back().second = r.second;
      else
        runs.push_back(r);
    }
  (void)world;
  if (runs.size() > kMaxRuns) {  // merge the smallest gaps (in edges)
    std::vector<uint64_t> gaps;
    for (size_t i = 1; i < runs.size(); ++i)
      gaps.push_back(a->csr_offsets[runs[i].first] - a->csr_offsets[runs[i - 1].second]);
    std::vector<uint64_t> sorted = gaps;
    const size_t drop = runs.size() - kMaxRuns;
    std::nth_element(sorted.begin(), sorted.begin() + (drop - 1), sorted.end());
    const uint64_t thr = sorted[drop - 1];
    std::vector<std::pair<uint32_t, uint32_t>> merged{runs[0]};
    size_t budget = drop;
    for (size_t i = 1; i < runs.size(); ++i) {
      if (gaps[i - 1] <= thr && budget > 0) {
        merged.back().second = runs[i].second;
        --budget;
      } else {
        merged.push_back(runs[i]);
      }
    }
    runs.swap(merged);
  }
  return runs;
}

cudaUUID_t device_uuid(int device) {
  cudaDeviceProp prop{};
  CK(cudaGetDeviceProperties(&prop, device));
  return prop.uuid;
}

// Grid of a rank's persistent kernel: ranks sharing a device split it.
// Their persistent kernels must run concurrently, which needs them on
// different hardware work queues: with the default 8 (CUDA_DEVICE_MAX_CONNECTIONS)
// and three streams per rank, 5-7 ranks on one GPU deadlock at the first
// cross-rank barrier (measured; 8 ranks work with 32 queues) -- refused
// up front instead of timing out.
void part_grid(egs_ctx* c, int ranks_on_device) {
  if (ranks_on_device <= 1) return;
  const char* q = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
  const int queues = q ? std::atoi(q) : 8;
  if (ranks_on_device > 4 && queues < 4 * ranks_on_device)
    throw Fail(EGS_ERR_INVALID_CONFIG,
               std::to_string(ranks_on_device) + " ranks share one GPU: set "
               "CUDA_DEVICE_MAX_CONNECTIONS=32 before CUDA initialises (or use at most 4)");
  c->grid = std::max(1, std::min(c->grid, c->full_grid / ranks_on_device));
}

}  // namespace

extern "C" {

int egs_part_plan_compute(const egs_arena_view* arena, int32_t world, egs_part_plan* plan) {
  return guarded([&] {
    if (!arena || !plan) throw Fail(EGS_ERR_INVALID_CONFIG, "null argument");
    plan_compute(arena, world, plan);
  });
}

int egs_part_create(const egs_arena_view* arena, const egs_gpu_opts* opts, int32_t rank,
                    int32_t world, egs_part** out, egs_part_plan* plan_out,
                    egs_gpu_stats* stats) {
  return guarded([&] {
    egs_gpu_opts o;
    if (opts)
      o = *opts;
    else
      egs_gpu_opts_default(&o);
    if (!arena || !out) throw Fail(EGS_ERR_INVALID_CONFIG, "null argument");
    if (world < 1 || world > egs::kMaxRanks || rank < 0 || rank >= world)
      throw Fail(EGS_ERR_INVALID_CONFIG, "rank must be in [0, world), world in [1, 8]");
    if (o.n_gpus != world) throw Fail(EGS_ERR_INVALID_CONFIG, "opts.n_gpus must equal world");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    auto* p = new egs_part();
    try {
      plan_compute(arena, world, &p->plan);
      p->c = ctx_create(arena, o, stats, rank, world, &p->plan);
    } catch (...) {
      delete p;
      throw;
    }
    if (world == 1) p->c->connected = true;
    if (plan_out) *plan_out = p->plan;
    *out = p;
  });
}

int egs_part_export(egs_part* part, void* handle) {
  return guarded([&] {
    if (!part || !handle) throw Fail(EGS_ERR_INVALID_CONFIG, "null argument");
    egs_ctx* c = part->c;
    if (!c->xbuf) throw Fail(EGS_ERR_INVALID_CONFIG, "a one-rank partition has nothing to export");
    CK(cudaSetDevice(c->device));
    static_assert(sizeof(cudaIpcMemHandle_t) + 16 <= EGS_IPC_HANDLE_BYTES, "export record size");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->xbuf));
    char rec[EGS_IPC_HANDLE_BYTES] = {};
    std::memcpy(rec, &h, sizeof(h));
    const cudaUUID_t u = device_uuid(c->device);
    std::memcpy(rec + sizeof(h), &u, 16);
    std::memcpy(handle, rec, sizeof(rec));
  });
}

int egs_part_connect(egs_part* part, const void* handles) {
  return guarded([&] {
    if (!part || !handles) throw Fail(EGS_ERR_INVALID_CONFIG, "null argument");
    egs_ctx* c = part->c;
    CK(cudaSetDevice(c->device));
    const cudaUUID_t mine = device_uuid(c->device);
    int same = 1;  // ranks on this GPU (their persistent grids must be co-resident)
    for (int q = 0; q < c->world; ++q) {
      if (q == c->rank) continue;
      const char* rec = static_cast<const char*>(handles) + (size_t)q * EGS_IPC_HANDLE_BYTES;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, rec, sizeof(h));
      if (std::memcmp(rec + sizeof(h), &mine, 16) == 0) ++same;
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      c->xpeer[q] = static_cast<char*>(ptr);
      c->xpeer_ipc[q] = true;
    }
    part_grid(c, same);
    c->connected = true;
  });
}

int egs_part_connect_local(egs_part* const* parts, int32_t world) {
  return guarded([&] {
    if (!parts || world < 1) throw Fail(EGS_ERR_INVALID_CONFIG, "null argument");
    for (int r = 0; r < world; ++r) {
      if (!parts[r] || parts[r]->c->rank != r || parts[r]->c->world != world)
        throw Fail(EGS_ERR_INVALID_CONFIG, "parts[r] must be rank r of the same world");
      if (parts[r]->c->xbytes != parts[0]->c->xbytes)
        throw Fail(EGS_ERR_INVALID_CONFIG, "parts of different arenas");
    }
    for (int r = 0; r < world; ++r) {
      egs_ctx* c = parts[r]->c;
      int same = 0;
      for (int q = 0; q < world; ++q) {
        egs_ctx* d = parts[q]->c;
        c->xpeer[q] = d->xbuf;
        if (d->device == c->device) {
          ++same;
        } else {
          CK(cudaSetDevice(c->device));
          const cudaError_t e = cudaDeviceEnablePeerAccess(d->device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
          cudaGetLastError();
        }
      }
      part_grid(c, same);
      c->connected = true;
    }
  });
}

int egs_part_solve(egs_part* part, egs_gpu_stats* stats) {
  return guarded([&] {
    if (!part) throw Fail(EGS_ERR_INVALID_CONFIG, "null partition");
    egs_ctx* c = part->c;
    if (!c->connected) throw Fail(EGS_ERR_INVALID_CONFIG, "partition not connected to its peers");
    auto t0 = Clock::now();
    if (stats) std::memset(stats, 0, sizeof(*stats));
    ctx_solve(c, stats);
    if (stats) stats->wall_seconds = secs_since(t0);
  });
}

int egs_part_read_measure(egs_part* part, int64_t* f_out) {
  return guarded([&] {
    if (!part) throw Fail(EGS_ERR_INVALID_CONFIG, "null partition");
    ctx_read(part->c, f_out);
  });
}

int egs_part_digest(egs_part* part, uint64_t* digest) {
  return guarded([&] {
    if (!part || !digest) throw Fail(EGS_ERR_INVALID_CONFIG, "null argument");
    egs_ctx* c = part->c;
    if (!c->solved) throw Fail(EGS_ERR_INVALID_CONFIG, "partition not solved");
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    g_alloc_stream = s;
    DevBuf d_out;
    unsigned long long* out = d_out.alloc<unsigned long long>(1);
    CK(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
    const uint32_t grid = grid_for(c->n, c->num_sms);
    if (c->vbits == 32)
      egs::k_digest<uint32_t><<<grid, 256, 0, s>>>(c->n, static_cast<const uint32_t*>(c->f), out);
    else
      egs::k_digest<uint64_t><<<grid, 256, 0, s>>>(c->n, static_cast<const uint64_t*>(c->f), out);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, out, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *digest = h;
  });
}

void egs_part_destroy(egs_part* part) {
  if (!part) return;
  ctx_free(part->c);
  delete part;
}

void egs_gpu_opts_default(egs_gpu_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->n_gpus = 1;
  o->device = -1;
  o->certify = 1;
  o->cert_interval = 1;
  o->cert_growth = 8;
  o->sparse_div = 8;
  o->mode = EGS_MODE_AUTO;
}

int egs_ctx_create(const egs_arena_view* arena, const egs_gpu_opts* opts, egs_ctx** out,
                   egs_gpu_stats* stats) {
  return guarded([&] {
    egs_gpu_opts o;
    if (opts)
      o = *opts;
    else
      egs_gpu_opts_default(&o);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    *out = ctx_create(arena, o, stats);
  });
}

int egs_ctx_solve(egs_ctx* ctx, egs_gpu_stats* stats) {
  return guarded([&] {
    if (!ctx) throw Fail(EGS_ERR_INVALID_CONFIG, "null context");
    auto t0 = Clock::now();
    if (stats) std::memset(stats, 0, sizeof(*stats));
    ctx_solve(ctx, stats);
    if (stats) stats->wall_seconds = secs_since(t0);
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

int64_t egs_ctx_write_solution(egs_ctx* ctx, char* buf, size_t cap) {
  int64_t r = 0;
  int rc = guarded([&] {
    if (!ctx) throw Fail(EGS_ERR_INVALID_CONFIG, "null context");
    if (!ctx->solved) throw Fail(EGS_ERR_INVALID_CONFIG, "context not solved");
    CK(cudaSetDevice(ctx->device));
    g_alloc_stream = ctx->stream;
    if (ctx->n == 0) {
      r = 0;
      return;
    }
    r = ctx->vbits == 32 ? write_solution_dev<uint32_t>(ctx, buf, cap)
                         : write_solution_dev<uint64_t>(ctx, buf, cap);
  });
  return rc == EGS_OK ? r : -rc;
}

int egs_ctx_is_fixpoint(egs_ctx* ctx, const int64_t* f) {
  int r = 0;
  int rc = guarded([&] {
    if (!ctx) throw Fail(EGS_ERR_INVALID_CONFIG, "null context");
    r = ctx_fixpoint(ctx, f);
  });
  return rc == EGS_OK ? r : -rc;
}

void egs_ctx_destroy(egs_ctx* ctx) { ctx_free(ctx); }

int egs_gpu_solve(const egs_arena_view* arena, const egs_gpu_opts* opts, int64_t* f_out,
                  egs_gpu_stats* stats) {
  return guarded([&] {
    auto t0 = Clock::now();
    egs_gpu_opts o;
    if (opts)
      o = *opts;
    else
      egs_gpu_opts_default(&o);
    egs_gpu_stats local{};
    egs_gpu_stats* st = stats ? stats : &local;
    std::memset(st, 0, sizeof(*st));
    egs_ctx* c = ctx_create(arena, o, st);
    try {
      const double up = st->upload_seconds;
      const uint64_t h2d = st->h2d_bytes;
      ctx_solve(c, st);
      st->h2d_bytes = h2d;
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
