// Roofline probe for the lift's access pattern on B200: 16M vertices x 16
// random successors, u32 values (the C4 shape).  Measures how fast random
// 4-byte gathers from a 64 MB array can be served with different mappings.
//   A  edge-centric: coalesced dst stream, one gather per thread per step
//   B  thread-per-row, 16 edges, direct row loads, ld.cg gathers
//   C  thread-per-row, ld.global.nc gathers
//   D  like B but gathers only half the rows (P1 half of an owner-sorted arena)
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t g_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t g_hint(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_last()));
  return v;
}
__device__ __forceinline__ uint32_t g_plain(const uint32_t* p) { return *(const volatile uint32_t*)p; }
// row per thread like lift_thread: f[v], off[v], off[v+1], clamped chunks, 64-bit ominus, stage write
template <int G>
__global__ void kL(const int2* __restrict__ e, const uint32_t* __restrict__ off, uint32_t n, const uint32_t* f,
                   uint32_t* stage, uint32_t* chg, int64_t cap) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (v & 1) continue;
    const uint32_t old = __ldcg(f + v);
    bool ch = false;
    if (old != 0xFFFFFFFFu) {
      const uint32_t b = __ldg(off + v), en = __ldg(off + v + 1);
      uint32_t acc = 0;
      for (uint32_t i = b; i < en; i += 8) {
        int2 r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __ldcs(e + min(i + k, en - 1));
        uint32_t c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = G == 0 ? g_cg(f + r[k].x) : G == 1 ? g_hint(f + r[k].x) : g_plain(f + r[k].x);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          int64_t x = (int64_t)c[k] - r[k].y; x = x < 0 ? 0 : x;
          uint32_t o = x > cap ? 0xFFFFFFFFu : (uint32_t)x; o = c[k] == 0xFFFFFFFFu ? 0xFFFFFFFFu : o;
          acc = o > acc ? o : acc;
        }
        if (acc == 0xFFFFFFFFu) break;
      }
      if (acc > old) { __stcg(stage + v, acc); ch = true; }
    }
    unsigned m = __ballot_sync(__activemask(), ch);
    if (m && (threadIdx.x & 31) == 0) atomicOr(chg + (v >> 5), m);
  }
}
__device__ __forceinline__ uint32_t g_nc(const uint32_t* p) { return __ldg(p); }

__global__ void kA(const int2* __restrict__ e, uint64_t m, const uint32_t* f, uint32_t* out, uint32_t mask) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    int2 r = __ldcs(e + i);
    acc = max(acc, g_cg(f + (r.x & mask)) - r.y);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <bool NC, int CH>
__global__ void kB(const int2* __restrict__ e, uint32_t n, uint32_t d, const uint32_t* f, uint32_t* out, uint32_t stride) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (stride > 1 && (v % stride)) continue;
    const int2* row = e + (uint64_t)v * d;
    uint32_t acc = 0;
    for (uint32_t k0 = 0; k0 < d; k0 += CH) {
      int2 r[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) r[k] = __ldcs(row + k0 + k);
      uint32_t c[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) c[k] = NC ? g_nc(f + r[k].x) : g_cg(f + r[k].x);
#pragma unroll
      for (int k = 0; k < CH; ++k) acc = max(acc, c[k] - r[k].y);
    }
    out[v] = acc;
  }
}

int main() {
  const uint32_t n = 16000000, d = 16;
  const uint64_t m = (uint64_t)n * d;
  std::vector<int2> he(m);
  uint64_t s = 1;
  for (uint64_t i = 0; i < m; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    he[i] = make_int2((int)((s >> 33) % n), (int)((s >> 20) & 255) - 100);
  }
  int2* e; uint32_t *f, *out;
  CK(cudaMalloc(&e, m * 8)); CK(cudaMalloc(&f, n * 4)); CK(cudaMalloc(&out, n * 4));
  CK(cudaMemcpy(e, he.data(), m * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(f, 1, n * 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch, double gathers, double bytes) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-40s %8.3f ms  %7.1f Ggather/s  %7.1f GB/s (edge stream)\n", name, ms, gathers / ms / 1e6, bytes / ms / 1e6);
  };
  for (int bpsm : {4, 8, 16}) {
    char nm[64]; snprintf(nm, 64, "A edge-centric grid=%dx", bpsm);
    run(nm, [&] { kA<<<sms * bpsm, 256>>>(e, m, f, out, 0xFFFFFFFFu); }, m, m * 8.0);
  }
  for (uint32_t mb : {32, 16, 8, 2}) {
    char nm[64]; snprintf(nm, 64, "A edge-centric target set %u MB", mb);
    uint32_t mask = mb * 1024u * 1024u / 4u - 1u;
    run(nm, [&] { kA<<<sms * 8, 256>>>(e, m, f, out, mask); }, m, m * 8.0);
  }
  for (int bpsm : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "B row/thread cg ch8 grid=%dx", bpsm);
    run(nm, [&] { kB<false, 8><<<sms * bpsm, 256>>>(e, n, d, f, out, 1); }, m, m * 8.0);
    snprintf(nm, 64, "B row/thread cg ch16 grid=%dx", bpsm);
    run(nm, [&] { kB<false, 16><<<sms * bpsm, 256>>>(e, n, d, f, out, 1); }, m, m * 8.0);
    snprintf(nm, 64, "C row/thread nc ch8 grid=%dx", bpsm);
    run(nm, [&] { kB<true, 8><<<sms * bpsm, 256>>>(e, n, d, f, out, 1); }, m, m * 8.0);
    snprintf(nm, 64, "D half rows cg ch8 grid=%dx", bpsm);
    run(nm, [&] { kB<false, 8><<<sms * bpsm, 256>>>(e, n, d, f, out, 2); }, m / 2, m * 4.0);
  }
  uint32_t *off, *stage, *chg;
  std::vector<uint32_t> hoff(n + 1);
  for (uint32_t v = 0; v <= n; ++v) hoff[v] = v * d;
  CK(cudaMalloc(&off, (n + 1) * 4)); CK(cudaMalloc(&stage, n * 4)); CK(cudaMalloc(&chg, n / 8 + 4));
  CK(cudaMemcpy(off, hoff.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(f, 0, n * 4));
  for (int bpsm : {2, 3, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "L lift-like cg grid=%dx", bpsm);
    run(nm, [&] { kL<0><<<sms * bpsm, 256>>>(e, off, n, f, stage, chg, 1400000000ll); }, m / 2, m * 4.0);
    snprintf(nm, 64, "L lift-like hint grid=%dx", bpsm);
    run(nm, [&] { kL<1><<<sms * bpsm, 256>>>(e, off, n, f, stage, chg, 1400000000ll); }, m / 2, m * 4.0);
    snprintf(nm, 64, "L lift-like volatile grid=%dx", bpsm);
    run(nm, [&] { kL<2><<<sms * bpsm, 256>>>(e, off, n, f, stage, chg, 1400000000ll); }, m / 2, m * 4.0);
  }
  return 0;
}
