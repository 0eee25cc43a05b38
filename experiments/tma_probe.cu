// Micro-test of the per-warp TMA bulk-copy + mbarrier pipeline used by
// dense_light_p1 (egs_solve.cuh).  Each warp streams tiles of a buffer
// through two shared-memory stages and sums them; a watchdog traps instead
// of hanging.
#include <cstdio>
#include <cstdint>
#include "../paper_1710_03647_b200/csrc/egs_device.cuh"
using namespace egs;
constexpr int W = 8, S = 2, R = 512;
__device__ __noinline__ void other_fn(unsigned long long* out) {
  __shared__ unsigned int junk[1234];
  junk[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && junk[5] != 5) atomicAdd(out, 1ull << 60);
}
template <bool NOINLINE>
struct Body;
__device__ __noinline__ void body_noinline(const int2* src, uint32_t ntiles, uint32_t tile_recs, unsigned long long* out);
__device__ __forceinline__ void body(const int2* src, uint32_t ntiles, uint32_t tile_recs, unsigned long long* out) {
  extern __shared__ __align__(128) int2 dsm[];
  __shared__ __align__(8) uint64_t bar[W][S];
  uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int2* st = dsm + warp * S * R;
  if (lane == 0) { for (int s = 0; s < S; ++s) mbar_init(&bar[warp][s], 1); mbar_init_fence(); }
  __syncwarp();
  uint32_t parity = 0, s = 0;
  unsigned long long acc = 0;
  uint32_t nw = gridDim.x * W, w0 = blockIdx.x * W + warp;
  auto issue = [&](uint32_t t, uint32_t ss) {
    if (lane == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bar[warp][ss], tile_recs * 8);
      bulk_g2s(st + ss * R, src + (size_t)t * tile_recs, tile_recs * 8, &bar[warp][ss]);
    }
  };
  if (w0 < ntiles) issue(w0, 0);
  for (uint32_t t = w0; t < ntiles; t += nw) {
    __syncwarp();
    if (t + nw < ntiles) issue(t + nw, s ^ 1);
    unsigned spins = 0;
    while (!mbar_try_wait(&bar[warp][s], (parity >> s) & 1)) { if (++spins > (1u << 24)) __trap(); }
    parity ^= 1u << s;
    for (uint32_t i = lane; i < tile_recs; i += 32) acc += (unsigned)st[s * R + i].x;
    s ^= 1;
  }
  atomicAdd(out, acc);
}
__device__ __noinline__ void body_noinline(const int2* src, uint32_t ntiles, uint32_t tile_recs, unsigned long long* out) {
  body(src, ntiles, tile_recs, out);
}
__global__ void k(const int2* src, uint32_t ntiles, uint32_t tile_recs, unsigned long long* out, int mode) {
  if (mode == 0) body(src, ntiles, tile_recs, out);
  else { other_fn(out); body_noinline(src, ntiles, tile_recs, out); }
}
int main() {
  const uint32_t ntiles = 100000, tr = 512;
  size_t n = (size_t)ntiles * tr;
  int2* h = (int2*)malloc(n * 8); unsigned long long want = 0;
  for (size_t i = 0; i < n; ++i) { h[i] = make_int2((int)(i % 1000), 0); want += i % 1000; }
  int2* d; cudaMalloc(&d, n * 8); cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  unsigned long long* o; cudaMalloc(&o, 8); cudaMemset(o, 0, 8);
  size_t smem = W * S * R * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int bad = 0;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(o, 0, 8);
    cudaEventRecord(a);
    k<<<148 * 3, 256, smem>>>(d, ntiles, tr, o, mode);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long got = 0; cudaMemcpy(&got, o, 8, cudaMemcpyDeviceToHost);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    printf("mode=%d err=%s got=%llu want=%llu %s  %.3f ms  %.1f GB/s\n", mode, cudaGetErrorString(e), got, want,
           got == want ? "OK" : "MISMATCH", ms, n * 8 / ms / 1e6);
    bad |= got != want;
    if (e != cudaSuccess) return 2;
  }
  return bad;
}
