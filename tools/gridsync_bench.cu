// Floor of a phase boundary in the persistent solve kernel (VERDICT r01,
// "time a bare grid.sync() at 296 CTAs"): per-iteration device time of
//   0  cg grid.sync() alone
//   1  grid.sync() + the round-1 block_flush (12 warp reductions, 2
//      __syncthreads, up to 12 same-address global atomics per CTA)
//   2  grid.sync() + one same-address atomicAdd per CTA (the phase sum the
//      control flow reads)
//   3  grid.sync() + one atomicAdd per WARP
//   4  hand-rolled barrier: one arrival atomic per CTA + acquire spin on a
//      generation word (what a phase boundary needs at least)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridsync_bench.bin tools/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ unsigned int g_arrive;
__device__ volatile unsigned int g_gen;

__device__ __forceinline__ void my_barrier(unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int want = gen + 1;
    __threadfence();
    const unsigned int a = atomicAdd(&g_arrive, 1u);
    if (a == gridDim.x - 1) {
      g_arrive = 0;
      __threadfence();
      g_gen = want;
    } else {
      unsigned int g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&g_gen));
      } while (g != want);
    }
    gen = want;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256, 2) k_bench(int mode, int iters, unsigned long long* ctr,
                                                  unsigned long long* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned int s_cnt[8 * 12];
  unsigned int gen = 0;
  if (threadIdx.x == 0) gen = g_gen;
  grid.sync();
  const unsigned long long t0 = gtimer();
  unsigned int v[12];
  for (int k = 0; k < 12; ++k) v[k] = threadIdx.x + k;
  for (int it = 0; it < iters; ++it) {
    if (mode == 1) {
#pragma unroll
      for (int k = 0; k < 12; ++k) v[k] = __reduce_add_sync(0xffffffffu, v[k] + it);
      __syncthreads();
      if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 12; ++k) s_cnt[(threadIdx.x >> 5) * 12 + k] = v[k];
      __syncthreads();
      if (threadIdx.x < 12) {
        unsigned long long s = 0;
        for (int w = 0; w < 8; ++w) s += s_cnt[w * 12 + threadIdx.x];
        atomicAdd(ctr + threadIdx.x, s);
      }
    } else if (mode == 2) {
      if (threadIdx.x == 0) atomicAdd(ctr, 1ull);
    } else if (mode == 3) {
      if ((threadIdx.x & 31) == 0) atomicAdd(ctr, 1ull);
    }
    if (mode == 4)
      my_barrier(gen);
    else
      grid.sync();
  }
  const unsigned long long t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

int main(int argc, char** argv) {
  int per_sm = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bench, 256, 0);
  unsigned long long *ctr, *out;
  cudaMalloc(&ctr, 64 * 8);
  cudaMalloc(&out, 8);
  const int iters = 2000;
  const int grids[] = {148, 296};
  for (int gi = 0; gi < 2; ++gi) {
    int grid = grids[gi];
    if (grid > per_sm * sms) continue;
    for (int mode = 0; mode < 5; ++mode) {
      double best = 1e30;
      for (int rep = 0; rep < 3; ++rep) {
        int m = mode, it = iters;
        void* args[] = {&m, &it, &ctr, &out};
        cudaLaunchCooperativeKernel((void*)k_bench, dim3(grid), dim3(256), args, 0, 0);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          std::printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        unsigned long long ns = 0;
        cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
        best = ns / (double)iters < best ? ns / (double)iters : best;
      }
      static const char* names[] = {"grid.sync", "grid.sync+block_flush", "grid.sync+atomic/CTA",
                                    "grid.sync+atomic/warp", "hand-rolled barrier"};
      std::printf("{\"grid\": %d, \"mode\": \"%s\", \"ns_per_phase\": %.1f}\n", grid, names[mode],
                  best);
    }
  }
  return 0;
}
