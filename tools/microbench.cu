// Microbenchmarks for ranking primitives on B200 (scratch tool, not product).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ __forceinline__ uint32_t lmlt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

template <int NB, int MODE>  // MODE 0 ballot peers, 1 match_any, 2 smem atomic, 3 match+leader LDS/STS, 4 atomic uniform addr
__global__ void kbench(uint32_t* sink, int iters, uint32_t skew) {
  __shared__ uint32_t hist[4][1 << NB];
  for (int i = threadIdx.x; i < 4 * (1 << NB); i += blockDim.x) (&hist[0][0])[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  const int warp = threadIdx.x >> 5;
  uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) * 7919u;
  for (int it = 0; it < iters; ++it) {
    uint32_t h = hash32(base + it);
    uint32_t b = (h & 0xffff) < skew ? 5u : (h >> 8) & ((1u << NB) - 1);
    if (MODE == 0) {
      uint32_t m = FULL;
#pragma unroll
      for (int i = 0; i < NB; ++i) { uint32_t bit = (b >> i) & 1; uint32_t bal = __ballot_sync(FULL, bit); m &= bit ? bal : ~bal; }
      acc += __popc(m & lmlt());
    } else if (MODE == 1) {
      uint32_t m = __match_any_sync(FULL, b);
      acc += __popc(m & lmlt());
    } else if (MODE == 2) {
      atomicAdd(&hist[warp & 3][b], 1u);
    } else if (MODE == 3) {
      uint32_t m = __match_any_sync(FULL, b);
      uint32_t before = __popc(m & lmlt());
      uint32_t old = hist[warp & 3][b];
      __syncwarp();
      if (before == 0) hist[warp & 3][b] = old + __popc(m);
      __syncwarp();
      acc += old + before;
    } else if (MODE == 5) {
      uint32_t m = FULL;
#pragma unroll
      for (int i = 0; i < NB; ++i) { uint32_t bit = (b >> i) & 1; uint32_t bal = __ballot_sync(FULL, bit); m &= bit ? bal : ~bal; }
      uint32_t before = __popc(m & lmlt());
      uint32_t old = hist[warp & 3][b];
      __syncwarp();
      if (before == 0) hist[warp & 3][b] = old + __popc(m);
      __syncwarp();
      acc += old + before;
    }
  }
  __syncthreads();
  if (MODE == 2) acc += hist[warp & 3][threadIdx.x & ((1 << NB) - 1)];
  if (acc == 0x12345678) sink[0] = acc;
}

template <int NB, int MODE>
void run(const char* name, uint32_t skew) {
  uint32_t* sink; cudaMalloc(&sink, 4);
  int iters = 4096; int blocks = 148 * 8, threads = 256;
  kbench<NB, MODE><<<blocks, threads>>>(sink, 16, skew);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kbench<NB, MODE><<<blocks, threads>>>(sink, iters, skew);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double keys = (double)blocks * threads * iters;
  printf("%-28s NB=%2d skew=%5u : %8.1f Gkeys/s  (%.3f ms)\n", name, NB, skew, keys / ms / 1e6, ms);
  cudaFree(sink);
}

int main() {
  for (uint32_t skew : {0u, 32768u, 65535u}) {
    run<8, 0>("ballot peers", skew);
    run<11, 0>("ballot peers", skew);
    run<8, 1>("match_any", skew);
    run<11, 1>("match_any", skew);
    run<8, 2>("smem atomicAdd", skew);
    run<11, 2>("smem atomicAdd", skew);
    run<8, 3>("match + leader LDS/STS", skew);
    run<11, 3>("match + leader LDS/STS", skew);
    run<8, 5>("ballot + leader LDS/STS", skew);
    run<11, 5>("ballot + leader LDS/STS", skew);
  }
  return 0;
}
