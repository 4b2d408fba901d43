// Ranking primitive microbenchmarks on B200 (scratch tool, not product).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ __forceinline__ uint32_t lmlt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

// MODE 0: 10 unrolled ballots + leader LDS/STS on per-warp u16 counts
// MODE 1: atomicOr peer mask + leader update (per-warp u32 mask table)
// MODE 2: atomicAdd with return (unordered slot) on a per-CTA table
template <int MODE, int NB>
__global__ void __launch_bounds__(256) kb(uint32_t* sink, int iters) {
  extern __shared__ uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint16_t* wh = reinterpret_cast<uint16_t*>(sm) + warp * NB;      // 8 warps x NB u16
  uint32_t* mk = sm + (8 * NB) / 2 + warp * NB;                    // 8 warps x NB u32
  for (int i = threadIdx.x; i < 8 * NB / 2 + 8 * NB; i += 256) sm[i] = 0;
  __syncthreads();
  uint32_t acc = 0, base = (blockIdx.x * 256 + threadIdx.x) * 7919u;
  for (int it = 0; it < iters; ++it) {
    const uint32_t b = hash32(base + it) & (NB - 1);
    if (MODE == 0) {
      uint32_t m = FULL;
#pragma unroll
      for (int i = 0; i < 10; ++i) { const uint32_t bit = (b >> i) & 1; const uint32_t bal = __ballot_sync(FULL, bit); m &= bit ? bal : ~bal; }
      const uint32_t before = __popc(m & lmlt());
      const uint32_t old = wh[b];
      __syncwarp();
      if (before == 0) wh[b] = (uint16_t)(old + __popc(m));
      __syncwarp();
      acc += old + before;
    } else if (MODE == 1) {
      atomicOr(&mk[b], 1u << lane);
      __syncwarp();
      const uint32_t m = mk[b];
      const uint32_t before = __popc(m & lmlt());
      const uint32_t old = wh[b];
      __syncwarp();
      if (before == 0) { wh[b] = (uint16_t)(old + __popc(m)); mk[b] = 0; }
      __syncwarp();
      acc += old + before;
    } else {
      acc += atomicAdd(&sm[b], 1u);
    }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int MODE, int NB>
void run(const char* name) {
  uint32_t* sink; cudaMalloc(&sink, 4);
  const size_t smem = 8 * NB * 2 + 8 * NB * 4;
  cudaFuncSetAttribute(kb<MODE, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int iters = 4096, blocks = 148 * 4;
  kb<MODE, NB><<<blocks, 256, smem>>>(sink, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kb<MODE, NB><<<blocks, 256, smem>>>(sink, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-34s NB=%5d : %8.1f Gkeys/s  err=%s\n", name, NB, (double)blocks * 256 * iters / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0, 1024>("ballot10 + leader LDS/STS");
  run<1, 1024>("atomicOr mask + leader");
  run<2, 1024>("atomicAdd with return");
  run<0, 512>("ballot10 + leader LDS/STS");
  run<1, 512>("atomicOr mask + leader");
  run<2, 512>("atomicAdd with return");
  return 0;
}
