// Do shared-memory accesses and global stores of one SM overlap, or do they
// queue behind each other?  And how fast are 64-byte TMA bulk stores
// (cp.async.bulk.global.shared::cta) compared with STG?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mb_mio tools/mb_mio.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
// role bits: 1 = STG warps (scattered 64-B chunks, 8 B per lane), 2 = STS warps (random 8-byte stores), 4 = TMA bulk stores of 64 B
__global__ void __launch_bounds__(512, 1) k(uint32_t* __restrict__ out, size_t span_words, int iters, unsigned long long* cyc,
                                           int stg_warps, int sts_warps, int tma_warps) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t nchunk = span_words / 16;
  uint32_t h = mix(blockIdx.x * 977u + warp * 131u + 1u);
  uint2* s2 = reinterpret_cast<uint2*>(sm);
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp < stg_warps) {
    for (int it = 0; it < iters; ++it) {
      h = mix(h + it);
      const size_t c = (size_t)(mix(h + (lane >> 3)) & (nchunk - 1));
      uint2* p = reinterpret_cast<uint2*>(out + c * 16) + (lane & 7);
      *p = make_uint2(it, lane);
    }
  } else if (warp < stg_warps + sts_warps) {
    uint32_t g = mix(threadIdx.x * 7u + 3u);
    for (int it = 0; it < iters * 4; ++it) {
      g = g * 1664525u + 1013904223u;
      s2[(g >> 8) & 8191] = make_uint2(it, lane);  // random 8-byte slots in 64 KB
    }
  } else if (warp < stg_warps + sts_warps + tma_warps) {
    // each lane: one 64-byte bulk store from its own 64-byte SMEM slot
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm + 65536 + (size_t)threadIdx.x * 64);
    for (int it = 0; it < iters; ++it) {
      h = mix(h + it);
      const size_t c = (size_t)(mix(h + lane) & (nchunk - 1));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 64;" ::"l"(out + c * 16), "r"(src) : "memory");
      if ((it & 7) == 7) {
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  unsigned long long t1 = clock64();
  // per-role elapsed cycles (max over the role's warps, block 0 only)
  const int role = warp < stg_warps ? 0 : warp < stg_warps + sts_warps ? 1 : warp < stg_warps + sts_warps + tma_warps ? 2 : 3;
  if (blockIdx.x == 0 && lane == 0 && role < 3) atomicMax(&cyc[role], t1 - t0);
}
int main() {
  const size_t words = (size_t)1 << 30;
  uint32_t* out; cudaMalloc(&out, words * 4);
  unsigned long long* cyc; cudaMallocManaged(&cyc, 148 * 8); 
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 20000;
  const size_t span = (size_t)1 << 24;  // 64 MB: L2-resident, so DRAM is not the limiter
  struct R { int stg, sts, tma; } runs[] = {{8, 0, 0}, {16, 0, 0}, {0, 8, 0}, {0, 16, 0}, {8, 8, 0}, {4, 12, 0}, {0, 0, 1}, {0, 0, 4}, {0, 0, 8}, {0, 8, 4}, {0, 8, 8}, {0, 12, 4}, {0, 15, 1}};
  for (int grid : {1, 148})
    for (auto r : runs) {
      for (int rep = 0; rep < 2; ++rep) { cyc[0] = cyc[1] = cyc[2] = 0; k<<<grid, 512, 100 * 1024>>>(out, span, iters, cyc, r.stg, r.sts, r.tma); cudaDeviceSynchronize(); }
      cudaError_t e = cudaGetLastError(); if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      printf("grid %3d stg %2d sts %2d tma %2d:", grid, r.stg, r.sts, r.tma);
      if (r.stg) printf("  STG %8llu cyc = %.1f B/clk", cyc[0], (double)iters * r.stg * 256 / cyc[0]);
      if (r.sts) printf("  STS %8llu cyc = %.2f cyc/warp-instr", cyc[1], (double)cyc[1] / ((double)iters * 4 * r.sts));
      if (r.tma) printf("  TMA %8llu cyc = %.1f B/clk", cyc[2], (double)iters * r.tma * 2048 / cyc[2]);
      printf("\n");
    }
  return 0;
}
