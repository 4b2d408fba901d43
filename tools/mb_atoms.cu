// Cost of SMEM atomicAdd-with-return when many lanes of a warp hit one address
// (a heavy key's bucket) against uniformly random buckets; and of a ballot-ranked
// alternative for the hot bucket.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mb_atoms tools/mb_atoms.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
// mode 0: plain atomics; mode 1: hot bucket 0 by ballot, others atomics
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, int iters, uint32_t hot_permille, unsigned long long* cyc) {
  __shared__ uint32_t wh[16][260];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * 260; i += 512) (&wh[0][0])[i] = 0;
  __syncthreads();
  uint32_t acc = 0, h = mix(threadIdx.x * 977u + blockIdx.x);
  uint32_t c0 = 0;
  const uint32_t lt = (1u << lane) - 1u;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 18; ++i) {
      h = h * 1664525u + 1013904223u;
      const uint32_t r = h >> 8;
      const uint32_t b = (r % 1000u) < hot_permille ? 0u : (r >> 10) % 512u;
      if (MODE == 1) {
        const bool h0 = b == 0u;
        const uint32_t m0 = __ballot_sync(0xffffffffu, h0);
        if (h0) acc += c0 + __popc(m0 & lt);
        else {
          const uint32_t sh = (b & 1u) << 4;
          acc += (atomicAdd(&wh[warp][b >> 1], 1u << sh) >> sh) & 0xffffu;
        }
        c0 += __popc(m0);
      } else {
        const uint32_t sh = (b & 1u) << 4;
        acc += (atomicAdd(&wh[warp][b >> 1], 1u << sh) >> sh) & 0xffffu;
      }
      __syncwarp();
    }
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * 512 + threadIdx.x] = acc + c0;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 512 * 4);
  unsigned long long* cyc; cudaMallocManaged(&cyc, 148 * 8);
  const int iters = 200;
  for (uint32_t hot : {0u, 60u, 150u, 380u, 800u})
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, 512>>>(out, iters, hot, cyc); else k<1><<<148, 512>>>(out, iters, hot, cyc);
        cudaDeviceSynchronize();
      }
      double c = 0; for (int i = 0; i < 148; ++i) c += cyc[i]; c /= 148;
      printf("hot %3u/1000 mode %d: %.3f clk per record and SM (%.0f cycles per 9216-record tile)\n", hot, mode,
             c / (iters * 18.0 * 512), c / iters);
    }
  return 0;
}
