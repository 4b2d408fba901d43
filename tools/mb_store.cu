// SM store-port microbenchmark: how many bytes per clock can one SM push to
// L2 with the write-out's access shape (each warp instruction = 32 lanes x 8 B
// covering 4 scattered 64-byte chunks) against contiguous 256/512-byte rows?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mb_store tools/mb_store.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
// mode 0: scattered 64-B chunks, STG.64; mode 1: contiguous STG.64 (256 B per warp instr);
// mode 2: contiguous STG.128; mode 3: scattered 64-B chunks as STG.128 (4 lanes per chunk)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(uint32_t* __restrict__ out, size_t words, int iters, unsigned long long* cyc, int active_warps, size_t span_words) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= active_warps) return;
  const size_t nchunk = span_words / 16;  // 64-B chunks (power of two)
  uint32_t h = mix(blockIdx.x * 977u + warp * 131u + 1u);
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      h = mix(h + it);
      const size_t c = (size_t)(mix(h + (lane >> 3)) & (nchunk - 1));
      uint2* p = reinterpret_cast<uint2*>(out + c * 16) + (lane & 7);
      *p = make_uint2(it, lane);
    } else if (MODE == 1) {
      h = mix(h + it);
      const size_t c = (size_t)(h & (nchunk / 4 - 1)) * 4;
      uint2* p = reinterpret_cast<uint2*>(out + c * 16) + lane;
      *p = make_uint2(it, lane);
    } else if (MODE == 2) {
      h = mix(h + it);
      const size_t c = (size_t)(h & (nchunk / 8 - 1)) * 8;
      uint4* p = reinterpret_cast<uint4*>(out + c * 16) + lane;
      *p = make_uint4(it, lane, 0, 1);
    } else {
      h = mix(h + it);
      const size_t c = (size_t)(mix(h + (lane >> 2)) & (nchunk - 1));
      uint4* p = reinterpret_cast<uint4*>(out + c * 16) + (lane & 3);
      *p = make_uint4(it, lane, 0, 1);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  const size_t words = (size_t)1 << 30;  // 4 GB
  uint32_t* out; cudaMalloc(&out, words * 4);
  unsigned long long* cyc; cudaMallocManaged(&cyc, 148 * 8);
  const int iters = 20000;
  for (size_t span : {(size_t)1 << 24, (size_t)1 << 30})
  for (int mode = 0; mode < 4; ++mode)
    for (int grid : {1, 148})
      for (int aw : {4, 8, 16}) {
        for (int rep = 0; rep < 2; ++rep) {
          if (mode == 0) k<0><<<grid, 512>>>(out, words, iters, cyc, aw, span);
          if (mode == 1) k<1><<<grid, 512>>>(out, words, iters, cyc, aw, span);
          if (mode == 2) k<2><<<grid, 512>>>(out, words, iters, cyc, aw, span);
          if (mode == 3) k<3><<<grid, 512>>>(out, words, iters, cyc, aw, span);
          cudaDeviceSynchronize();
        }
        double c = 0; for (int i = 0; i < grid; ++i) c += cyc[i]; c /= grid;
        const double bytes = (double)iters * aw * 32 * (mode >= 2 ? 16 : 8);
        printf("span %zu MB mode %d grid %3d warps %2d: %.1f B/clk/SM  (%.0f cycles)\n", span >> 18, mode, grid, aw, bytes / c, c);
      }
  return 0;
}
