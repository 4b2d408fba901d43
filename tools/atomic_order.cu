// Does B200 serve same-address shared atomics of one warp instruction in lane order? (probe)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void k(unsigned long long* viol, unsigned long long* coll, int iters, int nb) {
  __shared__ uint32_t c[8][1024];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * 1024; i += 256) (&c[0][0])[i] = 0;
  __syncthreads();
  unsigned long long v = 0, cc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t b = hash32((blockIdx.x * 256 + threadIdx.x) * 131 + it * 7919) % nb;
    const uint32_t old = atomicAdd(&c[w][b], 1u);
    __syncwarp();
    // check: every lower lane with the same bucket must have a smaller old
    for (int j = 0; j < 32; ++j) {
      const uint32_t bj = __shfl_sync(0xffffffffu, b, j), oj = __shfl_sync(0xffffffffu, old, j);
      if (j < lane && bj == b) { ++cc; if (oj > old) ++v; }
    }
    __syncwarp();
  }
  atomicAdd(viol, v); atomicAdd(coll, cc);
}
int main() {
  unsigned long long *v, *c; cudaMalloc(&v, 8); cudaMalloc(&c, 8);
  for (int nb : {2, 32, 512, 1024}) {
    cudaMemset(v, 0, 8); cudaMemset(c, 0, 8);
    k<<<148 * 8, 256>>>(v, c, 2000, nb);
    unsigned long long hv, hc; cudaMemcpy(&hv, v, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("nb=%4d colliding pairs=%llu out-of-lane-order=%llu\n", nb, hc, hv);
  }
  // also 16-bit packed variant
  return 0;
}
