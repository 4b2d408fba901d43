// Memory-pattern microbenchmarks on B200 (scratch tool, not product):
// what the scatter / local-sort data movement costs without any ranking.
//   mode 0: LDG.128 -> STG.128 copy (reference)
//   mode 1: persistent, TMA tile in (single buffer) -> coalesced STG out
//   mode 2: persistent, TMA tile in (double buffer) -> coalesced STG out
//   mode 3: persistent, TMA tile in (single buffer) -> STG in bucket runs
//           (NBK buckets; tile t's run for bucket r lands after tile t-1's)
//   mode 4: mode 3 with double buffering
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb_mem tools/mb_mem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 512, IPT = 9, T = NT * IPT;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(par)
      : "memory");
}

__global__ void k_copy(const uint4* a, uint4* b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <int MODE, int NBK, int CH = 8>
__global__ void __launch_bounds__(NT, 2) k_tile(const uint32_t* kin, const uint32_t* vin, uint32_t* kout,
                                                 uint32_t* vout, uint32_t ntile) {
  constexpr bool DB = (MODE == 2 || MODE == 4 || MODE == 6);
  constexpr bool STRIPE = MODE >= 5;  // CTA c takes tiles [c*tpc, (c+1)*tpc)
  // mode 7: stripes; each bucket stream gets whole 32-byte sectors only
  // (8 consecutive records of one bucket per 8 lanes): the write pattern of
  // an SMEM write-combined scatter
  extern __shared__ __align__(16) unsigned char sm[];
  uint32_t* sk[2] = {reinterpret_cast<uint32_t*>(sm), reinterpret_cast<uint32_t*>(sm + 2 * T * 4)};
  uint32_t* sv[2] = {reinterpret_cast<uint32_t*>(sm + T * 4), reinterpret_cast<uint32_t*>(sm + 3 * T * 4)};
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t ph[2] = {0, 0};
  int cur = 0;
  auto issue = [&](uint32_t t, int b) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    expect_tx(&bar[b], 2 * T * 4);
    tma1d(sk[b], kin + (size_t)t * T, T * 4, &bar[b]);
    tma1d(sv[b], vin + (size_t)t * T, T * 4, &bar[b]);
  };
  const uint32_t tpc = (ntile + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = STRIPE ? blockIdx.x * tpc : blockIdx.x;
  const uint32_t tend = STRIPE ? min(ntile, t0 + tpc) : ntile;
  const uint32_t step = STRIPE ? 1u : gridDim.x;
  if (DB && tid == 0 && t0 < tend) issue(t0, 0);
  for (uint32_t t = t0; t < tend; t += step) {
    const int b = DB ? cur : 0;
    if (tid == 0) {
      if (DB) {
        if (t + step < tend) issue(t + step, cur ^ 1);
      } else {
        issue(t, 0);
      }
    }
    mwait(&bar[b], ph[b]);
    ph[b] ^= 1;
    if (MODE == 1 || MODE == 2) {
      uint32_t* ko = kout + (size_t)t * T;
      uint32_t* vo = vout + (size_t)t * T;
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const int p = i * NT + tid;
        ko[p] = sk[b][p];
        vo[p] = sv[b][p];
      }
    } else if (MODE == 7) {
      // bucket r's stream: this CTA's region [(r * G + c) * tpc * T/NBK, ...),
      // tile t (i-th of the stripe) appends T/NBK records as whole sectors
      constexpr int L = T / NBK;
      const uint32_t i0 = t - t0;
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const int p = i * NT + tid;           // p-th record of the tile
        const uint32_t sec = p / CH, j = p % CH;
        const uint32_t r = sec % NBK;         // chunks round-robin over buckets
        const uint32_t k = sec / NBK;         // k-th chunk of bucket r in this tile
        const size_t d = (((size_t)r * gridDim.x + blockIdx.x) * tpc + i0) * (size_t)L + k * CH + j;
        kout[d] = sk[b][p];
        vout[d] = sv[b][p];
      }
    } else {
      // bucket r holds runs of L = T / NBK records; its region is
      // [r * ntile * L, (r+1) * ntile * L), tile t writes run t
      constexpr int L = T / NBK;
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const int p = i * NT + tid;
        const uint32_t r = p / L, q = p % L;
        const size_t d = ((size_t)r * ntile + t) * L + q;
        kout[d] = sk[b][p];
        vout[d] = sv[b][p];
      }
    }
    __syncthreads();
    cur ^= 1;
  }
}

template <int MODE, int NBK, int CH = 8>
float run_tile(const uint32_t* k, const uint32_t* v, uint32_t* ko, uint32_t* vo, uint32_t ntile, int sms, int per = 2) {
  auto fn = k_tile<MODE, NBK, CH>;
  const int smb = 4 * T * 4;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    fn<<<per * sms, NT, smb>>>(k, v, ko, vo, ntile);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t ntile = 1000000000u / T;
  const size_t n = (size_t)ntile * T;
  uint32_t *k, *v, *ko, *vo;
  cudaMalloc(&k, n * 4);
  cudaMalloc(&v, n * 4);
  const size_t nout = n + (size_t)2 * sms * 2 * T * 4;  // stripe-rounding slack
  cudaMalloc(&ko, nout * 4);
  cudaMalloc(&vo, nout * 4);
  cudaMemset(k, 1, n * 4);
  cudaMemset(v, 2, n * 4);
  const double bytes = 16.0 * n;
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      k_copy<<<sms * 8, 512>>>((const uint4*)k, (uint4*)ko, n / 4);
      k_copy<<<sms * 8, 512>>>((const uint4*)v, (uint4*)vo, n / 4);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("mode0 copy LDG/STG.128            %7.3f ms  %7.1f GB/s\n", best, bytes / best / 1e6);
  }
  float ms;
  ms = run_tile<1, 512>(k, v, ko, vo, ntile, sms);
  printf("mode1 TMA single -> coalesced      %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<2, 512>(k, v, ko, vo, ntile, sms);
  printf("mode2 TMA double -> coalesced      %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<3, 512>(k, v, ko, vo, ntile, sms);
  printf("mode3 TMA single -> 512 runs of 9  %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<4, 512>(k, v, ko, vo, ntile, sms);
  printf("mode4 TMA double -> 512 runs of 9  %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<3, 256>(k, v, ko, vo, ntile, sms);
  printf("mode3 TMA single -> 256 runs of 18 %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<4, 1024>(k, v, ko, vo, ntile, sms);
  printf("mode4 TMA double -> 1024 runs of 4 %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<4, 128>(k, v, ko, vo, ntile, sms);
  printf("mode4 TMA double -> 128 runs of 36 %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<5, 512>(k, v, ko, vo, ntile, sms);
  printf("mode5 stripes single -> 512 runs   %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<6, 512>(k, v, ko, vo, ntile, sms);
  printf("mode6 stripes double -> 512 runs   %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<6, 1024>(k, v, ko, vo, ntile, sms);
  printf("mode6 stripes double -> 1024 runs  %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<7, 576>(k, v, ko, vo, ntile, sms);
  printf("mode7 stripes, full sectors, 576 streams %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<7, 144>(k, v, ko, vo, ntile, sms);
  printf("mode7 stripes, full sectors, 144 streams %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<7, 288, 16>(k, v, ko, vo, ntile, sms);
  printf("mode7 stripes, 64B chunks, 288 streams %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<7, 144, 32>(k, v, ko, vo, ntile, sms);
  printf("mode7 stripes, 128B chunks, 144 streams %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<7, 288, 16>(k, v, ko, vo, ntile, sms, 1);
  printf("mode7 1 CTA/SM, 64B chunks, 288 streams %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<7, 144, 32>(k, v, ko, vo, ntile, sms, 1);
  printf("mode7 1 CTA/SM, 128B chunks, 144 streams %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<2, 512>(k, v, ko, vo, ntile, sms, 1);
  printf("mode2 1 CTA/SM TMA double -> coalesced %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  ms = run_tile<7, 72, 64>(k, v, ko, vo, ntile, sms);
  printf("mode7 stripes, 256B chunks, 72 streams %7.3f ms  %7.1f GB/s\n", ms, bytes / ms / 1e6);
  return 0;
}
