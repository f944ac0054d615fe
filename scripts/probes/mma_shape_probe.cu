// Micro-probe (sm_100a): tcgen05.mma kind::f16 (bf16, SS, K-major SW128) throughput for
// M=128 and N = 64 / 128 / 256, and the latency from issuing a K=128 chain (8 MMAs) to its
// commit landing on an mbarrier, for N=128 and for an N=64 half. Informs whether the attention
// S tile can be split into key halves.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2512_04025_b200/csrc
//   mma_shape_probe.cu -o /tmp/mma_shape_probe -lcuda
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

using namespace psa;

struct Smem {
  uint8_t a[128 * 128 * 2];  // 128 rows x 128 K (two 64-wide SW128 atoms)
  uint8_t b[256 * 128 * 2];
  uint64_t done;
  uint32_t tmem;
};

template <int N>
__global__ void __launch_bounds__(128, 1) thr_kernel(long long* cyc, int iters) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<Smem*>(smem_raw);
  for (int i = threadIdx.x; i < (int)sizeof(sm.a) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm.a)[i] = 0x3C003C00u;
  for (int i = threadIdx.x; i < (int)sizeof(sm.b) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm.b)[i] = 0x3C003C00u;
  if (threadIdx.x == 0) {
    mbar_init(&sm.done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    tmem_alloc(&sm.tmem, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  if (threadIdx.x < 32) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint64_t ad = umma_desc_sw128(smem_u32(sm.a), 16, 1024);
    const uint64_t bd = umma_desc_sw128(smem_u32(sm.b), 16, 1024);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tmem, ad + ((kk * 32) >> 4), bd + ((kk * 32) >> 4), idesc, 1u);
      }
      mma_commit(&sm.done);
    }
    __syncwarp();
    mbar_wait(&sm.done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// latency: chain of 8 K=16 MMAs (K = 128) at width N, commit, wait; repeated, averaged
template <int N>
__global__ void __launch_bounds__(128, 1) lat_kernel(long long* cyc, int iters) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<Smem*>(smem_raw);
  for (int i = threadIdx.x; i < (int)sizeof(sm.a) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm.a)[i] = 0x3C003C00u;
  for (int i = threadIdx.x; i < (int)sizeof(sm.b) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm.b)[i] = 0x3C003C00u;
  if (threadIdx.x == 0) {
    mbar_init(&sm.done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    tmem_alloc(&sm.tmem, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  if (threadIdx.x < 32) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint64_t ad = umma_desc_sw128(smem_u32(sm.a), 16, 1024);
    const uint64_t bd = umma_desc_sw128(smem_u32(sm.b), 16, 1024);
    long long tot = 0;
    for (int it = 0; it < iters; ++it) {
      long long t0 = clock64();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = ((kk >> 2) * 128 * 128 + (kk & 3) * 32) >> 4;
          mma_bf16_ss(tmem, ad + koff, bd + koff, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sm.done);
      }
      __syncwarp();
      mbar_wait(&sm.done, it & 1);
      tot += clock64() - t0;
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

#define CK(x)                                                           \
  do {                                                                  \
    cudaError_t e = (x);                                                \
    if (e != cudaSuccess) {                                             \
      printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); \
      exit(1);                                                          \
    }                                                                   \
  } while (0)

template <int N>
void run() {
  long long* cyc;
  CK(cudaMalloc(&cyc, 148 * 8));
  long long h[148];
  const int iters = 4096;
  auto k = thr_kernel<N>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
  for (int r = 0; r < 2; ++r) k<<<148, 128, sizeof(Smem)>>>(cyc, iters);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("SS M=128 N=%3d K=16: %.1f cycles per MMA (%.0f MAC/clk)\n", N, mx / (iters * 4.0),
         128.0 * N * 16 * iters * 4 / mx);
  auto l = lat_kernel<N>;
  CK(cudaFuncSetAttribute(l, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
  for (int r = 0; r < 2; ++r) l<<<148, 128, sizeof(Smem)>>>(cyc, 256);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
  printf("   issue -> commit landed, 8 MMAs (K=128) at N=%3d: %.0f cycles\n", N, mean);
  cudaFree(cyc);
}

int main() {
  run<64>();
  run<128>();
  run<256>();
  return 0;
}
