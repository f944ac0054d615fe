// Micro-probe (sm_100a): MUFU ex2 throughput per SMSP for f32 / f16x2 / bf16x2 operands, and
// tcgen05.mma kind::f16 M=128 N=128 K=16 cycles per instruction for SS (A and B in shared
// memory) and TS (A in TMEM) operands, alone and with 8 warps streaming shared-memory stores
// (the softmax P stores / TMA fills of the attention kernel). Informs the attention kernel's
// design. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include
//   -I../../paper_2512_04025_b200/csrc mufu_mma_probe.cu -o /tmp/mufu_mma_probe -lcuda
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

using namespace psa;

template <int MODE>
__global__ void mufu_kernel(float* out, long long* cyc, int iters) {
  uint32_t r[8];
  for (int i = 0; i < 8; ++i) {
    float a = -0.1f * (threadIdx.x % 7 + i);
    if (MODE == 0) r[i] = __float_as_uint(a);
    else r[i] = MODE == 1 ? 0xB800B800u : 0xBE00BE00u;  // f16 -0.5 pairs / bf16 -0.125 pairs
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint_as_float(r[i])));
        r[i] = __float_as_uint(y - 1.25f);
      } else if (MODE == 1) {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(r[i]));
        r[i] = y ^ 0x80008000u;  // negate both halves (stay in (-1, 0])
      } else {
        uint32_t y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(r[i]));
        r[i] = y ^ 0x80008000u;
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(acc);
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

struct MmaSmem {
  uint8_t a[128 * 64 * 2];
  uint8_t b[128 * 64 * 2];
  uint8_t scratch[8][32 * 16 * 16];  // per-store-warp 8 KB
  uint64_t done;
  uint64_t dummy[2];
  uint32_t tmem;
};

// MODE 0: SS; MODE 1: TS (A from TMEM). STORES: 8 warps stream 16-byte shared stores meanwhile.
template <int MODE, int STORES>
__global__ void __launch_bounds__(384, 1) mma_kernel(long long* cyc, int iters) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<MmaSmem*>(smem_raw);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (int)sizeof(sm.a) / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(sm.a)[i] = 0x3C003C00u ^ (i * 2654435761u & 0x00070007u);
    reinterpret_cast<uint32_t*>(sm.b)[i] = 0x3C003C00u ^ (i * 40503u & 0x00070007u);
  }
  if (threadIdx.x == 0) {
    mbar_init(&sm.done, 1);
    mbar_init(&sm.dummy[0], 1 << 20);
    mbar_init(&sm.dummy[1], 1 << 20);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&sm.tmem, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
    const uint64_t ad = umma_desc_sw128(smem_u32(sm.a), 16, 1024);
    const uint64_t bd = umma_desc_sw128(smem_u32(sm.b), 16, 1024);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t koff = (kk * 32) >> 4;
          if (MODE == 0 || MODE == 2)
            mma_bf16_ss(tmem, ad + koff, bd + koff, idesc, 1u);
          else
            mma_bf16_ts(tmem, tmem + 256 + kk * 8, bd + koff, idesc, 1u);
        }
        if (MODE == 2 && (it % 2 == 1)) {  // 8 MMAs then 2 commits, like the attention kernel
          mma_commit(&sm.dummy[0]);
          mma_commit(&sm.dummy[1]);
        }
      }
      mma_commit(&sm.done);
    }
    __syncwarp();
    mbar_wait(&sm.done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      cyc[blockIdx.x] = t1 - t0;
      stop = 1;
    }
  } else if (STORES == 2 && (warp == 5 || warp == 9 || warp == 6 || warp == 10)) {
    // TMEM traffic of softmax warps on the MMA warp's sub-partition (warp 1 -> SMSP 1): LDTM x32
    // of S and STTM x32 of P in a loop (lanes of this warp's TMEM quarter)
    const uint32_t tl = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 384;
    uint32_t v[32];
    for (int e = 0; e < 32; ++e) v[e] = e;
    while (!stop) {
      tmem_ld32(tl, v);
      tmem_ld_wait(v);
      for (int e = 0; e < 32; ++e) v[e] += 1;
      tmem_st32(tl + 64, v);
      tmem_st_wait();
    }
  } else if (STORES == 1 && warp >= 4) {
    uint4* dst = reinterpret_cast<uint4*>(sm.scratch[warp - 4]);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 16; ++i) dst[i * 32 + (threadIdx.x & 31)] = v;
      v.x += 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
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

template <int MODE>
void run_mufu(const char* name, int warps_per_smsp) {
  const int blocks = 148, threads = 128 * warps_per_smsp, iters = 4096;
  float* out;
  long long* cyc;
  CK(cudaMalloc(&out, blocks * threads * 4));
  CK(cudaMalloc(&cyc, blocks * threads / 32 * 8));
  mufu_kernel<MODE><<<blocks, threads>>>(out, cyc, iters);
  CK(cudaDeviceSynchronize());
  mufu_kernel<MODE><<<blocks, threads>>>(out, cyc, iters);
  CK(cudaDeviceSynchronize());
  long long h[148 * 32];
  CK(cudaMemcpy(h, cyc, blocks * threads / 32 * 8, cudaMemcpyDeviceToHost));
  double mx = 0;
  for (int i = 0; i < blocks * threads / 32; ++i) mx = h[i] > mx ? h[i] : mx;
  const double instr_per_smsp = double(iters) * 8 * warps_per_smsp;  // warp-instructions
  printf("MUFU %-8s warps/SMSP=%d: %.2f cycles per warp-instruction per SMSP (%.1f lanes/clk/SM)\n",
         name, warps_per_smsp, mx / instr_per_smsp, 4 * 32 * instr_per_smsp / mx);
  cudaFree(out);
  cudaFree(cyc);
}

template <int MODE, int STORES>
void run_mma(const char* name) {
  const int iters = 4096;
  long long* cyc;
  CK(cudaMalloc(&cyc, 148 * 8));
  auto k = mma_kernel<MODE, STORES>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MmaSmem)));
  k<<<148, 384, sizeof(MmaSmem)>>>(cyc, iters);
  CK(cudaDeviceSynchronize());
  k<<<148, 384, sizeof(MmaSmem)>>>(cyc, iters);
  CK(cudaDeviceSynchronize());
  long long h[148];
  CK(cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost));
  double mx = 0, mn = 1e30;
  for (int i = 0; i < 148; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    mn = h[i] < mn ? h[i] : mn;
  }
  printf("MMA %-22s: %.1f cycles per 128x128x16 (min SM %.1f)\n", name, mx / (iters * 4.0),
         mn / (iters * 4.0));
  cudaFree(cyc);
}

int main() {
  run_mufu<0>("f32", 1);
  run_mufu<0>("f32", 2);
  run_mufu<1>("f16x2", 1);
  run_mufu<1>("f16x2", 2);
  run_mufu<2>("bf16x2", 1);
  run_mufu<2>("bf16x2", 2);
  run_mma<0, 0>("SS");
  run_mma<1, 0>("TS");
  run_mma<2, 0>("SS + 2 commits / 8 MMAs");
  run_mma<0, 1>("SS + 8 warps STS.128");
  run_mma<0, 2>("SS + TMEM ld/st warps (SMSP1,2)");
  run_mma<2, 2>("SS+commits + TMEM ld/st");
  return 0;
}
