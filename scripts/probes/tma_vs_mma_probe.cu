// Micro-probe (sm_100a): does a busy tensor core slow TMA fills of shared memory? One warp keeps
// issuing tcgen05.mma M=128 N=128 K=16 (SS: A and B from shared memory, 8 KB of operand reads per
// 64 cycles; or TS: A from TMEM) while one thread streams 16 KB TMA boxes (128 rows x 128 B, L2
// resident, 4-slot ring, 2 in flight) into shared memory; prints the TMA bytes/clk per SM with
// the tensor core idle, SS-busy and TS-busy. Informs the attention kernel (DESIGN.md §3 K4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2512_04025_b200/csrc
//   tma_vs_mma_probe.cu -o tma_vs_mma_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace psa;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

struct Smem {
  uint8_t a[128 * 64 * 2];
  uint8_t b[128 * 64 * 2];
  uint8_t ring[4][16384];
  uint64_t bars[4];
  uint64_t done;
  uint32_t tmem;
  volatile int stop;
};

template <int MODE>  // 0: tensor idle, 1: SS MMAs, 2: TS MMAs
__global__ void __launch_bounds__(128, 1)
    probe(const __grid_constant__ CUtensorMap map, int rows_total, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (int)sizeof(sm.a) / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(sm.a)[i] = 0x3C003C00u;
    reinterpret_cast<uint32_t*>(sm.b)[i] = 0x3C003C00u;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) mbar_init(&sm.bars[s], 1);
    mbar_init(&sm.done, 1);
    sm.stop = 0;
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
  if (warp == 0 && MODE > 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
    const uint64_t ad = umma_desc_sw128(smem_u32(sm.a), 16, 1024);
    const uint64_t bd = umma_desc_sw128(smem_u32(sm.b), 16, 1024);
    int rounds = 0;
    while (!sm.stop) {
      if (elect_one()) {
        for (int it = 0; it < 16; ++it)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t koff = (kk * 32) >> 4;
            if (MODE == 1) mma_bf16_ss(tmem, ad + koff, bd + koff, idesc, 1u);
            else mma_bf16_ts(tmem, tmem + 256 + kk * 8, bd + koff, idesc, 1u);
          }
        mma_commit(&sm.done);
      }
      __syncwarp();
      mbar_wait(&sm.done, rounds & 1);
      ++rounds;
    }
  } else if (warp == 1 && threadIdx.x == 32) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    unsigned rng = 12345u + blockIdx.x * 7919u;
    const long long t0 = clock64();
    for (int it = 0; it < iters + 2; ++it) {
      const int s = it % 4;
      if (it >= 2) mbar_wait(&sm.bars[(it - 2) % 4], ((it - 2) / 4) & 1);
      if (it < iters) {
        rng = rng * 1664525u + 1013904223u;
        const int row = (rng >> 4) % (rows_total - 128);
        mbar_arrive_expect_tx(&sm.bars[s], 16384);
        tma_load_2d(&map, &sm.bars[s], sm.ring[s], 0, row);
      }
    }
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    sm.stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fnp);
  const int rows_total = 200000;  // 25.6 MB: L2 resident
  void* buf;
  cudaMalloc(&buf, static_cast<size_t>(rows_total) * 128);
  cudaMemset(buf, 0, static_cast<size_t>(rows_total) * 128);
  CUtensorMap map;
  cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows_total)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  long long* out;
  cudaMalloc(&out, 148 * 8);
  const int iters = 2048;
  const char* names[3] = {"tensor idle", "SS MMAs (A, B in smem)", "TS MMAs (A in TMEM)"};
  for (int mode = 0; mode < 3; ++mode) {
    auto k = mode == 0 ? probe<0> : (mode == 1 ? probe<1> : probe<2>);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    for (int r = 0; r < 2; ++r) k<<<148, 128, sizeof(Smem)>>>(map, rows_total, iters, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (long long v : h) mx = v > mx ? v : mx;
    printf("%-26s: TMA %.1f B/clk/SM (16 KB boxes, 2 in flight, one thread)\n", names[mode],
           double(iters) * 16384 / mx);
  }
  return 0;
}
