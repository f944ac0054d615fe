// Micro-probe (sm_100a): does tcgen05.mma operand traffic share shared-memory bandwidth with TMA
// fills? Warp 0 streams M=128 N=128 K=16 bf16 MMAs (SS: A and B from smem; TS: A from TMEM),
// warps 1..3 stream 16 KB TMA boxes from an L2-resident tensor into their own smem ring (depth 2).
// Reports MMA cycles per instruction and TMA bytes per clock per SM, alone and together.
#include <cstdio>
#include <vector>
#include "common.cuh"
using namespace psa;
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
struct Sm {
  uint8_t a[16384];
  uint8_t b[16384];
  uint8_t ring[3][2][16384];
  uint64_t bars[3][2];
  uint64_t done;
  uint32_t tmem;
  int stop;
};
// mode bit0: MMA on (bit1: TS), bit2: TMA on
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap map, int rows_total,
                                            int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Sm& sm = *reinterpret_cast<Sm*>(raw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 3; ++w)
      for (int s = 0; s < 2; ++s) mbar_init(&sm.bars[w][s], 1);
    mbar_init(&sm.done, 1);
    sm.stop = 0;
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&sm.tmem, 512);
    tmem_relinquish();
  }
  for (int i = threadIdx.x; i < 2 * 16384 / 4; i += 128) reinterpret_cast<uint32_t*>(sm.a)[i] = 0x3C003C00u;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  volatile int* stop = &sm.stop;
  if (warp == 0) {
    long long t0 = clock64();
    if (mode & 1) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
      const uint64_t ad = umma_desc_sw128(smem_u32(sm.a), 16, 1024);
      const uint64_t bd = umma_desc_sw128(smem_u32(sm.b), 16, 1024);
      if (elect_one()) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (mode & 2) mma_bf16_ts(tmem, tmem + 256 + kk * 8, bd + ((kk * 32) >> 4), idesc, 1u);
            else mma_bf16_ss(tmem, ad + ((kk * 32) >> 4), bd + ((kk * 32) >> 4), idesc, 1u);
          }
        mma_commit(&sm.done);
      }
      __syncwarp();
      mbar_wait(&sm.done, 0);
    } else {
      while (clock64() - t0 < (long long)iters * 4 * 64) { }
    }
    long long t1 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 4] = t1 - t0;
      *stop = 1;
    }
  } else if ((mode & 4) && lane == 0) {
    const int w = warp - 1;
    unsigned rng = 99u + blockIdx.x * 7919u + w * 31u;
    long long bytes = 0;
    for (int it = 0; ; ++it) {
      const int s = it & 1;
      if (it >= 2) mbar_wait(&sm.bars[w][s], ((it >> 1) - 1) & 1);
      if (*stop) break;
      rng = rng * 1664525u + 1013904223u;
      const int row = (rng >> 4) % (rows_total - 128);
      mbar_arrive_expect_tx(&sm.bars[w][s], 16384);
      tma_load_2d(&map, &sm.bars[w][s], sm.ring[w][s], 0, row);
      if (it >= 2) bytes += 16384;
    }
    out[blockIdx.x * 4 + 1 + w] = bytes;
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
  const int rows_total = 200000;
  void* buf;
  cudaMalloc(&buf, size_t(rows_total) * 128);
  cudaMemset(buf, 0, size_t(rows_total) * 128);
  long long* out;
  cudaMalloc(&out, 148 * 4 * 8);
  CUtensorMap map;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(Sm));
  const char* names[] = {"", "SS MMA alone", "", "TS MMA alone", "TMA alone (3 warps)", "SS MMA + TMA", "", "TS MMA + TMA"};
  for (int mode : {1, 3, 4, 5, 7}) {
    const int iters = 8192;
    for (int rep = 0; rep < 2; ++rep) k<<<148, 128, sizeof(Sm)>>>(map, rows_total, mode, iters, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<long long> h(148 * 4);
    cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    double cyc = 0, bytes = 0;
    for (int b = 0; b < 148; ++b) {
      cyc += h[b * 4] / 148.0;
      bytes += (h[b * 4 + 1] + h[b * 4 + 2] + h[b * 4 + 3]) / 148.0;
    }
    printf("%-20s: %.1f cycles per MMA, TMA %.1f B/clk/SM\n", names[mode], cyc / (iters * 4.0),
           (mode & 4) ? bytes / cyc : 0.0);
  }
  return 0;
}
