// Micro-probe (sm_100a): TMA tile-load latency and L2->SM bandwidth with every SM streaming
// 2D boxes (128 B wide rows, bf16 [rows, 64] boxes, 128B swizzle) from an L2-resident tensor, with
// `depth` loads in flight per SM. Mirrors the attention kernel's K/V tile traffic.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace psa;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

__global__ void __launch_bounds__(128, 1)
    tma_kernel(const __grid_constant__ CUtensorMap map, int rows_total, int box_rows, int depth,
               int iters, long long* out, int issuers) {
  extern __shared__ __align__(1024) unsigned char smem_all[];
  const bool lanes = issuers > 100;
  const int n_iss = lanes ? issuers - 100 : issuers;
  const int w = lanes ? (threadIdx.x < 32 ? threadIdx.x : 99) : (threadIdx.x % 32 == 0 ? threadIdx.x / 32 : 99);
  unsigned char* smem = smem_all + (w < n_iss ? w : 0) * (8 / n_iss) * 16384;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_all + 8 * 16384) + w * 8;
  if (w < n_iss) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    for (int s = 0; s < 8; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (w < n_iss) {
    const uint32_t bytes = box_rows * 128;
    unsigned rng = 12345u + blockIdx.x * 7919u + w * 104729u;
    long long lat_sum = 0;
    const long long t0 = clock64();
    long long issue[8];
    for (int it = 0; it < iters + depth; ++it) {
      const int s = it % depth;
      if (it >= depth) {  // retire the load issued depth iterations ago
        mbar_wait(&bars[s], ((it / depth) - 1) & 1);
        lat_sum += clock64() - issue[s];
      }
      if (it < iters) {
        rng = rng * 1664525u + 1013904223u;
        const int row = (rng >> 4) % (rows_total - box_rows);
        issue[s] = clock64();
        mbar_arrive_expect_tx(&bars[s], bytes);
        tma_load_2d(&map, &bars[s], smem + s * 16384, 0, row);
      }
    }
    const long long t1 = clock64();
    if (w == 0) {
      out[blockIdx.x * 2 + 0] = t1 - t0;
      out[blockIdx.x * 2 + 1] = lat_sum / iters;
    }
  }
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fnp);
  const int rows_total = 200000;  // 200000 x 64 bf16 = 25.6 MB (L2-resident)
  void* buf;
  cudaMalloc(&buf, static_cast<size_t>(rows_total) * 128);
  cudaMemset(buf, 0, static_cast<size_t>(rows_total) * 128);
  long long* out;
  cudaMalloc(&out, 148 * 2 * 8);
  auto kern = tma_kernel;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 512);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (int box_rows : {128, 64, 16}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows_total)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      return 1;
    }
    for (int cfgi = 0; cfgi < 6; ++cfgi) {
      const int issuers = cfgi < 2 ? 1 : (cfgi == 2 ? 4 : (cfgi == 3 ? 102 : (cfgi == 4 ? 104 : 108)));
      const int depth = cfgi < 2 ? (1 << cfgi) : (cfgi == 5 ? 1 : 2);
      const int iters = 2048;
      for (int rep = 0; rep < 2; ++rep)
        kern<<<148, 128, 8 * 16384 + 512>>>(map, rows_total, box_rows, depth, iters, out, issuers);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
      }
      std::vector<long long> h(148 * 2);
      cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
      double cyc = 0, lat = 0;
      for (int b = 0; b < 148; ++b) {
        cyc = h[2 * b] > cyc ? h[2 * b] : cyc;
        lat += h[2 * b + 1] / 148.0;
      }
      const int n_iss = issuers > 100 ? issuers - 100 : issuers;
      const double bytes_per_sm_clk = double(iters) * n_iss * box_rows * 128 / cyc;
      printf("box %3d rows (%5d B) issuers %d%s x depth %d: %.1f B/clk/SM, mean issue->landed %.0f clk\n",
             box_rows, box_rows * 128, n_iss, issuers > 100 ? " lanes of 1 warp" : " warps", depth, bytes_per_sm_clk, lat);
    }
  }
  return 0;
}
