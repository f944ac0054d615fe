// Micro-probe (sm_100a): the attention kernel's K/V load pattern without compute. Two producer
// warps (K and V) each stream 32 KB tiles (two 128-row x 64-column boxes, 128B swizzle) into a
// 2-stage ring, issuing tile t+2 once tile t has landed; rows are random in an L2-resident (or
// HBM-sized) tensor. Prints cycles per tile pair and B/clk per SM for: boxes from one lane vs two
// lanes, L2-resident vs 4 GB source. Informs DESIGN.md §3 K4.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2512_04025_b200/csrc
//   tma_pattern_probe.cu -o tma_pattern_probe -lcuda
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
  uint8_t ring[2][2][32768];  // [producer][stage][tile]
  uint64_t full[2][2];
};

template <int LANES, int STAGES>
__global__ void __launch_bounds__(64, 1)
    probe(const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv,
          int rows_total, int tiles, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int p = 0; p < 2; ++p)
      for (int s = 0; s < 2; ++s) mbar_init(&sm.full[p][s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const CUtensorMap* map = warp == 0 ? &mk : &mv;
  unsigned rng = 12345u + blockIdx.x * 7919u + warp * 104729u;
  const long long t0 = clock64();
  for (int t = 0; t < tiles + STAGES; ++t) {
    const int s = t % STAGES;
    if (t >= STAGES) mbar_wait(&sm.full[warp][s], ((t - STAGES) / STAGES) & 1);  // landed: reuse
    if (t < tiles) {
      rng = rng * 1664525u + 1013904223u;
      const int row = static_cast<int>((rng >> 3) % static_cast<unsigned>(rows_total - 128));
      if (lane == 0) mbar_arrive_expect_tx(&sm.full[warp][s], 32768);
      __syncwarp();
      for (int c = 0; c < 2; ++c)
        if ((LANES == 1 && lane == 0) || (LANES == 2 && lane == c))
          tma_load_2d(map, &sm.full[warp][s], sm.ring[warp][s] + c * 16384, c * 64, row);
    }
  }
  const long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 2 + warp] = t1 - t0;
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fnp);
  long long* out;
  cudaMalloc(&out, 148 * 2 * 8);
  for (int big = 0; big < 2; ++big) {
    const int rows_total = big ? 16000000 : 100000;  // 4 GB (HBM) or 25.6 MB (L2) per tensor
    void *bk, *bv;
    cudaMalloc(&bk, static_cast<size_t>(rows_total) * 256);
    cudaMalloc(&bv, static_cast<size_t>(rows_total) * 256);
    cudaMemset(bk, 0, static_cast<size_t>(rows_total) * 256);
    cudaMemset(bv, 0, static_cast<size_t>(rows_total) * 256);
    CUtensorMap mk, mv;
    cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows_total)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    for (int m = 0; m < 2; ++m)
      if (enc(m ? &mv : &mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m ? bv : bk, dims, strides, box,
              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
      }
    const int tiles = 1024;
    for (int variant = 0; variant < 2; ++variant) {
      auto k = variant == 0 ? probe<1, 2> : probe<2, 2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
      for (int r = 0; r < 2; ++r) k<<<148, 64, sizeof(Smem)>>>(mk, mv, rows_total, tiles, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
      }
      std::vector<long long> h(296);
      cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (long long v : h) mx = v > mx ? v : mx;
      printf("%s source, boxes from %d lane(s), 2 stages per producer: %.0f cycles per K+V tile pair, "
             "%.1f B/clk/SM\n", big ? "4 GB (HBM)" : "25.6 MB (L2)", variant + 1, mx / tiles,
             tiles * 65536.0 / mx);
    }
    cudaFree(bk);
    cudaFree(bv);
  }
  return 0;
}
