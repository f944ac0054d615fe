// Micro-probe (sm_100a): does a thread's cp.async.bulk.tensor issue block while its previous TMA
// loads are in flight? One thread issues 8 loads back to back (each on its own mbarrier) and
// stamps clock64 after each issue, then waits all. Every SM runs it concurrently.
#include <cstdio>
#include <vector>
#include "common.cuh"
using namespace psa;
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap map, int rows_total,
                                           int box_rows, int two_threads, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 8 * 16384);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const bool issuer = threadIdx.x == 0 || (two_threads && threadIdx.x == 1);
  if (issuer) {
    long long st[9];
    unsigned rng = 777u + blockIdx.x * 7919u + threadIdx.x * 31u;
    st[0] = clock64();
    for (int s = threadIdx.x; s < 8; s += (two_threads ? 2 : 1)) {
      rng = rng * 1664525u + 1013904223u;
      const int row = (rng >> 4) % (rows_total - box_rows);
      mbar_arrive_expect_tx(&bars[s], box_rows * 128);
      tma_load_2d(&map, &bars[s], smem + s * 16384, 0, row);
      st[s + 1] = clock64();
    }
    for (int s = threadIdx.x; s < 8; s += (two_threads ? 2 : 1)) mbar_wait(&bars[s], 0);
    const long long done = clock64();
    if (blockIdx.x == 5)
      for (int s = threadIdx.x; s < 8; s += (two_threads ? 2 : 1)) out[s] = st[s + 1] - st[0];
    if (blockIdx.x == 5 && threadIdx.x == 0) out[8] = done - st[0];
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
  cudaMalloc(&out, 16 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 128);
  for (int two = 0; two < 2; ++two)
    for (int box_rows : {128, 16}) {
      CUtensorMap map;
      cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
      cuuint64_t strides[1] = {128};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int rep = 0; rep < 3; ++rep) k<<<148, 64, 8 * 16384 + 128>>>(map, rows_total, box_rows, two, out);
      cudaDeviceSynchronize();
      long long h[16];
      cudaMemcpy(h, out, 9 * 8, cudaMemcpyDeviceToHost);
      printf("%s box %3d rows: cycles after each issue:", two ? "2 threads" : "1 thread ", box_rows);
      for (int s = 0; s < 8; ++s) printf(" %lld", h[s]);
      printf(" | all landed %lld\n", h[8]);
    }
  return 0;
}
