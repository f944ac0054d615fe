// Token-row gather for the space-filling-curve permutation (pkg/src/pyrattn/permute.py:131-137,
// apply_permutation: output row i = input row order[i]) applied to [bh, n, row] tensors.
// HBM-bound: one warp per output row, 16-byte vector copies when the row allows it.
#include "common.cuh"
#include "psa_internal.h"

namespace psa {

template <typename V>
__global__ void __launch_bounds__(256) gather_rows_kernel(const V* __restrict__ src,
                                                          int64_t n_rows, int64_t n,
                                                          int row_vecs,
                                                          const int64_t* __restrict__ index,
                                                          V* __restrict__ dst) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= n_rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t bh = r / n, i = r % n;
  const V* s = src + (bh * n + index[i]) * row_vecs;
  V* d = dst + r * row_vecs;
  for (int c = lane; c < row_vecs; c += 32) d[c] = __ldg(s + c);
}

}  // namespace psa

using namespace psa;

extern "C" int psa_gather_rows(const void* src, int64_t bh, int64_t n, int row_bytes,
                               const int64_t* index, void* dst, void* stream) {
  PSA_CHECK_ARG(src && index && dst, "null pointer argument");
  PSA_CHECK_ARG(bh >= 1 && n >= 1 && row_bytes >= 4 && row_bytes % 4 == 0,
                "gather: bh, n >= 1 and row_bytes a positive multiple of 4 required");
  PSA_CHECK_ARG(src != dst, "gather: src and dst must not alias");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t rows = bh * n;
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  if (row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src) % 16 == 0) &&
      (reinterpret_cast<uintptr_t>(dst) % 16 == 0))
    gather_rows_kernel<uint4><<<grid, 256, 0, s>>>(static_cast<const uint4*>(src), rows, n,
                                                    row_bytes / 16, index,
                                                    static_cast<uint4*>(dst));
  else
    gather_rows_kernel<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(src), rows, n,
                                                       row_bytes / 4, index,
                                                       static_cast<uint32_t*>(dst));
  return psa_check_launch("gather_rows_kernel");
}
