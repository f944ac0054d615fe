// K1: multi-level mean-pooled K/V pyramid (HBM-streaming) and the per-KV-block
// similarity cap (Alg. 3).
//
// Reference semantics:
//   build_pyramid / _pool_stack / mean_pool_rows   pkg/src/pyrattn/blocks.py:86-109,
//                                                  pkg/src/pyrattn/linalg.py:46-58
//   level_cap_from_similarity / _strided_block_similarity
//                                                  pkg/src/pyrattn/mask.py:182-234
//
// Pooling is a dyadic tree of 0.5*(a+b) over raw rows; because b_k is a multiple of
// 2^(H-1) and blocks start at multiples of b_k, level-h row t of the flattened
// [BH*N_h, d] array is exactly the mean of raw rows [t*2^(h-1), (t+1)*2^(h-1)), i.e.
// pooling never crosses a block (or head) boundary. We evaluate the same tree in fp64
// (the reference's precision) and round each level once to bf16 (RNE), so the stored
// pyramid equals bf16(reference fp64 pyramid) bit-for-bit.
#include "common.cuh"
#include "psa_internal.h"

namespace psa {

// One thread: 4 consecutive columns (8 bytes) of one group of G = 2^LOGG raw rows,
// for K (blockIdx.y == 0) or V (blockIdx.y == 1). A warp covers 128 contiguous columns
// so every row access is a fully coalesced 256-byte segment.
// GATHER: the token permutation of pipeline._run_head (pipeline.py:257-263) fused into the
// loads: row p of a head reads source row index[p] and is also written to the permuted level 1
// (k1/v1), so the permuted K/V and their pyramid cost one pass over K/V.
template <int LOGG, bool GATHER>
__global__ void __launch_bounds__(256) pyramid_kernel(const uint16_t* __restrict__ k,
                                                      const uint16_t* __restrict__ v,
                                                      int64_t groups, int d,
                                                      uint16_t* __restrict__ kp,
                                                      uint16_t* __restrict__ vp,
                                                      int64_t bh_rows /* bh*n */,
                                                      int32_t* __restrict__ nonfinite,
                                                      const int64_t* __restrict__ index, int64_t n,
                                                      uint16_t* __restrict__ k1,
                                                      uint16_t* __restrict__ v1) {
  constexpr int G = 1 << LOGG;
  const int tpg = d >> 2;  // threads per group
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t g = tid / tpg;
  if (g >= groups) return;
  const int c4 = static_cast<int>(tid - g * tpg) * 4;
  const uint16_t* src = blockIdx.y == 0 ? k : v;
  uint16_t* dst = blockIdx.y == 0 ? kp : vp;

  const int64_t row0 = g * G;
  uint2 raw[G];
  if (GATHER) {  // G divides n: the group lies in one head
    const int64_t head0 = row0 - row0 % n;
    const int64_t p0 = row0 - head0;
#pragma unroll
    for (int r = 0; r < G; ++r)
      raw[r] = __ldg(reinterpret_cast<const uint2*>(src + (head0 + __ldg(index + p0 + r)) * d + c4));
    uint16_t* dst1 = blockIdx.y == 0 ? k1 : v1;
#pragma unroll
    for (int r = 0; r < G; ++r) *reinterpret_cast<uint2*>(dst1 + (row0 + r) * d + c4) = raw[r];
  } else {
#pragma unroll
    for (int r = 0; r < G; ++r)
      raw[r] = __ldg(reinterpret_cast<const uint2*>(src + (row0 + r) * d + c4));
  }

  double stack[LOGG > 0 ? LOGG : 1][4];
  bool bad = false;
#pragma unroll
  for (int r = 0; r < G; ++r) {
    double x[4];
    x[0] = bf16_bits_to_dbl(static_cast<uint16_t>(raw[r].x & 0xFFFFu));
    x[1] = bf16_bits_to_dbl(static_cast<uint16_t>(raw[r].x >> 16));
    x[2] = bf16_bits_to_dbl(static_cast<uint16_t>(raw[r].y & 0xFFFFu));
    x[3] = bf16_bits_to_dbl(static_cast<uint16_t>(raw[r].y >> 16));
#pragma unroll
    for (int c = 0; c < 4; ++c) bad |= !isfinite(x[c]);
    // climb the dyadic tree: a right child at level lvl closes a level lvl+1 row
#pragma unroll
    for (int lvl = 1; lvl <= LOGG; ++lvl) {
      if ((r >> (lvl - 1)) & 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) x[c] = 0.5 * __dadd_rn(stack[lvl - 1][c], x[c]);
        // level (lvl+1) lives at offset sum_{h=2}^{lvl} (bh_rows >> (h-1)) rows
        int64_t off_rows = 0;
#pragma unroll
        for (int h = 2; h <= lvl; ++h) off_rows += bh_rows >> (h - 1);
        const int64_t out_row = off_rows + ((row0 + r) >> lvl);
        uint2 o;
        o.x = static_cast<uint32_t>(dbl_to_bf16_bits(x[0])) |
              (static_cast<uint32_t>(dbl_to_bf16_bits(x[1])) << 16);
        o.y = static_cast<uint32_t>(dbl_to_bf16_bits(x[2])) |
              (static_cast<uint32_t>(dbl_to_bf16_bits(x[3])) << 16);
        *reinterpret_cast<uint2*>(dst + out_row * d + c4) = o;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) stack[lvl - 1][c] = x[c];
        break;
      }
    }
  }
  if (bad && nonfinite != nullptr) atomicOr(nonfinite, 1);
}

// numpy pairwise sum (any n), recursive split above 128 exactly like numpy.
__device__ double np_pairwise_sum_any(const double* a, int n) {
  if (n <= 128) return np_pairwise_sum(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum_any(a, n2), np_pairwise_sum_any(a + n2, n - n2));
}

// One CTA per (kv head, KV block j). Dot products / squared norms of bf16 rows are exact
// in fp64 (order-free), sqrt/mul/div are single IEEE ops, and the mean uses numpy's
// pairwise order over the compacted "ok" pairs -> caps are identical to the reference.
__global__ void __launch_bounds__(128) simcap_kernel(const uint16_t* __restrict__ k, int64_t n,
                                                     int d, int b_k, int levels, int n_k,
                                                     SimTaus taus, int8_t* __restrict__ caps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint16_t* blk = reinterpret_cast<uint16_t*>(smem_raw);                    // b_k*d
  double* norms = reinterpret_cast<double*>(smem_raw + ((b_k * d * 2 + 15) & ~15));  // b_k
  double* cosv = norms + b_k;                                              // b_k
  int* okf = reinterpret_cast<int*>(cosv + b_k);                           // b_k
  __shared__ int cap_s;

  const int j = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const uint16_t* src = k + (bh * n + static_cast<int64_t>(j) * b_k) * d;
  const int nvec = b_k * d / 8;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x)
    reinterpret_cast<uint4*>(blk)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
  if (threadIdx.x == 0) cap_s = 1;
  __syncthreads();
  // one warp per row (pair): lanes take columns lane, lane + 32, ... (conflict-free shared
  // loads), then a shuffle reduction; the sums are exact, so the order does not matter
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  auto row_dot = [&](int ra, int rb) {
    double acc = 0.0;
    for (int c = lane; c < d; c += 32)
      acc = __fma_rn(bf16_bits_to_dbl(blk[ra * d + c]), bf16_bits_to_dbl(blk[rb * d + c]), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    return acc;
  };
  for (int r = warp; r < b_k; r += nwarps) {
    const double s = row_dot(r, r);
    if (lane == 0) norms[r] = __dsqrt_rn(s);
  }
  __syncthreads();
  for (int h = 2; h <= levels; ++h) {
    const int stride = 1 << (h - 1);
    const int np_ = b_k - stride;
    if (np_ <= 0) break;  // uniform across the CTA
    for (int r = warp; r < np_; r += nwarps) {
      const double na = norms[r], nb = norms[r + stride];
      const bool ok = (na > 0.0) && (nb > 0.0);  // warp-uniform
      double c = 0.0;
      if (ok) {
        c = __ddiv_rn(row_dot(r, r + stride), __dmul_rn(na, nb));
        c = fmin(fmax(c, -1.0), 1.0);
      }
      if (lane == 0) {
        cosv[r] = c;
        okf[r] = ok ? 1 : 0;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int m = 0;
      for (int r = 0; r < np_; ++r)
        if (okf[r]) cosv[m++] = cosv[r];  // in-place compaction keeps index order
      if (m > 0) {
        const double sim = __ddiv_rn(np_pairwise_sum_any(cosv, m), static_cast<double>(m));
        if (sim > taus.v[h - 2]) cap_s = h > cap_s ? h : cap_s;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) caps[bh * n_k + j] = static_cast<int8_t>(cap_s);
}

}  // namespace psa

using namespace psa;

static int pyramid_launch(const void* k, const void* v, int64_t bh, int64_t n, int d, int b_k,
                          int levels, void* k_pyr, void* v_pyr, int32_t* nonfinite,
                          const int64_t* index, void* k1, void* v1, void* stream) {
  PSA_CHECK_ARG(k && v, "K/V pointers must be non-null");
  PSA_CHECK_ARG(bh >= 1 && n >= 1, "bh and n must be positive");
  PSA_CHECK_ARG(d == 64 || d == 128, "head_dim must be 64 or 128 for the sm_100a path");
  PSA_CHECK_ARG(levels >= 1 && levels <= 8, "levels must lie in 1..8");
  PSA_CHECK_ARG(b_k >= 1 && n % b_k == 0, "seq_len not divisible by k_block");
  PSA_CHECK_ARG(b_k % (1 << (levels - 1)) == 0, "k_block not divisible by 2^(levels-1)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool gather = index != nullptr;
  if (gather) PSA_CHECK_ARG(k1 && v1, "permuted level-1 outputs must be non-null");
  if (levels == 1) {
    if (!gather) return PSA_OK;
    int rc = psa_gather_rows(k, bh, n, d * 2, index, k1, stream);
    return rc ? rc : psa_gather_rows(v, bh, n, d * 2, index, v1, stream);
  }
  PSA_CHECK_ARG(k_pyr && v_pyr, "pyramid output pointers must be non-null");
  const int logg = levels - 1;
  const int64_t rows = bh * n;
  const int64_t groups = rows >> logg;
  const int64_t threads = groups * (d / 4);
  dim3 grid(static_cast<unsigned>((threads + 255) / 256), 2);
  auto* kk = static_cast<const uint16_t*>(k);
  auto* vv = static_cast<const uint16_t*>(v);
  auto* kp = static_cast<uint16_t*>(k_pyr);
  auto* vp = static_cast<uint16_t*>(v_pyr);
  auto* k1p = static_cast<uint16_t*>(k1);
  auto* v1p = static_cast<uint16_t*>(v1);
  switch (logg) {
#define PSA_PYR_CASE(L)                                                                        \
  case L:                                                                                      \
    if (gather)                                                                                \
      pyramid_kernel<L, true><<<grid, 256, 0, s>>>(kk, vv, groups, d, kp, vp, rows, nonfinite, \
                                                   index, n, k1p, v1p);                         \
    else                                                                                       \
      pyramid_kernel<L, false><<<grid, 256, 0, s>>>(kk, vv, groups, d, kp, vp, rows,           \
                                                    nonfinite, nullptr, n, nullptr, nullptr);   \
    break;
    PSA_PYR_CASE(1)
    PSA_PYR_CASE(2)
    PSA_PYR_CASE(3)
    PSA_PYR_CASE(4)
    PSA_PYR_CASE(5)
    PSA_PYR_CASE(6)
    PSA_PYR_CASE(7)
#undef PSA_PYR_CASE
    default:
      return psa_fail(PSA_EINVAL, "unsupported level count");
  }
  return psa_check_launch("pyramid_kernel");
}

extern "C" int psa_pyramid_build(const void* k, const void* v, int64_t bh, int64_t n, int d,
                                 int b_k, int levels, void* k_pyr, void* v_pyr,
                                 int32_t* nonfinite, void* stream) {
  return pyramid_launch(k, v, bh, n, d, b_k, levels, k_pyr, v_pyr, nonfinite, nullptr, nullptr,
                        nullptr, stream);
}

extern "C" int psa_pyramid_build_gather(const void* k, const void* v, int64_t bh, int64_t n,
                                        int d, int b_k, int levels, const int64_t* index,
                                        void* k1, void* v1, void* k_pyr, void* v_pyr,
                                        int32_t* nonfinite, void* stream) {
  PSA_CHECK_ARG(index != nullptr, "index must be non-null");
  return pyramid_launch(k, v, bh, n, d, b_k, levels, k_pyr, v_pyr, nonfinite, index, k1, v1,
                        stream);
}

extern "C" int psa_similarity_caps(const void* k, int64_t bh, int64_t n, int d, int b_k,
                                   int levels, const double* sim_taus, int8_t* caps,
                                   void* stream) {
  PSA_CHECK_ARG(k && caps, "K/caps pointers must be non-null");
  PSA_CHECK_ARG(d == 64 || d == 128, "head_dim must be 64 or 128 for the sm_100a path");
  PSA_CHECK_ARG(levels >= 1 && levels <= 8, "levels must lie in 1..8");
  PSA_CHECK_ARG(b_k >= 1 && n % b_k == 0, "seq_len not divisible by k_block");
  PSA_CHECK_ARG(levels == 1 || sim_taus != nullptr, "need levels-1 similarity thresholds");
  SimTaus t{};
  for (int i = 0; i + 1 < levels; ++i) t.v[i] = sim_taus[i];
  const int n_k = static_cast<int>(n / b_k);
  const size_t smem = ((static_cast<size_t>(b_k) * d * 2 + 15) & ~static_cast<size_t>(15)) +
                      static_cast<size_t>(b_k) * (8 + 8 + 4);
  PSA_CHECK_ARG(smem <= 200 * 1024, "k_block too large for the similarity-cap kernel");
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(simcap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  dim3 grid(n_k, static_cast<unsigned>(bh));
  simcap_kernel<<<grid, 128, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(k), n, d, b_k, levels, n_k, t, caps);
  return psa_check_launch("simcap_kernel");
}
