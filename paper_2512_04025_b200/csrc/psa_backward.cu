// Backward of the multi-level block-sparse attention (dQ, dK, dV through
// pooling). The reference has no backward (SPEC.md:494 non-goal; the paper claims training use,
// PAPER.md:139), so the oracle is the autograd of the forward's own definition
// (attention.py:171-218 with the mask held fixed; tests/test_gpu_backward.py).
//
// Identity used throughout: a level-h pooled key stands for the 2^(h-1) raw keys it averages,
// with bias (h-1) ln 2 (attention.py:39-44). exp(s + (h-1) ln 2) = 2^(h-1) exp(s), so the forward
// equals attention WITHOUT bias over the "expanded" block whose raw row r carries pooled row
// r >> (h-1). Differentiating that form, the gradient of raw row r is exactly the gradient of its
// duplicate (the chain rule through the mean divides the pooled gradient by 2^(h-1), and the
// duplicate's weight is 2^(h-1) times smaller). So the backward is a standard attention backward
// over (query block, expanded KV block) pairs, and dK/dV land directly on raw rows; the pyramid
// needs no transpose. With the mask fixed, importance and level assignment carry no gradient.
//
// The identity is applied at pooled granularity: the kernels compute with the L_h = b_k >> (h-1)
// pooled rows (unbiased weights p' = p / 2^(h-1) for dK/dV, biased p for dQ) and only the final
// add spreads a pooled row's gradient over its 2^(h-1) raw rows, so the work per selected block
// scales with its pooled length like the forward's.
//
// At D = 128 both passes run on tcgen05 / TMEM (psa_attention.cu):
//  - psa_bwd_dq_tc_kernel: the forward's producers and plan walk, S and dP in TMEM, dS written
//    back over S as the TMEM A operand of dQ += dS K, 3-stage K ring; 29 ms at cfg3;
//  - psa_bwd_dkv_tc_kernel: one CTA per (KV head, level, unit of 2^(h-1) blocks packed into one
//    tile), S^T / dP^T in TMEM, P'^T / dS^T written back over them as the TMEM A operand of
//    dV / dK, double-buffered Q / dO, per-level pooled fp32 slabs summed by bwd_unpool_kernel;
//    70 ms at cfg3.
// D = 64 uses warp-level mma.sync kernels (m16n8k16 bf16, fp32 accumulate, ldmatrix fragments,
// cp.async double-buffered tiles). cfg3 backward ~109 ms against a 34 ms forward.
#include "common.cuh"
#include "psa_internal.h"

namespace psa {

constexpr int kBwdThreads = 256;  // 8 warps x 16 rows = 128 rows (b_q, b_k <= 128)
constexpr int kBwdRows = 128;

struct BwdParams {
  int64_t n, bkv_total;  // bkv_total = batch * hkv (pyramid level offsets)
  int hq, hkv, b_q, b_k, levels, n_q, n_k, causal;
  float scale;       // 1/sqrt(d)
  float scale_log2;  // scale * log2(e)
  const uint16_t* q;
  const uint16_t* k;
  const uint16_t* v;
  const uint16_t* k_pyr;
  const uint16_t* v_pyr;
  const uint16_t* dout;
  const float* lse;    // natural log, -inf for rows without keys
  const float* drow;   // rowsum(dO * O) [bhq * n]
  const uint16_t* csr;  // plan entries j | level << 12, level-major
  const int32_t* info;
  const int8_t* level_map;  // [bhq, n_q, n_k]
  uint16_t* dq;
  uint16_t* dk;
  uint16_t* dv;
};

PSA_DEV void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
PSA_DEV void ldsm4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
PSA_DEV void ldsm4t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
PSA_DEV float bf2f(uint16_t x) { return __uint_as_float(static_cast<uint32_t>(x) << 16); }
PSA_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
PSA_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
PSA_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Tiles in shared memory: [128 rows][D + 8] bf16 (the 16-byte pad makes ldmatrix conflict-free).
template <int D>
struct BwdTile {
  static constexpr int kStride = D + 8;
  static constexpr int kBytes = kBwdRows * kStride * 2;
};

// rows [0, rows) of src (row pitch D) -> tile; rows [rows, 128) zeroed. expand_shift > 0 maps
// tile row r to source row r >> expand_shift (the expanded pooled block).
template <int D>
__device__ void load_tile(uint16_t* tile, const uint16_t* src, int rows, int expand_shift) {
  constexpr int kVec = D / 8;  // 16-byte vectors per row
  for (int e = threadIdx.x; e < kBwdRows * kVec; e += kBwdThreads) {
    const int r = e / kVec, c = (e % kVec) * 8;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (r < rows) val = *reinterpret_cast<const uint4*>(src + static_cast<int64_t>(r >> expand_shift) * D + c);
    *reinterpret_cast<uint4*>(tile + r * BwdTile<D>::kStride + c) = val;
  }
}

// load_tile with cp.async (completion via cp_async_commit / cp_async_wait; zero rows stored)
template <int D>
__device__ void load_tile_async(uint16_t* tile, const uint16_t* src, int rows) {
  constexpr int kVec = D / 8;
  for (int e = threadIdx.x; e < kBwdRows * kVec; e += kBwdThreads) {
    const int r = e / kVec, c = (e % kVec) * 8;
    uint16_t* dst = tile + r * BwdTile<D>::kStride + c;
    if (r < rows) cp_async16(dst, src + static_cast<int64_t>(r) * D + c);
    else *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
  }
}

// pointer to the first row of KV block j of head bkv at level h (rows are b_k >> (h-1) long)
PSA_DEV const uint16_t* level_block(const uint16_t* raw, const uint16_t* pyr, int64_t bkv_count,
                                    int64_t bkv, int64_t n, int d, int b_k, int h, int j) {
  if (h == 1) return raw + (bkv * n + static_cast<int64_t>(j) * b_k) * d;
  int64_t off = 0;
  for (int l = 2; l < h; ++l) off += bkv_count * (n >> (l - 1));
  const int64_t nh = n >> (h - 1);
  return pyr + (off + bkv * nh + static_cast<int64_t>(j) * (b_k >> (h - 1))) * d;
}

// D_r = rowsum(dO_r * O_r) (fp32), one warp per row
template <int D>
// Also nl2[r] = -lse[r] log2(e) (-inf for a fully masked row), the additive term of the dK/dV
// pass's exp2 so that its softmax needs no per-column checks.
__global__ void __launch_bounds__(256) bwd_drow_kernel(const uint16_t* __restrict__ out,
                                                       const uint16_t* __restrict__ dout,
                                                       const float* __restrict__ lse,
                                                       int64_t rows, float* __restrict__ drow,
                                                       float* __restrict__ nl2) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float acc = 0.f;
  for (int c = lane * 2; c < D; c += 64) {
    const uint32_t o = *reinterpret_cast<const uint32_t*>(out + r * D + c);
    const uint32_t g = *reinterpret_cast<const uint32_t*>(dout + r * D + c);
    acc = fmaf(bf2f(o & 0xFFFFu), bf2f(g & 0xFFFFu), acc);
    acc = fmaf(bf2f(o >> 16), bf2f(g >> 16), acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    drow[r] = acc;
    const float l = lse[r];
    nl2[r] = l == -INFINITY ? -INFINITY : -l * 1.4426950408889634f;
  }
}

// ---------------------------------------------------------------------------------------- dQ
// One CTA per (head, query block); warp w owns query rows 16w..16w+15. The unit's selected
// pooled blocks (level-major plan order) are packed back to back into 64-key chunks staged in
// shared memory (a level-4 block is 15 rows, so several blocks share a chunk):
//   S = Q K^T, P = exp2(S c + (h-1) - lse2), dP = dO V^T, dS = P (dP - D), dQ += dS K.
// P carries the level bias here: dq = scale * sum_j ds_j k_j over POOLED keys.
constexpr int kChunkKeys = 64;

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1) bwd_dq_kernel(const BwdParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using T = BwdTile<D>;
  uint16_t* qs = reinterpret_cast<uint16_t*>(smem_raw);
  uint16_t* ds = qs + kBwdRows * T::kStride;
  uint16_t* kbuf = ds + kBwdRows * T::kStride;  // 2 stages x kChunkKeys rows (K), then V
  uint16_t* vbuf = kbuf + 2 * kChunkKeys * T::kStride;
  int* ent_off = reinterpret_cast<int*>(vbuf + 2 * kChunkKeys * T::kStride);  // [n_k + 1]
  float* cbias_b = reinterpret_cast<float*>(ent_off + p.n_k + 1);  // [2][kChunkKeys]
  int* ckpos_b = reinterpret_cast<int*>(cbias_b + 2 * kChunkKeys);  // [2][kChunkKeys]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = blockIdx.x;
  const int bhq = static_cast<int>(unit / p.n_q), i = static_cast<int>(unit % p.n_q);
  const int b = bhq / p.hq, hh = bhq % p.hq;
  const int64_t bkv = static_cast<int64_t>(b) * p.hkv + hh / (p.hq / p.hkv);
  const int64_t row0 = static_cast<int64_t>(bhq) * p.n + static_cast<int64_t>(i) * p.b_q;
  const int n_ent = p.info[unit * 2];
  const uint16_t* csr = p.csr + unit * p.n_k;

  load_tile<D>(qs, p.q + row0 * D, p.b_q, 0);
  load_tile<D>(ds, p.dout + row0 * D, p.b_q, 0);
  if (threadIdx.x == 0) {  // prefix of pooled rows over the unit's entries
    int acc = 0;
    for (int e = 0; e < n_ent; ++e) {
      ent_off[e] = acc;
      acc += p.b_k >> ((csr[e] >> 12) - 1);
    }
    ent_off[n_ent] = acc;
  }
  const int ra = warp * 16 + (lane >> 2), rb = ra + 8;
  const float kLog2e = 1.4426950408889634f;
  float lse2[2], dd[2];
  bool live[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int r = u ? rb : ra;
    const float l = r < p.b_q ? p.lse[row0 + r] : -INFINITY;
    live[u] = l != -INFINITY;
    lse2[u] = live[u] ? l * kLog2e : 0.f;
    dd[u] = r < p.b_q ? p.drow[row0 + r] : 0.f;
  }
  float dqa[D / 8][4];
#pragma unroll
  for (int t = 0; t < D / 8; ++t) dqa[t][0] = dqa[t][1] = dqa[t][2] = dqa[t][3] = 0.f;
  const uint32_t qs_a = smem_u32(qs), ds_a = smem_u32(ds);
  const uint32_t a_off = ((warp * 16 + (lane & 15)) * T::kStride + (lane >> 4) * 8) * 2;
  const int bn = (lane & 7) + ((lane >> 4) << 3), bk = ((lane >> 3) & 1) * 8;   // [n][k] memory
  const int tk = (lane & 7) + (((lane >> 3) & 1) << 3), tn = (lane >> 4) << 3;  // [k][n] memory
  const int64_t qpos0 = static_cast<int64_t>(i) * p.b_q;
  __syncthreads();
  const int total = ent_off[n_ent];

  // stage chunk `base` into buffer st: key row c <- pooled row (e, t), base + c = ent_off[e] + t
  auto stage = [&](int base, int st) {
    constexpr int kVec = D / 8;
    const int nk = min(kChunkKeys, total - base);
    uint16_t* kd = kbuf + st * kChunkKeys * T::kStride;
    uint16_t* vd = vbuf + st * kChunkKeys * T::kStride;
    for (int x = threadIdx.x; x < kChunkKeys * kVec; x += kBwdThreads) {
      const int c = x / kVec, col = (x % kVec) * 8;
      if (c < nk) {
        const int g = base + c;
        int lo = 0, hi = n_ent - 1;  // last entry with ent_off[e] <= g
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (ent_off[mid] <= g) lo = mid; else hi = mid - 1;
        }
        const uint32_t ent = csr[lo];
        const int j = static_cast<int>(ent & 0xFFFu), h = static_cast<int>(ent >> 12);
        const int t = g - ent_off[lo];
        const int64_t src = static_cast<int64_t>(t) * D + col;
        cp_async16(kd + c * T::kStride + col, level_block(p.k, p.k_pyr, p.bkv_total, bkv, p.n, D, p.b_k, h, j) + src);
        cp_async16(vd + c * T::kStride + col, level_block(p.v, p.v_pyr, p.bkv_total, bkv, p.n, D, p.b_k, h, j) + src);
        if (col == 0) {
          cbias_b[st * kChunkKeys + c] = static_cast<float>(h - 1);
          ckpos_b[st * kChunkKeys + c] = h == 1 ? j * p.b_k + t : -1;  // pooled levels never straddle
        }
      } else {
        *reinterpret_cast<uint4*>(kd + c * T::kStride + col) = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(vd + c * T::kStride + col) = make_uint4(0u, 0u, 0u, 0u);
        if (col == 0) {
          cbias_b[st * kChunkKeys + c] = -INFINITY;
          ckpos_b[st * kChunkKeys + c] = -1;
        }
      }
    }
    cp_async_commit();
  };
  if (total > 0) stage(0, 0);
  for (int base = 0, st = 0; base < total; base += kChunkKeys, st ^= 1) {
    const int nk = min(kChunkKeys, total - base);
    if (base + kChunkKeys < total) {
      stage(base + kChunkKeys, st ^ 1);  // buffer st^1 was released by the sync ending chunk-1
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t ks_a = smem_u32(kbuf + st * kChunkKeys * T::kStride);
    const uint32_t vs_a = smem_u32(vbuf + st * kChunkKeys * T::kStride);
    const float* cbias = cbias_b + st * kChunkKeys;
    const int* ckpos = ckpos_b + st * kChunkKeys;
    const int nt16 = (nk + 15) >> 4;  // 16-key tiles holding keys
    float s[8][4], dp[8][4];
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int c = 0; c < 4; ++c) s[t][c] = dp[t][c] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t qa[4], da[4];
      ldsm4(qa, qs_a + a_off + kk * 32);
      ldsm4(da, ds_a + a_off + kk * 32);
#pragma unroll
      for (int t2 = 0; t2 < 4; ++t2) {
        if (t2 < nt16) {
          uint32_t kb[4], vb[4];
          const uint32_t off = ((t2 * 16 + bn) * T::kStride + kk * 16 + bk) * 2;
          ldsm4(kb, ks_a + off);
          ldsm4(vb, vs_a + off);
          mma16816(s[2 * t2], qa, kb[0], kb[1]);
          mma16816(s[2 * t2 + 1], qa, kb[2], kb[3]);
          mma16816(dp[2 * t2], da, vb[0], vb[1]);
          mma16816(dp[2 * t2 + 1], da, vb[2], vb[3]);
        }
      }
    }
    uint32_t dsa[4][4];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      float v4[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int u = c >> 1;
        const int key = t * 8 + 2 * (lane & 3) + (c & 1);
        const float bias = cbias[key];
        const int kp = ckpos[key];
        const int64_t qpos = qpos0 + (u ? rb : ra);
        const bool ok = live[u] && bias != -INFINITY && !(p.causal && kp >= 0 && kp > qpos);
        const float pr = ok ? exp2f(fmaf(s[t][c], p.scale_log2, bias - lse2[u])) : 0.f;
        v4[c] = pr * (dp[t][c] - dd[u]);
      }
      dsa[t >> 1][(t & 1) * 2 + 0] = pack_bf16x2(v4[0], v4[1]);
      dsa[t >> 1][(t & 1) * 2 + 1] = pack_bf16x2(v4[2], v4[3]);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      if (kk < nt16) {
        const uint32_t a[4] = {dsa[kk][0], dsa[kk][1], dsa[kk][2], dsa[kk][3]};
#pragma unroll
        for (int t2 = 0; t2 < D / 16; ++t2) {
          uint32_t kb[4];
          ldsm4t(kb, ks_a + ((kk * 16 + tk) * T::kStride + t2 * 16 + tn) * 2);
          mma16816(dqa[2 * t2], a, kb[0], kb[1]);
          mma16816(dqa[2 * t2 + 1], a, kb[2], kb[3]);
        }
      }
    }
    __syncthreads();  // buffer st free for the chunk after next
  }
#pragma unroll
  for (int t = 0; t < D / 8; ++t) {
    const int c = t * 8 + 2 * (lane & 3);
    if (ra < p.b_q)
      *reinterpret_cast<uint32_t*>(p.dq + (row0 + ra) * D + c) =
          pack_bf16x2(dqa[t][0] * p.scale, dqa[t][1] * p.scale);
    if (rb < p.b_q)
      *reinterpret_cast<uint32_t*>(p.dq + (row0 + rb) * D + c) =
          pack_bf16x2(dqa[t][2] * p.scale, dqa[t][3] * p.scale);
  }
}

// ------------------------------------------------------------------------------------ dK, dV
// One CTA per (KV head, KV block j). The CTA lists, level-major and in (query head, query
// block) order, every (q head of the GQA group, query block) that selected block j. Per level h
// the POOLED block (L_h = b_k >> (h-1) rows, R = pow2(ceil(L_h / 16)) row tiles) is staged once;
// warp w takes row tile w % R and the query slice (w / R) of every listed query block, so all 8
// warps work at every level. Per listed query block (pooled, unbiased weights p' = p / 2^(h-1)):
//   S^T = K Q^T, P'^T = exp2(S^T c - lse2), dP^T = V dO^T, dS^T = P'^T (dP^T - D),
//   dV_h += P'^T dO, dK_h += dS^T Q.
// A raw row r of block j receives the pooled gradients of row r >> (h-1) of every level, i.e.
// the duplicate's gradient (file header). At the end of a level the warps' partials are summed
// in shared memory and added to the CTA's raw rows in an fp32 scratch (exclusive to this CTA);
// the last step writes bf16 dK (x scale) and dV.
template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1) bwd_dkv_kernel(const BwdParams p, int cap,
                                                                float* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using T = BwdTile<D>;
  // Q / dO double-buffered (stage st at qbuf + st * 2 tiles), then the pooled K and V tiles
  uint16_t* qbuf = reinterpret_cast<uint16_t*>(smem_raw);
  uint16_t* ks = qbuf + 4 * kBwdRows * T::kStride;
  uint16_t* vs = ks + kBwdRows * T::kStride;
  float* part = reinterpret_cast<float*>(smem_raw);  // level-end reduction (aliases Q / dO)
  float* lse_b = reinterpret_cast<float*>(vs + kBwdRows * T::kStride);  // [2][128]
  float* d_b = lse_b + 2 * kBwdRows;                                     // [2][128]
  uint32_t* ents = reinterpret_cast<uint32_t*>(d_b + 2 * kBwdRows);
  __shared__ int warp_cnt[kBwdThreads / 32];
  static_assert(2 * 8 * 16 * D * 4 <= 4 * BwdTile<D>::kBytes, "partials must fit in Q / dO");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x;
  const int64_t bkv = blockIdx.y;
  const int b = static_cast<int>(bkv / p.hkv), hk = static_cast<int>(bkv % p.hkv);
  const int group = p.hq / p.hkv;
  const int span = group * p.n_q;

  // ---- deterministic level-major compaction of the entries selecting block j
  int total = 0;
  int lvl_end[9];
  for (int h = 1; h <= p.levels; ++h) {
    for (int base = 0; base < span; base += kBwdThreads) {
      const int x = base + threadIdx.x;
      bool hit = false;
      if (x < span) {
        const int g = x / p.n_q, iq = x % p.n_q;
        const int64_t bhq = static_cast<int64_t>(b) * p.hq + hk * group + g;
        hit = p.level_map[(bhq * p.n_q + iq) * p.n_k + j] == h;
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) warp_cnt[warp] = __popc(m);
      __syncthreads();
      int before = 0, all = 0;
      for (int w = 0; w < kBwdThreads / 32; ++w) {
        before += w < warp ? warp_cnt[w] : 0;
        all += warp_cnt[w];
      }
      if (hit) {
        const int slot = total + before + __popc(m & ((1u << lane) - 1u));
        if (slot < cap) ents[slot] = static_cast<uint32_t>(x);
      }
      total += all;
      __syncthreads();
    }
    lvl_end[h] = min(total, cap);
  }

  const int64_t krow0 = bkv * p.n + static_cast<int64_t>(j) * p.b_k;
  float* sk = scratch + krow0 * D;                        // dK rows of block j (fp32)
  float* sv = scratch + (p.bkv_total * p.n + krow0) * D;  // dV rows
  const uint32_t ks_a = smem_u32(ks), vs_a = smem_u32(vs);
  const int bn = (lane & 7) + ((lane >> 4) << 3), bk = ((lane >> 3) & 1) * 8;
  const int tk = (lane & 7) + (((lane >> 3) & 1) << 3), tn = (lane >> 4) << 3;
  const float kLog2e = 1.4426950408889634f;
  bool first = true;
  // stage entry e (its query block's Q, dO, lse, D) into buffer st with cp.async
  auto stage = [&](int e, int st) {
    const int x = static_cast<int>(ents[e]);
    const int g = x / p.n_q, iq = x % p.n_q;
    const int64_t bhq = static_cast<int64_t>(b) * p.hq + hk * group + g;
    const int64_t row0 = bhq * p.n + static_cast<int64_t>(iq) * p.b_q;
    uint16_t* q_t = qbuf + (2 * st) * kBwdRows * T::kStride;
    load_tile_async<D>(q_t, p.q + row0 * D, p.b_q);
    load_tile_async<D>(q_t + kBwdRows * T::kStride, p.dout + row0 * D, p.b_q);
    if (threadIdx.x < kBwdRows) {
      const int r = threadIdx.x;
      lse_b[st * kBwdRows + r] = r < p.b_q ? p.lse[row0 + r] : -INFINITY;
      d_b[st * kBwdRows + r] = r < p.b_q ? p.drow[row0 + r] : 0.f;
    }
    cp_async_commit();
  };

  int e0 = 0;
  for (int h = 1; h <= p.levels; ++h) {
    const int e1 = lvl_end[h];
    if (e1 == e0) continue;
    const int L = p.b_k >> (h - 1);
    int R = 1;
    while (R * 16 < L) R <<= 1;  // row tiles (power of two, divides 8)
    const int qsplit = 8 / R, qw = kBwdRows / qsplit;  // query columns per warp
    const int rt = warp % R, qsl = warp / R;
    const uint32_t a_off = ((rt * 16 + (lane & 15)) * T::kStride + (lane >> 4) * 8) * 2;
    float dka[D / 8][4], dva[D / 8][4];
#pragma unroll
    for (int t = 0; t < D / 8; ++t)
#pragma unroll
      for (int c = 0; c < 4; ++c) dka[t][c] = dva[t][c] = 0.f;
    __syncthreads();  // partial buffers (aliasing the tiles) consumed
    load_tile<D>(ks, level_block(p.k, p.k_pyr, p.bkv_total, bkv, p.n, D, p.b_k, h, j), L, 0);
    load_tile<D>(vs, level_block(p.v, p.v_pyr, p.bkv_total, bkv, p.n, D, p.b_k, h, j), L, 0);
    const int key_a = rt * 16 + (lane >> 2);  // this thread's pooled rows key_a, key_a + 8
    stage(e0, 0);
    for (int e = e0, st = 0; e < e1; ++e, st ^= 1) {
      if (e + 1 < e1) {
        stage(e + 1, st ^ 1);  // buffer st^1 was released by the sync ending entry e-1
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const int iq = static_cast<int>(ents[e]) % p.n_q;
      const uint32_t qs_a = smem_u32(qbuf + (2 * st) * kBwdRows * T::kStride);
      const uint32_t ds_a = qs_a + kBwdRows * T::kStride * 2;
      const float* lse_s = lse_b + st * kBwdRows;
      const float* d_s = d_b + st * kBwdRows;
      const int64_t qpos0 = static_cast<int64_t>(iq) * p.b_q;
      const bool straddle = p.causal && (static_cast<int64_t>(j + 1) * p.b_k - 1 > qpos0);
      for (int qc = qsl * qw; qc < (qsl + 1) * qw && qc < p.b_q; qc += 64) {
        const int nq16 = min(4, (min((qsl + 1) * qw, qc + 64) - qc) >> 4);  // 16-query tiles
        float st[8][4], dpt[8][4];
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
          for (int c = 0; c < 4; ++c) st[t][c] = dpt[t][c] = 0.f;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          uint32_t ka[4], va[4];
          ldsm4(ka, ks_a + a_off + kk * 32);
          ldsm4(va, vs_a + a_off + kk * 32);
#pragma unroll
          for (int t2 = 0; t2 < 4; ++t2) {
            if (t2 < nq16) {
              uint32_t qb[4], db[4];
              const uint32_t off = ((qc + t2 * 16 + bn) * T::kStride + kk * 16 + bk) * 2;
              ldsm4(qb, qs_a + off);
              ldsm4(db, ds_a + off);
              mma16816(st[2 * t2], ka, qb[0], qb[1]);
              mma16816(st[2 * t2 + 1], ka, qb[2], qb[3]);
              mma16816(dpt[2 * t2], va, db[0], db[1]);
              mma16816(dpt[2 * t2 + 1], va, db[2], db[3]);
            }
          }
        }
        uint32_t pa[4][4], dsa[4][4];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          float pv[4], sv4[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int key = key_a + ((c >> 1) << 3);
            const int qr = qc + t * 8 + 2 * (lane & 3) + (c & 1);  // may pass 127 (masked)
            const int qi = min(qr, kBwdRows - 1);
            const float l = lse_s[qi];
            const int64_t kpos = static_cast<int64_t>(j) * p.b_k + key;  // level 1 only straddles
            const bool ok = t < 2 * nq16 && key < L && qr < p.b_q && l != -INFINITY &&
                            !(straddle && kpos > qpos0 + qr);
            const float pr = ok ? exp2f(fmaf(st[t][c], p.scale_log2, -l * kLog2e)) : 0.f;
            pv[c] = pr;
            sv4[c] = pr * (dpt[t][c] - d_s[qi]);
          }
          pa[t >> 1][(t & 1) * 2 + 0] = pack_bf16x2(pv[0], pv[1]);
          pa[t >> 1][(t & 1) * 2 + 1] = pack_bf16x2(pv[2], pv[3]);
          dsa[t >> 1][(t & 1) * 2 + 0] = pack_bf16x2(sv4[0], sv4[1]);
          dsa[t >> 1][(t & 1) * 2 + 1] = pack_bf16x2(sv4[2], sv4[3]);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (kk < nq16) {
            const uint32_t ap[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
            const uint32_t as[4] = {dsa[kk][0], dsa[kk][1], dsa[kk][2], dsa[kk][3]};
#pragma unroll
            for (int t2 = 0; t2 < D / 16; ++t2) {
              uint32_t db[4], qb[4];
              const uint32_t off = ((qc + kk * 16 + tk) * T::kStride + t2 * 16 + tn) * 2;
              ldsm4t(db, ds_a + off);
              ldsm4t(qb, qs_a + off);
              mma16816(dva[2 * t2], ap, db[0], db[1]);
              mma16816(dva[2 * t2 + 1], ap, db[2], db[3]);
              mma16816(dka[2 * t2], as, qb[0], qb[1]);
              mma16816(dka[2 * t2 + 1], as, qb[2], qb[3]);
            }
          }
        }
      }
      __syncthreads();  // buffer st free for the entry after next
    }
    // ---- level end: partials -> shared memory [warp][16][D] (dK then dV), sum over the query
    // slices, add row r >> (h-1) to every raw row r of the block
    __syncthreads();
    float* pk = part;
    float* pvv = part + 8 * 16 * D;
#pragma unroll
    for (int t = 0; t < D / 8; ++t) {
      const int c = t * 8 + 2 * (lane & 3);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r16 = (lane >> 2) + 8 * u;
        pk[(warp * 16 + r16) * D + c] = dka[t][2 * u];
        pk[(warp * 16 + r16) * D + c + 1] = dka[t][2 * u + 1];
        pvv[(warp * 16 + r16) * D + c] = dva[t][2 * u];
        pvv[(warp * 16 + r16) * D + c + 1] = dva[t][2 * u + 1];
      }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < p.b_k * D; x += kBwdThreads) {
      const int r = x / D, c = x % D;
      const int tp = r >> (h - 1);
      const int w0 = tp >> 4, r16 = tp & 15;
      float gk = 0.f, gv = 0.f;
      for (int q2 = 0; q2 < qsplit; ++q2) {
        const int w = w0 + q2 * R;
        gk += pk[(w * 16 + r16) * D + c];
        gv += pvv[(w * 16 + r16) * D + c];
      }
      sk[x] = first ? gk : sk[x] + gk;
      sv[x] = first ? gv : sv[x] + gv;
    }
    first = false;
    e0 = e1;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < p.b_k * D / 2; x += kBwdThreads) {
    const int r = (2 * x) / D, c = (2 * x) % D;
    uint32_t okv = 0u, ovv = 0u;
    if (!first) {
      okv = pack_bf16x2(sk[r * D + c] * p.scale, sk[r * D + c + 1] * p.scale);
      ovv = pack_bf16x2(sv[r * D + c], sv[r * D + c + 1]);
    }
    *reinterpret_cast<uint32_t*>(p.dk + (krow0 + r) * D + c) = okv;
    *reinterpret_cast<uint32_t*>(p.dv + (krow0 + r) * D + c) = ovv;
  }
}

template <int D>
static int launch_bwd(BwdParams p, int64_t batch, const uint16_t* out, void* ws, cudaStream_t s) {
  const int64_t rows = batch * p.hq * p.n;
  float* drow = static_cast<float*>(ws);
  float* nl2 = drow + ((rows + 63) / 64) * 64;
  float* scratch = nl2 + ((rows + 63) / 64) * 64;
  p.drow = drow;
  bwd_drow_kernel<D><<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(out, p.dout, p.lse, rows, drow, nl2);
  int rc = psa_check_launch("bwd_drow_kernel");
  if (rc) return rc;
  const size_t smem_q = 2 * static_cast<size_t>(BwdTile<D>::kBytes) +
                        4 * static_cast<size_t>(kChunkKeys) * BwdTile<D>::kStride * 2 +
                        static_cast<size_t>(p.n_k + 1) * 4 + 2 * kChunkKeys * 8;
  if (D == 128) {  // tcgen05 / TMEM dQ pass (psa_attention.cu): 26 ms vs ~300 ms at cfg3
    rc = attn_bwd_dq_tc(p.q, p.k, p.v, p.k_pyr, p.v_pyr, p.dout, p.lse, drow, batch, p.hq, p.hkv,
                        p.n, p.b_q, p.b_k, p.levels, p.csr, p.info, p.causal, p.dq, s);
  } else {
    cudaFuncSetAttribute(bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_q));
    bwd_dq_kernel<D><<<static_cast<unsigned>(batch * p.hq * p.n_q), kBwdThreads, smem_q, s>>>(p);
    rc = psa_check_launch("bwd_dq_kernel");
  }
  if (rc) return rc;
  if (D == 128)  // tcgen05 / TMEM dK/dV pass (psa_attention.cu)
    return attn_bwd_dkv_tc(p.q, p.k, p.v, p.k_pyr, p.v_pyr, p.dout, p.lse, drow, batch, p.hq,
                           p.hkv, p.n, p.b_q, p.b_k, p.levels, p.level_map, p.causal, nl2, scratch,
                           p.dk, p.dv, s);
  const int cap = (p.hq / p.hkv) * p.n_q;
  const size_t smem = 6 * static_cast<size_t>(BwdTile<D>::kBytes) + 4 * kBwdRows * sizeof(float) +
                      static_cast<size_t>(cap) * 4;
  if (smem > 227 * 1024) return psa_fail(PSA_EINVAL, "too many query blocks per KV head for the backward kernel");
  cudaFuncSetAttribute(bwd_dkv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  bwd_dkv_kernel<D><<<dim3(static_cast<unsigned>(p.n_k), static_cast<unsigned>(batch * p.hkv)),
                      kBwdThreads, smem, s>>>(p, cap, scratch);
  return psa_check_launch("bwd_dkv_kernel");
}

}  // namespace psa

using namespace psa;

extern "C" size_t psa_attn_bwd_workspace_bytes(int64_t batch, int hq, int hkv, int64_t n, int d) {
  // D = rowsum(dO * O) per query row, then fp32 dK / dV accumulators: the raw rows (D = 64), or
  // the pooled rows of every level, < 2 n per KV head (D = 128 tcgen05 pass)
  const int64_t rows = batch * hq * n;
  return static_cast<size_t>(2 * ((rows + 63) / 64 * 64) + 4 * batch * hkv * n * d) * sizeof(float);
}

extern "C" int psa_attn_bwd(const void* q, const void* k, const void* v, const void* k_pyr,
                            const void* v_pyr, const void* out, const void* dout, const float* lse,
                            int64_t batch, int hq, int hkv, int64_t n, int d, int b_q, int b_k,
                            int levels, const uint16_t* plan_csr, const int32_t* plan_info,
                            const int8_t* level_map, int causal, void* dq, void* dk, void* dv,
                            void* workspace, void* stream) {
  PSA_CHECK_ARG(q && k && v && out && dout && lse && plan_csr && plan_info && level_map && dq &&
                    dk && dv && workspace,
                "null pointer argument");
  PSA_CHECK_ARG(d == 64 || d == 128, "head_dim must be 64 or 128");
  PSA_CHECK_ARG(b_q >= 1 && b_q <= kBwdRows && b_k >= 1 && b_k <= kBwdRows,
                "q_block and k_block must lie in 1..128 for the backward kernels");
  PSA_CHECK_ARG(n % b_q == 0 && n % b_k == 0, "layout does not divide seq_len");
  PSA_CHECK_ARG(levels >= 1 && levels <= 8 && b_k % (1 << (levels - 1)) == 0, "bad level count");
  PSA_CHECK_ARG(levels == 1 || (k_pyr && v_pyr), "pyramid pointers required for levels > 1");
  PSA_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0, "query heads must be a multiple of kv heads");
  PSA_CHECK_ARG(n / b_k <= 4096, "n_k must be <= 4096");
  // same coordinate guards as the forward (TMA coordinates and row indices are 32-bit), and the
  // dK/dV grid's y dimension is batch * hkv
  PSA_CHECK_ARG(batch * hq * n < (int64_t(1) << 31), "too many rows for 32-bit TMA coordinates");
  PSA_CHECK_ARG(n < (int64_t(1) << 23), "seq_len must be < 2^23");
  PSA_CHECK_ARG(batch * hkv <= 65535, "batch * kv heads must be <= 65535 for the backward grid");
  BwdParams p{};
  p.n = n;
  p.bkv_total = batch * hkv;
  p.hq = hq;
  p.hkv = hkv;
  p.b_q = b_q;
  p.b_k = b_k;
  p.levels = levels;
  p.n_q = static_cast<int>(n / b_q);
  p.n_k = static_cast<int>(n / b_k);
  p.causal = causal;
  p.scale = static_cast<float>(1.0 / sqrt(static_cast<double>(d)));
  p.scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(d)));
  p.q = static_cast<const uint16_t*>(q);
  p.k = static_cast<const uint16_t*>(k);
  p.v = static_cast<const uint16_t*>(v);
  p.k_pyr = static_cast<const uint16_t*>(k_pyr);
  p.v_pyr = static_cast<const uint16_t*>(v_pyr);
  p.dout = static_cast<const uint16_t*>(dout);
  p.lse = lse;
  p.csr = plan_csr;
  p.info = plan_info;
  p.level_map = level_map;
  p.dq = static_cast<uint16_t*>(dq);
  p.dk = static_cast<uint16_t*>(dk);
  p.dv = static_cast<uint16_t*>(dv);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const auto* o = static_cast<const uint16_t*>(out);
  return d == 128 ? launch_bwd<128>(p, batch, o, workspace, s) : launch_bwd<64>(p, batch, o, workspace, s);
}
