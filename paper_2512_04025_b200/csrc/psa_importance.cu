// K2: sampled block importance (pkg/src/pyrattn/importance.py:52-85).
//
// Reference: q_s = Q[q_rows], k_s = K[k_rows] (rows drawn by one seeded generator,
// importance.py:68-79); probs = row_softmax(q_s @ k_s.T / sqrt(d)) over ALL n_k*s_k sampled
// keys (importance.py:80, linalg.py:38-43); S = max (or mean) over each s_q x s_k block.
//
// GPU formulation (no n_q*s_q x n_k*s_k probability matrix is ever materialised):
//   pass A (this file, stats kernel): per sampled query row a, stream the sampled keys in
//     chunks of whole KV blocks; logits X = dot(q_a, k_b) / sqrt(d) in fp64 on the DMMA pipe
//     (products and sums of bf16 values are exact in fp64, so the summation order is free);
//     keep the per-(a, block) max logit M_aj plus an online (max, sum-exp) pair (m_a, l_a).
//   pass B (finalize kernel): S_ij = max_{a in block i} exp(M_aj - m_a) / l_a. Because exp
//     and the division are monotone, this equals the reference's max over the block of the
//     individually normalised probabilities (same subtraction, exp and division per element).
//   The mean reducer re-runs pass A with the final (m_a, l_a) and accumulates block sums of
//   exp(x - m_a) / l_a.
#include "common.cuh"
#include "psa_internal.h"

namespace psa {

constexpr int kImpRows = 64;   // sampled query rows per CTA
constexpr int kImpCols = 64;   // sampled key rows per chunk (upper bound)
constexpr int kImpThreads = 256;

PSA_DEV void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int D>
struct ImpSmem {
  static constexpr int kLd = D + 8;  // padded bf16 row: 8 rows of a fragment hit distinct banks
  uint16_t qs[kImpRows * kLd];
  uint16_t ks[kImpCols * kLd];
  double x[kImpRows * (kImpCols + 1)];
};

// Row maps: local sampled index -> row inside the head.
struct TableRows {  // importance_sampled: rows drawn by the reference's generator (host table)
  const int32_t* rows;
  PSA_DEV int64_t operator()(int a) const { return rows[a]; }
};
struct StridedRows {  // antidiagonal: element a of class r = block (a / per) offset r + (a % per)*stride
  int per, block, r, stride;
  const int32_t* blocks;  // optional list of the call's blocks (query side of q-block work units)
  PSA_DEV int64_t operator()(int a) const {
    const int bi = blocks != nullptr ? blocks[a / per] : a / per;
    return static_cast<int64_t>(bi) * block + r + (a % per) * stride;
  }
};

// Load `count` gathered bf16 rows of length D into registers (16 B per vector).
template <int D, class Rows>
PSA_DEV void gather_rows_regs(const uint16_t* __restrict__ base, const Rows& rows, int first,
                              int count, uint4 (&buf)[kImpCols * D / 8 / kImpThreads]) {
  constexpr int kVecPerRow = D / 8;
  constexpr int kPer = kImpCols * D / 8 / kImpThreads;
#pragma unroll
  for (int p = 0; p < kPer; ++p) {
    const int idx = threadIdx.x + p * kImpThreads;
    const int r = idx / kVecPerRow, c = idx % kVecPerRow;
    if (r < count) {
      const int64_t row = rows(first + r);
      buf[p] = __ldg(reinterpret_cast<const uint4*>(base + row * D) + c);
    } else {
      buf[p] = make_uint4(0, 0, 0, 0);
    }
  }
}

template <int D>
PSA_DEV void store_rows_bf16(uint16_t* dst, const uint4 (&buf)[kImpCols * D / 8 / kImpThreads]) {
  constexpr int kVecPerRow = D / 8;
  constexpr int kPer = kImpCols * D / 8 / kImpThreads;
  constexpr int kLd = D + 8;
#pragma unroll
  for (int p = 0; p < kPer; ++p) {
    const int idx = threadIdx.x + p * kImpThreads;
    const int r = idx / kVecPerRow, c = idx % kVecPerRow;
    *reinterpret_cast<uint4*>(dst + r * kLd + c * 8) = buf[p];
  }
}

PSA_DEV double bf16_to_f64(uint16_t h) {
  return static_cast<double>(__uint_as_float(static_cast<uint32_t>(h) << 16));
}

// 64 x 64 fp64 logit tile on the DMMA pipe: x[r][c] = dot(qs[r], ks[c]) (exact for bf16
// inputs). 8 warps in a 2 x 4 grid, warp tile 32 x 16 (4 x 2 m8n8k4 tiles).
template <int D>
PSA_DEV void dmma_logit_tile(ImpSmem<D>& sm) {
  constexpr int kLd = ImpSmem<D>::kLd;
  constexpr int kXld = kImpCols + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp >> 2, wc = warp & 3;
  double acc[4][2][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  const uint16_t* qa = sm.qs + (wr * 32 + (lane >> 2)) * kLd + (lane & 3);
  const uint16_t* kb = sm.ks + (wc * 16 + (lane >> 2)) * kLd + (lane & 3);
#pragma unroll 4
  for (int k4 = 0; k4 < D / 4; ++k4) {
    double af[4], bf[2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) af[mt] = bf16_to_f64(qa[mt * 8 * kLd + k4 * 4]);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) bf[nt] = bf16_to_f64(kb[nt * 8 * kLd + k4 * 4]);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) dmma_m8n8k4(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = wr * 32 + mt * 8 + (lane >> 2);
        const int c = wc * 16 + nt * 8 + (lane & 3) * 2 + e;
        sm.x[r * kXld + c] = acc[mt][nt][e];
      }
}

template <int D, bool MEAN>
__global__ void __launch_bounds__(kImpThreads, 2)
    importance_stats_kernel(const uint16_t* __restrict__ q, const uint16_t* __restrict__ k,
                            int hq, int hkv, int64_t n, const int32_t* __restrict__ q_rows,
                            const int32_t* __restrict__ k_rows, int R, int s_k, int n_k,
                            double sqrt_d, double* __restrict__ M, double* __restrict__ mstat,
                            double* __restrict__ lstat, const int32_t* __restrict__ qflag,
                            const int32_t* __restrict__ kflag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<ImpSmem<D>*>(smem_raw);
  constexpr int kXld = kImpCols + 1;
  constexpr int kPer = kImpCols * D / 8 / kImpThreads;

  const int bhq = blockIdx.y;
  const int b = bhq / hq, h = bhq % hq;
  const int hk = h / (hq / hkv);
  // with flags: only the heads the int8 path (psa_xlogits.cu) handed over
  if (qflag != nullptr && !(qflag[bhq] | kflag[b * hkv + hk])) return;
  const uint16_t* qh = q + static_cast<int64_t>(bhq) * n * D;
  const uint16_t* kh = k + (static_cast<int64_t>(b) * hkv + hk) * n * D;
  const int a0 = blockIdx.x * kImpRows;
  const int rows_here = min(kImpRows, R - a0);

  // sampled query rows -> fp64 smem (reuse the chunk register buffer for the gather)
  {
    uint4 buf[kPer];
    gather_rows_regs<D>(qh, TableRows{q_rows}, a0, rows_here, buf);
    store_rows_bf16<D>(sm.qs, buf);
  }

  const int blocks_per_chunk = kImpCols / s_k;  // s_k <= 64 checked on the host
  const int cw = blocks_per_chunk * s_k;
  const int C = n_k * s_k;
  const int n_chunks = (C + cw - 1) / cw;

  const int a_loc = threadIdx.x >> 2, quad = threadIdx.x & 3;
  const int a_glob = a0 + a_loc;
  const bool row_ok = a_loc < rows_here;

  double m_run = -INFINITY, l_run = 0.0;
  const double inv_sqrt_d = 1.0 / sqrt_d;
  double m_fin = 0.0, l_fin = 1.0;
  if (MEAN && row_ok) {
    m_fin = mstat[static_cast<int64_t>(bhq) * R + a_glob];
    l_fin = lstat[static_cast<int64_t>(bhq) * R + a_glob];
  }

  uint4 pref[kPer];
  gather_rows_regs<D>(kh, TableRows{k_rows}, 0, min(cw, C), pref);

  for (int ch = 0; ch < n_chunks; ++ch) {
    const int b0 = ch * cw;
    const int cols = min(cw, C - b0);
    __syncthreads();  // previous chunk's X/K consumers are done
    store_rows_bf16<D>(sm.ks, pref);
    if (ch + 1 < n_chunks) gather_rows_regs<D>(kh, TableRows{k_rows}, b0 + cw, min(cw, C - b0 - cw), pref);
    __syncthreads();

    dmma_logit_tile<D>(sm);  // raw fp64 dots (exact) -> sm.x
    __syncthreads();

    // ---- per-row statistics; 4 threads per row, blocks interleaved over the quad
    const double* xr = sm.x + a_loc * kXld;
    const int nb = cols / s_k;
    const int j0 = b0 / s_k;
    if (!MEAN) {
      // block max of the RAW dots (the finalize kernel divides once: x -> fl(x / sqrt(d)) is
      // monotone, so fl(max(x) / sqrt(d)) is exactly the reference's block-max logit)
      double lmax = -INFINITY;
      for (int bb = quad; bb < nb; bb += 4) {
        double bm = -INFINITY;
        for (int t = 0; t < s_k; ++t) bm = fmax(bm, xr[bb * s_k + t]);
        lmax = fmax(lmax, bm);
        if (row_ok) M[(static_cast<int64_t>(bhq) * R + a_glob) * n_k + j0 + bb] = bm;
      }
      lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, 1));
      lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, 2));
      const double m_new = fmax(m_run, __ddiv_rn(lmax, sqrt_d));  // importance.py:80
      // softmax denominator (only its value, not its summation order, matters downstream)
      double part = 0.0;
      for (int bb = quad; bb < nb; bb += 4)
        for (int t = 0; t < s_k; ++t)
          part = __dadd_rn(part, exp(__fma_rn(xr[bb * s_k + t], inv_sqrt_d, -m_new)));
      part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, 1));
      part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, 2));
      l_run = __dadd_rn(__dmul_rn(l_run, exp(__dsub_rn(m_run, m_new))), part);
      m_run = m_new;
    } else {
      for (int bb = quad; bb < nb; bb += 4) {
        double s = 0.0;
        for (int t = 0; t < s_k; ++t)
          s = __dadd_rn(s, __ddiv_rn(exp(__dsub_rn(__ddiv_rn(xr[bb * s_k + t], sqrt_d), m_fin)), l_fin));
        if (row_ok) M[(static_cast<int64_t>(bhq) * R + a_glob) * n_k + j0 + bb] = s;
      }
    }
  }
  if (!MEAN && row_ok && quad == 0) {
    mstat[static_cast<int64_t>(bhq) * R + a_glob] = m_run;
    lstat[static_cast<int64_t>(bhq) * R + a_glob] = l_run;
  }
}

// S_ij = max_a exp(fl(M_aj / sqrt(d)) - m_a) / l_a, M_aj = raw block-max dot
// (or mean: sum_a M_aj / (s_q*s_k))
// MAX: the candidates are ranked by y_a = M_aj / sqrt(d) - (m_a + ln l_a) (one multiply and one
// subtraction each; |error| << 1e-12); only those within 1e-9 of the best are evaluated exactly
// as fl(fl(exp(fl(fl(M_aj / sqrt(d)) - m_a))) / l_a), the reference's arithmetic (softmax,
// linalg.py:38-43, then the block max), so S is the same value as evaluating every candidate
// (exp and division are monotone) with ~1 exp and 2 divisions per (i, j) instead of s_q.
template <bool MEAN>
__global__ void __launch_bounds__(128) importance_finalize_kernel(
    const double* __restrict__ M, const double* __restrict__ mstat,
    const double* __restrict__ lstat, int R, int s_q, int s_k, int n_q, int n_k, double sqrt_d,
    double* __restrict__ S) {
  const int i = blockIdx.x;
  const int64_t bhq = blockIdx.y;
  constexpr int kMaxSq = 64;
  __shared__ double nl[kMaxSq];
  if (!MEAN && s_q <= kMaxSq) {
    for (int t = threadIdx.x; t < s_q; t += blockDim.x) {
      const int64_t a = bhq * R + static_cast<int64_t>(i) * s_q + t;
      nl[t] = mstat[a] + log(lstat[a]);
    }
    __syncthreads();
    const double inv = 1.0 / sqrt_d;
    const double* Mi = M + (bhq * R + static_cast<int64_t>(i) * s_q) * n_k;
    for (int j = threadIdx.x; j < n_k; j += blockDim.x) {
      constexpr int kReg = 8;  // the s_q <= 8 candidates in registers (all loads in flight)
      double mv[kReg];
#pragma unroll
      for (int t = 0; t < kReg; ++t) mv[t] = t < s_q ? Mi[static_cast<int64_t>(t) * n_k + j] : 0.0;
      double ybest = -INFINITY;
#pragma unroll
      for (int t = 0; t < kReg; ++t)
        if (t < s_q) ybest = fmax(ybest, mv[t] * inv - nl[t]);
      for (int t = kReg; t < s_q; ++t) ybest = fmax(ybest, Mi[static_cast<int64_t>(t) * n_k + j] * inv - nl[t]);
      double acc = -INFINITY;
      auto cand = [&](int t, double m_) {
        if (!(m_ * inv - nl[t] >= ybest - 1e-9)) return;
        const int64_t a = bhq * R + static_cast<int64_t>(i) * s_q + t;
        const double logit = __ddiv_rn(m_, sqrt_d);  // importance.py:80
        acc = fmax(acc, __ddiv_rn(exp(__dsub_rn(logit, mstat[a])), lstat[a]));
      };
#pragma unroll
      for (int t = 0; t < kReg; ++t)
        if (t < s_q) cand(t, mv[t]);
      for (int t = kReg; t < s_q; ++t) cand(t, Mi[static_cast<int64_t>(t) * n_k + j]);
      S[(bhq * n_q + i) * n_k + j] = acc;
    }
    return;
  }
  for (int j = threadIdx.x; j < n_k; j += blockDim.x) {
    double acc = MEAN ? 0.0 : -INFINITY;
    for (int t = 0; t < s_q; ++t) {
      const int64_t a = bhq * R + static_cast<int64_t>(i) * s_q + t;
      const double mv = M[a * n_k + j];
      if (MEAN) {
        acc = __dadd_rn(acc, mv);
      } else {
        const double logit = __ddiv_rn(mv, sqrt_d);  // importance.py:80
        const double p = __ddiv_rn(exp(__dsub_rn(logit, mstat[a])), lstat[a]);
        acc = fmax(acc, p);
      }
    }
    if (MEAN) acc = __ddiv_rn(acc, static_cast<double>(s_q) * static_cast<double>(s_k));
    S[(bhq * n_q + i) * n_k + j] = acc;
  }
}


// ------------------------------------------------------------------ antidiagonal estimator
// Reference: importance_antidiagonal (pkg/src/pyrattn/importance.py:97-132). Query row p of a
// query block reads the keys whose in-block column c satisfies (p + c) % stride == 0, i.e. the
// residue class (-p) mod stride of every KV block (b_k % stride == 0); logits are
// fl(dot * fl(1/sqrt(d))) (importance.py:113,128: multiply by the reciprocal), softmaxed over
// the row's n_k * per picks, summed per block, averaged over the b_q rows of the query block.
//
// All query rows with the same residue r share one key set, so each residue class is one dense
// (n_q * c_r) x (n_k * per) fp64 GEMM on the DMMA pipe. The stats kernel streams the class's
// keys in chunks of whole KV blocks; per row and chunk it takes the chunk max m_c (merged into
// a running max), and per block the pairwise (numpy order) sum E of exp(logit - m_c). The
// finalize kernel rescales E by exp(m_c - m_row) / l_row and averages over the query block's
// rows sequentially (numpy's axis-0 mean). Only the rescaling step differs from the reference's
// per-element exp(logit - m_row) / l_row (ulps; the level map is unchanged).
template <int D>
__global__ void __launch_bounds__(kImpThreads, 2)
    antidiag_stats_kernel(const uint16_t* __restrict__ q, const uint16_t* __restrict__ k,
                          int hq, int hkv, int64_t n, int b_q, int b_k, int stride, int n_k,
                          double scale, int bpc, int n_chunks, int n_q,
                          const int32_t* __restrict__ qblk, double* __restrict__ E,
                          double* __restrict__ Mc, double* __restrict__ mstat,
                          double* __restrict__ lstat, const int32_t* __restrict__ qflag,
                          const int32_t* __restrict__ kflag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<ImpSmem<D>*>(smem_raw);
  constexpr int kXld = kImpCols + 1;
  constexpr int kPer = kImpCols * D / 8 / kImpThreads;

  const int r = blockIdx.z;
  const int c_r = r < b_q ? (b_q - r + stride - 1) / stride : 0;  // rows of class r per block
  const int R = n_q * c_r;
  const int a0 = blockIdx.x * kImpRows;
  if (a0 >= R) return;
  const int rows_here = min(kImpRows, R - a0);
  const int bhq = blockIdx.y;
  const int b = bhq / hq, h = bhq % hq;
  const int hk = h / (hq / hkv);
  if (qflag != nullptr && !(qflag[bhq] | kflag[b * hkv + hk])) return;
  const uint16_t* qh = q + static_cast<int64_t>(bhq) * n * D;
  const uint16_t* kh = k + (static_cast<int64_t>(b) * hkv + hk) * n * D;
  const int per = b_k / stride;
  const int kr = (stride - r % stride) % stride;
  const StridedRows qmap{c_r, b_q, r, stride, qblk};
  const StridedRows kmap{per, b_k, kr, stride, nullptr};

  {
    uint4 buf[kPer];
    gather_rows_regs<D>(qh, qmap, a0, rows_here, buf);
    store_rows_bf16<D>(sm.qs, buf);
  }
  const int cw = bpc * per;  // whole KV blocks per chunk (cw <= 64 checked on the host)
  const int C = n_k * per;

  const int a_loc = threadIdx.x >> 2, quad = threadIdx.x & 3;
  const bool row_ok = a_loc < rows_here;
  const int64_t grow = row_ok ? qmap(a0 + a_loc) : 0;  // row inside the head
  double* Erow = E + (static_cast<int64_t>(bhq) * n + grow) * n_k;
  double m_run = -INFINITY, l_run = 0.0;

  uint4 pref[kPer];
  gather_rows_regs<D>(kh, kmap, 0, min(cw, C), pref);
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int c0 = ch * cw;
    const int cols = min(cw, C - c0);
    __syncthreads();
    store_rows_bf16<D>(sm.ks, pref);
    if (ch + 1 < n_chunks) gather_rows_regs<D>(kh, kmap, c0 + cw, min(cw, C - c0 - cw), pref);
    __syncthreads();
    dmma_logit_tile<D>(sm);
    __syncthreads();

    const double* xr = sm.x + a_loc * kXld;
    const int nb = cols / per;
    const int j0 = c0 / per;
    double cmax = -INFINITY;
    for (int bb = quad; bb < nb; bb += 4)
      for (int t = 0; t < per; ++t) cmax = fmax(cmax, xr[bb * per + t]);
    cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, 1));
    cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, 2));
    // fl(x * scale) is monotone in x: the max of the scaled logits is the scaled max
    const double m_new = fmax(m_run, __dmul_rn(cmax, scale));
    double part = 0.0;
    for (int bb = quad; bb < nb; bb += 4) {
      const double* xb = xr + bb * per;
      const double e = np_pairwise_sum_fn(per, [&](int t) {
        return exp(__dsub_rn(__dmul_rn(xb[t], scale), m_new));
      });
      part = __dadd_rn(part, e);
      if (row_ok) Erow[j0 + bb] = e;
    }
    part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, 1));
    part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, 2));
    l_run = __dadd_rn(__dmul_rn(l_run, exp(__dsub_rn(m_run, m_new))), part);
    m_run = m_new;
    if (row_ok && quad == 0) Mc[(static_cast<int64_t>(bhq) * n + grow) * n_chunks + ch] = m_new;
  }
  if (row_ok && quad == 0) {
    mstat[static_cast<int64_t>(bhq) * n + grow] = m_run;
    lstat[static_cast<int64_t>(bhq) * n + grow] = l_run;
  }
}

// S_ij = (sum_{p < b_q} E[p, j] * w(p, c) ) / b_q, p ascending, with one weight
// w = exp(m_c - m_p) / l_p per (row, chunk) shared by the chunk's bpc blocks (one thread per
// chunk): an exp and a division per (row, chunk) instead of per (row, block).
__global__ void __launch_bounds__(128) antidiag_finalize_kernel(
    const double* __restrict__ E, const double* __restrict__ Mc, const double* __restrict__ mstat,
    const double* __restrict__ lstat, int64_t n, int b_q, int n_q, int n_k, int bpc, int n_chunks,
    const int32_t* __restrict__ qblk, double* __restrict__ S) {
  const int il = blockIdx.x;  // the call's query block il = block qblk[il] of the head
  const int i = qblk != nullptr ? qblk[il] : il;
  const int64_t bhq = blockIdx.y;
  constexpr int kMaxBpc = 8;  // blocks per work item (a chunk of bpc > 8 blocks spans several)
  const int subs = (bpc + kMaxBpc - 1) / kMaxBpc;
  for (int it = threadIdx.x; it < n_chunks * subs; it += blockDim.x) {
    const int c = it / subs, sub = it % subs;
    const int j0 = c * bpc + sub * kMaxBpc;
    const int nb = min(min(kMaxBpc, bpc - sub * kMaxBpc), n_k - j0);
    double acc[kMaxBpc];
#pragma unroll
    for (int u = 0; u < kMaxBpc; ++u) acc[u] = 0.0;
#pragma unroll 4
    for (int p = 0; p < b_q; ++p) {
      const int64_t a = bhq * n + static_cast<int64_t>(i) * b_q + p;
      const double w = __ddiv_rn(exp(__dsub_rn(Mc[a * n_chunks + c], mstat[a])), lstat[a]);
#pragma unroll
      for (int u = 0; u < kMaxBpc; ++u)
        if (u < nb) acc[u] = __dadd_rn(acc[u], __dmul_rn(E[a * n_k + j0 + u], w));
    }
#pragma unroll
    for (int u = 0; u < kMaxBpc; ++u)
      if (u < nb) S[(bhq * n_q + il) * n_k + j0 + u] = __ddiv_rn(acc[u], static_cast<double>(b_q));
  }
}

// Chunk geometry of the antidiagonal statistics: the int8 path's key tiles when it applies
// (so the fp64 fallback heads produce identically laid-out chunk maxima), else 64-key chunks.
struct AdGeom {
  int per, bpc, n_chunks, c_max;
  XlGeometry xl;
};
static AdGeom ad_geometry(int64_t bhq, int64_t bkv, int64_t n, int b_q, int b_k, int stride,
                          int n_q, bool allow_xl) {
  AdGeom a{};
  a.per = b_k / stride;
  a.c_max = (b_q + stride - 1) / stride;
  const int n_k = static_cast<int>(n / b_k);
  a.xl = xl_geometry(bhq, bkv, n_q, n_k, stride, n_q * a.c_max, a.per, bhq * n);
  a.xl.ok = a.xl.ok && allow_xl;
  a.bpc = a.xl.ok ? a.xl.bpt : kImpCols / a.per;
  a.n_chunks = (n_k + a.bpc - 1) / a.bpc;
  return a;
}

template <int D>
static int launch_antidiag_dmma(const void* q, const void* k, int64_t batch, int hq, int hkv,
                                int64_t n, int b_q, int b_k, int stride, int n_q,
                                const int32_t* qblk, const AdGeom& g, double* E, double* Mc,
                                double* mstat, double* lstat, const int32_t* qflag,
                                const int32_t* kflag, cudaStream_t s) {
  const int64_t bhq = batch * hq;
  const int n_k = static_cast<int>(n / b_k);
  const size_t smem = sizeof(ImpSmem<D>);
  cudaFuncSetAttribute(antidiag_stats_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  dim3 grid((n_q * g.c_max + kImpRows - 1) / kImpRows, static_cast<unsigned>(bhq), stride);
  antidiag_stats_kernel<D><<<grid, kImpThreads, smem, s>>>(
      static_cast<const uint16_t*>(q), static_cast<const uint16_t*>(k), hq, hkv, n, b_q, b_k,
      stride, n_k, 1.0 / sqrt(static_cast<double>(D)), g.bpc, g.n_chunks, n_q, qblk, E, Mc, mstat,
      lstat, qflag, kflag);
  return psa_check_launch("antidiag_stats_kernel");
}

}  // namespace psa

using namespace psa;

static size_t ad_fp64_bytes(int64_t bhq, int64_t n, int n_k, int n_chunks) {
  return static_cast<size_t>(bhq * n * (n_k + n_chunks + 2)) * sizeof(double);
}

extern "C" size_t psa_antidiag_workspace_bytes_rows(int64_t bhq, int64_t bkv, int64_t n, int b_q,
                                                    int b_k, int stride, int n_qsel) {
  if (stride < 1 || b_q < 1 || b_k % stride || b_k / stride > kImpCols || n % b_k || n % b_q ||
      n_qsel < 1)
    return 0;
  const AdGeom g = ad_geometry(bhq, bkv, n, b_q, b_k, stride, n_qsel, true);
  return ad_fp64_bytes(bhq, n, static_cast<int>(n / b_k), g.n_chunks) + (g.xl.ok ? g.xl.bytes : 0);
}

extern "C" size_t psa_antidiag_workspace_bytes(int64_t bhq, int64_t bkv, int64_t n, int b_q,
                                               int b_k, int stride) {
  if (b_q < 1 || n % b_q) return 0;
  return psa_antidiag_workspace_bytes_rows(bhq, bkv, n, b_q, b_k, stride, static_cast<int>(n / b_q));
}

extern "C" int psa_importance_antidiagonal_rows(const void* q, const void* k, int64_t batch,
                                                int hq, int hkv, int64_t n, int d, int b_q, int b_k,
                                                int stride, int flags, const int32_t* qblk,
                                                int n_qsel, double* scores, void* workspace,
                                                void* stream);

extern "C" int psa_importance_antidiagonal(const void* q, const void* k, int64_t batch, int hq,
                                           int hkv, int64_t n, int d, int b_q, int b_k,
                                           int stride, int flags, double* scores,
                                           void* workspace, void* stream) {
  PSA_CHECK_ARG(b_q >= 1 && n % b_q == 0, "layout does not divide seq_len");
  return psa_importance_antidiagonal_rows(q, k, batch, hq, hkv, n, d, b_q, b_k, stride, flags,
                                          nullptr, static_cast<int>(n / b_q), scores, workspace,
                                          stream);
}

extern "C" int psa_importance_antidiagonal_rows(const void* q, const void* k, int64_t batch,
                                                int hq, int hkv, int64_t n, int d, int b_q, int b_k,
                                                int stride, int flags, const int32_t* qblk,
                                                int n_qsel, double* scores, void* workspace,
                                                void* stream) {
  PSA_CHECK_ARG(q && k && scores && workspace, "null pointer argument");
  PSA_CHECK_ARG(d == 64 || d == 128, "head_dim must be 64 or 128 for the sm_100a path");
  PSA_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0, "query heads must be a multiple of kv heads");
  PSA_CHECK_ARG(b_q >= 1 && b_k >= 1 && n % b_q == 0 && n % b_k == 0, "layout does not divide seq_len");
  PSA_CHECK_ARG(stride >= 1 && b_k % stride == 0, "stride must divide k_block");
  PSA_CHECK_ARG(b_k / stride <= kImpCols,
                "k_block / stride > 64 is not supported by the sm_100a antidiagonal kernel");
  PSA_CHECK_ARG(n_qsel >= 1 && n_qsel <= n / b_q, "query-block count outside 1..n_q");
  PSA_CHECK_ARG(qblk != nullptr || n_qsel == n / b_q, "a query-block subset needs its block list");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t bhq = batch * hq, bkv = batch * hkv;
  const int n_q = n_qsel, n_k = static_cast<int>(n / b_k);
  const AdGeom g = ad_geometry(bhq, bkv, n, b_q, b_k, stride, n_q, !(flags & PSA_IMP_FP64_ONLY));
  double* E = static_cast<double*>(workspace);
  double* Mc = E + bhq * n * n_k;
  double* mstat = Mc + bhq * n * g.n_chunks;
  double* lstat = mstat + bhq * n;
  const int32_t* qflag = nullptr;
  const int32_t* kflag = nullptr;
  int rc = PSA_OK;
  if (g.xl.ok) {
    void* xws = static_cast<uint8_t*>(workspace) + ad_fp64_bytes(bhq, n, n_k, g.n_chunks);
    rc = xl_antidiag(q, k, batch, hq, hkv, n, d, b_q, b_k, stride, n_q, qblk, g.xl, xws, E, Mc,
                     mstat, lstat, s);
    if (rc) return rc;
    qflag = xl_qflags(g.xl, xws);
    kflag = qflag + bhq;
  }
  rc = d == 128 ? launch_antidiag_dmma<128>(q, k, batch, hq, hkv, n, b_q, b_k, stride, n_q, qblk,
                                            g, E, Mc, mstat, lstat, qflag, kflag, s)
                : launch_antidiag_dmma<64>(q, k, batch, hq, hkv, n, b_q, b_k, stride, n_q, qblk,
                                           g, E, Mc, mstat, lstat, qflag, kflag, s);
  if (rc) return rc;
  antidiag_finalize_kernel<<<dim3(n_q, bhq), 128, 0, s>>>(E, Mc, mstat, lstat, n, b_q, n_q, n_k,
                                                          g.bpc, g.n_chunks, qblk, scores);
  return psa_check_launch("antidiag_finalize_kernel");
}

static XlGeometry sampled_xl_geometry(int64_t bhq, int64_t bkv, int n_q, int s_q, int n_k,
                                      int s_k, bool allow) {
  XlGeometry g = xl_geometry(bhq, bkv, n_q, n_k, 1, n_q * s_q, s_k,
                             bhq * static_cast<int64_t>(n_q) * s_q);
  g.ok = g.ok && allow;
  return g;
}

static size_t sampled_fp64_bytes(int64_t bhq, int n_q, int s_q, int n_k) {
  const int64_t R = static_cast<int64_t>(n_q) * s_q;
  return static_cast<size_t>(bhq * R * n_k + 2 * bhq * R) * sizeof(double);
}

extern "C" size_t psa_importance_workspace_bytes(int64_t bhq, int64_t bkv, int n_q, int s_q,
                                                 int n_k, int s_k) {
  const XlGeometry g = sampled_xl_geometry(bhq, bkv, n_q, s_q, n_k, s_k, true);
  return sampled_fp64_bytes(bhq, n_q, s_q, n_k) + (g.ok ? g.bytes : 0);
}

template <int D>
static int launch_importance(const void* q, const void* k, int64_t batch, int hq, int hkv,
                             int64_t n, int b_q, const int32_t* q_rows, const int32_t* k_rows,
                             int R, int s_q, int s_k, int n_q, int n_k, int reducer, int flags,
                             double* scores, void* ws, cudaStream_t s) {
  const int64_t bhq = batch * hq, bkv = batch * hkv;
  double* M = static_cast<double*>(ws);
  double* mstat = M + bhq * R * n_k;
  double* lstat = mstat + bhq * R;
  const int32_t* qflag = nullptr;
  const int32_t* kflag = nullptr;
  int rc = PSA_OK;
  const XlGeometry g = sampled_xl_geometry(bhq, bkv, n_q, s_q, n_k, s_k,
                                           reducer == 0 && !(flags & PSA_IMP_FP64_ONLY));
  if (g.ok) {  // exact logits on the int8 tensor cores; DMMA only for the heads it flags
    void* xws = static_cast<uint8_t*>(ws) + sampled_fp64_bytes(bhq, n_q, s_q, n_k);
    rc = xl_sampled_max(q, k, batch, hq, hkv, n, D, b_q, static_cast<int>(n / n_k), n_q, q_rows,
                        k_rows, s_q, s_k, g, xws, M, mstat, lstat, s);
    if (rc) return rc;
    qflag = xl_qflags(g, xws);
    kflag = qflag + bhq;
  }
  const size_t smem = sizeof(ImpSmem<D>);
  cudaFuncSetAttribute(importance_stats_kernel<D, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaFuncSetAttribute(importance_stats_kernel<D, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  dim3 grid((R + kImpRows - 1) / kImpRows, static_cast<unsigned>(bhq));
  const double sqrt_d = sqrt(static_cast<double>(D));
  auto* qq = static_cast<const uint16_t*>(q);
  auto* kk = static_cast<const uint16_t*>(k);
  importance_stats_kernel<D, false><<<grid, kImpThreads, smem, s>>>(
      qq, kk, hq, hkv, n, q_rows, k_rows, R, s_k, n_k, sqrt_d, M, mstat, lstat, qflag, kflag);
  rc = psa_check_launch("importance_stats_kernel");
  if (rc) return rc;
  if (reducer == 1) {
    importance_stats_kernel<D, true><<<grid, kImpThreads, smem, s>>>(
        qq, kk, hq, hkv, n, q_rows, k_rows, R, s_k, n_k, sqrt_d, M, mstat, lstat, nullptr,
        nullptr);
    rc = psa_check_launch("importance_stats_kernel<mean>");
    if (rc) return rc;
    importance_finalize_kernel<true><<<dim3(n_q, bhq), 128, 0, s>>>(M, mstat, lstat, R, s_q, s_k,
                                                                     n_q, n_k, sqrt_d, scores);
  } else {
    importance_finalize_kernel<false><<<dim3(n_q, bhq), 128, 0, s>>>(M, mstat, lstat, R, s_q,
                                                                      s_k, n_q, n_k, sqrt_d, scores);
  }
  return psa_check_launch("importance_finalize_kernel");
}

extern "C" int psa_importance_sampled_rows(const void* q, const void* k, int64_t batch, int hq,
                                           int hkv, int64_t n, int d, int b_q, int b_k,
                                           const int32_t* q_rows, const int32_t* k_rows, int s_q,
                                           int s_k, int reducer, int flags, int n_qsel,
                                           double* scores, void* workspace, void* stream);

extern "C" int psa_importance_sampled(const void* q, const void* k, int64_t batch, int hq,
                                      int hkv, int64_t n, int d, int b_q, int b_k,
                                      const int32_t* q_rows, const int32_t* k_rows, int s_q,
                                      int s_k, int reducer, int flags, double* scores,
                                      void* workspace, void* stream) {
  PSA_CHECK_ARG(b_q >= 1 && n % b_q == 0, "layout does not divide seq_len");
  return psa_importance_sampled_rows(q, k, batch, hq, hkv, n, d, b_q, b_k, q_rows, k_rows, s_q,
                                     s_k, reducer, flags, static_cast<int>(n / b_q), scores,
                                     workspace, stream);
}

// q_rows: the sample rows of the call's n_qsel query blocks (n_qsel * s_q entries, block-major);
// scores: fp64 [batch*hq, n_qsel, n_k] (the q-block work units of the multi-GPU partition).
extern "C" int psa_importance_sampled_rows(const void* q, const void* k, int64_t batch, int hq,
                                           int hkv, int64_t n, int d, int b_q, int b_k,
                                           const int32_t* q_rows, const int32_t* k_rows, int s_q,
                                           int s_k, int reducer, int flags, int n_qsel,
                                           double* scores, void* workspace, void* stream) {
  PSA_CHECK_ARG(q && k && q_rows && k_rows && scores && workspace, "null pointer argument");
  PSA_CHECK_ARG(d == 64 || d == 128, "head_dim must be 64 or 128 for the sm_100a path");
  PSA_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0, "query heads must be a multiple of kv heads");
  PSA_CHECK_ARG(b_q >= 1 && b_k >= 1 && n % b_q == 0 && n % b_k == 0, "layout does not divide seq_len");
  PSA_CHECK_ARG(s_q >= 1 && s_q <= b_q, "s_q outside 1..q_block");
  PSA_CHECK_ARG(s_k >= 1 && s_k <= b_k, "s_k outside 1..k_block");
  PSA_CHECK_ARG(s_k <= kImpCols, "s_k > 64 is not supported by the sm_100a importance kernel");
  PSA_CHECK_ARG(reducer == 0 || reducer == 1, "reducer must be 0 (max) or 1 (mean)");
  PSA_CHECK_ARG(n_qsel >= 1 && n_qsel <= n / b_q, "query-block count outside 1..n_q");
  const int n_q = n_qsel, n_k = static_cast<int>(n / b_k);
  const int R = n_q * s_q;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (d == 128)
    return launch_importance<128>(q, k, batch, hq, hkv, n, b_q, q_rows, k_rows, R, s_q, s_k, n_q,
                                  n_k, reducer, flags, scores, workspace, s);
  return launch_importance<64>(q, k, batch, hq, hkv, n, b_q, q_rows, k_rows, R, s_q, s_k, n_q,
                               n_k, reducer, flags, scores, workspace, s);
}
