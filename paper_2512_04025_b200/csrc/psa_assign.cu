// K3: multi-level mask assignment + compact per-query-block plan.
//
// Reference semantics (pkg/src/pyrattn/mask.py):
//   _descending_order      :107-109  stable argsort of -s (ties -> ascending block index)
//   _compensated_cumsum    :112-125  sequential Neumaier, out[i] = total + comp
//   assign_threshold       :128-151  row/fsum(row) (uniform 1/n_k if the total is 0), clip 1.0,
//                                    searchsorted(taus, cum, 'left') -> level t+1, 0 past tau_H
//   binary_mask            :154-158  threshold with a single tau
//   assign_quantile        :167-179  rank levels via searchsorted(counts, rank, 'right')
//   combine_mask           :237-247  min(M, caps[j])
//   causal_premask         :324-349  future -> 0, straddling -> 1, visible -> keep
//
// One CTA (128 threads) per (head, query block) row. The sort is a bitonic network in shared
// memory; the row total is computed EXACTLY (a 256-bit fixed-point superaccumulator reduced
// across a warp, then rounded half-to-even), which is what CPython's math.fsum returns; the
// Neumaier recurrence is inherently sequential and runs on one thread with the same IEEE ops
// in the same order, so identical scores give identical levels.
#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"
#include "psa_internal.h"

namespace psa {

struct AssignParams {
  LevelRule rule;
  int n_q, n_k, hq, hkv, b_q, b_k, levels, causal, n_pad;
  const int32_t* qblk;  // optional: score row i is query block qblk[i] of the head (work units)
};

// Bits [lo, lo + cnt) (cnt <= 53) of a 256-bit little-endian limb array; bits below 0 read 0.
PSA_DEV uint64_t bits256(const uint32_t (&w)[8], int lo, int cnt) {
  auto word = [&](int i) -> uint64_t { return (i >= 0 && i < 8) ? w[i] : 0u; };
  uint64_t v;
  if (lo >= 0) {
    const int i = lo >> 5, sh = lo & 31;
    v = (word(i) | (word(i + 1) << 32)) >> sh;
    if (sh) v |= word(i + 2) << (64 - sh);
  } else {
    v = (lo > -64) ? (word(0) | (word(1) << 32)) << (-lo) : 0u;
  }
  return cnt >= 64 ? v : (v & ((1ull << cnt) - 1ull));
}
// Any bit set below bit `lo` (lo may be <= 0 or >= 256).
PSA_DEV bool any_below(const uint32_t (&w)[8], int lo) {
  if (lo <= 0) return false;
  const int full = min(lo >> 5, 8);
  bool any = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) any = any || (i < full && w[i] != 0u);
  if (full < 8 && (lo & 31)) any = any || (w[full] & ((1u << (lo & 31)) - 1u)) != 0u;
  return any;
}

// Correctly rounded (half-to-even) sum of n non-negative finite doubles, sorted descending
// (v[0] is the maximum). Called by the whole 128-thread block (red: 4 x 8 shared limbs); every
// thread gets the result. Equivalent to CPython math.fsum for this input class.
PSA_DEV double exact_sum_sorted_nonneg(const double* v, int n, unsigned long long* red,
                                       int* sticky_s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double vmax = v[0];
  if (!(vmax > 0.0)) return 0.0;
  const int emax = ilogb(vmax);
  const int lsb = emax - 243;  // window bit 0 weight 2^lsb; sum < 2^(emax+13) <= 2^(lsb+256)
  uint64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool sticky = false;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t bits = __double_as_longlong(v[i]);
    const int e = static_cast<int>((bits >> 52) & 0x7FF);
    uint64_t m = bits & 0xFFFFFFFFFFFFFull;
    if (e != 0) m |= 1ull << 52;
    if (m == 0) continue;
    int pos = (e != 0 ? e : 1) - 1075 - lsb;
    if (pos < 0) {
      const int sh = -pos;
      if (sh >= 64) {
        sticky = true;
        continue;
      }
      if (m & ((1ull << sh) - 1ull)) sticky = true;
      m >>= sh;
      pos = 0;
    }
    const int li = pos >> 5, s = pos & 31;
    const uint64_t lo = (m & 0xFFFFFFFFull) << s;
    const uint64_t hi = (m >> 32) << s;
    const uint64_t p0 = lo & 0xFFFFFFFFull;
    const uint64_t p1 = (lo >> 32) + (hi & 0xFFFFFFFFull);
    const uint64_t p2 = hi >> 32;
#pragma unroll
    for (int L = 0; L < 8; ++L)
      acc[L] += (L == li) ? p0 : (L == li + 1) ? p1 : (L == li + 2) ? p2 : 0ull;
  }
#pragma unroll
  for (int L = 0; L < 8; ++L)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[L] += __shfl_xor_sync(0xffffffffu, acc[L], o);
  sticky = __any_sync(0xffffffffu, sticky);
  if (threadIdx.x == 0) *sticky_s = 0;
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int L = 0; L < 8; ++L) red[warp * 8 + L] = acc[L];
    if (sticky) atomicOr(sticky_s, 1);
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int L = 0; L < 8; ++L) {
    acc[L] = 0;
    for (int w2 = 0; w2 < nw; ++w2) acc[L] += red[w2 * 8 + L];  // < 2^41 per limb: no overflow
  }
  sticky = *sticky_s != 0;
  uint32_t w[8];
  uint64_t carry = 0;
#pragma unroll
  for (int L = 0; L < 8; ++L) {
    const uint64_t t = acc[L] + carry;
    w[L] = static_cast<uint32_t>(t);
    carry = t >> 32;
  }
  int p = -1;
  for (int L = 7; L >= 0 && p < 0; --L)
    if (w[L]) p = L * 32 + 31 - __clz(w[L]);
  int r = p - 52;
  if (lsb + p < -1022) r = max(r, -1074 - lsb);  // subnormal result
  uint64_t mant = bits256(w, r, p - r + 1);
  const bool rbit = bits256(w, r - 1, 1) != 0;
  const bool st = sticky || any_below(w, r - 1);
  if (rbit && (st || (mant & 1ull))) mant += 1;
  return ldexp(static_cast<double>(mant), lsb + r);
}

PSA_DEV int slot_rows(int pooled) {  // power-of-two slot >= 8 rows (TMA/UMMA atom alignment)
  int s = 8;
  while (s < pooled) s <<= 1;
  return s;
}

// Level-major compaction of lvl[0..n_k) into the plan row; returns per-level counts in cnt.
PSA_DEV void emit_plan_row(const int8_t* lvl, int n_k, int levels, int b_k, int64_t unit,
                           uint16_t* __restrict__ csr, int32_t* __restrict__ info,
                           unsigned long long* __restrict__ level_counts, int* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  int base = 0;
  int64_t rows_total = 0;
  for (int h = 1; h <= levels; ++h) {
    const int start_h = base;
    for (int j0 = 0; j0 < n_k; j0 += blockDim.x) {
      const int j = j0 + threadIdx.x;
      const bool f = j < n_k && lvl[j] == h;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) warp_tot[warp] = __popc(bal);
      __syncthreads();
      int off = base;
      int tot = 0;
      for (int w = 0; w < nwarps; ++w) {
        if (w < warp) off += warp_tot[w];
        tot += warp_tot[w];
      }
      if (f)
        csr[unit * n_k + off + __popc(bal & ((1u << lane) - 1u))] =
            static_cast<uint16_t>(j | (h << 12));
      __syncthreads();
      base += tot;
    }
    const int cnt = base - start_h;
    if (threadIdx.x == 0) {
      rows_total += static_cast<int64_t>(cnt) * slot_rows(b_k >> (h - 1));
      if (level_counts && cnt) atomicAdd(level_counts + h, static_cast<unsigned long long>(cnt));
    }
  }
  if (threadIdx.x == 0) {
    info[unit * 2 + 0] = base;
    info[unit * 2 + 1] = static_cast<int32_t>(rows_total);  // slot rows; tiles = ceil(rows / tile)
    if (level_counts && n_k - base)
      atomicAdd(level_counts, static_cast<unsigned long long>(n_k - base));
  }
}

// Descending stable order of a row of n_k <= 128*IPT non-negative scores (numpy's stable argsort
// of -s, mask.py:107-109). The fp64 bit patterns are monotone for non-negative values (-0.0 is
// folded into +0.0 first, as the comparison-based sort treats them as equal). A CUB block radix
// sort orders the rows by the top 32 of the 63 value bits with the column index as payload
// (8 passes of 4-bit digits instead of 16); radix sort is stable, so equal keys keep ascending column order.
// Entries whose top 32 bits tie but whose low bits differ (rare) are then put in full order by
// an insertion pass with the same (value desc, column asc) comparator. Padding keys (0) follow
// every real score, zeros included.
#ifndef PSA_ASSIGN_RADIX_BITS
#define PSA_ASSIGN_RADIX_BITS 4  // A/B at cfg3: 4 bits 0.81 ms, 5 bits 0.85, 6 bits 0.92
#endif
template <int IPT, int RB = PSA_ASSIGN_RADIX_BITS>  // digit bits per radix pass
__global__ void __launch_bounds__(128) assign_levels_kernel(
    const double* __restrict__ S, const int8_t* __restrict__ caps, AssignParams p,
    int8_t* __restrict__ level_map, uint16_t* __restrict__ csr, int32_t* __restrict__ info,
    unsigned long long* __restrict__ level_counts) {
  using Sort = cub::BlockRadixSort<unsigned int, 128, IPT, int, RB>;
  __shared__ typename Sort::TempStorage sort_tmp;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* keys = reinterpret_cast<double*>(smem_raw);
  int* idx = reinterpret_cast<int*>(keys + p.n_pad);
  int8_t* lsorted = reinterpret_cast<int8_t*>(idx + p.n_pad);
  int8_t* lvl = lsorted + p.n_pad;
  double* row_s = reinterpret_cast<double*>(smem_raw + static_cast<size_t>(p.n_pad) * 14 + 16);
  __shared__ double total_s;
  __shared__ int unsorted_s;
  __shared__ unsigned long long red_s[4 * 8];
  __shared__ int sticky_s;
  __shared__ int warp_tot[4];

  const int i = blockIdx.x;
  const int64_t bhq = blockIdx.y;
  const int64_t unit = bhq * p.n_q + i;
  const double* row = S + unit * p.n_k;
  {
    unsigned int kb[IPT];
    int vb[IPT];
    if (threadIdx.x == 0) unsorted_s = 0;
#pragma unroll
    for (int e = 0; e < IPT; ++e) {  // blocked arrangement: thread t holds [t*IPT, t*IPT+IPT)
      const int t = threadIdx.x * IPT + e;
      double x = t < p.n_k ? row[t] : 0.0;
      x = x == 0.0 ? 0.0 : x;
      row_s[t] = x;
      kb[e] = static_cast<unsigned int>(static_cast<unsigned long long>(__double_as_longlong(x)) >> 31);
      vb[e] = t;
    }
    Sort(sort_tmp).SortDescending(kb, vb, 0, 32);  // value bits 62..31
    __syncthreads();  // row_s complete
#pragma unroll
    for (int e = 0; e < IPT; ++e) {
      const int t = threadIdx.x * IPT + e;
      keys[t] = row_s[vb[e]];
      idx[t] = vb[e];
    }
  }
  __syncthreads();
  for (int t = 1 + threadIdx.x; t < p.n_pad; t += blockDim.x)  // low-bit ties out of order?
    if (__double_as_longlong(keys[t]) > __double_as_longlong(keys[t - 1])) unsorted_s = 1;
  __syncthreads();
  if (unsorted_s && threadIdx.x == 0) {  // rare: insertion pass, (value desc, column asc)
    for (int t = 1; t < p.n_pad; ++t) {
      const double kv = keys[t];
      const int iv = idx[t];
      int u = t;
      while (u > 0 && (keys[u - 1] < kv || (keys[u - 1] == kv && idx[u - 1] > iv))) {
        keys[u] = keys[u - 1];
        idx[u] = idx[u - 1];
        --u;
      }
      keys[u] = kv;
      idx[u] = iv;
    }
  }
  __syncthreads();

  if (p.rule.mode == 0) {
    {
      const double tot = exact_sum_sorted_nonneg(keys, p.n_k, red_s, &sticky_s);  // math.fsum(row)
      if (threadIdx.x == 0) total_s = tot;
    }
    __syncthreads();
    const double tot = total_s;
    const double uni = 1.0 / static_cast<double>(p.n_k);
    for (int t = threadIdx.x; t < p.n_k; t += blockDim.x)
      keys[t] = tot > 0.0 ? __ddiv_rn(keys[t], tot) : uni;
    __syncthreads();
    // Fast path: fp64 prefix sums in parallel (blocked: thread t owns positions [t*IPT, t*IPT +
    // IPT)); they differ from the reference's sequential Neumaier sums by ~1e-15 at most (n_k <=
    // 4096 non-negative terms summing to 1), so the comparisons cum <= tau agree whenever no sum
    // lies within 1e-12 of a threshold. Otherwise (probability ~1e-8 per row) the row falls back
    // to the exact sequential recurrence below.
    {
      double loc[IPT];
      double run = 0.0;
#pragma unroll
      for (int e = 0; e < IPT; ++e) {
        const int t = threadIdx.x * IPT + e;
        run = __dadd_rn(run, t < p.n_k ? keys[t] : 0.0);
        loc[e] = run;
      }
      double excl = run;  // inclusive scan of the thread totals, then shifted
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, excl, o);
        if (lane >= o) excl = __dadd_rn(excl, y);
      }
      __shared__ double warp_sum[4];
      if (lane == 31) warp_sum[warp] = excl;
      __syncthreads();
      double wbase = 0.0;
      for (int w = 0; w < warp; ++w) wbase = __dadd_rn(wbase, warp_sum[w]);
      excl = __dadd_rn(__dsub_rn(excl, run), wbase);
      bool fragile = false;
#pragma unroll
      for (int e = 0; e < IPT; ++e) {
        const int t = threadIdx.x * IPT + e;
        loc[e] = fmin(__dadd_rn(excl, loc[e]), 1.0);
        if (t < p.n_k)
          for (int c = 0; c < p.rule.n_cuts; ++c)
            fragile |= fabs(loc[e] - p.rule.taus[c]) <= 1e-12;
      }
      fragile = __syncthreads_or(fragile) != 0;
      if (!fragile) {
#pragma unroll
        for (int e = 0; e < IPT; ++e) {
          const int t = threadIdx.x * IPT + e;
          if (t < p.n_k) keys[t] = loc[e];
        }
      } else if (threadIdx.x == 0) {
      // The recurrence is inherently sequential; keep only it on one thread and store
      // cum_t in place of e_t (read just before it is overwritten).
      // t = 0: total = 0 < x (the else branch of Neumaier's |total| >= |x| test); for t >= 1 the
      // test always holds since the values are sorted descending and non-negative (total >=
      // x_{t-1} >= x_t), so the loop carries no compare or select.
      double total = keys[0], comp = 0.0;  // fl(0 + x0) = x0, d = (x0 - x0) + 0 = 0
      keys[0] = fmin(total, 1.0);
#pragma unroll 8
      for (int t = 1; t < p.n_k; ++t) {
        const double x = keys[t];
        const double tt = __dadd_rn(total, x);
        comp = __dadd_rn(comp, __dadd_rn(__dsub_rn(total, tt), x));
        total = tt;
        keys[t] = fmin(__dadd_rn(total, comp), 1.0);
      }
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < p.n_k; t += blockDim.x) {
      const double cum = keys[t];
      int c = 0;
      while (c < p.rule.n_cuts && p.rule.taus[c] < cum) ++c;  // searchsorted 'left'
      lsorted[t] = static_cast<int8_t>(c < p.rule.n_cuts ? c + 1 : 0);
    }
  } else {
    for (int t = threadIdx.x; t < p.n_k; t += blockDim.x) {
      int c = 0;
      while (c < p.rule.n_cuts && p.rule.counts[c] <= t) ++c;  // searchsorted 'right'
      lsorted[t] = static_cast<int8_t>(c < p.rule.n_cuts ? c + 1 : 0);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < p.n_k; t += blockDim.x) lvl[idx[t]] = lsorted[t];
  __syncthreads();

  const int b = static_cast<int>(bhq / p.hq), h = static_cast<int>(bhq % p.hq);
  const int64_t bhkv = static_cast<int64_t>(b) * p.hkv + h / (p.hq / p.hkv);
  const int iq = p.qblk != nullptr ? p.qblk[i] : i;
  const int64_t q_lo = static_cast<int64_t>(iq) * p.b_q, q_hi = q_lo + p.b_q - 1;
  for (int j = threadIdx.x; j < p.n_k; j += blockDim.x) {
    int L = lvl[j];
    if (caps) L = min(L, static_cast<int>(caps[bhkv * p.n_k + j]));
    if (p.causal) {
      const int64_t k_lo = static_cast<int64_t>(j) * p.b_k, k_hi = k_lo + p.b_k - 1;
      if (k_lo > q_hi) L = 0;
      else if (!(k_hi <= q_lo)) L = 1;
    }
    lvl[j] = static_cast<int8_t>(L);
    level_map[unit * p.n_k + j] = static_cast<int8_t>(L);
  }
  __syncthreads();
  emit_plan_row(lvl, p.n_k, p.levels, p.b_k, unit, csr, info, level_counts, warp_tot);
}

// Plan from a caller-supplied mask (psa_streaming drop-in). Validates like
// attention.py:66-75 (_check_mask) and attention.py:88-108 (_causal_key_mask).
template <typename T>
__global__ void __launch_bounds__(128) mask_to_plan_kernel(
    const T* __restrict__ mask, int n_q, int n_k, int causal, int b_q, int b_k, int levels,
    uint16_t* __restrict__ csr, int32_t* __restrict__ info,
    unsigned long long* __restrict__ level_counts, int32_t* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int8_t* lvl = reinterpret_cast<int8_t*>(smem_raw);
  __shared__ int warp_tot[4];
  const int64_t unit = blockIdx.x;
  const int i = static_cast<int>(unit % n_q);
  const int64_t q_lo = static_cast<int64_t>(i) * b_q;
  for (int j = threadIdx.x; j < n_k; j += blockDim.x) {
    const long long L = static_cast<long long>(mask[unit * n_k + j]);
    int8_t v = 0;
    if (L < 0 || L > levels) {
      atomicOr(bad, 1);
    } else {
      v = static_cast<int8_t>(L);
      if (causal && L > 1) {
        const int64_t k_hi = static_cast<int64_t>(j + 1) * b_k - 1;
        if (!(k_hi <= q_lo)) atomicOr(bad, 2);  // pooled level on a straddling pair
      }
    }
    lvl[j] = v;
  }
  __syncthreads();
  emit_plan_row(lvl, n_k, levels, b_k, unit, csr, info, level_counts, warp_tot);
}

}  // namespace psa

using namespace psa;

extern "C" int psa_assign_levels_rows(const double* scores, int64_t batch, int hq, int hkv,
                                      int n_q, int n_k, int mode, const double* taus,
                                      const int32_t* counts, int n_cuts, const int8_t* caps,
                                      int causal, int b_q, int b_k, int levels,
                                      const int32_t* qblk, int8_t* level_map, uint16_t* plan_csr,
                                      int32_t* plan_info, unsigned long long* level_counts,
                                      void* stream);

extern "C" int psa_assign_levels(const double* scores, int64_t batch, int hq, int hkv, int n_q,
                                 int n_k, int mode, const double* taus, const int32_t* counts,
                                 int n_cuts, const int8_t* caps, int causal, int b_q, int b_k,
                                 int levels, int8_t* level_map, uint16_t* plan_csr,
                                 int32_t* plan_info, unsigned long long* level_counts,
                                 void* stream) {
  return psa_assign_levels_rows(scores, batch, hq, hkv, n_q, n_k, mode, taus, counts, n_cuts, caps,
                                causal, b_q, b_k, levels, nullptr, level_map, plan_csr, plan_info,
                                level_counts, stream);
}

// qblk (optional, device int32 [n_q]): score row i of every head is query block qblk[i] of the
// head, for the causal pre-pass (the q-block work units of the multi-GPU partition).
extern "C" int psa_assign_levels_rows(const double* scores, int64_t batch, int hq, int hkv,
                                      int n_q, int n_k, int mode, const double* taus,
                                      const int32_t* counts, int n_cuts, const int8_t* caps,
                                      int causal, int b_q, int b_k, int levels,
                                      const int32_t* qblk, int8_t* level_map, uint16_t* plan_csr,
                                      int32_t* plan_info, unsigned long long* level_counts,
                                      void* stream) {
  PSA_CHECK_ARG(scores && level_map && plan_csr && plan_info, "null pointer argument");
  PSA_CHECK_ARG(mode == 0 || mode == 1, "mode must be 0 (threshold) or 1 (quantile)");
  PSA_CHECK_ARG(n_cuts >= 1 && n_cuts <= kMaxCuts, "need 1..16 thresholds/cutpoints");
  PSA_CHECK_ARG(n_cuts <= levels, "more thresholds than pyramid levels");
  PSA_CHECK_ARG(levels >= 1 && levels <= 15, "levels must lie in 1..15");
  PSA_CHECK_ARG(n_k >= 1 && n_k <= 4096, "n_k must lie in 1..4096");
  PSA_CHECK_ARG(n_q >= 1, "n_q must be positive");
  PSA_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0, "query heads must be a multiple of kv heads");
  AssignParams p{};
  p.rule.mode = mode;
  p.rule.n_cuts = n_cuts;
  for (int c = 0; c < n_cuts; ++c) {
    if (mode == 0) {
      PSA_CHECK_ARG(taus != nullptr, "threshold mode needs taus");
      p.rule.taus[c] = taus[c];
    } else {
      PSA_CHECK_ARG(counts != nullptr, "quantile mode needs counts");
      p.rule.counts[c] = counts[c];
    }
  }
  p.n_q = n_q;
  p.n_k = n_k;
  p.hq = hq;
  p.hkv = hkv;
  p.b_q = b_q;
  p.b_k = b_k;
  p.levels = levels;
  p.causal = causal;
  p.qblk = qblk;
  static const int kIpt[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32};
  int ipt = 32;
  for (int v : kIpt)
    if (128 * v >= n_k) {
      ipt = v;
      break;
    }
  const int n_pad = 128 * ipt;
  p.n_pad = n_pad;
  const size_t smem = static_cast<size_t>(n_pad) * 14 + 16 + static_cast<size_t>(n_pad) * 8;
  dim3 grid(n_q, static_cast<unsigned>(batch * hq));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto launch = [&](auto kern) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    kern<<<grid, 128, smem, st>>>(scores, caps, p, level_map, plan_csr, plan_info, level_counts);
  };
  switch (ipt) {
    case 1: launch(assign_levels_kernel<1>); break;
    case 2: launch(assign_levels_kernel<2>); break;
    case 3: launch(assign_levels_kernel<3>); break;
    case 4: launch(assign_levels_kernel<4>); break;
    case 5: launch(assign_levels_kernel<5>); break;
    case 6: launch(assign_levels_kernel<6>); break;
    case 8: launch(assign_levels_kernel<8>); break;
    case 10: launch(assign_levels_kernel<10>); break;
    case 12: launch(assign_levels_kernel<12>); break;
    case 16: launch(assign_levels_kernel<16>); break;
    case 20: launch(assign_levels_kernel<20>); break;
    case 24: launch(assign_levels_kernel<24>); break;
    default: launch(assign_levels_kernel<32>); break;
  }
  return psa_check_launch("assign_levels_kernel");
}

extern "C" int psa_mask_to_plan(const void* mask, int mask_is_int64, int64_t units, int n_q,
                                int n_k, int causal, int b_q, int b_k, int levels,
                                uint16_t* plan_csr, int32_t* plan_info,
                                unsigned long long* level_counts, int32_t* bad_flag,
                                void* stream) {
  PSA_CHECK_ARG(mask && plan_csr && plan_info && bad_flag, "null pointer argument");
  PSA_CHECK_ARG(n_k >= 1 && n_k <= 4096, "n_k must lie in 1..4096");
  PSA_CHECK_ARG(levels >= 1 && levels <= 15, "levels must lie in 1..15");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = static_cast<size_t>(n_k) + 16;
  if (mask_is_int64)
    mask_to_plan_kernel<long long><<<static_cast<unsigned>(units), 128, smem, s>>>(
        static_cast<const long long*>(mask), n_q, n_k, causal, b_q, b_k, levels, plan_csr,
        plan_info, level_counts, bad_flag);
  else
    mask_to_plan_kernel<int8_t><<<static_cast<unsigned>(units), 128, smem, s>>>(
        static_cast<const int8_t*>(mask), n_q, n_k, causal, b_q, b_k, levels, plan_csr,
        plan_info, level_counts, bad_flag);
  return psa_check_launch("mask_to_plan_kernel");
}
