// K4: multi-level block-sparse attention forward on sm_100a (tcgen05 + TMEM + TMA).
//
// Reference semantics:
//   psa_streaming        pkg/src/pyrattn/attention.py:171-218  (online softmax over the selected
//                        (j, h) pairs; logits q.k*scale + (h-1)*ln2; empty rows -> 0, lse -inf)
//   level_bias           pkg/src/pyrattn/attention.py:39-44
//   _causal_key_mask     pkg/src/pyrattn/attention.py:88-108 (k_pos <= q_pos on straddling pairs)
//   execute_schedule     pkg/src/pyrattn/scheduler.py:203-269 (decoupled block tiles: pooled
//                        segments of several KV blocks packed into one fixed-size tile)
//
// One CTA per (head, query block) work unit; 12 warps:
//   warp 0  TMA producer: walks the unit's level-major plan and packs pooled segments into
//           128-row KV tiles. Segment sizes are padded to power-of-two slots (>= 8 rows) and
//           emitted largest-first, so every slot starts on a 1024-byte (8-row) swizzle atom and
//           the packing is perfect except for the last tile. Per 8-column chunk it publishes
//           (valid rows, level bias, causal flag, key position) through a 4-deep meta ring.
//           K and V have separate rings (K: 3 stages, freed when S = QK^T completes;
//           V: 2 stages, freed when O += PV completes).
//   warp 1  MMA issuer (one thread): S[sb] = Q K^T into TMEM (double-buffered), then
//           O += P V with P from shared memory; commits signal the other roles.
//   warp 2  TMEM allocator (512 columns: S0 | S1 | O).
//   warps 4-11  softmax + epilogue: two warpgroups, one TMEM lane (query row) per thread;
//           warpgroup g owns S columns [64g, 64g+64) and O columns [D/2 g, D/2 (g+1)), so every
//           SM sub-partition runs two softmax warps. Per tile the two halves exchange their row
//           max through shared memory (one named barrier). log2-domain online softmax with the
//           level bias exactly (h-1) in log2 units, packed f32x2 FMA/ADD, lazy O rescaling (only
//           when the running max grows by more than 2^8), P written as bf16 into a 128B-swizzled
//           K-major tile, final 1/l normalisation and lse.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "psa_internal.h"

namespace psa {

constexpr int kTileRows = 128;  // query rows per tile (MMA M) and KV rows per tile (MMA N)
constexpr int kChunks = kTileRows / 8;
constexpr int kMetaRing = 4;
constexpr int kSoftmaxWarps = 8;
constexpr int kSoftmaxThreads = kSoftmaxWarps * 32;
constexpr int kAttnThreads = 4 * 32 + kSoftmaxThreads;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kPolyFrom = 48;  // softmax columns [48, 64) of each warp use the FMA-pipe exp2
// TMEM columns: S0 | S1 | O (D) | P (64 packed bf16x2 columns)
constexpr uint32_t kTmemS = 0, kTmemO = 256, kTmemP = 384;

template <int D>
struct AttnCfg {
  static constexpr int kKStages = D == 128 ? 3 : 4;
  static constexpr int kVStages = D == 128 ? 2 : 4;
  static constexpr int kTileBytes = kTileRows * D * 2;  // one K or V tile
};

struct AttnMaps {
  CUtensorMap q;
  CUtensorMap k[kMaxLevels];
  CUtensorMap v[kMaxLevels];
};

struct AttnParams {
  int64_t n;
  int hq, hkv, b_q, b_k, levels, n_q, n_k, causal;
  float scale_log2;
  const int64_t* out_rows;  // optional scatter: O/lse row i of a head goes to row out_rows[i]
};

template <int D>
struct AttnSmem {
  using C = AttnCfg<D>;
  uint8_t q[kTileRows * D * 2];                   // [D/64][128 rows][128 B]
  uint8_t k[C::kKStages][C::kTileBytes];          // [D/64][128 rows][128 B]
  uint8_t v[C::kVStages][C::kTileBytes];
  float bias[kMetaRing][kTileRows];               // per KV column: level-1 (log2) or -inf
  uint32_t meta[kMetaRing][kChunks];              // causal: key position | straddle flag
  float red[2][2][kTileRows];                     // [tile parity][warpgroup][row]
  uint64_t q_full;
  uint64_t k_full[C::kKStages], k_empty[C::kKStages];
  uint64_t v_full[C::kVStages], v_empty[C::kVStages];
  uint64_t meta_full[kMetaRing], meta_empty[kMetaRing];
  uint64_t s_full[2], s_free[2], p_full, o_done;
  uint32_t tmem_base;
};

// Tile packing shared by the K and V producer warps: lane l (< 16) owns plan entry e + l; a
// warp inclusive scan of the slot sizes gives each segment's row offset in the tile, and the
// lanes whose running total fits in 128 rows form the tile.
struct TileSeg {
  int j, h, L, sz, off, row, total, nseg;
  bool fits;
};

struct PlanCursor {
  const uint16_t* plan;
  int n_ent, e, base;
  uint32_t cur, nxt;
  PSA_DEV void init(const uint16_t* pl, int n, int lane) {
    plan = pl;
    n_ent = n;
    e = 0;
    base = 0;
    cur = lane < n ? plan[lane] : 0u;
    nxt = 32 + lane < n ? plan[32 + lane] : 0u;
  }
  PSA_DEV TileSeg next(const AttnParams& p, int64_t bhkv, int lane) {
    TileSeg s;
    const int rel = e - base + lane;
    const uint32_t a = __shfl_sync(0xffffffffu, cur, rel & 31);
    const uint32_t b = __shfl_sync(0xffffffffu, nxt, rel & 31);
    const uint32_t ent = rel < 32 ? a : b;
    const bool valid = lane < kChunks && e + lane < n_ent;
    s.j = static_cast<int>(ent & 0xFFFu);
    s.h = valid ? static_cast<int>(ent >> 12) : 1;
    s.L = valid ? (p.b_k >> (s.h - 1)) : 0;
    s.sz = 256;  // never fits: keeps the fitting lanes a prefix
    if (valid) s.sz = s.L <= 8 ? 8 : (1 << (32 - __clz(s.L - 1)));
    int incl = s.sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    s.fits = incl <= kTileRows;
    s.nseg = __popc(__ballot_sync(0xffffffffu, s.fits));
    s.total = __shfl_sync(0xffffffffu, incl, s.nseg - 1);
    s.off = incl - s.sz;
    s.row = static_cast<int>(bhkv) * static_cast<int>(p.n >> (s.h - 1)) + s.j * s.L;
    e += s.nseg;
    if (e - base >= 32) {  // advance the two-window cache (warp-uniform)
      base += 32;
      cur = nxt;
      nxt = base + 32 + lane < n_ent ? plan[base + 32 + lane] : 0u;
    }
    return s;
  }
};

template <int D>
__global__ void __launch_bounds__(kAttnThreads, 1)
    psa_attn_fwd_kernel(const __grid_constant__ AttnMaps maps, const AttnParams p,
                        const uint16_t* __restrict__ csr, const int32_t* __restrict__ info,
                        uint16_t* __restrict__ out, float* __restrict__ lse,
                        int32_t* __restrict__ skipped) {
  using C = AttnCfg<D>;
  constexpr int KST = C::kKStages, VST = C::kVStages;
  constexpr int OC = D / 2;  // O columns per softmax warpgroup
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<AttnSmem<D>*>(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = blockIdx.x;
  const int bhq = static_cast<int>(unit / p.n_q);
  const int i = static_cast<int>(unit % p.n_q);
  const int b = bhq / p.hq, hh = bhq % p.hq;
  const int64_t bhkv = static_cast<int64_t>(b) * p.hkv + hh / (p.hq / p.hkv);
  const int n_ent = info[unit * 2 + 0];
  const int T = (info[unit * 2 + 1] + kTileRows - 1) / kTileRows;  // 128-row KV tiles
  const int64_t q_row0 = static_cast<int64_t>(bhq) * p.n + static_cast<int64_t>(i) * p.b_q;

  // ---------------------------------------------------------------- setup
  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();  // 128B-swizzle atoms need 1024-B alignment
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int s = 0; s < kMetaRing; ++s) {
      mbar_init(&sm.meta_full[s], 1);
      mbar_init(&sm.meta_empty[s], kSoftmaxThreads);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_free[s], kSoftmaxThreads);
    }
    mbar_init(&sm.p_full, kSoftmaxWarps);
    mbar_init(&sm.o_done, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    for (int h = 0; h < p.levels; ++h) {
      tma_prefetch_desc(&maps.k[h]);
      tma_prefetch_desc(&maps.v[h]);
    }
  }
  if (warp == 2) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  {  // K/V rows past the last filled slot of a tile are read by the MMA: keep them finite
    uint4* z = reinterpret_cast<uint4*>(&sm.k[0][0]);
    const int nvec = (KST + VST) * C::kTileBytes / 16;
    for (int t = threadIdx.x; t < nvec; t += kAttnThreads) z[t] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ================================================================ K producer (+ Q)
    if (T > 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&sm.q_full, kTileRows * D * 2);
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(&maps.q, &sm.q_full, sm.q + c * kTileRows * 128, c * 64,
                      static_cast<int>(q_row0));
      }
      PlanCursor pc;
      pc.init(csr + unit * p.n_k, n_ent, lane);
      for (int t = 0; t < T; ++t) {
        const int ks = t % KST;
        const TileSeg s = pc.next(p, bhkv, lane);
        if (t >= KST) mbar_wait(&sm.k_empty[ks], ((t / KST) - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&sm.k_full[ks], static_cast<uint32_t>(s.total) * D * 2);
        __syncwarp();
        if (s.fits)
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(&maps.k[s.h - 1], &sm.k_full[ks],
                        sm.k[ks] + c * kTileRows * 128 + s.off * 128, c * 64, s.row);
      }
    }
  } else if (warp == 2) {
    // ================================================================ bias/meta producer
    // per KV column: level-1 (log2 units) or -inf on pad rows; causal: straddle flag + key pos
    if (T > 0) {
      const int64_t q_lo = static_cast<int64_t>(i) * p.b_q;
      PlanCursor pc;
      pc.init(csr + unit * p.n_k, n_ent, lane);
      for (int t = 0; t < T; ++t) {
        const int ms = t % kMetaRing;
        const TileSeg s = pc.next(p, bhkv, lane);
        if (t >= kMetaRing) mbar_wait(&sm.meta_empty[ms], ((t / kMetaRing) - 1) & 1);
        {  // lane l fills columns [4l, 4l+4): find the owning segment (offsets ascend)
          int g = 0;
          for (int q = 1; q < s.nseg; ++q)
            if (__shfl_sync(0xffffffffu, s.off, q) <= 4 * lane) g = q;
          const int goff = __shfl_sync(0xffffffffu, s.off, g);
          const int gL = __shfl_sync(0xffffffffu, s.L, g);
          const int gh = __shfl_sync(0xffffffffu, s.h, g);
          const int r0 = 4 * lane - goff;  // row of column 4l inside its segment slot
          const float bv = static_cast<float>(gh - 1);
          float4 w = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
          if (4 * lane < s.total) {
            w.x = r0 + 0 < gL ? bv : -INFINITY;
            w.y = r0 + 1 < gL ? bv : -INFINITY;
            w.z = r0 + 2 < gL ? bv : -INFINITY;
            w.w = r0 + 3 < gL ? bv : -INFINITY;
          }
          *reinterpret_cast<float4*>(&sm.bias[ms][4 * lane]) = w;
        }
        if (p.causal && s.fits) {
          const bool straddle = static_cast<int64_t>(s.j + 1) * p.b_k - 1 > q_lo;
          for (int c = 0; c < s.sz / 8; ++c)
            sm.meta[ms][s.off / 8 + c] =
                (straddle ? 1u : 0u) | (static_cast<uint32_t>(s.j * p.b_k + c * 8) << 1);
        }
        if (p.causal && lane < kChunks && 8 * lane >= s.total) sm.meta[ms][lane] = 0u;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.meta_full[ms]);
      }
    }
  } else if (warp == 3) {
    // ================================================================ V producer
    if (T > 0) {
      PlanCursor pc;
      pc.init(csr + unit * p.n_k, n_ent, lane);
      for (int t = 0; t < T; ++t) {
        const int vs = t % VST;
        const TileSeg s = pc.next(p, bhkv, lane);
        if (t >= VST) mbar_wait(&sm.v_empty[vs], ((t / VST) - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&sm.v_full[vs], static_cast<uint32_t>(s.total) * D * 2);
        __syncwarp();
        if (s.fits)
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(&maps.v[s.h - 1], &sm.v_full[vs],
                        sm.v[vs] + c * kTileRows * 128 + s.off * 128, c * 64, s.row);
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    // warp-uniform loop; one elected lane issues the tcgen05 instructions
    if (T > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
      const uint64_t q_desc0 = umma_desc_sw128(smem_u32(sm.q), 16, 1024);
      auto issue_pv = [&](int u) {
        const int vs = u % VST;
        mbar_wait(&sm.v_full[vs], (u / VST) & 1);
        mbar_wait(&sm.p_full, u & 1);
        tc_fence_after();
        const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sm.v[vs]), kTileRows * 128, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kTileRows / 16; ++kk)
            mma_bf16_ts(tmem + kTmemO, tmem + kTmemP + kk * 8, v_desc0 + ((kk * 16 * 128) >> 4),
                        idesc_o, (u > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&sm.v_empty[vs]);
          mma_commit(&sm.o_done);
        }
        __syncwarp();
      };
      mbar_wait(&sm.q_full, 0);
      tc_fence_after();
      for (int t = 0; t < T; ++t) {
        const int ks = t % KST, sb = t & 1;
        mbar_wait(&sm.k_full[ks], (t / KST) & 1);
        if (t >= 2) mbar_wait(&sm.s_free[sb], ((t >> 1) - 1) & 1);
        tc_fence_after();
        const uint64_t k_desc0 = umma_desc_sw128(smem_u32(sm.k[ks]), 16, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
            mma_bf16_ss(tmem + kTmemS + sb * 128, q_desc0 + koff, k_desc0 + koff, idesc_s,
                        kk > 0 ? 1u : 0u);
          }
          mma_commit(&sm.k_empty[ks]);
          mma_commit(&sm.s_full[sb]);
        }
        __syncwarp();
        if (t >= 1) issue_pv(t - 1);
      }
      issue_pv(T - 1);
    }
  } else if (warp >= 4) {
    // ================================================================ softmax + epilogue
    const int wg = (warp - 4) >> 2;  // warpgroup: S columns [64 wg, 64 wg + 64)
    const int wq = warp & 3;         // TMEM lane quarter
    const int row = wq * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int qpos = i * p.b_q + row;
    const float2 scale2 = make_float2(p.scale_log2, p.scale_log2);
    float m_run = -INFINITY, l_run = 0.f;
    for (int t = 0; t < T; ++t) {
      const int sb = t & 1, ms = t % kMetaRing;
      mbar_wait(&sm.s_full[sb], (t >> 1) & 1);
      tc_fence_after();
      uint32_t s[2][32];
      tmem_ld32(t_lane + kTmemS + sb * 128 + wg * 64, s[0]);
      tmem_ld32(t_lane + kTmemS + sb * 128 + wg * 64 + 32, s[1]);
      tmem_ld_wait(s[0]);
      tmem_ld_wait(s[1]);
      tc_fence_before();
      mbar_arrive(&sm.s_free[sb]);

      // y = s * scale + bias_col  (bias: level-1 in log2 units; -inf on pad columns)
      mbar_wait(&sm.meta_full[ms], (t / kMetaRing) & 1);
      float y[64];
      const float4* bias4 = reinterpret_cast<const float4*>(&sm.bias[ms][wg * 64]);
#pragma unroll
      for (int q4 = 0; q4 < 16; ++q4) {
        const float4 bv = bias4[q4];
        const float* x = reinterpret_cast<const float*>(&s[q4 >> 3][(q4 & 7) * 4]);
        const float2 a = ffma2(make_float2(x[0], x[1]), scale2, make_float2(bv.x, bv.y));
        const float2 c = ffma2(make_float2(x[2], x[3]), scale2, make_float2(bv.z, bv.w));
        y[q4 * 4 + 0] = a.x;
        y[q4 * 4 + 1] = a.y;
        y[q4 * 4 + 2] = c.x;
        y[q4 * 4 + 3] = c.y;
      }
      if (p.causal) {  // token-level mask on straddling level-1 chunks (attention.py:88-108)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t w = sm.meta[ms][wg * 8 + c];
          if (w & 1u) {
            const int lim = qpos - static_cast<int>(w >> 1);  // key k visible iff k <= lim
#pragma unroll
            for (int e = 0; e < 8; ++e) y[c * 8 + e] = (e <= lim) ? y[c * 8 + e] : -INFINITY;
          }
        }
      }
      mbar_arrive(&sm.meta_empty[ms]);

      float mx0 = fmax3(y[0], y[1], y[2]), mx1 = fmax3(y[3], y[4], y[5]);
      float mx2 = fmax3(y[6], y[7], y[8]), mx3 = fmax3(y[9], y[10], y[11]);
#pragma unroll
      for (int e = 12; e < 60; e += 8) {
        mx0 = fmax3(mx0, y[e], y[e + 1]);
        mx1 = fmax3(mx1, y[e + 2], y[e + 3]);
        mx2 = fmax3(mx2, y[e + 4], y[e + 5]);
        mx3 = fmax3(mx3, y[e + 6], y[e + 7]);
      }
      mx0 = fmax3(mx0, y[60], y[61]);
      mx1 = fmax3(mx1, y[62], y[63]);
      float mt = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      sm.red[t & 1][wg][row] = mt;
      named_bar_sync(1, kSoftmaxThreads);
      mt = fmaxf(sm.red[t & 1][0][row], sm.red[t & 1][1][row]);

      const float m_new = fmaxf(m_run, mt);
      const bool resc = m_new > m_run + kRescaleThreshold;
      float alpha = 1.f;
      if (resc) {
        alpha = ex2_approx(m_run - m_new);
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      const float2 negm = make_float2(-m_use, -m_use);
      float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 64; e += 4) {
        float2 a = fadd2(make_float2(y[e], y[e + 1]), negm);
        float2 c = fadd2(make_float2(y[e + 2], y[e + 3]), negm);
        if (e >= kPolyFrom) {  // last quarter of the columns on the FMA pipe (MUFU offload)
          a = ex2_poly2(a);
          c = ex2_poly2(c);
        } else {
          a.x = ex2_approx(a.x);
          a.y = ex2_approx(a.y);
          c.x = ex2_approx(c.x);
          c.y = ex2_approx(c.y);
        }
        ls0 = fadd2(ls0, a);
        ls1 = fadd2(ls1, c);
        pk[e / 2] = pack_bf16x2(a.x, a.y);
        pk[e / 2 + 1] = pack_bf16x2(c.x, c.y);
      }
      const float2 ls = fadd2(ls0, ls1);
      l_run = l_run * alpha + (ls.x + ls.y);

      const bool need = (t > 0) && __any_sync(0xffffffffu, resc);
      if (t > 0) mbar_wait(&sm.o_done, (t - 1) & 1);  // PV(t-1) done: P columns free, O stable
      tc_fence_after();
      if (need) {
#pragma unroll
        for (int c4 = 0; c4 < OC / 32; ++c4) {
          uint32_t o[32];
          tmem_ld32(t_lane + kTmemO + wg * OC + c4 * 32, o);
          tmem_ld_wait(o);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tmem_st32(t_lane + kTmemO + wg * OC + c4 * 32, o);
        }
      }
      tmem_st32(t_lane + kTmemP + wg * 32, pk);  // P row half: keys [64 wg, 64 wg + 64)
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full);
    }

    // ---------------------------------------------------------------- epilogue
    named_bar_sync(1, kSoftmaxThreads);  // both halves finished reading red[]
    sm.red[0][wg][row] = l_run;
    named_bar_sync(1, kSoftmaxThreads);
    const float l_tot = sm.red[0][0][row] + sm.red[0][1][row];
    if (T > 0) {
      mbar_wait(&sm.o_done, (T - 1) & 1);
      tc_fence_after();
    }
    const bool valid = row < p.b_q;
    const bool alive = l_tot > 0.f;
    const float inv = alive ? 1.f / l_tot : 0.f;
    uint16_t* orow = out + (q_row0 + row) * D + wg * OC;
#pragma unroll
    for (int c4 = 0; c4 < OC / 32; ++c4) {
      uint32_t o[32];
      if (T > 0) {
        tmem_ld32(t_lane + kTmemO + wg * OC + c4 * 32, o);
        tmem_ld_wait(o);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0u;
      }
      uint32_t pkd[16];
#pragma unroll
      for (int e = 0; e < 16; ++e)
        pkd[e] = pack_bf16x2(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
      if (valid) {
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4)
          *reinterpret_cast<uint4*>(orow + c4 * 32 + v4 * 8) =
              make_uint4(pkd[v4 * 4], pkd[v4 * 4 + 1], pkd[v4 * 4 + 2], pkd[v4 * 4 + 3]);
      }
    }
    if (wg == 0) {
      if (valid)
        lse[q_row0 + row] = alive ? (m_run + log2f(l_tot)) * 0.69314718055994530942f : -INFINITY;
      const unsigned dead = __ballot_sync(0xffffffffu, valid && !alive);
      if (lane == 0 && dead) atomicAdd(skipped, __popc(dead));
    }
  }

  // ---------------------------------------------------------------- teardown
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ====================================================================== ping-pong kernel
// Same work unit, plan walk, producers and numerics as psa_attn_fwd_kernel, but the two
// softmax warpgroups are independent "lanes" that take ALTERNATE KV tiles of the unit, each
// with full 128-column rows, its own running (max, sum) and its own O accumulator in TMEM;
// the lanes merge once in the epilogue. While one lane runs its softmax, the tensor core
// computes the other lane's S and PV, so neither waits for the other (the v1 kernel's two
// warpgroups split one tile's columns and synchronised on every tile). P is written back into
// the lane's S columns (tcgen05 MMAs from one CTA execute in issue order, so S(t+2) cannot
// overwrite P(t) before PV(t) has read it). TMEM: S0 | S1 | O0 | O1 (512 columns at D=128).
// Register split via setmaxnreg within the CTA pool of 384 x 168: producer/MMA warpgroup 64,
// softmax warpgroups 216 (128*64 + 256*216 <= 384*168, else the increase never completes).
constexpr int kPPThreads = 384;
constexpr int kPPPolyFrom = 96;  // columns [96, 128) of a row use the FMA-pipe exp2

template <int D>
struct PPSmem {
  using C = AttnCfg<D>;
  uint8_t q[kTileRows * D * 2];
  uint8_t k[C::kKStages][C::kTileBytes];
  uint8_t v[C::kVStages][C::kTileBytes];
  float bias[kMetaRing][kTileRows];
  uint32_t meta[kMetaRing][kChunks];
  float red_m[2][kTileRows], red_l[2][kTileRows];
  uint64_t q_full;
  uint64_t k_full[C::kKStages], k_empty[C::kKStages];
  uint64_t v_full[C::kVStages], v_empty[C::kVStages];
  uint64_t meta_full[kMetaRing], meta_empty[kMetaRing];
  uint64_t s_full[2], p_full[2], o_done[2];
  uint32_t tmem_base;
};

template <uint32_t N>
PSA_DEV void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }
template <uint32_t N>
PSA_DEV void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }

template <int D, int POLY_FROM = kPPPolyFrom>
__global__ void __launch_bounds__(kPPThreads, 1)
    psa_attn_pp_kernel(const __grid_constant__ AttnMaps maps, const AttnParams p,
                       const uint16_t* __restrict__ csr, const int32_t* __restrict__ info,
                       uint16_t* __restrict__ out, float* __restrict__ lse,
                       int32_t* __restrict__ skipped) {
  using C = AttnCfg<D>;
  constexpr int KST = C::kKStages, VST = C::kVStages;
  constexpr uint32_t kO0 = 256;  // O_L at kO0 + L * D
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<PPSmem<D>*>(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = blockIdx.x;
  const int bhq = static_cast<int>(unit / p.n_q);
  const int i = static_cast<int>(unit % p.n_q);
  const int b = bhq / p.hq, hh = bhq % p.hq;
  const int64_t bhkv = static_cast<int64_t>(b) * p.hkv + hh / (p.hq / p.hkv);
  const int n_ent = info[unit * 2 + 0];
  const int T = (info[unit * 2 + 1] + kTileRows - 1) / kTileRows;  // 128-row KV tiles
  const int64_t q_row0 = static_cast<int64_t>(bhq) * p.n + static_cast<int64_t>(i) * p.b_q;

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int s = 0; s < kMetaRing; ++s) {
      mbar_init(&sm.meta_full[s], 1);
      mbar_init(&sm.meta_empty[s], kTileRows);  // one lane (128 threads) consumes a tile
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.p_full[s], 4);  // one arrive per warp of the lane
      mbar_init(&sm.o_done[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    for (int h = 0; h < p.levels; ++h) {
      tma_prefetch_desc(&maps.k[h]);
      tma_prefetch_desc(&maps.v[h]);
    }
  }
  if (warp == 2) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  {  // K/V rows past the last filled slot of a tile are read by the MMA: keep them finite
    uint4* z = reinterpret_cast<uint4*>(&sm.k[0][0]);
    const int nvec = (KST + VST) * C::kTileBytes / 16;
    for (int t = threadIdx.x; t < nvec; t += kPPThreads) z[t] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    regs_dec<64>();
    if (warp == 0) {
      // ============================================================ K producer (+ Q)
      if (T > 0) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm.q_full, kTileRows * D * 2);
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(&maps.q, &sm.q_full, sm.q + c * kTileRows * 128, c * 64,
                        static_cast<int>(q_row0));
        }
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int ks = t % KST;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= KST) mbar_wait(&sm.k_empty[ks], ((t / KST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.k_full[ks], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.k[sg.h - 1], &sm.k_full[ks],
                          sm.k[ks] + c * kTileRows * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 3) {
      // ============================================================ V producer
      if (T > 0) {
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int vs = t % VST;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= VST) mbar_wait(&sm.v_empty[vs], ((t / VST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.v_full[vs], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.v[sg.h - 1], &sm.v_full[vs],
                          sm.v[vs] + c * kTileRows * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 2) {
      // ============================================================ bias/meta producer
      if (T > 0) {
        const int64_t q_lo = static_cast<int64_t>(i) * p.b_q;
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int ms = t % kMetaRing;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= kMetaRing) mbar_wait(&sm.meta_empty[ms], ((t / kMetaRing) - 1) & 1);
          {
            int g = 0;
            for (int q = 1; q < sg.nseg; ++q)
              if (__shfl_sync(0xffffffffu, sg.off, q) <= 4 * lane) g = q;
            const int goff = __shfl_sync(0xffffffffu, sg.off, g);
            const int gL = __shfl_sync(0xffffffffu, sg.L, g);
            const int gh = __shfl_sync(0xffffffffu, sg.h, g);
            const int r0 = 4 * lane - goff;
            const float bv = static_cast<float>(gh - 1);
            float4 w = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            if (4 * lane < sg.total) {
              w.x = r0 + 0 < gL ? bv : -INFINITY;
              w.y = r0 + 1 < gL ? bv : -INFINITY;
              w.z = r0 + 2 < gL ? bv : -INFINITY;
              w.w = r0 + 3 < gL ? bv : -INFINITY;
            }
            *reinterpret_cast<float4*>(&sm.bias[ms][4 * lane]) = w;
          }
          if (p.causal && sg.fits) {
            const bool straddle = static_cast<int64_t>(sg.j + 1) * p.b_k - 1 > q_lo;
            for (int c = 0; c < sg.sz / 8; ++c)
              sm.meta[ms][sg.off / 8 + c] =
                  (straddle ? 1u : 0u) | (static_cast<uint32_t>(sg.j * p.b_k + c * 8) << 1);
          }
          if (p.causal && lane < kChunks && 8 * lane >= sg.total) sm.meta[ms][lane] = 0u;
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.meta_full[ms]);
        }
      }
    } else {
      // ============================================================ MMA issuer (warp 1)
      if (T > 0) {
        constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
        const uint64_t q_desc0 = umma_desc_sw128(smem_u32(sm.q), 16, 1024);
        auto issue_s = [&](int t) {
          const int ks = t % KST, L = t & 1;
          mbar_wait(&sm.k_full[ks], (t / KST) & 1);
          tc_fence_after();
          const uint64_t k_desc0 = umma_desc_sw128(smem_u32(sm.k[ks]), 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ss(tmem + L * 128, q_desc0 + koff, k_desc0 + koff, idesc_s,
                          kk > 0 ? 1u : 0u);
            }
            mma_commit(&sm.k_empty[ks]);
            mma_commit(&sm.s_full[L]);
          }
          __syncwarp();
        };
        auto issue_pv = [&](int t) {
          const int vs = t % VST, L = t & 1;
          mbar_wait(&sm.v_full[vs], (t / VST) & 1);
          mbar_wait(&sm.p_full[L], (t >> 1) & 1);
          tc_fence_after();
          const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sm.v[vs]), kTileRows * 128, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kTileRows / 16; ++kk)
              mma_bf16_ts(tmem + kO0 + L * D, tmem + L * 128 + kk * 8,
                          v_desc0 + ((kk * 16 * 128) >> 4), idesc_o,
                          (t >= 2 || kk > 0) ? 1u : 0u);
            mma_commit(&sm.v_empty[vs]);
            mma_commit(&sm.o_done[L]);
          }
          __syncwarp();
        };
        mbar_wait(&sm.q_full, 0);
        tc_fence_after();
        issue_s(0);
        if (T > 1) issue_s(1);
        issue_pv(0);
        for (int t = 2; t < T; ++t) {
          issue_s(t);       // program order after PV(t-2): S(t) may overwrite P(t-2)
          issue_pv(t - 1);
        }
        if (T > 1) issue_pv(T - 1);
      }
    }
  } else {
    regs_inc<216>();
    // ============================================================== softmax lanes
    const int L = (warp - 4) >> 2;  // lane L takes KV tiles t = L, L + 2, ...
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const uint32_t t_s = t_lane + L * 128;
    const int qpos = i * p.b_q + row;
    const float2 scale2 = make_float2(p.scale_log2, p.scale_log2);
    float m_run = -INFINITY, l_run = 0.f;
    for (int t = L; t < T; t += 2) {
      const int ms = t % kMetaRing;
      mbar_wait(&sm.s_full[L], (t >> 1) & 1);
      tc_fence_after();
      uint32_t s[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(t_s + c * 32, s[c]);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_wait(s[c]);
      // y = s * scale + bias_col (bias: level-1 in log2 units; -inf on pad columns)
      mbar_wait(&sm.meta_full[ms], (t / kMetaRing) & 1);
      float y[128];
      const float4* bias4 = reinterpret_cast<const float4*>(&sm.bias[ms][0]);
#pragma unroll
      for (int q4 = 0; q4 < 32; ++q4) {
        const float4 bv = bias4[q4];
        const float* x = reinterpret_cast<const float*>(&s[q4 >> 3][(q4 & 7) * 4]);
        const float2 a = ffma2(make_float2(x[0], x[1]), scale2, make_float2(bv.x, bv.y));
        const float2 c = ffma2(make_float2(x[2], x[3]), scale2, make_float2(bv.z, bv.w));
        y[q4 * 4 + 0] = a.x;
        y[q4 * 4 + 1] = a.y;
        y[q4 * 4 + 2] = c.x;
        y[q4 * 4 + 3] = c.y;
      }
      if (p.causal) {  // token-level mask on straddling level-1 chunks (attention.py:88-108)
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          const uint32_t w = sm.meta[ms][c];
          if (w & 1u) {
            const int lim = qpos - static_cast<int>(w >> 1);
#pragma unroll
            for (int e = 0; e < 8; ++e) y[c * 8 + e] = (e <= lim) ? y[c * 8 + e] : -INFINITY;
          }
        }
      }
      mbar_arrive(&sm.meta_empty[ms]);

      float mx[4] = {fmax3(y[0], y[1], y[2]), fmax3(y[3], y[4], y[5]), fmax3(y[6], y[7], y[8]),
                     fmax3(y[9], y[10], y[11])};
#pragma unroll
      for (int e = 12; e < 124; e += 8) {
        mx[0] = fmax3(mx[0], y[e], y[e + 1]);
        mx[1] = fmax3(mx[1], y[e + 2], y[e + 3]);
        mx[2] = fmax3(mx[2], y[e + 4], y[e + 5]);
        mx[3] = fmax3(mx[3], y[e + 6], y[e + 7]);
      }
      mx[0] = fmax3(mx[0], y[124], y[125]);
      mx[1] = fmax3(mx[1], y[126], y[127]);
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      const float m_new = fmaxf(m_run, mt);
      const bool resc = m_new > m_run + kRescaleThreshold;
      float alpha = 1.f;
      if (resc) {
        alpha = ex2_approx(m_run - m_new);
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      const float2 negm = make_float2(-m_use, -m_use);
      float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
      uint32_t pk[64];
#pragma unroll
      for (int e = 0; e < 128; e += 4) {
        float2 a = fadd2(make_float2(y[e], y[e + 1]), negm);
        float2 c = fadd2(make_float2(y[e + 2], y[e + 3]), negm);
        if (e >= POLY_FROM) {
          a = ex2_poly2(a);
          c = ex2_poly2(c);
        } else {
          a.x = ex2_approx(a.x);
          a.y = ex2_approx(a.y);
          c.x = ex2_approx(c.x);
          c.y = ex2_approx(c.y);
        }
        ls0 = fadd2(ls0, a);
        ls1 = fadd2(ls1, c);
        pk[e / 2] = pack_bf16x2(a.x, a.y);
        pk[e / 2 + 1] = pack_bf16x2(c.x, c.y);
      }
      const float2 ls = fadd2(ls0, ls1);
      l_run = l_run * alpha + (ls.x + ls.y);
      // S(t) complete => PV(t-2) of this lane complete (in-order tensor pipe): O is stable
      if (t >= 2 && __any_sync(0xffffffffu, resc)) {
#pragma unroll
        for (int c4 = 0; c4 < D / 32; ++c4) {
          uint32_t o[32];
          tmem_ld32(t_lane + kO0 + L * D + c4 * 32, o);
          tmem_ld_wait(o);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tmem_st32(t_lane + kO0 + L * D + c4 * 32, o);
        }
      }
      {  // P (bf16 pairs) into this lane's S columns [0, 64)
        uint32_t (&p0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&pk[0]);
        uint32_t (&p1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&pk[32]);
        tmem_st32(t_s, p0);
        tmem_st32(t_s + 32, p1);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full[L]);
    }

    // ---------------------------------------------------------------- merge + epilogue
    const int cnt0 = (T + 1) >> 1, cnt1 = T >> 1;  // tiles of lane 0 / lane 1
    sm.red_m[L][row] = m_run;
    sm.red_l[L][row] = l_run;
    named_bar_sync(1, 2 * kTileRows);
    const float m0 = sm.red_m[0][row], m1 = sm.red_m[1][row];
    const float l0 = sm.red_l[0][row], l1 = sm.red_l[1][row];
    const float m = fmaxf(m0, m1);
    const float a0 = (cnt0 > 0 && m0 != -INFINITY) ? ex2_approx(m0 - m) : 0.f;
    const float a1 = (cnt1 > 0 && m1 != -INFINITY) ? ex2_approx(m1 - m) : 0.f;
    const float l_tot = l0 * a0 + l1 * a1;
    if (cnt0 > 0) mbar_wait(&sm.o_done[0], (cnt0 - 1) & 1);
    if (cnt1 > 0) mbar_wait(&sm.o_done[1], (cnt1 - 1) & 1);
    tc_fence_after();
    const bool valid = row < p.b_q;
    const bool alive = l_tot > 0.f;
    const float inv = alive ? 1.f / l_tot : 0.f;
    const float w0 = a0 * inv, w1 = a1 * inv;
    constexpr int OC = D / 2;  // output columns per lane
    uint16_t* orow = out + (q_row0 + row) * D + L * OC;
#pragma unroll
    for (int c4 = 0; c4 < OC / 32; ++c4) {
      uint32_t o0[32], o1[32];
      const uint32_t col = L * OC + c4 * 32;
      if (cnt0 > 0) {
        tmem_ld32(t_lane + kO0 + col, o0);
        tmem_ld_wait(o0);
      }
      if (cnt1 > 0) {
        tmem_ld32(t_lane + kO0 + D + col, o1);
        tmem_ld_wait(o1);
      }
      uint32_t pkd[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float v0 = 0.f, v1 = 0.f;
        if (cnt0 > 0) {
          v0 = __uint_as_float(o0[2 * e]) * w0;
          v1 = __uint_as_float(o0[2 * e + 1]) * w0;
        }
        if (cnt1 > 0) {
          v0 = fmaf(__uint_as_float(o1[2 * e]), w1, v0);
          v1 = fmaf(__uint_as_float(o1[2 * e + 1]), w1, v1);
        }
        pkd[e] = pack_bf16x2(v0, v1);
      }
      if (valid) {
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4)
          *reinterpret_cast<uint4*>(orow + c4 * 32 + v4 * 8) =
              make_uint4(pkd[v4 * 4], pkd[v4 * 4 + 1], pkd[v4 * 4 + 2], pkd[v4 * 4 + 3]);
      }
    }
    if (L == 0) {
      if (valid) lse[q_row0 + row] = alive ? (m + log2f(l_tot)) * 0.69314718055994530942f : -INFINITY;
      const unsigned dead = __ballot_sync(0xffffffffu, valid && !alive);
      if (lane == 0 && dead) atomicAdd(skipped, __popc(dead));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ====================================================================== ping-pong, P in SMEM
// psa_attn_pp_kernel with P written to shared memory instead of back into the lane's S columns:
// a lane releases S right after tcgen05.ld, so the tensor core computes the lane's NEXT S(t+2)
// while its softmax of tile t is still running (the TMEM-P variant must wait for PV(t) before
// S(t+2) can overwrite P). PV reads P with a shared-memory descriptor (K-major, 128B swizzle).
// SMEM at D=128: Q 32K + K 2x32K + V 2x32K + P 2x32K. The lanes' final (max, sum) exchange
// reuses their P buffers.
template <int D>
struct PP2Cfg {
  static constexpr int kKStages = D == 128 ? 2 : 3;
  static constexpr int kVStages = D == 128 ? 2 : 3;
  static constexpr int kTileBytes = kTileRows * D * 2;
};

template <int D>
struct PP2Smem {
  using C = PP2Cfg<D>;
  uint8_t q[kTileRows * D * 2];
  uint8_t k[C::kKStages][C::kTileBytes];
  uint8_t v[C::kVStages][C::kTileBytes];
  uint8_t p[2][kTileRows * kTileRows * 2];
  float bias[kMetaRing][kTileRows];
  uint32_t meta[kMetaRing][kChunks];
  uint64_t q_full;
  uint64_t k_full[C::kKStages], k_empty[C::kKStages];
  uint64_t v_full[C::kVStages], v_empty[C::kVStages];
  uint64_t meta_full[kMetaRing], meta_empty[kMetaRing];
  uint64_t s_full[2], s_free[2], p_full[2], o_done[2];
  uint32_t tmem_base;
};

template <int D, int POLY_FROM = kPPPolyFrom>
__global__ void __launch_bounds__(kPPThreads, 1)
    psa_attn_pp2_kernel(const __grid_constant__ AttnMaps maps, const AttnParams p,
                       const uint16_t* __restrict__ csr, const int32_t* __restrict__ info,
                       uint16_t* __restrict__ out, float* __restrict__ lse,
                       int32_t* __restrict__ skipped) {
  using C = PP2Cfg<D>;
  constexpr int KST = C::kKStages, VST = C::kVStages;
  constexpr uint32_t kO0 = 256;  // O_L at kO0 + L * D
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<PP2Smem<D>*>(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = blockIdx.x;
  const int bhq = static_cast<int>(unit / p.n_q);
  const int i = static_cast<int>(unit % p.n_q);
  const int b = bhq / p.hq, hh = bhq % p.hq;
  const int64_t bhkv = static_cast<int64_t>(b) * p.hkv + hh / (p.hq / p.hkv);
  const int n_ent = info[unit * 2 + 0];
  const int T = (info[unit * 2 + 1] + kTileRows - 1) / kTileRows;  // 128-row KV tiles
  const int64_t q_row0 = static_cast<int64_t>(bhq) * p.n + static_cast<int64_t>(i) * p.b_q;

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int s = 0; s < kMetaRing; ++s) {
      mbar_init(&sm.meta_full[s], 1);
      mbar_init(&sm.meta_empty[s], kTileRows);  // one lane (128 threads) consumes a tile
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_free[s], 4);  // one arrive per warp of the lane
      mbar_init(&sm.p_full[s], 4);
      mbar_init(&sm.o_done[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    for (int h = 0; h < p.levels; ++h) {
      tma_prefetch_desc(&maps.k[h]);
      tma_prefetch_desc(&maps.v[h]);
    }
  }
  if (warp == 2) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  {  // K/V rows past the last filled slot of a tile are read by the MMA: keep them finite
    uint4* z = reinterpret_cast<uint4*>(&sm.k[0][0]);
    const int nvec = (KST + VST) * C::kTileBytes / 16;
    for (int t = threadIdx.x; t < nvec; t += kPPThreads) z[t] = make_uint4(0, 0, 0, 0);  // K, V
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    regs_dec<64>();
    if (warp == 0) {
      // ============================================================ K producer (+ Q)
      if (T > 0) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm.q_full, kTileRows * D * 2);
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(&maps.q, &sm.q_full, sm.q + c * kTileRows * 128, c * 64,
                        static_cast<int>(q_row0));
        }
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int ks = t % KST;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= KST) mbar_wait(&sm.k_empty[ks], ((t / KST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.k_full[ks], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.k[sg.h - 1], &sm.k_full[ks],
                          sm.k[ks] + c * kTileRows * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 3) {
      // ============================================================ V producer
      if (T > 0) {
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int vs = t % VST;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= VST) mbar_wait(&sm.v_empty[vs], ((t / VST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.v_full[vs], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.v[sg.h - 1], &sm.v_full[vs],
                          sm.v[vs] + c * kTileRows * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 2) {
      // ============================================================ bias/meta producer
      if (T > 0) {
        const int64_t q_lo = static_cast<int64_t>(i) * p.b_q;
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int ms = t % kMetaRing;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= kMetaRing) mbar_wait(&sm.meta_empty[ms], ((t / kMetaRing) - 1) & 1);
          {
            int g = 0;
            for (int q = 1; q < sg.nseg; ++q)
              if (__shfl_sync(0xffffffffu, sg.off, q) <= 4 * lane) g = q;
            const int goff = __shfl_sync(0xffffffffu, sg.off, g);
            const int gL = __shfl_sync(0xffffffffu, sg.L, g);
            const int gh = __shfl_sync(0xffffffffu, sg.h, g);
            const int r0 = 4 * lane - goff;
            const float bv = static_cast<float>(gh - 1);
            float4 w = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            if (4 * lane < sg.total) {
              w.x = r0 + 0 < gL ? bv : -INFINITY;
              w.y = r0 + 1 < gL ? bv : -INFINITY;
              w.z = r0 + 2 < gL ? bv : -INFINITY;
              w.w = r0 + 3 < gL ? bv : -INFINITY;
            }
            *reinterpret_cast<float4*>(&sm.bias[ms][4 * lane]) = w;
          }
          if (p.causal && sg.fits) {
            const bool straddle = static_cast<int64_t>(sg.j + 1) * p.b_k - 1 > q_lo;
            for (int c = 0; c < sg.sz / 8; ++c)
              sm.meta[ms][sg.off / 8 + c] =
                  (straddle ? 1u : 0u) | (static_cast<uint32_t>(sg.j * p.b_k + c * 8) << 1);
          }
          if (p.causal && lane < kChunks && 8 * lane >= sg.total) sm.meta[ms][lane] = 0u;
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.meta_full[ms]);
        }
      }
    } else {
      // ============================================================ MMA issuer (warp 1)
      if (T > 0) {
        constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
        const uint64_t q_desc0 = umma_desc_sw128(smem_u32(sm.q), 16, 1024);
        auto issue_s = [&](int t) {
          const int ks = t % KST, L = t & 1;
          mbar_wait(&sm.k_full[ks], (t / KST) & 1);
          if (t >= 2) mbar_wait(&sm.s_free[L], ((t >> 1) - 1) & 1);  // lane read S(t-2)
          tc_fence_after();
          const uint64_t k_desc0 = umma_desc_sw128(smem_u32(sm.k[ks]), 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ss(tmem + L * 128, q_desc0 + koff, k_desc0 + koff, idesc_s,
                          kk > 0 ? 1u : 0u);
            }
            mma_commit(&sm.k_empty[ks]);
            mma_commit(&sm.s_full[L]);
          }
          __syncwarp();
        };
        auto issue_pv = [&](int t) {
          const int vs = t % VST, L = t & 1;
          mbar_wait(&sm.v_full[vs], (t / VST) & 1);
          mbar_wait(&sm.p_full[L], (t >> 1) & 1);
          tc_fence_after();
          const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sm.v[vs]), kTileRows * 128, 1024);
          const uint64_t p_desc0 = umma_desc_sw128(smem_u32(sm.p[L]), 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kTileRows / 16; ++kk) {
              const uint32_t poff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ss(tmem + kO0 + L * D, p_desc0 + poff, v_desc0 + ((kk * 16 * 128) >> 4),
                          idesc_o, (t >= 2 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&sm.v_empty[vs]);
            mma_commit(&sm.o_done[L]);
          }
          __syncwarp();
        };
        mbar_wait(&sm.q_full, 0);
        tc_fence_after();
        issue_s(0);
        if (T > 1) issue_s(1);
        for (int t = 0; t < T; ++t) {
          if (t + 2 < T) issue_s(t + 2);  // as soon as lane (t&1) has read S(t)
          issue_pv(t);
        }
      }
    }
  } else {
    regs_inc<216>();
    // ============================================================== softmax lanes
    const int L = (warp - 4) >> 2;  // lane L takes KV tiles t = L, L + 2, ...
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const uint32_t t_s = t_lane + L * 128;
    const int qpos = i * p.b_q + row;
    const float2 scale2 = make_float2(p.scale_log2, p.scale_log2);
    float m_run = -INFINITY, l_run = 0.f;
    for (int t = L; t < T; t += 2) {
      const int ms = t % kMetaRing;
      mbar_wait(&sm.s_full[L], (t >> 1) & 1);
      tc_fence_after();
      uint32_t s[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(t_s + c * 32, s[c]);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_wait(s[c]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.s_free[L]);  // S_L may take tile t+2 now
      // y = s * scale + bias_col (bias: level-1 in log2 units; -inf on pad columns)
      mbar_wait(&sm.meta_full[ms], (t / kMetaRing) & 1);
      float y[128];
      const float4* bias4 = reinterpret_cast<const float4*>(&sm.bias[ms][0]);
#pragma unroll
      for (int q4 = 0; q4 < 32; ++q4) {
        const float4 bv = bias4[q4];
        const float* x = reinterpret_cast<const float*>(&s[q4 >> 3][(q4 & 7) * 4]);
        const float2 a = ffma2(make_float2(x[0], x[1]), scale2, make_float2(bv.x, bv.y));
        const float2 c = ffma2(make_float2(x[2], x[3]), scale2, make_float2(bv.z, bv.w));
        y[q4 * 4 + 0] = a.x;
        y[q4 * 4 + 1] = a.y;
        y[q4 * 4 + 2] = c.x;
        y[q4 * 4 + 3] = c.y;
      }
      if (p.causal) {  // token-level mask on straddling level-1 chunks (attention.py:88-108)
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          const uint32_t w = sm.meta[ms][c];
          if (w & 1u) {
            const int lim = qpos - static_cast<int>(w >> 1);
#pragma unroll
            for (int e = 0; e < 8; ++e) y[c * 8 + e] = (e <= lim) ? y[c * 8 + e] : -INFINITY;
          }
        }
      }
      mbar_arrive(&sm.meta_empty[ms]);

      float mx[4] = {fmax3(y[0], y[1], y[2]), fmax3(y[3], y[4], y[5]), fmax3(y[6], y[7], y[8]),
                     fmax3(y[9], y[10], y[11])};
#pragma unroll
      for (int e = 12; e < 124; e += 8) {
        mx[0] = fmax3(mx[0], y[e], y[e + 1]);
        mx[1] = fmax3(mx[1], y[e + 2], y[e + 3]);
        mx[2] = fmax3(mx[2], y[e + 4], y[e + 5]);
        mx[3] = fmax3(mx[3], y[e + 6], y[e + 7]);
      }
      mx[0] = fmax3(mx[0], y[124], y[125]);
      mx[1] = fmax3(mx[1], y[126], y[127]);
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      const float m_new = fmaxf(m_run, mt);
      const bool resc = m_new > m_run + kRescaleThreshold;
      float alpha = 1.f;
      if (resc) {
        alpha = ex2_approx(m_run - m_new);
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      const float2 negm = make_float2(-m_use, -m_use);
      float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
      uint32_t pk[64];
#pragma unroll
      for (int e = 0; e < 128; e += 4) {
        float2 a = fadd2(make_float2(y[e], y[e + 1]), negm);
        float2 c = fadd2(make_float2(y[e + 2], y[e + 3]), negm);
        if (e >= POLY_FROM) {
          a = ex2_poly2(a);
          c = ex2_poly2(c);
        } else {
          a.x = ex2_approx(a.x);
          a.y = ex2_approx(a.y);
          c.x = ex2_approx(c.x);
          c.y = ex2_approx(c.y);
        }
        ls0 = fadd2(ls0, a);
        ls1 = fadd2(ls1, c);
        pk[e / 2] = pack_bf16x2(a.x, a.y);
        pk[e / 2 + 1] = pack_bf16x2(c.x, c.y);
      }
      const float2 ls = fadd2(ls0, ls1);
      l_run = l_run * alpha + (ls.x + ls.y);
      // PV(t-2) done: P_L is free and O_L is stable
      if (t >= 2) {
        mbar_wait(&sm.o_done[L], ((t >> 1) - 1) & 1);
        tc_fence_after();
      }
      if (t >= 2 && __any_sync(0xffffffffu, resc)) {
#pragma unroll
        for (int c4 = 0; c4 < D / 32; ++c4) {
          uint32_t o[32];
          tmem_ld32(t_lane + kO0 + L * D + c4 * 32, o);
          tmem_ld_wait(o);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tmem_st32(t_lane + kO0 + L * D + c4 * 32, o);
        }
      }
      {  // P (bf16) -> shared memory, UMMA K-major 128B-swizzled: [key half][row][128 B]
        uint8_t* prow = sm.p[L] + row * 128;
        const int sw = row & 7;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            *reinterpret_cast<uint4*>(prow + c * kTileRows * 128 + ((ch ^ sw) << 4)) =
                make_uint4(pk[c * 32 + ch * 4], pk[c * 32 + ch * 4 + 1], pk[c * 32 + ch * 4 + 2],
                           pk[c * 32 + ch * 4 + 3]);
      }
      tmem_st_wait();  // O rescale stores
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full[L]);
    }

    // ---------------------------------------------------------------- merge + epilogue
    const int cnt0 = (T + 1) >> 1, cnt1 = T >> 1;  // tiles of lane 0 / lane 1
    const int cnt_me = L == 0 ? cnt0 : cnt1;
    if (cnt_me > 0) mbar_wait(&sm.o_done[L], (cnt_me - 1) & 1);  // P_L no longer read
    float* red = reinterpret_cast<float*>(sm.p[L]);
    red[row] = m_run;
    red[kTileRows + row] = l_run;
    named_bar_sync(1, 2 * kTileRows);
    const float* red0 = reinterpret_cast<const float*>(sm.p[0]);
    const float* red1 = reinterpret_cast<const float*>(sm.p[1]);
    const float m0 = red0[row], m1 = red1[row];
    const float l0 = red0[kTileRows + row], l1 = red1[kTileRows + row];
    const float m = fmaxf(m0, m1);
    const float a0 = (cnt0 > 0 && m0 != -INFINITY) ? ex2_approx(m0 - m) : 0.f;
    const float a1 = (cnt1 > 0 && m1 != -INFINITY) ? ex2_approx(m1 - m) : 0.f;
    const float l_tot = l0 * a0 + l1 * a1;
    if (cnt0 > 0) mbar_wait(&sm.o_done[0], (cnt0 - 1) & 1);
    if (cnt1 > 0) mbar_wait(&sm.o_done[1], (cnt1 - 1) & 1);
    tc_fence_after();
    const bool valid = row < p.b_q;
    const bool alive = l_tot > 0.f;
    const float inv = alive ? 1.f / l_tot : 0.f;
    const float w0 = a0 * inv, w1 = a1 * inv;
    constexpr int OC = D / 2;  // output columns per lane
    // unpermute (pipeline.py:312-313) fused into the store: row i of the head -> out_rows[i]
    const int64_t o_row = p.out_rows == nullptr || !valid
                              ? q_row0 + row
                              : static_cast<int64_t>(bhq) * p.n + p.out_rows[i * p.b_q + row];
    uint16_t* orow = out + o_row * D + L * OC;
#pragma unroll
    for (int c4 = 0; c4 < OC / 32; ++c4) {
      uint32_t o0[32], o1[32];
      const uint32_t col = L * OC + c4 * 32;
      if (cnt0 > 0) {
        tmem_ld32(t_lane + kO0 + col, o0);
        tmem_ld_wait(o0);
      }
      if (cnt1 > 0) {
        tmem_ld32(t_lane + kO0 + D + col, o1);
        tmem_ld_wait(o1);
      }
      uint32_t pkd[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float v0 = 0.f, v1 = 0.f;
        if (cnt0 > 0) {
          v0 = __uint_as_float(o0[2 * e]) * w0;
          v1 = __uint_as_float(o0[2 * e + 1]) * w0;
        }
        if (cnt1 > 0) {
          v0 = fmaf(__uint_as_float(o1[2 * e]), w1, v0);
          v1 = fmaf(__uint_as_float(o1[2 * e + 1]), w1, v1);
        }
        pkd[e] = pack_bf16x2(v0, v1);
      }
      if (valid) {
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4)
          *reinterpret_cast<uint4*>(orow + c4 * 32 + v4 * 8) =
              make_uint4(pkd[v4 * 4], pkd[v4 * 4 + 1], pkd[v4 * 4 + 2], pkd[v4 * 4 + 3]);
      }
    }
    if (L == 0) {
      if (valid) lse[o_row] = alive ? (m + log2f(l_tot)) * 0.69314718055994530942f : -INFINITY;
      const unsigned dead = __ballot_sync(0xffffffffu, valid && !alive);
      if (lane == 0 && dead) atomicAdd(skipped, __popc(dead));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ====================================================================== pp4: Q and P in TMEM
// Shared-memory traffic is what bounds psa_attn_pp2_kernel (Q, K, P, V operand reads + K/V TMA
// writes + P stores ~ 224 KB per 128x128 tile). pp4 keeps both Q (the S MMA's A operand) and P
// (the PV MMA's A operand) in tensor memory, so per KV row the SM only moves the K and V rows
// (TMA write + one tensor-core read each): ~128 B/clk at full MMA rate. The TMEM budget then
// forces 64-row KV tiles (N = 64):
//   cols [0, D/2) Q | S0, S1 (64 each) | P0, P1 (32 each) | O0, O1 (D each)      (512 at D=128)
// Level-1 blocks longer than 64 rows are split into 64-row pieces (the reference's schedule
// splits blocks across tiles too, scheduler.py:71-126); every other segment sits in a
// power-of-two slot, so ceil(R / 64) tiles hold the plan exactly (R = plan_info slot rows).
// Roles as in pp2: K producer (+Q TMA), bias/meta producer, V producer, one MMA issuer, two
// softmax lanes on alternate tiles (lane 0 also copies Q from shared memory into TMEM).
constexpr int kT4 = 64;             // KV rows per tile (MMA N)
constexpr int kT4Chunks = kT4 / 8;
constexpr int kT4Meta = 8;          // bias/meta ring depth

template <int D>
struct PP4Cfg {
  static constexpr int kKStages = 4;
  static constexpr int kVStages = 4;
  static constexpr int kTileBytes = kT4 * D * 2;
  static constexpr uint32_t kColQ = 0;
  static constexpr uint32_t kColS = D / 2;            // + 64 L
  static constexpr uint32_t kColP = kColS + 2 * kT4;  // + 32 L
  static constexpr uint32_t kColO = kColP + kT4;      // + D L
  static_assert(kColO + 2 * D <= 512, "TMEM budget");
};

template <int D>
struct PP4Smem {
  using C = PP4Cfg<D>;
  uint8_t q[kTileRows * D * 2];  // TMA landing of Q; reused for the final lane merge
  uint8_t k[C::kKStages][C::kTileBytes];
  uint8_t v[C::kVStages][C::kTileBytes];
  float bias[kT4Meta][kT4];
  uint32_t meta[kT4Meta][kT4Chunks];
  uint64_t q_full, q_tmem;
  uint64_t k_full[C::kKStages], k_empty[C::kKStages];
  uint64_t v_full[C::kVStages], v_empty[C::kVStages];
  uint64_t meta_full[kT4Meta], meta_empty[kT4Meta];
  uint64_t s_full[2], s_free[2], p_full[2], o_done[2];
  uint32_t tmem_base;
};

// Plan walk for 64-row tiles: segments of <= 64 rows pack as in PlanCursor; a segment longer
// than 64 rows (level 1 with b_k > 64) forms single-piece tiles of 64 rows.
struct PlanCursor64 {
  const uint16_t* plan;
  int n_ent, e, base, piece;
  uint32_t cur, nxt;
  PSA_DEV void init(const uint16_t* pl, int n, int lane) {
    plan = pl;
    n_ent = n;
    e = 0;
    base = 0;
    piece = 0;
    cur = lane < n ? plan[lane] : 0u;
    nxt = 32 + lane < n ? plan[32 + lane] : 0u;
  }
  PSA_DEV void advance(int k, int lane) {
    e += k;
    if (e - base >= 32) {
      base += 32;
      cur = nxt;
      nxt = base + 32 + lane < n_ent ? plan[base + 32 + lane] : 0u;
    }
  }
  // s.row: first global row of this lane's segment; s.rows: valid rows of the segment
  PSA_DEV TileSeg next(const AttnParams& p, int64_t bhkv, int lane, int& rows, int& key0) {
    TileSeg s;
    const int rel = e - base + lane;
    const uint32_t a = __shfl_sync(0xffffffffu, cur, rel & 31);
    const uint32_t b = __shfl_sync(0xffffffffu, nxt, rel & 31);
    const uint32_t ent = rel < 32 ? a : b;
    const int h0 = static_cast<int>(__shfl_sync(0xffffffffu, ent, 0) >> 12);
    const int L0 = p.b_k >> (h0 - 1);
    if (L0 > kT4) {  // one 64-row piece of a long block
      s.j = static_cast<int>(__shfl_sync(0xffffffffu, ent, 0) & 0xFFFu);
      s.h = h0;
      s.L = L0;
      s.sz = kT4;
      s.off = 0;
      s.nseg = 1;
      s.total = kT4;
      s.fits = lane == 0;
      rows = min(kT4, L0 - piece * kT4);
      key0 = s.j * p.b_k + piece * kT4;
      s.row = static_cast<int>(bhkv) * static_cast<int>(p.n >> (h0 - 1)) + s.j * L0 + piece * kT4;
      if (++piece * kT4 >= L0) {
        piece = 0;
        advance(1, lane);
      }
      return s;
    }
    const bool valid = lane < kT4Chunks && e + lane < n_ent;
    s.j = static_cast<int>(ent & 0xFFFu);
    s.h = valid ? static_cast<int>(ent >> 12) : 1;
    s.L = valid ? (p.b_k >> (s.h - 1)) : 0;
    s.sz = 256;
    if (valid) s.sz = s.L <= 8 ? 8 : (1 << (32 - __clz(s.L - 1)));
    int incl = s.sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    s.fits = incl <= kT4;
    s.nseg = __popc(__ballot_sync(0xffffffffu, s.fits));
    s.total = __shfl_sync(0xffffffffu, incl, s.nseg - 1);
    s.off = incl - s.sz;
    s.row = static_cast<int>(bhkv) * static_cast<int>(p.n >> (s.h - 1)) + s.j * s.L;
    rows = s.L;
    key0 = s.j * p.b_k;
    advance(s.nseg, lane);
    return s;
  }
};

template <int D>
__global__ void __launch_bounds__(kPPThreads, 1)
    psa_attn_pp4_kernel(const __grid_constant__ AttnMaps maps, const AttnParams p,
                        const uint16_t* __restrict__ csr, const int32_t* __restrict__ info,
                        uint16_t* __restrict__ out, float* __restrict__ lse,
                        int32_t* __restrict__ skipped) {
  using C = PP4Cfg<D>;
  constexpr int KST = C::kKStages, VST = C::kVStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<PP4Smem<D>*>(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = blockIdx.x;
  const int bhq = static_cast<int>(unit / p.n_q);
  const int i = static_cast<int>(unit % p.n_q);
  const int b = bhq / p.hq, hh = bhq % p.hq;
  const int64_t bhkv = static_cast<int64_t>(b) * p.hkv + hh / (p.hq / p.hkv);
  const int n_ent = info[unit * 2 + 0];
  const int T = (info[unit * 2 + 1] + kT4 - 1) / kT4;
  const int64_t q_row0 = static_cast<int64_t>(bhq) * p.n + static_cast<int64_t>(i) * p.b_q;

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_tmem, 4);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int s = 0; s < kT4Meta; ++s) {
      mbar_init(&sm.meta_full[s], 1);
      mbar_init(&sm.meta_empty[s], 4);  // the 4 warps of one lane
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_free[s], 4);
      mbar_init(&sm.p_full[s], 4);
      mbar_init(&sm.o_done[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    for (int h = 0; h < p.levels; ++h) {
      tma_prefetch_desc(&maps.k[h]);
      tma_prefetch_desc(&maps.v[h]);
    }
  }
  if (warp == 2) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  {  // K/V rows past the last filled slot of a tile are read by the MMA: keep them finite
    uint4* z = reinterpret_cast<uint4*>(&sm.k[0][0]);
    const int nvec = (KST + VST) * C::kTileBytes / 16;
    for (int t = threadIdx.x; t < nvec; t += kPPThreads) z[t] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    regs_dec<64>();
    if (warp == 0) {
      // ============================================================ K producer (+ Q)
      if (T > 0) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm.q_full, kTileRows * D * 2);
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(&maps.q, &sm.q_full, sm.q + c * kTileRows * 128, c * 64,
                        static_cast<int>(q_row0));
        }
        PlanCursor64 pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int ks = t % KST;
          int rows, key0;
          const TileSeg sg = pc.next(p, bhkv, lane, rows, key0);
          if (t >= KST) mbar_wait(&sm.k_empty[ks], ((t / KST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.k_full[ks], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.k[sg.h - 1], &sm.k_full[ks],
                          sm.k[ks] + c * kT4 * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 3) {
      // ============================================================ V producer
      if (T > 0) {
        PlanCursor64 pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int vs = t % VST;
          int rows, key0;
          const TileSeg sg = pc.next(p, bhkv, lane, rows, key0);
          if (t >= VST) mbar_wait(&sm.v_empty[vs], ((t / VST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.v_full[vs], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.v[sg.h - 1], &sm.v_full[vs],
                          sm.v[vs] + c * kT4 * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 2) {
      // ============================================================ bias/meta producer
      if (T > 0) {
        const int64_t q_lo = static_cast<int64_t>(i) * p.b_q;
        PlanCursor64 pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int ms = t % kT4Meta;
          int rows, key0;
          const TileSeg sg = pc.next(p, bhkv, lane, rows, key0);
          if (t >= kT4Meta) mbar_wait(&sm.meta_empty[ms], ((t / kT4Meta) - 1) & 1);
          {  // lane l fills columns 2l, 2l+1: find the owning segment (offsets ascend)
            int g = 0;
            for (int q = 1; q < sg.nseg; ++q)
              if (__shfl_sync(0xffffffffu, sg.off, q) <= 2 * lane) g = q;
            const int goff = __shfl_sync(0xffffffffu, sg.off, g);
            const int grows = __shfl_sync(0xffffffffu, rows, g);
            const int gh = __shfl_sync(0xffffffffu, sg.h, g);
            const int r0 = 2 * lane - goff;
            const float bv = static_cast<float>(gh - 1);
            float2 w = make_float2(-INFINITY, -INFINITY);
            if (2 * lane < sg.total) {
              w.x = r0 + 0 < grows ? bv : -INFINITY;
              w.y = r0 + 1 < grows ? bv : -INFINITY;
            }
            *reinterpret_cast<float2*>(&sm.bias[ms][2 * lane]) = w;
          }
          if (p.causal) {
            if (sg.fits) {
              const bool straddle = static_cast<int64_t>(sg.j + 1) * p.b_k - 1 > q_lo;
              for (int c = 0; c < sg.sz / 8; ++c)
                sm.meta[ms][sg.off / 8 + c] =
                    (straddle ? 1u : 0u) | (static_cast<uint32_t>(key0 + c * 8) << 1);
            }
            if (lane < kT4Chunks && 8 * lane >= sg.total) sm.meta[ms][lane] = 0u;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.meta_full[ms]);
        }
      }
    } else {
      // ============================================================ MMA issuer (warp 1)
      if (T > 0) {
        constexpr uint32_t idesc_s = umma_idesc_bf16(128, kT4, false, false);
        constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
        auto issue_s = [&](int t) {
          const int ks = t % KST, L = t & 1;
          mbar_wait(&sm.k_full[ks], (t / KST) & 1);
          if (t >= 2) mbar_wait(&sm.s_free[L], ((t >> 1) - 1) & 1);  // lane read S(t-2)
          tc_fence_after();
          const uint64_t k_desc0 = umma_desc_sw128(smem_u32(sm.k[ks]), 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t koff = ((kk >> 2) * kT4 * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ts(tmem + C::kColS + L * kT4, tmem + C::kColQ + kk * 8, k_desc0 + koff,
                          idesc_s, kk > 0 ? 1u : 0u);
            }
            mma_commit(&sm.k_empty[ks]);
            mma_commit(&sm.s_full[L]);
          }
          __syncwarp();
        };
        auto issue_pv = [&](int t) {
          const int vs = t % VST, L = t & 1;
          mbar_wait(&sm.v_full[vs], (t / VST) & 1);
          mbar_wait(&sm.p_full[L], (t >> 1) & 1);
          tc_fence_after();
          const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sm.v[vs]), kT4 * 128, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kT4 / 16; ++kk)
              mma_bf16_ts(tmem + C::kColO + L * D, tmem + C::kColP + L * (kT4 / 2) + kk * 8,
                          v_desc0 + ((kk * 16 * 128) >> 4), idesc_o,
                          (t >= 2 || kk > 0) ? 1u : 0u);
            mma_commit(&sm.v_empty[vs]);
            mma_commit(&sm.o_done[L]);
          }
          __syncwarp();
        };
        mbar_wait(&sm.q_tmem, 0);
        tc_fence_after();
        issue_s(0);
        if (T > 1) issue_s(1);
        for (int t = 0; t < T; ++t) {
          if (t + 2 < T) issue_s(t + 2);  // as soon as lane (t&1) has read S(t)
          issue_pv(t);
        }
      }
    }
  } else {
    regs_inc<216>();
    // ============================================================== softmax lanes
    const int L = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int qpos = i * p.b_q + row;
    if (L == 0 && T > 0) {  // Q (bf16 pairs, K-consecutive) from the swizzled TMA tile into TMEM
      mbar_wait(&sm.q_full, 0);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t qv[32];
        const uint8_t* qrow = sm.q + c * kTileRows * 128 + row * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const uint4 x = *reinterpret_cast<const uint4*>(qrow + ((ch ^ (row & 7)) << 4));
          qv[4 * ch] = x.x;
          qv[4 * ch + 1] = x.y;
          qv[4 * ch + 2] = x.z;
          qv[4 * ch + 3] = x.w;
        }
        tmem_st32(t_lane + C::kColQ + c * 32, qv);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.q_tmem);
    }
    const uint32_t t_s = t_lane + C::kColS + L * kT4;
    const uint32_t t_p = t_lane + C::kColP + L * (kT4 / 2);
    const uint32_t t_o = t_lane + C::kColO + L * D;
    const float2 scale2 = make_float2(p.scale_log2, p.scale_log2);
    float m_run = -INFINITY, l_run = 0.f;
    for (int t = L; t < T; t += 2) {
      const int ms = t % kT4Meta;
      mbar_wait(&sm.s_full[L], (t >> 1) & 1);
      tc_fence_after();
      uint32_t s[2][32];
      tmem_ld32(t_s, s[0]);
      tmem_ld32(t_s + 32, s[1]);
      tmem_ld_wait(s[0]);
      tmem_ld_wait(s[1]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.s_free[L]);  // S_L may take tile t+2 now
      mbar_wait(&sm.meta_full[ms], (t / kT4Meta) & 1);
      float y[kT4];
      const float4* bias4 = reinterpret_cast<const float4*>(&sm.bias[ms][0]);
#pragma unroll
      for (int q4 = 0; q4 < kT4 / 4; ++q4) {
        const float4 bv = bias4[q4];
        const float* x = reinterpret_cast<const float*>(&s[q4 >> 3][(q4 & 7) * 4]);
        const float2 a = ffma2(make_float2(x[0], x[1]), scale2, make_float2(bv.x, bv.y));
        const float2 c = ffma2(make_float2(x[2], x[3]), scale2, make_float2(bv.z, bv.w));
        y[q4 * 4 + 0] = a.x;
        y[q4 * 4 + 1] = a.y;
        y[q4 * 4 + 2] = c.x;
        y[q4 * 4 + 3] = c.y;
      }
      if (p.causal) {  // token-level mask on straddling level-1 chunks (attention.py:88-108)
#pragma unroll
        for (int c = 0; c < kT4Chunks; ++c) {
          const uint32_t w = sm.meta[ms][c];
          if (w & 1u) {
            const int lim = qpos - static_cast<int>(w >> 1);
#pragma unroll
            for (int e = 0; e < 8; ++e) y[c * 8 + e] = (e <= lim) ? y[c * 8 + e] : -INFINITY;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.meta_empty[ms]);

      float mx[4] = {fmax3(y[0], y[1], y[2]), fmax3(y[3], y[4], y[5]), fmax3(y[6], y[7], y[8]),
                     fmax3(y[9], y[10], y[11])};
#pragma unroll
      for (int e = 12; e < 60; e += 8) {
        mx[0] = fmax3(mx[0], y[e], y[e + 1]);
        mx[1] = fmax3(mx[1], y[e + 2], y[e + 3]);
        mx[2] = fmax3(mx[2], y[e + 4], y[e + 5]);
        mx[3] = fmax3(mx[3], y[e + 6], y[e + 7]);
      }
      mx[0] = fmax3(mx[0], y[60], y[61]);
      mx[1] = fmax3(mx[1], y[62], y[63]);
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      const float m_new = fmaxf(m_run, mt);
      const bool resc = m_new > m_run + kRescaleThreshold;
      float alpha = 1.f;
      if (resc) {
        alpha = ex2_approx(m_run - m_new);
        m_run = m_new;
      }
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      const float2 negm = make_float2(-m_use, -m_use);
      float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < kT4; e += 4) {
        float2 a = fadd2(make_float2(y[e], y[e + 1]), negm);
        float2 c = fadd2(make_float2(y[e + 2], y[e + 3]), negm);
        if (e >= 48) {  // last quarter on the FMA-pipe exp2
          a = ex2_poly2(a);
          c = ex2_poly2(c);
        } else {
          a.x = ex2_approx(a.x);
          a.y = ex2_approx(a.y);
          c.x = ex2_approx(c.x);
          c.y = ex2_approx(c.y);
        }
        ls0 = fadd2(ls0, a);
        ls1 = fadd2(ls1, c);
        pk[e / 2] = pack_bf16x2(a.x, a.y);
        pk[e / 2 + 1] = pack_bf16x2(c.x, c.y);
      }
      const float2 ls = fadd2(ls0, ls1);
      l_run = l_run * alpha + (ls.x + ls.y);
      if (t >= 2) {  // PV(t-2) done: P_L is free and O_L is stable
        mbar_wait(&sm.o_done[L], ((t >> 1) - 1) & 1);
        tc_fence_after();
      }
      if (t >= 2 && __any_sync(0xffffffffu, resc)) {
#pragma unroll
        for (int c4 = 0; c4 < D / 32; ++c4) {
          uint32_t o[32];
          tmem_ld32(t_o + c4 * 32, o);
          tmem_ld_wait(o);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tmem_st32(t_o + c4 * 32, o);
        }
      }
      tmem_st32(t_p, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.p_full[L]);
    }

    // ---------------------------------------------------------------- merge + epilogue
    const int cnt0 = (T + 1) >> 1, cnt1 = T >> 1;  // tiles of lane 0 / lane 1
    if (T > 0) mbar_wait(&sm.q_tmem, 0);  // lane 0 has finished reading the Q landing zone
    float* red = reinterpret_cast<float*>(sm.q);  // Q lives in TMEM now; its landing zone is free
    red[(2 * L) * kTileRows + row] = m_run;
    red[(2 * L + 1) * kTileRows + row] = l_run;
    named_bar_sync(1, 2 * kTileRows);
    const float m0 = red[row], l0 = red[kTileRows + row];
    const float m1 = red[2 * kTileRows + row], l1 = red[3 * kTileRows + row];
    const float m = fmaxf(m0, m1);
    const float a0 = (cnt0 > 0 && m0 != -INFINITY) ? ex2_approx(m0 - m) : 0.f;
    const float a1 = (cnt1 > 0 && m1 != -INFINITY) ? ex2_approx(m1 - m) : 0.f;
    const float l_tot = l0 * a0 + l1 * a1;
    if (cnt0 > 0) mbar_wait(&sm.o_done[0], (cnt0 - 1) & 1);
    if (cnt1 > 0) mbar_wait(&sm.o_done[1], (cnt1 - 1) & 1);
    tc_fence_after();
    const bool valid = row < p.b_q;
    const bool alive = l_tot > 0.f;
    const float inv = alive ? 1.f / l_tot : 0.f;
    const float w0 = a0 * inv, w1 = a1 * inv;
    constexpr int OC = D / 2;  // output columns per lane
    uint16_t* orow = out + (q_row0 + row) * D + L * OC;
#pragma unroll
    for (int c4 = 0; c4 < OC / 32; ++c4) {
      uint32_t o0[32], o1[32];
      const uint32_t col = L * OC + c4 * 32;
      if (cnt0 > 0) {
        tmem_ld32(t_lane + C::kColO + col, o0);
        tmem_ld_wait(o0);
      }
      if (cnt1 > 0) {
        tmem_ld32(t_lane + C::kColO + D + col, o1);
        tmem_ld_wait(o1);
      }
      uint32_t pkd[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float v0 = 0.f, v1 = 0.f;
        if (cnt0 > 0) {
          v0 = __uint_as_float(o0[2 * e]) * w0;
          v1 = __uint_as_float(o0[2 * e + 1]) * w0;
        }
        if (cnt1 > 0) {
          v0 = fmaf(__uint_as_float(o1[2 * e]), w1, v0);
          v1 = fmaf(__uint_as_float(o1[2 * e + 1]), w1, v1);
        }
        pkd[e] = pack_bf16x2(v0, v1);
      }
      if (valid) {
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4)
          *reinterpret_cast<uint4*>(orow + c4 * 32 + v4 * 8) =
              make_uint4(pkd[v4 * 4], pkd[v4 * 4 + 1], pkd[v4 * 4 + 2], pkd[v4 * 4 + 3]);
      }
    }
    if (L == 0) {
      if (valid) lse[q_row0 + row] = alive ? (m + log2f(l_tot)) * 0.69314718055994530942f : -INFINITY;
      const unsigned dead = __ballot_sync(0xffffffffu, valid && !alive);
      if (lane == 0 && dead) atomicAdd(skipped, __popc(dead));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side
EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 2D bf16 [rows, cols] row-major, box = [box_rows, 64 cols], 128-byte swizzle.
static int encode_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                     uint32_t box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (fn == nullptr) return psa_fail(PSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return psa_fail(PSA_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PSA_OK;
}

template <int D>
static int launch_attn(const void* q, const void* k, const void* v, const void* k_pyr,
                       const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n, int b_q,
                       int b_k, int levels, const uint16_t* csr, const int32_t* info, int causal,
                       void* out, float* lse, int32_t* skipped, const int64_t* out_rows,
                       cudaStream_t s) {
  AttnMaps maps;
  memset(&maps, 0, sizeof(maps));
  AttnParams p{};
  p.n = n;
  p.hq = hq;
  p.hkv = hkv;
  p.b_q = b_q;
  p.b_k = b_k;
  p.levels = levels;
  p.n_q = static_cast<int>(n / b_q);
  p.n_k = static_cast<int>(n / b_k);
  p.causal = causal;
  p.scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(D)));
  p.out_rows = out_rows;
  const int64_t bhkv = batch * hkv;
  int rc = encode_2d(&maps.q, q, static_cast<uint64_t>(batch * hq * n), D, kTileRows);
  if (rc) return rc;
  int64_t off_elems = 0;
  for (int h = 1; h <= levels; ++h) {
    const int L = b_k >> (h - 1);
    int sz = 8;
    while (sz < L) sz <<= 1;
    const uint64_t rows = static_cast<uint64_t>(bhkv * (n >> (h - 1)));
    const void* kb = h == 1 ? k : static_cast<const void*>(static_cast<const uint16_t*>(k_pyr) + off_elems);
    const void* vb = h == 1 ? v : static_cast<const void*>(static_cast<const uint16_t*>(v_pyr) + off_elems);
    if (h > 1) off_elems += static_cast<int64_t>(rows) * D;
    rc = encode_2d(&maps.k[h - 1], kb, rows, D, sz);
    if (rc) return rc;
    rc = encode_2d(&maps.v[h - 1], vb, rows, D, sz);
    if (rc) return rc;
  }
  const int64_t units = batch * hq * p.n_q;
  static const bool use_v1 = [] {
    const char* e = getenv("PSA_ATTN_KERNEL");
    return e != nullptr && strcmp(e, "v1") == 0;
  }();
  if (out_rows != nullptr && getenv("PSA_ATTN_KERNEL") != nullptr &&
      strcmp(getenv("PSA_ATTN_KERNEL"), "pp2") != 0)
    return psa_fail(PSA_EINVAL, "the scatter epilogue exists only in the default (pp2) kernel");
  if (use_v1) {
    const size_t smem = sizeof(AttnSmem<D>);
    cudaFuncSetAttribute(psa_attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    psa_attn_fwd_kernel<D><<<static_cast<unsigned>(units), kAttnThreads, smem, s>>>(
        maps, p, csr, info, static_cast<uint16_t*>(out), lse, skipped);
    return psa_check_launch("psa_attn_fwd_kernel");
  }
  static const bool use_pp4 = [] {
    const char* e = getenv("PSA_ATTN_KERNEL");
    return e != nullptr && strcmp(e, "pp4") == 0;
  }();
  if (use_pp4) {  // 64-row KV tiles: level maps with at most 64-row boxes
    AttnMaps m4 = maps;
    int64_t off4 = 0;
    for (int h = 1; h <= levels; ++h) {
      const int L = b_k >> (h - 1);
      int sz = 8;
      while (sz < L) sz <<= 1;
      sz = sz > kT4 ? kT4 : sz;
      const uint64_t rows = static_cast<uint64_t>(batch * hkv * (n >> (h - 1)));
      const void* kb = h == 1 ? k : static_cast<const void*>(static_cast<const uint16_t*>(k_pyr) + off4);
      const void* vb = h == 1 ? v : static_cast<const void*>(static_cast<const uint16_t*>(v_pyr) + off4);
      if (h > 1) off4 += static_cast<int64_t>(rows) * D;
      int rc4 = encode_2d(&m4.k[h - 1], kb, rows, D, sz);
      if (rc4) return rc4;
      rc4 = encode_2d(&m4.v[h - 1], vb, rows, D, sz);
      if (rc4) return rc4;
    }
    const size_t smem4 = sizeof(PP4Smem<D>);
    auto kern4 = psa_attn_pp4_kernel<D>;
    cudaFuncSetAttribute(kern4, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem4));
    kern4<<<static_cast<unsigned>(units), kPPThreads, smem4, s>>>(
        m4, p, csr, info, static_cast<uint16_t*>(out), lse, skipped);
    return psa_check_launch("psa_attn_pp4_kernel");
  }
  static const bool use_pp1 = [] {
    const char* e = getenv("PSA_ATTN_KERNEL");
    return e != nullptr && strcmp(e, "pp") == 0;
  }();
  if (!use_pp1) {
    const size_t smem2 = sizeof(PP2Smem<D>);
    auto kern2 = psa_attn_pp2_kernel<D>;
    cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem2));
    kern2<<<static_cast<unsigned>(units), kPPThreads, smem2, s>>>(
        maps, p, csr, info, static_cast<uint16_t*>(out), lse, skipped);
    return psa_check_launch("psa_attn_pp2_kernel");
  }
  const size_t smem = sizeof(PPSmem<D>);
  static const int poly = [] {  // experiment knob: first softmax column on the FMA-pipe exp2
    const char* e = getenv("PSA_PP_POLY");
    return e != nullptr ? atoi(e) : kPPPolyFrom;
  }();
  auto kern = poly >= 128 ? psa_attn_pp_kernel<D, 128>
            : poly >= 112 ? psa_attn_pp_kernel<D, 112>
            : poly >= 96 ? psa_attn_pp_kernel<D, 96>
            : poly >= 80 ? psa_attn_pp_kernel<D, 80> : psa_attn_pp_kernel<D, 64>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  kern<<<static_cast<unsigned>(units), kPPThreads, smem, s>>>(
      maps, p, csr, info, static_cast<uint16_t*>(out), lse, skipped);
  return psa_check_launch("psa_attn_pp_kernel");
}

}  // namespace psa

using namespace psa;

extern "C" int psa_attn_fwd_scatter(const void* q, const void* k, const void* v,
                                    const void* k_pyr, const void* v_pyr, int64_t batch, int hq,
                                    int hkv, int64_t n, int d, int b_q, int b_k, int levels,
                                    const uint16_t* plan_csr, const int32_t* plan_info, int causal,
                                    void* out, float* lse, int32_t* skipped_rows,
                                    const int64_t* out_rows, void* stream) {
  PSA_CHECK_ARG(q && k && v && plan_csr && plan_info && out && lse && skipped_rows,
                "null pointer argument");
  PSA_CHECK_ARG(d == 64 || d == 128, "head_dim must be 64 or 128 for the sm_100a path");
  PSA_CHECK_ARG(b_q >= 1 && b_q <= kTileRows, "q_block must lie in 1..128 for the sm_100a kernel");
  PSA_CHECK_ARG(b_k >= 1 && b_k <= kTileRows, "k_block must lie in 1..128 for the sm_100a kernel");
  PSA_CHECK_ARG(n % b_q == 0 && n % b_k == 0, "layout does not divide seq_len");
  PSA_CHECK_ARG(levels >= 1 && levels <= kMaxLevels, "levels must lie in 1..8");
  PSA_CHECK_ARG(levels == 1 || (k_pyr && v_pyr), "pyramid pointers required for levels > 1");
  PSA_CHECK_ARG(hq >= 1 && hkv >= 1 && hq % hkv == 0, "query heads must be a multiple of kv heads");
  PSA_CHECK_ARG(n / b_k <= 4096, "n_k must be <= 4096");
  PSA_CHECK_ARG(batch * hq * n < (int64_t(1) << 31), "too many rows for 32-bit TMA coordinates");
  PSA_CHECK_ARG(n < (int64_t(1) << 23), "seq_len must be < 2^23");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (d == 128)
    return launch_attn<128>(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, b_q, b_k, levels, plan_csr,
                            plan_info, causal, out, lse, skipped_rows, out_rows, s);
  return launch_attn<64>(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, b_q, b_k, levels, plan_csr,
                         plan_info, causal, out, lse, skipped_rows, out_rows, s);
}

extern "C" int psa_attn_fwd(const void* q, const void* k, const void* v, const void* k_pyr,
                            const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n, int d,
                            int b_q, int b_k, int levels, const uint16_t* plan_csr,
                            const int32_t* plan_info, int causal, void* out, float* lse,
                            int32_t* skipped_rows, void* stream) {
  return psa_attn_fwd_scatter(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, d, b_q, b_k, levels,
                              plan_csr, plan_info, causal, out, lse, skipped_rows, nullptr, stream);
}
