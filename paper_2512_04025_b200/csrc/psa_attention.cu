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
// psa_attn_pp2_kernel: one CTA per (head, query block) work unit, 12 warps:
//   warp 0  K TMA producer (+ the Q tile): walks the unit's level-major plan and packs pooled
//           segments into 128-row KV tiles. Segment sizes are padded to power-of-two slots
//           (>= 8 rows) and emitted largest-first, so every slot starts on a 1024-byte (8-row)
//           swizzle atom and the packing is perfect except for the last tile.
//   warp 3  V TMA producer (same walk); warp 2 bias/meta producer (per-column level bias in
//           log2 units or -inf on pad columns, causal chunk metadata) and TMEM allocator.
//   warp 1  MMA issuer (one elected thread): S_L = Q K^T into TMEM, O_L += P_L V with P from
//           shared memory.
//   warps 4-7 / 8-11  softmax "lanes" 0 / 1 taking alternate KV tiles, one query row per thread
//           (details at the kernel). Other variants measured during development (one lane with
//           the columns split across warpgroups; P kept in TMEM; Q and P in TMEM with 64-row KV
//           tiles) are described in DESIGN.md and live in the git history.
#include <cstring>

#include "common.cuh"
#include "psa_internal.h"

namespace psa {

constexpr int kTileRows = 128;  // query rows per tile (MMA M) and KV rows per tile (MMA N)
constexpr int kChunks = kTileRows / 8;
constexpr int kMetaRing = 4;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

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
  // optional q-block work units: unit u of head bhq is query block qblk[u % n_qs]; O/lse rows are
  // then compact, [bhq, n_qs * b_q) (NULL: n_qs = n_q, every block, rows in place)
  const int32_t* qblk;
  int n_qs;
  // forward: the level bias (h-1)*ln2 of attention.py:39-44 in raw logit units, (h-1)/scale_log2,
  // as three bf16 terms
  // hi | mid << 16, lo, i.e. the first 8 bytes of a key's augmentation row (see kAugPad)
  uint32_t aug[kMaxLevels][2];
};
// augmentation row of a pad key: -2^100 in the first column (S -> -1.3e30: exp2 -> 0, never the max)
constexpr uint32_t kAugPad = 0xF180u;

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

// ====================================================================== ping-pong lanes
// The two softmax warpgroups are independent "lanes" that take ALTERNATE KV tiles of the unit,
// each with full 128-column rows, its own running (max, sum) and its own O accumulator in TMEM;
// the lanes merge once in the epilogue. While one lane runs its softmax, the tensor core
// computes the other lane's S and PV. P goes to shared memory, so a lane releases S right after
// tcgen05.ld and the tensor core computes the lane's NEXT S(t+2) while its softmax of tile t is
// still running; PV reads P with a shared-memory descriptor (K-major, 128B swizzle).
// TMEM: S0 | S1 | O0 | O1 (512 columns at D=128). SMEM at D=128: Q 32K + K 2x32K + V 2x32K +
// P 2x32K; the lanes' final (max, sum) exchange reuses their P buffers.
// Register split via setmaxnreg within the CTA pool of 384 x 168: producer/MMA warpgroup 64,
// softmax warpgroups 216 (128*64 + 256*216 <= 384*168, else the increase never completes).
constexpr int kPPThreads = 384;
// mbarrier waits of the forward kernel: spin (try_wait re-polled after the system-dependent
// limit) or sleep (try_wait with a suspend-time hint)
// Pairs (e + 2, e + 3) of the softmax loop iterations e / 4 whose bit is set take the FMA-pipe
// exp2 polynomial instead of MUFU.EX2 (FA4-style offload of the exp unit). A/B at cfg3 (round 2,
// evenly interleaved): 0 / 8 / 16 / 24 polynomial pairs per row-tile: 24.7 / 25.0 / 25.5 / 26.1
// ms. The MUFU pipe is 64% busy but the lanes are dependency-latency-bound, so every extra
// instruction costs more than the exp-unit time it frees; all exps stay on MUFU.
#ifndef PSA_ATTN_POLY_MASK
#define PSA_ATTN_POLY_MASK 0x00000000u
#endif
constexpr uint32_t kPPPolyMask = PSA_ATTN_POLY_MASK;
#ifndef PSA_ATTN_SLEEP_SOFT
#define PSA_ATTN_SLEEP_SOFT 0
#endif
#ifndef PSA_ATTN_SLEEP_PROD
#define PSA_ATTN_SLEEP_PROD 0
#endif
#if PSA_ATTN_SLEEP_SOFT
#define PP_WAIT_SOFT(bar, par) mbar_wait_sleep(bar, par)
#else
#define PP_WAIT_SOFT(bar, par) mbar_wait(bar, par)
#endif
#if PSA_ATTN_SLEEP_PROD
#define PP_WAIT_PROD(bar, par) mbar_wait_sleep(bar, par)
#else
#define PP_WAIT_PROD(bar, par) mbar_wait(bar, par)
#endif


// PSA_ATTN_SHARED_P: one P buffer for both lanes (a lane stores P(t) once the other lane's
// PV(t-1) has read P(t-1)); the freed 32 KB give K a third stage at D = 128.
#ifndef PSA_ATTN_SHARED_P
#define PSA_ATTN_SHARED_P 0
#endif
constexpr bool kPPSharedP = PSA_ATTN_SHARED_P;
constexpr int kPPBufsP = kPPSharedP ? 1 : 2;
template <int D>
struct PP2Cfg {
  static constexpr int kKStages = D == 128 ? (kPPSharedP ? 3 : 2) : 3;
  static constexpr int kVStages = D == 128 ? 2 : 3;
  static constexpr int kAugStages = D == 128 ? 1 : 2;  // one 2 KB stage is all that fits at D=128
  static constexpr int kTileBytes = kTileRows * D * 2;
};

// The level bias enters S through the tensor core: S = [Q | Qa] [K | Ka]^T with one extra K=16
// step, Qa = (1, 1, 1, 0, ...) for every query row and Ka = (hi, mid, lo, 0, ...) of the key's
// bias (h-1)/scale_log2 (= (h-1) ln 2 after the softmax scale, exactly h-1 in the log2 domain)
// split into three bf16 terms (pad keys: -2^100). The softmax then works on
// raw S like dense attention (no per-column bias loads or adds; pad keys need no masking).
// Ka: no-swizzle K-major, 16 B per key (its second 8-column core matrix aliases the first: LBO = 0,
// matched by zeros in Qa's second core matrix); Qa: one core matrix broadcast to every row (SBO = 0).
template <int D>
struct PP2Smem {
  using C = PP2Cfg<D>;
  uint8_t q[kTileRows * D * 2];
  uint8_t k[C::kKStages][C::kTileBytes];
  uint8_t v[C::kVStages][C::kTileBytes];
  uint8_t p[kPPBufsP][kTileRows * kTileRows * 2];
  uint8_t kaug[C::kAugStages][kTileRows * 16];
  uint8_t qaug[256];
  uint32_t meta[kMetaRing][kChunks];
  uint64_t q_full;
  uint64_t k_full[C::kKStages], k_empty[C::kKStages];
  uint64_t v_full[C::kVStages], v_empty[C::kVStages];
  uint64_t aug_full[C::kAugStages], aug_empty[C::kAugStages];
  uint64_t meta_full[kMetaRing], meta_empty[kMetaRing];
  uint64_t s_full[2], s_free[2], p_full[2], o_done[2];
  uint32_t tmem_base;
};

// Optional clock64 trace (-DPSA_TRACE; scripts/probes/pp2_trace3.py): 8 CTAs spaced through the
// grid record per KV tile t < 256: 0 lane (t&1) starts waiting for S(t), 1 S(t) ready, 2 tile
// max done, 3 exp loop done, 4 P(t) stored and released, 5 S(t) issued, 6 PV(t) issued, 7 the MMA
// warp starts waiting for P(t), 8 K(t) TMA issued, 9 V(t) TMA issued, 10 segments (TMA boxes / 2)
// of K tile t (a count), 11 the MMA warp sees K(t) full, 12 ... s_free, 13 ... aug_full (the
// lanes' first warps, the MMA warp and the producers' lane 0).
#ifdef PSA_TRACE
__device__ long long g_pp2_trace[8][14][256];
#define PP2_TRACE(ev, t)                                                              \
  do {                                                                                \
    if (tslot >= 0 && (t) < 256) g_pp2_trace[tslot][ev][t] = clock64();               \
  } while (0)
#else
#define PP2_TRACE(ev, t) \
  do {                   \
  } while (0)
#endif

template <int D>
__global__ void __launch_bounds__(kPPThreads, 1)
    psa_attn_pp2_kernel(const __grid_constant__ AttnMaps maps, const AttnParams p,
                       const uint16_t* __restrict__ csr, const int32_t* __restrict__ info,
                       uint16_t* __restrict__ out, float* __restrict__ lse,
                       int32_t* __restrict__ skipped) {
  using C = PP2Cfg<D>;
  constexpr int KST = C::kKStages, VST = C::kVStages, AST = C::kAugStages;
  constexpr uint32_t kO0 = 256;  // O_L at kO0 + L * D
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<PP2Smem<D>*>(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = blockIdx.x;
#ifdef PSA_TRACE
  const int tstep = static_cast<int>(gridDim.x) / 8;
  const int tslot = (static_cast<int>(blockIdx.x) % tstep == tstep / 2) ? static_cast<int>(blockIdx.x) / tstep : -1;
#endif
  const int bhq = static_cast<int>(unit / p.n_qs);
  const int il = static_cast<int>(unit % p.n_qs);
  const int i = p.qblk != nullptr ? p.qblk[il] : il;
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
    for (int s = 0; s < AST; ++s) {
      mbar_init(&sm.aug_full[s], 1);
      mbar_init(&sm.aug_empty[s], 1);
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
    if (threadIdx.x < 16)  // Qa: core matrix 0 rows = (1, 1, 1, 0, 0, 0, 0, 0), core matrix 1 = 0
      reinterpret_cast<uint4*>(sm.qaug)[threadIdx.x] =
          threadIdx.x < 8 ? make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u) : make_uint4(0u, 0u, 0u, 0u);
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
          if (t >= KST) PP_WAIT_PROD(&sm.k_empty[ks], ((t / KST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.k_full[ks], static_cast<uint32_t>(sg.total) * D * 2);
          if (lane == 0) PP2_TRACE(8, t);
#ifdef PSA_TRACE
          if (lane == 0 && tslot >= 0 && t < 256) g_pp2_trace[tslot][10][t] = sg.nseg;
#endif
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
          if (t >= VST) PP_WAIT_PROD(&sm.v_empty[vs], ((t / VST) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.v_full[vs], static_cast<uint32_t>(sg.total) * D * 2);
          if (lane == 0) PP2_TRACE(9, t);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.v[sg.h - 1], &sm.v_full[vs],
                          sm.v[vs] + c * kTileRows * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 2) {
      // ============================================================ bias rows (Ka) + causal meta
      if (T > 0) {
        const int64_t q_lo = static_cast<int64_t>(i) * p.b_q;
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int as = t % AST;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= AST) PP_WAIT_PROD(&sm.aug_empty[as], ((t / AST) - 1) & 1);  // S(t - AST) done
          {  // lane owns keys 4 lane .. 4 lane + 3 (one segment: slots are >= 8 rows, aligned)
            int g = 0;
            for (int q = 1; q < sg.nseg; ++q)
              if (__shfl_sync(0xffffffffu, sg.off, q) <= 4 * lane) g = q;
            const int goff = __shfl_sync(0xffffffffu, sg.off, g);
            const int gL = __shfl_sync(0xffffffffu, sg.L, g);
            const int gh = __shfl_sync(0xffffffffu, sg.h, g);
            const int r0 = 4 * lane - goff;
            const bool in_tile = 4 * lane < sg.total;
            const uint4 live = make_uint4(p.aug[gh - 1][0], p.aug[gh - 1][1], 0u, 0u);
            const uint4 pad = make_uint4(kAugPad, 0u, 0u, 0u);
            uint4* row = reinterpret_cast<uint4*>(sm.kaug[as]) + 4 * lane;
#pragma unroll
            for (int e = 0; e < 4; ++e) row[e] = in_tile && r0 + e < gL ? live : pad;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.aug_full[as]);
          if (p.causal) {
            // per 8-key chunk: straddle flag, valid keys of the chunk (pad keys of a straddling
            // chunk are masked too, so a row with no visible key stays empty), first key position
            const int ms = t % kMetaRing;
            if (t >= kMetaRing) PP_WAIT_PROD(&sm.meta_empty[ms], ((t / kMetaRing) - 1) & 1);
            if (sg.fits) {
              const bool straddle = static_cast<int64_t>(sg.j + 1) * p.b_k - 1 > q_lo;
              for (int c = 0; c < sg.sz / 8; ++c) {
                const int nv = max(0, min(8, sg.L - 8 * c));
                sm.meta[ms][sg.off / 8 + c] = (straddle ? 1u : 0u) | (static_cast<uint32_t>(nv) << 1) |
                                              (static_cast<uint32_t>(sg.j * p.b_k + c * 8) << 5);
              }
            }
            if (lane < kChunks && 8 * lane >= sg.total) sm.meta[ms][lane] = 0u;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.meta_full[ms]);
          }
        }
      }
    } else {
      // ============================================================ MMA issuer (warp 1)
      if (T > 0) {
        constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
        const uint64_t q_desc0 = umma_desc_sw128(smem_u32(sm.q), 16, 1024);
        const uint64_t qa_desc = umma_desc_noswz(smem_u32(sm.qaug), 128, 0);
        auto issue_s = [&](int t) {
          const int ks = t % KST, as = t % AST, L = t & 1;
          PP_WAIT_PROD(&sm.k_full[ks], (t / KST) & 1);
          if (lane == 0) PP2_TRACE(11, t);
          if (t >= 2) PP_WAIT_PROD(&sm.s_free[L], ((t >> 1) - 1) & 1);  // lane read S(t-2)
          if (lane == 0) PP2_TRACE(12, t);
          PP_WAIT_PROD(&sm.aug_full[as], (t / AST) & 1);
          if (lane == 0) PP2_TRACE(13, t);
          tc_fence_after();
          const uint64_t k_desc0 = umma_desc_sw128(smem_u32(sm.k[ks]), 16, 1024);
          const uint64_t ka_desc = umma_desc_noswz(smem_u32(sm.kaug[as]), 0, 128);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ss(tmem + L * 128, q_desc0 + koff, k_desc0 + koff, idesc_s,
                          kk > 0 ? 1u : 0u);
            }
            mma_bf16_ss(tmem + L * 128, qa_desc, ka_desc, idesc_s, 1u);  // + level bias
            PP2_TRACE(5, t);
            mma_commit(&sm.k_empty[ks]);
            mma_commit(&sm.aug_empty[as]);
            mma_commit(&sm.s_full[L]);
          }
          __syncwarp();
        };
        auto issue_pv = [&](int t) {
          const int vs = t % VST, L = t & 1;
          PP_WAIT_PROD(&sm.v_full[vs], (t / VST) & 1);
          if (lane == 0) PP2_TRACE(7, t);
          PP_WAIT_PROD(&sm.p_full[L], (t >> 1) & 1);
          tc_fence_after();
          const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sm.v[vs]), kTileRows * 128, 1024);
          const uint64_t p_desc0 = umma_desc_sw128(smem_u32(sm.p[kPPSharedP ? 0 : L]), 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kTileRows / 16; ++kk) {
              const uint32_t poff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ss(tmem + kO0 + L * D, p_desc0 + poff, v_desc0 + ((kk * 16 * 128) >> 4),
                          idesc_o, (t >= 2 || kk > 0) ? 1u : 0u);
            }
            PP2_TRACE(6, t);
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
      const bool tr = wq == 0 && lane == 0;
      if (tr) PP2_TRACE(0, t);
      PP_WAIT_SOFT(&sm.s_full[L], (t >> 1) & 1);
      if (tr) PP2_TRACE(1, t);
      tc_fence_after();
      uint32_t s[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(t_s + c * 32, s[c]);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_wait(s[c]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.s_free[L]);  // S_L may take tile t+2 now
      // raw logits with the level bias already added by the tensor core (pad keys ~ -1.3e30)
      float y[128];
#pragma unroll
      for (int e = 0; e < 128; ++e) y[e] = __uint_as_float(s[e >> 5][e & 31]);
      if (p.causal) {  // token-level mask on straddling level-1 chunks (attention.py:88-108)
        PP_WAIT_SOFT(&sm.meta_full[ms], (t / kMetaRing) & 1);
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          const uint32_t w = sm.meta[ms][c];
          if (w & 1u) {
            const int lim = min(qpos - static_cast<int>(w >> 5), static_cast<int>((w >> 1) & 15u) - 1);
#pragma unroll
            for (int e = 0; e < 8; ++e) y[c * 8 + e] = (e <= lim) ? y[c * 8 + e] : -INFINITY;
          }
        }
        mbar_arrive(&sm.meta_empty[ms]);
      }

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
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
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
      if (tr) PP2_TRACE(2, t);
#pragma unroll
      for (int e = 0; e < 128; e += 4) {
        float2 a = ffma2(make_float2(y[e], y[e + 1]), scale2, negm);
        float2 c = ffma2(make_float2(y[e + 2], y[e + 3]), scale2, negm);
        a.x = ex2_approx(a.x);
        a.y = ex2_approx(a.y);
        if ((kPPPolyMask >> (e >> 2)) & 1u) {  // spread evenly: MUFU and FMA pipes overlap
          c = ex2_poly2(c);
        } else {
          c.x = ex2_approx(c.x);
          c.y = ex2_approx(c.y);
        }
        ls0 = fadd2(ls0, a);
        ls1 = fadd2(ls1, c);
        pk[e / 2] = pack_bf16x2(a.x, a.y);
        pk[e / 2 + 1] = pack_bf16x2(c.x, c.y);
      }
      if (tr) PP2_TRACE(3, t);
      const float2 ls = fadd2(ls0, ls1);
      l_run = l_run * alpha + (ls.x + ls.y);
      // PV(t-2) done: P_L is free and O_L is stable
      if (t >= 2) {
        PP_WAIT_SOFT(&sm.o_done[L], ((t >> 1) - 1) & 1);
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
      if (kPPSharedP && t >= 1) {  // the shared P buffer: the other lane's PV(t-1) has read it
        PP_WAIT_SOFT(&sm.o_done[L ^ 1], ((t - 1) >> 1) & 1);
        tc_fence_after();
      }
      {  // P (bf16) -> shared memory, UMMA K-major 128B-swizzled: [key half][row][128 B]
        uint8_t* prow = sm.p[kPPSharedP ? 0 : L] + row * 128;
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
      if (tr) PP2_TRACE(4, t);
    }

    // ---------------------------------------------------------------- merge + epilogue
    const int cnt0 = (T + 1) >> 1, cnt1 = T >> 1;  // tiles of lane 0 / lane 1
    const int cnt_me = L == 0 ? cnt0 : cnt1;
    if (kPPSharedP) {  // every PV has read the shared P buffer
      if (cnt0 > 0) mbar_wait(&sm.o_done[0], (cnt0 - 1) & 1);
      if (cnt1 > 0) mbar_wait(&sm.o_done[1], (cnt1 - 1) & 1);
    } else if (cnt_me > 0) {
      mbar_wait(&sm.o_done[L], (cnt_me - 1) & 1);  // P_L no longer read
    }
    constexpr int kRedStride = kPPSharedP ? 2 * kTileRows : kTileRows * kTileRows / 2;  // floats
    float* red = reinterpret_cast<float*>(sm.p[0]) + L * kRedStride;
    red[row] = m_run;
    red[kTileRows + row] = l_run;
    named_bar_sync(1, 2 * kTileRows);
    const float* red0 = reinterpret_cast<const float*>(sm.p[0]);
    const float* red1 = reinterpret_cast<const float*>(sm.p[0]) + kRedStride;
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
    const int64_t o_row =
        p.qblk != nullptr ? (static_cast<int64_t>(bhq) * p.n_qs + il) * p.b_q + row
        : p.out_rows == nullptr || !valid
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
// ------------------------------------------------------------------ host side
static uint32_t host_bf16_rne(double x) {  // finite x in bf16 range: fp32 then RNE to bf16
  const float f = static_cast<float>(x);
  uint32_t u;
  memcpy(&u, &f, 4);
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}
static double host_bf16_to_double(uint32_t b) {
  const uint32_t u = b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

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
                       const int32_t* qblk, int n_qs, cudaStream_t s) {
  AttnMaps maps;
  memset(&maps, 0, sizeof(maps));
  AttnParams p{};
  p.qblk = qblk;
  p.n_qs = n_qs;
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
  for (int h = 1; h <= levels; ++h) {  // bias (h-1)/scale_log2 as hi + mid + lo (bf16 terms)
    double r = (h - 1) / static_cast<double>(p.scale_log2);
    uint32_t t[3];
    for (int e = 0; e < 3; ++e) {
      t[e] = host_bf16_rne(r);
      r -= host_bf16_to_double(t[e]);
    }
    p.aug[h - 1][0] = t[0] | (t[1] << 16);
    p.aug[h - 1][1] = t[2];
  }
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
  const int64_t units = batch * hq * p.n_qs;
  const size_t smem2 = sizeof(PP2Smem<D>);
  auto kern2 = psa_attn_pp2_kernel<D>;
  cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2));
  kern2<<<static_cast<unsigned>(units), kPPThreads, smem2, s>>>(
      maps, p, csr, info, static_cast<uint16_t*>(out), lse, skipped);
  return psa_check_launch("psa_attn_pp2_kernel");
}


// ====================================================================== backward dQ (tcgen05)
// dQ of the multi-level attention for a fixed mask (psa_backward.cu has the derivation): the
// same work unit, plan walk and K/V producers as the forward, with
//   S = Q K^T and dP = dO V^T (SS MMAs into TMEM), P = exp2(S c + (h-1) - lse2) (lse known: no
//   running max), dS = P (dP - D) written back as bf16 pairs over the S columns it came from,
//   dQ += dS K with dS as the TMEM A operand (tcgen05.mma TS form; K read MN-major like V in the
//   forward's PV).
// Two softmax warpgroups split the 128 key columns of a tile (no cross-warp exchange is needed
// since the row statistics are final). TMEM: S0 | S1 | dP | dQ (512 columns at D = 128).
struct BwdQSmem {
  uint8_t q[kTileRows * 128 * 2];
  uint8_t dout[kTileRows * 128 * 2];
  uint8_t k[3][kTileRows * 128 * 2];  // K lives until dQ(t) has read it: one stage deeper than V
  uint8_t v[2][kTileRows * 128 * 2];
  float bias[kMetaRing][kTileRows];
  uint32_t meta[kMetaRing][kChunks];
  uint64_t q_full;
  uint64_t k_full[3], k_empty[3], v_full[2], v_empty[2];
  uint64_t meta_full[kMetaRing], meta_empty[kMetaRing];
  uint64_t s_full[2], sp_read, ds_full[2], dq_done;
  uint32_t tmem_base;
};

static_assert(sizeof(BwdQSmem) <= 227 * 1024, "dQ kernel shared memory exceeds the sm_100 limit");

struct BwdQMaps {
  AttnMaps a;  // q, k[], v[]
  CUtensorMap dout;
};

__global__ void __launch_bounds__(kPPThreads, 1)
    psa_bwd_dq_tc_kernel(const __grid_constant__ BwdQMaps maps, const AttnParams p,
                         const uint16_t* __restrict__ csr, const int32_t* __restrict__ info,
                         const float* __restrict__ lse, const float* __restrict__ drow,
                         float scale, uint16_t* __restrict__ dq) {
  constexpr int D = 128;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<BwdQSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit = blockIdx.x;
  const int bhq = static_cast<int>(unit / p.n_q);
  const int i = static_cast<int>(unit % p.n_q);
  const int b = bhq / p.hq, hh = bhq % p.hq;
  const int64_t bhkv = static_cast<int64_t>(b) * p.hkv + hh / (p.hq / p.hkv);
  const int n_ent = info[unit * 2 + 0];
  const int T = (info[unit * 2 + 1] + kTileRows - 1) / kTileRows;
  const int64_t q_row0 = static_cast<int64_t>(bhq) * p.n + static_cast<int64_t>(i) * p.b_q;
  constexpr uint32_t kDP = 256, kDQ = 384;

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < 3; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
      mbar_init(&sm.s_full[s], 1);
    }
    for (int s = 0; s < kMetaRing; ++s) {
      mbar_init(&sm.meta_full[s], 1);
      mbar_init(&sm.meta_empty[s], 8);  // one arrive per softmax warp
    }
    mbar_init(&sm.sp_read, 8);
    mbar_init(&sm.ds_full[0], 4);  // one per softmax warpgroup (key half)
    mbar_init(&sm.ds_full[1], 4);
    mbar_init(&sm.dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  {  // K/V rows past the last filled slot of a tile are read by the MMAs: keep them finite
    uint4* z = reinterpret_cast<uint4*>(&sm.k[0][0]);
    const int nvec = 5 * kTileRows * 128 * 2 / 16;  // k[3], v[2]
    for (int t = threadIdx.x; t < nvec; t += kPPThreads) z[t] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp < 4) {
    regs_dec<64>();
    if (warp == 0) {  // K producer (+ Q, dO)
      if (T > 0) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm.q_full, 2 * kTileRows * D * 2);
          for (int c = 0; c < D / 64; ++c) {
            tma_load_2d(&maps.a.q, &sm.q_full, sm.q + c * kTileRows * 128, c * 64,
                        static_cast<int>(q_row0));
            tma_load_2d(&maps.dout, &sm.q_full, sm.dout + c * kTileRows * 128, c * 64,
                        static_cast<int>(q_row0));
          }
        }
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int ks = t % 3;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= 3) mbar_wait(&sm.k_empty[ks], ((t / 3) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.k_full[ks], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.a.k[sg.h - 1], &sm.k_full[ks],
                          sm.k[ks] + c * kTileRows * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 3) {  // V producer
      if (T > 0) {
        PlanCursor pc;
        pc.init(csr + unit * p.n_k, n_ent, lane);
        for (int t = 0; t < T; ++t) {
          const int vs = t & 1;
          const TileSeg sg = pc.next(p, bhkv, lane);
          if (t >= 2) mbar_wait(&sm.v_empty[vs], ((t >> 1) - 1) & 1);
          if (lane == 0) mbar_arrive_expect_tx(&sm.v_full[vs], static_cast<uint32_t>(sg.total) * D * 2);
          __syncwarp();
          if (sg.fits)
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(&maps.a.v[sg.h - 1], &sm.v_full[vs],
                          sm.v[vs] + c * kTileRows * 128 + sg.off * 128, c * 64, sg.row);
        }
      }
    } else if (warp == 2) {  // bias / causal metadata (as in the forward)
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
    } else {  // MMA issuer (warp 1)
      if (T > 0) {
        constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_q = umma_idesc_bf16(128, D, false, true);
        const uint64_t q_desc0 = umma_desc_sw128(smem_u32(sm.q), 16, 1024);
        const uint64_t do_desc0 = umma_desc_sw128(smem_u32(sm.dout), 16, 1024);
        auto issue_sd = [&](int t) {  // S(t) = Q K^T into S[t & 1], dP(t) = dO V^T
          const int st = t & 1, kst = t % 3;
          mbar_wait(&sm.k_full[kst], (t / 3) & 1);
          mbar_wait(&sm.v_full[st], (t >> 1) & 1);
          tc_fence_after();
          const uint64_t k_desc0 = umma_desc_sw128(smem_u32(sm.k[kst]), 16, 1024);
          const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sm.v[st]), 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ss(tmem + st * 128, q_desc0 + koff, k_desc0 + koff, idesc_s,
                          kk > 0 ? 1u : 0u);
            }
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
              mma_bf16_ss(tmem + kDP, do_desc0 + koff, v_desc0 + koff, idesc_s,
                          kk > 0 ? 1u : 0u);
            }
            mma_commit(&sm.v_empty[st]);
            mma_commit(&sm.s_full[st]);
          }
          __syncwarp();
        };
        mbar_wait(&sm.q_full, 0);
        tc_fence_after();
        issue_sd(0);
        for (int t = 0; t < T; ++t) {
          const int st = t & 1;
          if (t + 1 < T) {
            mbar_wait(&sm.sp_read, t & 1);  // softmax read S(t) and dP(t)
            issue_sd(t + 1);
          }
          const uint64_t kmn_desc0 = umma_desc_sw128(smem_u32(sm.k[t % 3]), kTileRows * 128, 1024);
          // dS(t) (bf16 pairs) sits in S[t & 1]: key columns [64 g, 64 g + 64) packed into
          // [64 g, 64 g + 32); the A operand comes from tensor memory. Each key half goes to the
          // tensor core as soon as its warpgroup has packed it.
#pragma unroll
          for (int kh = 0; kh < 2; ++kh) {
            mbar_wait(&sm.ds_full[kh], t & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) {
                const int kk = 4 * kh + k4;
                const uint32_t acol = st * 128 + 64 * kh + k4 * 8;
                mma_bf16_ts(tmem + kDQ, tmem + acol, kmn_desc0 + ((kk * 16 * 128) >> 4), idesc_q,
                            (t > 0 || kk > 0) ? 1u : 0u);
              }
            }
            __syncwarp();
          }
          if (elect_one()) {
            mma_commit(&sm.k_empty[t % 3]);
            if (t + 1 == T) mma_commit(&sm.dq_done);
          }
          __syncwarp();
        }
      }
    }
  } else {
    regs_inc<216>();
    const int g = (warp - 4) >> 2;  // key columns [64 g, 64 g + 64)
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int qpos = i * p.b_q + row;
    const bool valid = row < p.b_q;
    const float l = valid ? lse[q_row0 + row] : -INFINITY;
    const bool live = l != -INFINITY;
    // -lse log2(e), -inf for a masked row: exp2 gives P = 0 without a per-column select
    const float nl2 = live ? -l * 1.4426950408889634f : -INFINITY;
    const float2 nl22 = make_float2(nl2, nl2);
    const float dd = valid ? drow[q_row0 + row] : 0.f;
    const float2 ndd2 = make_float2(-dd, -dd);
    const float2 scale2 = make_float2(p.scale_log2, p.scale_log2);
    for (int t = 0; t < T; ++t) {
      const int st = t & 1, ms = t % kMetaRing;
      mbar_wait(&sm.s_full[st], (t >> 1) & 1);
      tc_fence_after();
      uint32_t sv[2][32], pv[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) tmem_ld32(t_lane + st * 128 + 64 * g + c * 32, sv[c]);
#pragma unroll
      for (int c = 0; c < 2; ++c) tmem_ld32(t_lane + kDP + 64 * g + c * 32, pv[c]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tmem_ld_wait(sv[c]);
        tmem_ld_wait(pv[c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.sp_read);
      mbar_wait(&sm.meta_full[ms], (t / kMetaRing) & 1);
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 64; e += 2) {
        const int col = 64 * g + e;
        const float* x = reinterpret_cast<const float*>(&sv[e >> 5][e & 31]);
        const float* y = reinterpret_cast<const float*>(&pv[e >> 5][e & 31]);
        const float2 bv = *reinterpret_cast<const float2*>(&sm.bias[ms][col]);
        float2 a = ffma2(make_float2(x[0], x[1]), scale2, bv);
        a = fadd2(a, nl22);
        float p0 = ex2_approx(a.x), p1 = ex2_approx(a.y);
        if (p.causal) {
          const uint32_t w = sm.meta[ms][col >> 3];
          if (w & 1u) {
            const int kp = static_cast<int>(w >> 1) + (col & 7);
            if (kp > qpos) p0 = 0.f;
            if (kp + 1 > qpos) p1 = 0.f;
          }
        }
        const float2 ds = fmul2(make_float2(p0, p1), fadd2(make_float2(y[0], y[1]), ndd2));
        pk[e >> 1] = pack_bf16x2(ds.x, ds.y);
      }
      if (lane == 0) mbar_arrive(&sm.meta_empty[ms]);
      // dS (bf16 pairs) over this warpgroup's (already read) S columns: the dQ MMA's A operand.
      // S[t & 1] is next written by S(t + 2), which the MMA warp issues after dQ(t).
      tmem_st32(t_lane + st * 128 + 64 * g, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.ds_full[g]);
    }
    if (T > 0) {
      mbar_wait(&sm.dq_done, 0);
      tc_fence_after();
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t o[32];
      if (T > 0) {
        tmem_ld32(t_lane + kDQ + 64 * g + c * 32, o);
        tmem_ld_wait(o);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0u;
      }
      if (valid) {
        uint16_t* orow = dq + (q_row0 + row) * D + 64 * g + c * 32;
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          uint32_t w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            w[u] = pack_bf16x2(__uint_as_float(o[v4 * 8 + 2 * u]) * scale,
                               __uint_as_float(o[v4 * 8 + 2 * u + 1]) * scale);
          *reinterpret_cast<uint4*>(orow + v4 * 8) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int attn_bwd_dq_tc(const void* q, const void* k, const void* v, const void* k_pyr,
                   const void* v_pyr, const void* dout, const float* lse, const float* drow,
                   int64_t batch, int hq, int hkv, int64_t n, int b_q, int b_k, int levels,
                   const uint16_t* csr, const int32_t* info, int causal, void* dq,
                   cudaStream_t s) {
  constexpr int D = 128;
  BwdQMaps maps;
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
  const int64_t bhkv = batch * hkv;
  int rc = encode_2d(&maps.a.q, q, static_cast<uint64_t>(batch * hq * n), D, kTileRows);
  if (rc) return rc;
  rc = encode_2d(&maps.dout, dout, static_cast<uint64_t>(batch * hq * n), D, kTileRows);
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
    rc = encode_2d(&maps.a.k[h - 1], kb, rows, D, sz);
    if (rc) return rc;
    rc = encode_2d(&maps.a.v[h - 1], vb, rows, D, sz);
    if (rc) return rc;
  }
  const size_t smem = sizeof(BwdQSmem);
  cudaFuncSetAttribute(psa_bwd_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  psa_bwd_dq_tc_kernel<<<static_cast<unsigned>(batch * hq * p.n_q), kPPThreads, smem, s>>>(
      maps, p, csr, info, lse, drow, static_cast<float>(1.0 / sqrt(static_cast<double>(D))),
      static_cast<uint16_t*>(dq));
  return psa_check_launch("psa_bwd_dq_tc_kernel");
}


// ====================================================================== backward dK/dV (tcgen05)
// One CTA per (KV head, KV block j), as the mma.sync version in psa_backward.cu: the CTA lists
// (level-major) the (query head, query block) entries that selected block j; per level the
// pooled block K_h / V_h is one TMA tile (box = slot rows), and per entry
//   S^T = K_h Q^T and dP^T = V_h dO^T (SS MMAs, pooled keys as M = 128 TMEM lanes),
//   P'^T = exp2(S^T c - lse2) (unbiased: the raw-row gradient is the duplicate's, see
//   psa_backward.cu), dS^T = P'^T (dP^T - D) -> shared memory (128B-swizzled, queries as K),
//   dV_h += P'^T dO and dK_h += dS^T Q (dO / Q read MN-major like V in the forward) in TMEM.
// At the end of a level the pooled rows are spread over their 2^(h-1) raw rows into the CTA's
// fp32 scratch rows; the last step writes bf16 dK (x scale) and dV. TMEM: S^T | dP^T | dV | dK.
// dK/dV work unit: up to kDkvUnitBlocks KV blocks of one level packed into one tile
// (2^(h-1) blocks of L = b_k >> (h-1) rows at level h, capped at 16 so that the per-entry block
// mask fits its 16 bits for every level up to kMaxLevels).
constexpr int kDkvUnitBlocks = 16;
__host__ __device__ inline int dkv_unit_blocks(int h) {
  return (1 << (h - 1)) < kDkvUnitBlocks ? (1 << (h - 1)) : kDkvUnitBlocks;
}
__host__ __device__ inline int dkv_level_units(int n_k, int h) {
  const int f = dkv_unit_blocks(h);
  return (n_k + f - 1) / f;
}

struct BwdKVSmem {
  uint8_t kt[kTileRows * 128 * 2];
  uint8_t vt[kTileRows * 128 * 2];
  uint8_t q[2][kTileRows * 128 * 2];     // double-buffered per entry
  uint8_t dout[2][kTileRows * 128 * 2];
  float nl2[2][kTileRows];  // -lse log2(e) / D of the entry's query rows (double-buffered)
  float dd[2][kTileRows];
  uint64_t kv_full, q_full[2], q_free[2], s_full[2], pds_full[4], acc_done;
  uint32_t tmem_base;
  int n_ent;
  int warp_cnt[kPPThreads / 32];
};

// One CTA per (KV head, level h, unit u). A unit is the f = 2^(h-1) neighbouring KV blocks
// [u f, u f + f) whose level-h pooled rows (L = b_k >> (h-1) each) fill one tile of f L = b_k rows,
// so every level keeps the M = 128 MMAs full. The entries are the (query head, query block) pairs
// that selected at least one of the unit's blocks at level h, each with an f-bit row mask; rows of
// blocks the entry did not select at h get P = dS = 0. The unit writes its pooled dK / dV rows
// (fp32, unscaled) to the level-h slab of the scratch; bwd_unpool_kernel sums the levels per raw row.
__global__ void __launch_bounds__(kPPThreads, 1)
    psa_bwd_dkv_tc_kernel(const __grid_constant__ BwdQMaps maps, const AttnParams p,
                          const int8_t* __restrict__ level_map, const float* __restrict__ nl2,
                          const float* __restrict__ drow, int cap, float* __restrict__ scratch,
                          int64_t bkv_total) {
  constexpr int D = 128;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<BwdKVSmem*>(smem_raw);
  uint32_t* ents = reinterpret_cast<uint32_t*>(smem_raw + sizeof(BwdKVSmem));
  uint16_t* emask = reinterpret_cast<uint16_t*>(ents + cap);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bkv = blockIdx.y;
  const int b = static_cast<int>(bkv / p.hkv), hk = static_cast<int>(bkv % p.hkv);
  const int group = p.hq / p.hkv;
  const int span = group * p.n_q;
  // blockIdx.x -> (level h, unit u): level h has ceil(n_k / 2^(h-1)) units
  int h = 1, u = blockIdx.x;
  int64_t slab = 0;  // pooled rows of the levels before h (scratch slab offset, per KV head)
  while (u >= dkv_level_units(p.n_k, h)) {
    u -= dkv_level_units(p.n_k, h);
    slab += p.n >> (h - 1);
    ++h;
  }
  const int f = dkv_unit_blocks(h);
  const int L = p.b_k >> (h - 1);
  const int j0 = u * f;
  const int nb = min(f, p.n_k - j0);  // blocks in this unit
  const int64_t n_h = p.n >> (h - 1);
  const int rows_u = nb * L;          // pooled rows owned by this unit
  constexpr uint32_t kST = 0, kDPT = 128, kDV = 256, kDK = 384;

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    mbar_init(&sm.kv_full, 1);
    for (int w = 0; w < 2; ++w) {
      mbar_init(&sm.q_full[w], 1);
      mbar_init(&sm.q_free[w], 1);
      mbar_init(&sm.s_full[w], 1);   // query halves: one per softmax warpgroup
      mbar_init(&sm.pds_full[2 * w], 4);  // (half, 32-query chunk)
      mbar_init(&sm.pds_full[2 * w + 1], 4);
    }
    mbar_init(&sm.acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  {  // tile rows never written by a TMA box are read by the MMAs: keep them finite
    uint4* z = reinterpret_cast<uint4*>(sm.kt);
    const int nvec = 2 * kTileRows * 128 * 2 / 16;  // pooled K / V tiles
    for (int t = threadIdx.x; t < nvec; t += kPPThreads) z[t] = make_uint4(0, 0, 0, 0);
    for (int t = threadIdx.x; t < 2 * kTileRows; t += kPPThreads) {  // rows >= b_q: P = dS = 0
      (&sm.nl2[0][0])[t] = -INFINITY;
      (&sm.dd[0][0])[t] = 0.f;
    }
    fence_proxy_async_smem();
  }
  // ---- deterministic list of the entries that selected any block of the unit at level h
  int total = 0;
  for (int base = 0; base < span; base += kPPThreads) {
    const int x = base + threadIdx.x;
    uint32_t m16 = 0;
    if (x < span) {
      const int g = x / p.n_q, iq = x % p.n_q;
      const int64_t bhq = static_cast<int64_t>(b) * p.hq + hk * group + g;
      const int8_t* lm = level_map + (bhq * p.n_q + iq) * p.n_k + j0;
      for (int t = 0; t < nb; ++t) m16 |= (lm[t] == h ? 1u : 0u) << t;
    }
    const bool hit = m16 != 0;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) sm.warp_cnt[warp] = __popc(m);
    __syncthreads();
    int before = 0, all = 0;
    for (int w = 0; w < kPPThreads / 32; ++w) {
      before += w < warp ? sm.warp_cnt[w] : 0;
      all += sm.warp_cnt[w];
    }
    if (hit) {
      const int slot = total + before + __popc(m & ((1u << lane) - 1u));
      if (slot < cap) {
        ents[slot] = static_cast<uint32_t>(x);
        emask[slot] = static_cast<uint16_t>(m16);
      }
    }
    total += all;
    __syncthreads();
  }
  if (threadIdx.x == 0) sm.n_ent = min(total, cap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int n_ent = sm.n_ent;
  // level-h slab of this KV head: pooled rows [j0 L, j0 L + rows_u)
  const int64_t prow0 = bkv * (2 * p.n) + slab + static_cast<int64_t>(j0) * L;
  float* sk = scratch + prow0 * D;
  float* sv = scratch + (bkv_total * 2 * p.n + prow0) * D;

  if (warp < 4) {
    regs_dec<72>();  // 128 x 72 + 256 x 216 = 384 x 168
    if (warp == 0 && n_ent > 0) {  // producer: the unit's pooled K/V once, Q / dO / lse / D per entry
      const bool bulk_rows = p.b_q % 4 == 0 && p.n % 4 == 0;
      int sz = 8;
      while (sz < L) sz <<= 1;
      const int row = static_cast<int>(bkv * n_h + static_cast<int64_t>(j0) * L);
      if (lane == 0) {
        const int nbox = (rows_u + sz - 1) / sz;
        mbar_arrive_expect_tx(&sm.kv_full, 2u * nbox * sz * D * 2);
        for (int bx = 0; bx < nbox; ++bx)
          for (int c = 0; c < D / 64; ++c) {
            const int off = c * kTileRows * 128 + bx * sz * 128;
            tma_load_2d(&maps.a.k[h - 1], &sm.kv_full, sm.kt + off, c * 64, row + bx * sz);
            tma_load_2d(&maps.a.v[h - 1], &sm.kv_full, sm.vt + off, c * 64, row + bx * sz);
          }
      }
      for (int e = 0; e < n_ent; ++e) {
        const int qb = e & 1;
        if (e >= 2) mbar_wait(&sm.q_free[qb], ((e >> 1) - 1) & 1);  // entry e-2 done
        const int x = static_cast<int>(ents[e]);
        const int g = x / p.n_q, iq = x % p.n_q;
        const int64_t bhq = static_cast<int64_t>(b) * p.hq + hk * group + g;
        const int64_t q_row0 = bhq * p.n + static_cast<int64_t>(iq) * p.b_q;
        if (!bulk_rows)
          for (int r = lane; r < p.b_q; r += 32) {
            sm.nl2[qb][r] = nl2[q_row0 + r];
            sm.dd[qb][r] = drow[q_row0 + r];
          }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm.q_full[qb], 2u * kTileRows * D * 2 + (bulk_rows ? 8u * p.b_q : 0u));
          if (bulk_rows) {  // lse / D rows ride the same transaction (no serial global loads)
            bulk_load_1d(sm.nl2[qb], nl2 + q_row0, 4u * p.b_q, &sm.q_full[qb]);
            bulk_load_1d(sm.dd[qb], drow + q_row0, 4u * p.b_q, &sm.q_full[qb]);
          }
          for (int c = 0; c < D / 64; ++c) {
            tma_load_2d(&maps.a.q, &sm.q_full[qb], sm.q[qb] + c * kTileRows * 128, c * 64,
                        static_cast<int>(q_row0));
            tma_load_2d(&maps.dout, &sm.q_full[qb], sm.dout[qb] + c * kTileRows * 128, c * 64,
                        static_cast<int>(q_row0));
          }
        }
      }
    } else if (warp == 1 && n_ent > 0) {  // MMA issuer
      // Two query halves ping-pong with the softmax warpgroups: while one half's P'^T / dS^T
      // is being formed, the tensor core runs the other half's dV / dK and the next entry's S^T.
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
      const uint64_t kt_desc = umma_desc_sw128(smem_u32(sm.kt), 16, 1024);
      const uint64_t vt_desc = umma_desc_sw128(smem_u32(sm.vt), 16, 1024);
      auto issue_s = [&](int e, int half) {  // S^T / dP^T of queries [64 half, 64 half + 64)
        const int qb = e & 1;
        const uint64_t q_desc = umma_desc_sw128(smem_u32(sm.q[qb]), 16, 1024) + ((half * 64 * 128) >> 4);
        const uint64_t do_desc =
            umma_desc_sw128(smem_u32(sm.dout[qb]), 16, 1024) + ((half * 64 * 128) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
            mma_bf16_ss(tmem + kST + 64 * half, kt_desc + koff, q_desc + koff, idesc_s, kk > 0 ? 1u : 0u);
          }
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = ((kk >> 2) * kTileRows * 128 + (kk & 3) * 32) >> 4;
            mma_bf16_ss(tmem + kDPT + 64 * half, vt_desc + koff, do_desc + koff, idesc_s,
                        kk > 0 ? 1u : 0u);
          }
          mma_commit(&sm.s_full[half]);
        }
        __syncwarp();
      };
      // dV += P'^T dO, dK += dS^T Q over the 32 queries of (half, chunk)
      auto issue_acc = [&](int e, int half, int chunk, bool zero) {
        const int qb = e & 1;
        const uint64_t q_mn = umma_desc_sw128(smem_u32(sm.q[qb]), kTileRows * 128, 1024);
        const uint64_t do_mn = umma_desc_sw128(smem_u32(sm.dout[qb]), kTileRows * 128, 1024);
        if (elect_one()) {
          // P'^T / dS^T (bf16 pairs) sit in the first 32 S^T / dP^T columns of the half
#pragma unroll
          for (int k2 = 0; k2 < 2; ++k2) {
            const int kk = 2 * chunk + k2;
            const uint32_t boff = ((half * 64 + kk * 16) * 128) >> 4;
            const uint32_t acc = (zero && k2 == 0) ? 0u : 1u;
            mma_bf16_ts(tmem + kDV, tmem + kST + 64 * half + kk * 8, do_mn + boff, idesc_o, acc);
            mma_bf16_ts(tmem + kDK, tmem + kDPT + 64 * half + kk * 8, q_mn + boff, idesc_o, acc);
          }
        }
        __syncwarp();
      };
      mbar_wait(&sm.kv_full, 0);
      mbar_wait(&sm.q_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(0, 1);
      for (int e = 0; e < n_ent; ++e) {
        const bool more = e + 1 < n_ent;
        mbar_wait(&sm.pds_full[0], e & 1);
        tc_fence_after();
        issue_acc(e, 0, 0, e == 0);
        mbar_wait(&sm.pds_full[1], e & 1);
        tc_fence_after();
        issue_acc(e, 0, 1, false);
        if (more) {
          mbar_wait(&sm.q_full[(e + 1) & 1], ((e + 1) >> 1) & 1);
          tc_fence_after();
          issue_s(e + 1, 0);
        }
        mbar_wait(&sm.pds_full[2], e & 1);
        tc_fence_after();
        issue_acc(e, 1, 0, false);
        mbar_wait(&sm.pds_full[3], e & 1);
        tc_fence_after();
        issue_acc(e, 1, 1, false);
        if (elect_one()) {
          mma_commit(&sm.q_free[e & 1]);
          if (!more) mma_commit(&sm.acc_done);
        }
        __syncwarp();
        if (more) issue_s(e + 1, 1);
      }
    }
  } else {
    regs_inc<216>();
    const int g = (warp - 4) >> 2;  // query columns [64 g, 64 g + 64); d columns at the end
    const int wq = warp & 3;
    const int row = wq * 32 + lane;  // pooled key row of the unit (TMEM lane)
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const float2 scale2 = make_float2(p.scale_log2, p.scale_log2);
    const int blk = row / L;  // block of the unit this row belongs to
    for (int e = 0; e < n_ent; ++e) {
      mbar_wait(&sm.s_full[g], e & 1);
      tc_fence_after();
      const int iq = static_cast<int>(ents[e]) % p.n_q;
      const bool live = blk < nb && ((emask[e] >> blk) & 1u);
      const int qb = e & 1;
      // nl2 / D rows of this entry: acquire them from their own transaction (already complete,
      // since S^T read the Q tile of the same phase), not only through the MMA warp's commit
      mbar_wait(&sm.q_full[qb], (e >> 1) & 1);
      const bool straddle =  // causal diagonal blocks are always level 1 (f = 1)
          p.causal && h == 1 && static_cast<int64_t>(j0 + 1) * p.b_k - 1 > static_cast<int64_t>(iq) * p.b_q;
      const int kpos = j0 * p.b_k + row;
      const int qpos0 = iq * p.b_q + 64 * g;
      // rows of blocks this entry did not select at h: exp2(-inf) = 0 through the additive term
      const float kill = live ? 0.f : -INFINITY;
      const float2 kill2 = make_float2(kill, kill);
      uint32_t sva[32], dva[32], svb[32], dvb[32];  // both 32-query chunks in flight at once
      tmem_ld32(t_lane + kST + 64 * g, sva);
      tmem_ld32(t_lane + kDPT + 64 * g, dva);
      tmem_ld32(t_lane + kST + 64 * g + 32, svb);
      tmem_ld32(t_lane + kDPT + 64 * g + 32, dvb);
      tmem_ld_wait(sva);
      tmem_ld_wait(dva);
      tmem_ld_wait(svb);
      tmem_ld_wait(dvb);
#pragma unroll
      for (int c = 0; c < 2; ++c) {  // each chunk is handed to the MMA warp as soon as it is packed
        uint32_t (&sv2)[32] = c == 0 ? sva : svb;
        uint32_t (&dv2)[32] = c == 0 ? dva : dvb;
        uint32_t pp[16], sp[16];
#pragma unroll
        for (int e2 = 0; e2 < 32; e2 += 2) {
          const int cl = c * 32 + e2;  // column within this warpgroup's 64
          const int col = 64 * g + cl;
          const float2 nl = *reinterpret_cast<const float2*>(&sm.nl2[qb][col]);
          const float2 d2 = *reinterpret_cast<const float2*>(&sm.dd[qb][col]);
          const float2 a = ffma2(make_float2(__uint_as_float(sv2[e2]), __uint_as_float(sv2[e2 + 1])),
                                 scale2, fadd2(nl, kill2));
          float p0 = ex2_approx(a.x), p1 = ex2_approx(a.y);
          if (straddle) {  // causal diagonal block (warp-uniform, rare)
            if (kpos > qpos0 + cl) p0 = 0.f;
            if (kpos > qpos0 + cl + 1) p1 = 0.f;
          }
          pp[e2 >> 1] = pack_bf16x2(p0, p1);
          sp[e2 >> 1] = pack_bf16x2(p0 * (__uint_as_float(dv2[e2]) - d2.x),
                                    p1 * (__uint_as_float(dv2[e2 + 1]) - d2.y));
        }
        // P'^T / dS^T as bf16 pairs over already-read columns: chunk c -> [64 g + 16 c, + 16)
        tmem_st16(t_lane + kST + 64 * g + 16 * c, pp);
        tmem_st16(t_lane + kDPT + 64 * g + 16 * c, sp);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.pds_full[2 * g + c]);
      }
    }
    // ---- the unit's pooled rows -> the level-h slab (zeros when no entry selected them)
    if (n_ent > 0) {
      mbar_wait(&sm.acc_done, 0);
      tc_fence_after();
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t ok[32], ov[32];
      if (n_ent > 0) {
        tmem_ld32(t_lane + kDK + 64 * g + c * 32, ok);
        tmem_ld32(t_lane + kDV + 64 * g + c * 32, ov);
        tmem_ld_wait(ok);
        tmem_ld_wait(ov);
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t) ok[t] = ov[t] = 0u;
      }
      if (row < rows_u) {
        float4* pk4 = reinterpret_cast<float4*>(sk + static_cast<int64_t>(row) * D + 64 * g + c * 32);
        float4* pv4 = reinterpret_cast<float4*>(sv + static_cast<int64_t>(row) * D + 64 * g + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          pk4[q4] = make_float4(__uint_as_float(ok[4 * q4]), __uint_as_float(ok[4 * q4 + 1]),
                                __uint_as_float(ok[4 * q4 + 2]), __uint_as_float(ok[4 * q4 + 3]));
          pv4[q4] = make_float4(__uint_as_float(ov[4 * q4]), __uint_as_float(ov[4 * q4 + 1]),
                                __uint_as_float(ov[4 * q4 + 2]), __uint_as_float(ov[4 * q4 + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// dK / dV of raw row r = sum over levels of the level's pooled gradient row r >> (h-1) (the
// duplicate identity, psa_backward.cu header); dK takes the softmax scale. One thread per 4 columns.
__global__ void bwd_unpool_kernel(const float* __restrict__ scratch, int64_t bkv_total, int64_t n,
                                  int levels, float scale, uint16_t* __restrict__ dk,
                                  uint16_t* __restrict__ dv) {
  constexpr int D = 128;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= bkv_total * n * (D / 4)) return;
  const int c = static_cast<int>(t % (D / 4)) * 4;
  const int64_t rr = t / (D / 4);
  const int64_t bkv = rr / n, r = rr % n;
  const float* sk = scratch + bkv * (2 * n) * D;
  const float* sv = scratch + (bkv_total + bkv) * (2 * n) * D;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), w = a;
  int64_t slab = 0;
  for (int h = 1; h <= levels; ++h) {
    const int64_t pr = (slab + (r >> (h - 1))) * D + c;
    const float4 x = *reinterpret_cast<const float4*>(sk + pr);
    const float4 y = *reinterpret_cast<const float4*>(sv + pr);
    a = make_float4(a.x + x.x, a.y + x.y, a.z + x.z, a.w + x.w);
    w = make_float4(w.x + y.x, w.y + y.y, w.z + y.z, w.w + y.w);
    slab += n >> (h - 1);
  }
  uint2 ok, ov;
  ok.x = pack_bf16x2(a.x * scale, a.y * scale);
  ok.y = pack_bf16x2(a.z * scale, a.w * scale);
  ov.x = pack_bf16x2(w.x, w.y);
  ov.y = pack_bf16x2(w.z, w.w);
  *reinterpret_cast<uint2*>(dk + rr * D + c) = ok;
  *reinterpret_cast<uint2*>(dv + rr * D + c) = ov;
}

int attn_bwd_dkv_tc(const void* q, const void* k, const void* v, const void* k_pyr,
                    const void* v_pyr, const void* dout, const float* lse, const float* drow,
                    int64_t batch, int hq, int hkv, int64_t n, int b_q, int b_k, int levels,
                    const int8_t* level_map, int causal, const float* nl2, float* scratch,
                    void* dk, void* dv, cudaStream_t s) {
  constexpr int D = 128;
  BwdQMaps maps;
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
  const int64_t bhkv = batch * hkv;
  int rc = encode_2d(&maps.a.q, q, static_cast<uint64_t>(batch * hq * n), D, kTileRows);
  if (rc) return rc;
  rc = encode_2d(&maps.dout, dout, static_cast<uint64_t>(batch * hq * n), D, kTileRows);
  if (rc) return rc;
  int64_t off_elems = 0;
  int units = 0;
  for (int h = 1; h <= levels; ++h) {
    const int L = b_k >> (h - 1);
    int sz = 8;
    while (sz < L) sz <<= 1;
    const uint64_t rows = static_cast<uint64_t>(bhkv * (n >> (h - 1)));
    const void* kb = h == 1 ? k : static_cast<const void*>(static_cast<const uint16_t*>(k_pyr) + off_elems);
    const void* vb = h == 1 ? v : static_cast<const void*>(static_cast<const uint16_t*>(v_pyr) + off_elems);
    if (h > 1) off_elems += static_cast<int64_t>(rows) * D;
    rc = encode_2d(&maps.a.k[h - 1], kb, rows, D, sz);
    if (rc) return rc;
    rc = encode_2d(&maps.a.v[h - 1], vb, rows, D, sz);
    if (rc) return rc;
    units += dkv_level_units(p.n_k, h);
  }
  const int cap = (hq / hkv) * p.n_q;
  const size_t smem = sizeof(BwdKVSmem) + static_cast<size_t>(cap) * 6;
  if (smem > 227 * 1024) return psa_fail(PSA_EINVAL, "too many query blocks per KV head for the backward kernel");
  cudaFuncSetAttribute(psa_bwd_dkv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  psa_bwd_dkv_tc_kernel<<<dim3(static_cast<unsigned>(units), static_cast<unsigned>(bhkv)),
                          kPPThreads, smem, s>>>(maps, p, level_map, nl2, drow, cap, scratch, bhkv);
  rc = psa_check_launch("psa_bwd_dkv_tc_kernel");
  if (rc) return rc;
  const int64_t threads = bhkv * n * (D / 4);
  bwd_unpool_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
      scratch, bhkv, n, levels, static_cast<float>(1.0 / sqrt(static_cast<double>(D))),
      static_cast<uint16_t*>(dk), static_cast<uint16_t*>(dv));
  return psa_check_launch("bwd_unpool_kernel");
}

}  // namespace psa

using namespace psa;

static int attn_fwd_impl(const void* q, const void* k, const void* v, const void* k_pyr,
                         const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n, int d,
                         int b_q, int b_k, int levels, const uint16_t* plan_csr,
                         const int32_t* plan_info, int causal, void* out, float* lse,
                         int32_t* skipped_rows, const int64_t* out_rows, const int32_t* qblk,
                         int n_qs, void* stream) {
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
  PSA_CHECK_ARG(n_qs >= 1 && n_qs <= n / b_q, "query-block count outside 1..n_q");
  PSA_CHECK_ARG(qblk != nullptr || n_qs == n / b_q, "a query-block subset needs its block list");
  PSA_CHECK_ARG(qblk == nullptr || out_rows == nullptr,
                "the output row scatter and query-block subsets are exclusive");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (d == 128)
    return launch_attn<128>(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, b_q, b_k, levels, plan_csr,
                            plan_info, causal, out, lse, skipped_rows, out_rows, qblk, n_qs, s);
  return launch_attn<64>(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, b_q, b_k, levels, plan_csr,
                         plan_info, causal, out, lse, skipped_rows, out_rows, qblk, n_qs, s);
}

extern "C" int psa_attn_fwd_scatter(const void* q, const void* k, const void* v,
                                    const void* k_pyr, const void* v_pyr, int64_t batch, int hq,
                                    int hkv, int64_t n, int d, int b_q, int b_k, int levels,
                                    const uint16_t* plan_csr, const int32_t* plan_info, int causal,
                                    void* out, float* lse, int32_t* skipped_rows,
                                    const int64_t* out_rows, void* stream) {
  PSA_CHECK_ARG(b_q >= 1 && n % b_q == 0, "layout does not divide seq_len");
  return attn_fwd_impl(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, d, b_q, b_k, levels, plan_csr,
                       plan_info, causal, out, lse, skipped_rows, out_rows, nullptr,
                       static_cast<int>(n / b_q), stream);
}

extern "C" int psa_attn_fwd_rows(const void* q, const void* k, const void* v, const void* k_pyr,
                                 const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n,
                                 int d, int b_q, int b_k, int levels, const uint16_t* plan_csr,
                                 const int32_t* plan_info, int causal, const int32_t* qblk,
                                 int n_qsel, void* out, float* lse, int32_t* skipped_rows,
                                 void* stream) {
  PSA_CHECK_ARG(qblk != nullptr, "null query-block list");
  return attn_fwd_impl(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, d, b_q, b_k, levels, plan_csr,
                       plan_info, causal, out, lse, skipped_rows, nullptr, qblk, n_qsel, stream);
}

extern "C" int psa_attn_fwd(const void* q, const void* k, const void* v, const void* k_pyr,
                            const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n, int d,
                            int b_q, int b_k, int levels, const uint16_t* plan_csr,
                            const int32_t* plan_info, int causal, void* out, float* lse,
                            int32_t* skipped_rows, void* stream) {
  return psa_attn_fwd_scatter(q, k, v, k_pyr, v_pyr, batch, hq, hkv, n, d, b_q, b_k, levels,
                              plan_csr, plan_info, causal, out, lse, skipped_rows, nullptr, stream);
}

#ifdef PSA_TRACE
// Copies the forward kernel's clock64 trace (8 x 14 x 256 int64) to host memory.
extern "C" int psa_debug_pp2_trace(long long* host) {
  return cudaMemcpyFromSymbol(host, psa::g_pp2_trace, sizeof(psa::g_pp2_trace)) == cudaSuccess ? 0 : 1;
}
#endif
