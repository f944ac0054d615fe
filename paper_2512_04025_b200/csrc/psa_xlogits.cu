// Exact fp64 importance logits on the int8 tensor cores (tcgen05 kind::i8), for K2/K2b.
//
// Both estimators of pkg/src/pyrattn/importance.py need fp64 logits of bf16 rows:
//   importance_sampled      :52-85   fl(dot(q_a, k_b) / sqrt(d)) over sampled rows
//   importance_antidiagonal :97-132  fl(dot(q_p, k_c) * fl(1/sqrt(d))) over strided picks
// A dot product of bf16 vectors is an exact sum of 16-bit products, so BLAS (and the DMMA
// kernels in psa_importance.cu) return it exactly whenever it fits in 53 bits. The FP64 pipe is
// ~36 TFLOP/s; the int8 tensor cores are ~120x faster, so we compute the SAME exact value with
// integer arithmetic (an Ozaki-style split):
//
//   every gathered row x is put on the grid 2^(E-27), E = floor(log2 max|x|):
//     x = X * 2^(E-27) + r,  X integer, |X| < 2^28,  r = 0 unless |x_k| < 2^(E-20) ("tiny")
//   X = d3 * 2^21 + d2 * 2^14 + d1 * 2^7 + d0, int8 digits (d0..d2 in [0, 127], d3 signed)
//   dot(X, Y) = sum_{a,b} 2^(7(a+b)) * dot(x_a, y_b)        (16 int8 GEMMs, int32 exact)
//
// The 16 slice products accumulate into 7 int32 TMEM accumulators (one per weight class a+b);
// the epilogue forms the classes 0-3 and 4-6 as two exact int64 partial sums, converts both
// exactly to fp64 and adds them with ONE rounding (the correctly rounded exact dot), then scales
// by 2^(Ex+Ey-54). Pairs involving tiny elements (at most 4 per row; ~2e-4 of Gaussian rows)
// add the exact fp64 correction sum_k (x_k y_k - xm_k ym_k) over the tiny dimensions. Rows with
// more than 4 tiny elements (or non-finite values) mark their head for the fp64 DMMA kernel
// instead. Either way the logit is the exact dot up to the final fp64 rounding. From the logits on, the epilogue is the DMMA kernels' arithmetic: per KV block the
// max (sampled) or the numpy-ordered exp-sum (antidiagonal), and the online softmax (m, l).
//
// Kernel shape: one CTA per (head, residue class, 128 gathered query rows); 12 warps.
//   warp 0  TMA: the 3 query slice tiles once, then 3 x (32 keys x 128 B) per key tile
//   warp 1  MMA: per k-step, Q slice a x the 4 contiguous K slices as one N=128
//           tcgen05.mma.kind::i8 into the class columns a..a+3 (4 MMAs instead of 16 pairs)
//   warp 2  TMEM allocator (2 accumulator buffers x 7 classes x 32 columns)
//   warps 4-11  epilogue, two groups taking alternate key tiles (group g owns accumulator
//           buffer g; their running (m, l) merge at the end). The epilogue is FP64-pipe bound
//           (one fp64 exp per logit), so it keeps the tile's 32 logits in registers and
//           evaluates them as independent chains.
#include <algorithm>

#include "common.cuh"
#include "psa_internal.h"

namespace psa {

constexpr int kXlSlices = 4;
constexpr int kXlClasses = 2 * kXlSlices - 1;
constexpr int kXlRowBytes = 128;  // one slice row: K-major, one 128-byte swizzle atom wide
constexpr int kXlQRows = 128;     // MMA M
constexpr int kXlKeys = 32;       // MMA N = keys per tile
constexpr int kXlStages = 4;
constexpr int kXlAccBufs = 2;
constexpr int kXlMaxTiny = 4;
constexpr int kXlHalf = 16;         // keys per epilogue group and tile (half an MMA tile)
constexpr int kXlGroups = 4;        // epilogue warpgroups: (accumulator buffer, half) pairs
constexpr int kXlEpiThreads = kXlGroups * 128;
constexpr int kXlThreads = 128 + kXlEpiThreads;
constexpr int kXlGridShift = 27;
#ifndef PSA_XL_SLEEP_WAIT
#define PSA_XL_SLEEP_WAIT 1
#endif
#if PSA_XL_SLEEP_WAIT
#define XL_WAIT(bar, par) mbar_wait_sleep(bar, par)
#else
#define XL_WAIT(bar, par) mbar_wait(bar, par)
#endif

#ifndef PSA_XL_REGS_EPI
#define PSA_XL_REGS_EPI 112
#endif
// setmaxnreg redistributes the CTA's own pool (640 threads x 96 at launch): the increase only
// completes if 128 x producer + 512 x epilogue fits in it
#ifndef PSA_XL_REGS_PROD
#define PSA_XL_REGS_PROD 32
#endif
constexpr int kXlRegsProducer = PSA_XL_REGS_PROD, kXlRegsEpilogue = PSA_XL_REGS_EPI;
static_assert(128 * kXlRegsProducer + kXlEpiThreads * kXlRegsEpilogue <= (128 + kXlEpiThreads) * 96,
              "register pool");  // X = x * 2^(27 - E), |X| < 2^28

struct XlMeta {
  int32_t e;      // row exponent E (0 for an all-zero row)
  uint32_t tiny;  // count << 28 | four 7-bit dimensions of the tiny elements
};

// ------------------------------------------------------------------ row slicer
// Packed row p of a (head, class) set: p = g * G + j holds element g * cw + j (j < cw) of the
// set, else zeros. Keys use G = 32 (tiles hold whole KV blocks), queries G = cw = padded rows.
struct XlPack {
  int G, cw, total, pad_rows;
};

template <int D, class Rows>
__global__ void __launch_bounds__(256) xl_slice_kernel(const uint16_t* __restrict__ src,
                                                       int64_t n, Rows rows_base, int classes,
                                                       int stride, int block, XlPack pk,
                                                       int8_t* __restrict__ slices,
                                                       XlMeta* __restrict__ meta,
                                                       int32_t* __restrict__ flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * 8 + warp;
  if (p >= pk.pad_rows) return;
  const int64_t bh = blockIdx.y;
  const int cls = blockIdx.z;
  Rows rows = rows_base;
  rows.set_class(cls, stride, block);
  const int g = p / pk.G, j = p % pk.G;
  const int idx = g * pk.cw + j;
  const bool valid = j < pk.cw && idx < rows.count(pk.total);
  const int64_t set = (bh * classes + cls);
  int8_t* dst = slices + set * kXlSlices * static_cast<int64_t>(pk.pad_rows) * kXlRowBytes;

  // Integer decomposition of the bf16 elements |x| = sig * 2^eb (sig < 256): the row exponent
  // E = floor(log2 max|x|) is the max of the elements' eb + floor(log2 sig), and
  // X = trunc(x * 2^(27 - E)) is a shift of sig (a right shift drops bits only for "tiny" x).
  uint2 raw = make_uint2(0u, 0u);
  if (valid && lane * 4 < D)
    raw = *reinterpret_cast<const uint2*>(src + (bh * n + rows(idx)) * D + lane * 4);
  const uint32_t u[4] = {raw.x & 0xFFFFu, raw.x >> 16, raw.y & 0xFFFFu, raw.y >> 16};
  int sig[4], eb[4];
  bool fin = true;
  int emax = -100000;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int ex = static_cast<int>((u[e] >> 7) & 0xFFu), man = static_cast<int>(u[e] & 0x7Fu);
    fin = fin && ex != 0xFF;
    sig[e] = ex ? (128 | man) : man;
    eb[e] = ex ? ex - 134 : -133;
    if (sig[e]) emax = max(emax, eb[e] + 31 - __clz(sig[e]));
  }
  const bool finite = __all_sync(0xffffffffu, fin);
  emax = __reduce_max_sync(0xffffffffu, emax);
  const int E = (emax > -100000 && finite) ? emax : 0;
  uint32_t d[kXlSlices] = {0u, 0u, 0u, 0u};
  unsigned tiny_bits = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int sh = eb[e] + kXlGridShift - E;  // <= 20 (E >= the element's exponent)
    uint32_t mag;
    bool frac;
    if (sh >= 0) {
      mag = static_cast<uint32_t>(sig[e]) << sh;
      frac = false;
    } else {
      const int r = -sh;
      mag = r < 32 ? static_cast<uint32_t>(sig[e]) >> r : 0u;
      frac = r < 32 ? (static_cast<uint32_t>(sig[e]) & ((1u << r) - 1u)) != 0u : sig[e] != 0;
    }
    if (!finite) mag = 0u, frac = false;
    if (frac) tiny_bits |= 1u << e;
    const int X = (u[e] & 0x8000u) ? -static_cast<int>(mag) : static_cast<int>(mag);
    d[0] |= static_cast<uint32_t>(X & 127) << (8 * e);
    d[1] |= static_cast<uint32_t>((X >> 7) & 127) << (8 * e);
    d[2] |= static_cast<uint32_t>((X >> 14) & 127) << (8 * e);
    d[3] |= static_cast<uint32_t>((X >> 21) & 0xFF) << (8 * e);
  }
#pragma unroll
  for (int s = 0; s < kXlSlices; ++s)
    reinterpret_cast<uint32_t*>(dst + (static_cast<int64_t>(s) * pk.pad_rows + p) * kXlRowBytes)[lane] = d[s];
  // tiny elements: at most kXlMaxTiny per row, else the head goes to the fp64 fallback; slots
  // in element order (lane-major), counted with one ballot per element position
  int before = 0, total = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t b = __ballot_sync(0xffffffffu, (tiny_bits >> e) & 1u);
    before += __popc(b & lt);
    total += __popc(b);
  }
  uint32_t dims = 0;
  int slot = before;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if ((tiny_bits >> e) & 1u) {
      if (slot < kXlMaxTiny) dims |= static_cast<uint32_t>(lane * 4 + e) << (7 * slot);
      ++slot;
    }
  dims = __reduce_or_sync(0xffffffffu, dims);
  if (lane == 0) {
    XlMeta m;
    m.e = E;
    m.tiny = (static_cast<uint32_t>(min(total, 7)) << 28) | dims;
    meta[set * pk.pad_rows + p] = m;
    if (valid && (total > kXlMaxTiny || !finite)) atomicOr(flag + bh, 1);
  }
}

// Row maps (queries and keys of one class). count(total) = elements in the class.
struct XlTableRows {  // sampled rows (host table of the reference's generator), one class
  const int32_t* rows;
  PSA_DEV void set_class(int, int, int) {}
  PSA_DEV int count(int total) const { return total; }
  PSA_DEV int64_t operator()(int a) const { return rows[a]; }
};
struct XlQueryClass {  // antidiagonal query rows p = r (mod stride) of every (listed) query block
  int r, c_r, block, stride, n_blocks;
  const int32_t* blocks;  // optional: the query blocks of this call (q-block work units)
  PSA_DEV void set_class(int cls, int stride_, int block_) {
    r = cls;
    stride = stride_;
    block = block_;
    c_r = r < block ? (block - r + stride - 1) / stride : 0;
  }
  PSA_DEV int count(int) const { return n_blocks * c_r; }
  PSA_DEV int64_t operator()(int a) const {
    const int bi = blocks != nullptr ? blocks[a / c_r] : a / c_r;
    return static_cast<int64_t>(bi) * block + r + (a % c_r) * stride;
  }
};
struct XlKeyClass {  // antidiagonal key columns c = kr (mod stride) of every KV block
  int kr, per, block, stride, n_blocks;
  PSA_DEV void set_class(int cls, int stride_, int block_) {
    kr = cls;
    stride = stride_;
    block = block_;
    per = block / stride;
  }
  PSA_DEV int count(int) const { return n_blocks * per; }
  PSA_DEV int64_t operator()(int a) const {
    return static_cast<int64_t>(a / per) * block + kr + (a % per) * stride;
  }
};

// ------------------------------------------------------------------ stats kernel
enum XlMode { kXlMax = 0, kXlAntidiag = 1 };

struct XlParams {
  int64_t n;
  int hq, hkv, classes, stride, b_q, b_k, n_q, n_k;
  int r_total, rq_pad, kp, n_tiles, n_chunks, per, bpt;  // bpt: KV blocks per 16-key half
  int ksplit, tps;  // key tiles split over ksplit CTAs of tps tiles each (partial row stats)
  int64_t out_rows;  // rows of mstat / lstat
  double sqrt_d, inv_sqrt_d, scale;
  const uint16_t* q;
  const uint16_t* k;
  const int32_t* q_rows;  // sampled tables (MAX mode)
  const int32_t* k_rows;
  const XlMeta* qmeta;
  const XlMeta* kmeta;
  const int32_t* qflag;
  const int32_t* kflag;
  double* M;      // MAX: block maxima [bhq][R][n_k];  ANTIDIAG: E [bhq][n][n_k]
  double* Mc;     // ANTIDIAG: chunk maxima [bhq][n][n_tiles]
  double* mstat;  // [bhq][R or n]
  double* lstat;
  double* pm;     // ksplit > 1: per-split (m, l) [ksplit][out_rows], merged by xl_merge_kernel
  double* pl;
};

struct XlMaps {
  CUtensorMap qs;
  CUtensorMap ks;
};

template <int D>
struct XlSmem {
  uint8_t q[kXlSlices][kXlQRows * kXlRowBytes];
  uint8_t k[kXlStages][kXlSlices][kXlKeys * kXlRowBytes];
  double ex[kXlHalf][kXlEpiThreads];  // per-thread logits / exp terms of one half tile
  double exp_tab[64];                 // 2^(j/64)
  double red_m[kXlGroups][kXlQRows], red_l[kXlGroups][kXlQRows], red_x[kXlGroups][kXlQRows];
  uint64_t q_full;
  uint64_t k_full[kXlStages], k_empty[kXlStages];
  uint64_t acc_full[kXlAccBufs], acc_empty[kXlAccBufs];
  uint32_t tmem_base;
};

PSA_DEV void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
PSA_DEV void tmem_zero16(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1};" ::"r"(taddr), "r"(0u)
      : "memory");
}
PSA_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

PSA_DEV void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// kind::i8 instruction descriptor: s8 x s8 -> s32, both K-major.
constexpr uint32_t xl_idesc(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

PSA_DEV double pow2(int k) {  // exact 2^k for the normal range
  return __longlong_as_double(static_cast<long long>(k + 1023) << 52);
}
// exact int32 -> fp64 without a conversion instruction: 1.5*2^52 + 2^31 + x has x in the low
// word once the sign bit is flipped
PSA_DEV double i32_to_f64(int x) {
  return __dsub_rn(__hiloint2double(0x43380000, x ^ static_cast<int>(0x80000000u)),
                   6755401588539392.0);  // 1.5 * 2^52 + 2^31
}
// 64-bit a * b + c with a sign-extended 32-bit a
PSA_DEV long long mad_wide(int a, int b, long long c) {
  long long d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
// The exact dot from the 7 class sums c_k (weight 2^(7k), |c_k| < 2^23), rounded once.
//   lo = c0 + c1 2^7 + c2 2^14 + c3 2^21  (|lo| < 2^45),  hi = c4 + c5 2^7 + c6 2^14  (< 2^38)
// Default: four exact int32 -> fp64 conversions and three fmas (the partial sums below 2^53 are
// exact, the last fma rounds). kWide: lo and hi are built with integer
// multiply-adds directly as the bit patterns of 1.5 * 2^52 + lo / hi (doubles with ulp 1), and
// fma(hi - 1.5 * 2^24, 2^28, 1.5 * 2^52 + lo) = hi * 2^28 + lo (2 FP64 ops instead of 7, more
// integer work: A/B at cfg4 17.2 vs 17.75 ms, at cfg3 5.90 vs 5.77 ms, so only the antidiagonal
// estimator uses it).
template <bool kWide>
PSA_DEV double class_dot(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t c4,
                         uint32_t c5, uint32_t c6) {
  const int a = static_cast<int>(c0) + (static_cast<int>(c1) << 7);
  const int b = static_cast<int>(c2) + (static_cast<int>(c3) << 7);
  const int h = static_cast<int>(c4) + (static_cast<int>(c5) << 7);
  if constexpr (kWide) {
    constexpr long long kMagic = 0x4338000000000000LL;  // 1.5 * 2^52
    const long long lo_bits = mad_wide(b, 16384, mad_wide(a, 1, kMagic));
    const long long hi_bits = mad_wide(static_cast<int>(c6), 16384, mad_wide(h, 1, kMagic));
    const double hi_off = __dsub_rn(__longlong_as_double(hi_bits), 6755399466221568.0);  // 1.5*(2^52+2^24)
    return __fma_rn(hi_off, 268435456.0, __longlong_as_double(lo_bits));
  } else {
    const double lo = __fma_rn(i32_to_f64(b), 16384.0, i32_to_f64(a));
    const double hi = __fma_rn(i32_to_f64(static_cast<int>(c6)), 16384.0, i32_to_f64(h));
    return __fma_rn(hi, 268435456.0, lo);
  }
}
// 2^(j/64), j = 0..63, correctly rounded (host-computed)
__constant__ double kExp2Tab[64] = {1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284, 1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199, 1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418, 1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812, 1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687, 1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783, 1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303, 1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112, 1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647, 1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384, 1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267, 1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364, 1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062, 1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989, 1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656, 1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};

// exp(t) for finite t <= 0 without branches, so a thread's 32 independent exps interleave on
// the FP64 pipe: t = (64 e + j) ln2/64 + r with |r| <= ln2/128 (Cody-Waite, ln2_hi has 21
// trailing zero bits so n * ln2_hi/64 is exact), e^r by a degree-6 Taylor polynomial
// (truncation < 2^-60) evaluated as e^r - 1, 2^(j/64) from a shared-memory table joined with
// one fma, 2^e applied in two exact steps (correct subnormals). Max error 1 ulp against libm
// (numpy's and CUDA's exp differ from each other by as much).
__constant__ double kExpC[9] = {
    92.33248261689366,                           // 64 / ln2
    0.01083042469326756,                         // ln2_hi / 64
    2.9815858269852933e-12,                      // ln2_lo / 64
    8.3333333333333332177e-03,                   // 1/5!
    4.1666666666666664354e-02,                   // 1/4!
    1.6666666666666665741e-01,                   // 1/3!
    0.5, 1.0, 6755399441055744.0};               // 1/2!, 1/1!, 1.5 * 2^52
// Fast path for t >= -708 (2^e applied by an exponent-field add: exact for normal results);
// *slow (0/1) flags a t below that, which the caller recomputes with exp_nonpos_slow.
PSA_DEV double exp_nonpos(double t, const double* tab, int* slow) {
  const double kd = __fma_rn(t, kExpC[0], kExpC[8]);  // rint(t * 64/ln2)
  const int n = __double2loint(kd);
  const double nd = __dsub_rn(kd, kExpC[8]);
  double r = __fma_rn(-nd, kExpC[1], t);
  r = __fma_rn(-nd, kExpC[2], r);
  double pl = kExpC[3];                       // degree 5: truncation < 0.3 ulp for |r| <= ln2/128
  pl = __fma_rn(pl, r, kExpC[4]);
  pl = __fma_rn(pl, r, kExpC[5]);
  pl = __fma_rn(pl, r, kExpC[6]);
  pl = __fma_rn(pl, r, kExpC[7]);
  const double q = __dmul_rn(pl, r);  // e^r - 1
  const double tj = tab[n & 63];
  const double v = __fma_rn(tj, q, tj);  // in [1, 2)
  *slow |= (n < -65344) ? 1 : 0;         // e = n >> 6 < -1021: subnormal / zero result
  return __hiloint2double(__double2hiint(v) + ((n >> 6) << 20), __double2loint(v));
}
// exp(t) for any t <= 0 including -inf (two exact scaling steps: correct subnormals)
PSA_DEV double exp_nonpos_slow(double t, const double* tab) {
  t = fmax(t, -1100.0);
  const double kd = __fma_rn(t, kExpC[0], kExpC[8]);
  const int n = __double2loint(kd);
  const double nd = __dsub_rn(kd, kExpC[8]);
  double r = __fma_rn(-nd, kExpC[1], t);
  r = __fma_rn(-nd, kExpC[2], r);
  double pl = kExpC[3];
  pl = __fma_rn(pl, r, kExpC[4]);
  pl = __fma_rn(pl, r, kExpC[5]);
  pl = __fma_rn(pl, r, kExpC[6]);
  pl = __fma_rn(pl, r, kExpC[7]);
  const double q = __dmul_rn(pl, r);
  const double tj = tab[n & 63];
  const int e = n >> 6;
  const int ea = e >> 1;
  return __dmul_rn(__dmul_rn(__fma_rn(tj, q, tj), pow2(ea)), pow2(e - ea));
}
// exp(m_old - m_new) for the running-sum rescale; 0 before the first tile (m_old = -inf), and
// exactly 1 without the exp when the max did not move (most tiles after the first few)
PSA_DEV double rescale(double m_old, double m_new, const double* tab) {
  if (m_old == m_new) return 1.0;
  return m_old == -INFINITY ? 0.0 : exp_nonpos_slow(__dsub_rn(m_old, m_new), tab);
}
// value of x on row grid E (the part the int8 slices carry exactly)
PSA_DEV double grid_part(double x, int E) {
  return trunc(x * pow2(kXlGridShift - E)) * pow2(E - kXlGridShift);
}
PSA_DEV double bf16_at(const uint16_t* row, int c) {
  return static_cast<double>(__uint_as_float(static_cast<uint32_t>(row[c]) << 16));
}
// exact fp64 correction of dot(x, y) for the tiny dimensions of either row (rare path)
__device__ __noinline__ double tiny_correction(const uint16_t* xr, const uint16_t* yr,
                                               XlMeta mx, XlMeta my) {
  double c = 0.0;
  const int nx = min(static_cast<int>(mx.tiny >> 28), kXlMaxTiny);
  const int ny = min(static_cast<int>(my.tiny >> 28), kXlMaxTiny);
  for (int s = 0; s < nx + ny; ++s) {
    const int dim = s < nx ? (mx.tiny >> (7 * s)) & 127 : (my.tiny >> (7 * (s - nx))) & 127;
    bool dup = false;
    for (int u = 0; u < nx && s >= nx; ++u) dup = dup || (((mx.tiny >> (7 * u)) & 127) == dim);
    if (dup) continue;
    const double x = bf16_at(xr, dim), y = bf16_at(yr, dim);
    c = __dadd_rn(c, __fma_rn(x, y, -(grid_part(x, mx.e) * grid_part(y, my.e))));
  }
  return c;
}

// PER > 0: keys per KV block known at compile time (tile = 32/PER whole blocks; the block
// reductions are static register trees). PER == 0: runtime block size (shared-memory loops).
template <int D, class QRows, class KRows, int MODE, int PER>
__global__ void __launch_bounds__(kXlThreads, 1)
    xl_stats_kernel(const __grid_constant__ XlMaps maps, const XlParams p, QRows qrows0,
                    KRows krows0) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<XlSmem<D>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x;
  const int bhq = blockIdx.y;
  const int cls = blockIdx.z / p.ksplit, split = blockIdx.z % p.ksplit;
  const int b = bhq / p.hq, h = bhq % p.hq;
  const int bkv = b * p.hkv + h / (p.hq / p.hkv);
  if (p.qflag[bhq] | p.kflag[bkv]) return;  // head handled by the fp64 DMMA kernel
  QRows qrows = qrows0;
  qrows.set_class(cls, p.stride, p.b_q);
  const int rows_valid = qrows.count(p.r_total);  // gathered query rows of this class
  const int kcls = MODE == kXlAntidiag ? (p.stride - cls % p.stride) % p.stride : 0;
  KRows krows = krows0;
  krows.set_class(kcls, p.stride, p.b_k);
  if (qt * kXlQRows >= rows_valid) return;
  const int t0 = split * p.tps;                   // this CTA's key tiles [t0, t0 + T)
  const int T = min(p.n_tiles, t0 + p.tps) - t0;  // >= 1 (ksplit <= n_tiles)

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kXlStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kXlAccBufs; ++s) {
      mbar_init(&sm.acc_full[s], 1);
      mbar_init(&sm.acc_empty[s], 2 * 128);  // the two half-tile groups of the buffer
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.qs);
    tma_prefetch_desc(&maps.ks);
  }
  if (warp == 2) {
    tmem_alloc(&sm.tmem_base, 512);
    tmem_relinquish();
  }
  if (threadIdx.x < 64) sm.exp_tab[threadIdx.x] = kExp2Tab[threadIdx.x];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (warp >= 4 && warp < 8) {  // classes 4-6 start at zero (the MMAs only accumulate into them)
    const uint32_t tl = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    for (int ab = 0; ab < kXlAccBufs; ++ab)
      for (int c = kXlSlices; c < kXlClasses; ++c)
        for (int h2 = 0; h2 < kXlKeys / 16; ++h2)
          tmem_zero16(tl + ab * (kXlClasses * kXlKeys) + c * kXlKeys + h2 * 16);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp < 4) {
    // producer warpgroup (TMA, MMA, TMEM allocator, idle): few registers, so the epilogue
    // warpgroups get 112 (128 x 32 + 512 x 112 = 640 x 96) instead of the launch's 96
    if constexpr (kXlRegsEpilogue > 96) regs_dec<kXlRegsProducer>();
  if (warp == 0) {
    if (lane == 0) {
      const int qset = (bhq * p.classes + cls) * kXlSlices;
      mbar_arrive_expect_tx(&sm.q_full, kXlSlices * kXlQRows * kXlRowBytes);
      for (int a = 0; a < kXlSlices; ++a)
        tma_load_2d(&maps.qs, &sm.q_full, sm.q[a], 0, (qset + a) * p.rq_pad + qt * kXlQRows);
      const int kset = (bkv * p.classes + kcls) * kXlSlices;
      for (int t = 0; t < T; ++t) {
        const int s = t % kXlStages;
        if (t >= kXlStages) mbar_wait_backoff(&sm.k_empty[s], ((t / kXlStages) - 1) & 1);
        mbar_arrive_expect_tx(&sm.k_full[s], kXlSlices * kXlKeys * kXlRowBytes);
        for (int bb = 0; bb < kXlSlices; ++bb)
          tma_load_2d(&maps.ks, &sm.k_full[s], sm.k[s][bb], 0,
                      (kset + bb) * p.kp + (t0 + t) * kXlKeys);
      }
    }
  } else if (warp == 1) {
    // Class c = a + b accumulates at columns [c * 32, c * 32 + 32) of the buffer: slice a of Q
    // against the 4 contiguous K slices is ONE N = 128 MMA into columns [a * 32, a * 32 + 128).
    // Classes 0-3 are initialised by slice 0; classes 4-6 are zeroed by the epilogue after it
    // reads them, so slices 1-3 only accumulate. 4 MMAs per K step.
    constexpr uint32_t idesc128 = xl_idesc(kXlQRows, 4 * kXlKeys);
    static_assert(kXlSlices == 4, "class layout assumes 4 slices");
    mbar_wait(&sm.q_full, 0);
    tc_fence_after();
    for (int t = 0; t < T; ++t) {
      const int s = t % kXlStages, ab = t % kXlAccBufs;
      XL_WAIT(&sm.k_full[s], (t / kXlStages) & 1);
      if (t >= kXlAccBufs) mbar_wait_backoff(&sm.acc_empty[ab], ((t / kXlAccBufs) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t dbuf = tmem + ab * (kXlClasses * kXlKeys);
        const uint64_t b0 = umma_desc_sw128(smem_u32(sm.k[s][0]), 16, 1024);
#pragma unroll
        for (int a = 0; a < kXlSlices; ++a) {
          const uint64_t ad = umma_desc_sw128(smem_u32(sm.q[a]), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk) {
            const uint32_t ko = (kk * 32) >> 4;
            mma_i8_ss(dbuf + a * kXlKeys, ad + ko, b0 + ko, idesc128, (a > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit(&sm.k_empty[s]);
        mma_commit(&sm.acc_full[ab]);
      }
      __syncwarp();
    }
  }
  } else {
    if constexpr (kXlRegsEpilogue > 96) regs_inc<kXlRegsEpilogue>();
    // ---- epilogue: group g takes accumulator buffer g >> 1 (tiles t = g >> 1 mod 2) and
    // the 16-key half (g & 1) of each of those tiles; half index hx = 2 t + half holds the
    // whole KV blocks [hx * bpt, hx * bpt + bpt) (keys packed 16 per half by the slicer)
    const int e_tid = threadIdx.x - 128;
    const int grp = (warp - 4) >> 2;
    const int buf = grp >> 1, half = grp & 1;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const int a = qt * kXlQRows + row;  // gathered query row of this class
    const bool row_ok = a < rows_valid;
    const int qset = bhq * p.classes + cls;
    const XlMeta qm = p.qmeta[static_cast<int64_t>(qset) * p.rq_pad + a];
    const bool q_tiny = (qm.tiny >> 28) != 0;
    const int64_t qsrc = row_ok ? qrows(a) : 0;  // row inside the head
    const uint16_t* qrow_ptr = p.q + (static_cast<int64_t>(bhq) * p.n + qsrc) * D;
    const XlMeta* kmeta = p.kmeta + static_cast<int64_t>(bkv * p.classes + kcls) * p.kp;
    const uint16_t* kbase = p.k + static_cast<int64_t>(bkv) * p.n * D;
    const uint32_t t_acc = tmem + (static_cast<uint32_t>(wq * 32) << 16) +
                           buf * (kXlClasses * kXlKeys) + half * kXlHalf;
    const int cw = p.bpt * p.per;  // valid keys of a half
    const int64_t out_row = MODE == kXlMax ? static_cast<int64_t>(bhq) * rows_valid + a
                                           : static_cast<int64_t>(bhq) * p.n + qsrc;
    double* out_blocks = p.M + out_row * p.n_k;
    double m_run = -INFINITY, l_run = 0.0;
    double rmax = -INFINITY;  // MAX mode: exact running max of the raw dot products
    double* xs = &sm.ex[0][e_tid];  // this thread's column: 16 values, stride kXlEpiThreads

    for (int tl = buf; tl < T; tl += 2) {
      const int t = t0 + tl;  // global key tile
      const int hx = 2 * t + half;
      const int j0 = hx * p.bpt;  // first KV block of the half
      const int nb = max(0, min(p.bpt, p.n_k - j0));
      const int nvalid = nb * p.per;
      const uint32_t valid_mask = (1u << nvalid) - 1u;
      const XlMeta kml = kmeta[t * kXlKeys + half * kXlHalf + (lane & (kXlHalf - 1))];
      const int kinfo = (kml.e << 1) | ((kml.tiny >> 28) != 0u ? 1 : 0);
      XL_WAIT(&sm.acc_full[buf], (tl >> 1) & 1);
      tc_fence_after();
      double dv[kXlHalf];
#pragma unroll
      for (int c8 = 0; c8 < kXlHalf / 8; ++c8) {
        uint32_t cv[kXlClasses][8];
#pragma unroll
        for (int c = 0; c < kXlClasses; ++c) tmem_ld8(t_acc + c * kXlKeys + c8 * 8, cv[c]);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e)  // exact dot(X, Y) rounded once
          dv[c8 * 8 + e] = class_dot<MODE == kXlAntidiag>(cv[0][e], cv[1][e], cv[2][e], cv[3][e], cv[4][e], cv[5][e],
                                     cv[6][e]);
      }
#pragma unroll
      for (int c = kXlSlices; c < kXlClasses; ++c) tmem_zero16(t_acc + c * kXlKeys);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.acc_empty[buf]);
      if (nb == 0) continue;  // odd half count: this half of the last tile holds no block
      // exact corrections for tiny elements (rare: skipped unless some lane needs one)
      const uint32_t key_tiny = __ballot_sync(0xffffffffu, kinfo & 1) & valid_mask;
#pragma unroll
      for (int j = 0; j < kXlHalf; ++j) {
        const int kj = __shfl_sync(0xffffffffu, kinfo, j);
        dv[j] = __dmul_rn(dv[j], pow2((kj >> 1) + qm.e - 2 * kXlGridShift));
      }
      if (__any_sync(0xffffffffu, q_tiny && row_ok) || key_tiny != 0u) {
#pragma unroll 1
        for (int j = 0; j < nvalid; ++j)
          if (row_ok && (q_tiny || ((key_tiny >> j) & 1u))) {
            const XlMeta kmj = kmeta[t * kXlKeys + half * kXlHalf + j];
            const double c = tiny_correction(qrow_ptr, kbase + krows(hx * cw + j) * D, qm, kmj);
            xs[j * kXlEpiThreads] = c;  // staged: dv[] needs static indices
          }
#pragma unroll
        for (int j = 0; j < kXlHalf; ++j)
          if (row_ok && (q_tiny || ((key_tiny >> j) & 1u)) && j < nvalid)
            dv[j] = __dadd_rn(dv[j], xs[j * kXlEpiThreads]);
      }

      constexpr int kP = PER > 0 ? PER : 1;
      if (PER > 0) {
        // ---- static block structure: blocks are PER consecutive keys of the half
        constexpr int kB = kXlHalf / kP;
        if (MODE == kXlMax) {
          double hmax = -INFINITY;
#pragma unroll
          for (int bb = 0; bb < kB; ++bb) {  // raw block maxima (tree)
            double v[kP];
#pragma unroll
            for (int u = 0; u < kP; ++u) v[u] = dv[bb * kP + u];
#pragma unroll
            for (int w = 1; w < kP; w <<= 1)
#pragma unroll
              for (int u = 0; u + w < kP; u += 2 * w) v[u] = fmax(v[u], v[u + w]);
            if (bb < nb) {
              hmax = fmax(hmax, v[0]);
              if (row_ok) out_blocks[j0 + bb] = v[0];
            }
          }
          rmax = fmax(rmax, hmax);
          // exps use an offset within an ulp of the running max logit (no division on the
          // critical path); the exact max fl(max / sqrt(d)) is applied once per row at the end
          const double m_new = fmax(m_run, __dmul_rn(hmax, p.inv_sqrt_d));
          double ps[4] = {0.0, 0.0, 0.0, 0.0};
          int slow = 0;
#pragma unroll
          for (int j = 0; j < kXlHalf; ++j) {
            const bool ok = (valid_mask >> j) & 1u;
            const double e = exp_nonpos(ok ? __fma_rn(dv[j], p.inv_sqrt_d, -m_new) : 0.0,
                                        sm.exp_tab, &slow);
            ps[j & 3] = __dadd_rn(ps[j & 3], ok ? e : 0.0);
          }
          if (slow) {  // some term below e^-708: redo this half's sum with exact subnormals
            ps[0] = ps[1] = ps[2] = ps[3] = 0.0;
#pragma unroll
            for (int j = 0; j < kXlHalf; ++j)
              if ((valid_mask >> j) & 1u)
                ps[j & 3] = __dadd_rn(ps[j & 3], exp_nonpos_slow(__fma_rn(dv[j], p.inv_sqrt_d, -m_new),
                                                                 sm.exp_tab));
          }
          const double part = __dadd_rn(__dadd_rn(ps[0], ps[1]), __dadd_rn(ps[2], ps[3]));
          l_run = __dadd_rn(__dmul_rn(l_run, rescale(m_run, m_new, sm.exp_tab)), part);
          m_run = m_new;
        } else {
          auto xsc = [&](int j) { return __dmul_rn(dv[j], p.scale); };  // importance.py:128
          double cmax = -INFINITY;
#pragma unroll
          for (int j = 0; j < kXlHalf; ++j)
            cmax = fmax(cmax, ((valid_mask >> j) & 1u) ? dv[j] : -INFINITY);
          const double m_new = fmax(m_run, __dmul_rn(cmax, p.scale));
          double part = 0.0;
#pragma unroll
          for (int bb = 0; bb < kB; ++bb) {
            double ev[kP];
            int slow = 0;
#pragma unroll
            for (int u = 0; u < kP; ++u)
              ev[u] = exp_nonpos(__dsub_rn(xsc(bb * kP + u), m_new), sm.exp_tab, &slow);
            if (slow) {
#pragma unroll
              for (int u = 0; u < kP; ++u)
                ev[u] = exp_nonpos_slow(__dsub_rn(xsc(bb * kP + u), m_new), sm.exp_tab);
            }
            // numpy pairwise order for PER elements (np_pairwise_sum, common.cuh)
            double e;
            if (kP < 8) {
              e = 0.0;
#pragma unroll
              for (int u = 0; u < kP; ++u) e = __dadd_rn(e, ev[u]);
            } else {
              double r8[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) r8[u] = ev[u < kP ? u : 0];
#pragma unroll
              for (int u = 8; u < kP - (kP % 8); u += 8)
#pragma unroll
                for (int w = 0; w < 8; ++w) r8[w] = __dadd_rn(r8[w], ev[u + w]);
              e = __dadd_rn(__dadd_rn(__dadd_rn(r8[0], r8[1]), __dadd_rn(r8[2], r8[3])),
                            __dadd_rn(__dadd_rn(r8[4], r8[5]), __dadd_rn(r8[6], r8[7])));
#pragma unroll
              for (int u = kP - (kP % 8); u < kP; ++u) e = __dadd_rn(e, ev[u]);
            }
            if (bb < nb) {
              part = __dadd_rn(part, e);
              if (row_ok) out_blocks[j0 + bb] = e;
            }
          }
          l_run = __dadd_rn(__dmul_rn(l_run, rescale(m_run, m_new, sm.exp_tab)), part);
          m_run = m_new;
          if (row_ok) p.Mc[out_row * p.n_chunks + hx] = m_new;
        }
      } else if (MODE == kXlMax) {
        double hmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < kXlHalf; ++j) {
          xs[j * kXlEpiThreads] = dv[j];
          hmax = fmax(hmax, ((valid_mask >> j) & 1u) ? dv[j] : -INFINITY);
        }
        rmax = fmax(rmax, hmax);
        const double m_new = fmax(m_run, __dmul_rn(hmax, p.inv_sqrt_d));
        double ps[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < kXlHalf; ++j) {
          const double arg = __fma_rn(dv[j], p.inv_sqrt_d, -m_new);
          ps[j & 3] = __dadd_rn(ps[j & 3],
                                exp_nonpos_slow(((valid_mask >> j) & 1u) ? arg : -2000.0, sm.exp_tab));
        }
        const double part = __dadd_rn(__dadd_rn(ps[0], ps[1]), __dadd_rn(ps[2], ps[3]));
        l_run = __dadd_rn(__dmul_rn(l_run, rescale(m_run, m_new, sm.exp_tab)), part);
        m_run = m_new;
        // raw block maxima (the finalize kernel divides by sqrt(d) once per value)
        for (int bb = 0; bb < nb; ++bb) {
          double bm = xs[bb * p.per * kXlEpiThreads];
          for (int u = 1; u < p.per; ++u) bm = fmax(bm, xs[(bb * p.per + u) * kXlEpiThreads]);
          if (row_ok) out_blocks[j0 + bb] = bm;
        }
      } else {
        double cmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < kXlHalf; ++j)
          cmax = fmax(cmax, ((valid_mask >> j) & 1u) ? dv[j] : -INFINITY);
        const double m_new = fmax(m_run, __dmul_rn(cmax, p.scale));
#pragma unroll
        for (int j = 0; j < kXlHalf; ++j) {
          const double arg = __dsub_rn(__dmul_rn(dv[j], p.scale), m_new);
          xs[j * kXlEpiThreads] = exp_nonpos_slow(((valid_mask >> j) & 1u) ? arg : -2000.0, sm.exp_tab);
        }
        double part = 0.0;
        for (int bb = 0; bb < nb; ++bb) {  // numpy pairwise order inside each block
          const double* xb = xs + bb * p.per * kXlEpiThreads;
          const double e = np_pairwise_sum_fn(p.per, [&](int u) { return xb[u * kXlEpiThreads]; });
          part = __dadd_rn(part, e);
          if (row_ok) out_blocks[j0 + bb] = e;
        }
        l_run = __dadd_rn(__dmul_rn(l_run, rescale(m_run, m_new, sm.exp_tab)), part);
        m_run = m_new;
        if (row_ok) p.Mc[out_row * p.n_chunks + hx] = m_new;
      }
    }
    // merge the four groups' running (m, l); MAX mode re-bases l on the exact max logit
    sm.red_m[grp][row] = m_run;
    sm.red_l[grp][row] = l_run;
    sm.red_x[grp][row] = rmax;
    named_bar_sync(1, kXlEpiThreads);
    if (grp == 0 && row_ok) {
      double xm = -INFINITY, mm = -INFINITY;
#pragma unroll
      for (int g = 0; g < kXlGroups; ++g) {
        xm = fmax(xm, sm.red_x[g][row]);
        mm = fmax(mm, sm.red_m[g][row]);
      }
      const double m = MODE == kXlMax ? __ddiv_rn(xm, p.sqrt_d) : mm;  // importance.py:80
      double l = 0.0;
#pragma unroll
      for (int g = 0; g < kXlGroups; ++g) {
        const double mg = sm.red_m[g][row];
        if (mg != -INFINITY) l = __dadd_rn(l, __dmul_rn(sm.red_l[g][row], exp(__dsub_rn(mg, m))));
      }
      if (p.ksplit > 1) {
        p.pm[split * p.out_rows + out_row] = m;
        p.pl[split * p.out_rows + out_row] = l;
      } else {
        p.mstat[out_row] = m;
        p.lstat[out_row] = l;
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

// Key-split merge: m = max_s m_s, l = sum_s l_s exp(m_s - m) (the stats kernel's own group merge
// across CTAs). Heads flagged for the fp64 kernel are left to it.
__global__ void __launch_bounds__(256) xl_merge_kernel(const double* __restrict__ pm,
                                                       const double* __restrict__ pl, int ksplit,
                                                       int64_t out_rows, int64_t rows_per_head,
                                                       int hq, int hkv,
                                                       const int32_t* __restrict__ qflag,
                                                       const int32_t* __restrict__ kflag,
                                                       double* __restrict__ mstat,
                                                       double* __restrict__ lstat) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= out_rows) return;
  const int bhq = static_cast<int>(r / rows_per_head);
  const int b = bhq / hq, h = bhq % hq;
  if (qflag[bhq] | kflag[b * hkv + h / (hq / hkv)]) return;
  double m = -INFINITY;
  for (int s = 0; s < ksplit; ++s) m = fmax(m, pm[s * out_rows + r]);
  double l = 0.0;
  for (int s = 0; s < ksplit; ++s) {
    const double ms = pm[s * out_rows + r];
    if (ms != -INFINITY) l = __dadd_rn(l, __dmul_rn(pl[s * out_rows + r], exp(__dsub_rn(ms, m))));
  }
  mstat[r] = m;
  lstat[r] = l;
}

// ------------------------------------------------------------------ host side
static int xl_encode(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (fn == nullptr) return psa_fail(PSA_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(kXlRowBytes), rows};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(kXlRowBytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kXlRowBytes), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return psa_fail(PSA_ECUDA, "cuTensorMapEncodeTiled (int8) failed (%d)", (int)r);
  return PSA_OK;
}

XlGeometry xl_geometry(int64_t bhq, int64_t bkv, int n_q, int n_k, int classes, int rows_per_class,
                       int per, int64_t out_rows) {
  XlGeometry g{};
  g.ok = per >= 1 && per <= kXlHalf;
  if (!g.ok) return g;
  g.per = per;
  g.bpt = kXlHalf / per;  // whole KV blocks per 16-key half
  g.n_halves = (n_k + g.bpt - 1) / g.bpt;
  g.n_tiles = (g.n_halves + 1) / 2;
  g.kp = g.n_tiles * kXlKeys;
  // Key tiles per CTA ~32: a fixed property of the layout (not of the head count), so the grid
  // stays full when few heads run per GPU and every configuration merges the same way.
  g.ksplit = std::max(1, std::min(8, (g.n_tiles + 16) / 32));
  g.tps = (g.n_tiles + g.ksplit - 1) / g.ksplit;
  g.ksplit = (g.n_tiles + g.tps - 1) / g.tps;
  g.out_rows = out_rows;
  g.rq_pad = (rows_per_class + kXlQRows - 1) / kXlQRows * kXlQRows;
  g.classes = classes;
  const size_t qs = static_cast<size_t>(bhq) * classes * kXlSlices * g.rq_pad * kXlRowBytes;
  const size_t ks = static_cast<size_t>(bkv) * classes * kXlSlices * g.kp * kXlRowBytes;
  const size_t qm = static_cast<size_t>(bhq) * classes * g.rq_pad * sizeof(XlMeta);
  const size_t km = static_cast<size_t>(bkv) * classes * g.kp * sizeof(XlMeta);
  g.off_ks = qs;
  g.off_qm = g.off_ks + ks;
  g.off_km = g.off_qm + qm;
  g.off_flags = g.off_km + km;
  g.off_part = (g.off_flags + static_cast<size_t>(bhq + bkv) * sizeof(int32_t) + 255) / 256 * 256;
  g.bytes = g.off_part + (g.ksplit > 1 ? 2 * static_cast<size_t>(g.ksplit) * out_rows * sizeof(double) : 0);
  g.bytes = (g.bytes + 255) / 256 * 256;
  return g;
}

template <int D, int MODE, class QR, class KR>
static int xl_launch(const void* q, const void* k, int64_t batch, int hq, int hkv, int64_t n,
                     int b_q, int b_k, int stride, const XlGeometry& g, QR qr, KR kr,
                     int q_total, int k_total, void* ws, double* M, double* Mc, double* mstat,
                     double* lstat, cudaStream_t s) {
  const int64_t bhq = batch * hq, bkv = batch * hkv;
  auto* base = static_cast<uint8_t*>(ws);
  auto* qs = reinterpret_cast<int8_t*>(base);
  auto* ks = reinterpret_cast<int8_t*>(base + g.off_ks);
  auto* qm = reinterpret_cast<XlMeta*>(base + g.off_qm);
  auto* km = reinterpret_cast<XlMeta*>(base + g.off_km);
  auto* qflag = reinterpret_cast<int32_t*>(base + g.off_flags);
  int32_t* kflag = qflag + bhq;
  cudaMemsetAsync(qflag, 0, static_cast<size_t>(bhq + bkv) * sizeof(int32_t), s);
  const auto* qq = static_cast<const uint16_t*>(q);
  const auto* kk = static_cast<const uint16_t*>(k);
  XlPack qp{g.rq_pad, g.rq_pad, q_total, g.rq_pad};
  xl_slice_kernel<D, QR><<<dim3((g.rq_pad + 7) / 8, bhq, g.classes), 256, 0, s>>>(
      qq, n, qr, g.classes, stride, b_q, qp, qs, qm, qflag);
  int rc = psa_check_launch("xl_slice_kernel<q>");
  if (rc) return rc;
  XlPack kp{kXlHalf, g.bpt * g.per, k_total, g.kp};
  xl_slice_kernel<D, KR><<<dim3((g.kp + 7) / 8, bkv, g.classes), 256, 0, s>>>(
      kk, n, kr, g.classes, stride, b_k, kp, ks, km, kflag);
  rc = psa_check_launch("xl_slice_kernel<k>");
  if (rc) return rc;

  XlMaps maps;
  memset(&maps, 0, sizeof(maps));
  rc = xl_encode(&maps.qs, qs, static_cast<uint64_t>(bhq) * g.classes * kXlSlices * g.rq_pad,
                 kXlQRows);
  if (rc) return rc;
  rc = xl_encode(&maps.ks, ks, static_cast<uint64_t>(bkv) * g.classes * kXlSlices * g.kp, kXlKeys);
  if (rc) return rc;
  XlParams p{};
  p.n = n;
  p.hq = hq;
  p.hkv = hkv;
  p.classes = g.classes;
  p.stride = stride;
  p.b_q = b_q;
  p.b_k = b_k;
  p.n_q = static_cast<int>(n / b_q);
  p.n_k = static_cast<int>(n / b_k);
  p.r_total = q_total;
  p.rq_pad = g.rq_pad;
  p.kp = g.kp;
  p.n_tiles = g.n_tiles;
  p.ksplit = g.ksplit;
  p.tps = g.tps;
  p.out_rows = g.out_rows;
  p.pm = reinterpret_cast<double*>(base + g.off_part);
  p.pl = p.pm + static_cast<int64_t>(g.ksplit) * g.out_rows;
  p.n_chunks = g.n_halves;
  p.per = g.per;
  p.bpt = g.bpt;
  p.sqrt_d = sqrt(static_cast<double>(D));
  p.inv_sqrt_d = 1.0 / p.sqrt_d;
  p.scale = 1.0 / sqrt(static_cast<double>(D));
  p.q = qq;
  p.k = kk;
  p.qmeta = qm;
  p.kmeta = km;
  p.qflag = qflag;
  p.kflag = kflag;
  p.M = M;
  p.Mc = Mc;
  p.mstat = mstat;
  p.lstat = lstat;
  const size_t smem = sizeof(XlSmem<D>);
  auto kern = g.per == 8 ? xl_stats_kernel<D, QR, KR, MODE, 8> : xl_stats_kernel<D, QR, KR, MODE, 0>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  kern<<<dim3(g.rq_pad / kXlQRows, bhq, g.classes * g.ksplit), kXlThreads, smem, s>>>(maps, p, qr, kr);
  rc = psa_check_launch("xl_stats_kernel");
  if (rc || g.ksplit == 1) return rc;
  xl_merge_kernel<<<static_cast<unsigned>((g.out_rows + 255) / 256), 256, 0, s>>>(
      p.pm, p.pl, g.ksplit, g.out_rows, g.out_rows / bhq, hq, hkv, qflag, kflag, mstat, lstat);
  return psa_check_launch("xl_merge_kernel");
}

int xl_sampled_max(const void* q, const void* k, int64_t batch, int hq, int hkv, int64_t n, int d,
                   int b_q, int b_k, int n_q, const int32_t* q_rows, const int32_t* k_rows, int s_q,
                   int s_k, const XlGeometry& g, void* ws, double* M, double* mstat,
                   double* lstat, cudaStream_t s) {
  const int n_k = static_cast<int>(n / b_k);
  XlTableRows qr{q_rows}, kr{k_rows};
  if (d == 128)
    return xl_launch<128, kXlMax>(q, k, batch, hq, hkv, n, b_q, b_k, 1, g, qr, kr, n_q * s_q,
                                  n_k * s_k, ws, M, nullptr, mstat, lstat, s);
  return xl_launch<64, kXlMax>(q, k, batch, hq, hkv, n, b_q, b_k, 1, g, qr, kr, n_q * s_q,
                               n_k * s_k, ws, M, nullptr, mstat, lstat, s);
}

int xl_antidiag(const void* q, const void* k, int64_t batch, int hq, int hkv, int64_t n, int d,
                int b_q, int b_k, int stride, int n_q, const int32_t* qblk, const XlGeometry& g,
                void* ws, double* E, double* Mc, double* mstat, double* lstat, cudaStream_t s) {
  const int n_k = static_cast<int>(n / b_k);
  XlQueryClass qr{};
  qr.n_blocks = n_q;
  qr.blocks = qblk;
  XlKeyClass kr{};
  kr.n_blocks = n_k;
  if (d == 128)
    return xl_launch<128, kXlAntidiag>(q, k, batch, hq, hkv, n, b_q, b_k, stride, g, qr, kr, 0, 0,
                                       ws, E, Mc, mstat, lstat, s);
  return xl_launch<64, kXlAntidiag>(q, k, batch, hq, hkv, n, b_q, b_k, stride, g, qr, kr, 0, 0,
                                    ws, E, Mc, mstat, lstat, s);
}

const int32_t* xl_qflags(const XlGeometry& g, const void* ws) {
  return reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(ws) + g.off_flags);
}

}  // namespace psa
