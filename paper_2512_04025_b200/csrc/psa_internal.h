// Internal host-side helpers shared by the C-ABI translation units: thread-local error
// string, argument checks, launch checks, and small by-value parameter structs.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "../../include/psa.h"

namespace psa {

constexpr int kMaxLevels = 8;
constexpr int kMaxCuts = 16;

struct SimTaus {
  double v[kMaxLevels];
};

struct LevelRule {  // thresholds (mode 0) or quantile rank counts (mode 1)
  double taus[kMaxCuts];
  int32_t counts[kMaxCuts];
  int n_cuts;
  int mode;
};

// Exact int8-sliced importance logits (psa_xlogits.cu).
struct XlGeometry {
  bool ok;
  int per, bpt, n_halves, n_tiles, kp, rq_pad, classes;  // bpt: KV blocks per 16-key half
  int ksplit, tps;   // key tiles split over ksplit CTAs of tps tiles (merged by xl_merge_kernel)
  int64_t out_rows;  // rows of the (m, l) statistics
  size_t off_ks, off_qm, off_km, off_flags, off_part, bytes;
};
XlGeometry xl_geometry(int64_t bhq, int64_t bkv, int n_q, int n_k, int classes, int rows_per_class,
                       int per, int64_t out_rows);
// n_q: query blocks of the call (the q_rows table holds n_q * s_q rows); qblk: optional list of
// the call's query blocks (antidiagonal; NULL = blocks 0..n_q-1)
int xl_sampled_max(const void* q, const void* k, int64_t batch, int hq, int hkv, int64_t n, int d,
                   int b_q, int b_k, int n_q, const int32_t* q_rows, const int32_t* k_rows, int s_q,
                   int s_k, const XlGeometry& g, void* ws, double* M, double* mstat,
                   double* lstat, cudaStream_t s);
int xl_antidiag(const void* q, const void* k, int64_t batch, int hq, int hkv, int64_t n, int d,
                int b_q, int b_k, int stride, int n_q, const int32_t* qblk, const XlGeometry& g,
                void* ws, double* E, double* Mc, double* mstat, double* lstat, cudaStream_t s);
// device flags [bhq] then [bkv]: heads the int8 path could not represent exactly
const int32_t* xl_qflags(const XlGeometry& g, const void* ws);

// tcgen05 dQ pass of the backward (psa_attention.cu; D = 128)
int attn_bwd_dq_tc(const void* q, const void* k, const void* v, const void* k_pyr,
                   const void* v_pyr, const void* dout, const float* lse, const float* drow,
                   int64_t batch, int hq, int hkv, int64_t n, int b_q, int b_k, int levels,
                   const uint16_t* csr, const int32_t* info, int causal, void* dq,
                   cudaStream_t s);

// tcgen05 dK/dV pass of the backward (psa_attention.cu; D = 128)
int attn_bwd_dkv_tc(const void* q, const void* k, const void* v, const void* k_pyr,
                    const void* v_pyr, const void* dout, const float* lse, const float* drow,
                    int64_t batch, int hq, int hkv, int64_t n, int b_q, int b_k, int levels,
                    const int8_t* level_map, int causal, const float* nl2, float* scratch,
                    void* dk, void* dv, cudaStream_t s);

// cuTensorMapEncodeTiled from the driver (psa_attention.cu)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode_fn();

}  // namespace psa

int psa_fail(int code, const char* fmt, ...);
int psa_check_launch(const char* what);

#define PSA_CHECK_ARG(cond, msg)                           \
  do {                                                     \
    if (!(cond)) return psa_fail(PSA_EINVAL, "%s", (msg)); \
  } while (0)
