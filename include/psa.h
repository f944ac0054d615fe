/*
 * psa.h — C ABI of the B200-native Pyramid Sparse Attention (PSA) forward path.
 *
 * One shared library (libpsa.so, sm_100a) exports these entry points. Each one replaces a
 * function of the reference package `pyrattn` (mounted at /root/reference/pkg); the cited
 * file:line is the reference interface whose semantics it reproduces. The Python layer
 * `paper_2512_04025_b200` binds them with ctypes and keeps the reference names.
 *
 * Conventions (all entry points):
 *   - return PSA_OK (0) on success; PSA_EINVAL (-2) maps to ValidationError,
 *     PSA_ENUMERIC (-4) to NumericError, PSA_ECUDA (-5) to RuntimeError; psa_last_error()
 *     returns a thread-local message for the last failure.
 *   - tensor arguments are DEVICE pointers to contiguous row-major arrays; bf16 tensors are
 *     passed as `const void*` (raw 16-bit payloads). The caller allocates every output and
 *     workspace; the library never calls cudaMalloc.
 *   - `stream` is a cudaStream_t; every call is asynchronous and stream-ordered, no host
 *     synchronisation happens inside. Small host arrays (thresholds, counts) are copied into
 *     kernel parameters before the call returns.
 *   - Re-entrant: no mutable global state besides the thread-local error string and a cached
 *     driver entry point.
 *   - Shapes: `bh` = batch*heads; Q is [batch, hq, n, d], K/V are [batch, hkv, n, d]
 *     (hq % hkv == 0; q head h reads kv head h / (hq/hkv)).
 */
#ifndef PSA_H_
#define PSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSA_OK 0
#define PSA_EINVAL (-2)
#define PSA_ENUMERIC (-4)
#define PSA_ECUDA (-5)

/* Last error message of the calling thread ("" if none). */
const char* psa_last_error(void);

/* Library/ABI version (major*100 + minor). */
int psa_version(void);

/*
 * K1 — pyramid build.  Replaces build_pyramid / _pool_stack / mean_pool_rows
 * (pkg/src/pyrattn/blocks.py:86-109, pkg/src/pyrattn/linalg.py:46-58).
 * k, v      : bf16 [bh, n, d]
 * k_pyr/v_pyr: bf16 buffers holding levels 2..levels back to back; level h occupies
 *             [bh, n >> (h-1), d] starting at element offset d * sum_{h'=2}^{h-1} bh*(n >> (h'-1)).
 *             Level 1 is the raw K/V (not copied).
 * Each level is the fp64 dyadic mean of raw rows rounded once to bf16 (RNE).
 * nonfinite : optional device int32 flag, OR-ed with 1 if any K/V entry is NaN/Inf.
 */
int psa_pyramid_build(const void* k, const void* v, int64_t bh, int64_t n, int d, int b_k,
                      int levels, void* k_pyr, void* v_pyr, int32_t* nonfinite, void* stream);

/*
 * Pyramid of token-permuted K/V.  Fuses apply_permutation (pkg/src/pyrattn/permute.py:131-137,
 * as pipeline._run_head applies it before pooling, pipeline.py:257-263) into the pyramid build
 * (blocks.py:93-109): row p of each head reads source row index[p].  Writes the permuted K/V
 * (level 1) to k1/v1 [bh, n, d] and levels 2..H to k_pyr/v_pyr as psa_pyramid_build does.
 * index: DEVICE int64 [n], a bijection.
 */
int psa_pyramid_build_gather(const void* k, const void* v, int64_t bh, int64_t n, int d, int b_k,
                             int levels, const int64_t* index, void* k1, void* v1, void* k_pyr,
                             void* v_pyr, int32_t* nonfinite, void* stream);

/*
 * Similarity cap (Alg. 3).  Replaces level_cap_from_similarity / _strided_block_similarity
 * (pkg/src/pyrattn/mask.py:182-234).  sim_taus: HOST array of levels-1 thresholds.
 * caps: int8 [bh, n/b_k], each in 1..levels.
 */
int psa_similarity_caps(const void* k, int64_t bh, int64_t n, int d, int b_k, int levels,
                        const double* sim_taus, int8_t* caps, void* stream);

/* Importance flags (psa_importance_sampled / psa_importance_antidiagonal). */
#define PSA_IMP_FP64_ONLY 1 /* skip the int8-sliced tensor-core logits; fp64 DMMA for every head */

/*
 * K2 — sampled importance.  Replaces importance_sampled (pkg/src/pyrattn/importance.py:52-85).
 * q_rows/k_rows: DEVICE int32 tables of sampled row indices inside a head, in the order the
 *   reference's single seeded generator produces them (n_q*s_q and n_k*s_k entries).
 * reducer: 0 = max, 1 = mean.  scores: fp64 [batch*hq, n_q, n_k].
 * Logits are the exact dot products of the bf16 rows, rounded once to fp64 (max reducer with
 * s_k <= 32: int8-sliced tcgen05 GEMMs + exact corrections, psa_xlogits.cu; otherwise, for
 * heads it cannot represent, or with PSA_IMP_FP64_ONLY: fp64 DMMA), divided by sqrt(d) as the
 * reference does; the row softmax over all n_k*s_k sampled keys is fp64.
 * workspace: psa_importance_workspace_bytes(batch*hq, batch*hkv, n_q, s_q, n_k, s_k) bytes.
 */
size_t psa_importance_workspace_bytes(int64_t bhq, int64_t bkv, int n_q, int s_q, int n_k,
                                      int s_k);
int psa_importance_sampled(const void* q, const void* k, int64_t batch, int hq, int hkv,
                           int64_t n, int d, int b_q, int b_k, const int32_t* q_rows,
                           const int32_t* k_rows, int s_q, int s_k, int reducer, int flags,
                           double* scores, void* workspace, void* stream);

/*
 * K2b — antidiagonal importance.  Replaces importance_antidiagonal
 * (pkg/src/pyrattn/importance.py:97-132).  Query row p of a block reads the keys whose in-block
 * column c has (p + c) % stride == 0 (antidiagonal_selection, importance.py:88-94); logits are
 * fp64 dot products (exact for bf16 inputs) times fl(1/sqrt(d)); row softmax over all picks,
 * probability mass per KV block, mean over the query block's rows.
 * Logits as for psa_importance_sampled (int8-sliced tensor cores when b_k/stride <= 32).
 * Constraints: stride divides b_k, b_k / stride <= 64.  scores: fp64 [batch*hq, n_q, n_k].
 * workspace: psa_antidiag_workspace_bytes(batch*hq, batch*hkv, n, b_q, b_k, stride) bytes
 * (0 = invalid geometry).
 */
size_t psa_antidiag_workspace_bytes(int64_t bhq, int64_t bkv, int64_t n, int b_q, int b_k,
                                    int stride);
int psa_importance_antidiagonal(const void* q, const void* k, int64_t batch, int hq, int hkv,
                                int64_t n, int d, int b_q, int b_k, int stride, int flags,
                                double* scores, void* workspace, void* stream);

/*
 * K3 — level assignment + compact plan.  Replaces assign_threshold / binary_mask /
 * assign_quantile (pkg/src/pyrattn/mask.py:128-179), combine_mask (mask.py:237-247) and
 * causal_premask (mask.py:324-349), and emits the selected-block lists the attention
 * kernel walks.
 * mode 0 (threshold): taus = HOST array of n_cuts thresholds (Alg. 2: stable descending sort,
 *   exactly-rounded row total, sequential Neumaier cumulative sum, searchsorted 'left').
 * mode 1 (quantile) : counts = HOST array of n_cuts cumulative rank counts
 *   (mask.py:161-164 computed on the host exactly as the reference does).
 * caps: optional int8 [batch*hkv, n_k]; causal: apply the causal pre-pass.
 * Outputs: level_map int8 [batch*hq, n_q, n_k];
 *   plan_csr uint16 [batch*hq*n_q, n_k]: per (head, query block) the selected blocks as
 *     (j | (level << 12)), level-major (level 1 first), ascending j within a level;
 *   plan_info int32 [batch*hq*n_q, 2]: (number of entries, total slot rows R: every selected
 *     pooled segment rounded up to a power of two >= 8 rows; an executor with T-row tiles runs
 *     ceil(R / T) tiles — the segments pack perfectly in level-major order);
 *   level_counts uint64 [levels+1] (accumulated: caller zeroes it).
 */
int psa_assign_levels(const double* scores, int64_t batch, int hq, int hkv, int n_q, int n_k,
                      int mode, const double* taus, const int32_t* counts, int n_cuts,
                      const int8_t* caps, int causal, int b_q, int b_k, int levels,
                      int8_t* level_map, uint16_t* plan_csr, int32_t* plan_info,
                      unsigned long long* level_counts, void* stream);

/*
 * Plan from an explicit mask (int8 or int64 [units, n_k], units = batch*hq*n_q), used by the
 * psa_streaming drop-in (pkg/src/pyrattn/attention.py:171-218) when the caller supplies M.
 * Entries outside 0..levels, or pooled levels on causally straddling pairs, set *bad_flag.
 */
int psa_mask_to_plan(const void* mask, int mask_is_int64, int64_t units, int n_q, int n_k,
                     int causal, int b_q, int b_k, int levels, uint16_t* plan_csr,
                     int32_t* plan_info, unsigned long long* level_counts, int32_t* bad_flag,
                     void* stream);

/*
 * K4 — multi-level block-sparse attention forward (tcgen05/TMEM/TMA).  Replaces
 * psa_streaming (pkg/src/pyrattn/attention.py:171-218), level_bias (attention.py:39-44) and
 * the decoupled block-tile executor execute_schedule (pkg/src/pyrattn/scheduler.py:203-269).
 * q: bf16 [batch, hq, n, d]; k, v: bf16 [batch, hkv, n, d]; k_pyr/v_pyr: as produced by
 * psa_pyramid_build. Constraints of the sm_100a kernel: d in {64,128}, b_q <= 128,
 * b_k <= 128.
 * out: bf16 [batch, hq, n, d]; lse: fp32 [batch, hq, n] (natural log; -inf for rows with no
 * key); skipped_rows: device int32 counter (accumulated: caller zeroes it).
 */
int psa_attn_fwd(const void* q, const void* k, const void* v, const void* k_pyr,
                 const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n, int d, int b_q,
                 int b_k, int levels, const uint16_t* plan_csr, const int32_t* plan_info,
                 int causal, void* out, float* lse, int32_t* skipped_rows, void* stream);

/*
 * psa_attn_fwd with the unpermute of pipeline._run_head (pipeline.py:312-313) fused into the
 * epilogue: O and lse of row i of each head are stored at row out_rows[i] (out_rows: DEVICE int64
 * [n], the curve order; NULL = identity).  Only the default kernel has the scatter epilogue.
 */
int psa_attn_fwd_scatter(const void* q, const void* k, const void* v, const void* k_pyr,
                         const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n, int d,
                         int b_q, int b_k, int levels, const uint16_t* plan_csr,
                         const int32_t* plan_info, int causal, void* out, float* lse,
                         int32_t* skipped_rows, const int64_t* out_rows, void* stream);

/*
 * Backward of psa_attn_fwd for a fixed mask (the reference has none).
 * Inputs: the forward's Q, K, V, pyramid, O (out), lse and plan, the level map (int8
 * [batch, hq, n_q, n_k]) and dO (dout, bf16 like O).  Outputs dq [batch, hq, n, d] and dk, dv
 * [batch, hkv, n, d] (bf16, gradients w.r.t. the RAW K/V: pooled levels are differentiated
 * through their means).  workspace: psa_attn_bwd_workspace_bytes(batch, hq, hkv, n, d) bytes.
 * Limit: the dK/dV pass keeps the list of (query head, query block) entries of a KV head in
 * shared memory, 6 bytes each next to ~194 KB of tiles, so (hq / hkv) * n_q must stay below
 * about 5.6K entries per KV head (e.g. 8 query heads per KV head at n = 128K, b_q = 128 is
 * over); beyond it the call returns PSA_EINVAL ("too many query blocks per KV head").
 */
size_t psa_attn_bwd_workspace_bytes(int64_t batch, int hq, int hkv, int64_t n, int d);
int psa_attn_bwd(const void* q, const void* k, const void* v, const void* k_pyr,
                 const void* v_pyr, const void* out, const void* dout, const float* lse,
                 int64_t batch, int hq, int hkv, int64_t n, int d, int b_q, int b_k, int levels,
                 const uint16_t* plan_csr, const int32_t* plan_info, const int8_t* level_map,
                 int causal, void* dq, void* dk, void* dv, void* workspace, void* stream);

/*
 * Token permutation.  Replaces apply_permutation (pkg/src/pyrattn/permute.py:131-137) for the
 * space-filling-curve reorder of pipeline._run_head (pipeline.py:257-263, unpermute :312-313):
 * dst[b][i] = src[b][index[i]] for b < bh, i < n; rows of row_bytes bytes (multiple of 4).
 * index: DEVICE int64 [n] (a bijection; hilbert_order is generated by the Python layer).
 */
int psa_gather_rows(const void* src, int64_t bh, int64_t n, int row_bytes, const int64_t* index,
                    void* dst, void* stream);

/*
 * Query-block work units (a rank owns (batch, head, query-block set); the
 * reference's query blocks are independent given K/V, pkg/src/pyrattn/attention.py:187 and
 * importance.py:52-132 / mask.py:128-151 row by row).  Each *_rows entry point runs its
 * counterpart above on the n_qsel query blocks listed in qblk (DEVICE int32 [n_qsel], any order,
 * the same list for every head of the call); the per-block outputs are compact:
 *   psa_importance_sampled_rows:    q_rows holds the n_qsel * s_q sample rows of the listed
 *                                   blocks (block-major, the reference table's rows of those
 *                                   blocks); scores fp64 [batch*hq, n_qsel, n_k].  (The row list
 *                                   is the table itself, so no qblk is needed.)
 *   psa_importance_antidiagonal_rows: scores fp64 [batch*hq, n_qsel, n_k]; workspace
 *                                   psa_antidiag_workspace_bytes_rows(..., n_qsel) bytes.
 *   psa_assign_levels_rows:         scores / level map / plan rows are the listed blocks (n_q =
 *                                   n_qsel); qblk gives the causal pre-pass the true positions.
 *   psa_attn_fwd_rows:              plan units = batch*hq*n_qsel; out bf16 [batch, hq,
 *                                   n_qsel*b_q, d], lse fp32 [batch, hq, n_qsel*b_q] (compact).
 * Results are bit-identical to the same rows of the full-head call.
 */
int psa_importance_sampled_rows(const void* q, const void* k, int64_t batch, int hq, int hkv,
                                int64_t n, int d, int b_q, int b_k, const int32_t* q_rows,
                                const int32_t* k_rows, int s_q, int s_k, int reducer, int flags,
                                int n_qsel, double* scores, void* workspace, void* stream);
size_t psa_antidiag_workspace_bytes_rows(int64_t bhq, int64_t bkv, int64_t n, int b_q, int b_k,
                                         int stride, int n_qsel);
int psa_importance_antidiagonal_rows(const void* q, const void* k, int64_t batch, int hq, int hkv,
                                     int64_t n, int d, int b_q, int b_k, int stride, int flags,
                                     const int32_t* qblk, int n_qsel, double* scores,
                                     void* workspace, void* stream);
int psa_assign_levels_rows(const double* scores, int64_t batch, int hq, int hkv, int n_q, int n_k,
                           int mode, const double* taus, const int32_t* counts, int n_cuts,
                           const int8_t* caps, int causal, int b_q, int b_k, int levels,
                           const int32_t* qblk, int8_t* level_map, uint16_t* plan_csr,
                           int32_t* plan_info, unsigned long long* level_counts, void* stream);
int psa_attn_fwd_rows(const void* q, const void* k, const void* v, const void* k_pyr,
                      const void* v_pyr, int64_t batch, int hq, int hkv, int64_t n, int d,
                      int b_q, int b_k, int levels, const uint16_t* plan_csr,
                      const int32_t* plan_info, int causal, const int32_t* qblk, int n_qsel,
                      void* out, float* lse, int32_t* skipped_rows, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSA_H_ */
