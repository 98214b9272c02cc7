/*
 * infllm2.h — C ABI of the B200-native InfLLM v2 block-sparse attention library
 * (libinfllm2.so, sm_100a).
 *
 * The reference (/root/reference, "deskinfer") is pure Python/NumPy and exposes
 * this path only as Python functions; there is no FFI of its own.  Each entry
 * point below replaces one reference interface, cited as file:line into
 * /root/reference/pkg/src/deskinfer/.  INTEGRATION.md shows the ctypes binding a
 * maintainer would add on the reference side.
 *
 * Conventions (all entry points):
 *   - every pointer is a DEVICE pointer unless its comment says "host";
 *   - the library never allocates or frees device memory: the caller passes
 *     workspace (size it with the *_workspace_bytes queries);
 *   - work is enqueued on `stream`; no entry point synchronises the host;
 *   - arguments are validated on the host before any launch; a negative return
 *     is an error code (infllm2_strerror), 0 is success;
 *   - inputs are post-RoPE (the operator never applies rotary embeddings,
 *     matching model.py:427-432).
 *
 * Memory layout in HBM (the "blockized cache"):
 *   K, V cache   bf16  [HKV][cap][D]        (head-major: one KV group's 64-row
 *                                            block is one contiguous 16 KB run)
 *   fine means   f32   [HKV][means_cap][D]  window j = rows [j*s, min(j*s+p, L))
 *   means hi/lo  bf16  [HKV][means_cap][D]  optional split copy of the fine
 *                                            means (hi = bf16(mu), lo = bf16(mu-hi))
 *                                            feeding the tensor-core scorer
 *   q            bf16  (n, HQ, D) rows `q_row_stride` elements apart
 *   out          bf16 or f32 (n, HQ, D) contiguous
 *   lse          f32   (n, HQ)  natural-log normaliser of the stage-2 scores
 *   selection    i32   (n, HKV, max_sel)  ascending block ids, -1 padded,
 *                      max_sel = top_k + n_init_blocks + n_local_blocks
 */
#ifndef INFLLM2_H_
#define INFLLM2_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* infllm2_stream_t; /* a cudaStream_t (CUstream); NULL = legacy default */

/* Error codes.  ValidationError in the reference maps to -1..-5 and -9
 * (container.py:48-49, raised at sparse.py:42-51,407-420,265-266,365-374);
 * NumericError (model.py:24-25, sparse.py:176-177) maps to -8. */
enum {
  INFLLM2_OK = 0,
  INFLLM2_ERR_CONFIG = -1,       /* bad SparseAttentionConfig (sparse.py:42-51)        */
  INFLLM2_ERR_SHAPE = -2,        /* head counts / dims inconsistent (sparse.py:407-408) */
  INFLLM2_ERR_POSITION = -3,     /* query position beyond cache length (sparse.py:417) */
  INFLLM2_ERR_CAPACITY = -4,     /* cache or means capacity too small                  */
  INFLLM2_ERR_WORKSPACE = -5,    /* workspace missing or too small                     */
  INFLLM2_ERR_UNSUPPORTED = -6,  /* shape outside every kernel's envelope (D > 256 ...) */
  INFLLM2_ERR_CUDA = -7,         /* a launch failed                                    */
  INFLLM2_ERR_NUMERIC = -8,      /* non-finite input (debug check only)                */
  INFLLM2_ERR_EMPTY = -9         /* empty selection / nothing to attend                */
};

/* Mirrors SparseAttentionConfig (sparse.py:31-40). */
typedef struct infllm2_geometry {
  int32_t block_size;            /* m   */
  int32_t kernel_size;           /* p   */
  int32_t kernel_stride;         /* s   */
  int32_t coarse_stride;         /* s_c */
  int32_t top_k;                 /* k   */
  int32_t n_init_blocks;
  int32_t n_local_blocks;
  int32_t forced_consume_budget; /* 0/1 */
} infllm2_geometry;

/* flags for infllm2_select / infllm2_attend / infllm2_forward */
enum {
  INFLLM2_FLAG_EXACT_SIMT = 1 << 0,  /* force the CUDA-core float64 scorer (verifier) */
  INFLLM2_FLAG_CHECK_FINITE = 1 << 1,/* report non-finite q / means (costs a sync)    */
  INFLLM2_FLAG_OUT_F32 = 1 << 2,     /* `out` is float32 instead of bf16              */
  INFLLM2_FLAG_P_SPLIT = 1 << 3,     /* stage 2: softmax weights as bf16 hi + lo (two PV
                                        MMAs, ~1e-5 outputs) instead of bf16 P          */
  /* infllm2_decode_step: bits 8..11 = how many decode batches run CONCURRENTLY
   * on the device (micro-batches on separate streams); the fused kernel then
   * sizes its thread-block clusters so that many launches are co-resident. */
  INFLLM2_FLAG_DECODE_SHARE_SHIFT = 8
};

const char* infllm2_strerror(int code);
int infllm2_version(void);            /* major*10000 + minor*100 + patch */
int infllm2_validate_geometry(const infllm2_geometry* g);  /* sparse.py:42-51 */
int32_t infllm2_max_selected(const infllm2_geometry* g);
/* Number of kernel launches this library has enqueued since load (host counter;
 * lets callers report how many of the library's kernels ran in a region). */
uint64_t infllm2_launch_count(void);
/* Number of batched-decode steps launched with the early means stream (the
 * stream's previous decode step used another layer's table, so the lengths and
 * the means tiles are fetched before griddepcontrol.wait; DESIGN §4 K4). */
uint64_t infllm2_decode_early_count(void);

/* Append n_new rows to the blockized cache at rows [l_old, l_old+n_new).
 * k_new/v_new are (n_new, HKV, D), rows `src_row_stride` elements apart,
 * dtype bf16 (src_is_f32 = 0) or f32 (src_is_f32 = 1, rounded to bf16).
 * Replaces LayerCache.append's copy (model.py:322-336). */
int infllm2_append_kv(void* k_cache, void* v_cache, int64_t cap, int32_t hkv, int32_t d,
                      const void* k_new, const void* v_new, int64_t n_new,
                      int64_t src_row_stride, int32_t src_is_f32, int64_t l_old,
                      infllm2_stream_t stream);

/* Re-synchronise kernel means with stride `stride` after the cache length went
 * from l_old to l_new (append: l_new > l_old; truncate: l_new < l_old; full
 * build: l_old = 0).  Recomputes windows j >= first, first = the first window
 * whose rows changed (sparse.py:116-127), clipped to the windows that already
 * existed (reference defect F18).  means_count_old is the number of
 * windows valid before the call (l_old // stride for a cache kept in sync).
 * means_hi / means_lo may be NULL.  Bitwise equal to build_kernels
 * (sparse.py:70-91): sequential f64 sum, f64 divide, f32 round-to-nearest. */
int infllm2_compress(const void* k_cache, int64_t cap, int32_t hkv, int32_t d,
                     int64_t l_old, int64_t l_new, int64_t means_count_old,
                     int32_t kernel_size, int32_t stride,
                     float* means, void* means_hi, void* means_lo, int64_t means_cap,
                     infllm2_stream_t stream);

/* Fused append + re-sync of the fine (stride s) and coarse (stride s_c) kernel
 * means in ONE streaming pass (the prefill path of LayerCache.append +
 * BlockizedLayerCache.notify_append, model.py:322-336, sparse.py:111-133):
 * with n_new > 0 the rows [l_old, l_new = l_old + n_new) are read from k_new /
 * v_new (as infllm2_append_kv) and written to the cache while the dirty
 * windows are recomputed from the staged rows; with n_new = 0 it re-syncs
 * after a truncate (l_new < l_old) or rebuilds (l_old = 0).  fine_count_old /
 * coarse_count_old are the windows valid before the call (F18 clip).  coarse
 * (and its hi/lo split) may be NULL.  Bitwise equal to build_kernels. */
int infllm2_append_compress(void* k_cache, void* v_cache, int64_t cap, int32_t hkv, int32_t d, const void* k_new,
                            const void* v_new, int64_t n_new, int64_t src_row_stride, int32_t src_is_f32,
                            int64_t l_old, int64_t l_new, int64_t fine_count_old, int64_t coarse_count_old,
                            int32_t kernel_size, int32_t stride, int32_t coarse_stride, float* fine, void* fine_hi,
                            void* fine_lo, int64_t fine_cap, float* coarse, void* coarse_hi, void* coarse_lo,
                            int64_t coarse_cap, infllm2_stream_t stream);

/* Workspace for infllm2_select / infllm2_forward (bytes). */
size_t infllm2_select_workspace_bytes(const infllm2_geometry* g, int64_t n, int32_t hq,
                                      int32_t hkv, int32_t d, int64_t cache_len, int32_t flags);

/* Stage 1: per (query row, KV group) block selection.
 * Replaces the per-row scoring/selection of two_stage_attention
 * (sparse.py:415-451): kernel_scores (:163-180) + softmax_f64 (model.py:185-191)
 * + group_scores (:183-188) + block_scores (:201-215) + force_blocks (:218-227)
 * + select_topk (:247-277).  Query row i is at absolute position start + i and
 * sees kernels j < min((start+i)//s + 1, cache_len//s) (sparse.py:426).
 * sel_scores (optional, may be NULL): f64 (n, HKV, max_sel) relevance score of
 * each selected block (the traces' "scores_topk", sparse.py:465). */
int infllm2_select(const infllm2_geometry* g,
                   const void* q, int64_t q_row_stride, int64_t n, int64_t start,
                   int32_t hq, int32_t hkv, int32_t d,
                   const float* fine_means, const void* means_hi, const void* means_lo,
                   int64_t means_cap, int64_t cache_len,
                   int32_t* selection, double* sel_scores,
                   void* workspace, size_t workspace_bytes, int32_t flags,
                   infllm2_stream_t stream);

/* Stage 1 in the opt-in approx-LSE mode (the paper's
 * LSE-approximated stage 1): head h's kernel weights are
 * exp(z_hj - approx_lse(q_h, coarse[:nc_t])) with approx_lse as in
 * sparse.py:292-312 (logsumexp over coarse dots + ln(s_c/s)) and
 * nc_t = min(t // s_c + 1, cache_len // s_c); the rest as infllm2_select.  The
 * reference has no driver for this mode (it changes ~1/3 of selections, SURVEY
 * F3); with cache_len < s_c it is infllm2_select.  coarse_means f32
 * [HKV][coarse_cap][D]; coarse_hi/lo (bf16 split, may be NULL: CUDA-core path)
 * as the fine pair.  Same workspace as infllm2_select. */
int infllm2_select_approx(const infllm2_geometry* g,
                          const void* q, int64_t q_row_stride, int64_t n, int64_t start,
                          int32_t hq, int32_t hkv, int32_t d,
                          const float* fine_means, const void* means_hi, const void* means_lo,
                          int64_t means_cap,
                          const float* coarse_means, const void* coarse_hi, const void* coarse_lo,
                          int64_t coarse_cap, int64_t cache_len,
                          int32_t* selection, double* sel_scores,
                          void* workspace, size_t workspace_bytes, int32_t flags,
                          infllm2_stream_t stream);

/* Stage 2: attention over the selected blocks, causally clipped
 * (sparse_attend, sparse.py:347-384).  Writes out (n, HQ, D) and lse (n, HQ)
 * (lse may be NULL). */
int infllm2_attend(const infllm2_geometry* g,
                   const void* q, int64_t q_row_stride, int64_t n, int64_t start,
                   int32_t hq, int32_t hkv, int32_t d,
                   const void* k_cache, const void* v_cache, int64_t cap, int64_t cache_len,
                   const int32_t* selection, void* out, float* lse, int32_t flags,
                   infllm2_stream_t stream);

/* Stage 1 + stage 2: the whole two_stage_attention call (sparse.py:387-468). */
int infllm2_forward(const infllm2_geometry* g,
                    const void* q, int64_t q_row_stride, int64_t n, int64_t start,
                    int32_t hq, int32_t hkv, int32_t d,
                    const void* k_cache, const void* v_cache, int64_t cap, int64_t cache_len,
                    const float* fine_means, const void* means_hi, const void* means_lo,
                    int64_t means_cap,
                    int32_t* selection, double* sel_scores, void* out, float* lse,
                    void* workspace, size_t workspace_bytes, int32_t flags,
                    infllm2_stream_t stream);

/* Dense causal GQA attention over the cache (row i at position start + i sees
 * rows [0, start + i]): the path below the sparsity threshold (every block
 * selected) and the dense backend (model.py:194-253), on the tensor cores with
 * 8 query rows x 16 heads per MMA tile.  G = 16, D = 128 only
 * (INFLLM2_ERR_UNSUPPORTED otherwise).  out (n, HQ, D), lse (n, HQ) or NULL. */
int infllm2_dense_attend(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n, int64_t start,
                         int32_t hq, int32_t hkv, int32_t d, const void* k_cache, const void* v_cache, int64_t cap,
                         int64_t cache_len, void* out, float* lse, int32_t flags, infllm2_stream_t stream);
/* 1 when every row of the call selects every candidate block (select_topk's
 * budget covers all non-forced candidates of the last row, sparse.py:268). */
int infllm2_dense_regime(const infllm2_geometry* g, int64_t n, int64_t start, int64_t cache_len);

/* Tree-draft verification (specdec.py:565-625, the sparse counterpart of
 * forward_tree): all n query rows sit at the same `position` (the last cached
 * row; each draft node sees the whole prefix), so they share the candidate
 * blocks and forced set; selection per (row, KV group) by the float64 scorer,
 * stage 2 as infllm2_attend.  The tree rows themselves are attended by the
 * caller (a tiny masked attention) and merged by log-sum-exp. */
int infllm2_forward_at(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n,
                       int64_t position, int32_t hq, int32_t hkv, int32_t d, const void* k_cache,
                       const void* v_cache, int64_t cap, int64_t cache_len, const float* fine_means,
                       int64_t means_cap, int32_t* selection, double* sel_scores, void* out, float* lse,
                       void* workspace, size_t workspace_bytes, int32_t flags, infllm2_stream_t stream);
size_t infllm2_forward_at_workspace_bytes(const infllm2_geometry* g, int64_t n, int32_t hkv, int64_t position,
                                          int64_t cache_len);

/* Tree-draft verification on the tensor cores with the uint64 packed ancestor
 * mask (PackedMask specdec.py:117-157, the sparse
 * counterpart of forward_tree specdec.py:565-625).  The n draft nodes' K/V
 * rows must already sit in the cache at rows [prefix_len, prefix_len + n)
 * (written with infllm2_append_kv without advancing the cache length; cap >=
 * prefix_len + n).  Every node is a query at position prefix_len - 1 (it sees
 * every cached row): stage 1 selects its prefix blocks (tcgen05; the float64
 * scorer with INFLLM2_FLAG_EXACT_SIMT), stage 2 attends those blocks AND the
 * tree rows j whose bit j is set in tree_words[i * words_per_row + j / 64], in
 * one online softmax.  n <= 1024.  out (n, HQ, D), lse (n, HQ) or NULL. */
int infllm2_forward_tree(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n, int32_t hq,
                         int32_t hkv, int32_t d, const void* k_cache, const void* v_cache, int64_t cap,
                         int64_t prefix_len, const float* fine_means, const void* means_hi, const void* means_lo,
                         int64_t means_cap, const uint64_t* tree_words, int32_t words_per_row, int32_t* selection,
                         double* sel_scores, void* out, float* lse, void* workspace, size_t workspace_bytes,
                         int32_t flags, infllm2_stream_t stream);
size_t infllm2_forward_tree_workspace_bytes(const infllm2_geometry* g, int64_t n, int32_t hq, int32_t hkv,
                                            int32_t d, int64_t prefix_len);

/* ---------------------------------------------------------------- batched decode
 * S sequences (each its own blockized cache of one layer) append one token and
 * attend one query row: BASELINE configs[3].  The reference's decode is the same
 * per-row procedure with n = 1 (model.py:442-444, specdec.py:717-718). */
typedef struct infllm2_seq_desc {
  void* k_cache;            /* bf16 [HKV][cap][D] */
  void* v_cache;
  int64_t cap;
  float* fine_means;        /* f32 [HKV][means_cap][D] (stride 16) */
  void* means_hi;           /* bf16 split of fine_means */
  void* means_lo;
  int64_t means_cap;
  float* coarse_means;      /* f32 [HKV][coarse_cap][D] */
  int64_t coarse_cap;
} infllm2_seq_desc;

/* 1 when infllm2_decode_step covers this geometry ((G, D) = (16, 128) or
 * (8, 64), s = 16, p = 32, m = 64, max_selected <= 80), else 0: callers step
 * other shapes through infllm2_forward one sequence at a time. */
int infllm2_decode_supported(const infllm2_geometry* g, int32_t hq, int32_t hkv, int32_t d);
/* Device table (descriptors, TMA tensor maps, device-resident lengths). */
size_t infllm2_decode_table_bytes(int32_t n_seq);
/* Build it from HOST descriptors and lengths into `table` (device memory of
 * infllm2_decode_table_bytes bytes).  Synchronises `stream`; rebuild only when a
 * cache is reallocated or its length changes outside infllm2_decode_step. */
int infllm2_decode_table_build(const infllm2_seq_desc* seqs, const int64_t* lens, int32_t n_seq,
                               int32_t hkv, int32_t d, void* table, infllm2_stream_t stream);
/* Link `table` to the NEXT layer's table of the same sequences (or NULL to
 * unlink): while a decode step of this layer runs its dependent tail, each
 * CTA L2-prefetches the piece of the next layer's kernel means it will stream
 * next (a hint: no effect on results).  Stream-ordered; capture-safe.  The
 * link is cleared by infllm2_decode_table_build. */
int infllm2_decode_table_link(void* table, int32_t n_seq, const void* next_table, infllm2_stream_t stream);
/* Copy the table's device-resident lengths (advanced by every decode step,
 * including graph replays) into host `lens` (n_seq entries); synchronises
 * `stream`.  Lets a caller check its host bookkeeping after replays. */
int infllm2_decode_table_lengths(const void* table, int32_t n_seq, int64_t* lens, infllm2_stream_t stream);
size_t infllm2_decode_workspace_bytes(const infllm2_geometry* g, int32_t n_seq, int32_t hkv,
                                      int64_t max_cache_len);
/* One decode step for all sequences: append k_new/v_new ((S, HKV, D) bf16) at
 * each sequence's length (the device length is incremented), re-sync the kernel
 * means, select and attend q ((S, HQ, D) bf16).  max_len_after bounds every
 * sequence's length after the append (sizes the split-K grid).  Caches must have
 * room for one more row.  selection (S, HKV, max_sel), out (S, HQ, D), lse (S, HQ). */
int infllm2_decode_step(const infllm2_geometry* g, void* table, int32_t n_seq, int64_t max_len_after,
                        int32_t hq, int32_t hkv, int32_t d, const void* q, const void* k_new,
                        const void* v_new, int32_t* selection, void* out, float* lse,
                        void* workspace, size_t workspace_bytes, int32_t flags,
                        infllm2_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* INFLLM2_H_ */
