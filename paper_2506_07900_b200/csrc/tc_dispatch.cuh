// Tensor-core (tcgen05/TMEM/TMA) kernels for the production geometry and their
// dispatch predicates.  Implemented in select_tc.cu / attend_tc.cu.
#pragma once

#include "common.cuh"

namespace infllm2 {
bool tc_select_supported(const infllm2_geometry& g, const CallShape& cs, bool have_split_means);
size_t tc_select_workspace(const infllm2_geometry& g, const CallShape& cs, int flags);
cudaError_t launch_select_tc(const infllm2_geometry& g, const CallShape& cs, const void* q,
                             int64_t q_row_stride, const float* means, const void* means_hi,
                             const void* means_lo, int64_t means_cap, int32_t* selection,
                             double* sel_scores, void* ws, size_t ws_bytes, cudaStream_t stream,
                             const CoarseArgs* coarse = nullptr);
bool tc_attend_supported(const infllm2_geometry& g, const CallShape& cs);
bool dense_tc_supported(const CallShape& cs);
cudaError_t launch_dense_tc(const CallShape& cs, const void* q, int64_t q_row_stride, const void* k_cache,
                            const void* v_cache, int64_t cap, void* out, int out_f32, float* lse,
                            cudaStream_t stream);
// Tree-draft rows for stage 2 (infllm2_forward_tree): cache rows [row0, row0 + n)
// hold the draft nodes' K/V; row i of the call admits tree row j iff bit j of
// words[i * words_per_row + j / 64] is set.
struct TreeArgs {
  const uint64_t* words;
  int n, words_per_row;
  int64_t row0;
};
cudaError_t launch_attend_tc(const infllm2_geometry& g, const CallShape& cs, const void* q,
                             int64_t q_row_stride, const void* k_cache, const void* v_cache,
                             int64_t cap, const int32_t* selection, void* out, int out_f32,
                             float* lse, int p_split, cudaStream_t stream, const TreeArgs* tree = nullptr);
size_t decode_table_bytes(int n_seq);
int decode_table_build(const infllm2_seq_desc* host, const int64_t* lens, int n_seq, int hkv, int d,
                       void* table_dev, cudaStream_t stream);
cudaError_t decode_table_link(void* table, int n_seq, void* next_table, cudaStream_t stream);
cudaError_t decode_table_lengths(const void* table, int n_seq, int64_t* lens, cudaStream_t stream);
bool decode_supported(const infllm2_geometry& g, int hq, int hkv, int d);
size_t decode_workspace_bytes(const infllm2_geometry& g, int n_seq, int hkv, int64_t max_len);
int decode_step(const infllm2_geometry& g, void* table, int n_seq, int64_t max_len_after, int hq, int hkv, int d,
                const void* q, const void* k_new, const void* v_new, int32_t* selection, void* out, int out_f32,
                float* lse, void* ws, size_t ws_bytes, cudaStream_t stream, int share = 1);
}  // namespace infllm2
