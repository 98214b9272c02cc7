// Shared device/host helpers for libinfllm2 (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "infllm2.h"

namespace infllm2 {

constexpr int kNumSMs = 148;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ float bf16_to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float bf16bits_to_f32(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// Host-side derived geometry for one call.
struct CallShape {
  int64_t n, start, cache_len;
  int32_t hq, hkv, d, group;
  int32_t max_sel;
  int64_t nk_total;     // cache_len // s
  int64_t nb_max;       // candidate blocks of the last row
  int bcast = 0;        // 1: every row sits at position `start` (tree-draft nodes over a prefix)
};

// First kernel window whose rows change when the cache boundary moves
// (sparse.py:119-120).
__host__ __device__ inline int64_t first_dirty_window(int64_t boundary, int64_t p, int64_t s) {
  return boundary < p ? 0 : (boundary - p) / s + 1;
}

// Half-open kernel range intersecting block [start, end) (sparse.py:191-198).
__host__ __device__ inline void kernel_range_for_block(int64_t start, int64_t end, int64_t p,
                                                       int64_t s, int64_t n_kernels, int64_t* lo,
                                                       int64_t* hi) {
  int64_t l = start < p ? 0 : (start - p) / s + 1;
  int64_t h = (end + s - 1) / s;
  if (h > n_kernels) h = n_kernels;
  if (l > n_kernels) l = n_kernels;
  *lo = l;
  *hi = h;
}

}  // namespace infllm2

// Kernel-launch entry points implemented in the .cu files (host side).
namespace infllm2 {
void count_launch();  // host-side counter behind infllm2_launch_count()
// Raise `kernel`'s dynamic shared-memory limit to `bytes` once per (kernel,
// device): the attribute is per device, so a process driving several GPUs
// sets it on each (thread-safe; later calls are a map lookup).
cudaError_t smem_attr_once(const void* kernel, int bytes);
int current_device();
cudaError_t launch_append_kv(void* k_cache, void* v_cache, int64_t cap, int hkv, int d,
                             const void* k_new, const void* v_new, int64_t n_new,
                             int64_t src_row_stride, int src_is_f32, int64_t l_old,
                             cudaStream_t stream);
cudaError_t launch_compress(const void* k_cache, int64_t cap, int hkv, int d, int64_t first,
                            int64_t count, int64_t length, int p, int s, float* means,
                            void* hi, void* lo, int64_t means_cap, cudaStream_t stream);
// Coarse kernel means (stride s_c) for the opt-in approx-LSE selection mode
// (DESIGN §4 K2p): head weights exp(z - approx_lse) with approx_lse over the
// nc_t = min(t // s_c + 1, nc_total) coarse kernels (sparse.py:292-312).
struct CoarseArgs {
  const float* means;      // f32 [HKV][cap][D]
  const void* hi;          // bf16 split (tensor-core path)
  const void* lo;
  int64_t cap;
  int64_t nc_total;        // cache_len // s_c (>= 1)
};
cudaError_t launch_append_compress(void* k_cache, void* v_cache, int64_t cap, int hkv, int d, const void* k_new,
                                   const void* v_new, int64_t n_new, int64_t src_row_stride, int src_f32,
                                   int64_t l_old, int64_t l_new, int64_t jf0, int64_t count_f, int64_t c0,
                                   int64_t count_c, int p, int s, int sc, float* fine, void* fine_hi, void* fine_lo,
                                   int64_t fine_cap, float* coarse, void* coarse_hi, void* coarse_lo,
                                   int64_t coarse_cap, cudaStream_t stream);
size_t select_simt_workspace(int64_t items, int64_t nk_total, int64_t nb_max);
bool select_dense_regime(const infllm2_geometry& g, const CallShape& cs);
cudaError_t launch_select_dense(const infllm2_geometry& g, const CallShape& cs, int32_t* selection,
                                cudaStream_t stream);
cudaError_t launch_select_simt(const infllm2_geometry& g, const CallShape& cs, const void* q,
                               int64_t q_row_stride, const float* means, int64_t means_cap,
                               int32_t* selection, double* sel_scores, void* ws, size_t ws_bytes,
                               cudaStream_t stream, const CoarseArgs* coarse = nullptr);
cudaError_t launch_attend_simt(const infllm2_geometry& g, const CallShape& cs, const void* q,
                               int64_t q_row_stride, const void* k_cache, const void* v_cache,
                               int64_t cap, const int32_t* selection, void* out, int out_f32,
                               float* lse, cudaStream_t stream);
}  // namespace infllm2
