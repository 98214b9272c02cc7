// Blockized KV cache maintenance: row append and kernel-mean compression.
//
// Compression restates build_kernels/_window_mean (sparse.py:70-91) and the
// incremental re-sync (sparse.py:111-133): every window mean is a sequential
// float64 sum over the window's rows, a float64 divide by the clipped width and
// a round-to-nearest float32 — bitwise what numpy computes.  It is HBM-bound:
// each thread owns one (window, head, dim) element, threads of a warp walk
// consecutive dims so every row read is a coalesced run, and the p/s = 2x
// window overlap is served from L2.
#include "common.cuh"

namespace infllm2 {

template <bool kSrcF32>
__global__ void __launch_bounds__(256) append_kv_kernel(
    __nv_bfloat16* __restrict__ k_cache, __nv_bfloat16* __restrict__ v_cache, int64_t cap,
    int hkv, int d, const void* __restrict__ k_new, const void* __restrict__ v_new,
    int64_t n_new, int64_t src_row_stride, int64_t l_old) {
  const int64_t total = n_new * hkv * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / (hkv * d);
    const int rem = (int)(idx - r * hkv * d);
    const int g = rem / d, e = rem - g * d;
    const int64_t src = r * src_row_stride + (int64_t)g * d + e;
    const int64_t dst = ((int64_t)g * cap + l_old + r) * d + e;
    if constexpr (kSrcF32) {
      k_cache[dst] = __float2bfloat16_rn(static_cast<const float*>(k_new)[src]);
      v_cache[dst] = __float2bfloat16_rn(static_cast<const float*>(v_new)[src]);
    } else {
      k_cache[dst] = static_cast<const __nv_bfloat16*>(k_new)[src];
      v_cache[dst] = static_cast<const __nv_bfloat16*>(v_new)[src];
    }
  }
}

// One thread per (window j, head g, dim e) for j in [first, count).
__global__ void __launch_bounds__(256) compress_kernel(
    const __nv_bfloat16* __restrict__ k_cache, int64_t cap, int hkv, int d, int64_t first,
    int64_t count, int64_t length, int p, int s, float* __restrict__ means,
    __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo, int64_t means_cap) {
  const int64_t per_window = (int64_t)hkv * d;
  const int64_t total = (count - first) * per_window;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = first + idx / per_window;
    const int rem = (int)(idx % per_window);
    const int g = rem / d, e = rem - g * d;
    const int64_t row0 = j * s;
    int64_t row1 = row0 + p;
    if (row1 > length) row1 = length;
    const __nv_bfloat16* src = k_cache + ((int64_t)g * cap + row0) * d + e;
    // numpy's add.reduce seeds the accumulator with the first row, so a -0.0
    // first row survives exactly as in the reference.
    double acc = (double)bf16_to_f32(src[0]);
    for (int64_t r = 1; r < row1 - row0; ++r) acc += (double)bf16_to_f32(src[r * d]);
    const float mu = __double2float_rn(acc / (double)(row1 - row0));
    const int64_t dst = ((int64_t)g * means_cap + j) * d + e;
    means[dst] = mu;
    if (hi != nullptr) {
      const __nv_bfloat16 h = __float2bfloat16_rn(mu);
      hi[dst] = h;
      lo[dst] = __float2bfloat16_rn(mu - __bfloat162float(h));
    }
  }
}

static int grid_for(int64_t total, int threads) {
  int64_t blocks = ceil_div(total, threads);
  const int64_t cap = (int64_t)kNumSMs * 16;
  return (int)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

cudaError_t launch_append_kv(void* k_cache, void* v_cache, int64_t cap, int hkv, int d,
                             const void* k_new, const void* v_new, int64_t n_new,
                             int64_t src_row_stride, int src_is_f32, int64_t l_old,
                             cudaStream_t stream) {
  if (n_new <= 0) return cudaSuccess;
  const int grid = grid_for(n_new * hkv * d, 256);
  auto* kc = static_cast<__nv_bfloat16*>(k_cache);
  auto* vc = static_cast<__nv_bfloat16*>(v_cache);
  count_launch();
  if (src_is_f32)
    append_kv_kernel<true><<<grid, 256, 0, stream>>>(kc, vc, cap, hkv, d, k_new, v_new, n_new,
                                                      src_row_stride, l_old);
  else
    append_kv_kernel<false><<<grid, 256, 0, stream>>>(kc, vc, cap, hkv, d, k_new, v_new, n_new,
                                                       src_row_stride, l_old);
  return cudaGetLastError();
}

cudaError_t launch_compress(const void* k_cache, int64_t cap, int hkv, int d, int64_t first,
                            int64_t count, int64_t length, int p, int s, float* means, void* hi,
                            void* lo, int64_t means_cap, cudaStream_t stream) {
  if (count <= first) return cudaSuccess;
  const int grid = grid_for((count - first) * hkv * d, 256);
  count_launch();
  compress_kernel<<<grid, 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(k_cache), cap, hkv, d, first, count, length, p, s, means,
      static_cast<__nv_bfloat16*>(hi), static_cast<__nv_bfloat16*>(lo), means_cap);
  return cudaGetLastError();
}

}  // namespace infllm2
