// Blockized KV cache maintenance: row append and kernel-mean compression.
//
// Compression restates build_kernels/_window_mean (sparse.py:70-91) and the
// incremental re-sync (sparse.py:111-133): every window mean is a sequential
// float64 sum over the window's rows, a float64 divide by the clipped width and
// a round-to-nearest float32 — bitwise what numpy computes.  It is HBM-bound.
// The production kernel is stream_compress_kernel (append + fine + coarse
// means in one pass, 16-byte vectors, staged rows); append_kv_kernel and the
// scalar compress_kernel (one thread per (window, head, dim)) serve shapes
// outside its envelope (D % 8 != 0, kernel_size < stride, misaligned rows),
// e.g. the reference's own test geometry.
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

// ---------------------------------------------------------------- streaming append + compress
//
// One pass over the K rows a re-sync touches: a block owns K1_WIN consecutive fine
// windows of one KV head.  It stages their rows ((K1_WIN-1)*s + p of them, one
// contiguous run of the [HKV][cap][D] cache, or of the caller's new rows) in
// shared memory with 16-byte loads, writes the appended K/V rows it owns to the
// cache (16-byte stores), then every thread forms one window's means for 8
// dims from shared memory - the same sequential float64 sum seeded with the
// first row, float64 divide, round-to-nearest float32 as _window_mean
// (sparse.py:70-73) - and stores them (+ the bf16 hi/lo split) as 16-byte
// vectors.  Coarse windows (stride s_c = r*s, same kernel size p) cover the
// SAME rows as fine window j*r, so they are written by that fine window's
// thread: bitwise what build_kernels(keys, p, s_c) gives.  HBM traffic = the
// appended K/V once in, once out + 9/8 of the dirty K rows + the means.
#ifndef K1_WIN
#define K1_WIN 8
#endif
constexpr int kWinPerBlock = K1_WIN;   // windows per block (8: 36 KB of staged rows at s 16, p 32, D 128; measured 3.72 vs 3.58 TB/s for 16, 3.10 for 32)

struct StreamArgs {
  __nv_bfloat16* k_cache;
  __nv_bfloat16* v_cache;
  int64_t cap;
  int hkv, d, dg;                 // dg = d / 8 (16-byte groups per row)
  const void* k_src;              // rows >= l_old come from here (null: compress only)
  const void* v_src;
  int64_t src_row_stride;         // elements
  int src_f32;
  int64_t l_old, l_new;
  int p, s, r;                    // kernel size, stride, coarse stride / stride
  int64_t jf0, count_f;           // fine windows [jf0, count_f) recomputed
  int64_t c0, count_c;            // coarse windows [c0, count_c) written
  int nchunks;
  float* fine;
  __nv_bfloat16* fine_hi;
  __nv_bfloat16* fine_lo;
  int64_t fine_cap;
  float* coarse;
  __nv_bfloat16* coarse_hi;
  __nv_bfloat16* coarse_lo;
  int64_t coarse_cap;
};

__device__ __forceinline__ uint4 load_row8(const StreamArgs& a, const void* src, int64_t r_rel, int g, int dg) {
  const int64_t e = r_rel * a.src_row_stride + (int64_t)g * a.d + dg * 8;
  if (a.src_f32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(src) + e);
    const float4 x = __ldg(p), y = __ldg(p + 1);
    uint4 o;
    __nv_bfloat162 t;
    t = __floats2bfloat162_rn(x.x, x.y); o.x = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(x.z, x.w); o.y = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(y.x, y.y); o.z = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(y.z, y.w); o.w = *reinterpret_cast<uint32_t*>(&t);
    return o;
  }
  return __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(src) + e));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}

__global__ void __launch_bounds__(512) stream_compress_kernel(const StreamArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint4* rows = reinterpret_cast<uint4*>(smem_raw);
  const int g = blockIdx.y, c = blockIdx.x;
  const int64_t jb = a.jf0 + (int64_t)c * kWinPerBlock;
  const int64_t je = jb + kWinPerBlock < a.count_f ? jb + kWinPerBlock : a.count_f;
  // rows this block appends: [B(c), B(c+1)) within [l_old, l_new)
  const int64_t bc = c == 0 ? a.l_old : jb * a.s;
  const int64_t bn = c == a.nchunks - 1 ? a.l_new : (jb + kWinPerBlock) * a.s;
  const int64_t own0 = bc > a.l_old ? bc : a.l_old;
  const int64_t own1 = bn < a.l_new ? bn : a.l_new;
  // staged rows for the windows [jb, je)
  const int64_t st0 = jb * a.s;
  int64_t st1 = je > jb ? (je - 1) * a.s + a.p : st0;
  if (st1 > a.l_new) st1 = a.l_new;
  const __nv_bfloat16* kg = a.k_cache + (int64_t)g * a.cap * a.d;
  const bool append = a.k_src != nullptr;
  const int nth = blockDim.x;
  const int dg_t = threadIdx.x % a.dg;          // blockDim is a multiple of dg: fixed per thread
  const int r_t = threadIdx.x / a.dg, r_step = nth / a.dg;
  // 1. stage K: 16-byte asynchronous copies (every load in flight at once);
  //    a float32 source is converted on the way, four rows per batch
  if (!append || !a.src_f32) {
    for (int64_t r = st0 + r_t; r < st1; r += r_step) {
      const void* src = (append && r >= a.l_old)
                            ? static_cast<const void*>(static_cast<const __nv_bfloat16*>(a.k_src) +
                                                       (r - a.l_old) * a.src_row_stride + (int64_t)g * a.d + dg_t * 8)
                            : static_cast<const void*>(kg + r * a.d + dg_t * 8);
      cp_async16(&rows[(r - st0) * a.dg + dg_t], src);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    for (int64_t r = st0 + r_t; r < st1; r += 4 * r_step) {
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t rr = r + u * r_step;
        if (rr < st1)
          x[u] = rr >= a.l_old ? load_row8(a, a.k_src, rr - a.l_old, g, dg_t)
                               : __ldg(reinterpret_cast<const uint4*>(kg + rr * a.d + dg_t * 8));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (r + u * r_step < st1) rows[(r + u * r_step - st0) * a.dg + dg_t] = x[u];
    }
  }
  // 2. meanwhile: V rows (and K rows past the staged windows) this block owns,
  //    source -> cache, four rows per batch so the loads overlap
  if (append) {
    for (int64_t r = own0 + r_t; r < own1; r += 4 * r_step) {
      uint4 xv[4], xk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t rr = r + u * r_step;
        if (rr < own1) {
          xv[u] = load_row8(a, a.v_src, rr - a.l_old, g, dg_t);
          if (rr >= st1) xk[u] = load_row8(a, a.k_src, rr - a.l_old, g, dg_t);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t rr = r + u * r_step;
        if (rr < own1) {
          const int64_t dst = ((int64_t)g * a.cap + rr) * a.d + dg_t * 8;
          *reinterpret_cast<uint4*>(a.v_cache + dst) = xv[u];
          if (rr >= st1) *reinterpret_cast<uint4*>(a.k_cache + dst) = xk[u];
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // 3. the appended K rows inside the staged range: shared memory -> cache
  if (append) {
    const int64_t lo = own0 > st0 ? own0 : st0, hi = own1 < st1 ? own1 : st1;
    for (int64_t r = lo + r_t; r < hi; r += r_step)
      *reinterpret_cast<uint4*>(a.k_cache + ((int64_t)g * a.cap + r) * a.d + dg_t * 8) = rows[(r - st0) * a.dg + dg_t];
  }
  const int w = threadIdx.x / a.dg, dg = threadIdx.x % a.dg;
  const int64_t j = jb + w;
  if (w >= kWinPerBlock || j >= je) return;
  const int64_t r0 = j * a.s;
  const int64_t wr64 = a.l_new - r0 < a.p ? a.l_new - r0 : a.p;
  const int wr = (int)wr64;
  const uint4* src = rows + (r0 - st0) * a.dg + dg;
  double acc[8];
  {
    const uint4 x = src[0];
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&x);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = (double)__bfloat162float(h[e]);   // numpy's reduce seeds with row 0
  }
#ifdef K1_NOSUM
  if (wr < 0)
#endif
  for (int r = 1; r < wr; ++r) {
    const uint4 x = src[(int64_t)r * a.dg];
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&x);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += (double)__bfloat162float(h[e]);
  }
  float mu[8];
  uint4 hi, lo;
  __nv_bfloat16* hh = reinterpret_cast<__nv_bfloat16*>(&hi);
  __nv_bfloat16* ll = reinterpret_cast<__nv_bfloat16*>(&lo);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    mu[e] = __double2float_rn(acc[e] / (double)wr);
    hh[e] = __float2bfloat16_rn(mu[e]);
    ll[e] = __float2bfloat16_rn(mu[e] - __bfloat162float(hh[e]));
  }
  const int64_t fdst = ((int64_t)g * a.fine_cap + j) * a.d + dg * 8;
  float4* fo = reinterpret_cast<float4*>(a.fine + fdst);
  fo[0] = make_float4(mu[0], mu[1], mu[2], mu[3]);
  fo[1] = make_float4(mu[4], mu[5], mu[6], mu[7]);
  if (a.fine_hi != nullptr) {
    *reinterpret_cast<uint4*>(a.fine_hi + fdst) = hi;
    *reinterpret_cast<uint4*>(a.fine_lo + fdst) = lo;
  }
  if (a.coarse != nullptr && j % a.r == 0) {
    const int64_t jc = j / a.r;
    if (jc >= a.c0 && jc < a.count_c) {
      const int64_t cdst = ((int64_t)g * a.coarse_cap + jc) * a.d + dg * 8;
      float4* co = reinterpret_cast<float4*>(a.coarse + cdst);
      co[0] = fo[0];
      co[1] = fo[1];
      if (a.coarse_hi != nullptr) {
        *reinterpret_cast<uint4*>(a.coarse_hi + cdst) = hi;
        *reinterpret_cast<uint4*>(a.coarse_lo + cdst) = lo;
      }
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

namespace infllm2 {

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Fused append + fine/coarse re-sync (infllm2_append_compress).  Returns
// cudaErrorNotSupported when the shape is outside the vectorised kernel's
// envelope (the caller then runs append + two compress passes).
cudaError_t launch_append_compress(void* k_cache, void* v_cache, int64_t cap, int hkv, int d, const void* k_new,
                                   const void* v_new, int64_t n_new, int64_t src_row_stride, int src_f32,
                                   int64_t l_old, int64_t l_new, int64_t jf0, int64_t count_f, int64_t c0,
                                   int64_t count_c, int p, int s, int sc, float* fine, void* fine_hi, void* fine_lo,
                                   int64_t fine_cap, float* coarse, void* coarse_hi, void* coarse_lo,
                                   int64_t coarse_cap, cudaStream_t stream) {
  if (d % 8 != 0 || d > 256 || p < s || sc % s != 0) return cudaErrorNotSupported;
  const size_t smem = (size_t)((kWinPerBlock - 1) * s + p) * d * 2;
  if (smem > 160 * 1024) return cudaErrorNotSupported;
  if (!aligned16(k_cache) || !aligned16(v_cache) || !aligned16(fine) || (cap * d) % 8 != 0 ||
      (fine_cap * d) % 8 != 0)
    return cudaErrorNotSupported;
  if (fine_hi && (!aligned16(fine_hi) || !aligned16(fine_lo))) return cudaErrorNotSupported;
  if (coarse && (!aligned16(coarse) || (coarse_cap * d) % 8 != 0)) return cudaErrorNotSupported;
  if (coarse_hi && (!aligned16(coarse_hi) || !aligned16(coarse_lo))) return cudaErrorNotSupported;
  if (n_new > 0) {
    const int vec = src_f32 ? 4 : 8;
    if (!aligned16(k_new) || !aligned16(v_new) || src_row_stride % vec != 0) return cudaErrorNotSupported;
  }
  const int r = sc / s;
  // fine windows [jf, count_f) plus every coarse window's fine twin
  int64_t jf = jf0;
  if (coarse != nullptr && c0 < count_c && c0 * r < jf) jf = c0 * r;
  if (jf > count_f) jf = count_f;
  int64_t nch = ceil_div(count_f - jf, kWinPerBlock);
  if (n_new > 0) {
    const int64_t rows_from = jf * s;   // <= l_old: the first dirty window starts at or before the boundary
    const int64_t nr = ceil_div(l_new - rows_from, (int64_t)kWinPerBlock * s);
    if (nr > nch) nch = nr;
  }
  if (nch <= 0) return cudaSuccess;
  StreamArgs a;
  a.k_cache = static_cast<__nv_bfloat16*>(k_cache);
  a.v_cache = static_cast<__nv_bfloat16*>(v_cache);
  a.cap = cap;
  a.hkv = hkv;
  a.d = d;
  a.dg = d / 8;
  a.k_src = n_new > 0 ? k_new : nullptr;
  a.v_src = n_new > 0 ? v_new : nullptr;
  a.src_row_stride = src_row_stride;
  a.src_f32 = src_f32;
  a.l_old = l_old;
  a.l_new = l_new;
  a.p = p;
  a.s = s;
  a.r = r;
  a.jf0 = jf;
  a.count_f = count_f;
  a.c0 = c0;
  a.count_c = count_c;
  a.nchunks = (int)nch;
  a.fine = fine;
  a.fine_hi = static_cast<__nv_bfloat16*>(fine_hi);
  a.fine_lo = static_cast<__nv_bfloat16*>(fine_lo);
  a.fine_cap = fine_cap;
  a.coarse = coarse;
  a.coarse_hi = static_cast<__nv_bfloat16*>(coarse_hi);
  a.coarse_lo = static_cast<__nv_bfloat16*>(coarse_lo);
  a.coarse_cap = coarse_cap;
  cudaError_t e = smem_attr_once((const void*)stream_compress_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  count_launch();
  stream_compress_kernel<<<dim3((unsigned)nch, (unsigned)hkv), kWinPerBlock * (d / 8), smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace infllm2
