// Stage-2 attention over the selected blocks on CUDA cores (any geometry).
//
// Follows sparse_attend (sparse.py:347-384): the rows of the selected blocks,
// causally clipped to the query position, are scored per head
// (f32 dot -> f64 scale, sparse.py:381), softmax-normalised and mixed with V.
// Online softmax over chunks of kThreads rows keeps shared memory bounded;
// statistics and accumulators are float64.  Also emits the natural-log LSE of
// the same scores (not returned by the reference).
#include <float.h>

#include "common.cuh"

namespace infllm2 {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct AttendArgs {
  int m;
  const __nv_bfloat16* q;
  int64_t q_row_stride;
  int64_t n, start;
  int hq, hkv, d, group, max_sel;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  int64_t cap;
  const int32_t* selection;
  void* out;
  int out_f32;
  float* lse;
  int bcast;             // every row at position start
};

__global__ void __launch_bounds__(kThreads) attend_simt_kernel(AttendArgs a) {
  extern __shared__ double smem[];
  const int G = a.group, D = a.d;
  float* qs = reinterpret_cast<float*>(smem);                 // [G][D]
  double* zs = smem + (G * D + 1) / 2;                         // [G][kThreads]
  double* acc = zs + G * kThreads;                             // [G][D]
  double* mrun = acc + G * D;                                  // [G]
  double* lrun = mrun + G;                                     // [G]
  int* rows = reinterpret_cast<int*>(lrun + G);                // [kThreads]
  int* offs = rows + kThreads;                                 // [max_sel + 2]
  int* blk = offs + a.max_sel + 2;                             // [max_sel]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double scale = 1.0 / sqrt((double)D);
  const int64_t items = a.n * a.hkv;

  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t i = item / a.hkv;
    const int grp = (int)(item - i * a.hkv);
    const int64_t pos = a.bcast ? a.start : a.start + i;
    const int32_t* sel = a.selection + item * a.max_sel;
    for (int idx = tid; idx < G * D; idx += kThreads) {
      const int h = idx / D, e = idx - h * D;
      qs[idx] = bf16_to_f32(a.q[i * a.q_row_stride + (int64_t)(grp * G + h) * D + e]);
      acc[idx] = 0.0;
    }
    if (tid < G) { mrun[tid] = -DBL_MAX; lrun[tid] = 0.0; }
    if (tid == 0) {
      int total = 0, nb = 0;
      for (int x = 0; x < a.max_sel; ++x) {
        const int b = sel[x];
        if (b < 0) break;
        const int64_t s0 = (int64_t)b * a.m;
        if (s0 > pos) continue;
        int64_t e0 = s0 + a.m;
        if (e0 > pos + 1) e0 = pos + 1;
        offs[nb] = total;
        blk[nb] = b;
        total += (int)(e0 - s0);
        ++nb;
      }
      offs[nb] = total;
      offs[a.max_sel + 1] = nb;  // stash the block count in the last slot
    }
    __syncthreads();
    const int nb = offs[a.max_sel + 1];
    const int total = offs[nb];
    const __nv_bfloat16* kg = a.k + (int64_t)grp * a.cap * D;
    const __nv_bfloat16* vg = a.v + (int64_t)grp * a.cap * D;

    for (int c0 = 0; c0 < total; c0 += kThreads) {
      const int t = c0 + tid;
      int r = -1;
      if (t < total) {
        int x = 0;
        while (x + 1 < nb && offs[x + 1] <= t) ++x;
        r = blk[x] * a.m + (t - offs[x]);
      }
      rows[tid] = r;
      for (int h = 0; h < G; ++h) {
        double z = -INFINITY;
        if (r >= 0) {
          const __nv_bfloat16* kr = kg + (int64_t)r * D;
          const float* qh = qs + h * D;
          float dot = 0.f;
          for (int e = 0; e < D; ++e) dot = fmaf(bf16_to_f32(kr[e]), qh[e], dot);
          z = (double)dot * scale;
        }
        zs[h * kThreads + tid] = z;
      }
      __syncthreads();
      const int cnt = total - c0 < kThreads ? total - c0 : kThreads;
      for (int h = warp; h < G; h += kWarps) {
        double* zh = zs + h * kThreads;
        double cmax = -DBL_MAX;
        for (int x = lane; x < cnt; x += 32) cmax = fmax(cmax, zh[x]);
        for (int off = 16; off > 0; off >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
        const double mold = mrun[h];
        const double mnew = fmax(mold, cmax);
        const double corr = exp(mold - mnew);
        double psum = 0.0;
        for (int x = lane; x < cnt; x += 32) {
          const double pv = exp(zh[x] - mnew);
          zh[x] = pv;
          psum += pv;
        }
        for (int off = 16; off > 0; off >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
        __syncwarp();
        for (int e = lane; e < D; e += 32) {
          double av = acc[h * D + e] * corr;
          for (int x = 0; x < cnt; ++x) av = fma(zh[x], (double)bf16_to_f32(vg[(int64_t)rows[x] * D + e]), av);
          acc[h * D + e] = av;
        }
        if (lane == 0) {
          mrun[h] = mnew;
          lrun[h] = lrun[h] * corr + psum;
        }
      }
      __syncthreads();
    }

    for (int idx = tid; idx < G * D; idx += kThreads) {
      const int h = idx / D;
      const double o = lrun[h] > 0.0 ? acc[idx] / lrun[h] : 0.0;
      const int64_t dst = (i * a.hq + grp * G) * (int64_t)D + idx;
      if (a.out_f32)
        static_cast<float*>(a.out)[dst] = (float)o;
      else
        static_cast<__nv_bfloat16*>(a.out)[dst] = __float2bfloat16_rn((float)o);
    }
    if (a.lse && tid < G) a.lse[i * a.hq + grp * G + tid] = (float)(mrun[tid] + log(lrun[tid]));
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_attend_simt(const infllm2_geometry& g, const CallShape& cs, const void* q,
                               int64_t q_row_stride, const void* k_cache, const void* v_cache,
                               int64_t cap, const int32_t* selection, void* out, int out_f32,
                               float* lse, cudaStream_t stream) {
  AttendArgs a;
  a.m = g.block_size;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.q_row_stride = q_row_stride;
  a.n = cs.n;
  a.start = cs.start;
  a.hq = cs.hq;
  a.hkv = cs.hkv;
  a.d = cs.d;
  a.group = cs.group;
  a.max_sel = cs.max_sel;
  a.k = static_cast<const __nv_bfloat16*>(k_cache);
  a.v = static_cast<const __nv_bfloat16*>(v_cache);
  a.cap = cap;
  a.selection = selection;
  a.out = out;
  a.out_f32 = out_f32;
  a.lse = lse;
  a.bcast = cs.bcast;
  const int64_t items = cs.n * cs.hkv;
  const int grid = (int)(items < kNumSMs * 4 ? items : kNumSMs * 4);
  if (grid < 1) return cudaSuccess;
  const size_t smem = sizeof(double) * ((size_t)(cs.group * cs.d + 1) / 2 + (size_t)cs.group * kThreads +
                                        (size_t)cs.group * cs.d + 2 * cs.group) +
                      sizeof(int) * (kThreads + 2 * (size_t)cs.max_sel + 2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(attend_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  attend_simt_kernel<<<grid, kThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace infllm2
