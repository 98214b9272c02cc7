// Stage-1 block selection on CUDA cores, float64 throughout.
//
// This is the any-geometry scorer (any D <= 256, any group size) and the GPU
// verifier for the tensor-core scorer ("K2-exact"): it
// follows two_stage_attention's per-row stage-1 (sparse.py:421-451) with every
// dot product formed in float64, so its only difference from the reference is
// the reference's float32 BLAS rounding of the dots.
//
// One CTA owns one (query row, KV group) item at a time (persistent loop):
//   pass 1  per-head max and sum of exp over the visible kernels
//           (softmax_f64 normaliser, model.py:185-191);
//   pass 2  p_hj = exp(z_hj - max_h) / sum_h, group mean over heads in head
//           order (group_scores, sparse.py:183-188) -> S_j in workspace;
//   blocks  R_b = max S over the block's kernel range (sparse.py:191-215);
//   top-k   forced blocks (sparse.py:218-227) + `budget` best non-forced by
//           (-R, id) (sparse.py:247-277), written ascending.
#include <float.h>

#include "common.cuh"

namespace infllm2 {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct SelectArgs {
  infllm2_geometry g;
  const __nv_bfloat16* q;
  int64_t q_row_stride;
  int64_t n, start, cache_len, nk_total, nb_max;
  int hq, hkv, d, group, max_sel;
  const float* means;
  int64_t means_cap;
  int32_t* selection;
  double* sel_scores;
  double* ws;
  int64_t ws_per_cta;  // doubles
  const float* coarse;   // approx-LSE mode (nullptr: exact softmax)
  int64_t coarse_cap, nc_total;
  int bcast;             // every row at position start
};

__device__ __forceinline__ bool better(double ra, int64_t ba, double rb, int64_t bb) {
  // (score desc, id asc) — np.lexsort((cand, -scores)) order (sparse.py:273)
  return ra > rb || (ra == rb && ba < bb);
}

__global__ void __launch_bounds__(kThreads) select_simt_kernel(SelectArgs a) {
  extern __shared__ double smem[];
  const int G = a.group, D = a.d;
  const int ldq = D + 1;
  double* qs = smem;                            // [G][D+1]
  double* part_m = qs + G * ldq;                // [kThreads]
  double* part_s = part_m + kThreads;           // [kThreads]
  double* hmax = part_s + kThreads;             // [G]
  double* hsum = hmax + G;                      // [G]
  double* ptile = hsum + G;                     // [kThreads]
  double* red_v = ptile + kThreads;             // [kWarps]
  long long* red_b = reinterpret_cast<long long*>(red_v + kWarps);   // [kWarps]
  long long* list = red_b + kWarps;             // [max_sel]
  double* list_score = reinterpret_cast<double*>(list + a.max_sel); // [max_sel]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = a.g.block_size, p = a.g.kernel_size, s = a.g.kernel_stride;
  const double scale = 1.0 / sqrt((double)D);
  const int tj = kThreads / G;                  // kernels per pass-2 tile
  const int active = tj * G;                    // threads with a (kernel, head) slot
  double* S = a.ws + (int64_t)blockIdx.x * a.ws_per_cta;
  double* R = S + a.nk_total;
  const int64_t items = a.n * a.hkv;

  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t i = item / a.hkv;
    const int grp = (int)(item - i * a.hkv);
    const int64_t pos = a.bcast ? a.start : a.start + i;
    const int64_t n_cand = pos / m + 1;
    int64_t nk_t = pos / s + 1;
    if (nk_t > a.nk_total) nk_t = a.nk_total;
    const int64_t qb = pos / m;

    for (int idx = tid; idx < G * D; idx += kThreads) {
      const int h = idx / D, e = idx - h * D;
      qs[h * ldq + e] = (double)bf16_to_f32(a.q[i * a.q_row_stride + (int64_t)(grp * G + h) * D + e]);
    }
    __syncthreads();

    const int h_me = tid % G;
    const int jl_me = tid / G;
    const float* mu_g = a.means + (int64_t)grp * a.means_cap * D;

    // approx-LSE mode: pass 1 runs over the nc_t visible coarse kernels and the
    // normaliser gains ln(s_c / s) (sparse.py:292-312)
    int64_t nc_t = 0;
    if (a.coarse != nullptr) {
      nc_t = pos / a.g.coarse_stride + 1;
      if (nc_t > a.nc_total) nc_t = a.nc_total;
    }
    const bool approx = nc_t > 0;
    const float* p1_base = approx ? a.coarse + (int64_t)grp * a.coarse_cap * D : mu_g;
    const int64_t p1_n = approx ? nc_t : nk_t;

    if (nk_t > 0) {
      // ---- pass 1: per-head max / sum-exp
      double mloc = -DBL_MAX, sloc = 0.0;
      if (tid < active) {
        for (int64_t j = jl_me; j < p1_n; j += tj) {
          const float* mu = p1_base + j * D;
          const double* qh = qs + h_me * ldq;
          double dot = 0.0;
          for (int e = 0; e < D; ++e) dot = fma((double)mu[e], qh[e], dot);
          const double z = dot * scale;
          if (z > mloc) {
            sloc = sloc * exp(mloc - z) + 1.0;
            mloc = z;
          } else {
            sloc += exp(z - mloc);
          }
        }
      }
      part_m[tid] = mloc;
      part_s[tid] = sloc;
      __syncthreads();
      if (tid < G) {
        double M = -DBL_MAX;
        for (int t = tid; t < active; t += G) M = fmax(M, part_m[t]);
        double Ssum = 0.0;
        for (int t = tid; t < active; t += G)
          if (part_s[t] > 0.0) Ssum += part_s[t] * exp(part_m[t] - M);
        hmax[tid] = M;
        hsum[tid] = approx ? Ssum * ((double)a.g.coarse_stride / (double)s) : Ssum;
      }
      __syncthreads();

      // ---- pass 2: p_hj, group mean in head order -> S_j
      for (int64_t j0 = 0; j0 < nk_t; j0 += tj) {
        const int64_t j = j0 + jl_me;
        if (tid < active && j < nk_t) {
          const float* mu = mu_g + j * D;
          const double* qh = qs + h_me * ldq;
          double dot = 0.0;
          for (int e = 0; e < D; ++e) dot = fma((double)mu[e], qh[e], dot);
          ptile[tid] = exp(dot * scale - hmax[h_me]) / hsum[h_me];
        }
        __syncthreads();
        if (tid < tj && j0 + tid < nk_t) {
          double acc = ptile[tid * G];
          for (int h = 1; h < G; ++h) acc += ptile[tid * G + h];
          S[j0 + tid] = acc / (double)G;
        }
        __syncthreads();
      }
    }

    // ---- block scores over clipped candidate blocks
    for (int64_t b = tid; b < n_cand; b += kThreads) {
      double r = 0.0;
      if (nk_t > 0) {
        int64_t end = (b + 1) * m;
        if (end > pos + 1) end = pos + 1;
        int64_t lo, hi;
        kernel_range_for_block(b * m, end, p, s, nk_t, &lo, &hi);
        if (hi > lo) {
          r = S[lo];
          for (int64_t j = lo + 1; j < hi; ++j) r = fmax(r, S[j]);
        }
      }
      R[b] = r;
    }
    __syncthreads();

    // ---- forced set and budget
    const int64_t n_init = a.g.n_init_blocks < n_cand ? a.g.n_init_blocks : n_cand;
    int64_t local_lo = qb + 1;  // empty
    if (a.g.n_local_blocks > 0) {
      local_lo = qb - a.g.n_local_blocks + 1;
      if (local_lo < 0) local_lo = 0;
      if (local_lo < n_init) local_lo = n_init;
    }
    const int64_t n_forced = n_init + (qb + 1 - local_lo);
    int64_t budget = a.g.top_k;
    if (a.g.forced_consume_budget) budget = a.g.top_k - n_forced > 0 ? a.g.top_k - n_forced : 0;
    const int64_t n_free = n_cand - n_forced;
    int cnt = 0;
    if (tid == 0) {
      for (int64_t b = 0; b < n_init; ++b) { list[cnt] = b; list_score[cnt] = R[b]; ++cnt; }
      for (int64_t b = local_lo; b <= qb; ++b) { list[cnt] = b; list_score[cnt] = R[b]; ++cnt; }
    }
    if (budget >= n_free) {
      // dense regime: every candidate is selected
      if (tid == 0)
        for (int64_t b = n_init; b < local_lo; ++b) { list[cnt] = b; list_score[cnt] = R[b]; ++cnt; }
    } else {
      for (int64_t it = 0; it < budget; ++it) {
        double bv = -1.0;
        long long bb = -1;
        for (int64_t b = n_init + tid; b < local_lo; b += kThreads) {
          const double r = R[b];
          if (r >= 0.0 && (bb < 0 || better(r, b, bv, bb))) { bv = r; bb = b; }
        }
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
          const long long ob = __shfl_xor_sync(0xffffffffu, bb, off);
          if (ob >= 0 && (bb < 0 || better(ov, ob, bv, bb))) { bv = ov; bb = ob; }
        }
        if (lane == 0) { red_v[warp] = bv; red_b[warp] = bb; }
        __syncthreads();
        if (tid == 0) {
          double v = red_v[0];
          long long w = red_b[0];
          for (int k = 1; k < kWarps; ++k)
            if (red_b[k] >= 0 && (w < 0 || better(red_v[k], red_b[k], v, w))) { v = red_v[k]; w = red_b[k]; }
          list[cnt] = w;
          list_score[cnt] = v;
          ++cnt;
          R[w] = -1.0;  // taken
        }
        __syncthreads();
      }
    }
    if (tid == 0) {
      // insertion sort by id (<= max_sel entries)
      for (int x = 1; x < cnt; ++x) {
        const long long key = list[x];
        const double sv = list_score[x];
        int y = x - 1;
        while (y >= 0 && list[y] > key) { list[y + 1] = list[y]; list_score[y + 1] = list_score[y]; --y; }
        list[y + 1] = key;
        list_score[y + 1] = sv;
      }
      int32_t* out = a.selection + item * a.max_sel;
      double* osc = a.sel_scores ? a.sel_scores + item * a.max_sel : nullptr;
      for (int x = 0; x < a.max_sel; ++x) {
        out[x] = x < cnt ? (int32_t)list[x] : -1;
        if (osc) osc[x] = x < cnt ? list_score[x] : 0.0;
      }
    }
    __syncthreads();
  }
}

}  // namespace

size_t select_simt_workspace(int64_t items, int64_t nk_total, int64_t nb_max) {
  int64_t grid = items < kNumSMs * 4 ? items : kNumSMs * 4;
  if (grid < 1) grid = 1;
  return (size_t)grid * (size_t)(nk_total + nb_max) * sizeof(double);
}

// Dense regime (every row's budget covers all its non-forced candidates,
// select_topk sparse.py:268-276): the selection is every candidate block
// 0..t//m, ascending -- no scoring needed.  One thread per (row, group, slot).
__global__ void select_dense_kernel(int64_t n, int64_t start, int hkv, int m, int max_sel, int bcast,
                                    int32_t* selection) {
  const int64_t total = n * hkv * max_sel;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / ((int64_t)hkv * max_sel);
    const int slot = (int)(x % max_sel);
    const int64_t pos = bcast ? start : start + i;
    const int64_t n_cand = pos / m + 1;
    selection[x] = slot < n_cand ? slot : -1;
  }
}

bool select_dense_regime(const infllm2_geometry& g, const CallShape& cs) {
  // the last row has the most candidates; budget never grows with position
  const int64_t t = cs.bcast ? cs.start : cs.start + cs.n - 1;
  const int64_t qb = t / g.block_size, n_cand = qb + 1;
  const int64_t n_init = g.n_init_blocks < n_cand ? g.n_init_blocks : n_cand;
  int64_t local_lo = qb + 1;
  if (g.n_local_blocks > 0) {
    local_lo = qb - g.n_local_blocks + 1;
    if (local_lo < 0) local_lo = 0;
    if (local_lo < n_init) local_lo = n_init;
  }
  const int64_t n_forced = n_init + (qb + 1 - local_lo);
  int64_t budget = g.top_k;
  if (g.forced_consume_budget) budget = g.top_k - n_forced > 0 ? g.top_k - n_forced : 0;
  if (cs.max_sel < n_cand) return false;      // the output row could not hold every block
  return budget >= n_cand - n_forced;
}

cudaError_t launch_select_dense(const infllm2_geometry& g, const CallShape& cs, int32_t* selection,
                                cudaStream_t stream) {
  const int64_t total = cs.n * cs.hkv * cs.max_sel;
  const int threads = 256;
  const int64_t blocks64 = (total + threads - 1) / threads;
  const int blocks = (int)(blocks64 < 4 * kNumSMs ? blocks64 : 4 * kNumSMs);
  count_launch();
  select_dense_kernel<<<blocks, threads, 0, stream>>>(cs.n, cs.start, cs.hkv, g.block_size, cs.max_sel, cs.bcast,
                                                       selection);
  return cudaGetLastError();
}

cudaError_t launch_select_simt(const infllm2_geometry& g, const CallShape& cs, const void* q,
                               int64_t q_row_stride, const float* means, int64_t means_cap,
                               int32_t* selection, double* sel_scores, void* ws, size_t ws_bytes,
                               cudaStream_t stream, const CoarseArgs* coarse) {
  SelectArgs a;
  a.bcast = cs.bcast;
  a.coarse = coarse ? coarse->means : nullptr;
  a.coarse_cap = coarse ? coarse->cap : 0;
  a.nc_total = coarse ? coarse->nc_total : 0;
  a.g = g;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.q_row_stride = q_row_stride;
  a.n = cs.n;
  a.start = cs.start;
  a.cache_len = cs.cache_len;
  a.nk_total = cs.nk_total;
  a.nb_max = cs.nb_max;
  a.hq = cs.hq;
  a.hkv = cs.hkv;
  a.d = cs.d;
  a.group = cs.group;
  a.max_sel = cs.max_sel;
  a.means = means;
  a.means_cap = means_cap;
  a.selection = selection;
  a.sel_scores = sel_scores;
  a.ws = static_cast<double*>(ws);
  a.ws_per_cta = cs.nk_total + cs.nb_max;
  const int64_t items = cs.n * cs.hkv;
  int grid = (int)(items < kNumSMs * 4 ? items : kNumSMs * 4);
  if (grid < 1) return cudaSuccess;
  if ((size_t)grid * a.ws_per_cta * sizeof(double) > ws_bytes) return cudaErrorInvalidValue;
  const size_t smem = sizeof(double) * ((size_t)cs.group * (cs.d + 1) + 3 * kThreads + 2 * cs.group +
                                        2 * kWarps + 2 * (size_t)cs.max_sel);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(select_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  select_simt_kernel<<<grid, kThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace infllm2
