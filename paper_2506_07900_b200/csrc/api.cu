// C ABI of libinfllm2 (include/infllm2.h): host-side validation and dispatch.
//
// Validation mirrors the reference's ValidationError sites so the Python mirror
// can raise the same exception types: SparseAttentionConfig.__post_init__
// (sparse.py:42-51), two_stage_attention's head/position checks
// (sparse.py:407-420).
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_dispatch.cuh"

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

using namespace infllm2;

namespace infllm2 {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev;
}

cudaError_t smem_attr_once(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;   // (kernel, device) -> bytes set
  const auto key = std::make_pair(kernel, current_device());
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}
}  // namespace infllm2

namespace {

constexpr int kMaxHeadDim = 256;
constexpr int kMaxGroup = 256;
constexpr int64_t kMaxTreeNodes = 1024;

int cuda_status(cudaError_t e) { return e == cudaSuccess ? INFLLM2_OK : INFLLM2_ERR_CUDA; }

int make_shape(const infllm2_geometry* g, int64_t n, int64_t start, int32_t hq, int32_t hkv,
               int32_t d, int64_t cache_len, CallShape* cs) {
  int rc = infllm2_validate_geometry(g);
  if (rc) return rc;
  if (n < 0 || start < 0 || hq <= 0 || hkv <= 0 || d <= 0) return INFLLM2_ERR_SHAPE;
  if (hq % hkv) return INFLLM2_ERR_SHAPE;                       // sparse.py:407-408
  if (d > kMaxHeadDim || hq / hkv > kMaxGroup) return INFLLM2_ERR_UNSUPPORTED;
  if (n > 0 && start + n > cache_len) return INFLLM2_ERR_POSITION;  // sparse.py:417-420
  cs->n = n;
  cs->start = start;
  cs->cache_len = cache_len;
  cs->hq = hq;
  cs->hkv = hkv;
  cs->d = d;
  cs->group = hq / hkv;
  cs->max_sel = infllm2_max_selected(g);
  cs->nk_total = cache_len / g->kernel_stride;
  cs->nb_max = n > 0 ? (start + n - 1) / g->block_size + 1 : 0;
  return INFLLM2_OK;
}

}  // namespace

namespace infllm2 {
long long decode_early_launches();
}

extern "C" {

const char* infllm2_strerror(int code) {
  switch (code) {
    case INFLLM2_OK: return "ok";
    case INFLLM2_ERR_CONFIG: return "invalid sparse attention geometry";
    case INFLLM2_ERR_SHAPE: return "query heads not divisible by KV heads or bad dims";
    case INFLLM2_ERR_POSITION: return "query position beyond cache length";
    case INFLLM2_ERR_CAPACITY: return "cache capacity exceeded";
    case INFLLM2_ERR_WORKSPACE: return "workspace missing or too small";
    case INFLLM2_ERR_UNSUPPORTED: return "shape outside the supported envelope";
    case INFLLM2_ERR_CUDA: return "CUDA launch failed";
    case INFLLM2_ERR_NUMERIC: return "non-finite values in kernel scoring";
    case INFLLM2_ERR_EMPTY: return "empty block selection";
    default: return "unknown error";
  }
}

int infllm2_version(void) { return 100; }

uint64_t infllm2_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

uint64_t infllm2_decode_early_count(void) { return (uint64_t)infllm2::decode_early_launches(); }

int infllm2_validate_geometry(const infllm2_geometry* g) {
  if (!g) return INFLLM2_ERR_CONFIG;
  const int32_t mn = g->block_size < g->kernel_size ? g->block_size : g->kernel_size;
  int32_t smallest = mn < g->kernel_stride ? mn : g->kernel_stride;
  smallest = smallest < g->coarse_stride ? smallest : g->coarse_stride;
  smallest = smallest < g->top_k ? smallest : g->top_k;
  if (smallest <= 0) return INFLLM2_ERR_CONFIG;
  if (g->kernel_stride > g->kernel_size) return INFLLM2_ERR_CONFIG;
  if (g->coarse_stride < g->kernel_stride || g->coarse_stride % g->kernel_stride) return INFLLM2_ERR_CONFIG;
  if (g->n_init_blocks < 0 || g->n_local_blocks < 0) return INFLLM2_ERR_CONFIG;
  return INFLLM2_OK;
}

int32_t infllm2_max_selected(const infllm2_geometry* g) {
  return g->top_k + g->n_init_blocks + g->n_local_blocks;
}

int infllm2_append_kv(void* k_cache, void* v_cache, int64_t cap, int32_t hkv, int32_t d,
                      const void* k_new, const void* v_new, int64_t n_new, int64_t src_row_stride,
                      int32_t src_is_f32, int64_t l_old, infllm2_stream_t stream) {
  if (hkv <= 0 || d <= 0 || n_new < 0 || l_old < 0) return INFLLM2_ERR_SHAPE;
  if (l_old + n_new > cap) return INFLLM2_ERR_CAPACITY;
  return cuda_status(launch_append_kv(k_cache, v_cache, cap, hkv, d, k_new, v_new, n_new,
                                      src_row_stride, src_is_f32, l_old, (cudaStream_t)stream));
}

int infllm2_compress(const void* k_cache, int64_t cap, int32_t hkv, int32_t d, int64_t l_old,
                     int64_t l_new, int64_t means_count_old, int32_t kernel_size, int32_t stride,
                     float* means, void* means_hi, void* means_lo, int64_t means_cap,
                     infllm2_stream_t stream) {
  if (kernel_size <= 0 || stride <= 0 || hkv <= 0 || d <= 0) return INFLLM2_ERR_CONFIG;
  if (l_old < 0 || l_new < 0 || l_new > cap) return INFLLM2_ERR_CAPACITY;
  if ((means_hi == nullptr) != (means_lo == nullptr)) return INFLLM2_ERR_SHAPE;
  const int64_t count = l_new / stride;
  if (count > means_cap) return INFLLM2_ERR_CAPACITY;
  // boundary = old length on append, new length on truncate (sparse.py:129-133)
  const int64_t boundary = l_new >= l_old ? l_old : l_new;
  int64_t first = first_dirty_window(boundary, kernel_size, stride);
  if (first > count) first = count;
  if (first > means_count_old) first = means_count_old;  // F18: windows that never existed
  if (first < 0) first = 0;
  if (first >= count) return INFLLM2_OK;
  // the vectorised streaming kernel when the shape allows (d % 8, p >= stride, alignment)
  const cudaError_t e = launch_append_compress(const_cast<void*>(k_cache), nullptr, cap, hkv, d, nullptr, nullptr, 0, 0,
                                               0, l_new, l_new, first, count, 0, 0, kernel_size, stride, stride, means,
                                               means_hi, means_lo, means_cap, nullptr, nullptr, nullptr, 0,
                                               (cudaStream_t)stream);
  if (e != cudaErrorNotSupported) return cuda_status(e);
  return cuda_status(launch_compress(k_cache, cap, hkv, d, first, count, l_new, kernel_size, stride,
                                     means, means_hi, means_lo, means_cap, (cudaStream_t)stream));
}

int infllm2_append_compress(void* k_cache, void* v_cache, int64_t cap, int32_t hkv, int32_t d, const void* k_new,
                            const void* v_new, int64_t n_new, int64_t src_row_stride, int32_t src_is_f32,
                            int64_t l_old, int64_t l_new, int64_t fine_count_old, int64_t coarse_count_old,
                            int32_t kernel_size, int32_t stride, int32_t coarse_stride, float* fine, void* fine_hi,
                            void* fine_lo, int64_t fine_cap, float* coarse, void* coarse_hi, void* coarse_lo,
                            int64_t coarse_cap, infllm2_stream_t stream) {
  if (kernel_size <= 0 || stride <= 0 || coarse_stride <= 0 || hkv <= 0 || d <= 0) return INFLLM2_ERR_CONFIG;
  if (n_new < 0 || l_old < 0 || l_new < 0 || l_new > cap) return INFLLM2_ERR_CAPACITY;
  if (n_new > 0 && (l_new != l_old + n_new || !k_new || !v_new)) return INFLLM2_ERR_SHAPE;
  if ((fine_hi == nullptr) != (fine_lo == nullptr) || (coarse_hi == nullptr) != (coarse_lo == nullptr))
    return INFLLM2_ERR_SHAPE;
  const int64_t count_f = l_new / stride, count_c = l_new / coarse_stride;
  if (count_f > fine_cap || (coarse && count_c > coarse_cap)) return INFLLM2_ERR_CAPACITY;
  // boundary = old length on append, new length on truncate (sparse.py:129-133)
  const int64_t boundary = l_new >= l_old ? l_old : l_new;
  auto first_of = [&](int32_t st, int64_t count, int64_t count_old) {
    int64_t f = first_dirty_window(boundary, kernel_size, st);
    if (f > count) f = count;
    if (f > count_old) f = count_old;   // F18: windows that never existed
    return f < 0 ? (int64_t)0 : f;
  };
  const int64_t f0 = first_of(stride, count_f, fine_count_old);
  const int64_t c0 = first_of(coarse_stride, count_c, coarse_count_old);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_append_compress(k_cache, v_cache, cap, hkv, d, k_new, v_new, n_new, src_row_stride,
                                         src_is_f32, l_old, l_new, f0, count_f, c0, coarse ? count_c : 0, kernel_size,
                                         stride, coarse_stride, fine, fine_hi, fine_lo, fine_cap, coarse, coarse_hi,
                                         coarse_lo, coarse_cap, st);
  if (e != cudaErrorNotSupported) return cuda_status(e);
  // outside the vectorised envelope: copy, then one re-sync pass per stride
  if (n_new > 0) {
    e = launch_append_kv(k_cache, v_cache, cap, hkv, d, k_new, v_new, n_new, src_row_stride, src_is_f32, l_old, st);
    if (e != cudaSuccess) return INFLLM2_ERR_CUDA;
  }
  if (f0 < count_f) {
    e = launch_compress(k_cache, cap, hkv, d, f0, count_f, l_new, kernel_size, stride, fine, fine_hi, fine_lo,
                        fine_cap, st);
    if (e != cudaSuccess) return INFLLM2_ERR_CUDA;
  }
  if (coarse && c0 < count_c) {
    e = launch_compress(k_cache, cap, hkv, d, c0, count_c, l_new, kernel_size, coarse_stride, coarse, coarse_hi,
                        coarse_lo, coarse_cap, st);
    if (e != cudaSuccess) return INFLLM2_ERR_CUDA;
  }
  return INFLLM2_OK;
}

size_t infllm2_select_workspace_bytes(const infllm2_geometry* g, int64_t n, int32_t hq, int32_t hkv,
                                      int32_t d, int64_t cache_len, int32_t flags) {
  CallShape cs;
  if (make_shape(g, n, cache_len - n > 0 ? cache_len - n : 0, hq, hkv, d, cache_len, &cs)) return 0;
  // The tail rows have the most candidate blocks; size for the whole cache.
  cs.nb_max = cache_len / g->block_size + 1;
  size_t ws = select_simt_workspace(n * hkv, cs.nk_total, cs.nb_max);
  const size_t tc = tc_select_workspace(*g, cs, flags);
  return ws > tc ? ws : tc;
}

int infllm2_select(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n,
                   int64_t start, int32_t hq, int32_t hkv, int32_t d, const float* fine_means,
                   const void* means_hi, const void* means_lo, int64_t means_cap, int64_t cache_len,
                   int32_t* selection, double* sel_scores, void* workspace, size_t workspace_bytes,
                   int32_t flags, infllm2_stream_t stream) {
  CallShape cs;
  int rc = make_shape(g, n, start, hq, hkv, d, cache_len, &cs);
  if (rc) return rc;
  if (n == 0) return INFLLM2_OK;
  if (cs.nk_total > means_cap) return INFLLM2_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  // below the sparsity threshold every row selects every block (the dense
  // path of configs[4]): no scoring, unless the caller wants the scores
  if (sel_scores == nullptr && select_dense_regime(*g, cs))
    return cuda_status(launch_select_dense(*g, cs, selection, st));
  if (!(flags & INFLLM2_FLAG_EXACT_SIMT) && tc_select_supported(*g, cs, means_hi != nullptr)) {
    return cuda_status(launch_select_tc(*g, cs, q, q_row_stride, fine_means, means_hi, means_lo, means_cap,
                                        selection, sel_scores, workspace, workspace_bytes, st));
  }
  const size_t need = select_simt_workspace(n * hkv, cs.nk_total, cs.nb_max);
  if (workspace == nullptr || workspace_bytes < need) return INFLLM2_ERR_WORKSPACE;
  return cuda_status(launch_select_simt(*g, cs, q, q_row_stride, fine_means, means_cap, selection,
                                        sel_scores, workspace, workspace_bytes, st));
}

int infllm2_select_approx(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n,
                          int64_t start, int32_t hq, int32_t hkv, int32_t d, const float* fine_means,
                          const void* means_hi, const void* means_lo, int64_t means_cap,
                          const float* coarse_means, const void* coarse_hi, const void* coarse_lo,
                          int64_t coarse_cap, int64_t cache_len, int32_t* selection, double* sel_scores,
                          void* workspace, size_t workspace_bytes, int32_t flags, infllm2_stream_t stream) {
  CallShape cs;
  int rc = make_shape(g, n, start, hq, hkv, d, cache_len, &cs);
  if (rc) return rc;
  if (n == 0) return INFLLM2_OK;
  if (cs.nk_total > means_cap) return INFLLM2_ERR_CAPACITY;
  const int64_t nc_total = cache_len / g->coarse_stride;
  if (nc_total > 0 && (coarse_means == nullptr || nc_total > coarse_cap)) return INFLLM2_ERR_CAPACITY;
  CoarseArgs ca{coarse_means, coarse_hi, coarse_lo, coarse_cap, nc_total};
  const CoarseArgs* cp = nc_total > 0 ? &ca : nullptr;      // no coarse kernel yet: the exact softmax
  cudaStream_t st = (cudaStream_t)stream;
  if (sel_scores == nullptr && select_dense_regime(*g, cs))   // every block selected: the LSE cannot matter
    return cuda_status(launch_select_dense(*g, cs, selection, st));
  if (!(flags & INFLLM2_FLAG_EXACT_SIMT) && tc_select_supported(*g, cs, means_hi != nullptr) &&
      (cp == nullptr || coarse_hi != nullptr)) {
    return cuda_status(launch_select_tc(*g, cs, q, q_row_stride, fine_means, means_hi, means_lo, means_cap,
                                        selection, sel_scores, workspace, workspace_bytes, st, cp));
  }
  const size_t need = select_simt_workspace(n * hkv, cs.nk_total, cs.nb_max);
  if (workspace == nullptr || workspace_bytes < need) return INFLLM2_ERR_WORKSPACE;
  return cuda_status(launch_select_simt(*g, cs, q, q_row_stride, fine_means, means_cap, selection,
                                        sel_scores, workspace, workspace_bytes, st, cp));
}

int infllm2_attend(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n,
                   int64_t start, int32_t hq, int32_t hkv, int32_t d, const void* k_cache,
                   const void* v_cache, int64_t cap, int64_t cache_len, const int32_t* selection,
                   void* out, float* lse, int32_t flags, infllm2_stream_t stream) {
  CallShape cs;
  int rc = make_shape(g, n, start, hq, hkv, d, cache_len, &cs);
  if (rc) return rc;
  if (cache_len > cap) return INFLLM2_ERR_CAPACITY;
  if (n == 0) return INFLLM2_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int out_f32 = (flags & INFLLM2_FLAG_OUT_F32) ? 1 : 0;
  if (!(flags & INFLLM2_FLAG_EXACT_SIMT) && tc_attend_supported(*g, cs)) {
    return cuda_status(launch_attend_tc(*g, cs, q, q_row_stride, k_cache, v_cache, cap, selection, out, out_f32,
                                        lse, (flags & INFLLM2_FLAG_P_SPLIT) ? 1 : 0, st));
  }
  return cuda_status(launch_attend_simt(*g, cs, q, q_row_stride, k_cache, v_cache, cap, selection, out,
                                        out_f32, lse, st));
}

int infllm2_forward(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n,
                    int64_t start, int32_t hq, int32_t hkv, int32_t d, const void* k_cache,
                    const void* v_cache, int64_t cap, int64_t cache_len, const float* fine_means,
                    const void* means_hi, const void* means_lo, int64_t means_cap, int32_t* selection,
                    double* sel_scores, void* out, float* lse, void* workspace, size_t workspace_bytes,
                    int32_t flags, infllm2_stream_t stream) {
  int rc = infllm2_select(g, q, q_row_stride, n, start, hq, hkv, d, fine_means, means_hi, means_lo,
                          means_cap, cache_len, selection, sel_scores, workspace, workspace_bytes, flags,
                          stream);
  if (rc) return rc;
  return infllm2_attend(g, q, q_row_stride, n, start, hq, hkv, d, k_cache, v_cache, cap, cache_len,
                        selection, out, lse, flags, stream);
}

int infllm2_forward_at(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n,
                       int64_t position, int32_t hq, int32_t hkv, int32_t d, const void* k_cache,
                       const void* v_cache, int64_t cap, int64_t cache_len, const float* fine_means,
                       int64_t means_cap, int32_t* selection, double* sel_scores, void* out, float* lse,
                       void* workspace, size_t workspace_bytes, int32_t flags, infllm2_stream_t stream) {
  CallShape cs;
  int rc = make_shape(g, n > 0 ? 1 : 0, position, hq, hkv, d, cache_len, &cs);   // validates position < L
  if (rc) return rc;
  if (n == 0) return INFLLM2_OK;
  cs.n = n;
  cs.bcast = 1;
  if (cs.nk_total > means_cap) return INFLLM2_ERR_CAPACITY;
  if (cache_len > cap) return INFLLM2_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t need = select_simt_workspace(n * hkv, cs.nk_total, cs.nb_max);
  if (workspace == nullptr || workspace_bytes < need) return INFLLM2_ERR_WORKSPACE;
  rc = cuda_status(launch_select_simt(*g, cs, q, q_row_stride, fine_means, means_cap, selection, sel_scores,
                                      workspace, workspace_bytes, st));
  if (rc) return rc;
  const int out_f32 = (flags & INFLLM2_FLAG_OUT_F32) ? 1 : 0;
  if (!(flags & INFLLM2_FLAG_EXACT_SIMT) && tc_attend_supported(*g, cs))
    return cuda_status(launch_attend_tc(*g, cs, q, q_row_stride, k_cache, v_cache, cap, selection, out, out_f32,
                                        lse, (flags & INFLLM2_FLAG_P_SPLIT) ? 1 : 0, st));
  return cuda_status(launch_attend_simt(*g, cs, q, q_row_stride, k_cache, v_cache, cap, selection, out, out_f32,
                                        lse, st));
}

int infllm2_forward_tree(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n, int32_t hq,
                         int32_t hkv, int32_t d, const void* k_cache, const void* v_cache, int64_t cap,
                         int64_t prefix_len, const float* fine_means, const void* means_hi, const void* means_lo,
                         int64_t means_cap, const uint64_t* tree_words, int32_t words_per_row, int32_t* selection,
                         double* sel_scores, void* out, float* lse, void* workspace, size_t workspace_bytes,
                         int32_t flags, infllm2_stream_t stream) {
  if (prefix_len < 1) return INFLLM2_ERR_POSITION;
  CallShape cs;
  int rc = make_shape(g, n > 0 ? 1 : 0, prefix_len - 1, hq, hkv, d, prefix_len, &cs);   // nodes see every cached row
  if (rc) return rc;
  if (n == 0) return INFLLM2_OK;
  if (n > kMaxTreeNodes || !tree_words || words_per_row < (n + 63) / 64) return INFLLM2_ERR_SHAPE;
  if (prefix_len + n > cap) return INFLLM2_ERR_CAPACITY;   // the draft rows live at [prefix_len, prefix_len + n)
  cs.n = n;
  cs.bcast = 1;
  if (cs.nk_total > means_cap) return INFLLM2_ERR_CAPACITY;
  if (!tc_attend_supported(*g, cs)) return INFLLM2_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream;
  if (!(flags & INFLLM2_FLAG_EXACT_SIMT) && tc_select_supported(*g, cs, means_hi != nullptr)) {
    rc = cuda_status(launch_select_tc(*g, cs, q, q_row_stride, fine_means, means_hi, means_lo, means_cap, selection,
                                      sel_scores, workspace, workspace_bytes, st));
  } else {
    const size_t need = select_simt_workspace(n * hkv, cs.nk_total, cs.nb_max);
    if (workspace == nullptr || workspace_bytes < need) return INFLLM2_ERR_WORKSPACE;
    rc = cuda_status(launch_select_simt(*g, cs, q, q_row_stride, fine_means, means_cap, selection, sel_scores,
                                        workspace, workspace_bytes, st));
  }
  if (rc) return rc;
  const TreeArgs tree{tree_words, (int)n, words_per_row, prefix_len};
  return cuda_status(launch_attend_tc(*g, cs, q, q_row_stride, k_cache, v_cache, cap, selection, out,
                                      (flags & INFLLM2_FLAG_OUT_F32) ? 1 : 0, lse,
                                      (flags & INFLLM2_FLAG_P_SPLIT) ? 1 : 0, st, &tree));
}

size_t infllm2_forward_tree_workspace_bytes(const infllm2_geometry* g, int64_t n, int32_t hq, int32_t hkv,
                                            int32_t d, int64_t prefix_len) {
  CallShape cs;
  if (prefix_len < 1 || n <= 0 || make_shape(g, 1, prefix_len - 1, hq, hkv, d, prefix_len, &cs)) return 0;
  cs.n = n;
  cs.bcast = 1;
  const size_t a = select_simt_workspace(n * hkv, cs.nk_total, cs.nb_max);
  const size_t b = tc_select_workspace(*g, cs, 0);
  return a > b ? a : b;
}

size_t infllm2_forward_at_workspace_bytes(const infllm2_geometry* g, int64_t n, int32_t hkv, int64_t position,
                                          int64_t cache_len) {
  if (infllm2_validate_geometry(g) || n <= 0 || hkv <= 0) return 0;
  return select_simt_workspace(n * hkv, cache_len / g->kernel_stride, position / g->block_size + 1);
}

int infllm2_dense_attend(const infllm2_geometry* g, const void* q, int64_t q_row_stride, int64_t n, int64_t start,
                         int32_t hq, int32_t hkv, int32_t d, const void* k_cache, const void* v_cache, int64_t cap,
                         int64_t cache_len, void* out, float* lse, int32_t flags, infllm2_stream_t stream) {
  CallShape cs;
  int rc = make_shape(g, n, start, hq, hkv, d, cache_len, &cs);
  if (rc) return rc;
  if (cache_len > cap) return INFLLM2_ERR_CAPACITY;
  if (n == 0) return INFLLM2_OK;
  if (!dense_tc_supported(cs)) return INFLLM2_ERR_UNSUPPORTED;
  return cuda_status(launch_dense_tc(cs, q, q_row_stride, k_cache, v_cache, cap, out,
                                     (flags & INFLLM2_FLAG_OUT_F32) ? 1 : 0, lse, (cudaStream_t)stream));
}

int infllm2_dense_regime(const infllm2_geometry* g, int64_t n, int64_t start, int64_t cache_len) {
  CallShape cs;
  if (make_shape(g, n, start, 32, 2, 128, cache_len, &cs) || n == 0) return 0;
  return select_dense_regime(*g, cs) ? 1 : 0;
}

int infllm2_decode_supported(const infllm2_geometry* g, int32_t hq, int32_t hkv, int32_t d) {
  if (infllm2_validate_geometry(g) || hq <= 0 || hkv <= 0 || hq % hkv) return 0;
  return decode_supported(*g, hq, hkv, d) ? 1 : 0;
}

size_t infllm2_decode_table_bytes(int32_t n_seq) { return n_seq > 0 ? decode_table_bytes(n_seq) : 0; }

int infllm2_decode_table_build(const infllm2_seq_desc* seqs, const int64_t* lens, int32_t n_seq, int32_t hkv,
                               int32_t d, void* table, infllm2_stream_t stream) {
  if (n_seq <= 0 || !seqs || !lens || !table) return INFLLM2_ERR_SHAPE;
  for (int s = 0; s < n_seq; ++s)
    if (lens[s] < 0 || lens[s] > seqs[s].cap) return INFLLM2_ERR_CAPACITY;
  return decode_table_build(seqs, lens, n_seq, hkv, d, table, (cudaStream_t)stream);
}

int infllm2_decode_table_link(void* table, int32_t n_seq, const void* next_table, infllm2_stream_t stream) {
  if (n_seq <= 0 || !table) return INFLLM2_ERR_SHAPE;
  return cuda_status(decode_table_link(table, n_seq, const_cast<void*>(next_table), (cudaStream_t)stream));
}

int infllm2_decode_table_lengths(const void* table, int32_t n_seq, int64_t* lens, infllm2_stream_t stream) {
  if (n_seq <= 0 || !table || !lens) return INFLLM2_ERR_SHAPE;
  return cuda_status(decode_table_lengths(table, n_seq, lens, (cudaStream_t)stream));
}

size_t infllm2_decode_workspace_bytes(const infllm2_geometry* g, int32_t n_seq, int32_t hkv, int64_t max_cache_len) {
  if (infllm2_validate_geometry(g) || n_seq <= 0) return 0;
  return decode_workspace_bytes(*g, n_seq, hkv, max_cache_len);
}

int infllm2_decode_step(const infllm2_geometry* g, void* table, int32_t n_seq, int64_t max_len_after, int32_t hq,
                        int32_t hkv, int32_t d, const void* q, const void* k_new, const void* v_new,
                        int32_t* selection, void* out, float* lse, void* workspace, size_t workspace_bytes,
                        int32_t flags, infllm2_stream_t stream) {
  int rc = infllm2_validate_geometry(g);
  if (rc) return rc;
  if (n_seq <= 0 || hq <= 0 || hkv <= 0 || hq % hkv || max_len_after < 1) return INFLLM2_ERR_SHAPE;
  if (!decode_supported(*g, hq, hkv, d)) return INFLLM2_ERR_UNSUPPORTED;
  int share = (flags >> INFLLM2_FLAG_DECODE_SHARE_SHIFT) & 15;
  if (share < 1) share = 1;
  return decode_step(*g, table, n_seq, max_len_after, hq, hkv, d, q, k_new, v_new, selection, out,
                     (flags & INFLLM2_FLAG_OUT_F32) ? 1 : 0, lse, workspace, workspace_bytes, (cudaStream_t)stream,
                     share);
}

}  // extern "C"
