// Batched single-token decode (BASELINE configs[3]): S sequences, each with its
// own blockized cache, append one token and attend one query row per layer.
//
// Per layer-step, five launches, all batched over sequences:
//   1. decode_append_compress_kernel  new K/V row + the <= 3 kernel windows it
//      touches (fine, hi/lo split, coarse), bitwise as build_kernels
//      (sparse.py:70-91, 111-133); bumps the device-side length.
//   2. decode_stage1_kernel (tcgen05)  split-K over 256-kernel chunks of every
//      (sequence, group): z = mu . q for the 16 heads (M = 128 kernels, N = 16
//      heads, bf16 hi+lo), written to an L2-resident z buffer, plus per-chunk
//      (max, sum 2^z) partials.  HBM-bound on the means (8.4 MB per 128K seq-layer).
//   3. decode_scores_kernel  combine partials -> exact per-head LSE; group
//      score S_j = mean_h 2^(z - lse) (sparse.py:163-188); block max over each
//      block's kernels (sparse.py:191-215) for a range of 64 blocks.
//   4. decode_topk_kernel  one warp per (sequence, group): forced + top-k
//      (sparse.py:218-277) via topk::warp_select.
//   5. attend_tc_kernel with per-sequence K/V tensor maps (stage 2).
#include <float.h>
#include <string.h>

#include <mutex>
#include <unordered_map>
#include <utility>

#include "common.cuh"
#include "sm100.cuh"
#include "tc_dispatch.cuh"
#include "topk.cuh"
#include "decode_common.cuh"

namespace infllm2 {

using namespace dec;

cudaError_t launch_attend_tc_decode(int hq, int hkv, int d, int max_sel, int64_t n_seq, const void* q,
                                    const CUtensorMap* kv_maps, int map_stride, const int64_t* seq_len,
                                    const int32_t* selection, void* out, int out_f32, float* lse,
                                    float* split_ws, cudaStream_t stream);
size_t attend_split_workspace(int64_t n_seq, int hkv, int max_sel);
size_t decode_fused_workspace_bytes(int n_seq, int hkv);
bool decode_fused_supported(const infllm2_geometry& g, int n_seq, int hq, int hkv, int d, int64_t max_len_after,
                            int share);
int decode_fused_step(const infllm2_geometry& g, void* table, int n_seq, int64_t max_len_after, int hq, int hkv,
                      int d, const void* q, const void* k_new, const void* v_new, int32_t* selection, void* out,
                      int out_f32, float* lse, void* ws, cudaStream_t stream, int share, int early);

namespace {

using namespace sm100;

constexpr int kG = 16;
constexpr int kD = 128;
constexpr int kS = 16;             // fine stride
constexpr int kTile = 128;         // kernels per MMA tile
constexpr int kChunk = 1024;       // kernels per stage-1 work item (8 tiles)
constexpr int kBlkChunk = 64;      // blocks per scores work item
// PDL launch: the kernel may start while its predecessor drains; it calls
// pdl_wait() before reading the predecessor's output.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ 1. append + compress

// grid (n_seq, 3): y = 0 writes the new row and re-syncs the first dirty fine
// window, y = 1 the second, y = 2 the coarse window (sparse.py:116-127; first
// dirty window clipped to the windows that already existed, F18).
__global__ void __launch_bounds__(256) decode_append_compress_kernel(void* table, int n_seq, int hkv, int d,
                                                                     const __nv_bfloat16* __restrict__ k_new,
                                                                     const __nv_bfloat16* __restrict__ v_new,
                                                                     int coarse_stride) {
  pdl_launch_dependents();
  pdl_wait();
  const int s = blockIdx.x, role = blockIdx.y;
  TableView tv = table_view(table, n_seq);
  const SeqDesc ds = tv.desc[s];
  const int64_t l_old = tv.len[s];
  const int64_t l_new = l_old + 1;
  const int stride = role < 2 ? kS : coarse_stride;
  int64_t first = l_old < kP ? 0 : (l_old - kP) / stride + 1;
  const int64_t count_old = l_old / stride, count = l_new / stride;
  if (first > count_old) first = count_old;
  const int64_t j = first + (role == 1 ? 1 : 0);
  for (int idx = threadIdx.x; idx < hkv * d; idx += blockDim.x) {
    const int g = idx / d, e = idx - g * d;
    const float knew = __bfloat162float(k_new[(int64_t)s * hkv * d + idx]);
    if (role == 0) {
      ds.k[((int64_t)g * ds.cap + l_old) * d + e] = k_new[(int64_t)s * hkv * d + idx];
      ds.v[((int64_t)g * ds.cap + l_old) * d + e] = v_new[(int64_t)s * hkv * d + idx];
    }
    if (role < 2) {
      if (j >= count) continue;
      const float mu = window_mean(ds.k + (int64_t)g * ds.cap * d, d, j, stride, l_new, e, l_old, knew);
      const int64_t dst = ((int64_t)g * ds.means_cap + j) * d + e;
      ds.fine[dst] = mu;
      const __nv_bfloat16 h = __float2bfloat16_rn(mu);
      ds.hi[dst] = h;
      ds.lo[dst] = __float2bfloat16_rn(mu - __bfloat162float(h));
    } else {
      // every dirty coarse window (two when coarse_stride < kernel_size)
      for (int64_t jc = first; jc < count; ++jc)
        ds.coarse[((int64_t)g * ds.coarse_cap + jc) * d + e] =
            window_mean(ds.k + (int64_t)g * ds.cap * d, d, jc, stride, l_new, e, l_old, knew);
    }
  }
}

// ------------------------------------------------------------------ 2. stage-1 (tcgen05, split-K)

constexpr int kS1Stages = 3;
constexpr uint32_t kMuHalf = kTile * 128;          // 16 KB: 128 kernels x 64 dims
constexpr int kS1Threads = 192;                     // 0 TMA, 1 MMA, 2..5 epilogue

// Head geometries: (G, D) = (16, 128) MiniCPM4-8B, (8, 64) MiniCPM4-0.5B.
// Workspace strides are sized for G = 16 (kG) and shared by both.
template <int G, int D>
struct S1Cfg {
  static constexpr int kDH = D / 64;                          // 64-dim halves
  static constexpr uint32_t kMuStage = 2 * kDH * kMuHalf;     // hi halves, then lo halves
  static constexpr uint32_t kQB = G * D * 2;                  // one query row's group (4 KB / 1 KB)
  static constexpr uint32_t kQHalf = G * 128;                 // one 64-dim half of it
  struct Smem {
    static constexpr uint32_t mu = 0;
    static constexpr uint32_t q = mu + kS1Stages * kMuStage;
    static constexpr uint32_t red = q + 2 * kQB;              // [G][4] m, [G][4] s
    static constexpr uint32_t bars = red + 2 * 128 * G * 4;
    static constexpr uint32_t total = bars + 32 * 8;
  };
};

struct S1Params {
  void* table;
  int n_seq, hkv;
  int64_t nchunk;            // chunks per (seq, group)
  int64_t zstride;           // floats per (seq, group) in zbuf
  float* zbuf;               // [seq][g][kernel][16] log2-domain scores
  float* pstat;              // [seq][g][chunk][16][2]
  float zscale;
};

__device__ __forceinline__ void s1_item(const S1Params& p, const TableView& tv, int64_t item, int* s, int* g,
                                        int64_t* j0, int64_t* j1) {
  const int64_t sg = item / p.nchunk;
  const int64_t c = item - sg * p.nchunk;
  *s = (int)(sg / p.hkv);
  *g = (int)(sg - (int64_t)(*s) * p.hkv);
  const int64_t nk = (tv.len[*s] + 1) / kS;   // length after this step's append
  *j0 = c * kChunk;
  int64_t e = *j0 + kChunk;
  *j1 = e < nk ? e : nk;
}

template <int G, int D>
__global__ void __launch_bounds__(kS1Threads, 1)
decode_stage1_kernel(const __grid_constant__ CUtensorMap tm_q, const S1Params p) {
  using C = S1Cfg<G, D>;
  using S1Smem = typename C::Smem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by pointer arithmetic on the __shared__ array (a uintptr_t round trip
  // loses the address space: every access would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S1Smem::bars);
  uint64_t* mu_full = bars;          // [3]
  uint64_t* mu_empty = bars + 3;     // [3]
  uint64_t* q_full = bars + 6;       // [2]
  uint64_t* q_empty = bars + 8;      // [2]
  uint64_t* s_full = bars + 10;      // [2]
  uint64_t* s_empty = bars + 12;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  float* red_m = reinterpret_cast<float*>(smem + S1Smem::red);
  float* red_s = red_m + 128 * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TableView tv = table_view(p.table, p.n_seq);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kS1Stages; ++i) { mbar_init(mu_full + i, 1); mbar_init(mu_empty + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 4);
    }
    fence_barrier_init();
    tma_prefetch(&tm_q);
  }
  if (warp == 1) tmem_alloc<32>(tmem_slot);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();     // means / lengths of this step's append are visible past here
  const int64_t items = (int64_t)p.n_seq * p.hkv * p.nchunk;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        int s, g;
        int64_t j0, j1;
        s1_item(p, tv, item, &s, &g, &j0, &j1);
        if (j0 >= j1) continue;
        const int qb = it & 1;
        mbar_wait(q_empty + qb, ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(q_full + qb, C::kQB);
        uint8_t* qd = smem + S1Smem::q + qb * C::kQB;
        for (int hh = 0; hh < C::kDH; ++hh) tma_load_3d(qd + hh * C::kQHalf, &tm_q, q_full + qb, 64 * hh, g * G, s);
        const CUtensorMap* mhi = tv.maps + (int64_t)kMaps * s + 2;
        const CUtensorMap* mlo = tv.maps + (int64_t)kMaps * s + 3;
        for (int64_t t0 = j0; t0 < j1; t0 += kTile) {
          mbar_wait(mu_empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(mu_full + stage, C::kMuStage);
          uint8_t* dst = smem + S1Smem::mu + stage * C::kMuStage;
          for (int hh = 0; hh < C::kDH; ++hh) {
            tma_load_3d(dst + hh * kMuHalf, mhi, mu_full + stage, 64 * hh, (int)t0, g);
            tma_load_3d(dst + (C::kDH + hh) * kMuHalf, mlo, mu_full + stage, 64 * hh, (int)t0, g);
          }
          if (++stage == kS1Stages) { stage = 0; phase ^= 1; }
        }
        ++it;
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(128, G);
    int stage = 0, slot = 0;
    uint32_t phase = 0;
    uint32_t s_ph[2] = {0, 0};
    int it = 0;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
      int s, g;
      int64_t j0, j1;
      s1_item(p, tv, item, &s, &g, &j0, &j1);
      if (j0 >= j1) continue;
      const int qb = it & 1;
      mbar_wait(q_full + qb, (it >> 1) & 1);
      const uint32_t q_addr = smem_u32(smem + S1Smem::q + qb * C::kQB);
      for (int64_t t0 = j0; t0 < j1; t0 += kTile) {
        mbar_wait(mu_full + stage, phase);
        mbar_wait(s_empty + slot, s_ph[slot] ^ 1);
        s_ph[slot] ^= 1;
        tc_fence_after();
        if (elect_one()) {
          const uint32_t mu_s = smem_u32(smem + S1Smem::mu + stage * C::kMuStage);
          for (int part = 0; part < 2; ++part) {
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t koff = (k & 3) * 32;
              const uint32_t mu_k = mu_s + part * C::kDH * kMuHalf + (k >> 2) * kMuHalf + koff;
              const uint32_t q_k = q_addr + (k >> 2) * C::kQHalf + koff;
              umma_f16_ss(tmem + slot * 16, sdesc_k_sw128(mu_k), sdesc_k_sw128(q_k), idesc, (part | k) ? 1u : 0u);
            }
          }
          umma_commit(mu_empty + stage);
          umma_commit(s_full + slot);
          if (t0 + kTile >= j1) umma_commit(q_empty + qb);
        }
        __syncwarp();
        if (++stage == kS1Stages) { stage = 0; phase ^= 1; }
        slot ^= 1;
      }
      ++it;
    }
  } else {
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const int etid = (warp - 2) * 32 + lane;
    int slot = 0;
    uint32_t s_ph[2] = {0, 0};
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
      int s, g;
      int64_t j0, j1;
      s1_item(p, tv, item, &s, &g, &j0, &j1);
      float* ps = p.pstat + item * (2 * G);
      if (j0 >= j1) {
        if (etid < G) { ps[2 * etid] = -INFINITY; ps[2 * etid + 1] = 0.f; }
        continue;
      }
      float m[G], sm[G];
#pragma unroll
      for (int h = 0; h < G; ++h) { m[h] = -INFINITY; sm[h] = 0.f; }
      float* zg = p.zbuf + ((int64_t)s * p.hkv + g) * p.zstride;
      for (int64_t t0 = j0; t0 < j1; t0 += kTile) {
        mbar_wait(s_full + slot, s_ph[slot]);
        s_ph[slot] ^= 1;
        tc_fence_after();
        float v[G];
        tmem_ld_n<G>(tmem + lane_base + slot * 16, v);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + slot);
        slot ^= 1;
        const int64_t j = t0 + row;
        if (j < j1) {
#pragma unroll
          for (int h = 0; h < G; ++h) v[h] *= p.zscale;
          float4* dst = reinterpret_cast<float4*>(zg + j * G);
#pragma unroll
          for (int x = 0; x < G / 4; ++x) dst[x] = make_float4(v[4 * x], v[4 * x + 1], v[4 * x + 2], v[4 * x + 3]);
#pragma unroll
          for (int h = 0; h < G; ++h) {
            if (v[h] > m[h]) {
              sm[h] = sm[h] * ex2(m[h] - v[h]) + 1.f;
              m[h] = v[h];
            } else {
              sm[h] += ex2(v[h] - m[h]);
            }
          }
        }
      }
      // (max, sum) per head: warp butterfly, then the 4 warps through smem
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float mm = m[h], ss = sm[h];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const float om = __shfl_xor_sync(0xffffffffu, mm, off);
          const float os = __shfl_xor_sync(0xffffffffu, ss, off);
          const float nm = fmaxf(mm, om);
          ss = (mm == -INFINITY ? 0.f : ss * ex2(mm - nm)) + (om == -INFINITY ? 0.f : os * ex2(om - nm));
          mm = nm;
        }
        if (lane == 0) { red_m[h * 4 + quad] = mm; red_s[h * 4 + quad] = ss; }
      }
      named_bar_sync(1, 128);
      if (etid < G) {
        float M = -INFINITY;
        for (int x = 0; x < 4; ++x) M = fmaxf(M, red_m[etid * 4 + x]);
        float S = 0.f;
        for (int x = 0; x < 4; ++x) {
          const float mm = red_m[etid * 4 + x];
          if (mm != -INFINITY) S += red_s[etid * 4 + x] * ex2(mm - M);
        }
        ps[2 * etid] = M;
        ps[2 * etid + 1] = S;
      }
      named_bar_sync(1, 128);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<32>(tmem);
}

// ------------------------------------------------------------------ 3. block scores

struct ScoreParams {
  void* table;
  int n_seq, hkv, m, kpb;
  int top_k, n_init, n_local, consume, max_sel;
  int64_t nchunk, nbchunk, zstride, nb_cap;
  const float* zbuf;
  const float* pstat;
  float* rbuf;               // [seq][g][nb_cap]
  int32_t* selection;        // [seq][g][max_sel]
};

// Block scores for 64 blocks of one (sequence, group); the last CTA of the
// (sequence, group) to finish (device counter) then runs the top-k over all of
// them, so selection needs no extra launch.
template <int G>
__global__ void __launch_bounds__(256) decode_scores_kernel(const ScoreParams p) {
  __shared__ float lse2[G];
  __shared__ float sk[kBlkChunk * 8 + 8];   // kernels of this block range (kpb <= 8)
  __shared__ float lkey[topk::kListCap];
  __shared__ int lid[topk::kListCap];
  __shared__ int is_last;
  extern __shared__ float rs[];             // staged block scores for the top-k
  pdl_launch_dependents();
  pdl_wait();
  const TableView tv = table_view(p.table, p.n_seq);
  const int64_t item = blockIdx.x;
  const int64_t sg = item / p.nbchunk;
  const int64_t bc = item - sg * p.nbchunk;
  const int s = (int)(sg / p.hkv);
  const int g = (int)(sg - (int64_t)s * p.hkv);
  const int64_t pos = tv.len[s];            // the new token's position
  const int64_t L = pos + 1;
  int64_t nk_t = pos / kS + 1;
  if (nk_t > L / kS) nk_t = L / kS;
  const int64_t n_cand = pos / p.m + 1;
  const int64_t b0 = bc * kBlkChunk;
  if (b0 >= n_cand) return;
  const int64_t b1 = b0 + kBlkChunk < n_cand ? b0 + kBlkChunk : n_cand;
  {
    // per-head LSE from the chunk partials: 256 / G lanes per head, shuffle merge
    constexpr int kLanes = 256 / G;                             // 16 (G = 16) or 32 (G = 8)
    const float* ps = p.pstat + sg * p.nchunk * (2 * G);
    const int h = threadIdx.x / kLanes, sub = threadIdx.x % kLanes;
    float M = -INFINITY, S = 0.f;
    for (int64_t c = sub; c < p.nchunk; c += kLanes) {
      const float mm = ps[c * 2 * G + 2 * h], ss = ps[c * 2 * G + 2 * h + 1];
      if (mm == -INFINITY) continue;
      const float nm = fmaxf(M, mm);
      S = (M == -INFINITY ? 0.f : S * ex2(M - nm)) + ss * ex2(mm - nm);
      M = nm;
    }
#pragma unroll
    for (int off = kLanes / 2; off > 0; off >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, M, off);
      const float os = __shfl_xor_sync(0xffffffffu, S, off);
      const float nm = fmaxf(M, om);
      S = (M == -INFINITY ? 0.f : S * ex2(M - nm)) + (om == -INFINITY ? 0.f : os * ex2(om - nm));
      M = nm;
    }
    if (sub == 0) lse2[h] = M + log2f(S);
  }
  __syncthreads();
  int64_t jlo, jhi, tmp;
  kernel_range_for_block(b0 * p.m, b0 * p.m + p.m, kP, kS, nk_t, &jlo, &tmp);
  jhi = b1 * p.kpb < nk_t ? b1 * p.kpb : nk_t;
  const float* zg = p.zbuf + sg * p.zstride;
  for (int64_t j = jlo + threadIdx.x; j < jhi; j += blockDim.x) {
    const float4* z4 = reinterpret_cast<const float4*>(zg + j * G);
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int x = 0; x < G / 4; ++x) {
      const float4 z = z4[x];
      a0 += ex2(z.x - lse2[4 * x]) + ex2(z.z - lse2[4 * x + 2]);
      a1 += ex2(z.y - lse2[4 * x + 1]) + ex2(z.w - lse2[4 * x + 3]);
    }
    sk[j - jlo] = (a0 + a1) * (1.0f / G);
  }
  __syncthreads();
  float* rrow = p.rbuf + sg * p.nb_cap;
  for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    int64_t end = (b + 1) * p.m;
    if (end > pos + 1) end = pos + 1;
    int64_t lo, hi;
    kernel_range_for_block(b * p.m, end, kP, kS, nk_t, &lo, &hi);
    float r = 0.f;
    if (hi > lo) {
      r = sk[lo - jlo];
      for (int64_t j = lo + 1; j < hi; ++j) r = fmaxf(r, sk[j - jlo]);
    }
    rrow[b] = r;
  }
  // ---- last CTA of this (sequence, group) selects
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int n_active = (int)((n_cand + kBlkChunk - 1) / kBlkChunk);
    const int done = atomicAdd(&tv.counters[s * kMaxHkv + g], 1);
    is_last = (done == n_active - 1);
    if (is_last) tv.counters[s * kMaxHkv + g] = 0;   // reset for the next step
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int64_t b = threadIdx.x; b < n_cand; b += blockDim.x) rs[b] = __ldcg(rrow + b);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const topk::UnitSel us = topk::unit_sel(pos, p.m, p.top_k, p.n_init, p.n_local, p.consume);
  topk::warp_select(rs, us, threadIdx.x, lkey, lid, p.selection + sg * p.max_sel, nullptr, p.max_sel);
}

}  // namespace

// ------------------------------------------------------------------ host API

size_t decode_table_bytes(int n_seq) { return table_bytes(n_seq); }

__global__ void decode_table_link_kernel(void** slot, void* next) { *slot = next; }

cudaError_t decode_table_link(void* table, int n_seq, void* next_table, cudaStream_t stream) {
  const TableView tv = table_view(table, n_seq);
  decode_table_link_kernel<<<1, 1, 0, stream>>>(tv.next, next_table);
  return cudaGetLastError();
}

cudaError_t decode_table_lengths(const void* table, int n_seq, int64_t* lens, cudaStream_t stream) {
  const TableView tv = table_view(const_cast<void*>(table), n_seq);
  const cudaError_t e = cudaMemcpyAsync(lens, tv.len, sizeof(int64_t) * n_seq, cudaMemcpyDeviceToHost, stream);
  return e != cudaSuccess ? e : cudaStreamSynchronize(stream);
}

int decode_table_build(const infllm2_seq_desc* host, const int64_t* lens, int n_seq, int hkv, int d,
                       void* table_dev, cudaStream_t stream) {
  const size_t bytes = table_bytes(n_seq);
  uint8_t* staging = static_cast<uint8_t*>(malloc(bytes));
  if (!staging) return INFLLM2_ERR_CUDA;
  memset(staging, 0, bytes);
  TableView tv = table_view(staging, n_seq);
  SeqDesc* desc = const_cast<SeqDesc*>(tv.desc);
  CUtensorMap* maps = const_cast<CUtensorMap*>(tv.maps);
  int rc = INFLLM2_OK;
  for (int s = 0; s < n_seq && rc == INFLLM2_OK; ++s) {
    const infllm2_seq_desc& h = host[s];
    desc[s].k = static_cast<__nv_bfloat16*>(h.k_cache);
    desc[s].v = static_cast<__nv_bfloat16*>(h.v_cache);
    desc[s].cap = h.cap;
    desc[s].fine = h.fine_means;
    desc[s].hi = static_cast<__nv_bfloat16*>(h.means_hi);
    desc[s].lo = static_cast<__nv_bfloat16*>(h.means_lo);
    desc[s].means_cap = h.means_cap;
    desc[s].coarse = h.coarse_means;
    desc[s].coarse_cap = h.coarse_cap;
    tv.len[s] = lens[s];
    const uint64_t kdims[3] = {(uint64_t)d, (uint64_t)h.cap, (uint64_t)hkv};
    const uint64_t kstr[2] = {(uint64_t)d * 2, (uint64_t)h.cap * d * 2};
    const uint32_t kbox[3] = {64, 64, 1};
    const uint64_t mdims[3] = {(uint64_t)d, (uint64_t)h.means_cap, (uint64_t)hkv};
    const uint64_t mstr[2] = {(uint64_t)d * 2, (uint64_t)h.means_cap * d * 2};
    const uint32_t mbox[3] = {64, (uint32_t)kTile, 1};
    if (!encode_tmap_3d_bf16(&maps[kMaps * s + 0], h.k_cache, kdims, kstr, kbox) ||
        !encode_tmap_3d_bf16(&maps[kMaps * s + 1], h.v_cache, kdims, kstr, kbox) ||
        !encode_tmap_3d_bf16(&maps[kMaps * s + 2], h.means_hi, mdims, mstr, mbox) ||
        !encode_tmap_3d_bf16(&maps[kMaps * s + 3], h.means_lo, mdims, mstr, mbox))
      rc = INFLLM2_ERR_SHAPE;
  }
  if (rc == INFLLM2_OK) {
    // pageable source: the copy completes (staged) before cudaMemcpyAsync returns
    if (cudaMemcpyAsync(table_dev, staging, bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
      rc = INFLLM2_ERR_CUDA;
    else if (cudaStreamSynchronize(stream) != cudaSuccess)
      rc = INFLLM2_ERR_CUDA;
  }
  free(staging);
  return rc;
}

struct DecodeWs {
  float* zbuf;
  float* pstat;
  float* rbuf;
  float* split;
  void* fused;
  int64_t nchunk, nbchunk, zstride, nb_cap;
  size_t bytes;
};

static DecodeWs decode_ws_layout(const infllm2_geometry& g, int n_seq, int hkv, int64_t max_len, void* base) {
  DecodeWs w;
  const int64_t nk = max_len / kS + 1;
  w.nchunk = (nk + kChunk - 1) / kChunk;
  w.zstride = w.nchunk * kChunk * kG;
  w.nb_cap = max_len / g.block_size + 2;
  w.nbchunk = (w.nb_cap + kBlkChunk - 1) / kBlkChunk;
  uint8_t* b = static_cast<uint8_t*>(base);
  size_t off = 0;
  w.zbuf = reinterpret_cast<float*>(b + off);
  off += align_up(sizeof(float) * n_seq * hkv * w.zstride, 256);
  w.pstat = reinterpret_cast<float*>(b + off);
  off += align_up(sizeof(float) * n_seq * hkv * w.nchunk * 2 * kG, 256);
  w.rbuf = reinterpret_cast<float*>(b + off);
  off += align_up(sizeof(float) * n_seq * hkv * w.nb_cap, 256);
  w.split = reinterpret_cast<float*>(b + off);
  off += align_up(attend_split_workspace(n_seq, hkv, infllm2_max_selected(&g)), 256);
  w.fused = b + off;
  off += align_up(decode_fused_workspace_bytes(n_seq, hkv), 256);
  w.bytes = off;
  return w;
}

bool decode_supported(const infllm2_geometry& g, int hq, int hkv, int d) {
  const int G = hkv > 0 ? hq / hkv : 0;
  return hkv > 0 && hkv <= kMaxHkv && hq % hkv == 0 && ((G == 16 && d == 128) || (G == 8 && d == 64)) &&
         g.kernel_stride == kS && g.kernel_size == kP &&
         g.block_size == 64 && g.coarse_stride % kS == 0 && infllm2_max_selected(&g) <= 80;
}

size_t decode_workspace_bytes(const infllm2_geometry& g, int n_seq, int hkv, int64_t max_len) {
  return decode_ws_layout(g, n_seq, hkv, max_len, nullptr).bytes;
}

// Which fused decode table the stream's last decode launch used (nullptr: the
// five-launch path, whose kernels trigger their dependents before their own
// pdl_wait).  A fused step may read its lengths and means before pdl_wait only
// when the previous decode launch on the stream was a fused step of ANOTHER
// table: that step triggers its dependents after its own pdl_wait, so every
// kernel before it — including this table's previous step — has completed, and
// it does not write this table.  Kernels of other kinds in between only delay
// the launch (the append kernels do not use PDL; stage 2 writes no cache).
static long long g_early_launches = 0;
static int note_decode_launch(cudaStream_t stream, const void* table) {
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, const void*> last;
  std::lock_guard<std::mutex> lock(mu);
  auto it = last.find(stream);
  const int early = table != nullptr && it != last.end() && it->second != nullptr && it->second != table;
  last[stream] = table;
  g_early_launches += early;
  return early;
}
long long decode_early_launches() { return g_early_launches; }

// Launches 2-4 of the five-launch path for one head geometry.
template <int G, int D>
static int decode_select(const infllm2_geometry& g, void* table, int n_seq, int hq, int hkv, const void* q,
                         int32_t* selection, const DecodeWs& w, int max_sel, cudaStream_t stream) {
  using C = S1Cfg<G, D>;
  // 2. stage-1 split-K
  S1Params sp;
  sp.table = table;
  sp.n_seq = n_seq;
  sp.hkv = hkv;
  sp.nchunk = w.nchunk;
  sp.zstride = w.zstride;
  sp.zbuf = w.zbuf;
  sp.pstat = w.pstat;
  sp.zscale = 1.4426950408889634f / sqrtf((float)D);
  CUtensorMap tq;
  {
    const uint64_t dims[3] = {(uint64_t)D, (uint64_t)hq, (uint64_t)n_seq};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)hq * D * 2};
    const uint32_t box[3] = {64, (uint32_t)G, 1};
    if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return INFLLM2_ERR_SHAPE;
  }
  const size_t smem1 = C::Smem::total + 1024;
  if (smem_attr_once((const void*)decode_stage1_kernel<G, D>, (int)smem1) != cudaSuccess)
    return INFLLM2_ERR_CUDA;
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items1 = (int64_t)n_seq * hkv * w.nchunk;
  if (launch_pdl(decode_stage1_kernel<G, D>, dim3((unsigned)(items1 < sms ? items1 : sms)), dim3(kS1Threads), smem1,
                 stream, tq, sp) != cudaSuccess)
    return INFLLM2_ERR_CUDA;
  // 3. block scores + (last CTA) top-k
  ScoreParams scp;
  scp.table = table;
  scp.n_seq = n_seq;
  scp.hkv = hkv;
  scp.m = g.block_size;
  scp.kpb = g.block_size / kS;
  scp.top_k = g.top_k;
  scp.n_init = g.n_init_blocks;
  scp.n_local = g.n_local_blocks;
  scp.consume = g.forced_consume_budget;
  scp.max_sel = max_sel;
  scp.nchunk = w.nchunk;
  scp.nbchunk = w.nbchunk;
  scp.zstride = w.zstride;
  scp.nb_cap = w.nb_cap;
  scp.zbuf = w.zbuf;
  scp.pstat = w.pstat;
  scp.rbuf = w.rbuf;
  scp.selection = selection;
  const size_t sc_smem = sizeof(float) * (size_t)w.nb_cap;
  if (sc_smem > 40 * 1024 &&
      smem_attr_once((const void*)decode_scores_kernel<G>, (int)sc_smem) != cudaSuccess)
    return INFLLM2_ERR_UNSUPPORTED;
  if (launch_pdl(decode_scores_kernel<G>, dim3((unsigned)(n_seq * hkv * w.nbchunk)), dim3(256), sc_smem, stream,
                 scp) != cudaSuccess)
    return INFLLM2_ERR_CUDA;
  return INFLLM2_OK;
}

int decode_step(const infllm2_geometry& g, void* table, int n_seq, int64_t max_len_after, int hq, int hkv, int d,
                const void* q, const void* k_new, const void* v_new, int32_t* selection, void* out, int out_f32,
                float* lse, void* ws, size_t ws_bytes, cudaStream_t stream, int share) {
  DecodeWs w = decode_ws_layout(g, n_seq, hkv, max_len_after, ws);
  if (ws == nullptr || ws_bytes < w.bytes) return INFLLM2_ERR_WORKSPACE;
  if (!decode_supported(g, hq, hkv, d)) return INFLLM2_ERR_UNSUPPORTED;
  const int max_sel = infllm2_max_selected(&g);
  const TableView tvd = table_view(table, n_seq);
  const bool g16 = hq / hkv == kG && d == kD;     // else (8, 64): MiniCPM4-0.5B
  const bool fused = decode_fused_supported(g, n_seq, hq, hkv, d, max_len_after, share);
  const int early = note_decode_launch(stream, fused ? table : nullptr);
  if (fused)
    return decode_fused_step(g, table, n_seq, max_len_after, hq, hkv, d, q, k_new, v_new, selection, out, out_f32,
                             lse, w.fused, stream, share, early);
  // 1. append + compress (3 CTAs per sequence)
  if (launch_pdl(decode_append_compress_kernel, dim3(n_seq, 3), dim3(256), 0, stream, table, n_seq, hkv, d,
                 static_cast<const __nv_bfloat16*>(k_new), static_cast<const __nv_bfloat16*>(v_new),
                 (int)g.coarse_stride) != cudaSuccess)
    return INFLLM2_ERR_CUDA;
  // 2-4. stage-1 scores, block scores, top-k
  const int rc = g16 ? decode_select<16, 128>(g, table, n_seq, hq, hkv, q, selection, w, max_sel, stream)
                     : decode_select<8, 64>(g, table, n_seq, hq, hkv, q, selection, w, max_sel, stream);
  if (rc != INFLLM2_OK) return rc;
  // 5. stage 2
  cudaError_t e = launch_attend_tc_decode(hq, hkv, d, max_sel, n_seq, q, tvd.maps, kMaps, tvd.len, selection, out,
                                          out_f32, lse, w.split, stream);
  if (e != cudaSuccess) return INFLLM2_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? INFLLM2_OK : INFLLM2_ERR_CUDA;
}

}  // namespace infllm2
