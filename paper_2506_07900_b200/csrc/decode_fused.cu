// Batched single-token decode in ONE launch (BASELINE configs[3]).
//
// The five-launch path (decode.cu) spends most of a 128K layer-step in launch
// ramps and tails: each phase is a few microseconds of HBM traffic behind a
// kernel boundary.  Here the whole step is one launch of 8-CTA thread-block
// clusters (one CTA per SM); each cluster owns one (sequence, KV group)
// "segment" at a time and its eight CTAs ("pieces") exchange the small
// intermediate results through distributed shared memory, signalled by
// cluster-scope mbarrier arrivals — no global-memory round trips between the
// phases of a segment.  Stage 1's means stream (8.4 MB per 128K segment, the
// HBM-bound part) runs on every SM at once; the dependent tail costs a few
// microseconds.
//
// Per segment, piece r owns the contiguous candidate-block range
// [r*nb/8, (r+1)*nb/8) (nb = pos/64 + 1, pos = the new token's position).
// Warp 0 = TMA producer, warp 1 = MMA issuer, warps 2..5 = 128 epilogue threads.
//   A. append.  The kernel windows that contain the new row (the last one or
//      two) are recomputed bitwise as build_kernels (sparse.py:70-91, 116-127,
//      F18 clip) by every piece whose row range holds them (identical values,
//      so concurrent writers agree); piece 7 also writes the K/V row and the
//      dirty coarse window.
//   B. stage-1 scores z = mu . q for the piece's kernels [4*b0 - 1, 4*b1) (one
//      halo kernel on the left makes every block's kernel range [4b-1, 4b+4)
//      local) on tcgen05: M = 128 kernels, N = 16 heads, bf16 hi + lo means.
//      The z tiles STAY IN TMEM (16 columns per tile).  Per-head (max, sum 2^z)
//      over the owned kernels [4*b0, 4*b1) is exchanged across the cluster ->
//      exact LSE (model.py:172-191).
//   C. S_j = mean_h 2^(z - lse) (sparse.py:163-188) from TMEM, block max R_b
//      (sparse.py:191-215), local top-`budget` by (score desc, id asc)
//      (sparse.py:273); the eight local lists are exchanged and every piece
//      merges them (the global top-B lies in the union of the local top-Bs)
//      into the selection (force_blocks + select_topk, sparse.py:218-277).
//   D. stage 2: the selection's 64-row blocks in 128-row tiles, forced-only
//      tiles first (they do not wait for the selection) and assigned from the
//      last piece down, chosen tiles from piece 0 up.  Per tile: S^T = K . Q^T,
//      masked softmax (sparse.py:370-372), P as bf16 hi + lo, O^T = V^T . P^T,
//      kept as an unnormalised partial in shared memory; after the cluster
//      exchange piece r merges heads 2r, 2r+1 of all partials into the output
//      row and its LSE.
// Clusters loop over segments (the grid is co-resident); the last CTA to read
// the lengths at the start bumps every sequence's device-side length.
// Templated on the head geometry: (G, D) = (16, 128) (MiniCPM4-8B, described
// above) and (8, 64) (MiniCPM4-0.5B: N = 8 heads per MMA, one 64-dim half per
// operand, the combine merges 4 heads per pass).
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "decode_common.cuh"
#include "sm100.cuh"
#include "tc_dispatch.cuh"
#include "topk.cuh"

namespace infllm2 {

using namespace dec;

namespace {

using namespace sm100;

constexpr int kS = 16;
constexpr int kM = 64;
constexpr int kMaxCl = 8;                     // CTAs per cluster = pieces per segment (runtime 3..8)
constexpr int kThreads = 224;                 // warps 0 TMA, 1 MMA, 2..5 epilogue, 6 append
constexpr int kStages = 3;
constexpr int kMaxTiles = 28;                 // z tiles resident in TMEM (16 columns each)
constexpr int kMaxRows = kMaxTiles * 128;     // kernels per piece
constexpr int kMaxPieceBlocks = (kMaxRows - 1) / 4;
constexpr int kMaxBudget = 32;
constexpr int kMaxSeq = 160;
constexpr uint32_t kColS2 = 448;
constexpr uint32_t kColO = 464;

constexpr uint32_t kHalf = 128 * 128;         // 16 KB: 128 rows x 64 bf16
constexpr uint32_t kStageBytes = 4 * kHalf;   // 64 KB ring stage: mu hi/lo tile, or K + V tile

// Head geometry (G heads per KV group, head dim D): (16, 128) MiniCPM4-8B,
// (8, 64) MiniCPM4-0.5B.  With D = 64 a stage holds one 64-dim half of each
// operand (K at 0, V at 2 * kHalf); stage 2's PV still runs M = 128 over O^T
// (lanes >= D read the unused upper half of the V slot and are never stored).
template <int G, int D>
struct FCfg {
  static constexpr int kDH = D / 64;
  static constexpr uint32_t kMuBytes = 2 * kDH * kHalf;        // one stage-1 tile: hi halves, then lo halves
  static constexpr uint32_t kQB = G * D * 2;                    // 4 KB / 1 KB
  static constexpr uint32_t kQHalf = G * 128;                   // one 64-dim half of Q
  static constexpr uint32_t kPHalf = 128 * G * 2;               // P (hi or lo) of one 128-row tile
  static constexpr int kPartStride = G * D + 2 * G;             // floats per stage-2 partial
  struct Smem {
    static constexpr uint32_t ring = 0;
    static constexpr uint32_t q = ring + kStages * kStageBytes;
    static constexpr uint32_t p = q + kQB;                       // P hi/lo; top-k lists / merge flags alias it
    static constexpr uint32_t sarr = p + 2 * kPHalf;             // S_j; merge list; stage-2 partial slots
    static constexpr uint32_t rarr = sarr + kMaxRows * 4;        // R_b; filtered merge list
    static constexpr uint32_t xch = rarr + (kMaxPieceBlocks + 9) * 4;   // published: [2G] LSE partial, [64] candidates
    static constexpr uint32_t red = xch + (2 * G + 2 * kMaxBudget) * 4;
    static constexpr uint32_t bars = (red + (4 * G * 2 + 2 * G + 8) * 4 + 7) / 8 * 8;
    static constexpr uint32_t total = bars + (kMaxTiles + 24) * 8 + 16;
  };
  static_assert(Smem::total + 1024 + 2048 <= 232448, "fused decode shared memory");
  static_assert(topk::kListCap * 8 <= 2 * kPHalf, "top-k lists alias the P buffer");
  static_assert((128 + 2 * 256) * 4 <= 2 * kPHalf, "cta_topk scratch aliases the P buffer");
  static_assert(kPartStride * 4 <= Smem::xch - Smem::sarr, "the stage-2 partial fits the sarr/rarr region");
};

struct Params {
  void* table;
  int n_seq, hkv, hq;
  int top_k, n_init, n_local, consume, max_sel, coarse_stride;
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  int32_t* selection;      // [seq][g][max_sel]
  void* out;
  int out_f32;
  float* lse;
  float zscale;            // log2(e) / sqrt(D)
  int trace;
  int prefetch;            // 1: L2-prefetch the linked next layer's means (infllm2_decode_table_link)
  int early;               // 1: the stream's previous kernel is a fused decode step of ANOTHER table (host-tracked):
                           // the lengths and the first means tiles are read before griddepcontrol.wait
};

// One piece's view of one segment.
struct Info {
  int np;                      // pieces = cluster size
  int s, g;
  int64_t pos, nk, n_cand, b0, b1, r0, r1, dlo;
  int ntiles, dirty_tile;
  // selection geometry (force_blocks / select_topk rules)
  int n_init, local_lo, n_loc, budget, n_free, n_ch, n_sel, nf, tf, t2;
};

__device__ __forceinline__ void seg_info(const Params& p, const int64_t* len, int sg, int rank, int np, Info& I) {
  I.np = np;
  I.s = sg / p.hkv;
  I.g = sg - I.s * p.hkv;
  I.pos = len[I.s];
  const int64_t nb = I.pos / kM + 1;
  I.n_cand = nb;
  I.b0 = rank * nb / np;
  I.b1 = (rank + 1) * nb / np;
  const int64_t L = I.pos + 1;
  I.nk = L / kS;                                       // nk_t == nk for the newest row
  I.r0 = I.b0 == 0 ? 0 : 4 * I.b0 - 1;
  I.r1 = 4 * I.b1 < I.nk ? 4 * I.b1 : I.nk;
  if (I.b1 == I.b0 || I.r1 < I.r0) I.r1 = I.r0;
  I.ntiles = (int)((I.r1 - I.r0 + 127) / 128);
  int64_t first = I.pos < kP ? 0 : (I.pos - kP) / kS + 1;
  const int64_t count_old = I.pos / kS;
  if (first > count_old) first = count_old;
  I.dlo = first;
  I.dirty_tile = -1;
  {
    const int64_t lo = I.dlo > I.r0 ? I.dlo : I.r0;
    if (lo < I.r1) I.dirty_tile = (int)((lo - I.r0) / 128);
  }
  const topk::UnitSel u = topk::unit_sel(I.pos, kM, p.top_k, p.n_init, p.n_local, p.consume);
  I.n_init = (int)u.n_init;
  I.local_lo = (int)u.local_lo;
  I.n_loc = (int)(u.qb + 1 - u.local_lo);
  I.budget = (int)u.budget;
  I.n_free = (int)u.n_free;
  I.n_ch = I.budget >= I.n_free ? I.n_free : I.budget;
  I.n_sel = I.n_init + I.n_ch + I.n_loc;
  I.nf = I.n_init + I.n_loc;
  I.tf = (I.nf + 1) / 2;
  I.t2 = I.tf + (I.n_ch + 1) / 2;
}

// Stage-2 tiles: t < tf hold forced entries (init, then local) 2t, 2t+1; t >= tf
// hold chosen entries 2(t-tf), 2(t-tf)+1.  Forced tiles are owned from the last
// piece down, chosen ones from piece 0 up (round robin).
__device__ __forceinline__ int tile_owner(const Info& I, int t) {
  return t < I.tf ? (((I.np - 1 - t) % I.np) + I.np) % I.np : (t - I.tf) % I.np;
}
__device__ __forceinline__ int tile_blocks(const Info& I, int t) {
  const int n = t < I.tf ? I.nf - 2 * t : I.n_ch - 2 * (t - I.tf);
  return n >= 2 ? 2 : n;
}
__device__ __forceinline__ int tile_block(const Info& I, const int* sel_s, int t, int x) {
  if (x >= tile_blocks(I, t)) return -1;
  if (t < I.tf) {
    const int e = 2 * t + x;
    return e < I.n_init ? e : I.local_lo + (e - I.n_init);
  }
  return sel_s[I.n_init + 2 * (t - I.tf) + x];
}

// ---------------------------------------------------------------- cluster / sync helpers
// Optional phase timeline (INFLLM2_DECODE_TRACE=1): %globaltimer per CTA and
// phase of the first segment, read back with infllm2_debug_decode_trace
// (tools/decode_trace.py).  `on` = launch number + 1; the last kTraceRing
// launches are kept.
constexpr int kTracePts = 24;
constexpr int kTraceRing = 4;
constexpr int kTraceCtas = 160;
__device__ unsigned long long g_trace[kTraceRing * kTraceCtas * kTracePts];
__device__ __forceinline__ void trace(int on, int pt) {
  if (on && blockIdx.x < kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[(((on - 1) % kTraceRing) * kTraceCtas + blockIdx.x) * kTracePts + pt] = t;
  }
}

__device__ long long g_cyc[kTraceCtas * 32];
#define CYC(k)                                                                        \
  do {                                                                                \
    if (tr && tid == 0 && blockIdx.x < kTraceCtas) g_cyc[blockIdx.x * 32 + (k)] = clock64(); \
  } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
// One arrival (release at cluster scope) on the same barrier of every CTA of
// the cluster: called by a whole warp after a CTA barrier; lane r signals CTA r,
// so the eight remote arrivals are in flight together.
__device__ __forceinline__ void arrive_all(uint64_t* bar, int lane, int np) {
  if (lane < np)
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(map_rank(smem_u32(bar), lane))
                 : "memory");
  __syncwarp();
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ float ld_dsmem(const float* local, uint32_t rank) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(map_rank(smem_u32(local), rank)));
  return v;
}
__device__ __forceinline__ float2 ld_dsmem2(const float* local, uint32_t rank) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];"
               : "=f"(v.x), "=f"(v.y)
               : "r"(map_rank(smem_u32(local), rank)));
  return v;
}
// Same for (max, sum 2^(x - max)) pairs.
__device__ __forceinline__ void lse_merge(float& m, float& s, float om, float os) {
  const float nm = fmaxf(m, om);
  s = (m == -INFINITY ? 0.f : s * ex2(m - nm)) + (om == -INFINITY ? 0.f : os * ex2(om - nm));
  m = nm;
}
// (max, sum) pairs of N heads reduce-scattered across the warp: lane l ends
// with head reduce_head_n<N>(l) (lanes sharing bits 4..(5 - log2 N) agree).
template <int N>
__device__ __forceinline__ void warp_reduce_lse_n(float (&m)[N], float (&s)[N], int lane) {
#pragma unroll
  for (int w = N / 2, off = 16; w >= 1; w >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float sm_ = up ? m[i] : m[i + w], ss_ = up ? s[i] : s[i + w];
      float km = up ? m[i + w] : m[i], ks = up ? s[i + w] : s[i];
      lse_merge(km, ks, __shfl_xor_sync(0xffffffffu, sm_, off), __shfl_xor_sync(0xffffffffu, ss_, off));
      m[i] = km;
      s[i] = ks;
    }
  }
#pragma unroll
  for (int off = 16 / N; off >= 1; off >>= 1)
    lse_merge(m[0], s[0], __shfl_xor_sync(0xffffffffu, m[0], off), __shfl_xor_sync(0xffffffffu, s[0], off));
}

__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ int publish_arrive(int* ctr) {
  int old;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
  return old;
}

// Local top-`budget` of r[lo..hi) (indices relative to block id base) by
// (score desc, id asc), one warp; emits exactly `budget` (key, id) pairs, id -1
// padding.  Threshold T0 = budget-th largest lane maximum bounds the answer.
__device__ void local_topk(const float* r, int64_t base, int lo, int hi, int budget, int lane, float* lkey,
                           int* lid, float* out) {
  const int n = hi - lo;
  if (n <= budget) {
    for (int x = lane; x < budget; x += 32) {
      out[2 * x] = x < n ? r[lo + x] : -1.f;
      out[2 * x + 1] = __int_as_float(x < n ? (int)(base + lo + x) : -1);
    }
    return;
  }
  float m = -1.f;
  for (int b = lo + lane; b < hi; b += 32) m = fmaxf(m, r[b]);
  const float t0 = __shfl_sync(0xffffffffu, topk::warp_sort_desc(m, lane), budget - 1);
  int cnt = 0;
  const int cap = topk::kListCap;
  for (int b0 = lo; b0 < hi; b0 += 32) {
    const int b = b0 + lane;
    const float v = b < hi ? r[b] : -2.f;
    const bool f = v >= t0;
    const unsigned mask = __ballot_sync(0xffffffffu, f);
    const int pos = cnt + __popc(mask & ((1u << lane) - 1u));
    if (f && pos < cap) { lkey[pos] = v; lid[pos] = (int)(base + b); }
    cnt += __popc(mask);
  }
  __syncwarp();
  if (cnt <= cap) {
    int taken = 0;
    for (int x0 = 0; x0 < cnt; x0 += 32) {
      const int x = x0 + lane;
      bool keep = false;
      float rk = 0.f;
      int bk = -1;
      if (x < cnt) {
        rk = lkey[x];
        bk = lid[x];
        int rank = 0;
#pragma unroll 8
        for (int f = 0; f < cnt; ++f) rank += topk::better(lkey[f], lid[f], rk, bk) ? 1 : 0;
        keep = rank < budget;
      }
      const unsigned mask = __ballot_sync(0xffffffffu, keep);
      const int pos = taken + __popc(mask & ((1u << lane) - 1u));
      if (keep) { out[2 * pos] = rk; out[2 * pos + 1] = __int_as_float(bk); }
      taken += __popc(mask);
    }
  } else {
    // pathological ties: iterative order statistics
    float pv = INFINITY;
    int pb = -1;
    for (int it = 0; it < budget; ++it) {
      float bv = -1.f;
      int bb = -1;
      for (int b = lo + lane; b < hi; b += 32) {
        const float v = r[b];
        const int id = (int)(base + b);
        if ((pb < 0 || topk::better(pv, pb, v, id)) && (bb < 0 || topk::better(v, id, bv, bb))) { bv = v; bb = id; }
      }
      topk::warp_best_after(bv, bb);
      if (lane == 0) { out[2 * it] = bv; out[2 * it + 1] = __int_as_float(bb); }
      pv = bv;
      pb = bb;
    }
  }
}

// Top-`budget` (<= 32) of r[lo..hi) by (score desc, id asc), id = base + index,
// computed by the 128 epilogue threads (named barrier 1).  A threshold T0 with
// >= budget values reaching it bounds the answer to {r >= T0}; that set is
// compacted and ranked, and the
// result is written SORTED: out[2k], out[2k+1] = key, id bits of the k-th best
// (id -1 padding when fewer than `budget` values).  Returns false (nothing
// written) if the threshold set overflows `cap` (massive exact ties).
__device__ bool cta_topk(const float* r, int64_t base, int lo, int hi, int budget, int tid, int lane, int wq,
                         float* scratch, int* cnt, float* out) {
  const int n = hi - lo;
  float* wmax = scratch;                                  // [4]
  float* lk = scratch + 128;                              // [cap][2]
  const int cap = 256;
  if (n <= budget) {
    // fewer candidates than the budget: all of them (order irrelevant: list not full)
    for (int x = tid; x < budget; x += 128) {
      out[2 * x] = x < n ? r[lo + x] : -1.f;
      out[2 * x + 1] = __int_as_float(x < n ? (int)(base + lo + x) : -1);
    }
    return true;
  }
  float m = -1.f;
  for (int b = lo + tid; b < hi; b += 128) m = fmaxf(m, r[b]);
  const float ws = topk::warp_sort_desc(m, lane);
  if (tid == 0) *cnt = 0;
  // T0 = max over the 4 warps of the warp's budget-th largest thread maximum:
  // that warp alone has >= budget values >= T0, so the top-budget set lies in
  // {r >= T0} (no exact order statistic needed)
  if (lane == budget - 1) wmax[wq] = ws;
  named_bar_sync(1, 128);
  const float t0 = fmaxf(fmaxf(wmax[0], wmax[1]), fmaxf(wmax[2], wmax[3]));
  for (int b = lo + tid; b < hi; b += 128) {
    const float v = r[b];
    if (v >= t0) {
      const int slot = atomicAdd(cnt, 1);
      if (slot < cap) { lk[2 * slot] = v; lk[2 * slot + 1] = __int_as_float((int)(base + b)); }
    }
  }
  named_bar_sync(1, 128);
  const int mm = *cnt;
  if (mm > cap) return false;
  for (int x = tid; x < mm; x += 128) {
    const float rk = lk[2 * x];
    const int bk = __float_as_int(lk[2 * x + 1]);
    int rank = 0;
#pragma unroll 8
    for (int y = 0; y < mm; ++y) rank += topk::better(lk[2 * y], __float_as_int(lk[2 * y + 1]), rk, bk) ? 1 : 0;
    if (rank < budget) { out[2 * rank] = rk; out[2 * rank + 1] = __int_as_float(bk); }
  }
  return true;
}

template <int G, int D>
__global__ void __launch_bounds__(kThreads, 1)
decode_cluster_kernel(const __grid_constant__ CUtensorMap tm_q, const Params p) {
  using C = FCfg<G, D>;
  using Smem = typename C::Smem;
  constexpr int kG = G;
  constexpr int kD = D;
  constexpr int kDH = C::kDH;
  constexpr uint32_t kQB = C::kQB;
  constexpr uint32_t kPHalf = C::kPHalf;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by pointer arithmetic on the __shared__ array (a uintptr_t round trip
  // loses the address space: every access would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* full = bars;                 // [3]
  uint64_t* empty = bars + 3;            // [3]
  uint64_t* q_full = bars + 6;
  uint64_t* q_empty = bars + 7;
  uint64_t* appended = bars + 8;         // 32 append-warp arrivals: dirty windows + K/V row stored
  uint64_t* z_free = bars + 9;           // 128 epilogue arrivals: z tiles read, TMEM reusable
  uint64_t* s2_full = bars + 10;
  uint64_t* s2_empty = bars + 11;        // 4 warps
  uint64_t* p_full = bars + 12;          // 4 warps
  uint64_t* o_full = bars + 13;
  uint64_t* o_empty = bars + 14;         // 4 warps
  uint64_t* sel_ready = bars + 15;       // selection merged into sel_s
  uint64_t* x1 = bars + 16;              // cluster exchanges: 8 arrivals each
  uint64_t* x2 = bars + 17;
  uint64_t* x3 = bars + 18;
  uint64_t* s_full = bars + 24;          // [kMaxTiles], one phase per segment
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24 + kMaxTiles);
  float* red = reinterpret_cast<float*>(smem + Smem::red);
  float* xpart = reinterpret_cast<float*>(smem + Smem::xch);          // [G][2] (max, sum 2^z)
  float* xcand = xpart + 2 * kG;                                      // [budget][2] (key, id bits)
  __shared__ int sel_s[96];
  __shared__ int64_t len_s[kMaxSeq];
  __shared__ int s_cnt;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  uint32_t np_u;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(np_u));
  const int P = (int)np_u;
  const int ncl = gridDim.x / P;
  const int cid = blockIdx.x / P;
  const int nseg = p.n_seq * p.hkv;
  const TableView tv = table_view(p.table, p.n_seq);
  if (threadIdx.x == 0) {
    trace(p.trace, 0);
    if (p.trace && blockIdx.x < kTraceCtas)
      g_trace[(((p.trace - 1) % kTraceRing) * kTraceCtas + blockIdx.x) * kTracePts + 15] = clock64();
    for (int i = 0; i < kStages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(appended, 32);
    mbar_init(z_free, 128);
    mbar_init(s2_full, 1);
    mbar_init(s2_empty, 4);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    mbar_init(sel_ready, 1);
    mbar_init(x1, P);
    mbar_init(x2, P);
    mbar_init(x3, P);
    for (int t = 0; t < kMaxTiles; ++t) mbar_init(s_full + t, 1);
    fence_barrier_init();
    tma_prefetch(&tm_q);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                    // barrier inits visible to the cluster before any remote arrival
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch.  No input of this step (q, k_new, v_new)
  // is read before pdl_wait().  With p.early the lengths and the first means
  // tiles below the dirty window are read before it: this layer's table is not
  // written by the previous kernel, and every kernel before that one has
  // completed (each decode step triggers its dependents only after its own
  // pdl_wait).
  if (!p.early) {
    pdl_wait();
    pdl_launch_dependents();
  }
  for (int s = threadIdx.x; s < p.n_seq; s += blockDim.x) len_s[s] = tv.len[s];
  __syncthreads();
  if (threadIdx.x == 160) {
    // the last CTA to read the lengths advances them (the grid is co-resident
    // and every CTA reads them once, above): no serial work at kernel exit
    int* started = tv.fused + 4 * nseg;
    if (publish_arrive(started) == (int)gridDim.x - 1) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      *started = 0;
      for (int s = 0; s < p.n_seq; ++s) tv.len[s] = len_s[s] + 1;
    }
  }
  if (p.early && warp != 0 && warp != 6) {
    pdl_wait();
    pdl_launch_dependents();
  }

  if (warp == 0) {
    // ============================================================ producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      int pre = 0;                                     // stage-1 tiles of the first segment issued before pdl_wait
      if (p.early) {
        if (cid < nseg) {
          Info I;
          seg_info(p, len_s, cid, rank, P, I);
          const CUtensorMap* mhi = tv.maps + (int64_t)kMaps * I.s + 2;
          const CUtensorMap* mlo = tv.maps + (int64_t)kMaps * I.s + 3;
          tma_prefetch(mhi);
          tma_prefetch(mlo);
          for (int t = 0; t < I.ntiles && t < kStages && t != I.dirty_tile; ++t, ++pre) {
            mbar_wait(empty + stage, phase ^ 1);
            mbar_arrive_expect_tx(full + stage, C::kMuBytes);
            uint8_t* dst = smem + Smem::ring + stage * kStageBytes;
            const int row = (int)(I.r0 + 128 * t);
#pragma unroll
            for (int hh = 0; hh < kDH; ++hh) {
              tma_load_3d(dst + hh * kHalf, mhi, full + stage, 64 * hh, row, I.g);
              tma_load_3d(dst + (kDH + hh) * kHalf, mlo, full + stage, 64 * hh, row, I.g);
            }
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
        pdl_wait();
        pdl_launch_dependents();
      }
      void* next_table = p.prefetch ? *tv.next : nullptr;
      for (int sg = cid; sg < nseg; sg += ncl, ++it) {
        Info I;
        seg_info(p, len_s, sg, rank, P, I);
        const uint32_t par = it & 1;
        const CUtensorMap* mhi = tv.maps + (int64_t)kMaps * I.s + 2;
        const CUtensorMap* mlo = tv.maps + (int64_t)kMaps * I.s + 3;
        const CUtensorMap* mk = tv.maps + (int64_t)kMaps * I.s + 0;
        const CUtensorMap* mv = tv.maps + (int64_t)kMaps * I.s + 1;
        tma_prefetch(mhi);
        tma_prefetch(mlo);
        tma_prefetch(mk);
        tma_prefetch(mv);
        mbar_wait(q_empty, par ^ 1);
        mbar_arrive_expect_tx(q_full, kQB);
        uint8_t* qd = smem + Smem::q;
#pragma unroll
        for (int hh = 0; hh < kDH; ++hh) tma_load_3d(qd + hh * C::kQHalf, &tm_q, q_full, 64 * hh, I.g * kG, I.s);
        for (int t = it == 0 ? pre : 0; t < I.ntiles; ++t) {
          if (t == I.dirty_tile) mbar_wait(appended, par);   // this CTA's window re-sync is in global memory
          mbar_wait(empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, C::kMuBytes);
          uint8_t* dst = smem + Smem::ring + stage * kStageBytes;
          const int row = (int)(I.r0 + 128 * t);
#pragma unroll
          for (int hh = 0; hh < kDH; ++hh) {
            tma_load_3d(dst + hh * kHalf, mhi, full + stage, 64 * hh, row, I.g);
            tma_load_3d(dst + (kDH + hh) * kHalf, mlo, full + stage, 64 * hh, row, I.g);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (it == 0) trace(p.trace, 1);
        if (next_table != nullptr) {
          // this CTA's stream is issued: pull the SAME piece of the next
          // layer's means (hi + lo rows [r0, r1) of this segment) into L2 while
          // this layer's dependent tail keeps HBM otherwise idle
          const TableView tn = table_view(next_table, p.n_seq);
          Info In;
          seg_info(p, tn.len, sg, rank, P, In);
          const SeqDesc dn = tn.desc[In.s];
          const int64_t off = ((int64_t)In.g * dn.means_cap + In.r0) * kD;
          const int64_t bytes = (In.r1 - In.r0) * kD * 2;
          for (int64_t b = 0; b < bytes; b += 32768) {
            const uint32_t nb = (uint32_t)(bytes - b < 32768 ? bytes - b : 32768);
            l2_prefetch_bulk(reinterpret_cast<const uint8_t*>(dn.hi + off) + b, nb);
            l2_prefetch_bulk(reinterpret_cast<const uint8_t*>(dn.lo + off) + b, nb);
          }
        }
        for (int t = 0; t < I.t2; ++t) {
          if (tile_owner(I, t) != (int)rank) continue;
          // the K/V row of this step (piece 7) is published with the stage-1 exchange
          if (t < I.tf) mbar_wait_cluster(x1, par);
          else mbar_wait(sel_ready, par);
          fence_proxy_async_global();
          if (it == 0) trace(p.trace, 7);
          const int nt = tile_blocks(I, t);
          const int b0 = tile_block(I, sel_s, t, 0), b1 = tile_block(I, sel_s, t, 1);
          mbar_wait(empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, nt * 2 * kDH * (kM * 128));
          uint8_t* kd = smem + Smem::ring + stage * kStageBytes;
          uint8_t* vd = kd + 2 * kHalf;
          for (int x = 0; x < nt; ++x) {
            const int row0 = (x ? b1 : b0) * kM;
            const uint32_t off = x * kM * 128;
#pragma unroll
            for (int hh = 0; hh < kDH; ++hh) {
              tma_load_3d(kd + hh * kHalf + off, mk, full + stage, 64 * hh, row0, I.g);
              tma_load_3d(vd + hh * kHalf + off, mv, full + stage, 64 * hh, row0, I.g);
            }
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    } else if (p.early) {
      pdl_wait();
      pdl_launch_dependents();
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================================================ MMA issuer
    const uint32_t idesc = idesc_bf16_f32(128, kG);
    const uint32_t idesc_pv = idesc_bf16_f32_major(128, kG, 1, 1);
    const uint32_t q_addr = smem_u32(smem + Smem::q);
    int stage = 0;
    uint32_t phase = 0;
    int i2 = 0;
    int it = 0;
    for (int sg = cid; sg < nseg; sg += ncl, ++it) {
      Info I;
      seg_info(p, len_s, sg, rank, P, I);
      const uint32_t par = it & 1;
      mbar_wait(q_full, par);
      if (it > 0) mbar_wait(z_free, par ^ 1);      // previous segment's z tiles have been read
      for (int t = 0; t < I.ntiles; ++t) {
        mbar_wait(full + stage, phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t mu_s = smem_u32(smem + Smem::ring + stage * kStageBytes);
          for (int part = 0; part < 2; ++part)
            for (int k = 0; k < kD / 16; ++k) {
              const uint32_t koff = (k & 3) * 32;
              umma_f16_ss(tmem + t * kG, sdesc_k_sw128(mu_s + part * kDH * kHalf + (k >> 2) * kHalf + koff),
                          sdesc_k_sw128(q_addr + (k >> 2) * C::kQHalf + koff), idesc, (part | k) ? 1u : 0u);
            }
          umma_commit(empty + stage);
          umma_commit(s_full + t);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      int ti = 0;                                      // this piece's tile index within the segment
      for (int t = 0; t < I.t2; ++t) {
        if (tile_owner(I, t) != (int)rank) continue;
        const int nt = tile_blocks(I, t);
        const uint32_t tp = i2 & 1;                    // per-tile barrier parity (running count)
        ++i2;
        mbar_wait(full + stage, phase);
        mbar_wait(s2_empty, tp ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + Smem::ring + stage * kStageBytes);
        if (elect_one()) {
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
            const uint32_t qoff = (k >> 2) * C::kQHalf + (k & 3) * 32;
            umma_f16_ss(tmem + kColS2, sdesc_k_sw128(k_addr + off), sdesc_k_sw128(q_addr + qoff), idesc,
                        k > 0 ? 1u : 0u);
          }
          umma_commit(s2_full);
        }
        __syncwarp();
        mbar_wait(p_full, tp);
        if (ti == 0) mbar_wait(o_empty, par ^ 1);    // the previous segment's O has been read
        tc_fence_after();
        if (elect_one()) {
          const uint32_t v_addr = k_addr + 2 * kHalf;
          const uint32_t p_addr = smem_u32(smem + Smem::p);
          const int ksteps = nt == 2 ? 8 : 4;
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t vdesc = sdesc_mn_sw128(v_addr + k * 2048, kHalf, 1024);
            umma_f16_ss(tmem + kColO, vdesc, sdesc_interleave(p_addr + k * 32 * kG, 16 * kG, 128), idesc_pv,
                        (ti > 0 || k > 0) ? 1u : 0u);
            umma_f16_ss(tmem + kColO, vdesc, sdesc_interleave(p_addr + kPHalf + k * 32 * kG, 16 * kG, 128),
                        idesc_pv, 1u);
          }
          umma_commit(empty + stage);
          umma_commit(o_full);                         // after every PV: P buffer free, O stable
        }
        __syncwarp();
        ++ti;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(q_empty);          // every MMA reading this segment's Q is issued
      __syncwarp();
    }
  } else if (warp == 6) {
    // ============================================================ append (32 threads)
    // The kernel windows that contain the new row (at most two fine windows in
    // this piece's row range, nk - dlo <= 2) are recomputed bitwise as
    // build_kernels (sparse.py:70-91, 116-127, F18 clip) by every piece whose
    // range holds them; piece P-1 also writes the K/V row and the dirty coarse
    // windows.  A warp of its own: the epilogue starts reducing z tiles at
    // once instead of waiting out this work's load round trip (the producer
    // holds only the dirty tile's TMA until `appended`).  Lane = 4 dims, 8-byte
    // loads: the <= 48 rows of a window pair are one round of loads.
    const int d0 = lane * 4;
    const bool dact = d0 < kD;                       // D = 64: lanes 0..15 carry the dims
    int it = 0;
    for (int sg = cid; sg < nseg; sg += ncl, ++it) {
      Info I;
      seg_info(p, len_s, sg, rank, P, I);
      const SeqDesc ds = tv.desc[I.s];
      const int64_t L = I.pos + 1;
      const __nv_bfloat16* kg = ds.k + (int64_t)I.g * ds.cap * kD;
      const int64_t knew_idx = ((int64_t)I.s * p.hkv + I.g) * kD + d0;
      const int64_t jlo = I.dlo > I.r0 ? I.dlo : I.r0;
      const bool dirty = jlo < I.r1 && dact;
      // the raw bf16 quads stay packed until summed (96 registers, not 192)
      uint2 raw[kP + kS];
      if (dirty) {
        const int64_t row0 = jlo * kS;
#pragma unroll
        for (int i = 0; i < kP + kS; ++i) {
          const int64_t r = row0 + i;
          raw[i] = (r < L && r != I.pos) ? __ldg(reinterpret_cast<const uint2*>(kg + r * kD + d0)) : make_uint2(0u, 0u);
        }
      }
      if (it == 0 && p.early) {                      // k_new / v_new: this step's inputs
        pdl_wait();
        pdl_launch_dependents();
      }
      const uint2 kraw = dact ? *reinterpret_cast<const uint2*>(p.k_new + knew_idx) : make_uint2(0u, 0u);
      float knew[4];
      {
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&kraw.x);
        const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&kraw.y);
        knew[0] = __low2float(a);
        knew[1] = __high2float(a);
        knew[2] = __low2float(b);
        knew[3] = __high2float(b);
      }
      if (dirty) {
        const int64_t row0 = jlo * kS;
#pragma unroll
        for (int i = 0; i < kP + kS; ++i)
          if (row0 + i == I.pos) raw[i] = kraw;
        auto val = [&](int i, int e) {
          const uint32_t w = e < 2 ? raw[i].x : raw[i].y;
          return __uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16));
        };
        auto emit = [&](int64_t j, int i0) {
          const int64_t w64 = L - j * kS;
          const int w = (int)(w64 < kP ? w64 : kP);
          float mu[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            double acc = (double)val(i0, e);
#pragma unroll
            for (int r = 1; r < kP; ++r)
              if (r < w) acc += (double)val(i0 + r, e);   // sequential, as numpy's reduce
            mu[e] = __double2float_rn(acc / (double)w);
          }
          const int64_t dst = ((int64_t)I.g * ds.means_cap + j) * kD + d0;
          *reinterpret_cast<float4*>(ds.fine + dst) = make_float4(mu[0], mu[1], mu[2], mu[3]);
          __nv_bfloat16 h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            h[e] = __float2bfloat16_rn(mu[e]);
            l[e] = __float2bfloat16_rn(mu[e] - __bfloat162float(h[e]));
          }
          *reinterpret_cast<uint2*>(ds.hi + dst) = *reinterpret_cast<const uint2*>(h);
          *reinterpret_cast<uint2*>(ds.lo + dst) = *reinterpret_cast<const uint2*>(l);
        };
        emit(jlo, 0);
        if (jlo + 1 < I.r1) emit(jlo + 1, kS);
      }
      if ((int)rank == P - 1 && dact) {               // the new K/V row (read by the forced tiles after x1)
        const int64_t dst = ((int64_t)I.g * ds.cap + I.pos) * kD + d0;
        *reinterpret_cast<uint2*>(ds.k + dst) = kraw;
        *reinterpret_cast<uint2*>(ds.v + dst) = *reinterpret_cast<const uint2*>(p.v_new + knew_idx);
      }
      fence_proxy_async_global();
      mbar_arrive(appended);
      if (lane == 0 && it == 0) trace(p.trace, 13);
      if ((int)rank == P - 1 && dact) {
        // every dirty coarse window (two when coarse_stride < kernel_size): not
        // read by this step's stages
        const int cs = p.coarse_stride;
        int64_t first = I.pos < kP ? 0 : (I.pos - kP) / cs + 1;
        const int64_t count_old = I.pos / cs, count = L / cs;
        if (first > count_old) first = count_old;
        for (int64_t j = first; j < count; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float mu = window_mean(kg, kD, j, cs, L, d0 + e, I.pos, knew[e]);
            ds.coarse[((int64_t)I.g * ds.coarse_cap + j) * kD + d0 + e] = mu;
          }
      }
    }
  } else {
    // ============================================================ epilogue (128 threads)
    const int tid = threadIdx.x - 64;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;                // TMEM lane
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    float* red_m = red;
    float* red_s = red + 4 * kG;
    float* lse2 = red + 8 * kG;
    float* sarr = reinterpret_cast<float*>(smem + Smem::sarr);
    float* rarr = reinterpret_cast<float*>(smem + Smem::rarr);
    int i2 = 0;
    int it = 0;
    uint32_t sfpar = 0;                              // bit t: parity of the next s_full[t] phase
    for (int sg = cid; sg < nseg; sg += ncl, ++it) {
      Info I;
      seg_info(p, len_s, sg, rank, P, I);
      const uint32_t par = it & 1;
      const int tr = it == 0 ? p.trace : 0;
      const SeqDesc ds = tv.desc[I.s];
      const int64_t L = I.pos + 1;
      // ---- B. stage-1 partial (max, sum 2^z) over owned kernels [4*b0, r1)
      const int64_t own0 = 4 * I.b0;
      {
        float m[kG], sm[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) { m[h] = -INFINITY; sm[h] = 0.f; }
        for (int t = 0; t < I.ntiles; ++t) {
          mbar_wait(s_full + t, (sfpar >> t) & 1u);
          sfpar ^= 1u << t;
          tc_fence_after();
          float v[kG];
          tmem_ld_n<kG>(tmem + lane_base + t * kG, v);
          tmem_wait_ld();
          if (t == 0 && tid == 0) trace(tr, 12);
          const int64_t j = I.r0 + 128 * t + row;
          if (j >= own0 && j < I.r1) {
#pragma unroll
            for (int h = 0; h < kG; ++h) {
              const float z = v[h] * p.zscale;
              if (z > m[h]) {
                sm[h] = sm[h] * ex2(m[h] - z) + 1.f;
                m[h] = z;
              } else {
                sm[h] += ex2(z - m[h]);
              }
            }
          }
        }
        warp_reduce_lse_n<kG>(m, sm, lane);
        if (reduce_writer_n<kG>(lane)) {
          const int h = reduce_head_n<kG>(lane);
          red_m[h * 4 + quad] = m[0];
          red_s[h * 4 + quad] = sm[0];
        }
      }
      named_bar_sync(1, 128);
      if (tid < kG) {
        float M = -INFINITY;
        for (int x = 0; x < 4; ++x) M = fmaxf(M, red_m[tid * 4 + x]);
        float S = 0.f;
        for (int x = 0; x < 4; ++x) {
          const float mm = red_m[tid * 4 + x];
          if (mm != -INFINITY) S += red_s[tid * 4 + x] * ex2(mm - M);
        }
        xpart[2 * tid] = M;
        xpart[2 * tid + 1] = S;
      }
      named_bar_sync(1, 128);
      if (tid == 0) trace(tr, 2);
      mbar_wait(appended, par);                      // the append warp's stores precede this CTA's x1 arrival
      if (warp == 2) arrive_all(x1, lane, P);
      mbar_wait_cluster(x1, par);
      if (tid == 0) trace(tr, 3);
      CYC(0);
      // ---- C. LSE (all pieces' partials over DSMEM), group scores, block scores, local top-k
      {
        const int h = tid >> 3, r = tid & 7;           // G heads x 8 pieces (threads >= 8G idle)
        float M = -INFINITY, S = 0.f;
        if (r < P && h < kG) {
          const float2 ms = ld_dsmem2(xpart + 2 * h, r);
          M = ms.x;
          S = ms.y;
        }
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {
          const float om = __shfl_xor_sync(0xffffffffu, M, off);
          const float os = __shfl_xor_sync(0xffffffffu, S, off);
          const float nm = fmaxf(M, om);
          S = (M == -INFINITY ? 0.f : S * ex2(M - nm)) + (om == -INFINITY ? 0.f : os * ex2(om - nm));
          M = nm;
        }
        if (r == 0 && h < kG) lse2[h] = M == -INFINITY ? INFINITY : M + log2f(S);
      }
      named_bar_sync(1, 128);
      CYC(1);
      {
        float l2[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) l2[h] = lse2[h];
        tc_fence_after();
        // two TMEM tiles per wait: the load latency is paid once per pair
        for (int t = 0; t < I.ntiles; t += 2) {
          float v[kG], w[kG];
          tmem_ld_n<kG>(tmem + lane_base + t * kG, v);
          if (t + 1 < I.ntiles) tmem_ld_n<kG>(tmem + lane_base + (t + 1) * kG, w);
          tmem_wait_ld();
          const int64_t jl = 128 * t + row;
          if (I.r0 + jl < I.r1) {
            float a = 0.f;
#pragma unroll
            for (int h = 0; h < kG; ++h) a += ex2(v[h] * p.zscale - l2[h]);
            sarr[jl] = a * (1.0f / kG);
          }
          if (t + 1 < I.ntiles && I.r0 + jl + 128 < I.r1) {
            float a = 0.f;
#pragma unroll
            for (int h = 0; h < kG; ++h) a += ex2(w[h] * p.zscale - l2[h]);
            sarr[jl + 128] = a * (1.0f / kG);
          }
        }
        CYC(2);
        tc_fence_before();
        mbar_arrive(z_free);
      }
      named_bar_sync(1, 128);
      // R_b = max S_j over block b's kernels [lo, hi) (kernel_range_for_block,
      // sparse.py:191-215: lo = 4b - 1 for b >= 1, hi clipped to the row and nk):
      // <= 5 kernels, loaded together, in 32-bit offsets from r0
      for (int64_t b = I.b0 + tid; b < I.b1; b += 128) {
        int64_t end = (b + 1) * kM;
        if (end > L) end = L;
        int64_t hi64 = (end + kS - 1) / kS;
        if (hi64 > I.nk) hi64 = I.nk;
        const int lo = (int)((b == 0 ? 0 : 4 * b - 1) - I.r0);
        const int hi = (int)(hi64 - I.r0);
        float r = 0.f;
        if (hi > lo) {
          float x[kP / kS + 3];
#pragma unroll
          for (int k = 0; k < kP / kS + 3; ++k) x[k] = sarr[lo + k < kMaxRows ? lo + k : lo];
          r = x[0];
#pragma unroll
          for (int k = 1; k < kP / kS + 3; ++k) r = (lo + k < hi) ? fmaxf(r, x[k]) : r;
        }
        rarr[b - I.b0] = r;
      }
      named_bar_sync(1, 128);
      if (tid == 0) trace(tr, 4);
      CYC(3);
      const bool dense = I.budget >= I.n_free || I.budget == 0;
      if (!dense) {
        int lo = (int)((I.b0 > I.n_init ? I.b0 : I.n_init) - I.b0);
        int hi = (int)((I.b1 < I.local_lo ? I.b1 : I.local_lo) - I.b0);
        if (hi < lo) hi = lo;
        float* scratch = reinterpret_cast<float*>(smem + Smem::p);
        if (!cta_topk(rarr, I.b0, lo, hi, I.budget, tid, lane, warp - 2, scratch, &s_cnt, xcand) && warp == 2) {
          float* lkey = scratch;
          int* lid = reinterpret_cast<int*>(lkey + topk::kListCap);
          local_topk(rarr, I.b0, lo, hi, I.budget, lane, lkey, lid, xcand);   // massive ties: exact fallback
        }
      }
      named_bar_sync(1, 128);
      if (tid == 0) {
        trace(tr, 5);
        CYC(4);
      }
      // ---- D (part 1). stage-2 state of this piece: all its tiles accumulate
      // into one O^T in TMEM with a running per-head max (rescaled only when a
      // tile's max exceeds it by more than 2^8), per-thread row sums
      float m_run[kG], lrow[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h) { m_run[h] = -INFINITY; lrow[h] = 0.f; }
      int ti = 0;
      uint32_t tp_prev = 0;
      auto stage2_tile = [&](int t) {
        const uint32_t tp = i2 & 1;
        ++i2;
        const int bx = tile_block(I, sel_s, t, row >> 6);
        mbar_wait(s2_full, tp);
        tc_fence_after();
        float z[kG];
        tmem_ld_n<kG>(tmem + lane_base + kColS2, z);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s2_empty);
        const bool valid = bx >= 0 && (int64_t)bx * kM + (row & 63) <= I.pos;
#pragma unroll
        for (int h = 0; h < kG; ++h) z[h] = valid ? z[h] * p.zscale : -INFINITY;
        {
          float zz[kG];
#pragma unroll
          for (int h = 0; h < kG; ++h) zz[h] = z[h];
          const float v = warp_reduce_n<kG>(zz, lane, [](float a, float b) { return fmaxf(a, b); });
          if (reduce_writer_n<kG>(lane)) red_m[quad * kG + reduce_head_n<kG>(lane)] = v;
        }
        named_bar_sync(1, 128);
        float mnew[kG];
        bool need = ti == 0;
#pragma unroll
        for (int h = 0; h < kG; ++h) {
          const float tm = fmaxf(fmaxf(red_m[h], red_m[kG + h]), fmaxf(red_m[2 * kG + h], red_m[3 * kG + h]));
          mnew[h] = fmaxf(m_run[h], tm);
          need |= tm > m_run[h] + 8.f;
        }
        named_bar_sync(1, 128);                        // red_m reads done
        if (ti > 0) {
          mbar_wait(o_full, tp_prev);                  // PV of the previous tile: P buffer free, O stable
          tc_fence_after();
        }
        if (need) {
          float corr[kG];
          bool any = false;
#pragma unroll
          for (int h = 0; h < kG; ++h) {
            corr[h] = m_run[h] == -INFINITY ? 0.f : ex2(m_run[h] - mnew[h]);
            any |= ti > 0 && corr[h] != 1.f;
            lrow[h] *= corr[h];
            m_run[h] = mnew[h];
          }
          if (any) {
            float o[kG];
            tmem_ld_n<kG>(tmem + lane_base + kColO, o);
            tmem_wait_ld();
#pragma unroll
            for (int h = 0; h < kG; ++h) o[h] *= corr[h];
            tmem_st_n<kG>(tmem + lane_base + kColO, o);
            tmem_wait_st();
            tc_fence_before();
          }
        }
        uint32_t phi[kG / 2], plo[kG / 2];
#pragma unroll
        for (int h = 0; h < kG; h += 2) {
          const float a = ex2(z[h] - m_run[h]);
          const float b = ex2(z[h + 1] - m_run[h + 1]);
          lrow[h] += a;
          lrow[h + 1] += b;
          const __nv_bfloat162 hi2 = __floats2bfloat162_rn(a, b);
          const __nv_bfloat162 lo2 = __floats2bfloat162_rn(a - __low2float(hi2), b - __high2float(hi2));
          phi[h / 2] = *reinterpret_cast<const uint32_t*>(&hi2);
          plo[h / 2] = *reinterpret_cast<const uint32_t*>(&lo2);
        }
        uint8_t* pb = smem + Smem::p;
        // P^T [128 rows][G heads]: 8-row x 8-head core matrices, heads 8..15 at +128
        const uint32_t base = (row >> 3) * (16 * kG) + (row & 7) * 16;
#pragma unroll
        for (int c = 0; c < kG / 8; ++c) {
          *reinterpret_cast<uint4*>(pb + base + 128 * c) =
              make_uint4(phi[4 * c], phi[4 * c + 1], phi[4 * c + 2], phi[4 * c + 3]);
          *reinterpret_cast<uint4*>(pb + kPHalf + base + 128 * c) =
              make_uint4(plo[4 * c], plo[4 * c + 1], plo[4 * c + 2], plo[4 * c + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        tp_prev = tp;
        ++ti;
      };
      // forced-only tiles do not depend on the selection: run them while the
      // candidate exchange is in flight
      if (warp == 2) arrive_all(x2, lane, P);
      for (int t = 0; t < I.tf; ++t)
        if (tile_owner(I, t) == (int)rank) stage2_tile(t);
      mbar_wait_cluster(x2, par);
      CYC(5);
      {
        // ---- merge (every piece): the global top-B lies in the union of the local lists
        float* lk = sarr;                                         // [n][2] (key, id bits)
        // the P buffer doubles as the chosen-id list: the forced tiles' PV must be done with it
        if (ti > 0) mbar_wait(o_full, tp_prev);
        int* chosen = reinterpret_cast<int*>(smem + Smem::p);
        const int n = dense ? 0 : P * I.budget;
        for (int x = tid; x < n; x += 128) {
          const float2 kv = ld_dsmem2(xcand + 2 * (x % I.budget), x / I.budget);
          lk[2 * x] = kv.x;
          lk[2 * x + 1] = kv.y;
        }
        if (tid == 0) s_cnt = 0;
        named_bar_sync(1, 128);
        CYC(6);
        // a full local list's worst key tau_i is <= the global B-th best (that
        // list alone has B keys >= tau_i): keys < max_i tau_i cannot be chosen
        float tau = -INFINITY;
        if (tid < (dense ? 0 : P)) {
          float mn = INFINITY;
          bool full_list = true;
          for (int k = 0; k < I.budget; ++k) {
            full_list &= __float_as_int(lk[2 * (tid * I.budget + k) + 1]) >= 0;
            mn = fminf(mn, lk[2 * (tid * I.budget + k)]);
          }
          if (full_list) tau = mn;
        }
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) tau = fmaxf(tau, __shfl_xor_sync(0xffffffffu, tau, off));
        if (tid == 0) red_m[0] = tau;
        named_bar_sync(1, 128);
        tau = red_m[0];
        CYC(7);
        float* fl = rarr;                                          // filtered (key, id) pairs
        for (int x = tid; x < n; x += 128) {
          const float k = lk[2 * x];
          const int id = __float_as_int(lk[2 * x + 1]);
          if (id >= 0 && k >= tau) {
            const int slot = atomicAdd(&s_cnt, 1);
            fl[2 * slot] = k;
            fl[2 * slot + 1] = lk[2 * x + 1];
          }
        }
        named_bar_sync(1, 128);
        const int m = s_cnt;
        CYC(8);
        for (int x = tid; x < m; x += 128) {
          const float rk = fl[2 * x];
          const int bk = __float_as_int(fl[2 * x + 1]);
          int rnk = 0;
#pragma unroll 8
          for (int y = 0; y < m; ++y) rnk += topk::better(fl[2 * y], __float_as_int(fl[2 * y + 1]), rk, bk) ? 1 : 0;
          if (rnk < I.budget) chosen[rnk] = bk;          // ranks are distinct: exactly budget writers
        }
        named_bar_sync(1, 128);
        CYC(9);
        if (!dense && warp == 2) {
          // chosen ids ascending (select_topk returns sorted ids, sparse.py:277)
          const int id = lane < I.budget ? chosen[lane] : INT_MAX;
          const int srt = topk::warp_sort_asc(id, lane);
          if (lane < I.budget) sel_s[I.n_init + lane] = srt;
        }
        for (int x = tid; x < p.max_sel; x += 128) {
          int id = -2;
          // every candidate only when the budget covers them all; budget 0 with
          // free blocks left (forced_consume_budget) selects the forced blocks
          if (I.budget >= I.n_free) id = x < I.n_cand ? x : -1;
          else if (x < I.n_init) id = x;
          else if (x >= I.n_init + I.n_ch && x < I.n_sel) id = I.local_lo + (x - I.n_init - I.n_ch);
          else if (x >= I.n_sel) id = -1;
          if (id != -2) sel_s[x] = id;
        }
        named_bar_sync(1, 128);
        if (tid == 0) {
          mbar_arrive(sel_ready);
          trace(tr, 6);
        }
        CYC(10);
        if (rank == 0) {
          int32_t* sel_row = p.selection + (int64_t)sg * p.max_sel;
          for (int x = tid; x < p.max_sel; x += 128) sel_row[x] = sel_s[x];
        }
      }
      // ---- D (part 2). chosen tiles, then this piece's partial -> shared memory
      for (int t = I.tf; t < I.t2; ++t)
        if (tile_owner(I, t) == (int)rank) stage2_tile(t);
      if (tid == 0 && it == 0) trace(tr, 8);
      CYC(14);
      {
        float* pt = sarr;                                  // [16][128] O^T, [16][2] (max, sum)
        if (ti > 0) {
          mbar_wait(o_full, tp_prev);
          tc_fence_after();
          float o[kG];
          tmem_ld_n<kG>(tmem + lane_base + kColO, o);
          tmem_wait_ld();
          tc_fence_before();
          if (row < kD) {
#pragma unroll
            for (int h = 0; h < kG; ++h) pt[h * kD + row] = o[h];   // O^T lane == d
          }
          const float v = warp_reduce_n<kG>(lrow, lane, [](float a, float b) { return a + b; });
          if (reduce_writer_n<kG>(lane)) red_s[quad * kG + reduce_head_n<kG>(lane)] = v;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty);               // once per segment, with or without tiles
        named_bar_sync(1, 128);
        if (tid < kG) {
          pt[kG * kD + 2 * tid] = ti > 0 ? m_run[tid] : -INFINITY;
          pt[kG * kD + 2 * tid + 1] =
              ti > 0 ? red_s[tid] + red_s[kG + tid] + red_s[2 * kG + tid] + red_s[3 * kG + tid] : 0.f;
        }
        named_bar_sync(1, 128);
      }
      if (warp == 2) arrive_all(x3, lane, P);
      mbar_wait_cluster(x3, par);
      if (tid == 0) trace(tr, 14);
      CYC(15);
      {
        // ---- combine: piece r merges heads r, r + P, ... of the P partials (DSMEM);
        // a head is D/2 threads (float2 each), 256/D heads per pass
        constexpr int kHPass = 256 / kD;
        const int hh = tid / (kD / 2), dp = tid % (kD / 2);
        for (int j2 = 0; (int)rank + P * kHPass * j2 < kG; ++j2) {
          const int h = (int)rank + P * (kHPass * j2 + hh);
          const bool act = h < kG;
          const int hs = act ? h : (int)rank;
          float mq[kMaxCl], lq[kMaxCl];
          float2 oq[kMaxCl];
#pragma unroll
          for (int q = 0; q < kMaxCl; ++q) {
            if (q < P) {
              mq[q] = ld_dsmem(sarr + kG * kD + 2 * hs, q);
              lq[q] = ld_dsmem(sarr + kG * kD + 2 * hs + 1, q);
              oq[q] = ld_dsmem2(sarr + hs * kD + 2 * dp, q);
            }
          }
          float M = -INFINITY;
#pragma unroll
          for (int q = 0; q < kMaxCl; ++q)
            if (q < P) M = fmaxf(M, mq[q]);
          CYC(16);
          float Ls = 0.f, ax = 0.f, ay = 0.f;
#pragma unroll
          for (int q = 0; q < kMaxCl; ++q) {
            if (q < P && mq[q] != -INFINITY) {
              const float w = ex2(mq[q] - M);
              Ls += lq[q] * w;
              ax += oq[q].x * w;
              ay += oq[q].y * w;
            }
          }
          if (act) {
            const float il = 1.f / Ls;
            const int64_t oi = ((int64_t)I.s * p.hq + I.g * kG + h) * kD + 2 * dp;
            if (p.out_f32) {
              *reinterpret_cast<float2*>(static_cast<float*>(p.out) + oi) = make_float2(ax * il, ay * il);
            } else {
              *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(p.out) + oi) =
                  __floats2bfloat162_rn(ax * il, ay * il);
            }
            if (p.lse && dp == 0) p.lse[(int64_t)I.s * p.hq + I.g * kG + h] = (M + log2f(Ls)) * 0.6931471805599453f;
          }
        }
      }
      if (tid == 0) trace(tr, 9);
      CYC(17);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                     // no CTA leaves while its shared memory may still be read
  if (warp == 1) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {
    trace(p.trace, 10);
    if (p.trace && blockIdx.x < kTraceCtas)
      g_trace[(((p.trace - 1) % kTraceRing) * kTraceCtas + blockIdx.x) * kTracePts + 11] = clock64();
  }
}

}  // namespace

size_t decode_fused_workspace_bytes(int n_seq, int hkv) {
  (void)n_seq;
  (void)hkv;
  return 0;
}

template <int G, int D>
static int max_active_clusters(int np) {
  constexpr int kMaxDev = 64;
  static int cached[kMaxDev][kMaxCl + 1];
  static bool init = false;
  if (!init) {
    for (auto& row : cached)
      for (int& c : row) c = -1;
    init = true;
  }
  const int dev = current_device() % kMaxDev;   // occupancy is per device
  if (cached[dev][np] >= 0) return cached[dev][np];
  const size_t smem = FCfg<G, D>::Smem::total + 1024;
  if (smem_attr_once((const void*)decode_cluster_kernel<G, D>, (int)smem) != cudaSuccess) return cached[dev][np] = 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = np;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(np * 32);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, decode_cluster_kernel<G, D>, &cfg) != cudaSuccess) n = 0;
  return cached[dev][np] = n;
}

// Cluster size (= pieces per segment): the largest per-round parallelism
// np / rounds over the sizes whose pieces fit the TMEM-resident z tiles.  On a
// B200 (1 CTA/SM) 8-CTA clusters reach 15 co-resident clusters, 6-CTA ones 22.
// `share` launches of this kernel run concurrently (decode micro-batches on
// separate streams): each may use 1/share of the co-resident clusters.
template <int G, int D>
static int choose_cluster(int nseg, int64_t max_len_after, int share) {
  const int64_t nb_max = max_len_after / kM + 1;
  static const int forced = getenv("INFLLM2_DECODE_P") ? atoi(getenv("INFLLM2_DECODE_P")) : 0;   // diagnostic
  if (forced >= 3 && forced <= kMaxCl && (nb_max + forced - 1) / forced + 1 <= kMaxPieceBlocks &&
      max_active_clusters<G, D>(forced) / share > 0)
    return forced;
  int best = 0;
  double best_score = -1.0;
  for (int np = kMaxCl; np >= 3; --np) {
    if ((nb_max + np - 1) / np + 1 > kMaxPieceBlocks) continue;
    const int n = max_active_clusters<G, D>(np) / share;
    if (n <= 0) continue;
    const int rounds = (nseg + n - 1) / n;
    const double score = (double)np / rounds;
    if (score > best_score) {
      best_score = score;
      best = np;
    }
  }
  return best;
}

static int choose_cluster_geom(int hq, int hkv, int d, int nseg, int64_t max_len_after, int share) {
  if (hq == 16 * hkv && d == 128) return choose_cluster<16, 128>(nseg, max_len_after, share);
  if (hq == 8 * hkv && d == 64) return choose_cluster<8, 64>(nseg, max_len_after, share);
  return 0;
}

// Host-side eligibility: pieces must fit the TMEM-resident z tiles for every
// length up to max_len_after and budgets must fit the warp top-k.
bool decode_fused_supported(const infllm2_geometry& g, int n_seq, int hq, int hkv, int d, int64_t max_len_after,
                            int share) {
  if (getenv("INFLLM2_DECODE_LEGACY")) return false;
  if (n_seq > kMaxSeq || n_seq < 1) return false;
  if (g.top_k > kMaxBudget || g.top_k < 1) return false;
  if (infllm2_max_selected(&g) > 96) return false;
  return choose_cluster_geom(hq, hkv, d, n_seq * hkv, max_len_after, share) > 0;
}

template <int G, int D>
static int fused_launch(const Params& p, const void* q, int n_seq, int hq, int hkv, int64_t max_len_after, int share,
                        cudaStream_t stream) {
  CUtensorMap tq;
  const uint64_t dims[3] = {(uint64_t)D, (uint64_t)hq, (uint64_t)n_seq};
  const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)hq * D * 2};
  const uint32_t box[3] = {64, (uint32_t)G, 1};
  if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return INFLLM2_ERR_SHAPE;
  const int nseg = n_seq * hkv;
  const int np = choose_cluster<G, D>(nseg, max_len_after, share);
  if (np <= 0) return INFLLM2_ERR_UNSUPPORTED;
  int ncl = max_active_clusters<G, D>(np) / share;
  if (ncl > nseg) ncl = nseg;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = np;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = getenv("INFLLM2_DECODE_NOPDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * np));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = FCfg<G, D>::Smem::total + 1024;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  count_launch();
  if (cudaLaunchKernelEx(&cfg, decode_cluster_kernel<G, D>, tq, p) != cudaSuccess) return INFLLM2_ERR_CUDA;
  return INFLLM2_OK;
}

int decode_fused_step(const infllm2_geometry& g, void* table, int n_seq, int64_t max_len_after, int hq, int hkv,
                      int d, const void* q, const void* k_new, const void* v_new, int32_t* selection, void* out,
                      int out_f32, float* lse, void* ws, cudaStream_t stream, int share, int early) {
  (void)ws;
  Params p;
  static const bool no_early = getenv("INFLLM2_DECODE_NOEARLY") != nullptr;   // diagnostic
  p.early = early && !no_early;
  p.table = table;
  p.n_seq = n_seq;
  p.hkv = hkv;
  p.hq = hq;
  p.top_k = g.top_k;
  p.n_init = g.n_init_blocks;
  p.n_local = g.n_local_blocks;
  p.consume = g.forced_consume_budget;
  p.max_sel = infllm2_max_selected(&g);
  p.coarse_stride = (int)g.coarse_stride;
  p.k_new = static_cast<const __nv_bfloat16*>(k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(v_new);
  p.selection = selection;
  p.out = out;
  p.out_f32 = out_f32;
  p.lse = lse;
  p.zscale = 1.4426950408889634f / sqrtf((float)d);
  // L2 prefetch of the linked next layer's means: measured neutral to slightly
  // slower (the means stream already runs at ~6.2 TB/s; DESIGN §4 K4), so opt-in
  static const bool pf = getenv("INFLLM2_DECODE_PREFETCH") != nullptr;
  p.prefetch = pf ? 1 : 0;
  static const bool tr = getenv("INFLLM2_DECODE_TRACE") != nullptr;
  static int launches = 0;
  p.trace = tr ? 1 + (launches++ % kTraceRing) : 0;
  if (hq == 16 * hkv && d == 128) return fused_launch<16, 128>(p, q, n_seq, hq, hkv, max_len_after, share, stream);
  if (hq == 8 * hkv && d == 64) return fused_launch<8, 64>(p, q, n_seq, hq, hkv, max_len_after, share, stream);
  return INFLLM2_ERR_UNSUPPORTED;
}

}  // namespace infllm2

// Debug: copy the traced launches' per-CTA phase timestamps (ns,
// [4 launches][160 CTAs][16], ring by launch number) to host memory.
extern "C" int infllm2_debug_decode_cycles(long long* host, int max_entries) {
  const int cap = infllm2::kTraceCtas * 32;
  const int n = max_entries < cap ? max_entries : cap;
  return cudaMemcpyFromSymbol(host, infllm2::g_cyc, sizeof(long long) * n) == cudaSuccess ? 0 : -1;
}

extern "C" int infllm2_debug_decode_trace(unsigned long long* host, int max_entries) {
  const int cap = infllm2::kTraceRing * infllm2::kTraceCtas * infllm2::kTracePts;
  const int n = max_entries < cap ? max_entries : cap;
  return cudaMemcpyFromSymbol(host, infllm2::g_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
