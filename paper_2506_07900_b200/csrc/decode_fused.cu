// Batched single-token decode in ONE launch (BASELINE configs[3]).
//
// The five-launch path (decode.cu) spends most of a 128K layer-step in launch
// ramps and tails: each phase is a few microseconds of HBM traffic behind a
// kernel boundary.  Here one persistent CTA per SM runs the whole step and the
// phases of each (sequence, KV group) "segment" are chained by device-scope
// counters instead of kernel boundaries, so the means stream of stage 1 —
// the HBM-bound part, 8.4 MB per 128K segment — runs back to back on all SMs
// and the dependent tail (LSE merge, block scores, top-k, stage 2) costs a few
// microseconds per segment.
//
// Work split.  Segment sg = (s, g) has n_cand = pos/64 + 1 candidate blocks
// (pos = the new token's position).  Every CTA computes the same partition from
// the device-side lengths: each segment gets 1 + floor(avail * n_cand / total)
// CTAs ("pieces"), capped so the top-k merge list fits shared memory, and each
// piece owns a contiguous block range [b0, b1) of its segment.
//
// Per piece (warp 0 = TMA producer, warp 1 = MMA issuer, warps 2..5 = 128
// epilogue threads):
//   A. append.  Kernel windows containing the new row (the last one or two of
//      the segment) are recomputed, bitwise as build_kernels (sparse.py:70-91,
//      116-127, F18 clip), by every piece whose row range holds them (identical
//      values, so concurrent writers agree); the segment's last piece also
//      writes the K/V row and the dirty coarse window.
//   B. stage-1 scores z = mu . q for the piece's kernels [4*b0 - 1, 4*b1)
//      (one halo kernel on the left, so every block's kernel range
//      [4b-1, 4b+4) is local) on tcgen05: M = 128 kernels, N = 16 heads,
//      bf16 hi + lo means; the z tiles STAY IN TMEM (16 columns per tile).
//      Online per-head (max, sum 2^z) over the owned kernels [4*b0, 4*b1) ->
//      global partial; arrive on the segment's stage-1 counter.
//   C. when all pieces arrived: exact per-head LSE from the partials,
//      S_j = mean_h 2^(z - lse) (sparse.py:163-188) from TMEM, block max R_b
//      (sparse.py:191-215), local top-`budget` by (score desc, id asc)
//      (sparse.py:273) -> global candidates; the last piece to arrive merges
//      the candidate lists (the global top-B is contained in the union of the
//      local top-Bs) and publishes the selection (force_blocks + select_topk,
//      sparse.py:218-277).
//   D. stage 2: the selection's 64-row blocks, forced ones first, are cut into
//      128-row tiles; tile t goes to piece t mod c.  Forced-only tiles do not
//      wait for the selection.  Per tile: S^T = K . Q^T, masked softmax
//      (sparse.py:370-372), P as bf16 hi + lo, O^T = V^T . P^T, written as an
//      unnormalised partial; the last tile to finish merges the partials into
//      the output row and its LSE.
// The last CTA to finish bumps every sequence's device-side length and resets
// the counters for the next step.
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

constexpr int kG = 16;
constexpr int kD = 128;
constexpr int kS = 16;
constexpr int kM = 64;
constexpr int kThreads = 192;
constexpr int kStages = 3;
constexpr int kMaxTiles = 28;                 // z tiles resident in TMEM (16 columns each)
constexpr int kMaxRows = kMaxTiles * 128;     // kernels per piece
constexpr int kMaxPieceBlocks = (kMaxRows - 1) / 4;
constexpr int kCandCap = kMaxRows * 4 / 8;    // (key, id) pairs in the sarr alias
constexpr int kMaxPieces = 160;               // >= SM count
constexpr int kMaxT2 = 40;                    // stage-2 tiles per segment (max_sel <= 80)
constexpr int kPartStride = kG * kD + 2 * kG; // floats per stage-2 partial
constexpr uint32_t kColS2 = 448;
constexpr uint32_t kColO = 464;

constexpr uint32_t kHalf = 128 * 128;         // 16 KB: 128 rows x 64 bf16
constexpr uint32_t kStageBytes = 4 * kHalf;   // 64 KB: mu hi/lo tile, or K + V tile
constexpr uint32_t kQB = 2 * kG * 128;        // 4 KB
constexpr uint32_t kPHalf = 128 * kG * 2;     // 4 KB

struct Smem {
  static constexpr uint32_t ring = 0;
  static constexpr uint32_t q = ring + kStages * kStageBytes;
  static constexpr uint32_t p = q + kQB;                         // P hi/lo; top-k lists alias it
  static constexpr uint32_t sarr = p + 2 * kPHalf;               // S_j per kernel; merge list alias
  static constexpr uint32_t rarr = sarr + kMaxRows * 4;          // R_b per block
  static constexpr uint32_t red = rarr + (kMaxPieceBlocks + 9) * 4;
  static constexpr uint32_t bars = (red + (4 * kG * 2 + 2 * kG + 8) * 4 + 7) / 8 * 8;
  static constexpr uint32_t total = bars + (kMaxTiles + 16) * 8 + 16;
};
static_assert(Smem::total + 1024 <= 232448, "fused decode shared memory");
static_assert(topk::kListCap * 8 <= 2 * kPHalf, "top-k lists alias the P buffer");
static_assert(kCandCap * 4 <= 2 * kPHalf, "merge flags alias the P buffer");

struct Params {
  void* table;
  int n_seq, hkv, hq;
  int top_k, n_init, n_local, consume, max_sel, coarse_stride, cmax;
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  int32_t* selection;      // [seq][g][max_sel]
  void* out;
  int out_f32;
  float* lse;
  float* pstat;            // [seg][kMaxPieces][16][2]
  float* cand;             // [seg][kMaxPieces][32][2]  (key, id bits)
  float* part;             // [seg][kMaxT2][kPartStride]
  float zscale;            // log2(e) / sqrt(D)
  int trace;
};

// Per-CTA assignment (thread 0 computes, everyone reads).
struct Info {
  int active, s, g, sg, piece, c;
  int64_t pos, nk, n_cand, b0, b1, r0, r1;
  int ntiles, dirty_tile;
  int64_t dlo;                 // first dirty window (rows [dlo, nk) change this step)
  // selection geometry (force_blocks / select_topk rules)
  int n_init, local_lo, n_loc, budget, n_free, n_ch, n_sel, nf, t2;
};

// Optional phase timeline (INFLLM2_DECODE_TRACE=1): %globaltimer per CTA and
// phase, read back with infllm2_debug_decode_trace (tools/decode_trace.py).
// `on` = launch number + 1; the last kTraceRing launches are kept.
constexpr int kTracePts = 16;
constexpr int kTraceRing = 4;
__device__ unsigned long long g_trace[kTraceRing * kMaxPieces * kTracePts];
__device__ __forceinline__ void trace(int on, int pt) {
  if (on) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[(((on - 1) % kTraceRing) * kMaxPieces + blockIdx.x) * kTracePts + pt] = t;
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Bounded spin: a broken dependency chain traps (launch error) instead of
// hanging the GPU.
__device__ __forceinline__ void spin_until(const int* p, int target) {
  for (uint32_t n = 0; ld_acquire(p) < target; ++n) {
    __nanosleep(32);
    if (n > (1u << 26)) __trap();
  }
}
// Publish this CTA's prior global writes (made visible to thread 0 by the
// preceding bar.sync) and count one arrival: one gpu-scope fence per CTA.
__device__ __forceinline__ int publish_arrive(int* ctr) {
  int old;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
  return old;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

__device__ void compute_info(const Params& p, const int64_t* len, Info& I) {
  const int nseg = p.n_seq * p.hkv;
  int64_t total = 0;
  for (int s = 0; s < p.n_seq; ++s) total += (int64_t)p.hkv * (len[s] / kM + 1);
  const int64_t avail = (int64_t)gridDim.x - nseg;
  I.active = 0;
  int acc = 0;
  for (int sg = 0; sg < nseg; ++sg) {
    const int s = sg / p.hkv;
    const int64_t nb = len[s] / kM + 1;
    int64_t c = 1 + (avail > 0 ? avail * nb / total : 0);
    if (c > p.cmax) c = p.cmax;
    if (c > nb) c = nb;
    if ((int)blockIdx.x < acc + c) {
      I.active = 1;
      I.s = s;
      I.g = sg - s * p.hkv;
      I.sg = sg;
      I.piece = (int)blockIdx.x - acc;
      I.c = (int)c;
      I.pos = len[s];
      I.n_cand = nb;
      I.b0 = I.piece * nb / c;
      I.b1 = (I.piece + 1) * nb / c;
      break;
    }
    acc += (int)c;
  }
  if (!I.active) return;
  const int64_t L = I.pos + 1;
  I.nk = L / kS;                                       // nk_t == nk for the newest row
  I.r0 = I.b0 == 0 ? 0 : 4 * I.b0 - 1;
  I.r1 = 4 * I.b1 < I.nk ? 4 * I.b1 : I.nk;
  if (I.r1 < I.r0) I.r1 = I.r0;
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
  I.t2 = (I.n_sel + 1) / 2;
}

// Stage-2 order: forced blocks first (init, then local), then the chosen ones.
__device__ __forceinline__ bool tile_needs_sel(const Info& I, int t) {
  const int e1 = 2 * t + 1 < I.n_sel ? 2 * t + 1 : 2 * t;
  return e1 >= I.nf;
}
__device__ __forceinline__ int entry_block(const Info& I, const int* sel_s, int e) {
  if (e >= I.n_sel) return -1;
  if (e < I.n_init) return e;
  if (e < I.nf) return I.local_lo + (e - I.n_init);
  return sel_s[I.n_init + (e - I.nf)];
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

__global__ void __launch_bounds__(kThreads, 1)
decode_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* full = bars;                 // [3]
  uint64_t* empty = bars + 3;            // [3]
  uint64_t* q_full = bars + 6;
  uint64_t* appended = bars + 7;         // 128 epilogue arrivals
  uint64_t* s2_full = bars + 8;
  uint64_t* s2_empty = bars + 9;         // 4 warps
  uint64_t* p_full = bars + 10;          // 4 warps
  uint64_t* o_full = bars + 11;
  uint64_t* o_empty = bars + 12;         // 4 warps
  uint64_t* sel_ready = bars + 13;       // selection merged into sel_s
  uint64_t* s_full = bars + 16;          // [kMaxTiles], one phase each
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16 + kMaxTiles);
  float* red = reinterpret_cast<float*>(smem + Smem::red);
  __shared__ Info I;
  __shared__ int s_flag;
  __shared__ int sel_s[96];              // this segment's selection (every piece merges it)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TableView tv = table_view(p.table, p.n_seq);
  {
    int64_t* len_s = reinterpret_cast<int64_t*>(smem + Smem::sarr);   // free until phase C
    for (int s = threadIdx.x; s < p.n_seq; s += blockDim.x) len_s[s] = tv.len[s];
    __syncthreads();
    if (threadIdx.x == 0) {
      trace(p.trace, 0);
      if (p.trace) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace[(((p.trace - 1) % kTraceRing) * kMaxPieces + blockIdx.x) * kTracePts + 11] = smid;
      }
      compute_info(p, len_s, I);
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    mbar_init(q_full, 1);
    mbar_init(appended, 128);
    mbar_init(s2_full, 1);
    mbar_init(s2_empty, 4);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    mbar_init(sel_ready, 1);
    for (int t = 0; t < kMaxTiles; ++t) mbar_init(s_full + t, 1);
    fence_barrier_init();
    tma_prefetch(&tm_q);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int* seg_ctr = tv.fused + 4 * (I.active ? I.sg : 0);   // [0] stage-1, [1] candidates, [3] stage-2
  const SeqDesc ds = tv.desc[I.active ? I.s : 0];
  int32_t* sel_row = p.selection + (int64_t)(I.active ? I.sg : 0) * p.max_sel;   // output

  if (I.active) {
    if (warp == 0) {
      // ============================================================ producer
      if (elect_one()) {
        const CUtensorMap* mhi = tv.maps + (int64_t)kMaps * I.s + 2;
        const CUtensorMap* mlo = tv.maps + (int64_t)kMaps * I.s + 3;
        const CUtensorMap* mk = tv.maps + (int64_t)kMaps * I.s + 0;
        const CUtensorMap* mv = tv.maps + (int64_t)kMaps * I.s + 1;
        mbar_arrive_expect_tx(q_full, kQB);
        uint8_t* qd = smem + Smem::q;
        tma_load_3d(qd, &tm_q, q_full, 0, I.g * kG, I.s);
        tma_load_3d(qd + kQB / 2, &tm_q, q_full, 64, I.g * kG, I.s);
        int stage = 0;
        uint32_t phase = 0;
        for (int t = 0; t < I.ntiles; ++t) {
          if (t == I.dirty_tile) mbar_wait(appended, 0);   // this CTA's window re-sync is in global memory
          mbar_wait(empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, kStageBytes);
          uint8_t* dst = smem + Smem::ring + stage * kStageBytes;
          const int row = (int)(I.r0 + 128 * t);
          tma_load_3d(dst, mhi, full + stage, 0, row, I.g);
          tma_load_3d(dst + kHalf, mhi, full + stage, 64, row, I.g);
          tma_load_3d(dst + 2 * kHalf, mlo, full + stage, 0, row, I.g);
          tma_load_3d(dst + 3 * kHalf, mlo, full + stage, 64, row, I.g);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        trace(p.trace, 1);
        for (int t = I.piece; t < I.t2; t += I.c) {
          // K/V row of this step is written before the segment's stage-1 counter completes
          if (tile_needs_sel(I, t)) mbar_wait(sel_ready, 0);   // implies the segment's stage 1 is complete
          else spin_until(seg_ctr + 0, I.c);
          fence_proxy_async_global();
          if (t == I.piece) trace(p.trace, 7);
          const int b0 = entry_block(I, sel_s, 2 * t), b1 = entry_block(I, sel_s, 2 * t + 1);
          const int nt = b1 >= 0 ? 2 : 1;
          mbar_wait(empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, nt * 4 * (kM * 128));
          uint8_t* kd = smem + Smem::ring + stage * kStageBytes;
          uint8_t* vd = kd + 2 * kHalf;
          for (int x = 0; x < nt; ++x) {
            const int row0 = (x ? b1 : b0) * kM;
            const uint32_t off = x * kM * 128;
            tma_load_3d(kd + off, mk, full + stage, 0, row0, I.g);
            tma_load_3d(kd + kHalf + off, mk, full + stage, 64, row0, I.g);
            tma_load_3d(vd + off, mv, full + stage, 0, row0, I.g);
            tma_load_3d(vd + kHalf + off, mv, full + stage, 64, row0, I.g);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ============================================================ MMA issuer
      const uint32_t idesc = idesc_bf16_f32(128, kG);
      const uint32_t idesc_pv = idesc_bf16_f32_major(128, kG, 1, 1);
      mbar_wait(q_full, 0);
      const uint32_t q_addr = smem_u32(smem + Smem::q);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < I.ntiles; ++t) {
        mbar_wait(full + stage, phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t mu_s = smem_u32(smem + Smem::ring + stage * kStageBytes);
          for (int part = 0; part < 2; ++part)
            for (int k = 0; k < kD / 16; ++k) {
              const uint32_t koff = (k & 3) * 32;
              umma_f16_ss(tmem + t * kG, sdesc_k_sw128(mu_s + part * 2 * kHalf + (k >> 2) * kHalf + koff),
                          sdesc_k_sw128(q_addr + (k >> 2) * (kQB / 2) + koff), idesc, (part | k) ? 1u : 0u);
            }
          umma_commit(empty + stage);
          umma_commit(s_full + t);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      int i2 = 0;
      for (int t = I.piece; t < I.t2; t += I.c, ++i2) {
        const int nt = (I.n_sel - 2 * t) >= 2 ? 2 : 1;
        const uint32_t par = i2 & 1;
        mbar_wait(full + stage, phase);
        mbar_wait(s2_empty, par ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + Smem::ring + stage * kStageBytes);
        if (elect_one()) {
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
            const uint32_t qoff = (k >> 2) * (kQB / 2) + (k & 3) * 32;
            umma_f16_ss(tmem + kColS2, sdesc_k_sw128(k_addr + off), sdesc_k_sw128(q_addr + qoff), idesc, k > 0 ? 1u : 0u);
          }
          umma_commit(s2_full);
        }
        __syncwarp();
        mbar_wait(p_full, par);
        mbar_wait(o_empty, par ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t v_addr = k_addr + 2 * kHalf;
          const uint32_t p_addr = smem_u32(smem + Smem::p);
          const int ksteps = nt == 2 ? 8 : 4;
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t vdesc = sdesc_mn_sw128(v_addr + k * 2048, kHalf, 1024);
            umma_f16_ss(tmem + kColO, vdesc, sdesc_interleave(p_addr + k * 512, 256, 128), idesc_pv, k > 0 ? 1u : 0u);
            umma_f16_ss(tmem + kColO, vdesc, sdesc_interleave(p_addr + kPHalf + k * 512, 256, 128), idesc_pv, 1u);
          }
          umma_commit(empty + stage);
          umma_commit(o_full);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    } else {
      // ============================================================ epilogue (128 threads)
      const int tid = threadIdx.x - 64;
      const int quad = warp & 3;
      const int row = quad * 32 + lane;                // TMEM lane
      const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
      const int64_t L = I.pos + 1;
      // ---- A. append: dirty windows in [r0, r1) (+ K/V row and coarse window on the last piece)
      const int d = tid;
      const __nv_bfloat16* kg = ds.k + (int64_t)I.g * ds.cap * kD;
      const int64_t knew_idx = ((int64_t)I.s * p.hkv + I.g) * kD + d;
      {
        // at most two fine windows change (nk - dlo <= 2): their <= 48 rows are
        // loaded in ONE round (latency under the stage-1 stream is microseconds),
        // summed as window_mean does (sequential float64, numpy reduce order)
        const int64_t jlo = I.dlo > I.r0 ? I.dlo : I.r0;
        if (jlo < I.r1) {
          const float knew = __bfloat162float(p.k_new[knew_idx]);
          const int64_t row0 = jlo * kS;
          float x[kP + kS];
#pragma unroll
          for (int i = 0; i < kP + kS; ++i) {
            const int64_t r = row0 + i;
            x[i] = r < L && r != I.pos ? __bfloat162float(kg[r * kD + d]) : 0.f;
          }
#pragma unroll
          for (int i = 0; i < kP + kS; ++i)
            if (row0 + i == I.pos) x[i] = knew;
          auto emit = [&](int64_t j, const float* xs) {
            int64_t w64 = L - j * kS;
            const int w = (int)(w64 < kP ? w64 : kP);
            double acc = (double)xs[0];
#pragma unroll
            for (int r = 1; r < kP; ++r)
              if (r < w) acc += (double)xs[r];
            const float mu = __double2float_rn(acc / (double)w);
            const int64_t dst = ((int64_t)I.g * ds.means_cap + j) * kD + d;
            ds.fine[dst] = mu;
            const __nv_bfloat16 h = __float2bfloat16_rn(mu);
            ds.hi[dst] = h;
            ds.lo[dst] = __float2bfloat16_rn(mu - __bfloat162float(h));
          };
          emit(jlo, x);
          if (jlo + 1 < I.r1) emit(jlo + 1, x + kS);
        }
        fence_proxy_async_global();
        mbar_arrive(appended);
        if (tid == 0) trace(p.trace, 13);
        if (I.piece == I.c - 1) {   // not needed by stage 1: after the arrival
          const float knew = __bfloat162float(p.k_new[knew_idx]);
          ds.k[((int64_t)I.g * ds.cap + I.pos) * kD + d] = p.k_new[knew_idx];
          ds.v[((int64_t)I.g * ds.cap + I.pos) * kD + d] = p.v_new[knew_idx];
          const int cs = p.coarse_stride;
          int64_t first = I.pos < kP ? 0 : (I.pos - kP) / cs + 1;
          const int64_t count_old = I.pos / cs, count = L / cs;
          if (first > count_old) first = count_old;
          if (first < count) {
            const float mu = window_mean(kg, kD, first, cs, L, d, I.pos, knew);
            ds.coarse[((int64_t)I.g * ds.coarse_cap + first) * kD + d] = mu;
          }
        }
      }
      // ---- B. stage-1 partial (max, sum 2^z) over owned kernels [4*b0, r1)
      const int64_t own0 = 4 * I.b0;
      float m[kG], sm[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h) { m[h] = -INFINITY; sm[h] = 0.f; }
      for (int t = 0; t < I.ntiles; ++t) {
        mbar_wait(s_full + t, 0);
        tc_fence_after();
        float v[kG];
        tmem_ld16(tmem + lane_base + t * kG, v);
        tmem_wait_ld();
        if (t == 0 && tid == 0) trace(p.trace, 12);
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
      float* red_m = red;
      float* red_s = red + 4 * kG;
      float* lse2 = red + 8 * kG;
#pragma unroll
      for (int h = 0; h < kG; ++h) {
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
      float* ps_seg = p.pstat + (int64_t)I.sg * kMaxPieces * (2 * kG);
      if (tid < kG) {
        float M = -INFINITY;
        for (int x = 0; x < 4; ++x) M = fmaxf(M, red_m[tid * 4 + x]);
        float S = 0.f;
        for (int x = 0; x < 4; ++x) {
          const float mm = red_m[tid * 4 + x];
          if (mm != -INFINITY) S += red_s[tid * 4 + x] * ex2(mm - M);
        }
        ps_seg[I.piece * 2 * kG + 2 * tid] = M;
        ps_seg[I.piece * 2 * kG + 2 * tid + 1] = S;
      }
      named_bar_sync(1, 128);
      if (tid == 0) {
        trace(p.trace, 2);
        publish_arrive(seg_ctr + 0);
        spin_until(seg_ctr + 0, I.c);
        trace(p.trace, 3);
      }
      named_bar_sync(1, 128);
      // ---- C. LSE, group scores, block scores, local top-k
      float* sarr = reinterpret_cast<float*>(smem + Smem::sarr);
      for (int x = tid; x < I.c * 2 * kG; x += 128) sarr[x] = __ldcg(ps_seg + x);   // all partials in flight
      named_bar_sync(1, 128);
      if (tid < kG) {
        float M = -INFINITY, S = 0.f;
        for (int x = 0; x < I.c; ++x) {
          const float mm = sarr[x * 2 * kG + 2 * tid], ss = sarr[x * 2 * kG + 2 * tid + 1];
          if (mm == -INFINITY) continue;
          const float nm = fmaxf(M, mm);
          S = (M == -INFINITY ? 0.f : S * ex2(M - nm)) + ss * ex2(mm - nm);
          M = nm;
        }
        lse2[tid] = M == -INFINITY ? INFINITY : M + log2f(S);
      }
      named_bar_sync(1, 128);
      float* rarr = reinterpret_cast<float*>(smem + Smem::rarr);
      {
        float l2[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) l2[h] = lse2[h];
        tc_fence_after();
        for (int t = 0; t < I.ntiles; ++t) {
          float v[kG];
          tmem_ld16(tmem + lane_base + t * kG, v);
          tmem_wait_ld();
          const int64_t jl = 128 * t + row;
          if (I.r0 + jl < I.r1) {
            float a = 0.f;
#pragma unroll
            for (int h = 0; h < kG; ++h) a += ex2(v[h] * p.zscale - l2[h]);
            sarr[jl] = a * (1.0f / kG);
          }
        }
      }
      named_bar_sync(1, 128);
      for (int64_t b = I.b0 + tid; b < I.b1; b += 128) {
        int64_t end = (b + 1) * kM;
        if (end > L) end = L;
        int64_t lo, hi;
        kernel_range_for_block(b * kM, end, kP, kS, I.nk, &lo, &hi);
        float r = 0.f;
        if (hi > lo) {
          r = sarr[lo - I.r0];
          for (int64_t j = lo + 1; j < hi; ++j) r = fmaxf(r, sarr[j - I.r0]);
        }
        rarr[b - I.b0] = r;
      }
      named_bar_sync(1, 128);
      if (tid == 0) trace(p.trace, 4);
      const bool dense = I.budget >= I.n_free || I.budget == 0;
      float* cand_seg = p.cand + (int64_t)I.sg * kMaxPieces * 64;
      if (!dense && warp == 2) {
        int lo = (int)((I.b0 > I.n_init ? I.b0 : I.n_init) - I.b0);
        int hi = (int)((I.b1 < I.local_lo ? I.b1 : I.local_lo) - I.b0);
        if (hi < lo) hi = lo;
        float* lkey = reinterpret_cast<float*>(smem + Smem::p);
        int* lid = reinterpret_cast<int*>(lkey + topk::kListCap);
        local_topk(rarr, I.b0, lo, hi, I.budget, lane, lkey, lid, cand_seg + I.piece * 64);
      }
      named_bar_sync(1, 128);
      if (tid == 0) {
        trace(p.trace, 5);
        publish_arrive(seg_ctr + 1);
        spin_until(seg_ctr + 1, I.c);
      }
      named_bar_sync(1, 128);
      {
        // ---- merge (every piece, redundantly: no publish hop): the global
        // top-B lies in the union of the pieces' local top-B lists
        float* lk = sarr;                                         // [n][2] (key, id bits)
        int* chosen = reinterpret_cast<int*>(smem + Smem::p);    // flags (P buffer is idle here)
        const int n = dense ? 0 : I.c * I.budget;
        for (int x = tid; x < n; x += 128) {
          const int off = 2 * x + (x / I.budget) * (64 - 2 * I.budget);
          const float2 kv = __ldcg(reinterpret_cast<const float2*>(cand_seg + off));
          lk[2 * x] = kv.x;
          lk[2 * x + 1] = kv.y;
        }
        named_bar_sync(1, 128);
        // Filter: a full local list's worst key tau_i is <= the global B-th
        // best (that list alone has B keys >= tau_i), so keys < max_i tau_i
        // cannot be selected.  Typically leaves ~B..2B of the c*B candidates.
        int* cnt = reinterpret_cast<int*>(red + 8 * kG + kG);     // after lse2
        float* fl = rarr;                                          // filtered (key, id) pairs
        const int fcap = (kMaxPieceBlocks + 8) / 2;
        if (tid == 0) *cnt = 0;
        float tau = -INFINITY;
        for (int i = tid; i < (dense ? 0 : I.c); i += 128) {
          float mn = INFINITY;
          bool full_list = true;
          for (int k = 0; k < I.budget; ++k) {
            full_list &= __float_as_int(lk[2 * (i * I.budget + k) + 1]) >= 0;
            mn = fminf(mn, lk[2 * (i * I.budget + k)]);
          }
          if (full_list) tau = fmaxf(tau, mn);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) tau = fmaxf(tau, __shfl_xor_sync(0xffffffffu, tau, off));
        if (lane == 0) red_m[quad] = tau;
        named_bar_sync(1, 128);
        tau = fmaxf(fmaxf(red_m[0], red_m[1]), fmaxf(red_m[2], red_m[3]));
        for (int x = tid; x < n; x += 128) {
          const float k = lk[2 * x];
          const int id = __float_as_int(lk[2 * x + 1]);
          if (id >= 0 && k >= tau) {
            const int slot = atomicAdd(cnt, 1);
            if (slot < fcap) { fl[2 * slot] = k; fl[2 * slot + 1] = lk[2 * x + 1]; }
          }
        }
        named_bar_sync(1, 128);
        const int m = *cnt;
        const bool use_f = m <= fcap;
        const float* L2 = use_f ? fl : lk;
        const int nn = use_f ? m : n;
        for (int x = tid; x < nn; x += 128) {
          const float rk = L2[2 * x];
          const int bk = __float_as_int(L2[2 * x + 1]);
          int keep = 0;
          if (bk >= 0 && rk >= tau) {
            int rank = 0;
#pragma unroll 8
            for (int y = 0; y < nn; ++y) {
              const int by = __float_as_int(L2[2 * y + 1]);
              rank += (by >= 0 && topk::better(L2[2 * y], by, rk, bk)) ? 1 : 0;
            }
            keep = rank < I.budget;
          }
          chosen[x] = keep ? bk : -1;
        }
        named_bar_sync(1, 128);
        for (int x = tid; x < nn; x += 128) {
          const int bk = chosen[x];
          if (bk < 0) continue;
          int posn = 0;
#pragma unroll 8
          for (int y = 0; y < nn; ++y) {
            const int cy = chosen[y];
            posn += (cy >= 0 && cy < bk) ? 1 : 0;
          }
          sel_s[I.n_init + posn] = bk;
        }
        for (int x = tid; x < p.max_sel; x += 128) {
          int id = -2;
          if (dense) id = x < I.n_cand ? x : -1;
          else if (x < I.n_init) id = x;
          else if (x >= I.n_init + I.n_ch && x < I.n_sel) id = I.local_lo + (x - I.n_init - I.n_ch);
          else if (x >= I.n_sel) id = -1;
          if (id != -2) sel_s[x] = id;
        }
        named_bar_sync(1, 128);
        if (tid == 0) {
          mbar_arrive(sel_ready);
          trace(p.trace, 6);
        }
        if (I.piece == 0)
          for (int x = tid; x < p.max_sel; x += 128) sel_row[x] = sel_s[x];
      }
      // ---- D. stage 2 (this piece's tiles)
      const float c2 = p.zscale;
      int i2 = 0;
      float* part_seg = p.part + (int64_t)I.sg * kMaxT2 * kPartStride;
      for (int t = I.piece; t < I.t2; t += I.c, ++i2) {
        const uint32_t par = i2 & 1;
        const int bx = entry_block(I, sel_s, 2 * t + (row >> 6));
        mbar_wait(s2_full, par);
        tc_fence_after();
        float z[kG];
        tmem_ld16(tmem + lane_base + kColS2, z);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s2_empty);
        const bool valid = bx >= 0 && (int64_t)bx * kM + (row & 63) <= I.pos;
#pragma unroll
        for (int h = 0; h < kG; ++h) z[h] = valid ? z[h] * c2 : -INFINITY;
        // tile max per head across the 128 rows
#pragma unroll
        for (int h = 0; h < kG; ++h) {
          float v = z[h];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
          if (lane == h) red_m[quad * kG + h] = v;
        }
        named_bar_sync(1, 128);
        float mt[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h)
          mt[h] = fmaxf(fmaxf(red_m[h], red_m[kG + h]), fmaxf(red_m[2 * kG + h], red_m[3 * kG + h]));
        uint32_t phi[kG / 2], plo[kG / 2];
        float pl[kG];
#pragma unroll
        for (int h = 0; h < kG; h += 2) {
          const float a = ex2(z[h] - mt[h]);
          const float b = ex2(z[h + 1] - mt[h + 1]);
          pl[h] = a;
          pl[h + 1] = b;
          const __nv_bfloat162 hi2 = __floats2bfloat162_rn(a, b);
          const __nv_bfloat162 lo2 = __floats2bfloat162_rn(a - __low2float(hi2), b - __high2float(hi2));
          phi[h / 2] = *reinterpret_cast<const uint32_t*>(&hi2);
          plo[h / 2] = *reinterpret_cast<const uint32_t*>(&lo2);
        }
        uint8_t* pb = smem + Smem::p;
        const uint32_t base = (row >> 3) * 256 + (row & 7) * 16;
        *reinterpret_cast<uint4*>(pb + base) = make_uint4(phi[0], phi[1], phi[2], phi[3]);
        *reinterpret_cast<uint4*>(pb + base + 128) = make_uint4(phi[4], phi[5], phi[6], phi[7]);
        *reinterpret_cast<uint4*>(pb + kPHalf + base) = make_uint4(plo[0], plo[1], plo[2], plo[3]);
        *reinterpret_cast<uint4*>(pb + kPHalf + base + 128) = make_uint4(plo[4], plo[5], plo[6], plo[7]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        // row sums per head
#pragma unroll
        for (int h = 0; h < kG; ++h) {
          float v = pl[h];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
          if (lane == h) red_s[quad * kG + h] = v;
        }
        mbar_wait(o_full, par);
        tc_fence_after();
        float o[kG];
        tmem_ld16(tmem + lane_base + kColO, o);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty);
        float* pt = part_seg + (int64_t)t * kPartStride;
        const int d = row;                              // O^T lane == d
#pragma unroll
        for (int h = 0; h < kG; ++h) pt[h * kD + d] = o[h];
        named_bar_sync(1, 128);                         // red_s complete
        if (tid < kG) {
          pt[kG * kD + 2 * tid] = mt[tid];
          pt[kG * kD + 2 * tid + 1] = red_s[tid] + red_s[kG + tid] + red_s[2 * kG + tid] + red_s[3 * kG + tid];
        }
        named_bar_sync(1, 128);
        if (tid == 0) {
          if (i2 == 0) trace(p.trace, 8);
          s_flag = (publish_arrive(seg_ctr + 3) == I.t2 - 1);
          if (s_flag) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        named_bar_sync(1, 128);
        if (s_flag) {
          // ---- merge the segment's stage-2 partials -> output row + LSE
          if (tid == 0) trace(p.trace, 14);
          float* wgt = sarr;                             // [t2][16]
          float* inv_l = sarr + kMaxT2 * kG;
          float* ml = inv_l + kG;                        // [t2][16][2]
          for (int x = tid; x < I.t2 * 2 * kG; x += 128)
            ml[x] = __ldcg(part_seg + (int64_t)(x / (2 * kG)) * kPartStride + kG * kD + (x % (2 * kG)));
          named_bar_sync(1, 128);
          if (tid < kG) {
            float M = -INFINITY;
            for (int x = 0; x < I.t2; ++x) M = fmaxf(M, ml[(x * kG + tid) * 2]);
            float Lsum = 0.f;
            for (int x = 0; x < I.t2; ++x) {
              const float mm = ml[(x * kG + tid) * 2];
              const float w = mm == -INFINITY ? 0.f : ex2(mm - M);
              wgt[x * kG + tid] = w;
              Lsum += ml[(x * kG + tid) * 2 + 1] * w;
            }
            inv_l[tid] = 1.f / Lsum;
            if (p.lse) p.lse[(int64_t)I.s * p.hq + I.g * kG + tid] = (M + log2f(Lsum)) * 0.6931471805599453f;
          }
          named_bar_sync(1, 128);
          if (tid == 0) trace(p.trace, 15);
          // thread -> heads 4*hp..4*hp+3 at d in [4*c4, 4*c4+4): every partial's
          // float4 loads are independent, so many are in flight per thread
          const int c4 = tid & 31, hp = tid >> 5;        // hp in 0..3 -> heads 4*hp .. 4*hp+3
          float4 acc[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 5
          for (int x = 0; x < I.t2; ++x) {
            float4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              v[k] = __ldcg(reinterpret_cast<const float4*>(part_seg + (int64_t)x * kPartStride + (4 * hp + k) * kD) + c4);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float w = wgt[x * kG + 4 * hp + k];
              acc[k].x += v[k].x * w;
              acc[k].y += v[k].y * w;
              acc[k].z += v[k].z * w;
              acc[k].w += v[k].w * w;
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int h = 4 * hp + k;
            const float il = inv_l[h];
            const int64_t oi = ((int64_t)I.s * p.hq + I.g * kG + h) * kD + 4 * c4;
            if (p.out_f32) {
              *reinterpret_cast<float4*>(static_cast<float*>(p.out) + oi) =
                  make_float4(acc[k].x * il, acc[k].y * il, acc[k].z * il, acc[k].w * il);
            } else {
              __nv_bfloat162 a = __floats2bfloat162_rn(acc[k].x * il, acc[k].y * il);
              __nv_bfloat162 b = __floats2bfloat162_rn(acc[k].z * il, acc[k].w * il);
              uint2 u;
              u.x = *reinterpret_cast<uint32_t*>(&a);
              u.y = *reinterpret_cast<uint32_t*>(&b);
              *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.out) + oi) = u;
            }
          }
        }
        if (s_flag && tid == 0) trace(p.trace, 9);
        named_bar_sync(1, 128);                          // red_m / red_s / s_flag reuse
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {
    trace(p.trace, 10);
    const int nseg = p.n_seq * p.hkv;
    int* done = tv.fused + 4 * nseg;
    if (publish_arrive(done) == (int)gridDim.x - 1) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      // every CTA has finished: the new token is part of the caches now
      for (int s = 0; s < p.n_seq; ++s) tv.len[s] += 1;
      for (int x = 0; x < 4 * nseg; ++x) tv.fused[x] = 0;
      *done = 0;
      __threadfence();
    }
  }
}

}  // namespace

size_t decode_fused_workspace_bytes(int n_seq, int hkv) {
  const size_t nseg = (size_t)n_seq * hkv;
  return align_up(nseg * kMaxPieces * 2 * kG * sizeof(float), 256) + align_up(nseg * kMaxPieces * 64 * sizeof(float), 256) +
         align_up(nseg * kMaxT2 * kPartStride * sizeof(float), 256);
}

// Host-side eligibility: the partition must fit the TMEM-resident z tiles and
// the merge list for every length up to max_len_after.
bool decode_fused_supported(const infllm2_geometry& g, int n_seq, int hkv, int64_t max_len_after, int sms) {
  if (getenv("INFLLM2_DECODE_LEGACY")) return false;
  const int nseg = n_seq * hkv;
  if (nseg > sms || sms > kMaxPieces) return false;
  if (g.top_k > 32 || g.top_k < 1) return false;
  if (infllm2_max_selected(&g) > 2 * kMaxT2) return false;
  const int64_t nb_max = max_len_after / kM + 1;
  const int64_t avail = sms - nseg;
  const int cmax = kCandCap / g.top_k;
  int64_t per_piece = avail > 0 ? (nseg * nb_max + avail - 1) / avail : nb_max;
  const int64_t capped = (nb_max + cmax - 1) / cmax;
  if (capped > per_piece) per_piece = capped;
  return per_piece + 1 <= kMaxPieceBlocks;
}

int decode_fused_step(const infllm2_geometry& g, void* table, int n_seq, int hq, int hkv, const void* q,
                      const void* k_new, const void* v_new, int32_t* selection, void* out, int out_f32, float* lse,
                      void* ws, cudaStream_t stream, int sms) {
  Params p;
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
  p.cmax = kCandCap / g.top_k;
  if (p.cmax > kMaxPieces) p.cmax = kMaxPieces;
  p.k_new = static_cast<const __nv_bfloat16*>(k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(v_new);
  p.selection = selection;
  p.out = out;
  p.out_f32 = out_f32;
  p.lse = lse;
  const size_t nseg = (size_t)n_seq * hkv;
  uint8_t* b = static_cast<uint8_t*>(ws);
  p.pstat = reinterpret_cast<float*>(b);
  b += align_up(nseg * kMaxPieces * 2 * kG * sizeof(float), 256);
  p.cand = reinterpret_cast<float*>(b);
  b += align_up(nseg * kMaxPieces * 64 * sizeof(float), 256);
  p.part = reinterpret_cast<float*>(b);
  p.zscale = 1.4426950408889634f / sqrtf((float)kD);
  static const bool tr = getenv("INFLLM2_DECODE_TRACE") != nullptr;
  static int launches = 0;
  p.trace = tr ? 1 + (launches++ % kTraceRing) : 0;
  CUtensorMap tq;
  const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)hq, (uint64_t)n_seq};
  const uint64_t strides[2] = {(uint64_t)kD * 2, (uint64_t)hq * kD * 2};
  const uint32_t box[3] = {64, (uint32_t)kG, 1};
  if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return INFLLM2_ERR_SHAPE;
  const size_t smem = Smem::total + 1024;
  if (cudaFuncSetAttribute(decode_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return INFLLM2_ERR_CUDA;
  static const bool coop = getenv("INFLLM2_DECODE_NOCOOP") == nullptr;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  count_launch();
  if (cudaLaunchKernelEx(&cfg, decode_fused_kernel, tq, p) != cudaSuccess) return INFLLM2_ERR_CUDA;
  return INFLLM2_OK;
}

}  // namespace infllm2

// Debug: copy the traced launches' per-CTA phase timestamps (ns,
// [4 launches][kMaxPieces][12], ring by launch number) to host memory.
extern "C" int infllm2_debug_decode_trace(unsigned long long* host, int max_entries) {
  const int cap = infllm2::kTraceRing * infllm2::kMaxPieces * infllm2::kTracePts;
  const int n = max_entries < cap ? max_entries : cap;
  return cudaMemcpyFromSymbol(host, infllm2::g_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
