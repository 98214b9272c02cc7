// Stage-1 block selection on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Production geometry: GQA group G = 16 heads, D = 128, s = 16, p = 2s, m a
// multiple of s with (m/s) | 128.  Replaces, for every query row and KV group,
// kernel_scores + softmax_f64 + group_scores + block_scores + force_blocks +
// select_topk (sparse.py:163-277, model.py:185-191) as called per row by
// two_stage_attention (sparse.py:421-451).
//
// Work unit = 16 consecutive query positions t0..t0+15 (t0 % 16 == 0) of one
// KV group: 256 (query, head) rows.  Because 16 | s and 16 | m, all 16 rows
// see the same kernel count nk_t = min(t0/s + 1, L/s) (sparse.py:426) and the
// same candidate blocks, so one unit is one dense, masked-at-the-tail GEMM.
//
// Kernel means enter as a bf16 hi/lo split (mu = hi + lo to ~2^-17 relative,
// SURVEY F7): every product is formed twice and accumulated in f32 TMEM.
//
//   pass 1  S[row, j]   = Q(256x128) . mu^T        (A = Q rows, B = mu tile)
//           online max / sum of 2^z per row   ->  lse2[row]     (softmax normaliser)
//   pass 2  S^T[j, row] = mu(128x128) . Q^T        (A = mu tile, B = Q, N = 256)
//           p = 2^(z - lse2[row]); group score S_j = mean_h p    (in-thread: a thread
//           owns one kernel j and all 16 heads of a query -> no shuffles)
//           block max over each block's kernels (sparse.py:191-215) -> workspace
//   top-k   per query: forced blocks + budget best non-forced by (-R, id).
//
// Warp roles (10 warps): 0 = TMA producer, 1 = TMEM allocator + MMA issuer,
// 2..9 = epilogue (TMEM -> registers -> softmax math).  TMEM: 512 columns =
// two 256-column accumulator buffers, so the epilogue of tile c overlaps the
// MMAs of tile c+1.  Shared memory: Q 64 KB + 2 stages x 64 KB of mu.
#include <float.h>
#include <limits.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tc_dispatch.cuh"
#include "topk.cuh"

namespace infllm2 {

namespace {

using namespace sm100;

#ifdef SEL_PROFILE
// per-CTA cycle counters (variant builds only, tools/build_variant.sh -DSEL_PROFILE):
// [0] epilogue warp 2 total, [1] its acc_full waits, [2] its pass-1 time,
// [3] MMA warp total, [4] MMA mu_full waits, [5] MMA acc_empty waits
__device__ long long g_sel_cyc[160][8];
#define SEL_T0(v) long long v = clock64()
#define SEL_ADD(slot, v) (g_sel_cyc[blockIdx.x][slot] += clock64() - (v))
#else
#define SEL_T0(v)
#define SEL_ADD(slot, v)
#endif
constexpr int kQ = 16;            // query positions per work unit
constexpr int kG = 16;            // heads per KV group
constexpr int kRows = kQ * kG;    // 256 (query, head) rows
constexpr int kNT = 128;          // kernels per tile
constexpr int kStages = 2;
#ifndef SEL_POLY
#define SEL_POLY 0   // of every 4 odd element pairs, how many take 2^x on the FMA pipe
#endif
#ifndef SEL_P2N256
#define SEL_P2N256 1   // pass 2 as one N = 256 MMA per K-step: ~1 % faster than 2 x N = 128 (13.96 vs 14.11 ms per 128K layer)
#endif
#ifndef SEL_SPLIT
#define SEL_SPLIT 1   // 2 (16 epilogue warps, 80 registers): stage 1 alone -6 %, full step equal (clocks drop under sw_power_cap)
#endif
constexpr int kSplit = SEL_SPLIT;           // epilogue warps per TMEM quadrant and half
constexpr int kEpiWarps = 8 * kSplit;
constexpr int kTopkWarps = 4;     // dedicated selection warps (4 queries each)
constexpr int kThreads = 32 * (2 + kEpiWarps + kTopkWarps);
constexpr int kEpiThreads = 32 * kEpiWarps;
using topk::kListCap;
using topk::kOutCap;
using topk::UnitSel;
using topk::unit_sel;
using topk::warp_select;

constexpr uint32_t kMuHalfBytes = kNT * 64 * 2;            // 16 KB (128 rows x 128 B)
constexpr int kSTileLd = kNT + 4;                          // epilogue scratch (see the epilogue)

// Per-geometry constants: G heads per KV group, head dim D; a unit is always
// 256 (query, head) rows, i.e. kQ = 256 / G query positions (16 for the 8B
// shape, 32 for MiniCPM4-0.5B's G = 8, D = 64).
template <int G, int D>
struct SelCfg {
  static constexpr int kQ = kRows / G;
  static constexpr int kDH = D / 64;
  static constexpr uint32_t kQBytes = kRows * D * 2;
  static constexpr uint32_t kMuStageBytes = 2 * kDH * kMuHalfBytes;   // hi halves, then lo halves
  static_assert(2 * kSplit * kRows + 3 * 2 * kSplit * 8 * (128 / G / kSplit) <= kQ * kSTileLd, "epilogue scratch");
  struct Smem {
    static constexpr uint32_t q = 0;
    static constexpr uint32_t mu = q + kQBytes;
    static constexpr uint32_t stile = mu + kStages * kMuStageBytes;   // epilogue scratch
    static constexpr uint32_t lse2 = stile + kQ * kSTileLd * 4;       // float [kRows]
    static constexpr uint32_t bars = lse2 + kRows * 4;                // uint64 [..]
    static constexpr uint32_t topk = bars + 24 * 8;                   // per top-k warp lists
    static constexpr uint32_t topk_per_warp = kListCap * 8;
    static constexpr uint32_t total = topk + kTopkWarps * topk_per_warp + 16;
  };
};


struct Params {
  int64_t n, start, cache_len, nk_total;
  int hkv, max_sel;
  int m, kpb;                     // block size, kernels per block
  int top_k, n_init, n_local, consume;
  int64_t units_per_group, n_units;
  int64_t first_t0;               // aligned position of unit 0
  int32_t* selection;
  double* sel_scores;
  float* rbuf;                    // [grid][2][kQ][nb_cap]  block scores, double-buffered per unit
  int64_t nb_cap;
  float zscale;                   // log2(e)/sqrt(D)
  int kq;                         // query positions per unit (256 / G)
  int dbg;                        // INFLLM2_SELECT_DBG in -DSEL_PROFILE builds (experiments), else 0
  // approx-LSE mode (DESIGN §4 K2p): pass 1 over the nc_t coarse kernels,
  // LSE + log2(s_c / s); pass 2 unchanged
  int approx;
  int64_t nc_total;
  int p1hi;                       // experiment (INFLLM2_SELECT_P1HI=1): pass 1 over mu_hi only
  // broadcast position (tree-draft nodes, infllm2_forward_tree): every row
  // sits at position bpos; units are 16 consecutive ROWS (start = 0)
  int bcast;
  int64_t bpos;
  int sc;
  float lse_bias2;
};

// unit index -> (t0, group); heaviest (largest t0) units first
__device__ __forceinline__ void unit_coords(const Params& p, int64_t u, int64_t* t0, int* grp) {
  const int64_t tile = p.units_per_group - 1 - u / p.hkv;
  *grp = (int)(u % p.hkv);
  *t0 = p.first_t0 + tile * p.kq;
}

// position of unit coordinate t (the row's own position, or the broadcast one)
__device__ __forceinline__ int64_t upos(const Params& p, int64_t t) { return p.bcast ? p.bpos : t; }

// kernel count of query position t (sparse.py:426)
__device__ __forceinline__ int64_t pos_nk(const Params& p, int64_t t) {
  t = upos(p, t);
  int64_t nk = t / 16 + 1;
  return nk < p.nk_total ? nk : p.nk_total;
}
// largest kernel count in the unit (its last query)
__device__ __forceinline__ int64_t unit_nk(const Params& p, int64_t t0) { return pos_nk(p, t0 + p.kq - 1); }
// coarse kernel count of query position t (approx-LSE mode)
__device__ __forceinline__ int64_t pos_nc(const Params& p, int64_t t) {
  t = upos(p, t);
  const int64_t nc = t / p.sc + 1;
  return nc < p.nc_total ? nc : p.nc_total;
}
// pass-1 kernel count of position t: fine kernels, or coarse ones in approx mode
__device__ __forceinline__ int64_t pos_n1(const Params& p, int64_t t) { return p.approx ? pos_nc(p, t) : pos_nk(p, t); }

__device__ __forceinline__ int unit_tiles(const Params& p, int64_t t0, int64_t nk) {
  const int64_t qb = upos(p, t0) / p.m;
  int64_t need = (qb + 1) * p.kpb;
  if (nk > need) need = nk;
  return (int)((need + kNT - 1) / kNT);
}

template <int G, int D>
__global__ void __launch_bounds__(kThreads, 1)
select_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_hi,
                 const __grid_constant__ CUtensorMap tm_lo, const __grid_constant__ CUtensorMap tm_chi,
                 const __grid_constant__ CUtensorMap tm_clo, const Params p) {
  using C = SelCfg<G, D>;
  using SmemLayout = typename C::Smem;
  constexpr int kQ = C::kQ;
  constexpr int kG = G;
  constexpr int kD = D;
  constexpr uint32_t kQBytes = C::kQBytes;
  constexpr uint32_t kMuStageBytes = C::kMuStageBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by pointer arithmetic on the __shared__ array (a uintptr_t round trip
  // loses the address space: every access would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sq = smem + SmemLayout::q;
  uint8_t* smu = smem + SmemLayout::mu;
  float* stile = reinterpret_cast<float*>(smem + SmemLayout::stile);
  float* lse2 = reinterpret_cast<float*>(smem + SmemLayout::lse2);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout::bars);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* mu_full = bars + 2;             // [kStages]
  uint64_t* mu_empty = bars + 2 + kStages;  // [kStages]
  uint64_t* acc_full = bars + 2 + 2 * kStages;       // [2]
  uint64_t* acc_empty = bars + 4 + 2 * kStages;      // [2]
  uint64_t* rb_full = bars + 6 + 2 * kStages;        // [2] block scores of a unit ready
  uint64_t* rb_empty = bars + 8 + 2 * kStages;       // [2] top-k warps done with them
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(bars + 10 + 2 * kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SEL_T0(t_kernel);

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kStages; ++s) { mbar_init(mu_full + s, 1); mbar_init(mu_empty + s, 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, kEpiWarps);
      mbar_init(rb_full + b, kEpiWarps);
      mbar_init(rb_empty + b, kTopkWarps);
    }
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_hi);
    tma_prefetch(&tm_lo);
  }
  if (warp == 1) tmem_alloc<512>(tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0, q_phase = 0;
      for (int64_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        int64_t t0;
        int grp;
        unit_coords(p, u, &t0, &grp);
        const int64_t nk = unit_nk(p, t0);
        const int tiles = unit_tiles(p, t0, nk);
        const int tiles1 = p.approx ? (int)((pos_nc(p, t0 + p.kq - 1) + kNT - 1) / kNT) : tiles;
        mbar_wait(q_empty, q_phase ^ 1);
        q_phase ^= 1;
        mbar_arrive_expect_tx(q_full, kQBytes);
        const int i0 = (int)(t0 - p.start);
#pragma unroll
        for (int hh = 0; hh < C::kDH; ++hh) tma_load_3d(sq + hh * (kRows * 128), &tm_q, q_full, 64 * hh, grp * kG, i0);
        for (int pass = 0; pass < 2; ++pass) {
          const CUtensorMap* mh = (pass == 0 && p.approx) ? &tm_chi : &tm_hi;
          const CUtensorMap* ml = (pass == 0 && p.approx) ? &tm_clo : &tm_lo;
          for (int c = 0; c < (pass ? tiles : tiles1); ++c) {
            mbar_wait(mu_empty + stage, phase ^ 1);
            uint8_t* dst = smu + stage * kMuStageBytes;
            const bool hi_only = pass == 0 && p.p1hi;
            mbar_arrive_expect_tx(mu_full + stage, hi_only ? kMuStageBytes / 2 : kMuStageBytes);
#pragma unroll
            for (int hh = 0; hh < C::kDH; ++hh) {
              tma_load_3d(dst + hh * kMuHalfBytes, mh, mu_full + stage, 64 * hh, c * kNT, grp);
              if (!hi_only) tma_load_3d(dst + (C::kDH + hh) * kMuHalfBytes, ml, mu_full + stage, 64 * hh, c * kNT, grp);
            }
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc1 = idesc_bf16_f32(128, 128);
    [[maybe_unused]] const uint32_t idesc2 = idesc_bf16_f32(128, 256);
    const uint32_t q_addr = smem_u32(sq);
    const uint32_t mu_addr = smem_u32(smu);
    int stage = 0, buf = 0;
    uint32_t phase = 0, q_phase = 0;
    uint32_t acc_phase[2] = {0, 0};
    for (int64_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      int64_t t0;
      int grp;
      unit_coords(p, u, &t0, &grp);
      const int64_t nk = unit_nk(p, t0);
      const int tiles = unit_tiles(p, t0, nk);
      const int tiles1 = p.approx ? (int)((pos_nc(p, t0 + p.kq - 1) + kNT - 1) / kNT) : tiles;
      mbar_wait(q_full, q_phase);
      q_phase ^= 1;
      for (int pass = 0; pass < 2; ++pass) {
        for (int c = 0; c < (pass ? tiles : tiles1); ++c) {
          SEL_T0(tw0);
          mbar_wait(mu_full + stage, phase);
          if (lane == 0) SEL_ADD(4, tw0);
          SEL_T0(tw1);
          mbar_wait(acc_empty + buf, acc_phase[buf] ^ 1);
          if (lane == 0) SEL_ADD(5, tw1);
          acc_phase[buf] ^= 1;
          tc_fence_after();
          if (elect_one()) {
            const uint32_t mu_s = mu_addr + stage * kMuStageBytes;
            const uint32_t d0 = tmem + buf * 256;
            const int parts = (pass == 0 && p.p1hi) ? 1 : 2;
            for (int part = 0; part < parts; ++part) {       // hi, then lo
              const uint32_t mu_p = mu_s + part * C::kDH * kMuHalfBytes;
              for (int k = 0; k < kD / 16; ++k) {
                const uint32_t koff = (k >> 2) * 0 + (k & 3) * 32;
                const uint32_t mu_k = mu_p + (k >> 2) * kMuHalfBytes + koff;
                const uint32_t q_k = q_addr + (k >> 2) * (kRows * 128) + koff;
                const uint32_t acc = (part | k) ? 1u : 0u;
                if (pass == 0) {
                  umma_f16_ss(d0, sdesc_k_sw128(q_k), sdesc_k_sw128(mu_k), idesc1, acc);
                  umma_f16_ss(d0 + 128, sdesc_k_sw128(q_k + 128 * 128), sdesc_k_sw128(mu_k), idesc1, acc);
                } else {
#if SEL_P2N256
                  // one N = 256 MMA: the mu tile (A) is fetched once per K-step
                  // instead of twice (12 KB of SMEM operands instead of 16)
                  umma_f16_ss(d0, sdesc_k_sw128(mu_k), sdesc_k_sw128(q_k), idesc2, acc);
#else
                  // N = 256 split into two independent N = 128 accumulators
                  // (columns 0-127 / 128-255), issued alternately: a dependent
                  // N = 256 chain costs ~190 cycles per MMA, two interleaved
                  // N = 128 chains ~75 each (tools/mma_bench.cu)
                  umma_f16_ss(d0, sdesc_k_sw128(mu_k), sdesc_k_sw128(q_k), idesc1, acc);
                  umma_f16_ss(d0 + 128, sdesc_k_sw128(mu_k), sdesc_k_sw128(q_k + 128 * 128), idesc1, acc);
#endif
                }
              }
            }
            umma_commit(mu_empty + stage);
            umma_commit(acc_full + buf);
            if (pass == 1 && c == tiles - 1) umma_commit(q_empty);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
          buf ^= 1;
        }
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    // kEpiWarps = 8 * kSplit warps: groups ("subs") of four warps cover the
    // four TMEM lane quadrants; sub = (column part, half).  More warps per
    // SM sub-partition hide the TMEM-load / MUFU latency of each thread's
    // chain (the epilogue, not the tensor pipe, bounds this kernel).
    const int ew = warp - 2;                 // 0..kEpiWarps-1
    const int quad = warp & 3;               // TMEM lane quadrant this warp may access
    const int sub = ew >> 2;                 // 0..2*kSplit-1
    const int half = sub & 1;                // pass 1: row half; pass 2: query half
    const int cpart = sub >> 1;              // pass 1: column part; pass 2: query part
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    [[maybe_unused]] const int etid = ew * 32 + lane;   // kSplit > 1 only
    int buf = 0;
    uint32_t acc_phase[2] = {0, 0};
    int ucount = 0;
    constexpr int kQC = 32 / kG;                     // queries per 32-column chunk
    constexpr int kQH = 128 / kG;                    // queries per column half
    constexpr int kQS = kQH / kSplit;                // queries per sub in pass 2
    constexpr int kCols1 = 128 / kSplit;             // pass-1 columns per thread
    // scratch in the stile region: pass-1 partial (max, sum) per (part, row),
    // then pass-2 carries [3 slots][subs][2][4 quads][kQS]
    [[maybe_unused]] float* pm = stile;
    [[maybe_unused]] float* ps = stile + kSplit * kRows;
    float* carries = stile + 2 * kSplit * kRows;
    for (int64_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++ucount) {
      float* rbuf = p.rbuf + ((int64_t)blockIdx.x * 2 + (ucount & 1)) * kQ * p.nb_cap;
      int64_t t0;
      int grp;
      unit_coords(p, u, &t0, &grp);
      const int64_t nk = unit_nk(p, t0);
      const int tiles = unit_tiles(p, t0, nk);
      const int tiles1 = p.approx ? (int)((pos_nc(p, t0 + p.kq - 1) + kNT - 1) / kNT) : tiles;
      const int64_t qb = upos(p, t0) / p.m;
      const int64_t n_cand = qb + 1;

      SEL_T0(tp1);
      // ---- pass 1: row LSE (log2 domain).  Max on the raw accumulator
      // (zscale > 0), FFMA+ex2 with four independent partial sums; masking
      // only on the tail tile.
      {
        const int row = half * 128 + quad * 32 + lane;
        const int64_t nk_row = pos_n1(p, t0 + row / kG);    // rows of one query share its kernel count
        const int64_t nk_min = pos_n1(p, t0);
        float mrun = -INFINITY, srun = 0.f;
        for (int c = 0; c < tiles1; ++c) {
          SEL_T0(tw);
          mbar_wait(acc_full + buf, acc_phase[buf]);
          if (warp == 2 && lane == 0) SEL_ADD(1, tw);
          acc_phase[buf] ^= 1;
          tc_fence_after();
          if (p.dbg & 4) { __syncwarp(); if (lane == 0) mbar_arrive(acc_empty + buf); buf ^= 1; continue; }
          const int64_t jbase = (int64_t)c * kNT + cpart * kCols1;
          const bool tail = (int64_t)c * kNT + kNT > nk_min;
          // 32-column chunks, the next chunk's TMEM load in flight while this
          // one is reduced (tcgen05.wait::ld waits for all loads, so the wait
          // sits after the compute)
          const uint32_t cbase = tmem + lane_base + buf * 256 + half * 128 + cpart * kCols1;
          float va[32], vb[32];
          tmem_ld32(cbase, va);
          tmem_wait_ld();
#pragma unroll
          for (int ch = 0; ch < kCols1 / 32; ++ch) {
            float* v = (ch & 1) ? vb : va;
            if (ch + 1 < kCols1 / 32)
              tmem_ld32(cbase + (ch + 1) * 32, *reinterpret_cast<float(*)[32]>((ch & 1) ? va : vb));
            if (tail) {
              const int64_t j0 = jbase + ch * 32;
#pragma unroll
              for (int x = 0; x < 32; ++x) v[x] = (j0 + x < nk_row) ? v[x] : -INFINITY;
            }
            // packed fp32 pairs (FFMA2 / FADD2) and 3-input max: the same
            // per-element arithmetic and summation order as four scalar
            // partial sums a[x & 3]
            float mA = v[0], mB = v[1];
#pragma unroll
            for (int x = 2; x < 30; x += 4) { mA = fmax3(mA, v[x], v[x + 1]); mB = fmax3(mB, v[x + 2], v[x + 3]); }
            const float cmax = fmaxf(fmax3(mA, v[30], v[31]), mB) * p.zscale;
            const float mnew = fmaxf(mrun, cmax);
            if (mnew != -INFINITY) {
              const uint64_t zs2 = pk2(p.zscale, p.zscale), nm2 = pk2(-mnew, -mnew);
              uint64_t s01 = 0, s23 = 0;
#pragma unroll
              for (int x = 0; x < 32; x += 4) {
                float e0, e1, e2, e3;
                upk2(ffma2(pk2(v[x], v[x + 1]), zs2, nm2), e0, e1);
                const uint64_t x23 = ffma2(pk2(v[x + 2], v[x + 3]), zs2, nm2);
                upk2(x23, e2, e3);
                s01 = fadd2(s01, pk2(ex2(e0), ex2(e1)));
                // SEL_POLY of every 4 odd pairs on the FMA pipe (MUFU relief)
                s23 = fadd2(s23, ((x >> 2) & 3) < SEL_POLY ? ex2_poly2(x23) : pk2(ex2(e2), ex2(e3)));
              }
              float a0, a1, a2, a3;
              upk2(s01, a0, a1);
              upk2(s23, a2, a3);
              srun = srun * ex2(mrun - mnew) + ((a0 + a1) + (a2 + a3));
              mrun = mnew;
            }
            if (ch + 1 < kCols1 / 32) tmem_wait_ld();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty + buf);
          buf ^= 1;
        }
        if constexpr (kSplit == 1) {
          lse2[row] = -(mrun + log2f(srun) + p.lse_bias2);     // negated: the FFMA2 addend
        } else {
          pm[cpart * kRows + row] = mrun;
          ps[cpart * kRows + row] = srun;
        }
      }
      if (warp == 2 && lane == 0) SEL_ADD(2, tp1);
      named_bar_sync(1, kEpiThreads);
      if constexpr (kSplit > 1) {
        if (etid < kRows) {
          float m = pm[etid];
#pragma unroll
          for (int x = 1; x < kSplit; ++x) m = fmaxf(m, pm[x * kRows + etid]);
          float sum = 0.f;
#pragma unroll
          for (int x = 0; x < kSplit; ++x) {
            const float mx = pm[x * kRows + etid];
            sum += (mx == -INFINITY) ? 0.f : ps[x * kRows + etid] * ex2(mx - m);
          }
          lse2[etid] = -(m + log2f(sum) + p.lse_bias2);
        }
        named_bar_sync(1, kEpiThreads);
      }

      // ---- pass 2: group scores per kernel, block max.  A thread owns one
      // kernel (TMEM lane) and kQS queries; lanes hold consecutive kernels,
      // so block b's kernels [b*kpb - 1, (b+1)*kpb) (sparse.py:191-215: the
      // boundary kernel is shared with block b-1) are a shuffle-reduction
      // over kpb lanes plus the previous lane; the kernel before a warp's
      // lane 0 comes from the neighbouring quadrant (same tile) or the
      // previous tile through a small smem carry.
      mbar_wait(rb_empty + (ucount & 1), ((ucount >> 1) & 1) ^ 1);
      const int kpb = p.kpb;
      const int kpb_log2 = __ffs(kpb) - 1;                     // kpb is a power of two
      const int jl = quad * 32 + lane;
      const bool first = (jl & (kpb - 1)) == 0;
      const int q0 = half * kQH + cpart * kQS;                 // this sub's first query
      // a thread's queries lie in one 16-position group of the (16- or
      // 32-aligned) unit, so with s = 16 they share one kernel count
      const int64_t nk_thr = pos_nk(p, t0 + q0);
      for (int c = 0; c < tiles; ++c) {
        SEL_T0(tw);
        mbar_wait(acc_full + buf, acc_phase[buf]);
        if (warp == 2 && lane == 0) SEL_ADD(1, tw);
        acc_phase[buf] ^= 1;
        tc_fence_after();
        if (p.dbg & 2) {   // timing experiment: no pass-2 math (selection invalid)
          __syncwarp(); if (lane == 0) mbar_arrive(acc_empty + buf); buf ^= 1;
          if (sub == 0) named_bar_sync(2, 128); else if (sub == 1) named_bar_sync(3, 128);
          else if (sub == 2) named_bar_sync(4, 128); else named_bar_sync(5, 128);
          continue;
        }
        const int64_t jg = (int64_t)c * kNT + jl;               // this thread's kernel
        const int64_t b = jg >> kpb_log2;
        const bool writer = first && b < n_cand;
        const bool live = jg < nk_thr;
        // [slot][sub][carry | part0][quad][kQS]: lane-31 scores (the kernel
        // before the next quadrant's lane 0) and lane-0 partial block maxima;
        // three slots so tile c + 3's writes never race tile c + 1's reads
        const int slot = c % 3;
        float* carry = carries + (slot * 2 * kSplit + sub) * 8 * kQS;
        float* part0 = carry + 4 * kQS;
        const uint32_t cbase = tmem + lane_base + buf * 256 + q0 * kG;
        float va[32], vb[32];
        tmem_ld32(cbase, va);
        tmem_wait_ld();
#pragma unroll
        for (int qq = 0; qq < kQS; qq += kQC) {
          const int ch = qq / kQC;
          float* v = (ch & 1) ? vb : va;
          if (qq + kQC < kQS) tmem_ld32(cbase + (ch + 1) * 32, *reinterpret_cast<float(*)[32]>((ch & 1) ? va : vb));
          float sc[kQC];
#pragma unroll
          for (int u4 = 0; u4 < kQC; ++u4) {
            const int qi = q0 + qq + u4;
            const uint32_t l2 = smem_u32(lse2 + qi * kG);
            // packed pairs: acc = (a0, a1), a0 over even heads, a1 over odd
            // heads, in head order (the scalar two-accumulator order)
            const uint64_t zs2 = pk2(p.zscale, p.zscale);
            uint64_t acc = 0;
#pragma unroll
            for (int h = 0; h < kG; h += 4) {
              const float4 l4 = lds4(l2 + h * 4);                // -lse2
              float e0, e1, e2, e3;
              upk2(ffma2(pk2(v[u4 * kG + h], v[u4 * kG + h + 1]), zs2, pk2(l4.x, l4.y)), e0, e1);
              const uint64_t x23 = ffma2(pk2(v[u4 * kG + h + 2], v[u4 * kG + h + 3]), zs2, pk2(l4.z, l4.w));
              upk2(x23, e2, e3);
              acc = fadd2(acc, pk2(ex2(e0), ex2(e1)));
              acc = fadd2(acc, ((u4 * kG + h) / 4 & 3) < SEL_POLY ? ex2_poly2(x23) : pk2(ex2(e2), ex2(e3)));
            }
            float a0, a1;
            upk2(acc, a0, a1);
            sc[u4] = live ? (a0 + a1) * (1.0f / kG) : -INFINITY;
          }
          float r[kQC];
#pragma unroll
          for (int u4 = 0; u4 < kQC; ++u4) {
            const float up = __shfl_up_sync(0xffffffffu, sc[u4], 1);
            r[u4] = (first && lane > 0) ? fmaxf(sc[u4], up) : sc[u4];
          }
          // butterfly over the kpb lanes of a block: unconditional shuffles (a
          // loop bounded by the runtime kpb costs a WARPSYNC per step)
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            if (o >= 4 && o >= kpb) break;               // uniform; kpb <= 4 never takes it
#pragma unroll
            for (int u4 = 0; u4 < kQC; ++u4) {
              const float t = __shfl_xor_sync(0xffffffffu, r[u4], o);
              r[u4] = o < kpb ? fmaxf(r[u4], t) : r[u4];
            }
          }
#pragma unroll
          for (int u4 = 0; u4 < kQC; ++u4) {
            const int qi = q0 + qq + u4;
            st_shared_if(smem_u32(carry + quad * kQS + qq + u4), sc[u4], lane == 31);
            st_shared_if(smem_u32(part0 + quad * kQS + qq + u4), r[u4], lane == 0);
            st_global_if(rbuf + (int64_t)qi * p.nb_cap + b, (r[u4] == -INFINITY) ? 0.f : r[u4], writer && lane > 0);
          }
          if (qq + kQC < kQS) tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + buf);
        buf ^= 1;
        switch (sub) {                       // constant barrier ids (a variable id reserves all 16)
          case 0: named_bar_sync(2, 128); break;
          case 1: named_bar_sync(3, 128); break;
          case 2: named_bar_sync(4, 128); break;
          default: named_bar_sync(5, 128); break;
        }
        {   // lane 0's block also holds the previous kernel: lane x finishes query x
          const float* prev = (quad > 0) ? carry + (quad - 1) * kQS
                                         : carries + (((slot + 2) % 3) * 2 * kSplit + sub) * 8 * kQS + 3 * kQS;
          const int x = lane & (kQS - 1);
          const int64_t b0 = ((int64_t)c * kNT + quad * 32) >> kpb_log2;
          const float pr = (quad == 0 && c == 0) ? -INFINITY : prev[x];
          const float r = fmaxf(part0[quad * kQS + x], pr);
          st_global_if(rbuf + (int64_t)(q0 + x) * p.nb_cap + b0, (r == -INFINITY) ? 0.f : r,
                       lane < kQS && b0 < n_cand);
        }
      }

      // hand the unit's block scores to the top-k warps
      __threadfence_block();
      __syncwarp();
      if (lane == 0) mbar_arrive(rb_full + (ucount & 1));
    }
  } else {
    // ------------------------------------------------------------ top-k warps
    const int tw = warp - 2 - kEpiWarps;     // 0..kTopkWarps-1
    float* lkey = reinterpret_cast<float*>(smem + SmemLayout::topk + tw * SmemLayout::topk_per_warp);
    int* lid = reinterpret_cast<int*>(lkey + kListCap);
    int ucount = 0;
    for (int64_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++ucount) {
      int64_t t0;
      int grp;
      unit_coords(p, u, &t0, &grp);
      const UnitSel us = unit_sel(upos(p, t0), p.m, p.top_k, p.n_init, p.n_local, p.consume);
      const float* rbuf = p.rbuf + ((int64_t)blockIdx.x * 2 + (ucount & 1)) * kQ * p.nb_cap;
      mbar_wait(rb_full + (ucount & 1), (ucount >> 1) & 1);
      for (int qi = tw; qi < kQ; qi += kTopkWarps) {
        const int64_t i = t0 + qi - p.start;
        if (i < 0 || i >= p.n || (p.dbg & 1)) continue;     // warp-uniform
        const int64_t item = i * p.hkv + grp;
        warp_select(rbuf + (int64_t)qi * p.nb_cap, us, lane, lkey, lid, p.selection + item * p.max_sel,
                    p.sel_scores ? p.sel_scores + item * p.max_sel : nullptr, p.max_sel);
        __syncwarp();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(rb_empty + (ucount & 1));
    }
  }

  tc_fence_before();
  __syncthreads();
#ifdef SEL_PROFILE
  if (lane == 0 && warp == 2) SEL_ADD(0, t_kernel);
  if (lane == 0 && warp == 1) SEL_ADD(3, t_kernel);
#endif
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(ptr);
  }();
  return fn;
}

}  // namespace

bool encode_tmap_3d_bf16(CUtensorMap* map, const void* base, const uint64_t dims[3],
                         const uint64_t strides_bytes[2], const uint32_t box[3]) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t gd[3] = {dims[0], dims[1], dims[2]};
  cuuint64_t gs[2] = {strides_bytes[0], strides_bytes[1]};
  cuuint32_t bx[3] = {box[0], box[1], box[2]};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gd, gs, bx, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int tc_grid(int64_t n_units) {
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static const int cap = [] {
    const char* e = getenv("INFLLM2_SELECT_CTAS");
    return e ? atoi(e) : 0;
  }();
  if (cap > 0 && cap < sms) sms = cap;
  return (int)(n_units < sms ? n_units : sms);
}

bool tc_kernels_enabled() {
  static const bool on = [] {
    const char* e = getenv("INFLLM2_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool tc_select_shape(const CallShape& cs, int* kq) {
  if (cs.group == 16 && cs.d == 128) { *kq = 16; return true; }
  if (cs.group == 8 && cs.d == 64) { *kq = 32; return true; }
  return false;
}

bool tc_select_supported(const infllm2_geometry& g, const CallShape& cs, bool have_split_means) {
  if (!have_split_means || !tc_kernels_enabled()) return false;
  int kq;
  if (!tc_select_shape(cs, &kq)) return false;
  if (g.kernel_stride != 16 || g.kernel_size != 32) return false;
  // every query of a unit (kq consecutive positions) must share the candidate blocks
  // kernels per block (a power of two dividing the 128-kernel tile) must fit
  // in one warp: the block max is a shuffle reduction over lanes
  if (g.block_size % kq != 0 || kNT % (g.block_size / 16) != 0 || g.block_size / 16 > 32) return false;
  if (g.top_k + g.n_init_blocks + g.n_local_blocks > 80) return false;
  if (cs.nk_total < 1) return false;
  return true;
}

size_t tc_select_workspace(const infllm2_geometry& g, const CallShape& cs, int) {
  int kq;
  if (!tc_select_shape(cs, &kq)) return 0;
  const int64_t nb_cap = cs.cache_len / g.block_size + 2;
  return (size_t)kNumSMs * 2 * kq * nb_cap * sizeof(float);
}

template <int G, int D>
static cudaError_t launch_select_shape(const CallShape& cs, const void* q, int64_t q_row_stride, const void* means_hi,
                                       const void* means_lo, int64_t means_cap, Params& p, void* ws, size_t ws_bytes,
                                       cudaStream_t stream, const CoarseArgs* coarse) {
  using C = SelCfg<G, D>;
  constexpr int kQ = C::kQ;
  p.kq = kQ;
  p.bcast = cs.bcast;
  p.bpos = cs.start;
  if (cs.bcast) p.start = 0;          // unit coordinates are row indices; every row at position bpos
  p.first_t0 = p.start / kQ * kQ;
  const int64_t last = p.start + cs.n - 1;
  p.units_per_group = (last - p.first_t0) / kQ + 1;
  p.n_units = p.units_per_group * cs.hkv;
  p.zscale = 1.4426950408889634f / sqrtf((float)D);
  {
    const char* e = getenv("INFLLM2_SELECT_P1HI");
    p.p1hi = e && e[0] == '1';
  }
#ifdef SEL_PROFILE
  p.dbg = getenv("INFLLM2_SELECT_DBG") ? atoi(getenv("INFLLM2_SELECT_DBG")) : 0;   // experiments only
#else
  p.dbg = 0;
#endif
  const int grid = tc_grid(p.n_units);
  if ((size_t)grid * 2 * kQ * p.nb_cap * sizeof(float) > ws_bytes || ws == nullptr) return cudaErrorInvalidValue;
  p.rbuf = static_cast<float*>(ws);
  CUtensorMap tq, thi, tlo, tchi, tclo;
  {
    const uint64_t dims[3] = {(uint64_t)D, (uint64_t)cs.hq, (uint64_t)cs.n};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)q_row_stride * 2};
    const uint32_t box[3] = {64, (uint32_t)G, (uint32_t)kQ};
    if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {(uint64_t)D, (uint64_t)means_cap, (uint64_t)cs.hkv};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)means_cap * D * 2};
    const uint32_t box[3] = {64, (uint32_t)kNT, 1};
    if (!encode_tmap_3d_bf16(&thi, means_hi, dims, strides, box)) return cudaErrorInvalidValue;
    if (!encode_tmap_3d_bf16(&tlo, means_lo, dims, strides, box)) return cudaErrorInvalidValue;
  }
  if (p.approx) {
    const uint64_t dims[3] = {(uint64_t)D, (uint64_t)coarse->cap, (uint64_t)cs.hkv};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)coarse->cap * D * 2};
    const uint32_t box[3] = {64, (uint32_t)kNT, 1};
    if (!encode_tmap_3d_bf16(&tchi, coarse->hi, dims, strides, box)) return cudaErrorInvalidValue;
    if (!encode_tmap_3d_bf16(&tclo, coarse->lo, dims, strides, box)) return cudaErrorInvalidValue;
  } else {
    tchi = thi;
    tclo = tlo;
  }
  const size_t smem = C::Smem::total + 1024;
  {
    cudaError_t e = smem_attr_once((const void*)select_tc_kernel<G, D>, (int)smem);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  select_tc_kernel<G, D><<<grid, kThreads, smem, stream>>>(tq, thi, tlo, tchi, tclo, p);
  return cudaGetLastError();
}

cudaError_t launch_select_tc(const infllm2_geometry& g, const CallShape& cs, const void* q,
                             int64_t q_row_stride, const float* /*means*/, const void* means_hi,
                             const void* means_lo, int64_t means_cap, int32_t* selection,
                             double* sel_scores, void* ws, size_t ws_bytes, cudaStream_t stream,
                             const CoarseArgs* coarse) {
  Params p;
  p.approx = coarse != nullptr;
  p.nc_total = coarse ? coarse->nc_total : 0;
  p.sc = (int)g.coarse_stride;
  p.lse_bias2 = coarse ? log2f((float)g.coarse_stride / (float)g.kernel_stride) : 0.f;
  p.n = cs.n;
  p.start = cs.start;
  p.cache_len = cs.cache_len;
  p.nk_total = cs.nk_total;
  p.hkv = cs.hkv;
  p.max_sel = cs.max_sel;
  p.m = g.block_size;
  p.kpb = g.block_size / g.kernel_stride;
  p.top_k = g.top_k;
  p.n_init = g.n_init_blocks;
  p.n_local = g.n_local_blocks;
  p.consume = g.forced_consume_budget;
  p.selection = selection;
  p.sel_scores = sel_scores;
  p.nb_cap = cs.cache_len / g.block_size + 2;
  if (cs.group == 8 && cs.d == 64)
    return launch_select_shape<8, 64>(cs, q, q_row_stride, means_hi, means_lo, means_cap, p, ws, ws_bytes, stream,
                                      coarse);
  return launch_select_shape<16, 128>(cs, q, q_row_stride, means_hi, means_lo, means_cap, p, ws, ws_bytes, stream,
                                      coarse);
}

}  // namespace infllm2

extern "C" int infllm2_debug_select_cycles(long long* host, int max_entries) {
#ifdef SEL_PROFILE
  const int n = max_entries < 160 * 8 ? max_entries : 160 * 8;
  return cudaMemcpyFromSymbol(host, infllm2::g_sel_cyc, sizeof(long long) * n) == cudaSuccess ? 0 : -1;
#else
  for (int i = 0; i < max_entries; ++i) host[i] = 0;
  return 1;   // not a profiling build
#endif
}
