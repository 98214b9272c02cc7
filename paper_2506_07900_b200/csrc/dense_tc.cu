// Dense causal GQA attention on the tensor cores: the below-threshold path of
// InfLLM v2 (every block selected) and the dense backend of the
// model seam (model.py:194-253, masked grouped attention).  Query row i at
// position start + i attends cache rows [0, start + i].
//
// One work item = 8 consecutive query rows x one KV group = an M = 128 tile of
// (query, head) rows (row r = 16 q + h), so every K/V byte feeds 128 rows
// instead of the sparse kernel's 16:
//
//   S   [128 (q,h) x 128 keys] = Q (K-major) . K_tile^T            (TMEM, 2 slots)
//   softmax warps: thread = (q,h) row, causal mask, running max with a rare
//     rescale (threshold 8 in log2 units), P = 2^(z - M) -> bf16 -> smem
//     (K-major, 128-B swizzle); items below position 256 also keep the bf16
//     lo part (second PV MMA) so few-key rows stay exact to ~1e-5
//   O^T [128 d x 128 (q,h)]  += V_tile^T (MN-major) . P^T            (TMEM)
//
// Warp roles (12 warps): 0 = TMA producer (Q per item, K + V per tile, two
// stages), 1 = TMEM alloc + MMA issuer, 4..11 = softmax, then epilogue.  Warps
// w and w + 4 share TMEM lane quadrant w % 4: thread = (q,h) row r, the first
// four take keys 0..63 of every tile, the others keys 64..127 (half maxima
// exchanged through smem as bf16 rounded up; one OR-reducing barrier per tile
// is also the rescale vote); in the epilogue thread = d lane of O^T over its half of the
// (q,h) columns (divide by the row sums, store) and thread = row (LSE).
#include <float.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"
#include "tc_dispatch.cuh"

namespace infllm2 {

bool tc_kernels_enabled();

namespace {

using namespace sm100;

constexpr int kG = 16;
constexpr int kD = 128;
constexpr int kQR = 8;                        // query rows per item (8 x 16 heads = 128 MMA rows)
constexpr int kKT = 128;                      // keys per tile
constexpr int kThreads = 384;
#ifndef DENSE_SLOTS
#define DENSE_SLOTS 2   // 3 measured equal (softmax-bound)
#endif
constexpr int kSSlots = DENSE_SLOTS;          // S tiles in TMEM (QK runs up to kSSlots tiles ahead)
static_assert(kSSlots >= 2 && kSSlots <= 3, "S slots + O^T must fit 512 TMEM columns");
constexpr int64_t kSplitBelow = 256;          // items starting below this position carry P lo too
constexpr uint32_t kHalf = 128 * 128;         // 16 KB: 128 rows x 64 bf16 (one 128-B swizzle half)
constexpr uint32_t kTile = 2 * kHalf;         // 32 KB: 128 rows x 128 bf16

struct Smem {
  static constexpr uint32_t q = 0;                          // 32 KB
  static constexpr uint32_t kv = q + kTile;                 // [2 stages][K, V] 128 KB
  static constexpr uint32_t p = kv + 4 * kTile;             // [2] P tiles (hi; the lo part uses the other) 64 KB
  static constexpr uint32_t corr = p + 2 * kTile;           // [128] per-row rescale factors
  static constexpr uint32_t xch = corr + 128 * 4;           // [2 parities][2 key halves][128] bf16 row maxima
  static constexpr uint32_t bars = xch + 2 * 2 * 128 * 2;
  // the epilogue's row sums [2 halves][128] l, [2][128] l exact live in the
  // P region (idle once O is complete)
  static constexpr uint32_t total = bars + 20 * 8;
};
static_assert(Smem::total + 1024 <= 232448, "dense attention shared memory");

struct Params {
  int64_t n, start;
  int hq, hkv, out_f32;
  int64_t items;          // (n / 8 rounded up) x hkv
  void* out;
  float* lse;
};

// item w -> (first row i0, group): heaviest (latest rows) first
__device__ __forceinline__ void item_of(const Params& p, int64_t w, int64_t* i0, int* grp) {
  const int64_t nblk = (p.n + kQR - 1) / kQR;
  const int64_t b = nblk - 1 - w / p.hkv;
  *grp = (int)(w % p.hkv);
  *i0 = b * kQR;
}

__global__ void __launch_bounds__(kThreads, 1)
dense_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;      // [2]
  uint64_t* kv_empty = bars + 4;     // [2]
  uint64_t* s_full = bars + 6;       // [kSSlots <= 3]
  uint64_t* s_empty = bars + 9;      // [kSSlots <= 3]
  uint64_t* p_full = bars + 12;      // [2]
  uint64_t* p_empty = bars + 14;     // [2]
  uint64_t* o_full = bars + 16;
  uint64_t* o_empty = bars + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);
  float* corr = reinterpret_cast<float*>(smem + Smem::corr);
  __nv_bfloat16* xch = reinterpret_cast<__nv_bfloat16*>(smem + Smem::xch);
  float* st_l = reinterpret_cast<float*>(smem + Smem::p);          // [2][128], then l exact [2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
      mbar_init(p_full + i, 8);
      mbar_init(p_empty + i, 1);
    }
    for (int i = 0; i < kSSlots; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 8);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 8);
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kColO = kSSlots * 128;     // S slots at [0, kColO), O^T at [kColO, kColO + 128)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x, ++it) {
        int64_t i0;
        int grp;
        item_of(p, w, &i0, &grp);
        const int64_t last = i0 + kQR - 1 < p.n - 1 ? i0 + kQR - 1 : p.n - 1;
        const int tiles = (int)((p.start + last) / kKT) + 1;
        mbar_wait(q_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, kTile);
        uint8_t* qd = smem + Smem::q;
        tma_load_3d(qd, &tm_q, q_full, 0, grp * kG, (int)i0);
        tma_load_3d(qd + kHalf, &tm_q, q_full, 64, grp * kG, (int)i0);
        for (int t = 0; t < tiles; ++t) {
          mbar_wait(kv_empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(kv_full + stage, 2 * kTile);
          uint8_t* kd = smem + Smem::kv + stage * 2 * kTile;
          uint8_t* vd = kd + kTile;
          tma_load_3d(kd, &tm_k, kv_full + stage, 0, t * kKT, grp);
          tma_load_3d(kd + kHalf, &tm_k, kv_full + stage, 64, t * kKT, grp);
          tma_load_3d(vd, &tm_v, kv_full + stage, 0, t * kKT, grp);
          tma_load_3d(vd + kHalf, &tm_v, kv_full + stage, 64, t * kKT, grp);
          if (++stage == 2) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // QK(t) is issued before PV(t-1), so tile t's scores are computed while
    // the softmax works on tile t-1.
    const uint32_t idesc_qk = idesc_bf16_f32(128, 128);
    const uint32_t idesc_pv = idesc_bf16_f32_major(128, 128, 1, 0);   // A = V^T (MN-major), B = P (K-major)
    const uint64_t dq = sdesc_k_sw128(smem_u32(smem + Smem::q));
    int stage = 0;
    uint32_t phase = 0;
    uint32_t tcount = 0;       // tiles issued (S slot = tcount % kSSlots)
    uint32_t pcount = 0;       // PV tiles issued (P buffer = pcount & 1)
    int it = 0;
    for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x, ++it) {
      int64_t i0;
      int grp;
      item_of(p, w, &i0, &grp);
      const int64_t last = i0 + kQR - 1 < p.n - 1 ? i0 + kQR - 1 : p.n - 1;
      const int tiles = (int)((p.start + last) / kKT) + 1;
      const bool split = p.start + i0 < kSplitBelow;
      mbar_wait(q_full, it & 1);
      int pv_stage = stage;
      uint32_t pv_phase = phase;
      auto issue_pv = [&](int t) {
        const int pb = split ? 0 : (int)(pcount & 1);
        mbar_wait(p_full + (pcount & 1), (pcount >> 1) & 1);
        if (t == 0) mbar_wait(o_empty, (it & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint8_t* vd = smem + Smem::kv + pv_stage * 2 * kTile + kTile;
          const uint64_t dv = sdesc_mn_sw128(smem_u32(vd), kHalf, 1024);
          const uint64_t dp = sdesc_k_sw128(smem_u32(smem + Smem::p + pb * kTile));
          const uint64_t dpl = sdesc_k_sw128(smem_u32(smem + Smem::p + kTile));   // lo part (split items)
#pragma unroll
          for (int k = 0; k < kKT / 16; ++k) {
            const uint32_t poff = (k >> 2) * kHalf + (k & 3) * 32;
            umma_f16_ss(tmem + kColO, dv + (k * 2048 >> 4), dp + (poff >> 4), idesc_pv, (t > 0 || k > 0) ? 1u : 0u);
            if (split) umma_f16_ss(tmem + kColO, dv + (k * 2048 >> 4), dpl + (poff >> 4), idesc_pv, 1u);
          }
          umma_commit(kv_empty + pv_stage);        // K (used by QK(t) earlier) and V of this stage
          umma_commit(p_empty + (pcount & 1));
          if (t == tiles - 1) umma_commit(o_full);
        }
        __syncwarp();
        ++pcount;
        if (++pv_stage == 2) { pv_stage = 0; pv_phase ^= 1; }
      };
      for (int t = 0; t < tiles; ++t, ++tcount) {
        const int slot = tcount % kSSlots;
        mbar_wait(kv_full + stage, phase);
        mbar_wait(s_empty + slot, ((tcount / kSSlots) & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dk = sdesc_k_sw128(smem_u32(smem + Smem::kv + stage * 2 * kTile));
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
            umma_f16_ss(tmem + slot * 128, dq + (off >> 4), dk + (off >> 4), idesc_qk, k > 0 ? 1u : 0u);
          }
          umma_commit(s_full + slot);
          if (t == tiles - 1) umma_commit(q_empty);
        }
        __syncwarp();
        if (++stage == 2) { stage = 0; phase ^= 1; }
        if (t > 0) issue_pv(t - 1);
      }
      issue_pv(tiles - 1);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int quad = warp & 3;
    const int hf = (warp - 4) >> 2;                   // key half of every tile
    const int r = quad * 32 + lane;                   // S row (q, h) == O^T lane d
    const int qr = r >> 4, h = r & 15;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const float c2 = 1.4426950408889634f / sqrtf((float)kD);
    uint32_t tcount = 0, pcount = 0;
    uint32_t p_ph[2] = {0, 0};
    int it = 0;
    for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x, ++it) {
      int64_t i0;
      int grp;
      item_of(p, w, &i0, &grp);
      const int64_t last = i0 + kQR - 1 < p.n - 1 ? i0 + kQR - 1 : p.n - 1;
      const int tiles = (int)((p.start + last) / kKT) + 1;
      const bool split = p.start + i0 < kSplitBelow;
      const int64_t row_i = i0 + qr;                    // query row of this thread
      const bool row_ok = row_i < p.n;
      const int64_t pos = p.start + (row_ok ? row_i : last);
      float mrun = -INFINITY, lsum = 0.f, lsx = 0.f;
      for (int t = 0; t < tiles; ++t, ++tcount, ++pcount) {
        const int slot = tcount % kSSlots;
        mbar_wait(s_full + slot, (tcount / kSSlots) & 1);
        tc_fence_after();
        const int64_t key0 = (int64_t)t * kKT;
        // keys <= pos in this tile, counted from this half's first key
        const int nvalid = (int)(pos - key0 + 1 < kKT ? pos - key0 + 1 : kKT) - hf * 64;
        const uint32_t scol = tmem + lane_base + slot * 128 + hf * 64;
        // both halves take the max over the whole row (identical values, no
        // exchange); the barrier ORs the rescale vote: exact max on the first
        // tile, later a rescale only when some row's score exceeds its max by 8
        // (tiles wholly below the item's first row need no causal mask: the
        // max is taken on the raw scores, then scaled, c2 > 0)
        const bool full = key0 + kKT - 1 <= p.start + i0;
        float tmax = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < 64; c += 32) {
          float z[32];
          tmem_ld32(scol + c, z);
          tmem_wait_ld();
          if (full) {
#pragma unroll
            for (int x = 0; x < 32; x += 2) tmax = fmax3(tmax, z[x], z[x + 1]);
          } else {
#pragma unroll
            for (int x = 0; x < 32; ++x) tmax = fmaxf(tmax, c + x < nvalid ? z[x] : -INFINITY);
          }
        }
        // row max of both halves through smem, rounded UP to bf16 on both
        // sides (the two threads of a row then hold the same M >= the true
        // max; M only needs to bound the scores, the LSE and O are exact for
        // any M); slots double-buffered by tile parity: a slot is rewritten
        // only after every reader passed the next tile's barrier
        __nv_bfloat16* xb = xch + (tcount & 1) * 256;
        const __nv_bfloat16 mine = __float2bfloat16_ru(tmax * c2);
        xb[hf * 128 + r] = mine;
        tmax = __bfloat162float(mine);
        const bool over_own = tmax > mrun + 8.f;
        const bool need = named_bar_or(1, 256, t == 0 || over_own);
        tmax = fmaxf(tmax, __bfloat162float(xb[(hf ^ 1) * 128 + r]));
        if (need) {
          const float mnew = fmaxf(mrun, tmax);
          const float cf = mrun == -INFINITY ? 1.f : ex2(mrun - mnew);
          lsum *= mrun == -INFINITY ? 0.f : cf;
          lsx *= mrun == -INFINITY ? 0.f : cf;
          mrun = mnew;
          if (t > 0) {
            if (hf == 0) corr[r] = cf;
            // O^T holds PV(t-1) once p_empty of its buffer completes again
            const int pb = (int)((pcount - 1) & 1);
            mbar_wait(p_empty + pb, p_ph[pb] ^ 1);
            named_bar_sync(1, 256);
            tc_fence_after();
            // this thread's O^T lane over its half of the (q,h) columns
#pragma unroll 1
            for (int c = hf * 64; c < hf * 64 + 64; c += 32) {
              float o[32];
              tmem_ld32(tmem + lane_base + kColO + c, o);
              tmem_wait_ld();
#pragma unroll
              for (int x = 0; x < 32; ++x) o[x] *= corr[c + x];
              tmem_st16(tmem + lane_base + kColO + c, *reinterpret_cast<float(*)[16]>(o));
              tmem_st16(tmem + lane_base + kColO + c + 16, *reinterpret_cast<float(*)[16]>(o + 16));
            }
            tmem_wait_st();
            tc_fence_before();
          }
        }
        // P = 2^(z - M) as bf16 (hi; lo into the second buffer for split items),
        // K-major with the 128-B swizzle: 16-byte chunk c of row r at c ^ (r & 7);
        // key half hf is swizzle half hf of the tile
        const int pb = split ? 0 : (int)(pcount & 1);
        mbar_wait(p_empty + (pcount & 1), p_ph[pcount & 1] ^ 1);   // PV(tile - 2) done
        p_ph[pcount & 1] ^= 1;
        if (split && pcount > 0) {
          // split items use both buffers every tile: PV(tile - 1) must be done
          // too (the next completion of its p_empty; no other can intervene)
          const int ob = (int)((pcount - 1) & 1);
          mbar_wait(p_empty + ob, p_ph[ob] ^ 1);
        }
        uint8_t* ph = smem + Smem::p + pb * kTile + hf * kHalf;
        uint8_t* pl = smem + Smem::p + kTile + hf * kHalf;
        // one body per (split, masked) combination: packed fp32 pairs for the
        // scale (FFMA2) and the row sums (FADD2)
        uint64_t lsum2 = 0, lsx2 = 0;
        const uint64_t c2x2 = pk2(c2, c2), nm2 = pk2(-mrun, -mrun), neg1 = pk2(-1.f, -1.f);
        auto emit = [&](auto split_c, auto masked_c) {
          constexpr bool kSplit = decltype(split_c)::value, kMasked = decltype(masked_c)::value;
#pragma unroll 1
          for (int c = 0; c < 64; c += 32) {
            float z[32];
            tmem_ld32(scol + c, z);
            tmem_wait_ld();
#pragma unroll
            for (int c8 = 0; c8 < 4; ++c8) {
              uint32_t hw[4], lw[4];
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                float xa, xb;
                upk2(ffma2(pk2(z[c8 * 8 + e], z[c8 * 8 + e + 1]), c2x2, nm2), xa, xb);
                float a = ex2(xa), b = ex2(xb);
                if constexpr (kMasked) {
                  const int k0 = c + c8 * 8 + e;
                  a = k0 < nvalid ? a : 0.f;
                  b = k0 + 1 < nvalid ? b : 0.f;
                }
                const __nv_bfloat162 hi2 = __floats2bfloat162_rn(a, b);
                const uint32_t hb = *reinterpret_cast<const uint32_t*>(&hi2);
                const uint64_t ab = pk2(a, b);
                const uint64_t hf2 = pk2(__uint_as_float(hb << 16), __uint_as_float(hb & 0xffff0000u));
                lsx2 = fadd2(lsx2, ab);
                hw[e / 2] = hb;
                if constexpr (kSplit) {
                  float la, lb;
                  upk2(ffma2(hf2, neg1, ab), la, lb);       // a - hi(a), exact
                  const __nv_bfloat162 lo2 = __floats2bfloat162_rn(la, lb);
                  lw[e / 2] = *reinterpret_cast<const uint32_t*>(&lo2);
                  lsum2 = fadd2(lsum2, ab);
                } else {
                  lsum2 = fadd2(lsum2, hf2);
                }
              }
              const int chunk = (c >> 3) + c8;               // 16-byte chunk within the half (0..7)
              const uint32_t off = r * 128 + ((chunk ^ (r & 7)) * 16);
              *reinterpret_cast<uint4*>(ph + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
              if constexpr (kSplit) *reinterpret_cast<uint4*>(pl + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
          }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        if (split) {
          if (full) emit(T_{}, F_{}); else emit(T_{}, T_{});
        } else {
          if (full) emit(F_{}, F_{}); else emit(F_{}, T_{});
        }
        {
          float s0, s1, x0, x1;
          upk2(lsum2, s0, s1);
          upk2(lsx2, x0, x1);
          lsum += s0 + s1;
          lsx += x0 + x1;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + slot);       // S slot read for the last time
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full + (pcount & 1));
      }
      // ---- epilogue: thread = O^T lane d over its half of the (q,h) columns;
      // row sums of both key halves via smem (the P region: every PV is done)
      mbar_wait(o_full, it & 1);
      st_l[hf * 128 + r] = lsum;
      st_l[256 + hf * 128 + r] = lsx;
      named_bar_sync(1, 256);
      tc_fence_after();
      const int d = r;
#pragma unroll 1
      for (int c = hf * 64; c < hf * 64 + 64; c += 32) {
        float o[32];
        tmem_ld32(tmem + lane_base + kColO + c, o);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < 32; ++x) {
          const int col = c + x;                         // (q, h) column
          const int64_t ri = i0 + (col >> 4);
          if (ri < p.n) {
            const float v = o[x] / (st_l[col] + st_l[128 + col]);
            const int64_t idx = (ri * p.hq + (int64_t)grp * kG + (col & 15)) * kD + d;
            if (p.out_f32) static_cast<float*>(p.out)[idx] = v;
            else static_cast<__nv_bfloat16*>(p.out)[idx] = __float2bfloat16_rn(v);
          }
        }
      }
      if (p.lse && row_ok && hf == 0)
        p.lse[row_i * p.hq + grp * kG + h] = (mrun + log2f(st_l[256 + r] + st_l[384 + r])) * 0.6931471805599453f;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

bool dense_tc_supported(const CallShape& cs) {
  return tc_kernels_enabled() && cs.group == kG && cs.d == kD && cs.n > 0 && !cs.bcast;
}

cudaError_t launch_dense_tc(const CallShape& cs, const void* q, int64_t q_row_stride, const void* k_cache,
                            const void* v_cache, int64_t cap, void* out, int out_f32, float* lse,
                            cudaStream_t stream) {
  Params p;
  p.n = cs.n;
  p.start = cs.start;
  p.hq = cs.hq;
  p.hkv = cs.hkv;
  p.out_f32 = out_f32;
  p.items = (cs.n + kQR - 1) / kQR * cs.hkv;
  p.out = out;
  p.lse = lse;
  CUtensorMap tq, tk, tv;
  {
    const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)cs.hq, (uint64_t)cs.n};
    const uint64_t strides[2] = {(uint64_t)kD * 2, (uint64_t)q_row_stride * 2};
    const uint32_t box[3] = {64, (uint32_t)kG, (uint32_t)kQR};
    if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)cap, (uint64_t)cs.hkv};
    const uint64_t strides[2] = {(uint64_t)kD * 2, (uint64_t)cap * kD * 2};
    const uint32_t box[3] = {64, (uint32_t)kKT, 1};
    if (!encode_tmap_3d_bf16(&tk, k_cache, dims, strides, box)) return cudaErrorInvalidValue;
    if (!encode_tmap_3d_bf16(&tv, v_cache, dims, strides, box)) return cudaErrorInvalidValue;
  }
  const size_t smem = Smem::total + 1024;
  {
    cudaError_t e = smem_attr_once((const void*)dense_tc_kernel, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(p.items < sms ? p.items : sms);
  count_launch();
  dense_tc_kernel<<<grid, kThreads, smem, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace infllm2
