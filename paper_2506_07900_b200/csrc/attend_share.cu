// Stage-2 block-sparse attention with the forced blocks shared across query
// rows (tcgen05 + TMEM + TMA), for prefill rows at positions >= 2048 of the
// production geometries (G = 16, D = 128 and G = 8, D = 64; m = 64, one init
// block, two local blocks: the MiniCPM4 defaults), every top-k up to 80
// selected blocks.  (The description below uses the 8B numbers; the 0.5B shape
// runs U = 8 rows per unit with the same N = 64 shared tiles.)
//
// attend_tc.cu gathers every selected block once per (row, KV group) item and
// is bound by shared-memory traffic: each 128-key tile moves 64 KB by TMA and
// 64 KB through the tensor-core operand reads for only 16 heads (DESIGN §4
// K3p).  The three forced blocks of a row (init block 0, local blocks qb-1 and
// qb, force_blocks, sparse.py:218-227) are the same for every row of a 64-row
// query block, so here a work unit is U = 4 consecutive rows of one query
// block and one KV group:
//
//   shared tile A = blocks (0, qb-1), shared tile B = block qb (half tile):
//     S^T[128 keys x 64] = K . [Q_0 .. Q_3]^T          (N = 16 U, one MMA chain)
//     softmax per row over A and B together (exact max of the shared keys,
//     the causal mask of block qb per row, sparse.py:370-372)
//     O^T[128 d x 64] += V^T . P^T                     (N = 16 U)
//   then each row's chosen blocks (its selection minus the forced ones, in
//   ascending order) in 128-key tiles with N = 16, online softmax continuing
//   from the shared pass, exactly as attend_tc.cu.
//
// Per row that is 8 chosen tiles + 1.5 / U shared tiles instead of 9.5 tiles:
// ~12 % less shared-memory and L2 traffic per row.  The per-row running state
// of the shared pass (max per head, per-warp partial row sums) is stashed in
// shared memory until the row's own tiles run.  Summation order differs from
// attend_tc.cu (forced keys first), so outputs agree to rounding.
//
// Warp roles (16 warps, as attend_tc.cu): 0 = Q + K TMA, 1 = QK issuer,
// 2..9 = softmax (thread = tile row x 8 heads), 10 = PV issuer, 11..14 =
// epilogue (thread = d lane of O^T), 15 = V TMA.  The producers and the QK
// issuer walk a unit's rows with the row index unrolled: a per-tile search
// over runtime-indexed register arrays kept both TMA warps ~90 % busy
// (-DSHARE_PROF role counters, DESIGN §4 K3s).
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tc_dispatch.cuh"

namespace infllm2 {

namespace {

using namespace sm100;

constexpr int kM = 64;
constexpr int kNS = 64;                       // shared-tile MMA N = U * G (both geometries)
#ifndef SHARE_KST
#define SHARE_KST 2
#endif
#ifndef SHARE_SLOTS
#define SHARE_SLOTS 6
#endif
constexpr int kSlots = SHARE_SLOTS;           // row-tile S^T slots (G columns each, <= 8)
static_assert(kSlots <= 8, "S^T slots: TMEM columns [0, 128) and 8 barrier pairs");
constexpr int kSoftWarps = 8;
constexpr int kPvWarp = 2 + kSoftWarps;       // 10
constexpr int kVWarp = kPvWarp + 5;           // 15
constexpr int kThreads = 32 * (kVWarp + 1);   // 512
#ifdef SHARE_PROF
// per-role wait cycles (variant builds: tools/build_variant.sh ... -DSHARE_PROF; tools/share_prof.py):
// [0] K producer total, [1] its ring waits, [2] V producer total, [3] its ring waits, [4] QK total,
// [5] QK k_full, [6] QK s_empty, [7] PV total, [8] PV v_full, [9] PV p_full, [10] PV o_empty,
// [11] softmax (warp 2) total, [12] s_full, [13] p_empty, [14] epilogue (warp 11) total, [15] o_full
__device__ long long g_sp[160][16];
#define SP_INIT()                                  \
  long long sp_acc[16];                            \
  for (int i_ = 0; i_ < 16; ++i_) sp_acc[i_] = 0;  \
  const long long sp_t0 = clock64()
#define SP_W(slot, call) do { const long long t_ = clock64(); call; sp_acc[slot] += clock64() - t_; } while (0)
#define SP_FLUSH()                                                                                       \
  do {                                                                                                   \
    const int tot_ = warp == 0 ? 0 : warp == kVWarp ? 2 : warp == 1 ? 4 : warp == kPvWarp ? 7 :          \
                     warp == 2 ? 11 : warp == 11 ? 14 : -1;                                              \
    if (tot_ >= 0) sp_acc[tot_] = clock64() - sp_t0;                                                     \
    if (lane == 0 && blockIdx.x < 160 && tot_ >= 0)                                                      \
      for (int i_ = 0; i_ < 16; ++i_)                                                                    \
        if (sp_acc[i_]) atomicAdd(reinterpret_cast<unsigned long long*>(&g_sp[blockIdx.x][i_]),         \
                                  (unsigned long long)sp_acc[i_]);                                       \
  } while (0)
#else
#define SP_INIT()
#define SP_W(slot, call) call
#define SP_FLUSH()
#endif
constexpr int kMaxSel = 80;
constexpr int64_t kShareFrom = 2048;          // first position on this kernel
constexpr uint32_t kHalf = 128 * 128;         // 16 KB: 128 rows x 64 d (bf16)

// TMEM columns: row S^T slots [0, G kSlots), shared S^T A [128, 192), B [192, 256),
// O^T double buffer [256, 512): buffer b = [256 + 128 b, +128), O_a(u) at +G u,
// O_b(u) at +64 + G u (even / odd K-steps, summed by the epilogue).
constexpr uint32_t kColSA = 128;
constexpr uint32_t kColSB = kColSA + kNS;
constexpr uint32_t kColO = 256;

// Per-geometry constants: (G, D) = (16, 128) MiniCPM4-8B, (8, 64) MiniCPM4-0.5B.
// U = 64 / G rows per unit keep the shared tiles at N = 64.
template <int G, int D>
struct SC {
  static constexpr int kG = G, kD = D;
  static constexpr int kU = kNS / G;                             // 4 / 8
  static constexpr int kDH = D / 64;                             // 64-d halves per row
  static constexpr int kSH = G / 2;                              // heads per softmax thread (two head halves)
  static constexpr uint32_t kTile = kDH * kHalf;                 // K or V tile (128 rows)
  // ring: 8B 2 + 3 stages of 32 KB; 0.5B 4 + 6 of 16 KB (+ a 16 KB pad: PV runs
  // M = 128 over a half-width V tile, its operand spans kHalf past the ring)
  static constexpr int kKSt = D == 128 ? SHARE_KST : 4;
  static constexpr int kVSt = D == 128 ? 5 - SHARE_KST : 6;
  static constexpr uint32_t kPad = D == 64 ? kHalf : 0;
  static constexpr uint32_t kQHalf = kNS * 128;                  // 8 KB: U x G rows x 64 d
  static constexpr uint32_t kQB = kDH * kQHalf;
  static constexpr uint32_t kPRow = 128 * G * 2;                 // P^T of a row tile (128 keys x G)
  static constexpr uint32_t kPSh = 128 * kNS * 2;                // 16 KB: P^T of shared tile A
  static constexpr uint32_t kPB = 64 * kNS * 2;                  // 8 KB: P^T of shared tile B (64 keys)
  static constexpr bool kPBAlias = 2 * kPRow == kPB;             // 8B: B aliases the two row buffers
  struct Smem {
    static constexpr uint32_t kv = 0;                                 // K ring, then V ring (+ pad)
    static constexpr uint32_t q = kv + (kKSt + kVSt) * kTile + kPad;  // [2] Q buffers
    static constexpr uint32_t prow = q + 2 * kQB;                     // [2] row P^T
    static constexpr uint32_t pb = kPBAlias ? prow : prow + 2 * kPRow;
    static constexpr uint32_t psh = pb + (kPBAlias ? 2 * kPRow : kPB);
    static constexpr uint32_t stats = psh + kPSh;                     // [2] x 9 x 16 floats (as attend_tc.cu)
    static constexpr uint32_t red = stats + 2 * 9 * 16 * 4;           // [8 warps][16]
    // per row u of the unit: m[G] (shared-pass max per head), then per softmax
    // warp kSH heads x (rounded row sum, exact row sum) of the shared pass
    static constexpr uint32_t stash_row = G + 2 * kSoftWarps * kSH;   // floats
    static constexpr uint32_t stash = red + kSoftWarps * 16 * 4;
    static constexpr uint32_t bars = (stash + kU * stash_row * 4 + 7) / 8 * 8;
    static constexpr uint32_t total = bars + 96 * 8;
  };
  static_assert(Smem::total + 1024 <= 232448, "attend_share shared memory");
};

struct Params {
  int64_t n, start;          // rows [start, start + n): start % U == 0, n % U == 0, start >= kShareFrom
  int hq, hkv, max_sel, out_f32;
  const int32_t* sel;
  void* out;
  float* lse;
  int64_t units;             // hkv * n / U, group-major
};

// The unit's selection rows: lane-parallel entries (lane, lane+32, lane+64) of
// each of the U rows, and each row's chosen-block count.  A row's selection is
// [0, chosen (ascending, all in [1, qb-1)), qb-1, qb] (force_blocks +
// select_topk with n_init = 1, n_local = 2), so chosen entry j is index 1 + j.
template <int kU>
struct UnitRows {
  int r[kU][3];
  int nch[kU];
  // register arrays indexed by a runtime row: selects, not local memory
  __device__ __forceinline__ int pick(int u, int x) const {
    int v = r[0][x];
#pragma unroll
    for (int k = 1; k < kU; ++k) v = u == k ? r[k][x] : v;
    return v;
  }
  __device__ __forceinline__ int nchosen(int u) const {
    int v = nch[0];
#pragma unroll
    for (int k = 1; k < kU; ++k) v = u == k ? nch[k] : v;
    return v;
  }
  __device__ __forceinline__ int get(int u, int j) const {
    const int v = j < 32 ? pick(u, 0) : (j < 64 ? pick(u, 1) : pick(u, 2));
    return __shfl_sync(0xffffffffu, v, j & 31);
  }
  __device__ __forceinline__ int chosen(int u, int j) const { return get(u, 1 + (j < 94 ? j : 94)); }
  __device__ __forceinline__ int tiles(int u) const { return (nchosen(u) + 1) >> 1; }
};

template <int kU>
__device__ __forceinline__ void unit_of(const Params& p, int64_t w, int* grp, int64_t* i0) {
  const int64_t per = p.n / kU;
  *grp = (int)(w / per);
  *i0 = (w - (int64_t)(*grp) * per) * kU;
}

template <int kU>
__device__ __forceinline__ UnitRows<kU> load_unit(const Params& p, int64_t w, int lane) {
  int grp;
  int64_t i0;
  unit_of<kU>(p, w, &grp, &i0);
  UnitRows<kU> ur;
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int32_t* s = p.sel + ((i0 + u) * p.hkv + grp) * p.max_sel;
    ur.r[u][0] = lane < p.max_sel ? s[lane] : -1;
    ur.r[u][1] = lane + 32 < p.max_sel ? s[lane + 32] : -1;
    ur.r[u][2] = lane + 64 < p.max_sel ? s[lane + 64] : -1;
    const int64_t pos = p.start + i0 + u;
    auto ok = [&](int b) { return b >= 0 && (int64_t)b * kM <= pos; };
    const int nb = __popc(__ballot_sync(0xffffffffu, ok(ur.r[u][0]))) +
                   __popc(__ballot_sync(0xffffffffu, ok(ur.r[u][1]))) +
                   __popc(__ballot_sync(0xffffffffu, ok(ur.r[u][2])));
    ur.nch[u] = nb - 3;
  }
  return ur;
}

template <int G, int D>
__global__ void __launch_bounds__(kThreads, 1)
attend_share_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = SC<G, D>;
  using Smem = typename C::Smem;
  constexpr int kG = G, kD = D, kU = C::kU, kDH = C::kDH, kSH = C::kSH;
  constexpr int kKSt = C::kKSt, kVSt = C::kVSt;
  constexpr uint32_t kTile = C::kTile, kQHalf = C::kQHalf, kQB = C::kQB, kPRow = C::kPRow;
  using URows = UnitRows<kU>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* v_full = bars + 0;      // [kVSt <= 8]
  uint64_t* v_empty = bars + 8;     // [kVSt <= 8]
  uint64_t* k_full = bars + 16;     // [kKSt <= 8]
  uint64_t* k_empty = bars + 24;    // [kKSt <= 8]
  uint64_t* q_full = bars + 32;     // [2]
  uint64_t* q_empty = bars + 34;    // [2]
  uint64_t* s_full = bars + 36;     // [kSlots <= 8]
  uint64_t* s_empty = bars + 44;    // [kSlots <= 8]
  uint64_t* p_full = bars + 52;     // [2]
  uint64_t* p_empty = bars + 54;    // [2]
  uint64_t* st_full = bars + 56;    // [2]
  uint64_t* st_empty = bars + 58;   // [2]
  uint64_t* o_empty = bars + 60;    // [2]
  uint64_t* ssh_full = bars + 62;   // shared S^T A and B written
  uint64_t* ssh_empty = bars + 63;  // shared S^T read by the softmax
  uint64_t* psh_full = bars + 64;   // shared P^T (A and B) written
  uint64_t* psh_empty = bars + 65;  // PV of tile A done with P^T A
  uint64_t* pb_empty = bars + 66;   // PV of tile B done with P^T B (0.5B: its own buffer)
  uint64_t* osh_done = bars + 67;   // shared PVs done (O of the unit initialised)
  // O of row u in buffer b is complete: one barrier per (buffer, row), so the
  // PV issuer (gated per buffer by o_empty) is never two phases ahead of the
  // epilogue on any of them
  uint64_t* o_full = bars + 68;     // [2][kU <= 8]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 84);
  float* stats = reinterpret_cast<float*>(smem + Smem::stats);
  float* red = reinterpret_cast<float*>(smem + Smem::red);
  float* stash = reinterpret_cast<float*>(smem + Smem::stash);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kKSt; ++i) { mbar_init(k_full + i, 1); mbar_init(k_empty + i, 1); }
    for (int i = 0; i < kVSt; ++i) { mbar_init(v_full + i, 1); mbar_init(v_empty + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
      mbar_init(p_full + i, kSoftWarps);
      mbar_init(p_empty + i, 1);
      mbar_init(st_full + i, kSoftWarps);
      mbar_init(st_empty + i, 4);
      mbar_init(o_empty + i, 4);
    }
    for (int i = 0; i < kSlots; ++i) { mbar_init(s_full + i, 1); mbar_init(s_empty + i, kSoftWarps); }
    for (int i = 0; i < 2 * kU; ++i) mbar_init(o_full + i, 1);
    mbar_init(ssh_full, 1);
    mbar_init(ssh_empty, kSoftWarps);
    mbar_init(psh_full, kSoftWarps);
    mbar_init(psh_empty, 1);
    mbar_init(pb_empty, 1);
    mbar_init(osh_done, 1);
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
  SP_INIT();

  if (warp == 0 || warp == kVWarp) {
    // ------------------------------------------------------------ producers
    const bool is_k = warp == 0;
    uint64_t* ring_full = is_k ? k_full : v_full;
    uint64_t* ring_empty = is_k ? k_empty : v_empty;
    uint8_t* ring = smem + Smem::kv + (is_k ? 0 : kKSt * kTile);
    const int nst = is_k ? kKSt : kVSt;
    const CUtensorMap* mm = is_k ? &tm_k : &tm_v;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int64_t w = blockIdx.x; w < p.units; w += gridDim.x, ++it) {
      int grp;
      int64_t i0;
      unit_of<kU>(p, w, &grp, &i0);
      const URows ur = load_unit<kU>(p, w, lane);
      const int64_t qb = (p.start + i0) / kM;
      if (is_k && lane == 0) {
        const int qbuf = it & 1;
        mbar_wait(q_empty + qbuf, ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(q_full + qbuf, kQB);
        uint8_t* qd = smem + Smem::q + qbuf * kQB;
#pragma unroll
        for (int hh = 0; hh < kDH; ++hh)
          tma_load_3d_hint(qd + hh * kQHalf, &tm_q, q_full + qbuf, 64 * hh, grp * kG, (int)i0, pol_stream);
      }
      auto issue = [&](int b0, int b1, int nt) {
        if (lane == 0) {
          SP_W(is_k ? 1 : 3, mbar_wait(ring_empty + stage, phase ^ 1));
          mbar_arrive_expect_tx(ring_full + stage, nt * kDH * (kM * 128));
          uint8_t* dst = ring + stage * kTile;
          for (int x = 0; x < nt; ++x) {
            const int row0 = (x ? b1 : b0) * kM;
            const uint32_t off = x * kM * 128;
#pragma unroll
            for (int hh = 0; hh < kDH; ++hh)
              tma_load_3d_hint(dst + hh * kHalf + off, mm, ring_full + stage, 64 * hh, row0, grp, pol_keep);
          }
        }
        __syncwarp();
        if (++stage == nst) { stage = 0; phase ^= 1; }
      };
      issue(0, (int)qb - 1, 2);           // shared tile A
      issue((int)qb, -1, 1);               // shared tile B
      // the rows' chosen tiles; u unrolled so the unit's registers are
      // addressed directly (no per-tile row search or select chains)
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int nch = ur.nch[u];
        for (int k = 0; 2 * k < nch; ++k) {
          const int nt = 2 * k + 1 < nch ? 2 : 1;
          const int b0 = ur.chosen(u, 2 * k);
          const int b1 = ur.chosen(u, 2 * k + 1);       // shuffled by every lane; unused when nt == 1
          issue(b0, b1, nt);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ QK issuer
    const uint32_t idesc_sh = idesc_bf16_f32(128, kNS);
    const uint32_t idesc_row = idesc_bf16_f32(128, kG);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t tcount = 0;
    int it = 0;
    for (int64_t w = blockIdx.x; w < p.units; w += gridDim.x, ++it) {
      const URows ur = load_unit<kU>(p, w, lane);
      const int qbuf = it & 1;
      mbar_wait(q_full + qbuf, (it >> 1) & 1);
      const uint32_t qa = smem_u32(smem + Smem::q + qbuf * kQB);
      // shared tiles A, B: S^T = K . [Q_0..Q_3]^T (N = 64)
      mbar_wait(ssh_empty, (it & 1) ^ 1);
      for (int x = 0; x < 2; ++x) {
        mbar_wait(k_full + stage, phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t ka = smem_u32(smem + Smem::kv + stage * kTile);
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
            const uint32_t qoff = (k >> 2) * kQHalf + (k & 3) * 32;
            umma_f16_ss(tmem + (x ? kColSB : kColSA), sdesc_k_sw128(ka + off), sdesc_k_sw128(qa + qoff), idesc_sh,
                        k > 0 ? 1u : 0u);
          }
          umma_commit(k_empty + stage);
          if (x == 1) umma_commit(ssh_full);
        }
        __syncwarp();
        if (++stage == kKSt) { stage = 0; phase ^= 1; }
      }
      // row tiles: S^T = K . Q_u^T (N = 16) through the slot ring
#pragma unroll
      for (int u = 0; u < kU; ++u)
      for (int k = 0; k < ur.tiles(u); ++k, ++tcount) {
        const int slot = tcount % kSlots;
        SP_W(5, mbar_wait(k_full + stage, phase));
        SP_W(6, mbar_wait(s_empty + slot, ((tcount / kSlots) & 1) ^ 1));
        tc_fence_after();
        if (elect_one()) {
          const uint32_t ka = smem_u32(smem + Smem::kv + stage * kTile);
#pragma unroll
          for (int k2 = 0; k2 < kD / 16; ++k2) {
            const uint32_t off = (k2 >> 2) * kHalf + (k2 & 3) * 32;
            const uint32_t qoff = (k2 >> 2) * kQHalf + u * (kG * 128) + (k2 & 3) * 32;
            umma_f16_ss(tmem + slot * kG, sdesc_k_sw128(ka + off), sdesc_k_sw128(qa + qoff), idesc_row,
                        k2 > 0 ? 1u : 0u);
          }
          umma_commit(k_empty + stage);
          umma_commit(s_full + slot);
        }
        __syncwarp();
        if (++stage == kKSt) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(q_empty + qbuf);   // every MMA reading this Q buffer is issued
      __syncwarp();
    }
  } else if (warp == kPvWarp) {
    // ------------------------------------------------------------ PV issuer
    const uint32_t idesc_sh = idesc_bf16_f32_major(128, kNS, 1, 1);
    const uint32_t idesc_row = idesc_bf16_f32_major(128, kG, 1, 1);
    int stage = 0;
    uint32_t vphase = 0;
    uint32_t pcount = 0;
    int it = 0;
    for (int64_t w = blockIdx.x; w < p.units; w += gridDim.x, ++it) {
      const URows ur = load_unit<kU>(p, w, lane);
      const int ob = it & 1;
      const uint32_t obase = tmem + kColO + 128 * ob;
      SP_W(10, mbar_wait(o_empty + ob, ((it >> 1) & 1) ^ 1));
      mbar_wait(psh_full, it & 1);
      // shared PVs: O^T[all U rows] = V_A^T . P_A^T + V_B^T . P_B^T (N = 64);
      // even K-steps -> O_a region, odd -> O_b region
      for (int x = 0; x < 2; ++x) {
        mbar_wait(v_full + stage, vphase);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dv = sdesc_mn_sw128(smem_u32(smem + Smem::kv + (kKSt + stage) * kTile), kHalf, 1024);
          const uint64_t dp = sdesc_interleave(smem_u32(smem + (x ? Smem::pb : Smem::psh)), 16 * kNS, 128);
          const int ksteps = x ? 4 : 8;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (k < ksteps)
              umma_f16_ss(obase + (k & 1) * kNS, dv + (k * 2048 >> 4), dp + (k * 32 * kNS >> 4), idesc_sh,
                          (x | (k >> 1)) ? 1u : 0u);
          }
          umma_commit(v_empty + stage);
          if (x == 0) {
            umma_commit(psh_empty);
          } else {
            if (C::kPBAlias) {
              umma_commit(p_empty + 0);    // P^T B occupied both row buffers
              umma_commit(p_empty + 1);
            } else {
              umma_commit(pb_empty);       // P^T B buffer free
            }
            umma_commit(osh_done);
          }
        }
        __syncwarp();
        if (++stage == kVSt) { stage = 0; vphase ^= 1; }
      }
      // row tiles: O_u^T += V^T . P^T (N = 16)
      int c = 0;
      for (int u = 0; u < kU; ++u) {
        const int tiles = ur.tiles(u);
        const int nch = ur.nchosen(u);
        for (int k = 0; k < tiles; ++k, ++c, ++pcount) {
          const int pbuf = pcount & 1;
          SP_W(8, mbar_wait(v_full + stage, vphase));
          SP_W(9, mbar_wait(p_full + pbuf, (pcount >> 1) & 1));
          tc_fence_after();
          const int ksteps = 2 * k + 1 < nch ? 8 : 4;
          if (elect_one()) {
            const uint64_t dv = sdesc_mn_sw128(smem_u32(smem + Smem::kv + (kKSt + stage) * kTile), kHalf, 1024);
            const uint64_t dp = sdesc_interleave(smem_u32(smem + Smem::prow + pbuf * kPRow), 16 * kG, 128);
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) {
              if (k2 < ksteps)
                umma_f16_ss(obase + (k2 & 1) * kNS + u * kG, dv + (k2 * 2048 >> 4), dp + (k2 * 32 * kG >> 4),
                            idesc_row, 1u);
            }
            umma_commit(v_empty + stage);
            umma_commit(p_empty + pbuf);
            if (k == tiles - 1) umma_commit(o_full + ob * kU + u);
          }
          __syncwarp();
          if (++stage == kVSt) { stage = 0; vphase ^= 1; }
        }
        if (tiles == 0 && elect_one()) umma_commit(o_full + ob * kU + u);   // a row without chosen blocks (budget 0)
        __syncwarp();
      }
    }
  } else if (warp < kPvWarp) {
    // ------------------------------------------------------------ softmax
    const int ws = warp - 2;                            // 0..7
    const int quad = warp & 3;
    const int half = ws >> 2;                           // head half: heads h0 .. h0 + 7
    const int h0 = kSH * half;
    const int row = quad * 32 + lane;                   // tile row == TMEM lane
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const float c2 = 1.4426950408889634f / sqrtf((float)kD);
    const uint64_t c2x2 = pk2(c2, c2);
    uint32_t p_ph[2] = {0, 0};
    int pbuf = 0;
    uint32_t tcount = 0;
    uint32_t rcount = 0;                                // rows finished (stats double buffer)
    int it = 0;
    for (int64_t w = blockIdx.x; w < p.units; w += gridDim.x, ++it) {
      int grp;
      int64_t i0;
      unit_of<kU>(p, w, &grp, &i0);
      const URows ur = load_unit<kU>(p, w, lane);
      const int64_t qb = (p.start + i0) / kM;
      // ---- shared pass: rows u = 0..U-1 over tiles A (keys of blocks 0,
      // qb-1: all visible) and B (block qb: key row <= the row's position)
      mbar_wait(ssh_full, it & 1);
      mbar_wait(psh_empty, (it & 1) ^ 1);
      if (C::kPBAlias) {
        // P^T B aliases both row P buffers: their previous PVs must be done
        mbar_wait(p_empty + 0, p_ph[0] ^ 1);
        p_ph[0] ^= 1;
        mbar_wait(p_empty + 1, p_ph[1] ^ 1);
        p_ph[1] ^= 1;
      } else {
        mbar_wait(pb_empty, (it & 1) ^ 1);
      }
      tc_fence_after();
      for (int u = 0; u < kU; ++u) {
        const int64_t pos = p.start + i0 + u;
        float za[kSH], zb[kSH];
        tmem_ld_n<kSH>(tmem + lane_base + kColSA + u * kG + h0, za);
        tmem_ld_n<kSH>(tmem + lane_base + kColSB + u * kG + h0, zb);
        tmem_wait_ld();
        const bool vb = row < kM && qb * kM + row <= pos;
#pragma unroll
        for (int h = 0; h < kSH; h += 2) {
          upk2(ffma2(pk2(za[h], za[h + 1]), c2x2, 0ull), za[h], za[h + 1]);
          upk2(ffma2(pk2(zb[h], zb[h + 1]), c2x2, 0ull), zb[h], zb[h + 1]);
        }
#pragma unroll
        for (int h = 0; h < kSH; ++h) zb[h] = vb ? zb[h] : -INFINITY;
        float mx[kSH];
#pragma unroll
        for (int h = 0; h < kSH; ++h) mx[h] = fmaxf(za[h], zb[h]);
        {
          const float v = warp_reduce_n<kSH>(mx, lane, [](float a, float b) { return fmaxf(a, b); });
          if (reduce_writer_n<kSH>(lane)) red[ws * 16 + reduce_head_n<kSH>(lane)] = v;
        }
        named_bar_sync(2 + half, 128);
        float m[kSH];
        const int hb = 4 * half;
#pragma unroll
        for (int h = 0; h < kSH; ++h)
          m[h] = fmaxf(fmaxf(red[(hb + 0) * 16 + h], red[(hb + 1) * 16 + h]),
                       fmaxf(red[(hb + 2) * 16 + h], red[(hb + 3) * 16 + h]));
        named_bar_sync(2 + half, 128);
        float ls[kSH], lx[kSH];
        uint32_t pa[kSH / 2], pbv[kSH / 2];
#pragma unroll
        for (int h = 0; h < kSH; h += 2) {
          float xa, xb, ya, yb;
          upk2(fadd2(pk2(za[h], za[h + 1]), pk2(-m[h], -m[h + 1])), xa, xb);
          upk2(fadd2(pk2(zb[h], zb[h + 1]), pk2(-m[h], -m[h + 1])), ya, yb);
          const float a0 = ex2(xa), a1 = ex2(xb), b0 = ex2(ya), b1 = ex2(yb);
          const __nv_bfloat162 ah = __floats2bfloat162_rn(a0, a1);
          const __nv_bfloat162 bh = __floats2bfloat162_rn(b0, b1);
          pa[h / 2] = *reinterpret_cast<const uint32_t*>(&ah);
          pbv[h / 2] = *reinterpret_cast<const uint32_t*>(&bh);
          // row sums of the ROUNDED weights (what PV multiplies) and of the exact ones (LSE)
          ls[h] = __low2float(ah) + __low2float(bh);
          ls[h + 1] = __high2float(ah) + __high2float(bh);
          lx[h] = a0 + b0;
          lx[h + 1] = a1 + b1;
        }
        // P^T A: 8-key groups 16 * 64 bytes apart, 8-column groups 128 B apart; column = u * 16 + h
        {
          const int col = u * kG + h0;
          const uint32_t base = (row >> 3) * (16 * kNS) + (row & 7) * 16 + 128 * (col >> 3) + 2 * (col & 7);
          if constexpr (kSH == 8) {
            *reinterpret_cast<uint4*>(smem + Smem::psh + base) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
            if (row < kM)
              *reinterpret_cast<uint4*>(smem + Smem::pb + base) = make_uint4(pbv[0], pbv[1], pbv[2], pbv[3]);
          } else {
            *reinterpret_cast<uint2*>(smem + Smem::psh + base) = make_uint2(pa[0], pa[1]);
            if (row < kM) *reinterpret_cast<uint2*>(smem + Smem::pb + base) = make_uint2(pbv[0], pbv[1]);
          }
        }
        // stash: the max per head and this warp's partial row sums
        {
          const float v = warp_reduce_n<kSH>(ls, lane, [](float a, float b) { return a + b; });
          const float vx = warp_reduce_n<kSH>(lx, lane, [](float a, float b) { return a + b; });
          float* su = stash + u * Smem::stash_row;
          if (reduce_writer_n<kSH>(lane)) {
            su[kG + (ws * kSH + reduce_head_n<kSH>(lane)) * 2] = v;
            su[kG + (ws * kSH + reduce_head_n<kSH>(lane)) * 2 + 1] = vx;
          }
          if (quad == 0 && lane < kSH) {
            float mine = m[0];
#pragma unroll
            for (int h = 1; h < kSH; ++h) mine = (lane == h) ? m[h] : mine;
            su[h0 + lane] = mine;
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(ssh_empty);
        mbar_arrive(psh_full);
      }
      named_bar_sync(2 + half, 128);                    // the stash of this head half is complete
      // ---- row pass: each row's chosen tiles, online softmax from the stash
      for (int u = 0; u < kU; ++u) {
        const float* su = stash + u * Smem::stash_row;
        float mrun[kSH], mst[kSH], lsum[kSH], lsx[kSH];
#pragma unroll
        for (int h = 0; h < kSH; ++h) { mst[h] = su[h0 + h]; mrun[h] = mst[h]; lsum[h] = 0.f; lsx[h] = 0.f; }
        const int tiles = ur.tiles(u);
        const int nch = ur.nchosen(u);
        const int ob = it & 1;
        const uint32_t oa = tmem + lane_base + kColO + 128 * ob + u * kG + h0;
        for (int k = 0; k < tiles; ++k) {
          const int sslot = tcount % kSlots;
          SP_W(12, mbar_wait(s_full + sslot, (tcount / kSlots) & 1));
          ++tcount;
          tc_fence_after();
          float z[kSH];
          tmem_ld_n<kSH>(tmem + lane_base + sslot * kG + h0, z);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty + sslot);
          const bool valid = 2 * k + (row >> 6) < nch;   // chosen blocks lie below qb - 1
#pragma unroll
          for (int h = 0; h < kSH; h += 2) upk2(ffma2(pk2(z[h], z[h + 1]), c2x2, 0ull), z[h], z[h + 1]);
#pragma unroll
          for (int h = 0; h < kSH; ++h) z[h] = valid ? z[h] : -INFINITY;
          bool over = false;
#pragma unroll
          for (int h = 0; h < kSH; ++h) over |= z[h] > mrun[h] + 8.f;
          if (named_bar_or(2 + half, 128, over)) {
            {
              float zz[kSH];
#pragma unroll
              for (int h = 0; h < kSH; ++h) zz[h] = z[h];
              const float v = warp_reduce_n<kSH>(zz, lane, [](float a, float b) { return fmaxf(a, b); });
              if (reduce_writer_n<kSH>(lane)) red[ws * 16 + reduce_head_n<kSH>(lane)] = v;
            }
            named_bar_sync(2 + half, 128);
            float corr[kSH];
            bool any = false;
            const int hb = 4 * half;
#pragma unroll
            for (int h = 0; h < kSH; ++h) {
              const float tm = fmaxf(fmaxf(red[(hb + 0) * 16 + h], red[(hb + 1) * 16 + h]),
                                     fmaxf(red[(hb + 2) * 16 + h], red[(hb + 3) * 16 + h]));
              const float mnew = fmaxf(mrun[h], tm);
              corr[h] = ex2(mrun[h] - mnew);
              any |= corr[h] != 1.f;
              lsum[h] *= corr[h];
              lsx[h] *= corr[h];
              mrun[h] = mnew;
            }
            named_bar_sync(2 + half, 128);
            if (any) {
              // O_u holds the shared PVs and this row's earlier tiles: wait for
              // the last of them (the shared pass, or the previous tile's PV)
              if (k == 0) mbar_wait(osh_done, it & 1);
              else mbar_wait(p_empty + (pbuf ^ 1), p_ph[pbuf ^ 1] ^ 1);
              tc_fence_after();
              float o[kSH], o2[kSH];
              tmem_ld_n<kSH>(oa, o);
              tmem_ld_n<kSH>(oa + kNS, o2);
              tmem_wait_ld();
#pragma unroll
              for (int h = 0; h < kSH; ++h) { o[h] *= corr[h]; o2[h] *= corr[h]; }
              tmem_st_n<kSH>(oa, o);
              tmem_st_n<kSH>(oa + kNS, o2);
              tmem_wait_st();
              tc_fence_before();
            }
          }
          SP_W(13, mbar_wait(p_empty + pbuf, p_ph[pbuf] ^ 1));
          p_ph[pbuf] ^= 1;
          uint32_t phi[kSH / 2];
#pragma unroll
          for (int h = 0; h < kSH; h += 2) {
            float xa, xb;
            upk2(fadd2(pk2(z[h], z[h + 1]), pk2(-mrun[h], -mrun[h + 1])), xa, xb);
            const float a = ex2(xa), b = ex2(xb);
            const __nv_bfloat162 hi2 = __floats2bfloat162_rn(a, b);
            phi[h / 2] = *reinterpret_cast<const uint32_t*>(&hi2);
            upk2(fadd2(pk2(lsx[h], lsx[h + 1]), pk2(a, b)), lsx[h], lsx[h + 1]);
            upk2(fadd2(pk2(lsum[h], lsum[h + 1]), pk2(__low2float(hi2), __high2float(hi2))), lsum[h], lsum[h + 1]);
          }
          uint8_t* pb = smem + Smem::prow + pbuf * kPRow;
          const uint32_t base = (row >> 3) * (16 * kG) + (row & 7) * 16 + 128 * (h0 >> 3) + 2 * (h0 & 7);
          if constexpr (kSH == 8) *reinterpret_cast<uint4*>(pb + base) = make_uint4(phi[0], phi[1], phi[2], phi[3]);
          else *reinterpret_cast<uint2*>(pb + base) = make_uint2(phi[0], phi[1]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full + pbuf);
          pbuf ^= 1;
        }
        // ---- row stats: this row's tiles + the stashed shared-pass sums,
        // rescaled from the shared-pass max to the final one
        const int sb = rcount & 1;
        mbar_wait(st_empty + sb, ((rcount >> 1) & 1) ^ 1);
        float* st = stats + sb * 9 * 16;
        {
          const float v = warp_reduce_n<kSH>(lsum, lane, [](float a, float b) { return a + b; });
          const float vx = warp_reduce_n<kSH>(lsx, lane, [](float a, float b) { return a + b; });
          if (reduce_writer_n<kSH>(lane)) {
            const int hl = reduce_head_n<kSH>(lane);
            float ms = mst[0], mf = mrun[0];
#pragma unroll
            for (int h = 1; h < kSH; ++h) {
              ms = (hl == h) ? mst[h] : ms;
              mf = (hl == h) ? mrun[h] : mf;
            }
            const float cf = ex2(ms - mf);
            st[quad * 16 + h0 + hl] = v + su[kG + (ws * kSH + hl) * 2] * cf;
            st[80 + quad * 16 + h0 + hl] = vx + su[kG + (ws * kSH + hl) * 2 + 1] * cf;
          }
        }
        if (quad == 0 && lane < kSH) {
          float mine = mrun[0];
#pragma unroll
          for (int h = 1; h < kSH; ++h) mine = (lane == h) ? mrun[h] : mine;
          st[64 + h0 + lane] = mine;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(st_full + sb);
        ++rcount;
      }
      // the next unit's shared pass rewrites the stash: every warp of this head
      // half has read it (the stats barrier above orders the reads)
      named_bar_sync(2 + half, 128);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;
    const int d = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    uint32_t rcount = 0;
    int it = 0;
    for (int64_t w = blockIdx.x; w < p.units; w += gridDim.x, ++it) {
      int grp;
      int64_t i0;
      unit_of<kU>(p, w, &grp, &i0);
      const int ob = it & 1;
      for (int u = 0; u < kU; ++u, ++rcount) {
        const int sb = rcount & 1;
        SP_W(15, mbar_wait(o_full + ob * kU + u, (it >> 1) & 1));
        mbar_wait(st_full + sb, (rcount >> 1) & 1);
        tc_fence_after();
        float o[kG], o2[kG];
        tmem_ld_n<kG>(tmem + lane_base + kColO + 128 * ob + u * kG, o);
        tmem_ld_n<kG>(tmem + lane_base + kColO + 128 * ob + kNS + u * kG, o2);
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < kG; ++h) o[h] += o2[h];
        const float* st = stats + sb * 9 * 16;
        float l[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) l[h] = st[h] + st[16 + h] + st[32 + h] + st[48 + h];
        const int64_t i = i0 + u;
        const int64_t obase = (i * p.hq + (int64_t)grp * kG) * kD + d;
        if (d >= kD) {
          // O^T lanes >= D (D = 64 runs PV with M = 128 over a half-width V tile): unused
        } else if (p.out_f32) {
          float* out = static_cast<float*>(p.out);
#pragma unroll
          for (int h = 0; h < kG; ++h) st_global_hint(out + obase + h * kD, o[h] / l[h], pol_stream);
        } else {
          __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
#pragma unroll
          for (int h = 0; h < kG; ++h) st_global_hint(out + obase + h * kD, __float2bfloat16_rn(o[h] / l[h]), pol_stream);
        }
        if (p.lse && quad == 0 && lane < kG) {
          const float lx = st[80 + lane] + st[96 + lane] + st[112 + lane] + st[128 + lane];
          p.lse[i * p.hq + grp * kG + lane] = (st[64 + lane] + log2f(lx)) * 0.6931471805599453f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(st_empty + sb);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty + ob);
    }
  }

  tc_fence_before();
  __syncthreads();
  SP_FLUSH();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

// Rows [row0, row1) of a prefill call that the shared-forced-block kernel
// covers: positions >= 2048, U-aligned, MiniCPM4 forced-block layout and head
// geometry (8B: G = 16, D = 128; 0.5B: G = 8, D = 64), plain prefill (no tree
// rows, no broadcast position, no hi + lo weights).
bool attend_share_range(const infllm2_geometry& g, const CallShape& cs, int p_split, bool tree, int64_t* row0,
                        int64_t* row1) {
  static const bool off = [] {
    const char* e = getenv("INFLLM2_ATTEND_SHARE");
    return e && e[0] == '0';
  }();
  if (off || p_split || tree || cs.bcast) return false;
  const bool shape_ok = (cs.group == 16 && cs.d == 128) || (cs.group == 8 && cs.d == 64);
  if (!shape_ok || g.block_size != kM || g.n_init_blocks != 1 || g.n_local_blocks != 2) return false;
  if (cs.max_sel > kMaxSel) return false;
  // a selection of little more than the forced blocks (forced_consume_budget
  // with top-k <= 4) attends too few keys for bf16 weights: attend_tc.cu's
  // hi + lo weights serve it
  if (g.forced_consume_budget && g.top_k <= 4) return false;
  // 0.5B runs here at every top-k since the producer-loop fix (128K stage 2 vs
  // attend_tc: k = 32 15.7 -> 11.4 ms, k = 64 27.4 -> 20.4 ms; before it, k >= 32
  // was neutral or slower and stayed on attend_tc)
  const int u = kNS / cs.group;
  // rows below position 2048 attend at most 32 blocks and carry the largest
  // relative bf16-weight rounding error: they stay on attend_tc.cu (whose
  // rows below 256 use hi + lo weights), so the two kernels share one envelope
  int64_t a = cs.start > kShareFrom ? cs.start : kShareFrom;
  a = (a + u - 1) / u * u;
  const int64_t b = (cs.start + cs.n) / u * u;
  if (b - a < 2 * u * kNumSMs) return false;   // too few units to pay for a second launch
  *row0 = a - cs.start;
  *row1 = b - cs.start;
  return true;
}

template <int G, int D>
static cudaError_t launch_share(const CallShape& cs, int64_t row0, int64_t row1, const void* q, int64_t q_row_stride,
                                const void* k_cache, const void* v_cache, int64_t cap, const int32_t* selection,
                                void* out, int out_f32, float* lse, cudaStream_t stream) {
  using C = SC<G, D>;
  const int64_t n = row1 - row0;
  Params p;
  p.n = n;
  p.start = cs.start + row0;
  p.hq = cs.hq;
  p.hkv = cs.hkv;
  p.max_sel = cs.max_sel;
  p.out_f32 = out_f32;
  p.sel = selection + row0 * cs.hkv * cs.max_sel;
  p.out = static_cast<uint8_t*>(out) + row0 * cs.hq * D * (out_f32 ? 4 : 2);
  p.lse = lse ? lse + row0 * cs.hq : nullptr;
  p.units = cs.hkv * (n / C::kU);
  const __nv_bfloat16* qr = static_cast<const __nv_bfloat16*>(q) + row0 * q_row_stride;
  CUtensorMap tq, tk, tv;
  {
    const uint64_t dims[3] = {(uint64_t)D, (uint64_t)cs.hq, (uint64_t)n};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)q_row_stride * 2};
    const uint32_t box[3] = {64, (uint32_t)G, (uint32_t)C::kU};
    if (!encode_tmap_3d_bf16(&tq, qr, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {(uint64_t)D, (uint64_t)cs.cache_len, (uint64_t)cs.hkv};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)cap * D * 2};
    const uint32_t box[3] = {64, (uint32_t)kM, 1};
    if (!encode_tmap_3d_bf16(&tk, k_cache, dims, strides, box)) return cudaErrorInvalidValue;
    if (!encode_tmap_3d_bf16(&tv, v_cache, dims, strides, box)) return cudaErrorInvalidValue;
  }
  const size_t smem = C::Smem::total + 1024;
  cudaError_t e = smem_attr_once((const void*)attend_share_kernel<G, D>, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(p.units < sms ? p.units : sms);
  count_launch();
  attend_share_kernel<G, D><<<grid, kThreads, smem, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

cudaError_t launch_attend_share(const CallShape& cs, int64_t row0, int64_t row1, const void* q, int64_t q_row_stride,
                                const void* k_cache, const void* v_cache, int64_t cap, const int32_t* selection,
                                void* out, int out_f32, float* lse, cudaStream_t stream) {
  if (cs.group == 8 && cs.d == 64)
    return launch_share<8, 64>(cs, row0, row1, q, q_row_stride, k_cache, v_cache, cap, selection, out, out_f32, lse,
                               stream);
  return launch_share<16, 128>(cs, row0, row1, q, q_row_stride, k_cache, v_cache, cap, selection, out, out_f32, lse,
                               stream);
}

}  // namespace infllm2

#ifdef SHARE_PROF
extern "C" int infllm2_debug_share_cycles(long long* host) {
  return cudaMemcpyFromSymbol(host, infllm2::g_sp, sizeof(long long) * 160 * 16) == cudaSuccess ? 0 : -1;
}
#endif
