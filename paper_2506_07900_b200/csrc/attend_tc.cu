// Stage-2 block-sparse attention on the tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces sparse_attend (sparse.py:347-384) for the production geometry
// (G = 16 heads per KV group, D = 128, m = 64).  One work item is one
// (query row, KV group); its selected blocks (ascending, from stage 1) are
// gathered by TMA two at a time into 128-row K/V tiles:
//
//   S^T[128 rows x 16 heads] = K_tile (128x128, K-major) . Q^T      (TMEM)
//   softmax warps: thread = row; mask rows beyond the query position
//     (causal clip, sparse.py:370-372) and the empty half of a 1-block tile;
//     P = 2^(z - M_h) -> bf16 -> smem (MN-major, no swizzle)
//   O^T[128 d x 16 heads] += V_tile^T (MN-major, 128-B swizzle) . P^T (TMEM)
//
// Every K/V byte feeds only the 16 heads of its group, so the kernel is bound
// by the gather bandwidth (L2 -> SMEM), not by the tensor pipe:
// three 64 KB K/V stages keep ~128 KB in flight per SM.  The running max M_h
// is the exact max of the first tile (which always holds the forced init
// block); later tiles only trigger a rescale of O (TMEM ld/scale/st) when a
// score exceeds M_h + 8 (log2 units), so P stays <= 256 and the rescale is rare.
//
// Warp roles (10 warps): 0 = TMA producer, 1 = TMEM alloc + MMA issuer,
// 2..5 = softmax (128 threads = tile rows), 6..9 = epilogue (thread = d lane
// of O^T: normalise, store bf16/f32 output and the natural-log LSE).
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tc_dispatch.cuh"

namespace infllm2 {

bool tc_kernels_enabled();

namespace {

using namespace sm100;

constexpr int kG = 16;
constexpr int kD = 128;
#ifdef ATT_PROFILE
// per-CTA cycle counters (variant builds only, tools/build_variant.sh -DATT_PROFILE;
// read by tools/attend_profile.py): [0] QK warp total [1] softmax in tile loops
// [2] QK s_empty wait [3] PV warp total [4] PV v_full wait [5] PV p_full wait
// [6] softmax P fence+arrive [7] softmax warp 2 total [8] its s_full wait
// [9] vote barrier [10] need path [11] p_empty wait [12] K TMA k_empty wait
// [13] V TMA v_empty wait [14] K TMA total [15] softmax S TMEM load + wait
__device__ long long g_att_cyc[160][24];
#define ATT_T0(v) long long v = clock64()
#define ATT_ADD(slot, v) (att_acc[slot] += clock64() - (v))   // registers; flushed once at kernel end
#else
#define ATT_T0(v)
#define ATT_ADD(slot, v)
#endif
constexpr int kM = 64;                 // block size
constexpr int kRowsT = 128;            // rows per tile (two blocks)
#ifndef ATT_KSTAGES
#define ATT_KSTAGES 2   // K ring 2 + V ring 4: 12.24 vs 12.34 ms (3 + 3) per 128K layer
#endif
#ifndef ATT_HS
#define ATT_HS 2   // softmax head groups per tile row (8B shape): 2 -> 8 softmax warps, 4 -> 16
#endif
#ifndef ATT_SLOTS
#define ATT_SLOTS 6   // 4 / 5 / 6 measured 12.75 / 12.61 / 12.59 ms per 128K layer
#endif
constexpr int kSlots = ATT_SLOTS;       // S^T slots in TMEM (QK runs up to kSlots tiles ahead of softmax)
static_assert(kSlots <= 6, "(kSlots + 2) * 2 * G TMEM columns must fit the 256-column allocation at G = 16");
#ifndef ATT_QK_SPLIT
#define ATT_QK_SPLIT 0   // 1 measured ~1.5 % slower now that the softmax bounds the kernel
#endif
constexpr bool kQkSplit = ATT_QK_SPLIT;  // S^T as two interleaved accumulators (summed by the softmax)
constexpr int kMaxSel = 80;
// Rows at positions below this attend few keys, where bf16 softmax weights
// would cost up to 2^-9 |v0 - v1| (two keys): they always carry the weights as
// bf16 hi + lo (a second PV MMA per k-step on <= 2 tiles per item); so do rows
// of any position that attend at most kSplitPBlocks blocks (a budget-0
// forced_consume_budget selection: the forced blocks alone)
constexpr int64_t kSplitPBelow = 256;
constexpr int kSplitPBlocks = 4;

constexpr uint32_t kHalfBytes = kRowsT * 128;           // 16 KB: 128 rows x 64 d (bf16)

// Per-geometry constants: G heads per KV group (16 or 8), head dim D (128 or
// 64).  MiniCPM4-8B is (16, 128), MiniCPM4-0.5B (8, 64).  Tiles stay 128 rows;
// a D = 64 tile is one 128-B swizzle half, so the ring holds twice the stages.
template <int G, int D>
struct AttCfg {
  static constexpr int kDH = D / 64;                              // 64-d halves per row
  static constexpr uint32_t kTileBytes = kDH * kHalfBytes;        // K or V tile
  static constexpr int kStages = 3 * (128 / D);                   // K + V stage pairs of smem
  static constexpr int kKStages = ATT_KSTAGES * (128 / D);        // K ring depth
  static constexpr int kVStages = 2 * kStages - kKStages;         // V ring depth
  static_assert(kKStages <= 8 && kVStages <= 8 && kKStages >= 1 && kVStages >= 1, "ring depths");
  static constexpr uint32_t kQBytes = kDH * G * 128;
  static constexpr uint32_t kPHalf = kRowsT * G * 2;
  static constexpr uint32_t kPBytes = 2 * kPHalf;
  // Every accumulator is split in two (even / odd K-steps, summed by the
  // reader) so consecutive MMAs never write the same TMEM columns: a dependent
  // N = 16 chain costs ~75 cycles per MMA, two interleaved ones ~50
  // (tools/mma_bench.cu).  S^T slot s: columns [2Gs, 2Gs + 2G); O^T buffer b:
  // [kColO + 2Gb, kColO + 2Gb + 2G).
  static constexpr uint32_t kColO = kSlots * 2 * G;
  static constexpr uint32_t kTmemCols = (kSlots + 2) * 2 * G <= 64 ? 64 : (kSlots + 2) * 2 * G <= 128 ? 128 : 256;
  // softmax: kHS head groups x 4 TMEM lane quadrants = 4*kHS warps, kSH heads per thread
  static constexpr int kHS = G == 16 ? ATT_HS : 2;
  static constexpr int kSH = G / kHS;                             // heads per softmax thread
  static constexpr int kSoftWarps = 4 * kHS;
  // warp roles: 0 K TMA, 1 QK issuer, [2, 2 + kSoftWarps) softmax, then the PV
  // issuer, 4 epilogue warps (one per TMEM lane quadrant of O^T), the V TMA warp
  static constexpr int kPvWarp = 2 + kSoftWarps;
  static constexpr int kVWarp = kPvWarp + 5;
  static constexpr int kThreads = 32 * (kVWarp + 1);
  struct Smem {
    static constexpr uint32_t kv = 0;
    // D = 64: PV runs M = 128 over a half-width V tile, so the last stage's V
    // operand spans kHalfBytes past the ring: pad, never read back
    static constexpr uint32_t q = kv + (kKStages + kVStages) * kTileBytes + (kDH == 1 ? kHalfBytes : 0);   // 2 buffers
    static constexpr uint32_t p = q + 2 * kQBytes;                // 2 buffers
    static constexpr uint32_t stats = p + 2 * kPBytes;            // [2] x ([4 warps][16] l, [16] M, [4][16] l exact)
    static constexpr uint32_t red = stats + 2 * 9 * 16 * 4;       // [softmax warps][16] reduction scratch
    static constexpr uint32_t flags = red + kSoftWarps * 16 * 4;  // (unused)
    static constexpr uint32_t bars = flags + 2 * 8 * 4;
    static constexpr uint32_t total = bars + 88 * 8;
  };
};

struct Params {
  int64_t n, start;
  int hq, hkv, max_sel, out_f32;
  const int32_t* sel;
  void* out;
  float* lse;
  // batched decode: row i is sequence i with its own cache; its K/V tensor maps
  // are kv_maps[map_stride*i + 0/1] (device memory) and its query position is
  // seq_len[i] - 1.  Both null for prefill (one cache, pos = start + i).
  const CUtensorMap* kv_maps;
  int map_stride;
  const int64_t* seq_len;
  int bcast;          // prefill rows all at position start (tree-draft nodes)
  // split-K (decode): each work unit is (item, part) covering tiles
  // [part*split, (part+1)*split); partial O^T (unnormalised), max and row sum go
  // to part_o / part_ml and attend_combine_kernel merges them.  split == 0: off.
  int split;
  int p_split;        // 1: P as bf16 hi + lo (two PV MMAs per k-step), 0: P in bf16
  int group_major;    // prefill: items ordered (group, row) so one group's K/V is the L2 working set
  int64_t parts;
  float* part_o;      // [item][part][16][128]
  float* part_ml;     // [item][part][16][2]
  // tree-draft verification (infllm2_forward_tree): after its selected prefix
  // blocks every row also attends the tree rows [tree_row0, tree_row0 +
  // tree_n) of the cache, row j admitted iff bit j of its packed ancestor mask
  // (PackedMask, specdec.py:117-157) is set: word j / 64 of tree_words[row]
  const uint64_t* tree_words;
  int tree_n, tree_nw;
  int64_t tree_row0;
};

// Tiles of one item: prefix tiles (pairs of selected blocks) first, then the
// tree tiles (pairs of 64-row tree blocks).
struct Tiles {
  int nb, tp, tb, tt;
  __device__ __forceinline__ Tiles(const Params& p, int nb_) : nb(nb_), tp((nb_ + 1) / 2) {
    tb = p.tree_n > 0 ? (p.tree_n + kM - 1) / kM : 0;
    tt = (tb + 1) / 2;
  }
  __device__ __forceinline__ int total() const { return tp + tt; }
  __device__ __forceinline__ bool tree(int c) const { return c >= tp; }
  // 64-row blocks in tile c (1 or 2)
  __device__ __forceinline__ int blocks(int c) const {
    const int left = c < tp ? nb - 2 * c : tb - 2 * (c - tp);
    return left >= 2 ? 2 : 1;
  }
};

__device__ __forceinline__ void tile_range(const Params& p, int64_t part, int tiles, int* c0, int* c1) {
  if (p.split == 0) { *c0 = 0; *c1 = tiles; return; }
  const int64_t a = part * p.split, b = a + p.split;
  *c0 = (int)(a < tiles ? a : tiles);
  *c1 = (int)(b < tiles ? b : tiles);
}

// Work unit w -> (selection/output item = i*hkv + grp, split part, row i, group).
__device__ __forceinline__ void unit_of(const Params& p, int64_t w, int64_t* item, int64_t* part, int64_t* i,
                                        int* grp) {
  // 32-bit divisions whenever the unit space fits (a 64-bit division is a
  // ~100-instruction subroutine, paid by every warp role once per item)
  if (w < 0x7fffffff && p.n < 0x7fffffff) {
    const uint32_t w32 = (uint32_t)w, parts = (uint32_t)p.parts;
    const uint32_t u = parts == 1 ? w32 : w32 / parts;
    *part = (int64_t)(w32 - u * parts);
    uint32_t i32, g32;
    if (p.group_major) {
      g32 = u / (uint32_t)p.n;
      i32 = u - g32 * (uint32_t)p.n;
    } else {
      i32 = u / (uint32_t)p.hkv;
      g32 = u - i32 * (uint32_t)p.hkv;
    }
    *i = (int64_t)i32;
    *grp = (int)g32;
  } else {
    const int64_t u = w / p.parts;
    *part = w - u * p.parts;
    if (p.group_major) {
      *grp = (int)(u / p.n);
      *i = u - (int64_t)(*grp) * p.n;
    } else {
      *i = u / p.hkv;
      *grp = (int)(u - *i * p.hkv);
    }
  }
  *item = *i * p.hkv + *grp;
}

__device__ __forceinline__ int64_t item_pos(const Params& p, int64_t i) {
  // decode: seq_len holds the length before this step's append = the new
  // token's position
  return p.seq_len ? p.seq_len[i] : p.bcast ? p.start : p.start + i;
}

// The item's selection row, read once per warp with lane-parallel loads
// (entries lane, lane+32, lane+64); nb = blocks that start at or before pos.
struct SelRow {
  int r0, r1, r2;
  int nb;
  __device__ __forceinline__ int get(int j) const {
    const int v = j < 32 ? r0 : (j < 64 ? r1 : r2);
    return __shfl_sync(0xffffffffu, v, j & 31);
  }
};

__device__ __forceinline__ SelRow sel_raw(const Params& p, int64_t item, int lane) {
  const int32_t* s = p.sel + item * p.max_sel;
  SelRow r;
  r.r0 = lane < p.max_sel ? s[lane] : -1;
  r.r1 = lane + 32 < p.max_sel ? s[lane + 32] : -1;
  r.r2 = lane + 64 < p.max_sel ? s[lane + 64] : -1;
  r.nb = 0;
  return r;
}
__device__ __forceinline__ SelRow sel_finish(SelRow r, int64_t pos) {
  auto ok = [&](int b) { return b >= 0 && (int64_t)b * kM <= pos; };
  r.nb = __popc(__ballot_sync(0xffffffffu, ok(r.r0))) + __popc(__ballot_sync(0xffffffffu, ok(r.r1))) +
         __popc(__ballot_sync(0xffffffffu, ok(r.r2)));
  return r;
}
__device__ __forceinline__ SelRow load_sel(const Params& p, int64_t item, int64_t pos, int lane) {
  return sel_finish(sel_raw(p, item, lane), pos);
}
// Selection rows of a warp's item stream, fetched one item ahead so the
// global-memory latency hides behind the current item.
struct SelPrefetch {
  SelRow nxt;
  __device__ __forceinline__ void init(const Params& p, int64_t w, int64_t items, int lane) {
    if (w < items) {
      int64_t item, part, i;
      int grp;
      unit_of(p, w, &item, &part, &i, &grp);
      nxt = sel_raw(p, item, lane);
    }
  }
  // row of unit w (which must be the prefetched one); prefetches w + stride
  __device__ __forceinline__ SelRow take(const Params& p, int64_t w, int64_t items, int64_t pos, int lane) {
    const SelRow cur = nxt;
    const int64_t w2 = w + gridDim.x;
    if (w2 < items) {
      int64_t item, part, i;
      int grp;
      unit_of(p, w2, &item, &part, &i, &grp);
      nxt = sel_raw(p, item, lane);
    }
    return sel_finish(cur, pos);
  }
};


template <int G, int D>
__global__ void __launch_bounds__(AttCfg<G, D>::kThreads, 1)
attend_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const Params p) {
  using C = AttCfg<G, D>;
  using Smem = typename C::Smem;
  constexpr int kG = G;
  constexpr int kD = D;
  constexpr uint32_t kTileBytes = C::kTileBytes;
  constexpr uint32_t kQBytes = C::kQBytes;
  constexpr uint32_t kPBytes = C::kPBytes;
  constexpr uint32_t kPHalf = C::kPHalf;
  constexpr uint32_t kColO = C::kColO;
  constexpr int kSH = C::kSH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by pointer arithmetic on the __shared__ array (a uintptr_t round trip
  // loses the address space: every access would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  // K and V have separate rings: a K stage frees as soon as its QK is done, so
  // QK runs ahead of the softmax / PV chain instead of waiting for PV to free
  // a shared K+V stage
  uint64_t* k_full = bars + 38;           // [kKStages <= 8]
  uint64_t* k_empty = bars + 46;
  uint64_t* v_full = bars + 54;           // [kVStages <= 8]
  uint64_t* v_empty = bars + 62;
  uint64_t* q_full = bars + 6;            // [2]
  uint64_t* q_empty = bars + 8;           // [2]
  uint64_t* s_full = bars + 70;           // [kSlots <= 8]
  uint64_t* s_empty = bars + 78;          // [kSlots <= 8]
  uint64_t* p_full = bars + 14;           // [2]
  uint64_t* p_empty = bars + 16;          // [2]
  uint64_t* o_full = bars + 18;           // [2]
  uint64_t* o_empty = bars + 20;          // [2]
  uint64_t* st_full = bars + 22;          // [2]
  uint64_t* st_empty = bars + 24;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 36);
  float* stats = reinterpret_cast<float*>(smem + Smem::stats);
  float* red = reinterpret_cast<float*>(smem + Smem::red);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // q rows and outputs stream through L2 once; the gathered K/V blocks are
  // re-read by many items: keep them (DRAM re-fetches of evicted K/V were
  // ~0.85 GB per 128K layer, ncu r1)
  const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
  ATT_T0(t_kernel);
#ifdef ATT_PROFILE
  long long att_acc[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) att_acc[i] = 0;
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kKStages; ++i) { mbar_init(k_full + i, 1); mbar_init(k_empty + i, 1); }
    for (int i = 0; i < C::kVStages; ++i) { mbar_init(v_full + i, 1); mbar_init(v_empty + i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
      mbar_init(p_full + i, C::kSoftWarps);
      mbar_init(p_empty + i, 1);
      mbar_init(o_full + i, 1);
      mbar_init(o_empty + i, 4);
      mbar_init(st_full + i, C::kSoftWarps);
      mbar_init(st_empty + i, 4);
    }
    for (int i = 0; i < kSlots; ++i) { mbar_init(s_full + i, 1); mbar_init(s_empty + i, C::kSoftWarps); }
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;       // cols [0,64): S slots, [64,96): O buffers
  pdl_wait();                             // no-op unless launched as a dependent
  const int64_t items = p.n * p.hkv * p.parts;   // work units (item, part)

  if (warp == 0 || warp == C::kVWarp) {
    // -------------------------------------------------------------- producers
    // warp 0: Q + K tiles into the K ring; warp 15: V tiles into the V ring
    const bool is_k = warp == 0;
    uint64_t* ring_full = is_k ? k_full : v_full;
    uint64_t* ring_empty = is_k ? k_empty : v_empty;
    uint8_t* ring = smem + Smem::kv + (is_k ? 0 : C::kKStages * kTileBytes);
    const int nstages = is_k ? C::kKStages : C::kVStages;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    SelPrefetch pf;
    pf.init(p, blockIdx.x, items, lane);
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
      int64_t item, part, i;
      int grp;
      unit_of(p, w, &item, &part, &i, &grp);
      const int64_t pos = item_pos(p, i);
      const CUtensorMap* mk = p.kv_maps ? p.kv_maps + (int64_t)p.map_stride * i : &tm_k;
      const CUtensorMap* mv = p.kv_maps ? p.kv_maps + (int64_t)p.map_stride * i + 1 : &tm_v;
      const CUtensorMap* mm = is_k ? mk : mv;
      const SelRow sr = pf.take(p, w, items, pos, lane);
      const Tiles tl(p, sr.nb);
      int c0, c1;
      tile_range(p, part, tl.total(), &c0, &c1);
      if (c0 >= c1) continue;
      const int qb = it & 1;
      const uint32_t q_par = ((it >> 1) & 1) ^ 1;
      ++it;
      if (is_k && lane == 0) {
        mbar_wait(q_empty + qb, q_par);
        mbar_arrive_expect_tx(q_full + qb, kQBytes);
        uint8_t* qd = smem + Smem::q + qb * kQBytes;
#pragma unroll
        for (int hh = 0; hh < C::kDH; ++hh)
          tma_load_3d_hint(qd + hh * kG * 128, &tm_q, q_full + qb, 64 * hh, grp * kG, (int)i, pol_stream);
      }
      for (int c = c0; c < c1; ++c) {
        const int nt = tl.blocks(c);
        const int b0 = sr.get(2 * c < 96 ? 2 * c : 95);
        const int b1 = sr.get(2 * c + 1 < 96 ? 2 * c + 1 : 95);
        const bool tree = tl.tree(c);
        if (lane == 0) {
          ATT_T0(t0w);
          mbar_wait(ring_empty + stage, phase ^ 1);
          if (is_k) ATT_ADD(12, t0w); else ATT_ADD(13, t0w);
          mbar_arrive_expect_tx(ring_full + stage, nt * C::kDH * (kM * 128));
          uint8_t* dst = ring + stage * kTileBytes;
          for (int x = 0; x < nt; ++x) {
            const int row0 = tree ? (int)(p.tree_row0 + (int64_t)kM * (2 * (c - tl.tp) + x)) : (x ? b1 : b0) * kM;
            const uint32_t off = x * kM * 128;
#pragma unroll
            for (int hh = 0; hh < C::kDH; ++hh)
              tma_load_3d_hint(dst + hh * kHalfBytes + off, mm, ring_full + stage, 64 * hh, row0, grp, pol_keep);
          }
        }
        __syncwarp();
        if (++stage == nstages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- QK issuer
    // S^T[slot] = K_tile . Q^T for every tile of the CTA's item stream, up to
    // kSlots tiles ahead of the softmax warps.  QK and PV are issued from two
    // warps: each tcgen05.mma costs ~50 cycles of A-operand fetch whatever N
    // (N = 16 here), so one issuer stalled on a barrier leaves the tensor
    // pipe idle.
    const uint32_t idesc_qk = idesc_bf16_f32(128, kG);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t tcount = 0;
    int it = 0;
    SelPrefetch pf;
    pf.init(p, blockIdx.x, items, lane);
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
      int64_t item, part, i;
      int grp;
      unit_of(p, w, &item, &part, &i, &grp);
      const int64_t pos = item_pos(p, i);
      const SelRow sr = pf.take(p, w, items, pos, lane);
      int c0, c1;
      tile_range(p, part, Tiles(p, sr.nb).total(), &c0, &c1);
      if (c0 >= c1) continue;
      const int qb = it & 1;
      mbar_wait(q_full + qb, (it >> 1) & 1);
      const uint64_t dq = sdesc_k_sw128(smem_u32(smem + Smem::q + qb * kQBytes));
      for (int c = c0; c < c1; ++c, ++tcount) {
        const int slot = tcount % kSlots;
        mbar_wait(k_full + stage, phase);
        ATT_T0(q1);
        mbar_wait(s_empty + slot, ((tcount / kSlots) & 1) ^ 1);
        if (lane == 0) ATT_ADD(2, q1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dk = sdesc_k_sw128(smem_u32(smem + Smem::kv + stage * kTileBytes));
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t off = (k >> 2) * kHalfBytes + (k & 3) * 32;
            const uint32_t qoff = (k >> 2) * (kG * 128) + (k & 3) * 32;
            if constexpr (kQkSplit)
              umma_f16_ss(tmem + slot * 2 * kG + (k & 1) * kG, dk + (off >> 4), dq + (qoff >> 4), idesc_qk,
                          k > 1 ? 1u : 0u);
            else
              umma_f16_ss(tmem + slot * 2 * kG, dk + (off >> 4), dq + (qoff >> 4), idesc_qk, k > 0 ? 1u : 0u);
          }
          umma_commit(k_empty + stage);                // K tile consumed: its stage may refill
          umma_commit(s_full + slot);
          if (c == c1 - 1) umma_commit(q_empty + qb);
        }
        __syncwarp();
        if (++stage == C::kKStages) { stage = 0; phase ^= 1; }
      }
      ++it;
    }
  } else if (warp == C::kPvWarp) {
    // -------------------------------------------------------------- PV issuer
    const uint32_t idesc_pv = idesc_bf16_f32_major(128, kG, 1, 1);
    int stage = 0;
    uint32_t vphase = 0;
    uint32_t pcount = 0;
    int it = 0;
    SelPrefetch pf;
    pf.init(p, blockIdx.x, items, lane);
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
      int64_t item, part, i;
      int grp;
      unit_of(p, w, &item, &part, &i, &grp);
      const int64_t pos = item_pos(p, i);
      const SelRow sr = pf.take(p, w, items, pos, lane);
      const Tiles tl(p, sr.nb);
      int c0, c1;
      tile_range(p, part, tl.total(), &c0, &c1);
      if (c0 >= c1) continue;
      const int ob = it & 1;
      for (int c = c0; c < c1; ++c, ++pcount) {
        const int pbuf = pcount & 1;
        ATT_T0(v0);
        mbar_wait(v_full + stage, vphase);
        if (lane == 0) ATT_ADD(4, v0);
        ATT_T0(v1);
        mbar_wait(p_full + pbuf, (pcount >> 1) & 1);
        if (lane == 0) ATT_ADD(5, v1);
        if (c == c0) mbar_wait(o_empty + ob, ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const int ksteps = tl.blocks(c) == 2 ? 8 : 4;
        if (elect_one()) {
          const uint64_t dv = sdesc_mn_sw128(smem_u32(smem + Smem::kv + (C::kKStages + stage) * kTileBytes),
                                             kHalfBytes, 1024);
          // P^T (K = rows, N = heads, no swizzle): 8-row K groups of 16*G bytes, 8-head groups 128 B apart
          const uint64_t dp = sdesc_interleave(smem_u32(smem + Smem::p + pbuf * kPBytes), 16 * kG, 128);
          const uint32_t ocol = tmem + kColO + ob * 2 * kG;
          const uint32_t acc0 = c > c0 ? 1u : 0u;
          if (p.p_split || pos < kSplitPBelow || tl.nb <= kSplitPBlocks) {      // hi -> O_a, lo -> O_b
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              if (k < ksteps) {
                umma_f16_ss(ocol, dv + (k * 2048 >> 4), dp + (k * 32 * kG >> 4), idesc_pv, (acc0 | k) ? 1u : 0u);
                umma_f16_ss(ocol + kG, dv + (k * 2048 >> 4), dp + ((kPHalf + k * 32 * kG) >> 4), idesc_pv,
                            (acc0 | k) ? 1u : 0u);
              }
            }
          } else {              // even K-steps -> O_a, odd -> O_b
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              if (k < ksteps)
                umma_f16_ss(ocol + (k & 1) * kG, dv + (k * 2048 >> 4), dp + (k * 32 * kG >> 4), idesc_pv,
                            (acc0 | (k >> 1)) ? 1u : 0u);
            }
          }
          umma_commit(v_empty + stage);
          umma_commit(p_empty + pbuf);
          if (c == c1 - 1) umma_commit(o_full + ob);
        }
        __syncwarp();
        if (++stage == C::kVStages) { stage = 0; vphase ^= 1; }
      }
      ++it;
    }
  } else if (warp < C::kPvWarp) {
    // -------------------------------------------------------------- softmax
    // 8 warps: warps w and w+4 share TMEM lane quadrant w%4 (tile rows); the
    // first four take heads 0..7, the others heads 8..15 of every row.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;                 // head group 0..kHS-1 (its own 128-thread barrier)
    const int h0 = kSH * half;
    const int ws = warp - 2;                           // scratch row
    const int row = quad * 32 + lane;                  // tile row == TMEM lane
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const float c2 = 1.4426950408889634f / sqrtf((float)kD);
    int pbuf = 0;
    uint32_t p_ph[2] = {0, 0};
    uint32_t tcount = 0;
    int it = 0;
    SelPrefetch pf;
    pf.init(p, blockIdx.x, items, lane);
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
      int64_t item, part, i;
      int grp;
      unit_of(p, w, &item, &part, &i, &grp);
      const int64_t pos = item_pos(p, i);
      ATT_T0(s16);
      const SelRow sr = pf.take(p, w, items, pos, lane);
      if (warp == 2 && lane == 0) ATT_ADD(16, s16);
      const Tiles tl(p, sr.nb);
      int c0, c1;
      tile_range(p, part, tl.total(), &c0, &c1);
      if (c0 >= c1) continue;
      const int ob = it & 1;
      const bool splitp = p.p_split || pos < kSplitPBelow || tl.nb <= kSplitPBlocks;
      float mrun[kSH], lsum[kSH], lsx[kSH];     // lsum: weights as used by PV; lsx: unrounded (LSE)
#pragma unroll
      for (int h = 0; h < kSH; ++h) { mrun[h] = -INFINITY; lsum[h] = 0.f; lsx[h] = 0.f; }
      ATT_T0(sloop);
      for (int c = c0; c < c1; ++c) {
        const int sslot = tcount % kSlots;
        ATT_T0(s0);
        mbar_wait(s_full + sslot, (tcount / kSlots) & 1);
        if (warp == 2 && lane == 0) ATT_ADD(8, s0);
        ++tcount;
        tc_fence_after();
        float z[kSH], z2[kSH];
        ATT_T0(s4);
        tmem_ld_n<kSH>(tmem + lane_base + sslot * 2 * kG + h0, z);
        if constexpr (kQkSplit) tmem_ld_n<kSH>(tmem + lane_base + sslot * 2 * kG + kG + h0, z2);
        tmem_wait_ld();
        if (warp == 2 && lane == 0) ATT_ADD(15, s4);
        if constexpr (kQkSplit) {
#pragma unroll
          for (int h = 0; h < kSH; ++h) z[h] += z2[h];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + sslot);
        ATT_T0(s19);
        const int x = row >> 6;
        const int b0 = sr.get(2 * c < 96 ? 2 * c : 95), b1 = sr.get(2 * c + 1 < 96 ? 2 * c + 1 : 95);
        bool valid;
        if (!tl.tree(c)) {
          valid = (2 * c + x) < tl.nb;
          if (valid) valid = (int64_t)(x ? b1 : b0) * kM + (row & 63) <= pos;
        } else {   // tree row j: admitted by the packed ancestor-or-self mask
          const int j = kM * (2 * (c - tl.tp) + x) + (row & 63);
          valid = j < p.tree_n && ((p.tree_words[i * p.tree_nw + (j >> 6)] >> (j & 63)) & 1ull);
        }
        {
          // z * c2 as packed pairs (FFMA2, zero addend); masked rows -inf by
          // select (a row past the tile's blocks may hold stale smem: NaN)
          const uint64_t c2x2 = pk2(c2, c2);
#pragma unroll
          for (int h = 0; h < kSH; h += 2) upk2(ffma2(pk2(z[h], z[h + 1]), c2x2, 0ull), z[h], z[h + 1]);
#pragma unroll
          for (int h = 0; h < kSH; ++h) z[h] = valid ? z[h] : -INFINITY;
        }
        // running max: exact on the first tile, rescale later only if z > M + 8.
        // The max is per head, so only the four warps of a head half vote (one
        // OR-reducing 128-thread barrier per tile)
        if (warp == 2 && lane == 0) ATT_ADD(19, s19);
        bool need = (c == c0);
        if (c > c0) {
          bool over = false;
#pragma unroll
          for (int h = 0; h < kSH; h += 2) {
            float t0, t1;
            upk2(fadd2(pk2(mrun[h], mrun[h + 1]), pk2(8.f, 8.f)), t0, t1);
            over |= (z[h] > t0) | (z[h + 1] > t1);
          }
          // the half's 128-thread barrier ORs the votes (bar.red)
          ATT_T0(s1);
          need = named_bar_or(2 + half, 128, over);
          if (warp == 2 && lane == 0) ATT_ADD(9, s1);
        }
        ATT_T0(s2);
        if (need) {
          {
            float zz[kSH];
#pragma unroll
            for (int h = 0; h < kSH; ++h) zz[h] = z[h];
            const float v = warp_reduce_n<kSH>(zz, lane, [](float a, float b) { return fmaxf(a, b); });
            if (reduce_writer_n<kSH>(lane)) red[ws * 16 + reduce_head_n<kSH>(lane)] = v;
          }
          named_bar_sync(2 + half, 128);
          float corr[kSH];
          bool any_corr = false;
#pragma unroll
          for (int h = 0; h < kSH; ++h) {
            const int hb = 4 * half;                    // this half's four warps: scratch rows hb..hb+3
            const float tm = fmaxf(fmaxf(red[(hb + 0) * 16 + h], red[(hb + 1) * 16 + h]),
                                   fmaxf(red[(hb + 2) * 16 + h], red[(hb + 3) * 16 + h]));
            const float mnew = fmaxf(mrun[h], tm);
            corr[h] = (mrun[h] == -INFINITY) ? 1.f : ex2(mrun[h] - mnew);
            any_corr |= (c > c0) && (corr[h] != 1.f);
            lsum[h] *= (mrun[h] == -INFINITY) ? 0.f : corr[h];
            lsx[h] *= (mrun[h] == -INFINITY) ? 0.f : corr[h];
            mrun[h] = mnew;
          }
          named_bar_sync(2 + half, 128);
          if (c > c0 && any_corr) {
            // rescale this thread's 8 O^T columns (d lane == row): wait for
            // PV(c-1), whose completion is the next phase of p_empty[its buffer]
            mbar_wait(p_empty + (pbuf ^ 1), p_ph[pbuf ^ 1] ^ 1);
            tc_fence_after();
            float o[kSH], o2[kSH];
            tmem_ld_n<kSH>(tmem + lane_base + kColO + ob * 2 * kG + h0, o);
            tmem_ld_n<kSH>(tmem + lane_base + kColO + ob * 2 * kG + kG + h0, o2);
            tmem_wait_ld();
#pragma unroll
            for (int h = 0; h < kSH; ++h) { o[h] *= corr[h]; o2[h] *= corr[h]; }
            tmem_st_n<kSH>(tmem + lane_base + kColO + ob * 2 * kG + h0, o);
            tmem_st_n<kSH>(tmem + lane_base + kColO + ob * 2 * kG + kG + h0, o2);
            tmem_wait_st();
            tc_fence_before();
          }
        }
        if (warp == 2 && lane == 0) ATT_ADD(10, s2);
        // P = 2^(z - M) as bf16 into the MN-major interleaved buffer
        ATT_T0(s3);
        mbar_wait(p_empty + pbuf, p_ph[pbuf] ^ 1);
        if (warp == 2 && lane == 0) ATT_ADD(11, s3);
        p_ph[pbuf] ^= 1;
        // P in bf16 for one PV MMA per k-step; the row sums use the ROUNDED
        // weights, so O = sum P~ V / sum P~ stays a convex combination (error
        // ~2^-9 |V| / sqrt(rows)).  p_split: P also as a bf16 lo part (second
        // PV MMA), ~16-bit weights, for callers that want 1e-5 outputs.
        ATT_T0(s20);
        uint32_t phi[kSH / 2], plo[kSH / 2];
#pragma unroll
        for (int h = 0; h < kSH; h += 2) {
          // packed pairs: z - M (FADD2), the row sums (FADD2), a - hi (FFMA2)
          float xa, xb;
          upk2(fadd2(pk2(z[h], z[h + 1]), pk2(-mrun[h], -mrun[h + 1])), xa, xb);
          const float a = ex2(xa);
          const float b = ex2(xb);
          const __nv_bfloat162 hi2 = __floats2bfloat162_rn(a, b);
          const uint32_t hb = *reinterpret_cast<const uint32_t*>(&hi2);
          const uint64_t ab = pk2(a, b);
          const uint64_t hf2 = pk2(__uint_as_float(hb << 16), __uint_as_float(hb & 0xffff0000u));
          upk2(fadd2(pk2(lsx[h], lsx[h + 1]), ab), lsx[h], lsx[h + 1]);
          upk2(fadd2(pk2(lsum[h], lsum[h + 1]), splitp ? ab : hf2), lsum[h], lsum[h + 1]);
          float la, lb;
          upk2(ffma2(hf2, pk2(-1.f, -1.f), ab), la, lb);    // a - hi(a), exact
          const __nv_bfloat162 lo2 = __floats2bfloat162_rn(la, lb);
          phi[h / 2] = hb;
          plo[h / 2] = *reinterpret_cast<const uint32_t*>(&lo2);
        }
        uint8_t* pb = smem + Smem::p + pbuf * kPBytes;
        // P^T core matrices: 8 rows x 8 heads (128 B), 8-row groups 16*G bytes apart
        const uint32_t base = (row >> 3) * (16 * kG) + (row & 7) * 16 + 128 * (h0 >> 3) + 2 * (h0 & 7);
        if constexpr (kSH == 8) {
          *reinterpret_cast<uint4*>(pb + base) = make_uint4(phi[0], phi[1], phi[2], phi[3]);
          if (splitp) *reinterpret_cast<uint4*>(pb + kPHalf + base) = make_uint4(plo[0], plo[1], plo[2], plo[3]);
        } else {
          *reinterpret_cast<uint2*>(pb + base) = make_uint2(phi[0], phi[1]);
          if (splitp) *reinterpret_cast<uint2*>(pb + kPHalf + base) = make_uint2(plo[0], plo[1]);
        }
        if (warp == 2 && lane == 0) ATT_ADD(20, s20);
        ATT_T0(s5);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full + pbuf);
        if (warp == 2 && lane == 0) ATT_ADD(6, s5);
        pbuf ^= 1;
      }
      if (warp == 2 && lane == 0) ATT_ADD(1, sloop);
      // per-head row sums -> stats for the epilogue
      ATT_T0(s17);
      mbar_wait(st_empty + ob, ((it >> 1) & 1) ^ 1);
      if (warp == 2 && lane == 0) ATT_ADD(17, s17);
      ATT_T0(s18);
      float* st = stats + ob * 9 * 16;
      {
        const float v = warp_reduce_n<kSH>(lsum, lane, [](float a, float b) { return a + b; });
        const float vx = warp_reduce_n<kSH>(lsx, lane, [](float a, float b) { return a + b; });
        if (reduce_writer_n<kSH>(lane)) {
          st[quad * 16 + h0 + reduce_head_n<kSH>(lane)] = v;
          st[80 + quad * 16 + h0 + reduce_head_n<kSH>(lane)] = vx;
        }
      }
      if (quad == 0 && lane < kSH) {
        float mine = mrun[0];
#pragma unroll
        for (int h = 1; h < kSH; ++h) mine = (lane == h) ? mrun[h] : mine;
        st[64 + h0 + lane] = mine;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(st_full + ob);
      if (warp == 2 && lane == 0) ATT_ADD(18, s18);
      ++it;
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int quad = warp & 3;
    const int d = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    int it = 0;
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
      int64_t item, part, i;
      int grp;
      unit_of(p, w, &item, &part, &i, &grp);
      if (p.split) {
        const SelRow sr = load_sel(p, item, item_pos(p, i), lane);
        int c0, c1;
        tile_range(p, part, Tiles(p, sr.nb).total(), &c0, &c1);
        if (c0 >= c1) {   // empty part: neutral partial for the combine
          if (quad == 0 && lane < kG) {
            p.part_ml[(w * kG + lane) * 2] = -INFINITY;
            p.part_ml[(w * kG + lane) * 2 + 1] = 0.f;
          }
          continue;
        }
      }
      const int ob = it & 1;
      const uint32_t par = (it >> 1) & 1;
      ++it;
      mbar_wait(o_full + ob, par);
      mbar_wait(st_full + ob, par);
      tc_fence_after();
      float o[kG], o2[kG];
      tmem_ld_n<kG>(tmem + lane_base + kColO + ob * 2 * kG, o);
      tmem_ld_n<kG>(tmem + lane_base + kColO + ob * 2 * kG + kG, o2);
      tmem_wait_ld();
#pragma unroll
      for (int h = 0; h < kG; ++h) o[h] += o2[h];
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty + ob);
      const float* st = stats + ob * 9 * 16;
      float l[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h) l[h] = st[h] + st[16 + h] + st[32 + h] + st[48 + h];
      auto lsum_exact = [&](int h) { return st[80 + h] + st[96 + h] + st[112 + h] + st[128 + h]; };
      if (p.split) {
        float* po = p.part_o + w * (kG * kD) + d;
        if (d < kD) {     // D = 64: O^T lanes >= D unused
#pragma unroll
          for (int h = 0; h < kG; ++h) po[h * kD] = o[h];
        }
        if (quad == 0 && lane < kG) {
          float lh = l[0];
#pragma unroll
          for (int h = 1; h < kG; ++h) lh = (lane == h) ? l[h] : lh;
          p.part_ml[(w * kG + lane) * 2] = st[64 + lane];
          p.part_ml[(w * kG + lane) * 2 + 1] = lh;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(st_empty + ob);
        continue;
      }
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
      if (p.lse && quad == 0 && lane < kG)
        p.lse[i * p.hq + grp * kG + lane] = (st[64 + lane] + log2f(lsum_exact(lane))) * 0.6931471805599453f;
      __syncwarp();
      if (lane == 0) mbar_arrive(st_empty + ob);
    }
  }

  tc_fence_before();
  __syncthreads();
#ifdef ATT_PROFILE
  if (lane == 0 && warp == 1) ATT_ADD(0, t_kernel);
  if (lane == 0 && warp == C::kPvWarp) ATT_ADD(3, t_kernel);
  if (lane == 0 && warp == 2) ATT_ADD(7, t_kernel);
  if (lane == 0 && warp == 0) ATT_ADD(14, t_kernel);
#ifdef ATT_PROFILE
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 24; ++i)
      if (att_acc[i]) atomicAdd(reinterpret_cast<unsigned long long*>(&g_att_cyc[blockIdx.x][i]), (unsigned long long)att_acc[i]);
#endif
#endif
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

// Merge split-K partials of each (row, group) item: O = sum_p O_p 2^(m_p - M) /
// sum_p l_p 2^(m_p - M).  One CTA per item; part weights computed once into
// shared memory, then thread (h, d-slice) streams the parts with independent loads.
template <int kG, int kD>
__global__ void __launch_bounds__(512) attend_combine_kernel(const float* __restrict__ part_o,
                                                             const float* __restrict__ part_ml, int64_t parts, int hq,
                                                             int hkv, void* out, int out_f32, float* lse,
                                                             int64_t* seq_len) {
  __shared__ float wgt[(kMaxSel / 2 + 1) * kG];   // [part][h]
  __shared__ float inv_l[kG];
  pdl_launch_dependents();
  pdl_wait();
  const int64_t item = blockIdx.x;
  const int64_t i = item / hkv;
  const int grp = (int)(item - i * hkv);
  const int t = threadIdx.x;
  if (t < kG) {
    float M = -INFINITY;
    for (int64_t q = 0; q < parts; ++q) M = fmaxf(M, part_ml[((item * parts + q) * kG + t) * 2]);
    float L = 0.f;
    for (int64_t q = 0; q < parts; ++q) {
      const float m = part_ml[((item * parts + q) * kG + t) * 2];
      const float w = m == -INFINITY ? 0.f : ex2(m - M);
      wgt[q * kG + t] = w;
      L += part_ml[((item * parts + q) * kG + t) * 2 + 1] * w;
    }
    inv_l[t] = 1.f / L;
    if (lse) lse[i * hq + grp * kG + t] = (M + log2f(L)) * 0.6931471805599453f;
  }
  __syncthreads();
  for (int x = t; x < kG * kD; x += blockDim.x) {
    const int h = x / kD;
    float acc = 0.f;
#pragma unroll 4
    for (int64_t q = 0; q < parts; ++q) {
      const float w = wgt[q * kG + h];
      if (w != 0.f) acc += part_o[(item * parts + q) * (kG * kD) + x] * w;
    }
    const int64_t o = (i * hq + (int64_t)grp * kG) * kD + x;
    if (out_f32)
      static_cast<float*>(out)[o] = acc * inv_l[h];
    else
      static_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(acc * inv_l[h]);
  }
  // end of the decode step: the new token is now part of the cache
  if (seq_len && grp == 0 && t == 0) seq_len[i] += 1;
}

}  // namespace

size_t attend_split_workspace(int64_t n_seq, int hkv, int max_sel) {
  const int64_t parts = (max_sel + 1) / 2;
  return (size_t)n_seq * hkv * parts * (kG * kD + 2 * kG) * sizeof(float);
}

// Batched decode: one query row per sequence, per-sequence K/V tensor maps in
// device memory (maps[stride*s + 0] = K, + 1 = V), positions seq_len[s] - 1.
template <int G, int D>
static cudaError_t attend_decode(int hq, int hkv, int max_sel, int64_t n_seq, const void* q,
                                 const CUtensorMap* kv_maps, int map_stride, const int64_t* seq_len,
                                 const int32_t* selection, void* out, int out_f32, float* lse, float* split_ws,
                                 cudaStream_t stream) {
  Params p;
  p.n = n_seq;
  p.start = 0;
  p.hq = hq;
  p.hkv = hkv;
  p.max_sel = max_sel;
  p.out_f32 = out_f32;
  p.sel = selection;
  p.out = out;
  p.lse = lse;
  p.kv_maps = kv_maps;
  p.map_stride = map_stride;
  p.seq_len = seq_len;
  p.bcast = 0;
  // split-K: one 2-block tile per CTA so n_seq*hkv*10 CTAs share the gather
  p.split = split_ws ? 1 : 0;
  p.p_split = 1;
  p.group_major = 0;
  p.parts = split_ws ? (max_sel + 1) / 2 : 1;
  p.part_o = split_ws;
  p.part_ml = split_ws ? split_ws + n_seq * hkv * p.parts * (G * D) : nullptr;
  p.tree_words = nullptr;
  p.tree_n = p.tree_nw = 0;
  p.tree_row0 = 0;
  CUtensorMap tq;
  const uint64_t dims[3] = {(uint64_t)D, (uint64_t)hq, (uint64_t)n_seq};
  const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)hq * D * 2};
  const uint32_t box[3] = {64, (uint32_t)G, 1};
  if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return cudaErrorInvalidValue;
  const size_t smem = AttCfg<G, D>::Smem::total + 1024;
  cudaError_t e = smem_attr_once((const void*)attend_tc_kernel<G, D>, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t items = n_seq * hkv * p.parts;
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(items < sms ? items : sms);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(AttCfg<G, D>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  e = cudaLaunchKernelEx(&cfg, attend_tc_kernel<G, D>, tq, tq, tq, p);
  if (e != cudaSuccess) return e;
  if (split_ws) {
    cfg.gridDim = dim3((unsigned)(n_seq * hkv));
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 0;
    count_launch();
    e = cudaLaunchKernelEx(&cfg, attend_combine_kernel<G, D>, (const float*)p.part_o, (const float*)p.part_ml,
                           p.parts, hq, hkv, out, out_f32, lse, const_cast<int64_t*>(seq_len));
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_attend_tc_decode(int hq, int hkv, int d, int max_sel, int64_t n_seq, const void* q,
                                    const CUtensorMap* kv_maps, int map_stride, const int64_t* seq_len,
                                    const int32_t* selection, void* out, int out_f32, float* lse,
                                    float* split_ws, cudaStream_t stream) {
  if (hq / hkv == 16 && d == 128)
    return attend_decode<16, 128>(hq, hkv, max_sel, n_seq, q, kv_maps, map_stride, seq_len, selection, out, out_f32,
                                  lse, split_ws, stream);
  if (hq / hkv == 8 && d == 64)
    return attend_decode<8, 64>(hq, hkv, max_sel, n_seq, q, kv_maps, map_stride, seq_len, selection, out, out_f32,
                                lse, split_ws, stream);
  return cudaErrorInvalidValue;
}

static int group_major_enabled() {
  static const int v = [] {
    const char* e = getenv("INFLLM2_ATTEND_ORDER");
    return (e && e[0] == 'r') ? 0 : 1;     // default: group-major
  }();
  return v;
}

template <int G, int D>
static cudaError_t launch_attend_prefill(const CallShape& cs, const void* q, int64_t q_row_stride,
                                         const void* k_cache, const void* v_cache, int64_t cap, const Params& p,
                                         cudaStream_t stream) {
  CUtensorMap tq, tk, tv;
  {
    const uint64_t dims[3] = {(uint64_t)D, (uint64_t)cs.hq, (uint64_t)cs.n};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)q_row_stride * 2};
    const uint32_t box[3] = {64, (uint32_t)G, 1};
    if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    // rows past the cache length are visible only to tree tiles (the draft rows)
    const uint64_t rows = (uint64_t)(p.tree_n > 0 ? p.tree_row0 + p.tree_n : cs.cache_len);
    const uint64_t dims[3] = {(uint64_t)D, rows, (uint64_t)cs.hkv};
    const uint64_t strides[2] = {(uint64_t)D * 2, (uint64_t)cap * D * 2};
    const uint32_t box[3] = {64, (uint32_t)kM, 1};
    if (!encode_tmap_3d_bf16(&tk, k_cache, dims, strides, box)) return cudaErrorInvalidValue;
    if (!encode_tmap_3d_bf16(&tv, v_cache, dims, strides, box)) return cudaErrorInvalidValue;
  }
  const size_t smem = AttCfg<G, D>::Smem::total + 1024;
  {
    cudaError_t e = smem_attr_once((const void*)attend_tc_kernel<G, D>, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = cs.n * cs.hkv;
  static const int ctas_cap = [] {
    const char* e = getenv("INFLLM2_ATTEND_CTAS");
    return e ? atoi(e) : 0;
  }();
  if (ctas_cap > 0 && ctas_cap < sms) sms = ctas_cap;
  const int grid = (int)(items < sms ? items : sms);
  count_launch();
  attend_tc_kernel<G, D><<<grid, AttCfg<G, D>::kThreads, smem, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

bool tc_attend_supported(const infllm2_geometry& g, const CallShape& cs) {
  if (!tc_kernels_enabled()) return false;
  const bool shape_ok = (cs.group == 16 && cs.d == 128) || (cs.group == 8 && cs.d == 64);
  if (!shape_ok || g.block_size != kM) return false;
  if (cs.max_sel > kMaxSel) return false;
  return cs.n > 0;
}

bool attend_share_range(const infllm2_geometry& g, const CallShape& cs, int p_split, bool tree, int64_t* row0,
                        int64_t* row1);
cudaError_t launch_attend_share(const CallShape& cs, int64_t row0, int64_t row1, const void* q, int64_t q_row_stride,
                                const void* k_cache, const void* v_cache, int64_t cap, const int32_t* selection,
                                void* out, int out_f32, float* lse, cudaStream_t stream);

static cudaError_t launch_attend_rows(const infllm2_geometry& g, const CallShape& cs, const void* q,
                                     int64_t q_row_stride, const void* k_cache, const void* v_cache, int64_t cap,
                                     const int32_t* selection, void* out, int out_f32, float* lse, int p_split,
                                     cudaStream_t stream, const TreeArgs* tree);

cudaError_t launch_attend_tc(const infllm2_geometry& g, const CallShape& cs, const void* q, int64_t q_row_stride,
                             const void* k_cache, const void* v_cache, int64_t cap, const int32_t* selection,
                             void* out, int out_f32, float* lse, int p_split, cudaStream_t stream,
                             const TreeArgs* tree) {
  // prefill rows at positions >= 256 of the MiniCPM4 geometry: forced blocks
  // shared by 4 rows (attend_share.cu); the rows around them here
  int64_t r0, r1;
  if (attend_share_range(g, cs, p_split, tree != nullptr, &r0, &r1)) {
    const size_t ob = out_f32 ? 4 : 2;
    auto part = [&](int64_t a, int64_t b) -> cudaError_t {
      if (b <= a) return cudaSuccess;
      CallShape c2 = cs;
      c2.start = cs.start + a;
      c2.n = b - a;
      return launch_attend_rows(g, c2, static_cast<const __nv_bfloat16*>(q) + a * q_row_stride, q_row_stride,
                                k_cache, v_cache, cap, selection + a * cs.hkv * cs.max_sel,
                                static_cast<uint8_t*>(out) + a * cs.hq * cs.d * ob, out_f32,
                                lse ? lse + a * cs.hq : nullptr, p_split, stream, nullptr);
    };
    cudaError_t e = part(0, r0);
    if (e != cudaSuccess) return e;
    e = launch_attend_share(cs, r0, r1, q, q_row_stride, k_cache, v_cache, cap, selection, out, out_f32, lse, stream);
    if (e != cudaSuccess) return e;
    return part(r1, cs.n);
  }
  return launch_attend_rows(g, cs, q, q_row_stride, k_cache, v_cache, cap, selection, out, out_f32, lse, p_split,
                            stream, tree);
}

static cudaError_t launch_attend_rows(const infllm2_geometry& g, const CallShape& cs, const void* q,
                                     int64_t q_row_stride, const void* k_cache, const void* v_cache, int64_t cap,
                                     const int32_t* selection, void* out, int out_f32, float* lse, int p_split,
                                     cudaStream_t stream, const TreeArgs* tree) {
  Params p;
  p.n = cs.n;
  p.start = cs.start;
  p.hq = cs.hq;
  p.hkv = cs.hkv;
  p.max_sel = cs.max_sel;
  p.out_f32 = out_f32;
  p.sel = selection;
  p.out = out;
  p.lse = lse;
  p.kv_maps = nullptr;
  p.map_stride = 0;
  p.seq_len = nullptr;
  p.bcast = cs.bcast;
  p.split = 0;
  p.p_split = p_split;
  p.group_major = group_major_enabled();
  p.parts = 1;
  p.part_o = nullptr;
  p.part_ml = nullptr;
  p.tree_words = tree ? tree->words : nullptr;
  p.tree_n = tree ? tree->n : 0;
  p.tree_nw = tree ? tree->words_per_row : 0;
  p.tree_row0 = tree ? tree->row0 : 0;
  if (cs.group == 8 && cs.d == 64) return launch_attend_prefill<8, 64>(cs, q, q_row_stride, k_cache, v_cache, cap, p, stream);
  return launch_attend_prefill<16, 128>(cs, q, q_row_stride, k_cache, v_cache, cap, p, stream);
}

}  // namespace infllm2

extern "C" int infllm2_debug_attend_cycles(long long* host, int max_entries) {
#ifdef ATT_PROFILE
  const int n = max_entries < 160 * 16 ? max_entries : 160 * 16;
  return cudaMemcpyFromSymbol(host, infllm2::g_att_cyc, sizeof(long long) * n) == cudaSuccess ? 0 : -1;
#else
  for (int i = 0; i < max_entries; ++i) host[i] = 0;
  return 1;   // not a profiling build
#endif
}
