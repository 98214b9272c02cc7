// Stage-2 prefill attention, two-team tcgen05 pipeline.
//
// Same math as attend_tc.cu (sparse_attend, sparse.py:347-384): per (query
// row, KV group) item, TMA gathers the selected 64-row blocks two at a time,
// S^T = K_tile . Q^T and O^T += V_tile^T . P^T on the tensor cores (P split
// into bf16 hi + lo), softmax in float32 with an exact first-tile max.
//
// The single-team kernel alternates MMA -> softmax -> MMA on one item, so the
// tensor pipe idles while the softmax warps work and vice versa (ncu: softmax
// warps waited 38 % of their time for S).  Here two softmax teams own
// alternate items of the CTA's work list; the MMA issuer walks both items'
// tiles interleaved and keeps a two-deep FIFO of issued QK's, issuing each PV
// only after the next QK — so team A's softmax overlaps team B's MMAs.
//
// Warps: 0 = TMA producer, 1 = TMEM alloc + MMA issuer, 2..5 = team 0,
// 6..9 = team 1 (softmax + the item's epilogue).  TMEM (128 columns): per team
// two 16-column S slots and two 16-column O buffers.
#include <float.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tc_dispatch.cuh"

namespace infllm2 {

bool tc_kernels_enabled();

namespace {

using namespace sm100;

constexpr int kG = 16;
constexpr int kD = 128;
constexpr int kM = 64;
constexpr int kRowsT = 128;
constexpr int kStages = 3;
constexpr int kThreads = 320;
constexpr int kMaxSel = 80;

constexpr uint32_t kHalfBytes = kRowsT * 128;       // 16 KB
constexpr uint32_t kTileBytes = 2 * kHalfBytes;     // 32 KB (K or V)
constexpr uint32_t kStageBytes = 2 * kTileBytes;    // 64 KB
constexpr uint32_t kQBytes = 2 * kG * 128;          // 4 KB
constexpr uint32_t kPHalf = kRowsT * kG * 2;        // 4 KB
constexpr uint32_t kPBytes = 2 * kPHalf;            // hi + lo

struct Smem {
  static constexpr uint32_t kv = 0;
  static constexpr uint32_t q = kv + kStages * kStageBytes;       // [2 teams]
  static constexpr uint32_t p = q + 2 * kQBytes;                  // [2 teams]
  static constexpr uint32_t red = p + 2 * kPBytes;                // [2 teams][4][16]
  static constexpr uint32_t lsum = red + 2 * 64 * 4;              // [2 teams][4][16]
  static constexpr uint32_t bars = lsum + 2 * 64 * 4;
  static constexpr uint32_t total = bars + 40 * 8;
};

struct Params {
  int64_t n, start;
  int hq, hkv, max_sel, out_f32;
  const int32_t* sel;
  void* out;
  float* lse;
};

struct SelRow {
  int r0, r1, r2;
  int nb;
  __device__ __forceinline__ int get(int j) const {
    const int v = j < 32 ? r0 : (j < 64 ? r1 : r2);
    return __shfl_sync(0xffffffffu, v, j & 31);
  }
};

__device__ __forceinline__ SelRow load_sel(const Params& p, int64_t item, int64_t pos, int lane) {
  const int32_t* s = p.sel + item * p.max_sel;
  SelRow r;
  r.r0 = lane < p.max_sel ? s[lane] : -1;
  r.r1 = lane + 32 < p.max_sel ? s[lane + 32] : -1;
  r.r2 = lane + 64 < p.max_sel ? s[lane + 64] : -1;
  auto ok = [&](int b) { return b >= 0 && (int64_t)b * kM <= pos; };
  r.nb = __popc(__ballot_sync(0xffffffffu, ok(r.r0))) + __popc(__ballot_sync(0xffffffffu, ok(r.r1))) +
         __popc(__ballot_sync(0xffffffffu, ok(r.r2)));
  return r;
}

// One team's item stream: items k = team, team+2, ... of this CTA's list.
struct Stream {
  int64_t k;        // index in the CTA's work list
  int64_t item;
  int c, tiles;
  bool done;
  SelRow sr;
  int grp;
  int64_t i, pos;
};

__device__ __forceinline__ void stream_load(const Params& p, Stream& s, int lane) {
  const int64_t items = p.n * p.hkv;
  s.item = blockIdx.x + s.k * gridDim.x;
  s.done = s.item >= items;
  s.c = 0;
  if (s.done) return;
  s.i = s.item / p.hkv;
  s.grp = (int)(s.item - s.i * p.hkv);
  s.pos = p.start + s.i;
  s.sr = load_sel(p, s.item, s.pos, lane);
  s.tiles = (s.sr.nb + 1) / 2;
}

// Walks both streams' tiles interleaved (A, B, A, B, ...; one stream alone when
// the other is exhausted).  Producer and MMA issuer run the same walk.
struct Walker {
  Stream st[2];
  int cur;
  int nitems[2];    // items started per team (for buffer parities)
  __device__ __forceinline__ void init(const Params& p, int lane) {
    for (int t = 0; t < 2; ++t) {
      st[t].k = t;
      stream_load(p, st[t], lane);
      nitems[t] = 0;
    }
    cur = 0;
  }
  // next tile: returns false when both streams are exhausted
  __device__ __forceinline__ bool next(int* team) {
    if (st[cur].done) cur ^= 1;
    if (st[cur].done) return false;
    *team = cur;
    return true;
  }
  __device__ __forceinline__ void advance(const Params& p, int lane) {
    Stream& s = st[cur];
    if (++s.c == s.tiles) {
      s.k += 2;
      ++nitems[cur];
      stream_load(p, s, lane);
    }
    if (!st[cur ^ 1].done) cur ^= 1;
  }
};

__global__ void __launch_bounds__(kThreads, 1)
attend_tc2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* kv_full = bars;            // [3]
  uint64_t* kv_empty = bars + 3;       // [3]
  uint64_t* q_full = bars + 6;         // [team]
  uint64_t* q_empty = bars + 8;        // [team]
  uint64_t* s_full = bars + 10;        // [team][slot]
  uint64_t* s_empty = bars + 14;       // [team][slot]
  uint64_t* p_full = bars + 18;        // [team]
  uint64_t* p_empty = bars + 20;       // [team]
  uint64_t* o_full = bars + 22;        // [team][buf]
  uint64_t* o_empty = bars + 26;       // [team][buf]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
    for (int t = 0; t < 2; ++t) {
      mbar_init(q_full + t, 1);
      mbar_init(q_empty + t, 1);
      mbar_init(p_full + t, 4);
      mbar_init(p_empty + t, 1);
      for (int x = 0; x < 2; ++x) {
        mbar_init(s_full + 2 * t + x, 1);
        mbar_init(s_empty + 2 * t + x, 4);
        mbar_init(o_full + 2 * t + x, 1);
        mbar_init(o_empty + 2 * t + x, 4);
      }
    }
    fence_barrier_init();
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto s_col = [&](int t, int slot) { return tmem + t * 64 + slot * kG; };
  auto o_col = [&](int t, int buf) { return tmem + t * 64 + 32 + buf * kG; };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    Walker wk;
    wk.init(p, lane);
    int stage = 0;
    uint32_t phase = 0;
    int team;
    while (wk.next(&team)) {
      Stream& s = wk.st[team];
      const int c = s.c;
      const int nt = (s.sr.nb - 2 * c) >= 2 ? 2 : 1;
      const int b0 = s.sr.get(2 * c), b1 = s.sr.get(2 * c + 1 < 96 ? 2 * c + 1 : 95);
      if (lane == 0) {
        if (c == 0) {
          mbar_wait(q_empty + team, (wk.nitems[team] & 1) ^ 1);
          mbar_arrive_expect_tx(q_full + team, kQBytes);
          uint8_t* qd = smem + Smem::q + team * kQBytes;
          tma_load_3d(qd, &tm_q, q_full + team, 0, s.grp * kG, (int)s.i);
          tma_load_3d(qd + kQBytes / 2, &tm_q, q_full + team, 64, s.grp * kG, (int)s.i);
        }
        mbar_wait(kv_empty + stage, phase ^ 1);
        mbar_arrive_expect_tx(kv_full + stage, nt * 4 * (kM * 128));
        uint8_t* kd = smem + Smem::kv + stage * kStageBytes;
        uint8_t* vd = kd + kTileBytes;
        for (int x = 0; x < nt; ++x) {
          const int row0 = (x ? b1 : b0) * kM;
          const uint32_t off = x * kM * 128;
          tma_load_3d(kd + off, &tm_k, kv_full + stage, 0, row0, s.grp);
          tma_load_3d(kd + kHalfBytes + off, &tm_k, kv_full + stage, 64, row0, s.grp);
          tma_load_3d(vd + off, &tm_v, kv_full + stage, 0, row0, s.grp);
          tma_load_3d(vd + kHalfBytes + off, &tm_v, kv_full + stage, 64, row0, s.grp);
        }
      }
      __syncwarp();
      if (++stage == kStages) { stage = 0; phase ^= 1; }
      wk.advance(p, lane);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc_qk = idesc_bf16_f32(128, kG);
    const uint32_t idesc_pv = idesc_bf16_f32_major(128, kG, 1, 1);
    Walker wk;
    wk.init(p, lane);
    int stage = 0;
    uint32_t phase = 0;
    int sslot[2] = {0, 0};
    uint32_t s_ph[2][2] = {{0, 0}, {0, 0}};
    uint32_t p_ph[2] = {0, 0};
    // FIFO of issued QK's awaiting their PV (depth <= 2)
    struct Pend { int team, stage, ksteps, first, last, buf, nbuf_par; };
    Pend fifo[2];
    int nf = 0;
    auto issue_pv = [&](const Pend& y) {
      mbar_wait(p_full + y.team, p_ph[y.team]);
      p_ph[y.team] ^= 1;
      if (y.first) mbar_wait(o_empty + 2 * y.team + y.buf, y.nbuf_par ^ 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t v_addr = smem_u32(smem + Smem::kv + y.stage * kStageBytes + kTileBytes);
        const uint32_t p_addr = smem_u32(smem + Smem::p + y.team * kPBytes);
        for (int k = 0; k < y.ksteps; ++k) {
          const uint64_t vdesc = sdesc_mn_sw128(v_addr + k * 2048, kHalfBytes, 1024);
          umma_f16_ss(o_col(y.team, y.buf), vdesc, sdesc_interleave(p_addr + k * 512, 256, 128), idesc_pv,
                      (!y.first || k > 0) ? 1u : 0u);
          umma_f16_ss(o_col(y.team, y.buf), vdesc, sdesc_interleave(p_addr + kPHalf + k * 512, 256, 128), idesc_pv,
                      1u);
        }
        umma_commit(kv_empty + y.stage);
        umma_commit(p_empty + y.team);
        if (y.last) umma_commit(o_full + 2 * y.team + y.buf);
      }
      __syncwarp();
    };
    int team;
    while (wk.next(&team)) {
      Stream& s = wk.st[team];
      const int c = s.c;
      const int item_no = wk.nitems[team];     // items of this team started before
      if (c == 0) mbar_wait(q_full + team, item_no & 1);
      mbar_wait(kv_full + stage, phase);
      const int slot = sslot[team];
      mbar_wait(s_empty + 2 * team + slot, s_ph[team][slot] ^ 1);
      s_ph[team][slot] ^= 1;
      tc_fence_after();
      if (elect_one()) {
        const uint32_t k_addr = smem_u32(smem + Smem::kv + stage * kStageBytes);
        const uint32_t q_addr = smem_u32(smem + Smem::q + team * kQBytes);
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t off = (k >> 2) * kHalfBytes + (k & 3) * 32;
          const uint32_t qoff = (k >> 2) * (kQBytes / 2) + (k & 3) * 32;
          umma_f16_ss(s_col(team, slot), sdesc_k_sw128(k_addr + off), sdesc_k_sw128(q_addr + qoff), idesc_qk,
                      k > 0 ? 1u : 0u);
        }
        umma_commit(s_full + 2 * team + slot);
        if (c == s.tiles - 1) umma_commit(q_empty + team);
      }
      __syncwarp();
      sslot[team] ^= 1;
      Pend x;
      x.team = team;
      x.stage = stage;
      x.ksteps = (s.sr.nb - 2 * c) >= 2 ? 8 : 4;
      x.first = (c == 0);
      x.last = (c == s.tiles - 1);
      x.buf = item_no & 1;
      x.nbuf_par = (item_no >> 1) & 1;
      if (nf == 2) {
        issue_pv(fifo[0]);
        fifo[0] = fifo[1];
        nf = 1;
      }
      fifo[nf++] = x;
      if (nf == 2) {
        issue_pv(fifo[0]);
        fifo[0] = fifo[1];
        nf = 1;
      }
      if (++stage == kStages) { stage = 0; phase ^= 1; }
      wk.advance(p, lane);
    }
    for (int x = 0; x < nf; ++x) issue_pv(fifo[x]);
  } else {
    // ------------------------------------------------------------ softmax teams
    const int team = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;        // tile row == TMEM lane (and O^T d lane)
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const float c2 = 1.4426950408889634f / sqrtf((float)kD);
    float* red = reinterpret_cast<float*>(smem + Smem::red) + team * 64;
    float* lred = reinterpret_cast<float*>(smem + Smem::lsum) + team * 64;
    const uint32_t bar_id = 2 + team;
    int slot = 0;
    uint32_t s_ph[2] = {0, 0};
    uint32_t p_ph = 0;
    int item_no = 0;
    Stream s;
    s.k = team;
    for (stream_load(p, s, lane); !s.done; s.k += 2, stream_load(p, s, lane), ++item_no) {
      float mrun[kG], lsum[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h) { mrun[h] = -INFINITY; lsum[h] = 0.f; }
      const int buf = item_no & 1;
      for (int c = 0; c < s.tiles; ++c) {
        mbar_wait(s_full + 2 * team + slot, s_ph[slot]);
        s_ph[slot] ^= 1;
        tc_fence_after();
        float z[kG];
        tmem_ld16(s_col(team, slot) + lane_base, z);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + 2 * team + slot);
        slot ^= 1;
        const int x = row >> 6;
        const int b0 = s.sr.get(2 * c), b1 = s.sr.get(2 * c + 1 < 96 ? 2 * c + 1 : 95);
        bool valid = (2 * c + x) < s.sr.nb;
        if (valid) valid = (int64_t)(x ? b1 : b0) * kM + (row & 63) <= s.pos;
#pragma unroll
        for (int h = 0; h < kG; ++h) z[h] = valid ? z[h] * c2 : -INFINITY;
        bool need = (c == 0);
        if (c > 0) {
          bool over = false;
#pragma unroll
          for (int h = 0; h < kG; ++h) over |= z[h] > mrun[h] + 8.f;
          const unsigned any = __ballot_sync(0xffffffffu, over);
          if (lane == 0) red[quad * 16] = any ? 1.f : 0.f;
          named_bar_sync(bar_id, 128);
          need = (red[0] + red[16] + red[32] + red[48]) > 0.f;
          named_bar_sync(bar_id, 128);
        }
        // the previous PV of this team must be done before P (single buffer)
        // is rewritten or O is rescaled
        mbar_wait(p_empty + team, p_ph ^ 1);
        p_ph ^= 1;
        if (need) {
          float tmax[kG];
#pragma unroll
          for (int h = 0; h < kG; ++h) {
            float v = z[h];
            for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
            tmax[h] = v;
          }
          if (lane < kG) {
            float mine = tmax[0];
#pragma unroll
            for (int h = 1; h < kG; ++h) mine = (lane == h) ? tmax[h] : mine;
            red[quad * 16 + lane] = mine;
          }
          named_bar_sync(bar_id, 128);
          float corr[kG];
          bool any_corr = false;
#pragma unroll
          for (int h = 0; h < kG; ++h) {
            const float tm = fmaxf(fmaxf(red[h], red[16 + h]), fmaxf(red[32 + h], red[48 + h]));
            const float mnew = fmaxf(mrun[h], tm);
            corr[h] = (mrun[h] == -INFINITY) ? 1.f : ex2(mrun[h] - mnew);
            any_corr |= (c > 0) && (corr[h] != 1.f);
            lsum[h] *= (mrun[h] == -INFINITY) ? 0.f : corr[h];
            mrun[h] = mnew;
          }
          named_bar_sync(bar_id, 128);
          if (any_corr) {
            tc_fence_after();
            float o[kG];
            tmem_ld16(o_col(team, buf) + lane_base, o);
            tmem_wait_ld();
#pragma unroll
            for (int h = 0; h < kG; ++h) o[h] *= corr[h];
            tmem_st16(o_col(team, buf) + lane_base, o);
            tmem_wait_st();
            tc_fence_before();
          }
        }
        uint32_t phi[kG / 2], plo[kG / 2];
#pragma unroll
        for (int h = 0; h < kG; h += 2) {
          const float a = ex2(z[h] - mrun[h]);
          const float b = ex2(z[h + 1] - mrun[h + 1]);
          lsum[h] += a;
          lsum[h + 1] += b;
          const __nv_bfloat162 hi2 = __floats2bfloat162_rn(a, b);
          const __nv_bfloat162 lo2 = __floats2bfloat162_rn(a - __low2float(hi2), b - __high2float(hi2));
          phi[h / 2] = *reinterpret_cast<const uint32_t*>(&hi2);
          plo[h / 2] = *reinterpret_cast<const uint32_t*>(&lo2);
        }
        uint8_t* pb = smem + Smem::p + team * kPBytes;
        const uint32_t base = (row >> 3) * 256 + (row & 7) * 16;
        *reinterpret_cast<uint4*>(pb + base) = make_uint4(phi[0], phi[1], phi[2], phi[3]);
        *reinterpret_cast<uint4*>(pb + base + 128) = make_uint4(phi[4], phi[5], phi[6], phi[7]);
        *reinterpret_cast<uint4*>(pb + kPHalf + base) = make_uint4(plo[0], plo[1], plo[2], plo[3]);
        *reinterpret_cast<uint4*>(pb + kPHalf + base + 128) = make_uint4(plo[4], plo[5], plo[6], plo[7]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full + team);
      }
      // ---- epilogue of the item: row sums across the team, normalise O
#pragma unroll
      for (int h = 0; h < kG; ++h) {
        float v = lsum[h];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) lred[quad * 16 + h] = v;
      }
      named_bar_sync(bar_id, 128);
      float l[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h) l[h] = lred[h] + lred[16 + h] + lred[32 + h] + lred[48 + h];
      mbar_wait(o_full + 2 * team + buf, (item_no >> 1) & 1);
      tc_fence_after();
      float o[kG];
      tmem_ld16(o_col(team, buf) + lane_base, o);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty + 2 * team + buf);
      const int d = row;
      const int64_t obase = (s.i * p.hq + (int64_t)s.grp * kG) * kD + d;
      if (p.out_f32) {
        float* out = static_cast<float*>(p.out);
#pragma unroll
        for (int h = 0; h < kG; ++h) out[obase + h * kD] = o[h] / l[h];
      } else {
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
#pragma unroll
        for (int h = 0; h < kG; ++h) out[obase + h * kD] = __float2bfloat16_rn(o[h] / l[h]);
      }
      if (p.lse && quad == 0 && lane < kG) {
        float lh = l[0], mh = mrun[0];
#pragma unroll
        for (int h = 1; h < kG; ++h) {
          lh = (lane == h) ? l[h] : lh;
          mh = (lane == h) ? mrun[h] : mh;
        }
        p.lse[s.i * p.hq + s.grp * kG + lane] = (mh + log2f(lh)) * 0.6931471805599453f;
      }
      named_bar_sync(bar_id, 128);     // lred reuse by the next item
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<128>(tmem);
}

}  // namespace

cudaError_t launch_attend_tc2(const CallShape& cs, const void* q, int64_t q_row_stride, const void* k_cache,
                              const void* v_cache, int64_t cap, const int32_t* selection, void* out, int out_f32,
                              float* lse, cudaStream_t stream) {
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
  CUtensorMap tq, tk, tv;
  {
    const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)cs.hq, (uint64_t)cs.n};
    const uint64_t strides[2] = {(uint64_t)kD * 2, (uint64_t)q_row_stride * 2};
    const uint32_t box[3] = {64, (uint32_t)kG, 1};
    if (!encode_tmap_3d_bf16(&tq, q, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)cs.cache_len, (uint64_t)cs.hkv};
    const uint64_t strides[2] = {(uint64_t)kD * 2, (uint64_t)cap * kD * 2};
    const uint32_t box[3] = {64, (uint32_t)kM, 1};
    if (!encode_tmap_3d_bf16(&tk, k_cache, dims, strides, box)) return cudaErrorInvalidValue;
    if (!encode_tmap_3d_bf16(&tv, v_cache, dims, strides, box)) return cudaErrorInvalidValue;
  }
  const size_t smem = Smem::total + 1024;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attend_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = cs.n * cs.hkv;
  const int grid = (int)(items < sms ? items : sms);
  count_launch();
  attend_tc2_kernel<<<grid, kThreads, smem, stream>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace infllm2
