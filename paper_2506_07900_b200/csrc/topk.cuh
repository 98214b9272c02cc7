// Warp-level block selection shared by the prefill and decode stage-1 kernels:
// forced blocks (force_blocks, sparse.py:218-227) plus the `budget` best
// candidates by (score desc, id asc) (select_topk, sparse.py:247-277).
#pragma once

#include <limits.h>
#include <stdint.h>

namespace infllm2 {
namespace topk {

constexpr int kListCap = 352;     // per-warp threshold-compaction list (+ staging tail)
constexpr int kOutCap = 96;

__device__ __forceinline__ bool better(float ra, int ba, float rb, int bb) {
  return ra > rb || (ra == rb && ba < bb);   // (score desc, id asc), sparse.py:273
}

// Forced set / budget of a unit (all 16 rows share it): force_blocks
// (sparse.py:218-227) and the budget rule of select_topk (sparse.py:268).
struct UnitSel {
  int64_t qb, n_cand, n_init, local_lo, budget, n_free;
};
__device__ __forceinline__ UnitSel unit_sel(int64_t pos, int m, int top_k, int n_init_cfg, int n_local,
                                            int consume) {
  UnitSel u;
  u.qb = pos / m;
  u.n_cand = u.qb + 1;
  u.n_init = n_init_cfg < u.n_cand ? n_init_cfg : u.n_cand;
  u.local_lo = u.qb + 1;
  if (n_local > 0) {
    u.local_lo = u.qb - n_local + 1;
    if (u.local_lo < 0) u.local_lo = 0;
    if (u.local_lo < u.n_init) u.local_lo = u.n_init;
  }
  const int64_t n_forced = u.n_init + (u.qb + 1 - u.local_lo);
  u.budget = top_k;
  if (consume) u.budget = top_k - n_forced > 0 ? top_k - n_forced : 0;
  u.n_free = u.n_cand - n_forced;
  return u;
}

// Warp bitonic sort of one value per lane: descending floats / ascending ints.
__device__ __forceinline__ float warp_sort_desc(float x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const float y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool keep_max = (((lane & k) == 0) == ((lane & j) == 0));
      x = keep_max ? fmaxf(x, y) : fminf(x, y);
    }
  return x;
}
__device__ __forceinline__ int warp_sort_asc(int x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool keep_min = (((lane & k) == 0) == ((lane & j) == 0));
      x = keep_min ? min(x, y) : max(x, y);
    }
  return x;
}

// Warp argmax over (score desc, id asc) strictly after (prev_v, prev_b) in that order.
__device__ __forceinline__ void warp_best_after(float& bv, int& bb) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int ob = __shfl_xor_sync(0xffffffffu, bb, off);
    if (ob >= 0 && (bb < 0 || better(ov, ob, bv, bb))) { bv = ov; bb = ob; }
  }
}

// One query's selection by one warp: forced init blocks, the `budget` best
// candidates of rq[n_init, local_lo) by (score desc, id asc), forced local
// blocks; written ascending with -1 padding (select_topk, sparse.py:247-277).
// Fast path (budget <= 64): threshold T0 = budget-th largest of the lanes' top
// K values (K = 1 / 2 / 4 for budget <= 16 / 32 / 64) -- at least `budget`
// candidates reach it, so the answer lies in {r >= T0} -- compact that set in
// id order, rank it exactly, and the ballot-compacted survivors come out
// ascending.  Iterative order statistics only when the set overflows the list
// (massive exact ties) or budget > 64.
__device__ __forceinline__ void warp_select(const float* rq, const UnitSel& u, int lane, float* lkey, int* lid, int32_t* out,
                            double* osc, int max_sel) {
  const int lo = (int)u.n_init, hi = (int)u.local_lo;
  const int budget = (int)u.budget;
  int chosen0 = INT_MAX, chosen1 = INT_MAX;   // lane x holds the x-th / (32+x)-th chosen id
  bool fast = false;
  if (budget >= u.n_free) {
    // dense regime: every candidate is selected (assembled below)
  } else if (budget > 0 && budget <= 64) {
    // each lane keeps its K largest values, K = 1 / 2 / 4 for budget <= 16 /
    // 32 / 64, so T0 (the budget-th largest of those 32K values) sits about
    // halfway down their sorted order: a tight threshold, ~budget survivors
    float m[4] = {-1.f, -1.f, -1.f, -1.f};
    const int K = budget <= 16 ? 1 : budget <= 32 ? 2 : 4;
    for (int b = lo + lane; b < hi; b += 32) {
      const float a = rq[b];
      if (a > m[3]) {
        if (a > m[0]) { m[3] = m[2]; m[2] = m[1]; m[1] = m[0]; m[0] = a; }
        else if (a > m[1]) { m[3] = m[2]; m[2] = m[1]; m[1] = a; }
        else if (a > m[2]) { m[3] = m[2]; m[2] = a; }
        else m[3] = a;
      }
    }
    float t0;
    if (K == 1) {
      t0 = __shfl_sync(0xffffffffu, warp_sort_desc(m[0], lane), budget - 1);
    } else {
      // budget-th largest of the 32K values: count values above / at least each of mine
      int gt[4] = {0, 0, 0, 0}, ge[4] = {0, 0, 0, 0};
      for (int x = 0; x < 32; ++x) {
        float a[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = __shfl_sync(0xffffffffu, m[j], x);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (j < K) {
              gt[i] += a[j] > m[i];
              ge[i] += a[j] >= m[i];
            }
          }
      }
      t0 = -1.f;
      bool done = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool hit = i < K && gt[i] < budget && ge[i] >= budget;
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (!done && bal) {
          t0 = __shfl_sync(0xffffffffu, m[i], __ffs(bal) - 1);
          done = true;
        }
      }
    }
    int cnt = 0;
    for (int base = lo; base < hi; base += 128) {
      float r4[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int b = base + 32 * x + lane;
        r4[x] = b < hi ? rq[b] : -2.f;
      }
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int b = base + 32 * x + lane;
        const bool f = r4[x] >= t0;
        const unsigned mask = __ballot_sync(0xffffffffu, f);
        const int pos = cnt + __popc(mask & ((1u << lane) - 1u));
        if (f && pos < kListCap - kOutCap) { lkey[pos] = r4[x]; lid[pos] = b; }
        cnt += __popc(mask);
      }
    }
    __syncwarp();
    if (cnt <= kListCap - kOutCap) {
      // rank every listed candidate against the whole list (no dependent
      // chains), keep rank < budget; the list is in id order, so a ballot
      // compaction emits the chosen ids already ascending.
      int taken = 0;
      for (int base = 0; base < cnt; base += 32) {
        const int x = base + lane;
        bool keep = false;
        if (x < cnt) {
          const float rk = lkey[x];
          const int bk = lid[x];
          int rank = 0;
#pragma unroll 4
          for (int f = 0; f < cnt; ++f) rank += better(lkey[f], lid[f], rk, bk) ? 1 : 0;
          keep = rank < budget;
        }
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        const int pos = taken + __popc(mask & ((1u << lane) - 1u));
        if (keep) lid[kListCap - kOutCap + pos] = lid[x];   // staging area at the list tail
        taken += __popc(mask);
      }
      __syncwarp();
      chosen0 = lane < budget ? lid[kListCap - kOutCap + lane] : INT_MAX;
      chosen1 = lane + 32 < budget ? lid[kListCap - kOutCap + 32 + lane] : INT_MAX;
      __syncwarp();
      fast = true;
    }
  }
  if (budget < u.n_free && budget > 0 && !fast) {
    // rare: iterative order statistics over the whole range (massive ties or budget > 64)
    float pv = INFINITY;
    int pb = -1;
    for (int it = 0; it < budget; ++it) {
      float bv = -1.f;
      int bb = -1;
      for (int b = lo + lane; b < hi; b += 32) {
        const float r = rq[b];
        if ((pb < 0 || better(pv, pb, r, b)) && (bb < 0 || better(r, b, bv, bb))) { bv = r; bb = b; }
      }
      warp_best_after(bv, bb);
      if (lane == 0) lid[it] = bb;  // staged in smem, sorted below
      pv = bv;
      pb = bb;
    }
    __syncwarp();
    // insertion-free ascending order: ids are distinct, rank = #smaller
    for (int x = lane; x < budget; x += 32) {
      const int me = lid[x];
      int rank = 0;
      for (int y = 0; y < budget; ++y) rank += lid[y] < me;
      lkey[rank] = __int_as_float(me);
    }
    __syncwarp();
  }
  // assemble: [0, lo) + chosen + [local_lo, qb]
  const int n_ch = budget >= u.n_free ? (int)u.n_free : budget;
  const int n_loc = (int)(u.qb + 1 - u.local_lo);
  for (int x = lane; x < max_sel; x += 32) {
    int id = -1;
    if (x < lo) id = x;
    else if (x < lo + n_ch) {
      const int c = x - lo;
      if (budget >= u.n_free) id = lo + c;
      else if (fast) id = -2;  // filled from registers below
      else id = __float_as_int(lkey[c]);
    } else if (x < lo + n_ch + n_loc) id = (int)u.local_lo + (x - lo - n_ch);
    if (id != -2) {
      out[x] = id;
      if (osc) osc[x] = id >= 0 ? (double)rq[id] : 0.0;
    }
  }
  if (fast) {
    if (lane < budget) {
      out[lo + lane] = chosen0;
      if (osc) osc[lo + lane] = (double)rq[chosen0];
    }
    if (lane + 32 < budget) {
      out[lo + 32 + lane] = chosen1;
      if (osc) osc[lo + 32 + lane] = (double)rq[chosen1];
    }
  }
}


}  // namespace topk
}  // namespace infllm2
