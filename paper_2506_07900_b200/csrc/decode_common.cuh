// Device-side decode table shared by the five-launch decode path (decode.cu)
// and the fused single-launch path (decode_fused.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"

namespace infllm2 {
namespace dec {

constexpr int kMaps = 4;           // per sequence: K, V, hi, lo
constexpr int kMaxHkv = 8;
constexpr int kP = 32;             // kernel size (decode geometry)

// Device-side table: [n_seq] descriptors, [n_seq][4] tensor maps, [n_seq]
// lengths, [n_seq][8] legacy counters, [n_seq*8][4] fused-path counters + 1.
struct SeqDesc {
  __nv_bfloat16* k;
  __nv_bfloat16* v;
  int64_t cap;
  float* fine;
  __nv_bfloat16* hi;
  __nv_bfloat16* lo;
  int64_t means_cap;
  float* coarse;
  int64_t coarse_cap;
};

struct TableView {
  const SeqDesc* desc;
  const CUtensorMap* maps;
  int64_t* len;        // OLD length during a step; bumped by the last kernel
  int* counters;       // [n_seq][8] last-CTA-done counters of the scores kernel
  int* fused;          // [n_seq*kMaxHkv][4] per-segment counters, then the CTA-done counter
  void** next;         // the next layer's table (same sequences), or null: L2 prefetch target
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline TableView table_view(void* base, int n_seq) {
  uint8_t* b = static_cast<uint8_t*>(base);
  TableView t;
  const size_t maps_off = align_up(sizeof(SeqDesc) * n_seq, 128);
  const size_t len_off = maps_off + sizeof(CUtensorMap) * kMaps * n_seq;
  t.desc = reinterpret_cast<const SeqDesc*>(b);
  t.maps = reinterpret_cast<const CUtensorMap*>(b + maps_off);
  t.len = reinterpret_cast<int64_t*>(b + len_off);
  t.counters = reinterpret_cast<int*>(b + len_off + sizeof(int64_t) * n_seq);
  t.fused = t.counters + kMaxHkv * n_seq;
  const size_t next_off = align_up(len_off + sizeof(int64_t) * n_seq + sizeof(int) * kMaxHkv * n_seq +
                                       sizeof(int) * (4 * kMaxHkv * n_seq + 4), 16);
  t.next = reinterpret_cast<void**>(b + next_off);
  return t;
}

inline size_t table_bytes(int n_seq) {
  return align_up(sizeof(SeqDesc) * n_seq, 128) + sizeof(CUtensorMap) * kMaps * n_seq + sizeof(int64_t) * n_seq +
         sizeof(int) * kMaxHkv * n_seq + sizeof(int) * (4 * kMaxHkv * n_seq + 4) + 32;
}

// Window mean over the cache rows, with row `new_row` taken from `knew` (the
// token being appended in this step) so no CTA waits for the cache write.
__device__ __forceinline__ float window_mean(const __nv_bfloat16* kg, int d, int64_t j, int stride, int64_t length,
                                             int e, int64_t new_row, float knew) {
  const int64_t r0 = j * stride;
  int64_t r1 = r0 + kP;
  if (r1 > length) r1 = length;
  const int w = (int)(r1 - r0);
  float x[kP];
#pragma unroll
  for (int r = 0; r < kP; ++r)   // all loads in flight together
    x[r] = r < w ? (r0 + r == new_row ? knew : __bfloat162float(__ldg(&kg[(r0 + r) * d + e]))) : 0.f;
  double acc = (double)x[0];
#pragma unroll
  for (int r = 1; r < kP; ++r)
    if (r < w) acc += (double)x[r];   // sequential, as numpy's reduce
  return __double2float_rn(acc / (double)w);
}


}  // namespace dec
}  // namespace infllm2
