// TMA gather micro-benchmark: per-SM throughput of the stage-2 K/V block
// gather (random 64-row blocks of a 128K x 128 bf16 cache, two blocks per
// 64 KB "tile") for several tensor-map box shapes, no compute.
//   mode 0: 4 boxes {64 d, 64 rows} per block (128B swizzle)  [attend_tc today]
//   mode 1: 2 boxes {64 d, 64 rows, 2 halves} per block (3-D, 128B swizzle)
//   mode 2: 2 boxes {128 d, 64 rows} per block (no swizzle, 256 B inner)
//   mode 3: 4 boxes {64 d, 128 rows}: 2 CONSECUTIVE blocks per box (upper bound: contiguous)
// Usage: tma_bench <mode> <stages> [ctas]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su(dst)), "l"(m), "r"(su(b)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(su(dst)), "l"(m), "r"(su(b)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

constexpr uint32_t kTile = 65536;

__global__ void __launch_bounds__(64, 1) gather(const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv,
                                               const int* blocks, int tiles_per_cta, int mode, int stages) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[8], empty[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { bar_init(full + i, 1); bar_init(empty + i, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int* bl = blocks + (size_t)blockIdx.x * tiles_per_cta * 2;
  const uint32_t stage_bytes = kTile;
  if (threadIdx.x == 0) {
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int st = t % stages;
      const uint32_t ph = (t / stages) & 1;
      bar_wait(empty + st, ph ^ 1);
      bar_expect(full + st, kTile);
      uint8_t* kd = s + st * stage_bytes;
      uint8_t* vd = kd + kTile / 2;
      for (int x = 0; x < 2; ++x) {
        const int row0 = bl[2 * t + x] * 64;
        const uint32_t off = x * 8192;
        if (mode == 0) {
          tma2(kd + off, &mk, full + st, 0, row0);
          tma2(kd + 16384 + off, &mk, full + st, 64, row0);
          tma2(vd + off, &mv, full + st, 0, row0);
          tma2(vd + 16384 + off, &mv, full + st, 64, row0);
        } else if (mode == 1) {
          tma3(kd + off * 2, &mk, full + st, 0, row0, 0);
          tma3(vd + off * 2, &mv, full + st, 0, row0, 0);
        } else if (mode == 2) {
          tma2(kd + off * 2, &mk, full + st, 0, row0);
          tma2(vd + off * 2, &mv, full + st, 0, row0);
        }
      }
      if (mode == 3) {
        const int row0 = bl[2 * t] * 64;
        tma2(kd, &mk, full + st, 0, row0);
        tma2(kd + 16384, &mk, full + st, 64, row0);
        tma2(vd, &mv, full + st, 0, row0);
        tma2(vd + 16384, &mv, full + st, 64, row0);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int st = t % stages;
      bar_wait(full + st, (t / stages) & 1);
      bar_arrive(empty + st);
    }
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int stages = argc > 2 ? atoi(argv[2]) : 3;
  int ctas = argc > 3 ? atoi(argv[3]) : 148;
  const int tiles = 2000;
  const size_t rows = 131072, d = 128;
  void *k, *v;
  CK(cudaMalloc(&k, rows * d * 2));
  CK(cudaMalloc(&v, rows * d * 2));
  CK(cudaMemset(k, 0, rows * d * 2));
  CK(cudaMemset(v, 0, rows * d * 2));
  std::vector<int> hb((size_t)ctas * tiles * 2);
  std::mt19937 rng(1);
  for (auto& x : hb) x = rng() % (rows / 64 - 1);
  int* db;
  CK(cudaMalloc(&db, hb.size() * 4));
  CK(cudaMemcpy(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  CUtensorMap mk, mv;
  CUresult r1, r2;
  cuuint32_t es[3] = {1, 1, 1};
  if (mode == 0 || mode == 3) {
    cuuint64_t gd[2] = {d, rows};
    cuuint64_t gs[1] = {d * 2};
    cuuint32_t bx[2] = {64, (cuuint32_t)(mode == 3 ? 128 : 64)};
    r1 = enc(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    r2 = enc(&mv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (mode == 1) {
    cuuint64_t gd[3] = {64, rows, 2};
    cuuint64_t gs[2] = {d * 2, 128};
    cuuint32_t bx[3] = {64, 64, 2};
    r1 = enc(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, k, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    r2 = enc(&mv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, v, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t gd[2] = {d, rows};
    cuuint64_t gs[1] = {d * 2};
    cuuint32_t bx[2] = {128, 64};
    r1 = enc(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    r2 = enc(&mv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) { printf("mode %d: encode failed (%d, %d)\n", mode, (int)r1, (int)r2); return 0; }
  const size_t smem = (size_t)stages * kTile + 1024;
  CK(cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gather<<<ctas, 64, smem>>>(mk, mv, db, 100, mode, stages);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  gather<<<ctas, 64, smem>>>(mk, mv, db, tiles, mode, stages);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)ctas * tiles * kTile;
  printf("mode %d stages %d ctas %d: %.3f ms, %.1f GB/s total, %.1f GB/s per SM\n", mode, stages, ctas, ms,
         bytes / ms / 1e6, bytes / ms / 1e6 / ctas);
  return 0;
}
