// Stage-1 MMA -> epilogue pipeline in isolation: one MMA warp writes 256x128
// fp32 score tiles (32 tcgen05.mma M=128 N=128 K=16 per tile, two interleaved
// accumulators, like select_tc pass 1) into two TMEM buffers; 8 epilogue warps
// run the pass-1 reduction (max, ex2, sums) on each tile.  Handshake with
// mbarriers exactly as the kernel (acc_full / acc_empty).  Prints cycles per
// tile for: mode 0 pipeline, 1 MMA only (epilogue skips math), 2 epilogue only
// (MMA skips issue), 3 pipeline plus a producer streaming 64 KB L2 -> smem per
// tile (the mu stage of the real kernel).
// Usage: pipe_bench <mode>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>

#include "../paper_2506_07900_b200/csrc/sm100.cuh"
using namespace infllm2::sm100;

__global__ void __launch_bounds__(320, 1) pipe(int iters, int mode, long long* out, float* sink, const float* gsrc) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sm = dsm + ((1024u - (smem_u32(dsm) & 1023u)) & 1023u);
  __shared__ uint64_t full[2], empty[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) { mbar_init(full + b, 1); mbar_init(empty + b, 8); }
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (warp == 9) {
    // TMA-like producer: 64 KB of L2 -> smem bulk copies per tile (mode 3 only),
    // into a region the MMA does not read, paced by the MMA's empty barrier
    if (mode == 3 && lane == 0) {
      __shared__ uint64_t tb;
      mbar_init(&tb, 1);
      fence_barrier_init();
      for (int t = 0; t < iters; ++t) {
        mbar_wait(empty + (t & 1), ((t >> 1) & 1) ^ 1);   // one 64 KB stage per tile, like the mu ring
        mbar_arrive_expect_tx(&tb, 65536);
        for (int c = 0; c < 4; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                       ::"r"(smem_u32(sm + 65536 + 16384 * c)),
                       "l"(gsrc + ((size_t)(blockIdx.x * 97 + t * 4 + c) & 4095) * 4096), "r"(smem_u32(&tb))
                       : "memory");
        mbar_wait(&tb, t & 1);
      }
    }
  } else if (warp == 8) {
    const uint32_t idesc = idesc_bf16_f32(128, 128);
    const uint64_t da = sdesc_k_sw128(smem_u32(sm));
    const uint64_t db = sdesc_k_sw128(smem_u32(sm + 32768));
    for (int t = 0; t < iters; ++t) {
      const int b = t & 1;
      mbar_wait(empty + b, ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      if (elect_one()) {
        if (mode != 2) {   // modes 0, 1, 3
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            umma_f16_ss(tmem + b * 256, da + ((k & 3) * 32 >> 4), db + ((k & 3) * 32 >> 4), idesc, k > 0 ? 1u : 0u);
            umma_f16_ss(tmem + b * 256 + 128, da + ((k & 3) * 32 >> 4), db + ((k & 3) * 32 >> 4), idesc,
                        k > 0 ? 1u : 0u);
          }
        }
        umma_commit(full + b);
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3, half = warp >> 2;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const float zscale = 0.127f;
    float mrun = -INFINITY, srun = 0.f;
    for (int t = 0; t < iters; ++t) {
      const int b = t & 1;
      mbar_wait(full + b, (t >> 1) & 1);
      tc_fence_after();
      if (mode != 1) {
        const uint32_t cbase = tmem + lane_base + b * 256 + half * 128;
        float va[32], vb[32];
        tmem_ld32(cbase, va);
        tmem_wait_ld();
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          float* v = (ch & 1) ? vb : va;
          if (ch < 3) tmem_ld32(cbase + (ch + 1) * 32, *reinterpret_cast<float(*)[32]>((ch & 1) ? va : vb));
          float m4[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
          for (int x = 4; x < 32; ++x) m4[x & 3] = fmaxf(m4[x & 3], v[x]);
          const float cmax = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * zscale;
          const float mnew = fmaxf(mrun, cmax);
          float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int x = 0; x < 32; ++x) a4[x & 3] += ex2(fmaf(v[x], zscale, -mnew));
          srun = srun * ex2(mrun - mnew) + ((a4[0] + a4[1]) + (a4[2] + a4[3]));
          mrun = mnew;
          if (ch < 3) tmem_wait_ld();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + b);
    }
    sink[blockIdx.x * 256 + threadIdx.x] = mrun + srun;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<512>(tmem);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int iters = 2000;
  long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 256 * 4);
  float* gsrc;
  cudaMalloc(&gsrc, 4096ull * 4096 * 4);
  cudaFuncSetAttribute(pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 132 * 1024);
  pipe<<<148, 320, 132 * 1024>>>(10, mode, d, sink, gsrc);
  pipe<<<148, 320, 132 * 1024>>>(iters, mode, d, sink, gsrc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  printf("mode=%d (%s): %.0f cycles per tile %s\n", mode, mode == 0 ? "pipeline" : mode == 1 ? "MMA only" : mode == 2 ? "epilogue only" : "pipeline + 64 KB TMA per tile",
         avg / 148 / iters, cudaGetErrorString(e));
  return 0;
}
