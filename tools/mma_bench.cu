// tcgen05.mma issue-rate micro-benchmark: cycles per kind::f16 M=128 x N x K=16
// MMA (both operands in shared memory, K-major 128-B swizzle), one CTA per SM,
// one issuing thread, commits every `group` MMAs (like stage 2's QK / PV).
// Usage: mma_bench <N> <group> [iters] [ts] [nowait] [nacc]  (nacc = 2/4 independent
// accumulators, MMA k writes accumulator k % nacc, 16 MMAs per commit)
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>

#include "../paper_2506_07900_b200/csrc/sm100.cuh"

using namespace infllm2::sm100;

__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

template <int NACC>
__global__ void __launch_bounds__(128, 1) bench(int n, int group, int iters, long long* out, int ts, int nowait) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {   // whole warp runs the loop (uniform operands), one elected lane issues
    const uint32_t idesc = idesc_bf16_f32(128, n);
    const uint64_t da = sdesc_k_sw128(smem_u32(sm));
    const uint64_t db = sdesc_k_sw128(smem_u32(sm + 32768));
    uint32_t ph = 0;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (NACC > 1) {
        // NACC independent accumulators (columns k % NACC * max(n, 64)), 16 MMAs per group
        if (elect_one())
#pragma unroll
        for (int k = 0; k < 16; ++k)
          umma_f16_ss(tmem + (k % NACC) * (n < 64 ? 64 : n), da + ((k & 3) * 32 >> 4), db + ((k & 3) * 32 >> 4), idesc,
                      k >= NACC ? 1u : 0u);
      } else {
        if (elect_one())
        for (int k = 0; k < group; ++k) {
          if (ts) umma_ts(tmem, tmem + 256 + (k & 3) * 8, db + ((k & 3) * 32 >> 4), idesc, k > 0 ? 1u : 0u);
          else umma_f16_ss(tmem, da + ((k & 3) * 32 >> 4), db + ((k & 3) * 32 >> 4), idesc, k > 0 ? 1u : 0u);
        }
      }
      if (elect_one()) umma_commit(&bar);
      __syncwarp();
      if (!nowait || it == iters - 1) {
        mbar_wait(&bar, ph);
      }
      ph ^= 1;
    }
    t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 16;
  const int group = argc > 2 ? atoi(argv[2]) : 8;
  const int iters = argc > 3 ? atoi(argv[3]) : 2000;
  const int ts = argc > 4 ? atoi(argv[4]) : 0;
  const int nowait = argc > 5 ? atoi(argv[5]) : 0;
  const int nacc = argc > 6 ? atoi(argv[6]) : 1;   // 1, 2 or 4 (N <= 64); >1 forces group = 16
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto* fn = nacc == 4 ? bench<4> : nacc == 2 ? bench<2> : bench<1>;
  const int grp = nacc > 1 ? 16 : group;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  fn<<<148, 128, 66 * 1024>>>(n, grp, 10, d, ts, nowait);
  fn<<<148, 128, 66 * 1024>>>(n, grp, iters, d, ts, nowait);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("nacc=%d %s%s N=%3d group=%2d: %.1f cycles per MMA (%.1f per group incl. commit+wait) %s\n", nacc, ts ? "TS" : "SS", nowait ? " nowait" : "", n, grp,
         avg / (iters * (double)grp), avg / iters, cudaGetErrorString(e));
  return 0;
}
