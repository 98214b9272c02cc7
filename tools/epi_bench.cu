// Stage-1 pass-1 epilogue in isolation: W warps (W/4 per TMEM lane quadrant)
// run the select_tc pass-1 chunk loop over a resident TMEM tile `iters`
// times, no MMA / TMA.  Prints cycles per 256x128 tile (both halves, i.e. one
// tile-pass of the real kernel when W = 8).
// Usage: epi_bench <warps> <mode>   mode 0: as the kernel, 1: no TMEM loads,
//        2: no ex2 (FFMA only), 3: no max tree, 4: pass 2 (group sums + block max)
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>

#include "../paper_2506_07900_b200/csrc/sm100.cuh"
using namespace infllm2::sm100;

template <int MODE>
__global__ void bench(int iters, long long* out, float* sink, int mma, const float* gsrc, int tma, int idle) {
  extern __shared__ __align__(1024) uint8_t dsm_raw[];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int quad = warp & 3;
  const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
  const int nw = (blockDim.x >> 5) - (mma ? 1 : 0) - (tma ? 1 : 0) - idle;
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  // fill: each warp writes its quadrant's columns it owns
  {
    float v[32];
    for (int x = 0; x < 32; ++x) v[x] = 0.01f * ((lane * 7 + x * 13) % 97) - 0.5f;
    for (int c = (warp >> 2) * 32; c < 512; c += (nw >> 2) * 32) {
      uint32_t* r = reinterpret_cast<uint32_t*>(v);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + lane_base + c),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == nw) {   // concurrent MMA issuer: SS, M=128 N=128 K=16, 2 interleaved accumulators
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    if (lane == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    __syncwarp();
    const uint32_t idesc = idesc_bf16_f32(128, 128);
    const uint64_t da = sdesc_k_sw128(smem_u32(sm));
    const uint64_t db = sdesc_k_sw128(smem_u32(sm + 32768));
    uint32_t ph = 0;
    while (!stop) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          umma_f16_ss(tmem + (k & 1) * 128, da + ((k & 3) * 32 >> 4), db + ((k & 3) * 32 >> 4), idesc, 1u);
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    return;
  }
  if (tma && warp == nw + (mma ? 1 : 0)) {   // concurrent bulk copies L2 -> smem, 16 KB each
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t tbar;
    if (lane == 0) { mbar_init(&tbar, 1); fence_barrier_init(); }
    __syncwarp();
    uint32_t ph = 0;
    int k = 0;
    while (!stop) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&tbar, 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                     ::"r"(smem_u32(sm + 16384 * (k & 3))), "l"(gsrc + (size_t)((blockIdx.x * 64 + k) & 4095) * 4096),
                     "r"(smem_u32(&tbar)) : "memory");
      }
      __syncwarp();
      mbar_wait(&tbar, ph);
      ph ^= 1;
      ++k;
    }
    return;
  }
  if (warp >= nw + (mma ? 1 : 0) + (tma ? 1 : 0)) {   // idle warps parked on an mbarrier (like the top-k warps)
    __shared__ uint64_t ibar;
    if (threadIdx.x == (nw + (mma ? 1 : 0) + (tma ? 1 : 0)) * 32) { mbar_init(&ibar, 1); fence_barrier_init(); }
    __syncwarp();
    while (!stop) {
      uint32_t done;
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, 10000000;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&ibar)), "r"(0u) : "memory");
    }
    return;
  }
  // each warp covers (256 columns / (nw/4)) of every tile
  const int parts = nw >> 2;
  const int part = warp >> 2;
  const int cols = 256 / parts;
  const float zscale = 0.127f;
  float mrun = -INFINITY, srun = 0.f;
  long long t0 = clock64();
  if (MODE != 4)
  for (int it = 0; it < iters; ++it) {
    const uint32_t cbase = tmem + lane_base + (it & 1) * 256 + part * cols;
    float va[32], vb[32];
    if (MODE != 1) { tmem_ld32(cbase, va); tmem_wait_ld(); }
    else for (int x = 0; x < 32; ++x) va[x] = vb[x] = 0.01f * x + mrun * 1e-9f;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      if (ch >= cols / 32) break;
      float* v = (ch & 1) ? vb : va;
      if (MODE != 1 && ch + 1 < cols / 32) tmem_ld32(cbase + (ch + 1) * 32, *reinterpret_cast<float(*)[32]>((ch & 1) ? va : vb));
      float mnew = mrun;
      if (MODE != 3) {
        float m4[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
        for (int x = 4; x < 32; ++x) m4[x & 3] = fmaxf(m4[x & 3], v[x]);
        const float cmax = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * zscale;
        mnew = fmaxf(mrun, cmax);
      } else {
        mnew = fmaxf(mrun, 1.0f);
      }
      float a4[4] = {0.f, 0.f, 0.f, 0.f};
      if (MODE == 2) {
#pragma unroll
        for (int x = 0; x < 32; ++x) a4[x & 3] += fmaf(v[x], zscale, -mnew);
      } else {
#pragma unroll
        for (int x = 0; x < 32; ++x) a4[x & 3] += ex2(fmaf(v[x], zscale, -mnew));
      }
      srun = srun * ex2(mrun - mnew) + ((a4[0] + a4[1]) + (a4[2] + a4[3]));
      mrun = mnew;
      if (MODE != 1 && ch + 1 < cols / 32) tmem_wait_ld();
    }
  }
  if (MODE == 4) {
    // pass 2 (G = 16): thread = kernel lane, kQH = 8 queries x 16 heads of its half,
    // lse from smem, shuffle block max, predicated stores to a global row buffer
    __shared__ __align__(16) float lse2[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lse2[i] = 0.3f + 0.001f * i;
    __syncthreads();
    const int half = part & 1;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t cbase = tmem + lane_base + (it & 1) * 256 + half * 128;
      float va[32], vb[32];
      tmem_ld32(cbase, va);
      tmem_wait_ld();
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        float* v = (ch & 1) ? vb : va;
        if (ch < 3) tmem_ld32(cbase + (ch + 1) * 32, *reinterpret_cast<float(*)[32]>((ch & 1) ? va : vb));
        float sc[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t l2 = smem_u32(lse2 + (half * 8 + ch * 2 + u) * 16);
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int h = 0; h < 16; h += 4) {
            const float4 l4 = lds4(l2 + h * 4);
            a0 += ex2(fmaf(v[u * 16 + h], zscale, -l4.x));
            a1 += ex2(fmaf(v[u * 16 + h + 1], zscale, -l4.y));
            a0 += ex2(fmaf(v[u * 16 + h + 2], zscale, -l4.z));
            a1 += ex2(fmaf(v[u * 16 + h + 3], zscale, -l4.w));
          }
          sc[u] = (a0 + a1) * 0.0625f;
        }
        float r[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float up = __shfl_up_sync(0xffffffffu, sc[u], 1);
          r[u] = ((lane & 3) == 0 && lane > 0) ? fmaxf(sc[u], up) : sc[u];
        }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1)
#pragma unroll
          for (int u = 0; u < 2; ++u) r[u] = fmaxf(r[u], __shfl_xor_sync(0xffffffffu, r[u], o));
#pragma unroll
        for (int u = 0; u < 2; ++u)
          st_global_if(sink + 148 * 1024 + ((half * 8 + ch * 2 + u) * 64 + quad * 8 + (lane >> 2)), r[u], (lane & 3) == 0);
        if (ch < 3) tmem_wait_ld();
      }
      srun += va[0];
    }
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = srun + mrun;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (threadIdx.x == 0) stop = 1;
  asm volatile("bar.sync 1, %0;" ::"r"(nw * 32));
  if (threadIdx.x == 0) { while (false) {} }
  __threadfence_block();
  if (warp == 0) { for (volatile int i = 0; i < 100000; ++i) {} tmem_dealloc<512>(tmem); }
}

int main(int argc, char** argv) {
  const int warps = argc > 1 ? atoi(argv[1]) : 8;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  const int iters = 2000;
  long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4 + 65536);
  auto fn = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : mode == 3 ? bench<3> : bench<4>;
  const int mma = argc > 3 ? atoi(argv[3]) : 0;
  const int tma = argc > 4 ? atoi(argv[4]) : 0;
  const int idle = argc > 5 ? atoi(argv[5]) : 0;
  float* gsrc;
  cudaMalloc(&gsrc, 4096ull * 4096 * 4);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  fn<<<148, (warps + mma + tma + idle) * 32, 66 * 1024>>>(10, d, sink, mma, gsrc, tma, idle);
  fn<<<148, (warps + mma + tma + idle) * 32, 66 * 1024>>>(iters, d, sink, mma, gsrc, tma, idle);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("idle=%d tma=%d mma=%d warps=%2d mode=%d: %.0f cycles per 256x128 tile (MUFU bound 2048) %s\n", idle, tma, mma, warps, mode, avg / iters,
         cudaGetErrorString(e));
  return 0;
}
