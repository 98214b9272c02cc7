// MUFU.EX2 vs FMA-pipe exp2 throughput per SM: each thread runs 8 independent
// chains of `iters` steps; prints warp-instructions per cycle per SM.
// Usage: mufu_bench [threads_per_block]
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]) - 1.0f;
      else v[i] = fmaf(v[i], 0.999f, -1e-4f);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main(int argc, char** argv) {
  int tpb = argc > 1 ? atoi(argv[1]) : 512;
  int iters = 4096;
  float* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  for (int mode = 0; mode < 2; ++mode) {
    auto fn = mode ? k<1> : k<0>;
    fn<<<148, tpb>>>(o, 16, c);
    fn<<<148, tpb>>>(o, iters, c);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    // MODE 0: 2 instr per element (MUFU + FADD); count MUFU lanes/clk/SM
    double lanes = (double)tpb * iters * 8;
    printf("%s tpb=%d: %.2f %s lanes/clk/SM\n", mode ? "FFMA" : "MUFU.EX2", tpb, lanes / avg, mode ? "ffma" : "ex2");
  }
  return 0;
}
