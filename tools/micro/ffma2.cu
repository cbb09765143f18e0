// FMA-pipe throughput: FFMA vs FFMA2 vs FADD2 vs F2FP (cycles per warp instruction per SMSP).
#include <cstdio>
#include <cstdint>
#include "../../paper_2605_16839_b200/csrc/common.cuh"
using namespace cpa;
template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, long long* cyc, int iters) {
  float2 a[8]; float s[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); s[i] = a[i].x; u[i] = i; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) s[i] = fmaf(s[i], 0.999f, 0.37f);
      if (MODE == 1) a[i] = ffma2(a[i], 0.999f, 0.37f);
      if (MODE == 2) a[i] = fadd2(a[i], make_float2(0.37f, 0.11f));
      if (MODE == 3) u[i] += pack_f16x2(s[i], s[(i + 1) & 7]);
      if (MODE == 4) s[i] = fmax3(s[i], s[(i + 3) & 7], 0.5f);
    }
  }
  long long t1 = clock64();
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i].x + a[i].y + s[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(float* o, long long* c, const char* n, int warps) {
  int iters = 4000;
  k<MODE><<<148, warps * 32>>>(o, c, iters); cudaDeviceSynchronize();
  k<MODE><<<148, warps * 32>>>(o, c, iters); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-6s warps/SM=%2d: %.2f cycles per warp-instr per SMSP\n", n, warps, (double)h / (iters * 8.0) / (warps / 4.0));
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 1 << 22); cudaMalloc(&c, 1 << 16);
  for (int w : {4, 8, 16}) {
    run<0>(o, c, "FFMA", w); run<1>(o, c, "FFMA2", w); run<2>(o, c, "FADD2", w); run<3>(o, c, "F2FP", w); run<4>(o, c, "FMNMX3", w);
  }
  return 0;
}
