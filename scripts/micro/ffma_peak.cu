// Measures the sustainable FP32 FMA rate of one B200 with scalar FFMA and packed FFMA2 streams
// (register operands only), for the roofline denominator of the tile-MLP kernel.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>  // 0 scalar FFMA, 1 packed FFMA2, 2 FFMA2 + one LDS.128 per 8 (like the layer loop)
__global__ void k(float* out, int iters, float a) {
  __shared__ float4 sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = make_float4(a, a, a, a);
  __syncthreads();
  float2 acc[16];
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  float2 x = make_float2(a, a * 0.5f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      float w = a + r;
      if (MODE == 2) { float4 v = sm[(threadIdx.x + r + it) & 63]; w = v.x; x = make_float2(v.y, v.z); }
#pragma unroll
      for (int i = 0; i < 16; i++) {
        if (MODE == 0) { acc[i].x = __fmaf_rn(x.x, w, acc[i].x); acc[i].y = __fmaf_rn(x.y, w, acc[i].y); }
        else acc[i] = __ffma2_rn(x, make_float2(w, w), acc[i]);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> void run(const char* name, int warps_per_sm) {
  int threads = 32 * warps_per_sm, blocks = 148, iters = 20000;
  float* out; cudaMalloc(&out, blocks * threads * 4);
  k<MODE><<<blocks, threads>>>(out, 100, 1.0001f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<MODE><<<blocks, threads>>>(out, iters, 1.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = (double)blocks * threads * iters * 8 * 16 * 2;
  printf("%-28s warps/SM %2d: %.2f ms  %.1f TFLOP/s  (%.1f FMA/clk/SM at 1.965 GHz)\n", name, warps_per_sm, ms, 2 * fma / ms / 1e9,
         fma / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(out);
}
int main() {
  for (int w : {4, 8, 16, 32}) { run<0>("scalar FFMA", w); run<1>("packed FFMA2", w); run<2>("FFMA2 + LDS.128/16", w); }
  return 0;
}
