// hmma_split.cu -- (1) accuracy of fp32 dot products evaluated on the tensor cores as exact 3-way
// bf16 splits (x = x1 + x2 + x3, 8 bits each) with mma.sync.m16n8k16 (SASS HMMA.16816.F32.BF16), against
// fp64 and against the k-ordered fp32 FMA chain the reference's sgemm performs; (2) the HMMA issue rate of
// one B200 alone and interleaved with a packed-FFMA2 stream (does the tensor pipe overlap the FMA pipe?).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o hmma_split hmma_split.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ uint32_t pack_hi(float lo, float hi) { return __byte_perm(__float_as_uint(lo), __float_as_uint(hi), 0x7632); }
__device__ __forceinline__ float trunc_bf16(float x) { return __uint_as_float(__float_as_uint(x) & 0xffff0000u); }

// three exact pieces of (lo, hi), truncation split
__device__ __forceinline__ void split3(float lo, float hi, uint32_t& p1, uint32_t& p2, uint32_t& p3) {
  p1 = pack_hi(lo, hi);
  float rl = __fsub_rn(lo, trunc_bf16(lo)), rh = __fsub_rn(hi, trunc_bf16(hi));
  p2 = pack_hi(rl, rh);
  rl = __fsub_rn(rl, trunc_bf16(rl));
  rh = __fsub_rn(rh, trunc_bf16(rh));
  p3 = pack_hi(rl, rh);
}

// Y[64 x 32] = X[64 x K] . W[K x 32] per warp; variant selects the accumulation strategy.
//  0: one accumulator, small products first (all k-tiles), x1w1 last
//  1: two accumulators (small, big), summed with one rounded add
//  2: small accumulator + one fresh accumulator per k-tile for x1w1, summed with rounded adds
//  3: like 1 with only 6 products (x2w3, x3w2 dropped too)
template <int K>
__global__ void dot_kernel(const float* __restrict__ X, const float* __restrict__ W, float* __restrict__ Y, int variant) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float* Xt = X + (size_t)blockIdx.x * 64 * K;
  float* Yt = Y + (size_t)blockIdx.x * 64 * 32;
  constexpr int KT = K / 16;
  for (int m = 0; m < 4; m++) {
    uint32_t a[KT][3][4];
    for (int kt = 0; kt < KT; kt++)
      for (int h = 0; h < 4; h++) {
        int row = 16 * m + g + ((h & 1) ? 8 : 0), col = 16 * kt + 2 * t + ((h & 2) ? 8 : 0);
        split3(Xt[row * K + col], Xt[row * K + col + 1], a[kt][0][h], a[kt][1][h], a[kt][2][h]);
      }
    for (int nt = 0; nt < 4; nt++) {
      uint32_t b[KT][3][2];
      for (int kt = 0; kt < KT; kt++)
        for (int h = 0; h < 2; h++) {
          int k = 16 * kt + 2 * t + (h ? 8 : 0), n = 8 * nt + g;
          split3(W[k * 32 + n], W[(k + 1) * 32 + n], b[kt][0][h], b[kt][1][h], b[kt][2][h]);
        }
      float ds[4] = {0, 0, 0, 0}, db[4] = {0, 0, 0, 0}, out[4];
      for (int kt = 0; kt < KT; kt++) {
        if (variant != 3) {
          hmma(ds, a[kt][2], b[kt][1]);
          hmma(ds, a[kt][1], b[kt][2]);
        }
        hmma(ds, a[kt][2], b[kt][0]);
        hmma(ds, a[kt][0], b[kt][2]);
        hmma(ds, a[kt][1], b[kt][1]);
        hmma(ds, a[kt][1], b[kt][0]);
        hmma(ds, a[kt][0], b[kt][1]);
      }
      if (variant == 0) {
        for (int kt = 0; kt < KT; kt++) hmma(ds, a[kt][0], b[kt][0]);
        for (int i = 0; i < 4; i++) out[i] = ds[i];
      } else if (variant == 1 || variant == 3) {
        for (int kt = 0; kt < KT; kt++) hmma(db, a[kt][0], b[kt][0]);
        for (int i = 0; i < 4; i++) out[i] = __fadd_rn(db[i], ds[i]);
      } else {
        for (int kt = 0; kt < KT; kt++) {
          float f[4] = {0, 0, 0, 0};
          hmma(f, a[kt][0], b[kt][0]);
          for (int i = 0; i < 4; i++) db[i] = __fadd_rn(db[i], f[i]);
        }
        for (int i = 0; i < 4; i++) out[i] = __fadd_rn(db[i], ds[i]);
      }
      int r0 = 16 * m + g, c0 = 8 * nt + 2 * t;
      Yt[r0 * 32 + c0] = out[0];
      Yt[r0 * 32 + c0 + 1] = out[1];
      Yt[(r0 + 8) * 32 + c0] = out[2];
      Yt[(r0 + 8) * 32 + c0 + 1] = out[3];
    }
  }
}

template <int K>
void accuracy(const char* what, bool positive_inputs) {
  const int tiles = 8192, rows = tiles * 64;
  std::vector<float> X((size_t)rows * K), W((size_t)K * 32), Y((size_t)rows * 32);
  srand(12345);
  auto u = []() { return (rand() + 0.5) / (RAND_MAX + 1.0); };
  auto gauss = [&]() { return sqrt(-2 * log(u())) * cos(6.283185307179586 * u()); };
  for (auto& x : X) {
    double v = gauss() * 1.5;
    x = positive_inputs ? (float)(log1p(exp(-fabs(v))) + fmax(v, 0.0)) : (float)sin(v * 3.0);
  }
  double lim = sqrt(6.0 / K);
  for (auto& w : W) w = (float)((2 * u() - 1) * lim);
  std::vector<double> exact((size_t)rows * 32), mag((size_t)rows * 32);
  std::vector<float> chain((size_t)rows * 32);
  for (int r = 0; r < rows; r++)
    for (int n = 0; n < 32; n++) {
      double s = 0, m = 0;
      float c = 0;
      for (int k = 0; k < K; k++) {
        m += fabs((double)X[(size_t)r * K + k] * (double)W[k * 32 + n]);
        s += (double)X[(size_t)r * K + k] * (double)W[k * 32 + n];
        c = fmaf(X[(size_t)r * K + k], W[k * 32 + n], c);
      }
      exact[(size_t)r * 32 + n] = s;
      mag[(size_t)r * 32 + n] = m;
      chain[(size_t)r * 32 + n] = c;
    }
  auto report = [&](const char* name, const float* y) {
    double se = 0, sa = 0, sb = 0, mx = 0, sabs = 0, worst_rel = 0;
    size_t n = exact.size(), differ = 0;
    for (size_t i = 0; i < n; i++) {
      double e = (double)y[i] - exact[i];
      double ulp = ldexp(1.0, ilogb(fabs(exact[i]) + 1e-300) - 23);
      double eu = e / ulp;
      se += eu * eu; sa += fabs(eu); sb += eu * (exact[i] >= 0 ? 1 : -1); mx = fmax(mx, fabs(eu)); sabs += fabs(e);
      differ += (y[i] != chain[i]);
      worst_rel = fmax(worst_rel, fabs(e) / (mag[i] + 1e-300));
    }
    printf("  %-44s mean|e| %.3f ulp  rms %.3f  max %.2f  bias(toward +|y|) %+.3f  mean abs %.3e  differs from fp32 chain %.1f %%  worst |e| / sum|x w| = %.3e = 2^%.1f\n", name,
           sa / n, sqrt(se / n), mx, sb / n, sabs / n, 100.0 * differ / n, worst_rel, log2(worst_rel));
  };
  printf("%s (K=%d, %d rows x 32 outputs)\n", what, K, rows);
  report("fp32 k-ordered FMA chain (reference sgemm)", chain.data());
  float *dX, *dW, *dY;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dW, W.size() * 4); cudaMalloc(&dY, Y.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  const char* names[4] = {"HMMA 8 products, one accumulator", "HMMA 8 products, small + big accumulators", "HMMA 8 products, fresh accumulator per k-tile",
                          "HMMA 6 products, small + big accumulators"};
  for (int v = 0; v < 4; v++) {
    dot_kernel<K><<<tiles, 32>>>(dX, dW, dY, v);
    cudaMemcpy(Y.data(), dY, Y.size() * 4, cudaMemcpyDeviceToHost);
    report(names[v], Y.data());
  }
  cudaFree(dX); cudaFree(dW); cudaFree(dY);
}

// ---- throughput ---------------------------------------------------------------------------------------
// MODE 0: HMMA only (8 independent accumulator tiles per warp); 1: FFMA2 only; 2: 1 HMMA per FPER FFMA2.
template <int MODE, int FPER>
__global__ void rate_kernel(float* out, int iters, float seed) {
  float d[8][4];
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; i++) a[i] = 0x3f803f80u + threadIdx.x;
  b[0] = 0x3f803c00u; b[1] = 0x3c003f80u + threadIdx.x;
  for (int j = 0; j < 8; j++) for (int i = 0; i < 4; i++) d[j][i] = seed * j;
  float2 acc[FPER];
  for (int i = 0; i < FPER; i++) acc[i] = make_float2(seed + i, seed - i);
  const float2 x = make_float2(seed, seed * 0.5f), w = make_float2(0.999f, 0.999f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (MODE != 1) hmma(d[j], a, b);
      if (MODE != 0) {
#pragma unroll
        for (int i = 0; i < FPER; i++) acc[i] = __ffma2_rn(x, w, acc[i]);
      }
    }
  }
  float s = 0;
  for (int j = 0; j < 8; j++) for (int i = 0; i < 4; i++) s += d[j][i];
  for (int i = 0; i < FPER; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE, int FPER>
void rate(const char* name, int warps_per_sm) {
  int threads = 32 * warps_per_sm, blocks = 148, iters = 20000;
  float* out; cudaMalloc(&out, blocks * threads * 4);
  rate_kernel<MODE, FPER><<<blocks, threads>>>(out, 100, 1.0001f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); rate_kernel<MODE, FPER><<<blocks, threads>>>(out, iters, 1.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double clk = ms * 1e-3 * 1.965e9;  // SM cycles (assuming the boost clock)
  double hm = (MODE != 1) ? (double)warps_per_sm * iters * 8 : 0, ff = (MODE != 0) ? (double)warps_per_sm * iters * 8 * FPER : 0;
  printf("  %-34s warps/SM %2d: %7.2f ms  HMMA/clk/SM %.3f (%.0f bf16 TFLOP/s)  FFMA2 lane-FMA/clk/SM %.1f\n", name, warps_per_sm, ms, hm / clk,
         hm * 4096 * 148 / (ms * 1e-3) / 1e12, ff * 64 / clk);
  cudaFree(out);
}

int main() {
  accuracy<32>("hidden layer, softplus-like positive inputs", true);
  accuracy<48>("first layer, sin/cos-like inputs", false);
  printf("issue rates (148 CTAs, clock assumed 1.965 GHz)\n");
  for (int w : {4, 8, 12, 16}) {
    rate<0, 1>("HMMA.16816 bf16 only", w);
    rate<1, 8>("FFMA2 only", w);
    rate<2, 2>("1 HMMA : 2 FFMA2", w);
    rate<2, 4>("1 HMMA : 4 FFMA2", w);
    rate<2, 8>("1 HMMA : 8 FFMA2", w);
  }
  return 0;
}
