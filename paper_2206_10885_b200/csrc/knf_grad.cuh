// knf_grad.cuh -- analytic gradient of the SDF tile MLP (north_star subsystem 2: "also emits the SDF gradient for
// normals").  Forward-mode differentiation of the cell's network d(x) = w3 . softplus(W2 softplus(W1 enc(x) + b1) + b2)
// + b3 through nn.fourier_encode (nn.py:66-93): every feature depends on one coordinate, d sin(2^o pi x_a) / d x_a =
// 2^o pi cos(2^o pi x_a), so the first layer's Jacobian costs one extra FMA per weight and the second layer three.
//
// This is NOT what the reference renders with: grid.grad_fd / normal_batch are global central differences over the
// whole field (grid.py:440-461), which see the jumps between neighbouring cells' networks; the parity path implements
// those exactly (knf_rays.cuh).  The analytic gradient is an extra output (knf_sdf_gradient, grid.grad_analytic) whose
// deviation from the FD normals is reported by tests/test_gpu_forward.py::test_analytic_gradient.
//
// Same tiles and weight blobs as mlp_warp_kernel; one lane differentiates one point (two per tile pass), weights are
// broadcast reads from shared memory, the point's features and hidden vectors (value + 3 partials) live in two
// per-lane shared-memory panels.  A utility kernel, not a hot one: ~6 700 FMAs per point.
#pragma once

#include "knf_mlp.cuh"

namespace knf {

struct GradSmem {
  alignas(16) float w[SdfBlob::floats];
  alignas(16) float feat[2 * pad_k(kSdfIn)][32];  // [k][lane] value, [pad + k][lane] d/dx_axis(k)
  alignas(16) float hid[4 * kHidden][32];         // [4 m + c][lane]: c = 0 value, 1..3 partials
  alignas(8) uint64_t bar;
};

struct GradParams {
  MlpParams P;
  float* dist;  // per request slot (nullable)
  float* grad;  // (n,3) per request slot
};

__device__ __forceinline__ float sigmoid_of_softplus_arg(float z) {
  // softplus'(z) = 1 / (1 + exp(-z)); plain fp32 (this output is not bit-matched to anything)
  return __fdividef(1.0f, 1.0f + __expf(-z));
}

static __global__ void __launch_bounds__(32, 5) sdf_gradient_kernel(GradParams G) {
  using Blob = SdfBlob;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GradSmem& S = *reinterpret_cast<GradSmem*>(smem_raw);
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const MlpParams& P = G.P;
  const int n_tiles = P.ctr->n_tiles;
  uint32_t parity = 0;
  constexpr int KP = pad_k(kSdfIn);
  const float pi_f = 3.14159274101257324e+00f;
  for (;;) {
    const int t = next_tile(P.ctr, lane);
    if (t >= n_tiles) break;
    const Tile tile = P.tiles[t];
    fetch_weights<Blob>(S.w, P.blobs, tile.cell, &S.bar, lane);
    mbar_wait(&S.bar, parity);
    parity ^= 1;
    const float* W1 = S.w + Blob::w1;  // [k][32]
    const float* W2 = S.w + Blob::w2;  // [m][32]
    const float* W3 = S.w + Blob::w3;  // [m][12]
    for (int half = 0; half < 2; half++) {
      const int p = 32 * half + lane;
      if (32 * half >= tile.count) break;  // warp-uniform
      const bool act = p < tile.count;
      int slot = -1;
      float x[3] = {0.f, 0.f, 0.f};
      if (act) {
        slot = P.perm[tile.start + p];
        const float4 pt = P.req_pt[slot];
        x[0] = pt.x; x[1] = pt.y; x[2] = pt.z;
      }
      // features and their derivative with respect to their own axis (feature k of axis a: k = a, 3 + 6 o + a, 3 + 6 o + 3 + a)
#pragma unroll
      for (int a = 0; a < 3; a++) {
        S.feat[a][lane] = x[a];
        S.feat[KP + a][lane] = 1.0f;
        float s, c;
        np_sincosf(__fmul_rn(pi_f, x[a]), s, c);
        float scale = pi_f;
#pragma unroll
        for (int o = 0; o < kSdfFreqs; o++) {
          S.feat[3 + 6 * o + a][lane] = s;
          S.feat[3 + 6 * o + 3 + a][lane] = c;
          S.feat[KP + 3 + 6 * o + a][lane] = scale * c;
          S.feat[KP + 3 + 6 * o + 3 + a][lane] = -scale * s;
          const float two_s = __fmul_rn(2.0f, s);
          const float ns = __fmul_rn(two_s, c), nc = __fsub_rn(1.0f, __fmul_rn(two_s, s));
          s = ns;
          c = nc;
          scale *= 2.0f;
        }
      }
      // layer 1: z1[n] and its three partials, eight neurons at a time
#pragma unroll 1
      for (int n0 = 0; n0 < kHidden; n0 += 8) {
        float z[8], dz[8][3];
#pragma unroll
        for (int j = 0; j < 8; j++) z[j] = dz[j][0] = dz[j][1] = dz[j][2] = 0.0f;
#pragma unroll
        for (int k = 0; k < kSdfIn; k++) {
          const int a = k < 3 ? k : (k - 3) % 3;  // compile-time after unrolling
          const float f = S.feat[k][lane], df = S.feat[KP + k][lane];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const float w = W1[k * kHidden + n0 + j];
            z[j] = fmaf(f, w, z[j]);
            dz[j][a] = fmaf(df, w, dz[j][a]);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const float zz = z[j] + S.w[Blob::b1 + n0 + j];
          const float sg = sigmoid_of_softplus_arg(zz);
          S.hid[4 * (n0 + j) + 0][lane] = fmaxf(zz, 0.0f) + log1pf(__expf(-fabsf(zz)));
#pragma unroll
          for (int a = 0; a < 3; a++) S.hid[4 * (n0 + j) + 1 + a][lane] = sg * dz[j][a];
        }
      }
      // layer 2 + output layer (distance row): accumulate d and grad directly
      float d = 0.0f, g[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll 1
      for (int n0 = 0; n0 < kHidden; n0 += 8) {
        float z[8], dz[8][3];
#pragma unroll
        for (int j = 0; j < 8; j++) z[j] = dz[j][0] = dz[j][1] = dz[j][2] = 0.0f;
#pragma unroll 4
        for (int m = 0; m < kHidden; m++) {
          const float h = S.hid[4 * m][lane], h0 = S.hid[4 * m + 1][lane], h1 = S.hid[4 * m + 2][lane], h2 = S.hid[4 * m + 3][lane];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const float w = W2[m * kHidden + n0 + j];
            z[j] = fmaf(h, w, z[j]);
            dz[j][0] = fmaf(h0, w, dz[j][0]);
            dz[j][1] = fmaf(h1, w, dz[j][1]);
            dz[j][2] = fmaf(h2, w, dz[j][2]);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const float zz = z[j] + S.w[Blob::b2 + n0 + j];
          const float sg = sigmoid_of_softplus_arg(zz);
          const float w3 = W3[(n0 + j) * kSdfOutPad];
          d = fmaf(fmaxf(zz, 0.0f) + log1pf(__expf(-fabsf(zz))), w3, d);
#pragma unroll
          for (int a = 0; a < 3; a++) g[a] = fmaf(sg * dz[j][a], w3, g[a]);
        }
      }
      if (act) {
        if (G.dist) G.dist[slot] = d + S.w[Blob::b3];
        G.grad[3 * (size_t)slot + 0] = g[0];
        G.grad[3 * (size_t)slot + 1] = g[1];
        G.grad[3 * (size_t)slot + 2] = g[2];
      }
    }
    __syncwarp();
  }
}

}  // namespace knf
