// knf_mlp.cuh -- fused tiny-MLP tile kernels (north_star subsystem 2).
//
// Replaces nn.fourier_encode (nn.py:66-93) + grid.grid_forward (grid.py:241-294) + the
// activations (nn.py:26-50) for one family of per-cell MLPs.
//
// Work unit: a *tile* = up to 256 evaluation requests that fall in the same grid cell
// (produced by the routing pass, knf_route.cuh).  One CTA of 4 warps owns a tile:
//   * thread 0 pulls the cell's 10.9 KB weight blob into shared memory with ONE TMA bulk copy
//     (cp.async.bulk -> UBLKCP) signalled on an mbarrier; the copy overlaps the encode;
//   * each warp owns 64 of the tile's points.  It encodes them (NumPy-exact sin/cos + the fp32
//     double-angle recurrence) into a k-major shared-memory panel X[k][64];
//   * hidden layers are register-tiled SGEMMs: every lane accumulates an 8 point x 8 neuron
//     block, reading 8 activations + 8 weights (4 LDS.128) per k for 64 FFMAs.  The k loop is
//     sequential from k = 0 with one FFMA per step and the bias is added afterwards as its own
//     rounded add -- exactly the arithmetic OpenBLAS sgemm + NumPy's `+ b` perform in the
//     reference's per-cell path, so given the same layer inputs the pre-activations are
//     bit-identical to the reference's;
//   * the 32 -> N3 output layer is evaluated two points per lane and written straight to the
//     caller's buffers in request order (no unsort pass).
//
// FP32 FFMA, not tensor cores: TF32/BF16 mma gives ~1e-3 absolute SDF error, 1000x over the
// parity budget that FD normals (x 1/2h = 500 amplification) need.  See DESIGN.md.
#pragma once

#include "knf_common.cuh"

namespace knf {

constexpr int kPanelLd = kWarpPts + 4;  // 68: row stride of the per-warp activation panels (floats)

enum { ACT_RELU = 1, ACT_SOFTPLUS = 2 };

struct MlpParams {
  const float* blobs;          // n_cells * Blob::floats
  const int* perm;             // sorted position -> request slot
  const Tile* tiles;
  RouteCounters* ctr;          // n_tiles, tile_cursor
  // SDF inputs
  const float4* req_pt;        // request slot -> fp32 point
  // colour inputs (request slot -> row)
  const float* col_v;          // (n,3) fp32 view dirs
  const float* col_n;          // (n,3) fp32 normals
  const float* col_z;          // (n,F) fp32 features
  // outputs, indexed by request slot
  float* out_first;            // SDF: distance per slot (nullable)
  float* out_full;             // SDF: (n, 1+F) rows; colour: (n,3) rows (nullable)
};

template <int K1, int N3, int N3P, int HIDDEN_ACT, bool IS_COLOR>
struct MlpSmem {
  using Blob = BlobLayout<K1, N3P>;
  alignas(16) float w[Blob::floats];
  alignas(16) float x[kTileWarps][K1 * kPanelLd];       // layer-1 input panel, later layer-2 output
  alignas(16) float h[kTileWarps][kHidden * kPanelLd];  // layer-1 output panel
  alignas(8) uint64_t bar;
  int tile_idx[2];
};

template <int ACT>
__device__ __forceinline__ float hidden_act(float z) {
  if (ACT == ACT_RELU) return fmaxf(z, 0.0f);
  return softplus_acc(z);
}

// acc[i][j] = sum_k In[k][pt_i] * Wt[k][nr_j], k ascending, one FFMA per k.
template <int K>
__device__ __forceinline__ void layer_8x8(const float* __restrict__ In, const float* __restrict__ Wt, int pg, int ng,
                                          float (&acc)[8][8]) {
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = 0.0f;
  const float* xp = In + pg * 4;
  const float* wp = Wt + ng * 4;
#pragma unroll 3
  for (int k = 0; k < K; k++) {
    float4 xa = *reinterpret_cast<const float4*>(xp + k * kPanelLd);
    float4 xb = *reinterpret_cast<const float4*>(xp + k * kPanelLd + 32);
    float4 wa = *reinterpret_cast<const float4*>(wp + k * kHidden);
    float4 wb = *reinterpret_cast<const float4*>(wp + k * kHidden + 16);
    const float xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    const float ws[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[i][j] = __fmaf_rn(xs[i], ws[j], acc[i][j]);
  }
}

// z = acc + b ; h = act(z) ; Out[neuron][point] (k-major panel for the next layer)
template <int ACT>
__device__ __forceinline__ void store_hidden(float (&acc)[8][8], const float* __restrict__ bias, float* __restrict__ Out,
                                             int pg, int ng) {
#pragma unroll
  for (int j = 0; j < 8; j++) {
    int neuron = (j < 4) ? (ng * 4 + j) : (16 + ng * 4 + (j - 4));
    float b = bias[neuron];
    float4 lo, hi;
    lo.x = hidden_act<ACT>(__fadd_rn(acc[0][j], b));
    lo.y = hidden_act<ACT>(__fadd_rn(acc[1][j], b));
    lo.z = hidden_act<ACT>(__fadd_rn(acc[2][j], b));
    lo.w = hidden_act<ACT>(__fadd_rn(acc[3][j], b));
    hi.x = hidden_act<ACT>(__fadd_rn(acc[4][j], b));
    hi.y = hidden_act<ACT>(__fadd_rn(acc[5][j], b));
    hi.z = hidden_act<ACT>(__fadd_rn(acc[6][j], b));
    hi.w = hidden_act<ACT>(__fadd_rn(acc[7][j], b));
    *reinterpret_cast<float4*>(Out + neuron * kPanelLd + pg * 4) = lo;
    *reinterpret_cast<float4*>(Out + neuron * kPanelLd + 32 + pg * 4) = hi;
  }
}

// nn.fourier_encode (nn.py:66-93) of a 3-vector into panel rows [row0, row0 + 3 + 6*L) at column p.
template <int L>
__device__ __forceinline__ void encode_into(float* __restrict__ panel, int row0, int p, float x, float y, float z) {
  const float pi_f = 3.14159274101257324e+00f;  // float32(np.pi)
  panel[(row0 + 0) * kPanelLd + p] = x;
  panel[(row0 + 1) * kPanelLd + p] = y;
  panel[(row0 + 2) * kPanelLd + p] = z;
  float s[3], c[3];
  np_sincosf(__fmul_rn(pi_f, x), s[0], c[0]);
  np_sincosf(__fmul_rn(pi_f, y), s[1], c[1]);
  np_sincosf(__fmul_rn(pi_f, z), s[2], c[2]);
#pragma unroll
  for (int o = 0; o < L; o++) {
    int r = row0 + 3 + 6 * o;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      panel[(r + a) * kPanelLd + p] = s[a];
      panel[(r + 3 + a) * kPanelLd + p] = c[a];
      float two_s = __fmul_rn(2.0f, s[a]);
      float ns = __fmul_rn(two_s, c[a]);                      // 2 s c
      float nc = __fsub_rn(1.0f, __fmul_rn(two_s, s[a]));     // 1 - 2 s s
      s[a] = ns;
      c[a] = nc;
    }
  }
}

template <int K1, int N3, int N3P, int HIDDEN_ACT, bool IS_COLOR>
static __global__ void __launch_bounds__(kTileWarps * 32, 2) mlp_tile_kernel(MlpParams P) {
  using Blob = BlobLayout<K1, N3P>;
  using Smem = MlpSmem<K1, N3, N3P, HIDDEN_ACT, IS_COLOR>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int pg = lane >> 2;  // 8 point groups of 4(+4) points
  const int ng = lane & 3;   // 4 neuron groups of 4(+4) neurons

  if (tid == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncthreads();

  const int n_tiles = P.ctr->n_tiles;
  uint32_t parity = 0;
  float* X = S.x[warp];
  float* H = S.h[warp];

  for (;;) {
    if (tid == 0) S.tile_idx[parity] = atomicAdd(&P.ctr->tile_cursor, 1);
    __syncthreads();  // also: every warp is done reading S.w of the previous tile
    const int t = S.tile_idx[parity];
    if (t >= n_tiles) break;
    const Tile tile = P.tiles[t];
    if (tid == 0) {
      fence_proxy_async();
      mbar_expect_tx(&S.bar, Blob::bytes);
      bulk_copy_g2s(S.w, P.blobs + (size_t)tile.cell * Blob::floats, Blob::bytes, &S.bar);
    }

    const int wcount = min(kWarpPts, tile.count - warp * kWarpPts);  // points of this warp (may be <= 0)
    int slot[2] = {-1, -1};
    if (wcount > 0) {
      // ---- gather + encode two points per lane -------------------------------------------------
#pragma unroll
      for (int q = 0; q < 2; q++) {
        int p = lane + 32 * q;
        float px = 0.f, py = 0.f, pz = 0.f;
        if (p < wcount) {
          slot[q] = P.perm[tile.start + warp * kWarpPts + p];
          float4 pt = P.req_pt[slot[q]];
          px = pt.x; py = pt.y; pz = pt.z;
        }
        if (!IS_COLOR) {
          encode_into<kSdfFreqs>(X, 0, p, px, py, pz);
        } else {
          // grid.color_query (grid.py:397): [x | enc_L4(v) | n | z]
          float vx = 0.f, vy = 0.f, vz = 0.f, nx = 0.f, ny = 0.f, nz = 0.f;
          float zf[kFeat];
#pragma unroll
          for (int f = 0; f < kFeat; f++) zf[f] = 0.f;
          if (p < wcount) {
            const float* v = P.col_v + (size_t)slot[q] * 3;
            const float* nn = P.col_n + (size_t)slot[q] * 3;
            const float* zz = P.col_z + (size_t)slot[q] * kFeat;
            vx = v[0]; vy = v[1]; vz = v[2];
            nx = nn[0]; ny = nn[1]; nz = nn[2];
#pragma unroll
            for (int f = 0; f < kFeat; f++) zf[f] = zz[f];
          }
          X[0 * kPanelLd + p] = px;
          X[1 * kPanelLd + p] = py;
          X[2 * kPanelLd + p] = pz;
          encode_into<kDirFreqs>(X, 3, p, vx, vy, vz);
          constexpr int r = 3 + 3 + 6 * kDirFreqs;
          X[(r + 0) * kPanelLd + p] = nx;
          X[(r + 1) * kPanelLd + p] = ny;
          X[(r + 2) * kPanelLd + p] = nz;
#pragma unroll
          for (int f = 0; f < kFeat; f++) X[(r + 3 + f) * kPanelLd + p] = zf[f];
        }
      }
      __syncwarp();
    }

    mbar_wait(&S.bar, parity);  // weights have landed (all threads observe the phase)
    parity ^= 1;

    if (wcount > 0) {
      float acc[8][8];
      // ---- layer 1: K1 -> 32 ---------------------------------------------------------------------
      layer_8x8<K1>(X, S.w + Blob::w1, pg, ng, acc);
      store_hidden<HIDDEN_ACT>(acc, S.w + Blob::b1, H, pg, ng);
      __syncwarp();
      // ---- layer 2: 32 -> 32 (output panel reuses X) ----------------------------------------------
      layer_8x8<kHidden>(H, S.w + Blob::w2, pg, ng, acc);
      __syncwarp();  // all lanes finished reading... X is not read in layer 2, H is; X is free
      store_hidden<HIDDEN_ACT>(acc, S.w + Blob::b2, X, pg, ng);
      __syncwarp();
      // ---- layer 3: 32 -> N3, two points per lane ---------------------------------------------------
      float o0[N3P], o1[N3P];
#pragma unroll
      for (int j = 0; j < N3P; j++) o0[j] = o1[j] = 0.0f;
      const float* W3 = S.w + Blob::w3;
#pragma unroll 4
      for (int k = 0; k < kHidden; k++) {
        float a0 = X[k * kPanelLd + lane];
        float a1 = X[k * kPanelLd + 32 + lane];
#pragma unroll
        for (int j4 = 0; j4 < N3P; j4 += 4) {
          float4 w = *reinterpret_cast<const float4*>(W3 + k * N3P + j4);
          o0[j4 + 0] = __fmaf_rn(a0, w.x, o0[j4 + 0]);
          o0[j4 + 1] = __fmaf_rn(a0, w.y, o0[j4 + 1]);
          o0[j4 + 2] = __fmaf_rn(a0, w.z, o0[j4 + 2]);
          o0[j4 + 3] = __fmaf_rn(a0, w.w, o0[j4 + 3]);
          o1[j4 + 0] = __fmaf_rn(a1, w.x, o1[j4 + 0]);
          o1[j4 + 1] = __fmaf_rn(a1, w.y, o1[j4 + 1]);
          o1[j4 + 2] = __fmaf_rn(a1, w.z, o1[j4 + 2]);
          o1[j4 + 3] = __fmaf_rn(a1, w.w, o1[j4 + 3]);
        }
      }
      const float* B3 = S.w + Blob::b3;
#pragma unroll
      for (int q = 0; q < 2; q++) {
        if (slot[q] < 0) continue;
        float* o = q ? o1 : o0;
        if (!IS_COLOR) {
          float d = __fadd_rn(o[0], B3[0]);
          if (P.out_first) P.out_first[slot[q]] = d;
          if (P.out_full) {
            float* row = P.out_full + (size_t)slot[q] * N3;
            row[0] = d;
#pragma unroll
            for (int j = 1; j < N3; j++) row[j] = __fadd_rn(o[j], B3[j]);
          }
        } else {
          float* row = P.out_full + (size_t)slot[q] * N3;
#pragma unroll
          for (int j = 0; j < N3; j++) row[j] = np_sigmoidf(__fadd_rn(o[j], B3[j]));
        }
      }
    }
    // loop: the __syncthreads at the top orders these reads of S.w before the next bulk copy
  }
}

using SdfKernelSmem = MlpSmem<kSdfIn, kSdfOut, kSdfOutPad, ACT_SOFTPLUS, false>;
using ColKernelSmem = MlpSmem<kColIn, kColOut, kColOutPad, ACT_RELU, true>;

}  // namespace knf
