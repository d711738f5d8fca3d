// knf_mlp.cuh -- fused tiny-MLP tile kernels (north_star subsystem 2).
//
// Replaces nn.fourier_encode (nn.py:66-93) + grid.grid_forward (grid.py:241-294) + the
// activations (nn.py:26-50) for one family of per-cell MLPs.
//
// Work unit: a *tile* = up to 64 evaluation requests that fall in the same grid cell (produced by
// the routing pass, knf_route.cuh).  ONE WARP owns a tile (one-warp CTAs, 10 per SM): no block
// barriers, so a warp never waits for a slower sibling (the 4-warp version spent 21 % of its
// samples at the per-tile __syncthreads, ncu v3):
//   * lane 0 pulls the cell's 10.9 KB weight blob into shared memory with ONE TMA bulk copy
//     (cp.async.bulk -> UBLKCP) signalled on an mbarrier; the copy overlaps the encode;
//   * the warp encodes its 64 points (NumPy-exact sin/cos + the fp32 double-angle recurrence)
//     into a k-major shared-memory panel X[k][64];
//   * hidden layers are register-tiled SGEMMs: every lane accumulates an 8 point x 8 neuron
//     block, reading 8 activations + 8 weights (4 LDS.128) per k for 64 FFMAs.  The k loop is
//     sequential from k = 0 with one FFMA per step and the bias is added afterwards as its own
//     rounded add -- exactly the arithmetic OpenBLAS sgemm + NumPy's `+ b` perform in the
//     reference's per-cell path, so given the same layer inputs the pre-activations are
//     bit-identical to the reference's;
//   * pre-activations go back into the SAME panel (the layer's inputs are dead once every lane
//     holds its accumulators), and softplus runs over the panel in a rolled loop -- one copy of
//     the softplus code instead of 128 inlined ones keeps the kernel inside the instruction
//     cache (ncu on the first version: "no_instruction" was the top stall);
//   * the 32 -> N3 output layer is evaluated two points per lane and written straight to the
//     caller's buffers in request order (no unsort pass).
// Shared memory: 10.9 KB weights + 10.6 KB panel = 21.5 KB per one-warp CTA -> 10 CTAs per SM.
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
  const float4* sorted;        // march kernels: sorted position -> (point, ray id bits in .w)
  // colour inputs (request slot -> row)
  const float* col_v;          // (n,3) fp32 view dirs
  const float* col_n;          // (n,3) fp32 normals
  const float* col_z;          // (n,F) fp32 features
  // outputs, indexed by request slot
  float* out_first;            // SDF: distance per slot (nullable)
  float* out_full;             // SDF: (n, 1+F) rows; colour: (n,3) rows (nullable)
};

template <int K1, int N3P>
struct MlpSmem {
  using Blob = BlobLayout<K1, N3P>;
  alignas(16) float w[Blob::floats];
  alignas(16) float x[pad_k(K1) * kPanelLd];  // the warp's activation panel, reused by every layer
  alignas(8) uint64_t bar;
};

__device__ __forceinline__ float2 splat(float v) { return make_float2(v, v); }

// acc[ip][j] = (point 2ip, point 2ip+1) x neuron j: sum_k In[k][pt] * Wt[k][nr], k ascending, one
// IEEE fma per k and lane -- issued as packed FFMA2 (Blackwell fma.rn.f32x2: the weight is the
// scalar-broadcast operand, two points share an instruction), which halves the issue slots of the
// FFMA stream without changing a bit of the result.
struct LayerOperands {
  float4 xa, xb, wa, wb;
};
__device__ __forceinline__ void load_operands(LayerOperands& o, const float* __restrict__ xp, const float* __restrict__ wp,
                                              int k) {
  o.xa = *reinterpret_cast<const float4*>(xp + k * kPanelLd);
  o.xb = *reinterpret_cast<const float4*>(xp + k * kPanelLd + 32);
  o.wa = *reinterpret_cast<const float4*>(wp + k * kHidden);
  o.wb = *reinterpret_cast<const float4*>(wp + k * kHidden + 16);
}
__device__ __forceinline__ void fma_block(const LayerOperands& o, float2 (&acc)[4][8]) {
  const float2 xs[4] = {make_float2(o.xa.x, o.xa.y), make_float2(o.xa.z, o.xa.w), make_float2(o.xb.x, o.xb.y),
                        make_float2(o.xb.z, o.xb.w)};
  const float ws[8] = {o.wa.x, o.wa.y, o.wa.z, o.wa.w, o.wb.x, o.wb.y, o.wb.z, o.wb.w};
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = __ffma2_rn(xs[i], splat(ws[j]), acc[i][j]);
}

// K is a multiple of 8: the k loop runs as fully unrolled chunks of 8 steps (288 instructions,
// ptxas pipelines the LDS inside the chunk).  Rolled-up variants made ptxas rotate the operand
// registers with ~30 MOVs per iteration (ncu v3/v4: 9-13 % of all issued instructions).
template <int K>
__device__ __forceinline__ void layer_8x8(const float* __restrict__ In, const float* __restrict__ Wt, int pg, int ng,
                                          float2 (&acc)[4][8]) {
  static_assert(K % 8 == 0, "pad K to a multiple of 8");
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.0f, 0.0f);
  const float* xp = In + pg * 4;
  const float* wp = Wt + ng * 4;
#ifndef KNF_LAYER_CHUNK
#define KNF_LAYER_CHUNK 8
#endif
  constexpr int kChunk = KNF_LAYER_CHUNK == 0 ? K : KNF_LAYER_CHUNK;
  static_assert(K % kChunk == 0, "chunk must divide K");
#pragma unroll 1
  for (int k0 = 0; k0 < K; k0 += kChunk) {
#pragma unroll
    for (int kk = 0; kk < kChunk; kk++) {
      LayerOperands o;
      load_operands(o, xp, wp, k0 + kk);
      fma_block(o, acc);
    }
    // keep ptxas from prefetching the next chunk's operands across the back-edge: that rotation cost
    // ~35 MOVs per chunk (ncu v5); the other resident warps cover the one exposed LDS latency
    asm volatile("" ::: "memory");
  }
}

// Out[neuron][point] = act(acc + b), k-major panel for the next layer.  RELU is applied here;
// SOFTPLUS stores the pre-activation and leaves the transcendental to softplus_panel().
template <int ACT>
__device__ __forceinline__ void store_hidden(float2 (&acc)[4][8], const float* __restrict__ bias,
                                             float* __restrict__ Out, int pg, int ng) {
#pragma unroll
  for (int j = 0; j < 8; j++) {
    int neuron = (j < 4) ? (ng * 4 + j) : (16 + ng * 4 + (j - 4));
    float2 b = splat(bias[neuron]);
    float2 v[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      v[i] = __fadd2_rn(acc[i][j], b);
      if (ACT == ACT_RELU) v[i] = make_float2(fmaxf(v[i].x, 0.0f), fmaxf(v[i].y, 0.0f));
    }
    *reinterpret_cast<float4*>(Out + neuron * kPanelLd + pg * 4) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
    *reinterpret_cast<float4*>(Out + neuron * kPanelLd + 32 + pg * 4) = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
  }
}

// In-place softplus over a 32 x 64 panel: lane owns the adjacent columns 2*lane, 2*lane+1 and
// runs both through one packed evaluation (LDS.64 / STS.64, conflict-free).
#ifndef KNF_SP_UNROLL
#define KNF_SP_UNROLL 4
#endif
constexpr int kSoftplusUnroll = KNF_SP_UNROLL;
// __noinline__: the exact kernel calls this four times per pass shape; one copy keeps it inside the instruction cache
// (ncu on the 97 KB version: no_instruction was the top stall, 1.9 per issue).
static __device__ __noinline__ void softplus_panel(float* __restrict__ panel, int lane) {
#pragma unroll 1
  for (int j = 0; j < kHidden; j += kSoftplusUnroll) {
    float2 v[kSoftplusUnroll];
#pragma unroll
    for (int u = 0; u < kSoftplusUnroll; u++) v[u] = *reinterpret_cast<float2*>(panel + (j + u) * kPanelLd + 2 * lane);
    softplus_tile<kSoftplusUnroll>(v);
#pragma unroll
    for (int u = 0; u < kSoftplusUnroll; u++) *reinterpret_cast<float2*>(panel + (j + u) * kPanelLd + 2 * lane) = v[u];
  }
}

// Column swizzle of the compact panels (mid: 32 columns, small: 16).  A lane of the register-tiled layers stores its
// pre-activations as float4 at (row = neuron, columns 4 pg ..): with the plain layout the row strides 8 * 36 and 4 * 20 words
// are multiples of 32 and 16 banks, so the lanes of one 8-lane store phase that differ only in their neuron group hit the same
// banks -- 4-way conflicts on every STS.128 of store_hidden_mid / _small (ncu: 16 % of the mid kernel's shared-memory
// wavefronts were excess).  XOR-ing the float4-column index with a function of row / 8 spreads them over all banks; every
// reader and writer of these panels goes through panel_col (the in-place softplus does not care where a column lives).
template <int PLD>
__device__ __forceinline__ int panel_col4(int row, int c4) { return c4; }  // physical float4-column of logical float4-column c4 in `row` (other strides: plain)
constexpr int kMidPanelLdFwd = 36, kSmallPanelLdFwd = 20;  // (= kMidPanelLd / kSmallPanelLd, defined with their tile shapes below)
template <>
__device__ __forceinline__ int panel_col4<kMidPanelLdFwd>(int row, int c4) { return c4 ^ (((row >> 3) & 3) << 1); }
template <>
__device__ __forceinline__ int panel_col4<kSmallPanelLdFwd>(int row, int c4) { return c4 ^ ((row >> 3) & 3); }
template <int PLD>
__device__ __forceinline__ int panel_col(int row, int p) { return 4 * panel_col4<PLD>(row, p >> 2) + (p & 3); }

// nn.fourier_encode (nn.py:66-93) of a 3-vector into rows [0, 3 + 6*L) of a swizzled compact panel at logical column p.
template <int L, int PLD>
static __device__ __noinline__ void encode_into_swz(float* __restrict__ panel, int p, float x, float y, float z) {
  const float pi_f = 3.14159274101257324e+00f;  // float32(np.pi)
  panel[0 * PLD + panel_col<PLD>(0, p)] = x;
  panel[1 * PLD + panel_col<PLD>(1, p)] = y;
  panel[2 * PLD + panel_col<PLD>(2, p)] = z;
  float s[3], c[3];
  np_sincosf(__fmul_rn(pi_f, x), s[0], c[0]);
  np_sincosf(__fmul_rn(pi_f, y), s[1], c[1]);
  np_sincosf(__fmul_rn(pi_f, z), s[2], c[2]);
#pragma unroll
  for (int o = 0; o < L; o++) {
    const int r = 3 + 6 * o;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      panel[(r + a) * PLD + panel_col<PLD>(r + a, p)] = s[a];
      panel[(r + 3 + a) * PLD + panel_col<PLD>(r + 3 + a, p)] = c[a];
      float two_s = __fmul_rn(2.0f, s[a]);
      float ns = __fmul_rn(two_s, c[a]);                      // 2 s c
      float nc = __fsub_rn(1.0f, __fmul_rn(two_s, s[a]));     // 1 - 2 s s
      s[a] = ns;
      c[a] = nc;
    }
  }
}

// nn.fourier_encode (nn.py:66-93) of a 3-vector into panel rows [row0, row0 + 3 + 6*L) at column p.
// __noinline__ (one copy per instantiation): three sin/cos evaluations and the recurrence are ~300 instructions, and
// the exact kernel used to inline them three times.
template <int L, int PLD = kPanelLd>
static __device__ __noinline__ void encode_into(float* __restrict__ panel, int row0, int p, float x, float y, float z) {
  constexpr int kPanelLd = PLD;  // row stride of this panel
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

// Rows K1 .. pad_k(K1)-1 of the input panel must be zero for the lane's two columns.
template <int K1>
__device__ __forceinline__ void zero_pad_rows(float* __restrict__ X, int lane) {
#pragma unroll
  for (int r = K1; r < pad_k(K1); r++) *reinterpret_cast<float2*>(X + r * kPanelLd + 2 * lane) = make_float2(0.f, 0.f);
}

// ---- the same arithmetic for a SMALL tile (<= 16 points in panel columns 0..15) ---------------------------------
// Late in a march the exact queue holds a handful of rays per cell; a 64-column pass would spend 3/4 of its FFMA2
// on empty columns.  Here a lane accumulates 4 points x 4 neurons (4 point groups x 8 neuron groups), one LDS.128
// of activations + one of weights per 8 FFMA2.  Every output is still the k-ordered FMA chain from zero followed by
// the rounded bias add, so a point's value does not depend on which tile shape evaluated it.
constexpr int kSmallTilePts = 16;

constexpr int kSmallPanelLd = kSmallTilePts + 4;  // 20: row stride of the compact panel of the small-tile kernel
static_assert(kSmallPanelLd == kSmallPanelLdFwd, "panel_col4 is specialised for this stride");

template <int K, int PLD>
__device__ __forceinline__ void layer_4x4(const float* __restrict__ In, const float* __restrict__ Wt, int pg, int ng,
                                          float2 (&acc)[2][4]) {
  constexpr int kPanelLd = PLD;
  static_assert(K % 8 == 0, "pad K to a multiple of 8");
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.0f, 0.0f);
  const float* wp = Wt + ng * 4;
#pragma unroll 1
  for (int k0 = 0; k0 < K; k0 += 8) {
    const float* xp = In + 4 * panel_col4<PLD>(k0, pg);  // (rows k0 .. k0 + 7 share one swizzle)
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
      const float4 x = *reinterpret_cast<const float4*>(xp + (k0 + kk) * kPanelLd);
      const float4 w = *reinterpret_cast<const float4*>(wp + (k0 + kk) * kHidden);
      const float2 x01 = make_float2(x.x, x.y), x23 = make_float2(x.z, x.w);
      const float ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 4; j++) {
        acc[0][j] = __ffma2_rn(x01, splat(ws[j]), acc[0][j]);
        acc[1][j] = __ffma2_rn(x23, splat(ws[j]), acc[1][j]);
      }
    }
  }
}

template <int ACT, int PLD>
__device__ __forceinline__ void store_hidden_small(float2 (&acc)[2][4], const float* __restrict__ bias, float* __restrict__ Out,
                                                   int pg, int ng) {
  constexpr int kPanelLd = PLD;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int neuron = ng * 4 + j;
    const float2 b = splat(bias[neuron]);
    float2 v0 = __fadd2_rn(acc[0][j], b), v1 = __fadd2_rn(acc[1][j], b);
    if (ACT == ACT_RELU) {
      v0 = make_float2(fmaxf(v0.x, 0.0f), fmaxf(v0.y, 0.0f));
      v1 = make_float2(fmaxf(v1.x, 0.0f), fmaxf(v1.y, 0.0f));
    }
    *reinterpret_cast<float4*>(Out + neuron * kPanelLd + 4 * panel_col4<PLD>(neuron, pg)) = make_float4(v0.x, v0.y, v1.x, v1.y);
  }
}

// In-place softplus over panel rows 0..31, columns 0..15: lane owns columns 2 (lane & 7), +1 of rows (lane >> 3) + 4 i.
template <int PLD>
static __device__ __noinline__ void softplus_panel_small(float* __restrict__ panel, int lane) {
  constexpr int kPanelLd = PLD;
  float* base = panel + (lane >> 3) * kPanelLd + 2 * (lane & 7);
#pragma unroll 1
  for (int i0 = 0; i0 < 8; i0 += 4) {
    float2 v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = *reinterpret_cast<float2*>(base + 4 * (i0 + u) * kPanelLd);
    softplus_tile<4>(v);
#pragma unroll
    for (int u = 0; u < 4; u++) *reinterpret_cast<float2*>(base + 4 * (i0 + u) * kPanelLd) = v[u];
  }
}

template <int K1, int N3P, int HIDDEN_ACT, int PLD>
__device__ __forceinline__ void hidden_layers_small(float* __restrict__ X, const float* __restrict__ W, int lane) {
  using Blob = BlobLayout<K1, N3P>;
  const int pg = lane >> 3;  // 4 point groups of 4 points
  const int ng = lane & 7;   // 8 neuron groups of 4 neurons
  float2 acc[2][4];
  layer_4x4<pad_k(K1), PLD>(X, W + Blob::w1, pg, ng, acc);
  __syncwarp();
  store_hidden_small<HIDDEN_ACT, PLD>(acc, W + Blob::b1, X, pg, ng);
  __syncwarp();
  if (HIDDEN_ACT == ACT_SOFTPLUS) {
    softplus_panel_small<PLD>(X, lane);
    __syncwarp();
  }
  layer_4x4<kHidden, PLD>(X, W + Blob::w2, pg, ng, acc);
  __syncwarp();
  store_hidden_small<HIDDEN_ACT, PLD>(acc, W + Blob::b2, X, pg, ng);
  __syncwarp();
  if (HIDDEN_ACT == ACT_SOFTPLUS) {
    softplus_panel_small<PLD>(X, lane);
    __syncwarp();  // the output layer reads column `lane`, written by other lanes
  }
}


// ---- the same arithmetic for a MID tile (<= 32 points, panel column = lane) ----------------------------------------
// Dense wavefronts of the exact march: a lane accumulates 4 points x 8 neurons (8 point groups x 4 neuron groups), 32
// accumulator registers instead of the 128 of the 8 x 8 tiles, so 13 one-warp CTAs share an SM instead of 8.  Every
// output is still the k-ordered FMA chain from zero followed by the rounded bias add: same bits as the other shapes.
constexpr int kMidTilePts = 32;
constexpr int kMidPanelLd = kMidTilePts + 4;  // 36
static_assert(kMidPanelLd == kMidPanelLdFwd, "panel_col4 is specialised for this stride");

template <int K, int PLD>
__device__ __forceinline__ void layer_4x8(const float* __restrict__ In, const float* __restrict__ Wt, int pg, int ng, float2 (&acc)[2][8]) {
  static_assert(K % 8 == 0, "pad K to a multiple of 8");
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.0f, 0.0f);
  const float* wp = Wt + ng * 8;
#pragma unroll 1
  for (int k0 = 0; k0 < K; k0 += 8) {
    const float* xp = In + 4 * panel_col4<PLD>(k0, pg);  // (rows k0 .. k0 + 7 share one swizzle)
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
      const float4 x = *reinterpret_cast<const float4*>(xp + (k0 + kk) * PLD);
      const float4 wa = *reinterpret_cast<const float4*>(wp + (k0 + kk) * kHidden);
      const float4 wb = *reinterpret_cast<const float4*>(wp + (k0 + kk) * kHidden + 4);
      const float2 x01 = make_float2(x.x, x.y), x23 = make_float2(x.z, x.w);
      const float ws[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
      for (int j = 0; j < 8; j++) {
        acc[0][j] = __ffma2_rn(x01, splat(ws[j]), acc[0][j]);
        acc[1][j] = __ffma2_rn(x23, splat(ws[j]), acc[1][j]);
      }
    }
    asm volatile("" ::: "memory");  // (as in layer_8x8: no operand prefetch across the back-edge)
  }
}

template <int ACT, int PLD>
__device__ __forceinline__ void store_hidden_mid(float2 (&acc)[2][8], const float* __restrict__ bias, float* __restrict__ Out, int pg, int ng) {
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const int neuron = ng * 8 + j;
    const float2 b = splat(bias[neuron]);
    float2 v0 = __fadd2_rn(acc[0][j], b), v1 = __fadd2_rn(acc[1][j], b);
    if (ACT == ACT_RELU) {
      v0 = make_float2(fmaxf(v0.x, 0.0f), fmaxf(v0.y, 0.0f));
      v1 = make_float2(fmaxf(v1.x, 0.0f), fmaxf(v1.y, 0.0f));
    }
    *reinterpret_cast<float4*>(Out + neuron * PLD + 4 * panel_col4<PLD>(neuron, pg)) = make_float4(v0.x, v0.y, v1.x, v1.y);
  }
}

// In-place softplus over panel rows 0..31, columns 0..31: lane owns columns 2 (lane & 15), +1 of rows (lane >> 4) + 2 i.
template <int PLD>
static __device__ __noinline__ void softplus_panel_mid(float* __restrict__ panel, int lane) {
  float* base = panel + (lane >> 4) * PLD + 2 * (lane & 15);
#pragma unroll 1
  for (int i0 = 0; i0 < 16; i0 += 4) {
    float2 v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = *reinterpret_cast<float2*>(base + 2 * (i0 + u) * PLD);
    softplus_tile<4>(v);
#pragma unroll
    for (int u = 0; u < 4; u++) *reinterpret_cast<float2*>(base + 2 * (i0 + u) * PLD) = v[u];
  }
}

template <int K1, int N3P, int HIDDEN_ACT, int PLD>
__device__ __forceinline__ void hidden_layers_mid(float* __restrict__ X, const float* __restrict__ W, int lane) {
  using Blob = BlobLayout<K1, N3P>;
  const int pg = lane >> 2;  // 8 point groups of 4 points
  const int ng = lane & 3;   // 4 neuron groups of 8 neurons
  float2 acc[2][8];
  layer_4x8<pad_k(K1), PLD>(X, W + Blob::w1, pg, ng, acc);
  __syncwarp();
  store_hidden_mid<HIDDEN_ACT, PLD>(acc, W + Blob::b1, X, pg, ng);
  __syncwarp();
  if (HIDDEN_ACT == ACT_SOFTPLUS) {
    softplus_panel_mid<PLD>(X, lane);
    __syncwarp();
  }
  layer_4x8<kHidden, PLD>(X, W + Blob::w2, pg, ng, acc);
  __syncwarp();
  store_hidden_mid<HIDDEN_ACT, PLD>(acc, W + Blob::b2, X, pg, ng);
  __syncwarp();
  if (HIDDEN_ACT == ACT_SOFTPLUS) {
    softplus_panel_mid<PLD>(X, lane);
    __syncwarp();  // the output layer reads column `lane`, written by other lanes
  }
}

// Output 0 (the distance) of the 32 -> N3 layer for panel column p (same chain as output_distance).
template <int N3P, int PLD>
__device__ __forceinline__ float output_distance_col(const float* __restrict__ X, const float* __restrict__ W3,
                                                     const float* __restrict__ B3, int p) {
  constexpr int kPanelLd = PLD;
  float d = 0.0f;
#pragma unroll
  for (int k0 = 0; k0 < kHidden; k0 += 8) {
    const int pc = panel_col<PLD>(k0, p);  // the swizzled column of rows k0 .. k0 + 7
#pragma unroll
    for (int kk = 0; kk < 8; kk++) d = __fmaf_rn(X[(k0 + kk) * kPanelLd + pc], W3[(k0 + kk) * N3P], d);
  }
  return __fadd_rn(d, B3[0]);
}

// Layers 1 and 2 (+ activations) of one 64-point warp tile; leaves h2 in the panel.
template <int K1, int N3P, int HIDDEN_ACT>
__device__ __forceinline__ void hidden_layers(float* __restrict__ X, const float* __restrict__ W, int lane) {
  using Blob = BlobLayout<K1, N3P>;
  const int pg = lane >> 2;  // 8 point groups of 4(+4) points
  const int ng = lane & 3;   // 4 neuron groups of 4(+4) neurons
  float2 acc[4][8];
  layer_8x8<pad_k(K1)>(X, W + Blob::w1, pg, ng, acc);
  __syncwarp();  // every lane holds its accumulators: the input rows are dead
  store_hidden<HIDDEN_ACT>(acc, W + Blob::b1, X, pg, ng);
  __syncwarp();
  if (HIDDEN_ACT == ACT_SOFTPLUS) {
    softplus_panel(X, lane);
    __syncwarp();
  }
  layer_8x8<kHidden>(X, W + Blob::w2, pg, ng, acc);
  __syncwarp();
  store_hidden<HIDDEN_ACT>(acc, W + Blob::b2, X, pg, ng);
  __syncwarp();
  if (HIDDEN_ACT == ACT_SOFTPLUS) softplus_panel(X, lane);  // the output layer reads back only the lane's own columns
}

// Output 0 (the distance) of the 32 -> N3 layer for the lane's two columns.
template <int N3P>
__device__ __forceinline__ float2 output_distance(const float* __restrict__ X, const float* __restrict__ W3,
                                                  const float* __restrict__ B3, int lane) {
  const float* Xc = X + 2 * lane;
  float2 d = make_float2(0.0f, 0.0f);
#pragma unroll 8
  for (int k = 0; k < kHidden; k++)
    d = __ffma2_rn(*reinterpret_cast<const float2*>(Xc + k * kPanelLd), splat(W3[k * N3P]), d);
  return __fadd2_rn(d, splat(B3[0]));
}

// Weight fetch for one tile: one elected lane arms the mbarrier and issues the TMA bulk copy.
template <class Blob>
__device__ __forceinline__ void fetch_weights(float* smem_w, const float* __restrict__ blobs, int cell, uint64_t* bar,
                                              int lane) {
  if (lane == 0) {
    fence_proxy_async();
    mbar_expect_tx(bar, Blob::bytes);
    bulk_copy_g2s(smem_w, blobs + (size_t)cell * Blob::floats, Blob::bytes, bar);
  }
}

__device__ __forceinline__ int next_tile(RouteCounters* ctr, int lane) {
  int t = 0;
  if (lane == 0) t = atomicAdd(&ctr->tile_cursor, 1);
  return __shfl_sync(0xffffffffu, t, 0);
}

// Batched-forward kernel (grid.sdf_query / color_query, shading probes): ONE WARP per CTA, each
// warp a persistent worker that pulls 64-request tiles from the routing pass's tile list.
template <int K1, int N3, int N3P, int HIDDEN_ACT, bool IS_COLOR>
static __global__ void __launch_bounds__(32, kFwdCtasPerSm) mlp_warp_kernel(MlpParams P) {
  using Blob = BlobLayout<K1, N3P>;
  using Smem = MlpSmem<K1, N3P>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const int n_tiles = P.ctr->n_tiles;
  uint32_t parity = 0;
  float* X = S.x;

  for (;;) {
    const int t = next_tile(P.ctr, lane);
    if (t >= n_tiles) break;
    const Tile tile = P.tiles[t];
    fetch_weights<Blob>(S.w, P.blobs, tile.cell, &S.bar, lane);

    int slot[2] = {-1, -1};
#pragma unroll
    for (int q = 0; q < 2; q++) {
      int p = 2 * lane + q;  // the lane's two adjacent panel columns
      float px = 0.f, py = 0.f, pz = 0.f;
      if (p < tile.count) {
        slot[q] = P.perm[tile.start + p];
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
        if (p < tile.count) {
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
    zero_pad_rows<K1>(X, lane);
    __syncwarp();
    mbar_wait(&S.bar, parity);  // weights have landed
    parity ^= 1;

    hidden_layers<K1, N3P, HIDDEN_ACT>(X, S.w, lane);

    const float* W3 = S.w + Blob::w3;
    const float* B3 = S.w + Blob::b3;
    if (!IS_COLOR && P.out_full == nullptr) {
      float2 d = output_distance<N3P>(X, W3, B3, lane);
      if (slot[0] >= 0) P.out_first[slot[0]] = d.x;
      if (slot[1] >= 0) P.out_first[slot[1]] = d.y;
    } else {
      const float* Xc = X + 2 * lane;
      float2 o01[N3P];
#pragma unroll
      for (int j = 0; j < N3P; j++) o01[j] = make_float2(0.0f, 0.0f);
#pragma unroll 4
      for (int k = 0; k < kHidden; k++) {
        float2 a = *reinterpret_cast<const float2*>(Xc + k * kPanelLd);
#pragma unroll
        for (int j4 = 0; j4 < N3P; j4 += 4) {
          float4 w = *reinterpret_cast<const float4*>(W3 + k * N3P + j4);
          o01[j4 + 0] = __ffma2_rn(a, splat(w.x), o01[j4 + 0]);
          o01[j4 + 1] = __ffma2_rn(a, splat(w.y), o01[j4 + 1]);
          o01[j4 + 2] = __ffma2_rn(a, splat(w.z), o01[j4 + 2]);
          o01[j4 + 3] = __ffma2_rn(a, splat(w.w), o01[j4 + 3]);
        }
      }
#pragma unroll
      for (int q = 0; q < 2; q++) {
        if (slot[q] < 0) continue;
        float* row = P.out_full + (size_t)slot[q] * N3;
#pragma unroll
        for (int j = 0; j < N3; j++) {
          float v = __fadd_rn(q ? o01[j].y : o01[j].x, B3[j]);
          if (IS_COLOR) v = np_sigmoidf(v);
          row[j] = v;
          if (!IS_COLOR && j == 0 && P.out_first) P.out_first[slot[q]] = v;
        }
      }
    }
    __syncwarp();  // every lane is done reading S.w and the panel before the next tile overwrites them
  }
}

// Shared memory of the small-tile-only kernel: the same weight blob, a 40 x 20 panel -- 14.3 KB, 14 one-warp CTAs per SM.
template <int K1, int N3P>
struct SmallSmem {
  using Blob = BlobLayout<K1, N3P>;
  alignas(16) float w[Blob::floats];
  alignas(16) float x[pad_k(K1) * kSmallPanelLd];
  alignas(8) uint64_t bar;
};
// ... and of the mid-tile kernel: a 40 x 36 panel -- 16.8 KB, 13 one-warp CTAs per SM.
template <int K1, int N3P>
struct MidSmem {
  using Blob = BlobLayout<K1, N3P>;
  alignas(16) float w[Blob::floats];
  alignas(16) float x[pad_k(K1) * kMidPanelLd];
  alignas(8) uint64_t bar;
};
using SdfMidSmem = MidSmem<kSdfIn, kSdfOutPad>;
using SdfKernelSmem = MlpSmem<kSdfIn, kSdfOutPad>;
using SdfSmallSmem = SmallSmem<kSdfIn, kSdfOutPad>;
using ColKernelSmem = MlpSmem<kColIn, kColOutPad>;

}  // namespace knf
