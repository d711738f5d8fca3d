// knf_mma.cuh -- the SDF tile MLP on the tensor cores (north_star subsystem 2: "hidden layers as
// warp-level mma tiles where the per-cell batch is a real dense contraction").
//
// Same work unit as knf_mlp.cuh (one warp owns a tile of <= 64 requests of one cell), same inputs,
// same outputs, different arithmetic for the two hidden contractions (39->32, 32->32):
//
//   * every fp32 operand is split EXACTLY into three bf16 pieces, x = x1 + x2 + x3 (8 significand
//     bits each, round-to-nearest splits), weights once on the host, activations in registers;
//   * x.w is evaluated as the six piece products x1w1 + x1w2 + x2w1 + x2w2 + x1w3 + x3w1 (every
//     bf16 x bf16 product is exact in fp32; the three dropped terms are <= 2^-26 of |x||w|, measured
//     7e-9 mean absolute on a 32-term dot) with mma.sync.m16n8k16 bf16 -> fp32 (SASS HMMA.16816.F32.BF16);
//   * the five small products accumulate in one fp32 accumulator, x1w1 in another, and the two are
//     added with one rounded add: measured on B200 (scripts/micro/hmma_split.cu, profiles/hmma_split_r1.txt)
//     the result is 3x CLOSER to the exact dot product than the reference's own k-ordered fp32 FMA
//     chain (mean |err| 4.1e-8 vs 1.2e-7 at K = 32), so it differs from the reference by the
//     reference's own rounding error and nothing else.  It is not bit-identical to the chain: the
//     chain kernels (knf_mlp.cuh) remain available as KNF_PRECISION_FP32_CHAIN.
//
// Layers are chained in REGISTERS: the m16n8 accumulator fragment of layer l (rows g, g+8; columns
// 2t, 2t+1 of each 8-wide n-tile) is exactly the m16k16 A fragment of layer l+1, so bias, softplus and
// the bf16 split run on the accumulator registers and no activation ever touches shared memory.  The
// first layer's A fragments are produced in place as well: the Fourier features are ordered so that
// lane t of a quad owns axis t's twelve sin/cos values (t = 3 owns the raw coordinates), i.e. each
// lane runs nn.fourier_encode's recurrence for one axis of its eight rows.  Shared memory holds only
// the cell's weight fragments (one TMA bulk copy) and a 64 x 3 coordinate exchange.
//
// Work per 64-point pass and warp: 480 HMMA (bf16 x 3) or 240 (fp16 x 2) on the tensor pipe + 64 packed softplus +
// ~80 operand splits (FMA / ALU pipes) instead of 2336 FFMA2 + 64 packed softplus.
//
// Three users: sdf_mma_kernel (batched forward in the KNF_PRECISION_TENSOR_* modes), march_mma_kernel<P, false>
// (the march in those modes) and march_mma_kernel<2, true> -- the DECISION FILTER of the exact mode (knf_march.cuh),
// which is where the default configuration spends most of its time.
#pragma once

#include "knf_common.cuh"
#include "knf_mlp.cuh"
#include "knf_rays.cuh"

namespace knf {

// ---- per-cell blob for the MMA path -------------------------------------------------------------
// P = pieces per operand: 3 -> bf16 x 3 (exact split, six products), 2 -> fp16 x 2 (22-23 significand bits, the
// second piece scaled by 2^11 to stay normal, three products).
//   frag1[kt 0..2][nt 0..3][lane 0..31][piece 0..P-1] uint2   B fragments of W1 (K order permuted, see mma_feature_of)
//   frag2[kt 0..1][nt 0..3][lane 0..31][piece 0..P-1] uint2   B fragments of W2   (P = 2: one LDS.128 per lane)
//   b1[32] b2[32] fp32 | w3d[32] fp32 (output-layer column 0: the distance) | b3[12] fp32      <- march kernels copy up to here
//   W3t[32][12] fp32 (k-major, like BlobLayout: all nine outputs, batched-forward kernel only)
template <int P>
struct MmaBlobT {
  static constexpr int pieces = P;
  static constexpr int kt1 = 3, kt2 = 2;
  static constexpr int frag1 = 0;  // in 32-bit words
  static constexpr int frag2 = frag1 + kt1 * 4 * P * 32 * 2;
  static constexpr int b1 = frag2 + kt2 * 4 * P * 32 * 2;
  static constexpr int b2 = b1 + kHidden;
  static constexpr int w3d = b2 + kHidden;
  static constexpr int b3 = w3d + kHidden;
  static constexpr int march_words = b3 + kSdfOutPad + 4;  // + 4 words of filter constants; P = 3: 3952 (15808 B), P = 2: 2672 (10688 B)
  static constexpr int w3 = march_words;
  static constexpr int words = w3 + kHidden * kSdfOutPad;  // P = 3: 4336 (17344 B); P = 2: 3056 (12224 B)
  static constexpr int bytes = words * 4;
  static constexpr int march_bytes = march_words * 4;
  static_assert(bytes % 16 == 0 && march_bytes % 16 == 0, "blob (parts) must be multiples of 16 B for cp.async.bulk");
};
using MmaBlob = MmaBlobT<3>;
using MmaBlobH = MmaBlobT<2>;
// per-cell constants of the decision filter, stored after b3 (b3[9..11] = per-axis Lipschitz bounds, then 4 words):
constexpr int kFilterLipSlot = kSdfOut;           // b3[9 + a]: proven bound on |d d / d x_a| over the cell, a = 0, 1, 2
constexpr int kFilterDeltaSlot = kSdfOutPad;      // b3[12]: proven bound on |tensor distance - exact distance| in this cell
constexpr float kHalfPieceScale = 2048.0f;  // 2^11: the fp16 second piece carries (x - x1) * 2^11

// Which reference feature (nn.fourier_encode column, nn.py:84-93) sits at position `kslot` of k-tile
// `kt` of the permuted first-layer K axis; -1 = zero padding.  Lane t of a quad holds k = 2t, 2t+1,
// 2t+8, 2t+9 of every k-tile: (sin, cos) of octaves 2kt and 2kt+1 of axis t, or (x, y, z, 0) for t = 3.
__host__ __device__ inline int mma_feature_of(int kt, int kslot) {
  const int t = (kslot % 8) / 2;
  const int j = (kslot % 2) + 2 * (kslot / 8);
  if (t == 3) return (kt == 0 && j < 3) ? j : -1;
  const int octave = 2 * kt + j / 2;
  return 3 + 6 * octave + 3 * (j % 2) + t;
}

template <int P>
struct MmaSmemT {
  alignas(16) uint32_t w[MmaBlobT<P>::words];
  alignas(16) float pts[3][72];  // coordinate exchange: pts[axis][point], stride 72 keeps the quad reads conflict-free
  int slot[64];                  // batched-forward kernel: request slot of every tile point
  alignas(8) uint64_t bar;
};
// The march kernels also park the resident rays' origins and directions here (k-major: conflict-free 8-byte
// accesses) instead of in 48 registers per lane, which is what lets 13 one-warp CTAs share an SM.
template <int P>
struct MmaMarchSmemT {
  alignas(16) uint32_t w[MmaBlobT<P>::march_words];
  alignas(16) float pts[3][72];
  alignas(16) double od[6][64];  // [component][32 q + lane]: each lane touches only its own two slots
  alignas(8) uint64_t bar;
};

// ---- device helpers -------------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], const uint2 b) {
  if (P == 3)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

// (lo, hi) -> three packed bf16 pairs with lo + hi pieces summing exactly to the inputs.
__device__ __forceinline__ void split3(float lo, float hi, uint32_t& p1, uint32_t& p2, uint32_t& p3) {
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p1) : "f"(hi), "f"(lo));
  float rl = __fsub_rn(lo, __uint_as_float(p1 << 16));
  float rh = __fsub_rn(hi, __uint_as_float(p1 & 0xffff0000u));
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p2) : "f"(rh), "f"(rl));
  rl = __fsub_rn(rl, __uint_as_float(p2 << 16));
  rh = __fsub_rn(rh, __uint_as_float(p2 & 0xffff0000u));
  p3 = __byte_perm(__float_as_uint(rl), __float_as_uint(rh), 0x7632);  // the remainder is exact in bf16
}
// (lo, hi) -> packed fp16 pairs p1 = rn16(x), p2 = rn16((x - p1) * 2^11): x = p1 + p2 / 2^11 to 2^-24 relative.
__device__ __forceinline__ void split2h(float lo, float hi, uint32_t& p1, uint32_t& p2) {
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(p1) : "f"(hi), "f"(lo));
  float fl, fh;
  asm("{ .reg .f16 l, h; mov.b32 {l, h}, %2; cvt.f32.f16 %0, l; cvt.f32.f16 %1, h; }" : "=f"(fl), "=f"(fh) : "r"(p1));
  const float2 r = __fmul2_rn(__fadd2_rn(make_float2(lo, hi), make_float2(-fl, -fh)), make_float2(kHalfPieceScale, kHalfPieceScale));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(p2) : "f"(r.y), "f"(r.x));
}

// One 16-row x 16-k slab of activations, P pieces, in A-fragment registers.
template <int P>
struct APieces {
  uint32_t p[P][4];
};
// v0 = (row g: k 2t, 2t+1), v1 = (row g+8: same k), v2 = (row g: k 2t+8, 2t+9), v3 = (row g+8: same)
template <int P>
__device__ __forceinline__ void make_a(APieces<P>& A, float2 v0, float2 v1, float2 v2, float2 v3) {
  const float2 v[4] = {v0, v1, v2, v3};
#pragma unroll
  for (int i = 0; i < 4; i++) {
    if (P == 3) split3(v[i].x, v[i].y, A.p[0][i], A.p[1][i], A.p[P - 1][i]);
    else split2h(v[i].x, v[i].y, A.p[0][i], A.p[1][i]);
  }
}

// One layer of one m-tile.  HMMA issue order: k-tile, then piece product, then n-tile -- consecutive HMMAs hit
// different accumulators (an accumulator is revisited every 4th instruction), so a single warp keeps the tensor
// pipe busy without waiting on HMMA latency.
//   P = 3: small += x3w1 + x1w3 + x2w2 + x2w1 + x1w2 ; big += x1w1          (pre-activation = big + small)
//   P = 2: small += x2'w1 + x1w2'                    ; big += x1w1          (pre-activation = big + small / 2^11)
template <int P, int KT>
__device__ __forceinline__ void mma_layer(const APieces<P> (&A)[KT], const uint2* __restrict__ frag /* [kt][nt][lane][piece] */,
                                          int lane, float (&small)[4][4], float (&big)[4][4]) {
#pragma unroll
  for (int nt = 0; nt < 4; nt++)
#pragma unroll
    for (int i = 0; i < 4; i++) small[nt][i] = 0.0f;  // `big` arrives holding its initial value (zero, or the bias)
#pragma unroll
  for (int kt = 0; kt < KT; kt++) {
    uint2 w[4][P];
#pragma unroll
    for (int nt = 0; nt < 4; nt++) {
      const uint2* f = frag + ((kt * 4 + nt) * 32 + lane) * P;
      if (P == 2) {
        const uint4 q = *reinterpret_cast<const uint4*>(f);
        w[nt][0] = make_uint2(q.x, q.y);
        w[nt][1] = make_uint2(q.z, q.w);
      } else {
#pragma unroll
        for (int pc = 0; pc < P; pc++) w[nt][pc] = f[pc];
      }
    }
    if (P == 3) {
#pragma unroll
      for (int nt = 0; nt < 4; nt++) hmma<P>(small[nt], A[kt].p[P - 1], w[nt][0]);
#pragma unroll
      for (int nt = 0; nt < 4; nt++) hmma<P>(small[nt], A[kt].p[0], w[nt][P - 1]);
#pragma unroll
      for (int nt = 0; nt < 4; nt++) hmma<P>(small[nt], A[kt].p[1], w[nt][1]);
    }
#pragma unroll
    for (int nt = 0; nt < 4; nt++) hmma<P>(small[nt], A[kt].p[1], w[nt][0]);
#pragma unroll
    for (int nt = 0; nt < 4; nt++) hmma<P>(big[nt], A[kt].p[0], w[nt][0]);  // between the two small products: an accumulator is revisited every 8th HMMA
#pragma unroll
    for (int nt = 0; nt < 4; nt++) hmma<P>(small[nt], A[kt].p[0], w[nt][1]);
  }
}

// h = softplus(big + small [/ 2^11] + bias) on the accumulator fragments: eight independent packed evaluations in flight.
// The filter (FAST) starts the big accumulator at the bias instead of adding it afterwards (one packed add less per
// pair; the sum order differs from the other modes by design -- only the proven bound matters there).
template <bool FAST>
__device__ __forceinline__ void init_big(float (&big)[4][4], const float* __restrict__ bias, int t) {
#pragma unroll
  for (int nt = 0; nt < 4; nt++) {
    const float2 b = FAST ? *reinterpret_cast<const float2*>(bias + 8 * nt + 2 * t) : make_float2(0.0f, 0.0f);
    big[nt][0] = b.x; big[nt][1] = b.y; big[nt][2] = b.x; big[nt][3] = b.y;
  }
}

template <int P, bool FAST>
__device__ __forceinline__ void finish_hidden(const float (&small)[4][4], const float (&big)[4][4], const float* __restrict__ bias,
                                              int t, float (&h)[4][4]) {
  float2 r[8];
#pragma unroll
  for (int nt = 0; nt < 4; nt++) {
    const float2 b = FAST ? make_float2(0.0f, 0.0f) : *reinterpret_cast<const float2*>(bias + 8 * nt + 2 * t);
#pragma unroll
    for (int hh = 0; hh < 2; hh++) {
      const float2 bg = make_float2(big[nt][2 * hh], big[nt][2 * hh + 1]), sm = make_float2(small[nt][2 * hh], small[nt][2 * hh + 1]);
      const float2 z = (P == 3) ? __fadd2_rn(bg, sm) : __ffma2_rn(sm, make_float2(1.0f / kHalfPieceScale, 1.0f / kHalfPieceScale), bg);
      r[2 * nt + hh] = FAST ? z : __fadd2_rn(z, b);
    }
  }
#ifndef KNF_FILTER_SOFTPLUS
#define KNF_FILTER_SOFTPLUS 0  // 0: MUFU ex2 + lg2 (XU pipe), 1: the packed polynomial softplus_f2xN (FMA pipe; |err| 5e-7)
#endif
  if (FAST && KNF_FILTER_SOFTPLUS == 0) softplus_fast_f2xN<8>(r);
  else if (FAST) softplus_f2xN<8>(r);
  else softplus_tile<8>(r);
#pragma unroll
  for (int nt = 0; nt < 4; nt++) {
    h[nt][0] = r[2 * nt].x; h[nt][1] = r[2 * nt].y; h[nt][2] = r[2 * nt + 1].x; h[nt][3] = r[2 * nt + 1].y;
  }
}

// First-layer inputs of m-tile `m` of the warp's 64 points, as the lane's A-fragment values: v[i] = (row g, row g+8)
// of the lane's i-th input (k-tile major).  Lane t < 3 runs nn.fourier_encode's recurrence for axis t of its two
// rows; lane t = 3 carries the raw coordinates.  Coordinates come from S.pts.
template <int P, class SmemT>
__device__ __forceinline__ void mma_encode(const SmemT& S, int m, int lane, float2 (&v)[12]) {
  const int g = lane >> 2, t = lane & 3;
  const float pi_f = 3.14159274101257324e+00f;  // float32(np.pi)
  const int p0 = 16 * m + g;
  if (t < 3) {
    const float2 c = make_float2(S.pts[t][p0], S.pts[t][p0 + 8]);
    const float2 a = __fmul2_rn(make_float2(pi_f, pi_f), c);
    float2 s, co;
    np_sincosf2(a, s, co);
#pragma unroll
    for (int o = 0; o < kSdfFreqs; o++) {
      v[2 * o] = s;
      v[2 * o + 1] = co;
      if (o + 1 < kSdfFreqs) {
        const float2 two_s = __fmul2_rn(make_float2(2.0f, 2.0f), s);
        const float2 ns = __fmul2_rn(two_s, co);                                                       // 2 s c      (nn.py:88-92)
        const float2 ss = __fmul2_rn(two_s, s);
        co = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-ss.x, -ss.y));                           // 1 - 2 s s
        s = ns;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 12; i++) v[i] = make_float2(0.0f, 0.0f);
    v[0] = make_float2(S.pts[0][p0], S.pts[0][p0 + 8]);
    v[1] = make_float2(S.pts[1][p0], S.pts[1][p0 + 8]);
    v[2] = make_float2(S.pts[2][p0], S.pts[2][p0 + 8]);
  }
}

// Hidden activations h2 (after both softplus layers) of one m-tile from its encoded inputs, in accumulator layout:
// h2[nt][0..1] = row g, columns 8nt+2t, +1 ; h2[nt][2..3] = row g+8.
template <int P, bool FAST, class SmemT>
__device__ __forceinline__ void mma_hidden_from(const SmemT& S, const float2 (&v)[12], int lane, float (&h2)[4][4]) {
  using Blob = MmaBlobT<P>;
  const int t = lane & 3;
  float h1[4][4], small[4][4], big[4][4];
  {
    APieces<P> A[Blob::kt1];
#pragma unroll
    for (int kt = 0; kt < Blob::kt1; kt++)
      make_a<P>(A[kt], make_float2(v[4 * kt].x, v[4 * kt + 1].x), make_float2(v[4 * kt].y, v[4 * kt + 1].y),
                make_float2(v[4 * kt + 2].x, v[4 * kt + 3].x), make_float2(v[4 * kt + 2].y, v[4 * kt + 3].y));
    init_big<FAST>(big, reinterpret_cast<const float*>(S.w + Blob::b1), t);
    mma_layer<P, Blob::kt1>(A, reinterpret_cast<const uint2*>(S.w + Blob::frag1), lane, small, big);
  }
  finish_hidden<P, FAST>(small, big, reinterpret_cast<const float*>(S.w + Blob::b1), t, h1);
  // ---- second layer: the accumulator fragment is the next A fragment ------------------------------------
  {
    APieces<P> A[Blob::kt2];
#pragma unroll
    for (int kt = 0; kt < Blob::kt2; kt++)
      make_a<P>(A[kt], make_float2(h1[2 * kt][0], h1[2 * kt][1]), make_float2(h1[2 * kt][2], h1[2 * kt][3]),
                make_float2(h1[2 * kt + 1][0], h1[2 * kt + 1][1]), make_float2(h1[2 * kt + 1][2], h1[2 * kt + 1][3]));
    init_big<FAST>(big, reinterpret_cast<const float*>(S.w + Blob::b2), t);
    mma_layer<P, Blob::kt2>(A, reinterpret_cast<const uint2*>(S.w + Blob::frag2), lane, small, big);
  }
  finish_hidden<P, FAST>(small, big, reinterpret_cast<const float*>(S.w + Blob::b2), t, h2);
}

template <int P, bool FAST, class SmemT>
__device__ __forceinline__ void mma_hidden(const SmemT& S, int m, int lane, float (&h2)[4][4]) {
  float2 v[12];
  mma_encode<P, SmemT>(S, m, lane, v);
  mma_hidden_from<P, FAST, SmemT>(S, v, lane, h2);
}

// Output column j of the 32 -> N3 layer for rows g (.x) and g+8 (.y): the lane's eight hidden units first
// (fp32 FMA, fixed order), then the quad butterfly; every lane of the quad ends up with the full sum.
template <int LD = kSdfOutPad>
__device__ __forceinline__ float2 mma_output(const float (&h2)[4][4], const float* __restrict__ W3t, float bias, int t, int j) {
  float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int nt = 0; nt < 4; nt++) {
    const int k = 8 * nt + 2 * t;
    acc = __ffma2_rn(make_float2(h2[nt][0], h2[nt][2]), splat(W3t[k * LD + j]), acc);
    acc = __ffma2_rn(make_float2(h2[nt][1], h2[nt][3]), splat(W3t[(k + 1) * LD + j]), acc);
  }
  acc.x = __fadd_rn(acc.x, __shfl_xor_sync(0xffffffffu, acc.x, 1));
  acc.y = __fadd_rn(acc.y, __shfl_xor_sync(0xffffffffu, acc.y, 1));
  acc.x = __fadd_rn(acc.x, __shfl_xor_sync(0xffffffffu, acc.x, 2));
  acc.y = __fadd_rn(acc.y, __shfl_xor_sync(0xffffffffu, acc.y, 2));
  return __fadd2_rn(acc, splat(bias));
}

template <int P, int BYTES, class SmemT>
__device__ __forceinline__ void fetch_mma_weights(SmemT& S, const uint32_t* __restrict__ blobs, int cell, int lane) {
  if (lane == 0) {
    fence_proxy_async();
    mbar_expect_tx(&S.bar, BYTES);
    bulk_copy_g2s(S.w, blobs + (size_t)cell * MmaBlobT<P>::words, BYTES, &S.bar);
  }
}

#ifndef KNF_MMA_CTAS_PER_SM
#define KNF_MMA_CTAS_PER_SM 12
#endif
constexpr int kMmaCtasPerSm = KNF_MMA_CTAS_PER_SM;
#ifndef KNF_FILTER_CTAS_PER_SM
#define KNF_FILTER_CTAS_PER_SM 14
#endif
// one-warp CTAs per SM of the march kernels: P = 3 is bound by its 21 KB of shared memory, P = 2 by 16 KB
template <int P>
constexpr int march_ctas_per_sm() { return P == 2 ? KNF_FILTER_CTAS_PER_SM : 12; }

// ---- batched forward (grid.sdf_query, shading probes) ---------------------------------------------------
// Tile point p is owned by lane (g = p % 8 ... ) : point 16 t + g (+ 8): lane 4 g + t.
template <int PC>
static __global__ void __launch_bounds__(32, kMmaCtasPerSm) sdf_mma_kernel(MlpParams P) {
  using Blob = MmaBlobT<PC>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MmaSmemT<PC>& S = *reinterpret_cast<MmaSmemT<PC>*>(smem_raw);
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const int n_tiles = P.ctr->n_tiles;
  const uint32_t* blobs = reinterpret_cast<const uint32_t*>(P.blobs);
  uint32_t parity = 0;
  for (;;) {
    const int tix = next_tile(P.ctr, lane);
    if (tix >= n_tiles) break;
    const Tile tile = P.tiles[tix];
    fetch_mma_weights<PC, Blob::bytes>(S, blobs, tile.cell, lane);
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const int p = 16 * t + g + 8 * q;
      int slot = -1;
      float4 pt = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < tile.count) {
        slot = P.perm[tile.start + p];
        pt = P.req_pt[slot];
      }
      S.slot[p] = slot;
      S.pts[0][p] = pt.x;
      S.pts[1][p] = pt.y;
      S.pts[2][p] = pt.z;
    }
    __syncwarp();
    mbar_wait(&S.bar, parity);
    parity ^= 1;
    const float* W3t = reinterpret_cast<const float*>(S.w + Blob::w3);
    const float* B3 = reinterpret_cast<const float*>(S.w + Blob::b3);
    const int m_tiles = (tile.count + 15) >> 4;
    for (int m = 0; m < m_tiles; m++) {
      float h2[4][4];
      mma_hidden<PC, false, MmaSmemT<PC>>(S, m, lane, h2);
      const int s0 = S.slot[16 * m + g], s1 = S.slot[16 * m + g + 8];
      if (P.out_full == nullptr) {
        const float2 d = mma_output(h2, W3t, B3[0], t, 0);
        if (t == 0) {
          if (s0 >= 0) P.out_first[s0] = d.x;
          if (s1 >= 0) P.out_first[s1] = d.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < kSdfOut; j++) {
          const float2 o = mma_output(h2, W3t, B3[j], t, j);
          if ((j & 3) == t) {  // spread the stores over the quad
            if (s0 >= 0) P.out_full[(size_t)s0 * kSdfOut + j] = o.x;
            if (s1 >= 0) P.out_full[(size_t)s1 * kSdfOut + j] = o.y;
            if (j == 0 && P.out_first) {
              if (s0 >= 0) P.out_first[s0] = o.x;
              if (s1 >= 0) P.out_first[s1] = o.y;
            }
          }
        }
      }
    }
    __syncwarp();  // every lane is done with S.w / S.pts / S.slot before the next tile overwrites them
  }
}

}  // namespace knf
