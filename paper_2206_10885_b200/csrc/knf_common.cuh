// knf_common.cuh -- shared definitions for libknf_b200 (sm_100a only).
//
// Compile the whole library with -fmad=false: the reference's fp64 ray bookkeeping and its
// fp32 encoder recurrence are sequences of individually rounded NumPy operations, so the
// compiler must never contract a*b+c on its own.  Fused multiply-adds appear only where the
// reference itself fuses (OpenBLAS sgemm's k-ordered FMA chain, NumPy's SIMD sin/cos/exp
// polynomials) and are written explicitly with __fmaf_rn.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/knf_b200.h"

namespace knf {

// ---- compiled architecture (reference defaults, grid.py:32-68) -----------------------------
constexpr int kHidden = 32;
constexpr int kSdfFreqs = 6;
constexpr int kDirFreqs = 4;
constexpr int kFeat = 8;
constexpr int kSdfIn = 3 + 6 * kSdfFreqs;              // 39
constexpr int kSdfOut = 1 + kFeat;                      // 9
constexpr int kSdfOutPad = 12;                          // padded to a float4 multiple
constexpr int kColIn = 3 + (3 + 6 * kDirFreqs) + 3 + kFeat;  // 41
constexpr int kColOut = 3;
constexpr int kColOutPad = 4;

// Per-cell weight blob, all k-major ("transposed") so a thread reads W[k][j..j+3] as one float4:
//   W1t[K1][32] | b1[32] | W2t[32][32] | b2[32] | W3t[32][N3P] | b3[N3P]
// The first layer's K is padded to a multiple of 8 with zero rows (39 -> 40, 41 -> 48) so the k loop
// runs in fully unrolled chunks of 8; a zero row adds fma(0, 0, acc) = acc, which changes no bit.
__host__ __device__ constexpr int pad_k(int k) { return (k + 7) / 8 * 8; }

template <int K1, int N3P>
struct BlobLayout {
  static constexpr int rows1 = pad_k(K1);
  static constexpr int w1 = 0;
  static constexpr int b1 = w1 + rows1 * kHidden;
  static constexpr int w2 = b1 + kHidden;
  static constexpr int b2 = w2 + kHidden * kHidden;
  static constexpr int w3 = b2 + kHidden;
  static constexpr int b3 = w3 + kHidden * N3P;
  static constexpr int floats = b3 + N3P;
  static constexpr int bytes = floats * 4;
  static_assert(bytes % 16 == 0, "blob must be a multiple of 16 B for cp.async.bulk");
};
using SdfBlob = BlobLayout<kSdfIn, kSdfOutPad>;    // 2764 floats = 11056 B
using ColBlob = BlobLayout<kColIn, kColOutPad>;    // 2756 floats = 11024 B

// A tile is <= kTilePts requests of one cell and is processed by one warp (one-warp CTAs).
constexpr int kWarpPts = 64;
constexpr int kTilePts = kWarpPts;
#ifndef KNF_CTAS_PER_SM
#define KNF_CTAS_PER_SM 8
#endif
constexpr int kWarpCtasPerSm = KNF_CTAS_PER_SM;  // march_warp_kernel: 21.9 KB of shared memory each (192 registers: 8 is the measured optimum)
#ifndef KNF_FWD_CTAS_PER_SM
#define KNF_FWD_CTAS_PER_SM 10
#endif
constexpr int kFwdCtasPerSm = KNF_FWD_CTAS_PER_SM;  // mlp_warp_kernel (batched forward, 125 registers): 10 fit the shared memory; 16.8 M points 3.76 -> 4.19 Gq/s

// Certified skipping (decision filter) measures |p - p0| against per-cell Lipschitz bounds that hold on the cell box extended
// by a small margin (knf_bounds.cuh); a filter kernel only skips from an evaluated sample p0 that lies within kLipSlack x the
// cell extent of the cell box (samples routed from outside the grid are clamped into boundary cells and fail this test).
constexpr float kLipSlack = 1.0e-5f;

struct GridGeom {
  int resolution;
  int n_cells;
  double lo[3];
  double hi[3];
  double fd_step;
};

// One tile of work for the MLP kernels.
struct Tile {
  int cell;
  int start;  // offset into the sorted permutation
  int count;  // 1..kTilePts
  int pad;
};

// Device-resident counters of one routing pass.
struct RouteCounters {
  int n_requests;  // how many evaluation requests were emitted
  int n_tiles;
  int tile_cursor;  // dynamic tile scheduler of the MLP kernel
  int pad;
};

// ---- device math that reproduces NumPy's fp32 SIMD routines bit for bit --------------------
// Validated in the build container against numpy 2.3.5 (AVX512F/AVX2+FMA dispatch) on 4e6
// random arguments each: zero mismatches.  See DESIGN.md "Numerics".

// np.sin / np.cos on float32 (loops_trigonometric): 3-term Cody-Waite reduction by pi/2 and
// two minimax polynomials.  Valid for |x| < 71476 (beyond that NumPy calls libm).
__device__ __forceinline__ void np_sincosf(float x, float& s_out, float& c_out) {
  const float two_over_pi = 0x1.45f306p-1f;
  const float cw1 = -0x1.921fb0p+00f, cw2 = -0x1.5110b4p-22f, cw3 = -0x1.846988p-48f;
  const float magic = 0x1.8p+23f;
  float q = __fsub_rn(__fmaf_rn(x, two_over_pi, magic), magic);
  float r = __fmaf_rn(q, cw1, x);
  r = __fmaf_rn(q, cw2, r);
  r = __fmaf_rn(q, cw3, r);
  float r2 = __fmul_rn(r, r);
  float pc = __fmaf_rn(0x1.98e616p-16f, r2, -0x1.6c06dcp-10f);
  pc = __fmaf_rn(pc, r2, 0x1.55553cp-05f);
  pc = __fmaf_rn(pc, r2, -0x1.000000p-01f);
  pc = __fmaf_rn(pc, r2, 0x1.000000p+00f);
  float ps = __fmaf_rn(0x1.7d3bbcp-19f, r2, -0x1.a06bbap-13f);
  ps = __fmaf_rn(ps, r2, 0x1.11119ap-07f);
  ps = __fmaf_rn(ps, r2, -0x1.555556p-03f);
  ps = __fmul_rn(ps, r2);
  ps = __fmaf_rn(ps, r, r);
  int iq = (int)q;
  float sv = (iq & 1) ? pc : ps;
  s_out = (iq & 2) ? -sv : sv;
  int ic = iq + 1;
  float cv = (ic & 1) ? pc : ps;
  c_out = (ic & 2) ? -cv : cv;
}

// Two np_sincosf evaluations in one packed (f32x2) instruction stream: identical operations per component, so identical
// bits; used by the tensor tile kernels, where a lane encodes one axis of two rows.
__device__ __forceinline__ void np_sincosf2(float2 x, float2& s_out, float2& c_out) {
#define KNF_P2(v) make_float2(v, v)
  const float2 magic = KNF_P2(0x1.8p+23f);
  float2 q = __fadd2_rn(__ffma2_rn(x, KNF_P2(0x1.45f306p-1f), magic), KNF_P2(-0x1.8p+23f));
  float2 r = __ffma2_rn(q, KNF_P2(-0x1.921fb0p+00f), x);
  r = __ffma2_rn(q, KNF_P2(-0x1.5110b4p-22f), r);
  r = __ffma2_rn(q, KNF_P2(-0x1.846988p-48f), r);
  const float2 r2 = __fmul2_rn(r, r);
  float2 pc = __ffma2_rn(KNF_P2(0x1.98e616p-16f), r2, KNF_P2(-0x1.6c06dcp-10f));
  pc = __ffma2_rn(pc, r2, KNF_P2(0x1.55553cp-05f));
  pc = __ffma2_rn(pc, r2, KNF_P2(-0x1.000000p-01f));
  pc = __ffma2_rn(pc, r2, KNF_P2(0x1.000000p+00f));
  float2 ps = __ffma2_rn(KNF_P2(0x1.7d3bbcp-19f), r2, KNF_P2(-0x1.a06bbap-13f));
  ps = __ffma2_rn(ps, r2, KNF_P2(0x1.11119ap-07f));
  ps = __ffma2_rn(ps, r2, KNF_P2(-0x1.555556p-03f));
  ps = __fmul2_rn(ps, r2);
  ps = __ffma2_rn(ps, r, r);
#undef KNF_P2
  const int iq0 = (int)q.x, iq1 = (int)q.y;
  const float sv0 = (iq0 & 1) ? pc.x : ps.x, sv1 = (iq1 & 1) ? pc.y : ps.y;
  s_out = make_float2((iq0 & 2) ? -sv0 : sv0, (iq1 & 2) ? -sv1 : sv1);
  const int ic0 = iq0 + 1, ic1 = iq1 + 1;
  const float cv0 = (ic0 & 1) ? pc.x : ps.x, cv1 = (ic1 & 1) ? pc.y : ps.y;
  c_out = make_float2((ic0 & 2) ? -cv0 : cv0, (ic1 & 2) ? -cv1 : cv1);
}

// np.exp on float32 (loops_exponent_log): Cody-Waite by ln2, rational P5/Q2, scalef.
__device__ __forceinline__ float np_expf(float x) {
  const float magic = 0x1.8p+23f;
  float q = __fmul_rn(x, 1.442695040888963407359924681f);
  q = __fsub_rn(__fadd_rn(q, magic), magic);
  float r = __fmaf_rn(q, -6.93145752e-1f, x);
  r = __fmaf_rn(q, -1.42860677e-6f, r);
  float num = __fmaf_rn(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
  num = __fmaf_rn(num, r, 5.114512081637298353406e-02f);
  num = __fmaf_rn(num, r, 2.473615434895520810817e-01f);
  num = __fmaf_rn(num, r, 7.257664613233124478488e-01f);
  num = __fmaf_rn(num, r, 9.999999999980870924916e-01f);
  float den = __fmaf_rn(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
  den = __fmaf_rn(den, r, 1.0f);
  return ldexpf(__fdiv_rn(num, den), (int)q);
}

// nn.sigmoid (nn.py:36-38) with NumPy's exp: bit-exact given the same input.
__device__ __forceinline__ float np_sigmoidf(float x) {
  float t = np_expf(-fabsf(x));
  float den = __fadd_rn(1.0f, t);
  return x >= 0.0f ? __fdiv_rn(1.0f, den) : __fdiv_rn(t, den);
}

// nn.softplus (nn.py:26-33): log1p(exp(-|x|)) + max(x,0).  NumPy's log1p is Intel SVML and cannot be
// reproduced bit for bit, so this is a fresh evaluation of the same formula: e = exp(-|x|) by
// Cody-Waite + a degree-6 polynomial and an integer exponent add; log1p(e) = 2 atanh(e / (2 + e)) with
// s = e/(2+e) <= 1/3 (MUFU.RCP + one Newton step, odd polynomial in s).  Emulated in fp32 against
// float64 on 2e6 N(0,1.5) arguments: mean |error| 0.416 ulp, max 2.7 ulp -- NumPy's own softplus32
// measures 0.428 / 3.3 on the same inputs; the two agree bit-for-bit on 64-67 % of arguments and never
// differ by more than 4.8e-7 (tests/test_gpu_forward.py::test_device_math_against_reference_golden).
// Two evaluations share one packed (f32x2) instruction stream: every polynomial step is an
// FFMA2/FMUL2/FADD2, so a pair costs ~24 packed + ~10 scalar issue slots, one MUFU each, no
// conversions and no slow paths.
__device__ __forceinline__ float2 softplus_f2(float2 x) {
  const float2 yn = make_float2(fmaxf(-fabsf(x.x), -87.0f), fmaxf(-fabsf(x.y), -87.0f));  // -min(|x|, 87)
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  float2 tm = __ffma2_rn(yn, make_float2(1.4426950408889634f, 1.4426950408889634f), magic);
  float2 nf = __fadd2_rn(tm, make_float2(-12582912.0f, -12582912.0f));
  float2 r = __ffma2_rn(nf, make_float2(-0.693145751953125f, -0.693145751953125f), yn);
  r = __ffma2_rn(nf, make_float2(-1.42860677e-6f, -1.42860677e-6f), r);
  float2 p = __ffma2_rn(make_float2(0.0013943214435130358f, 0.0013943214435130358f), r,
                        make_float2(0.00836438313126564f, 0.00836438313126564f));
  p = __ffma2_rn(p, r, make_float2(0.04166635125875473f, 0.04166635125875473f));
  p = __ffma2_rn(p, r, make_float2(0.1666657030582428f, 0.1666657030582428f));
  p = __ffma2_rn(p, r, make_float2(0.5f, 0.5f));
  float2 q = __ffma2_rn(p, __fmul2_rn(r, r), r);
  float2 er = __fadd2_rn(make_float2(1.0f, 1.0f), q);
  float2 e = make_float2(__int_as_float(__float_as_int(er.x) + (__float_as_int(tm.x) << 23)),
                         __int_as_float(__float_as_int(er.y) + (__float_as_int(tm.y) << 23)));
  float2 nden = __ffma2_rn(e, make_float2(-1.0f, -1.0f), make_float2(-2.0f, -2.0f));  // -(2 + e), exact same rounding
  float2 rc;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.x) : "f"(-nden.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.y) : "f"(-nden.y));
  float2 s0 = __fmul2_rn(e, rc);
  float2 s = __ffma2_rn(__ffma2_rn(s0, nden, e), rc, s0);
  float2 s2 = __fmul2_rn(s, s);
  float2 g = __ffma2_rn(make_float2(0.2493898570537567f, 0.2493898570537567f), s2,
                        make_float2(0.21339640021324158f, 0.21339640021324158f));
  g = __ffma2_rn(g, s2, make_float2(0.28616610169410706f, 0.28616610169410706f));
  g = __ffma2_rn(g, s2, make_float2(0.3999920189380646f, 0.3999920189380646f));
  g = __ffma2_rn(g, s2, make_float2(0.6666666865348816f, 0.6666666865348816f));
  float2 l = __ffma2_rn(__fmul2_rn(s, s2), g, __fadd2_rn(s, s));
  return __fadd2_rn(make_float2(fmaxf(x.x, 0.0f), fmaxf(x.y, 0.0f)), l);
}

// N independent softplus_f2 evaluations advanced in lock step (same arithmetic, same bits): written stage by stage
// so that every packed instruction has N-1 independent neighbours and a lone warp can fill the FMA pipe.
template <int N>
__device__ __forceinline__ void softplus_f2xN(float2 (&x)[N]) {
#define KNF_EACH _Pragma("unroll") for (int i = 0; i < N; i++)
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  float2 yn[N], tm[N], r[N], p[N], e[N], nden[N], s[N], s2[N], g[N];
  KNF_EACH yn[i] = make_float2(fmaxf(-fabsf(x[i].x), -87.0f), fmaxf(-fabsf(x[i].y), -87.0f));
  KNF_EACH tm[i] = __ffma2_rn(yn[i], make_float2(1.4426950408889634f, 1.4426950408889634f), magic);
  KNF_EACH r[i] = __fadd2_rn(tm[i], make_float2(-12582912.0f, -12582912.0f));
  KNF_EACH { const float2 nf = r[i]; r[i] = __ffma2_rn(nf, make_float2(-0.693145751953125f, -0.693145751953125f), yn[i]);
             r[i] = __ffma2_rn(nf, make_float2(-1.42860677e-6f, -1.42860677e-6f), r[i]); }
  KNF_EACH p[i] = __ffma2_rn(make_float2(0.0013943214435130358f, 0.0013943214435130358f), r[i],
                             make_float2(0.00836438313126564f, 0.00836438313126564f));
  KNF_EACH p[i] = __ffma2_rn(p[i], r[i], make_float2(0.04166635125875473f, 0.04166635125875473f));
  KNF_EACH p[i] = __ffma2_rn(p[i], r[i], make_float2(0.1666657030582428f, 0.1666657030582428f));
  KNF_EACH p[i] = __ffma2_rn(p[i], r[i], make_float2(0.5f, 0.5f));
  KNF_EACH p[i] = __ffma2_rn(p[i], __fmul2_rn(r[i], r[i]), r[i]);
  KNF_EACH p[i] = __fadd2_rn(make_float2(1.0f, 1.0f), p[i]);
  KNF_EACH e[i] = make_float2(__int_as_float(__float_as_int(p[i].x) + (__float_as_int(tm[i].x) << 23)),
                              __int_as_float(__float_as_int(p[i].y) + (__float_as_int(tm[i].y) << 23)));
  KNF_EACH nden[i] = __ffma2_rn(e[i], make_float2(-1.0f, -1.0f), make_float2(-2.0f, -2.0f));
  KNF_EACH { float2 rc;
             asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.x) : "f"(-nden[i].x));
             asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.y) : "f"(-nden[i].y));
             const float2 s0 = __fmul2_rn(e[i], rc);
             s[i] = __ffma2_rn(__ffma2_rn(s0, nden[i], e[i]), rc, s0); }
  KNF_EACH s2[i] = __fmul2_rn(s[i], s[i]);
  KNF_EACH g[i] = __ffma2_rn(make_float2(0.2493898570537567f, 0.2493898570537567f), s2[i],
                             make_float2(0.21339640021324158f, 0.21339640021324158f));
  KNF_EACH g[i] = __ffma2_rn(g[i], s2[i], make_float2(0.28616610169410706f, 0.28616610169410706f));
  KNF_EACH g[i] = __ffma2_rn(g[i], s2[i], make_float2(0.3999920189380646f, 0.3999920189380646f));
  KNF_EACH g[i] = __ffma2_rn(g[i], s2[i], make_float2(0.6666666865348816f, 0.6666666865348816f));
  KNF_EACH { const float2 l = __ffma2_rn(__fmul2_rn(s[i], s2[i]), g[i], __fadd2_rn(s[i], s[i]));
             x[i] = __fadd2_rn(make_float2(fmaxf(x[i].x, 0.0f), fmaxf(x[i].y, 0.0f)), l); }
#undef KNF_EACH
}

// nn.softplus (nn.py:26-33) BIT FOR BIT as NumPy evaluates it on an AVX-512 host: np.exp (np_expf above: Cody-Waite,
// P5/Q2, IEEE division, scalef) followed by np.log1p, which NumPy dispatches to Intel SVML's __svml_log1pf16
// (numpy/_core/src/umath/svml, linked into _multiarray_umath): 1 + e as a two-piece sum (A, Al), reduction of A
// to [2/3, 4/3) by integer exponent arithmetic, a degree-8 polynomial in R = (mantissa - 1) + Al * 2^-N, then
// N * ln2 + poly.  The constants below are the routine's own data table (__svml_slog1p_data_internal), read from
// the installed numpy 2.3.5 binary; the operation order was restated from its main path and checked against
// np.log1p / np.exp / the composed softplus on 7e6 + 11e6 float32 arguments in the build container: 0 mismatches
// (tests/test_oracle_golden.py::test_softplus_restatement_bit_exact pins the same restatement in C).
// The IEEE division is a Markstein sequence (MUFU.RCP, one Newton step, residual correction): correctly rounded
// for the operand range here (num in [0.7, 1.42], den in [0.9, 1.1]).  |x| is clamped at 87 (e stays normal).
// N evaluations advance in lock step; every FMA-pipe step is a packed f32x2 instruction.
template <int N>
__device__ __forceinline__ void softplus_np_f2xN(float2 (&x)[N]) {
#define KNF_EACH _Pragma("unroll") for (int i = 0; i < N; i++)
#define KNF_S2(v) make_float2(v, v)
  float2 yn[N], tm[N], r[N], num[N], den[N], e[N];
  KNF_EACH yn[i] = make_float2(fmaxf(-fabsf(x[i].x), -87.0f), fmaxf(-fabsf(x[i].y), -87.0f));
  KNF_EACH tm[i] = __fadd2_rn(__fmul2_rn(yn[i], KNF_S2(1.442695040888963407359924681f)), KNF_S2(12582912.0f));
  KNF_EACH { const float2 nf = __fadd2_rn(tm[i], KNF_S2(-12582912.0f));
             r[i] = __ffma2_rn(nf, KNF_S2(-6.93145752e-1f), yn[i]);
             r[i] = __ffma2_rn(nf, KNF_S2(-1.42860677e-6f), r[i]); }
  KNF_EACH num[i] = __ffma2_rn(KNF_S2(5.082762527590693718096e-04f), r[i], KNF_S2(6.757896990527504603057e-03f));
  KNF_EACH den[i] = __ffma2_rn(KNF_S2(2.159509375685829852307e-02f), r[i], KNF_S2(-2.742335390411667452936e-01f));
  KNF_EACH num[i] = __ffma2_rn(num[i], r[i], KNF_S2(5.114512081637298353406e-02f));
  KNF_EACH den[i] = __ffma2_rn(den[i], r[i], KNF_S2(1.0f));
  KNF_EACH num[i] = __ffma2_rn(num[i], r[i], KNF_S2(2.473615434895520810817e-01f));
  KNF_EACH num[i] = __ffma2_rn(num[i], r[i], KNF_S2(7.257664613233124478488e-01f));
  KNF_EACH num[i] = __ffma2_rn(num[i], r[i], KNF_S2(9.999999999980870924916e-01f));
  KNF_EACH { float2 rc;
             asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.x) : "f"(den[i].x));
             asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc.y) : "f"(den[i].y));
             const float2 nd = make_float2(-den[i].x, -den[i].y);
             rc = __ffma2_rn(rc, __ffma2_rn(nd, rc, KNF_S2(1.0f)), rc);
             float2 q = __fmul2_rn(num[i], rc);
             q = __ffma2_rn(__ffma2_rn(nd, q, num[i]), rc, q);
             e[i] = make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(tm[i].x) << 23)),
                                __int_as_float(__float_as_int(q.y) + (__float_as_int(tm[i].y) << 23))); }
  // ---- log1p(e), e in (0, 1]: xh = 1, xl = e ---------------------------------------------------------------
  float2 A[N], Al[N], R[N], fN[N], p[N];
  KNF_EACH A[i] = __fadd2_rn(KNF_S2(1.0f), e[i]);
  KNF_EACH Al[i] = __fadd2_rn(__fadd2_rn(KNF_S2(1.0f), make_float2(-A[i].x, -A[i].y)), e[i]);
  // The routine's integer reduction (ia = bits(A) - 0x3f2aaaab; N = ia >> 23; mantissa re-biased to [2/3, 4/3)) with
  // A = 1 + e in (1, 2]: N is 1 exactly when bits(A) >= 0x3faaaaab, i.e. A >= 1.3333334f, and then the re-biased mantissa
  // is A / 2 and the scale 2^-N is 0.5 (else A and 1) -- the same values from one compare, two selects and one exact packed
  // multiplication by a power of two instead of seven integer operations per element.
  KNF_EACH {
    const float thr = __int_as_float(0x3faaaaab);
    const bool hi0 = A[i].x >= thr, hi1 = A[i].y >= thr;
    fN[i] = make_float2(hi0 ? 1.0f : 0.0f, hi1 ? 1.0f : 0.0f);
    const float2 sc = make_float2(hi0 ? 0.5f : 1.0f, hi1 ? 0.5f : 1.0f);
    const float2 r0 = __fmul2_rn(A[i], sc);
    R[i] = __fadd2_rn(__fadd2_rn(r0, KNF_S2(-1.0f)), __fmul2_rn(Al[i], sc));
  }
  KNF_EACH p[i] = __ffma2_rn(R[i], KNF_S2(0x1.1b09dap-3f), KNF_S2(-0x1.35b3c6p-3f));
  KNF_EACH p[i] = __ffma2_rn(p[i], R[i], KNF_S2(0x1.1f9624p-3f));
  KNF_EACH p[i] = __ffma2_rn(p[i], R[i], KNF_S2(-0x1.515a6ep-3f));
  KNF_EACH p[i] = __ffma2_rn(p[i], R[i], KNF_S2(0x1.99c32p-3f));
  KNF_EACH p[i] = __ffma2_rn(p[i], R[i], KNF_S2(-0x1.000b1cp-2f));
  KNF_EACH p[i] = __ffma2_rn(p[i], R[i], KNF_S2(0x1.555528p-2f));
  KNF_EACH p[i] = __ffma2_rn(p[i], R[i], KNF_S2(-0.5f));
  KNF_EACH p[i] = __ffma2_rn(__fmul2_rn(p[i], R[i]), R[i], R[i]);
  KNF_EACH { const float2 l = __ffma2_rn(fN[i], KNF_S2(0x1.62e43p-1f), p[i]);
             x[i] = __fadd2_rn(l, make_float2(fmaxf(x[i].x, 0.0f), fmaxf(x[i].y, 0.0f))); }
#undef KNF_S2
#undef KNF_EACH
}
__device__ __forceinline__ float2 softplus_np_f2(float2 x) {
  float2 a[1] = {x};
  softplus_np_f2xN<1>(a);
  return a[0];
}

// Decision-filter softplus (knf_march.cuh): MUFU.EX2 / MUFU.LG2, absolute error below kFastSoftplusErr (PTX ISA:
// ex2.approx.ftz.f32 max relative error 2^-22, lg2.approx.ftz.f32 max absolute error 2^-22 on (0.5, 2); plus four
// fp32 roundings of values <= max(1, y)).  Never reaches a result: it only feeds the filter's predicate.
constexpr float kFastSoftplusErr = 1.0e-6f;  // + 2^-22 * y, accounted for in the filter bound
template <int N>
__device__ __forceinline__ void softplus_fast_f2xN(float2 (&x)[N]) {
#pragma unroll
  for (int i = 0; i < N; i++) {
    // 2^(-|x| log2 e): one packed multiply, the -|.| rides on the MUFU operand
    const float2 u = __fmul2_rn(x[i], make_float2(1.4426950408889634f, 1.4426950408889634f));
    float2 e, l;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(-fabsf(u.x)));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(-fabsf(u.y)));
    e = __fadd2_rn(e, make_float2(1.0f, 1.0f));
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l.x) : "f"(e.x));
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l.y) : "f"(e.y));
    x[i] = __ffma2_rn(l, make_float2(0.6931471805599453f, 0.6931471805599453f), make_float2(fmaxf(x[i].x, 0.0f), fmaxf(x[i].y, 0.0f)));
  }
}

// One-MUFU variant for the tcgen05 filter (knf_tc5.cuh), where the XU pipe (ex2 + lg2 of 64 activations per evaluation) is
// the busiest pipe: e = 2^(-|x| log2 e) by MUFU.EX2 as above, ln(1 + e) on [0, 1] by a degree-5 minimax polynomial on the
// FMA pipe (packed) instead of MUFU.LG2.  Polynomial fitted in float64, evaluated here in fp32 Horner form: max |error|
// 8.8e-6 on 200 001 grid points of [0, 1] (scripts/fit_log1p.py), + 2^-22 e from ex2.approx + three fp32 roundings <= 1:
// kFastSoftplusPolyErr covers it with margin.  Like softplus_fast it only ever feeds the filter's predicate.
constexpr float kFastSoftplusPolyErr = 1.0e-5f;  // + 2^-22 * y, accounted for in the filter bound
template <int N>
__device__ __forceinline__ void softplus_fast_poly_f2xN(float2 (&x)[N]) {
#define KNF_C2(v) make_float2(v, v)
#pragma unroll
  for (int i = 0; i < N; i++) {
    const float2 u = __fmul2_rn(x[i], KNF_C2(1.4426950408889634f));
    float2 e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(-fabsf(u.x)));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(-fabsf(u.y)));
    float2 p = __ffma2_rn(KNF_C2(0.0311028603464365f), e, KNF_C2(-0.1332147866487503f));
    p = __ffma2_rn(p, e, KNF_C2(0.28669968247413635f));
    p = __ffma2_rn(p, e, KNF_C2(-0.4907394051551819f));
    p = __ffma2_rn(p, e, KNF_C2(0.9992988109588623f));
    p = __ffma2_rn(p, e, KNF_C2(8.732203241379466e-06f));
    x[i] = __fadd2_rn(p, make_float2(fmaxf(x[i].x, 0.0f), fmaxf(x[i].y, 0.0f)));
  }
#undef KNF_C2
}

// Which softplus the tile kernels run: 1 = softplus_np (NumPy bit-exact, 34 packed FMA-pipe steps per pair),
// 0 = softplus_f2 (same accuracy against float64, 24 steps, agrees with NumPy on 64 % of arguments).
#ifndef KNF_SOFTPLUS_EXACT
#define KNF_SOFTPLUS_EXACT 1
#endif
template <int N>
__device__ __forceinline__ void softplus_tile(float2 (&x)[N]) {
  if (KNF_SOFTPLUS_EXACT) softplus_np_f2xN<N>(x);
  else softplus_f2xN<N>(x);
}

// grid._cell_triples (grid.py:176-179) for one coordinate: fp64 arithmetic on the fp32 point.
__device__ __forceinline__ int cell_coord(double p, double lo, double hi, int n) {
  double t = (p - lo) / (hi - lo) * (double)n;
  double fl = floor(t);
  // np.floor(t).astype(int64) then clip: NaN / +-inf / |t| >= 2^63 convert to INT64_MIN on x86 -> 0
  if (!(fl >= 0.0)) return 0;
  if (fl >= 9.2233720368547758e18) return 0;
  if (fl >= (double)n) return n - 1;
  return (int)fl;
}

// Out-of-line copy for the march kernels, which need it only for the few samples near a cell face (three fp64
// divisions: ~300 instructions per inlined copy).
static __device__ __noinline__ int cell_of_slow(float x, float y, float z, double lo0, double lo1, double lo2, double hi0, double hi1, double hi2, int n) {
  int i = cell_coord((double)x, lo0, hi0, n);
  int j = cell_coord((double)y, lo1, hi1, n);
  int k = cell_coord((double)z, lo2, hi2, n);
  return (i * n + j) * n + k;
}

// cell_of_slow's result without its three fp64 divisions in the common case: t is estimated as (p - lo) * scale with the
// precomputed scale = n / (hi - lo).  The estimate and the reference's ((p - lo) / (hi - lo)) * n each carry <= 3 roundings
// (|difference| < 1e-12 for n <= 2^12), so unless the estimate lies within 1e-9 of an integer -- a cell face, 0 or n
// included -- both have the same floor and the same clamp; anything closer, or not finite, takes the exact path.
__device__ __forceinline__ int cell_of_quick(float x, float y, float z, const double (&lo)[3], const double (&hi)[3], const double (&scale)[3], int n) {
  const float p[3] = {x, y, z};
  int idx[3];
  bool exact = false;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const double te = ((double)p[a] - lo[a]) * scale[a];
    const double fl = floor(te);
    const double frac = te - fl;
    exact = exact || !(frac > 1e-9 && frac < 1.0 - 1e-9) || !(fabs(te) < 1e9);
    idx[a] = fl < 0.0 ? 0 : (fl >= (double)n ? n - 1 : (int)fl);
  }
  if (exact) return cell_of_slow(x, y, z, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], n);
  return (idx[0] * n + idx[1]) * n + idx[2];
}

__device__ __forceinline__ int cell_of(double x, double y, double z, const GridGeom& g) {
  int i = cell_coord(x, g.lo[0], g.hi[0], g.resolution);
  int j = cell_coord(y, g.lo[1], g.hi[1], g.resolution);
  int k = cell_coord(z, g.lo[2], g.hi[2], g.resolution);
  return (i * g.resolution + j) * g.resolution + k;
}

// ---- small PTX helpers: mbarrier + TMA 1-D bulk copy (UBLKCP) -------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// 8-byte asynchronous global -> shared copy (LDGSTS): no register staging, completion via cp_async_wait_all().
__device__ __forceinline__ void cp_async_8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Warp-aggregated append: every active lane with `want` gets a unique slot from *counter.
// Must be reached by all 32 lanes of the warp (callers keep their loops warp-uniform).
__device__ __forceinline__ int warp_append(int* counter, bool want) {
  unsigned mask = __ballot_sync(0xffffffffu, want);
  if (!want) return -1;
  int lane = threadIdx.x & 31;
  int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mask));
  base = __shfl_sync(mask, base, leader);
  return base + __popc(mask & ((1u << lane) - 1));
}

}  // namespace knf
