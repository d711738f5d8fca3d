/* oracle/np_softplus.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * C restatement of how NumPy 2.3 evaluates nn.softplus (reference nn.py:26-33,
 *     np.log1p(np.exp(-np.abs(x))) + np.maximum(x, 0)      in float32)
 * on an AVX-512 host, operation for operation:
 *   - np.exp  : numpy/_core/src/umath/loops_exponent_log.dispatch.c.src (Cody-Waite by ln2, rational P5/Q2,
 *               IEEE division, scalef) -- a NumPy source loop;
 *   - np.log1p: Intel SVML __svml_log1pf16 (numpy/_core/src/umath/svml/linux/avx512/svml_z0_log1p_s_la.s), a
 *               third-party routine linked into _multiarray_umath and absent from /root/reference; pinned here
 *               to the installed numpy 2.3.5 binary: the constants are its __svml_slog1p_data_internal table and
 *               the operation order follows its main path (1 + x as a two-piece sum, reduction to [2/3, 4/3) by
 *               integer exponent arithmetic, degree-8 polynomial, N ln2 + poly).
 * tests/test_oracle_golden.py checks it against NumPy itself on millions of arguments (0 mismatches on the
 * build host) -- this is what the device routine softplus_np_f2xN (csrc/knf_common.cuh) reproduces.
 * Valid for the arguments the path produces: exp of x <= 0, log1p of e in [0, 1].
 * Build: gcc -O2 -mfma -ffp-contract=off -shared -fPIC -o oracle/_build/libnp_softplus.so oracle/np_softplus.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

float knf_np_expf(float x) {
  const float magic = 0x1.8p+23f;
  float q = x * 1.442695040888963407359924681f;
  q = (q + magic) - magic;
  float r = fmaf(q, -6.93145752e-1f, x);
  r = fmaf(q, -1.42860677e-6f, r);
  float num = fmaf(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
  num = fmaf(num, r, 5.114512081637298353406e-02f);
  num = fmaf(num, r, 2.473615434895520810817e-01f);
  num = fmaf(num, r, 7.257664613233124478488e-01f);
  num = fmaf(num, r, 9.999999999980870924916e-01f);
  float den = fmaf(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
  den = fmaf(den, r, 1.0f);
  return ldexpf(num / den, (int)q);
}

float knf_svml_log1pf(float x) {
  const float xh = fmaxf(1.0f, x), xl = fminf(1.0f, x);
  const float A = xh + xl;
  const float Al = (xh - A) + xl;
  const int32_t iA = (int32_t)(f2u(A) - 0x3f2aaaabu);
  const int32_t N = iA >> 23;
  const float scale = u2f(0x3f800000u - ((uint32_t)N << 23));
  float R = u2f(((uint32_t)iA & 0x007fffffu) + 0x3f2aaaabu) - 1.0f;
  R = R + Al * scale;
  float p = fmaf(R, u2f(0x3e0d84edu), u2f(0xbe1ad9e3u));
  p = fmaf(p, R, u2f(0x3e0fcb12u));
  p = fmaf(p, R, u2f(0xbe28ad37u));
  p = fmaf(p, R, u2f(0x3e4ce190u));
  p = fmaf(p, R, u2f(0xbe80058eu));
  p = fmaf(p, R, u2f(0x3eaaaa94u));
  p = fmaf(p, R, u2f(0xbf000000u));
  float q = p * R;
  q = fmaf(q, R, R);
  return fmaf((float)N, u2f(0x3f317218u), q);
}

void knf_np_softplus(const float* x, float* y, long n) {
  for (long i = 0; i < n; i++) y[i] = knf_svml_log1pf(knf_np_expf(-fabsf(x[i]))) + fmaxf(x[i], 0.0f);
}
void knf_np_exp(const float* x, float* y, long n) {
  for (long i = 0; i < n; i++) y[i] = knf_np_expf(x[i]);
}
void knf_np_log1p(const float* x, float* y, long n) {
  for (long i = 0; i < n; i++) y[i] = knf_svml_log1pf(x[i]);
}
