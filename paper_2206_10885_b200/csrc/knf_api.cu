// knf_api.cu -- the extern "C" surface declared in include/knf_b200.h.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "knf_engine.h"
#include "knf_mlp.cuh"
#include "knf_grad.cuh"
#include "knf_mma.cuh"
#define KNF_TC5_LAYOUT_ONLY  // the blob layout, not the kernels (those are compiled in knf_engine.cu)
#include "knf_tc5.cuh"
#include "knf_rays.cuh"
#define KNF_BOUNDS_LAYOUT_ONLY  // the per-cell constants, not the kernels (compiled in knf_engine.cu)
#include "knf_bounds.cuh"

using namespace knf;

namespace knf {
const std::string& last_error();
}

#define KNF_TRY(expr)         \
  do {                        \
    int _rc = (expr);         \
    if (_rc != 0) return _rc; \
  } while (0)

namespace {

inline int blocks_for(size_t n, int threads = 256) {
  size_t b = (n + threads - 1) / threads;
  return (int)std::max<size_t>(1, std::min<size_t>(b, 148 * 16));
}

// Host<->device staging for KNF_MEM_HOST calls.  in(): device mirror of a host input;
// out(): device buffer whose contents are copied back by finish().
struct Stager {
  Field* F;  // may be null (field-less entry points use own buffers)
  int mem;
  cudaStream_t st;
  std::vector<DevBuf> own;
  struct Pending {
    void* host;
    void* dev;
    size_t bytes;
  };
  std::vector<Pending> outs;
  int slot = 0;
  int rc = 0;

  Stager(Field* f, int m, cudaStream_t s) : F(f), mem(m), st(s) { own.reserve(16); }
  ~Stager() {
    for (DevBuf& b : own) b.release();
  }
  void* buffer(size_t bytes) {
    if (F && slot < 12) {
      DevBuf& b = F->ws.stage[slot++];
      if (b.ensure(std::max<size_t>(bytes, 16)) != 0) {
        rc = KNF_E_NOMEM;
        return nullptr;
      }
      return b.p;
    }
    own.emplace_back();
    if (own.back().ensure(std::max<size_t>(bytes, 16)) != 0) {
      rc = KNF_E_NOMEM;
      return nullptr;
    }
    return own.back().p;
  }
  template <class T>
  const T* in(const T* p, size_t count) {
    if (mem == KNF_MEM_DEVICE || p == nullptr) return p;
    void* d = buffer(count * sizeof(T));
    if (!d) return nullptr;
    cudaError_t e = cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "H2D staging copy");
    return reinterpret_cast<const T*>(d);
  }
  template <class T>
  T* out(T* p, size_t count) {
    if (mem == KNF_MEM_DEVICE || p == nullptr) return p;
    void* d = buffer(count * sizeof(T));
    if (!d) return nullptr;
    outs.push_back({p, d, count * sizeof(T)});
    return reinterpret_cast<T*>(d);
  }
  int finish() {
    if (rc) return rc;
    if (mem == KNF_MEM_DEVICE) return 0;
    for (auto& o : outs) {
      cudaError_t e = cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_fail(e, "D2H staging copy");
    }
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return 0;
  }
};

int check_field(knf_field_t f) {
  if (!f) return fail(KNF_E_INVALID, "null field handle");
  return 0;
}

int check_settings(const KnfSettings* s) {
  if (!s) return fail(KNF_E_INVALID, "null settings");
  if (!(s->step_scale > 0.0 && s->step_scale <= 1.0)) return fail(KNF_E_INVALID, "step_scale must be in (0, 1]");
  if (s->max_steps < 0) return fail(KNF_E_INVALID, "max_steps must be >= 0");
  return 0;
}

CameraDev make_camera(const KnfCamera& c, int ss) {
  CameraDev d;
  for (int i = 0; i < 3; i++) d.pos[i] = c.position[i];
  for (int i = 0; i < 9; i++) d.rot[i] = c.rotation[i];
  d.width = c.width * ss;
  d.height = c.height * ss;
  d.scale = 2.0 * std::tan(c.fov_y / 2) / d.height;  // cameras.py:68-69
  return d;
}

// Pack one family into cell-major, k-major blobs (see knf_common.cuh BlobLayout).
template <int K1, int N3, int N3P>
void pack_family(int n_cells, const float* const w[3], const float* const b[3], std::vector<float>& out) {
  using L = BlobLayout<K1, N3P>;
  out.assign((size_t)n_cells * L::floats, 0.0f);
  for (int c = 0; c < n_cells; c++) {
    float* blob = out.data() + (size_t)c * L::floats;
    const float* w1 = w[0] + (size_t)c * kHidden * K1;  // (32, K1)
    for (int j = 0; j < kHidden; j++)
      for (int k = 0; k < K1; k++) blob[L::w1 + k * kHidden + j] = w1[j * K1 + k];
    std::memcpy(blob + L::b1, b[0] + (size_t)c * kHidden, kHidden * sizeof(float));
    const float* w2 = w[1] + (size_t)c * kHidden * kHidden;
    for (int j = 0; j < kHidden; j++)
      for (int k = 0; k < kHidden; k++) blob[L::w2 + k * kHidden + j] = w2[j * kHidden + k];
    std::memcpy(blob + L::b2, b[1] + (size_t)c * kHidden, kHidden * sizeof(float));
    const float* w3 = w[2] + (size_t)c * N3 * kHidden;  // (N3, 32)
    for (int j = 0; j < N3; j++)
      for (int k = 0; k < kHidden; k++) blob[L::w3 + k * N3P + j] = w3[j * kHidden + k];
    std::memcpy(blob + L::b3, b[2] + (size_t)c * N3, N3 * sizeof(float));
  }
}

// bf16 round-to-nearest-even of an fp32 value, returned as fp32 (the host side of knf_mma.cuh split3)
static inline float bf16_rn(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
static inline uint16_t bf16_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return (uint16_t)(u >> 16);
}
// w = p[0] + p[1] + p[2] exactly, each piece a bf16 value
static inline void split_bf16x3(float w, uint16_t p[3]) {
  const float a = bf16_rn(w), r1 = w - a, b = bf16_rn(r1), r2 = r1 - b;
  p[0] = bf16_bits(a);
  p[1] = bf16_bits(b);
  p[2] = bf16_bits(r2);
}

// fp16 pieces of the P = 2 split: w ~= h[0] + h[1] / 2^11 (to 2^-24 relative), both fp16 bit patterns
static inline void split_fp16x2(float w, uint16_t p[2]) {
  const __half a = __float2half_rn(w);
  const float r = (w - __half2float(a)) * kHalfPieceScale;
  const __half b = __float2half_rn(r);
  std::memcpy(&p[0], &a, 2);
  std::memcpy(&p[1], &b, 2);
}

// Pack the SDF family into knf_mma.cuh MmaBlobT<P>: mma.sync.m16n8k16 B fragments of W1 (permuted K) and W2
// as P pieces each (bf16 x 3 or fp16 x 2), then fp32 biases and the k-major output layer.
// Proven bound on |distance from the tensor-core tile kernel with the fast softplus - distance from the exact
// fp32 chain kernel| for one cell, by forward error analysis over the cell's weights (all sums of magnitudes):
//   * operand representation: P = 3 pieces are exact; P = 2 leaves |x~ - x| <= 2^-22 |x| per operand and drops
//     x2 w2 <= 2^-22 |x||w|                                             -> e_rep = 3.1 * 2^-22 (0 for P = 3);
//   * HMMA accumulation: every mma.sync adds <= 17 addends aligned to the largest exponent, each truncated below
//     2^-24 of it; <= 9 instructions per output (3 k-tiles x 3 products), then two fp32 roundings
//                                                                          -> e_acc = 155 * 2^-24 of sum |x||w|
//     (worst case measured on B200 over 1.7e7 outputs of 16-24 HMMAs each: 2^-22.5, scripts/micro/hmma_split.cu);
//   * the exact kernel's own distance to real arithmetic: fp32 FMA chains of <= 48 terms, gamma_48 < 2^-18;
//   * softplus is 1-Lipschitz; the fast softplus adds kFastSoftplusErr + 2^-22 y, NumPy's adds <= 2^-22 y.
// Inputs are bounded by 1 (sin / cos) and by the box (raw coordinates).
constexpr double kFp16Safe = 60000.0;  // below the largest finite fp16 (65504) with room for the rounding of a piece
static double filter_delta(int pieces, const float* w1, const float* b1, const float* w2, const float* b2, const float* w3,
                           const float* b3, double x_raw, bool bias1_in_mma = false, double softplus_abs_err = (double)kFastSoftplusErr) {
  const double e_rep = pieces == 2 ? 3.1 * std::ldexp(1.0, -22) : 0.0;
  const double e = e_rep + 155.0 * std::ldexp(1.0, -24) + std::ldexp(1.0, -18);
  const double sp_rel = 2.0 * std::ldexp(1.0, -22), sp_abs = softplus_abs_err;
  auto softplus = [](double z) { return std::log1p(std::exp(-std::fabs(z))) + std::max(z, 0.0); };
  double eh1[kHidden], H1[kHidden], eh2[kHidden], H2[kHidden];
  for (int n = 0; n < kHidden; n++) {
    double s = 0.0;
    for (int k = 0; k < kSdfIn; k++) s += std::fabs((double)w1[n * kSdfIn + k]) * (k < 3 ? x_raw : 1.0);
    // knf_tc5.cuh feeds b1 through the tensor core as the weight of a constant-1 feature: one more product term
    const double s_mma = s + (bias1_in_mma ? std::fabs((double)b1[n]) : 0.0);
    H1[n] = softplus(std::fabs((double)b1[n]) + s);
    eh1[n] = e * s_mma + std::ldexp(1.0, -22) * (std::fabs((double)b1[n]) + s) + sp_abs + sp_rel * H1[n];
  }
  for (int n = 0; n < kHidden; n++) {
    double s = 0.0, err = 0.0;
    for (int k = 0; k < kHidden; k++) {
      const double a = std::fabs((double)w2[n * kHidden + k]);
      s += a * H1[k];
      err += a * (eh1[k] + e * (H1[k] + eh1[k]));
    }
    H2[n] = softplus(std::fabs((double)b2[n]) + s);
    eh2[n] = err + std::ldexp(1.0, -22) * (std::fabs((double)b2[n]) + s) + sp_abs + sp_rel * H2[n];
  }
  double err = 0.0, s = std::fabs((double)b3[0]);
  for (int k = 0; k < kHidden; k++) {
    const double a = std::fabs((double)w3[k]);  // output 0 = the distance
    s += a * H2[k];
    err += a * eh2[k];
  }
  // fp16 operand pieces: a hidden activation (bounded by H1 / H2) or a first-layer input beyond the fp16 range turns
  // into inf inside the tensor-core evaluation and the analysis above says nothing: no bound for this cell.
  double h_max = x_raw;
  for (int n = 0; n < kHidden; n++) h_max = std::max(h_max, std::max(H1[n], H2[n]));
  if (pieces == 2 && !(h_max < kFp16Safe)) return INFINITY;
  const double delta = 1.05 * (err + std::ldexp(1.0, -17) * s) + 1e-6;
  return std::isfinite(delta) ? delta : INFINITY;
}

// Proven Lipschitz bound of one cell's distance network d(x) = w3 . softplus(W2 softplus(W1 enc(x) + b1) + b2) + b3:
// softplus' <= 1, so L <= |w3|_2 * |W2|_2 * sup_x |W1 J_enc(x)|_2.  |W2|_2 is bounded by Gershgorin on (W2^T W2)^16
// (within 2 % of the true spectral norm).  J_enc is block diagonal per axis a: d/dx_a of (x_a, sin(2^o pi x_a),
// cos(2^o pi x_a))_o = (1, 2^o pi cos, -2^o pi sin)_o; (cos, -sin) is a unit vector, so the axis-a column of W1 J
// has norm <= |w_raw_a| + sum_o 2^o pi sigma_max([w_sin_o,a | w_cos_o,a]).
// Returns the three per-axis bounds L_a = |w3| |W2| |column a of W1 J|: |d(p) - d(q)| <= sum_a L_a |p_a - q_a| (triangle
// inequality over the axes -- tighter than one constant times the Euclidean distance for rays near an axis).
static void lipschitz_bound(const float* w1, const float* w2, const float* w3, double out[3], LipCellConst* cc = nullptr) {
  double n3 = 0.0;
  for (int k = 0; k < kHidden; k++) n3 += (double)w3[k] * (double)w3[k];
  n3 = std::sqrt(n3);
  std::vector<double> G(kHidden * kHidden), T(kHidden * kHidden);
  for (int i = 0; i < kHidden; i++)
    for (int j = 0; j < kHidden; j++) {
      double a = 0.0;
      for (int n = 0; n < kHidden; n++) a += (double)w2[n * kHidden + i] * (double)w2[n * kHidden + j];
      G[i * kHidden + j] = a;
    }
  double log_scale = 0.0;  // G is rescaled between squarings so large weights cannot overflow
  for (int sq = 0; sq < 4; sq++) {
    double mx = 0.0;
    for (double v : G) mx = std::max(mx, std::fabs(v));
    if (mx > 0.0) {
      for (double& v : G) v /= mx;
      log_scale = 2.0 * (log_scale + std::log(mx));
    } else {
      log_scale *= 2.0;
    }
    for (int i = 0; i < kHidden; i++)
      for (int j = 0; j < kHidden; j++) {
        double a = 0.0;
        for (int n = 0; n < kHidden; n++) a += G[i * kHidden + n] * G[n * kHidden + j];
        T[i * kHidden + j] = a;
      }
    G.swap(T);
  }
  double row = 0.0;
  for (int i = 0; i < kHidden; i++) {
    double a = 0.0;
    for (int j = 0; j < kHidden; j++) a += std::fabs(G[i * kHidden + j]);
    row = std::max(row, a);
  }
  // lambda_max(W2^T W2)^16 <= row * exp(log_scale)  =>  |W2|_2 <= (row * exp(log_scale))^(1/32)
  const double n2 = row > 0.0 ? std::exp((std::log(row) + log_scale) / 32.0) : 0.0;
  for (int a = 0; a < 3; a++) {
    double m = 0.0;
    for (int n = 0; n < kHidden; n++) m += (double)w1[n * kSdfIn + a] * (double)w1[n * kSdfIn + a];
    m = std::sqrt(m);
    for (int o = 0; o < kSdfFreqs; o++) {
      double aa = 0.0, bb = 0.0, ab = 0.0;
      for (int n = 0; n < kHidden; n++) {
        const double s = w1[n * kSdfIn + 3 + 6 * o + a], c = w1[n * kSdfIn + 3 + 6 * o + 3 + a];
        aa += s * s;
        bb += c * c;
        ab += s * c;
      }
      const double lam = 0.5 * (aa + bb) + std::sqrt(0.25 * (aa - bb) * (aa - bb) + ab * ab);
      m += std::ldexp(3.14159265358979323846, o) * std::sqrt(lam);
    }
    out[a] = 1.001 * n3 * n2 * m + 1e-12;
  }
  if (cc) {  // constants of the sub-box refinement (knf_bounds.cuh), rounded up
    cc->n3 = n3 * (1.0 + 1e-12);
    cc->n2 = n2 * 1.0001;
    double fro = 0.0;
    for (int i = 0; i < kHidden * kHidden; i++) fro += (double)w2[i] * (double)w2[i];
    cc->n2f = std::sqrt(fro) * (1.0 + 1e-12);
    for (int a = 0; a < 3; a++) {
      double k3 = 0.0;
      for (int o = 0; o < kSdfFreqs; o++) {
        double aa = 0.0, bb = 0.0, ab = 0.0;
        for (int n = 0; n < kHidden; n++) {
          const double sn = w1[n * kSdfIn + 3 + 6 * o + a], cs = w1[n * kSdfIn + 3 + 6 * o + 3 + a];
          aa += sn * sn;
          bb += cs * cs;
          ab += sn * cs;
        }
        const double lam = 0.5 * (aa + bb) + std::sqrt(0.25 * (aa - bb) * (aa - bb) + ab * ab);
        const double f = std::ldexp(3.14159265358979323846, o);
        k3 += f * f * f * std::sqrt(lam);
      }
      cc->k3[a] = k3 * (1.0 + 1e-9);
    }
  }
}

// Certified skipping compares the exact kernel's distances at two points of a cell through a Lipschitz bound of the
// REAL-arithmetic network on the TRUE Fourier features, so the error of the fp32 features themselves (NumPy's float32 sin / cos
// of fl(pi_f x) at octave 0, then the rounded double-angle recurrence, which roughly doubles the error per octave) enters at
// both points.  scripts/feature_error.py measures max |fp32 feature - true feature| per octave EXHAUSTIVELY over all
// 2 130 723 212 float32 inputs with |x| <= 1.001 (profiles/feature_error_r2b.json: 3.5, 9.9, 19.8, 45.4, 108.4, 273.0 units of
// 2^-24); the constants below are those maxima x 1.25.  The dominant part is the angle error, proportional to |x|, so a larger
// box scales them by x_raw / 1.001 (an extrapolation, not a measurement).  Through the layers (softplus' <= 1):
//   |F(phi~) - F(phi)| <= |w3| |W2| sum_k |W1[:, k]|_2 |phi~_k - phi_k|   =: E_phi,
// and 2 E_phi is added to the cell's filter bound delta, which is what both the filter's decision and the skip budget use.
constexpr double kFeatureErrU[kSdfFreqs] = {4.5, 12.5, 25.0, 57.0, 136.0, 342.0};
static double feature_error_allowance(const float* w1, double n3, double n2, double x_raw) {
  const double unit = std::max(1.0, x_raw / 1.001) * std::ldexp(1.0, -24);
  double s = 0.0;
  for (int o = 0; o < kSdfFreqs; o++)
    for (int c = 0; c < 6; c++) {  // the octave's three sin and three cos columns
      double nn = 0.0;
      for (int n = 0; n < kHidden; n++) nn += (double)w1[n * kSdfIn + 3 + 6 * o + c] * (double)w1[n * kSdfIn + 3 + 6 * o + c];
      s += std::sqrt(nn) * kFeatureErrU[o] * unit;
    }
  return n3 * n2 * s * 1.0001;
}

template <int P>
void pack_sdf_mma(int n_cells, const float* const w[3], const float* const b[3], double x_raw, std::vector<uint32_t>& out,
                  double* delta_max, int* cells_off = nullptr) {
  using Blob = MmaBlobT<P>;
  out.assign((size_t)n_cells * Blob::words, 0u);
  for (int c = 0; c < n_cells; c++) {
    uint32_t* blob = out.data() + (size_t)c * Blob::words;
    const float* w1 = w[0] + (size_t)c * kHidden * kSdfIn;   // (32, 39)
    const float* w2 = w[1] + (size_t)c * kHidden * kHidden;  // (32, 32)
    const float* w3 = w[2] + (size_t)c * kSdfOut * kHidden;  // (9, 32)
    for (int layer = 0; layer < 2; layer++) {
      const int kts = layer == 0 ? Blob::kt1 : Blob::kt2;
      uint32_t* frag = blob + (layer == 0 ? Blob::frag1 : Blob::frag2);
      for (int kt = 0; kt < kts; kt++)
        for (int nt = 0; nt < 4; nt++)
          for (int lane = 0; lane < 32; lane++) {
            const int g = lane >> 2, t = lane & 3, n = 8 * nt + g;
            for (int h = 0; h < 2; h++) {
              uint16_t lo[3], hi[3];
              float wv[2];
              for (int e = 0; e < 2; e++) {
                const int kslot = 2 * t + 8 * h + e;
                if (layer == 0) {
                  const int feat = mma_feature_of(kt, kslot);
                  wv[e] = feat >= 0 ? w1[n * kSdfIn + feat] : 0.0f;
                } else {
                  wv[e] = w2[n * kHidden + 16 * kt + kslot];
                }
              }
              if (P == 3) {
                split_bf16x3(wv[0], lo);
                split_bf16x3(wv[1], hi);
              } else {
                split_fp16x2(wv[0], lo);
                split_fp16x2(wv[1], hi);
              }
              for (int piece = 0; piece < P; piece++)
                frag[((((kt * 4 + nt) * 32) + lane) * P + piece) * 2 + h] = (uint32_t)lo[piece] | ((uint32_t)hi[piece] << 16);
            }
          }
    }
    std::memcpy(blob + Blob::b1, b[0] + (size_t)c * kHidden, kHidden * sizeof(float));
    std::memcpy(blob + Blob::b2, b[1] + (size_t)c * kHidden, kHidden * sizeof(float));
    float* w3t = reinterpret_cast<float*>(blob + Blob::w3);
    for (int j = 0; j < kSdfOut; j++)
      for (int k = 0; k < kHidden; k++) w3t[k * kSdfOutPad + j] = w3[j * kHidden + k];
    std::memcpy(blob + Blob::w3d, w3, kHidden * sizeof(float));  // row 0 of (9, 32): the distance output
    std::memcpy(blob + Blob::b3, b[2] + (size_t)c * kSdfOut, kSdfOut * sizeof(float));
    double lip[3];
    LipCellConst lcc{};
    lipschitz_bound(w1, w2, w3, lip, &lcc);
    const double delta = filter_delta(P, w1, b[0] + (size_t)c * kHidden, w2, b[1] + (size_t)c * kHidden, w3, b[2] + (size_t)c * kSdfOut, x_raw) +
                         2.0 * feature_error_allowance(w1, lcc.n3, lcc.n2, x_raw);
    // delta = +inf switches the filter off for this cell: -(eps + inf) = -inf, no distance is ever below it
    const float delta_f = delta < 1e30 ? std::nextafter((float)delta, INFINITY) : INFINITY;
    std::memcpy(blob + Blob::b3 + kFilterDeltaSlot, &delta_f, sizeof(float));
    if (delta_max && std::isfinite(delta_f)) *delta_max = std::max(*delta_max, (double)delta_f);
    if (cells_off && !std::isfinite(delta_f)) *cells_off += 1;
    for (int a = 0; a < 3; a++) {
      const float lip_f = std::nextafter((float)lip[a], INFINITY);
      std::memcpy(blob + Blob::b3 + kFilterLipSlot + a, &lip_f, sizeof(float));
    }
  }
}

// Pack the SDF family into knf_tc5.cuh Tc5Blob: fp16 x 2 weight pieces as K-major no-swizzle tcgen05 B operands (8-row x
// 16-byte core matrices: [K chunk][row][8 fp16]), rows 0..31 first pieces, rows 32..63 second pieces (x 2^11); layer 1 carries
// its bias as the weight of the constant-1 feature k = 39.  Then the fp32 constants, the filter bound delta and the Lipschitz
// bounds (same analysis as pack_sdf_mma<2>: same operand pieces, same number of tensor-core accumulation steps per output).
void pack_sdf_tc5(int n_cells, const float* const w[3], const float* const b[3], double x_raw, std::vector<uint8_t>& out,
                  double* delta_max, int* cells_off, std::vector<LipCellConst>* lip_consts = nullptr, std::vector<float>* lip_out = nullptr) {
  if (lip_consts) lip_consts->assign((size_t)n_cells, LipCellConst{});
  if (lip_out) lip_out->assign((size_t)n_cells * 3, 0.0f);
  out.assign((size_t)n_cells * Tc5Blob::bytes, 0);
  for (int c = 0; c < n_cells; c++) {
    uint8_t* blob = out.data() + (size_t)c * Tc5Blob::bytes;
    const float* w1 = w[0] + (size_t)c * kHidden * kSdfIn;
    const float* w2 = w[1] + (size_t)c * kHidden * kHidden;
    const float* w3 = w[2] + (size_t)c * kSdfOut * kHidden;
    const float* b1 = b[0] + (size_t)c * kHidden;
    const float* b2 = b[1] + (size_t)c * kHidden;
    const float* b3 = b[2] + (size_t)c * kSdfOut;
    uint16_t* B1 = reinterpret_cast<uint16_t*>(blob + Tc5Blob::off_b1);
    uint16_t* B2 = reinterpret_cast<uint16_t*>(blob + Tc5Blob::off_b2);
    for (int n = 0; n < kHidden; n++) {
      for (int k = 0; k < kTc5K1; k++) {
        const float v = k < kSdfIn ? w1[n * kSdfIn + k] : (k == kTc5BiasK ? b1[n] : 0.0f);
        uint16_t p[2];
        split_fp16x2(v, p);
        B1[((k / 8) * 64 + n) * 8 + (k % 8)] = p[0];
        B1[((k / 8) * 64 + 32 + n) * 8 + (k % 8)] = p[1];
      }
      for (int k = 0; k < kHidden; k++) {
        uint16_t p[2];
        split_fp16x2(w2[n * kHidden + k], p);
        B2[((k / 8) * 64 + n) * 8 + (k % 8)] = p[0];
        B2[((k / 8) * 64 + 32 + n) * 8 + (k % 8)] = p[1];
      }
    }
    float* f = reinterpret_cast<float*>(blob + Tc5Blob::off_f32);
    std::memcpy(f + Tc5Blob::f_b2, b2, kHidden * sizeof(float));
    std::memcpy(f + Tc5Blob::f_w3d, w3, kHidden * sizeof(float));
    std::memcpy(f + Tc5Blob::f_b3, b3, kSdfOut * sizeof(float));
    for (int j = 0; j < kSdfOut; j++)
      for (int k = 0; k < kHidden; k++) f[Tc5Blob::f_w3t + k * kSdfOutPad + j] = w3[j * kHidden + k];
    double lip[3];
    LipCellConst lcc{};
    lipschitz_bound(w1, w2, w3, lip, &lcc);
    if (lip_consts) (*lip_consts)[c] = lcc;
    const double delta = filter_delta(2, w1, b1, w2, b2, w3, b3, x_raw, true, (double)kTc5SoftplusErr) + 2.0 * feature_error_allowance(w1, lcc.n3, lcc.n2, x_raw);
    const float delta_f = delta < 1e30 ? std::nextafter((float)delta, INFINITY) : INFINITY;
    f[Tc5Blob::f_delta] = delta_f;
    if (delta_max && std::isfinite(delta_f)) *delta_max = std::max(*delta_max, (double)delta_f);
    if (cells_off && !std::isfinite(delta_f)) *cells_off += 1;
    for (int a = 0; a < 3; a++) {
      f[Tc5Blob::f_lip + a] = std::nextafter((float)lip[a], INFINITY);
      if (lip_out) (*lip_out)[(size_t)c * 3 + a] = f[Tc5Blob::f_lip + a];
    }
  }
}

int validate_desc(const KnfFieldDesc* d) {
  if (!d) return fail(KNF_E_INVALID, "null field description");
  if (d->resolution < 1) return fail(KNF_E_INVALID, "resolution must be >= 1");
  if ((int64_t)d->resolution * d->resolution * d->resolution > (1 << 24))
    return fail(KNF_E_UNSUPPORTED, "resolution^3 exceeds 2^24 cells");
  for (int a = 0; a < 3; a++)
    if (!(d->bbox_min[a] < d->bbox_max[a])) return fail(KNF_E_INVALID, "bbox_min must be < bbox_max componentwise");
  if (!(d->fd_step > 0)) return fail(KNF_E_INVALID, "fd_step must be > 0");
  if (d->sdf_freqs != kSdfFreqs || d->dir_freqs != kDirFreqs || d->feature_dim != kFeat)
    return fail(KNF_E_UNSUPPORTED,
                "kernels are compiled for the reference widths only: sdf_freqs=6, dir_freqs=4, feature_dim=8 "
                "(39-32-32-9 / 41-32-32-3)");
  for (int k = 0; k < 3; k++)
    if (!d->sdf_w[k] || !d->sdf_b[k] || !d->color_w[k] || !d->color_b[k])
      return fail(KNF_E_INVALID, "null weight/bias stack");
  return 0;
}

int create_from_stacks(const KnfFieldDesc* d, int device, knf_field_t* out) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(KNF_E_CUDA, "no CUDA device available: libknf_b200 has no CPU fallback");
  }
  if (device < 0 || device >= ndev) return fail(KNF_E_INVALID, "device index out of range");
  KNF_CUDA(cudaSetDevice(device));
  std::unique_ptr<knf_field_s> h(new knf_field_s());
  Field& F = h->f;
  F.device = device;
  F.geom.resolution = d->resolution;
  F.geom.n_cells = d->resolution * d->resolution * d->resolution;
  for (int a = 0; a < 3; a++) {
    F.geom.lo[a] = d->bbox_min[a];
    F.geom.hi[a] = d->bbox_max[a];
  }
  F.geom.fd_step = d->fd_step;
  if (const char* env = std::getenv("KNF_MARCH_MAX_INNER")) F.march_max_inner = F.filter_max_inner = std::max(1, std::atoi(env));  // tuning knob
  std::vector<float> packed;
  pack_family<kSdfIn, kSdfOut, kSdfOutPad>(F.geom.n_cells, d->sdf_w, d->sdf_b, packed);
  KNF_CUDA(cudaMalloc(&F.sdf_blobs, packed.size() * sizeof(float)));
  KNF_CUDA(cudaMemcpy(F.sdf_blobs, packed.data(), packed.size() * sizeof(float), cudaMemcpyHostToDevice));
  pack_family<kColIn, kColOut, kColOutPad>(F.geom.n_cells, d->color_w, d->color_b, packed);
  KNF_CUDA(cudaMalloc(&F.col_blobs, packed.size() * sizeof(float)));
  KNF_CUDA(cudaMemcpy(F.col_blobs, packed.data(), packed.size() * sizeof(float), cudaMemcpyHostToDevice));
  {
    std::vector<uint32_t> frags;
    double x_raw = 0.0;
    for (int a = 0; a < 3; a++) x_raw = std::max(x_raw, std::max(std::fabs(d->bbox_min[a]), std::fabs(d->bbox_max[a])));
    x_raw *= 1.001;
    pack_sdf_mma<3>(F.geom.n_cells, d->sdf_w, d->sdf_b, x_raw, frags, nullptr);
    KNF_CUDA(cudaMalloc(&F.sdf_mma_blobs, frags.size() * sizeof(uint32_t)));
    KNF_CUDA(cudaMemcpy(F.sdf_mma_blobs, frags.data(), frags.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    // fp16 pieces need |w| < 65504 in the two hidden layers (true of any trained or random-init field)
    F.fp16_ok = true;
    const size_t n1 = (size_t)F.geom.n_cells * kHidden * kSdfIn, n2 = (size_t)F.geom.n_cells * kHidden * kHidden;
    for (size_t i = 0; i < n1 && F.fp16_ok; i++) F.fp16_ok = std::fabs(d->sdf_w[0][i]) < 60000.0f;
    for (size_t i = 0; i < n2 && F.fp16_ok; i++) F.fp16_ok = std::fabs(d->sdf_w[1][i]) < 60000.0f;
    if (F.fp16_ok) {
      F.filter_delta_max = 0.0;
      F.filter_x_raw = (float)x_raw;
      F.filter_cells_off = 0;
      pack_sdf_mma<2>(F.geom.n_cells, d->sdf_w, d->sdf_b, x_raw, frags, &F.filter_delta_max, &F.filter_cells_off);
      if (F.filter_cells_off == F.geom.n_cells) F.fp16_ok = false;  // nothing left for the filter to decide
    }
    if (F.fp16_ok) {
      KNF_CUDA(cudaMalloc(&F.sdf_mmah_blobs, frags.size() * sizeof(uint32_t)));
      KNF_CUDA(cudaMemcpy(F.sdf_mmah_blobs, frags.data(), frags.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
      std::vector<uint8_t> tc5;
      double dmax = 0.0;
      int off = 0;
      std::vector<LipCellConst> lipc;
      pack_sdf_tc5(F.geom.n_cells, d->sdf_w, d->sdf_b, x_raw, tc5, &dmax, &off, &lipc, &F.lip_closed_form);
      KNF_CUDA(cudaMalloc(&F.lip_consts, lipc.size() * sizeof(LipCellConst)));
      KNF_CUDA(cudaMemcpy(F.lip_consts, lipc.data(), lipc.size() * sizeof(LipCellConst), cudaMemcpyHostToDevice));
      KNF_CUDA(cudaMalloc(&F.lip_cur, F.lip_closed_form.size() * sizeof(float)));
      KNF_CUDA(cudaMemcpy(F.lip_cur, F.lip_closed_form.data(), F.lip_closed_form.size() * sizeof(float), cudaMemcpyHostToDevice));
      KNF_CUDA(cudaMalloc(&F.lip_max, F.lip_closed_form.size() * sizeof(unsigned long long)));
      F.filter_delta_max = std::max(F.filter_delta_max, dmax);  // crawl_below must cover whichever filter kernel runs
      KNF_CUDA(cudaMalloc(&F.sdf_tc5_blobs, tc5.size()));
      KNF_CUDA(cudaMemcpy(F.sdf_tc5_blobs, tc5.data(), tc5.size(), cudaMemcpyHostToDevice));
    }
  }
  F.precision = KNF_PRECISION_DEFAULT;
  if (const char* env = std::getenv("KNF_PRECISION")) {
    const std::string v(env);
    if (v == "fp32_chain" || v == "0") F.precision = KNF_PRECISION_FP32_CHAIN;
    else if (v == "tensor_bf16x3" || v == "1") F.precision = KNF_PRECISION_TENSOR_BF16X3;
    else if (v == "tensor_fp16x2" || v == "2") F.precision = KNF_PRECISION_TENSOR_FP16X2;
    else return fail(KNF_E_INVALID, "KNF_PRECISION must be fp32_chain, tensor_bf16x3 or tensor_fp16x2");
  }
  if (F.precision == KNF_PRECISION_TENSOR_FP16X2 && (!F.fp16_ok || F.filter_cells_off > 0)) F.precision = KNF_PRECISION_TENSOR_BF16X3;  // bf16 pieces keep fp32's range
  if (const char* env = std::getenv("KNF_LIP_WIDTH")) F.lip_width = std::max(0.0, std::atof(env));
  if (const char* env = std::getenv("KNF_LIP_FINE")) F.lip_fine = std::max(1, std::min(kLipMaxFine, std::atoi(env)));
  if (const char* env = std::getenv("KNF_FILTER_SKIP")) F.filter_skip = std::max(0, std::min(2, std::atoi(env)));
  if (const char* env = std::getenv("KNF_SPARSE_SMALL")) F.sparse_small_kernel = std::atoi(env) != 0;
  if (const char* env = std::getenv("KNF_FILTER_KEEP")) F.filter_keep_div = std::max(1, std::atoi(env));
  if (const char* env = std::getenv("KNF_FILTER_INNER")) F.filter_max_inner = std::max(1, std::atoi(env));
  if (const char* env = std::getenv("KNF_SPARSE_DIV")) F.sparse_div = std::max(1, std::atoi(env));
  if (const char* env = std::getenv("KNF_SPARSE_INNER")) F.sparse_max_inner = std::max(1, std::atoi(env));
  if (const char* env = std::getenv("KNF_SPARSE_KEEP")) F.sparse_keep_div = std::max(1, std::atoi(env));
  if (const char* env = std::getenv("KNF_EXACT_MID")) F.exact_mid = std::atoi(env) != 0;
  if (const char* env = std::getenv("KNF_SCAN_SPLIT")) F.scan_split = std::max(64, std::atoi(env));
  if (const char* env = std::getenv("KNF_FILTER_GRID")) F.filter_grid_ctas = std::max(1, std::atoi(env));
  if (const char* env = std::getenv("KNF_FILTER_SKIP_CAP")) F.filter_skip_cap = std::max(0, std::atoi(env));
  if (const char* env = std::getenv("KNF_OVERLAP")) F.overlap_queues = std::atoi(env) != 0;
  if (const char* env = std::getenv("KNF_EXACT_GRID")) F.exact_grid_ctas = std::max(0, std::atoi(env));
  if (const char* env = std::getenv("KNF_EXACT_FIRST")) F.exact_first = std::atoi(env) != 0;
  if (const char* env = std::getenv("KNF_FIRST_SPLIT")) F.first_split_eighths = std::max(0, std::min(8, std::atoi(env)));
  if (const char* env = std::getenv("KNF_FILTER_FIRST")) F.filter_first = std::atoi(env) != 0;
  if (const char* env = std::getenv("KNF_TAIL_SKIP")) F.tail_skip = std::atoi(env) != 0;
  if (const char* env = std::getenv("KNF_TAIL")) F.tail_threshold = std::max(0, std::atoi(env));
  if (const char* env = std::getenv("KNF_FILTER_KERNEL")) {
    const std::string v(env);
    if (v == "tc5" || v == "1") F.filter_kernel = 1;
    else if (v == "mma" || v == "0") F.filter_kernel = 0;
    else return fail(KNF_E_INVALID, "KNF_FILTER_KERNEL must be tc5 or mma");
  }
  if (const char* env = std::getenv("KNF_FILTER")) {
    const std::string v(env);
    if (v == "off" || v == "0") F.filter_mode = KNF_FILTER_OFF;
    else if (v == "on" || v == "1") F.filter_mode = KNF_FILTER_ON;
    else if (v == "auto" || v == "2") F.filter_mode = KNF_FILTER_AUTO;
    else return fail(KNF_E_INVALID, "KNF_FILTER must be off, on or auto");
  }
  *out = h.release();
  return 0;
}

// zlib-compatible CRC32 (modelio.py:124, 153)
uint32_t crc32_bytes(const unsigned char* p, size_t n) {
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; i++) {
      uint32_t c = i;
      for (int k = 0; k < 8; k++) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
      table[i] = c;
    }
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; i++) c = table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

__global__ void fourier_encode_kernel(const float* __restrict__ x, long long n, int L, float* __restrict__ out) {
  const float pi_f = 3.14159274101257324e+00f;
  const int width = 3 + 6 * L;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    float* row = out + i * width;
    float s[3], c[3];
    for (int a = 0; a < 3; a++) {
      float v = x[3 * i + a];
      row[a] = v;
      if (L > 0) np_sincosf(__fmul_rn(pi_f, v), s[a], c[a]);
    }
    for (int o = 0; o < L; o++)
      for (int a = 0; a < 3; a++) {
        row[3 + 6 * o + a] = s[a];
        row[3 + 6 * o + 3 + a] = c[a];
        float two_s = __fmul_rn(2.0f, s[a]);
        float ns = __fmul_rn(two_s, c[a]);
        float nc = __fsub_rn(1.0f, __fmul_rn(two_s, s[a]));
        s[a] = ns;
        c[a] = nc;
      }
  }
}
__global__ void activation_kernel(const float* __restrict__ x, long long n, int which, float* __restrict__ out) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = which == 0 ? (KNF_SOFTPLUS_EXACT ? softplus_np_f2(make_float2(x[i], x[i])).x : softplus_f2(make_float2(x[i], x[i])).x) : np_sigmoidf(x[i]);
}

__global__ void pass_u8_kernel(int pass, long long n, const float* __restrict__ color, const float* __restrict__ depth,
                               const float* __restrict__ normal, const unsigned char* __restrict__ hit,
                               unsigned char* __restrict__ out) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double v[3];
    if (pass == KNF_PASS_COLOR) {
      for (int a = 0; a < 3; a++) v[a] = (double)color[3 * i + a];
    } else if (pass == KNF_PASS_NORMAL) {
      for (int a = 0; a < 3; a++) v[a] = hit[i] ? 0.5 * ((double)normal[3 * i + a] + 1.0) : 0.0;
    } else {
      float d = depth[i];
      double g = isfinite(d) ? 1.0 / (1.0 + (double)d) : 0.0;
      v[0] = v[1] = v[2] = g;
    }
    for (int a = 0; a < 3; a++) out[3 * i + a] = (unsigned char)(fmin(fmax(v[a], 0.0), 1.0) * 255.0 + 0.5);
  }
}
__global__ void tonemap_u8_kernel(const double* __restrict__ img, long long n, double divisor, int gamma22,
                                  unsigned char* __restrict__ out) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = fmin(fmax(img[i] / divisor, 0.0), 1.0);
    if (gamma22) v = pow(v, 1.0 / 2.2);
    out[i] = (unsigned char)(fmin(fmax(v, 0.0), 1.0) * 255.0 + 0.5);
  }
}
struct LatticeDev {
  double start[3], stop[3], step[3];
  int res;
};
// np.linspace: arange(num) * step + start with the last sample forced to `stop`; meshgrid(indexing="ij").
__global__ void lattice_emit_kernel(RouteBuffers R, GridGeom G, LatticeDev L, long long base, int n) {
  int stride = gridDim.x * blockDim.x;
  int n_round = (n + 31) & ~31;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_round; s += stride) {
    bool act = s < n;
    float p[3] = {0.f, 0.f, 0.f};
    if (act) {
      long long idx = base + s;
      int ijk[3] = {(int)(idx / ((long long)L.res * L.res)), (int)((idx / L.res) % L.res), (int)(idx % L.res)};
      for (int a = 0; a < 3; a++) {
        double c = ijk[a] == L.res - 1 ? L.stop[a] : (double)ijk[a] * L.step[a] + L.start[a];
        p[a] = __double2float_rn(c);
      }
    }
    route_emit(R, G, act, s, p[0], p[1], p[2]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) R.ctr->n_requests = n;
}

int unary_op(const float* x, int64_t n, int which, float* out, int device, int mem, void* stream) {
  if (n < 0 || (n > 0 && (!x || !out))) return fail(KNF_E_INVALID, "bad arguments to an activation operator");
  if (n == 0) return 0;
  KNF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  Stager S(nullptr, mem, st);
  const float* dx = S.in(x, (size_t)n);
  float* dout = S.out(out, (size_t)n);
  if (S.rc) return S.rc;
  activation_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(dx, (long long)n, which, dout);
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

}  // namespace

extern "C" {

int knf_fourier_encode(const float* x, int64_t n, int32_t L, float* out, int device, int mem, void* stream) {
  if (n < 0 || (n > 0 && (!x || !out))) return fail(KNF_E_INVALID, "bad arguments to knf_fourier_encode");
  if (L < 0) return fail(KNF_E_INVALID, "L must be >= 0");
  if (L > 8) return fail(KNF_E_UNSUPPORTED, "L > 8 is not supported");
  if (n == 0) return 0;
  KNF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  Stager S(nullptr, mem, st);
  const float* dx = S.in(x, (size_t)n * 3);
  float* dout = S.out(out, (size_t)n * (3 + 6 * L));
  if (S.rc) return S.rc;
  fourier_encode_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(dx, (long long)n, L, dout);
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}
int knf_softplus(const float* x, int64_t n, float* out, int device, int mem, void* stream) {
  return unary_op(x, n, 0, out, device, mem, stream);
}
int knf_sigmoid(const float* x, int64_t n, float* out, int device, int mem, void* stream) {
  return unary_op(x, n, 1, out, device, mem, stream);
}

int knf_abi_version(void) { return KNF_ABI_VERSION; }
const char* knf_last_error(void) { return knf::last_error().c_str(); }

int knf_device_count(void) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(KNF_E_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  return n;
}

int knf_field_create(const KnfFieldDesc* desc, int device, knf_field_t* out) {
  if (!out) return fail(KNF_E_INVALID, "null output handle");
  *out = nullptr;
  KNF_TRY(validate_desc(desc));
  return create_from_stacks(desc, device, out);
}

// modelio.load_model (modelio.py:127-165): header, layer specs, payload, CRC32 trailer.
int knf_field_create_from_knf(const char* path, int device, knf_field_t* out) {
  if (!out) return fail(KNF_E_INVALID, "null output handle");
  *out = nullptr;
  if (!path) return fail(KNF_E_INVALID, "null path");
  FILE* fh = std::fopen(path, "rb");
  if (!fh) return fail(KNF_E_IO, std::string("cannot open ") + path);
  std::vector<unsigned char> buf;
  std::fseek(fh, 0, SEEK_END);
  long size = std::ftell(fh);
  std::fseek(fh, 0, SEEK_SET);
  buf.resize(size > 0 ? (size_t)size : 0);
  size_t got = buf.empty() ? 0 : std::fread(buf.data(), 1, buf.size(), fh);
  std::fclose(fh);
  if (got != buf.size()) return fail(KNF_E_IO, "short read");
  auto u32 = [&](size_t off) {
    uint32_t v;
    std::memcpy(&v, buf.data() + off, 4);
    return v;
  };
  if (buf.size() < 48 || std::memcmp(buf.data(), "KNSF", 4) != 0) return fail(KNF_E_IO, "bad magic: expected KNSF");
  if (u32(4) != 1) return fail(KNF_E_IO, "format version mismatch: supported 1");
  KnfFieldDesc d{};
  d.resolution = (int32_t)u32(8);
  float bbox[6];
  std::memcpy(bbox, buf.data() + 12, 24);
  for (int a = 0; a < 3; a++) {
    d.bbox_min[a] = bbox[a];
    d.bbox_max[a] = bbox[3 + a];
  }
  d.feature_dim = (int32_t)u32(36);
  d.sdf_freqs = (int32_t)u32(40);
  d.dir_freqs = (int32_t)u32(44);
  d.fd_step = 1e-3;  // not stored in the file; GridConfig default (grid.py:40)
  size_t off = 48;
  int dims[2][4];
  for (int fam = 0; fam < 2; fam++) {
    if (off + 4 > buf.size()) return fail(KNF_E_IO, "truncated header");
    uint32_t nl = u32(off);
    off += 4;
    if (nl != 3) return fail(KNF_E_UNSUPPORTED, "only 3-layer MLPs are supported");
    if (off + 4 * 7 > buf.size()) return fail(KNF_E_IO, "truncated header");
    for (int k = 0; k < 4; k++) dims[fam][k] = (int)u32(off + 4 * k);
    off += 16;
    uint32_t acts[3] = {u32(off), u32(off + 4), u32(off + 8)};
    off += 12;
    const uint32_t want_sdf[3] = {2, 2, 0}, want_col[3] = {1, 1, 3};  // nn.py:22 codes
    const uint32_t* want = fam == 0 ? want_sdf : want_col;
    for (int k = 0; k < 3; k++)
      if (acts[k] != want[k]) return fail(KNF_E_UNSUPPORTED, "unsupported activation sequence");
  }
  const int want_dims[2][4] = {{kSdfIn, kHidden, kHidden, kSdfOut}, {kColIn, kHidden, kHidden, kColOut}};
  for (int fam = 0; fam < 2; fam++)
    for (int k = 0; k < 4; k++)
      if (dims[fam][k] != want_dims[fam][k]) return fail(KNF_E_UNSUPPORTED, "unsupported layer widths");
  if (d.resolution < 1 || (int64_t)d.resolution * d.resolution * d.resolution > (1 << 24))
    return fail(KNF_E_UNSUPPORTED, "unsupported resolution");
  const size_t n_cells = (size_t)d.resolution * d.resolution * d.resolution;
  const size_t per_sdf = kSdfIn * kHidden + kHidden + kHidden * kHidden + kHidden + kHidden * kSdfOut + kSdfOut;
  const size_t per_col = kColIn * kHidden + kHidden + kHidden * kHidden + kHidden + kHidden * kColOut + kColOut;
  const size_t payload = 4 * (1 + n_cells * (per_sdf + per_col));
  if (buf.size() < off + payload + 4) return fail(KNF_E_IO, "truncated payload");
  if (crc32_bytes(buf.data() + off, payload) != u32(off + payload)) return fail(KNF_E_IO, "payload CRC32 mismatch");
  // Payload rows are cell-major [W1 | b1 | W2 | b2 | W3 | b3] (modelio.py:72-78); split them into the
  // stacked layout knf_field_create expects.
  const float* vals = reinterpret_cast<const float*>(buf.data() + off) + 1;
  std::vector<float> w[2][3], b[2][3];
  const float* cursor = vals;
  for (int fam = 0; fam < 2; fam++) {
    const int* dm = want_dims[fam];
    for (int k = 0; k < 3; k++) {
      w[fam][k].resize(n_cells * dm[k + 1] * dm[k]);
      b[fam][k].resize(n_cells * dm[k + 1]);
    }
    for (size_t c = 0; c < n_cells; c++)
      for (int k = 0; k < 3; k++) {
        size_t nw = (size_t)dm[k + 1] * dm[k], nb = dm[k + 1];
        std::memcpy(w[fam][k].data() + c * nw, cursor, nw * 4);
        cursor += nw;
        std::memcpy(b[fam][k].data() + c * nb, cursor, nb * 4);
        cursor += nb;
      }
  }
  for (int k = 0; k < 3; k++) {
    d.sdf_w[k] = w[0][k].data();
    d.sdf_b[k] = b[0][k].data();
    d.color_w[k] = w[1][k].data();
    d.color_b[k] = b[1][k].data();
  }
  KNF_TRY(validate_desc(&d));
  return create_from_stacks(&d, device, out);
}

int knf_field_destroy(knf_field_t f) {
  if (!f) return 0;
  int prev_device = -1;
  if (cudaGetDevice(&prev_device) != cudaSuccess) prev_device = -1;
  cudaSetDevice(f->f.device);
  {
    std::lock_guard<std::mutex> lk(f->f.mu);
    if (f->f.last_call_valid) cudaEventSynchronize(f->f.last_call_done);  // asynchronous (KNF_MEM_DEVICE) calls may still be using the workspace
    if (f->f.last_call_done) cudaEventDestroy(f->f.last_call_done);
    if (f->f.side_stream) {
      cudaStreamSynchronize(f->f.side_stream);
      cudaStreamDestroy(f->f.side_stream);
      cudaEventDestroy(f->f.ev_fork);
      cudaEventDestroy(f->f.ev_join);
    }
    f->f.ws.release_all();
    for (cudaEvent_t e : f->f.events) cudaEventDestroy(e);
    if (f->f.host_poll) cudaFreeHost(f->f.host_poll);
    if (f->f.sdf_blobs) cudaFree(f->f.sdf_blobs);
    if (f->f.col_blobs) cudaFree(f->f.col_blobs);
    if (f->f.sdf_mma_blobs) cudaFree(f->f.sdf_mma_blobs);
    if (f->f.sdf_mmah_blobs) cudaFree(f->f.sdf_mmah_blobs);
    if (f->f.sdf_tc5_blobs) cudaFree(f->f.sdf_tc5_blobs);
    if (f->f.lip_consts) cudaFree(f->f.lip_consts);
    if (f->f.lip_cur) cudaFree(f->f.lip_cur);
    if (f->f.lip_max) cudaFree(f->f.lip_max);
  }
  delete f;
  if (prev_device >= 0) cudaSetDevice(prev_device);
  cudaGetLastError();
  return 0;
}

int knf_field_describe(knf_field_t f, KnfFieldDesc* desc) {
  KNF_TRY(check_field(f));
  if (!desc) return fail(KNF_E_INVALID, "null desc");
  std::memset(desc, 0, sizeof(*desc));
  desc->resolution = f->f.geom.resolution;
  for (int a = 0; a < 3; a++) {
    desc->bbox_min[a] = f->f.geom.lo[a];
    desc->bbox_max[a] = f->f.geom.hi[a];
  }
  desc->sdf_freqs = f->f.sdf_freqs;
  desc->dir_freqs = f->f.dir_freqs;
  desc->feature_dim = f->f.feature_dim;
  desc->fd_step = f->f.geom.fd_step;
  return 0;
}

int knf_field_stats(knf_field_t f, KnfStats* out) {
  KNF_TRY(check_field(f));
  if (!out) return fail(KNF_E_INVALID, "null stats");
  std::lock_guard<std::mutex> lk(f->f.mu);
  KNF_CUDA(cudaSetDevice(f->f.device));
  KNF_CUDA(cudaDeviceSynchronize());
  if (f->f.ws.counters.p) KNF_TRY(finish_stats(f->f, 0));
  KNF_TRY(collect_profile(f->f));
  *out = f->f.stats;
  return 0;
}

int knf_field_stats_reset(knf_field_t f) {
  KNF_TRY(check_field(f));
  std::lock_guard<std::mutex> lk(f->f.mu);
  KNF_CUDA(cudaSetDevice(f->f.device));
  KNF_CUDA(cudaDeviceSynchronize());
  KNF_TRY(collect_profile(f->f));
  f->f.stats = KnfStats{};
  if (f->f.ws.counters.p) KNF_CUDA(cudaMemset(stat_counter(f->f, 0), 0, 8 * sizeof(unsigned long long)));
  return 0;
}

int knf_field_set_profiling(knf_field_t f, int enable) {
  KNF_TRY(check_field(f));
  std::lock_guard<std::mutex> lk(f->f.mu);
  f->f.profiling = enable != 0;
  return 0;
}

int knf_field_set_precision(knf_field_t f, int mode) {
  KNF_TRY(check_field(f));
  if (mode != KNF_PRECISION_FP32_CHAIN && mode != KNF_PRECISION_TENSOR_BF16X3 && mode != KNF_PRECISION_TENSOR_FP16X2)
    return fail(KNF_E_INVALID, "unknown KNF_PRECISION_* mode");
  if (mode == KNF_PRECISION_TENSOR_FP16X2 && (!f->f.fp16_ok || f->f.filter_cells_off > 0))
    return fail(KNF_E_UNSUPPORTED, "KNF_PRECISION_TENSOR_FP16X2 needs hidden-layer weights and activation bounds below 6e4 in magnitude");
  std::lock_guard<std::mutex> lk(f->f.mu);
  f->f.precision = mode;
  return 0;
}

int knf_field_get_precision(knf_field_t f) {
  KNF_TRY(check_field(f));
  return f->f.precision;
}

int knf_field_set_filter(knf_field_t f, int mode) {
  KNF_TRY(check_field(f));
  if (mode != KNF_FILTER_OFF && mode != KNF_FILTER_ON && mode != KNF_FILTER_AUTO) return fail(KNF_E_INVALID, "unknown KNF_FILTER_* mode");
  std::lock_guard<std::mutex> lk(f->f.mu);
  f->f.filter_mode = mode;
  return 0;
}

double knf_field_filter_delta(knf_field_t f) {
  if (check_field(f) != 0) return -1.0;
  return f->f.filter_delta_max;
}

const char* knf_field_filter_kernel(knf_field_t f) {
  if (check_field(f) != 0) return "";
  return (f->f.filter_kernel == 1 && f->f.sdf_tc5_blobs) ? "march_tc5_kernel" : "march_mma_kernel<2, true>";
}

int knf_field_filter_cells_off(knf_field_t f) {
  KNF_TRY(check_field(f));
  return f->f.fp16_ok ? f->f.filter_cells_off : f->f.geom.n_cells;
}

int knf_field_lipschitz(knf_field_t f, float* closed_form, float* refined, float* refine_ms, void* stream) {
  KNF_TRY(check_field(f));
  Field& F = f->f;
  if (!F.lip_cur) return fail(KNF_E_UNSUPPORTED, "this field has no decision-filter blobs (weights beyond the fp16 range): no Lipschitz bounds");
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  const size_t n = (size_t)F.geom.n_cells * 3;
  if (closed_form) std::memcpy(closed_form, F.lip_closed_form.data(), n * sizeof(float));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool timed = refine_ms && !F.lip_refined;
  if (timed) {
    KNF_CUDA(cudaEventCreate(&e0));
    KNF_CUDA(cudaEventCreate(&e1));
    KNF_CUDA(cudaEventRecord(e0, st));
  }
  KNF_TRY(ensure_lipschitz_refined(F, st));
  if (timed) KNF_CUDA(cudaEventRecord(e1, st));
  if (refined) KNF_CUDA(cudaMemcpyAsync(refined, F.lip_cur, n * sizeof(float), cudaMemcpyDeviceToHost, st));
  KNF_CUDA(cudaStreamSynchronize(st));
  if (timed) {
    KNF_CUDA(cudaEventElapsedTime(&F.lip_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (refine_ms) *refine_ms = F.lip_ms;
  return 0;
}

// ---- routing ---------------------------------------------------------------------------------------
extern "C++" {
template <class T>
static int cell_index_impl(knf_field_t f, const T* pts, int64_t n, int32_t* cell, int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!pts || !cell))) return fail(KNF_E_INVALID, "bad arguments to knf_cell_index");
  if (n == 0) return 0;
  if (n > INT32_MAX / 4) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const T* dp = S.in(pts, (size_t)n * 3);
  int32_t* dc = S.out(cell, (size_t)n);
  if (S.rc) return S.rc;
  cell_index_kernel<T><<<blocks_for((size_t)n), 256, 0, st>>>(F.geom, dp, (int)n, dc);
  F.stats.kernel_launches += 1;
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}
}  // extern "C++"

int knf_cell_index(knf_field_t f, const float* pts, int64_t n, int32_t* cell, int mem, void* stream) {
  return cell_index_impl<float>(f, pts, n, cell, mem, stream);
}
int knf_cell_index_f64(knf_field_t f, const double* pts, int64_t n, int32_t* cell, int mem, void* stream) {
  return cell_index_impl<double>(f, pts, n, cell, mem, stream);
}

int knf_route(knf_field_t f, const float* pts, int64_t n, int32_t* cell, int32_t* order, int32_t* seg_cell,
              int32_t* seg_start, int32_t* n_seg, int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && !pts)) return fail(KNF_E_INVALID, "bad arguments to knf_route");
  if ((seg_cell == nullptr) != (seg_start == nullptr)) return fail(KNF_E_INVALID, "seg_cell and seg_start go together");
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  size_t nseg_cap = std::min<size_t>((size_t)std::max<int64_t>(n, 1), (size_t)F.geom.n_cells);
  const float* dp = S.in(pts, (size_t)n * 3);
  int32_t* dcell = S.out(cell, (size_t)n);
  int32_t* dorder = S.out(order, (size_t)n);
  int32_t* dsc = S.out(seg_cell, nseg_cap);
  int32_t* dss = S.out(seg_start, nseg_cap + 1);
  int32_t* dns = S.out(n_seg, 1);
  if (S.rc) return S.rc;
  KNF_TRY(ensure_requests(F, (size_t)std::max<int64_t>(n, 1)));
  RouteBuffers R = route_buffers(F, 2, -1);
  route_emit_points_kernel<<<blocks_for((size_t)std::max<int64_t>(n, 1)), 256, 0, st>>>(R, F.geom, dp, (int)n, dcell);
  F.stats.kernel_launches += 1;
  KNF_TRY(launch_scan_scatter(F, R, (size_t)std::max<int64_t>(n, 1), st, dsc, dss, dns));
  if (dorder && n > 0)
    KNF_CUDA(cudaMemcpyAsync(dorder, R.perm, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, st));
  return S.finish();
}

// ---- batched forward -----------------------------------------------------------------------------------
int knf_sdf_forward(knf_field_t f, const float* pts, int64_t n, float* out, int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!pts || !out))) return fail(KNF_E_INVALID, "bad arguments to knf_sdf_forward");
  if (n == 0) return 0;
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const float* dp = S.in(pts, (size_t)n * 3);
  float* dout = S.out(out, (size_t)n * kSdfOut);
  if (S.rc) return S.rc;
  KNF_TRY(sdf_forward_device(F, dp, n, dout, nullptr, nullptr, st));
  return S.finish();
}

int knf_sdf_values(knf_field_t f, const float* pts, int64_t n, float* dist, int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!pts || !dist))) return fail(KNF_E_INVALID, "bad arguments to knf_sdf_values");
  if (n == 0) return 0;
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const float* dp = S.in(pts, (size_t)n * 3);
  float* dd = S.out(dist, (size_t)n);
  if (S.rc) return S.rc;
  KNF_TRY(sdf_forward_device(F, dp, n, nullptr, dd, nullptr, st));
  return S.finish();
}

int knf_sdf_gradient(knf_field_t f, const float* pts, int64_t n, float* dist, float* grad, int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!pts || !grad))) return fail(KNF_E_INVALID, "bad arguments to knf_sdf_gradient");
  if (n == 0) return 0;
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const float* dp = S.in(pts, (size_t)n * 3);
  float* dd = dist ? S.out(dist, (size_t)n) : nullptr;
  float* dg = S.out(grad, (size_t)n * 3);
  if (S.rc) return S.rc;
  KNF_TRY(ensure_requests(F, (size_t)n));
  RouteBuffers R = route_buffers(F, 2, -1);
  route_emit_points_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(R, F.geom, dp, (int)n, nullptr);
  KNF_TRY(launch_scan_scatter(F, R, (size_t)n, st));
  static bool configured = false;
  if (!configured) {
    KNF_CUDA(cudaFuncSetAttribute(sdf_gradient_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(GradSmem)));
    configured = true;
  }
  GradParams G{};
  G.P.blobs = F.sdf_blobs;
  G.P.perm = R.perm;
  G.P.tiles = R.tiles;
  G.P.ctr = R.ctr;
  G.P.req_pt = R.req_pt;
  G.dist = dd;
  G.grad = dg;
  const size_t tiles_upper = (size_t)n / kSmallTile + std::min<size_t>((size_t)n, (size_t)F.geom.n_cells) + 1;
  sdf_gradient_kernel<<<(int)std::min<size_t>(tiles_upper, 148 * 5), 32, sizeof(GradSmem), st>>>(G);
  F.stats.kernel_launches += 4;
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

int knf_color_forward(knf_field_t f, const float* x, const float* v, const float* nrm, const float* z, int64_t n,
                      float* rgb, int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!x || !v || !nrm || !z || !rgb))) return fail(KNF_E_INVALID, "bad arguments to knf_color_forward");
  if (n == 0) return 0;
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const float* dx = S.in(x, (size_t)n * 3);
  const float* dv = S.in(v, (size_t)n * 3);
  const float* dn = S.in(nrm, (size_t)n * 3);
  const float* dz = S.in(z, (size_t)n * kFeat);
  float* drgb = S.out(rgb, (size_t)n * 3);
  if (S.rc) return S.rc;
  KNF_TRY(color_forward_device(F, dx, dv, dn, dz, n, drgb, st));
  return S.finish();
}

// ---- FD normals -----------------------------------------------------------------------------------------
int knf_fd_gradient(knf_field_t f, const double* pts, int64_t n, double* grad, int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!pts || !grad))) return fail(KNF_E_INVALID, "bad arguments to knf_fd_gradient");
  if (n == 0) return 0;
  if (n > INT32_MAX / 128) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const double* dp = S.in(pts, (size_t)n * 3);
  double* dg = S.out(grad, (size_t)n * 3);
  if (S.rc) return S.rc;
  ShadeTargets T;
  T.grad = dg;
  KNF_TRY(shade_points_device(F, dp, nullptr, n, T, st));
  return S.finish();
}

int knf_fd_normals(knf_field_t f, const double* pts, int64_t n, double eps, double* nrm, uint8_t* ok, int mem,
                   void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!pts || !nrm))) return fail(KNF_E_INVALID, "bad arguments to knf_fd_normals");
  if (n == 0) return 0;
  if (n > INT32_MAX / 128) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const double* dp = S.in(pts, (size_t)n * 3);
  double* dn = S.out(nrm, (size_t)n * 3);
  uint8_t* dok = S.out(ok, (size_t)n);
  if (S.rc) return S.rc;
  ShadeTargets T;
  T.normals = dn;
  T.ok = dok;
  T.eps = eps;
  KNF_TRY(shade_points_device(F, dp, nullptr, n, T, st));
  return S.finish();
}

// ---- rays -------------------------------------------------------------------------------------------------
int knf_pixel_rays(const KnfCamera* cam, const int32_t* pixel_xy, const double* jitter, int64_t n, double* origins,
                   double* dirs, int device, int mem, void* stream) {
  if (!cam || n < 0 || (n > 0 && (!origins || !dirs))) return fail(KNF_E_INVALID, "bad arguments to knf_pixel_rays");
  if (cam->width <= 0 || cam->height <= 0) return fail(KNF_E_INVALID, "image dimensions must be positive");
  if (!pixel_xy && n != (int64_t)cam->width * cam->height)
    return fail(KNF_E_INVALID, "n must equal width*height when pixel_xy is NULL");
  if (n == 0) return 0;
  KNF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  Stager S(nullptr, mem, st);
  const int32_t* dpx = S.in(pixel_xy, (size_t)n * 2);
  const double* dj = S.in(jitter, (size_t)n * 2);
  double* dorig = S.out(origins, (size_t)n * 3);
  double* ddir = S.out(dirs, (size_t)n * 3);
  if (S.rc) return S.rc;
  pixel_rays_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(make_camera(*cam, 1), dpx, dj, (long long)n, dorig, ddir);
  KNF_CUDA(cudaGetLastError());
  int rc = S.finish();
  if (rc == 0 && mem == KNF_MEM_HOST) return 0;
  return rc;
}

int knf_ray_aabb(const double* origins, const double* dirs, int64_t n, const double bbox_min[3],
                 const double bbox_max[3], double* t_near, double* t_far, uint8_t* hit, int device, int mem,
                 void* stream) {
  if (n < 0 || (n > 0 && (!origins || !dirs || !t_near || !t_far)) || !bbox_min || !bbox_max)
    return fail(KNF_E_INVALID, "bad arguments to knf_ray_aabb");
  if (n == 0) return 0;
  KNF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  Stager S(nullptr, mem, st);
  const double* dorig = S.in(origins, (size_t)n * 3);
  const double* ddir = S.in(dirs, (size_t)n * 3);
  double* dtn = S.out(t_near, (size_t)n);
  double* dtf = S.out(t_far, (size_t)n);
  uint8_t* dh = S.out(hit, (size_t)n);
  if (S.rc) return S.rc;
  GridGeom box{};
  for (int a = 0; a < 3; a++) {
    box.lo[a] = bbox_min[a];
    box.hi[a] = bbox_max[a];
  }
  ray_aabb_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(dorig, ddir, (long long)n, box, dtn, dtf, dh, 0);
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

// ---- sphere tracing + shading ----------------------------------------------------------------------------------
int knf_march(knf_field_t f, const double* origins, const double* dirs, const double* t_near, const double* t_far,
              int64_t n, const KnfSettings* s, uint8_t* hit, double* t, double* position, int32_t* steps, int mem,
              void* stream) {
  KNF_TRY(check_field(f));
  KNF_TRY(check_settings(s));
  if (n < 0 || (n > 0 && (!origins || !dirs || !t_near || !t_far || !hit || !t)))
    return fail(KNF_E_INVALID, "bad arguments to knf_march");
  if (n == 0) return 0;
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const double* dorig = S.in(origins, (size_t)n * 3);
  const double* ddir = S.in(dirs, (size_t)n * 3);
  const double* dtn = S.in(t_near, (size_t)n);
  const double* dtf = S.in(t_far, (size_t)n);
  uint8_t* dh = S.out(hit, (size_t)n);
  double* dt = S.out(t, (size_t)n);
  double* dpos = S.out(position, (size_t)n * 3);
  int32_t* dsteps = S.out(steps, (size_t)n);
  if (S.rc) return S.rc;
  KNF_TRY(march_device(F, dorig, ddir, dtn, dtf, n, *s, dh, dt, dpos, dsteps, false, st));
  return S.finish();
}

int knf_shade(knf_field_t f, const double* pts, const double* view_dirs, int64_t n, double* colors, double* normals,
              int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (n < 0 || (n > 0 && (!pts || !view_dirs || !colors || !normals)))
    return fail(KNF_E_INVALID, "bad arguments to knf_shade");
  if (n == 0) return 0;
  if (n > INT32_MAX / 128) return fail(KNF_E_INVALID, "too many points for one call");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const double* dp = S.in(pts, (size_t)n * 3);
  const double* dv = S.in(view_dirs, (size_t)n * 3);
  double* dc = S.out(colors, (size_t)n * 3);
  double* dn = S.out(normals, (size_t)n * 3);
  if (S.rc) return S.rc;
  ShadeTargets T;
  T.normals = dn;
  T.colors = dc;
  T.fallback = true;
  KNF_TRY(shade_points_device(F, dp, dv, n, T, st));
  return S.finish();
}

// Shared by knf_trace_and_shade and knf_render_frame: march, then shade the hits in chunks.
static int trace_shade_device(Field& F, const double* o, const double* d, const double* tn, const double* tf, int64_t n,
                              const KnfSettings& s, uint8_t* hit, double* t, double* pos, int32_t* steps,
                              double* normals, double* colors, cudaStream_t st) {
  KNF_TRY(march_device(F, o, d, tn, tf, n, s, hit, t, pos, steps, true, st));
  KNF_CUDA(cudaMemsetAsync(normals, 0, (size_t)n * 3 * sizeof(double), st));
  KNF_CUDA(cudaMemsetAsync(colors, 0, (size_t)n * 3 * sizeof(double), st));
  int m = 0;
  KNF_TRY(read_hit_count(F, st, &m));
  if (m > 0) {
    ShadeTargets T;
    T.normals = normals;
    T.colors = colors;
    T.fallback = true;
    T.scatter_by_ray = true;
    T.clip_colors = true;
    // chunk so that 7 * chunk requests stay within 32-bit routing indices and modest scratch
    const int64_t chunk = 1 << 20;
    for (int64_t base = 0; base < m; base += chunk) {
      int64_t cnt = std::min<int64_t>(chunk, m - base);
      KNF_TRY(shade_hits_device(F, o, d, base, cnt, T, st));
    }
  }
  return 0;
}

int knf_trace_and_shade(knf_field_t f, const double* origins, const double* dirs, int64_t n, const KnfSettings* s,
                        uint8_t* hit, double* t, double* position, int32_t* steps, double* normals, double* colors,
                        int mem, void* stream) {
  KNF_TRY(check_field(f));
  KNF_TRY(check_settings(s));
  if (n < 0 || (n > 0 && (!origins || !dirs || !hit || !t || !normals || !colors)))
    return fail(KNF_E_INVALID, "bad arguments to knf_trace_and_shade");
  if (n == 0) return 0;
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  Stager S(&F, mem, st);
  const double* dorig = S.in(origins, (size_t)n * 3);
  const double* ddir = S.in(dirs, (size_t)n * 3);
  uint8_t* dh = S.out(hit, (size_t)n);
  double* dt = S.out(t, (size_t)n);
  double* dpos = S.out(position, (size_t)n * 3);
  int32_t* dsteps = S.out(steps, (size_t)n);
  double* dnrm = S.out(normals, (size_t)n * 3);
  double* dcol = S.out(colors, (size_t)n * 3);
  if (S.rc) return S.rc;
  Workspace& W = F.ws;
  KNF_TRY(W.t_near.ensure((size_t)n * 8));
  KNF_TRY(W.t_far.ensure((size_t)n * 8));
  ray_aabb_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(dorig, ddir, (long long)n, F.geom, W.t_near.as<double>(),
                                                       W.t_far.as<double>(), nullptr, 1);
  F.stats.kernel_launches += 1;
  KNF_TRY(trace_shade_device(F, dorig, ddir, W.t_near.as<double>(), W.t_far.as<double>(), n, *s, dh, dt, dpos, dsteps,
                             dnrm, dcol, st));
  return S.finish();
}

// Rows [row0,row1) of a frame into device buffers (shared by knf_render_frame and knf_render_pass_u8).
static int render_rows_device(Field& F, const KnfCamera& cam, const KnfSettings& s, const double background[3], int ss,
                              int row0, int row1, float* dcolor, float* ddepth, float* dnormal, uint8_t* dhit,
                              cudaStream_t st) {
  const int W_ = cam.width;
  const int rows = row1 - row0;
  CameraDev cd = make_camera(cam, ss);
  // process row chunks so a chunk holds at most ~4M sub-rays
  const int64_t per_row = (int64_t)W_ * ss * ss;
  int rows_per_chunk = (int)std::max<int64_t>(1, (4ll << 20) / per_row);
  Workspace& W = F.ws;
  for (int r = 0; r < rows; r += rows_per_chunk) {
    int rc_rows = std::min(rows_per_chunk, rows - r);
    int64_t n = (int64_t)rc_rows * per_row;
    KNF_TRY(W.origins.ensure((size_t)n * 24));
    KNF_TRY(W.dirs.ensure((size_t)n * 24));
    KNF_TRY(W.t_near.ensure((size_t)n * 8));
    KNF_TRY(W.t_far.ensure((size_t)n * 8));
    KNF_TRY(W.normals64.ensure((size_t)n * 24));
    KNF_TRY(W.colors64.ensure((size_t)n * 24));
    KNF_TRY(ensure_rays(F, (size_t)n));
    primary_rays_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(cd, F.geom, (row0 + r) * ss, (long long)n,
                                                             W.origins.as<double>(), W.dirs.as<double>(),
                                                             W.t_near.as<double>(), W.t_far.as<double>());
    F.stats.kernel_launches += 1;
    KNF_TRY(trace_shade_device(F, W.origins.as<double>(), W.dirs.as<double>(), W.t_near.as<double>(),
                               W.t_far.as<double>(), n, s, nullptr, nullptr, nullptr, nullptr,
                               W.normals64.as<double>(), W.colors64.as<double>(), st));
    compose_kernel<<<blocks_for((size_t)rc_rows * W_), 256, 0, st>>>(
        rc_rows, W_, ss, W.hit.as<unsigned char>(), W.t_hit.as<double>(), W.normals64.as<double>(),
        W.colors64.as<double>(), background[0], background[1], background[2], dcolor + (size_t)r * W_ * 3,
        ddepth + (size_t)r * W_, dnormal + (size_t)r * W_ * 3, dhit + (size_t)r * W_);
    F.stats.kernel_launches += 1;
    KNF_CUDA(cudaGetLastError());
  }
  return 0;
}

static int check_frame_args(const KnfCamera* cam, const double* background, int supersample, int row0, int row1) {
  if (!cam || !background) return fail(KNF_E_INVALID, "null camera or background");
  if (supersample < 1) return fail(KNF_E_INVALID, "supersample must be >= 1");
  if (cam->width <= 0 || cam->height <= 0) return fail(KNF_E_INVALID, "image dimensions must be positive");
  if (row0 < 0 || row1 > cam->height || row0 >= row1) return fail(KNF_E_INVALID, "row range out of bounds");
  return 0;
}

int knf_render_frame(knf_field_t f, const KnfCamera* cam, const KnfSettings* s, const double background[3],
                     int supersample, int row0, int row1, float* color, float* depth, float* normal, uint8_t* hit,
                     int mem, void* stream) {
  KNF_TRY(check_field(f));
  KNF_TRY(check_settings(s));
  KNF_TRY(check_frame_args(cam, background, supersample, row0, row1));
  if (!color || !depth || !normal || !hit) return fail(KNF_E_INVALID, "null argument to knf_render_frame");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  const size_t px = (size_t)(row1 - row0) * cam->width;
  Stager S(&F, mem, st);
  float* dcolor = S.out(color, px * 3);
  float* ddepth = S.out(depth, px);
  float* dnormal = S.out(normal, px * 3);
  uint8_t* dhit = S.out(hit, px);
  if (S.rc) return S.rc;
  KNF_TRY(render_rows_device(F, *cam, *s, background, supersample, row0, row1, dcolor, ddepth, dnormal, dhit, st));
  return S.finish();
}

// SURVEY 8(f).2, the interactive caller (service._render_once, service.py:279-288): render_frame ->
// surface.pass_image (surface.py:339-350) -> images.to_uint8 (images.py:15-17), all on the device, so
// only 3 bytes per pixel cross PCIe instead of 29.
int knf_render_pass_u8(knf_field_t f, const KnfCamera* cam, const KnfSettings* s, const double background[3],
                       int supersample, int render_pass, int row0, int row1, uint8_t* rgb, int mem, void* stream) {
  KNF_TRY(check_field(f));
  KNF_TRY(check_settings(s));
  KNF_TRY(check_frame_args(cam, background, supersample, row0, row1));
  if (!rgb) return fail(KNF_E_INVALID, "null output image");
  if (render_pass < KNF_PASS_COLOR || render_pass > KNF_PASS_DEPTH) return fail(KNF_E_INVALID, "unknown pass");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  const size_t px = (size_t)(row1 - row0) * cam->width;
  Stager S(&F, mem, st);
  uint8_t* drgb = S.out(rgb, px * 3);
  if (S.rc) return S.rc;
  Workspace& W = F.ws;
  KNF_TRY(W.frame_color.ensure(px * 12));
  KNF_TRY(W.frame_depth.ensure(px * 4));
  KNF_TRY(W.frame_normal.ensure(px * 12));
  KNF_TRY(W.frame_hit.ensure(px));
  KNF_TRY(render_rows_device(F, *cam, *s, background, supersample, row0, row1, W.frame_color.as<float>(),
                             W.frame_depth.as<float>(), W.frame_normal.as<float>(), W.frame_hit.as<uint8_t>(), st));
  pass_u8_kernel<<<blocks_for(px), 256, 0, st>>>(render_pass, (long long)px, W.frame_color.as<float>(),
                                                W.frame_depth.as<float>(), W.frame_normal.as<float>(),
                                                W.frame_hit.as<uint8_t>(), drgb);
  F.stats.kernel_launches += 1;
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

// images.to_uint8 of an fp64 image, optionally after the path tracer's display transform
// clip(hdr / divisor, 0, 1) ** (1 / 2.2) (service.py:297-299, pathtrace.py:470).
int knf_tonemap_u8(const double* img, int64_t n, double divisor, int gamma22, uint8_t* out, int device, int mem, void* stream) {
  if (n < 0 || (n > 0 && (!img || !out)) || !(divisor > 0)) return fail(KNF_E_INVALID, "bad arguments to knf_tonemap_u8");
  if (n == 0) return 0;
  KNF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  Stager S(nullptr, mem, st);
  const double* din = S.in(img, (size_t)n);
  uint8_t* dout = S.out(out, (size_t)n);
  if (S.rc) return S.rc;
  tonemap_u8_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(din, (long long)n, divisor, gamma22, dout);
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

// SURVEY 8(f).4, mesh._sample_volume (mesh.py:43-57): SDF values on an R^3 np.linspace lattice
// (x-major, "ij" order), lattice points generated on the device.
int knf_sample_volume(knf_field_t f, int32_t resolution, const double bbox_min[3], const double bbox_max[3], float* values,
                      int mem, void* stream) {
  KNF_TRY(check_field(f));
  if (resolution < 2 || !bbox_min || !bbox_max || !values) return fail(KNF_E_INVALID, "bad arguments to knf_sample_volume");
  if (resolution > 1024) return fail(KNF_E_UNSUPPORTED, "resolution > 1024 is not supported");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  const int64_t R = resolution, total = R * R * R;
  Stager S(&F, mem, st);
  float* dvals = S.out(values, (size_t)total);
  if (S.rc) return S.rc;
  LatticeDev L;
  for (int a = 0; a < 3; a++) {
    L.start[a] = bbox_min[a];
    L.stop[a] = bbox_max[a];
    L.step[a] = (bbox_max[a] - bbox_min[a]) / (double)(resolution - 1);  // np.linspace's step
  }
  L.res = resolution;
  const int64_t chunk = 16ll << 20;
  for (int64_t base = 0; base < total; base += chunk) {
    const int64_t n = std::min(chunk, total - base);
    KNF_TRY(ensure_requests(F, (size_t)n));
    RouteBuffers Rb = route_buffers(F, 2, -1);
    Rb.eval_counter = stat_counter(F, 0);
    lattice_emit_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(Rb, F.geom, L, (long long)base, (int)n);
    F.stats.kernel_launches += 1;
    KNF_TRY(launch_scan_scatter(F, Rb, (size_t)n, st));
    KNF_TRY(launch_sdf_mlp(F, Rb, (size_t)n, dvals + base, nullptr, st));
  }
  return S.finish();
}

}  // extern "C"
