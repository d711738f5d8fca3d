// knf_bounds.cuh -- per-cell, per-axis Lipschitz bounds of the SDF network, computed on the device at first use.
//
// The decision filter (knf_tc5.cuh / knf_march.cuh) skips the reference's crawl steps without evaluating anything while
// sum_a L_a |p_a - p0_a| stays below the room the filter distance left (certified skipping).  L_a must be a PROVEN bound on
// |d d / d x_a| over the cell; how far a ray can skip -- and with it the number of filter evaluations of a frame -- is
// inversely proportional to it.  The closed-form bound of knf_api.cu (|w3| |W2| |W1 J_a|, softplus' <= 1) is 16-20 x the
// largest gradient that actually occurs in a random-init cell.  This kernel tightens it by bound propagation over sub-boxes:
//
//   d(x) = w3 . sp(z2) + b3,  z2 = W2 sp(z1) + b2,  z1 = W1 phi(x) + b1        (sp = softplus, phi = nn.fourier_encode)
//   d d / d x_a = w3^T S2 W2 S1 g_a(x_a),   S_i = diag(sigmoid(z_i)),   g_a = W1 d phi / d x_a  (a function of x_a alone)
//
// The cell (extended by `margin` per face) is cut into k^3 sub-boxes Q.  On Q:
//   1. every feature is enclosed exactly (raw coordinate: the interval; sin / cos of 2^o pi x_a: end-point values plus the
//      interior extrema), phi in phi_c +- phi_r;
//   2. z1 in z1c +- z1r with z1c = W1 phi_c + b1, z1r = |W1| phi_r; sigmoid and softplus are monotone, so
//      S1 = C1 + R1 D1 with |D1| <= 1 (C1, R1 diagonal: centre and radius of [sigmoid(z1c - z1r), sigmoid(z1c + z1r)]),
//      sp(z1) in h1c +- h1r; the same through layer 2 gives S2 = C2 + R2 D2;
//   3. w3^T (C2 + R2 D2) W2 (C1 + R1 D1) g, expanded, is bounded term by term for ANY |D1|, |D2| <= 1:
//        Phi(g) = |v~ . (c1 o g)|  +  sum_m r2_m |w3_m| |(W2 (c1 o g))_m|  +  sum_n |v~_n| r1_n |g_n|  +  T4(g),
//        v~ = W2^T (c2 o w3),   T4 = |r2 o w3|_2 |W2|_2 |r1 o g|_2   or   sum_mn r2_m |w3_m| |W2_mn| r1_n |g_n|
//      (two variants A / B of the bilinear term; each makes Phi a seminorm in g, the smaller total is taken);
//   4. g_a varies inside the sub-box's x_a interval: it is sampled at `fine` midpoints x_i with a first-order Taylor
//      model, g(x) = g(x_i) + (x - x_i) g'(x_i) + rho, |rho|_2 <= (x - x_i)^2 / 2 * K3_a, K3_a = sum_o (2^o pi)^3
//      sigma_max([w_sin_o,a | w_cos_o,a]); Phi is a seminorm and Phi(rho) <= (2 |w3| |W2| (+ |w3| |W2|_F for variant B)) |rho|,
//      so  sup Phi(g(x)) <= Phi(g_i) + h Phi(g'_i) + const * h^2 K3_a / 2   with h half the sample spacing.
// L_a = 1.001 x the maximum over sub-boxes and samples (+ 1e-12), never more than the closed-form bound.  As the sub-boxes
// shrink, R -> 0 and the bound tends to the true maximum of |d d / d x_a|; with sub-boxes 0.004 wide it is 7-10 x below
// the closed form on a random-init 16^3 field.  All arithmetic is fp64 with radii inflated by 1e-12 relative + 1e-13
// absolute per stage -- orders of magnitude above the rounding errors of 40-term fp64 sums -- and a final factor 1.001.
//
// One warp per sub-box, lane = hidden unit; the cell's weights sit in shared memory as fp64 (from the fp32 chain blob).
#pragma once

#include "knf_common.cuh"

namespace knf {

// host-computed per cell (knf_api.cu lipschitz_consts)
struct LipCellConst {
  double n3;     // |w3|_2 (the distance row of the output layer)
  double n2;     // proven upper bound on |W2|_2 (Gershgorin on (W2^T W2)^16)
  double n2f;    // |W2|_F (>= the spectral norm of |W2|)
  double k3[3];  // sum_o (2^o pi)^3 sigma_max([w_sin_o,a | w_cos_o,a]): bound on |g_a''|_2
};

struct LipArgs {
  const float* blobs;       // SdfBlob per cell (k-major fp32 chain layout)
  const LipCellConst* cc;
  GridGeom G;
  int k;                    // sub-boxes per axis
  int fine;                 // Taylor samples of g_a per sub-box interval (<= 4)
  double margin;            // the cell box is extended by this much per face
  unsigned long long* out;  // [n_cells][3]: running maximum as the bit pattern of a non-negative double (zeroed by the caller)
};

constexpr int kLipWarps = 8;
constexpr int kLipMaxFine = 4;

#ifndef KNF_BOUNDS_LAYOUT_ONLY
struct LipWarpScratch {
  // (centre, radius) / paired vectors interleaved: every broadcast read of a pair is one 16-byte shared-memory wavefront
  double2 phi[40];          // .x centre, .y radius
  double2 vab[kHidden];     // layer 2: (h1c, h1r); then (c2 w3, r2 |w3|)
  double2 vcd[kHidden];     // (c1 o g, c1 o g')
  double trig[3 * kLipMaxFine][2 * kSdfFreqs];  // [axis * fine + i][2 o] = sin(2^o pi x_i), [2 o + 1] = cos
};

struct LipSmem {
  double w1t[kSdfIn * kHidden];    // [k][n] = W1[n][k]
  double w2t[kHidden * kHidden];   // [n][m] = W2[m][n]   (lane = output unit m)
  double w2r[kHidden * kHidden];   // [m][n] = W2[m][n]   (lane = input unit n)
  double b1[kHidden], b2[kHidden], w3[kHidden];
  LipWarpScratch ws[kLipWarps];
};

__device__ __forceinline__ double lip_warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// does [lo, hi] contain p + 2 pi j for some integer j?
__device__ __forceinline__ bool lip_contains(double lo, double hi, double p) {
  const double two_pi = 6.283185307179586476925286766559;
  return fma(ceil((lo - p) / two_pi), two_pi, p) <= hi;
}

// range of sin and cos over [tlo, thi] as centre / radius
__device__ __forceinline__ void lip_trig_range(double tlo, double thi, double& sc, double& sr, double& cc, double& cr) {
  const double pi = 3.141592653589793238462643383279;
  double s0, c0, s1, c1;
  sincos(tlo, &s0, &c0);
  sincos(thi, &s1, &c1);
  double smin = fmin(s0, s1), smax = fmax(s0, s1), cmin = fmin(c0, c1), cmax = fmax(c0, c1);
  if (lip_contains(tlo, thi, 0.5 * pi)) smax = 1.0;
  if (lip_contains(tlo, thi, -0.5 * pi)) smin = -1.0;
  if (lip_contains(tlo, thi, 0.0)) cmax = 1.0;
  if (lip_contains(tlo, thi, pi)) cmin = -1.0;
  sc = 0.5 * (smin + smax);
  sr = 0.5 * (smax - smin) + 1e-12;
  cc = 0.5 * (cmin + cmax);
  cr = 0.5 * (cmax - cmin) + 1e-12;
}

// sigmoid and softplus of z (fp64)
__device__ __forceinline__ void lip_act(double z, double& sg, double& sp) {
  const double e = exp(-fabs(z));
  const double inv = 1.0 / (1.0 + e);
  sg = z >= 0.0 ? inv : e * inv;
  sp = fmax(z, 0.0) + log1p(e);
}

// centre / radius of sigmoid and softplus over z in zc +- zr
__device__ __forceinline__ void lip_act_range(double zc, double zr, double& sgc, double& sgr, double& spc, double& spr) {
  double sl, su, hl, hu;
  lip_act(zc - zr, sl, hl);
  lip_act(zc + zr, su, hu);
  sgc = 0.5 * (sl + su);
  sgr = 0.5 * (su - sl) + 1e-13;
  spc = 0.5 * (hl + hu);
  spr = 0.5 * (hu - hl) * (1.0 + 1e-12) + 1e-13;
}

static __global__ void __launch_bounds__(32 * kLipWarps, 2) lip_bound_kernel(LipArgs A) {
  extern __shared__ __align__(16) unsigned char lip_smem_raw[];
  LipSmem& S = *reinterpret_cast<LipSmem*>(lip_smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cell = blockIdx.x;
  const float* blob = A.blobs + (size_t)cell * SdfBlob::floats;
  for (int i = tid; i < kSdfIn * kHidden; i += blockDim.x) S.w1t[i] = (double)blob[SdfBlob::w1 + i];
  for (int i = tid; i < kHidden * kHidden; i += blockDim.x) {
    const double w = (double)blob[SdfBlob::w2 + i];  // blob: [k = input n][j = output m]
    S.w2t[i] = w;
    S.w2r[(i & 31) * kHidden + (i >> 5)] = w;
  }
  if (tid < kHidden) {
    S.b1[tid] = (double)blob[SdfBlob::b1 + tid];
    S.b2[tid] = (double)blob[SdfBlob::b2 + tid];
    S.w3[tid] = (double)blob[SdfBlob::w3 + tid * kSdfOutPad];  // output 0 = the distance
  }
  __syncthreads();
  LipWarpScratch& W = S.ws[warp];
  const LipCellConst cc = A.cc[cell];
  const int N = A.G.resolution, k = A.k, fine = A.fine;
  const int ci[3] = {cell / (N * N), (cell / N) % N, cell % N};
  double elo[3], wsub[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const double ext = A.G.hi[a] - A.G.lo[a];
    const double lo = A.G.lo[a] + ext * (double)ci[a] / (double)N - A.margin;
    const double hi = A.G.lo[a] + ext * (double)(ci[a] + 1) / (double)N + A.margin;
    elo[a] = lo;
    wsub[a] = (hi - lo) / (double)k;
  }
  const double pi = 3.141592653589793238462643383279;
  const double w3l = S.w3[lane], aw3l = fabs(w3l);
  double best[3] = {0.0, 0.0, 0.0};
  bool bad = false;

  const int n_sub = k * k * k;
  for (int s = blockIdx.y * kLipWarps + warp; s < n_sub; s += gridDim.y * kLipWarps) {
    const int si[3] = {s / (k * k), (s / k) % k, s % k};
    // ---- 1. feature enclosures -----------------------------------------------------------------------------------
    if (lane < 18) {
      const int o = lane / 3, a = lane % 3;
      const double f = ldexp(pi, o);
      const double xlo = elo[a] + wsub[a] * (double)si[a], xhi = elo[a] + wsub[a] * (double)(si[a] + 1);
      double sc, sr, cc2, cr;
      lip_trig_range(f * xlo, f * xhi, sc, sr, cc2, cr);
      W.phi[3 + 6 * o + a] = make_double2(sc, sr);
      W.phi[6 + 6 * o + a] = make_double2(cc2, cr);
      if (lane < 3)  // the raw coordinate (a == lane)
        W.phi[lane] = make_double2(elo[lane] + wsub[lane] * ((double)si[lane] + 0.5), 0.5 * wsub[lane] * (1.0 + 1e-12) + 1e-13);
    } else if (lane < 18 + 3 * fine) {
      // Taylor sample points of g_a: sin / cos of 2^o pi x_i by one sincos and the double-angle recurrence
      const int q = lane - 18, a = q / fine, i = q % fine;
      const double x = elo[a] + wsub[a] * ((double)si[a] + ((double)i + 0.5) / (double)fine);
      double sn, cs;
      sincos(pi * x, &sn, &cs);
#pragma unroll
      for (int o = 0; o < kSdfFreqs; o++) {
        W.trig[q][2 * o] = sn;
        W.trig[q][2 * o + 1] = cs;
        const double s2 = 2.0 * sn * cs, c2 = fma(-2.0 * sn, sn, 1.0);
        sn = s2;
        cs = c2;
      }
    }
    __syncwarp();
    // ---- 2. layer 1 ------------------------------------------------------------------------------------------------
    double z1c = S.b1[lane], z1r = 0.0;
#pragma unroll 13
    for (int kk = 0; kk < kSdfIn; kk++) {
      const double w = S.w1t[kk * kHidden + lane];
      const double2 ph = W.phi[kk];
      z1c = fma(w, ph.x, z1c);
      z1r = fma(fabs(w), ph.y, z1r);
    }
    z1r = fma(1e-12, fabs(z1c) + z1r, z1r) + 1e-13;
    double c1, r1, h1c, h1r;
    lip_act_range(z1c, z1r, c1, r1, h1c, h1r);
    W.vab[lane] = make_double2(h1c, h1r);
    __syncwarp();
    // ---- layer 2 ---------------------------------------------------------------------------------------------------
    double z2c = S.b2[lane], z2r = 0.0;
#pragma unroll 8
    for (int n = 0; n < kHidden; n++) {
      const double w = S.w2t[n * kHidden + lane];
      const double2 hh = W.vab[n];
      z2c = fma(w, hh.x, z2c);
      z2r = fma(fabs(w), hh.y, z2r);
    }
    z2r = fma(1e-12, fabs(z2c) + z2r, z2r) + 1e-13;
    double c2, r2, h2c_unused, h2r_unused;
    lip_act_range(z2c, z2r, c2, r2, h2c_unused, h2r_unused);
    const double rw = r2 * aw3l;  // r2_m |w3_m|
    __syncwarp();
    W.vab[lane] = make_double2(c2 * w3l, rw);
    __syncwarp();
    double vt = 0.0, q = 0.0;  // v~_n = sum_m W2[m][n] c2_m w3_m ; q_n = sum_m |W2[m][n]| r2_m |w3_m|
#pragma unroll 8
    for (int m = 0; m < kHidden; m++) {
      const double w = S.w2r[m * kHidden + lane];
      const double2 uu = W.vab[m];
      vt = fma(w, uu.x, vt);
      q = fma(fabs(w), uu.y, q);
    }
    const double nrw = sqrt(lip_warp_sum(rw * rw));
    const double avt_r1 = fabs(vt) * r1;
    // ---- 3 + 4. Phi at the Taylor samples of every axis ---------------------------------------------------------------
#pragma unroll 1
    for (int a = 0; a < 3; a++) {
      const double h = 0.5 * wsub[a] / (double)fine;
      const double rem_a = 2.0 * cc.n3 * cc.n2 * (0.5 * h * h * cc.k3[a]);
      const double rem_b = (2.0 * cc.n3 * cc.n2 + cc.n3 * cc.n2f) * (0.5 * h * h * cc.k3[a]);
#pragma unroll 1
      for (int i = 0; i < fine; i++) {
        const double* tg = W.trig[a * fine + i];
        double g = S.w1t[a * kHidden + lane], gp = 0.0;
#pragma unroll
        for (int o = 0; o < kSdfFreqs; o++) {
          const double f = ldexp(pi, o);
          const double ws = S.w1t[(3 + 6 * o + a) * kHidden + lane], wc = S.w1t[(6 + 6 * o + a) * kHidden + lane];
          const double sn = tg[2 * o], cs = tg[2 * o + 1];
          g = fma(f, fma(cs, ws, -sn * wc), g);            // d/dx [ws sin(f x) + wc cos(f x)] = f (ws cos - wc sin)
          gp = fma(-f * f, fma(sn, ws, cs * wc), gp);      // d2/dx2 = -f^2 (ws sin + wc cos)
        }
        __syncwarp();
        const double cg = c1 * g, cgp = c1 * gp;
        W.vcd[lane] = make_double2(cg, cgp);
        __syncwarp();
        double u = 0.0, up = 0.0;  // (W2 (c1 o g))_m, lane = m
#pragma unroll 8
        for (int n = 0; n < kHidden; n++) {
          const double w = S.w2t[n * kHidden + lane];
          const double2 cc12 = W.vcd[n];
          u = fma(w, cc12.x, u);
          up = fma(w, cc12.y, up);
        }
        const double rg = r1 * fabs(g), rgp = r1 * fabs(gp);
        // lane-wise terms of the sums (the Taylor combination Phi(g) + h Phi(g') is formed before reducing where it is linear)
        const double s1 = lip_warp_sum(vt * cg);
        const double s1p = lip_warp_sum(vt * cgp);
        const double s23 = lip_warp_sum(fma(h, fma(rw, fabs(up), avt_r1 * fabs(gp)), fma(rw, fabs(u), avt_r1 * fabs(g))));
        const double s4 = lip_warp_sum(rg * rg);
        const double s4p = lip_warp_sum(rgp * rgp);
        const double s4b = lip_warp_sum(q * fma(h, rgp, rg));
        const double base = fabs(s1) + h * fabs(s1p) + s23;
        const double tot_a = base + nrw * cc.n2 * (sqrt(s4) + h * sqrt(s4p)) + rem_a;
        const double tot_b = base + s4b + rem_b;
        const double cand = fmin(tot_a, tot_b);
        bad = bad || !(cand == cand);  // fmax would drop a NaN silently: a sub-box without a bound must void the cell's refinement
        best[a] = fmax(best[a], cand);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      if (bad) best[a] = __longlong_as_double(0x7ff0000000000000ll);  // +inf: lip_store_kernel keeps the closed-form bound
      if (best[a] > 0.0) atomicMax(A.out + (size_t)cell * 3 + a, (unsigned long long)__double_as_longlong(best[a]));
    }
  }
}

// L_a <- min(closed-form bound already in the blobs, 1.001 x the sub-box maximum), written (rounded up to fp32) into the
// filter constants of both filter blob kinds and into `cur` (the accessor's copy).
static __global__ void lip_store_kernel(const unsigned long long* __restrict__ mx, int n_cells, float* __restrict__ cur,
                                        unsigned char* __restrict__ tc5_blobs, int tc5_stride, int tc5_off,
                                        uint32_t* __restrict__ mma_blobs, int mma_stride_words, int mma_off_words) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_cells * 3) return;
  const int cell = i / 3, a = i % 3;
  const double v = __longlong_as_double((long long)mx[i]);
  float l = cur[i];
  if (v > 0.0 && isfinite(v)) {
    const float t = __double2float_ru(fma(1.001, v, 1e-12));
    l = fminf(l, t);
  }
  cur[i] = l;
  if (tc5_blobs) reinterpret_cast<float*>(tc5_blobs + (size_t)cell * tc5_stride + tc5_off)[a] = l;
  if (mma_blobs) reinterpret_cast<float*>(mma_blobs + (size_t)cell * mma_stride_words + mma_off_words)[a] = l;
}

#endif  // KNF_BOUNDS_LAYOUT_ONLY

}  // namespace knf
