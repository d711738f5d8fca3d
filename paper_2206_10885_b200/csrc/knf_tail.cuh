// knf_tail.cuh -- the END of a march without global wavefronts: one warp per ray, to completion.
//
// Late in a march only stragglers are left (a few rays per cell, each with dozens of steps to go); every further global
// wavefront then costs a routing pass and two latency-bound tile launches for a handful of evaluations (measured: the
// last ~17 of 34 wavefronts of the 1080p frame hold < 2 % of its evaluations and take ~1.5 ms of its ~10).  Once the live
// rays drop below a threshold the engine hands ALL of them -- both queues -- to this kernel instead:
//
//   * a group of 8 lanes takes one ray and steps it until it is done (hit, miss, or out of steps), then claims the next: no
//     routing, no queues; the four groups of a warp evaluate in lock step and run their march steps side by side;
//   * lane q of a group owns hidden units 4 q .. 4 q + 3: each pre-activation is the k-ordered fp32 FMA chain from zero plus
//     the rounded bias add, NumPy's softplus bit for bit, and the distance is the k-ordered chain over the 32 hidden units --
//     the very arithmetic of the tile kernels (knf_mlp.cuh), so a sample's distance does not depend on which kernel
//     evaluated it and results stay bit-identical.  (Round 2 started with one ray per warp, lane = hidden unit: every
//     instruction served one evaluation -- ~900 warp instructions each, ten times the tile kernels' cost -- and the kernel
//     was issue-bound at 0.5 ms for 47 k rays; four rays per warp share every instruction of the evaluation);
//   * weights are read straight from the cell's k-major blob (a row of W^T is one coalesced 128-byte load per group;
//     consecutive steps of a ray stay in one cell, so the rows come from L1 / L2);
//   * crawling rays from the filter queue are evaluated exactly too (the filter only ever answered predicates), and CERTIFIED
//     SKIPPING works here as in the filter kernel, with the exact distance in place of the filter's: from a sample p0 with
//     d_exact(p0) < -(eps + delta) every further sample p of the ray in the same cell with sum_a L_a |p_a - p0_a| below
//     -(eps + delta) - d_exact(p0) has an exact distance below -eps (L_a: the cell's proven Lipschitz bounds,
//     knf_bounds.cuh; delta, the cell's filter bound, contains twice over the exact kernel's own distance to real
//     arithmetic, which is all that separates d_exact from the function the bounds are about), so the reference's crawl
//     steps there are taken without evaluating: closed-form run (cell-exit DDA + Lipschitz budget, J rounded fp64 additions
//     in O(1)) and then sample by sample -- the logic of march_tc5_kernel, one ray per warp.
#pragma once

#include "knf_common.cuh"
#include "knf_march.cuh"
#include "knf_mlp.cuh"
#include "knf_rays.cuh"

namespace knf {

struct MarchTailArgs {
  const float* blobs;        // SdfBlob per cell (the exact kernels' blobs)
  GridGeom G;
  MarchState M;
  double cell_scale[3];
  // the two pending queues: request slot -> (ray, point, cell)
  const int* live_a;
  const float4* pt_a;
  const int* cell_a;
  const RouteCounters* ctr_a;
  const int* live_b;
  const float4* pt_b;
  const int* cell_b;
  const RouteCounters* ctr_b;
  int* cursor;               // zero on entry: next unclaimed ray
  unsigned long long* eval_counter;
  // certified skipping: per-cell filter constants (delta, L_a) inside the decision-filter blobs; null disables it
  const unsigned char* fconst;
  int fconst_stride;         // bytes per cell
  int off_delta, off_lip;    // byte offsets of delta (1 float) and L_a (3 floats) inside a cell's blob
  int skip_cap;              // most certified steps taken sample by sample after one evaluation
  double inv_resolution;
};

// `m` certified crawl steps of the reference (surface.py:217-223 with max(d, eps / 2) = eps / 2) from the ray's current t:
// J = n rounded fp64 additions t <- fl(t + dt), taken in closed form inside one binade (see march_tc5_kernel), or one by one.
// Stops early at the first step that passes t_far or exhausts max_steps (returns true: the ray is done, a miss).
__device__ __forceinline__ bool crawl_run(RayRegs& R, const MarchState& M, int ray, int n, double dt, unsigned long long& skipped) {
  if (n <= 0) return false;
  const double t0 = R.t;
  const long long eb = __double_as_longlong(t0) & 0x7ff0000000000000ll;
  const double top = __longlong_as_double(eb + 0x0010000000000000ll);  // 2^(e+1)
  const double u = __longlong_as_double(eb - (52ll << 52));            // 2^(e-52)
  const double D = (t0 + dt) - t0;
  bool done = false;
  if (t0 > 0.0 && eb > (60ll << 52) && D > 0.0 && fabs(dt - D) * 2.0 != u && n < (1 << 20) && t0 + (double)(n + 2) * dt < top) {
    int m = n;
    const int m_steps = max(1, M.max_steps - R.steps);
    if (m_steps <= m) { m = m_steps; done = true; }
    if (t0 + (double)m * D > R.t_far) {
      int mf = (int)fmin(floor((R.t_far - t0) / D), 2.0e6) + 1;
      mf = max(1, min(mf, m));
      while (mf > 1 && t0 + (double)(mf - 1) * D > R.t_far) mf--;
      while (mf < m && !(t0 + (double)mf * D > R.t_far)) mf++;
      m = mf;
      done = true;
    }
    R.steps += m;
    R.t_prev = t0 + (double)(m - 1) * D;
    R.t = t0 + (double)m * D;
    skipped += (unsigned long long)m;
  } else {
    for (int j = 0; j < n && !done; j++) {
      R.steps += 1;
      R.t_prev = R.t;
      R.t = R.t + dt;
      skipped += 1;
      done = R.t > R.t_far || R.steps >= M.max_steps;
    }
  }
  if (done) {
    M.phase[ray] = PH_DONE;
    M.steps[ray] = R.steps;
  }
  return done;
}

constexpr int kTailGroup = 8;   // lanes per ray
constexpr int kTailUnits = kHidden / kTailGroup;  // hidden units per lane
static_assert(kTailUnits == 4, "tail_eval is written for four hidden units per lane (float4 weight rows)");

// exact SDF distance at (x, y, z) in the cell whose blob is `blob`: the 8 lanes [gbase, gbase + 8) call it with the same
// point and all get the same value; the four groups of a warp call it together (the shuffles are warp-wide)
__device__ __forceinline__ float tail_eval(const float* __restrict__ blob, int q, int gbase, float x, float y, float z) {
  using Blob = SdfBlob;
  const float pi_f = 3.14159274101257324e+00f;  // float32(np.pi)
  // nn.fourier_encode, operation for operation (every lane computes the 39 features of its group's point)
  float f[kSdfIn];
  f[0] = x; f[1] = y; f[2] = z;
  float s[3], c[3];
  np_sincosf(__fmul_rn(pi_f, x), s[0], c[0]);
  np_sincosf(__fmul_rn(pi_f, y), s[1], c[1]);
  np_sincosf(__fmul_rn(pi_f, z), s[2], c[2]);
#pragma unroll
  for (int o = 0; o < kSdfFreqs; o++) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      f[3 + 6 * o + a] = s[a];
      f[3 + 6 * o + 3 + a] = c[a];
      const float two_s = __fmul_rn(2.0f, s[a]);
      const float ns = __fmul_rn(two_s, c[a]);
      c[a] = __fsub_rn(1.0f, __fmul_rn(two_s, s[a]));
      s[a] = ns;
    }
  }
  // layer 1: acc_j = fma(x_k, W1[j][k], acc_j), k ascending, from zero, for the lane's units j = 4 q + u; then the rounded bias add
  const float4* w1 = reinterpret_cast<const float4*>(blob + Blob::w1) + q;  // row k of W1^T: 32 floats = 8 float4, the lane's is number q
  float acc[kTailUnits] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < kSdfIn; k++) {
    const float4 w = __ldg(w1 + k * (kHidden / 4));
    acc[0] = __fmaf_rn(f[k], w.x, acc[0]);
    acc[1] = __fmaf_rn(f[k], w.y, acc[1]);
    acc[2] = __fmaf_rn(f[k], w.z, acc[2]);
    acc[3] = __fmaf_rn(f[k], w.w, acc[3]);
  }
  float4 b = __ldg(reinterpret_cast<const float4*>(blob + Blob::b1) + q);
  float2 h[2] = {make_float2(__fadd_rn(acc[0], b.x), __fadd_rn(acc[1], b.y)), make_float2(__fadd_rn(acc[2], b.z), __fadd_rn(acc[3], b.w))};
  softplus_np_f2xN<2>(h);
  const float h1[kTailUnits] = {h[0].x, h[0].y, h[1].x, h[1].y};
  // layer 2: h1[k] comes from lane k / 4 of the group, component k % 4
  const float4* w2 = reinterpret_cast<const float4*>(blob + Blob::w2) + q;
  acc[0] = acc[1] = acc[2] = acc[3] = 0.0f;
#pragma unroll
  for (int sl = 0; sl < kTailGroup; sl++)
#pragma unroll
    for (int u = 0; u < kTailUnits; u++) {
      const float hv = __shfl_sync(0xffffffffu, h1[u], gbase + sl);
      const float4 w = __ldg(w2 + (kTailUnits * sl + u) * (kHidden / 4));
      acc[0] = __fmaf_rn(hv, w.x, acc[0]);
      acc[1] = __fmaf_rn(hv, w.y, acc[1]);
      acc[2] = __fmaf_rn(hv, w.z, acc[2]);
      acc[3] = __fmaf_rn(hv, w.w, acc[3]);
    }
  b = __ldg(reinterpret_cast<const float4*>(blob + Blob::b2) + q);
  h[0] = make_float2(__fadd_rn(acc[0], b.x), __fadd_rn(acc[1], b.y));
  h[1] = make_float2(__fadd_rn(acc[2], b.z), __fadd_rn(acc[3], b.w));
  softplus_np_f2xN<2>(h);
  const float h2[kTailUnits] = {h[0].x, h[0].y, h[1].x, h[1].y};
  // output 0: the distance, the k-ordered chain over the 32 hidden units (every lane of the group runs it)
  const float* w3 = blob + Blob::w3;
  float d = 0.0f;
#pragma unroll
  for (int sl = 0; sl < kTailGroup; sl++)
#pragma unroll
    for (int u = 0; u < kTailUnits; u++) {
      const float hv = __shfl_sync(0xffffffffu, h2[u], gbase + sl);
      d = __fmaf_rn(hv, __ldg(w3 + (kTailUnits * sl + u) * kSdfOutPad), d);
    }
  return __fadd_rn(d, __ldg(blob + Blob::b3));
}

#ifndef KNF_TAIL_MIN_BLOCKS
#define KNF_TAIL_MIN_BLOCKS 3
#endif
constexpr int kTailWarps = 4;
static __global__ void __launch_bounds__(32 * kTailWarps, KNF_TAIL_MIN_BLOCKS) march_tail_kernel(MarchTailArgs A) {
  const int lane = threadIdx.x & 31, q = lane & (kTailGroup - 1), gbase = lane & ~(kTailGroup - 1);
  const int n_a = A.ctr_a->n_requests, n_b = A.ctr_b ? A.ctr_b->n_requests : 0;
  const double dt = A.M.step_scale * (A.M.eps / 2);
  unsigned long long evals = 0, skipped = 0, rays_done = 0;  // per group (counted in its lane 0)
  bool have = false, exhausted = false;  // the group holds a live ray / the queue has run dry
  int ray = 0, cell = 0;
  float4 pt = make_float4(0.f, 0.f, 0.f, 0.f);
  RayRegs rr;
  for (;;) {
    // ---- groups without a ray claim the next one --------------------------------------------------------------------
    int i = -1;
    if (!have && !exhausted && q == 0) i = atomicAdd(A.cursor, 1);
    i = __shfl_sync(0xffffffffu, i, gbase);
    if (!have && !exhausted) {
      if (i < n_a + n_b) {
        const bool from_a = i < n_a;
        const int slot = from_a ? i : i - n_a;
        ray = (from_a ? A.live_a : A.live_b)[slot];
        pt = (from_a ? A.pt_a : A.pt_b)[slot];
        cell = (from_a ? A.cell_a : A.cell_b)[slot];
        ray_load(rr, A.M, ray);
        rays_done += 1;
        have = true;
      } else {
        exhausted = true;
      }
    }
    if (!__any_sync(0xffffffffu, have)) break;
    // ---- one exact evaluation per group, in lock step (a group without a ray evaluates cell 0 at the origin: finite, ignored)
    const float d = tail_eval(A.blobs + (size_t)(have ? cell : 0) * SdfBlob::floats, q, gbase, have ? pt.x : 0.f, have ? pt.y : 0.f,
                              have ? pt.z : 0.f);
    if (have) {
      evals += 1;
      double t_next = 0.0;
      double safe_below = -INFINITY;
      const float* fc = nullptr;
      if (A.fconst) {
        fc = reinterpret_cast<const float*>(A.fconst + (size_t)cell * A.fconst_stride);
        safe_below = -(A.M.eps + (double)__ldg(fc + A.off_delta / 4));  // delta = +inf (filter off for the cell): never below
      }
      // every lane of the group steps its copy of the ray: same writes, same values
      const int code = ray_step(rr, A.M, ray, d, t_next, safe_below);
      bool done = code == STEP_DONE, known_cell = false;
      if (code == STEP_FILTER) {
        // ---- certified skipping from p0 = pt, d_exact(p0) = d < -(eps + delta): the logic of march_tc5_kernel ---------------
        const float lip[3] = {__ldg(fc + A.off_lip / 4), __ldg(fc + A.off_lip / 4 + 1), __ldg(fc + A.off_lip / 4 + 2)};
        const int N = A.G.resolution;
        const int ci[3] = {cell / (N * N), (cell / N) % N, cell % N};
        const float p0[3] = {pt.x, pt.y, pt.z};
        float in_lo[3], in_hi[3];
        bool p0_in = true;
#pragma unroll
        for (int a = 0; a < 3; a++) {
          const double ext = A.G.hi[a] - A.G.lo[a];
          in_lo[a] = (float)(A.G.lo[a] + ext * ((double)ci[a] * A.inv_resolution) + 1e-6 * ext);
          in_hi[a] = (float)(A.G.lo[a] + ext * ((double)(ci[a] + 1) * A.inv_resolution) - 1e-6 * ext);
          const float pad = (float)((1e-6 + (double)kLipSlack * A.inv_resolution) * ext);
          p0_in = p0_in && p0[a] >= in_lo[a] - pad && p0[a] <= in_hi[a] + pad;
        }
        const float room = p0_in ? __fmul_rd(__fsub_rd(__double2float_rd(safe_below), d), 0.99999f) : 0.0f;
        const unsigned long long skipped_before = skipped;
        if (room > 0.0f) {
          // part 1: closed-form run (per axis |p_j - p0| <= j dt |d_a| (1 + 2^-20) + two fp32 roundings; 2 samples short of
          // the cell exit and of the Lipschitz budget, scaled by 0.999 against the fp32 arithmetic here)
          const float dtf = __double2float_ru(dt);
          float run = 1.0e9f, rise_per_step = 0.0f, lip_sum = 0.0f;
#pragma unroll
          for (int a = 0; a < 3; a++) {
            const float ad = __double2float_ru(fabs(rr.d[a])) * 1.000002f;
            const float gap = rr.d[a] > 0.0 ? in_hi[a] - p0[a] : p0[a] - in_lo[a];
            const float stepa = ad * dtf;
            if (stepa > 0.0f) run = fminf(run, __fdividef(fmaxf(gap, 0.0f), stepa));
            rise_per_step += lip[a] * stepa;
            lip_sum += lip[a];
          }
          const float budget = room - 1.0e-6f * lip_sum;
          if (rise_per_step > 0.0f) run = fminf(run, budget > 0.0f ? __fdividef(budget, rise_per_step) : 0.0f);
          const int J = (int)fminf(run * 0.999f, 1.0e6f) - 2;
          done = crawl_run(rr, A.M, ray, J, dt, skipped);
          t_next = rr.t;
        }
        // part 2: the remaining samples, one by one (exact point, exact box test, exact rise)
        for (int it = 0; !done; it++) {
          pt.x = __double2float_rn(rr.o[0] + t_next * rr.d[0]);
          pt.y = __double2float_rn(rr.o[1] + t_next * rr.d[1]);
          pt.z = __double2float_rn(rr.o[2] + t_next * rr.d[2]);
          known_cell = pt.x > in_lo[0] && pt.x < in_hi[0] && pt.y > in_lo[1] && pt.y < in_hi[1] && pt.z > in_lo[2] && pt.z < in_hi[2];
          if (!known_cell || it >= A.skip_cap) break;
          const float rise = lip[0] * (fabsf(pt.x - p0[0]) + 1e-6f) + lip[1] * (fabsf(pt.y - p0[1]) + 1e-6f) + lip[2] * (fabsf(pt.z - p0[2]) + 1e-6f);
          if (!(rise < room)) break;
          done = crawl_run(rr, A.M, ray, 1, dt, skipped);
          t_next = rr.t;
        }
        // t_prev moved past samples nobody evaluated: d_prev (exact, at p0) is now only good as a predicate, and a ray that
        // converges next re-evaluates it at t_prev first (PH_RECHECK), as after filtered steps
        if (skipped != skipped_before) rr.approx = 1;
      } else if (!done) {
        pt.x = __double2float_rn(rr.o[0] + t_next * rr.d[0]);
        pt.y = __double2float_rn(rr.o[1] + t_next * rr.d[1]);
        pt.z = __double2float_rn(rr.o[2] + t_next * rr.d[2]);
      }
      if (done) have = false;
      else if (!known_cell) cell = cell_of_quick(pt.x, pt.y, pt.z, A.G.lo, A.G.hi, A.cell_scale, A.G.resolution);
    }
    __syncwarp();
  }
  if (A.eval_counter) {
    if (q != 0) evals = skipped = rays_done = 0;  // one count per group
#pragma unroll
    for (int off = 16; off >= kTailGroup; off >>= 1) {
      evals += __shfl_xor_sync(0xffffffffu, evals, off);
      skipped += __shfl_xor_sync(0xffffffffu, skipped, off);
      rays_done += __shfl_xor_sync(0xffffffffu, rays_done, off);
    }
    if (lane == 0 && evals) {
      atomicAdd(A.eval_counter, evals);
      atomicAdd(A.eval_counter + 8, evals);  // diagnostics (KNF_DEBUG_TAIL): the tail's own evaluations and rays
      atomicAdd(A.eval_counter + 9, rays_done);
      if (skipped) atomicAdd(A.eval_counter + 6, skipped);  // certified steps (same counter as the filter kernel's)
    }
  }
}

}  // namespace knf
