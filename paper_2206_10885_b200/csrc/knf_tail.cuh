// knf_tail.cuh -- the END of a march without global wavefronts: one warp per ray, to completion.
//
// Late in a march only stragglers are left (a few rays per cell, each with dozens of steps to go); every further global
// wavefront then costs a routing pass and two latency-bound tile launches for a handful of evaluations (measured: the
// last ~17 of 34 wavefronts of the 1080p frame hold < 2 % of its evaluations and take ~1.5 ms of its ~10).  Once the live
// rays drop below a threshold the engine hands ALL of them -- both queues -- to this kernel instead:
//
//   * a warp takes one ray and steps it until it is done (hit, miss, or out of steps): no routing, no queues;
//   * lane j owns hidden unit j: its layer-1 / layer-2 pre-activation is the k-ordered fp32 FMA chain from zero plus the
//     rounded bias add, NumPy's softplus bit for bit, and the distance is the k-ordered chain over the 32 hidden units --
//     the very arithmetic of the tile kernels (knf_mlp.cuh), so a sample's distance does not depend on which kernel
//     evaluated it and results stay bit-identical;
//   * weights are read straight from the cell's k-major blob (a row of W^T is one coalesced 128-byte load; consecutive
//     steps of a ray stay in one cell, so the rows come from L1 / L2);
//   * crawling rays from the filter queue are simply evaluated exactly (the filter only ever answered predicates).
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
};

// exact SDF distance at (x, y, z) in `cell`; all 32 lanes call it with the same point, all get the same value
__device__ __forceinline__ float tail_eval(const float* __restrict__ blob, int lane, float x, float y, float z) {
  using Blob = SdfBlob;
  const float pi_f = 3.14159274101257324e+00f;  // float32(np.pi)
  // nn.fourier_encode, operation for operation (every lane computes the 39 features of the shared point)
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
  // layer 1: lane = hidden unit; acc = fma(x_k, W1[j][k], acc), k ascending, from zero; then the rounded bias add
  const float* w1 = blob + Blob::w1 + lane;
  float acc = 0.0f;
#pragma unroll
  for (int k = 0; k < kSdfIn; k++) acc = __fmaf_rn(f[k], __ldg(w1 + k * kHidden), acc);
  float2 h = softplus_np_f2(splat(__fadd_rn(acc, __ldg(blob + Blob::b1 + lane))));
  const float h1 = h.x;
  // layer 2: h1[k] comes from lane k
  const float* w2 = blob + Blob::w2 + lane;
  acc = 0.0f;
#pragma unroll
  for (int k = 0; k < kHidden; k++) acc = __fmaf_rn(__shfl_sync(0xffffffffu, h1, k), __ldg(w2 + k * kHidden), acc);
  h = softplus_np_f2(splat(__fadd_rn(acc, __ldg(blob + Blob::b2 + lane))));
  const float h2 = h.x;
  // output 0: the distance
  const float* w3 = blob + Blob::w3;
  acc = 0.0f;
#pragma unroll
  for (int k = 0; k < kHidden; k++) acc = __fmaf_rn(__shfl_sync(0xffffffffu, h2, k), __ldg(w3 + k * kSdfOutPad), acc);
  return __fadd_rn(acc, __ldg(blob + Blob::b3));
}

constexpr int kTailWarps = 4;
static __global__ void __launch_bounds__(32 * kTailWarps) march_tail_kernel(MarchTailArgs A) {
  const int lane = threadIdx.x & 31;
  const int n_a = A.ctr_a->n_requests, n_b = A.ctr_b ? A.ctr_b->n_requests : 0;
  unsigned long long evals = 0;
  for (;;) {
    int i = 0;
    if (lane == 0) i = atomicAdd(A.cursor, 1);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= n_a + n_b) break;
    const bool from_a = i < n_a;
    const int slot = from_a ? i : i - n_a;
    const int ray = (from_a ? A.live_a : A.live_b)[slot];
    float4 pt = (from_a ? A.pt_a : A.pt_b)[slot];
    int cell = (from_a ? A.cell_a : A.cell_b)[slot];
    RayRegs rr;
    ray_load(rr, A.M, ray);
    for (;;) {
      const float d = tail_eval(A.blobs + (size_t)cell * SdfBlob::floats, lane, pt.x, pt.y, pt.z);
      evals += 1;
      double t_next = 0.0;
      const int code = ray_step(rr, A.M, ray, d, t_next, -INFINITY);  // every lane steps its copy of the ray: same writes, same values
      if (code == STEP_DONE) break;
      // pts = origins + t * dirs in fp64 (surface.py:184), then the fp32 cast of grid.py:375
      pt.x = __double2float_rn(rr.o[0] + t_next * rr.d[0]);
      pt.y = __double2float_rn(rr.o[1] + t_next * rr.d[1]);
      pt.z = __double2float_rn(rr.o[2] + t_next * rr.d[2]);
      cell = cell_of_quick(pt.x, pt.y, pt.z, A.G.lo, A.G.hi, A.cell_scale, A.G.resolution);
    }
  }
  if (lane == 0 && evals && A.eval_counter) atomicAdd(A.eval_counter, evals);
}

}  // namespace knf
