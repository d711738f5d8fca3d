// knf_rays.cuh -- ray generation, ray/AABB slabs, the wavefront sphere-trace step with secant
// refinement, FD-normal shading and the frame composite (north_star subsystems 1, 3, 4;
// SURVEY K1, K5, K6).  All ray state is fp64 exactly as in the reference; only the point handed
// to the MLP is rounded to fp32 (grid.py:375) and its cell is computed in fp64 from that fp32
// point (grid.py:176-179).  The library is compiled with -fmad=false, so every a*b+c below is two
// roundings like NumPy's; the FMA chains written out with fma() are where NumPy goes through
// dgemm (verified bit-exact against numpy in the build container).
#pragma once

#include "knf_common.cuh"
#include "knf_route.cuh"

namespace knf {

// 3-vector times 3x3 the way `v @ M` (dgemm) evaluates it: k-ordered FMA chain from zero.
// m is row-major; out_i = sum_k v_k * m[k][i]   (v @ M)
__device__ __forceinline__ void vec_mat(const double v[3], const double* m, double out[3]) {
#pragma unroll
  for (int i = 0; i < 3; i++) out[i] = fma(v[2], m[6 + i], fma(v[1], m[3 + i], fma(v[0], m[i], 0.0)));
}
// out_i = sum_k v_k * m[i][k]   (v @ M^T)
__device__ __forceinline__ void vec_matT(const double v[3], const double* m, double out[3]) {
#pragma unroll
  for (int i = 0; i < 3; i++) out[i] = fma(v[2], m[3 * i + 2], fma(v[1], m[3 * i + 1], fma(v[0], m[3 * i], 0.0)));
}
// np.linalg.norm(axis=1) on 3-vectors: sqrt((x^2 + y^2) + z^2)
__device__ __forceinline__ double norm3(const double v[3]) { return sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]); }

struct CameraDev {
  double pos[3];
  double rot[9];
  double scale;  // 2 tan(fov_y / 2) / H, computed on the host in fp64
  int width;
  int height;
};

// cameras.pixel_rays (cameras.py:57-76) for one pixel.
__device__ __forceinline__ void pixel_ray(const CameraDev& c, double col, double row, double offx, double offy,
                                          double dir[3]) {
  double px = (col + offx - c.width / 2.0) * c.scale;
  double py = (c.height / 2.0 - row - offy) * c.scale;
  double local[3] = {px, py, -1.0};
  vec_matT(local, c.rot, dir);
  double len = norm3(dir);
  dir[0] /= len;
  dir[1] /= len;
  dir[2] /= len;
}

// surface.ray_aabb_batch (surface.py:131-149) for one ray.
__device__ __forceinline__ bool slab(const double o[3], const double d[3], const double lo[3], const double hi[3],
                                     double& t_near, double& t_far) {
  double enter = -INFINITY, leave = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double e, l;
    if (d[a] == 0.0) {
      bool inside = (o[a] >= lo[a]) && (o[a] <= hi[a]);
      e = inside ? -INFINITY : INFINITY;
      l = inside ? INFINITY : -INFINITY;
    } else {
      double inv = 1.0 / d[a];
      double ta = (lo[a] - o[a]) * inv;
      double tb = (hi[a] - o[a]) * inv;
      e = fmin(ta, tb);
      l = fmax(ta, tb);
    }
    enter = fmax(enter, e);
    leave = fmin(leave, l);
  }
  t_near = fmax(enter, 0.0);
  t_far = leave;
  return (leave >= enter) && (leave >= 0.0);
}

static __global__ void pixel_rays_kernel(CameraDev cam, const int* __restrict__ pixel_xy, const double* __restrict__ jitter,
                                  long long n, double* __restrict__ origins, double* __restrict__ dirs) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double col, row;
    if (pixel_xy) {
      col = pixel_xy[2 * i];
      row = pixel_xy[2 * i + 1];
    } else {
      col = (double)(i % cam.width);
      row = (double)(i / cam.width);
    }
    double ox = jitter ? jitter[2 * i] : 0.5, oy = jitter ? jitter[2 * i + 1] : 0.5;
    double d[3];
    pixel_ray(cam, col, row, ox, oy, d);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      origins[3 * i + a] = cam.pos[a];
      dirs[3 * i + a] = d[a];
    }
  }
}

static __global__ void ray_aabb_kernel(const double* __restrict__ o, const double* __restrict__ d, long long n, GridGeom box,
                                double* __restrict__ t_near, double* __restrict__ t_far, unsigned char* __restrict__ hit,
                                int trace_convention) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
    double dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
    double tn, tf;
    bool h = slab(oo, dd, box.lo, box.hi, tn, tf);
    if (trace_convention && !h) {  // surface.py:231-232: a missed box can never become active
      tn = 1.0;
      tf = 0.0;
    }
    t_near[i] = tn;
    t_far[i] = tf;
    if (hit) hit[i] = h;
  }
}

// Primary rays of rows [row0,row1) of a (W*ss x H*ss) raster + box test, fused (K1).
static __global__ void primary_rays_kernel(CameraDev cam, GridGeom box, int sub_row0, long long n, double* __restrict__ origins,
                                    double* __restrict__ dirs, double* __restrict__ t_near, double* __restrict__ t_far) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double col = (double)(i % cam.width);
    double row = (double)(sub_row0 + i / cam.width);
    double d[3];
    pixel_ray(cam, col, row, 0.5, 0.5, d);
    double tn, tf;
    if (!slab(cam.pos, d, box.lo, box.hi, tn, tf)) {
      tn = 1.0;
      tf = 0.0;
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
      origins[3 * i + a] = cam.pos[a];
      dirs[3 * i + a] = d[a];
    }
    t_near[i] = tn;
    t_far[i] = tf;
  }
}

// ---- wavefront march (surface.march_rays, surface.py:162-226) ---------------------------------
// PH_RECHECK: the ray converged while its d_prev came from the low-precision decision filter; the exact distance
// at t_prev is being fetched before the secant step (surface.py:190-195) may use it.
enum : unsigned char { PH_MARCH = 0, PH_REFINE = 1, PH_DONE = 2, PH_RECHECK = 3 };
constexpr unsigned char kPhaseMask = 3, kApproxPrevBit = 0x80;  // stored phase byte: phase | (d_prev is approximate ? 0x80 : 0)
// What a step asks for next.
enum { STEP_DONE = 0, STEP_EXACT = 1, STEP_FILTER = 2 };

struct MarchState {
  const double* o;   // (n,3)
  const double* d;   // (n,3)
  const double* t_far;
  double* t;         // current parameter (or the secant candidate while PH_REFINE)
  double* t_prev;
  double* d_prev;
  double* t_conv;    // t at convergence (PH_REFINE only)
  double* d_conv;    // d at convergence
  double* t_hit;
  int* steps;
  unsigned char* phase;
  unsigned char* hit;
  int* live[4];      // request slot -> ray id: [queue * 2 + wavefront parity], queue 0 = exact, 1 = decision filter
  double eps;
  double step_scale;
  int max_steps;
};

__device__ __forceinline__ void emit_at(const RouteBuffers& R, const GridGeom& G, const MarchState& M, int* live_out,
                                        bool want, int ray, double t) {
  int slot = warp_append(&R.ctr->n_requests, want);
  float x = 0.f, y = 0.f, z = 0.f;
  if (want) {
    // pts = origins + t * dirs in fp64 (surface.py:184), then the fp32 cast of grid.py:375
    x = __double2float_rn(M.o[3 * (size_t)ray + 0] + t * M.d[3 * (size_t)ray + 0]);
    y = __double2float_rn(M.o[3 * (size_t)ray + 1] + t * M.d[3 * (size_t)ray + 1]);
    z = __double2float_rn(M.o[3 * (size_t)ray + 2] + t * M.d[3 * (size_t)ray + 2]);
    live_out[slot] = ray;
  }
  route_emit(R, G, want, slot, x, y, z);
}

// First samples go to queue R (its live list: live_out); with `exact_eighths` > 0 that many of every 8 consecutive 32-ray blocks
// go to the second queue R2 / live_out2 instead (the exact queue when R is the filter queue: both kernels of wavefront 0 then
// have work, instead of the filter evaluating every first sample alone and handing three quarters of them on undecided).
static __global__ void march_init_kernel(RouteBuffers R, GridGeom G, MarchState M, const double* __restrict__ t_near, int n, int* __restrict__ live_out,
                                         RouteBuffers R2, int* __restrict__ live_out2, int exact_eighths) {
  int stride = gridDim.x * blockDim.x;
  int n_round = (n + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    bool want = false;
    double t0 = 0.0;
    if (i < n) {
      t0 = t_near[i];
      want = t0 < M.t_far[i];
      M.t[i] = t0;
      M.t_prev[i] = NAN;
      M.d_prev[i] = NAN;
      M.t_hit[i] = 0.0;
      M.steps[i] = 0;
      M.hit[i] = 0;
      M.phase[i] = want ? PH_MARCH : PH_DONE;
    }
    const bool second = exact_eighths > 0 && ((i >> 5) & 7) < exact_eighths;  // warp-uniform: i >> 5 is the same for the whole warp
    if (exact_eighths > 0 && second) emit_at(R2, G, M, live_out2, want, i, t0);
    else emit_at(R, G, M, live_out, want, i, t0);
  }
}

// A ray's marching state held in registers while it is resident in a tile.
struct RayRegs {
  double o[3], d[3];
  double t, t_far, t_prev, d_prev;
  int steps;
  int phase;
  int approx;  // d_prev was produced by the decision filter (knf_march.cuh) and is only good as a predicate
};
__device__ __forceinline__ void ray_load(RayRegs& R, const MarchState& M, int ray) {
  const size_t r3 = 3 * (size_t)ray;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    R.o[a] = M.o[r3 + a];
    R.d[a] = M.d[r3 + a];
  }
  R.t = M.t[ray];
  R.t_far = M.t_far[ray];
  R.t_prev = M.t_prev[ray];
  R.d_prev = M.d_prev[ray];
  R.steps = M.steps[ray];
  const int ph = M.phase[ray];
  R.phase = ph & kPhaseMask;
  R.approx = (ph & kApproxPrevBit) ? 1 : 0;
}
// The same without origin / direction (kernels that park those in shared memory with cp.async).
__device__ __forceinline__ void ray_load_scalars(RayRegs& R, const MarchState& M, int ray) {
  R.t = M.t[ray];
  R.t_far = M.t_far[ray];
  R.t_prev = M.t_prev[ray];
  R.d_prev = M.d_prev[ray];
  R.steps = M.steps[ray];
  const int ph = M.phase[ray];
  R.phase = ph & kPhaseMask;
  R.approx = (ph & kApproxPrevBit) ? 1 : 0;
}
// Write back what a later tile visit (or the finish kernel) needs.
__device__ __forceinline__ void ray_store(const RayRegs& R, const MarchState& M, int ray) {
  M.t[ray] = R.t;
  M.t_prev[ray] = R.t_prev;
  M.d_prev[ray] = R.d_prev;
  M.steps[ray] = R.steps;
  M.phase[ray] = (unsigned char)(R.phase | (R.approx ? kApproxPrevBit : 0));
}

// IEEE fp64 division out of line: the inlined sequence (~50 instructions with its slow path) sat in every copy of the step.
static __device__ __noinline__ double div_f64(double a, double b) { return a / b; }

// One sphere-trace step of one ray (the body of the reference loop, surface.py:185-223) given the EXACT fp32
// distance `dval` the MLP produced at the ray's requested parameter.  Returns STEP_DONE when the ray is finished
// (its result has been written to global memory), otherwise the ray needs another evaluation at t_next:
// STEP_EXACT, or STEP_FILTER when the ray just took a march step from a distance below `crawl_below` -- it is
// inside the negative region, where the reference only asks "is d still < -eps?" (decision filter, knf_march.cuh).
__device__ __forceinline__ int ray_step(RayRegs& R, const MarchState& M, int ray, float dval, double& t_next, double crawl_below) {
  double dv = (double)dval;
  double t = R.t;
  if (R.phase == PH_REFINE) {
    // surface.py:203-206: keep the secant point unless it is farther from the surface
    M.t_hit[ray] = (fabs(dv) > fabs(M.d_conv[ray])) ? M.t_conv[ray] : t;
    M.hit[ray] = 1;
    M.phase[ray] = PH_DONE;
    M.steps[ray] = R.steps;
    return STEP_DONE;
  }
  bool converged;
  if (R.phase == PH_RECHECK) {
    // dval is the exact distance at t_prev; resume the convergence branch with the stored (t, d)
    R.d_prev = dv;
    R.approx = 0;
    t = M.t_conv[ray];
    dv = M.d_conv[ray];
    converged = true;
  } else {
    R.steps += 1;
    converged = fabs(dv) <= M.eps;
    if (converged && R.approx && isfinite(R.t_prev)) {
      M.t_conv[ray] = t;
      M.d_conv[ray] = dv;
      R.phase = PH_RECHECK;
      t_next = R.t_prev;
      return STEP_EXACT;
    }
  }
  if (converged) {
    const double tp = R.t_prev, dp = R.d_prev;
    if (isfinite(tp) && (fabs(dv - dp) > 1e-12)) {
      double root = t - div_f64(dv * (t - tp), dv - dp);
      const double a = fmin(t, tp), b = fmax(t, tp);
      root = fmin(fmax(root, a), b + (b - a));  // np.clip(root, a, b + (b - a))
      M.t_conv[ray] = t;
      M.d_conv[ray] = dv;
      R.t = root;
      R.phase = PH_REFINE;
      t_next = root;
      return STEP_EXACT;
    }
    M.t_hit[ray] = t;
    M.hit[ray] = 1;
    M.phase[ray] = PH_DONE;
    M.steps[ray] = R.steps;
    return STEP_DONE;
  }
  R.t_prev = t;
  R.d_prev = dv;
  R.approx = 0;
  const double tn = t + M.step_scale * fmax(dv, M.eps / 2);
  R.t = tn;
  if (tn > R.t_far || R.steps >= M.max_steps) {
    M.phase[ray] = PH_DONE;  // left the box, or the step budget is spent: a miss
    M.steps[ray] = R.steps;
    return STEP_DONE;
  }
  t_next = tn;
  return dv < crawl_below ? STEP_FILTER : STEP_EXACT;
}

// The same step driven by an APPROXIMATE distance d_f with |d_f - d_exact| < delta (decision filter).  Only a
// PH_MARCH ray in the negative region comes here.  If d_f < -(eps + delta) the exact distance is certainly below
// -eps: the reference neither converges nor uses the value (max(d, eps/2) = eps/2), so the step is taken with the
// reference's own arithmetic and d_f is remembered as a predicate-only d_prev.  Otherwise nothing is changed and
// the caller re-queues the same sample for the exact kernel (STEP_EXACT, t_next = t).
__device__ __forceinline__ int ray_filter_step(RayRegs& R, const MarchState& M, int ray, float d_f, double safe_below, double& t_next,
                                               bool trusted = true) {
  const double dv = (double)d_f;
  // Undecided: not provably below -eps; NaN; -inf (a hidden activation left the fp16 range: the bound delta says
  // nothing about such a value); or a sample the bound was not derived for (`trusted` false: outside the box).
  if (!(dv < safe_below) || !(dv >= -3.0e38) || !trusted) {
    t_next = R.t;
    return STEP_EXACT;
  }
  R.steps += 1;
  R.t_prev = R.t;
  R.d_prev = dv;
  R.approx = 1;
  const double tn = R.t + M.step_scale * fmax(dv, M.eps / 2);
  R.t = tn;
  if (tn > R.t_far || R.steps >= M.max_steps) {
    M.phase[ray] = PH_DONE;
    M.steps[ray] = R.steps;
    return STEP_DONE;
  }
  t_next = tn;
  return STEP_FILTER;
}

// Write the TraceResult arrays (surface.py:225-226) and, optionally, compact the hit rays.
static __global__ void march_finish_kernel(MarchState M, int n, unsigned char* __restrict__ hit_out, double* __restrict__ t_out,
                                    double* __restrict__ pos_out, int* __restrict__ steps_out, int* __restrict__ hit_list,
                                    int* __restrict__ hit_count) {
  int stride = gridDim.x * blockDim.x;
  int n_round = (n + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    bool h = false;
    if (i < n) {
      h = M.hit[i] != 0;
      double th = M.t_hit[i];
      if (hit_out) hit_out[i] = h;
      if (t_out) t_out[i] = th;
      if (steps_out) steps_out[i] = M.steps[i];
      if (pos_out) {
#pragma unroll
        for (int a = 0; a < 3; a++) pos_out[3 * (size_t)i + a] = M.o[3 * (size_t)i + a] + th * M.d[3 * (size_t)i + a];
      }
    }
    if (hit_list) {
      int k = warp_append(hit_count, h);
      if (h) hit_list[k] = i;
    }
  }
}

// ---- shading (FieldSurface.shade, surface.py:93-99; grid._fd_probes / grad_fd / normal_batch) ---
// A shading point j owns `np` consecutive request slots: +x,+y,+z,-x,-y,-z probes and, when
// np == 7, the point itself (the "second sdf_query" that fetches the features).
struct ShadePoints {
  // either explicit points/dirs ...
  const double* pts;   // (m,3) or null
  const double* dirs;  // (m,3) or null
  // ... or rays + hit list: point = o[r] + t_hit[r] * d[r], dir = d[r]
  const double* o;
  const double* d;
  const double* t_hit;
  const int* list;
  const int* count;  // device count (null => m_host)
  int m_host;
};

__device__ __forceinline__ int shade_count(const ShadePoints& S) { return S.count ? *S.count : S.m_host; }

__device__ __forceinline__ void shade_point(const ShadePoints& S, int j, double p[3], double v[3]) {
  if (S.list) {
    int r = S.list[j];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      v[a] = S.d[3 * (size_t)r + a];
      p[a] = S.o[3 * (size_t)r + a] + S.t_hit[r] * v[a];
    }
  } else {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      p[a] = S.pts[3 * (size_t)j + a];
      v[a] = S.dirs ? S.dirs[3 * (size_t)j + a] : 0.0;
    }
  }
}

// grid._fd_probes (grid.py:416-437) for axis a of point p.
__device__ __forceinline__ void fd_pair(const GridGeom& G, const double p[3], int a, double& up, double& dn) {
  bool inside = (p[a] >= G.lo[a]) && (p[a] <= G.hi[a]);
  up = p[a] + G.fd_step;
  dn = p[a] - G.fd_step;
  if (inside) {
    up = fmin(up, G.hi[a]);
    dn = fmax(dn, G.lo[a]);
  }
}

static __global__ void shade_emit_kernel(RouteBuffers R, GridGeom G, ShadePoints S, int np) {
  const int m = shade_count(S);
  const int total = m * np;
  int stride = gridDim.x * blockDim.x;
  int n_round = (total + 31) & ~31;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_round; s += stride) {
    bool act = s < total;
    float x = 0.f, y = 0.f, z = 0.f;
    if (act) {
      int j = s / np, q = s - j * np;
      double p[3], v[3];
      shade_point(S, j, p, v);
      if (q < 6) {
        int a = q % 3;
        double up, dn;
        fd_pair(G, p, a, up, dn);
        p[a] = (q < 3) ? up : dn;
      }
      x = __double2float_rn(p[0]);
      y = __double2float_rn(p[1]);
      z = __double2float_rn(p[2]);
    }
    route_emit(R, G, act, s, x, y, z);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) R.ctr->n_requests = total;
}

// Gradient / normal from the probe distances; optionally set up the colour-MLP requests.
//   sdf_out : (m*np, 1+F) rows from the SDF kernel
//   grad_out: (m,3) f64 raw gradient (nullable)        -- grid.grad_fd
//   nrm_out : (m,3) f64 normal (zeros when degenerate unless fallback) (nullable)
//   ok_out  : (m) u8 (nullable)                         -- grid.normal_batch
//   fallback: replace degenerate normals by -view_dir    -- surface.py:96
//   colour request j (slot j): x = f32(p), v = f32(dir), n = f32(normal), z = features
static __global__ void shade_finish_kernel(RouteBuffers Rcol, GridGeom G, ShadePoints S, int np, const float* __restrict__ sdf_out,
                                    double eps, int fallback, double* __restrict__ grad_out, double* __restrict__ nrm_out,
                                    unsigned char* __restrict__ ok_out, int scatter_by_ray, float* __restrict__ col_v,
                                    float* __restrict__ col_n, float* __restrict__ col_z, int want_color) {
  const int m = shade_count(S);
  int stride = gridDim.x * blockDim.x;
  int n_round = (m + 31) & ~31;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_round; j += stride) {
    bool act = j < m;
    float x = 0.f, y = 0.f, z = 0.f;
    if (act) {
      double p[3], v[3], g[3];
      shade_point(S, j, p, v);
#pragma unroll
      for (int a = 0; a < 3; a++) {
        double up, dn;
        fd_pair(G, p, a, up, dn);
        double d_hi = (double)sdf_out[(size_t)(j * np + a) * kSdfOut];
        double d_lo = (double)sdf_out[(size_t)(j * np + 3 + a) * kSdfOut];
        g[a] = (d_hi - d_lo) / (up - dn);
      }
      double len = norm3(g);
      bool ok = len > eps;
      double nrm[3] = {0.0, 0.0, 0.0};
      if (ok) {
        nrm[0] = g[0] / len;
        nrm[1] = g[1] / len;
        nrm[2] = g[2] / len;
      } else if (fallback) {
        nrm[0] = -v[0];
        nrm[1] = -v[1];
        nrm[2] = -v[2];
      }
      size_t o = scatter_by_ray && S.list ? (size_t)S.list[j] : (size_t)j;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        if (grad_out) grad_out[3 * o + a] = g[a];
        if (nrm_out) nrm_out[3 * o + a] = nrm[a];
      }
      if (ok_out) ok_out[o] = ok;
      if (want_color) {
        x = __double2float_rn(p[0]);
        y = __double2float_rn(p[1]);
        z = __double2float_rn(p[2]);
#pragma unroll
        for (int a = 0; a < 3; a++) {
          col_v[3 * (size_t)j + a] = __double2float_rn(v[a]);
          col_n[3 * (size_t)j + a] = __double2float_rn(nrm[a]);
        }
        const float* feat = sdf_out + (size_t)(j * np + 6) * kSdfOut + 1;
#pragma unroll
        for (int f = 0; f < kFeat; f++) col_z[(size_t)j * kFeat + f] = feat[f];
      }
    }
    if (want_color) route_emit(Rcol, G, act, j, x, y, z);
  }
  if (want_color && blockIdx.x == 0 && threadIdx.x == 0) Rcol.ctr->n_requests = m;
}

// colors.astype(float64) (surface.py:99) [+ clip to [0,1] (surface.py:239)], scattered by ray or dense.
static __global__ void shade_colors_kernel(ShadePoints S, const float* __restrict__ rgb, int scatter_by_ray, int clip,
                                    double* __restrict__ colors_out) {
  const int m = shade_count(S);
  int stride = gridDim.x * blockDim.x;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    size_t o = scatter_by_ray && S.list ? (size_t)S.list[j] : (size_t)j;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      double c = (double)rgb[3 * (size_t)j + a];
      if (clip) c = fmin(fmax(c, 0.0), 1.0);
      colors_out[3 * o + a] = c;
    }
  }
}

// ---- frame composite (render_band epilogue, surface.py:310-324) ------------------------------------
// One thread per output pixel; sub-rays are laid out as a (rows*ss, W*ss) raster.
static __global__ void compose_kernel(int rows, int W, int ss, const unsigned char* __restrict__ hit,
                               const double* __restrict__ t_hit, const double* __restrict__ nrm,
                               const double* __restrict__ col, double bg0, double bg1, double bg2,
                               float* __restrict__ color_out, float* __restrict__ depth_out, float* __restrict__ normal_out,
                               unsigned char* __restrict__ hit_out) {
  long long n = (long long)rows * W;
  long long stride = (long long)gridDim.x * blockDim.x;
  const double bg[3] = {bg0, bg1, bg2};
  for (long long px = blockIdx.x * (long long)blockDim.x + threadIdx.x; px < n; px += stride) {
    int r = (int)(px / W), c = (int)(px % W);
    double acc[3] = {0.0, 0.0, 0.0};
    double best = INFINITY;
    long long best_i = -1;
    bool best_hit = false;
    for (int sr = 0; sr < ss; sr++)
      for (int sc = 0; sc < ss; sc++) {
        long long i = (long long)(r * ss + sr) * (W * ss) + (c * ss + sc);
        bool h = hit[i] != 0;
        double dep = h ? t_hit[i] : INFINITY;
#pragma unroll
        for (int a = 0; a < 3; a++) acc[a] += h ? col[3 * i + a] : bg[a];
        if (best_i < 0 || dep < best) {  // np.argmin: first minimum wins
          best = dep;
          best_i = i;
          best_hit = h;
        }
      }
    double inv_n = (double)(ss * ss);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      color_out[3 * px + a] = (float)(acc[a] / inv_n);
      normal_out[3 * px + a] = best_hit ? (float)nrm[3 * best_i + a] : 0.0f;
    }
    depth_out[px] = (float)best;
    hit_out[px] = best_hit;
  }
}

}  // namespace knf
