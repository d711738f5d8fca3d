// knf_pathtrace.cu -- the Lambertian path tracer over analytic shapes + neural grid objects
// (north_star subsystem 4).  Device restatement of pathtrace.py:
//   Rng (counter hash, :30-49), SphereObj / QuadObj / BoxObj (:115-222), NeuralObject (:225-274),
//   sample_lambertian (:287-304) + teacher.orthonormal_tangents (teacher.py:302-309),
//   intersect_scene (:311-330), _trace_batch (:340-420), render_pathtraced (:436-471).
// All path state is fp64 like the reference.  Paths are processed as one wavefront per bounce;
// each neural object is intersected with the fused march kernel (knf_march.cuh) in its local frame
// and its winning lanes are shaded with the FD-normal + colour-MLP pass (knf_rays.cuh).
// Compiled with -fmad=false; fma() appears only where NumPy goes through BLAS (`@`).
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "knf_engine.h"
#include "knf_rays.cuh"

using namespace knf;

#define KNF_TRY(expr)         \
  do {                        \
    int _rc = (expr);         \
    if (_rc != 0) return _rc; \
  } while (0)

namespace {

constexpr int kMaxObjects = 32;
constexpr unsigned long long kGold = 0x9E3779B97F4A7C15ull, kMul1 = 0xBF58476D1CE4E5B9ull, kMul2 = 0x94D049BB133111EBull;
constexpr int kRouletteStart = 3;
constexpr int kJitterSlot = 1 << 20;

struct ObjDev {
  int kind, material;
  double rgb[3];
  double a[3], b[3], c[3];
  double rot[9];
  double s;
  double nrm[3];  // quad: unit normal
  double uu[3];   // quad: edge_u / |edge_u|^2
  double vv[3];
  double bias;
  int neural_slot;  // index into the per-neural-object buffers, or -1
};

struct SceneDev {
  ObjDev obj[kMaxObjects];
  int n_obj;
  double env[3];
};

inline int blocks_for(size_t n, int threads = 256) {
  size_t b = (n + threads - 1) / threads;
  return (int)std::max<size_t>(1, std::min<size_t>(b, 148 * 16));
}

// ---- pathtrace.Rng ---------------------------------------------------------------------------------
__host__ __device__ inline unsigned long long mix64(unsigned long long x) {
  x = (x ^ (x >> 30)) * kMul1;
  x = (x ^ (x >> 27)) * kMul2;
  return x ^ (x >> 31);
}
__host__ __device__ inline double rng_uniform(unsigned long long seed, unsigned long long pixel, unsigned long long sample,
                                              unsigned long long slot) {
  unsigned long long h = mix64(seed + kGold);
  h = mix64(h ^ (pixel * kGold + kMul2));
  h = mix64(h ^ (sample * kGold + kMul2));
  h = mix64(h ^ (slot * kGold + kMul2));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void rng_kernel(unsigned long long seed, const unsigned long long* pixel, const unsigned long long* sample,
                           const unsigned long long* slot, long long n, double* u) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    u[i] = rng_uniform(seed, pixel[i], sample[i], slot[i]);
}

// ---- small vector helpers with NumPy's evaluation order --------------------------------------------
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {  // np.sum(a*b, axis=1)
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
__device__ __forceinline__ double mv3(const double a[3], const double b[3]) {  // a @ b through BLAS
  return fma(a[2], b[2], fma(a[1], b[1], fma(a[0], b[0], 0.0)));
}
__device__ __forceinline__ void cross3(const double a[3], const double b[3], double out[3]) {  // np.cross
  out[0] = a[1] * b[2] - a[2] * b[1];
  out[1] = a[2] * b[0] - a[0] * b[2];
  out[2] = a[0] * b[1] - a[1] * b[0];
}

// ---- analytic shapes: intersect_t --------------------------------------------------------------------
__device__ double sphere_t(const ObjDev& ob, const double o[3], const double d[3]) {
  double oc[3] = {o[0] - ob.a[0], o[1] - ob.a[1], o[2] - ob.a[2]};
  double b = dot3(oc, d);
  double c = dot3(oc, oc) - ob.s * ob.s;
  double disc = b * b - c;
  if (!(disc >= 0)) return INFINITY;
  double sq = sqrt(disc);
  double t0 = -b - sq, t1 = -b + sq;
  return t0 > 1e-9 ? t0 : (t1 > 1e-9 ? t1 : INFINITY);
}
__device__ double quad_t(const ObjDev& ob, const double o[3], const double d[3]) {
  double den = mv3(d, ob.nrm);
  if (!(fabs(den) > 1e-12)) return INFINITY;
  double co[3] = {ob.a[0] - o[0], ob.a[1] - o[1], ob.a[2] - o[2]};
  double tt = mv3(co, ob.nrm) / den;
  double rel[3];
#pragma unroll
  for (int a = 0; a < 3; a++) rel[a] = (o[a] + tt * d[a]) - ob.a[a];
  double su = mv3(rel, ob.uu), sv = mv3(rel, ob.vv);
  bool inside = (tt > 1e-9) && (su >= 0) && (su <= 1) && (sv >= 0) && (sv <= 1);
  return inside ? tt : INFINITY;
}
__device__ double box_t(const ObjDev& ob, const double o[3], const double d[3]) {
  double tn, tf;
  bool hit = slab(o, d, ob.a, ob.b, tn, tf);
  return (hit && tn > 1e-9) ? tn : ((hit && tf > 1e-9) ? tf : INFINITY);
}

// ---- analytic shapes: surface_at -----------------------------------------------------------------------
__device__ void analytic_normal(const ObjDev& ob, const double pos[3], const double d[3], double n[3]) {
  if (ob.kind == KNF_OBJ_SPHERE) {
#pragma unroll
    for (int a = 0; a < 3; a++) n[a] = (pos[a] - ob.a[a]) / ob.s;
  } else if (ob.kind == KNF_OBJ_QUAD) {
#pragma unroll
    for (int a = 0; a < 3; a++) n[a] = ob.nrm[a];
  } else {
    double best = INFINITY;
    int face = 0;
#pragma unroll
    for (int f = 0; f < 6; f++) {
      double w = f < 3 ? fabs(pos[f] - ob.a[f]) : fabs(pos[f - 3] - ob.b[f - 3]);
      if (w < best) {  // np.argmin: first minimum
        best = w;
        face = f;
      }
    }
    n[0] = n[1] = n[2] = 0.0;
    n[face % 3] = face < 3 ? -1.0 : 1.0;
  }
  if (dot3(n, d) > 0) {
    n[0] = -n[0];
    n[1] = -n[1];
    n[2] = -n[2];
  }
}

// teacher.orthonormal_tangents + pathtrace.sample_lambertian
__device__ void lambert_dir(const double n[3], double u1, double u2, double out[3]) {
  double helper[3] = {0.0, 0.0, 1.0};
  if (!(fabs(n[2]) < 0.9)) {
    helper[0] = 1.0;
    helper[2] = 0.0;
  }
  double t[3], b[3];
  cross3(helper, n, t);
  double len = norm3(t);
  t[0] /= len;
  t[1] /= len;
  t[2] /= len;
  cross3(n, t, b);
  double r = sqrt(u1);
  double phi = 2 * 3.141592653589793 * u2;
  double cz = sqrt(fmax(0.0, 1.0 - u1));
  double rc = r * cos(phi), rs = r * sin(phi);
#pragma unroll
  for (int a = 0; a < 3; a++) out[a] = (rc * t[a] + rs * b[a]) + cz * n[a];
}

__global__ void sample_lambertian_kernel(const double* nrm, const double* u1, const double* u2, long long n, double* out,
                                         double* pdf) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double nn[3] = {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]}, d[3];
    lambert_dir(nn, u1[i], u2[i], d);
    out[3 * i] = d[0];
    out[3 * i + 1] = d[1];
    out[3 * i + 2] = d[2];
    if (pdf) pdf[i] = sqrt(fmax(0.0, 1.0 - u1[i])) / 3.141592653589793;
  }
}

// ---- path state ------------------------------------------------------------------------------------------
struct PathState {
  double* o;     // (n,3)
  double* d;     // (n,3)
  double* thr;   // (n,3)
  double* rad;   // (n,3)
  double* best_t;
  int* best_obj;
  double* pos;   // (n,3) hit position (world)
  double* nrm;   // (n,3)
  double* alb;   // (n,3)
  double* bias;
  unsigned char* active;
  unsigned char* lambert;
  const unsigned long long* pixel;
  int n;
};

__global__ void pt_init_kernel(PathState P, const double* o, const double* d) {
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      P.o[3 * i + a] = o[3 * i + a];
      P.d[3 * i + a] = d[3 * i + a];
      P.thr[3 * i + a] = 1.0;
      P.rad[3 * i + a] = 0.0;
    }
    P.active[i] = 1;
  }
}

__global__ void pt_begin_kernel(PathState P) {
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    P.best_t[i] = INFINITY;
    P.best_obj[i] = -1;
  }
}

// One analytic object: t = intersect_t; strict '<' keeps the earlier object on ties (pathtrace.py:327).
__global__ void pt_analytic_kernel(PathState P, const SceneDev* S, int oi, double t_max, const unsigned char* mask) {
  const ObjDev ob = S->obj[oi];
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    if (mask && !mask[i]) continue;
    double o[3] = {P.o[3 * i], P.o[3 * i + 1], P.o[3 * i + 2]}, d[3] = {P.d[3 * i], P.d[3 * i + 1], P.d[3 * i + 2]};
    double t = ob.kind == KNF_OBJ_SPHERE ? sphere_t(ob, o, d) : (ob.kind == KNF_OBJ_QUAD ? quad_t(ob, o, d) : box_t(ob, o, d));
    if (t > t_max) t = INFINITY;
    if (t < P.best_t[i]) {
      P.best_t[i] = t;
      P.best_obj[i] = oi;
    }
  }
}

// NeuralObject.to_local + the box test (pathtrace.py:243-253); lanes that cannot hit get t_near=1, t_far=0.
__global__ void pt_neural_prepare_kernel(PathState P, const SceneDev* S, int oi, GridGeom box, const unsigned char* mask,
                                         double* ol, double* dl, double* tn, double* tf) {
  const ObjDev ob = S->obj[oi];
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    double near = 1.0, far = 0.0;
    double lo[3] = {0, 0, 0}, ld[3] = {0, 0, 1};
    if (!mask || mask[i]) {
      double rel[3] = {P.o[3 * i] - ob.a[0], P.o[3 * i + 1] - ob.a[1], P.o[3 * i + 2] - ob.a[2]};
      double d[3] = {P.d[3 * i], P.d[3 * i + 1], P.d[3 * i + 2]};
      vec_mat(rel, ob.rot, lo);
      lo[0] /= ob.s;
      lo[1] /= ob.s;
      lo[2] /= ob.s;
      vec_mat(d, ob.rot, ld);
      double a, b;
      if (slab(lo, ld, box.lo, box.hi, a, b) && a < b) {
        near = a;
        far = b;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
      ol[3 * i + a] = lo[a];
      dl[3 * i + a] = ld[a];
    }
    tn[i] = near;
    tf[i] = far;
  }
}

__global__ void pt_neural_best_kernel(PathState P, const SceneDev* S, int oi, double t_max, const unsigned char* hit,
                                      const double* t_local) {
  const double scale = S->obj[oi].s;
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    if (!hit[i]) continue;
    double t = t_local[i] * scale;
    if (t > t_max) continue;
    if (t < P.best_t[i]) {
      P.best_t[i] = t;
      P.best_obj[i] = oi;
    }
  }
}

// Environment for misses, hit positions, analytic normals/materials (pathtrace.py:354-387).
__global__ void pt_resolve_kernel(PathState P, const SceneDev* S, int last_bounce) {
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    if (!P.active[i]) continue;
    P.lambert[i] = 0;
    double t = P.best_t[i];
    int oi = P.best_obj[i];
    if (!isfinite(t)) {
#pragma unroll
      for (int a = 0; a < 3; a++) P.rad[3 * i + a] += P.thr[3 * i + a] * S->env[a];
      P.active[i] = 0;
      continue;
    }
    if (last_bounce) {
      P.active[i] = 0;
      continue;
    }
    double o[3] = {P.o[3 * i], P.o[3 * i + 1], P.o[3 * i + 2]}, d[3] = {P.d[3 * i], P.d[3 * i + 1], P.d[3 * i + 2]};
    double pos[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      pos[a] = o[a] + t * d[a];
      P.pos[3 * i + a] = pos[a];
    }
    const ObjDev& ob = S->obj[oi];
    if (ob.kind == KNF_OBJ_NEURAL) continue;  // shaded by the neural pass
    double n[3];
    analytic_normal(ob, pos, d, n);
    if (ob.material == KNF_MAT_EMISSIVE) {
#pragma unroll
      for (int a = 0; a < 3; a++) P.rad[3 * i + a] += P.thr[3 * i + a] * ob.rgb[a];
      P.active[i] = 0;
      continue;
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
      P.nrm[3 * i + a] = n[a];
      P.alb[3 * i + a] = ob.rgb[a];
    }
    P.bias[i] = ob.bias;
    P.lambert[i] = 1;
  }
}

// Winners of neural object oi -> dense (position_local, dir_local) list for FieldSurface.shade.
__global__ void pt_neural_collect_kernel(PathState P, int oi, const double* ol, const double* dl, const double* t_local,
                                         int* list, int* count, double* pts, double* dirs) {
  int stride = gridDim.x * blockDim.x;
  int n_round = (P.n + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    bool want = i < P.n && P.active[i] && P.best_obj[i] == oi && isfinite(P.best_t[i]);
    int j = warp_append(count, want);
    if (want) {
      list[j] = i;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        double dd = dl[3 * i + a];
        pts[3 * j + a] = ol[3 * i + a] + t_local[i] * dd;  // res.position = origins + t_hit * dirs (local frame)
        dirs[3 * j + a] = dd;
      }
    }
  }
}

// NeuralObject.surface_at_indices (pathtrace.py:270-274): rotate, renormalise, face the ray, clip albedo.
__global__ void pt_neural_apply_kernel(PathState P, const SceneDev* S, int oi, const int* list, int m, const double* nrm_local,
                                       const double* colors) {
  const ObjDev ob = S->obj[oi];
  int stride = gridDim.x * blockDim.x;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    int i = list[j];
    double nl[3] = {nrm_local[3 * j], nrm_local[3 * j + 1], nrm_local[3 * j + 2]}, nw[3];
    vec_matT(nl, ob.rot, nw);
    double len = norm3(nw);
    nw[0] /= len;
    nw[1] /= len;
    nw[2] /= len;
    double d[3] = {P.d[3 * i], P.d[3 * i + 1], P.d[3 * i + 2]};
    if (dot3(nw, d) > 0) {
      nw[0] = -nw[0];
      nw[1] = -nw[1];
      nw[2] = -nw[2];
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
      P.nrm[3 * i + a] = nw[a];
      P.alb[3 * i + a] = fmin(fmax(colors[3 * j + a], 0.0), 1.0);
    }
    P.bias[i] = ob.bias;
    P.lambert[i] = 1;
  }
}

// Throughput, Russian roulette, cosine sampling (pathtrace.py:396-418).
__global__ void pt_bounce_kernel(PathState P, unsigned long long seed, unsigned long long sample, int bounce) {
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    if (!P.active[i] || !P.lambert[i]) continue;
    double thr[3];
#pragma unroll
    for (int a = 0; a < 3; a++) thr[a] = P.thr[3 * i + a] * P.alb[3 * i + a];
    unsigned long long pix = P.pixel[i];
    if (bounce >= kRouletteStart) {
      double p = fmin(fmax(fmax(fmax(thr[0], thr[1]), thr[2]), 0.05), 0.95);
      double u = rng_uniform(seed, pix, sample, (unsigned long long)(bounce * 3));
      if (u > p) {
        P.active[i] = 0;
#pragma unroll
        for (int a = 0; a < 3; a++) P.thr[3 * i + a] = thr[a];
        continue;
      }
#pragma unroll
      for (int a = 0; a < 3; a++) thr[a] /= p;
    }
    double u1 = rng_uniform(seed, pix, sample, (unsigned long long)(bounce * 3 + 1));
    double u2 = rng_uniform(seed, pix, sample, (unsigned long long)(bounce * 3 + 2));
    double n[3] = {P.nrm[3 * i], P.nrm[3 * i + 1], P.nrm[3 * i + 2]}, nd[3];
    lambert_dir(n, u1, u2, nd);
    double bias = P.bias[i];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      P.thr[3 * i + a] = thr[a];
      P.o[3 * i + a] = P.pos[3 * i + a] + n[a] * bias;
      P.d[3 * i + a] = nd[a];
    }
  }
}

__global__ void pt_jitter_rays_kernel(CameraDev cam, int row0, long long n, unsigned long long seed, unsigned long long sample,
                                      unsigned long long* pixel_ids, double* o, double* d) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    long long col = i % cam.width, row = row0 + i / cam.width;
    unsigned long long pid = (unsigned long long)(row * cam.width + col);
    pixel_ids[i] = pid;
    double jx = rng_uniform(seed, pid, sample, (unsigned long long)kJitterSlot);
    double jy = rng_uniform(seed, pid, sample, (unsigned long long)(kJitterSlot + 1));
    double dir[3];
    pixel_ray(cam, (double)col, (double)row, jx, jy, dir);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      o[3 * i + a] = cam.pos[a];
      d[3 * i + a] = dir[a];
    }
  }
}

__global__ void pt_accumulate_kernel(const double* rad, double* acc, long long n3, int first) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n3; i += stride) acc[i] = first ? rad[i] : acc[i] + rad[i];
}
__global__ void pt_average_kernel(double* acc, long long n3, double spp) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n3; i += stride) acc[i] = acc[i] / spp;
}

__global__ void pt_export_kernel(PathState P, double* t_out, int* obj_out) {
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += stride) {
    if (t_out) t_out[i] = P.best_t[i];
    if (obj_out) obj_out[i] = P.best_obj[i];
  }
}

}  // namespace

struct knf_scene_s {
  int device = 0;
  SceneDev host{};
  SceneDev* dev = nullptr;
  std::vector<knf_field_t> fields;      // per object (null for analytic)
  std::vector<KnfSettings> settings;    // per object
  int n_neural = 0;
  std::mutex mu;
  // path workspace
  DevBuf o, d, thr, rad, best_t, best_obj, pos, nrm, alb, bias, active, lambert, pixel, acc, ray_o, ray_d;
  struct NeuralBufs {
    DevBuf ol, dl, tn, tf, t, hit, list, count, pts, dirs, nrm, col;
  };
  std::vector<NeuralBufs> nb;
  int* host_count = nullptr;
};

namespace {

int ensure_paths(knf_scene_s& sc, size_t n) {
  KNF_TRY(sc.o.ensure(n * 24));
  KNF_TRY(sc.d.ensure(n * 24));
  KNF_TRY(sc.thr.ensure(n * 24));
  KNF_TRY(sc.rad.ensure(n * 24));
  KNF_TRY(sc.best_t.ensure(n * 8));
  KNF_TRY(sc.best_obj.ensure(n * 4));
  KNF_TRY(sc.pos.ensure(n * 24));
  KNF_TRY(sc.nrm.ensure(n * 24));
  KNF_TRY(sc.alb.ensure(n * 24));
  KNF_TRY(sc.bias.ensure(n * 8));
  KNF_TRY(sc.active.ensure(n));
  KNF_TRY(sc.lambert.ensure(n));
  for (auto& b : sc.nb) {
    KNF_TRY(b.ol.ensure(n * 24));
    KNF_TRY(b.dl.ensure(n * 24));
    KNF_TRY(b.tn.ensure(n * 8));
    KNF_TRY(b.tf.ensure(n * 8));
    KNF_TRY(b.t.ensure(n * 8));
    KNF_TRY(b.hit.ensure(n));
    KNF_TRY(b.list.ensure(n * 4));
    KNF_TRY(b.count.ensure(16));
    KNF_TRY(b.pts.ensure(n * 24));
    KNF_TRY(b.dirs.ensure(n * 24));
    KNF_TRY(b.nrm.ensure(n * 24));
    KNF_TRY(b.col.ensure(n * 24));
  }
  return 0;
}

PathState path_state(knf_scene_s& sc, int n, const unsigned long long* pixel) {
  PathState P;
  P.o = sc.o.as<double>();
  P.d = sc.d.as<double>();
  P.thr = sc.thr.as<double>();
  P.rad = sc.rad.as<double>();
  P.best_t = sc.best_t.as<double>();
  P.best_obj = sc.best_obj.as<int>();
  P.pos = sc.pos.as<double>();
  P.nrm = sc.nrm.as<double>();
  P.alb = sc.alb.as<double>();
  P.bias = sc.bias.as<double>();
  P.active = sc.active.as<unsigned char>();
  P.lambert = sc.lambert.as<unsigned char>();
  P.pixel = pixel;
  P.n = n;
  return P;
}

// intersect_scene over the current path origins/dirs (pathtrace.py:311-330); `mask` restricts lanes.
int intersect_scene_device(knf_scene_s& sc, PathState& P, double t_max, const unsigned char* mask, cudaStream_t st) {
  const int nb = blocks_for((size_t)P.n);
  pt_begin_kernel<<<nb, 256, 0, st>>>(P);
  for (int oi = 0; oi < sc.host.n_obj; oi++) {
    const ObjDev& ob = sc.host.obj[oi];
    if (ob.kind != KNF_OBJ_NEURAL) {
      pt_analytic_kernel<<<nb, 256, 0, st>>>(P, sc.dev, oi, t_max, mask);
      continue;
    }
    knf_scene_s::NeuralBufs& B = sc.nb[ob.neural_slot];
    Field& F = sc.fields[oi]->f;
    std::lock_guard<std::mutex> lk(F.mu);
    CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
    pt_neural_prepare_kernel<<<nb, 256, 0, st>>>(P, sc.dev, oi, F.geom, mask, B.ol.as<double>(), B.dl.as<double>(),
                                                 B.tn.as<double>(), B.tf.as<double>());
    KNF_TRY(march_device(F, B.ol.as<double>(), B.dl.as<double>(), B.tn.as<double>(), B.tf.as<double>(), P.n,
                         sc.settings[oi], B.hit.as<unsigned char>(), B.t.as<double>(), nullptr, nullptr, false, st));
    pt_neural_best_kernel<<<nb, 256, 0, st>>>(P, sc.dev, oi, t_max, B.hit.as<unsigned char>(), B.t.as<double>());
  }
  KNF_CUDA(cudaGetLastError());
  return 0;
}

// pathtrace._trace_batch for device rays (o, d, pixel ids) -> P.rad
int trace_batch_device(knf_scene_s& sc, const double* o, const double* d, const unsigned long long* pixel, int n,
                       unsigned long long sample, unsigned long long seed, int max_bounces, cudaStream_t st) {
  KNF_TRY(ensure_paths(sc, (size_t)n));
  PathState P = path_state(sc, n, pixel);
  const int nb = blocks_for((size_t)n);
  pt_init_kernel<<<nb, 256, 0, st>>>(P, o, d);
  for (int bounce = 0; bounce <= max_bounces; bounce++) {
    KNF_TRY(intersect_scene_device(sc, P, INFINITY, P.active, st));
    pt_resolve_kernel<<<nb, 256, 0, st>>>(P, sc.dev, bounce == max_bounces ? 1 : 0);
    if (bounce == max_bounces) break;
    for (int oi = 0; oi < sc.host.n_obj; oi++) {
      const ObjDev& ob = sc.host.obj[oi];
      if (ob.kind != KNF_OBJ_NEURAL) continue;
      knf_scene_s::NeuralBufs& B = sc.nb[ob.neural_slot];
      Field& F = sc.fields[oi]->f;
      KNF_CUDA(cudaMemsetAsync(B.count.p, 0, 16, st));
      pt_neural_collect_kernel<<<nb, 256, 0, st>>>(P, oi, B.ol.as<double>(), B.dl.as<double>(), B.t.as<double>(),
                                                  B.list.as<int>(), B.count.as<int>(), B.pts.as<double>(),
                                                  B.dirs.as<double>());
      KNF_CUDA(cudaMemcpyAsync(sc.host_count, B.count.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      KNF_CUDA(cudaStreamSynchronize(st));
      int m = *sc.host_count;
      if (m <= 0) continue;
      std::lock_guard<std::mutex> lk(F.mu);
      CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
      ShadeTargets T;
      T.normals = B.nrm.as<double>();
      T.colors = B.col.as<double>();
      T.fallback = true;
      KNF_TRY(shade_points_device(F, B.pts.as<double>(), B.dirs.as<double>(), m, T, st));
      pt_neural_apply_kernel<<<blocks_for((size_t)m), 256, 0, st>>>(P, sc.dev, oi, B.list.as<int>(), m, B.nrm.as<double>(),
                                                                  B.col.as<double>());
    }
    pt_bounce_kernel<<<nb, 256, 0, st>>>(P, seed, sample, bounce);
  }
  KNF_CUDA(cudaGetLastError());
  return 0;
}

// Host<->device staging (same contract as knf_api.cu's).
struct Stage {
  int mem;
  cudaStream_t st;
  std::vector<DevBuf> bufs;
  struct Out {
    void* host;
    void* dev;
    size_t bytes;
  };
  std::vector<Out> outs;
  int rc = 0;
  Stage(int m, cudaStream_t s) : mem(m), st(s) { bufs.reserve(16); }
  ~Stage() {
    for (auto& b : bufs) b.release();
  }
  void* buf(size_t bytes) {
    bufs.emplace_back();
    if (bufs.back().ensure(std::max<size_t>(bytes, 16)) != 0) {
      rc = KNF_E_NOMEM;
      return nullptr;
    }
    return bufs.back().p;
  }
  template <class T>
  const T* in(const T* p, size_t count) {
    if (mem == KNF_MEM_DEVICE || !p) return p;
    void* d = buf(count * sizeof(T));
    if (!d) return nullptr;
    if (cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, st) != cudaSuccess) rc = KNF_E_CUDA;
    return reinterpret_cast<const T*>(d);
  }
  template <class T>
  T* out(T* p, size_t count) {
    if (mem == KNF_MEM_DEVICE || !p) return p;
    void* d = buf(count * sizeof(T));
    if (!d) return nullptr;
    outs.push_back({p, d, count * sizeof(T)});
    return reinterpret_cast<T*>(d);
  }
  int finish() {
    if (rc) return fail(rc, "staging failed");
    if (mem == KNF_MEM_DEVICE) return 0;
    for (auto& o : outs) KNF_CUDA(cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, st));
    KNF_CUDA(cudaStreamSynchronize(st));
    return 0;
  }
};

CameraDev camera_dev(const KnfCamera& c) {
  CameraDev d;
  for (int i = 0; i < 3; i++) d.pos[i] = c.position[i];
  for (int i = 0; i < 9; i++) d.rot[i] = c.rotation[i];
  d.width = c.width;
  d.height = c.height;
  d.scale = 2.0 * std::tan(c.fov_y / 2) / c.height;
  return d;
}

}  // namespace

extern "C" {

int knf_scene_create(const KnfObject* objects, int32_t n_objects, const double env_rgb[3], int device, knf_scene_t* out) {
  if (!out) return fail(KNF_E_INVALID, "null output handle");
  *out = nullptr;
  if (n_objects < 0 || (n_objects > 0 && !objects) || !env_rgb) return fail(KNF_E_INVALID, "bad arguments to knf_scene_create");
  if (n_objects > kMaxObjects) return fail(KNF_E_UNSUPPORTED, "at most 32 scene objects are supported");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(KNF_E_CUDA, "no CUDA device available: libknf_b200 has no CPU fallback");
  }
  KNF_CUDA(cudaSetDevice(device));
  std::unique_ptr<knf_scene_s> sc(new knf_scene_s());
  sc->device = device;
  sc->host.n_obj = n_objects;
  for (int a = 0; a < 3; a++) sc->host.env[a] = env_rgb[a];
  sc->fields.assign(n_objects, nullptr);
  sc->settings.assign(n_objects, KnfSettings{1e-3, 128, 0.8});
  for (int i = 0; i < n_objects; i++) {
    const KnfObject& in = objects[i];
    ObjDev& ob = sc->host.obj[i];
    std::memset(&ob, 0, sizeof(ob));
    ob.kind = in.kind;
    ob.material = in.material;
    ob.neural_slot = -1;
    for (int a = 0; a < 3; a++) {
      ob.rgb[a] = in.rgb[a];
      ob.a[a] = in.a[a];
      ob.b[a] = in.b[a];
      ob.c[a] = in.c[a];
    }
    for (int a = 0; a < 9; a++) ob.rot[a] = in.rot[a];
    ob.s = in.s;
    ob.bias = 1e-6;  // pathtrace.py:333-337
    switch (in.kind) {
      case KNF_OBJ_SPHERE:
        if (!(in.s > 0)) return fail(KNF_E_INVALID, "radius must be > 0");
        break;
      case KNF_OBJ_QUAD: {
        double n[3] = {in.b[1] * in.c[2] - in.b[2] * in.c[1], in.b[2] * in.c[0] - in.b[0] * in.c[2],
                       in.b[0] * in.c[1] - in.b[1] * in.c[0]};
        double ln = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        if (ln < 1e-12) return fail(KNF_E_INVALID, "degenerate quad");
        double uu = in.b[0] * in.b[0] + in.b[1] * in.b[1] + in.b[2] * in.b[2];
        double vv = in.c[0] * in.c[0] + in.c[1] * in.c[1] + in.c[2] * in.c[2];
        for (int a = 0; a < 3; a++) {
          ob.nrm[a] = n[a] / ln;
          ob.uu[a] = in.b[a] / uu;
          ob.vv[a] = in.c[a] / vv;
        }
        break;
      }
      case KNF_OBJ_BOX:
        for (int a = 0; a < 3; a++)
          if (!(in.a[a] < in.b[a])) return fail(KNF_E_INVALID, "bmin must be < bmax");
        break;
      case KNF_OBJ_NEURAL:
        if (!in.field) return fail(KNF_E_INVALID, "neural object without a field");
        if (!(in.s > 0)) return fail(KNF_E_INVALID, "scale must be > 0");
        if (in.field->f.device != device) return fail(KNF_E_INVALID, "neural object's field lives on another device");
        if (!(in.settings.step_scale > 0 && in.settings.step_scale <= 1)) return fail(KNF_E_INVALID, "step_scale must be in (0, 1]");
        sc->fields[i] = in.field;
        sc->settings[i] = in.settings;
        ob.bias = 4.0 * in.settings.eps_hit;
        ob.neural_slot = sc->n_neural++;
        break;
      default:
        return fail(KNF_E_INVALID, "unknown object kind");
    }
    if (in.kind != KNF_OBJ_NEURAL && in.material != KNF_MAT_LAMBERTIAN && in.material != KNF_MAT_EMISSIVE)
      return fail(KNF_E_INVALID, "unknown material");
  }
  sc->nb.resize(sc->n_neural);
  KNF_CUDA(cudaMalloc(&sc->dev, sizeof(SceneDev)));
  KNF_CUDA(cudaMemcpy(sc->dev, &sc->host, sizeof(SceneDev), cudaMemcpyHostToDevice));
  KNF_CUDA(cudaMallocHost(&sc->host_count, 64));
  *out = sc.release();
  return 0;
}

int knf_scene_destroy(knf_scene_t sc) {
  if (!sc) return 0;
  cudaSetDevice(sc->device);
  DevBuf* all[] = {&sc->o, &sc->d, &sc->thr, &sc->rad, &sc->best_t, &sc->best_obj, &sc->pos, &sc->nrm, &sc->alb,
                   &sc->bias, &sc->active, &sc->lambert, &sc->pixel, &sc->acc, &sc->ray_o, &sc->ray_d};
  for (DevBuf* b : all) b->release();
  for (auto& b : sc->nb) {
    DevBuf* nbs[] = {&b.ol, &b.dl, &b.tn, &b.tf, &b.t, &b.hit, &b.list, &b.count, &b.pts, &b.dirs, &b.nrm, &b.col};
    for (DevBuf* x : nbs) x->release();
  }
  if (sc->dev) cudaFree(sc->dev);
  if (sc->host_count) cudaFreeHost(sc->host_count);
  delete sc;
  return 0;
}

int knf_rng_uniform(uint64_t seed, const uint64_t* pixel, const uint64_t* sample, const uint64_t* slot, int64_t n, double* u,
                    int device, int mem, void* stream) {
  if (n < 0 || (n > 0 && (!pixel || !sample || !slot || !u))) return fail(KNF_E_INVALID, "bad arguments to knf_rng_uniform");
  if (n == 0) return 0;
  KNF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  Stage S(mem, st);
  auto* dp = reinterpret_cast<const unsigned long long*>(S.in(pixel, (size_t)n));
  auto* ds = reinterpret_cast<const unsigned long long*>(S.in(sample, (size_t)n));
  auto* dl = reinterpret_cast<const unsigned long long*>(S.in(slot, (size_t)n));
  double* du = S.out(u, (size_t)n);
  if (S.rc) return fail(S.rc, "staging failed");
  rng_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(seed, dp, ds, dl, (long long)n, du);
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

int knf_sample_lambertian(const double* normals, const double* u1, const double* u2, int64_t n, double* dirs, double* pdf,
                          int device, int mem, void* stream) {
  if (n < 0 || (n > 0 && (!normals || !u1 || !u2 || !dirs))) return fail(KNF_E_INVALID, "bad arguments to knf_sample_lambertian");
  if (n == 0) return 0;
  KNF_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  Stage S(mem, st);
  const double* dn = S.in(normals, (size_t)n * 3);
  const double* d1 = S.in(u1, (size_t)n);
  const double* d2 = S.in(u2, (size_t)n);
  double* dd = S.out(dirs, (size_t)n * 3);
  double* dpdf = S.out(pdf, (size_t)n);
  if (S.rc) return fail(S.rc, "staging failed");
  sample_lambertian_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(dn, d1, d2, (long long)n, dd, dpdf);
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

int knf_intersect_scene(knf_scene_t sc, const double* origins, const double* dirs, int64_t n, double t_max, double* t,
                        int32_t* obj, int mem, void* stream) {
  if (!sc) return fail(KNF_E_INVALID, "null scene");
  if (n < 0 || (n > 0 && (!origins || !dirs))) return fail(KNF_E_INVALID, "bad arguments to knf_intersect_scene");
  if (n == 0) return 0;
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "too many rays for one call");
  std::lock_guard<std::mutex> lk(sc->mu);
  KNF_CUDA(cudaSetDevice(sc->device));
  cudaStream_t st = (cudaStream_t)stream;
  Stage S(mem, st);
  const double* dorig = S.in(origins, (size_t)n * 3);
  const double* ddir = S.in(dirs, (size_t)n * 3);
  double* dt = S.out(t, (size_t)n);
  int32_t* dobj = S.out(obj, (size_t)n);
  if (S.rc) return fail(S.rc, "staging failed");
  KNF_TRY(ensure_paths(*sc, (size_t)n));
  PathState P = path_state(*sc, (int)n, nullptr);
  pt_init_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(P, dorig, ddir);
  KNF_TRY(intersect_scene_device(*sc, P, t_max, nullptr, st));
  pt_export_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(P, dt, dobj);
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

int knf_trace_paths(knf_scene_t sc, const double* origins, const double* dirs, const uint64_t* pixel_ids, int64_t n,
                    uint64_t sample, uint64_t seed, int32_t max_bounces, double* radiance, int mem, void* stream) {
  if (!sc) return fail(KNF_E_INVALID, "null scene");
  if (n < 0 || (n > 0 && (!origins || !dirs || !pixel_ids || !radiance)) || max_bounces < 0)
    return fail(KNF_E_INVALID, "bad arguments to knf_trace_paths");
  if (n == 0) return 0;
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "too many paths for one call");
  std::lock_guard<std::mutex> lk(sc->mu);
  KNF_CUDA(cudaSetDevice(sc->device));
  cudaStream_t st = (cudaStream_t)stream;
  Stage S(mem, st);
  const double* dorig = S.in(origins, (size_t)n * 3);
  const double* ddir = S.in(dirs, (size_t)n * 3);
  auto* dpix = reinterpret_cast<const unsigned long long*>(S.in(pixel_ids, (size_t)n));
  double* drad = S.out(radiance, (size_t)n * 3);
  if (S.rc) return fail(S.rc, "staging failed");
  KNF_TRY(trace_batch_device(*sc, dorig, ddir, dpix, (int)n, sample, seed, max_bounces, st));
  KNF_CUDA(cudaMemcpyAsync(drad, sc->rad.p, (size_t)n * 24, cudaMemcpyDeviceToDevice, st));
  return S.finish();
}

int knf_pathtrace(knf_scene_t sc, const KnfCamera* cam, int32_t spp, uint64_t seed, int32_t max_bounces,
                  int32_t sample_offset, int row0, int row1, double* hdr, int mem, void* stream) {
  if (!sc) return fail(KNF_E_INVALID, "null scene");
  if (!cam || !hdr) return fail(KNF_E_INVALID, "null argument to knf_pathtrace");
  if (spp < 1) return fail(KNF_E_INVALID, "spp must be >= 1");
  if (max_bounces < 0 || sample_offset < 0) return fail(KNF_E_INVALID, "max_bounces and sample_offset must be >= 0");
  if (cam->width <= 0 || cam->height <= 0) return fail(KNF_E_INVALID, "image dimensions must be positive");
  if (row0 < 0 || row1 > cam->height || row0 >= row1) return fail(KNF_E_INVALID, "row range out of bounds");
  std::lock_guard<std::mutex> lk(sc->mu);
  KNF_CUDA(cudaSetDevice(sc->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int W = cam->width, rows = row1 - row0;
  Stage S(mem, st);
  double* dhdr = S.out(hdr, (size_t)rows * W * 3);
  if (S.rc) return fail(S.rc, "staging failed");
  CameraDev cd = camera_dev(*cam);
  // bands of at most ~2M paths, like the reference's row bands (pathtrace.py:450-469)
  const int rows_per_band = (int)std::max<int64_t>(1, (2ll << 20) / W);
  for (int r = 0; r < rows; r += rows_per_band) {
    const int br = std::min(rows_per_band, rows - r);
    const int64_t n = (int64_t)br * W;
    KNF_TRY(sc->pixel.ensure((size_t)n * 8));
    KNF_TRY(sc->ray_o.ensure((size_t)n * 24));
    KNF_TRY(sc->ray_d.ensure((size_t)n * 24));
    double* acc = dhdr + (size_t)r * W * 3;
    for (int s = 0; s < spp; s++) {
      const unsigned long long sample = (unsigned long long)(sample_offset + s);
      pt_jitter_rays_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(cd, row0 + r, (long long)n, seed, sample,
                                                                 sc->pixel.as<unsigned long long>(), sc->ray_o.as<double>(),
                                                                 sc->ray_d.as<double>());
      KNF_TRY(trace_batch_device(*sc, sc->ray_o.as<double>(), sc->ray_d.as<double>(), sc->pixel.as<unsigned long long>(),
                                 (int)n, sample, seed, max_bounces, st));
      pt_accumulate_kernel<<<blocks_for((size_t)n * 3), 256, 0, st>>>(sc->rad.as<double>(), acc, (long long)n * 3, s == 0 ? 1 : 0);
    }
    pt_average_kernel<<<blocks_for((size_t)n * 3), 256, 0, st>>>(acc, (long long)n * 3, (double)spp);
  }
  KNF_CUDA(cudaGetLastError());
  return S.finish();
}

}  // extern "C"
