// knf_volume.cu -- SURVEY 8(f).3: forward pass of the S-density volume renderer
// (training._volume_forward, training.py:330-415) -- the "NeuS volume samples" consumer of the batched
// multi-network forward.  Forward only (photometric-loss evaluation); the backward pass is training
// and stays out of scope.
//
// Per ray: n_s stratified samples inside the box; SDF + features at every sample; FD normals only
// where |d| <= 20/s (elsewhere a facing placeholder, training.py:373-383); colour at the left
// sample of each of the m = n_s - 1 intervals; opacity = clipped relative drop of sigmoid(s d);
// sequential transmittance product; background for what is left; clip to [0,1].
#include <cmath>

#include "knf_engine.h"
#include "knf_rays.cuh"

using namespace knf;

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

struct VolArgs {
  const double* o;       // (B,3)
  const double* d;       // (B,3)
  const double* jitter;  // (B,n_s) or null (0.5)
  int B, n_s;
  double* t0;            // (B) box entry
  double* dt;            // (B) sample spacing; <= 0 marks an inactive ray
};

// fp64 sample parameter and position exactly as training.py:362-364
__device__ __forceinline__ double sample_t(const VolArgs& V, int r, int j) {
  const double jit = V.jitter ? V.jitter[(size_t)r * V.n_s + j] : 0.5;
  return V.t0[r] + ((double)j + jit) * V.dt[r];
}

__global__ void vol_box_kernel(VolArgs V, GridGeom G, unsigned char* active) {
  int stride = gridDim.x * blockDim.x;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < V.B; r += stride) {
    double o[3] = {V.o[3 * r], V.o[3 * r + 1], V.o[3 * r + 2]}, d[3] = {V.d[3 * r], V.d[3 * r + 1], V.d[3 * r + 2]};
    double t0, t1;
    bool hit = slab(o, d, G.lo, G.hi, t0, t1);
    bool act = hit && (t0 < t1);
    V.t0[r] = t0;
    V.dt[r] = act ? (t1 - t0) / (double)V.n_s : 0.0;
    active[r] = act;
  }
}

// One request per (ray, sample); slots of inactive rays carry cell -1 and are skipped by the scatter.
__global__ void vol_emit_kernel(RouteBuffers R, GridGeom G, VolArgs V, const unsigned char* active) {
  const int total = V.B * V.n_s;
  int stride = gridDim.x * blockDim.x;
  int n_round = (total + 31) & ~31;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_round; s += stride) {
    bool act = false;
    float p[3] = {0.f, 0.f, 0.f};
    if (s < total) {
      int r = s / V.n_s, j = s - r * V.n_s;
      act = active[r] != 0;
      if (act) {
        double t = sample_t(V, r, j);
#pragma unroll
        for (int a = 0; a < 3; a++) p[a] = __double2float_rn(V.o[3 * r + a] + t * V.d[3 * r + a]);
      } else {
        R.req_cell[s] = -1;
      }
    }
    route_emit(R, G, act, s, p[0], p[1], p[2]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) R.ctr->n_requests = total;
}

// Interval samples close enough to the surface to matter get FD normals: compact them.
__global__ void vol_near_kernel(VolArgs V, const unsigned char* active, const float* sdf_out, double s_param, int* list,
                                int* count, double* pts, double* nrm_all) {
  const int m = V.n_s - 1, total = V.B * m;
  int stride = gridDim.x * blockDim.x;
  int n_round = (total + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    bool want = false;
    int r = 0, j = 0;
    if (i < total) {
      r = i / m;
      j = i - r * m;
      if (active[r]) {
        // placeholder normal: facing the ray (training.py:378)
#pragma unroll
        for (int a = 0; a < 3; a++) nrm_all[3 * (size_t)i + a] = -V.d[3 * r + a];
        double dv = (double)sdf_out[((size_t)r * V.n_s + j) * kSdfOut];
        want = fabs(dv) <= 20.0 / s_param;
      }
    }
    int k = warp_append(count, want);
    if (want) {
      list[k] = i;
      double t = sample_t(V, r, j);
#pragma unroll
      for (int a = 0; a < 3; a++) pts[3 * (size_t)k + a] = V.o[3 * r + a] + t * V.d[3 * r + a];
    }
  }
}

// normals of the compacted near samples -> the per-interval normal array (degenerate: keep -v)
__global__ void vol_near_apply_kernel(const int* list, int n_near, const double* nrm, const unsigned char* ok, double* nrm_all) {
  int stride = gridDim.x * blockDim.x;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_near; k += stride) {
    if (!ok[k]) continue;
    size_t i = (size_t)list[k];
#pragma unroll
    for (int a = 0; a < 3; a++) nrm_all[3 * i + a] = nrm[3 * (size_t)k + a];
  }
}

// Colour requests: one per (active ray, interval), routed by the fp32 sample position.
__global__ void vol_color_emit_kernel(RouteBuffers R, GridGeom G, VolArgs V, const unsigned char* active, const float* sdf_out,
                                      const double* nrm_all, float* col_v, float* col_n, float* col_z) {
  const int m = V.n_s - 1, total = V.B * m;
  int stride = gridDim.x * blockDim.x;
  int n_round = (total + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    bool act = false;
    float p[3] = {0.f, 0.f, 0.f};
    if (i < total) {
      int r = i / m, j = i - r * m;
      act = active[r] != 0;
      if (act) {
        double t = sample_t(V, r, j);
#pragma unroll
        for (int a = 0; a < 3; a++) {
          p[a] = __double2float_rn(V.o[3 * r + a] + t * V.d[3 * r + a]);
          col_v[3 * (size_t)i + a] = __double2float_rn(V.d[3 * r + a]);
          col_n[3 * (size_t)i + a] = __double2float_rn(nrm_all[3 * (size_t)i + a]);
        }
        const float* feat = sdf_out + ((size_t)r * V.n_s + j) * kSdfOut + 1;
#pragma unroll
        for (int f = 0; f < kFeat; f++) col_z[(size_t)i * kFeat + f] = feat[f];
      } else {
        R.req_cell[i] = -1;
      }
    }
    route_emit(R, G, act, i, p[0], p[1], p[2]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) R.ctr->n_requests = total;
}

__device__ __forceinline__ double sigmoid64(double x) {  // training.py:418-424
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  double e = exp(x);
  return e / (1.0 + e);
}

// training.py:391-403, one thread per ray
__global__ void vol_composite_kernel(VolArgs V, const unsigned char* active, const float* sdf_out, const float* rgb, double s_param,
                                     double bg0, double bg1, double bg2, double* colors) {
  const int m = V.n_s - 1;
  const double bg[3] = {bg0, bg1, bg2};
  int stride = gridDim.x * blockDim.x;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < V.B; r += stride) {
    double out[3];
    if (!active[r]) {
#pragma unroll
      for (int a = 0; a < 3; a++) out[a] = bg[a];
    } else {
      double acc[3] = {0.0, 0.0, 0.0};
      double T = 1.0;  // transmittance before interval j (np.cumprod, sequential)
      double phi = sigmoid64(s_param * (double)sdf_out[((size_t)r * V.n_s) * kSdfOut]);
      for (int j = 0; j < m; j++) {
        double phi_next = sigmoid64(s_param * (double)sdf_out[((size_t)r * V.n_s + j + 1) * kSdfOut]);
        double ratio = (phi - phi_next) / fmax(phi, 1e-12);
        double alpha = fmin(fmax(ratio, 0.0), 1.0);
        double w = T * alpha;
#pragma unroll
        for (int a = 0; a < 3; a++) acc[a] += w * (double)rgb[((size_t)r * m + j) * 3 + a];
        T = T * (1.0 - alpha);
        phi = phi_next;
      }
#pragma unroll
      for (int a = 0; a < 3; a++) out[a] = acc[a] + T * bg[a];
    }
#pragma unroll
    for (int a = 0; a < 3; a++) colors[3 * (size_t)r + a] = fmin(fmax(out[a], 0.0), 1.0);
  }
}

}  // namespace

extern "C" int knf_volume_forward(knf_field_t f, const double* origins, const double* dirs, int64_t n_rays, int32_t n_s,
                                  const double* jitter, const double background[3], double s_param, double* colors, int mem,
                                  void* stream) {
  if (!f) return fail(KNF_E_INVALID, "null field handle");
  if (n_rays < 0 || (n_rays > 0 && (!origins || !dirs || !colors)) || !background)
    return fail(KNF_E_INVALID, "bad arguments to knf_volume_forward");
  if (n_s < 2) return fail(KNF_E_INVALID, "n_s must be >= 2");
  if (!(s_param > 0)) return fail(KNF_E_INVALID, "s must be > 0");
  if (n_rays == 0) return 0;
  if (n_rays * (int64_t)n_s > (int64_t)(INT32_MAX / 16)) return fail(KNF_E_INVALID, "too many samples for one call; split the ray batch");
  Field& F = f->f;
  std::lock_guard<std::mutex> lk(F.mu);
  cudaStream_t st = (cudaStream_t)stream;
  CallScope call_scope(F, st);
  KNF_TRY(call_scope.rc);
  const int B = (int)n_rays, m = n_s - 1;
  const size_t n_samples = (size_t)B * n_s, n_int = (size_t)B * m;

  // staging (host mode) through the handle's stage buffers
  DevBuf* stg = F.ws.stage;
  const double *d_o = origins, *d_d = dirs, *d_j = jitter;
  double* d_col = colors;
  if (mem == KNF_MEM_HOST) {
    KNF_TRY(stg[0].ensure((size_t)B * 24));
    KNF_TRY(stg[1].ensure((size_t)B * 24));
    KNF_TRY(stg[3].ensure((size_t)B * 24));
    KNF_CUDA(cudaMemcpyAsync(stg[0].p, origins, (size_t)B * 24, cudaMemcpyHostToDevice, st));
    KNF_CUDA(cudaMemcpyAsync(stg[1].p, dirs, (size_t)B * 24, cudaMemcpyHostToDevice, st));
    d_o = stg[0].as<double>();
    d_d = stg[1].as<double>();
    d_col = stg[3].as<double>();
    if (jitter) {
      KNF_TRY(stg[2].ensure(n_samples * 8));
      KNF_CUDA(cudaMemcpyAsync(stg[2].p, jitter, n_samples * 8, cudaMemcpyHostToDevice, st));
      d_j = stg[2].as<double>();
    }
  }

  Workspace& W = F.ws;
  KNF_TRY(ensure_requests(F, n_samples));
  KNF_TRY(W.t_near.ensure((size_t)B * 8));
  KNF_TRY(W.t_far.ensure((size_t)B * 8));
  KNF_TRY(W.hit.ensure((size_t)B));
  KNF_TRY(W.sdf_out.ensure(n_samples * kSdfOut * sizeof(float)));
  KNF_TRY(W.normals64.ensure(n_int * 24));
  KNF_TRY(W.hit_list.ensure(n_int * 4));
  KNF_TRY(W.hit_count.ensure(16));
  KNF_TRY(W.origins.ensure(n_int * 24));   // compacted near-sample positions
  KNF_TRY(W.dirs.ensure(n_int * 24));      // their FD normals
  KNF_TRY(W.phase.ensure(n_int));          // ok flags
  KNF_TRY(W.col_v.ensure(n_int * 3 * sizeof(float)));
  KNF_TRY(W.col_n.ensure(n_int * 3 * sizeof(float)));
  KNF_TRY(W.col_z.ensure(n_int * kFeat * sizeof(float)));
  KNF_TRY(W.rgb.ensure(n_int * 3 * sizeof(float)));

  VolArgs V{d_o, d_d, d_j, B, n_s, W.t_near.as<double>(), W.t_far.as<double>()};
  unsigned char* active = W.hit.as<unsigned char>();
  vol_box_kernel<<<blocks_for((size_t)B), 256, 0, st>>>(V, F.geom, active);
  // 1. SDF + features at every sample
  RouteBuffers R = route_buffers(F, 2, -1);
  R.eval_counter = stat_counter(F, 0);
  vol_emit_kernel<<<blocks_for(n_samples), 256, 0, st>>>(R, F.geom, V, active);
  KNF_TRY(launch_scan_scatter(F, R, n_samples, st));
  KNF_TRY(launch_sdf_mlp(F, R, n_samples, nullptr, W.sdf_out.as<float>(), st));
  // 2. FD normals where the sample can influence the pixel
  KNF_CUDA(cudaMemsetAsync(W.hit_count.p, 0, 16, st));
  vol_near_kernel<<<blocks_for(n_int), 256, 0, st>>>(V, active, W.sdf_out.as<float>(), s_param, W.hit_list.as<int>(),
                                                    W.hit_count.as<int>(), W.origins.as<double>(), W.normals64.as<double>());
  int n_near = 0;
  KNF_CUDA(cudaMemcpyAsync(F.host_poll, W.hit_count.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  KNF_CUDA(cudaStreamSynchronize(st));
  n_near = *F.host_poll;
  F.stats.kernel_launches += 3;
  if (n_near > 0) {
    // shade_points_device re-uses ws.sdf_out for its probes: keep the sample outputs in a second buffer
    KNF_TRY(W.colors64.ensure(n_samples * kSdfOut * sizeof(float)));
    KNF_CUDA(cudaMemcpyAsync(W.colors64.p, W.sdf_out.p, n_samples * kSdfOut * sizeof(float), cudaMemcpyDeviceToDevice, st));
    ShadeTargets T;
    T.normals = W.dirs.as<double>();
    T.ok = W.phase.as<unsigned char>();
    T.eps = 1e-8;
    KNF_TRY(shade_points_device(F, W.origins.as<double>(), nullptr, n_near, T, st));
    vol_near_apply_kernel<<<blocks_for((size_t)n_near), 256, 0, st>>>(W.hit_list.as<int>(), n_near, W.dirs.as<double>(),
                                                                     W.phase.as<unsigned char>(), W.normals64.as<double>());
  }
  const float* sdf_samples = n_near > 0 ? W.colors64.as<float>() : W.sdf_out.as<float>();
  // 3. colour at the left sample of every interval
  RouteBuffers Rc = route_buffers(F, 3, -1);
  Rc.eval_counter = stat_counter(F, 1);
  vol_color_emit_kernel<<<blocks_for(n_int), 256, 0, st>>>(Rc, F.geom, V, active, sdf_samples, W.normals64.as<double>(),
                                                          W.col_v.as<float>(), W.col_n.as<float>(), W.col_z.as<float>());
  KNF_TRY(launch_scan_scatter(F, Rc, n_int, st));
  KNF_TRY(launch_col_mlp(F, Rc, n_int, W.col_v.as<float>(), W.col_n.as<float>(), W.col_z.as<float>(), W.rgb.as<float>(), st));
  // 4. composite
  vol_composite_kernel<<<blocks_for((size_t)B), 256, 0, st>>>(V, active, sdf_samples, W.rgb.as<float>(), s_param, background[0],
                                                             background[1], background[2], d_col);
  F.stats.kernel_launches += 3;
  KNF_CUDA(cudaGetLastError());
  if (mem == KNF_MEM_HOST) {
    KNF_CUDA(cudaMemcpyAsync(colors, d_col, (size_t)B * 24, cudaMemcpyDeviceToHost, st));
    KNF_CUDA(cudaStreamSynchronize(st));
  }
  return 0;
}
