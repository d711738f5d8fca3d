/*
 * knf_b200.h -- C-ABI of libknf_b200.so: the B200-native (sm_100a) replacement for the
 * KiloNeuS render hot path of the reference package `kilofield`
 * (/root/reference/pkg/src/kilofield).  Plain pointers and sizes only; no torch types.
 *
 * Every entry point names the reference function it stands in for (file:line relative to
 * /root/reference/pkg/src/kilofield/).  INTEGRATION.md shows the ctypes binding a
 * reference maintainer would add.
 *
 * Conventions
 *   - return value: 0 on success, negative KNF_E_* on failure; knf_last_error() returns a
 *     thread-local message for the last failing call on this thread.
 *   - `mem` says where EVERY array argument of that call lives: KNF_MEM_DEVICE (device
 *     pointers on the field's GPU, nothing is copied, the call is asynchronous on `stream`)
 *     or KNF_MEM_HOST (ordinary host memory; the library stages host->device, runs, copies
 *     device->host and synchronises `stream` before returning).
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - arrays are C-contiguous; "(n,3) f64" means n rows of 3 doubles.
 *   - the library owns only the opaque handles and their internal scratch; callers own
 *     every buffer they pass.  A handle serialises concurrent calls internally, so it may be
 *     shared between host threads (reference contract: SPEC.md:190-191).
 *   - there is no CPU fallback: without a CUDA device every compute call fails with
 *     KNF_E_CUDA.
 */
#ifndef KNF_B200_H
#define KNF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNF_ABI_VERSION 2
#define KNF_PRECISION_DEFAULT 0 /* KNF_PRECISION_FP32_CHAIN */

enum {
  KNF_OK = 0,
  KNF_E_INVALID = -1,     /* contract violation -> Python ValueError (surface.py:72-75, grid.py:409) */
  KNF_E_UNSUPPORTED = -2, /* field architecture the kernels are not compiled for */
  KNF_E_CUDA = -3,        /* CUDA runtime / no device */
  KNF_E_IO = -4,          /* .knf file problems (modelio.py:30-47) */
  KNF_E_NOMEM = -5
};

enum { KNF_MEM_DEVICE = 0, KNF_MEM_HOST = 1 };

/* Arithmetic of the two hidden contractions of the SDF tile MLP (grid.grid_forward, grid.py:253-265).
 *   KNF_PRECISION_FP32_CHAIN     k-ordered fp32 FMA chain from zero + rounded bias add on the FP32 pipe:
 *                                bit-identical to the reference's OpenBLAS sgemm for cells with >= 47 rows.
 *   KNF_PRECISION_TENSOR_BF16X3  exact 3-way bf16 split of every fp32 operand, six piece products on the
 *                                tensor cores (mma.sync bf16 -> fp32): closer to the exact dot product than
 *                                the fp32 chain itself (mean |err| 4e-8 vs 1.2e-7), ~2x faster, but not
 *                                bit-identical to the chain.
 * All are deterministic and independent of batch composition.  The colour MLP always uses the chain.
 *   KNF_PRECISION_TENSOR_FP16X2  two fp16 pieces per operand (22-23 significand bits, second piece scaled by
 *                                2^11), three piece products: half the tensor work of BF16X3, about as accurate
 *                                as the fp32 chain itself (mean |err| 1e-7).  Needs |w| < 6e4 in the hidden layers.
 */
enum { KNF_PRECISION_FP32_CHAIN = 0, KNF_PRECISION_TENSOR_BF16X3 = 1, KNF_PRECISION_TENSOR_FP16X2 = 2 };

typedef struct knf_field_s* knf_field_t;
typedef struct knf_scene_s* knf_scene_t;

/* grid.py:32-154 GridConfig + MlpGrid stacks, exactly as the reference holds them in host
 * memory: weights[k] is (n_cells, out_k, in_k) row-major fp32, biases[k] is (n_cells, out_k). */
typedef struct {
  int32_t resolution;
  double bbox_min[3];
  double bbox_max[3];
  int32_t sdf_freqs;   /* L_x, 6 */
  int32_t dir_freqs;   /* L_v, 4 */
  int32_t feature_dim; /* F, 8 */
  double fd_step;      /* h, 1e-3 */
  const float* sdf_w[3];
  const float* sdf_b[3];
  const float* color_w[3];
  const float* color_b[3];
} KnfFieldDesc;

/* cameras.py:10-36 CameraPose */
typedef struct {
  double position[3];
  double rotation[9]; /* row-major 3x3, columns = right/up/back */
  double fov_y;
  int32_t width;
  int32_t height;
} KnfCamera;

/* surface.py:64-75 RenderSettings (render_pass is host-side only) */
typedef struct {
  double eps_hit;
  int32_t max_steps;
  double step_scale;
} KnfSettings;

/* device-side statistics of the last march/render call on a handle (for roofline accounting) */
typedef struct {
  int64_t sdf_evals;    /* SDF MLP evaluations issued (march + refinement + shading probes) */
  int64_t color_evals;  /* colour MLP evaluations */
  int64_t rays;         /* rays marched */
  int64_t hits;
  int64_t wavefronts;   /* march iterations executed */
  int64_t kernel_launches;
  /* filled only while profiling is enabled (knf_field_set_profiling): CUDA-event time of the
   * SDF tile-MLP launches and of the routing launches (emit/advance + scan + scatter) */
  int64_t sdf_mlp_launches;
  int64_t route_launches;
  double sdf_mlp_ms;
  double route_ms;
  double color_mlp_ms;
  double other_ms;
  int64_t march_lane_slots; /* 64 x tile passes of the fused march kernel: sdf march evals / this = tile fill */
  int64_t march_routed_requests; /* march evaluations that went through a global routing pass (the rest stepped in place) */
  /* decision filter of the exact march (knf_field_set_filter): tensor-core predicate evaluations, how many of them
   * could not be decided and were re-evaluated exactly, and (while profiling) the filter launches' CUDA-event time */
  int64_t filter_evals;
  int64_t filter_deferred;
  int64_t filter_skipped; /* march steps taken without any evaluation: certified by the cell's Lipschitz bound */
  int64_t filter_lane_slots; /* 16 x m-tiles the filter kernel computed: filter_evals / this = its tile fill */
  int64_t filter_launches;
  double filter_ms;
} KnfStats;

int knf_abi_version(void);
const char* knf_last_error(void);
/* number of CUDA devices visible, or KNF_E_CUDA */
int knf_device_count(void);

/* ---- field lifetime --------------------------------------------------------------------- */
/* Packs the stacks into cell-major, k-major blobs and uploads them to `device`
 * (replaces nothing in the reference: this is the one-time upload of grid.KiloField). */
int knf_field_create(const KnfFieldDesc* desc, int device, knf_field_t* out);
/* modelio.load_model (modelio.py:127-165) straight to the device layout;
 * same magic / version / truncation / CRC32 checks. */
int knf_field_create_from_knf(const char* path, int device, knf_field_t* out);
int knf_field_destroy(knf_field_t f);
/* fills the GridConfig part of `desc` (pointers are set to NULL) */
int knf_field_describe(knf_field_t f, KnfFieldDesc* desc);
/* Statistics accumulate over calls until reset.  knf_field_stats synchronises the device. */
int knf_field_stats(knf_field_t f, KnfStats* out);
int knf_field_stats_reset(knf_field_t f);
/* Bracket every kernel launch with CUDA events on the call's stream (adds ~1 us of host work per launch). */
int knf_field_set_profiling(knf_field_t f, int enable);
/* Select / query the KNF_PRECISION_* mode of the SDF tile kernels (grid.grid_forward's arithmetic).  A new
 * handle starts in the mode named by the environment variable KNF_PRECISION ("fp32_chain" | "tensor_bf16x3" | "tensor_fp16x2"),
 * default KNF_PRECISION_DEFAULT. */
int knf_field_set_precision(knf_field_t f, int mode);
int knf_field_get_precision(knf_field_t f);
/* Decision filter of surface.march_rays in KNF_PRECISION_FP32_CHAIN mode (surface.py:185-223).  A ray inside a
 * negative region advances by the fixed step scale * eps / 2 and the reference consults the distance there only
 * as the predicate d < -eps (plus, once, as d_prev of the secant step).  With the filter on, those predicates are
 * answered by a tensor-core evaluation with a per-cell error bound (forward error analysis over the cell's
 * weights with a measured model of the tensor-core accumulation); every sample it cannot decide, and
 * every value the reference uses as a number, is evaluated by the exact fp32 chain kernel.  Results are
 * bit-identical to filter off.  KNF_FILTER_AUTO probes the first wavefront and switches the filter off when fewer
 * than 1/8 of the live rays are in a negative region (always the case on a real surface).  Environment variable
 * KNF_FILTER ("off" | "on" | "auto") sets the initial mode of new handles; default auto. */
enum { KNF_FILTER_OFF = 0, KNF_FILTER_ON = 1, KNF_FILTER_AUTO = 2 };
int knf_field_set_filter(knf_field_t f, int mode);
/* largest per-cell bound |filter distance - exact distance| the field was packed with (for reports) */
double knf_field_filter_delta(knf_field_t f);
/* number of cells the filter is switched off for (bound = +inf): cells whose hidden activations could leave the
 * fp16 range of the tensor-core operand pieces (very large weights); their samples all go to the exact kernel */
int knf_field_filter_cells_off(knf_field_t f);
/* name of the decision-filter kernel this handle launches: "march_tc5_kernel" (tcgen05.mma, accumulators in tensor
 * memory; the default) or "march_mma_kernel<2, true>" (mma.sync; environment KNF_FILTER_KERNEL=mma).  For reports. */
const char* knf_field_filter_kernel(knf_field_t f);

/* Per-cell, per-axis Lipschitz bounds L_a >= sup |d d / d x_a| of the SDF network behind the decision filter's certified
 * skipping (no reference counterpart: the reference evaluates every crawl sample, surface.py:217-223; a sample p of a ray
 * in the cell of an evaluated sample p0 with sum_a L_a |p_a - p0_a| below the room the filter distance left has an exact
 * distance below -eps, so the reference's step there is taken without evaluating).  `closed_form` receives the bounds the
 * field was packed with (|w3| |W2| |W1 J_a|), `refined` the bounds after the sub-box bound propagation of
 * csrc/knf_bounds.cuh, which this call runs if no march has triggered it yet (both n_cells * 3 floats, HOST pointers,
 * either may be NULL); `refine_ms` (may be NULL) the device time of that refinement, 0 if it ran untimed earlier.
 * Environment: KNF_LIP_WIDTH (target sub-box width, default 0.004; 0 keeps the closed-form bounds), KNF_LIP_FINE.
 * KNF_E_UNSUPPORTED for a field without filter blobs. */
int knf_field_lipschitz(knf_field_t f, float* closed_form, float* refined, float* refine_ms, void* stream);

/* ---- routing: grid.py:176-213 ------------------------------------------------------------ */
/* grid.cell_index_flat (grid.py:182-185) on fp32 points (fp64 arithmetic, bit-exact). */
int knf_cell_index(knf_field_t f, const float* pts, int64_t n, int32_t* cell, int mem, void* stream);
/* same for fp64 points (grid.cell_index, grid.py:166-173, passes fp64 straight through). */
int knf_cell_index_f64(knf_field_t f, const double* pts, int64_t n, int32_t* cell, int mem, void* stream);
/* grid.route (grid.py:207-213): cell ids, a sort-by-cell permutation (`order[r]` = input row of
 * sorted row r; rows of one cell are contiguous, order inside a cell is unspecified), and the
 * occupied segments.  seg_cell/seg_start need room for min(n, n_cells) entries (+1 for
 * seg_start, which gets the closing n); *n_seg receives the count. Any output may be NULL. */
int knf_route(knf_field_t f, const float* pts, int64_t n, int32_t* cell, int32_t* order,
              int32_t* seg_cell, int32_t* seg_start, int32_t* n_seg, int mem, void* stream);

/* ---- batched multi-network forward: grid.py:373-409 -------------------------------------- */
/* grid.sdf_query (grid.py:373-380): out is (n, 1+F) fp32, column 0 = distance. */
int knf_sdf_forward(knf_field_t f, const float* pts, int64_t n, float* out, int mem, void* stream);
/* grid.sdf_values (grid.py:383-384): distances only. */
int knf_sdf_values(knf_field_t f, const float* pts, int64_t n, float* dist, int mem, void* stream);
/* grid.color_query (grid.py:387-400): x,v,nrm (n,3) fp32, z (n,F) fp32 -> rgb (n,3) fp32. */
int knf_color_forward(knf_field_t f, const float* x, const float* v, const float* nrm, const float* z,
                      int64_t n, float* rgb, int mem, void* stream);

/* ---- encoder + activations as stand-alone operators: nn.py:26-93 ----------------------------- */
/* nn.fourier_encode (nn.py:66-93) for 3-vectors: x (n,3) fp32 -> out (n, 3 + 6*L) fp32, 0 <= L <= 8;
 * bit-exact with NumPy's fp32 sin/cos + double-angle recurrence for |pi*x| < 71476. */
int knf_fourier_encode(const float* x, int64_t n, int32_t L, float* out, int device, int mem, void* stream);
/* nn.softplus / nn.sigmoid (nn.py:26-38), elementwise on fp32: the device routines the MLP kernels use. */
int knf_softplus(const float* x, int64_t n, float* out, int device, int mem, void* stream);
int knf_sigmoid(const float* x, int64_t n, float* out, int device, int mem, void* stream);

/* north_star subsystem 2 ("also emits the SDF gradient"): the ANALYTIC gradient of the owning cell's SDF network at each
 * fp32 point, by forward-mode differentiation through nn.fourier_encode and the softplus layers (no reference
 * counterpart: grid.grad_fd, grid.py:440-451, is a global finite difference and stays the parity path).  dist (n) may
 * be NULL; grad is (n,3) fp32. */
int knf_sdf_gradient(knf_field_t f, const float* pts, int64_t n, float* dist, float* grad, int mem, void* stream);

/* ---- FD normals: grid.py:416-461 ---------------------------------------------------------- */
/* grid.grad_fd (grid.py:440-451): pts (n,3) f64 -> grad (n,3) f64. */
int knf_fd_gradient(knf_field_t f, const double* pts, int64_t n, double* grad, int mem, void* stream);
/* grid.normal_batch (grid.py:454-461): unit normals or zeros, ok mask. */
int knf_fd_normals(knf_field_t f, const double* pts, int64_t n, double eps, double* nrm, uint8_t* ok,
                   int mem, void* stream);

/* ---- rays: cameras.py:57-76, surface.py:131-149 ------------------------------------------- */
/* cameras.pixel_rays: pixel_xy (n,2) int32 (col,row) or NULL for the full raster (n = W*H);
 * jitter (n,2) f64 or NULL for pixel centres. */
int knf_pixel_rays(const KnfCamera* cam, const int32_t* pixel_xy, const double* jitter, int64_t n,
                   double* origins, double* dirs, int device, int mem, void* stream);
/* surface.ray_aabb_batch. */
int knf_ray_aabb(const double* origins, const double* dirs, int64_t n, const double bbox_min[3],
                 const double bbox_max[3], double* t_near, double* t_far, uint8_t* hit, int device, int mem,
                 void* stream);

/* ---- sphere tracing + shading: surface.py:82-99, 162-258 ---------------------------------- */
/* surface.march_rays(FieldSurface(field), ...): hit (n) u8, t (n) f64, position (n,3) f64,
 * steps (n) i32.  position/steps may be NULL. */
int knf_march(knf_field_t f, const double* origins, const double* dirs, const double* t_near,
              const double* t_far, int64_t n, const KnfSettings* s, uint8_t* hit, double* t, double* position,
              int32_t* steps, int mem, void* stream);
/* FieldSurface.shade (surface.py:93-99): FD normals (fallback -view_dir), feature re-query,
 * colour MLP.  colors/normals (n,3) f64. */
int knf_shade(knf_field_t f, const double* pts, const double* view_dirs, int64_t n, double* colors,
              double* normals, int mem, void* stream);
/* surface.trace_and_shade (surface.py:229-241): AABB -> march -> shade; colours clipped to
 * [0,1], zeros at misses. */
int knf_trace_and_shade(knf_field_t f, const double* origins, const double* dirs, int64_t n,
                        const KnfSettings* s, uint8_t* hit, double* t, double* position, int32_t* steps,
                        double* normals, double* colors, int mem, void* stream);

/* ---- frame driver: surface.py:273-336 ------------------------------------------------------ */
/* Rows [row0,row1) of surface.render_frame: ray generation, AABB, march, shade, background
 * composite and supersample reduction, all on the device.  Buffers cover ONLY the requested
 * rows: color (rows,W,3) f32, depth (rows,W) f32 (+inf at misses), normal (rows,W,3) f32,
 * hit (rows,W) u8. */
int knf_render_frame(knf_field_t f, const KnfCamera* cam, const KnfSettings* s, const double background[3],
                     int supersample, int row0, int row1, float* color, float* depth, float* normal,
                     uint8_t* hit, int mem, void* stream);

/* ---- next rows: the interactive caller and the mesh-sampling caller ------------------- */
enum { KNF_PASS_COLOR = 0, KNF_PASS_NORMAL = 1, KNF_PASS_DEPTH = 2 };
/* 8(f).2 service._render_once (service.py:279-288): render_frame -> surface.pass_image (surface.py:339-350)
 * -> images.to_uint8 (images.py:15-17) on the device; rgb is (rows,W,3) u8. */
int knf_render_pass_u8(knf_field_t f, const KnfCamera* cam, const KnfSettings* s, const double background[3],
                       int supersample, int render_pass, int row0, int row1, uint8_t* rgb, int mem, void* stream);
/* images.to_uint8 of an fp64 image after clip(img / divisor, 0, 1) and, if gamma22, ** (1/2.2)
 * (the progressive path-trace display transform, service.py:297-299). */
int knf_tonemap_u8(const double* img, int64_t n, double divisor, int gamma22, uint8_t* out, int device, int mem, void* stream);
/* 8(f).4 mesh._sample_volume (mesh.py:43-57): fp32 SDF values on the R^3 np.linspace lattice of
 * [bbox_min, bbox_max], "ij" order (x slowest); values has R^3 entries. */
int knf_sample_volume(knf_field_t f, int32_t resolution, const double bbox_min[3], const double bbox_max[3], float* values,
                      int mem, void* stream);

/* 8(f).3 training._volume_forward (training.py:330-415), forward only: S-density volume rendering of a ray
 * batch with n_s stratified samples per ray.  jitter (n_rays,n_s) f64 in [0,1) or NULL for 0.5; s_param =
 * exp(inv_std_param); colors (n_rays,3) f64 in [0,1]. */
int knf_volume_forward(knf_field_t f, const double* origins, const double* dirs, int64_t n_rays, int32_t n_s,
                       const double* jitter, const double background[3], double s_param, double* colors, int mem,
                       void* stream);

/* ---- path tracer: pathtrace.py -------------------------------------------------------------- */
enum { KNF_OBJ_SPHERE = 0, KNF_OBJ_QUAD = 1, KNF_OBJ_BOX = 2, KNF_OBJ_NEURAL = 3 };
enum { KNF_MAT_LAMBERTIAN = 0, KNF_MAT_EMISSIVE = 1 };

/* One entry of pathtrace.Scene.objects (pathtrace.py:115-280), in scene order. */
typedef struct {
  int32_t kind;
  int32_t material;  /* analytic objects only */
  double rgb[3];     /* albedo or radiance */
  /* sphere: a = centre, s = radius.  quad: a = corner, b = edge_u, c = edge_v.
   * box: a = bmin, b = bmax.  neural: a = translation, rot = rotation (row-major), s = scale. */
  double a[3];
  double b[3];
  double c[3];
  double rot[9];
  double s;
  knf_field_t field;    /* neural only */
  KnfSettings settings; /* neural only */
} KnfObject;

/* pathtrace.Scene with a ConstantEnv (pathtrace.py:76-84, 277-280). */
int knf_scene_create(const KnfObject* objects, int32_t n_objects, const double env_rgb[3], int device,
                     knf_scene_t* out);
int knf_scene_destroy(knf_scene_t sc);
/* pathtrace.Rng.uniform (pathtrace.py:37-49), bit-exact: u[i] = hash(seed, pixel[i], sample[i], slot[i]). */
int knf_rng_uniform(uint64_t seed, const uint64_t* pixel, const uint64_t* sample, const uint64_t* slot,
                    int64_t n, double* u, int device, int mem, void* stream);
/* pathtrace.sample_lambertian (pathtrace.py:287-304) with teacher.orthonormal_tangents (teacher.py:302-309):
 * normals (n,3), u1/u2 (n) -> dirs (n,3), pdf (n, nullable). */
int knf_sample_lambertian(const double* normals, const double* u1, const double* u2, int64_t n, double* dirs, double* pdf,
                          int device, int mem, void* stream);
/* pathtrace.intersect_scene (pathtrace.py:311-330): nearest hit over all objects; t = +inf and obj = -1 on a miss. */
int knf_intersect_scene(knf_scene_t sc, const double* origins, const double* dirs, int64_t n, double t_max, double* t,
                        int32_t* obj, int mem, void* stream);
/* Rows [row0,row1) of pathtrace.render_pathtraced (pathtrace.py:436-471): hdr (rows,W,3) f64 mean
 * radiance over samples sample_offset .. sample_offset+spp-1. */
int knf_pathtrace(knf_scene_t sc, const KnfCamera* cam, int32_t spp, uint64_t seed, int32_t max_bounces,
                  int32_t sample_offset, int row0, int row1, double* hdr, int mem, void* stream);
/* pathtrace._trace_batch (pathtrace.py:340-420) for caller-supplied rays (trace_path is n = 1). */
int knf_trace_paths(knf_scene_t sc, const double* origins, const double* dirs, const uint64_t* pixel_ids,
                    int64_t n, uint64_t sample, uint64_t seed, int32_t max_bounces, double* radiance, int mem,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KNF_B200_H */
