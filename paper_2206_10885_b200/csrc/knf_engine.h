// knf_engine.h -- host-side engine behind the C-ABI: field handle, workspace, and the device
// drivers (route -> MLP, wavefront march, shade) shared by knf_api.cu and knf_pathtrace.cu.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "knf_common.cuh"
#include "knf_route.cuh"

namespace knf {

struct LipCellConst;  // knf_bounds.cuh

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define KNF_CUDA(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
  } while (0)

// A lazily grown device allocation.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes);  // 0 or KNF_E_*
  void release();
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct Workspace {
  // routing
  DevBuf req_pt, req_cell, req_rank, perm, tiles;
  DevBuf req_pt1, req_cell1, req_rank1;  // second request list: the fused march kernel reads one list while filling the other
  DevBuf req_pt2, req_cell2, req_rank2, req_pt3, req_cell3, req_rank3;  // the decision filter's two request lists
  DevBuf sorted;                         // march queues: (point, ray) per sorted position
  DevBuf cell_count_f;                   // per-cell request counts of the filter queue
  DevBuf sorted_f, tiles_f, cell_offset_f, tile_base_f;  // the filter queue's own sorted view and tile list: its tile kernel runs
                                         // concurrently with the exact queue's (two streams), so the two cannot share them
  DevBuf live2, live3;
  DevBuf cell_count, cell_offset, tile_base;
  DevBuf counters;  // RouteCounters[4] + stats counters
  // march state
  DevBuf t, t_prev, d_prev, t_conv, d_conv, t_hit, steps, phase, hit, live0, live1;
  // shading
  DevBuf tail_cursor, scan_part;
  DevBuf hit_list, hit_count, sdf_out, col_v, col_n, col_z, rgb;
  // render-frame ray buffers
  DevBuf origins, dirs, t_near, t_far, normals64, colors64;
  DevBuf frame_color, frame_depth, frame_normal, frame_hit;  // knf_render_pass_u8 intermediates
  // host staging (KNF_MEM_HOST calls): input/output mirrors
  DevBuf stage[12];
  size_t req_cap = 0;
  size_t ray_cap = 0;
  void release_all();
};

struct Field {
  int device = 0;
  GridGeom geom{};
  int sdf_freqs = kSdfFreqs, dir_freqs = kDirFreqs, feature_dim = kFeat;
  float* sdf_blobs = nullptr;
  float* col_blobs = nullptr;
  uint32_t* sdf_mma_blobs = nullptr;   // knf_mma.cuh MmaBlobT<3> per cell (bf16 x 3 B fragments)
  uint32_t* sdf_mmah_blobs = nullptr;  // MmaBlobT<2> per cell (fp16 x 2 B fragments); null when a weight exceeds the fp16 range
  uint8_t* sdf_tc5_blobs = nullptr;    // knf_tc5.cuh Tc5Blob per cell (fp16 x 2 pieces as tcgen05 B operands); null when !fp16_ok
  int filter_kernel = 1;               // decision filter kernel: 1 = march_tc5_kernel (tcgen05 / TMEM), 0 = march_mma_kernel<2, true> (mma.sync); KNF_FILTER_KERNEL
  bool fp16_ok = false;
  double filter_delta_max = 0.0;       // largest FINITE per-cell decision-filter bound (knf_api.cu filter_delta)
  float filter_x_raw = 0.0f;           // coordinate magnitude the bounds were derived for (1.001 x the box's largest |coordinate|)
  // sub-box refinement of the per-cell Lipschitz bounds behind certified skipping (knf_bounds.cuh): run on the device the
  // first time a march uses the decision filter; until then (and wherever it is no tighter) the closed-form bounds apply
  LipCellConst* lip_consts = nullptr;        // device, per cell
  float* lip_cur = nullptr;                  // device, [n_cells][3]: the bounds the filter kernels currently read
  unsigned long long* lip_max = nullptr;     // device, [n_cells][3]: the refinement's running maxima
  std::vector<float> lip_closed_form;        // host copy of the closed-form bounds
  bool lip_refined = false;
  double lip_width = 0.004;                  // target sub-box width (KNF_LIP_WIDTH; 0: keep the closed-form bounds)
  int lip_fine = 2;                          // Taylor samples per sub-box interval (KNF_LIP_FINE, 1..4)
  float lip_ms = 0.f;                        // device time of the refinement (0 until it has run with profiling on)
  int filter_cells_off = 0;            // cells whose activations can leave the fp16 range: delta = +inf, the filter decides nothing there
  int sparse_max_inner = 8;            // residency cap and keep rule of sparse exact wavefronts (KNF_SPARSE_INNER / KNF_SPARSE_KEEP)
  int sparse_keep_div = 2;   // measured: (16, 4) gains 3 % on the distilled frame and loses 1.3 % on the random-init one; (32, 8) and up lose more
  int sparse_div = 6;                  // a wavefront is sparse when its exact queue holds < n / sparse_div rays (KNF_SPARSE_DIV; 8 until round 2b: 6 / 4 / 3 take 3 % off the trained 16^3 frame and leave the others unchanged)
  bool sparse_small_kernel = true;     // exact march: sparse wavefronts by march_small_kernel (KNF_SPARSE_SMALL=0 disables)
  bool exact_mid = true;               // dense exact wavefronts by march_mid_kernel (32-request tiles, 13 CTAs per SM) instead of march_warp_kernel (KNF_EXACT_MID=0)
  int scan_split = 65536;              // grids with more cells scan in chunks over many CTAs (two launches) instead of one CTA per queue (KNF_SCAN_SPLIT)
  int filter_grid_ctas = 6;            // CTAs per SM the tcgen05 filter's grid asks for (KNF_FILTER_GRID; fewer leaves room for the concurrent exact kernel)
  int filter_skip_cap = 1 << 20;       // cap on the certified steps taken after one evaluation (KNF_FILTER_SKIP_CAP)
  int filter_skip = 2;                 // certified (Lipschitz) skipping inside the filter: 0 off, 1 sample by sample, 2 closed-form run (cell-exit DDA + Lipschitz budget) then sample by sample (the default since the refined bounds made runs long); KNF_FILTER_SKIP
  int filter_hint = 0;                 // auto mode: what the previous march on this handle learnt (0 unknown, 1 rays crawl, 2 they do not)
  int filter_mode = 2;                 // decision filter of the exact march: 0 off, 1 on, 2 auto (probe the first wavefront)
  int precision = 0;                  // KNF_PRECISION_*: which SDF tile kernels run
  Workspace ws;
  std::mutex mu;
  KnfStats stats{};
  bool smem_configured = false;
  // optional per-launch event timing
  bool profiling = false;
  std::vector<cudaEvent_t> events;
  struct Span {
    int kind;
    size_t e0, e1;
  };
  std::vector<Span> spans;
  size_t events_used = 0;
  size_t prof_last_end = (size_t)-1;  // event index of the last finished span (shared with the next span's start)
  void* prof_last_stream = nullptr;
  bool prof_chain = false;            // set by the march loop
  int* host_poll = nullptr;  // pinned; early-out polling of the march loop
  cudaStream_t side_stream = nullptr;    // the exact queue's tile kernels run here, beside the filter kernel on the caller's stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int tail_threshold = 24576;            // hand the march to march_tail_kernel (one warp per ray) once this few rays are live (twice as many when the tail can skip certified crawl steps); 0: never (KNF_TAIL)
  int exact_grid_ctas = 0;               // cap on the exact kernels' CTAs per SM while a filter pass runs beside them (KNF_EXACT_GRID; 0: none)
  bool exact_first = false;              // launch the exact queue's kernel before the filter's (KNF_EXACT_FIRST)
  int first_split_eighths = 0;           // with filter_first: this many of every 8 ray blocks start in the exact queue instead (KNF_FIRST_SPLIT)
  bool filter_first = true;              // first samples through the filter queue once the handle knows its rays crawl (KNF_FILTER_FIRST=0: always the exact queue)
  bool tail_skip = true;                 // certified skipping inside march_tail_kernel (KNF_TAIL_SKIP=0 disables)
  bool overlap_queues = true;            // KNF_OVERLAP=0: one stream, filter then exact (the round-1 schedule)
  cudaEvent_t last_call_done = nullptr;  // recorded at the end of every call (CallScope)
  void* last_call_stream = nullptr;
  bool last_call_valid = false;
  int march_max_inner = 8;    // tile-residency cap (steps in place per tile visit), exact / tensor march kernels
  int filter_keep_div = 2;    // the filter keeps stepping a tile in place while n_stay * this >= its size (KNF_FILTER_KEEP)
  int filter_max_inner = 12;  // ... of the decision-filter kernel (measured optimum: 8 -> 15.97 ms, 12 -> 15.80, 16 -> 16.06)
};

enum { SPAN_SDF_MLP = 0, SPAN_ROUTE = 1, SPAN_COLOR_MLP = 2, SPAN_OTHER = 3, SPAN_FILTER = 4 };
// RAII: records an event pair around the launches issued in its scope when F.profiling is set.
struct ProfScope {
  Field& F;
  cudaStream_t st;
  int kind;
  size_t e0 = 0;
  bool on;
  ProfScope(Field& f, cudaStream_t s, int k);
  ~ProfScope();
};
int collect_profile(Field& F);  // syncs; folds finished spans into F.stats

// ---- drivers (all asynchronous on `st`; pointers are device pointers) -------------------------
int ensure_requests(Field& F, size_t n_requests);
int ensure_rays(Field& F, size_t n_rays);
RouteBuffers route_buffers(Field& F, int counter_slot, int next_slot, int list = 0);  // list 0/1: exact queue, 2/3: filter queue
RouteCounters* counters(Field& F, int slot);
unsigned long long* stat_counter(Field& F, int which);  // 0 = sdf evals, 1 = colour evals
int begin_call(Field& F, cudaStream_t st);              // reset routing invariants (device already selected by CallScope)
// One API call on a field handle (the caller holds F.mu).  All scratch belongs to the handle but work is ordered only on
// the caller's stream, so a call on another stream than the previous one first waits (on the device) for that call's
// kernels: two torch streams or threads sharing a handle are serialised instead of racing on the workspace.  The
// thread's current device is saved and restored (a library call must not change torch.cuda.current_device()).
struct CallScope {
  Field& F;
  cudaStream_t st;
  int prev_device = -1;
  int rc = 0;
  CallScope(Field& f, cudaStream_t s);
  ~CallScope();
  CallScope(const CallScope&) = delete;
  CallScope& operator=(const CallScope&) = delete;
};
int finish_stats(Field& F, cudaStream_t st);            // pull device counters into F.stats (syncs)
int ensure_lipschitz_refined(Field& F, cudaStream_t st);  // knf_bounds.cuh, once per handle (asynchronous on `st`)

int launch_scan_scatter(Field& F, const RouteBuffers& R, size_t n_upper, cudaStream_t st, int* seg_cell = nullptr,
                        int* seg_start = nullptr, int* n_seg = nullptr);
int launch_sdf_mlp(Field& F, const RouteBuffers& R, size_t n_upper, float* out_first, float* out_full, cudaStream_t st);
int launch_col_mlp(Field& F, const RouteBuffers& R, size_t n_upper, const float* v, const float* nrm, const float* z,
                   float* rgb, cudaStream_t st);

int sdf_forward_device(Field& F, const float* pts, int64_t n, float* out_full, float* out_first, int* cell_out,
                       cudaStream_t st);
int color_forward_device(Field& F, const float* x, const float* v, const float* nrm, const float* z, int64_t n,
                         float* rgb, cudaStream_t st);

// surface.march_rays; optionally compacts the hit rays into ws.hit_list / ws.hit_count.
int march_device(Field& F, const double* o, const double* d, const double* t_near, const double* t_far, int64_t n,
                 const KnfSettings& s, unsigned char* hit, double* t, double* pos, int* steps, bool want_hit_list,
                 cudaStream_t st);

struct ShadeTargets {
  double* grad = nullptr;       // (m,3)
  double* normals = nullptr;    // (m,3)
  unsigned char* ok = nullptr;  // (m)
  double* colors = nullptr;     // (m,3); null => no colour pass
  bool fallback = false;        // degenerate normal -> -view_dir
  bool scatter_by_ray = false;  // write outputs at the ray index of the hit list instead of densely
  bool clip_colors = false;
  double eps = 1e-8;
};
// Shade explicit points (pts/dirs, m known) ...
int shade_points_device(Field& F, const double* pts, const double* dirs, int64_t m, const ShadeTargets& T,
                        cudaStream_t st);
// ... or the hits of the last march_device(want_hit_list=true) over rays (o, d); m_hits is the
// host copy of the hit count; [first_hit, first_hit + m_hits) selects a chunk of the hit list.
int shade_hits_device(Field& F, const double* o, const double* d, int64_t first_hit, int64_t m_hits,
                      const ShadeTargets& T, cudaStream_t st);
int read_hit_count(Field& F, cudaStream_t st, int* out);  // syncs the stream

}  // namespace knf

struct knf_field_s {
  knf::Field f;
};
