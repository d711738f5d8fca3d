// knf_engine.cu -- workspace management and the device drivers: routing -> tile MLP, the wavefront
// sphere-trace loop, and shading.  Everything here is stream-ordered; nothing synchronises except
// read_hit_count / finish_stats.
#include "knf_engine.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "knf_march.cuh"
#include "knf_mlp.cuh"
#include "knf_mma.cuh"
#include "knf_rays.cuh"
#include "knf_tail.cuh"
#include "knf_tc5.cuh"
#include "knf_bounds.cuh"

namespace knf {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }
const std::string& last_error() { return g_error; }
int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_error = std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what;
  cudaGetLastError();  // clear sticky-less errors
  return KNF_E_CUDA;
}

int DevBuf::ensure(size_t bytes) {
  if (bytes <= cap) return 0;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  size_t want = bytes + bytes / 8 + 256;
  cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return fail(KNF_E_NOMEM, std::string("cudaMalloc of ") + std::to_string(want) + " bytes failed: " + cudaGetErrorString(e));
  }
  cap = want;
  return 0;
}
void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
}

void Workspace::release_all() {
  DevBuf* all[] = {&scan_part, &tail_cursor, &sorted_f, &tiles_f, &cell_offset_f, &tile_base_f, &req_pt2, &req_cell2, &req_rank2, &req_pt3, &req_cell3, &req_rank3, &cell_count_f, &sorted, &live2, &live3, &tile_base, &req_pt1, &req_cell1, &req_rank1, &req_pt, &req_cell, &req_rank, &perm, &tiles, &cell_count, &cell_offset, &counters, &t, &t_prev,
                   &d_prev, &t_conv, &d_conv, &t_hit, &steps, &phase, &hit, &live0, &live1, &hit_list,
                   &hit_count, &sdf_out, &col_v, &col_n, &col_z, &rgb, &origins, &dirs, &t_near, &t_far, &normals64,
                   &colors64, &frame_color, &frame_depth, &frame_normal, &frame_hit};
  for (DevBuf* b : all) b->release();
  for (DevBuf& b : stage) b.release();
  req_cap = ray_cap = 0;
}

static inline int blocks_for(size_t n, int threads = 256) {
  size_t b = (n + threads - 1) / threads;
  return (int)std::max<size_t>(1, std::min<size_t>(b, 148 * 16));
}

#define KNF_TRY(expr)       \
  do {                      \
    int _rc = (expr);       \
    if (_rc != 0) return _rc; \
  } while (0)

constexpr int kRouteSlots = 6;    // 0/1 exact march queue (ping-pong), 2 SDF forward, 3 colour forward, 4/5 filter march queue
constexpr int kStatCounters = 32;  // see finish_stats; [16..25]: optional section cycles of march_tc5_kernel (-DKNF_TC5_TIMING)
constexpr size_t kCounterBytes = kRouteSlots * sizeof(RouteCounters) + kStatCounters * sizeof(unsigned long long);

int ensure_requests(Field& F, size_t n) {
  Workspace& W = F.ws;
  n = std::max<size_t>(n, 1024);
  if (n > (size_t)INT32_MAX / 16) return fail(KNF_E_INVALID, "request batch too large for 32-bit routing indices");
  KNF_TRY(W.req_pt.ensure(n * sizeof(float4)));
  KNF_TRY(W.req_cell.ensure(n * sizeof(int)));
  KNF_TRY(W.req_rank.ensure(n * sizeof(int)));
  KNF_TRY(W.perm.ensure(n * sizeof(int)));
  KNF_TRY(W.tiles.ensure((n / kSmallTile + (size_t)F.geom.n_cells + 2) * sizeof(Tile)));  // worst case: every tile holds <= 16 requests
  bool fresh = W.cell_count.p == nullptr;
  KNF_TRY(W.cell_count.ensure((size_t)F.geom.n_cells * sizeof(int)));
  KNF_TRY(W.cell_offset.ensure(((size_t)F.geom.n_cells + 1) * sizeof(int)));
  KNF_TRY(W.tile_base.ensure(((size_t)F.geom.n_cells + 1) * sizeof(int)));
  KNF_TRY(W.counters.ensure(kCounterBytes));
  if (fresh) {
    KNF_CUDA(cudaMemset(W.cell_count.p, 0, W.cell_count.cap));
    KNF_CUDA(cudaMemset(W.counters.p, 0, W.counters.cap));
  }
  W.req_cap = std::max(W.req_cap, n);
  return 0;
}

int ensure_rays(Field& F, size_t n) {
  Workspace& W = F.ws;
  n = std::max<size_t>(n, 1024);
  KNF_TRY(W.t.ensure(n * 8));
  KNF_TRY(W.t_prev.ensure(n * 8));
  KNF_TRY(W.d_prev.ensure(n * 8));
  KNF_TRY(W.t_conv.ensure(n * 8));
  KNF_TRY(W.d_conv.ensure(n * 8));
  KNF_TRY(W.t_hit.ensure(n * 8));
  KNF_TRY(W.steps.ensure(n * 4));
  KNF_TRY(W.phase.ensure(n));
  KNF_TRY(W.hit.ensure(n));
  KNF_TRY(W.live0.ensure(n * 4));
  KNF_TRY(W.live1.ensure(n * 4));
  KNF_TRY(W.req_pt1.ensure(n * sizeof(float4)));
  KNF_TRY(W.req_cell1.ensure(n * sizeof(int)));
  KNF_TRY(W.req_rank1.ensure(n * sizeof(int)));
  KNF_TRY(W.req_pt2.ensure(n * sizeof(float4)));
  KNF_TRY(W.req_cell2.ensure(n * sizeof(int)));
  KNF_TRY(W.req_rank2.ensure(n * sizeof(int)));
  KNF_TRY(W.req_pt3.ensure(n * sizeof(float4)));
  KNF_TRY(W.req_cell3.ensure(n * sizeof(int)));
  KNF_TRY(W.req_rank3.ensure(n * sizeof(int)));
  KNF_TRY(W.sorted.ensure(n * sizeof(float4)));
  KNF_TRY(W.sorted_f.ensure(n * sizeof(float4)));
  KNF_TRY(W.tiles_f.ensure((n / 32 + (size_t)F.geom.n_cells + 2) * sizeof(Tile)));  // filter tiles hold >= 32 requests except one per cell
  KNF_TRY(W.cell_offset_f.ensure(((size_t)F.geom.n_cells + 1) * sizeof(int)));
  KNF_TRY(W.tile_base_f.ensure(((size_t)F.geom.n_cells + 1) * sizeof(int)));
  KNF_TRY(W.live2.ensure(n * 4));
  KNF_TRY(W.live3.ensure(n * 4));
  {
    const bool fresh_f = W.cell_count_f.p == nullptr;
    KNF_TRY(W.cell_count_f.ensure((size_t)F.geom.n_cells * sizeof(int)));
    if (fresh_f) KNF_CUDA(cudaMemset(W.cell_count_f.p, 0, W.cell_count_f.cap));
  }
  KNF_TRY(W.hit_list.ensure(n * 4));
  KNF_TRY(W.hit_count.ensure(16));
  KNF_TRY(W.tail_cursor.ensure(16));
  W.ray_cap = std::max(W.ray_cap, n);
  return ensure_requests(F, n);
}

RouteCounters* counters(Field& F, int slot) { return F.ws.counters.as<RouteCounters>() + slot; }
unsigned long long* stat_counter(Field& F, int which) {
  return reinterpret_cast<unsigned long long*>(F.ws.counters.as<RouteCounters>() + kRouteSlots) + which;
}

RouteBuffers route_buffers(Field& F, int slot, int next_slot, int list) {
  Workspace& W = F.ws;
  RouteBuffers R;
  DevBuf* pts[4] = {&W.req_pt, &W.req_pt1, &W.req_pt2, &W.req_pt3};
  DevBuf* cells[4] = {&W.req_cell, &W.req_cell1, &W.req_cell2, &W.req_cell3};
  DevBuf* ranks[4] = {&W.req_rank, &W.req_rank1, &W.req_rank2, &W.req_rank3};
  R.req_pt = pts[list]->as<float4>();
  R.req_cell = cells[list]->as<int>();
  R.req_rank = ranks[list]->as<int>();
  R.cell_count = (list >= 2 ? W.cell_count_f : W.cell_count).as<int>();
  R.cell_offset = (list >= 2 ? W.cell_offset_f : W.cell_offset).as<int>();
  R.tile_base = (list >= 2 ? W.tile_base_f : W.tile_base).as<int>();
  R.perm = W.perm.as<int>();
  R.tiles = (list >= 2 ? W.tiles_f : W.tiles).as<Tile>();
  R.ctr = counters(F, slot);
  R.next_ctr = next_slot >= 0 ? counters(F, next_slot) : nullptr;
  R.eval_counter = nullptr;
  R.small_tiles = 0;
  R.sorted = nullptr;
  R.live = nullptr;
  return R;
}

CallScope::CallScope(Field& f, cudaStream_t s) : F(f), st(s) {
  if (cudaGetDevice(&prev_device) != cudaSuccess) {
    cudaGetLastError();
    prev_device = -1;
  }
  cudaError_t e = cudaSetDevice(F.device);
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "cudaSetDevice");
    return;
  }
  if (F.last_call_valid && F.last_call_stream != (void*)st) {
    e = cudaStreamWaitEvent(st, F.last_call_done, 0);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "cudaStreamWaitEvent");
      return;
    }
  }
  rc = begin_call(F, st);
}
CallScope::~CallScope() {
  if (!F.last_call_done && cudaEventCreateWithFlags(&F.last_call_done, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    F.last_call_done = nullptr;
  }
  if (F.last_call_done && cudaEventRecord(F.last_call_done, st) == cudaSuccess) {
    F.last_call_stream = (void*)st;
    F.last_call_valid = true;
  } else {
    cudaGetLastError();
    cudaStreamSynchronize(st);  // no event: fall back to finishing this call's work before the next one may start
    F.last_call_valid = false;
  }
  if (prev_device >= 0 && prev_device != F.device) cudaSetDevice(prev_device);
}

int begin_call(Field& F, cudaStream_t st) {
  F.prof_chain = false;
  KNF_TRY(ensure_requests(F, 1024));
  KNF_CUDA(cudaMemsetAsync(F.ws.cell_count.p, 0, (size_t)F.geom.n_cells * sizeof(int), st));
  KNF_CUDA(cudaMemsetAsync(F.ws.counters.p, 0, kRouteSlots * sizeof(RouteCounters), st));  // stat counters persist
  if (!F.smem_configured) {
    KNF_CUDA(cudaFuncSetAttribute(mlp_warp_kernel<kSdfIn, kSdfOut, kSdfOutPad, ACT_SOFTPLUS, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SdfKernelSmem)));
    KNF_CUDA(cudaFuncSetAttribute(mlp_warp_kernel<kColIn, kColOut, kColOutPad, ACT_RELU, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ColKernelSmem)));
    KNF_CUDA(cudaFuncSetAttribute(march_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(SdfKernelSmem)));
    KNF_CUDA(cudaFuncSetAttribute(march_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SdfSmallSmem)));
    KNF_CUDA(cudaFuncSetAttribute(march_mid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SdfMidSmem)));
    KNF_CUDA(cudaFuncSetAttribute(march_mid_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    KNF_CUDA(cudaFuncSetAttribute(march_mma_kernel<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MmaMarchSmemT<3>)));
    KNF_CUDA(cudaFuncSetAttribute(sdf_mma_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MmaSmemT<3>)));
    KNF_CUDA(cudaFuncSetAttribute(march_mma_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MmaMarchSmemT<2>)));
    KNF_CUDA(cudaFuncSetAttribute(march_mma_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MmaMarchSmemT<2>)));
    KNF_CUDA(cudaFuncSetAttribute(sdf_mma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MmaSmemT<2>)));
    KNF_CUDA(cudaFuncSetAttribute(march_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Tc5MarchSmem)));
    KNF_CUDA(cudaFuncSetAttribute(march_tc5_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));  // several 40 KB CTAs per SM
    KNF_CUDA(cudaFuncSetAttribute(sdf_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Tc5FwdSmem)));
    KNF_CUDA(cudaFuncSetAttribute(sdf_tc5_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    if (!F.host_poll) KNF_CUDA(cudaMallocHost(&F.host_poll, 64));
    if (!F.side_stream) {
      KNF_CUDA(cudaStreamCreateWithFlags(&F.side_stream, cudaStreamNonBlocking));
      KNF_CUDA(cudaEventCreateWithFlags(&F.ev_fork, cudaEventDisableTiming));
      KNF_CUDA(cudaEventCreateWithFlags(&F.ev_join, cudaEventDisableTiming));
    }
    F.smem_configured = true;
  }
  return 0;
}

static cudaEvent_t next_event(Field& F) {
  if (F.events_used == F.events.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    F.events.push_back(e);
  }
  return F.events[F.events_used++];
}
ProfScope::ProfScope(Field& f, cudaStream_t s, int k) : F(f), st(s), kind(k), on(f.profiling) {
  if (!on) return;
  // back-to-back scopes on one stream share an event: the previous scope's end is this scope's start
  if (F.prof_chain && F.prof_last_end != (size_t)-1 && F.prof_last_stream == (void*)st) {
    e0 = F.prof_last_end;
  } else {
    e0 = F.events_used;
    cudaEventRecord(next_event(F), st);
  }
}
ProfScope::~ProfScope() {
  if (!on) return;
  size_t e1 = F.events_used;
  cudaEventRecord(next_event(F), st);
  F.spans.push_back({kind, e0, e1});
  F.prof_last_end = e1;
  F.prof_last_stream = (void*)st;
}
int collect_profile(Field& F) {
  KNF_CUDA(cudaDeviceSynchronize());
  for (const Field::Span& sp : F.spans) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, F.events[sp.e0], F.events[sp.e1]) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    switch (sp.kind) {
      case SPAN_SDF_MLP: F.stats.sdf_mlp_ms += ms; F.stats.sdf_mlp_launches += 1; break;
      case SPAN_ROUTE: F.stats.route_ms += ms; F.stats.route_launches += 1; break;
      case SPAN_COLOR_MLP: F.stats.color_mlp_ms += ms; break;
      case SPAN_FILTER: F.stats.filter_ms += ms; F.stats.filter_launches += 1; break;
      default: F.stats.other_ms += ms; break;
    }
  }
  F.spans.clear();
  F.events_used = 0;
  F.prof_last_end = (size_t)-1;
  return 0;
}

int finish_stats(Field& F, cudaStream_t st) {
  unsigned long long host[kStatCounters] = {};
  KNF_CUDA(cudaMemcpyAsync(host, stat_counter(F, 0), sizeof(host), cudaMemcpyDeviceToHost, st));
  KNF_CUDA(cudaStreamSynchronize(st));
  F.stats.sdf_evals = (int64_t)host[0];
  F.stats.color_evals = (int64_t)host[1];
  F.stats.march_lane_slots = (int64_t)host[2];
  F.stats.march_routed_requests = (int64_t)host[3];
  F.stats.filter_evals = (int64_t)host[4];
  F.stats.filter_deferred = (int64_t)host[5];
  F.stats.filter_skipped = (int64_t)host[6];
  F.stats.filter_lane_slots = (int64_t)host[7];
  if (std::getenv("KNF_DEBUG_TAIL"))
    fprintf(stderr, "march_tail_kernel since the last stats reset: %llu rays, %llu evaluations\n", host[9], host[8]);
#ifdef KNF_TC5_TIMING
  {
    static const char* names[10] = {"tile setup", "encode+split+store", "barriers", "layer-1 MMA wait", "h1 epilogue", "layer-2 MMA wait", "h2 epilogue+output",
                                    "march step+skip", "emit", "loop top"};
    double tot = 0;
    for (int i = 0; i < 10; i++) tot += (double)host[16 + i];
    fprintf(stderr, "march_tc5_kernel warp-cycles by section (total %.3g):", tot);
    for (int i = 0; i < 10; i++) fprintf(stderr, " %s %.1f%% |", names[i], 100.0 * (double)host[16 + i] / (tot > 0 ? tot : 1));
    fprintf(stderr, "\n");
  }
#endif
  return 0;
}

// grids beyond scan_split cells: the scan runs over <= 1024 chunks of >= 4096 cells in two launches (knf_route.cuh)
static inline void scan_chunks(const Field& F, int& chunks, int& chunk) {
  const int n = F.geom.n_cells;
  chunk = std::max(std::min(4096, F.scan_split > 0 ? F.scan_split : 4096), (n + kScanThreads - 1) / kScanThreads);
  chunks = (n + chunk - 1) / chunk;
}

int launch_scan_scatter(Field& F, const RouteBuffers& R, size_t n_upper, cudaStream_t st, int* seg_cell, int* seg_start,
                        int* n_seg) {
  ProfScope prof(F, st, SPAN_ROUTE);
  if (F.geom.n_cells > F.scan_split) {
    int chunks, chunk;
    scan_chunks(F, chunks, chunk);
    KNF_TRY(F.ws.scan_part.ensure(2 * (size_t)chunks * sizeof(ScanPart)));
    route_scan_part_kernel<<<dim3(chunks, 1), kScanThreads, 0, st>>>(R, R, F.geom.n_cells, chunk, F.ws.scan_part.as<ScanPart>());
    route_scan_apply_kernel<<<dim3(chunks, 1), kScanThreads, 0, st>>>(R, R, F.geom.n_cells, chunk, F.ws.scan_part.as<ScanPart>(), seg_cell, seg_start, n_seg);
    F.stats.kernel_launches += 1;
  } else
  route_scan_kernel<<<1, kScanThreads, 0, st>>>(R, F.geom.n_cells, seg_cell, seg_start, n_seg);
  route_scatter_kernel<<<blocks_for(std::max<size_t>(n_upper, (size_t)F.geom.n_cells)), 256, 0, st>>>(R, F.geom.n_cells);
  F.stats.kernel_launches += 2;
  KNF_CUDA(cudaGetLastError());
  return 0;
}

// scan + scatter of the two queues of one march wavefront in two launches instead of four
static int launch_scan_scatter2(Field& F, const RouteBuffers& Ra, const RouteBuffers& Rb, size_t n_upper, cudaStream_t st) {
  ProfScope prof(F, st, SPAN_ROUTE);
  if (F.geom.n_cells > F.scan_split) {
    int chunks, chunk;
    scan_chunks(F, chunks, chunk);
    KNF_TRY(F.ws.scan_part.ensure(2 * (size_t)chunks * sizeof(ScanPart)));
    route_scan_part_kernel<<<dim3(chunks, 2), kScanThreads, 0, st>>>(Ra, Rb, F.geom.n_cells, chunk, F.ws.scan_part.as<ScanPart>());
    route_scan_apply_kernel<<<dim3(chunks, 2), kScanThreads, 0, st>>>(Ra, Rb, F.geom.n_cells, chunk, F.ws.scan_part.as<ScanPart>(), nullptr, nullptr, nullptr);
    F.stats.kernel_launches += 1;
  } else
  route_scan2_kernel<<<2, kScanThreads, 0, st>>>(Ra, Rb, F.geom.n_cells);
  route_scatter2_kernel<<<blocks_for(std::max<size_t>(n_upper, (size_t)F.geom.n_cells)), 256, 0, st>>>(Ra, Rb, F.geom.n_cells);
  F.stats.kernel_launches += 2;
  KNF_CUDA(cudaGetLastError());
  return 0;
}

static inline int mlp_grid(const Field& F, size_t n_upper, int ctas_per_sm = kWarpCtasPerSm) {
  size_t tiles_upper = n_upper / kSmallTile + std::min<size_t>(n_upper, (size_t)F.geom.n_cells) + 1;
  return (int)std::max<size_t>(1, std::min<size_t>(tiles_upper, (size_t)148 * ctas_per_sm));
}

// tile shape of the batched SDF forward: 128-request tiles for the tcgen05 kernel of KNF_PRECISION_TENSOR_FP16X2
static inline int sdf_forward_tile_mode(const Field& F) {
  return (F.precision == KNF_PRECISION_TENSOR_FP16X2 && F.sdf_tc5_blobs && F.filter_kernel == 1) ? 3 : 0;
}

int launch_sdf_mlp(Field& F, const RouteBuffers& R, size_t n_upper, float* out_first, float* out_full, cudaStream_t st) {
  MlpParams P{};
  P.blobs = F.sdf_blobs;
  P.perm = R.perm;
  P.tiles = R.tiles;
  P.ctr = R.ctr;
  P.req_pt = R.req_pt;
  P.out_first = out_first;
  P.out_full = out_full;
  ProfScope prof(F, st, SPAN_SDF_MLP);
  if (F.precision == KNF_PRECISION_TENSOR_BF16X3) {
    P.blobs = reinterpret_cast<const float*>(F.sdf_mma_blobs);
    sdf_mma_kernel<3><<<mlp_grid(F, n_upper, kMmaCtasPerSm), 32, sizeof(MmaSmemT<3>), st>>>(P);
  } else if (F.precision == KNF_PRECISION_TENSOR_FP16X2 && R.small_tiles == 3) {
    // routed in tiles of <= 128 (launch_scan_scatter callers pass small_tiles = 3 for this mode): tcgen05 / TMEM kernel
    P.blobs = reinterpret_cast<const float*>(F.sdf_tc5_blobs);
    const size_t tiles_upper = n_upper / 64 + std::min<size_t>(n_upper, (size_t)F.geom.n_cells) + 1;
    sdf_tc5_kernel<<<(int)std::max<size_t>(1, std::min<size_t>(tiles_upper, (size_t)148 * kTc5CtasPerSm)), kTc5Tile, sizeof(Tc5FwdSmem), st>>>(P);
  } else if (F.precision == KNF_PRECISION_TENSOR_FP16X2) {
    P.blobs = reinterpret_cast<const float*>(F.sdf_mmah_blobs);
    sdf_mma_kernel<2><<<mlp_grid(F, n_upper, kMmaCtasPerSm), 32, sizeof(MmaSmemT<2>), st>>>(P);
  } else {
    mlp_warp_kernel<kSdfIn, kSdfOut, kSdfOutPad, ACT_SOFTPLUS, false>
        <<<mlp_grid(F, n_upper, kFwdCtasPerSm), 32, sizeof(SdfKernelSmem), st>>>(P);
  }
  F.stats.kernel_launches += 1;
  KNF_CUDA(cudaGetLastError());
  return 0;
}

int launch_col_mlp(Field& F, const RouteBuffers& R, size_t n_upper, const float* v, const float* nrm, const float* z,
                   float* rgb, cudaStream_t st) {
  MlpParams P{};
  P.blobs = F.col_blobs;
  P.perm = R.perm;
  P.tiles = R.tiles;
  P.ctr = R.ctr;
  P.req_pt = R.req_pt;
  P.col_v = v;
  P.col_n = nrm;
  P.col_z = z;
  P.out_full = rgb;
  ProfScope prof(F, st, SPAN_COLOR_MLP);
  mlp_warp_kernel<kColIn, kColOut, kColOutPad, ACT_RELU, true>
      <<<mlp_grid(F, n_upper, kFwdCtasPerSm), 32, sizeof(ColKernelSmem), st>>>(P);
  F.stats.kernel_launches += 1;
  KNF_CUDA(cudaGetLastError());
  return 0;
}

int sdf_forward_device(Field& F, const float* pts, int64_t n, float* out_full, float* out_first, int* cell_out,
                       cudaStream_t st) {
  if (n <= 0) return 0;
  KNF_TRY(ensure_requests(F, (size_t)n));
  RouteBuffers R = route_buffers(F, 2, -1);
  R.eval_counter = stat_counter(F, 0);
  R.small_tiles = sdf_forward_tile_mode(F);
  route_emit_points_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(R, F.geom, pts, (int)n, cell_out);
  F.stats.kernel_launches += 1;
  KNF_TRY(launch_scan_scatter(F, R, (size_t)n, st));
  return launch_sdf_mlp(F, R, (size_t)n, out_first, out_full, st);
}

int color_forward_device(Field& F, const float* x, const float* v, const float* nrm, const float* z, int64_t n,
                         float* rgb, cudaStream_t st) {
  if (n <= 0) return 0;
  KNF_TRY(ensure_requests(F, (size_t)n));
  RouteBuffers R = route_buffers(F, 3, -1);
  R.eval_counter = stat_counter(F, 1);
  route_emit_points_kernel<<<blocks_for((size_t)n), 256, 0, st>>>(R, F.geom, x, (int)n, nullptr);
  F.stats.kernel_launches += 1;
  KNF_TRY(launch_scan_scatter(F, R, (size_t)n, st));
  return launch_col_mlp(F, R, (size_t)n, v, nrm, z, rgb, st);
}

// Sub-box refinement of the per-cell Lipschitz bounds (knf_bounds.cuh), once per handle, on the stream of the first march
// that uses the decision filter: the filter blobs keep the closed-form bounds until the store kernel has run, and both are
// proven bounds, so there is no window in which a kernel could read an invalid one.
int ensure_lipschitz_refined(Field& F, cudaStream_t st) {
  if (F.lip_refined || !F.lip_cur || !F.lip_consts) return 0;
  F.lip_refined = true;
  if (!(F.lip_width > 0.0)) return 0;
  const int N = F.geom.resolution, n_cells = F.geom.n_cells;
  double cell_w = 0.0, coord = 0.0;
  for (int a = 0; a < 3; a++) {
    cell_w = std::max(cell_w, (F.geom.hi[a] - F.geom.lo[a]) / (double)N);
    coord = std::max(coord, std::max(std::fabs(F.geom.lo[a]), std::fabs(F.geom.hi[a])));
  }
  LipArgs A{};
  A.blobs = F.sdf_blobs;
  A.cc = F.lip_consts;
  A.G = F.geom;
  A.k = (int)std::max(1.0, std::min(64.0, std::ceil(cell_w / F.lip_width)));
  A.fine = F.lip_fine;
  // certified skipping requires the evaluated sample p0 within kLipSlack of the cell box (knf_tc5.cuh / knf_march.cuh
  // `p0_in`): cover that, the fp32 rounding of the kernels' box test and the inner-box margin with room to spare
  A.margin = 4.0 * (double)kLipSlack * cell_w + 4e-7 * coord;
  A.out = F.lip_max;
  KNF_CUDA(cudaMemsetAsync(F.lip_max, 0, (size_t)n_cells * 3 * sizeof(unsigned long long), st));
  const long long n_sub = (long long)A.k * A.k * A.k;
  // enough CTAs to fill the GPU several times over, each warp still looping over many sub-boxes of its cell
  int chunks = (int)std::max<long long>(1, std::min<long long>((n_sub + 8 * kLipWarps - 1) / (8 * kLipWarps), (148 * 16 + n_cells - 1) / n_cells));
  KNF_CUDA(cudaFuncSetAttribute(lip_bound_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LipSmem)));
  lip_bound_kernel<<<dim3(n_cells, chunks), 32 * kLipWarps, sizeof(LipSmem), st>>>(A);
  const bool tc5 = F.sdf_tc5_blobs != nullptr, mma = F.sdf_mmah_blobs != nullptr;
  lip_store_kernel<<<(n_cells * 3 + 255) / 256, 256, 0, st>>>(
      F.lip_max, n_cells, F.lip_cur, tc5 ? F.sdf_tc5_blobs : nullptr, Tc5Blob::bytes, Tc5Blob::off_f32 + Tc5Blob::f_lip * 4,
      mma ? F.sdf_mmah_blobs : nullptr, MmaBlobT<2>::words, MmaBlobT<2>::b3 + kFilterLipSlot);
  F.stats.kernel_launches += 2;
  KNF_CUDA(cudaGetLastError());
  return 0;
}

int march_device(Field& F, const double* o, const double* d, const double* t_near, const double* t_far, int64_t n,
                 const KnfSettings& s, unsigned char* hit, double* t, double* pos, int* steps, bool want_hit_list,
                 cudaStream_t st) {
  if (n <= 0) return 0;
  if (n > INT32_MAX / 16) return fail(KNF_E_INVALID, "march batch too large; split the rays");
  KNF_TRY(ensure_rays(F, (size_t)n));
  Workspace& W = F.ws;
  MarchState M{};
  M.o = o;
  M.d = d;
  M.t_far = t_far;
  M.t = W.t.as<double>();
  M.t_prev = W.t_prev.as<double>();
  M.d_prev = W.d_prev.as<double>();
  M.t_conv = W.t_conv.as<double>();
  M.d_conv = W.d_conv.as<double>();
  M.t_hit = W.t_hit.as<double>();
  M.steps = W.steps.as<int>();
  M.phase = W.phase.as<unsigned char>();
  M.hit = W.hit.as<unsigned char>();
  M.live[0] = W.live0.as<int>();
  M.live[1] = W.live1.as<int>();
  M.live[2] = W.live2.as<int>();
  M.live[3] = W.live3.as<int>();
  M.eps = s.eps_hit;
  M.step_scale = s.step_scale;
  M.max_steps = s.max_steps;

  KNF_CUDA(cudaMemsetAsync(counters(F, 0), 0, 2 * sizeof(RouteCounters), st));
  KNF_CUDA(cudaMemsetAsync(counters(F, 4), 0, 2 * sizeof(RouteCounters), st));
  KNF_CUDA(cudaMemsetAsync(W.cell_count_f.p, 0, (size_t)F.geom.n_cells * sizeof(int), st));
  const int nb = blocks_for((size_t)n);
  // The decision filter (knf_march.cuh) serves the exact mode only; the tensor modes evaluate everything on the
  // tensor cores anyway.  auto: let the first global wavefront (one sample per ray) show whether rays enter the
  // negative region at all -- on a real surface they never do and the filter passes would be empty launches.
  const bool exact_mode = F.precision == KNF_PRECISION_FP32_CHAIN;
  bool use_filter = exact_mode && F.fp16_ok && F.filter_mode != 0;
  // auto: probe the first wavefront unless the previous march on this handle already showed which way it goes
  // (consecutive frames of one field look alike; a wrong hint costs time, never a result)
  if (use_filter && F.filter_mode == 2 && F.filter_hint == 2) use_filter = false;
  const bool probing = use_filter && F.filter_mode == 2 && F.filter_hint == 0;
  if (use_filter && !probing && F.filter_skip > 0) KNF_TRY(ensure_lipschitz_refined(F, st));  // (a probing march refines once it has seen rays crawl)
  // When the previous march on this handle has shown that rays crawl, every ray's FIRST sample goes to the filter queue too:
  // about half of them are decided there at tensor-core speed (the rest move, unchanged, to the exact queue of wavefront 1,
  // beside the filter's second pass) instead of all of them paying a dense exact launch that nothing overlaps.
  const bool filter_first = use_filter && !probing && F.filter_first;
  {
    ProfScope prof(F, st, SPAN_ROUTE);
    RouteBuffers R0 = filter_first ? route_buffers(F, 4, 5, 2) : route_buffers(F, 0, 1, 0);
    march_init_kernel<<<nb, 256, 0, st>>>(R0, F.geom, M, t_near, (int)n, filter_first ? M.live[2] : M.live[0], route_buffers(F, 0, 1, 0), M.live[0],
                                          filter_first ? F.first_split_eighths : 0);
    F.stats.kernel_launches += 1;
  }
  size_t seen_filter = 0, seen_total = 0;
  bool filter_drained = false;  // the filter queue was seen empty after the filter had been switched off
  bool exact_sparse = false;    // last poll: the exact queue holds < 1/16 of the rays -> small-tile-only kernel
  const double crawl_on = -(s.eps_hit + 2.0 * F.filter_delta_max);
  // Global wavefronts.  Every ray queued in a wavefront either advances a step, fetches (once each) its secant / re-check
  // sample, or -- a filter-queue ray whose sample the filter cannot decide -- moves to the next exact queue unchanged and
  // advances there, so 2 * max_steps + 6 bounds the count; tile residency usually finishes in far fewer, which the host
  // learns by polling the request counts.
  // KNF_DEBUG_TIMELINE=1: events at the phase boundaries of every wavefront, printed (relative to the march's start) after the march
  static const bool debug_timeline = std::getenv("KNF_DEBUG_TIMELINE") != nullptr;
  struct Mark { const char* what; int w; cudaEvent_t ev; };
  std::vector<Mark> marks;
  auto mark = [&](const char* what, int w, cudaStream_t s_) {
    if (!debug_timeline) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s_);
    marks.push_back({what, w, e});
  };
  mark("start", -1, st);
  F.prof_chain = true;  // spans inside the loop are back to back on `st`: one shared event between neighbours
  F.prof_last_end = (size_t)-1;
  size_t live_upper = (size_t)n;  // upper bound on the size of any queue from here on: sizes the routing and tile grids
  const int max_wavefronts = 2 * s.max_steps + 6;
  // hand-over point to the one-warp-per-ray tail kernel: a fixed count for large marches, 1/16 of the rays for small ones
  // (twice as early when the tail kernel can skip certified crawl steps: measured 4.58 -> 4.30 ms on the random-init frame;
  // a trained field, whose tail evaluates every step, loses 0.4 ms with the larger hand-over)
  auto tail_threshold_now = [&]() {
    const int base = (use_filter && F.tail_skip && F.filter_skip > 0 && F.sdf_tc5_blobs && F.filter_kernel == 1) ? 2 * F.tail_threshold : F.tail_threshold;
    return base > 0 ? (int)std::min<int64_t>(base, std::max<int64_t>(n / 16, 2048)) : 0;
  };
  for (int w = 0; w < max_wavefronts; w++) {
    const int cur = w & 1, nxt = cur ^ 1;
    const bool filter_pass = exact_mode && F.fp16_ok && F.filter_mode != 0 && !filter_drained && (w > 0 || filter_first);
    MarchTileArgs A{};
    A.G = F.geom;
    A.M = M;
    A.next = route_buffers(F, nxt, -1, nxt);
    A.next_filter = route_buffers(F, 4 + nxt, -1, 2 + nxt);
    A.live_out = M.live[nxt];
    A.live_filter = M.live[2 + nxt];
    A.eval_counter = stat_counter(F, 0);
    A.max_inner = (probing && w == 0) ? 1 : F.march_max_inner;
    A.crawl_below = use_filter ? crawl_on : -INFINITY;
    A.max_skip = F.filter_skip;
    A.skip_cap = F.filter_skip_cap;
    A.inv_resolution = 1.0 / (double)F.geom.resolution;
    A.filter_x_raw = F.filter_x_raw;
    for (int a = 0; a < 3; a++) A.cell_scale[a] = (double)F.geom.resolution / (F.geom.hi[a] - F.geom.lo[a]);
    // Both queues of this wavefront were filled by the previous wavefront's kernels and hold different rays, so their tile
    // kernels are independent: route both, then run the filter kernel on the caller's stream and the exact kernel beside
    // it on the side stream (the exact launches of a frame are sparse and latency-bound; alone on the GPU they cost 2.6 ms
    // per 1080p frame).  Samples the filter cannot decide join the exact queue of the NEXT wavefront.
    const bool tc5 = F.filter_kernel == 1 && F.sdf_tc5_blobs != nullptr;
    RouteBuffers Rf = route_buffers(F, 4 + cur, 4 + nxt, 2 + cur);
    if (filter_pass) {
      Rf.sorted = W.sorted_f.as<float4>();
      Rf.live = M.live[2 + cur];
      Rf.small_tiles = tc5 ? 3 : 0;  // tcgen05 filter: tiles of <= 128 requests (one per thread of a 128-thread CTA)
    }
    RouteBuffers R = route_buffers(F, cur, nxt, cur);
    R.eval_counter = stat_counter(F, 3);  // requests that went through global routing
    R.sorted = W.sorted.as<float4>();
    R.live = M.live[cur];
    const bool small_only = exact_mode && exact_sparse && F.sparse_small_kernel;
    const bool mid = exact_mode && !small_only && F.exact_mid;
    R.small_tiles = small_only ? 2 : (mid ? 4 : 0);  // dense wavefronts: <= 32-request tiles for march_mid_kernel (or 64 for march_warp_kernel); sparse: <= 16 for march_small_kernel
    mark("wavefront", w, st);
    if (filter_pass) KNF_TRY(launch_scan_scatter2(F, Rf, R, live_upper, st));
    else KNF_TRY(launch_scan_scatter(F, R, live_upper, st));
    mark("routed", w, st);
    cudaStream_t st_exact = st;
    if (filter_pass && F.overlap_queues && F.side_stream) {
      KNF_CUDA(cudaEventRecord(F.ev_fork, st));
      KNF_CUDA(cudaStreamWaitEvent(F.side_stream, F.ev_fork, 0));
      st_exact = F.side_stream;
    }
    auto launch_filter = [&]() -> int {
      MarchTileArgs Af = A;
      Af.P.blobs = reinterpret_cast<const float*>(F.sdf_mmah_blobs);
      Af.P.perm = Rf.perm;
      Af.P.tiles = Rf.tiles;
      Af.P.ctr = Rf.ctr;
      Af.P.req_pt = Rf.req_pt;
      Af.P.sorted = Rf.sorted;
      Af.live_in = M.live[2 + cur];
      Af.max_inner = F.filter_max_inner;
      Af.keep_div = F.filter_keep_div;
      Af.defer = A.next;  // undecided samples: the exact queue of the next wavefront
      Af.live_defer = A.live_out;
      {
        ProfScope prof(F, st, SPAN_FILTER);
        if (tc5) {
          Af.P.blobs = reinterpret_cast<const float*>(F.sdf_tc5_blobs);
          const size_t tiles_upper = live_upper / 64 + std::min<size_t>(live_upper, (size_t)F.geom.n_cells) + 1;
          const int grid = (int)std::max<size_t>(1, std::min<size_t>(tiles_upper, (size_t)148 * std::min(kTc5CtasPerSm, F.filter_grid_ctas)));
          march_tc5_kernel<<<grid, kTc5Tile, sizeof(Tc5MarchSmem), st>>>(Af);
        } else {
          march_mma_kernel<2, true><<<mlp_grid(F, live_upper, march_ctas_per_sm<2>()), 32, sizeof(MmaMarchSmemT<2>), st>>>(Af);
        }
      }
      F.stats.kernel_launches += 1;
      mark("filter done", w, st);
      return 0;
    };
    // the exact queue's launch; beside a filter pass its grid may be capped (KNF_EXACT_GRID CTAs per SM) so that both kernels'
    // CTAs are resident together instead of the first-launched one holding every register of the SM until it drains
    const bool beside_filter = filter_pass && st_exact != st;
    auto exact_ctas = [&](int full) { return beside_filter && F.exact_grid_ctas > 0 ? std::min(full, F.exact_grid_ctas) : full; };
    auto launch_exact = [&]() -> int {
    MarchTileArgs& Ax = A;
    Ax.P.blobs = F.sdf_blobs;
    Ax.P.perm = R.perm;
    Ax.P.tiles = R.tiles;
    Ax.P.ctr = R.ctr;
    Ax.P.req_pt = R.req_pt;
    Ax.P.sorted = R.sorted;
    Ax.live_in = M.live[cur];
    {
      ProfScope prof(F, st_exact, SPAN_SDF_MLP);
      if (F.precision == KNF_PRECISION_TENSOR_BF16X3) {
        A.P.blobs = reinterpret_cast<const float*>(F.sdf_mma_blobs);
        march_mma_kernel<3, false><<<mlp_grid(F, live_upper, march_ctas_per_sm<3>()), 32, sizeof(MmaMarchSmemT<3>), st_exact>>>(A);
      } else if (F.precision == KNF_PRECISION_TENSOR_FP16X2) {
        A.P.blobs = reinterpret_cast<const float*>(F.sdf_mmah_blobs);
        march_mma_kernel<2, false><<<mlp_grid(F, live_upper, march_ctas_per_sm<2>()), 32, sizeof(MmaMarchSmemT<2>), st_exact>>>(A);
      } else if (small_only) {
        // sparse wavefront: few tiles, the GPU is far from full -- a ray that stays in its cell keeps stepping there
        // rather than paying another routing round trip (the long tail of a frame is a chain of such round trips)
        A.max_inner = F.sparse_max_inner;
        A.keep_div = F.sparse_keep_div;
        march_small_kernel<<<mlp_grid(F, live_upper, exact_ctas(kSmallCtasPerSm)), 32, sizeof(SdfSmallSmem), st_exact>>>(A);
      } else if (mid) {
        march_mid_kernel<<<mlp_grid(F, live_upper, exact_ctas(kMidCtasPerSm)), 32, sizeof(SdfMidSmem), st_exact>>>(A);
      } else {
        march_warp_kernel<<<mlp_grid(F, live_upper), 32, sizeof(SdfKernelSmem), st_exact>>>(A);
      }
    }
    mark("exact done", w, st_exact);
    return 0;
    };
    if (filter_pass && beside_filter && F.exact_first) {
      KNF_TRY(launch_exact());
      KNF_TRY(launch_filter());
    } else {
      if (filter_pass) KNF_TRY(launch_filter());
      KNF_TRY(launch_exact());
    }
    if (st_exact != st) {
      KNF_CUDA(cudaEventRecord(F.ev_join, st_exact));
      KNF_CUDA(cudaStreamWaitEvent(st, F.ev_join, 0));
    }
    F.stats.kernel_launches += 1;
    F.stats.wavefronts += 1;
    // (more often once the live count nears the tail threshold, so the hand-over is not missed by several wavefronts)
    const int tail_at = tail_threshold_now();
    const bool near_tail = exact_mode && tail_at > 0 && live_upper <= (size_t)tail_at * 6 && w > 3;
    const bool poll = (w == 0 && probing) || (w == 1) || (w == 3) || (w % 8 == 7) || (near_tail && (w & 1));
    if (poll && w + 1 < max_wavefronts) {
      // n_requests of the next exact queue and of the next filter queue
      KNF_CUDA(cudaMemcpyAsync(F.host_poll, &counters(F, nxt)->n_requests, sizeof(int), cudaMemcpyDeviceToHost, st));
      KNF_CUDA(cudaMemcpyAsync(F.host_poll + 1, &counters(F, 4 + nxt)->n_requests, sizeof(int), cudaMemcpyDeviceToHost, st));
      KNF_CUDA(cudaStreamSynchronize(st));
      F.prof_last_end = (size_t)-1;  // the GPU idled during the poll: the next span records its own start
      const int n_exact = F.host_poll[0], n_filter = F.host_poll[1];
      if (w <= 1) {
        seen_filter = (size_t)n_filter;
        seen_total = (size_t)n_exact + (size_t)n_filter;
      }
      if (n_exact == 0 && n_filter == 0) break;
      if (exact_mode && tail_at > 0 && n_exact + n_filter <= tail_at) {
        // few rays left: one warp per ray to completion instead of more global wavefronts (knf_tail.cuh)
        MarchTailArgs T{};
        T.blobs = F.sdf_blobs;
        T.G = F.geom;
        T.M = M;
        for (int a = 0; a < 3; a++) T.cell_scale[a] = A.cell_scale[a];
        const RouteBuffers Qa = route_buffers(F, nxt, -1, nxt), Qb = route_buffers(F, 4 + nxt, -1, 2 + nxt);
        T.live_a = M.live[nxt]; T.pt_a = Qa.req_pt; T.cell_a = Qa.req_cell; T.ctr_a = Qa.ctr;
        T.live_b = M.live[2 + nxt]; T.pt_b = Qb.req_pt; T.cell_b = Qb.req_cell; T.ctr_b = Qb.ctr;
        T.cursor = W.tail_cursor.as<int>();
        T.eval_counter = stat_counter(F, 0);
        T.inv_resolution = A.inv_resolution;
        T.skip_cap = F.filter_skip_cap;
        if (use_filter && F.filter_skip > 0 && F.tail_skip && tc5) {  // certified skipping in the tail: delta / L_a from the tcgen05 filter blobs
          T.fconst = F.sdf_tc5_blobs;
          T.fconst_stride = Tc5Blob::bytes;
          T.off_delta = Tc5Blob::off_f32 + Tc5Blob::f_delta * 4;
          T.off_lip = Tc5Blob::off_f32 + Tc5Blob::f_lip * 4;
        }
        KNF_CUDA(cudaMemsetAsync(W.tail_cursor.p, 0, 16, st));
        const int rays_left = n_exact + n_filter;
        const int rays_per_cta = kTailWarps * (32 / kTailGroup);  // a group of kTailGroup lanes per ray
        const int grid = std::max(1, std::min((rays_left + rays_per_cta - 1) / rays_per_cta, 148 * 8));
        static const bool debug_tail = std::getenv("KNF_DEBUG_TAIL") != nullptr;
        cudaEvent_t dbg0 = nullptr, dbg1 = nullptr;
        if (debug_tail) {
          cudaEventCreate(&dbg0);
          cudaEventCreate(&dbg1);
          cudaEventRecord(dbg0, st);
        }
        {
          ProfScope prof(F, st, SPAN_SDF_MLP);
          march_tail_kernel<<<grid, 32 * kTailWarps, 0, st>>>(T);
        }
        if (debug_tail) {
          cudaEventRecord(dbg1, st);
          cudaEventSynchronize(dbg1);
          float tms = 0.f;
          cudaEventElapsedTime(&tms, dbg0, dbg1);
          fprintf(stderr, "march_tail_kernel: %d rays handed over at wavefront %d, %.3f ms\n", rays_left, w, tms);
          cudaEventDestroy(dbg0);
          cudaEventDestroy(dbg1);
        }
        F.stats.kernel_launches += 1;
        // the pending queues were consumed without a routing pass: leave their per-cell counts as a pass would
        KNF_CUDA(cudaMemsetAsync(W.cell_count.p, 0, (size_t)F.geom.n_cells * sizeof(int), st));
        KNF_CUDA(cudaMemsetAsync(W.cell_count_f.p, 0, (size_t)F.geom.n_cells * sizeof(int), st));
        break;
      }
      exact_sparse = (size_t)n_exact * (size_t)F.sparse_div < (size_t)n;
      live_upper = std::max<size_t>((size_t)n_exact + (size_t)n_filter, 1);  // rays only retire: an upper bound for every later queue
      if (probing && w == 0 && (size_t)n_filter * 8 < (size_t)(n_exact + n_filter)) use_filter = false;  // < 1/8 of the live rays crawl
      if (probing && w == 0 && use_filter && F.filter_skip > 0) KNF_TRY(ensure_lipschitz_refined(F, st));
      if (!use_filter && n_filter == 0) filter_drained = true;
    }
  }
  F.prof_chain = false;
  if (debug_timeline) {
    mark("march end", -1, st);
    cudaStreamSynchronize(st);
    if (F.side_stream) cudaStreamSynchronize(F.side_stream);
    fprintf(stderr, "timeline of a march of %lld rays (ms since start):", (long long)n);
    int last_w = -2;
    for (size_t i = 1; i < marks.size(); i++) {
      float ms_ = 0.f;
      cudaEventElapsedTime(&ms_, marks[0].ev, marks[i].ev);
      if (marks[i].w != last_w) fprintf(stderr, "\n  w%-3d", marks[i].w);
      last_w = marks[i].w;
      fprintf(stderr, " %s %.3f |", marks[i].what, ms_);
    }
    fprintf(stderr, "\n");
    for (Mark& m : marks) cudaEventDestroy(m.ev);
  }
  if (std::getenv("KNF_DEBUG_HINT"))
    fprintf(stderr, "march n=%lld hint_before=%d probing=%d filter_first=%d use_filter_end=%d seen_filter=%zu seen_total=%zu wavefronts=%lld\n", (long long)n, F.filter_hint,
            (int)probing, (int)filter_first, (int)use_filter, seen_filter, seen_total, (long long)F.stats.wavefronts);
  if (exact_mode && F.fp16_ok && F.filter_mode == 2 && seen_total > 0) {
    // The hint errs towards the filter: a march that crawls without it pays for every crawl step with an exact evaluation,
    // a march that carries it in vain pays a few empty launches.  Marches on one handle differ (path tracing alternates
    // primary and bounce rays, late bounces are small and their statistics noisy), so "rays crawl" is sticky: only a LARGE
    // march that is (almost) crawl-free sends the handle back to probing, and only such a march sets "no crawl" (large by
    // its LIVE rays after the first wavefronts: the path tracer marches whole bands whose late bounces hold a handful).
    const bool crawl = seen_filter * 8 >= seen_total, none = seen_filter * 64 < seen_total, large = seen_total >= 16384;
    if (F.filter_hint == 1) {
      if (none && large) F.filter_hint = 0;
    } else if (F.filter_hint == 0) {
      if (crawl) F.filter_hint = 1;
      else if (none && large) F.filter_hint = 2;
    } else if (n >= 4096) {
      F.filter_hint = 0;  // a "no crawl" hint is re-examined by probing the next large march
    }
  }
  if (want_hit_list) KNF_CUDA(cudaMemsetAsync(W.hit_count.p, 0, 16, st));
  march_finish_kernel<<<nb, 256, 0, st>>>(M, (int)n, hit, t, pos, steps, want_hit_list ? W.hit_list.as<int>() : nullptr,
                                          want_hit_list ? W.hit_count.as<int>() : nullptr);
  F.stats.kernel_launches += 1;
  F.stats.rays += n;
  KNF_CUDA(cudaGetLastError());
  return 0;
}

int read_hit_count(Field& F, cudaStream_t st, int* out) {
  KNF_CUDA(cudaMemcpyAsync(out, F.ws.hit_count.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  KNF_CUDA(cudaStreamSynchronize(st));
  F.stats.hits += *out;
  return 0;
}

static int shade_common(Field& F, ShadePoints S, int64_t m, const ShadeTargets& T, cudaStream_t st) {
  if (m <= 0) return 0;
  const bool color = T.colors != nullptr;
  const int np = color ? 7 : 6;
  const size_t nreq = (size_t)m * np;
  KNF_TRY(ensure_requests(F, nreq));
  Workspace& W = F.ws;
  KNF_TRY(W.sdf_out.ensure(nreq * kSdfOut * sizeof(float)));
  if (color) {
    KNF_TRY(W.col_v.ensure((size_t)m * 3 * sizeof(float)));
    KNF_TRY(W.col_n.ensure((size_t)m * 3 * sizeof(float)));
    KNF_TRY(W.col_z.ensure((size_t)m * kFeat * sizeof(float)));
    KNF_TRY(W.rgb.ensure((size_t)m * 3 * sizeof(float)));
  }
  S.m_host = (int)m;
  S.count = nullptr;
  RouteBuffers R = route_buffers(F, 2, -1);
  R.eval_counter = stat_counter(F, 0);
  R.small_tiles = sdf_forward_tile_mode(F);
  shade_emit_kernel<<<blocks_for(nreq), 256, 0, st>>>(R, F.geom, S, np);
  F.stats.kernel_launches += 1;
  KNF_TRY(launch_scan_scatter(F, R, nreq, st));
  KNF_TRY(launch_sdf_mlp(F, R, nreq, nullptr, W.sdf_out.as<float>(), st));
  RouteBuffers Rc = route_buffers(F, 3, -1);
  Rc.eval_counter = stat_counter(F, 1);
  shade_finish_kernel<<<blocks_for((size_t)m), 256, 0, st>>>(
      Rc, F.geom, S, np, W.sdf_out.as<float>(), T.eps, T.fallback ? 1 : 0, T.grad, T.normals, T.ok,
      T.scatter_by_ray ? 1 : 0, W.col_v.as<float>(), W.col_n.as<float>(), W.col_z.as<float>(), color ? 1 : 0);
  F.stats.kernel_launches += 1;
  if (color) {
    KNF_TRY(launch_scan_scatter(F, Rc, (size_t)m, st));
    KNF_TRY(launch_col_mlp(F, Rc, (size_t)m, W.col_v.as<float>(), W.col_n.as<float>(), W.col_z.as<float>(),
                           W.rgb.as<float>(), st));
    shade_colors_kernel<<<blocks_for((size_t)m), 256, 0, st>>>(S, W.rgb.as<float>(), T.scatter_by_ray ? 1 : 0,
                                                              T.clip_colors ? 1 : 0, T.colors);
    F.stats.kernel_launches += 1;
  }
  KNF_CUDA(cudaGetLastError());
  return 0;
}

int shade_points_device(Field& F, const double* pts, const double* dirs, int64_t m, const ShadeTargets& T,
                        cudaStream_t st) {
  ShadePoints S{};
  S.pts = pts;
  S.dirs = dirs;
  return shade_common(F, S, m, T, st);
}

int shade_hits_device(Field& F, const double* o, const double* d, int64_t first_hit, int64_t m_hits,
                      const ShadeTargets& T, cudaStream_t st) {
  ShadePoints S{};
  S.o = o;
  S.d = d;
  S.t_hit = F.ws.t_hit.as<double>();
  S.list = F.ws.hit_list.as<int>() + first_hit;
  return shade_common(F, S, m_hits, T, st);
}

}  // namespace knf
