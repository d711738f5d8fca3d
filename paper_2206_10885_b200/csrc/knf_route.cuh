// knf_route.cuh -- cell routing: the counting sort that groups evaluation requests by grid cell
// (north_star subsystem 1).  Replaces grid._cell_triples / cell_index_flat / route
// (grid.py:176-213: fp64 cell arithmetic, np.argsort(kind="stable"), np.unique).
//
// A routing pass is three kernels over the request list:
//   emit    (fused into whatever produces the requests): cell id in fp64 from the fp32 point,
//           rank = warp-aggregated atomicAdd on the cell's counter (__match_any_sync so one
//           atomic serves all lanes of a warp that share a cell -- neighbouring rays usually do);
//   scan    one CTA: exclusive scan of the per-cell counts -> cell offsets, the tile list for the
//           MLP kernel, optionally the occupied-segment list of grid.route; re-zeroes the counts
//           and the NEXT pass's counters so no memset launches are needed;
//   scatter perm[offset[cell] + rank] = request slot.
// Only 4-byte indices move; points and results stay in request order.  Rank order inside a cell
// depends on atomic timing, but every request is evaluated independently with a fixed FMA order,
// so results are deterministic.
#pragma once

#include "knf_common.cuh"

namespace knf {

struct RouteBuffers {
  float4* req_pt;     // [cap] request slot -> fp32 point (w unused)
  int* req_cell;      // [cap]
  int* req_rank;      // [cap]
  int* cell_count;    // [n_cells], zero on entry to a pass
  int* cell_offset;   // [n_cells + 1]
  int* perm;          // [cap]
  Tile* tiles;        // [cap / kTilePts + n_cells + 1]
  RouteCounters* ctr; // this pass
  RouteCounters* next_ctr;  // zeroed by scan (may equal nullptr)
  unsigned long long* eval_counter;  // += n_requests per pass (nullable); statistics only
};

// Record request `slot` at fp32 point (x,y,z) whose cell is already known.  Must be reached by
// all 32 lanes; `active` is false for lanes that have nothing to emit.
__device__ __forceinline__ void route_emit_cell(const RouteBuffers& R, bool active, int slot, float x, float y, float z,
                                                int cell) {
  if (!active) cell = -1;
  unsigned peers = __match_any_sync(0xffffffffu, cell);  // all 32 lanes reach this (warp-uniform loops)
  if (active) {
    int lane = threadIdx.x & 31;
    int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&R.cell_count[cell], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    int rank = base + __popc(peers & ((1u << lane) - 1));
    R.req_pt[slot] = make_float4(x, y, z, 0.f);
    R.req_cell[slot] = cell;
    R.req_rank[slot] = rank;
  }
}

__device__ __forceinline__ void route_emit(const RouteBuffers& R, const GridGeom& G, bool active, int slot, float x,
                                           float y, float z) {
  route_emit_cell(R, active, slot, x, y, z, active ? cell_of(x, y, z, G) : -1);
}

// grid.cell_index_flat on caller points + emit, slot = row index (the batched-forward entry).
static __global__ void route_emit_points_kernel(RouteBuffers R, GridGeom G, const float* __restrict__ pts, int n,
                                         int* __restrict__ cell_out) {
  int stride = gridDim.x * blockDim.x;
  int n_round = (n + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
    bool act = i < n;
    float x = 0.f, y = 0.f, z = 0.f;
    if (act) {
      x = pts[3 * (size_t)i + 0];
      y = pts[3 * (size_t)i + 1];
      z = pts[3 * (size_t)i + 2];
    }
    route_emit(R, G, act, i, x, y, z);
    if (act && cell_out) cell_out[i] = R.req_cell[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) R.ctr->n_requests = n;
}

// cell ids only (grid.cell_index_flat), no routing state touched.
template <class T>
static __global__ void cell_index_kernel(GridGeom G, const T* __restrict__ pts, int n, int* __restrict__ cell_out) {
  int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    cell_out[i] = cell_of((double)pts[3 * (size_t)i], (double)pts[3 * (size_t)i + 1], (double)pts[3 * (size_t)i + 2], G);
}

constexpr int kScanThreads = 1024;

// One CTA.  Optionally emits grid.route's occupied segments (cells ascending, starts).
static __global__ void __launch_bounds__(kScanThreads) route_scan_kernel(RouteBuffers R, int n_cells, int* __restrict__ seg_cell,
                                                                  int* __restrict__ seg_start,
                                                                  int* __restrict__ n_seg_out) {
  __shared__ int s_pts[kScanThreads];
  __shared__ int s_tiles[kScanThreads];
  __shared__ int s_segs[kScanThreads];
  const int tid = threadIdx.x;
  const int per = (n_cells + kScanThreads - 1) / kScanThreads;
  const int c0 = min(tid * per, n_cells);
  const int c1 = min(c0 + per, n_cells);
  int pts = 0, tl = 0, sg = 0;
  for (int c = c0; c < c1; c++) {
    int k = R.cell_count[c];
    pts += k;
    tl += (k + kTilePts - 1) / kTilePts;
    sg += (k > 0);
  }
  s_pts[tid] = pts;
  s_tiles[tid] = tl;
  s_segs[tid] = sg;
  __syncthreads();
  // Hillis-Steele inclusive scan over 1024 partials (three lanes of data)
  for (int off = 1; off < kScanThreads; off <<= 1) {
    int a = 0, b = 0, c = 0;
    if (tid >= off) {
      a = s_pts[tid - off];
      b = s_tiles[tid - off];
      c = s_segs[tid - off];
    }
    __syncthreads();
    s_pts[tid] += a;
    s_tiles[tid] += b;
    s_segs[tid] += c;
    __syncthreads();
  }
  int p_base = s_pts[tid] - pts;
  int t_base = s_tiles[tid] - tl;
  int g_base = s_segs[tid] - sg;
  for (int c = c0; c < c1; c++) {
    int k = R.cell_count[c];
    R.cell_offset[c] = p_base;
    R.cell_count[c] = 0;  // ready for the next pass
    if (k > 0 && seg_cell) {
      seg_cell[g_base] = c;
      seg_start[g_base] = p_base;
      g_base++;
    }
    for (int s = 0; s < k; s += kTilePts) {
      Tile t;
      t.cell = c;
      t.start = p_base + s;
      t.count = min(kTilePts, k - s);
      t.pad = 0;
      R.tiles[t_base++] = t;
    }
    p_base += k;
  }
  if (tid == kScanThreads - 1) {
    R.cell_offset[n_cells] = s_pts[tid];
    R.ctr->n_tiles = s_tiles[tid];
    R.ctr->tile_cursor = 0;
    if (R.eval_counter) *R.eval_counter += (unsigned long long)s_pts[tid];
    if (seg_start) seg_start[s_segs[tid]] = s_pts[tid];
    if (n_seg_out) *n_seg_out = s_segs[tid];
    if (R.next_ctr) {
      R.next_ctr->n_requests = 0;
      R.next_ctr->n_tiles = 0;
      R.next_ctr->tile_cursor = 0;
    }
  }
}

static __global__ void route_scatter_kernel(RouteBuffers R) {
  const int n = R.ctr->n_requests;
  int stride = gridDim.x * blockDim.x;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += stride)
    R.perm[R.cell_offset[R.req_cell[s]] + R.req_rank[s]] = s;
}

}  // namespace knf
