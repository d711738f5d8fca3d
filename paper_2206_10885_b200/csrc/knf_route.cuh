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
  int* tile_base;     // [n_cells + 1] first tile of each cell
  int* perm;          // [cap]
  Tile* tiles;        // [cap / kTilePts + n_cells + 1]
  RouteCounters* ctr; // this pass
  RouteCounters* next_ctr;  // zeroed by scan (may equal nullptr)
  unsigned long long* eval_counter;  // += n_requests per pass (nullable); statistics only
  float4* sorted;     // march queues: sorted position -> (point, ray id in .w): one coalesced load per tile point (nullable)
  const int* live;    // march queues: request slot -> ray id (read by scatter when `sorted` is set)
  int small_tiles;    // 1: cut the last < 49 requests of a cell into tiles of <= 16 (kernels with a small-tile path); 2: every tile <= 16;
                      // 4: every tile <= 32 (march_mid_kernel); 3: tiles of <= 128 requests, a cell's requests split evenly (knf_tc5.cuh: one request per thread of a 128-thread CTA)
};

// How a cell's k requests are cut into tiles: full 64-request tiles, then the remainder r either as one tile
// (r >= 49, or small tiles off) or as ceil(r / 16) tiles of <= 16 requests.
constexpr int kSmallTile = 16, kSmallTileMaxRemainder = 48;
constexpr int kBigTile = 128, kMidTile = 32;
__device__ __forceinline__ int tiles_of_cell(int k, int small_tiles) {
  if (small_tiles == 3) return (k + kBigTile - 1) / kBigTile;
  if (small_tiles == 4) return (k + kMidTile - 1) / kMidTile;
  if (small_tiles == 2) return (k + kSmallTile - 1) / kSmallTile;
  const int full = k / kTilePts, r = k - full * kTilePts;
  if (r == 0) return full;
  return full + ((small_tiles && r <= kSmallTileMaxRemainder) ? (r + kSmallTile - 1) / kSmallTile : 1);
}

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

// Three-lane block-wide exclusive scan step built from warp shuffles (2 block barriers).
__device__ __forceinline__ void block_scan3(int& a, int& b, int& c, int* s_warp /*[3*32]*/, int& ta, int& tb, int& tc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ia = a, ib = b, ic = c;  // inclusive within the warp
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int xa = __shfl_up_sync(0xffffffffu, ia, off), xb = __shfl_up_sync(0xffffffffu, ib, off),
        xc = __shfl_up_sync(0xffffffffu, ic, off);
    if (lane >= off) {
      ia += xa;
      ib += xb;
      ic += xc;
    }
  }
  if (lane == 31) {
    s_warp[warp] = ia;
    s_warp[32 + warp] = ib;
    s_warp[64 + warp] = ic;
  }
  __syncthreads();
  if (warp == 0) {
    int wa = s_warp[lane], wb = s_warp[32 + lane], wc = s_warp[64 + lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int xa = __shfl_up_sync(0xffffffffu, wa, off), xb = __shfl_up_sync(0xffffffffu, wb, off),
          xc = __shfl_up_sync(0xffffffffu, wc, off);
      if (lane >= off) {
        wa += xa;
        wb += xb;
        wc += xc;
      }
    }
    s_warp[lane] = wa;  // inclusive warp totals
    s_warp[32 + lane] = wb;
    s_warp[64 + lane] = wc;
  }
  __syncthreads();
  const int pa = warp ? s_warp[warp - 1] : 0, pb = warp ? s_warp[32 + warp - 1] : 0, pc = warp ? s_warp[64 + warp - 1] : 0;
  ta = s_warp[31];
  tb = s_warp[63];
  tc = s_warp[95];
  a = pa + ia - a;  // exclusive prefix of this thread
  b = pb + ib - b;
  c = pc + ic - c;
}

// Per-cell request offsets and per-cell tile bases of cells [c_begin, c_end) given the totals of all cells before them
// (the tile descriptors themselves are written in parallel by route_scatter_kernel).  Optionally emits grid.route's
// occupied segments (cells ascending, starts).  Re-zeroes the cell counters; the chunk that ends at n_cells also writes
// the totals and resets the next pass's counters.
__device__ __forceinline__ void route_scan_chunk(const RouteBuffers& R, int c_begin, int c_end, int n_cells, int base_p, int base_t, int base_g,
                                                 int* __restrict__ seg_cell, int* __restrict__ seg_start, int* __restrict__ n_seg_out, int* s_warp) {
  const int tid = threadIdx.x;
  const int per = (c_end - c_begin + kScanThreads - 1) / kScanThreads;
  const int c0 = min(c_begin + tid * per, c_end);
  const int c1 = min(c0 + per, c_end);
  int pts = 0, tl = 0, sg = 0;
  for (int c = c0; c < c1; c++) {
    int k = R.cell_count[c];
    pts += k;
    tl += tiles_of_cell(k, R.small_tiles);
    sg += (k > 0);
  }
  int p_base = pts, t_base = tl, g_base = sg, tot_p, tot_t, tot_g;
  block_scan3(p_base, t_base, g_base, s_warp, tot_p, tot_t, tot_g);
  p_base += base_p;
  t_base += base_t;
  g_base += base_g;
  for (int c = c0; c < c1; c++) {
    int k = R.cell_count[c];
    R.cell_offset[c] = p_base;
    R.tile_base[c] = t_base;
    R.cell_count[c] = 0;  // ready for the next pass
    if (k > 0 && seg_cell) {
      seg_cell[g_base] = c;
      seg_start[g_base] = p_base;
      g_base++;
    }
    t_base += tiles_of_cell(k, R.small_tiles);
    p_base += k;
  }
  if (c_end == n_cells && tid == kScanThreads - 1) {
    tot_p += base_p;
    tot_t += base_t;
    tot_g += base_g;
    R.cell_offset[n_cells] = tot_p;
    R.tile_base[n_cells] = tot_t;
    R.ctr->n_tiles = tot_t;
    R.ctr->tile_cursor = 0;
    if (R.eval_counter) *R.eval_counter += (unsigned long long)tot_p;
    if (seg_start) seg_start[tot_g] = tot_p;
    if (n_seg_out) *n_seg_out = tot_g;
    if (R.next_ctr) {
      R.next_ctr->n_requests = 0;
      R.next_ctr->n_tiles = 0;
      R.next_ctr->tile_cursor = 0;
    }
  }
}
// One CTA per queue: the whole grid in one chunk (up to a few 10^4 cells).
static __global__ void __launch_bounds__(kScanThreads) route_scan_kernel(RouteBuffers R, int n_cells, int* __restrict__ seg_cell,
                                                                  int* __restrict__ seg_start,
                                                                  int* __restrict__ n_seg_out) {
  __shared__ int s_warp[96];
  route_scan_chunk(R, 0, n_cells, n_cells, 0, 0, 0, seg_cell, seg_start, n_seg_out, s_warp);
}
// The two queues of a march wavefront (filter, exact) in one launch: CTA 0 scans the first, CTA 1 the second.
static __global__ void __launch_bounds__(kScanThreads) route_scan2_kernel(RouteBuffers Ra, RouteBuffers Rb, int n_cells) {
  __shared__ int s_warp[96];
  route_scan_chunk(blockIdx.x == 0 ? Ra : Rb, 0, n_cells, n_cells, 0, 0, 0, nullptr, nullptr, nullptr, s_warp);
}

// ---- large grids: the scan in two launches over gridDim.x chunks of `chunk` cells (gridDim.y = queues) -------------------
// part: per queue and chunk the totals (requests, tiles, occupied cells); apply: every CTA sums the parts before its chunk
// (<= 1024 chunks: one block-wide scan) and runs the chunk scan from those bases.
struct ScanPart {
  int p, t, g, pad;
};
static __global__ void __launch_bounds__(kScanThreads) route_scan_part_kernel(RouteBuffers Ra, RouteBuffers Rb, int n_cells, int chunk,
                                                                       ScanPart* __restrict__ part) {
  __shared__ int s_warp[96];
  const RouteBuffers& R = blockIdx.y == 0 ? Ra : Rb;
  const int c_begin = min((int)blockIdx.x * chunk, n_cells), c_end = min(c_begin + chunk, n_cells);
  const int per = (c_end - c_begin + kScanThreads - 1) / kScanThreads;
  const int c0 = min(c_begin + (int)threadIdx.x * per, c_end), c1 = min(c0 + per, c_end);
  int pts = 0, tl = 0, sg = 0;
  for (int c = c0; c < c1; c++) {
    int k = R.cell_count[c];
    pts += k;
    tl += tiles_of_cell(k, R.small_tiles);
    sg += (k > 0);
  }
  int tp, tt, tg;
  block_scan3(pts, tl, sg, s_warp, tp, tt, tg);
  if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = ScanPart{tp, tt, tg, 0};
}
static __global__ void __launch_bounds__(kScanThreads) route_scan_apply_kernel(RouteBuffers Ra, RouteBuffers Rb, int n_cells, int chunk,
                                                                        const ScanPart* __restrict__ part, int* __restrict__ seg_cell,
                                                                        int* __restrict__ seg_start, int* __restrict__ n_seg_out) {
  __shared__ int s_warp[96];
  const RouteBuffers& R = blockIdx.y == 0 ? Ra : Rb;
  const ScanPart* mine = part + blockIdx.y * gridDim.x;
  int a = 0, b = 0, c = 0, base_p, base_t, base_g;
  if ((int)threadIdx.x < (int)blockIdx.x) {
    const ScanPart v = mine[threadIdx.x];
    a = v.p; b = v.t; c = v.g;
  }
  block_scan3(a, b, c, s_warp, base_p, base_t, base_g);  // totals over the chunks before this one
  __syncthreads();                                        // s_warp is reused by the chunk scan
  const int c_begin = min((int)blockIdx.x * chunk, n_cells), c_end = min(c_begin + chunk, n_cells);
  route_scan_chunk(R, c_begin, c_end, n_cells, base_p, base_t, base_g, seg_cell, seg_start, n_seg_out, s_warp);
}

// perm[offset[cell] + rank] = request slot, and (in the same launch) the tile descriptors of every cell.
__device__ __forceinline__ void route_scatter_body(const RouteBuffers& R, int n_cells) {
  const int n = R.ctr->n_requests;
  const int stride = gridDim.x * blockDim.x;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int s = gid; s < n; s += stride) {
    const int c = R.req_cell[s];  // -1: a slot its producer left empty (knf_volume.cu)
    if (c >= 0) {
      const int pos = R.cell_offset[c] + R.req_rank[s];
      if (R.sorted) {  // march queues: the tile kernels read (point, ray) straight from the sorted position
        float4 v = R.req_pt[s];
        v.w = __int_as_float(R.live[s]);
        R.sorted[pos] = v;
      } else {
        R.perm[pos] = s;
      }
    }
  }
  // tile descriptors, one thread per TILE (a cell of a coarse grid can own thousands): the tile's cell is found by
  // bisection over the per-cell tile bases the scan wrote
  const int n_tiles = R.ctr->n_tiles;
  for (int ti = gid; ti < n_tiles; ti += stride) {
    int lo = 0, hi = n_cells;  // invariant: tile_base[lo] <= ti < tile_base[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (R.tile_base[mid] <= ti) lo = mid;
      else hi = mid;
    }
    const int c = lo, j = ti - R.tile_base[c];
    const int start = R.cell_offset[c], k = R.cell_offset[c + 1] - start;
    int off, take;
    if (R.small_tiles == 3) {
      // n = ceil(k / 128) tiles of an even share rounded up to whole warps (so only the last tile holds a partly filled
      // warp): per <= 128, and (n - 1) * per < k, so the last tile is never empty
      const int n = (k + kBigTile - 1) / kBigTile, per = ((k + n - 1) / n + 31) & ~31;
      off = j * per;
      take = min(per, k - off);
    } else if (R.small_tiles == 4) {
      off = j * kMidTile;
      take = min(kMidTile, k - off);
    } else if (R.small_tiles == 2) {
      off = j * kSmallTile;
      take = min(kSmallTile, k - off);
    } else {
      const int full = k / kTilePts;
      if (j < full) {
        off = j * kTilePts;
        take = kTilePts;
      } else {
        const int r = k - full * kTilePts, jr = j - full;
        if (R.small_tiles && r <= kSmallTileMaxRemainder) {
          off = full * kTilePts + jr * kSmallTile;
          take = min(kSmallTile, k - off);
        } else {
          off = full * kTilePts;
          take = r;
        }
      }
    }
    Tile t;
    t.cell = c;
    t.start = start + off;
    t.count = take;
    t.pad = 0;
    R.tiles[ti] = t;
  }
}
static __global__ void route_scatter_kernel(RouteBuffers R, int n_cells) { route_scatter_body(R, n_cells); }
static __global__ void route_scatter2_kernel(RouteBuffers Ra, RouteBuffers Rb, int n_cells) {
  route_scatter_body(Ra, n_cells);
  route_scatter_body(Rb, n_cells);
}

}  // namespace knf
