// knf_march.cuh -- the fused sphere-trace kernel (north_star subsystems 2 + 3; SURVEY K3 + K5).
//
// march_warp_kernel = the SDF tile MLP of knf_mlp.cuh with the march step of surface.march_rays
// (surface.py:180-223) as its epilogue, plus *tile residency*: after a step, every ray whose next
// sample still falls in the tile's cell is evaluated again right away by the same warp -- the
// cell's weights are already in shared memory and the ray is already in a lane -- and only rays
// that changed cell (or tiles that thinned out below half their size) go back through the global
// routing pass.  Rays inside a random-init or a real field crawl through a cell for many steps
// (step 0.8 * max(d, eps/2) against a cell edge of 0.125), so the number of global wavefronts
// drops from max_steps + 1 to a few dozen, and the per-step ray-state traffic is overlapped with
// other warps' FFMA work instead of being a separate HBM-bound kernel.
// Every ray still sees exactly the reference's sequence of evaluations; only their order across
// rays changes, and no result depends on that order.
#pragma once

#include "knf_mlp.cuh"
#include "knf_mma.cuh"
#include "knf_rays.cuh"

namespace knf {

struct MarchTileArgs {
  MlpParams P;              // current wavefront: blobs, perm, tiles, counters, request points
  RouteBuffers next;        // exact queue of the next wavefront: rays that leave their tile and need an exact distance
  RouteBuffers next_filter; // filter queue of the next wavefront: rays crawling through the negative region
  RouteBuffers defer;       // filter kernel only: exact queue of THIS wavefront, for samples the filter cannot decide
  GridGeom G;
  MarchState M;
  const int* live_in;       // request slot -> ray id (the list being consumed)
  int* live_out;            // ... of `next`
  int* live_filter;         // ... of `next_filter`
  int* live_defer;          // ... of `defer`
  unsigned long long* eval_counter;  // statistics: [0] SDF evaluations, [2] lane slots, [4] filter evaluations, [5] deferred, [6] certified skips, [7] filter lane slots
  int max_inner;            // cap on consecutive in-place steps of one tile
  int max_skip;             // filter kernel: 0 disables certified skipping
  int skip_cap;             // filter kernel: most certified steps taken sample by sample after one evaluation
  int keep_div;             // a tile keeps stepping in place while n_stay * keep_div >= its size (2 = half; 0 is read as 2)
  double inv_resolution;    // 1 / grid resolution (host-computed)
  double crawl_below;       // exact kernels: a march step from a distance below this continues in the filter queue (-inf: never)
  double cell_scale[3];     // resolution / (hi - lo) per axis (host-computed): cell_of_quick's estimate
  float filter_x_raw;       // filter kernel: the coordinate magnitude the per-cell bounds delta were derived for (knf_api.cu filter_delta);
                            // a sample with a larger |coordinate| (outside the box: caller-supplied t ranges) is left to the exact kernel
};

// Queue one ray's next sample (warp-uniform call; `emit` selects the lanes that take part).
__device__ __forceinline__ void march_emit(const RouteBuffers& Q, int* live, bool emit, int ray, const RayRegs& rr, const MarchState& M,
                                           float x, float y, float z, int cell) {
  if (!__any_sync(0xffffffffu, emit)) return;  // skip the collectives when nobody leaves
  const int slot = warp_append(&Q.ctr->n_requests, emit);
  if (emit) {
    live[slot] = ray;
    ray_store(rr, M, ray);
  }
  route_emit_cell(Q, emit, slot, x, y, z, cell);
}

// One tile visit of the exact kernel.  PTS = 64: up to 64 rays, two per lane (panel columns 2 lane, 2 lane + 1), 8 x 8
// register tiles; PTS = 32 / 16: one ray per lane (panel column = lane; lanes 0..15 for 16), evaluated by the 4 x 8 /
// 4 x 4 register tiles of knf_mlp.cuh -- the mid shape trades register-tile size for resident warps in dense wavefronts,
// the small one is a quarter of the work for the sparse tiles that dominate once the decision filter has taken the
// crawling rays away.  Same chains, same bits in every shape.
template <int PTS, class SmemT, int PLD>
__device__ __forceinline__ void march_exact_tile(const MarchTileArgs& A, SmemT& S, const Tile& tile, int lane,
                                                 uint32_t& parity, unsigned long long& evals, unsigned long long& slots) {
  using Blob = SdfBlob;
  constexpr bool SMALL = PTS < 64;  // one ray per lane
  static_assert(SMALL || PLD == kPanelLd, "the 64-point path needs the full panel");
  static_assert(PTS == 64 || PTS == 32 || PTS == 16, "tile shapes: 64, 32 or 16 requests");
  constexpr int NQ = SMALL ? 1 : 2;
  const MlpParams& P = A.P;
  float* X = S.x;
  bool active[NQ];
  int ray[NQ], col[NQ];
  float px[NQ], py[NQ], pz[NQ];
  RayRegs rr[NQ];  // the lane's rays live in registers for the whole tile visit
#pragma unroll
  for (int q = 0; q < NQ; q++) {
    col[q] = SMALL ? lane : 2 * lane + q;
    active[q] = col[q] < tile.count;
    ray[q] = 0;
    px[q] = py[q] = pz[q] = 0.f;
    if (active[q]) {
      const float4 pt = P.sorted[tile.start + col[q]];  // (point, ray id): written by the routing scatter
      ray[q] = __float_as_int(pt.w);
      px[q] = pt.x; py[q] = pt.y; pz[q] = pt.z;
      ray_load(rr[q], A.M, ray[q]);  // in flight during the first MLP pass
    }
  }
  if (PLD == kPanelLd) {
    zero_pad_rows<kSdfIn>(X, lane);
  } else if (lane < PTS) {
#pragma unroll
    for (int r = kSdfIn; r < pad_k(kSdfIn); r++) X[r * PLD + lane] = 0.f;
  }
  // fp32 box strictly inside the tile's cell: a point inside it is in this cell without redoing the
  // fp64 cell arithmetic (cell_coord is monotone and its rounding error is ~1e-16 of the extent, the
  // margin is 1e-6 of it); anything closer to a face takes the exact path.
  float in_lo[3], in_hi[3];
  {
    const int N = A.G.resolution;
    const double inv_n = A.inv_resolution;
    const int ci[3] = {tile.cell / (N * N), (tile.cell / N) % N, tile.cell % N};
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double ext = A.G.hi[a] - A.G.lo[a];  // (a multiplication by 1/N instead of a division: the 1e-6 margin absorbs the ulp)
      in_lo[a] = (float)(A.G.lo[a] + ext * ((double)ci[a] * inv_n) + 1e-6 * ext);
      in_hi[a] = (float)(A.G.lo[a] + ext * ((double)(ci[a] + 1) * inv_n) - 1e-6 * ext);
    }
  }
  int n_active = tile.count;

  for (int inner = 0;; inner++) {
    if (SMALL) {
      if (lane < PTS) encode_into_swz<kSdfFreqs, PLD>(X, lane, px[0], py[0], pz[0]);
    } else {
#pragma unroll
      for (int q = 0; q < NQ; q++) encode_into<kSdfFreqs>(X, 0, col[q], px[q], py[q], pz[q]);
    }
    __syncwarp();
    if (inner == 0) {
      mbar_wait(&S.bar, parity);  // weights have landed
      parity ^= 1;
    }
    float dist[NQ];
    if (SMALL) {
      if (PTS == 32) hidden_layers_mid<kSdfIn, kSdfOutPad, ACT_SOFTPLUS, PLD>(X, S.w, lane);
      else hidden_layers_small<kSdfIn, kSdfOutPad, ACT_SOFTPLUS, PLD>(X, S.w, lane);
      dist[0] = lane < PTS ? output_distance_col<kSdfOutPad, PLD>(X, S.w + Blob::w3, S.w + Blob::b3, lane) : 0.0f;
    } else if (PLD == kPanelLd) {
      hidden_layers<kSdfIn, kSdfOutPad, ACT_SOFTPLUS>(X, S.w, lane);
      const float2 d2 = output_distance<kSdfOutPad>(X, S.w + Blob::w3, S.w + Blob::b3, lane);
      dist[0] = d2.x;
      dist[NQ - 1] = d2.y;
    }
    evals += (lane == 0) ? (unsigned long long)n_active : 0ull;
    slots += PTS;

    // ---- the march step for the lane's rays -----------------------------------------------------------
    int code[NQ], cell[NQ];
    bool stay[NQ];
    int n_stay = 0;
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      code[q] = STEP_DONE;
      cell[q] = -1;
      if (active[q]) {
        double t_next = 0.0;
        code[q] = ray_step(rr[q], A.M, ray[q], dist[q], t_next, A.crawl_below);
        if (code[q] != STEP_DONE) {
          // pts = origins + t * dirs in fp64 (surface.py:184), then the fp32 cast of grid.py:375
          px[q] = __double2float_rn(rr[q].o[0] + t_next * rr[q].d[0]);
          py[q] = __double2float_rn(rr[q].o[1] + t_next * rr[q].d[1]);
          pz[q] = __double2float_rn(rr[q].o[2] + t_next * rr[q].d[2]);
          const bool well_inside = px[q] > in_lo[0] && px[q] < in_hi[0] && py[q] > in_lo[1] && py[q] < in_hi[1] &&
                                   pz[q] > in_lo[2] && pz[q] < in_hi[2];
          cell[q] = well_inside ? tile.cell : cell_of_quick(px[q], py[q], pz[q], A.G.lo, A.G.hi, A.cell_scale, A.G.resolution);
          // a sample outside the box is not the filter's to decide (its bound was derived for coordinates inside it): keep
          // the ray in the exact queue instead of bouncing it through the filter queue
          if (code[q] == STEP_FILTER && !(fmaxf(fmaxf(fabsf(px[q]), fabsf(py[q])), fabsf(pz[q])) <= A.filter_x_raw)) code[q] = STEP_EXACT;
        }
      }
      stay[q] = code[q] == STEP_EXACT && cell[q] == tile.cell;
      n_stay += __popc(__ballot_sync(0xffffffffu, stay[q]));
    }
    // keep stepping in place while at least half of the tile's rays are still here
    const bool cont = n_stay > 0 && (A.keep_div > 0 ? A.keep_div : 2) * n_stay >= tile.count && inner + 1 < A.max_inner;
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      march_emit(A.next, A.live_out, code[q] == STEP_EXACT && !(cont && stay[q]), ray[q], rr[q], A.M, px[q], py[q], pz[q], cell[q]);
      march_emit(A.next_filter, A.live_filter, code[q] == STEP_FILTER, ray[q], rr[q], A.M, px[q], py[q], pz[q], cell[q]);
      active[q] = cont && stay[q];
      if (!active[q]) px[q] = py[q] = pz[q] = 0.f;
    }
    if (!cont) break;
    n_active = n_stay;
    __syncwarp();
  }
}

static __global__ void __launch_bounds__(32, kWarpCtasPerSm) march_warp_kernel(MarchTileArgs A) {
  using Blob = SdfBlob;
  using Smem = MlpSmem<kSdfIn, kSdfOutPad>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const MlpParams& P = A.P;
  const int n_tiles = P.ctr->n_tiles;
  uint32_t parity = 0;
  unsigned long long evals = 0, slots = 0;

  for (;;) {
    const int t = next_tile(P.ctr, lane);
    if (t >= n_tiles) break;
    const Tile tile = P.tiles[t];
    fetch_weights<Blob>(S.w, P.blobs, tile.cell, &S.bar, lane);
#ifdef KNF_MIXED_TILE_KERNEL
    if (tile.count <= kSmallTilePts) march_exact_tile<16, Smem, kPanelLd>(A, S, tile, lane, parity, evals, slots);
    else
#endif
      march_exact_tile<64, Smem, kPanelLd>(A, S, tile, lane, parity, evals, slots);  // one tile shape per kernel: half the instruction footprint
    __syncwarp();  // every lane is done reading S.w and the panel before the next tile overwrites them
  }
  if (lane == 0 && evals && A.eval_counter) {
    atomicAdd(A.eval_counter, evals);
    atomicAdd(A.eval_counter + 2, slots);  // lane slots spent (tile-fill statistic)
  }
}

// The exact kernel for SPARSE wavefronts: every tile was cut to <= 16 requests (RouteBuffers::small_tiles = 2) and this
// kernel holds nothing but the 4 x 4 path -- 14.3 KB of shared memory, half the registers and less than half the
// instruction footprint of march_warp_kernel, whose top stall in such wavefronts was instruction fetch.
#ifndef KNF_SMALL_CTAS_PER_SM
#define KNF_SMALL_CTAS_PER_SM 14
#endif
constexpr int kSmallCtasPerSm = KNF_SMALL_CTAS_PER_SM;
static __global__ void __launch_bounds__(32, kSmallCtasPerSm) march_small_kernel(MarchTileArgs A) {
  using Blob = SdfBlob;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SdfSmallSmem& S = *reinterpret_cast<SdfSmallSmem*>(smem_raw);
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const MlpParams& P = A.P;
  const int n_tiles = P.ctr->n_tiles;
  uint32_t parity = 0;
  unsigned long long evals = 0, slots = 0;
  for (;;) {
    const int t = next_tile(P.ctr, lane);
    if (t >= n_tiles) break;
    const Tile tile = P.tiles[t];
    fetch_weights<Blob>(S.w, P.blobs, tile.cell, &S.bar, lane);
    march_exact_tile<16, SdfSmallSmem, kSmallPanelLd>(A, S, tile, lane, parity, evals, slots);
    __syncwarp();
  }
  if (lane == 0 && evals && A.eval_counter) {
    atomicAdd(A.eval_counter, evals);
    atomicAdd(A.eval_counter + 2, slots);
  }
}

// The exact kernel for DENSE wavefronts in the mid shape: tiles of <= 32 requests (RouteBuffers::small_tiles = 4), 4 x 8
// register tiles, 16.8 KB of shared memory, 13 one-warp CTAs per SM (march_warp_kernel: 192 registers, 8 per SM).
#ifndef KNF_MID_CTAS_PER_SM
#define KNF_MID_CTAS_PER_SM 13
#endif
constexpr int kMidCtasPerSm = KNF_MID_CTAS_PER_SM;
static __global__ void __launch_bounds__(32, kMidCtasPerSm) march_mid_kernel(MarchTileArgs A) {
  using Blob = SdfBlob;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SdfMidSmem& S = *reinterpret_cast<SdfMidSmem*>(smem_raw);
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const MlpParams& P = A.P;
  const int n_tiles = P.ctr->n_tiles;
  uint32_t parity = 0;
  unsigned long long evals = 0, slots = 0;
  for (;;) {
    const int t = next_tile(P.ctr, lane);
    if (t >= n_tiles) break;
    const Tile tile = P.tiles[t];
    fetch_weights<Blob>(S.w, P.blobs, tile.cell, &S.bar, lane);
    march_exact_tile<32, SdfMidSmem, kMidPanelLd>(A, S, tile, lane, parity, evals, slots);
    __syncwarp();
  }
  if (lane == 0 && evals && A.eval_counter) {
    atomicAdd(A.eval_counter, evals);
    atomicAdd(A.eval_counter + 2, slots);
  }
}

// ---- the same kernel with the hidden layers on the tensor cores (knf_mma.cuh) ------------------------------
// Lane (g, t) owns tile points 16 t + g and 16 t + g + 8 (rows g, g + 8 of m-tile t), so the distance the quad
// butterfly leaves in every lane of quad g is picked up by the lane whose t equals the m-tile index.
//
// FILTER = false: the tensor-core distance IS the evaluation (KNF_PRECISION_TENSOR_*).
// FILTER = true : the DECISION FILTER of the exact mode.  98.5 % of the march evaluations of the BASELINE frame are
//   taken by rays crawling through a negative region with the fixed step scale * eps / 2 (surface.py:217-219): the
//   reference looks at such a distance only to see that it is still below -eps.  This kernel answers that
//   predicate from a tensor-core evaluation with a proven error bound delta (per cell, stored in the blob):
//   d_f < -(eps + delta) => d_exact < -eps, and the step is taken with the reference's own fp64 arithmetic.  Every
//   sample it cannot decide is handed, unchanged, to the exact kernel's queue of the same wavefront; a ray that
//   converges after filtered steps re-evaluates d_prev exactly first (PH_RECHECK).  Results are bit-identical to
//   running the exact kernel on every sample (tests/test_gpu_march.py::test_decision_filter_is_exact).
template <int PC, bool FILTER>
// A plain register cap instead of __launch_bounds__(32, n): with the latter ptxas squeezed the filter into 128 registers
// (spills) although 14 one-warp CTAs leave room for 146; measured 8.2 ms vs 8.6-8.9 ms of filter time per frame.
#ifndef KNF_MARCH_MMA_MAXNREG
#define KNF_MARCH_MMA_MAXNREG 144
#endif
static __global__ void __maxnreg__(KNF_MARCH_MMA_MAXNREG) march_mma_kernel(MarchTileArgs A) {
  using Blob = MmaBlobT<PC>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MmaMarchSmemT<PC>& S = *reinterpret_cast<MmaMarchSmemT<PC>*>(smem_raw);
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const MlpParams& P = A.P;
  const int n_tiles = P.ctr->n_tiles;
  const uint32_t* blobs = reinterpret_cast<const uint32_t*>(P.blobs);
  uint32_t parity = 0;
  unsigned evals = 0, slots = 0, deferred = 0, skipped = 0;  // per warp and launch: far below 2^32

  for (;;) {
    const int tix = next_tile(P.ctr, lane);
    if (tix >= n_tiles) break;
    const Tile tile = P.tiles[tix];
    fetch_mma_weights<PC, Blob::march_bytes>(S, blobs, tile.cell, lane);

    bool active[2];
    int ray[2] = {0, 0};
    int pidx[2];
    float px[2], py[2], pz[2];
    RayRegs rr[2];
#pragma unroll
    for (int q = 0; q < 2; q++) {
      pidx[q] = 16 * t + g + 8 * q;
      active[q] = pidx[q] < tile.count;
      px[q] = py[q] = pz[q] = 0.f;
      if (active[q]) {
        const float4 pt = P.sorted[tile.start + pidx[q]];  // (point, ray id): written by the routing scatter
        ray[q] = __float_as_int(pt.w);
        px[q] = pt.x; py[q] = pt.y; pz[q] = pt.z;
        ray_load_scalars(rr[q], A.M, ray[q]);  // in flight during the first pass
#pragma unroll
        for (int a = 0; a < 3; a++) {  // origin and direction go straight to shared memory (own slots only), also in flight
          cp_async_8(&S.od[a][32 * q + lane], A.M.o + 3 * (size_t)ray[q] + a);
          cp_async_8(&S.od[3 + a][32 * q + lane], A.M.d + 3 * (size_t)ray[q] + a);
        }
      }
    }
    float in_lo[3], in_hi[3], lip_pad[3];
    {
      const int N = A.G.resolution;
      const double inv_n = A.inv_resolution;
      const int ci[3] = {tile.cell / (N * N), (tile.cell / N) % N, tile.cell % N};
#pragma unroll
      for (int a = 0; a < 3; a++) {
        const double ext = A.G.hi[a] - A.G.lo[a];
        in_lo[a] = (float)(A.G.lo[a] + ext * ((double)ci[a] * inv_n) + 1e-6 * ext);
        in_hi[a] = (float)(A.G.lo[a] + ext * ((double)(ci[a] + 1) * inv_n) - 1e-6 * ext);
        lip_pad[a] = (float)((1e-6 + (double)kLipSlack * inv_n) * ext);  // inner box -> cell box + kLipSlack cell widths
      }
    }
    int n_active = tile.count;
    const float* W3d = reinterpret_cast<const float*>(S.w + Blob::w3d);  // output-layer column 0
    double safe_below = 0.0;
    float safe_below_f = 0.f;  // safe_below rounded down
    float lip[3] = {0.f, 0.f, 0.f};

    for (int inner = 0;; inner++) {
#pragma unroll
      for (int q = 0; q < 2; q++) {
        S.pts[0][pidx[q]] = px[q];
        S.pts[1][pidx[q]] = py[q];
        S.pts[2][pidx[q]] = pz[q];
      }
      // m-tiles that hold no active ray are skipped (warp-uniform): lanes with t == m own m-tile m
      const unsigned act_mask = __ballot_sync(0xffffffffu, active[0] || active[1]);
      __syncwarp();
      if (inner == 0) {
        mbar_wait(&S.bar, parity);
        parity ^= 1;
        if (FILTER) {
          safe_below = -(A.M.eps + (double)reinterpret_cast<const float*>(S.w + Blob::b3)[kFilterDeltaSlot]);
          safe_below_f = __double2float_rd(safe_below);
#pragma unroll
          for (int a = 0; a < 3; a++) lip[a] = reinterpret_cast<const float*>(S.w + Blob::b3)[kFilterLipSlot + a];
        }
      }
      const float b3 = reinterpret_cast<const float*>(S.w + Blob::b3)[0];
      float2 dist = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int m = 0; m < 4; m++) {
        if ((act_mask & (0x11111111u << m)) == 0) continue;
        float h2[4][4];
        mma_hidden<PC, FILTER, MmaMarchSmemT<PC>>(S, m, lane, h2);
        const float2 d = mma_output<1>(h2, W3d, b3, t, 0);
        if (m == t) dist = d;
        slots += 16;
      }
      evals += (lane == 0) ? (unsigned)n_active : 0u;
      if (inner == 0) cp_async_wait_all();  // the lane's own origin / direction slots

      int code[2], cell[2];
      bool stay[2];
#pragma unroll
      for (int q = 0; q < 2; q++) {
        code[q] = STEP_DONE;
        cell[q] = -1;
        if (active[q]) {
          double t_next = 0.0;
          code[q] = FILTER ? ray_filter_step(rr[q], A.M, ray[q], q ? dist.y : dist.x, safe_below, t_next,
                                             fmaxf(fmaxf(fabsf(px[q]), fabsf(py[q])), fabsf(pz[q])) <= A.filter_x_raw)
                           : ray_step(rr[q], A.M, ray[q], q ? dist.y : dist.x, t_next, A.crawl_below);
          if (FILTER && code[q] == STEP_EXACT) {
            cell[q] = tile.cell;  // undecided: the same sample goes to the exact queue of this wavefront
          } else if (code[q] != STEP_DONE) {
            const float x0 = px[q], y0 = py[q], z0 = pz[q];  // where d_f was evaluated
            // |d(p) - d(p0)| <= sum_a L_a |p_a - p0_a| inside the cell (L_a: proven per-axis Lipschitz bounds of the cell's
            // network), so every sample whose bound stays below `room` still has an exact distance below -eps: the
            // reference's evaluation there can only say "keep crawling", and its step is taken without evaluating.
            // (fp32, rounded towards less room: the fp64 pipe is the scarce one in this kernel)
            // (the bounds hold on the cell box plus a small margin, knf_bounds.cuh: no skipping from a sample clamped into this
            // cell from outside the grid)
            const bool p0_in = x0 >= in_lo[0] - lip_pad[0] && x0 <= in_hi[0] + lip_pad[0] && y0 >= in_lo[1] - lip_pad[1] &&
                               y0 <= in_hi[1] + lip_pad[1] && z0 >= in_lo[2] - lip_pad[2] && z0 <= in_hi[2] + lip_pad[2];
            const float room = (FILTER && A.max_skip > 0 && p0_in) ? __fmul_rd(__fsub_rd(safe_below_f, q ? dist.y : dist.x), 0.99999f) : 0.0f;
            for (;;) {
              px[q] = __double2float_rn(S.od[0][32 * q + lane] + t_next * S.od[3][32 * q + lane]);
              py[q] = __double2float_rn(S.od[1][32 * q + lane] + t_next * S.od[4][32 * q + lane]);
              pz[q] = __double2float_rn(S.od[2][32 * q + lane] + t_next * S.od[5][32 * q + lane]);
              const bool well_inside = px[q] > in_lo[0] && px[q] < in_hi[0] && py[q] > in_lo[1] && py[q] < in_hi[1] &&
                                       pz[q] > in_lo[2] && pz[q] < in_hi[2];
              cell[q] = well_inside ? tile.cell : cell_of_quick(px[q], py[q], pz[q], A.G.lo, A.G.hi, A.cell_scale, A.G.resolution);
              if (!FILTER || !well_inside) break;
              // (+ 1e-6 per axis: the fp32 roundings of the two points; the 0.99999 on `room` covers the fp32 arithmetic here)
              const float rise = lip[0] * (fabsf(px[q] - x0) + 1e-6f) + lip[1] * (fabsf(py[q] - y0) + 1e-6f) + lip[2] * (fabsf(pz[q] - z0) + 1e-6f);
              if (!(rise < room)) break;
              // the reference's march step at t_next (surface.py:217-223) with max(d, eps/2) = eps/2
              rr[q].steps += 1;
              rr[q].t_prev = rr[q].t;
              rr[q].t = rr[q].t + A.M.step_scale * (A.M.eps / 2);
              skipped += 1;
              if (rr[q].t > rr[q].t_far || rr[q].steps >= A.M.max_steps) {
                A.M.phase[ray[q]] = PH_DONE;
                A.M.steps[ray[q]] = rr[q].steps;
                code[q] = STEP_DONE;
                cell[q] = -1;
                break;
              }
              t_next = rr[q].t;
            }
          }
        }
        // rays that keep this kernel's kind of evaluation and stay in the cell may step in place
        stay[q] = code[q] == (FILTER ? STEP_FILTER : STEP_EXACT) && cell[q] == tile.cell;
      }
      const int n_stay = __popc(__ballot_sync(0xffffffffu, stay[0])) + __popc(__ballot_sync(0xffffffffu, stay[1]));
      const bool cont = n_stay > 0 && (A.keep_div > 0 ? A.keep_div : 2) * n_stay >= tile.count && inner + 1 < A.max_inner;
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const bool leaves = !(cont && stay[q]);
        if (FILTER) {
          march_emit(A.next_filter, A.live_filter, code[q] == STEP_FILTER && leaves, ray[q], rr[q], A.M, px[q], py[q], pz[q], cell[q]);
          march_emit(A.defer, A.live_defer, code[q] == STEP_EXACT, ray[q], rr[q], A.M, px[q], py[q], pz[q], cell[q]);
          deferred += (code[q] == STEP_EXACT) ? 1u : 0u;
        } else {
          march_emit(A.next, A.live_out, code[q] == STEP_EXACT && leaves, ray[q], rr[q], A.M, px[q], py[q], pz[q], cell[q]);
          march_emit(A.next_filter, A.live_filter, code[q] == STEP_FILTER, ray[q], rr[q], A.M, px[q], py[q], pz[q], cell[q]);
        }
        active[q] = cont && stay[q];
        if (!active[q]) px[q] = py[q] = pz[q] = 0.f;
      }
      if (!cont) break;
      n_active = n_stay;
      __syncwarp();
    }
    __syncwarp();
  }
  if (A.eval_counter) {
    if (FILTER) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        deferred += __shfl_xor_sync(0xffffffffu, deferred, off);
        skipped += __shfl_xor_sync(0xffffffffu, skipped, off);
      }
    }
    if (lane == 0 && evals) {
      atomicAdd(A.eval_counter + (FILTER ? 4 : 0), (unsigned long long)evals);
      if (FILTER) {
        atomicAdd(A.eval_counter + 5, (unsigned long long)deferred);
        atomicAdd(A.eval_counter + 6, (unsigned long long)skipped);
        atomicAdd(A.eval_counter + 7, (unsigned long long)slots);
      }
      else atomicAdd(A.eval_counter + 2, (unsigned long long)slots);
    }
  }
}

}  // namespace knf
