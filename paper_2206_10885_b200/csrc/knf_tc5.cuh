// knf_tc5.cuh -- the SDF tile MLP on Blackwell's 5th-generation tensor cores: tcgen05.mma issued by one thread per
// CTA, accumulators in tensor memory (TMEM), epilogues through tcgen05.ld (SASS UTCHMMA / LDTM).
//
// Work unit: a tile of <= 128 requests of ONE cell, one request per thread of a 128-thread CTA -- thread r owns TMEM
// lane r, i.e. row r of every accumulator, so bias / softplus / operand split / the 32 -> 1 output layer are all
// in-thread and nothing is shuffled.  Arithmetic is the fp16 x 2 operand split of knf_mma.cuh (x = x1 + x2' / 2^11,
// three piece products) laid out for M = 128 MMAs:
//
//   layer 1 (39 -> 32, K padded to 48; feature 39 is the constant 1 whose weight row is the bias b1):
//     D[:, 0:64]  = X1  . [W1a ; W1b']^T      3 x (M128 N64 K16)      big | small
//     D[:, 32:64] += X2' . W1a^T              3 x (M128 N32 K16)             small
//     z = D[:, 0:32] + D[:, 32:64] / 2^11 ; h1 = softplus(z)
//   layer 2 (32 -> 32):  the same with H1 pieces and [W2a ; W2b'], 2 + 2 MMAs, + b2, softplus
//   layer 3 (32 -> 1 or 32 -> 9): fp32 FMAs in the thread.
//
// 10 MMAs per 128 requests instead of 960 mma.sync.m16n8k16 (8 m-tiles x 120), and the warps' instruction streams hold
// only the Fourier features, the operand splits, the activations and the sphere-trace step.  Operands: A (activation
// pieces) is written by the threads into shared memory in the canonical K-major no-swizzle layout (8-row x 16-byte core
// matrices; thread r stores 16 contiguous bytes per K chunk: conflict-free STS.128); B (weight pieces) arrives in that
// layout from the per-cell blob with one TMA bulk copy.  Descriptors are built by hand (validated on B200 by
// scripts/micro/tc5_probe.cu: exact products, A from shared or tensor memory, kind::f16 / kind::tf32).
//
// Measured on B200 (profiles/tc5_probe_r2.txt): a K-chained MMA on one accumulator completes every ~200 cycles, MMAs on
// independent accumulators every ~105 per CTA, and CTAs overlap (8 CTAs per SM: 27 cycles per MMA per SM), so the kernel
// keeps several 128-thread CTAs per SM resident (64 TMEM columns each) instead of pipelining inside one CTA.
//
// Users: march_tc5_kernel -- the DECISION FILTER of the exact march (knf_march.cuh explains the filter; same predicate,
// same certified skipping, same proven-bound contract, results bit-identical to the exact kernel on every sample) --
// and sdf_tc5_kernel, the batched forward of KNF_PRECISION_TENSOR_FP16X2.
#pragma once

#include "knf_common.cuh"
#ifndef KNF_TC5_LAYOUT_ONLY
#include "knf_march.cuh"
#include "knf_mlp.cuh"
#include "knf_mma.cuh"
#include "knf_rays.cuh"
#endif

namespace knf {

// Activation of the filter kernel: 1 = one MUFU (ex2) + degree-5 polynomial ln(1 + e) (softplus_fast_poly_f2xN), 0 = two MUFU
// (ex2 + lg2, softplus_fast_f2xN).  The blob's bound delta is computed for the matching error constant (kTc5SoftplusErr).
#ifndef KNF_TC5_SOFTPLUS_POLY
#define KNF_TC5_SOFTPLUS_POLY 1
#endif
constexpr int kTc5Tile = 128;     // requests per tile = threads per CTA = TMEM lanes
constexpr int kTc5K1 = 48;        // layer-1 K: 39 features + the constant-1 bias feature + 8 zero columns
constexpr int kTc5BiasK = kSdfIn; // index of the constant-1 feature
constexpr int kTc5TmemCols = 64;  // D: big (0..31) | small (32..63)
constexpr float kTc5SoftplusErr = KNF_TC5_SOFTPLUS_POLY ? kFastSoftplusPolyErr : kFastSoftplusErr;
constexpr int kTc5AChunks = 5;    // K chunks (8 fp16 each) of an A piece the threads write: k = 0..39 (chunk 5 meets zero weights, see tc5_issue_layer)

// ---- per-cell blob ----------------------------------------------------------------------------------------------
//   B1: [chunk 0..5][row 0..63][8 fp16]   rows 0..31 = first pieces of W1 (row n = neuron n, k = chunk * 8 + i),
//                                         rows 32..63 = second pieces (scaled 2^11); k = 39 holds the bias pieces
//   B2: [chunk 0..3][row 0..63][8 fp16]   the same for W2
//   fp32: b2[32] | w3d[32] (output row 0: the distance) | b3[12] | delta | lip[3]        <- march kernels copy up to here
//         W3t[32][12] (k-major: all nine outputs, batched forward only)
struct Tc5Blob {
  static constexpr int b1_bytes = 6 * 64 * 16;   // 6144
  static constexpr int b2_bytes = 4 * 64 * 16;   // 4096
  static constexpr int off_b1 = 0;
  static constexpr int off_b2 = off_b1 + b1_bytes;
  static constexpr int off_f32 = off_b2 + b2_bytes;           // byte offset of the fp32 section
  static constexpr int f_b2 = 0, f_w3d = 32, f_b3 = 64, f_delta = 76, f_lip = 77, f_march_end = 80, f_w3t = 80;
  static constexpr int march_bytes = off_f32 + f_march_end * 4;          // 10560
  static constexpr int bytes = off_f32 + (f_w3t + kHidden * kSdfOutPad) * 4;  // 12096
  static_assert(march_bytes % 16 == 0 && bytes % 16 == 0, "blob (parts) must be multiples of 16 B for cp.async.bulk");
};

#ifndef KNF_TC5_LAYOUT_ONLY
// ---- PTX wrappers -----------------------------------------------------------------------------------------------
__device__ __forceinline__ void tc5_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc5_dealloc(uint32_t addr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols) : "memory");
}
__device__ __forceinline__ void tc5_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc5_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// K-major, no swizzle: element (row, k) of a [rows x K] fp16 operand lives at
//   base + (k / 8) * lbo + (row / 8) * 128 + (row % 8) * 16 + (k % 8) * 2
__device__ __forceinline__ uint64_t tc5_smem_desc(uint32_t addr, uint32_t lbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) | ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}
// kind::f16 instruction descriptor: D fp32, A = B = fp16, both K-major, M = 128
__host__ __device__ constexpr uint32_t tc5_idesc(int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }
__device__ __forceinline__ void tc5_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, bool accumulate) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem), "l"(a), "l"(b),
               "r"(idesc), "r"((uint32_t)accumulate)
               : "memory");
}
__device__ __forceinline__ void tc5_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// mbarrier wait for the tensor-core commits: the hardware parks the thread for up to `ns` before try_wait returns false, so
// the 128 waiting threads spend a couple of instructions per MMA batch instead of spinning through issue slots.
__device__ __forceinline__ void tc5_mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(20000u)
        : "memory");
  } while (!done);
}
// 16 consecutive TMEM columns of the thread's lane
__device__ __forceinline__ void tc5_ld16(uint32_t taddr, float (&r)[16]) {
  uint32_t u[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]), "=r"(u[8]), "=r"(u[9]),
                 "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; i++) r[i] = __uint_as_float(u[i]);
}
__device__ __forceinline__ void tc5_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- shared memory of one CTA -------------------------------------------------------------------------------------
struct Tc5MarchSmem {
  alignas(128) uint8_t w[Tc5Blob::march_bytes];      // B1 | B2 | fp32 constants
  alignas(128) uint8_t a[2 * kTc5AChunks * kTc5Tile * 16];  // A pieces: [piece][chunk 0..4][row][16 B] (layer 2 uses chunks 0..3)
  alignas(16) double od[6][kTc5Tile];                // resident rays' origins / directions, [component][thread]
  alignas(8) uint64_t bar_w;                         // weights landed (TMA transaction barrier)
  alignas(8) uint64_t bar_mma;                       // MMAs of the current layer done (tcgen05.commit)
  uint32_t tmem_slot;
  int tile_ix;
};

// fp16 x 2 split of 8 consecutive k (v[0..7]) -> the thread's 16 bytes of both A pieces at chunk `chunk`
__device__ __forceinline__ void tc5_store_chunk(uint8_t* a_base, int chunk, int row, const float (&v)[8]) {
  uint32_t p1[4], p2[4];
#pragma unroll
  for (int i = 0; i < 4; i++) split2h(v[2 * i], v[2 * i + 1], p1[i], p2[i]);
  *reinterpret_cast<uint4*>(a_base + ((0 * kTc5AChunks + chunk) * kTc5Tile + row) * 16) = make_uint4(p1[0], p1[1], p1[2], p1[3]);
  *reinterpret_cast<uint4*>(a_base + ((1 * kTc5AChunks + chunk) * kTc5Tile + row) * 16) = make_uint4(p2[0], p2[1], p2[2], p2[3]);
}

// nn.fourier_encode (nn.py:66-93) of the thread's point, operation for operation (the features the exact kernel sees),
// split and stored as layer-1 A pieces.  Feature k = 39 is the constant 1 (bias); k = 40..47 (chunk 5) is never stored.
__device__ __forceinline__ void tc5_encode_store(uint8_t* a_base, int row, float px, float py, float pz) {
  const float pi_f = 3.14159274101257324e+00f;  // float32(np.pi)
  float f[8 * kTc5AChunks];
  f[0] = px; f[1] = py; f[2] = pz;
  float2 sxy, cxy;
  np_sincosf2(__fmul2_rn(make_float2(pi_f, pi_f), make_float2(px, py)), sxy, cxy);
  float sz, cz;
  np_sincosf(__fmul_rn(pi_f, pz), sz, cz);
#pragma unroll
  for (int o = 0; o < kSdfFreqs; o++) {
    f[3 + 6 * o + 0] = sxy.x; f[3 + 6 * o + 1] = sxy.y; f[3 + 6 * o + 2] = sz;
    f[3 + 6 * o + 3] = cxy.x; f[3 + 6 * o + 4] = cxy.y; f[3 + 6 * o + 5] = cz;
    if (o + 1 < kSdfFreqs) {
      const float2 two_s = __fmul2_rn(make_float2(2.0f, 2.0f), sxy);
      const float2 ns = __fmul2_rn(two_s, cxy);                                    // 2 s c      (nn.py:88-92)
      const float2 ss = __fmul2_rn(two_s, sxy);
      cxy = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-ss.x, -ss.y));        // 1 - 2 s s
      sxy = ns;
      const float two_sz = __fmul_rn(2.0f, sz);
      const float nsz = __fmul_rn(two_sz, cz);
      cz = __fsub_rn(1.0f, __fmul_rn(two_sz, sz));
      sz = nsz;
    }
  }
  f[kTc5BiasK] = 1.0f;
  static_assert(kTc5BiasK == 8 * kTc5AChunks - 1, "the bias feature closes chunk 4");
#pragma unroll
  for (int c = 0; c < kTc5AChunks; c++) {
    const float v[8] = {f[8 * c], f[8 * c + 1], f[8 * c + 2], f[8 * c + 3], f[8 * c + 4], f[8 * c + 5], f[8 * c + 6], f[8 * c + 7]};
    tc5_store_chunk(a_base, c, row, v);
  }
}

// Issued by ONE thread: the MMAs of one layer (KS k-steps), then the commit that arrives on `bar` when they are done.
// K step 2 of layer 1 covers chunks 4 and 5.  The weights of chunk 5 (k = 40..47) are zero in the blob, so what the A side
// supplies there only has to be finite: its descriptor uses a leading-dimension stride of 0 and reads chunk 4 (finite
// features) a second time instead of 2 x 2 KB of stored zeros per CTA.
template <int KS>
__device__ __forceinline__ void tc5_issue_layer(uint32_t tmem, uint32_t a_addr, uint32_t b_addr, uint64_t* bar) {
  constexpr uint32_t a_lbo = kTc5Tile * 16, b_lbo = 64 * 16, a_piece = kTc5AChunks * kTc5Tile * 16;
#pragma unroll
  for (int pc = 0; pc < 2; pc++)    // pc 0: big | small = X1 . [Wa ; Wb']^T (N = 64);  pc 1: small += X2' . Wa^T (N = 32)
#pragma unroll
    for (int ks = 0; ks < KS; ks++) {
      const uint32_t a0 = a_addr + pc * a_piece + ks * 2 * a_lbo;
      const uint32_t lbo = (ks == 2) ? 0u : a_lbo;
      tc5_mma(tmem + 32 * pc, tc5_smem_desc(a0, lbo), tc5_smem_desc(b_addr + ks * 2 * b_lbo, b_lbo), tc5_idesc(pc ? 32 : 64), pc > 0 || ks > 0);
    }
  tc5_commit(bar);
}

// Pre-activations of hidden units [16 h, 16 h + 16) of the thread's row from TMEM: big + small / 2^11 (+ bias).
__device__ __forceinline__ void tc5_load_half(uint32_t taddr_lane, int h, const float* __restrict__ bias, float2 (&z)[8]) {
  float big[16], small[16];
  tc5_ld16(taddr_lane + 16 * h, big);
  tc5_ld16(taddr_lane + 32 + 16 * h, small);
  tc5_ld_wait();
#pragma unroll
  for (int i = 0; i < 8; i++) {
    z[i] = __ffma2_rn(make_float2(small[2 * i], small[2 * i + 1]), make_float2(1.0f / kHalfPieceScale, 1.0f / kHalfPieceScale),
                      make_float2(big[2 * i], big[2 * i + 1]));
    if (bias) z[i] = __fadd2_rn(z[i], *reinterpret_cast<const float2*>(bias + 16 * h + 2 * i));
  }
}

#ifndef KNF_TC5_LAYOUT_ONLY
template <int N>
__device__ __forceinline__ void tc5_softplus(float2 (&z)[N]) {
  if (KNF_TC5_SOFTPLUS_POLY) softplus_fast_poly_f2xN<N>(z);
  else softplus_fast_f2xN<N>(z);
}
#endif

#ifndef KNF_TC5_CTAS_PER_SM
#define KNF_TC5_CTAS_PER_SM 6
#endif
constexpr int kTc5CtasPerSm = KNF_TC5_CTAS_PER_SM;

// ---- the decision filter on tcgen05 --------------------------------------------------------------------------------
// Same contract as march_mma_kernel<2, true> (knf_march.cuh): a filter distance d_f with |d_f - d_exact| < delta (per
// cell, stored in the blob) answers the reference's predicate d < -eps; undecided samples go, unchanged, to the exact
// queue of this wavefront; certified skipping by the per-axis Lipschitz bounds; tile residency.
static __global__ void __launch_bounds__(kTc5Tile, kTc5CtasPerSm) march_tc5_kernel(MarchTileArgs A) {
  extern __shared__ __align__(128) unsigned char tc5_smem_raw[];
  Tc5MarchSmem& S = *reinterpret_cast<Tc5MarchSmem*>(tc5_smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&S.bar_w, 1);
    mbar_init(&S.bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tc5_alloc(&S.tmem_slot, kTc5TmemCols);
  tc5_fence_before();
  __syncthreads();
  tc5_fence_after();
  const uint32_t tmem = S.tmem_slot;
  const uint32_t tmem_lane = tmem + ((uint32_t)(warp * 32) << 16);
  const MlpParams& P = A.P;
  const int n_tiles = P.ctr->n_tiles;
  const uint8_t* blobs = reinterpret_cast<const uint8_t*>(P.blobs);
  const float* F32 = reinterpret_cast<const float*>(S.w + Tc5Blob::off_f32);
  uint32_t par_w = 0, par_mma = 0;
  unsigned evals = 0, slots = 0, deferred = 0, skipped = 0;

  for (;;) {
    if (tid == 0) S.tile_ix = atomicAdd(&P.ctr->tile_cursor, 1);
    __syncthreads();  // also: every thread is done with the previous tile's shared memory
    const int tix = S.tile_ix;
    if (tix >= n_tiles) break;
    const Tile tile = P.tiles[tix];
    if (tid == 0) {
      fence_proxy_async();
      mbar_expect_tx(&S.bar_w, Tc5Blob::march_bytes);
      bulk_copy_g2s(S.w, blobs + (size_t)tile.cell * Tc5Blob::bytes, Tc5Blob::march_bytes, &S.bar_w);
    }
    bool active = tid < tile.count;
    int ray = 0;
    float px = 0.f, py = 0.f, pz = 0.f;
    RayRegs rr;
    if (active) {
      const float4 pt = P.sorted[tile.start + tid];  // (point, ray id): written by the routing scatter
      ray = __float_as_int(pt.w);
      px = pt.x; py = pt.y; pz = pt.z;
      ray_load_scalars(rr, A.M, ray);
#pragma unroll
      for (int a = 0; a < 3; a++) {
        cp_async_8(&S.od[a][tid], A.M.o + 3 * (size_t)ray + a);
        cp_async_8(&S.od[3 + a][tid], A.M.d + 3 * (size_t)ray + a);
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
    double safe_below = 0.0;
    float safe_below_f = 0.f, lip[3] = {0.f, 0.f, 0.f}, b3 = 0.f;

    for (int inner = 0;; inner++) {
      // ---- layer 1 operands ---------------------------------------------------------------------------------------
      const bool warp_active = __any_sync(0xffffffffu, active);
      if (warp_active) tc5_encode_store(S.a, tid, px, py, pz);  // (inactive lanes of a live warp encode the origin: finite, ignored)
      fence_proxy_async();  // the threads' shared-memory writes -> visible to the tensor core (async proxy)
      tc5_fence_before();
      __syncthreads();
      if (tid == 0) {
        if (inner == 0) {
          mbar_wait(&S.bar_w, par_w);  // weights have landed
        }
        tc5_fence_after();
        tc5_issue_layer<3>(tmem, smem_u32(S.a), smem_u32(S.w + Tc5Blob::off_b1), &S.bar_mma);
      }
      if (inner == 0) {
        mbar_wait(&S.bar_w, par_w);  // every thread reads the cell's constants below
        par_w ^= 1;
        safe_below = -(A.M.eps + (double)F32[Tc5Blob::f_delta]);
        safe_below_f = __double2float_rd(safe_below);
#pragma unroll
        for (int a = 0; a < 3; a++) lip[a] = F32[Tc5Blob::f_lip + a];
        b3 = F32[Tc5Blob::f_b3];
      }
      tc5_mbar_wait(&S.bar_mma, par_mma);
      par_mma ^= 1;
      tc5_fence_after();
      // ---- h1 = softplus(layer 1) -> layer-2 operands ----------------------------------------------------------------
#pragma unroll
      for (int h = 0; h < 2; h++) {
        float2 z[8];
        tc5_load_half(tmem_lane, h, nullptr, z);  // the bias came in through feature 39
        if (warp_active) {
          tc5_softplus<8>(z);
#pragma unroll
          for (int c = 0; c < 2; c++) {
            const float v[8] = {z[4 * c].x, z[4 * c].y, z[4 * c + 1].x, z[4 * c + 1].y, z[4 * c + 2].x, z[4 * c + 2].y, z[4 * c + 3].x, z[4 * c + 3].y};
            tc5_store_chunk(S.a, 2 * h + c, tid, v);
          }
        }
      }
      fence_proxy_async();
      tc5_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc5_fence_after();
        tc5_issue_layer<2>(tmem, smem_u32(S.a), smem_u32(S.w + Tc5Blob::off_b2), &S.bar_mma);
      }
      tc5_mbar_wait(&S.bar_mma, par_mma);
      par_mma ^= 1;
      tc5_fence_after();
      // ---- h2 = softplus(layer 2 + b2); d_f = w3 . h2 + b3 -------------------------------------------------------------
      float dist = b3;
      {
        float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int h = 0; h < 2; h++) {
          float2 z[8];
          tc5_load_half(tmem_lane, h, F32 + Tc5Blob::f_b2, z);
          if (warp_active) {
            tc5_softplus<8>(z);
#pragma unroll
            for (int i = 0; i < 8; i++) acc = __ffma2_rn(z[i], *reinterpret_cast<const float2*>(F32 + Tc5Blob::f_w3d + 16 * h + 2 * i), acc);
          }
        }
        dist = __fadd_rn(__fadd_rn(acc.x, acc.y), b3);
      }
      evals += (tid == 0) ? (unsigned)n_active : 0u;
      slots += (lane == 0 && warp_active) ? 32u : 0u;  // lane slots spent: warps without a live ray skip the arithmetic
      if (inner == 0) cp_async_wait_all();  // the thread's own origin / direction slots

      // ---- the march step (identical to march_mma_kernel<2, true>) ---------------------------------------------------------
      int code = STEP_DONE, cell = -1;
      if (active) {
        double t_next = 0.0;
        code = ray_filter_step(rr, A.M, ray, dist, safe_below, t_next, fmaxf(fmaxf(fabsf(px), fabsf(py)), fabsf(pz)) <= A.filter_x_raw);
        if (code == STEP_EXACT) {
          cell = tile.cell;  // undecided: the same sample goes to the exact queue of this wavefront
        } else if (code != STEP_DONE) {
          const float x0 = px, y0 = py, z0 = pz;  // where d_f was evaluated
          // the Lipschitz bounds hold on the cell box plus a small margin (knf_bounds.cuh): no skipping from a sample that was
          // clamped into this cell from outside the grid
          const bool p0_in = x0 >= in_lo[0] - lip_pad[0] && x0 <= in_hi[0] + lip_pad[0] && y0 >= in_lo[1] - lip_pad[1] &&
                             y0 <= in_hi[1] + lip_pad[1] && z0 >= in_lo[2] - lip_pad[2] && z0 <= in_hi[2] + lip_pad[2];
          const float room = (A.max_skip > 0 && p0_in) ? __fmul_rd(__fsub_rd(safe_below_f, dist), 0.99999f) : 0.0f;
          const double dt = A.M.step_scale * (A.M.eps / 2);  // the crawl step (surface.py:217-223 with max(d, eps/2) = eps/2)
          // ---- certified skipping, part 1: a run of samples certified in closed form (the ray's cell-exit parameter from
          // the grid DDA and the Lipschitz budget bound the run; no per-sample arithmetic).  Sample j (j = 1 is t_next)
          // lies j * dt along the ray from p0, so per axis |p_j - p0| <= j dt |d_a| (1 + 2^-20) + two fp32 roundings, and
          // it is certified when it stays inside the cell's inner box and sum_a L_a (|p_j - p0|_a + 1e-6) < room.  J is
          // taken 2 samples short of either limit and scaled by 0.999 against the fp32 arithmetic here; part 2 below
          // re-checks the remaining samples one by one with the exact per-sample test.
          if (room > 0.0f && A.max_skip > 1) {
            const float dtf = __double2float_ru(dt);
            float run = 1.0e9f, rise_per_step = 0.0f, lip_sum = 0.0f;
            const float p0[3] = {x0, y0, z0};
#pragma unroll
            for (int a = 0; a < 3; a++) {
              const double da = S.od[3 + a][tid];
              const float ad = __double2float_ru(fabs(da)) * 1.000002f;
              const float gap = da > 0.0 ? in_hi[a] - p0[a] : p0[a] - in_lo[a];  // distance to the face the ray moves towards
              const float stepa = ad * dtf;
              if (stepa > 0.0f) run = fminf(run, __fdividef(fmaxf(gap, 0.0f), stepa));
              rise_per_step += lip[a] * stepa;
              lip_sum += lip[a];
            }
            const float budget = room - 1.0e-6f * lip_sum;
            if (rise_per_step > 0.0f) run = fminf(run, budget > 0.0f ? __fdividef(budget, rise_per_step) : 0.0f);
            int J = (int)fminf(run * 0.999f, 1.0e6f) - 2;  // samples 1 .. J are certified
            // The reference's steps through samples 1 .. J: J rounded fp64 additions t <- fl(t + dt).  Inside one binade
            // [2^e, 2^(e+1)) every t is a multiple of u = 2^(e-52), so fl(t + dt) = t + D with the SAME D = rn_u(dt) at every
            // step (unless dt's remainder is an exact tie, where the parity of t / u decides): t_j = t0 + j D, and j D and the
            // sum are exactly representable.  D = fl(t0 + dt) - t0 is the first of those additions itself.  So the run -- and
            // the step at which it would pass t_far or exhaust max_steps -- is taken in closed form, bit for bit; a run that
            // could leave the binade (t crossing a power of two), a tie, or t0 <= 0 takes the loop below instead.
            if (J > 0) {
              const double t0 = rr.t;
              const long long eb = __double_as_longlong(t0) & 0x7ff0000000000000ll;
              const double top = __longlong_as_double(eb + 0x0010000000000000ll);  // 2^(e+1)
              const double u = __longlong_as_double(eb - (52ll << 52));            // 2^(e-52)
              const double D = (t0 + dt) - t0;
              const bool closed = t0 > 0.0 && eb > (60ll << 52) && D > 0.0 && fabs(dt - D) * 2.0 != u && J < (1 << 20) &&
                                  t0 + (double)(J + 2) * dt < top;
              if (closed) {
                int m = J;
                bool done = false;
                const int m_steps = max(1, A.M.max_steps - rr.steps);  // the addition after which steps reaches max_steps
                if (m_steps <= m) { m = m_steps; done = true; }
                if (t0 + (double)m * D > rr.t_far) {  // the first m additions pass t_far: find the first that does
                  int mf = (int)fmin(floor((rr.t_far - t0) / D), 2.0e6) + 1;
                  mf = max(1, min(mf, m));
                  while (mf > 1 && t0 + (double)(mf - 1) * D > rr.t_far) mf--;
                  while (mf < m && !(t0 + (double)mf * D > rr.t_far)) mf++;
                  m = mf;
                  done = true;
                }
                rr.steps += m;
                rr.t_prev = t0 + (double)(m - 1) * D;
                rr.t = t0 + (double)m * D;
                skipped += (unsigned)m;
                if (done) {
                  A.M.phase[ray] = PH_DONE;
                  A.M.steps[ray] = rr.steps;
                  code = STEP_DONE;
                }
              } else {
                for (int j = 0; j < J; j++) {
                  rr.steps += 1;
                  rr.t_prev = rr.t;
                  rr.t = rr.t + dt;
                  skipped += 1;
                  if (rr.t > rr.t_far || rr.steps >= A.M.max_steps) {
                    A.M.phase[ray] = PH_DONE;
                    A.M.steps[ray] = rr.steps;
                    code = STEP_DONE;
                    break;
                  }
                }
              }
            }
            t_next = rr.t;
          }
          // ---- part 2: the remaining samples, one by one (exact point, exact box test, exact rise) ---------------------
          for (int it = 0; code != STEP_DONE; it++) {
            px = __double2float_rn(S.od[0][tid] + t_next * S.od[3][tid]);
            py = __double2float_rn(S.od[1][tid] + t_next * S.od[4][tid]);
            pz = __double2float_rn(S.od[2][tid] + t_next * S.od[5][tid]);
            const bool well_inside = px > in_lo[0] && px < in_hi[0] && py > in_lo[1] && py < in_hi[1] && pz > in_lo[2] && pz < in_hi[2];
            cell = well_inside ? tile.cell : cell_of_quick(px, py, pz, A.G.lo, A.G.hi, A.cell_scale, A.G.resolution);
            if (!well_inside || it >= A.skip_cap) break;  // (the cap bounds how long one lane can hold up its warp and CTA)
            const float rise = lip[0] * (fabsf(px - x0) + 1e-6f) + lip[1] * (fabsf(py - y0) + 1e-6f) + lip[2] * (fabsf(pz - z0) + 1e-6f);
            if (!(rise < room)) break;
            rr.steps += 1;
            rr.t_prev = rr.t;
            rr.t = rr.t + dt;
            skipped += 1;
            if (rr.t > rr.t_far || rr.steps >= A.M.max_steps) {
              A.M.phase[ray] = PH_DONE;
              A.M.steps[ray] = rr.steps;
              code = STEP_DONE;
              cell = -1;
              break;
            }
            t_next = rr.t;
          }
          if (code == STEP_DONE) cell = -1;
        }
      }
      const bool stay = code == STEP_FILTER && cell == tile.cell;
      const int n_stay = __syncthreads_count(stay);
      const bool cont = n_stay > 0 && (A.keep_div > 0 ? A.keep_div : 2) * n_stay >= tile.count && inner + 1 < A.max_inner;
      const bool leaves = !(cont && stay);
      march_emit(A.next_filter, A.live_filter, code == STEP_FILTER && leaves, ray, rr, A.M, px, py, pz, cell);
      march_emit(A.defer, A.live_defer, code == STEP_EXACT, ray, rr, A.M, px, py, pz, cell);
      deferred += (code == STEP_EXACT) ? 1u : 0u;
      active = cont && stay;
      if (!active) px = py = pz = 0.f;
      if (!cont) break;
      n_active = n_stay;
    }
  }
  if (A.eval_counter) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      deferred += __shfl_xor_sync(0xffffffffu, deferred, off);
      skipped += __shfl_xor_sync(0xffffffffu, skipped, off);
    }
    if (lane == 0) {
      if (evals) atomicAdd(A.eval_counter + 4, (unsigned long long)evals);
      if (deferred) atomicAdd(A.eval_counter + 5, (unsigned long long)deferred);
      if (skipped) atomicAdd(A.eval_counter + 6, (unsigned long long)skipped);
      if (slots) atomicAdd(A.eval_counter + 7, (unsigned long long)slots);
    }
  }
  tc5_fence_before();
  __syncthreads();
  if (warp == 0) tc5_dealloc(tmem, kTc5TmemCols);
}


// ---- batched forward on tcgen05 (grid.sdf_query / sdf_values in KNF_PRECISION_TENSOR_FP16X2) -------------------------
// Same tile, same operand pieces, an accurate polynomial softplus (softplus_f2xN: 0.42 ulp mean against float64, like
// NumPy's) instead of the filter's MUFU one, and all nine outputs: out[j] = sum_k h2[k] W3[j][k] + b3[j] as in-thread fp32 FMAs in ascending k.
struct Tc5FwdSmem {
  alignas(128) uint8_t w[Tc5Blob::bytes];            // B1 | B2 | fp32 constants | W3t
  alignas(128) uint8_t a[2 * kTc5AChunks * kTc5Tile * 16];
  alignas(8) uint64_t bar_w;
  alignas(8) uint64_t bar_mma;
  uint32_t tmem_slot;
  int tile_ix;
};

static __global__ void __launch_bounds__(kTc5Tile, kTc5CtasPerSm) sdf_tc5_kernel(MlpParams P) {
  extern __shared__ __align__(128) unsigned char tc5_smem_raw[];
  Tc5FwdSmem& S = *reinterpret_cast<Tc5FwdSmem*>(tc5_smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&S.bar_w, 1);
    mbar_init(&S.bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tc5_alloc(&S.tmem_slot, kTc5TmemCols);
  tc5_fence_before();
  __syncthreads();
  tc5_fence_after();
  const uint32_t tmem = S.tmem_slot;
  const uint32_t tmem_lane = tmem + ((uint32_t)(warp * 32) << 16);
  const int n_tiles = P.ctr->n_tiles;
  const uint8_t* blobs = reinterpret_cast<const uint8_t*>(P.blobs);
  const float* F32 = reinterpret_cast<const float*>(S.w + Tc5Blob::off_f32);
  uint32_t par_w = 0, par_mma = 0;

  for (;;) {
    if (tid == 0) S.tile_ix = atomicAdd(&P.ctr->tile_cursor, 1);
    __syncthreads();  // also: every thread is done with the previous tile's shared memory
    const int tix = S.tile_ix;
    if (tix >= n_tiles) break;
    const Tile tile = P.tiles[tix];
    if (tid == 0) {
      fence_proxy_async();
      mbar_expect_tx(&S.bar_w, Tc5Blob::bytes);
      bulk_copy_g2s(S.w, blobs + (size_t)tile.cell * Tc5Blob::bytes, Tc5Blob::bytes, &S.bar_w);
    }
    int slot = -1;
    float4 pt = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid < tile.count) {
      slot = P.perm[tile.start + tid];
      pt = P.req_pt[slot];
    }
    const bool warp_active = __any_sync(0xffffffffu, slot >= 0);
    if (warp_active) tc5_encode_store(S.a, tid, pt.x, pt.y, pt.z);
    fence_proxy_async();
    tc5_fence_before();
    __syncthreads();
    if (tid == 0) {
      mbar_wait(&S.bar_w, par_w);
      tc5_fence_after();
      tc5_issue_layer<3>(tmem, smem_u32(S.a), smem_u32(S.w + Tc5Blob::off_b1), &S.bar_mma);
    }
    tc5_mbar_wait(&S.bar_mma, par_mma);
    par_mma ^= 1;
    tc5_fence_after();
#pragma unroll
    for (int h = 0; h < 2; h++) {
      float2 z[8];
      tc5_load_half(tmem_lane, h, nullptr, z);
      if (warp_active) {
        softplus_f2xN<8>(z);  // 24 packed steps per pair; as accurate against float64 as NumPy's own (knf_common.cuh), not bit-equal to it
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const float v[8] = {z[4 * c].x, z[4 * c].y, z[4 * c + 1].x, z[4 * c + 1].y, z[4 * c + 2].x, z[4 * c + 2].y, z[4 * c + 3].x, z[4 * c + 3].y};
          tc5_store_chunk(S.a, 2 * h + c, tid, v);
        }
      }
    }
    fence_proxy_async();
    tc5_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc5_fence_after();
      tc5_issue_layer<2>(tmem, smem_u32(S.a), smem_u32(S.w + Tc5Blob::off_b2), &S.bar_mma);
    }
    mbar_wait(&S.bar_w, par_w);  // (long complete: the fp32 constants are read below by every thread)
    par_w ^= 1;
    tc5_mbar_wait(&S.bar_mma, par_mma);
    par_mma ^= 1;
    tc5_fence_after();
    // outputs 0..8 (+ 3 pad columns) as six packed accumulators, ascending k
    float2 acc[6];
#pragma unroll
    for (int j = 0; j < 6; j++) acc[j] = *reinterpret_cast<const float2*>(F32 + Tc5Blob::f_b3 + 2 * j);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      float2 z[8];
      tc5_load_half(tmem_lane, h, F32 + Tc5Blob::f_b2, z);
      if (warp_active) {
        softplus_f2xN<8>(z);  // 24 packed steps per pair; as accurate against float64 as NumPy's own (knf_common.cuh), not bit-equal to it
#pragma unroll
        for (int i = 0; i < 16; i++) {
          const float hv = (i & 1) ? z[i >> 1].y : z[i >> 1].x;
          const float4* wrow = reinterpret_cast<const float4*>(F32 + Tc5Blob::f_w3t + (16 * h + i) * kSdfOutPad);
          const float4 w0 = wrow[0], w1 = wrow[1], w2 = wrow[2];
          acc[0] = __ffma2_rn(splat(hv), make_float2(w0.x, w0.y), acc[0]);
          acc[1] = __ffma2_rn(splat(hv), make_float2(w0.z, w0.w), acc[1]);
          acc[2] = __ffma2_rn(splat(hv), make_float2(w1.x, w1.y), acc[2]);
          acc[3] = __ffma2_rn(splat(hv), make_float2(w1.z, w1.w), acc[3]);
          acc[4] = __ffma2_rn(splat(hv), make_float2(w2.x, w2.y), acc[4]);
        }
      }
    }
    if (slot >= 0) {
      if (P.out_first) P.out_first[slot] = acc[0].x;
      if (P.out_full) {
        float* o = P.out_full + (size_t)slot * kSdfOut;
        o[0] = acc[0].x; o[1] = acc[0].y; o[2] = acc[1].x; o[3] = acc[1].y; o[4] = acc[2].x;
        o[5] = acc[2].y; o[6] = acc[3].x; o[7] = acc[3].y; o[8] = acc[4].x;
      }
    }
  }
  tc5_fence_before();
  __syncthreads();
  if (warp == 0) tc5_dealloc(tmem, kTc5TmemCols);
}

#endif  // KNF_TC5_LAYOUT_ONLY

}  // namespace knf
