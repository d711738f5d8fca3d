// tc5_probe.cu -- what the decision filter needs to know about tcgen05 on B200 before it is built on it:
//  (1) do hand-made shared-memory descriptors (K-major, no swizzle: 8-row x 16-byte core matrices, LBO between
//      K chunks, SBO between 8-row groups) and the instruction descriptor give D = A . B^T for M = 128, N = 32;
//  (2) the same with A read from tensor memory (written by tcgen05.st, one TMEM lane per row);
//  (3) kind::tf32: are the low 13 mantissa bits of an fp32 container ignored (truncation), so x itself can be
//      the leading piece of a split;
//  (4) the accumulation error model: worst |error| / sum |a||b| of a K = 48 / K = 32 dot product of exactly
//      representable operands (the term the filter's proven bound delta needs);
//  (5) issue rate: back-to-back M128 N32 K16 MMAs per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc5_probe tc5_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t addr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// K-major, no swizzle: element (row, k) of a [rows x K] operand lives at
//   base + (k / EPC) * lbo + (row / 8) * sbo + (row % 8) * 16 + (k % EPC) * sizeof(elem),  EPC = 16 / sizeof(elem)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;                // base offset 0, layout type 0 = no swizzle
}
// kind::f16 / kind::tf32 instruction descriptor: D fp32, A and B of format `fmt` (0 f16, 1 bf16, 2 tf32), K-major.
__host__ __device__ constexpr uint32_t instr_desc(int fmt, int M, int N) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <bool TF32>
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  if (TF32)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc) : "memory");
}
template <bool TF32>
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, bool acc) {
  if (TF32)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem), "r"(a_tmem), "l"(b), "r"(idesc), "r"((uint32_t)acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem), "r"(a_tmem), "l"(b), "r"(idesc), "r"((uint32_t)acc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]),
        "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
               "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One CTA of 128 threads: D[128 x 32] = A[128 x K] . B[32 x K]^T.  A, B given in global memory as raw 32-bit words per
// row (K * sizeof(elem) / 4 words per row), row-major.  mode 0: A from shared memory, 1: A from tensor memory.
template <bool TF32, int K>
__global__ void __launch_bounds__(128) mma_probe(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B, float* __restrict__ D, int mode,
                                                 int reps, long long* cycles) {
  constexpr int ES = TF32 ? 4 : 2;          // element size
  constexpr int EPC = 16 / ES;              // elements per 16-byte chunk
  constexpr int KC = K / EPC;               // chunks along K
  constexpr int KSTEP = TF32 ? 8 : 16;      // K per MMA
  constexpr int WPR = K * ES / 4;           // words per row
  __shared__ __align__(128) uint8_t sA[KC * 128 * 16];
  __shared__ __align__(128) uint8_t sB[KC * 32 * 16];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_slot;
  const uint32_t lane_base = ((uint32_t)(warp * 32)) << 16;
  // operands -> shared memory (canonical layout); row = tid for A
  for (int c = 0; c < KC; c++) {
    uint4 v = *reinterpret_cast<const uint4*>(A + (size_t)tid * WPR + c * 4);
    *reinterpret_cast<uint4*>(sA + (size_t)c * 128 * 16 + tid * 16) = v;
    if (tid < 32) {
      uint4 w = *reinterpret_cast<const uint4*>(B + (size_t)tid * WPR + c * 4);
      *reinterpret_cast<uint4*>(sB + (size_t)c * 32 * 16 + tid * 16) = w;
    }
  }
  constexpr uint32_t A_COL0 = 64;  // TMEM columns of the A operand (mode 1): K * ES / 4 columns
  if (mode == 1) {
    for (int c8 = 0; c8 < WPR / 8; c8++) {
      uint32_t r[8];
      for (int i = 0; i < 8; i++) r[i] = A[(size_t)tid * WPR + c8 * 8 + i];
      tmem_st8(tmem + lane_base + A_COL0 + c8 * 8, r);
    }
    tmem_st_wait();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t idesc = instr_desc(TF32 ? 2 : 0, 128, 32);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int rep = 0; rep < reps; rep++) {
      for (int ks = 0; ks < K / KSTEP; ks++) {
        const int chunk = ks * (KSTEP / EPC);
        const uint64_t bdesc = smem_desc(smem_u32(sB) + chunk * 32 * 16, 32 * 16, 128);
        if (mode == 0) {
          const uint64_t adesc = smem_desc(smem_u32(sA) + chunk * 128 * 16, 128 * 16, 128);
          mma_ss<TF32>(tmem, adesc, bdesc, idesc, ks > 0);
        } else {
          mma_ts<TF32>(tmem, tmem + A_COL0 + ks * (KSTEP * ES / 4), bdesc, idesc, ks > 0);
        }
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  if (tid == 0) {
    t1 = clock64();
    if (cycles) cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_after();
  uint32_t r[32];
  tmem_ld32(tmem + lane_base, r);
  for (int j = 0; j < 32; j++) D[(size_t)blockIdx.x * 128 * 32 + (size_t)tid * 32 + j] = __uint_as_float(r[j]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}


// Issue-rate probe: `reps` rounds of MMAs (M128 x N x K16, f16) from one thread per CTA, rotating over n_acc independent
// accumulators (TMEM columns acc * N); operands are whatever shared memory holds.
template <int N>
__global__ void __launch_bounds__(128) mma_rate(int n_acc, int reps, int a_tmem, long long* cycles, int cols) {
  extern __shared__ __align__(128) uint8_t dyn[];
  uint8_t* sA = dyn;                 // 2 chunks x 128 rows x 16 B
  uint8_t* sB = dyn + 2 * 128 * 16;  // 2 chunks x N rows x 16 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (2 * 128 * 16 + 2 * N * 16) / 4; i += 128) reinterpret_cast<uint32_t*>(dyn)[i] = 0;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_slot, cols);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_slot;
  const uint32_t idesc = instr_desc(0, 128, N);
  if (tid == 0) {
    const uint64_t adesc = smem_desc(smem_u32(sA), 128 * 16, 128);
    const uint64_t bdesc = smem_desc(smem_u32(sB), N * 16, 128);
    const long long t0 = clock64();
    for (int rep = 0; rep < reps; rep++)
      for (int acc = 0; acc < n_acc; acc++) {
        if (a_tmem) mma_ts<false>(tmem + acc * N, tmem + cols - 8, bdesc, idesc, true);
        else mma_ss<false>(tmem + acc * N, adesc, bdesc, idesc, true);
      }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, cols);
}
template <int N>
static void rate(int n_acc, int a_tmem, int ctas_per_sm) {
  long long* dC;
  const int grid = 148 * ctas_per_sm;
  CK(cudaMalloc(&dC, grid * 8));
  const int reps = 4000 / n_acc;
  const int smem = 2 * 128 * 16 + 2 * N * 16;
  const int cols = 512 / ctas_per_sm;
  mma_rate<N><<<grid, 128, smem>>>(n_acc, reps, a_tmem, dC, cols);
  CK(cudaDeviceSynchronize());
  std::vector<long long> c(grid);
  CK(cudaMemcpy(c.data(), dC, grid * 8, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (auto v : c) avg += (double)v;
  avg /= grid;
  printf("rate N=%3d acc=%d A-%s ctas/SM=%d: %.1f cycles per MMA per CTA -> %.1f per SM\n", N, n_acc, a_tmem ? "tmem" : "smem", ctas_per_sm, avg / (reps * n_acc), avg / (reps * n_acc) / ctas_per_sm);
  cudaFree(dC);
}

static float half_round(float x) { return __half2float(__float2half_rn(x)); }

template <bool TF32, int K>
static void run(const char* name, int mode, std::vector<float>& a, std::vector<float>& b, bool report_model) {
  constexpr int ES = TF32 ? 4 : 2;
  constexpr int WPR = K * ES / 4;
  std::vector<uint32_t> ha(128 * WPR), hb(32 * WPR);
  auto pack = [&](const std::vector<float>& src, std::vector<uint32_t>& dst, int rows) {
    for (int r = 0; r < rows; r++)
      for (int k = 0; k < K; k++) {
        if (TF32) {
          memcpy(&dst[r * WPR + k], &src[r * K + k], 4);
        } else {
          __half h = __float2half_rn(src[r * K + k]);
          uint16_t u;
          memcpy(&u, &h, 2);
          uint32_t& w = dst[r * WPR + k / 2];
          if (k % 2 == 0) w = (w & 0xffff0000u) | u;
          else w = (w & 0x0000ffffu) | ((uint32_t)u << 16);
        }
      }
  };
  pack(a, ha, 128);
  pack(b, hb, 32);
  uint32_t *dA, *dB;
  float* dD;
  long long* dC;
  CK(cudaMalloc(&dA, ha.size() * 4));
  CK(cudaMalloc(&dB, hb.size() * 4));
  CK(cudaMalloc(&dD, 128 * 32 * 4));
  CK(cudaMalloc(&dC, 8));
  CK(cudaMemcpy(dA, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
  mma_probe<TF32, K><<<1, 128>>>(dA, dB, dD, mode, 1, dC);
  CK(cudaDeviceSynchronize());
  std::vector<float> d(128 * 32);
  CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0, worst_rel = 0, worst_trunc = 0;
  for (int r = 0; r < 128; r++)
    for (int n = 0; n < 32; n++) {
      double exact = 0, mag = 0, exact_trunc = 0;
      for (int k = 0; k < K; k++) {
        float x = a[r * K + k], w = b[n * K + k];
        if (!TF32) { x = half_round(x); w = half_round(w); }
        exact += (double)x * (double)w;
        mag += fabs((double)x * (double)w);
        if (TF32) {
          uint32_t xu, wu;
          memcpy(&xu, &x, 4); memcpy(&wu, &w, 4);
          xu &= 0xffffe000u; wu &= 0xffffe000u;
          float xt, wt;
          memcpy(&xt, &xu, 4); memcpy(&wt, &wu, 4);
          exact_trunc += (double)xt * (double)wt;
        }
      }
      double e = fabs((double)d[r * 32 + n] - exact);
      worst = fmax(worst, e);
      worst_rel = fmax(worst_rel, e / mag);
      if (TF32) worst_trunc = fmax(worst_trunc, fabs((double)d[r * 32 + n] - exact_trunc) / mag);
    }
  printf("%-34s mode %d (%s): worst |err| %.3e, worst |err|/sum|xw| %.3e = 2^%.2f", name, mode, mode ? "A in TMEM" : "A in smem", worst, worst_rel,
         log2(worst_rel));
  if (TF32) printf(", vs truncated-operand product 2^%.2f", log2(worst_trunc + 1e-300));
  printf("\n");
  (void)report_model;
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dC);
}


// Alignment probe: one product of 1.0 plus fifteen equal tiny products p = 1.5 * 2^-q in one K = 16 MMA.  What the fp32
// result keeps of the tiny addends shows where the tensor core truncates addends relative to the largest exponent.
static void alignment_probe() {
  std::vector<float> a(128 * 16), b(32 * 16);
  for (int r = 0; r < 128; r++) {
    const int q = 14 + (r % 32);          // p = 1.5 * 2^-q, q = 14 .. 45
    const int qa = q / 2, qb = q - qa;    // a = 1.5 * 2^-qa, b = 2^-qb (both normal fp16 for q <= 28; beyond: via subnormals / zero)
    a[r * 16] = 1.0f;
    for (int k = 1; k < 16; k++) a[r * 16 + k] = (r / 32 == 1 ? -1.0f : 1.0f) * ldexpf(1.5f, -std::min(qa, 14));
    (void)qb;
  }
  // B differs per column group: column n uses b = 2^-(q - qa) for the row's q -- but B is shared by all rows, so instead fix
  // b = 2^-14 (columns 0..7), 2^-10 (8..15), 2^-6 (16..23), 2^-2 (24..31) and let the row choose a's exponent.
  for (int n = 0; n < 32; n++) {
    b[n * 16] = 1.0f;
    for (int k = 1; k < 16; k++) b[n * 16 + k] = ldexpf(1.0f, -(14 - 4 * (n / 8)));
  }
  for (int r = 0; r < 128; r++) {
    const int ea = (r % 32) / 2;  // a = (1.5 or 1.0) * 2^-ea, ea = 0 .. 15 (fp16 normal down to 2^-14, 2^-15 subnormal but exact)
    const float mant = (r % 2) ? 1.5f : 1.0f;
    for (int k = 1; k < 16; k++) a[r * 16 + k] = (r / 32 == 1 ? -1.0f : 1.0f) * ldexpf(mant, -ea);
    if (r / 32 >= 2) a[r * 16] = (r / 32 == 2) ? 0.0f : 1024.0f;  // no large addend / a larger one
  }
  std::vector<uint32_t> ha(128 * 8), hb(32 * 8);
  auto packh = [](const std::vector<float>& src, std::vector<uint32_t>& dst, int rows) {
    for (int r = 0; r < rows; r++)
      for (int k = 0; k < 16; k += 2) {
        __half h0 = __float2half_rn(src[r * 16 + k]), h1 = __float2half_rn(src[r * 16 + k + 1]);
        uint16_t u0, u1;
        memcpy(&u0, &h0, 2); memcpy(&u1, &h1, 2);
        dst[r * 8 + k / 2] = u0 | ((uint32_t)u1 << 16);
      }
  };
  packh(a, ha, 128);
  packh(b, hb, 32);
  uint32_t *dA, *dB; float* dD;
  CK(cudaMalloc(&dA, ha.size() * 4)); CK(cudaMalloc(&dB, hb.size() * 4)); CK(cudaMalloc(&dD, 128 * 32 * 4));
  CK(cudaMemcpy(dA, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
  mma_probe<false, 16><<<1, 128>>>(dA, dB, dD, 0, 1, nullptr);
  CK(cudaDeviceSynchronize());
  std::vector<float> d(128 * 32);
  CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
  printf("alignment probe (K = 16, one MMA): big addend B0, fifteen addends p each; shown: log2(p / B0), exact (sum - B0) / ulp(B0), measured\n");
  double worst_rel = 0;
  for (int grp = 0; grp < 4; grp++) {
    const double big = grp == 2 ? 0.0 : (grp == 3 ? 1024.0 : 1.0);
    for (int r = grp * 32; r < grp * 32 + 32; r++)
      for (int n = 0; n < 32; n += 8) {
        const double p = (double)a[r * 16 + 1] * (double)b[n * 16 + 1];
        const double exact = big + 15.0 * p;
        const double ulp = big > 0 ? ldexp(1.0, (int)floor(log2(big)) - 23) : 0.0;
        const double meas = d[r * 32 + n];
        const double err = fabs(meas - exact);
        const double mag = fabs(big) + 15.0 * fabs(p);
        worst_rel = fmax(worst_rel, err / mag);
        if (big > 0 && fabs(p) / big < ldexp(1.0, -17) && fabs(p) / big > ldexp(1.0, -30) && (r % 2 == 1))
          printf("  grp %d log2(|p|/B0) = %6.2f  exact %+9.3f ulp  measured %+9.3f ulp\n", grp, log2(fabs(p) / big), (exact - big) / ulp, (meas - big) / ulp);
      }
  }
  printf("alignment probe: worst |err| / sum|xw| over all patterns = 2^%.2f\n", log2(worst_rel));
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

int main() {
  srand(1);
  alignment_probe();
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.0f - 1.0f; };
  {
    std::vector<float> a(128 * 48), b(32 * 48);
    for (auto& v : a) v = rnd();
    for (auto& v : b) v = rnd() * 0.4f;
    run<false, 48>("f16 K=48 random", 0, a, b, true);
    run<false, 48>("f16 K=48 random", 1, a, b, true);
    // structured: A[r][k] = r + k / 64 (exactly representable), B[n][k] = (k == n % 48): D[r][n] = A[r][n % 48]: layout check
    for (int r = 0; r < 128; r++) for (int k = 0; k < 48; k++) a[r * 48 + k] = (float)r + (float)k / 64.0f;
    for (int n = 0; n < 32; n++) for (int k = 0; k < 48; k++) b[n * 48 + k] = (k == (n * 5) % 48) ? 1.0f : 0.0f;
    run<false, 48>("f16 K=48 selector (layout)", 0, a, b, false);
    run<false, 48>("f16 K=48 selector (layout)", 1, a, b, false);
  }
  {
    std::vector<float> a(128 * 32), b(32 * 32);
    for (auto& v : a) v = rnd();
    for (auto& v : b) v = rnd() * 0.4f;
    run<false, 32>("f16 K=32 random", 0, a, b, true);
    run<false, 32>("f16 K=32 random", 1, a, b, true);
  }
  {
    std::vector<float> a(128 * 48), b(32 * 48);
    for (auto& v : a) v = rnd();
    for (auto& v : b) v = rnd() * 0.4f;
    run<true, 48>("tf32 K=48 random full fp32 bits", 0, a, b, true);
    run<true, 48>("tf32 K=48 random full fp32 bits", 1, a, b, true);
    for (auto& v : a) { uint32_t u; memcpy(&u, &v, 4); u &= 0xffffe000u; memcpy(&v, &u, 4); }
    for (auto& v : b) { uint32_t u; memcpy(&u, &v, 4); u &= 0xffffe000u; memcpy(&v, &u, 4); }
    run<true, 48>("tf32 K=48 pre-truncated operands", 0, a, b, true);
    run<true, 48>("tf32 K=48 pre-truncated operands", 1, a, b, true);
  }
  // accumulation model over many random draws (f16, exactly representable operands): worst error / sum |x w|
  {
    double worst48 = 0, worst32 = 0;
    (void)worst32;
    std::vector<float> a(128 * 48), b(32 * 48);
    uint32_t *dA, *dB; float* dD;
    CK(cudaMalloc(&dA, 128 * 24 * 4)); CK(cudaMalloc(&dB, 32 * 24 * 4)); CK(cudaMalloc(&dD, 128 * 32 * 4));
    std::vector<uint32_t> ha(128 * 24), hb(32 * 24);
    std::vector<float> d(128 * 32);
    for (int trial = 0; trial < 400; trial++) {
      const float sa = (trial % 4 == 0) ? 1.0f : (trial % 4 == 1) ? 30.0f : (trial % 4 == 2) ? 0.01f : 1.0f;
      for (auto& v : a) v = half_round(rnd() * sa * ((trial % 4 == 3 && rand() % 8 == 0) ? 1000.0f : 1.0f));
      for (auto& v : b) v = half_round(rnd() * 0.4f);
      for (int r = 0; r < 128; r++) for (int k = 0; k < 48; k += 2) {
        __half h0 = __float2half_rn(a[r * 48 + k]), h1 = __float2half_rn(a[r * 48 + k + 1]);
        uint16_t u0, u1; memcpy(&u0, &h0, 2); memcpy(&u1, &h1, 2);
        ha[r * 24 + k / 2] = u0 | ((uint32_t)u1 << 16);
      }
      for (int r = 0; r < 32; r++) for (int k = 0; k < 48; k += 2) {
        __half h0 = __float2half_rn(b[r * 48 + k]), h1 = __float2half_rn(b[r * 48 + k + 1]);
        uint16_t u0, u1; memcpy(&u0, &h0, 2); memcpy(&u1, &h1, 2);
        hb[r * 24 + k / 2] = u0 | ((uint32_t)u1 << 16);
      }
      CK(cudaMemcpy(dA, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dB, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
      mma_probe<false, 48><<<1, 128>>>(dA, dB, dD, trial & 1, 1, nullptr);
      CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
      for (int r = 0; r < 128; r++) for (int n = 0; n < 32; n++) {
        double exact = 0, mag = 0;
        for (int k = 0; k < 48; k++) { exact += (double)a[r * 48 + k] * b[n * 48 + k]; mag += fabs((double)a[r * 48 + k] * b[n * 48 + k]); }
        if (mag > 0) worst48 = fmax(worst48, fabs(d[r * 32 + n] - exact) / mag);
      }
    }
    printf("accumulation model, f16 K=48 (3 chained MMAs), 400 x 4096 outputs: worst |err|/sum|xw| = %.3e = 2^%.2f\n", worst48, log2(worst48));
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
  }
  // issue rate: reps x 3 MMAs (M128 N32 K16) from one thread, one CTA per SM
  {
    uint32_t *dA, *dB; float* dD; long long* dC;
    CK(cudaMalloc(&dA, 128 * 24 * 4)); CK(cudaMalloc(&dB, 32 * 24 * 4)); CK(cudaMalloc(&dD, (size_t)148 * 128 * 32 * 4)); CK(cudaMalloc(&dC, 148 * 8));
    CK(cudaMemset(dA, 0, 128 * 24 * 4)); CK(cudaMemset(dB, 0, 32 * 24 * 4));
    for (int mode = 0; mode < 2; mode++) {
      const int reps = 2000;
      mma_probe<false, 48><<<148, 128>>>(dA, dB, dD, mode, reps, dC);
      CK(cudaDeviceSynchronize());
      long long c[148];
      CK(cudaMemcpy(c, dC, sizeof(c), cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int i = 0; i < 148; i++) avg += (double)c[i];
      avg /= 148;
      printf("issue rate mode %d: %d MMAs (M128 N32 K16) in %.0f cycles -> %.1f cycles per MMA per SM\n", mode, reps * 3, avg, avg / (reps * 3));
    }
  }
  for (int a_tmem = 0; a_tmem < 2; a_tmem++) {
    rate<32>(1, a_tmem, 1); rate<32>(2, a_tmem, 1); rate<32>(4, a_tmem, 1); rate<32>(8, a_tmem, 1);
    rate<64>(1, a_tmem, 1); rate<64>(4, a_tmem, 1);
    rate<128>(1, a_tmem, 1); rate<128>(2, a_tmem, 1);
    rate<256>(1, a_tmem, 1);
    rate<32>(1, a_tmem, 2); rate<32>(2, a_tmem, 2); rate<32>(1, a_tmem, 4); rate<32>(2, a_tmem, 4); rate<32>(1, a_tmem, 8); rate<64>(1, a_tmem, 4); rate<64>(2, a_tmem, 2);
  }
  return 0;
}
