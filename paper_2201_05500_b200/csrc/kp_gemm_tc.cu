// fp32-accurate GEMM on the 5th-generation tensor cores (tcgen05, 3xTF32).
//
//   C[m][n] = epi( sum_k A[m][k] * B[n][k] )      A, B K-major fp32
//
// The MLP's forward (Z = X W^T) and input-gradient (dX = dZ W, with W^T kept
// as a K-major copy) products. Inputs stay fp32 in HBM; each operand x is
// split as hi = x with the low 13 mantissa bits ignored (what kind::tf32
// reads) and lo = x - hi, and three tcgen05.mma per k-step accumulate
// A*B + A*B_lo + A_lo*B in a TMEM fp32 accumulator (the dropped lo*lo term is
// ~2^-21 relative): fp32-level accuracy at tensor-core rate.
//
// CTA = one 128 x BN output tile, 192 threads, warp-specialised:
//   warp 0    TMA producer: A tile (128x32) + B, B_lo tiles (BNx32) per stage,
//             128B-swizzled (the canonical K-major SW128 UMMA layout)
//   warp 1    TMEM allocator + single-thread MMA issuer (tcgen05.mma/commit)
//   warps 2-5 A_lo converters (smem -> smem, fence.proxy.async), then the
//             epilogue (tcgen05.ld 32x32b -> bias/activation/derivative -> HBM)
// Pipelines: full[s] (TMA tx bytes) -> conv[s] (128 arrivals) -> MMA ->
// empty[s] (tcgen05.commit) back to the producer; done -> epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "kp_internal.cuh"

namespace kp {
namespace {

constexpr int TC_BM = 128, TC_BN = 128, TC_BK = 32, TC_STAGES = 3;
constexpr int TC_THREADS = 192;
constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4;   // 16 KB
constexpr uint32_t B_BYTES = TC_BN * TC_BK * 4;   // 16 KB
constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr uint32_t SMEM_BYTES = TC_STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major, 128B-swizzled UMMA shared-memory descriptor (sm100 version bits)
__device__ __forceinline__ uint64_t sdesc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);       // start address
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                        // version = 1 (Blackwell)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, K-major both, M=128, N=TC_BN
constexpr uint32_t idesc_tf32() {
  return (1u << 4)            // c_format F32
         | (2u << 7)          // a_format TF32
         | (2u << 10)         // b_format TF32
         | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc_tf32()), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// x -> (hi, lo): hi = tf32 round-to-nearest of x, lo = x - hi (exact in fp32);
// the MMA reads lo as tf32 too, leaving ~2^-21 relative error per product.
__device__ __forceinline__ void split3(float& x, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  lo = __fsub_rn(x, __uint_as_float(h));
  x = __uint_as_float(h);
}

__device__ __forceinline__ float act_fwd(int act, float z) {
  return act == 0 ? (z > 0.f ? z : 0.f) : tanhf(z);
}
__device__ __forceinline__ float act_bwd(int act, float y) {
  return act == 0 ? (y > 0.f ? 1.f : 0.f) : __fsub_rn(1.f, __fmul_rn(y, y));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%"
      "15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// Two-level accumulation: the tensor-core accumulator adds are not IEEE
// round-to-nearest, so its error grows ~linearly with K. Every TC_CH k-blocks
// (128 of K) the MMA switches to the other of two TMEM accumulators and the
// epilogue warps fold the finished chunk into fp32 registers with RN adds.
constexpr int TC_CH = 4;

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmBlo, int M, int N, int K, float* __restrict__ C,
              int ldc, GemmEpi ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TC_STAGES * STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* conv = bars + TC_STAGES;
  uint64_t* empty = bars + 2 * TC_STAGES;
  uint64_t* tfull = bars + 3 * TC_STAGES;       // [2] chunk accumulated (MMA commit)
  uint64_t* tempty = bars + 3 * TC_STAGES + 2;  // [2] chunk drained (128 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * TC_STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * TC_BM, n0 = blockIdx.x * TC_BN;
  const int nk = (K + TC_BK - 1) / TC_BK;
  const int nchunks = (nk + TC_CH - 1) / TC_CH;
  auto sA = [&](int s) { return smem + s * STAGE_BYTES; };
  auto sAlo = [&](int s) { return smem + s * STAGE_BYTES + A_BYTES; };
  auto sB = [&](int s) { return smem + s * STAGE_BYTES + 2 * A_BYTES; };
  auto sBlo = [&](int s) { return smem + s * STAGE_BYTES + 2 * A_BYTES + B_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * TC_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBlo)) : "memory");
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % TC_STAGES;
        const uint32_t ph = (kb / TC_STAGES) & 1;
        if (kb >= TC_STAGES) mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], A_BYTES + 2 * B_BYTES);
        tma_load_2d(sA(s), &tmA, &full[s], kb * TC_BK, m0);
        tma_load_2d(sB(s), &tmB, &full[s], kb * TC_BK, n0);
        tma_load_2d(sBlo(s), &tmBlo, &full[s], kb * TC_BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % TC_STAGES;
        const uint32_t ph = (kb / TC_STAGES) & 1;
        const int c = kb / TC_CH, buf = c & 1, kin = kb % TC_CH;
        if (kin == 0 && c >= 2) mbar_wait(&tempty[buf], ((c >> 1) - 1) & 1);
        mbar_wait(&full[s], ph);
        mbar_wait(&conv[s], ph);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * TC_BN);
        const uint32_t a = smem_u32(sA(s)), alo = smem_u32(sAlo(s));
        const uint32_t b = smem_u32(sB(s)), blo = smem_u32(sBlo(s));
#pragma unroll
        for (int kk = 0; kk < TC_BK / 8; ++kk) {
          const uint32_t off = kk * 32;  // 8 tf32 = 32 B along K inside the swizzle atom
          mma_tf32(d, sdesc_k_sw128(a + off), sdesc_k_sw128(b + off), (kin | kk) != 0);
          mma_tf32(d, sdesc_k_sw128(a + off), sdesc_k_sw128(blo + off), 1);
          mma_tf32(d, sdesc_k_sw128(alo + off), sdesc_k_sw128(b + off), 1);
        }
        mma_commit(&empty[s]);
        if (kin == TC_CH - 1 || kb == nk - 1) mma_commit(&tfull[buf]);
      }
    }
  } else {
    const int ct = threadIdx.x - 64;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    float acc[TC_BN];
#pragma unroll
    for (int j = 0; j < TC_BN; ++j) acc[j] = 0.f;
    int drained = 0;
    auto drain = [&](int c) {
      const int buf = c & 1;
      mbar_wait(&tfull[buf], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < TC_BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * TC_BN + c0), r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[c0 + j] = __fadd_rn(acc[c0 + j], __uint_as_float(r[j]));
      }
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
    };
    // ---- A hi/lo converters, draining finished chunks as they go ----
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TC_STAGES;
      const uint32_t ph = (kb / TC_STAGES) & 1;
      mbar_wait(&full[s], ph);
      float4* hi = reinterpret_cast<float4*>(sA(s));
      float4* lo = reinterpret_cast<float4*>(sAlo(s));
#pragma unroll
      for (int i = 0; i < (int)(A_BYTES / 16 / 128); ++i) {
        float4 x = hi[ct + 128 * i], l;
        split3(x.x, l.x);
        split3(x.y, l.y);
        split3(x.z, l.z);
        split3(x.w, l.w);
        hi[ct + 128 * i] = x;
        lo[ct + 128 * i] = l;
      }
      fence_proxy_async();
      mbar_arrive(&conv[s]);
      while (drained < kb / TC_CH) drain(drained++);
    }
    while (drained < nchunks) drain(drained++);
    // ---- epilogue: registers -> HBM ----
    const int row = q * 32 + lane;
    const int m = m0 + row;
    if (m < M) {
      float* crow = C + (size_t)m * ldc;
#pragma unroll
      for (int j = 0; j < TC_BN; ++j) {
        const int n = n0 + j;
        if (n < N) {
          float v = acc[j];
          if (ep.mode == 1) v = act_fwd(ep.act, __fadd_rn(v, ep.bias[n]));
          else if (ep.mode == 2) v = __fmul_rn(v, act_bwd(ep.act, ep.aux[(size_t)m * ep.ld_aux + n]));
          else if (ep.mode == 3) v = __fmul_rn(v, ep.coeff[(size_t)m * ep.S + n / ep.e]);
          acc[j] = v;
        }
      }
      if (n0 + TC_BN <= N && (ldc & 3) == 0) {
#pragma unroll
        for (int j = 0; j < TC_BN; j += 4)
          *reinterpret_cast<float4*>(crow + n0 + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < TC_BN; ++j)
          if (n0 + j < N) crow[n0 + j] = acc[j];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_BN));
}

// ---- host side ---------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// row-major [rows][cols] fp32 with leading dimension ld, box = box_rows x 32 cols
bool make_map(CUtensorMap* m, const float* base, uint64_t rows, uint64_t cols, uint64_t ld,
              uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__global__ void k_split(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                        size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v = x[i], l;
    split3(v, l);
    hi[i] = v;
    lo[i] = l;
  }
}

}  // namespace

bool tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("KP_GEMM");
    return !(e && std::string(e) == "simt");
  }();
  return on;
}

bool tc_gemm_supported(int M, int N, int K, const float* A, int lda, const float* B, int ldb) {
  if (M <= 0 || N <= 0 || K <= 0) return false;
  if (lda % 4 || ldb % 4) return false;
  if (reinterpret_cast<uintptr_t>(A) % 16 || reinterpret_cast<uintptr_t>(B) % 16) return false;
  return encode_fn() != nullptr;
}

void split_hilo(const float* x, float* hi, float* lo, size_t n, cudaStream_t s) {
  unsigned g = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
  k_split<<<g ? g : 1, 256, 0, s>>>(x, hi, lo, n); ::kp::count_launch();
}

// C = epi(A[M][K] . B[N][K]^T); (B_hi, B_lo) = split_hilo(B) precomputed by the caller.
void tc_gemm_nt(int M, int N, int K, const float* A, int lda, const float* B, const float* Blo,
                int ldb, float* C, int ldc, const GemmEpi& ep, cudaStream_t s) {
  CUtensorMap ta, tb, tbl;
  KP_CHECK(make_map(&ta, A, M, K, lda, TC_BM) && make_map(&tb, B, N, K, ldb, TC_BN) &&
               make_map(&tbl, Blo, N, K, ldb, TC_BN),
           kErrCuda, "cuTensorMapEncodeTiled failed");
  static bool attr = false;
  if (!attr) {
    KP_CUDA(cudaFuncSetAttribute(k_tc_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr = true;
  }
  dim3 grid(ceil_div(N, TC_BN), ceil_div(M, TC_BM));
  k_tc_gemm<<<grid, TC_THREADS, SMEM_BYTES, s>>>(ta, tb, tbl, M, N, K, C, ldc, ep); ::kp::count_launch();
}

}  // namespace kp
