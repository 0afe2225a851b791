// fp32-accurate GEMM on the 5th-generation tensor cores (tcgen05, 3xTF32).
//
//   C[z][m][n] = epi( sum_{k in split z} A(m,k) * B(n,k) )
//
// Operands stay fp32 in HBM and are read by TMA in either major order:
//   K-major  (X[row][k], k contiguous):   the forward Z = X W^T and the
//            input gradient dX = dZ W (with W^T kept K-major);
//   MN-major (X[k][row], row contiguous): the weight gradient dW = dZ^T X, whose
//            contraction runs over the batch.
// Each operand tile x is split in shared memory into hi = tf32_rn(x) and
// lo = x - hi; three tcgen05.mma per k-step accumulate hi*hi + hi*lo + lo*hi
// (the dropped lo*lo term is ~2^-21 relative). The tensor-core accumulator's
// adds are not IEEE round-to-nearest (its error grows with K), so every
// TC_CH k-blocks the MMA switches between two TMEM accumulators and the
// epilogue warps fold the finished one into fp32 registers with RN adds:
// fp32-level accuracy, independent of K, at tensor-core rate.
//
// Layout: a persistent, warp-specialised kernel of 18 warps per CTA (TMA
// producer, TMEM allocator + MMA issuer, 8 splitter warps, 8 drain/epilogue
// warps; CTA pairs with cta_group::2) -- see the block above k_tc_gemm.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <string>

#include "kp_internal.cuh"

namespace kp {
namespace {

constexpr int TC_BM = 128, TC_BN = 128, TC_BK = 32, TC_CH = 4;
constexpr uint32_t A_BYTES = TC_BM * TC_BK * 4;  // 16 KB
constexpr int EPI_LD = 20;  // epilogue transpose row stride (floats): conflict-free float4 rows
constexpr uint32_t EPI_BYTES = 8 * 32 * EPI_LD * 4;  // 8 epilogue warps x 32 rows x 16 columns

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

// UMMA shared-memory descriptors (sm100 version bits).
//  K-major : SWIZZLE_128B; 8-row groups of 128 B rows at SBO = 1024 B.
//  MN-major: tf32 MN-major operands only come in SWIZZLE_128B_BASE32B (32 B
//            swizzle atoms, TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 32-element
//            (128 B) MN atoms at LBO = 4096 B (one 32x32 TMA box), 4-row K
//            groups at SBO = 512 B.
template <bool MN>
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(MN ? (4096 >> 4) : 1) << 16;
  d |= (uint64_t)(MN ? (512 >> 4) : (1024 >> 4)) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(MN ? 1 : 2) << 61;
  return d;
}
// byte offset of UMMA k-step kk (8 tf32) inside a stage tile
template <bool MN>
__device__ __forceinline__ uint32_t kstep_off(int kk) {
  return MN ? (uint32_t)kk * 1024u : (uint32_t)kk * 32u;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Split mode. Truncating (default): the tensor core reads a raw fp32 operand
// as tf32 by dropping the 13 low mantissa bits, so hi needs no conversion and
// no copy -- the TMA-loaded fp32 tile IS the hi operand -- and only
// lo = x - trunc(x) (exact) is produced: half the TMEM/smem split traffic.
// KP_TC_RN selects the round-to-nearest split (hi = tf32_rn(x)).
#ifdef KP_TC_RN
constexpr bool kTrunc = false;
#else
constexpr bool kTrunc = true;
#endif
// KP_ALO_SMEM: A lo operand in shared memory (all three MMAs SS, TMEM holds
// only the accumulators). Measured slower (shared memory bandwidth is the
// scarcer resource: +7% GEMM time); the default keeps A lo in TMEM.
#ifdef KP_ALO_SMEM
constexpr bool kAloSmem = kTrunc;
#else
constexpr bool kAloSmem = false;
#endif
__device__ __forceinline__ float lo_trunc(float x) {
  return __fsub_rn(x, __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
}

// x -> (hi, lo): hi = tf32 round-to-nearest of x, lo = x - hi (exact in fp32)
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// Persistent, warp-specialised kernel. A work unit is one CTA (CG = 1) or one
// CTA pair (CG = 2, a 2-CTA cluster on one TPC issuing tcgen05.mma.cta_group::2
// with M = 256: each CTA holds 128 rows of A and HALF of the B tile, so every
// SM streams half the B bytes per MMA cycle -- the L2->SM operand stream is
// what bounds 3xTF32). Units walk work items (m-block, n-block, k-split)
// w = unit, +units, ...; the smem pipeline, the TMEM chunk buffers and their
// barriers run continuously across work items, so the epilogue of one tile
// overlaps the mainloop of the next.
//   warp 0      TMA producer (this CTA's A rows and B half -> local full[s])
//   warp 1      TMEM allocator; lane 0 of the leader CTA issues the MMAs
//   warps 2-9   splitters: A (fp32 in smem) -> hi/lo in TMEM (the MMA's A
//               operand comes from TMEM, so shared memory only feeds B); B is
//               split in smem too unless it arrives pre-split (BPRE); then one
//               arrival per CTA on the leader's conv[s]
//   warps 10-17 drain + epilogue: warp w owns TMEM lane quarter w%4 and column
//               half (w-10)/4 -> 64 fp32 register accumulators per thread;
//               one arrival per CTA on the leader's tempty[b]
// TMEM (per CTA): [0,256) two 128-column accumulator chunks; [256,512) per
// stage A hi (32 columns) + A lo (32 columns).
constexpr int TC_NBUF = 2;
constexpr int TC_ASLOTS = 4;  // TMEM A (hi+lo) k-block slots: 4 x 64 columns
constexpr int TC_WARPS = 18;
constexpr int TC_EPI_T = 256;  // drain/epilogue threads
constexpr uint32_t TC_ACOL = TC_NBUF * TC_BN;  // first A-operand column

// H: fp16 operands (kind::f16, 2x the tf32 rate) -- A split on chip into
// fp16 hi/lo with a per-row power-of-two scale, B pre-split fp16 hi/lo (64-byte
// K-major rows, SWIZZLE_64B) with per-row scales; see k_tc_gemm.
template <int CG, bool H = false, bool AR = false>
struct TcCfg {
  static constexpr int BROWS = TC_BN / CG;  // B rows held by one CTA
  static constexpr uint32_t B_BYTES = BROWS * TC_BK * (H ? 2 : 4);
  // A fp32, B (hi), B lo, and (kAloSmem) the A lo tile. AR: a stage holds
  // EITHER an A tile (unit start) or a B hi/lo pair, so stages are small and
  // the ring deep -- B streams from L2 with nothing else to hide its latency
  static constexpr uint32_t STAGE =
      AR ? (A_BYTES > 2 * B_BYTES ? A_BYTES : 2 * B_BYTES)
         : A_BYTES + 2 * B_BYTES + (kAloSmem ? A_BYTES : 0);
  // smem ring depth (a deeper ring, 6 stages at CG = 2 with separate TMEM A
  // slot barriers, measured no faster in the streaming-A modes)
  static constexpr int STAGES = AR ? 8 : H ? 6 : (kAloSmem && CG == 1) ? 3 : 4;
  // fp16 A slot in TMEM = 32 columns (hi 16 + lo 16): the 256 free columns hold
  // 8 slots, >= STAGES, so a slot is free whenever its smem stage is refilled
  static constexpr uint32_t ASLOT_COLS = H ? 32 : 64;
  // CG == 2: per epilogue warp two dense 32x16 fp32 tiles (TMA-store sources)
  static constexpr uint32_t EPI_DENSE = CG == 2 ? 8 * 2 * 32 * 16 * 4 : 0;
  static constexpr uint32_t EPI_CS = H ? 8 * 64 * 4 : 0;  // (H) per-warp column scales
  static constexpr uint32_t SMEM =
      STAGES * STAGE + EPI_BYTES + EPI_DENSE + EPI_CS + 1024 /*align*/ + 512 /*barriers*/;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// one arrival on barrier `b` of the leader CTA (rank 0) of the pair
template <int CG>
__device__ __forceinline__ void arrive_leader(uint64_t* b) {
  if (CG == 1) {
    mbar_arrive(b);
  } else {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(b)));
    // default (.release.cta) semantics: a .cluster-scoped release costs a
    // MEMBAR.ALL.GPU per arrival; the TMEM/smem operands are ordered by the
    // tcgen05 / proxy fences before the named barrier
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t parity) {
  mbar_wait(b, parity);
}
// instruction descriptor: D f32, A/B tf32, M = 128*CG, N = TC_BN, per-operand major
template <bool AMN, bool BMN, int CG>
__host__ __device__ constexpr uint32_t idesc_tf32_cg() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
         ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)((TC_BM * CG) >> 4) << 24);
}
// A (hi or lo) from TMEM (lane = row, 32-bit column = k), B from smem
template <bool BMN, int CG>
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t accum) {
  if (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc_tf32_cg<false, BMN, 1>()), "r"(accum));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc_tf32_cg<false, BMN, 2>()), "r"(accum));
  }
}
// A and B from shared memory
template <bool AMN, bool BMN, int CG>
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
  if (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc_tf32_cg<AMN, BMN, 1>()), "r"(accum));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc_tf32_cg<AMN, BMN, 2>()), "r"(accum));
  }
}
// fp16 K-major operand with 64-byte rows (32 halves), SWIZZLE_64B: 8-row
// groups at SBO = 512 B
__device__ __forceinline__ uint64_t sdesc_h64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
template <int CG>
__host__ __device__ constexpr uint32_t idesc_f16_cg() {
  // D f32, A/B f16 (format 0), both K-major
  return (1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)((TC_BM * CG) >> 4) << 24);
}
template <int CG>
__device__ __forceinline__ void mma_h_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t accum) {
  if (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc_f16_cg<1>()), "r"(accum));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc_f16_cg<2>()), "r"(accum));
  }
}
// power-of-two scale e of a row with max |x| = mx: mx * 2^e in [2^14, 2^15)
__host__ __device__ __forceinline__ int row_exp(float mx) {
  if (!(mx > 0.f) || !(mx < 3.0e38f)) return 0;
  int ex;
  frexpf(mx, &ex);
  const int e = 15 - ex;
  return e > 126 ? 126 : (e < -126 ? -126 : e);
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((e + 127) << 23); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
      "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}

// MMA completion -> barrier b in this CTA (CG = 1) or in both CTAs of the pair
template <int CG>
__device__ __forceinline__ void commit_cg(uint64_t* b) {
  if (CG == 1) {
    mma_commit(b);
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(b)),
        "h"((uint16_t)3)
        : "memory");
  }
}

// TMA `rows` x 32-k operand rows into smem (one K-major box, or rows/32
// 32x32 MN-major boxes at LBO spacing)
template <bool MN, int ROWS>
__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int k0,
                                          int r0) {
  if (MN) {
#pragma unroll
    for (int i = 0; i < ROWS / 32; ++i) tma_load_2d(dst + i * 4096, map, bar, r0 + 32 * i, k0);
  } else {
    tma_load_2d(dst, map, bar, k0, r0);
  }
}

// 256 splitter threads split this CTA's B tile in place (hi) + into lo
template <int CG>
__device__ __forceinline__ void split_tile(uint8_t* tile, uint8_t* lo_tile, int ct) {
  float4* hi = reinterpret_cast<float4*>(tile);
  float4* lo = reinterpret_cast<float4*>(lo_tile);
  constexpr int PER = (int)(TcCfg<CG>::B_BYTES / 16 / 256);
  float4 x[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) x[i] = hi[ct + 256 * i];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    float4 l;
    if (kTrunc) {  // hi stays the raw tile
      l = make_float4(lo_trunc(x[i].x), lo_trunc(x[i].y), lo_trunc(x[i].z), lo_trunc(x[i].w));
    } else {
      split3(x[i].x, l.x);
      split3(x[i].y, l.y);
      split3(x[i].z, l.z);
      split3(x[i].w, l.w);
      hi[ct + 256 * i] = x[i];
    }
    lo[ct + 256 * i] = l;
  }
}

// row r, k columns [k0, k0+16) of the stage's A tile -> 16 floats
template <bool MN>
__device__ __forceinline__ void load_a_row16(const uint8_t* tile, int r, int k0, float (&v)[16]) {
  if (!MN) {
    // K-major SW128: row r is 128 B; 16-byte chunk c sits at chunk c ^ (r & 7)
    const uint8_t* row = tile + r * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = (k0 >> 2) + i;
      const float4 x = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 4));
      v[4 * i] = x.x, v[4 * i + 1] = x.y, v[4 * i + 2] = x.z, v[4 * i + 3] = x.w;
    }
  } else {
    // MN-major SWIZZLE_128B_ATOM_32B: 32x32 boxes (4 KB) along m; in a box,
    // element (m, k) at k*128 + ((m%32)*4 ^ ((k & 3) << 5))
    const uint8_t* box = tile + (r >> 5) * 4096;
    const int mm = (r & 31) * 4;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k = k0 + j;
      v[j] = *reinterpret_cast<const float*>(box + k * 128 + (mm ^ ((k & 3) << 5)));
    }
  }
}

// inverse of load_a_row16: 16 values (bit patterns) -> row r, k [k0, k0+16)
template <bool MN>
__device__ __forceinline__ void store_a_row16(uint8_t* tile, int r, int k0, const uint32_t (&v)[16]) {
  if (!MN) {
    uint8_t* row = tile + r * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = (k0 >> 2) + i;
      *reinterpret_cast<uint4*>(row + ((c ^ (r & 7)) << 4)) =
          make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  } else {
    uint8_t* box = tile + (r >> 5) * 4096;
    const int mm = (r & 31) * 4;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k = k0 + j;
      *reinterpret_cast<uint32_t*>(box + k * 128 + (mm ^ ((k & 3) << 5))) = v[j];
    }
  }
}

// AR (A resident, fp16 only, K <= 256): a work unit is (m-block, run of
// n-blocks); A is split into TMEM once per unit (hi at columns [256,384), lo at
// [384,512)) and only B streams per n-block -- for dX = dZ.W1 (K = 256,
// N = 6400) this removes re-reading the A tile 50 times through TMA/smem.
template <bool AMN, bool BMN, bool BPRE, int CG, bool H = false, bool AR = false>
__global__ void __launch_bounds__(TC_WARPS * 32, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ CUtensorMap tmC,
              int c_tma, int M, int N, int K, int kps, float* __restrict__ C, int ldc, GemmEpi ep) {
  static_assert(!H || (!AMN && !BMN && BPRE), "fp16 mode: K-major A, pre-split K-major B");
  static_assert(!AR || H, "A-resident mode is fp16 only");
  constexpr uint32_t AR_COL = TC_NBUF * TC_BN;  // resident A hi; lo at +128
  // k-blocks per accumulator chunk: fp16 products are exact in fp32 and the
  // chunk error stays below the fp32 SIMT GEMM's at 8 (256 k); tf32 keeps 4
  constexpr int CH = H ? 2 * TC_CH : TC_CH;
  using Cfg = TcCfg<CG, H, AR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NS = Cfg::STAGES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * Cfg::STAGE);
  uint64_t* full = bars;                     // TMA -> splitters (local)
  uint64_t* conv = bars + NS;                // splitters -> MMA (leader; CG arrivals)
  uint64_t* empty = bars + 2 * NS;           // MMA -> producer (both CTAs)
  uint64_t* afree = bars + 3 * NS;           // MMA -> splitters: TMEM A slot free (both CTAs)
  uint64_t* tfull = afree + TC_ASLOTS;       // MMA -> drain (both CTAs)
  uint64_t* tempty = tfull + TC_NBUF;        // drain -> MMA (leader; CG arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + TC_NBUF);
  float* epi_smem = reinterpret_cast<float*>(smem + NS * Cfg::STAGE + 512);
  float* epi_dense = reinterpret_cast<float*>(smem + NS * Cfg::STAGE + 512 + EPI_BYTES);
  float* epi_cs = reinterpret_cast<float*>(smem + NS * Cfg::STAGE + 512 + EPI_BYTES + Cfg::EPI_DENSE);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const int unit = blockIdx.x / CG, units = gridDim.x / CG;
  const int TM = TC_BM * CG;
  const int mblocks = (M + TM - 1) / TM, nblocks = (N + TC_BN - 1) / TC_BN;
  const int splits = (K + kps - 1) / kps;
  // AR: n-blocks of an m-block split into nparts runs (kps carries nparts)
  const int nparts = AR ? kps : 1;
  const int nper = (nblocks + nparts - 1) / nparts;
  const int works = AR ? mblocks * nparts : mblocks * nblocks * splits;
  const int nkA = (K + TC_BK - 1) / TC_BK;  // AR: k-blocks of the resident A
  auto ar_work = [&](int w, int& m0, int& nb_lo, int& nb_hi) {
    const int mb = w / nparts, pt = w % nparts;
    m0 = mb * TM + (int)rank * TC_BM;
    nb_lo = pt * nper;
    nb_hi = min(nblocks, nb_lo + nper);
  };
  // work w -> (n-block fastest, then m-block, then split): units in flight share A rows
  auto decode = [&](int w, int& m0, int& n0, int& z, int& nk) {
    const int nb = w % nblocks, r = w / nblocks, mb = r % mblocks;
    z = r / mblocks;
    m0 = mb * TM + (int)rank * TC_BM;  // this CTA's rows
    n0 = nb * TC_BN;
    const int kbeg = z * kps, kend = min(K, kbeg + kps);
    nk = kend > kbeg ? (kend - kbeg + TC_BK - 1) / TC_BK : 0;
  };
  auto sA = [&](int s) { return smem + s * Cfg::STAGE; };
  auto sB = [&](int s) { return smem + s * Cfg::STAGE + (AR ? 0 : A_BYTES); };
  auto sBlo = [&](int s) { return smem + s * Cfg::STAGE + (AR ? 0 : A_BYTES) + Cfg::B_BYTES; };
  auto sAlo = [&](int s) { return smem + s * Cfg::STAGE + A_BYTES + 2 * Cfg::B_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], CG);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < TC_ASLOTS; ++a) mbar_init(&afree[a], 1);
    for (int b = 0; b < TC_NBUF; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote arrival
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      if (BPRE) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmBlo)) : "memory");
      int g = 0;  // global k-block counter (stage pipeline)
      if constexpr (AR) {
        for (int w = unit; w < works; w += units) {
          int m0, nlo, nhi;
          ar_work(w, m0, nlo, nhi);
          for (int kb = 0; kb < nkA; ++kb, ++g) {  // the unit's A, once
            const int s = g % NS;
            if (g >= NS) mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);
            mbar_expect_tx(&full[s], A_BYTES);
            load_rows<false, TC_BM>(sA(s), &tmA, &full[s], kb * TC_BK, m0);
          }
          for (int nb = nlo; nb < nhi; ++nb) {  // then only B per n-block
            const int nb0 = nb * TC_BN + (int)rank * Cfg::BROWS;
            for (int kb = 0; kb < nkA; ++kb, ++g) {
              const int s = g % NS;
              if (g >= NS) mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);
              mbar_expect_tx(&full[s], 2 * Cfg::B_BYTES);
              load_rows<false, Cfg::BROWS>(sB(s), &tmB, &full[s], kb * TC_BK, nb0);
              load_rows<false, Cfg::BROWS>(sBlo(s), &tmBlo, &full[s], kb * TC_BK, nb0);
            }
          }
        }
      } else
      for (int w = unit; w < works; w += units) {
        int m0, n0, z, nk;
        decode(w, m0, n0, z, nk);
        const int nb0 = n0 + (int)rank * Cfg::BROWS;  // this CTA's half of the B tile
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % NS;
          const uint32_t ph = (g / NS) & 1;
          if (g >= NS) mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], A_BYTES + (BPRE ? 2 : 1) * Cfg::B_BYTES);
          const int k0 = z * kps + kb * TC_BK;
          load_rows<AMN, TC_BM>(sA(s), &tmA, &full[s], k0, m0);
          load_rows<BMN, Cfg::BROWS>(sB(s), &tmB, &full[s], k0, nb0);  // (H: one 64 B-row box)
          if (BPRE) load_rows<BMN, Cfg::BROWS>(sBlo(s), &tmBlo, &full[s], k0, nb0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      int g = 0, c = 0;  // global k-block and chunk counters
      if constexpr (AR) {
        for (int w = unit; w < works; w += units) {
          int m0, nlo, nhi;
          ar_work(w, m0, nlo, nhi);
          for (int kb = 0; kb < nkA; ++kb, ++g) {  // A split into TMEM: free the smem stage
            const int s = g % NS;
            mbar_wait_cl<CG>(&conv[s], (g / NS) & 1);
            tc_fence_after();
            commit_cg<CG>(&empty[s]);
          }
          for (int nb = nlo; nb < nhi; ++nb, ++c) {
            const int buf = c % TC_NBUF;
            if (c >= TC_NBUF) mbar_wait_cl<CG>(&tempty[buf], ((c / TC_NBUF) - 1) & 1);
            const uint32_t d = tmem + (uint32_t)(buf * TC_BN);
            for (int kb = 0; kb < nkA; ++kb, ++g) {
              const int s = g % NS;
              mbar_wait_cl<CG>(&conv[s], (g / NS) & 1);
              tc_fence_after();
              const uint32_t b = smem_u32(sB(s)), blo = smem_u32(sBlo(s));
#pragma unroll
              for (int kk = 0; kk < TC_BK / 16; ++kk) {
                const uint64_t bh = sdesc_h64(b + 32u * kk), bl = sdesc_h64(blo + 32u * kk);
                const uint32_t ah = tmem + AR_COL + 16u * kb + 8u * kk;
                mma_h_ts<CG>(d, ah, bh, (kb | kk) != 0);
                mma_h_ts<CG>(d, ah, bl, 1);
                mma_h_ts<CG>(d, ah + 128u, bh, 1);
              }
              commit_cg<CG>(&empty[s]);
            }
            commit_cg<CG>(&tfull[buf]);
          }
          commit_cg<CG>(&afree[0]);  // the resident A may be overwritten
        }
      } else
      for (int w = unit; w < works; w += units) {
        int m0, n0, z, nk;
        decode(w, m0, n0, z, nk);
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % NS;
          const uint32_t ph = (g / NS) & 1;
          const int kin = kb % CH, buf = c % TC_NBUF;
          if (kin == 0 && c >= TC_NBUF) mbar_wait_cl<CG>(&tempty[buf], ((c / TC_NBUF) - 1) & 1);
          mbar_wait_cl<CG>(&conv[s], ph);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * TC_BN);
          const uint32_t ahi = tmem + TC_ACOL +
                               Cfg::ASLOT_COLS * (uint32_t)(H ? g % NS : g % TC_ASLOTS),
                         alo = ahi + 32u;
          const uint32_t b = smem_u32(sB(s)), blo = smem_u32(sBlo(s));
          const uint32_t asm_ = smem_u32(sA(s));
          if constexpr (H) {
            // A hi at slot columns [0,16), A lo at [16,32): 2 halves per column
#pragma unroll
            for (int kk = 0; kk < TC_BK / 16; ++kk) {
              const uint64_t bh = sdesc_h64(b + 32u * kk), bl = sdesc_h64(blo + 32u * kk);
              mma_h_ts<CG>(d, ahi + 8u * kk, bh, (kin | kk) != 0);
              mma_h_ts<CG>(d, ahi + 8u * kk, bl, 1);
              mma_h_ts<CG>(d, ahi + 16u + 8u * kk, bh, 1);
            }
          } else {
#pragma unroll
          for (int kk = 0; kk < TC_BK / 8; ++kk) {
            const uint32_t ob = kstep_off<BMN>(kk);
            if (kTrunc) {
              const uint64_t ad = sdesc<AMN>(asm_ + kstep_off<AMN>(kk));
              mma_ss<AMN, BMN, CG>(d, ad, sdesc<BMN>(b + ob), (kin | kk) != 0);
              mma_ss<AMN, BMN, CG>(d, ad, sdesc<BMN>(blo + ob), 1);
            } else {
              mma_ts<BMN, CG>(d, ahi + 8u * kk, sdesc<BMN>(b + ob), (kin | kk) != 0);
              mma_ts<BMN, CG>(d, ahi + 8u * kk, sdesc<BMN>(blo + ob), 1);
            }
            if (kAloSmem)
              mma_ss<AMN, BMN, CG>(d, sdesc<AMN>(smem_u32(sAlo(s)) + kstep_off<AMN>(kk)), sdesc<BMN>(b + ob), 1);
            else
              mma_ts<BMN, CG>(d, alo + 8u * kk, sdesc<BMN>(b + ob), 1);
          }
          }
          commit_cg<CG>(&empty[s]);
          if (!H && NS > TC_ASLOTS) commit_cg<CG>(&afree[g % TC_ASLOTS]);
          if (kin == CH - 1 || kb == nk - 1) {
            commit_cg<CG>(&tfull[buf]);
            ++c;
          }
        }
      }
    }
  } else if (warp < 10) {
    // ---- splitters: A -> TMEM hi/lo (+ B in smem unless pre-split) ----
    const int ct = threadIdx.x - 64;
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int r = q * 32 + lane;  // tile row == TMEM lane
    float h_scale = 1.f;          // (H) this row's 2^e
    int g = 0;
    if constexpr (AR) {
      int wi = 0;
      for (int w = unit; w < works; w += units, ++wi) {
        int m0, nlo, nhi;
        ar_work(w, m0, nlo, nhi);
        // the previous unit's MMAs have finished reading the resident A
        if (wi > 0) mbar_wait(&afree[0], (wi - 1) & 1);
        {
          const int m = m0 + r;
          h_scale = pow2f(m < M ? row_exp(ep.a_rowmax[m]) : 0);
        }
        for (int kb = 0; kb < nkA; ++kb, ++g) {
          const int s = g % NS;
          mbar_wait(&full[s], (g / NS) & 1);
          float v[16];
          load_a_row16<false>(sA(s), r, h * 16, v);
          uint32_t hp[8], lp[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x0 = __fmul_rn(v[2 * j], h_scale), x1 = __fmul_rn(v[2 * j + 1], h_scale);
            const __half2 hh = __floats2half2_rn(x0, x1);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(__fsub_rn(x0, hf.x), __fsub_rn(x1, hf.y));
            hp[j] = *reinterpret_cast<const uint32_t*>(&hh);
            lp[j] = *reinterpret_cast<const uint32_t*>(&ll);
          }
          tc_fence_after();
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + AR_COL + 16u * kb + 8u * h;
          tmem_st8(ta, hp);
          tmem_st8(ta + 128u, lp);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          named_sync(1, 256);
          if (ct == 0) arrive_leader<CG>(&conv[s]);
        }
        // B stages: forward TMA completion to the (leader's) MMA issuer
        for (int nb = nlo; nb < nhi; ++nb)
          for (int kb = 0; kb < nkA; ++kb, ++g) {
            if (ct == 0) {
              const int s = g % NS;
              mbar_wait(&full[s], (g / NS) & 1);
              arrive_leader<CG>(&conv[s]);
            }
          }
      }
    } else
    for (int w = unit; w < works; w += units) {
      int m0, n0, z, nk;
      decode(w, m0, n0, z, nk);
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % NS;
        const uint32_t ph = (g / NS) & 1;
        mbar_wait(&full[s], ph);
        float v[16];
        load_a_row16<AMN>(sA(s), r, h * 16, v);
        if constexpr (H) {
          // row scale: the row's max |x| (a_rowmax) -> 2^e
          if (kb == 0) {
            const int m = m0 + r;
            h_scale = pow2f(m < M ? row_exp(ep.a_rowmax[m]) : 0);
          }
          uint32_t hp[8], lp[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            // packed conversions: cvt.rn.f16x2.f32 (low half = even k)
            const float x0 = __fmul_rn(v[2 * j], h_scale), x1 = __fmul_rn(v[2 * j + 1], h_scale);
            const __half2 hh = __floats2half2_rn(x0, x1);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(__fsub_rn(x0, hf.x), __fsub_rn(x1, hf.y));
            hp[j] = *reinterpret_cast<const uint32_t*>(&hh);
            lp[j] = *reinterpret_cast<const uint32_t*>(&ll);
          }
          const int as = g % NS;  // (fp16: 8 slots >= NS, see TcCfg)
          tc_fence_after();
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + TC_ACOL + Cfg::ASLOT_COLS * (uint32_t)as + 8u * h;
          tmem_st8(ta, hp);
          tmem_st8(ta + 16u, lp);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          named_sync(1, 256);
          if (ct == 0) arrive_leader<CG>(&conv[s]);
          continue;
        }
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float x = v[j], l;
          if (kTrunc) {
            l = lo_trunc(x);
          } else {
            split3(x, l);
          }
          hi[j] = __float_as_uint(x);
          lo[j] = __float_as_uint(l);
        }
        // the MMAs of k-block g - TC_ASLOTS have finished reading this TMEM A slot
        const int as = g % TC_ASLOTS;
        // (NS == TC_ASLOTS: implied by empty[s] -> TMA -> full[s])
        if (NS > TC_ASLOTS && g >= TC_ASLOTS) mbar_wait(&afree[as], ((g / TC_ASLOTS) - 1) & 1);
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + TC_ACOL + 64u * (uint32_t)as + 16u * h;
        if (kAloSmem) {
          store_a_row16<AMN>(sAlo(s), r, h * 16, lo);
        } else {
          if (!kTrunc) tmem_st16(ta, hi);  // truncating: the MMA reads hi from the smem tile
          tmem_st16(ta + 32u, lo);
        }
        if (!BPRE) split_tile<CG>(sB(s), sBlo(s), ct);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async();
        tc_fence_before();
        named_sync(1, 256);
        if (ct == 0) arrive_leader<CG>(&conv[s]);
      }
    }
  } else {
    // ---- drain + epilogue (256 threads) ----
    const int q = warp & 3;               // TMEM lane quarter
    const int half = (warp - 10) >> 2;    // column half of the 128-wide tile
    const int et = threadIdx.x - 320;
    uint32_t tma_seq = 0;  // TMA stores issued by this warp (dense buffer parity)
    int c = 0;
    for (int w = unit; w < works; w += units) {
      int m0, n0 = 0, z = 0, nk, nlo = 0, nhi = 1;
      if constexpr (AR) {
        ar_work(w, m0, nlo, nhi);
        nk = nkA;
      } else {
        decode(w, m0, n0, z, nk);
      }
      for (int nbi = nlo; nbi < nhi; ++nbi) {  // AR: the unit's n-blocks; else one tile
      if constexpr (AR) n0 = nbi * TC_BN;
      if (ep.mode == 2) {
        // activation-derivative operand: pull this lane's 64-column row
        // segment into L2 while the tile's MMAs run, so the epilogue's
        // loads do not pay an HBM round trip per 16-column group
        const int m = min(m0 + q * 32 + lane, M - 1);
        const int nb = min(n0 + half * 64, N - 1);
        const char* a0 = reinterpret_cast<const char*>(ep.aux + (size_t)m * ep.ld_aux + nb);
        const char* a1 = reinterpret_cast<const char*>(ep.aux + (size_t)m * ep.ld_aux + min(nb + 63, N - 1));
        for (const char* pp = a0; pp <= a1; pp += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pp));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a1));
      }
      float acc[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) acc[j] = 0.f;
      const int nch = (nk + CH - 1) / CH;
      for (int ci = 0; ci < nch; ++ci, ++c) {
        const int buf = c % TC_NBUF;
        mbar_wait(&tfull[buf], (c / TC_NBUF) & 1);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * TC_BN + half * 64 + c0), r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[c0 + j] = __fadd_rn(acc[c0 + j], __uint_as_float(r[j]));
        }
        tc_fence_before();
        named_sync(2, TC_EPI_T);
        if (et == 0) arrive_leader<CG>(&tempty[buf]);
      }
      // Epilogue through a per-warp smem transpose: the drain holds one ROW
      // per lane (tcgen05.ld 32x32b); stores want consecutive COLUMNS per
      // lane. Per 16-column group: lane -> smem row, then 4 lanes per row
      // (float4 each, 64 B contiguous) x 8 rows per instruction -> HBM, with
      // the epilogue's bias / activation-derivative / coefficient loads
      // coalesced the same way.
      float* st = epi_smem + (warp - 10) * (32 * EPI_LD);
      const int rsub = lane >> 2, c4 = (lane & 3) * 4;
      const bool cvec = (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
      float rs[4] = {1.f, 1.f, 1.f, 1.f};  // (H) 2^-ea of this thread's 4 output rows
      float* csw = epi_cs + (warp - 10) * 64;  // (H) 2^-eb of this warp's 64 columns
      if constexpr (H) {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int m = m0 + q * 32 + it * 8 + rsub;
          rs[it] = m < M ? pow2f(-row_exp(__ldg(ep.a_rowmax + m))) : 1.f;
        }
        __syncwarp();
        for (int j = lane; j < 64; j += 32) {
          const int nn = n0 + half * 64 + j;
          csw[j] = nn < N ? pow2f(-__ldg(ep.b_exp + nn)) : 1.f;
        }
        __syncwarp();
      }
      if (Cfg::EPI_DENSE && c_tma) {
        // TMA-store epilogue, row per lane: each lane writes its row's 16
        // columns into a SWIZZLE_64B 32x16 smem tile (conflict-free float4
        // stores) and one bulk tensor store moves it; no transpose. Rows and
        // columns outside C are clipped by the store.
        const int m = m0 + q * 32 + lane;
        const int mc = min(m, M - 1);
        float ra = 1.f;
        if constexpr (H) ra = m < M ? pow2f(-row_exp(__ldg(ep.a_rowmax + m))) : 1.f;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          uint8_t* dense = reinterpret_cast<uint8_t*>(epi_dense + ((warp - 10) * 2 + (tma_seq & 1)) * 512);
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          const int nb = n0 + half * 64 + c0;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = acc[c0 + j];
          if constexpr (H) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __fmul_rn(__fmul_rn(v[j], ra), csw[c0 + j]);
          }
          if (ep.mode == 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = act_fwd(ep.act, __fadd_rn(v[j], __ldg(ep.bias + min(nb + j, N - 1))));
          } else if (ep.mode == 2) {
            const float* ap = ep.aux + (size_t)mc * ep.ld_aux;
            if (nb + 16 <= N && ((reinterpret_cast<uintptr_t>(ap + nb) & 15) == 0)) {
              float a[16];
#pragma unroll
              for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(a + j) = __ldg(reinterpret_cast<const float4*>(ap + nb + j));
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = __fmul_rn(v[j], act_bwd(ep.act, a[j]));
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = __fmul_rn(v[j], act_bwd(ep.act, __ldg(ap + min(nb + j, N - 1))));
            }
          } else if (ep.mode == 3) {
            const float* cp = ep.coeff + (size_t)mc * ep.S;
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __fmul_rn(v[j], __ldg(cp + min(nb + j, N - 1) / ep.e));
          }
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            *reinterpret_cast<float4*>(dense + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4)) =
                make_float4(v[4 * cc], v[4 * cc + 1], v[4 * cc + 2], v[4 * cc + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            const int cy = z * M + m0 + q * 32;
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmC)),
                "r"(smem_u32(dense)), "r"(nb), "r"(cy)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++tma_seq;
        }
        continue;
      }
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(st + lane * EPI_LD + j) =
              make_float4(acc[c0 + j], acc[c0 + j + 1], acc[c0 + j + 2], acc[c0 + j + 3]);
        __syncwarp();
        const int n = n0 + half * 64 + c0 + c4;
        float cs[4] = {1.f, 1.f, 1.f, 1.f};  // (H) 2^-eb of the 4 columns
        if constexpr (H) {
          const float4 c4v = *reinterpret_cast<const float4*>(csw + c0 + c4);
          cs[0] = c4v.x, cs[1] = c4v.y, cs[2] = c4v.z, cs[3] = c4v.w;
        }
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int rr = it * 8 + rsub;
          const int m = m0 + q * 32 + rr;
          if (m >= M || n >= N) continue;
          float4 v = *reinterpret_cast<const float4*>(st + rr * EPI_LD + c4);
          float* vv = reinterpret_cast<float*>(&v);
          const bool full4 = n + 4 <= N;
          if constexpr (H) {  // undo the operand scales: x 2^-(ea + eb[n]), exact
#pragma unroll
            for (int t = 0; t < 4; ++t) vv[t] = __fmul_rn(__fmul_rn(vv[t], rs[it]), cs[t]);
          }
          if (ep.mode == 1) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (n + t < N) vv[t] = act_fwd(ep.act, __fadd_rn(vv[t], ep.bias[n + t]));
          } else if (ep.mode == 2) {
            const float* ap = ep.aux + (size_t)m * ep.ld_aux + n;
            if (full4 && ((ep.ld_aux & 3) == 0) && ((reinterpret_cast<uintptr_t>(ep.aux) & 15) == 0)) {
              const float4 a = __ldg(reinterpret_cast<const float4*>(ap));
              vv[0] = __fmul_rn(vv[0], act_bwd(ep.act, a.x));
              vv[1] = __fmul_rn(vv[1], act_bwd(ep.act, a.y));
              vv[2] = __fmul_rn(vv[2], act_bwd(ep.act, a.z));
              vv[3] = __fmul_rn(vv[3], act_bwd(ep.act, a.w));
            } else {
#pragma unroll
              for (int t = 0; t < 4; ++t)
                if (n + t < N) vv[t] = __fmul_rn(vv[t], act_bwd(ep.act, ap[t]));
            }
          } else if (ep.mode == 3) {
            const float* cp = ep.coeff + (size_t)m * ep.S;
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (n + t < N) vv[t] = __fmul_rn(vv[t], cp[(n + t) / ep.e]);
          }
          float* crow = C + (size_t)z * M * ldc + (size_t)m * ldc + n;
          if (full4 && cvec) {
            *reinterpret_cast<float4*>(crow) = v;
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (n + t < N) crow[t] = vv[t];
          }
        }
      }
      }
    }
    if (Cfg::EPI_DENSE && c_tma && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
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

// row-major [rows][cols] fp32 (leading dimension ld) with a box of
// box_rows x 32 columns, 128B swizzle
bool make_map(CUtensorMap* m, const float* base, uint64_t rows, uint64_t cols, uint64_t ld,
              uint32_t box_rows, bool atom32 = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp16 [rows][cols] (leading dimension ld halves), boxes of box_rows x 32
// halves (64-byte rows), 64B swizzle
bool make_map_h(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// one block per row of W [N][K]: row max -> exponent e (row_exp), then the
// fp16 split of W * 2^e: hi = rn(x), lo = rn(x - hi)
__global__ void k_split_h(const float* __restrict__ w, int K, int ld, __half* __restrict__ hi,
                          __half* __restrict__ lo, int* __restrict__ exps) {
  __shared__ float red[32];
  const float* row = w + (size_t)blockIdx.x * ld;
  float mx = 0.f;
#pragma unroll 4
  for (int k = threadIdx.x; k < K; k += blockDim.x) mx = fmaxf(mx, fabsf(row[k]));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) red[0] = mx;
  }
  __syncthreads();
  const int e = row_exp(red[0]);
  if (threadIdx.x == 0) exps[blockIdx.x] = e;
  const float sc = pow2f(e);
#pragma unroll 4
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float x = __fmul_rn(row[k], sc);
    const __half h = __float2half_rn(x);
    hi[(size_t)blockIdx.x * ld + k] = h;
    lo[(size_t)blockIdx.x * ld + k] = __float2half_rn(__fsub_rn(x, __half2float(h)));
  }
}

// one warp per row: max |A[m][k]| (the per-row scale of the fp16 A operand)
__global__ void k_rowmax(const float* __restrict__ a, int M, int K, int lda, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int m = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; m < M; m += (gridDim.x * blockDim.x) >> 5) {
    const float* row = a + (size_t)m * lda;
    float mx = 0.f;
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(row[k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) out[m] = mx;
  }
}

__global__ void k_split(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                        size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v = x[i], l;
    if (kTrunc) l = lo_trunc(v);
    else split3(v, l);
    hi[i] = v;
    lo[i] = l;
  }
}

thread_local int g_reserve_sms = 0;

bool tma_store_enabled() {  // KP_GEMM_TMA_STORE=0: per-thread global stores
  static const bool on = [] {
    const char* e = getenv("KP_GEMM_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CTA-pair (cta_group::2) mode for M > 128; KP_GEMM_CG=1 forces single-CTA tiles
int choose_cg(int M) {
  static const int force = [] {
    const char* e = getenv("KP_GEMM_CG");
    return e ? atoi(e) : 0;
  }();
  if (force == 1 || force == 2) return force;
  return M > TC_BM ? 2 : 1;
}

// concurrently resident work units (CTAs or CTA pairs)
template <bool AMN, bool BMN, bool BPRE, int CG, bool H = false, bool AR = false>
int resident_units() {
  static int units = 0;
  if (units) return units;
  int sms = 0;
  int dev = 0;
  KP_CUDA(cudaGetDevice(&dev));
  KP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  units = sms / CG;
  if (CG > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * CG, 1, 1);
    cfg.blockDim = dim3(TC_WARPS * 32, 1, 1);
    cfg.dynamicSmemBytes = TcCfg<CG, H, AR>::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_tc_gemm<AMN, BMN, BPRE, CG, H, AR>, &cfg) == cudaSuccess && n > 0)
      units = std::min(units, n);
    cudaGetLastError();
  }
  return units;
}

template <bool AMN, bool BMN, bool BPRE, int CG, bool H = false, bool AR = false>
int launch_cg(int M, int N, int K, const float* A, int lda, const void* B, const void* Blo, int ldb,
              float* C, int ldc, int splits, const GemmEpi& ep, cudaStream_t s) {
  using Cfg = TcCfg<CG, H, AR>;
  CUtensorMap ta, tb, tbl;
  // K-major: [rows][K] with box_rows-row boxes; MN-major: [K][rows] with 32x32 boxes
  auto mk = [&](CUtensorMap* m, const void* p, bool mn, int rows, int ld, int box_rows) {
    if (H && p != A) return make_map_h(m, p, rows, K, ld, box_rows);
    const float* f = static_cast<const float*>(p);
    return mn ? make_map(m, f, K, rows, ld, 32, true) : make_map(m, f, rows, K, ld, box_rows);
  };
  const bool ok = mk(&ta, A, AMN, M, lda, TC_BM) && mk(&tb, B, BMN, N, ldb, Cfg::BROWS) &&
                  (!BPRE || mk(&tbl, Blo, BMN, N, ldb, Cfg::BROWS));
  if (!BPRE) tbl = tb;
  KP_CHECK(ok, kErrCuda, "cuTensorMapEncodeTiled failed");
  // TMA-store epilogue (CTA pairs): C as a [nz*M][N] fp32 tensor, 32x16 boxes;
  // split-K partials are stacked along rows, so it needs M % 128 == 0 there
  int c_tma = 0;
  CUtensorMap tc = ta;
  {
    int kps0 = (K + splits - 1) / splits;
    kps0 = (kps0 + TC_BK - 1) / TC_BK * TC_BK;
    const unsigned nz0 = ceil_div(K, kps0);
    if (Cfg::EPI_DENSE && (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0 &&
        (nz0 == 1 || M % TC_BM == 0) && tma_store_enabled()) {
      auto fn = encode_fn();
      cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M * nz0};
      cuuint64_t strides[1] = {(cuuint64_t)ldc * 4};
      cuuint32_t box[2] = {16, 32};
      cuuint32_t es[2] = {1, 1};
      c_tma = fn && fn(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  // the smem opt-in is per device: one bit per device this instantiation ran on
  static std::atomic<uint64_t> attr{0};
  int dev = 0;
  KP_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr.load(std::memory_order_acquire) & bit)) {
    KP_CUDA(cudaFuncSetAttribute(k_tc_gemm<AMN, BMN, BPRE, CG, H, AR>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr.fetch_or(bit, std::memory_order_release);
  }
  int kps = (K + splits - 1) / splits;
  kps = (kps + TC_BK - 1) / TC_BK * TC_BK;
  const unsigned nz = ceil_div(K, kps);
  const uint64_t works = (uint64_t)ceil_div(N, TC_BN) * ceil_div(M, TC_BM * CG) * nz;
  const int units = std::max(1, resident_units<AMN, BMN, BPRE, CG, H, AR>() - (g_reserve_sms + CG - 1) / CG);
  const unsigned grid = (unsigned)std::min<uint64_t>(works, (uint64_t)units) * CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(TC_WARPS * 32, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int kparam = kps;
  uint64_t works_l = works;
  if constexpr (AR) {
    // runs of n-blocks per m-block: enough units for balance, A loaded per run
    const int mb = (int)ceil_div(M, TC_BM * CG), nbl = (int)ceil_div(N, TC_BN);
    kparam = std::max(1, std::min(nbl, (int)ceil_div((uint64_t)4 * units, (uint64_t)mb)));
    works_l = (uint64_t)mb * kparam;
    cfg.gridDim = dim3((unsigned)std::min<uint64_t>(works_l, (uint64_t)units) * CG, 1, 1);
  }
  KP_CUDA(cudaLaunchKernelEx(&cfg, k_tc_gemm<AMN, BMN, BPRE, CG, H, AR>, ta, tb, tbl, tc, c_tma, M, N, K,
                             kparam, C, ldc, ep));
  ::kp::count_launch();
  return (int)nz;
}

template <bool AMN, bool BMN, bool BPRE>
int launch(int M, int N, int K, const float* A, int lda, const float* B, const float* Blo, int ldb,
           float* C, int ldc, int splits, const GemmEpi& ep, cudaStream_t s) {
  if (choose_cg(M) == 2)
    return launch_cg<AMN, BMN, BPRE, 2>(M, N, K, A, lda, B, Blo, ldb, C, ldc, splits, ep, s);
  return launch_cg<AMN, BMN, BPRE, 1>(M, N, K, A, lda, B, Blo, ldb, C, ldc, splits, ep, s);
}

}  // namespace

void tc_reserve_sms(int n) { g_reserve_sms = n < 0 ? 0 : n; }

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

// split-K count: best wave efficiency (units / (waves * resident units)) with
// >= 16 k-blocks per split; ties go to fewer splits (less partial traffic)
int tc_splits(int M, int N, int K) {
  const int cg = choose_cg(M);
  const int tiles = (int)(ceil_div(M, TC_BM * cg) * ceil_div(N, TC_BN));
  const int slots = std::max(1, (cg == 2 ? resident_units<true, true, false, 2>()
                                         : resident_units<true, true, false, 1>()) -
                                     (g_reserve_sms + cg - 1) / cg);
  const int max_sp = std::max(1, std::min(64, K / 512));
  int best = 1;
  double best_eff = 0;
  for (int sp = 1; sp <= max_sp; ++sp) {
    const int u = tiles * sp;
    const int waves = (u + slots - 1) / slots;
    const double eff = (double)u / ((double)waves * slots) - 0.004 * sp;
    if (eff > best_eff + 1e-9) best_eff = eff, best = sp;
  }
  return best;
}

// C[m][n] = epi(sum_k A[m][k] B[n][k])   (both K-major; B split in smem)
void tc_gemm_nt(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
                int ldc, const GemmEpi& ep, cudaStream_t s) {
  launch<false, false, false>(M, N, K, A, lda, B, nullptr, ldb, C, ldc, 1, ep, s);
}
// same with (B, B_lo) = split_hilo(B) precomputed (weights)
void tc_gemm_nt_pre(int M, int N, int K, const float* A, int lda, const float* Bhi, const float* Blo,
                    int ldb, float* C, int ldc, const GemmEpi& ep, cudaStream_t s) {
  launch<false, false, true>(M, N, K, A, lda, Bhi, Blo, ldb, C, ldc, 1, ep, s);
}

// fp16 operands (see TcCfg): C = epi(2^-(ea[m]+eb[n]) * (A*2^ea)(B*2^eb)^T)
void tc_gemm_nt_h(int M, int N, int K, const float* A, int lda, const float* a_rowmax,
                  const __half* Bhi, const __half* Blo, const int* b_exp, int ldb, float* C, int ldc,
                  const GemmEpi& ep, cudaStream_t s) {
  GemmEpi e2 = ep;
  e2.a_rowmax = a_rowmax;
  e2.b_exp = b_exp;
  static const bool ar_on = [] {
    const char* e = getenv("KP_GEMM_AR");
    return !(e && e[0] == '0');
  }();
  const bool ar = ar_on && K <= 2 * TC_BN;  // the whole K of A fits the 256 free TMEM columns
  if (choose_cg(M) == 2) {
    if (ar) launch_cg<false, false, true, 2, true, true>(M, N, K, A, lda, Bhi, Blo, ldb, C, ldc, 1, e2, s);
    else launch_cg<false, false, true, 2, true>(M, N, K, A, lda, Bhi, Blo, ldb, C, ldc, 1, e2, s);
  } else {
    if (ar) launch_cg<false, false, true, 1, true, true>(M, N, K, A, lda, Bhi, Blo, ldb, C, ldc, 1, e2, s);
    else launch_cg<false, false, true, 1, true>(M, N, K, A, lda, Bhi, Blo, ldb, C, ldc, 1, e2, s);
  }
}
void split_h(const float* W, int N, int K, int ld, __half* hi, __half* lo, int* exps, cudaStream_t s) {
  // one block per row; long rows (the 6400-wide W1) get 1024 threads so the
  // 256-row grid keeps enough loads in flight
  k_split_h<<<N, K >= 4096 ? 1024 : 256, 0, s>>>(W, K, ld, hi, lo, exps); ::kp::count_launch();
}
void rowmax(const float* A, int M, int K, int lda, float* out, cudaStream_t s) {
  k_rowmax<<<std::min<unsigned>(ceil_div((uint64_t)M * 32, 256), 148 * 16), 256, 0, s>>>(A, M, K, lda, out); ::kp::count_launch();
}
bool tc_h_enabled() {
  static const bool on = [] {
    const char* e = getenv("KP_GEMM_F16");
    return !(e && e[0] == '0');
  }();
  return on;
}

// C[z][m][n] = sum_{k in split z} A[k][m] B[k][n]   (both MN-major); returns #splits
int tc_gemm_tn(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
               int ldc, int splits, cudaStream_t s) {
  GemmEpi ep{0, 0, nullptr, nullptr, 0, nullptr, 1, 1};
  return launch<true, true, false>(M, N, K, A, lda, B, nullptr, ldb, C, ldc, splits, ep, s);
}

}  // namespace kp
