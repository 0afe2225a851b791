// fp32-accurate GEMM on pre-split fp16 operands ("3xFP16", tcgen05 kind::f16).
//
//   C = epi( 2^-(ea[m] + eb[n]) * sum_k (Ah*Bh + Ah*Bl + Al*Bh)(m, n, k) )
//
// Every operand arrives in HBM as two fp16 planes, hi = rn(x * 2^e) and
// lo = rn(x * 2^e - hi), with a power-of-two scale per row of A (ea) and per
// row of B (eb) that puts the row's max |x| in [2^14, 2^15): hi + lo carries 22
// significant bits like tf32 hi + lo, at the fp16 tensor rate (2x tf32), and
// the dropped lo*lo term is ~2^-22 relative. The planes are produced by the
// kernels that write the operands anyway (the pooling kernel writes the MLP
// input as planes, the weight and upstream-gradient splits below), so the
// GEMM itself only streams them: no on-chip split, TMA straight into the
// UMMA layouts, both MMA operands from shared memory.
//
// Layer 1 of the CTR MLP (proj/src/model.cpp:100-191) at configs[1]
// (B = 65536, S*e = 6400, hidden 256) runs three of these:
//   forward   Z = X W1^T       A = X planes [B][6400] (K-major), B = W1 [256][6400]
//   dX        dX = dZ W1       A = dZ1 [B][256] (K-major), B = W1^T [6400][256]
//   dW        dW = dZ^T X      A = dZ' [B][256] (MN-major), B = X [B][6400] (MN-major),
//             split over the batch (stream-K, deterministic fix-up)
//
// CTA pair (cluster of 2, tcgen05.mma.cta_group::2): tile M = 256 (128 rows
// per CTA) x N = 256 (each CTA holds 128 of the B rows), k-block 32. TMEM:
// two 256-column fp32 accumulators; the tensor core's accumulation is not
// IEEE round-to-nearest and its error grows with K, so the MMA switches
// accumulator every H3_CH k-blocks (512 k) and the epilogue warps fold the
// finished one into fp32 registers with RN adds -- fp32-level accuracy
// independent of K (the same scheme as kp_gemm_tc.cu).
// Warps (per CTA): 0 TMA producer; 1 TMEM allocator, the leader's lane 0
// issues the MMAs, the peer's lane 0 relays its TMA completions; 2-3 idle;
// 4-19 drain + epilogue (warp w: TMEM lane quarter w%4, 64-column quarter
// (w-4)/4, TMA store of 32x16 fp32 boxes). setmaxnreg moves registers from
// warpgroup 0 to the epilogue warpgroups (64 fp32 running sums per thread).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kp_internal.cuh"
#include "kp_tcgen05.cuh"

namespace kp {
namespace {

using namespace tc;

constexpr int H3_BM = 128;   // rows per CTA (pair: 256)
constexpr int H3_BN = 256;   // tile columns (each CTA holds 128 B rows)
constexpr int H3_BK = 32;    // k per stage
// epilogue store box: H3_EB fp32 columns x 32 rows per TMA store (16: SW64,
// 2 KB; 32: SW128, 4 KB), one per epilogue warp; the smaller box leaves
// room for a fifth operand stage
constexpr int H3_EB = 16;
constexpr int H3_EPIB = 2;   // store boxes per epilogue warp (double-buffered)
constexpr int H3_NS = 4;     // smem stages
constexpr int H3_CH = 16;    // k-blocks per accumulator chunk (512 k)
constexpr int H3_WARPS = 20;  // warpgroup 0: producer, MMA, 2 idle; warpgroups 1-4: epilogue
constexpr int H3_EPI_T = 512;
constexpr uint32_t H3_PLANE = H3_BM * H3_BK * 2;  // 8 KB: one plane tile per CTA
constexpr uint32_t H3_STAGE = 4 * H3_PLANE;       // A hi, A lo, B hi, B lo
constexpr uint32_t H3_EPI = 16 * H3_EPIB * 32 * H3_EB * 4;  // per epilogue warp H3_EPIB 32 x H3_EB fp32 store tiles
// register split (setmaxnreg, per warpgroup): the epilogue holds 64 fp32
// running sums per thread; the TMA / MMA warps need few
constexpr int H3_REG_LO = 64, H3_REG_HI = 104;  // 128*64 + 512*104 <= 640*96 (the CTA pool)
constexpr uint32_t H3_COLP = 16 * 2 * 64 * 4;  // per epilogue warp: 64 column scales + 64 biases
constexpr uint32_t H3_SMEM = H3_NS * H3_STAGE + H3_EPI + H3_COLP + 1024 + 256;
// Tile width BN = 256 (2 TMEM accumulators; each CTA holds BN/2 rows of B).
// (A 128-wide variant with 4 accumulators in flight measured slower for dX,
// 702 vs 556 us, and was dropped.)
// GA (gathered A): A's rows are fetched as fp32 by TMA gather4 from a row
// table (one feature per slot: A[m][slot*e + j] = src[rowocc[m*S + slot]][j]),
// into NG staging slots, and split into the A planes on chip by warps 2-3.
template <int BN, bool GA = false>
struct H3Cfg {
  static constexpr int NBUF = 512 / BN;
  static constexpr int BROWS = BN / 2;
  static constexpr uint32_t B_PLANE = BROWS * H3_BK * 2;
  static constexpr uint32_t STAGE = 2 * H3_PLANE + 2 * B_PLANE;
  static constexpr int NS = BN == 256 ? 4 : 6;
  static constexpr int CW = BN / 4;  // columns per epilogue warp
  static constexpr int EPIB = GA ? 1 : H3_EPIB;  // (GA: one store box per warp, room for the staging)
  static constexpr uint32_t EPI = 16 * EPIB * 32 * H3_EB * 4;
  static constexpr int NG = GA ? 2 : 0;
  static constexpr uint32_t GSLOT = H3_BM * H3_BK * 4;  // 128 rows x 32 fp32
  static constexpr uint32_t GEXP = GA ? H3_BM * 4 : 0;  // the tile rows' exponents
  static constexpr uint32_t SMEM = NS * STAGE + EPI + H3_COLP + NG * GSLOT + GEXP + 1024 + 256;
};
static_assert(H3Cfg<256>::SMEM <= 232448 && H3Cfg<256, true>::SMEM <= 232448, "h3 smem");
// stream-K virtual units (the partition depends only on the problem shape,
// not on the grid): 148, or fewer so that each owns >= 8 k-blocks
constexpr int H3_VUNITS = 148;
__host__ __device__ __forceinline__ int h3_vunits(int64_t T) {
  const int64_t v = T / 8;
  return v < 1 ? 1 : (v > H3_VUNITS ? H3_VUNITS : (int)v);
}

struct H3Args {
  int M, N, K;
  int nblocks_m, nblocks_n, nk;  // tiles and k-blocks
  int splitk;                    // stream-K over vunits virtual units
  int vunits;
  int tiles_dp;                  // stream-K kernels: whole tiles [0, tiles_dp) first, the rest stream-K
  const int* ea;                 // per-row exponents of A (nullable = 0)
  const int* eb;                 // per-row exponents of B (nullable = 0)
  int keep_a, keep_b;            // L2 policy per operand: 1 evict_last (re-read), 0 evict_first
  int dbg;                       // timing experiments only (KP_H3_DBG): 1 no stores, 2 no drain,
                                 // 3 no A conversion, 4 no A gathers (GA)
  int mode;                      // 0 store, 1 act(x + bias[n]), 3 x * coeff[m*S + n/e]
  int act;
  const float* bias;
  const float* coeff;
  uint32_t S, e;
  // GA: row of (m, slot) in the gather source, S slots of gkps k-blocks;
  // gstore: also store the A planes (for a later GEMM over the same input)
  const uint32_t* grow;
  uint32_t gS, gkps;
  int gstore;
};

// the k-block range of virtual unit v over T = tiles * nk iterations
__device__ __forceinline__ int64_t vstart(int64_t v, int64_t T, int V) { return v * T / V; }

// Iterates the (tile, kb0, kb1) segments of one physical unit: data-parallel
// (whole tiles w = unit, unit+units, ...) or stream-K: first the whole tiles
// [0, tiles_dp) as in data-parallel, then the virtual units v = unit,
// unit+units, ... each owning [vstart(v), vstart(v+1)) of the flattened
// (tail tile x k-block) space; a stream-K segment's partial-tile id is
// (tile - tiles_dp) + v (unique). The split depends only on the shape.
template <bool SK>
struct SegIter {
  int tiles, nk, units, V, tdp, u0;
  int v;  // current whole tile, then (stream-K) virtual unit
  bool whole;
  int64_t T, t, tend;
  __device__ SegIter(const H3Args& a, int unit, int units_)
      : tiles(a.nblocks_m * a.nblocks_n), nk(a.nk), units(units_), V(a.vunits) {
    v = unit;
    u0 = unit;
    if constexpr (SK) {
      tdp = a.tiles_dp;
      whole = v < tdp;
      T = (int64_t)(tiles - tdp) * nk;
      t = tend = 0;
      if (!whole) start_sk(unit);
    }
  }
  __device__ void start_sk(int u) {
    v = u;
    t = tend = 0;
    if (v < V) {
      t = vstart(v, T, V);
      tend = vstart(v + 1, T, V);
    }
  }
  // next segment: tile index, [kb0, kb1), partial-tile id (stream-K part),
  // partial; false when done
  __device__ bool next(int& tile, int& kb0, int& kb1, int& sid, bool& partial) {
    if constexpr (!SK) {
      if (v >= tiles) return false;
      tile = v;
      kb0 = 0;
      kb1 = nk;
      sid = v;
      partial = false;
      v += units;
      return true;
    } else {
      if (whole) {
        tile = v;
        kb0 = 0;
        kb1 = nk;
        sid = v;
        partial = false;
        v += units;
        if (v >= tdp) {
          whole = false;
          start_sk(u0);
        }
        return true;
      }
      while (t >= tend) {
        v += units;
        if (v >= V) return false;
        t = vstart(v, T, V);
        tend = vstart(v + 1, T, V);
      }
      const int lt = (int)(t / nk);
      tile = tdp + lt;
      kb0 = (int)(t % nk);
      const int64_t e = kb0 + (tend - t);
      kb1 = (int)(e < nk ? e : nk);
      sid = lt + v;
      partial = true;
      t += kb1 - kb0;
      return true;
    }
  }
};

// tile -> (m-block, n-block), n fastest: concurrently running units share A rows
__device__ __forceinline__ void tile_mn(const H3Args& a, int tile, int& mb, int& nb) {
  nb = tile % a.nblocks_n;
  mb = tile / a.nblocks_n;
}

__device__ __forceinline__ float act_fwd(int act, float z) { return act == 0 ? (z > 0.f ? z : 0.f) : tanhf(z); }

// one plane tile (ROWS of this CTA's rows x 32 k) of a K-major or MN-major operand
template <bool MN, int ROWS = 128>
__device__ __forceinline__ void load_plane(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int k0, int r0,
                                           uint64_t pol) {
  if (MN) {  // 64(mn) x 32(k) SW128 boxes, LBO = 4 KB apart
#pragma unroll
    for (int i = 0; i < ROWS / 64; ++i) tma_load_2d_hint(dst + 4096 * i, map, bar, r0 + 64 * i, k0, pol);
  } else {   // one 32(k) x ROWS SW64 box
    tma_load_2d_hint(dst, map, bar, k0, r0, pol);
  }
}
template <bool MN>
__device__ __forceinline__ uint64_t plane_desc(uint32_t base, int kk) {
  return MN ? sdesc_mn128(base + (uint32_t)kk * 2048u, 4096u) : sdesc_k64(base + (uint32_t)kk * 32u);
}

template <bool AMN, bool BMN, bool SK, int BN, bool GA, int EM>
__global__ void __launch_bounds__(H3_WARPS * 32, 1)
    k_h3(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
         const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
         const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmP,
         const __grid_constant__ CUtensorMap tmG, H3Args a) {
  static_assert(!GA || (!AMN && BN == 256), "gathered A: K-major, 256-wide tiles");
  using Cfg = H3Cfg<BN, GA>;
  // (NG: the staging ring's modulus, 1 without staging)
  constexpr int NS = Cfg::NS, NBUF = Cfg::NBUF, CW = Cfg::CW, EPIB = Cfg::EPIB, NG = Cfg::NG > 0 ? Cfg::NG : 1;
  constexpr uint32_t STAGE = Cfg::STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stages = smem;
  uint8_t* epi = stages + NS * STAGE;
  float* colp = reinterpret_cast<float*>(epi + Cfg::EPI);
  uint8_t* gstage = reinterpret_cast<uint8_t*>(colp) + H3_COLP;  // GA: fp32 staging slots
  int* gexp = reinterpret_cast<int*>(gstage + Cfg::NG * Cfg::GSLOT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(gexp) + Cfg::GEXP);
  uint64_t* full = bars;              // TMA -> MMA (local)
  uint64_t* conv = bars + NS;         // peer's TMA landed -> leader's MMA (1 arrival)
  uint64_t* empty = bars + 2 * NS;    // MMA done with stage -> producers (both CTAs)
  uint64_t* tfull = bars + 3 * NS;    // chunk accumulated -> drains (both CTAs)
  uint64_t* tempty = tfull + NBUF;    // drained -> MMA (leader; 2 arrivals)
  uint64_t* cvt = tempty + NBUF;      // GA: A planes written -> MMA / relay (local)
  uint64_t* gfull = cvt + NS;         // GA: gathered rows landed -> converters
  uint64_t* gempty = gfull + Cfg::NG; // GA: staging slot read -> producer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gempty + Cfg::NG);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int unit = blockIdx.x >> 1, units = gridDim.x >> 1;
  auto sAh = [&](int s) { return stages + s * STAGE; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2);
    }
    if constexpr (GA) {
      for (int s = 0; s < NS; ++s) mbar_init(&cvt[s], 1);
      for (int j = 0; j < NG; ++j) {
        mbar_init(&gfull[j], 1);
        mbar_init(&gempty[j], 1);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(H3_REG_LO));
  if (GA && warp == 0) {
    // ---- gathered-A producer: lane l fetches A rows 4l..4l+3 (fp32, 32 k of
    // their slot's source row) with one gather4 per k-block; lane 0 also the
    // B planes. The next slot's row indices are loaded one slot ahead.
    if (lane == 0) {
      prefetch_map(&tmBh);
      prefetch_map(&tmBl);
      prefetch_map(&tmG);
    }
    const uint64_t pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
    const uint64_t pb = a.keep_b ? pol_keep : pol_stream;
    SegIter<SK> it(a, unit, units);
    int tile, kb0, kb1, sid, g = 0;
    bool partial;
    while (it.next(tile, kb0, kb1, sid, partial)) {
      int mb, nb;
      tile_mn(a, tile, mb, nb);
      const int m0 = mb * 2 * H3_BM + (int)rank * H3_BM;
      const int n0 = nb * BN + (int)rank * Cfg::BROWS;
      auto rows_of = [&](int slot, uint32_t (&r)[4]) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int m = m0 + 4 * lane + t;
          r[t] = (m < a.M && slot < (int)a.gS) ? __ldg(a.grow + (size_t)m * a.gS + slot) : 0u;
        }
      };
      int slot = kb0 / (int)a.gkps;
      uint32_t ri[4], nx[4];
      rows_of(slot, ri);
      rows_of(slot + 1, nx);
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % NS, j = g % NG;
        const int sl = kb / (int)a.gkps;
        if (sl != slot) {  // (slots advance one at a time inside a segment)
          slot = sl;
#pragma unroll
          for (int t = 0; t < 4; ++t) ri[t] = nx[t];
          rows_of(slot + 1, nx);
        }
        if (lane == 0) {
          if (g >= NS) mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);
          mbar_expect_tx(&full[s], 2 * Cfg::B_PLANE);
          uint8_t* st = sAh(s);
          load_plane<BMN, Cfg::BROWS>(st + 2 * H3_PLANE, &tmBh, &full[s], kb * H3_BK, n0, pb);
          load_plane<BMN, Cfg::BROWS>(st + 2 * H3_PLANE + Cfg::B_PLANE, &tmBl, &full[s], kb * H3_BK, n0, pb);
          if (g >= NG) mbar_wait(&gempty[j], ((g / NG) & 1) ^ 1);
          if (a.dbg == 4) mbar_arrive(&gfull[j]);  // timing experiment: no gathers
          else mbar_expect_tx(&gfull[j], Cfg::GSLOT);
        }
        __syncwarp();
        if (a.dbg != 4)
          tma_gather4(gstage + j * Cfg::GSLOT + lane * (4 * H3_BK * 4), &tmG, &gfull[j],
                      (kb % (int)a.gkps) * H3_BK, ri);
      }
    }
  } else if (GA && (warp == 2 || warp == 3)) {
    // ---- converters: staging fp32 rows -> x * 2^e(row) -> hi/lo fp16 in the
    // SW64 K-major layout the A planes' TMA would have produced; optionally
    // stored to the planes in HBM (TMA) for a later GEMM
    const int ct = threadIdx.x - 64, w2 = warp - 2;
    SegIter<SK> it(a, unit, units);
    int tile, kb0, kb1, sid, g = 0;
    bool partial;
    while (it.next(tile, kb0, kb1, sid, partial)) {
      int mb, nb;
      tile_mn(a, tile, mb, nb);
      const int m0 = mb * 2 * H3_BM + (int)rank * H3_BM;
      named_sync(2, 64);  // the previous segment's conversions are done with gexp
      for (int r = ct; r < H3_BM; r += 64) gexp[r] = (a.ea && m0 + r < a.M) ? __ldg(a.ea + m0 + r) : 0;
      named_sync(2, 64);
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % NS, j = g % NG;
        mbar_wait(&gfull[j], (g / NG) & 1);
        if (g >= NS) mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);  // the MMAs are done with the A slots
        if (ct == 0 && g >= NS && a.gstore)  // ... and so is this slot's previous plane store
          asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(2 * NS - 2) : "memory");
        named_sync(2, 64);
        const uint8_t* gs = gstage + j * Cfg::GSLOT;
        uint8_t* ah = sAh(s);
#pragma unroll 4
        for (int i = 0; i < (a.dbg == 3 ? 0 : 16); ++i) {  // (dbg 3: timing experiment, no conversion)
          // 8 lanes per row (one 128-byte row per quarter warp: conflict-free)
          const int r = w2 * 64 + i * 4 + (lane >> 3), c = lane & 7;
          const float4 v = *reinterpret_cast<const float4*>(gs + r * (H3_BK * 4) + c * 16);
          const float sc = pow2f(gexp[r]);
          uint32_t h0, l0, h1, l1;
          split_h2(__fmul_rn(v.x, sc), __fmul_rn(v.y, sc), h0, l0);
          split_h2(__fmul_rn(v.z, sc), __fmul_rn(v.w, sc), h1, l1);
          // SW64: row r's 16-byte chunk q at q ^ ((r >> 1) & 3); halves 4c..4c+3 = 8 bytes
          const uint32_t off = (uint32_t)(r * 64) + ((uint32_t)((c >> 1) ^ ((r >> 1) & 3)) << 4) + ((c & 1) << 3);
          st_shared_v2(smem_u32(ah) + off, h0, h1);
          st_shared_v2(smem_u32(ah + H3_PLANE) + off, l0, l1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_sync(2, 64);
        if (ct == 0) {
          mbar_arrive(&gempty[j]);
          if (a.gstore) {
            tma_store_2d(&tmAh, ah, kb * H3_BK, m0);
            tma_store_2d(&tmAl, ah + H3_PLANE, kb * H3_BK, m0);
          }
          mbar_arrive(&cvt[s]);
        }
      }
    }
    if (ct == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp == 0) {
    // ---- TMA producer: this CTA's 128 A rows and 128 B rows per k-block
    if (lane == 0) {
      prefetch_map(&tmAh);
      prefetch_map(&tmAl);
      prefetch_map(&tmBh);
      prefetch_map(&tmBl);
      // the operand re-read across tiles stays in L2, the streamed one goes first
      const uint64_t pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
      const uint64_t pa = a.keep_a ? pol_keep : pol_stream, pb = a.keep_b ? pol_keep : pol_stream;
      SegIter<SK> it(a, unit, units);
      int tile, kb0, kb1, sid, g = 0;
      bool partial;
      while (it.next(tile, kb0, kb1, sid, partial)) {
        int mb, nb;
        tile_mn(a, tile, mb, nb);
        const int m0 = mb * 2 * H3_BM + (int)rank * H3_BM;
        const int n0 = nb * BN + (int)rank * Cfg::BROWS;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % NS;
          if (g >= NS) mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);
          mbar_expect_tx(&full[s], STAGE);
          uint8_t* st = sAh(s);
          load_plane<AMN>(st, &tmAh, &full[s], kb * H3_BK, m0, pa);
          load_plane<AMN>(st + H3_PLANE, &tmAl, &full[s], kb * H3_BK, m0, pa);
          load_plane<BMN, Cfg::BROWS>(st + 2 * H3_PLANE, &tmBh, &full[s], kb * H3_BK, n0, pb);
          load_plane<BMN, Cfg::BROWS>(st + 2 * H3_PLANE + Cfg::B_PLANE, &tmBl, &full[s], kb * H3_BK, n0, pb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---- MMA issuer (leader CTA): both CTAs' tiles, M = 256
      constexpr uint32_t idesc = idesc_f16(AMN, BMN, 2 * H3_BM, BN);
      SegIter<SK> it(a, unit, units);
      int tile, kb0, kb1, sid, g = 0, c = 0;
      bool partial;
      while (it.next(tile, kb0, kb1, sid, partial)) {
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % NS;
          const int kin = (kb - kb0) % H3_CH, buf = c % NBUF;
          if (kin == 0 && c >= NBUF) mbar_wait(&tempty[buf], ((c / NBUF) - 1) & 1);
          mbar_wait(&full[s], (g / NS) & 1);
          if constexpr (GA) mbar_wait(&cvt[s], (g / NS) & 1);
          mbar_wait(&conv[s], (g / NS) & 1);
          fence_after();
          const uint32_t d = tmem + (uint32_t)(buf * BN);
          const uint32_t ah = smem_u32(sAh(s)), al = ah + H3_PLANE, bh = ah + 2 * H3_PLANE,
                         bl = bh + Cfg::B_PLANE;
#pragma unroll
          for (int kk = 0; kk < H3_BK / 16; ++kk) {
            const uint64_t dah = plane_desc<AMN>(ah, kk), dal = plane_desc<AMN>(al, kk);
            const uint64_t dbh = plane_desc<BMN>(bh, kk), dbl = plane_desc<BMN>(bl, kk);
            mma_f16_pair(d, dah, dbh, idesc, (kin | kk) != 0);
            mma_f16_pair(d, dah, dbl, idesc, 1);
            mma_f16_pair(d, dal, dbh, idesc, 1);
          }
          commit_pair(&empty[s]);
          if (kin == H3_CH - 1 || kb == kb1 - 1) {
            commit_pair(&tfull[buf]);
            ++c;
          }
        }
      }
    } else if (lane == 0) {
      // ---- peer CTA: relay "my TMA landed" to the leader's MMA issuer
      SegIter<SK> it(a, unit, units);
      int tile, kb0, kb1, sid, g = 0;
      bool partial;
      while (it.next(tile, kb0, kb1, sid, partial))
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % NS;
          mbar_wait(&full[s], (g / NS) & 1);
          if constexpr (GA) mbar_wait(&cvt[s], (g / NS) & 1);
          mbar_arrive_leader(&conv[s]);
        }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(H3_REG_HI));
    // ---- drain + epilogue (16 warps): TMEM lane quarter q, columns [cq*64, +64)
    const int q = warp & 3, cq = (warp - 4) >> 2;
    const int et = threadIdx.x - 128;
    uint8_t* dense_base = epi + (warp - 4) * (EPIB * 32 * H3_EB * 4);
    uint32_t tma_seq = 0;
    SegIter<SK> it(a, unit, units);
    int tile, kb0, kb1, sid, c = 0;
    bool partial;
    while (it.next(tile, kb0, kb1, sid, partial)) {
      int mb, nb;
      tile_mn(a, tile, mb, nb);
      const int mrow0 = mb * 2 * H3_BM + (int)rank * H3_BM + q * 32;  // this warp's 32 rows
      const int ncol0 = nb * BN + cq * CW;                             // this warp's CW columns
      // column scales / biases and the row scale, loaded while the MMAs run
      float* csb = colp + (warp - 4) * 128;
      __syncwarp();  // the previous tile's epilogue is done reading csb
#pragma unroll
      for (int h = 0; h < CW / 32; ++h) {
        const int nn = min(ncol0 + lane + 32 * h, a.N - 1);
        csb[lane + 32 * h] = a.eb ? pow2f(-__ldg(a.eb + nn)) : 1.f;
        csb[64 + lane + 32 * h] = EM == 1 ? __ldg(a.bias + nn) : 0.f;
      }
      const int m = mrow0 + lane;
      const float sa = (a.ea && m < a.M) ? pow2f(-__ldg(a.ea + m)) : 1.f;
      // the epilogue op is a template parameter (EM): one op's code per kernel
      // keeps the unrolled epilogue small (the runtime-selected version with
      // every op inlined 64-wide measured instruction-fetch stalls on top);
      // partial tiles: plain scaled sums (the fix-up applies the op)
      const int mode = partial ? 0 : EM;
      float acc[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) acc[j] = 0.f;
      const int nch = (kb1 - kb0 + H3_CH - 1) / H3_CH;
      for (int ci = 0; ci < nch; ++ci, ++c) {
        const int buf = c % NBUF;
        mbar_wait(&tfull[buf], (c / NBUF) & 1);
        fence_after();
#pragma unroll
        for (int c0 = 0; c0 < CW; c0 += 16) {
          uint32_t r[16];
          if (a.dbg == 2) {
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = 0;
          } else {
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN + cq * CW + c0), r);
            tmem_ld_wait();
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[c0 + j] = __fadd_rn(acc[c0 + j], __uint_as_float(r[j]));
        }
        fence_before();
        named_sync(1, H3_EPI_T);
        if (et == 0) mbar_arrive_leader(&tempty[buf]);
      }
      // epilogue: row per lane; exact power-of-two unscaling, then the op;
      // 32 x H3_EB fp32 boxes, one TMA store each (lane = row; its 16-byte
      // chunks XOR-swizzled by the row, conflict-free)
      __syncwarp();  // csb visible to the warp
#pragma unroll
      for (int h = 0; h < CW / H3_EB; ++h, ++tma_seq) {
        uint8_t* box = dense_base + (tma_seq % EPIB) * (32 * H3_EB * 4);
        const uint32_t dense = smem_u32(box);
        const int c0 = H3_EB * h;
        const int n = ncol0 + c0;
        float* v = acc + c0;  // transformed in place (registers)
#pragma unroll
        for (int j = 0; j < H3_EB; ++j) {
          v[j] = __fmul_rn(__fmul_rn(v[j], sa), csb[c0 + j]);
          if (mode == 1) v[j] = act_fwd(a.act, __fadd_rn(v[j], csb[64 + c0 + j]));
        }
        if (mode == 3) {  // mean-pooling coefficient of the column's slot (few distinct per box)
          const float* cp = a.coeff + (size_t)min(m, a.M - 1) * a.S;
          int slot = -1;
          float cf = 1.f;
#pragma unroll
          for (int j = 0; j < H3_EB; ++j) {
            const int sj = min(n + j, a.N - 1) / (int)a.e;
            if (sj != slot) slot = sj, cf = __ldg(cp + sj);
            v[j] = __fmul_rn(v[j], cf);
          }
        }
        // the store that last used this buffer has read it out of shared memory
        if (lane == 0) {
          if (EPIB == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < H3_EB / 4; ++cc) {
          const uint32_t sw = H3_EB == 32 ? (uint32_t)(cc ^ (lane & 7)) : (uint32_t)(cc ^ ((lane >> 1) & 3));
          st_shared_v4(dense + lane * (H3_EB * 4) + (sw << 4), v[4 * cc], v[4 * cc + 1], v[4 * cc + 2],
                       v[4 * cc + 3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && a.dbg != 1) {
          if (SK && partial)  // partial tile of segment sid: rows sid*256 + local row
            tma_store_2d(&tmP, box, cq * CW + c0, sid * 2 * H3_BM + (int)rank * H3_BM + q * 32);
          else
            tma_store_2d(&tmC, box, n, mrow0);
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

// stream-K fix-up: C tile = op(sum of its segments' partials in k order),
// for the stream-K tiles tdp + blockIdx.y (op: mode 0 store, 1 act(x + bias))
__global__ void k_h3_fixup(const float* __restrict__ part, int nblocks_n, int nk, int tdp, int64_t T, int V,
                           int M, int N, float* __restrict__ C, int ldc, int mode, int act,
                           const float* __restrict__ bias) {
  const int lt = blockIdx.y, tile = tdp + lt;
  const int mb = tile / nblocks_n, nb = tile % nblocks_n;
  const int64_t t0 = (int64_t)lt * nk, t1 = t0 + nk - 1;
  // unit(t) = max v with vstart(v) <= t = floor(((t+1)*V - 1) / T)
  const int v0 = (int)(((t0 + 1) * V - 1) / T), v1 = (int)(((t1 + 1) * V - 1) / T);
  // the tile's contributing virtual units, once per block (some own no k-block
  // when the k-blocks are fewer than the units)
  __shared__ int vlist[H3_VUNITS];
  __shared__ int nv;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int v = v0; v <= v1; ++v)
      if (vstart(v + 1, T, V) > vstart(v, T, V)) vlist[c++] = v;
    nv = c;
  }
  __syncthreads();
  // 4 consecutive columns per thread (float4 partial loads)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * H3_BM * H3_BN / 4; i += gridDim.x * blockDim.x) {
    const int r = (4 * i) / H3_BN, cc = (4 * i) % H3_BN;
    const int m = mb * 2 * H3_BM + r, n = nb * H3_BN + cc;
    if (m >= M || n >= N) continue;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < nv; ++j) {
      const float4 p = *reinterpret_cast<const float4*>(part + ((size_t)(lt + vlist[j]) * 2 * H3_BM + r) * H3_BN + cc);
      s.x = __fadd_rn(s.x, p.x), s.y = __fadd_rn(s.y, p.y), s.z = __fadd_rn(s.z, p.z), s.w = __fadd_rn(s.w, p.w);
    }
    float v[4] = {s.x, s.y, s.z, s.w};
    if (mode == 1)
#pragma unroll
      for (int t = 0; t < 4; ++t) v[t] = act_fwd(act, __fadd_rn(v[t], __ldg(bias + min(n + t, N - 1))));
    float* c = C + (size_t)m * ldc + n;
    if (n + 3 < N && (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
      *reinterpret_cast<float4*>(c) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
      for (int t = 0; t < 4 && n + t < N; ++t) c[t] = v[t];
    }
  }
}

// ---- host ------------------------------------------------------------------
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

// fp16 plane [rows][cols] (ld halves): K-major boxes 32(k) x box_rows SW64,
// MN-major boxes 64(mn) x 32(k) SW128 (rows = K, cols = MN)
bool map_plane(CUtensorMap* m, const __half* p, uint64_t rows, uint64_t cols, uint64_t ld, bool mn,
               uint32_t box_rows = 128) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {mn ? 64u : 32u, mn ? 32u : box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(p), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, mn ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// fp32 [rows][cols] output, H3_EB x 32 boxes (the epilogue's store tiles)
bool map_out(CUtensorMap* m, float* p, uint64_t rows, uint64_t cols, uint64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)H3_EB, 32};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            H3_EB == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// gather source rows [nrows][e] fp32: boxes of 32 columns x 1 row (gather4
// fetches four of them)
bool map_rows(CUtensorMap* m, const float* p, uint64_t nrows, uint32_t e) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {e, nrows};
  cuuint64_t strides[1] = {(cuuint64_t)e * 4};
  cuuint32_t box[2] = {(cuuint32_t)H3_BK, 1};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fprintf(stderr, "map_rows: cuTensorMapEncodeTiled %d (rows %llu, e %u, p %p)\n", (int)r,
                                 (unsigned long long)nrows, e, (const void*)p);
  return r == CUDA_SUCCESS;
}

thread_local int g_h3_reserve = 0;

template <bool AMN, bool BMN, bool SK, int BN, bool GA, int EM>
void launch_h3_t(const H3Operand& A, const H3Operand& B, int M, int N, int K, float* C, int ldc, float* ws,
                 const H3Args& a0, cudaStream_t s, int split, const H3Gather* ga);
// one kernel per epilogue op (EM): the ops each operand layout uses -- the
// forward's bias + activation and the input gradient's mean-pool coefficient
// on K-major operands, plain stores everywhere
template <bool AMN, bool BMN, bool SK, bool GA>
void launch_em(const H3Operand& A, const H3Operand& B, int M, int N, int K, float* C, int ldc, float* ws,
               const H3Args& a, cudaStream_t s, int split, const H3Gather* ga) {
  if (a.mode == 1) {
    if constexpr (!AMN && !BMN) {
      launch_h3_t<AMN, BMN, SK, 256, GA, 1>(A, B, M, N, K, C, ldc, ws, a, s, split, ga);
      return;
    }
  } else if (a.mode == 3) {
    if constexpr (!AMN && !BMN && !SK && !GA) {
      launch_h3_t<AMN, BMN, SK, 256, GA, 3>(A, B, M, N, K, C, ldc, ws, a, s, split, ga);
      return;
    }
  } else if (a.mode == 0) {
    if constexpr (!GA) {
      launch_h3_t<AMN, BMN, SK, 256, GA, 0>(A, B, M, N, K, C, ldc, ws, a, s, split, ga);
      return;
    }
  }
  KP_CHECK(false, kErrGeneric, "h3_gemm: epilogue op not built for this operand layout");
}

// stream-K and data-parallel variants are separate kernels (no 64-bit
// stream-K state in the data-parallel ones)
template <bool AMN, bool BMN>
void launch_h3(const H3Operand& A, const H3Operand& B, int M, int N, int K, float* C, int ldc, int splitk,
               float* ws, const H3Args& a, cudaStream_t s, const H3Gather* ga = nullptr) {
  static const bool hybrid = [] {
    const char* e = getenv("KP_H3_HYBRID");
    return !(e && e[0] == '0');
  }();
  if (splitk == 2) {
    // whole tiles in full waves of the 74 pairs, the last partial wave
    // stream-K (shape-only split); all whole: the data-parallel kernel
    const int tiles = (int)(ceil_div(M, 2 * H3_BM) * ceil_div(N, H3_BN));
    // (below one full wave -- short-K small batches -- the fix-up costs more
    // than the balance gains; at configs[1] the split measured -5 us in situ)
    if (tiles % (H3_VUNITS / 2) == 0 || tiles < H3_VUNITS / 2 || !hybrid) splitk = 0;
  }
  if constexpr (!AMN && !BMN) {
    if (ga) {
      if (splitk) launch_em<false, false, true, true>(A, B, M, N, K, C, ldc, ws, a, s, splitk, ga);
      else launch_em<false, false, false, true>(A, B, M, N, K, C, ldc, ws, a, s, 0, ga);
      return;
    }
  }
  KP_CHECK(!ga, kErrGeneric, "h3_gemm: gathered A must be K-major");
  if (splitk) launch_em<AMN, BMN, true, false>(A, B, M, N, K, C, ldc, ws, a, s, splitk, nullptr);
  else launch_em<AMN, BMN, false, false>(A, B, M, N, K, C, ldc, ws, a, s, 0, nullptr);
}

template <bool AMN, bool BMN, bool SK, int BN, bool GA, int EM>
int h3_units() {
  static int units = 0;
  if (units) return units;
  int dev = 0, sms = 0;
  KP_CUDA(cudaGetDevice(&dev));
  KP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  units = sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(4, 1, 1);
  cfg.blockDim = dim3(H3_WARPS * 32, 1, 1);
  cfg.dynamicSmemBytes = H3Cfg<BN, GA>::SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_h3<AMN, BMN, SK, BN, GA, EM>, &cfg) == cudaSuccess && n > 0)
    units = std::min(units, n);
  cudaGetLastError();
  return units;
}

template <bool AMN, bool BMN, bool SK, int BN, bool GA, int EM>
void launch_h3_t(const H3Operand& A, const H3Operand& B, int M, int N, int K, float* C, int ldc, float* ws,
                 const H3Args& a0, cudaStream_t s, int split, const H3Gather* ga) {
  static_assert(!SK || BN == 256, "stream-K partial tiles are 256 wide");
  constexpr bool splitk = SK;
  CUtensorMap tah, tal, tbh, tbl, tcm, tpm, tgm;
  // K-major operand [rows][K]; MN-major [K][rows]
  auto mk = [&](CUtensorMap* m, const __half* p, const H3Operand& op, int rows, bool mn, uint32_t box_rows) {
    return mn ? map_plane(m, p, K, rows, op.ld, true) : map_plane(m, p, rows, K, op.ld, false, box_rows);
  };
  bool ok = mk(&tah, A.hi, A, M, AMN, 128) && mk(&tal, A.lo, A, M, AMN, 128) &&
            mk(&tbh, B.hi, B, N, BMN, BN / 2) && mk(&tbl, B.lo, B, N, BMN, BN / 2);
  H3Args a = a0;
  a.M = M;
  a.N = N;
  a.K = K;
  a.nblocks_m = (int)ceil_div(M, 2 * H3_BM);
  a.nblocks_n = (int)ceil_div(N, BN);
  a.nk = (int)ceil_div(K, H3_BK);
  a.splitk = splitk ? 1 : 0;
  a.ea = A.exp;
  a.eb = B.exp;
  const int tiles = a.nblocks_m * a.nblocks_n;
  // stream-K: all tiles (split 1), or the tiles past the last full wave of
  // H3_VUNITS/2 pairs (split 2), over up to H3_VUNITS virtual units
  a.tiles_dp = split == 2 ? tiles / (H3_VUNITS / 2) * (H3_VUNITS / 2) : 0;
  a.vunits = split == 2 ? std::min(h3_vunits((int64_t)(tiles - a.tiles_dp) * a.nk), H3_VUNITS / 2)
                        : h3_vunits((int64_t)tiles * a.nk);
  // the output map is used by whole tiles only (stream-K writes partials)
  KP_CHECK(a.tiles_dp == 0 || (reinterpret_cast<uintptr_t>(C) % 16 == 0 && ((size_t)ldc * 4) % 16 == 0),
           kErrGeneric, "h3_gemm: whole tiles need a 16-byte aligned output");
  const int tail = tiles - a.tiles_dp;
  const int64_t T = (int64_t)tail * a.nk;
  if (!splitk || a.tiles_dp > 0) ok = ok && map_out(&tcm, C, M, N, ldc);
  if (splitk) {
    KP_CHECK(ws != nullptr, kErrGeneric, "h3_gemm: stream-K needs a workspace");
    ok = ok && map_out(&tpm, ws, (uint64_t)(tail + H3_VUNITS) * 2 * H3_BM, H3_BN, H3_BN);
    if (a.tiles_dp == 0) tcm = tpm;
  } else {
    tpm = tcm;
  }
  if constexpr (GA) {
    // A = rows of ga->src, (m, slot) -> ga->rowocc[m*S + slot]; its planes
    // (A.hi / A.lo) are outputs when ga->store
    KP_CHECK(ga && ga->e % H3_BK == 0 && (uint64_t)ga->S * ga->e == (uint64_t)K && A.exp, kErrGeneric,
             "h3_gemm: gathered A needs K = S*e, e % 32 == 0 and row exponents");
    a.grow = ga->rowocc;
    a.gS = ga->S;
    a.gkps = ga->e / H3_BK;
    a.gstore = ga->store ? 1 : 0;
    ok = ok && map_rows(&tgm, ga->src, ga->nrows, ga->e);
  } else {
    tgm = tah;
  }
  KP_CHECK(ok, kErrCuda, "cuTensorMapEncodeTiled failed (3xFP16 GEMM operands)");
  constexpr uint32_t SMEM = H3Cfg<BN, GA>::SMEM;
  static std::atomic<uint64_t> attr{0};
  int dev = 0;
  KP_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr.load(std::memory_order_acquire) & bit)) {
    KP_CUDA(cudaFuncSetAttribute(k_h3<AMN, BMN, SK, BN, GA, EM>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr.fetch_or(bit, std::memory_order_release);
  }
  const int units_all = std::max(1, h3_units<AMN, BMN, SK, BN, GA, EM>() - (g_h3_reserve + 1) / 2);
  const int work = splitk ? std::max(a.vunits, a.tiles_dp > 0 ? H3_VUNITS / 2 : 0) : tiles;
  const unsigned grid = (unsigned)std::min(work, units_all) * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(H3_WARPS * 32, 1, 1);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KP_CUDA(cudaLaunchKernelEx(&cfg, k_h3<AMN, BMN, SK, BN, GA, EM>, tah, tal, tbh, tbl, tcm, tpm, tgm, a));
  ::kp::count_launch();
  if (splitk && tail > 0) {
    k_h3_fixup<<<dim3(64, tail), 256, 0, s>>>(ws, a.nblocks_n, a.nk, a.tiles_dp, T, a.vunits, M, N, C, ldc,
                                              a.mode, a.act, a.bias);
    ::kp::count_launch();
  }
}

// ---- plane producers ----------------------------------------------------------
// one warp per row of X [rows][K] (K <= 1024): max |x| -> e = row_exp, planes of x * 2^e
__global__ void k_split_rows(const float* __restrict__ x, int rows, int K, int ld, __half* __restrict__ hi,
                             __half* __restrict__ lo, int* __restrict__ exps) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += (gridDim.x * blockDim.x) >> 5) {
    const float* row = x + (size_t)r * ld;
    float mx = 0.f;
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(row[k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int e = row_exp(mx);
    if (lane == 0) exps[r] = e;
    const float sc = pow2f(e);
    for (int k = 2 * lane; k < K; k += 64) {
      const float x0 = __fmul_rn(row[k], sc), x1 = k + 1 < K ? __fmul_rn(row[k + 1], sc) : 0.f;
      uint32_t h, l;
      split_h2(x0, x1, h, l);
      if (k + 1 < K) {
        *reinterpret_cast<uint32_t*>(hi + (size_t)r * K + k) = h;
        *reinterpret_cast<uint32_t*>(lo + (size_t)r * K + k) = l;
      } else {
        hi[(size_t)r * K + k] = __ushort_as_half((unsigned short)(h & 0xFFFF));
        lo[(size_t)r * K + k] = __ushort_as_half((unsigned short)(l & 0xFFFF));
      }
    }
  }
}

// W [N][K] -> planes of W^T ([K][N]) with one exponent per row of W^T (per
// column k of W): a block owns 32 columns of W, stages the 32 x N tile in
// shared memory (N <= 256), reduces each column's max and writes the
// transposed planes -- the transpose and the per-row split of round 1 in one
// read of W.
__global__ void k_split_t(const float* __restrict__ w, int N, int K, __half* __restrict__ hi,
                          __half* __restrict__ lo, int* __restrict__ exps) {
  __shared__ float tile[256][33];
  __shared__ float cmax[8][32];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  const int k0 = blockIdx.x * 32, k = k0 + tx;
  float mx = 0.f;
  for (int n = ty; n < N; n += 8) {
    const float v = k < K ? w[(size_t)n * K + k] : 0.f;
    tile[n][tx] = v;
    mx = fmaxf(mx, fabsf(v));
  }
  cmax[ty][tx] = mx;
  __syncthreads();
  if (ty == 0) {
    float m = cmax[0][tx];
    for (int i = 1; i < 8; ++i) m = fmaxf(m, cmax[i][tx]);
    cmax[0][tx] = pow2f(row_exp(m));
    if (k < K) exps[k] = row_exp(m);
  }
  __syncthreads();
  // row kk of W^T = column k0 + kk of W: consecutive threads take consecutive n
  for (int kk = ty; kk < 32; kk += 8) {
    const int kr = k0 + kk;
    if (kr >= K) break;
    const float sc = cmax[0][kk];
    for (int n2 = 2 * tx; n2 < N; n2 += 64) {
      const float x0 = __fmul_rn(tile[n2][kk], sc), x1 = n2 + 1 < N ? __fmul_rn(tile[n2 + 1][kk], sc) : 0.f;
      uint32_t h, l;
      split_h2(x0, x1, h, l);
      if (n2 + 1 < N) {
        *reinterpret_cast<uint32_t*>(hi + (size_t)kr * N + n2) = h;
        *reinterpret_cast<uint32_t*>(lo + (size_t)kr * N + n2) = l;
      } else {
        hi[(size_t)kr * N + n2] = __ushort_as_half((unsigned short)(h & 0xFFFF));
        lo[(size_t)kr * N + n2] = __ushort_as_half((unsigned short)(l & 0xFFFF));
      }
    }
  }
}

// dW's A operand: D[b][o] = dZ[b][o] * 2^-xe[b] (X's row scale moved onto the
// other factor, so the sum over b needs no per-k scale), split with a scale
// per COLUMN o (the GEMM row of dW): pass 1 column maxima, pass 2 planes.
// Layout for both: a thread owns 4 consecutive columns (float4) of a row,
// blockDim.x = N/4 threads span a row, blockDim.y rows per block step.
// (csum, optional: the plain column sums of dz -- the layer's bias gradient --
// as per-block partials [gridDim.x][N] in a fixed order, reduced after)
__global__ void k_colmax_scaled(const float* __restrict__ dz, int B, int N, const int* __restrict__ xe,
                                unsigned* __restrict__ cmax, float* __restrict__ csum) {
  __shared__ float red[1024];  // [blockDim.y][4 * blockDim.x] <= 1024
  const int n4 = blockIdx.y * blockDim.x + threadIdx.x;  // column quad (slab blockIdx.y)
  const bool in = n4 < N / 4;
  float4 mx = make_float4(0.f, 0.f, 0.f, 0.f), sm = mx;
  for (int b = blockIdx.x * blockDim.y + threadIdx.y; in && b < B; b += gridDim.x * blockDim.y) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(dz + (size_t)b * N) + n4);
    const float xs = xe ? pow2f(-__ldg(xe + b)) : 1.f;
    mx.x = fmaxf(mx.x, fabsf(__fmul_rn(v.x, xs)));
    mx.y = fmaxf(mx.y, fabsf(__fmul_rn(v.y, xs)));
    mx.z = fmaxf(mx.z, fabsf(__fmul_rn(v.z, xs)));
    mx.w = fmaxf(mx.w, fabsf(__fmul_rn(v.w, xs)));
    sm.x = __fadd_rn(sm.x, v.x), sm.y = __fadd_rn(sm.y, v.y);
    sm.z = __fadd_rn(sm.z, v.z), sm.w = __fadd_rn(sm.w, v.w);
  }
  const int W = 4 * blockDim.x;  // slab width (columns)
  float* rr = red + threadIdx.y * W + 4 * threadIdx.x;
  rr[0] = mx.x, rr[1] = mx.y, rr[2] = mx.z, rr[3] = mx.w;
  __syncthreads();
  for (int c = threadIdx.y * blockDim.x + threadIdx.x; c < W; c += blockDim.x * blockDim.y) {
    float m = 0.f;
    for (int r = 0; r < (int)blockDim.y; ++r) m = fmaxf(m, red[r * W + c]);
    const int col = blockIdx.y * W + c;
    if (m > 0.f && col < N) atomicMax(cmax + col, __float_as_uint(m));
  }
  if (!csum) return;
  __syncthreads();
  rr[0] = sm.x, rr[1] = sm.y, rr[2] = sm.z, rr[3] = sm.w;
  __syncthreads();
  for (int c = threadIdx.y * blockDim.x + threadIdx.x; c < W; c += blockDim.x * blockDim.y) {
    float t = 0.f;
    for (int r = 0; r < (int)blockDim.y; ++r) t = __fadd_rn(t, red[r * W + c]);  // rows in y order
    const int col = blockIdx.y * W + c;
    if (col < N) csum[(size_t)blockIdx.x * N + col] = t;
  }
}

__device__ __forceinline__ void sum_parts_warp(const float* __restrict__ part, int nparts, int N, int n, int lane,
                                               float* __restrict__ out) {
  float v = 0.f;
  for (int c = lane; c < nparts; c += 32) v = __fadd_rn(v, part[(size_t)c * N + n]);
#pragma unroll
  for (int o = 16; o; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) out[n] = v;
}

// k_split_rows (dX's A operand) and k_colmax_scaled (dW's column scales and
// the bias-gradient partials) from ONE read of dz, for N % 128 == 0, N <= 1024
// (one slab; a row spans N/128 whole warps): the colmax layout and row order,
// the row max through shared memory. Bit for bit the two kernels' outputs.
__global__ void k_rows_colmax(const float* __restrict__ dz, int B, int N, const int* __restrict__ xe,
                              unsigned* __restrict__ cmax, float* __restrict__ csum, __half* __restrict__ rhi,
                              __half* __restrict__ rlo, int* __restrict__ rexps) {
  constexpr int RU = 4;  // rows in flight per thread (one barrier per RU rows)
  __shared__ float red[1024];
  __shared__ float rm[2][RU][8][8];  // [iteration parity][row u][row ty][warp of the row]
  const int n4 = threadIdx.x, lane = threadIdx.x & 31, wr = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int step = gridDim.x * blockDim.y;
  float4 mx = make_float4(0.f, 0.f, 0.f, 0.f), sm = mx;
  int it = 0;
  for (int b0 = blockIdx.x * blockDim.y; b0 < B; b0 += RU * step, ++it) {  // block-uniform
    float4 v[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int b = b0 + u * step + threadIdx.y;
      v[u] = b < B ? __ldg(reinterpret_cast<const float4*>(dz + (size_t)b * N) + n4)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      float m = fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w)));
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) rm[it & 1][u][threadIdx.y][wr] = m;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < RU; ++u) {  // rows in the colmax kernel's order (b ascending)
      const int b = b0 + u * step + threadIdx.y;
      if (b >= B) break;
      float r = rm[it & 1][u][threadIdx.y][0];
      for (int i = 1; i < nw; ++i) r = fmaxf(r, rm[it & 1][u][threadIdx.y][i]);
      const int e = row_exp(r);
      if (n4 == 0) rexps[b] = e;
      const float sc = pow2f(e);
      uint2 h, l;
      split_h2(__fmul_rn(v[u].x, sc), __fmul_rn(v[u].y, sc), h.x, l.x);
      split_h2(__fmul_rn(v[u].z, sc), __fmul_rn(v[u].w, sc), h.y, l.y);
      reinterpret_cast<uint2*>(rhi + (size_t)b * N)[n4] = h;
      reinterpret_cast<uint2*>(rlo + (size_t)b * N)[n4] = l;
      const float xs = xe ? pow2f(-__ldg(xe + b)) : 1.f;
      mx.x = fmaxf(mx.x, fabsf(__fmul_rn(v[u].x, xs)));
      mx.y = fmaxf(mx.y, fabsf(__fmul_rn(v[u].y, xs)));
      mx.z = fmaxf(mx.z, fabsf(__fmul_rn(v[u].z, xs)));
      mx.w = fmaxf(mx.w, fabsf(__fmul_rn(v[u].w, xs)));
      sm.x = __fadd_rn(sm.x, v[u].x), sm.y = __fadd_rn(sm.y, v[u].y);
      sm.z = __fadd_rn(sm.z, v[u].z), sm.w = __fadd_rn(sm.w, v[u].w);
    }
  }
  const int W = 4 * blockDim.x;
  float* rr = red + threadIdx.y * W + 4 * threadIdx.x;
  rr[0] = mx.x, rr[1] = mx.y, rr[2] = mx.z, rr[3] = mx.w;
  __syncthreads();
  for (int c = threadIdx.y * blockDim.x + threadIdx.x; c < W; c += blockDim.x * blockDim.y) {
    float mm = 0.f;
    for (int q = 0; q < (int)blockDim.y; ++q) mm = fmaxf(mm, red[q * W + c]);
    if (mm > 0.f) atomicMax(cmax + c, __float_as_uint(mm));
  }
  if (!csum) return;
  __syncthreads();
  rr[0] = sm.x, rr[1] = sm.y, rr[2] = sm.z, rr[3] = sm.w;
  __syncthreads();
  for (int c = threadIdx.y * blockDim.x + threadIdx.x; c < W; c += blockDim.x * blockDim.y) {
    float t = 0.f;
    for (int q = 0; q < (int)blockDim.y; ++q) t = __fadd_rn(t, red[q * W + c]);  // rows in y order
    csum[(size_t)blockIdx.x * N + c] = t;
  }
}

// out[n] = sum over the per-block partials in block order (deterministic)
__global__ void k_sum_parts(const float* __restrict__ part, int nparts, int N, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < N; n += (gridDim.x * blockDim.x) >> 5)
    sum_parts_warp(part, nparts, N, n, lane, out);
}
// (part/sum_out, optional: k_sum_parts folded in -- the warps of the first
// slab's blocks reduce the colsum partials, same order, bit for bit)
__global__ void k_split_cols_scaled(const float* __restrict__ dz, int B, int N, const int* __restrict__ xe,
                                    const unsigned* __restrict__ cmax, __half* __restrict__ hi,
                                    __half* __restrict__ lo, int* __restrict__ exps,
                                    const float* __restrict__ part = nullptr, int nparts = 0,
                                    float* __restrict__ sum_out = nullptr) {
  if (sum_out && blockIdx.y == 0) {
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, wpb = (blockDim.x * blockDim.y) >> 5;
    for (int n = blockIdx.x * wpb + (tid >> 5); n < N; n += gridDim.x * wpb)
      sum_parts_warp(part, nparts, N, n, tid & 31, sum_out);
  }
  const int n4 = blockIdx.y * blockDim.x + threadIdx.x;
  if (n4 >= N / 4) return;
  int ex[4];
  float sc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    ex[j] = row_exp(__uint_as_float(cmax[4 * n4 + j]));
    sc[j] = pow2f(ex[j]);
  }
  if (blockIdx.x == 0 && threadIdx.y == 0)
#pragma unroll
    for (int j = 0; j < 4; ++j) exps[4 * n4 + j] = ex[j];
  for (int b = blockIdx.x * blockDim.y + threadIdx.y; b < B; b += gridDim.x * blockDim.y) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(dz + (size_t)b * N) + n4);
    const float xs = xe ? pow2f(-__ldg(xe + b)) : 1.f;
    uint2 h, l;
    split_h2(__fmul_rn(__fmul_rn(v.x, xs), sc[0]), __fmul_rn(__fmul_rn(v.y, xs), sc[1]), h.x, l.x);
    split_h2(__fmul_rn(__fmul_rn(v.z, xs), sc[2]), __fmul_rn(__fmul_rn(v.w, xs), sc[3]), h.y, l.y);
    reinterpret_cast<uint2*>(hi + (size_t)b * N)[n4] = h;
    reinterpret_cast<uint2*>(lo + (size_t)b * N)[n4] = l;
  }
}

}  // namespace

void h3_reserve_sms(int n) { g_h3_reserve = n < 0 ? 0 : n; }

bool h3_enabled() {
  static const bool on = [] {
    const char* e = getenv("KP_GEMM_H3");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool h3_supported(int M, int N, int K, const H3Operand& A, const H3Operand& B) {
  if (M <= 0 || N <= 0 || K <= 0 || !encode_fn()) return false;
  for (const H3Operand* o : {&A, &B}) {
    if ((o->ld * 2) % 16) return false;
    if (reinterpret_cast<uintptr_t>(o->hi) % 16 || reinterpret_cast<uintptr_t>(o->lo) % 16) return false;
  }
  return true;
}

// C[m][n] = epi(sum_k A(m,k) B(n,k)); A/B K-major ([rows][K]) unless *_mn
void h3_gemm(const H3Operand& A, bool a_mn, const H3Operand& B, bool b_mn, int M, int N, int K, float* C,
             int ldc, const GemmEpi& ep, int splitk, float* ws, cudaStream_t s, int keep, const H3Gather* ga) {
  H3Args a{};
  static const int dbg = [] {
    const char* e = getenv("KP_H3_DBG");
    return e ? atoi(e) : 0;
  }();
  a.dbg = dbg;
  a.keep_a = keep & 1;
  a.keep_b = (keep >> 1) & 1;
  a.mode = ep.mode;
  a.act = ep.act;
  a.bias = ep.bias;
  a.coeff = ep.coeff;
  a.S = ep.S;
  a.e = ep.e;
  KP_CHECK(ep.mode == 0 || ep.mode == 1 || ep.mode == 3, kErrGeneric, "h3_gemm: unsupported epilogue");
  KP_CHECK(splitk == 0 || ep.mode != 3, kErrGeneric, "h3_gemm: stream-K fix-up has no coefficient epilogue");
  KP_CHECK(!ga || !a_mn, kErrGeneric, "h3_gemm: gathered A is K-major");
  KP_CHECK(a_mn == b_mn, kErrGeneric, "h3_gemm: both operands K-major or both MN-major");
  if (!a_mn) launch_h3<false, false>(A, B, M, N, K, C, ldc, splitk, ws, a, s, ga);
  else launch_h3<true, true>(A, B, M, N, K, C, ldc, splitk, ws, a, s);
}

size_t split_cols_colsum_ws_floats(int B, int N) {
  const int W = std::min(N, 1024);
  const int by = std::max(1, std::min(8, 256 / (W / 4)));
  return (size_t)std::min<uint64_t>(ceil_div(B, by), std::max<uint64_t>(1, 148 * 8 / ceil_div(N, W))) * N;
}

size_t h3_splitk_ws_floats(int M, int N, bool tail_only) {
  size_t tiles = ceil_div(M, 2 * H3_BM) * ceil_div(N, H3_BN);
  if (tail_only) tiles = std::min<size_t>(tiles, H3_VUNITS / 2);
  return (tiles + H3_VUNITS) * 2 * H3_BM * H3_BN;
}

void split_t_h(const float* W, int N, int K, __half* hi, __half* lo, int* exps, cudaStream_t s) {
  KP_CHECK(N <= 256 && N % 2 == 0, kErrConfig, "split_t_h: N must be even and <= 256");
  k_split_t<<<ceil_div(K, 32), 256, 0, s>>>(W, N, K, hi, lo, exps);
  ::kp::count_launch();
}

void split_rows_h(const float* X, int rows, int K, int ld, __half* hi, __half* lo, int* exps, cudaStream_t s) {
  k_split_rows<<<std::min<unsigned>(ceil_div((uint64_t)rows * 32, 256), 148 * 16), 256, 0, s>>>(X, rows, K, ld, hi,
                                                                                                lo, exps);
  ::kp::count_launch();
}

static dim3 cols_block(int N) {
  const int W = std::min(N, 1024);
  return dim3(W / 4, std::max(1, std::min(8, 256 / (W / 4))));
}
static dim3 cols_grid(int B, int N, dim3 blk) {
  const int W = std::min(N, 1024);
  const unsigned slabs = ceil_div(N, W);
  return dim3((unsigned)std::min<uint64_t>(ceil_div(B, blk.y), std::max<uint64_t>(1, 148 * 8 / slabs)), slabs);
}

bool rows_colmax_fusable(int N) {
  const char* e = getenv("KP_SPLIT_FUSE");  // (per call: tests toggle it)
  return !(e && e[0] == '0') && N % 128 == 0 && N <= 1024;
}

void split_rows_colmax_h(const float* dz, int B, int N, const int* xe, unsigned* cmax_ws, __half* rhi,
                         __half* rlo, int* rexps, float* colsum_ws, cudaStream_t s) {
  KP_CHECK(rows_colmax_fusable(N), kErrConfig, "split_rows_colmax_h: N must be a multiple of 128, <= 1024");
  KP_CUDA(cudaMemsetAsync(cmax_ws, 0, (size_t)N * 4, s));
  const dim3 blk = cols_block(N), g = cols_grid(B, N, blk);
  k_rows_colmax<<<g, blk, 0, s>>>(dz, B, N, xe, cmax_ws, colsum_ws, rhi, rlo, rexps);
  ::kp::count_launch();
}

void split_cols_after_h(const float* dz, int B, int N, const int* xe, const unsigned* cmax_ws, __half* hi, __half* lo,
                        int* exps, float* colsum_out, const float* colsum_ws, cudaStream_t s) {
  const dim3 blk = cols_block(N), g = cols_grid(B, N, blk);
  k_split_cols_scaled<<<g, blk, 0, s>>>(dz, B, N, xe, cmax_ws, hi, lo, exps, colsum_ws, (int)g.x,
                                        colsum_out);
  ::kp::count_launch();
}

void split_cols_scaled_h(const float* dz, int B, int N, const int* xe, unsigned* cmax_ws, __half* hi, __half* lo,
                         int* exps, cudaStream_t s, float* colsum_out, float* colsum_ws) {
  KP_CHECK(N % 4 == 0, kErrConfig, "split_cols_scaled_h: N must be a multiple of 4");
  KP_CUDA(cudaMemsetAsync(cmax_ws, 0, (size_t)N * 4, s));
  // slabs of up to 1024 columns (blockIdx.y), rows strided over blockIdx.x
  const int W = std::min(N, 1024);
  const dim3 blk(W / 4, std::max(1, std::min(8, 256 / (W / 4))));
  const unsigned slabs = ceil_div(N, W);
  const dim3 g((unsigned)std::min<uint64_t>(ceil_div(B, blk.y), std::max<uint64_t>(1, 148 * 8 / slabs)), slabs);
  k_colmax_scaled<<<g, blk, 0, s>>>(dz, B, N, xe, cmax_ws, colsum_out ? colsum_ws : nullptr);
  ::kp::count_launch();
  if (colsum_out) {
    k_sum_parts<<<std::min<unsigned>(ceil_div((uint64_t)N * 32, 256), 148 * 16), 256, 0, s>>>(colsum_ws, (int)g.x, N,
                                                                                          colsum_out);
    ::kp::count_launch();
  }
  k_split_cols_scaled<<<g, blk, 0, s>>>(dz, B, N, xe, cmax_ws, hi, lo, exps);
  ::kp::count_launch();
}

}  // namespace kp
