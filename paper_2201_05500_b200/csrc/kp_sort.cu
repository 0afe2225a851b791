// Key dedup for the working set: LSD radix sort of (key, occurrence) pairs,
// then unique + inverse index + segment starts; and the key % G owner bucket.
//
// Replaces the reference's std::set working-set build
// (proj/src/trainer.cpp:121-124) and the per-key owner map
// (proj/src/trainer.cpp:83). Output order is ascending key -- bit-identical to
// std::set iteration order.
//
// Design (HBM-bound integer work, no tensor cores):
//  * only the bits where keys differ are sorted: digits of (key - min), so a
//    100M key space costs 4 passes of 8 bits, not 8;
//  * per pass: upsweep histogram (warp-aggregated smem atomics), per-digit
//    scan, downsweep with a stable block rank (ballot digit match) and a
//    shared-memory staged scatter so global writes are digit-run coalesced;
//  * tiles of 2048 pairs (256 threads x 8), grids are multiples of the SM
//    count for every config that matters.
#include <cstdlib>
#include <vector>

#include <type_traits>

#include "kp_internal.cuh"

namespace kp {
namespace {

constexpr int ST = 256;              // threads per sort block
constexpr int IPT = 8;               // items per thread
constexpr int TILE = ST * IPT;       // 2048
constexpr int RADIX = 256;
constexpr int NW = ST / 32;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of one value per thread (256 threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  uint32_t wpre = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t t = s_warp[w];
    if (w < warp) wpre += t;
    total += t;
  }
  __syncthreads();
  return wpre + x - v;
}

__global__ void k_minmax_init(unsigned long long* mm) {
  mm[0] = ~0ull;
  mm[1] = 0ull;
}

__global__ void k_minmax(const uint64_t* __restrict__ keys, uint32_t n, unsigned long long* mm) {
  uint64_t lo = ~0ull, hi = 0;
  // 4 x 16-byte loads in flight per thread; an 8-byte-aligned start peels
  // its first key
  const uint32_t peel = (reinterpret_cast<uintptr_t>(keys) & 15) ? 1u : 0u;
  if (peel && n && blockIdx.x == 0 && threadIdx.x == 0) lo = hi = keys[0];
  keys += peel;
  n = n > peel ? n - peel : 0;
  const uint32_t n2 = n / 2;
  const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys);
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    ulonglong2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(k2 + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      lo = min(lo, (uint64_t)min(v[u].x, v[u].y));
      hi = max(hi, (uint64_t)max(v[u].x, v[u].y));
    }
  }
  for (; i < n2; i += stride) {
    const ulonglong2 v = __ldg(k2 + i);
    lo = min(lo, (uint64_t)min(v.x, v.y));
    hi = max(hi, (uint64_t)max(v.x, v.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    lo = min(lo, keys[n - 1]);
    hi = max(hi, keys[n - 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o);
    const uint64_t b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  // block reduce, then one atomic pair per block (per-warp atomics on the
  // same two words serialised at L2)
  __shared__ uint64_t s_lo[32], s_hi[32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) s_lo[w] = lo, s_hi[w] = hi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < nw; ++j) lo = min(lo, s_lo[j]), hi = max(hi, s_hi[j]);
    atomicMin(&mm[0], (unsigned long long)lo);
    atomicMax(&mm[1], (unsigned long long)hi);
  }
}

// digit of an input key: (key - kmin) >> shift for raw u64 keys, key >> shift
// for u32 keys that already are (key - kmin)
template <typename KIN>
__device__ __forceinline__ uint32_t digit_of(KIN k, uint64_t kmin, int shift, uint32_t mask) {
  if constexpr (sizeof(KIN) == 4) return (uint32_t)(k >> shift) & mask;
  else return (uint32_t)((k - kmin) >> shift) & mask;
}

// lanes holding the same digit d in [0, R] (R = invalid): one ballot per
// digit bit instead of MATCH.ANY (which issues through the MIO queue and
// dominated the rank loop's stalls)
// (full: no lane holds R -- a full tile -- so the validity bit is skipped)
template <int R>
__device__ __forceinline__ uint32_t match_digit(uint32_t d, bool full = false) {
  constexpr int BITS = R == 256 ? 8 : R == 512 ? 9 : R == 1024 ? 10 : 16;
  uint32_t peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool on = (d >> b) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, on);
    peers &= on ? bal : ~bal;
  }
  if (!full) {
    const bool on = (d >> BITS) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, on);
    peers &= on ? bal : ~bal;
  }
  return peers;
}

template <typename KIN, int R>
__global__ void __launch_bounds__(ST) k_upsweep(const KIN* __restrict__ keys, uint32_t n,
                                                const unsigned long long* __restrict__ mm,
                                                int shift, uint32_t* __restrict__ counts,
                                                uint32_t nb) {
  __shared__ uint32_t hist[R];
  for (int i = threadIdx.x; i < R; i += ST) hist[i] = 0;
  __syncthreads();
  const uint64_t kmin = mm[0];
  const uint32_t base = blockIdx.x * TILE;
  // counts only (no ranks): one shared-memory atomic per item; integer adds,
  // so the histogram is exact whatever order they land in
  uint32_t d[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t idx = base + r * ST + threadIdx.x;
    d[r] = idx < n ? digit_of<KIN>(keys[idx], kmin, shift, R - 1) : R;
  }
#pragma unroll
  for (int r = 0; r < IPT; ++r)
    if (d[r] < R) atomicAdd(&hist[d[r]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < R; i += ST) counts[i * nb + blockIdx.x] = hist[i];
}

// rows of `counts` ([rows][nb]) scanned exclusive in place; totals[row].
__global__ void __launch_bounds__(ST) k_scan_rows(uint32_t* __restrict__ counts, uint32_t nb,
                                                  uint32_t* __restrict__ totals) {
  __shared__ uint32_t s_warp[NW];
  uint32_t* row = counts + (size_t)blockIdx.x * nb;
  uint32_t running = 0;
  for (uint32_t base = 0; base < nb; base += ST * 4) {
    uint32_t v[4], sum = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t j = base + threadIdx.x * 4 + i;
      v[i] = j < nb ? row[j] : 0;
      sum += v[i];
    }
    uint32_t total;
    uint32_t pre = block_excl_scan(sum, s_warp, total) + running;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t j = base + threadIdx.x * 4 + i;
      if (j < nb) row[j] = pre;
      pre += v[i];
    }
    running += total;
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = running;
}

// Stable rank of the tile's items within their digit. Items are striped:
// item r of thread t is tile element r*ST + t, so processing rounds r in
// order, warps in order, lanes in order is element order. d == R: invalid.
template <int R>
__device__ __forceinline__ void stable_rank(const uint32_t (&d)[IPT], uint32_t (&rank)[IPT],
                                            uint32_t* s_run, uint16_t (*s_wcnt)[NW][R]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int buf = r & 1;
    const uint32_t peers = __match_any_sync(0xffffffffu, d[r]);
    const bool leader = lane == __ffs(peers) - 1;
    const uint32_t cnt = __popc(peers);
    const uint32_t rw = __popc(peers & lt);
    if (leader && d[r] < R) s_wcnt[buf][warp][d[r]] = (uint16_t)cnt;
    __syncthreads();
    if (d[r] < R) {
      uint32_t pre = s_run[d[r]];
      for (int w = 0; w < warp; ++w) pre += s_wcnt[buf][w][d[r]];
      rank[r] = pre + rw;
    }
    __syncthreads();
    if (leader && d[r] < R) {
      atomicAdd(&s_run[d[r]], cnt);
      s_wcnt[buf][warp][d[r]] = 0;
    }
  }
  __syncthreads();
}

// exclusive scan of R (256 or 512) values held as RPT consecutive values per thread
template <int R>
__device__ __forceinline__ void scan_digits(const uint32_t* in, uint32_t* out, uint32_t* s_warp) {
  constexpr int RPT = R / ST;
  uint32_t v[RPT], sum = 0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    v[i] = in[threadIdx.x * RPT + i];
    sum += v[i];
  }
  uint32_t tot;
  uint32_t pre = block_excl_scan(sum, s_warp, tot);
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    out[threadIdx.x * RPT + i] = pre;
    pre += v[i];
  }
}

// One LSD pass. KIN -> KOUT: u64 -> u64 (raw keys), u64 -> u32 (first pass of
// the narrow mode: keys become key - kmin), u32 -> u32.
template <typename KIN, typename KOUT, int R>
__global__ void __launch_bounds__(ST, 4) k_downsweep(
    const KIN* __restrict__ kin, const uint32_t* __restrict__ vin, KOUT* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, const unsigned long long* __restrict__ mm, int shift,
    const uint32_t* __restrict__ counts, const uint32_t* __restrict__ totals, uint32_t nb) {
  // Warp-striped items (warp w owns tile elements [w*IPT*32, (w+1)*IPT*32),
  // round r lane l -> w*IPT*32 + r*32 + l): element order = (warp, round,
  // lane), so a warp-local running count per digit gives a stable rank with
  // no block barrier per round; one scan over the [warp][digit] counts in
  // (digit, warp) order then turns (digit, warp, rank-in-warp) into the tile
  // position. (Warp-major rows: a warp's lanes hit banks by digit, and the
  // scan reads each digit's column with consecutive threads -- the digit-major
  // layout had 8- and 16-way bank conflicts in those two places.)
  __shared__ KOUT s_keys[TILE];
  __shared__ uint32_t s_vals[TILE];
  // [warp][digit] counts -> exclusive tile positions (both <= TILE: 16 bits
  // suffice, which keeps the 1024-digit table inside the static 48 KB)
  using WT = std::conditional_t<(R > 512), uint16_t, uint32_t>;
  __shared__ __align__(16) WT s_wh[NW * R];
  __shared__ uint32_t s_start[R], s_off[R];
  __shared__ uint32_t s_warp[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < R * NW; i += ST) s_wh[i] = 0;
  __syncthreads();
  const uint64_t kmin = mm[0];
  const uint32_t base = blockIdx.x * TILE;
  const uint32_t tile_n = min((uint32_t)TILE, n - base);
  const bool full = tile_n == (uint32_t)TILE;
  const uint32_t lt = lanemask_lt();
  KOUT k[IPT];
  uint32_t v[IPT], d[IPT], rw[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t i = (uint32_t)warp * (IPT * 32) + r * 32 + lane;
    if (i < tile_n) {
      const KIN x = kin[base + i];
      d[r] = digit_of<KIN>(x, kmin, shift, R - 1);
      if constexpr (sizeof(KOUT) == 4 && sizeof(KIN) == 8) k[r] = (KOUT)(x - kmin);
      else k[r] = (KOUT)x;
      v[r] = vin ? vin[base + i] : base + i;
    } else {
      d[r] = R;
    }
  }
  WT* wrow = s_wh + warp * R;
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t peers = match_digit<R>(d[r], full);
    const bool leader = lane == __ffs(peers) - 1;
    uint32_t before = 0;
    if (d[r] < R) before = wrow[d[r]];
    __syncwarp();
    if (d[r] < R) {
      rw[r] = before + __popc(peers & lt);
      if (leader) wrow[d[r]] = (WT)(before + __popc(peers));
    }
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan in (digit, warp) order: thread t owns digits [t*DPT, +DPT);
  // the column is read twice (sums, then positions) instead of held
  if constexpr (R / ST == 4) {
    // 1024 digits (16-bit entries)
    uint32_t tt[4] = {0, 0, 0, 0};
#pragma unroll
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int j = 0; j < 4; ++j) tt[j] += s_wh[w * R + 4 * tid + j];
    uint32_t tot;
    uint32_t p[4];
    p[0] = block_excl_scan(tt[0] + tt[1] + tt[2] + tt[3], s_warp, tot);
    p[1] = p[0] + tt[0];
    p[2] = p[1] + tt[1];
    p[3] = p[2] + tt[2];
#pragma unroll
    for (int j = 0; j < 4; ++j) s_start[tid * 4 + j] = p[j];  // first tile position of the digit
#pragma unroll
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = s_wh[w * R + 4 * tid + j];
        s_wh[w * R + 4 * tid + j] = (WT)p[j];
        p[j] += x;
      }
  } else {
    constexpr int DPT = R / ST;
    static_assert(DPT == 1 || DPT == 2, "256, 512 or 1024 digits");
    uint32_t t0 = 0, t1 = 0;  // the owned digits' totals
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if constexpr (DPT == 2) {
        const uint2 x = *reinterpret_cast<const uint2*>(s_wh + w * R + 2 * tid);
        t0 += x.x;
        t1 += x.y;
      } else {
        t0 += s_wh[w * R + tid];
      }
    }
    uint32_t tot;
    uint32_t p0 = block_excl_scan(t0 + t1, s_warp, tot), p1 = p0 + t0;
    s_start[tid * DPT] = p0;  // first tile position of the digit
    if constexpr (DPT == 2) s_start[tid * DPT + 1] = p1;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if constexpr (DPT == 2) {
        uint2* q = reinterpret_cast<uint2*>(s_wh + w * R + 2 * tid);
        const uint2 x = *q;
        *q = make_uint2(p0, p1);
        p0 += x.x;
        p1 += x.y;
      } else {
        const uint32_t x = s_wh[w * R + tid];
        s_wh[w * R + tid] = p0;
        p0 += x;
      }
    }
  }
  for (int i = tid; i < R; i += ST) s_off[i] = totals[i];
  __syncthreads();
  scan_digits<R>(s_off, s_off, s_warp);  // global digit starts (in place: values read first)
  __syncthreads();
  for (int i = tid; i < R; i += ST) s_off[i] += counts[i * nb + blockIdx.x] - s_start[i];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    if (d[r] < R) {
      const uint32_t p = wrow[d[r]] + rw[r];
      s_keys[p] = k[r];
      s_vals[p] = v[r];
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < tile_n; i += ST) {
    const KOUT key = s_keys[i];
    const uint32_t dd = digit_of<KOUT>(key, kmin, shift, R - 1);
    const uint32_t g = s_off[dd] + i;
    kout[g] = key;
    vout[g] = s_vals[i];
  }
}

// ---- unique / inverse / segments -----------------------------------------
template <typename KT>
__global__ void __launch_bounds__(ST) k_head_count(const KT* __restrict__ sk, uint32_t n,
                                                   uint32_t* __restrict__ bcount) {
  __shared__ uint32_t s_warp[NW];
  const uint32_t base = blockIdx.x * TILE + threadIdx.x * IPT;
  KT kv[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) kv[r] = base + r < n ? sk[base + r] : KT(0);
  const KT prev = base > 0 && base - 1 < n ? sk[base - 1] : KT(0);
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t i = base + r;
    if (i < n && (i == 0 || kv[r] != (r ? kv[r - 1] : prev))) ++c;
  }
  uint32_t tot;
  block_excl_scan(c, s_warp, tot);
  if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

template <typename KT>
__global__ void __launch_bounds__(ST) k_dedup_emit(const KT* __restrict__ sk,
                                                   const unsigned long long* __restrict__ mm,
                                                   const uint32_t* __restrict__ sv, uint32_t n,
                                                   const uint32_t* __restrict__ bbase,
                                                   uint64_t* __restrict__ uniq,
                                                   uint32_t* __restrict__ inverse,
                                                   uint32_t* __restrict__ seg,
                                                   uint32_t* __restrict__ nuniq, uint32_t nb,
                                                   const uint32_t* __restrict__ occ_map,
                                                   uint32_t* __restrict__ sorted_mapped,
                                                   const uint32_t* __restrict__ occ_ident) {
  __shared__ uint32_t s_warp[NW];
  const uint32_t base = blockIdx.x * TILE + threadIdx.x * IPT;
  // every load first (keys, the predecessor key, occurrences, then the
  // occ_map gathers), so one latency covers the thread's IPT positions
  KT kv[IPT];
  uint32_t occ[IPT], mp[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) kv[r] = base + r < n ? sk[base + r] : KT(0);
  const KT prev = base > 0 && base - 1 < n ? sk[base - 1] : KT(0);
#pragma unroll
  for (int r = 0; r < IPT; ++r) occ[r] = base + r < n ? sv[base + r] : 0;
  bool f[IPT];
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t i = base + r;
    f[r] = i < n && (i == 0 || kv[r] != (r ? kv[r - 1] : prev));
    c += f[r];
  }
  // identity map (one feature per slot): the bag IS the occurrence, no gather
  const bool ident = occ_ident && *occ_ident == 0xFFFFFFFFu;
  if (occ_map) {
#pragma unroll
    for (int r = 0; r < IPT; ++r) mp[r] = base + r < n ? (ident ? occ[r] : occ_map[occ[r]]) : 0;
  }
  uint32_t tot;
  uint32_t uid = bbase[blockIdx.x] + block_excl_scan(c, s_warp, tot);  // uniques before my items
  const uint64_t kmin = sizeof(KT) == 4 ? (uint64_t)mm[0] : 0;
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t i = base + r;
    if (i >= n) break;
    if (f[r]) {
      uniq[uid] = kmin + (uint64_t)kv[r];
      seg[uid] = i;
      ++uid;
    }
    inverse[occ[r]] = uid - 1;
    if (occ_map && !ident) sorted_mapped[i] = mp[r];  // e.g. bag of each sorted position (identity: = sv)
  }
  if (blockIdx.x == nb - 1 && threadIdx.x == 0) {
    const uint32_t U = bbase[blockIdx.x] + tot;
    seg[U] = n;
    *nuniq = U;
  }
}

// ---- owner bucket (key % G) ---------------------------------------------
constexpr int MAXG = 64;

__global__ void __launch_bounds__(ST) k_shard_count(const uint64_t* __restrict__ keys, uint32_t n,
                                                    uint32_t G, uint32_t* __restrict__ counts,
                                                    uint32_t nb, const uint32_t* __restrict__ dn) {
  if (dn) n = min(n, *dn);  // (the key count on the device, n its bound)
  __shared__ uint32_t hist[MAXG];
  if (threadIdx.x < MAXG) hist[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * TILE;
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t i = base + r * ST + threadIdx.x;
    if (i < n) atomicAdd(&hist[keys[i] % G], 1u);
  }
  __syncthreads();
  if (threadIdx.x < G) counts[threadIdx.x * nb + blockIdx.x] = hist[threadIdx.x];
}

__global__ void __launch_bounds__(ST) k_shard_emit(const uint64_t* __restrict__ keys, uint32_t n,
                                                   uint32_t G, const uint32_t* __restrict__ counts,
                                                   const uint32_t* __restrict__ totals,
                                                   uint32_t nb, uint32_t* __restrict__ perm,
                                                   uint32_t* __restrict__ pos, const uint32_t* __restrict__ dn) {
  if (dn) n = min(n, *dn);
  __shared__ uint32_t s_off[MAXG], s_run[MAXG];
  __shared__ uint16_t s_wcnt[2][NW][MAXG];
  const int tid = threadIdx.x;
  if (tid < MAXG) {
    s_run[tid] = 0;
    uint32_t pre = 0;
    for (uint32_t g = 0; g < (uint32_t)tid && g < G; ++g) pre += totals[g];
    s_off[tid] = tid < (int)G ? pre + counts[tid * nb + blockIdx.x] : 0;
  }
  for (int i = tid; i < 2 * NW * MAXG; i += ST) (&s_wcnt[0][0][0])[i] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * TILE;
  uint32_t d[IPT], rank[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t i = base + r * ST + tid;
    d[r] = i < n ? (uint32_t)(keys[i] % G) : MAXG;
  }
  stable_rank<MAXG>(d, rank, s_run, s_wcnt);
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t i = base + r * ST + tid;
    if (i < n) {
      const uint32_t p = s_off[d[r]] + rank[r];
      perm[p] = i;
      pos[i] = p;
    }
  }
}

__global__ void k_key_iota(uint32_t* __restrict__ v, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

// ---- merge of sorted runs (owner side of the exchange) --------------------
// Up to kMaxRuns pairs per level; block b -> (pair, output tile) through the
// per-pair tile prefix. A wins ties (stable: lower source first).
constexpr int kMaxRuns = 64;
struct MergeLevel {
  int pairs;
  uint32_t a0[kMaxRuns / 2], na[kMaxRuns / 2], nb[kMaxRuns / 2];  // A = [a0, a0+na), B follows
  uint32_t tile0[kMaxRuns / 2 + 1];                               // first block of each pair
};

__device__ __forceinline__ uint32_t merge_path(const uint64_t* A, uint32_t na, const uint64_t* B,
                                               uint32_t nb, uint32_t d) {
  uint32_t lo = d > nb ? d - nb : 0, hi = min(d, na);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(ST) k_merge_level(const uint64_t* __restrict__ kin,
                                                    const uint32_t* __restrict__ vin,
                                                    uint64_t* __restrict__ kout,
                                                    uint32_t* __restrict__ vout, MergeLevel L) {
  __shared__ uint64_t sk[TILE];
  __shared__ uint32_t sv[TILE];
  __shared__ uint32_t s_split[2];
  int pr = 0;
  while (pr + 1 < L.pairs && blockIdx.x >= L.tile0[pr + 1]) ++pr;
  const uint32_t a0 = L.a0[pr], na = L.na[pr], nb = L.nb[pr];
  const uint64_t* A = kin + a0;
  const uint64_t* B = A + na;
  const uint32_t d0 = (blockIdx.x - L.tile0[pr]) * TILE, d1 = min(na + nb, d0 + TILE);
  if (threadIdx.x < 2) s_split[threadIdx.x] = merge_path(A, na, B, nb, threadIdx.x ? d1 : d0);
  __syncthreads();
  const uint32_t ia0 = s_split[0], ia1 = s_split[1];
  const uint32_t ib0 = d0 - ia0, ib1 = d1 - ia1;
  const uint32_t la = ia1 - ia0, lb = ib1 - ib0;
  for (uint32_t i = threadIdx.x; i < la + lb; i += ST) {
    if (i < la) {
      sk[i] = A[ia0 + i];
      sv[i] = vin ? vin[a0 + ia0 + i] : a0 + ia0 + i;
    } else {
      sk[i] = B[ib0 + i - la];
      sv[i] = vin ? vin[a0 + na + ib0 + i - la] : a0 + na + ib0 + i - la;
    }
  }
  __syncthreads();
  // this thread's IPT outputs: diagonal t*IPT inside the tile
  const uint32_t dt = min(threadIdx.x * IPT, la + lb);
  uint32_t ia = merge_path(sk, la, sk + la, lb, dt), ib = dt - ia;
  uint64_t ok[IPT];
  uint32_t ov[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const bool takeA = ib >= lb || (ia < la && sk[ia] <= sk[la + ib]);
    const uint32_t src = takeA ? ia : la + ib;
    ok[r] = sk[src < la + lb ? src : 0];
    ov[r] = sv[src < la + lb ? src : 0];
    if (takeA) ++ia; else ++ib;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const uint32_t o = threadIdx.x * IPT + r;
    if (o < la + lb) {
      sk[o] = ok[r];
      sv[o] = ov[r];
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < la + lb; i += ST) {
    kout[a0 + d0 + i] = sk[i];
    vout[a0 + d0 + i] = sv[i];
  }
}

}  // namespace

// narrow-mode pass plan for a key span of `bits` bits (<= 32): the fewest
// passes of at most 10-bit digits, digits as even as possible
__host__ __device__ inline void narrow_plan(int bits, int& np, int& db) {
  np = bits == 0 ? 1 : (bits + 9) / 10;
  db = bits == 0 ? 1 : (bits + np - 1) / np;
}

template <int R>
void pass_u64_to_u32(const uint64_t* kin, uint32_t* kout, uint32_t* vout, uint32_t n, const unsigned long long* mm,
                     int shift, uint32_t* counts, uint32_t* totals, uint32_t nb, cudaStream_t s) {
  k_upsweep<uint64_t, R><<<nb, ST, 0, s>>>(kin, n, mm, shift, counts, nb); ::kp::count_launch();
  k_scan_rows<<<R, ST, 0, s>>>(counts, nb, totals); ::kp::count_launch();
  k_downsweep<uint64_t, uint32_t, R><<<nb, ST, 0, s>>>(kin, nullptr, kout, vout, n, mm, shift, counts, totals, nb);
  ::kp::count_launch();
}
template <int R>
void pass_u32(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout, uint32_t n,
              const unsigned long long* mm, int shift, uint32_t* counts, uint32_t* totals, uint32_t nb,
              cudaStream_t s) {
  k_upsweep<uint32_t, R><<<nb, ST, 0, s>>>(kin, n, mm, shift, counts, nb); ::kp::count_launch();
  k_scan_rows<<<R, ST, 0, s>>>(counts, nb, totals); ::kp::count_launch();
  k_downsweep<uint32_t, uint32_t, R><<<nb, ST, 0, s>>>(kin, vin, kout, vout, n, mm, shift, counts, totals, nb);
  ::kp::count_launch();
}

// The radix passes + unique/inverse/segments for a key span of `bits` bits
// (any plan whose passes cover the actual span sorts correctly).
static void dedup_sort(const uint64_t* d_keys, uint32_t n, DedupWs& ws, cudaStream_t s,
                       const uint32_t* d_occ_map, const uint32_t* d_occ_ident, int bits,
                       const unsigned long long* mm, uint32_t nb) {
  uint32_t* va = ws.vals_a.get<uint32_t>(n);
  uint32_t* vb = ws.vals_b.get<uint32_t>(n);
  uint32_t* bcount = ws.bcount.get<uint32_t>(nb);
  ws.d_unique = ws.unique.get<uint64_t>(n);
  ws.d_inverse = ws.inverse.get<uint32_t>(n);
  ws.d_seg = ws.seg.get<uint32_t>(n + 1);
  ws.d_sorted_mapped = d_occ_map ? ws.mapped.get<uint32_t>(n) : nullptr;
  if (bits <= 32) {
    // narrow mode: the first pass turns keys into u32 (key - kmin); digits of
    // up to 10 bits, the fewest passes: a 27-bit span (1e8 keys) takes 3
    // passes of 9 bits, a 20-bit one (1e6 keys) 2 of 10, 29 bits (5e8) 3 of 10
    int np, db;
    narrow_plan(bits, np, db);
    uint32_t* ka = reinterpret_cast<uint32_t*>(ws.keys_a.get<uint64_t>((n + 1) / 2));
    uint32_t* kb = reinterpret_cast<uint32_t*>(ws.keys_b.get<uint64_t>((n + 1) / 2));
    uint32_t* counts = ws.counts.get<uint32_t>((size_t)1024 * nb);
    uint32_t* totals = ws.totals.get<uint32_t>(1024);
    const uint32_t* kin32 = nullptr;
    const uint32_t* vin = nullptr;
    uint32_t* kout = ka;
    uint32_t* vout = va;
    for (int p = 0; p < np; ++p) {
      const int shift = p * db;
      // digits of db bits, masked with R-1: R = 2^db rounded up to 256/512/1024
      if (p == 0) {
        if (db > 9) pass_u64_to_u32<1024>(d_keys, kout, vout, n, mm, shift, counts, totals, nb, s);
        else if (db > 8) pass_u64_to_u32<512>(d_keys, kout, vout, n, mm, shift, counts, totals, nb, s);
        else pass_u64_to_u32<256>(d_keys, kout, vout, n, mm, shift, counts, totals, nb, s);
      } else {
        if (db > 9) pass_u32<1024>(kin32, vin, kout, vout, n, mm, shift, counts, totals, nb, s);
        else if (db > 8) pass_u32<512>(kin32, vin, kout, vout, n, mm, shift, counts, totals, nb, s);
        else pass_u32<256>(kin32, vin, kout, vout, n, mm, shift, counts, totals, nb, s);
      }
      kin32 = kout;
      vin = vout;
      kout = (kout == ka) ? kb : ka;
      vout = (vout == va) ? vb : va;
    }
    ws.sorted_keys = nullptr;
    ws.sorted_vals = vin;
    k_head_count<uint32_t><<<nb, ST, 0, s>>>(kin32, n, bcount); ::kp::count_launch();
    k_scan_rows<<<1, ST, 0, s>>>(bcount, nb, ws.d_nunique + 1); ::kp::count_launch();
    k_dedup_emit<uint32_t><<<nb, ST, 0, s>>>(kin32, mm, vin, n, bcount, ws.d_unique, ws.d_inverse, ws.d_seg,
                                             ws.d_nunique, nb, d_occ_map, ws.d_sorted_mapped, d_occ_ident); ::kp::count_launch();
  } else {
    const int passes = (bits + 7) / 8;
    uint64_t* ka = ws.keys_a.get<uint64_t>(n);
    uint64_t* kb = ws.keys_b.get<uint64_t>(n);
    uint32_t* counts = ws.counts.get<uint32_t>((size_t)RADIX * nb);
    uint32_t* totals = ws.totals.get<uint32_t>(RADIX);
    const uint64_t* kin = d_keys;
    const uint32_t* vin = nullptr;
    uint64_t* kout = ka;
    uint32_t* vout = va;
    for (int p = 0; p < passes; ++p) {
      const int shift = p * 8;
      k_upsweep<uint64_t, RADIX><<<nb, ST, 0, s>>>(kin, n, mm, shift, counts, nb); ::kp::count_launch();
      k_scan_rows<<<RADIX, ST, 0, s>>>(counts, nb, totals); ::kp::count_launch();
      k_downsweep<uint64_t, uint64_t, RADIX><<<nb, ST, 0, s>>>(kin, vin, kout, vout, n, mm, shift, counts, totals, nb); ::kp::count_launch();
      kin = kout;
      vin = vout;
      kout = (kout == ka) ? kb : ka;
      vout = (vout == va) ? vb : va;
    }
    ws.sorted_keys = kin;
    ws.sorted_vals = vin;
    k_head_count<uint64_t><<<nb, ST, 0, s>>>(kin, n, bcount); ::kp::count_launch();
    k_scan_rows<<<1, ST, 0, s>>>(bcount, nb, ws.d_nunique + 1); ::kp::count_launch();
    k_dedup_emit<uint64_t><<<nb, ST, 0, s>>>(kin, mm, vin, n, bcount, ws.d_unique, ws.d_inverse, ws.d_seg,
                                             ws.d_nunique, nb, d_occ_map, ws.d_sorted_mapped, d_occ_ident); ::kp::count_launch();
  }
}

static int span_bits(const unsigned long long* h_mm) {
  const uint64_t span = h_mm[1] - h_mm[0];
  return span == 0 ? 0 : 64 - __builtin_clzll(span);
}

// does a sort planned for `planned` span bits cover an actual span of `bits`?
static bool plan_covers(int planned, int bits) {
  if (planned > 32) return ((planned + 7) / 8) * 8 >= bits;  // wide: 8-bit digit passes
  if (bits > 32) return false;                               // narrow keys are u32 (key - kmin)
  int np, db;
  narrow_plan(planned, np, db);
  return np * db >= bits;
}

static bool spec_enabled() {
  static const bool on = [] {
    const char* v = getenv("KP_DEDUP_SPEC");
    return !(v && v[0] == '0');
  }();
  return on;
}

// the batch's key span against the planned passes' (a miss aborts the step)
__global__ void k_plan_check(const unsigned long long* __restrict__ mm, int planned, uint32_t* abort_word,
                             const uint32_t* __restrict__ ident_word, int expect_ident) {
  if (expect_ident >= 0 && (*ident_word == 0xFFFFFFFFu) != (expect_ident != 0)) atomicOr(abort_word, kAbortPlan);
  const uint64_t span = mm[1] - mm[0];
  const int bits = span == 0 ? 0 : 64 - __clzll((long long)span);
  bool ok;
  if (planned > 32) ok = ((planned + 7) / 8) * 8 >= bits;
  else if (bits > 32) ok = false;
  else {
    int np, db;
    narrow_plan(planned, np, db);
    ok = np * db >= bits;
  }
  if (!ok) atomicOr(abort_word, kAbortPlan);
}

bool dedup_async_ready(const DedupWs& ws, uint32_t n) { return n > 0 && spec_enabled() && ws.spec_bits >= 0; }

bool dedup(const uint64_t* d_keys, uint32_t n, DedupWs& ws, cudaStream_t s,
           const uint32_t* d_occ_map, const uint32_t* d_occ_ident, uint32_t* d_abort, int expect_ident) {
  ws.n = n;
  ws.d_nunique = ws.scalars.get<uint32_t>(4);
  if (n == 0) {
    ws.n_unique = 0;
    ws.d_unique = ws.unique.get<uint64_t>(1);
    ws.d_inverse = ws.inverse.get<uint32_t>(1);
    ws.d_seg = ws.seg.get<uint32_t>(1);
    KP_CUDA(cudaMemsetAsync(ws.d_seg, 0, 4, s));
    KP_CUDA(cudaMemsetAsync(ws.d_nunique, 0, 4, s));
    return false;
  }
  const uint32_t nb = ceil_div(n, TILE);
  auto* mm = ws.minmax.get<unsigned long long>(2);
  k_minmax_init<<<1, 1, 0, s>>>(mm); ::kp::count_launch();
  k_minmax<<<min(nb * 2, 1184u), 256, 0, s>>>(d_keys, n, mm); ::kp::count_launch();
  if (spec_enabled() && ws.spec_bits >= 0 && d_abort) {
    // no readback at all: the plan is checked on the device
    const int planned = ws.spec_bits;
    dedup_sort(d_keys, n, ws, s, d_occ_map, d_occ_ident, planned, mm, nb);
    k_plan_check<<<1, 1, 0, s>>>(mm, planned, d_abort, d_occ_ident, d_occ_ident ? expect_ident : -1);
    ::kp::count_launch();
    ws.n_unique = kUnknownU;
    return true;
  }
  if (spec_enabled() && ws.spec_bits >= 0) {
    // Plan the passes from the previous call's key span and check it with
    // the final readback (one host sync per dedup instead of two); a batch
    // whose span outgrows the plan is sorted again with the exact plan.
    const int planned = ws.spec_bits;
    dedup_sort(d_keys, n, ws, s, d_occ_map, d_occ_ident, planned, mm, nb);
    unsigned long long h_mm[2];
    KP_CUDA(cudaMemcpyAsync(h_mm, mm, 16, cudaMemcpyDeviceToHost, s));
    KP_CUDA(cudaMemcpyAsync(&ws.n_unique, ws.d_nunique, 4, cudaMemcpyDeviceToHost, s));
    KP_CUDA(cudaStreamSynchronize(s));
    const int bits = span_bits(h_mm);
    ws.spec_bits = bits;
    if (plan_covers(planned, bits)) return false;
    dedup_sort(d_keys, n, ws, s, d_occ_map, d_occ_ident, bits, mm, nb);
    KP_CUDA(cudaMemcpyAsync(&ws.n_unique, ws.d_nunique, 4, cudaMemcpyDeviceToHost, s));
    KP_CUDA(cudaStreamSynchronize(s));
    return false;
  }
  unsigned long long h_mm[2];
  KP_CUDA(cudaMemcpyAsync(h_mm, mm, 16, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaStreamSynchronize(s));
  const int bits = span_bits(h_mm);
  ws.spec_bits = bits;
  dedup_sort(d_keys, n, ws, s, d_occ_map, d_occ_ident, bits, mm, nb);
  KP_CUDA(cudaMemcpyAsync(&ws.n_unique, ws.d_nunique, 4, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaStreamSynchronize(s));
  return false;
}

// Same outputs as dedup() when the keys are R runs that are each strictly
// ascending (the owner's received keys: each source sends its unique keys in
// order): a pairwise merge tree (log2 R levels of merge path) replaces the
// radix passes.
void dedup_runs(const uint64_t* d_keys, uint32_t n, const std::vector<uint64_t>& run_off,
                DedupWs& ws, cudaStream_t s, bool readback) {
  const int R = (int)run_off.size() - 1;
  if (n == 0 || R < 1 || R > kMaxRuns) {
    dedup(d_keys, n, ws, s);
    return;
  }
  ws.n = n;
  ws.d_nunique = ws.scalars.get<uint32_t>(4);
  const uint32_t nb = ceil_div(n, TILE);
  uint64_t* ka = ws.keys_a.get<uint64_t>(n);
  uint64_t* kb = ws.keys_b.get<uint64_t>(n);
  uint32_t* va = ws.vals_a.get<uint32_t>(n);
  uint32_t* vb = ws.vals_b.get<uint32_t>(n);
  std::vector<uint64_t> runs(run_off);
  const uint64_t* kin = d_keys;
  const uint32_t* vin = nullptr;
  uint64_t* kout = ka;
  uint32_t* vout = va;
  if (R == 1) {  // already sorted
    KP_CUDA(cudaMemcpyAsync(ka, d_keys, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    k_key_iota<<<std::min<uint32_t>(nb * 8, 148 * 16), 256, 0, s>>>(va, n); ::kp::count_launch();
    kin = ka;
    vin = va;
  }
  while (runs.size() > 2) {
    MergeLevel L{};
    std::vector<uint64_t> next{runs[0]};
    uint32_t tiles = 0;
    for (size_t i = 0; i + 1 < runs.size(); i += 2) {
      const uint64_t a0 = runs[i], am = runs[i + 1];
      const uint64_t b1 = i + 2 < runs.size() ? runs[i + 2] : am;  // odd run: merged with nothing
      L.a0[L.pairs] = (uint32_t)a0;
      L.na[L.pairs] = (uint32_t)(am - a0);
      L.nb[L.pairs] = (uint32_t)(b1 - am);
      L.tile0[L.pairs] = tiles;
      tiles += ceil_div((uint32_t)(b1 - a0), TILE);
      ++L.pairs;
      next.push_back(b1);
    }
    L.tile0[L.pairs] = tiles;
    if (tiles) {
      k_merge_level<<<tiles, ST, 0, s>>>(kin, vin, kout, vout, L); ::kp::count_launch();
    }
    runs.swap(next);
    kin = kout;
    vin = vout;
    kout = (kout == ka) ? kb : ka;
    vout = (vout == va) ? vb : va;
  }
  ws.sorted_keys = kin;
  ws.sorted_vals = vin;
  uint32_t* bcount = ws.bcount.get<uint32_t>(nb);
  ws.d_unique = ws.unique.get<uint64_t>(n);
  ws.d_inverse = ws.inverse.get<uint32_t>(n);
  ws.d_seg = ws.seg.get<uint32_t>(n + 1);
  ws.d_sorted_mapped = nullptr;
  auto* mm = ws.minmax.get<unsigned long long>(2);
  k_head_count<uint64_t><<<nb, ST, 0, s>>>(kin, n, bcount); ::kp::count_launch();
  k_scan_rows<<<1, ST, 0, s>>>(bcount, nb, ws.d_nunique + 1); ::kp::count_launch();
  k_dedup_emit<uint64_t><<<nb, ST, 0, s>>>(kin, mm, vin, n, bcount, ws.d_unique, ws.d_inverse, ws.d_seg,
                                           ws.d_nunique, nb, nullptr, nullptr, nullptr); ::kp::count_launch();
  if (!readback) {  // U stays on the device (ws.d_nunique)
    ws.n_unique = kUnknownU;
    return;
  }
  KP_CUDA(cudaMemcpyAsync(&ws.n_unique, ws.d_nunique, 4, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaStreamSynchronize(s));
}

__global__ void k_counts_u64(const uint32_t* __restrict__ in, uint32_t G, uint64_t* __restrict__ out) {
  if (threadIdx.x < G) out[threadIdx.x] = in[threadIdx.x];
}

__global__ void k_pack_step_flags(const uint32_t* __restrict__ pflag, const uint32_t* __restrict__ err,
                                  uint64_t* __restrict__ out) {
  out[0] = pflag ? *pflag : 0u;
  out[1] = (uint64_t)err[0] | ((uint64_t)err[1] << 32);
}

void pack_step_flags(const uint32_t* d_pflag, const uint32_t* d_err, uint64_t* d_out, cudaStream_t s) {
  k_pack_step_flags<<<1, 1, 0, s>>>(d_pflag, d_err, d_out); ::kp::count_launch();
}

void shard(const uint64_t* d_unique, uint32_t n, uint32_t G, uint32_t* d_perm, uint32_t* d_pos,
           uint64_t* h_counts, ShardWs& ws, cudaStream_t s, uint64_t* d_counts, const uint32_t* d_n) {
  KP_CHECK(G >= 1 && G <= MAXG, kErrConfig, "shard: G must be in [1, 64]");
  KP_CHECK(h_counts || d_counts, kErrGeneric, "shard: no output for the counts");
  if (h_counts)
    for (uint32_t g = 0; g < G; ++g) h_counts[g] = 0;
  if (n == 0) {
    if (d_counts) KP_CUDA(cudaMemsetAsync(d_counts, 0, G * 8, s));
    return;
  }
  const uint32_t nb = ceil_div(n, TILE);
  uint32_t* counts = ws.bcount.get<uint32_t>((size_t)G * nb);
  uint32_t* totals = ws.scalars.get<uint32_t>(MAXG);
  k_shard_count<<<nb, ST, 0, s>>>(d_unique, n, G, counts, nb, d_n); ::kp::count_launch();
  k_scan_rows<<<G, ST, 0, s>>>(counts, nb, totals); ::kp::count_launch();
  k_shard_emit<<<nb, ST, 0, s>>>(d_unique, n, G, counts, totals, nb, d_perm, d_pos, d_n); ::kp::count_launch();
  if (d_counts) {
    k_counts_u64<<<1, MAXG, 0, s>>>(totals, G, d_counts); ::kp::count_launch();
  }
  if (!h_counts) return;
  uint32_t h[MAXG];
  KP_CUDA(cudaMemcpyAsync(h, totals, G * 4, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaStreamSynchronize(s));
  for (uint32_t g = 0; g < G; ++g) h_counts[g] = h[g];
}

}  // namespace kp
