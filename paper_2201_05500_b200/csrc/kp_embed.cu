// Embedding pull + per-slot sum pooling, and the backward segmented reduce
// fused with the in-place sparse update (the "push").
//
// Reference: pooling in CtrModel::forward (proj/src/model.cpp:88-99) via the
// per-occurrence EmbeddingSource lookup (proj/src/trainer.cpp:137-139); sparse
// grads scattered per key in backward (proj/src/model.cpp:180-188), summed over
// workers in ascending order (proj/src/trainer.cpp:180-186), scaled by 1/N
// (:202-207) and pushed through AdaGrad (proj/src/store.cpp:191-208).
//
// Layout: a "bag" is one (instance, slot) pair; bag b = instance*S + slot and
// pooled rows are [bags][e] = [B][S*e] (S=1: the reference's one pooled vector
// per instance). Rows move as float4 (16 B per lane, e/4 lanes per row).
// Sums run in occurrence order inside a lane, so pooling is bit-identical to
// the fp32 oracle; the backward reduce is a fixed-order two-level segmented
// sum (chunk partials combined in chunk order) -- deterministic, no float
// atomics.
#include <cstdlib>

#include "kp_table.cuh"
#include "kp_tcgen05.cuh"

namespace kp {
namespace {

unsigned grid_cap(uint64_t blocks) {
  if (blocks < 1) blocks = 1;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  return (unsigned)blocks;
}

__global__ void k_prepare_bags(const uint32_t* __restrict__ offs, uint32_t occ_base,
                               const uint16_t* __restrict__ slots, uint32_t n_inst, uint32_t S,
                               uint32_t* __restrict__ bag_offs, uint32_t* __restrict__ bag_of_occ,
                               uint32_t* __restrict__ err,
                               uint32_t* __restrict__ abort_word, int maps) {
  // (maps == 0: only the checks -- the caller predicted one feature per slot,
  // whose maps are the identity and go unread; a miss aborts the step)
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  bool nonid = false;  // some bag_of_occ[o] != o
  for (uint32_t i = w0; i < n_inst; i += nw) {
    const uint32_t o0 = offs[i] - occ_base, o1 = offs[i + 1] - occ_base;
    if (S == 1) {
      if (lane == 0) bag_offs[i] = o0;
      for (uint32_t o = o0 + lane; o < o1; o += 32) {
        bag_of_occ[o] = i;
        nonid |= o != i;
      }
    } else {
      if (o0 == o1) {
        if (maps)
          for (uint32_t s = lane; s < S; s += 32) bag_offs[(uint64_t)i * S + s] = o0;
        nonid = true;  // an empty instance: not one feature in every slot
        continue;
      }
      for (uint32_t ob = o0; ob < o1; ob += 128) {
        // the instance's slot ids (and predecessors) for 4 rounds in flight at once
        uint32_t sv[4];
        int pv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t o = ob + lane + 32 * k;
          sv[k] = o < o1 ? slots[o] : 0;
          pv[k] = o < o1 && o > o0 ? (int)slots[o - 1] : -1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t o = ob + lane + 32 * k;
          if (o >= o1) break;
          const uint32_t s = sv[k];
          const int prev = pv[k];
          if (s >= S || (int)s < prev) {
            atomicMin(err, o);
            if (abort_word) atomicOr(abort_word, kAbortPlan);
            nonid = true;
            if (maps) bag_of_occ[o] = i * S;  // keep downstream indexing in bounds; the batch is rejected
            continue;
          }
          if (maps) {
            for (int t = prev + 1; t <= (int)s; ++t) bag_offs[(uint64_t)i * S + t] = o;
            if (o == o1 - 1)
              for (uint32_t t = s + 1; t < S; ++t) bag_offs[(uint64_t)i * S + t] = o1;
            bag_of_occ[o] = i * S + s;
          }
          nonid |= o != i * S + s;
        }
      }
    }
  }
  if (maps && blockIdx.x == 0 && threadIdx.x == 0) bag_offs[(uint64_t)n_inst * S] = offs[n_inst] - occ_base;
  // one store per warp that saw a mismatch, skipped once another landed
  if (__any_sync(0xffffffffu, nonid) && lane == 0 && *(volatile uint32_t*)(err + 1) != 0u) err[1] = 0u;
}

// ---- row access policies -------------------------------------------------
// V4: lane gl of an LPG-lane group owns dims [4*gl, 4*gl+4); e == 4*LPG.
// Scalar: LPG = 32, lane owns dims gl + 32*q (q < NV), masked by j < e.
template <int LPG, int NV, bool V4>
struct Row {
  float v[V4 ? 4 : NV];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < (V4 ? 4 : NV); ++q) v[q] = 0.f;
  }
  __device__ __forceinline__ void load(const float* __restrict__ p, int gl, uint32_t e) {
    if (V4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(p) + gl);
      v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
    } else {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const uint32_t j = gl + 32 * q;
        v[q] = j < e ? __ldg(p + j) : 0.f;
      }
    }
  }
  __device__ __forceinline__ void store(float* __restrict__ p, int gl, uint32_t e) const {
    if (V4) {
      reinterpret_cast<float4*>(p)[gl] = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const uint32_t j = gl + 32 * q;
        if (j < e) p[j] = v[q];
      }
    }
  }
  __device__ __forceinline__ void add(const Row& o) {
#pragma unroll
    for (int q = 0; q < (V4 ? 4 : NV); ++q) v[q] = __fadd_rn(v[q], o.v[q]);
  }
  __device__ __forceinline__ void scale(float s) {
#pragma unroll
    for (int q = 0; q < (V4 ? 4 : NV); ++q) v[q] = __fmul_rn(v[q], s);
  }
  __device__ __forceinline__ int dim(int gl, int q) const { return V4 ? 4 * gl + q : gl + 32 * q; }
};

// Each group pools PB consecutive bags per iteration: their row loads are
// independent, so PB rows are in flight even for one-feature bags (S slots of
// one feature each); inside a bag rows are still summed in occurrence order.
constexpr int PB = 4;

template <int LPG, int NV, bool V4>
__global__ void __launch_bounds__(256, 5) k_pool(const uint32_t* __restrict__ bag_offs, uint32_t n_bags,
                                              const uint32_t* __restrict__ rowocc,
                                              const float* __restrict__ src, uint32_t e, int mean,
                                              float* __restrict__ pooled,
                                              float* __restrict__ inv_count,
                                              unsigned* __restrict__ inst_max, uint32_t S) {
  const int gl = threadIdx.x % LPG;
  const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPG;
  const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / LPG;
  for (uint64_t b0 = g0 * PB; b0 < n_bags; b0 += ng * PB) {
    uint32_t o[PB + 1];
#pragma unroll
    for (int i = 0; i <= PB; ++i) o[i] = bag_offs[b0 + i < n_bags ? b0 + i : n_bags];
    Row<LPG, NV, V4> acc[PB], r[PB];
    uint32_t maxlen = 0;
#pragma unroll
    for (int i = 0; i < PB; ++i) {
      acc[i].zero();
      maxlen = max(maxlen, o[i + 1] - o[i]);
    }
    for (uint32_t j = 0; j < maxlen; ++j) {
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        if (o[i] + j < o[i + 1]) {
          const uint32_t rr = rowocc[o[i] + j];
          if (rr == kNoRow) r[i].zero();  // table full: error raised at the batch end
          else r[i].load(src + (uint64_t)rr * e, gl, e);
        }
      }
#pragma unroll
      for (int i = 0; i < PB; ++i)
        if (o[i] + j < o[i + 1]) acc[i].add(r[i]);  // occurrence order (model.cpp:93)
    }
#pragma unroll
    for (int i = 0; i < PB; ++i) {
      const uint64_t b = b0 + i;
      if (b >= n_bags) break;
      const uint32_t len = o[i + 1] - o[i];
      if (mean) {
        const float inv = len ? __fdiv_rn(1.f, (float)len) : 1.f;  // model.cpp:95-97
        if (len) acc[i].scale(inv);
        if (gl == 0) inv_count[b] = inv;
      }
      acc[i].store(pooled + b * e, gl, e);
    }
    if (inst_max) {
      // max |pooled| per instance (= per row of the [B][S*e] MLP input), the
      // row scale of the fp16-operand first layer. S >= PB: the group's PB
      // consecutive bags touch at most two instances -> two lane reductions
      // and at most two atomics per group; else one per bag.
      if (S >= PB) {
        const uint64_t i0 = b0 / S;
        float m0 = 0.f, m1 = 0.f;
#pragma unroll
        for (int i = 0; i < PB; ++i) {
          if (b0 + i >= n_bags) break;
          float mx = 0.f;
#pragma unroll
          for (int q = 0; q < (V4 ? 4 : NV); ++q) mx = fmaxf(mx, fabsf(acc[i].v[q]));
          if ((b0 + i) / S == i0) m0 = fmaxf(m0, mx);
          else m1 = fmaxf(m1, mx);
        }
#pragma unroll
        for (int o = LPG / 2; o; o >>= 1) {
          m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o, LPG));
          m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o, LPG));
        }
        if (gl == 0) {
          if (m0 > 0.f) atomicMax(inst_max + i0, __float_as_uint(m0));
          if (m1 > 0.f) atomicMax(inst_max + i0 + 1, __float_as_uint(m1));
        }
      } else {
#pragma unroll
        for (int i = 0; i < PB; ++i) {
          float mx = 0.f;
#pragma unroll
          for (int q = 0; q < (V4 ? 4 : NV); ++q) mx = fmaxf(mx, fabsf(acc[i].v[q]));
#pragma unroll
          for (int o = LPG / 2; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o, LPG));
          const uint64_t b = b0 + i;
          if (gl == 0 && b < n_bags && mx > 0.f) atomicMax(inst_max + b / S, __float_as_uint(mx));
        }
      }
    }
  }
}

// Instance-major pooling (S >= 2*PB, row maxima requested): one warp owns an
// instance's S bags -- its two 16-lane groups take PB bags each per
// iteration -- so the max |pooled| of the instance (the fp16 first layer's row
// scale) is a warp reduction and one store, no atomics. Same per-bag
// arithmetic as k_pool.
template <int LPG, int NV, bool V4>
__global__ void __launch_bounds__(256, 5) k_pool_inst(const uint32_t* __restrict__ bag_offs,
                                                      uint32_t n_inst, uint32_t S,
                                                      const uint32_t* __restrict__ rowocc,
                                                      const float* __restrict__ src, uint32_t e, int mean,
                                                      float* __restrict__ pooled,
                                                      float* __restrict__ inv_count,
                                                      float* __restrict__ inst_max) {
  constexpr int GPW = 32 / LPG;  // groups per warp
  const int lane = threadIdx.x & 31, gl = lane % LPG, gw = lane / LPG;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t inst = w0; inst < n_inst; inst += nw) {
    const uint64_t bend = (inst + 1) * S;
    float wmax = 0.f;
    for (uint64_t b0 = inst * S + (uint64_t)gw * PB; b0 < bend; b0 += (uint64_t)GPW * PB) {
      uint32_t o[PB + 1];
#pragma unroll
      for (int i = 0; i <= PB; ++i) o[i] = bag_offs[b0 + i < bend ? b0 + i : bend];
      Row<LPG, NV, V4> acc[PB], r[PB];
      uint32_t maxlen = 0;
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        acc[i].zero();
        maxlen = max(maxlen, o[i + 1] - o[i]);
      }
      for (uint32_t j = 0; j < maxlen; ++j) {
#pragma unroll
        for (int i = 0; i < PB; ++i) {
          if (o[i] + j < o[i + 1]) {
            const uint32_t rr = rowocc[o[i] + j];
            if (rr == kNoRow) r[i].zero();
            else r[i].load(src + (uint64_t)rr * e, gl, e);
          }
        }
#pragma unroll
        for (int i = 0; i < PB; ++i)
          if (o[i] + j < o[i + 1]) acc[i].add(r[i]);
      }
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        const uint64_t b = b0 + i;
        if (b >= bend) break;
        const uint32_t len = o[i + 1] - o[i];
        if (mean) {
          const float inv = len ? __fdiv_rn(1.f, (float)len) : 1.f;
          if (len) acc[i].scale(inv);
          if (gl == 0) inv_count[b] = inv;
        }
        acc[i].store(pooled + b * e, gl, e);
#pragma unroll
        for (int q = 0; q < (V4 ? 4 : NV); ++q) wmax = fmaxf(wmax, fabsf(acc[i].v[q]));
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
    if (lane == 0) inst_max[inst] = wmax;
  }
}

// Pooling straight into the first layer's fp16 operand planes (kp_gemm_h3.cu):
// one block per instance holds the instance's whole pooled row (S*e floats,
// NP float4 cells per thread) in registers, reduces its max |x|, and writes
// hi = rn(x * 2^e), lo = rn(x * 2^e - hi) with e = row_exp(max) -- the same 4
// bytes per element as the fp32 row, so the GEMMs never split on chip. Cell
// c = (bag c / (e/4), float4 column c % (e/4)); a bag's rows are summed in
// occurrence order (model.cpp:93), bit-identical to k_pool before the split.
template <int NT, int NP>
__global__ void __launch_bounds__(NT, NP <= 4 ? 4 : 2) k_pool_planes(const uint32_t* __restrict__ bag_offs, uint32_t n_inst,
                                                    uint32_t S, const uint32_t* __restrict__ rowocc,
                                                    const float* __restrict__ src, uint32_t e, int mean,
                                                    __half* __restrict__ hi, __half* __restrict__ lo,
                                                    int* __restrict__ inst_exp, float* __restrict__ inv_count) {
  __shared__ float red[NT / 32];
  const uint32_t lpr = e >> 2, ncell = S * lpr;
  for (uint64_t inst = blockIdx.x; inst < n_inst; inst += gridDim.x) {
    uint32_t o0[NP], o1[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t c = threadIdx.x + p * NT;
      const uint64_t b = inst * S + (c < ncell ? c / lpr : 0);
      o0[p] = c < ncell ? bag_offs[b] : 0;
      o1[p] = c < ncell ? bag_offs[b + 1] : 0;
    }
    float4 v[NP];
    // first occurrence of every cell's bag: NP independent row loads in flight
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t c = threadIdx.x + p * NT;
      v[p] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (o0[p] < o1[p]) {
        const uint32_t rr = rowocc[o0[p]];
        if (rr != kNoRow) v[p] = __ldg(reinterpret_cast<const float4*>(src + (uint64_t)rr * e) + c % lpr);
      }
    }
    float mx = 0.f;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t c = threadIdx.x + p * NT;
      for (uint32_t o = o0[p] + 1; o < o1[p]; ++o) {  // multi-feature bags, occurrence order
        const uint32_t rr = rowocc[o];
        if (rr == kNoRow) continue;
        const float4 x = __ldg(reinterpret_cast<const float4*>(src + (uint64_t)rr * e) + c % lpr);
        v[p].x = __fadd_rn(v[p].x, x.x), v[p].y = __fadd_rn(v[p].y, x.y);
        v[p].z = __fadd_rn(v[p].z, x.z), v[p].w = __fadd_rn(v[p].w, x.w);
      }
      if (mean && c < ncell) {
        const uint32_t len = o1[p] - o0[p];
        const float inv = len ? __fdiv_rn(1.f, (float)len) : 1.f;  // model.cpp:95-97
        if (len) v[p].x = __fmul_rn(v[p].x, inv), v[p].y = __fmul_rn(v[p].y, inv),
                 v[p].z = __fmul_rn(v[p].z, inv), v[p].w = __fmul_rn(v[p].w, inv);
        if (c % lpr == 0) inv_count[inst * S + c / lpr] = inv;
      }
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[p].x), fabsf(v[p].y)), fmaxf(fabsf(v[p].z), fabsf(v[p].w))));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.f;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) mx = fmaxf(mx, red[w]);
    __syncthreads();  // red is reused by the next instance
    const int ex = tc::row_exp(mx);
    if (threadIdx.x == 0) inst_exp[inst] = ex;
    const float sc = tc::pow2f(ex);
    uint2* h2 = reinterpret_cast<uint2*>(hi + inst * ncell * 4);
    uint2* l2 = reinterpret_cast<uint2*>(lo + inst * ncell * 4);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t c = threadIdx.x + p * NT;
      if (c >= ncell) break;
      uint2 hh, ll;
      tc::split_h2(__fmul_rn(v[p].x, sc), __fmul_rn(v[p].y, sc), hh.x, ll.x);
      tc::split_h2(__fmul_rn(v[p].z, sc), __fmul_rn(v[p].w, sc), hh.y, ll.y);
      h2[c] = hh;
      l2[c] = ll;
    }
  }
}

// The same for the common layout of one feature per slot (bag b = occurrence
// b, flagged by prepare_bags): no bag offsets, cell c's row is rowocc[inst*S
// + c / (e/4)], and the next instance's row indices are loaded while this
// instance's rows are in flight (the index -> row chain is the latency).
// (inverse set: rowocc is the unique -> row map and the row of occurrence o is
// rowocc[inverse[o]] -- the compose pass folded into the index prefetch)
template <int NT, int NP>
__global__ void __launch_bounds__(NT, 4) k_pool_planes_ident(uint32_t n_inst, uint32_t S,
                                                             const uint32_t* __restrict__ rowocc,
                                                             const uint32_t* __restrict__ inverse,
                                                             const float* __restrict__ src, uint32_t e,
                                                             __half* __restrict__ hi, __half* __restrict__ lo,
                                                             int* __restrict__ inst_exp,
                                                             float* __restrict__ inv_count, int mean) {
  __shared__ float red[2][NT / 32];
  const uint32_t lpr = e >> 2, ncell = S * lpr;
  uint32_t rr[NP];
  uint64_t inst = blockIdx.x;
  auto load_idx = [&](uint64_t i, uint32_t (&r)[NP]) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t c = threadIdx.x + p * NT;
      r[p] = (i < n_inst && c < ncell) ? __ldg((inverse ? inverse : rowocc) + i * S + c / lpr) : kNoRow;
    }
    if (inverse) {
#pragma unroll
      for (int p = 0; p < NP; ++p)
        if (r[p] != kNoRow) r[p] = __ldg(rowocc + r[p]);
    }
  };
  load_idx(inst, rr);
  for (int it = 0; inst < n_inst; inst += gridDim.x, ++it) {
    float4 v[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t c = threadIdx.x + p * NT;
      v[p] = rr[p] != kNoRow ? __ldg(reinterpret_cast<const float4*>(src + (uint64_t)rr[p] * e) + c % lpr)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    load_idx(inst + gridDim.x, rr);  // next instance's indices, overlapping the row loads
    float mx = 0.f;
#pragma unroll
    for (int p = 0; p < NP; ++p)
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[p].x), fabsf(v[p].y)), fmaxf(fabsf(v[p].z), fabsf(v[p].w))));
#pragma unroll
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if ((threadIdx.x & 31) == 0) red[it & 1][threadIdx.x >> 5] = mx;  // double-buffered: one sync
    __syncthreads();
    mx = 0.f;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) mx = fmaxf(mx, red[it & 1][w]);
    const int ex = tc::row_exp(mx);
    if (threadIdx.x == 0) inst_exp[inst] = ex;
    if (mean && threadIdx.x < S) inv_count[inst * S + threadIdx.x] = 1.f;  // one feature per bag
    const float sc = tc::pow2f(ex);
    uint2* h2 = reinterpret_cast<uint2*>(hi + inst * ncell * 4);
    uint2* l2 = reinterpret_cast<uint2*>(lo + inst * ncell * 4);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t c = threadIdx.x + p * NT;
      if (c >= ncell) break;
      uint2 hh, ll;
      tc::split_h2(__fmul_rn(v[p].x, sc), __fmul_rn(v[p].y, sc), hh.x, ll.x);
      tc::split_h2(__fmul_rn(v[p].z, sc), __fmul_rn(v[p].w, sc), hh.y, ll.y);
      h2[c] = hh;
      l2[c] = ll;
    }
  }
}

// max |x| of each unique key's source row (half a warp per row of e <= 64
// floats as float4s; kNoRow -> 0)
__global__ void k_unique_maxabs(const float* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t U,
                                uint32_t e, float* __restrict__ umax) {
  const uint32_t lpr = e >> 2;  // float4 lanes per row (<= 16)
  const uint32_t lane = threadIdx.x & 31, sub = lane / lpr, per = 32 / lpr;
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const unsigned gmask = lpr == 32 ? 0xffffffffu : (((1u << lpr) - 1u) << (sub * lpr));
  for (uint64_t u0 = (uint64_t)w0 * per; u0 < U; u0 += (uint64_t)nw * per) {
    const uint64_t u = u0 + sub;
    float mx = 0.f;
    if (u < U && sub < per) {
      const uint32_t r = __ldg(idx + u);
      if (r != kNoRow) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src + (uint64_t)r * e) + lane % lpr);
        mx = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
      }
    }
    for (uint32_t o = lpr / 2; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, o, lpr));
    if (u < U && sub < per && lane % lpr == 0) umax[u] = mx;
  }
}

// per instance: row_exp(max over its S slots of umax[inverse[i*S + s]]) --
// the exponent k_pool_planes_ident computes from the pooled row itself
__global__ void k_inst_exp(const uint32_t* __restrict__ inverse, const float* __restrict__ umax,
                           uint32_t n_inst, uint32_t S, int* __restrict__ inst_exp, float* __restrict__ inv_count,
                           int mean) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w0; i < n_inst; i += nw) {
    float mx = 0.f;
    for (uint32_t s = lane; s < S; s += 32) {
      mx = fmaxf(mx, __ldg(umax + __ldg(inverse + i * S + s)));
      if (mean) inv_count[i * S + s] = 1.f;  // one feature per bag
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) inst_exp[i] = tc::row_exp(mx);
  }
}

__global__ void k_compose(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ inverse,
                          uint32_t n, uint32_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = idx[inverse[i]];
}

// ---- segmented reduce + sparse rule ---------------------------------------
struct SegArgs {
  const uint32_t* seg;
  uint32_t U;
  const uint32_t* sorted_vals;
  const uint32_t* bag_of_occ;
  uint32_t n_pos;
  const float* rows_src;
  uint32_t e;
  float inv_n;
  const uint32_t* table_rows;
  float* grad_out;
  const uint32_t* out_idx;
  float* partials;
  const uint32_t* first;  // [nchunks] segment holding the chunk's first position
  uint32_t CH;
  int apply;
  int peer;     // store through pm (remote windows) instead of grad_out
  PeerMap pm;
  int rule;
  float lr, b1, b2;
};

template <int LPG, int NV, bool V4>
__device__ __forceinline__ void finalize(const SegArgs& a, const TView& t, uint32_t u,
                                         Row<LPG, NV, V4>& g, int gl) {
  g.scale(a.inv_n);  // trainer.cpp:204-206 (x 1/N)
  if (!a.apply) {
    const uint32_t o = a.out_idx ? a.out_idx[u] : u;
    float* dst = a.peer ? reinterpret_cast<float*>(peer_dst(a.pm, o)) : a.grad_out + (uint64_t)o * a.e;
    g.store(dst, gl, a.e);
    return;
  }
  if (a.table_rows[u] == kNoRow) return;  // table full: error raised at the batch end
  const uint64_t o = (uint64_t)a.table_rows[u] * a.e;
#pragma unroll
  for (int q = 0; q < (V4 ? 4 : NV); ++q) {
    const int j = g.dim(gl, q);
    if (j >= (int)a.e) continue;
    if (a.rule == 0) {
      float w = t.w[o + j], acc = t.s1[o + j];
      adagrad1(w, acc, g.v[q], a.lr);
      t.w[o + j] = w;
      t.s1[o + j] = acc;
    } else {
      float w = t.w[o + j], m = t.s1[o + j], v = t.s2[o + j];
      adam1(w, m, v, g.v[q], a.lr, a.b1, a.b2);
      t.w[o + j] = w;
      t.s1[o + j] = m;
      t.s2[o + j] = v;
    }
  }
}

__device__ __forceinline__ uint32_t src_row(const SegArgs& a, uint32_t p) {
  const uint32_t occ = a.sorted_vals[p];
  return a.bag_of_occ ? a.bag_of_occ[occ] : occ;
}

template <int LPG, int NV, bool V4>
__device__ __forceinline__ void sum_range(const SegArgs& a, uint32_t p, uint32_t q,
                                          Row<LPG, NV, V4>& acc, int gl) {
  constexpr int UR = V4 ? 8 : 4;  // rows in flight per group
  Row<LPG, NV, V4> r[UR];
  for (; p + UR <= q; p += UR) {
    uint32_t sr[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) sr[u] = src_row(a, p + u);
#pragma unroll
    for (int u = 0; u < UR; ++u) r[u].load(a.rows_src + (uint64_t)sr[u] * a.e, gl, a.e);
#pragma unroll
    for (int u = 0; u < UR; ++u) acc.add(r[u]);
  }
  // (the tail one row at a time: batching its loads with predicates
  // measured slower, 0.76 vs 0.70 ms -- registers/occupancy)
  for (; p < q; ++p) {
    r[0].load(a.rows_src + (uint64_t)src_row(a, p) * a.e, gl, a.e);
    acc.add(r[0]);
  }
}

// Pipelined chunk walk (float4 rows, LPG >= 8 lanes per row, CH <= 64):
//  * the chunk's source-row indices are loaded up front, KP per lane
//    (position p0 + gl + LPG*k), and broadcast by shuffles -- no
//    index -> row dependency inside the row loop;
//  * a segment that ends inside the chunk has its table row index and its
//    current state (w, s1[, s2]) loaded BEFORE its gradient rows are summed,
//    so the read-modify-write overlaps the sum: a one-feature key costs two
//    dependent latencies instead of four.
// Arithmetic (sum order, x 1/N, the rule) is the scalar path's, bit for bit.
template <int LPG, int KP>
__device__ __forceinline__ uint32_t pos_row(const uint32_t (&srow)[KP], uint32_t rel) {
  // the two groups of a warp walk different chunks: shuffle within the group
  const uint32_t gmask = LPG == 32 ? 0xffffffffu : (((1u << LPG) - 1u) << ((threadIdx.x & 31) & ~(LPG - 1)));
  const uint32_t k = rel / LPG;
  uint32_t v = srow[0];
#pragma unroll
  for (int i = 1; i < KP; ++i) v = k == (uint32_t)i ? srow[i] : v;
  return __shfl_sync(gmask, v, (int)(rel % LPG), LPG);
}

template <int LPG, int NV, bool V4>
__device__ __forceinline__ void sum_range_pre(const SegArgs& a, const uint32_t (&srow)[64 / LPG], uint32_t p0,
                                              uint32_t p, uint32_t q, Row<LPG, NV, V4>& acc, int gl) {
  constexpr int UR = 8;
  Row<LPG, NV, V4> r[UR];
  // group-uniform loop bounds: every lane takes part in the shuffles
  for (; p + UR <= q; p += UR) {
    uint32_t sr[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) sr[u] = pos_row<LPG, 64 / LPG>(srow, p + u - p0);
#pragma unroll
    for (int u = 0; u < UR; ++u) r[u].load(a.rows_src + (uint64_t)sr[u] * a.e, gl, a.e);
#pragma unroll
    for (int u = 0; u < UR; ++u) acc.add(r[u]);
  }
  if (p < q) {
    uint32_t sr[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) sr[u] = pos_row<LPG, 64 / LPG>(srow, min(p + u, q - 1) - p0);
#pragma unroll
    for (int u = 0; u < UR; ++u)
      if (p + u < q) r[u].load(a.rows_src + (uint64_t)sr[u] * a.e, gl, a.e);
#pragma unroll
    for (int u = 0; u < UR; ++u)
      if (p + u < q) acc.add(r[u]);
  }
}

template <int LPG, int NV, bool V4>
__global__ void __launch_bounds__(256, 3) k_seg_chunks_pre(SegArgs a, TView t) {
  static_assert(V4 && LPG >= 8, "pipelined walk: float4 rows, >= 8 lanes");
  constexpr int KP = 64 / LPG;
  if (aborted(t.abort)) return;  // no row updates after a peer timeout
  const int gl = threadIdx.x % LPG;
  const uint32_t nchunks = (a.n_pos + a.CH - 1) / a.CH;
  const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPG;
  const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / LPG;
  for (uint64_t c = g0; c < nchunks; c += ng) {
    const uint32_t p0 = (uint32_t)c * a.CH, p1 = min(a.n_pos, p0 + a.CH);
    uint32_t srow[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const uint32_t p = p0 + gl + LPG * k;
      srow[k] = p < p1 ? src_row(a, p) : 0u;
    }
    uint32_t u = a.first[c];  // largest u with seg[u] <= p0
    uint32_t s0 = a.seg[u], s1 = a.seg[u + 1];
    for (;;) {
      const uint32_t s2 = s1 < p1 ? a.seg[u + 2] : 0u;  // next segment's end, in flight
      const bool before = s0 < p0, after = s1 > p1;
      const bool fin = !before && !after;
      // the finalized segment's row state, loaded while its gradients are summed
      uint32_t trow = kNoRow;
      float4 w4 = make_float4(0.f, 0.f, 0.f, 0.f), m4 = w4, v4 = w4;
      if (fin && a.apply) {
        trow = a.table_rows[u];
        if (trow != kNoRow) {
          const uint64_t o = (uint64_t)trow * a.e;
          w4 = reinterpret_cast<const float4*>(t.w + o)[gl];
          m4 = reinterpret_cast<const float4*>(t.s1 + o)[gl];
          if (a.rule != 0) v4 = reinterpret_cast<const float4*>(t.s2 + o)[gl];
        }
      }
      Row<LPG, NV, V4> acc;
      acc.zero();
      sum_range_pre(a, srow, p0, max(s0, p0), min(s1, p1), acc, gl);
      if (fin) {
        if (!a.apply) {
          finalize(a, t, u, acc, gl);
        } else if (trow != kNoRow) {
          acc.scale(a.inv_n);  // trainer.cpp:204-206 (x 1/N)
          float* wv = &w4.x;
          float* mv = &m4.x;
          float* vv = &v4.x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (a.rule == 0) adagrad1(wv[q], mv[q], acc.v[q], a.lr);
            else adam1(wv[q], mv[q], vv[q], acc.v[q], a.lr, a.b1, a.b2);
          }
          const uint64_t o = (uint64_t)trow * a.e;
          reinterpret_cast<float4*>(t.w + o)[gl] = w4;
          reinterpret_cast<float4*>(t.s1 + o)[gl] = m4;
          if (a.rule != 0) reinterpret_cast<float4*>(t.s2 + o)[gl] = v4;
        }
      } else {
        acc.store(a.partials + ((uint64_t)c * 2 + (before ? 0 : 1)) * a.e, gl, a.e);
        if (before && after) {  // spans the chunk: its (unused) tail slot reads as 0
          acc.zero();
          acc.store(a.partials + ((uint64_t)c * 2 + 1) * a.e, gl, a.e);
        }
      }
      if (s1 >= p1) break;
      ++u;
      s0 = s1;
      s1 = s2;
    }
  }
  if (a.peer) __threadfence_system();  // remote stores complete before the signal
}

// Phase 1: one group per chunk of CH sorted positions.
template <int LPG, int NV, bool V4>
__global__ void __launch_bounds__(256, 6) k_seg_chunks(SegArgs a, TView t) {
  if (aborted(t.abort)) return;  // no row updates after a peer timeout
  const int gl = threadIdx.x % LPG;
  const uint32_t nchunks = (a.n_pos + a.CH - 1) / a.CH;
  const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPG;
  const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / LPG;
  const uint32_t pw = (uint32_t)(a.e * (V4 ? 1 : 1));
  (void)pw;
  for (uint64_t c = g0; c < nchunks; c += ng) {
    const uint32_t p0 = (uint32_t)c * a.CH, p1 = min(a.n_pos, p0 + a.CH);
    uint32_t u = a.first[c];  // largest u with seg[u] <= p0
    for (;;) {
      const uint32_t s0 = a.seg[u], s1 = a.seg[u + 1];
      Row<LPG, NV, V4> acc;
      acc.zero();
      sum_range(a, max(s0, p0), min(s1, p1), acc, gl);
      const bool before = s0 < p0, after = s1 > p1;
      if (!before && !after) {
        finalize(a, t, u, acc, gl);
      } else {
        acc.store(a.partials + ((uint64_t)c * 2 + (before ? 0 : 1)) * a.e, gl, a.e);
        if (before && after) {  // spans the chunk: its (unused) tail slot reads as 0
          acc.zero();
          acc.store(a.partials + ((uint64_t)c * 2 + 1) * a.e, gl, a.e);
        }
      }
      if (s1 >= p1) break;
      ++u;
    }
  }
  if (a.peer) __threadfence_system();  // remote stores complete before the signal
}

// Phase 2: a segment spanning chunks c0 < c1 owns the contiguous flattened
// partial range P[2c0+1 .. 2c1] (tail of c0, then head of each later chunk;
// the unused tail slots in between hold 0). Short ranges are summed in order;
// long ones (Zipf-hot keys) as loose head + QB-entry block sums Q + loose tail,
// the hottest (more than 2*QB Q blocks) with a second level Q2 of QB-Q sums.
// QB = 16: the fix-up's loose head/tail walks are what a hot key waits on
// (configs[1] push 0.712 -> 0.705 ms, configs[0] 0.051 -> 0.039 ms vs 64).
constexpr uint32_t QB = 16;
static_assert(QB % 16 == 0, "block sums load 16 (float4) or 4 rows per round");

template <int LPG, int NV, bool V4>
__global__ void __launch_bounds__(256) k_seg_blocksum(const float* __restrict__ src, uint32_t nP, uint32_t e,
                                                      float* __restrict__ Q) {
  const int gl = threadIdx.x % LPG;
  const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPG;
  const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / LPG;
  for (uint64_t j = g0; j < nP / QB; j += ng) {
    constexpr int UB = V4 ? 16 : 4;  // rows in flight (the Q2 level is latency-bound)
    Row<LPG, NV, V4> acc, r[UB];
    acc.zero();
    for (uint32_t i = 0; i < QB; i += UB) {
#pragma unroll
      for (int u = 0; u < UB; ++u) r[u].load(src + (j * QB + i + u) * e, gl, e);
#pragma unroll
      for (int u = 0; u < UB; ++u) acc.add(r[u]);
    }
    acc.store(Q + j * e, gl, e);
  }
}

// Both block-sum levels in one launch (LPG <= 4, small rows: the step is
// latency-bound there, configs[0]): block j's QB groups form
// Q[QB*j .. QB*j+QB-1] as k_seg_blocksum does, then (a full block) its first
// group sums those 64 in order into Q2[j] -- the second level's sum, bit for
// bit, without the second launch.
template <int LPG, int NV, bool V4>
__global__ void __launch_bounds__(256) k_seg_blocksum12(const float* __restrict__ src, uint32_t nP, uint32_t e,
                                                         float* Q, float* __restrict__ Q2) {
  const int gl = threadIdx.x % LPG, g = threadIdx.x / LPG;  // QB groups
  const uint64_t nQ = nP / QB, j = (uint64_t)blockIdx.x * QB + g;
  constexpr int UB = V4 ? 16 : 4;
  Row<LPG, NV, V4> acc, r[UB];
  if (j < nQ) {
    acc.zero();
    for (uint32_t i = 0; i < QB; i += UB) {
#pragma unroll
      for (int u = 0; u < UB; ++u) r[u].load(src + (j * QB + i + u) * e, gl, e);
#pragma unroll
      for (int u = 0; u < UB; ++u) acc.add(r[u]);
    }
    acc.store(Q + j * e, gl, e);
  }
  if ((uint64_t)(blockIdx.x + 1) * QB > nQ) return;  // (block-uniform) partial block: no Q2 entry
  __syncthreads();
  if (g != 0) return;
  acc.zero();
  const float* q0 = Q + (uint64_t)blockIdx.x * QB * e;
  for (uint32_t i = 0; i < QB; i += UB) {
#pragma unroll
    for (int u = 0; u < UB; ++u) {  // (written by this block: L2 loads, not the read-only path)
      if (V4) {
        const float4 x = __ldcg(reinterpret_cast<const float4*>(q0 + (i + u) * e) + gl);
        r[u].v[0] = x.x, r[u].v[1] = x.y, r[u].v[2] = x.z, r[u].v[3] = x.w;
      } else {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const uint32_t jj = gl + 32 * q;
          r[u].v[q] = jj < e ? __ldcg(q0 + (i + u) * e + jj) : 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) acc.add(r[u]);
  }
  acc.store(Q2 + (uint64_t)blockIdx.x * e, gl, e);
}

template <int LPG, int NV, bool V4>
__device__ __forceinline__ void sum_p(const float* P, uint64_t lo, uint64_t hi, uint32_t e,
                                      Row<LPG, NV, V4>& acc, int gl) {
  constexpr int UR = V4 ? 16 : 4;  // partial rows in flight (latency-bound tail of hot keys)
  Row<LPG, NV, V4> r[UR];
  for (; lo + UR <= hi; lo += UR) {
#pragma unroll
    for (int u = 0; u < UR; ++u) r[u].load(P + (lo + u) * e, gl, e);
#pragma unroll
    for (int u = 0; u < UR; ++u) acc.add(r[u]);
  }
  for (; lo < hi; ++lo) {
    r[0].load(P + lo * e, gl, e);
    acc.add(r[0]);
  }
}

// chunk c's first position c*CH lies in segment first[c]: one thread per
// chunk, binary search over the segment starts (a per-segment fill would put
// a Zipf-hot key's thousands of chunks on one thread)
__global__ void k_chunk_first(const uint32_t* __restrict__ seg, uint32_t U, uint32_t CH,
                              uint32_t nchunks, uint32_t* __restrict__ first, const uint32_t* __restrict__ dU) {
  if (dU) U = *dU;  // (U on the device only: the sync-free step)
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += gridDim.x * blockDim.x) {
    const uint32_t p0 = c * CH;
    uint32_t lo = 0, hi = U;  // largest u with seg[u] <= p0
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (seg[mid] <= p0) lo = mid;
      else hi = mid;
    }
    first[c] = lo;
  }
}

// Segments crossing a chunk boundary: each is handled once, at the first
// boundary it crosses (c = its start chunk + 1), found through first[c].
template <int LPG, int NV, bool V4>
__global__ void __launch_bounds__(256) k_seg_fix(SegArgs a, TView t, const float* __restrict__ Q,
                                                 const float* __restrict__ Q2) {
  if (aborted(t.abort)) return;
  const int gl = threadIdx.x % LPG;
  const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPG;
  const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / LPG;
  const uint32_t nchunks = (a.n_pos + a.CH - 1) / a.CH;
  for (uint64_t c = 1 + g0; c < nchunks; c += ng) {
    const uint32_t u = a.first[c];
    const uint32_t s0 = a.seg[u], s1 = a.seg[u + 1];
    const uint32_t c0 = s0 / a.CH, c1 = (s1 - 1) / a.CH;
    if (c0 + 1 != c || c1 == c0) continue;
    const uint64_t lo = 2ull * c0 + 1, hi = 2ull * c1 + 1;  // [lo, hi)
    Row<LPG, NV, V4> acc;
    acc.zero();
    if (hi - lo <= 2 * QB) {
      sum_p(a.partials, lo, hi, a.e, acc, gl);
    } else {
      const uint64_t qa = (lo + QB - 1) / QB, qb = hi / QB;
      sum_p(a.partials, lo, qa * QB, a.e, acc, gl);
      if (qb - qa <= 2 * QB) {
        sum_p(Q, qa, qb, a.e, acc, gl);
      } else {  // the hottest keys: a second level of QB-block sums
        const uint64_t q2a = (qa + QB - 1) / QB, q2b = qb / QB;
        sum_p(Q, qa, q2a * QB, a.e, acc, gl);
        sum_p(Q2, q2a, q2b, a.e, acc, gl);
        sum_p(Q, q2b * QB, qb, a.e, acc, gl);
      }
      sum_p(a.partials, qb * QB, hi, a.e, acc, gl);
    }
    finalize(a, t, u, acc, gl);
  }
  if (a.peer) __threadfence_system();
}

template <int LPG, int NV, bool V4>
void launch_seg(const SegArgs& a, const TView& t, float* Q, cudaStream_t s) {
  const uint32_t nchunks = (a.n_pos + a.CH - 1) / a.CH;
  const uint32_t nP = 2 * nchunks;
  static const bool pre_on = [] {  // measured slower at configs[1] (DESIGN 4.1): opt-in
    const char* e = getenv("KP_SEG_PRE");
    return e && e[0] == '1';
  }();
  if constexpr (V4 && LPG >= 8) {
    if (pre_on && a.CH <= 64) {
      k_seg_chunks_pre<LPG, NV, V4><<<grid_cap(((uint64_t)nchunks * LPG + 255) / 256), 256, 0, s>>>(a, t);
      ::kp::count_launch();
    } else {
      k_seg_chunks<LPG, NV, V4><<<grid_cap(((uint64_t)nchunks * LPG + 255) / 256), 256, 0, s>>>(a, t);
      ::kp::count_launch();
    }
  } else {
    k_seg_chunks<LPG, NV, V4><<<grid_cap(((uint64_t)nchunks * LPG + 255) / 256), 256, 0, s>>>(a, t);
    ::kp::count_launch();
  }
  const uint32_t nQ = nP / QB;
  float* Q2 = Q + (uint64_t)(nQ + 1) * a.e;
  const char* bs_env = getenv("KP_SEG_BS12");  // =0: the two block-sum levels as two launches
  const bool one = LPG <= 4 && !(bs_env && bs_env[0] == '0');
  if (nQ && one) {
    k_seg_blocksum12<LPG, NV, V4><<<(nQ + QB - 1) / QB, QB * LPG, 0, s>>>(a.partials, nP, a.e, Q, Q2);
    ::kp::count_launch();
  } else if (nQ) {
    k_seg_blocksum<LPG, NV, V4><<<grid_cap(((uint64_t)nQ * LPG + 255) / 256), 256, 0, s>>>(a.partials, nP, a.e, Q); ::kp::count_launch();
  }
  if (nQ >= QB && !one) {
    k_seg_blocksum<LPG, NV, V4><<<grid_cap(((uint64_t)(nQ / QB) * LPG + 255) / 256), 256, 0, s>>>(Q, nQ, a.e, Q2); ::kp::count_launch();
  }
  if (nchunks > 1) {
    k_seg_fix<LPG, NV, V4><<<grid_cap(((uint64_t)nchunks * LPG + 255) / 256), 256, 0, s>>>(a, t, Q, Q2); ::kp::count_launch();
  }
}

template <int LPG, int NV, bool V4>
void launch_pool(const uint32_t* bag_offs, uint32_t n_bags, const uint32_t* rowocc,
                 const float* src, uint32_t e, bool mean, float* pooled, float* inv_count,
                 float* inst_max, uint32_t S, cudaStream_t s) {
  if (inst_max && S >= 2 * PB && LPG <= 16) {
    const uint32_t n_inst = n_bags / S;
    k_pool_inst<LPG, NV, V4><<<grid_cap(((uint64_t)n_inst * 32 + 255) / 256), 256, 0, s>>>(
        bag_offs, n_inst, S, rowocc, src, e, mean ? 1 : 0, pooled, inv_count, inst_max); ::kp::count_launch();
    return;
  }
  if (inst_max) KP_CUDA(cudaMemsetAsync(inst_max, 0, (size_t)(n_bags / S) * 4, s));
  k_pool<LPG, NV, V4><<<grid_cap(((uint64_t)(n_bags + PB - 1) / PB * LPG + 255) / 256), 256, 0, s>>>(
      bag_offs, n_bags, rowocc, src, e, mean ? 1 : 0, pooled, inv_count,
      reinterpret_cast<unsigned*>(inst_max), S); ::kp::count_launch();
}

// Dispatch on the embedding width: float4 groups for e in {4,8,...,128},
// 32-lane scalar groups otherwise (e <= 256).
template <template <int, int, bool> class F, class... Args>
void dispatch_e(uint32_t e, Args&&... args) {
  switch (e) {
    case 4: F<1, 4, true>::run(args...); return;
    case 8: F<2, 4, true>::run(args...); return;
    case 16: F<4, 4, true>::run(args...); return;
    case 32: F<8, 4, true>::run(args...); return;
    case 64: F<16, 4, true>::run(args...); return;
    case 128: F<32, 4, true>::run(args...); return;
    default: break;
  }
  KP_CHECK(e <= 256, kErrConfig, "embedding_dim > 256 not supported");
  if (e <= 32) F<32, 1, false>::run(args...);
  else if (e <= 64) F<32, 2, false>::run(args...);
  else if (e <= 128) F<32, 4, false>::run(args...);
  else F<32, 8, false>::run(args...);
}

template <int LPG, int NV, bool V4>
struct PoolF {
  template <class... A>
  static void run(A... a) { launch_pool<LPG, NV, V4>(a...); }
};
template <int LPG, int NV, bool V4>
struct SegF {
  static void run(const SegArgs& a, const TView& t, float* Q, cudaStream_t s) {
    launch_seg<LPG, NV, V4>(a, t, Q, s);
  }
};

__global__ void k_gather_rows(const float* __restrict__ src, const uint32_t* __restrict__ idx,
                              uint32_t n, uint32_t e, float* __restrict__ out) {
  const uint64_t total = (uint64_t)n * e;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = q / e, j = q % e;
    out[q] = idx[i] == kNoRow ? 0.f : src[(uint64_t)idx[i] * e + j];
  }
}

}  // namespace

void prepare_bags(const uint32_t* d_offs, uint32_t occ_base, const uint16_t* d_slots,
                  uint32_t n_inst, uint32_t S, uint32_t* d_bag_offs, uint32_t* d_bag_of_occ,
                  uint32_t* d_err, cudaStream_t s, uint32_t* d_abort, bool maps) {
  KP_CUDA(cudaMemsetAsync(d_err + 1, 0xFF, 4, s));
  k_prepare_bags<<<grid_cap(((uint64_t)n_inst * 32 + 255) / 256), 256, 0, s>>>(
      d_offs, occ_base, d_slots, n_inst, S, d_bag_offs, d_bag_of_occ, d_err, d_abort, maps ? 1 : 0); ::kp::count_launch();
}

void compose(const uint32_t* d_idx, const uint32_t* d_inverse, uint32_t n, uint32_t* d_out,
             cudaStream_t s) {
  if (n == 0) return;
  k_compose<<<grid_cap(((uint64_t)n + 255) / 256), 256, 0, s>>>(d_idx, d_inverse, n, d_out); ::kp::count_launch();
}

void pool(const uint32_t* d_bag_offs, uint32_t n_bags, const uint32_t* d_row_of_occ,
          const float* d_src, uint32_t e, bool mean, float* d_pooled, float* d_inv_count,
          cudaStream_t s, float* d_inst_max, uint32_t S) {
  if (n_bags == 0) return;
  dispatch_e<PoolF>(e, d_bag_offs, n_bags, d_row_of_occ, d_src, e, mean, d_pooled, d_inv_count,
                    d_inst_max, S, s);
}

// one feature per slot, 256 < S*e/4 <= 2048 cells: k_pool_planes_ident
bool planes_ident_kernel(uint32_t S, uint32_t e) {
  const uint32_t cells = S * e / 4;
  return cells > 256 && cells <= 256 * 8 && S <= 256;
}

bool pool_planes_supported(uint32_t S, uint32_t e) {
  return e % 4 == 0 && e <= 128 && (S * e) % 8 == 0 && S * e / 4 <= 256 * 16;
}

void pool_planes(const uint32_t* d_bag_offs, uint32_t n_inst, uint32_t S, const uint32_t* d_row_of_occ,
                 const float* d_src, uint32_t e, bool mean, __half* d_hi, __half* d_lo, int* d_inst_exp,
                 float* d_inv_count, cudaStream_t s, bool ident, const uint32_t* d_inverse) {
  KP_CHECK(pool_planes_supported(S, e), kErrConfig, "pool_planes: unsupported S*e");
  KP_CHECK(!d_inverse || (ident && planes_ident_kernel(S, e)), kErrGeneric,
           "pool_planes: the unique -> row map form is for one feature per slot");
  if (n_inst == 0) return;
  const uint32_t cells = S * e / 4;
  if (ident && planes_ident_kernel(S, e)) {
    const unsigned grid = (unsigned)std::min<uint64_t>(n_inst, 148ull * 4);
    if (cells <= 256 * 4)
      k_pool_planes_ident<256, 4><<<grid, 256, 0, s>>>(n_inst, S, d_row_of_occ, d_inverse, d_src, e, d_hi, d_lo,
                                                        d_inst_exp, d_inv_count, mean ? 1 : 0);
    else
      k_pool_planes_ident<256, 8><<<grid, 256, 0, s>>>(n_inst, S, d_row_of_occ, d_inverse, d_src, e, d_hi, d_lo,
                                                        d_inst_exp, d_inv_count, mean ? 1 : 0);
    ::kp::count_launch();
    return;
  }
  const unsigned grid = (unsigned)std::min<uint64_t>(n_inst, 148ull * 64);
  // threads per instance: the cells rounded up to warps (<= 256), then the
  // fewest float4 cells per thread that cover the row
  if (cells <= 64) {
    k_pool_planes<64, 1><<<grid, 64, 0, s>>>(d_bag_offs, n_inst, S, d_row_of_occ, d_src, e, mean, d_hi, d_lo,
                                              d_inst_exp, d_inv_count);
  } else if (cells <= 256) {
    k_pool_planes<256, 1><<<grid, 256, 0, s>>>(d_bag_offs, n_inst, S, d_row_of_occ, d_src, e, mean, d_hi, d_lo,
                                                d_inst_exp, d_inv_count);
  } else if (cells <= 256 * 4) {
    k_pool_planes<256, 4><<<grid, 256, 0, s>>>(d_bag_offs, n_inst, S, d_row_of_occ, d_src, e, mean, d_hi, d_lo,
                                                d_inst_exp, d_inv_count);
  } else if (cells <= 256 * 8) {
    k_pool_planes<256, 8><<<grid, 256, 0, s>>>(d_bag_offs, n_inst, S, d_row_of_occ, d_src, e, mean, d_hi, d_lo,
                                                d_inst_exp, d_inv_count);
  } else {
    k_pool_planes<256, 16><<<grid, 256, 0, s>>>(d_bag_offs, n_inst, S, d_row_of_occ, d_src, e, mean, d_hi, d_lo,
                                                 d_inst_exp, d_inv_count);
  }
  ::kp::count_launch();
}

void inst_exps_ident(const float* d_src, const uint32_t* d_idx, uint32_t U, uint32_t e,
                     const uint32_t* d_inverse, uint32_t n_inst, uint32_t S, float* d_umax_ws,
                     int* d_inst_exp, float* d_inv_count, bool mean, cudaStream_t s) {
  KP_CHECK(e % 4 == 0 && e <= 128, kErrConfig, "inst_exps_ident: e must be a multiple of 4, <= 128");
  if (n_inst == 0) return;
  if (U) {
    const uint64_t per = 32 / (e / 4);
    k_unique_maxabs<<<grid_cap(((U + per - 1) / per * 32 + 255) / 256), 256, 0, s>>>(d_src, d_idx, U, e, d_umax_ws);
    ::kp::count_launch();
  }
  k_inst_exp<<<grid_cap(((uint64_t)n_inst * 32 + 255) / 256), 256, 0, s>>>(d_inverse, d_umax_ws, n_inst, S,
                                                                           d_inst_exp, d_inv_count, mean ? 1 : 0);
  ::kp::count_launch();
}

void seg_reduce_apply(const uint32_t* d_seg, uint32_t n_unique, const uint32_t* d_sorted_vals,
                      const uint32_t* d_bag_of_occ, uint32_t n_pos, const float* d_rows_src,
                      uint32_t e, float inv_n, Table* t, const uint32_t* d_table_rows,
                      const SparseRule& r, float* d_grad_out, const uint32_t* d_out_idx,
                      SegWs& ws, cudaStream_t s, const PeerMap* pm,
                      const uint32_t* d_nunique) {
  if (n_unique == 0 || n_pos == 0) return;
  SegArgs a;
  a.seg = d_seg;
  a.U = n_unique;
  a.sorted_vals = d_sorted_vals;
  a.bag_of_occ = d_bag_of_occ;
  a.n_pos = n_pos;
  a.rows_src = d_rows_src;
  a.e = e;
  a.inv_n = inv_n;
  a.table_rows = d_table_rows;
  a.grad_out = d_grad_out;
  a.out_idx = d_out_idx;
  // chunk length: 64 positions, shorter for small batches so the
  // latency-bound chunk walks still fill the GPU (C1: 106K positions -> 4)
  // (floor 4: configs[0]'s 106K positions -> 26.6K chunks, push 61 -> 55 us
  // against a floor of 8; KP_SEG_MINCH overrides)
  static const uint32_t min_ch = [] {
    const char* e = getenv("KP_SEG_MINCH");
    const int v = e ? atoi(e) : 4;
    return (uint32_t)(v >= 1 && v <= 64 ? v : 4);
  }();
  a.CH = 64;
  while (a.CH > min_ch && n_pos / a.CH < 148u * 128u) a.CH /= 2;
  const uint32_t nchunks = (n_pos + a.CH - 1) / a.CH;
  a.partials = ws.partials.get<float>((size_t)nchunks * 2 * e);
  uint32_t* first = ws.first.get<uint32_t>(nchunks);
  k_chunk_first<<<grid_cap(((uint64_t)nchunks + 255) / 256), 256, 0, s>>>(d_seg, n_unique, a.CH, nchunks, first,
                                                                           d_nunique); ::kp::count_launch();
  a.first = first;
  a.apply = t != nullptr;
  a.peer = pm != nullptr;
  if (pm) a.pm = *pm;
  a.rule = r.rule;
  a.lr = r.lr;
  a.b1 = r.beta1;
  a.b2 = r.beta2;
  TView tv{};
  if (t) tv = view(t);
  float* Q = ws.qsums.get<float>((size_t)(2 * nchunks / QB + 1 + 2 * nchunks / QB / QB + 1) * e);
  dispatch_e<SegF>(e, a, tv, Q, s);
}

void gather_rows(const float* d_src, const uint32_t* d_idx, uint32_t n, uint32_t e, float* d_out,
                 cudaStream_t s) {
  if (n == 0) return;
  k_gather_rows<<<grid_cap(((uint64_t)n * e + 255) / 256), 256, 0, s>>>(d_src, d_idx, n, e, d_out); ::kp::count_launch();
}

}  // namespace kp
