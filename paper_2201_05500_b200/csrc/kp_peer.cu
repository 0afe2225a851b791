// NVLink peer-memory exchange (G > 1, one process per GPU).
//
// The reference exchanges nothing (one process, trainer.cpp:163,180-186 sums
// worker gradients in a std::map); the B200 design shards the table by
// key % G and moves keys, rows and gradients between GPUs.
// Instead of staging into send buffers for an NCCL all-to-all, the producing
// kernels store their output directly into the destination rank's exchange
// window (CUDA IPC mapping, NVSwitch P2P), so the transfer overlaps the
// kernel's own HBM-bound work:
//   keys   unique keys in owner order      -> owner's key window
//   rows   owner's table rows               -> requester's row window
//   grads  per-unique reduced gradients     -> owner's gradient window
//          (stored by the segmented reduction's finalize, kp_embed.cu)
// Completion is a per-(phase, source) sequence flag written with a
// system-scope release after the data; the consumer spins on its own flags
// (bounded, error bit instead of a hang) before reading the window.
#include <cstdlib>

#include "kp_internal.cuh"

namespace kp {
namespace {

__global__ void k_send_keys(const uint64_t* __restrict__ unique, const uint32_t* __restrict__ perm,
                            uint32_t n, PeerMap pm) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    *reinterpret_cast<uint64_t*>(peer_dst(pm, t)) = unique[perm[t]];
  __threadfence_system();
}

// one 16-lane group per row, float4 lanes (e % 4 == 0) or scalar fallback
__global__ void k_send_rows(const float* __restrict__ src, const uint32_t* __restrict__ idx,
                            uint32_t n, uint32_t e, PeerMap pm) {
  const uint32_t gl = threadIdx.x & 15;
  const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 4;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) >> 4;
  const bool v4 = (e & 3) == 0;
  for (uint64_t i = g0; i < n; i += ng) {
    float* dst = reinterpret_cast<float*>(peer_dst(pm, (uint32_t)i));
    const uint32_t r = idx[i];
    if (v4) {
      const float4* sp = reinterpret_cast<const float4*>(src + (uint64_t)r * e);
      for (uint32_t j = gl; j < e / 4; j += 16)
        reinterpret_cast<float4*>(dst)[j] = r == kNoRow ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(sp + j);
    } else {
      for (uint32_t j = gl; j < e; j += 16) dst[j] = r == kNoRow ? 0.f : __ldg(src + (uint64_t)r * e + j);
    }
  }
  __threadfence_system();
}

__global__ void k_signal(PeerFlags f, int R, uint64_t seq) {
  const int p = threadIdx.x;
  __threadfence_system();
  if (p < R) {
    volatile unsigned long long* q = reinterpret_cast<volatile unsigned long long*>(f.flag[p]);
    *q = seq;
  }
  __threadfence_system();
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until every peer's flag reached seq. A peer that never signals (gone,
// or slower than timeout_ns of wall time -- KP_PEER_TIMEOUT_S, default 120 s)
// sets kAbortTimeout in *err instead of hanging the stream: every later
// state-writing kernel of the step then returns without writing (aborted()),
// and the host raises at the batch-end readback.
__global__ void k_wait(const uint64_t* flags, int R, uint64_t seq, uint32_t* err, uint64_t timeout_ns) {
  const int p = threadIdx.x;
  if (p < R) {
    const volatile unsigned long long* q = reinterpret_cast<const volatile unsigned long long*>(flags + p);
    const uint64_t t0 = globaltimer_ns();
    while (*q < seq) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicOr(err, kAbortTimeout);
        break;
      }
      __nanosleep(256);
    }
  }
  __threadfence_system();
}

// centered mean over all N = R*W global workers of elements [c0, c1):
// worker i = (rank p, local l) at src[p] + l*D (remote loads over NVLink),
// result stored into dst[p] of every rank (remote stores). Same expression
// tree and worker order as k_cmean (common.hpp:27-45).
__global__ void k_cmean_peer(PeerVecs pv, int R, uint32_t W, uint64_t D, uint64_t c0, uint64_t c1,
                             const uint32_t* abort) {
  if (aborted(abort)) return;
  const float n = (float)(R * W);
  for (uint64_t j = c0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < c1;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const float base = reinterpret_cast<const float*>(pv.src[0])[j];
    float acc = 0.f;
    for (int p = 0; p < R; ++p) {
      const float* sp = reinterpret_cast<const float*>(pv.src[p]);
      for (uint32_t l = 0; l < W; ++l) acc = __fadd_rn(acc, __fsub_rn(sp[(uint64_t)l * D + j], base));
    }
    const float r = __fadd_rn(base, __fdiv_rn(acc, n));
    for (int p = 0; p < R; ++p) reinterpret_cast<float*>(pv.dst[p])[j] = r;
  }
  __threadfence_system();
}

// k_cmean_peer (v) -> merge_terms on every rank -> k_cmean_peer (terms) in
// one kernel: the owner of chunk [c0, c1) reads every rank's v, x and m
// there, so the merge needs one exchange round instead of two; the same
// expression trees and worker order, so the result is bitwise the two-round
// one's. It writes only its own chunk of every rank's x (worker 0), which no
// other owner reads.
__global__ void k_merge_peer(PeerMerge pm, int R, uint32_t W, uint64_t D, uint64_t c0, uint64_t c1, float alpha,
                             const uint32_t* abort) {
  if (aborted(abort)) return;
  const float n = (float)(R * W);
  for (uint64_t j = c0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < c1;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const float vbase = reinterpret_cast<const float*>(pm.v[0])[j];
    float acc = 0.f;
    for (int p = 0; p < R; ++p) {
      const float* vp = reinterpret_cast<const float*>(pm.v[p]);
      for (uint32_t l = 0; l < W; ++l) acc = __fadd_rn(acc, __fsub_rn(vp[(uint64_t)l * D + j], vbase));
    }
    const float vb = __fadd_rn(vbase, __fdiv_rn(acc, n));
    const float sq = __fsqrt_rn(vb);
    auto term = [&](int p, uint32_t l) {
      const float xv = reinterpret_cast<const float*>(pm.x[p])[(uint64_t)l * D + j];
      const float mv = reinterpret_cast<const float*>(pm.m[p])[(uint64_t)l * D + j];
      return __fsub_rn(xv, __fdiv_rn(__fmul_rn(alpha, mv), sq));
    };
    const float tbase = term(0, 0);
    float tacc = 0.f;
    for (int p = 0; p < R; ++p)
      for (uint32_t l = 0; l < W; ++l) tacc = __fadd_rn(tacc, __fsub_rn(term(p, l), tbase));
    const float xb = __fadd_rn(tbase, __fdiv_rn(tacc, n));
    for (int p = 0; p < R; ++p) {
      reinterpret_cast<float*>(pm.vb[p])[j] = vb;
      reinterpret_cast<float*>(pm.x[p])[j] = xb;
    }
  }
  __threadfence_system();
}

// The same with RW = R * W <= 8 known at compile time: each element's R*W
// remote v loads are issued together, then its R*W x and m loads, so one
// element costs two NVLink round trips instead of 3*R*W dependent ones. The
// adds run in the same (rank, worker) order: bitwise k_merge_peer's result.
template <int RW>
__global__ void k_merge_peer_rw(PeerMerge pm, uint32_t W, uint64_t D, uint64_t c0, uint64_t c1, float alpha,
                                const uint32_t* abort) {
  if (aborted(abort)) return;
  const float n = (float)RW;
  const float* vp[RW];
  const float* xp[RW];
  const float* mp[RW];
#pragma unroll
  for (int i = 0; i < RW; ++i) {
    const uint32_t p = i / W, l = i % W;
    vp[i] = reinterpret_cast<const float*>(pm.v[p]) + (uint64_t)l * D;
    xp[i] = reinterpret_cast<const float*>(pm.x[p]) + (uint64_t)l * D;
    mp[i] = reinterpret_cast<const float*>(pm.m[p]) + (uint64_t)l * D;
  }
  for (uint64_t j = c0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < c1;
       j += (uint64_t)gridDim.x * blockDim.x) {
    float vv[RW], xv[RW], mv[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) vv[i] = vp[i][j];
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      xv[i] = xp[i][j];
      mv[i] = mp[i][j];
    }
    const float vbase = vv[0];
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < RW; ++i) acc = __fadd_rn(acc, __fsub_rn(vv[i], vbase));
    const float vb = __fadd_rn(vbase, __fdiv_rn(acc, n));
    const float sq = __fsqrt_rn(vb);
    float t[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) t[i] = __fsub_rn(xv[i], __fdiv_rn(__fmul_rn(alpha, mv[i]), sq));
    float tacc = 0.f;
#pragma unroll
    for (int i = 0; i < RW; ++i) tacc = __fadd_rn(tacc, __fsub_rn(t[i], t[0]));
    const float xb = __fadd_rn(t[0], __fdiv_rn(tacc, n));
#pragma unroll
    for (int i = 0; i < RW; i += (int)W) {
      const uint32_t p = i / W;
      reinterpret_cast<float*>(pm.vb[p])[j] = vb;
      reinterpret_cast<float*>(pm.x[p])[j] = xb;
    }
  }
  __threadfence_system();
}

}  // namespace

void peer_merge(const PeerMerge& pm, int R, uint32_t W, uint64_t D, uint64_t c0, uint64_t c1, float alpha,
                cudaStream_t s) {
  if (c1 <= c0) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((c1 - c0 + 255) / 256, 148 * 8);
  static const bool rw_on = [] {
    const char* e = getenv("KP_MERGE_RW");
    return !(e && e[0] == '0');
  }();
  const uint64_t rw = (uint64_t)R * W;
#define KP_MERGE_RW_CASE(N) \
  case N: k_merge_peer_rw<N><<<grid, 256, 0, s>>>(pm, W, D, c0, c1, alpha, g_abort); break;
  if (rw_on && rw <= 8) {
    switch (rw) {
      KP_MERGE_RW_CASE(1) KP_MERGE_RW_CASE(2) KP_MERGE_RW_CASE(3) KP_MERGE_RW_CASE(4)
      KP_MERGE_RW_CASE(5) KP_MERGE_RW_CASE(6) KP_MERGE_RW_CASE(7) KP_MERGE_RW_CASE(8)
    }
  } else {
    k_merge_peer<<<grid, 256, 0, s>>>(pm, R, W, D, c0, c1, alpha, g_abort);
  }
#undef KP_MERGE_RW_CASE
  ::kp::count_launch();
}

void peer_cmean(const PeerVecs& pv, int R, uint32_t W, uint64_t D, uint64_t c0, uint64_t c1,
                cudaStream_t s) {
  if (c1 <= c0) return;
  k_cmean_peer<<<(unsigned)std::min<uint64_t>((c1 - c0 + 255) / 256, 148 * 8), 256, 0, s>>>(pv, R, W, D, c0, c1, g_abort); ::kp::count_launch();
}

void peer_send_keys(const uint64_t* d_unique, const uint32_t* d_perm, uint32_t n, const PeerMap& pm,
                    cudaStream_t s) {
  if (n == 0) return;
  k_send_keys<<<std::min<uint32_t>(ceil_div(n, 256), 148 * 8), 256, 0, s>>>(d_unique, d_perm, n, pm); ::kp::count_launch();
}

void peer_send_rows(const float* d_src, const uint32_t* d_idx, uint32_t n, uint32_t e,
                    const PeerMap& pm, cudaStream_t s) {
  if (n == 0) return;
  const uint64_t groups = n;
  k_send_rows<<<(unsigned)std::min<uint64_t>((groups * 16 + 255) / 256, 148 * 16), 256, 0, s>>>(
      d_src, d_idx, n, e, pm); ::kp::count_launch();
}

void peer_signal(const PeerFlags& f, int R, uint64_t seq, cudaStream_t s) {
  k_signal<<<1, 32, 0, s>>>(f, R, seq); ::kp::count_launch();
}

void peer_wait(const uint64_t* d_my_flags, int R, uint64_t seq, uint32_t* d_err, cudaStream_t s) {
  static const uint64_t timeout_ns = [] {
    const char* e = getenv("KP_PEER_TIMEOUT_S");
    const double sec = e ? atof(e) : 120.0;
    return (uint64_t)((sec > 0 ? sec : 120.0) * 1e9);
  }();
  k_wait<<<1, 32, 0, s>>>(d_my_flags, R, seq, d_err, timeout_ns); ::kp::count_launch();
}

}  // namespace kp
