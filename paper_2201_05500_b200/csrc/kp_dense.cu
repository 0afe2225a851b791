// Dense k-step Adam: local step, moment accumulation, fixed-order centered
// mean merge, state checks; plus the host-side dense initializer.
//
// Reference: accumulate_moments / local_adam_step / global_merge
// (proj/src/optimizer.cpp:39-84), centered_mean_vectors
// (proj/include/kpsim/common.hpp:27-45), KStepEngine::step checks
// (proj/src/optimizer.cpp:135-142), CtrModel::init_dense (model.cpp:68-74).
// Every kernel keeps the reference's expression tree with round-to-nearest
// intrinsics (no FMA contraction): the fp32 results are bit-identical to the
// fp32 oracle given the same gradients, and the centered mean makes N identical
// replicas bit-identical to one (the replica-invariance contract).
#include <cmath>

#include "kp_internal.cuh"

namespace kp {
namespace {

unsigned grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 148ull * 16) g = 148ull * 16;
  return (unsigned)g;
}

__device__ __forceinline__ void moments(float& m, float& v, float g, float b1, float b2) {
  m = __fadd_rn(__fmul_rn(b1, m), __fmul_rn(__fsub_rn(1.f, b1), g));
  v = __fadd_rn(__fmul_rn(b2, v), __fmul_rn(__fsub_rn(1.f, b2), __fmul_rn(g, g)));
}

__global__ void k_local_step(float* __restrict__ x, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ vbar, const float* __restrict__ g,
                             uint64_t D, float alpha, float b1, float b2, const uint32_t* abort) {
  if (aborted(abort)) return;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x) {
    float mj = m[j], vj = v[j];
    moments(mj, vj, g[j], b1, b2);
    m[j] = mj;
    v[j] = vj;
    x[j] = __fsub_rn(x[j], __fdiv_rn(__fmul_rn(alpha, mj), __fsqrt_rn(vbar[j])));
  }
}

__global__ void k_moments(float* __restrict__ m, float* __restrict__ v, const float* __restrict__ g,
                          uint64_t D, float b1, float b2, const uint32_t* abort) {
  if (aborted(abort)) return;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x) {
    float mj = m[j], vj = v[j];
    moments(mj, vj, g[j], b1, b2);
    m[j] = mj;
    v[j] = vj;
  }
}

// base + sum_i (v_i - base) / n, ascending i (common.hpp:27-45)
__global__ void k_cmean(const float* __restrict__ vecs, uint64_t stride, uint32_t n, uint64_t D,
                        float* __restrict__ out, const uint32_t* abort) {
  if (aborted(abort)) return;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const float base = vecs[j];
    float acc = 0.f;
    for (uint32_t i = 0; i < n; ++i) acc = __fadd_rn(acc, __fsub_rn(vecs[i * stride + j], base));
    out[j] = __fadd_rn(base, __fdiv_rn(acc, (float)n));
  }
}

__global__ void k_terms(const float* __restrict__ x, const float* __restrict__ m,
                        const float* __restrict__ vbar, uint64_t D, float alpha,
                        float* __restrict__ out, const uint32_t* abort) {
  if (aborted(abort)) return;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = __fsub_rn(x[j], __fdiv_rn(__fmul_rn(alpha, m[j]), __fsqrt_rn(vbar[j])));
}

// One worker on one rank: the whole merge in one pass, the same expression
// tree as k_cmean (n = 1) -> k_terms -> k_cmean (n = 1) -> copies, so the
// result is bitwise the general path's (including x = -0 -> +0).
__global__ void k_merge_single(float* __restrict__ x, const float* __restrict__ m,
                               float* __restrict__ v, float* __restrict__ vbar, uint64_t D,
                               float alpha, int reset, const uint32_t* abort) {
  if (aborted(abort)) return;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const float vj = v[j];
    const float vb = __fadd_rn(vj, __fdiv_rn(__fadd_rn(0.f, __fsub_rn(vj, vj)), 1.f));
    const float t = __fsub_rn(x[j], __fdiv_rn(__fmul_rn(alpha, m[j]), __fsqrt_rn(vb)));
    x[j] = __fadd_rn(t, __fdiv_rn(__fadd_rn(0.f, __fsub_rn(t, t)), 1.f));
    vbar[j] = vb;
    if (reset) v[j] = vb;
  }
}

__global__ void k_copy(float* __restrict__ dst, const float* __restrict__ src, uint64_t D,
                       const uint32_t* abort) {
  if (aborted(abort)) return;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x)
    dst[j] = src[j];
}

// bit 0: non-finite x or v; bit 1: v or v_bar lost positivity (optimizer.cpp:135-142)
// done (nullable): +1 once per call unless the step was aborted -- the count
// of steps that applied their updates (the host rolls its counters back to it)
__global__ void k_check(const float* __restrict__ v, const float* __restrict__ vbar,
                        const float* __restrict__ x, uint64_t D, uint32_t* flag, uint32_t* done,
                        const uint32_t* abort) {
  if (done && blockIdx.x == 0 && threadIdx.x == 0 && !aborted(abort)) atomicAdd(done, 1u);
  uint32_t f = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x) {
    if (!isfinite(x[j]) || !isfinite(v[j])) f |= 1;
    if (!(v[j] > 0.f) || !(vbar[j] > 0.f)) f |= 2;
  }
  if (f) atomicOr(flag, f);
}

// One worker on one GPU, the whole dense step in one pass: moments, then the
// local step or the single-worker merge, then the state checks -- the same
// expression trees as k_moments / k_local_step / k_merge_single / k_check in
// sequence (bitwise their results), one read and write of each vector.
__global__ void k_dense_step_single(float* __restrict__ x, float* __restrict__ m, float* __restrict__ v,
                                    float* __restrict__ vbar, const float* __restrict__ g, uint64_t D,
                                    float alpha, float b1, float b2, int merge, int reset, uint32_t* flag,
                                    uint32_t* done, const uint32_t* abort) {
  if (aborted(abort)) return;
  if (done && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(done, 1u);
  uint32_t f = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < D;
       j += (uint64_t)gridDim.x * blockDim.x) {
    float mj = m[j], vj = v[j], xj = x[j], vb;
    moments(mj, vj, g[j], b1, b2);
    if (!merge) {
      vb = vbar[j];
      xj = __fsub_rn(xj, __fdiv_rn(__fmul_rn(alpha, mj), __fsqrt_rn(vb)));
    } else {
      vb = __fadd_rn(vj, __fdiv_rn(__fadd_rn(0.f, __fsub_rn(vj, vj)), 1.f));
      const float t = __fsub_rn(xj, __fdiv_rn(__fmul_rn(alpha, mj), __fsqrt_rn(vb)));
      xj = __fadd_rn(t, __fdiv_rn(__fadd_rn(0.f, __fsub_rn(t, t)), 1.f));
      vbar[j] = vb;
      if (reset) vj = vb;
    }
    m[j] = mj;
    v[j] = vj;
    x[j] = xj;
    if (!isfinite(xj) || !isfinite(vj)) f |= 1;
    if (!(vj > 0.f) || !(vb > 0.f)) f |= 2;
  }
  if (f) atomicOr(flag, f);
}

}  // namespace

void dense_step_single(float* x, float* m, float* v, float* vbar, const float* g, uint64_t D, const AdamParams& h,
                       bool merge, bool reset, uint32_t* d_flag, uint32_t* d_done, cudaStream_t s) {
  k_dense_step_single<<<grid_for(D), 256, 0, s>>>(x, m, v, vbar, g, D, h.alpha, h.beta1, h.beta2, merge ? 1 : 0,
                                                  reset ? 1 : 0, d_flag, d_done, g_abort); ::kp::count_launch();
}

void dense_local_step(float* x, float* m, float* v, const float* vbar, const float* g, uint64_t D,
                      const AdamParams& h, cudaStream_t s) {
  k_local_step<<<grid_for(D), 256, 0, s>>>(x, m, v, vbar, g, D, h.alpha, h.beta1, h.beta2, g_abort); ::kp::count_launch();
}
void dense_moments(float* m, float* v, const float* g, uint64_t D, const AdamParams& h,
                   cudaStream_t s) {
  k_moments<<<grid_for(D), 256, 0, s>>>(m, v, g, D, h.beta1, h.beta2, g_abort); ::kp::count_launch();
}
void centered_mean(const float* vecs, uint64_t stride, uint32_t n, uint64_t D, float* out,
                   cudaStream_t s) {
  k_cmean<<<grid_for(D), 256, 0, s>>>(vecs, stride, n, D, out, g_abort); ::kp::count_launch();
}
void merge_single(float* x, const float* m, float* v, float* vbar, uint64_t D, float alpha,
                  bool reset, cudaStream_t s) {
  k_merge_single<<<grid_for(D), 256, 0, s>>>(x, m, v, vbar, D, alpha, reset ? 1 : 0, g_abort); ::kp::count_launch();
}
void merge_terms(const float* x, const float* m, const float* vbar, uint64_t D, float alpha,
                 float* out, cudaStream_t s) {
  k_terms<<<grid_for(D), 256, 0, s>>>(x, m, vbar, D, alpha, out, g_abort); ::kp::count_launch();
}
void dense_copy(float* dst, const float* src, uint64_t D, cudaStream_t s) {
  k_copy<<<grid_for(D), 256, 0, s>>>(dst, src, D, g_abort); ::kp::count_launch();
}
void dense_check(const float* v, const float* vbar, const float* x, uint64_t D, uint32_t* d_flag,
                 cudaStream_t s, uint32_t* d_done) {
  k_check<<<grid_for(D), 256, 0, s>>>(v, vbar, x, D, d_flag, d_done, g_abort); ::kp::count_launch();
}

uint64_t splitmix64_host(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// std::mt19937_64 + libstdc++'s uniform_real_distribution<double>(-0.05, 0.05):
// generate_canonical from one 64-bit draw, u*(b-a)+a.
void init_dense_host(uint64_t seed, uint64_t dim, double* out) {
  uint64_t mt[312];
  int idx = 312;
  mt[0] = splitmix64_host(seed ^ 0xD15EA5E0ULL);
  for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
  for (uint64_t q = 0; q < dim; ++q) {
    if (idx >= 312) {
      for (int i = 0; i < 312; ++i) {
        const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
        uint64_t xa = x >> 1;
        if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
        mt[i] = mt[(i + 156) % 312] ^ xa;
      }
      idx = 0;
    }
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    double u = (double)y / 18446744073709551616.0;
    if (u >= 1.0) u = std::nextafter(1.0, 0.0);
    out[q] = u * (0.05 - -0.05) + -0.05;
  }
}

}  // namespace kp
