// Dense MLP forward/backward over pooled embeddings (fp32).
//
// Reference: CtrModel::forward/backward (proj/src/model.cpp:76-191); flat dense
// layout per layer W(out x in, row-major) then bias (:55-66); hidden
// activation relu/tanh, linear logit head, sigmoid, mean BCE (:34-38,126-135);
// upstream (p - y)/n with n the worker's minibatch size (:153-155).
//
// GEMMs: the first layer (the wide S*e contraction) runs on the 3xFP16
// tcgen05 kernel over pre-split fp16 planes (kp_gemm_h3.cu) when the pooling
// kernel wrote its output as planes, else on the on-chip-split tcgen05
// kernels (kp_gemm_tc.cu: 3xFP16 forward/dX, 3xTF32 dW); the other layers on
// 3xTF32 tcgen05. Products below KP_TC_MIN_MFLOP (512 MFLOP: every layer of
// configs[0]) run on the small-tile fp32 SIMT GEMM (k_gemm_s, 32x64 tiles),
// where a tcgen05 launch costs more than the arithmetic; the 128x128x8 SIMT
// GEMM is the fallback for shapes TMA cannot describe.
// Epilogues are fused (bias+activation, activation derivative, mean-pooling
// coefficient); weight gradients use deterministic split-K; the out=1 head
// is a warp-per-instance GEMV fused with sigmoid, loss and the upstream
// gradient.
#include <cstdlib>

#include <cuda_fp16.h>

#include "kp_internal.cuh"

namespace kp {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, GT = 256;

enum Epi : int { kStore = 0, kBiasAct = 1, kDAct = 2, kCoeff = 3 };

using EpiArgs = GemmEpi;

__device__ __forceinline__ float act_fwd(int act, float z) {
  return act == 0 ? (z > 0.f ? z : 0.f) : tanhf(z);
}
// derivative from the layer OUTPUT y (relu: y>0 <=> z>0; tanh: 1-y^2), model.cpp:45-51
__device__ __forceinline__ float act_bwd(int act, float y) {
  return act == 0 ? (y > 0.f ? 1.f : 0.f) : __fsub_rn(1.f, __fmul_rn(y, y));
}

// C[m][n] (+ split offset) = sum_k A(m,k) * B(n,k)
//   A(m,k) = A_K ? A[m*lda+k] : A[k*lda+m];  B(n,k) = B_K ? B[n*ldb+k] : B[k*ldb+n]
template <bool A_K, bool B_K, bool VEC>
__global__ void __launch_bounds__(GT) k_gemm(int M, int N, int K, const float* __restrict__ A,
                                             int lda, const float* __restrict__ B, int ldb,
                                             float* __restrict__ C, int ldc, int kps, EpiArgs ep) {
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb = blockIdx.z * kps, ke = min(K, kb + kps);
  if (blockIdx.z > 0) C += (size_t)blockIdx.z * M * ldc;

  // loader coordinates (4 elements per thread per operand)
  float ra[4], rb[4];
  auto load_a = [&](int k0) {
    if (A_K) {
      const int m = tid >> 1, k = (tid & 1) * 4;
      const int gm = m0 + m, gk = k0 + k;
      if (VEC && gm < M && gk + 3 < ke) {
        const float4 v = *reinterpret_cast<const float4*>(A + (size_t)gm * lda + gk);
        ra[0] = v.x, ra[1] = v.y, ra[2] = v.z, ra[3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ra[q] = (gm < M && gk + q < ke) ? A[(size_t)gm * lda + gk + q] : 0.f;
      }
    } else {
      const int k = tid >> 5, m = (tid & 31) * 4;
      const int gm = m0 + m, gk = k0 + k;
      if (VEC && gk < ke && gm + 3 < M) {
        const float4 v = *reinterpret_cast<const float4*>(A + (size_t)gk * lda + gm);
        ra[0] = v.x, ra[1] = v.y, ra[2] = v.z, ra[3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ra[q] = (gk < ke && gm + q < M) ? A[(size_t)gk * lda + gm + q] : 0.f;
      }
    }
  };
  auto load_b = [&](int k0) {
    if (B_K) {
      const int n = tid >> 1, k = (tid & 1) * 4;
      const int gn = n0 + n, gk = k0 + k;
      if (VEC && gn < N && gk + 3 < ke) {
        const float4 v = *reinterpret_cast<const float4*>(B + (size_t)gn * ldb + gk);
        rb[0] = v.x, rb[1] = v.y, rb[2] = v.z, rb[3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          rb[q] = (gn < N && gk + q < ke) ? B[(size_t)gn * ldb + gk + q] : 0.f;
      }
    } else {
      const int k = tid >> 5, n = (tid & 31) * 4;
      const int gn = n0 + n, gk = k0 + k;
      if (VEC && gk < ke && gn + 3 < N) {
        const float4 v = *reinterpret_cast<const float4*>(B + (size_t)gk * ldb + gn);
        rb[0] = v.x, rb[1] = v.y, rb[2] = v.z, rb[3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          rb[q] = (gk < ke && gn + q < N) ? B[(size_t)gk * ldb + gn + q] : 0.f;
      }
    }
  };
  auto store_ab = [&](int buf) {
    if (A_K) {
      const int m = tid >> 1, k = (tid & 1) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) As[buf][k + q][m] = ra[q];
    } else {
      const int k = tid >> 5, m = (tid & 31) * 4;
      *reinterpret_cast<float4*>(&As[buf][k][m]) = make_float4(ra[0], ra[1], ra[2], ra[3]);
    }
    if (B_K) {
      const int n = tid >> 1, k = (tid & 1) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) Bs[buf][k + q][n] = rb[q];
    } else {
      const int k = tid >> 5, n = (tid & 31) * 4;
      *reinterpret_cast<float4*>(&Bs[buf][k][n]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
    }
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const int tx = tid & 15, ty = tid >> 4;
  int buf = 0;
  if (kb < ke) {
    load_a(kb);
    load_b(kb);
    store_ab(0);
  }
  __syncthreads();
  for (int k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) {
      load_a(k0 + BK);
      load_b(k0 + BK);
    }
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
      a[0] = a0.x, a[1] = a0.y, a[2] = a0.z, a[3] = a0.w;
      a[4] = a1.x, a[5] = a1.y, a[6] = a1.z, a[7] = a1.w;
      b[0] = b0.x, b[1] = b0.y, b[2] = b0.z, b[3] = b0.w;
      b[4] = b1.x, b[5] = b1.y, b[6] = b1.z, b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_ab(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= N) continue;
      float v = acc[i][j];
      if (ep.mode == kBiasAct) {
        v = act_fwd(ep.act, __fadd_rn(v, ep.bias[n]));
      } else if (ep.mode == kDAct) {
        v = __fmul_rn(v, act_bwd(ep.act, ep.aux[(size_t)m * ep.ld_aux + n]));
      } else if (ep.mode == kCoeff) {
        v = __fmul_rn(v, ep.coeff[(size_t)m * ep.S + n / ep.e]);
      }
      C[(size_t)m * ldc + n] = v;
    }
  }
}

// Small tiles (32 x 64, 8 outputs per thread) for the skinny products of small
// batches (configs[0]'s [208->64->32->1] at 4096 instances): the 128 x 128 tile
// leaves most of the GPU idle there -- 32 CTAs for a 4096 x 32 layer.
constexpr int SBM = 32, SBN = 64, SBK = 32;
template <bool A_K, bool B_K>
__global__ void __launch_bounds__(256) k_gemm_s(int M, int N, int K, const float* __restrict__ A, int lda,
                                                const float* __restrict__ B, int ldb, float* __restrict__ C,
                                                int ldc, int kps, EpiArgs ep) {
  __shared__ __align__(16) float As[SBK][SBM + 4];  // [k][m]
  __shared__ __align__(16) float Bs[SBK][SBN + 4];  // [k][n]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // columns tx*4.., rows ty*2..
  const int m0 = blockIdx.y * SBM, n0 = blockIdx.x * SBN;
  const int kb = blockIdx.z * kps, ke = min(K, kb + kps);
  if (blockIdx.z > 0) C += (size_t)blockIdx.z * M * ldc;
  float acc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // the next k-chunk's operands are loaded into registers while this one is
  // multiplied (loads run along each operand's contiguous dimension)
  constexpr int NA = SBM * SBK / 256, NB = SBN * SBK / 256;
  float ra[NA], rb[NB];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int i = threadIdx.x + q * 256;
      const int m = A_K ? i / SBK : i % SBM, k = A_K ? i % SBK : i / SBM;
      const int gm = m0 + m, gk = k0 + k;
      ra[q] = (gm < M && gk < ke) ? (A_K ? A[(size_t)gm * lda + gk] : A[(size_t)gk * lda + gm]) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int i = threadIdx.x + q * 256;
      const int n = B_K ? i / SBK : i % SBN, k = B_K ? i % SBK : i / SBN;
      const int gn = n0 + n, gk = k0 + k;
      rb[q] = (gn < N && gk < ke) ? (B_K ? B[(size_t)gn * ldb + gk] : B[(size_t)gk * ldb + gn]) : 0.f;
    }
  };
  if (kb < ke) load(kb);
  for (int k0 = kb; k0 < ke; k0 += SBK) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int i = threadIdx.x + q * 256;
      As[A_K ? i % SBK : i / SBM][A_K ? i / SBK : i % SBM] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int i = threadIdx.x + q * 256;
      Bs[B_K ? i % SBK : i / SBN][B_K ? i / SBK : i % SBN] = rb[q];
    }
    __syncthreads();
    if (k0 + SBK < ke) load(k0 + SBK);
#pragma unroll 8
    for (int k = 0; k < SBK; ++k) {
      const float2 a = *reinterpret_cast<const float2*>(&As[k][ty * 2]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float av[2] = {a.x, a.y}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float out[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int m = m0 + ty * 2 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      out[i][j] = 0.f;
      if (m >= M || n >= N) continue;
      float v = acc[i][j];
      if (ep.mode == kBiasAct) {
        v = act_fwd(ep.act, __fadd_rn(v, ep.bias[n]));
      } else if (ep.mode == kDAct) {
        v = __fmul_rn(v, act_bwd(ep.act, ep.aux[(size_t)m * ep.ld_aux + n]));
      } else if (ep.mode == kCoeff) {
        v = __fmul_rn(v, ep.coeff[(size_t)m * ep.S + n / ep.e]);
      }
      C[(size_t)m * ldc + n] = v;
      out[i][j] = v;
    }
  }
  if (ep.csum_part) {  // (one K split) this tile's column sums: row pairs in order
    float* red = &As[0][0];  // 16 x 64 <= 32 x 36 floats; free after the k loop's last barrier
#pragma unroll
    for (int j = 0; j < 4; ++j) red[ty * SBN + tx * 4 + j] = __fadd_rn(out[0][j], out[1][j]);
    __syncthreads();
    if (tid < SBN && n0 + tid < N) {
      float t = red[tid];
      for (int q = 1; q < 16; ++q) t = __fadd_rn(t, red[q * SBN + tid]);
      ep.csum_part[(size_t)blockIdx.y * N + n0 + tid] = t;
    }
  }
}

// the small tiles when the 128 x 128 ones would not cover the SMs
bool small_tiles(int M, int N) { return ceil_div(M, BM) * ceil_div(N, BN) < 148; }

template <bool A_K, bool B_K>
int gemm(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C, int ldc,
          int splits, const EpiArgs& ep, cudaStream_t s) {
  if (M <= 0 || N <= 0) return 0;
  splits = splits < 1 ? 1 : splits;
  if (small_tiles(M, N)) {
    int kps = (K + splits - 1) / splits;
    kps = std::max(SBK, (kps + SBK - 1) / SBK * SBK);
    splits = K > 0 ? (K + kps - 1) / kps : 1;
    dim3 grid(ceil_div(N, SBN), ceil_div(M, SBM), splits);
    k_gemm_s<A_K, B_K><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, kps, ep);
    ::kp::count_launch();
    return splits;
  }
  int kps = (K + splits - 1) / splits;
  kps = (kps + BK - 1) / BK * BK;
  splits = K > 0 ? (K + kps - 1) / kps : 1;
  if (kps == 0) kps = BK;
  dim3 grid(ceil_div(N, BN), ceil_div(M, BM), splits);
  const bool vec = (lda % 4 == 0) && (ldb % 4 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(B) % 16 == 0);
  if (vec)
    k_gemm<A_K, B_K, true><<<grid, GT, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, kps, ep);
  else
    k_gemm<A_K, B_K, false><<<grid, GT, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, kps, ep);
  ::kp::count_launch();
  return splits;
}

// out[i] = sum_z part[z][i], z ascending (deterministic split-K reduce)
// small outputs with many splits (the SIMT weight gradients of configs[0]):
// 32 outputs per block, 8 thread rows each summing a fixed z-range, then the
// 8 range sums in order -- a fixed tree, deterministic like the flat one
__global__ void k_reduce_splits_wide(const float* __restrict__ part, int splits, size_t n,
                                     float* __restrict__ out) {
  __shared__ float red[8][33];
  const size_t i = blockIdx.x * (size_t)32 + threadIdx.x;
  const int z0 = threadIdx.y * splits / 8, z1 = (threadIdx.y + 1) * splits / 8;
  float v = 0.f;
  if (i < n) {
    int z = z0;
    for (; z + 4 <= z1; z += 4) {
      const float a = part[(size_t)z * n + i], b = part[(size_t)(z + 1) * n + i];
      const float c = part[(size_t)(z + 2) * n + i], d = part[(size_t)(z + 3) * n + i];
      v = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(v, a), b), c), d);
    }
    for (; z < z1; ++z) v = __fadd_rn(v, part[(size_t)z * n + i]);
  }
  red[threadIdx.y][threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.y == 0 && i < n) {
    float t = red[0][threadIdx.x];
#pragma unroll
    for (int r = 1; r < 8; ++r) t = __fadd_rn(t, red[r][threadIdx.x]);
    out[i] = t;
  }
}

__global__ void k_reduce_splits(const float* __restrict__ part, int splits, size_t n,
                                float* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float v = part[i];
    int z = 1;
    for (; z + 4 <= splits; z += 4) {  // loads in flight, adds in z order
      const float a = part[(size_t)z * n + i], b = part[(size_t)(z + 1) * n + i];
      const float c = part[(size_t)(z + 2) * n + i], d = part[(size_t)(z + 3) * n + i];
      v = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(v, a), b), c), d);
    }
    for (; z < splits; ++z) v = __fadd_rn(v, part[(size_t)z * n + i]);
    out[i] = v;
  }
}

// column sums (optionally weighted): partial[c][n] = sum_{b in chunk c} w[b]*X[b][n]
// column sums (optionally weighted): part[c][n] = sum_{b in chunk c} w[b]*X[b][n];
// block (32 columns x 8 row lanes), fixed-order combine of the 8 lanes.
// Rows per chunk: 512, or fewer for small batches so at least ~128 chunks
// run in parallel (configs[0]: 4096 rows -> 32-row chunks; configs[1]
// unchanged).
constexpr int COLSUM_ROWS = 512;
int colsum_rows(int B) {
  if (B >= 128 * COLSUM_ROWS) return COLSUM_ROWS;
  const int r = (B / 128 + 31) / 32 * 32;
  return r < 32 ? 32 : r;
}
__global__ void k_colsum_part(const float* __restrict__ X, const float* __restrict__ w, int B,
                              int N, float* __restrict__ part, int rows) {
  __shared__ float red[8][33];
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int c = blockIdx.y;
  const int b0 = c * rows, b1 = min(B, b0 + rows);
  float acc = 0.f;
  if (n < N) {
    int b = b0 + threadIdx.y;
    for (; b + 24 < b1; b += 32) {  // 4 independent loads in flight
      float x0 = X[(size_t)b * N + n], x1 = X[(size_t)(b + 8) * N + n];
      float x2 = X[(size_t)(b + 16) * N + n], x3 = X[(size_t)(b + 24) * N + n];
      if (w) {
        x0 = __fmul_rn(w[b], x0), x1 = __fmul_rn(w[b + 8], x1);
        x2 = __fmul_rn(w[b + 16], x2), x3 = __fmul_rn(w[b + 24], x3);
      }
      acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, x0), x1), x2), x3);
    }
    for (; b < b1; b += 8) {
      const float x = X[(size_t)b * N + n];
      acc = __fadd_rn(acc, w ? __fmul_rn(w[b], x) : x);
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    float t = red[0][threadIdx.x];
    for (int i = 1; i < 8; ++i) t = __fadd_rn(t, red[i][threadIdx.x]);
    part[(size_t)c * N + n] = t;
  }
}

// Head (out = 1): logit = b + w . a ; pred = sigmoid (model.cpp:34-38,118-123)
__global__ void k_head_fwd(const float* __restrict__ in, int B, int W, const float* __restrict__ w,
                           const float* __restrict__ bias, float* __restrict__ logits,
                           float* __restrict__ preds) {
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int b = wid; b < B; b += nw) {
    const float* a = in + (size_t)b * W;
    float s = 0.f;
    for (int i = lane; i < W; i += 32) s = fmaf(w[i], a[i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const float z = __fadd_rn(s, bias[0]);
      float p;
      if (z >= 0.f) {
        p = __fdiv_rn(1.f, __fadd_rn(1.f, expf(-z)));
      } else {
        const float e = expf(z);
        p = __fdiv_rn(e, __fadd_rn(1.f, e));
      }
      logits[b] = z;
      preds[b] = p;
    }
  }
}

// delta = (p - y)/n; loss term softplus(z) - y z (model.cpp:126-135,153-155);
// dprev[b][i] = (delta * w[i]) * act'(a[b][i])  or  * coeff  (layer-0 input)
__global__ void k_head_bwd(const float* __restrict__ in, int B, int W, const float* __restrict__ w,
                           const float* __restrict__ logits, const float* __restrict__ preds,
                           const int32_t* __restrict__ labels, float nb,
                           float* __restrict__ delta, float* __restrict__ dprev, int mode, int act,
                           const float* __restrict__ coeff, uint32_t S, uint32_t e,
                           double* __restrict__ loss_part, unsigned* __restrict__ done,
                           double* __restrict__ loss_sum, int n_loss, float* __restrict__ cpart, int W2) {
  __shared__ double s_loss[8];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double lsum = 0.0;
  if (cpart) {
    // (W <= 256) the head's three column sums from the rows in registers:
    // sum_b delta*a[b][i] (head weights), sum_b dprev[b][i] (the hidden
    // layer's bias, W2 = W), sum_b delta (head bias) -- per lane over its
    // rows in order, then the block's warps in order into cpart[block][NT]
    constexpr int MAXC = 8;
    float wacc[MAXC], bacc[MAXC], dacc = 0.f;
#pragma unroll
    for (int q = 0; q < MAXC; ++q) wacc[q] = 0.f, bacc[q] = 0.f;
    for (int b = wid; b < B; b += nw) {
      const float y = (float)labels[b];
      const float d = __fdiv_rn(__fsub_rn(preds[b], y), nb);
      if (lane == 0) {
        delta[b] = d;
        const float z = logits[b];
        const float sp = __fadd_rn(fmaxf(z, 0.f), log1pf(expf(-fabsf(z))));
        lsum += (double)__fsub_rn(sp, __fmul_rn(y, z));
        dacc = __fadd_rn(dacc, d);
      }
#pragma unroll
      for (int q = 0; q < MAXC; ++q) {
        const int i = lane + 32 * q;
        if (i < W) {
          const float av = in[(size_t)b * W + i];
          wacc[q] = __fadd_rn(wacc[q], __fmul_rn(d, av));
          if (dprev) {
            float g = __fmul_rn(d, w[i]);
            if (mode == kDAct) g = __fmul_rn(g, act_bwd(act, av));
            else if (mode == kCoeff) g = __fmul_rn(g, coeff[(size_t)b * S + i / e]);
            dprev[(size_t)b * W + i] = g;
            if (W2) bacc[q] = __fadd_rn(bacc[q], g);
          }
        }
      }
    }
    __shared__ float s_col[8][2 * 256 + 1];
    const int NT = W + W2 + 1;
#pragma unroll
    for (int q = 0; q < MAXC; ++q) {
      const int i = lane + 32 * q;
      if (i < W) {
        s_col[warp][i] = wacc[q];
        if (W2) s_col[warp][W + i] = bacc[q];
      }
    }
    if (lane == 0) s_col[warp][W + W2] = dacc;
    __syncthreads();
    for (int n = threadIdx.x; n < NT; n += blockDim.x) {
      float t = s_col[0][n];
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q) t = __fadd_rn(t, s_col[q][n]);
      cpart[(size_t)blockIdx.x * NT + n] = t;
    }
  } else {
    for (int b = wid; b < B; b += nw) {
      const float y = (float)labels[b];
      const float d = __fdiv_rn(__fsub_rn(preds[b], y), nb);
      if (lane == 0) {
        delta[b] = d;
        const float z = logits[b];
        const float sp = __fadd_rn(fmaxf(z, 0.f), log1pf(expf(-fabsf(z))));
        lsum += (double)__fsub_rn(sp, __fmul_rn(y, z));
      }
      if (dprev) {
        for (int i = lane; i < W; i += 32) {
          float g = __fmul_rn(d, w[i]);
          if (mode == kDAct) g = __fmul_rn(g, act_bwd(act, in[(size_t)b * W + i]));
          else if (mode == kCoeff) g = __fmul_rn(g, coeff[(size_t)b * S + i / e]);
          dprev[(size_t)b * W + i] = g;
        }
      }
    }
  }
  if (lane == 0) s_loss[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += s_loss[q];
    loss_part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;  // the last block finalizes
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // loss_sum += (sum / n) * n, the reference's loss_sum += bwd.loss * mb.size
  // (trainer.cpp:177): every thread of the last block sums a strided set of
  // partials (four loads in flight -- one lane walking them was a chain of
  // L2 round trips), then the block's sums combine in thread order
  __shared__ double s_fin[32];
  const int nt = (int)blockDim.x, ng = (int)gridDim.x;
  double t = 0.0;
  int i = (int)threadIdx.x;
  for (; i + 3 * nt < ng; i += 4 * nt) {
    const double a = *reinterpret_cast<volatile double*>(loss_part + i);
    const double b = *reinterpret_cast<volatile double*>(loss_part + i + nt);
    const double c = *reinterpret_cast<volatile double*>(loss_part + i + 2 * nt);
    const double d = *reinterpret_cast<volatile double*>(loss_part + i + 3 * nt);
    t += a;
    t += b;
    t += c;
    t += d;
  }
  for (; i < ng; i += nt) t += *reinterpret_cast<volatile double*>(loss_part + i);
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);  // fixed butterfly
  if (lane == 0) s_fin[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int q = 0; q < (nt >> 5); ++q) u += s_fin[q];
    *loss_sum += (u / (double)n_loss) * (double)n_loss;
    *done = 0u;  // ready for the next launch (stream order)
  }
}

unsigned grid_cap(uint64_t blocks) {
  if (blocks < 1) blocks = 1;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  return (unsigned)blocks;
}

// split-K reduce: the wide form when few outputs would leave the GPU idle
void reduce_splits_any(const float* part, int splits, size_t n, float* out, cudaStream_t s) {
  if (n < 148 * 256 && splits >= 16) {
    k_reduce_splits_wide<<<(unsigned)ceil_div(n, 32), dim3(32, 8), 0, s>>>(part, splits, n, out);
  } else {
    k_reduce_splits<<<grid_cap(ceil_div(n, 256)), 256, 0, s>>>(part, splits, n, out);
  }
  ::kp::count_launch();
}

// split-K count: enough CTAs to cover ~2 waves of 148 SMs
int pick_splits(int M, int N, int K) {
  const bool sm = small_tiles(M, N);
  const int tiles = sm ? (int)(ceil_div(M, SBM) * ceil_div(N, SBN)) : (int)(ceil_div(M, BM) * ceil_div(N, BN));
  int sp = (2 * 148 + tiles - 1) / tiles;
  const int max_sp = sm ? (K + 63) / 64 : (K + 255) / 256;  // >= 64 / 256 rows per split
  if (sp > max_sp) sp = max_sp;
  return sp < 1 ? 1 : sp;
}

}  // namespace

void simt_gemm_nt(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
                  int ldc, cudaStream_t s) {
  EpiArgs plain{kStore, 0, nullptr, nullptr, 0, nullptr, 1, 1};
  gemm<true, true>(M, N, K, A, lda, B, ldb, C, ldc, 1, plain, s);
}

void simt_gemm_tn(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
                  int ldc, cudaStream_t s) {
  EpiArgs plain{kStore, 0, nullptr, nullptr, 0, nullptr, 1, 1};
  gemm<false, false>(M, N, K, A, lda, B, ldb, C, ldc, 1, plain, s);
}

void reduce_splits(const float* part, int splits, size_t n, float* out, cudaStream_t s) {
  reduce_splits_any(part, splits, n, out, s);
}

static bool gemm_pre() {
  static const bool on = [] {
    const char* e = getenv("KP_GEMM_PRE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// small GEMMs (all of configs[0]'s layers: <= 109 MFLOP at 4096 instances)
// finish sooner on the small-tile SIMT kernel than a persistent tcgen05 launch
// with its TMEM/barrier set-up and operand splits
bool tc_worth(int M, int N, int K, double min_flop) { return 2.0 * M * N * K >= min_flop; }

// fp16-operand GEMM for the first layer: K-major, 16-byte aligned, K % 8 == 0
static bool use_h(int M, int N, int K, const float* A, const float* W, double min_flop) {
  return tc_enabled() && tc_h_enabled() && tc_worth(M, N, K, min_flop) && K % 8 == 0 &&
         tc_gemm_supported(M, N, K, A, K, W, K);
}

void mlp_forward(const MlpShape& m, const float* d_x, const float* d_in, uint32_t B,
                 float* d_preds, MlpWs& ws, cudaStream_t s) {
  if (B == 0) return;
  const float* in = d_in;
  const uint32_t L = m.n_layers;
  for (uint32_t l = 0; l + 1 < L; ++l) {
    const int K = m.widths[l], N = m.widths[l + 1];
    float* out = ws.act[l].get<float>((size_t)B * N);
    EpiArgs ep{kBiasAct, m.activation, d_x + m.b_off[l], nullptr, 0, nullptr, 1, 1};
    const float* W = d_x + m.w_off[l];
    if (l == 0 && ws.in_hi) {
      // first layer on the pooling kernel's fp16 planes: 3xFP16 on pre-split
      // operands (kp_gemm_h3.cu), W1 split per row
      __half* hh = reinterpret_cast<__half*>(ws.hhi.get<uint16_t>((size_t)N * K));
      __half* hl = reinterpret_cast<__half*>(ws.hlo.get<uint16_t>((size_t)N * K));
      int* he = ws.hexp.get<int>(N);
      split_h(W, N, K, K, hh, hl, he, s);
      // (the last partial wave of tiles stream-K: 256 tiles = 3.46 waves at B = 65536)
      // one feature per slot: the GEMM gathers the table rows itself (TMA
      // gather4) and writes the planes on the way -- no pooling pass
      const H3Gather ga{ws.ga_src, ws.ga_nrows, ws.ga_rowocc, ws.ga_S, ws.ga_e, true};
      h3_gemm(H3Operand{ws.in_hi, ws.in_lo, ws.in_exp, K}, false, H3Operand{hh, hl, he, K}, false, B, N, K,
              out, N, ep, 2, ws.skws.get<float>(h3_splitk_ws_floats(B, N, true)), s, /*keep W1*/ 2,
              ws.ga_src ? &ga : nullptr);
    } else if (l == 0 && use_h(B, N, K, in, W, ws.tc_min_flop)) {
      // first layer (the wide S*e contraction): fp16 operands, per-row scales
      const float* am = ws.in_rowmax;
      if (!am) {
        float* t = ws.amax.get<float>(B);
        rowmax(in, B, K, K, t, s);
        am = t;
      }
      __half* hh = reinterpret_cast<__half*>(ws.hhi.get<uint16_t>((size_t)N * K));
      __half* hl = reinterpret_cast<__half*>(ws.hlo.get<uint16_t>((size_t)N * K));
      int* he = ws.hexp.get<int>(N);
      split_h(W, N, K, K, hh, hl, he, s);
      tc_gemm_nt_h(B, N, K, in, K, am, hh, hl, he, K, out, N, ep, s);
    } else if (tc_enabled() && tc_worth(B, N, K, ws.tc_min_flop) && tc_gemm_supported(B, N, K, in, K, W, K)) {
      float* whi = ws.whi.get<float>((size_t)N * K);
      float* wlo = ws.wlo.get<float>((size_t)N * K);
      if (gemm_pre()) {
        split_hilo(W, whi, wlo, (size_t)N * K, s);
        tc_gemm_nt_pre(B, N, K, in, K, whi, wlo, K, out, N, ep, s);
      } else {
        tc_gemm_nt(B, N, K, in, K, W, K, out, N, ep, s);
      }
    } else {
      gemm<true, true>(B, N, K, in, K, W, K, out, N, 1, ep, s);
    }
    in = out;
  }
  const int W = m.widths[L - 1];
  float* logits = ws.logits.get<float>(B);
  k_head_fwd<<<grid_cap(((uint64_t)B * 32 + 255) / 256), 256, 0, s>>>(
      in, B, W, d_x + m.w_off[L - 1], d_x + m.b_off[L - 1], logits, d_preds); ::kp::count_launch();
}

namespace {
__global__ void k_transpose(const float* __restrict__ in, int R, int Cc, float* __restrict__ out) {
  __shared__ float t[32][33];
  const int c = blockIdx.x * 32 + threadIdx.x, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (r0 + i < R && c < Cc) t[i][threadIdx.x] = in[(size_t)(r0 + i) * Cc + c];
  __syncthreads();
  const int r = r0 + threadIdx.x, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (c0 + i < Cc && r < R) out[(size_t)(c0 + i) * R + r] = t[threadIdx.x][i];
}

// dX[B][K] = dZ[B][N] . W[N][K]  (W^T kept K-major for the tensor-core path)
// (returns true when the small-tile path also wrote ep.csum_part; the other
// paths ignore it)
bool dx_gemm(int B, int K, int N, const float* dZ, const float* W, float* out, EpiArgs ep,
             MlpWs& ws, cudaStream_t s, bool first = false) {
  float* const csum = ep.csum_part;
  ep.csum_part = nullptr;
  if (first && N % 8 == 0 && use_h(B, K, N, dZ, W, ws.tc_min_flop)) {
    // first layer's input gradient (the wide output): fp16 operands
    float* wt = ws.wt.get<float>((size_t)N * K);
    dim3 g(ceil_div(K, 32), ceil_div(N, 32));
    k_transpose<<<g, dim3(32, 8), 0, s>>>(W, N, K, wt); ::kp::count_launch();
    __half* th = reinterpret_cast<__half*>(ws.thi.get<uint16_t>((size_t)N * K));
    __half* tl = reinterpret_cast<__half*>(ws.tlo.get<uint16_t>((size_t)N * K));
    int* te = ws.texp.get<int>(K);
    split_h(wt, K, N, N, th, tl, te, s);
    float* am = ws.amax.get<float>(B);
    rowmax(dZ, B, N, N, am, s);
    tc_gemm_nt_h(B, K, N, dZ, N, am, th, tl, te, N, out, K, ep, s);
    return false;
  }
  if (tc_enabled() && tc_worth(B, K, N, ws.tc_min_flop) && tc_gemm_supported(B, K, N, dZ, N, W, N)) {
    float* wt = ws.wt.get<float>((size_t)N * K);
    dim3 g(ceil_div(K, 32), ceil_div(N, 32));
    k_transpose<<<g, dim3(32, 8), 0, s>>>(W, N, K, wt); ::kp::count_launch();
    float* wthi = ws.wthi.get<float>((size_t)N * K);
    float* wtlo = ws.wtlo.get<float>((size_t)N * K);
    if (gemm_pre()) {
      split_hilo(wt, wthi, wtlo, (size_t)N * K, s);
      tc_gemm_nt_pre(B, K, N, dZ, N, wthi, wtlo, N, out, K, ep, s);
    } else {
      tc_gemm_nt(B, K, N, dZ, N, wt, N, out, K, ep, s);
    }
    return false;
  }
  const bool cs = csum && small_tiles(B, K);  // (one K split on the small tiles)
  if (cs) ep.csum_part = csum;
  gemm<true, false>(B, K, N, dZ, N, W, K, out, K, 1, ep, s);
  return cs;
}

// The head's three reductions in one pass (model.cpp:163-177 for the last
// two layers): virtual column n < W: sum_b delta[b] * a[b][n] (head weight
// gradient), W <= n < W + W2: sum_b dz[b][n - W] (the hidden layer's bias
// gradient), n == W + W2: sum_b delta[b] (head bias). Per 512-row chunk
// partials like k_colsum_part (fixed order), reduced by k_reduce_chunks_to.
__global__ void k_colsum_head(const float* __restrict__ a, const float* __restrict__ delta,
                              const float* __restrict__ dz, int B, int W, int W2, float* __restrict__ part,
                              int rows) {
  __shared__ float red[8][33];
  const int NT = W + W2 + 1;
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int c = blockIdx.y;
  const int b0 = c * rows, b1 = min(B, b0 + rows);
  float acc = 0.f;
  if (n < NT) {
    // the column's source, then 4 independent loads in flight per step
    const float* src = n < W ? a + n : (n < W + W2 ? dz + (n - W) : delta);
    const int ld = n < W ? W : (n < W + W2 ? W2 : 1);
    const bool wt = n < W;
    int b = b0 + threadIdx.y;
    for (; b + 24 < b1; b += 32) {
      float x0 = src[(size_t)b * ld], x1 = src[(size_t)(b + 8) * ld];
      float x2 = src[(size_t)(b + 16) * ld], x3 = src[(size_t)(b + 24) * ld];
      if (wt) {
        x0 = __fmul_rn(delta[b], x0), x1 = __fmul_rn(delta[b + 8], x1);
        x2 = __fmul_rn(delta[b + 16], x2), x3 = __fmul_rn(delta[b + 24], x3);
      }
      acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, x0), x1), x2), x3);
    }
    for (; b < b1; b += 8) {
      const float x = src[(size_t)b * ld];
      acc = __fadd_rn(acc, wt ? __fmul_rn(delta[b], x) : x);
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && n < NT) {
    float t = red[0][threadIdx.x];
    for (int i = 1; i < 8; ++i) t = __fadd_rn(t, red[i][threadIdx.x]);
    part[(size_t)c * NT + n] = t;
  }
}

// k_reduce_chunks writing column n to out0[n] (n < n0), out1[n - n0]
// (n < n0 + n1), out2[n - n0 - n1]
__global__ void k_reduce_chunks_to(const float* __restrict__ part, int chunks, int N, int n0, int n1,
                                   float* __restrict__ out0, float* __restrict__ out1, float* __restrict__ out2) {
  const int lane = threadIdx.x & 31;
  for (int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < N; n += (gridDim.x * blockDim.x) >> 5) {
    float v = 0.f;
    for (int c = lane; c < chunks; c += 32) v = __fadd_rn(v, part[(size_t)c * N + n]);
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) {
      if (n < n0) out0[n] = v;
      else if (n < n0 + n1) out1[n - n0] = v;
      else out2[n - n0 - n1] = v;
    }
  }
}

// column sums of the chunk partials [chunks][N]: one warp per column, lane j
// adds chunks j, j+32, ... in order, then a fixed xor tree (deterministic)
__global__ void k_reduce_chunks(const float* __restrict__ part, int chunks, int N,
                                float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < N; n += (gridDim.x * blockDim.x) >> 5) {
    float v = 0.f;
    for (int c = lane; c < chunks; c += 32) v = __fadd_rn(v, part[(size_t)c * N + n]);
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) out[n] = v;
  }
}

void colsum(const float* X, const float* w, int B, int N, float* out, MlpWs& ws, cudaStream_t s) {
  const int rows = colsum_rows(B);
  const int chunks = std::max(1, (B + rows - 1) / rows);
  float* part = ws.partials.get<float>((size_t)chunks * N);
  dim3 g(ceil_div(N, 32), chunks);
  k_colsum_part<<<g, dim3(32, 8), 0, s>>>(X, w, B, N, part, rows); ::kp::count_launch();
  if (chunks >= 32 && N <= 4096) {
    k_reduce_chunks<<<grid_cap(ceil_div((uint64_t)N * 32, 256)), 256, 0, s>>>(part, chunks, N, out); ::kp::count_launch();
  } else {
    k_reduce_splits<<<grid_cap(ceil_div(N, 256)), 256, 0, s>>>(part, chunks, (size_t)N, out); ::kp::count_launch();
  }
}
}  // namespace

void mlp_backward(const MlpShape& m, const float* d_x, const float* d_in, uint32_t B,
                  const float* d_preds, const int32_t* d_labels, float* d_grad, float* d_dinput,
                  const float* d_coeff, uint32_t S, uint32_t e, double* d_loss_sum, MlpWs& ws,
                  cudaStream_t s, const std::function<void()>* after_dinput) {
  const uint32_t L = m.n_layers;
  if (B == 0) {
    KP_CUDA(cudaMemsetAsync(d_grad, 0, m.D * 4, s));
    return;
  }
  auto layer_in = [&](uint32_t l) -> const float* {
    return l == 0 ? d_in : static_cast<const float*>(ws.act[l - 1].p);
  };
  // ---- head (out = 1) ----
  const int W = m.widths[L - 1];
  float* delta = ws.delta.get<float>(B);
  float* dprev = nullptr;
  int mode = kStore;
  if (L >= 2) {
    dprev = ws.dz[0].get<float>((size_t)B * W);
    mode = kDAct;
  } else if (d_dinput) {
    dprev = d_dinput;
    mode = d_coeff ? kCoeff : kStore;
  }
  // head weight + bias gradients, and (with hidden layers) the last hidden
  // layer's bias gradient (the column sums of dprev = its dZ): in the head's
  // backward pass itself (W <= 256: per-block partials, ~8 rows per warp), or
  // one extra pass over a and dprev
  const bool fused_bias = L >= 2;
  const int W2 = fused_bias ? W : 0;
  const int NT = W + W2 + 1;
  const char* hf_env = getenv("KP_HEAD_FUSE");  // =0: the separate column-sum pass
  const bool head_cols = W <= 256 && !(hf_env && hf_env[0] == '0');
  // (fused: ~8 rows per warp, but at least two blocks per SM for small batches)
  const unsigned hb = head_cols ? grid_cap(std::max<uint64_t>((B + 63) / 64, std::min<uint64_t>(296, (B + 7) / 8)))
                                : grid_cap(((uint64_t)B * 32 + 255) / 256);
  double* lossp = ws.lossp.get<double>(hb);
  if (!ws.hdone.p) {
    ws.hdone.get<unsigned>(1);
    KP_CUDA(cudaMemsetAsync(ws.hdone.p, 0, 4, s));
  }
  float* cpart = head_cols ? ws.partials.get<float>((size_t)hb * NT) : nullptr;
  k_head_bwd<<<hb, 256, 0, s>>>(layer_in(L - 1), B, W, d_x + m.w_off[L - 1],
                                 static_cast<const float*>(ws.logits.p), d_preds, d_labels,
                                 (float)B, delta, dprev, mode, m.activation, d_coeff, S, e, lossp,
                                 static_cast<unsigned*>(ws.hdone.p), d_loss_sum, (int)B, cpart, W2);
  ::kp::count_launch();
  if (head_cols) {
    k_reduce_chunks_to<<<grid_cap(ceil_div((uint64_t)NT * 32, 256)), 256, 0, s>>>(
        cpart, (int)hb, NT, W, W2, d_grad + m.w_off[L - 1], fused_bias ? d_grad + m.b_off[L - 2] : nullptr,
        d_grad + m.b_off[L - 1]); ::kp::count_launch();
  } else {
    const int rows = colsum_rows((int)B);
    const int chunks = std::max(1, (int)((B + rows - 1) / rows));
    float* part = ws.partials.get<float>((size_t)chunks * NT);
    k_colsum_head<<<dim3(ceil_div(NT, 32), chunks), dim3(32, 8), 0, s>>>(layer_in(L - 1), delta, dprev, B, W, W2,
                                                                          part, rows); ::kp::count_launch();
    k_reduce_chunks_to<<<grid_cap(ceil_div((uint64_t)NT * 32, 256)), 256, 0, s>>>(
        part, chunks, NT, W, W2, d_grad + m.w_off[L - 1], fused_bias ? d_grad + m.b_off[L - 2] : nullptr,
        d_grad + m.b_off[L - 1]); ::kp::count_launch();
  }
  // ---- hidden layers, top down ----
  int cur = 0;
  bool csum_ready = false;  // ws.cpart holds this layer's bias-gradient partials
  for (int l = (int)L - 2; l >= 0; --l) {
    const int N = m.widths[l + 1], K = m.widths[l];
    float* dZ = static_cast<float*>(ws.dz[cur].p);
    const float* in = layer_in(l);
    if (l == 0 && ws.in_hi) {
      // first layer on fp16 planes (kp_gemm_h3.cu): dX = dZ1 W1 (dZ1 split per
      // row, W1^T per row), then dW = dZ'^T X over the batch with X's row
      // scales moved onto dZ' (split per column) and X's planes read MN-major
      // (the layer's bias gradient = column sums of dZ, from the same read)
      const bool bias_here = l != (int)L - 2;
      float* colsum_ws = bias_here ? ws.partials.get<float>(split_cols_colsum_ws_floats(B, N)) : nullptr;
      unsigned* cmax = ws.cmax.get<unsigned>(N);
      const bool fuse = d_dinput && rows_colmax_fusable(N);
      if (d_dinput) {
        __half* dzh = reinterpret_cast<__half*>(ws.dzh.get<uint16_t>((size_t)B * N));
        __half* dzl = reinterpret_cast<__half*>(ws.dzl.get<uint16_t>((size_t)B * N));
        int* dze = ws.dze.get<int>(B);
        // dX's row-split operand and dW's column scales (+ bias partials) in one read
        if (fuse) split_rows_colmax_h(dZ, B, N, ws.in_exp, cmax, dzh, dzl, dze, colsum_ws, s);
        else split_rows_h(dZ, B, N, N, dzh, dzl, dze, s);
        __half* th = reinterpret_cast<__half*>(ws.thi.get<uint16_t>((size_t)N * K));
        __half* tl = reinterpret_cast<__half*>(ws.tlo.get<uint16_t>((size_t)N * K));
        int* te = ws.texp.get<int>(K);
        if (N <= 256 && N % 2 == 0) {
          split_t_h(d_x + m.w_off[l], N, K, th, tl, te, s);  // transpose + split in one pass
        } else {
          float* wt = ws.wt.get<float>((size_t)N * K);
          dim3 g(ceil_div(K, 32), ceil_div(N, 32));
          k_transpose<<<g, dim3(32, 8), 0, s>>>(d_x + m.w_off[l], N, K, wt); ::kp::count_launch();
          split_h(wt, K, N, N, th, tl, te, s);
        }
        EpiArgs ep{d_coeff ? kCoeff : kStore, 0, nullptr, nullptr, 0, d_coeff, S, e};
        h3_gemm(H3Operand{dzh, dzl, dze, N}, false, H3Operand{th, tl, te, N}, false, B, K, N, d_dinput, K, ep,
                false, nullptr, s);
        if (after_dinput) (*after_dinput)();
      }
      __half* dwh = reinterpret_cast<__half*>(ws.dwh.get<uint16_t>((size_t)B * N));
      __half* dwl = reinterpret_cast<__half*>(ws.dwl.get<uint16_t>((size_t)B * N));
      int* dwe = ws.dwe.get<int>(N);
      if (fuse)
        split_cols_after_h(dZ, B, N, ws.in_exp, cmax, dwh, dwl, dwe, bias_here ? d_grad + m.b_off[l] : nullptr,
                           colsum_ws, s);
      else
        split_cols_scaled_h(dZ, B, N, ws.in_exp, cmax, dwh, dwl, dwe, s, bias_here ? d_grad + m.b_off[l] : nullptr,
                            colsum_ws);
      EpiArgs plain{kStore, 0, nullptr, nullptr, 0, nullptr, 1, 1};
      h3_gemm(H3Operand{dwh, dwl, dwe, N}, true, H3Operand{ws.in_hi, ws.in_lo, nullptr, K}, true, N, K, B,
              d_grad + m.w_off[l], K, plain, true, ws.skws.get<float>(h3_splitk_ws_floats(N, K)), s,
              /*keep dZ', stream X*/ 1);
      continue;
    }
    // first layer: the input gradient goes first so its consumer can overlap
    // the weight-gradient GEMM
    if (l == 0 && d_dinput) {
      EpiArgs ep{d_coeff ? kCoeff : kStore, 0, nullptr, nullptr, 0, d_coeff, S, e};
      dx_gemm(B, K, N, dZ, d_x + m.w_off[l], d_dinput, ep, ws, s, true);
      if (after_dinput) (*after_dinput)();
    }
    // dW_l[o][i] = sum_b dZ[b][o] in[b][i]   (deterministic split-K)
    EpiArgs plain{kStore, 0, nullptr, nullptr, 0, nullptr, 1, 1};
    if (tc_enabled() && tc_worth(N, K, B, ws.tc_min_flop) && tc_gemm_supported(N, K, B, dZ, N, in, K)) {
      const int tsp = tc_splits(N, K, B);
      if (tsp == 1) {
        tc_gemm_tn(N, K, B, dZ, N, in, K, d_grad + m.w_off[l], K, 1, s);
      } else {
        float* part = ws.partials.get<float>((size_t)tsp * N * K);
        const int got = tc_gemm_tn(N, K, B, dZ, N, in, K, part, K, tsp, s);
        reduce_splits_any(part, got, (size_t)N * K, d_grad + m.w_off[l], s);
      }
    } else if (const int sp = pick_splits(N, K, B); sp == 1) {
      gemm<false, false>(N, K, B, dZ, N, in, K, d_grad + m.w_off[l], K, 1, plain, s);
    } else {
      float* part = ws.partials.get<float>((size_t)sp * N * K);
      const int got = gemm<false, false>(N, K, B, dZ, N, in, K, part, K, sp, plain, s);
      reduce_splits_any(part, got, (size_t)N * K, d_grad + m.w_off[l], s);
    }
    if (l != (int)L - 2) {  // (L-2: with the head's)
      if (csum_ready) {  // partials from the GEMM that produced dZ (one per 32-row tile)
        const int chunks = (int)ceil_div(B, 32);
        if (chunks >= 32 && N <= 4096) {
          k_reduce_chunks<<<grid_cap(ceil_div((uint64_t)N * 32, 256)), 256, 0, s>>>(
              static_cast<const float*>(ws.cpart.p), chunks, N, d_grad + m.b_off[l]);
        } else {
          k_reduce_splits<<<grid_cap(ceil_div(N, 256)), 256, 0, s>>>(static_cast<const float*>(ws.cpart.p), chunks,
                                                                      (size_t)N, d_grad + m.b_off[l]);
        }
        ::kp::count_launch();
      } else {
        colsum(dZ, nullptr, B, N, d_grad + m.b_off[l], ws, s);
      }
    }
    csum_ready = false;
    // upstream for the layer below: dX = dZ . W_l, then act' or pooling coeff
    if (l > 0) {
      float* next = ws.dz[cur ^ 1].get<float>((size_t)B * K);
      EpiArgs ep{kDAct, m.activation, nullptr, static_cast<const float*>(ws.act[l - 1].p), K, nullptr, 1, 1};
      // (the layer below's bias gradient partials from the same epilogue when
      // that layer takes the plain column-sum path: small tiles, not layer L-2)
      const char* cf_env = getenv("KP_COLSUM_FUSE");
      if (l - 1 != (int)L - 2 && !(l - 1 == 0 && ws.in_hi) && !(cf_env && cf_env[0] == '0'))
        ep.csum_part = ws.cpart.get<float>((size_t)ceil_div(B, 32) * K);
      // hidden layers: the 3xTF32 path (measured faster than fp16 at K = 128,
      // where the row-max/split passes and the A split per unit dominate)
      csum_ready = dx_gemm(B, K, N, dZ, d_x + m.w_off[l], next, ep, ws, s, false);
      cur ^= 1;
    }
  }
}

}  // namespace kp
