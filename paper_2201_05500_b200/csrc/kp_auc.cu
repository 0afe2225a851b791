// Online AUC on the device.
//
// Reference: compute_auc (proj/src/eval.cpp:8-39) -- rank-sum with tie
// averaging -- and AucAccumulator (eval.cpp:41-50), which pools every score
// seen so far and re-ranks on each value() call.
//
// Scores are mapped to order-preserving u32 keys and ranked by the dedup
// machinery (stable radix sort + unique + inverse + segment starts): a tie
// group g occupies sorted positions [seg[g], seg[g+1]) and its average 1-based
// rank is (seg[g] + 1 + seg[g+1]) / 2. Every partial sum of such half-integers
// is exact in f64 (< 2^52), so the positive rank-sum -- and the AUC -- is
// bit-identical to the reference's sequential loop on the same scores.
#include <cmath>
#include <vector>

#include "kp_internal.cuh"

namespace kp {
namespace {

__global__ void k_score_keys(const float* __restrict__ s, uint32_t n, uint64_t* __restrict__ keys) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t u = __float_as_uint(s[i]);
    u ^= (u >> 31) ? 0xFFFFFFFFu : 0x80000000u;  // ascending float order
    keys[i] = u;
  }
}

// per block: sum of average ranks of positives (f64, exact) and counts
__global__ void k_auc_part(const int32_t* __restrict__ labels, const uint32_t* __restrict__ inverse,
                           const uint32_t* __restrict__ seg, uint32_t n,
                           double* __restrict__ part_rank, unsigned long long* __restrict__ part_pos,
                           uint32_t* __restrict__ bad) {
  double r = 0.0;
  unsigned long long p = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t y = labels[i];
    if (y != 0 && y != 1) atomicMin(bad, i);
    if (y == 1) {
      const uint32_t g = inverse[i];
      r += 0.5 * (double)((uint64_t)seg[g] + 1 + seg[g + 1]);
      ++p;
    }
  }
  __shared__ double sr[256];
  __shared__ unsigned long long sp[256];
  sr[threadIdx.x] = r;
  sp[threadIdx.x] = p;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sr[threadIdx.x] += sr[threadIdx.x + o];
      sp[threadIdx.x] += sp[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part_rank[blockIdx.x] = sr[0];
    part_pos[blockIdx.x] = sp[0];
  }
}

}  // namespace

double device_auc(const float* d_scores, const int32_t* d_labels, uint32_t n, AucWs& ws,
                  cudaStream_t s) {
  if (n == 0) return std::nan("");
  uint64_t* keys = ws.keys.get<uint64_t>(n);
  const unsigned g = std::min<unsigned>(ceil_div(n, 256), 148 * 4);
  k_score_keys<<<g, 256, 0, s>>>(d_scores, n, keys); ::kp::count_launch();
  dedup(keys, n, ws.dd, s);
  double* pr = ws.part.get<double>(g);
  auto* pp = reinterpret_cast<unsigned long long*>(ws.part2.get<uint64_t>(g));
  uint32_t* bad = ws.bad.get<uint32_t>(1);
  KP_CUDA(cudaMemcpyAsync(bad, &n, 4, cudaMemcpyHostToDevice, s));
  k_auc_part<<<g, 256, 0, s>>>(d_labels, ws.dd.d_inverse, ws.dd.d_seg, n, pr, pp, bad); ::kp::count_launch();
  std::vector<double> hr(g);
  std::vector<unsigned long long> hp(g);
  uint32_t h_bad = n;
  KP_CUDA(cudaMemcpyAsync(hr.data(), pr, g * 8, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaMemcpyAsync(hp.data(), pp, g * 8, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaStreamSynchronize(s));
  KP_CHECK(h_bad == n, kErrGeneric, "compute_auc: label outside {0,1}");
  double prs = 0.0;
  uint64_t pos = 0;
  for (unsigned i = 0; i < g; ++i) {
    prs += hr[i];
    pos += hp[i];
  }
  const uint64_t neg = n - pos;
  if (pos == 0 || neg == 0) return std::nan("");
  const double p = (double)pos, m = (double)neg;
  return (prs - p * (p + 1.0) / 2.0) / (p * m);  // eval.cpp:36-37
}

}  // namespace kp
