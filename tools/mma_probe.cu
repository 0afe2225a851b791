// Microbenchmark: cycles per tcgen05.mma (kind::tf32 / kind::f16, M=128,
// cta_group::1) for N in {64,128,256}, A from TMEM (ts) or shared memory (ss).
// Data is whatever shared memory holds; only the issue rate is measured.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, bool F16>
__host__ __device__ constexpr uint32_t idesc() {
  // c_format f32 (bit 4); a/b format: tf32 = 2, f16 = 0
  return (1u << 4) | ((F16 ? 0u : 2u) << 7) | ((F16 ? 0u : 2u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

template <int N, bool TS, bool F16>
__global__ void __launch_bounds__(128, 1) k_probe(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t b = smem_u32(sm), a = smem_u32(sm + 65536);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i & 1) * 0);  // one accumulator
      const uint64_t bd = sdesc(b + (i & 3) * 32);
      if (TS) {
        if (F16)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(tmem + 256u + (uint32_t)((i & 3) * 8)), "l"(bd), "r"(idesc<N, F16>()), "r"(1));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(tmem + 256u + (uint32_t)((i & 3) * 8)), "l"(bd), "r"(idesc<N, F16>()), "r"(1));
      } else {
        const uint64_t ad = sdesc(a + (i & 3) * 32);
        if (F16)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(idesc<N, F16>()), "r"(1));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(idesc<N, F16>()), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool TS, bool F16>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = 2 * 65536 + 1024;
  cudaFuncSetAttribute(k_probe<N, TS, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  k_probe<N, TS, F16><<<148, 128, smem>>>(iters, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_probe<N, TS, F16><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double kk = F16 ? 16 : 8;
  const double flops = 2.0 * 128 * N * kk * iters * 148;
  printf("%-22s N=%3d: %6.1f cycles/MMA, %7.1f TFLOP/s (%s)\n", name, N, (double)cyc / iters,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, true, false>("tf32 A=TMEM");
  run<128, true, false>("tf32 A=TMEM");
  run<256, true, false>("tf32 A=TMEM");
  run<128, false, false>("tf32 A=smem");
  run<256, false, false>("tf32 A=smem");
  run<128, true, true>("f16 A=TMEM");
  run<256, true, true>("f16 A=TMEM");
  run<128, false, true>("f16 A=smem");
  run<256, false, true>("f16 A=smem");
  return 0;
}
