// Shared helpers for the sm_100a hot-path kernels.
#pragma once

#include <atomic>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace kp {

// Error kinds mirror the reference's exception hierarchy
// (proj/include/kpsim/common.hpp:13-22, store.hpp:17-20).
enum Status : int {
  kOk = 0,
  kErrGeneric = 1,   // kpsim::Error
  kErrConfig = 2,    // kpsim::ConfigError
  kErrStore = 3,     // kpsim::StoreError
  kErrCuda = 4,
  kErrNccl = 5,
  kErrTableFull = 6,
};

struct KpError : std::runtime_error {
  int status;
  KpError(int s, const std::string& w) : std::runtime_error(w), status(s) {}
};

#define KP_CUDA(x)                                                              \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess)                                                      \
      throw ::kp::KpError(::kp::kErrCuda, std::string("CUDA error ") +         \
                                              cudaGetErrorString(e_) + " at " + \
                                              __FILE__ + ":" +                  \
                                              std::to_string(__LINE__));        \
  } while (0)

#define KP_CHECK(cond, status, msg)                  \
  do {                                                \
    if (!(cond)) throw ::kp::KpError((status), (msg)); \
  } while (0)

constexpr uint64_t kEmptyKey = ~0ull;     // empty-slot sentinel (u64 max has a side slot)
constexpr uint32_t kNoRow = 0xFFFFFFFFu;

// process-wide count of kernels launched by this library (kp_launch_count)
void count_launch();
// bumped whenever a DevBuf (re)allocates: CUDA graphs captured over the old
// buffers are stale
std::atomic<uint64_t>& devbuf_generation();

inline unsigned ceil_div(uint64_t a, uint64_t b) { return (unsigned)((a + b - 1) / b); }

// Grow-only device buffer (cudaMallocAsync-free; reused across steps).
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void* ensure(size_t bytes) {
    if (bytes <= cap) return p;
    // (the new block first: a failed allocation -- e.g. refused inside a
    // CUDA-graph capture -- leaves the old one intact)
    size_t n = bytes + bytes / 4 + 256;
    void* q = nullptr;
    KP_CUDA(cudaMalloc(&q, n));
    if (p) KP_CUDA(cudaFree(p));
    p = q;
    cap = n;
    devbuf_generation().fetch_add(1, std::memory_order_relaxed);
    return p;
  }
  template <class T>
  T* get(size_t n) {
    return static_cast<T*>(ensure(n * sizeof(T)));
  }
  // grow keeping the first `used` bytes (history buffers)
  template <class T>
  T* get_keep(size_t n, size_t used_elems) {
    const size_t bytes = n * sizeof(T);
    if (bytes <= cap) return static_cast<T*>(p);
    void* q = nullptr;
    const size_t nc = bytes * 2 + 256;
    KP_CUDA(cudaMalloc(&q, nc));
    if (p && used_elems) KP_CUDA(cudaMemcpy(q, p, used_elems * sizeof(T), cudaMemcpyDeviceToDevice));
    if (p) KP_CUDA(cudaFree(p));
    p = q;
    cap = nc;
    devbuf_generation().fetch_add(1, std::memory_order_relaxed);
    return static_cast<T*>(p);
  }
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace kp
