// HBM open-addressing embedding table: insert-if-absent with fresh init,
// lookup, working-set stamps, export.
//
// Replaces TieredStore's std::unordered_map cache + resolve/fresh-init
// (proj/src/store.cpp:153-189; kFreshAccumulator=1e-6 store.hpp:49) with a
// table sized to fit HBM (the reference's cold tier / eviction are out of
// scope). Key u64max (a legitimate reference key) lives in
// a side slot so the empty sentinel never shadows it.
#include "kp_table.cuh"

namespace kp {
namespace {

constexpr uint32_t kPending = 0xFFFFFFFEu;
constexpr uint32_t kFullRow = 0xFFFFFFFDu;  // slot claimed but the table had no free row
// lanes per probing group = slots per bucket line: lane i reads slot i's key
// and row (two independent loads of the same 128-byte line), four keys per
// warp in flight
constexpr int GS = kSlotsPerLine;

__device__ __forceinline__ void init_row(const TView& t, uint32_t row, int gl) {
  const uint64_t o = (uint64_t)row * t.dim;
  for (uint32_t j = gl; j < t.dim; j += GS) {
    t.w[o + j] = t.iw;
    t.s1[o + j] = t.is1;
    if (t.rule == 1) t.s2[o + j] = t.is2;
  }
}

// One 16-lane group resolves one key. Returns the row (kNoRow if absent and
// !INSERT, or when the table is full).
template <bool INSERT>
__device__ uint32_t probe(const TView& t, uint64_t key, int gl, uint32_t gmask, int gbase) {
  if (key == kEmptyKey) {
    volatile uint32_t* side = t.sc + 1;
    uint32_t r = *side;
    if (r == kNoRow && INSERT) {
      uint32_t claim = 0;
      if (gl == 0) claim = atomicCAS(t.sc + 1, kNoRow, kPending);
      claim = __shfl_sync(gmask, claim, gbase);
      if (claim == kNoRow) {
        uint32_t row = 0;
        if (gl == 0) {
          row = atomicAdd(t.sc, 1u);
          if (row >= t.capacity) {
            t.sc[2] = 1;
            row = kNoRow;
          } else {
            t.row_key[row] = key;
          }
        }
        row = __shfl_sync(gmask, row, gbase);
        if (row != kNoRow) init_row(t, row, gl);
        __threadfence();
        if (gl == 0) *side = row;
        return row;
      }
      r = *side;
    }
    while (r == kPending) r = *side;
    return r;
  }
  uint64_t b = mix64(key) & t.bmask;
  uint64_t probes = 0;
  for (;;) {
    const uint64_t k = *(volatile uint64_t*)line_key(t.lines, b, gl);
    const uint32_t rv = *(volatile uint32_t*)line_row(t.lines, b, gl);
    const uint32_t match = (__ballot_sync(gmask, k == key) >> gbase) & 0xFFu;
    if (match) {
      const int i = __ffs(match) - 1;
      uint32_t r = __shfl_sync(gmask, rv, gbase + i);
      if (r == kNoRow && INSERT) {  // inserter in flight (same key, same launch)
        volatile uint32_t* rp = line_row(t.lines, b, i);
        while (r == kNoRow) r = *rp;
      }
      return r >= kFullRow ? kNoRow : r;
    }
    const uint32_t empty = (__ballot_sync(gmask, k == kEmptyKey) >> gbase) & 0xFFu;
    if (empty) {
      if (!INSERT) return kNoRow;
      const int el = __ffs(empty) - 1;
      unsigned long long old = 0;
      if (gl == el)
        old = atomicCAS((unsigned long long*)line_key(t.lines, b, el), (unsigned long long)kEmptyKey,
                        (unsigned long long)key);
      old = __shfl_sync(gmask, old, gbase + el);
      if (old == kEmptyKey) {
        uint32_t row = 0;
        if (gl == el) {
          row = atomicAdd(t.sc, 1u);
          if (row >= t.capacity) {
            t.sc[2] = 1;
            row = kNoRow;
          } else {
            t.row_key[row] = key;
          }
        }
        row = __shfl_sync(gmask, row, gbase + el);
        if (row != kNoRow) init_row(t, row, gl);
        __threadfence();
        if (gl == el) *(volatile uint32_t*)line_row(t.lines, b, el) = row == kNoRow ? kFullRow : row;
        return row;
      }
      if (old == key) {
        volatile uint32_t* rp = line_row(t.lines, b, el);
        uint32_t r = *rp;
        while (r == kNoRow) r = *rp;
        return r >= kFullRow ? kNoRow : r;
      }
      continue;  // lost the slot to another key: re-read this bucket
    }
    b = (b + 1) & t.bmask;
    if (++probes > t.bmask) {  // every bucket visited: no slot left
      if (gl == 0) t.sc[2] = 1;
      return kNoRow;
    }
  }
}

template <bool INSERT>
__global__ void k_probe(TView t, const uint64_t* __restrict__ keys, uint32_t n,
                        uint32_t* __restrict__ rows_out, uint32_t epoch, const uint32_t* __restrict__ d_n) {
  if (d_n) n = min(n, *d_n);
  if (INSERT && aborted(t.abort)) {
    // no inserts after a peer timeout / plan miss -- but defined outputs: the
    // rest of the (discarded) step still indexes rows with them
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
      rows_out[i] = kNoRow;
    return;
  }
  const int lane = threadIdx.x & 31;
  const int gl = lane & (GS - 1), gbase = lane & ~(GS - 1);
  const uint32_t gmask = ((1u << GS) - 1u) << gbase;
  const uint64_t g0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / GS;
  const uint64_t ng = (uint64_t)gridDim.x * blockDim.x / GS;
  // (two keys' lines in flight per group measured slower: 108 vs 95 us)
  for (uint64_t i = g0; i < n; i += ng) {
    const uint32_t r = probe<INSERT>(t, keys[i], gl, gmask, gbase);
    if (gl == 0) {
      rows_out[i] = r;
      if (epoch && r != kNoRow) t.epoch[r] = epoch;
    }
  }
}

__global__ void k_export(TView t, uint64_t nslots, uint64_t* __restrict__ out_keys,
                         uint32_t* __restrict__ out_rows, unsigned long long* __restrict__ cnt) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nslots;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = s / kSlotsPerLine;
    const int i = (int)(s % kSlotsPerLine);
    const uint32_t r = *line_row(t.lines, b, i);
    if (r < t.capacity) {
      const unsigned long long p = atomicAdd(cnt, 1ull);
      out_keys[p] = *line_key(t.lines, b, i);
      out_rows[p] = r;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t r = t.sc[1];
    if (r != kNoRow && r < t.capacity) {
      const unsigned long long p = atomicAdd(cnt, 1ull);
      out_keys[p] = kEmptyKey;
      out_rows[p] = r;
    }
  }
}

// rows of keys that are absent or not stamped with `epoch` -> min index
__global__ void k_ws_check(const uint32_t* __restrict__ rows, uint32_t n, const uint32_t* epoch_arr,
                           uint32_t epoch, uint32_t* __restrict__ first_bad) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t r = rows[i];
    if (r == kNoRow || epoch_arr[r] != epoch) atomicMin(first_bad, i);
  }
}

__global__ void k_apply_grads(TView t, const uint32_t* __restrict__ rows,
                              const float* __restrict__ grads, uint32_t n, float lr, float b1,
                              float b2) {
  if (aborted(t.abort)) return;
  const uint64_t total = (uint64_t)n * t.dim;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = q / t.dim, j = q % t.dim;
    const uint64_t o = (uint64_t)rows[i] * t.dim + j;
    const float g = grads[q];
    if (t.rule == 0) {
      float w = t.w[o], a = t.s1[o];
      adagrad1(w, a, g, lr);
      t.w[o] = w;
      t.s1[o] = a;
    } else {
      float w = t.w[o], m = t.s1[o], v = t.s2[o];
      adam1(w, m, v, g, lr, b1, b2);
      t.w[o] = w;
      t.s1[o] = m;
      t.s2[o] = v;
    }
  }
}

__global__ void k_gather_state(TView t, const uint32_t* __restrict__ rows, uint32_t n,
                               float* __restrict__ w, float* __restrict__ s1,
                               float* __restrict__ s2) {
  const uint64_t total = (uint64_t)n * t.dim;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = q / t.dim, j = q % t.dim;
    const uint32_t r = rows[i];
    const bool ok = r != kNoRow;
    const uint64_t o = (uint64_t)r * t.dim + j;
    if (w) w[q] = ok ? t.w[o] : 0.f;
    if (s1) s1[q] = ok ? t.s1[o] : 0.f;
    if (s2) s2[q] = ok && t.rule == 1 ? t.s2[o] : 0.f;
  }
}

__global__ void k_set_state(TView t, const uint32_t* __restrict__ rows, uint32_t n,
                            const float* __restrict__ w, const float* __restrict__ s1,
                            const float* __restrict__ s2) {
  const uint64_t total = (uint64_t)n * t.dim;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = q / t.dim, j = q % t.dim;
    const uint64_t o = (uint64_t)rows[i] * t.dim + j;
    if (w) t.w[o] = w[q];
    if (s1) t.s1[o] = s1[q];
    if (s2 && t.rule == 1) t.s2[o] = s2[q];
  }
}

unsigned grid_for(uint64_t work, unsigned per_block) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 148ull * 64) g = 148ull * 64;
  return (unsigned)g;
}

}  // namespace

Table* table_create(int device, uint64_t capacity, uint32_t dim, int rule, float init_w,
                    float init_s1, float init_s2) {
  KP_CHECK(capacity >= 1 && capacity < kPending, kErrStore, "table capacity must be in [1, 2^32-2]");
  KP_CHECK(dim >= 1, kErrStore, "embedding_dim must be >= 1");
  KP_CHECK(rule == 0 || rule == 1, kErrConfig, "sparse rule must be adagrad or adam");
  KP_CUDA(cudaSetDevice(device));
  auto* t = new Table();
  t->device = device;
  t->capacity = capacity;
  t->dim = dim;
  t->rule = rule;
  t->init_w = init_w;
  t->init_s1 = init_s1;
  t->init_s2 = init_s2;
  uint64_t ns = 16;
  while (ns < 2 * capacity) ns <<= 1;  // load factor <= 0.5 (>= 2 bucket lines)
  t->nslots = ns;
  try {
    KP_CUDA(cudaMalloc(&t->d_lines, ns / kSlotsPerLine * kLineBytes));
    KP_CUDA(cudaMalloc(&t->d_row_key, capacity * 8));
    KP_CUDA(cudaMalloc(&t->d_w, capacity * dim * 4));
    KP_CUDA(cudaMalloc(&t->d_s1, capacity * dim * 4));
    if (rule == 1) KP_CUDA(cudaMalloc(&t->d_s2, capacity * dim * 4));
    KP_CUDA(cudaMalloc(&t->d_epoch, capacity * 4));
    KP_CUDA(cudaMalloc(&t->d_scalars, 64));
    KP_CUDA(cudaMemset(t->d_lines, 0xFF, ns / kSlotsPerLine * kLineBytes));  // empty keys, kNoRow rows
    KP_CUDA(cudaMemset(t->d_epoch, 0, capacity * 4));
    uint32_t sc[16] = {0, kNoRow, 0, 0};
    KP_CUDA(cudaMemcpy(t->d_scalars, sc, 64, cudaMemcpyHostToDevice));
  } catch (...) {
    table_destroy(t);
    throw;
  }
  return t;
}

void table_destroy(Table* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  cudaFree(t->d_lines);
  cudaFree(t->d_row_key);
  cudaFree(t->d_w);
  cudaFree(t->d_s1);
  cudaFree(t->d_s2);
  cudaFree(t->d_epoch);
  cudaFree(t->d_scalars);
  delete t;
}

void table_pull(Table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows_out,
                bool stamp_epoch, cudaStream_t s, const uint32_t* d_n) {
  if (n == 0) return;
  // (a device count: n is an upper bound -- the occurrences; U is ~1/6 of it
  // at configs[1], the grid is sized for that and strides)
  const uint64_t work = d_n ? std::max<uint64_t>(n / 4, 1) : n;
  k_probe<true><<<grid_for(work * GS, 256), 256, 0, s>>>(view(t), d_keys, n, d_rows_out,
                                                          stamp_epoch ? t->epoch : 0, d_n); ::kp::count_launch();
}

void table_lookup(const Table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows_out,
                  cudaStream_t s) {
  if (n == 0) return;
  k_probe<false><<<grid_for((uint64_t)n * GS, 256), 256, 0, s>>>(view(t), d_keys, n, d_rows_out, 0, nullptr); ::kp::count_launch();
}

uint64_t table_size(const Table* t, cudaStream_t s) {
  uint32_t h[4];
  KP_CUDA(cudaMemcpyAsync(h, t->d_scalars, 16, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaStreamSynchronize(s));
  return h[0] < t->capacity ? h[0] : t->capacity;
}

void table_check_full(const Table* t, cudaStream_t s) {
  uint32_t h[4];
  KP_CUDA(cudaMemcpyAsync(h, t->d_scalars, 16, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaStreamSynchronize(s));
  KP_CHECK(h[2] == 0, kErrTableFull,
           "embedding table full: capacity " + std::to_string(t->capacity) + " rows");
}

// ---- helpers used by the C ABI (TieredStore surface) ---------------------
void table_export(const Table* t, uint64_t* d_keys_out, uint32_t* d_rows_out,
                  unsigned long long* d_cnt, cudaStream_t s) {
  KP_CUDA(cudaMemsetAsync(d_cnt, 0, 8, s));
  k_export<<<grid_for(t->nslots, 256), 256, 0, s>>>(view(t), t->nslots, d_keys_out, d_rows_out, d_cnt); ::kp::count_launch();
}

void table_ws_check(const Table* t, const uint32_t* d_rows, uint32_t n, uint32_t* d_first_bad,
                    cudaStream_t s) {
  KP_CUDA(cudaMemcpyAsync(d_first_bad, &n, 4, cudaMemcpyHostToDevice, s));
  if (n) k_ws_check<<<grid_for(n, 256), 256, 0, s>>>(d_rows, n, t->d_epoch, t->epoch, d_first_bad); ::kp::count_launch();
}

void table_apply(Table* t, const uint32_t* d_rows, const float* d_grads, uint32_t n, float lr,
                 float b1, float b2, cudaStream_t s) {
  if (n == 0) return;
  k_apply_grads<<<grid_for((uint64_t)n * t->dim, 256), 256, 0, s>>>(view(t), d_rows, d_grads, n,
                                                                     lr, b1, b2); ::kp::count_launch();
}

void table_set_rows(Table* t, const uint32_t* d_rows, uint32_t n, const float* d_w,
                    const float* d_s1, const float* d_s2, cudaStream_t s) {
  if (n == 0) return;
  k_set_state<<<grid_for((uint64_t)n * t->dim, 256), 256, 0, s>>>(view(t), d_rows, n, d_w, d_s1, d_s2); ::kp::count_launch();
}

void table_gather(const Table* t, const uint32_t* d_rows, uint32_t n, float* d_w, float* d_s1,
                  float* d_s2, cudaStream_t s) {
  if (n == 0) return;
  k_gather_state<<<grid_for((uint64_t)n * t->dim, 256), 256, 0, s>>>(view(t), d_rows, n, d_w, d_s1,
                                                                      d_s2); ::kp::count_launch();
}

}  // namespace kp
