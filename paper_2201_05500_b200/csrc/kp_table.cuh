// Device view of the HBM embedding table + the in-place sparse rules.
#pragma once
#include "kp_internal.cuh"

namespace kp {

// Open addressing in 128-byte bucket lines: 8 slot keys u64 (bytes 0-63)
// and their 8 row indices u32 (bytes 64-95) in the same line, so one
// coalesced load of a 16-lane group (8 key lanes + 8 row lanes) resolves a
// hit; two ballots find a match / an empty slot. Rows are dense SoA fp32
// arrays w[rows][dim], s1[rows][dim] (AdaGrad acc | Adam m), s2 (Adam v).
constexpr int kSlotsPerLine = 8;
constexpr int kLineBytes = 128;
struct TView {
  uint8_t* lines;
  uint64_t* row_key;
  float* w;
  float* s1;
  float* s2;
  uint32_t* epoch;
  uint32_t* sc;  // [0] rows used, [1] row of key u64max, [2] full flag
  uint64_t bmask;
  uint64_t capacity;
  uint32_t dim;
  int rule;
  float iw, is1, is2;
  const uint32_t* abort;  // g_abort at view time (null: unguarded)
};

__host__ __device__ __forceinline__ uint64_t* line_key(uint8_t* lines, uint64_t b, int i) {
  return reinterpret_cast<uint64_t*>(lines + b * kLineBytes) + i;
}
__host__ __device__ __forceinline__ uint32_t* line_row(uint8_t* lines, uint64_t b, int i) {
  return reinterpret_cast<uint32_t*>(lines + b * kLineBytes + 64) + i;
}

inline TView view(const Table* t) {
  TView v;
  v.lines = t->d_lines;
  v.row_key = t->d_row_key;
  v.w = t->d_w;
  v.s1 = t->d_s1;
  v.s2 = t->d_s2;
  v.epoch = t->d_epoch;
  v.sc = t->d_scalars;
  v.bmask = t->nslots / kSlotsPerLine - 1;
  v.capacity = t->capacity;
  v.dim = t->dim;
  v.rule = t->rule;
  v.iw = t->init_w;
  v.is1 = t->init_s1;
  v.is2 = t->init_s2;
  v.abort = g_abort;
  return v;
}

// AdaGrad (proj/src/optimizer.cpp:86-95): acc += g*g; w -= lr*g/sqrt(acc).
// Round-to-nearest intrinsics keep the reference's expression tree (no FMA
// contraction), matching the fp32 oracle bit for bit given the same g.
__device__ __forceinline__ void adagrad1(float& w, float& acc, float g, float lr) {
  acc = __fadd_rn(acc, __fmul_rn(g, g));
  w = __fsub_rn(w, __fdiv_rn(__fmul_rn(lr, g), __fsqrt_rn(acc)));
}
// Sparse Adam = KStepEngine N=1,k=1 per row (optimizer.cpp:39-46,56-84).
__device__ __forceinline__ void adam1(float& w, float& m, float& v, float g, float lr, float b1,
                                      float b2) {
  m = __fadd_rn(__fmul_rn(b1, m), __fmul_rn(__fsub_rn(1.f, b1), g));
  v = __fadd_rn(__fmul_rn(b2, v), __fmul_rn(__fsub_rn(1.f, b2), __fmul_rn(g, g)));
  w = __fsub_rn(w, __fdiv_rn(__fmul_rn(lr, m), __fsqrt_rn(v)));
}

}  // namespace kp
