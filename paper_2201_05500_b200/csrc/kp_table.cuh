// Device view of the HBM embedding table + the in-place sparse rules.
#pragma once
#include "kp_internal.cuh"

namespace kp {

// Open addressing: slot keys u64 [nslots] + slot rows u32 [nslots]; a bucket is
// 16 consecutive slots = one 128 B line of keys, probed by a 16-lane group with
// one coalesced load and two ballots. Rows are dense SoA fp32 arrays
// w[rows][dim], s1[rows][dim] (AdaGrad acc | Adam m), s2 (Adam v).
struct TView {
  uint64_t* keys;
  uint32_t* rows;
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

inline TView view(const Table* t) {
  TView v;
  v.keys = t->d_keys;
  v.rows = t->d_rows;
  v.row_key = t->d_row_key;
  v.w = t->d_w;
  v.s1 = t->d_s1;
  v.s2 = t->d_s2;
  v.epoch = t->d_epoch;
  v.sc = t->d_scalars;
  v.bmask = t->nslots / 16 - 1;
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
