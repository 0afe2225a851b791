// The C ABI (include/kpsim_b200.h) and the per-batch trainer orchestration.
//
// Trainer::process_batch (proj/src/trainer.cpp:115-259) becomes, per
// minibatch step on each rank:
//   dedup(step keys) -> [G>1: owner bucket, key all-to-all, owner dedup]
//   -> table pull (insert-if-absent) -> [G>1: row all-to-all] -> bag pooling
//   -> per local worker MLP fwd/bwd -> segmented reduce by unique key
//   -> [G>1: grad all-to-all, owner reduce in source order] -> x 1/N + rule
//   -> dense k-step Adam (allgather + centered mean at merges).
// NCCL runs on the trainer's stream; one process per GPU.
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <map>
#include <set>
#include <tuple>
#include <vector>

#include "kp_table.cuh"
#include "../../include/kpsim_b200.h"

using namespace kp;

namespace {
thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return KP_OK;
  } catch (const KpError& e) {
    return set_err(e.status, e.what());
  } catch (const std::exception& e) {
    return set_err(KP_ERR, e.what());
  }
}

#define KP_NCCL(x)                                                                        \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      throw KpError(kErrNccl, std::string("NCCL error ") + ncclGetErrorString(r_) + " at " + \
                                  __FILE__ + ":" + std::to_string(__LINE__));             \
  } while (0)

cudaStream_t st(kp_stream s) { return reinterpret_cast<cudaStream_t>(s); }

__global__ void k_gather_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx,
                             uint32_t n, uint64_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}
__global__ void k_compose(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint32_t n,
                          uint32_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a[b[i]];
}
__global__ void k_key_range(uint64_t start, uint64_t step, uint32_t n, uint64_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = start + (uint64_t)i * step;
}
unsigned grid1(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, 148 * 16));
}
}  // namespace

thread_local const uint32_t* kp::g_abort = nullptr;
std::atomic<uint64_t> g_launches{0};
void kp::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
std::atomic<uint64_t>& kp::devbuf_generation() {
  static std::atomic<uint64_t> g{0};
  return g;
}

struct MergeWs {
  DevBuf allg, cm, terms, chunk, full;
};

struct kp_table {
  Table* t = nullptr;
  cudaStream_t s = nullptr;
  DevBuf keys, rows, w, s1, s2, grads, scratch;
};

struct kp_comm {
  ncclComm_t nc = nullptr;
  ncclComm_t nc2 = nullptr;  // second channel: gradient exchange overlapping the GEMM
  int rank = 0, world = 1, device = 0;
};

// ---------------------------------------------------------------------------
struct kp_trainer {
  kp_trainer_config cfg{};
  int device = 0;
  cudaStream_t s = nullptr;
  kp_comm* comm = nullptr;
  int rank = 0, world = 1;
  uint32_t W = 1, N = 1, S = 1, e = 1;
  MlpShape shape;
  kp_table tab;
  float *x = nullptr, *m = nullptr, *v = nullptr, *vbar = nullptr, *g = nullptr;
  uint64_t D = 0;
  uint64_t t_global = 0, merges = 0;
  // all replicas (every worker on every rank) hold the same x: initial state
  // and right after a merge. Cleared by local steps and set_worker_state
  // (which, with several ranks, must be called symmetrically on all of them).
  bool x_uniform = true;
  // inputs
  DevBuf in_offs, in_keys, in_slots, in_labels;
  std::vector<uint32_t> h_offs;
  // double-buffered staged batches (H2D on a copy stream overlapping compute)
  struct Staged {
    DevBuf offs, keys, slots, labels;
    uint32_t n = 0;
    bool has_slots = false, ready = false, used_set = false;
    cudaEvent_t ev = nullptr;    // H2D of this slot done (copy stream)
    cudaEvent_t used = nullptr;  // last step reading this slot done (compute stream)
    // H2D not issued yet (host sources, caller-owned until train_staged)
    bool pending = false;
    const uint32_t* h_src_offs = nullptr;
    const uint64_t* h_src_keys = nullptr;
    const uint16_t* h_src_slots = nullptr;
    const int32_t* h_src_labels = nullptr;
  } stage[2];
  cudaStream_t copy_s = nullptr;
  // gradient exchange stream (G > 1): the all-to-all overlaps the last GEMM
  cudaStream_t xs = nullptr;
  cudaEvent_t ev_dinput = nullptr, ev_xdone = nullptr;
  // step buffers
  DevBuf st_offs, st_keys, st_slots, st_labels;
  DedupWs dd, dd_owner;
  ShardWs sh;
  SegWs sg, sg_owner;
  MlpWs mlp;
  MergeWs mws;
  AucWs aucws;
  DevBuf hist_scores, hist_labels, all_preds, all_labels, gather_tmp;
  uint64_t hist_n = 0;
  DevBuf rows, rowocc, bag_offs, bag_of_occ, pooled, inv_count, dpooled, preds, err, loss, check;
  DevBuf inst_max;  // max |pooled row| per instance, from the pool kernel
  // planes mode: the pooling kernel writes the first layer's input as fp16
  // hi/lo planes (in the `pooled` buffer, same bytes) + an exponent per instance
  bool planes = false;
  // this step's first layer gathers its rows (one feature per slot, planes;
  // KP_FUSED_POOL=1 at trainer creation; else the pooling pass writes the planes)
  bool fused_pool = false;
  bool ga_on = false;
  const float* ga_src = nullptr;
  uint64_t ga_nrows = 0;
  const uint32_t* ga_rowocc = nullptr;
  DevBuf umax;
  DevBuf inst_exp;
  const __half* plane_hi(size_t nb) const { return static_cast<const __half*>(pooled.p); }
  const __half* plane_lo(size_t nb) const { return static_cast<const __half*>(pooled.p) + nb * e; }
  DevBuf xbar, pred_keep, lossg;
  // exchange buffers (G > 1)
  DevBuf perm, pos, send_keys, recv_keys, owner_rows, owner_idx, send_rows, recv_rows, send_grads,
      recv_grads, counts_dev;
  std::vector<uint64_t> cnt_send, cnt_recv, off_send, off_recv;
  std::vector<uint64_t> mat;  // [R][R] unique keys rank p sends to owner q (mat[p*R+q])
  // NVLink peer windows (kp_peer.cu); mode -1 undecided, 0 NCCL, 1 peer
  struct PeerWin {
    void* local = nullptr;
    size_t bytes = 0;
    bool owned = true;  // false: an exported trainer buffer (x, v)
    std::vector<void*> remote;
  };
  struct {
    int mode = -1;
    PeerWin keys, rows, grads, flags;
    PeerWin dv, dx, dm, vb;  // k-step merge over NVLink (the trainer's v, x, m; v_bar)
    uint64_t seq[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    DevBuf scratch;
  } peer;
  // communication ledger (ledger.hpp TransferCategory order): bytes this
  // rank SENT over NVLink, and the transmissions (one per peer and step)
  uint64_t led_bytes[5] = {0, 0, 0, 0, 0}, led_count[5] = {0, 0, 0, 0, 0};
  // dense trajectory (Trainer::dense_trajectory, trainer.cpp:215-227), opt-in
  struct TrajStep {
    uint64_t step = 0;
    int merged = 0;
    double loss = 0, a3 = 0;
    std::vector<float> x_bar, v_bar;
  };
  bool traj_on = false;
  // sync-free single-GPU step: no dedup readback -- the pass
  // plan and the one-feature-per-slot layout are predicted from the previous
  // batch and checked on the device (kAbortPlan: the batch wrote nothing and
  // is rerun with the readbacks)
  bool async_step = false, force_sync = false, pred_ident = false;
  bool sync_free = true;  // KP_SYNC_FREE=0 at trainer creation: every step reads back
  // The sync-free single-GPU batch as a CUDA graph (KP_GRAPH=0 at trainer
  // creation: off): captured the first time a batch with these inputs
  // (pointers, sizes) and step-dependent choices runs sync-free, replayed
  // after; the readbacks land in pinned host memory.
  bool graphs = true;
  struct GraphKey {
    const void* p[4];
    uint64_t n, n_occ, gn, gfirst;
    int flags;  // predict_first | preds | fused | merged | pred_ident
    int spec;
    bool operator<(const GraphKey& o) const {
      return std::tie(p[0], p[1], p[2], p[3], n, n_occ, gn, gfirst, flags, spec) <
             std::tie(o.p[0], o.p[1], o.p[2], o.p[3], o.n, o.n_occ, o.gn, o.gfirst, o.flags, o.spec);
    }
  };
  struct GraphEnt {
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
  };
  std::map<GraphKey, GraphEnt> gcache;
  std::set<GraphKey> gseen;
  uint64_t ggen = 0;  // devbuf generation the cache was built at
  void graphs_clear() {
    for (auto& kv : gcache)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    gcache.clear();
  }
  // pinned readback block: [0..1] err words, [2..3] check words, [4] U,
  // [5..8] table scalars; then the losses (double) and the predictions
  uint32_t* rb = nullptr;
  size_t rb_bytes = 0;
  void* rb_ensure(size_t bytes) {
    if (bytes > rb_bytes) {
      if (rb) cudaFreeHost(rb);
      graphs_clear();  // captured graphs point at the old block
      KP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&rb), bytes));
      rb_bytes = bytes;
    }
    return rb;
  }
  DevBuf pflag;           // G > 1: the local dedup's plan-miss flag (travels with the counts)
  std::vector<TrajStep> traj;
  std::vector<float> traj_prev_vbar;  // frozen v_bar before the step (a3)
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  double stage_ms[7] = {0};
  uint64_t prof_steps = 0, prof_unique = 0, prof_occ = 0, prof_owner_unique = 0, prof_recv = 0;
  std::vector<std::pair<int, int>> marks;  // (stage, event index) pairs for this batch
  int ev_used = 0;

  cudaEvent_t next_event() {
    if (ev_used >= (int)ev.size()) {
      cudaEvent_t e;
      KP_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
    return ev[ev_used++];
  }
  // mark the END of `stage` (the previous mark is its start)
  void mark(int stage) {
    static const bool dbg = getenv("KP_SYNC_DEBUG") != nullptr;
    if (dbg) {  // localise asynchronous faults to a stage
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess)
        throw KpError(kErrCuda, std::string("stage ") + std::to_string(stage) + ": " + cudaGetErrorString(e));
    }
    if (!prof) return;
    cudaEvent_t e = next_event();
    KP_CUDA(cudaEventRecord(e, s));
    marks.push_back({stage, ev_used - 1});
  }
  void harvest() {
    if (!prof) return;
    KP_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 1; i < marks.size(); ++i) {
      if (marks[i].first < 0) continue;
      float ms = 0;
      KP_CUDA(cudaEventElapsedTime(&ms, ev[marks[i - 1].second], ev[marks[i].second]));
      stage_ms[marks[i].first] += ms;
    }
    marks.clear();
    ev_used = 0;
  }
  ~kp_trainer() {
    for (auto e : ev) cudaEventDestroy(e);
    for (auto& st : stage) {
      if (st.ev) cudaEventDestroy(st.ev);
      if (st.used) cudaEventDestroy(st.used);
    }
    if (copy_s) cudaStreamDestroy(copy_s);
    if (xs) cudaStreamDestroy(xs);
    for (PeerWin* w : {&peer.keys, &peer.rows, &peer.grads, &peer.flags, &peer.dv, &peer.dx,
                       &peer.dm, &peer.vb}) {
      for (size_t p = 0; p < w->remote.size(); ++p)
        if (w->remote[p] && w->remote[p] != w->local) cudaIpcCloseMemHandle(w->remote[p]);
      if (w->local && w->owned) cudaFree(w->local);
    }
    graphs_clear();
    if (rb) cudaFreeHost(rb);
    if (ev_dinput) cudaEventDestroy(ev_dinput);
    if (ev_xdone) cudaEventDestroy(ev_xdone);
    if (tab.t) table_destroy(tab.t);
    if (tab.s) cudaStreamDestroy(tab.s);
    cudaFree(x);
    cudaFree(m);
    cudaFree(v);
    cudaFree(vbar);
    cudaFree(g);
    if (s) cudaStreamDestroy(s);
  }
};

namespace {

void all_to_all(kp_trainer* tr, const void* send, const std::vector<uint64_t>& scnt,
                const std::vector<uint64_t>& soff, void* recv, const std::vector<uint64_t>& rcnt,
                const std::vector<uint64_t>& roff, size_t elem, ncclDataType_t dt,
                cudaStream_t st = nullptr, ncclComm_t nc = nullptr) {
  if (!st) st = tr->s;
  if (!nc) nc = tr->comm->nc;
  const int R = tr->world, me = tr->rank;
  auto* sb = static_cast<const char*>(send);
  auto* rb = static_cast<char*>(recv);
  const size_t dts = (dt == ncclUint64 || dt == ncclFloat64) ? 8 : 4;
  const size_t per = elem / dts;  // datatype elements per logical element
  if (scnt[me])
    KP_CUDA(cudaMemcpyAsync(rb + roff[me] * elem, sb + soff[me] * elem, scnt[me] * elem,
                            cudaMemcpyDeviceToDevice, st));
  KP_NCCL(ncclGroupStart());
  for (int p = 0; p < R; ++p) {
    if (p == me) continue;
    if (scnt[p]) KP_NCCL(ncclSend(sb + soff[p] * elem, scnt[p] * per, dt, p, nc, st));
    if (rcnt[p]) KP_NCCL(ncclRecv(rb + roff[p] * elem, rcnt[p] * per, dt, p, nc, st));
  }
  KP_NCCL(ncclGroupEnd());
}


// Chunked exchange for the merge (SURVEY.md 8e "recommended merge for large
// D"): rank c owns chunk c = [c*C, c*C + len_c) of the D parameters and
// receives every global worker's slice of it, [N][C] in ascending global
// worker order (rank-major, then local worker).
void exchange_chunks(kp_comm* comm, cudaStream_t s, uint32_t W, uint64_t D, uint64_t C,
                     const float* src, float* dst) {
  const int R = comm->world, me = comm->rank;
  const uint64_t my_len = std::min<uint64_t>(C, D > me * C ? D - me * C : 0);
  KP_NCCL(ncclGroupStart());
  for (int p = 0; p < R; ++p) {
    const uint64_t len_p = std::min<uint64_t>(C, D > p * C ? D - p * C : 0);
    for (uint32_t l = 0; l < W; ++l) {
      const float* sp = src + (size_t)l * D + (size_t)p * C;
      float* rp = dst + ((size_t)p * W + l) * C;
      if (p == me) {
        if (my_len) KP_CUDA(cudaMemcpyAsync(dst + ((size_t)me * W + l) * C, sp, my_len * 4,
                                            cudaMemcpyDeviceToDevice, s));
        continue;
      }
      if (len_p) KP_NCCL(ncclSend(sp, len_p, ncclFloat32, p, comm->nc, s));
      if (my_len) KP_NCCL(ncclRecv(rp, my_len, ncclFloat32, p, comm->nc, s));
    }
  }
  KP_NCCL(ncclGroupEnd());
}

// global_merge (optimizer.cpp:56-84) over W local workers x all ranks; moments
// already accumulated. v_bar = cmean(v_i); x_i = cmean(x_j - a m_j/sqrt(v_bar)).
// Multi-rank: two rounds (v, then the term) of chunk exchange -> owner
// centered mean over its chunk -> allgather, ~2*2*(R-1)/R*4D bytes per rank.
// The centered mean is elementwise in a fixed worker order, so the result is
// bitwise the one a single process computes over all N workers.
void merge_states(kp_comm* comm, cudaStream_t s, uint32_t W, uint64_t D, float* x, float* m,
                  float* v, float* vbar, float alpha, bool reset, MergeWs& ws) {
  const bool local = !comm || comm->world == 1;
  if (local && W == 1) {
    merge_single(x, m, v, vbar, D, alpha, reset, s);
    return;
  }
  float* vb = ws.cm.get<float>(D);
  float* terms = ws.terms.get<float>((size_t)W * D);
  // small models / few ranks: one allgather per round beats the three-step
  // chunked exchange on latency; same fixed-order arithmetic either way
  const bool gather_all = !local && (uint64_t)(comm->world - 1) * W * D * 4 <= (24ull << 20);
  if (local || gather_all) {
    const uint32_t N = W * (local ? 1 : comm->world);
    float* all = local ? nullptr : ws.allg.get<float>((size_t)N * D);
    if (!local) KP_NCCL(ncclAllGather(v, all, (size_t)W * D, ncclFloat32, comm->nc, s));
    centered_mean(local ? v : all, D, N, D, vb, s);
    for (uint32_t l = 0; l < W; ++l) merge_terms(x + l * D, m + l * D, vb, D, alpha, terms + l * D, s);
    if (!local) KP_NCCL(ncclAllGather(terms, all, (size_t)W * D, ncclFloat32, comm->nc, s));
    centered_mean(local ? terms : all, D, N, D, x, s);  // merged x into worker 0
  } else {
    const int R = comm->world, me = comm->rank;
    const uint32_t N = W * R;
    const uint64_t C = (D + R - 1) / R;
    const uint64_t my_len = std::min<uint64_t>(C, D > me * C ? D - me * C : 0);
    float* recv = ws.allg.get<float>((size_t)N * C);
    float* mine = ws.chunk.get<float>(C);
    float* full = ws.full.get<float>((size_t)R * C);
    // round 1: v_bar
    exchange_chunks(comm, s, W, D, C, v, recv);
    KP_CUDA(cudaMemsetAsync(mine, 0, C * 4, s));
    if (my_len) centered_mean(recv, C, N, my_len, mine, s);
    KP_NCCL(ncclAllGather(mine, full, C, ncclFloat32, comm->nc, s));
    KP_CUDA(cudaMemcpyAsync(vb, full, D * 4, cudaMemcpyDeviceToDevice, s));
    // round 2: x = cmean(x_j - a m_j / sqrt(v_bar))
    for (uint32_t l = 0; l < W; ++l) merge_terms(x + l * D, m + l * D, vb, D, alpha, terms + l * D, s);
    exchange_chunks(comm, s, W, D, C, terms, recv);
    KP_CUDA(cudaMemsetAsync(mine, 0, C * 4, s));
    if (my_len) centered_mean(recv, C, N, my_len, mine, s);
    KP_NCCL(ncclAllGather(mine, full, C, ncclFloat32, comm->nc, s));
    KP_CUDA(cudaMemcpyAsync(x, full, D * 4, cudaMemcpyDeviceToDevice, s));
  }
  for (uint32_t l = 0; l < W; ++l) {
    if (l) KP_CUDA(cudaMemcpyAsync(x + l * D, x, D * 4, cudaMemcpyDeviceToDevice, s));
    KP_CUDA(cudaMemcpyAsync(vbar + l * D, vb, D * 4, cudaMemcpyDeviceToDevice, s));
    if (reset) KP_CUDA(cudaMemcpyAsync(v + l * D, vb, D * 4, cudaMemcpyDeviceToDevice, s));
  }
}

void compute_xbar(kp_trainer* tr, float* out) {
  const uint64_t D = tr->D;
  if (tr->x_uniform) {
    // every replica holds the same x (initial state, or just merged): the
    // centered mean of identical vectors is that vector, bit for bit
    KP_CUDA(cudaMemcpyAsync(out, tr->x, D * 4, cudaMemcpyDeviceToDevice, tr->s));
    return;
  }
  if (tr->world == 1) {
    centered_mean(tr->x, D, tr->N, D, out, tr->s);
    return;
  }
  const int R = tr->world, me = tr->rank;
  const uint64_t C = (D + R - 1) / R;
  const uint64_t my_len = std::min<uint64_t>(C, D > me * C ? D - me * C : 0);
  float* recv = tr->mws.allg.get<float>((size_t)tr->N * C);
  float* mine = tr->mws.chunk.get<float>(C);
  float* full = tr->mws.full.get<float>((size_t)R * C);
  exchange_chunks(tr->comm, tr->s, tr->W, D, C, tr->x, recv);
  KP_CUDA(cudaMemsetAsync(mine, 0, C * 4, tr->s));
  if (my_len) centered_mean(recv, C, tr->N, my_len, mine, tr->s);
  KP_NCCL(ncclAllGather(mine, full, C, ncclFloat32, tr->comm->nc, tr->s));
  KP_CUDA(cudaMemcpyAsync(out, full, D * 4, cudaMemcpyDeviceToDevice, tr->s));
}

struct StepView {
  const uint32_t* offs;  // device, n_inst+1 entries, absolute values with occ_base
  uint32_t occ_base;
  const uint64_t* keys;  // device, starting at the step's first occurrence
  const uint16_t* slots;
  const int32_t* labels;
  uint32_t n_inst, n_occ;
  std::vector<uint32_t> wlo, whi;  // local worker instance ranges in step coords
};

// Embedding stage for a step: dedup, (exchange), pull, pool. Leaves the
// segment structure in tr->dd and the per-unique source index for the push.
struct PullResult {
  const float* src;
  const uint32_t* idx;
  uint32_t U;          // unique keys (an upper bound when dU is set)
  const uint32_t* dU;  // U on the device (sync-free step), else null
};

// ---- NVLink peer windows ------------------------------------------------
// all ranks: min over ranks of `ok` (also a barrier)
bool all_ok(kp_trainer* tr, bool ok) {
  int* d = tr->peer.scratch.get<int>(2);
  const int h = ok ? 1 : 0;
  KP_CUDA(cudaMemcpyAsync(d, &h, 4, cudaMemcpyHostToDevice, tr->s));
  KP_NCCL(ncclAllReduce(d, d + 1, 1, ncclInt32, ncclMin, tr->comm->nc, tr->s));
  int r = 0;
  KP_CUDA(cudaMemcpyAsync(&r, d + 1, 4, cudaMemcpyDeviceToHost, tr->s));
  KP_CUDA(cudaStreamSynchronize(tr->s));
  return r == 1;
}

void win_release(kp_trainer* tr, kp_trainer::PeerWin& w) {
  if (!w.local) return;
  KP_CUDA(cudaStreamSynchronize(tr->s));
  all_ok(tr, true);  // every rank is past its last use of the window
  for (size_t p = 0; p < w.remote.size(); ++p)
    if (w.remote[p] && w.remote[p] != w.local) cudaIpcCloseMemHandle(w.remote[p]);
  all_ok(tr, true);  // every mapping of ours is closed
  if (w.owned) KP_CUDA(cudaFree(w.local));
  w.local = nullptr;
  w.remote.clear();
  w.bytes = 0;
}

// collective: (re)allocate a window of `bytes` on every rank (or export the
// existing allocation `existing`) and map the peers'
bool win_alloc(kp_trainer* tr, kp_trainer::PeerWin& w, size_t bytes, void* existing = nullptr) {
  const int R = tr->world, me = tr->rank;
  win_release(tr, w);
  if (existing) {
    w.local = existing;
    w.owned = false;
  } else {
    KP_CUDA(cudaMalloc(&w.local, bytes));
    KP_CUDA(cudaMemset(w.local, 0, bytes));
    w.owned = true;
  }
  w.bytes = bytes;
  cudaIpcMemHandle_t h;
  bool ok = cudaIpcGetMemHandle(&h, w.local) == cudaSuccess;
  cudaGetLastError();
  char* d = tr->peer.scratch.get<char>((size_t)R * 64 + 64);
  KP_CUDA(cudaMemcpyAsync(d + (size_t)me * 64, &h, 64, cudaMemcpyHostToDevice, tr->s));
  KP_NCCL(ncclAllGather(d + (size_t)me * 64, d, 64, ncclChar, tr->comm->nc, tr->s));
  std::vector<cudaIpcMemHandle_t> hs(R);
  KP_CUDA(cudaMemcpyAsync(hs.data(), d, (size_t)R * 64, cudaMemcpyDeviceToHost, tr->s));
  KP_CUDA(cudaStreamSynchronize(tr->s));
  w.remote.assign(R, nullptr);
  for (int p = 0; p < R; ++p) {
    if (p == me) {
      w.remote[p] = w.local;
      continue;
    }
    if (ok && cudaIpcOpenMemHandle(&w.remote[p], hs[p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      w.remote[p] = nullptr;
      ok = false;
    }
  }
  return ok;
}

// Decide (collectively) whether this step's exchange runs over peer windows,
// growing them when the global counts matrix needs more room. Every rank holds
// the same matrix, so every rank takes the same decisions.
bool peer_ready(kp_trainer* tr) {
  auto& P = tr->peer;
  if (P.mode == 0) return false;
  const int R = tr->world;
  if (P.mode == -1) {
    const char* e = getenv("KP_PEER");
    if (R > kMaxPeers || (e && e[0] == '0')) {
      P.mode = 0;
      return false;
    }
  }
  uint64_t maxcol = 1, maxrow = 1;
  for (int r = 0; r < R; ++r) {
    uint64_t c = 0, w = 0;
    for (int p = 0; p < R; ++p) {
      c += tr->mat[(size_t)p * R + r];
      w += tr->mat[(size_t)r * R + p];
    }
    maxcol = std::max(maxcol, c);
    maxrow = std::max(maxrow, w);
  }
  const size_t row = (size_t)tr->e * 4;
  auto room = [](uint64_t n, size_t b) { return (size_t)((n + n / 4 + 1024) * b); };
  // every grow decision below depends only on the shared counts matrix, so
  // all ranks (re)allocate the same windows; `grew` makes the agreement
  // collective whenever any window changed, on every rank alike
  bool ok = true, grew = false;
  if (P.mode == -1) ok = win_alloc(tr, P.flags, 8 * kMaxPeers * 8);
  if (P.keys.bytes < maxcol * 8) ok = win_alloc(tr, P.keys, room(maxcol, 8)) && ok, grew = true;
  if (P.grads.bytes < maxcol * row) ok = win_alloc(tr, P.grads, room(maxcol, row)) && ok, grew = true;
  if (P.rows.bytes < maxrow * row) ok = win_alloc(tr, P.rows, room(maxrow, row)) && ok, grew = true;
  const bool first = P.mode == -1;
  if (first) {
    // the k-step merge's windows too, now: a one-time collective setup must
    // not land in the middle of a run (the first merge may be k steps away)
    const uint64_t D = tr->D;
    const uint32_t W = tr->W;
    ok = win_alloc(tr, P.dv, (size_t)W * D * 4, tr->v) && ok;
    ok = win_alloc(tr, P.dx, (size_t)W * D * 4, tr->x) && ok;
    ok = win_alloc(tr, P.dm, (size_t)W * D * 4, tr->m) && ok;
    ok = win_alloc(tr, P.vb, (size_t)D * 4) && ok;
  }
  if (first || grew) {
    P.mode = all_ok(tr, ok) ? 1 : 0;
    if (P.mode == 0)
      for (auto* w : {&P.keys, &P.rows, &P.grads, &P.flags, &P.dv, &P.dx, &P.dm, &P.vb})
        win_release(tr, *w);
  }
  return P.mode == 1;
}

// phase 0 keys (requester -> owner), 2 grads (requester -> owner): element i of
// the local send order goes to owner p's window after the segments of the
// lower ranks; phase 1 rows (owner -> requester): received element i goes
// back to requester p's window at p's own send position.
PeerMap peer_map(kp_trainer* tr, int phase, uint32_t n_local) {
  const int R = tr->world, me = tr->rank;
  const auto& P = tr->peer;
  PeerMap pm{};
  pm.R = R;
  const size_t row = (size_t)tr->e * 4;
  pm.stride = phase == 0 ? 8 : (uint32_t)row;
  const kp_trainer::PeerWin& w = phase == 0 ? P.keys : phase == 1 ? P.rows : P.grads;
  for (int p = 0; p < R; ++p) {
    uint64_t before = 0;  // my segment's offset inside p's window
    for (int q = 0; q < me; ++q) before += phase == 1 ? tr->mat[(size_t)p * R + q] : tr->mat[(size_t)q * R + p];
    pm.start[p] = (uint32_t)(phase == 1 ? tr->off_recv[p] : tr->off_send[p]);
    pm.base[p] = reinterpret_cast<uintptr_t>(w.remote[p]) + before * pm.stride;
  }
  pm.start[R] = n_local;
  return pm;
}

void peer_exchange_sync(kp_trainer* tr, int phase, bool signal, bool wait,
                        cudaStream_t sig_stream = nullptr) {
  const int R = tr->world, me = tr->rank;
  auto& P = tr->peer;
  if (signal) {
    PeerFlags f{};
    for (int p = 0; p < R; ++p)
      f.flag[p] = reinterpret_cast<uintptr_t>(P.flags.remote[p]) + ((size_t)phase * kMaxPeers + me) * 8;
    peer_signal(f, R, ++P.seq[phase], sig_stream ? sig_stream : tr->s);
  }
  if (wait)
    peer_wait(static_cast<const uint64_t*>(P.flags.local) + (size_t)phase * kMaxPeers, R, P.seq[phase],
              static_cast<uint32_t*>(tr->check.p), tr->s);
}

// k-step merge over NVLink (peer mode): the owner of chunk c reads every
// rank's workers' v (then x - a m / sqrt(v_bar)) for its chunk straight from
// their HBM, computes the fixed-order centered mean and stores the result into
// every rank; four flag phases order the rounds. Same arithmetic and worker
// order as merge_states, so the result is bitwise the same.
void merge_states_peer(kp_trainer* tr, float alpha, bool reset) {
  auto& P = tr->peer;
  const int R = tr->world, me = tr->rank;
  const uint32_t W = tr->W;
  const uint64_t D = tr->D;
  cudaStream_t s = tr->s;
  KP_CHECK(P.dv.local != nullptr, kErrCuda, "peer merge: dense-state windows not mapped");
  const uint64_t C = (D + R - 1) / R;
  const uint64_t c0 = std::min<uint64_t>(D, (uint64_t)me * C), c1 = std::min<uint64_t>(D, c0 + C);
  // one round: every rank's v, x and m are final -> each owner merges its
  // chunk straight from the peers' buffers into every rank -> all stored
  peer_exchange_sync(tr, 3, true, true);
  PeerMerge pm{};
  for (int p = 0; p < R; ++p) {
    pm.v[p] = reinterpret_cast<uintptr_t>(P.dv.remote[p]);
    pm.x[p] = reinterpret_cast<uintptr_t>(P.dx.remote[p]);
    pm.m[p] = reinterpret_cast<uintptr_t>(P.dm.remote[p]);
    pm.vb[p] = reinterpret_cast<uintptr_t>(P.vb.remote[p]);
  }
  peer_merge(pm, R, W, D, c0, c1, alpha, s);
  peer_exchange_sync(tr, 4, true, true);  // v_bar and x complete everywhere
  const float* vb = static_cast<const float*>(P.vb.local);
  float* x = tr->x;
  // guarded copies (not cudaMemcpy): a timed-out merge must not publish v_bar
  for (uint32_t l = 0; l < W; ++l) {
    if (l) dense_copy(x + l * D, x, D, s);
    dense_copy(tr->vbar + l * D, vb, D, s);
    if (reset) dense_copy(tr->v + l * D, vb, D, s);
  }
}

// Issue the H2D of staged batches waiting for it (one slot, or all with
// slot < 0). The copy is ordered after the last step that read the slot.
void issue_staged(kp_trainer* tr, int slot) {
  for (int i = 0; i < 2; ++i) {
    if (slot >= 0 && i != slot) continue;
    auto& st = tr->stage[i];
    if (!st.pending) continue;
    if (st.used_set) KP_CUDA(cudaStreamWaitEvent(tr->copy_s, st.used, 0));
    const uint32_t n = st.n, O = st.h_src_offs[n];
    KP_CUDA(cudaMemcpyAsync(st.offs.p, st.h_src_offs, (size_t)(n + 1) * 4, cudaMemcpyHostToDevice, tr->copy_s));
    KP_CUDA(cudaMemcpyAsync(st.keys.p, st.h_src_keys, (size_t)O * 8, cudaMemcpyHostToDevice, tr->copy_s));
    if (st.has_slots)
      KP_CUDA(cudaMemcpyAsync(st.slots.p, st.h_src_slots, (size_t)O * 2, cudaMemcpyHostToDevice, tr->copy_s));
    KP_CUDA(cudaMemcpyAsync(st.labels.p, st.h_src_labels, (size_t)n * 4, cudaMemcpyHostToDevice, tr->copy_s));
    KP_CUDA(cudaEventRecord(st.ev, tr->copy_s));
    st.pending = false;
  }
}

PullResult pull_and_pool(kp_trainer* tr, const StepView& sv, bool stamp) {
  cudaStream_t s = tr->s;
  // bags first, so dedup can emit the bag of every sorted position
  const uint32_t nb = sv.n_inst * tr->S;
  uint32_t* bag_offs = tr->bag_offs.get<uint32_t>(nb + 1);
  uint32_t* bag_of_occ = tr->bag_of_occ.get<uint32_t>(std::max<uint32_t>(sv.n_occ, 1));
  uint32_t* err = tr->err.get<uint32_t>(4);
  uint32_t* chk = static_cast<uint32_t*>(tr->check.p);
  // (sync-free, predicted one feature per slot on the planes path: the bag
  // maps are the identity and unread -- only the checks run; the device
  // check of the prediction aborts the step otherwise)
  const bool skip_maps = tr->async_step && tr->pred_ident && tr->planes && sv.n_occ == nb &&
                         planes_ident_kernel(tr->S, tr->e) && !tr->fused_pool &&
                         dedup_async_ready(tr->dd, sv.n_occ);
  prepare_bags(sv.offs, sv.occ_base, sv.slots, sv.n_inst, tr->S, bag_offs, bag_of_occ, err, s,
               tr->async_step ? chk : nullptr, !skip_maps);
  // [0] first bad slot id, [1] all-ones iff every bag holds exactly its own
  // occurrence (one feature per slot), read with dedup's one host sync --
  // or, on the sync-free step, predicted and checked on the device
  uint32_t h_errw[2] = {0xFFFFFFFFu, 0};
  // G > 1: no readback after the local dedup either -- its plan check goes to
  // a flag word that travels with the send counts in the counts allgather
  // (one readback for all three; a miss anywhere redoes the sort and the
  // counts on every rank, before anything was sent or written)
  const bool g_async = tr->world > 1 && tr->sync_free && !tr->fused_pool && dedup_async_ready(tr->dd, sv.n_occ);
  uint32_t* pflag = g_async ? tr->pflag.get<uint32_t>(1) : nullptr;
  if (g_async) {
    KP_CUDA(cudaMemsetAsync(pflag, 0, 4, s));
    dedup(sv.keys, sv.n_occ, tr->dd, s, bag_of_occ, err + 1, pflag, -1);
  }
  const bool ran_async = g_async || (tr->async_step && dedup(sv.keys, sv.n_occ, tr->dd, s, bag_of_occ, err + 1, chk,
                                                             tr->pred_ident ? 1 : 0));
  if (!ran_async) {
    KP_CUDA(cudaMemcpyAsync(h_errw, err, 8, cudaMemcpyDeviceToHost, s));
    dedup(sv.keys, sv.n_occ, tr->dd, s, bag_of_occ, err + 1);  // synchronises the stream
    if (sv.n_occ == 0) KP_CUDA(cudaStreamSynchronize(s));
    tr->pred_ident = h_errw[1] == 0xFFFFFFFFu;
  }
  // G > 1: the send counts (+ this rank's plan flag and error words) of every
  // rank in one allgather and one readback; a plan miss anywhere redoes the
  // sort with the exact plan (and the readback) and the counts on every rank
  std::vector<uint64_t> gath;
  auto gather_counts = [&](uint32_t n_bound, const uint32_t* dn) {
    const int R = tr->world;
    const size_t RS = (size_t)R + 2;
    uint32_t* perm = tr->perm.get<uint32_t>(std::max<uint32_t>(n_bound, 1));
    uint32_t* pos = tr->pos.get<uint32_t>(std::max<uint32_t>(n_bound, 1));
    uint64_t* cd = tr->counts_dev.get<uint64_t>(RS * (R + 1));
    shard(tr->dd.d_unique, n_bound, R, perm, pos, nullptr, tr->sh, s, cd, dn);
    pack_step_flags(pflag, err, cd + R, s);
    KP_NCCL(ncclAllGather(cd, cd + RS, RS, ncclUint64, tr->comm->nc, s));
    gath.assign(RS * R, 0);
    KP_CUDA(cudaMemcpyAsync(gath.data(), cd + RS, RS * R * 8, cudaMemcpyDeviceToHost, s));
    KP_CUDA(cudaStreamSynchronize(s));
  };
  if (g_async) {
    const int R = tr->world;
    gather_counts(sv.n_occ, tr->dd.d_nunique);
    bool miss = false;
    for (int p = 0; p < R; ++p) miss |= gath[(size_t)p * (R + 2) + R] != 0;
    if (miss) {  // (collective: every rank saw the same flags)
      dedup(sv.keys, sv.n_occ, tr->dd, s, bag_of_occ, err + 1);  // exact plan, readback
      pflag = nullptr;
      gather_counts(tr->dd.n_unique, nullptr);
    }
    const uint64_t ew = gath[(size_t)tr->rank * (R + 2) + R + 1];
    h_errw[0] = (uint32_t)ew;
    h_errw[1] = (uint32_t)(ew >> 32);
    tr->pred_ident = h_errw[1] == 0xFFFFFFFFu;
    uint64_t u = 0;
    for (int q = 0; q < R; ++q) u += gath[(size_t)tr->rank * (R + 2) + q];
    tr->dd.n_unique = (uint32_t)u;  // this rank's unique keys = what it sends
  }
  const uint32_t h_err = h_errw[0];
  const bool ident_word = (ran_async && !g_async) ? tr->pred_ident : h_errw[1] == 0xFFFFFFFFu;
  const bool ident_bags = ident_word && sv.n_occ == nb;
  // the identity occurrence -> bag map: the bag of sorted position p is the
  // sorted occurrence itself (dedup skipped writing the copy)
  if (ident_word && sv.n_occ > 0) tr->dd.d_sorted_mapped = const_cast<uint32_t*>(tr->dd.sorted_vals);
  // reject bad slot ids before any state (table, weights) changes (the
  // sync-free step: its state writes are guarded, the batch end raises)
  KP_CHECK(h_err == 0xFFFFFFFFu, kErrConfig,
           "slot ids must be < n_slots and non-decreasing within an instance (occurrence " +
               std::to_string(h_err) + ")");
  tr->mark(0);
  const bool u_dev = ran_async && !g_async;
  const uint32_t U = u_dev ? sv.n_occ : tr->dd.n_unique;
  PullResult pr{};
  pr.U = U;
  pr.dU = u_dev ? tr->dd.d_nunique : nullptr;
  if (tr->world == 1) {
    uint32_t* rows = tr->rows.get<uint32_t>(std::max<uint32_t>(U, 1));
    table_pull(tr->tab.t, tr->dd.d_unique, U, rows, stamp, s, pr.dU);
    pr.src = tr->tab.t->d_w;
    pr.idx = rows;
    tr->mark(1);
  } else {
    const int R = tr->world;
    // counts matrix via allgather, straight from the shard's device counts
    // (one host readback: this rank's row is its send counts)
    if (!g_async) gather_counts(U, nullptr);
    uint32_t* perm = static_cast<uint32_t*>(tr->perm.p);
    uint32_t* pos = static_cast<uint32_t*>(tr->pos.p);
    tr->mat.assign((size_t)R * R, 0);
    for (int p = 0; p < R; ++p)
      for (int q = 0; q < R; ++q) tr->mat[(size_t)p * R + q] = gath[(size_t)p * (R + 2) + q];
    const std::vector<uint64_t>& mat = tr->mat;
    tr->cnt_send.assign(mat.begin() + (size_t)tr->rank * R, mat.begin() + (size_t)(tr->rank + 1) * R);
    tr->cnt_recv.assign(R, 0);
    tr->off_send.assign(R, 0);
    tr->off_recv.assign(R, 0);
    uint64_t tot = 0;
    for (int p = 0; p < R; ++p) {
      tr->cnt_recv[p] = mat[(size_t)p * R + tr->rank];
      tr->off_recv[p] = tot;
      tot += tr->cnt_recv[p];
    }
    for (int p = 1; p < R; ++p) tr->off_send[p] = tr->off_send[p - 1] + tr->cnt_send[p - 1];
    const uint32_t Rn = (uint32_t)tot;
    // GpuPull: keys to each remote owner and its rows back (ledger.hpp)
    for (int p = 0; p < R; ++p)
      if (p != tr->rank && tr->cnt_send[p]) {
        tr->led_bytes[kLedPull] += tr->cnt_send[p] * (8 + 4ull * tr->e);
        tr->led_count[kLedPull] += 1;
      }
    const bool peer = peer_ready(tr);
    uint64_t* rk;
    if (peer) {
      // keys straight into the owners' windows over NVLink
      peer_send_keys(tr->dd.d_unique, perm, U, peer_map(tr, 0, U), s);
      peer_exchange_sync(tr, 0, true, true);
      rk = static_cast<uint64_t*>(tr->peer.keys.local);
    } else {
      uint64_t* sk = tr->send_keys.get<uint64_t>(std::max<uint32_t>(U, 1));
      if (U) k_gather_u64<<<grid1(U), 256, 0, s>>>(tr->dd.d_unique, perm, U, sk); ::kp::count_launch();
      rk = tr->recv_keys.get<uint64_t>(std::max<uint32_t>(Rn, 1));
      all_to_all(tr, sk, tr->cnt_send, tr->off_send, rk, tr->cnt_recv, tr->off_recv, 8, ncclUint64);
    }
    tr->mark(6);
    // owner side: dedup received keys (stable: source order inside a key)
    {
      // each source's keys arrive ascending: merge the R runs
      std::vector<uint64_t> run_off(R + 1, 0);
      for (int p = 0; p < R; ++p) run_off[p + 1] = run_off[p] + tr->cnt_recv[p];
      dedup_runs(rk, Rn, run_off, tr->dd_owner, s, /*readback*/ false);
    }
    tr->mark(0);
    // (the owner's U stays on the device: Rn bounds it)
    const bool uo_dev = tr->dd_owner.n_unique == kUnknownU;
    const uint32_t Uo = uo_dev ? Rn : tr->dd_owner.n_unique;
    const uint32_t* dUo = uo_dev ? tr->dd_owner.d_nunique : nullptr;
    uint32_t* orows = tr->owner_rows.get<uint32_t>(std::max<uint32_t>(Uo, 1));
    table_pull(tr->tab.t, tr->dd_owner.d_unique, Uo, orows, stamp, s, dUo);
    uint32_t* oidx = tr->owner_idx.get<uint32_t>(std::max<uint32_t>(Rn, 1));
    if (Rn) k_compose<<<grid1(Rn), 256, 0, s>>>(orows, tr->dd_owner.d_inverse, Rn, oidx); ::kp::count_launch();
    float* rrows;
    if (peer) {
      // rows straight back into the requesters' windows
      peer_send_rows(tr->tab.t->d_w, oidx, Rn, tr->e, peer_map(tr, 1, Rn), s);
      tr->mark(1);
      peer_exchange_sync(tr, 1, true, true);
      rrows = static_cast<float*>(tr->peer.rows.local);
    } else {
      float* srows = tr->send_rows.get<float>((size_t)std::max<uint32_t>(Rn, 1) * tr->e);
      gather_rows(tr->tab.t->d_w, oidx, Rn, tr->e, srows, s);
      tr->mark(1);
      rrows = tr->recv_rows.get<float>((size_t)std::max<uint32_t>(U, 1) * tr->e);
      all_to_all(tr, srows, tr->cnt_recv, tr->off_recv, rrows, tr->cnt_send, tr->off_send,
                 4 * (size_t)tr->e, ncclFloat32);
    }
    tr->mark(6);
    pr.src = rrows;
    pr.idx = pos;
  }
  // pooling over the composed per-occurrence source rows (the one-feature
  // planes kernel composes on the fly: its index prefetch reads inverse, then
  // the unique's row)
  tr->ga_on = tr->fused_pool && tr->planes && ident_bags && tr->e % 32 == 0 && sv.n_occ > 0 && !pr.dU;
  // (measured: pool 0.52 vs 0.48 ms against compose's 0.02 -- off; KP_POOL_COMPOSE=1)
  static const bool pool_compose = [] {
    const char* e = getenv("KP_POOL_COMPOSE");
    return e && e[0] == '1';
  }();
  const bool compose_in_pool =
      pool_compose && tr->planes && ident_bags && !tr->ga_on && planes_ident_kernel(tr->S, tr->e);
  uint32_t* rowocc = tr->rowocc.get<uint32_t>(std::max<uint32_t>(sv.n_occ, 1));
  if (!compose_in_pool) compose(pr.idx, tr->dd.d_inverse, sv.n_occ, rowocc, s);
  float* pooled = tr->pooled.get<float>((size_t)std::max<uint32_t>(nb, 1) * tr->e);
  float* invc = tr->inv_count.get<float>(std::max<uint32_t>(nb, 1));
  // one feature per slot, KP_FUSED_POOL=1: the first layer's forward gathers
  // the rows itself (kp_gemm_h3.cu, TMA gather4) and writes the planes; only
  // the instance exponents here
  if (tr->ga_on) {
    int* iexp = tr->inst_exp.get<int>(std::max<uint32_t>(sv.n_inst, 1));
    float* umax = tr->umax.get<float>(std::max<uint32_t>(U, 1));
    inst_exps_ident(pr.src, pr.idx, U, tr->e, tr->dd.d_inverse, sv.n_inst, tr->S, umax, iexp, invc,
                    tr->cfg.pooling == 1, s);
    tr->ga_src = pr.src;
    tr->ga_nrows = tr->world == 1 ? tr->tab.t->capacity : std::max<uint32_t>(U, 1);
    tr->ga_rowocc = rowocc;
  } else if (tr->planes) {
    // the first layer's input as fp16 planes (hi at pooled, lo behind it)
    __half* hi = reinterpret_cast<__half*>(pooled);
    int* iexp = tr->inst_exp.get<int>(std::max<uint32_t>(sv.n_inst, 1));
    pool_planes(bag_offs, sv.n_inst, tr->S, compose_in_pool ? pr.idx : rowocc, pr.src, tr->e,
                tr->cfg.pooling == 1, hi, hi + (size_t)nb * tr->e, iexp, invc, s, ident_bags,
                compose_in_pool ? tr->dd.d_inverse : nullptr);
  } else {
    // max |row| of the MLP input per instance (fp16-operand first layer)
    float* imax = tr->inst_max.get<float>(std::max<uint32_t>(sv.n_inst, 1));
    pool(bag_offs, nb, rowocc, pr.src, tr->e, tr->cfg.pooling == 1, pooled, invc, s, imax, tr->S);
  }
  tr->mark(2);
  issue_staged(tr, -1);  // this step's host readbacks are done
  return pr;
}

// Bytes this rank sends over the fabric for one merge (two rounds, v then
// the term), per path: peer (owner reads every rank's W chunk slices and
// stores its result into every other rank), NCCL chunked (send W slices of
// each peer's chunk + ring allgather), NCCL allgather of every worker vector.
uint64_t merge_bytes_sent(const kp_trainer* tr) {
  const uint64_t R = tr->world, W = tr->W, D = tr->D, me = tr->rank;
  const uint64_t C = (D + R - 1) / R;
  const uint64_t my_len = std::min<uint64_t>(C, D > me * C ? D - me * C : 0);
  uint64_t per_round;
  if (tr->peer.mode == 1) {
    // one round (k_merge_peer): every other owner reads its chunk of my W
    // workers' v, x and m; I store my merged chunk's v_bar and x into every
    // other rank
    return 3 * (D - my_len) * W * 4 + 2 * (R - 1) * my_len * 4;
  } else if ((R - 1) * W * D * 4 <= (24ull << 20)) {
    per_round = (R - 1) * W * D * 4;  // ring allgather of W*D per rank
  } else {
    per_round = (D - my_len) * W * 4 + (R - 1) * C * 4;
  }
  return 2 * per_round;
}

// StepRecord (optimizer.hpp:55-63) for the step just taken: x_bar (a
// collective when G > 1 and the replicas differ), the frozen v_bar of worker
// 0, merged, a3 = sum_j |1/sqrt(v_bar_before) - 1/sqrt(v_bar_after)| at
// merges (optimizer.cpp:126-131). The loss is filled in at batch end.
void record_trajectory(kp_trainer* tr, uint64_t t, bool merged) {
  const uint64_t D = tr->D;
  kp_trainer::TrajStep r;
  r.step = t;
  r.merged = merged ? 1 : 0;
  r.x_bar.resize(D);
  r.v_bar.resize(D);
  float* xb = tr->xbar.get<float>(D);
  compute_xbar(tr, xb);
  KP_CUDA(cudaMemcpyAsync(r.x_bar.data(), xb, D * 4, cudaMemcpyDeviceToHost, tr->s));
  KP_CUDA(cudaMemcpyAsync(r.v_bar.data(), tr->vbar, D * 4, cudaMemcpyDeviceToHost, tr->s));
  KP_CUDA(cudaStreamSynchronize(tr->s));
  if (merged) {
    double a3 = 0.0;
    for (uint64_t j = 0; j < D; ++j)
      a3 += std::abs(1.0 / std::sqrt((double)tr->traj_prev_vbar[j]) - 1.0 / std::sqrt((double)r.v_bar[j]));
    r.a3 = a3;
  }
  tr->traj_prev_vbar = r.v_bar;
  tr->traj.push_back(std::move(r));
}

void run_step(kp_trainer* tr, const StepView& sv, double* d_loss_slot, float* fused_preds) {
  cudaStream_t s = tr->s;
  const uint64_t D = tr->D;
  const uint32_t in_w = tr->S * tr->e;
  tr->mark(-1);
  PullResult pr = pull_and_pool(tr, sv, false);
  if (tr->prof) {
    if (!pr.dU) tr->prof_unique += pr.U;  // (sync-free step: added at the batch-end readback)
    tr->prof_occ += sv.n_occ;
    if (tr->world > 1) {
      if (tr->dd_owner.n_unique != kUnknownU) tr->prof_owner_unique += tr->dd_owner.n_unique;
      for (auto c : tr->cnt_recv) tr->prof_recv += c;
    }
  }
  const float* pooled = static_cast<const float*>(tr->pooled.p);
  const float* invc = static_cast<const float*>(tr->inv_count.p);
  float* dpooled = tr->dpooled.get<float>((size_t)std::max<uint32_t>(sv.n_inst, 1) * in_w);
  float* preds = tr->preds.get<float>(std::max<uint32_t>(sv.n_inst, 1));
  SparseRule rule{tr->cfg.sparse_rule, (float)tr->cfg.sparse_lr, (float)tr->cfg.sparse_beta1,
                  (float)tr->cfg.sparse_beta2};
  const float inv_n = (float)(1.0 / (double)tr->N);
  // G > 1: per-unique gradients for the owners, then the all-to-all. With
  // overlap (default), both are issued right after the first layer's input
  // gradient: the reduction on the compute stream, the all-to-all on the
  // exchange stream (own NCCL channel) while the weight-gradient GEMM runs on
  // all but kXReserve SMs.
  float* sgr = nullptr;
  float* rgr = nullptr;
  uint64_t Rn = 0;
  const bool peer = tr->world > 1 && tr->peer.mode == 1;
  PeerMap pmg{};
  if (tr->world > 1) {
    for (auto c : tr->cnt_recv) Rn += c;
    if (peer) {
      // reduced gradients go straight into the owners' windows (NVLink)
      pmg = peer_map(tr, 2, pr.U);
      rgr = static_cast<float*>(tr->peer.grads.local);
    } else {
      sgr = tr->send_grads.get<float>((size_t)std::max<uint32_t>(pr.U, 1) * tr->e);
      rgr = tr->recv_grads.get<float>((size_t)std::max<uint64_t>(Rn, 1) * tr->e);
    }
  }
  // Gradients: reduce into a local buffer, then the copy engines move each
  // owner's segment into its peer window on the exchange stream (no SMs,
  // overlaps the weight-gradient GEMM; measured +1.5% at G=4 over remote
  // stores from the reduction itself, which KP_PEER_CE=0 selects)
  static const bool peer_ce = [] {
    const char* e = getenv("KP_PEER_CE");
    return !(e && e[0] == '0');
  }();
  auto send_grads = [&] {
    if (peer && peer_ce) {
      float* loc = tr->send_grads.get<float>((size_t)std::max<uint32_t>(pr.U, 1) * tr->e);
      seg_reduce_apply(tr->dd.d_seg, pr.U, tr->dd.d_sorted_mapped, nullptr, sv.n_occ, dpooled, tr->e,
                       1.0f, nullptr, nullptr, rule, loc, static_cast<const uint32_t*>(tr->pos.p),
                       tr->sg, s, nullptr);
      if (!tr->xs) {
        KP_CUDA(cudaStreamCreateWithFlags(&tr->xs, cudaStreamNonBlocking));
        KP_CUDA(cudaEventCreateWithFlags(&tr->ev_dinput, cudaEventDisableTiming));
        KP_CUDA(cudaEventCreateWithFlags(&tr->ev_xdone, cudaEventDisableTiming));
      }
      KP_CUDA(cudaEventRecord(tr->ev_dinput, s));
      KP_CUDA(cudaStreamWaitEvent(tr->xs, tr->ev_dinput, 0));
      const size_t row = (size_t)tr->e * 4;
      for (int p = 0; p < tr->world; ++p) {
        if (!tr->cnt_send[p]) continue;
        KP_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(pmg.base[p]),
                                reinterpret_cast<const char*>(loc) + tr->off_send[p] * row,
                                tr->cnt_send[p] * row, cudaMemcpyDeviceToDevice, tr->xs));
      }
      peer_exchange_sync(tr, 2, true, false, tr->xs);
      KP_CUDA(cudaEventRecord(tr->ev_xdone, tr->xs));
      return;
    }
    seg_reduce_apply(tr->dd.d_seg, pr.U, tr->dd.d_sorted_mapped, nullptr, sv.n_occ, dpooled, tr->e,
                     1.0f, nullptr, nullptr, rule, sgr, static_cast<const uint32_t*>(tr->pos.p),
                     tr->sg, s, peer ? &pmg : nullptr);
    if (peer) peer_exchange_sync(tr, 2, true, false);
  };
  static const int reserve = [] {
    const char* e = getenv("KP_XRESERVE");
    return e ? atoi(e) : 16;
  }();
  const bool overlap = tr->world > 1 && (reserve > 0 || peer);
  bool exchanged = false;
  std::function<void()> hook = [&] {
    tr->mark(3);  // the backward so far is MLP time; the reduction is push time
    send_grads();
    tr->mark(4);
    exchanged = true;
    if (peer) return;  // the reduction itself moved the data; no SMs to reserve
    if (!tr->xs) {
      KP_CUDA(cudaStreamCreateWithFlags(&tr->xs, cudaStreamNonBlocking));
      KP_CUDA(cudaEventCreateWithFlags(&tr->ev_dinput, cudaEventDisableTiming));
      KP_CUDA(cudaEventCreateWithFlags(&tr->ev_xdone, cudaEventDisableTiming));
    }
    KP_CUDA(cudaEventRecord(tr->ev_dinput, s));
    KP_CUDA(cudaStreamWaitEvent(tr->xs, tr->ev_dinput, 0));
    all_to_all(tr, sgr, tr->cnt_send, tr->off_send, rgr, tr->cnt_recv, tr->off_recv,
               4 * (size_t)tr->e, ncclFloat32, tr->xs, tr->comm->nc2);
    KP_CUDA(cudaEventRecord(tr->ev_xdone, tr->xs));
    tc_reserve_sms(reserve);
    exchanged = true;
  };
  for (uint32_t l = 0; l < tr->W; ++l) {
    const uint32_t lo = sv.wlo[l], hi = sv.whi[l], Bw = hi - lo;
    if (Bw == 0) {
      KP_CUDA(cudaMemsetAsync(tr->g + l * D, 0, D * 4, s));
      continue;
    }
    tr->mlp.in_rowmax = static_cast<const float*>(tr->inst_max.p) + lo;
    if (tr->planes) {
      const size_t nbags = (size_t)sv.n_inst * tr->S;
      tr->mlp.in_hi = tr->plane_hi(nbags) + (size_t)lo * in_w;
      tr->mlp.in_lo = tr->plane_lo(nbags) + (size_t)lo * in_w;
      tr->mlp.in_exp = static_cast<const int*>(tr->inst_exp.p) + lo;
      if (tr->ga_on) {
        tr->mlp.ga_src = tr->ga_src;
        tr->mlp.ga_nrows = tr->ga_nrows;
        tr->mlp.ga_rowocc = tr->ga_rowocc + (size_t)lo * tr->S;
        tr->mlp.ga_S = tr->S;
        tr->mlp.ga_e = tr->e;
      }
    }
    mlp_forward(tr->shape, tr->x + l * D, pooled + (size_t)lo * in_w, Bw, preds + lo, tr->mlp, s);
    tr->mlp.in_rowmax = nullptr;
    mlp_backward(tr->shape, tr->x + l * D, pooled + (size_t)lo * in_w, Bw, preds + lo,
                 sv.labels + lo, tr->g + l * D, dpooled + (size_t)lo * in_w,
                 tr->cfg.pooling == 1 ? invc + (size_t)lo * tr->S : nullptr, tr->S, tr->e,
                 d_loss_slot, tr->mlp, s, (overlap && l + 1 == tr->W) ? &hook : nullptr);
    tr->mlp.in_hi = tr->mlp.in_lo = nullptr;
    tr->mlp.in_exp = nullptr;
    tr->mlp.ga_src = nullptr;
    tr->mlp.ga_rowocc = nullptr;
  }
  tc_reserve_sms(0);
  if (fused_preds)
    KP_CUDA(cudaMemcpyAsync(fused_preds, preds, (size_t)sv.n_inst * 4, cudaMemcpyDeviceToDevice, s));
  tr->mark(3);
  // sparse push (x 1/N, trainer.cpp:202-207)
  if (tr->world == 1) {
    seg_reduce_apply(tr->dd.d_seg, pr.U, tr->dd.d_sorted_mapped, nullptr, sv.n_occ, dpooled, tr->e,
                     inv_n, tr->tab.t, pr.idx, rule, nullptr, nullptr, tr->sg, s, nullptr, pr.dU);
    tr->mark(4);
  } else {
    if (!exchanged) {
      send_grads();
      tr->mark(4);
      if (!peer)
        all_to_all(tr, sgr, tr->cnt_send, tr->off_send, rgr, tr->cnt_recv, tr->off_recv,
                   4 * (size_t)tr->e, ncclFloat32);
    } else if (!peer) {
      KP_CUDA(cudaStreamWaitEvent(s, tr->ev_xdone, 0));
    }
    if (peer && peer_ce) KP_CUDA(cudaStreamWaitEvent(s, tr->ev_xdone, 0));
    if (peer) peer_exchange_sync(tr, 2, false, true);
    tr->mark(6);
    const bool uo_dev = tr->dd_owner.n_unique == kUnknownU;  // (U on the device: Rn bounds it)
    seg_reduce_apply(tr->dd_owner.d_seg, uo_dev ? (uint32_t)Rn : tr->dd_owner.n_unique, tr->dd_owner.sorted_vals,
                     nullptr, (uint32_t)Rn, rgr, tr->e, inv_n, tr->tab.t,
                     static_cast<const uint32_t*>(tr->owner_rows.p), rule, nullptr, nullptr,
                     tr->sg_owner, s, nullptr, uo_dev ? tr->dd_owner.d_nunique : nullptr);
    tr->mark(4);
  }
  if (tr->world > 1)  // GpuPush: per-key gradients to each remote owner
    for (int p = 0; p < tr->world; ++p)
      if (p != tr->rank && tr->cnt_send[p]) {
        tr->led_bytes[kLedPush] += tr->cnt_send[p] * 4ull * tr->e;
        tr->led_count[kLedPush] += 1;
      }
  // dense k-step Adam (KStepEngine::step, optimizer.cpp:113-144)
  const uint64_t t = tr->t_global + 1;
  const bool merged = (t % tr->cfg.k) == 0;
  AdamParams h{(float)tr->cfg.alpha, (float)tr->cfg.beta1, (float)tr->cfg.beta2};
  uint32_t* chk = static_cast<uint32_t*>(tr->check.p);
  if (tr->W == 1 && tr->world == 1) {
    // one pass: moments, the local step or the single-worker merge, checks
    dense_step_single(tr->x, tr->m, tr->v, tr->vbar, tr->g, D, h, merged, tr->cfg.reset_local_v != 0, chk,
                      chk + 1, s);
    if (merged) {
      tr->merges++;
      tr->x_uniform = true;
    } else {
      tr->x_uniform = false;
    }
    tr->t_global = t;
    tr->mark(5);
    if (tr->traj_on) record_trajectory(tr, t, merged);
    return;
  }
  if (!merged) {
    for (uint32_t l = 0; l < tr->W; ++l)
      dense_local_step(tr->x + l * D, tr->m + l * D, tr->v + l * D, tr->vbar + l * D, tr->g + l * D,
                       D, h, s);
    tr->x_uniform = false;
  } else {
    for (uint32_t l = 0; l < tr->W; ++l) dense_moments(tr->m + l * D, tr->v + l * D, tr->g + l * D, D, h, s);
    if (tr->world > 1 && tr->peer.mode == 1)
      merge_states_peer(tr, h.alpha, tr->cfg.reset_local_v != 0);
    else
      merge_states(tr->comm, s, tr->W, D, tr->x, tr->m, tr->v, tr->vbar, h.alpha,
                   tr->cfg.reset_local_v != 0, tr->mws);
    tr->merges++;
    tr->x_uniform = true;
    if (tr->world > 1) {  // DenseMerge: one model transmission per worker (trainer.cpp:99-107)
      tr->led_bytes[kLedDense] += merge_bytes_sent(tr);
      tr->led_count[kLedDense] += tr->W;
    }
  }
  tr->t_global = t;
  for (uint32_t l = 0; l < tr->W; ++l)
    dense_check(tr->v + l * D, tr->vbar + l * D, tr->x + l * D, D, chk, s, l == 0 ? chk + 1 : nullptr);
  tr->mark(5);
  if (tr->traj_on) record_trajectory(tr, t, merged);
}

void predict_pass(kp_trainer* tr, const StepView& sv, float* d_preds_out) {
  float* xb = tr->xbar.get<float>(tr->D);
  compute_xbar(tr, xb);
  pull_and_pool(tr, sv, false);
  tr->mlp.in_rowmax = static_cast<const float*>(tr->inst_max.p);
  if (tr->planes) {
    const size_t nbags = (size_t)sv.n_inst * tr->S;
    tr->mlp.in_hi = tr->plane_hi(nbags);
    tr->mlp.in_lo = tr->plane_lo(nbags);
    tr->mlp.in_exp = static_cast<const int*>(tr->inst_exp.p);
    if (tr->ga_on) {
      tr->mlp.ga_src = tr->ga_src;
      tr->mlp.ga_nrows = tr->ga_nrows;
      tr->mlp.ga_rowocc = tr->ga_rowocc;
      tr->mlp.ga_S = tr->S;
      tr->mlp.ga_e = tr->e;
    }
  }
  mlp_forward(tr->shape, xb, static_cast<const float*>(tr->pooled.p), sv.n_inst, d_preds_out,
              tr->mlp, tr->s);
  tr->mlp.in_rowmax = nullptr;
  tr->mlp.in_hi = tr->mlp.in_lo = nullptr;
  tr->mlp.in_exp = nullptr;
  tr->mlp.ga_src = nullptr;
  tr->mlp.ga_rowocc = nullptr;
  tr->mark(3);
}

void train_batch_impl(kp_trainer* tr, const uint32_t* h_offs, const uint32_t* d_offs,
                      const uint64_t* d_keys, const uint16_t* d_slots, const int32_t* d_labels,
                      uint32_t n, uint64_t global_n, uint64_t global_first, bool predict_first,
                      float* h_preds, kp_batch_result* out) {
  KP_CHECK(n >= 1 || tr->world > 1, kErrGeneric, "train_batch: empty batch");
  KP_CHECK(global_n >= 1, kErrGeneric, "train_batch: empty batch");
  KP_CHECK(tr->S == 1 || d_slots != nullptr, kErrConfig, "slots must be given when n_slots > 1");
  cudaStream_t s = tr->s;
  const uint64_t N = tr->N, W = tr->W, r = tr->rank;
  const uint64_t mb = tr->cfg.minibatch_size;
  const uint64_t n_mb = std::max<uint64_t>(1, (global_n + N * mb - 1) / (N * mb));
  const uint64_t cells = N * n_mb, base = global_n / cells, extra = global_n % cells;
  auto cstart = [&](uint64_t c) { return c * base + std::min(c, extra); };
  const uint64_t my_lo = cstart(r * W * n_mb), my_hi = cstart((r + 1) * W * n_mb);
  KP_CHECK(global_first == my_lo && global_first + n == my_hi, kErrConfig,
           "train_batch: slice [" + std::to_string(global_first) + ", " +
               std::to_string(global_first + n) + ") is not this rank's shard_batch range [" +
               std::to_string(my_lo) + ", " + std::to_string(my_hi) + ")");
  KP_CHECK(h_offs[0] == 0, kErrGeneric, "offs[0] must be 0");
  uint32_t* err = tr->err.get<uint32_t>(4);
  uint32_t* chk_w = tr->check.get<uint32_t>(2);  // [0] flags [1] steps applied
  // the sync-free single-GPU step: one minibatch step per batch, no
  // per-step host work that needs U (trajectory, gathered-A forward)
  struct AsyncReset {
    kp_trainer* t;
    ~AsyncReset() { t->async_step = false; }
  } async_reset{tr};
  tr->async_step = tr->sync_free && !tr->force_sync && tr->world == 1 && n_mb == 1 && !tr->traj_on && !tr->fused_pool;
  // G > 1 (and the sync-free step): every state-writing kernel of this batch
  // (predict pass included) checks the abort bits of the check word first
  AbortScope abort_guard(tr->world > 1 || tr->async_step ? static_cast<const uint32_t*>(tr->check.p) : nullptr);
  double* d_loss = tr->loss.get<double>(n_mb);
  // predictions use x_bar (trainer.cpp:141-151); when every replica holds
  // the same x (initial state, right after a merge, no set_worker_state
  // since) x_bar IS each worker's x, and the training forward doubles as the
  // prediction
  const bool fused = predict_first && n_mb == 1 && tr->x_uniform;
  float* d_pred_keep = predict_first ? tr->pred_keep.get<float>(std::max<uint32_t>(n, 1)) : nullptr;
  const uint64_t steps_before = tr->t_global, merges_before = tr->merges;
  const bool uniform_before = tr->x_uniform;
  // pinned readback block (see kp_trainer::rb)
  uint32_t* rb = static_cast<uint32_t*>(tr->rb_ensure(64 + n_mb * 8 + (size_t)(predict_first ? n : 0) * 4));
  double* rb_loss = reinterpret_cast<double*>(reinterpret_cast<char*>(rb) + 64);
  float* rb_preds = reinterpret_cast<float*>(reinterpret_cast<char*>(rb) + 64 + n_mb * 8);
  // CUDA graph of the whole sync-free batch: replayed when this exact batch
  // shape (inputs, sizes, step-dependent choices) was captured before
  const bool merged_next = ((tr->t_global + 1) % tr->cfg.k) == 0;
  static const bool sync_debug = getenv("KP_SYNC_DEBUG") != nullptr;
  const bool gmode = tr->graphs && tr->async_step && W == 1 && !tr->prof && n_mb == 1 && !sync_debug &&
                     dedup_async_ready(tr->dd, h_offs[n]);
  kp_trainer::GraphKey gk{};
  if (gmode) {
    const uint64_t gen = devbuf_generation().load();
    if (gen != tr->ggen) {
      tr->graphs_clear();
      tr->ggen = gen;
    }
    gk.p[0] = d_offs;
    gk.p[1] = d_keys;
    gk.p[2] = d_slots;
    gk.p[3] = d_labels;
    gk.n = n;
    gk.n_occ = h_offs[n];
    gk.gn = global_n;
    gk.gfirst = global_first;
    gk.flags = (predict_first ? 1 : 0) | (fused ? 4 : 0) | (merged_next ? 8 : 0) | (tr->pred_ident ? 16 : 0);
    gk.spec = tr->dd.spec_bits;
  }
  auto it = gmode ? tr->gcache.find(gk) : tr->gcache.end();
  const bool replay = gmode && it != tr->gcache.end();
  const bool capture = gmode && !replay;
  auto body = [&]() {
  KP_CUDA(cudaMemsetAsync(err, 0xFF, 4, s));
  KP_CUDA(cudaMemsetAsync(chk_w, 0, 8, s));
  KP_CUDA(cudaMemsetAsync(d_loss, 0, n_mb * 8, s));
  if (predict_first) {
    if (!fused) {
      StepView pv;
      pv.offs = d_offs;
      pv.occ_base = 0;
      pv.keys = d_keys;
      pv.slots = d_slots;
      pv.labels = d_labels;
      pv.n_inst = n;
      pv.n_occ = h_offs[n];
      tr->mark(-1);
      predict_pass(tr, pv, d_pred_keep);
    }
  }
  for (uint64_t j = 0; j < n_mb; ++j) {
    StepView sv;
    sv.wlo.resize(W);
    sv.whi.resize(W);
    std::vector<uint64_t> lo(W), hi(W);
    for (uint64_t l = 0; l < W; ++l) {
      const uint64_t c = (r * W + l) * n_mb + j;
      lo[l] = cstart(c) - global_first;
      hi[l] = cstart(c + 1) - global_first;
    }
    const bool contiguous = W == 1 || n_mb == 1;
    if (contiguous) {
      const uint64_t a = lo[0], b = hi[W - 1];
      sv.offs = d_offs + a;
      sv.occ_base = h_offs[a];
      sv.keys = d_keys + h_offs[a];
      sv.slots = d_slots ? d_slots + h_offs[a] : nullptr;
      sv.labels = d_labels + a;
      sv.n_inst = (uint32_t)(b - a);
      sv.n_occ = h_offs[b] - h_offs[a];
      for (uint64_t l = 0; l < W; ++l) {
        sv.wlo[l] = (uint32_t)(lo[l] - a);
        sv.whi[l] = (uint32_t)(hi[l] - a);
      }
    } else {
      // gather the local workers' cells for minibatch j into step buffers
      uint32_t ninst = 0, nocc = 0;
      for (uint64_t l = 0; l < W; ++l) {
        ninst += (uint32_t)(hi[l] - lo[l]);
        nocc += h_offs[hi[l]] - h_offs[lo[l]];
      }
      std::vector<uint32_t> so(ninst + 1);
      uint64_t* sk = tr->st_keys.get<uint64_t>(std::max<uint32_t>(nocc, 1));
      uint16_t* ss = d_slots ? tr->st_slots.get<uint16_t>(std::max<uint32_t>(nocc, 1)) : nullptr;
      int32_t* sl = tr->st_labels.get<int32_t>(std::max<uint32_t>(ninst, 1));
      uint32_t* sof = tr->st_offs.get<uint32_t>(ninst + 1);
      uint32_t ci = 0, co = 0;
      so[0] = 0;
      for (uint64_t l = 0; l < W; ++l) {
        sv.wlo[l] = ci;
        const uint32_t o0 = h_offs[lo[l]], o1 = h_offs[hi[l]];
        for (uint64_t i = lo[l]; i < hi[l]; ++i) so[++ci] = co + (h_offs[i + 1] - o0);
        if (o1 > o0) {
          KP_CUDA(cudaMemcpyAsync(sk + co, d_keys + o0, (size_t)(o1 - o0) * 8, cudaMemcpyDeviceToDevice, s));
          if (ss) KP_CUDA(cudaMemcpyAsync(ss + co, d_slots + o0, (size_t)(o1 - o0) * 2, cudaMemcpyDeviceToDevice, s));
        }
        if (hi[l] > lo[l])
          KP_CUDA(cudaMemcpyAsync(sl + sv.wlo[l], d_labels + lo[l], (hi[l] - lo[l]) * 4, cudaMemcpyDeviceToDevice, s));
        co += o1 - o0;
        sv.whi[l] = ci;
      }
      KP_CUDA(cudaMemcpyAsync(sof, so.data(), (ninst + 1) * 4, cudaMemcpyHostToDevice, s));
      KP_CUDA(cudaStreamSynchronize(s));  // `so` is a host temporary
      sv.offs = sof;
      sv.occ_base = 0;
      sv.keys = sk;
      sv.slots = ss;
      sv.labels = sl;
      sv.n_inst = ninst;
      sv.n_occ = nocc;
    }
    run_step(tr, sv, d_loss + j, fused && j == 0 ? d_pred_keep : nullptr);
  }
  // error flags, loss, predictions -> the pinned readback block
  KP_CUDA(cudaMemcpyAsync(rb, err, 8, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaMemcpyAsync(rb + 2, tr->check.p, 8, cudaMemcpyDeviceToHost, s));
  if (tr->async_step && tr->dd.d_nunique)
    KP_CUDA(cudaMemcpyAsync(rb + 4, tr->dd.d_nunique, 4, cudaMemcpyDeviceToHost, s));
  KP_CUDA(cudaMemcpyAsync(rb_loss, d_loss, n_mb * 8, cudaMemcpyDeviceToHost, s));
  if (predict_first)
    KP_CUDA(cudaMemcpyAsync(rb_preds, d_pred_keep, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
  // table scalars ([2] = full flag), same readback
  KP_CUDA(cudaMemcpyAsync(rb + 5, tr->tab.t->d_scalars, 16, cudaMemcpyDeviceToHost, s));
  };  // body
  if (replay) {
    KP_CUDA(cudaGraphLaunch(it->second.exec, s));
    issue_staged(tr, -1);  // a pending next-batch copy: outside the graph, after its launch
    g_launches.fetch_add(it->second.launches, std::memory_order_relaxed);
    // the host-side effects of the captured step (run_step, W = 1, one GPU)
    tr->t_global += 1;
    if (merged_next) tr->merges++;
    tr->x_uniform = merged_next;
  } else if (capture) {
    issue_staged(tr, -1);
    const uint64_t l0 = g_launches.load(), gen0 = devbuf_generation().load();
    KP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    bool ok = true;
    try {
      body();
    } catch (...) {
      ok = false;
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ex = nullptr;
    ok = ok && ec == cudaSuccess && g && devbuf_generation().load() == gen0 &&
         cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      // undo the capture pass's host effects and run the batch directly; the
      // first failure for a shape (a buffer that had to grow: allocations are
      // refused inside a capture) defers the capture to the next batch of the
      // shape, a second one turns graphs off for this trainer
      cudaGetLastError();
      if (ex) cudaGraphExecDestroy(ex);
      const bool again = tr->gseen.count(gk) > 0;
      tr->graphs_clear();
      if (again) tr->graphs = false;
      else tr->gseen.insert(gk);
      tr->t_global = steps_before;
      tr->merges = merges_before;
      tr->x_uniform = uniform_before;
      tr->marks.clear();
      tr->ev_used = 0;
      train_batch_impl(tr, h_offs, d_offs, d_keys, d_slots, d_labels, n, global_n, global_first, predict_first,
                       h_preds, out);
      return;
    }
    if (tr->gcache.size() >= 16) tr->graphs_clear();  // (bounded: many shapes -> recapture)
    tr->gcache[gk] = kp_trainer::GraphEnt{ex, g_launches.load() - l0};
    g_launches.store(l0);  // counted when it runs, below
    KP_CUDA(cudaGraphLaunch(ex, s));
    g_launches.fetch_add(tr->gcache[gk].launches, std::memory_order_relaxed);
  } else {
    body();
  }
  KP_CUDA(cudaStreamSynchronize(s));
  uint32_t h_errw2[2] = {rb[0], rb[1]}, h_chkw[2] = {rb[2], rb[3]};
  const uint32_t h_nu = rb[4];
  uint32_t h_sc[4] = {rb[5], rb[6], rb[7], rb[8]};
  const uint32_t& h_err = h_errw2[0];
  const uint32_t h_chk = h_chkw[0];
  std::vector<double> lsum(rb_loss, rb_loss + n_mb);
  if (predict_first && h_preds) std::memcpy(h_preds, rb_preds, (size_t)n * 4);
  if (tr->async_step) {
    if (h_chkw[0] & kAbortPlan) {
      // the device found the pass plan or the predicted layout wrong (or a
      // bad slot id): nothing was written -- roll the host counters back and
      // rerun the batch with the readbacks (or raise the slot error)
      tr->marks.clear();
      tr->ev_used = 0;
      tr->t_global = steps_before;
      tr->merges = merges_before;
      tr->x_uniform = uniform_before;
      tr->pred_ident = h_errw2[1] == 0xFFFFFFFFu;
      KP_CHECK(h_err == 0xFFFFFFFFu, kErrConfig,
               "slot ids must be < n_slots and non-decreasing within an instance (occurrence " +
                   std::to_string(h_err) + ")");
      tr->force_sync = true;
      struct Unforce {
        kp_trainer* t;
        ~Unforce() { t->force_sync = false; }
      } unforce{tr};
      train_batch_impl(tr, h_offs, d_offs, d_keys, d_slots, d_labels, n, global_n, global_first, predict_first,
                       h_preds, out);
      return;
    }
    tr->pred_ident = h_errw2[1] == 0xFFFFFFFFu;
    if (tr->prof) tr->prof_unique += h_nu;
  }
  tr->harvest();
  if (tr->prof) tr->prof_steps += n_mb;
  KP_CHECK(h_err == 0xFFFFFFFFu, kErrConfig,
           "slot ids must be < n_slots and non-decreasing within an instance (occurrence " +
               std::to_string(h_err) + ")");
  KP_CHECK(h_sc[2] == 0, kErrTableFull,
           "embedding table full: capacity " + std::to_string(tr->tab.t->capacity) + " rows");
  if (h_chk & kAbortTimeout) {
    // the steps before the timed-out one applied their updates, the rest
    // wrote nothing: roll the host counters back to the applied count
    const uint64_t applied = h_chkw[1];
    if (applied < tr->t_global - steps_before) {
      uint64_t merges = merges_before;
      for (uint64_t t = steps_before + 1; t <= steps_before + applied; ++t)
        if (t % tr->cfg.k == 0) ++merges;
      tr->t_global = steps_before + applied;
      tr->merges = merges;
      tr->x_uniform = applied ? (tr->t_global % tr->cfg.k == 0) : uniform_before;
    }
  }
  KP_CHECK(!(h_chk & kAbortTimeout), kErrCuda,
           "peer exchange timed out waiting for another rank (NVLink window flags, "
           "KP_PEER_TIMEOUT_S): the timed-out minibatch step and the rest of the batch "
           "wrote no table or dense state");
  KP_CHECK(!(h_chk & 1), kErrGeneric, "non-finite worker state after step " + std::to_string(tr->t_global));
  KP_CHECK(!(h_chk & 2), kErrGeneric, "second moment lost positivity at step " + std::to_string(tr->t_global));
  // per-step loss = sum_workers loss_i*|mb_i| / sum |mb_i|  (trainer.cpp:177-178,221-223)
  if (tr->world > 1) {
    double* dl = tr->lossg.get<double>((size_t)n_mb * tr->world);
    KP_CUDA(cudaMemcpyAsync(d_loss, lsum.data(), n_mb * 8, cudaMemcpyHostToDevice, s));
    KP_NCCL(ncclAllGather(d_loss, dl, n_mb, ncclFloat64, tr->comm->nc, s));
    std::vector<double> all((size_t)n_mb * tr->world);
    KP_CUDA(cudaMemcpyAsync(all.data(), dl, all.size() * 8, cudaMemcpyDeviceToHost, s));
    KP_CUDA(cudaStreamSynchronize(s));
    for (uint64_t j = 0; j < n_mb; ++j) {
      double t = 0;
      for (int p = 0; p < tr->world; ++p) t += all[(size_t)p * n_mb + j];
      lsum[j] = t;
    }
  }
  double total = 0;
  uint64_t cnt = 0;
  for (uint64_t j = 0; j < n_mb; ++j) {
    uint64_t count = 0;
    for (uint64_t w = 0; w < N; ++w) count += cstart(w * n_mb + j + 1) - cstart(w * n_mb + j);
    if (count > 0) {
      total += lsum[j] / (double)count;
      ++cnt;
    }
  }
  out->loss = cnt ? total / (double)cnt : std::nan("");
  if (tr->traj_on && tr->traj.size() >= n_mb) {  // per-step losses (trainer.cpp:217-223)
    const size_t first = tr->traj.size() - n_mb;
    for (uint64_t j = 0; j < n_mb; ++j) {
      uint64_t count = 0;
      for (uint64_t w = 0; w < N; ++w) count += cstart(w * n_mb + j + 1) - cstart(w * n_mb + j);
      tr->traj[first + j].loss = count ? lsum[j] / (double)count : std::nan("");
    }
  }
  out->auc = out->cumulative_auc = std::nan("");
  out->has_auc = 0;
  if (predict_first) {
    // online AUC over the GLOBAL batch (trainer.cpp:141-151): gather every
    // rank's predictions/labels, then rank on the device
    const float* gp = d_pred_keep;
    const int32_t* gl = d_labels;
    uint32_t gn = n;
    if (tr->world > 1) {
      const int R = tr->world;
      std::vector<uint32_t> ns(R);
      uint32_t* dn = tr->gather_tmp.get<uint32_t>(2 * R);
      KP_CUDA(cudaMemcpyAsync(dn, &n, 4, cudaMemcpyHostToDevice, s));
      KP_NCCL(ncclAllGather(dn, dn + R, 1, ncclUint32, tr->comm->nc, s));
      KP_CUDA(cudaMemcpyAsync(ns.data(), dn + R, R * 4, cudaMemcpyDeviceToHost, s));
      KP_CUDA(cudaStreamSynchronize(s));
      uint32_t mx = 0;
      gn = 0;
      for (auto v : ns) mx = std::max(mx, v), gn += v;
      float* pp = tr->all_preds.get<float>((size_t)mx * R + mx);
      int32_t* ll = tr->all_labels.get<int32_t>((size_t)mx * R + mx);
      float* pad_p = pp + (size_t)mx * R;
      int32_t* pad_l = ll + (size_t)mx * R;
      KP_CUDA(cudaMemcpyAsync(pad_p, d_pred_keep, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
      KP_CUDA(cudaMemcpyAsync(pad_l, d_labels, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
      KP_NCCL(ncclAllGather(pad_p, pp, mx, ncclFloat32, tr->comm->nc, s));
      KP_NCCL(ncclAllGather(pad_l, ll, mx, ncclInt32, tr->comm->nc, s));
      // compact the rank slices (rank order = global instance order) into
      // separate buffers (in-place compaction would overlap)
      float* cp = tr->hist_scores.get_keep<float>(tr->hist_n + gn, tr->hist_n) + tr->hist_n;
      int32_t* cl = tr->hist_labels.get_keep<int32_t>(tr->hist_n + gn, tr->hist_n) + tr->hist_n;
      uint32_t off = 0;
      for (int r = 0; r < R; ++r) {
        if (ns[r]) {
          KP_CUDA(cudaMemcpyAsync(cp + off, pp + (size_t)r * mx, (size_t)ns[r] * 4, cudaMemcpyDeviceToDevice, s));
          KP_CUDA(cudaMemcpyAsync(cl + off, ll + (size_t)r * mx, (size_t)ns[r] * 4, cudaMemcpyDeviceToDevice, s));
        }
        off += ns[r];
      }
      gp = cp;
      gl = cl;
    }
    out->auc = device_auc(gp, gl, gn, tr->aucws, s);
    // AucAccumulator: every score so far, re-ranked (eval.cpp:41-50)
    float* hs = tr->hist_scores.get_keep<float>(tr->hist_n + gn, tr->hist_n);
    int32_t* hl = tr->hist_labels.get_keep<int32_t>(tr->hist_n + gn, tr->hist_n);
    if (gp != hs + tr->hist_n) {
      KP_CUDA(cudaMemcpyAsync(hs + tr->hist_n, gp, (size_t)gn * 4, cudaMemcpyDeviceToDevice, s));
      KP_CUDA(cudaMemcpyAsync(hl + tr->hist_n, gl, (size_t)gn * 4, cudaMemcpyDeviceToDevice, s));
    }
    tr->hist_n += gn;
    out->cumulative_auc = device_auc(hs, hl, (uint32_t)tr->hist_n, tr->aucws, s);
    out->has_auc = 1;
  }
  out->minibatch_steps = tr->t_global - steps_before;
  out->merges = tr->merges - merges_before;
  out->steps_total = tr->t_global;
  out->merges_total = tr->merges;
}

}  // namespace

// ============================================================== C ABI ====
extern "C" {

const char* kp_last_error(void) { return g_err.c_str(); }
const char* kp_version(void) { return "kpsim_b200 0.1.0 (sm_100a)"; }
uint64_t kp_launch_count(void) { return g_launches.load(); }

int kp_device_count(int* n) {
  return guard([&] { KP_CUDA(cudaGetDeviceCount(n)); });
}
int kp_host_alloc(size_t bytes, void** out) {
  return guard([&] { KP_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocDefault)); });
}
int kp_host_free(void* p) {
  return guard([&] { KP_CUDA(cudaFreeHost(p)); });
}
int kp_set_device(int device) {
  return guard([&] { KP_CUDA(cudaSetDevice(device)); });
}
int kp_dev_alloc(size_t bytes, void** out) {
  return guard([&] { KP_CUDA(cudaMalloc(out, bytes ? bytes : 1)); });
}
int kp_dev_free(void* p) {
  return guard([&] { KP_CUDA(cudaFree(p)); });
}
int kp_memcpy_h2d(void* d_dst, const void* src, size_t bytes) {
  return guard([&] { if (bytes) KP_CUDA(cudaMemcpy(d_dst, src, bytes, cudaMemcpyHostToDevice)); });
}
int kp_memcpy_d2h(void* dst, const void* d_src, size_t bytes) {
  return guard([&] { if (bytes) KP_CUDA(cudaMemcpy(dst, d_src, bytes, cudaMemcpyDeviceToHost)); });
}
int kp_memset_d(void* d_dst, int value, size_t bytes) {
  return guard([&] { if (bytes) KP_CUDA(cudaMemset(d_dst, value, bytes)); });
}

// ---- table ----
int kp_table_create(int device, uint64_t capacity, uint32_t dim, int rule, float init_w,
                    float init_s1, float init_s2, kp_table** out) {
  return guard([&] {
    auto h = std::make_unique<kp_table>();
    h->t = table_create(device, capacity, dim, rule, init_w, init_s1, init_s2);
    KP_CUDA(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    *out = h.release();
  });
}
int kp_table_destroy(kp_table* t) {
  return guard([&] {
    if (!t) return;
    if (t->s) cudaStreamDestroy(t->s);
    table_destroy(t->t);
    delete t;
  });
}
int kp_table_size(kp_table* t, uint64_t* n) {
  return guard([&] { *n = table_size(t->t, t->s); });
}
int kp_table_pull(kp_table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows, kp_stream s) {
  return guard([&] { table_pull(t->t, d_keys, n, d_rows, false, st(s)); });
}
int kp_table_insert_range(kp_table* t, uint64_t start, uint64_t step, uint64_t count, kp_stream s) {
  return guard([&] {
    KP_CUDA(cudaSetDevice(t->t->device));
    const uint64_t chunk = 1ull << 24;
    uint64_t* dk = t->keys.get<uint64_t>(std::min(count, chunk));
    uint32_t* dr = t->rows.get<uint32_t>(std::min(count, chunk));
    for (uint64_t i = 0; i < count; i += chunk) {
      const uint32_t n = (uint32_t)std::min(chunk, count - i);
      k_key_range<<<grid1(n), 256, 0, st(s)>>>(start + i * step, step, n, dk); ::kp::count_launch();
      table_pull(t->t, dk, n, dr, false, st(s));
    }
    KP_CUDA(cudaStreamSynchronize(st(s)));
    table_check_full(t->t, st(s));
  });
}
int kp_table_lookup(kp_table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows, kp_stream s) {
  return guard([&] { table_lookup(t->t, d_keys, n, d_rows, st(s)); });
}
int kp_table_gather(kp_table* t, const uint32_t* d_rows, uint32_t n, float* d_w, float* d_s1,
                    float* d_s2, kp_stream s) {
  return guard([&] { table_gather(t->t, d_rows, n, d_w, d_s1, d_s2, st(s)); });
}
int kp_table_set_rows(kp_table* t, const uint32_t* d_rows, uint32_t n, const float* d_w,
                      const float* d_s1, const float* d_s2, kp_stream s) {
  return guard([&] { table_set_rows(t->t, d_rows, n, d_w, d_s1, d_s2, st(s)); });
}
int kp_table_apply(kp_table* t, const uint32_t* d_rows, const float* d_grads, uint32_t n, float lr,
                   float beta1, float beta2, kp_stream s) {
  return guard([&] { table_apply(t->t, d_rows, d_grads, n, lr, beta1, beta2, st(s)); });
}

int kp_store_pull_batch(kp_table* t, const uint64_t* keys, uint32_t n, float* w, float* s1,
                        float* s2) {
  return guard([&] {
    KP_CHECK(n >= 1, kErrStore, "pull_batch: empty key set");
    Table* tb = t->t;
    KP_CUDA(cudaSetDevice(tb->device));
    uint64_t* dk = t->keys.get<uint64_t>(n);
    uint32_t* dr = t->rows.get<uint32_t>(n);
    KP_CUDA(cudaMemcpyAsync(dk, keys, (size_t)n * 8, cudaMemcpyHostToDevice, t->s));
    tb->epoch++;  // new working set (store.cpp:187)
    table_pull(tb, dk, n, dr, true, t->s);
    const size_t rn = (size_t)n * tb->dim;
    float* dw = t->w.get<float>(rn);
    float* d1 = t->s1.get<float>(rn);
    float* d2 = t->s2.get<float>(rn);
    table_gather(tb, dr, n, dw, d1, tb->rule == 1 ? d2 : nullptr, t->s);
    if (w) KP_CUDA(cudaMemcpyAsync(w, dw, rn * 4, cudaMemcpyDeviceToHost, t->s));
    if (s1) KP_CUDA(cudaMemcpyAsync(s1, d1, rn * 4, cudaMemcpyDeviceToHost, t->s));
    if (s2 && tb->rule == 1) KP_CUDA(cudaMemcpyAsync(s2, d2, rn * 4, cudaMemcpyDeviceToHost, t->s));
    KP_CUDA(cudaStreamSynchronize(t->s));
    table_check_full(tb, t->s);
  });
}

int kp_store_push_updates(kp_table* t, const uint64_t* keys, const float* grads, uint32_t n,
                          float lr, float beta1, float beta2, uint32_t* applied) {
  if (applied) *applied = 0;
  return guard([&] {
    if (n == 0) return;
    Table* tb = t->t;
    KP_CUDA(cudaSetDevice(tb->device));
    uint64_t* dk = t->keys.get<uint64_t>(n);
    uint32_t* dr = t->rows.get<uint32_t>(n);
    uint32_t* bad = t->scratch.get<uint32_t>(1);
    float* dg = t->grads.get<float>((size_t)n * tb->dim);
    KP_CUDA(cudaMemcpyAsync(dk, keys, (size_t)n * 8, cudaMemcpyHostToDevice, t->s));
    KP_CUDA(cudaMemcpyAsync(dg, grads, (size_t)n * tb->dim * 4, cudaMemcpyHostToDevice, t->s));
    table_lookup(tb, dk, n, dr, t->s);
    table_ws_check(tb, dr, n, bad, t->s);
    uint32_t h_bad = n;
    KP_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, t->s));
    KP_CUDA(cudaStreamSynchronize(t->s));
    table_apply(tb, dr, dg, h_bad, lr, beta1, beta2, t->s);
    KP_CUDA(cudaStreamSynchronize(t->s));
    if (applied) *applied = h_bad;
    KP_CHECK(h_bad == n, kErrStore,
             "push_updates: key " + std::to_string(keys[h_bad]) + " not in the current working set");
  });
}

int kp_store_lookup(kp_table* t, uint64_t key, float* w, float* s1, float* s2) {
  return guard([&] {
    Table* tb = t->t;
    KP_CUDA(cudaSetDevice(tb->device));
    uint64_t* dk = t->keys.get<uint64_t>(1);
    uint32_t* dr = t->rows.get<uint32_t>(1);
    uint32_t* bad = t->scratch.get<uint32_t>(1);
    KP_CUDA(cudaMemcpyAsync(dk, &key, 8, cudaMemcpyHostToDevice, t->s));
    table_lookup(tb, dk, 1, dr, t->s);
    table_ws_check(tb, dr, 1, bad, t->s);
    uint32_t h_bad = 1;
    KP_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, t->s));
    KP_CUDA(cudaStreamSynchronize(t->s));
    KP_CHECK(h_bad == 1, kErrStore, "lookup: key " + std::to_string(key) + " not in the current working set");
    float* dw = t->w.get<float>(tb->dim);
    float* d1 = t->s1.get<float>(tb->dim);
    float* d2 = t->s2.get<float>(tb->dim);
    table_gather(tb, dr, 1, dw, d1, tb->rule == 1 ? d2 : nullptr, t->s);
    if (w) KP_CUDA(cudaMemcpyAsync(w, dw, tb->dim * 4, cudaMemcpyDeviceToHost, t->s));
    if (s1) KP_CUDA(cudaMemcpyAsync(s1, d1, tb->dim * 4, cudaMemcpyDeviceToHost, t->s));
    if (s2 && tb->rule == 1) KP_CUDA(cudaMemcpyAsync(s2, d2, tb->dim * 4, cudaMemcpyDeviceToHost, t->s));
    KP_CUDA(cudaStreamSynchronize(t->s));
  });
}

int kp_table_export(kp_table* t, uint64_t* keys, float* w, float* s1, float* s2, uint64_t cap,
                    uint64_t* n_out) {
  return guard([&] {
    Table* tb = t->t;
    KP_CUDA(cudaSetDevice(tb->device));
    const uint64_t n = table_size(tb, t->s);
    *n_out = n;
    if (!keys) return;
    KP_CHECK(cap >= n, kErrGeneric, "table_export: output capacity too small");
    if (n == 0) return;
    uint64_t* dk = t->keys.get<uint64_t>(n);
    uint32_t* dr = t->rows.get<uint32_t>(n);
    auto* cnt = reinterpret_cast<unsigned long long*>(t->scratch.get<uint64_t>(1));
    table_export(tb, dk, dr, cnt, t->s);
    std::vector<uint64_t> hk(n);
    std::vector<uint32_t> hr(n);
    KP_CUDA(cudaMemcpyAsync(hk.data(), dk, n * 8, cudaMemcpyDeviceToHost, t->s));
    KP_CUDA(cudaMemcpyAsync(hr.data(), dr, n * 4, cudaMemcpyDeviceToHost, t->s));
    KP_CUDA(cudaStreamSynchronize(t->s));
    std::vector<uint64_t> order(n);
    for (uint64_t i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return hk[a] < hk[b]; });
    std::vector<uint32_t> sr(n);
    for (uint64_t i = 0; i < n; ++i) {
      keys[i] = hk[order[i]];
      sr[i] = hr[order[i]];
    }
    KP_CUDA(cudaMemcpyAsync(dr, sr.data(), n * 4, cudaMemcpyHostToDevice, t->s));
    const size_t rn = (size_t)n * tb->dim;
    float* dw = t->w.get<float>(rn);
    float* d1 = t->s1.get<float>(rn);
    float* d2 = t->s2.get<float>(rn);
    table_gather(tb, dr, (uint32_t)n, dw, d1, tb->rule == 1 ? d2 : nullptr, t->s);
    if (w) KP_CUDA(cudaMemcpyAsync(w, dw, rn * 4, cudaMemcpyDeviceToHost, t->s));
    if (s1) KP_CUDA(cudaMemcpyAsync(s1, d1, rn * 4, cudaMemcpyDeviceToHost, t->s));
    if (s2 && tb->rule == 1) KP_CUDA(cudaMemcpyAsync(s2, d2, rn * 4, cudaMemcpyDeviceToHost, t->s));
    KP_CUDA(cudaStreamSynchronize(t->s));
  });
}

// ---- dedup / shard ----
// Workspaces of the stand-alone entry points live on the device they were
// first used on, so keep one per (thread, device).
extern "C++" {
template <class W>
W& dev_ws() {
  static thread_local W ws[16];
  int dev = 0;
  KP_CUDA(cudaGetDevice(&dev));
  KP_CHECK(dev >= 0 && dev < 16, kErrConfig, "device ordinal out of range");
  return ws[dev];
}
}
int kp_dedup(const uint64_t* d_keys, uint32_t n, uint64_t* d_unique, uint32_t* d_inverse,
             uint32_t* d_seg, uint32_t* n_unique, kp_stream s) {
  return guard([&] {
    DedupWs& ws = dev_ws<DedupWs>();
    dedup(d_keys, n, ws, st(s));
    const uint32_t U = ws.n_unique;
    *n_unique = U;
    if (U) KP_CUDA(cudaMemcpyAsync(d_unique, ws.d_unique, (size_t)U * 8, cudaMemcpyDeviceToDevice, st(s)));
    if (n && d_inverse)
      KP_CUDA(cudaMemcpyAsync(d_inverse, ws.d_inverse, (size_t)n * 4, cudaMemcpyDeviceToDevice, st(s)));
    if (d_seg) KP_CUDA(cudaMemcpyAsync(d_seg, ws.d_seg, (size_t)(U + 1) * 4, cudaMemcpyDeviceToDevice, st(s)));
    KP_CUDA(cudaStreamSynchronize(st(s)));
  });
}
int kp_dedup_runs(const uint64_t* d_keys, uint32_t n, const uint64_t* run_off, uint32_t n_runs,
                  uint64_t* d_unique, uint32_t* d_inverse, uint32_t* d_seg, uint32_t* d_sorted_pos,
                  uint32_t* n_unique, kp_stream s) {
  return guard([&] {
    KP_CHECK(n_runs >= 1 && run_off && run_off[0] == 0 && run_off[n_runs] == n, kErrConfig,
             "dedup_runs: run offsets must start at 0 and end at n");
    DedupWs& ws = dev_ws<DedupWs>();
    std::vector<uint64_t> ro(run_off, run_off + n_runs + 1);
    dedup_runs(d_keys, n, ro, ws, st(s));
    const uint32_t U = ws.n_unique;
    *n_unique = U;
    if (U) KP_CUDA(cudaMemcpyAsync(d_unique, ws.d_unique, (size_t)U * 8, cudaMemcpyDeviceToDevice, st(s)));
    if (n && d_inverse)
      KP_CUDA(cudaMemcpyAsync(d_inverse, ws.d_inverse, (size_t)n * 4, cudaMemcpyDeviceToDevice, st(s)));
    if (d_seg) KP_CUDA(cudaMemcpyAsync(d_seg, ws.d_seg, (size_t)(U + 1) * 4, cudaMemcpyDeviceToDevice, st(s)));
    if (n && d_sorted_pos)
      KP_CUDA(cudaMemcpyAsync(d_sorted_pos, ws.sorted_vals, (size_t)n * 4, cudaMemcpyDeviceToDevice, st(s)));
    KP_CUDA(cudaStreamSynchronize(st(s)));
  });
}
int kp_shard(const uint64_t* d_unique, uint32_t n, uint32_t G, uint32_t* d_perm, uint32_t* d_pos,
             uint64_t* counts, kp_stream s) {
  return guard([&] {
    ShardWs& ws = dev_ws<ShardWs>();
    shard(d_unique, n, G, d_perm, d_pos, counts, ws, st(s));
  });
}

// ---- dense ----
int kp_dense_local_step(float* d_x, float* d_m, float* d_v, const float* d_vbar, const float* d_g,
                        uint64_t D, float alpha, float beta1, float beta2, kp_stream s) {
  return guard([&] { dense_local_step(d_x, d_m, d_v, d_vbar, d_g, D, {alpha, beta1, beta2}, st(s)); });
}
int kp_dense_moments(float* d_m, float* d_v, const float* d_g, uint64_t D, float beta1, float beta2,
                     kp_stream s) {
  return guard([&] { dense_moments(d_m, d_v, d_g, D, {0.f, beta1, beta2}, st(s)); });
}
int kp_centered_mean(const float* d_vecs, uint64_t stride, uint32_t n, uint64_t D, float* d_out,
                     kp_stream s) {
  return guard([&] {
    KP_CHECK(n >= 1, kErrGeneric, "global_merge: empty worker list");
    centered_mean(d_vecs, stride, n, D, d_out, st(s));
  });
}
int kp_kstep_merge(kp_comm* comm, float* d_x, float* d_m, float* d_v, float* d_vbar, uint32_t W,
                   uint64_t D, float alpha, int reset_local_v, kp_stream s) {
  return guard([&] {
    KP_CHECK(W >= 1, kErrGeneric, "global_merge: empty worker list");
    MergeWs& ws = dev_ws<MergeWs>();
    merge_states(comm, st(s), W, D, d_x, d_m, d_v, d_vbar, alpha, reset_local_v != 0, ws);
    KP_CUDA(cudaStreamSynchronize(st(s)));
  });
}

// ---- AUC ----
int kp_compute_auc(const float* d_scores, const int32_t* d_labels, uint32_t n, double* auc,
                   kp_stream s) {
  return guard([&] {
    AucWs& ws = dev_ws<AucWs>();
    *auc = device_auc(d_scores, d_labels, n, ws, st(s));
  });
}

// ---- GEMM ----
int kp_gemm_nt(const float* d_A, int lda, const float* d_B, int ldb, float* d_C, int ldc, int M,
               int N, int K, int engine, kp_stream s) {
  return guard([&] {
    const bool tc_ok = tc_gemm_supported(M, N, K, d_A, lda, d_B, ldb);
    KP_CHECK(engine < 2 || tc_ok, kErrConfig, "gemm_nt: shape/alignment not supported by tcgen05 path");
    KP_CHECK(engine != 3 || (ldb % 8 == 0 && K % 8 == 0), kErrConfig,
             "gemm_nt: fp16 path needs K and ldb multiples of 8");
    KP_CHECK(engine < 4 || (lda == K && ldb == K && K % 8 == 0), kErrConfig,
             "gemm_nt: pre-split fp16 path needs contiguous rows and K % 8 == 0");
    if (engine == 1 || !tc_ok) {
      simt_gemm_nt(M, N, K, d_A, lda, d_B, ldb, d_C, ldc, st(s));
    } else if (engine >= 4 && engine <= 6) {
      // 3xFP16 on pre-split planes (kp_gemm_h3.cu): split both operands per
      // row, then the all-TMA GEMM; engine 5 runs it stream-K over K
      struct PWs {
        DevBuf ah, al, ae, bh, bl, be, ws;
      };
      PWs& w = dev_ws<PWs>();
      auto* ah = reinterpret_cast<__half*>(w.ah.get<uint16_t>((size_t)M * K));
      auto* al = reinterpret_cast<__half*>(w.al.get<uint16_t>((size_t)M * K));
      auto* bh = reinterpret_cast<__half*>(w.bh.get<uint16_t>((size_t)N * K));
      auto* bl = reinterpret_cast<__half*>(w.bl.get<uint16_t>((size_t)N * K));
      int* ae = w.ae.get<int>(M);
      int* be = w.be.get<int>(N);
      split_rows_h(d_A, M, K, K, ah, al, ae, st(s));
      split_rows_h(d_B, N, K, K, bh, bl, be, st(s));
      GemmEpi ep{0, 0, nullptr, nullptr, 0, nullptr, 1, 1};
      h3_gemm(H3Operand{ah, al, ae, K}, false, H3Operand{bh, bl, be, K}, false, M, N, K, d_C, ldc, ep,
              engine - 4, engine > 4 ? w.ws.get<float>(h3_splitk_ws_floats(M, N)) : nullptr, st(s));
      KP_CUDA(cudaStreamSynchronize(st(s)));
    } else if (engine == 3) {
      // fp16-operand path (per-row scaled 3xFP16), as used for the first MLP layer
      struct HWs {
        DevBuf amax, bhi, blo, bexp;
      };
      HWs& hw = dev_ws<HWs>();
      DevBuf &amax = hw.amax, &bhi = hw.bhi, &blo = hw.blo, &bexp = hw.bexp;
      float* am = amax.get<float>(M);
      rowmax(d_A, M, K, lda, am, st(s));
      __half* h = reinterpret_cast<__half*>(bhi.get<uint16_t>((size_t)N * ldb));
      __half* l = reinterpret_cast<__half*>(blo.get<uint16_t>((size_t)N * ldb));
      int* ex = bexp.get<int>(N);
      split_h(d_B, N, K, ldb, h, l, ex, st(s));
      GemmEpi ep{0, 0, nullptr, nullptr, 0, nullptr, 1, 1};
      tc_gemm_nt_h(M, N, K, d_A, lda, am, h, l, ex, ldb, d_C, ldc, ep, st(s));
      KP_CUDA(cudaStreamSynchronize(st(s)));
    } else {
      GemmEpi ep{0, 0, nullptr, nullptr, 0, nullptr, 1, 1};
      tc_gemm_nt(M, N, K, d_A, lda, d_B, ldb, d_C, ldc, ep, st(s));
      KP_CUDA(cudaStreamSynchronize(st(s)));
    }
    KP_CUDA(cudaGetLastError());
  });
}

int kp_gemm_tn(const float* d_A, int lda, const float* d_B, int ldb, float* d_C, int ldc, int M,
               int N, int K, int engine, kp_stream s) {
  return guard([&] {
    const bool tc_ok = tc_gemm_supported(M, N, K, d_A, lda, d_B, ldb);
    KP_CHECK(engine != 2 || tc_ok, kErrConfig, "gemm_tn: shape/alignment not supported by tcgen05 path");
    KP_CHECK(engine < 4 || (lda == M && ldb == N && M % 8 == 0 && N % 8 == 0), kErrConfig,
             "gemm_tn: pre-split fp16 path needs contiguous rows and M, N % 8 == 0");
    if (engine == 1 || !tc_ok) {
      simt_gemm_tn(M, N, K, d_A, lda, d_B, ldb, d_C, ldc, st(s));
    } else if (engine >= 4 && engine <= 6) {
      // both operands MN-major ([K][M], [K][N]): planes with one exponent per
      // column, the all-TMA 3xFP16 GEMM (engine 5: stream-K over K)
      struct PWs {
        DevBuf ah, al, ae, bh, bl, be, cm, ws;
      };
      PWs& w = dev_ws<PWs>();
      auto* ah = reinterpret_cast<__half*>(w.ah.get<uint16_t>((size_t)M * K));
      auto* al = reinterpret_cast<__half*>(w.al.get<uint16_t>((size_t)M * K));
      auto* bh = reinterpret_cast<__half*>(w.bh.get<uint16_t>((size_t)N * K));
      auto* bl = reinterpret_cast<__half*>(w.bl.get<uint16_t>((size_t)N * K));
      int* ae = w.ae.get<int>(M);
      int* be = w.be.get<int>(N);
      unsigned* cm = w.cm.get<unsigned>(std::max(M, N));
      split_cols_scaled_h(d_A, K, M, nullptr, cm, ah, al, ae, st(s));
      split_cols_scaled_h(d_B, K, N, nullptr, cm, bh, bl, be, st(s));
      GemmEpi ep{0, 0, nullptr, nullptr, 0, nullptr, 1, 1};
      h3_gemm(H3Operand{ah, al, ae, M}, true, H3Operand{bh, bl, be, N}, true, M, N, K, d_C, ldc, ep,
              engine - 4, engine > 4 ? w.ws.get<float>(h3_splitk_ws_floats(M, N)) : nullptr, st(s));
      KP_CUDA(cudaStreamSynchronize(st(s)));
    } else {
      const int sp = tc_splits(M, N, K);
      if (sp == 1) {
        tc_gemm_tn(M, N, K, d_A, lda, d_B, ldb, d_C, ldc, 1, st(s));
      } else {
        DevBuf& part = dev_ws<DevBuf>();
        float* p = part.get<float>((size_t)sp * M * ldc);
        const int got = tc_gemm_tn(M, N, K, d_A, lda, d_B, ldb, p, ldc, sp, st(s));
        reduce_splits(p, got, (size_t)M * ldc, d_C, st(s));
        KP_CUDA(cudaStreamSynchronize(st(s)));
      }
    }
    KP_CUDA(cudaStreamSynchronize(st(s)));
    KP_CUDA(cudaGetLastError());
  });
}

// ---- comm ----
int kp_comm_unique_id(uint8_t id[128]) {
  return guard([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    KP_NCCL(ncclGetUniqueId(&u));
    std::memcpy(id, &u, 128);
  });
}
int kp_comm_init(const uint8_t id[128], int rank, int world, int device, kp_comm** out) {
  return guard([&] {
    KP_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<kp_comm>();
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    KP_NCCL(ncclCommInitRank(&c->nc, world, u, rank));
    KP_NCCL(ncclCommSplit(c->nc, 0, rank, &c->nc2, nullptr));
    c->rank = rank;
    c->world = world;
    c->device = device;
    *out = c.release();
  });
}
int kp_comm_destroy(kp_comm* c) {
  return guard([&] {
    if (!c) return;
    if (c->nc2) ncclCommDestroy(c->nc2);
    if (c->nc) ncclCommDestroy(c->nc);
    delete c;
  });
}
int kp_comm_rank(kp_comm* c, int* rank, int* world) {
  return guard([&] {
    *rank = c->rank;
    *world = c->world;
  });
}

// ---- trainer ----
int kp_trainer_create(const kp_trainer_config* cfg, kp_comm* comm, int device, kp_trainer** out) {
  return guard([&] {
    const kp_trainer_config& c = *cfg;
    KP_CHECK(c.n_workers >= 1 && c.local_workers >= 1, kErrConfig, "workers must be >= 1");
    const int world = comm ? comm->world : 1;
    KP_CHECK((uint64_t)c.local_workers * world == c.n_workers, kErrConfig,
             "n_workers must equal world_size * local_workers");
    KP_CHECK(c.minibatch_size >= 1, kErrConfig, "minibatch_size must be >= 1");
    KP_CHECK(c.alpha > 0, kErrConfig, "adam: alpha must be > 0");
    KP_CHECK(c.beta1 >= 0 && c.beta1 < 1, kErrConfig, "adam: beta1 must be in [0,1)");
    KP_CHECK(c.beta2 >= 0 && c.beta2 < 1, kErrConfig, "adam: beta2 must be in [0,1)");
    KP_CHECK(c.epsilon > 0, kErrConfig, "adam: epsilon must be > 0");
    KP_CHECK(c.k >= 1, kErrConfig, "adam: k must be >= 1");
    KP_CHECK(c.embedding_dim >= 1, kErrConfig, "model: embedding_dim must be >= 1");
    KP_CHECK(c.n_slots >= 1 && c.n_slots <= 65535, kErrConfig, "n_slots must be in [1, 65535]");
    KP_CHECK(c.n_hidden <= 8, kErrConfig, "at most 8 hidden layers");
    for (uint32_t i = 0; i < c.n_hidden; ++i)
      KP_CHECK(c.hidden[i] >= 1, kErrConfig, "model: hidden widths must be >= 1");
    KP_CHECK(c.table_capacity >= 1, kErrConfig, "table_capacity must be >= 1");
    KP_CUDA(cudaSetDevice(device));
    auto tr = std::make_unique<kp_trainer>();
    tr->cfg = c;
    tr->device = device;
    tr->comm = comm;
    tr->world = world;
    tr->rank = comm ? comm->rank : 0;
    tr->W = c.local_workers;
    tr->N = c.n_workers;
    tr->S = c.n_slots;
    tr->e = c.embedding_dim;
    KP_CUDA(cudaStreamCreateWithFlags(&tr->s, cudaStreamNonBlocking));
    // model shape, flat layout per layer W then bias (model.cpp:55-66)
    MlpShape& m = tr->shape;
    m.widths[0] = c.n_slots * c.embedding_dim;
    for (uint32_t i = 0; i < c.n_hidden; ++i) m.widths[i + 1] = c.hidden[i];
    m.widths[c.n_hidden + 1] = 1;
    m.n_layers = c.n_hidden + 1;
    m.activation = c.activation;
    for (uint32_t l = 0; l < m.n_layers; ++l) {
      m.w_off[l] = m.D;
      m.D += (uint64_t)m.widths[l] * m.widths[l + 1];
      m.b_off[l] = m.D;
      m.D += m.widths[l + 1];
    }
    tr->D = m.D;
    // layer 1 on pre-split fp16 planes written by the pooling kernel
    {
      // opt-in (KP_FUSED_POOL=1): measured slower, see DESIGN.md §4.3
      const char* e = getenv("KP_FUSED_POOL");
      tr->fused_pool = e && e[0] == '1';
      const char* f = getenv("KP_SYNC_FREE");
      tr->sync_free = !(f && f[0] == '0');
      const char* g = getenv("KP_GRAPH");
      tr->graphs = !(g && g[0] == '0');
    }
    // (the backward's plane operands [B][hidden1] and W1^T [S*e][hidden1]
    // need 16-byte rows: hidden1 % 8 == 0)
    if (const char* e = getenv("KP_TC_MIN_MFLOP")) tr->mlp.tc_min_flop = atof(e) * 1e6;
    tr->planes = c.n_hidden >= 1 && tc_enabled() && tc_h_enabled() && h3_enabled() &&
                 pool_planes_supported(c.n_slots, c.embedding_dim) && m.widths[1] % 8 == 0 &&
                 tc_worth((int)std::min<uint64_t>(c.minibatch_size, 1u << 30), (int)m.widths[1],
                          (int)m.widths[0], tr->mlp.tc_min_flop);
    const uint64_t D = m.D, W = tr->W;
    std::vector<double> x0(D);
    init_dense_host(c.seed, D, x0.data());
    std::vector<float> hx(D), hv(D, (float)c.epsilon);
    for (uint64_t j = 0; j < D; ++j) hx[j] = (float)x0[j];
    KP_CUDA(cudaMalloc(&tr->x, W * D * 4));
    KP_CUDA(cudaMalloc(&tr->m, W * D * 4));
    KP_CUDA(cudaMalloc(&tr->v, W * D * 4));
    KP_CUDA(cudaMalloc(&tr->vbar, W * D * 4));
    KP_CUDA(cudaMalloc(&tr->g, W * D * 4));
    KP_CUDA(cudaMemset(tr->m, 0, W * D * 4));
    for (uint64_t l = 0; l < W; ++l) {
      KP_CUDA(cudaMemcpy(tr->x + l * D, hx.data(), D * 4, cudaMemcpyHostToDevice));
      KP_CUDA(cudaMemcpy(tr->v + l * D, hv.data(), D * 4, cudaMemcpyHostToDevice));
      KP_CUDA(cudaMemcpy(tr->vbar + l * D, hv.data(), D * 4, cudaMemcpyHostToDevice));
    }
    const int rule = c.sparse_rule;
    tr->tab.t = table_create(device, c.table_capacity, c.embedding_dim, rule, 0.f,
                             rule == 0 ? 1e-6f : 0.f, rule == 0 ? 0.f : (float)c.sparse_eps);
    tr->tab.s = nullptr;
    tr->check.get<uint32_t>(2);
    *out = tr.release();
  });
}

int kp_trainer_destroy(kp_trainer* tr) {
  return guard([&] {
    if (!tr) return;
    cudaSetDevice(tr->device);
    delete tr;
  });
}

int kp_trainer_train_batch(kp_trainer* tr, const uint32_t* offs, const uint64_t* keys,
                           const uint16_t* slots, const int32_t* labels, uint32_t n,
                           uint64_t global_n, uint64_t global_first, int predict_first,
                           float* preds, kp_batch_result* out) {
  return guard([&] {
    KP_CUDA(cudaSetDevice(tr->device));
    const uint32_t O = offs[n];
    uint32_t* d_offs = tr->in_offs.get<uint32_t>(n + 1);
    uint64_t* d_keys = tr->in_keys.get<uint64_t>(std::max<uint32_t>(O, 1));
    uint16_t* d_slots = slots ? tr->in_slots.get<uint16_t>(std::max<uint32_t>(O, 1)) : nullptr;
    int32_t* d_labels = tr->in_labels.get<int32_t>(std::max<uint32_t>(n, 1));
    KP_CUDA(cudaMemcpyAsync(d_offs, offs, (size_t)(n + 1) * 4, cudaMemcpyHostToDevice, tr->s));
    KP_CUDA(cudaMemcpyAsync(d_keys, keys, (size_t)O * 8, cudaMemcpyHostToDevice, tr->s));
    if (slots) KP_CUDA(cudaMemcpyAsync(d_slots, slots, (size_t)O * 2, cudaMemcpyHostToDevice, tr->s));
    KP_CUDA(cudaMemcpyAsync(d_labels, labels, (size_t)n * 4, cudaMemcpyHostToDevice, tr->s));
    train_batch_impl(tr, offs, d_offs, d_keys, d_slots, d_labels, n, global_n, global_first,
                     predict_first != 0, preds, out);
  });
}

int kp_trainer_stage_batch(kp_trainer* tr, int slot, const uint32_t* offs, const uint64_t* keys,
                           const uint16_t* slots, const int32_t* labels, uint32_t n) {
  return guard([&] {
    KP_CHECK(slot == 0 || slot == 1, kErrGeneric, "stage slot must be 0 or 1");
    KP_CUDA(cudaSetDevice(tr->device));
    if (!tr->copy_s) KP_CUDA(cudaStreamCreateWithFlags(&tr->copy_s, cudaStreamNonBlocking));
    auto& st = tr->stage[slot];
    if (!st.ev) KP_CUDA(cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming));
    const uint32_t O = offs[n];
    st.offs.get<uint32_t>(n + 1);
    st.keys.get<uint64_t>(std::max<uint32_t>(O, 1));
    if (slots) st.slots.get<uint16_t>(std::max<uint32_t>(O, 1));
    st.labels.get<int32_t>(std::max<uint32_t>(n, 1));
    // The H2D itself is issued at the next point where the trainer has no
    // host readback left in its current step (issue_staged), so the step's
    // small D2H readbacks never queue behind a 66 MB copy.
    st.h_src_offs = offs;
    st.h_src_keys = keys;
    st.h_src_slots = slots;
    st.h_src_labels = labels;
    st.pending = true;
    st.n = n;  // (offs stays the caller's: valid until train_staged returns)
    st.has_slots = slots != nullptr;
    st.ready = true;
  });
}

int kp_trainer_train_staged(kp_trainer* tr, int slot, uint64_t global_n, uint64_t global_first,
                            int predict_first, float* preds, kp_batch_result* out) {
  return guard([&] {
    KP_CHECK(slot == 0 || slot == 1, kErrGeneric, "stage slot must be 0 or 1");
    auto& st = tr->stage[slot];
    KP_CHECK(st.ready, kErrGeneric, "train_staged: nothing staged in this slot");
    KP_CUDA(cudaSetDevice(tr->device));
    if (st.pending) issue_staged(tr, slot);
    KP_CUDA(cudaStreamWaitEvent(tr->s, st.ev, 0));
    st.ready = false;
    train_batch_impl(tr, st.h_src_offs, static_cast<const uint32_t*>(st.offs.p),
                     static_cast<const uint64_t*>(st.keys.p),
                     st.has_slots ? static_cast<const uint16_t*>(st.slots.p) : nullptr,
                     static_cast<const int32_t*>(st.labels.p), st.n, global_n, global_first,
                     predict_first != 0, preds, out);
    if (!st.used) KP_CUDA(cudaEventCreateWithFlags(&st.used, cudaEventDisableTiming));
    KP_CUDA(cudaEventRecord(st.used, tr->s));
    st.used_set = true;
  });
}

int kp_trainer_train_batch_device(kp_trainer* tr, const uint32_t* h_offs, const uint32_t* d_offs,
                                  const uint64_t* d_keys, const uint16_t* d_slots,
                                  const int32_t* d_labels, uint32_t n, uint64_t global_n,
                                  uint64_t global_first, int predict_first, float* preds,
                                  kp_batch_result* out) {
  return guard([&] {
    KP_CUDA(cudaSetDevice(tr->device));
    train_batch_impl(tr, h_offs, d_offs, d_keys, d_slots, d_labels, n, global_n, global_first,
                     predict_first != 0, preds, out);
  });
}

int kp_trainer_dense_dim(kp_trainer* tr, uint64_t* D) {
  return guard([&] { *D = tr->D; });
}

int kp_trainer_worker_state(kp_trainer* tr, uint32_t l, float* x, float* m, float* v, float* vbar) {
  return guard([&] {
    KP_CHECK(l < tr->W, kErrGeneric, "worker index out of range");
    KP_CUDA(cudaSetDevice(tr->device));
    const uint64_t D = tr->D;
    // a read-only getter: x_uniform must stay rank-symmetric (it selects a
    // collective path in compute_xbar), so reading a state never clears it
    if (x) KP_CUDA(cudaMemcpyAsync(x, tr->x + l * D, D * 4, cudaMemcpyDeviceToHost, tr->s));
    if (m) KP_CUDA(cudaMemcpyAsync(m, tr->m + l * D, D * 4, cudaMemcpyDeviceToHost, tr->s));
    if (v) KP_CUDA(cudaMemcpyAsync(v, tr->v + l * D, D * 4, cudaMemcpyDeviceToHost, tr->s));
    if (vbar) KP_CUDA(cudaMemcpyAsync(vbar, tr->vbar + l * D, D * 4, cudaMemcpyDeviceToHost, tr->s));
    KP_CUDA(cudaStreamSynchronize(tr->s));
  });
}

int kp_trainer_set_worker_state(kp_trainer* tr, uint32_t l, const float* x, const float* m,
                                const float* v, const float* vbar) {
  return guard([&] {
    KP_CHECK(l < tr->W, kErrGeneric, "worker index out of range");
    KP_CUDA(cudaSetDevice(tr->device));
    const uint64_t D = tr->D;
    if (x) tr->x_uniform = false;
    if (x) KP_CUDA(cudaMemcpyAsync(tr->x + l * D, x, D * 4, cudaMemcpyHostToDevice, tr->s));
    if (m) KP_CUDA(cudaMemcpyAsync(tr->m + l * D, m, D * 4, cudaMemcpyHostToDevice, tr->s));
    if (v) KP_CUDA(cudaMemcpyAsync(tr->v + l * D, v, D * 4, cudaMemcpyHostToDevice, tr->s));
    if (vbar) KP_CUDA(cudaMemcpyAsync(tr->vbar + l * D, vbar, D * 4, cudaMemcpyHostToDevice, tr->s));
    KP_CUDA(cudaStreamSynchronize(tr->s));
  });
}

int kp_trainer_xbar(kp_trainer* tr, float* out) {
  return guard([&] {
    KP_CUDA(cudaSetDevice(tr->device));
    float* xb = tr->xbar.get<float>(tr->D);
    compute_xbar(tr, xb);
    KP_CUDA(cudaMemcpyAsync(out, xb, tr->D * 4, cudaMemcpyDeviceToHost, tr->s));
    KP_CUDA(cudaStreamSynchronize(tr->s));
  });
}

int kp_trainer_table(kp_trainer* tr, kp_table** out) {
  return guard([&] {
    if (!tr->tab.s) KP_CUDA(cudaStreamCreateWithFlags(&tr->tab.s, cudaStreamNonBlocking));
    *out = &tr->tab;
  });
}

int kp_trainer_profile(kp_trainer* tr, int enable, double* stage_ms, uint64_t* counters) {
  return guard([&] {
    if (stage_ms)
      for (int i = 0; i < 7; ++i) stage_ms[i] = tr->stage_ms[i];
    if (counters) {
      counters[0] = tr->prof_steps;
      counters[1] = tr->prof_unique;
      counters[2] = tr->prof_occ;
      counters[3] = tr->prof_owner_unique;
      counters[4] = tr->prof_recv;
    }
    for (double& d : tr->stage_ms) d = 0;
    tr->prof_steps = tr->prof_unique = tr->prof_occ = tr->prof_owner_unique = tr->prof_recv = 0;
    tr->prof = enable != 0;
  });
}

int kp_trainer_ledger(kp_trainer* tr, uint64_t bytes[5], uint64_t count[5]) {
  return guard([&] {
    for (int i = 0; i < 5; ++i) {
      bytes[i] = tr->led_bytes[i];
      count[i] = tr->led_count[i];
    }
  });
}

int kp_trainer_record_trajectory(kp_trainer* tr, int enable) {
  return guard([&] {
    if (enable && !tr->traj_on) {
      tr->traj_prev_vbar.resize(tr->D);
      KP_CUDA(cudaSetDevice(tr->device));
      KP_CUDA(cudaMemcpyAsync(tr->traj_prev_vbar.data(), tr->vbar, tr->D * 4, cudaMemcpyDeviceToHost, tr->s));
      KP_CUDA(cudaStreamSynchronize(tr->s));
    }
    tr->traj_on = enable != 0;
  });
}

int kp_trainer_trajectory(kp_trainer* tr, uint64_t i, uint64_t* step, int* merged, double* loss,
                          double* a3, float* x_bar, float* v_bar, uint64_t* n_steps) {
  return guard([&] {
    if (n_steps) *n_steps = tr->traj.size();
    if (!step && !x_bar && !v_bar && !merged && !loss && !a3) return;
    KP_CHECK(i < tr->traj.size(), kErrGeneric, "trajectory step index out of range");
    const auto& r = tr->traj[i];
    if (step) *step = r.step;
    if (merged) *merged = r.merged;
    if (loss) *loss = r.loss;
    if (a3) *a3 = r.a3;
    if (x_bar) std::memcpy(x_bar, r.x_bar.data(), tr->D * 4);
    if (v_bar) std::memcpy(v_bar, r.v_bar.data(), tr->D * 4);
  });
}

int kp_trainer_stream(kp_trainer* tr, kp_stream* s) {
  return guard([&] { *s = tr->s; });
}

}  // extern "C"
