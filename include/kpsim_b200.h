/* kpsim_b200 -- C ABI of the B200-native sparse-embedding training hot path.
 *
 * This is the drop-in boundary for the reference's per-batch training path
 * (kpsim, /root/reference/proj). Each entry point names the reference interface
 * it replaces. Rules:
 *   - no C++ exceptions cross this boundary: every call returns a status code
 *     (KP_OK = 0) and kp_last_error() holds the message of the last failure on
 *     the calling thread. Status codes map to the reference's exception types
 *     (kpsim::Error / ConfigError / StoreError, proj/include/kpsim/common.hpp:13-22,
 *     store.hpp:17-20);
 *   - "d_" pointers are caller-owned DEVICE memory, calls taking a kp_stream
 *     are stream-ordered; plain pointers are HOST memory and those calls are
 *     synchronous (the reference's value-returning semantics);
 *   - tables, trainers and communicators are opaque handles.
 * There is no CPU fallback: every compute call runs sm_100a kernels and fails
 * with KP_ERR_CUDA when no B200 is present.
 */
#ifndef KPSIM_B200_H
#define KPSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KP_OK 0
#define KP_ERR 1             /* kpsim::Error */
#define KP_ERR_CONFIG 2      /* kpsim::ConfigError */
#define KP_ERR_STORE 3       /* kpsim::StoreError */
#define KP_ERR_CUDA 4
#define KP_ERR_NCCL 5
#define KP_ERR_TABLE_FULL 6

#define KP_RULE_ADAGRAD 0
#define KP_RULE_ADAM 1

typedef struct kp_table kp_table;
typedef struct kp_trainer kp_trainer;
typedef struct kp_comm kp_comm;
typedef void* kp_stream; /* cudaStream_t; NULL = legacy default stream */

const char* kp_last_error(void);
const char* kp_version(void);
int kp_device_count(int* n);
/* Pinned host memory for end-to-end host->device feeds. */
int kp_host_alloc(size_t bytes, void** out);
int kp_host_free(void* p);
/* Number of kernels this library launched (process-wide counter). */
uint64_t kp_launch_count(void);
/* Device memory plumbing for host shims (synchronous). */
int kp_set_device(int device);
int kp_dev_alloc(size_t bytes, void** out);
int kp_dev_free(void* p);
int kp_memcpy_h2d(void* d_dst, const void* src, size_t bytes);
int kp_memcpy_d2h(void* dst, const void* d_src, size_t bytes);
int kp_memset_d(void* d_dst, int value, size_t bytes);

/* ------------------------------------------------------------ table ---
 * The embedding table that replaces kpsim::TieredStore
 * (proj/include/kpsim/store.hpp:47-97, proj/src/store.cpp:53-245) with an
 * HBM-resident open-addressing table: keys u64 -> dense fp32 rows.
 * rule KP_RULE_ADAGRAD: state {w, acc}, fresh {init_w, init_s1}
 *   (reference: w = 0, acc = kFreshAccumulator = 1e-6, store.hpp:49);
 * rule KP_RULE_ADAM: state {w, m, v}, fresh {init_w, init_s1, init_s2}. */
int kp_table_create(int device, uint64_t capacity, uint32_t dim, int rule, float init_w,
                    float init_s1, float init_s2, kp_table** out);
/* ~TieredStore */
int kp_table_destroy(kp_table* t);
/* TieredStore::cache_size (store.hpp:82) */
int kp_table_size(kp_table* t, uint64_t* n);
/* TieredStore::resolve, device batch form (store.cpp:153-168): insert-if-absent,
 * d_rows[i] = row of d_keys[i]. */
int kp_table_pull(kp_table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows, kp_stream s);
/* insert keys start + i*step (i < count) -- pre-populates a table shard with
 * a key range without host traffic (benchmarks at steady state) */
int kp_table_insert_range(kp_table* t, uint64_t start, uint64_t step, uint64_t count, kp_stream s);
/* lookup only; d_rows[i] = 0xFFFFFFFF when absent */
int kp_table_lookup(kp_table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows,
                    kp_stream s);
/* row snapshot (w, s1, s2 may be NULL): [n][dim] each */
int kp_table_gather(kp_table* t, const uint32_t* d_rows, uint32_t n, float* d_w, float* d_s1,
                    float* d_s2, kp_stream s);
/* overwrite row state from device buffers [n][dim] (NULL = keep) */
int kp_table_set_rows(kp_table* t, const uint32_t* d_rows, uint32_t n, const float* d_w,
                      const float* d_s1, const float* d_s2, kp_stream s);
/* adagrad_sparse_update (proj/src/optimizer.cpp:86-95) / sparse Adam applied in
 * place to rows with per-row gradients d_grads[n][dim]. */
int kp_table_apply(kp_table* t, const uint32_t* d_rows, const float* d_grads, uint32_t n,
                   float lr, float beta1, float beta2, kp_stream s);
/* TieredStore::pull_batch (store.hpp:56-60, store.cpp:176-189): keys ascending
 * and unique (a std::set), n >= 1 else KP_ERR_STORE "pull_batch: empty key set".
 * Inserts missing keys, makes them the working set, returns value snapshots
 * (host [n][dim] each; s1/s2 may be NULL). */
int kp_store_pull_batch(kp_table* t, const uint64_t* keys, uint32_t n, float* w, float* s1,
                        float* s2);
/* TieredStore::push_updates (store.hpp:62-65, store.cpp:191-208): keys
 * ascending; applies the rule to each key in order and fails with KP_ERR_STORE
 * ("push_updates: key K not in the current working set") at the first key
 * outside the last pull_batch working set, leaving earlier keys updated.
 * *applied = number of keys updated. */
int kp_store_push_updates(kp_table* t, const uint64_t* keys, const float* grads, uint32_t n,
                          float lr, float beta1, float beta2, uint32_t* applied);
/* TieredStore::lookup (store.cpp:210-218), copying the live row out */
int kp_store_lookup(kp_table* t, uint64_t key, float* w, float* s1, float* s2);
/* Every key with its state, ascending key (parity dumps; the reference
 * exposes this only through flush() + the cold files, store.cpp:238-245).
 * Pass keys == NULL to query *n_out. */
int kp_table_export(kp_table* t, uint64_t* keys, float* w, float* s1, float* s2, uint64_t cap,
                    uint64_t* n_out);

/* ------------------------------------------------------- dedup/shard ---
 * Working-set dedup (proj/src/trainer.cpp:121-124): d_unique[U] ascending
 * (std::set order, bit-exact), d_inverse[n] occurrence -> unique index,
 * d_seg[U+1] (nullable) segment starts in sorted order. */
int kp_dedup(const uint64_t* d_keys, uint32_t n, uint64_t* d_unique, uint32_t* d_inverse,
             uint32_t* d_seg, uint32_t* n_unique, kp_stream s);
/* Owner-side dedup of the G > 1 exchange: the keys are R runs (one per source
 * rank, run r = [run_off[r], run_off[r+1]), host array), each strictly
 * ascending. Same outputs as kp_dedup (the cross-worker sparse_sum key union of
 * proj/src/trainer.cpp:163,180-186, ties in source order), plus d_sorted_pos[p]
 * = input position of sorted position p (may be NULL). */
int kp_dedup_runs(const uint64_t* d_keys, uint32_t n, const uint64_t* run_off, uint32_t n_runs,
                  uint64_t* d_unique, uint32_t* d_inverse, uint32_t* d_seg, uint32_t* d_sorted_pos,
                  uint32_t* n_unique, kp_stream s);
/* Owner shard = key % G (proj/src/trainer.cpp:83): stable bucket of ascending
 * unique keys; d_perm[slot] = unique index, d_pos[unique] = slot, counts[G] host. */
int kp_shard(const uint64_t* d_unique, uint32_t n, uint32_t G, uint32_t* d_perm, uint32_t* d_pos,
             uint64_t* counts, kp_stream s);

/* ---------------------------------------------------- dense k-step Adam ---
 * proj/include/kpsim/optimizer.hpp:77-126, proj/src/optimizer.cpp:39-153.
 * All vectors fp32 device [D]; worker blocks are [W][D] contiguous. */
/* local_adam_step (optimizer.cpp:48-54) */
int kp_dense_local_step(float* d_x, float* d_m, float* d_v, const float* d_vbar, const float* d_g,
                        uint64_t D, float alpha, float beta1, float beta2, kp_stream s);
/* accumulate_moments (optimizer.cpp:39-46) */
int kp_dense_moments(float* d_m, float* d_v, const float* d_g, uint64_t D, float beta1,
                     float beta2, kp_stream s);
/* centered_mean_vectors (common.hpp:36-45) over n vectors at d_vecs + i*stride */
int kp_centered_mean(const float* d_vecs, uint64_t stride, uint32_t n, uint64_t D, float* d_out,
                     kp_stream s);
/* global_merge (optimizer.cpp:56-84) over W local worker states [W][D] and,
 * with a communicator, every rank's workers (ascending global worker order).
 * Moments must already be accumulated. */
int kp_kstep_merge(kp_comm* comm, float* d_x, float* d_m, float* d_v, float* d_vbar, uint32_t W,
                   uint64_t D, float alpha, int reset_local_v, kp_stream s);

/* -------------------------------------------------------------- AUC ---
 * compute_auc (proj/src/eval.cpp:8-39) on the device: rank-sum with tie
 * averaging over n (score, label) pairs; *auc = NaN when a class is absent,
 * KP_ERR for labels outside {0,1}. Bit-identical to the reference's loop on
 * the same scores (all partial sums are exact in f64). Synchronous. */
int kp_compute_auc(const float* d_scores, const int32_t* d_labels, uint32_t n, double* auc,
                   kp_stream s);

/* ------------------------------------------------------------- GEMM ---
 * C[M][N] = A[M][K] . B[N][K]^T in fp32 (the MLP's contraction, model.cpp:107-109).
 * engine 0 = auto (tcgen05 3xTF32 when the shapes allow TMA), 1 = SIMT fp32,
 * 2 = tcgen05 3xTF32 only (KP_ERR_CONFIG if unsupported), 3 = tcgen05 fp16
 * operands with per-row power-of-two scales (3xFP16, the first-layer path),
 * 4 = 3xFP16 on operands pre-split into fp16 planes (the planes-mode first
 * layer, kp_gemm_h3.cu), 5 = the same with the deterministic stream-K split,
 * 6 = whole tiles for the full waves and stream-K for the last partial wave. */
int kp_gemm_nt(const float* d_A, int lda, const float* d_B, int ldb, float* d_C, int ldc, int M,
               int N, int K, int engine, kp_stream s);
/* C[M][N] = A[K][M]^T . B[K][N] (the weight gradient dW = dZ^T X of
 * model.cpp:184-186, contracted over the minibatch); deterministic split-K. */
int kp_gemm_tn(const float* d_A, int lda, const float* d_B, int ldb, float* d_C, int ldc, int M,
               int N, int K, int engine, kp_stream s);

/* ------------------------------------------------------------- comm ---
 * One process per GPU; NCCL over NVLink/NVSwitch. The caller broadcasts the
 * 128-byte id from rank 0 (e.g. with torch.distributed) before kp_comm_init. */
int kp_comm_unique_id(uint8_t id[128]);
int kp_comm_init(const uint8_t id[128], int rank, int world, int device, kp_comm** out);
int kp_comm_destroy(kp_comm* c);
int kp_comm_rank(kp_comm* c, int* rank, int* world);

/* ---------------------------------------------------------- trainer ---
 * kpsim::Trainer (proj/include/kpsim/trainer.hpp:66-106): per batch, working
 * set dedup, pull (insert-if-absent), per-slot pooling, per-worker MLP
 * forward/backward, averaged sparse push, k-step Adam on the dense block.
 * Field names follow TrainerConfig / ModelConfig / AdamHyper. */
typedef struct kp_trainer_config {
  uint64_t seed;
  uint32_t n_workers;      /* N: all workers over all ranks */
  uint32_t local_workers;  /* workers on this rank (N = world * local_workers) */
  uint64_t minibatch_size;
  double sparse_lr;
  double alpha, beta1, beta2, epsilon; /* AdamHyper */
  uint64_t k;
  int32_t reset_local_v;
  uint32_t embedding_dim;
  uint32_t n_slots;        /* S >= 1; S = 1 is the reference model */
  uint32_t n_hidden;
  uint32_t hidden[8];
  int32_t activation;      /* 0 relu, 1 tanh */
  int32_t pooling;         /* 0 sum, 1 mean */
  int32_t sparse_rule;     /* KP_RULE_ADAGRAD | KP_RULE_ADAM */
  double sparse_beta1, sparse_beta2, sparse_eps;
  uint64_t table_capacity; /* rows held by this rank's table shard */
} kp_trainer_config;

typedef struct kp_batch_result {
  double loss;             /* BatchRecord::loss (mean of minibatch-step losses) */
  uint64_t minibatch_steps;
  uint64_t merges;
  uint64_t steps_total;
  uint64_t merges_total;
  /* predict_first only: online AUC of this batch and over every batch so far
   * (BatchRecord::auc / cumulative_auc, trainer.hpp:36-42), computed on the
   * device over the global batch; NaN when a class is absent */
  int32_t has_auc;
  double auc;
  double cumulative_auc;
} kp_batch_result;

int kp_trainer_create(const kp_trainer_config* cfg, kp_comm* comm, int device, kp_trainer** out);
int kp_trainer_destroy(kp_trainer* tr);
/* Trainer::train_batch / process_batch (trainer.cpp:115-259) for this rank's
 * contiguous slice [global_first, global_first + n) of a global batch of
 * global_n instances (the slice shard_batch assigns to this rank's workers).
 * HOST buffers: offs[n+1] (u32 CSR), keys[offs[n]], slots (NULL => S = 1),
 * labels[n]. predict_first = online_eval's predict-then-train; preds (host,
 * nullable) receives this slice's predictions. */
int kp_trainer_train_batch(kp_trainer* tr, const uint32_t* offs, const uint64_t* keys,
                           const uint16_t* slots, const int32_t* labels, uint32_t n,
                           uint64_t global_n, uint64_t global_first, int predict_first,
                           float* preds, kp_batch_result* out);
/* Same with the batch already resident in HBM (h_offs is the host copy of
 * d_offs, used for step bookkeeping). */
int kp_trainer_train_batch_device(kp_trainer* tr, const uint32_t* h_offs, const uint32_t* d_offs,
                                  const uint64_t* d_keys, const uint16_t* d_slots,
                                  const int32_t* d_labels, uint32_t n, uint64_t global_n,
                                  uint64_t global_first, int predict_first, float* preds,
                                  kp_batch_result* out);
/* Pipelined ingestion: stage a HOST batch (pinned memory for true overlap)
 * into one of two device buffer slots, then train on it. The async H2D (copy
 * stream) is issued once the running step has passed its last host readback
 * (or at train_staged of that slot), so staging batch i+1 right before
 * training batch i hides the copy behind batch i's compute. The host arrays
 * must stay valid and unmodified until train_staged(slot) returns. */
int kp_trainer_stage_batch(kp_trainer* tr, int slot, const uint32_t* offs, const uint64_t* keys,
                           const uint16_t* slots, const int32_t* labels, uint32_t n);
int kp_trainer_train_staged(kp_trainer* tr, int slot, uint64_t global_n, uint64_t global_first,
                            int predict_first, float* preds, kp_batch_result* out);
int kp_trainer_dense_dim(kp_trainer* tr, uint64_t* D);
/* KStepEngine::states()[w] (optimizer.hpp:118), host copies [D] */
int kp_trainer_worker_state(kp_trainer* tr, uint32_t local_worker, float* x, float* m, float* v,
                            float* vbar);
int kp_trainer_set_worker_state(kp_trainer* tr, uint32_t local_worker, const float* x,
                                const float* m, const float* v, const float* vbar);
/* KStepEngine::x_bar / Trainer::dense_model (optimizer.cpp:146-153) */
int kp_trainer_xbar(kp_trainer* tr, float* out);
/* borrowed handle of the trainer's table shard */
int kp_trainer_table(kp_trainer* tr, kp_table** out);
/* CUDA-event stage times on the trainer's stream accumulated since the last
 * call (ms): [0] dedup [1] pull [2] pool [3] mlp [4] push [5] dense
 * [6] exchange; counters: [0] steps [1] unique keys [2] occurrences
 * [3] owner-side unique keys [4] keys received (G > 1). Returns and resets. */
int kp_trainer_profile(kp_trainer* tr, int enable, double* stage_ms, uint64_t* counters);
int kp_trainer_stream(kp_trainer* tr, kp_stream* s);
/* Trainer::ledger (proj/include/kpsim/trainer.hpp:81, ledger.hpp:13-19) from
 * MEASURED traffic: bytes this rank sent over NVLink since creation and the
 * transmissions, indexed by TransferCategory: [0] gpu_pull (keys to remote
 * owners + their rows back), [1] gpu_push (per-key gradients to remote
 * owners), [2] dense_merge (the k-step merge's two rounds; one transmission
 * per worker per merge), [3] sparse_sync and [4] cold_tier_io (0: one node,
 * the sparse sync IS the push; no cold tier). All zero at G = 1. */
int kp_trainer_ledger(kp_trainer* tr, uint64_t bytes[5], uint64_t count[5]);
/* Trainer::dense_trajectory (trainer.hpp:82, recorded at trainer.cpp:215-227):
 * opt-in (per-step x_bar readback; with G > 1 a collective, so enable it on
 * every rank alike). */
int kp_trainer_record_trajectory(kp_trainer* tr, int enable);
/* StepRecord i (optimizer.hpp:55-63): step (1-based), merged, loss, a3
 * increment, x_bar[D], frozen v_bar[D] (any output may be NULL);
 * *n_steps = records so far. */
int kp_trainer_trajectory(kp_trainer* tr, uint64_t i, uint64_t* step, int* merged, double* loss,
                          double* a3, float* x_bar, float* v_bar, uint64_t* n_steps);

#ifdef __cplusplus
}
#endif
#endif /* KPSIM_B200_H */
