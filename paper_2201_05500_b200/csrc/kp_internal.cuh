// Internal (C++) interfaces between the kernel files; the C ABI in
// include/kpsim_b200.h is built on these.
#pragma once

#include <cuda_fp16.h>

#include <functional>
#include <vector>
#include "kp_common.cuh"

namespace kp {

// ------------------------------------------------------------- abort -----
// Peer-exchange timeout guard (G > 1). k_wait sets kAbortTimeout in the
// trainer's device check word when a peer's flag never arrives; every kernel
// that writes PERSISTENT state (table inserts and row updates, dense x/m/v/
// v_bar, the merge) reads the word at entry and returns without writing, so
// a timed-out step leaves the table and the dense state exactly as they were
// before the wait (stream order makes k_wait's store visible to every later
// kernel). g_abort is the word for the kernels launched on this host thread
// (nullptr: no guard, single GPU); set it with AbortScope.
// kAbortPlan: the single-GPU step ran without the dedup readback (pass plan
// from the previous batch's key span, U on the device only) and the batch's
// span outgrew the plan -- the same guard keeps every state write out and the
// host reruns the batch with the exact plan.
constexpr uint32_t kAbortTimeout = 16u;
constexpr uint32_t kAbortPlan = 32u;
// ledger categories (proj/include/kpsim/ledger.hpp TransferCategory)
enum LedgerCat : int { kLedPull = 0, kLedPush = 1, kLedDense = 2, kLedSparse = 3, kLedCold = 4 };
extern thread_local const uint32_t* g_abort;
struct AbortScope {
  explicit AbortScope(const uint32_t* p) { g_abort = p; }
  ~AbortScope() { g_abort = nullptr; }
};
__device__ __forceinline__ bool aborted(const uint32_t* a) {
  return a != nullptr && (*reinterpret_cast<const volatile uint32_t*>(a) & (kAbortTimeout | kAbortPlan));
}

// ------------------------------------------------------------- dedup ----
// Workspace for one dedup: sorted (key, occurrence) pairs, unique keys,
// inverse index and segment starts. All device memory, grown on demand.
struct DedupWs {
  DevBuf keys_a, keys_b, vals_a, vals_b;  // radix ping-pong
  DevBuf counts, totals, minmax, bcount, scalars;
  DevBuf unique, inverse, seg, mapped;
  // results of the last run (device pointers into the buffers above)
  const uint64_t* sorted_keys = nullptr;
  const uint32_t* sorted_vals = nullptr;  // occurrence index per sorted position
  uint64_t* d_unique = nullptr;           // [U] ascending
  uint32_t* d_inverse = nullptr;          // [n] occurrence -> unique index
  uint32_t* d_seg = nullptr;              // [U+1] segment starts in sorted order
  uint32_t* d_nunique = nullptr;          // device scalar U
  uint32_t* d_sorted_mapped = nullptr;    // occ_map[sorted_vals[p]] (when requested)
  uint32_t n = 0, n_unique = 0;
  int spec_bits = -1;  // key-span bits of the last call (planned passes of the next)
};

// Radix sort (stable) of (key, occurrence index) + unique + inverse + segment
// starts. Writes U to ws.n_unique (host; one sync) and ws.d_nunique.
// d_occ_map (optional): per-occurrence map materialised in sorted order
// (ws.d_sorted_mapped[p] = occ_map[sorted_vals[p]]), e.g. the bag of each occurrence.
// d_occ_ident (optional, device word): 0xFFFFFFFF when occ_map is the identity
// (one feature in every slot), which skips its random gather -- and the
// d_sorted_mapped write: the caller then uses sorted_vals (equal).
// d_abort (optional): no host sync when a pass plan exists (the previous
// call's key span): U stays on the device (ws.n_unique = kUnknownU) and a
// span that outgrows the plan sets kAbortPlan in *d_abort (the caller's
// state writes are guarded by it and it reruns the batch); returns whether
// it ran that way.
constexpr uint32_t kUnknownU = 0xFFFFFFFFu;
struct DedupWs;
// would dedup() of n keys with d_abort run without the readback?
bool dedup_async_ready(const DedupWs& ws, uint32_t n);
// expect_ident (0/1; -1 none): the caller's prediction of *d_occ_ident ==
// all-ones, checked on the device the same way.
bool dedup(const uint64_t* d_keys, uint32_t n, DedupWs& ws, cudaStream_t s,
           const uint32_t* d_occ_map = nullptr, const uint32_t* d_occ_ident = nullptr,
           uint32_t* d_abort = nullptr, int expect_ident = -1);
// dedup() of keys made of runs [run_off[i], run_off[i+1]), each strictly
// ascending: merge tree instead of the radix sort, identical outputs
// (readback false: no host sync, ws.n_unique = kUnknownU, U on the device)
void dedup_runs(const uint64_t* d_keys, uint32_t n, const std::vector<uint64_t>& run_off,
                DedupWs& ws, cudaStream_t s, bool readback = true);

// Stable bucket of ascending unique keys by owner = key % G.
// perm[i] = unique index placed at bucket slot i; pos[u] = slot of unique u;
// counts[G] on host -- or, with d_counts (h_counts null), as u64 on the
// device only, with no host sync (the trainer allgathers them first).
struct ShardWs {
  DevBuf bcount, scalars;
};
void shard(const uint64_t* d_unique, uint32_t n, uint32_t G, uint32_t* d_perm,
           uint32_t* d_pos, uint64_t* h_counts, ShardWs& ws, cudaStream_t s,
           uint64_t* d_counts = nullptr, const uint32_t* d_n = nullptr);
// out[0] = *d_pflag (0 when null), out[1] = err[0] | err[1] << 32 (the step's
// plan flag and error words, allgathered with the counts)
void pack_step_flags(const uint32_t* d_pflag, const uint32_t* d_err, uint64_t* d_out, cudaStream_t s);

// ------------------------------------------------------------- table ----
struct Table {
  int device = 0;
  uint64_t capacity = 0;  // max rows
  uint64_t nslots = 0;    // power of two, 8 slots per 128 B bucket line (keys + rows)
  uint32_t dim = 0;
  int rule = 0;  // 0 adagrad {w, acc}; 1 adam {w, m, v}
  float init_w = 0.f, init_s1 = 0.f, init_s2 = 0.f;
  uint8_t* d_lines = nullptr;  // [nslots / 8] x 128 B: 8 keys u64 + 8 rows u32 + pad
  uint64_t* d_row_key = nullptr;
  float* d_w = nullptr;
  float* d_s1 = nullptr;
  float* d_s2 = nullptr;
  uint32_t* d_epoch = nullptr;    // working-set stamp per row (TieredStore API)
  uint32_t* d_scalars = nullptr;  // [0]=rows used, [1]=row of key u64max, [2]=full flag, [3]=error idx
  uint32_t epoch = 0;
};
Table* table_create(int device, uint64_t capacity, uint32_t dim, int rule, float init_w,
                    float init_s1, float init_s2);
void table_destroy(Table* t);
// insert-if-absent; rows_out[i] = row of keys[i] (kNoRow if the table is full)
// (d_n: the key count on the device, n its upper bound)
void table_pull(Table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows_out,
                bool stamp_epoch, cudaStream_t s, const uint32_t* d_n = nullptr);
// lookup only; kNoRow when absent
void table_lookup(const Table* t, const uint64_t* d_keys, uint32_t n, uint32_t* d_rows_out,
                  cudaStream_t s);
uint64_t table_size(const Table* t, cudaStream_t s);
void table_check_full(const Table* t, cudaStream_t s);  // throws kErrTableFull
void table_export(const Table* t, uint64_t* d_keys_out, uint32_t* d_rows_out,
                  unsigned long long* d_cnt, cudaStream_t s);
void table_ws_check(const Table* t, const uint32_t* d_rows, uint32_t n, uint32_t* d_first_bad,
                    cudaStream_t s);
void table_apply(Table* t, const uint32_t* d_rows, const float* d_grads, uint32_t n, float lr,
                 float b1, float b2, cudaStream_t s);
void table_set_rows(Table* t, const uint32_t* d_rows, uint32_t n, const float* d_w,
                    const float* d_s1, const float* d_s2, cudaStream_t s);
void table_gather(const Table* t, const uint32_t* d_rows, uint32_t n, float* d_w, float* d_s1,
                  float* d_s2, cudaStream_t s);

// ----------------------------------------------------------- embedding ---
// bags: CSR over occurrences; bag b = instance*S + slot. d_err[0]: first bad
// occurrence (caller presets 0xFFFFFFFF); d_err[1]: 0xFFFFFFFF iff
// bag_of_occ[o] == o for every occurrence (set here).
// (d_abort: a bad slot id also sets kAbortPlan there -- the sync-free step
// keeps its state writes out and raises at the batch-end readback; maps =
// false: only the checks, for a batch predicted to hold one feature per slot
// -- its maps are the identity and nothing reads them)
void prepare_bags(const uint32_t* d_offs, uint32_t occ_base, const uint16_t* d_slots,
                  uint32_t n_inst, uint32_t S, uint32_t* d_bag_offs, uint32_t* d_bag_of_occ,
                  uint32_t* d_err, cudaStream_t s, uint32_t* d_abort = nullptr, bool maps = true);
// row_of_occ[o] = idx[inverse[o]]  (source row of every occurrence)
void compose(const uint32_t* d_idx, const uint32_t* d_inverse, uint32_t n, uint32_t* d_out,
             cudaStream_t s);
// pooled[bag][e] = sum_{o in bag} src[row_of_occ[o]][e]  (x 1/|bag| when mean);
// d_inst_max (optional): max |pooled| over each instance's S bags
void pool(const uint32_t* d_bag_offs, uint32_t n_bags, const uint32_t* d_row_of_occ,
          const float* d_src, uint32_t e, bool mean, float* d_pooled, float* d_inv_count,
          cudaStream_t s, float* d_inst_max = nullptr, uint32_t S = 1);
// Deterministic segmented reduce of coefficient-scaled upstream rows by
// unique key, times inv_n, then the sparse rule applied in place to the row.
struct SegWs {
  DevBuf partials, qsums, first;
};
// ---------------------------------------------------------- peer memory ----
// Destination map for kernels that write their output straight into the
// peers' exchange windows over NVLink (CUDA IPC mappings): local element i
// belongs to peer p with start[p] <= i < start[p+1] and lands at
// base[p] + (i - start[p]) * stride bytes (base already holds the offset of
// this rank's segment inside peer p's window).
constexpr int kMaxPeers = 16;
struct PeerMap {
  int R;
  uint32_t stride;
  uint32_t start[kMaxPeers + 1];
  uintptr_t base[kMaxPeers];
};
__device__ __forceinline__ char* peer_dst(const PeerMap& pm, uint32_t i) {
  int p = 0;
#pragma unroll 1
  while (p + 1 < pm.R && i >= pm.start[p + 1]) ++p;
  return reinterpret_cast<char*>(pm.base[p]) + (uint64_t)(i - pm.start[p]) * pm.stride;
}
struct PeerFlags {
  uintptr_t flag[kMaxPeers];  // &flags_p[phase][me] in every peer p's window
};
struct PeerVecs {
  uintptr_t src[kMaxPeers];  // rank p's [W][D] worker vectors
  uintptr_t dst[kMaxPeers];  // rank p's [D] result
};
// centered mean of elements [c0, c1) over all ranks' workers, into every rank
void peer_cmean(const PeerVecs& pv, int R, uint32_t W, uint64_t D, uint64_t c0, uint64_t c1,
                cudaStream_t s);
// The whole k-step merge of elements [c0, c1) in one pass over NVLink: v_bar =
// cmean(v), terms x - alpha*m/sqrt(v_bar) of every rank's workers, x = cmean(
// terms) -- stored into every rank's v_bar window and worker-0 x.
struct PeerMerge {
  uintptr_t v[kMaxPeers], x[kMaxPeers], m[kMaxPeers];  // rank p's [W][D] worker vectors
  uintptr_t vb[kMaxPeers];                             // rank p's [D] v_bar window
};
void peer_merge(const PeerMerge& pm, int R, uint32_t W, uint64_t D, uint64_t c0, uint64_t c1, float alpha,
                cudaStream_t s);
// keys[t] = unique[perm[t]] -> peer windows (the owner's received keys)
void peer_send_keys(const uint64_t* d_unique, const uint32_t* d_perm, uint32_t n, const PeerMap& pm,
                    cudaStream_t s);
// rows src[idx[i]] (e floats; kNoRow -> zeros) -> peer windows
void peer_send_rows(const float* d_src, const uint32_t* d_idx, uint32_t n, uint32_t e,
                    const PeerMap& pm, cudaStream_t s);
// after this stream's writes: flag_p = seq in every peer (system-scope release)
void peer_signal(const PeerFlags& f, int R, uint64_t seq, cudaStream_t s);
// wait until every peer's flag in this rank's window reached seq (bit 4 of
// *d_err on timeout instead of hanging)
void peer_wait(const uint64_t* d_my_flags, int R, uint64_t seq, uint32_t* d_err, cudaStream_t s);

struct SparseRule {
  int rule;  // 0 adagrad, 1 adam
  float lr, beta1, beta2;
};
// Segments are [seg[u], seg[u+1]) of sorted positions p; the upstream row of
// position p is rows_src[map(p)] with map(p) = bag_of_occ[sorted_vals[p]]
// (bag_of_occ may be null: identity; sorted_vals null: map(p) = p, rows
// already in sorted order). Output: apply the rule to table row
// table_rows[u] (fused push) when `t` is set, else store to grad_out[out_idx[u]]
// -- or, with `pm`, to peer_dst(pm, out_idx[u]) in the owners' windows.
// d_nunique: U on the device (n_unique is then only an upper bound).
void seg_reduce_apply(const uint32_t* d_seg, uint32_t n_unique, const uint32_t* d_sorted_vals,
                      const uint32_t* d_bag_of_occ, uint32_t n_pos, const float* d_rows_src,
                      uint32_t e, float inv_n, Table* t, const uint32_t* d_table_rows,
                      const SparseRule& r, float* d_grad_out, const uint32_t* d_out_idx,
                      SegWs& ws, cudaStream_t s, const PeerMap* pm = nullptr,
                      const uint32_t* d_nunique = nullptr);
void gather_rows(const float* d_src, const uint32_t* d_idx, uint32_t n, uint32_t e, float* d_out,
                 cudaStream_t s);

// --------------------------------------------------------------- GEMM ----
// epilogue: 0 store, 1 act(acc + bias[n]), 2 acc * act'(aux[m][n]),
//           3 acc * coeff[m*S + n/e] (mean-pooling coefficient)
struct GemmEpi {
  int mode;
  int act;
  const float* bias;
  const float* aux;
  int ld_aux;
  const float* coeff;
  uint32_t S, e;
  // fp16-operand GEMM (tc_gemm_nt_h): per-row max |A| and per-row exponent of B
  const float* a_rowmax = nullptr;
  const int* b_exp = nullptr;
  // (small-tile SIMT GEMM, one K split) column sums of each 32-row tile's
  // outputs -> csum_part[m-tile][N]: the next layer's bias gradient partials
  float* csum_part = nullptr;
};
// tcgen05 3xTF32 GEMMs (operands split hi/lo on the fly in shared memory)
bool tc_gemm_supported(int M, int N, int K, const float* A, int lda, const float* B, int ldb);
// C = epi(A[M][K] . B[N][K]^T)
void tc_gemm_nt(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
                int ldc, const GemmEpi& ep, cudaStream_t s);
void tc_gemm_nt_pre(int M, int N, int K, const float* A, int lda, const float* Bhi, const float* Blo,
                    int ldb, float* C, int ldc, const GemmEpi& ep, cudaStream_t s);
// C[z] = A[K][M]^T . B[K][N] over K split z (deterministic split-K partials); returns #splits
int tc_gemm_tn(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
               int ldc, int splits, cudaStream_t s);
int tc_splits(int M, int N, int K);
// fp16-operand GEMM ("3xFP16": A, B split into fp16 hi + lo after a per-row
// power-of-two scale; hi*hi + hi*lo + lo*hi at the f16 tensor rate). A is fp32
// K-major with a_rowmax[m] = max_k |A[m][k]|; B is pre-split by split_h.
void tc_gemm_nt_h(int M, int N, int K, const float* A, int lda, const float* a_rowmax,
                  const __half* Bhi, const __half* Blo, const int* b_exp, int ldb, float* C, int ldc,
                  const GemmEpi& ep, cudaStream_t s);
void split_h(const float* W, int N, int K, int ld, __half* hi, __half* lo, int* exps, cudaStream_t s);
void rowmax(const float* A, int M, int K, int lda, float* out, cudaStream_t s);
bool tc_h_enabled();  // KP_GEMM_F16=0 keeps every GEMM on 3xTF32
void split_hilo(const float* x, float* hi, float* lo, size_t n, cudaStream_t s);
bool tc_enabled();  // KP_GEMM=simt disables the tensor-core path
// leave `n` SMs free of persistent GEMM CTAs (for kernels overlapping the GEMM
// on another stream, e.g. NCCL); 0 = use every SM
void tc_reserve_sms(int n);
// C = A . B^T on the SIMT fp32 path (reference engine for the tensor-core path)
void simt_gemm_nt(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
                  int ldc, cudaStream_t s);
// C = A[K][M]^T . B[K][N] on the SIMT fp32 path
void simt_gemm_tn(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
                  int ldc, cudaStream_t s);
// out[i] = sum_z part[z][i] in z order
void reduce_splits(const float* part, int splits, size_t n, float* out, cudaStream_t s);

// 3xFP16 GEMM on pre-split fp16 operand planes (kp_gemm_h3.cu). An operand
// is hi/lo planes of x * 2^exp[row] (exp nullable = 0), ld in halves.
struct H3Operand {
  const __half* hi;
  const __half* lo;
  const int* exp;
  int ld;
};
bool h3_enabled();  // KP_GEMM_H3=0 keeps layer 1 on the on-chip-split kernels
bool h3_supported(int M, int N, int K, const H3Operand& A, const H3Operand& B);
// C[m][n] = epi(2^-(ea[m]+eb[n]) sum_k A(m,k) B(n,k)); a_mn / b_mn: operand
// stored [K][rows] (MN-major) instead of [rows][K]. splitk: 0 data-parallel
// tiles; 1 deterministic stream-K over all tiles' K ranges into `ws`
// (h3_splitk_ws_floats) + fix-up; 2 whole tiles for the full waves of the
// GPU's pairs and stream-K for the last partial wave. Stream-K: epilogue
// modes 0 and 1 (applied by the fix-up), the split depends only on the shape.
// keep: operands re-read across tiles (bit 0 A, bit 1 B) load with an L2
// evict_last policy, the others evict_first
// Gathered A (one feature per slot): A[m][slot*e + j] = src[rowocc[m*S + slot]][j],
// fetched by TMA gather4 and split into planes on chip with the row exponents
// A.exp; with `store` the planes also go to A.hi / A.lo (for a later GEMM).
struct H3Gather {
  const float* src;
  uint64_t nrows;
  const uint32_t* rowocc;
  uint32_t S, e;
  bool store;
};
void h3_gemm(const H3Operand& A, bool a_mn, const H3Operand& B, bool b_mn, int M, int N, int K, float* C,
             int ldc, const GemmEpi& ep, int splitk, float* ws, cudaStream_t s, int keep = 3,
             const H3Gather* ga = nullptr);
size_t h3_splitk_ws_floats(int M, int N, bool tail_only = false);
void h3_reserve_sms(int n);
// planes of W^T ([K][N], one exponent per row of W^T) from W [N][K], N <= 256
void split_t_h(const float* W, int N, int K, __half* hi, __half* lo, int* exps, cudaStream_t s);
// planes of each row of X [rows][K] with its own exponent (one warp per row)
void split_rows_h(const float* X, int rows, int K, int ld, __half* hi, __half* lo, int* exps, cudaStream_t s);
// planes of D[b][n] = dz[b][n] * 2^-xe[b] with one exponent per column n
// colsum_out (optional): the plain column sums of dz (a bias gradient) from the
// same read, via colsum_ws (split_cols_colsum_ws_floats)
void split_cols_scaled_h(const float* dz, int B, int N, const int* xe, unsigned* cmax_ws, __half* hi,
                         __half* lo, int* exps, cudaStream_t s, float* colsum_out = nullptr,
                         float* colsum_ws = nullptr);
size_t split_cols_colsum_ws_floats(int B, int N);
// split_rows_h(dz) + the column pass of split_cols_scaled_h from one read of
// dz (N % 128 == 0, N <= 1024; KP_SPLIT_FUSE=0: off), then the planes (and the
// colsum reduction) after: bit for bit the unfused pair
bool rows_colmax_fusable(int N);
void split_rows_colmax_h(const float* dz, int B, int N, const int* xe, unsigned* cmax_ws, __half* rhi,
                         __half* rlo, int* rexps, float* colsum_ws, cudaStream_t s);
void split_cols_after_h(const float* dz, int B, int N, const int* xe, const unsigned* cmax_ws, __half* hi, __half* lo,
                        int* exps, float* colsum_out, const float* colsum_ws, cudaStream_t s);
// pooling written as the first layer's planes (see kp_embed.cu k_pool_planes)
bool pool_planes_supported(uint32_t S, uint32_t e);
void pool_planes(const uint32_t* d_bag_offs, uint32_t n_inst, uint32_t S, const uint32_t* d_row_of_occ,
                 const float* d_src, uint32_t e, bool mean, __half* d_hi, __half* d_lo, int* d_inst_exp,
                 float* d_inv_count, cudaStream_t s, bool ident = false,
                 const uint32_t* d_inverse = nullptr);
// (d_inverse set: d_row_of_occ is the unique -> row map, row of occurrence o
// = d_row_of_occ[d_inverse[o]]; one feature per slot with planes_ident_kernel)
bool planes_ident_kernel(uint32_t S, uint32_t e);
// One feature per slot, pooling fused into the first layer (the forward GEMM
// gathers the rows itself): only the per-instance exponents of the planes the
// pooling kernel would write -- row_exp(max over the instance's S rows of
// max |x|), from one max per unique key -- and the mean coefficients (1).
void inst_exps_ident(const float* d_src, const uint32_t* d_idx, uint32_t U, uint32_t e,
                     const uint32_t* d_inverse, uint32_t n_inst, uint32_t S, float* d_umax_ws,
                     int* d_inst_exp, float* d_inv_count, bool mean, cudaStream_t s);

// is an M x N x K product big enough for the tcgen05 kernels (else the SIMT one)
bool tc_worth(int M, int N, int K, double min_flop);

// ---------------------------------------------------------------- MLP ----
struct MlpShape {
  uint32_t n_layers = 0;          // hidden + 1
  uint32_t widths[10] = {0};      // in, hidden..., 1
  uint64_t w_off[9] = {0}, b_off[9] = {0};
  uint64_t D = 0;
  int activation = 0;             // 0 relu, 1 tanh
};
struct MlpWs {
  DevBuf act[9];    // per hidden layer activations [B][width]
  DevBuf dz[2];     // ping-pong upstream grads
  DevBuf logits, delta, partials, lossp, whi, wlo, wt, wthi, wtlo;
  // fp16-operand first layer: split weights (+ exponents) and row maxima
  DevBuf hhi, hlo, hexp, thi, tlo, texp, amax;
  const float* in_rowmax = nullptr;  // max |input row| from the producer (pool), else computed
  // first-layer input as fp16 planes from the pooling kernel (3xFP16 GEMMs on
  // pre-split operands); null: fp32 input
  const __half* in_hi = nullptr;
  const __half* in_lo = nullptr;
  const int* in_exp = nullptr;
  DevBuf dzh, dzl, dze, dwh, dwl, dwe, cmax, skws;  // layer-1 backward planes, stream-K partials
  DevBuf hdone;  // head backward's last-block counter (the loss finalize)
  DevBuf cpart;  // bias-gradient partials from a small-tile dX epilogue
  // planes mode, one feature per slot: the forward gathers its input rows
  // (row of (b, slot) = ga_rowocc[b*S + slot] of ga_src [ga_nrows][e]) and
  // writes the planes at in_hi / in_lo for the weight gradient
  // products below this many flops run on the small-tile SIMT kernel
  // (KP_TC_MIN_MFLOP at trainer creation; 512 MFLOP: configs[0] is all SIMT)
  double tc_min_flop = 512e6;
  const float* ga_src = nullptr;
  uint64_t ga_nrows = 0;
  const uint32_t* ga_rowocc = nullptr;
  uint32_t ga_S = 0, ga_e = 0;
};
// Forward over B instances (input [B][in]); writes preds (sigmoid) and
// logits; keeps activations in ws for backward.
void mlp_forward(const MlpShape& m, const float* d_x, const float* d_in, uint32_t B,
                 float* d_preds, MlpWs& ws, cudaStream_t s);
// Backward: d_grad[D] (overwritten), d_dinput[B][in] scaled by d_coeff
// (per bag; null = 1), loss sum (f64, device) accumulated into d_loss.
// `after_dinput` (optional) runs right after d_dinput is enqueued and before
// the first layer's weight gradient, so a caller can start consuming it
// (e.g. the gradient exchange) while the last GEMM runs.
void mlp_backward(const MlpShape& m, const float* d_x, const float* d_in, uint32_t B,
                  const float* d_preds, const int32_t* d_labels, float* d_grad, float* d_dinput, const float* d_coeff,
                  uint32_t S, uint32_t e, double* d_loss_sum, MlpWs& ws, cudaStream_t s,
                  const std::function<void()>* after_dinput = nullptr);

// -------------------------------------------------------------- dense ----
struct AdamParams {
  float alpha, beta1, beta2;
};
void dense_local_step(float* x, float* m, float* v, const float* vbar, const float* g, uint64_t D,
                      const AdamParams& h, cudaStream_t s);
void dense_moments(float* m, float* v, const float* g, uint64_t D, const AdamParams& h,
                   cudaStream_t s);
// out[j] = centered mean over n vectors at vecs + i*stride (ascending i)
void centered_mean(const float* vecs, uint64_t stride, uint32_t n, uint64_t D, float* out,
                   cudaStream_t s);
// local merge of a single worker (W = 1, one rank), fused; bitwise the general path
void merge_single(float* x, const float* m, float* v, float* vbar, uint64_t D, float alpha,
                  bool reset, cudaStream_t s);
void merge_terms(const float* x, const float* m, const float* vbar, uint64_t D, float alpha,
                 float* out, cudaStream_t s);
void dense_check(const float* v, const float* vbar, const float* x, uint64_t D, uint32_t* d_flag,
                 cudaStream_t s, uint32_t* d_done = nullptr);
// one worker on one GPU: moments + local step or merge + checks in one pass
// (bitwise the separate kernels' results)
void dense_step_single(float* x, float* m, float* v, float* vbar, const float* g, uint64_t D, const AdamParams& h,
                       bool merge, bool reset, uint32_t* d_flag, uint32_t* d_done, cudaStream_t s);
// dst = src (D floats), skipped when the step was aborted (g_abort)
void dense_copy(float* dst, const float* src, uint64_t D, cudaStream_t s);

// ---------------------------------------------------------------- AUC ----
struct AucWs {
  DevBuf keys, part, part2, bad;
  DedupWs dd;
};
// rank-sum AUC with tie averaging over n (score, label) pairs; NaN when a
// class is absent (proj/src/eval.cpp:8-39). Synchronises the stream.
double device_auc(const float* d_scores, const int32_t* d_labels, uint32_t n, AucWs& ws,
                  cudaStream_t s);

// init_dense (proj/src/model.cpp:68-74): mt19937_64 + libstdc++ uniform(-0.05,0.05)
void init_dense_host(uint64_t seed, uint64_t dim, double* out);
uint64_t splitmix64_host(uint64_t x);

}  // namespace kp
