// C++ host shim over the C ABI (include/kpsim_b200.h) that keeps the
// reference's class and function names (namespace kpsim -> kpsim_b200):
//   TieredStore        proj/include/kpsim/store.hpp:47-97
//   AdamHyper, WorkerState, accumulate_moments, local_adam_step,
//   global_merge, adagrad_sparse_update, KStepEngine
//                      proj/include/kpsim/optimizer.hpp:15-126
//   Trainer            proj/include/kpsim/trainer.hpp:66-106
//   compute_auc        proj/include/kpsim/eval.hpp:13-27 (host parity metric)
// Errors are rethrown with the reference's types and messages.
// Values cross the API as double (reference signatures); the device computes
// in fp32 (the stated tolerance).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "kpsim_b200.h"

namespace kpsim_b200 {

using ParameterKey = std::uint64_t;

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
class ConfigError : public Error {
 public:
  explicit ConfigError(const std::string& w) : Error(w) {}
};
class StoreError : public Error {
 public:
  explicit StoreError(const std::string& w) : Error(w) {}
};
class DeviceError : public Error {
 public:
  explicit DeviceError(const std::string& w) : Error(w) {}
};

// status code from the C ABI -> exception of the reference's type
void check(int status);

// ------------------------------------------------------------ optimizer --
struct AdamHyper {
  double alpha = 0.01;
  double beta1 = 0.0;
  double beta2 = 0.999;
  double epsilon = 0.01;
  std::uint64_t k = 1;
  bool reset_local_v = true;
  void validate() const;
};

struct WorkerState {
  std::vector<double> x, m, v, v_bar;
  std::uint64_t t = 0;
  static WorkerState init(std::span<const double> x0, double epsilon);
  std::size_t dim() const { return x.size(); }
};

void accumulate_moments(WorkerState& s, std::span<const double> g, const AdamHyper& h);
void local_adam_step(WorkerState& s, std::span<const double> g, const AdamHyper& h);
void global_merge(std::vector<WorkerState>& states, const AdamHyper& h);
void adagrad_sparse_update(std::span<double> weight, std::span<double> accumulator,
                           std::span<const double> g, double lr);

// Device-resident engine: N worker states in HBM, one synchronized step from
// per-worker host gradients (KStepEngine, optimizer.hpp:103-126).
class KStepEngine {
 public:
  KStepEngine(const AdamHyper& h, std::size_t n_workers, std::span<const double> x0,
              int device = 0);
  ~KStepEngine();
  KStepEngine(const KStepEngine&) = delete;
  KStepEngine& operator=(const KStepEngine&) = delete;
  struct StepInfo {
    bool merged = false;
    double a3_increment = 0.0;
  };
  StepInfo step(std::span<const std::vector<double>> gradients);
  std::uint64_t completed_steps() const { return t_; }
  std::size_t workers() const { return n_; }
  std::size_t dim() const { return d_; }
  std::vector<WorkerState> states() const;
  std::vector<double> frozen_v() const;
  std::vector<double> x_bar() const;

 private:
  AdamHyper h_;
  std::size_t n_, d_;
  std::uint64_t t_ = 0;
  float *x_ = nullptr, *m_ = nullptr, *v_ = nullptr, *vbar_ = nullptr, *g_ = nullptr,
        *tmp_ = nullptr;
};

// --------------------------------------------------------------- store --
struct TierConfig {
  std::size_t cache_capacity = 1;
  std::string cold_path;
  std::size_t hbm_capacity = 0;  // table rows; 0 = max(cache_capacity, 1<<20)
  int device = 0;
};

struct EmbeddingEntry {
  std::vector<double> weights;
  std::vector<double> adagrad_acc;
  std::uint64_t access_count = 0;
  std::uint64_t last_access = 0;
};

class TieredStore {
 public:
  static constexpr double kFreshAccumulator = 1e-6;
  TieredStore(TierConfig config, std::size_t embedding_dim);
  ~TieredStore();
  TieredStore(const TieredStore&) = delete;
  TieredStore& operator=(const TieredStore&) = delete;

  std::map<ParameterKey, EmbeddingEntry> pull_batch(const std::set<ParameterKey>& keys);
  void push_updates(const std::map<ParameterKey, std::vector<double>>& updates, double lr);
  EmbeddingEntry lookup(ParameterKey key) const;
  // HBM-resident table: there is no cold tier to evict to.
  std::size_t evict() { return 0; }
  // Writes every row in the reference's cold-file format (store.cpp:18-22):
  // <cold_path>/cold.dat "KPSC" v1 records, cold.idx "KPSI" v1 (key, offset).
  void flush();
  std::size_t cache_size() const;
  std::size_t embedding_dim() const { return dim_; }
  std::size_t capacity() const { return capacity_; }
  int device() const { return config_.device; }

  // ascending keys + rows (w, acc), for parity dumps
  void export_all(std::vector<ParameterKey>& keys, std::vector<float>& w,
                  std::vector<float>& acc) const;
  kp_table* handle() const { return t_; }
  // rebinds this store to a trainer-owned table (Trainer ctor)
  void bind(kp_table* t);

 private:
  TierConfig config_;
  std::size_t dim_;
  std::size_t capacity_;
  kp_table* t_ = nullptr;
  bool owned_ = true;
};

// ------------------------------------------------------------- trainer --
struct ModelConfig {
  std::uint64_t vocab = 10000;
  std::size_t embedding_dim = 8;
  std::vector<std::size_t> hidden = {16};
  std::string activation = "relu";  // relu | tanh
  std::string pooling = "sum";      // sum | mean
  std::size_t n_slots = 1;          // B200 extension: per-slot pooling (1 = reference)
};

struct TrainerConfig {
  std::uint64_t seed = 42;
  std::size_t n_workers = 4;
  std::uint64_t minibatch_size = 128;
  double sparse_lr = 0.05;
  AdamHyper adam;
  ModelConfig model;
  std::string sparse_rule = "adagrad";  // adagrad (reference) | adam
  double sparse_beta1 = 0.9, sparse_beta2 = 0.999, sparse_eps = 1e-8;
};

struct Instance {
  std::vector<ParameterKey> feature_ids;
  int label = 0;
  std::vector<std::uint16_t> slots;  // empty => slot 0
};
struct Batch {
  std::vector<Instance> instances;
  std::uint64_t id = 0;
};

// Replayable dataset file, one instance per line "label<TAB>id,id,..."
// (proj/include/kpsim/data.hpp:45-51, proj/src/data.cpp:59-124): same
// parsing rules and error messages as the reference.
std::vector<Instance> read_instances(const std::string& path);
void write_instances(const std::string& path, const std::vector<Instance>& instances);
std::vector<Batch> make_batches(std::vector<Instance> instances, std::uint64_t batch_size);
// read_instances straight into the CSR layout the trainer consumes:
// offs[n+1], keys[offs[n]] (each instance's ids ascending, deduped), labels[n]
void read_instances_csr(const std::string& path, std::vector<std::uint32_t>& offs,
                        std::vector<ParameterKey>& keys, std::vector<std::int32_t>& labels);

// ------------------------------------------------------------- ledger --
// proj/include/kpsim/ledger.hpp:13-68, filled from MEASURED traffic (bytes
// this rank sent over NVLink, kp_trainer_ledger) instead of a cost model.
enum class TransferCategory : std::uint8_t { GpuPull, GpuPush, DenseMerge, SparseSync, ColdTierIo };
const char* to_string(TransferCategory c);
struct CategoryTotals {
  std::uint64_t bytes = 0;
  std::uint64_t count = 0;
};
struct KStepRatios {
  double dense_bytes = 0.0;  // DenseMerge bytes, k-step over baseline
  double total_bytes = 0.0;  // all bytes, k-step over baseline
};
struct LedgerReport {
  std::map<TransferCategory, CategoryTotals> categories;
  CategoryTotals total;
  std::uint64_t bytes(TransferCategory c) const;
};
// kstep_ratio (proj/src/ledger.cpp:132-145); throws Error on a zero-byte baseline
KStepRatios kstep_ratio(const LedgerReport& kstep, const LedgerReport& baseline);

// ------------------------------------------------------- trajectory ----
struct StepRecord {  // proj/include/kpsim/optimizer.hpp:55-63
  std::uint64_t step = 0;
  bool merged = false;
  double loss = 0.0;
  double a3_increment = 0.0;
  std::vector<double> x_bar, v_bar;
};
struct Trajectory {
  std::size_t dim = 0, workers = 0;
  std::vector<StepRecord> steps;
};

struct BatchRecord {
  std::uint64_t batch = 0;
  std::size_t instances = 0;
  double loss = 0.0;
  std::optional<double> auc;
  std::optional<double> cumulative_auc;
};

struct TrainMetrics {
  std::vector<BatchRecord> batches;
  std::optional<double> cumulative_auc;
  std::uint64_t minibatch_steps = 0;
  std::uint64_t merge_events = 0;
};

std::optional<double> compute_auc(std::span<const double> scores, std::span<const int> labels);

class AucAccumulator {
 public:
  void add(std::span<const double> scores, std::span<const int> labels);
  std::optional<double> value() const;
  std::size_t size() const { return scores_.size(); }

 private:
  std::vector<double> scores_;
  std::vector<int> labels_;
};

// Per-batch result of the CSR entry point.
struct CsrResult {
  double loss = 0.0;
  std::uint64_t minibatch_steps = 0, merges = 0;
  std::vector<float> preds;  // predict_first only
  std::optional<double> auc, cumulative_auc;  // predict_first only (device AUC)
};

class Trainer {
 public:
  // comm == nullptr: single process (all n_workers on this GPU).
  Trainer(const TrainerConfig& config, TieredStore& store, const void* topology = nullptr,
          kp_comm* comm = nullptr);
  ~Trainer();
  Trainer(const Trainer&) = delete;
  Trainer& operator=(const Trainer&) = delete;

  BatchRecord train_batch(const Batch& b);
  TrainMetrics online_eval(std::span<const Batch> stream);

  // CSR form (this rank's slice of a global batch)
  CsrResult train_csr(const std::uint32_t* offs, const ParameterKey* keys,
                      const std::uint16_t* slots, const std::int32_t* labels, std::uint32_t n,
                      std::uint64_t global_n, std::uint64_t global_first, bool predict_first);
  CsrResult train_csr_device(const std::uint32_t* h_offs, const std::uint32_t* d_offs,
                             const ParameterKey* d_keys, const std::uint16_t* d_slots,
                             const std::int32_t* d_labels, std::uint32_t n,
                             std::uint64_t global_n, std::uint64_t global_first,
                             bool predict_first);

  const TrainMetrics& metrics() const { return metrics_; }
  std::vector<double> dense_model() const;  // x_bar
  std::vector<WorkerState> worker_states() const;
  void set_worker_state(std::size_t local_worker, const WorkerState& s);
  std::size_t dense_dim() const { return D_; }
  std::size_t local_workers() const { return W_; }
  std::uint64_t completed_steps() const { return steps_; }
  kp_trainer* handle() const { return tr_; }
  // Trainer::ledger (trainer.hpp:81): measured bytes per category
  LedgerReport ledger() const;
  // Trainer::dense_trajectory (trainer.hpp:82); recording is opt-in
  // (record_trajectory(true) before training; collective when G > 1)
  void record_trajectory(bool on);
  Trajectory dense_trajectory() const;
  int rank() const { return rank_; }
  int world() const { return world_; }

 private:
  BatchRecord process(const Batch& b, bool predict_first);
  TrainerConfig config_;
  TieredStore& store_;
  kp_trainer* tr_ = nullptr;
  std::size_t D_ = 0, W_ = 1;
  int rank_ = 0, world_ = 1;
  std::uint64_t steps_ = 0;
  TrainMetrics metrics_;
  AucAccumulator cumulative_;
};

}  // namespace kpsim_b200
