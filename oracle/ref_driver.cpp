// TEST INFRASTRUCTURE ONLY (oracle/): a C-ABI driver around the UNMODIFIED
// reference library compiled from /root/reference/proj/src by oracle/Makefile.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load it. It is the checker, never the product.
//
// The reference has no key-enumeration API and no Trainer binding
// (SURVEY.md §8c), so this driver owns a kpsim::TieredStore + kpsim::Trainer,
// feeds CSR batches through Trainer::train_batch / online_eval
// (proj/src/trainer.cpp:219-221,369-373), and dumps the dense worker states
// (KStepEngine::states, proj/include/kpsim/optimizer.hpp:118) and the full
// table (TieredStore::pull_batch over every key ever seen,
// proj/src/store.cpp:176-189 -- values are not modified by a pull).
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "kpsim/data.hpp"
#include "kpsim/eval.hpp"
#include "kpsim/model.hpp"
#include "kpsim/optimizer.hpp"
#include "kpsim/store.hpp"
#include "kpsim/trainer.hpp"

using namespace kpsim;

namespace {
thread_local std::string g_err;

struct RefTrainer {
  std::unique_ptr<TieredStore> store;
  std::unique_ptr<Trainer> trainer;
  std::set<ParameterKey> seen;
  std::size_t dim = 0;
};

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Batch make_batch(const uint64_t* offs, const uint64_t* keys, const int32_t* labels,
                 uint64_t n, uint64_t id) {
  Batch b;
  b.id = id;
  b.instances.resize(n);
  for (uint64_t i = 0; i < n; ++i) {
    // read_instances semantics (proj/src/data.cpp:153-168): ids deduped+sorted
    std::set<ParameterKey> s(keys + offs[i], keys + offs[i + 1]);
    b.instances[i].feature_ids.assign(s.begin(), s.end());
    b.instances[i].label = labels[i];
  }
  return b;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_trainer_create(const char* cold_dir, uint64_t seed, uint64_t n_workers,
                         uint64_t minibatch, double sparse_lr, double alpha,
                         double beta1, double beta2, double eps, uint64_t k,
                         int reset_v, uint64_t emb_dim, const uint64_t* hidden,
                         int n_hidden, int activation, int pooling,
                         uint64_t vocab) {
  RefTrainer* t = nullptr;
  int rc = guard([&] {
    auto r = std::make_unique<RefTrainer>();
    TierConfig tier;
    tier.cache_capacity = std::size_t(1) << 40;  // never evict (HBM-resident)
    tier.cold_path = cold_dir;
    r->store = std::make_unique<TieredStore>(tier, emb_dim);
    TrainerConfig c;
    c.seed = seed;
    c.n_workers = n_workers;
    c.minibatch_size = minibatch;
    c.sparse_lr = sparse_lr;
    c.adam.alpha = alpha;
    c.adam.beta1 = beta1;
    c.adam.beta2 = beta2;
    c.adam.epsilon = eps;
    c.adam.k = k;
    c.adam.reset_local_v = reset_v != 0;
    c.model.vocab = vocab;
    c.model.embedding_dim = emb_dim;
    c.model.hidden.assign(hidden, hidden + n_hidden);
    c.model.activation = activation ? Activation::Tanh : Activation::Relu;
    c.model.pooling = pooling ? Pooling::Mean : Pooling::Sum;
    r->dim = emb_dim;
    r->trainer = std::make_unique<Trainer>(c, *r->store, nullptr);
    t = r.release();
  });
  return rc == 0 ? t : nullptr;
}

void ref_trainer_destroy(void* h) { delete static_cast<RefTrainer*>(h); }

// One batch through Trainer::train_batch (predict_first=0) or
// Trainer::online_eval (predict_first=1). auc outputs are NaN when undefined.
int ref_trainer_batch(void* h, const uint64_t* offs, const uint64_t* keys,
                      const int32_t* labels, uint64_t n, uint64_t batch_id,
                      int predict_first, double* loss, double* auc,
                      double* cum_auc) {
  auto* t = static_cast<RefTrainer*>(h);
  return guard([&] {
    Batch b = make_batch(offs, keys, labels, n, batch_id);
    for (const auto& inst : b.instances)
      t->seen.insert(inst.feature_ids.begin(), inst.feature_ids.end());
    const double nan = std::nan("");
    if (predict_first) {
      std::vector<Batch> one{std::move(b)};
      t->trainer->online_eval(one);
      const auto& rec = t->trainer->metrics().batches.back();
      *loss = rec.loss;
      *auc = rec.auc ? *rec.auc : nan;
      *cum_auc = rec.cumulative_auc ? *rec.cumulative_auc : nan;
    } else {
      const auto rec = t->trainer->train_batch(b);
      *loss = rec.loss;
      *auc = nan;
      *cum_auc = nan;
    }
  });
}

uint64_t ref_trainer_dense_dim(void* h) {
  return static_cast<RefTrainer*>(h)->trainer->engine().dim();
}
uint64_t ref_trainer_steps(void* h) {
  return static_cast<RefTrainer*>(h)->trainer->engine().completed_steps();
}
uint64_t ref_trainer_merges(void* h) {
  return static_cast<RefTrainer*>(h)->trainer->metrics().merge_events;
}

int ref_trainer_worker_state(void* h, uint64_t worker, double* x, double* m,
                             double* v, double* vbar) {
  auto* t = static_cast<RefTrainer*>(h);
  return guard([&] {
    const auto& s = t->trainer->engine().states().at(worker);
    std::memcpy(x, s.x.data(), s.x.size() * 8);
    std::memcpy(m, s.m.data(), s.m.size() * 8);
    std::memcpy(v, s.v.data(), s.v.size() * 8);
    std::memcpy(vbar, s.v_bar.data(), s.v_bar.size() * 8);
  });
}

int ref_trainer_xbar(void* h, double* out) {
  auto* t = static_cast<RefTrainer*>(h);
  return guard([&] {
    const auto xb = t->trainer->dense_model();
    std::memcpy(out, xb.data(), xb.size() * 8);
  });
}

// per-step dense trajectory (x_bar, v_bar) recorded by Trainer::process_batch
// (proj/src/trainer.cpp:325-335)
int ref_trainer_trajectory(void* h, uint64_t step, double* xbar, double* vbar,
                           double* loss) {
  auto* t = static_cast<RefTrainer*>(h);
  return guard([&] {
    const auto& s = t->trainer->dense_trajectory().steps.at(step);
    std::memcpy(xbar, s.x_bar.data(), s.x_bar.size() * 8);
    std::memcpy(vbar, s.v_bar.data(), s.v_bar.size() * 8);
    *loss = s.loss;
  });
}

// the same StepRecord's merged flag and a3 increment (optimizer.hpp:55-63)
int ref_trainer_trajectory_flags(void* h, uint64_t step, int* merged, double* a3,
                                 uint64_t* n_steps) {
  auto* t = static_cast<RefTrainer*>(h);
  return guard([&] {
    const auto& steps = t->trainer->dense_trajectory().steps;
    *n_steps = steps.size();
    if (step >= steps.size()) return;
    *merged = steps[step].merged ? 1 : 0;
    *a3 = steps[step].a3_increment;
  });
}

uint64_t ref_trainer_table_size(void* h) {
  return static_cast<RefTrainer*>(h)->store->cache_size();
}

// every key ever pulled, ascending, with its weights and accumulators
int ref_trainer_table(void* h, uint64_t* keys, double* w, double* acc) {
  auto* t = static_cast<RefTrainer*>(h);
  return guard([&] {
    if (t->seen.empty()) return;
    const auto snap = t->store->pull_batch(t->seen);
    std::size_t i = 0;
    for (const auto& [key, e] : snap) {
      keys[i] = key;
      std::memcpy(w + i * t->dim, e.weights.data(), t->dim * 8);
      std::memcpy(acc + i * t->dim, e.adagrad_acc.data(), t->dim * 8);
      ++i;
    }
  });
}

// x0 = CtrModel::init_dense(seed) (proj/src/model.cpp:68-74)
int ref_init_dense(uint64_t emb_dim, const uint64_t* hidden, int n_hidden,
                   uint64_t seed, double* out, uint64_t* dim_out) {
  return guard([&] {
    ModelConfig c;
    c.embedding_dim = emb_dim;
    c.hidden.assign(hidden, hidden + n_hidden);
    CtrModel m(c);
    const auto x = m.init_dense(seed);
    *dim_out = x.size();
    if (out) std::memcpy(out, x.data(), x.size() * 8);
  });
}

// working-set dedup exactly as Trainer::process_batch builds it
// (proj/src/trainer.cpp:121-124): std::set insert over every occurrence.
uint64_t ref_dedup(const uint64_t* keys, uint64_t n, uint64_t* unique_out) {
  std::set<ParameterKey> s(keys, keys + n);
  uint64_t i = 0;
  for (auto k : s) unique_out[i++] = k;
  return i;
}

// AdaGrad rule (proj/src/optimizer.cpp:86-95)
int ref_adagrad(double* w, double* acc, const double* g, uint64_t n, double lr) {
  return guard([&] {
    adagrad_sparse_update(std::span<double>(w, n), std::span<double>(acc, n),
                          std::span<const double>(g, n), lr);
  });
}

// KStepEngine over N workers with caller-provided gradients
// (proj/src/optimizer.cpp:102-144). grads: [steps][workers][dim]. Outputs
// per step per worker x,m,v and frozen v_bar: [steps][workers][dim].
int ref_kstep(double alpha, double beta1, double beta2, double eps, uint64_t k,
              int reset_v, uint64_t workers, uint64_t dim, const double* x0,
              uint64_t steps, const double* grads, double* xs, double* ms,
              double* vs, double* vbars, int32_t* merged) {
  return guard([&] {
    AdamHyper h;
    h.alpha = alpha;
    h.beta1 = beta1;
    h.beta2 = beta2;
    h.epsilon = eps;
    h.k = k;
    h.reset_local_v = reset_v != 0;
    KStepEngine e(h, workers, std::span<const double>(x0, dim));
    std::vector<std::vector<double>> g(workers, std::vector<double>(dim));
    for (uint64_t t = 0; t < steps; ++t) {
      for (uint64_t i = 0; i < workers; ++i)
        std::memcpy(g[i].data(), grads + (t * workers + i) * dim, dim * 8);
      const auto info = e.step(g);
      merged[t] = info.merged ? 1 : 0;
      for (uint64_t i = 0; i < workers; ++i) {
        const auto& s = e.states()[i];
        const uint64_t o = (t * workers + i) * dim;
        std::memcpy(xs + o, s.x.data(), dim * 8);
        std::memcpy(ms + o, s.m.data(), dim * 8);
        std::memcpy(vs + o, s.v.data(), dim * 8);
        std::memcpy(vbars + o, s.v_bar.data(), dim * 8);
      }
    }
  });
}

// AUC rank-sum (proj/src/eval.cpp:8-39); NaN when undefined
double ref_auc(const double* scores, const int32_t* labels, uint64_t n) {
  std::vector<int> l(labels, labels + n);
  const auto a = compute_auc(std::span<const double>(scores, n), l);
  return a ? *a : std::nan("");
}

// The reference's own synthetic CTR stream (SyntheticCtr, proj/src/data.cpp:11-57,
// resolved from ExperimentConfig as in proj/src/experiment.cpp:35-44), flattened
// to CSR in stream order. Call with offs == NULL to size: *n_out instances,
// *nnz_out feature ids.
int ref_synthetic(uint64_t seed, uint64_t n_instances, uint64_t vocab, double nnz_mean,
                  double signal_scale, uint64_t* offs, uint64_t* keys, int32_t* labels,
                  uint64_t* n_out, uint64_t* nnz_out) {
  return guard([&] {
    SyntheticSpec spec;
    spec.seed = seed;
    spec.n_instances = n_instances;
    spec.vocab = vocab;
    spec.nnz_mean = nnz_mean;
    spec.signal_scale = signal_scale;
    SyntheticCtr gen(spec);
    uint64_t o = 0;
    for (uint64_t i = 0; i < n_instances; ++i) {
      const Instance inst = gen.next();
      if (offs) {
        offs[i] = o;
        std::memcpy(keys + o, inst.feature_ids.data(), inst.feature_ids.size() * 8);
        labels[i] = inst.label;
      }
      o += inst.feature_ids.size();
    }
    if (offs) offs[n_instances] = o;
    *n_out = n_instances;
    *nnz_out = o;
  });
}

// read_instances (proj/src/data.cpp:72-110) on a TSV file, flattened to CSR.
// Same two-call sizing protocol as ref_synthetic.
int ref_read_instances(const char* path, uint64_t* offs, uint64_t* keys, int32_t* labels,
                       uint64_t* n_out, uint64_t* nnz_out) {
  return guard([&] {
    const auto insts = read_instances(path);
    uint64_t o = 0;
    for (uint64_t i = 0; i < insts.size(); ++i) {
      if (offs) {
        offs[i] = o;
        std::memcpy(keys + o, insts[i].feature_ids.data(), insts[i].feature_ids.size() * 8);
        labels[i] = insts[i].label;
      }
      o += insts[i].feature_ids.size();
    }
    if (offs) offs[insts.size()] = o;
    *n_out = insts.size();
    *nnz_out = o;
  });
}

}  // extern "C"
