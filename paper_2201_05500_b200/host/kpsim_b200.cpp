// C++ host shim: the reference's API names over the C ABI. No CUDA headers:
// every device operation goes through include/kpsim_b200.h.
#include "kpsim_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <numeric>

namespace kpsim_b200 {

void check(int status) {
  if (status == KP_OK) return;
  const std::string msg = kp_last_error();
  switch (status) {
    case KP_ERR_CONFIG: throw ConfigError(msg);
    case KP_ERR_STORE:
    case KP_ERR_TABLE_FULL: throw StoreError(msg);
    case KP_ERR_CUDA:
    case KP_ERR_NCCL: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

namespace {

// RAII device buffer through the C ABI
struct Dev {
  void* p = nullptr;
  explicit Dev(std::size_t bytes) { check(kp_dev_alloc(bytes, &p)); }
  ~Dev() {
    if (p) kp_dev_free(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

std::vector<float> to_f32(std::span<const double> v) {
  return std::vector<float>(v.begin(), v.end());
}
void to_f64(const std::vector<float>& f, std::vector<double>& out) {
  out.assign(f.begin(), f.end());
}

void check_gradient_input(const WorkerState& s, std::span<const double> g) {
  if (g.size() != s.dim())
    throw Error("gradient dimension " + std::to_string(g.size()) + " != state dimension " +
                std::to_string(s.dim()));
  for (std::size_t j = 0; j < g.size(); ++j)
    if (!std::isfinite(g[j])) throw Error("non-finite gradient coordinate " + std::to_string(j));
}

}  // namespace

// ---------------------------------------------------------------------------
void AdamHyper::validate() const {
  if (!(alpha > 0.0)) throw ConfigError("adam: alpha must be > 0");
  if (beta1 < 0.0 || beta1 >= 1.0) throw ConfigError("adam: beta1 must be in [0,1)");
  if (beta2 < 0.0 || beta2 >= 1.0) throw ConfigError("adam: beta2 must be in [0,1)");
  if (!(epsilon > 0.0)) throw ConfigError("adam: epsilon must be > 0");
  if (k < 1) throw ConfigError("adam: k must be >= 1");
}

WorkerState WorkerState::init(std::span<const double> x0, double epsilon) {
  WorkerState s;
  s.x.assign(x0.begin(), x0.end());
  s.m.assign(x0.size(), 0.0);
  s.v.assign(x0.size(), epsilon);
  s.v_bar.assign(x0.size(), epsilon);
  return s;
}

// One worker's state in HBM for the free functions below.
struct DevState {
  std::size_t d;
  Dev x, m, v, vb, g;
  explicit DevState(std::size_t dim)
      : d(dim), x(dim * 4), m(dim * 4), v(dim * 4), vb(dim * 4), g(dim * 4) {}
  void upload(const WorkerState& s, std::span<const double> grad) {
    auto fx = to_f32(s.x), fm = to_f32(s.m), fv = to_f32(s.v), fb = to_f32(s.v_bar);
    check(kp_memcpy_h2d(x.p, fx.data(), d * 4));
    check(kp_memcpy_h2d(m.p, fm.data(), d * 4));
    check(kp_memcpy_h2d(v.p, fv.data(), d * 4));
    check(kp_memcpy_h2d(vb.p, fb.data(), d * 4));
    if (!grad.empty()) {
      auto fg = to_f32(grad);
      check(kp_memcpy_h2d(g.p, fg.data(), d * 4));
    }
  }
  void download(WorkerState& s) const {
    std::vector<float> f(d);
    check(kp_memcpy_d2h(f.data(), x.p, d * 4));
    to_f64(f, s.x);
    check(kp_memcpy_d2h(f.data(), m.p, d * 4));
    to_f64(f, s.m);
    check(kp_memcpy_d2h(f.data(), v.p, d * 4));
    to_f64(f, s.v);
    check(kp_memcpy_d2h(f.data(), vb.p, d * 4));
    to_f64(f, s.v_bar);
  }
};

void accumulate_moments(WorkerState& s, std::span<const double> g, const AdamHyper& h) {
  check_gradient_input(s, g);
  DevState d(s.dim());
  d.upload(s, g);
  check(kp_dense_moments(d.m.as<float>(), d.v.as<float>(), d.g.as<float>(), s.dim(),
                         (float)h.beta1, (float)h.beta2, nullptr));
  d.download(s);
}

void local_adam_step(WorkerState& s, std::span<const double> g, const AdamHyper& h) {
  check_gradient_input(s, g);
  DevState d(s.dim());
  d.upload(s, g);
  check(kp_dense_local_step(d.x.as<float>(), d.m.as<float>(), d.v.as<float>(), d.vb.as<float>(),
                            d.g.as<float>(), s.dim(), (float)h.alpha, (float)h.beta1,
                            (float)h.beta2, nullptr));
  d.download(s);
  s.t += 1;
}

void global_merge(std::vector<WorkerState>& states, const AdamHyper& h) {
  if (states.empty()) throw Error("global_merge: empty worker list");
  const std::size_t d = states.front().dim();
  for (const auto& s : states)
    if (s.dim() != d) throw Error("global_merge: mismatched dimensions");
  const std::size_t n = states.size();
  Dev x(n * d * 4), m(n * d * 4), v(n * d * 4), vb(n * d * 4);
  std::vector<float> hx(n * d), hm(n * d), hv(n * d), hb(n * d);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < d; ++j) {
      hx[i * d + j] = (float)states[i].x[j];
      hm[i * d + j] = (float)states[i].m[j];
      hv[i * d + j] = (float)states[i].v[j];
      hb[i * d + j] = (float)states[i].v_bar[j];
    }
  check(kp_memcpy_h2d(x.p, hx.data(), n * d * 4));
  check(kp_memcpy_h2d(m.p, hm.data(), n * d * 4));
  check(kp_memcpy_h2d(v.p, hv.data(), n * d * 4));
  check(kp_memcpy_h2d(vb.p, hb.data(), n * d * 4));
  check(kp_kstep_merge(nullptr, x.as<float>(), m.as<float>(), v.as<float>(), vb.as<float>(),
                       (uint32_t)n, d, (float)h.alpha, h.reset_local_v ? 1 : 0, nullptr));
  check(kp_memcpy_d2h(hx.data(), x.p, n * d * 4));
  check(kp_memcpy_d2h(hv.data(), v.p, n * d * 4));
  check(kp_memcpy_d2h(hb.data(), vb.p, n * d * 4));
  for (std::size_t i = 0; i < n; ++i) {
    for (std::size_t j = 0; j < d; ++j) {
      states[i].x[j] = hx[i * d + j];
      states[i].v[j] = hv[i * d + j];
      states[i].v_bar[j] = hb[i * d + j];
    }
    states[i].t += 1;
  }
}

void adagrad_sparse_update(std::span<double> weight, std::span<double> accumulator,
                           std::span<const double> g, double lr) {
  if (weight.size() != accumulator.size() || weight.size() != g.size())
    throw Error("adagrad_sparse_update: dimension mismatch");
  const std::size_t n = g.size();
  if (n == 0) return;
  // the caller's (w, acc) becomes one row of a scratch table; the device rule
  // updates it in place (the same kernel the trainer's push uses)
  kp_table* t = nullptr;
  auto fw = to_f32(weight), fa = to_f32(accumulator), fg = to_f32(g);
  check(kp_table_create(0, 1, (uint32_t)n, KP_RULE_ADAGRAD, 0.f, 0.f, 0.f, &t));
  try {
    Dev key(8), rows(4), dg(n * 4), dw(n * 4), da(n * 4);
    const uint64_t k0 = 0;
    check(kp_memcpy_h2d(key.p, &k0, 8));
    check(kp_table_pull(t, key.as<uint64_t>(), 1, rows.as<uint32_t>(), nullptr));
    check(kp_memcpy_h2d(dw.p, fw.data(), n * 4));
    check(kp_memcpy_h2d(da.p, fa.data(), n * 4));
    check(kp_table_set_rows(t, rows.as<uint32_t>(), 1, dw.as<float>(), da.as<float>(), nullptr,
                            nullptr));
    check(kp_memcpy_h2d(dg.p, fg.data(), n * 4));
    check(kp_table_apply(t, rows.as<uint32_t>(), dg.as<float>(), 1, (float)lr, 0.f, 0.f, nullptr));
    check(kp_table_gather(t, rows.as<uint32_t>(), 1, dw.as<float>(), da.as<float>(), nullptr,
                          nullptr));
    check(kp_memcpy_d2h(fw.data(), dw.p, n * 4));
    check(kp_memcpy_d2h(fa.data(), da.p, n * 4));
  } catch (...) {
    kp_table_destroy(t);
    throw;
  }
  kp_table_destroy(t);
  for (std::size_t j = 0; j < n; ++j) {
    weight[j] = fw[j];
    accumulator[j] = fa[j];
  }
}

// ---------------------------------------------------------------------------
KStepEngine::KStepEngine(const AdamHyper& h, std::size_t n_workers, std::span<const double> x0,
                         int device)
    : h_(h), n_(n_workers), d_(x0.size()) {
  h_.validate();
  if (n_workers < 1) throw Error("KStepEngine: need at least one worker");
  if (x0.empty()) throw Error("KStepEngine: empty initial model");
  check(kp_set_device(device));
  const std::size_t b = n_ * d_ * 4;
  void* p;
  check(kp_dev_alloc(b, &p));
  x_ = static_cast<float*>(p);
  check(kp_dev_alloc(b, &p));
  m_ = static_cast<float*>(p);
  check(kp_dev_alloc(b, &p));
  v_ = static_cast<float*>(p);
  check(kp_dev_alloc(b, &p));
  vbar_ = static_cast<float*>(p);
  check(kp_dev_alloc(b, &p));
  g_ = static_cast<float*>(p);
  check(kp_dev_alloc(d_ * 4, &p));
  tmp_ = static_cast<float*>(p);
  std::vector<float> fx = to_f32(x0), fe(d_, (float)h_.epsilon);
  check(kp_memset_d(m_, 0, b));
  for (std::size_t i = 0; i < n_; ++i) {
    check(kp_memcpy_h2d(x_ + i * d_, fx.data(), d_ * 4));
    check(kp_memcpy_h2d(v_ + i * d_, fe.data(), d_ * 4));
    check(kp_memcpy_h2d(vbar_ + i * d_, fe.data(), d_ * 4));
  }
}

KStepEngine::~KStepEngine() {
  for (float* p : {x_, m_, v_, vbar_, g_, tmp_})
    if (p) kp_dev_free(p);
}

KStepEngine::StepInfo KStepEngine::step(std::span<const std::vector<double>> gradients) {
  if (gradients.size() != n_) throw Error("KStepEngine::step: gradient count != worker count");
  std::vector<float> fg(n_ * d_);
  for (std::size_t i = 0; i < n_; ++i) {
    if (gradients[i].size() != d_)
      throw Error("gradient dimension " + std::to_string(gradients[i].size()) +
                  " != state dimension " + std::to_string(d_));
    for (std::size_t j = 0; j < d_; ++j) {
      if (!std::isfinite(gradients[i][j]))
        throw Error("non-finite gradient coordinate " + std::to_string(j));
      fg[i * d_ + j] = (float)gradients[i][j];
    }
  }
  check(kp_memcpy_h2d(g_, fg.data(), n_ * d_ * 4));
  const std::uint64_t t = t_ + 1;
  StepInfo info;
  info.merged = (t % h_.k) == 0;
  std::vector<float> before;
  if (info.merged) {
    before.resize(d_);
    check(kp_memcpy_d2h(before.data(), vbar_, d_ * 4));
    for (std::size_t i = 0; i < n_; ++i)
      check(kp_dense_moments(m_ + i * d_, v_ + i * d_, g_ + i * d_, d_, (float)h_.beta1,
                             (float)h_.beta2, nullptr));
    check(kp_kstep_merge(nullptr, x_, m_, v_, vbar_, (uint32_t)n_, d_, (float)h_.alpha,
                         h_.reset_local_v ? 1 : 0, nullptr));
    std::vector<float> after(d_);
    check(kp_memcpy_d2h(after.data(), vbar_, d_ * 4));
    for (std::size_t j = 0; j < d_; ++j)
      info.a3_increment +=
          std::abs(1.0 / std::sqrt((double)before[j]) - 1.0 / std::sqrt((double)after[j]));
  } else {
    for (std::size_t i = 0; i < n_; ++i)
      check(kp_dense_local_step(x_ + i * d_, m_ + i * d_, v_ + i * d_, vbar_ + i * d_, g_ + i * d_,
                                d_, (float)h_.alpha, (float)h_.beta1, (float)h_.beta2, nullptr));
  }
  t_ = t;
  // finite / positivity checks (optimizer.cpp:135-142)
  for (const auto& s : states()) {
    for (std::size_t j = 0; j < d_; ++j) {
      if (!std::isfinite(s.x[j]) || !std::isfinite(s.v[j]))
        throw Error("non-finite worker state after step " + std::to_string(t));
      if (!(s.v[j] > 0.0) || !(s.v_bar[j] > 0.0))
        throw Error("second moment lost positivity at step " + std::to_string(t));
    }
  }
  return info;
}

std::vector<WorkerState> KStepEngine::states() const {
  std::vector<WorkerState> out(n_);
  std::vector<float> f(d_);
  for (std::size_t i = 0; i < n_; ++i) {
    check(kp_memcpy_d2h(f.data(), x_ + i * d_, d_ * 4));
    to_f64(f, out[i].x);
    check(kp_memcpy_d2h(f.data(), m_ + i * d_, d_ * 4));
    to_f64(f, out[i].m);
    check(kp_memcpy_d2h(f.data(), v_ + i * d_, d_ * 4));
    to_f64(f, out[i].v);
    check(kp_memcpy_d2h(f.data(), vbar_ + i * d_, d_ * 4));
    to_f64(f, out[i].v_bar);
    out[i].t = t_;
  }
  return out;
}

std::vector<double> KStepEngine::frozen_v() const {
  std::vector<float> f(d_);
  check(kp_memcpy_d2h(f.data(), vbar_, d_ * 4));
  return std::vector<double>(f.begin(), f.end());
}

std::vector<double> KStepEngine::x_bar() const {
  check(kp_centered_mean(x_, d_, (uint32_t)n_, d_, tmp_, nullptr));
  std::vector<float> f(d_);
  check(kp_memcpy_d2h(f.data(), tmp_, d_ * 4));
  return std::vector<double>(f.begin(), f.end());
}

// ---------------------------------------------------------------------------
TieredStore::TieredStore(TierConfig config, std::size_t embedding_dim)
    : config_(std::move(config)), dim_(embedding_dim) {
  if (config_.cache_capacity < 1) throw StoreError("cache_capacity must be >= 1");
  if (dim_ < 1) throw StoreError("embedding_dim must be >= 1");
  if (config_.cold_path.empty()) throw StoreError("cold_path must be a directory path");
  capacity_ = config_.hbm_capacity ? config_.hbm_capacity
                                   : std::max<std::size_t>(config_.cache_capacity, 1u << 20);
  check(kp_table_create(config_.device, capacity_, (uint32_t)dim_, KP_RULE_ADAGRAD, 0.f,
                        (float)kFreshAccumulator, 0.f, &t_));
}

TieredStore::~TieredStore() {
  if (t_ && owned_) kp_table_destroy(t_);
}

void TieredStore::bind(kp_table* t) {
  if (cache_size() != 0) throw StoreError("trainer: store must be empty when the trainer binds it");
  if (t_ && owned_) kp_table_destroy(t_);
  t_ = t;
  owned_ = false;
}

std::map<ParameterKey, EmbeddingEntry> TieredStore::pull_batch(const std::set<ParameterKey>& keys) {
  if (keys.empty()) throw StoreError("pull_batch: empty key set");
  std::vector<ParameterKey> k(keys.begin(), keys.end());
  const std::size_t n = k.size();
  std::vector<float> w(n * dim_), a(n * dim_);
  check(kp_store_pull_batch(t_, k.data(), (uint32_t)n, w.data(), a.data(), nullptr));
  std::map<ParameterKey, EmbeddingEntry> out;
  for (std::size_t i = 0; i < n; ++i) {
    EmbeddingEntry e;
    e.weights.assign(w.begin() + i * dim_, w.begin() + (i + 1) * dim_);
    e.adagrad_acc.assign(a.begin() + i * dim_, a.begin() + (i + 1) * dim_);
    out.emplace(k[i], std::move(e));
  }
  return out;
}

void TieredStore::push_updates(const std::map<ParameterKey, std::vector<double>>& updates,
                               double lr) {
  // reference order: per key ascending, working-set check then dimension check
  std::vector<ParameterKey> k;
  std::vector<float> g;
  std::size_t bad_dim = updates.size();
  std::size_t i = 0;
  for (const auto& [key, grad] : updates) {
    if (grad.size() != dim_) {
      bad_dim = i;
      break;
    }
    k.push_back(key);
    g.insert(g.end(), grad.begin(), grad.end());
    ++i;
  }
  uint32_t applied = 0;
  int rc = KP_OK;
  if (!k.empty())
    rc = kp_store_push_updates(t_, k.data(), g.data(), (uint32_t)k.size(), (float)lr, 0.f, 0.f,
                               &applied);
  if (rc != KP_OK) check(rc);
  if (bad_dim < updates.size()) {
    // the key with the wrong dimension must still pass the working-set check first
    auto it = std::next(updates.begin(), (long)bad_dim);
    ParameterKey key = it->first;
    std::vector<float> w(dim_), a(dim_);
    int lr2 = kp_store_lookup(t_, key, w.data(), a.data(), nullptr);
    if (lr2 != KP_OK)
      throw StoreError("push_updates: key " + std::to_string(key) +
                       " not in the current working set");
    throw StoreError("push_updates: gradient dimension mismatch");
  }
}

EmbeddingEntry TieredStore::lookup(ParameterKey key) const {
  std::vector<float> w(dim_), a(dim_);
  check(kp_store_lookup(t_, key, w.data(), a.data(), nullptr));
  EmbeddingEntry e;
  e.weights.assign(w.begin(), w.end());
  e.adagrad_acc.assign(a.begin(), a.end());
  return e;
}

std::size_t TieredStore::cache_size() const {
  uint64_t n = 0;
  check(kp_table_size(t_, &n));
  return n;
}

void TieredStore::export_all(std::vector<ParameterKey>& keys, std::vector<float>& w,
                             std::vector<float>& acc) const {
  uint64_t n = 0;
  check(kp_table_export(t_, nullptr, nullptr, nullptr, nullptr, 0, &n));
  keys.resize(n);
  w.resize(n * dim_);
  acc.resize(n * dim_);
  if (n) check(kp_table_export(t_, keys.data(), w.data(), acc.data(), nullptr, n, &n));
}

void TieredStore::flush() {
  namespace fs = std::filesystem;
  std::vector<ParameterKey> keys;
  std::vector<float> w, a;
  export_all(keys, w, a);
  fs::create_directories(config_.cold_path);
  const std::string dp = (fs::path(config_.cold_path) / "cold.dat").string();
  const std::string ip = (fs::path(config_.cold_path) / "cold.idx").string();
  std::ofstream dat(dp, std::ios::binary | std::ios::trunc);
  std::ofstream idx(ip, std::ios::binary | std::ios::trunc);
  if (!dat || !idx) throw StoreError("cold tier: cannot open " + dp);
  dat.write("KPSC\x01", 5);
  idx.write("KPSI\x01", 5);
  uint64_t off = 5;
  const uint32_t d32 = (uint32_t)dim_;
  for (std::size_t i = 0; i < keys.size(); ++i) {
    dat.write(reinterpret_cast<const char*>(&keys[i]), 8);
    dat.write(reinterpret_cast<const char*>(&d32), 4);
    for (std::size_t j = 0; j < dim_; ++j) {
      const double x = w[i * dim_ + j];
      dat.write(reinterpret_cast<const char*>(&x), 8);
    }
    for (std::size_t j = 0; j < dim_; ++j) {
      const double x = a[i * dim_ + j];
      dat.write(reinterpret_cast<const char*>(&x), 8);
    }
    idx.write(reinterpret_cast<const char*>(&keys[i]), 8);
    idx.write(reinterpret_cast<const char*>(&off), 8);
    off += 12 + 16ull * dim_;
  }
  if (!dat || !idx) throw StoreError("cold tier: write failure on " + dp);
}

// ---------------------------------------------------------------------------
std::optional<double> compute_auc(std::span<const double> scores, std::span<const int> labels) {
  if (scores.size() != labels.size()) throw Error("compute_auc: scores/labels length mismatch");
  const std::size_t n = scores.size();
  std::size_t pos = 0;
  for (int y : labels) {
    if (y != 0 && y != 1) throw Error("compute_auc: label outside {0,1}");
    pos += (std::size_t)y;
  }
  const std::size_t neg = n - pos;
  if (pos == 0 || neg == 0) return std::nullopt;
  std::vector<std::size_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return scores[a] < scores[b]; });
  double prs = 0.0;
  std::size_t i = 0;
  while (i < n) {
    std::size_t j = i;
    while (j < n && scores[order[j]] == scores[order[i]]) ++j;
    const double avg = 0.5 * (double)(i + 1 + j);
    for (std::size_t t = i; t < j; ++t)
      if (labels[order[t]] == 1) prs += avg;
    i = j;
  }
  const double p = (double)pos, m = (double)neg;
  return (prs - p * (p + 1.0) / 2.0) / (p * m);
}

void AucAccumulator::add(std::span<const double> scores, std::span<const int> labels) {
  scores_.insert(scores_.end(), scores.begin(), scores.end());
  labels_.insert(labels_.end(), labels.begin(), labels.end());
}
std::optional<double> AucAccumulator::value() const {
  if (scores_.empty()) return std::nullopt;
  return compute_auc(scores_, labels_);
}

// ---------------------------------------------------------------------------
Trainer::Trainer(const TrainerConfig& config, TieredStore& store, const void* /*topology*/,
                 kp_comm* comm)
    : config_(config), store_(store) {
  config_.adam.validate();
  if (store_.embedding_dim() != config_.model.embedding_dim)
    throw Error("trainer: store embedding_dim != model embedding_dim");
  if (config_.model.hidden.size() > 8) throw ConfigError("at most 8 hidden layers");
  if (comm) check(kp_comm_rank(comm, &rank_, &world_));
  if (config_.n_workers % (std::size_t)world_ != 0)
    throw ConfigError("n_workers must be a multiple of the world size");
  W_ = config_.n_workers / world_;
  kp_trainer_config c{};
  c.seed = config_.seed;
  c.n_workers = (uint32_t)config_.n_workers;
  c.local_workers = (uint32_t)W_;
  c.minibatch_size = config_.minibatch_size;
  c.sparse_lr = config_.sparse_lr;
  c.alpha = config_.adam.alpha;
  c.beta1 = config_.adam.beta1;
  c.beta2 = config_.adam.beta2;
  c.epsilon = config_.adam.epsilon;
  c.k = config_.adam.k;
  c.reset_local_v = config_.adam.reset_local_v ? 1 : 0;
  c.embedding_dim = (uint32_t)config_.model.embedding_dim;
  c.n_slots = (uint32_t)config_.model.n_slots;
  c.n_hidden = (uint32_t)config_.model.hidden.size();
  for (std::size_t i = 0; i < config_.model.hidden.size(); ++i)
    c.hidden[i] = (uint32_t)config_.model.hidden[i];
  if (config_.model.activation == "relu") c.activation = 0;
  else if (config_.model.activation == "tanh") c.activation = 1;
  else throw ConfigError("unknown activation '" + config_.model.activation + "' (relu|tanh)");
  if (config_.model.pooling == "sum") c.pooling = 0;
  else if (config_.model.pooling == "mean") c.pooling = 1;
  else throw ConfigError("unknown pooling '" + config_.model.pooling + "' (sum|mean)");
  if (config_.sparse_rule == "adagrad") c.sparse_rule = KP_RULE_ADAGRAD;
  else if (config_.sparse_rule == "adam") c.sparse_rule = KP_RULE_ADAM;
  else throw ConfigError("unknown sparse rule '" + config_.sparse_rule + "' (adagrad|adam)");
  c.sparse_beta1 = config_.sparse_beta1;
  c.sparse_beta2 = config_.sparse_beta2;
  c.sparse_eps = config_.sparse_eps;
  c.table_capacity = store_.capacity();
  check(kp_trainer_create(&c, comm, store_.device(), &tr_));
  uint64_t D = 0;
  check(kp_trainer_dense_dim(tr_, &D));
  D_ = D;
  kp_table* t = nullptr;
  check(kp_trainer_table(tr_, &t));
  store_.bind(t);
}

Trainer::~Trainer() {
  if (tr_) kp_trainer_destroy(tr_);
}

CsrResult Trainer::train_csr(const std::uint32_t* offs, const ParameterKey* keys,
                             const std::uint16_t* slots, const std::int32_t* labels,
                             std::uint32_t n, std::uint64_t global_n, std::uint64_t global_first,
                             bool predict_first) {
  CsrResult r;
  if (predict_first) r.preds.resize(n);
  kp_batch_result br{};
  check(kp_trainer_train_batch(tr_, offs, keys, slots, labels, n, global_n, global_first,
                               predict_first ? 1 : 0, predict_first ? r.preds.data() : nullptr,
                               &br));
  r.loss = br.loss;
  r.minibatch_steps = br.minibatch_steps;
  r.merges = br.merges;
  if (br.has_auc) {
    if (std::isfinite(br.auc)) r.auc = br.auc;
    if (std::isfinite(br.cumulative_auc)) r.cumulative_auc = br.cumulative_auc;
  }
  steps_ = br.steps_total;
  metrics_.minibatch_steps += br.minibatch_steps;
  metrics_.merge_events += br.merges;
  return r;
}

CsrResult Trainer::train_csr_device(const std::uint32_t* h_offs, const std::uint32_t* d_offs,
                                    const ParameterKey* d_keys, const std::uint16_t* d_slots,
                                    const std::int32_t* d_labels, std::uint32_t n,
                                    std::uint64_t global_n, std::uint64_t global_first,
                                    bool predict_first) {
  CsrResult r;
  if (predict_first) r.preds.resize(n);
  kp_batch_result br{};
  check(kp_trainer_train_batch_device(tr_, h_offs, d_offs, d_keys, d_slots, d_labels, n, global_n,
                                      global_first, predict_first ? 1 : 0,
                                      predict_first ? r.preds.data() : nullptr, &br));
  r.loss = br.loss;
  r.minibatch_steps = br.minibatch_steps;
  r.merges = br.merges;
  if (br.has_auc) {
    if (std::isfinite(br.auc)) r.auc = br.auc;
    if (std::isfinite(br.cumulative_auc)) r.cumulative_auc = br.cumulative_auc;
  }
  steps_ = br.steps_total;
  metrics_.minibatch_steps += br.minibatch_steps;
  metrics_.merge_events += br.merges;
  return r;
}

BatchRecord Trainer::process(const Batch& b, bool predict_first) {
  if (b.instances.empty()) throw Error("train_batch: empty batch");
  if (world_ != 1) throw Error("Trainer::train_batch(Batch): use train_csr for multi-rank slices");
  std::vector<std::uint32_t> offs{0};
  std::vector<ParameterKey> keys;
  std::vector<std::uint16_t> slots;
  std::vector<std::int32_t> labels;
  bool any_slots = false;
  for (const auto& inst : b.instances) {
    if (inst.label != 0 && inst.label != 1) throw Error("backward: label outside {0,1}");
    keys.insert(keys.end(), inst.feature_ids.begin(), inst.feature_ids.end());
    if (!inst.slots.empty()) {
      any_slots = true;
      if (inst.slots.size() != inst.feature_ids.size()) throw Error("slots/feature_ids mismatch");
    }
    offs.push_back((std::uint32_t)keys.size());
    labels.push_back(inst.label);
  }
  if (any_slots) {
    for (const auto& inst : b.instances) {
      if (inst.slots.empty()) slots.insert(slots.end(), inst.feature_ids.size(), 0);
      else slots.insert(slots.end(), inst.slots.begin(), inst.slots.end());
    }
  }
  CsrResult r = train_csr(offs.data(), keys.data(), any_slots ? slots.data() : nullptr,
                          labels.data(), (std::uint32_t)b.instances.size(), b.instances.size(), 0,
                          predict_first);
  BatchRecord rec;
  rec.batch = b.id;
  rec.instances = b.instances.size();
  rec.loss = r.loss;
  if (predict_first) {  // online AUC computed on the device (kp_auc.cu)
    rec.auc = r.auc;
    rec.cumulative_auc = r.cumulative_auc;
  }
  metrics_.batches.push_back(rec);
  return rec;
}

BatchRecord Trainer::train_batch(const Batch& b) { return process(b, false); }

TrainMetrics Trainer::online_eval(std::span<const Batch> stream) {
  for (const auto& b : stream) metrics_.cumulative_auc = process(b, true).cumulative_auc;
  return metrics_;
}

std::vector<double> Trainer::dense_model() const {
  std::vector<float> f(D_);
  check(kp_trainer_xbar(tr_, f.data()));
  return std::vector<double>(f.begin(), f.end());
}

std::vector<WorkerState> Trainer::worker_states() const {
  std::vector<WorkerState> out(W_);
  std::vector<float> x(D_), m(D_), v(D_), vb(D_);
  for (std::size_t l = 0; l < W_; ++l) {
    check(kp_trainer_worker_state(tr_, (uint32_t)l, x.data(), m.data(), v.data(), vb.data()));
    to_f64(x, out[l].x);
    to_f64(m, out[l].m);
    to_f64(v, out[l].v);
    to_f64(vb, out[l].v_bar);
    out[l].t = steps_;
  }
  return out;
}

void Trainer::set_worker_state(std::size_t l, const WorkerState& s) {
  if (s.dim() != D_) throw Error("set_worker_state: dimension mismatch");
  auto x = to_f32(s.x), m = to_f32(s.m), v = to_f32(s.v), vb = to_f32(s.v_bar);
  check(kp_trainer_set_worker_state(tr_, (uint32_t)l, x.data(), m.data(), v.data(), vb.data()));
}

// ---------------------------------------------------------------- ledger --
LedgerReport Trainer::ledger() const {
  uint64_t bytes[5], count[5];
  check(kp_trainer_ledger(tr_, bytes, count));
  LedgerReport rep;
  for (int i = 0; i < 5; ++i) {
    if (!count[i] && !bytes[i]) continue;
    rep.categories[static_cast<TransferCategory>(i)] = {bytes[i], count[i]};
    rep.total.bytes += bytes[i];
    rep.total.count += count[i];
  }
  return rep;
}

const char* to_string(TransferCategory c) {
  switch (c) {
    case TransferCategory::GpuPull: return "gpu_pull";
    case TransferCategory::GpuPush: return "gpu_push";
    case TransferCategory::DenseMerge: return "dense_merge";
    case TransferCategory::SparseSync: return "sparse_sync";
    case TransferCategory::ColdTierIo: return "cold_tier_io";
  }
  return "?";
}

std::uint64_t LedgerReport::bytes(TransferCategory c) const {
  auto it = categories.find(c);
  return it == categories.end() ? 0 : it->second.bytes;
}

KStepRatios kstep_ratio(const LedgerReport& kstep, const LedgerReport& baseline) {
  const auto base_dense = baseline.bytes(TransferCategory::DenseMerge);
  const auto base_total = baseline.total.bytes;
  if (base_total == 0) throw Error("kstep_ratio: zero-byte baseline ledger");
  KStepRatios r;
  r.dense_bytes = base_dense == 0 ? 0.0
                                  : static_cast<double>(kstep.bytes(TransferCategory::DenseMerge)) /
                                        static_cast<double>(base_dense);
  r.total_bytes = static_cast<double>(kstep.total.bytes) / static_cast<double>(base_total);
  return r;
}

// ------------------------------------------------------------ trajectory --
void Trainer::record_trajectory(bool on) { check(kp_trainer_record_trajectory(tr_, on ? 1 : 0)); }

Trajectory Trainer::dense_trajectory() const {
  Trajectory tj;
  tj.dim = D_;
  tj.workers = config_.n_workers;
  uint64_t n = 0;
  check(kp_trainer_trajectory(tr_, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &n));
  std::vector<float> xb(D_), vb(D_);
  for (uint64_t i = 0; i < n; ++i) {
    StepRecord r;
    int merged = 0;
    check(kp_trainer_trajectory(tr_, i, &r.step, &merged, &r.loss, &r.a3_increment, xb.data(),
                                vb.data(), nullptr));
    r.merged = merged != 0;
    to_f64(xb, r.x_bar);
    to_f64(vb, r.v_bar);
    tj.steps.push_back(std::move(r));
  }
  return tj;
}

// -------------------------------------------------------------- data file --
namespace {
// one line of the instance file (proj/src/data.cpp:72-110): "label<TAB>ids"
// with ids comma separated (empty tokens skipped), parsed by std::stoull
// (base 10, leading blanks and a sign accepted, trailing junk ignored),
// collected into a std::set (ascending, deduped)
void parse_line(const std::string& line, int lineno, std::set<ParameterKey>& seen, int& label) {
  const auto tab = line.find('\t');
  if (tab == std::string::npos)
    throw Error("instance file line " + std::to_string(lineno) + ": missing tab separator");
  const std::string label_s = line.substr(0, tab);
  if (label_s != "0" && label_s != "1")
    throw Error("instance file line " + std::to_string(lineno) + ": label must be 0 or 1");
  label = label_s == "1" ? 1 : 0;
  seen.clear();
  std::size_t pos = tab + 1;
  while (pos <= line.size()) {
    std::size_t end = line.find(',', pos);
    if (end == std::string::npos) end = line.size();
    if (end > pos) {
      const std::string tok = line.substr(pos, end - pos);
      try {
        seen.insert(std::stoull(tok));
      } catch (const std::exception&) {
        throw Error("instance file line " + std::to_string(lineno) + ": bad feature id '" + tok + "'");
      }
    }
    pos = end + 1;
  }
  if (seen.empty()) throw Error("instance file line " + std::to_string(lineno) + ": no feature ids");
}
}  // namespace

void read_instances_csr(const std::string& path, std::vector<std::uint32_t>& offs,
                        std::vector<ParameterKey>& keys, std::vector<std::int32_t>& labels) {
  std::ifstream in(path);
  if (!in) throw Error("cannot open instance file: " + path);
  offs.assign(1, 0);
  keys.clear();
  labels.clear();
  std::string line;
  std::set<ParameterKey> seen;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    int label = 0;
    parse_line(line, lineno, seen, label);
    keys.insert(keys.end(), seen.begin(), seen.end());
    if (keys.size() > 0xFFFFFFFFull) throw Error("instance file: more than 2^32 feature ids");
    offs.push_back(static_cast<std::uint32_t>(keys.size()));
    labels.push_back(label);
  }
}

std::vector<Instance> read_instances(const std::string& path) {
  std::vector<std::uint32_t> offs;
  std::vector<ParameterKey> keys;
  std::vector<std::int32_t> labels;
  read_instances_csr(path, offs, keys, labels);
  std::vector<Instance> out(labels.size());
  for (std::size_t i = 0; i < labels.size(); ++i) {
    out[i].feature_ids.assign(keys.begin() + offs[i], keys.begin() + offs[i + 1]);
    out[i].label = labels[i];
  }
  return out;
}

void write_instances(const std::string& path, const std::vector<Instance>& instances) {
  std::ofstream out(path);
  if (!out) throw Error("cannot write instance file: " + path);
  for (const auto& inst : instances) {
    out << inst.label << '\t';
    for (std::size_t i = 0; i < inst.feature_ids.size(); ++i) {
      if (i > 0) out << ',';
      out << inst.feature_ids[i];
    }
    out << '\n';
  }
}

std::vector<Batch> make_batches(std::vector<Instance> instances, std::uint64_t batch_size) {
  if (batch_size < 1) throw ConfigError("batch_size must be >= 1");
  std::vector<Batch> batches;
  Batch current;
  current.id = 0;
  for (auto& inst : instances) {
    current.instances.push_back(std::move(inst));
    if (current.instances.size() == batch_size) {
      batches.push_back(std::move(current));
      current = Batch{};
      current.id = batches.size();
    }
  }
  if (!current.instances.empty()) batches.push_back(std::move(current));
  return batches;
}

}  // namespace kpsim_b200
