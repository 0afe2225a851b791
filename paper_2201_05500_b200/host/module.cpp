// Python module `_kpsim_b200`: the reference's `_core` names for the hot path
// (proj/bindings/module.cpp:83-296, re-exported by proj/python/kpsim/__init__.py)
// bound to the C++ shim, plus array-level entry points (numpy) for the
// trainer and the primitives.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <memory>

#include "kpsim_b200.hpp"

namespace py = pybind11;
using namespace kpsim_b200;

namespace {

template <class T>
using Arr = py::array_t<T, py::array::c_style | py::array::forcecast>;

// python-owned communicator handle
struct Comm {
  kp_comm* c = nullptr;
  Comm(py::bytes id, int rank, int world, int device) {
    std::string s = id;
    if (s.size() != 128) throw ConfigError("nccl unique id must be 128 bytes");
    check(kp_comm_init(reinterpret_cast<const uint8_t*>(s.data()), rank, world, device, &c));
  }
  ~Comm() {
    if (c) kp_comm_destroy(c);
  }
};

// Trainer bound to its own store (python owns both)
struct PyTrainer {
  std::unique_ptr<TieredStore> store;
  std::unique_ptr<Trainer> tr;
  std::shared_ptr<Comm> comm;
  // host arrays of the staged batches: the H2D reads them until train_staged
  py::object staged[2];
};

TrainerConfig config_from_kwargs(const py::kwargs& kw) {
  TrainerConfig c;
  auto get = [&](const char* k, auto& out) {
    if (kw.contains(k)) out = kw[k].cast<std::decay_t<decltype(out)>>();
  };
  get("seed", c.seed);
  get("n_workers", c.n_workers);
  get("minibatch_size", c.minibatch_size);
  get("sparse_lr", c.sparse_lr);
  get("alpha", c.adam.alpha);
  get("beta1", c.adam.beta1);
  get("beta2", c.adam.beta2);
  get("epsilon", c.adam.epsilon);
  get("k", c.adam.k);
  get("reset_local_v", c.adam.reset_local_v);
  get("vocab", c.model.vocab);
  get("embedding_dim", c.model.embedding_dim);
  get("hidden", c.model.hidden);
  get("activation", c.model.activation);
  get("pooling", c.model.pooling);
  get("n_slots", c.model.n_slots);
  get("sparse_rule", c.sparse_rule);
  get("sparse_beta1", c.sparse_beta1);
  get("sparse_beta2", c.sparse_beta2);
  get("sparse_eps", c.sparse_eps);
  return c;
}

py::dict ledger_to_dict(const LedgerReport& r) {
  py::dict d;
  for (int i = 0; i < 5; ++i) {
    const auto c = static_cast<TransferCategory>(i);
    auto it = r.categories.find(c);
    py::dict e;
    e["bytes"] = it == r.categories.end() ? 0 : it->second.bytes;
    e["count"] = it == r.categories.end() ? 0 : it->second.count;
    d[to_string(c)] = e;
  }
  py::dict t;
  t["bytes"] = r.total.bytes;
  t["count"] = r.total.count;
  d["total"] = t;
  return d;
}

LedgerReport ledger_from_dict(const py::dict& d) {
  LedgerReport r;
  for (int i = 0; i < 5; ++i) {
    const auto c = static_cast<TransferCategory>(i);
    if (!d.contains(to_string(c))) continue;
    py::dict e = d[to_string(c)];
    CategoryTotals t{e["bytes"].cast<std::uint64_t>(), e["count"].cast<std::uint64_t>()};
    if (!t.bytes && !t.count) continue;
    r.categories[c] = t;
    r.total.bytes += t.bytes;
    r.total.count += t.count;
  }
  return r;
}

}  // namespace

PYBIND11_MODULE(_kpsim_b200, m) {
  m.doc() = "B200-native sparse-embedding training hot path (kpsim drop-in)";
  // translators run newest-first, so the base class registers first
  auto& base = py::register_exception<Error>(m, "KpsimError", PyExc_RuntimeError);
  py::register_exception<ConfigError>(m, "ConfigError", PyExc_ValueError);
  py::register_exception<StoreError>(m, "StoreError", base.ptr());
  py::register_exception<DeviceError>(m, "DeviceError", base.ptr());

  m.def("version", [] { return std::string(kp_version()); });
  m.def("device_count", [] {
    int n = 0;
    return kp_device_count(&n) == KP_OK ? n : 0;
  });
  m.def("launch_count", [] { return kp_launch_count(); });
  // ---- data file (proj/src/data.cpp:72-124) + ledger arithmetic ----
  m.def(
      "read_instances",
      [](const std::string& path) {
        std::vector<std::uint32_t> offs;
        std::vector<ParameterKey> keys;
        std::vector<std::int32_t> labels;
        read_instances_csr(path, offs, keys, labels);
        return py::make_tuple(Arr<std::uint32_t>((py::ssize_t)offs.size(), offs.data()),
                              Arr<std::uint64_t>((py::ssize_t)keys.size(), keys.data()),
                              Arr<std::int32_t>((py::ssize_t)labels.size(), labels.data()));
      },
      py::arg("path"));
  m.def(
      "write_instances",
      [](const std::string& path, Arr<std::uint32_t> offs, Arr<std::uint64_t> keys,
         Arr<std::int32_t> labels) {
        const std::size_t n = labels.size();
        if ((std::size_t)offs.size() != n + 1) throw Error("offs must have n+1 entries");
        if ((std::size_t)keys.size() != offs.data()[n]) throw Error("keys size != offs[n]");
        std::vector<Instance> insts(n);
        for (std::size_t i = 0; i < n; ++i) {
          insts[i].feature_ids.assign(keys.data() + offs.data()[i], keys.data() + offs.data()[i + 1]);
          insts[i].label = labels.data()[i];
        }
        write_instances(path, insts);
      },
      py::arg("path"), py::arg("offs"), py::arg("keys"), py::arg("labels"));
  m.def(
      "kstep_ratio",
      [](const py::dict& kstep, const py::dict& baseline) {
        const KStepRatios r = kstep_ratio(ledger_from_dict(kstep), ledger_from_dict(baseline));
        py::dict d;
        d["dense_bytes"] = r.dense_bytes;
        d["total_bytes"] = r.total_bytes;
        return d;
      },
      py::arg("kstep"), py::arg("baseline"));

  // ---- optimizer ----
  py::class_<AdamHyper>(m, "AdamHyper")
      .def(py::init<>())
      .def_readwrite("alpha", &AdamHyper::alpha)
      .def_readwrite("beta1", &AdamHyper::beta1)
      .def_readwrite("beta2", &AdamHyper::beta2)
      .def_readwrite("epsilon", &AdamHyper::epsilon)
      .def_readwrite("k", &AdamHyper::k)
      .def_readwrite("reset_local_v", &AdamHyper::reset_local_v);

  py::class_<WorkerState>(m, "WorkerState")
      .def_static("init", [](const std::vector<double>& x0, double eps) { return WorkerState::init(x0, eps); },
                  py::arg("x0"), py::arg("epsilon"))
      .def_readwrite("x", &WorkerState::x)
      .def_readwrite("m", &WorkerState::m)
      .def_readwrite("v", &WorkerState::v)
      .def_readwrite("v_bar", &WorkerState::v_bar)
      .def_readonly("t", &WorkerState::t);

  m.def("local_adam_step",
        [](WorkerState& s, const std::vector<double>& g, const AdamHyper& h) {
          local_adam_step(s, g, h);
          return s;
        },
        py::arg("state"), py::arg("gradient"), py::arg("hyper"));
  m.def("accumulate_moments",
        [](WorkerState& s, const std::vector<double>& g, const AdamHyper& h) {
          accumulate_moments(s, g, h);
          return s;
        },
        py::arg("state"), py::arg("gradient"), py::arg("hyper"));
  m.def("global_merge",
        [](std::vector<WorkerState> states, const AdamHyper& h) {
          global_merge(states, h);
          return states;
        },
        py::arg("states"), py::arg("hyper"));
  m.def("adagrad_sparse_update",
        [](std::vector<double> w, std::vector<double> acc, const std::vector<double>& g, double lr) {
          adagrad_sparse_update(w, acc, g, lr);
          return py::make_tuple(w, acc);
        },
        py::arg("weight"), py::arg("accumulator"), py::arg("gradient"), py::arg("lr"));

  py::class_<KStepEngine>(m, "KStepEngine")
      .def(py::init([](const AdamHyper& h, std::size_t n, const std::vector<double>& x0, int dev) {
             return std::make_unique<KStepEngine>(h, n, x0, dev);
           }),
           py::arg("hyper"), py::arg("workers"), py::arg("x0"), py::arg("device") = 0)
      .def("step",
           [](KStepEngine& e, const std::vector<std::vector<double>>& g) {
             auto info = e.step(g);
             return py::make_tuple(info.merged, info.a3_increment);
           },
           py::arg("gradients"))
      .def("states", &KStepEngine::states)
      .def("x_bar", &KStepEngine::x_bar)
      .def("frozen_v", &KStepEngine::frozen_v)
      .def_property_readonly("completed_steps", &KStepEngine::completed_steps);

  // ---- store ----
  py::class_<TieredStore>(m, "TieredStore")
      .def(py::init([](std::size_t cache_capacity, const std::string& cold_dir, std::size_t dim,
                       std::size_t hbm_capacity, int device) {
             TierConfig t;
             t.cache_capacity = cache_capacity;
             t.cold_path = cold_dir;
             t.hbm_capacity = hbm_capacity;
             t.device = device;
             return std::make_unique<TieredStore>(t, dim);
           }),
           py::arg("cache_capacity"), py::arg("cold_dir"), py::arg("embedding_dim"),
           py::arg("hbm_capacity") = 0, py::arg("device") = 0)
      .def("pull",
           [](TieredStore& s, const std::vector<ParameterKey>& keys) {
             const auto got = s.pull_batch(std::set<ParameterKey>(keys.begin(), keys.end()));
             py::dict out;
             for (const auto& [key, e] : got) out[py::int_(key)] = py::make_tuple(e.weights, e.adagrad_acc);
             return out;
           },
           py::arg("keys"))
      .def("push",
           [](TieredStore& s, const std::map<ParameterKey, std::vector<double>>& updates, double lr) {
             s.push_updates(updates, lr);
           },
           py::arg("updates"), py::arg("lr"))
      .def("lookup",
           [](const TieredStore& s, ParameterKey k) {
             auto e = s.lookup(k);
             return py::make_tuple(e.weights, e.adagrad_acc);
           })
      .def("evict", &TieredStore::evict)
      .def("flush", &TieredStore::flush)
      .def("export",
           [](const TieredStore& s) {
             std::vector<ParameterKey> k;
             std::vector<float> w, a;
             s.export_all(k, w, a);
             const py::ssize_t n = (py::ssize_t)k.size(), d = (py::ssize_t)s.embedding_dim();
             Arr<uint64_t> K(n);
             Arr<float> W({n, d}), A({n, d});
             std::copy(k.begin(), k.end(), K.mutable_data());
             std::copy(w.begin(), w.end(), W.mutable_data());
             std::copy(a.begin(), a.end(), A.mutable_data());
             return py::make_tuple(K, W, A);
           })
      .def_property_readonly("cache_size", &TieredStore::cache_size)
      .def_property_readonly("embedding_dim", &TieredStore::embedding_dim);

  // ---- data + eval ----
  m.def("compute_auc",
        [](const std::vector<double>& scores, const std::vector<int>& labels) -> py::object {
          const auto a = compute_auc(scores, labels);
          if (!a) return py::none();
          return py::float_(*a);
        },
        py::arg("scores"), py::arg("labels"));

  // ---- primitives on numpy arrays (device round trip) ----
  m.def("dedup",
        [](Arr<uint64_t> keys, int device) {
          check(kp_set_device(device));
          const uint32_t n = (uint32_t)keys.size();
          void *dk, *du, *di, *ds;
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 8, &dk));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 8, &du));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 4, &di));
          check(kp_dev_alloc((std::max<size_t>(n, 1) + 1) * 4, &ds));
          uint32_t U = 0;
          int rc = kp_memcpy_h2d(dk, keys.data(), (size_t)n * 8);
          if (rc == KP_OK)
            rc = kp_dedup((const uint64_t*)dk, n, (uint64_t*)du, (uint32_t*)di, (uint32_t*)ds, &U, nullptr);
          Arr<uint64_t> uq(U);
          Arr<uint32_t> inv(n), seg(U + 1);
          if (rc == KP_OK) rc = kp_memcpy_d2h(uq.mutable_data(), du, (size_t)U * 8);
          if (rc == KP_OK) rc = kp_memcpy_d2h(inv.mutable_data(), di, (size_t)n * 4);
          if (rc == KP_OK) rc = kp_memcpy_d2h(seg.mutable_data(), ds, (size_t)(U + 1) * 4);
          for (void* p : {dk, du, di, ds}) kp_dev_free(p);
          check(rc);
          return py::make_tuple(uq, inv, seg);
        },
        py::arg("keys"), py::arg("device") = 0);
  m.def("dedup_runs",
        [](Arr<uint64_t> keys, Arr<uint64_t> run_lengths, int device) {
          check(kp_set_device(device));
          const uint32_t n = (uint32_t)keys.size();
          const uint32_t R = (uint32_t)run_lengths.size();
          std::vector<uint64_t> off(R + 1, 0);
          for (uint32_t r = 0; r < R; ++r) off[r + 1] = off[r] + run_lengths.data()[r];
          void *dk, *du, *di, *ds, *dp;
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 8, &dk));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 8, &du));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 4, &di));
          check(kp_dev_alloc((std::max<size_t>(n, 1) + 1) * 4, &ds));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 4, &dp));
          uint32_t U = 0;
          int rc = kp_memcpy_h2d(dk, keys.data(), (size_t)n * 8);
          if (rc == KP_OK)
            rc = kp_dedup_runs((const uint64_t*)dk, n, off.data(), R, (uint64_t*)du, (uint32_t*)di,
                               (uint32_t*)ds, (uint32_t*)dp, &U, nullptr);
          Arr<uint64_t> uq(U);
          Arr<uint32_t> inv(n), seg(U + 1), pos(n);
          if (rc == KP_OK) rc = kp_memcpy_d2h(uq.mutable_data(), du, (size_t)U * 8);
          if (rc == KP_OK) rc = kp_memcpy_d2h(inv.mutable_data(), di, (size_t)n * 4);
          if (rc == KP_OK) rc = kp_memcpy_d2h(seg.mutable_data(), ds, (size_t)(U + 1) * 4);
          if (rc == KP_OK) rc = kp_memcpy_d2h(pos.mutable_data(), dp, (size_t)n * 4);
          for (void* p : {dk, du, di, ds, dp}) kp_dev_free(p);
          check(rc);
          return py::make_tuple(uq, inv, seg, pos);
        },
        py::arg("keys"), py::arg("run_lengths"), py::arg("device") = 0);
  m.def("shard",
        [](Arr<uint64_t> uniq, uint32_t G, int device) {
          check(kp_set_device(device));
          const uint32_t n = (uint32_t)uniq.size();
          void *du, *dp, *dq;
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 8, &du));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 4, &dp));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 4, &dq));
          std::vector<uint64_t> counts(G);
          int rc = kp_memcpy_h2d(du, uniq.data(), (size_t)n * 8);
          if (rc == KP_OK)
            rc = kp_shard((const uint64_t*)du, n, G, (uint32_t*)dp, (uint32_t*)dq, counts.data(), nullptr);
          Arr<uint32_t> perm(n), pos(n);
          if (rc == KP_OK) rc = kp_memcpy_d2h(perm.mutable_data(), dp, (size_t)n * 4);
          if (rc == KP_OK) rc = kp_memcpy_d2h(pos.mutable_data(), dq, (size_t)n * 4);
          for (void* p : {du, dp, dq}) kp_dev_free(p);
          check(rc);
          Arr<uint64_t> c(G);
          std::copy(counts.begin(), counts.end(), c.mutable_data());
          return py::make_tuple(perm, pos, c);
        },
        py::arg("unique"), py::arg("G"), py::arg("device") = 0);

  m.def("gemm_nt",
        [](Arr<float> A, Arr<float> B, int engine, int device) {
          if (A.ndim() != 2 || B.ndim() != 2 || A.shape(1) != B.shape(1))
            throw Error("gemm_nt: A[M][K], B[N][K] expected");
          check(kp_set_device(device));
          const int M = (int)A.shape(0), K = (int)A.shape(1), N = (int)B.shape(0);
          void *da, *db, *dc;
          check(kp_dev_alloc((size_t)M * K * 4, &da));
          check(kp_dev_alloc((size_t)N * K * 4, &db));
          check(kp_dev_alloc((size_t)M * N * 4, &dc));
          int rc = kp_memcpy_h2d(da, A.data(), (size_t)M * K * 4);
          if (rc == KP_OK) rc = kp_memcpy_h2d(db, B.data(), (size_t)N * K * 4);
          if (rc == KP_OK)
            rc = kp_gemm_nt((const float*)da, K, (const float*)db, K, (float*)dc, N, M, N, K, engine, nullptr);
          Arr<float> C({(py::ssize_t)M, (py::ssize_t)N});
          if (rc == KP_OK) rc = kp_memcpy_d2h(C.mutable_data(), dc, (size_t)M * N * 4);
          for (void* p2 : {da, db, dc}) kp_dev_free(p2);
          check(rc);
          return C;
        },
        py::arg("A"), py::arg("B"), py::arg("engine") = 0, py::arg("device") = 0);

  m.def("auc_device",
        [](Arr<float> scores, Arr<int32_t> labels, int device) -> py::object {
          if (scores.size() != labels.size()) throw Error("compute_auc: scores/labels length mismatch");
          check(kp_set_device(device));
          const uint32_t n = (uint32_t)scores.size();
          void *ds, *dl;
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 4, &ds));
          check(kp_dev_alloc(std::max<size_t>(n, 1) * 4, &dl));
          double auc = 0;
          int rc = kp_memcpy_h2d(ds, scores.data(), (size_t)n * 4);
          if (rc == KP_OK) rc = kp_memcpy_h2d(dl, labels.data(), (size_t)n * 4);
          if (rc == KP_OK) rc = kp_compute_auc((const float*)ds, (const int32_t*)dl, n, &auc, nullptr);
          kp_dev_free(ds);
          kp_dev_free(dl);
          check(rc);
          if (!(auc == auc)) return py::none();
          return py::float_(auc);
        },
        py::arg("scores"), py::arg("labels"), py::arg("device") = 0);
  m.def("gemm_tn",
        [](Arr<float> A, Arr<float> B, int engine, int device) {
          if (A.ndim() != 2 || B.ndim() != 2 || A.shape(0) != B.shape(0))
            throw Error("gemm_tn: A[K][M], B[K][N] expected");
          check(kp_set_device(device));
          const int K = (int)A.shape(0), M = (int)A.shape(1), N = (int)B.shape(1);
          void *da, *db, *dc;
          check(kp_dev_alloc((size_t)M * K * 4, &da));
          check(kp_dev_alloc((size_t)N * K * 4, &db));
          check(kp_dev_alloc((size_t)M * N * 4, &dc));
          int rc = kp_memcpy_h2d(da, A.data(), (size_t)M * K * 4);
          if (rc == KP_OK) rc = kp_memcpy_h2d(db, B.data(), (size_t)N * K * 4);
          if (rc == KP_OK)
            rc = kp_gemm_tn((const float*)da, M, (const float*)db, N, (float*)dc, N, M, N, K, engine, nullptr);
          Arr<float> C({(py::ssize_t)M, (py::ssize_t)N});
          if (rc == KP_OK) rc = kp_memcpy_d2h(C.mutable_data(), dc, (size_t)M * N * 4);
          for (void* p2 : {da, db, dc}) kp_dev_free(p2);
          check(rc);
          return C;
        },
        py::arg("A"), py::arg("B"), py::arg("engine") = 0, py::arg("device") = 0);

  // ---- comm ----
  m.def("comm_unique_id", [] {
    uint8_t id[128];
    check(kp_comm_unique_id(id));
    return py::bytes(reinterpret_cast<const char*>(id), 128);
  });
  py::class_<Comm, std::shared_ptr<Comm>>(m, "Comm")
      .def(py::init<py::bytes, int, int, int>(), py::arg("unique_id"), py::arg("rank"),
           py::arg("world"), py::arg("device"));

  // ---- trainer ----
  py::class_<PyTrainer>(m, "Trainer")
      .def(py::init([](std::shared_ptr<Comm> comm, std::size_t table_capacity, int device,
                       const py::kwargs& kw) {
             auto p = std::make_unique<PyTrainer>();
             TrainerConfig c = config_from_kwargs(kw);
             c.adam.validate();  // config errors before any device work
             TierConfig t;
             t.cache_capacity = table_capacity;
             t.cold_path = kw.contains("cold_dir") ? kw["cold_dir"].cast<std::string>() : "/tmp/kpsim_b200_cold";
             t.hbm_capacity = table_capacity;
             t.device = device;
             p->store = std::make_unique<TieredStore>(t, c.model.embedding_dim);
             p->comm = comm;
             p->tr = std::make_unique<Trainer>(c, *p->store, nullptr, comm ? comm->c : nullptr);
             return p;
           }),
           py::arg("comm") = nullptr, py::arg("table_capacity") = (std::size_t)1 << 22,
           py::arg("device") = 0)
      .def("train_batch",
           [](PyTrainer& p, Arr<uint32_t> offs, Arr<uint64_t> keys, Arr<int32_t> labels,
              py::object slots, bool predict_first, py::object global_n, uint64_t global_first) {
             const uint32_t n = (uint32_t)labels.size();
             if ((uint32_t)offs.size() != n + 1) throw Error("offs must have n+1 entries");
             if ((uint64_t)keys.size() != offs.data()[n]) throw Error("keys size != offs[n]");
             Arr<uint16_t> sl;
             const uint16_t* sp = nullptr;
             if (!slots.is_none()) {
               sl = slots.cast<Arr<uint16_t>>();
               if (sl.size() != keys.size()) throw Error("slots size != keys size");
               sp = sl.data();
             }
             const uint64_t gn = global_n.is_none() ? n : global_n.cast<uint64_t>();
             CsrResult r;
             {
               py::gil_scoped_release rel;
               r = p.tr->train_csr(offs.data(), keys.data(), sp, labels.data(), n, gn, global_first,
                                   predict_first);
             }
             py::dict d;
             d["loss"] = r.loss;
             d["minibatch_steps"] = r.minibatch_steps;
             d["merges"] = r.merges;
             if (predict_first) {
               Arr<float> pr(n);
               std::copy(r.preds.begin(), r.preds.end(), pr.mutable_data());
               d["preds"] = pr;
               d["auc"] = r.auc ? py::object(py::float_(*r.auc)) : py::object(py::none());
               d["cumulative_auc"] =
                   r.cumulative_auc ? py::object(py::float_(*r.cumulative_auc)) : py::object(py::none());
             }
             return d;
           },
           py::arg("offs"), py::arg("keys"), py::arg("labels"), py::arg("slots") = py::none(),
           py::arg("predict_first") = false, py::arg("global_n") = py::none(),
           py::arg("global_first") = 0)
      .def("train_batch_device",
           [](PyTrainer& p, Arr<uint32_t> h_offs, uintptr_t d_offs, uintptr_t d_keys, uintptr_t d_slots,
              uintptr_t d_labels, uint32_t n, py::object global_n, uint64_t global_first,
              bool predict_first) {
             const uint64_t gn = global_n.is_none() ? n : global_n.cast<uint64_t>();
             CsrResult r;
             {
               py::gil_scoped_release rel;
               r = p.tr->train_csr_device(h_offs.data(), (const uint32_t*)d_offs,
                                          (const uint64_t*)d_keys, (const uint16_t*)d_slots,
                                          (const int32_t*)d_labels, n, gn, global_first,
                                          predict_first);
             }
             py::dict d;
             d["loss"] = r.loss;
             d["minibatch_steps"] = r.minibatch_steps;
             d["merges"] = r.merges;
             if (predict_first) {
               Arr<float> pr(n);
               std::copy(r.preds.begin(), r.preds.end(), pr.mutable_data());
               d["preds"] = pr;
             }
             return d;
           },
           py::arg("h_offs"), py::arg("d_offs"), py::arg("d_keys"), py::arg("d_slots"),
           py::arg("d_labels"), py::arg("n"), py::arg("global_n") = py::none(),
           py::arg("global_first") = 0, py::arg("predict_first") = false)
      .def("stage_batch",
           [](PyTrainer& p, int slot, Arr<uint32_t> offs, Arr<uint64_t> keys, Arr<int32_t> labels,
              py::object slots) {
             const uint32_t n = (uint32_t)labels.size();
             if ((uint32_t)offs.size() != n + 1) throw Error("offs must have n+1 entries");
             if ((uint64_t)keys.size() != offs.data()[n]) throw Error("keys size != offs[n]");
             Arr<uint16_t> sl;
             const uint16_t* sp = nullptr;
             if (!slots.is_none()) {
               sl = slots.cast<Arr<uint16_t>>();
               if (sl.size() != keys.size()) throw Error("slots size != keys size");
               sp = sl.data();
             }
             check(kp_trainer_stage_batch(p.tr->handle(), slot, offs.data(), keys.data(), sp,
                                          labels.data(), n));
             p.staged[slot] = py::make_tuple(offs, keys, labels, sl);
           },
           py::arg("slot"), py::arg("offs"), py::arg("keys"), py::arg("labels"),
           py::arg("slots") = py::none())
      .def("train_staged",
           [](PyTrainer& p, int slot, py::object global_n, uint64_t global_first, bool predict_first,
              uint32_t n_local) {
             kp_batch_result br{};
             std::vector<float> preds(predict_first ? n_local : 0);
             const uint64_t gn = global_n.is_none() ? n_local : global_n.cast<uint64_t>();
             {
               py::gil_scoped_release rel;
               check(kp_trainer_train_staged(p.tr->handle(), slot, gn, global_first,
                                             predict_first ? 1 : 0,
                                             predict_first ? preds.data() : nullptr, &br));
             }
             p.staged[slot] = py::none();  // its H2D has completed
             py::dict d;
             d["loss"] = br.loss;
             d["minibatch_steps"] = br.minibatch_steps;
             d["merges"] = br.merges;
             if (predict_first) {
               Arr<float> pr((py::ssize_t)preds.size());
               std::copy(preds.begin(), preds.end(), pr.mutable_data());
               d["preds"] = pr;
             }
             return d;
           },
           py::arg("slot"), py::arg("global_n") = py::none(), py::arg("global_first") = 0,
           py::arg("predict_first") = false, py::arg("n_local") = 0)
      .def("worker_state",
           [](PyTrainer& p, std::size_t l) {
             const auto st = p.tr->worker_states().at(l);
             py::dict d;
             d["x"] = Arr<double>((py::ssize_t)st.x.size(), st.x.data());
             d["m"] = Arr<double>((py::ssize_t)st.m.size(), st.m.data());
             d["v"] = Arr<double>((py::ssize_t)st.v.size(), st.v.data());
             d["v_bar"] = Arr<double>((py::ssize_t)st.v_bar.size(), st.v_bar.data());
             return d;
           })
      .def("xbar",
           [](PyTrainer& p) {
             const auto x = p.tr->dense_model();
             return Arr<double>((py::ssize_t)x.size(), x.data());
           })
      .def("table",
           [](PyTrainer& p) {
             uint64_t n = 0;
             kp_table* t = p.store->handle();
             check(kp_table_export(t, nullptr, nullptr, nullptr, nullptr, 0, &n));
             const py::ssize_t d = (py::ssize_t)p.store->embedding_dim();
             Arr<uint64_t> K((py::ssize_t)n);
             Arr<float> W({(py::ssize_t)n, d}), S1({(py::ssize_t)n, d}), S2({(py::ssize_t)n, d});
             if (n)
               check(kp_table_export(t, K.mutable_data(), W.mutable_data(), S1.mutable_data(),
                                     S2.mutable_data(), n, &n));
             return py::make_tuple(K, W, S1, S2);
           })
      .def("prefill",
           [](PyTrainer& p, uint64_t start, uint64_t step, uint64_t count) {
             py::gil_scoped_release rel;
             check(kp_table_insert_range(p.store->handle(), start, step, count, nullptr));
           },
           py::arg("start"), py::arg("step"), py::arg("count"))
      .def("profile",
           [](PyTrainer& p, bool enable) {
             double ms[7];
             uint64_t c[5] = {0};
             check(kp_trainer_profile(p.tr->handle(), enable ? 1 : 0, ms, c));
             py::dict d;
             const char* names[7] = {"dedup", "pull", "pool", "mlp", "push", "dense", "exchange"};
             for (int i = 0; i < 7; ++i) d[names[i]] = ms[i];
             d["steps"] = c[0];
             d["unique"] = c[1];
             d["occurrences"] = c[2];
             d["owner_unique"] = c[3];
             d["received"] = c[4];
             return d;
           },
           py::arg("enable"))
      .def("ledger", [](PyTrainer& p) { return ledger_to_dict(p.tr->ledger()); })
      .def("record_trajectory", [](PyTrainer& p, bool on) { p.tr->record_trajectory(on); },
           py::arg("on") = true)
      .def("dense_trajectory",
           [](PyTrainer& p) {
             const Trajectory tj = p.tr->dense_trajectory();
             py::list out;
             for (const auto& r : tj.steps) {
               py::dict d;
               d["step"] = r.step;
               d["merged"] = r.merged;
               d["loss"] = r.loss;
               d["a3_increment"] = r.a3_increment;
               d["x_bar"] = Arr<double>((py::ssize_t)r.x_bar.size(), r.x_bar.data());
               d["v_bar"] = Arr<double>((py::ssize_t)r.v_bar.size(), r.v_bar.data());
               out.append(d);
             }
             return out;
           })
      .def("stream",
           [](PyTrainer& p) {
             kp_stream s = nullptr;
             check(kp_trainer_stream(p.tr->handle(), &s));
             return reinterpret_cast<uintptr_t>(s);
           })
      .def_property_readonly("dense_dim", [](PyTrainer& p) { return p.tr->dense_dim(); })
      .def_property_readonly("completed_steps", [](PyTrainer& p) { return p.tr->completed_steps(); })
      .def_property_readonly("merges", [](PyTrainer& p) { return p.tr->metrics().merge_events; })
      .def_property_readonly("table_size", [](PyTrainer& p) { return p.store->cache_size(); });
}
