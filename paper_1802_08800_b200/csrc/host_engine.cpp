// Layer 2 of include/sgdb.h: the reference's epoch loops as host C++ over the
// device ops of layer 1, plus the sgdb:: C++ training API (sgdb_b200.hpp).
//
//   sync loop     <- sync::train        (proj/src/sync_engine.cpp:56-121)
//   hogwild loop  <- hogwild::train     (proj/src/async_engine.cpp:425-460)
//   dual loop     <- numa_dual_train    (proj/src/async_engine.cpp:462-520)
//
// The host keeps exactly the reference's loop semantics: mt19937_64(seed)
// schedule with one std::shuffle per epoch (untimed), compute-only epoch
// timing through the injectable clock, loss outside the timed region, the
// epoch hook, divergence reported in-band and the wall-clock budget checked
// after the loss.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool attached

#include "device.hpp"
#include "errors.hpp"
#include "sgdb_b200.hpp"

namespace sgdb {

void throw_status(sgdb_status st) {
  if (st == SGDB_OK) return;
  const std::string msg = sgdb_last_error();
  switch (st) {
    case SGDB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SGDB_ERR_DOMAIN: throw std::domain_error(msg);
    case SGDB_ERR_PARSE: throw ParseError(msg, detail::parse_line());
    case SGDB_ERR_CAPACITY: throw CapacityError(msg);
    case SGDB_ERR_UNSUPPORTED: throw detail::UnsupportedError(msg);
    case SGDB_ERR_CUDA: throw detail::DeviceError(msg);
    default: throw std::runtime_error(msg);
  }
}

namespace engine {

struct LoopOptions {
  std::function<double()> now;
  std::function<void(std::size_t, double)> hook;
  double max_seconds = 0.0;
  std::vector<double> initial_model;
  bool shuffle = true;
};

struct LoopResult {
  std::vector<double> model;
  LossTrace trace;
  std::vector<std::size_t> evals;
};

namespace {

struct ModelHandle {
  sgdb_model* m = nullptr;
  ModelHandle(sgdb_ctx* ctx, std::size_t d, const std::vector<double>& init) {
    throw_status(sgdb_model_create(ctx, d, init.empty() ? nullptr : init.data(), &m));
  }
  ~ModelHandle() { sgdb_model_free(m); }
  void reset(sgdb_ctx* ctx, const std::vector<double>& w) const {
    if (!w.empty()) throw_status(sgdb_model_set(ctx, m, w.data()));
  }
};

std::vector<double> initial(const LoopOptions& o, std::size_t d) {
  std::vector<double> w = o.initial_model.empty() ? std::vector<double>(d, 0.0) : o.initial_model;
  if (w.size() != d) throw std::invalid_argument("initial model dimension mismatch");
  return w;
}

double device_loss(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, Task task) {
  double l = 0.0;
  throw_status(sgdb_loss(ctx, ds, m, static_cast<int32_t>(task), &l));
  return l;
}

bool over_budget(const LoopOptions& o, double run_start) {
  return o.max_seconds > 0.0 && o.now() - run_start >= o.max_seconds;
}

}  // namespace

LoopResult sync_loop(sgdb_ctx* ctx, sgdb_dataset* ds, Task task, const Hyperparams& hyper,
                     std::uint64_t seed, const LoopOptions& o) {
  const std::size_t n = ds->n_global, d = ds->d;
  hyper.validate(n);
  if (n == 0) throw std::invalid_argument("cannot train on an empty dataset");
  LoopResult r;
  const std::vector<double> init = initial(o, d);
  ModelHandle model(ctx, d, init);
  const std::size_t b = hyper.batch_b;
  const bool full = b >= n;  // one full-batch step: membership is every row
  std::mt19937_64 rng(seed);
  std::vector<std::uint32_t> order;
  if (!full) {
    order.resize(n);
    std::iota(order.begin(), order.end(), 0u);
  }
  // Engine setup before the run clock starts, as the reference builds its
  // engine state before run_start (sync_engine.cpp / async_engine.cpp:436):
  // one untimed epoch allocates the lazily built per-dataset and per-model
  // device state (partition, partial buffers, captured step graph) and loads
  // the kernels; the model is then reset to its initial value.
  int32_t setup_finite = 1;
  throw_status(sgdb_sync_epoch(ctx, ds, model.m, static_cast<int32_t>(task), hyper.step_size(1),
                               full ? nullptr : order.data(), b, &setup_finite));
  model.reset(ctx, init);
  const double run_start = o.now();
  for (std::size_t epoch = 1; epoch <= hyper.epochs; ++epoch) {
    const double alpha = hyper.step_size(epoch);
    if (o.shuffle && !full) std::shuffle(order.begin(), order.end(), rng);
    const double t0 = o.now();
    int32_t finite = 1;
    nvtxRangePushA("sgdb sync epoch");
    throw_status(sgdb_sync_epoch(ctx, ds, model.m, static_cast<int32_t>(task), alpha,
                                 full ? nullptr : order.data(), b, &finite));
    nvtxRangePop();
    const double t1 = o.now();
    const double loss = device_loss(ctx, ds, model.m, task);
    r.trace.epochs.push_back({epoch, loss, t1 - t0});
    if (o.hook) o.hook(epoch, loss);
    if (!finite || !std::isfinite(loss)) {
      r.trace.diverged = true;
      r.trace.divergence_note = !finite ? "non-finite gradient in epoch " + std::to_string(epoch)
                                        : "non-finite loss after epoch " + std::to_string(epoch);
      break;
    }
    if (over_budget(o, run_start)) break;
  }
  r.model.resize(d);
  throw_status(sgdb_model_get(ctx, model.m, r.model.data()));
  return r;
}

LoopResult hogwild_loop(sgdb_ctx* ctx, sgdb_dataset* ds, Task task, const Hyperparams& hyper,
                        const ExecutionPlan& plan, const LoopOptions& o, bool dual) {
  const sgdb_plan cp = to_c(plan);
  throw_status(sgdb_validate_plan(&cp, ds->layout_in));
  if (ds->n_global == 0) throw std::invalid_argument("cannot train on an empty dataset");
  hyper.validate(ds->n_global);
  const std::size_t d = ds->d;
  LoopResult r;
  const std::vector<double> init = initial(o, d);
  ModelHandle a(ctx, d, init);
  std::unique_ptr<ModelHandle> b, merged;
  if (dual) {
    b = std::make_unique<ModelHandle>(ctx, d, init);
    merged = std::make_unique<ModelHandle>(ctx, d, init);
  }
  {  // untimed engine setup, as in sync_loop (the reference's Instance is
     // built before run_start, async_engine.cpp:436)
    uint64_t ea = 0;
    throw_status(sgdb_hogwild_epoch(ctx, ds, a.m, static_cast<int32_t>(task), hyper.step_size(1), &cp,
                                    &ea));
    if (dual) {
      throw_status(sgdb_hogwild_epoch(ctx, ds, b->m, static_cast<int32_t>(task), hyper.step_size(1), &cp,
                                      &ea));
      sgdb_model* pair[2] = {a.m, b->m};
      throw_status(sgdb_models_average(ctx, pair, 2, nullptr, merged->m, 1));
      b->reset(ctx, init);
      merged->reset(ctx, init);
    }
    a.reset(ctx, init);
  }
  const double run_start = o.now();
  for (std::size_t epoch = 1; epoch <= hyper.epochs; ++epoch) {
    const double alpha = hyper.step_size(epoch);
    const double t0 = o.now();
    uint64_t ea = 0, eb = 0;
    nvtxRangePushA("sgdb hogwild epoch");
    throw_status(sgdb_hogwild_epoch(ctx, ds, a.m, static_cast<int32_t>(task), alpha, &cp, &ea));
    sgdb_model* view = a.m;
    if (dual) {
      throw_status(sgdb_hogwild_epoch(ctx, ds, b->m, static_cast<int32_t>(task), alpha, &cp, &eb));
      const bool merge_due = plan.merge_period_epochs > 0 && epoch % plan.merge_period_epochs == 0;
      sgdb_model* pair[2] = {a.m, b->m};
      throw_status(sgdb_models_average(ctx, pair, 2, nullptr, merged->m, merge_due ? 1 : 0));
      view = merged->m;
    }
    // Multi-GPU (an NCCL communicator on the context): every rank trains its
    // replica, averaged across ranks every merge period (numa_dual_train's
    // merge generalised to N ranks, async_engine.cpp:478-501).
    int32_t rank = 0, nranks = 1;
    throw_status(sgdb_ctx_world(ctx, &rank, &nranks));
    if (!dual && nranks > 1 && plan.merge_period_epochs > 0 && epoch % plan.merge_period_epochs == 0)
      throw_status(sgdb_model_average_ranks(ctx, a.m, static_cast<uint64_t>(nranks)));
    throw_status(sgdb_ctx_synchronize(ctx));  // epoch work is stream-asynchronous
    nvtxRangePop();
    const double t1 = o.now();
    r.evals.push_back(static_cast<std::size_t>(ea + eb));
    const double loss = device_loss(ctx, ds, view, task);
    r.trace.epochs.push_back({epoch, loss, t1 - t0});
    if (o.hook) o.hook(epoch, loss);
    if (!std::isfinite(loss)) {
      r.trace.diverged = true;
      r.trace.divergence_note = "non-finite loss after epoch " + std::to_string(epoch);
      break;
    }
    if (over_budget(o, run_start)) break;
  }
  r.model.resize(d);
  throw_status(sgdb_model_get(ctx, dual ? merged->m : a.m, r.model.data()));
  return r;
}

LoopOptions from_c(const sgdb_train_options* c) {
  LoopOptions o;
  Clock default_clock;
  o.now = default_clock.now_seconds;
  if (!c) return o;
  if (c->clock) {
    auto fn = c->clock;
    void* user = c->clock_user;
    o.now = [fn, user] { return fn(user); };
  }
  if (c->epoch_hook) {
    auto fn = c->epoch_hook;
    void* user = c->hook_user;
    o.hook = [fn, user](std::size_t e, double l) { fn(user, e, l); };
  }
  o.max_seconds = c->max_seconds;
  if (c->initial_model) o.initial_model.assign(c->initial_model, c->initial_model + c->initial_model_len);
  o.shuffle = c->shuffle != 0;
  return o;
}

Hyperparams from_c(const sgdb_hyperparams* h) {
  if (!h) throw std::invalid_argument("null hyperparams");
  Hyperparams p;
  p.alpha = h->alpha;
  p.batch_b = h->batch_b;
  p.epochs = h->epochs;
  p.task = static_cast<Task>(h->task);
  p.step_decay = h->step_decay;
  return p;
}

void export_result(const LoopResult& r, double* model_out, sgdb_trace* t) {
  if (model_out) std::copy(r.model.begin(), r.model.end(), model_out);
  if (!t) return;
  t->count = r.trace.epochs.size();
  t->diverged = r.trace.diverged ? 1 : 0;
  std::snprintf(t->divergence_note, sizeof(t->divergence_note), "%s", r.trace.divergence_note.c_str());
  for (std::size_t i = 0; i < r.trace.epochs.size() && i < t->capacity; ++i) {
    if (t->epochs) t->epochs[i] = {r.trace.epochs[i].epoch, r.trace.epochs[i].loss, r.trace.epochs[i].seconds};
    if (t->evals_per_epoch && i < r.evals.size()) t->evals_per_epoch[i] = r.evals[i];
  }
}

}  // namespace engine

// ---- C++ API ------------------------------------------------------------------

Device::Device(int ordinal, void* stream) { throw_status(sgdb_ctx_create(ordinal, stream, &ctx_)); }
Device::~Device() { sgdb_ctx_destroy(ctx_); }
Device& Device::default_device() {
  static Device dev(0);
  return dev;
}

namespace {
std::atomic<int> g_precision{-1};
}

void set_default_precision(Precision p) { g_precision = static_cast<int>(p); }

Precision default_precision() {
  int p = g_precision.load();
  if (p < 0) {
    const char* e = std::getenv("SGDB_PRECISION");
    p = static_cast<int>(e && (std::string(e) == "exact" || std::string(e) == "fp64")
                             ? Precision::ExactFp64
                             : Precision::Fp32);
    g_precision = p;
  }
  return static_cast<Precision>(p);
}

DeviceDataset::DeviceDataset(Device& dev, const Dataset& ds, std::size_t row_base,
                             std::size_t n_global, Precision precision) {
  const sgdb_dataset_view v = ds.view();
  throw_status(sgdb_dataset_upload_ex(
      dev.get(), &v, row_base, n_global,
      precision == Precision::ExactFp64 ? SGDB_UPLOAD_EXACT_FP64 : 0u, &ds_));
}
DeviceDataset::~DeviceDataset() { sgdb_dataset_free(ds_); }

namespace {
engine::LoopOptions loop_opts(const Clock& clock, const std::function<void(std::size_t, double)>& hook,
                              double max_seconds, const std::vector<double>& init, bool shuffle) {
  engine::LoopOptions o;
  o.now = clock.now_seconds;
  o.hook = hook;
  o.max_seconds = max_seconds;
  o.initial_model = init;
  o.shuffle = shuffle;
  return o;
}
}  // namespace

double dataset_loss(Task task, const Dataset& ds, std::span<const double> w) {
  if (w.size() != ds.n_features) throw std::invalid_argument("model/dataset dim mismatch");
  Device& dev = Device::default_device();
  DeviceDataset dds(dev, ds);
  sgdb_model* m = nullptr;
  throw_status(sgdb_model_create(dev.get(), ds.n_features, w.data(), &m));
  double l = 0.0;
  sgdb_status st = sgdb_loss(dev.get(), dds.get(), m, static_cast<int32_t>(task), &l);
  sgdb_model_free(m);
  throw_status(st);
  return l;
}

namespace sync {

std::vector<double> batch_gradient(Task task, const Dataset& ds, std::span<const std::uint32_t> rows,
                                   std::span<const double> w, unsigned,
                                   const Dataset* transposed) {
  if (w.size() != ds.n_features) throw std::invalid_argument("matvec: dimension mismatch");
  Device& dev = Device::default_device();
  DeviceDataset dds(dev, ds);
  std::vector<double> g(ds.n_features, 0.0);
  throw_status(sgdb_batch_gradient(dev.get(), dds.get(), static_cast<int32_t>(task), rows.data(),
                                   rows.size(), w.data(), transposed != nullptr, g.data()));
  return g;
}

double epoch_batch(Task task, const Dataset& ds, std::vector<double>& w, double alpha, unsigned) {
  Device& dev = Device::default_device();
  DeviceDataset dds(dev, ds);
  sgdb_model* m = nullptr;
  throw_status(sgdb_model_create(dev.get(), ds.n_features, w.data(), &m));
  double norm = 0.0;
  sgdb_status st = sgdb_epoch_batch(dev.get(), dds.get(), m, static_cast<int32_t>(task), alpha, &norm);
  if (st == SGDB_OK) st = sgdb_model_get(dev.get(), m, w.data());
  sgdb_model_free(m);
  throw_status(st);
  return norm;
}

TrainResult train(Device& dev, DeviceDataset& dds, Task task, const Hyperparams& hyper,
                  std::uint64_t seed, const TrainOptions& options) {
  auto r = engine::sync_loop(dev.get(), dds.get(), task, hyper, seed,
                             loop_opts(options.clock, options.epoch_hook, options.max_seconds,
                                       options.initial_model, options.shuffle));
  return TrainResult{std::move(r.model), std::move(r.trace)};
}

TrainResult train(Task task, const Dataset& ds, const Hyperparams& hyper, std::uint64_t seed,
                  const TrainOptions& options) {
  hyper.validate(ds.n_examples);
  if (ds.n_examples == 0) throw std::invalid_argument("cannot train on an empty dataset");
  Device& dev = Device::default_device();
  DeviceDataset dds(dev, ds);
  return train(dev, dds, task, hyper, seed, options);
}

}  // namespace sync

namespace hogwild {

Result train(Device& dev, DeviceDataset& dds, Task task, const Hyperparams& hyper,
             const ExecutionPlan& plan, std::uint64_t, const Options& options) {
  auto r = engine::hogwild_loop(dev.get(), dds.get(), task, hyper, plan,
                                loop_opts(options.clock, options.epoch_hook, options.max_seconds,
                                          options.initial_model, true),
                                false);
  return Result{std::move(r.model), std::move(r.trace), std::move(r.evals)};
}

Result train(Task task, const Dataset& ds, const Hyperparams& hyper, const ExecutionPlan& plan,
             std::uint64_t seed, const Options& options) {
  validate_plan(plan, ds);
  if (ds.n_examples == 0) throw std::invalid_argument("cannot train on an empty dataset");
  hyper.validate(ds.n_examples);
  Device& dev = Device::default_device();
  DeviceDataset dds(dev, ds);
  return train(dev, dds, task, hyper, plan, seed, options);
}

Result numa_dual_train(Task task, const Dataset& ds, const Hyperparams& hyper,
                       const ExecutionPlan& plan, std::uint64_t, const Options& options) {
  validate_plan(plan, ds);
  if (ds.n_examples == 0) throw std::invalid_argument("cannot train on an empty dataset");
  hyper.validate(ds.n_examples);
  Device& dev = Device::default_device();
  DeviceDataset dds(dev, ds);
  auto r = engine::hogwild_loop(dev.get(), dds.get(), task, hyper, plan,
                                loop_opts(options.clock, options.epoch_hook, options.max_seconds,
                                          options.initial_model, true),
                                true);
  return Result{std::move(r.model), std::move(r.trace), std::move(r.evals)};
}

// merge_models (async_engine.cpp:133-156): a host utility over host vectors.
std::vector<double> merge_models(std::vector<std::vector<double>>& replicas,
                                 const std::vector<double>* weights) {
  if (replicas.empty()) throw std::invalid_argument("merge_models: no replicas");
  const std::size_t d = replicas.front().size();
  for (const auto& r : replicas)
    if (r.size() != d) throw std::invalid_argument("merge_models: dimension mismatch");
  double total = 0.0;
  if (weights) {
    if (weights->size() != replicas.size()) throw std::invalid_argument("merge_models: weight count mismatch");
    for (double w : *weights) total += w;
    if (total == 0.0) throw std::invalid_argument("merge_models: zero total weight");
  } else {
    total = static_cast<double>(replicas.size());
  }
  std::vector<double> merged(d, 0.0);
  for (std::size_t r = 0; r < replicas.size(); ++r) {
    const double w = weights ? (*weights)[r] : 1.0;
    for (std::size_t j = 0; j < d; ++j) merged[j] += w * replicas[r][j];
  }
  for (double& v : merged) v /= total;
  for (auto& r : replicas) r = merged;
  return merged;
}

}  // namespace hogwild
}  // namespace sgdb

// ---- C-ABI: whole runs ----------------------------------------------------------

namespace {
void check_trace(const sgdb_trace* t, std::size_t epochs) {
  if (t && t->capacity < epochs) throw std::invalid_argument("trace capacity below hyper.epochs");
}
}  // namespace

extern "C" {

sgdb_status sgdb_sync_train(sgdb_ctx* ctx, sgdb_dataset* ds, const sgdb_hyperparams* hyper,
                            uint64_t seed, const sgdb_train_options* options, double* model_out,
                            sgdb_trace* trace) {
  return sgdb_guard([&] {
    const sgdb::Hyperparams h = sgdb::engine::from_c(hyper);
    check_trace(trace, h.epochs);
    auto r = sgdb::engine::sync_loop(ctx, ds, static_cast<sgdb::Task>(hyper->task), h, seed,
                                     sgdb::engine::from_c(options));
    sgdb::engine::export_result(r, model_out, trace);
  });
}

sgdb_status sgdb_hogwild_train(sgdb_ctx* ctx, sgdb_dataset* ds, const sgdb_hyperparams* hyper,
                               const sgdb_plan* plan, uint64_t, const sgdb_train_options* options,
                               double* model_out, sgdb_trace* trace) {
  return sgdb_guard([&] {
    if (!plan) throw std::invalid_argument("null plan");
    const sgdb::Hyperparams h = sgdb::engine::from_c(hyper);
    check_trace(trace, h.epochs);
    auto r = sgdb::engine::hogwild_loop(ctx, ds, static_cast<sgdb::Task>(hyper->task), h,
                                        sgdb::from_c(*plan), sgdb::engine::from_c(options), false);
    sgdb::engine::export_result(r, model_out, trace);
  });
}

sgdb_status sgdb_numa_dual_train(sgdb_ctx* ctx, sgdb_dataset* ds, const sgdb_hyperparams* hyper,
                                 const sgdb_plan* plan, uint64_t, const sgdb_train_options* options,
                                 double* model_out, sgdb_trace* trace) {
  return sgdb_guard([&] {
    if (!plan) throw std::invalid_argument("null plan");
    const sgdb::Hyperparams h = sgdb::engine::from_c(hyper);
    check_trace(trace, h.epochs);
    auto r = sgdb::engine::hogwild_loop(ctx, ds, static_cast<sgdb::Task>(hyper->task), h,
                                        sgdb::from_c(*plan), sgdb::engine::from_c(options), true);
    sgdb::engine::export_result(r, model_out, trace);
  });
}

}  // extern "C"
