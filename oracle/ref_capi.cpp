// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrappers over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile). They let the Python tests,
// tests/golden/make_golden.py and bench.py's `cpu_baseline` / `--impl
// reference` leg drive the reference's own entry points:
//   fixtures::dense_classification / sparse_classification  (proj/src/fixtures.cpp:30-100)
//   sync::train / batch_gradient / epoch_batch               (proj/src/sync_engine.cpp:22-121)
//   hogwild::train / numa_dual_train / merge_models          (proj/src/async_engine.cpp:133-520)
//   dataset_loss                                             (proj/src/glm.cpp:85-94)
//   parse_libsvm / convert_layout / assign                   (proj/src/dataset.cpp:167-503)
// Only ref_sync_train_dump is a loop of our own: it replays sync::train's
// schedule (mt19937_64 + std::shuffle + std::sort, sync_engine.cpp:75-99)
// through the reference's batch_gradient + axpy so that the per-epoch model
// can be captured; it is checked bit-exact against sync::train in the tests.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "sgdbench/async_engine.hpp"
#include "sgdbench/dataset.hpp"
#include "sgdbench/fixtures.hpp"
#include "sgdbench/glm.hpp"
#include "sgdbench/linalg.hpp"
#include "sgdbench/sync_engine.hpp"
#include "sgdbench/simd_sim.hpp"
#include "sgdbench/harness.hpp"

using namespace sgdbench;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}
Dataset* D(void* h) { return static_cast<Dataset*>(h); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_fixture_dense(uint64_t n, uint64_t d, uint64_t seed, double noise) {
  return new Dataset(fixtures::dense_classification(n, d, seed, noise));
}

void* ref_fixture_sparse(uint64_t n, uint64_t d, double avg, uint64_t seed, double noise) {
  return new Dataset(fixtures::sparse_classification(n, d, avg, seed, noise));
}

void ref_ds_free(void* h) { delete D(h); }

void ref_ds_info(void* h, uint64_t* out /* n,d,layout,n_values,n_indices,n_offsets,pw */) {
  Dataset* ds = D(h);
  out[0] = ds->n_examples;
  out[1] = ds->n_features;
  out[2] = static_cast<uint64_t>(ds->layout);
  out[3] = ds->values.size();
  out[4] = ds->indices.size();
  out[5] = ds->row_offsets.size();
  out[6] = ds->padded_width;
}

void ref_ds_copy(void* h, double* labels, double* values, uint32_t* indices, uint64_t* offsets) {
  Dataset* ds = D(h);
  if (labels) std::copy(ds->labels.begin(), ds->labels.end(), labels);
  if (values) std::copy(ds->values.begin(), ds->values.end(), values);
  if (indices) std::copy(ds->indices.begin(), ds->indices.end(), indices);
  if (offsets)
    for (std::size_t i = 0; i < ds->row_offsets.size(); ++i) offsets[i] = ds->row_offsets[i];
}

void* ref_ds_from_arrays(uint64_t n, uint64_t d, int layout, const double* labels,
                         const double* values, uint64_t n_values, const uint32_t* indices,
                         uint64_t n_indices, const uint64_t* offsets, uint64_t n_offsets,
                         uint64_t padded_width) {
  auto* ds = new Dataset();
  ds->n_examples = n;
  ds->n_features = d;
  ds->layout = static_cast<Layout>(layout);
  ds->labels.assign(labels, labels + n);
  if (n_values) ds->values.assign(values, values + n_values);
  if (n_indices) ds->indices.assign(indices, indices + n_indices);
  for (uint64_t i = 0; i < n_offsets; ++i) ds->row_offsets.push_back(offsets[i]);
  ds->padded_width = padded_width;
  return ds;
}

// Rounds stored values to fp32 (the GPU storage precision) in place, so that
// oracle and device runs differ only in arithmetic.
void ref_ds_round_f32(void* h) {
  for (double& v : D(h)->values) v = static_cast<double>(static_cast<float>(v));
}

int ref_convert_layout(void* h, int layout, uint64_t max_dense_bytes, void** out) {
  try {
    *out = new Dataset(convert_layout(*D(h), static_cast<Layout>(layout),
                                      max_dense_bytes ? max_dense_bytes : kDefaultMaxDenseBytes));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_validate(void* h) {
  try {
    D(h)->validate();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Returns 0 ok, 1 ParseError (line in *line_out), 2 other error.
int ref_parse_libsvm(const char* text, uint64_t len, int64_t declared_d, void** out,
                     uint64_t* line_out) {
  try {
    std::istringstream in(std::string(text, len));
    std::optional<std::size_t> dd;
    if (declared_d >= 0) dd = static_cast<std::size_t>(declared_d);
    *out = new Dataset(parse_libsvm(in, dd));
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    *line_out = e.line_number;
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

uint64_t ref_write_libsvm(void* h, char* buf, uint64_t cap) {
  std::ostringstream os;
  write_libsvm(*D(h), os);
  std::string s = os.str();
  if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  return s.size();
}

double ref_dataset_loss(void* h, int task, const double* w) {
  return dataset_loss(static_cast<Task>(task), *D(h),
                      std::span<const double>(w, D(h)->n_features));
}

int ref_batch_gradient(void* h, int task, const uint32_t* rows, uint64_t n_rows, const double* w,
                       unsigned workers, double* g_out) {
  try {
    Dataset* ds = D(h);
    std::optional<Dataset> tr;
    if (ds->layout == Layout::DenseRowMajor) tr = transpose_dense(*ds);
    auto g = sync::batch_gradient(static_cast<Task>(task), *ds,
                                  std::span<const std::uint32_t>(rows, n_rows),
                                  std::span<const double>(w, ds->n_features), workers,
                                  tr ? &*tr : nullptr);
    std::copy(g.begin(), g.end(), g_out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_epoch_batch(void* h, int task, double* w, double alpha, unsigned workers) {
  std::vector<double> wv(w, w + D(h)->n_features);
  double norm = sync::epoch_batch(static_cast<Task>(task), *D(h), wv, alpha, workers);
  std::copy(wv.begin(), wv.end(), w);
  return norm;
}

// sync::train verbatim. Outputs: model (d), per-epoch loss and seconds.
int ref_sync_train(void* h, int task, double alpha, uint64_t batch_b, uint64_t epochs,
                   double decay, uint64_t seed, unsigned workers, int shuffle,
                   const double* init, double* model_out, double* losses, double* seconds,
                   uint64_t* n_epochs, int* diverged) {
  try {
    Hyperparams hp;
    hp.task = static_cast<Task>(task);
    hp.alpha = alpha;
    hp.batch_b = batch_b;
    hp.epochs = epochs;
    hp.step_decay = decay;
    sync::TrainOptions o;
    o.workers = workers;
    o.shuffle = shuffle != 0;
    if (init) o.initial_model.assign(init, init + D(h)->n_features);
    auto r = sync::train(hp.task, *D(h), hp, seed, o);
    std::copy(r.model.begin(), r.model.end(), model_out);
    *n_epochs = r.trace.epochs.size();
    for (std::size_t i = 0; i < r.trace.epochs.size(); ++i) {
      if (losses) losses[i] = r.trace.epochs[i].loss;
      if (seconds) seconds[i] = r.trace.epochs[i].seconds;
    }
    *diverged = r.trace.diverged ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Replays sync::train's schedule through the reference primitives and records
// the model after every epoch (models: epochs x d, row-major).
int ref_sync_train_dump(void* h, int task, double alpha, uint64_t batch_b, uint64_t epochs,
                        double decay, uint64_t seed, unsigned workers, int shuffle,
                        double* models, double* losses) {
  try {
    Dataset* ds = D(h);
    Hyperparams hp;
    hp.task = static_cast<Task>(task);
    hp.alpha = alpha;
    hp.batch_b = batch_b;
    hp.epochs = epochs;
    hp.step_decay = decay;
    hp.validate(ds->n_examples);
    std::optional<Dataset> tr;
    if (ds->layout == Layout::DenseRowMajor) tr = transpose_dense(*ds);
    std::vector<double> w(ds->n_features, 0.0);
    std::mt19937_64 rng(seed);
    std::vector<std::uint32_t> order(ds->n_examples);
    std::iota(order.begin(), order.end(), 0u);
    std::vector<std::uint32_t> batch;
    for (uint64_t epoch = 1; epoch <= epochs; ++epoch) {
      double a = hp.step_size(epoch);
      if (shuffle) std::shuffle(order.begin(), order.end(), rng);
      for (std::size_t lo = 0; lo < ds->n_examples; lo += batch_b) {
        std::size_t hi = std::min<std::size_t>(ds->n_examples, lo + batch_b);
        batch.assign(order.begin() + lo, order.begin() + hi);
        std::sort(batch.begin(), batch.end());
        auto g = sync::batch_gradient(hp.task, *ds, batch, w, workers, tr ? &*tr : nullptr);
        linalg::axpy(w, a, g, workers);
      }
      std::copy(w.begin(), w.end(), models + (epoch - 1) * ds->n_features);
      losses[epoch - 1] = dataset_loss(hp.task, *ds, w);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

struct RefPlanOut {
  int32_t access_path;
  int32_t replication;
  uint64_t k;
};

int ref_parse_plan(const char* text, RefPlanOut* out) {
  try {
    ExecutionPlan p = parse_plan(text);
    out->access_path = static_cast<int32_t>(p.access_path);
    out->replication = static_cast<int32_t>(p.model_replication);
    out->k = p.data_replication_k;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_validate_plan(const char* text, void* h) {
  try {
    validate_plan(parse_plan(text), *D(h));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// hogwild::train / numa_dual_train verbatim (dual != 0 selects the latter).
int ref_hogwild_train(void* h, int task, double alpha, uint64_t epochs, double decay,
                      const char* plan_text, uint64_t workers, uint64_t group_size,
                      int circular_offsets, uint64_t merge_period, int dual, const double* init,
                      double* model_out, double* losses, double* seconds, uint64_t* evals,
                      uint64_t* n_epochs) {
  try {
    Hyperparams hp;
    hp.task = static_cast<Task>(task);
    hp.alpha = alpha;
    hp.batch_b = 1;
    hp.epochs = epochs;
    hp.step_decay = decay;
    ExecutionPlan plan = parse_plan(plan_text);
    plan.workers = workers;
    plan.group_size = group_size;
    plan.circular_offsets = circular_offsets != 0;
    plan.merge_period_epochs = merge_period;
    hogwild::Options o;
    if (init) o.initial_model.assign(init, init + D(h)->n_features);
    auto r = dual ? hogwild::numa_dual_train(hp.task, *D(h), hp, plan, 0, o)
                  : hogwild::train(hp.task, *D(h), hp, plan, 0, o);
    std::copy(r.model.begin(), r.model.end(), model_out);
    *n_epochs = r.trace.epochs.size();
    for (std::size_t i = 0; i < r.trace.epochs.size(); ++i) {
      if (losses) losses[i] = r.trace.epochs[i].loss;
      if (seconds) seconds[i] = r.trace.epochs[i].seconds;
      if (evals) evals[i] = r.evals_per_epoch[i];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// assign(): lists flattened into out (total entries) with offsets (workers+1).
uint64_t ref_assign(uint64_t n, uint64_t workers, int strategy, uint64_t k, uint32_t* out,
                    uint64_t* offsets) {
  Assignment a = assign(n, workers, static_cast<Strategy>(strategy), k);
  uint64_t pos = 0;
  if (offsets) offsets[0] = 0;
  for (uint64_t w = 0; w < workers; ++w) {
    for (uint32_t id : a.per_worker[w]) {
      if (out) out[pos] = id;
      ++pos;
    }
    if (offsets) offsets[w + 1] = pos;
  }
  return pos;
}

void ref_merge_models(double* replicas, uint64_t r, uint64_t d, const double* weights,
                      double* merged) {
  std::vector<std::vector<double>> reps(r);
  for (uint64_t i = 0; i < r; ++i) reps[i].assign(replicas + i * d, replicas + (i + 1) * d);
  std::vector<double> wts;
  if (weights) wts.assign(weights, weights + r);
  auto m = hogwild::merge_models(reps, weights ? &wts : nullptr);
  std::copy(m.begin(), m.end(), merged);
}

double ref_point_coefficient(int task, double z, double y) {
  return point_gradient_coefficient(static_cast<Task>(task), z, y);
}

double ref_point_loss_from_margin(int task, double z, double y) {
  return point_loss_from_margin(static_cast<Task>(task), z, y);
}

unsigned ref_hardware_threads() { return std::thread::hardware_concurrency(); }

// linalg:: primitives (proj/src/linalg.cpp:26-183), verbatim calls.
int ref_matvec(void* h, const uint32_t* rows, uint64_t n_rows, const double* v, unsigned workers,
               double* out) {
  try {
    Dataset* ds = D(h);
    auto r = linalg::matvec(*ds, std::span<const std::uint32_t>(rows, n_rows),
                            std::span<const double>(v, ds->n_features), workers);
    std::copy(r.begin(), r.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_matvec_transposed(void* h, const uint32_t* rows, uint64_t n_rows, const double* a,
                          uint64_t a_len, unsigned workers, double* out) {
  try {
    Dataset* ds = D(h);
    auto r = linalg::matvec_transposed(*ds, std::span<const std::uint32_t>(rows, n_rows),
                                       std::span<const double>(a, a_len), workers);
    std::copy(r.begin(), r.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// op 0..4 = linalg::ElementwiseOp, 5 = ew_sigmoid, 6 = ew_hinge_indicator.
int ref_elementwise(int op, const double* a, const double* b, uint64_t n, double scalar,
                    unsigned workers, double* out) {
  try {
    std::span<const double> sa(a, n), sb(b, b ? n : 0);
    linalg::DenseVector r;
    if (op == 5)
      r = linalg::ew_sigmoid(sa, workers);
    else if (op == 6)
      r = linalg::ew_hinge_indicator(sa, workers);
    else
      r = linalg::elementwise(static_cast<linalg::ElementwiseOp>(op), sa, sb, scalar, workers);
    std::copy(r.begin(), r.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_axpy(double* w, double alpha, const double* g, uint64_t n, unsigned workers) {
  linalg::axpy(std::span<double>(w, n), alpha, std::span<const double>(g, n), workers);
}

// harness (proj/src/harness.cpp): run / estimate_optimal_loss /
// grid_search_alpha with the Sync or Async engine. losses_out: the first
// repetition's losses (n_out entries); epochs_to_out[4]: epochs to 10/5/2/1 %
// of the loss used (0 = not reached).
namespace {
harness::RunConfig harness_config(int engine, int task, double alpha, uint64_t batch_b,
                                  uint64_t epochs, const char* plan_text, uint64_t workers,
                                  uint64_t repetitions, uint64_t seed, double optimal_loss) {
  harness::RunConfig c;
  c.engine = engine == 0 ? harness::Engine::Sync : harness::Engine::Async;
  c.task = static_cast<Task>(task);
  c.hyper.task = c.task;
  c.hyper.alpha = alpha;
  c.hyper.batch_b = batch_b;
  c.hyper.epochs = epochs;
  c.workers = workers;
  if (plan_text && *plan_text) {
    ExecutionPlan p = parse_plan(plan_text);
    p.workers = workers;
    c.plan = p;
  }
  c.repetitions = repetitions;
  c.seed = seed;
  c.wall_clock_budget_seconds = 600.0;
  if (!std::isnan(optimal_loss)) c.optimal_loss = optimal_loss;
  return c;
}
void report_out(const harness::RunReport& r, double* losses_out, uint64_t* n_out, int64_t* epochs_to_out,
                double* l_used) {
  *n_out = r.trace.epochs.size();
  for (std::size_t i = 0; i < r.trace.epochs.size(); ++i) losses_out[i] = r.trace.epochs[i].loss;
  const int tols[4] = {10, 5, 2, 1};
  for (int k = 0; k < 4; ++k) {
    auto it = r.epochs_to.find(tols[k]);
    epochs_to_out[k] = it != r.epochs_to.end() && it->second ? static_cast<int64_t>(*it->second) : 0;
  }
  *l_used = r.optimal_loss_used;
}
}  // namespace

int ref_harness_run(void* h, int engine, int task, double alpha, uint64_t batch_b, uint64_t epochs,
                    const char* plan_text, uint64_t workers, uint64_t repetitions, uint64_t seed,
                    double optimal_loss, double* losses_out, uint64_t* n_out, int64_t* epochs_to_out,
                    double* l_used) {
  try {
    const auto c = harness_config(engine, task, alpha, batch_b, epochs, plan_text, workers, repetitions,
                                  seed, optimal_loss);
    report_out(harness::run(c, *D(h)), losses_out, n_out, epochs_to_out, l_used);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// estimate_optimal_loss with the default probes' construction
// (harness.cpp:275-289: batch GD over default_alpha_grid) but `epochs`
// epochs each instead of 100,000 under a wall-clock budget.
double ref_estimate_optimal_loss(void* h, int task, uint64_t epochs) {
  harness::clear_optimal_loss_cache();
  std::vector<harness::RunConfig> probes;
  for (double alpha : harness::default_alpha_grid()) {
    harness::RunConfig c;
    c.engine = harness::Engine::Sync;
    c.task = static_cast<Task>(task);
    c.hyper.task = c.task;
    c.hyper.alpha = alpha;
    c.hyper.batch_b = D(h)->n_examples;
    c.hyper.epochs = epochs;
    c.max_epochs = epochs;
    probes.push_back(std::move(c));
  }
  return harness::estimate_optimal_loss(static_cast<Task>(task), *D(h), probes, 600.0);
}

int ref_grid_search_alpha(void* h, int engine, int task, uint64_t batch_b, uint64_t epochs,
                          const char* plan_text, uint64_t workers, uint64_t seed, double optimal_loss,
                          const double* grid, uint64_t n_grid, double* best_alpha, int* converged,
                          double* l_used) {
  try {
    auto c = harness_config(engine, task, grid[0], batch_b, epochs, plan_text, workers, 1, seed,
                            optimal_loss);
    const auto r = harness::grid_search_alpha(c, *D(h), std::vector<double>(grid, grid + n_grid));
    *best_alpha = r.best_alpha;
    *converged = r.converged ? 1 : 0;
    *l_used = r.optimal_loss_used;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// warpsim (proj/src/simd_sim.cpp): one lockstep epoch of the warp simulator;
// stats_out = {attempted, surviving, memory_transactions, micro_steps}.
int ref_warpsim_epoch(void* h, int task, double alpha, const char* plan_text, uint64_t warp_width,
                      uint64_t segment_size, int offsets, double* w_inout, uint64_t* stats_out) {
  try {
    ExecutionPlan plan = parse_plan(plan_text);
    warpsim::WarpConfig warp;
    warp.warp_width = warp_width;
    warp.segment_size = segment_size;
    warp.offsets_enabled = offsets != 0;
    std::vector<double> w(w_inout, w_inout + D(h)->n_features);
    const auto st = warpsim::simulate_epoch(static_cast<Task>(task), *D(h), w, alpha, plan, warp, 0);
    std::copy(w.begin(), w.end(), w_inout);
    stats_out[0] = st.attempted_updates;
    stats_out[1] = st.surviving_updates;
    stats_out[2] = st.memory_transactions;
    stats_out[3] = st.micro_steps;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// warpsim::count_transactions over lanes given as one flat array + offsets.
uint64_t ref_count_transactions(const uint64_t* flat, const uint64_t* lane_off, uint64_t lanes,
                                uint64_t segment_size) {
  std::vector<std::vector<std::uint64_t>> streams(lanes);
  for (uint64_t l = 0; l < lanes; ++l) streams[l].assign(flat + lane_off[l], flat + lane_off[l + 1]);
  return warpsim::count_transactions(streams, segment_size);
}

}  // extern "C"
