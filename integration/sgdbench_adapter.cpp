// Drop-in adapter: the reference's training entry points, implemented on the
// B200 engine through the C-ABI of include/sgdb.h.
//
// Compiled against the reference's own headers (proj/include/sgdbench), it
// defines exactly the symbols a maintainer replaces:
//   sgdbench::sync::batch_gradient   proj/include/sgdbench/sync_engine.hpp:33-36
//   sgdbench::sync::epoch_batch      proj/include/sgdbench/sync_engine.hpp:40-41
//   sgdbench::sync::train            proj/include/sgdbench/sync_engine.hpp:51-52
//   sgdbench::hogwild::train         proj/include/sgdbench/async_engine.hpp:96-97
//   sgdbench::hogwild::numa_dual_train proj/include/sgdbench/async_engine.hpp:102-104
//   sgdbench::linalg::{matvec, matvec_transposed, ew_*, elementwise, axpy}
//                                    proj/include/sgdbench/linalg.hpp:23-58
// Datasets are uploaded in the exact-fp64 mode (SGDB_UPLOAD_EXACT_FP64), so
// results are bit-identical to the reference's; SGDB_PRECISION=fp32 selects
// the fused fp32 kernels (the benchmarked path) instead.
// Multi-GPU (one process per GPU): with SGDB_NRANKS=N,
// SGDB_RANK=r and SGDB_NCCL_ID_FILE=<path on a shared filesystem> the context
// attaches the engine's own NCCL communicator (rank 0 writes the id, the
// others wait for it); sync::train / batch_gradient / epoch_batch then train
// on the rank's contiguous row shard with the gradient all-reduced every step,
// and hogwild::train runs each rank's shard with the replicas averaged every
// merge_period_epochs (numa_dual_train's merge generalised to N ranks,
// proj/src/async_engine.cpp:462-520). SGDB_DEVICE (default LOCAL_RANK, else
// r) picks the GPU. Sharding needs row-major dense or CSR data.
// Everything else (dataset I/O, plan grammar, harness, warp simulator) stays
// the reference's. See INTEGRATION.md for the two ways to link it (replace
// sync_engine.cpp / the engine half of async_engine.cpp, or interpose the
// shared library ahead of libsgdbench).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sgdb.h"
#include "sgdbench/async_engine.hpp"
#include "sgdbench/linalg.hpp"
#include "sgdbench/sync_engine.hpp"

namespace {

void throw_for(sgdb_status st) {
  if (st == SGDB_OK) return;
  const std::string msg = sgdb_last_error();
  switch (st) {
    case SGDB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SGDB_ERR_DOMAIN: throw std::domain_error(msg);
    case SGDB_ERR_CAPACITY: throw sgdbench::CapacityError(msg);
    default: throw std::runtime_error(msg);
  }
}

long env_long(const char* name, long fallback) {
  const char* e = std::getenv(name);
  return e && *e ? std::strtol(e, nullptr, 10) : fallback;
}

struct Ranks {
  int rank = 0, nranks = 1;
};
const Ranks& ranks() {
  static const Ranks r = [] {
    Ranks x;
    x.nranks = static_cast<int>(env_long("SGDB_NRANKS", 1));
    x.rank = static_cast<int>(env_long("SGDB_RANK", 0));
    if (x.nranks < 1 || x.rank < 0 || x.rank >= x.nranks)
      throw std::invalid_argument("SGDB_RANK / SGDB_NRANKS out of range");
    return x;
  }();
  return r;
}

// File rendezvous for the 128-byte NCCL id: rank 0 writes <path>.tmp and
// renames it (atomic), the others poll for <path>.
void exchange_id(const std::string& path, int rank, uint8_t* id) {
  if (rank == 0) {
    throw_for(sgdb_nccl_get_unique_id(id));
    const std::string tmp = path + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f || std::fwrite(id, 1, 128, f) != 128) throw std::runtime_error("cannot write " + tmp);
    std::fclose(f);
    if (std::rename(tmp.c_str(), path.c_str()) != 0) throw std::runtime_error("cannot publish " + path);
    return;
  }
  for (int t = 0; t < 6000; ++t) {  // up to 120 s
    if (FILE* f = std::fopen(path.c_str(), "rb")) {
      const size_t got = std::fread(id, 1, 128, f);
      std::fclose(f);
      if (got == 128) return;
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
  }
  throw std::runtime_error("timed out waiting for the NCCL id in " + path);
}

sgdb_ctx* context() {
  static sgdb_ctx* ctx = [] {
    const Ranks& r = ranks();
    const int device = static_cast<int>(env_long("SGDB_DEVICE", env_long("LOCAL_RANK", r.rank)));
    sgdb_ctx* c = nullptr;
    throw_for(sgdb_ctx_create(device, nullptr, &c));
    const char* idf = std::getenv("SGDB_NCCL_ID_FILE");
    if (r.nranks > 1 && !(idf && *idf))
      throw std::invalid_argument("SGDB_NRANKS > 1 needs SGDB_NCCL_ID_FILE for the NCCL id rendezvous");
    if (idf && *idf) {
      uint8_t id[128];
      exchange_id(idf, r.rank, id);
      throw_for(sgdb_ctx_init_nccl(c, r.nranks, r.rank, id));
    }
    return c;
  }();
  return ctx;
}

// sgdbench::Dataset and sgdb_dataset_view carry the same fields.
sgdb_dataset_view view_of(const sgdbench::Dataset& ds) {
  static_assert(sizeof(std::size_t) == sizeof(std::uint64_t));
  sgdb_dataset_view v{};
  v.n_examples = ds.n_examples;
  v.n_features = ds.n_features;
  v.layout = static_cast<int32_t>(ds.layout);
  v.labels = ds.labels.data();
  v.values = ds.values.data();
  v.n_values = ds.values.size();
  v.indices = ds.indices.data();
  v.n_indices = ds.indices.size();
  v.row_offsets = reinterpret_cast<const std::uint64_t*>(ds.row_offsets.data());
  v.n_row_offsets = ds.row_offsets.size();
  v.padded_width = ds.padded_width;
  return v;
}

uint32_t upload_flags() {
  static const uint32_t flags = [] {
    const char* e = std::getenv("SGDB_PRECISION");
    return e && std::string(e) == "fp32" ? 0u : SGDB_UPLOAD_EXACT_FP64;
  }();
  return flags;
}

// How a dataset is placed on a multi-rank context: the whole dataset on every
// rank, a row shard of one logical dataset (sync: ids stay global, the
// gradient is all-reduced), or a row shard trained as a dataset of its own
// (Hogwild replicas averaged across ranks).
enum class Placement { Whole, Shard, ShardAlone };

struct Uploaded {
  sgdb_dataset* ds = nullptr;
  std::vector<std::uint64_t> offs;  // rebased CSR row offsets of a shard
  explicit Uploaded(const sgdbench::Dataset& d, Placement place = Placement::Shard) {
    sgdb_dataset_view v = view_of(d);
    const Ranks& r = ranks();
    uint64_t base = 0, n_global = 0;
    if (r.nranks > 1 && place != Placement::Whole) {
      // The chunk rule of assign() (dataset.cpp:484-490): ceil(N / ranks) rows each.
      const uint64_t n = d.n_examples, chunk = (n + r.nranks - 1) / r.nranks;
      base = std::min<uint64_t>(n, chunk * static_cast<uint64_t>(r.rank));
      const uint64_t cnt = std::min<uint64_t>(n, base + chunk) - base;
      if (d.layout == sgdbench::Layout::DenseRowMajor) {
        v.values += base * d.n_features;
        v.n_values = cnt * d.n_features;
      } else if (d.layout == sgdbench::Layout::Csr) {
        const uint64_t o0 = d.row_offsets[base];
        offs.resize(cnt + 1);
        for (uint64_t i = 0; i <= cnt; ++i) offs[i] = d.row_offsets[base + i] - o0;
        v.values += o0;
        v.indices += o0;
        v.n_values = v.n_indices = offs[cnt];
        v.row_offsets = offs.data();
        v.n_row_offsets = cnt + 1;
      } else {
        throw std::invalid_argument("multi-GPU sharding needs row-major dense or CSR data");
      }
      v.labels += base;
      v.n_examples = cnt;
      n_global = place == Placement::Shard ? n : cnt;
      if (place == Placement::ShardAlone) base = 0;
    }
    throw_for(sgdb_dataset_upload_ex(context(), &v, base, n_global, upload_flags(), &ds));
  }
  ~Uploaded() { sgdb_dataset_free(ds); }
};

struct Model {
  sgdb_model* m = nullptr;
  Model(std::size_t d, const double* init) { throw_for(sgdb_model_create(context(), d, init, &m)); }
  ~Model() { sgdb_model_free(m); }
};

sgdb_plan plan_of(const sgdbench::ExecutionPlan& p) {
  sgdb_plan c{};
  c.access_path = static_cast<int32_t>(p.access_path);
  c.replication = static_cast<int32_t>(p.model_replication);
  c.data_replication_k = p.data_replication_k;
  c.workers = p.workers;
  c.group_size = p.group_size;
  c.circular_offsets = p.circular_offsets ? 1 : 0;
  c.merge_period_epochs = p.merge_period_epochs;
  c.lanes_per_worker = 0;
  return c;
}

sgdb_hyperparams hyper_of(sgdbench::Task task, const sgdbench::Hyperparams& h) {
  return sgdb_hyperparams{h.alpha, h.batch_b, h.epochs, static_cast<int32_t>(task), h.step_decay};
}

// Trampolines for the injectable Clock and epoch hook.
struct Callbacks {
  const sgdbench::Clock* clock;
  const std::function<void(std::size_t, double)>* hook;
};
double clock_tramp(void* u) { return static_cast<Callbacks*>(u)->clock->now_seconds(); }
void hook_tramp(void* u, uint64_t e, double l) { (*static_cast<Callbacks*>(u)->hook)(e, l); }

sgdb_train_options options_of(Callbacks& cb, bool shuffle, double max_seconds,
                              const std::vector<double>& init) {
  sgdb_train_options o{};
  o.workers = 1;
  o.shuffle = shuffle ? 1 : 0;
  o.max_seconds = max_seconds;
  o.initial_model = init.empty() ? nullptr : init.data();
  o.initial_model_len = init.size();
  o.clock = clock_tramp;
  o.clock_user = &cb;
  if (*cb.hook) {
    o.epoch_hook = hook_tramp;
    o.hook_user = &cb;
  }
  return o;
}

sgdbench::LossTrace trace_of(const sgdb_trace& t, const std::vector<sgdb_epoch_record>& recs) {
  sgdbench::LossTrace lt;
  for (std::size_t i = 0; i < t.count; ++i) lt.epochs.push_back({recs[i].epoch, recs[i].loss, recs[i].seconds});
  lt.diverged = t.diverged != 0;
  lt.divergence_note = t.divergence_note;
  return lt;
}

sgdbench::hogwild::Result run_hogwild(bool dual, sgdbench::Task task, const sgdbench::Dataset& ds,
                                      const sgdbench::Hyperparams& hyper,
                                      const sgdbench::ExecutionPlan& plan, std::uint64_t seed,
                                      const sgdbench::hogwild::Options& options) {
  sgdbench::validate_plan(plan, ds);
  if (ds.n_examples == 0) throw std::invalid_argument("cannot train on an empty dataset");
  hyper.validate(ds.n_examples);
  Uploaded up(ds, Placement::ShardAlone);
  const sgdb_hyperparams h = hyper_of(task, hyper);
  const sgdb_plan p = plan_of(plan);
  Callbacks cb{&options.clock, &options.epoch_hook};
  const sgdb_train_options o = options_of(cb, true, options.max_seconds, options.initial_model);
  std::vector<sgdb_epoch_record> recs(hyper.epochs);
  std::vector<uint64_t> evals(hyper.epochs);
  sgdb_trace t{};
  t.epochs = recs.data();
  t.evals_per_epoch = evals.data();
  t.capacity = hyper.epochs;
  sgdbench::hogwild::Result r;
  r.model.resize(ds.n_features);
  throw_for(dual ? sgdb_numa_dual_train(context(), up.ds, &h, &p, seed, &o, r.model.data(), &t)
                 : sgdb_hogwild_train(context(), up.ds, &h, &p, seed, &o, r.model.data(), &t));
  r.trace = trace_of(t, recs);
  r.evals_per_epoch.assign(evals.begin(), evals.begin() + static_cast<std::ptrdiff_t>(t.count));
  return r;
}

}  // namespace

namespace sgdbench {
namespace sync {

linalg::DenseVector batch_gradient(Task task, const Dataset& ds,
                                   std::span<const std::uint32_t> rows,
                                   std::span<const double> w, unsigned,
                                   const Dataset* transposed) {
  if (w.size() != ds.n_features) throw std::invalid_argument("matvec: dimension mismatch");
  Uploaded up(ds);
  linalg::DenseVector g(ds.n_features, 0.0);
  throw_for(sgdb_batch_gradient(context(), up.ds, static_cast<int32_t>(task), rows.data(),
                                rows.size(), w.data(), transposed != nullptr, g.data()));
  return g;
}

double epoch_batch(Task task, const Dataset& ds, std::vector<double>& w, double alpha, unsigned) {
  Uploaded up(ds);
  Model m(ds.n_features, w.data());
  double norm = 0.0;
  throw_for(sgdb_epoch_batch(context(), up.ds, m.m, static_cast<int32_t>(task), alpha, &norm));
  throw_for(sgdb_model_get(context(), m.m, w.data()));
  return norm;
}

TrainResult train(Task task, const Dataset& ds, const Hyperparams& hyper, std::uint64_t seed,
                  const TrainOptions& options) {
  hyper.validate(ds.n_examples);
  if (ds.n_examples == 0) throw std::invalid_argument("cannot train on an empty dataset");
  Uploaded up(ds);
  const sgdb_hyperparams h = hyper_of(task, hyper);
  Callbacks cb{&options.clock, &options.epoch_hook};
  const sgdb_train_options o = options_of(cb, options.shuffle, options.max_seconds,
                                          options.initial_model);
  std::vector<sgdb_epoch_record> recs(hyper.epochs);
  sgdb_trace t{};
  t.epochs = recs.data();
  t.capacity = hyper.epochs;
  TrainResult r;
  r.model.resize(ds.n_features);
  throw_for(sgdb_sync_train(context(), up.ds, &h, seed, &o, r.model.data(), &t));
  r.trace = trace_of(t, recs);
  return r;
}

}  // namespace sync

namespace hogwild {

Result train(Task task, const Dataset& ds, const Hyperparams& hyper, const ExecutionPlan& plan,
             std::uint64_t seed, const Options& options) {
  return run_hogwild(false, task, ds, hyper, plan, seed, options);
}

Result numa_dual_train(Task task, const Dataset& ds, const Hyperparams& hyper,
                       const ExecutionPlan& plan, std::uint64_t seed, const Options& options) {
  return run_hogwild(true, task, ds, hyper, plan, seed, options);
}

}  // namespace hogwild
namespace linalg {

DenseVector matvec(const Dataset& x, std::span<const std::uint32_t> rows, std::span<const double> v,
                   unsigned) {
  if (v.size() != x.n_features) throw std::invalid_argument("matvec: dimension mismatch");
  Uploaded up(x, Placement::Whole);
  DenseVector out(rows.empty() ? x.n_examples : rows.size(), 0.0);
  throw_for(sgdb_matvec(context(), up.ds, rows.data(), rows.size(), v.data(), v.size(),
                        out.data()));
  return out;
}

DenseVector matvec(const Dataset& x, std::span<const double> v, unsigned workers) {
  return matvec(x, std::span<const std::uint32_t>{}, v, workers);
}

DenseVector matvec_transposed(const Dataset& x, std::span<const std::uint32_t> rows,
                              std::span<const double> a_by_position, unsigned) {
  const std::size_t n = rows.empty() ? x.n_examples : rows.size();
  if (a_by_position.size() != n)
    throw std::invalid_argument("matvec_transposed: dimension mismatch");
  if (n == 0) return DenseVector(x.n_features, 0.0);
  Uploaded up(x, Placement::Whole);
  DenseVector out(x.n_features, 0.0);
  throw_for(sgdb_matvec_transposed(context(), up.ds, rows.data(), rows.size(),
                                   a_by_position.data(), a_by_position.size(), out.data()));
  return out;
}

DenseVector matvec_transposed(const Dataset& x, std::span<const double> a, unsigned workers) {
  return matvec_transposed(x, std::span<const std::uint32_t>{}, a, workers);
}

namespace {
DenseVector ew(int32_t op, std::span<const double> a, std::span<const double> b, double s) {
  DenseVector out(a.size());
  throw_for(sgdb_elementwise(context(), op, a.data(), b.empty() ? nullptr : b.data(), a.size(), s,
                             out.data()));
  return out;
}
void same_length(std::span<const double> a, std::span<const double> b, const char* what) {
  if (a.size() != b.size()) throw std::invalid_argument(std::string(what) + ": length mismatch");
}
}  // namespace

DenseVector ew_mul(std::span<const double> a, std::span<const double> b, unsigned) {
  same_length(a, b, "ew_mul");
  return ew(SGDB_EW_MUL, a, b, 0.0);
}
DenseVector ew_div(std::span<const double> a, std::span<const double> b, unsigned) {
  same_length(a, b, "ew_div");
  return ew(SGDB_EW_DIV, a, b, 0.0);
}
DenseVector ew_exp(std::span<const double> a, unsigned) { return ew(SGDB_EW_EXP, a, {}, 0.0); }
DenseVector ew_neg(std::span<const double> a, unsigned) { return ew(SGDB_EW_NEG, a, {}, 0.0); }
DenseVector ew_add_scalar(double s, std::span<const double> a, unsigned) {
  return ew(SGDB_EW_ADD_SCALAR, a, {}, s);
}
DenseVector ew_sigmoid(std::span<const double> a, unsigned) {
  return ew(SGDB_EW_SIGMOID, a, {}, 0.0);
}
DenseVector ew_hinge_indicator(std::span<const double> a, unsigned) {
  return ew(SGDB_EW_HINGE_INDICATOR, a, {}, 0.0);
}
DenseVector elementwise(ElementwiseOp op, std::span<const double> a, std::span<const double> b,
                        double scalar, unsigned workers) {
  switch (op) {
    case ElementwiseOp::Mul: return ew_mul(a, b, workers);
    case ElementwiseOp::Div: return ew_div(a, b, workers);
    case ElementwiseOp::Exp: return ew_exp(a, workers);
    case ElementwiseOp::Neg: return ew_neg(a, workers);
    case ElementwiseOp::AddScalar: return ew_add_scalar(scalar, a, workers);
  }
  throw std::invalid_argument("unknown elementwise op");
}

void axpy(std::span<double> w, double alpha, std::span<const double> g, unsigned) {
  if (w.size() != g.size()) throw std::invalid_argument("axpy: length mismatch");
  throw_for(sgdb_axpy(context(), w.data(), alpha, g.data(), w.size()));
}

}  // namespace linalg
}  // namespace sgdbench
