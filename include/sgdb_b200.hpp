// sgdb_b200.hpp — C++ host API of the B200 GLM SGD engine.
//
// Mirrors the reference's C++ interface (proj/include/sgdbench/*.hpp) name
// for name under namespace `sgdb` — same types, argument meaning and error
// behaviour — with the training entry points executed on the GPU through the
// C-ABI in sgdb.h. The reference header each declaration follows is cited
// beside it. INTEGRATION.md shows the adapter that binds these to the
// reference's own `sgdbench::` symbols so its harness runs unchanged.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "sgdb.h"

namespace sgdb {

// ---- glm.hpp ---------------------------------------------------------------
enum class Task { LR, SVM };                                   // glm.hpp:15
const char* task_name(Task t);
std::optional<Task> task_from_name(std::string_view name);

struct Hyperparams {                                            // glm.hpp:22-35
  double alpha = 0.01;
  std::size_t batch_b = 1;
  std::size_t epochs = 10;
  Task task = Task::LR;
  double step_decay = 1.0;
  double step_size(std::size_t epoch) const {
    double a = alpha;
    for (std::size_t i = 1; i < epoch; ++i) a *= step_decay;
    return a;
  }
  void validate(std::size_t n_examples) const;
};

// ---- dataset.hpp -----------------------------------------------------------
enum class Layout { DenseRowMajor, DenseColMajor, Csr, PaddedDense };  // dataset.hpp:13
const char* layout_name(Layout layout);
std::optional<Layout> layout_from_name(std::string_view name);

struct ParseError : std::runtime_error {                        // dataset.hpp:22-26
  ParseError(const std::string& msg, std::size_t line)
      : std::runtime_error(msg + " (line " + std::to_string(line) + ")"), line_number(line) {}
  std::size_t line_number;
};
struct CapacityError : std::runtime_error {                     // dataset.hpp:28-30
  using std::runtime_error::runtime_error;
};

struct Dataset {                                                // dataset.hpp:42-61
  std::size_t n_examples = 0;
  std::size_t n_features = 0;
  Layout layout = Layout::Csr;
  std::vector<double> labels;
  std::vector<double> values;
  std::vector<std::uint32_t> indices;
  std::vector<std::size_t> row_offsets;
  std::size_t padded_width = 0;

  std::uint32_t pad_sentinel() const { return static_cast<std::uint32_t>(n_features); }
  bool is_sparse_layout() const { return layout == Layout::Csr || layout == Layout::PaddedDense; }
  std::size_t nnz() const;
  void validate() const;
  sgdb_dataset_view view() const;  // borrowed C view of this object
};
Dataset from_view(const sgdb_dataset_view& v);

Dataset parse_libsvm(std::istream& in, std::optional<std::size_t> declared_d = std::nullopt);
Dataset parse_libsvm_file(const std::string& path,
                          std::optional<std::size_t> declared_d = std::nullopt);
void write_libsvm(const Dataset& ds, std::ostream& out);
void save_binary(const Dataset& ds, const std::string& path);
Dataset load_binary(const std::string& path);

inline constexpr std::size_t kDefaultMaxDenseBytes = std::size_t{2} << 30;
Dataset convert_layout(const Dataset& ds, Layout target,
                       std::size_t max_dense_bytes = kDefaultMaxDenseBytes);
Dataset append_bias_feature(const Dataset& ds);
Dataset transpose_dense(const Dataset& ds);

enum class Strategy { RoundRobin, Chunk };                      // dataset.hpp:133
struct Assignment {                                             // dataset.hpp:140-151
  std::size_t worker_count = 0;
  Strategy strategy = Strategy::Chunk;
  std::size_t replication_k = 0;
  std::vector<std::vector<std::uint32_t>> per_worker;
  std::size_t total_assigned() const {
    std::size_t t = 0;
    for (const auto& w : per_worker) t += w.size();
    return t;
  }
};
Assignment assign(std::size_t n, std::size_t workers, Strategy strategy, std::size_t k);

// ---- fixtures.hpp ----------------------------------------------------------
namespace fixtures {
Dataset dense_classification(std::size_t n, std::size_t d, std::uint64_t seed,
                             double label_noise = 0.1);
Dataset sparse_classification(std::size_t n, std::size_t d, double avg_nnz, std::uint64_t seed,
                              double label_noise = 0.1);
}  // namespace fixtures

// ---- trace.hpp -------------------------------------------------------------
struct Clock {                                                  // trace.hpp:14-19
  std::function<double()> now_seconds;
  Clock();
};
struct EpochRecord {
  std::size_t epoch = 0;
  double loss = 0.0;
  double seconds = 0.0;
};
struct LossTrace {                                              // trace.hpp:27-49
  std::vector<EpochRecord> epochs;
  bool diverged = false;
  std::string divergence_note;
  std::vector<double> losses() const;
  double final_loss() const { return epochs.empty() ? 0.0 : epochs.back().loss; }
  double min_loss() const;
  double total_seconds() const;
};

// ---- async_engine.hpp (plan grammar) ----------------------------------------
enum class AccessPath { RowRR, RowCh, ColRR, ColCh };
enum class ModelReplication { Kernel, Block, Thread, Example };
struct ExecutionPlan {                                          // async_engine.hpp:25-33
  AccessPath access_path = AccessPath::RowCh;
  ModelReplication model_replication = ModelReplication::Kernel;
  std::size_t data_replication_k = 0;
  std::size_t workers = 1;
  std::size_t group_size = 32;
  bool circular_offsets = true;
  std::size_t merge_period_epochs = 1;
  int lanes_per_worker = 0;  // device knob: 0 = auto
};
const char* access_path_name(AccessPath p);
const char* replication_name(ModelReplication r);
Strategy plan_strategy(AccessPath p);
ExecutionPlan parse_plan(std::string_view text);
std::string plan_to_string(const ExecutionPlan& plan);
void validate_plan(const ExecutionPlan& plan, const Dataset& ds);
sgdb_plan to_c(const ExecutionPlan& p);
ExecutionPlan from_c(const sgdb_plan& c);

// ---- device handles (RAII over sgdb.h) ---------------------------------------
class Device {
 public:
  explicit Device(int ordinal = 0, void* stream = nullptr);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  sgdb_ctx* get() const { return ctx_; }
  static Device& default_device();  // lazily created on device 0

 private:
  sgdb_ctx* ctx_ = nullptr;
};

// Arithmetic of device datasets: Fp32 = the fused fp32 kernels (default);
// ExactFp64 = SGDB_UPLOAD_EXACT_FP64, results bit-identical to the reference.
// The process default starts from the environment (SGDB_PRECISION=exact).
enum class Precision { Fp32, ExactFp64 };
void set_default_precision(Precision p);
Precision default_precision();

class DeviceDataset {
 public:
  DeviceDataset(Device& dev, const Dataset& ds, std::size_t row_base = 0,
                std::size_t n_global = 0, Precision precision = default_precision());
  ~DeviceDataset();
  DeviceDataset(const DeviceDataset&) = delete;
  DeviceDataset& operator=(const DeviceDataset&) = delete;
  sgdb_dataset* get() const { return ds_; }

 private:
  sgdb_dataset* ds_ = nullptr;
};

// Throws the reference's exception type for a failed status.
void throw_status(sgdb_status st);

double dataset_loss(Task task, const Dataset& ds, std::span<const double> w);  // glm.hpp:70

// ---- sync_engine.hpp ---------------------------------------------------------
namespace sync {
struct TrainOptions {                                           // sync_engine.hpp:15-25
  unsigned workers = 1;
  bool shuffle = true;
  Clock clock;
  std::function<void(std::size_t epoch, double loss)> epoch_hook;
  double max_seconds = 0.0;
  std::vector<double> initial_model;
};
struct TrainResult {
  std::vector<double> model;
  LossTrace trace;
};
std::vector<double> batch_gradient(Task task, const Dataset& ds,
                                   std::span<const std::uint32_t> rows,
                                   std::span<const double> w, unsigned workers = 1,
                                   const Dataset* transposed = nullptr);
double epoch_batch(Task task, const Dataset& ds, std::vector<double>& w, double alpha,
                   unsigned workers = 1);
TrainResult train(Task task, const Dataset& ds, const Hyperparams& hyper, std::uint64_t seed,
                  const TrainOptions& options = {});
// Same loop over an already uploaded dataset.
TrainResult train(Device& dev, DeviceDataset& dds, Task task, const Hyperparams& hyper,
                  std::uint64_t seed, const TrainOptions& options = {});
}  // namespace sync

// ---- async_engine.hpp ---------------------------------------------------------
namespace hogwild {
struct Options {                                                // async_engine.hpp:77-82
  Clock clock;
  std::function<void(std::size_t epoch, double loss)> epoch_hook;
  double max_seconds = 0.0;
  std::vector<double> initial_model;
};
struct Result {
  std::vector<double> model;
  LossTrace trace;
  std::vector<std::size_t> evals_per_epoch;
};
Result train(Task task, const Dataset& ds, const Hyperparams& hyper, const ExecutionPlan& plan,
             std::uint64_t seed, const Options& options = {});
Result numa_dual_train(Task task, const Dataset& ds, const Hyperparams& hyper,
                       const ExecutionPlan& plan, std::uint64_t seed, const Options& options = {});
Result train(Device& dev, DeviceDataset& dds, Task task, const Hyperparams& hyper,
             const ExecutionPlan& plan, std::uint64_t seed, const Options& options = {});
std::vector<double> merge_models(std::vector<std::vector<double>>& replicas,
                                 const std::vector<double>* weights = nullptr);
}  // namespace hogwild

}  // namespace sgdb
