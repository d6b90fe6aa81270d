// Host data layer of the engine (layer 3 of include/sgdb.h) and the
// sgdb:: C++ mirror of the reference's dataset / fixtures / plan API.
//
// This file is a PORT of the reference's host code, not a redesign (paths
// relative to /root/reference/proj): the bit-exactness contract leaves no
// freedom in parse order, rounding, <random> draw order, byte format or error
// text, so each function follows its reference counterpart step by step:
//   parse_libsvm / write_libsvm     <- src/dataset.cpp:145-230 (label
//                                      normalisation, error lines)
//   save_binary / load_binary       <- src/dataset.cpp:257-327 (sgdbds01)
//   transpose_dense, convert_layout,
//   append_bias_feature             <- src/dataset.cpp:333-446
//   assign                          <- src/dataset.cpp:470-503
//   fixtures                        <- src/fixtures.cpp:12-100
//   plan grammar / validation       <- src/async_engine.cpp:12-117 (same
//                                      error strings: part of the exception
//                                      contract)
// Fixtures and the mini-batch schedule go through libstdc++ <random> exactly
// as the reference does, which makes them bit-identical to it (checked in
// tests/test_host.py). None of this is on the CUDA hot path.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <istream>
#include <limits>
#include <numeric>
#include <ostream>
#include <random>
#include <sstream>
#include <unordered_set>

#include "errors.hpp"
#include "sgdb_b200.hpp"

namespace sgdb {

// ---- names ------------------------------------------------------------------
const char* task_name(Task t) { return t == Task::LR ? "lr" : "svm"; }
std::optional<Task> task_from_name(std::string_view name) {
  if (name == "lr") return Task::LR;
  if (name == "svm") return Task::SVM;
  return std::nullopt;
}
const char* layout_name(Layout layout) {
  switch (layout) {
    case Layout::DenseRowMajor: return "dense-row";
    case Layout::DenseColMajor: return "dense-col";
    case Layout::Csr: return "csr";
    case Layout::PaddedDense: return "padded";
  }
  return "?";
}
std::optional<Layout> layout_from_name(std::string_view name) {
  if (name == "dense-row") return Layout::DenseRowMajor;
  if (name == "dense-col") return Layout::DenseColMajor;
  if (name == "csr") return Layout::Csr;
  if (name == "padded") return Layout::PaddedDense;
  return std::nullopt;
}

// glm.cpp:16-22
void Hyperparams::validate(std::size_t n_examples) const {
  if (!(alpha > 0.0)) throw std::invalid_argument("alpha must be positive");
  if (batch_b < 1 || batch_b > n_examples)
    throw std::invalid_argument("batch size must be in [1, N]");
  if (epochs < 1) throw std::invalid_argument("epoch count must be >= 1");
  if (!(step_decay > 0.0)) throw std::invalid_argument("step decay must be positive");
}

// ---- trace ------------------------------------------------------------------
Clock::Clock()
    : now_seconds([] {
        using namespace std::chrono;
        return duration<double>(steady_clock::now().time_since_epoch()).count();
      }) {}
std::vector<double> LossTrace::losses() const {
  std::vector<double> out;
  out.reserve(epochs.size());
  for (const auto& e : epochs) out.push_back(e.loss);
  return out;
}
double LossTrace::min_loss() const {
  double m = epochs.empty() ? 0.0 : epochs.front().loss;
  for (const auto& e : epochs) m = std::min(m, e.loss);
  return m;
}
double LossTrace::total_seconds() const {
  double s = 0.0;
  for (const auto& e : epochs) s += e.seconds;
  return s;
}

// ---- Dataset ------------------------------------------------------------------
std::size_t Dataset::nnz() const {
  switch (layout) {
    case Layout::Csr: return values.size();
    case Layout::PaddedDense:
      return static_cast<std::size_t>(
          std::count_if(indices.begin(), indices.end(), [&](std::uint32_t j) { return j != pad_sentinel(); }));
    default:
      return static_cast<std::size_t>(
          std::count_if(values.begin(), values.end(), [](double v) { return v != 0.0; }));
  }
}

// dataset.cpp:61-101
void Dataset::validate() const {
  if (labels.size() != n_examples)
    throw std::invalid_argument("label count does not match example count");
  for (double y : labels)
    if (y != 1.0 && y != -1.0) throw std::invalid_argument("label not in {+1,-1}");
  switch (layout) {
    case Layout::Csr:
      if (row_offsets.size() != n_examples + 1)
        throw std::invalid_argument("csr row_offsets size mismatch");
      if (row_offsets.front() != 0 || row_offsets.back() != values.size())
        throw std::invalid_argument("csr row_offsets endpoints invalid");
      for (std::size_t i = 0; i + 1 < row_offsets.size(); ++i)
        if (row_offsets[i] > row_offsets[i + 1])
          throw std::invalid_argument("csr row_offsets not nondecreasing");
      if (indices.size() != values.size())
        throw std::invalid_argument("csr index/value size mismatch");
      for (std::uint32_t j : indices)
        if (j >= n_features) throw std::invalid_argument("csr feature index out of range");
      break;
    case Layout::PaddedDense:
      if (values.size() != n_examples * padded_width || indices.size() != n_examples * padded_width)
        throw std::invalid_argument("padded storage size mismatch");
      for (std::size_t i = 0; i < indices.size(); ++i) {
        if (indices[i] > pad_sentinel()) throw std::invalid_argument("padded feature index out of range");
        if (indices[i] == pad_sentinel() && values[i] != 0.0)
          throw std::invalid_argument("padded sentinel slot with nonzero value");
      }
      break;
    default:
      if (values.size() != n_examples * n_features)
        throw std::invalid_argument("dense storage size mismatch");
  }
}

sgdb_dataset_view Dataset::view() const {
  static_assert(sizeof(std::size_t) == sizeof(std::uint64_t));
  sgdb_dataset_view v{};
  v.n_examples = n_examples;
  v.n_features = n_features;
  v.layout = static_cast<int32_t>(layout);
  v.labels = labels.data();
  v.values = values.data();
  v.n_values = values.size();
  v.indices = indices.data();
  v.n_indices = indices.size();
  v.row_offsets = reinterpret_cast<const std::uint64_t*>(row_offsets.data());
  v.n_row_offsets = row_offsets.size();
  v.padded_width = padded_width;
  return v;
}

Dataset from_view(const sgdb_dataset_view& v) {
  Dataset ds;
  ds.n_examples = v.n_examples;
  ds.n_features = v.n_features;
  ds.layout = static_cast<Layout>(v.layout);
  if (v.n_examples) ds.labels.assign(v.labels, v.labels + v.n_examples);
  if (v.n_values) ds.values.assign(v.values, v.values + v.n_values);
  if (v.n_indices) ds.indices.assign(v.indices, v.indices + v.n_indices);
  for (std::uint64_t i = 0; i < v.n_row_offsets; ++i) ds.row_offsets.push_back(v.row_offsets[i]);
  ds.padded_width = v.padded_width;
  return ds;
}

namespace {

// Visits example e's (index, value) slots in storage order, padded sentinels
// skipped (dataset.hpp:176-187).
template <class F>
void visit(const Dataset& ds, std::size_t e, F&& f) {
  switch (ds.layout) {
    case Layout::DenseRowMajor:
      for (std::size_t j = 0; j < ds.n_features; ++j) f(static_cast<std::uint32_t>(j), ds.values[e * ds.n_features + j]);
      break;
    case Layout::DenseColMajor:
      for (std::size_t j = 0; j < ds.n_features; ++j) f(static_cast<std::uint32_t>(j), ds.values[j * ds.n_examples + e]);
      break;
    case Layout::Csr:
      for (std::size_t s = ds.row_offsets[e]; s < ds.row_offsets[e + 1]; ++s) f(ds.indices[s], ds.values[s]);
      break;
    case Layout::PaddedDense:
      for (std::size_t s = 0; s < ds.padded_width; ++s) {
        std::uint32_t j = ds.indices[s * ds.n_examples + e];
        if (j == ds.pad_sentinel()) continue;
        f(j, ds.values[s * ds.n_examples + e]);
      }
      break;
  }
}

double normalize_label(double raw) {  // dataset.cpp:147-151
  if (raw <= 0.0) return -1.0;
  if (raw == 2.0) return -1.0;
  return 1.0;
}

bool parse_double(std::string_view s, double& out) {
  if (!s.empty() && s.front() == '+') s.remove_prefix(1);
  if (s.empty()) return false;
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), out);
  return ec == std::errc{} && p == s.data() + s.size();
}

bool parse_index(std::string_view s, std::uint64_t& out) {
  auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), out);
  return ec == std::errc{} && p == s.data() + s.size();
}

Dataset to_csr(const Dataset& ds) {
  if (ds.layout == Layout::Csr) return ds;
  Dataset out;
  out.n_examples = ds.n_examples;
  out.n_features = ds.n_features;
  out.layout = Layout::Csr;
  out.labels = ds.labels;
  out.row_offsets.reserve(ds.n_examples + 1);
  out.row_offsets.push_back(0);
  for (std::size_t e = 0; e < ds.n_examples; ++e) {
    visit(ds, e, [&](std::uint32_t j, double x) {
      if (x == 0.0) return;
      out.indices.push_back(j);
      out.values.push_back(x);
    });
    out.row_offsets.push_back(out.values.size());
  }
  return out;
}

constexpr char kMagic[8] = {'s', 'g', 'd', 'b', 'd', 's', '0', '1'};

}  // namespace

// dataset.cpp:167-230
Dataset parse_libsvm(std::istream& in, std::optional<std::size_t> declared_d) {
  Dataset ds;
  ds.layout = Layout::Csr;
  ds.row_offsets.push_back(0);
  std::uint64_t max_index = 0;
  std::string line;
  std::size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (auto pos = line.find('#'); pos != std::string::npos) line.resize(pos);
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ' || line.back() == '\t'))
      line.pop_back();
    std::size_t start = line.find_first_not_of(" \t");
    if (start == std::string::npos) continue;
    std::string_view rest(line.data() + start, line.size() - start);
    auto next = [&rest]() -> std::string_view {
      std::size_t b = rest.find_first_not_of(" \t");
      if (b == std::string_view::npos) return {};
      std::size_t e = rest.find_first_of(" \t", b);
      std::string_view tok = rest.substr(b, e == std::string_view::npos ? e : e - b);
      rest = e == std::string_view::npos ? std::string_view{} : rest.substr(e);
      return tok;
    };
    std::string_view label_tok = next();
    double raw;
    if (!parse_double(label_tok, raw))
      throw ParseError("malformed label '" + std::string(label_tok) + "'", line_no);
    ds.labels.push_back(normalize_label(raw));
    std::uint64_t prev = 0;
    for (std::string_view tok = next(); !tok.empty(); tok = next()) {
      std::size_t colon = tok.find(':');
      if (colon == std::string_view::npos)
        throw ParseError("malformed feature '" + std::string(tok) + "', expected idx:val", line_no);
      std::uint64_t i1;
      double v;
      if (!parse_index(tok.substr(0, colon), i1) || i1 == 0)
        throw ParseError("malformed feature index in '" + std::string(tok) + "'", line_no);
      if (!parse_double(tok.substr(colon + 1), v))
        throw ParseError("malformed feature value in '" + std::string(tok) + "'", line_no);
      if (i1 <= prev) throw ParseError("feature indices not strictly increasing", line_no);
      prev = i1;
      if (declared_d && i1 > *declared_d)
        throw ParseError("feature index " + std::to_string(i1) + " exceeds declared " +
                             std::to_string(*declared_d),
                         line_no);
      max_index = std::max(max_index, i1);
      if (v == 0.0) continue;
      ds.values.push_back(v);
      ds.indices.push_back(static_cast<std::uint32_t>(i1 - 1));
    }
    ds.row_offsets.push_back(ds.values.size());
  }
  ds.n_examples = ds.labels.size();
  ds.n_features = declared_d ? *declared_d : static_cast<std::size_t>(max_index);
  return ds;
}

Dataset parse_libsvm_file(const std::string& path, std::optional<std::size_t> declared_d) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  return parse_libsvm(in, declared_d);
}

// dataset.cpp:238-249
void write_libsvm(const Dataset& ds, std::ostream& out) {
  char buf[64];
  for (std::size_t e = 0; e < ds.n_examples; ++e) {
    out << (ds.labels[e] > 0 ? "+1" : "-1");
    visit(ds, e, [&](std::uint32_t j, double x) {
      if (x == 0.0) return;
      std::snprintf(buf, sizeof(buf), " %u:%.17g", j + 1, x);
      out << buf;
    });
    out << '\n';
  }
}

// dataset.cpp:287-327
void save_binary(const Dataset& ds, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  auto pod = [&](auto v) { out.write(reinterpret_cast<const char*>(&v), sizeof(v)); };
  auto vec = [&](const auto& v) {
    pod(static_cast<std::uint64_t>(v.size()));
    out.write(reinterpret_cast<const char*>(v.data()),
              static_cast<std::streamsize>(v.size() * sizeof(v[0])));
  };
  out.write(kMagic, sizeof(kMagic));
  pod(static_cast<std::uint64_t>(ds.n_examples));
  pod(static_cast<std::uint64_t>(ds.n_features));
  pod(static_cast<std::uint32_t>(ds.layout));
  pod(static_cast<std::uint64_t>(ds.padded_width));
  vec(ds.labels);
  vec(ds.values);
  vec(ds.indices);
  vec(ds.row_offsets);
  if (!out) throw std::runtime_error("write failed: " + path);
}

Dataset load_binary(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  char magic[8];
  in.read(magic, sizeof(magic));
  if (!in || std::memcmp(magic, kMagic, sizeof(magic)) != 0)
    throw std::runtime_error("not a dataset cache file: " + path);
  auto pod = [&](auto& v) { in.read(reinterpret_cast<char*>(&v), sizeof(v)); };
  auto vec = [&](auto& v) {
    std::uint64_t n = 0;
    pod(n);
    if (!in) return;
    v.resize(n);
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(v[0])));
  };
  Dataset ds;
  std::uint64_t n = 0, d = 0, pw = 0;
  std::uint32_t layout = 0;
  pod(n);
  pod(d);
  pod(layout);
  pod(pw);
  ds.n_examples = n;
  ds.n_features = d;
  ds.layout = static_cast<Layout>(layout);
  ds.padded_width = pw;
  vec(ds.labels);
  vec(ds.values);
  vec(ds.indices);
  vec(ds.row_offsets);
  if (!in) throw std::runtime_error("truncated dataset cache file: " + path);
  ds.validate();
  return ds;
}

// dataset.cpp:406-446
Dataset transpose_dense(const Dataset& ds) {
  if (ds.layout != Layout::DenseRowMajor && ds.layout != Layout::DenseColMajor)
    throw std::invalid_argument("transpose_dense requires a dense layout");
  Dataset out;
  out.n_examples = ds.n_examples;
  out.n_features = ds.n_features;
  out.labels = ds.labels;
  out.layout = ds.layout == Layout::DenseRowMajor ? Layout::DenseColMajor : Layout::DenseRowMajor;
  const std::size_t rows = ds.layout == Layout::DenseRowMajor ? ds.n_examples : ds.n_features;
  const std::size_t cols = ds.layout == Layout::DenseRowMajor ? ds.n_features : ds.n_examples;
  out.values.resize(ds.values.size());
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t c = 0; c < cols; ++c) out.values[c * rows + r] = ds.values[r * cols + c];
  return out;
}

Dataset convert_layout(const Dataset& ds, Layout target, std::size_t max_dense_bytes) {
  if (ds.layout == target) return ds;
  if ((ds.layout == Layout::DenseRowMajor && target == Layout::DenseColMajor) ||
      (ds.layout == Layout::DenseColMajor && target == Layout::DenseRowMajor))
    return transpose_dense(ds);
  Dataset csr = to_csr(ds);
  if (target == Layout::Csr) return csr;
  const std::size_t n = csr.n_examples, d = csr.n_features;
  Dataset out;
  out.n_examples = n;
  out.n_features = d;
  out.layout = target;
  out.labels = csr.labels;
  if (target == Layout::PaddedDense) {
    std::size_t width = 0;
    for (std::size_t e = 0; e < n; ++e) width = std::max(width, csr.row_offsets[e + 1] - csr.row_offsets[e]);
    out.padded_width = width;
    out.values.assign(n * width, 0.0);
    out.indices.assign(n * width, out.pad_sentinel());
    for (std::size_t e = 0; e < n; ++e)
      for (std::size_t s = 0; s < csr.row_offsets[e + 1] - csr.row_offsets[e]; ++s) {
        out.values[s * n + e] = csr.values[csr.row_offsets[e] + s];
        out.indices[s * n + e] = csr.indices[csr.row_offsets[e] + s];
      }
    return out;
  }
  if (d != 0 && n > std::numeric_limits<std::size_t>::max() / d / sizeof(double))
    throw CapacityError("dense materialization overflows size arithmetic");
  const std::size_t bytes = n * d * sizeof(double);
  if (bytes > max_dense_bytes)
    throw CapacityError("dense materialization of " + std::to_string(n) + "x" + std::to_string(d) +
                        " needs " + std::to_string(bytes) + " bytes, above the " +
                        std::to_string(max_dense_bytes) + " byte cap");
  out.values.assign(n * d, 0.0);
  for (std::size_t e = 0; e < n; ++e)
    for (std::size_t s = csr.row_offsets[e]; s < csr.row_offsets[e + 1]; ++s) {
      const std::uint32_t j = csr.indices[s];
      if (target == Layout::DenseRowMajor) out.values[e * d + j] = csr.values[s];
      else out.values[static_cast<std::size_t>(j) * n + e] = csr.values[s];
    }
  return out;
}

// dataset.cpp:448-468
Dataset append_bias_feature(const Dataset& ds) {
  Dataset out;
  out.n_examples = ds.n_examples;
  out.n_features = ds.n_features + 1;
  out.layout = Layout::Csr;
  out.labels = ds.labels;
  const auto bias = static_cast<std::uint32_t>(ds.n_features);
  out.row_offsets.push_back(0);
  for (std::size_t e = 0; e < ds.n_examples; ++e) {
    visit(ds, e, [&](std::uint32_t j, double x) {
      if (x == 0.0) return;
      out.indices.push_back(j);
      out.values.push_back(x);
    });
    out.indices.push_back(bias);
    out.values.push_back(1.0);
    out.row_offsets.push_back(out.values.size());
  }
  return out;
}

// dataset.cpp:470-503
Assignment assign(std::size_t n, std::size_t workers, Strategy strategy, std::size_t k) {
  if (workers < 1) throw std::invalid_argument("assign: workers must be >= 1");
  if (n < 1) throw std::invalid_argument("assign: n must be >= 1");
  Assignment a;
  a.worker_count = workers;
  a.strategy = strategy;
  a.replication_k = k;
  a.per_worker.resize(workers);
  if (strategy == Strategy::RoundRobin) {
    for (std::size_t w = 0; w < workers; ++w)
      for (std::size_t i = w; i < n; i += workers) a.per_worker[w].push_back(static_cast<std::uint32_t>(i));
  } else {
    const std::size_t chunk = (n + workers - 1) / workers;
    for (std::size_t w = 0; w < workers; ++w)
      for (std::size_t i = w * chunk; i < std::min(n, (w + 1) * chunk); ++i)
        a.per_worker[w].push_back(static_cast<std::uint32_t>(i));
  }
  if (k > 0)
    for (auto& list : a.per_worker) {
      if (list.empty()) continue;
      const std::size_t boundary = static_cast<std::size_t>(list.back()) + 1;
      for (std::size_t i = 0; i < k; ++i) list.push_back(static_cast<std::uint32_t>((boundary + i) % n));
    }
  return a;
}

// fixtures.cpp:12-100 — same <random> draws in the same order.
namespace fixtures {
namespace {
std::vector<double> hidden_model(std::size_t d, std::mt19937_64& rng) {
  std::normal_distribution<double> normal(0.0, 1.0);
  std::vector<double> w(d);
  for (double& v : w) v = normal(rng);
  return w;
}
double label_for(double z, double noise, std::mt19937_64& rng) {
  double y = z >= 0.0 ? 1.0 : -1.0;
  if (noise > 0.0) {
    std::uniform_real_distribution<double> u(0.0, 1.0);
    if (u(rng) < noise) y = -y;
  }
  return y;
}
}  // namespace

Dataset dense_classification(std::size_t n, std::size_t d, std::uint64_t seed, double noise) {
  std::mt19937_64 rng(seed);
  std::vector<double> w_true = hidden_model(d, rng);
  std::uniform_real_distribution<double> uval(-1.0, 1.0);
  Dataset ds;
  ds.n_examples = n;
  ds.n_features = d;
  ds.layout = Layout::DenseRowMajor;
  ds.values.resize(n * d);
  ds.labels.resize(n);
  for (std::size_t e = 0; e < n; ++e) {
    double z = 0.0;
    for (std::size_t j = 0; j < d; ++j) {
      const double v = uval(rng);
      ds.values[e * d + j] = v;
      z += v * w_true[j];
    }
    ds.labels[e] = label_for(z, noise, rng);
  }
  return ds;
}

Dataset sparse_classification(std::size_t n, std::size_t d, double avg_nnz, std::uint64_t seed,
                              double noise) {
  std::mt19937_64 rng(seed);
  std::vector<double> w_true = hidden_model(d, rng);
  std::uniform_real_distribution<double> uval(-1.0, 1.0);
  std::uniform_real_distribution<double> u01(std::nextafter(0.0, 1.0), 1.0);
  std::uniform_int_distribution<std::uint32_t> uidx(0, static_cast<std::uint32_t>(d - 1));
  const double x_m = avg_nnz / 2.0;  // Pareto(x_m, 2) has mean avg_nnz
  const auto max_nnz = static_cast<std::size_t>(
      std::min<double>(static_cast<double>(d), std::max(1.0, 20.0 * avg_nnz)));
  Dataset ds;
  ds.n_examples = n;
  ds.n_features = d;
  ds.layout = Layout::Csr;
  ds.labels.resize(n);
  ds.row_offsets.reserve(n + 1);
  ds.row_offsets.push_back(0);
  ds.values.reserve(static_cast<std::size_t>(n * avg_nnz * 1.05));
  ds.indices.reserve(static_cast<std::size_t>(n * avg_nnz * 1.05));
  std::vector<std::uint32_t> row;
  std::unordered_set<std::uint32_t> seen;
  for (std::size_t e = 0; e < n; ++e) {
    const double pareto = x_m / std::sqrt(u01(rng));
    const std::size_t nnz =
        std::clamp<std::size_t>(static_cast<std::size_t>(std::lround(pareto)), 1, max_nnz);
    row.clear();
    seen.clear();
    while (row.size() < nnz) {
      const std::uint32_t j = uidx(rng);
      if (seen.insert(j).second) row.push_back(j);
    }
    std::sort(row.begin(), row.end());
    double z = 0.0;
    for (std::uint32_t j : row) {
      const double v = uval(rng);
      ds.indices.push_back(j);
      ds.values.push_back(v);
      z += v * w_true[j];
    }
    ds.row_offsets.push_back(ds.values.size());
    ds.labels[e] = label_for(z, noise, rng);
  }
  return ds;
}
}  // namespace fixtures

// ---- plan grammar (async_engine.cpp:12-117) -------------------------------------
const char* access_path_name(AccessPath p) {
  switch (p) {
    case AccessPath::RowRR: return "row-rr";
    case AccessPath::RowCh: return "row-ch";
    case AccessPath::ColRR: return "col-rr";
    case AccessPath::ColCh: return "col-ch";
  }
  return "?";
}
const char* replication_name(ModelReplication r) {
  switch (r) {
    case ModelReplication::Kernel: return "kernel";
    case ModelReplication::Block: return "block";
    case ModelReplication::Thread: return "thread";
    case ModelReplication::Example: return "example";
  }
  return "?";
}
Strategy plan_strategy(AccessPath p) {
  return (p == AccessPath::RowRR || p == AccessPath::ColRR) ? Strategy::RoundRobin : Strategy::Chunk;
}

namespace {
std::string trim(std::string_view s) {
  std::size_t b = s.find_first_not_of(" \t");
  if (b == std::string_view::npos) return {};
  std::size_t e = s.find_last_not_of(" \t");
  return std::string(s.substr(b, e - b + 1));
}
}  // namespace

ExecutionPlan parse_plan(std::string_view text) {
  std::vector<std::string> tok;
  std::string cur;
  for (char ch : text) {
    if (ch == ':' || ch == '+') {
      tok.push_back(trim(cur));
      cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  tok.push_back(trim(cur));
  if (tok.size() != 3)
    throw std::invalid_argument("plan '" + std::string(text) +
                                "' must have three parts: <access>:<replication>:<k>");
  ExecutionPlan plan;
  if (tok[0] == "row-rr") plan.access_path = AccessPath::RowRR;
  else if (tok[0] == "row-ch") plan.access_path = AccessPath::RowCh;
  else if (tok[0] == "col-rr") plan.access_path = AccessPath::ColRR;
  else if (tok[0] == "col-ch") plan.access_path = AccessPath::ColCh;
  else throw std::invalid_argument("unknown access path '" + tok[0] + "'");
  if (tok[1] == "kernel") plan.model_replication = ModelReplication::Kernel;
  else if (tok[1] == "block") plan.model_replication = ModelReplication::Block;
  else if (tok[1] == "thread") plan.model_replication = ModelReplication::Thread;
  else if (tok[1] == "example") plan.model_replication = ModelReplication::Example;
  else throw std::invalid_argument("unknown model replication '" + tok[1] + "'");
  std::string k = tok[2];
  if (k == "no-rep") k = "0";
  else if (k.rfind("rep-", 0) == 0) k = k.substr(4);
  try {
    std::size_t pos = 0;
    long long v = std::stoll(k, &pos);
    if (pos != k.size() || v < 0) throw std::invalid_argument("");
    plan.data_replication_k = static_cast<std::size_t>(v);
  } catch (...) {
    throw std::invalid_argument("bad replication factor '" + tok[2] + "'");
  }
  return plan;
}

std::string plan_to_string(const ExecutionPlan& plan) {
  return std::string(access_path_name(plan.access_path)) + ":" +
         replication_name(plan.model_replication) + ":" + std::to_string(plan.data_replication_k);
}

namespace {
void validate_plan_layout(const ExecutionPlan& plan, Layout layout) {
  if (plan.workers < 1) throw std::invalid_argument("plan needs at least one worker");
  if (plan.group_size < 1) throw std::invalid_argument("group size must be >= 1");
  const bool col = plan.access_path == AccessPath::ColRR || plan.access_path == AccessPath::ColCh;
  if (col && layout == Layout::Csr)
    throw std::invalid_argument("column access paths on sparse data require the padded dense layout");
  if (col && layout == Layout::DenseRowMajor)
    throw std::invalid_argument("column access paths require column-major dense storage");
  if (!col && layout == Layout::DenseColMajor)
    throw std::invalid_argument("row access paths require row-major dense storage");
  if (plan.model_replication == ModelReplication::Example &&
      !(layout == Layout::Csr || layout == Layout::PaddedDense))
    throw std::invalid_argument("example replication requires a sparse layout");
}
}  // namespace

void validate_plan(const ExecutionPlan& plan, const Dataset& ds) { validate_plan_layout(plan, ds.layout); }

sgdb_plan to_c(const ExecutionPlan& p) {
  sgdb_plan c{};
  c.access_path = static_cast<int32_t>(p.access_path);
  c.replication = static_cast<int32_t>(p.model_replication);
  c.data_replication_k = p.data_replication_k;
  c.workers = p.workers;
  c.group_size = p.group_size;
  c.circular_offsets = p.circular_offsets ? 1 : 0;
  c.merge_period_epochs = p.merge_period_epochs;
  c.lanes_per_worker = p.lanes_per_worker;
  return c;
}

ExecutionPlan from_c(const sgdb_plan& c) {
  ExecutionPlan p;
  p.access_path = static_cast<AccessPath>(c.access_path);
  p.model_replication = static_cast<ModelReplication>(c.replication);
  p.data_replication_k = c.data_replication_k;
  p.workers = c.workers;
  p.group_size = c.group_size;
  p.circular_offsets = c.circular_offsets != 0;
  p.merge_period_epochs = c.merge_period_epochs;
  p.lanes_per_worker = c.lanes_per_worker;
  return p;
}

}  // namespace sgdb

// ---- C-ABI: host helpers ------------------------------------------------------------

struct sgdb_host_dataset {
  sgdb::Dataset ds;
};

struct sgdb_schedule {
  std::mt19937_64 rng;
  std::vector<std::uint32_t> order;
  bool shuffle;
};

namespace {
sgdb_host_dataset* wrap(sgdb::Dataset&& ds) {
  auto* h = new sgdb_host_dataset();
  h->ds = std::move(ds);
  return h;
}
void need(const void* p) {
  if (!p) throw std::invalid_argument("null argument");
}
}  // namespace

extern "C" {

sgdb_status sgdb_fixture_dense(uint64_t n, uint64_t d, uint64_t seed, double noise,
                               sgdb_host_dataset** out) {
  return sgdb_guard([&] {
    need(out);
    *out = wrap(sgdb::fixtures::dense_classification(n, d, seed, noise));
  });
}

sgdb_status sgdb_fixture_sparse(uint64_t n, uint64_t d, double avg, uint64_t seed, double noise,
                                sgdb_host_dataset** out) {
  return sgdb_guard([&] {
    need(out);
    if (d == 0) throw std::invalid_argument("sparse fixture needs d >= 1");
    *out = wrap(sgdb::fixtures::sparse_classification(n, d, avg, seed, noise));
  });
}

sgdb_status sgdb_parse_libsvm(const char* text, uint64_t len, int64_t declared_d,
                              sgdb_host_dataset** out, uint64_t* error_line) {
  sgdb_status st = sgdb_guard([&] {
    need(out);
    std::istringstream in(std::string(text ? text : "", len));
    std::optional<std::size_t> dd;
    if (declared_d >= 0) dd = static_cast<std::size_t>(declared_d);
    *out = wrap(sgdb::parse_libsvm(in, dd));
  });
  if (st == SGDB_ERR_PARSE && error_line) *error_line = sgdb::detail::parse_line();
  return st;
}

sgdb_status sgdb_write_libsvm(const sgdb_dataset_view* view, char* buf, uint64_t cap,
                              uint64_t* len_out) {
  return sgdb_guard([&] {
    need(view);
    std::ostringstream os;
    sgdb::write_libsvm(sgdb::from_view(*view), os);
    const std::string s = os.str();
    if (len_out) *len_out = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  });
}

sgdb_status sgdb_save_binary(const sgdb_dataset_view* view, const char* path) {
  return sgdb_guard([&] {
    need(view);
    need(path);
    sgdb::save_binary(sgdb::from_view(*view), path);
  });
}

sgdb_status sgdb_load_binary(const char* path, sgdb_host_dataset** out) {
  return sgdb_guard([&] {
    need(path);
    need(out);
    *out = wrap(sgdb::load_binary(path));
  });
}

sgdb_status sgdb_convert_layout(const sgdb_dataset_view* view, int32_t target,
                                uint64_t max_dense_bytes, sgdb_host_dataset** out) {
  return sgdb_guard([&] {
    need(view);
    need(out);
    if (target < 0 || target > 3) throw std::invalid_argument("unknown target layout");
    *out = wrap(sgdb::convert_layout(sgdb::from_view(*view), static_cast<sgdb::Layout>(target),
                                     max_dense_bytes ? max_dense_bytes : sgdb::kDefaultMaxDenseBytes));
  });
}

sgdb_status sgdb_validate_dataset(const sgdb_dataset_view* view) {
  return sgdb_guard([&] {
    need(view);
    sgdb::from_view(*view).validate();
  });
}

sgdb_status sgdb_host_dataset_view(const sgdb_host_dataset* h, sgdb_dataset_view* out) {
  return sgdb_guard([&] {
    need(h);
    need(out);
    *out = h->ds.view();
  });
}

sgdb_status sgdb_host_dataset_free(sgdb_host_dataset* h) {
  return sgdb_guard([&] { delete h; });
}

sgdb_status sgdb_assign(uint64_t n, uint64_t workers, int32_t strategy, uint64_t k,
                        uint32_t* ids_out, uint64_t* offsets_out, uint64_t* total) {
  return sgdb_guard([&] {
    sgdb::Assignment a = sgdb::assign(n, workers, static_cast<sgdb::Strategy>(strategy), k);
    uint64_t pos = 0;
    if (offsets_out) offsets_out[0] = 0;
    for (uint64_t w = 0; w < workers; ++w) {
      for (std::uint32_t id : a.per_worker[w]) {
        if (ids_out) ids_out[pos] = id;
        ++pos;
      }
      if (offsets_out) offsets_out[w + 1] = pos;
    }
    if (total) *total = pos;
  });
}

sgdb_status sgdb_parse_plan(const char* text, sgdb_plan* out) {
  return sgdb_guard([&] {
    need(text);
    need(out);
    *out = sgdb::to_c(sgdb::parse_plan(text));
  });
}

sgdb_status sgdb_plan_to_string(const sgdb_plan* plan, char* buf, uint64_t cap) {
  return sgdb_guard([&] {
    need(plan);
    const std::string s = sgdb::plan_to_string(sgdb::from_c(*plan));
    if (!buf || cap < s.size() + 1) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

sgdb_status sgdb_validate_plan(const sgdb_plan* plan, int32_t layout) {
  return sgdb_guard([&] {
    need(plan);
    sgdb::validate_plan_layout(sgdb::from_c(*plan), static_cast<sgdb::Layout>(layout));
  });
}

sgdb_status sgdb_schedule_create(uint64_t seed, uint64_t n, int32_t shuffle, sgdb_schedule** out) {
  return sgdb_guard([&] {
    need(out);
    auto* s = new sgdb_schedule{std::mt19937_64(seed), std::vector<std::uint32_t>(n), shuffle != 0};
    std::iota(s->order.begin(), s->order.end(), 0u);
    *out = s;
  });
}

// One epoch of the schedule: sync_engine.cpp:84 (std::shuffle with the run's rng).
sgdb_status sgdb_schedule_next(sgdb_schedule* s, uint32_t* order_out) {
  return sgdb_guard([&] {
    need(s);
    if (s->shuffle) std::shuffle(s->order.begin(), s->order.end(), s->rng);
    if (order_out) std::copy(s->order.begin(), s->order.end(), order_out);
  });
}

sgdb_status sgdb_schedule_free(sgdb_schedule* s) {
  return sgdb_guard([&] { delete s; });
}

}  // extern "C"
