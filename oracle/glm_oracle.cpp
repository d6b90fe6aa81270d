// TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into, or called by,
// the product path (paper_1802_08800_b200/). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg load it, and only as the checker.
//
// A from-scratch fp64 restatement of the reference's algorithms for the hot
// path, each function citing the reference file:line it follows (paths are
// relative to /root/reference/proj). It is compiled with g++ against the same
// libstdc++ as the reference so that <random> (mt19937_64, std::shuffle and
// the distributions) reproduces the reference's fixtures and mini-batch
// schedules bit for bit. It is PINNED by tests/test_oracle.py against
//   * the unmodified reference built in oracle/_ref (bit-exact, where present)
//   * the golden vectors in tests/golden/ (generated from that reference by
//     tests/golden/make_golden.py) and the reference tests' known answers.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

enum Layout { kDenseRow = 0, kDenseCol = 1, kCsr = 2, kPadded = 3 };
enum Task { kLR = 0, kSVM = 1 };

// Mirrors the field set of sgdbench::Dataset (include/sgdbench/dataset.hpp:42-61).
struct Data {
  uint64_t n = 0, d = 0;
  int layout = kCsr;
  std::vector<double> labels, values;
  std::vector<uint32_t> indices;
  std::vector<uint64_t> offsets;
  uint64_t pw = 0;
};

thread_local std::string g_err;

// include/sgdbench/math.hpp:10-16
double sigmoid(double u) {
  if (u <= 0.0) {
    double e = std::exp(u);
    return e / (1.0 + e);
  }
  return 1.0 / (1.0 + std::exp(-u));
}
// include/sgdbench/math.hpp:19-22
double softplus(double u) {
  if (u > 0.0) return u + std::log1p(std::exp(-u));
  return std::log1p(std::exp(u));
}
// src/glm.cpp:24-28
double loss_from_margin(int task, double z, double y) {
  double m = y * z;
  if (task == kLR) return softplus(-m);
  return m < 1.0 ? 1.0 - m : 0.0;
}
// src/glm.cpp:30-34
double coefficient(int task, double z, double y) {
  double m = y * z;
  if (task == kLR) return sigmoid(-m) * -y;
  return m < 1.0 ? -y : 0.0;
}

// Strided example view (src/dataset.cpp:103-132).
struct View {
  const double* val;
  const uint32_t* idx;
  uint64_t len, stride;
  double value(uint64_t s) const { return val[s * stride]; }
  uint32_t index(uint64_t s) const { return idx ? idx[s * stride] : static_cast<uint32_t>(s); }
};
View view(const Data& ds, uint64_t e) {
  switch (ds.layout) {
    case kDenseRow: return {ds.values.data() + e * ds.d, nullptr, ds.d, 1};
    case kDenseCol: return {ds.values.data() + e, nullptr, ds.d, ds.n};
    case kCsr: {
      uint64_t b = ds.offsets[e];
      return {ds.values.data() + b, ds.indices.data() + b, ds.offsets[e + 1] - b, 1};
    }
    default: return {ds.values.data() + e, ds.indices.data() + e, ds.pw, ds.n};
  }
}
// for_example: storage order, padded sentinels skipped (dataset.hpp:176-187).
template <class F>
void for_example(const Data& ds, uint64_t e, F&& f) {
  View v = view(ds, e);
  for (uint64_t s = 0; s < v.len; ++s) {
    uint32_t j = v.index(s);
    if (j == ds.d) continue;
    f(j, v.value(s));
  }
}

// src/glm.cpp:85-94 — sequential in example id order.
double dataset_loss(int task, const Data& ds, const double* w) {
  double total = 0.0;
  for (uint64_t e = 0; e < ds.n; ++e) {
    double z = 0.0;
    for_example(ds, e, [&](uint32_t j, double x) { z += x * w[j]; });
    total += loss_from_margin(task, z, ds.labels[e]);
  }
  return total;
}

// Dense storage transpose (src/dataset.cpp:422-446); content-only restatement.
Data transpose(const Data& ds) {
  Data out = ds;
  out.layout = ds.layout == kDenseRow ? kDenseCol : kDenseRow;
  uint64_t rows = ds.layout == kDenseRow ? ds.n : ds.d;
  uint64_t cols = ds.layout == kDenseRow ? ds.d : ds.n;
  for (uint64_t r = 0; r < rows; ++r)
    for (uint64_t c = 0; c < cols; ++c) out.values[c * rows + r] = ds.values[r * cols + c];
  return out;
}

// sync::batch_gradient (src/sync_engine.cpp:22-42) built from matvec
// (src/linalg.cpp:30-44), the elementwise chain (linalg.cpp:124-174) and
// matvec_transposed (linalg.cpp:50-109) with its exact summation order:
// column streaming for DenseColMajor, else 256-row dense partials combined by
// a fixed stride-doubling pairwise tree.
std::vector<double> batch_gradient(int task, const Data& ds, const std::vector<uint32_t>& rows,
                                   const double* w, const Data* transposed) {
  const uint64_t n = rows.size(), d = ds.d;
  std::vector<double> c(n);
  for (uint64_t p = 0; p < n; ++p) {
    double z = 0.0;
    for_example(ds, rows[p], [&](uint32_t j, double x) { z += x * w[j]; });
    double y = ds.labels[rows[p]];
    double m = y * z;
    if (task == kLR) {
      c[p] = sigmoid(-m) * (-y);
    } else {
      double active = m < 1.0 ? 1.0 : 0.0;
      c[p] = active * (-y);
    }
  }
  const Data& X = transposed ? *transposed : ds;
  std::vector<double> g(d, 0.0);
  if (n == 0) return g;
  if (X.layout == kDenseCol) {
    for (uint64_t j = 0; j < d; ++j) {
      const double* col = X.values.data() + j * X.n;
      double s = 0.0;
      for (uint64_t p = 0; p < n; ++p) s += c[p] * col[rows[p]];
      g[j] = s;
    }
    return g;
  }
  const uint64_t kBlock = 256;
  uint64_t nb = (n + kBlock - 1) / kBlock;
  std::vector<std::vector<double>> part(nb, std::vector<double>(d, 0.0));
  for (uint64_t b = 0; b < nb; ++b) {
    for (uint64_t p = b * kBlock; p < std::min(n, (b + 1) * kBlock); ++p) {
      double s = c[p];
      for_example(X, rows[p], [&](uint32_t j, double x) { part[b][j] += s * x; });
    }
  }
  for (uint64_t stride = 1; stride < nb; stride *= 2)
    for (uint64_t i = 0; i + stride < nb; i += 2 * stride)
      for (uint64_t j = 0; j < d; ++j) part[i][j] += part[i + stride][j];
  return part[0];
}

// assign (src/dataset.cpp:470-503).
std::vector<std::vector<uint32_t>> assign(uint64_t n, uint64_t workers, int rr, uint64_t k) {
  std::vector<std::vector<uint32_t>> lists(workers);
  if (rr) {
    for (uint64_t w = 0; w < workers; ++w)
      for (uint64_t i = w; i < n; i += workers) lists[w].push_back(static_cast<uint32_t>(i));
  } else {
    uint64_t chunk = (n + workers - 1) / workers;
    for (uint64_t w = 0; w < workers; ++w)
      for (uint64_t i = w * chunk; i < std::min(n, (w + 1) * chunk); ++i)
        lists[w].push_back(static_cast<uint32_t>(i));
  }
  if (k > 0)
    for (auto& l : lists) {
      if (l.empty()) continue;
      uint64_t boundary = static_cast<uint64_t>(l.back()) + 1;
      for (uint64_t i = 0; i < k; ++i) l.push_back(static_cast<uint32_t>((boundary + i) % n));
    }
  return lists;
}

// process_examples (src/async_engine.cpp:178-195): dot over ALL slots (padded
// sentinels read the guard slot w[d] == 0), coefficient, rotated update.
void process_examples(std::vector<double>& m, const Data& ds, int task,
                      const std::vector<uint32_t>& list, double alpha, bool offsets,
                      uint64_t wid) {
  for (uint32_t e : list) {
    View x = view(ds, e);
    double z = 0.0;
    for (uint64_t s = 0; s < x.len; ++s) z += x.value(s) * m[x.index(s)];
    double c = coefficient(task, z, ds.labels[e]);
    if (x.len == 0) continue;
    uint64_t s = offsets ? wid % x.len : 0;
    for (uint64_t i = 0; i < x.len; ++i) {
      uint32_t j = x.index(s);
      m[j] = m[j] - alpha * (c * x.value(s));
      if (++s == x.len) s = 0;
    }
  }
}

double step_size(double alpha, double decay, uint64_t epoch) {  // include/sgdbench/glm.hpp:29-33
  double a = alpha;
  for (uint64_t i = 1; i < epoch; ++i) a *= decay;
  return a;
}

Data* H(void* h) { return static_cast<Data*>(h); }

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// --- data handles -------------------------------------------------------------

void* orc_ds_from_arrays(uint64_t n, uint64_t d, int layout, const double* labels,
                         const double* values, uint64_t n_values, const uint32_t* indices,
                         uint64_t n_indices, const uint64_t* offsets, uint64_t n_offsets,
                         uint64_t pw) {
  auto* ds = new Data();
  ds->n = n;
  ds->d = d;
  ds->layout = layout;
  ds->labels.assign(labels, labels + n);
  if (n_values) ds->values.assign(values, values + n_values);
  if (n_indices) ds->indices.assign(indices, indices + n_indices);
  if (n_offsets) ds->offsets.assign(offsets, offsets + n_offsets);
  ds->pw = pw;
  return ds;
}
void orc_ds_free(void* h) { delete H(h); }
void orc_ds_info(void* h, uint64_t* out) {
  Data* ds = H(h);
  out[0] = ds->n;
  out[1] = ds->d;
  out[2] = static_cast<uint64_t>(ds->layout);
  out[3] = ds->values.size();
  out[4] = ds->indices.size();
  out[5] = ds->offsets.size();
  out[6] = ds->pw;
}
void orc_ds_copy(void* h, double* labels, double* values, uint32_t* indices, uint64_t* offsets) {
  Data* ds = H(h);
  if (labels) std::copy(ds->labels.begin(), ds->labels.end(), labels);
  if (values) std::copy(ds->values.begin(), ds->values.end(), values);
  if (indices) std::copy(ds->indices.begin(), ds->indices.end(), indices);
  if (offsets) std::copy(ds->offsets.begin(), ds->offsets.end(), offsets);
}

// --- fixtures (src/fixtures.cpp:12-100) ---------------------------------------------

void* orc_fixture_dense(uint64_t n, uint64_t d, uint64_t seed, double noise) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  std::vector<double> wt(d);
  for (double& v : wt) v = normal(rng);  // hidden model, fixtures.cpp:12-17
  std::uniform_real_distribution<double> uval(-1.0, 1.0);
  auto* ds = new Data();
  ds->n = n;
  ds->d = d;
  ds->layout = kDenseRow;
  ds->values.resize(n * d);
  ds->labels.resize(n);
  for (uint64_t e = 0; e < n; ++e) {
    double z = 0.0;
    for (uint64_t j = 0; j < d; ++j) {
      double v = uval(rng);
      ds->values[e * d + j] = v;
      z += v * wt[j];
    }
    double y = z >= 0.0 ? 1.0 : -1.0;  // label_for, fixtures.cpp:19-26
    if (noise > 0.0) {
      std::uniform_real_distribution<double> u(0.0, 1.0);
      if (u(rng) < noise) y = -y;
    }
    ds->labels[e] = y;
  }
  return ds;
}

void* orc_fixture_sparse(uint64_t n, uint64_t d, double avg, uint64_t seed, double noise) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  std::vector<double> wt(d);
  for (double& v : wt) v = normal(rng);
  std::uniform_real_distribution<double> uval(-1.0, 1.0);
  std::uniform_real_distribution<double> u01(std::nextafter(0.0, 1.0), 1.0);
  std::uniform_int_distribution<uint32_t> uidx(0, static_cast<uint32_t>(d - 1));
  const double xm = avg / 2.0;
  const auto max_nnz = static_cast<uint64_t>(
      std::min<double>(static_cast<double>(d), std::max(1.0, 20.0 * avg)));
  auto* ds = new Data();
  ds->n = n;
  ds->d = d;
  ds->layout = kCsr;
  ds->labels.resize(n);
  ds->offsets.push_back(0);
  std::vector<uint32_t> row;
  std::unordered_set<uint32_t> seen;
  for (uint64_t e = 0; e < n; ++e) {
    double pareto = xm / std::sqrt(u01(rng));
    uint64_t nnz = std::clamp<uint64_t>(static_cast<uint64_t>(std::lround(pareto)), 1, max_nnz);
    row.clear();
    seen.clear();
    while (row.size() < nnz) {
      uint32_t j = uidx(rng);
      if (seen.insert(j).second) row.push_back(j);
    }
    std::sort(row.begin(), row.end());
    double z = 0.0;
    for (uint32_t j : row) {
      double v = uval(rng);
      ds->indices.push_back(j);
      ds->values.push_back(v);
      z += v * wt[j];
    }
    ds->offsets.push_back(ds->values.size());
    double y = z >= 0.0 ? 1.0 : -1.0;
    if (noise > 0.0) {
      std::uniform_real_distribution<double> u(0.0, 1.0);
      if (u(rng) < noise) y = -y;
    }
    ds->labels[e] = y;
  }
  return ds;
}

void orc_round_f32(void* h) {
  for (double& v : H(h)->values) v = static_cast<double>(static_cast<float>(v));
}

// --- layout conversion (src/dataset.cpp:333-446) -------------------------------------

void* orc_convert_layout(void* h, int target) {
  const Data& ds = *H(h);
  if (ds.layout == target) return new Data(ds);
  if ((ds.layout == kDenseRow && target == kDenseCol) ||
      (ds.layout == kDenseCol && target == kDenseRow))
    return new Data(transpose(ds));
  // canonical CSR: storage order, zeros dropped
  Data csr;
  csr.n = ds.n;
  csr.d = ds.d;
  csr.layout = kCsr;
  csr.labels = ds.labels;
  csr.offsets.push_back(0);
  for (uint64_t e = 0; e < ds.n; ++e) {
    for_example(ds, e, [&](uint32_t j, double x) {
      if (x == 0.0) return;
      csr.indices.push_back(j);
      csr.values.push_back(x);
    });
    csr.offsets.push_back(csr.values.size());
  }
  if (target == kCsr) return new Data(csr);
  auto* out = new Data();
  out->n = ds.n;
  out->d = ds.d;
  out->layout = target;
  out->labels = ds.labels;
  if (target == kPadded) {
    uint64_t width = 0;
    for (uint64_t e = 0; e < ds.n; ++e) width = std::max(width, csr.offsets[e + 1] - csr.offsets[e]);
    out->pw = width;
    out->values.assign(ds.n * width, 0.0);
    out->indices.assign(ds.n * width, static_cast<uint32_t>(ds.d));
    for (uint64_t e = 0; e < ds.n; ++e)
      for (uint64_t s = 0; s < csr.offsets[e + 1] - csr.offsets[e]; ++s) {
        out->values[s * ds.n + e] = csr.values[csr.offsets[e] + s];
        out->indices[s * ds.n + e] = csr.indices[csr.offsets[e] + s];
      }
    return out;
  }
  out->values.assign(ds.n * ds.d, 0.0);
  for (uint64_t e = 0; e < ds.n; ++e)
    for (uint64_t s = csr.offsets[e]; s < csr.offsets[e + 1]; ++s) {
      uint32_t j = csr.indices[s];
      if (target == kDenseRow) out->values[e * ds.d + j] = csr.values[s];
      else out->values[static_cast<uint64_t>(j) * ds.n + e] = csr.values[s];
    }
  return out;
}

// --- schedule: mt19937_64(seed) + per-epoch std::shuffle (sync_engine.cpp:75-84) ------

void orc_schedule(uint64_t seed, uint64_t n, uint64_t epochs, int shuffle, uint32_t* out) {
  std::mt19937_64 rng(seed);
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  for (uint64_t e = 0; e < epochs; ++e) {
    if (shuffle) std::shuffle(order.begin(), order.end(), rng);
    std::copy(order.begin(), order.end(), out + e * n);
  }
}

// --- primitives ------------------------------------------------------------------------

double orc_dataset_loss(void* h, int task, const double* w) { return dataset_loss(task, *H(h), w); }

double orc_point_coefficient(int task, double z, double y) { return coefficient(task, z, y); }
double orc_point_loss_from_margin(int task, double z, double y) {
  return loss_from_margin(task, z, y);
}

void orc_batch_gradient(void* h, int task, const uint32_t* rows, uint64_t n_rows, const double* w,
                        double* g_out) {
  const Data& ds = *H(h);
  std::vector<uint32_t> r;
  if (n_rows == 0) {
    r.resize(ds.n);
    std::iota(r.begin(), r.end(), 0u);
  } else {
    r.assign(rows, rows + n_rows);
  }
  Data tr;
  bool use_tr = ds.layout == kDenseRow;
  if (use_tr) tr = transpose(ds);
  auto g = batch_gradient(task, ds, r, w, use_tr ? &tr : nullptr);
  std::copy(g.begin(), g.end(), g_out);
}

// sync::train (src/sync_engine.cpp:56-121): per-epoch model dump (epochs x d),
// loss per epoch, divergence. Returns the number of epochs run.
uint64_t orc_sync_train(void* h, int task, double alpha, uint64_t batch_b, uint64_t epochs,
                        double decay, uint64_t seed, int shuffle, const double* init,
                        double* models, double* losses, int* diverged) {
  const Data& ds = *H(h);
  std::vector<double> w(ds.d, 0.0);
  if (init) w.assign(init, init + ds.d);
  Data tr;
  bool use_tr = ds.layout == kDenseRow;
  if (use_tr) tr = transpose(ds);
  std::mt19937_64 rng(seed);
  std::vector<uint32_t> order(ds.n), batch;
  std::iota(order.begin(), order.end(), 0u);
  *diverged = 0;
  uint64_t ran = 0;
  for (uint64_t epoch = 1; epoch <= epochs; ++epoch) {
    double a = step_size(alpha, decay, epoch);
    if (shuffle) std::shuffle(order.begin(), order.end(), rng);
    bool finite = true;
    for (uint64_t lo = 0; lo < ds.n && finite; lo += batch_b) {
      uint64_t hi = std::min(ds.n, lo + batch_b);
      batch.assign(order.begin() + lo, order.begin() + hi);
      std::sort(batch.begin(), batch.end());
      auto g = batch_gradient(task, ds, batch, w.data(), use_tr ? &tr : nullptr);
      for (double v : g)
        if (!std::isfinite(v)) finite = false;
      for (uint64_t j = 0; j < ds.d; ++j) w[j] -= a * g[j];  // axpy, linalg.cpp:176-181
    }
    double loss = dataset_loss(task, ds, w.data());
    if (models) std::copy(w.begin(), w.end(), models + (epoch - 1) * ds.d);
    if (losses) losses[epoch - 1] = loss;
    ran = epoch;
    if (!finite || !std::isfinite(loss)) {
      *diverged = 1;
      break;
    }
  }
  return ran;
}

// Hogwild (src/async_engine.cpp:178-460) with the workers SERIALIZED in worker
// order — one legal interleaving of the "do in parallel" loop, deterministic,
// and identical to the reference for workers == 1. replication: 0 kernel,
// 1 block (group replicas reset from the global model at epoch start and
// merged by unweighted mean at epoch end, :293-331), 2 thread (per-worker).
// rr != 0 selects round-robin assignment (row-rr / col-rr).
uint64_t orc_hogwild_serial(void* h, int task, double alpha, uint64_t epochs, double decay, int rr,
                            int replication, uint64_t k, uint64_t workers, uint64_t group_size,
                            int offsets, const double* init, double* models, double* losses,
                            uint64_t* evals) {
  const Data& ds = *H(h);
  auto lists = assign(ds.n, workers, rr, k);
  std::vector<double> global(ds.d + 1, 0.0);
  if (init) std::copy(init, init + ds.d, global.begin());
  uint64_t n_rep = replication == 1 ? (workers + group_size - 1) / group_size
                   : replication == 2 ? workers
                                      : 0;
  std::vector<std::vector<double>> reps(n_rep);
  for (uint64_t epoch = 1; epoch <= epochs; ++epoch) {
    double a = step_size(alpha, decay, epoch);
    for (auto& r : reps) r = global, r[ds.d] = 0.0;
    uint64_t total = 0;
    for (uint64_t w = 0; w < workers; ++w) {
      std::vector<double>& m = replication == 0   ? global
                               : replication == 1 ? reps[w / group_size]
                                                  : reps[w];
      process_examples(m, ds, task, lists[w], a, offsets != 0, w);
      total += lists[w].size();
    }
    if (n_rep) {  // merge_models (async_engine.cpp:133-156): sum in replica order, / R
      for (uint64_t j = 0; j < ds.d; ++j) {
        double s = 0.0;
        for (uint64_t r = 0; r < n_rep; ++r) s += 1.0 * reps[r][j];
        global[j] = s / static_cast<double>(n_rep);
      }
    }
    if (models) std::copy(global.begin(), global.begin() + ds.d, models + (epoch - 1) * ds.d);
    double loss = dataset_loss(task, ds, global.data());
    if (losses) losses[epoch - 1] = loss;
    if (evals) evals[epoch - 1] = total;
    if (!std::isfinite(loss)) return epoch;
  }
  return epochs;
}

uint64_t orc_assign(uint64_t n, uint64_t workers, int rr, uint64_t k, uint32_t* out,
                    uint64_t* offs) {
  auto lists = assign(n, workers, rr, k);
  uint64_t pos = 0;
  if (offs) offs[0] = 0;
  for (uint64_t w = 0; w < workers; ++w) {
    for (uint32_t id : lists[w]) {
      if (out) out[pos] = id;
      ++pos;
    }
    if (offs) offs[w + 1] = pos;
  }
  return pos;
}

// merge_models with optional weights (src/async_engine.cpp:133-156).
void orc_merge_models(const double* replicas, uint64_t r, uint64_t d, const double* weights,
                      double* merged) {
  double total = 0.0;
  if (weights)
    for (uint64_t i = 0; i < r; ++i) total += weights[i];
  else
    total = static_cast<double>(r);
  for (uint64_t j = 0; j < d; ++j) merged[j] = 0.0;
  for (uint64_t i = 0; i < r; ++i) {
    double wt = weights ? weights[i] : 1.0;
    for (uint64_t j = 0; j < d; ++j) merged[j] += wt * replicas[i * d + j];
  }
  for (uint64_t j = 0; j < d; ++j) merged[j] /= total;
}

// --- LIBSVM parsing (src/dataset.cpp:145-230) ---------------------------------------
// Returns 0 ok, 1 parse error (line number in *line_out), 2 other.

int orc_parse_libsvm(const char* text, uint64_t len, int64_t declared_d, void** out,
                     uint64_t* line_out) {
  auto parse_double = [](std::string_view s, double& v) {
    if (!s.empty() && s.front() == '+') s.remove_prefix(1);
    if (s.empty()) return false;
    auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    return ec == std::errc{} && p == s.data() + s.size();
  };
  auto parse_index = [](std::string_view s, uint64_t& v) {
    auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    return ec == std::errc{} && p == s.data() + s.size();
  };
  auto* ds = new Data();
  ds->layout = kCsr;
  ds->offsets.push_back(0);
  uint64_t max_seen = 0, line_no = 0;
  std::string_view all(text, len);
  std::size_t pos = 0;
  auto bad = [&](const std::string& msg) {
    g_err = msg + " (line " + std::to_string(line_no) + ")";
    *line_out = line_no;
    delete ds;
    return 1;
  };
  while (pos < all.size()) {
    std::size_t nl = all.find('\n', pos);
    std::string line(all.substr(pos, nl == std::string_view::npos ? std::string_view::npos : nl - pos));
    pos = nl == std::string_view::npos ? all.size() : nl + 1;
    ++line_no;
    if (auto c = line.find('#'); c != std::string::npos) line.resize(c);
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ' || line.back() == '\t'))
      line.pop_back();
    std::size_t start = line.find_first_not_of(" \t");
    if (start == std::string::npos) continue;
    std::string_view rest(line.data() + start, line.size() - start);
    auto next = [&rest]() -> std::string_view {
      std::size_t b = rest.find_first_not_of(" \t");
      if (b == std::string_view::npos) return {};
      std::size_t e = rest.find_first_of(" \t", b);
      std::string_view t = rest.substr(b, e == std::string_view::npos ? e : e - b);
      rest = e == std::string_view::npos ? std::string_view{} : rest.substr(e);
      return t;
    };
    std::string_view lt = next();
    double raw;
    if (!parse_double(lt, raw)) return bad("malformed label");
    ds->labels.push_back(raw <= 0.0 ? -1.0 : (raw == 2.0 ? -1.0 : 1.0));
    uint64_t prev = 0;
    for (std::string_view t = next(); !t.empty(); t = next()) {
      std::size_t colon = t.find(':');
      if (colon == std::string_view::npos) return bad("malformed feature");
      uint64_t i1;
      double v;
      if (!parse_index(t.substr(0, colon), i1) || i1 == 0) return bad("malformed feature index");
      if (!parse_double(t.substr(colon + 1), v)) return bad("malformed feature value");
      if (i1 <= prev) return bad("feature indices not strictly increasing");
      prev = i1;
      if (declared_d >= 0 && i1 > static_cast<uint64_t>(declared_d))
        return bad("feature index exceeds declared dimension");
      max_seen = std::max(max_seen, i1);
      if (v == 0.0) continue;
      ds->values.push_back(v);
      ds->indices.push_back(static_cast<uint32_t>(i1 - 1));
    }
    ds->offsets.push_back(ds->values.size());
  }
  ds->n = ds->labels.size();
  ds->d = declared_d >= 0 ? static_cast<uint64_t>(declared_d) : max_seen;
  *out = ds;
  return 0;
}

}  // extern "C"

// --- K9 restatement: the Philox dense generator (paper_1802_08800_b200/csrc/
// kernels_gen.cu, philox.hpp), written independently here. Distribution of
// fixtures::dense_classification (src/fixtures.cpp:30-52); exact bit-level
// definition: Philox-4x32-10, value = 2*(r>>8)*2^-24 - 1, hidden model by
// Box-Muller, label = sign of the fp64 dot product accumulated lane-strided
// over feature quads (lane l takes quads l, l+32, ...) and combined by an xor
// butterfly (16, 8, 4, 2, 1), flipped when the Philox flip draw < noise. ----

namespace {
struct P4 {
  uint32_t v[4];
};
P4 philox10(P4 c, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c.v[0];
    uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c.v[2];
    P4 n{{static_cast<uint32_t>(p1 >> 32) ^ c.v[1] ^ k0, static_cast<uint32_t>(p1),
          static_cast<uint32_t>(p0 >> 32) ^ c.v[3] ^ k1, static_cast<uint32_t>(p0)}};
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}
float unit_val(uint32_t r) { return static_cast<float>(r >> 8) * (1.0f / 16777216.0f) * 2.0f - 1.0f; }
}  // namespace

extern "C" {

void orc_philox_hidden_model(uint64_t seed, uint64_t d, double* w) {
  const uint32_t k0 = static_cast<uint32_t>(seed) ^ 0x9E3779B9u;
  const uint32_t k1 = static_cast<uint32_t>(seed >> 32) ^ 0x7F4A7C15u;
  for (uint64_t i = 0; 2 * i < d; ++i) {
    P4 r = philox10(P4{{static_cast<uint32_t>(i), 0u, 0u, 0x5EED0003u}}, k0, k1);
    uint64_t a = (static_cast<uint64_t>(r.v[0]) << 20) | (r.v[1] >> 12);
    uint64_t b = (static_cast<uint64_t>(r.v[2]) << 20) | (r.v[3] >> 12);
    double u1 = static_cast<double>(a + 1) * 0x1p-52, u2 = static_cast<double>(b) * 0x1p-52;
    double rad = std::sqrt(-2.0 * std::log(u1)), th = 6.283185307179586 * u2;
    w[2 * i] = rad * std::cos(th);
    if (2 * i + 1 < d) w[2 * i + 1] = rad * std::sin(th);
  }
}

// Rows [row_base, row_base + n) of the generated dataset: values (row-major,
// n*d doubles holding the fp32 values) and labels.
void orc_philox_dense(uint64_t n, uint64_t d, uint64_t row_base, uint64_t seed, double noise,
                      double* values, double* labels) {
  std::vector<double> w(d);
  orc_philox_hidden_model(seed, d, w.data());
  const uint64_t nq = (d + 3) / 4;
  for (uint64_t r = 0; r < n; ++r) {
    const uint64_t e = row_base + r;
    double part[32] = {0.0};
    for (uint64_t q = 0; q < nq; ++q) {
      P4 u = philox10(P4{{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32),
                          static_cast<uint32_t>(q), 0x5EED0001u}},
                      static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
      for (int t = 0; t < 4; ++t) {
        const uint64_t j = 4 * q + t;
        if (j >= d) continue;
        const float v = unit_val(u.v[t]);
        values[r * d + j] = static_cast<double>(v);
        part[q % 32] = part[q % 32] + static_cast<double>(v) * w[j];
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      double nx[32];
      for (int l = 0; l < 32; ++l) nx[l] = part[l] + part[l ^ off];
      for (int l = 0; l < 32; ++l) part[l] = nx[l];
    }
    double y = part[0] >= 0.0 ? 1.0 : -1.0;
    if (noise > 0.0) {
      P4 f = philox10(P4{{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), 0u, 0x5EED0002u}},
                      static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
      const float u = static_cast<float>(f.v[0] >> 8) * (1.0f / 16777216.0f);
      if (static_cast<double>(u) < noise) y = -y;
    }
    labels[r] = y;
  }
}

// Streaming full-batch gradient over rows [row_base, row_base + n) of the
// generated dataset at model w, without materialising it (the 25M x 1000
// shard of C5 is 100 GB in fp32): every row is regenerated from its Philox
// counters (exactly the values orc_philox_dense produces), its margin is the
// fp64 dot in ascending feature order (src/linalg.cpp:30-44), the coefficient
// is src/glm.cpp:30-34, and g = sum_e c_e x_e (src/linalg.cpp:58-76) is
// accumulated in fp64. Rows are split into `threads` contiguous ranges, each
// accumulated in row order, and the per-thread partials added in thread order
// (deterministic for a fixed thread count). loss_out (may be NULL) receives
// dataset_loss at w (src/glm.cpp:85-94).
void orc_philox_dense_gradient(uint64_t n, uint64_t d, uint64_t row_base, uint64_t seed,
                               double noise, int task, const double* w, uint32_t threads,
                               double* g_out, double* loss_out) {
  if (threads == 0) threads = 1;
  std::vector<double> wt(d);
  orc_philox_hidden_model(seed, d, wt.data());
  std::vector<std::vector<double>> part(threads, std::vector<double>(d, 0.0));
  std::vector<double> lpart(threads, 0.0);
  auto work = [&](uint32_t t) {
    const uint64_t r0 = n * t / threads, r1 = n * (t + 1) / threads;
    std::vector<double> x(d);
    std::vector<double>& g = part[t];
    double lsum = 0.0;
    const uint64_t nq = (d + 3) / 4;
    for (uint64_t r = r0; r < r1; ++r) {
      const uint64_t e = row_base + r;
      double lane[32] = {0.0};
      for (uint64_t q = 0; q < nq; ++q) {
        P4 u = philox10(P4{{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32),
                            static_cast<uint32_t>(q), 0x5EED0001u}},
                        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
        for (int k = 0; k < 4; ++k) {
          const uint64_t j = 4 * q + k;
          if (j >= d) continue;
          x[j] = static_cast<double>(unit_val(u.v[k]));
          lane[q % 32] = lane[q % 32] + x[j] * wt[j];
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        double nx[32];
        for (int l = 0; l < 32; ++l) nx[l] = lane[l] + lane[l ^ off];
        for (int l = 0; l < 32; ++l) lane[l] = nx[l];
      }
      double y = lane[0] >= 0.0 ? 1.0 : -1.0;
      if (noise > 0.0) {
        P4 f = philox10(P4{{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), 0u, 0x5EED0002u}},
                        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
        const float uf = static_cast<float>(f.v[0] >> 8) * (1.0f / 16777216.0f);
        if (static_cast<double>(uf) < noise) y = -y;
      }
      double z = 0.0;
      for (uint64_t j = 0; j < d; ++j) z = z + x[j] * w[j];
      lsum = lsum + loss_from_margin(task, z, y);
      const double c = coefficient(task, z, y);
      if (c != 0.0)
        for (uint64_t j = 0; j < d; ++j) g[j] = g[j] + c * x[j];
    }
    lpart[t] = lsum;
  };
  std::vector<std::thread> pool;
  for (uint32_t t = 0; t < threads; ++t) pool.emplace_back(work, t);
  for (auto& th : pool) th.join();
  double l = 0.0;
  for (uint64_t j = 0; j < d; ++j) g_out[j] = 0.0;
  for (uint32_t t = 0; t < threads; ++t) {
    for (uint64_t j = 0; j < d; ++j) g_out[j] = g_out[j] + part[t][j];
    l = l + lpart[t];
  }
  if (loss_out) *loss_out = l;
}

}  // extern "C"

