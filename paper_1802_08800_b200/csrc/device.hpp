// Internal device-side objects behind the C-ABI handles of include/sgdb.h and
// the kernel launchers (kernels_*.cu). Host-only header (no device code).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "errors.hpp"
#include "sgdb.h"

namespace sgdb::dev {

using CudaError = sgdb::detail::DeviceError;
using Unsupported = sgdb::detail::UnsupportedError;

inline void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device allocation.
template <class T>
struct DBuf {
  T* p = nullptr;
  uint64_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(uint64_t count) {
    if (count <= n && p) return;
    release();
    check(cudaMalloc(&p, (count ? count : 1) * sizeof(T)), "cudaMalloc");
    n = count;
  }
  void zero(cudaStream_t s) {
    if (p) check(cudaMemsetAsync(p, 0, n * sizeof(T), s), "cudaMemsetAsync");
  }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int max_threads_per_sm = 2048;
  size_t max_smem_optin = 227 * 1024;
  uint64_t launches = 0;
  sgdb_allreduce_fn allreduce = nullptr;
  void* allreduce_user = nullptr;
  // In-library NCCL communicator (sgdb_ctx_init_nccl): SUM all-reduces are
  // issued on the context stream (CUDA-graph capturable, no host hop).
  void* nccl_comm = nullptr;
  int nccl_rank = 0, nccl_nranks = 1;
  DBuf<double> loss_partials;  // per-block loss sums
  DBuf<double> loss_out;       // [0] loss, [1] scratch
  DBuf<unsigned> tickets;      // [0] loss ticket
  int* pinned_flag = nullptr;  // pinned host word for flag read-back
  cudaStream_t capture_stream = nullptr;  // private stream for CUDA-graph capture
  // Optional per-launch CUDA-event timing (sgdb_ctx_set_profiling).
  bool profiling = false;
  struct LaunchRec {
    const char* name;
    cudaEvent_t start, stop;
  };
  std::vector<LaunchRec> recs;
};

// Bracket every kernel launch: prof_begin before, launched after.
inline void prof_begin(Ctx& c, const char* name) {
  if (!c.profiling) return;
  Ctx::LaunchRec r{name, nullptr, nullptr};
  check(cudaEventCreate(&r.start), "cudaEventCreate");
  check(cudaEventCreate(&r.stop), "cudaEventCreate");
  check(cudaEventRecord(r.start, c.stream), "cudaEventRecord");
  c.recs.push_back(r);
}
inline void launched(Ctx& c, const char* what) {
  ++c.launches;
  check(cudaGetLastError(), what);
  if (c.profiling && !c.recs.empty()) check(cudaEventRecord(c.recs.back().stop, c.stream), "cudaEventRecord");
}

// Launch-configuration queries cached per (device, kernel, threads, smem):
// cudaFuncSetAttribute / cudaOccupancy* / cudaFuncGetAttributes cost host
// microseconds each, which showed up as idle GPU time between the kernels of
// one small epoch. Defined in capi_device.cu.
void set_max_dyn_smem(const void* kern, size_t smem, const char* what);
int blocks_per_sm(const void* kern, int threads, size_t smem);
size_t static_smem_of(const void* kern);

// Device storage kind chosen at upload.
enum class Kind { Dense, Csr };

// A blocked, segmented copy of the nonzeros (kernels_sparse.cu). The major
// dimension (rows for the gradient pass's CSC, columns for the wide margin
// pass) is split into nblk blocks of rb (< 2^16, % 8 == 0) entries; segment
// (b, m) = block b's entries of minor index m, at segptr[b*nminor + m] ..
// segptr[b*nminor + m + 1], stored as fp32 values + 16-bit block-local major
// ids in (block, minor, major) order; its head bitmap (bit s = slot s starts
// a non-empty segment) + word prefix; ord_of_seg (exclusive count of the
// non-empty segments before each) when some segments are empty; cpb nnz-balanced minor ranges (cta) shared by all blocks; arrival
// tickets (monotonic: gen launches since they were zeroed).
struct Blocked {
  uint32_t rb = 0, nblk = 0, cpb = 0;
  DBuf<float> val;
  DBuf<uint16_t> id;
  DBuf<uint32_t> segptr, bm, bm_pre, ord_of_seg, cta;
  bool segs_empty = false;
  DBuf<unsigned> tickets;
  unsigned gen = 0;
};

struct Dataset {
  Ctx* ctx = nullptr;
  uint64_t uid = 0;  // unique per upload (keys cached epoch graphs)
  uint64_t n = 0;  // local rows
  uint64_t d = 0;
  uint64_t row_base = 0, n_global = 0;
  int layout_in = SGDB_LAYOUT_CSR;
  Kind kind = Kind::Csr;
  uint64_t nnz = 0;  // stored entries (CSR) or n*d (dense)
  uint64_t max_row = 0;  // longest CSR row (slots)
  DBuf<float> labels;  // n (padded to a multiple of 4 + tile slack)
  // Dense row-major fp32, n*d (+ slack so bulk copies may round up to 16 B).
  DBuf<float> x;
  // CSR.
  DBuf<float> val;
  DBuf<uint32_t> idx;
  DBuf<uint32_t> rowptr;
  DBuf<uint16_t> idx16;  // staging for sgdb_dataset_refresh_idx16
  // Full-batch sparse step (kernels_sparse.cu), built on the device by
  // sparse_prep at upload and again after a refresh (sparse_ready = false):
  //  * row-head bitmap rbm (bit s = slot s starts a non-empty row) and the
  //    exclusive popcount prefix of its words (rbm_pre); row_of_ord maps a
  //    non-empty row's ordinal to its row id when some rows are empty;
  //  * 16-bit column ids (d <= 65536) for the margin pass;
  //  * margin-pass CTA ranges (cta_n CTAs, each starting at a row start);
  //  * the row-blocked CSC of the gradient pass (csc) and, for models too
  //    large for shared memory, the column-blocked CSR of the margin pass
  //    (wide; see Blocked).
  bool sparse_ready = false;
  DBuf<uint32_t> rbm, rbm_pre, row_of_ord;
  bool rows_empty = false;
  DBuf<uint16_t> cidx16;
  uint32_t cta_n = 0;
  DBuf<uint32_t> cta_slot;
  DBuf<uint32_t> cta_row;  // first row of each margin CTA (cta_n + 1)
  DBuf<unsigned> blk_ready, blk_expect;  // K23g: per row block, released / expected margin CTAs
  Blocked csc;       // major = rows, minor = columns
  bool wide = false;  // margin pass over `wmajor` below instead of the CSR stream
  Blocked wmajor;    // major = columns, minor = rows
  DBuf<float> mpart;  // wmajor.nblk * n partial margins
  // sparse_prep's scratch, kept so a rebuild after every refresh (bench
  // e2e) neither allocates nor frees (cudaFree synchronises the device).
  struct {
    DBuf<uint32_t> k_in, k_out, a, b, c;
    DBuf<uint64_t> p_in, p_out;
    DBuf<unsigned char> tmp;
    DBuf<unsigned> cnt;
  } prep;
  // Column-major copies for the col-* access paths (built lazily).
  bool col_built = false;
  DBuf<float> xcol;    // dense: d*n
  DBuf<float> pval;    // padded slot-major: pw*n
  DBuf<uint32_t> pidx;
  uint64_t pw = 0;
  // Host copies kept for lazy builds (CSR arrays, only when needed).
  std::vector<float> h_val;
  std::vector<uint32_t> h_idx;
  std::vector<uint32_t> h_rowptr;
  std::vector<float> h_xcol;
  // Example-scope Hogwild replicas (async_engine.cpp:266-290): one fp32 copy
  // of the model at every stored slot (aligned with val/idx), plus the
  // per-example claim / ready epoch words of ensure_replica (:333-344).
  DBuf<float> ex_rep;
  DBuf<double> ex_rep64;  // exact-fp64 mode
  DBuf<unsigned> ex_claim, ex_ready;
  unsigned ex_epoch = 0;
  // Scratch.
  DBuf<float> coef;        // per local row coefficient (sparse full batch)
  DBuf<uint32_t> order;    // n_global ids of the current epoch
  bool order_iota = false; // order holds 0..n_global-1 (sync_epoch with no order)
  // Sparse mini-batch chunk plan (K3c): rows of ids[0..mb_count) cut into
  // chunks of mb_ch slots; mb_off = exclusive prefix of the chunk counts
  // (mb_count + 1 entries), mb_z = per-chunk partial margins of one step.
  const uint32_t* mb_ids = nullptr;
  uint64_t mb_count = 0;
  uint32_t mb_ch = 0;
  DBuf<uint32_t> mb_cnt, mb_off;
  DBuf<uint4> mb_meta;     // per chunk {slot begin, slot end, position, local row}
  uint64_t mb_cap = 0;     // chunks mb_meta holds (steps beyond it search mb_off)
  DBuf<float> mb_z;
  DBuf<unsigned char> mb_tmp;
  size_t mb_tmp_bytes = 0;
  // Exact-fp64 mode (SGDB_UPLOAD_EXACT_FP64): fp64 copies of the values and
  // the scratch of the reference-order kernels (kernels_linalg.cu).
  bool exact = false;
  DBuf<double> x64;        // dense: n*d row-major
  DBuf<double> val64;      // CSR (and wide dense): nnz, aligned with idx
  DBuf<double> ex_a, ex_c, ex_part, ex_stack, ex_reps;
  DBuf<int> ex_live;
};

struct Model {
  Ctx* ctx = nullptr;
  uint64_t d = 0;
  DBuf<float> w32;       // d+1 (guard slot d == 0)
  DBuf<double> w64;      // d, master
  DBuf<double> g64;      // d, gradient accumulator (kept zeroed between steps)
  DBuf<double> partials; // per-block gradient partials, deterministic full batch
  DBuf<float> part32;    // per-(row block, column) sums of the full-batch sparse step
  DBuf<unsigned> ticket; // [0] grad ticket
  DBuf<double> g3;       // 3*d rotating gradient buffers of the persistent epoch (K1c)
  DBuf<unsigned> gbar;   // grid barrier words (K1c), zero between uses
  DBuf<int> finite;      // [0] 1 while every gradient entry was finite
  DBuf<double> scal;     // [0] ||g||^2
  DBuf<float> replicas;  // Hogwild replicas, R x ld
  DBuf<float> spread;    // kernel-scope Hogwild model, slice-spread layout
  // Which copy holds the latest model: the dense w32/w64 pair and/or the
  // spread copy (kept authoritative across back-to-back Hogwild epochs).
  bool dense_current = true;
  bool spread_current = false;
  uint32_t spread_ms = 1;
  uint64_t n_replicas = 0, replica_ld = 0;
  // Captured mini-batch epoch (one kernel sequence per step), replayed each
  // epoch; key = (dataset uid, batch size, task).
  cudaGraphExec_t epoch_graph = nullptr;
  uint64_t graph_ds = 0, graph_b = 0, graph_nodes = 0;
  int graph_task = -1;
  void* graph_comm = nullptr;  // the NCCL communicator captured into the graph
  DBuf<double> alpha_dev;
  Model() = default;
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;
  ~Model() {
    if (epoch_graph) cudaGraphExecDestroy(epoch_graph);
  }
};

// A cross-rank collective is attached (NCCL communicator or host hook).
inline bool has_collective(const Ctx& c) { return c.nccl_comm != nullptr || c.allreduce != nullptr; }

// ---- launchers (kernels_*.cu) -------------------------------------------------

struct StepArgs {
  int task = 0;
  double alpha = 0.0;
  const double* alpha_dev = nullptr;  // device step size (graph-captured epochs)
  bool apply = true;      // fuse w -= alpha*g (else g64 holds the gradient)
  bool want_norm = false; // accumulate ||g||^2 into model.scal[0]
  // Sparse mini-batch steps update the fp64 master directly (no gradient
  // buffer, no apply launch); the epoch ends with sync_w32_from_w64.
  bool direct = false;
};

// Dense, all local rows: one full-batch gradient (deterministic).
void dense_full_step(Dataset& ds, Model& m, const StepArgs& a);
// Dense, rows = global ids ids[0..nb) (device pointer), mini-batch gradient.
// K1c: a whole dense mini-batch epoch (ids in ds.order, batches of B) in one
// persistent cooperative launch; no allreduce hook. Returns false (nothing
// launched) for shapes the per-step kernels serve better.
bool dense_epoch(Dataset& ds, Model& m, int task, double alpha, uint64_t B);
void dense_batch_step(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb,
                      const StepArgs& a);
// Sparse, all local rows: margin/coef pass + CSC gradient pass
// (kernels_sparse.cu); sparse_prep builds the device structures it reads.
void sparse_prep(Dataset& ds);
void sparse_full_step(Dataset& ds, Model& m, const StepArgs& a);
// Sparse mini-batch: chunk plan of the ids a sequence of steps walks (device
// ids[0..count), steps of at most max_step positions); steps whose ids lie
// outside the current plan build their own.
void csr_batch_plan(Dataset& ds, const uint32_t* ids, uint64_t count, uint64_t max_step);
// Sparse mini-batch step: chunk margins, then coefficient + scatter with fp64
// atomics, then apply.
void csr_batch_step(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb, const StepArgs& a);
// w -= alpha*g64; w32 = w64; finite; g64 = 0. alpha_dev (if set) overrides alpha.
void apply_update(Model& m, double alpha, bool want_norm, const double* alpha_dev = nullptr);
// dst[i] = src[i] (u16 -> u32) on c's stream; src 16-byte aligned.
void widen_u16(Ctx& c, const uint16_t* src, uint32_t* dst, uint64_t n);
// fp64 loss over all local rows; result left in ctx.loss_out[0] (device).
void loss_launch(Dataset& ds, Model& m, int task);
// w64 = (double) w32[0..d)
void sync_w64_from_w32(Model& m);
// w32 = (float) w64[0..d) (after directly-updated sparse mini-batch steps)
void sync_w32_from_w64(Model& m);
// Weighted mean of models (w64) -> out; refresh copies it back to each input.
void average_models(Ctx& c, Model* const* models, uint64_t count, const double* weights,
                    Model& out, bool refresh);

struct HogwildArgs {
  int task = 0;
  float alpha = 0.f;
  int access = 0;        // sgdb_access_path
  int replication = 0;   // sgdb_replication
  uint64_t k = 0, workers = 1, group_size = 32;
  bool offsets = true;
  int lanes = 0;         // resolved lanes per worker
  uint32_t seg = 0, nseg = 1;  // run list positions [total*seg/nseg, total*(seg+1)/nseg)
  double alpha_f64 = 0.0;      // exact-fp64 mode step size
};
int hogwild_auto_lanes(const Dataset& ds, int access);
// Lane groups of one resident wave of the kernel-scope Hogwild kernel this
// dataset would use (the long-row variant holds more registers).
uint64_t hogwild_resident_workers(const Ctx& c, const Dataset& ds, int lanes);
void hogwild_epoch(Dataset& ds, Model& m, const HogwildArgs& a);

// Make w32/w64 current (gathers the spread Hogwild copy if it is newer).
void materialize(Model& m);
// Mark the dense model as written (the spread copy is stale afterwards).
inline void dense_written(Model& m) {
  m.dense_current = true;
  m.spread_current = false;
}

// w64 *= scale; w32 = w64 (rank averaging after a SUM all-reduce).
void scale_model(Model& m, double scale);

uint64_t next_dataset_uid();

// fp64 operator primitives and the exact-fp64 mode (kernels_linalg.cu).
void lin_matvec(Dataset& ds, const uint32_t* rows, uint64_t nr, const double* v, double* out);
void lin_matvec_t(Dataset& ds, const uint32_t* rows, uint64_t nr, const double* a, bool col_order,
                  double* out);
void exact_batch_gradient(Dataset& ds, const uint32_t* rows_host, uint64_t n_rows,
                          const double* w_host, int task, bool transposed, double* g_host);
void exact_sync_epoch(Dataset& ds, Model& m, int task, double alpha, const uint32_t* order,
                      uint64_t batch_b);
void exact_epoch_batch(Dataset& ds, Model& m, int task, double alpha);
void exact_loss(Dataset& ds, Model& m, int task);
void exact_hogwild(Dataset& ds, Model& m, const HogwildArgs& a);
void build_col(Dataset& ds);
// Slot-major padded copy (pval / pidx, width = longest row, sentinel d) of the
// uploaded CSR, on the device (convert_layout(Csr -> PaddedDense)).
void build_padded_from_csr(Dataset& ds);

}  // namespace sgdb::dev

// Opaque C handles are the internal objects.
struct sgdb_ctx : sgdb::dev::Ctx {};
struct sgdb_dataset : sgdb::dev::Dataset {};
struct sgdb_model : sgdb::dev::Model {};
