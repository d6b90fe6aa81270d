// Layer 1 of include/sgdb.h: device context, device-resident dataset and
// model, and the per-epoch device ops (sync epoch, batch gradient, Hogwild
// epoch, replica averaging, loss). Host code only; kernels live in
// kernels_sync.cu / kernels_hogwild.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <map>
#include <mutex>
#include <tuple>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "device.hpp"
#include "errors.hpp"

using namespace sgdb::dev;

namespace sgdb::detail {
namespace {
thread_local std::string g_last_error;
thread_local uint64_t g_parse_line = 0;
}  // namespace
void set_last_error(const std::string& msg) { g_last_error = msg; }
void set_parse_line(uint64_t line) { g_parse_line = line; }
uint64_t parse_line() { return g_parse_line; }
}  // namespace sgdb::detail

namespace {

void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}


template <class T>
void h2d(T* dst, const T* src, uint64_t count, cudaStream_t s) {
  if (count) check(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
}

void upload_csr(sgdb_dataset* ds, std::vector<uint32_t>& rowptr, std::vector<uint32_t>& idx,
                std::vector<float>& val) {
  cudaStream_t s = ds->ctx->stream;
  ds->kind = Kind::Csr;
  ds->nnz = idx.size();
  ds->max_row = 0;
  for (size_t r = 0; r + 1 < rowptr.size(); ++r)
    ds->max_row = std::max<uint64_t>(ds->max_row, rowptr[r + 1] - rowptr[r]);
  // +8 slack: vectorised kernels read whole aligned 16-byte groups around a row.
  ds->val.alloc(ds->nnz + 8);
  ds->idx.alloc(ds->nnz + 8);
  ds->val.zero(s);
  ds->idx.zero(s);
  ds->rowptr.alloc(ds->n + 1);
  h2d(ds->val.p, val.data(), ds->nnz, s);
  h2d(ds->idx.p, idx.data(), ds->nnz, s);
  h2d(ds->rowptr.p, rowptr.data(), ds->n + 1, s);
  // The full-batch structures (head bitmaps, blocked CSC) are built on the
  // device on first use (sparse_prep).
  ds->sparse_ready = false;
  check(cudaStreamSynchronize(s), "upload sync");  // host vectors die with the caller
}

uint64_t nonempty_workers(uint64_t n, uint64_t T, bool rr) {
  if (rr) return std::min(n, T);
  const uint64_t chunk = (n + T - 1) / T;
  return (n + chunk - 1) / chunk;
}

// Evaluations in segment seg of nseg: per worker, list positions
// [total*seg/nseg, total*(seg+1)/nseg) of its assign() list (n + k per
// non-empty worker in all), as run_worker splits them.
uint64_t segment_evals(uint64_t n, uint64_t T, bool rr, uint64_t k, uint32_t seg, uint32_t nseg) {
  if (nseg == 1) return n + nonempty_workers(n, T, rr) * k;
  const uint64_t chunk = (n + T - 1) / T;
  uint64_t total_evals = 0;
  for (uint64_t w = 0; w < T; ++w) {
    uint64_t cnt;
    if (rr) {
      cnt = w < n ? (n - 1 - w) / T + 1 : 0;
    } else {
      const uint64_t b = std::min(n, w * chunk), e = std::min(n, b + chunk);
      cnt = e - b;
    }
    if (cnt == 0) {
      if (!rr) break;  // chunk lists are empty from here on
      continue;
    }
    const uint64_t t = cnt + k;
    total_evals += t * (seg + 1) / nseg - t * seg / nseg;
  }
  return total_evals;
}

// The finite flag is any nonzero value while every gradient entry was
// finite; kernels write 0. Reset with a device memset (no host staging) and
// read back through pinned memory.
void set_finite(sgdb_model* m) {
  check(cudaMemsetAsync(m->finite.p, 0x01, sizeof(int), m->ctx->stream), "set finite");
}

int read_finite(sgdb_model* m) {
  Ctx& c = *m->ctx;
  if (!c.pinned_flag) check(cudaMallocHost(&c.pinned_flag, sizeof(int)), "cudaMallocHost");
  check(cudaMemcpyAsync(c.pinned_flag, m->finite.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream),
        "read finite");
  check(cudaStreamSynchronize(c.stream), "sync");
  return *c.pinned_flag != 0 ? 1 : 0;
}

// NCCL, resolved at run time (dlopen "libnccl.so.2": the copy already in the
// process when a host framework loaded one, else the system library), so the
// engine carries no link dependency and single-GPU use never needs NCCL.
// Types and entry points follow nccl.h (NCCL 2.x ABI).
struct NcclUid {
  char internal[128];
};
struct NcclApi {
  using GetUid = int (*)(NcclUid*);
  using InitRank = int (*)(void**, int, NcclUid, int);
  using AllReduce = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  using Destroy = int (*)(void*);
  using ErrStr = const char* (*)(int);
  GetUid get_uid = nullptr;
  InitRank init_rank = nullptr;
  AllReduce all_reduce = nullptr;
  Destroy destroy = nullptr;
  ErrStr err = nullptr;
};
constexpr int kNcclSum = 0, kNcclFloat32 = 7, kNcclFloat64 = 8;

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_uid = reinterpret_cast<NcclApi::GetUid>(dlsym(h, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<NcclApi::InitRank>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<NcclApi::AllReduce>(dlsym(h, "ncclAllReduce"));
    a.destroy = reinterpret_cast<NcclApi::Destroy>(dlsym(h, "ncclCommDestroy"));
    a.err = reinterpret_cast<NcclApi::ErrStr>(dlsym(h, "ncclGetErrorString"));
    return a;
  }();
  if (!api.get_uid || !api.init_rank || !api.all_reduce || !api.destroy)
    throw std::runtime_error("NCCL (libnccl.so.2) is not available");
  return api;
}

void nccl_check(int r, const char* what) {
  if (r != 0)
    throw std::runtime_error(std::string(what) + ": " + (nccl().err ? nccl().err(r) : "NCCL error"));
}

void call_allreduce(Ctx& c, void* ptr, uint64_t count, int dtype) {
  if (c.nccl_comm) {
    nccl_check(nccl().all_reduce(ptr, ptr, count, dtype == 0 ? kNcclFloat32 : kNcclFloat64, kNcclSum,
                                 c.nccl_comm, c.stream),
               "ncclAllReduce");
    return;
  }
  if (!c.allreduce) return;
  if (c.allreduce(c.allreduce_user, ptr, count, dtype, c.stream) != 0)
    throw std::runtime_error("allreduce hook failed");
}

void validate_device_plan(const sgdb_plan& p, int layout) {
  sgdb_status st = sgdb_validate_plan(&p, layout);
  if (st != SGDB_OK) throw std::invalid_argument(sgdb_last_error());
}

void model_init(sgdb_model* m, Ctx* c, uint64_t d) {
  m->ctx = c;
  m->d = d;
  m->w32.alloc(((d + 1) + 3) & ~uint64_t(3));  // whole 16-byte groups (bulk copies)
  m->w64.alloc(std::max<uint64_t>(1, d) + 2);  // +2: whole 16-byte units for L2 bulk prefetches
  m->g64.alloc(std::max<uint64_t>(1, d));
  m->ticket.alloc(1);
  m->finite.alloc(1);
  m->scal.alloc(2);
  m->w32.zero(c->stream);
  m->w64.zero(c->stream);
  m->g64.zero(c->stream);
  m->ticket.zero(c->stream);
  m->scal.zero(c->stream);
  set_finite(m);
}

void model_set(sgdb_model* m, const double* w) {
  Ctx& c = *m->ctx;
  dense_written(*m);
  std::vector<float> w32(m->d + 1, 0.f);
  for (uint64_t j = 0; j < m->d; ++j) w32[j] = static_cast<float>(w[j]);
  h2d(m->w64.p, w, m->d, c.stream);
  h2d(m->w32.p, w32.data(), m->d + 1, c.stream);
  check(cudaStreamSynchronize(c.stream), "model_set sync");
}

void full_step(sgdb_dataset* ds, sgdb_model* m, const StepArgs& a) {
  if (ds->kind == Kind::Dense) dense_full_step(*ds, *m, a);
  else sparse_full_step(*ds, *m, a);
}

}  // namespace

extern "C" {

const char* sgdb_last_error(void) { return sgdb::detail::g_last_error.c_str(); }
const char* sgdb_version(void) { return "sgdb_b200 0.1 (sm_100a)"; }

sgdb_status sgdb_ctx_create(int32_t device, void* cuda_stream, sgdb_ctx** out) {
  return sgdb_guard([&] {
    require(out != nullptr, "out is null");
    check(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new sgdb_ctx();
    c->device = device;
    cudaDeviceProp prop{};
    check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10)
      throw sgdb::detail::UnsupportedError("sgdb_b200 is built for sm_100a (Blackwell); found sm_" +
                                           std::to_string(prop.major * 10 + prop.minor));
    c->num_sms = prop.multiProcessorCount;
    c->max_threads_per_sm = prop.maxThreadsPerMultiProcessor;
    c->max_smem_optin = prop.sharedMemPerBlockOptin;
    if (cuda_stream) {
      c->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
      check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
      c->own_stream = true;
    }
    check(cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->loss_out.alloc(2);
    c->tickets.alloc(4);
    c->tickets.zero(c->stream);
    *out = c;
  });
}

sgdb_status sgdb_ctx_destroy(sgdb_ctx* ctx) {
  return sgdb_guard([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->pinned_flag) cudaFreeHost(ctx->pinned_flag);
    if (ctx->capture_stream) cudaStreamDestroy(ctx->capture_stream);
    if (ctx->nccl_comm) nccl().destroy(ctx->nccl_comm);
    delete ctx;
  });
}

sgdb_status sgdb_ctx_stream(sgdb_ctx* ctx, void** stream_out) {
  return sgdb_guard([&] { *stream_out = ctx->stream; });
}

sgdb_status sgdb_ctx_synchronize(sgdb_ctx* ctx) {
  return sgdb_guard([&] { check(cudaStreamSynchronize(ctx->stream), "synchronize"); });
}

sgdb_status sgdb_ctx_launch_count(sgdb_ctx* ctx, uint64_t* out) {
  return sgdb_guard([&] { *out = ctx->launches; });
}

sgdb_status sgdb_ctx_set_allreduce(sgdb_ctx* ctx, sgdb_allreduce_fn fn, void* user) {
  return sgdb_guard([&] {
    ctx->allreduce = fn;
    ctx->allreduce_user = user;
  });
}

sgdb_status sgdb_ctx_set_profiling(sgdb_ctx* ctx, int32_t enable) {
  return sgdb_guard([&] {
    check(cudaStreamSynchronize(ctx->stream), "profiling sync");
    for (auto& r : ctx->recs) {
      cudaEventDestroy(r.start);
      cudaEventDestroy(r.stop);
    }
    ctx->recs.clear();
    ctx->profiling = enable != 0;
  });
}

sgdb_status sgdb_ctx_kernel_stats(sgdb_ctx* ctx, uint64_t i, char* name, uint64_t cap,
                                  uint64_t* launches, double* total_ms, uint64_t* n_entries) {
  return sgdb_guard([&] {
    check(cudaStreamSynchronize(ctx->stream), "stats sync");
    std::vector<std::string> names;
    std::vector<std::pair<uint64_t, double>> agg;
    for (auto& r : ctx->recs) {
      float ms = 0.f;
      check(cudaEventElapsedTime(&ms, r.start, r.stop), "cudaEventElapsedTime");
      auto it = std::find(names.begin(), names.end(), std::string(r.name));
      if (it == names.end()) {
        names.emplace_back(r.name);
        agg.push_back({1, ms});
      } else {
        auto& a = agg[static_cast<size_t>(it - names.begin())];
        a.first += 1;
        a.second += ms;
      }
    }
    if (n_entries) *n_entries = names.size();
    if (i < names.size()) {
      if (name && cap) std::snprintf(name, cap, "%s", names[i].c_str());
      if (launches) *launches = agg[i].first;
      if (total_ms) *total_ms = agg[i].second;
    }
  });
}

sgdb_status sgdb_nccl_get_unique_id(uint8_t* id_out) {
  return sgdb_guard([&] {
    require(id_out != nullptr, "null argument");
    NcclUid uid{};
    nccl_check(nccl().get_uid(&uid), "ncclGetUniqueId");
    std::memcpy(id_out, uid.internal, sizeof(uid.internal));
  });
}

sgdb_status sgdb_ctx_init_nccl(sgdb_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id) {
  return sgdb_guard([&] {
    require(ctx && id, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "rank out of range");
    require(ctx->nccl_comm == nullptr, "the context already has a communicator");
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    NcclUid uid{};
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    void* comm = nullptr;
    nccl_check(nccl().init_rank(&comm, nranks, uid, rank), "ncclCommInitRank");
    ctx->nccl_comm = comm;
    ctx->nccl_rank = rank;
    ctx->nccl_nranks = nranks;
  });
}

sgdb_status sgdb_ctx_world(sgdb_ctx* ctx, int32_t* rank, int32_t* nranks) {
  return sgdb_guard([&] {
    require(ctx != nullptr, "null argument");
    if (rank) *rank = ctx->nccl_rank;
    if (nranks) *nranks = ctx->nccl_nranks;
  });
}

sgdb_status sgdb_model_average_ranks(sgdb_ctx* ctx, sgdb_model* m, uint64_t world) {
  return sgdb_guard([&] {
    require(world >= 1, "world size must be >= 1");
    if (world == 1 && !has_collective(*ctx)) return;
    if (!has_collective(*ctx))
      throw std::invalid_argument("no collective on the context (sgdb_ctx_init_nccl or an allreduce hook)");
    materialize(*m);
    dense_written(*m);
    call_allreduce(*ctx, m->w64.p, m->d, 1);
    scale_model(*m, 1.0 / static_cast<double>(world));
    // No host sync: the hook's collective is ordered on the context stream
    // (NCCL through torch's current stream), so the next epoch's kernels see
    // the averaged model; a per-average host round trip would stall every
    // ~25 us epoch of the multi-GPU bench.
  });
}

sgdb_status sgdb_ctx_resident_workers(sgdb_ctx* ctx, const sgdb_dataset* ds, int32_t lanes,
                                      uint64_t* out) {
  return sgdb_guard([&] {
    int g = lanes > 0 ? lanes : hogwild_auto_lanes(*ds, SGDB_ACCESS_ROW_CH);
    *out = hogwild_resident_workers(*ctx, *ds, g);
  });
}

sgdb_status sgdb_dataset_upload(sgdb_ctx* ctx, const sgdb_dataset_view* v, uint64_t row_base,
                                uint64_t n_global, sgdb_dataset** out) {
  return sgdb_dataset_upload_ex(ctx, v, row_base, n_global, 0, out);
}

sgdb_status sgdb_dataset_upload_ex(sgdb_ctx* ctx, const sgdb_dataset_view* v, uint64_t row_base,
                                   uint64_t n_global, uint32_t flags, sgdb_dataset** out) {
  return sgdb_guard([&] {
    require(ctx && v && out, "null argument");
    require((flags & ~uint32_t(SGDB_UPLOAD_EXACT_FP64 | SGDB_UPLOAD_PADDED)) == 0, "unknown upload flags");
    if (flags & SGDB_UPLOAD_PADDED) {
      require(v->layout == SGDB_LAYOUT_CSR, "SGDB_UPLOAD_PADDED converts a CSR view");
      if (flags & SGDB_UPLOAD_EXACT_FP64)
        throw Unsupported("SGDB_UPLOAD_PADDED with the exact-fp64 mode: convert on the host");
    }
    const uint64_t n = v->n_examples, d = v->n_features;
    require(n == 0 || v->labels != nullptr, "labels missing");
    if (n_global == 0) n_global = n;
    require(row_base + n <= n_global, "shard exceeds n_global");
    require(n_global <= 0xFFFFFFFFull, "example ids must fit in 32 bits");
    auto* ds = new sgdb_dataset();
    std::unique_ptr<sgdb_dataset> guard(ds);
    ds->ctx = ctx;
    ds->uid = next_dataset_uid();
    ds->n = n;
    ds->d = d;
    ds->row_base = row_base;
    ds->n_global = n_global;
    ds->layout_in = v->layout;
    cudaStream_t s = ctx->stream;

    const uint64_t nlab = ((n + 3) & ~uint64_t(3)) + 8;
    std::vector<float> lab(nlab, 0.f);
    for (uint64_t e = 0; e < n; ++e) lab[e] = static_cast<float>(v->labels[e]);
    ds->labels.alloc(nlab);
    h2d(ds->labels.p, lab.data(), nlab, s);

    switch (v->layout) {
      case SGDB_LAYOUT_DENSE_ROW:
      case SGDB_LAYOUT_DENSE_COL: {
        require(v->n_values == n * d, "dense storage size mismatch");
        const bool colmajor = v->layout == SGDB_LAYOUT_DENSE_COL;
        if (d <= 1024) {
          ds->kind = Kind::Dense;
          ds->nnz = n * d;
          std::vector<float> x(n * d + 8, 0.f);
          for (uint64_t e = 0; e < n; ++e)
            for (uint64_t j = 0; j < d; ++j)
              x[e * d + j] = static_cast<float>(colmajor ? v->values[j * n + e] : v->values[e * d + j]);
          ds->x.alloc(x.size());
          h2d(ds->x.p, x.data(), x.size(), s);
          check(cudaStreamSynchronize(s), "upload sync");
        } else {
          // Wide dense data: CSR with every coordinate stored (zeros kept so the
          // dot products visit all d slots as for_example does).
          require(n * d < 0xFFFFFFFFull, "dense matrix too large for 32-bit offsets");
          std::vector<uint32_t> rowptr(n + 1), idx(n * d);
          std::vector<float> val(n * d);
          for (uint64_t e = 0; e < n; ++e) {
            rowptr[e] = static_cast<uint32_t>(e * d);
            for (uint64_t j = 0; j < d; ++j) {
              idx[e * d + j] = static_cast<uint32_t>(j);
              val[e * d + j] =
                  static_cast<float>(colmajor ? v->values[j * n + e] : v->values[e * d + j]);
            }
          }
          rowptr[n] = static_cast<uint32_t>(n * d);
          upload_csr(ds, rowptr, idx, val);
        }
        break;
      }
      case SGDB_LAYOUT_CSR: {
        require(v->n_row_offsets == n + 1 && v->row_offsets, "csr row_offsets size mismatch");
        require(v->n_indices == v->n_values, "csr index/value size mismatch");
        const uint64_t nnz = v->n_values;
        require(nnz < 0xFFFFFFFFull, "nnz must fit in 32-bit row offsets");
        std::vector<uint32_t> rowptr(n + 1), idx(v->indices, v->indices + nnz);
        std::vector<float> val(nnz);
        for (uint64_t e = 0; e <= n; ++e) rowptr[e] = static_cast<uint32_t>(v->row_offsets[e]);
        for (uint64_t s2 = 0; s2 < nnz; ++s2) {
          require(idx[s2] < d, "csr feature index out of range");
          val[s2] = static_cast<float>(v->values[s2]);
        }
        upload_csr(ds, rowptr, idx, val);
        break;
      }
      case SGDB_LAYOUT_PADDED: {
        const uint64_t pw = v->padded_width;
        require(v->n_values == n * pw && v->n_indices == n * pw, "padded storage size mismatch");
        std::vector<uint32_t> rowptr(n + 1, 0), idx;
        std::vector<float> val;
        for (uint64_t e = 0; e < n; ++e) {
          for (uint64_t sl = 0; sl < pw; ++sl) {
            const uint32_t j = v->indices[sl * n + e];
            if (j == d) continue;  // sentinel
            require(j < d, "padded feature index out of range");
            idx.push_back(j);
            val.push_back(static_cast<float>(v->values[sl * n + e]));
          }
          rowptr[e + 1] = static_cast<uint32_t>(idx.size());
        }
        std::vector<float> pval(std::max<uint64_t>(1, n * pw));
        for (uint64_t i = 0; i < n * pw; ++i) pval[i] = static_cast<float>(v->values[i]);
        ds->pw = pw;
        ds->pval.alloc(pval.size());
        ds->pidx.alloc(std::max<uint64_t>(1, n * pw));
        h2d(ds->pval.p, pval.data(), n * pw, s);
        h2d(ds->pidx.p, v->indices, n * pw, s);
        ds->col_built = true;
        upload_csr(ds, rowptr, idx, val);
        break;
      }
      default:
        throw std::invalid_argument("unknown layout");
    }
    if (flags & SGDB_UPLOAD_PADDED) {
      build_padded_from_csr(*ds);  // device-side csr_to_padded
      ds->layout_in = SGDB_LAYOUT_PADDED;
    }
    if (flags & SGDB_UPLOAD_EXACT_FP64) {
      // fp64 copy aligned with the fp32 storage built above.
      std::vector<double> v64;
      if (v->layout == SGDB_LAYOUT_DENSE_ROW || v->layout == SGDB_LAYOUT_DENSE_COL) {
        const bool colmajor = v->layout == SGDB_LAYOUT_DENSE_COL;
        v64.resize(n * d);
        for (uint64_t e = 0; e < n; ++e)
          for (uint64_t j = 0; j < d; ++j)
            v64[e * d + j] = colmajor ? v->values[j * n + e] : v->values[e * d + j];
      } else if (v->layout == SGDB_LAYOUT_CSR) {
        v64.assign(v->values, v->values + v->n_values);
      } else {
        const uint64_t pw = v->padded_width;
        for (uint64_t e = 0; e < n; ++e)
          for (uint64_t sl = 0; sl < pw; ++sl)
            if (v->indices[sl * n + e] != d) v64.push_back(v->values[sl * n + e]);
      }
      DBuf<double>& dst = ds->kind == Kind::Dense ? ds->x64 : ds->val64;
      dst.alloc(std::max<uint64_t>(1, v64.size()));
      h2d(dst.p, v64.data(), v64.size(), s);
      check(cudaStreamSynchronize(s), "upload sync");
      ds->exact = true;
    }
    ds->order.alloc(std::max<uint64_t>(1, n_global));
    check(cudaStreamSynchronize(s), "upload sync");
    *out = guard.release();
  });
}

sgdb_status sgdb_dataset_refresh_f32(sgdb_ctx* ctx, sgdb_dataset* ds, const float* values,
                                     const float* labels, const uint32_t* indices,
                                     const uint32_t* row_offsets32) {
  return sgdb_guard([&] {
    require(ctx && ds, "null argument");
    if (ds->exact || ds->layout_in == SGDB_LAYOUT_PADDED)
      throw Unsupported("refresh: exact-fp64 and padded-layout datasets keep derived copies; upload again");
    cudaStream_t s = ctx->stream;
    if (labels) h2d(ds->labels.p, labels, ds->n, s);
    if (ds->kind == Kind::Dense) {
      if (values) {
        h2d(ds->x.p, values, ds->n * ds->d, s);
        ds->col_built = false;  // the column-major copy is rebuilt on next use
      }
      return;
    }
    if (row_offsets32) {
      // Row offsets size the mini-batch chunk plans (max_row): validate and
      // recompute from the host array before it is copied.
      require(row_offsets32[0] == 0 && row_offsets32[ds->n] == ds->nnz,
              "refresh: row offsets must start at 0 and end at nnz");
      uint64_t mr = 0;
      for (uint64_t r = 0; r < ds->n; ++r) {
        require(row_offsets32[r + 1] >= row_offsets32[r], "refresh: row offsets must be non-decreasing");
        mr = std::max<uint64_t>(mr, row_offsets32[r + 1] - row_offsets32[r]);
      }
      ds->max_row = mr;
      ds->mb_ids = nullptr;  // chunk plans refer to the old row extents
      h2d(ds->rowptr.p, row_offsets32, ds->n + 1, s);
    }
    if (values) h2d(ds->val.p, values, ds->nnz, s);
    if (indices) h2d(ds->idx.p, indices, ds->nnz, s);
    // The full-batch structures (bitmaps, 16-bit ids, blocked CSC) are
    // rebuilt on the device at the next full-batch step.
    if (values || indices || row_offsets32) ds->sparse_ready = false;
  });
}

sgdb_status sgdb_dataset_refresh_idx16(sgdb_ctx* ctx, sgdb_dataset* ds, const uint16_t* indices16) {
  return sgdb_guard([&] {
    require(ctx && ds && indices16, "null argument");
    require(ds->kind == Kind::Csr, "refresh_idx16: the dataset is not stored as CSR");
    require(ds->d <= 65536, "refresh_idx16: column ids need d <= 65536");
    if (ds->exact || ds->layout_in == SGDB_LAYOUT_PADDED)
      throw Unsupported("refresh: exact-fp64 and padded-layout datasets keep derived copies; upload again");
    cudaStream_t s = ctx->stream;
    ds->idx16.alloc(ds->nnz + 8);
    h2d(ds->idx16.p, indices16, ds->nnz, s);
    widen_u16(*ctx, ds->idx16.p, ds->idx.p, ds->nnz);
    ds->sparse_ready = false;  // as sgdb_dataset_refresh_f32
  });
}

sgdb_status sgdb_dataset_free(sgdb_dataset* ds) {
  return sgdb_guard([&] {
    if (!ds) return;
    cudaStreamSynchronize(ds->ctx->stream);
    delete ds;
  });
}

sgdb_status sgdb_dataset_sweep_bytes(const sgdb_dataset* ds, uint64_t* out) {
  return sgdb_guard([&] {
    if (ds->kind == Kind::Dense) *out = ds->n * ds->d * 4 + ds->n * 4;
    else *out = ds->nnz * 8 + (ds->n + 1) * 4 + ds->n * 4;
  });
}

sgdb_status sgdb_dataset_shape(const sgdb_dataset* ds, uint64_t* n_local, uint64_t* d,
                               uint64_t* nnz, uint64_t* row_base, uint64_t* n_global) {
  return sgdb_guard([&] {
    if (n_local) *n_local = ds->n;
    if (d) *d = ds->d;
    if (nnz) *nnz = ds->nnz;
    if (row_base) *row_base = ds->row_base;
    if (n_global) *n_global = ds->n_global;
  });
}

sgdb_status sgdb_model_create(sgdb_ctx* ctx, uint64_t d, const double* init, sgdb_model** out) {
  return sgdb_guard([&] {
    auto* m = new sgdb_model();
    std::unique_ptr<sgdb_model> guard(m);
    model_init(m, ctx, d);
    if (init) model_set(m, init);
    check(cudaStreamSynchronize(ctx->stream), "model sync");
    *out = guard.release();
  });
}

sgdb_status sgdb_model_set(sgdb_ctx*, sgdb_model* m, const double* w) {
  return sgdb_guard([&] { model_set(m, w); });
}

sgdb_status sgdb_model_get(sgdb_ctx*, sgdb_model* m, double* w_out) {
  return sgdb_guard([&] {
    Ctx& c = *m->ctx;
    materialize(*m);
    if (m->d)
      check(cudaMemcpyAsync(w_out, m->w64.p, m->d * sizeof(double), cudaMemcpyDeviceToHost,
                            c.stream),
            "D2H model");
    check(cudaStreamSynchronize(c.stream), "model_get sync");
  });
}

sgdb_status sgdb_model_device_ptrs(sgdb_model* m, float** w32, double** w64) {
  return sgdb_guard([&] {
    materialize(*m);
    dense_written(*m);  // the caller may write through the pointers
    if (w32) *w32 = m->w32.p;
    if (w64) *w64 = m->w64.p;
  });
}

sgdb_status sgdb_model_free(sgdb_model* m) {
  return sgdb_guard([&] {
    if (!m) return;
    cudaStreamSynchronize(m->ctx->stream);
    delete m;
  });
}

sgdb_status sgdb_sync_epoch(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                            double alpha, const uint32_t* order, uint64_t batch_b,
                            int32_t* finite_out) {
  return sgdb_guard([&] {
    require(ctx && ds && m, "null argument");
    require(m->d == ds->d, "model/dataset dim mismatch");
    require(batch_b >= 1, "batch size must be in [1, N]");
    Ctx& c = *ctx;
    materialize(*m);
    dense_written(*m);
    set_finite(m);
    if (ds->exact) {
      exact_sync_epoch(*ds, *m, task, alpha, order, std::min<uint64_t>(batch_b, ds->n));
      if (finite_out) *finite_out = read_finite(m);
      return;
    }
    // With a cross-rank collective every step's gradient is SUM-reduced
    // before the identical update on every rank.
    const bool hook = has_collective(c);
    StepArgs a;
    a.task = task;
    a.alpha = alpha;
    a.apply = !hook;
    if (batch_b >= ds->n_global) {
      full_step(ds, m, a);
      if (hook) {
        call_allreduce(c, m->g64.p, m->d, 1);
        apply_update(*m, alpha, false);
      }
    } else {
      const uint64_t ng = ds->n_global;
      if (order) {
        h2d(ds->order.p, order, ng, c.stream);
        ds->order_iota = false;
      } else if (!ds->order_iota) {  // identity order: uploaded once, kept
        std::vector<uint32_t> iota(ng);
        std::iota(iota.begin(), iota.end(), 0u);
        h2d(ds->order.p, iota.data(), ng, c.stream);
        check(cudaStreamSynchronize(c.stream), "order sync");
        ds->order_iota = true;
      }
      // Chunk plan of this epoch's order for the sparse steps (outside any
      // captured graph: it may allocate; the graph re-reads it every replay).
      if (ds->kind == Kind::Csr) csr_batch_plan(*ds, ds->order.p, ng, batch_b);
      // Sparse steps without a collective update the fp64 master directly;
      // the fp32 copy is refreshed once at the end of the epoch.
      const bool direct = !hook && ds->kind == Kind::Csr;
      auto run_steps = [&](const StepArgs& sa0) {
        StepArgs sa = sa0;
        sa.direct = direct;
        for (uint64_t lo = 0; lo < ng; lo += batch_b) {
          const uint64_t nb = std::min(batch_b, ng - lo);
          const uint32_t* ids = ds->order.p + lo;
          if (ds->kind == Kind::Dense) dense_batch_step(*ds, *m, ids, nb, sa);
          else csr_batch_step(*ds, *m, ids, nb, sa);
          if (hook) {
            call_allreduce(c, m->g64.p, m->d, 1);
            apply_update(*m, alpha, false, sa.alpha_dev);
          }
        }
        if (direct) sync_w32_from_w64(*m);
      };
      if (!hook && ds->kind == Kind::Dense && ng > batch_b &&
          dense_epoch(*ds, *m, task, alpha, batch_b)) {
        // K1c: the whole epoch in one persistent launch
      } else if (c.allreduce || ng / batch_b < 4) {
        // (a host hook cannot be captured; NCCL steps are graph-replayed)
        run_steps(a);
      } else {
        // Launch-bound many-step epoch: replay a captured CUDA graph of the
        // whole step sequence (captured once per dataset / batch size / task;
        // the step size is read from device memory).
        if (!(m->epoch_graph && m->graph_ds == ds->uid && m->graph_b == batch_b &&
              m->graph_task == task && m->graph_comm == c.nccl_comm)) {
          if (m->epoch_graph) cudaGraphExecDestroy(m->epoch_graph);
          m->epoch_graph = nullptr;
          m->alpha_dev.alloc(1);
          StepArgs ga = a;
          ga.alpha_dev = m->alpha_dev.p;
          const cudaStream_t saved = c.stream;
          const bool prof = c.profiling;
          const uint64_t l0 = c.launches;
          c.stream = c.capture_stream;
          c.profiling = false;
          cudaGraph_t graph = nullptr;
          check(cudaStreamBeginCapture(c.capture_stream, cudaStreamCaptureModeThreadLocal),
                "cudaStreamBeginCapture");
          try {
            run_steps(ga);
          } catch (...) {
            cudaStreamEndCapture(c.capture_stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            c.stream = saved;
            c.profiling = prof;
            throw;
          }
          check(cudaStreamEndCapture(c.capture_stream, &graph), "cudaStreamEndCapture");
          c.stream = saved;
          c.profiling = prof;
          m->graph_nodes = c.launches - l0;
          c.launches = l0;
          check(cudaGraphInstantiate(&m->epoch_graph, graph, 0), "cudaGraphInstantiate");
          cudaGraphDestroy(graph);
          m->graph_ds = ds->uid;
          m->graph_b = batch_b;
          m->graph_task = task;
          m->graph_comm = c.nccl_comm;
        }
        h2d(m->alpha_dev.p, &alpha, 1, c.stream);  // pageable source: staged before return
        prof_begin(c, "sync_epoch_graph");
        check(cudaGraphLaunch(m->epoch_graph, c.stream), "cudaGraphLaunch");
        launched(c, "sync_epoch_graph");
        c.launches += m->graph_nodes - 1;
      }
    }
    // finite_out == NULL: fully asynchronous on the context stream.
    if (finite_out) *finite_out = read_finite(m);
  });
}

sgdb_status sgdb_batch_gradient(sgdb_ctx* ctx, sgdb_dataset* ds, int32_t task,
                                const uint32_t* rows, uint64_t n_rows, const double* w,
                                int32_t transposed, double* g_out) {
  return sgdb_guard([&] {
    require(ctx && ds && w && g_out, "null argument");
    if (ds->exact) {
      exact_batch_gradient(*ds, rows, n_rows, w, task, transposed != 0, g_out);
      return;
    }
    Ctx& c = *ctx;
    sgdb_model tmp;
    model_init(&tmp, ctx, ds->d);
    model_set(&tmp, w);
    StepArgs a;
    a.task = task;
    a.apply = false;
    if (n_rows == 0) {
      full_step(ds, &tmp, a);
    } else {
      DBuf<uint32_t> ids;
      ids.alloc(n_rows);
      h2d(ids.p, rows, n_rows, c.stream);
      if (ds->kind == Kind::Dense) {
        dense_batch_step(*ds, tmp, ids.p, n_rows, a);
      } else {
        csr_batch_plan(*ds, ids.p, n_rows, n_rows);
        csr_batch_step(*ds, tmp, ids.p, n_rows, a);
        ds->mb_ids = nullptr;  // the plan refers to this call's ids
      }
      check(cudaStreamSynchronize(c.stream), "batch_gradient sync");
    }
    call_allreduce(c, tmp.g64.p, ds->d, 1);
    if (ds->d)
      check(cudaMemcpyAsync(g_out, tmp.g64.p, ds->d * sizeof(double), cudaMemcpyDeviceToHost,
                            c.stream),
            "D2H gradient");
    check(cudaStreamSynchronize(c.stream), "batch_gradient sync");
  });
}

sgdb_status sgdb_epoch_batch(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                             double alpha, double* grad_norm_out) {
  return sgdb_guard([&] {
    require(m->d == ds->d, "model/dataset dim mismatch");
    Ctx& c = *ctx;
    if (ds->exact) {
      exact_epoch_batch(*ds, *m, task, alpha);
      double sq = 0.0;
      check(cudaMemcpyAsync(&sq, m->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream),
            "D2H norm");
      check(cudaStreamSynchronize(c.stream), "epoch_batch sync");
      if (grad_norm_out) *grad_norm_out = std::sqrt(sq);
      return;
    }
    materialize(*m);
    dense_written(*m);
    check(cudaMemsetAsync(m->scal.p, 0, sizeof(double), c.stream), "memset norm");
    StepArgs a;
    a.task = task;
    a.alpha = alpha;
    a.apply = !has_collective(c);
    a.want_norm = true;
    set_finite(m);
    full_step(ds, m, a);
    if (has_collective(c)) {
      call_allreduce(c, m->g64.p, m->d, 1);
      apply_update(*m, alpha, true);
    }
    double sq = 0.0;
    check(cudaMemcpyAsync(&sq, m->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream),
          "D2H norm");
    check(cudaStreamSynchronize(c.stream), "epoch_batch sync");
    if (grad_norm_out) *grad_norm_out = std::sqrt(sq);
  });
}

sgdb_status sgdb_hogwild_epoch(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                               double alpha, const sgdb_plan* plan, uint64_t* evals_out) {
  return sgdb_hogwild_segment(ctx, ds, m, task, alpha, plan, 0, 1, evals_out);
}

sgdb_status sgdb_hogwild_segment(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                                 double alpha, const sgdb_plan* plan, uint32_t seg, uint32_t nseg,
                                 uint64_t* evals_out) {
  return sgdb_guard([&] {
    require(ctx && ds && m && plan, "null argument");
    require(nseg >= 1 && seg < nseg, "segment out of range");
    require(m->d == ds->d, "model/dataset dim mismatch");
    require(ds->n >= 1, "cannot train on an empty dataset");
    validate_device_plan(*plan, ds->layout_in);
    HogwildArgs a;
    a.task = task;
    a.alpha = static_cast<float>(alpha);
    a.access = plan->access_path;
    a.replication = plan->replication;
    a.k = plan->data_replication_k;
    a.workers = plan->workers;
    a.group_size = plan->group_size;
    a.offsets = plan->circular_offsets != 0;
    a.lanes = plan->lanes_per_worker > 0 ? plan->lanes_per_worker
                                         : hogwild_auto_lanes(*ds, plan->access_path);
    require(a.lanes == 1 || a.lanes == 2 || a.lanes == 4 || a.lanes == 8 || a.lanes == 16 ||
                a.lanes == 32,
            "lanes_per_worker must be 1, 2, 4, 8, 16 or 32");
    a.seg = seg;
    a.nseg = nseg;
    a.alpha_f64 = alpha;
    if (ds->exact) exact_hogwild(*ds, *m, a);
    else hogwild_epoch(*ds, *m, a);
    if (evals_out) {
      const bool rr = plan->access_path == SGDB_ACCESS_ROW_RR || plan->access_path == SGDB_ACCESS_COL_RR;
      *evals_out = segment_evals(ds->n, plan->workers, rr, plan->data_replication_k, seg, nseg);
    }
  });
}

sgdb_status sgdb_models_average(sgdb_ctx* ctx, sgdb_model* const* models, uint64_t count,
                                const double* weights, sgdb_model* out, int32_t refresh) {
  return sgdb_guard([&] {
    require(count > 0, "merge_models: no replicas");
    std::vector<Model*> ms(count);
    for (uint64_t i = 0; i < count; ++i) {
      ms[i] = models[i];
      materialize(*ms[i]);
      if (refresh) dense_written(*ms[i]);
    }
    materialize(*out);
    dense_written(*out);
    average_models(*ctx, ms.data(), count, weights, *out, refresh != 0);
  });
}

sgdb_status sgdb_loss(sgdb_ctx* ctx, sgdb_dataset* ds, sgdb_model* m, int32_t task,
                      double* loss_out) {
  return sgdb_guard([&] {
    require(m->d == ds->d, "model/dataset dim mismatch");
    Ctx& c = *ctx;
    materialize(*m);
    if (ds->exact) exact_loss(*ds, *m, task);
    else loss_launch(*ds, *m, task);
    call_allreduce(c, c.loss_out.p, 1, 1);
    double l = 0.0;
    check(cudaMemcpyAsync(&l, c.loss_out.p, sizeof(double), cudaMemcpyDeviceToHost, c.stream),
          "D2H loss");
    check(cudaStreamSynchronize(c.stream), "loss sync");
    *loss_out = l;
  });
}

}  // extern "C"

namespace sgdb::dev {

namespace {
std::mutex g_cfg_mu;
std::map<std::pair<int, const void*>, size_t> g_dyn_smem;
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;
std::map<std::pair<int, const void*>, size_t> g_static_smem;
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
}  // namespace

void set_max_dyn_smem(const void* kern, size_t smem, const char* what) {
  if (smem <= 48 * 1024) return;
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  size_t& cur = g_dyn_smem[{current_device(), kern}];
  if (smem <= cur) return;
  check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)), what);
  cur = smem;
}

int blocks_per_sm(const void* kern, int threads, size_t smem) {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  const auto key = std::make_tuple(current_device(), kern, threads, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem), "occupancy");
  g_occ[key] = per_sm;
  return per_sm;
}

size_t static_smem_of(const void* kern) {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  const auto key = std::make_pair(current_device(), kern);
  auto it = g_static_smem.find(key);
  if (it != g_static_smem.end()) return it->second;
  cudaFuncAttributes fa{};
  check(cudaFuncGetAttributes(&fa, kern), "cudaFuncGetAttributes");
  g_static_smem[key] = fa.sharedSizeBytes;
  return fa.sharedSizeBytes;
}

}  // namespace sgdb::dev

namespace sgdb::dev {
uint64_t next_dataset_uid() {
  static std::atomic<uint64_t> counter{1};
  return counter.fetch_add(1);
}

}  // namespace sgdb::dev
