// fp64 device kernels that follow the reference's arithmetic exactly:
//
// 1. The §4 linear-algebra operator API (proj/include/sgdbench/linalg.hpp:23-58,
//    proj/src/linalg.cpp:26-183): the primitives the paper's GPU sync SGD
//    chains (§4, Eq. 2), for callers of the reference's linalg:: API.
// 2. The exact-fp64 mode of the engine (datasets uploaded with
//    SGDB_UPLOAD_EXACT_FP64): sync epochs run the reference's own primitive
//    chain (sync_engine.cpp:22-121), Hogwild runs a warp-per-worker fp64
//    process_examples (async_engine.cpp:178-195), and the loss sums in id
//    order (glm.cpp:85-94) — on an fp64 copy of the data, with glibc's exp
//    restated bit-for-bit (libm_exp.hpp). The fused fp32 kernels remain the
//    fast path; this mode is what makes results bit-identical to the
//    reference (up to log1p in the LR loss).
//
// Summation orders reproduced:
//   matvec             one writer per row, ascending slots        (linalg.cpp:30-44)
//   matvec_transposed  per column sequential when the data is (or is passed
//                      as) column-major (linalg.cpp:58-76); otherwise 256-row
//                      block partials + the fixed pairwise tree   (linalg.cpp:78-109)
//   elementwise, axpy  one rounding per reference operation       (linalg.cpp:113-183)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "device.hpp"
#include "libm_exp.hpp"

namespace sgdb::dev {
namespace {

constexpr uint32_t kReduceBlock = 256;  // linalg.hpp:18

__device__ __forceinline__ double as_d(float v) { return static_cast<double>(v); }
__device__ __forceinline__ double as_d(double v) { return v; }

// ---- matvec ---------------------------------------------------------------

template <class T>
__global__ void matvec_dense_kernel(const T* __restrict__ x, uint64_t n_local, uint64_t row_base,
                                    uint32_t d, const uint32_t* __restrict__ rows, uint64_t nr,
                                    const double* __restrict__ v, double* __restrict__ out) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nr;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = (rows ? rows[p] : p) - row_base;
    double z = 0.0;
    if (r < n_local)
      for (uint32_t j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(as_d(x[r * d + j]), v[j]));
    out[p] = z;
  }
}

template <class T>
__global__ void matvec_csr_kernel(const T* __restrict__ val, const uint32_t* __restrict__ idx,
                                  const uint32_t* __restrict__ rowptr, uint64_t n_local,
                                  uint64_t row_base, const uint32_t* __restrict__ rows, uint64_t nr,
                                  const double* __restrict__ v, double* __restrict__ out) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nr;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = (rows ? rows[p] : p) - row_base;
    double z = 0.0;
    if (r < n_local)
      for (uint32_t s = rowptr[r]; s < rowptr[r + 1]; ++s)
        z = __dadd_rn(z, __dmul_rn(as_d(val[s]), v[idx[s]]));
    out[p] = z;
  }
}

// ---- matvec_transposed ------------------------------------------------------

// Column order: thread j walks the positions in order, reading column j of
// the row-major store.
template <class T>
__global__ void matvec_t_col_kernel(const T* __restrict__ x, uint64_t n_local, uint64_t row_base,
                                    uint32_t d, const uint32_t* __restrict__ rows, uint64_t nr,
                                    const double* __restrict__ a, double* __restrict__ out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint64_t p = 0; p < nr; ++p) {
      const uint64_t r = (rows ? rows[p] : p) - row_base;
      if (r < n_local) s = __dadd_rn(s, __dmul_rn(a[p], as_d(x[r * d + j])));
    }
    out[j] = s;
  }
}

// Tree order. The pairwise combine over blocks equals a binary counter:
// pushing block k merges it with the stacked complete subtrees for the
// trailing one bits of k (left += right), and the final collapse adds the
// remaining subtrees right to left. The per-coordinate stack (one value per
// bit level) lives in global memory so blocks stream in bounded chunks.

// Phase 1, dense: thread (block-in-chunk, j) sums its block sequentially.
template <class T>
__global__ void partials_dense_kernel(const T* __restrict__ x, uint64_t n_local, uint64_t row_base,
                                      uint32_t d, const uint32_t* __restrict__ rows, uint64_t nr,
                                      uint64_t blk0, const double* __restrict__ a,
                                      double* __restrict__ part) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const uint64_t blk = blk0 + blockIdx.y;
  const uint64_t lo = blk * kReduceBlock, hi = min(nr, lo + kReduceBlock);
  double s = 0.0;
  for (uint64_t p = lo; p < hi; ++p) {
    const uint64_t r = (rows ? rows[p] : p) - row_base;
    if (r < n_local) s = __dadd_rn(s, __dmul_rn(a[p], as_d(x[r * d + j])));
  }
  part[(uint64_t)blockIdx.y * d + j] = s;
}

// Phase 1, CSR: one warp per block walks its rows in order; the slots of a row
// have distinct columns, so lanes split them and __syncwarp orders rows.
template <class T>
__global__ void partials_csr_kernel(const T* __restrict__ val, const uint32_t* __restrict__ idx,
                                    const uint32_t* __restrict__ rowptr, uint64_t n_local,
                                    uint64_t row_base, uint32_t d, const uint32_t* __restrict__ rows,
                                    uint64_t nr, uint64_t blk0, const double* __restrict__ a,
                                    double* __restrict__ part) {
  const uint64_t blk = blk0 + blockIdx.x;
  const uint32_t lane = threadIdx.x;
  double* dst = part + (uint64_t)blockIdx.x * d;
  const uint64_t lo = blk * kReduceBlock, hi = min(nr, lo + kReduceBlock);
  for (uint64_t p = lo; p < hi; ++p) {
    const uint64_t r = (rows ? rows[p] : p) - row_base;
    if (r < n_local) {
      const double ap = a[p];
      for (uint32_t s = rowptr[r] + lane; s < rowptr[r + 1]; s += 32) {
        const uint32_t j = idx[s];
        dst[j] = __dadd_rn(dst[j], __dmul_rn(ap, as_d(val[s])));
      }
    }
    __syncwarp();
  }
}

// Phase 2: push the chunk's block partials onto each coordinate's stack.
// stack[l*d + j] holds the complete subtree of 2^l blocks for set bit l of k.
__global__ void tree_push_kernel(const double* __restrict__ part, uint32_t nblk, uint32_t d,
                                 uint64_t k0, double* __restrict__ stack) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  uint64_t k = k0;
  for (uint32_t b = 0; b < nblk; ++b, ++k) {
    double v = part[(uint64_t)b * d + j];
    uint32_t level = 0;
    while ((k >> level) & 1u) {  // left subtree (earlier blocks) += right
      v = __dadd_rn(stack[(uint64_t)level * d + j], v);
      ++level;
    }
    stack[(uint64_t)level * d + j] = v;
  }
}

// Phase 3: out[j] = S_high + (... + (S_low)) over the set bits of nblocks.
__global__ void tree_collapse_kernel(const double* __restrict__ stack, uint32_t d, uint64_t nblocks,
                                     double* __restrict__ out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  bool have = false;
  double acc = 0.0;
  for (uint32_t level = 0; level < 64; ++level) {
    if (!((nblocks >> level) & 1u)) continue;
    const double v = stack[(uint64_t)level * d + j];
    acc = have ? __dadd_rn(v, acc) : v;
    have = true;
  }
  out[j] = acc;
}

// ---- elementwise / axpy -----------------------------------------------------

// ElementwiseOp (linalg.hpp:40) + the fused sigmoid / hinge indicator.
__global__ void elementwise_kernel(int op, const double* __restrict__ a, const double* __restrict__ b,
                                   double scalar, uint64_t n, double* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double x = a[i];
    double r;
    switch (op) {
      case SGDB_EW_MUL: r = __dmul_rn(x, b[i]); break;
      case SGDB_EW_DIV: r = __ddiv_rn(x, b[i]); break;
      case SGDB_EW_EXP: r = libm::exp(x); break;
      case SGDB_EW_NEG: r = -x; break;
      case SGDB_EW_ADD_SCALAR: r = __dadd_rn(scalar, x); break;
      case SGDB_EW_SIGMOID: r = libm::stable_sigmoid(x); break;  // math.hpp:10-16
      default: r = x < 1.0 ? 1.0 : 0.0; break;                   // SGDB_EW_HINGE_INDICATOR
    }
    out[i] = r;
  }
}

// w <- w - alpha g (no FMA: the reference rounds twice). With `live`, a
// no-op once an earlier batch of the epoch produced a non-finite gradient.
__global__ void axpy_kernel(double* w, double alpha, const double* __restrict__ g, uint64_t n,
                            const int* live) {
  if (live && *live == 0) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    w[i] = __dsub_rn(w[i], __dmul_rn(alpha, g[i]));
}

// ---- exact-mode sync helpers --------------------------------------------------

// c_p from the reference chain (sync_engine.cpp:30-40): m = y.a; LR
// c = sigma(-m) * (-y), SVM c = [m < 1] * (-y).
__global__ void chain_coef_kernel(int task, const float* __restrict__ labels, uint64_t row_base,
                                  const uint32_t* __restrict__ rows, uint64_t nr,
                                  const double* __restrict__ a, double* __restrict__ c) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nr;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const double y = static_cast<double>(labels[(rows ? rows[p] : p) - row_base]);
    const double m = __dmul_rn(y, a[p]);
    const double act = task == 0 ? libm::stable_sigmoid(-m) : (m < 1.0 ? 1.0 : 0.0);
    c[p] = __dmul_rn(act, -y);
  }
}

// finite &= all(isfinite(g)); the batch's own axpy still applies (the
// reference checks, applies, then stops: sync_engine.cpp:94-97).
__global__ void finite_kernel(const double* __restrict__ g, uint64_t d, int* finite) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x)
    if (!isfinite(g[j])) *finite = 0;
}

__global__ void snapshot_kernel(const int* finite, int* live) { *live = *finite; }

// sum_j g_j^2 in index order (sync_engine.cpp:50-51).
__global__ void sq_norm_kernel(const double* __restrict__ g, uint64_t d, double* out) {
  double s = 0.0;
  for (uint64_t j = 0; j < d; ++j) s = __dadd_rn(s, __dmul_rn(g[j], g[j]));
  *out = s;
}

__global__ void w32_from_w64_kernel(const double* __restrict__ w64, uint64_t d,
                                    float* __restrict__ w32) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x)
    w32[j] = static_cast<float>(w64[j]);
}

// ---- exact-mode loss: per-example point loss, then the id-order sum ---------

__device__ __forceinline__ double point_loss(int task, double z, double y) {
  const double m = __dmul_rn(y, z);  // glm.cpp:24-28
  if (task == 0) {
    const double u = -m;  // stable_softplus (math.hpp:18-22)
    return u > 0.0 ? __dadd_rn(u, log1p(libm::exp(-u))) : log1p(libm::exp(u));
  }
  return m < 1.0 ? __dsub_rn(1.0, m) : 0.0;
}

template <class T, bool DENSE>
__global__ void example_loss_kernel(int task, const T* __restrict__ val,
                                    const uint32_t* __restrict__ idx,
                                    const uint32_t* __restrict__ rowptr,
                                    const float* __restrict__ labels, uint64_t n, uint32_t d,
                                    const double* __restrict__ w, double* __restrict__ out) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    double z = 0.0;
    if (DENSE) {
      for (uint32_t j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(as_d(val[e * d + j]), w[j]));
    } else {
      for (uint32_t s = rowptr[e]; s < rowptr[e + 1]; ++s)
        z = __dadd_rn(z, __dmul_rn(as_d(val[s]), w[idx[s]]));
    }
    out[e] = point_loss(task, z, static_cast<double>(labels[e]));
  }
}

__global__ void ordered_sum_kernel(const double* __restrict__ v, uint64_t n, double* out) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s = __dadd_rn(s, v[i]);
  *out = s;
}

// ---- exact-mode Hogwild: process_examples (async_engine.cpp:178-195) --------
//
// One warp per worker over its assign() list segment. z is summed in slot
// order (lanes form the products, every lane adds them in sequence through
// shuffles), c from the reference's scalar core, then each lane applies
// w_j <- w_j - alpha (c x_j) to its slots. With one worker the schedule is
// sequential Alg. 3 and the result is bit-identical to the reference; with
// more workers the model is shared racily in fp64, like the reference's
// relaxed atomics.
struct ExactHog {
  const double* val;  // dense row-major (DENSE) or CSR values, fp64
  const uint32_t* idx;
  const uint32_t* rowptr;
  const float* y;
  uint64_t n, d, T, k, gs, ld;
  int rr;
  double* model;  // kernel scope: w64; replica scopes: replica 0 (+ (w/gs)*ld)
  double alpha;
  uint32_t seg, nseg;
};

template <int TASK, bool DENSE>
__global__ void __launch_bounds__(256) hogwild_exact_kernel(ExactHog p) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t hw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const uint64_t HW = ((uint64_t)gridDim.x * blockDim.x) / 32;
  for (uint64_t w = hw; w < p.T; w += HW) {
    double* m = p.model + (w / p.gs) * p.ld;
    const WorkerList l = assign_list(p.n, p.T, p.k, p.rr != 0, w);
    const uint32_t lo = static_cast<uint32_t>(uint64_t(l.total) * p.seg / p.nseg);
    const uint32_t hi = static_cast<uint32_t>(uint64_t(l.total) * (p.seg + 1) / p.nseg);
    for (uint32_t i = lo; i < hi; ++i) {
      const uint32_t e = assign_at(p.n, l, i);
      const uint64_t b = DENSE ? uint64_t(e) * p.d : p.rowptr[e];
      const uint32_t len = DENSE ? static_cast<uint32_t>(p.d) : p.rowptr[e + 1] - p.rowptr[e];
      double z = 0.0;
      for (uint32_t base = 0; base < len; base += 32) {
        double prod = 0.0;
        if (base + lane < len) {
          const uint32_t j = DENSE ? base + lane : p.idx[b + base + lane];
          prod = __dmul_rn(p.val[b + base + lane], __ldcg(m + j));
        }
        const uint32_t cnt = min(32u, len - base);
        for (uint32_t t = 0; t < cnt; ++t) z = __dadd_rn(z, __shfl_sync(0xffffffffu, prod, t));
      }
      const double y = static_cast<double>(p.y[e]);
      const double mm = __dmul_rn(y, z);  // glm.cpp:30-34
      const double c = TASK == 0 ? __dmul_rn(libm::stable_sigmoid(-mm), -y) : (mm < 1.0 ? -y : 0.0);
      for (uint32_t s = lane; s < len; s += 32) {
        const uint32_t j = DENSE ? s : p.idx[b + s];
        const double upd = __dmul_rn(p.alpha, __dmul_rn(c, p.val[b + s]));
        __stcg(m + j, __dsub_rn(__ldcg(m + j), upd));
      }
      __syncwarp();
    }
  }
}

// Example scope in the reference's order (async_engine.cpp:333-370): the
// claim/ready protocol of K5x (kernels_hogwild.cu) with fp64 replicas; margin
// summed in slot order, updates cur - alpha*(c*x), replicas stored into the
// shared model when the worker's list is done.
template <int TASK>
__global__ void __launch_bounds__(256) hogwild_exact_example_kernel(ExactHog p, double* rep,
                                                                    unsigned* claim, unsigned* ready,
                                                                    unsigned epoch) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t hw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const uint64_t HW = ((uint64_t)gridDim.x * blockDim.x) / 32;
  double* m = p.model;
  for (uint64_t w = hw; w < p.T; w += HW) {
    const WorkerList l = assign_list(p.n, p.T, p.k, p.rr != 0, w);
    const uint32_t lo = static_cast<uint32_t>(uint64_t(l.total) * p.seg / p.nseg);
    const uint32_t hi = static_cast<uint32_t>(uint64_t(l.total) * (p.seg + 1) / p.nseg);
    for (uint32_t i = lo; i < hi; ++i) {
      const uint32_t e = assign_at(p.n, l, i);
      const uint32_t b = p.rowptr[e], len = p.rowptr[e + 1] - b;
      int role = 0;
      if (lane == 0) {
        unsigned r;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(ready + e) : "memory");
        if (r != epoch) role = atomicExch(claim + e, epoch) != epoch ? 1 : 2;
      }
      role = __shfl_sync(0xffffffffu, role, 0);
      if (role == 1) {
        for (uint32_t s = lane; s < len; s += 32) __stcg(rep + b + s, __ldcg(m + p.idx[b + s]));
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + e), "r"(epoch) : "memory");
        }
      } else if (role == 2) {
        if (lane == 0) {
          unsigned r;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(ready + e) : "memory");
          } while (r != epoch);
        }
        __syncwarp();
      }
      if (len == 0) continue;
      double z = 0.0;
      for (uint32_t base = 0; base < len; base += 32) {
        double prod = 0.0;
        if (base + lane < len) prod = __dmul_rn(p.val[b + base + lane], __ldcg(rep + b + base + lane));
        const uint32_t cnt = min(32u, len - base);
        for (uint32_t t = 0; t < cnt; ++t) z = __dadd_rn(z, __shfl_sync(0xffffffffu, prod, t));
      }
      const double y = static_cast<double>(p.y[e]);
      const double mm = __dmul_rn(y, z);
      const double c = TASK == 0 ? __dmul_rn(libm::stable_sigmoid(-mm), -y) : (mm < 1.0 ? -y : 0.0);
      for (uint32_t s = lane; s < len; s += 32) {
        const double upd = __dmul_rn(p.alpha, __dmul_rn(c, p.val[b + s]));
        __stcg(rep + b + s, __dsub_rn(__ldcg(rep + b + s), upd));
      }
      __syncwarp();
    }
    for (uint32_t i = lo; i < hi; ++i) {
      const uint32_t e = assign_at(p.n, l, i);
      const uint32_t b = p.rowptr[e], len = p.rowptr[e + 1] - b;
      for (uint32_t s = lane; s < len; s += 32) __stcg(m + p.idx[b + s], __ldcg(rep + b + s));
    }
  }
}

// Replica prepare (async_engine.cpp:372-383): every replica = the global
// model, guard slot 0.
__global__ void replicas_fill_kernel(double* reps, uint64_t R, uint64_t d, const double* w) {
  const uint64_t total = R * (d + 1);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = i % (d + 1);
    reps[i] = j < d ? w[j] : 0.0;
  }
}

// merge_models (async_engine.cpp:133-156), unweighted: sum in replica order, / R.
__global__ void replicas_merge_kernel(const double* reps, uint64_t R, uint64_t d, double* w) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint64_t r = 0; r < R; ++r) s = __dadd_rn(s, __dmul_rn(1.0, reps[r * (d + 1) + j]));
    w[j] = __ddiv_rn(s, static_cast<double>(R));
  }
}

unsigned grid_1d(const Ctx& c, uint64_t n) {
  return static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, c.num_sms * 16ull)));
}

template <class T>
void h2d_vec(DBuf<T>& buf, const T* src, uint64_t n, cudaStream_t s) {
  buf.alloc(std::max<uint64_t>(1, n));
  if (n) check(cudaMemcpyAsync(buf.p, src, n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
}

void d2h_sync(double* dst, const double* src, uint64_t n, cudaStream_t s) {
  if (n) check(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
  check(cudaStreamSynchronize(s), "linalg sync");
}

void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

bool dense_layout(const Dataset& ds) {
  return ds.layout_in == SGDB_LAYOUT_DENSE_ROW || ds.layout_in == SGDB_LAYOUT_DENSE_COL;
}

// Calls f(x_rowmajor_or_null, csr_values) with the fp64 copies in exact
// mode, the fp32 arrays otherwise. Dense data wider than the dense kernels'
// limit is stored as CSR with every slot kept (rowptr[e] = e*d), so its
// values double as a row-major matrix.
template <class F>
void with_values(Dataset& ds, F&& f) {
  if (ds.exact) {
    const double* xr = ds.kind == Kind::Dense ? ds.x64.p : (dense_layout(ds) ? ds.val64.p : nullptr);
    f(xr, ds.val64.p);
  } else {
    const float* xr = ds.kind == Kind::Dense ? ds.x.p : (dense_layout(ds) ? ds.val.p : nullptr);
    f(xr, ds.val.p);
  }
}

}  // namespace

// ---- device-vector primitives (all pointers on the device) ------------------

void lin_matvec(Dataset& ds, const uint32_t* rows, uint64_t nr, const double* v, double* out) {
  Ctx& c = *ds.ctx;
  const unsigned grid = grid_1d(c, nr);
  const uint32_t d = static_cast<uint32_t>(ds.d);
  with_values(ds, [&](auto xr, auto val) {
    prof_begin(c, "matvec_kernel");
    if (ds.kind == Kind::Dense)
      matvec_dense_kernel<<<grid, 256, 0, c.stream>>>(xr, ds.n, ds.row_base, d, rows, nr, v, out);
    else
      matvec_csr_kernel<<<grid, 256, 0, c.stream>>>(val, ds.idx.p, ds.rowptr.p, ds.n, ds.row_base,
                                                    rows, nr, v, out);
    launched(c, "matvec_kernel");
  });
}

// out (d, device) = X^T a over `rows`; col_order selects the per-column
// sequential order (the reference's DenseColMajor branch; only dense data).
void lin_matvec_t(Dataset& ds, const uint32_t* rows, uint64_t nr, const double* a, bool col_order,
                  double* out) {
  Ctx& c = *ds.ctx;
  const uint32_t d = static_cast<uint32_t>(ds.d);
  const unsigned gd = (d + 255) / 256;
  if (d == 0) return;
  if (nr == 0) {
    check(cudaMemsetAsync(out, 0, uint64_t(d) * sizeof(double), c.stream), "memset");
    return;
  }
  col_order = (col_order && dense_layout(ds)) || ds.layout_in == SGDB_LAYOUT_DENSE_COL;
  with_values(ds, [&](auto xr, auto val) {
    if (col_order) {
      prof_begin(c, "matvec_t_kernel");
      matvec_t_col_kernel<<<grid_1d(c, d), 256, 0, c.stream>>>(xr, ds.n, ds.row_base, d, rows, nr,
                                                               a, out);
      launched(c, "matvec_t_kernel");
      return;
    }
    const uint64_t nblocks = (nr + kReduceBlock - 1) / kReduceBlock;
    // Partials of at most ~256 MiB per chunk (and <= 65535 grid rows).
    const uint64_t chunk = std::max<uint64_t>(
        1, std::min<uint64_t>({nblocks, (256ull << 20) / (8ull * d), 65535}));
    ds.ex_part.alloc(chunk * d);
    ds.ex_stack.alloc(64ull * d);
    for (uint64_t b0 = 0; b0 < nblocks; b0 += chunk) {
      const uint32_t nb = static_cast<uint32_t>(std::min(chunk, nblocks - b0));
      if (ds.kind == Kind::Dense) {
        prof_begin(c, "matvec_t_partials");
        partials_dense_kernel<<<dim3(gd, nb), 256, 0, c.stream>>>(xr, ds.n, ds.row_base, d, rows,
                                                                  nr, b0, a, ds.ex_part.p);
      } else {
        check(cudaMemsetAsync(ds.ex_part.p, 0, uint64_t(nb) * d * sizeof(double), c.stream),
              "memset");
        prof_begin(c, "matvec_t_partials");
        partials_csr_kernel<<<nb, 32, 0, c.stream>>>(val, ds.idx.p, ds.rowptr.p, ds.n, ds.row_base,
                                                     d, rows, nr, b0, a, ds.ex_part.p);
      }
      launched(c, "matvec_t_partials");
      prof_begin(c, "matvec_t_tree");
      tree_push_kernel<<<gd, 256, 0, c.stream>>>(ds.ex_part.p, nb, d, b0, ds.ex_stack.p);
      launched(c, "matvec_t_tree");
    }
    prof_begin(c, "matvec_t_tree");
    tree_collapse_kernel<<<gd, 256, 0, c.stream>>>(ds.ex_stack.p, d, nblocks, out);
    launched(c, "matvec_t_tree");
  });
}

// ---- exact-fp64 mode ----------------------------------------------------------

namespace {

void require_exact(const Dataset& ds) {
  if (!ds.exact) throw std::logic_error("exact-mode op on a dataset uploaded without fp64 values");
  if (ds.n != ds.n_global || ds.row_base != 0)
    throw Unsupported("the exact-fp64 mode runs on whole (unsharded) datasets");
}

void refresh_w32(Model& m) {
  Ctx& c = *m.ctx;
  prof_begin(c, "w32_from_w64");
  w32_from_w64_kernel<<<grid_1d(c, m.d), 256, 0, c.stream>>>(m.w64.p, m.d, m.w32.p);
  launched(c, "w32_from_w64");
  dense_written(m);
}

// g = batch_gradient(rows) (sync_engine.cpp:22-42) into `g` (device).
void chain_gradient(Dataset& ds, const uint32_t* rows, uint64_t nr, const double* w, int task,
                    bool col_order, double* g) {
  Ctx& c = *ds.ctx;
  ds.ex_a.alloc(std::max<uint64_t>(1, nr));
  ds.ex_c.alloc(std::max<uint64_t>(1, nr));
  lin_matvec(ds, rows, nr, w, ds.ex_a.p);
  prof_begin(c, "chain_coef_kernel");
  chain_coef_kernel<<<grid_1d(c, nr), 256, 0, c.stream>>>(task, ds.labels.p, ds.row_base, rows, nr,
                                                          ds.ex_a.p, ds.ex_c.p);
  launched(c, "chain_coef_kernel");
  lin_matvec_t(ds, rows, nr, ds.ex_c.p, col_order, g);
}

}  // namespace

void exact_batch_gradient(Dataset& ds, const uint32_t* rows_host, uint64_t n_rows, const double* w_host,
                          int task, bool transposed, double* g_host) {
  require_exact(ds);
  Ctx& c = *ds.ctx;
  DBuf<uint32_t> rows;
  DBuf<double> w, g;
  if (n_rows) h2d_vec(rows, rows_host, n_rows, c.stream);
  h2d_vec(w, w_host, ds.d, c.stream);
  g.alloc(std::max<uint64_t>(1, ds.d));
  chain_gradient(ds, n_rows ? rows.p : nullptr, n_rows ? n_rows : ds.n, w.p, task, transposed, g.p);
  d2h_sync(g_host, g.p, ds.d, c.stream);
}

// sync::train's epoch body (sync_engine.cpp:80-98): batches of the order,
// each sorted, gradient by the chain (dense data through its column-major
// transpose, as train materialises it), finite check, axpy. m.finite is left
// 0 if a gradient was non-finite; later batches are skipped like the
// reference's loop.
void exact_sync_epoch(Dataset& ds, Model& m, int task, double alpha, const uint32_t* order,
                      uint64_t batch_b) {
  require_exact(ds);
  Ctx& c = *ds.ctx;
  materialize(m);
  const uint64_t n = ds.n;
  std::vector<uint32_t> ord(n);
  if (order) std::copy(order, order + n, ord.begin());
  else std::iota(ord.begin(), ord.end(), 0u);
  for (uint64_t lo = 0; lo < n; lo += batch_b)
    std::sort(ord.begin() + lo, ord.begin() + std::min(n, lo + batch_b));
  check(cudaMemcpyAsync(ds.order.p, ord.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                        c.stream),
        "H2D order");
  ds.order_iota = false;
  ds.ex_live.alloc(1);
  for (uint64_t lo = 0; lo < n; lo += batch_b) {
    const uint64_t nb = std::min(batch_b, n - lo);
    snapshot_kernel<<<1, 1, 0, c.stream>>>(m.finite.p, ds.ex_live.p);
    launched(c, "snapshot_kernel");
    chain_gradient(ds, ds.order.p + lo, nb, m.w64.p, task, true, m.g64.p);
    finite_kernel<<<grid_1d(c, ds.d), 256, 0, c.stream>>>(m.g64.p, ds.d, m.finite.p);
    launched(c, "finite_kernel");
    prof_begin(c, "axpy_kernel");
    axpy_kernel<<<grid_1d(c, ds.d), 256, 0, c.stream>>>(m.w64.p, alpha, m.g64.p, ds.d, ds.ex_live.p);
    launched(c, "axpy_kernel");
  }
  check(cudaStreamSynchronize(c.stream), "exact epoch sync");  // `ord` is pageable
  refresh_w32(m);
}

// epoch_batch (sync_engine.cpp:44-54): full-batch gradient (dense data through
// its transpose), ||g||^2 in index order into m.scal, then the step.
void exact_epoch_batch(Dataset& ds, Model& m, int task, double alpha) {
  require_exact(ds);
  Ctx& c = *ds.ctx;
  materialize(m);
  chain_gradient(ds, nullptr, ds.n, m.w64.p, task, true, m.g64.p);
  sq_norm_kernel<<<1, 1, 0, c.stream>>>(m.g64.p, ds.d, m.scal.p);
  launched(c, "sq_norm_kernel");
  axpy_kernel<<<grid_1d(c, ds.d), 256, 0, c.stream>>>(m.w64.p, alpha, m.g64.p, ds.d, nullptr);
  launched(c, "axpy_kernel");
  refresh_w32(m);
}

// dataset_loss (glm.cpp:85-94) into ctx.loss_out[0]: point losses in
// parallel, summed in id order.
void exact_loss(Dataset& ds, Model& m, int task) {
  require_exact(ds);
  Ctx& c = *ds.ctx;
  materialize(m);
  ds.ex_c.alloc(std::max<uint64_t>(1, ds.n));
  const uint32_t d = static_cast<uint32_t>(ds.d);
  prof_begin(c, "exact_loss_kernel");
  if (ds.kind == Kind::Dense)
    example_loss_kernel<double, true><<<grid_1d(c, ds.n), 256, 0, c.stream>>>(
        task, ds.x64.p, nullptr, nullptr, ds.labels.p, ds.n, d, m.w64.p, ds.ex_c.p);
  else
    example_loss_kernel<double, false><<<grid_1d(c, ds.n), 256, 0, c.stream>>>(
        task, ds.val64.p, ds.idx.p, ds.rowptr.p, ds.labels.p, ds.n, d, m.w64.p, ds.ex_c.p);
  launched(c, "exact_loss_kernel");
  ordered_sum_kernel<<<1, 1, 0, c.stream>>>(ds.ex_c.p, ds.n, c.loss_out.p);
  launched(c, "ordered_sum_kernel");
}

void exact_hogwild(Dataset& ds, Model& m, const HogwildArgs& a) {
  require_exact(ds);
  Ctx& c = *ds.ctx;
  materialize(m);
  ExactHog p{};
  const bool dense = ds.kind == Kind::Dense;
  p.val = dense ? ds.x64.p : ds.val64.p;
  p.idx = ds.idx.p;
  p.rowptr = ds.rowptr.p;
  p.y = ds.labels.p;
  p.n = ds.n;
  p.d = ds.d;
  p.T = a.workers;
  p.k = a.k;
  p.rr = a.access == SGDB_ACCESS_ROW_RR || a.access == SGDB_ACCESS_COL_RR;
  p.alpha = a.alpha_f64;
  p.seg = a.seg;
  p.nseg = a.nseg;
  uint64_t R = 0;
  if (a.replication == SGDB_REPL_EXAMPLE) {
    if (dense) throw std::invalid_argument("example replication requires a sparse layout");
    if (ds.ex_rep64.n < ds.nnz || !ds.ex_rep64.p || ds.ex_claim.n < ds.n || !ds.ex_claim.p) {
      ds.ex_rep64.alloc(std::max<uint64_t>(1, ds.nnz));
      ds.ex_claim.alloc(ds.n);
      ds.ex_ready.alloc(ds.n);
      ds.ex_claim.zero(c.stream);
      ds.ex_ready.zero(c.stream);
      ds.ex_epoch = 0;
    }
    if (a.seg == 0) ++ds.ex_epoch;
    p.model = m.w64.p;
    const unsigned egrid = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((a.workers + 7) / 8, c.num_sms * 8ull)));
    prof_begin(c, "hogwild_exact_kernel");
    if (a.task == 0)
      hogwild_exact_example_kernel<0><<<egrid, 256, 0, c.stream>>>(p, ds.ex_rep64.p, ds.ex_claim.p,
                                                                   ds.ex_ready.p, ds.ex_epoch);
    else
      hogwild_exact_example_kernel<1><<<egrid, 256, 0, c.stream>>>(p, ds.ex_rep64.p, ds.ex_claim.p,
                                                                   ds.ex_ready.p, ds.ex_epoch);
    launched(c, "hogwild_exact_kernel");
    refresh_w32(m);
    return;
  }
  if (a.replication == SGDB_REPL_KERNEL) {
    p.model = m.w64.p;
    p.gs = a.workers;  // one "group": w / gs == 0
    p.ld = 0;
  } else {
    p.gs = a.replication == SGDB_REPL_BLOCK ? a.group_size : 1;
    R = (a.workers + p.gs - 1) / p.gs;
    p.ld = ds.d + 1;
    const uint64_t bytes = R * p.ld * sizeof(double);
    if (bytes > (64ull << 30))
      throw sgdb::CapacityError("exact-mode replicas need " + std::to_string(bytes) + " bytes");
    ds.ex_reps.alloc(R * p.ld);
    replicas_fill_kernel<<<grid_1d(c, R * p.ld), 256, 0, c.stream>>>(ds.ex_reps.p, R, ds.d,
                                                                     m.w64.p);
    launched(c, "replicas_fill_kernel");
    p.model = ds.ex_reps.p;
  }
  const uint64_t warps = a.workers;
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, c.num_sms * 8ull)));
  prof_begin(c, "hogwild_exact_kernel");
  if (a.task == 0) {
    if (dense) hogwild_exact_kernel<0, true><<<grid, 256, 0, c.stream>>>(p);
    else hogwild_exact_kernel<0, false><<<grid, 256, 0, c.stream>>>(p);
  } else {
    if (dense) hogwild_exact_kernel<1, true><<<grid, 256, 0, c.stream>>>(p);
    else hogwild_exact_kernel<1, false><<<grid, 256, 0, c.stream>>>(p);
  }
  launched(c, "hogwild_exact_kernel");
  if (R) {
    replicas_merge_kernel<<<grid_1d(c, ds.d), 256, 0, c.stream>>>(ds.ex_reps.p, R, ds.d, m.w64.p);
    launched(c, "replicas_merge_kernel");
  }
  refresh_w32(m);
}

}  // namespace sgdb::dev

// ---- the operator API's C-ABI ----------------------------------------------

extern "C" {

sgdb_status sgdb_matvec(sgdb_ctx* ctx, sgdb_dataset* ds, const uint32_t* rows, uint64_t n_rows,
                        const double* v, uint64_t v_len, double* out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    require(ctx && ds, "null argument");
    require(v_len == ds->d, "matvec: dimension mismatch");
    Ctx& c = *ctx;
    const uint64_t nr = n_rows ? n_rows : ds->n_global;
    DBuf<uint32_t> drows;
    DBuf<double> dv, dout;
    if (n_rows) h2d_vec(drows, rows, n_rows, c.stream);
    h2d_vec(dv, v, ds->d, c.stream);
    dout.alloc(std::max<uint64_t>(1, nr));
    lin_matvec(*ds, n_rows ? drows.p : nullptr, nr, dv.p, dout.p);
    d2h_sync(out, dout.p, nr, c.stream);
  });
}

sgdb_status sgdb_matvec_transposed(sgdb_ctx* ctx, sgdb_dataset* ds, const uint32_t* rows,
                                   uint64_t n_rows, const double* a, uint64_t a_len, double* out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    require(ctx && ds, "null argument");
    const uint64_t nr = n_rows ? n_rows : ds->n_global;
    require(a_len == nr, "matvec_transposed: dimension mismatch");
    Ctx& c = *ctx;
    DBuf<uint32_t> drows;
    DBuf<double> da, dout;
    if (n_rows) h2d_vec(drows, rows, n_rows, c.stream);
    h2d_vec(da, a, nr, c.stream);
    dout.alloc(std::max<uint64_t>(1, ds->d));
    lin_matvec_t(*ds, n_rows ? drows.p : nullptr, nr, da.p, false, dout.p);
    d2h_sync(out, dout.p, ds->d, c.stream);
  });
}

sgdb_status sgdb_elementwise(sgdb_ctx* ctx, int32_t op, const double* a, const double* b,
                             uint64_t n, double scalar, double* out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    require(ctx != nullptr, "null argument");
    require(op >= SGDB_EW_MUL && op <= SGDB_EW_HINGE_INDICATOR, "unknown elementwise op");
    const bool binary = op == SGDB_EW_MUL || op == SGDB_EW_DIV;
    require(!binary || b != nullptr || n == 0, "binary elementwise op needs b");
    if (op == SGDB_EW_DIV)
      for (uint64_t i = 0; i < n; ++i)
        if (b[i] == 0.0)
          throw std::domain_error("ew_div: division by zero at position " + std::to_string(i));
    Ctx& c = *ctx;
    DBuf<double> da, db, dout;
    h2d_vec(da, a, n, c.stream);
    if (binary) h2d_vec(db, b, n, c.stream);
    dout.alloc(std::max<uint64_t>(1, n));
    prof_begin(c, "elementwise_kernel");
    elementwise_kernel<<<grid_1d(c, n), 256, 0, c.stream>>>(op, da.p, binary ? db.p : nullptr, scalar,
                                                            n, dout.p);
    launched(c, "elementwise_kernel");
    d2h_sync(out, dout.p, n, c.stream);
  });
}

sgdb_status sgdb_axpy(sgdb_ctx* ctx, double* w, double alpha, const double* g, uint64_t n) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    require(ctx != nullptr, "null argument");
    Ctx& c = *ctx;
    DBuf<double> dw, dg;
    h2d_vec(dw, w, n, c.stream);
    h2d_vec(dg, g, n, c.stream);
    prof_begin(c, "axpy_kernel");
    axpy_kernel<<<grid_1d(c, n), 256, 0, c.stream>>>(dw.p, alpha, dg.p, n, nullptr);
    launched(c, "axpy_kernel");
    d2h_sync(w, dw.p, n, c.stream);
  });
}

}  // extern "C"
