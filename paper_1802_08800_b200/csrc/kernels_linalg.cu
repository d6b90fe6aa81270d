// The §4 linear-algebra operator API on the device (proj/include/sgdbench/
// linalg.hpp:23-58, proj/src/linalg.cpp:26-181): the primitives the paper's
// GPU sync SGD chains (§4, Eq. 2). The training path uses the fused
// kernels of kernels_sync.cu; these are the stand-alone operators, for callers
// of the reference's linalg:: API. Arithmetic is fp64 on the fp32-stored
// matrix (the reference's precision), with the reference's summation order
// where it is a per-output sequential loop:
//   matvec               one writer per row, ascending slots   (linalg.cpp:30-44)
//   matvec_transposed    dense: one writer per column, ascending positions
//                        (linalg.cpp:58-76); CSR: fp64 atomics (order effects
//                        ~1e-16 instead of the 256-row partial tree)
//   ew_* / axpy          elementwise                           (linalg.cpp:113-181)
#include <cuda_runtime.h>

#include <cmath>
#include <memory>
#include <vector>

#include "device.hpp"

namespace sgdb::dev {
namespace {

__global__ void matvec_dense_kernel(const float* __restrict__ x, uint64_t n_local, uint64_t row_base,
                                    uint32_t d, const uint32_t* __restrict__ rows, uint64_t nr,
                                    const double* __restrict__ v, double* __restrict__ out) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nr;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = (rows ? rows[p] : p) - row_base;
    double z = 0.0;
    if (r < n_local)
      for (uint32_t j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(static_cast<double>(x[r * d + j]), v[j]));
    out[p] = z;
  }
}

__global__ void matvec_csr_kernel(const float* __restrict__ val, const uint32_t* __restrict__ idx,
                                  const uint32_t* __restrict__ rowptr, uint64_t n_local,
                                  uint64_t row_base, const uint32_t* __restrict__ rows, uint64_t nr,
                                  const double* __restrict__ v, double* __restrict__ out) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nr;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = (rows ? rows[p] : p) - row_base;
    double z = 0.0;
    if (r < n_local)
      for (uint32_t s = rowptr[r]; s < rowptr[r + 1]; ++s)
        z = __dadd_rn(z, __dmul_rn(static_cast<double>(val[s]), v[idx[s]]));
    out[p] = z;
  }
}

// Dense X^T a: thread j walks the positions in order (the reference's
// DenseColMajor branch), reading column j of the row-major store.
__global__ void matvec_t_dense_kernel(const float* __restrict__ x, uint64_t n_local,
                                      uint64_t row_base, uint32_t d, const uint32_t* __restrict__ rows,
                                      uint64_t nr, const double* __restrict__ a,
                                      double* __restrict__ out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint64_t p = 0; p < nr; ++p) {
      const uint64_t r = (rows ? rows[p] : p) - row_base;
      if (r < n_local) s = __dadd_rn(s, __dmul_rn(a[p], static_cast<double>(x[r * d + j])));
    }
    out[j] = s;
  }
}

// Row-major / CSR X^T a in the reference's order (linalg.cpp:78-109): a
// partial per kReduceBlock positions (ascending p within the block), then a
// fixed pairwise tree over blocks. The tree equals a binary counter: pushing
// block k merges it with the stacked complete subtrees for the trailing one
// bits of k (left += right), and the final collapse adds the remaining
// subtrees right to left. The per-coordinate stack (one value per bit level)
// lives in global memory so the blocks can be streamed in bounded chunks.
constexpr uint32_t kReduceBlock = 256;  // linalg.hpp:18

// Phase 1, dense: thread (block-in-chunk, j) sums its block sequentially.
__global__ void partials_dense_kernel(const float* __restrict__ x, uint64_t n_local,
                                      uint64_t row_base, uint32_t d,
                                      const uint32_t* __restrict__ rows, uint64_t nr,
                                      uint64_t blk0, const double* __restrict__ a,
                                      double* __restrict__ part) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const uint64_t blk = blk0 + blockIdx.y;
  const uint64_t lo = blk * kReduceBlock, hi = min(nr, lo + kReduceBlock);
  double s = 0.0;
  for (uint64_t p = lo; p < hi; ++p) {
    const uint64_t r = (rows ? rows[p] : p) - row_base;
    if (r < n_local) s = __dadd_rn(s, __dmul_rn(a[p], static_cast<double>(x[r * d + j])));
  }
  part[(uint64_t)blockIdx.y * d + j] = s;
}

// Phase 1, CSR: one warp per block walks its rows in order; the slots of a row
// have distinct columns, so lanes split them and __syncwarp orders rows.
__global__ void partials_csr_kernel(const float* __restrict__ val, const uint32_t* __restrict__ idx,
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
        dst[j] = __dadd_rn(dst[j], __dmul_rn(ap, static_cast<double>(val[s])));
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

// ElementwiseOp (linalg.hpp:40) + the fused sigmoid / hinge indicator.
__global__ void elementwise_kernel(int op, const double* __restrict__ a, const double* __restrict__ b,
                                   double scalar, uint64_t n, double* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double x = a[i];
    double r;
    switch (op) {
      case SGDB_EW_MUL: r = x * b[i]; break;
      case SGDB_EW_DIV: r = x / b[i]; break;
      case SGDB_EW_EXP: r = exp(x); break;
      case SGDB_EW_NEG: r = -x; break;
      case SGDB_EW_ADD_SCALAR: r = scalar + x; break;
      case SGDB_EW_SIGMOID:  // stable split (math.hpp:10-16); exp within 1 ulp of libm
        if (x <= 0.0) {
          const double e = exp(x);
          r = e / __dadd_rn(1.0, e);
        } else {
          r = 1.0 / __dadd_rn(1.0, exp(-x));
        }
        break;
      default: r = x < 1.0 ? 1.0 : 0.0; break;  // SGDB_EW_HINGE_INDICATOR
    }
    out[i] = r;
  }
}

__global__ void axpy_kernel(double* w, double alpha, const double* __restrict__ g, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    w[i] = __dsub_rn(w[i], __dmul_rn(alpha, g[i]));  // no FMA: the reference rounds twice
}

unsigned grid_1d(const Ctx& c, uint64_t n) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, c.num_sms * 16ull)));
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

}  // namespace
}  // namespace sgdb::dev

extern "C" {

sgdb_status sgdb_matvec(sgdb_ctx* ctx, sgdb_dataset* ds, const uint32_t* rows, uint64_t n_rows,
                        const double* v, uint64_t v_len, double* out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    require(v_len == ds->d, "matvec: dimension mismatch");
    Ctx& c = *ctx;
    const uint64_t nr = n_rows ? n_rows : ds->n_global;
    DBuf<uint32_t> drows;
    DBuf<double> dv, dout;
    if (n_rows) h2d_vec(drows, rows, n_rows, c.stream);
    h2d_vec(dv, v, ds->d, c.stream);
    dout.alloc(std::max<uint64_t>(1, nr));
    const unsigned grid = grid_1d(c, nr);
    prof_begin(c, "matvec_kernel");
    if (ds->kind == Kind::Dense)
      matvec_dense_kernel<<<grid, 256, 0, c.stream>>>(ds->x.p, ds->n, ds->row_base,
                                                      static_cast<uint32_t>(ds->d),
                                                      n_rows ? drows.p : nullptr, nr, dv.p, dout.p);
    else
      matvec_csr_kernel<<<grid, 256, 0, c.stream>>>(ds->val.p, ds->idx.p, ds->rowptr.p, ds->n,
                                                    ds->row_base, n_rows ? drows.p : nullptr, nr,
                                                    dv.p, dout.p);
    launched(c, "matvec_kernel");
    d2h_sync(out, dout.p, nr, c.stream);
  });
}

sgdb_status sgdb_matvec_transposed(sgdb_ctx* ctx, sgdb_dataset* ds, const uint32_t* rows,
                                   uint64_t n_rows, const double* a, uint64_t a_len, double* out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    const uint64_t nr = n_rows ? n_rows : ds->n_global;
    require(a_len == nr, "matvec_transposed: dimension mismatch");
    Ctx& c = *ctx;
    const uint32_t d = static_cast<uint32_t>(ds->d);
    DBuf<uint32_t> drows;
    DBuf<double> da, dout;
    if (n_rows) h2d_vec(drows, rows, n_rows, c.stream);
    h2d_vec(da, a, nr, c.stream);
    dout.alloc(std::max<uint64_t>(1, d));
    dout.zero(c.stream);
    const uint32_t* rp = n_rows ? drows.p : nullptr;
    const unsigned gd = (d + 255) / 256;
    if (nr == 0 || d == 0) {
      // zeros (linalg.cpp:56)
    } else if (ds->layout_in == SGDB_LAYOUT_DENSE_COL) {
      prof_begin(c, "matvec_t_kernel");
      matvec_t_dense_kernel<<<grid_1d(c, d), 256, 0, c.stream>>>(ds->x.p, ds->n, ds->row_base, d,
                                                                 rp, nr, da.p, dout.p);
      launched(c, "matvec_t_kernel");
    } else {
      const uint64_t nblocks = (nr + kReduceBlock - 1) / kReduceBlock;
      // Partials of at most ~256 MiB per chunk (and <= 65535 grid rows).
      const uint64_t chunk = std::max<uint64_t>(
          1, std::min<uint64_t>({nblocks, (256ull << 20) / (8ull * d), 65535}));
      DBuf<double> part, stack;
      part.alloc(chunk * d);
      stack.alloc(64ull * d);
      for (uint64_t b0 = 0; b0 < nblocks; b0 += chunk) {
        const uint32_t nb = static_cast<uint32_t>(std::min(chunk, nblocks - b0));
        if (ds->kind == Kind::Dense) {
          prof_begin(c, "matvec_t_partials");
          partials_dense_kernel<<<dim3(gd, nb), 256, 0, c.stream>>>(ds->x.p, ds->n, ds->row_base, d,
                                                                    rp, nr, b0, da.p, part.p);
        } else {
          check(cudaMemsetAsync(part.p, 0, uint64_t(nb) * d * sizeof(double), c.stream), "memset");
          prof_begin(c, "matvec_t_partials");
          partials_csr_kernel<<<nb, 32, 0, c.stream>>>(ds->val.p, ds->idx.p, ds->rowptr.p, ds->n,
                                                       ds->row_base, d, rp, nr, b0, da.p, part.p);
        }
        launched(c, "matvec_t_partials");
        prof_begin(c, "matvec_t_tree");
        tree_push_kernel<<<gd, 256, 0, c.stream>>>(part.p, nb, d, b0, stack.p);
        launched(c, "matvec_t_tree");
      }
      prof_begin(c, "matvec_t_tree");
      tree_collapse_kernel<<<gd, 256, 0, c.stream>>>(stack.p, d, nblocks, dout.p);
      launched(c, "matvec_t_tree");
    }
    d2h_sync(out, dout.p, d, c.stream);
  });
}

sgdb_status sgdb_elementwise(sgdb_ctx* ctx, int32_t op, const double* a, const double* b,
                             uint64_t n, double scalar, double* out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
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
    Ctx& c = *ctx;
    DBuf<double> dw, dg;
    h2d_vec(dw, w, n, c.stream);
    h2d_vec(dg, g, n, c.stream);
    prof_begin(c, "axpy_kernel");
    axpy_kernel<<<grid_1d(c, n), 256, 0, c.stream>>>(dw.p, alpha, dg.p, n);
    launched(c, "axpy_kernel");
    d2h_sync(w, dw.p, n, c.stream);
  });
}

}  // extern "C"
