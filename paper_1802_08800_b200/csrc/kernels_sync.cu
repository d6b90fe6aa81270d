// Synchronous mini-batch SGD kernels (sm_100a).
//
// Replaces the reference's §4 primitive chain for one mini-batch
// (proj/src/sync_engine.cpp:22-42): matvec (linalg.cpp:30-44) -> elementwise
// LR/SVM derivative (linalg.cpp:124-174) -> matvec_transposed
// (linalg.cpp:50-109) -> axpy (linalg.cpp:176-181) + the finite scan
// (sync_engine.cpp:97-98), fused so each batch is one (dense) or two
// (sparse full batch) HBM sweeps. See DESIGN.md §Kernels for the rooflines.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "device.hpp"

namespace sgdb::dev {

namespace {

// ---------------------------------------------------------------------------
// Shared tail: fixed-order fp64 reduction of per-block gradient partials by
// the last block to finish, then the fused update.
// ---------------------------------------------------------------------------
struct GradTail {
  double* partials;  // [gridDim.x][d]
  unsigned* ticket;
  int d;
  double alpha;
  int apply;
  int want_norm;
  double* w64;
  float* w32;
  double* g64;
  int* finite;
  double* norm2;
};

__device__ __forceinline__ double block_sum_d(double v, double* sh) {
  v = warp_sum_d(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  return t;  // valid in thread 0
}

// Called by every thread of every block after its partial is in
// partials[blockIdx.x]. Returns after the last block applied the tail.
__device__ void grad_tail(const GradTail& t) {
  __shared__ unsigned s_last;
  __shared__ double s_red[32];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(t.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double nrm = 0.0;
  int bad = 0;
  for (int j = threadIdx.x; j < t.d; j += blockDim.x) {
    double g = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) g += __ldcg(&t.partials[(size_t)b * t.d + j]);
    if (!isfinite(g)) bad = 1;
    if (t.apply) {
      double w = t.w64[j] - t.alpha * g;
      t.w64[j] = w;
      t.w32[j] = static_cast<float>(w);
    } else {
      t.g64[j] = g;
    }
    nrm += g * g;
  }
  if (bad) *t.finite = 0;
  if (t.want_norm) {
    double s = block_sum_d(nrm, s_red);
    if (threadIdx.x == 0) *t.norm2 += s;
  }
  if (threadIdx.x == 0) *t.ticket = 0u;
}

// ---------------------------------------------------------------------------
// K1: dense row-major, all local rows (full batch). Persistent CTAs, one per
// SM; warp 0 lane 0 streams contiguous row tiles (rows x d floats + labels)
// into a shared-memory ring with cp.async.bulk (1-D TMA) on mbarriers; WC
// consumer warps map L lanes to a row (F features per lane, feature
// q + L*k), keep the model slice and the gradient accumulators in
// registers, so each nonzero is read from HBM exactly once.
// ---------------------------------------------------------------------------
struct DenseFullParams {
  const float* x;
  const float* y;
  uint64_t n;
  int d;
  int R;          // rows per tile (multiple of 4)
  int S;          // pipeline stages
  uint64_t ntiles;
  uint32_t x_floats;      // R*d
  uint32_t stage_floats;  // x_floats + R, rounded to 32
  const float* w32;
  GradTail tail;
};

template <int L, int F, int TASK, int WC>
__global__ void __launch_bounds__(32 * (WC + 1), 1) dense_full_kernel(DenseFullParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + p.S;
  float* stages = reinterpret_cast<float*>(smem + 128 * ((16 * p.S + 127) / 128));
  float* red = stages + (size_t)p.S * p.stage_floats;  // [WC][d]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = p.d;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WC);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      uint64_t i = 0;
      for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++i) {
        const int s = static_cast<int>(i % p.S);
        if (i >= (uint64_t)p.S) mbar_wait(&empty[s], static_cast<uint32_t>(((i / p.S) - 1) & 1));
        const uint64_t r0 = t * p.R;
        const uint64_t rows = min(static_cast<uint64_t>(p.R), p.n - r0);
        const uint32_t xb = round_up16(rows * d * 4ull), yb = round_up16(rows * 4ull);
        float* st = stages + (size_t)s * p.stage_floats;
        mbar_arrive_expect_tx(&full[s], xb + yb);
        bulk_g2s(st, p.x + r0 * d, xb, &full[s]);
        bulk_g2s(st + p.x_floats, p.y + r0, yb, &full[s]);
      }
    }
  } else {
    constexpr int RS = 32 / L;
    const int cw = warp - 1, q = lane % L, slot = lane / L;
    float wr[F], acc[F];
#pragma unroll
    for (int k = 0; k < F; ++k) {
      const int j = q + L * k;
      wr[k] = j < d ? p.w32[j] : 0.f;
      acc[k] = 0.f;
    }
    uint64_t i = 0;
    for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++i) {
      const int s = static_cast<int>(i % p.S);
      mbar_wait(&full[s], static_cast<uint32_t>((i / p.S) & 1));
      const float* xs = stages + (size_t)s * p.stage_floats;
      const float* ys = xs + p.x_floats;
      const int rows = static_cast<int>(min(static_cast<uint64_t>(p.R), p.n - t * p.R));
      for (int rb = cw * RS; rb < rows; rb += WC * RS) {
        const int r = rb + slot;
        const bool valid = r < rows;
        float xv[F];
        float z = 0.f;
#pragma unroll
        for (int k = 0; k < F; ++k) {
          const int j = q + L * k;
          xv[k] = (valid && j < d) ? xs[r * d + j] : 0.f;
          z = fmaf(xv[k], wr[k], z);
        }
        z = group_sum<L>(z);
        const float c = valid ? coef_f<TASK>(z, ys[r]) : 0.f;
#pragma unroll
        for (int k = 0; k < F; ++k) acc[k] = fmaf(c, xv[k], acc[k]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int k = 0; k < F; ++k) acc[k] = cross_group_sum<L>(acc[k]);
    if (slot == 0) {
#pragma unroll
      for (int k = 0; k < F; ++k) {
        const int j = q + L * k;
        if (j < d) red[cw * d + j] = acc[k];
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < WC; ++w) s += red[w * d + j];
    p.tail.partials[(size_t)blockIdx.x * d + j] = s;
  }
  grad_tail(p.tail);
}

// ---------------------------------------------------------------------------
// K1b: dense row-major, rows gathered from a list of global ids (mini-batch).
// Block partials are folded into g64 with fp64 atomics; the last block
// applies the update and re-zeroes g64.
// ---------------------------------------------------------------------------
struct DenseBatchParams {
  const float* x;
  const float* y;
  uint64_t n_local, row_base;
  int d;
  const uint32_t* ids;
  uint64_t nb;
  const float* w32;
  double* g64;
  unsigned* ticket;
  int* finite;
  double* w64;
  float* w32_out;
  double* norm2;
  double alpha;
  int apply;
  int want_norm;
  const double* alpha_dev;
};

template <int L, int F, int TASK, int W>
__global__ void __launch_bounds__(32 * W) dense_batch_kernel(DenseBatchParams p) {
  extern __shared__ __align__(16) float red[];  // [W][d]
  __shared__ unsigned s_last;
  __shared__ double s_red[32];
  if (p.apply && *p.finite == 0) return;  // the epoch already stopped
  constexpr int RS = 32 / L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane % L, slot = lane / L, d = p.d;
  const uint64_t gw = (uint64_t)blockIdx.x * W + warp, tw = (uint64_t)gridDim.x * W;
  float wr[F], acc[F];
#pragma unroll
  for (int k = 0; k < F; ++k) {
    const int j = q + L * k;
    wr[k] = j < d ? p.w32[j] : 0.f;
    acc[k] = 0.f;
  }
  for (uint64_t pb = gw * RS; pb < p.nb; pb += tw * RS) {
    const uint64_t pos = pb + slot;
    uint64_t row = 0;
    bool valid = pos < p.nb;
    if (valid) {
      row = static_cast<uint64_t>(p.ids[pos]) - p.row_base;
      valid = row < p.n_local;
    }
    const float* xr = p.x + row * d;
    float xv[F];
    float z = 0.f;
#pragma unroll
    for (int k = 0; k < F; ++k) {
      const int j = q + L * k;
      xv[k] = (valid && j < d) ? __ldg(xr + j) : 0.f;
      z = fmaf(xv[k], wr[k], z);
    }
    z = group_sum<L>(z);
    const float c = valid ? coef_f<TASK>(z, __ldg(p.y + row)) : 0.f;
#pragma unroll
    for (int k = 0; k < F; ++k) acc[k] = fmaf(c, xv[k], acc[k]);
  }
#pragma unroll
  for (int k = 0; k < F; ++k) acc[k] = cross_group_sum<L>(acc[k]);
  if (slot == 0) {
#pragma unroll
    for (int k = 0; k < F; ++k) {
      const int j = q + L * k;
      if (j < d) red[warp * d + j] = acc[k];
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < W; ++w) s += red[w * d + j];
    if (s != 0.0) atomicAdd(&p.g64[j], s);
  }
  if (!p.apply) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(p.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double alpha = p.alpha_dev ? *p.alpha_dev : p.alpha;
  double nrm = 0.0;
  int bad = 0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const double g = __ldcg(&p.g64[j]);
    if (!isfinite(g)) bad = 1;
    const double w = p.w64[j] - alpha * g;
    p.w64[j] = w;
    p.w32_out[j] = static_cast<float>(w);
    p.g64[j] = 0.0;
    nrm += g * g;
  }
  if (bad) *p.finite = 0;
  if (p.want_norm) {
    double s = block_sum_d(nrm, s_red);
    if (threadIdx.x == 0) *p.norm2 += s;
  }
  if (threadIdx.x == 0) *p.ticket = 0u;
}

// Barrier across a co-resident grid (cooperative launch). `count` only grows:
// barrier k of the launch completes when it reaches k * gridDim.x, so an
// arrival is one atomic and the wait one acquire-load poll (no reset, no
// generation word). Thread 0 fences the block's global writes (the gradient
// REDs, ordered before it by the __syncthreads) before arriving.
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(count, 1u);
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
      if (v >= target) break;
      __nanosleep(20);
    }
  }
  __syncthreads();
}

// K1c: a whole dense mini-batch epoch in one persistent launch. Step s takes
// ids order[s*B, s*B+nb): warps compute margins, coefficients and CTA partial
// gradients as in K1b and fold them into g3[s % 3] with fp64 REDs; one grid
// barrier; then EVERY CTA applies the identical fp64 step to its own shared
// copy of the master model (so no second barrier), and CTA 0 clears the
// buffer of step s+2. The next step's first rows do not depend on the model,
// so they are loaded before the barrier. Non-finite gradients stop every CTA
// at the same step, after its update (sync_engine.cpp:94-97).
struct DenseEpochParams {
  const float* x;
  const float* y;
  uint64_t n_local, row_base;
  int d;
  const uint32_t* order;
  uint64_t n_ids, B;
  double* g3;     // 3*d, zero on entry
  unsigned* bar;  // arrivals (monotonic within the launch, zero on entry)
  int* finite;
  double* w64;
  float* w32;
  double alpha;
};

template <int L, int F, int TASK, int W>
__global__ void __launch_bounds__(32 * W) dense_epoch_kernel(DenseEpochParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* w64s = reinterpret_cast<double*>(smem_raw);  // [d] master copy
  float* red = reinterpret_cast<float*>(w64s + p.d);    // [W][d]
  constexpr int RS = 32 / L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane % L, slot = lane / L, d = p.d;
  const uint64_t gw = (uint64_t)blockIdx.x * W + warp, tw = (uint64_t)gridDim.x * W;
  for (int j = threadIdx.x; j < d; j += blockDim.x) w64s[j] = p.w64[j];
  __syncthreads();
  float wr[F];
#pragma unroll
  for (int k = 0; k < F; ++k) {
    const int j = q + L * k;
    wr[k] = j < d ? static_cast<float>(w64s[j]) : 0.f;
  }
  auto load_row = [&](uint64_t lo, uint64_t nb, uint64_t pb, float(&xv)[F], float& yv,
                      bool& valid) {
    const uint64_t pos = pb + slot;
    valid = pos < nb;
    uint64_t row = 0;
    if (valid) {
      row = static_cast<uint64_t>(p.order[lo + pos]) - p.row_base;
      valid = row < p.n_local;
    }
    const float* xr = p.x + row * d;
#pragma unroll
    for (int k = 0; k < F; ++k) {
      const int j = q + L * k;
      xv[k] = (valid && j < d) ? __ldg(xr + j) : 0.f;
    }
    yv = valid ? __ldg(p.y + row) : 0.f;
  };
  const uint64_t nsteps = (p.n_ids + p.B - 1) / p.B;
  float xn[F], yn;
  bool vn;
  load_row(0, min(p.B, p.n_ids), gw * RS, xn, yn, vn);
  for (uint64_t s = 0; s < nsteps; ++s) {
    const uint64_t lo = s * p.B, nb = min(p.B, p.n_ids - lo);
    double* g = p.g3 + (s % 3) * static_cast<uint64_t>(d);
    float acc[F];
    {
      float z = 0.f;
#pragma unroll
      for (int k = 0; k < F; ++k) z = fmaf(xn[k], wr[k], z);
      z = group_sum<L>(z);
      const float c = vn ? coef_f<TASK>(z, yn) : 0.f;
#pragma unroll
      for (int k = 0; k < F; ++k) acc[k] = c * xn[k];
    }
    for (uint64_t pb = (gw + tw) * RS; pb < nb; pb += tw * RS) {
      float xv[F], yv;
      bool v;
      load_row(lo, nb, pb, xv, yv, v);
      float z = 0.f;
#pragma unroll
      for (int k = 0; k < F; ++k) z = fmaf(xv[k], wr[k], z);
      z = group_sum<L>(z);
      const float c = v ? coef_f<TASK>(z, yv) : 0.f;
#pragma unroll
      for (int k = 0; k < F; ++k) acc[k] = fmaf(c, xv[k], acc[k]);
    }
    if (s + 1 < nsteps) load_row(lo + p.B, min(p.B, p.n_ids - lo - p.B), gw * RS, xn, yn, vn);
#pragma unroll
    for (int k = 0; k < F; ++k) acc[k] = cross_group_sum<L>(acc[k]);
    if (slot == 0) {
#pragma unroll
      for (int k = 0; k < F; ++k) {
        const int j = q + L * k;
        if (j < d) red[warp * d + j] = acc[k];
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < W; ++w) sum += red[w * d + j];
      if (sum != 0.0) atomicAdd(&g[j], sum);
    }
    grid_sync(p.bar, static_cast<unsigned>(s + 1) * gridDim.x);
    int bad = 0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      const double gj = __ldcg(&g[j]);
      if (!isfinite(gj)) bad = 1;
      w64s[j] = w64s[j] - p.alpha * gj;
    }
    if (blockIdx.x == 0) {
      double* g2 = p.g3 + ((s + 2) % 3) * static_cast<uint64_t>(d);
      for (int j = threadIdx.x; j < d; j += blockDim.x) g2[j] = 0.0;
    }
    bad = __syncthreads_or(bad);
#pragma unroll
    for (int k = 0; k < F; ++k) {
      const int j = q + L * k;
      wr[k] = j < d ? static_cast<float>(w64s[j]) : 0.f;
    }
    if (bad) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *p.finite = 0;
      break;
    }
  }
  if (blockIdx.x == 0) {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      p.w64[j] = w64s[j];
      p.w32[j] = static_cast<float>(w64s[j]);
    }
  }
}

// Lane-strided sparse dot x_row . w over slots [b, e): U slots per batch so
// U index loads and then U independent model gathers are in flight at once.
template <int G, bool SMEM = false>
__device__ __forceinline__ float gather_dot(const float* __restrict__ val,
                                            const uint32_t* __restrict__ idx, uint32_t b,
                                            uint32_t e, int lg, const float* __restrict__ w) {
  constexpr int U = 4;
  float z = 0.f;
  for (uint32_t s0 = b + lg; s0 < e; s0 += G * U) {
    uint32_t jv[U];
    float xv[U], wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t s = s0 + u * G;
      jv[u] = s < e ? __ldg(idx + s) : 0u;
      xv[u] = s < e ? __ldg(val + s) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) wv[u] = s0 + u * G < e ? (SMEM ? w[jv[u]] : __ldg(w + jv[u])) : 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) z = fmaf(xv[u], wv[u], z);
  }
  return z;
}

// ---------------------------------------------------------------------------
// K2: sparse margins + coefficients for all local rows. G lanes per row,
// coalesced val/idx, model gathered from L2 (d <= 1.4M floats stays resident).
// ---------------------------------------------------------------------------
template <int G, int TASK>
__global__ void __launch_bounds__(256) csr_coef_kernel(const float* __restrict__ val,
                                                       const uint32_t* __restrict__ idx,
                                                       const uint32_t* __restrict__ rowptr,
                                                       const float* __restrict__ y, uint64_t n,
                                                       const float* __restrict__ w32,
                                                       float* __restrict__ coef) {
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = gw * RW; base < n; base += tw * RW) {
    const uint64_t row = base + grp;
    float z = 0.f;
    if (row < n) z = gather_dot<G>(val, idx, rowptr[row], rowptr[row + 1], lg, w32);
    z = group_sum<G>(z);
    if (row < n && lg == 0) coef[row] = coef_f<TASK>(z, y[row]);
  }
}

// ---------------------------------------------------------------------------
// K2p: K2 with a 2-stage software pipeline across the rows a warp walks:
// while row i reduces, the extent (and label) of row i+2 and the first slot
// batch of row i+1 are in flight, so a warp is never idle on a dependent
// rowptr -> idx -> gather chain. SMEM = stage the fp32 model in shared memory
// (d <= 48K floats) and gather from it.
// ---------------------------------------------------------------------------
struct SegBatch {
  uint32_t j[4];
  float x[4];
};

template <int G>
__device__ __forceinline__ SegBatch seg_batch(const float* __restrict__ val,
                                              const uint32_t* __restrict__ idx, uint32_t s0,
                                              uint32_t e) {
  SegBatch bt;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t s = s0 + u * G;
    bt.j[u] = s < e ? __ldg(idx + s) : 0u;
    bt.x[u] = s < e ? __ldg(val + s) : 0.f;
  }
  return bt;
}

template <int G, bool SMEM>
__device__ __forceinline__ float seg_dot(const float* __restrict__ val,
                                         const uint32_t* __restrict__ idx, uint32_t b, uint32_t e,
                                         int lg, const SegBatch& first, const float* __restrict__ w) {
  float z = 0.f;
  {
    float wv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) wv[u] = b + lg + u * G < e ? (SMEM ? w[first.j[u]] : __ldg(w + first.j[u])) : 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) z = fmaf(first.x[u], wv[u], z);
  }
  for (uint32_t s0 = b + lg + G * 4; s0 < e; s0 += G * 4) {
    const SegBatch bt = seg_batch<G>(val, idx, s0, e);
    float wv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) wv[u] = s0 + u * G < e ? (SMEM ? w[bt.j[u]] : __ldg(w + bt.j[u])) : 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) z = fmaf(bt.x[u], wv[u], z);
  }
  return z;
}

template <int G, int TASK, bool SMEM>
__global__ void __launch_bounds__(SMEM ? 1024 : 256) csr_coef_pipe_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const float* __restrict__ y, uint64_t n,
    const float* __restrict__ w32, uint32_t d, float* __restrict__ coef) {
  extern __shared__ float ws[];
  const float* w = w32;
  if (SMEM) {
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) ws[j] = w32[j];
    __syncthreads();
    w = ws;
  }
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t step = (((uint64_t)gridDim.x * blockDim.x) >> 5) * RW;
  uint64_t base = gw * RW;
  auto extent = [&](uint64_t bs, uint32_t& b, uint32_t& e, float& yy) {
    const uint64_t r = bs + grp;
    if (r < n) {
      b = rowptr[r];
      e = rowptr[r + 1];
      yy = y[r];
    } else {
      b = e = 0u;
      yy = 0.f;
    }
  };
  uint32_t cb, ce, nb, ne;
  float cy, ny;
  extent(base, cb, ce, cy);
  extent(base + step, nb, ne, ny);
  SegBatch cur = seg_batch<G>(val, idx, cb + lg, ce);
  for (; base < n; base += step) {
    const SegBatch nxt = seg_batch<G>(val, idx, nb + lg, ne);
    uint32_t ab, ae;
    float ay;
    extent(base + 2 * step, ab, ae, ay);
    float z = seg_dot<G, SMEM>(val, idx, cb, ce, lg, cur, w);
    z = group_sum<G>(z);
    const uint64_t row = base + grp;
    if (row < n && lg == 0) coef[row] = coef_f<TASK>(z, cy);
    cur = nxt;
    cb = nb, ce = ne, cy = ny;
    nb = ab, ne = ae, ny = ay;
  }
}

// ---------------------------------------------------------------------------
// K2v: warp-per-row margin pass with 16-byte vector loads. Lane l of the
// warp loads the aligned group 4l of the window [b & ~3, e) — a float4 of
// values and a uint4 of indices — and gathers only its in-row slots, so a
// row costs ~2 vector loads + 4 gathers per lane instead of 8 scalar loads.
// Same 2-stage row pipeline as K2p (extent two rows ahead, first vector
// group one row ahead). The CSR arrays carry 8 elements of zero slack.
// ---------------------------------------------------------------------------
struct VecGroup {
  float4 v;
  uint4 j;
};

__device__ __forceinline__ VecGroup vec_group(const float* __restrict__ val,
                                              const uint32_t* __restrict__ idx, uint32_t a) {
  return VecGroup{__ldg(reinterpret_cast<const float4*>(val + a)),
                  __ldg(reinterpret_cast<const uint4*>(idx + a))};
}

__device__ __forceinline__ float vec_dot(const VecGroup& g, uint32_t a, uint32_t b, uint32_t e,
                                         const float* __restrict__ w) {
  float z = 0.f;
  if (a >= b && a + 3 < e) {  // whole group inside the row (the common case)
    z = fmaf(g.v.x, __ldg(w + g.j.x), z);
    z = fmaf(g.v.y, __ldg(w + g.j.y), z);
    z = fmaf(g.v.z, __ldg(w + g.j.z), z);
    z = fmaf(g.v.w, __ldg(w + g.j.w), z);
  } else {
    if (a + 0 >= b && a + 0 < e) z = fmaf(g.v.x, __ldg(w + g.j.x), z);
    if (a + 1 >= b && a + 1 < e) z = fmaf(g.v.y, __ldg(w + g.j.y), z);
    if (a + 2 >= b && a + 2 < e) z = fmaf(g.v.z, __ldg(w + g.j.z), z);
    if (a + 3 >= b && a + 3 < e) z = fmaf(g.v.w, __ldg(w + g.j.w), z);
  }
  return z;
}

template <int TASK>
__global__ void __launch_bounds__(256) csr_coef_vec_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const float* __restrict__ y, uint64_t n,
    const float* __restrict__ w, float* __restrict__ coef) {
  const int lane = threadIdx.x & 31;
  const uint64_t step = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t row = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  auto extent = [&](uint64_t r, uint32_t& b, uint32_t& e, float& yy) {
    if (r < n) {
      b = rowptr[r];
      e = rowptr[r + 1];
      yy = y[r];
    } else {
      b = e = 0u;
      yy = 0.f;
    }
  };
  uint32_t cb, ce, nb, ne;
  float cy, ny;
  extent(row, cb, ce, cy);
  extent(row + step, nb, ne, ny);
  uint32_t ca = (cb & ~3u) + 4u * lane;
  VecGroup cur = vec_group(val, idx, ca < ce ? ca : 0u);
  for (; row < n; row += step) {
    const uint32_t na = (nb & ~3u) + 4u * lane;
    const VecGroup nxt = vec_group(val, idx, na < ne ? na : 0u);
    uint32_t ab, ae;
    float ay;
    extent(row + 2 * step, ab, ae, ay);
    float z = ca < ce ? vec_dot(cur, ca, cb, ce, w) : 0.f;
    for (uint32_t a = ca + 128; a < ce; a += 128) z += vec_dot(vec_group(val, idx, a), a, cb, ce, w);
    z = group_sum<32>(z);
    if (lane == 0) coef[row] = coef_f<TASK>(z, cy);
    cur = nxt;
    ca = na, cb = nb, ce = ne, cy = ny;
    nb = ab, ne = ae, ny = ay;
  }
}

// ---------------------------------------------------------------------------
// K3: g = X^T c over the row-blocked CSC. CTA (block b, column range k)
// stages c[rows of b] in SMEM, then G lanes per column reduce
// cval * c_smem[crow] in fp64 into partials[b][j]; K3f sums the partials over
// b in fixed order, so the gradient is deterministic.
// ---------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(1024) csc_block_kernel(
    const float* __restrict__ cval, const uint16_t* __restrict__ crow,
    const uint32_t* __restrict__ colptr, const float* __restrict__ coef, uint64_t n, uint32_t d,
    uint32_t rb, uint32_t nblk, uint32_t cpb, double* __restrict__ partials) {
  extern __shared__ float cs[];
  const uint32_t b = blockIdx.x / cpb, k = blockIdx.x % cpb;
  if (b >= nblk) return;
  const uint64_t r0 = static_cast<uint64_t>(b) * rb;
  const uint32_t rows = static_cast<uint32_t>(min(static_cast<uint64_t>(rb), n - r0));
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) cs[i] = coef[r0 + i];
  __syncthreads();
  const uint32_t j0 = static_cast<uint32_t>(static_cast<uint64_t>(d) * k / cpb);
  const uint32_t j1 = static_cast<uint32_t>(static_cast<uint64_t>(d) * (k + 1) / cpb);
  const uint32_t* cp = colptr + static_cast<uint64_t>(b) * (d + 1);
  constexpr int CW = 32 / G;
  constexpr int U = 4;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint32_t warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // 2-stage pipeline over the columns this warp walks (as in K2p).
  const uint32_t step = nw * CW;
  uint32_t base = j0 + warp * CW;
  auto extent = [&](uint32_t bs, uint32_t& sb, uint32_t& se) {
    const uint32_t j = bs + grp;
    if (j < j1) {
      sb = cp[j];
      se = cp[j + 1];
    } else {
      sb = se = 0u;
    }
  };
  auto batch = [&](uint32_t s0, uint32_t se, float* xv, uint32_t* rv) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t s = s0 + u * G;
      xv[u] = s < se ? __ldg(cval + s) : 0.f;
      rv[u] = s < se ? __ldg(crow + s) : 0u;
    }
  };
  uint32_t cb, ce, nb, ne;
  extent(base, cb, ce);
  extent(base + step, nb, ne);
  float cx[U];
  uint32_t cr[U];
  batch(cb + lg, ce, cx, cr);
  for (; base < j1; base += step) {
    float nx[U];
    uint32_t nr[U];
    batch(nb + lg, ne, nx, nr);
    uint32_t ab, ae;
    extent(base + 2 * step, ab, ae);
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) acc += static_cast<double>(cx[u] * cs[cr[u]]);
    for (uint32_t s0 = cb + lg + G * U; s0 < ce; s0 += G * U) {
      float xv[U];
      uint32_t rv[U];
      batch(s0, ce, xv, rv);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += static_cast<double>(xv[u] * cs[rv[u]]);
    }
    acc = group_sum<G>(acc);
    const uint32_t j = base + grp;
    if (j < j1 && lg == 0) partials[static_cast<uint64_t>(b) * d + j] = acc;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cx[u] = nx[u];
      cr[u] = nr[u];
    }
    cb = nb, ce = ne;
    nb = ab, ne = ae;
  }
}

// K3f: g_j = sum_b partials[b][j] (fixed order), fused w -= alpha*g_j (one
// writer per coordinate), finite flag, ||g||^2.
__global__ void apply_partials_kernel(uint64_t d, uint32_t nblk, const double* __restrict__ partials,
                                      double alpha, int apply, int want_norm, double* w64,
                                      float* w32, double* g64, int* finite, double* norm2) {
  double nrm = 0.0;
  int bad = 0;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    // Sum over blocks in block order; 16 loads in flight per thread (only
    // ~d threads exist, so memory parallelism has to come from each one).
    double g = 0.0;
    uint32_t b = 0;
    for (; b + 16 <= nblk; b += 16) {
      double v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = partials[static_cast<uint64_t>(b + k) * d + j];
#pragma unroll
      for (int k = 0; k < 16; ++k) g += v[k];
    }
    for (; b < nblk; ++b) g += partials[static_cast<uint64_t>(b) * d + j];
    if (!isfinite(g)) bad = 1;
    if (apply) {
      const double w = w64[j] - alpha * g;
      w64[j] = w;
      w32[j] = static_cast<float>(w);
    } else {
      g64[j] = g;
    }
    nrm += g * g;
  }
  if (bad) *finite = 0;
  if (want_norm) {
    nrm = warp_sum_d(nrm);
    if ((threadIdx.x & 31) == 0 && nrm != 0.0) atomicAdd(norm2, nrm);
  }
}

// ---------------------------------------------------------------------------
// K3b: sparse mini-batch: margin, coefficient and scatter of c*x into g64
// with fp64 atomics (red.global.add.f64) — order effects ~1e-16, invisible
// after fp32 rounding.
// ---------------------------------------------------------------------------
template <int G, int TASK>
__global__ void __launch_bounds__(256) csr_batch_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const float* __restrict__ y, uint64_t n_local,
    uint64_t row_base, const uint32_t* __restrict__ ids, uint64_t nb,
    const float* __restrict__ w32, double* g64, const int* finite, int check_finite) {
  if (check_finite && *finite == 0) return;
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = gw * RW; base < nb; base += tw * RW) {
    const uint64_t pos = base + grp;
    uint64_t row = 0;
    bool valid = pos < nb;
    if (valid) {
      row = static_cast<uint64_t>(ids[pos]) - row_base;
      valid = row < n_local;
    }
    uint32_t b = 0, e = 0;
    if (valid) {
      b = rowptr[row];
      e = rowptr[row + 1];
    }
    const float z = group_sum<G>(gather_dot<G>(val, idx, b, e, lg, w32));
    if (!valid) continue;
    const float c = coef_f<TASK>(z, y[row]);
    if (c == 0.f) continue;
    for (uint32_t s = b + lg; s < e; s += G)
      atomicAdd(&g64[__ldg(idx + s)], static_cast<double>(c * __ldg(val + s)));
  }
}

__global__ void apply_kernel(uint64_t d, double alpha_in, const double* alpha_dev, double* w64,
                             float* w32, double* g64, int* finite, double* norm2, int want_norm) {
  const double alpha = alpha_dev ? *alpha_dev : alpha_in;
  double nrm = 0.0;
  int bad = 0;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double g = g64[j];
    if (!isfinite(g)) bad = 1;
    const double w = w64[j] - alpha * g;
    w64[j] = w;
    w32[j] = static_cast<float>(w);
    g64[j] = 0.0;
    nrm += g * g;
  }
  if (bad) *finite = 0;
  if (want_norm) {
    nrm = warp_sum_d(nrm);
    if ((threadIdx.x & 31) == 0 && nrm != 0.0) atomicAdd(norm2, nrm);
  }
}

// ---------------------------------------------------------------------------
// K4: loss (untimed, fp64): per-row margin in fp64 against the fp64 master,
// per-block partials, fixed-order final sum by the last block.
// ---------------------------------------------------------------------------
struct LossTail {
  double* partials;
  unsigned* ticket;
  double* out;
};

__device__ void loss_tail(double v, const LossTail& t) {
  __shared__ double s_red[32];
  __shared__ unsigned s_last;
  double s = block_sum_d(v, s_red);
  if (threadIdx.x == 0) t.partials[blockIdx.x] = s;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(t.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) tot += __ldcg(&t.partials[b]);
    *t.out = tot;
    *t.ticket = 0u;
  }
}

template <int L, int F>
__global__ void __launch_bounds__(256) dense_loss_kernel(const float* __restrict__ x,
                                                         const float* __restrict__ y, uint64_t n,
                                                         int d, const double* __restrict__ w64,
                                                         int task, LossTail t) {
  constexpr int RS = 32 / L;
  const int lane = threadIdx.x & 31, q = lane % L, slot = lane / L;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double wr[F];
#pragma unroll
  for (int k = 0; k < F; ++k) wr[k] = (q + L * k) < d ? w64[q + L * k] : 0.0;
  double lsum = 0.0;
  for (uint64_t base = gw * RS; base < n; base += tw * RS) {
    const uint64_t row = base + slot;
    const bool valid = row < n;
    double z = 0.0;
#pragma unroll
    for (int k = 0; k < F; ++k) {
      const int j = q + L * k;
      if (valid && j < d) z += static_cast<double>(__ldg(x + row * d + j)) * wr[k];
    }
    z = group_sum<L>(z);
    if (valid && q == 0) lsum += loss_d(task, z, static_cast<double>(y[row]));
  }
  loss_tail(lsum, t);
}

template <int G>
__global__ void __launch_bounds__(256) csr_loss_kernel(const float* __restrict__ val,
                                                       const uint32_t* __restrict__ idx,
                                                       const uint32_t* __restrict__ rowptr,
                                                       const float* __restrict__ y, uint64_t n,
                                                       const double* __restrict__ w64, int task,
                                                       LossTail t) {
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double lsum = 0.0;
  for (uint64_t base = gw * RW; base < n; base += tw * RW) {
    const uint64_t row = base + grp;
    double z = 0.0;
    if (row < n) {
      const uint32_t b = rowptr[row], e = rowptr[row + 1];
      constexpr int U = 4;
      for (uint32_t s0 = b + lg; s0 < e; s0 += G * U) {
        uint32_t jv[U];
        float xv[U];
        double wv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t s = s0 + u * G;
          jv[u] = s < e ? __ldg(idx + s) : 0u;
          xv[u] = s < e ? __ldg(val + s) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) wv[u] = s0 + u * G < e ? __ldg(w64 + jv[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) z += static_cast<double>(xv[u]) * wv[u];
      }
    }
    z = group_sum<G>(z);
    if (row < n && lg == 0) lsum += loss_d(task, z, static_cast<double>(y[row]));
  }
  loss_tail(lsum, t);
}

__global__ void w64_from_w32_kernel(uint64_t d, const float* w32, double* w64) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x)
    w64[j] = static_cast<double>(w32[j]);
}

// ---- host-side dispatch -----------------------------------------------------

int lanes_for(double avg) {
  if (avg <= 6.0) return 4;
  if (avg <= 16.0) return 8;
  if (avg <= 40.0) return 16;
  return 32;
}

int env_lanes(const char* name, int fallback) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : fallback;
}

unsigned grid_for(const Ctx& c, uint64_t items_per_block_unit, uint64_t units, unsigned per_sm) {
  uint64_t want = (units + items_per_block_unit - 1) / items_per_block_unit;
  uint64_t cap = static_cast<uint64_t>(c.num_sms) * per_sm;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
}

template <int L, int F, int TASK>
void launch_dense_full_LF(Dataset& ds, Model& m, const StepArgs& a) {
  Ctx& c = *ds.ctx;
  // Consumer warps scale with the register budget of F accumulators per lane.
  constexpr int WC = F <= 8 ? 24 : (F <= 16 ? 12 : 8);
  constexpr int RS = 32 / L;
  const int d = static_cast<int>(ds.d);
  const int row_bytes = d * 4;
  // Rows per tile: ~32 KB, a multiple of the rows all consumer warps take per
  // pass (balanced warps) and of 4 (16-byte bulk-copy granularity).
  const int unit = std::max(4, WC * RS);
  int R = std::max(unit, ((32768 / row_bytes) / unit) * unit);
  R = (R + 3) & ~3;
  DenseFullParams p{};
  p.x = ds.x.p;
  p.y = ds.labels.p;
  p.n = ds.n;
  p.d = d;
  p.R = R;
  p.ntiles = (ds.n + R - 1) / R;
  p.x_floats = static_cast<uint32_t>(R * d);
  p.stage_floats = (p.x_floats + R + 31) & ~31u;
  const size_t red_bytes = static_cast<size_t>(WC) * d * 4;
  const size_t budget = std::min<size_t>(c.max_smem_optin, 220 * 1024) - red_bytes - 256;
  int S = static_cast<int>(std::min<size_t>(8, budget / (p.stage_floats * 4ull)));
  if (S < 2) throw Unsupported("dense tile does not fit shared memory");
  p.S = S;
  const size_t smem = 128 * ((16 * S + 127) / 128) + (size_t)S * p.stage_floats * 4 + red_bytes;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(p.ntiles, c.num_sms));
  m.partials.alloc(static_cast<uint64_t>(grid) * d);
  p.w32 = m.w32.p;
  p.tail = GradTail{m.partials.p, m.ticket.p, d, a.alpha, a.apply ? 1 : 0, a.want_norm ? 1 : 0,
                    m.w64.p, m.w32.p, m.g64.p, m.finite.p, m.scal.p};
  auto kern = dense_full_kernel<L, F, TASK, WC>;
  check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)),
        "cudaFuncSetAttribute(dense_full)");
  prof_begin(c, "dense_full_kernel");
  kern<<<grid, 32 * (WC + 1), smem, c.stream>>>(p);
  launched(c, "dense_full_kernel");
}

template <int L, int F, int TASK>
void launch_dense_batch_LF(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb,
                           const StepArgs& a) {
  Ctx& c = *ds.ctx;
  constexpr int W = 8;
  constexpr int RS = 32 / L;
  const int d = static_cast<int>(ds.d);
  DenseBatchParams p{ds.x.p,  ds.labels.p, ds.n,     ds.row_base, d,
                     ids,     nb,          m.w32.p,  m.g64.p,     m.ticket.p,
                     m.finite.p, m.w64.p,  m.w32.p,  m.scal.p,    a.alpha,
                     a.apply ? 1 : 0, a.want_norm ? 1 : 0, a.alpha_dev};
  const unsigned grid = grid_for(c, static_cast<uint64_t>(W) * RS * 2, nb, 8);
  const size_t smem = static_cast<size_t>(W) * d * 4;
  auto kern = dense_batch_kernel<L, F, TASK, W>;
  if (smem > 48 * 1024)
    check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)),
          "cudaFuncSetAttribute(dense_batch)");
  prof_begin(c, "dense_batch_kernel");
  kern<<<grid, 32 * W, smem, c.stream>>>(p);
  launched(c, "dense_batch_kernel");
}

template <int L, int F, int TASK, int W>
void launch_dense_epoch_LFW(Dataset& ds, Model& m, uint64_t B, double alpha) {
  Ctx& c = *ds.ctx;
  constexpr int RS = 32 / L;
  const int d = static_cast<int>(ds.d);
  const size_t smem = static_cast<size_t>(d) * 8 + static_cast<size_t>(W) * d * 4;
  auto kern = dense_epoch_kernel<L, F, TASK, W>;
  if (smem > 48 * 1024)
    check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)),
          "cudaFuncSetAttribute(dense_epoch)");
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem), "occupancy");
  const uint64_t want = (B + W * RS - 1) / (W * RS);
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(std::max(1, per_sm)) * c.num_sms)));
  m.g3.alloc(3 * ds.d);
  m.gbar.alloc(2);
  check(cudaMemsetAsync(m.g3.p, 0, 3 * ds.d * sizeof(double), c.stream), "memset g3");
  check(cudaMemsetAsync(m.gbar.p, 0, 2 * sizeof(unsigned), c.stream), "memset barrier");
  DenseEpochParams p{ds.x.p, ds.labels.p, ds.n, ds.row_base, d, ds.order.p, ds.n_global, B,
                     m.g3.p, m.gbar.p, m.finite.p, m.w64.p, m.w32.p, alpha};
  void* args[] = {&p};
  prof_begin(c, "dense_epoch_kernel");
  check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(32 * W), args,
                                    smem, c.stream),
        "cudaLaunchCooperativeKernel(dense_epoch)");
  launched(c, "dense_epoch_kernel");
}

template <int L, int F>
void launch_dense_loss_LF(Dataset& ds, Model& m, int task) {
  Ctx& c = *ds.ctx;
  constexpr int RS = 32 / L;
  const unsigned grid = grid_for(c, 8ull * RS * 4, ds.n, 8);
  c.loss_partials.alloc(grid);
  prof_begin(c, "dense_loss_kernel");
  dense_loss_kernel<L, F><<<grid, 256, 0, c.stream>>>(
      ds.x.p, ds.labels.p, ds.n, static_cast<int>(ds.d), m.w64.p, task,
      LossTail{c.loss_partials.p, c.tickets.p, c.loss_out.p});
  launched(c, "dense_loss_kernel");
}

// (L, F) per d: L lanes per row, F features per lane, L*F >= d.
template <class Fn>
void dispatch_dense(uint64_t d, Fn&& fn) {
  if (d <= 32) fn.template operator()<4, 8>();
  else if (d <= 64) fn.template operator()<8, 8>();
  else if (d <= 128) fn.template operator()<16, 8>();
  else if (d <= 256) fn.template operator()<32, 8>();
  else if (d <= 512) fn.template operator()<32, 16>();
  else if (d <= 1024) fn.template operator()<32, 32>();
  else throw Unsupported("dense kernels handle d <= 1024 (wider data is stored as CSR)");
}

template <int G, int TASK>
void launch_csr_coef_G(Dataset& ds, Model& m) {
  Ctx& c = *ds.ctx;
  const unsigned grid = grid_for(c, 8ull * (32 / G) * 4, ds.n, 8);
  prof_begin(c, "csr_coef_kernel");
  csr_coef_kernel<G, TASK><<<grid, 256, 0, c.stream>>>(ds.val.p, ds.idx.p, ds.rowptr.p,
                                                       ds.labels.p, ds.n, m.w32.p, ds.coef.p);
  launched(c, "csr_coef_kernel");
}

template <int G, int TASK, bool SMEM>
void launch_csr_coef_pipe_G(Dataset& ds, Model& m) {
  Ctx& c = *ds.ctx;
  const size_t smem = SMEM ? ds.d * sizeof(float) : 0;
  const int threads = SMEM ? 1024 : 256;
  auto kern = csr_coef_pipe_kernel<G, TASK, SMEM>;
  if (smem > 48 * 1024)
    check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
          "cudaFuncSetAttribute(csr_coef_pipe)");
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem), "occupancy");
  const uint64_t want = (ds.n * G + threads - 1) / threads;
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(std::max(1, per_sm)) * c.num_sms)));
  prof_begin(c, "csr_coef_kernel");
  kern<<<grid, threads, smem, c.stream>>>(ds.val.p, ds.idx.p, ds.rowptr.p, ds.labels.p, ds.n, m.w32.p,
                                          static_cast<uint32_t>(ds.d), ds.coef.p);
  launched(c, "csr_coef_kernel");
}

template <int TASK>
void launch_csr_coef_vec(Dataset& ds, Model& m) {
  Ctx& c = *ds.ctx;
  auto kern = csr_coef_vec_kernel<TASK>;
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0), "occupancy");
  const uint64_t want = (ds.n * 32 + 255) / 256;
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(std::max(1, per_sm)) * c.num_sms)));
  prof_begin(c, "csr_coef_kernel");
  kern<<<grid, 256, 0, c.stream>>>(ds.val.p, ds.idx.p, ds.rowptr.p, ds.labels.p, ds.n, m.w32.p, ds.coef.p);
  launched(c, "csr_coef_kernel");
}

template <int G>
void launch_csc_block_G(Dataset& ds, Model& m) {
  Ctx& c = *ds.ctx;
  const size_t smem = static_cast<size_t>(ds.csc_rb) * sizeof(float);
  auto kern = csc_block_kernel<G>;
  if (smem > 48 * 1024)
    check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
          "cudaFuncSetAttribute(csc_block)");
  int per_sm = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1024, smem), "occupancy");
  const uint32_t slots = static_cast<uint32_t>(std::max(1, per_sm) * c.num_sms);
  const uint32_t cpb = std::max<uint32_t>(1, slots / ds.csc_nblk);
  m.partials.alloc(static_cast<uint64_t>(ds.csc_nblk) * ds.d);
  prof_begin(c, "csc_grad_kernel");
  kern<<<cpb * ds.csc_nblk, 1024, smem, c.stream>>>(ds.cval.p, ds.crow.p, ds.colptr.p, ds.coef.p, ds.n,
                                                    static_cast<uint32_t>(ds.d), ds.csc_rb,
                                                    ds.csc_nblk, cpb, m.partials.p);
  launched(c, "csc_grad_kernel");
}

void launch_apply_partials(Dataset& ds, Model& m, const StepArgs& a) {
  Ctx& c = *ds.ctx;
  const unsigned grid = grid_for(c, 256ull * 4, ds.d, 8);
  prof_begin(c, "apply_partials_kernel");
  apply_partials_kernel<<<grid, 256, 0, c.stream>>>(ds.d, ds.csc_nblk, m.partials.p, a.alpha,
                                                    a.apply ? 1 : 0, a.want_norm ? 1 : 0, m.w64.p,
                                                    m.w32.p, m.g64.p, m.finite.p, m.scal.p);
  launched(c, "apply_partials_kernel");
}

template <int G, int TASK>
void launch_csr_batch_G(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb, bool check) {
  Ctx& c = *ds.ctx;
  const unsigned grid = grid_for(c, 8ull * (32 / G) * 2, nb, 8);
  prof_begin(c, "csr_batch_kernel");
  csr_batch_kernel<G, TASK><<<grid, 256, 0, c.stream>>>(
      ds.val.p, ds.idx.p, ds.rowptr.p, ds.labels.p, ds.n, ds.row_base, ids, nb, m.w32.p,
      m.g64.p, m.finite.p, check ? 1 : 0);
  launched(c, "csr_batch_kernel");
}

template <int G>
void launch_csr_loss_G(Dataset& ds, Model& m, int task) {
  Ctx& c = *ds.ctx;
  const unsigned grid = grid_for(c, 8ull * (32 / G) * 4, ds.n, 8);
  c.loss_partials.alloc(grid);
  prof_begin(c, "csr_loss_kernel");
  csr_loss_kernel<G><<<grid, 256, 0, c.stream>>>(
      ds.val.p, ds.idx.p, ds.rowptr.p, ds.labels.p, ds.n, m.w64.p, task,
      LossTail{c.loss_partials.p, c.tickets.p, c.loss_out.p});
  launched(c, "csr_loss_kernel");
}

template <class Fn>
void dispatch_G(int g, Fn&& fn) {
  switch (g) {
    case 4: fn.template operator()<4>(); break;
    case 8: fn.template operator()<8>(); break;
    case 16: fn.template operator()<16>(); break;
    default: fn.template operator()<32>(); break;
  }
}

}  // namespace

void dense_full_step(Dataset& ds, Model& m, const StepArgs& a) {
  if (ds.n == 0) return;
  dispatch_dense(ds.d, [&]<int L, int F>() {
    if (a.task == kTaskLR) launch_dense_full_LF<L, F, kTaskLR>(ds, m, a);
    else launch_dense_full_LF<L, F, kTaskSVM>(ds, m, a);
  });
}

bool dense_epoch(Dataset& ds, Model& m, int task, double alpha, uint64_t B) {
  const char* e = std::getenv("SGDB_EPOCH_WARPS");
  const int w_env = e ? std::atoi(e) : 0;
  bool handled = true;
  dispatch_dense(ds.d, [&]<int L, int F>() {
    // Large batches of wide rows stream better through the per-step kernels
    // (measured: d = 1000, B = 65536: 72 vs 86 us per step).
    if (F > 16 && B > 16384) {
      handled = false;
      return;
    }
    // Measured (scripts/minibatch_time.py): 16 warps per CTA for F <= 8, else 8.
    const int w = w_env ? w_env : (F <= 8 ? 16 : 8);
    auto go = [&]<int W>() {
      if (task == kTaskLR) launch_dense_epoch_LFW<L, F, kTaskLR, W>(ds, m, B, alpha);
      else launch_dense_epoch_LFW<L, F, kTaskSVM, W>(ds, m, B, alpha);
    };
    if (w == 16) go.template operator()<16>();
    else if (w == 32) go.template operator()<32>();
    else go.template operator()<8>();
  });
  return handled;
}

void dense_batch_step(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb,
                      const StepArgs& a) {
  dispatch_dense(ds.d, [&]<int L, int F>() {
    if (a.task == kTaskLR) launch_dense_batch_LF<L, F, kTaskLR>(ds, m, ids, nb, a);
    else launch_dense_batch_LF<L, F, kTaskSVM>(ds, m, ids, nb, a);
  });
}

void csr_full_step(Dataset& ds, Model& m, const StepArgs& a) {
  build_csc(ds);
  if (ds.n > 0) {
    const int g = env_lanes("SGDB_ROW_LANES", lanes_for(static_cast<double>(ds.nnz) / static_cast<double>(ds.n)));
    // SMEM staging of the model: opt-in (SGDB_COEF_SMEM=1); measured slower on
    // rcv1 because one 189 KB CTA per SM halves the resident warps.
    static const bool smem_pref = [] {
      const char* e = std::getenv("SGDB_COEF_SMEM");
      return e && std::atoi(e) != 0;
    }();
    const bool smem_model = smem_pref && ds.d * sizeof(float) <= 192 * 1024;
    static const bool vec_pref = [] {
      const char* e = std::getenv("SGDB_ROW_VEC");
      return !e || std::atoi(e) != 0;
    }();
    if (g == 32 && vec_pref && !smem_model) {
      if (a.task == kTaskLR) launch_csr_coef_vec<kTaskLR>(ds, m);
      else launch_csr_coef_vec<kTaskSVM>(ds, m);
    } else dispatch_G(g, [&]<int G>() {
      if (smem_model) {
        if (a.task == kTaskLR) launch_csr_coef_pipe_G<G, kTaskLR, true>(ds, m);
        else launch_csr_coef_pipe_G<G, kTaskSVM, true>(ds, m);
      } else {
        if (a.task == kTaskLR) launch_csr_coef_pipe_G<G, kTaskLR, false>(ds, m);
        else launch_csr_coef_pipe_G<G, kTaskSVM, false>(ds, m);
      }
    });
  }
  const double per_col = static_cast<double>(ds.nnz) /
                         static_cast<double>(std::max<uint64_t>(1, ds.d) * std::max(1u, ds.csc_nblk));
  // Column segments: narrow groups amortise the per-column reduction over
  // more columns per warp (measured: rcv1 8 lanes, news20/real-sim 4).
  const int gc = per_col <= 16.0 ? 4 : (per_col <= 128.0 ? 8 : 16);
  dispatch_G(env_lanes("SGDB_COL_LANES", gc), [&]<int G>() { launch_csc_block_G<G>(ds, m); });
  launch_apply_partials(ds, m, a);
}

void csr_batch_step(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb, const StepArgs& a) {
  const int g = lanes_for(ds.n ? static_cast<double>(ds.nnz) / static_cast<double>(ds.n) : 1.0);
  dispatch_G(g, [&]<int G>() {
    if (a.task == kTaskLR) launch_csr_batch_G<G, kTaskLR>(ds, m, ids, nb, a.apply);
    else launch_csr_batch_G<G, kTaskSVM>(ds, m, ids, nb, a.apply);
  });
  if (a.apply) apply_update(m, a.alpha, a.want_norm, a.alpha_dev);
}

void apply_update(Model& m, double alpha, bool want_norm, const double* alpha_dev) {
  Ctx& c = *m.ctx;
  const unsigned grid = grid_for(c, 256ull * 4, m.d, 8);
  prof_begin(c, "apply_kernel");
  apply_kernel<<<grid, 256, 0, c.stream>>>(m.d, alpha, alpha_dev, m.w64.p, m.w32.p, m.g64.p, m.finite.p,
                                           m.scal.p, want_norm ? 1 : 0);
  launched(c, "apply_kernel");
}

void loss_launch(Dataset& ds, Model& m, int task) {
  Ctx& c = *ds.ctx;
  if (ds.n == 0) {
    check(cudaMemsetAsync(c.loss_out.p, 0, sizeof(double), c.stream), "memset loss");
    return;
  }
  if (ds.kind == Kind::Dense) {
    dispatch_dense(ds.d, [&]<int L, int F>() { launch_dense_loss_LF<L, F>(ds, m, task); });
  } else {
    const int g = lanes_for(static_cast<double>(ds.nnz) / static_cast<double>(ds.n));
    dispatch_G(g, [&]<int G>() { launch_csr_loss_G<G>(ds, m, task); });
  }
}

void sync_w64_from_w32(Model& m) {
  Ctx& c = *m.ctx;
  const unsigned grid = grid_for(c, 256ull * 4, m.d, 8);
  prof_begin(c, "w64_from_w32_kernel");
  w64_from_w32_kernel<<<grid, 256, 0, c.stream>>>(m.d, m.w32.p, m.w64.p);
  launched(c, "w64_from_w32_kernel");
}

}  // namespace sgdb::dev
