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
#include "segstream.cuh"
#include <cub/cub.cuh>

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
// scratch: `cap` doubles of shared memory free by the time the tail runs.
__device__ void grad_tail(const GradTail& t, double* s_part, int cap) {
  __shared__ unsigned s_last;
  __shared__ double s_red[32];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(t.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // The last CTA reduces gridDim.x partials per coordinate while every other
  // SM idles, so the sum is spread over all its threads: `parts` threads per
  // coordinate each add a contiguous run of blocks (16 loads in flight), then
  // the runs are added in order. Fixed order; a per-CTA timeline showed the
  // one-thread-per-coordinate tail taking ~11 us of a 37 us covtype epoch
  // (now ~9 us; covtype epoch 43 -> 41 us).
  const int d = t.d;
  const unsigned G = gridDim.x;
  const int parts = max(1, min(16, min(static_cast<int>(blockDim.x) / max(1, d), cap / max(1, d))));
  const unsigned run = (G + parts - 1) / parts;
  if (parts > 1) {
    const int part = threadIdx.x / d, j = threadIdx.x % d;
    if (part < parts) {
      const unsigned b0 = part * run, b1 = min(G, b0 + run);
      double g = 0.0;
      unsigned b = b0;
      for (; b + 16 <= b1; b += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = __ldcg(&t.partials[(size_t)(b + q) * d + j]);
#pragma unroll
        for (int q = 0; q < 16; ++q) g += v[q];
      }
      for (; b < b1; ++b) g += __ldcg(&t.partials[(size_t)b * d + j]);
      s_part[part * d + j] = g;
    }
    __syncthreads();
  }
  double nrm = 0.0;
  int bad = 0;
  for (int j = threadIdx.x; j < t.d; j += blockDim.x) {
    double g = 0.0;
    if (parts > 1) {
      for (int q = 0; q < parts; ++q) g += s_part[q * d + j];
    } else {
      unsigned b = 0;
      for (; b + 16 <= G; b += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = __ldcg(&t.partials[(size_t)(b + q) * d + j]);
#pragma unroll
        for (int q = 0; q < 16; ++q) g += v[q];
      }
      for (; b < G; ++b) g += __ldcg(&t.partials[(size_t)b * d + j]);
    }
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

  // Stage index and phase bit advance as counters (a runtime `i % S` cost a
  // ~20-instruction division per tile per warp).
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;  // phase of the ring pass this tile is in
      uint64_t i = 0;
      for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++i) {
        if (i >= (uint64_t)p.S) mbar_wait(&empty[s], ph ^ 1u);
        const uint64_t r0 = t * p.R;
        const uint64_t rows = min(static_cast<uint64_t>(p.R), p.n - r0);
        const uint32_t xb = round_up16(rows * d * 4ull), yb = round_up16(rows * 4ull);
        float* st = stages + (size_t)s * p.stage_floats;
        mbar_arrive_expect_tx(&full[s], xb + yb);
        bulk_g2s(st, p.x + r0 * d, xb, &full[s]);
        bulk_g2s(st + p.x_floats, p.y + r0, yb, &full[s]);
        if (++s == p.S) {
          s = 0;
          ph ^= 1u;
        }
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
    int s = 0;
    uint32_t ph = 0;
    for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      mbar_wait(&full[s], ph);
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
        const float c = valid ? coef_fast<TASK>(z, ys[r]) : 0.f;
#pragma unroll
        for (int k = 0; k < F; ++k) acc[k] = fmaf(c, xv[k], acc[k]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == p.S) {
        s = 0;
        ph ^= 1u;
      }
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
  // The stage ring is idle now: it holds the tail's per-run sums.
  grad_tail(p.tail, reinterpret_cast<double*>(stages),
            static_cast<int>(min(static_cast<unsigned long long>(p.S) * p.stage_floats / 2, 1ull << 20)));
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
      const float c = vn ? coef_fast<TASK>(z, yn) : 0.f;
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
      const float c = v ? coef_fast<TASK>(z, yv) : 0.f;
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

// Extents of a warp's contiguous row (or column) range, cached 32 at a time:
// lane l holds the pointer (and label) of entry r0 + 32q + l, `end` the
// pointer after the chunk. Extents are read with shuffles, so the only
// dependent global load left in an entry's chain is its own window.
struct RowChunk {
  uint32_t rp, end;
  float y;
};

// One pipeline stage: an entry's extent and its first window.
template <class W>
struct Stage {
  uint32_t b, e;
  float y;
  W g;
};


// ---------------------------------------------------------------------------
// K2t: margin pass as a segmented warp stream (segstream.cuh): each warp
// walks the nonzeros of a contiguous row range in 128-slot tiles regardless
// of row lengths; the model is staged in SMEM when it fits (SMEM), else
// gathered through L1/L2. Per-row sums are fp32, as in K2/K2v.
// ---------------------------------------------------------------------------
// Elements per lane per tile: 4 = one float4 + one index vector, so every
// warp-wide load is a contiguous 512 B (E = 8 doubles L1 wavefronts per load
// and made the kernels L1-bound; ncu l1tex 90 %).
constexpr int kSegE = 4;

// Warp w streams the nonzeros [w*nnz/NW, (w+1)*nnz/NW) whatever the row
// boundaries (news20's rows run to 9,100 slots; a row-balanced split left
// one warp with ~5x the average work). orow[w] = first row starting at or
// after warp w's first element (orow[NW] = n). A row cut by warp boundaries
// is finished from the per-warp pieces — pf[w]: the part of a row continued
// into warp w up to its tail, pl[w]: the part of a row up to warp w's end —
// by csr_coef_fixup_kernel. Used when one row could outweigh a warp's share
// (split); otherwise each warp takes whole rows, n / NW of them.
__host__ __device__ __forceinline__ uint32_t seg_pos(uint64_t nnz, uint32_t w, uint32_t nw) {
  return static_cast<uint32_t>(nnz * w / nw);
}

template <int TASK, bool SMEM, int NT>
__global__ void __launch_bounds__(NT, 1) csr_coef_seg_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const float* __restrict__ y, uint32_t n,
    const float* __restrict__ w32, uint32_t d, float* __restrict__ coef,
    const uint32_t* __restrict__ orow, float* __restrict__ pf, float* __restrict__ pl, int split) {
  // Dynamic SMEM: [model (SMEM) | per-warp scratch].
  extern __shared__ __align__(16) unsigned char dsm[];
  float* ws = reinterpret_cast<float*>(dsm);
  auto* scratch = reinterpret_cast<SegScratch<float, kSegE>*>(
      dsm + (SMEM ? round_up16(uint64_t(d) * 4) : 0u));
  __shared__ uint64_t bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = lane; k < kSegE * 8; k += 32) scratch[warp].flags[k] = 0u;
  if (SMEM && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint32_t total = round_up16(uint64_t(d) * 4);  // w32 is allocated in 16-byte groups
    mbar_arrive_expect_tx(&bar, total);
    for (uint32_t off = 0; off < total; off += 32768)
      bulk_g2s(reinterpret_cast<char*>(ws) + off, reinterpret_cast<const char*>(w32) + off,
               min(32768u, total - off), &bar);
  }
  __syncthreads();
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nnz = __ldg(rowptr + n);
  uint32_t P0, P1, g0, g1;
  bool cont = false;
  if (split) {
    P0 = seg_pos(nnz, gw, nw);
    P1 = seg_pos(nnz, gw + 1, nw);
    const uint32_t o0 = __ldg(orow + gw), o1 = __ldg(orow + gw + 1);
    // Continued row: the one before o0, if it runs past P0.
    cont = o0 > 0 && __ldg(rowptr + o0) > P0 && __ldg(rowptr + o0 - 1) < P0;
    g0 = cont ? o0 - 1 : o0;
    g1 = o1;
  } else {  // whole rows, n / NW per warp
    g0 = static_cast<uint32_t>(uint64_t(n) * gw / nw);
    g1 = static_cast<uint32_t>(uint64_t(n) * (gw + 1) / nw);
    P0 = __ldg(rowptr + g0);
    P1 = __ldg(rowptr + g1);
  }
  const float* w = SMEM ? ws : w32;
  bool model_ready = !SMEM;  // the first tiles' loads overlap the model's bulk copy
  const float open = segment_stream<float, kSegE, 2, VecGroup>(
      rowptr, y, g0, g1, P0, P1, [&](uint32_t a, int k) { return vec_group(val, idx, a + 4 * k); },
      [&](const VecGroup (&g)[kSegE / 4], float* p) {
        if (!model_ready) {
          mbar_wait(&bar, 0);
          model_ready = true;
        }
#pragma unroll
        for (int k = 0; k < kSegE / 4; ++k) {
          if (SMEM) {
            p[4 * k + 0] = g[k].v.x * w[g[k].j.x];
            p[4 * k + 1] = g[k].v.y * w[g[k].j.y];
            p[4 * k + 2] = g[k].v.z * w[g[k].j.z];
            p[4 * k + 3] = g[k].v.w * w[g[k].j.w];
          } else {
            p[4 * k + 0] = g[k].v.x * __ldg(w + g[k].j.x);
            p[4 * k + 1] = g[k].v.y * __ldg(w + g[k].j.y);
            p[4 * k + 2] = g[k].v.z * __ldg(w + g[k].j.z);
            p[4 * k + 3] = g[k].v.w * __ldg(w + g[k].j.w);
          }
        }
      },
      [&](uint32_t r, float z, float yy, bool ok) {
        const float c = coef_fast<TASK>(z, yy);
        if (ok) {
          if (cont && r == g0) pf[gw] = z;
          else coef[r] = c;
        }
      },
      scratch[warp]);
  if (split && lane == 0 && g1 > g0 && __ldg(rowptr + g1) > P1) pl[gw] = open;
}

// Finishes the rows cut by warp boundaries (split mode): the warp where row
// r starts adds its pl, every warp lying wholly inside r adds its pl, the
// warp holding r's tail adds its pf — in warp order — and the coefficient is
// formed.
template <int TASK>
__global__ void csr_coef_fixup_kernel(const uint32_t* __restrict__ rowptr, const float* __restrict__ y,
                                      uint32_t n, const uint32_t* __restrict__ orow, uint32_t nw,
                                      const float* __restrict__ pf, const float* __restrict__ pl,
                                      float* __restrict__ coef) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  const uint64_t nnz = rowptr[n];
  const uint32_t o0 = orow[w], o1 = orow[w + 1];
  if (o1 <= o0) return;  // no row starts in this warp
  const uint32_t r = o1 - 1;
  if (rowptr[r + 1] <= seg_pos(nnz, w + 1, nw)) return;  // the row ends inside the warp
  float z = pl[w];
  for (uint32_t v = w + 1; v < nw; ++v) {
    if (rowptr[r + 1] > seg_pos(nnz, v + 1, nw)) {
      z += pl[v];  // warp v lies wholly inside row r
    } else {
      z += pf[v];
      break;
    }
  }
  coef[r] = coef_fast<TASK>(z, y[r]);
}

// orow[w] = first row whose start is >= warp w's first element (binary
// search over rowptr); orow[nw] = n.
__global__ void seg_partition_kernel(const uint32_t* __restrict__ rowptr, uint32_t n, uint32_t nw,
                                     uint32_t* __restrict__ orow) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w > nw) return;
  if (w == nw) {
    orow[w] = n;
    return;
  }
  const uint32_t P = seg_pos(rowptr[n], w, nw);
  uint32_t lo = 0, hi = n;  // first r in [0, n] with rowptr[r] >= P
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (rowptr[mid] >= P) hi = mid;
    else lo = mid + 1;
  }
  orow[w] = lo;
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

// K3v: K3 with the coefficient slice bulk-copied (1-D TMA) into SMEM, each
// warp walking a contiguous column range with its column pointers cached 32
// at a time (read by shuffles), and aligned 4-slot windows (float4 values +
// 4 packed u16 rows) two columns ahead, so no dependent load sits in a
// column's chain except its own window. Per lane, a window's four fp32
// products are summed in fp32 and added to the fp64 accumulator; the
// per-(block, column) sum order is fixed, so the gradient is deterministic.
struct CscWin {
  float4 v;
  uint2 r;
};

// Update applied straight from the column sums when there is a single row
// block (news20: 19,996 rows): no partials, no apply_partials_kernel.
struct DirectApply {
  int on;
  double alpha;
  int apply, want_norm;
  double* w64;
  float* w32;
  double* g64;
  int* finite;
  double* norm2;
  // Several row blocks, cooperative launch: after a grid barrier the CTAs
  // sum the partials and apply (K3f's arithmetic) instead of a second launch.
  unsigned* gbar;  // non-null: grid-apply mode (on == 0)
};

// K3f's per-coordinate work, shared by apply_partials_kernel and the
// grid-apply tail of K3t: g_j = sum_b partials[b][j] in block order.
template <bool CG>
__device__ __forceinline__ void apply_partials_range(uint64_t j0, uint64_t stride, uint64_t d,
                                                     uint32_t nblk, const double* partials,
                                                     double alpha, int apply, int want_norm,
                                                     double* w64, float* w32, double* g64,
                                                     int* finite, double* norm2) {
  double nrm = 0.0;
  int bad = 0;
  for (uint64_t j = j0; j < d; j += stride) {
    // Sum over blocks in block order; 16 loads in flight per thread (only
    // ~d threads exist, so memory parallelism has to come from each one).
    double g = 0.0;
    uint32_t b = 0;
    for (; b + 16 <= nblk; b += 16) {
      double v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const double* q = partials + static_cast<uint64_t>(b + k) * d + j;
        v[k] = CG ? __ldcg(q) : *q;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) g += v[k];
    }
    for (; b < nblk; ++b) {
      const double* q = partials + static_cast<uint64_t>(b) * d + j;
      g += CG ? __ldcg(q) : *q;
    }
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

template <int G, class ACC>
__global__ void __launch_bounds__(1024, 1) csc_vec_kernel(
    const float* __restrict__ cval, const uint16_t* __restrict__ crow,
    const uint32_t* __restrict__ colptr, const float* __restrict__ coef, uint64_t n, uint32_t d,
    uint32_t rb, uint32_t nblk, uint32_t cpb, double* __restrict__ partials, DirectApply da) {
  extern __shared__ __align__(16) float cs[];
  __shared__ uint64_t bar;
  const uint32_t b = blockIdx.x / cpb, k = blockIdx.x % cpb;
  if (b >= nblk) return;
  const uint64_t r0 = static_cast<uint64_t>(b) * rb;  // rb % 4 == 0: 16-byte aligned slice
  const uint32_t rows = static_cast<uint32_t>(min(static_cast<uint64_t>(rb), n - r0));
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint32_t total = round_up16(uint64_t(rows) * 4);  // coef carries 16-byte slack
    mbar_arrive_expect_tx(&bar, total);
    for (uint32_t off = 0; off < total; off += 32768)
      bulk_g2s(reinterpret_cast<char*>(cs) + off, reinterpret_cast<const char*>(coef + r0) + off,
               min(32768u, total - off), &bar);
  }
  constexpr uint32_t CW = 32 / G;   // columns per warp step
  constexpr uint32_t SPC = 32 / CW;  // steps per 32-column chunk
  const int lane = threadIdx.x & 31, lg = lane % G, gi = lane / G;
  const uint32_t warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t j0 = static_cast<uint32_t>(static_cast<uint64_t>(d) * k / cpb);
  const uint32_t j1 = static_cast<uint32_t>(static_cast<uint64_t>(d) * (k + 1) / cpb);
  const uint32_t c0 = j0 + static_cast<uint32_t>(static_cast<uint64_t>(j1 - j0) * warp / nw);
  const uint32_t c1 = j0 + static_cast<uint32_t>(static_cast<uint64_t>(j1 - j0) * (warp + 1) / nw);
  const uint32_t nsteps = (c1 - c0 + CW - 1) / CW;
  const uint32_t* cp = colptr + static_cast<uint64_t>(b) * (d + 1);
  auto load_chunk = [&](uint32_t q) {
    RowChunk ch;
    ch.rp = cp[min(c0 + 32 * q + lane, c1)];
    ch.end = cp[min(c0 + 32 * q + 32, c1)];
    ch.y = 0.f;
    return ch;
  };
  auto window = [&](uint32_t a) {
    CscWin w;
    w.v = __ldg(reinterpret_cast<const float4*>(cval + a));
    w.r = __ldg(reinterpret_cast<const uint2*>(crow + a));
    return w;
  };
  auto dot = [&](const CscWin& w, uint32_t a, uint32_t sb, uint32_t se) {
    const int lo = static_cast<int>(sb - a), hi = static_cast<int>(se - a);
    const float x0 = (0 >= lo && 0 < hi) ? w.v.x : 0.f;
    const float x1 = (1 >= lo && 1 < hi) ? w.v.y : 0.f;
    const float x2 = (2 >= lo && 2 < hi) ? w.v.z : 0.f;
    const float x3 = (3 >= lo && 3 < hi) ? w.v.w : 0.f;
    float t = x0 * cs[w.r.x & 0xffffu];
    t = fmaf(x1, cs[w.r.x >> 16], t);
    t = fmaf(x2, cs[w.r.y & 0xffffu], t);
    t = fmaf(x3, cs[w.r.y >> 16], t);
    return static_cast<ACC>(t);
  };
  constexpr bool kThird = SPC < 8;
  RowChunk A = load_chunk(0), B = load_chunk(1), C;
  if constexpr (kThird) C = load_chunk(2);
  uint32_t qa = 0;
  auto issue = [&](uint32_t s, Stage<CscWin>& st) {
    if (s / SPC != qa) {
      A = B;
      ++qa;
      if constexpr (kThird) {
        B = C;
        C = load_chunk(qa + 2);
      } else {
        B = load_chunk(qa + 1);
      }
    }
    const uint32_t l = (s % SPC) * CW + gi;
    st.b = __shfl_sync(0xffffffffu, A.rp, l);
    const uint32_t nx = __shfl_sync(0xffffffffu, A.rp, (l + 1) & 31);
    st.e = l == 31 ? A.end : nx;
    if (s >= nsteps) st.e = st.b;
    const uint32_t a = (st.b & ~3u) + 4u * lg;
    st.g = window(a < st.e ? a : 0u);
  };
  auto consume = [&](uint32_t s, const Stage<CscWin>& st) {
    const uint32_t a = (st.b & ~3u) + 4u * lg;
    ACC acc = dot(st.g, a, st.b, st.e);
    for (uint32_t aa = a + 4 * G; aa < st.e; aa += 4 * G) acc += dot(window(aa), aa, st.b, st.e);
    acc = group_sum<G>(acc);
    const uint32_t j = c0 + s * CW + gi;
    if (j < c1 && lg == 0) partials[static_cast<uint64_t>(b) * d + j] = static_cast<double>(acc);
  };
  Stage<CscWin> s0, s1, s2;
  issue(0, s0);
  issue(1, s1);
  __syncthreads();
  mbar_wait(&bar, 0);
  for (uint32_t s = 0; s < nsteps; s += 3) {
    issue(s + 2, s2);
    consume(s, s0);
    if (s + 1 >= nsteps) break;
    issue(s + 3, s0);
    consume(s + 1, s1);
    if (s + 2 >= nsteps) break;
    issue(s + 4, s1);
    consume(s + 2, s2);
  }
  if (da.gbar) {  // grid-apply tail (cooperative launch), as in K3t
    grid_sync(da.gbar, gridDim.x);
    apply_partials_range<true>(static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                               static_cast<uint64_t>(gridDim.x) * blockDim.x, d, nblk, partials,
                               da.alpha, da.apply, da.want_norm, da.w64, da.w32, da.g64,
                               da.finite, da.norm2);
  }
}

// K3t: the gradient pass over the blocked CSC as a segmented warp stream:
// CTA (block b, column range k) stages c[rows of b] in SMEM by bulk copy;
// each warp streams the nonzeros of a contiguous column range (columns are
// segments) in 128-slot tiles. Used for short columns (a few slots per
// block): fp32 products and fp32 segment sums (an fp64 scan was bound by
// the FP64 / conversion pipes, ncu math_pipe_throttle), stored as fp64
// partials.
template <int NT>
__global__ void __launch_bounds__(NT, 1) csc_seg_kernel(
    const float* __restrict__ cval, const uint16_t* __restrict__ crow,
    const uint32_t* __restrict__ colptr, const float* __restrict__ coef, uint64_t n, uint32_t d,
    uint32_t rb, uint32_t nblk, uint32_t cpb, double* __restrict__ partials, DirectApply da) {
  // Dynamic SMEM: [coefficient slice | per-warp scratch].
  extern __shared__ __align__(16) unsigned char dsm[];
  float* cs = reinterpret_cast<float*>(dsm);
  auto* scratch = reinterpret_cast<SegScratch<float, kSegE>*>(dsm + round_up16(uint64_t(rb) * 4));
  __shared__ uint64_t bar;
  const uint32_t b = blockIdx.x / cpb, k = blockIdx.x % cpb;
  if (b >= nblk) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = lane; q < kSegE * 8; q += 32) scratch[warp].flags[q] = 0u;
  const uint64_t r0 = static_cast<uint64_t>(b) * rb;  // rb % 4 == 0: 16-byte aligned slice
  const uint32_t rows = static_cast<uint32_t>(min(static_cast<uint64_t>(rb), n - r0));
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint32_t total = round_up16(uint64_t(rows) * 4);  // coef carries 16-byte slack
    mbar_arrive_expect_tx(&bar, total);
    for (uint32_t off = 0; off < total; off += 32768)
      bulk_g2s(reinterpret_cast<char*>(cs) + off, reinterpret_cast<const char*>(coef + r0) + off,
               min(32768u, total - off), &bar);
  }
  __syncthreads();
  const uint32_t nw = blockDim.x >> 5;
  const uint32_t j0 = static_cast<uint32_t>(static_cast<uint64_t>(d) * k / cpb);
  const uint32_t j1 = static_cast<uint32_t>(static_cast<uint64_t>(d) * (k + 1) / cpb);
  const uint32_t c0 = j0 + static_cast<uint32_t>(static_cast<uint64_t>(j1 - j0) * warp / nw);
  const uint32_t c1 = j0 + static_cast<uint32_t>(static_cast<uint64_t>(j1 - j0) * (warp + 1) / nw);
  const uint32_t* cp = colptr + static_cast<uint64_t>(b) * (d + 1);
  double* out = partials + static_cast<uint64_t>(b) * d;
  mbar_wait(&bar, 0);
  int bad = 0;
  double nrm = 0.0;
  segment_stream<float, kSegE, 2, CscWin>(
      cp, nullptr, c0, c1, __ldg(cp + c0), __ldg(cp + c1),
      [&](uint32_t a, int q) {
        CscWin w;
        w.v = __ldg(reinterpret_cast<const float4*>(cval + a + 4 * q));
        w.r = __ldg(reinterpret_cast<const uint2*>(crow + a + 4 * q));
        return w;
      },
      [&](const CscWin (&w)[kSegE / 4], float* p) {
#pragma unroll
        for (int q = 0; q < kSegE / 4; ++q) {
          p[4 * q + 0] = w[q].v.x * cs[w[q].r.x & 0xffffu];
          p[4 * q + 1] = w[q].v.y * cs[w[q].r.x >> 16];
          p[4 * q + 2] = w[q].v.z * cs[w[q].r.y & 0xffffu];
          p[4 * q + 3] = w[q].v.w * cs[w[q].r.y >> 16];
        }
      },
      [&](uint32_t j, float v, float, bool ok) {
        if (!ok) return;
        if (!da.on) {
          out[j] = static_cast<double>(v);
          return;
        }
        // One row block: this lane's sum IS g_j, so apply it here (K3f's
        // arithmetic) instead of staging partials for a separate pass.
        const double g = static_cast<double>(v);
        if (!isfinite(g)) bad = 1;
        if (da.apply) {
          const double w = da.w64[j] - da.alpha * g;
          da.w64[j] = w;
          da.w32[j] = static_cast<float>(w);
        } else {
          da.g64[j] = g;
        }
        nrm += g * g;
      },
      scratch[warp]);
  if (da.on) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) *da.finite = 0;
    if (da.want_norm) {
      nrm = warp_sum_d(nrm);
      if (lane == 0 && nrm != 0.0) atomicAdd(da.norm2, nrm);
    }
  } else if (da.gbar) {
    grid_sync(da.gbar, gridDim.x);  // every block's partials are written
    apply_partials_range<true>(static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                               static_cast<uint64_t>(gridDim.x) * blockDim.x, d, nblk, partials,
                               da.alpha, da.apply, da.want_norm, da.w64, da.w32, da.g64,
                               da.finite, da.norm2);
  }
}

// K3f: g_j = sum_b partials[b][j] (fixed order), fused w -= alpha*g_j (one
// writer per coordinate), finite flag, ||g||^2.
__global__ void apply_partials_kernel(uint64_t d, uint32_t nblk, const double* __restrict__ partials,
                                      double alpha, int apply, int want_norm, double* w64,
                                      float* w32, double* g64, int* finite, double* norm2) {
  apply_partials_range<false>((uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
                              (uint64_t)gridDim.x * blockDim.x, d, nblk, partials, alpha, apply,
                              want_norm, w64, w32, g64, finite, norm2);
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
    float yr = 0.f;
    if (valid) {  // the label is loaded with the extent, off the margin's chain
      b = rowptr[row];
      e = rowptr[row + 1];
      yr = y[row];
    }
    const float z = group_sum<G>(gather_dot<G>(val, idx, b, e, lg, w32));
    if (!valid) continue;
    const float c = coef_f<TASK>(z, yr);
    if (c == 0.f) continue;
    // Slots in batches of U: the U loads are in flight together instead of
    // one load -> red round trip per slot (ncu: 79 % long-scoreboard on the
    // one-deep loop, news20 B = 4096).
    constexpr int U = 8;
    for (uint32_t s0 = b + lg; s0 < e; s0 += G * U) {
      uint32_t jv[U];
      float xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t s = s0 + u * G;
        jv[u] = s < e ? __ldg(idx + s) : 0u;
        xv[u] = s < e ? __ldg(val + s) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (s0 + u * G < e) atomicAdd(&g64[jv[u]], static_cast<double>(c * xv[u]));
    }
  }
}


// ---------------------------------------------------------------------------
// K3c: sparse mini-batch in row chunks. A batch's rows are heavy-tailed (the
// longest of 4,096 rcv1 rows is ~18x the mean, news20 ~20x), and with one
// lane group per row the step lasted as long as its longest row's load chain
// (news20: 85 us for 1.9M slots). The rows are cut into chunks of CH = G*8
// slots; the plan (per epoch: chunk counts + exclusive scan over the order)
// lets every lane group take one chunk:
//   K3c-m: partial margin of each chunk -> mb_z (one slot per chunk);
//   K3c-s: the row margin = its chunks' partials summed in chunk order
//          (deterministic), coefficient, scatter of the chunk's c*x into g64
//          with fp64 atomics (red.global.add.f64).
// ---------------------------------------------------------------------------
__global__ void mb_count_kernel(const uint32_t* __restrict__ ids, uint64_t count,
                                const uint32_t* __restrict__ rowptr, uint64_t n_local,
                                uint64_t row_base, uint32_t ch, uint32_t* __restrict__ cnt) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= count;
       p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t k = 0;
    if (p < count) {
      const uint64_t row = static_cast<uint64_t>(ids[p]) - row_base;  // wraps if not local
      if (row < n_local) k = (rowptr[row + 1] - rowptr[row] + ch - 1) / ch;
    }
    cnt[p] = k;
  }
}

// Largest p in [lo, hi) with off[p] <= q (off[lo] <= q < off[hi]): the
// position owning chunk q (positions with no chunk share their successor's
// offset and are skipped).
__device__ __forceinline__ uint64_t chunk_owner(const uint32_t* __restrict__ off, uint64_t lo,
                                                uint64_t hi, uint32_t q) {
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct ChunkRef {
  uint64_t p = 0, row = 0;
  uint32_t b = 0, e = 0;
};

// Chunk q of the plan: one 16-byte load from the per-chunk table when the
// plan holds it (every permutation order), else the owner search.
template <int G, int U>
__device__ __forceinline__ ChunkRef chunk_ref(const uint4* __restrict__ meta, uint64_t cap,
                                              const uint32_t* __restrict__ off,
                                              const uint32_t* __restrict__ ids,
                                              const uint32_t* __restrict__ rowptr, uint64_t row_base,
                                              uint64_t lo, uint64_t hi, uint32_t q, bool direct) {
  ChunkRef r;
  if (direct) {
    const uint4 m = __ldg(meta + q);
    r.b = m.x;
    r.e = m.y;
    r.p = m.z;
    r.row = m.w;
    return r;
  }
  r.p = chunk_owner(off, lo, hi, q);
  const uint32_t sub = q - __ldg(off + r.p);
  r.row = static_cast<uint64_t>(__ldg(ids + r.p)) - row_base;
  const uint32_t rb = __ldg(rowptr + r.row), re = __ldg(rowptr + r.row + 1);
  r.b = rb + sub * static_cast<uint32_t>(G * U);
  r.e = min(r.b + static_cast<uint32_t>(G * U), re);
  return r;
}

__global__ void mb_fill_kernel(const uint32_t* __restrict__ ids, uint64_t count,
                               const uint32_t* __restrict__ rowptr, uint64_t row_base, uint32_t ch,
                               const uint32_t* __restrict__ off, uint4* __restrict__ meta,
                               uint64_t cap) {
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < count;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q0 = off[p], q1 = off[p + 1];
    if (q0 == q1) continue;
    const uint32_t row = static_cast<uint32_t>(static_cast<uint64_t>(ids[p]) - row_base);
    const uint32_t rb = rowptr[row], re = rowptr[row + 1];
    for (uint32_t q = q0; q < q1 && q < cap; ++q) {
      const uint32_t b = rb + (q - q0) * ch;
      meta[q] = make_uint4(b, min(b + ch, re), static_cast<uint32_t>(p), row);
    }
  }
}

template <int G, int U>
__global__ void __launch_bounds__(256) mb_margin_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const uint32_t* __restrict__ ids,
    const uint32_t* __restrict__ off, const uint4* __restrict__ meta, uint64_t cap, uint64_t lo,
    uint64_t hi, uint64_t row_base, const float* __restrict__ w32, float* __restrict__ zpart,
    const int* finite, int check_finite) {
  if (check_finite && *finite == 0) return;
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint32_t c0 = __ldg(off + lo), c1 = __ldg(off + hi);
  const bool direct = c1 <= cap;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = c0 + gw * RW; base < c1; base += tw * RW) {
    const uint64_t q = base + grp;
    const bool valid = q < c1;
    uint32_t b = 0, e = 0;
    if (valid) {
      const ChunkRef r = chunk_ref<G, U>(meta, cap, off, ids, rowptr, row_base, lo, hi,
                                         static_cast<uint32_t>(q), direct);
      b = r.b;
      e = r.e;
    }
    uint32_t jv[U];
    float xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t s = b + lg + u * G;
      jv[u] = s < e ? __ldg(idx + s) : 0u;
      xv[u] = s < e ? __ldg(val + s) : 0.f;
    }
    float z = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) z = fmaf(xv[u], b + lg + u * G < e ? __ldg(w32 + jv[u]) : 0.f, z);
    z = group_sum<G>(z);
    if (valid && lg == 0) zpart[q - c0] = z;
  }
}

template <int G, int U, int TASK>
__global__ void __launch_bounds__(256) mb_scatter_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const float* __restrict__ y,
    const uint32_t* __restrict__ ids, const uint32_t* __restrict__ off,
    const uint4* __restrict__ meta, uint64_t cap, uint64_t lo, uint64_t hi, uint64_t row_base,
    const float* __restrict__ zpart, double* g64, const int* finite, int check_finite,
    int prefetch_next, uint64_t count) {
  if (check_finite && *finite == 0) return;
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint32_t c0 = __ldg(off + lo), c1 = __ldg(off + hi);
  const bool direct = c1 <= cap;
  const uint64_t total = prefetch_next ? __ldg(off + count) : 0;  // chunks of the whole plan
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t q = c0 + gw * RW + grp; q < c1; q += tw * RW) {  // no shuffles: per group
    const ChunkRef r = chunk_ref<G, U>(meta, cap, off, ids, rowptr, row_base, lo, hi,
                                       static_cast<uint32_t>(q), direct);
    uint32_t jv[U];
    float xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // the chunk's slots load while the margin is summed
      const uint32_t s = r.b + lg + u * G;
      jv[u] = s < r.e ? __ldg(idx + s) : 0u;
      xv[u] = s < r.e ? __ldg(val + s) : 0.f;
    }
    const uint32_t z0 = __ldg(off + r.p) - c0, z1 = __ldg(off + r.p + 1) - c0;
    float z = 0.f;
    for (uint32_t k = z0; k < z1; ++k) z += __ldg(zpart + k);  // chunk order
    const float c = coef_f<TASK>(z, __ldg(y + r.row));
    if (c != 0.f) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r.b + lg + u * G < r.e) atomicAdd(&g64[jv[u]], static_cast<double>(c * xv[u]));
    }
    if (prefetch_next && total <= cap) {
      // Pull the slots of the chunk at the same position of the next step
      // into L2, so that step's margin pass reads them from L2, not HBM.
      const uint64_t qn = q + (c1 - c0);
      if (qn < total && lg < 16) {  // total <= cap: table entries below it are written
        const uint4 mn = __ldg(meta + qn);
        const uint32_t lines = min((mn.y - mn.x + 31) / 32, (U * G + 31) / 32u);  // 128-byte lines
        const char* base = lg < 8 ? reinterpret_cast<const char*>(idx + mn.x)
                                  : reinterpret_cast<const char*>(val + mn.x);
        for (uint32_t l = lg & 7; l < lines; l += 8)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(base + 128ull * l));
      }
    }
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
  static const int tile_bytes = [] {
    const char* e = std::getenv("SGDB_DENSE_TILE");
    return e ? std::atoi(e) : 32768;
  }();
  int R = std::max(unit, ((tile_bytes / row_bytes) / unit) * unit);
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
  set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(dense_full)");
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
    set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(dense_batch)");
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
    set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(dense_epoch)");
  int per_sm = 0;
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), 32 * W, smem);
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
  static const bool lf416 = [] {
    const char* e = std::getenv("SGDB_DENSE_LF416");
    return e && std::atoi(e) != 0;
  }();
  if (d <= 32) fn.template operator()<4, 8>();
  else if (d <= 64 && lf416) fn.template operator()<4, 16>();
  else if (d <= 64) fn.template operator()<8, 8>();
  else if (d <= 128) fn.template operator()<16, 8>();
  else if (d <= 256) fn.template operator()<32, 8>();
  else if (d <= 512) fn.template operator()<32, 16>();
  else if (d <= 1024) fn.template operator()<32, 32>();
  else throw Unsupported("dense kernels handle d <= 1024 (wider data is stored as CSR)");
}


template <int G, int TASK, bool SMEM>
void launch_csr_coef_pipe_G(Dataset& ds, Model& m) {
  Ctx& c = *ds.ctx;
  const size_t smem = SMEM ? ds.d * sizeof(float) : 0;
  const int threads = SMEM ? 1024 : 256;
  auto kern = csr_coef_pipe_kernel<G, TASK, SMEM>;
  if (smem > 48 * 1024)
    set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(csr_coef_pipe)");
  int per_sm = 0;
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), threads, smem);
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
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), 256, 0);
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
    set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(csc_block)");
  int per_sm = 0;
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), 1024, smem);
  const uint32_t slots = static_cast<uint32_t>(std::max(1, per_sm) * c.num_sms);
  const uint32_t cpb = std::max<uint32_t>(1, slots / ds.csc_nblk);
  m.partials.alloc(static_cast<uint64_t>(ds.csc_nblk) * ds.d);
  prof_begin(c, "csc_grad_kernel");
  kern<<<cpb * ds.csc_nblk, 1024, smem, c.stream>>>(ds.cval.p, ds.crow.p, ds.colptr.p, ds.coef.p, ds.n,
                                                    static_cast<uint32_t>(ds.d), ds.csc_rb,
                                                    ds.csc_nblk, cpb, m.partials.p);
  launched(c, "csc_grad_kernel");
}

template <int G>
void launch_csc_vec_G(Dataset& ds, Model& m, const DirectApply& da) {
  Ctx& c = *ds.ctx;
  const size_t smem = round_up16(static_cast<uint64_t>(ds.csc_rb) * sizeof(float));
  // fp64 per-(block, column) sums (fp32 sums measured no faster: 85 vs 83 us on rcv1).
  auto kern = csc_vec_kernel<G, double>;
  set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(csc_vec)");
  int per_sm = 0;
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), 1024, smem);
  const uint32_t slots = static_cast<uint32_t>(std::max(1, per_sm) * c.num_sms);
  const uint32_t cpb = std::max<uint32_t>(1, slots / ds.csc_nblk);
  m.partials.alloc(static_cast<uint64_t>(ds.csc_nblk) * ds.d);
  prof_begin(c, "csc_grad_kernel");
  if (da.gbar) {
    check(cudaMemsetAsync(da.gbar, 0, sizeof(unsigned), c.stream), "memset barrier");
    const float* cval = ds.cval.p;
    const uint16_t* crow = ds.crow.p;
    const uint32_t* colptr = ds.colptr.p;
    const float* coef = ds.coef.p;
    uint64_t n = ds.n;
    uint32_t d = static_cast<uint32_t>(ds.d), rb = ds.csc_rb, nblk = ds.csc_nblk, cpb_ = cpb;
    double* partials = m.partials.p;
    DirectApply dav = da;
    void* args[] = {&cval, &crow, &colptr, &coef, &n, &d, &rb, &nblk, &cpb_, &partials, &dav};
    check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(cpb * ds.csc_nblk),
                                      dim3(1024), args, smem, c.stream),
          "cudaLaunchCooperativeKernel(csc_vec)");
  } else {
    kern<<<cpb * ds.csc_nblk, 1024, smem, c.stream>>>(ds.cval.p, ds.crow.p, ds.colptr.p, ds.coef.p,
                                                      ds.n, static_cast<uint32_t>(ds.d), ds.csc_rb,
                                                      ds.csc_nblk, cpb, m.partials.p, da);
  }
  launched(c, "csc_grad_kernel");
}

template <int TASK, bool SMEM, int NT>
bool launch_csr_coef_seg_N(Dataset& ds, Model& m) {
  Ctx& c = *ds.ctx;
  const size_t smem = (SMEM ? round_up16(ds.d * sizeof(float)) : 0) +
                      (NT / 32) * sizeof(SegScratch<float, kSegE>);
  auto kern = csr_coef_seg_kernel<TASK, SMEM, NT>;
  const size_t static_smem = static_smem_of(reinterpret_cast<const void*>(kern));
  if (static_smem + smem > c.max_smem_optin) return false;  // try fewer threads
  if (smem > 48 * 1024)
    set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(csr_coef_seg)");
  int per_sm = 0;
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), NT, smem);
  if (per_sm < 1) return false;
  // ~2 tiles per warp at least keeps short inputs spread out.
  const uint64_t want = std::max<uint64_t>(1, (ds.nnz / 512 + NT / 32 - 1) / (NT / 32));
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(per_sm) * c.num_sms)));
  const uint32_t nw = grid * (NT / 32);
  // Split rows across warps when one row could outweigh a warp's share
  // several times over (news20: 9,100-slot rows vs ~1,950 slots per warp);
  // otherwise whole rows per warp need no fix-up pass.
  // Also on large inputs, where the balance gain outweighs the fix-up launch
  // (rcv1: 135 -> 114 + 9 us; w8a / real-sim lose a few us).
  const char* se = std::getenv("SGDB_SEG_SPLIT");  // 1 / 0 force it (tests, A/B)
  const bool split = se ? std::atoi(se) != 0
                        : (ds.max_row > 4 * (ds.nnz / std::max<uint32_t>(1, nw)) || ds.nnz > (16ull << 20));
  if (split && ds.seg_nw != nw) {  // warp partition of the nonzeros (cached per dataset and warp count)
    ds.seg_orow.alloc(nw + 1);
    ds.seg_pf.alloc(nw);
    ds.seg_pl.alloc(nw);
    prof_begin(c, "seg_partition_kernel");
    seg_partition_kernel<<<(nw + 256) / 256, 256, 0, c.stream>>>(ds.rowptr.p, static_cast<uint32_t>(ds.n), nw,
                                                               ds.seg_orow.p);
    launched(c, "seg_partition_kernel");
    ds.seg_nw = nw;
  }
  prof_begin(c, "csr_coef_kernel");
  kern<<<grid, NT, smem, c.stream>>>(ds.val.p, ds.idx.p, ds.rowptr.p, ds.labels.p,
                                     static_cast<uint32_t>(ds.n), m.w32.p,
                                     static_cast<uint32_t>(ds.d), ds.coef.p, ds.seg_orow.p,
                                     ds.seg_pf.p, ds.seg_pl.p, split ? 1 : 0);
  launched(c, "csr_coef_kernel");
  if (split) {
    prof_begin(c, "csr_coef_fixup_kernel");
    csr_coef_fixup_kernel<TASK><<<(nw + 255) / 256, 256, 0, c.stream>>>(
        ds.rowptr.p, ds.labels.p, static_cast<uint32_t>(ds.n), ds.seg_orow.p, nw, ds.seg_pf.p,
        ds.seg_pl.p, ds.coef.p);
    launched(c, "csr_coef_fixup_kernel");
  }
  return true;
}

template <int NT>
bool launch_csc_seg_N(Dataset& ds, Model& m, const DirectApply& da) {
  Ctx& c = *ds.ctx;
  const size_t smem = round_up16(static_cast<uint64_t>(ds.csc_rb) * sizeof(float)) +
                      (NT / 32) * sizeof(SegScratch<float, kSegE>);
  auto kern = csc_seg_kernel<NT>;
  const size_t static_smem = static_smem_of(reinterpret_cast<const void*>(kern));
  if (static_smem + smem > c.max_smem_optin) return false;
  set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(csc_seg)");
  int per_sm = 0;
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), NT, smem);
  if (per_sm < 1) return false;
  const uint32_t slots = static_cast<uint32_t>(per_sm * c.num_sms);
  const uint32_t cpb = std::max<uint32_t>(1, slots / ds.csc_nblk);
  m.partials.alloc(static_cast<uint64_t>(ds.csc_nblk) * ds.d);
  prof_begin(c, "csc_grad_kernel");
  if (da.gbar) {  // grid-apply tail: co-residency guaranteed by the cooperative launch
    check(cudaMemsetAsync(da.gbar, 0, sizeof(unsigned), c.stream), "memset barrier");
    const float* cval = ds.cval.p;
    const uint16_t* crow = ds.crow.p;
    const uint32_t* colptr = ds.colptr.p;
    const float* coef = ds.coef.p;
    uint64_t n = ds.n;
    uint32_t d = static_cast<uint32_t>(ds.d), rb = ds.csc_rb, nblk = ds.csc_nblk, cpb_ = cpb;
    double* partials = m.partials.p;
    DirectApply dav = da;
    void* args[] = {&cval, &crow, &colptr, &coef, &n, &d, &rb, &nblk, &cpb_, &partials, &dav};
    check(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(cpb * ds.csc_nblk),
                                      dim3(NT), args, smem, c.stream),
          "cudaLaunchCooperativeKernel(csc_seg)");
  } else {
    kern<<<cpb * ds.csc_nblk, NT, smem, c.stream>>>(ds.cval.p, ds.crow.p, ds.colptr.p, ds.coef.p,
                                                    ds.n, static_cast<uint32_t>(ds.d), ds.csc_rb,
                                                    ds.csc_nblk, cpb, m.partials.p, da);
  }
  launched(c, "csc_grad_kernel");
  return true;
}

// CTA size: the largest of 1024 / 768 / 512 threads whose per-warp scratch
// fits next to the staged model (or coefficient slice); SGDB_SEG_THREADS
// caps it for A/B runs.
int seg_threads() {
  static const int nt = [] {
    const char* e = std::getenv("SGDB_SEG_THREADS");
    return e ? std::atoi(e) : 1024;
  }();
  return nt;
}

template <int TASK>
void launch_csr_coef_seg(Dataset& ds, Model& m, bool smem_model) {
  const int nt = seg_threads();
  auto go = [&]<bool SM>() {
    if (nt >= 1024 && launch_csr_coef_seg_N<TASK, SM, 1024>(ds, m)) return true;
    if (nt >= 768 && launch_csr_coef_seg_N<TASK, SM, 768>(ds, m)) return true;
    return launch_csr_coef_seg_N<TASK, SM, 512>(ds, m);
  };
  if (smem_model && go.template operator()<true>()) return;
  if (!go.template operator()<false>()) throw CudaError("csr_coef_seg: no launchable configuration");
}

// Grid-apply tail (several row blocks): the gradient kernel sums the partials
// and applies after a grid barrier. SGDB_CSC_GRID_APPLY=0 keeps the separate
// K3f launch (A/B).
DirectApply grid_apply_args(Model& m, const StepArgs& a) {
  static const bool on = [] {
    const char* e = std::getenv("SGDB_CSC_GRID_APPLY");
    return !(e && std::atoi(e) == 0);
  }();
  if (!on) return DirectApply{};
  m.gbar.alloc(2);
  return DirectApply{0, a.alpha, a.apply ? 1 : 0, a.want_norm ? 1 : 0, m.w64.p, m.w32.p, m.g64.p,
                     m.finite.p, m.scal.p, m.gbar.p};
}

// Returns true when the update was applied in the kernel (one row block).
bool launch_csc_seg(Dataset& ds, Model& m, const StepArgs& a) {
  const int nt = seg_threads();
  DirectApply da{};
  if (ds.csc_nblk == 1)
    da = DirectApply{1, a.alpha, a.apply ? 1 : 0, a.want_norm ? 1 : 0, m.w64.p, m.w32.p, m.g64.p,
                     m.finite.p, m.scal.p, nullptr};
  else
    da = grid_apply_args(m, a);
  const bool applied = da.on || da.gbar;
  if (nt >= 1024 && launch_csc_seg_N<1024>(ds, m, da)) return applied;
  if (nt >= 768 && launch_csc_seg_N<768>(ds, m, da)) return applied;
  if (!launch_csc_seg_N<512>(ds, m, da)) throw CudaError("csc_seg: no launchable configuration");
  return applied;
}

void launch_apply_partials(Dataset& ds, Model& m, const StepArgs& a) {
  Ctx& c = *ds.ctx;
  // One coordinate per thread: each thread's 16-deep load batch is the only
  // memory parallelism this d-sized pass has.
  const unsigned grid = grid_for(c, 256, ds.d, 64);
  prof_begin(c, "apply_partials_kernel");
  apply_partials_kernel<<<grid, 256, 0, c.stream>>>(ds.d, ds.csc_nblk, m.partials.p, a.alpha,
                                                    a.apply ? 1 : 0, a.want_norm ? 1 : 0, m.w64.p,
                                                    m.w32.p, m.g64.p, m.finite.p, m.scal.p);
  launched(c, "apply_partials_kernel");
}

template <int G, int TASK>
void launch_csr_batch_G(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb, bool check) {
  Ctx& c = *ds.ctx;
  // One row group per warp: each row is a chain of dependent loads (id ->
  // extent -> slots -> model gather), so rows are spread over as many warps
  // as the batch has, not walked two deep (rcv1 B = 4096: 24.9 -> see
  // profiles/round1_sync_sweep.jsonl).
  const unsigned grid = grid_for(c, 8ull * (32 / G), nb, 16);
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
    // K2t (segmented warp stream; model in SMEM when it fits, SGDB_SEG_SMEM=0
    // gathers it through L1 instead). SGDB_SEG=0 selects the lane-group
    // kernels measured before it (K2v for 32 lanes, else K2p).
    static const bool seg = [] {
      const char* e = std::getenv("SGDB_SEG");
      return !e || std::atoi(e) != 0;
    }();
    static const bool seg_smem = [] {
      const char* e = std::getenv("SGDB_SEG_SMEM");
      return !e || std::atoi(e) != 0;
    }();
    const bool fits = round_up16(ds.d * sizeof(float)) + 8192 <= ds.ctx->max_smem_optin;
    if (seg) {
      if (a.task == kTaskLR) launch_csr_coef_seg<kTaskLR>(ds, m, fits && seg_smem);
      else launch_csr_coef_seg<kTaskSVM>(ds, m, fits && seg_smem);
    } else if (g == 32) {
      if (a.task == kTaskLR) launch_csr_coef_vec<kTaskLR>(ds, m);
      else launch_csr_coef_vec<kTaskSVM>(ds, m);
    } else {
      dispatch_G(g, [&]<int G>() {
        if (a.task == kTaskLR) launch_csr_coef_pipe_G<G, kTaskLR, false>(ds, m);
        else launch_csr_coef_pipe_G<G, kTaskSVM, false>(ds, m);
      });
    }
  }
  const double per_col = static_cast<double>(ds.nnz) /
                         static_cast<double>(std::max<uint64_t>(1, ds.d) * std::max(1u, ds.csc_nblk));
  // Column segments: narrow groups amortise the per-column reduction over
  // more columns per warp (measured: rcv1 8 lanes, news20/real-sim 4).
  const int gc = per_col <= 16.0 ? 4 : (per_col <= 128.0 ? 8 : 16);
  static const bool csc_vec = [] {
    const char* e = std::getenv("SGDB_CSC_VEC");
    return !e || std::atoi(e) != 0;
  }();
  // SGDB_CSC: 0 = K3, 1 = K3v, 2 = K3t, unset = by column length. Measured
  // (profiles/round1_sync_kernels_ab.jsonl): the segmented stream wins when
  // columns are a few slots long (news20: 72 vs 84 us), K3v with 8-lane
  // groups when they run to tens of slots (rcv1: 82 vs 125-143 us).
  static const int csc_mode = [] {
    const char* e = std::getenv("SGDB_CSC");
    if (e) return std::atoi(e);
    const char* v = std::getenv("SGDB_CSC_VEC");
    return v && std::atoi(v) == 0 ? 0 : -1;
  }();
  const bool aligned = ds.csc_rb % 4 == 0;
  const int mode = !aligned ? 0 : (csc_mode >= 0 ? csc_mode : (per_col < 12.0 ? 2 : 1));
  bool applied = false;
  if (mode == 2) {
    applied = launch_csc_seg(ds, m, a);
  } else if (mode == 1) {
    // 4-slot windows: one window per lane group covers 4G slots of a column.
    const int gv = per_col <= 24.0 ? 4 : 8;
    const DirectApply da = grid_apply_args(m, a);
    dispatch_G(env_lanes("SGDB_COL_LANES", gv), [&]<int G>() { launch_csc_vec_G<G>(ds, m, da); });
    applied = da.gbar != nullptr;
  } else {
    dispatch_G(env_lanes("SGDB_COL_LANES", gc), [&]<int G>() { launch_csc_block_G<G>(ds, m); });
  }
  if (!applied) launch_apply_partials(ds, m, a);
}

namespace {
// Slots per lane per chunk (CH = G * U): 4 by default (measured against 2 / 8
// / 16, profiles/round1_minibatch_chunk_u_ab.jsonl); SGDB_BATCH_CHUNK_U selects.
int chunk_u() {
  static const int u = [] {
    const char* e = std::getenv("SGDB_BATCH_CHUNK_U");
    const int v = e ? std::atoi(e) : 4;
    return v == 2 || v == 8 || v == 16 ? v : 4;
  }();
  return u;
}

int batch_lanes(const Dataset& ds) {
  return env_lanes("SGDB_BATCH_LANES",
                   lanes_for(ds.n ? static_cast<double>(ds.nnz) / static_cast<double>(ds.n) : 1.0));
}

bool chunked_batches() {
  static const bool on = [] {
    const char* e = std::getenv("SGDB_BATCH_CHUNKS");  // 0 = one lane group per row (K3b)
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

bool mb_prefetch() {
  static const bool on = [] {  // SGDB_BATCH_PREFETCH=0: no L2 prefetch of the next step
    const char* e = std::getenv("SGDB_BATCH_PREFETCH");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

template <int G, int TASK, int U>
void launch_mb_chunks_U(Dataset& ds, Model& m, uint64_t lo, uint64_t nb, bool check) {
  Ctx& c = *ds.ctx;
  constexpr int RW = 32 / G;
  // Chunks of one step: the rows plus one per CH slots of their mean length.
  const double avg = ds.n ? static_cast<double>(ds.nnz) / static_cast<double>(ds.n) : 1.0;
  const uint64_t est = nb + static_cast<uint64_t>(nb * avg / (G * U));
  const unsigned grid = grid_for(c, 8ull * RW, est, 16);
  const uint64_t hi = lo + nb;
  prof_begin(c, "mb_margin_kernel");
  mb_margin_kernel<G, U><<<grid, 256, 0, c.stream>>>(
      ds.val.p, ds.idx.p, ds.rowptr.p, ds.mb_ids, ds.mb_off.p, ds.mb_meta.p, ds.mb_cap, lo, hi,
      ds.row_base, m.w32.p, ds.mb_z.p, m.finite.p, check ? 1 : 0);
  launched(c, "mb_margin_kernel");
  prof_begin(c, "mb_scatter_kernel");
  mb_scatter_kernel<G, U, TASK><<<grid, 256, 0, c.stream>>>(
      ds.val.p, ds.idx.p, ds.rowptr.p, ds.labels.p, ds.mb_ids, ds.mb_off.p, ds.mb_meta.p,
      ds.mb_cap, lo, hi, ds.row_base, ds.mb_z.p, m.g64.p, m.finite.p, check ? 1 : 0,
      mb_prefetch() && hi < ds.mb_count ? 1 : 0, ds.mb_count);
  launched(c, "mb_scatter_kernel");
}

template <int G, int TASK>
void launch_mb_chunks(Dataset& ds, Model& m, uint64_t lo, uint64_t nb, bool check) {
  switch (chunk_u()) {
    case 2: launch_mb_chunks_U<G, TASK, 2>(ds, m, lo, nb, check); break;
    case 8: launch_mb_chunks_U<G, TASK, 8>(ds, m, lo, nb, check); break;
    case 16: launch_mb_chunks_U<G, TASK, 16>(ds, m, lo, nb, check); break;
    default: launch_mb_chunks_U<G, TASK, 4>(ds, m, lo, nb, check); break;
  }
}
}  // namespace

void csr_batch_plan(Dataset& ds, const uint32_t* ids, uint64_t count, uint64_t max_step) {
  if (!chunked_batches() || count == 0) return;
  Ctx& c = *ds.ctx;
  const uint32_t ch = static_cast<uint32_t>(batch_lanes(ds) * chunk_u());
  const uint64_t per_row = ds.max_row ? (ds.max_row + ch - 1) / ch : 1;
  const uint64_t zcap = std::min(max_step, count) * per_row;
  // Chunk table: every chunk of a permutation order (sum over the local rows
  // of ceil(len / ch) <= nnz / ch + n); larger plans (repeated ids) search.
  const uint64_t cap = std::min<uint64_t>(count * per_row, ds.nnz / ch + ds.n + 1);
  const bool grow = !ds.mb_cnt.p || ds.mb_cnt.n < count + 1 || ds.mb_z.n < zcap ||
                    ds.mb_meta.n < cap;
  ds.mb_cnt.alloc(count + 1);
  ds.mb_off.alloc(count + 1);
  ds.mb_z.alloc(std::max<uint64_t>(1, zcap));
  ds.mb_meta.alloc(std::max<uint64_t>(1, cap));
  ds.mb_cap = cap;
  size_t bytes = 0;
  check(cub::DeviceScan::ExclusiveSum(nullptr, bytes, ds.mb_cnt.p, ds.mb_off.p,
                                      static_cast<int64_t>(count + 1), c.stream),
        "cub scan size");
  if (bytes > ds.mb_tmp.n) ds.mb_tmp.alloc(bytes);
  // New buffers invalidate epoch graphs captured against the old ones.
  if (grow) ds.uid = next_dataset_uid();
  const unsigned grid = grid_for(c, 256, count + 1, 8);
  prof_begin(c, "mb_count_kernel");
  mb_count_kernel<<<grid, 256, 0, c.stream>>>(ids, count, ds.rowptr.p, ds.n, ds.row_base, ch,
                                              ds.mb_cnt.p);
  launched(c, "mb_count_kernel");
  bytes = ds.mb_tmp.n;
  check(cub::DeviceScan::ExclusiveSum(ds.mb_tmp.p, bytes, ds.mb_cnt.p, ds.mb_off.p,
                                      static_cast<int64_t>(count + 1), c.stream),
        "cub scan");
  prof_begin(c, "mb_fill_kernel");
  mb_fill_kernel<<<grid, 256, 0, c.stream>>>(ids, count, ds.rowptr.p, ds.row_base, ch, ds.mb_off.p,
                                             ds.mb_meta.p, cap);
  launched(c, "mb_fill_kernel");
  ds.mb_ids = ids;
  ds.mb_count = count;
  ds.mb_ch = ch;
}

void csr_batch_step(Dataset& ds, Model& m, const uint32_t* ids, uint64_t nb, const StepArgs& a) {
  const int g = batch_lanes(ds);
  if (chunked_batches()) {
    if (!(ds.mb_ids && ids >= ds.mb_ids && ids + nb <= ds.mb_ids + ds.mb_count &&
          ds.mb_ch == static_cast<uint32_t>(g * chunk_u())))
      csr_batch_plan(ds, ids, nb, nb);
    const uint64_t lo = static_cast<uint64_t>(ids - ds.mb_ids);
    dispatch_G(g, [&]<int G>() {
      if (a.task == kTaskLR) launch_mb_chunks<G, kTaskLR>(ds, m, lo, nb, a.apply);
      else launch_mb_chunks<G, kTaskSVM>(ds, m, lo, nb, a.apply);
    });
  } else {
    dispatch_G(g, [&]<int G>() {
      if (a.task == kTaskLR) launch_csr_batch_G<G, kTaskLR>(ds, m, ids, nb, a.apply);
      else launch_csr_batch_G<G, kTaskSVM>(ds, m, ids, nb, a.apply);
    });
  }
  if (a.apply) apply_update(m, a.alpha, a.want_norm, a.alpha_dev);
}

void apply_update(Model& m, double alpha, bool want_norm, const double* alpha_dev) {
  Ctx& c = *m.ctx;
  // One coordinate per thread (each iteration is a dependent load chain).
  const unsigned grid = grid_for(c, 256, m.d, 64);
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
