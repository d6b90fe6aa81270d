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
// generation word). Thread 0 arrives with a release-add, which orders the
// block's global writes (the gradient REDs, ordered before it by the
// __syncthreads) before the arrival.
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // Release-add: the CTA's REDs (ordered before it by the barrier; release
    // is cumulative) are visible to whoever acquires the count — no separate
    // full fence.
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
      if (v >= target) break;
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

// W64: the model is read from the fp64 master, rounded to fp32 at the load
// (the value w32 would hold), for epochs whose steps update w64 directly.
template <int G, int U, bool W64>
__global__ void __launch_bounds__(256) mb_margin_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const uint32_t* __restrict__ ids,
    const uint32_t* __restrict__ off, const uint4* __restrict__ meta, uint64_t cap, uint64_t lo,
    uint64_t hi, uint64_t row_base, const float* __restrict__ w32, const double* __restrict__ w64,
    float* __restrict__ zpart, const int* finite, int check_finite) {
  // PDL: the chunk table and the slots are fixed for the epoch, so they load
  // while the previous step's update drains; the model is read after the wait.
  pdl_launch_dependents();
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint32_t c0 = __ldg(off + lo), c1 = __ldg(off + hi);
  const bool direct = c1 <= cap;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  bool waited = false;
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
    if (!waited) {
      pdl_wait();
      waited = true;
      if (check_finite && *finite == 0) return;
    }
    float z = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = b + lg + u * G < e;
      const float wv = W64 ? (ok ? static_cast<float>(w64[jv[u]]) : 0.f) : (ok ? w32[jv[u]] : 0.f);
      z = fmaf(xv[u], wv, z);
    }
    z = group_sum<G>(z);
    if (valid && lg == 0) zpart[q - c0] = z;
  }
}

// DIRECT: each step's update goes straight into the fp64 master
// (w64 -= alpha * c * x with red.add.f64; the step size from alpha_dev when
// set) and the finite flag follows the products, so no gradient buffer and no
// apply launch are needed; otherwise c * x is accumulated into g64.
template <int G, int U, int TASK, bool DIRECT>
__global__ void __launch_bounds__(256) mb_scatter_kernel(
    const float* __restrict__ val, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ rowptr, const float* __restrict__ y,
    const uint32_t* __restrict__ ids, const uint32_t* __restrict__ off,
    const uint4* __restrict__ meta, uint64_t cap, uint64_t lo, uint64_t hi, uint64_t row_base,
    const float* __restrict__ zpart, double* g64, int* finite, int check_finite,
    int prefetch_next, uint64_t count, double alpha_in, const double* alpha_dev) {
  pdl_launch_dependents();
  constexpr int RW = 32 / G;
  const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
  const uint32_t c0 = __ldg(off + lo), c1 = __ldg(off + hi);
  const bool direct = c1 <= cap;
  const uint64_t total = prefetch_next ? __ldg(off + count) : 0;  // chunks of the whole plan
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  bool waited = false;
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
    if (!waited) {  // the chunk margins (and the zeroed gradient) come from the predecessors
      pdl_wait();
      waited = true;
      if (check_finite && *finite == 0) return;
    }
    float z = 0.f;
    for (uint32_t k = z0; k < z1; ++k) z += __ldcg(zpart + k);  // chunk order
    const float c = coef_f<TASK>(z, __ldg(y + r.row));
    if (c != 0.f) {
      if (DIRECT) {
        const double alpha = alpha_dev ? *alpha_dev : alpha_in;
        bool bad = false;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (r.b + lg + u * G < r.e) {
            const double gx = static_cast<double>(c * xv[u]);
            bad = bad || !isfinite(gx);
            atomicAdd(&g64[jv[u]], -alpha * gx);  // g64 = the master here
          }
        if (bad) *finite = 0;
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (r.b + lg + u * G < r.e) atomicAdd(&g64[jv[u]], static_cast<double>(c * xv[u]));
      }
    }
    if (prefetch_next && total <= cap) {
      // Pull the slots of the chunk at the same position of the next step
      // into L2, so that step's margin pass reads them from L2, not HBM.
      const uint64_t qn = q + (c1 - c0);
      if (qn < total && lg < 16) {  // total <= cap: table entries below it are written
        const uint4 mn = __ldg(meta + qn);
        // 128-byte lines spanned by slots [mn.x, mn.y), counted from the line
        // holding mn.x (a chunk rarely starts on a line boundary).
        const uint32_t lines = min(((mn.x & 31u) + (mn.y - mn.x) + 31) / 32, (U * G) / 32u + 1);
        const char* base = lg < 8 ? reinterpret_cast<const char*>(idx + (mn.x & ~31u))
                                  : reinterpret_cast<const char*>(val + (mn.x & ~31u));
        for (uint32_t l = lg & 7; l < lines; l += 8)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(base + 128ull * l));
      }
    }
  }
}

__global__ void apply_kernel(uint64_t d, double alpha_in, const double* alpha_dev, double* w64,
                             float* w32, double* g64, int* finite, double* norm2, int want_norm) {
  pdl_launch_dependents();
  pdl_wait();  // g (and w) come from the step's kernels
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

__global__ void w32_from_w64_kernel(uint64_t d, const double* w64, float* w32) {
  pdl_wait();
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x)
    w32[j] = static_cast<float>(w64[j]);
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

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while its predecessor on the stream drains (it calls pdl_wait before
// touching the predecessor's results). Captured into CUDA graphs as
// programmatic edges.
template <class... KArgs, class... Args>
void launch_pdl(Ctx& c, void (*kern)(KArgs...), unsigned grid, unsigned block, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  check(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "cudaLaunchKernelEx");
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
  // Tile bytes (profiles/round2_dense_tile_sweep.jsonl): 96 KB (two stages)
  // for rows of >= 1 KB — C5's 25M x 1000 shard 14.8 -> 13.5 ms — and 64 KB
  // (three stages) for short rows (covtype 34.8 -> 32.8 us).
  const int tile_bytes = row_bytes >= 1024 ? 98304 : 65536;
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
  if (d <= 32) fn.template operator()<4, 8>();
  else if (d <= 56) fn.template operator()<4, 14>();
  else if (d <= 64) fn.template operator()<8, 8>();
  else if (d <= 128) fn.template operator()<16, 8>();
  else if (d <= 256) fn.template operator()<32, 8>();
  else if (d <= 512) fn.template operator()<32, 16>();
  else if (d <= 1024) fn.template operator()<32, 32>();
  else throw Unsupported("dense kernels handle d <= 1024 (wider data is stored as CSR)");
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
  bool handled = true;
  dispatch_dense(ds.d, [&]<int L, int F>() {
    // Large batches of wide rows stream better through the per-step kernels
    // (measured: d = 1000, B = 65536: 72 vs 86 us per step).
    if (F > 16 && B > 16384) {
      handled = false;
      return;
    }
    // Measured (scripts/minibatch_time.py): 16 warps per CTA for F <= 8, else
    // 8 (only these instances are built: wider CTAs at F = 32 spill).
    constexpr int W = F <= 8 ? 16 : 8;
    if (task == kTaskLR) launch_dense_epoch_LFW<L, F, kTaskLR, W>(ds, m, B, alpha);
    else launch_dense_epoch_LFW<L, F, kTaskSVM, W>(ds, m, B, alpha);
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

namespace {
// Slots per lane per chunk (CH = G * U): 4 (measured against 2 / 8 / 16,
// profiles/round1_minibatch_chunk_u_ab.jsonl).
constexpr int kChunkU = 4;

int batch_lanes(const Dataset& ds) {
  return lanes_for(ds.n ? static_cast<double>(ds.nnz) / static_cast<double>(ds.n) : 1.0);
}

template <int G, int TASK, int U>
void launch_mb_chunks_U(Dataset& ds, Model& m, uint64_t lo, uint64_t nb, bool check, const StepArgs& a) {
  Ctx& c = *ds.ctx;
  constexpr int RW = 32 / G;
  // Chunks of one step: the rows plus one per CH slots of their mean length.
  const double avg = ds.n ? static_cast<double>(ds.nnz) / static_cast<double>(ds.n) : 1.0;
  const uint64_t est = nb + static_cast<uint64_t>(nb * avg / (G * U));
  const unsigned grid = grid_for(c, 8ull * RW, est, 16);
  const uint64_t hi = lo + nb;
  auto go = [&]<bool D>() {
    prof_begin(c, "mb_margin_kernel");
    launch_pdl(c, mb_margin_kernel<G, U, D>, grid, 256, ds.val.p, ds.idx.p, ds.rowptr.p,
               static_cast<const uint32_t*>(ds.mb_ids), static_cast<const uint32_t*>(ds.mb_off.p),
               static_cast<const uint4*>(ds.mb_meta.p), ds.mb_cap, lo, hi, ds.row_base,
               static_cast<const float*>(m.w32.p), static_cast<const double*>(m.w64.p), ds.mb_z.p,
               static_cast<const int*>(m.finite.p), check ? 1 : 0);
    launched(c, "mb_margin_kernel");
    prof_begin(c, "mb_scatter_kernel");
    launch_pdl(c, mb_scatter_kernel<G, U, TASK, D>, grid, 256, ds.val.p, ds.idx.p, ds.rowptr.p,
               static_cast<const float*>(ds.labels.p), static_cast<const uint32_t*>(ds.mb_ids),
               static_cast<const uint32_t*>(ds.mb_off.p), static_cast<const uint4*>(ds.mb_meta.p),
               ds.mb_cap, lo, hi, ds.row_base, static_cast<const float*>(ds.mb_z.p),
               D ? m.w64.p : m.g64.p, m.finite.p, check ? 1 : 0, hi < ds.mb_count ? 1 : 0,
               ds.mb_count, a.alpha, a.alpha_dev);
    launched(c, "mb_scatter_kernel");
  };
  if (a.direct) go.template operator()<true>();
  else go.template operator()<false>();
}

template <int G, int TASK>
void launch_mb_chunks(Dataset& ds, Model& m, uint64_t lo, uint64_t nb, bool check, const StepArgs& a) {
  launch_mb_chunks_U<G, TASK, kChunkU>(ds, m, lo, nb, check, a);
}
}  // namespace

void csr_batch_plan(Dataset& ds, const uint32_t* ids, uint64_t count, uint64_t max_step) {
  if (count == 0) return;
  Ctx& c = *ds.ctx;
  const uint32_t ch = static_cast<uint32_t>(batch_lanes(ds) * kChunkU);
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
  if (!(ds.mb_ids && ids >= ds.mb_ids && ids + nb <= ds.mb_ids + ds.mb_count &&
        ds.mb_ch == static_cast<uint32_t>(g * kChunkU)))
    csr_batch_plan(ds, ids, nb, nb);
  const uint64_t lo = static_cast<uint64_t>(ids - ds.mb_ids);
  dispatch_G(g, [&]<int G>() {
    if (a.task == kTaskLR) launch_mb_chunks<G, kTaskLR>(ds, m, lo, nb, a.apply, a);
    else launch_mb_chunks<G, kTaskSVM>(ds, m, lo, nb, a.apply, a);
  });
  if (a.apply && !a.direct) apply_update(m, a.alpha, a.want_norm, a.alpha_dev);
}

void apply_update(Model& m, double alpha, bool want_norm, const double* alpha_dev) {
  Ctx& c = *m.ctx;
  // One coordinate per thread (each iteration is a dependent load chain).
  const unsigned grid = grid_for(c, 256, m.d, 64);
  prof_begin(c, "apply_kernel");
  launch_pdl(c, apply_kernel, grid, 256, m.d, alpha, alpha_dev, m.w64.p, m.w32.p, m.g64.p, m.finite.p,
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

void sync_w32_from_w64(Model& m) {
  Ctx& c = *m.ctx;
  const unsigned grid = grid_for(c, 256ull * 4, m.d, 8);
  prof_begin(c, "w32_from_w64_kernel");
  launch_pdl(c, w32_from_w64_kernel, grid, 256, m.d, static_cast<const double*>(m.w64.p), m.w32.p);
  launched(c, "w32_from_w64_kernel");
}

void sync_w64_from_w32(Model& m) {
  Ctx& c = *m.ctx;
  const unsigned grid = grid_for(c, 256ull * 4, m.d, 8);
  prof_begin(c, "w64_from_w32_kernel");
  w64_from_w32_kernel<<<grid, 256, 0, c.stream>>>(m.d, m.w32.p, m.w64.p);
  launched(c, "w64_from_w32_kernel");
}

}  // namespace sgdb::dev
