// Asynchronous Hogwild kernels (sm_100a) — the paper's accelerator
// contribution (§5 "do in parallel" Alg. 3).
//
// Replaces hogwild::Instance::worker_loop + process_examples
// (proj/src/async_engine.cpp:178-195, :372-396) and the replica prepare /
// merge (:293-331, merge_models :133-156). A reference "worker" walking its
// assign() list (proj/src/dataset.cpp:470-503) is a group of G lanes here
// (G = 32: one warp per example); the group gathers the model at the
// example's support, reduces the margin with shuffles, and writes the update
// back without locks. Lost updates between workers are allowed by design
// (async_engine.hpp:49-52); within a group every lane owns distinct
// coordinates.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "device.hpp"

namespace sgdb::dev {

namespace {

constexpr int kKindDenseRow = 0;  // row-major dense, idx implicit
constexpr int kKindCsr = 1;       // CSR rows
constexpr int kKindDenseCol = 2;  // column-major dense (stride n)
constexpr int kKindPaddedCol = 3; // slot-major padded (stride n, sentinel d)

constexpr int kScopeGlobalRep = 1;// replicas in global memory, replica = worker / gs
constexpr int kScopeSharedAtomic = 2;      // one model, red.global.add, slice-spread layout
constexpr int kScopeSharedAtomicFlat = 3;  // one model, red.global.add, contiguous layout
constexpr int kScopeGlobalRepAtomic = 4;   // replicas in global memory, red.global.add
constexpr uint32_t kSpread = 64;           // floats between coordinates (256 B)

struct HogParams {
  const float* val;
  const uint32_t* idx;
  const uint32_t* rowptr;
  const float* y;
  uint64_t n;
  uint64_t d;
  uint64_t pw;
  uint64_t T;
  uint64_t k;
  int rr;
  uint64_t gs;
  int offsets;
  float* model;
  uint64_t ld;
  float alpha;
  uint32_t ms;       // kernel scope: float stride between model coordinates in global
  uint32_t seg, nseg;  // this launch runs list positions [total*seg/nseg, total*(seg+1)/nseg)
};

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if (G == 32) return 0xffffffffu;
  const unsigned lane = threadIdx.x & 31;
  return ((1u << G) - 1u) << (lane & ~(G - 1u));
}

template <int G>
__device__ __forceinline__ float group_sum_m(float v, unsigned mask) {
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off);
  return v;
}

// Model access policies. `add(j, delta)` is the reference's
// m.store(j, m.load(j) - alpha*(c*x)) with delta = -(alpha*(c*x)), which is the
// same IEEE result (a - b == a + (-b)).
struct GlobalModel {  // plain load / store: lost updates allowed (Hogwild)
  float* m;
  uint32_t ms;
  __device__ GlobalModel at(uint64_t) const { return *this; }
  __device__ float load(uint32_t j) const { return ld_model(m + uint64_t(j) * ms); }
  __device__ void add(uint32_t j, float delta) const {
    st_model(m + uint64_t(j) * ms, ld_model(m + uint64_t(j) * ms) + delta);
  }
};
// red.global.add.f32: every update lands (no lost updates). MS = float stride
// between coordinates (64 = the slice-spread layout, a compile-time constant
// so the gather address is a shift).
template <uint32_t MS>
struct GlobalAtomicModel {
  float* m;
  __device__ GlobalAtomicModel at(uint64_t) const { return *this; }
  __device__ float load(uint32_t j) const { return ld_model(m + uint64_t(j) * MS); }
  __device__ void add(uint32_t j, float delta) const { atomicAdd(m + uint64_t(j) * MS, delta); }
};
struct SmemModel {  // block-scope replica in shared memory, plain RMW
  volatile float* m;
  __device__ SmemModel at(uint64_t) const { return *this; }
  __device__ float load(uint64_t j) const { return m[j]; }
  __device__ void add(uint64_t j, float delta) const { m[j] = m[j] + delta; }
};
// ---- one worker: its assign() list, a 2-stage prefetch pipeline, and the
// per-example body of process_examples (async_engine.cpp:178-195) ----------

constexpr int kU = 4;  // slots per lane per batch (U loads / gathers in flight)

__device__ __forceinline__ WorkerList worker_list(const HogParams& p, uint64_t w) {
  return assign_list(p.n, p.T, p.k, p.rr != 0, w);
}
__device__ __forceinline__ uint32_t list_at(const HogParams& p, const WorkerList& l, uint32_t i) {
  return assign_at(p.n, l, i);
}

// Example e's slots. Contiguous kinds (CSR, dense row): slots [b, bend).
// Strided kinds (dense col, padded col): base b = e, bend = slot count.
struct Row {
  uint32_t e;
  uint32_t b, bend;  // CSR offsets (< 2^32, enforced at upload) or strided base/count
  float y;           // label, prefetched with the extent
};
template <int KIND>
__device__ __forceinline__ Row make_row(const HogParams& p, uint32_t e) {
  const float y = __ldg(p.y + e);  // loads issued here are consumed iterations later
  if (KIND == kKindCsr) return {e, p.rowptr[e], p.rowptr[e + 1], y};
  if (KIND == kKindDenseRow) return {e, 0u, static_cast<uint32_t>(p.d), y};  // base = e*d
  if (KIND == kKindDenseCol) return {e, e, static_cast<uint32_t>(p.d), y};
  return {e, e, static_cast<uint32_t>(p.pw), y};
}
template <int KIND>
__device__ __forceinline__ uint32_t row_len(const Row& r) {
  return KIND == kKindCsr ? r.bend - r.b : r.bend;
}
template <int KIND>
__device__ __forceinline__ uint64_t row_base(const HogParams& p, const Row& r) {
  return KIND == kKindDenseRow ? uint64_t(r.e) * p.d : uint64_t(r.b);
}
template <int KIND>
__device__ __forceinline__ uint32_t slot_index(const HogParams& p, const Row& r, uint32_t s) {
  if (KIND == kKindCsr) return __ldg(p.idx + r.b + s);
  if (KIND == kKindPaddedCol) return __ldg(p.idx + r.b + uint64_t(s) * p.n);
  return s;
}
template <int KIND>
__device__ __forceinline__ float slot_value(const HogParams& p, const Row& r, uint32_t s) {
  if (KIND == kKindCsr) return __ldg(p.val + r.b + s);
  if (KIND == kKindDenseRow) return __ldg(p.val + row_base<KIND>(p, r) + s);
  return __ldg(p.val + r.b + uint64_t(s) * p.n);
}

struct Batch {
  uint32_t j[kU];
  float x[kU];
};
// Lane lg's U slots s0, s0+G, ... of row r (zeros past the end). Slots
// 1..U-1 sit behind a group-uniform branch (s0 - lg + G < len), so rows that
// fit one slot per lane — most rows of the sparse configs — do not issue
// their loads at all.
template <int G, int KIND>
__device__ __forceinline__ Batch load_batch(const HogParams& p, const Row& r, uint32_t s0,
                                            uint32_t len, int lg) {
  Batch bt;
  {
    const bool ok = s0 < len;
    bt.j[0] = ok ? slot_index<KIND>(p, r, s0) : 0u;
    bt.x[0] = ok ? slot_value<KIND>(p, r, s0) : 0.f;
  }
#pragma unroll
  for (int u = 1; u < kU; ++u) {
    bt.j[u] = 0u;
    bt.x[u] = 0.f;
  }
  if (s0 - lg + G < len) {
#pragma unroll
    for (int u = 1; u < kU; ++u) {
      const uint32_t s = s0 + u * G;
      const bool ok = s < len;
      bt.j[u] = ok ? slot_index<KIND>(p, r, s) : 0u;
      bt.x[u] = ok ? slot_value<KIND>(p, r, s) : 0.f;
    }
  }
  return bt;
}

// One example: margin over every slot (padded sentinels read the guard slot
// w[d] == 0), coefficient (glm.cpp:30-34), lock-free update. `first` holds
// this lane's first batch, prefetched by the worker loop.
template <int G, int TASK, int KIND, class M, bool LONG = false>
__device__ __forceinline__ void process_example(const HogParams& p, const M& m, const Row& r,
                                                const Batch& first, uint64_t wid, int lg,
                                                unsigned mask) {
  const uint32_t len = row_len<KIND>(r);
  // A worker is sequential (Alg. 3): the lanes of the group must see each
  // other's updates of the previous example before reading the model again;
  // under independent thread scheduling a lane with fewer slots could
  // otherwise run ahead into this dot product.
  __syncwarp(mask);
  const bool wide = G < len;  // group-uniform: slots 1..U-1 of the first batch in use
  float z = 0.f;
  {
    float mv[kU];
    mv[0] = lg < static_cast<int>(len) ? m.load(first.j[0]) : 0.f;
    z = first.x[0] * mv[0];
    if (wide) {
#pragma unroll
      for (int u = 1; u < kU; ++u) mv[u] = (lg + u * G < len) ? m.load(first.j[u]) : 0.f;
#pragma unroll
      for (int u = 1; u < kU; ++u) z = fmaf(first.x[u], mv[u], z);
    }
  }
  // Remaining slots. LONG (datasets whose rows run to thousands of slots —
  // news20's Pareto tail reaches 9,100, all walked by one worker): two
  // batches per trip, so each dependent round trip carries 2U loads and 2U
  // gathers per lane (same summation order). Off by default: the second
  // batch costs ~16 registers, i.e. a quarter of the resident workers.
  for (uint32_t s0 = lg + G * kU; s0 < len; s0 += (LONG ? 2 : 1) * G * kU) {
    const Batch bt = load_batch<G, KIND>(p, r, s0, len, lg);
    const bool two = LONG && s0 - lg + G * kU < len;  // group-uniform
    Batch b2{};
    if (two) b2 = load_batch<G, KIND>(p, r, s0 + G * kU, len, lg);
    float mv[kU], mv2[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) mv[u] = (s0 + u * G < len) ? m.load(bt.j[u]) : 0.f;
    if (two) {
#pragma unroll
      for (int u = 0; u < kU; ++u) mv2[u] = (s0 + (kU + u) * G < len) ? m.load(b2.j[u]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) z = fmaf(bt.x[u], mv[u], z);
    if (two) {
#pragma unroll
      for (int u = 0; u < kU; ++u) z = fmaf(b2.x[u], mv2[u], z);
    }
  }
  z = group_sum_m<G>(z, mask);
  const float c = coef_f<TASK>(z, r.y);
  if (c == 0.f || len == 0) return;  // w - alpha*(0*x) == w: skip the no-op stores
  const float ac = p.alpha;
  if (G == 1 && p.offsets) {
    // Circular offsets (async_engine.cpp:188-193): start at wid mod len.
    uint32_t s = static_cast<uint32_t>(wid % len);
    for (uint32_t i = 0; i < len; ++i) {
      m.add(slot_index<KIND>(p, r, s), -(ac * (c * slot_value<KIND>(p, r, s))));
      if (++s == len) s = 0;
    }
    return;
  }
  if (lg < static_cast<int>(len)) m.add(first.j[0], -(ac * (c * first.x[0])));
  if (wide) {
#pragma unroll
    for (int u = 1; u < kU; ++u)
      if (lg + u * G < len) m.add(first.j[u], -(ac * (c * first.x[u])));
  }
  for (uint32_t s0 = lg + G * kU; s0 < len; s0 += (LONG ? 2 : 1) * G * kU) {
    const Batch bt = load_batch<G, KIND>(p, r, s0, len, lg);
    const bool two = LONG && s0 - lg + G * kU < len;  // group-uniform
    Batch b2{};
    if (two) b2 = load_batch<G, KIND>(p, r, s0 + G * kU, len, lg);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (s0 + u * G < len) m.add(bt.j[u], -(ac * (c * bt.x[u])));
    if (two) {
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (s0 + (kU + u) * G < len) m.add(b2.j[u], -(ac * (c * b2.x[u])));
    }
  }
}

// Worker w walks its list with a 2-stage software pipeline: while example i
// runs, the row extent of example i+2 and the first slot batch of example
// i+1 are already in flight (data only — the model is always read fresh, so
// the single-worker schedule is exactly sequential Alg. 3).
template <int G, int TASK, int KIND, class M, bool LONG = false>
__device__ __forceinline__ void run_worker(const HogParams& p, const M& m, uint64_t w, int lg,
                                           unsigned mask) {
  const WorkerList l = worker_list(p, w);
  // Segment of the list (multi-GPU replicas averaged every segment; 0 of 1 = epoch).
  const uint32_t lo = static_cast<uint32_t>(uint64_t(l.total) * p.seg / p.nseg);
  const uint32_t hi = static_cast<uint32_t>(uint64_t(l.total) * (p.seg + 1) / p.nseg);
  if (lo >= hi) return;
  Row cur = make_row<KIND>(p, list_at(p, l, lo));
  Row nxt = lo + 1 < hi ? make_row<KIND>(p, list_at(p, l, lo + 1)) : cur;
  Batch bcur = load_batch<G, KIND>(p, cur, lg, row_len<KIND>(cur), lg);
  for (uint32_t i = lo; i < hi; ++i) {
    Batch bnxt = bcur;
    Row after = nxt;
    if (i + 1 < hi) bnxt = load_batch<G, KIND>(p, nxt, lg, row_len<KIND>(nxt), lg);
    if (i + 2 < hi) after = make_row<KIND>(p, list_at(p, l, i + 2));
    process_example<G, TASK, KIND, decltype(m.at(cur.e)), LONG>(p, m.at(cur.e), cur, bcur, w, lg, mask);
    cur = nxt;
    bcur = bnxt;
    nxt = after;
  }
}

// K5x: example-scope replication (ModelReplication::Example,
// async_engine.cpp:346-370). Every example owns a replica of the model
// restricted to its support, stored at its slots (rep[s] for s in the row's
// CSR range). The first worker to reach an example in an epoch claims it and
// copies the shared model into the replica (ensure_replica, :333-344; the
// claim is an atomicExch of the epoch number, readiness a release/acquire
// epoch word); the example's margin and update use only its replica; when a
// worker has walked its list it stores the replicas of the examples it
// processed into the shared model (plain stores, last writer wins, :365-369).
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int G, int TASK>
__global__ void __launch_bounds__(256) hogwild_example_kernel(HogParams p, float* rep,
                                                              unsigned* claim, unsigned* ready,
                                                              unsigned epoch) {
  const int lg = threadIdx.x % G;
  const unsigned mask = group_mask<G>();
  const int leader = (threadIdx.x & 31) & ~(G - 1);
  const uint64_t hg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const uint64_t HG = ((uint64_t)gridDim.x * blockDim.x) / G;
  for (uint64_t w = hg; w < p.T; w += HG) {
    const WorkerList l = worker_list(p, w);
    const uint32_t lo = static_cast<uint32_t>(uint64_t(l.total) * p.seg / p.nseg);
    const uint32_t hi = static_cast<uint32_t>(uint64_t(l.total) * (p.seg + 1) / p.nseg);
    for (uint32_t i = lo; i < hi; ++i) {
      const uint32_t e = list_at(p, l, i);
      const uint32_t b = __ldg(p.rowptr + e), en = __ldg(p.rowptr + e + 1);
      // ensure_replica
      int role = 0;  // 0 ready, 1 initialise, 2 wait
      if (lg == 0 && ld_acquire_u32(ready + e) != epoch)
        role = atomicExch(claim + e, epoch) != epoch ? 1 : 2;
      role = __shfl_sync(mask, role, leader);
      if (role == 1) {
        for (uint32_t s = b + lg; s < en; s += G) __stcg(rep + s, ld_model(p.model + __ldg(p.idx + s)));
        __syncwarp(mask);
        if (lg == 0) {
          __threadfence();
          st_release_u32(ready + e, epoch);
        }
      } else if (role == 2) {
        if (lg == 0)
          while (ld_acquire_u32(ready + e) != epoch) __nanosleep(32);
        __syncwarp(mask);
      }
      const uint32_t len = en - b;
      if (len == 0) continue;
      float z = 0.f;
      for (uint32_t s = b + lg; s < en; s += G) z = fmaf(__ldg(p.val + s), __ldcg(rep + s), z);
      z = group_sum_m<G>(z, mask);
      const float c = coef_f<TASK>(z, __ldg(p.y + e));
      if (c != 0.f) {
        const float ac = p.alpha;
        // Circular offsets (async_engine.cpp:357-362) for one-lane workers.
        const uint32_t s0 = (G == 1 && p.offsets) ? static_cast<uint32_t>(w % len) : 0u;
        for (uint32_t t = lg; t < len; t += G) {
          uint32_t q = s0 + t;
          if (q >= len) q -= len;
          const uint32_t s = b + q;
          __stcg(rep + s, __ldcg(rep + s) - ac * (c * __ldg(p.val + s)));
        }
      }
      __syncwarp(mask);
    }
    // Copy the replicas of the processed examples into the shared model.
    for (uint32_t i = lo; i < hi; ++i) {
      const uint32_t e = list_at(p, l, i);
      const uint32_t b = __ldg(p.rowptr + e), en = __ldg(p.rowptr + e + 1);
      for (uint32_t s = b + lg; s < en; s += G) st_model(p.model + __ldg(p.idx + s), __ldcg(rep + s));
    }
  }
}

// K5 (kernel scope, shared model) and the global-replica variant (block scope
// with replicas too large for shared memory, thread scope).
template <int G, int TASK, int KIND, int SCOPE, bool LONG = false>
__global__ void __launch_bounds__(256) hogwild_kernel(HogParams p) {
  const int lg = threadIdx.x % G;
  const unsigned mask = group_mask<G>();
  const uint64_t hg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const uint64_t HG = ((uint64_t)gridDim.x * blockDim.x) / G;
  for (uint64_t w = hg; w < p.T; w += HG) {
    if (SCOPE == kScopeSharedAtomic) {
      run_worker<G, TASK, KIND, GlobalAtomicModel<kSpread>, LONG>(p, GlobalAtomicModel<kSpread>{p.model}, w, lg,
                                                                 mask);
    } else if (SCOPE == kScopeSharedAtomicFlat) {
      run_worker<G, TASK, KIND, GlobalAtomicModel<1>, LONG>(p, GlobalAtomicModel<1>{p.model}, w, lg, mask);
    } else if (SCOPE == kScopeGlobalRepAtomic) {
      run_worker<G, TASK, KIND, GlobalAtomicModel<1>>(p, GlobalAtomicModel<1>{p.model + (w / p.gs) * p.ld},
                                                      w, lg, mask);
    } else {  // kScopeGlobalRep
      run_worker<G, TASK, KIND>(p, GlobalModel{p.model + (w / p.gs) * p.ld, 1u}, w, lg, mask);
    }
  }
}

// K6 (block scope): CTA r owns replica r in shared memory, loaded from the
// global snapshot at epoch start (async_engine.cpp:298-301) and written to
// replicas[r] at the end for K7. Workers r*gs .. r*gs+gs-1 run in the CTA.
template <int G, int TASK, int KIND>
__global__ void __launch_bounds__(1024) hogwild_smem_kernel(HogParams p, const float* w32,
                                                            uint64_t R) {
  extern __shared__ __align__(16) float rep[];
  __shared__ uint64_t bar;
  const int lg = threadIdx.x % G;
  const unsigned mask = group_mask<G>();
  const uint64_t gi = threadIdx.x / G, NG = blockDim.x / G;
  // The replica (w32 and its zero guard slot, allocated in whole 16-byte
  // groups) arrives by bulk copy: a thread loop left ~10 % of the epoch's
  // stall samples on the stores waiting for their loads (ncu, rcv1 block).
  const uint32_t bytes = round_up16((p.d + 1) * 4ull);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  for (uint64_t r = blockIdx.x; r < R; r += gridDim.x, phase ^= 1u) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, bytes);
      for (uint32_t off = 0; off < bytes; off += 32768)
        bulk_g2s(reinterpret_cast<char*>(rep) + off, reinterpret_cast<const char*>(w32) + off,
                 min(32768u, bytes - off), &bar);
    }
    mbar_wait(&bar, phase);
    for (uint64_t t = gi; t < p.gs; t += NG) {
      const uint64_t w = r * p.gs + t;
      if (w >= p.T) break;
      run_worker<G, TASK, KIND>(p, SmemModel{rep}, w, lg, mask);
    }
    __syncthreads();
    for (uint64_t j = threadIdx.x; j < p.d; j += blockDim.x) p.model[r * p.ld + j] = rep[j];
    __syncthreads();
  }
}

// Slice-spread copy of the shared model for kernel scope: coordinate j at
// float offset j*ms (ms*4 = 256 B), so concurrent red.add updates to
// different coordinates land in different L2 slices instead of serialising on
// the few lines a small model occupies (B300_MICROARCH.md, "L2-atom
// multi-CTA": distinct >=128 B-spaced addresses are ~63x faster).
__global__ void spread_kernel(uint64_t d, uint32_t ms, const float* w32, float* ws) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= d;
       j += (uint64_t)gridDim.x * blockDim.x)
    ws[j * ms] = j < d ? w32[j] : 0.f;
}
__global__ void gather_kernel(uint64_t d, uint32_t ms, const float* ws, float* w32, double* w64) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const float v = ws[j * ms];
    w32[j] = v;
    w64[j] = static_cast<double>(v);
  }
}

// Replica prepare for the global-replica scope: every replica <- snapshot.
__global__ void replicas_fill_kernel(float* reps, uint64_t R, uint64_t ld, uint64_t d,
                                     const float* w32) {
  const uint64_t total = R * ld;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = i % ld;
    reps[i] = j < d ? w32[j] : 0.f;
  }
}

// K7: global = unweighted mean of the replicas, summed in replica order in
// fp64 (merge_models, async_engine.cpp:148-153).
__global__ void replicas_merge_kernel(const float* reps, uint64_t R, uint64_t ld, uint64_t d,
                                      double* w64, float* w32) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    // Replica order as merge_models sums; eight loads in flight per thread.
    double s = 0.0;
    uint64_t r = 0;
    for (; r + 8 <= R; r += 8) {
      float v8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v8[k] = reps[(r + k) * ld + j];
#pragma unroll
      for (int k = 0; k < 8; ++k) s += 1.0 * static_cast<double>(v8[k]);
    }
    for (; r < R; ++r) s += 1.0 * static_cast<double>(reps[r * ld + j]);
    const double v = s / static_cast<double>(R);
    w64[j] = v;
    w32[j] = static_cast<float>(v);
  }
}

// Weighted mean over models' fp64 masters (merge_models with weights).
__global__ void models_mean_kernel(const double* const* ws, const double* wts, uint64_t count,
                                   double total, uint64_t d, double* out64, float* out32) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint64_t r = 0; r < count; ++r) s += (wts ? wts[r] : 1.0) * ws[r][j];
    const double v = s / total;
    out64[j] = v;
    out32[j] = static_cast<float>(v);
  }
}

__global__ void scale_model_kernel(uint64_t d, double scale, double* w64, float* w32) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double v = w64[j] * scale;
    w64[j] = v;
    w32[j] = static_cast<float>(v);
  }
}

__global__ void copy_model_kernel(uint64_t d, const double* src64, double* dst64, float* dst32) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < d;
       j += (uint64_t)gridDim.x * blockDim.x) {
    dst64[j] = src64[j];
    dst32[j] = static_cast<float>(src64[j]);
  }
}

// K8p: CSR -> slot-major padded (proj/src/dataset.cpp:380-402): thread per
// row, slot s of row e at s*n + e (coalesced over e), padding = (0, d).
__global__ void csr_to_padded_kernel(const float* __restrict__ val, const uint32_t* __restrict__ idx,
                                     const uint32_t* __restrict__ rowptr, uint64_t n, uint64_t d,
                                     uint64_t pw, float* pval, uint32_t* pidx) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = rowptr[e], len = rowptr[e + 1] - b;
    for (uint64_t s = 0; s < pw; ++s) {
      const bool in = s < len;
      pval[s * n + e] = in ? val[b + s] : 0.f;
      pidx[s * n + e] = in ? idx[b + s] : static_cast<uint32_t>(d);
    }
  }
}

// K8: dense row-major -> column-major (32x32 tiles through shared memory).
__global__ void transpose_kernel(const float* __restrict__ in, float* __restrict__ out,
                                 uint64_t rows, uint64_t cols) {
  __shared__ float tile[32][33];
  const uint64_t bx = (uint64_t)blockIdx.x * 32, by = (uint64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const uint64_t r = by + i, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const uint64_t c = bx + i, r = by + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
  }
}

template <class Fn>
void dispatch_lanes(int g, Fn&& fn) {
  switch (g) {
    case 1: fn.template operator()<1>(); break;
    case 2: fn.template operator()<2>(); break;
    case 4: fn.template operator()<4>(); break;
    case 8: fn.template operator()<8>(); break;
    case 16: fn.template operator()<16>(); break;
    default: fn.template operator()<32>(); break;
  }
}

template <class Fn>
void dispatch_kind(int kind, Fn&& fn) {
  switch (kind) {
    case kKindDenseRow: fn.template operator()<kKindDenseRow>(); break;
    case kKindCsr: fn.template operator()<kKindCsr>(); break;
    case kKindDenseCol: fn.template operator()<kKindDenseCol>(); break;
    default: fn.template operator()<kKindPaddedCol>(); break;
  }
}

}  // namespace

int hogwild_auto_lanes(const Dataset& ds, int access) {
  if (access == SGDB_ACCESS_COL_RR || access == SGDB_ACCESS_COL_CH) return 1;
  // Row paths: one warp per example (the paper's GPU kernel). Narrower lane
  // groups pack more workers per warp but lose on Pareto-tail rows; measured
  // on w8a (avg 11.7 nnz) G=32 was fastest (scripts/hogwild_lanes.py).
  const double avg = ds.kind == Kind::Dense
                         ? static_cast<double>(ds.d)
                         : (ds.n ? static_cast<double>(ds.nnz) / static_cast<double>(ds.n) : 1.0);
  return avg <= 2.0 ? 8 : 32;
}

// One resident wave: CTAs/SM from the occupancy calculator for this kernel
// instance, capped by the CTAs the workers need.
template <class K>
unsigned wave_grid(const Ctx& c, K kern, size_t smem, uint64_t workers, int lanes) {
  int per_sm = 0;
  per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), 256, smem);
  const uint64_t cap = static_cast<uint64_t>(std::max(1, per_sm)) * c.num_sms;
  const uint64_t need = (workers * static_cast<uint64_t>(lanes) + 255) / 256;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min(need, cap)));
}

bool hogwild_long_rows(const Dataset& ds) {
  return ds.kind == Kind::Csr && ds.n && ds.nnz / ds.n >= 256;
}

uint64_t hogwild_resident_workers(const Ctx& c, const Dataset& ds, int lanes) {
  uint64_t out = 0;
  dispatch_lanes(lanes, [&]<int GL>() {
    const unsigned grid =
        (GL == 32 && hogwild_long_rows(ds))
            ? wave_grid(c, hogwild_kernel<GL, kTaskSVM, kKindCsr, kScopeSharedAtomic, true>, 0,
                        ~uint64_t(0) / 64, GL)
            : wave_grid(c, hogwild_kernel<GL, kTaskSVM, kKindCsr, kScopeSharedAtomic>, 0,
                        ~uint64_t(0) / 64, GL);
    out = static_cast<uint64_t>(grid) * 256 / GL;
  });
  return out;
}

void hogwild_epoch(Dataset& ds, Model& m, const HogwildArgs& a) {
  Ctx& c = *ds.ctx;
  const bool col = a.access == SGDB_ACCESS_COL_RR || a.access == SGDB_ACCESS_COL_CH;
  const bool rr = a.access == SGDB_ACCESS_ROW_RR || a.access == SGDB_ACCESS_COL_RR;
  if (ds.n_global != ds.n || ds.row_base != 0)
    throw Unsupported("Hogwild epochs run on whole (replicated) datasets");

  HogParams p{};
  int kind;
  if (col) {
    build_col(ds);
    if (ds.layout_in == SGDB_LAYOUT_PADDED) {
      kind = kKindPaddedCol;
      p.val = ds.pval.p;
      p.idx = ds.pidx.p;
      p.pw = ds.pw;
    } else {
      kind = kKindDenseCol;
      p.val = ds.xcol.p;
    }
  } else if (ds.kind == Kind::Dense) {
    kind = kKindDenseRow;
    p.val = ds.x.p;
  } else {
    kind = kKindCsr;
    p.val = ds.val.p;
    p.idx = ds.idx.p;
    p.rowptr = ds.rowptr.p;
  }
  p.y = ds.labels.p;
  p.n = ds.n;
  p.d = ds.d;
  p.T = a.workers;
  p.k = a.k;
  p.rr = rr ? 1 : 0;
  p.offsets = a.offsets ? 1 : 0;
  p.alpha = a.alpha;
  if (a.nseg == 0 || a.seg >= a.nseg) throw std::invalid_argument("hogwild segment out of range");
  p.seg = a.seg;
  p.nseg = a.nseg;
  const int G = a.lanes;


  if (a.replication == SGDB_REPL_EXAMPLE) {
    if (kind != kKindCsr) throw std::invalid_argument("example replication requires a sparse layout");
    materialize(m);
    m.spread_current = false;
    if (ds.ex_rep.n < ds.nnz || !ds.ex_rep.p) {
      ds.ex_rep.alloc(std::max<uint64_t>(1, ds.nnz));
      ds.ex_claim.alloc(ds.n);
      ds.ex_ready.alloc(ds.n);
      ds.ex_claim.zero(c.stream);
      ds.ex_ready.zero(c.stream);
      ds.ex_epoch = 0;
    }
    if (a.seg == 0) ++ds.ex_epoch;  // one replica generation per epoch (segments share it)
    p.model = m.w32.p;
    p.ms = 1;
    dispatch_lanes(G, [&]<int GL>() {
      auto kern = a.task == kTaskLR ? hogwild_example_kernel<GL, kTaskLR> : hogwild_example_kernel<GL, kTaskSVM>;
      const unsigned grid = wave_grid(c, kern, 0, a.workers, GL);
      prof_begin(c, "hogwild_example_kernel");
      kern<<<grid, 256, 0, c.stream>>>(p, ds.ex_rep.p, ds.ex_claim.p, ds.ex_ready.p, ds.ex_epoch);
    });
    launched(c, "hogwild_example_kernel");
    sync_w64_from_w32(m);
    return;
  }

  if (a.replication == SGDB_REPL_KERNEL) {
    p.gs = 1;
    p.ld = 0;
    // Slice-spread layout for models that stay L2-resident when spread.
    const uint32_t ms = ds.d <= (uint64_t{1} << 17) ? kSpread : 1u;
    if (ms > 1) {
      if (!(m.spread_current && m.spread_ms == ms)) {
        materialize(m);
        m.spread.alloc((ds.d + 1) * ms);
        const unsigned dgrid = static_cast<unsigned>(
            std::max<uint64_t>(1, std::min<uint64_t>((ds.d + 256) / 256, c.num_sms * 8ull)));
        prof_begin(c, "spread_kernel");
        spread_kernel<<<dgrid, 256, 0, c.stream>>>(ds.d, ms, m.w32.p, m.spread.p);
        launched(c, "spread_kernel");
        m.spread_ms = ms;
      }
      p.model = m.spread.p;
    } else {
      materialize(m);
      p.model = m.w32.p;
    }
    p.ms = ms;
    // Average row of hundreds of slots (news20: 461): the batch chain of the
    // longest rows dominates, and the worker count (n / chunk) is small anyway.
    const bool long_rows = kind == kKindCsr && hogwild_long_rows(ds);
    {
      dispatch_lanes(G, [&]<int GL>() {
        dispatch_kind(kind, [&]<int KD>() {
          void (*kern)(HogParams);
          if (long_rows && GL == 32 && KD == kKindCsr) {
            // Long rows: two slot batches per round trip (see process_example).
            if (ms > 1)
              kern = a.task == kTaskLR ? hogwild_kernel<GL, kTaskLR, KD, kScopeSharedAtomic, true>
                                       : hogwild_kernel<GL, kTaskSVM, KD, kScopeSharedAtomic, true>;
            else
              kern = a.task == kTaskLR ? hogwild_kernel<GL, kTaskLR, KD, kScopeSharedAtomicFlat, true>
                                       : hogwild_kernel<GL, kTaskSVM, KD, kScopeSharedAtomicFlat, true>;
          } else if (ms > 1) {
            kern = a.task == kTaskLR ? hogwild_kernel<GL, kTaskLR, KD, kScopeSharedAtomic>
                                     : hogwild_kernel<GL, kTaskSVM, KD, kScopeSharedAtomic>;
          } else {
            kern = a.task == kTaskLR ? hogwild_kernel<GL, kTaskLR, KD, kScopeSharedAtomicFlat>
                                     : hogwild_kernel<GL, kTaskSVM, KD, kScopeSharedAtomicFlat>;
          }
          const unsigned grid = wave_grid(c, kern, 0, a.workers, GL);
          prof_begin(c, "hogwild_kernel");
          kern<<<grid, 256, 0, c.stream>>>(p);
        });
      });
    }
    launched(c, "hogwild_kernel");
    if (ms > 1) {
      // The spread copy stays authoritative until someone reads the dense
      // model (materialize) — no gather between back-to-back epochs.
      m.spread_current = true;
      m.dense_current = false;
    } else {
      sync_w64_from_w32(m);
    }
    return;
  }

  // Block (group_size workers per replica) or thread (one per worker) scope.
  materialize(m);
  m.spread_current = false;
  const uint64_t gs = a.replication == SGDB_REPL_THREAD ? 1 : a.group_size;
  const uint64_t R = (a.workers + gs - 1) / gs;
  const uint64_t ld = (ds.d + 1 + 31) & ~uint64_t(31);
  m.replicas.alloc(R * ld);
  m.n_replicas = R;
  m.replica_ld = ld;
  p.gs = gs;
  p.ld = ld;
  p.ms = 1;
  p.model = m.replicas.p;
  const size_t rep_bytes = round_up16((ds.d + 1) * sizeof(float));
  // Shared-memory replicas (K6) when every SM gets one: a CTA per replica.
  // Fewer replicas than SMs (large groups, R sized to the data) keep them in
  // global memory (L2) and let every resident warp work (K6g, red.add
  // updates within a replica).
  const bool smem_ok = a.replication == SGDB_REPL_BLOCK && rep_bytes + 1024 <= c.max_smem_optin &&
                       R >= static_cast<uint64_t>(c.num_sms);
  if (smem_ok) {
    uint64_t threads = std::min<uint64_t>(1024, gs * G);
    threads = std::max<uint64_t>(32, (threads + 31) & ~uint64_t(31));
    int blocks_per_sm = static_cast<int>(std::max<size_t>(1, (c.max_smem_optin) / (rep_bytes + 1024)));
    blocks_per_sm = std::min<int>(blocks_per_sm, static_cast<int>(c.max_threads_per_sm / threads));
    blocks_per_sm = std::max(1, blocks_per_sm);
    const unsigned grid = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>(R, static_cast<uint64_t>(c.num_sms) * blocks_per_sm)));
    dispatch_lanes(G, [&]<int GL>() {
      dispatch_kind(kind, [&]<int KD>() {
        auto kern = a.task == kTaskLR ? hogwild_smem_kernel<GL, kTaskLR, KD>
                                      : hogwild_smem_kernel<GL, kTaskSVM, KD>;
        set_max_dyn_smem(reinterpret_cast<const void*>(kern), rep_bytes, "cudaFuncSetAttribute(hogwild_smem)");
        prof_begin(c, "hogwild_smem_kernel");
        kern<<<grid, static_cast<unsigned>(threads), rep_bytes, c.stream>>>(p, m.w32.p, R);
      });
    });
    launched(c, "hogwild_smem_kernel");
  } else {
    const unsigned fill_grid = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((R * ld + 255) / 256, c.num_sms * 8ull)));
    prof_begin(c, "replicas_fill_kernel");
    replicas_fill_kernel<<<fill_grid, 256, 0, c.stream>>>(m.replicas.p, R, ld, ds.d, m.w32.p);
    launched(c, "replicas_fill_kernel");
    const bool shared_rep = gs > 1;  // several workers race on a replica
    dispatch_lanes(G, [&]<int GL>() {
      dispatch_kind(kind, [&]<int KD>() {
        void (*kern)(HogParams);
        if (shared_rep)
          kern = a.task == kTaskLR ? hogwild_kernel<GL, kTaskLR, KD, kScopeGlobalRepAtomic>
                                   : hogwild_kernel<GL, kTaskSVM, KD, kScopeGlobalRepAtomic>;
        else
          kern = a.task == kTaskLR ? hogwild_kernel<GL, kTaskLR, KD, kScopeGlobalRep>
                                   : hogwild_kernel<GL, kTaskSVM, KD, kScopeGlobalRep>;
        const unsigned grid = wave_grid(c, kern, 0, a.workers, GL);
        prof_begin(c, "hogwild_kernel(replicas)");
        kern<<<grid, 256, 0, c.stream>>>(p);
      });
    });
    launched(c, "hogwild_kernel(replicas)");
  }
  const unsigned mgrid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>((ds.d + 255) / 256, c.num_sms * 8ull)));
  prof_begin(c, "replicas_merge_kernel");
  replicas_merge_kernel<<<mgrid, 256, 0, c.stream>>>(m.replicas.p, R, ld, ds.d, m.w64.p, m.w32.p);
  launched(c, "replicas_merge_kernel");
}

void average_models(Ctx& c, Model* const* models, uint64_t count, const double* weights,
                    Model& out, bool refresh) {
  const uint64_t d = out.d;
  std::vector<const double*> ptrs(count);
  double total = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    if (models[i]->d != d) throw std::invalid_argument("merge_models: dimension mismatch");
    ptrs[i] = models[i]->w64.p;
    total += weights ? weights[i] : 1.0;
  }
  if (weights && total == 0.0) throw std::invalid_argument("merge_models: zero total weight");
  DBuf<const double*> dptrs;
  dptrs.alloc(count);
  DBuf<double> dw;
  check(cudaMemcpyAsync(dptrs.p, ptrs.data(), count * sizeof(double*), cudaMemcpyHostToDevice,
                        c.stream),
        "H2D model ptrs");
  if (weights) {
    dw.alloc(count);
    check(cudaMemcpyAsync(dw.p, weights, count * sizeof(double), cudaMemcpyHostToDevice, c.stream),
          "H2D weights");
  }
  const unsigned grid =
      static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((d + 255) / 256, c.num_sms * 8ull)));
  prof_begin(c, "models_mean_kernel");
  models_mean_kernel<<<grid, 256, 0, c.stream>>>(dptrs.p, weights ? dw.p : nullptr, count, total, d,
                                                 out.w64.p, out.w32.p);
  launched(c, "models_mean_kernel");
  if (refresh) {
    for (uint64_t i = 0; i < count; ++i) {
      if (models[i] == &out) continue;
      prof_begin(c, "copy_model_kernel");
      copy_model_kernel<<<grid, 256, 0, c.stream>>>(d, out.w64.p, models[i]->w64.p, models[i]->w32.p);
      launched(c, "copy_model_kernel");
    }
  }
  // dptrs / dw are freed on scope exit; make sure the kernels consumed them.
  check(cudaStreamSynchronize(c.stream), "average_models sync");
}

void materialize(Model& m) {
  if (m.dense_current) return;
  Ctx& c = *m.ctx;
  const unsigned dgrid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>((m.d + 256) / 256, c.num_sms * 8ull)));
  prof_begin(c, "gather_kernel");
  gather_kernel<<<dgrid, 256, 0, c.stream>>>(m.d, m.spread_ms, m.spread.p, m.w32.p, m.w64.p);
  launched(c, "gather_kernel");
  m.dense_current = true;
}

void scale_model(Model& m, double scale) {
  Ctx& c = *m.ctx;
  const unsigned grid =
      static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((m.d + 255) / 256, c.num_sms * 8ull)));
  prof_begin(c, "scale_model_kernel");
  scale_model_kernel<<<grid, 256, 0, c.stream>>>(m.d, scale, m.w64.p, m.w32.p);
  launched(c, "scale_model_kernel");
}

void build_padded_from_csr(Dataset& ds) {
  Ctx& c = *ds.ctx;
  const uint64_t n = ds.n, pw = ds.max_row;
  ds.pw = pw;
  ds.pval.alloc(std::max<uint64_t>(1, n * pw));
  ds.pidx.alloc(std::max<uint64_t>(1, n * pw));
  if (n && pw) {
    const unsigned grid =
        static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, c.num_sms * 8ull)));
    prof_begin(c, "csr_to_padded_kernel");
    csr_to_padded_kernel<<<grid, 256, 0, c.stream>>>(ds.val.p, ds.idx.p, ds.rowptr.p, n, ds.d, pw, ds.pval.p,
                                                     ds.pidx.p);
    launched(c, "csr_to_padded_kernel");
  }
  check(cudaStreamSynchronize(c.stream), "padded build");
  ds.col_built = true;
}

void build_col(Dataset& ds) {
  if (ds.col_built) return;
  Ctx& c = *ds.ctx;
  if (ds.layout_in == SGDB_LAYOUT_PADDED) {
    if (!ds.pval.p) throw Unsupported("padded column arrays were not uploaded");
  } else if (ds.kind == Kind::Dense) {
    ds.xcol.alloc(ds.n * ds.d);
    dim3 grid(static_cast<unsigned>((ds.d + 31) / 32), static_cast<unsigned>((ds.n + 31) / 32));
    prof_begin(c, "transpose_kernel");
    transpose_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(ds.x.p, ds.xcol.p, ds.n, ds.d);
    launched(c, "transpose_kernel");
  } else {
    throw std::invalid_argument("column access paths on sparse data require the padded dense layout");
  }
  ds.col_built = true;
}

}  // namespace sgdb::dev
