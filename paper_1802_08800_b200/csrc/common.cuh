// Device helpers shared by the sm_100a kernels: GLM scalar cores, lane-group
// reductions, fp64 atomics and the mbarrier / cp.async.bulk (1-D TMA) PTX used
// by the streaming kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Device-side bounds checks of the check build (make XFLAGS=-DSGDB_CHECKS):
// a failed check traps the kernel (cudaErrorAssert). Compiled out otherwise.
#ifdef SGDB_CHECKS
#include <cassert>
#define SGDB_CHECK(c) assert(c)
#else
#define SGDB_CHECK(c) ((void)0)
#endif

namespace sgdb::dev {

constexpr int kTaskLR = 0;
constexpr int kTaskSVM = 1;

// Scalar cores in fp32, following proj/src/glm.cpp:24-34 and the stable
// sigmoid split of proj/include/sgdbench/math.hpp:10-16.
__device__ __forceinline__ float sigmoid_f(float u) {
  if (u <= 0.0f) {
    float e = expf(u);
    return e / (1.0f + e);
  }
  return 1.0f / (1.0f + expf(-u));
}

// c such that the point gradient is c * x (glm.cpp:30-34).
template <int TASK>
__device__ __forceinline__ float coef_f(float z, float y) {
  float m = y * z;
  if (TASK == kTaskLR) return sigmoid_f(-m) * -y;
  return m < 1.0f ? -y : 0.0f;
}

// coef_f with the fast-math exponential and division (__expf, __fdividef:
// a few ulp) for the streaming passes, where the exact division's slow path
// would cost more issue slots than the rest of a row. Same stable split.
template <int TASK>
__device__ __forceinline__ float coef_fast(float z, float y) {
  const float m = y * z;
  if (TASK == kTaskLR) {
    const float u = -m;
    const float e = __expf(-fabsf(u));
    const float s = u <= 0.0f ? __fdividef(e, 1.0f + e) : __fdividef(1.0f, 1.0f + e);
    return s * -y;
  }
  return m < 1.0f ? -y : 0.0f;
}

// Point loss in fp64 (glm.cpp:24-28, math.hpp:19-22).
__device__ __forceinline__ double softplus_d(double u) {
  if (u > 0.0) return u + log1p(exp(-u));
  return log1p(exp(u));
}
__device__ __forceinline__ double loss_d(int task, double z, double y) {
  double m = y * z;
  if (task == kTaskLR) return softplus_d(-m);
  return m < 1.0 ? 1.0 - m : 0.0;
}

// Sum over an aligned group of G lanes (G power of two, <= 32); every lane of
// the group receives the total. All 32 lanes must execute it.
template <int G, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Sum across the 32/G groups of a warp for a fixed in-group lane (lanes with
// equal lane % G), i.e. xor over the high lane bits.
template <int G, typename T>
__device__ __forceinline__ T cross_group_sum(T v) {
#pragma unroll
  for (int off = G; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// L2-coherent model accesses for the Hogwild kernels: the shared model is
// written by every SM, so reads bypass L1 (ld.global.cg) to see the latest
// L2 value; Hogwild permits stale reads and lost updates between workers
// (proj/include/sgdbench/async_engine.hpp:49-52), not arbitrarily stale L1.
__device__ __forceinline__ float ld_model(const float* p) { return __ldcg(p); }
__device__ __forceinline__ void st_model(float* p, float v) { __stcg(p, v); }

// ---- programmatic dependent launch ---------------------------------------------
// A kernel launched with cudaLaunchAttributeProgrammaticStreamSerialization
// may start while its predecessor drains: it issues the loads that do not
// depend on the predecessor first, then waits here (griddepcontrol.wait:
// the predecessor grid has completed and its writes are visible).
// Arrival on a gpu-scope counter with acquire-release semantics: after a CTA
// barrier the CTA's prior writes are ordered before it (release is
// cumulative), and the arriving thread sees every earlier arrival's writes.
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- mbarrier + cp.async.bulk (1-D TMA, no tensor map) ------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Bulk global -> shared copy completing on `bar` (bytes % 16 == 0, both
// addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__host__ __device__ __forceinline__ uint32_t round_up16(uint64_t b) {
  return static_cast<uint32_t>((b + 15) & ~uint64_t(15));
}

// Worker w's assign() list (dataset.cpp:470-503), generated on the fly:
// base ids then k wrapped extras after the last base id. Round robin: ids
// w, w+T, ...; chunk: [w*ceil(n/T), min((w+1)*ceil(n/T), n)).
// (Example ids fit 32 bits: n_global <= 2^32 is enforced at upload.)
struct WorkerList {
  uint32_t first, step, cnt, total, last;
};
__device__ __forceinline__ WorkerList assign_list(uint64_t n, uint64_t T, uint64_t k, bool rr,
                                                  uint64_t w) {
  WorkerList l;
  if (rr) {
    l.cnt = w < n ? static_cast<uint32_t>((n - 1 - w) / T + 1) : 0u;
    l.first = static_cast<uint32_t>(w);
    l.step = static_cast<uint32_t>(T);
  } else {
    const uint64_t chunk = (n + T - 1) / T;
    const uint64_t b = w * chunk, e = min(n, b + chunk);
    l.cnt = e > b ? static_cast<uint32_t>(e - b) : 0u;
    l.first = static_cast<uint32_t>(min(b, n));
    l.step = 1;
  }
  l.total = l.cnt ? l.cnt + static_cast<uint32_t>(k) : 0u;
  l.last = l.cnt ? l.first + (l.cnt - 1) * l.step : 0u;
  return l;
}
__device__ __forceinline__ uint32_t assign_at(uint64_t n, const WorkerList& l, uint32_t i) {
  return i < l.cnt ? l.first + i * l.step
                   : static_cast<uint32_t>((uint64_t(l.last) + 1 + (i - l.cnt)) % n);
}

}  // namespace sgdb::dev
