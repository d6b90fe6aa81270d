// Diagnostic probe (not part of the library): how fast can a warp-per-range
// kernel stream an rcv1-sized CSR (49M float values + 49M u32 indices) on
// B200, with and without the per-element work of the margin pass?
//   mode 0: stream val+idx, sum (no gathers)
//   mode 1: + SMEM gathers from a 189 KB model
//   mode 2: + a 5-step warp scan per tile (the segmented-scan skeleton)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, int E>
__global__ void __launch_bounds__(768, 1) probe(const float* __restrict__ val, const uint32_t* __restrict__ idx,
                                                uint32_t nnz, uint32_t d, float* out) {
  extern __shared__ float ws[];
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) ws[j] = 0.001f * j;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t s0 = (uint64_t(nnz) * gw / nw) & ~3u, s1 = uint64_t(nnz) * (gw + 1) / nw;
  float acc = 0.f;
  for (uint32_t t = s0; t < s1; t += 32 * E) {
    const uint32_t a = t + E * lane;
    float4 v[E / 4];
    uint4 j[E / 4];
#pragma unroll
    for (int k = 0; k < E / 4; ++k) {
      v[k] = __ldg(reinterpret_cast<const float4*>(val + a + 4 * k));
      j[k] = __ldg(reinterpret_cast<const uint4*>(idx + a + 4 * k));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < E / 4; ++k) {
      if (MODE == 0) {
        s += v[k].x + v[k].y + v[k].z + v[k].w + __uint_as_float(j[k].x ^ j[k].y ^ j[k].z ^ j[k].w);
      } else {
        s = fmaf(v[k].x, ws[j[k].x], s);
        s = fmaf(v[k].y, ws[j[k].y], s);
        s = fmaf(v[k].z, ws[j[k].z], s);
        s = fmaf(v[k].w, ws[j[k].w], s);
      }
    }
    if (MODE == 2) {
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const float o = __shfl_up_sync(0xffffffffu, s, off);
        const int f = __shfl_up_sync(0xffffffffu, (int)(j[0].x & 1), off);
        if (lane >= off && !f) s += o;
      }
    }
    acc += s;
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const uint32_t nnz = 48930591, d = 47236;
  float* val;
  uint32_t* idx;
  float* out;
  cudaMalloc(&val, (nnz + 64) * 4ull);
  cudaMalloc(&idx, (nnz + 64) * 4ull);
  cudaMalloc(&out, 4);
  cudaMemset(val, 0, (nnz + 64) * 4ull);
  cudaMemset(idx, 0, (nnz + 64) * 4ull);
  // idx: pseudo-random in [0, d)
  {
    uint32_t* h = (uint32_t*)malloc(nnz * 4ull);
    uint64_t x = 88172645463325252ull;
    for (uint32_t i = 0; i < nnz; ++i) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      h[i] = (uint32_t)(x % d);
    }
    cudaMemcpy(idx, h, nnz * 4ull, cudaMemcpyHostToDevice);
    free(h);
  }
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, const char* name, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, d * 4);
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemsetAsync(flush, it, 256 << 20);
      cudaEventRecord(a);
      kern<<<148, threads, d * 4>>>(val, idx, nnz, d, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    printf("%-28s %8.1f us  %6.0f GB/s  err=%s\n", name, best * 1e3, nnz * 8.0 / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(probe<0, 4>, "stream E=4", 768);
  run(probe<0, 8>, "stream E=8", 768);
  run(probe<0, 16>, "stream E=16", 768);
  run(probe<1, 4>, "stream+gather E=4", 768);
  run(probe<1, 8>, "stream+gather E=8", 768);
  run(probe<1, 16>, "stream+gather E=16", 768);
  run(probe<2, 8>, "stream+gather+scan E=8", 768);
  run(probe<2, 16>, "stream+gather+scan E=16", 768);
  return 0;
}
