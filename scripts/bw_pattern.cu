// HBM read bandwidth of the access patterns the sparse passes use, against a
// plain grid-stride read (diagnostic; not part of the library).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bw_pattern scripts/bw_pattern.cu
//   ./bw_pattern
//
// Patterns over a 307 MB working set (rcv1's per-pass bytes), one CTA of 1024
// threads per SM, 256-bit loads:
//   stride   grid-stride: consecutive warps read consecutive 1 KB blocks
//   chunk1   each warp streams its own contiguous 1/(148*32) share (one stream)
//   chunk3   as chunk1, but three streams per warp in the K2s proportions
//            (4 B values, 2 B ids, 1/8 B bitmap per slot)
//   chunkNB  chunk3 with 2 tiles in flight per warp (the kernels' NB = 2)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const float* p, float4& a, float4& b) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
}

__global__ void __launch_bounds__(1024, 1) k_stride(const float* x, size_t nf, float* out) {
  float s = 0.f;
  const size_t step = size_t(gridDim.x) * blockDim.x * 8;
  for (size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i + 8 <= nf; i += step) {
    float4 a, b;
    ld256(x + i, a, b);
    s += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
  }
  if (s == 12345.f) out[0] = s;
}

// Grid-stride with U independent 256-bit loads in flight per thread.
template <int U>
__global__ void __launch_bounds__(1024, 1) k_stride_u(const float* x, size_t nf, float* out) {
  float s = 0.f;
  const size_t step = size_t(gridDim.x) * blockDim.x * 8;
  size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  for (; i + (U - 1) * step + 8 <= nf; i += U * step) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ld256(x + i + u * step, a[u], b[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s += a[u].x + a[u].y + a[u].z + a[u].w + b[u].x + b[u].y + b[u].z + b[u].w;
  }
  for (; i + 8 <= nf; i += step) {
    float4 a, b;
    ld256(x + i, a, b);
    s += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
  }
  if (s == 12345.f) out[0] = s;
}

// One stream per warp: slots [P, Q) of nf floats.
__global__ void __launch_bounds__(1024, 1) k_chunk1(const float* x, size_t nf, float* out) {
  const size_t W = size_t(gridDim.x) * 32, w = size_t(blockIdx.x) * 32 + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const size_t P = (nf * w / W) & ~size_t(255), Q = (nf * (w + 1) / W) & ~size_t(255);
  float s = 0.f;
  for (size_t t = P; t < Q; t += 256) {
    float4 a, b;
    ld256(x + t + 8 * lane, a, b);
    s += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
  }
  if (s == 12345.f) out[0] = s;
}

// Three streams per warp (values, 16-bit ids, bitmap), NB tiles in flight.
template <int NB>
__global__ void __launch_bounds__(1024, 1) k_chunk3(const float* v, const uint16_t* id, const uint32_t* bm,
                                                    size_t ns, float* out) {
  const size_t W = size_t(gridDim.x) * 32, w = size_t(blockIdx.x) * 32 + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const size_t P = (ns * w / W) & ~size_t(255), Q = (ns * (w + 1) / W) & ~size_t(255);
  float s = 0.f;
  float4 a[NB], b[NB];
  uint4 j[NB];
  uint32_t m[NB];
  auto fetch = [&](size_t t, int k) {
    const size_t q = t < Q ? t : P;
    ld256(v + q + 8 * lane, a[k], b[k]);
    j[k] = __ldg(reinterpret_cast<const uint4*>(id + q + 8 * lane));
    m[k] = __ldg(bm + (q + 8 * lane) / 32);
  };
#pragma unroll
  for (int k = 0; k < NB; ++k) fetch(P + 256 * k, k);
  for (size_t t = P; t < Q; t += 256 * NB) {
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      s += a[k].x + a[k].y + a[k].z + a[k].w + b[k].x + b[k].y + b[k].z + b[k].w +
           float(j[k].x ^ j[k].y ^ j[k].z ^ j[k].w ^ m[k]);
      fetch(t + 256 * (k + NB), k);
    }
  }
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t ns = size_t(49) << 20;  // 51.4M slots: 206 MB values + 103 MB ids + 6 MB bitmap
  float *v, *out;
  uint16_t* id;
  uint32_t* bm;
  char* fl;
  cudaMalloc(&v, ns * 4 + 4096);
  cudaMalloc(&id, ns * 2 + 4096);
  cudaMalloc(&bm, ns / 8 + 4096);
  cudaMalloc(&out, 64);
  cudaMalloc(&fl, size_t(256) << 20);
  cudaMemset(v, 0, ns * 4);
  cudaMemset(id, 0, ns * 2);
  cudaMemset(bm, 0, ns / 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t nf_all = (ns * 4 + ns * 2 + ns / 8) / 4;  // same total bytes as one pass
  float* big;
  cudaMalloc(&big, nf_all * 4 + 4096);
  cudaMemset(big, 0, nf_all * 4);
  auto flush = [&] {
    cudaMemset(fl, 1, size_t(256) << 20);
    k_stride<<<sms, 1024>>>(reinterpret_cast<const float*>(fl), (size_t(256) << 20) / 4, out);
  };
  auto time = [&](const char* name, auto launch, double bytes) {
    float best = 1e30f, sum = 0.f;
    for (int i = 0; i < 13; ++i) {
      flush();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 3) sum += ms, best = best < ms ? best : ms;
    }
    printf("{\"pattern\": \"%s\", \"us\": %.1f, \"GBps\": %.0f}\n", name, 1e3 * sum / 10,
           bytes / (sum / 10 / 1e3) / 1e9);
  };
  const double bytes = double(nf_all) * 4;
  time("stride", [&] { k_stride<<<sms, 1024>>>(big, nf_all, out); }, bytes);
  time("chunk1", [&] { k_chunk1<<<sms, 1024>>>(big, nf_all, out); }, bytes);
  time("chunk3_nb1", [&] { k_chunk3<1><<<sms, 1024>>>(v, id, bm, ns, out); }, bytes);
  time("chunk3_nb2", [&] { k_chunk3<2><<<sms, 1024>>>(v, id, bm, ns, out); }, bytes);
  time("chunk3_nb3", [&] { k_chunk3<3><<<sms, 1024>>>(v, id, bm, ns, out); }, bytes);
  time("stride_2cta", [&] { k_stride<<<2 * sms, 1024>>>(big, nf_all, out); }, bytes);
  time("stride_u2", [&] { k_stride_u<2><<<sms, 1024>>>(big, nf_all, out); }, bytes);
  time("stride_u4", [&] { k_stride_u<4><<<sms, 1024>>>(big, nf_all, out); }, bytes);
  {  // two passes: one launch over 2x the bytes vs two launches back to back
    float* big2;
    if (cudaMalloc(&big2, nf_all * 8 + 4096) == cudaSuccess) {
      cudaMemset(big2, 0, nf_all * 8);
      time("stride_2x_one_launch", [&] { k_stride<<<sms, 1024>>>(big2, 2 * nf_all, out); }, 2 * bytes);
      time("stride_2x_two_launches", [&] {
        k_stride<<<sms, 1024>>>(big2, nf_all, out);
        k_stride<<<sms, 1024>>>(big2 + nf_all, nf_all, out);
      }, 2 * bytes);
      cudaFree(big2);
    }
  }
  {  // a 4 GiB read (the copy peak's size) with 4 loads in flight per thread
    float* huge;
    const size_t nh = size_t(1) << 30;
    if (cudaMalloc(&huge, nh * 4) == cudaSuccess) {
      cudaMemset(huge, 0, nh * 4);
      time("stride_u4_4GiB", [&] { k_stride_u<4><<<sms, 1024>>>(huge, nh, out); }, double(nh) * 4);
      cudaFree(huge);
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}
