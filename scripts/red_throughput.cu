// Throughput of scattered fp32 reductions into L2 (red.global.add.f32), the
// update primitive of the kernel-scope Hogwild kernel K5 (diagnostic; not
// part of the library). Addresses come from an in-register hash (no index
// loads), coordinate j lives at float offset j * stride (K5's slice-spread
// layout: stride 64 = 256 B), one warp-wide red per 32 updates.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/red_throughput.bin scripts/red_throughput.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// fp64 reductions (the sparse mini-batch step's update of the fp64 master).
__global__ void __launch_bounds__(256) k64(double* m, uint32_t d, uint32_t stride, uint64_t total, uint32_t salt) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t j = mix(static_cast<uint32_t>(i) ^ salt) % d;
    atomicAdd(m + uint64_t(j) * stride, 1e-9);
  }
}

template <int MODE>  // 0: red.add.f32, 1: plain store, 2: load (gather) only
__global__ void __launch_bounds__(256) k(float* m, uint32_t d, uint32_t stride, uint64_t total, float* out) {
  float acc = 0.f;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t j = mix(static_cast<uint32_t>(i)) % d;
    float* p = m + uint64_t(j) * stride;
    if (MODE == 0) atomicAdd(p, 1e-7f);
    else if (MODE == 1) __stcg(p, 1e-7f);
    else acc += __ldcg(p);
  }
  if (MODE == 2 && acc == 12345.f) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *m, *out;
  cudaMalloc(&m, size_t(1) << 30);
  cudaMalloc(&out, 64);
  cudaMemset(m, 0, size_t(1) << 30);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case {
    const char* name;
    uint32_t d, stride;
    uint64_t total;
  } cases[] = {
      {"rcv1-like: 47,236 coords, 256 B apart, 48.9M updates", 47236, 64, 48995496},
      {"rcv1-like, contiguous coords", 47236, 1, 48995496},
      {"real-sim-like: 20,958 coords, 256 B apart, 3.7M updates", 20958, 64, 3709431},
      {"w8a-like: 300 coords, 256 B apart, 0.75M updates", 300, 64, 753755},
      {"w8a-like, contiguous coords", 300, 1, 753755},
  };
  const char* modes[] = {"red.add.f32", "st.cg (plain)", "ld.cg (gather)"};
  for (auto& c : cases) {
    for (int mode = 0; mode < 3; ++mode) {
      auto launch = [&] {
        const unsigned grid = sms * 8;
        if (mode == 0) k<0><<<grid, 256>>>(m, c.d, c.stride, c.total, out);
        else if (mode == 1) k<1><<<grid, 256>>>(m, c.d, c.stride, c.total, out);
        else k<2><<<grid, 256>>>(m, c.d, c.stride, c.total, out);
      };
      float sum = 0.f;
      for (int r = 0; r < 13; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 3) sum += ms;
      }
      const double us = 1e3 * sum / 10;
      printf("{\"case\": \"%s\", \"op\": \"%s\", \"us\": %.1f, \"G_ops_per_s\": %.1f}\n", c.name, modes[mode], us,
             c.total / us / 1e3);
    }
  }
  // One rcv1 mini-batch step's worth of fp64 reductions (4,096 rows x 73 slots).
  for (uint32_t stride : {1u, 4u, 32u}) {
    float sum = 0.f;
    for (int r = 0; r < 13; ++r) {
      cudaEventRecord(e0);
      k64<<<sms * 4, 256>>>(reinterpret_cast<double*>(m), 47236, stride, 299662, r);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) sum += ms;
    }
    printf("{\"case\": \"rcv1 mini-batch step: 300K fp64 red.add on 47,236 coords, stride %u doubles\", \"us\": %.2f}\n",
           stride, 1e3 * sum / 10);
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}
