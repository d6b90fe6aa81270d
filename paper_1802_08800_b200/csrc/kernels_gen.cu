// K9: device-side generator for the dense synthetic configuration
// (BASELINE.json configs[4]: 200M x 1,000). The reference's
// fixtures::dense_classification (proj/src/fixtures.cpp:30-52: uniform(-1,1)
// values, w_true ~ N(0,1), y = sign(x . w_true), 10% flipped labels) draws
// from one sequential mt19937_64, which cannot produce 800 GB on a host nor
// be split across GPUs. This generator keeps the distribution and makes every
// row a pure function of (seed, global row id): Philox-4x32-10 for the values
// and the flip draw, a host-computed Box-Muller hidden model, and a label dot
// product in a fixed order (lane-strided fp64 partials, then an xor butterfly,
// no FMA contraction) — so oracle/glm_oracle.cpp re-creates any slice bit for
// bit (tests/test_gpu_generator.py).
#include <cuda_runtime.h>

#include <cmath>
#include <memory>
#include <vector>

#include "device.hpp"
#include "philox.hpp"

namespace sgdb::dev {

namespace {

__global__ void __launch_bounds__(256) gen_dense_kernel(uint64_t n_local, uint32_t d,
                                                        uint64_t row_base, uint64_t seed,
                                                        double noise, const double* __restrict__ w,
                                                        float* __restrict__ x, float* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t tw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t nq = (d + 3) / 4;
  const bool vec = (d % 4) == 0;
  for (uint64_t r = gw; r < n_local; r += tw) {
    const uint64_t e = row_base + r;
    float* row = x + r * d;
    double part = 0.0;
    for (uint32_t q = lane; q < nq; q += 32) {
      const gen::U4 u = gen::value_quad(seed, e, q);
      const float v[4] = {gen::unit_value(u.x), gen::unit_value(u.y), gen::unit_value(u.z),
                          gen::unit_value(u.w)};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t j = 4 * q + t;
        if (j < d) part = __dadd_rn(part, __dmul_rn(static_cast<double>(v[t]), w[j]));
      }
      if (vec) {
        reinterpret_cast<float4*>(row)[q] = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * q + t < d) row[4 * q + t] = v[t];
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off));
    if (lane == 0) {
      float lab = part >= 0.0 ? 1.f : -1.f;
      if (noise > 0.0 && static_cast<double>(gen::flip_u(seed, e)) < noise) lab = -lab;
      y[r] = lab;
    }
  }
}

}  // namespace

// w_true ~ N(0,1) by Box-Muller over Philox draws (host; d is small).
std::vector<double> gen_hidden_model(uint64_t seed, uint64_t d) {
  std::vector<double> w(d);
  const uint32_t k0 = static_cast<uint32_t>(seed) ^ 0x9E3779B9u;
  const uint32_t k1 = static_cast<uint32_t>(seed >> 32) ^ 0x7F4A7C15u;
  for (uint64_t i = 0; 2 * i < d; ++i) {
    const gen::U4 r = gen::philox4x32_10(gen::U4{static_cast<uint32_t>(i), 0u, 0u, gen::kTagModel}, k0, k1);
    const uint64_t a = (static_cast<uint64_t>(r.x) << 20) | (r.y >> 12);
    const uint64_t b = (static_cast<uint64_t>(r.z) << 20) | (r.w >> 12);
    const double u1 = static_cast<double>(a + 1) * 0x1p-52;  // (0, 1]
    const double u2 = static_cast<double>(b) * 0x1p-52;      // [0, 1)
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 6.283185307179586 * u2;
    w[2 * i] = rad * std::cos(th);
    if (2 * i + 1 < d) w[2 * i + 1] = rad * std::sin(th);
  }
  return w;
}

// Widen 16-bit CSR column ids (host transfer format when d <= 65536) into the
// 32-bit ids the kernels read: 8 ids per thread, 16-byte loads.
__global__ void __launch_bounds__(256) widen_u16_kernel(const uint16_t* __restrict__ src,
                                                        uint32_t* __restrict__ dst, uint64_t n) {
  const uint64_t groups = n / 8;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(src)[g];
    uint4* o = reinterpret_cast<uint4*>(dst + g * 8);
    o[0] = make_uint4(v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16);
    o[1] = make_uint4(v.z & 0xFFFFu, v.z >> 16, v.w & 0xFFFFu, v.w >> 16);
  }
  if (blockIdx.x == 0 && threadIdx.x < n % 8) dst[groups * 8 + threadIdx.x] = src[groups * 8 + threadIdx.x];
}

void widen_u16(Ctx& c, const uint16_t* src, uint32_t* dst, uint64_t n) {
  if (n == 0) return;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
      std::max<uint64_t>(1, (n / 8 + 255) / 256), static_cast<uint64_t>(c.num_sms) * 8));
  prof_begin(c, "widen_u16_kernel");
  widen_u16_kernel<<<grid, 256, 0, c.stream>>>(src, dst, n);
  launched(c, "widen_u16_kernel");
}

void gen_dense(Dataset& ds, uint64_t seed, double noise) {
  Ctx& c = *ds.ctx;
  const std::vector<double> w = gen_hidden_model(seed, ds.d);
  DBuf<double> dw;
  dw.alloc(ds.d);
  check(cudaMemcpyAsync(dw.p, w.data(), ds.d * sizeof(double), cudaMemcpyHostToDevice, c.stream),
        "H2D hidden model");
  const uint64_t warps = std::max<uint64_t>(1, std::min<uint64_t>(ds.n, static_cast<uint64_t>(c.num_sms) * 64));
  const unsigned grid = static_cast<unsigned>((warps * 32 + 255) / 256);
  prof_begin(c, "gen_dense_kernel");
  gen_dense_kernel<<<grid, 256, 0, c.stream>>>(ds.n, static_cast<uint32_t>(ds.d), ds.row_base, seed,
                                               noise, dw.p, ds.x.p, ds.labels.p);
  launched(c, "gen_dense_kernel");
  check(cudaStreamSynchronize(c.stream), "gen sync");
}

}  // namespace sgdb::dev

extern "C" {

sgdb_status sgdb_generate_hidden_model(uint64_t seed, uint64_t d, double* out) {
  return sgdb_guard([&] {
    if (!out && d) throw std::invalid_argument("null output");
    const auto w = sgdb::dev::gen_hidden_model(seed, d);
    std::copy(w.begin(), w.end(), out);
  });
}

sgdb_status sgdb_dataset_generate_dense(sgdb_ctx* ctx, uint64_t n_local, uint64_t d,
                                        uint64_t row_base, uint64_t n_global, uint64_t seed,
                                        double label_noise, sgdb_dataset** out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    if (!ctx || !out) throw std::invalid_argument("null argument");
    if (d < 1 || d > 1024) throw std::invalid_argument("generated dense data needs 1 <= d <= 1024");
    if (n_global == 0) n_global = n_local;
    if (row_base + n_local > n_global) throw std::invalid_argument("shard exceeds n_global");
    if (n_global > 0xFFFFFFFFull) throw std::invalid_argument("example ids must fit in 32 bits");
    auto* ds = new sgdb_dataset();
    std::unique_ptr<sgdb_dataset> guard(ds);
    ds->ctx = ctx;
    ds->uid = next_dataset_uid();
    ds->n = n_local;
    ds->d = d;
    ds->row_base = row_base;
    ds->n_global = n_global;
    ds->layout_in = SGDB_LAYOUT_DENSE_ROW;
    ds->kind = Kind::Dense;
    ds->nnz = n_local * d;
    const uint64_t nlab = ((n_local + 3) & ~uint64_t(3)) + 8;
    ds->labels.alloc(nlab);
    ds->labels.zero(ctx->stream);
    ds->x.alloc(n_local * d + 8);
    check(cudaMemsetAsync(ds->x.p + n_local * d, 0, 8 * sizeof(float), ctx->stream), "memset tail");
    ds->order.alloc(std::max<uint64_t>(1, n_global));
    gen_dense(*ds, seed, label_noise);
    *out = guard.release();
  });
}

sgdb_status sgdb_dataset_read_dense(sgdb_ctx* ctx, const sgdb_dataset* ds, uint64_t row0,
                                    uint64_t nrows, float* values_out, float* labels_out) {
  using namespace sgdb::dev;
  return sgdb_guard([&] {
    if (ds->kind != Kind::Dense) throw std::invalid_argument("not a dense device dataset");
    if (row0 + nrows > ds->n) throw std::invalid_argument("rows out of range");
    if (values_out && nrows)
      check(cudaMemcpyAsync(values_out, ds->x.p + row0 * ds->d, nrows * ds->d * sizeof(float),
                            cudaMemcpyDeviceToHost, ctx->stream),
            "D2H values");
    if (labels_out && nrows)
      check(cudaMemcpyAsync(labels_out, ds->labels.p + row0, nrows * sizeof(float),
                            cudaMemcpyDeviceToHost, ctx->stream),
            "D2H labels");
    check(cudaStreamSynchronize(ctx->stream), "read sync");
  });
}

}  // extern "C"
