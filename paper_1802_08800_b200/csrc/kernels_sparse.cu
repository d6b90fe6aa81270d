// Full-batch sparse step (B = N) over CSR data — the hot path of sync::train
// at B = N on rcv1 / real-sim / news20 / w8a-shaped inputs
// (proj/src/sync_engine.cpp:22-42 -> linalg::matvec, the LR/SVM coefficient,
// linalg::matvec_transposed; proj/src/linalg.cpp:30-109, glm.cpp:30-34).
//
//   K2s  margin pass   z = X w, c = coef(z, y)                (CSR stream, model in SMEM)
//   K2w  margin pass of a model too large for SMEM                (column-blocked CSR stream)
//   K3s  gradient pass g = X^T c, w -= alpha g                    (row-blocked CSC stream)
//   K23g K2s then K3s in ONE launch (models in SMEM; the default), the
//        dependency between them carried by per-row-block release counts
//
// Both passes are one segmented stream over a CTA's contiguous range of
// nonzeros: each warp walks its share in 256-slot tiles (lane l holds slots
// 8l..8l+7 of a tile: one 256-bit load of values + 8 ids), multiplies with the
// staged operand (the model, or the row block's coefficient slice, in SMEM),
// and recovers the per-segment sums (rows, or (block, column) segments) with
// a segmented warp scan. Segment boundaries come from a HEAD BITMAP (bit s =
// slot s starts a non-empty segment) built once per upload, so a lane finds
// its boundaries with one 32-bit load and a shift — no row-pointer walking,
// no per-slot masks on full tiles. A segment's identity is its ordinal among
// the heads (the prefix popcount of the bitmap words, also built once); the
// ordinal maps to a row / (block, column) directly unless the data has empty
// segments, in which case a compaction map translates it.
//
// CTA ranges start at segment starts, so a segment is only ever cut between
// warps of the same CTA; those pieces are combined in SMEM after the stream,
// in slot order. The gradient pass writes fp32 per-(block, column) sums; the
// last CTA of each column range (arrival ticket) sums them over the row
// blocks in block order and applies the update: deterministic, no atomics on
// data, no grid barrier, any grid size.
//
// K2w and K3s are the same blocked pass (blocked_pass_kernel) over a blocked
// copy of the nonzeros with 16-bit block-local major ids (Blocked in
// device.hpp): rows blocked for K3s (operand slice: the coefficients),
// columns blocked for K2w (operand slice: the model). Both copies are built
// on the device by a stable radix sort of (block, minor) keys, at upload and
// after a refresh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "device.hpp"

namespace sgdb::dev {
namespace {

constexpr int kNT = 1024;  // threads per CTA of both passes
constexpr int kNW = kNT / 32;
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kMaxRowBlock = 49152;  // coefficient slice <= 192 KB of SMEM

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Eight consecutive fp32 values in one 256-bit load (LDG.E.256, sm_100+):
// the warp's 32 lanes read 1 KB of contiguous values in one instruction; two
// 128-bit loads per lane would each touch every line of the 1 KB half-used.
__device__ __forceinline__ void ldg256(const float* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Number of heads in slots [0, P): word prefix + partial word.
__device__ __forceinline__ int32_t heads_before(const uint32_t* __restrict__ bm,
                                                const uint32_t* __restrict__ pre, uint32_t P) {
  const uint32_t wd = P >> 5, sh = P & 31u;
  uint32_t c = __ldg(pre + wd);
  if (sh) c += __popc(__ldg(bm + wd) & ((1u << sh) - 1u));
  return static_cast<int32_t>(c);
}

// One warp's segmented stream over slots [P, Q), in tiles of 32*E slots
// (lane l holds slots E*l .. E*l+E-1 of a tile).
//   ld(s) -> the lane's E-slot window at s (s % E == 0)
//   prod(win, p[E]) -> the E products
//   close(X, z, first) -> segment ordinal X ends with sum z (the warp's first
//                          closing is flagged: its segment began before P)
// ord: ordinal of the segment holding slot P-1 on entry, of the segment open
// at Q on exit; carry: the open segment's sum over [.., Q); had: a head was seen.
// NB window buffers rotate through registers (static indices), so NB-1 tiles
// of loads stay in flight while one is reduced.
template <int E, int NB, class Win, class Ld, class Prod, class Close>
__device__ __forceinline__ void seg_stream(uint32_t P, uint32_t Q, const uint32_t* __restrict__ bm,
                                           int32_t& ord, float& carry, bool& had, Ld ld,
                                           Prod prod, Close close) {
  static_assert(E == 4 || E == 8, "4 or 8 slots per lane");
  constexpr uint32_t TILE = 32 * E;
  constexpr uint32_t EM = (1u << E) - 1u;
  if (P >= Q) return;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint32_t base = P & ~uint32_t(E - 1);
  auto fetch = [&](uint32_t t, Win& w, uint32_t& m) {
    uint32_t s = t + E * lane;
    s = s < Q ? s : base;  // past the range: re-read a live line (no new traffic)
    w = ld(s);
    m = __ldg(bm + (s >> 5));
  };
  auto tile = [&](uint32_t t, Win& w, uint32_t& m) {
    float p[E];
    prod(w, p);
    const uint32_t s0 = t + E * lane;
    uint32_t hd = (m >> (s0 & 31u)) & EM;  // head bits of the lane's slots
    fetch(t + TILE * NB, w, m);
    if (!(t >= P && t + TILE <= Q)) {  // warp-uniform: first / last tile only
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const bool in = s0 + u >= P && s0 + u < Q;
        p[u] = in ? p[u] : 0.f;
        hd = in ? hd : (hd & ~(1u << u));
      }
    }
    const uint32_t H = __ballot_sync(kFull, hd != 0u);
    const bool multi = __any_sync(kFull, (hd & (hd - 1u)) != 0u);
    float pre = 0.f, post = 0.f;
    int32_t hb;
    int32_t heads;
    if (!multi) {  // at most one head per lane (segments of >= E slots)
      const int u0 = hd ? __ffs(hd) - 1 : E;
#pragma unroll
      for (int u = 0; u < E; ++u) {
        if (u < u0) pre += p[u];
        else post += p[u];
      }
      hb = __popc(H & lt);
      heads = __popc(H);
    } else {  // short segments: several heads in a lane
      hb = 0;
      heads = 0;
#pragma unroll
      for (int u = 0; u < E; ++u) {
        const uint32_t B = __ballot_sync(kFull, (hd >> u) & 1u);
        hb += __popc(B & lt);
        heads += __popc(B);
      }
      float run = 0.f;
      int seen = 0;
#pragma unroll
      for (int u = 0; u < E; ++u) {
        if ((hd >> u) & 1u) {
          if (seen) close(ord + hb + seen, run, false);  // began at this lane's previous head
          else pre = run;
          run = 0.f;
          ++seen;
        }
        run += p[u];
      }
      if (seen) post = run;
      else pre = run;
    }
    // Segmented inclusive scan of the lanes' open sums; a lane with a head
    // starts a new segment, the carried sum enters at lane 0.
    float v = hd ? post : pre;
    if (lane == 0 && !hd) v += carry;
    const uint32_t Hle = H & (lt | (1u << lane));
    const int src = Hle ? 31 - __clz(Hle) : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float o = __shfl_up_sync(kFull, v, off);
      if (lane - off >= src) v += o;
    }
    float excl = __shfl_up_sync(kFull, v, 1);
    if (lane == 0) excl = carry;
    if (hd) close(ord + hb, excl + pre, !had && lane == __ffs(H) - 1);
    carry = __shfl_sync(kFull, v, 31);
    had = had || H != 0u;
    ord += heads;
  };
  uint32_t t = base;
  Win wb[NB];
  uint32_t mb[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) fetch(t + TILE * k, wb[k], mb[k]);
  while (true) {
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      tile(t, wb[k], mb[k]);
      t += TILE;
      if (t >= Q) return;
    }
  }
}

struct CtaScratch {
  float pl[kNW], pf[kNW];
  int32_t pf_ord[kNW];
  int32_t had[kNW], has_pf[kNW];
  int32_t last;
};

// The CTA's slots [S0, S1) (S0 a segment start, S1 the next CTA's start):
// split evenly over the warps (E-slot aligned), streamed, and the segments
// cut between warps finished in slot order. emit(X, z) receives every
// complete segment once.
// emit(X, z) receives the segments the warps complete inside their streams
// (each warp's are the consecutive ordinals [lo, hi) reported to
// warp_done(lo, hi), called by every lane of the warp as soon as its stream
// ends, before the CTA barrier); emit_final(X, z) the segments assembled
// after the barrier (cut between warps, or closed by the CTA end).
template <int E, int NB, class Win, class Ld, class Prod, class Emit, class EmitFinal, class WarpDone>
__device__ __forceinline__ void cta_segments(uint32_t S0, uint32_t S1, const uint32_t* __restrict__ bm,
                                             const uint32_t* __restrict__ bpre, Ld ld, Prod prod,
                                             Emit emit, EmitFinal emit_final, WarpDone warp_done,
                                             CtaScratch& sc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  auto split = [&](int k) -> uint32_t {
    if (k <= 0) return S0;
    if (k >= kNW) return S1;
    const uint32_t s = static_cast<uint32_t>(S0 + (uint64_t(S1 - S0) * k) / kNW) & ~uint32_t(E - 1);
    return max(s, S0);
  };
  const uint32_t P = split(w), Q = split(w + 1);
  if (lane == 0) sc.has_pf[w] = 0;
  __syncwarp();
  // Ordinal of the CTA's first segment: closings of lower ordinals (the
  // segment ending at S0 - 1) belong to the previous CTA and are dropped.
  const int32_t xmin = S1 > S0 ? heads_before(bm, bpre, S0) : 0;
  const int32_t ord0 = S1 > S0 ? heads_before(bm, bpre, P) - 1 : 0;
  int32_t ord = ord0;
  float carry = 0.f;
  bool had = false;
  seg_stream<E, NB, Win>(P, Q, bm, ord, carry, had, ld, prod, [&](int32_t X, float z, bool first) {
    if (X < xmin) return;
    if (!first) {
      emit(X, z);
    } else {
      sc.pf[w] = z;
      sc.pf_ord[w] = X;
      sc.has_pf[w] = 1;
    }
  });
  __syncwarp();
  // The warp's first closing (ordinal ord0) is a piece; the rest are whole.
  warp_done(had ? ord0 + 1 : ord, ord);
  if (lane == 0) {
    sc.pl[w] = carry;
    sc.had[w] = had;
    if (w == kNW - 1 && S1 > S0) {  // the CTA end closes the open segment
      if (had) {
        emit_final(ord, carry);
      } else {
        sc.pf[w] = carry;
        sc.pf_ord[w] = ord;
        sc.has_pf[w] = 1;
      }
    }
  }
  __syncthreads();
  // Segments cut between warps: the pieces in slot order — from the last
  // warp before t that saw a head (its piece starts there), through the
  // head-free warps, to warp t's piece up to its first closing.
  if (threadIdx.x > 0 && threadIdx.x < kNW && sc.has_pf[threadIdx.x]) {
    const int t = threadIdx.x;
    int v0 = t - 1;
    while (v0 > 0 && !sc.had[v0]) --v0;
    float z = 0.f;
    for (int v = v0; v < t; ++v) z += sc.pl[v];
    emit_final(sc.pf_ord[t], z + sc.pf[t]);
  }
}

// E = 8 slots per lane: two float4 of values + eight ids.
struct WinR16 {
  float4 v0, v1;
  uint4 j;  // eight u16
};
struct WinC {
  float4 v0, v1;
  uint4 r;  // eight u16 block-local rows
};
constexpr int kE = 8;

// K2s: margins and coefficients c = coef(z, y) of all local rows
// (glm.cpp:30-34). The stream emits each row's margin z in place; each warp
// then turns its own (consecutive) rows into coefficients with coalesced
// label loads while the CTA's other warps still stream — no label load on
// the stream's emission path; rows finished after the CTA barrier (cut
// between warps) get their coefficient directly. One CTA per SM; the fp32
// model is bulk-copied (1-D TMA) into SMEM (models too large for SMEM take
// the column-blocked margin pass K2w instead, so d < 65,536 here and the
// column ids are 16-bit).
struct K2sArgs {
  const float* val;
  const uint16_t* idx;
  const uint32_t* bm;
  const uint32_t* bpre;
  const uint32_t* cta_slot;
  const uint32_t* row_of_ord;  // RMAP only
  const float* y;
  uint32_t n;
  const float* w32;
  uint32_t d;
  float* coef;
};

template <int TASK, bool RMAP>  // RMAP: empty rows, ordinals map through row_of_ord
__device__ __forceinline__ void k2s_phase(const K2sArgs& a, float* ws, CtaScratch& sc, uint64_t* bar) {
  // PDL: launched while the previous step drains. The CSR stream is static
  // data, so every warp issues its first tiles' loads at once; only the model
  // (and the coefficients this pass overwrites) belong to the previous step:
  // thread 0 waits for it before bulk-copying the model, and the first
  // product of every warp waits for that copy (or, with the model in global
  // memory, for the previous step itself). Coefficient writes all come after
  // a warp's first product, hence after the wait.
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pdl_wait();
    const uint32_t total = round_up16(uint64_t(a.d + 1) * 4);  // w32 holds whole 16-byte groups
    mbar_arrive_expect_tx(bar, total);
    for (uint32_t off = 0; off < total; off += 32768)
      bulk_g2s(reinterpret_cast<char*>(ws) + off, reinterpret_cast<const char*>(a.w32) + off,
               min(32768u, total - off), bar);
  }
  const uint32_t S0 = __ldg(a.cta_slot + blockIdx.x), S1 = __ldg(a.cta_slot + blockIdx.x + 1);
  bool ready = false;  // the first tiles' loads overlap the wait and the model's bulk copy
  using Win = WinR16;
  const float* __restrict__ y = a.y;
  const uint32_t* __restrict__ row_of_ord = a.row_of_ord;
  float* __restrict__ coef = a.coef;
  cta_segments<kE, 2, Win>(
      S0, S1, a.bm, a.bpre,
      [&](uint32_t s) {
        Win q;
        ldg256(a.val + s, q.v0, q.v1);
        q.j = __ldg(reinterpret_cast<const uint4*>(a.idx + s));
        return q;
      },
      [&](const Win& q, float* p) {
        if (!ready) {
          mbar_wait(bar, 0);
          ready = true;
        }
        uint32_t j[8];
        j[0] = q.j.x & 0xffffu, j[1] = q.j.x >> 16, j[2] = q.j.y & 0xffffu, j[3] = q.j.y >> 16;
        j[4] = q.j.z & 0xffffu, j[5] = q.j.z >> 16, j[6] = q.j.w & 0xffffu, j[7] = q.j.w >> 16;
        const float x[8] = {q.v0.x, q.v0.y, q.v0.z, q.v0.w, q.v1.x, q.v1.y, q.v1.z, q.v1.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          SGDB_CHECK(j[u] <= a.d);
          p[u] = x[u] * ws[j[u]];
        }
      },
      [&](int32_t X, float z) {
        SGDB_CHECK(X >= 0 && (RMAP || static_cast<uint32_t>(X) < a.n));
        coef[RMAP ? __ldg(row_of_ord + X) : static_cast<uint32_t>(X)] = z;
      },
      [&](int32_t X, float z) {
        const uint32_t r = RMAP ? __ldg(row_of_ord + X) : static_cast<uint32_t>(X);
        SGDB_CHECK(r < a.n);
        coef[r] = coef_fast<TASK>(z, __ldg(y + r));
      },
      [&](int32_t lo, int32_t hi) {
        // The warp's own rows turn their margins into coefficients while the
        // CTA's other warps still stream (coalesced, all loads in flight).
        for (int32_t o0 = lo + (threadIdx.x & 31); o0 < hi; o0 += 32 * 4) {
          uint32_t r[4];
          float z[4], yy[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int32_t o = o0 + 32 * i;
            r[i] = o < hi ? (RMAP ? __ldg(row_of_ord + o) : static_cast<uint32_t>(o)) : 0u;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            z[i] = coef[r[i]];
            yy[i] = __ldg(y + r[i]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (o0 + 32 * i < hi) coef[r[i]] = coef_fast<TASK>(z[i], yy[i]);
        }
      },
      sc);
  if (!ready && threadIdx.x == 0) mbar_wait(bar, 0);  // the bulk copy must land before exit
}

template <int TASK, bool RMAP>
__global__ void __launch_bounds__(kNT, 1) k2s_margin_kernel(K2sArgs a) {
  extern __shared__ __align__(16) float ws[];
  __shared__ CtaScratch sc;
  __shared__ uint64_t bar;
  k2s_phase<TASK, RMAP>(a, ws, sc, &bar);
}

struct ApplyArgs {
  double alpha;
  int apply, want_norm;
  double* w64;
  float* w32;
  double* g64;
  int* finite;
  double* norm2;
};

struct PassArgs {
  const float* val;
  const uint16_t* id;
  const uint32_t* bm;
  const uint32_t* bpre;
  const uint32_t* segptr;
  const uint32_t* cta;
  uint32_t cpb, nblk, nminor, rb, nmajor;
  const float* slice;           // gradient: the coefficients; margin: the fp32 model
  const uint32_t* ord_of_seg;   // SMAP only: ordinal of segment q = exclusive count of non-empty segments
  float* part;                  // partial sums: nblk * nminor, or (SMAP) one per non-empty segment
  unsigned* tickets;
  unsigned gen;
  int coop;
  ApplyArgs aa;                 // gradient pass: the update
  const float* y;               // margin pass: labels -> coefficients
  float* coef;
};

constexpr int kPassGrad = 0;
constexpr int kPassMargin = 1;

// One blocked segmented pass (Blocked in device.hpp). CTA (major block b,
// minor range k) bulk-copies the block's slice of the operand into SMEM
// (gradient pass: the coefficients of rows [b*rb, ..); margin pass of a wide
// model: the model's columns [b*rb, ..)), streams the block's segments of
// minor indices [cta[k], cta[k+1]) against it and writes fp32
// per-(block, minor) sums. Then, per minor index, the sum over blocks in
// fixed block order (fp64):
//   K3s, gradient pass: g_j, w -= alpha g (or g64 = g), finite flag, |g|^2;
//   K2w, margin pass:   z_i, coef_i = coef(z_i, y_i) (glm.cpp:30-34).
// The finish is spread over the minor range's nblk CTAs once all of them
// have arrived (coop: at most one CTA per SM and no more CTAs than SMs, so
// every CTA is resident once the previous pass drains and the arrival wait
// cannot deadlock); otherwise the last CTA to arrive finishes the whole
// range. Arrival tickets count up by nblk per launch (gen = launch number),
// so they are never reset. SMAP: some segments are empty; the partials are
// stored compactly by segment ordinal (the stream's emission index, no
// lookup on the hot path) and the finish finds segment q's through
// ord_of_seg (empty segments contribute 0).
// GLUED (the one-launch epoch, K23g): the slice's coefficients come from the
// margin phase of other CTAs of the same launch; thread 0 acquires block b's
// ready count (every margin CTA holding rows of the block has released it)
// instead of waiting for a previous grid, then orders the async-proxy bulk
// copy after that acquire.
template <int MODE, int TASK, bool SMAP, bool GLUED>
__device__ __forceinline__ void blocked_phase(const PassArgs& p, uint32_t item, float* cs, CtaScratch& sc,
                                              uint64_t* bar, const unsigned* blk_ready, const unsigned* blk_expect) {
  const uint32_t b = item / p.cpb, k = item % p.cpb;
  SGDB_CHECK(b < p.nblk && b * p.rb < p.nmajor);
  const uint32_t r0 = b * p.rb, len = min(p.rb, p.nmajor - r0);  // rb % 8 == 0: 32-byte aligned slice
  // PDL: the blocked stream is static, so the first tiles' loads go out
  // while the previous pass drains; thread 0 waits for it before
  // bulk-copying the slice, and every warp's first product waits for that.
  if (!GLUED) pdl_launch_dependents();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  const uint32_t j0 = __ldg(p.cta + k), j1 = __ldg(p.cta + k + 1);
  const uint64_t q0 = uint64_t(b) * p.nminor;
  __syncthreads();  // the barrier init is visible to every waiter
  if (threadIdx.x == 0) {
    if (GLUED) {
      const unsigned target = p.gen * __ldg(blk_expect + b);
      SGDB_CHECK(__ldg(blk_expect + b) > 0);
      while (ld_acquire_gpu(blk_ready + b) < target) {
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
    } else {
      pdl_wait();  // the slice comes from the previous pass
    }
    const uint32_t total = round_up16(uint64_t(len) * 4);  // both operands carry 16-byte slack
    mbar_arrive_expect_tx(bar, total);
    for (uint32_t off = 0; off < total; off += 32768)
      bulk_g2s(reinterpret_cast<char*>(cs) + off, reinterpret_cast<const char*>(p.slice + r0) + off,
               min(32768u, total - off), bar);
  }
  const uint32_t S0 = __ldg(p.segptr + q0 + j0), S1 = __ldg(p.segptr + q0 + j1);
  if (MODE == kPassGrad && p.coop && threadIdx.x == 32) {
    // The finish's operands head for L2 while the stream runs: this CTA's
    // share of the fp64 master (read-modify-written per index there) and,
    // with empty segments, the ordinal map of its indices (L2-flushed between
    // epochs, they would otherwise cost an HBM round trip per finish round;
    // news20's gradient finish 41 -> 37 us). The margin pass (K2w, 28 column
    // blocks of ordinals per index) measured slower with the same prefetch.
    const uint32_t f0 = j0 + static_cast<uint32_t>(uint64_t(j1 - j0) * b / p.nblk);
    const uint32_t f1 = j0 + static_cast<uint32_t>(uint64_t(j1 - j0) * (b + 1) / p.nblk);
    if (p.aa.apply && f1 > f0) {
      const uint64_t lo = uint64_t(f0) & ~uint64_t(1), hi = (uint64_t(f1) + 1) & ~uint64_t(1);  // 16-byte units
      for (uint64_t x = lo; x < hi; x += 4096)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.aa.w64 + x),
                     "r"(static_cast<uint32_t>(min(uint64_t(4096), hi - x) * 8)) : "memory");
    }
    if (SMAP) {
      for (uint32_t bb = 0; bb < p.nblk; ++bb) {
        const uint64_t lo = (uint64_t(bb) * p.nminor + f0) & ~uint64_t(3);
        const uint64_t hi = (uint64_t(bb) * p.nminor + f1 + 1 + 3) & ~uint64_t(3);
        for (uint64_t x = lo; x < hi; x += 8192)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.ord_of_seg + x),
                       "r"(static_cast<uint32_t>(min(uint64_t(8192), hi - x) * 4)) : "memory");
      }
    }
  }
  bool ready = false;  // the first tiles' loads overlap the slice's bulk copy
  float* __restrict__ part = p.part;
  cta_segments<kE, 2, WinC>(
      S0, S1, p.bm, p.bpre,
      [&](uint32_t s) {
        WinC q;
        ldg256(p.val + s, q.v0, q.v1);
        q.r = __ldg(reinterpret_cast<const uint4*>(p.id + s));
        return q;
      },
      [&](const WinC& q, float* pr) {
        if (!ready) {
          mbar_wait(bar, 0);
          ready = true;
        }
        // Inside the staged slice's SMEM (rb entries). Slots outside the
        // warp's range (re-read windows, masked after the product) may carry
        // another block's ids, so the bound is rb, not this block's len.
        SGDB_CHECK((q.r.x & 0xffffu) < p.rb && (q.r.x >> 16) < p.rb && (q.r.y & 0xffffu) < p.rb &&
                   (q.r.y >> 16) < p.rb && (q.r.z & 0xffffu) < p.rb && (q.r.z >> 16) < p.rb &&
                   (q.r.w & 0xffffu) < p.rb && (q.r.w >> 16) < p.rb);
        pr[0] = q.v0.x * cs[q.r.x & 0xffffu], pr[1] = q.v0.y * cs[q.r.x >> 16];
        pr[2] = q.v0.z * cs[q.r.y & 0xffffu], pr[3] = q.v0.w * cs[q.r.y >> 16];
        pr[4] = q.v1.x * cs[q.r.z & 0xffffu], pr[5] = q.v1.y * cs[q.r.z >> 16];
        pr[6] = q.v1.z * cs[q.r.w & 0xffffu], pr[7] = q.v1.w * cs[q.r.w >> 16];
      },
      [&](int32_t X, float z) {
        SGDB_CHECK(X >= 0 && uint64_t(X) < uint64_t(p.nblk) * p.nminor);
        part[static_cast<uint32_t>(X)] = z;
      },
      [&](int32_t X, float z) {
        SGDB_CHECK(X >= 0 && uint64_t(X) < uint64_t(p.nblk) * p.nminor);
        part[static_cast<uint32_t>(X)] = z;
      },
      [&](int32_t, int32_t) {},
      sc);
  if (!ready && threadIdx.x == 0) mbar_wait(bar, 0);  // the bulk copy must land before exit
  __syncthreads();
  const unsigned target = p.gen * p.nblk;
  if (threadIdx.x == 0) {
    const unsigned t = atom_add_acq_rel_gpu(p.tickets + k, 1u) + 1u;
    sc.last = t == target;
    if (p.coop)
      while (ld_acquire_gpu(p.tickets + k) < target) __nanosleep(32);
  }
  __syncthreads();
  uint32_t a0 = j0, a1 = j1;  // the minor indices this CTA finishes
  if (p.coop) {
    a0 = j0 + static_cast<uint32_t>(uint64_t(j1 - j0) * b / p.nblk);
    a1 = j0 + static_cast<uint32_t>(uint64_t(j1 - j0) * (b + 1) / p.nblk);
  } else if (!sc.last) {
    return;
  }
  __threadfence();
  double nrm = 0.0;
  int bad = 0;
  for (uint32_t j = a0 + threadIdx.x; j < a1; j += kNT) {
    // The master's old value loads alongside the partials (not after them).
    const double wold = MODE == kPassGrad && p.aa.apply ? __ldcg(p.aa.w64 + j) : 0.0;
    // Block order; 8 loads in flight per thread.
    double g = 0.0;
    uint32_t bb = 0;
    // Segment (b, j)'s partial: at b*nminor + j, or (SMAP) at its ordinal
    // when the segment is non-empty.
    auto partial = [&](uint32_t b2) -> float {
      const uint64_t q = uint64_t(b2) * p.nminor + j;
      if (!SMAP) return __ldcg(part + q);
      const uint32_t o0 = __ldg(p.ord_of_seg + q), o1 = __ldg(p.ord_of_seg + q + 1);
      return o1 > o0 ? __ldcg(part + o0) : 0.f;
    };
    for (; bb + 8 <= p.nblk; bb += 8) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = partial(bb + i);
#pragma unroll
      for (int i = 0; i < 8; ++i) g += static_cast<double>(v[i]);
    }
    for (; bb < p.nblk; ++bb) g += static_cast<double>(partial(bb));
    if (MODE == kPassMargin) {
      p.coef[j] = coef_fast<TASK>(static_cast<float>(g), __ldg(p.y + j));
      continue;
    }
    if (!isfinite(g)) bad = 1;
    if (p.aa.apply) {
      const double wn = wold - p.aa.alpha * g;
      p.aa.w64[j] = wn;
      p.aa.w32[j] = static_cast<float>(wn);
    } else {
      p.aa.g64[j] = g;
    }
    nrm += g * g;
  }
  if (MODE == kPassGrad) {
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) *p.aa.finite = 0;
    if (p.aa.want_norm) {
      nrm = warp_sum_d(nrm);
      if ((threadIdx.x & 31) == 0 && nrm != 0.0) atomicAdd(p.aa.norm2, nrm);
    }
  }
}

template <int MODE, int TASK, bool SMAP>
__global__ void __launch_bounds__(kNT, 1) blocked_pass_kernel(PassArgs p) {
  extern __shared__ __align__(16) float cs[];
  __shared__ CtaScratch sc;
  __shared__ uint64_t bar;
  blocked_phase<MODE, TASK, SMAP, false>(p, blockIdx.x, cs, sc, &bar, nullptr, nullptr);
}

// K23g: the whole full-batch step in ONE launch when the model fits in SMEM:
// CTA x runs K2s's slot range x, releases the row blocks its rows belong to
// (blk_ready, monotonic: gen launches), then runs K3s's work item x once
// every margin CTA of that item's row block has released it. Same streams,
// same sums, same order as K2s -> K3s; no kernel boundary between them (the
// dynamic SMEM holds the model, then the coefficient slice). Every CTA must
// be resident: grid = SMs, one CTA per SM.
template <int TASK, bool RMAP, bool SMAP>
__global__ void __launch_bounds__(kNT, 1)
    glued_step_kernel(K2sArgs ka, PassArgs pa, const uint32_t* cta_row, uint32_t rb, unsigned* blk_ready,
                      const unsigned* blk_expect) {
  extern __shared__ __align__(16) float smem[];
  __shared__ CtaScratch sc;
  __shared__ uint64_t bar_a, bar_b;
  k2s_phase<TASK, RMAP>(ka, smem, sc, &bar_a);
  __syncthreads();  // every coefficient of this CTA's rows is written
  if (threadIdx.x == 0) {
    const uint32_t r0 = __ldg(cta_row + blockIdx.x), r1 = __ldg(cta_row + blockIdx.x + 1);
    if (r1 > r0)
      for (uint32_t bb = r0 / rb; bb <= (r1 - 1) / rb; ++bb) {
        SGDB_CHECK(bb < pa.nblk);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(blk_ready + bb) : "memory");
      }
  }
  if (blockIdx.x < pa.nblk * pa.cpb)
    blocked_phase<kPassGrad, TASK, SMAP, true>(pa, blockIdx.x, smem, sc, &bar_b, blk_ready, blk_expect);
}

// ---- preparation (once per upload / refresh) ---------------------------------

__global__ void row_heads_kernel(const uint32_t* __restrict__ rowptr, uint32_t n, uint32_t* bm,
                                 uint32_t* nonempty, unsigned* n_empty) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t s = rowptr[r], e = rowptr[r + 1];
  const bool ne = e > s;
  nonempty[r] = ne ? 1u : 0u;
  if (ne) atomicOr(bm + (s >> 5), 1u << (s & 31u));
  else atomicAdd(n_empty, 1u);
}

__global__ void popc_kernel(const uint32_t* __restrict__ bm, uint64_t nwords, uint32_t* out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nwords) out[i] = __popc(bm[i]);
  else if (i == nwords) out[i] = 0u;
}

// dst[pos[i]] = i where flag[i] (pos = exclusive prefix of flag).
__global__ void compact_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                               uint64_t count, uint32_t* dst) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count && flag[i]) dst[pos[i]] = static_cast<uint32_t>(i);
}

// CTA k of the margin pass starts at the first row starting at or after
// k*nnz/nc (a slot position).
__global__ void cta_slot_kernel(const uint32_t* __restrict__ rowptr, uint32_t n, uint32_t nc,
                                uint32_t* cta_slot, uint32_t* cta_row) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nc) return;
  const uint64_t nnz = rowptr[n];
  if (k == nc) {
    cta_slot[k] = static_cast<uint32_t>(nnz);
    cta_row[k] = n;
    return;
  }
  const uint32_t target = static_cast<uint32_t>(nnz * k / nc);
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (rowptr[mid] >= target) hi = mid;
    else lo = mid + 1;
  }
  cta_slot[k] = rowptr[lo];
  cta_row[k] = lo;
}

// K23g: how many margin CTAs hold rows of each row block (x's rows are
// [cta_row[x], cta_row[x+1])).
__global__ void blk_expect_kernel(const uint32_t* __restrict__ cta_row, uint32_t nc, uint32_t rb,
                                  unsigned* expect) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nc) return;
  const uint32_t r0 = cta_row[x], r1 = cta_row[x + 1];
  if (r1 > r0)
    for (uint32_t b = r0 / rb; b <= (r1 - 1) / rb; ++b) atomicAdd(expect + b, 1u);
}

__global__ void narrow_u16_kernel(const uint32_t* __restrict__ src, uint64_t n, uint16_t* dst) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = static_cast<uint16_t>(src[i]);
}

// Sort keys and payloads of every nonzero (row r, column j), warp per row:
// by rows (the CSC): key = (r / rb) * d + j, payload = value bits << 16 | r % rb;
// by columns (the wide margin pass): key = (j / rb) * n + r, payload = value
// bits << 16 | j % rb.
template <bool BY_COL>
__global__ void blocked_keys_kernel(const float* __restrict__ val, const uint32_t* __restrict__ idx,
                                    const uint32_t* __restrict__ rowptr, uint32_t n, uint32_t d,
                                    uint32_t rb, uint32_t* keys, uint64_t* pay) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const uint32_t b = static_cast<uint32_t>(r / rb), lr = static_cast<uint32_t>(r - uint64_t(b) * rb);
    const uint32_t s1 = rowptr[r + 1];
    for (uint32_t s = rowptr[r] + lane; s < s1; s += 32) {
      const uint32_t j = idx[s];
      const uint64_t v = uint64_t(__float_as_uint(val[s])) << 16;
      if (BY_COL) {
        const uint32_t jb = j / rb;
        keys[s] = jb * n + static_cast<uint32_t>(r);
        pay[s] = v | (j - jb * rb);
      } else {
        keys[s] = b * d + j;
        pay[s] = v | lr;
      }
    }
  }
}

// Unpack the sorted payloads, write the CSC head bitmap (one ballot per 32
// slots) and the segment pointers (segptr[q] = first slot of key >= q).
__global__ void blocked_unpack_kernel(const uint32_t* __restrict__ keys, const uint64_t* __restrict__ pay,
                                      uint32_t nnz, uint32_t nseg, float* cval, uint16_t* crow,
                                      uint32_t* bm, uint32_t* segptr) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t total = (uint64_t(nnz) + 32) & ~uint64_t(31);  // whole warps, one past the end
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    bool head = false;
    if (i < nnz) {
      const uint64_t p = pay[i];
      cval[i] = __uint_as_float(static_cast<uint32_t>(p >> 16));
      crow[i] = static_cast<uint16_t>(p & 0xffffu);
      const uint32_t key = keys[i];
      const uint32_t prev = i ? keys[i - 1] : 0u;
      head = i == 0 || key != prev;
      if (head)
        for (uint32_t q = i ? prev + 1 : 0u; q <= key; ++q) segptr[q] = static_cast<uint32_t>(i);
    } else if (i == nnz) {
      for (uint32_t q = nnz ? keys[nnz - 1] + 1 : 0u; q <= nseg; ++q) segptr[q] = nnz;
    }
    const uint32_t word = __ballot_sync(kFull, head);
    if ((threadIdx.x & 31) == 0) bm[i >> 5] = word;
  }
}

__global__ void seg_nonempty_kernel(const uint32_t* __restrict__ segptr, uint32_t nseg, uint32_t* flag,
                                    unsigned* n_empty) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nseg) return;
  const bool ne = segptr[q + 1] > segptr[q];
  flag[q] = ne ? 1u : 0u;
  if (!ne) atomicAdd(n_empty, 1u);
}

// Column totals over the row blocks (for nnz-balanced column ranges).
__global__ void minor_count_kernel(const uint32_t* __restrict__ segptr, uint32_t d, uint32_t nblk,
                                   uint32_t* cnt) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  uint32_t c = 0;
  for (uint32_t b = 0; b < nblk; ++b) c += segptr[uint64_t(b) * d + j + 1] - segptr[uint64_t(b) * d + j];
  cnt[j] = c;
}

// cta_col[k] = first minor index whose inclusive count prefix exceeds k*nnz/cpb.
__global__ void cta_minor_kernel(const uint32_t* __restrict__ incl, uint32_t d, uint32_t cpb,
                                 uint64_t nnz, uint32_t* cta_col) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > cpb) return;
  if (k == 0 || k == cpb) {
    cta_col[k] = k == 0 ? 0u : d;
    return;
  }
  const uint64_t target = nnz * k / cpb;
  uint32_t lo = 0, hi = d;  // first j with incl[j] > target
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (incl[mid] > target) hi = mid;
    else lo = mid + 1;
  }
  cta_col[k] = lo;
}

unsigned grid_1d(uint64_t n, unsigned threads = 256) {
  return static_cast<unsigned>(std::max<uint64_t>(1, (n + threads - 1) / threads));
}

// Exclusive prefix (nwords + 1 entries) of the popcounts of bitmap words.
void word_prefix(Ctx& c, const uint32_t* bm, uint64_t nwords, DBuf<uint32_t>& pre, DBuf<unsigned char>& tmp,
                 DBuf<uint32_t>& cnt) {
  cnt.alloc(nwords + 1);
  pre.alloc(nwords + 1);
  prof_begin(c, "sparse_prep_kernel");
  popc_kernel<<<grid_1d(nwords + 1), 256, 0, c.stream>>>(bm, nwords, cnt.p);
  launched(c, "sparse_prep_kernel");
  size_t bytes = 0;
  check(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, pre.p, static_cast<int64_t>(nwords + 1), c.stream),
        "cub scan size");
  tmp.alloc(bytes);
  bytes = tmp.n;
  check(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, pre.p, static_cast<int64_t>(nwords + 1), c.stream),
        "cub scan");
}

// Compaction map of the set flags (count entries), exclusive-scan based.
void compaction(Ctx& c, const uint32_t* flag, uint64_t count, DBuf<uint32_t>& map, DBuf<unsigned char>& tmp,
                DBuf<uint32_t>& pos) {
  pos.alloc(count + 1);
  size_t bytes = 0;
  check(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag, pos.p, static_cast<int64_t>(count), c.stream),
        "cub scan size");
  tmp.alloc(bytes);
  bytes = tmp.n;
  check(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, flag, pos.p, static_cast<int64_t>(count), c.stream),
        "cub scan");
  map.alloc(std::max<uint64_t>(1, count));
  prof_begin(c, "sparse_prep_kernel");
  compact_kernel<<<grid_1d(count), 256, 0, c.stream>>>(flag, pos.p, count, map.p);
  launched(c, "sparse_prep_kernel");
}

// Row-block geometry: blocks of at most 49,152 rows (u16 ids, <= 192 KB
// slice), and as many CTAs (blocks x column ranges) as SMs, one per SM.
void choose_blocks(const Ctx& c, uint64_t n, uint32_t& rb, uint32_t& nblk, uint32_t& cpb) {
  // Blocks of at most 49,152 rows (16-bit ids, <= 192 KB slice). From the
  // fewest such blocks up to twice as many, the count whose grid
  // nblk * floor(SMs / nblk) leaves the fewest SMs idle (ties: fewer blocks —
  // more blocks add nblk * d partial sums to the apply). rcv1: 21 blocks x 7
  // column ranges = 147 CTAs instead of 14 x 10 = 140.
  const uint64_t nb0 = std::max<uint64_t>(1, (n + kMaxRowBlock - 1) / kMaxRowBlock);
  const uint64_t sms = static_cast<uint64_t>(std::max(1, c.num_sms));
  uint64_t nb = nb0, best = 0;
  for (uint64_t k = nb0; k <= std::min<uint64_t>(2 * nb0, sms); ++k) {
    const uint64_t used = k * (sms / k);
    if (used > best) best = used, nb = k;
  }
  // rb % 8 == 0 keeps every coefficient slice 32-byte aligned (bulk copies).
  rb = static_cast<uint32_t>(std::max<uint64_t>(8, ((n + nb - 1) / nb + 7) & ~uint64_t(7)));
  nblk = static_cast<uint32_t>(std::max<uint64_t>(1, (n + rb - 1) / rb));
  cpb = static_cast<uint32_t>(std::max<uint64_t>(1, sms / nblk));
}

// The blocked segmented copy (see Blocked in device.hpp) by a stable radix
// sort of (block, minor) keys: within a segment the major ids stay ascending
// (deterministic sums). by_col: major = columns (the wide margin pass).
void build_blocked(Dataset& ds, bool by_col, Blocked& B) {
  Ctx& c = *ds.ctx;
  cudaStream_t s = c.stream;
  auto& sp = ds.prep;
  const uint64_t n = ds.n, d = ds.d, nnz = ds.nnz;
  const uint64_t nmajor = by_col ? d : n, nminor = by_col ? n : d;
  choose_blocks(c, nmajor, B.rb, B.nblk, B.cpb);
  const uint64_t nseg = uint64_t(B.nblk) * nminor;
  if (nseg >= (uint64_t(1) << 31))
    throw Unsupported("full-batch sparse step: (blocks x minor) segments must fit 31 bits");
  const uint64_t nwords = (nnz + 256) / 32 + 2;
  B.val.alloc(nnz + 1024);
  B.id.alloc(nnz + 1024);
  check(cudaMemsetAsync(B.val.p + nnz, 0, 1024 * sizeof(float), s), "memset");
  check(cudaMemsetAsync(B.id.p + nnz, 0, 1024 * sizeof(uint16_t), s), "memset");
  B.segptr.alloc(nseg + 1);
  B.bm.alloc(nwords);
  B.bm.zero(s);
  if (nnz > 0) {
    sp.k_in.alloc(nnz);
    sp.k_out.alloc(nnz);
    sp.p_in.alloc(nnz);
    sp.p_out.alloc(nnz);
    prof_begin(c, "sparse_prep_kernel");
    auto keys = by_col ? blocked_keys_kernel<true> : blocked_keys_kernel<false>;
    keys<<<c.num_sms * 8, 256, 0, s>>>(ds.val.p, ds.idx.p, ds.rowptr.p, static_cast<uint32_t>(n),
                                       static_cast<uint32_t>(d), B.rb, sp.k_in.p, sp.p_in.p);
    launched(c, "sparse_prep_kernel");
    int end_bit = 1;
    while (end_bit < 32 && (uint64_t(1) << end_bit) < nseg) ++end_bit;
    size_t bytes = 0;
    check(cub::DeviceRadixSort::SortPairs(nullptr, bytes, sp.k_in.p, sp.k_out.p, sp.p_in.p, sp.p_out.p,
                                          static_cast<int64_t>(nnz), 0, end_bit, s),
          "cub sort size");
    sp.tmp.alloc(bytes);
    bytes = sp.tmp.n;
    check(cub::DeviceRadixSort::SortPairs(sp.tmp.p, bytes, sp.k_in.p, sp.k_out.p, sp.p_in.p, sp.p_out.p,
                                          static_cast<int64_t>(nnz), 0, end_bit, s),
          "cub sort");
    prof_begin(c, "sparse_prep_kernel");
    blocked_unpack_kernel<<<c.num_sms * 8, 256, 0, s>>>(sp.k_out.p, sp.p_out.p, static_cast<uint32_t>(nnz),
                                                        static_cast<uint32_t>(nseg), B.val.p, B.id.p, B.bm.p,
                                                        B.segptr.p);
    launched(c, "sparse_prep_kernel");
  } else {
    B.segptr.zero(s);
  }
  word_prefix(c, B.bm.p, nwords, B.bm_pre, sp.tmp, sp.b);
  sp.c.alloc(nseg + 1);  // non-empty segment flags (+ a zero for the prefix's end)
  check(cudaMemsetAsync(sp.cnt.p + 1, 0, sizeof(unsigned), s), "memset");
  prof_begin(c, "sparse_prep_kernel");
  seg_nonempty_kernel<<<grid_1d(nseg), 256, 0, s>>>(B.segptr.p, static_cast<uint32_t>(nseg), sp.c.p,
                                                     sp.cnt.p + 1);
  launched(c, "sparse_prep_kernel");
  {  // nnz-balanced minor ranges, shared by every block
    sp.k_in.alloc(std::max<uint64_t>(1, nminor));  // per-minor counts (the sort keys are consumed)
    sp.b.alloc(std::max<uint64_t>(nwords + 1, nminor));
    prof_begin(c, "sparse_prep_kernel");
    minor_count_kernel<<<grid_1d(nminor), 256, 0, s>>>(B.segptr.p, static_cast<uint32_t>(nminor), B.nblk,
                                                        sp.k_in.p);
    launched(c, "sparse_prep_kernel");
    size_t bytes = 0;
    check(cub::DeviceScan::InclusiveSum(nullptr, bytes, sp.k_in.p, sp.b.p, static_cast<int64_t>(nminor), s),
          "cub scan size");
    sp.tmp.alloc(bytes);
    bytes = sp.tmp.n;
    check(cub::DeviceScan::InclusiveSum(sp.tmp.p, bytes, sp.k_in.p, sp.b.p, static_cast<int64_t>(nminor), s),
          "cub scan");
    B.cta.alloc(B.cpb + 1);
    prof_begin(c, "sparse_prep_kernel");
    cta_minor_kernel<<<grid_1d(B.cpb + 1), 256, 0, s>>>(sp.b.p, static_cast<uint32_t>(nminor), B.cpb, nnz,
                                                         B.cta.p);
    launched(c, "sparse_prep_kernel");
  }
  unsigned empty = 0;
  check(cudaMemcpyAsync(&empty, sp.cnt.p + 1, sizeof(empty), cudaMemcpyDeviceToHost, s), "D2H");
  check(cudaStreamSynchronize(s), "prep sync");
  B.segs_empty = empty != 0;
  if (B.segs_empty) {  // ord_of_seg: exclusive prefix of the non-empty flags (nseg + 1 entries)
    check(cudaMemsetAsync(sp.c.p + nseg, 0, sizeof(uint32_t), s), "memset");
    B.ord_of_seg.alloc(nseg + 4);  // + slack: whole 16-byte units for L2 bulk prefetches
    size_t bytes = 0;
    check(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sp.c.p, B.ord_of_seg.p, static_cast<int64_t>(nseg + 1), s),
          "cub scan size");
    sp.tmp.alloc(bytes);
    bytes = sp.tmp.n;
    check(cub::DeviceScan::ExclusiveSum(sp.tmp.p, bytes, sp.c.p, B.ord_of_seg.p, static_cast<int64_t>(nseg + 1), s),
          "cub scan");
  }
  B.tickets.alloc(B.cpb);
  B.tickets.zero(s);  // arrival counts restart with the launch numbers
  B.gen = 0;
}

}  // namespace

void sparse_prep(Dataset& ds) {
  if (ds.sparse_ready) return;
  Ctx& c = *ds.ctx;
  cudaStream_t s = c.stream;
  const uint64_t n = ds.n, d = ds.d, nnz = ds.nnz;
  if (n >= (uint64_t(1) << 31))
    throw Unsupported("full-batch sparse step: rows must fit 31 bits");
  auto& sp = ds.prep;
  sp.cnt.alloc(2);
  check(cudaMemsetAsync(sp.cnt.p, 0, 2 * sizeof(unsigned), s), "memset");
  const uint64_t nwords = (nnz + 256) / 32 + 2;
  // Row heads, 16-bit ids, margin CTA partition.
  ds.rbm.alloc(nwords);
  ds.rbm.zero(s);
  sp.a.alloc(std::max<uint64_t>(1, n));  // non-empty row flags
  prof_begin(c, "sparse_prep_kernel");
  row_heads_kernel<<<grid_1d(n), 256, 0, s>>>(ds.rowptr.p, static_cast<uint32_t>(n), ds.rbm.p, sp.a.p, sp.cnt.p);
  launched(c, "sparse_prep_kernel");
  word_prefix(c, ds.rbm.p, nwords, ds.rbm_pre, sp.tmp, sp.b);
  const size_t model_bytes = round_up16(uint64_t(d + 1) * 4);
  ds.wide = model_bytes + sizeof(CtaScratch) + 64 > c.max_smem_optin;
  if (!ds.wide) {  // K2s: the model fits in SMEM, so d < 65,536
    ds.cidx16.alloc(nnz + 1024);
    check(cudaMemsetAsync(ds.cidx16.p + nnz, 0, 1024 * sizeof(uint16_t), s), "memset");
    prof_begin(c, "sparse_prep_kernel");
    narrow_u16_kernel<<<c.num_sms * 8, 256, 0, s>>>(ds.idx.p, nnz, ds.cidx16.p);
    launched(c, "sparse_prep_kernel");
  }
  ds.cta_n = static_cast<uint32_t>(std::max(1, c.num_sms));
  ds.cta_slot.alloc(ds.cta_n + 1);
  ds.cta_row.alloc(ds.cta_n + 1);
  prof_begin(c, "sparse_prep_kernel");
  cta_slot_kernel<<<grid_1d(ds.cta_n + 1), 256, 0, s>>>(ds.rowptr.p, static_cast<uint32_t>(n), ds.cta_n,
                                                         ds.cta_slot.p, ds.cta_row.p);
  launched(c, "sparse_prep_kernel");

  build_blocked(ds, false, ds.csc);
  if (!ds.wide) {  // K23g's row-block readiness counts
    ds.blk_ready.alloc(ds.csc.nblk);
    ds.blk_ready.zero(s);
    ds.blk_expect.alloc(ds.csc.nblk);
    ds.blk_expect.zero(s);
    prof_begin(c, "sparse_prep_kernel");
    blk_expect_kernel<<<grid_1d(ds.cta_n), 256, 0, s>>>(ds.cta_row.p, ds.cta_n, ds.csc.rb, ds.blk_expect.p);
    launched(c, "sparse_prep_kernel");
  }
  // Models too large for shared memory: the margin pass runs blocked too.
  if (ds.wide) {
    build_blocked(ds, true, ds.wmajor);
    ds.mpart.alloc(uint64_t(ds.wmajor.nblk) * n + 1);
  }
  // One host read-back: are there empty rows (ordinal map needed)?
  unsigned empty = 0;
  check(cudaMemcpyAsync(&empty, sp.cnt.p, sizeof(empty), cudaMemcpyDeviceToHost, s), "D2H");
  check(cudaStreamSynchronize(s), "prep sync");
  ds.rows_empty = empty != 0;
  if (ds.rows_empty) compaction(c, sp.a.p, n, ds.row_of_ord, sp.tmp, sp.b);
  if (ds.coef.n < n + 8) {
    ds.coef.alloc(n + 8);
    ds.coef.zero(s);
  }
  ds.sparse_ready = true;
}

namespace {
// Launch one blocked pass over B (PDL unless the structures were just
// rebuilt by the previous kernels on the stream).
template <int MODE>
void launch_pass(Dataset& ds, Blocked& B, uint64_t nminor, uint64_t nmajor, const float* slice, float* part,
                 int task, const ApplyArgs& aa, bool pdl, const char* name) {
  Ctx& c = *ds.ctx;
  const size_t smem = round_up16(uint64_t(B.rb) * 4);
  void (*kern)(PassArgs);
  if (task == kTaskLR)
    kern = B.segs_empty ? blocked_pass_kernel<MODE, kTaskLR, true> : blocked_pass_kernel<MODE, kTaskLR, false>;
  else
    kern = B.segs_empty ? blocked_pass_kernel<MODE, kTaskSVM, true> : blocked_pass_kernel<MODE, kTaskSVM, false>;
  set_max_dyn_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(blocked_pass)");
  const unsigned grid = B.nblk * B.cpb;
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), kNT, smem);
  PassArgs p{B.val.p, B.id.p, B.bm.p, B.bm_pre.p, B.segptr.p, B.cta.p, B.cpb, B.nblk,
             static_cast<uint32_t>(nminor), B.rb, static_cast<uint32_t>(nmajor), slice,
             B.segs_empty ? B.ord_of_seg.p : nullptr, part, B.tickets.p, ++B.gen,
             // With one CTA per SM and grid <= SMs every CTA becomes resident
             // once the previous pass has drained: the arrival wait cannot deadlock.
             per_sm >= 1 && grid <= static_cast<unsigned>(c.num_sms) ? 1 : 0, aa, ds.labels.p, ds.coef.p};
  prof_begin(c, name);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  check(cudaLaunchKernelEx(&cfg, kern, p), "cudaLaunchKernelEx(blocked_pass)");
  launched(c, name);
}
}  // namespace

void sparse_full_step(Dataset& ds, Model& m, const StepArgs& a) {
  // The first pass issues its first static-data loads before its PDL wait,
  // so it may overlap its predecessor only when that predecessor cannot be
  // writing the derived structures, i.e. not right after they were (re)built.
  const bool rebuilt = !ds.sparse_ready;
  sparse_prep(ds);
  Ctx& c = *ds.ctx;
  if (ds.n == 0) return;
  const uint32_t d = static_cast<uint32_t>(ds.d);
  ApplyArgs aa{a.alpha, a.apply ? 1 : 0, a.want_norm ? 1 : 0, m.w64.p, m.w32.p, m.g64.p, m.finite.p, m.scal.p};
  if (ds.wide) {
    // K2w: margins of a model too large for SMEM, blocked by columns.
    launch_pass<kPassMargin>(ds, ds.wmajor, ds.n, d, m.w32.p, ds.mpart.p, a.task, aa, !rebuilt,
                             "k2w_margin_kernel");
  } else {  // K2s (d < 65,536 here: the 16-bit ids exist)
    const size_t model_bytes = round_up16(uint64_t(d + 1) * 4);
    const K2sArgs ka{ds.val.p, ds.cidx16.p, ds.rbm.p, ds.rbm_pre.p, ds.cta_slot.p,
                     ds.rows_empty ? ds.row_of_ord.p : nullptr, ds.labels.p, static_cast<uint32_t>(ds.n), m.w32.p, d,
                     ds.coef.p};
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.blockDim = dim3(kNT);
    cfg.stream = c.stream;
    cfg.attrs = attr;
    cfg.numAttrs = rebuilt ? 0 : 1;
    Blocked& B = ds.csc;
    const size_t gsmem = std::max<size_t>(model_bytes, round_up16(uint64_t(B.rb) * 4));
    // K23g: both passes in one launch whenever every work item of the
    // gradient pass has a CTA (more row blocks than SMs: K2s -> K3s below).
    if (B.nblk * B.cpb <= ds.cta_n && ds.cta_n == static_cast<uint32_t>(c.num_sms)) {
      void (*kern)(K2sArgs, PassArgs, const uint32_t*, uint32_t, unsigned*, const unsigned*);
      const bool rm = ds.rows_empty, sm = B.segs_empty;
      if (a.task == kTaskLR)
        kern = rm ? (sm ? glued_step_kernel<kTaskLR, true, true> : glued_step_kernel<kTaskLR, true, false>)
                  : (sm ? glued_step_kernel<kTaskLR, false, true> : glued_step_kernel<kTaskLR, false, false>);
      else
        kern = rm ? (sm ? glued_step_kernel<kTaskSVM, true, true> : glued_step_kernel<kTaskSVM, true, false>)
                  : (sm ? glued_step_kernel<kTaskSVM, false, true> : glued_step_kernel<kTaskSVM, false, false>);
      set_max_dyn_smem(reinterpret_cast<const void*>(kern), gsmem, "cudaFuncSetAttribute(k23g)");
      if (blocks_per_sm(reinterpret_cast<const void*>(kern), kNT, gsmem) >= 1) {
        m.part32.alloc(uint64_t(B.nblk) * d + 1);
        const PassArgs pa{B.val.p, B.id.p, B.bm.p, B.bm_pre.p, B.segptr.p, B.cta.p, B.cpb, B.nblk, d, B.rb,
                          static_cast<uint32_t>(ds.n), ds.coef.p, B.segs_empty ? B.ord_of_seg.p : nullptr,
                          m.part32.p, B.tickets.p, ++B.gen, 1, aa, ds.labels.p, ds.coef.p};
        cfg.gridDim = dim3(ds.cta_n);
        cfg.dynamicSmemBytes = gsmem;
        prof_begin(c, "k23g_step_kernel");
        check(cudaLaunchKernelEx(&cfg, kern, ka, pa, static_cast<const uint32_t*>(ds.cta_row.p), B.rb,
                                 ds.blk_ready.p, static_cast<const unsigned*>(ds.blk_expect.p)),
              "cudaLaunchKernelEx(k23g)");
        launched(c, "k23g_step_kernel");
        return;
      }
    }
    auto kern = a.task == kTaskLR
                    ? (ds.rows_empty ? k2s_margin_kernel<kTaskLR, true> : k2s_margin_kernel<kTaskLR, false>)
                    : (ds.rows_empty ? k2s_margin_kernel<kTaskSVM, true> : k2s_margin_kernel<kTaskSVM, false>);
    set_max_dyn_smem(reinterpret_cast<const void*>(kern), model_bytes, "cudaFuncSetAttribute(k2s)");
    prof_begin(c, "k2s_margin_kernel");
    cfg.gridDim = dim3(ds.cta_n);
    cfg.dynamicSmemBytes = model_bytes;
    check(cudaLaunchKernelEx(&cfg, kern, ka), "cudaLaunchKernelEx(k2s)");
    launched(c, "k2s_margin_kernel");
  }
  // K3s: the gradient pass and the update.
  m.part32.alloc(uint64_t(ds.csc.nblk) * d + 1);
  launch_pass<kPassGrad>(ds, ds.csc, d, ds.n, ds.coef.p, m.part32.p, a.task, aa, true, "k3s_grad_kernel");
}

}  // namespace sgdb::dev
