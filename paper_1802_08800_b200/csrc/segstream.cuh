// Segmented warp stream (sm_100a): one warp reduces a contiguous run of
// segments — CSR rows (the margin pass X.w, proj/src/linalg.cpp:30-44) or the
// columns of a row block of the blocked CSC (the gradient pass X^T c,
// linalg.cpp:50-109) — whose elements lie back to back in memory.
//
// Why: with a lane group per segment, every segment pays its own extent
// shuffles, window address math, group reduction and loop control; the
// sparse configs have 5-500 nonzeros per row, so such kernels issue ~300
// warp instructions per row and are issue-bound (ncu: issue-active 75-80 %)
// well before HBM is. Here the warp walks the stream in tiles of 32*E
// elements — lane l holds elements E*l .. E*l+E-1 (E/4 float4 windows of
// values and indices) — whatever the segment lengths, and recovers segment
// sums with a segmented warp scan, so the cost per tile does not depend on
// how many segments it touches, and a segment longer than a tile is carried
// across tiles.
//
// Bookkeeping: segment pointers are cached 32 at a time (lane l holds the
// start of segment gA + l) with the next chunk prefetched; the owner lane of
// a segment marks its head in a per-warp flag line (one byte per element);
// after the scan every lane parks its inclusive values in a per-warp SMEM
// line and the owner of each segment whose last element lies in the current
// (sub)tile reads the sum there and emits it. Empty segments are emitted
// with 0 when their chunk is entered. A tile crossing a chunk boundary is
// processed as two sub-tiles from the same registers. The summation order is
// fixed by the warp's tiling, so results are deterministic for a launch shape.
#pragma once

#include <cstdint>

namespace sgdb::dev {

// Per-warp scratch: TILE flag bytes (zero on entry, left zero) and TILE
// staged inclusive values, element-major (incl[u*32 + lane]) so the staging
// stores are bank-conflict free.
template <typename T, int E>
struct SegScratch {
  uint32_t flags[E * 8];  // 32*E bytes
  T incl[32 * E];
};

// Load(a, k) -> window k (elements a+4k .. a+4k+3) of the lane's run starting
// at a; Prod(win[E/4], p[E]) -> the E products; Emit(g, sum, aux_g, ok)
// stores segment g when ok (called by every lane, so it may be branch-free);
// aux_g = aux[g] is a per-segment payload fetched with the pointer chunk
// (e.g. the label; 0 when aux is null).
// NB = window buffers per lane: 2 keeps the next tile's loads in flight
// while a tile is scanned (more registers), 1 issues them at the top of the
// tile (for CTAs with many warps, which supply the memory parallelism).
//
// Element range: the warp streams elements [P0, P1). P0 may lie inside
// segment g0 (a segment continued from the previous warp: its head is not
// seen, and the sum emitted at its tail covers only [P0, tail]) and P1 may
// lie inside segment g1-1 (its tail is not reached: nothing is emitted for
// it). Returns the open segment's sum at P1 (the cut segment's partial).
// P0 = ptr[g0], P1 = ptr[g1] gives whole segments.
template <typename T, int E, int NB, class Win, class Load, class Prod, class Emit>
__device__ __forceinline__ T segment_stream(const uint32_t* __restrict__ ptr,
                                            const float* __restrict__ aux, uint32_t g0,
                                            uint32_t g1, uint32_t P0, uint32_t P1, Load load,
                                            Prod prod, Emit emit, SegScratch<T, E>& sc) {
  constexpr uint32_t TILE = 32 * E;
  constexpr int NW = E / 4;
  const int lane = threadIdx.x & 31;
  if (g0 >= g1) return T(0);
  const uint32_t S1 = P1;
  auto chunk_start = [&](uint32_t g) { return __ldg(ptr + min(g + lane, g1)); };
  auto chunk_end = [&](uint32_t g) { return __ldg(ptr + min(g + 32, g1)); };
  auto chunk_aux = [&](uint32_t g) { return aux && g + lane < g1 ? __ldg(aux + g + lane) : 0.f; };
  uint32_t gA = g0, rpA = chunk_start(gA), endA = chunk_end(gA);
  float axA = chunk_aux(gA);
  uint32_t rpB = chunk_start(gA + 32), endB = chunk_end(gA + 32);
  float axB = chunk_aux(gA + 32);
  uint32_t nxA;  // start of segment gA+lane+1
  bool liveA;    // segment gA+lane exists and is non-empty
  auto enter = [&]() {
    const uint32_t dn = __shfl_down_sync(0xffffffffu, rpA, 1);
    nxA = lane == 31 ? endA : dn;
    const bool exists = gA + lane < g1;
    liveA = exists && rpA < nxA;
    emit(gA + lane, T(0), axA, exists && rpA == nxA);
  };
  auto advance = [&]() {
    gA += 32;
    rpA = rpB;
    endA = endB;
    axA = axB;
    rpB = chunk_start(gA + 32);
    endB = chunk_end(gA + 32);
    axB = chunk_aux(gA + 32);
    enter();
  };
  enter();
  uint32_t pos = P0;
  T carry = T(0);
  uint8_t* f8 = reinterpret_cast<uint8_t*>(sc.flags);

  auto fill = [&](Win (&w)[NW], uint32_t t) {
    const uint32_t a = t + E * lane;
    const uint32_t aa = a < S1 ? a : 0u;
#pragma unroll
    for (int k = 0; k < NW; ++k) w[k] = load(aa, k);
  };
  // One tile: products from w, refill w with the tile two ahead, then the
  // sub-tiles' segmented scans and emissions.
  auto tile = [&](uint32_t Tt, Win (&w)[NW]) {
    float p[E];
    prod(w, p);
    fill(w, Tt + NB * TILE);
    const uint32_t tend = min(Tt + TILE, S1);
    const uint32_t e0 = Tt + E * lane;
    while (pos < tend) {  // warp-uniform
      while (pos == endA && gA + 32 < g1) advance();  // chunk exhausted (or only empty segments left)
      const uint32_t hi = min(tend, endA);
      if (liveA && rpA >= pos && rpA < hi) f8[rpA - Tt] = 1;
      __syncwarp();
      uint32_t fw[NW];
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        fw[k] = sc.flags[NW * lane + k];
        sc.flags[NW * lane + k] = 0u;  // only this lane reads these bytes
      }
      const bool full = pos <= Tt && hi == Tt + TILE;  // warp-uniform: no element masked
      T loc[E];
      int any = 0;
      {
        T acc = T(0);
#pragma unroll
        for (int u = 0; u < E; ++u) {
          T x = static_cast<T>(p[u]);
          if (!full) {
            const uint32_t e = e0 + u;
            x = (e >= pos && e < hi) ? x : T(0);
          }
          const bool h = (fw[u / 4] >> (8 * (u % 4))) & 1u;
          acc = (u == 0 || h) ? x : acc + x;
          loc[u] = acc;
        }
#pragma unroll
        for (int k = 0; k < NW; ++k) any |= fw[k] != 0u;
      }
      // Segmented inclusive scan of the lane totals (a head resets).
      T s = (lane == 0 && !any) ? carry + loc[E - 1] : loc[E - 1];
      int f = any;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const T os = __shfl_up_sync(0xffffffffu, s, off);
        const int of = __shfl_up_sync(0xffffffffu, f, off);
        if (lane >= off) {
          if (!f) s += os;
          f |= of;
        }
      }
      T ex = __shfl_up_sync(0xffffffffu, s, 1);
      if (lane == 0) ex = carry;
      // Inclusive value of every element: the lane's local run, plus the
      // carried-in sum for elements before the lane's first head.
      {
        bool seen = false;
#pragma unroll
        for (int u = 0; u < E; ++u) {
          seen = seen || ((fw[u / 4] >> (8 * (u % 4))) & 1u);
          sc.incl[32 * u + lane] = seen ? loc[u] : ex + loc[u];
        }
      }
      __syncwarp();
      // Owners whose last element lies in [pos, hi) emit the value there.
      const uint32_t t = nxA - 1;
      const bool done = liveA && t >= pos && t < hi;
      const uint32_t o = done ? t - Tt : 0u;  // element o = lane o / E, slot o % E
      const T v = sc.incl[32 * (o % E) + o / E];
      carry = sc.incl[32 * (E - 1) + 31];
      emit(gA + lane, v, axA, done);
      __syncwarp();  // incl / flags reused by the next sub-tile
      pos = hi;
    }
  };
  uint32_t Tt = pos & ~3u;
  Win wa[NW];
  fill(wa, Tt);
  if constexpr (NB == 1) {
    for (; Tt < S1; Tt += TILE) tile(Tt, wa);
  } else {
    Win wb[NW];
    fill(wb, Tt + TILE);
    // Two tiles per iteration so the window buffers never move between registers.
    while (Tt < S1) {
      tile(Tt, wa);
      Tt += TILE;
      if (Tt >= S1) break;
      tile(Tt, wb);
      Tt += TILE;
    }
  }
  // Trailing empty segments after the last element.
  while (gA + 32 < g1) advance();
  return carry;
}

}  // namespace sgdb::dev
