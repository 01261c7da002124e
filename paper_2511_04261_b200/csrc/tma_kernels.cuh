// tma_kernels.cuh -- the TMA-staged kernels (K1 k_stats_tma, K2 k_expand_tma)
// and their per-(C, b, n) selection templates. Instantiated per channel count
// in tma_c1.cu / tma_c3.cu (separate translation units build in parallel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "dppx_device.cuh"
#include "dppx_params.h"
#include "stats_common.cuh"

namespace dppx {

// ============================================================================
// K1: TMA-staged persistent kernel (fast path)
// ============================================================================
constexpr int kConsumers = 128;            // 4 consumer warps, one 4-px strip each
constexpr int kTilePx = 4 * kConsumers;    // 512 px per tile
constexpr int kStatsThreads = kConsumers + 32;
constexpr int kMaxStages = 4;
// Direct complex draws take two vertical subcells per iteration from this n up
// (A/B knob at build time).
#ifndef DPPX_PAIRS_MIN
#define DPPX_PAIRS_MIN 8
#endif
constexpr int kPairsMinNsub = DPPX_PAIRS_MIN;

// Ring position of unit k in an S-stage ring (S in {2, 3, 4}, the host's
// choice at run time): slot and lap without a runtime integer division (a
// division by a non-constant is ~25 instructions, and these run per unit).
__device__ __forceinline__ int ring_slot(int k, int S) {
  return S == 2 ? (k & 1) : S == 4 ? (k & 3) : k % 3;
}
__device__ __forceinline__ int ring_lap(int k, int S) {
  return S == 2 ? (k >> 1) : S == 4 ? (k >> 2) : k / 3;
}

struct UnitPos {
  int fg, r, tile, px0;  // frame group (frames fg*pack + j), grid row, column tile
};

// TILE: pixels per unit column tile (512 for power-of-two cells; general cell
// widths use whole cells per warp, see k_stats_tma).
template <bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ UnitPos decode_unit(const StatsArgs& a, int u) {
  UnitPos p;
  const uint32_t rest = a.div_tiles.div(static_cast<uint32_t>(u));
  p.tile = u - static_cast<int>(rest * a.div_tiles.d);
  const uint32_t fg = a.div_rows.div(rest);
  p.r = a.row_begin + static_cast<int>(rest - fg * a.div_rows.d);
  p.fg = static_cast<int>(fg);
  p.px0 = PACKED ? 0 : p.tile * TILE;  // packed units are one tile wide
  return p;
}

// Slot geometry: compile-time for wide frames (one TILE-px slot per unit).
template <bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ int slot_px(const StatsArgs& a) {
  return PACKED ? a.slot_px : TILE;
}
template <bool PACKED>
__device__ __forceinline__ int units_pack(const StatsArgs& a) {
  return PACKED ? a.pack : 1;
}

// Real bytes of a slot row starting at column px0.
template <int C, bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ int valid_bytes(const StatsArgs& a, int px0) {
  return min(slot_px<PACKED, TILE>(a), a.g.N - px0) * C;
}

// A band whose rows run past M needs mirrored rows (image.cpp:105-110): it is
// staged row by row with 1-D bulk copies; every other band is one 3-D box.
template <int B>
__device__ __forceinline__ bool band_reflects(const StatsArgs& a, int r) {
  return (r + 1) * B > a.g.M;
}

// Bytes per row a 1-D bulk copy stages (multiple of 16): rounded up into the
// pitch slack when the rows have it, else down (the rest is filled by threads).
template <int C, bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ int bulk_row_bytes(const StatsArgs& a, int px0) {
  const int v = valid_bytes<C, PACKED, TILE>(a, px0);
  return a.row_slack ? min(slot_px<PACKED, TILE>(a) * C, (v + 15) & ~15) : (v & ~15);
}

// Bytes of each smem slot row that the producer's copies deliver.
template <int C, int B, bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ int staged_bytes(const StatsArgs& a, const UnitPos& p) {
  if (band_reflects<B>(a, p.r)) return bulk_row_bytes<C, PACKED, TILE>(a, p.px0);
  return max(0, min(slot_px<PACKED, TILE>(a) * C, a.tensor_in_bytes - p.px0 * C));
}

template <int C, int B, bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ void load_unit(const StatsArgs& a, const CUtensorMap* tm, int u,
                                          uint8_t* st, uint64_t* bar) {
  const UnitPos p = decode_unit<PACKED, TILE>(a, u);
  const int srb = slot_px<PACKED, TILE>(a) * C;
  const int pk = units_pack<PACKED>(a);
  const int nf = PACKED ? min(pk, a.g.F - p.fg * pk) : 1;
  if (!band_reflects<B>(a, p.r)) {
    mbar_arrive_expect_tx(bar, nf * B * srb);  // full boxes, OOB bytes zero-filled
    for (int j = 0; j < nf; ++j)
      tma_load_3d(st + j * a.slot_stride, tm, p.px0 * C / 8, p.r * B, p.fg * pk + j, bar);
    return;
  }
  const uint32_t copy = static_cast<uint32_t>(bulk_row_bytes<C, PACKED, TILE>(a, p.px0));
  mbar_arrive_expect_tx(bar, copy * B * nf);
  if (copy == 0) return;
#pragma unroll 1
  for (int j = 0; j < nf; ++j) {
    const uint8_t* src = a.img + static_cast<int64_t>(p.fg * pk + j) * a.fstride +
                         static_cast<int64_t>(p.px0) * C;
#pragma unroll 1
    for (int i = 0; i < B; ++i) {
      const int srow = reflect_index(p.r * B + i, a.g.M);
      bulk_g2s(st + j * a.slot_stride + i * srb, src + static_cast<int64_t>(srow) * a.pitch, copy,
               bar);
    }
  }
}

// One 3-D box store per slot: rows >= M and bytes past the tensor's row are
// clipped by the TMA unit; the consumers write the (< 16) bytes past
// tensor_out_bytes.
template <int C, int B, bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ void store_unit(const StatsArgs& a, const CUtensorMap* tm, int u,
                                           const uint8_t* st) {
  const UnitPos p = decode_unit<PACKED, TILE>(a, u);
  if (p.px0 * C >= a.tensor_out_bytes) return;
  const int pk = units_pack<PACKED>(a);
  const int nf = PACKED ? min(pk, a.g.F - p.fg * pk) : 1;
  for (int j = 0; j < nf; ++j)
    tma_store_3d(tm, p.px0 * C / 8, p.r * B, p.fg * pk + j, st + j * a.slot_stride);
  bulk_commit();
  bulk_wait_read_all();
}

// The < 16 bytes of an output row past the store tensor map's extent: the
// extent is a multiple of 16 bytes and rows / smem slot rows are 16-byte
// aligned, so the tail is at most four aligned stores (8, 4, 2, 1 bytes)
// instead of one store per byte (CelebA rows: 6 tail bytes per row).
__device__ __forceinline__ void copy_row_tail(uint8_t* dst, const uint8_t* src, int n) {
  if (n >= 16 || ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 7)) {
    for (int x = 0; x < n; ++x) dst[x] = src[x];
    return;
  }
  int o = 0;
  if (n & 8) {
    *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(src);
    o = 8;
  }
  if (n & 4) {
    *reinterpret_cast<uint32_t*>(dst + o) = *reinterpret_cast<const uint32_t*>(src + o);
    o += 4;
  }
  if (n & 2) {
    *reinterpret_cast<uint16_t*>(dst + o) = *reinterpret_cast<const uint16_t*>(src + o);
    o += 2;
  }
  if (n & 1) dst[o] = src[o];
}

// Output bytes of a unit past the output tensor map's row extent (< 16 per row:
// the TMA store covers [0, tensor_out_bytes)), written by the 32 producer lanes.
template <int C, int B, bool PACKED, int TILE = kTilePx>
__device__ __forceinline__ void store_tail(const StatsArgs& a, int u, const uint8_t* st, int lane) {
  const UnitPos p = decode_unit<PACKED, TILE>(a, u);
  const int srb = slot_px<PACKED, TILE>(a) * C;
  const int vbytes = valid_bytes<C, PACKED, TILE>(a, p.px0);
  const int scopy = max(0, min(srb, a.tensor_out_bytes - p.px0 * C));
  if (scopy >= vbytes) return;
  const int span = vbytes - scopy;
  const int rows = min(B, a.g.M - p.r * B);
  const int pk = units_pack<PACKED>(a);
  const int nf = PACKED ? min(pk, a.g.F - p.fg * pk) : 1;
  for (int e = lane; e < nf * rows; e += 32) {  // one row per lane
    const int j = e / rows, i = e - j * rows;
    copy_row_tail(a.out + static_cast<int64_t>(p.fg * pk + j) * a.ofstride +
                      static_cast<int64_t>(p.r * B + i) * a.opitch + static_cast<int64_t>(p.px0) * C + scopy,
                  st + j * a.slot_stride + i * srb + scopy, span);
  }
}

// Byte k (0..4C-1) of a 4-pixel strip of value v[] (interleaved channels).
template <int C>
__device__ __forceinline__ void pattern_words(const uint32_t (&v)[C], uint32_t (&w)[C]) {
  if constexpr (C == 1) {
    w[0] = v[0] * 0x01010101u;
  } else if constexpr (C == 3) {
    w[0] = v[0] | (v[1] << 8) | (v[2] << 16) | (v[0] << 24);
    w[1] = v[1] | (v[2] << 8) | (v[0] << 16) | (v[1] << 24);
    w[2] = v[2] | (v[0] << 8) | (v[1] << 16) | (v[2] << 24);
  } else {  // C == 4: one pixel per word
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
  }
}

// Per-channel byte sums of one 4-px strip row held in C words, added to acc.
// Each row's partial starts from zero so rows form independent dp4a chains.
template <int C>
__device__ __forceinline__ void accumulate_row(const uint8_t* row, uint32_t (&acc)[C]) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row);
  if constexpr (C == 1) {
    acc[0] += __dp4a(w[0], 0x01010101u, 0u);
  } else if constexpr (C == 3) {
    const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
    // bytes: w0 = R G B R, w1 = G B R G, w2 = B R G B (little-endian)
    acc[0] += __dp4a(w0, 0x01000001u, __dp4a(w1, 0x00010000u, __dp4a(w2, 0x00000100u, 0u)));
    acc[1] += __dp4a(w0, 0x00000100u, __dp4a(w1, 0x01000001u, __dp4a(w2, 0x00010000u, 0u)));
    acc[2] += __dp4a(w0, 0x00010000u, __dp4a(w1, 0x00000100u, __dp4a(w2, 0x01000001u, 0u)));
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t x = w[k];
      acc[0] += x & 0xFF;
      acc[1] += (x >> 8) & 0xFF;
      acc[2] += (x >> 16) & 0xFF;
      acc[3] += x >> 24;
    }
  }
}

// Per-channel byte sums of the pixels selected by m (m[ch][q]: dp4a weights of
// word q for channel ch) of one 4-px strip row: a subcell boundary inside the
// strip (subcell sides that are not a multiple of 4 px).
template <int C>
__device__ __forceinline__ void accumulate_row_masked(const uint8_t* row,
                                                      const uint32_t (&m)[C][C == 4 ? 4 : C],
                                                      uint32_t (&acc)[C]) {
  constexpr int NW = C == 4 ? 4 : C;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row);
  uint32_t x[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) x[q] = w[q];
#pragma unroll
  for (int ch = 0; ch < C; ++ch) {
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < NW; ++q) s = __dp4a(x[q], m[ch][q], s);
    acc[ch] += s;
  }
}

// Strip words whose pixels [0, split) take va[] and the rest vb[].
template <int C>
__device__ __forceinline__ void pattern_words_split(const uint32_t (&va)[C], const uint32_t (&vb)[C],
                                                    int split, uint32_t (&w)[C == 4 ? 4 : C]) {
  constexpr int NW = C == 4 ? 4 : C;
#pragma unroll
  for (int q = 0; q < NW; ++q) w[q] = 0;
#pragma unroll
  for (int pos = 0; pos < 4 * C; ++pos) {
    const int k = pos / C, ch = pos % C;
    w[pos / 4] |= (k < split ? va[ch] : vb[ch]) << (8 * (pos % 4));
  }
}

// Sum of squares of all bytes of one 4-px strip row (variance extension).
template <int C>
__device__ __forceinline__ uint32_t square_row(const uint8_t* row, uint32_t acc) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row);
#pragma unroll
  for (int k = 0; k < (C == 4 ? 4 : C); ++k) acc = __dp4a(w[k], w[k], acc);
  return acc;
}

// Sum over an aligned group of G lanes (a cell or subcell), result in every lane
// of the group: butterfly for power-of-two G, else gather at the group's first
// lane and broadcast (groups never straddle a warp: see k_stats_tma's LPW).
template <int G>
__device__ __forceinline__ uint32_t group_sum(uint32_t x) {
  if constexpr ((G & (G - 1)) == 0) {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    return x;
  } else {
    const int lane = threadIdx.x & 31;
    uint32_t sum = x;
#pragma unroll
    for (int o = 1; o < G; ++o) sum += __shfl_down_sync(0xFFFFFFFFu, x, o);
    return __shfl_sync(0xFFFFFFFFu, sum, lane - lane % G);
  }
}

// Values of the C channels of one statistic, computed by the GL lanes of a
// lane group (each lane draws a subset of channels) and shared by shuffles.
// KSPLIT: the keyed case also gets its own exact-fallback and shuffle code
// (measured faster for wide frames; the packed narrow-frame instantiation
// spills with it, so it shares them).
template <int C, int GL, bool KSPLIT = true>
__device__ __forceinline__ void group_values(const StatsArgs& a, const DrawEnv& env, bool active,
                                             const uint32_t (&sum)[C], const uint64_t (&cs)[C],
                                             int f, int r, int c, int sr, int sc,
                                             uint32_t (&val)[C]) {
  constexpr int NV = (C + GL - 1) / GL;  // channels this lane draws
  if (!__any_sync(0xFFFFFFFFu, active)) {  // warp-uniform: nothing to draw
#pragma unroll
    for (int k = 0; k < C; ++k) val[k] = 0;
    return;
  }
  const int lane = threadIdx.x & 31;
  const int li = lane % GL;
  const int gb = lane - li;
  uint32_t s[NV], q[NV];
  uint64_t bits[NV];
  uint64_t stv[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int ch = j * GL + li;
    s[j] = sum[0];
    stv[j] = cs[0];
#pragma unroll
    for (int k = 1; k < C; ++k)
      if (ch == k) {
        s[j] = sum[k];
        stv[j] = cs[k];
      }
  }
  if (env.kind == DPPX_NOISE_KEYED && !env.exact_only) {
    // The common case on its own path: no Philox / injected-noise arguments
    // are formed (the compiler would otherwise compute them for every draw).
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      bits[j] = key_sub(stv[j], sr, sc);
      q[j] = fast_quantize(s[j], env.inv_area, bits[j], env.sln2, env.margin);
    }
    if constexpr (KSPLIT) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int ch = j * GL + li;
        if (active && ch < C && q[j] == 0xFFFFFFFFu)
          q[j] = exact_quantize(s[j], env.area, DPPX_NOISE_KEYED, bits[j], env.sigma, 0.0);
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) {
#pragma unroll
        for (int k = j * GL; k < C && k < (j + 1) * GL; ++k)
          val[k] = (GL == 1) ? q[j] : __shfl_sync(0xFFFFFFFFu, q[j], gb + (k - j * GL));
      }
      return;
    }
  } else {
#pragma unroll
    for (int j = 0; j < NV; ++j) bits[j] = draw_bits(a, stv[j], f, j * GL + li, r, c, sr, sc);
    // Phase 1: branch-free bounded estimates for all channels (independent
    // chains the scheduler can interleave); phase 2: the rare exact draws.
    if (!env.exact_only && env.kind == DPPX_NOISE_PHILOX) {
#pragma unroll
      for (int j = 0; j < NV; ++j) q[j] = fast_quantize(s[j], env.inv_area, bits[j], env.sln2, env.margin);
    } else if (!env.exact_only && env.kind == DPPX_NOISE_NONE && env.pow2) {
#pragma unroll
      for (int j = 0; j < NV; ++j)  // sum * 2^-k + 0.5 is exact in f32
        q[j] = static_cast<uint32_t>(floorf(static_cast<float>(s[j]) * env.inv_area + 0.5f));
    } else {
#pragma unroll
      for (int j = 0; j < NV; ++j) q[j] = 0xFFFFFFFFu;
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int ch = j * GL + li;
    if (active && ch < C && q[j] == 0xFFFFFFFFu)
      q[j] = exact_quantize(s[j], env.area, env.kind, bits[j], env.sigma,
                            env.kind == DPPX_NOISE_INJECTED ? inj_at(a, f, ch, r * a.g.GC + c, sr, sc)()
                                                            : 0.0);
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
#pragma unroll
    for (int k = j * GL; k < C && k < (j + 1) * GL; ++k)
      val[k] = (GL == 1) ? q[j] : __shfl_sync(0xFFFFFFFFu, q[j], gb + (k - j * GL));
  }
}

// RPU: cell rows per unit. Uniform b = 4 stages two cell rows (an 8-row band)
// per unit (RPU = 2) so the per-unit work -- claim, metadata, mirror fill,
// barriers, store bookkeeping -- is paid once per 6 draws per lane instead of
// 3 (the b = 4 kernel is instruction-bound, profiles/r02p_k1_uniform_b4_full.md).
template <int C, int B4, int NSUB, bool ADAPTIVE, bool PACKED, bool VAR = false, int RPU = 1>
#ifndef DPPX_RPU2_MINB
#define DPPX_RPU2_MINB 5
#endif
__global__ void __launch_bounds__(kStatsThreads, (!ADAPTIVE && B4 == 1) ? (RPU > 1 ? DPPX_RPU2_MINB : 6) : 0)
    k_stats_tma(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                const StatsArgs a) {
  constexpr int B = 4 * B4;
  constexpr int BR = B * RPU;  // rows of a unit's band
  static_assert(RPU == 1 || (!ADAPTIVE && !PACKED && !VAR), "multi-row units: uniform wide frames");
  constexpr int SB = B / NSUB;
  constexpr int SB4 = SB / 4;
  // Subcell sides that are not a multiple of 4 px (b = 24 n = 4: 6 px; 2 or
  // 3 px): a strip can straddle two subcells; each lane splits its strip sums at the
  // boundary and the subcell sums meet in per-warp smem (compact draw mode).
  // PIX (n = b, 1-px subcells: the diagonal of the paper's PPM-100 (b, n) grid,
  // CelebA b4 n4 / b16 n16): every pixel of a complex cell is its own
  // statistic; each lane draws its strip's 4 px x C per row in place.
  // In-lane subcells (SB = 1 or 2 px: n = b, n = b/2 -- the PPM-100 grid's
  // diagonals, CelebA b4 n4 / b8 n4 / b16 n8 / b16 n16): a strip holds 4/SB
  // whole subcells per row, so each lane sums, draws and writes its own
  // subcells in place -- no cross-lane tables.
  // (packed narrow frames keep the split-strip tables for 2-px subcells: their
  // compacted draws measured faster there, CelebA b8 n4 2.5 vs 3.1 ms)
  constexpr bool PIX = NSUB > 1 && (SB == 1 || (SB == 2 && !PACKED));
  constexpr int KS = PIX ? 4 / SB : 1;  // subcells per strip and subcell row
  constexpr bool STR = (SB % 4) != 0 && !PIX;
  // Strips per warp: whole cells only (a cell is B4 adjacent lanes), so for
  // B4 not a power of two (b = 12, 24) the last 32 % B4 lanes of each warp
  // idle and the tile is 16 * LPW px (480 at b = 12 or 24) instead of 512.
  constexpr int LPW = (32 / B4) * B4;
  constexpr int TILE = 4 * (kConsumers / 32) * LPW;
  constexpr int ROWB = TILE * C;
  constexpr uint32_t STAGE = BR * ROWB;
  // (SB >= 2: a strip meets at most two subcells.)
  static_assert(B4 <= 32 && (PIX ? (ADAPTIVE && !VAR && NSUB == B / SB) : STR ? (SB >= 2 && ADAPTIVE && !VAR) : B4 % SB4 == 0),
                "fast-path geometry");
  static_assert(TILE == kTilePx || !PACKED, "packed slots use 512-px tiles");
  static_assert(!VAR || (ADAPTIVE && !PACKED), "variance staging: wide adaptive frames only");

  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];  // TMA bytes landed
  __shared__ __align__(8) uint64_t id_bar[kMaxStages];    // stage_unit[s] published
  __shared__ __align__(8) uint64_t done_bar[kMaxStages];  // consumers finished the stage
  __shared__ int stage_unit[kMaxStages];                  // unit in stage s, -1 = no more work

  const int S = a.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&id_bar[s], 1);
      mbar_init(&done_bar[s], kConsumers);
    }
    fence_mbarrier_init();
  }
  __syncthreads();

  if (warp == kConsumers / 32) {
    // ---------------- producer warp: TMA loads + bulk stores ----------------
    // Units (frame, grid row, TILE-px tile) are claimed from a global counter so
    // heavy (complex-cell) tiles spread over all CTAs.
    // The whole warp stays in the loop: lane 0 claims units and issues the TMA
    // copies; all 32 lanes write the few output bytes past the output tensor
    // map's row extent (keeps that byte loop off the consumer warps).
    if (lane == 0) {
      prefetch_tmap(&tm_in);
      prefetch_tmap(&tm_out);
    }
    auto finish_unit = [&](int s, int use) {  // after consumers released stage s
      mbar_wait(&done_bar[s], use & 1);        // every lane acquires the smem writes
      if (a.out) {
        const int uu = stage_unit[s];
        store_tail<C, BR, PACKED, TILE>(a, uu, smem + s * STAGE, lane);
        if (lane == 0) store_unit<C, BR, PACKED, TILE>(a, &tm_out, uu, smem + s * STAGE);
      }
      __syncwarp();
    };
    int k = 0;
    int done_units = 0;  // units of this CTA already stored
    for (;; ++k) {
      const int s = ring_slot(k, S);
      if (k >= S) {
        finish_unit(s, ring_lap(k, S) - 1);
        ++done_units;
      }
      int u = 0;
      if (lane == 0) {
        u = atomicAdd(a.work_counter, 1);
        if (u >= a.units) {
          // Every producer makes exactly one failing claim; the last one resets
          // the counter for the next launch (no memset per launch).
          if (u == a.units + static_cast<int>(gridDim.x) - 1) atomicExch(a.work_counter, 0);
          u = -1;
        }
        stage_unit[s] = u;
        mbar_arrive(&id_bar[s]);
        if (u < 0)
          mbar_arrive_expect_tx(&full_bar[s], 0);
        else
          load_unit<C, BR, PACKED, TILE>(a, &tm_in, u, smem + s * STAGE, &full_bar[s]);
      }
      u = __shfl_sync(0xFFFFFFFFu, u, 0);
      if (u < 0) break;
    }
    // k units were loaded; units [done_units, k) still need their store.
    for (int j = done_units; j < k; ++j) finish_unit(ring_slot(j, S), ring_lap(j, S));
    if (lane == 0) bulk_wait_all();
    return;
  }

  // ---------------- consumer warps ----------------
  const int t = threadIdx.x;  // strip index within the tile
  const BatchGeom& g = a.g;
  const DrawEnv env_cell = make_env(a.noise.kind, a.exact_noise != 0, a.area, a.sigma);
  const DrawEnv env_sub = make_env(a.noise.kind, a.exact_noise != 0, a.sub_area, a.sigma_sub);
  // Per-unit metadata (K0's cell info, row prefix, simple total, plane seeds)
  // is loaded one unit ahead so its L2 latency hides behind a unit of work.
  struct Meta {
    int u;
    UnitPos pos;
    uint32_t info, rowpre, stot;
    uint64_t seed[C];
  };
  // This thread's 4-px strip in the tile: lanes >= LPW of a warp have none
  // (only when B4 is not a power of two) and compute on strip 0, inactive.
  const bool strip_ok = (t & 31) < LPW;
  const int sx = strip_ok ? (t >> 5) * LPW + (t & 31) : 0;  // strip index
  // Slot of the strip (fixed for the kernel). Wide frames (PACKED = false)
  // have one TILE-px slot: the compiler folds all of this.
  const int my_j = PACKED ? (4 * sx) / a.slot_px : 0;
  const bool in_slot = strip_ok && my_j < (PACKED ? a.pack : 1);
  const int jj = in_slot ? my_j : 0;
  const int lpx = 4 * sx - jj * (PACKED ? a.slot_px : TILE);  // strip column in its slot
  const int srb = PACKED ? a.slot_px * C : TILE * C;         // smem bytes per slot row
  // Packed mode: byte offsets of the mirrored sources of the padding bytes
  // [N*C, GC*b*C) of a slot row (image.cpp:105-110), shared by all units.
  __shared__ uint16_t fill_src[128];
  // Per-warp complex-draw tables (see the complex-cell block below).
  constexpr int CPW = 32 / B4;           // cells per consumer warp
  constexpr int NN = NSUB * NSUB;
  using SumT = typename std::conditional<(SB * SB * 255 < 65536 && !STR), uint16_t, uint32_t>::type;
  constexpr bool TABLES = VAR || STR;
  struct CellRec {
    int cw, f, cell, gidx;
    int64_t off;
  };
  __shared__ SumT csum[TABLES ? kConsumers / 32 : 1][TABLES ? CPW : 1][TABLES ? NN * C : 1];
  __shared__ CellRec crec[TABLES ? kConsumers / 32 : 1][TABLES ? CPW : 1];
  __shared__ uint64_t cstate[TABLES ? kConsumers / 32 : 1][TABLES ? CPW : 1][C];
  const int wq = TABLES ? (t >> 5) : 0;          // consumer warp
  const int cw = TABLES ? ((t & 31) / B4) : 0;   // cell within the warp
  // STR: this strip's first subcell column, the pixels [0, split) in it, and
  // the dp4a weights selecting those pixels per channel.
  const int str_px = 4 * (sx % B4);
  const int str_sa = STR ? str_px / SB : 0;
  const int str_split = STR ? min(4, (str_sa + 1) * SB - str_px) : 4;
  uint32_t str_m[C][C == 4 ? 4 : C];
#pragma unroll
  for (int ch = 0; ch < C; ++ch)
#pragma unroll
    for (int q = 0; q < (C == 4 ? 4 : C); ++q) str_m[ch][q] = 0;
  if constexpr (STR) {
#pragma unroll
    for (int pos = 0; pos < 4 * C; ++pos)
      if (pos / C < str_split) str_m[pos % C][pos / 4] |= 1u << (8 * (pos % 4));
  }
  if (PACKED) {
    const int v0 = g.N * C, pad = (g.GC * B - g.N) * C;
    for (int x = t; x < pad && x < 128; x += kConsumers) {
      const int cpx = (v0 + x) / C, ch = (v0 + x) - cpx * C;
      fill_src[x] = static_cast<uint16_t>(reflect_index(cpx, g.N) * C + ch);
    }
    named_bar_sync(1, kConsumers);
  }
  // (ring slot and lap of each unit are advanced incrementally, and the unit
  // is decoded once, here: both ran per unit and per thread)
  auto load_meta = [&](int sn, int lap) {
    Meta m;
    mbar_wait(&id_bar[sn], lap & 1);
    m.u = *reinterpret_cast<volatile int*>(&stage_unit[sn]);
    m.info = 1u;
    m.rowpre = m.stot = 0;
#pragma unroll
    for (int ch = 0; ch < C; ++ch) m.seed[ch] = 0;
    m.pos = UnitPos{0, 0, 0, 0};
    if (m.u >= 0) {
      const UnitPos q = decode_unit<PACKED, TILE>(a, m.u);
      if (!PACKED) m.pos = q;
      const int qf = q.fg * units_pack<PACKED>(a) + jj;
      const int qcell = PACKED ? (q.px0 + lpx) / B : q.px0 / B + sx / B4;
      if (!PACKED || qf < g.F) {
        if (ADAPTIVE && !VAR && qcell < g.GC) {
          m.info = __ldg(&a.cellinfo[static_cast<int64_t>(qf) * g.G + q.r * g.GC + qcell]);
          m.rowpre = __ldg(&a.rowprefix[static_cast<int64_t>(qf) * g.GR + q.r]);
          m.stot = __ldg(&a.totals[qf]);
        }
        if (a.noise.kind == DPPX_NOISE_KEYED) {
#pragma unroll
          for (int ch = 0; ch < C; ++ch)
            m.seed[ch] = a.noise.seed(static_cast<int64_t>(qf) * C + ch);
        }
      }
    }
    return m;
  };
  Meta next = load_meta(0, 0);
  for (int s = 0, lap = 0;;) {
    const int s_next = s + 1 == S ? 0 : s + 1;
    const int lap_next = s_next == 0 ? lap + 1 : lap;
    uint8_t* st = smem + s * STAGE;
    const Meta cur = next;
    const int u = cur.u;
    if (u < 0) break;
    // (packed units decode here again: carrying the position in Meta costs the
    // packed instantiation registers it spills)
    const UnitPos p = PACKED ? decode_unit<PACKED, TILE>(a, u) : cur.pos;
    const int f = p.fg * units_pack<PACKED>(a) + jj;  // this thread's frame
    const int cell = PACKED ? (p.px0 + lpx) / B : p.px0 / B + sx / B4;
    const int lic = sx % B4;       // lane within cell
    const int sc = lic / (SB4 > 0 ? SB4 : 1);  // subcell column (unused for split strips)
    const bool active = in_slot && (!PACKED || f < g.F) && cell < g.GC;
    const int gidx = p.r * g.GC + cell;
    const bool simple0 = !ADAPTIVE || (cur.info & 1u);  // VAR: decided after the sums
    const uint32_t slot_s = cur.rowpre + (cur.info >> 1);
    const uint32_t S_tot = cur.stot;
    const int vbytes = valid_bytes<C, PACKED, TILE>(a, p.px0);
    const int copy = staged_bytes<C, BR, PACKED, TILE>(a, p);  // bytes per row the producer staged
    const int need = min(slot_px<PACKED, TILE>(a), g.GC * B - p.px0) * C;
    const int nf = PACKED ? min(a.pack, g.F - p.fg * a.pack) : 1;
    uint64_t cs[C];
#pragma unroll
    for (int ch = 0; ch < C; ++ch)
      cs[ch] = a.noise.kind == DPPX_NOISE_KEYED ? key_cell(cur.seed[ch], p.r, cell) : 0ull;

    mbar_wait(&full_bar[s], lap & 1);

    // Row tail not covered by the staged copy and mirrored padding columns
    // (image.cpp:105-110), including stray pitch-slack bytes a rounded-up copy
    // brought in. Work is split as (slot row, column lane) so no index needs a
    // runtime division. A mirrored byte is read from the staged row in smem when
    // it is there (sources lie in [0, fs), targets in [fs, need): disjoint),
    // else from global memory.
    if (PACKED && a.row_slack) {
      // Packed slots always start at column 0 and the staged rows always cover
      // the real bytes: the mirror map of the padding is the same for every
      // row of every unit (precomputed in fill_src).
      const int span = need - vbytes;
      if (span > 0) {
        constexpr int kLanes = 8;
        for (int pr = t / kLanes; pr < nf * B; pr += kConsumers / kLanes) {
          const int j = pr / B, i = pr - j * B;
          uint8_t* rowp = st + j * a.slot_stride + i * srb;
          for (int x = t % kLanes; x < span; x += kLanes) rowp[vbytes + x] = rowp[fill_src[x]];
        }
        named_bar_sync(1, kConsumers);
      }
    } else {
      const int fs = min(copy, vbytes);
      if (fs < need) {
        constexpr int kLanes = 4;  // consumer threads per slot row
        const int rows_total = nf * BR;
        for (int pr = t / kLanes; pr < rows_total; pr += kConsumers / kLanes) {
          const int j = pr / BR, i = pr - j * BR;  // BR is a compile-time power of two
          uint8_t* rowp = st + j * (PACKED ? a.slot_stride : 0) + i * srb;
          const int frame = p.fg * units_pack<PACKED>(a) + j;
          const int srow = reflect_index(p.r * BR + i, g.M);
          const uint8_t* grow = a.img + static_cast<int64_t>(frame) * a.fstride +
                                static_cast<int64_t>(srow) * a.pitch;
          for (int x = fs + (t % kLanes); x < need; x += kLanes) {
            const int cpx = x / C, ch = x - cpx * C;  // C is a compile-time constant
            const int spx = reflect_index(p.px0 + cpx, g.N);
            const int sx = (spx - p.px0) * C + ch;
            rowp[x] = (sx >= 0 && sx < fs) ? rowp[sx]
                                           : __ldg(grow + static_cast<int64_t>(spx) * C + ch);
          }
        }
        named_bar_sync(1, kConsumers);
      }
    }

    const bool emit = a.out != nullptr;
    uint8_t* mystrip = st + jj * a.slot_stride + lpx * C;
    uint32_t tot[C];
#pragma unroll
    for (int ch = 0; ch < C; ++ch) tot[ch] = 0;
    bool simple = simple0;
    if constexpr (VAR) {
      // Pass 1 over the staged rows: per-channel cell sums and the sum of
      // squares; the variance test on the whole cell (same integers and IEEE
      // divide as K0 mode 2 / or_classify_variance).
      uint32_t sq = 0;
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const uint8_t* row = mystrip + i * srb;
        accumulate_row<C>(row, tot);
        sq = square_row<C>(row, sq);
      }
      next = load_meta(s_next, lap_next);
      uint32_t s1 = 0;
#pragma unroll
      for (int ch = 0; ch < C; ++ch) s1 += tot[ch];
      s1 = group_sum<B4>(s1);
      sq = group_sum<B4>(sq);
      const long long ns = static_cast<long long>(C) * B * B;
      const double num = static_cast<double>(ns * static_cast<long long>(sq) -
                                             static_cast<long long>(s1) * static_cast<long long>(s1));
      simple = !(__ddiv_rn(num, __dmul_rn(static_cast<double>(ns), static_cast<double>(ns))) >=
                 a.var_tau);
      if (active && lic == 0) a.var_flags[static_cast<int64_t>(f) * g.G + gidx] = simple ? 1 : 0;
    }

    if constexpr (ADAPTIVE) {
      // Complex cells. Direct mode (mask classification): the owner lanes of
      // each subcell draw its C values (NSUB * ceil(C / SB4) serial draws per
      // lane); masks are spatially coherent, so warps are mostly all-simple or
      // all-complex. Compact mode (variance classification, which scatters
      // complex cells): the owner lanes put the subcell sums into this warp's
      // smem table and the warp's complex draws (cells x n*n x C) are dealt
      // round-robin to all 32 lanes, so the lanes of simple cells do not idle
      // through the serial draws (tools/k1_complex_sweep.py measures both).
      constexpr bool compact = VAR || STR;
      const bool cx = active && !simple;
      const unsigned cx_any = __ballot_sync(0xFFFFFFFFu, cx);
      __syncwarp();  // the previous unit's reads of this warp's tables are done
      if constexpr (STR) {
        if (cx_any) {  // subcell sums accumulate with smem atomics
          for (int i = t & 31; i < CPW * NN * C; i += 32) (&csum[wq][0][0])[i] = 0;
          __syncwarp();
        }
      }
      // Direct mode with many vertical subcells (NSUB >= 8): two at a time, so
      // the two subcells' draw chains overlap (a store of one subcell's pattern
      // would otherwise order the next subcell's smem reads behind its draws).
      constexpr bool PAIRS = !compact && !PIX && NSUB >= kPairsMinNsub && NSUB % 2 == 0;
      if constexpr (PIX) {
        // whole-cell sums for the simple cells (tot), then the complex cells'
        // subcells: each lane's KS subcells per subcell row, summed from its own
        // strip, one keyed draw per (subcell, channel) at sigma_sub, written back
        // into the strip
#pragma unroll 4
        for (int i = 0; i < B; ++i) accumulate_row<C>(mystrip + i * srb, tot);
        if (cx_any) {
          const int sc0 = KS * lic;  // this strip's first subcell column in the cell
          const int64_t off0 = cx ? complex_offset<NSUB * NSUB>(a, gidx, slot_s, S_tot, 0) : 0;
#pragma unroll 1
          for (int sr = 0; sr < NSUB; ++sr) {
            if (cx) {
              uint8_t* row0p = mystrip + sr * SB * srb;
#pragma unroll
              for (int q = 0; q < KS * C; ++q) {
                const int k = q / C, ch = q - k * C;
                uint32_t sum = 0;
#pragma unroll
                for (int y = 0; y < SB; ++y)
#pragma unroll
                  for (int x = 0; x < SB; ++x) sum += row0p[y * srb + (k * SB + x) * C + ch];
                const uint32_t v = draw_stat(a, env_sub, sum, cs[ch], f, ch, p.r, cell, sr, sc0 + k, gidx);
                a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + off0 + sr * NSUB + sc0 + k] =
                    static_cast<uint8_t>(v);
                if (emit) {
#pragma unroll
                  for (int y = 0; y < SB; ++y)
#pragma unroll
                    for (int x = 0; x < SB; ++x) row0p[y * srb + (k * SB + x) * C + ch] = static_cast<uint8_t>(v);
                }
              }
            }
          }
        }
      }
      if constexpr (PAIRS) {
#pragma unroll 1
        for (int vs = 0; vs < NSUB; vs += 2) {
          uint32_t acc0[C], acc1[C];
#pragma unroll
          for (int ch = 0; ch < C; ++ch) acc0[ch] = acc1[ch] = 0;
#pragma unroll
          for (int i = 0; i < SB; ++i) {
            accumulate_row<C>(mystrip + (vs * SB + i) * srb, acc0);
            accumulate_row<C>(mystrip + ((vs + 1) * SB + i) * srb, acc1);
          }
#pragma unroll
          for (int ch = 0; ch < C; ++ch) tot[ch] += acc0[ch] + acc1[ch];
          if (cx_any) {
#pragma unroll
            for (int ch = 0; ch < C; ++ch) {
              acc0[ch] = group_sum<SB4>(acc0[ch]);
              acc1[ch] = group_sum<SB4>(acc1[ch]);
            }
            uint32_t val0[C], val1[C];
            group_values<C, SB4, !PACKED>(a, env_sub, cx, acc0, cs, f, p.r, cell, vs, sc, val0);
            group_values<C, SB4, !PACKED>(a, env_sub, cx, acc1, cs, f, p.r, cell, vs + 1, sc, val1);
            if (cx) {
              if (lic % SB4 == 0) {
                const int64_t off = complex_offset<NSUB * NSUB>(a, gidx, slot_s, S_tot, vs * NSUB + sc);
#pragma unroll
                for (int ch = 0; ch < C; ++ch) {
                  a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + off] = static_cast<uint8_t>(val0[ch]);
                  a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + off + NSUB] =
                      static_cast<uint8_t>(val1[ch]);
                }
              }
              if (emit) {
                uint32_t w0[C], w1[C];
                pattern_words<C>(val0, w0);
                pattern_words<C>(val1, w1);
#pragma unroll
                for (int i = 0; i < SB; ++i)
#pragma unroll
                  for (int q = 0; q < C; ++q) {
                    reinterpret_cast<uint32_t*>(mystrip + (vs * SB + i) * srb)[q] = w0[q];
                    reinterpret_cast<uint32_t*>(mystrip + ((vs + 1) * SB + i) * srb)[q] = w1[q];
                  }
              }
            }
          }
        }
      }
      if constexpr (!PIX) if (!PAIRS && (!VAR || cx_any)) {
#pragma unroll 1
        for (int vs = 0; vs < NSUB; ++vs) {
          uint32_t acc[C];
#pragma unroll
          for (int ch = 0; ch < C; ++ch) acc[ch] = 0;
#pragma unroll
          for (int i = 0; i < SB; ++i) accumulate_row<C>(mystrip + (vs * SB + i) * srb, acc);
          if constexpr (!VAR) {
#pragma unroll
            for (int ch = 0; ch < C; ++ch) tot[ch] += acc[ch];
          }
          if constexpr (STR) {
            if (cx_any) {
              uint32_t part[C];
#pragma unroll
              for (int ch = 0; ch < C; ++ch) part[ch] = 0;
#pragma unroll
              for (int i = 0; i < SB; ++i)
                accumulate_row_masked<C>(mystrip + (vs * SB + i) * srb, str_m, part);
              if (cx) {
                SumT* cs0 = &csum[wq][cw][(vs * NSUB + str_sa) * C];
#pragma unroll
                for (int ch = 0; ch < C; ++ch) {
                  atomicAdd(cs0 + ch, part[ch]);
                  if (str_split < 4) atomicAdd(cs0 + C + ch, acc[ch] - part[ch]);
                }
              }
            }
          } else if (cx_any) {
#pragma unroll
            for (int ch = 0; ch < C; ++ch) acc[ch] = group_sum<SB4>(acc[ch]);
            if constexpr (compact) {
              if (cx && lic % SB4 == 0) {
#pragma unroll
                for (int ch = 0; ch < C; ++ch)
                  csum[wq][cw][(vs * NSUB + sc) * C + ch] = static_cast<SumT>(acc[ch]);
              }
            } else {
              uint32_t val[C];
              group_values<C, SB4, !PACKED>(a, env_sub, cx, acc, cs, f, p.r, cell, vs, sc, val);
              if (cx) {
                if (lic % SB4 == 0) {
                  const int64_t off =
                      VAR ? a.stage_cx + static_cast<int64_t>(gidx) * NN + vs * NSUB + sc
                          : complex_offset<NSUB * NSUB>(a, gidx, slot_s, S_tot, vs * NSUB + sc);
                  uint8_t* dst = VAR ? a.stage : a.stats;
                  const int64_t pst = VAR ? a.stage_stride : a.sstride;
#pragma unroll
                  for (int ch = 0; ch < C; ++ch)
                    dst[static_cast<int64_t>(f * C + ch) * pst + off] = static_cast<uint8_t>(val[ch]);
                }
                if (emit) {
                  uint32_t w[C];
                  pattern_words<C>(val, w);
#pragma unroll
                  for (int i = 0; i < SB; ++i)
#pragma unroll
                    for (int q = 0; q < C; ++q)
                      reinterpret_cast<uint32_t*>(mystrip + (vs * SB + i) * srb)[q] = w[q];
                }
              }
            }
          }
        }
      }
      if constexpr (!VAR) next = load_meta(s_next, lap_next);
      if (compact && cx_any) {
        const unsigned leaders = __ballot_sync(0xFFFFFFFFu, cx && lic == 0);
        if (cx && lic == 0) {
          const int rank = __popc(leaders & ((1u << (t & 31)) - 1u));
          CellRec& rec = crec[wq][rank];
          rec.cw = cw;
          rec.f = f;
          rec.cell = cell;
          rec.gidx = gidx;
          rec.off = VAR ? a.stage_cx + static_cast<int64_t>(gidx) * NN
                        : complex_offset<NSUB * NSUB>(a, gidx, slot_s, S_tot, 0);
#pragma unroll
          for (int ch = 0; ch < C; ++ch) cstate[wq][rank][ch] = cs[ch];
        }
        __syncwarp();
        const int work = __popc(leaders) * NN * C;
        // Keyed stream, bounded fast path: batches of kBatch draws per lane with
        // no calls in the first phase (sums, keys and f32 estimates of all
        // kBatch draws are independent chains the scheduler interleaves; the
        // K1 CTAs run few warps, so one draw at a time is latency-bound), then
        // the rare exact draws and the stores.
        // (Not for VAR: measured slower there, its kernel is register-bound.)
        const bool keyed_fast = !VAR && !env_sub.exact_only && a.noise.kind == DPPX_NOISE_KEYED;
        constexpr int kBatch = 4;
        if (keyed_fast) {
          for (int i0 = 0; i0 < work; i0 += 32 * kBatch) {
            uint32_t sum[kBatch], q[kBatch];
            uint64_t bits[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
              const int i = min(i0 + j * 32 + (t & 31), work - 1);  // clamped: always valid
              const int kk = i / (NN * C), rem = i - kk * (NN * C);
              const int sidx = rem / C, ch = rem - sidx * C;
              const int vs = sidx / NSUB, sc2 = sidx - vs * NSUB;
              sum[j] = csum[wq][crec[wq][kk].cw][rem];
              bits[j] = key_sub(cstate[wq][kk][ch], vs, sc2);
              q[j] = fast_quantize(sum[j], env_sub.inv_area, bits[j], env_sub.sln2, env_sub.margin);
            }
            __syncwarp();  // all of the batch's sums are read before any is overwritten
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
              const int i = i0 + j * 32 + (t & 31);
              if (i < work) {
                const int kk = i / (NN * C), rem = i - kk * (NN * C);
                const int sidx = rem / C, ch = rem - sidx * C;
                const CellRec& rec = crec[wq][kk];
                uint32_t v = q[j];
                if (v == 0xFFFFFFFFu) v = exact_quantize(sum[j], env_sub.area, env_sub.kind, bits[j], env_sub.sigma, 0.0);
                uint8_t* base = VAR ? a.stage + static_cast<int64_t>(rec.f * C + ch) * a.stage_stride
                                    : a.stats + static_cast<int64_t>(rec.f * C + ch) * a.sstride;
                base[rec.off + sidx] = static_cast<uint8_t>(v);
                csum[wq][rec.cw][rem] = static_cast<SumT>(v);
              }
            }
          }
        } else {
          for (int i = t & 31; i < work; i += 32) {
            const int kk = i / (NN * C), rem = i - kk * (NN * C);
            const int sidx = rem / C, ch = rem - sidx * C;
            const int vs = sidx / NSUB, sc2 = sidx - vs * NSUB;
            const CellRec& rec = crec[wq][kk];
            const uint32_t sum = csum[wq][rec.cw][rem];
            const uint32_t v =
                draw_stat(a, env_sub, sum, cstate[wq][kk][ch], rec.f, ch, p.r, rec.cell, vs, sc2, rec.gidx);
            uint8_t* base = VAR ? a.stage + static_cast<int64_t>(rec.f * C + ch) * a.stage_stride
                                : a.stats + static_cast<int64_t>(rec.f * C + ch) * a.sstride;
            base[rec.off + sidx] = static_cast<uint8_t>(v);
            csum[wq][rec.cw][rem] = static_cast<SumT>(v);
          }
        }
        __syncwarp();
        if (emit && cx) {
#pragma unroll 1
          for (int vs = 0; vs < NSUB; ++vs) {
            uint32_t val[C];
            uint32_t w[C];
            if constexpr (STR) {
              uint32_t vb[C];
              const SumT* cs0 = &csum[wq][cw][(vs * NSUB + str_sa) * C];
#pragma unroll
              for (int ch = 0; ch < C; ++ch) {
                val[ch] = cs0[ch];
                vb[ch] = str_split < 4 ? cs0[C + ch] : val[ch];
              }
              pattern_words_split<C>(val, vb, str_split, w);
            } else {
#pragma unroll
              for (int ch = 0; ch < C; ++ch) val[ch] = csum[wq][cw][(vs * NSUB + sc) * C + ch];
              pattern_words<C>(val, w);
            }
#pragma unroll
            for (int i = 0; i < SB; ++i)
#pragma unroll
              for (int q = 0; q < C; ++q)
                reinterpret_cast<uint32_t*>(mystrip + (vs * SB + i) * srb)[q] = w[q];
          }
        }
      }
    } else if constexpr (RPU == 1) {
#pragma unroll
      for (int i = 0; i < B; ++i) accumulate_row<C>(mystrip + i * srb, tot);
      // Next unit's metadata: requested here (after the staged rows are
      // summed) rather than at the top, so a 2-stage ring never stalls on the
      // producer's previous store; its latency hides behind the epilogue.
      next = load_meta(s_next, lap_next);
    }

    if constexpr (RPU > 1) {
      // Uniform, RPU cell rows of this band: the same per-cell work as below,
      // once per cell row (a band's last rows may lie past the grid: skipped).
#ifndef DPPX_META_AT
#define DPPX_META_AT 2
#endif
      if (DPPX_META_AT == 0) next = load_meta(s_next, lap_next);
#pragma unroll 1
      for (int q = 0; q < RPU; ++q) {
        const int rq = p.r * RPU + q;
        const bool rok = active && rq < a.row_begin + a.row_count;
        uint32_t tq[C];
#pragma unroll
        for (int ch = 0; ch < C; ++ch) tq[ch] = 0;
#pragma unroll
        for (int i = 0; i < B; ++i) accumulate_row<C>(mystrip + (q * B + i) * srb, tq);
        if (DPPX_META_AT == 1 && q == RPU - 1) next = load_meta(s_next, lap_next);
#pragma unroll
        for (int ch = 0; ch < C; ++ch) tq[ch] = group_sum<B4>(tq[ch]);
        uint64_t csq[C];
#pragma unroll
        for (int ch = 0; ch < C; ++ch)
          csq[ch] = a.noise.kind == DPPX_NOISE_KEYED ? key_cell(cur.seed[ch], rq, cell) : 0ull;
        uint32_t val[C];
        group_values<C, B4, !PACKED>(a, env_cell, rok, tq, csq, f, rq, cell, 0, 0, val);
        if (rok) {
          if (lic == 0) {
            const int64_t off = static_cast<int64_t>(rq) * g.GC + cell;
#pragma unroll
            for (int ch = 0; ch < C; ++ch)
              a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + off] = static_cast<uint8_t>(val[ch]);
          }
          if (emit) {
            uint32_t w[C];
            pattern_words<C>(val, w);
#pragma unroll
            for (int i = 0; i < B; ++i)
#pragma unroll
              for (int qq = 0; qq < C; ++qq)
                reinterpret_cast<uint32_t*>(mystrip + (q * B + i) * srb)[qq] = w[qq];
          }
        }
      }
      if (DPPX_META_AT == 2) next = load_meta(s_next, lap_next);
    }

    // whole cell (uniform, or adaptive simple): reduce over B4 strips.
    if constexpr (RPU == 1) {
#pragma unroll
    for (int ch = 0; ch < C; ++ch) tot[ch] = group_sum<B4>(tot[ch]);
    {
      uint32_t val[C];
      group_values<C, B4, !PACKED>(a, env_cell, active && simple, tot, cs, f, p.r, cell, 0, 0, val);
      if (active && simple) {
        if (lic == 0) {
          if constexpr (VAR) {
#pragma unroll
            for (int ch = 0; ch < C; ++ch)
              a.stage[static_cast<int64_t>(f * C + ch) * a.stage_stride + gidx] =
                  static_cast<uint8_t>(val[ch]);
          } else {
            const int64_t off = stat_offset(a, true, gidx, slot_s, S_tot, 0, 0);
#pragma unroll
            for (int ch = 0; ch < C; ++ch)
              a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + off] =
                  static_cast<uint8_t>(val[ch]);
          }
        }
        if (emit) {
          uint32_t w[C];
          pattern_words<C>(val, w);
#pragma unroll
          for (int i = 0; i < B; ++i)
#pragma unroll
            for (int q = 0; q < C; ++q) reinterpret_cast<uint32_t*>(mystrip + i * srb)[q] = w[q];
        }
      }
    }
    }  // RPU == 1

    fence_proxy_async_smem();
    mbar_arrive(&done_bar[s]);
    s = s_next;
    lap = lap_next;
  }
}

// ============================================================================
// K1u: uniform pixelization (n = 1) for grid sides that are not a multiple of
// 4 px (the paper's b = 2..20 sweep, b = 30 for Venice-2). Same producer (TMA
// box loads / stores, 2-stage ring, dynamic unit claims) as K1; tiles are whole
// cells and a multiple of 16 px (TILE = lcm(b, 16) * k <= 512). A consumer's
// 4-px strip meets at most two cells (b >= 2): it splits its per-channel row
// sums at the cell boundary (dp4a byte masks), both parts meet in a per-CTA
// smem cell table (shared-memory atomics), one thread per (cell, channel)
// draws, and each strip writes its reconstructed pixels from the table.
// ============================================================================
constexpr int ku_gcd(int x, int y) { return y == 0 ? x : ku_gcd(y, x % y); }
constexpr int ku_lcm16(int b) { return b * 16 / ku_gcd(b, 16); }
// Whole cells, a multiple of 16 px, <= 512 px and <= ~100 KB per RGB stage
// (b = 128: 256-px tiles, two 98 KB stages).
constexpr int ku_tile(int b) {
  return ku_lcm16(b) * (((512 < 102400 / (3 * b)) ? 512 : 102400 / (3 * b)) / ku_lcm16(b) > 0
                            ? ((512 < 102400 / (3 * b)) ? 512 : 102400 / (3 * b)) / ku_lcm16(b)
                            : 1);
}

// K1a / K2a tiles (b = 128: 128 px, so the subcell tables fit beside two stages).
constexpr int ka_tile(int b) { return b == 128 ? 128 : ku_tile(b); }

template <int C, int B>
__global__ void __launch_bounds__(kStatsThreads)
    k_uniform_tma(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                  const StatsArgs a) {
  constexpr int TILE = ku_tile(B);
  constexpr int ROWB = TILE * C;
  constexpr uint32_t STAGE = (B * ROWB + 127) & ~127;  // TMA destinations: 128-byte aligned
  constexpr int NCELL = TILE / B;  // cells per tile
  constexpr int NSTRIP = TILE / 4;
  static_assert(B >= 2 && (B % 4 != 0 || B == 128) && TILE % B == 0 && TILE % 16 == 0 &&
                    NSTRIP <= kConsumers,
                "K1u geometry");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t id_bar[kMaxStages];
  __shared__ __align__(8) uint64_t done_bar[kMaxStages];
  __shared__ int stage_unit[kMaxStages];
  __shared__ uint32_t cellsum[NCELL * C];
  __shared__ uint8_t cellval[NCELL * C];

  const int S = a.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&id_bar[s], 1);
      mbar_init(&done_bar[s], kConsumers);
    }
    fence_mbarrier_init();
  }
  for (int i = threadIdx.x; i < NCELL * C; i += blockDim.x) cellsum[i] = 0;
  __syncthreads();

  if (warp == kConsumers / 32) {  // producer warp, as in k_stats_tma
    if (lane == 0) {
      prefetch_tmap(&tm_in);
      prefetch_tmap(&tm_out);
    }
    auto finish_unit = [&](int s, int use) {
      mbar_wait(&done_bar[s], use & 1);
      if (a.out) {
        const int uu = stage_unit[s];
        store_tail<C, B, false, TILE>(a, uu, smem + s * STAGE, lane);
        if (lane == 0) store_unit<C, B, false, TILE>(a, &tm_out, uu, smem + s * STAGE);
      }
      __syncwarp();
    };
    int k = 0, done_units = 0;
    for (;; ++k) {
      const int s = ring_slot(k, S);
      if (k >= S) {
        finish_unit(s, ring_lap(k, S) - 1);
        ++done_units;
      }
      int u = 0;
      if (lane == 0) {
        u = atomicAdd(a.work_counter, 1);
        if (u >= a.units) {
          if (u == a.units + static_cast<int>(gridDim.x) - 1) atomicExch(a.work_counter, 0);
          u = -1;
        }
        stage_unit[s] = u;
        mbar_arrive(&id_bar[s]);
        if (u < 0)
          mbar_arrive_expect_tx(&full_bar[s], 0);
        else
          load_unit<C, B, false, TILE>(a, &tm_in, u, smem + s * STAGE, &full_bar[s]);
      }
      u = __shfl_sync(0xFFFFFFFFu, u, 0);
      if (u < 0) break;
    }
    for (int j = done_units; j < k; ++j) finish_unit(ring_slot(j, S), ring_lap(j, S));
    if (lane == 0) bulk_wait_all();
    return;
  }

  // ---------------- consumer warps ----------------
  const int t = threadIdx.x;
  const BatchGeom& g = a.g;
  const DrawEnv env_cell = make_env(a.noise.kind, a.exact_noise != 0, a.area, a.sigma);
  const bool strip_ok = t < NSTRIP;
  const int lpx = 4 * (strip_ok ? t : 0);
  const int ca = lpx / B;                          // first cell of the strip (in the tile)
  const int split = min(4, (ca + 1) * B - lpx);    // pixels [0, split) are in cell ca
  uint32_t m[C][C == 4 ? 4 : C];
#pragma unroll
  for (int ch = 0; ch < C; ++ch)
#pragma unroll
    for (int q = 0; q < (C == 4 ? 4 : C); ++q) m[ch][q] = 0;
#pragma unroll
  for (int pos = 0; pos < 4 * C; ++pos)
    if (pos / C < split) m[pos % C][pos / 4] |= 1u << (8 * (pos % 4));

  for (int k = 0;; ++k) {
    const int s = ring_slot(k, S);
    uint8_t* st = smem + s * STAGE;
    mbar_wait(&id_bar[s], ring_lap(k, S) & 1);
    const int u = *reinterpret_cast<volatile int*>(&stage_unit[s]);
    if (u < 0) break;
    const UnitPos p = decode_unit<false, TILE>(a, u);
    const int f = p.fg;
    const int cell0 = p.px0 / B;
    const int ncell = min(NCELL, g.GC - cell0);
    const bool active = strip_ok && ca < ncell;
    const bool has_b = split < 4 && ca + 1 < ncell;
    const int vbytes = valid_bytes<C, false, TILE>(a, p.px0);
    const int copy = staged_bytes<C, B, false, TILE>(a, p);
    const int need = min(TILE, g.GC * B - p.px0) * C;

    mbar_wait(&full_bar[s], ring_lap(k, S) & 1);
    // Mirrored padding columns and any unstaged row tail (as k_stats_tma).
    const int fs = min(copy, vbytes);
    if (fs < need) {
      constexpr int kLanes = 4;
      for (int pr = t / kLanes; pr < B; pr += kConsumers / kLanes) {
        uint8_t* rowp = st + pr * ROWB;
        const int srow = reflect_index(p.r * B + pr, g.M);
        const uint8_t* grow = a.img + static_cast<int64_t>(f) * a.fstride + static_cast<int64_t>(srow) * a.pitch;
        for (int x = fs + (t % kLanes); x < need; x += kLanes) {
          const int cpx = x / C, ch = x - cpx * C;
          const int spx = reflect_index(p.px0 + cpx, g.N);
          const int sx = (spx - p.px0) * C + ch;
          rowp[x] = (sx >= 0 && sx < fs) ? rowp[sx] : __ldg(grow + static_cast<int64_t>(spx) * C + ch);
        }
      }
      named_bar_sync(1, kConsumers);
    }

    // Strip sums over the band, split at the cell boundary.
    uint32_t acc[C], part[C];
#pragma unroll
    for (int ch = 0; ch < C; ++ch) acc[ch] = part[ch] = 0;
    const uint8_t* mystrip = st + lpx * C;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      accumulate_row<C>(mystrip + i * ROWB, acc);
      accumulate_row_masked<C>(mystrip + i * ROWB, m, part);
    }
    if constexpr (B == 2) {
      // b = 2: a strip holds exactly its two cells, so the lane draws them
      // itself (no cell table, atomics or barriers); neighbouring lanes'
      // statistic stores stay contiguous per plane.
      if (active) {
        uint32_t va[C], vb[C];
        const int gca = cell0 + ca, gidx = p.r * g.GC + gca;
#pragma unroll
        for (int ch = 0; ch < C; ++ch) {
          uint8_t* plane = a.stats + static_cast<int64_t>(f * C + ch) * a.sstride + gidx;
          va[ch] = draw_stat(a, env_cell, part[ch], cell_state(a, f, ch, p.r, gca), f, ch, p.r, gca, 0, 0, gidx);
          plane[0] = static_cast<uint8_t>(va[ch]);
          vb[ch] = va[ch];
          if (has_b) {
            vb[ch] = draw_stat(a, env_cell, acc[ch] - part[ch], cell_state(a, f, ch, p.r, gca + 1), f, ch, p.r,
                               gca + 1, 0, 0, gidx + 1);
            plane[1] = static_cast<uint8_t>(vb[ch]);
          }
        }
        if (a.out) {
          uint32_t w[C == 4 ? 4 : C];
          pattern_words_split<C>(va, vb, split, w);
          uint8_t* ms = st + lpx * C;
#pragma unroll
          for (int i = 0; i < B; ++i)
#pragma unroll
            for (int q = 0; q < (C == 4 ? 4 : C); ++q) reinterpret_cast<uint32_t*>(ms + i * ROWB)[q] = w[q];
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&done_bar[s]);
      continue;
    }
    if (active) {
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        atomicAdd(&cellsum[ca * C + ch], part[ch]);
        if (has_b) atomicAdd(&cellsum[(ca + 1) * C + ch], acc[ch] - part[ch]);
      }
    }
    named_bar_sync(1, kConsumers);
    // One draw per (cell, channel): channel-major items so a warp's statistic
    // stores are contiguous in each plane.
    // Channel-major items. Small cells (many draws per unit): the compile-time
    // tile cell count as divisor, skipping cells past the frame (last tile);
    // larger cells: the runtime count (measured faster there, e.g. b = 11).
    constexpr bool kStaticItems = B <= 8;
    const int icell = kStaticItems ? NCELL : ncell;
    for (int item = t; item < icell * C; item += kConsumers) {
      const int ch = kStaticItems ? item / NCELL : item / ncell;
      const int c = item - ch * icell;
      if (kStaticItems && c >= ncell) continue;
      const int gc = cell0 + c, gidx = p.r * g.GC + gc;
      const uint32_t sum = cellsum[c * C + ch];
      cellsum[c * C + ch] = 0;  // ready for the next unit
      const uint32_t v = draw_stat(a, env_cell, sum, cell_state(a, f, ch, p.r, gc), f, ch, p.r, gc, 0, 0, gidx);
      a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + gidx] = static_cast<uint8_t>(v);
      cellval[c * C + ch] = static_cast<uint8_t>(v);
    }
    named_bar_sync(1, kConsumers);
    if (a.out && active) {
      uint32_t va[C], vb[C];
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        va[ch] = cellval[ca * C + ch];
        vb[ch] = has_b ? cellval[(ca + 1) * C + ch] : va[ch];
      }
      uint32_t w[C == 4 ? 4 : C];
      pattern_words_split<C>(va, vb, split, w);
      uint8_t* ms = st + lpx * C;
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q < (C == 4 ? 4 : C); ++q) reinterpret_cast<uint32_t*>(ms + i * ROWB)[q] = w[q];
    }
    fence_proxy_async_smem();
    mbar_arrive(&done_bar[s]);
  }
}


// ============================================================================
// K2 fast path: one CTA per (frame, grid row, TILE-px tile); each thread owns a
// 4-px strip, looks up its cell's statistics per channel plane (packed slots
// from K0's per-plane scan), writes the strip pattern into a smem tile and one
// thread bulk-stores the tile with a 3-D TMA box (clipped at M and N).
// ============================================================================
// Packed (narrow-frame) instantiations run 256 threads: a 1024-px tile holds
// more frame slots per CTA (5 CelebA frames instead of 2).
constexpr int kExpandPackedThreads = 256;

// HALF: a unit is half a band (B/2 rows; b >= 32): half the smem per CTA, so
// twice the CTAs per SM hide the statistics-load latency (4K b32 n8: a 49 KB
// tile allowed 4 CTAs/SM).
template <int C, int B4, int NSUB, bool ADAPTIVE, bool PACKED, int H = 1>
__global__ void __launch_bounds__(PACKED ? kExpandPackedThreads : kConsumers)
    k_expand_tma(const __grid_constant__ CUtensorMap tm_out, const ExpandArgs a) {
  constexpr int B = 4 * B4, SB = B / NSUB, SB4 = SB / 4;
  constexpr bool HALF = H > 1;
  constexpr int RU = B / H;                             // rows per unit
  constexpr int NV = NSUB >= H ? NSUB / H : 1;          // vertical subcells per unit
  constexpr int SBR = NSUB >= H ? SB : RU;              // rows per emitted subcell
  static_assert(!HALF || (!PACKED && (NSUB == 1 || NSUB % H == 0) && RU % 4 == 0), "band-split geometry");
  constexpr bool PIX = SB <= 2 && NSUB > 1;  // 1- or 2-px subcells: each pixel's own payload byte
  constexpr int KS = PIX ? 4 / SB : 1;       // subcells per strip and subcell row
  constexpr bool STR = (SB % 4) != 0 && !PIX;  // strips meet two subcells (as K1)
  static_assert(!STR || (ADAPTIVE && SB >= 2), "split strips: adaptive, subcells of >= 2 px");
  static_assert(!PIX || (ADAPTIVE && H == 1), "per-pixel subcells: adaptive, whole bands");
  constexpr int LPW = (32 / B4) * B4;                    // whole cells per warp (as K1)
  constexpr int NT = PACKED ? kExpandPackedThreads : kConsumers;
  constexpr int TILE = 4 * (NT / 32) * LPW;
  static_assert(!PACKED || LPW == 32, "packed slots need power-of-two cells");
  extern __shared__ __align__(128) uint8_t smem[];
  const BatchGeom& g = a.g;
  const int t = threadIdx.x;
  const bool strip_ok = (t & 31) < LPW;
  const int sx = strip_ok ? (t >> 5) * LPW + (t & 31) : 0;  // strip index in the tile
  // This thread's slot (frame within the group) and strip column in it.
  const int slot_px = PACKED ? a.slot_px : TILE;
  const int my_j = PACKED ? (4 * sx) / slot_px : 0;
  const bool in_slot = strip_ok && my_j < (PACKED ? a.pack : 1);
  const int jj = in_slot ? my_j : 0;
  const int lpx = 4 * sx - jj * slot_px;
  const int srb = slot_px * C;  // smem bytes per slot row
  const int sc = (STR || PIX) ? 0 : (sx % B4) / (SB4 > 0 ? SB4 : 1);
  const int str_px = 4 * (sx % B4);
  const int str_sa = STR ? str_px / SB : 0;
  const int str_split = STR ? min(4, (str_sa + 1) * SB - str_px) : 4;
  for (int u = blockIdx.x, k = 0; u < a.units; u += gridDim.x, ++k) {
    uint8_t* buf = smem;
    // A capped grid loops: the previous unit's store must have read the tile.
    if (t == 0 && k > 0) bulk_wait_read_all();
    __syncthreads();
    const int hh = HALF ? (u % H) : 0;  // which part of the band
    const int uu = HALF ? (u / H) : u;
    const uint32_t rest = a.div_tiles.div(static_cast<uint32_t>(uu));
    const int tile = uu - static_cast<int>(rest * a.div_tiles.d);
    const uint32_t fq = a.div_rows.div(rest);
    const int r = static_cast<int>(rest - fq * a.div_rows.d);
    const int fg = static_cast<int>(fq);
    const int row0 = r * B + hh * RU;  // first frame row of this unit
    const int pk = PACKED ? a.pack : 1;
    const int nf = PACKED ? min(pk, g.F - fg * pk) : 1;
    const int f = fg * pk + jj;
    const int px0 = PACKED ? 0 : tile * TILE;
    const int cell = (px0 + lpx) / B;
    const bool active = in_slot && jj < nf && cell < g.GC;
    const int gidx = r * g.GC + cell;
    if constexpr (PIX) {
      // simple cells: one value per channel over the band; complex cells: the
      // payload byte of every pixel (row i, column 4 * lane-in-cell + px)
      if (active) {
        uint8_t* mystrip = buf + jj * (PACKED ? a.slot_stride : 0) + lpx * C;
        const int64_t base = 4ll * g.G + 4;
        const int sc0 = KS * (sx % B4);
        const int64_t plane0 = static_cast<int64_t>(f) * C;
        const uint32_t info = __ldg(&a.cellinfo[plane0 * g.G + gidx]);
        const uint32_t slot_s = __ldg(&a.rowprefix[plane0 * g.GR + r]) + (info >> 1);
        if (info & 1u) {
          uint32_t vv[C];
#pragma unroll
          for (int ch = 0; ch < C; ++ch) vv[ch] = __ldg(a.stats + (plane0 + ch) * a.sstride + base + slot_s);
          uint32_t w[C];
          pattern_words<C>(vv, w);
#pragma unroll 4
          for (int i = 0; i < RU; ++i)
#pragma unroll
            for (int q = 0; q < C; ++q) reinterpret_cast<uint32_t*>(mystrip + i * srb)[q] = w[q];
        } else {
          const uint8_t* sub[C];
#pragma unroll
          for (int ch = 0; ch < C; ++ch)
            sub[ch] = a.stats + (plane0 + ch) * a.sstride + base + __ldg(&a.totals[plane0 + ch]) +
                      static_cast<int64_t>(static_cast<uint32_t>(gidx) - slot_s) * NSUB * NSUB + sc0;
#pragma unroll 1
          for (int i = 0; i < RU; ++i) {
            uint8_t* row = mystrip + i * srb;
#pragma unroll
            for (int q = 0; q < 4 * C; ++q) row[q] = __ldg(sub[q % C] + (i / SB) * NSUB + (q / C) / SB);
          }
        }
      }
    } else {
    uint32_t val[NV][C];
    uint32_t valb[STR ? NV : 1][C];  // STR: the strip's second subcell
    if (active) {
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        const int64_t plane = static_cast<int64_t>(f) * C + ch;
        const uint8_t* st = a.stats + plane * a.sstride;
        if constexpr (!ADAPTIVE) {
          const uint32_t v = __ldg(st + gidx);
#pragma unroll
          for (int vs = 0; vs < NV; ++vs) val[vs][ch] = v;
        } else {
          const uint32_t info = __ldg(&a.cellinfo[plane * g.G + gidx]);
          const uint32_t slot_s = __ldg(&a.rowprefix[plane * g.GR + r]) + (info >> 1);
          const int64_t base = 4ll * g.G + 4;
          if (info & 1u) {
            const uint32_t v = __ldg(st + base + slot_s);
#pragma unroll
            for (int vs = 0; vs < NV; ++vs) {
              val[vs][ch] = v;
              if constexpr (STR) valb[vs][ch] = v;
            }
          } else {
            const uint8_t* sub = st + base + __ldg(&a.totals[plane]) +
                                 static_cast<int64_t>(static_cast<uint32_t>(gidx) - slot_s) * NSUB * NSUB;
#pragma unroll
            for (int vs = 0; vs < NV; ++vs) {
              const int vg = NSUB >= H ? hh * NV + vs : 0;  // vertical subcell in the cell
              if constexpr (STR) {
                val[vs][ch] = __ldg(sub + vg * NSUB + str_sa);
                valb[vs][ch] = str_split < 4 ? __ldg(sub + vg * NSUB + str_sa + 1) : val[vs][ch];
              } else {
                val[vs][ch] = __ldg(sub + vg * NSUB + sc);
              }
            }
          }
        }
      }
      uint8_t* mystrip = buf + jj * (PACKED ? a.slot_stride : 0) + lpx * C;
#pragma unroll
      for (int vs = 0; vs < NV; ++vs) {
        uint32_t w[C];
        if constexpr (STR)
          pattern_words_split<C>(val[vs], valb[vs], str_split, w);
        else
          pattern_words<C>(val[vs], w);
#pragma unroll
        for (int i = 0; i < SBR; ++i)
#pragma unroll
          for (int q = 0; q < C; ++q)
            reinterpret_cast<uint32_t*>(mystrip + (vs * SBR + i) * srb)[q] = w[q];
      }
    }
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int scopy = max(0, min(srb, a.tensor_out_bytes - px0 * C));
    if (t == 0 && scopy > 0) {
      for (int j = 0; j < nf; ++j)
        tma_store_3d(&tm_out, px0 * C / 8, row0, fg * pk + j, buf + j * (PACKED ? a.slot_stride : 0));
    }
    if (t == 0) bulk_commit();  // one group per unit (possibly empty)
    // Bytes past the tensor's row extent (< 16 per row and slot), from the smem
    // tile, spread over the whole CTA (one thread per byte, not per strip).
    const int vbytes = min(slot_px, g.N - px0) * C;
    const int span = vbytes - scopy;
    if (span > 0) {
      const int rows = min(RU, g.M - row0);
      for (int e = t; e < nf * rows; e += NT) {  // one row per thread
        const int j = e / rows, i = e - j * rows;
        copy_row_tail(a.out + static_cast<int64_t>(fg * pk + j) * a.ofstride +
                          static_cast<int64_t>(row0 + i) * a.opitch + static_cast<int64_t>(px0) * C + scopy,
                      buf + j * (PACKED ? a.slot_stride : 0) + i * srb + scopy, span);
      }
    }
  }
  if (t == 0) bulk_wait_read_all();  // smem must outlive the stores' reads
}

// K2u: broadcast_means for the K1u grid sides (uniform, b % 4 != 0 or b = 128):
// K1u's tiles of whole cells; each 4-px strip takes the values of the (at most
// two) cells it meets and writes its pixels into a smem tile, stored with one
// 3-D TMA box (the < 16 bytes past the tensor's row extent by the CTA).
template <int C, int B>
__global__ void __launch_bounds__(kConsumers) k_expand_uany(const __grid_constant__ CUtensorMap tm_out,
                                                            const ExpandArgs a) {
  constexpr int TILE = ku_tile(B);
  constexpr int ROWB = TILE * C;
  constexpr int NCELL = TILE / B;
  constexpr int NSTRIP = TILE / 4;
  static_assert(NSTRIP <= kConsumers && TILE % B == 0, "K2u geometry");
  extern __shared__ __align__(128) uint8_t smem[];
  const BatchGeom& g = a.g;
  const int t = threadIdx.x;
  const bool strip_ok = t < NSTRIP;
  const int lpx = 4 * (strip_ok ? t : 0);
  const int ca = lpx / B;
  const int split = min(4, (ca + 1) * B - lpx);
  for (int u = blockIdx.x, k = 0; u < a.units; u += gridDim.x, ++k) {
    if (t == 0 && k > 0) bulk_wait_read_all();
    __syncthreads();
    const uint32_t rest = a.div_tiles.div(static_cast<uint32_t>(u));
    const int tile = u - static_cast<int>(rest * a.div_tiles.d);
    const uint32_t fq = a.div_rows.div(rest);
    const int r = static_cast<int>(rest - fq * a.div_rows.d);
    const int f = static_cast<int>(fq);
    const int px0 = tile * TILE;
    const int cell0 = px0 / B;
    const int ncell = min(NCELL, g.GC - cell0);
    const bool active = strip_ok && ca < ncell;
    const bool has_b = split < 4 && ca + 1 < ncell;
    if (active) {
      uint32_t va[C], vb[C];
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        const uint8_t* st = a.stats + (static_cast<int64_t>(f) * C + ch) * a.sstride + r * g.GC + cell0 + ca;
        va[ch] = __ldg(st);
        vb[ch] = has_b ? __ldg(st + 1) : va[ch];
      }
      uint32_t w[C == 4 ? 4 : C];
      pattern_words_split<C>(va, vb, split, w);
#pragma unroll 4
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int q = 0; q < (C == 4 ? 4 : C); ++q)
          reinterpret_cast<uint32_t*>(smem + i * ROWB + lpx * C)[q] = w[q];
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int scopy = max(0, min(ROWB, a.tensor_out_bytes - px0 * C));
    if (t == 0 && scopy > 0) tma_store_3d(&tm_out, px0 * C / 8, r * B, f, smem);
    if (t == 0) bulk_commit();
    const int vbytes = min(TILE, g.N - px0) * C;
    const int span = vbytes - scopy;
    if (span > 0) {
      const int rows = min(B, g.M - r * B);
      for (int i = t; i < rows; i += kConsumers)  // one row per thread
        copy_row_tail(a.out + static_cast<int64_t>(f) * a.ofstride + static_cast<int64_t>(r * B + i) * a.opitch +
                          static_cast<int64_t>(px0) * C + scopy,
                      smem + i * ROWB + scopy, span);
    }
  }
  if (t == 0) bulk_wait_read_all();
}

// K2a: reassemble for the K1a grid sides (adaptive b = 30, b = 128): K1a's
// tiles; per vertical subcell each strip takes the values of the (at most
// two) subcell columns it meets — a simple cell's value or the complex cell's
// subcell value from the packed payload (K0 run on the payload) — and writes
// its pixels into a smem tile stored with one TMA box.
template <int C, int B, int NSUB>
__global__ void __launch_bounds__(kConsumers) k_expand_aany(const __grid_constant__ CUtensorMap tm_out,
                                                            const ExpandArgs a) {
  constexpr int TILE = ka_tile(B);
  constexpr int ROWB = TILE * C;
  constexpr int SB = B / NSUB;
  constexpr int NSTRIP = TILE / 4;
  constexpr int NN = NSUB * NSUB;
  static_assert(NSTRIP <= kConsumers && TILE % B == 0 && SB >= 2, "K2a geometry");
  extern __shared__ __align__(128) uint8_t smem[];
  const BatchGeom& g = a.g;
  const int t = threadIdx.x;
  const bool strip_ok = t < NSTRIP;
  const int lpx = 4 * (strip_ok ? t : 0);
  const int sa = lpx / SB;
  const int split = min(4, (sa + 1) * SB - lpx);
  const int ca = sa / NSUB, sca = sa - ca * NSUB;
  const int cb = (sa + 1) / NSUB, scb = (sa + 1) - cb * NSUB;
  for (int u = blockIdx.x, k = 0; u < a.units; u += gridDim.x, ++k) {
    if (t == 0 && k > 0) bulk_wait_read_all();
    __syncthreads();
    const uint32_t rest = a.div_tiles.div(static_cast<uint32_t>(u));
    const int tile = u - static_cast<int>(rest * a.div_tiles.d);
    const uint32_t fq = a.div_rows.div(rest);
    const int r = static_cast<int>(rest - fq * a.div_rows.d);
    const int f = static_cast<int>(fq);
    const int px0 = tile * TILE;
    const int cell0 = px0 / B;
    const int nsc = min(TILE / B, g.GC - cell0) * NSUB;
    const bool active = strip_ok && sa < nsc;
    const bool has_b = split < 4 && sa + 1 < nsc;
    if (active) {
      // Per channel: where the strip's two subcell columns take their values.
      const uint8_t* pa[C];
      const uint8_t* pb[C];
      int stepa[C], stepb[C];  // 0: simple cell (one value), NSUB: complex (per vertical subcell)
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        const int64_t plane = static_cast<int64_t>(f) * C + ch;
        const uint8_t* st = a.stats + plane * a.sstride;
        const uint32_t rowpre = __ldg(&a.rowprefix[plane * g.GR + r]);
        const uint32_t tot = __ldg(&a.totals[plane]);
        const int64_t base = 4ll * g.G + 4;
        auto where = [&](int c, int sc, const uint8_t*& ptr, int& step) {
          const int gidx = r * g.GC + cell0 + c;
          const uint32_t info = __ldg(&a.cellinfo[plane * g.G + gidx]);
          const uint32_t slot_s = rowpre + (info >> 1);
          if (info & 1u) {
            ptr = st + base + slot_s;
            step = 0;
          } else {
            ptr = st + base + tot + static_cast<int64_t>(static_cast<uint32_t>(gidx) - slot_s) * NN + sc;
            step = NSUB;
          }
        };
        where(ca, sca, pa[ch], stepa[ch]);
        if (has_b) {
          where(cb, scb, pb[ch], stepb[ch]);
        } else {
          pb[ch] = pa[ch];
          stepb[ch] = stepa[ch];
        }
      }
#pragma unroll 1
      for (int vs = 0; vs < NSUB; ++vs) {
        uint32_t va[C], vb[C];
#pragma unroll
        for (int ch = 0; ch < C; ++ch) {
          va[ch] = __ldg(pa[ch] + vs * stepa[ch]);
          vb[ch] = __ldg(pb[ch] + vs * stepb[ch]);
        }
        uint32_t w[C == 4 ? 4 : C];
        pattern_words_split<C>(va, vb, has_b ? split : 4, w);
#pragma unroll 2
        for (int i = 0; i < SB; ++i)
#pragma unroll
          for (int q = 0; q < (C == 4 ? 4 : C); ++q)
            reinterpret_cast<uint32_t*>(smem + (vs * SB + i) * ROWB + lpx * C)[q] = w[q];
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int scopy = max(0, min(ROWB, a.tensor_out_bytes - px0 * C));
    if (t == 0 && scopy > 0) tma_store_3d(&tm_out, px0 * C / 8, r * B, f, smem);
    if (t == 0) bulk_commit();
    const int vbytes = min(TILE, g.N - px0) * C;
    const int span = vbytes - scopy;
    if (span > 0) {
      const int rows = min(B, g.M - r * B);
      for (int i = t; i < rows; i += kConsumers)  // one row per thread
        copy_row_tail(a.out + static_cast<int64_t>(f) * a.ofstride + static_cast<int64_t>(r * B + i) * a.opitch +
                          static_cast<int64_t>(px0) * C + scopy,
                      smem + i * ROWB + scopy, span);
    }
  }
  if (t == 0) bulk_wait_read_all();
}

using StatsKernel = void (*)(const CUtensorMap, const CUtensorMap, const StatsArgs);
using ExpandKernel = void (*)(const CUtensorMap, const ExpandArgs);

// K1a: the adaptive counterpart of K1u (PPM-100's b = 128 with n = 2..32, and
// b = 30): same producer and tiles of whole cells (b = 128: 128-px tiles, one
// cell, so the subcell tables fit beside two 49 KB stages). Per vertical
// subcell row, each strip splits its row sums at the subcell boundary into a
// per-CTA smem subcell table (atomics); then one pass over (vertical subcell,
// subcell column, channel): complex cells draw their subcells at sigma_sub,
// the (0, 0) item of a simple cell sums its n x n entries and draws the cell at
// sigma; the strips then write their pixels from the value tables.

template <int C, int B, int NSUB>
__global__ void __launch_bounds__(kStatsThreads)
    k_adaptive_any_tma(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                       const StatsArgs a) {
  constexpr int TILE = ka_tile(B);
  constexpr int ROWB = TILE * C;
  constexpr uint32_t STAGE = (B * ROWB + 127) & ~127;
  constexpr int SB = B / NSUB;            // subcell side
  constexpr int NCELL = TILE / B;
  constexpr int SC = TILE / SB;           // subcell columns per tile
  constexpr int NSTRIP = TILE / 4;
  static_assert(B % NSUB == 0 && SB >= 2 && TILE % B == 0 && TILE % 16 == 0 && NSTRIP <= kConsumers &&
                    NCELL <= kConsumers,
                "K1a geometry");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t id_bar[kMaxStages];
  __shared__ __align__(8) uint64_t done_bar[kMaxStages];
  __shared__ int stage_unit[kMaxStages];
  __shared__ uint32_t subsum[NSUB * SC * C];
  __shared__ uint8_t subval[NSUB * SC * C];
  __shared__ uint8_t cellval[NCELL * C];
  __shared__ uint8_t cflag[NCELL];
  __shared__ uint32_t cslot[NCELL];
  __shared__ uint32_t cellsum[NCELL * C];
  __shared__ int cxlist[NCELL];  // complex cells of the unit (compacted)
  __shared__ int ncx_s;

  const int S = a.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&id_bar[s], 1);
      mbar_init(&done_bar[s], kConsumers);
    }
    fence_mbarrier_init();
  }
  for (int i = threadIdx.x; i < NSUB * SC * C; i += blockDim.x) subsum[i] = 0;
  for (int i = threadIdx.x; i < NCELL * C; i += blockDim.x) cellsum[i] = 0;
  __syncthreads();

  if (warp == kConsumers / 32) {  // producer warp, as in k_stats_tma
    if (lane == 0) {
      prefetch_tmap(&tm_in);
      prefetch_tmap(&tm_out);
    }
    auto finish_unit = [&](int s, int use) {
      mbar_wait(&done_bar[s], use & 1);
      if (a.out) {
        const int uu = stage_unit[s];
        store_tail<C, B, false, TILE>(a, uu, smem + s * STAGE, lane);
        if (lane == 0) store_unit<C, B, false, TILE>(a, &tm_out, uu, smem + s * STAGE);
      }
      __syncwarp();
    };
    int k = 0, done_units = 0;
    for (;; ++k) {
      const int s = ring_slot(k, S);
      if (k >= S) {
        finish_unit(s, ring_lap(k, S) - 1);
        ++done_units;
      }
      int u = 0;
      if (lane == 0) {
        u = atomicAdd(a.work_counter, 1);
        if (u >= a.units) {
          if (u == a.units + static_cast<int>(gridDim.x) - 1) atomicExch(a.work_counter, 0);
          u = -1;
        }
        stage_unit[s] = u;
        mbar_arrive(&id_bar[s]);
        if (u < 0)
          mbar_arrive_expect_tx(&full_bar[s], 0);
        else
          load_unit<C, B, false, TILE>(a, &tm_in, u, smem + s * STAGE, &full_bar[s]);
      }
      u = __shfl_sync(0xFFFFFFFFu, u, 0);
      if (u < 0) break;
    }
    for (int j = done_units; j < k; ++j) finish_unit(ring_slot(j, S), ring_lap(j, S));
    if (lane == 0) bulk_wait_all();
    return;
  }

  // ---------------- consumer warps ----------------
  const int t = threadIdx.x;
  const BatchGeom& g = a.g;
  const DrawEnv env_cell = make_env(a.noise.kind, a.exact_noise != 0, a.area, a.sigma);
  const DrawEnv env_sub = make_env(a.noise.kind, a.exact_noise != 0, a.sub_area, a.sigma_sub);
  const int cA = (4 * (t < NSTRIP ? t : 0) / SB) / NSUB;                  // cell of column sa
  const int cB = ((4 * (t < NSTRIP ? t : 0) / SB) + 1) / NSUB;            // cell of column sa + 1
  const bool strip_ok = t < NSTRIP;
  const int lpx = 4 * (strip_ok ? t : 0);
  const int sa = lpx / SB;                          // first subcell column of the strip
  const int split = min(4, (sa + 1) * SB - lpx);    // pixels [0, split) are in column sa
  uint32_t m[C][C == 4 ? 4 : C];
#pragma unroll
  for (int ch = 0; ch < C; ++ch)
#pragma unroll
    for (int q = 0; q < (C == 4 ? 4 : C); ++q) m[ch][q] = 0;
#pragma unroll
  for (int pos = 0; pos < 4 * C; ++pos)
    if (pos / C < split) m[pos % C][pos / 4] |= 1u << (8 * (pos % 4));

  for (int k = 0;; ++k) {
    const int s = ring_slot(k, S);
    uint8_t* st = smem + s * STAGE;
    mbar_wait(&id_bar[s], ring_lap(k, S) & 1);
    const int u = *reinterpret_cast<volatile int*>(&stage_unit[s]);
    if (u < 0) break;
    const UnitPos p = decode_unit<false, TILE>(a, u);
    const int f = p.fg;
    const int cell0 = p.px0 / B;
    const int ncell = min(NCELL, g.GC - cell0);
    const int nsc = ncell * NSUB;                    // real subcell columns in the tile
    const bool active = strip_ok && sa < nsc;
    const bool has_b = split < 4 && sa + 1 < nsc;
    const int vbytes = valid_bytes<C, false, TILE>(a, p.px0);
    const int copy = staged_bytes<C, B, false, TILE>(a, p);
    const int need = min(TILE, g.GC * B - p.px0) * C;
    const uint32_t rowpre = __ldg(&a.rowprefix[static_cast<int64_t>(f) * g.GR + p.r]);
    const uint32_t S_tot = __ldg(&a.totals[f]);
    uint32_t info = 1u;  // cell class and packed slot (K0), published after the barrier below
    if (t < ncell) info = __ldg(&a.cellinfo[static_cast<int64_t>(f) * g.G + p.r * g.GC + cell0 + t]);

    mbar_wait(&full_bar[s], ring_lap(k, S) & 1);
    const int fs = min(copy, vbytes);
    if (fs < need) {
      constexpr int kLanes = 4;
      for (int pr = t / kLanes; pr < B; pr += kConsumers / kLanes) {
        uint8_t* rowp = st + pr * ROWB;
        const int srow = reflect_index(p.r * B + pr, g.M);
        const uint8_t* grow = a.img + static_cast<int64_t>(f) * a.fstride + static_cast<int64_t>(srow) * a.pitch;
        for (int x = fs + (t % kLanes); x < need; x += kLanes) {
          const int cpx = x / C, ch = x - cpx * C;
          const int spx = reflect_index(p.px0 + cpx, g.N);
          const int sx = (spx - p.px0) * C + ch;
          rowp[x] = (sx >= 0 && sx < fs) ? rowp[sx] : __ldg(grow + static_cast<int64_t>(spx) * C + ch);
        }
      }
    }
    named_bar_sync(1, kConsumers);  // staged rows complete; previous unit's tables free
    if (t < ncell) {
      cflag[t] = info & 1u;
      cslot[t] = rowpre + (info >> 1);
    }
    if (t == 0) {  // compact list of the unit's complex cells
      int q = 0;
      for (int c = 0; c < ncell; ++c) {
        const uint32_t ic = __ldg(&a.cellinfo[static_cast<int64_t>(f) * g.G + p.r * g.GC + cell0 + c]);
        if (!(ic & 1u)) cxlist[q++] = c;
      }
      ncx_s = q;
    }

    const uint8_t* mystrip = st + lpx * C;
    uint32_t tot_a[C], tot_b[C];  // whole-band sums left / right of the boundary
#pragma unroll
    for (int ch = 0; ch < C; ++ch) tot_a[ch] = tot_b[ch] = 0;
#pragma unroll 1
    for (int vs = 0; vs < NSUB; ++vs) {
      uint32_t acc[C], part[C];
#pragma unroll
      for (int ch = 0; ch < C; ++ch) acc[ch] = part[ch] = 0;
#pragma unroll
      for (int i = 0; i < SB; ++i) {
        accumulate_row<C>(mystrip + (vs * SB + i) * ROWB, acc);
        accumulate_row_masked<C>(mystrip + (vs * SB + i) * ROWB, m, part);
      }
      if (active) {
        uint32_t* row = &subsum[(vs * SC + sa) * C];
#pragma unroll
        for (int ch = 0; ch < C; ++ch) {
          atomicAdd(row + ch, part[ch]);
          if (has_b) atomicAdd(row + C + ch, acc[ch] - part[ch]);
          tot_a[ch] += part[ch];
          tot_b[ch] += acc[ch] - part[ch];
        }
      }
    }
    if (active) {  // whole-cell sums (for simple cells)
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        if (has_b && cB != cA) {
          atomicAdd(&cellsum[cA * C + ch], tot_a[ch]);
          atomicAdd(&cellsum[cB * C + ch], tot_b[ch]);
        } else {
          atomicAdd(&cellsum[cA * C + ch], tot_a[ch] + (has_b ? tot_b[ch] : 0u));
        }
      }
    }
    named_bar_sync(1, kConsumers);
    // Simple cells: one draw per (cell, channel) at sigma.
    for (int item = t; item < ncell * C; item += kConsumers) {
      const int ch = item / ncell, c = item - ch * ncell;
      if (!cflag[c]) continue;
      const int gc = cell0 + c, gidx = p.r * g.GC + gc;
      const uint32_t v = draw_stat(a, env_cell, cellsum[c * C + ch], cell_state(a, f, ch, p.r, gc), f, ch, p.r, gc, 0,
                                   0, gidx);
      a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + stat_offset(a, true, gidx, cslot[c], S_tot, 0, 0)] =
          static_cast<uint8_t>(v);
      cellval[c * C + ch] = static_cast<uint8_t>(v);
    }
    // Complex cells: n x n x C draws each at sigma_sub (compacted cell list).
    const int ncx = ncx_s;
    constexpr int NN = NSUB * NSUB;
    for (int item = t; item < ncx * NN * C; item += kConsumers) {
      const int kk = item / (NN * C), rem = item - kk * (NN * C);
      const int ch = rem / NN, ss = rem - ch * NN;
      const int vs = ss / NSUB, sc = ss - vs * NSUB;
      const int c = cxlist[kk];
      const int gc = cell0 + c, gidx = p.r * g.GC + gc;
      const int sidx = c * NSUB + sc;
      const uint32_t v = draw_stat(a, env_sub, subsum[(vs * SC + sidx) * C + ch], cell_state(a, f, ch, p.r, gc), f, ch,
                                   p.r, gc, vs, sc, gidx);
      a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + stat_offset(a, false, gidx, cslot[c], S_tot, vs, sc)] =
          static_cast<uint8_t>(v);
      subval[(vs * SC + sidx) * C + ch] = static_cast<uint8_t>(v);
    }
    named_bar_sync(1, kConsumers);
    for (int i = t; i < NSUB * nsc * C; i += kConsumers) {  // reset for the next unit
      const int vs = i / (nsc * C), r2 = i - vs * (nsc * C);
      subsum[vs * SC * C + r2] = 0;
    }
    for (int i = t; i < ncell * C; i += kConsumers) cellsum[i] = 0;
    if (a.out && active) {
      const int ca = sa / NSUB, cb = (sa + 1) / NSUB;
#pragma unroll 1
      for (int vs = 0; vs < NSUB; ++vs) {
        uint32_t va[C], vb[C];
#pragma unroll
        for (int ch = 0; ch < C; ++ch) {
          va[ch] = cflag[ca] ? cellval[ca * C + ch] : subval[(vs * SC + sa) * C + ch];
          vb[ch] = !has_b ? va[ch] : (cflag[cb] ? cellval[cb * C + ch] : subval[(vs * SC + sa + 1) * C + ch]);
        }
        uint32_t w[C == 4 ? 4 : C];
        pattern_words_split<C>(va, vb, split, w);
#pragma unroll 1
        for (int i = 0; i < SB; ++i)
#pragma unroll
          for (int q = 0; q < (C == 4 ? 4 : C); ++q)
            reinterpret_cast<uint32_t*>(st + lpx * C + (vs * SB + i) * ROWB)[q] = w[q];
      }
    }
    fence_proxy_async_smem();
    mbar_arrive(&done_bar[s]);
  }
}

template <int C>
StatsKernel pick_adaptive_any(int b, int n) {
#define DPPX_CASE(BV, NS) \
  if (b == (BV) && n == (NS)) return k_adaptive_any_tma<C, BV, NS>;
  // b = 128 with n <= 16 stays on K1r (measured 5-10 % faster there)
  DPPX_CASE(128, 32)
  DPPX_CASE(30, 2)
  DPPX_CASE(30, 3)
  DPPX_CASE(30, 5)
  DPPX_CASE(30, 6)
  DPPX_CASE(30, 10)
#undef DPPX_CASE
  return nullptr;
}

template <int C>
StatsKernel pick_uniform_any(int b) {
#define DPPX_CASE(BV) \
  if (b == (BV)) return k_uniform_tma<C, BV>;
  DPPX_CASE(2)
  DPPX_CASE(3)
  DPPX_CASE(5)
  DPPX_CASE(6)
  DPPX_CASE(7)
  DPPX_CASE(9)
  DPPX_CASE(10)
  DPPX_CASE(11)
  DPPX_CASE(13)
  DPPX_CASE(14)
  DPPX_CASE(15)
  DPPX_CASE(17)
  DPPX_CASE(18)
  DPPX_CASE(19)
  DPPX_CASE(30)
  DPPX_CASE(128)  // PPM-100's largest grid (K1 stages would not fit two per CTA)
#undef DPPX_CASE
  return nullptr;
}

template <int C, bool AD, bool PK>
StatsKernel pick_b(int b, int n) {
#define DPPX_CASE(B4v, NS)                 \
  if (b == 4 * (B4v) && n == (NS)) return k_stats_tma<C, B4v, NS, AD, PK>;
  DPPX_CASE(1, 1)
  DPPX_CASE(2, 1)
  DPPX_CASE(4, 1)
  DPPX_CASE(8, 1)
  if constexpr (!PK) {  // the paper's b = 12, 20, 24, 40 (whole cells per warp, 480-px tiles)
    DPPX_CASE(3, 1)
    DPPX_CASE(5, 1)
    DPPX_CASE(6, 1)
    DPPX_CASE(10, 1)
    DPPX_CASE(16, 1)  // b = 64: 98 KB stages, 1 CTA/SM
  }
  if constexpr (AD) {
    DPPX_CASE(2, 2)
    DPPX_CASE(4, 2)
    DPPX_CASE(4, 4)
    DPPX_CASE(8, 2)
    DPPX_CASE(8, 4)
    DPPX_CASE(8, 8)
    if constexpr (!PK) {
      DPPX_CASE(3, 3)
      DPPX_CASE(5, 5)
      DPPX_CASE(6, 2)
      DPPX_CASE(6, 3)
      DPPX_CASE(6, 6)
      DPPX_CASE(10, 2)
      DPPX_CASE(10, 5)
      DPPX_CASE(10, 10)
      DPPX_CASE(16, 2)
      DPPX_CASE(16, 4)
      DPPX_CASE(16, 8)
      DPPX_CASE(16, 16)
      // subcell sides that are not a multiple of 4 px (STR: split strips)
      DPPX_CASE(3, 2)
      DPPX_CASE(5, 2)
      DPPX_CASE(5, 4)
      DPPX_CASE(6, 4)
      DPPX_CASE(10, 4)
      DPPX_CASE(10, 8)
      DPPX_CASE(2, 4)   // subcells of 2 or 3 px
      DPPX_CASE(3, 4)
      DPPX_CASE(4, 8)
      DPPX_CASE(6, 8)
    }
    if constexpr (PK) {  // narrow frames, 2-px subcells (CelebA b8 n4, b16 n8)
      DPPX_CASE(2, 4)
      DPPX_CASE(4, 8)
    }
    // 1-px subcells (n = b): per-pixel complex cells
    DPPX_CASE(1, 4)
    DPPX_CASE(2, 8)
    DPPX_CASE(4, 16)
    if constexpr (!PK) {
      DPPX_CASE(8, 32)
      DPPX_CASE(16, 64)
      // 2-px subcells of the PPM-100 grid (in-lane, no subcell tables)
      DPPX_CASE(1, 2)
      DPPX_CASE(8, 16)
      DPPX_CASE(16, 32)
    }
  }
#undef DPPX_CASE
  return nullptr;
}

template <int C>
StatsKernel pick_var(int b, int n) {
#define DPPX_CASE(B4v, NS) \
  if (b == 4 * (B4v) && n == (NS)) return k_stats_tma<C, B4v, NS, true, false, true>;
  DPPX_CASE(2, 2)
  DPPX_CASE(4, 2)
  DPPX_CASE(4, 4)
  DPPX_CASE(8, 2)
  DPPX_CASE(8, 4)
  DPPX_CASE(8, 8)
#undef DPPX_CASE
  return nullptr;
}

// Band-split K2 (b = 32, 64: 49 / 98 KB RGB tiles otherwise): H parts per band.
template <int C, bool AD, int H>
ExpandKernel pick_expand_split(int b, int n) {
#define DPPX_CASE(B4v, NS) \
  if (b == 4 * (B4v) && n == (NS)) return k_expand_tma<C, B4v, NS, AD, false, H>;
  DPPX_CASE(8, 1)
  DPPX_CASE(16, 1)
  if constexpr (AD) {
    if constexpr (H <= 2) {
      DPPX_CASE(8, 2)
      DPPX_CASE(16, 2)
    }
    DPPX_CASE(8, 4)
    DPPX_CASE(8, 8)
    DPPX_CASE(16, 4)
    DPPX_CASE(16, 8)
    DPPX_CASE(16, 16)
  }
#undef DPPX_CASE
  return nullptr;
}

template <int C, bool AD, bool PK>
ExpandKernel pick_expand(int b, int n) {
#define DPPX_CASE(B4v, NS) \
  if (b == 4 * (B4v) && n == (NS)) return k_expand_tma<C, B4v, NS, AD, PK>;
  DPPX_CASE(1, 1)
  DPPX_CASE(2, 1)
  DPPX_CASE(4, 1)
  DPPX_CASE(8, 1)
  if constexpr (!PK) {  // whole-cell warps / large cells (same set as K1)
    DPPX_CASE(3, 1)
    DPPX_CASE(5, 1)
    DPPX_CASE(6, 1)
    DPPX_CASE(10, 1)
    DPPX_CASE(16, 1)
    if constexpr (AD) {
      DPPX_CASE(3, 3)
      DPPX_CASE(5, 5)
      DPPX_CASE(6, 2)
      DPPX_CASE(6, 3)
      DPPX_CASE(6, 6)
      DPPX_CASE(10, 2)
      DPPX_CASE(10, 5)
      DPPX_CASE(10, 10)
      DPPX_CASE(16, 2)
      DPPX_CASE(16, 4)
      DPPX_CASE(16, 8)
      DPPX_CASE(16, 16)
      // split strips, subcells of 2 or 3 px (K2r measured faster for the
      // 5, 6 and 10 px subcells: 0.84-0.92 vs 0.69-0.79 of HBM)
      DPPX_CASE(2, 4)
      DPPX_CASE(3, 4)
      DPPX_CASE(4, 8)
      DPPX_CASE(6, 8)
    }
  }
  if constexpr (AD) {
    DPPX_CASE(2, 2)
    DPPX_CASE(4, 2)
    DPPX_CASE(4, 4)
    DPPX_CASE(8, 2)
    DPPX_CASE(8, 4)
    DPPX_CASE(8, 8)
    if constexpr (PK) {  // narrow frames, 2-px subcells (CelebA b8 n4, b16 n8)
      DPPX_CASE(2, 4)
      DPPX_CASE(4, 8)
    }
    // 1-px subcells (n = b): per-pixel complex values
    DPPX_CASE(1, 4)
    DPPX_CASE(2, 8)
    DPPX_CASE(4, 16)
    if constexpr (!PK) {
      DPPX_CASE(8, 32)
      DPPX_CASE(16, 64)
      DPPX_CASE(1, 2)
      DPPX_CASE(8, 16)
      DPPX_CASE(16, 32)
    }
  }
#undef DPPX_CASE
  return nullptr;
}

template <int C>
ExpandKernel pick_expand_uany(int b) {
#define DPPX_CASE(BV) \
  if (b == (BV)) return k_expand_uany<C, BV>;
  DPPX_CASE(2)
  DPPX_CASE(3)
  DPPX_CASE(5)
  DPPX_CASE(6)
  DPPX_CASE(7)
  DPPX_CASE(9)
  DPPX_CASE(10)
  DPPX_CASE(11)
  DPPX_CASE(13)
  DPPX_CASE(14)
  DPPX_CASE(15)
  DPPX_CASE(17)
  DPPX_CASE(18)
  DPPX_CASE(19)
  DPPX_CASE(30)
  DPPX_CASE(128)
#undef DPPX_CASE
  return nullptr;
}

template <int C>
ExpandKernel pick_expand_aany(int b, int n) {
#define DPPX_CASE(BV, NS) \
  if (b == (BV) && n == (NS)) return k_expand_aany<C, BV, NS>;
  DPPX_CASE(30, 2)  // (b = 30 n = 3, 5: K2r measured faster, 0.92 / 0.84 vs 0.80 / 0.76)
  DPPX_CASE(30, 6)
  DPPX_CASE(30, 10)
  DPPX_CASE(128, 2)
  DPPX_CASE(128, 4)
  DPPX_CASE(128, 8)
  DPPX_CASE(128, 16)
  DPPX_CASE(128, 32)
#undef DPPX_CASE
  return nullptr;
}

// Per-channel-count selectors (defined in tma_c1.cu / tma_c3.cu).
StatsKernel select_stats_tma_c1(int b, int n, bool adaptive, bool packed);
StatsKernel select_stats_tma_c3(int b, int n, bool adaptive, bool packed);
StatsKernel select_stats_var_c1(int b, int n);
StatsKernel select_uniform_any_c1(int b);
StatsKernel select_adaptive_any_c1(int b, int n);
ExpandKernel select_expand_uany_c1(int b);
ExpandKernel select_expand_aany_c1(int b, int n);
ExpandKernel select_expand_aany_c3(int b, int n);
ExpandKernel select_expand_uany_c3(int b);
StatsKernel select_adaptive_any_c3(int b, int n);
StatsKernel select_uniform_any_c3(int b);
StatsKernel select_stats_var_c3(int b, int n);
ExpandKernel select_expand_tma_c1(int b, int n, bool adaptive, bool packed, int split);
ExpandKernel select_expand_tma_c3(int b, int n, bool adaptive, bool packed, int split);

}  // namespace dppx
