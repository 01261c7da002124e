// stats_common.cuh -- per-statistic helpers shared by every statistics kernel
// (K1 TMA, K1g, K1r): packed destination, noise bits, lazy injected noise.
#pragma once
#include <cstdint>

#include "dppx_device.cuh"
#include "dppx_params.h"

namespace dppx {

// ============================================================================
// Shared helpers for K1 / K1g: per-statistic value and packed destination
// ============================================================================

// Packed destination of a statistic of plane p (uniform: means[g];
// adaptive simple: 4G+4+slot; adaptive complex: 4G+4+S+slot*n*n+sr*n+sc).
__device__ __forceinline__ int64_t stat_offset(const StatsArgs& a, bool simple, int g_idx,
                                               uint32_t slot_s, uint32_t S_tot, int sr, int sc) {
  if (!a.adaptive) return g_idx;
  const int64_t base = 4ll * a.g.G + 4;
  if (simple) return base + slot_s;
  const uint32_t slot_c = static_cast<uint32_t>(g_idx) - slot_s;
  return base + S_tot + static_cast<int64_t>(slot_c) * a.g.n * a.g.n + sr * a.g.n + sc;
}

// stat_offset of complex subcell k = sr * n + sc with n known at compile time
// (NN = n * n): no 64-bit multiply by the runtime n.
template <int NN>
__device__ __forceinline__ int64_t complex_offset(const StatsArgs& a, int g_idx, uint32_t slot_s,
                                                 uint32_t S_tot, int k) {
  return 4ll * a.g.G + 4 + S_tot + static_cast<int64_t>(static_cast<uint32_t>(g_idx) - slot_s) * NN + k;
}

// 64 noise bits of statistic (r, c, sr, sc) of plane (f, ch). `cs` is the
// KEYED per-cell state key_cell(mix64(seed), r, c) (noise.cpp:86-91).
static __device__ __noinline__ uint64_t philox_call(uint64_t seed, uint32_t frame, uint32_t ch, uint32_t r,
                                             uint32_t c, uint32_t sr, uint32_t sc) {
  return philox_bits(seed, frame, ch, r, c, sr, sc);
}

__device__ __forceinline__ uint64_t draw_bits(const StatsArgs& a, uint64_t cs, int f, int ch, int r,
                                              int c, int sr, int sc) {
  if (a.noise.kind == DPPX_NOISE_KEYED) return key_sub(cs, sr, sc);
  if (a.noise.kind == DPPX_NOISE_PHILOX)  // out of line: keeps the hot loop small
    return philox_call(a.noise.seed(0), a.noise.frame_base + f, ch, r, c, sr, sc);
  return 0ull;
}

static __device__ __noinline__ double injected_value(const double* inj, int64_t plane, int G, int n,
                                              int g_idx, int sr, int sc) {
  return inj[((plane * G + g_idx) * n + sr) * n + sc];
}

// Lazy handle on one statistic's injected noise value (see quantize_stat):
// only scalars are captured, so nothing of StatsArgs is copied to local memory.
struct InjAt {
  const double* inj;
  int64_t plane;
  int G, n, g_idx, sr, sc;
  __device__ __forceinline__ double operator()() const {
    return injected_value(inj, plane, G, n, g_idx, sr, sc);
  }
};

__device__ __forceinline__ InjAt inj_at(const StatsArgs& a, int f, int ch, int g_idx, int sr, int sc) {
  return InjAt{a.noise.injected, static_cast<int64_t>(f) * a.g.C + ch, a.g.G, a.g.n, g_idx, sr, sc};
}

__device__ __forceinline__ uint64_t cell_state(const StatsArgs& a, int f, int ch, int r, int c) {
  return a.noise.kind == DPPX_NOISE_KEYED
             ? key_cell(a.noise.seed(static_cast<int64_t>(f) * a.g.C + ch), r, c)
             : 0ull;
}

// One statistic of plane (f, ch): the keyed stream (the common case) on its
// own path, so no Philox / injected-noise arguments are formed per draw
// (measured 7 % of K1's instructions at b = 4); every other kind through
// quantize_stat. `cs` is cell_state(a, f, ch, r, c); gidx = r * GC + c.
__device__ __forceinline__ uint32_t draw_stat(const StatsArgs& a, const DrawEnv& env, uint32_t sum, uint64_t cs,
                                              int f, int ch, int r, int c, int sr, int sc, int gidx) {
  if (env.kind == DPPX_NOISE_KEYED && !env.exact_only) {
    const uint64_t bits = key_sub(cs, sr, sc);
    const uint32_t q = fast_quantize(sum, env.inv_area, bits, env.sln2, env.margin);
    return q != 0xFFFFFFFFu ? q : exact_quantize(sum, env.area, DPPX_NOISE_KEYED, bits, env.sigma, 0.0);
  }
  return quantize_stat(env, sum, draw_bits(a, cs, f, ch, r, c, sr, sc), inj_at(a, f, ch, gidx, sr, sc));
}


}  // namespace dppx
