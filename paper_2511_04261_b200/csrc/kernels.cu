// kernels.cu -- sm_100a kernels of the dppix pixelization path.
//
//  K0  k_classify      mask (or stored mask means) -> per-cell simple/complex
//                      flag, intra-row packed-slot prefix, per-row counts; the
//                      last CTA of each plane scans the rows (no spin waits).
//                      classify_regions adaptive.cpp:34-65 + the exclusive scan
//                      adaptive.cpp:123-141.
//  K1  k_stats_tma     persistent, warp-specialized: one producer warp stages
//                      b-row x 512-px tiles of interleaved u8 frames into shared
//                      memory with cp.async.bulk (TMA) on an mbarrier ring; four
//                      consumer warps reduce 4-px strips with dp4a + warp
//                      shuffles, draw the keyed Laplace noise, write the compact
//                      statistics, and overwrite the tile in place with the
//                      reconstructed pixels that the producer bulk-stores back.
//                      grid_mean/block_sum image.cpp:154-189 adaptive.cpp:70-79,
//                      noise adaptive.cpp:147-170 pixelize.cpp:109-117,
//                      broadcast_means pixelize.cpp:126-150, reassemble
//                      adaptive.cpp:181-245.
//  K1g k_stats_generic same semantics for any b, n, C and alignment.
//  K2  k_expand        statistics -> pixels (broadcast_means / reassemble).
#include <cuda.h>  // CUtensorMap (type only; encoded on the host via the driver entry point)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "dppx_device.cuh"
#include "dppx_params.h"

namespace dppx {

// ============================================================================
// K0: classification + slot scan
// ============================================================================
constexpr int kClassifyThreads = 128;

__device__ __forceinline__ uint32_t sum_bytes4(uint32_t w) { return __dp4a(w, 0x01010101u, 0u); }

// Exclusive block scan of 0/1 flags (kClassifyThreads threads). Returns the
// exclusive prefix; *total receives the block total. Uses `warp_tot` of smem.
__device__ __forceinline__ uint32_t block_scan_flags(bool flag, uint32_t* warp_tot,
                                                     uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, flag);
  const uint32_t in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[warp] = __popc(bal);
  __syncthreads();
  uint32_t before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kClassifyThreads / 32; ++w) {
    const uint32_t v = warp_tot[w];
    before += (w < warp) ? v : 0u;
    all += v;
  }
  __syncthreads();
  *total = all;
  return before + in_warp;
}

// Exclusive block scan of u32 values (kClassifyThreads threads).
__device__ __forceinline__ uint32_t block_scan_u32(uint32_t v, uint32_t* warp_tot,
                                                   uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  uint32_t before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kClassifyThreads / 32; ++w) {
    const uint32_t t = warp_tot[w];
    before += (w < warp) ? t : 0u;
    all += t;
  }
  __syncthreads();
  *total = all;
  return before + x - v;
}

// Mask sum of cell (r, c). Rows are reflected (image.cpp:105-110); interior
// cells use aligned vector loads with all rows issued before the reduction.
template <int B>
__device__ __forceinline__ uint32_t mask_cell_sum_vec(const ClassifyArgs& a, const uint8_t* base,
                                                      int r, int j0) {
  uint32_t s = 0;
  if constexpr (B % 16 == 0) {
    constexpr int K = B / 16;
    uint4 v[B][K];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const uint4* p = reinterpret_cast<const uint4*>(
          base + static_cast<int64_t>(reflect_index(r * B + i, a.g.M)) * a.mpitch + j0);
#pragma unroll
      for (int k = 0; k < K; ++k) v[i][k] = __ldg(p + k);
    }
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int k = 0; k < K; ++k)
        s += sum_bytes4(v[i][k].x) + sum_bytes4(v[i][k].y) + sum_bytes4(v[i][k].z) +
             sum_bytes4(v[i][k].w);
  } else {
    constexpr int K = B / 4;
    uint32_t v[B][K];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(
          base + static_cast<int64_t>(reflect_index(r * B + i, a.g.M)) * a.mpitch + j0);
#pragma unroll
      for (int k = 0; k < K; ++k) v[i][k] = __ldg(p + k);
    }
#pragma unroll
    for (int i = 0; i < B; ++i)
#pragma unroll
      for (int k = 0; k < K; ++k) s += sum_bytes4(v[i][k]);
  }
  return s;
}

// Mask sum of cell (r, c) from bit-packed rows (host pipeline transport,
// maskpack.h): bit (j % 32) of word (j / 32) is mask[i][j] in {0, 1}.
// Scalars only: a reference to the kernel's parameter struct would force a
// per-thread local-memory copy of it.
__device__ __noinline__ uint32_t mask_cell_sum_bits(const uint8_t* base, int64_t mpitch, int M, int N,
                                                    int b, int r, int c) {
  const int j0 = c * b;
  uint32_t s = 0;
  if (j0 + b <= N) {
    const int j1 = j0 + b - 1;
    const int w0 = j0 >> 5, w1 = j1 >> 5;
    const uint32_t m0 = ~0u << (j0 & 31), m1 = ~0u >> (31 - (j1 & 31));
    for (int i = r * b; i < r * b + b; ++i) {
      const uint32_t* row =
          reinterpret_cast<const uint32_t*>(base + static_cast<int64_t>(reflect_index(i, M)) * mpitch);
      if (w0 == w1) {
        s += __popc(__ldg(row + w0) & m0 & m1);
      } else {
        s += __popc(__ldg(row + w0) & m0) + __popc(__ldg(row + w1) & m1);
        for (int w = w0 + 1; w < w1; ++w) s += __popc(__ldg(row + w));
      }
    }
    return s;
  }
  for (int i = r * b; i < r * b + b; ++i) {
    const uint32_t* row =
        reinterpret_cast<const uint32_t*>(base + static_cast<int64_t>(reflect_index(i, M)) * mpitch);
    for (int j = j0; j < j0 + b; ++j) {
      const int jj = reflect_index(j, N);
      s += (__ldg(row + (jj >> 5)) >> (jj & 31)) & 1u;
    }
  }
  return s;
}

__device__ __forceinline__ uint32_t mask_cell_sum(const ClassifyArgs& a, const uint8_t* base,
                                                  int r, int c) {
  const BatchGeom& g = a.g;
  const int b = g.b;
  const int j0 = c * b;
  if (a.mask_bits) return mask_cell_sum_bits(base, a.mpitch, g.M, g.N, b, r, c);
  if (j0 + b <= g.N && a.vec > 1) {
    if (a.vec == 16) {
      if (b == 16) return mask_cell_sum_vec<16>(a, base, r, j0);
      if (b == 32) return mask_cell_sum_vec<32>(a, base, r, j0);
    } else {
      if (b == 4) return mask_cell_sum_vec<4>(a, base, r, j0);
      if (b == 8) return mask_cell_sum_vec<8>(a, base, r, j0);
    }
  }
  uint32_t s = 0;
  for (int i = r * b; i < r * b + b; ++i) {
    const uint8_t* row = base + static_cast<int64_t>(reflect_index(i, g.M)) * a.mpitch;
    for (int j = j0; j < j0 + b; ++j) s += __ldg(row + reflect_index(j, g.N));
  }
  return s;
}

// EXTENSION (variance complexity): exact S1 = sum x, S2 = sum x^2 over the
// C*b*b samples of mirror-padded cell (r, c); dp4a(w, w) gives sum of squares.
__device__ __forceinline__ bool cell_is_complex_var(const ClassifyArgs& a, const uint8_t* base,
                                                   int r, int c) {
  const BatchGeom& g = a.g;
  const int b = g.b, C = g.C;
  const int j0 = c * b;
  uint64_t s1 = 0, s2 = 0;
  const bool inside = j0 + b <= g.N;
  for (int i = r * b; i < r * b + b; ++i) {
    const uint8_t* row = base + static_cast<int64_t>(reflect_index(i, g.M)) * a.pitch;
    if (inside && a.img_vec4) {
      const uint32_t* p = reinterpret_cast<const uint32_t*>(row + static_cast<int64_t>(j0) * C);
      uint32_t t1 = 0, t2 = 0;
      for (int k = 0; k < b * C / 4; ++k) {
        const uint32_t w = __ldg(p + k);
        t1 = __dp4a(w, 0x01010101u, t1);
        t2 = __dp4a(w, w, t2);
      }
      s1 += t1;
      s2 += t2;
    } else {
      for (int j = j0; j < j0 + b; ++j) {
        const uint8_t* px = row + static_cast<int64_t>(reflect_index(j, g.N)) * C;
        for (int k = 0; k < C; ++k) {
          const uint32_t v = __ldg(px + k);
          s1 += v;
          s2 += v * v;
        }
      }
    }
  }
  const long long ns = static_cast<long long>(C) * b * b;
  const double num = static_cast<double>(ns * static_cast<long long>(s2) -
                                         static_cast<long long>(s1) * static_cast<long long>(s1));
  const double var = __ddiv_rn(num, __dmul_rn(static_cast<double>(ns), static_cast<double>(ns)));
  return var >= a.var_tau;
}

// Band column sums for grid sides without a per-cell vector path (b = 12, 20,
// 24, 40, 64, 128 ...): the block sums its b mask rows column by column with
// coalesced 16-byte loads (SWAR, two u16 counters per u32: b <= 257), then a
// cell's sum is b smem reads. One thread per cell reading b x b bytes would
// leave most of the block idle at large b (30 cells per 1080p row at b = 64).
__device__ void mask_band_colsums(const ClassifyArgs& a, const uint8_t* mbase, int r,
                                  uint32_t* colsum) {
  const BatchGeom& g = a.g;
  const int W = g.GC * g.b;  // padded columns
  const bool vec = a.vec == 16;
  for (int x0 = threadIdx.x * 16; x0 < W; x0 += kClassifyThreads * 16) {
    uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
    const bool fast = vec && x0 + 16 <= g.N;
#pragma unroll 4
    for (int i = 0; i < g.b; ++i) {
      const uint8_t* row = mbase + static_cast<int64_t>(reflect_index(r * g.b + i, g.M)) * a.mpitch;
      uint32_t w[4];
      if (fast) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + x0));
        w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t acc = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int x = x0 + 4 * j + k;
            const uint32_t byte = x < W ? __ldg(row + reflect_index(x, g.N)) : 0u;
            acc |= byte << (8 * k);
          }
          w[j] = acc;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lo[j] += w[j] & 0x00FF00FFu;
        hi[j] += (w[j] >> 8) & 0x00FF00FFu;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int x = x0 + 4 * j;
      if (x + 0 < W) colsum[x + 0] = lo[j] & 0xFFFFu;
      if (x + 1 < W) colsum[x + 1] = hi[j] & 0xFFFFu;
      if (x + 2 < W) colsum[x + 2] = lo[j] >> 16;
      if (x + 3 < W) colsum[x + 3] = hi[j] >> 16;
    }
  }
}

// Bit-packed masks (host pipeline) at large b: items (cell, row) over the
// whole block, popc per row segment, smem atomics into the cell sums.
__device__ void mask_band_cellsums_bits(const ClassifyArgs& a, const uint8_t* mbase, int r,
                                        uint32_t* cellsum) {
  const BatchGeom& g = a.g;
  for (int c = threadIdx.x; c < g.GC; c += kClassifyThreads) cellsum[c] = 0;
  __syncthreads();
  const FastDiv div_b = make_fastdiv(static_cast<uint32_t>(g.b));
  for (int item = threadIdx.x; item < g.GC * g.b; item += kClassifyThreads) {
    const int c = static_cast<int>(div_b.div(static_cast<uint32_t>(item))), i = item - c * g.b;
    const uint32_t* row = reinterpret_cast<const uint32_t*>(
        mbase + static_cast<int64_t>(reflect_index(r * g.b + i, g.M)) * a.mpitch);
    const int j0 = c * g.b;
    uint32_t sum = 0;
    if (j0 + g.b <= g.N) {
      const int j1 = j0 + g.b - 1, w0 = j0 >> 5, w1 = j1 >> 5;
      const uint32_t m0 = ~0u << (j0 & 31), m1 = ~0u >> (31 - (j1 & 31));
      if (w0 == w1) {
        sum = __popc(__ldg(row + w0) & m0 & m1);
      } else {
        sum = __popc(__ldg(row + w0) & m0) + __popc(__ldg(row + w1) & m1);
        for (int w = w0 + 1; w < w1; ++w) sum += __popc(__ldg(row + w));
      }
    } else {
      for (int j = j0; j < j0 + g.b; ++j) {
        const int jj = reflect_index(j, g.N);
        sum += (__ldg(row + (jj >> 5)) >> (jj & 31)) & 1u;
      }
    }
    atomicAdd(&cellsum[c], sum);
  }
}

template <bool BAND>
__global__ void __launch_bounds__(kClassifyThreads, BAND ? 10 : 8) k_classify(const ClassifyArgs a) {
  __shared__ uint32_t warp_tot[kClassifyThreads / 32];
  __shared__ uint32_t s_last;
  extern __shared__ uint32_t colsum[];  // a.band: per padded column mask sums of the band
  const BatchGeom& g = a.g;
  const int r = blockIdx.x;
  for (int p = blockIdx.y; p < a.planes; p += gridDim.y) {
    const uint8_t* mbase = a.from_payload ? nullptr : a.mask + static_cast<int64_t>(p) * a.mfstride;
    const float* mm_in =
        a.from_payload == 1 ? reinterpret_cast<const float*>(a.payload_in + p * a.pstride) : nullptr;
    if constexpr (BAND) {
      if (a.band == 2) mask_band_cellsums_bits(a, mbase, r, colsum);
      else mask_band_colsums(a, mbase, r, colsum);
      __syncthreads();
    }
    uint32_t carry = 0;
    for (int c0 = 0; c0 < g.GC; c0 += kClassifyThreads) {
      const int c = c0 + threadIdx.x;
      bool simple = false;
      if (c < g.GC) {
        const int cell = r * g.GC + c;
        float mean;
        if (a.from_payload == 1) {
          mean = mm_in[cell];
        } else if (a.from_payload >= 2) {
          const bool cx = a.from_payload == 2
                              ? cell_is_complex_var(a, a.img + static_cast<int64_t>(p) * a.fstride, r, c)
                              : a.flags[static_cast<int64_t>(p) * g.G + cell] == 0;
          mean = cx ? 0.0f : 1.0f;
          for (int ch = 0; ch < g.C; ++ch)
            reinterpret_cast<float*>(a.payload + (static_cast<int64_t>(p) * g.C + ch) * a.pstride)
                [cell] = mean;
        } else {
          uint32_t s = 0;
          if constexpr (BAND) {
            if (a.band == 2) {
              s = colsum[c];
            } else {
              for (int k = 0; k < g.b; ++k) s += colsum[c * g.b + k];
            }
          } else {
            s = mask_cell_sum(a, mbase, r, c);
          }
          // mask_grid_mean (image.cpp:191-202) then static_cast<float>
          // (adaptive.cpp:59-60).
          mean = __double2float_rn(__ddiv_rn(static_cast<double>(s), a.area));
          for (int ch = 0; ch < g.C; ++ch)
            reinterpret_cast<float*>(a.payload + (static_cast<int64_t>(p) * g.C + ch) * a.pstride)
                [cell] = mean;
        }
        simple = mean > 0.5f;  // simple_from_mean, adaptive.cpp:30-32
      }
      uint32_t tot;
      const uint32_t pre = block_scan_flags(simple, warp_tot, &tot);
      if (c < g.GC)
        a.cellinfo[static_cast<int64_t>(p) * g.G + r * g.GC + c] =
            ((carry + pre) << 1) | (simple ? 1u : 0u);
      carry += tot;
    }
    if (threadIdx.x == 0) {
      a.rowcnt[static_cast<int64_t>(p) * g.GR + r] = carry;
      __threadfence();
      const uint32_t ticket = atomicAdd(&a.counters[p], 1u);
      s_last = (ticket == static_cast<uint32_t>(g.GR - 1)) ? 1u : 0u;
    }
    __syncthreads();
    if (s_last) {  // last row of plane p: exclusive scan over rows
      __threadfence();
      uint32_t rcarry = 0;
      for (int r0 = 0; r0 < g.GR; r0 += kClassifyThreads) {
        const int rr = r0 + threadIdx.x;
        const uint32_t v = rr < g.GR ? __ldcg(&a.rowcnt[static_cast<int64_t>(p) * g.GR + rr]) : 0u;
        uint32_t tot;
        const uint32_t pre = block_scan_u32(v, warp_tot, &tot);
        if (rr < g.GR) a.rowprefix[static_cast<int64_t>(p) * g.GR + rr] = rcarry + pre;
        rcarry += tot;
      }
      if (threadIdx.x == 0) {
        const uint32_t S = rcarry;
        a.totals[p] = S;
        a.counters[p] = 0u;  // ready for the next launch
        const uint64_t nn = static_cast<uint64_t>(g.n) * g.n;
        const uint32_t len = static_cast<uint32_t>(4ull * g.G + 4 + S + (g.G - S) * nn);
        if (a.from_payload == 1) {
          const uint8_t* q = a.payload_in + p * a.pstride + 4ll * g.G;
          const uint32_t stored = static_cast<uint32_t>(q[0]) | (static_cast<uint32_t>(q[1]) << 8) |
                                  (static_cast<uint32_t>(q[2]) << 16) |
                                  (static_cast<uint32_t>(q[3]) << 24);
          // decode's simple-count and length checks (record.cpp:253-270).
          if (stored != S || (a.in_len && a.in_len[p] != len) || len > a.pstride)
            atomicExch(a.status, DPPX_ERR_CORRUPT);
        } else {
          for (int ch = 0; ch < g.C; ++ch) {
            const int64_t q = (static_cast<int64_t>(p) * g.C + ch) * a.pstride + 4ll * g.G;
            *reinterpret_cast<uint32_t*>(a.payload + q) = S;
            if (a.payload_len) a.payload_len[static_cast<int64_t>(p) * g.C + ch] = len;
          }
        }
      }
    }
    __syncthreads();
  }
}

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

// 64 noise bits of statistic (r, c, sr, sc) of plane (f, ch). `cs` is the
// KEYED per-cell state key_cell(mix64(seed), r, c) (noise.cpp:86-91).
__device__ __noinline__ uint64_t philox_call(uint64_t seed, uint32_t frame, uint32_t ch, uint32_t r,
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

__device__ __noinline__ double injected_value(const double* inj, int64_t plane, int G, int n,
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

// ============================================================================
// K1: TMA-staged persistent kernel (fast path)
// ============================================================================
constexpr int kConsumers = 128;            // 4 consumer warps, one 4-px strip each
constexpr int kTilePx = 4 * kConsumers;    // 512 px per tile
constexpr int kStatsThreads = kConsumers + 32;
constexpr int kMaxStages = 4;

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

// Slot geometry: compile-time for wide frames (one 512-px slot per unit).
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
// clipped by the TMA unit; the consumers write the (< 8) bytes past
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

// Output bytes of a unit past the output tensor map's row extent (< 8 per row:
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
  for (int e = lane; e < nf * rows * span; e += 32) {
    const int jr = e / span, x = scopy + (e - jr * span);
    const int j = jr / rows, i = jr - j * rows;
    a.out[static_cast<int64_t>(p.fg * pk + j) * a.ofstride +
          static_cast<int64_t>(p.r * B + i) * a.opitch + static_cast<int64_t>(p.px0) * C + x] =
        st[j * a.slot_stride + i * srb + x];
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
template <int C, int GL>
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
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int ch = j * GL + li;
    s[j] = sum[0];
    uint64_t st = cs[0];
#pragma unroll
    for (int k = 1; k < C; ++k)
      if (ch == k) {
        s[j] = sum[k];
        st = cs[k];
      }
    bits[j] = draw_bits(a, st, f, ch, r, c, sr, sc);
  }
  // Phase 1: branch-free bounded estimates for all channels (independent
  // chains the scheduler can interleave); phase 2: the rare exact draws.
  if (!env.exact_only && (env.kind == DPPX_NOISE_KEYED || env.kind == DPPX_NOISE_PHILOX)) {
#pragma unroll
    for (int j = 0; j < NV; ++j) q[j] = fast_quantize(s[j], env.inv_area, bits[j], env.sigmaf, env.margin);
  } else if (!env.exact_only && env.kind == DPPX_NOISE_NONE && env.pow2) {
#pragma unroll
    for (int j = 0; j < NV; ++j)  // sum * 2^-k + 0.5 is exact in f32
      q[j] = static_cast<uint32_t>(floorf(static_cast<float>(s[j]) * env.inv_area + 0.5f));
  } else {
#pragma unroll
    for (int j = 0; j < NV; ++j) q[j] = 0xFFFFFFFFu;
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

template <int C, int B4, int NSUB, bool ADAPTIVE, bool PACKED, bool VAR = false>
__global__ void __launch_bounds__(kStatsThreads)
    k_stats_tma(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                const StatsArgs a) {
  constexpr int B = 4 * B4;
  constexpr int SB = B / NSUB;
  constexpr int SB4 = SB / 4;
  // Strips per warp: whole cells only (a cell is B4 adjacent lanes), so for
  // B4 not a power of two (b = 12, 24) the last 32 % B4 lanes of each warp
  // idle and the tile is 16 * LPW px (480 at b = 12 or 24) instead of 512.
  constexpr int LPW = (32 / B4) * B4;
  constexpr int TILE = 4 * (kConsumers / 32) * LPW;
  constexpr int ROWB = TILE * C;
  constexpr uint32_t STAGE = B * ROWB;
  static_assert(SB % 4 == 0 && B4 <= 32 && B4 % SB4 == 0, "fast-path geometry");
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
    // Units (frame, grid row, 512-px tile) are claimed from a global counter so
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
        store_tail<C, B, PACKED, TILE>(a, uu, smem + s * STAGE, lane);
        if (lane == 0) store_unit<C, B, PACKED, TILE>(a, &tm_out, uu, smem + s * STAGE);
      }
      __syncwarp();
    };
    int k = 0;
    int done_units = 0;  // units of this CTA already stored
    for (;; ++k) {
      const int s = k % S;
      if (k >= S) {
        finish_unit(s, (k / S) - 1);
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
          load_unit<C, B, PACKED, TILE>(a, &tm_in, u, smem + s * STAGE, &full_bar[s]);
      }
      u = __shfl_sync(0xFFFFFFFFu, u, 0);
      if (u < 0) break;
    }
    // k units were loaded; units [done_units, k) still need their store.
    for (int j = done_units; j < k; ++j) finish_unit(j % S, j / S);
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
  using SumT = typename std::conditional<(SB * SB * 255 < 65536), uint16_t, uint32_t>::type;
  struct CellRec {
    int cw, f, cell, gidx;
    int64_t off;
  };
  __shared__ SumT csum[VAR ? kConsumers / 32 : 1][VAR ? CPW : 1][VAR ? NN * C : 1];
  __shared__ CellRec crec[VAR ? kConsumers / 32 : 1][VAR ? CPW : 1];
  __shared__ uint64_t cstate[VAR ? kConsumers / 32 : 1][VAR ? CPW : 1][C];
  const int wq = VAR ? (t >> 5) : 0;          // consumer warp
  const int cw = VAR ? ((t & 31) / B4) : 0;   // cell within the warp
  if (PACKED) {
    const int v0 = g.N * C, pad = (g.GC * B - g.N) * C;
    for (int x = t; x < pad && x < 128; x += kConsumers) {
      const int cpx = (v0 + x) / C, ch = (v0 + x) - cpx * C;
      fill_src[x] = static_cast<uint16_t>(reflect_index(cpx, g.N) * C + ch);
    }
    named_bar_sync(1, kConsumers);
  }
  auto load_meta = [&](int k_next) {
    Meta m;
    const int sn = k_next % S;
    mbar_wait(&id_bar[sn], (k_next / S) & 1);
    m.u = *reinterpret_cast<volatile int*>(&stage_unit[sn]);
    m.info = 1u;
    m.rowpre = m.stot = 0;
#pragma unroll
    for (int ch = 0; ch < C; ++ch) m.seed[ch] = 0;
    if (m.u >= 0) {
      const UnitPos q = decode_unit<PACKED, TILE>(a, m.u);
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
  Meta next = load_meta(0);
  for (int k = 0;; ++k) {
    const int s = k % S;
    uint8_t* st = smem + s * STAGE;
    const Meta cur = next;
    const int u = cur.u;
    if (u < 0) break;
    const UnitPos p = decode_unit<PACKED, TILE>(a, u);
    const int f = p.fg * units_pack<PACKED>(a) + jj;  // this thread's frame
    const int cell = PACKED ? (p.px0 + lpx) / B : p.px0 / B + sx / B4;
    const int lic = sx % B4;       // lane within cell
    const int sc = lic / SB4;      // subcell column
    const bool active = in_slot && (!PACKED || f < g.F) && cell < g.GC;
    const int gidx = p.r * g.GC + cell;
    const bool simple0 = !ADAPTIVE || (cur.info & 1u);  // VAR: decided after the sums
    const uint32_t slot_s = cur.rowpre + (cur.info >> 1);
    const uint32_t S_tot = cur.stot;
    const int vbytes = valid_bytes<C, PACKED, TILE>(a, p.px0);
    const int copy = staged_bytes<C, B, PACKED, TILE>(a, p);  // bytes per row the producer staged
    const int need = min(slot_px<PACKED, TILE>(a), g.GC * B - p.px0) * C;
    const int nf = PACKED ? min(a.pack, g.F - p.fg * a.pack) : 1;
    uint64_t cs[C];
#pragma unroll
    for (int ch = 0; ch < C; ++ch)
      cs[ch] = a.noise.kind == DPPX_NOISE_KEYED ? key_cell(cur.seed[ch], p.r, cell) : 0ull;

    mbar_wait(&full_bar[s], (k / S) & 1);

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
        const int rows_total = nf * B;
        for (int pr = t / kLanes; pr < rows_total; pr += kConsumers / kLanes) {
          const int j = pr / B, i = pr - j * B;  // B is a compile-time power of two
          uint8_t* rowp = st + j * (PACKED ? a.slot_stride : 0) + i * srb;
          const int frame = p.fg * units_pack<PACKED>(a) + j;
          const int srow = reflect_index(p.r * B + i, g.M);
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
      next = load_meta(k + 1);
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
      constexpr bool compact = VAR;
      const bool cx = active && !simple;
      const unsigned cx_any = __ballot_sync(0xFFFFFFFFu, cx);
      __syncwarp();  // the previous unit's reads of this warp's tables are done
      if (!VAR || cx_any) {
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
          if (cx_any) {
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
              group_values<C, SB4>(a, env_sub, cx, acc, cs, f, p.r, cell, vs, sc, val);
              if (cx) {
                if (lic % SB4 == 0) {
                  const int64_t off =
                      VAR ? a.stage_cx + static_cast<int64_t>(gidx) * NN + vs * NSUB + sc
                          : stat_offset(a, false, gidx, slot_s, S_tot, vs, sc);
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
      if constexpr (!VAR) next = load_meta(k + 1);
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
                        : stat_offset(a, false, gidx, slot_s, S_tot, 0, 0);
#pragma unroll
          for (int ch = 0; ch < C; ++ch) cstate[wq][rank][ch] = cs[ch];
        }
        __syncwarp();
        const int work = __popc(leaders) * NN * C;
        for (int i = t & 31; i < work; i += 32) {
          const int kk = i / (NN * C), rem = i - kk * (NN * C);
          const int sidx = rem / C, ch = rem - sidx * C;
          const int vs = sidx / NSUB, sc2 = sidx - vs * NSUB;
          const CellRec& rec = crec[wq][kk];
          const uint32_t sum = csum[wq][rec.cw][rem];
          const uint32_t v =
              quantize_stat(env_sub, sum, draw_bits(a, cstate[wq][kk][ch], rec.f, ch, p.r, rec.cell, vs, sc2),
                            inj_at(a, rec.f, ch, rec.gidx, vs, sc2));
          uint8_t* base = VAR ? a.stage + static_cast<int64_t>(rec.f * C + ch) * a.stage_stride
                              : a.stats + static_cast<int64_t>(rec.f * C + ch) * a.sstride;
          base[rec.off + sidx] = static_cast<uint8_t>(v);
          csum[wq][rec.cw][rem] = static_cast<SumT>(v);
        }
        __syncwarp();
        if (emit && cx) {
#pragma unroll 1
          for (int vs = 0; vs < NSUB; ++vs) {
            uint32_t val[C];
#pragma unroll
            for (int ch = 0; ch < C; ++ch) val[ch] = csum[wq][cw][(vs * NSUB + sc) * C + ch];
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
    } else {
#pragma unroll
      for (int i = 0; i < B; ++i) accumulate_row<C>(mystrip + i * srb, tot);
      // Next unit's metadata: requested here (after the staged rows are
      // summed) rather than at the top, so a 2-stage ring never stalls on the
      // producer's previous store; its latency hides behind the epilogue.
      next = load_meta(k + 1);
    }

    // whole cell (uniform, or adaptive simple): reduce over B4 strips.
#pragma unroll
    for (int ch = 0; ch < C; ++ch) tot[ch] = group_sum<B4>(tot[ch]);
    {
      uint32_t val[C];
      group_values<C, B4>(a, env_cell, active && simple, tot, cs, f, p.r, cell, 0, 0, val);
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

    fence_proxy_async_smem();
    mbar_arrive(&done_bar[s]);
  }
}

// ============================================================================
// K1g: generic kernel (any b, n, C <= 4, any pitch / alignment)
// ============================================================================
constexpr int kGenericThreads = 128;

__global__ void __launch_bounds__(kGenericThreads) k_stats_generic(const StatsArgs a) {
  const BatchGeom& g = a.g;
  const int c = blockIdx.x * kGenericThreads + threadIdx.x;
  if (c >= g.GC) return;
  // grid-stride over rows and frames: GR or F may exceed the 65535 grid limit
  for (int r = a.row_begin + blockIdx.y; r < a.row_begin + a.row_count; r += gridDim.y)
  for (int f = blockIdx.z; f < g.F; f += gridDim.z) {
    const int gidx = r * g.GC + c;
    const uint8_t* img = a.img + static_cast<int64_t>(f) * a.fstride;
    bool simple = true;
    uint32_t slot_s = 0, S_tot = 0;
    if (a.adaptive) {
      const uint32_t info = a.cellinfo[static_cast<int64_t>(f) * g.G + gidx];
      simple = info & 1u;
      slot_s = a.rowprefix[static_cast<int64_t>(f) * g.GR + r] + (info >> 1);
      S_tot = a.totals[f];
    }
    const int nsub = simple ? 1 : g.n;
    const int side = simple ? g.b : g.sb;
    if (a.partial_borders) {
      // pixelize_reference (pixelize.cpp:50-84): the border cell (r, c) covers
      // h x w real pixels, mean = sum / (h*w), noise keyed (r, c, 0, 0) at sigma.
      const int i0 = r * g.b, j0 = c * g.b;
      const int h = min(g.b, g.M - i0), w = min(g.b, g.N - j0);
      const DrawEnv env = make_env(a.noise.kind, a.exact_noise != 0, static_cast<double>(h) * w,
                                   a.sigma);
      for (int ch = 0; ch < g.C; ++ch) {
        uint32_t sum = 0;
        for (int i = i0; i < i0 + h; ++i) {
          const uint8_t* row = img + static_cast<int64_t>(i) * a.pitch;
          for (int j = j0; j < j0 + w; ++j) sum += row[j * g.C + ch];
        }
        const uint32_t v = quantize_stat(env, sum, draw_bits(a, cell_state(a, f, ch, r, c), f, ch, r, c, 0, 0),
                                         inj_at(a, f, ch, gidx, 0, 0));
        a.stats[static_cast<int64_t>(f * g.C + ch) * a.sstride + gidx] = static_cast<uint8_t>(v);
        if (a.out) {
          uint8_t* o = a.out + static_cast<int64_t>(f) * a.ofstride;
          for (int i = i0; i < i0 + h; ++i)
            for (int j = j0; j < j0 + w; ++j)
              o[static_cast<int64_t>(i) * a.opitch + j * g.C + ch] = static_cast<uint8_t>(v);
        }
      }
      continue;
    }
    const DrawEnv env = make_env(a.noise.kind, a.exact_noise != 0, simple ? a.area : a.sub_area,
                                 simple ? a.sigma : a.sigma_sub);
    for (int ch = 0; ch < g.C; ++ch) {
      const uint64_t cs = cell_state(a, f, ch, r, c);
      for (int sr = 0; sr < nsub; ++sr)
        for (int sc = 0; sc < nsub; ++sc) {
          const int i0 = r * g.b + sr * side, j0 = c * g.b + sc * side;
          uint32_t sum = 0;
          for (int i = i0; i < i0 + side; ++i) {
            const uint8_t* row = img + static_cast<int64_t>(reflect_index(i, g.M)) * a.pitch;
            for (int j = j0; j < j0 + side; ++j) sum += row[reflect_index(j, g.N) * g.C + ch];
          }
          const uint32_t v = quantize_stat(env, sum, draw_bits(a, cs, f, ch, r, c, sr, sc),
                                           inj_at(a, f, ch, gidx, sr, sc));
          a.stats[static_cast<int64_t>(f * g.C + ch) * a.sstride +
                  stat_offset(a, simple, gidx, slot_s, S_tot, sr, sc)] = static_cast<uint8_t>(v);
          if (a.out) {
            uint8_t* o = a.out + static_cast<int64_t>(f) * a.ofstride;
            for (int i = i0; i < min(i0 + side, g.M); ++i)
              for (int j = j0; j < min(j0 + side, g.N); ++j)
                o[static_cast<int64_t>(i) * a.opitch + j * g.C + ch] = static_cast<uint8_t>(v);
          }
        }
    }
  }
}

// ============================================================================
// K1r / K2r: row-streaming kernels for grid sides the TMA kernels do not cover
// (PAPER.md recommends b = 12, 24, 30, 40 and uses up to b = 128): one CTA per
// (frame, grid row). The b rows of the band are streamed through registers in
// 16-byte chunks (coalesced, SWAR byte-column sums: two u16 counters per u32),
// one vertical subcell row (sb rows) at a time; the byte-column sums go to a
// u16 smem row, subcell sums are reduced from it, complex subcells are drawn
// immediately and simple cells accumulate in smem; after the band the simple
// cells are drawn and the reconstructed rows are emitted from one pattern row
// per vertical subcell (each output row written once, coalesced).
// ============================================================================
constexpr int kRowThreads = 256;

struct RowSmem {  // byte offsets into dynamic smem (host and device agree)
  int vg;  // vertical subcells whose byte-column sums are held at once
  int vsum, cellsum, flag, slot, simpleval, subval, pattern, cstate, total;
};

__host__ __device__ inline int rows_align16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline RowSmem row_smem_layout(const BatchGeom& g) {
  RowSmem L;
  const int PB = g.GC * g.b * g.C;  // padded row bytes
  const int NS = g.GC * g.n;        // subcell columns per band
  L.vg = max(1, min(g.n, (24 * 1024) / (2 * PB)));
  L.vsum = 0;
  L.cellsum = L.vsum + rows_align16(2 * PB * L.vg);
  L.flag = L.cellsum + rows_align16(4 * g.GC * g.C);
  L.slot = L.flag + rows_align16(g.GC * g.C);
  L.simpleval = L.slot + rows_align16(4 * g.GC);
  L.subval = L.simpleval + rows_align16(g.GC * g.C);
  L.pattern = L.subval + rows_align16(g.n * NS * g.C);
  L.cstate = L.pattern + rows_align16(g.N * g.C);
  L.total = L.cstate + 8 * g.GC * g.C;
  return L;
}

// Emits rows [r*b, min(r*b + b, M)) of frame f from the smem value tables:
// pixel x, channel ch of vertical subcell vs takes simpleval[c][ch] (simple
// cell c = x / b) or subval[vs][x / sb][ch]. One pattern row per vs.
template <int C, bool ADAPTIVE>
__device__ void rows_emit(const BatchGeom& g, int r, uint8_t* out_frame, int64_t opitch,
                          const uint8_t* flag, const uint8_t* simpleval, const uint8_t* subval,
                          uint8_t* pattern, const FastDiv& div_n, bool vec16) {
  const int t = threadIdx.x;
  const int RB = g.N * C, NS = g.GC * g.n;
  for (int vs = 0; vs < g.n; ++vs) {
    const int y0 = r * g.b + vs * g.sb;
    if (y0 >= g.M) break;
    const int y1 = min(y0 + g.sb, g.M);
    // pattern row: one thread per subcell column (sb pixels of C fixed values)
    for (int sidx = t; sidx < NS; sidx += kRowThreads) {
      const int c = static_cast<int>(div_n.div(static_cast<uint32_t>(sidx)));
      uint8_t v[C];
#pragma unroll
      for (int ch = 0; ch < C; ++ch)
        v[ch] = (!ADAPTIVE || flag[c * C + ch]) ? simpleval[c * C + ch] : subval[(vs * NS + sidx) * C + ch];
      const int px0 = sidx * g.sb, px1 = min(px0 + g.sb, g.N);
      for (int px = px0; px < px1; ++px)
#pragma unroll
        for (int ch = 0; ch < C; ++ch) pattern[px * C + ch] = v[ch];
    }
    __syncthreads();
    for (int y = y0; y < y1; ++y) {
      uint8_t* orow = out_frame + static_cast<int64_t>(y) * opitch;
      if (vec16) {
        const int n16 = RB >> 4;
        for (int q = t; q < n16; q += kRowThreads)
          reinterpret_cast<uint4*>(orow)[q] = reinterpret_cast<const uint4*>(pattern)[q];
        for (int x = (n16 << 4) + t; x < RB; x += kRowThreads) orow[x] = pattern[x];
      } else {
        for (int x = t; x < RB; x += kRowThreads) orow[x] = pattern[x];
      }
    }
    __syncthreads();
  }
}

template <int C, bool ADAPTIVE, bool VEC16>
__global__ void __launch_bounds__(kRowThreads, 4) k_stats_rows(const StatsArgs a) {
  extern __shared__ __align__(16) uint8_t rsm[];
  const BatchGeom& g = a.g;
  const RowSmem L = row_smem_layout(g);
  uint16_t* vsum = reinterpret_cast<uint16_t*>(rsm + L.vsum);
  uint32_t* cellsum = reinterpret_cast<uint32_t*>(rsm + L.cellsum);
  uint8_t* flag = rsm + L.flag;
  uint32_t* slot = reinterpret_cast<uint32_t*>(rsm + L.slot);
  uint8_t* simpleval = rsm + L.simpleval;
  uint8_t* subval = rsm + L.subval;
  uint8_t* pattern = rsm + L.pattern;
  uint64_t* cstate = reinterpret_cast<uint64_t*>(rsm + L.cstate);  // key_cell per (cell, ch)
  const int t = threadIdx.x;
  const int RB = g.N * C, PB = g.GC * g.b * C, NS = g.GC * g.n;
  const FastDiv div_n = make_fastdiv(static_cast<uint32_t>(g.n));
  const DrawEnv env_cell = make_env(a.noise.kind, a.exact_noise != 0, a.area, a.sigma);
  const DrawEnv env_sub = make_env(a.noise.kind, a.exact_noise != 0, a.sub_area, a.sigma_sub);
  const bool out_vec16 = a.out && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0 &&
                         (a.opitch & 15) == 0 && (a.ofstride & 15) == 0;
  for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
    const int f = static_cast<int>(a.div_rows.div(static_cast<uint32_t>(u)));
    const int r = a.row_begin + (u - f * a.row_count);
    const uint8_t* frame = a.img + static_cast<int64_t>(f) * a.fstride;
    uint32_t S_tot = 0;
    if (ADAPTIVE) {
      S_tot = __ldg(&a.totals[f]);
      const uint32_t rowpre = __ldg(&a.rowprefix[static_cast<int64_t>(f) * g.GR + r]);
      for (int c = t; c < g.GC; c += kRowThreads) {
        const uint32_t info = __ldg(&a.cellinfo[static_cast<int64_t>(f) * g.G + r * g.GC + c]);
#pragma unroll
        for (int ch = 0; ch < C; ++ch) flag[c * C + ch] = info & 1u;
        slot[c] = rowpre + (info >> 1);
      }
    }
    for (int e = t; e < g.GC * C; e += kRowThreads) {
      cellsum[e] = 0;
      const int c = e / C, ch = e - c * C;
      cstate[e] = cell_state(a, f, ch, r, c);  // one mix64 per cell and channel
    }
    __syncthreads();
    for (int v0 = 0; v0 < g.n; v0 += L.vg) {
      const int nv = min(L.vg, g.n - v0);
      // ---- byte-column sums of vertical subcells [v0, v0 + nv) ----
      // Chunk-major: each thread owns 16-byte column chunks and walks the rows
      // of one chunk at a time (8 live SWAR counters, flushed per vertical
      // subcell; rows unrolled so several loads are in flight); a warp reads
      // 512 contiguous bytes per row.
      for (int x0 = t * 16; x0 < PB; x0 += kRowThreads * 16) {
        const uint8_t* colp = frame + x0;
        const bool fast = VEC16 && x0 + 16 <= RB;
        for (int vg = 0; vg < nv; ++vg) {
          uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
          const int row0 = r * g.b + (v0 + vg) * g.sb;
#pragma unroll 4
          for (int i = 0; i < g.sb; ++i) {
            const int srow = reflect_index(row0 + i, g.M);
            const uint8_t* rowp = colp + static_cast<int64_t>(srow) * a.pitch;
            uint32_t w[4];
            if (fast) {
              const uint4 v = __ldg(reinterpret_cast<const uint4*>(rowp));
              w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
            } else {
              const uint8_t* rowbase = rowp - x0;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint32_t acc = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int x = x0 + 4 * j + k;
                  uint32_t byte = 0;
                  if (x < RB) {
                    byte = __ldg(rowbase + x);
                  } else if (x < PB) {  // mirrored padding column (image.cpp:105-110)
                    const int px = x / C, ch = x - px * C;
                    byte = __ldg(rowbase + static_cast<int64_t>(reflect_index(px, g.N)) * C + ch);
                  }
                  acc |= byte << (8 * k);
                }
                w[j] = acc;
              }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              lo[j] += w[j] & 0x00FF00FFu;
              hi[j] += (w[j] >> 8) & 0x00FF00FFu;
            }
          }
          uint16_t* vrow = vsum + vg * PB;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int x = x0 + 4 * j;
            if (x + 0 < PB) vrow[x + 0] = static_cast<uint16_t>(lo[j] & 0xFFFFu);
            if (x + 1 < PB) vrow[x + 1] = static_cast<uint16_t>(hi[j] & 0xFFFFu);
            if (x + 2 < PB) vrow[x + 2] = static_cast<uint16_t>(lo[j] >> 16);
            if (x + 3 < PB) vrow[x + 3] = static_cast<uint16_t>(hi[j] >> 16);
          }
        }
      }
      __syncthreads();
      // ---- subcell sums; complex subcells drawn now, simple cells accumulate ----
      for (int item = t; item < nv * NS * C; item += kRowThreads) {
        const int vi = item / (NS * C);
        const int rem = item - vi * (NS * C);
        const int vs = v0 + vi;
        const int sidx = rem / C, ch = rem - sidx * C;
        const int c = static_cast<int>(div_n.div(static_cast<uint32_t>(sidx))), sc = sidx - c * g.n;
        uint32_t sum = 0;
        const uint16_t* vp = vsum + vi * PB + sidx * g.sb * C + ch;
        for (int k = 0; k < g.sb; ++k) sum += vp[k * C];
        const int gidx = r * g.GC + c;
        if (!ADAPTIVE) {  // n == 1: the subcell is the cell
          const uint64_t cs = cstate[c * C + ch];
          const uint32_t v = quantize_stat(env_cell, sum, draw_bits(a, cs, f, ch, r, c, 0, 0),
                                           inj_at(a, f, ch, gidx, 0, 0));
          a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + gidx] = static_cast<uint8_t>(v);
          simpleval[c * C + ch] = static_cast<uint8_t>(v);
        } else if (flag[c * C + ch]) {
          atomicAdd(&cellsum[c * C + ch], sum);
        } else {
          const uint64_t cs = cstate[c * C + ch];
          const uint32_t v = quantize_stat(env_sub, sum, draw_bits(a, cs, f, ch, r, c, vs, sc),
                                           inj_at(a, f, ch, gidx, vs, sc));
          a.stats[static_cast<int64_t>(f * C + ch) * a.sstride +
                  stat_offset(a, false, gidx, slot[c], S_tot, vs, sc)] = static_cast<uint8_t>(v);
          subval[(vs * NS + sidx) * C + ch] = static_cast<uint8_t>(v);
        }
      }
      __syncthreads();
    }
    if (ADAPTIVE) {  // simple cells: one draw per channel at sigma
      for (int item = t; item < g.GC * C; item += kRowThreads) {
        const int c = item / C, ch = item - c * C;
        if (!flag[item]) continue;
        const int gidx = r * g.GC + c;
        const uint64_t cs = cstate[item];
        const uint32_t v = quantize_stat(env_cell, cellsum[item], draw_bits(a, cs, f, ch, r, c, 0, 0),
                                         inj_at(a, f, ch, gidx, 0, 0));
        a.stats[static_cast<int64_t>(f * C + ch) * a.sstride +
                stat_offset(a, true, gidx, slot[c], S_tot, 0, 0)] = static_cast<uint8_t>(v);
        simpleval[item] = static_cast<uint8_t>(v);
      }
      __syncthreads();
    }
    if (a.out)
      rows_emit<C, ADAPTIVE>(g, r, a.out + static_cast<int64_t>(f) * a.ofstride, a.opitch, flag,
                             simpleval, subval, pattern, div_n, out_vec16);
    __syncthreads();
  }
}

// K2r: statistics -> pixels for the same grid sides (broadcast_means /
// reassemble), one CTA per (plane group = frame, grid row): value tables from
// the payload slots (K0 run on the payload), then rows_emit.
template <int C, bool ADAPTIVE>
__global__ void __launch_bounds__(kRowThreads) k_expand_rows(const ExpandArgs a, int units,
                                                             FastDiv div_rows) {
  extern __shared__ __align__(16) uint8_t rsm[];
  const BatchGeom& g = a.g;
  const RowSmem L = row_smem_layout(g);
  uint8_t* flag = rsm + L.flag;
  uint8_t* simpleval = rsm + L.simpleval;
  uint8_t* subval = rsm + L.subval;
  uint8_t* pattern = rsm + L.pattern;
  const int t = threadIdx.x;
  const int NS = g.GC * g.n, nn = g.n * g.n;
  const FastDiv div_n = make_fastdiv(static_cast<uint32_t>(g.n));
  const bool out_vec16 = (reinterpret_cast<uintptr_t>(a.out) & 15) == 0 && (a.opitch & 15) == 0 &&
                         (a.ofstride & 15) == 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int f = static_cast<int>(div_rows.div(static_cast<uint32_t>(u)));
    const int r = u - f * g.GR;
    for (int e = t; e < g.GC * C; e += kRowThreads) {
      const int c = e / C, ch = e - c * C;
      const int64_t plane = static_cast<int64_t>(f) * C + ch;
      const uint8_t* st = a.stats + plane * a.sstride;
      const int gidx = r * g.GC + c;
      if (!ADAPTIVE) {
        simpleval[e] = __ldg(st + gidx);
        continue;
      }
      const uint32_t info = __ldg(&a.cellinfo[plane * g.G + gidx]);
      const uint32_t slot_s = __ldg(&a.rowprefix[plane * g.GR + r]) + (info >> 1);
      const int64_t base = 4ll * g.G + 4;
      flag[e] = info & 1u;
      if (info & 1u) {
        simpleval[e] = __ldg(st + base + slot_s);
      } else {
        const uint8_t* sub = st + base + __ldg(&a.totals[plane]) +
                             static_cast<int64_t>(static_cast<uint32_t>(gidx) - slot_s) * nn;
        for (int k = 0; k < nn; ++k) {
          const int vs = k / g.n, sc = k - vs * g.n;
          subval[(vs * NS + c * g.n + sc) * C + ch] = __ldg(sub + k);
        }
      }
    }
    __syncthreads();
    rows_emit<C, ADAPTIVE>(g, r, a.out + static_cast<int64_t>(f) * a.ofstride, a.opitch, flag,
                           simpleval, subval, pattern, div_n, out_vec16);
    __syncthreads();
  }
}

// ============================================================================
// K2: statistics -> pixels (broadcast_means pixelize.cpp:126-150,
//     reassemble adaptive.cpp:181-245). One thread per (plane, grid row, cell).
// ============================================================================
__global__ void __launch_bounds__(kGenericThreads) k_expand(const ExpandArgs a) {
  const BatchGeom& g = a.g;
  const int c = blockIdx.x * kGenericThreads + threadIdx.x;
  if (c >= g.GC) return;
  const int P = g.F * g.C;
  for (int r = blockIdx.y; r < g.GR; r += gridDim.y)
  for (int p = blockIdx.z; p < P; p += gridDim.z) {
    const int gidx = r * g.GC + c;
    const int f = p / g.C, ch = p % g.C;
    const uint8_t* st = a.stats + static_cast<int64_t>(p) * a.sstride;
    uint8_t* o = a.out + static_cast<int64_t>(f) * a.ofstride;
    const int i0 = r * g.b, j0 = c * g.b;
    const int i1 = min(i0 + g.b, g.M), j1 = min(j0 + g.b, g.N);
    if (!a.adaptive) {
      const uint8_t v = st[gidx];
      for (int i = i0; i < i1; ++i)
        for (int j = j0; j < j1; ++j) o[static_cast<int64_t>(i) * a.opitch + j * g.C + ch] = v;
      continue;
    }
    const uint32_t info = a.cellinfo[static_cast<int64_t>(p) * g.G + gidx];
    const uint32_t slot_s = a.rowprefix[static_cast<int64_t>(p) * g.GR + r] + (info >> 1);
    const int64_t base = 4ll * g.G + 4;
    if (info & 1u) {
      const uint8_t v = st[base + slot_s];
      for (int i = i0; i < i1; ++i)
        for (int j = j0; j < j1; ++j) o[static_cast<int64_t>(i) * a.opitch + j * g.C + ch] = v;
    } else {
      const uint32_t slot_c = static_cast<uint32_t>(gidx) - slot_s;
      const uint8_t* sub = st + base + a.totals[p] + static_cast<int64_t>(slot_c) * g.n * g.n;
      for (int i = i0; i < i1; ++i)
        for (int j = j0; j < j1; ++j)
          o[static_cast<int64_t>(i) * a.opitch + j * g.C + ch] =
              sub[((i - i0) / g.sb) * g.n + (j - j0) / g.sb];
    }
  }
}

// ============================================================================
// K2 fast path: one CTA per (frame, grid row, 512-px tile); each thread owns a
// 4-px strip, looks up its cell's statistics per channel plane (packed slots
// from K0's per-plane scan), writes the strip pattern into a smem tile and one
// thread bulk-stores the tile with a 3-D TMA box (clipped at M and N).
// ============================================================================
// Packed (narrow-frame) instantiations run 256 threads: a 1024-px tile holds
// more frame slots per CTA (5 CelebA frames instead of 2).
constexpr int kExpandPackedThreads = 256;

template <int C, int B4, int NSUB, bool ADAPTIVE, bool PACKED>
__global__ void __launch_bounds__(PACKED ? kExpandPackedThreads : kConsumers)
    k_expand_tma(const __grid_constant__ CUtensorMap tm_out, const ExpandArgs a) {
  constexpr int B = 4 * B4, SB = B / NSUB, SB4 = SB / 4;
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
  const int sc = (sx % B4) / SB4;
  for (int u = blockIdx.x, k = 0; u < a.units; u += gridDim.x, ++k) {
    uint8_t* buf = smem;
    // A capped grid loops: the previous unit's store must have read the tile.
    if (t == 0 && k > 0) bulk_wait_read_all();
    __syncthreads();
    const uint32_t rest = a.div_tiles.div(static_cast<uint32_t>(u));
    const int tile = u - static_cast<int>(rest * a.div_tiles.d);
    const uint32_t fq = a.div_rows.div(rest);
    const int r = static_cast<int>(rest - fq * a.div_rows.d);
    const int fg = static_cast<int>(fq);
    const int pk = PACKED ? a.pack : 1;
    const int nf = PACKED ? min(pk, g.F - fg * pk) : 1;
    const int f = fg * pk + jj;
    const int px0 = PACKED ? 0 : tile * TILE;
    const int cell = (px0 + lpx) / B;
    const bool active = in_slot && jj < nf && cell < g.GC;
    const int gidx = r * g.GC + cell;
    uint32_t val[NSUB][C];
    if (active) {
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        const int64_t plane = static_cast<int64_t>(f) * C + ch;
        const uint8_t* st = a.stats + plane * a.sstride;
        if constexpr (!ADAPTIVE) {
          const uint32_t v = __ldg(st + gidx);
#pragma unroll
          for (int vs = 0; vs < NSUB; ++vs) val[vs][ch] = v;
        } else {
          const uint32_t info = __ldg(&a.cellinfo[plane * g.G + gidx]);
          const uint32_t slot_s = __ldg(&a.rowprefix[plane * g.GR + r]) + (info >> 1);
          const int64_t base = 4ll * g.G + 4;
          if (info & 1u) {
            const uint32_t v = __ldg(st + base + slot_s);
#pragma unroll
            for (int vs = 0; vs < NSUB; ++vs) val[vs][ch] = v;
          } else {
            const uint8_t* sub = st + base + __ldg(&a.totals[plane]) +
                                 static_cast<int64_t>(static_cast<uint32_t>(gidx) - slot_s) * NSUB * NSUB;
#pragma unroll
            for (int vs = 0; vs < NSUB; ++vs) val[vs][ch] = __ldg(sub + vs * NSUB + sc);
          }
        }
      }
      uint8_t* mystrip = buf + jj * (PACKED ? a.slot_stride : 0) + lpx * C;
#pragma unroll
      for (int vs = 0; vs < NSUB; ++vs) {
        uint32_t w[C];
        pattern_words<C>(val[vs], w);
#pragma unroll
        for (int i = 0; i < SB; ++i)
#pragma unroll
          for (int q = 0; q < C; ++q)
            reinterpret_cast<uint32_t*>(mystrip + (vs * SB + i) * srb)[q] = w[q];
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int scopy = max(0, min(srb, a.tensor_out_bytes - px0 * C));
    if (t == 0 && scopy > 0) {
      for (int j = 0; j < nf; ++j)
        tma_store_3d(&tm_out, px0 * C / 8, r * B, fg * pk + j, buf + j * (PACKED ? a.slot_stride : 0));
    }
    if (t == 0) bulk_commit();  // one group per unit (possibly empty)
    // Bytes past the tensor's row extent (< 8 per row and slot), from the smem
    // tile, spread over the whole CTA (one thread per byte, not per strip).
    const int vbytes = min(slot_px, g.N - px0) * C;
    const int span = vbytes - scopy;
    if (span > 0) {
      const int rows = min(B, g.M - r * B);
      for (int e = t; e < nf * rows * span; e += NT) {
        const int jr = e / span, x = scopy + (e - jr * span);
        const int j = jr / rows, i = jr - j * rows;
        a.out[static_cast<int64_t>(fg * pk + j) * a.ofstride + static_cast<int64_t>(r * B + i) * a.opitch +
              static_cast<int64_t>(px0) * C + x] = buf[j * (PACKED ? a.slot_stride : 0) + i * srb + x];
      }
    }
  }
  if (t == 0) bulk_wait_read_all();  // smem must outlive the stores' reads
}

// ============================================================================
// Utility metrics: mse / ssim of metrics.cpp:26-183, per
// channel plane of interleaved frames a (pitch/fstride) and b (opitch/ofstride).
// ============================================================================
struct MetricArgs {
  int M, N, C, F;
  const uint8_t* a;
  int64_t pitch, fstride;
  const uint8_t* b;
  int64_t bpitch, bfstride;
  unsigned long long* sums;  // mse: [F*C] exact u64 sums of squared differences
  double* row_sums;          // ssim: [F*C][M-6] per-window-row partials
};

// Exact SSD per plane: one block per (frame, row band), byte channels by offset.
__global__ void __launch_bounds__(256) k_mse(const MetricArgs m) {
  __shared__ unsigned long long part[4];
  if (threadIdx.x < 4) part[threadIdx.x] = 0ull;
  __syncthreads();
  unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
  const int rows_per_block = 8;
  const int row_bytes = m.N * m.C;
  for (int f = blockIdx.y; f < m.F; f += gridDim.y) {  // F may exceed the 65535 grid limit
  for (int ch = 0; ch < 4; ++ch) acc[ch] = 0ull;
  __syncthreads();
  if (threadIdx.x < 4) part[threadIdx.x] = 0ull;
  __syncthreads();
  for (int i = blockIdx.x * rows_per_block; i < min(m.M, (blockIdx.x + 1) * rows_per_block); ++i) {
    const uint8_t* ra = m.a + static_cast<int64_t>(f) * m.fstride + static_cast<int64_t>(i) * m.pitch;
    const uint8_t* rb = m.b + static_cast<int64_t>(f) * m.bfstride + static_cast<int64_t>(i) * m.bpitch;
    for (int x = threadIdx.x; x < row_bytes; x += blockDim.x) {
      const int d = static_cast<int>(__ldg(ra + x)) - static_cast<int>(__ldg(rb + x));
      const int ch = m.C == 1 ? 0 : x % m.C;
      acc[ch] += static_cast<unsigned long long>(d * d);
    }
  }
  for (int ch = 0; ch < m.C; ++ch) atomicAdd(&part[ch], acc[ch]);
  __syncthreads();
  if (threadIdx.x < m.C) atomicAdd(&m.sums[static_cast<int64_t>(f) * m.C + threadIdx.x], part[threadIdx.x]);
  }
}

// One thread per (plane, window row): slides the 7x7 window along the row with
// exact integer column sums and accumulates the local SSIM in the reference's
// order (metrics.cpp:144-177): the row partial is bit-identical.
__global__ void __launch_bounds__(128) k_ssim_rows(const MetricArgs m) {
  constexpr int W = 7;
  const int pr = m.M - W + 1, pc = m.N - W + 1;
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t planes = static_cast<int64_t>(m.F) * m.C;
  if (idx >= planes * pr) return;
  const int64_t p = idx / pr;
  const int i = static_cast<int>(idx - p * pr);
  const int f = static_cast<int>(p / m.C), ch = static_cast<int>(p - static_cast<int64_t>(f) * m.C);
  const uint8_t* a = m.a + static_cast<int64_t>(f) * m.fstride + static_cast<int64_t>(i) * m.pitch + ch;
  const uint8_t* b = m.b + static_cast<int64_t>(f) * m.bfstride + static_cast<int64_t>(i) * m.bpitch + ch;
  uint32_t ring[W][5];
  uint32_t win[5] = {0u, 0u, 0u, 0u, 0u};
  auto column = [&](int c, uint32_t (&out)[5]) {
    uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
    for (int y = 0; y < W; ++y) {
      const uint32_t va = __ldg(a + static_cast<int64_t>(y) * m.pitch + static_cast<int64_t>(c) * m.C);
      const uint32_t vb = __ldg(b + static_cast<int64_t>(y) * m.bpitch + static_cast<int64_t>(c) * m.C);
      s0 += va;
      s1 += vb;
      s2 += va * va;
      s3 += vb * vb;
      s4 += va * vb;
    }
    out[0] = s0, out[1] = s1, out[2] = s2, out[3] = s3, out[4] = s4;
  };
#pragma unroll
  for (int c = 0; c < W; ++c) {
    column(c, ring[c]);
#pragma unroll
    for (int q = 0; q < 5; ++q) win[q] += ring[c][q];
  }
  const double area = 49.0, c1 = 6.5025, c2 = 58.5225;
  double acc = 0.0;
  for (int j = 0; j < pc; ++j) {
    if (j > 0) {  // slide: drop column j-1, add column j+6 (ring slot (j-1) % 7)
      const int slot = (j - 1) % W;
      uint32_t nc[5];
      column(j + W - 1, nc);
#pragma unroll
      for (int k = 0; k < W; ++k)
        if (k == slot) {
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            win[q] = win[q] - ring[k][q] + nc[q];
            ring[k][q] = nc[q];
          }
        }
    }
    const double mu_a = __ddiv_rn(static_cast<double>(win[0]), area);
    const double mu_b = __ddiv_rn(static_cast<double>(win[1]), area);
    const double raw_aa = __ddiv_rn(static_cast<double>(win[2]), area);
    const double raw_bb = __ddiv_rn(static_cast<double>(win[3]), area);
    const double raw_ab = __ddiv_rn(static_cast<double>(win[4]), area);
    const double mu_aa = __dmul_rn(mu_a, mu_a), mu_bb = __dmul_rn(mu_b, mu_b),
                 mu_ab = __dmul_rn(mu_a, mu_b);
    const double var_a = __dsub_rn(raw_aa, mu_aa), var_b = __dsub_rn(raw_bb, mu_bb),
                 cov = __dsub_rn(raw_ab, mu_ab);
    const double num = __dmul_rn(__dadd_rn(__dmul_rn(2.0, mu_ab), c1), __dadd_rn(__dmul_rn(2.0, cov), c2));
    const double den = __dmul_rn(__dadd_rn(__dadd_rn(mu_aa, mu_bb), c1),
                                 __dadd_rn(__dadd_rn(var_a, var_b), c2));
    acc = __dadd_rn(acc, __ddiv_rn(num, den));
  }
  m.row_sums[p * pr + i] = acc;
}

cudaError_t launch_metrics(const MetricArgs& m, bool ssim, cudaStream_t s) {
  if (!ssim) {
    dim3 grid((m.M + 7) / 8, m.F < 65535 ? m.F : 65535);
    k_mse<<<grid, 256, 0, s>>>(m);
  } else {
    const int64_t threads = static_cast<int64_t>(m.F) * m.C * (m.M - 6);
    k_ssim_rows<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, s>>>(m);
  }
  return cudaGetLastError();
}

// ============================================================================
// Synthetic workload generator (mirrors oracle/dppx_oracle.c or_synth_*)
// ============================================================================
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void k_synth(BatchGeom g, uint32_t data_seed, uint32_t f0, uint8_t* img, int64_t pitch,
                        int64_t fstride, uint8_t* mask, int64_t mpitch, int64_t mfstride) {
  const int64_t total = static_cast<int64_t>(g.F) * g.M * g.N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e % g.N);
    const int i = static_cast<int>((e / g.N) % g.M);
    const uint32_t f = f0 + static_cast<uint32_t>(e / (static_cast<int64_t>(g.N) * g.M));
    const int ff = static_cast<int>(f - f0);
    const int jj = static_cast<int>((static_cast<long long>(j) + f) % g.N);
    const long long dy = 2LL * i + 1 - g.M, dx = 2LL * jj + 1 - g.N;
    const long long rad = (g.M < g.N ? g.M : g.N) / 2;
    for (int k = 0; k < g.C; ++k) {
      int v = (i + 2 * jj + 85 * k) & 255;
      if (dy * dy + dx * dx < rad * rad) v = 200 - 40 * k;
      if (i < g.M / 2 && jj < g.N / 2 && (((i >> 3) + (jj >> 3)) & 1) == 0) v = 255 - v;
      const uint32_t h =
          hash32(data_seed ^ hash32(f * 0x9E3779B1u ^
                                    hash32(static_cast<uint32_t>(k) * 0x85EBCA77u ^
                                           hash32(static_cast<uint32_t>(i) * 0xC2B2AE3Du ^
                                                  static_cast<uint32_t>(j)))));
      img[ff * fstride + static_cast<int64_t>(i) * pitch + static_cast<int64_t>(j) * g.C + k] =
          static_cast<uint8_t>(v ^ static_cast<int>(h & 0x3F));
    }
    if (mask) {
      const long long ay = (4LL * g.M) / 5, ax = (2LL * g.N) / 5;
      const long long cx2 = (static_cast<long long>(g.N) + 4LL * f) % (2LL * g.N);
      long long mdx = 2LL * j + 1 - cx2;
      if (mdx > g.N) mdx -= 2LL * g.N;
      if (mdx < -g.N) mdx += 2LL * g.N;
      const long long mdy = 2LL * i + 1 - g.M;
      uint8_t mv = 1;
      if (ay != 0 && ax != 0)
        mv = (mdy * mdy * ax * ax + mdx * mdx * ay * ay < ax * ax * ay * ay) ? 0 : 1;
      mask[ff * mfstride + static_cast<int64_t>(i) * mpitch + j] = mv;
    }
  }
}

// Max |lg2.approx(m) - log2(m)| over every f32 mantissa m in [1, 2): the
// bound the fast quantization path relies on (dppx_device.cuh).
__global__ void k_debug_lg2(unsigned int* max_bits) {
  float worst = 0.f;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (1u << 23);
       i += gridDim.x * blockDim.x) {
    const float m = __uint_as_float(0x3F800000u | i);
    const double exact = log2(static_cast<double>(m));
    worst = fmaxf(worst, static_cast<float>(fabs(static_cast<double>(__log2f(m)) - exact)));
  }
  atomicMax(max_bits, __float_as_uint(worst));
}

// Row re-pitch for the host pipeline: PCIe moves dense rows (one linear copy),
// the kernels want 16-byte pitched rows (TMA). rows x width bytes.
__global__ void k_repitch(uint8_t* __restrict__ dst, int64_t dpitch, const uint8_t* __restrict__ src,
                          int64_t spitch, int64_t width, int64_t rows) {
  const int64_t chunks = (width + 15) / 16;
  const int64_t total = rows * chunks;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / chunks, x0 = (e - r * chunks) * 16;
    const uint8_t* sp = src + r * spitch + x0;
    uint8_t* dp = dst + r * dpitch + x0;
    const int64_t n = width - x0 < 16 ? width - x0 : 16;
    if (n == 16 && ((reinterpret_cast<uintptr_t>(dp) | reinterpret_cast<uintptr_t>(sp)) & 15) == 0) {
      *reinterpret_cast<uint4*>(dp) = __ldg(reinterpret_cast<const uint4*>(sp));
    } else {
      uint8_t v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = k < n ? __ldg(sp + k) : 0;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < n) dp[k] = v[k];
    }
  }
}

__global__ void k_debug_laplace(uint64_t mixed_seed, const uint32_t* keys, int count, double sigma,
                                double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint32_t* k = keys + 4 * i;
  out[i] = laplace_from_uniform(uniform_from_bits(key_sub(key_cell(mixed_seed, k[0], k[1]), k[2], k[3])),
                                sigma);
}

// ============================================================================
// Fused-variance compaction: staged per-cell statistics -> DPPX payload slots
// (simple value at 4G+4+slot, complex block at 4G+4+S+slot_c*n*n), using the
// slots K0 (mode 3) derived from the flags K1 wrote.
// ============================================================================
__global__ void __launch_bounds__(kGenericThreads) k_gather_stage(const GatherArgs a) {
  const BatchGeom& g = a.g;
  const int nn = g.n * g.n;
  const int P = g.F * g.C;
  for (int p = blockIdx.y; p < P; p += gridDim.y) {
    const int f = p / g.C;
    const uint8_t* src = a.stage + static_cast<int64_t>(p) * a.stage_stride;
    uint8_t* dst = a.payload + static_cast<int64_t>(p) * a.pstride + 4ll * g.G + 4;
    const uint32_t S = __ldg(&a.totals[f]);
    for (int gi = blockIdx.x * kGenericThreads + threadIdx.x; gi < g.G; gi += gridDim.x * kGenericThreads) {
      const uint32_t info = __ldg(&a.cellinfo[static_cast<int64_t>(f) * g.G + gi]);
      const int r = gi / g.GC;
      const uint32_t slot_s = __ldg(&a.rowprefix[static_cast<int64_t>(f) * g.GR + r]) + (info >> 1);
      if (info & 1u) {
        dst[slot_s] = __ldg(src + gi);
        continue;
      }
      const uint8_t* cs = src + a.stage_cx + static_cast<int64_t>(gi) * nn;
      uint8_t* d = dst + S + static_cast<int64_t>(static_cast<uint32_t>(gi) - slot_s) * nn;
      if (nn % 4 == 0 && (reinterpret_cast<uintptr_t>(d) & 3) == 0) {
        for (int k = 0; k < nn; k += 4)
          *reinterpret_cast<uint32_t*>(d + k) = __ldg(reinterpret_cast<const uint32_t*>(cs + k));
      } else {
        for (int k = 0; k < nn; k += 4) {  // staged blocks are 4-byte aligned when nn % 4 == 0
          const int m = min(4, nn - k);
          for (int q = 0; q < m; ++q) d[k + q] = __ldg(cs + k + q);
        }
      }
    }
  }
}

// ============================================================================
// Host-side launchers (called from capi.cu)
// ============================================================================
using StatsKernel = void (*)(const CUtensorMap, const CUtensorMap, const StatsArgs);

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

// Fused variance classification (wide frames only; else the 2-pass path).
StatsKernel select_stats_kernel_var(int C, int b, int n) {
  if (C == 1) return pick_var<1>(b, n);
  if (C == 3) return pick_var<3>(b, n);
  return nullptr;
}

cudaError_t launch_gather_stage(const GatherArgs& a, cudaStream_t s) {
  const int P = a.g.F * a.g.C;
  const int bx = std::min((a.g.G + kGenericThreads - 1) / kGenericThreads, 64);
  dim3 grid(bx > 0 ? bx : 1, P < 65535 ? P : 65535);
  k_gather_stage<<<grid, kGenericThreads, 0, s>>>(a);
  return cudaGetLastError();
}

StatsKernel select_stats_kernel(int C, int b, int n, bool adaptive, bool packed) {
  if (!adaptive && n != 1) return nullptr;
  if (C == 1) {
    if (packed) return adaptive ? pick_b<1, true, true>(b, n) : pick_b<1, false, true>(b, n);
    return adaptive ? pick_b<1, true, false>(b, n) : pick_b<1, false, false>(b, n);
  }
  if (C == 3) {
    if (packed) return adaptive ? pick_b<3, true, true>(b, n) : pick_b<3, false, true>(b, n);
    return adaptive ? pick_b<3, true, false>(b, n) : pick_b<3, false, false>(b, n);
  }
  return nullptr;
}

using ExpandKernel = void (*)(const CUtensorMap, const ExpandArgs);

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
    }
  }
  if constexpr (AD) {
    DPPX_CASE(2, 2)
    DPPX_CASE(4, 2)
    DPPX_CASE(4, 4)
    DPPX_CASE(8, 2)
    DPPX_CASE(8, 4)
    DPPX_CASE(8, 8)
  }
#undef DPPX_CASE
  return nullptr;
}

ExpandKernel select_expand_kernel(int C, int b, int n, bool adaptive, bool packed) {
  if (!adaptive && n != 1) return nullptr;
  if (C == 1) {
    if (packed) return adaptive ? pick_expand<1, true, true>(b, n) : pick_expand<1, false, true>(b, n);
    return adaptive ? pick_expand<1, true, false>(b, n) : pick_expand<1, false, false>(b, n);
  }
  if (C == 3) {
    if (packed) return adaptive ? pick_expand<3, true, true>(b, n) : pick_expand<3, false, true>(b, n);
    return adaptive ? pick_expand<3, true, false>(b, n) : pick_expand<3, false, false>(b, n);
  }
  return nullptr;
}

cudaError_t launch_expand_tma(ExpandKernel k, const CUtensorMap& tout, const ExpandArgs& a,
                              int grid, size_t smem, cudaStream_t s) {
  k<<<grid, a.pack > 1 ? kExpandPackedThreads : kConsumers, smem, s>>>(tout, a);
  return cudaGetLastError();
}

int expand_packed_tile_px() { return 4 * kExpandPackedThreads; }

int stats_threads() { return kStatsThreads; }
int stats_tile_px() { return kTilePx; }

// Tile width of the staged kernel for grid side b (whole cells per warp).
int stats_tile_px_for(int b) {
  const int b4 = b / 4;
  if (b % 4 != 0 || b4 < 1 || b4 > 32) return kTilePx;
  return 4 * (kConsumers / 32) * ((32 / b4) * b4);
}
int stats_max_stages() { return kMaxStages; }

cudaError_t launch_classify(const ClassifyArgs& a, cudaStream_t s) {
  dim3 grid(a.g.GR, a.planes < 65535 ? a.planes : 65535);
  if (!a.band) {
    k_classify<false><<<grid, kClassifyThreads, 0, s>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = static_cast<size_t>(a.g.GC) * (a.band == 2 ? 1 : a.g.b) * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_classify<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  k_classify<true><<<grid, kClassifyThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_stats_tma(StatsKernel k, const CUtensorMap& tin, const CUtensorMap& tout,
                             const StatsArgs& a, int grid, size_t smem, cudaStream_t s) {
  k<<<grid, kStatsThreads, smem, s>>>(tin, tout, a);
  return cudaGetLastError();
}

cudaError_t launch_stats_generic(const StatsArgs& a, cudaStream_t s) {
  dim3 grid((a.g.GC + kGenericThreads - 1) / kGenericThreads,
            a.row_count < 65535 ? (a.row_count > 0 ? a.row_count : 1) : 65535,
            a.g.F < 65535 ? a.g.F : 65535);
  k_stats_generic<<<grid, kGenericThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// Row-streaming kernels: smem bytes needed (0 = not applicable).
int rows_smem_bytes(const BatchGeom& g) {
  if (g.C != 1 && g.C != 3 && g.C != 4) return 0;
  if (g.sb > 257) return 0;  // u16 byte-column counters
  if (static_cast<int64_t>(g.GC) * g.b * g.C > (1 << 20)) return 0;
  const RowSmem L = row_smem_layout(g);
  return L.total <= 200 * 1024 ? L.total : 0;
}

template <int C>
cudaError_t launch_rows_c(const StatsArgs& a, size_t smem, bool vec16, cudaStream_t s) {
  auto k = a.adaptive ? (vec16 ? k_stats_rows<C, true, true> : k_stats_rows<C, true, false>)
                      : (vec16 ? k_stats_rows<C, false, true> : k_stats_rows<C, false, false>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = a.units < 0x7FFFFFFF ? a.units : 0x7FFFFFFF;
  k<<<grid, kRowThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_stats_rows(const StatsArgs& a, size_t smem, cudaStream_t s) {
  const bool vec16 = (reinterpret_cast<uintptr_t>(a.img) & 15) == 0 && (a.pitch & 15) == 0 &&
                     (a.fstride & 15) == 0;
  if (a.g.C == 1) return launch_rows_c<1>(a, smem, vec16, s);
  if (a.g.C == 3) return launch_rows_c<3>(a, smem, vec16, s);
  return launch_rows_c<4>(a, smem, vec16, s);
}

template <int C>
cudaError_t launch_expand_rows_c(const ExpandArgs& a, size_t smem, cudaStream_t s) {
  auto k = a.adaptive ? k_expand_rows<C, true> : k_expand_rows<C, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t units = static_cast<int64_t>(a.g.F) * a.g.GR;
  const int grid = units < 0x7FFFFFFF ? static_cast<int>(units) : 0x7FFFFFFF;
  k<<<grid, kRowThreads, smem, s>>>(a, static_cast<int>(std::min<int64_t>(units, 0x7FFFFFFF)),
                                    make_fastdiv(static_cast<uint32_t>(a.g.GR)));
  return cudaGetLastError();
}

cudaError_t launch_expand_rows(const ExpandArgs& a, size_t smem, cudaStream_t s) {
  if (a.g.C == 1) return launch_expand_rows_c<1>(a, smem, s);
  if (a.g.C == 3) return launch_expand_rows_c<3>(a, smem, s);
  return launch_expand_rows_c<4>(a, smem, s);
}

cudaError_t launch_expand(const ExpandArgs& a, cudaStream_t s) {
  const int P = a.g.F * a.g.C;
  dim3 grid((a.g.GC + kGenericThreads - 1) / kGenericThreads, a.g.GR < 65535 ? a.g.GR : 65535,
            P < 65535 ? P : 65535);
  k_expand<<<grid, kGenericThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_synth(const BatchGeom& g, uint32_t seed, uint32_t f0, uint8_t* img,
                         int64_t pitch, int64_t fstride, uint8_t* mask, int64_t mpitch,
                         int64_t mfstride, cudaStream_t s) {
  k_synth<<<148 * 8, 256, 0, s>>>(g, seed, f0, img, pitch, fstride, mask, mpitch, mfstride);
  return cudaGetLastError();
}

cudaError_t launch_repitch(uint8_t* dst, int64_t dpitch, const uint8_t* src, int64_t spitch,
                           int64_t width, int64_t rows, cudaStream_t s) {
  const int64_t work = rows * ((width + 15) / 16);
  const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 148 * 16));
  k_repitch<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(dst, dpitch, src, spitch, width, rows);
  return cudaGetLastError();
}

cudaError_t launch_debug_lg2(unsigned int* out, cudaStream_t s) {
  k_debug_lg2<<<148 * 4, 256, 0, s>>>(out);
  return cudaGetLastError();
}

cudaError_t launch_debug_laplace(uint64_t mixed, const uint32_t* keys, int count, double sigma,
                                 double* out, cudaStream_t s) {
  k_debug_laplace<<<(count + 127) / 128, 128, 0, s>>>(mixed, keys, count, sigma, out);
  return cudaGetLastError();
}

}  // namespace dppx
