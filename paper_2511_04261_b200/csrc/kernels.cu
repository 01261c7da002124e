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
//                      (K1 and its staged K2 k_expand_tma live in
//                      tma_kernels.cuh, instantiated in tma_c1.cu / tma_c3.cu.)
//  K1r k_stats_rows    row-streaming statistics for the other grid sides.
//  K1g k_stats_generic same semantics for any b, n, C and alignment
//  K1p k_stats_px      b = 1, 2 with b, n, C compile-time (K2p k_expand_px: reconstruction)
//                      (Algorithm 1, and shapes K1r cannot hold).
//  K2  k_expand        statistics -> pixels (broadcast_means / reassemble);
//                      K2r k_expand_rows for the K1r grid sides.
#include <cuda.h>  // CUtensorMap (type only; encoded on the host via the driver entry point)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include "dppx_device.cuh"
#include "dppx_params.h"
#include "stats_common.cuh"
#include "tma_kernels.cuh"

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
  if (b == 1) return __ldg(base + static_cast<int64_t>(r) * a.mpitch + c);  // grid = pixels
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
    if (fast) {
      // 8 rows' loads in flight per thread before any of them is summed
      for (int i0 = 0; i0 < g.b; i0 += 8) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[k] = make_uint4(0u, 0u, 0u, 0u);
          if (i0 + k < g.b)
            v[k] = __ldg(reinterpret_cast<const uint4*>(
                mbase + static_cast<int64_t>(reflect_index(r * g.b + i0 + k, g.M)) * a.mpitch + x0));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            lo[j] += w[j] & 0x00FF00FFu;
            hi[j] += (w[j] >> 8) & 0x00FF00FFu;
          }
        }
      }
    }
    for (int i = 0; i < (fast ? 0 : g.b); ++i) {
      const uint8_t* row = mbase + static_cast<int64_t>(reflect_index(r * g.b + i, g.M)) * a.mpitch;
      uint32_t w[4];
      {
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
  // A programmatic dependent (the zero-copy K1z) may start now: it waits for
  // this grid's results itself (griddepcontrol.wait); no-op for other launches.
  asm volatile("griddepcontrol.launch_dependents;");
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
          mean = __double2float_rn(a.inv_area_pow2 != 0.0  // b = 2^k: exact product, no DDIV
                                       ? static_cast<double>(s) * a.inv_area_pow2
                                       : __ddiv_rn(static_cast<double>(s), a.area));
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
          if (stored != S || (a.in_len && a.in_len[p] != len) || len > a.plen_limit) {
            atomicExch(a.status, DPPX_ERR_CORRUPT);
            s_last = 2u;  // plane p is corrupt: neutralise its slots below
          }
        } else {
          for (int ch = 0; ch < g.C; ++ch) {
            const int64_t q = (static_cast<int64_t>(p) * g.C + ch) * a.pstride + 4ll * g.G;
            *reinterpret_cast<uint32_t*>(a.payload + q) = S;
            if (a.payload_len) a.payload_len[static_cast<int64_t>(p) * g.C + ch] = len;
          }
        }
      }
      __syncthreads();
      if (s_last == 2u) {
        // Corrupt payload (reassemble throws RecordError, adaptive.cpp:192-210):
        // the expanders launched after this kernel must not follow its slot
        // offsets past the payload. Every cell becomes "simple, slot 0", which
        // reads byte 4G+4 (the host requires payload_stride >= 5G+4, the
        // shortest valid payload), and the plane's output is discarded.
        for (int64_t i = threadIdx.x; i < g.G; i += kClassifyThreads)
          a.cellinfo[static_cast<int64_t>(p) * g.G + i] = 1u;
        for (int i = threadIdx.x; i < g.GR; i += kClassifyThreads)
          a.rowprefix[static_cast<int64_t>(p) * g.GR + i] = 0u;
        if (threadIdx.x == 0) a.totals[p] = 0u;
      }
    }
    __syncthreads();
  }
}

// K0 for narrow frames (few cells per grid row, e.g. 178-px CelebA faces:
// 12 cells per row would leave 116 of k_classify's 128 threads idle, one CTA
// per row): one CTA per frame. Pass 1 (mode 0) sums the mask's b rows of
// every cell row column by column into smem (coalesced, one column per
// thread, 4 rows in flight, mirrored at the edges like image.cpp:105-110);
// pass 2 walks the frame's cells in row-major order in chunks of the block:
// mean (mode 0: mask_grid_mean -> f32; mode 1: the payload's stored mean),
// flag, and the frame-wide exclusive simple prefix; pass 3 derives the
// per-row prefixes, the intra-row prefixes (cell info), S and the payload
// lengths -- the same outputs as k_classify, without cross-CTA tickets.
__global__ void __launch_bounds__(kClassifyThreads) k_classify_frames(const ClassifyArgs a) {
  extern __shared__ __align__(16) uint8_t csm[];
  __shared__ uint32_t warp_tot[kClassifyThreads / 32];
  __shared__ uint32_t s_corrupt;
  const BatchGeom& g = a.g;
  const int t = threadIdx.x;
  const int PW = g.GC * g.b;
  const bool mode0 = a.from_payload == 0;
  uint32_t* gpre = reinterpret_cast<uint32_t*>(csm);                 // [G]: prefix | simple << 31
  uint16_t* colsum = reinterpret_cast<uint16_t*>(csm + 4ll * g.G);   // [GR][PW] (mode 0)
  for (int p = blockIdx.x; p < a.planes; p += gridDim.x) {
    if (mode0) {
      const uint8_t* mbase = a.mask + static_cast<int64_t>(p) * a.mfstride;
      for (int it = t; it < g.GR * PW; it += kClassifyThreads) {
        const int r = it / PW, x = it - r * PW;
        const uint8_t* col = mbase + reflect_index(x, g.N);
        const int y0 = r * g.b;
        uint32_t acc[4] = {0, 0, 0, 0};  // four rows in flight per step
        int i = 0;
        if (y0 + g.b <= g.M) {  // band inside the frame: no reflection
          const uint8_t* cp = col + static_cast<int64_t>(y0) * a.mpitch;
          for (; i + 4 <= g.b; i += 4)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] += __ldg(cp + static_cast<int64_t>(i + k) * a.mpitch);
        }
        for (; i < g.b; ++i) acc[0] += __ldg(col + static_cast<int64_t>(reflect_index(y0 + i, g.M)) * a.mpitch);
        colsum[it] = static_cast<uint16_t>(acc[0] + acc[1] + acc[2] + acc[3]);
      }
      __syncthreads();
    }
    const float* mm_in =
        a.from_payload == 1 ? reinterpret_cast<const float*>(a.payload_in + p * a.pstride) : nullptr;
    uint32_t carry = 0;
    for (int c0 = 0; c0 < g.G; c0 += kClassifyThreads) {
      const int cell = c0 + t;
      bool simple = false;
      if (cell < g.G) {
        float mean;
        if (mode0) {
          const int r = cell / g.GC, c = cell - r * g.GC;
          uint32_t sum = 0;
          const uint16_t* cs = colsum + r * PW + c * g.b;
          for (int k = 0; k < g.b; ++k) sum += cs[k];
          // mask_grid_mean (image.cpp:191-202) then static_cast<float> (adaptive.cpp:59-60)
          mean = __double2float_rn(a.inv_area_pow2 != 0.0  // b = 2^k: exact product, no DDIV
                                       ? static_cast<double>(sum) * a.inv_area_pow2
                                       : __ddiv_rn(static_cast<double>(sum), a.area));
          for (int ch = 0; ch < g.C; ++ch)
            reinterpret_cast<float*>(a.payload + (static_cast<int64_t>(p) * g.C + ch) * a.pstride)[cell] = mean;
        } else {
          mean = mm_in[cell];
        }
        simple = mean > 0.5f;  // simple_from_mean, adaptive.cpp:30-32
      }
      uint32_t tot;
      const uint32_t pre = block_scan_flags(simple, warp_tot, &tot);
      if (cell < g.G) gpre[cell] = (carry + pre) | (simple ? 0x80000000u : 0u);
      carry += tot;
    }
    __syncthreads();
    const uint32_t S = carry;
    const int64_t pg = static_cast<int64_t>(p) * g.G;
    for (int cell = t; cell < g.G; cell += kClassifyThreads) {
      const int r = cell / g.GC;
      const uint32_t rp = gpre[r * g.GC] & 0x7FFFFFFFu;
      const uint32_t v = gpre[cell];
      a.cellinfo[pg + cell] = (((v & 0x7FFFFFFFu) - rp) << 1) | (v >> 31);
    }
    for (int r = t; r < g.GR; r += kClassifyThreads) {
      const uint32_t rp = gpre[r * g.GC] & 0x7FFFFFFFu;
      const uint32_t next = r + 1 < g.GR ? (gpre[(r + 1) * g.GC] & 0x7FFFFFFFu) : S;
      a.rowprefix[static_cast<int64_t>(p) * g.GR + r] = rp;
      a.rowcnt[static_cast<int64_t>(p) * g.GR + r] = next - rp;
    }
    if (t == 0) {
      a.totals[p] = S;
      s_corrupt = 0u;
      const uint64_t nn = static_cast<uint64_t>(g.n) * g.n;
      const uint32_t len = static_cast<uint32_t>(4ull * g.G + 4 + S + (g.G - S) * nn);
      if (a.from_payload == 1) {
        const uint8_t* q = a.payload_in + p * a.pstride + 4ll * g.G;
        const uint32_t stored = static_cast<uint32_t>(q[0]) | (static_cast<uint32_t>(q[1]) << 8) |
                                (static_cast<uint32_t>(q[2]) << 16) | (static_cast<uint32_t>(q[3]) << 24);
        // decode's simple-count and length checks (record.cpp:253-270)
        if (stored != S || (a.in_len && a.in_len[p] != len) || len > a.plen_limit) {
          atomicExch(a.status, DPPX_ERR_CORRUPT);
          s_corrupt = 1u;
        }
      } else {
        for (int ch = 0; ch < g.C; ++ch) {
          const int64_t q = (static_cast<int64_t>(p) * g.C + ch) * a.pstride + 4ll * g.G;
          *reinterpret_cast<uint32_t*>(a.payload + q) = S;
          if (a.payload_len) a.payload_len[static_cast<int64_t>(p) * g.C + ch] = len;
        }
      }
    }
    __syncthreads();
    if (s_corrupt) {  // as k_classify: every cell "simple, slot 0", output discarded
      for (int i = t; i < g.G; i += kClassifyThreads) a.cellinfo[pg + i] = 1u;
      for (int i = t; i < g.GR; i += kClassifyThreads) a.rowprefix[static_cast<int64_t>(p) * g.GR + i] = 0u;
      if (t == 0) a.totals[p] = 0u;
    }
    __syncthreads();  // gpre / colsum reused by the next frame
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
        const uint32_t v = draw_stat(a, env, sum, cell_state(a, f, ch, r, c), f, ch, r, c, 0, 0, gidx);
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
          const uint32_t v = draw_stat(a, env, sum, cs, f, ch, r, c, sr, sc, gidx);
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

// K1p: grid sides b = 1, 2 (the paper's PPM grid starts at b = 1): one thread
// per cell as in K1g, but with b, n and C compile-time, so the pixel loops,
// reflections and subcell loops unroll to straight-line code and both draw
// environments are formed once per thread (K1g spent ~375 instructions per
// draw here, mostly loop control). Same statistics, slots and emitted pixels.
template <int C, int B, int NN>
__global__ void __launch_bounds__(kGenericThreads) k_stats_px(const StatsArgs a) {
  static_assert(B == 1 || B == 2, "K1p: b = 1, 2");
  static_assert(NN >= 1 && NN <= B, "K1p: n <= b");
  constexpr int SB = B / NN;  // complex subcell side
  const BatchGeom& g = a.g;
  const int c = blockIdx.x * kGenericThreads + threadIdx.x;
  if (c >= g.GC) return;
  const bool exact = a.exact_noise != 0;
  const DrawEnv env_s = make_env(a.noise.kind, exact, a.area, a.sigma);
  const DrawEnv env_c = make_env(a.noise.kind, exact, a.sub_area, a.sigma_sub);
  int jx[B];
  bool jin[B];
#pragma unroll
  for (int x = 0; x < B; ++x) {
    const int j = c * B + x;
    jx[x] = reflect_index(j, g.N) * C;
    jin[x] = j < g.N;
  }
  for (int r = a.row_begin + blockIdx.y; r < a.row_begin + a.row_count; r += gridDim.y)
  for (int f = blockIdx.z; f < g.F; f += gridDim.z) {
    const int gidx = r * g.GC + c;
    const uint8_t* img = a.img + static_cast<int64_t>(f) * a.fstride;
    bool simple = true;
    uint32_t slot_s = 0, S_tot = 0;
    if (a.adaptive) {
      const uint32_t info = __ldg(a.cellinfo + static_cast<int64_t>(f) * g.G + gidx);
      simple = info & 1u;
      slot_s = __ldg(a.rowprefix + static_cast<int64_t>(f) * g.GR + r) + (info >> 1);
      S_tot = __ldg(a.totals + f);
    }
    uint32_t px[B][B][C];
    int iy[B];
    bool iin[B];
#pragma unroll
    for (int y = 0; y < B; ++y) {
      const int i = r * B + y;
      iin[y] = i < g.M;
      iy[y] = reflect_index(i, g.M);
      const uint8_t* row = img + static_cast<int64_t>(iy[y]) * a.pitch;
#pragma unroll
      for (int x = 0; x < B; ++x)
#pragma unroll
        for (int ch = 0; ch < C; ++ch) px[y][x][ch] = __ldg(row + jx[x] + ch);
    }
    uint8_t* o = a.out ? a.out + static_cast<int64_t>(f) * a.ofstride : nullptr;
#pragma unroll
    for (int ch = 0; ch < C; ++ch) {
      const uint64_t cs = cell_state(a, f, ch, r, c);
      uint8_t* plane = a.stats + static_cast<int64_t>(f * C + ch) * a.sstride;
      if (simple || NN == 1) {
        uint32_t sum = 0;
#pragma unroll
        for (int y = 0; y < B; ++y)
#pragma unroll
          for (int x = 0; x < B; ++x) sum += px[y][x][ch];
        const uint32_t v = draw_stat(a, simple ? env_s : env_c, sum, cs, f, ch, r, c, 0, 0, gidx);
        plane[stat_offset(a, simple, gidx, slot_s, S_tot, 0, 0)] = static_cast<uint8_t>(v);
        if (o) {
#pragma unroll
          for (int y = 0; y < B; ++y)
#pragma unroll
            for (int x = 0; x < B; ++x)
              if (iin[y] && jin[x]) o[static_cast<int64_t>(r * B + y) * a.opitch + jx[x] + ch] = static_cast<uint8_t>(v);
        }
      } else {
#pragma unroll
        for (int sr = 0; sr < NN; ++sr)
#pragma unroll
          for (int sc = 0; sc < NN; ++sc) {
            uint32_t sum = 0;
#pragma unroll
            for (int y = sr * SB; y < sr * SB + SB; ++y)
#pragma unroll
              for (int x = sc * SB; x < sc * SB + SB; ++x) sum += px[y][x][ch];
            const uint32_t v = draw_stat(a, env_c, sum, cs, f, ch, r, c, sr, sc, gidx);
            plane[stat_offset(a, false, gidx, slot_s, S_tot, sr, sc)] = static_cast<uint8_t>(v);
            if (o) {
#pragma unroll
              for (int y = sr * SB; y < sr * SB + SB; ++y)
#pragma unroll
                for (int x = sc * SB; x < sc * SB + SB; ++x)
                  if (iin[y] && jin[x])
                    o[static_cast<int64_t>(r * B + y) * a.opitch + jx[x] + ch] = static_cast<uint8_t>(v);
            }
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
// K1r CTAs grow to 1024 threads when there are too few (frame, grid row) units
// to fill the GPU (large b on few frames: 8 x 4K at b = 128 is 136 units).
// (kRowThreadsMax, 1) caps registers at 64 like (256, 4) did.
constexpr int kRowThreadsMax = 1024;

struct RowSmem {  // byte offsets into dynamic smem (host and device agree)
  int vg;  // vertical subcells whose byte-column sums are held at once
  int sub_global;  // complex values too many for smem (large n): emit reads the payload
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
  L.sub_global = g.n * NS * g.C > 48 * 1024;
  L.pattern = L.subval + (L.sub_global ? rows_align16(4 * g.GC * g.C) : rows_align16(g.n * NS * g.C));
  L.cstate = L.pattern + rows_align16(g.N * g.C);
  L.total = L.cstate + 8 * g.GC * g.C;
  return L;
}

// Emits rows [r*b, min(r*b + b, M)) of frame f from the smem value tables:
// pixel x, channel ch of vertical subcell vs takes simpleval[c][ch] (simple
// cell c = x / b) or subval[vs][x / sb][ch]. One pattern row per vs.
// `sub(vs, sidx, c, ch)`: value of complex subcell column sidx (cell c) in
// vertical subcell vs, from the smem table or, at large n, the payload.
template <int C, bool ADAPTIVE, class SubFn>
__device__ void rows_emit(const BatchGeom& g, int r, uint8_t* out_frame, int64_t opitch,
                          const uint8_t* flag, const uint8_t* simpleval, const SubFn& sub,
                          uint8_t* pattern, const FastDiv& div_n, bool vec16) {
  const int t = threadIdx.x;
  const int RB = g.N * C, NS = g.GC * g.n;
  for (int vs = 0; vs < g.n; ++vs) {
    const int y0 = r * g.b + vs * g.sb;
    if (y0 >= g.M) break;
    const int y1 = min(y0 + g.sb, g.M);
    // pattern row: one thread per subcell column (sb pixels of C fixed values)
    for (int sidx = t; sidx < NS; sidx += static_cast<int>(blockDim.x)) {
      const int c = static_cast<int>(div_n.div(static_cast<uint32_t>(sidx)));
      uint8_t v[C];
#pragma unroll
      for (int ch = 0; ch < C; ++ch)
        v[ch] = (!ADAPTIVE || flag[c * C + ch]) ? simpleval[c * C + ch] : sub(vs, sidx, c, ch);
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
        for (int q = t; q < n16; q += static_cast<int>(blockDim.x))
          reinterpret_cast<uint4*>(orow)[q] = reinterpret_cast<const uint4*>(pattern)[q];
        for (int x = (n16 << 4) + t; x < RB; x += static_cast<int>(blockDim.x)) orow[x] = pattern[x];
      } else {
        for (int x = t; x < RB; x += static_cast<int>(blockDim.x)) orow[x] = pattern[x];
      }
    }
    __syncthreads();
  }
}

// CW: bytes per column chunk (16, or 8 when 16-byte chunks would leave the
// CTA's last pass mostly idle: 5775-byte padded rows = 361 chunks of 16 over
// 256 threads, the load phase then ends at a barrier half the block waits at).
template <int C, bool ADAPTIVE, bool VEC16, int CW, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_stats_rows(const StatsArgs a) {
  constexpr int NW = CW / 4;
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
      for (int c = t; c < g.GC; c += NT) {
        const uint32_t info = __ldg(&a.cellinfo[static_cast<int64_t>(f) * g.G + r * g.GC + c]);
#pragma unroll
        for (int ch = 0; ch < C; ++ch) flag[c * C + ch] = info & 1u;
        slot[c] = rowpre + (info >> 1);
      }
    }
    for (int e = t; e < g.GC * C; e += NT) {
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
      for (int x0 = t * CW; x0 < PB; x0 += NT * CW) {
        const uint8_t* colp = frame + x0;
        const bool fast = VEC16 && x0 + CW <= RB;
        for (int vg = 0; vg < nv; ++vg) {
          uint32_t lo[NW], hi[NW];
#pragma unroll
          for (int j = 0; j < NW; ++j) lo[j] = hi[j] = 0u;
          const int row0 = r * g.b + (v0 + vg) * g.sb;
#pragma unroll 4
          for (int i = 0; i < g.sb; ++i) {
            const int srow = reflect_index(row0 + i, g.M);
            const uint8_t* rowp = colp + static_cast<int64_t>(srow) * a.pitch;
            uint32_t w[NW];
            if (fast) {
              if constexpr (CW == 16) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(rowp));
                w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
              } else {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(rowp));
                w[0] = v.x, w[1] = v.y;
              }
            } else {
              const uint8_t* rowbase = rowp - x0;
#pragma unroll
              for (int j = 0; j < NW; ++j) {
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
            for (int j = 0; j < NW; ++j) {
              lo[j] += w[j] & 0x00FF00FFu;
              hi[j] += (w[j] >> 8) & 0x00FF00FFu;
            }
          }
          uint16_t* vrow = vsum + vg * PB;
#pragma unroll
          for (int j = 0; j < NW; ++j) {
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
      // (vi, rem) walked without a division: rem advances by NT and wraps
      const int nsc = NS * C;
      int vi = t / nsc, rem = t - vi * nsc;
      for (int item = t; item < nv * nsc; item += NT) {
        if (item != t) {
          rem += NT;
          while (rem >= nsc) rem -= nsc, ++vi;
        }
        const int vs = v0 + vi;
        const int sidx = rem / C, ch = rem - sidx * C;
        const int c = static_cast<int>(div_n.div(static_cast<uint32_t>(sidx))), sc = sidx - c * g.n;
        uint32_t sum = 0;
        const uint16_t* vp = vsum + vi * PB + sidx * g.sb * C + ch;
        if (g.sb == 1) {  // 1- and 2-px subcells (n = b, b / 2): no loop
          sum = vp[0];
        } else if (g.sb == 2) {
          sum = vp[0] + vp[C];
        } else {
          for (int k = 0; k < g.sb; ++k) sum += vp[k * C];
        }
        const int gidx = r * g.GC + c;
        if (!ADAPTIVE) {  // n == 1: the subcell is the cell
          const uint64_t cs = cstate[c * C + ch];
          const uint32_t v = draw_stat(a, env_cell, sum, cs, f, ch, r, c, 0, 0, gidx);
          a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + gidx] = static_cast<uint8_t>(v);
          simpleval[c * C + ch] = static_cast<uint8_t>(v);
        } else if (flag[c * C + ch]) {
          atomicAdd(&cellsum[c * C + ch], sum);
        } else {
          const uint64_t cs = cstate[c * C + ch];
          const uint32_t v = draw_stat(a, env_sub, sum, cs, f, ch, r, c, vs, sc, gidx);
          a.stats[static_cast<int64_t>(f * C + ch) * a.sstride +
                  stat_offset(a, false, gidx, slot[c], S_tot, vs, sc)] = static_cast<uint8_t>(v);
          if (!L.sub_global) subval[(vs * NS + sidx) * C + ch] = static_cast<uint8_t>(v);
        }
      }
      __syncthreads();
    }
    if (ADAPTIVE) {  // simple cells: one draw per channel at sigma
      for (int item = t; item < g.GC * C; item += NT) {
        const int c = item / C, ch = item - c * C;
        if (!flag[item]) continue;
        const int gidx = r * g.GC + c;
        const uint64_t cs = cstate[item];
        const uint32_t v = draw_stat(a, env_cell, cellsum[item], cs, f, ch, r, c, 0, 0, gidx);
        a.stats[static_cast<int64_t>(f * C + ch) * a.sstride +
                stat_offset(a, true, gidx, slot[c], S_tot, 0, 0)] = static_cast<uint8_t>(v);
        simpleval[item] = static_cast<uint8_t>(v);
      }
      __syncthreads();
    }
    if (a.out) {
      auto sub = [&](int vs, int sidx, int c, int ch) -> uint8_t {
        if (!L.sub_global) return subval[(vs * NS + sidx) * C + ch];
        const int gidx = r * g.GC + c;  // written above by this block (visible after the barrier)
        return a.stats[static_cast<int64_t>(f * C + ch) * a.sstride +
                       stat_offset(a, false, gidx, slot[c], S_tot, vs, sidx - c * g.n)];
      };
      rows_emit<C, ADAPTIVE>(g, r, a.out + static_cast<int64_t>(f) * a.ofstride, a.opitch, flag,
                             simpleval, sub, pattern, div_n, out_vec16);
    }
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
  int* cbase = reinterpret_cast<int*>(rsm + L.subval);  // sub_global: complex block offsets
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
        const int64_t cb = base + __ldg(&a.totals[plane]) +
                           static_cast<int64_t>(static_cast<uint32_t>(gidx) - slot_s) * nn;
        if (L.sub_global) {
          cbase[e] = static_cast<int>(cb);  // complex block of (cell, channel) in its plane
        } else {
          for (int k = 0; k < nn; ++k) {
            const int vs = k / g.n, sc = k - vs * g.n;
            subval[(vs * NS + c * g.n + sc) * C + ch] = __ldg(st + cb + k);
          }
        }
      }
    }
    __syncthreads();
    auto sub = [&](int vs, int sidx, int c, int ch) -> uint8_t {
      if (!L.sub_global) return subval[(vs * NS + sidx) * C + ch];
      const uint8_t* st = a.stats + (static_cast<int64_t>(f) * C + ch) * a.sstride;
      return __ldg(st + cbase[c * C + ch] + vs * g.n + (sidx - c * g.n));
    };
    rows_emit<C, ADAPTIVE>(g, r, a.out + static_cast<int64_t>(f) * a.ofstride, a.opitch, flag,
                           simpleval, sub, pattern, div_n, out_vec16);
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

// K2p: reconstruction for b = 1, 2 (K1p's counterpart): one thread per cell
// and all channels of a frame, b, n, C compile-time; per channel plane the
// cell's slot (K0 on the payload means) gives one simple value or the n x n
// complex values, written to the b x b pixels.
template <int C, int B, int NN>
__global__ void __launch_bounds__(kGenericThreads) k_expand_px(const ExpandArgs a) {
  constexpr int SB = B / NN;
  const BatchGeom& g = a.g;
  const int c = blockIdx.x * kGenericThreads + threadIdx.x;
  if (c >= g.GC) return;
  const int64_t base = 4ll * g.G + 4;
  for (int r = blockIdx.y; r < g.GR; r += gridDim.y)
  for (int f = blockIdx.z; f < g.F; f += gridDim.z) {
    const int gidx = r * g.GC + c;
    uint8_t v[C][B][B];
#pragma unroll
    for (int ch = 0; ch < C; ++ch) {
      const int64_t p = static_cast<int64_t>(f) * C + ch;
      const uint8_t* st = a.stats + p * a.sstride;
      if (!a.adaptive) {
        const uint8_t x = __ldg(st + gidx);
#pragma unroll
        for (int y = 0; y < B; ++y)
#pragma unroll
          for (int xx = 0; xx < B; ++xx) v[ch][y][xx] = x;
        continue;
      }
      const uint32_t info = __ldg(a.cellinfo + p * g.G + gidx);
      const uint32_t slot_s = __ldg(a.rowprefix + p * g.GR + r) + (info >> 1);
      if ((info & 1u) || NN == 1) {
        const uint8_t x = (info & 1u)
                              ? __ldg(st + base + slot_s)
                              : __ldg(st + base + __ldg(a.totals + p) + (static_cast<uint32_t>(gidx) - slot_s));
#pragma unroll
        for (int y = 0; y < B; ++y)
#pragma unroll
          for (int xx = 0; xx < B; ++xx) v[ch][y][xx] = x;
      } else {
        const uint8_t* sub = st + base + __ldg(a.totals + p) +
                             static_cast<int64_t>(static_cast<uint32_t>(gidx) - slot_s) * NN * NN;
#pragma unroll
        for (int y = 0; y < B; ++y)
#pragma unroll
          for (int xx = 0; xx < B; ++xx) v[ch][y][xx] = __ldg(sub + (y / SB) * NN + xx / SB);
      }
    }
    uint8_t* o = a.out + static_cast<int64_t>(f) * a.ofstride;
#pragma unroll
    for (int y = 0; y < B; ++y) {
      const int i = r * B + y;
      if (i >= g.M) break;
#pragma unroll
      for (int xx = 0; xx < B; ++xx) {
        const int j = c * B + xx;
        if (j >= g.N) break;
        uint8_t* q = o + static_cast<int64_t>(i) * a.opitch + static_cast<int64_t>(j) * C;
#pragma unroll
        for (int ch = 0; ch < C; ++ch) q[ch] = v[ch][y][xx];
      }
    }
  }
}

cudaError_t launch_expand_px(const ExpandArgs& a, cudaStream_t s) {
  void (*k)(const ExpandArgs) = nullptr;
  const int b = a.g.b, n = a.adaptive ? a.g.n : 1;
  if (a.g.C == 1) k = b == 1 ? k_expand_px<1, 1, 1> : n == 2 ? k_expand_px<1, 2, 2> : k_expand_px<1, 2, 1>;
  else if (a.g.C == 3) k = b == 1 ? k_expand_px<3, 1, 1> : n == 2 ? k_expand_px<3, 2, 2> : k_expand_px<3, 2, 1>;
  if (!k || b > 2) return cudaErrorNotSupported;
  const int rows = (a.g.GR + 3) / 4;  // 4 grid rows per thread
  dim3 grid((a.g.GC + kGenericThreads - 1) / kGenericThreads, rows < 65535 ? rows : 65535,
            a.g.F < 65535 ? a.g.F : 65535);
  k<<<grid, kGenericThreads, 0, s>>>(a);
  return cudaGetLastError();
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

// x / 49 for the integer window sums (x <= 49 * 255^2): RN(x * RN(1/49))
// corrected by one exact-remainder fma. Checked exhaustively against IEEE
// division for every x in [0, 3186225] (tools/div49_check.c), so the local
// SSIM below stays bit-identical to metrics.cpp's `/ area` without a DDIV.
__device__ __forceinline__ double div49(uint32_t x) {
  const double a = static_cast<double>(x), r = 1.0 / 49.0;
  const double q = __dmul_rn(a, r);
  return __fma_rn(__fma_rn(-q, 49.0, a), r, q);
}

// SSIM of one plane band: one CTA per (plane, SSR window rows), 7-row column
// sums and local SSIM values computed in parallel over 128-column chunks, then
// each window row's values folded left to right by one lane in the reference's
// order (metrics.cpp:144-177): the row partial is bit-identical.
//   warps 1..4: local SSIM of chunk c (thread = row r, 8 consecutive windows);
//   warp 0:     folds chunk c-1 meanwhile (lane r = window row r);
//   all:        7-row column sums of the next chunk.
constexpr int SSR = 8, SCW = 128, SVS = 152;  // rows per CTA, windows per chunk, V row stride
__device__ __forceinline__ int ssim_vx(int x) { return x + (x >> 3); }  // 16 lanes x 8 cols: no bank clash

__global__ void __launch_bounds__(160, 4) k_ssim_bands(const MetricArgs m) {
  constexpr int W = 7;
  __shared__ uint32_t V[5][SSR][SVS];
  __shared__ double Q[2][SSR][SCW + 1];
  const int pr = m.M - W + 1, pc = m.N - W + 1;
  const int nb = (pr + SSR - 1) / SSR;
  const int64_t p = blockIdx.x / nb;
  const int i0 = static_cast<int>(blockIdx.x - p * nb) * SSR;
  const int rows = min(SSR, pr - i0);
  const int f = static_cast<int>(p / m.C), ch = static_cast<int>(p - static_cast<int64_t>(f) * m.C);
  const uint8_t* a = m.a + static_cast<int64_t>(f) * m.fstride + static_cast<int64_t>(i0) * m.pitch + ch;
  const uint8_t* b = m.b + static_cast<int64_t>(f) * m.bfstride + static_cast<int64_t>(i0) * m.bpitch + ch;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int nchunk = (pc + SCW - 1) / SCW;
  double acc = 0.0;  // warp 0, lane r: window row i0 + r
  auto fold = [&](int c) {
    if (lane < rows) {
      const double* q = Q[c & 1][lane];
      const int n = min(SCW, pc - c * SCW);
      for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, q[k]);
    }
  };
  for (int c = 0; c < nchunk; ++c) {
    const int j0 = c * SCW;
    // ---- 7-row column sums of columns j0 .. j0+SCW+5 ----
    if (t < SCW + W - 1) {
      const int col = j0 + t;
      if (col < m.N) {
        const uint8_t* pa = a + static_cast<int64_t>(col) * m.C;
        const uint8_t* pb = b + static_cast<int64_t>(col) * m.C;
        uint32_t va[SSR + W - 1], vb[SSR + W - 1];
#pragma unroll
        for (int y = 0; y < SSR + W - 1; ++y) {
          va[y] = y < rows + W - 1 ? __ldg(pa + static_cast<int64_t>(y) * m.pitch) : 0u;
          vb[y] = y < rows + W - 1 ? __ldg(pb + static_cast<int64_t>(y) * m.bpitch) : 0u;
        }
        uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
#pragma unroll
        for (int y = 0; y < W; ++y) {
          s0 += va[y], s1 += vb[y], s2 += va[y] * va[y], s3 += vb[y] * vb[y], s4 += va[y] * vb[y];
        }
        const int x = ssim_vx(t);
#pragma unroll
        for (int r = 0; r < SSR; ++r) {
          if (r > 0) {
            const uint32_t oa = va[r - 1], ob = vb[r - 1], na = va[r + W - 1], nb2 = vb[r + W - 1];
            s0 += na - oa, s1 += nb2 - ob, s2 += na * na - oa * oa, s3 += nb2 * nb2 - ob * ob;
            s4 += na * nb2 - oa * ob;
          }
          V[0][r][x] = s0, V[1][r][x] = s1, V[2][r][x] = s2, V[3][r][x] = s3, V[4][r][x] = s4;
        }
      }
    }
    __syncthreads();
    if (warp == 0) {
      if (c > 0) fold(c - 1);
    } else {
      const int u = t - 32, r = u >> 4, g = u & 15;
      const int jl = g * 8;
      if (r < rows && j0 + jl < pc) {
        uint32_t win[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          uint32_t s = 0;
#pragma unroll
          for (int x = 0; x < W; ++x) s += V[q][r][ssim_vx(jl + x)];
          win[q] = s;
        }
        const double c1 = 6.5025, c2 = 58.5225;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k > 0) {
#pragma unroll
            for (int q = 0; q < 5; ++q)
              win[q] = win[q] - V[q][r][ssim_vx(jl + k - 1)] + V[q][r][ssim_vx(jl + k + W - 1)];
          }
          const double mu_a = div49(win[0]), mu_b = div49(win[1]);
          const double raw_aa = div49(win[2]), raw_bb = div49(win[3]), raw_ab = div49(win[4]);
          const double mu_aa = __dmul_rn(mu_a, mu_a), mu_bb = __dmul_rn(mu_b, mu_b),
                       mu_ab = __dmul_rn(mu_a, mu_b);
          const double var_a = __dsub_rn(raw_aa, mu_aa), var_b = __dsub_rn(raw_bb, mu_bb),
                       cov = __dsub_rn(raw_ab, mu_ab);
          const double num =
              __dmul_rn(__dadd_rn(__dmul_rn(2.0, mu_ab), c1), __dadd_rn(__dmul_rn(2.0, cov), c2));
          const double den = __dmul_rn(__dadd_rn(__dadd_rn(mu_aa, mu_bb), c1),
                                       __dadd_rn(__dadd_rn(var_a, var_b), c2));
          Q[c & 1][r][jl + k] = __ddiv_rn(num, den);  // windows past pc are never folded
        }
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
    fold(nchunk - 1);
    if (lane < rows) m.row_sums[p * pr + i0 + lane] = acc;
  }
}

cudaError_t launch_metrics(const MetricArgs& m, bool ssim, cudaStream_t s) {
  if (!ssim) {
    dim3 grid((m.M + 7) / 8, m.F < 65535 ? m.F : 65535);
    k_mse<<<grid, 256, 0, s>>>(m);
  } else {
    const int64_t ctas = static_cast<int64_t>(m.F) * m.C * ((m.M - 6 + SSR - 1) / SSR);
    if (ctas > 0x7fffffff) return cudaErrorInvalidConfiguration;
    k_ssim_bands<<<static_cast<unsigned>(ctas), 160, 0, s>>>(m);
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
    worst = fmaxf(worst, static_cast<float>(fabs(static_cast<double>(lg2_approx(m)) - exact)));
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
// Fused variance classification (wide frames only; else the 2-pass path).
StatsKernel select_stats_kernel_var(int C, int b, int n) {
  if (C == 1) return select_stats_var_c1(b, n);
  if (C == 3) return select_stats_var_c3(b, n);
  return nullptr;
}

cudaError_t launch_gather_stage(const GatherArgs& a, cudaStream_t s) {
  const int P = a.g.F * a.g.C;
  const int bx = std::min((a.g.G + kGenericThreads - 1) / kGenericThreads, 64);
  dim3 grid(bx > 0 ? bx : 1, P < 65535 ? P : 65535);
  k_gather_stage<<<grid, kGenericThreads, 0, s>>>(a);
  return cudaGetLastError();
}

StatsKernel select_uniform_b4_rows2_c1();
StatsKernel select_uniform_b4_rows2_c3();
StatsKernel select_uniform_b4_rows2(int C) {
  if (C == 1) return select_uniform_b4_rows2_c1();
  if (C == 3) return select_uniform_b4_rows2_c3();
  return nullptr;
}

StatsKernel select_stats_kernel(int C, int b, int n, bool adaptive, bool packed) {
  if (!adaptive && n != 1) return nullptr;
  if (adaptive && !packed && (b % 4 != 0 || b == 128)) {  // K1a (DPPX_NO_K1A: K1r, for A/B runs)
    static const bool off = std::getenv("DPPX_NO_K1A") != nullptr;
    if (off) return nullptr;
    if (C == 1) return select_adaptive_any_c1(b, n);
    if (C == 3) return select_adaptive_any_c3(b, n);
    return nullptr;
  }
  if (!adaptive && !packed && (b % 4 != 0 || b == 128)) {  // K1u: uniform, b % 4 != 0 or b = 128
    if (C == 1) return select_uniform_any_c1(b);
    if (C == 3) return select_uniform_any_c3(b);
    return nullptr;
  }
  if (C == 1) return select_stats_tma_c1(b, n, adaptive, packed);
  if (C == 3) return select_stats_tma_c3(b, n, adaptive, packed);
  return nullptr;
}

ExpandKernel select_expand_kernel(int C, int b, int n, bool adaptive, bool packed, int split) {
  if (!adaptive && n != 1) return nullptr;
  if (adaptive && !packed && (b % 4 != 0 || b == 128)) {  // K2a
    if (C == 1) return select_expand_aany_c1(b, n);
    if (C == 3) return select_expand_aany_c3(b, n);
    return nullptr;
  }
  if (!adaptive && !packed && (b % 4 != 0 || b == 128)) {  // K2u
    if (C == 1) return select_expand_uany_c1(b);
    if (C == 3) return select_expand_uany_c3(b);
    return nullptr;
  }
  if (C == 1) return select_expand_tma_c1(b, n, adaptive, packed, split);
  if (C == 3) return select_expand_tma_c3(b, n, adaptive, packed, split);
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
int stats_tile_px_for(int b, bool adaptive) {
  if ((b % 4 != 0 && b >= 2 && b <= 32) || b == 128) return adaptive ? ka_tile(b) : ku_tile(b);  // K1u / K1a
  const int b4 = b / 4;
  if (b % 4 != 0 || b4 < 1 || b4 > 32) return kTilePx;
  return 4 * (kConsumers / 32) * ((32 / b4) * b4);
}
int stats_max_stages() { return kMaxStages; }

cudaError_t launch_classify(const ClassifyArgs& a, cudaStream_t s) {
  // Narrow frames (a grid row at most half the block): one CTA per frame.
  // (DPPX_NO_K0_FRAMES: A/B knob)
  static const bool frames_off = std::getenv("DPPX_NO_K0_FRAMES") != nullptr;
  // ... and only when that gives enough CTAs or the frames are small: one CTA
  // per 1080p frame at b = 128 (GC = 15) left 120 CTAs on 148 SMs (1.37 ms;
  // the per-row kernel: GR CTAs per frame).
  const bool many = a.planes >= 2 * 148 ||
                    static_cast<int64_t>(a.g.M) * a.g.N <= (int64_t{1} << 16);
  if ((a.from_payload == 0 || a.from_payload == 1) && !a.mask_bits && a.g.GC * 2 <= kClassifyThreads &&
      many && !frames_off) {
    const size_t smem = 4 * static_cast<size_t>(a.g.G) +
                        (a.from_payload == 0 ? 2 * static_cast<size_t>(a.g.GR) * a.g.GC * a.g.b : 0);
    if (smem <= 48 * 1024 && a.g.b <= 257) {
      const int grid = a.planes < 148 * 16 ? a.planes : 148 * 16;
      k_classify_frames<<<grid > 0 ? grid : 1, kClassifyThreads, smem, s>>>(a);
      return cudaGetLastError();
    }
  }
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

// K1p for b = 1, 2 (C = 1, 3; not Algorithm 1's partial borders).
cudaError_t launch_stats_px(const StatsArgs& a, cudaStream_t s) {
  void (*k)(const StatsArgs) = nullptr;
  const int b = a.g.b, n = a.adaptive ? a.g.n : 1;
  if (a.g.C == 1) k = b == 1 ? k_stats_px<1, 1, 1> : n == 2 ? k_stats_px<1, 2, 2> : k_stats_px<1, 2, 1>;
  else if (a.g.C == 3) k = b == 1 ? k_stats_px<3, 1, 1> : n == 2 ? k_stats_px<3, 2, 2> : k_stats_px<3, 2, 1>;
  if (!k || b > 2 || a.partial_borders) return cudaErrorNotSupported;
  // several grid rows per thread (DPPX_K1P_ROWS, default 4): the per-thread
  // setup (two draw environments, column offsets) is paid once per 4 cells
  static const int rpt = [] {
    const char* e = std::getenv("DPPX_K1P_ROWS");
    const int v = e ? std::atoi(e) : 4;
    return v > 0 ? v : 4;
  }();
  const int rows = a.row_count > 0 ? (a.row_count + rpt - 1) / rpt : 1;
  dim3 grid((a.g.GC + kGenericThreads - 1) / kGenericThreads, rows < 65535 ? rows : 65535,
            a.g.F < 65535 ? a.g.F : 65535);
  k<<<grid, kGenericThreads, 0, s>>>(a);
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

template <int C, int CW>
cudaError_t launch_rows_cw(const StatsArgs& a, size_t smem, bool vec16, cudaStream_t s) {
  const int grid = a.units < 0x7FFFFFFF ? a.units : 0x7FFFFFFF;
  // few units: 1024-thread CTAs (DPPX_ROWS_THREADS=256 / 1024 forces one);
  // separate instantiations, so the 256-thread code keeps its (256, 4) bounds
  static const int forced = std::getenv("DPPX_ROWS_THREADS") ? std::atoi(std::getenv("DPPX_ROWS_THREADS")) : 0;
  const bool wide = forced ? forced == kRowThreadsMax : static_cast<int64_t>(grid) * kRowThreads < 148ll * 1024;
  using K = void (*)(const StatsArgs);
  K k;
  if (wide)
    k = a.adaptive ? (vec16 ? k_stats_rows<C, true, true, CW, kRowThreadsMax> : k_stats_rows<C, true, false, CW, kRowThreadsMax>)
                   : (vec16 ? k_stats_rows<C, false, true, CW, kRowThreadsMax> : k_stats_rows<C, false, false, CW, kRowThreadsMax>);
  else
    k = a.adaptive ? (vec16 ? k_stats_rows<C, true, true, CW, kRowThreads> : k_stats_rows<C, true, false, CW, kRowThreads>)
                   : (vec16 ? k_stats_rows<C, false, true, CW, kRowThreads> : k_stats_rows<C, false, false, CW, kRowThreads>);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, wide ? kRowThreadsMax : kRowThreads, smem, s>>>(a);
  return cudaGetLastError();
}

// Busy fraction of the CTA's column-chunk passes for chunk width cw.
inline double rows_chunk_balance(int pb, int cw) {
  const int chunks = (pb + cw - 1) / cw;
  const int passes = (chunks + kRowThreads - 1) / kRowThreads;
  return static_cast<double>(chunks) / (static_cast<double>(passes) * kRowThreads);
}

template <int C>
cudaError_t launch_rows_c(const StatsArgs& a, size_t smem, bool vec16, cudaStream_t s) {
  // Measured (tools/b_sweep.py uniform, 1080p RGB): 8-byte chunks win only when
  // the row has mirrored padding columns (b = 7, 9, 11, 13, 14, 17-19: 5-11 %
  // faster) and lose 10-14 % on unpadded rows (b = 6, 10, 15, 30, 128).
  const int pb = a.g.GC * a.g.b * C;
  if (pb != a.g.N * C && rows_chunk_balance(pb, 8) > rows_chunk_balance(pb, 16) + 0.15)
    return launch_rows_cw<C, 8>(a, smem, vec16, s);
  return launch_rows_cw<C, 16>(a, smem, vec16, s);
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

// Per-frame equality of two pitched frame batches (rows of `width` bytes):
// eq[f] is cleared when any byte of frame f differs (the batch runner's
// reconstruct check, cli.cpp:135-146, done where both images already live).
__global__ void k_frames_equal(const uint8_t* a, const uint8_t* b, int64_t pitch, int64_t fstride,
                               int64_t width, int rows, uint32_t* eq) {
  const int f = blockIdx.y;
  const int64_t w16 = width / 16;
  const int64_t work = static_cast<int64_t>(rows) * (w16 + 1);
  bool same = true;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < work;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / (w16 + 1), q = e - r * (w16 + 1);
    const uint8_t* pa = a + f * fstride + r * pitch;
    const uint8_t* pb = b + f * fstride + r * pitch;
    if (q < w16) {
      const uint4 x = reinterpret_cast<const uint4*>(pa)[q], y = reinterpret_cast<const uint4*>(pb)[q];
      same &= x.x == y.x && x.y == y.y && x.z == y.z && x.w == y.w;
    } else {
      for (int64_t k = w16 * 16; k < width; ++k) same &= pa[k] == pb[k];
    }
  }
  if (!__all_sync(0xFFFFFFFFu, same) && (threadIdx.x & 31) == 0) atomicAnd(&eq[f], 0u);
}

cudaError_t launch_frames_equal(const uint8_t* a, const uint8_t* b, int64_t pitch, int64_t fstride,
                                int64_t width, int rows, int frames, uint32_t* eq, cudaStream_t s) {
  if (frames <= 0) return cudaSuccess;
  const int64_t work = static_cast<int64_t>(rows) * (width / 16 + 1);
  const int bx = static_cast<int>(std::min<int64_t>((work + 255) / 256, 64));
  k_frames_equal<<<dim3(bx > 0 ? bx : 1, frames), 256, 0, s>>>(a, b, pitch, fstride, width, rows, eq);
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
