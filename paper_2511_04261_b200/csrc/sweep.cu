// sweep.cu -- K1s: one HBM read of the frames for every run of a uniform
// grid-size / epsilon sweep (the reference's run_sweep, cli.cpp:231-288, and
// b in {4, 8, 16, 32} x eps in {0.1, 0.5, 1} on
// 1917 x 1083 frames).
//
// The reference computes each (b, eps) run from scratch (pixelize_parallel,
// pixelize.cpp:86-124). Mirror reflection is b-independent (image.cpp:105-110:
// padded index len + k reads len - 1 - k), so 4-px cell sums taken over the
// LARGEST padded extent aggregate exactly (integer adds) to every larger
// power-of-two grid side, and for one plane seed and one cell the keyed bits
// -- hence u and -log1p(-2|u|) -- do not depend on eps (noise.cpp:86-117):
// only sigma = 255 m / (b^2 eps) scales them. Two kernels:
//  * K1s-sum: streams each frame once (TMA-staged BMAX-row bands, 512-px
//    tiles, dp4a strip sums), aggregates 2x2 per level in registers and writes
//    every level's cell sums (u16 / u32, ~17 % of the frame's bytes);
//  * K1s-draw: a flat, high-occupancy pass over the statistics. A thread takes
//    4 consecutive cells of one plane row, computes their keyed bits and
//    Laplace magnitude once, quantizes them for every eps and stores 4 bytes
//    per run at once. Statistics whose f32 estimate sits within the proven
//    error margin of a rounding boundary go to a per-warp queue that the warp
//    drains 32 at a time with the reference's exact f64 arithmetic
//    (exact_quantize), so the f64 path never diverges a warp.
// Statistics only: the runs' images are broadcast_means of these statistics
// (K2, issued by the host entry point).
#include "tma_kernels.cuh"

namespace dppx {

constexpr int kSweepMaxLevels = 4;  // b = 4, 8, 16, 32
constexpr int kSweepMaxEps = 4;

struct SweepLevels {
  int nlev;          // levels k = 0 .. nlev-1 have grid side 4 << k (BMAX = 4 << (nlev-1))
  int ne;            // eps runs per level
  uint32_t active;   // levels with outputs (bit k)
  int GR[kSweepMaxLevels], GC[kSweepMaxLevels];
  int64_t G[kSweepMaxLevels];
  double area[kSweepMaxLevels];
  double sigma[kSweepMaxLevels][kSweepMaxEps];
  float sln2[kSweepMaxLevels][kSweepMaxEps];  // f32(sigma * ln 2)
  float margin[kSweepMaxLevels][kSweepMaxEps];
  uint8_t* means[kSweepMaxLevels][kSweepMaxEps];  // run (k, j): F*C planes of G[k] bytes
  // level sums written by K1s-sum: plane p, cell (r, c) of level k at
  // sums[k] + (p * srows[k] + r) * scols[k] + c (u16; level 3: u32)
  void* sums[kSweepMaxLevels];
  int srows[kSweepMaxLevels], scols[kSweepMaxLevels];
  // K1s-draw work items: 4 consecutive cells of one (plane, row) of level k
  // (planes x GR[k] rows x groups[k]); items [item0[k], item0[k+1]) are level k's
  int64_t item0[kSweepMaxLevels + 1];
  int64_t item_begin, item_end;      // this launch's items (one or more levels)
  int groups[kSweepMaxLevels];       // ceil(GC[k] / 4)
  FastDiv div_groups[kSweepMaxLevels], div_rows[kSweepMaxLevels];  // by groups[k], by GR[k]
  int planes;
};

// ============================================================================
// K1s-sum
// ============================================================================
template <int C, int NLEV>
__global__ void __launch_bounds__(kStatsThreads, 3)
    k_sweep_sums(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ StatsArgs a,
                 const __grid_constant__ SweepLevels L) {
  constexpr int BMAX = 4 << (NLEV - 1);
  constexpr int TILE = kTilePx;        // 512 px: a multiple of every grid side
  constexpr int ROWB = TILE * C;
  constexpr uint32_t STAGE = BMAX * ROWB;
  constexpr int Q = BMAX / 4;          // 4-px cell rows per band
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t id_bar[kMaxStages];
  __shared__ __align__(8) uint64_t done_bar[kMaxStages];
  __shared__ int stage_unit[kMaxStages];

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
    // ---------------- producer: unit claims + TMA loads ----------------
    if (lane == 0) {
      prefetch_tmap(&tm_in);
      for (int k = 0;; ++k) {
        const int s = ring_slot(k, S);
        if (k >= S) mbar_wait(&done_bar[s], (ring_lap(k, S) - 1) & 1);
        int u = atomicAdd(a.work_counter, 1);
        if (u >= a.units) {
          if (u == a.units + static_cast<int>(gridDim.x) - 1) atomicExch(a.work_counter, 0);
          u = -1;
        }
        stage_unit[s] = u;
        mbar_arrive(&id_bar[s]);
        if (u < 0) {
          mbar_arrive_expect_tx(&full_bar[s], 0);
          break;
        }
        load_unit<C, BMAX, false, TILE>(a, &tm_in, u, smem + s * STAGE, &full_bar[s]);
      }
    }
    return;
  }

  // ---------------- consumers: one 4-px strip each ----------------
  const int t = threadIdx.x;
  const BatchGeom& g = a.g;  // geometry of the BMAX grid (bands, tiles, padding)
  for (int k = 0;; ++k) {
    const int s = ring_slot(k, S);
    mbar_wait(&id_bar[s], ring_lap(k, S) & 1);
    const int u = *reinterpret_cast<volatile int*>(&stage_unit[s]);
    if (u < 0) break;
    const UnitPos p = decode_unit<false, TILE>(a, u);
    const int f = p.fg;
    uint8_t* st = smem + s * STAGE;
    const int vbytes = valid_bytes<C, false, TILE>(a, p.px0);
    const int copy = staged_bytes<C, BMAX, false, TILE>(a, p);
    const int need = min(TILE, g.GC * BMAX - p.px0) * C;
    mbar_wait(&full_bar[s], ring_lap(k, S) & 1);
    // Mirrored padding columns / unstaged row tail (image.cpp:105-110), as K1.
    const int fs = min(copy, vbytes);
    if (fs < need) {
      constexpr int kLanes = 4;
      for (int pr = t / kLanes; pr < BMAX; pr += kConsumers / kLanes) {
        uint8_t* rowp = st + pr * ROWB;
        const int srow = reflect_index(p.r * BMAX + pr, g.M);
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
    // 4-px cell sums of this strip (exact u32, dp4a), then the stage is free.
    uint32_t acc[Q][C];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
#pragma unroll
      for (int ch = 0; ch < C; ++ch) acc[q][ch] = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) accumulate_row<C>(st + (4 * q + i) * ROWB + 4 * t * C, acc[q]);
    }
    mbar_arrive(&done_bar[s]);
    // Level sums: 2x2 aggregation per level (vertical in registers, horizontal
    // across lanes) -- exact integers. Stores of a (plane, row) are contiguous
    // across the owner lanes.
    const int tile_cells = p.px0 / 4;  // first 4-px cell column of the tile
    const int64_t P = static_cast<int64_t>(f) * C;
    auto put16 = [&](int lv, int r, int c, int ch, uint32_t v) {
      if (c < L.scols[lv])
        static_cast<uint16_t*>(L.sums[lv])[((P + ch) * L.srows[lv] + r) * L.scols[lv] + c] =
            static_cast<uint16_t>(v);
    };
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int ch = 0; ch < C; ++ch) put16(0, p.r * Q + q, tile_cells + t, ch, acc[q][ch]);
    if constexpr (NLEV > 1) {
      uint32_t v8[Q / 2][C];
#pragma unroll
      for (int q = 0; q < Q / 2; ++q)
#pragma unroll
        for (int ch = 0; ch < C; ++ch) {
          v8[q][ch] = acc[2 * q][ch] + acc[2 * q + 1][ch];
          v8[q][ch] += __shfl_xor_sync(0xFFFFFFFFu, v8[q][ch], 1);
        }
      if ((t & 1) == 0)
#pragma unroll
        for (int q = 0; q < Q / 2; ++q)
#pragma unroll
          for (int ch = 0; ch < C; ++ch) put16(1, p.r * (Q / 2) + q, tile_cells / 2 + (t >> 1), ch, v8[q][ch]);
      if constexpr (NLEV > 2) {
        uint32_t v16[Q / 4 > 0 ? Q / 4 : 1][C];
#pragma unroll
        for (int q = 0; q < Q / 4; ++q)
#pragma unroll
          for (int ch = 0; ch < C; ++ch) {
            v16[q][ch] = v8[2 * q][ch] + v8[2 * q + 1][ch];
            v16[q][ch] += __shfl_xor_sync(0xFFFFFFFFu, v16[q][ch], 2);
          }
        if ((t & 3) == 0)
#pragma unroll
          for (int q = 0; q < Q / 4; ++q)
#pragma unroll
            for (int ch = 0; ch < C; ++ch)
              put16(2, p.r * (Q / 4) + q, tile_cells / 4 + (t >> 2), ch, v16[q][ch]);
        if constexpr (NLEV > 3) {
          uint32_t v32[C];
#pragma unroll
          for (int ch = 0; ch < C; ++ch) {
            v32[ch] = v16[0][ch] + v16[1][ch];
            v32[ch] += __shfl_xor_sync(0xFFFFFFFFu, v32[ch], 4);
          }
          const int c32 = tile_cells / 8 + (t >> 3);
          if ((t & 7) == 0 && c32 < L.scols[3])
#pragma unroll
            for (int ch = 0; ch < C; ++ch)
              static_cast<uint32_t*>(L.sums[3])[((P + ch) * L.srows[3] + p.r) * L.scols[3] + c32] = v32[ch];
        }
      }
    }
  }
}

// ============================================================================
// K1s-draw
// ============================================================================
constexpr int kDrawThreads = 256;
constexpr int kDrawWarps = kDrawThreads / 32;
constexpr int kDrawQueue = 64;  // per warp; drained 32 at a time

struct ExactJob {
  uint64_t bits;
  uint8_t* dst;
  uint32_t sum;
  uint16_t lv, j;
};

// Signed f32 Laplace magnitude of 64 keyed bits in log2 units,
// +-(-log2(1 - 2|u|)) (the noise is this times sigma * ln 2; see fast_quantize,
// dppx_device.cuh, for the arithmetic and its error budget).
__device__ __forceinline__ float laplace_log2_signed(uint64_t bits) {
  const uint64_t y = bits >> 11;
  uint32_t lo_w, hi_w;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo_w), "=r"(hi_w) : "l"(bits));
  (void)lo_w;
  const bool neg = static_cast<int32_t>(hi_w) >= 0;
  const uint64_t W = neg ? y : (1ull << 53) - y;
  const uint32_t wb = __float_as_uint(fmaxf(__ull2float_rn(W), 1.0f));
  const int e = static_cast<int>(wb >> 23) - 127;
  const float lg_m = lg2_approx(__uint_as_float(0x3F800000u | (wb & 0x7FFFFFu)));
  const float L2 = static_cast<float>(52 - e) - lg_m;
  return neg ? -L2 : L2;
}

template <int NE, int KIND>
__global__ void __launch_bounds__(kDrawThreads)
    k_sweep_draw(const __grid_constant__ StatsArgs a, const __grid_constant__ SweepLevels L) {
  __shared__ ExactJob queue[kDrawWarps][kDrawQueue];
  __shared__ int qn[kDrawWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) qn[w] = 0;
  __syncwarp();
  constexpr int kind = KIND;  // noise kind: no per-statistic branches
  const bool exact_only = a.exact_noise != 0;
  const int ne = NE > 0 ? NE : L.ne;
  // Drain the top `cnt` queued statistics (one per lane) with the exact arithmetic.
  auto drain = [&](int cnt) {
    __syncwarp();
    const int base = qn[w] - cnt;
    if (lane < cnt) {
      const ExactJob e = queue[w][base + lane];
      *e.dst = static_cast<uint8_t>(exact_quantize(e.sum, L.area[e.lv], kind, e.bits, L.sigma[e.lv][e.j], 0.0));
    }
    __syncwarp();
    if (lane == 0) qn[w] = base;
    __syncwarp();
  };
  const int64_t total = L.item_end - L.item_begin;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kDrawThreads;
  // Every warp runs the same number of passes (the queue drains are warp-collective).
  const int64_t passes = (total + stride - 1) / stride;
  for (int64_t pass = 0; pass < passes; ++pass) {
    const int64_t rel_item = pass * stride + static_cast<int64_t>(blockIdx.x) * kDrawThreads + threadIdx.x;
    const int64_t item = L.item_begin + rel_item;
    bool any = rel_item < total;
    int lv = 0;
    if (any) {
#pragma unroll
      for (int k = 1; k < kSweepMaxLevels; ++k)
        if (k < L.nlev && item >= L.item0[k]) lv = k;
      any = (L.active >> lv) & 1u;
    }
    uint32_t sum[4] = {0, 0, 0, 0};
    uint64_t bits[4] = {0, 0, 0, 0};
    int nvalid = 0;
    int64_t off = 0;
    if (any) {
      const uint32_t rel = static_cast<uint32_t>(item - L.item0[lv]);
      const uint32_t prow = L.div_groups[lv].div(rel);         // plane * rows + row
      const int grp = static_cast<int>(rel - prow * static_cast<uint32_t>(L.groups[lv]));
      const uint32_t plane = L.div_rows[lv].div(prow);
      const int GRk = L.GR[lv], GCk = L.GC[lv];
      const int r = static_cast<int>(prow - plane * static_cast<uint32_t>(GRk));
      const int c0 = 4 * grp;
      nvalid = max(0, min(4, GCk - c0));
      const int f = static_cast<int>(plane / static_cast<uint32_t>(a.g.C));
      const int ch = static_cast<int>(plane) - f * a.g.C;
      const int64_t srow = (static_cast<int64_t>(plane) * L.srows[lv] + r) * L.scols[lv] + c0;
      if (lv < 3) {
        const uint16_t* s16 = static_cast<const uint16_t*>(L.sums[lv]) + srow;
#pragma unroll
        for (int v = 0; v < 4; ++v) sum[v] = v < nvalid ? __ldg(s16 + v) : 0u;
      } else {
        const uint32_t* s32 = static_cast<const uint32_t*>(L.sums[3]) + srow;
#pragma unroll
        for (int v = 0; v < 4; ++v) sum[v] = v < nvalid ? __ldg(s32 + v) : 0u;
      }
      if (kind == DPPX_NOISE_KEYED) {
        const uint64_t seed = a.noise.seed(plane);
#pragma unroll
        for (int v = 0; v < 4; ++v) bits[v] = key_sub(key_cell(seed, r, c0 + v), 0, 0);  // key (r, c, 0, 0)
      } else if (kind == DPPX_NOISE_PHILOX) {
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (v < nvalid) bits[v] = philox_call(a.noise.seed(0), a.noise.frame_base + f, ch, r, c0 + v, 0, 0);
      }
      off = static_cast<int64_t>(plane) * L.G[lv] + static_cast<int64_t>(r) * GCk + c0;
    }
    // quantize every cell for every eps; 4 bytes per run at once when aligned.
    // The mean + 0.5 and the signed log2 magnitude do not depend on eps: one
    // FFMA per (cell, eps) remains (the same arithmetic as fast_quantize).
    float Ls[4], m5[4];
    const float inv_area = any ? 1.0f / static_cast<float>(L.area[lv]) : 0.0f;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      m5[v] = fmaf(static_cast<float>(sum[v]), inv_area, 0.5f);
      Ls[v] = kind == DPPX_NOISE_NONE ? 0.0f : laplace_log2_signed(bits[v]);
    }
#pragma unroll
    for (int j = 0; j < ne; ++j) {
      uint32_t amb = 0;  // cells whose estimate is ambiguous
      if (any && nvalid > 0) {
        const float sl = L.sln2[lv][j], mg = L.margin[lv][j];
        uint32_t word = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint32_t q;
          const float t = kind == DPPX_NOISE_NONE ? m5[v] : fmaf(Ls[v], sl, m5[v]);
          if (kind == DPPX_NOISE_NONE) {
            q = static_cast<uint32_t>(floorf(t));  // area = 16^k: exact in f32
          } else {
            q = fast_finish(t, mg);
            if (exact_only || q == 0xFFFFFFFFu) amb |= 1u << v;
            q &= 0xFFu;  // (an ambiguous byte is overwritten when the queue drains)
          }
          word |= q << (8 * v);
        }
        uint8_t* dst = L.means[lv][j] + off;
        if (nvalid == 4 && (reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
          *reinterpret_cast<uint32_t*>(dst) = word;
        } else {
          for (int v = 0; v < nvalid; ++v) dst[v] = static_cast<uint8_t>(word >> (8 * v));
        }
        amb &= (1u << nvalid) - 1u;
      }
      // queue the ambiguous ones (their stored byte is overwritten when drained);
      // cell index v is static in every step, so nothing spills to local memory
      if (__any_sync(0xFFFFFFFFu, amb != 0)) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const bool mine = (amb >> v) & 1u;
          const unsigned want = __ballot_sync(0xFFFFFFFFu, mine);
          if (!want) continue;
          if (qn[w] > kDrawQueue - 32) drain(32);
          const int base = qn[w];
          if (mine)
            queue[w][base + __popc(want & ((1u << lane) - 1u))] =
                ExactJob{bits[v], L.means[lv][j] + off + v, sum[v], static_cast<uint16_t>(lv),
                         static_cast<uint16_t>(j)};
          __syncwarp();
          if (lane == 0) qn[w] = base + __popc(want);
          __syncwarp();
        }
      }
    }
    if (qn[w] >= 32) drain(32);
  }
  __syncwarp();
  if (qn[w] > 0) drain(qn[w]);
}

using SweepSumsKernel = void (*)(const CUtensorMap, const StatsArgs, const SweepLevels);
using SweepDrawKernel = void (*)(const StatsArgs, const SweepLevels);

SweepSumsKernel select_sweep_kernel(int C, int nlev) {
#define DPPX_SWEEP(Cv, NL) \
  if (C == (Cv) && nlev == (NL)) return k_sweep_sums<Cv, NL>;
  DPPX_SWEEP(1, 2)
  DPPX_SWEEP(1, 3)
  DPPX_SWEEP(1, 4)
  DPPX_SWEEP(3, 2)
  DPPX_SWEEP(3, 3)
  DPPX_SWEEP(3, 4)
#undef DPPX_SWEEP
  return nullptr;
}

cudaError_t launch_sweep_sums(SweepSumsKernel k, const CUtensorMap& tin, const StatsArgs& a,
                              const SweepLevels& L, int grid, size_t smem, cudaStream_t s) {
  k<<<grid, kStatsThreads, smem, s>>>(tin, a, L);
  return cudaGetLastError();
}

// Draws of items [L.item_begin, L.item_end) (one or more levels).
cudaError_t launch_sweep_draw(const StatsArgs& a, const SweepLevels& L, int max_grid, cudaStream_t s) {
  const int64_t items = L.item_end - L.item_begin;
  if (items <= 0) return cudaSuccess;
  const int draw_grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((items + kDrawThreads - 1) / kDrawThreads, max_grid)));
  const int kind = a.noise.kind;
  SweepDrawKernel d;
  if (kind == DPPX_NOISE_KEYED)
    d = L.ne == 3 ? k_sweep_draw<3, DPPX_NOISE_KEYED> : k_sweep_draw<0, DPPX_NOISE_KEYED>;
  else if (kind == DPPX_NOISE_PHILOX)
    d = L.ne == 3 ? k_sweep_draw<3, DPPX_NOISE_PHILOX> : k_sweep_draw<0, DPPX_NOISE_PHILOX>;
  else
    d = k_sweep_draw<0, DPPX_NOISE_NONE>;
  d<<<draw_grid, kDrawThreads, 0, s>>>(a, L);
  return cudaGetLastError();
}

int sweep_draw_threads() { return kDrawThreads; }

}  // namespace dppx

