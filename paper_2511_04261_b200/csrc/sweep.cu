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
// only sigma = 255 m / (b^2 eps) scales them. So one unit of work (frame,
// BMAX-row band, 512-px column tile) is staged once by TMA, summed once, and
// every level's cells draw their bits and Laplace magnitude once and quantize
// once per eps, each with the reference's own f64 fallback for values near a
// rounding boundary (fast_quantize / exact_quantize, dppx_device.cuh).
// Statistics only: the reconstructed images of the runs are broadcast_means of
// these statistics (K2, written by the host entry point).
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
  float sigmaf[kSweepMaxLevels][kSweepMaxEps];
  float margin[kSweepMaxLevels][kSweepMaxEps];
  uint8_t* means[kSweepMaxLevels][kSweepMaxEps];  // run (k, j): F*C planes of G[k] bytes
};

// A statistic whose f32 estimate was ambiguous: evaluated with the exact f64
// arithmetic after the unit's draw pass, by all consumers together (in line,
// ~1 in 4 warps would diverge into the f64 path on every pass at b = 4,
// eps = 0.1, where sigma = 2550 widens the margin).
struct ExactJob {
  uint64_t bits;
  uint8_t* dst;
  uint32_t sum;
  uint16_t lv, j;
};
constexpr int kSweepQueue = 256;

// Per-eps quantization of one statistic whose noise magnitude is shared:
// bits -> (sign, L = -ln(1 - 2|u|) in f32), then q_j for every sigma_j with
// the exact reference arithmetic when the f32 estimate is ambiguous. Runs
// j0 .. j0 + NE - 1 of level k.
template <int NE>
__device__ __forceinline__ void sweep_quantize(const SweepLevels& L, int k, int j0, uint32_t sum,
                                               uint64_t bits, int kind, bool exact_only, int64_t off,
                                               ExactJob* queue, int* qn) {
  const double area = L.area[k];
  const float inv_area = 1.0f / static_cast<float>(area);
  if (kind == DPPX_NOISE_NONE) {
    // area = 16^k is a power of two: sum * 2^-m + 0.5 is exact in f32
    const uint8_t q = static_cast<uint8_t>(floorf(static_cast<float>(sum) * inv_area + 0.5f));
#pragma unroll
    for (int j = 0; j < NE; ++j) L.means[k][j0 + j][off] = q;
    return;
  }
  const uint64_t y = bits >> 11;
  const bool neg = static_cast<int32_t>(bits >> 32) >= 0;
  const uint64_t W = neg ? y : (1ull << 53) - y;
  const uint32_t wb = __float_as_uint(fmaxf(__ull2float_rn(W), 1.0f));
  const int e = static_cast<int>(wb >> 23) - 127;
  const float lg_m = lg2_approx(__uint_as_float(0x3F800000u | (wb & 0x7FFFFFu)));
  const float Lf = (static_cast<float>(52 - e) - lg_m) * 0.693147180559945f;
  const float mean_f = static_cast<float>(sum) * inv_area + 0.5f;
#pragma unroll
  for (int j = 0; j < NE; ++j) {
    uint32_t q = 0xFFFFFFFFu;
    if (!exact_only) {
      const float sf = L.sigmaf[k][j0 + j];
      const float t = mean_f + (neg ? -sf * Lf : sf * Lf);
      const float jr = rintf(t);
      if (!(fabsf(t - jr) <= L.margin[k][j0 + j] && jr >= 1.0f && jr <= 255.0f))
        q = static_cast<uint32_t>(min(max(__float2int_rd(t), 0), 255));
    }
    if (q == 0xFFFFFFFFu) {
      const int slot = atomicAdd(qn, 1);
      if (slot < kSweepQueue) {
        queue[slot] = ExactJob{bits, L.means[k][j0 + j] + off, sum, static_cast<uint16_t>(k),
                               static_cast<uint16_t>(j0 + j)};
        continue;
      }
      q = exact_quantize(sum, area, kind, bits, L.sigma[k][j0 + j], 0.0);  // queue full
    }
    L.means[k][j0 + j][off] = static_cast<uint8_t>(q);
  }
}

template <int C, int NLEV>
__global__ void __launch_bounds__(kStatsThreads, 3)
    k_sweep_stats(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ StatsArgs a,
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
  // Level sums of the unit's cells, [level][cell row][cell col][channel]
  // (4-px level: every strip; b = 8 << k: owner lanes). u16 holds up to 257 * 255.
  __shared__ uint16_t t4[Q][kConsumers][C];
  __shared__ uint16_t t8[NLEV > 1 ? Q / 2 : 1][kConsumers / 2][C];
  __shared__ uint16_t t16[NLEV > 2 ? Q / 4 : 1][kConsumers / 4][C];
  __shared__ uint32_t t32[NLEV > 3 ? 1 : 1][kConsumers / 8][C];
  __shared__ ExactJob queue[kSweepQueue];
  __shared__ int qn;

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
    // ---------------- producer: unit claims + TMA loads (no stores) ----------------
    if (lane == 0) {
      prefetch_tmap(&tm_in);
      for (int k = 0;; ++k) {
        const int s = k % S;
        if (k >= S) mbar_wait(&done_bar[s], ((k / S) - 1) & 1);
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
  const bool keyed = a.noise.kind == DPPX_NOISE_KEYED;
  const bool exact_only = a.exact_noise != 0;
  if (t == 0) qn = 0;
  named_bar_sync(1, kConsumers);
  for (int k = 0;; ++k) {
    const int s = k % S;
    mbar_wait(&id_bar[s], (k / S) & 1);
    const int u = *reinterpret_cast<volatile int*>(&stage_unit[s]);
    if (u < 0) break;
    const UnitPos p = decode_unit<false, TILE>(a, u);
    const int f = p.fg;
    uint8_t* st = smem + s * STAGE;
    const int vbytes = valid_bytes<C, false, TILE>(a, p.px0);
    const int copy = staged_bytes<C, BMAX, false, TILE>(a, p);
    const int need = min(TILE, g.GC * BMAX - p.px0) * C;
    mbar_wait(&full_bar[s], (k / S) & 1);
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
    // Larger grid sides: 2x2 aggregation per level (vertical in registers,
    // horizontal across lanes) -- exact integers, b-independent reflection.
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int ch = 0; ch < C; ++ch) t4[q][t][ch] = static_cast<uint16_t>(acc[q][ch]);
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
          for (int ch = 0; ch < C; ++ch) t8[q][t >> 1][ch] = static_cast<uint16_t>(v8[q][ch]);
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
            for (int ch = 0; ch < C; ++ch) t16[q][t >> 2][ch] = static_cast<uint16_t>(v16[q][ch]);
        if constexpr (NLEV > 3) {
          uint32_t v32[C];
#pragma unroll
          for (int ch = 0; ch < C; ++ch) {
            v32[ch] = v16[0][ch] + v16[1][ch];
            v32[ch] += __shfl_xor_sync(0xFFFFFFFFu, v32[ch], 4);
          }
          if ((t & 7) == 0)
#pragma unroll
            for (int ch = 0; ch < C; ++ch) t32[0][t >> 3][ch] = v32[ch];
        }
      }
    }
    named_bar_sync(1, kConsumers);
    // Draws: every statistic of every active level, dealt round-robin to the
    // 128 consumers; within a level, consecutive threads take consecutive
    // cells of one plane row (coalesced byte stores into every eps run). Each
    // thread takes U statistics per pass and computes their keyed bits first:
    // U independent mix64 chains the scheduler interleaves.
    constexpr int U = 4;
#pragma unroll 1
    for (int lv = 0; lv < NLEV; ++lv) {
      if (!((L.active >> lv) & 1u)) continue;
      const int lgc = 7 - lv;  // log2(cells per tile row) = log2(512 / (4 << lv))
      const int rows = Q >> lv;
      const int count = (rows * C) << lgc;
      const int r0 = p.r * rows, c0 = p.px0 >> (2 + lv);
      const int GRk = L.GR[lv], GCk = L.GC[lv];
      const int64_t Gk = L.G[lv];
#pragma unroll 1
      for (int i0 = t; i0 < count; i0 += U * kConsumers) {
        uint64_t bits[U];
        uint32_t sum[U];
        int64_t off[U];
        bool ok[U];
#pragma unroll
        for (int v = 0; v < U; ++v) {
          const int i = min(i0 + v * kConsumers, count - 1);
          const int c = i & ((1 << lgc) - 1);
          const int rest = i >> lgc;
          const int ch = rest % C, q = rest / C;
          const int rk = r0 + q, ck = c0 + c;
          ok[v] = i0 + v * kConsumers < count && rk < GRk && ck < GCk;
          sum[v] = lv == 0 ? t4[q][c][ch]
                   : lv == 1 ? t8[NLEV > 1 ? q : 0][c][ch]
                   : lv == 2 ? t16[NLEV > 2 ? q : 0][c][ch]
                             : t32[0][c][ch];
          const int64_t plane = static_cast<int64_t>(f) * C + ch;
          bits[v] = keyed ? key_sub(key_cell(a.noise.seed(plane), rk, ck), 0, 0) : 0ull;  // key (r, c, 0, 0)
          off[v] = plane * Gk + static_cast<int64_t>(rk) * GCk + ck;
          if (a.noise.kind == DPPX_NOISE_PHILOX && ok[v])
            bits[v] = philox_call(a.noise.seed(0), a.noise.frame_base + f, ch, rk, ck, 0, 0);
        }
#pragma unroll
        for (int v = 0; v < U; ++v) {
          if (!ok[v]) continue;
          if (L.ne == 3) {
            sweep_quantize<3>(L, lv, 0, sum[v], bits[v], a.noise.kind, exact_only, off[v], queue, &qn);
          } else {
#pragma unroll 1
            for (int j = 0; j < L.ne; ++j)
              sweep_quantize<1>(L, lv, j, sum[v], bits[v], a.noise.kind, exact_only, off[v], queue, &qn);
          }
        }
      }
    }
    named_bar_sync(1, kConsumers);
    // the unit's ambiguous statistics, exact f64 reference arithmetic, compacted
    const int nq = min(qn, kSweepQueue);
    for (int i = t; i < nq; i += kConsumers) {
      const ExactJob& e = queue[i];
      *e.dst = static_cast<uint8_t>(exact_quantize(e.sum, L.area[e.lv], a.noise.kind, e.bits,
                                                   L.sigma[e.lv][e.j], 0.0));
    }
    named_bar_sync(1, kConsumers);  // tables and queue are rewritten by the next unit
    if (t == 0) qn = 0;
  }
}

using SweepKernel = void (*)(const CUtensorMap, const StatsArgs, const SweepLevels);

SweepKernel select_sweep_kernel(int C, int nlev) {
#define DPPX_SWEEP(Cv, NL) \
  if (C == (Cv) && nlev == (NL)) return k_sweep_stats<Cv, NL>;
  DPPX_SWEEP(1, 2)
  DPPX_SWEEP(1, 3)
  DPPX_SWEEP(1, 4)
  DPPX_SWEEP(3, 2)
  DPPX_SWEEP(3, 3)
  DPPX_SWEEP(3, 4)
#undef DPPX_SWEEP
  return nullptr;
}

cudaError_t launch_sweep(SweepKernel k, const CUtensorMap& tin, const StatsArgs& a, const SweepLevels& L,
                         int grid, size_t smem, cudaStream_t s) {
  k<<<grid, kStatsThreads, smem, s>>>(tin, a, L);
  return cudaGetLastError();
}

}  // namespace dppx
