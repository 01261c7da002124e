// K1z: uniform statistics + reconstruction for small host frames read and
// written over PCIe by the SMs themselves (zero-copy on the caller's mapped
// page-locked buffers; the `run_single` shape, cli.cpp:108-130).
//
// A single PETS frame (768 x 576 RGB, 1.33 MB) gains nothing from a staged
// H2D -> K1 -> D2H chain: each copy-engine transfer costs ~30 us and the two
// run back to back (tools/pcie_probe.cu). Here every CTA streams units (one
// grid row x a slab of S cells) through a two-deep cp.async ring: the PCIe
// reads of unit k+1 are in flight while unit k's sums, draws, statistics and
// output rows are produced, so the inbound and outbound halves of the link
// run at the same time instead of one after the other.
//
// Same arithmetic as every other statistics kernel (pixelize.cpp:86-124): the
// exact u32 cell sum, keyed / Philox / injected noise through quantize_stat,
// statistics plane-major at (f*C + ch)*sstride + r*GC + c, every pixel of the
// cell set to the cell's value. Eligible shapes (host checks): n == 1, no
// padding (b divides M and N), 16-byte rows, no row bands.
#include <cuda_runtime.h>

#include <cstdint>

#include "dppx_device.cuh"
#include "dppx_params.h"
#include "stats_common.cuh"

namespace dppx {

constexpr int kZcThreads = 256;

__device__ __forceinline__ void zc_cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void zc_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void zc_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct ZcArgs {
  int S;            // cells per slab
  int nslab;        // slabs per grid row
  int units;        // F * GR * nslab
  int unit_stride;  // bytes of one ring slot (>= b * S * b * C, 16-byte multiple)
  int vals_bytes;   // S * C (adaptive: S * n * n * C) rounded up to 16
  int pattern_bytes;  // adaptive: n * S * b * C rounded up to 16
};

template <int C>
__global__ void __launch_bounds__(kZcThreads) k_stats_zc(const StatsArgs a, const ZcArgs z) {
  extern __shared__ __align__(16) uint8_t zs[];
  const BatchGeom& g = a.g;
  const int b = g.b;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint8_t* vals = zs + 2 * z.unit_stride;
  uint8_t* pattern = vals + z.vals_bytes;
  const DrawEnv env = make_env(a.noise.kind, a.exact_noise != 0, a.area, a.sigma);
  auto coords = [&](int u, int& f, int& r, int& s) {
    s = u % z.nslab;
    const int q = u / z.nslab;
    r = q % g.GR;
    f = q / g.GR;
  };
  auto issue = [&](int u, uint8_t* dst) {
    int f, r, s;
    coords(u, f, r, s);
    const int s0 = s * z.S, su = min(z.S, g.GC - s0);
    const int sbytes = su * b * C, per_row = sbytes >> 4;
    const uint8_t* src = a.img + static_cast<int64_t>(f) * a.fstride + static_cast<int64_t>(r) * b * a.pitch +
                         static_cast<int64_t>(s0) * b * C;
    for (int i = t; i < per_row * b; i += kZcThreads) {
      const int y = i / per_row, q = i - y * per_row;
      zc_cp16(dst + y * sbytes + q * 16, src + static_cast<int64_t>(y) * a.pitch + q * 16);
    }
    zc_commit();
  };
  int u = blockIdx.x;
  if (u < z.units) issue(u, zs);
  for (int k = 0; u < z.units; ++k, u += gridDim.x) {
    const int un = u + gridDim.x;
    if (un < z.units) {
      issue(un, zs + ((k + 1) & 1) * z.unit_stride);
      zc_wait<1>();
    } else {
      zc_wait<0>();
    }
    __syncthreads();
    const uint8_t* tile = zs + (k & 1) * z.unit_stride;
    int f, r, s;
    coords(u, f, r, s);
    const int s0 = s * z.S, su = min(z.S, g.GC - s0), sbytes = su * b * C;
    // exact cell sums, one warp per (cell, channel); lane 0 draws the noise
    for (int p = w; p < su * C; p += kZcThreads / 32) {
      const int c = p / C, ch = p - c * C;
      uint32_t sum = 0;
      for (int i = lane; i < b * b; i += 32) {
        const int y = i / b, x = i - y * b;
        sum += tile[y * sbytes + (c * b + x) * C + ch];
      }
      sum = __reduce_add_sync(0xffffffffu, sum);
      if (lane == 0) {
        const int cg = s0 + c;
        const uint64_t cs = cell_state(a, f, ch, r, cg);
        vals[p] = static_cast<uint8_t>(
            draw_stat(a, env, sum, cs, f, ch, r, cg, 0, 0, r * g.GC + cg));
      }
    }
    __syncthreads();
    // statistics: one run of su bytes per channel plane (coalesced stores)
    for (int e = t; e < su * C; e += kZcThreads) {
      const int ch = e / su, c = e - ch * su;
      a.stats[static_cast<int64_t>(f * C + ch) * a.sstride + r * g.GC + s0 + c] = vals[c * C + ch];
    }
    if (a.out) {  // the b output rows of the unit are one repeated pattern row
      for (int x = t; x < sbytes; x += kZcThreads) {
        const int px = x / C, ch = x - px * C;
        pattern[x] = vals[(px / b) * C + ch];
      }
      __syncthreads();
      uint8_t* dst = a.out + static_cast<int64_t>(f) * a.ofstride + static_cast<int64_t>(r) * b * a.opitch +
                     static_cast<int64_t>(s0) * b * C;
      const int per_row = sbytes >> 4;
      for (int i = t; i < per_row * b; i += kZcThreads) {
        const int y = i / per_row, q = i - y * per_row;
        *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(y) * a.opitch + q * 16) =
            reinterpret_cast<const uint4*>(pattern)[q];
      }
    }
    __syncthreads();  // ring slot, vals and pattern free for reuse
  }
}

// Adaptive (pixelize_adaptive, adaptive.cpp:88-179) counterpart: K0 has
// classified the cells (cellinfo / rowprefix / totals in HBM, the mask means
// already in the payload); the frame streams in as above. A warp takes one
// (cell, channel): a simple cell is one sum over b x b pixels drawn at sigma,
// a complex cell n x n subcell sums (one lane per subcell) drawn at sigma_sub;
// values go to the payload slot (stat_offset) and into a per-unit table
// vals[cell][sr][sc][ch], from which one pattern row per vertical subcell
// band is built and stored sb times.
template <int C>
__global__ void __launch_bounds__(kZcThreads) k_adaptive_zc(const StatsArgs a, const ZcArgs z) {
  extern __shared__ __align__(16) uint8_t zs[];
  const BatchGeom& g = a.g;
  const int b = g.b, n = g.n, sb = g.sb, NN = n * n;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint8_t* vals = zs + 2 * z.unit_stride;              // S * n * n * C
  uint8_t* pattern = vals + z.vals_bytes;              // n rows of S * b * C
  uint32_t* meta = reinterpret_cast<uint32_t*>(pattern + z.pattern_bytes);  // S cell infos
  const DrawEnv env_cell = make_env(a.noise.kind, a.exact_noise != 0, a.area, a.sigma);
  const DrawEnv env_sub = make_env(a.noise.kind, a.exact_noise != 0, a.sub_area, a.sigma_sub);
  auto coords = [&](int u, int& f, int& r, int& s) {
    s = u % z.nslab;
    const int q = u / z.nslab;
    r = q % g.GR;
    f = q / g.GR;
  };
  auto issue = [&](int u, uint8_t* dst) {
    int f, r, s;
    coords(u, f, r, s);
    const int s0 = s * z.S, su = min(z.S, g.GC - s0);
    const int sbytes = su * b * C, per_row = sbytes >> 4;
    const uint8_t* src = a.img + static_cast<int64_t>(f) * a.fstride + static_cast<int64_t>(r) * b * a.pitch +
                         static_cast<int64_t>(s0) * b * C;
    for (int i = t; i < per_row * b; i += kZcThreads) {
      const int y = i / per_row, q = i - y * per_row;
      zc_cp16(dst + y * sbytes + q * 16, src + static_cast<int64_t>(y) * a.pitch + q * 16);
    }
    zc_commit();
  };
  int u = blockIdx.x;
  if (u < z.units) issue(u, zs);
  // The frame loads above do not depend on K0; its classification does.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int k = 0; u < z.units; ++k, u += gridDim.x) {
    const int un = u + gridDim.x;
    if (un < z.units) {
      issue(un, zs + ((k + 1) & 1) * z.unit_stride);
      zc_wait<1>();
    } else {
      zc_wait<0>();
    }
    int f, r, s;
    coords(u, f, r, s);
    const int s0 = s * z.S, su = min(z.S, g.GC - s0), sbytes = su * b * C;
    // (K0's results, written by a grid that may still have been running when
    // this one started: read through L2, not the non-coherent path)
    for (int c = t; c < su; c += kZcThreads)
      meta[c] = __ldcg(&a.cellinfo[static_cast<int64_t>(f) * g.G + r * g.GC + s0 + c]);
    __syncthreads();
    const uint8_t* tile = zs + (k & 1) * z.unit_stride;
    const uint32_t rowpre = __ldcg(&a.rowprefix[static_cast<int64_t>(f) * g.GR + r]);
    const uint32_t S_tot = __ldcg(&a.totals[f]);
    for (int p = w; p < su * C; p += kZcThreads / 32) {
      const int c = p / C, ch = p - c * C;
      const int cg = s0 + c, gidx = r * g.GC + cg;
      const uint32_t info = meta[c];
      const bool simple = info & 1u;
      const uint32_t slot_s = rowpre + (info >> 1);
      const uint64_t cs = cell_state(a, f, ch, r, cg);
      uint8_t* plane = a.stats + static_cast<int64_t>(f * C + ch) * a.sstride;
      uint8_t* cv = vals + static_cast<int64_t>(c) * NN * C + ch;  // vals[c][sr][sc][ch]
      if (simple) {
        uint32_t sum = 0;
        for (int i = lane; i < b * b; i += 32) {
          const int y = i / b, x = i - y * b;
          sum += tile[y * sbytes + (c * b + x) * C + ch];
        }
        sum = __reduce_add_sync(0xffffffffu, sum);
        uint32_t v = 0;
        if (lane == 0) {
          v = draw_stat(a, env_cell, sum, cs, f, ch, r, cg, 0, 0, gidx);
          plane[stat_offset(a, true, gidx, slot_s, S_tot, 0, 0)] = static_cast<uint8_t>(v);
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        for (int i = lane; i < NN; i += 32) cv[i * C] = static_cast<uint8_t>(v);
      } else {
        for (int i = lane; i < NN; i += 32) {
          const int sr = i / n, sc = i - sr * n;
          uint32_t sum = 0;
          for (int y = sr * sb; y < sr * sb + sb; ++y) {
            const uint8_t* row = tile + y * sbytes + (c * b + sc * sb) * C + ch;
            for (int x = 0; x < sb; ++x) sum += row[x * C];
          }
          const uint32_t v = draw_stat(a, env_sub, sum, cs, f, ch, r, cg, sr, sc, gidx);
          plane[stat_offset(a, false, gidx, slot_s, S_tot, sr, sc)] = static_cast<uint8_t>(v);
          cv[i * C] = static_cast<uint8_t>(v);
        }
      }
    }
    __syncthreads();
    if (a.out) {
      // one pattern row per vertical subcell band
      for (int e = t; e < n * sbytes; e += kZcThreads) {
        const int sr = e / sbytes, x = e - sr * sbytes;
        const int px = x / C, ch = x - px * C;
        const int c = px / b, sc = (px - c * b) / sb;
        pattern[e] = vals[((c * n + sr) * n + sc) * C + ch];
      }
      __syncthreads();
      uint8_t* dst = a.out + static_cast<int64_t>(f) * a.ofstride + static_cast<int64_t>(r) * b * a.opitch +
                     static_cast<int64_t>(s0) * b * C;
      const int per_row = sbytes >> 4;
      for (int i = t; i < per_row * b; i += kZcThreads) {
        const int y = i / per_row, q = i - y * per_row;
        *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(y) * a.opitch + q * 16) =
            reinterpret_cast<const uint4*>(pattern + (y / sb) * sbytes)[q];
      }
    }
    __syncthreads();  // ring slot, tables and pattern free for reuse
  }
}

// *launched = false if the shape is not eligible; else launches (dry_run: only
// reports eligibility). `unit_target`: bytes per unit (<= 16 KB), `ctas`: grid
// (0: automatic).
cudaError_t launch_stats_zc(const StatsArgs& a, int unit_target, int ctas, int sms, cudaStream_t s, bool* launched,
                            bool dry_run) {
  *launched = false;
  const BatchGeom& g = a.g;
  const int b = g.b, C = g.C;
  if ((!a.adaptive && g.n != 1) || g.PR != 0 || g.PC != 0 || a.partial_borders || a.row_begin != 0 ||
      a.row_count != g.GR || (C != 1 && C != 3) || b > 64 || a.var_flags)
    return cudaSuccess;
  if ((static_cast<int64_t>(g.N) * C) % 16 || a.pitch % 16 || a.fstride % 16 ||
      (reinterpret_cast<uintptr_t>(a.img) & 15))
    return cudaSuccess;
  if (a.out && (a.opitch % 16 || a.ofstride % 16 || (reinterpret_cast<uintptr_t>(a.out) & 15))) return cudaSuccess;
  // Slab rows on whole 128-byte lines where the width allows (measured: rows
  // of 240 / 480 / 1008 bytes read and write over PCIe 15-55 % slower than
  // 384 / 768-byte ones, profiles/r02_zerocopy.txt), else on 16 bytes.
  int base = 1;
  while ((base * b * C) % 128 && base <= g.GC) ++base;
  if (base > g.GC) {
    base = 1;
    while ((base * b * C) % 16) ++base;
  }
  if (base > g.GC) return cudaSuccess;
  unit_target = unit_target < 2048 ? 2048 : (unit_target > 16384 ? 16384 : unit_target);
  int S = base;
  while (S + base <= g.GC && (S + base) * b * b * C <= unit_target && (S + base) * C <= 1024) S += base;
  // the last slab must end on a 16-byte boundary too: it ends at N*C
  const int nslab = (g.GC + S - 1) / S;
  ZcArgs z;
  z.S = S;
  z.nslab = nslab;
  const int64_t units = static_cast<int64_t>(g.F) * g.GR * nslab;
  if (units > 0x7FFFFFFF) return cudaSuccess;
  z.units = static_cast<int>(units);
  z.unit_stride = (S * b * b * C + 127) / 128 * 128;
  const int nn = a.adaptive ? g.n * g.n : 1;
  z.vals_bytes = (S * nn * C + 15) / 16 * 16;
  z.pattern_bytes = ((a.adaptive ? g.n : 1) * S * b * C + 15) / 16 * 16;
  const size_t smem = 2 * static_cast<size_t>(z.unit_stride) + z.vals_bytes + z.pattern_bytes +
                      (a.adaptive ? 4 * static_cast<size_t>(S) : 0);
  if (smem > 200 * 1024) return cudaSuccess;
  if (dry_run) {
    *launched = true;
    return cudaSuccess;
  }
  auto k = a.adaptive ? (C == 1 ? k_adaptive_zc<1> : k_adaptive_zc<3>) : (C == 1 ? k_stats_zc<1> : k_stats_zc<3>);
  if (cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)))
    return e;
  // Default: about three units per CTA, so each CTA's PCIe reads of its next
  // unit overlap the writes of its current one.
  int grid = ctas > 0 ? ctas : (z.units + 2) / 3;
  grid = grid < 1 ? 1 : (grid > 4 * sms ? 4 * sms : grid);
  if (grid > z.units) grid = z.units;
  if (a.adaptive) {
    // Programmatic dependent launch: the kernel starts while K0 (which
    // releases its dependents at entry) still runs, streams its first frame
    // units in, and waits for K0's results at griddepcontrol.wait.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kZcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaError_t e = cudaLaunchKernelEx(&cfg, k, a, z)) return e;
  } else {
    k<<<grid, kZcThreads, smem, s>>>(a, z);
  }
  *launched = true;
  return cudaGetLastError();
}

}  // namespace dppx
