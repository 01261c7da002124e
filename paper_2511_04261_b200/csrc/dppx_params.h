// dppx_params.h -- launch-argument structs shared by the host runtime
// (capi.cu) and the kernels (kernels.cu). Plain data, passed by value.
#pragma once

#include <cstdint>

#include "../../include/dppx_gpu.h"

namespace dppx {

// n / d for n < 2^31 by multiply-shift: s = 31 + ceil(log2 d), m = ceil(2^s / d)
// (then n*m / 2^s < n/d + 1/d, so the floor is exact).
struct FastDiv {
  uint32_t d, m, s;
#ifdef __CUDACC__
  __host__ __device__
#endif
  uint32_t div(uint32_t n) const {
    return static_cast<uint32_t>((static_cast<uint64_t>(n) * m) >> s);
  }
};

#ifdef __CUDACC__
__host__ __device__
#endif
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  FastDiv f;
  f.d = d;
  f.s = 31 + l;
  f.m = static_cast<uint32_t>(((1ull << f.s) + d - 1) / d);
  return f;
}

// Geometry of one batch (GridGeometry image.hpp:71-82, plus batch shape).
struct BatchGeom {
  int M, N, C, F;         // rows, cols, channels, frames
  int b, n, sb;           // grid side, subgrid factor, subgrid side
  int GR, GC, G, PR, PC;  // grid_dims (image.cpp:48-72)
};

constexpr int kInlineSeeds = 48;  // planes whose seeds ride in the kernel parameters

struct NoiseArgs {
  int kind;
  uint32_t frame_base;
  const uint64_t* mixed_seeds;  // device: KEYED mix64(seed) per plane; PHILOX [0]=seed
  const double* injected;       // device
  int inline_count;             // > 0: seeds are in `inline_seeds` (no H2D copy per call)
  uint64_t inline_seeds[kInlineSeeds];

#ifdef __CUDACC__
  __device__ __forceinline__ uint64_t seed(int64_t plane) const {
    return inline_count > 0 ? inline_seeds[plane] : __ldg(&mixed_seeds[plane]);
  }
#endif
};

// K0: region classification + packed-slot scan.
struct ClassifyArgs {
  BatchGeom g;
  int planes;                // P: F (mask per frame) or F*C (payload per plane)
  int from_payload;          // 0: sum the u8 mask; 1: mask means read from payloads
  const uint8_t* mask;       // from_payload == 0
  int64_t mpitch, mfstride;
  int vec;                   // 16, 4 or 1: widest aligned load for the mask rows
  int mask_bits;             // mask rows are packed bits (u32 words, maskpack.h), mpitch in bytes
  const uint8_t* flags;      // mode 3: per-cell simple flags [F][G] from the fused variance K1
  int band;                  // mode 0: band column sums in dynamic smem (GC*b u32)
  uint8_t* payload;          // from_payload == 0: mask means + S written for C planes
  const uint8_t* payload_in; // from_payload == 1
  int64_t pstride;
  int64_t plen_limit;        // from_payload == 1: longest legal payload (caller's stride)
  uint32_t* payload_len;     // nullable (written)
  const uint32_t* in_len;    // nullable (checked, from_payload == 1)
  uint32_t* cellinfo;        // [P][G]  (intra-row exclusive simple prefix << 1) | simple
  uint32_t* rowcnt;          // [P][GR]
  uint32_t* rowprefix;       // [P][GR]
  uint32_t* totals;          // [P]
  uint32_t* counters;        // [P] self-resetting arrival tickets
  int* status;               // set to DPPX_ERR_CORRUPT on inconsistent payloads
  double area;               // (double)b*b
  double inv_area_pow2;      // 1 / area when b is a power of two (exact), else 0: K0 multiplies
  // from_payload == 2: variance classification (extension): cell complex iff
  // var(C*b*b samples) >= var_tau, computed from the frames themselves.
  const uint8_t* img;
  int64_t pitch, fstride;
  int img_vec4;              // rows/cells 4-byte aligned: word loads
  double var_tau;
};

// K1 / K1g: fused statistics, noise, compact store and reconstruction.
struct StatsArgs {
  BatchGeom g;
  int adaptive;
  const uint8_t* img;
  int64_t pitch, fstride;
  uint8_t* out;              // nullable
  int64_t opitch, ofstride;
  uint8_t* stats;            // uniform: means; adaptive: payload slots
  int64_t sstride;           // bytes between planes of `stats`
  const uint32_t* cellinfo;  // adaptive: [F][G]
  const uint32_t* rowprefix; // adaptive: [F][GR]
  const uint32_t* totals;    // adaptive: [F]
  double area, sub_area, sigma, sigma_sub;
  NoiseArgs noise;
  int exact_noise;           // 1: always evaluate the f64 reference arithmetic
  int partial_borders;       // 1: Algorithm 1 (pixelize_reference): border cells average
                             //    only their h x w real pixels, no mirror padding
  // K1 (staged) only
  int tiles_per_row;
  int units;
  int stages;
  int* work_counter;         // zeroed before each launch; units are claimed dynamically
  FastDiv div_tiles, div_rows;
  int tensor_in_bytes;       // row bytes covered by the input tensor map (N*C rounded down to 8)
  int tensor_out_bytes;      // same for the output tensor map
  // A unit stages `pack` frames side by side ("slots"): narrow frames (e.g.
  // 178 px) share one tile instead of leaving most lanes idle. Wide frames use
  // pack = 1 and a 512-px slot. Smem: slot j at j*slot_stride, its rows at
  // slot_px*C bytes (the TMA box is stored densely).
  int pack, slot_px, slot_stride;
  int row_slack;             // 1: input pitch >= roundup(N*C, 16), loads may read the slack
  // Grid rows [row_begin, row_begin + row_count) of every frame are processed
  // (the host pipeline's row bands for single-frame calls); 0 / GR otherwise.
  int row_begin, row_count;
  // EXTENSION, fused variance classification (k_stats_tma<..., VAR = true>):
  // each cell is classified by its own variance in the same pass; statistics
  // go to a per-cell staging area (slot positions need the whole frame's simple
  // count) that K0 (mode 3) + k_gather_stage compact into the payload.
  double var_tau;
  uint8_t* var_flags;        // [F][G]: 1 simple, 0 complex
  uint8_t* stage;            // [F*C][stage_stride]: simple value of cell g at g,
                             // complex block at stage_cx + g*n*n (+ sr*n + sc)
  int64_t stage_stride, stage_cx;
};

// Compaction of fused-variance staging into DPPX payloads (after K0 mode 3).
struct GatherArgs {
  BatchGeom g;
  const uint8_t* stage;
  int64_t stage_stride, stage_cx;
  const uint32_t* cellinfo;  // [F][G]
  const uint32_t* rowprefix; // [F][GR]
  const uint32_t* totals;    // [F]
  uint8_t* payload;
  int64_t pstride;
};

// K2: statistics -> pixels.
struct ExpandArgs {
  BatchGeom g;
  int adaptive;
  const uint8_t* stats;
  int64_t sstride;
  const uint32_t* cellinfo;  // adaptive: [F*C][G]
  const uint32_t* rowprefix; // adaptive: [F*C][GR]
  const uint32_t* totals;    // adaptive: [F*C]
  uint8_t* out;
  int64_t opitch, ofstride;
  // K2 (staged) only: one CTA per unit (frame group, grid row, tile).
  int tiles_per_row;
  int tensor_out_bytes;
  FastDiv div_tiles, div_rows;
  int units;
  int pack, slot_px, slot_stride;  // narrow frames: `pack` frames side by side per tile
  int stage_bytes;                 // bytes of the smem tile
};

}  // namespace dppx
