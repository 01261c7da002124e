// dppx_device.cuh -- device-side building blocks of the sm_100a pixelization
// path: reflection, the reference's keyed Laplace stream, Philox, the
// clip/quantize epilogue, and thin PTX wrappers for mbarrier + bulk async copy
// (TMA, cp.async.bulk) used by the staged kernels.
//
// Floating-point parity rules:
//  * every rounding step of the reference is an explicit __d*_rn intrinsic, so
//    nvcc can never contract mean + noise or sign*sigma*L into an FMA;
//  * cell means are one correctly rounded f64 divide of an exact integer sum
//    (image.cpp:184-189, adaptive.cpp:161-162);
//  * quantization is round-half-away-from-zero (llround, pixelize.cpp:29-31).
#pragma once

#include <cstdint>

#include "dppx_params.h"

namespace dppx {

__device__ __forceinline__ int reflect_index(int i, int len) {
  // image.cpp:105-110: appended index len+k reads len-1-k.
  return i < len ? i : len - 1 - (i - len);
}

// splitmix64 finalizer, noise.cpp:77-82.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// keyed_bits (noise.cpp:86-91) split in its per-plane, per-cell and
// per-subcell stages so the first two are computed once and reused.
__device__ __forceinline__ uint64_t key_cell(uint64_t mixed_seed, uint32_t r, uint32_t c) {
  return mix64(mixed_seed ^ ((static_cast<uint64_t>(r) << 32) | c));
}
__device__ __forceinline__ uint64_t key_sub(uint64_t cell_state, uint32_t sr, uint32_t sc) {
  return mix64(cell_state ^ ((static_cast<uint64_t>(sr) << 32) | sc));
}

// Philox4x32-10 extension (oracle/dppx_oracle.c or_philox_bits).
__device__ __forceinline__ uint64_t philox_bits(uint64_t seed, uint32_t frame, uint32_t channel,
                                                uint32_t r, uint32_t c, uint32_t sr,
                                                uint32_t sc) {
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  uint32_t x0 = r, x1 = c, x2 = (sr & 0xFFFFu) | (sc << 16), x3 = (frame << 2) | (channel & 3u);
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, x0), lo0 = 0xD2511F53u * x0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, x2), lo1 = 0xCD9E8D57u * x2;
    const uint32_t y0 = hi1 ^ x1 ^ k0, y2 = hi0 ^ x3 ^ k1;
    x0 = y0;
    x1 = lo1;
    x2 = y2;
    x3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return (static_cast<uint64_t>(x1) << 32) | x0;
}

// uniform_from_bits, noise.cpp:93-105 (every step exact; kept explicit).
__device__ __forceinline__ double uniform_from_bits(uint64_t bits) {
  const double kTwoNeg53 = 0x1.0p-53;
  const double kHalfOpen = 0.5 - kTwoNeg53;
  const double u = __dsub_rn(__dmul_rn(__ull2double_rn(bits >> 11), kTwoNeg53), 0.5);
  if (u <= -kHalfOpen) return -kHalfOpen;
  if (u >= kHalfOpen) return kHalfOpen;
  return u;
}

// laplace_from_uniform, noise.cpp:107-110: (sign * sigma) * -log1p(-2|u|).
__device__ __forceinline__ double laplace_from_uniform(double u, double sigma) {
  const double sign = u < 0.0 ? -1.0 : 1.0;
  const double l = log1p(__dmul_rn(-2.0, fabs(u)));
  return __dmul_rn(__dmul_rn(sign, sigma), -l);
}

// clip_intensity + quantize_intensity (pixelize.cpp:25-31) of mean + noise.
__device__ __forceinline__ uint32_t finalize_value(double mean, double noise) {
  double v = __dadd_rn(mean, noise);
  v = fmin(fmax(v, 0.0), 255.0);
  return static_cast<uint32_t>(round(v));  // half away from zero == llround
}

__device__ __forceinline__ double cell_mean(uint32_t sum, double area) {
  return __ddiv_rn(static_cast<double>(sum), area);
}

// Noise for one statistic of plane `plane` (= f*C + ch) at key (r, c, sr, sc).
// cell_state is key_cell(mix64(seed), r, c) for the KEYED stream.
struct NoiseView {
  int kind;
  uint32_t frame_base;
  const uint64_t* mixed_seeds;  // KEYED: mix64(seed) per plane; PHILOX: [0] = base seed
  const double* injected;       // INJECTED: ((plane*G + g)*n + sr)*n + sc
};

__device__ __forceinline__ double draw_noise(const NoiseView& nz, uint32_t plane, uint32_t frame,
                                             uint32_t ch, uint64_t cell_state, uint32_t r,
                                             uint32_t c, uint32_t sr, uint32_t sc, uint32_t g,
                                             uint32_t G, uint32_t n, double sigma) {
  switch (nz.kind) {
    case DPPX_NOISE_KEYED:
      return laplace_from_uniform(uniform_from_bits(key_sub(cell_state, sr, sc)), sigma);
    case DPPX_NOISE_PHILOX:
      return laplace_from_uniform(
          uniform_from_bits(philox_bits(nz.mixed_seeds[0], nz.frame_base + frame, ch, r, c, sr,
                                        sc)),
          sigma);
    case DPPX_NOISE_INJECTED:
      return nz.injected[((static_cast<size_t>(plane) * G + g) * n + sr) * n + sc];
    default:
      return 0.0;
  }
}

// ---- PTX wrappers: mbarrier + bulk async copies (sm_90+ / sm_100a) ---------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbarrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global bulk copy (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Make this thread's generic-proxy shared-memory writes visible to the async
// proxy (the bulk store that follows reads them).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace dppx
