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

#include <math_constants.h>

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

// log1p exactly as the reference's libm evaluates it. std::log1p (noise.cpp:110)
// resolves to glibc 2.39's sysdeps/ieee754/dbl-64/s_log1p.c (the fdlibm
// algorithm with an Estrin-split polynomial) in its x86-64 FMA/AVX2 ifunc
// variant, i.e. with GCC's FMA contractions. Every operation below, including
// which ones are fused, follows that compiled sequence, so the noise doubles
// are bit-identical to the reference's (oracle twin: or_log1p_glibc, checked
// against the host libm in tests/test_oracle_kats.py). Domain used here:
// x = -2|u| in (-1, 0]; the other branches are kept for completeness.
static __device__ __noinline__ double glibc_log1p(double x) {
  const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
  const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2,
               Lp3 = 0x1.2492494229359p-2, Lp4 = 0x1.c71c51d8e78afp-3,
               Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3,
               Lp7 = 0x1.2f112df3e5244p-3;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -CUDART_INF : CUDART_NAN;
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return __fma_rn(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= static_cast<int>(0xbfd2bec3)) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return __dadd_rn(x, x);
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = __dadd_rn(x, 1.0);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
  const double dk = static_cast<double>(k);
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
    const double R = __dmul_rn(__fma_rn(-f, 0x1.5555555555555p-1, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
  const double z = __dmul_rn(s, s);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double t = __dmul_rn(__dadd_rn(R, hfsq), s);
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  const double w = __dsub_rn(hfsq, __dadd_rn(__fma_rn(dk, ln2_lo, c), t));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(w, f));
}

// laplace_from_uniform, noise.cpp:107-110: (sign * sigma) * -log1p(-2|u|).
__device__ __forceinline__ double laplace_from_uniform(double u, double sigma) {
  const double sign = u < 0.0 ? -1.0 : 1.0;
  const double l = glibc_log1p(__dmul_rn(-2.0, fabs(u)));
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

// ---- quantized statistic: fast bounded path + exact fallback ---------------
//
// The reference computes q = llround(clip(mean + noise)) in f64 with
// noise = (sign*sigma) * -log1p(-2|u|) (noise.cpp:107-110, pixelize.cpp:25-31).
// q only depends on which interval [j - 0.5, j + 0.5) the f64 value falls in,
// so a cheap f32 estimate v_est with a proven error bound decides q whenever
// v_est is farther than `margin` from every rounding boundary (0.5 ... 254.5);
// otherwise (a few per mille of draws) the exact f64 arithmetic runs. The
// emitted bytes are therefore those of the exact evaluation. Error budget of
// the estimate:
//   log2 of w = 1 - 2|u| = W * 2^-52 (W an exact integer): W converted to
//   f32 (relative error <= 2^-24, so <= 8.6e-8 in log2), lg2.approx (<= 2^-21,
//   checked exhaustively on the device by tests/test_gpu_parity.py)
//   => |d noise| <= sigma * ln2 * 6.6e-7 <= sigma * 4.6e-7;
//   f32 rounding of mean + 0.5 (one FFMA), of -log2(1-2|u|), of sigma * ln 2
//   and of the final FFMA (each relative to |t|, |noise| <= 512 where it
//   matters) <= 1.2e-4 <= 2.5e-4.
// margin = 5e-4 + sigma * 1e-6 keeps a factor >= 2 over that budget (round 1
// used 2e-3 + 4e-6 sigma, a factor 8: 4x as many exact f64 evaluations, the
// dominant cost of draw-bound shapes such as b = 4 at eps = 0.1, sigma = 2550).
__host__ __device__ __forceinline__ float fast_margin(double sigma) {
  return 5e-4f + static_cast<float>(sigma) * 1e-6f;
}

// MUFU lg2 (no denormal fix-up: the argument is a mantissa in [1, 2)); its
// error on [1, 2) is measured exhaustively by k_debug_lg2.
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// q = clip(floor(t), 0, 255) for t = mean + noise + 0.5, or 0xFFFFFFFF when t
// lies within `margin` of a rounding boundary inside [1, 255]. Clamping t to
// [0.5, 255.5] first makes the range test implicit (an integer within margin
// < 0.5 of the clamped value lies in [1, 255]) and floor(clamped) is the
// clipped floor: two instructions fewer than testing the range and clipping.
__device__ __forceinline__ uint32_t fast_finish(float t, float margin) {
  const float tc = fminf(fmaxf(t, 0.5f), 255.5f);
  const float j = rintf(tc);
  if (fabsf(tc - j) <= margin) return 0xFFFFFFFFu;
  return static_cast<uint32_t>(__float2int_rd(tc));
}

// Returns the quantized value, or 0xFFFFFFFF when v_est is ambiguous.
// sln2 = f32(sigma * ln 2) (DrawEnv): noise = -log2(1 - 2|u|) * sigma * ln 2.
__device__ __forceinline__ uint32_t fast_quantize(uint32_t sum, float inv_area, uint64_t bits,
                                                  float sln2, float margin) {
  const uint64_t y = bits >> 11;                    // 53-bit integer of uniform_from_bits
  uint32_t lo_w, hi_w;  // top-bit test on the high word alone (on the 64-bit value the
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo_w), "=r"(hi_w) : "l"(bits));  // compiler emits 2 compares)
  (void)lo_w;
  const bool neg = static_cast<int32_t>(hi_w) >= 0;  // y < 2^52, i.e. u < 0
  // 1 - 2|u| = W * 2^-52: W = y for u < 0 (at least 1: the +-(0.5 - 2^-53)
  // clamp of noise.cpp:99-104, applied below on the f32 value), 2^53 - y
  // otherwise; W in [1, 2^52].
  const uint64_t W = neg ? y : (1ull << 53) - y;
  // W as f32 (hardware conversion, mantissa rounded to nearest: relative error
  // <= 2^-24; W = 0 becomes 1); exponent and mantissa taken from its bits.
  const uint32_t wb = __float_as_uint(fmaxf(__ull2float_rn(W), 1.0f));
  const int e = static_cast<int>(wb >> 23) - 127;  // floor(log2 Wf)
  const float lg_m = lg2_approx(__uint_as_float(0x3F800000u | (wb & 0x7FFFFFu)));  // log2 of [1,2)
  const float L2 = static_cast<float>(52 - e) - lg_m;  // -log2(1 - 2|u|)
  const float t = fmaf(L2, neg ? -sln2 : sln2, fmaf(static_cast<float>(sum), inv_area, 0.5f));
  return fast_finish(t, margin);
}

// The reference's f64 arithmetic, step for step (rare path).
static __device__ __noinline__ uint32_t exact_quantize(uint32_t sum, double area, int kind, uint64_t bits,
                                                double sigma, double injected) {
  const double mean = cell_mean(sum, area);
  double noise = 0.0;
  if (kind == DPPX_NOISE_KEYED || kind == DPPX_NOISE_PHILOX)
    noise = laplace_from_uniform(uniform_from_bits(bits), sigma);
  else if (kind == DPPX_NOISE_INJECTED)
    noise = injected;
  return finalize_value(mean, noise);
}

// Per-(unit, statistic kind) constants.
struct DrawEnv {
  int kind;
  bool exact_only;  // test switch: always take the f64 path
  bool pow2;        // area is a power of two: sum * inv_area is exact in f32
  double area, sigma;
  float inv_area, sln2, margin;
};

__device__ __forceinline__ DrawEnv make_env(int kind, bool exact_only, double area, double sigma) {
  DrawEnv e;
  e.kind = kind;
  e.exact_only = exact_only;
  const uint32_t ia = static_cast<uint32_t>(area);
  e.pow2 = (ia & (ia - 1)) == 0 && static_cast<double>(ia) == area;
  e.area = area;
  e.sigma = sigma;
  e.inv_area = 1.0f / static_cast<float>(area);
  e.sln2 = static_cast<float>(sigma * 0.6931471805599453);
  e.margin = fast_margin(sigma);
  return e;
}

// `inj` yields the caller-injected noise value (DPPX_NOISE_INJECTED only); it is
// evaluated lazily so its index arithmetic stays off the common path.
template <class Inj>
__device__ __forceinline__ uint32_t quantize_stat(const DrawEnv& e, uint32_t sum, uint64_t bits,
                                                  const Inj& inj) {
  if (!e.exact_only) {
    if (e.kind == DPPX_NOISE_KEYED || e.kind == DPPX_NOISE_PHILOX) {
      const uint32_t q = fast_quantize(sum, e.inv_area, bits, e.sln2, e.margin);
      if (q != 0xFFFFFFFFu) return q;
    } else if (e.kind == DPPX_NOISE_NONE && e.pow2) {
      // sum * 2^-k + 0.5 is exact in f32 (< 24 significant bits).
      return static_cast<uint32_t>(floorf(static_cast<float>(sum) * e.inv_area + 0.5f));
    }
  }
  return exact_quantize(sum, e.area, e.kind, bits, e.sigma,
                        e.kind == DPPX_NOISE_INJECTED ? inj() : 0.0);
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

// Blocking wait for the phase with `parity`; the thread is suspended in
// hardware (suspend-time hint) instead of spinning, so a waiting producer or
// consumer does not steal issue slots from the warps doing the work.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1, %2;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(0x100000u)
      : "memory");
}

// global -> shared bulk copy, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 3-D tensor TMA (cp.async.bulk.tensor): box {x, y, z} of the tensor map
// `tmap` (a __grid_constant__ kernel parameter) into / out of shared memory.
// Loads zero-fill and stores clip out-of-bounds elements.
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const void* tmap, int x, int y, int z,
                                             const void* smem_src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(x), "r"(y), "r"(z), "r"(smem_u32(smem_src))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
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
