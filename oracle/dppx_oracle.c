/*
 * dppx_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C CPU restatement of the reference `dppix` pixelization path
 * (/root/reference/proj, C++20). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this file's shared object. The product
 * (paper_2511_04261_b200/csrc) never links or calls it.
 *
 * Every function cites the reference file:line it restates. Paths are
 * relative to /root/reference/proj.
 *
 * Parity pinning: tests/test_oracle_*.py check this restatement against
 *   (1) the known-answer tests in the reference's own unit suites
 *       (tests/test_image.cpp, test_noise.cpp, test_pixelize.cpp,
 *        test_adaptive.cpp, test_record.cpp), restated in Python, and
 *   (2) outputs of the reference itself, compiled from its sources by
 *       oracle/Makefile into oracle/_ref/libdppix_ref.so, live when present and
 *       through the committed fixtures in tests/golden/ (made by
 *       tests/golden/make_golden.py from that library).
 *
 * Extensions that have NO reference counterpart (documented in DESIGN.md):
 *   - interleaved multi-channel (RGB) frames: plane k of a frame is processed
 *     exactly as the reference processes one GrayImage;
 *   - per-(frame, channel) seed derivation (or_derive_plane_seed);
 *   - the Philox4x32-10 noise stream (north-star option);
 *   - injected noise (parity testing);
 *   - the synthetic frame/mask generator used by bench.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID (-1)
#define OR_CORRUPT (-2)

enum { OR_NOISE_NONE = 0, OR_NOISE_KEYED = 1, OR_NOISE_PHILOX = 2, OR_NOISE_INJECTED = 3 };

typedef struct {
  int b, grid_rows, grid_cols, pad_rows, pad_cols;
} or_geom;

/* grid_dims: image.cpp:48-72 (64-bit intermediates, b <= max(M, N)). */
int or_grid_dims(int M, int N, int b, or_geom* g) {
  if (M < 1 || N < 1 || b < 1) return OR_INVALID;
  if (b > (M > N ? M : N)) return OR_INVALID;
  g->b = b;
  g->grid_rows = (int)(((long long)M + b - 1) / b);
  g->grid_cols = (int)(((long long)N + b - 1) / b);
  g->pad_rows = (int)((long long)g->grid_rows * b - M);
  g->pad_cols = (int)((long long)g->grid_cols * b - N);
  return OR_OK;
}

/* mirror_pad_buffer precondition: image.cpp:94-98, applied only when the pad
 * is not the identity (pixelize.cpp:95-102, adaptive.cpp:107-112, 47-49). */
static int pad_ok(const or_geom* g, int M, int N) {
  if (g->pad_rows == 0 && g->pad_cols == 0) return 1;
  return g->pad_rows < M && g->pad_cols < N;
}

/* Edge-inclusive reflection, rows first then columns: image.cpp:105-110. */
static inline int reflect(int i, int len) { return i < len ? i : len - 1 - (i - len); }

/* sensitivity / noise_scale / make_privacy_params: noise.cpp:22-68. */
typedef struct {
  double epsilon;
  int m, b, n, subgrid_side;
  double delta, sigma, delta_sub, sigma_sub;
} or_params;

int or_make_privacy_params(double epsilon, int m, int b, int n, or_params* p) {
  if (!(epsilon > 0.0) || m < 1 || b < 1 || n < 1 || b % n != 0) return OR_INVALID;
  p->epsilon = epsilon;
  p->m = m;
  p->b = b;
  p->n = n;
  p->subgrid_side = b / n;
  p->delta = 255.0 * m / ((double)b * b);
  p->sigma = p->delta / epsilon;
  p->delta_sub = 255.0 * m / ((double)p->subgrid_side * p->subgrid_side);
  p->sigma_sub = p->sigma * ((double)n * n); /* noise.cpp:64-66: sigma*n^2 */
  return OR_OK;
}

/* splitmix64 finalizer: noise.cpp:77-82. */
static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* keyed_bits: noise.cpp:86-91. */
uint64_t or_keyed_bits(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc) {
  uint64_t s = mix64(seed);
  s = mix64(s ^ (((uint64_t)r << 32) | c));
  s = mix64(s ^ (((uint64_t)sr << 32) | sc));
  return s;
}

/* uniform_from_bits: noise.cpp:93-105. */
double or_uniform_from_bits(uint64_t bits) {
  const double two_neg53 = 0x1.0p-53;
  const double half_open = 0.5 - two_neg53;
  const double u = (double)(bits >> 11) * two_neg53 - 0.5;
  if (u <= -half_open) return -half_open;
  if (u >= half_open) return half_open;
  return u;
}

/* glibc 2.39 log1p (sysdeps/ieee754/dbl-64/s_log1p.c, fdlibm algorithm with
 * an Estrin-split polynomial) as its x86-64 FMA ifunc variant evaluates it --
 * the libm the reference's std::log1p (noise.cpp:110) resolves to on FMA
 * hosts. Test infrastructure: pins the device twin (glibc_log1p in
 * dppx_device.cuh) against the host libm; the oracle's own noise keeps calling
 * libm's log1p. Built with -ffp-contract=off, so only the explicit fma() calls
 * are fused. */
static uint32_t hi32(double x) { uint64_t b; memcpy(&b, &x, 8); return (uint32_t)(b >> 32); }
static double with_hi32(double x, uint32_t hi) {
  uint64_t b; memcpy(&b, &x, 8);
  b = ((uint64_t)hi << 32) | (b & 0xffffffffu);
  memcpy(&x, &b, 8);
  return x;
}
double or_log1p_glibc(double x) {
  const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
  const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2,
               Lp3 = 0x1.2492494229359p-2, Lp4 = 0x1.c71c51d8e78afp-3,
               Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3,
               Lp7 = 0x1.2f112df3e5244p-3;
  const int32_t hx = (int32_t)hi32(x);
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) return ax < 0x3c900000 ? x : fma(-(x * x), 0.5, x);
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) { k = 0; f = x; hu = 1; }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = x + 1.0;
      hu = (int32_t)hi32(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = (int32_t)hi32(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi32(u, (uint32_t)(hu | 0x3ff00000));
    } else {
      k += 1;
      u = with_hi32(u, (uint32_t)(hu | 0x3fe00000));
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = (f * 0.5) * f;
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : fma(dk, ln2_hi, fma(dk, ln2_lo, c));
    const double R = fma(-f, 0x1.5555555555555p-1, 1.0) * hfsq;
    if (k == 0) return f - R;
    return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
  }
  const double s = f / (f + 2.0);
  const double z = s * s;
  const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
  const double z2 = z * z, z4 = z2 * z2, z6 = z2 * z4;
  double R = fma(z, Lp1, z2 * R2);
  R = fma(z4, R3, R);
  R = fma(z6, R4, R);
  const double t = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - t);
  return fma(dk, ln2_hi, -((hfsq - (fma(dk, ln2_lo, c) + t)) - f));
}

/* Number of xs where or_log1p_glibc and the linked libm's log1p differ in any bit. */
long or_log1p_glibc_mismatches(const double* xs, long n, double* first_bad) {
  long bad = 0;
  for (long i = 0; i < n; ++i) {
    const double a = or_log1p_glibc(xs[i]), b = log1p(xs[i]);
    if (memcmp(&a, &b, 8) != 0 && !(isnan(a) && isnan(b))) {
      if (bad == 0 && first_bad) *first_bad = xs[i];
      ++bad;
    }
  }
  return bad;
}

/* laplace_from_uniform: noise.cpp:107-110, evaluation order kept:
 * (sign * sigma) * -log1p(-2|u|). */
double or_laplace_from_uniform(double u, double sigma) {
  const double sign = u < 0.0 ? -1.0 : 1.0;
  return sign * sigma * -log1p(-2.0 * fabs(u));
}

/* laplace_at: noise.cpp:112-117 (sigma > 0 checked by callers). */
double or_laplace_at(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc,
                     double sigma) {
  return or_laplace_from_uniform(or_uniform_from_bits(or_keyed_bits(seed, r, c, sr, sc)),
                                 sigma);
}

/* ---- extensions (no reference counterpart) ------------------------------ */

/* Per-(frame, channel) seed: keyed_bits(seed, {f, k, ~0, ~0}). Real keys have
 * sr, sc < n <= 65535, so the derivation never collides with a draw key. */
uint64_t or_derive_plane_seed(uint64_t seed, uint32_t frame, uint32_t channel) {
  return or_keyed_bits(seed, frame, channel, 0xFFFFFFFFu, 0xFFFFFFFFu);
}

/* Philox4x32-10 (Salmon et al., SC'11). key = (lo32, hi32) of the plane seed,
 * counter = (r, c, sr | sc << 16, frame << 2 | channel). */
uint64_t or_philox_bits(uint64_t seed, uint32_t frame, uint32_t channel, uint32_t r,
                        uint32_t c, uint32_t sr, uint32_t sc) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint32_t x0 = r, x1 = c, x2 = (sr & 0xFFFFu) | (sc << 16), x3 = (frame << 2) | (channel & 3u);
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * x0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
    const uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
    const uint32_t y1 = (uint32_t)p1;
    const uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
    const uint32_t y3 = (uint32_t)p0;
    x0 = y0;
    x1 = y1;
    x2 = y2;
    x3 = y3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ((uint64_t)x1 << 32) | x0;
}

/* ---- per-cell finalize ---------------------------------------------------- */

typedef struct {
  int kind;
  uint64_t seed;           /* plane seed (KEYED / PHILOX) */
  uint32_t frame, channel; /* PHILOX counter fields */
  const double* injected;  /* INJECTED: G * n * n per plane, index (g*n + sr)*n + sc */
  int n;                   /* subgrid factor used to index `injected` */
  int grid_cols;
} or_noise;

static double noise_for(const or_noise* nz, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc,
                        double sigma) {
  switch (nz->kind) {
    case OR_NOISE_KEYED:
      return or_laplace_at(nz->seed, r, c, sr, sc, sigma);
    case OR_NOISE_PHILOX:
      return or_laplace_from_uniform(
          or_uniform_from_bits(or_philox_bits(nz->seed, nz->frame, nz->channel, r, c, sr, sc)),
          sigma);
    case OR_NOISE_INJECTED: {
      const size_t g = (size_t)r * nz->grid_cols + c;
      return nz->injected[(g * nz->n + sr) * nz->n + sc];
    }
    default:
      return 0.0;
  }
}

/* clip_intensity + quantize_intensity: pixelize.cpp:25-31 (clamp, llround). */
static inline uint8_t finalize(double mean, double noise) {
  double v = mean + noise;
  if (v < 0.0) v = 0.0;
  if (v > 255.0) v = 255.0;
  return (uint8_t)llround(v);
}

/* Pixel (i, j) of channel ch of the mirror-padded plane (image.cpp:87-133). */
#define PX(img, pitch, C, ch, M, N, i, j) \
  ((img)[(size_t)reflect((i), (M)) * (pitch) + (size_t)reflect((j), (N)) * (C) + (ch)])

/* tile_sum over padded (r*b.., c*b..) of side s at offset (i0, j0):
 * image.cpp:154-171, adaptive.cpp:70-79. */
static uint64_t block_sum(const uint8_t* img, long pitch, int C, int ch, int M, int N, int i0,
                          int j0, int s) {
  uint64_t sum = 0;
  for (int i = i0; i < i0 + s; ++i)
    for (int j = j0; j < j0 + s; ++j) sum += PX(img, pitch, C, ch, M, N, i, j);
  return sum;
}

/* pixelize_parallel for one channel plane: pixelize.cpp:86-124 (means) and
 * broadcast_means pixelize.cpp:126-150 (image). means: G bytes. out (nullable):
 * interleaved M x N x C with pitch out_pitch, only channel ch written. */
int or_pixelize_uniform_plane(const uint8_t* img, int M, int N, long pitch, int C, int ch, int b,
                              double sigma, int noise_kind, uint64_t seed, uint32_t frame,
                              const double* injected, uint8_t* means, uint8_t* out,
                              long out_pitch) {
  or_geom g;
  if (or_grid_dims(M, N, b, &g) != OR_OK || !pad_ok(&g, M, N)) return OR_INVALID;
  if (noise_kind != OR_NOISE_NONE && noise_kind != OR_NOISE_INJECTED && !(sigma > 0.0))
    return OR_INVALID;
  or_noise nz = {noise_kind, seed, frame, (uint32_t)ch, injected, 1, g.grid_cols};
  const double area = (double)b * b; /* image.cpp:187-188 */
  for (int r = 0; r < g.grid_rows; ++r)
    for (int c = 0; c < g.grid_cols; ++c) {
      const uint64_t s = block_sum(img, pitch, C, ch, M, N, r * b, c * b, b);
      const double mean = (double)s / area;
      means[(size_t)r * g.grid_cols + c] =
          finalize(mean, noise_for(&nz, (uint32_t)r, (uint32_t)c, 0, 0, sigma));
    }
  if (out) {
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j)
        out[(size_t)i * out_pitch + (size_t)j * C + ch] =
            means[(size_t)(i / b) * g.grid_cols + j / b];
  }
  return OR_OK;
}

/* classify_regions: adaptive.cpp:34-65 (double mean -> float -> > 0.5f). */
static void classify(const uint8_t* mask, long mask_pitch, int M, int N, const or_geom* g,
                     float* mask_means, uint8_t* is_simple) {
  const int b = g->b;
  const double area = (double)b * b;
  for (int r = 0; r < g->grid_rows; ++r)
    for (int c = 0; c < g->grid_cols; ++c) {
      const uint64_t s = block_sum(mask, mask_pitch, 1, 0, M, N, r * b, c * b, b);
      const float mean = (float)((double)s / area);
      const size_t k = (size_t)r * g->grid_cols + c;
      mask_means[k] = mean;
      is_simple[k] = mean > 0.5f ? 1 : 0; /* simple_from_mean adaptive.cpp:30-32 */
    }
}

static void put_u32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v;
  p[1] = (uint8_t)(v >> 8);
  p[2] = (uint8_t)(v >> 16);
  p[3] = (uint8_t)(v >> 24);
}

/* Payload capacity of one adaptive plane: G f32 + u32 + worst case G*n*n. */
size_t or_adaptive_payload_capacity(int M, int N, int b, int n) {
  or_geom g;
  if (or_grid_dims(M, N, b, &g) != OR_OK) return 0;
  const size_t G = (size_t)g.grid_rows * g.grid_cols;
  return 4 * G + 4 + G * (size_t)n * n;
}

/* pixelize_adaptive for one channel plane: adaptive.cpp:88-179, with the
 * result serialized in the DPPX v1 adaptive payload layout (record.hpp:48-54,
 * record.cpp:153-171): G x f32 LE mask means | u32 S | S simple means |
 * (G-S)*n*n complex submeans. out (nullable) is reassemble (adaptive.cpp:181-245)
 * of that payload for channel ch. */
static int adaptive_core(const uint8_t* img, const uint8_t* mask, const float* mm_in, int M, int N,
                         long pitch, long mask_pitch, int C, int ch, int b, int n, double sigma,
                         double sigma_sub, int noise_kind, uint64_t seed, uint32_t frame,
                         const double* injected, uint8_t* payload, uint32_t* payload_len,
                         uint8_t* out, long out_pitch);

int or_pixelize_adaptive_plane(const uint8_t* img, const uint8_t* mask, int M, int N, long pitch,
                               long mask_pitch, int C, int ch, int b, int n, double sigma,
                               double sigma_sub, int noise_kind, uint64_t seed, uint32_t frame,
                               const double* injected, uint8_t* payload, uint32_t* payload_len,
                               uint8_t* out, long out_pitch) {
  return adaptive_core(img, mask, NULL, M, N, pitch, mask_pitch, C, ch, b, n, sigma, sigma_sub,
                       noise_kind, seed, frame, injected, payload, payload_len, out, out_pitch);
}

/* EXTENSION (no reference counterpart; north-star "complexity measure"):
 * cell (r, c) of the mirror-padded frame is complex iff the variance of its
 * C*b*b samples, (n*S2 - S1^2) / n^2 with exact integer sums, is >= tau.
 * Writes mask means 1.0f (simple) / 0.0f (complex) so the DPPX payload
 * classifies identically on decode. */
int or_classify_variance(const uint8_t* img, int M, int N, long pitch, int C, int b, double tau,
                         float* mm_out) {
  or_geom g;
  if (or_grid_dims(M, N, b, &g) != OR_OK || !pad_ok(&g, M, N)) return OR_INVALID;
  const long long ns = (long long)C * b * b;
  for (int r = 0; r < g.grid_rows; ++r)
    for (int c = 0; c < g.grid_cols; ++c) {
      uint64_t s1 = 0, s2 = 0;
      for (int i = r * b; i < r * b + b; ++i)
        for (int j = c * b; j < c * b + b; ++j)
          for (int k = 0; k < C; ++k) {
            const uint64_t v = PX(img, pitch, C, k, M, N, i, j);
            s1 += v;
            s2 += v * v;
          }
      const double num = (double)((long long)(ns * (long long)s2) - (long long)(s1 * s1));
      const double var = num / ((double)ns * (double)ns);
      mm_out[(size_t)r * g.grid_cols + c] = var >= tau ? 0.0f : 1.0f;
    }
  return OR_OK;
}

/* Adaptive plane with per-cell mask means supplied (e.g. by or_classify_variance). */
int or_pixelize_adaptive_plane_mm(const uint8_t* img, const float* mm, int M, int N, long pitch,
                                  int C, int ch, int b, int n, double sigma, double sigma_sub,
                                  int noise_kind, uint64_t seed, uint32_t frame,
                                  const double* injected, uint8_t* payload, uint32_t* payload_len,
                                  uint8_t* out, long out_pitch) {
  return adaptive_core(img, NULL, mm, M, N, pitch, 0, C, ch, b, n, sigma, sigma_sub, noise_kind,
                       seed, frame, injected, payload, payload_len, out, out_pitch);
}

static int adaptive_core(const uint8_t* img, const uint8_t* mask, const float* mm_in, int M, int N,
                         long pitch, long mask_pitch, int C, int ch, int b, int n, double sigma,
                         double sigma_sub, int noise_kind, uint64_t seed, uint32_t frame,
                         const double* injected, uint8_t* payload, uint32_t* payload_len,
                         uint8_t* out, long out_pitch) {
  or_geom g;
  if (n < 1 || b % n != 0) return OR_INVALID;
  if (or_grid_dims(M, N, b, &g) != OR_OK || !pad_ok(&g, M, N)) return OR_INVALID;
  if (noise_kind != OR_NOISE_NONE && noise_kind != OR_NOISE_INJECTED &&
      (!(sigma > 0.0) || !(sigma_sub > 0.0)))
    return OR_INVALID;
  const int G = g.grid_rows * g.grid_cols;
  const int sb = b / n;
  float* mm = (float*)malloc(sizeof(float) * (size_t)G);
  uint8_t* simple = (uint8_t*)malloc((size_t)G);
  if (!mm || !simple) {
    free(mm);
    free(simple);
    return OR_INVALID;
  }
  if (mm_in) {
    for (int k = 0; k < G; ++k) {
      mm[k] = mm_in[k];
      simple[k] = mm_in[k] > 0.5f ? 1 : 0;
    }
  } else {
    classify(mask, mask_pitch, M, N, &g, mm, simple);
  }
  uint32_t S = 0;
  for (int k = 0; k < G; ++k) S += simple[k];
  memcpy(payload, mm, sizeof(float) * (size_t)G); /* little-endian host */
  put_u32(payload + 4 * (size_t)G, S);
  uint8_t* simple_out = payload + 4 * (size_t)G + 4;
  uint8_t* complex_out = simple_out + S;
  or_noise nz = {noise_kind, seed, frame, (uint32_t)ch, injected, n, g.grid_cols};
  /* Sequential exclusive scan for packed slots: adaptive.cpp:123-141. */
  size_t si = 0, ci = 0;
  const double area = (double)b * b, sub_area = (double)sb * sb;
  for (int r = 0; r < g.grid_rows; ++r)
    for (int c = 0; c < g.grid_cols; ++c) {
      const size_t k = (size_t)r * g.grid_cols + c;
      if (simple[k]) { /* adaptive.cpp:147-152 */
        const double mean = (double)block_sum(img, pitch, C, ch, M, N, r * b, c * b, b) / area;
        simple_out[si++] = finalize(mean, noise_for(&nz, (uint32_t)r, (uint32_t)c, 0, 0, sigma));
      } else { /* adaptive.cpp:153-170 */
        uint8_t* o = complex_out + ci * (size_t)n * n;
        for (int sr = 0; sr < n; ++sr)
          for (int sc = 0; sc < n; ++sc) {
            const double mean =
                (double)block_sum(img, pitch, C, ch, M, N, r * b + sr * sb, c * b + sc * sb, sb) /
                sub_area;
            o[sr * n + sc] = finalize(
                mean, noise_for(&nz, (uint32_t)r, (uint32_t)c, (uint32_t)sr, (uint32_t)sc,
                                sigma_sub));
          }
        ++ci;
      }
    }
  *payload_len = (uint32_t)(4 * (size_t)G + 4 + S + ci * (size_t)n * n);
  free(mm);
  free(simple);
  if (out) {
    /* reassemble: adaptive.cpp:223-243 (walk grids, crop to M x N). */
    size_t sa = 0, ca = 0;
    for (int r = 0; r < g.grid_rows; ++r)
      for (int c = 0; c < g.grid_cols; ++c) {
        const float mean = ((const float*)payload)[(size_t)r * g.grid_cols + c];
        const int i0 = r * b, j0 = c * b;
        const int h = b < M - i0 ? b : M - i0, w = b < N - j0 ? b : N - j0;
        if (mean > 0.5f) {
          const uint8_t v = simple_out[sa++];
          for (int i = i0; i < i0 + h; ++i)
            for (int j = j0; j < j0 + w; ++j) out[(size_t)i * out_pitch + (size_t)j * C + ch] = v;
        } else {
          const uint8_t* sub = complex_out + ca++ * (size_t)n * n;
          for (int i = i0; i < i0 + h; ++i)
            for (int j = j0; j < j0 + w; ++j)
              out[(size_t)i * out_pitch + (size_t)j * C + ch] =
                  sub[((i - i0) / sb) * n + (j - j0) / sb];
        }
      }
  }
  return OR_OK;
}

/* reassemble from a DPPX adaptive payload (adaptive.cpp:181-245 plus the
 * length checks of record.cpp:241-270). Returns OR_CORRUPT on inconsistent
 * lengths or a simple count that disagrees with the mask means. */
int or_reassemble_plane(const uint8_t* payload, size_t payload_len, int M, int N, int b, int n,
                        int C, int ch, uint8_t* out, long out_pitch) {
  or_geom g;
  if (or_grid_dims(M, N, b, &g) != OR_OK) return OR_INVALID;
  if (n < 1 || b % n != 0) return OR_CORRUPT;
  const size_t G = (size_t)g.grid_rows * g.grid_cols;
  if (payload_len < 4 * G + 4) return OR_CORRUPT;
  const float* mm = (const float*)payload;
  size_t S = 0;
  for (size_t k = 0; k < G; ++k) S += mm[k] > 0.5f;
  const uint8_t* p = payload + 4 * G;
  const uint32_t stored = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
                          ((uint32_t)p[3] << 24);
  if (stored != S) return OR_CORRUPT;
  if (payload_len != 4 * G + 4 + S + (G - S) * (size_t)n * n) return OR_CORRUPT;
  const uint8_t* simple_in = payload + 4 * G + 4;
  const uint8_t* complex_in = simple_in + S;
  const int sb = b / n;
  size_t sa = 0, ca = 0;
  for (int r = 0; r < g.grid_rows; ++r)
    for (int c = 0; c < g.grid_cols; ++c) {
      const int i0 = r * b, j0 = c * b;
      const int h = b < M - i0 ? b : M - i0, w = b < N - j0 ? b : N - j0;
      if (mm[(size_t)r * g.grid_cols + c] > 0.5f) {
        const uint8_t v = simple_in[sa++];
        for (int i = i0; i < i0 + h; ++i)
          for (int j = j0; j < j0 + w; ++j) out[(size_t)i * out_pitch + (size_t)j * C + ch] = v;
      } else {
        const uint8_t* sub = complex_in + ca++ * (size_t)n * n;
        for (int i = i0; i < i0 + h; ++i)
          for (int j = j0; j < j0 + w; ++j)
            out[(size_t)i * out_pitch + (size_t)j * C + ch] = sub[((i - i0) / sb) * n + (j - j0) / sb];
      }
    }
  return OR_OK;
}

/* broadcast_means: pixelize.cpp:126-150. */
int or_broadcast_plane(const uint8_t* means, int M, int N, int b, int C, int ch, uint8_t* out,
                       long out_pitch) {
  or_geom g;
  if (or_grid_dims(M, N, b, &g) != OR_OK) return OR_INVALID;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j)
      out[(size_t)i * out_pitch + (size_t)j * C + ch] = means[(size_t)(i / b) * g.grid_cols + j / b];
  return OR_OK;
}

/* pixelize_reference (Algorithm 1, no padding, partial border grids):
 * pixelize.cpp:50-84. Gray only. */
int or_pixelize_reference(const uint8_t* img, int M, int N, int b, double sigma, int noise_kind,
                          uint64_t seed, uint8_t* out) {
  or_geom g;
  if (or_grid_dims(M, N, b, &g) != OR_OK) return OR_INVALID;
  or_noise nz = {noise_kind, seed, 0, 0, NULL, 1, g.grid_cols};
  for (int r = 0; r < g.grid_rows; ++r) {
    const int i0 = r * b, h = b < M - i0 ? b : M - i0;
    for (int c = 0; c < g.grid_cols; ++c) {
      const int j0 = c * b, w = b < N - j0 ? b : N - j0;
      uint64_t s = 0;
      for (int i = i0; i < i0 + h; ++i)
        for (int j = j0; j < j0 + w; ++j) s += img[(size_t)i * N + j];
      const double mean = (double)s / ((double)h * w);
      const uint8_t v = finalize(mean, noise_for(&nz, (uint32_t)r, (uint32_t)c, 0, 0, sigma));
      for (int i = i0; i < i0 + h; ++i)
        for (int j = j0; j < j0 + w; ++j) out[(size_t)i * N + j] = v;
    }
  }
  return OR_OK;
}

/* ---- synthetic workload (bench + tests; mirrored by the device generator) -- */

static inline uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

/* Plane k of frame f: a gradient + disc + checker pattern (in the spirit of
 * the reference's synthetic_image, tests/support/oracles.cpp:43-63) drifting
 * one column per frame, XOR a 6-bit counter-hash texture. Integer-only so the
 * device generator reproduces it bit for bit. */
uint8_t or_synth_pixel(uint32_t data_seed, uint32_t f, uint32_t k, int M, int N, int i, int j) {
  const int jj = (int)(((long long)j + f) % N);
  int v = (i + 2 * jj + 85 * (int)k) & 255;
  const long long dy = 2LL * i + 1 - M, dx = 2LL * jj + 1 - N;
  const long long rad = (M < N ? M : N) / 2; /* diameter/2 in doubled coords */
  if (dy * dy + dx * dx < rad * rad) v = 200 - 40 * (int)k;
  if (i < M / 2 && jj < N / 2 && (((i >> 3) + (jj >> 3)) & 1) == 0) v = 255 - v;
  const uint32_t h = hash32(data_seed ^ hash32(f * 0x9E3779B1u ^ hash32(k * 0x85EBCA77u ^
                                        hash32((uint32_t)i * 0xC2B2AE3Du ^ (uint32_t)j))));
  return (uint8_t)(v ^ (int)(h & 0x3F));
}

/* Mask of frame f: 1 = simple/background, 0 = complex/foreground inside a
 * centred ellipse with semi-axes 0.4*M x 0.2*N whose centre drifts +2 px per
 * frame (wrapping). */
uint8_t or_synth_mask(uint32_t f, int M, int N, int i, int j) {
  const long long ay = (4LL * M) / 5, ax = (2LL * N) / 5; /* doubled semi-axes */
  const long long cx2 = ((long long)N + 4LL * f) % (2LL * N); /* doubled centre col */
  long long dx = 2LL * j + 1 - cx2;
  if (dx > N) dx -= 2LL * N;
  if (dx < -N) dx += 2LL * N;
  const long long dy = 2LL * i + 1 - M;
  if (ay == 0 || ax == 0) return 1;
  return (dy * dy * ax * ax + dx * dx * ay * ay < ax * ax * ay * ay) ? 0 : 1;
}

void or_synth_frames(uint32_t data_seed, uint32_t f0, int F, int M, int N, int C, long pitch,
                     long frame_stride, uint8_t* dst) {
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j)
        for (int k = 0; k < C; ++k)
          dst[(size_t)f * frame_stride + (size_t)i * pitch + (size_t)j * C + k] =
              or_synth_pixel(data_seed, f0 + (uint32_t)f, (uint32_t)k, M, N, i, j);
}

void or_synth_masks(uint32_t f0, int F, int M, int N, long pitch, long frame_stride,
                    uint8_t* dst) {
  for (int f = 0; f < F; ++f)
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j)
        dst[(size_t)f * frame_stride + (size_t)i * pitch + j] =
            or_synth_mask(f0 + (uint32_t)f, M, N, i, j);
}

/* ---- utility metrics (next row) ------------------------------ */

/* mse: metrics.cpp:26-37 (exact u64 sum of squared differences, one divide). */
double or_mse(const uint8_t* a, const uint8_t* b, long n) {
  uint64_t s = 0;
  for (long i = 0; i < n; ++i) {
    const int64_t d = (int64_t)a[i] - b[i];
    s += (uint64_t)(d * d);
  }
  return (double)s / (double)n;
}

/* ssim: metrics.cpp:73-183. Window sums are exact integers (the reference's
 * summed-area tables give the same integers); the per-window f64 sequence and
 * the row-ordered accumulation follow metrics.cpp:144-182. */
double or_ssim(const uint8_t* a, const uint8_t* b, int M, int N) {
  const int W = 7;
  const double area = 49.0, c1 = 6.5025, c2 = 58.5225;
  if (M < W || N < W) return -1.0;
  const int pr = M - W + 1, pc = N - W + 1;
  double total = 0.0;
  for (int i = 0; i < pr; ++i) {
    double acc = 0.0;
    for (int j = 0; j < pc; ++j) {
      uint64_t sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
      for (int y = i; y < i + W; ++y)
        for (int x = j; x < j + W; ++x) {
          const uint64_t va = a[(size_t)y * N + x], vb = b[(size_t)y * N + x];
          sa += va;
          sb += vb;
          saa += va * va;
          sbb += vb * vb;
          sab += va * vb;
        }
      const double mu_a = (double)sa / area, mu_b = (double)sb / area;
      const double raw_aa = (double)saa / area, raw_bb = (double)sbb / area,
                   raw_ab = (double)sab / area;
      const double mu_aa = mu_a * mu_a, mu_bb = mu_b * mu_b, mu_ab = mu_a * mu_b;
      const double var_a = raw_aa - mu_aa, var_b = raw_bb - mu_bb, cov = raw_ab - mu_ab;
      const double num = (2.0 * mu_ab + c1) * (2.0 * cov + c2);
      const double den = ((mu_aa + mu_bb) + c1) * ((var_a + var_b) + c2);
      acc += num / den;
    }
    total += acc;
  }
  return total / ((double)pr * pc);
}
