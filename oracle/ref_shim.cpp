// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled where they lie by oracle/Makefile
// into oracle/_ref/libdppix_ref.so). Used to (a) pin the C restatement in
// oracle/dppx_oracle.c, (b) generate tests/golden/ fixtures, and (c) time the
// reference CPU path for bench.py's cpu_baseline / --impl reference arm.
// Nothing here is shipped or called by the product.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <zlib.h>

#include "dppix/adaptive.hpp"
#include "dppix/errors.hpp"
#include "dppix/image.hpp"
#include "dppix/metrics.hpp"
#include "dppix/noise.hpp"
#include "dppix/pixelize.hpp"
#include "dppix/record.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_GUARD(...)                                          \
  try {                                                         \
    __VA_ARGS__;                                                \
    return 0;                                                   \
  } catch (const dppix::RecordError& e) {                       \
    return fail(e, -2);                                         \
  } catch (const std::invalid_argument& e) {                    \
    return fail(e, -1);                                         \
  } catch (const std::exception& e) {                           \
    return fail(e, -3);                                         \
  }

dppix::GrayImage to_image(const uint8_t* p, int M, int N) {
  dppix::GrayImage img;
  img.height = M;
  img.width = N;
  img.pixels.assign(p, p + static_cast<size_t>(M) * N);
  return img;
}

dppix::RegionMask to_mask(const uint8_t* p, int M, int N) {
  dppix::RegionMask m;
  m.height = M;
  m.width = N;
  m.values.assign(p, p + static_cast<size_t>(M) * N);
  return m;
}

std::optional<dppix::NoiseSeed> seed_of(int has_seed, uint64_t seed) {
  if (!has_seed) return std::nullopt;
  return dppix::NoiseSeed{seed};
}

// DPPX v1 adaptive payload (record.hpp:48-54) from an AdaptiveMeans.
uint32_t serialize(const dppix::AdaptiveMeans& am, uint8_t* out) {
  size_t pos = 0;
  for (float f : am.classification.mask_means) {
    std::memcpy(out + pos, &f, 4);
    pos += 4;
  }
  const uint32_t S = static_cast<uint32_t>(am.simple_means.size());
  std::memcpy(out + pos, &S, 4);
  pos += 4;
  std::memcpy(out + pos, am.simple_means.data(), am.simple_means.size());
  pos += am.simple_means.size();
  std::memcpy(out + pos, am.complex_submeans.data(), am.complex_submeans.size());
  pos += am.complex_submeans.size();
  return static_cast<uint32_t>(pos);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_make_privacy_params(double eps, int m, int b, int n, double* out5, int* sub_side) {
  REF_GUARD({
    const dppix::PrivacyParams p = dppix::make_privacy_params(eps, m, b, n);
    out5[0] = p.epsilon;
    out5[1] = p.delta;
    out5[2] = p.sigma;
    out5[3] = p.delta_sub;
    out5[4] = p.sigma_sub;
    *sub_side = p.subgrid_side;
  });
}

int ref_grid_dims(int M, int N, int b, int* out5) {
  REF_GUARD({
    const dppix::GridGeometry g = dppix::grid_dims(M, N, b);
    out5[0] = g.b;
    out5[1] = g.grid_rows;
    out5[2] = g.grid_cols;
    out5[3] = g.pad_rows;
    out5[4] = g.pad_cols;
  });
}

uint64_t ref_keyed_bits(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc) {
  return dppix::keyed_bits(dppix::NoiseSeed{seed}, dppix::NoiseKey{r, c, sr, sc});
}

double ref_uniform_from_bits(uint64_t bits) { return dppix::uniform_from_bits(bits); }

double ref_laplace_at(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc,
                      double sigma) {
  return dppix::laplace_at(dppix::NoiseSeed{seed}, dppix::NoiseKey{r, c, sr, sc}, sigma);
}

int ref_pixelize_parallel(const uint8_t* img, int M, int N, double eps, int m, int b,
                          int has_seed, uint64_t seed, int threads, uint8_t* out_image,
                          uint8_t* out_means) {
  REF_GUARD({
    const dppix::PrivacyParams p = dppix::make_privacy_params(eps, m, b);
    const dppix::UniformResult r =
        dppix::pixelize_parallel(to_image(img, M, N), p, seed_of(has_seed, seed), threads);
    if (out_image) std::memcpy(out_image, r.image.pixels.data(), r.image.pixels.size());
    if (out_means) std::memcpy(out_means, r.means.values.data(), r.means.values.size());
  });
}

int ref_pixelize_reference(const uint8_t* img, int M, int N, double eps, int m, int b,
                           int has_seed, uint64_t seed, uint8_t* out_image) {
  REF_GUARD({
    const dppix::PrivacyParams p = dppix::make_privacy_params(eps, m, b);
    const dppix::GrayImage r =
        dppix::pixelize_reference(to_image(img, M, N), p, seed_of(has_seed, seed));
    std::memcpy(out_image, r.pixels.data(), r.pixels.size());
  });
}

int ref_pixelize_adaptive(const uint8_t* img, const uint8_t* mask, int M, int N, double eps,
                          int m, int b, int n, int has_seed, uint64_t seed, int threads,
                          uint8_t* out_image, uint8_t* out_payload, uint32_t* payload_len) {
  REF_GUARD({
    const dppix::PrivacyParams p = dppix::make_privacy_params(eps, m, b, n);
    const dppix::AdaptiveResult r = dppix::pixelize_adaptive(
        to_image(img, M, N), to_mask(mask, M, N), p, seed_of(has_seed, seed), threads);
    if (out_image) std::memcpy(out_image, r.image.pixels.data(), r.image.pixels.size());
    if (out_payload) *payload_len = serialize(r.means, out_payload);
  });
}

// reassemble over a DPPX adaptive payload, via the reference's own decode
// (record.cpp:177-278) of a freshly encoded record, then reconstruct.
int ref_reconstruct_adaptive(const uint8_t* payload, uint32_t payload_len, int M, int N, int b,
                             int n, uint8_t* out_image) {
  REF_GUARD({
    std::vector<uint8_t> rec(20);
    std::memcpy(rec.data(), "DPPX", 4);
    rec[4] = 1;
    rec[5] = 0;
    rec[6] = 2;
    rec[7] = 0;
    std::memcpy(rec.data() + 8, &M, 4);
    std::memcpy(rec.data() + 12, &N, 4);
    const uint16_t b16 = static_cast<uint16_t>(b), n16 = static_cast<uint16_t>(n);
    std::memcpy(rec.data() + 16, &b16, 2);
    std::memcpy(rec.data() + 18, &n16, 2);
    rec.insert(rec.end(), payload, payload + payload_len);
    // CRC32 (zlib, as record.cpp:35-39) over all preceding bytes.
    const uint32_t crc = static_cast<uint32_t>(::crc32(0L, rec.data(), static_cast<uInt>(rec.size())));
    rec.resize(rec.size() + 4);
    std::memcpy(rec.data() + rec.size() - 4, &crc, 4);
    const dppix::PixelRecord pr = dppix::decode(rec);
    const dppix::GrayImage img = dppix::reconstruct(pr);
    std::memcpy(out_image, img.pixels.data(), img.pixels.size());
  });
}

// Full .dppx record bytes from the reference's encode (record.cpp:124-175).
int ref_encode_adaptive(const uint8_t* img, const uint8_t* mask, int M, int N, double eps, int m,
                        int b, int n, int has_seed, uint64_t seed, uint8_t* out, uint32_t cap,
                        uint32_t* len) {
  REF_GUARD({
    const dppix::PrivacyParams p = dppix::make_privacy_params(eps, m, b, n);
    dppix::AdaptiveResult r = dppix::pixelize_adaptive(
        to_image(img, M, N), to_mask(mask, M, N), p, seed_of(has_seed, seed), 1);
    dppix::PixelRecord rec{M, N, std::move(r.means)};
    const std::vector<uint8_t> bytes = dppix::encode(rec);
    if (bytes.size() > cap) throw std::runtime_error("ref_encode_adaptive: capacity");
    std::memcpy(out, bytes.data(), bytes.size());
    *len = static_cast<uint32_t>(bytes.size());
  });
}

int ref_encode_uniform(const uint8_t* img, int M, int N, double eps, int m, int b, int has_seed,
                       uint64_t seed, uint8_t* out, uint32_t cap, uint32_t* len) {
  REF_GUARD({
    const dppix::PrivacyParams p = dppix::make_privacy_params(eps, m, b);
    dppix::UniformResult r =
        dppix::pixelize_parallel(to_image(img, M, N), p, seed_of(has_seed, seed), 1);
    dppix::PixelRecord rec{M, N, std::move(r.means)};
    const std::vector<uint8_t> bytes = dppix::encode(rec);
    if (bytes.size() > cap) throw std::runtime_error("ref_encode_uniform: capacity");
    std::memcpy(out, bytes.data(), bytes.size());
    *len = static_cast<uint32_t>(bytes.size());
  });
}

double ref_mse(const uint8_t* a, const uint8_t* b, int M, int N) {
  try {
    return dppix::mse(to_image(a, M, N), to_image(b, M, N));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

double ref_ssim(const uint8_t* a, const uint8_t* b, int M, int N, int threads) {
  try {
    return dppix::ssim(to_image(a, M, N), to_image(b, M, N), threads);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// CPU baseline timing: `planes` gray planes (already de-interleaved upstream,
// as SPEC.md:92 prescribes for color) run through pixelize_adaptive (n >= 1)
// or pixelize_parallel (uniform=1), file-parallel over `workers` std::threads
// with threads=1 inside each call -- run_batch's scheme (cli.cpp:175-213)
// without its nested oversubscription. Only the pixelize calls are timed
// (cli.cpp:108-130). Returns wall seconds, or a negative value on error.
double ref_time_planes(const uint8_t* planes, const uint8_t* masks, int n_planes, int M, int N,
                       int uniform, double eps, int m, int b, int n, uint64_t seed,
                       int workers) {
  try {
    const size_t plane_bytes = static_cast<size_t>(M) * N;
    std::vector<dppix::GrayImage> imgs(n_planes);
    std::vector<dppix::RegionMask> msk(uniform ? 0 : n_planes);
    for (int i = 0; i < n_planes; ++i) {
      imgs[i] = to_image(planes + i * plane_bytes, M, N);
      if (!uniform) msk[i] = to_mask(masks + i * plane_bytes, M, N);
    }
    const dppix::PrivacyParams p = dppix::make_privacy_params(eps, m, b, uniform ? 1 : n);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    std::vector<int> bad(workers, 0);
    for (int w = 0; w < workers; ++w) {
      pool.emplace_back([&, w] {
        try {
          for (int i = w; i < n_planes; i += workers) {
            if (uniform) {
              volatile auto r = dppix::pixelize_parallel(imgs[i], p, dppix::NoiseSeed{seed}, 1)
                                    .means.values.size();
              (void)r;
            } else {
              volatile auto r =
                  dppix::pixelize_adaptive(imgs[i], msk[i], p, dppix::NoiseSeed{seed}, 1)
                      .means.simple_means.size();
              (void)r;
            }
          }
        } catch (...) {
          bad[w] = 1;
        }
      });
    }
    for (auto& t : pool) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    for (int v : bad)
      if (v) return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

}  // extern "C"
