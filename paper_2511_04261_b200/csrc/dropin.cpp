// dropin.cpp -- the reference's dppix:: C++ API (include/dppix/*.hpp) over the
// C ABI of libdppx_gpu.so. Callers written against /root/reference/proj/include
// (run_single-style code, the reference's own unit tests) link this library
// instead of libdppix.a. Pixelization, classification, broadcast and
// reassembly run on the GPU; a missing or unusable device raises
// std::runtime_error (there is no CPU fallback).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "dppix/adaptive.hpp"
#include "dppix/errors.hpp"
#include "dppix/image.hpp"
#include "dppix/metrics.hpp"
#include "dppix/noise.hpp"
#include "dppix/pixelize.hpp"
#include "dppix/record.hpp"
#include "dppx_gpu.h"

namespace dppix {
namespace {

struct CtxDeleter {
  void operator()(dppx_ctx* c) const { dppx_ctx_destroy(c); }
};

// One context per host thread: the reference functions are reentrant and may
// be called concurrently; a dppx_ctx is single-threaded.
dppx_ctx* thread_ctx() {
  thread_local std::unique_ptr<dppx_ctx, CtxDeleter> ctx;
  if (!ctx) {
    int device = 0;
    if (const char* env = std::getenv("DPPX_DEVICE")) device = std::atoi(env);
    dppx_ctx* c = nullptr;
    const int rc = dppx_ctx_create(device, &c);
    if (rc != DPPX_OK)
      throw std::runtime_error("dppix: no usable sm_100 GPU for the pixelization path (status " +
                               std::to_string(rc) + ")");
    ctx.reset(c);
  }
  return ctx.get();
}

[[noreturn]] void raise(int rc, const char* who) {
  const std::string msg = std::string(who) + ": " + dppx_ctx_last_error(thread_ctx());
  switch (rc) {
    case DPPX_ERR_INVALID:
      throw std::invalid_argument(msg);
    case DPPX_ERR_CORRUPT:
      throw RecordError(RecordErrorKind::corrupt_record, msg);
    case DPPX_ERR_OOM:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(msg);
  }
}

void check(int rc, const char* who) {
  if (rc != DPPX_OK) raise(rc, who);
}

dppx_frames_desc gray_desc(int M, int N) {
  dppx_frames_desc d{};
  d.height = M;
  d.width = N;
  d.channels = 1;
  d.frames = 1;
  d.pitch = d.mask_pitch = d.out_pitch = N;
  d.frame_stride = d.mask_frame_stride = d.out_frame_stride = static_cast<int64_t>(M) * N;
  return d;
}

dppx_privacy_params to_c(const PrivacyParams& p) {
  dppx_privacy_params c{};
  c.epsilon = p.epsilon;
  c.m = p.m;
  c.b = p.b;
  c.n = p.n;
  c.subgrid_side = p.subgrid_side;
  c.delta = p.delta;
  c.sigma = p.sigma;
  c.delta_sub = p.delta_sub;
  c.sigma_sub = p.sigma_sub;
  return c;
}

void check_image(const GrayImage& img, const char* who) {  // pixelize.cpp:40-46
  if (img.height < 1 || img.width < 1 ||
      img.pixels.size() != static_cast<std::size_t>(img.height) * img.width)
    throw std::invalid_argument(std::string(who) + ": malformed image");
}

template <typename T>
std::vector<T> mirror_pad_impl(const std::vector<T>& src, int h, int w, const GridGeometry& g) {
  if (g.b < 1 || g.padded_height() != h + g.pad_rows || g.padded_width() != w + g.pad_cols ||
      g.pad_rows < 0 || g.pad_rows >= g.b || g.pad_cols < 0 || g.pad_cols >= g.b)
    throw std::invalid_argument("mirror_pad: geometry does not match image dimensions");
  if (g.pad_rows >= h || g.pad_cols >= w)
    throw std::invalid_argument("mirror_pad: padding exceeds image size (use b <= min(M, N))");
  const int oh = g.padded_height(), ow = g.padded_width();
  std::vector<T> out(static_cast<std::size_t>(oh) * ow);
  for (int i = 0; i < oh; ++i) {
    const int si = i < h ? i : h - 1 - (i - h);
    for (int j = 0; j < ow; ++j) {
      const int sj = j < w ? j : w - 1 - (j - w);
      out[static_cast<std::size_t>(i) * ow + j] = src[static_cast<std::size_t>(si) * w + sj];
    }
  }
  return out;
}

template <typename T>
std::uint64_t tile_sum(const std::vector<T>& data, int stride, const GridGeometry& g, int r,
                       int c, const char* who) {
  if (r < 0 || r >= g.grid_rows || c < 0 || c >= g.grid_cols)
    throw std::invalid_argument(std::string(who) + ": grid index out of range");
  std::uint64_t s = 0;
  for (int i = r * g.b; i < (r + 1) * g.b; ++i)
    for (int j = c * g.b; j < (c + 1) * g.b; ++j) s += data[static_cast<std::size_t>(i) * stride + j];
  return s;
}

}  // namespace

dppx_ctx* dropin_thread_ctx() { return thread_ctx(); }  // used by runner.cpp

// ---------------------------------------------------------------- image.hpp
GrayImage make_image(int height, int width, std::uint8_t fill) {
  if (height < 1 || width < 1) throw std::invalid_argument("make_image: dimensions must be >= 1");
  GrayImage img;
  img.height = height;
  img.width = width;
  img.pixels.assign(static_cast<std::size_t>(height) * width, fill);
  return img;
}

RegionMask make_mask(int height, int width, std::uint8_t fill) {
  if (height < 1 || width < 1) throw std::invalid_argument("make_mask: dimensions must be >= 1");
  if (fill > 1) throw std::invalid_argument("make_mask: mask values must be 0 or 1");
  RegionMask m;
  m.height = height;
  m.width = width;
  m.values.assign(static_cast<std::size_t>(height) * width, fill);
  return m;
}

GridGeometry grid_dims(int height, int width, int b) {
  if (height < 1 || width < 1) throw std::invalid_argument("grid_dims: dimensions must be >= 1");
  if (b < 1) throw std::invalid_argument("grid_dims: grid side b must be >= 1");
  dppx_geometry g;
  if (dppx_grid_dims(height, width, b, &g) != DPPX_OK)
    throw std::invalid_argument("grid_dims: grid side b exceeds both image dimensions");
  return GridGeometry{g.b, g.grid_rows, g.grid_cols, g.pad_rows, g.pad_cols};
}

GrayImage mirror_pad(const GrayImage& img, const GridGeometry& g) {
  GrayImage out;
  out.pixels = mirror_pad_impl(img.pixels, img.height, img.width, g);
  out.height = g.padded_height();
  out.width = g.padded_width();
  return out;
}

RegionMask mirror_pad(const RegionMask& mask, const GridGeometry& g) {
  RegionMask out;
  out.values = mirror_pad_impl(mask.values, mask.height, mask.width, g);
  out.height = g.padded_height();
  out.width = g.padded_width();
  return out;
}

GrayImage crop(const GrayImage& img, int height, int width) {
  if (height < 1 || width < 1 || height > img.height || width > img.width)
    throw std::invalid_argument("crop: target size out of range");
  GrayImage out = make_image(height, width);
  for (int i = 0; i < height; ++i) std::memcpy(out.row(i), img.row(i), static_cast<std::size_t>(width));
  return out;
}

std::uint64_t grid_sum(const GrayImage& padded, const GridGeometry& g, int r, int c) {
  if (padded.height != g.padded_height() || padded.width != g.padded_width())
    throw std::invalid_argument("grid_sum: image is not padded to geometry");
  return tile_sum(padded.pixels, padded.width, g, r, c, "grid_sum");
}

double grid_mean(const GrayImage& padded, const GridGeometry& g, int r, int c) {
  return static_cast<double>(grid_sum(padded, g, r, c)) / (static_cast<double>(g.b) * g.b);
}

double mask_grid_mean(const RegionMask& padded, const GridGeometry& g, int r, int c) {
  if (padded.height != g.padded_height() || padded.width != g.padded_width())
    throw std::invalid_argument("mask_grid_mean: mask is not padded to geometry");
  return static_cast<double>(tile_sum(padded.values, padded.width, g, r, c, "mask_grid_mean")) /
         (static_cast<double>(g.b) * g.b);
}

// ---------------------------------------------------------------- noise.hpp
double sensitivity(int b, int m) {
  if (b < 1 || m < 1) throw std::invalid_argument("sensitivity: b and m must be >= 1");
  return dppx_sensitivity(b, m);
}

double noise_scale(double delta, double epsilon) {
  if (!(epsilon > 0.0)) throw std::invalid_argument("noise_scale: epsilon must be > 0");
  if (!(delta > 0.0)) throw std::invalid_argument("noise_scale: delta must be > 0");
  return delta / epsilon;
}

PrivacyParams make_privacy_params(double epsilon, int m, int b, int n) {
  if (!(epsilon > 0.0)) throw std::invalid_argument("make_privacy_params: epsilon must be > 0");
  if (m < 1) throw std::invalid_argument("make_privacy_params: m must be >= 1");
  if (b < 1) throw std::invalid_argument("make_privacy_params: b must be >= 1");
  if (n < 1) throw std::invalid_argument("make_privacy_params: n must be >= 1");
  if (b % n != 0) throw std::invalid_argument("make_privacy_params: n must divide b");
  dppx_privacy_params c;
  dppx_make_privacy_params(epsilon, m, b, n, &c);
  PrivacyParams p;
  p.epsilon = c.epsilon;
  p.m = c.m;
  p.b = c.b;
  p.n = c.n;
  p.subgrid_side = c.subgrid_side;
  p.delta = c.delta;
  p.sigma = c.sigma;
  p.delta_sub = c.delta_sub;
  p.sigma_sub = c.sigma_sub;
  return p;
}

double subgrid_sensitivity(const PrivacyParams& p) { return sensitivity(p.subgrid_side, p.m); }

std::uint64_t keyed_bits(NoiseSeed seed, const NoiseKey& k) {
  return dppx_keyed_bits(seed.value, k.r, k.c, k.sr, k.sc);
}

double uniform_from_bits(std::uint64_t bits) { return dppx_uniform_from_bits(bits); }

double laplace_from_uniform(double u, double sigma) {
  const double sign = u < 0.0 ? -1.0 : 1.0;
  return sign * sigma * -std::log1p(-2.0 * std::abs(u));
}

double laplace_at(NoiseSeed seed, const NoiseKey& k, double sigma) {
  if (!(sigma > 0.0)) throw std::invalid_argument("laplace_at: sigma must be > 0");
  return laplace_from_uniform(uniform_from_bits(keyed_bits(seed, k)), sigma);
}

// ------------------------------------------------------------- pixelize.hpp
double clip_intensity(double v) { return v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v); }

std::uint8_t quantize_intensity(double v) { return static_cast<std::uint8_t>(std::llround(v)); }

UniformResult pixelize_parallel(const GrayImage& img, const PrivacyParams& params,
                                const std::optional<NoiseSeed>& seed, int /*threads*/) {
  check_image(img, "pixelize_parallel");
  if (params.n != 1) throw std::invalid_argument("pixelize_parallel: requires n == 1");
  const GridGeometry geom = grid_dims(img.height, img.width, params.b);
  UniformResult res;
  res.image = make_image(img.height, img.width);
  res.means.geometry = geom;
  res.means.values.resize(geom.grid_count());
  const dppx_frames_desc d = gray_desc(img.height, img.width);
  const dppx_privacy_params p = to_c(params);
  const std::uint64_t s = seed ? seed->value : 0;
  dppx_noise nz{seed ? DPPX_NOISE_KEYED : DPPX_NOISE_NONE, 0, &s, nullptr};
  check(dppx_pixelize_uniform(thread_ctx(), &d, img.pixels.data(), &p, &nz,
                              res.means.values.data(), res.image.pixels.data()),
        "pixelize_parallel");
  return res;
}

GrayImage pixelize_reference(const GrayImage& img, const PrivacyParams& params,
                             const std::optional<NoiseSeed>& seed) {
  check_image(img, "pixelize_reference");
  if (params.n != 1) throw std::invalid_argument("pixelize_reference: requires n == 1");
  const GridGeometry geom = grid_dims(img.height, img.width, params.b);
  GrayImage out = make_image(img.height, img.width);
  std::vector<std::uint8_t> means(geom.grid_count());
  const dppx_frames_desc d = gray_desc(img.height, img.width);
  const dppx_privacy_params p = to_c(params);
  const std::uint64_t s = seed ? seed->value : 0;
  dppx_noise nz{seed ? DPPX_NOISE_KEYED : DPPX_NOISE_NONE, 0, &s, nullptr};
  check(dppx_pixelize_reference(thread_ctx(), &d, img.pixels.data(), &p, &nz, means.data(),
                                out.pixels.data()),
        "pixelize_reference");
  return out;
}

GrayImage broadcast_means(const GridMeans& means, int height, int width) {
  if (height < 1 || width < 1) throw std::invalid_argument("broadcast_means: dimensions must be >= 1");
  const GridGeometry expected = grid_dims(height, width, means.geometry.b);
  if (means.geometry != expected ||
      means.values.size() != static_cast<std::size_t>(expected.grid_count()))
    throw std::invalid_argument("broadcast_means: means do not fit the target dimensions");
  GrayImage out = make_image(height, width);
  const dppx_frames_desc d = gray_desc(height, width);
  check(dppx_broadcast_means(thread_ctx(), &d, means.values.data(), means.geometry.b,
                             out.pixels.data()),
        "broadcast_means");
  return out;
}

// ------------------------------------------------------------- adaptive.hpp
int RegionClassification::simple_count() const {
  int s = 0;
  for (std::uint8_t v : is_simple) s += v == 1;
  return s;
}

bool simple_from_mean(float mask_mean) { return mask_mean > 0.5f; }

RegionClassification classify_regions(const RegionMask& mask, const GridGeometry& geom) {
  if (mask.height < 1 || mask.width < 1 ||
      mask.values.size() != static_cast<std::size_t>(mask.height) * mask.width)
    throw std::invalid_argument("classify_regions: malformed mask");
  if (geom != grid_dims(mask.height, mask.width, geom.b))
    throw std::invalid_argument("classify_regions: geometry does not match mask dimensions");
  RegionClassification cls;
  cls.geometry = geom;
  cls.mask_means.resize(geom.grid_count());
  const dppx_frames_desc d = gray_desc(mask.height, mask.width);
  check(dppx_classify_regions(thread_ctx(), &d, mask.values.data(), geom.b, cls.mask_means.data()),
        "classify_regions");
  cls.is_simple.resize(geom.grid_count());
  for (std::size_t g = 0; g < cls.mask_means.size(); ++g)
    cls.is_simple[g] = simple_from_mean(cls.mask_means[g]) ? 1 : 0;
  return cls;
}

namespace {

// Parse one DPPX adaptive payload (record.hpp:52-54) into AdaptiveMeans.
void parse_payload(const std::uint8_t* p, const GridGeometry& geom, int n, AdaptiveMeans* out) {
  const std::size_t G = geom.grid_count();
  out->geometry = geom;
  out->n = n;
  out->classification.geometry = geom;
  out->classification.mask_means.resize(G);
  std::memcpy(out->classification.mask_means.data(), p, 4 * G);
  out->classification.is_simple.resize(G);
  for (std::size_t g = 0; g < G; ++g)
    out->classification.is_simple[g] = simple_from_mean(out->classification.mask_means[g]) ? 1 : 0;
  std::uint32_t S;
  std::memcpy(&S, p + 4 * G, 4);
  const std::uint8_t* sm = p + 4 * G + 4;
  out->simple_means.assign(sm, sm + S);
  out->complex_submeans.assign(sm + S, sm + S + (G - S) * static_cast<std::size_t>(n) * n);
}

}  // namespace

AdaptiveResult pixelize_adaptive(const GrayImage& img, const RegionMask& mask,
                                 const PrivacyParams& params,
                                 const std::optional<NoiseSeed>& seed, int /*threads*/) {
  check_image(img, "pixelize_adaptive");
  if (mask.height != img.height || mask.width != img.width)
    throw std::invalid_argument("pixelize_adaptive: mask dimensions do not match image");
  if (mask.values.size() != static_cast<std::size_t>(mask.height) * mask.width)
    throw std::invalid_argument("classify_regions: malformed mask");
  if (params.n < 1 || params.b % params.n != 0 || params.subgrid_side * params.n != params.b)
    throw std::invalid_argument("pixelize_adaptive: invalid subgrid factor");
  const GridGeometry geom = grid_dims(img.height, img.width, params.b);
  const std::size_t cap = dppx_adaptive_payload_capacity(img.height, img.width, params.b, params.n);
  std::vector<std::uint8_t> payload((cap + 3) & ~static_cast<std::size_t>(3));
  std::uint32_t len = 0;
  AdaptiveResult res;
  res.image = make_image(img.height, img.width);
  const dppx_frames_desc d = gray_desc(img.height, img.width);
  const dppx_privacy_params p = to_c(params);
  const std::uint64_t s = seed ? seed->value : 0;
  dppx_noise nz{seed ? DPPX_NOISE_KEYED : DPPX_NOISE_NONE, 0, &s, nullptr};
  check(dppx_pixelize_adaptive(thread_ctx(), &d, img.pixels.data(), mask.values.data(), &p, &nz,
                               payload.data(), static_cast<int64_t>(payload.size()), &len,
                               res.image.pixels.data()),
        "pixelize_adaptive");
  parse_payload(payload.data(), geom, params.n, &res.means);
  return res;
}

GrayImage reassemble(const AdaptiveMeans& means, int height, int width) {
  if (height < 1 || width < 1) throw std::invalid_argument("reassemble: dimensions must be >= 1");
  const GridGeometry geom = means.geometry;
  if (geom != grid_dims(height, width, geom.b))
    throw std::invalid_argument("reassemble: geometry does not match the target dimensions");
  const int n = means.n;
  if (n < 1 || geom.b % n != 0)
    throw RecordError(RecordErrorKind::corrupt_record,
                      "reassemble: subgrid factor does not divide grid side");
  const std::size_t G = geom.grid_count();
  const RegionClassification& cls = means.classification;
  if (cls.geometry != geom || cls.mask_means.size() != G || cls.is_simple.size() != G)
    throw RecordError(RecordErrorKind::corrupt_record, "reassemble: classification length mismatch");
  const std::size_t S = static_cast<std::size_t>(cls.simple_count());
  if (means.simple_means.size() != S ||
      means.complex_submeans.size() != (G - S) * static_cast<std::size_t>(n) * n)
    throw RecordError(RecordErrorKind::corrupt_record, "reassemble: mean array length mismatch");
  // Wire payload whose mask means classify exactly like is_simple (the
  // reference walks is_simple, adaptive.cpp:223-243).
  std::vector<std::uint8_t> payload(((4 * G + 4 + S + (G - S) * n * n) + 3) & ~std::size_t{3});
  for (std::size_t g = 0; g < G; ++g) {
    float mm = cls.mask_means[g];
    if (simple_from_mean(mm) != (cls.is_simple[g] != 0)) mm = cls.is_simple[g] ? 1.0f : 0.0f;
    std::memcpy(payload.data() + 4 * g, &mm, 4);
  }
  const std::uint32_t S32 = static_cast<std::uint32_t>(S);
  std::memcpy(payload.data() + 4 * G, &S32, 4);
  std::memcpy(payload.data() + 4 * G + 4, means.simple_means.data(), S);
  std::memcpy(payload.data() + 4 * G + 4 + S, means.complex_submeans.data(),
              means.complex_submeans.size());
  GrayImage out = make_image(height, width);
  const dppx_frames_desc d = gray_desc(height, width);
  const std::uint32_t len = static_cast<std::uint32_t>(4 * G + 4 + S + (G - S) * n * n);
  check(dppx_reassemble(thread_ctx(), &d, payload.data(), static_cast<int64_t>(payload.size()), &len,
                        geom.b, n, out.pixels.data()),
        "reassemble");
  return out;
}

// --------------------------------------------------------------- record.hpp
RecordMode PixelRecord::mode() const {
  return std::holds_alternative<GridMeans>(payload) ? RecordMode::uniform : RecordMode::adaptive;
}

int PixelRecord::grid_side() const {
  return std::holds_alternative<GridMeans>(payload) ? std::get<GridMeans>(payload).geometry.b
                                                    : std::get<AdaptiveMeans>(payload).geometry.b;
}

int PixelRecord::subgrid_factor() const {
  return std::holds_alternative<GridMeans>(payload) ? 1 : std::get<AdaptiveMeans>(payload).n;
}

std::vector<std::uint8_t> encode(const PixelRecord& record) {
  const int b = record.grid_side(), n = record.subgrid_factor();
  if (record.height < 1 || record.width < 1)
    throw std::invalid_argument("encode: dimensions must be >= 1");
  if (b < 1 || b > std::max(record.height, record.width))
    throw std::invalid_argument("encode: invalid grid side");
  if (n < 1 || b % n != 0) throw std::invalid_argument("encode: subgrid factor must divide grid side");
  const GridGeometry geom = grid_dims(record.height, record.width, b);
  const std::size_t G = geom.grid_count();
  std::vector<std::uint8_t> payload;
  if (const GridMeans* u = std::get_if<GridMeans>(&record.payload)) {  // record.cpp:143-147
    if (u->geometry != geom || u->values.size() != G)
      throw std::invalid_argument("encode: uniform payload length mismatch");
    payload = u->values;
  } else {  // record.cpp:148-171
    const AdaptiveMeans& am = std::get<AdaptiveMeans>(record.payload);
    const RegionClassification& cls = am.classification;
    const std::size_t S = static_cast<std::size_t>(cls.simple_count());
    if (am.geometry != geom || cls.geometry != geom || cls.mask_means.size() != G ||
        cls.is_simple.size() != G || am.simple_means.size() != S ||
        am.complex_submeans.size() != (G - S) * static_cast<std::size_t>(n) * n)
      throw std::invalid_argument("encode: adaptive payload length mismatch");
    for (std::size_t g = 0; g < G; ++g)
      if ((cls.is_simple[g] != 0) != simple_from_mean(cls.mask_means[g]))
        throw std::invalid_argument("encode: classification disagrees with mask means");
    payload.resize(4 * G + 4);
    std::memcpy(payload.data(), cls.mask_means.data(), 4 * G);
    const std::uint32_t S32 = static_cast<std::uint32_t>(S);
    std::memcpy(payload.data() + 4 * G, &S32, 4);
    payload.insert(payload.end(), am.simple_means.begin(), am.simple_means.end());
    payload.insert(payload.end(), am.complex_submeans.begin(), am.complex_submeans.end());
  }
  std::vector<std::uint8_t> out(dppx_record_size(payload.size()));
  std::size_t len = 0;
  if (dppx_encode_record(record.height, record.width, b, n, static_cast<int>(record.mode()),
                         payload.data(), payload.size(), out.data(), out.size(), &len) != DPPX_OK)
    throw std::invalid_argument("encode: payload inconsistent with header fields");
  out.resize(len);
  return out;
}

PixelRecord decode(const std::vector<std::uint8_t>& bytes) {
  dppx_record_info info{};
  switch (dppx_decode_record(bytes.data(), bytes.size(), &info)) {
    case DPPX_OK:
      break;
    case DPPX_ERR_NOT_A_RECORD:
      throw RecordError(RecordErrorKind::not_a_record, "decode: missing DPPX magic");
    case DPPX_ERR_CORRUPTION:
      throw RecordError(RecordErrorKind::corruption, "decode: CRC mismatch");
    case DPPX_ERR_UNSUPPORTED_VERSION:
      throw RecordError(RecordErrorKind::unsupported_version, "decode: unsupported format version");
    default:
      throw RecordError(RecordErrorKind::corrupt_record, "decode: inconsistent record");
  }
  PixelRecord rec;
  rec.height = info.height;
  rec.width = info.width;
  const GridGeometry geom = grid_dims(info.height, info.width, info.b);
  const std::uint8_t* p = bytes.data() + info.payload_offset;
  if (info.mode == 1) {
    GridMeans m;
    m.geometry = geom;
    m.values.assign(p, p + info.payload_len);
    rec.payload = std::move(m);
  } else {
    AdaptiveMeans am;
    parse_payload(p, geom, info.n, &am);
    rec.payload = std::move(am);
  }
  return rec;
}

GrayImage reconstruct(const PixelRecord& record) {  // record.cpp:280-286
  if (const GridMeans* u = std::get_if<GridMeans>(&record.payload))
    return broadcast_means(*u, record.height, record.width);
  return reassemble(std::get<AdaptiveMeans>(record.payload), record.height, record.width);
}

PixelRecord read_record(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("read_record: cannot open " + path);
  std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(in)),
                                  std::istreambuf_iterator<char>());
  if (in.bad()) throw IoError("read_record: read failed for " + path);
  return decode(bytes);
}

void write_record(const PixelRecord& record, const std::string& path) {
  const std::vector<std::uint8_t> bytes = encode(record);
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("write_record: cannot open " + path);
  out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
  out.flush();
  if (!out) throw IoError("write_record: write failed for " + path);
}

// -------------------------------------------------------------- metrics.hpp
namespace {
double metric(const GrayImage& a, const GrayImage& b, bool ssim_metric) {
  const char* who = ssim_metric ? "ssim" : "mse";
  if (!a.same_dims(b) || a.height < 1 || a.width < 1)
    throw std::invalid_argument(std::string(who) +
                                (ssim_metric ? ": images must share dimensions"
                                             : ": images must share valid dimensions"));
  if (ssim_metric && (a.height < 7 || a.width < 7))
    throw std::invalid_argument("ssim: images smaller than the 7x7 window");
  dppx_frames_desc d = gray_desc(a.height, a.width);
  double out = 0.0;
  const int rc = ssim_metric ? dppx_ssim(thread_ctx(), &d, a.pixels.data(), b.pixels.data(), &out)
                             : dppx_mse(thread_ctx(), &d, a.pixels.data(), b.pixels.data(), &out);
  check(rc, who);
  return out;
}
}  // namespace

double mse(const GrayImage& a, const GrayImage& b) { return metric(a, b, false); }

double ssim(const GrayImage& a, const GrayImage& b, int /*threads*/) { return metric(a, b, true); }

std::string format_double(double value) {  // metrics.cpp:185-194 semantics
  char buf[40];
  for (const int precision : {15, 16, 17}) {
    std::snprintf(buf, sizeof(buf), "%.*g", precision, value);
    if (std::strtod(buf, nullptr) == value) break;
  }
  return buf;
}

std::string csv_header() { return "epsilon,m,b,n,seed,mse,ssim,runtime_ms,record_bytes"; }

std::string csv_row(const MetricReport& r) {
  return format_double(r.epsilon) + ',' + std::to_string(r.m) + ',' + std::to_string(r.b) + ',' +
         std::to_string(r.n) + ',' + std::to_string(r.seed) + ',' + format_double(r.mse) + ',' +
         format_double(r.ssim) + ',' + format_double(r.runtime_ms) + ',' +
         std::to_string(r.record_bytes);
}

}  // namespace dppix
