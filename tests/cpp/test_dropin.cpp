// test_dropin.cpp -- the reference's own unit-test cases (proj/tests/test_*.cpp),
// restated against the GPU drop-in (include/dppix/*.hpp, libdppix_gpu.so):
// a caller written for libdppix.a compiles unchanged and gets the same answers.
// Exit status 0 iff every check passes (run by tests/test_gpu_dropin.py).
#include <algorithm>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>

#include "dppix/adaptive.hpp"
#include "dppix/errors.hpp"
#include "dppix/image.hpp"
#include "dppix/noise.hpp"
#include "dppix/pixelize.hpp"
#include "dppix/batch.hpp"
#include "dppix/metrics.hpp"
#include "dppix/pgm.hpp"
#include "dppix/record.hpp"

using namespace dppix;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (cond) {                                                             \
      ++g_pass;                                                             \
    } else {                                                                \
      ++g_fail;                                                             \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
    }                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, T)      \
  do {                                \
    bool thrown_ = false;             \
    try {                             \
      (void)(expr);                   \
    } catch (const T&) {              \
      thrown_ = true;                 \
    } catch (...) {                   \
    }                                 \
    CHECK(thrown_ && #T);             \
  } while (0)

static GrayImage random_image(std::mt19937_64& rng, int h, int w) {
  GrayImage img = make_image(h, w);
  for (auto& p : img.pixels) p = static_cast<std::uint8_t>(rng() & 255);
  return img;
}

static RegionMask random_mask(std::mt19937_64& rng, int h, int w) {
  RegionMask m = make_mask(h, w);
  for (auto& v : m.values) v = static_cast<std::uint8_t>(rng() & 1);
  return m;
}

static bool piecewise_constant(const GrayImage& img, int b) {
  for (int i = 0; i < img.height; ++i)
    for (int j = 0; j < img.width; ++j)
      if (img.at(i, j) != img.at(i - i % b, j - j % b)) return false;
  return true;
}

int main() {
  const std::optional<NoiseSeed> none;
  // test_noise.cpp:29-63 -- exact calibration values.
  CHECK(sensitivity(16, 16) == 15.9375);
  CHECK(sensitivity(32, 32) == 7.96875);
  CHECK(noise_scale(15.9375, 0.5) == 31.875);
  {
    const PrivacyParams p = make_privacy_params(0.5, 16, 16, 4);
    CHECK(p.subgrid_side == 4 && p.sigma == 31.875 && p.sigma_sub == p.sigma * 16.0);
    CHECK_THROWS_AS(make_privacy_params(1.0, 1, 4, 3), std::invalid_argument);
  }
  // test_pixelize.cpp:53-90 -- quantization and KATs.
  CHECK(quantize_intensity(127.5) == 128 && quantize_intensity(2.5) == 3 &&
        quantize_intensity(2.49) == 2);
  CHECK(clip_intensity(-5.0) == 0.0 && clip_intensity(300.0) == 255.0);
  {
    GrayImage img = make_image(2, 2);
    img.pixels = {0, 0, 255, 255};
    const UniformResult r = pixelize_parallel(img, make_privacy_params(1.0, 1, 2), none);
    for (auto px : r.image.pixels) CHECK(px == 128);
  }
  {
    GrayImage img = make_image(4, 4);
    std::iota(img.pixels.begin(), img.pixels.end(), std::uint8_t{0});
    const UniformResult r = pixelize_parallel(img, make_privacy_params(1.0, 1, 2), none);
    CHECK((r.means.values == std::vector<std::uint8_t>{3, 5, 11, 13}));
    GrayImage expected = make_image(4, 4);
    expected.pixels = {3, 3, 5, 5, 3, 3, 5, 5, 11, 11, 13, 13, 11, 11, 13, 13};
    CHECK(r.image == expected);
    const AdaptiveResult a =
        pixelize_adaptive(img, make_mask(4, 4, 0), make_privacy_params(1.0, 1, 4, 2), none);
    CHECK(a.means.simple_means.empty());
    CHECK((a.means.complex_submeans == std::vector<std::uint8_t>{3, 5, 11, 13}));
    CHECK(a.image == expected);
  }
  // Algorithm 1 == Algorithm 2 when grids tile the image (test_pixelize.cpp:92-106)
  {
    std::mt19937_64 rng(21);
    for (int round = 0; round < 15; ++round) {
      const int b = 1 << (rng() % 4);
      const int h = b * (1 + static_cast<int>(rng() % 12)), w = b * (1 + static_cast<int>(rng() % 12));
      const GrayImage img = random_image(rng, h, w);
      const PrivacyParams p = make_privacy_params(0.5, 16, b);
      const std::optional<NoiseSeed> seed = NoiseSeed{rng()};
      CHECK(pixelize_reference(img, p, seed) == pixelize_parallel(img, p, seed).image);
    }
  }
  // constant image is a fixed point (test_pixelize.cpp:127-135)
  for (int b : {2, 3, 5}) {
    const GrayImage img = make_image(11, 13, 77);
    CHECK(pixelize_parallel(img, make_privacy_params(1.0, 1, b), none).image == img);
  }
  // noisy output piecewise constant (test_pixelize.cpp:151-165)
  {
    std::mt19937_64 rng(24);
    for (int round = 0; round < 10; ++round) {
      const int h = 9 + static_cast<int>(rng() % 40), w = 9 + static_cast<int>(rng() % 40);
      const int b = 2 + static_cast<int>(rng() % 7);
      const GrayImage img = random_image(rng, h, w);
      const UniformResult r =
          pixelize_parallel(img, make_privacy_params(0.1, 16, b), NoiseSeed{rng()});
      CHECK(piecewise_constant(r.image, b));
    }
  }
  // thread count never changes the result (test_pixelize.cpp:194-207)
  {
    std::mt19937_64 rng(26);
    const GrayImage img = random_image(rng, 45, 37);
    const PrivacyParams p = make_privacy_params(0.5, 16, 8);
    const UniformResult one = pixelize_parallel(img, p, NoiseSeed{99}, 1);
    const UniformResult many = pixelize_parallel(img, p, NoiseSeed{99}, 16);
    CHECK(one.image == many.image && one.means == many.means);
  }
  // broadcast_means KATs + errors (test_pixelize.cpp:209-235)
  {
    GridMeans cropped;
    cropped.geometry = grid_dims(3, 3, 2);
    cropped.values = {1, 2, 3, 4};
    GrayImage e = make_image(3, 3);
    e.pixels = {1, 1, 2, 1, 1, 2, 3, 3, 4};
    CHECK(broadcast_means(cropped, 3, 3) == e);
    CHECK_THROWS_AS(broadcast_means(cropped, 9, 9), std::invalid_argument);
    GridMeans short_values = cropped;
    short_values.values = {1, 2, 3};
    CHECK_THROWS_AS(broadcast_means(short_values, 3, 3), std::invalid_argument);
  }
  CHECK_THROWS_AS(pixelize_parallel(make_image(8, 8), make_privacy_params(1.0, 1, 4, 2), none),
                  std::invalid_argument);
  // classification tie -> complex (test_adaptive.cpp:44-67)
  {
    RegionMask half = make_mask(2, 2, 0);
    half.at(0, 0) = 1;
    half.at(0, 1) = 1;
    const RegionClassification tie = classify_regions(half, grid_dims(2, 2, 2));
    CHECK(tie.mask_means[0] == 0.5f && tie.is_simple[0] == 0);
    CHECK(classify_regions(make_mask(4, 4, 1), grid_dims(4, 4, 2)).simple_count() == 4);
    CHECK_THROWS_AS(classify_regions(make_mask(4, 6, 1), grid_dims(6, 4, 2)), std::invalid_argument);
  }
  // n = 1 collapse and all-simple == uniform (test_adaptive.cpp:75-108)
  {
    std::mt19937_64 rng(31);
    for (int round = 0; round < 15; ++round) {
      const int h = 4 + static_cast<int>(rng() % 40), w = 4 + static_cast<int>(rng() % 40);
      const int b = 1 + static_cast<int>(rng() % std::min({h, w, 8}));
      const GrayImage img = random_image(rng, h, w);
      const RegionMask mask = random_mask(rng, h, w);
      const PrivacyParams p = make_privacy_params(0.4, 9, b, 1);
      const NoiseSeed seed{rng()};
      CHECK(pixelize_adaptive(img, mask, p, seed).image == pixelize_parallel(img, p, seed).image);
    }
    const GrayImage img = random_image(rng, 24, 32);
    for (int n : {2, 4}) {
      const AdaptiveResult a =
          pixelize_adaptive(img, make_mask(24, 32, 1), make_privacy_params(0.8, 4, 8, n), NoiseSeed{5});
      CHECK(a.image == pixelize_parallel(img, make_privacy_params(0.8, 4, 8), NoiseSeed{5}).image);
      CHECK(a.means.complex_submeans.empty());
    }
  }
  // per-subgrid keyed noise at sigma_sub (test_adaptive.cpp:124-144)
  {
    const PrivacyParams p = make_privacy_params(2.0, 3, 4, 2);
    const AdaptiveResult out =
        pixelize_adaptive(make_image(4, 4, 100), make_mask(4, 4, 0), p, NoiseSeed{77});
    for (std::uint32_t sr = 0; sr < 2; ++sr)
      for (std::uint32_t sc = 0; sc < 2; ++sc) {
        const double noise = laplace_at(NoiseSeed{77}, NoiseKey{0, 0, sr, sc}, p.sigma_sub);
        CHECK(out.means.complex_submeans[sr * 2 + sc] ==
              quantize_intensity(clip_intensity(100.0 + noise)));
      }
  }
  // reassemble KATs and corrupt lengths (test_adaptive.cpp:185-234)
  {
    AdaptiveMeans mixed;
    mixed.geometry = grid_dims(2, 4, 2);
    mixed.n = 2;
    mixed.classification.geometry = mixed.geometry;
    mixed.classification.mask_means = {1.0f, 0.0f};
    mixed.classification.is_simple = {1, 0};
    mixed.simple_means = {9};
    mixed.complex_submeans = {1, 2, 3, 4};
    GrayImage e = make_image(2, 4);
    e.pixels = {9, 9, 1, 2, 9, 9, 3, 4};
    CHECK(reassemble(mixed, 2, 4) == e);
    AdaptiveMeans broken = mixed;
    broken.complex_submeans = {1, 2, 3};
    CHECK_THROWS_AS(reassemble(broken, 2, 4), RecordError);
    try {
      reassemble(broken, 2, 4);
    } catch (const RecordError& err) {
      CHECK(err.kind() == RecordErrorKind::corrupt_record);
    }
  }
  CHECK_THROWS_AS(pixelize_adaptive(make_image(8, 8), make_mask(8, 6, 1),
                                    make_privacy_params(1.0, 1, 4, 2), none),
                  std::invalid_argument);
  // round trip: reassemble(means) == emitted image (acceptance criterion 6)
  {
    std::mt19937_64 rng(41);
    for (int round = 0; round < 20; ++round) {
      const int h = 8 + static_cast<int>(rng() % 100), w = 8 + static_cast<int>(rng() % 100);
      const int b = 1 << (1 + rng() % 3);
      const int n = 1 << (rng() % 2);
      const GrayImage img = random_image(rng, h, w);
      const AdaptiveResult r = pixelize_adaptive(img, random_mask(rng, h, w),
                                                 make_privacy_params(0.5, 16, b, n), NoiseSeed{rng()});
      CHECK(reassemble(r.means, h, w) == r.image);
    }
  }
  // records: size law, decode(encode) identity, reconstruct == emitted image,
  // failure taxonomy (test_record.cpp:83-293)
  {
    std::mt19937_64 rng(47);
    for (int round = 0; round < 10; ++round) {
      const int h = 6 + static_cast<int>(rng() % 50), w = 6 + static_cast<int>(rng() % 50);
      const int b = 1 + static_cast<int>(rng() % std::min({h, w, 8}));
      const GrayImage img = random_image(rng, h, w);
      if (round % 2 == 0) {
        UniformResult r = pixelize_parallel(img, make_privacy_params(0.5, 16, b), NoiseSeed{rng()});
        const PixelRecord rec{h, w, r.means};
        const std::vector<std::uint8_t> bytes = encode(rec);
        CHECK(bytes.size() == 24 + static_cast<std::size_t>(r.means.geometry.grid_count()));
        CHECK(decode(bytes) == rec);
        CHECK(reconstruct(decode(bytes)) == r.image);
      } else {
        const int n = b % 2 == 0 ? 2 : 1;
        AdaptiveResult r = pixelize_adaptive(img, random_mask(rng, h, w),
                                             make_privacy_params(0.5, 16, b, n), NoiseSeed{rng()});
        const PixelRecord rec{h, w, r.means};
        const std::vector<std::uint8_t> bytes = encode(rec);
        CHECK(decode(bytes) == rec);
        CHECK(reconstruct(decode(bytes)) == r.image);
      }
    }
    GridMeans one;
    one.geometry = grid_dims(16, 16, 16);
    one.values = {200};
    std::vector<std::uint8_t> bytes = encode(PixelRecord{16, 16, one});
    CHECK(bytes.size() == 25);
    std::vector<std::uint8_t> bad = bytes;
    bad[0] = 'X';
    try {
      decode(bad);
      CHECK(false);
    } catch (const RecordError& e) {
      CHECK(e.kind() == RecordErrorKind::not_a_record);
    }
    bad = bytes;
    bad[21] ^= 0x40;
    try {
      decode(bad);
      CHECK(false);
    } catch (const RecordError& e) {
      CHECK(e.kind() == RecordErrorKind::corruption);
    }
  }
  // metrics (test_metrics.cpp:32-117): KATs and symmetry
  {
    GrayImage a = make_image(8, 8, 0), b = make_image(8, 8, 255);
    CHECK(mse(a, b) == 65025.0);
    CHECK(mse(a, a) == 0.0);
    std::mt19937_64 rng(51);
    const GrayImage x = random_image(rng, 40, 50), y = random_image(rng, 40, 50);
    CHECK(ssim(x, x) == 1.0);
    CHECK(ssim(x, y) == ssim(y, x));
    CHECK(ssim(x, y, 1) == ssim(x, y, 8));
    CHECK_THROWS_AS(ssim(make_image(6, 9), make_image(6, 9)), std::invalid_argument);
    CHECK(csv_header() == "epsilon,m,b,n,seed,mse,ssim,runtime_ms,record_bytes");
  }
  // GPU batch runner == run_single per file (cli.cpp:93-213 semantics)
  {
    namespace fs = std::filesystem;
    const fs::path dir = fs::temp_directory_path() / "dppx_batch_test";
    fs::remove_all(dir);
    fs::create_directories(dir / "in");
    fs::create_directories(dir / "masks");
    std::mt19937_64 rng(77);
    const int shapes[5][2] = {{48, 64}, {48, 64}, {33, 70}, {48, 64}, {33, 70}};
    std::vector<GrayImage> imgs;
    for (int i = 0; i < 5; ++i) {
      imgs.push_back(random_image(rng, shapes[i][0], shapes[i][1]));
      write_pgm(imgs.back(), (dir / "in" / ("f" + std::to_string(i) + ".pgm")).string());
      GrayImage m = make_image(shapes[i][0], shapes[i][1]);
      for (auto& v : m.pixels) v = (rng() & 1) ? 255 : 0;
      if (i != 4) write_pgm(m, (dir / "masks" / ("f" + std::to_string(i) + ".pgm")).string());
    }
    { std::ofstream bad((dir / "in" / "zz.pgm").string()); bad << "P2\n1 1\n255\n0\n"; }
    BatchConfig cfg;
    cfg.input = (dir / "in").string();
    cfg.out_dir = (dir / "out").string();
    cfg.mode = BatchMode::adaptive;
    cfg.epsilon = 0.5;
    cfg.m = 16;
    cfg.b = 8;
    cfg.n = 2;
    cfg.seed = NoiseSeed{1234};
    cfg.mask_path = (dir / "masks").string();
    cfg.frames_per_call = 2;
    const std::vector<BatchFileReport> reps = run_batch_gpu(cfg);
    CHECK(reps.size() == 6);
    for (int i = 0; i < 4; ++i) {
      CHECK(reps[i].exit_code == 0);
      const RegionMask mask = read_mask_pgm((dir / "masks" / ("f" + std::to_string(i) + ".pgm")).string());
      const AdaptiveResult want = pixelize_adaptive(imgs[i], mask, make_privacy_params(0.5, 16, 8, 2),
                                                    NoiseSeed{1234});
      CHECK(read_pgm((dir / "out" / ("f" + std::to_string(i) + ".pix.pgm")).string()) == want.image);
      const PixelRecord rec = read_record((dir / "out" / ("f" + std::to_string(i) + ".dppx")).string());
      CHECK(rec == (PixelRecord{imgs[i].height, imgs[i].width, want.means}));
      CHECK(reps[i].report.mse == mse(imgs[i], want.image));
      CHECK(reps[i].report.ssim == ssim(imgs[i], want.image));
      CHECK(reps[i].report.record_bytes == encode(rec).size());
    }
    CHECK(reps[4].exit_code == 3);  // no mask for f4 (IoError)
    CHECK(reps[5].exit_code == 3);  // P2 input (IoError)
    cfg.mode = BatchMode::uniform;
    cfg.seed.reset();  // noise-free: epsilon is a label
    const std::vector<BatchFileReport> u = run_batch_gpu(cfg);
    CHECK(u[4].exit_code == 0 &&
          read_pgm((dir / "out" / "f4.pix.pgm").string()) ==
              pixelize_parallel(imgs[4], make_privacy_params(0.5, 16, 8), std::nullopt).image);
    cfg.mode = BatchMode::reference;
    bool usage = false;
    try {
      run_batch_gpu(cfg);  // reference mode cannot emit records (cli.cpp:82-85)
    } catch (const UsageError&) {
      usage = true;
    }
    CHECK(usage);
    fs::remove_all(dir);
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
