// Host mask bit packing (paper_2511_04261_b200/csrc/maskpack.cpp), no GPU:
// packed words equal a naive per-pixel packing for ragged widths, strided
// sources and several worker counts; a byte outside {0, 1} is reported.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2511_04261_b200/csrc/maskpack.h"

static int fails = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                        \
    }                                                                 \
  } while (0)

int main() {
  std::mt19937 rng(7);
  for (int threads : {1, 2, 5}) {
    dppx::MaskPacker* p = dppx::mask_packer_create(threads);
    CHECK(dppx::mask_packer_threads(p) == threads);
    for (int N : {1, 7, 31, 32, 33, 64, 100, 178, 1920, 1917}) {
      const int M = 1 + static_cast<int>(rng() % 40), F = 1 + static_cast<int>(rng() % 3);
      const int64_t pitch = N + static_cast<int>(rng() % 9), fstride = pitch * M + 5;
      std::vector<uint8_t> src(static_cast<size_t>(fstride) * F, 0xAB);  // junk in the gaps
      for (int f = 0; f < F; ++f)
        for (int i = 0; i < M; ++i)
          for (int j = 0; j < N; ++j) src[f * fstride + i * pitch + j] = rng() & 1;
      const int64_t wpr = dppx::mask_words_per_row(N);
      std::vector<uint32_t> dst(static_cast<size_t>(wpr) * M * F, 0xFFFFFFFFu);
      CHECK(dppx::pack_mask_bits(p, src.data(), pitch, fstride, M, N, F, dst.data(), wpr));
      for (int f = 0; f < F; ++f)
        for (int i = 0; i < M; ++i)
          for (int w = 0; w < wpr; ++w) {
            uint32_t want = 0;
            for (int k = 0; k < 32 && 32 * w + k < N; ++k)
              want |= static_cast<uint32_t>(src[f * fstride + i * pitch + 32 * w + k]) << k;
            CHECK(dst[(static_cast<size_t>(f) * M + i) * wpr + w] == want);
          }
      // one non-binary byte anywhere (incl. the ragged tail) is reported
      const int f = static_cast<int>(rng() % F), i = static_cast<int>(rng() % M),
                j = static_cast<int>(rng() % N);
      src[f * fstride + i * pitch + j] = static_cast<uint8_t>(2 + rng() % 254);
      CHECK(!dppx::pack_mask_bits(p, src.data(), pitch, fstride, M, N, F, dst.data(), wpr));
    }
    dppx::mask_packer_destroy(p);
  }
  if (fails) return 1;
  std::printf("test_maskpack: all checks passed\n");
  return 0;
}
