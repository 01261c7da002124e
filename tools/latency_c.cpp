// Single-frame host-call latency from C (no Python in the loop): PETS
// 768x576 RGB, uniform b16 and adaptive b16 n4, page-locked buffers
// (dppx_host_alloc), median / p10 / p90 of 2000 calls per small-frame path.
// Build: g++ -O2 -std=c++17 -Iinclude tools/latency_c.cpp -Lpaper_2511_04261_b200/lib -ldppx_gpu
//        -Wl,-rpath,$PWD/paper_2511_04261_b200/lib -o tools/latency_c
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "dppx_gpu.h"

int main() {
  const int M = 576, N = 768, C = 3;
  dppx_ctx* ctx = nullptr;
  if (dppx_ctx_create(0, &ctx) != DPPX_OK) {
    std::fprintf(stderr, "no device\n");
    return 1;
  }
  const size_t fb = static_cast<size_t>(M) * N * C;
  void *img, *out, *mask, *stats;
  dppx_host_alloc(fb, &img);
  dppx_host_alloc(fb, &out);
  dppx_host_alloc(static_cast<size_t>(M) * N, &mask);
  const int64_t stride = (dppx_adaptive_payload_capacity(M, N, 16, 4) + 3) & ~3ll;
  dppx_host_alloc(static_cast<size_t>(stride) * C, &stats);
  for (size_t i = 0; i < fb; ++i) static_cast<uint8_t*>(img)[i] = static_cast<uint8_t>(i * 131 + (i >> 7));
  for (int y = 0; y < M; ++y)
    for (int x = 0; x < N; ++x)
      static_cast<uint8_t*>(mask)[y * N + x] = (x - 384) * (x - 384) + (y - 288) * (y - 288) * 2 < 40000 ? 0 : 1;
  dppx_frames_desc d = {M, N, C, 1, static_cast<int64_t>(N) * C, static_cast<int64_t>(fb), N,
                        static_cast<int64_t>(M) * N, static_cast<int64_t>(N) * C, static_cast<int64_t>(fb)};
  uint64_t seeds[3] = {1, 2, 3};
  dppx_noise nz = {DPPX_NOISE_KEYED, 0, seeds, nullptr};
  uint32_t lens[3];
  const char* names[] = {"auto", "graph", "zerocopy", "staged"};
  for (int adaptive = 0; adaptive < 2; ++adaptive) {
    dppx_privacy_params p;
    dppx_make_privacy_params(0.5, 16, 16, adaptive ? 4 : 1, &p);
    for (int path : {DPPX_SMALL_AUTO, DPPX_SMALL_GRAPH, DPPX_SMALL_STAGED}) {
      dppx_ctx_set_small_frame_path(ctx, path);
      auto call = [&] {
        return adaptive ? dppx_pixelize_adaptive(ctx, &d, static_cast<uint8_t*>(img), static_cast<uint8_t*>(mask),
                                                 &p, &nz, static_cast<uint8_t*>(stats), stride, lens,
                                                 static_cast<uint8_t*>(out))
                        : dppx_pixelize_uniform(ctx, &d, static_cast<uint8_t*>(img), &p, &nz,
                                                static_cast<uint8_t*>(stats), static_cast<uint8_t*>(out));
      };
      for (int i = 0; i < 100; ++i)
        if (call() != DPPX_OK) {
          std::fprintf(stderr, "%s\n", dppx_ctx_last_error(ctx));
          return 1;
        }
      std::vector<double> us;
      for (int i = 0; i < 2000; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        call();
        const auto t1 = std::chrono::steady_clock::now();
        us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      }
      std::sort(us.begin(), us.end());
      std::printf("{\"mode\": \"%s\", \"path\": \"%s\", \"median_us\": %.2f, \"p10_us\": %.2f, \"p90_us\": %.2f}\n",
                  adaptive ? "adaptive b16 n4" : "uniform b16", names[path], us[us.size() / 2], us[us.size() / 10],
                  us[us.size() * 9 / 10]);
    }
  }
  dppx_host_free(img);
  dppx_host_free(out);
  dppx_host_free(mask);
  dppx_host_free(stats);
  dppx_ctx_destroy(ctx);
  return 0;
}
