// run_batch_gpu (include/dppix/batch.hpp) timed around the call; the GPU arm of
// tools/batch_bench.py (same arguments as oracle/batch_ref_main.cpp).
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "dppix/batch.hpp"
#include "dppix/pixelize.hpp"

int main(int argc, char** argv) {
  if (argc != 11 && argc != 12) {
    std::fprintf(stderr, "usage: %s in out u|a masks eps m b n seed threads [frames_per_call]\n", argv[0]);
    return 2;
  }
  dppix::BatchConfig cfg;
  cfg.input = argv[1];
  cfg.out_dir = argv[2];
  cfg.mode = argv[3][0] == 'a' ? dppix::BatchMode::adaptive : dppix::BatchMode::uniform;
  cfg.mask_path = argv[4];
  cfg.epsilon = std::atof(argv[5]);
  cfg.m = std::atoi(argv[6]);
  cfg.b = std::atoi(argv[7]);
  cfg.n = std::atoi(argv[8]);
  cfg.seed = dppix::NoiseSeed{std::strtoull(argv[9], nullptr, 10)};
  if (argc == 12) cfg.frames_per_call = std::atoi(argv[11]);
  {  // context creation and module loading happen here, outside the timed region
    dppix::GrayImage tiny = dppix::make_image(8, 8, 7);
    (void)dppix::pixelize_parallel(tiny, dppix::make_privacy_params(1.0, 1, 4), std::nullopt);
  }
  const auto t0 = std::chrono::steady_clock::now();
  const auto reports = dppix::run_batch_gpu(cfg);
  const auto t1 = std::chrono::steady_clock::now();
  int failures = 0;
  for (const auto& r : reports) failures += r.exit_code != 0;
  std::printf("{\"files\": %zu, \"seconds\": %.6f, \"failures\": %d}\n", reports.size(),
              std::chrono::duration<double>(t1 - t0).count(), failures);
  return failures ? 1 : 0;
}
