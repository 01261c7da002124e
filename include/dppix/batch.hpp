// dppix/batch.hpp -- GPU batch runner: the reference's run_batch
// (proj/src/cli.cpp:175-213 over run_single cli.cpp:93-173) re-planned for the
// GPU. Files are read by host threads, grouped by shape, and pixelized F frames
// per call through the pinned pipeline, the calls spread over every GPU of the
// node (one host thread + ctx per GPU); results and side effects match running
// run_single on each file (same seed for every file, cli.cpp:200-201).
// dppix::run_batch (dppix/cli.hpp) is this runner behind the reference's
// RunConfig signature.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "dppix/metrics.hpp"
#include "dppix/noise.hpp"

namespace dppix {

enum class BatchMode { uniform, adaptive, reference };

struct BatchConfig {
  std::string input;          // a .pgm file or a directory of them (sorted)
  std::string out_dir = ".";
  BatchMode mode = BatchMode::uniform;
  double epsilon = 0.0;
  int m = 1;
  int b = 1;
  int n = 1;
  std::optional<NoiseSeed> seed;  // nullopt: no noise (epsilon is a label)
  std::string mask_path;          // adaptive: a mask file or a directory paired by stem
  bool emit_image = true;         // <stem>.pix.pgm
  bool emit_record = true;        // <stem>.dppx
  bool reconstruct_check = true;  // decode + reconstruct must equal the image
  int frames_per_call = 64;       // GPU batch size per shape group
  int io_threads = 0;             // 0: hardware_concurrency
  // GPUs the chunks are spread over (one host thread + ctx each, dppx_group);
  // empty: env DPPX_BATCH_DEVICES ("0,1,...") if set, else every visible sm_100 GPU.
  std::vector<int> devices;
};

struct BatchFileReport {
  std::string input;
  MetricReport report;
  std::vector<std::string> written;
  std::string error;
  int exit_code = 0;  // cli.hpp:28-32: 0 ok, 1 other, 2 usage, 3 io, 4 record, 5 consistency
};

std::vector<BatchFileReport> run_batch_gpu(const BatchConfig& cfg);

// exit_code_for (cli.cpp:386-401).
int batch_exit_code_for(const std::exception& err);

}  // namespace dppix
