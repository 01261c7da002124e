// dppix/metrics.hpp -- utility scores of a pixelized image (reference:
// proj/include/dppix/metrics.hpp:25-53). mse and ssim run on the GPU and are
// bit-identical to the reference; the CSV helpers are host formatting.
#pragma once

#include <cstdint>
#include <string>

#include "dppix/image.hpp"

namespace dppix {

double mse(const GrayImage& a, const GrayImage& b);
double ssim(const GrayImage& a, const GrayImage& b, int threads = 0);  // threads ignored

struct MetricReport {
  double epsilon = 0.0;
  int m = 0;
  int b = 0;
  int n = 1;
  std::uint64_t seed = 0;
  double mse = 0.0;
  double ssim = 0.0;
  double runtime_ms = 0.0;
  std::uint64_t record_bytes = 0;
};

std::string format_double(double value);  // shortest round-trip %.15g..%.17g
std::string csv_header();
std::string csv_row(const MetricReport& report);

}  // namespace dppix
