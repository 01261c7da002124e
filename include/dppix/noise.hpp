// dppix/noise.hpp -- privacy calibration and the keyed Laplace stream
// (reference: proj/include/dppix/noise.hpp:21-80). The device kernels draw the
// same stream; these host functions exist for callers and parity checks.
#pragma once

#include <cstdint>

namespace dppix {

struct NoiseSeed {
  std::uint64_t value = 0;
};

struct NoiseKey {
  std::uint32_t r = 0;
  std::uint32_t c = 0;
  std::uint32_t sr = 0;
  std::uint32_t sc = 0;
};

struct PrivacyParams {
  double epsilon = 0.0;
  int m = 0;
  int b = 0;
  int n = 1;
  int subgrid_side = 0;
  double delta = 0.0;
  double sigma = 0.0;
  double delta_sub = 0.0;
  double sigma_sub = 0.0;
};

PrivacyParams make_privacy_params(double epsilon, int m, int b, int n = 1);
double sensitivity(int b, int m);
double noise_scale(double delta, double epsilon);
double subgrid_sensitivity(const PrivacyParams& params);
std::uint64_t keyed_bits(NoiseSeed seed, const NoiseKey& key);
double uniform_from_bits(std::uint64_t bits);
double laplace_from_uniform(double u, double sigma);
double laplace_at(NoiseSeed seed, const NoiseKey& key, double sigma);

}  // namespace dppix
