// dppix/pixelize.hpp -- uniform pixelization (Algorithm 2) on the GPU
// (reference: proj/include/dppix/pixelize.hpp:26-62).
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "dppix/image.hpp"
#include "dppix/noise.hpp"

namespace dppix {

struct GridMeans {
  GridGeometry geometry;
  std::vector<std::uint8_t> values;
  bool operator==(const GridMeans&) const = default;
};

double clip_intensity(double v);
std::uint8_t quantize_intensity(double v);

// Algorithm 1: no padding, border grids average only their real pixels.
GrayImage pixelize_reference(const GrayImage& img, const PrivacyParams& params,
                             const std::optional<NoiseSeed>& seed);

struct UniformResult {
  GrayImage image;
  GridMeans means;
};

// Runs on the calling thread's GPU context (device DPPX_DEVICE, default 0).
// `threads` is accepted for source compatibility and ignored: results never
// depend on it (reference acceptance criterion 9).
UniformResult pixelize_parallel(const GrayImage& img, const PrivacyParams& params,
                                const std::optional<NoiseSeed>& seed, int threads = 0);

GrayImage broadcast_means(const GridMeans& means, int height, int width);

}  // namespace dppix
