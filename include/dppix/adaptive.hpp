// dppix/adaptive.hpp -- region-adaptive pixelization (Algorithm 3) on the GPU
// (reference: proj/include/dppix/adaptive.hpp:29-78).
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "dppix/image.hpp"
#include "dppix/noise.hpp"
#include "dppix/pixelize.hpp"

namespace dppix {

struct RegionClassification {
  GridGeometry geometry;
  std::vector<float> mask_means;
  std::vector<std::uint8_t> is_simple;

  int simple_count() const;
  bool operator==(const RegionClassification&) const = default;
};

bool simple_from_mean(float mask_mean);

RegionClassification classify_regions(const RegionMask& mask, const GridGeometry& geom);

struct AdaptiveMeans {
  GridGeometry geometry;
  int n = 1;
  RegionClassification classification;
  std::vector<std::uint8_t> simple_means;
  std::vector<std::uint8_t> complex_submeans;
  bool operator==(const AdaptiveMeans&) const = default;
};

struct AdaptiveResult {
  GrayImage image;
  AdaptiveMeans means;
};

AdaptiveResult pixelize_adaptive(const GrayImage& img, const RegionMask& mask,
                                 const PrivacyParams& params,
                                 const std::optional<NoiseSeed>& seed, int threads = 0);

GrayImage reassemble(const AdaptiveMeans& means, int height, int width);

}  // namespace dppix
