// dppix/record.hpp -- the .dppx record (reference: proj/include/dppix/record.hpp:28-69).
// encode/decode wrap the compact store's payload with the 20-byte header and a
// CRC32 trailer; reconstruct expands it on the GPU.
#pragma once

#include <cstdint>
#include <string>
#include <variant>
#include <vector>

#include "dppix/adaptive.hpp"
#include "dppix/image.hpp"
#include "dppix/pixelize.hpp"

namespace dppix {

enum class RecordMode : std::uint8_t { uniform = 1, adaptive = 2 };

struct PixelRecord {
  int height = 0;
  int width = 0;
  std::variant<GridMeans, AdaptiveMeans> payload;

  RecordMode mode() const;
  int grid_side() const;
  int subgrid_factor() const;
  bool operator==(const PixelRecord&) const = default;
};

std::vector<std::uint8_t> encode(const PixelRecord& record);
PixelRecord decode(const std::vector<std::uint8_t>& bytes);
GrayImage reconstruct(const PixelRecord& record);
PixelRecord read_record(const std::string& path);
void write_record(const PixelRecord& record, const std::string& path);

}  // namespace dppix
