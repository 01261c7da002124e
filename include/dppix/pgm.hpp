// dppix/pgm.hpp -- binary PGM (P5, maxval 255) ingest (reference:
// proj/include/dppix/pgm.hpp:25-33). Masks: pixel >= 128 -> 1 (simple),
// following pgm.cpp:112-119 (not README.md:81).
#pragma once

#include <string>

#include "dppix/image.hpp"

namespace dppix {

GrayImage read_pgm(const std::string& path);
void write_pgm(const GrayImage& img, const std::string& path);
RegionMask read_mask_pgm(const std::string& path);

}  // namespace dppix
