// test_pgm.cpp -- PGM ingest (no GPU needed): the reference's PGM tests
// (proj/tests/test_image.cpp:199-255) against include/dppix/pgm.hpp.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <random>
#include <string>

#include "dppix/errors.hpp"
#include "dppix/pgm.hpp"

using namespace dppix;
static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (c) ++g_pass;                                                  \
    else { ++g_fail; std::fprintf(stderr, "FAIL %d: %s\n", __LINE__, #c); } \
  } while (0)

static void raw(const std::string& path, const std::string& bytes) {
  std::ofstream f(path, std::ios::binary);
  f << bytes;
}

static bool io_error(const std::string& path) {
  try {
    read_pgm(path);
  } catch (const IoError&) {
    return true;
  } catch (...) {
  }
  return false;
}

int main() {
  const auto dir = std::filesystem::temp_directory_path() / "dppx_pgm_test";
  std::filesystem::create_directories(dir);
  std::mt19937_64 rng(15);
  GrayImage img = make_image(37, 53);
  for (auto& p : img.pixels) p = static_cast<std::uint8_t>(rng());
  const std::string f = (dir / "a.pgm").string();
  write_pgm(img, f);
  CHECK(read_pgm(f) == img);  // round trip
  raw((dir / "c.pgm").string(), std::string("P5\n# comment\n2 1\n# more\n255\n") + "\x07\x09");
  const GrayImage c = read_pgm((dir / "c.pgm").string());
  CHECK(c.width == 2 && c.height == 1 && c.pixels[0] == 7 && c.pixels[1] == 9);
  raw((dir / "p2.pgm").string(), "P2\n2 1\n255\n7 9\n");
  CHECK(io_error((dir / "p2.pgm").string()));  // only P5 (pgm.cpp:57)
  raw((dir / "mv.pgm").string(), std::string("P5\n2 1\n65535\n") + std::string(4, '\0'));
  CHECK(io_error((dir / "mv.pgm").string()));
  raw((dir / "tr.pgm").string(), std::string("P5\n4 4\n255\n") + "abc");
  CHECK(io_error((dir / "tr.pgm").string()));
  CHECK(io_error((dir / "missing.pgm").string()));
  GrayImage m = make_image(1, 4);
  m.pixels = {0, 127, 128, 255};
  write_pgm(m, (dir / "m.pgm").string());
  const RegionMask mk = read_mask_pgm((dir / "m.pgm").string());
  CHECK((mk.values == std::vector<std::uint8_t>{0, 0, 1, 1}));  // test_image.cpp:247-255
  std::filesystem::remove_all(dir);
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
