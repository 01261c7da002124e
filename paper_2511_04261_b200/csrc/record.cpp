// record.cpp -- the .dppx record codec around the compact store
// (reference: proj/include/dppix/record.hpp:48-71, proj/src/record.cpp:124-278).
//
// Wire layout (little-endian): "DPPX" | u16 version = 1 | u8 mode | u8 0 |
// u32 M | u32 N | u16 b | u16 n | payload | u32 CRC32 of all preceding bytes.
// The payload is exactly what the K0/K1 kernels write into a statistics slot,
// so encoding a GPU result is a header + CRC around bytes already in hand.
// Host code: the record is O(G) bytes per plane.
#include <cstdint>
#include <cstring>

#include "../../include/dppx_gpu.h"

namespace {

constexpr size_t kHeader = 20;

// CRC-32 (IEEE 802.3, reflected 0xEDB88320 -- the polynomial of zlib's crc32,
// record.cpp:35-39), slicing-by-8.
struct Crc32Tables {
  uint32_t t[8][256];
  Crc32Tables() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
      t[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int s = 1; s < 8; ++s) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xFF];
  }
};

const Crc32Tables& tables() {
  static const Crc32Tables tb;
  return tb;
}

uint32_t rd32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) |
         (static_cast<uint32_t>(p[2]) << 16) | (static_cast<uint32_t>(p[3]) << 24);
}
uint16_t rd16(const uint8_t* p) {
  return static_cast<uint16_t>(p[0] | (static_cast<uint16_t>(p[1]) << 8));
}
void wr32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
void wr16(uint8_t* p, uint16_t v) {
  p[0] = static_cast<uint8_t>(v);
  p[1] = static_cast<uint8_t>(v >> 8);
}

// validate_header_fields, record.cpp:93-112.
bool header_fields_ok(int64_t M, int64_t N, int64_t b, int64_t n, int mode) {
  if (M < 1 || N < 1) return false;
  if (b < 1 || b > (M > N ? M : N)) return false;
  if (n < 1 || b % n != 0) return false;
  if (mode == 1 && n != 1) return false;
  return true;
}

// Expected payload length, or 0 if the payload is internally inconsistent.
// Uniform: G bytes. Adaptive: 4G + 4 + S + (G - S) n^2 with S the stored count,
// which must equal the number of mask means > 0.5f (record.cpp:241-270).
size_t expected_payload(const uint8_t* payload, size_t avail, int M, int N, int b, int n, int mode,
                        bool* count_ok) {
  dppx_geometry g;
  if (dppx_grid_dims(M, N, b, &g) != DPPX_OK) return 0;
  const size_t G = static_cast<size_t>(g.grid_rows) * g.grid_cols;
  *count_ok = true;
  if (mode == 1) return G;
  if (avail < 4 * G + 4) return 4 * G + 4;  // too short: caller reports
  size_t S = 0;
  for (size_t k = 0; k < G; ++k) {
    float f;
    std::memcpy(&f, payload + 4 * k, 4);
    S += f > 0.5f;  // simple_from_mean, adaptive.cpp:30-32
  }
  const uint32_t stored = rd32(payload + 4 * G);
  if (stored != S) *count_ok = false;
  return 4 * G + 4 + S + (G - S) * static_cast<size_t>(n) * n;
}

}  // namespace

extern "C" {

uint32_t dppx_crc32(uint32_t crc, const uint8_t* data, size_t len) {
  const Crc32Tables& tb = tables();
  uint32_t c = ~crc;
  while (len >= 8) {
    const uint32_t lo = rd32(data) ^ c, hi = rd32(data + 4);
    c = tb.t[7][lo & 0xFF] ^ tb.t[6][(lo >> 8) & 0xFF] ^ tb.t[5][(lo >> 16) & 0xFF] ^
        tb.t[4][lo >> 24] ^ tb.t[3][hi & 0xFF] ^ tb.t[2][(hi >> 8) & 0xFF] ^
        tb.t[1][(hi >> 16) & 0xFF] ^ tb.t[0][hi >> 24];
    data += 8;
    len -= 8;
  }
  while (len--) c = (c >> 8) ^ tb.t[0][(c ^ *data++) & 0xFF];
  return ~c;
}

size_t dppx_record_size(size_t payload_len) { return kHeader + payload_len + 4; }

// encode, record.cpp:124-175.
int dppx_encode_record(int32_t height, int32_t width, int32_t b, int32_t n, int32_t mode,
                       const uint8_t* payload, size_t payload_len, uint8_t* out, size_t cap,
                       size_t* out_len) {
  if (!out_len || (mode != 1 && mode != 2)) return DPPX_ERR_INVALID;
  if (!header_fields_ok(height, width, b, n, mode)) return DPPX_ERR_INVALID;
  if (!payload && payload_len) return DPPX_ERR_INVALID;
  bool count_ok = true;
  const size_t want = expected_payload(payload, payload_len, height, width, b, n, mode, &count_ok);
  if (want == 0 || want != payload_len || !count_ok) return DPPX_ERR_INVALID;
  const size_t total = dppx_record_size(payload_len);
  *out_len = total;
  if (!out || cap < total) return DPPX_ERR_INVALID;
  std::memcpy(out, "DPPX", 4);
  wr16(out + 4, 1);
  out[6] = static_cast<uint8_t>(mode);
  out[7] = 0;
  wr32(out + 8, static_cast<uint32_t>(height));
  wr32(out + 12, static_cast<uint32_t>(width));
  wr16(out + 16, static_cast<uint16_t>(b));
  wr16(out + 18, static_cast<uint16_t>(n));
  std::memcpy(out + kHeader, payload, payload_len);
  wr32(out + kHeader + payload_len, dppx_crc32(0, out, kHeader + payload_len));
  return DPPX_OK;
}

// decode, record.cpp:177-278: the checks run in the reference's order.
int dppx_decode_record(const uint8_t* bytes, size_t len, dppx_record_info* info) {
  if (!info || (!bytes && len)) return DPPX_ERR_INVALID;
  if (len < 4 || std::memcmp(bytes, "DPPX", 4) != 0) return DPPX_ERR_NOT_A_RECORD;
  if (len < kHeader + 4) return DPPX_ERR_CORRUPT;  // truncated header
  const size_t body = len - 4;
  if (dppx_crc32(0, bytes, body) != rd32(bytes + body)) return DPPX_ERR_CORRUPTION;
  if (rd16(bytes + 4) != 1) return DPPX_ERR_UNSUPPORTED_VERSION;
  const int mode = bytes[6];
  if ((mode != 1 && mode != 2) || bytes[7] != 0) return DPPX_ERR_CORRUPT;
  const uint32_t M = rd32(bytes + 8), N = rd32(bytes + 12);
  if (M < 1 || N < 1 || M > 0x7FFFFFFFu || N > 0x7FFFFFFFu) return DPPX_ERR_CORRUPT;
  const int b = rd16(bytes + 16), n = rd16(bytes + 18);
  if (!header_fields_ok(M, N, b, n, mode)) return DPPX_ERR_CORRUPT;
  const uint8_t* payload = bytes + kHeader;
  const size_t plen = body - kHeader;
  bool count_ok = true;
  const size_t want = expected_payload(payload, plen, static_cast<int>(M), static_cast<int>(N), b,
                                       n, mode, &count_ok);
  if (want == 0 || !count_ok || want != plen) return DPPX_ERR_CORRUPT;
  info->height = static_cast<int32_t>(M);
  info->width = static_cast<int32_t>(N);
  info->b = b;
  info->n = n;
  info->mode = mode;
  info->payload_offset = static_cast<uint32_t>(kHeader);
  info->payload_len = static_cast<uint32_t>(plen);
  return DPPX_OK;
}

}  // extern "C"
