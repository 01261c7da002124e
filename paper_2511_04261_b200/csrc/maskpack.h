// Host-side mask transport encoding for the pinned host pipeline.
//
// The reference's RegionMask is one byte per pixel holding 0 or 1
// (image.hpp:49-54). Only the bits cross PCIe: rows of ceil(N/32) u32 words,
// bit (j % 32) of word (j / 32) = mask[i][j]. That cuts the adaptive call's
// host->device bytes per 1080p RGB frame from 8.29 MB to 6.48 MB. K0 counts
// the bits with popc and produces the same mask sums, so the statistics are
// unchanged. A mask byte outside {0, 1} (not a RegionMask value, but accepted
// by the reference arithmetic) makes the packer report failure and the caller
// sends that chunk's bytes instead.
#pragma once
#include <cstdint>
#include <functional>

namespace dppx {

struct MaskPacker;

MaskPacker* mask_packer_create(int threads);  // threads <= 0: automatic
void mask_packer_destroy(MaskPacker* p);
int mask_packer_threads(const MaskPacker* p);

inline int64_t mask_words_per_row(int N) { return (static_cast<int64_t>(N) + 31) / 32; }

// Pack F frames of M rows x N bytes (row pitch `pitch`, frame stride `fstride`)
// into dst (rows of `wpr` words, frame stride M * wpr words). Returns false if
// any byte is > 1 (dst contents are then unspecified).
bool pack_mask_bits(MaskPacker* p, const uint8_t* src, int64_t pitch, int64_t fstride, int M, int N,
                    int F, uint32_t* dst, int64_t wpr);

// Runs body(begin, end) over [0, n) split evenly across the pool's threads
// (the caller takes one share). Used for pageable <-> pinned staging copies.
void pool_for(MaskPacker* p, int64_t n, const std::function<void(int64_t, int64_t)>& body);

}  // namespace dppx
