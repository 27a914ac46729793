// Host-side bit packing of uint8 {0,1} image batches (ts_hostpack.cpp).
#pragma once
#include <cstdint>

namespace ts {
// [n][h][w] uint8 -> [n][h][ww] uint32 bit rows (LSB = leftmost pixel);
// false if any byte is not 0 or 1 (the output is then unspecified)
bool pack_images(const uint8_t *in, uint32_t *out, int64_t n, int h, int w, int ww);
// the same for `planes` (<= 3) batches at once -- image, keep, avoid -- in one parallel region
bool pack_planes(const uint8_t *const *in, uint32_t *const *out, int planes, int64_t n, int h, int w, int ww);
// inverse of pack_images
void unpack_images(const uint32_t *in, uint8_t *out, int64_t n, int h, int w, int ww);
}  // namespace ts
