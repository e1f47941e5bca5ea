// covap_half.cuh — the reference's fp16 wire conversion on the device
// (compress.cpp:157-224), shared by the dense filter kernels.  Internal.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace covapb {

// half_bits_from_float (compress.cpp:157-205).  The reference rounds to
// nearest even on the normal and subnormal half grids, which is what the
// hardware conversion (cvt.rn.f16.f32) does for |x| in [2^-24, 65504]; its
// three departures from IEEE are patched explicitly: NaN -> 0x7e00,
// |x| > 65504 (inf included) -> +-65504 and counted as saturated (IEEE
// would round 65504 < |x| < 65520 down and give inf above), and
// |x| < 2^-24 -> signed zero (IEEE rounds (2^-25, 2^-24) up).
__device__ __forceinline__ uint16_t half_bits(float value, bool& saturated) {
  const uint32_t bits = __float_as_uint(value);
  const uint32_t sign = (bits >> 16) & 0x8000u;
  const uint32_t a = bits & 0x7fffffffu;
  if (a > 0x7f800000u) return static_cast<uint16_t>(sign | 0x7e00u);
  if (a > 0x477fe000u) {  // 65504.0f
    saturated = true;
    return static_cast<uint16_t>(sign | 0x7bffu);
  }
  if (a < 0x33800000u) return static_cast<uint16_t>(sign);  // 2^-24
  return __half_as_ushort(__float2half_rn(value));
}

// float_from_half_bits (compress.cpp:207-224).
__device__ __forceinline__ float half_to_float(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu;
  const uint32_t m = h & 0x3ffu;
  if (e == 0) {
    if (m == 0) return __uint_as_float(sign);
    const int s = __clz(m) - 21;  // shifts until bit 10 is set
    const uint32_t mm = (m << s) & 0x3ffu;
    return __uint_as_float(sign | (static_cast<uint32_t>(-14 - s + 127) << 23) | (mm << 13));
  }
  if (e == 31) return __uint_as_float(sign | 0x7f800000u | (m << 13));
  return __uint_as_float(sign | ((e - 15 + 127) << 23) | (m << 13));
}

}  // namespace covapb
