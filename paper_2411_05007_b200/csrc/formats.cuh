// formats.cuh -- device half of the number formats (DESIGN.md "Readings" Q5-Q13):
// E2M1 / E4M3 conversions via the sm_100 cvt instructions, 16-bit scale
// rounding, and the NVFP4 128x4 scale-factor tile layout.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

namespace svdq {

// Two fp32 values -> one E2M1x2 byte, RNE, saturating; lo goes to bits [0,4).
__device__ __forceinline__ uint32_t e2m1x2(float lo, float hi) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .b8 b;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b, %2, %1;\n\t"
      "cvt.u32.u8 %0, b;\n\t}\n"
      : "=r"(r)
      : "f"(lo), "f"(hi));
  return r;
}
// Eight fp32 values -> 32 bits of packed E2M1 (element 0 in the lowest nibble).
__device__ __forceinline__ uint32_t e2m1x8(const float (&v)[8]) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}\n"
      : "=r"(r)
      : "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
  return r;
}

// fp32 (>= 0) -> UE4M3 byte, RNE, satfinite.
__device__ __forceinline__ uint32_t e4m3_rn_sat(float v) {
  return static_cast<uint32_t>(__nv_cvt_float_to_fp8(v, __NV_SATFINITE, __NV_E4M3));
}
// UE4M3 byte -> fp32 (exact).
__device__ __forceinline__ float e4m3_to_f32(uint32_t b) {
  __half_raw h = __nv_cvt_fp8_to_halfraw(static_cast<__nv_fp8_storage_t>(b), __NV_E4M3);
  return __half2float(__half(h));
}

// 16-bit scale storage, RNE + satfinite.  kBf16 selects bf16 vs fp16.
template <bool kBf16>
__device__ __forceinline__ uint16_t scale16_rn_sat(float v) {
  if constexpr (kBf16) {
    v = fminf(v, 3.3895313892515355e38f);
    return __bfloat16_as_ushort(__float2bfloat16_rn(v));
  } else {
    v = fminf(v, 65504.0f);
    return __half_as_ushort(__float2half_rn(v));
  }
}
template <bool kBf16>
__device__ __forceinline__ float scale16_to_f32(uint16_t b) {
  if constexpr (kBf16) return __bfloat162float(__ushort_as_bfloat16(b));
  else return __half2float(__ushort_as_half(b));
}

// Byte offset of NVFP4 scale factor (row, c), c = k/16, K = reduction length.
__host__ __device__ __forceinline__ int64_t sf_offset(int64_t row, int64_t c, int64_t K) {
  const int64_t nkt = K / 64;
  return (row >> 7) * (nkt * 512) + (c >> 2) * 512 + (row & 31) * 16 + ((row & 127) >> 5) * 4 +
         (c & 3);
}

}  // namespace svdq
