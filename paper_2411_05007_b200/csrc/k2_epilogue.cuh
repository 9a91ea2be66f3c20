// Shared epilogue of the NVFP4 GEMMs (K2): TMEM -> registers -> alpha, bias ->
// 16-bit (or fp32) -> 128-B-swizzled smem staging -> TMA bulk tensor store.
//   Y[m,n] = out_rn(fl32(alpha * acc[m,n]) + bias[n])        (App. B.5, reading Q16)
// One warp owns one TMEM lane quadrant (32 rows).  Each 32-row x 128-byte chunk is
// staged in a 4 KB buffer (two per warp, so the TMA store of one overlaps the next
// chunk) whose 16-byte columns are XOR-swizzled by row, matching the store map's
// SWIZZLE_128B layout; TMA clips rows >= M and columns >= N.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sm100.cuh"

namespace svdq {

__device__ __forceinline__ uint32_t pack2(float a, float b, int dt) {
  if (dt == 0)
    return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
           (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
  return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(a))) |
         (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(b))) << 16);
}

// Drains `ncols` accumulator columns of this warp's 32 TMEM lanes.  `release` is invoked
// once every tcgen05.ld of the tile has completed (the accumulator buffer may be reused).
template <int NCOLS, typename Release>
__device__ __forceinline__ void epilogue_tile(uint32_t tmem_acc_lane, const float *bias_s, float alpha, int y_dtype,
                                              const CUtensorMap *tmY, int32_t row0, int32_t col0, uint8_t *stage,
                                              int &buf, int lane, Release release) {
  const int cpc = y_dtype == 2 ? 32 : 64;                 // columns per 128-byte chunk
  const int nchunks = NCOLS / cpc;
  for (int ch = 0; ch < nchunks; ++ch) {
    float v[64];
    if (y_dtype == 2) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_acc_lane + ch * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    } else {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_acc_lane + ch * 64, r);
      uint32_t r2[32];
      tmem_ld_32x32b_x32(tmem_acc_lane + ch * 64 + 32, r2);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        v[j] = __uint_as_float(r[j]);
        v[32 + j] = __uint_as_float(r2[j]);
      }
    }
    if (ch == nchunks - 1) release();
    // staging buffer of this chunk: wait until the TMA store that last used it has read it
    uint8_t *sb = stage + buf * 4096;
    if (lane == 0) bulk_wait_group_read<1>();
    __syncwarp();
    const float *bs = bias_s + ch * cpc;
    uint8_t *rowp = sb + lane * 128;
    const uint32_t sw = static_cast<uint32_t>(lane & 7);
    if (y_dtype == 2) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float4 o;
        o.x = __fadd_rn(__fmul_rn(alpha, v[4 * c + 0]), bs[4 * c + 0]);
        o.y = __fadd_rn(__fmul_rn(alpha, v[4 * c + 1]), bs[4 * c + 1]);
        o.z = __fadd_rn(__fmul_rn(alpha, v[4 * c + 2]), bs[4 * c + 2]);
        o.w = __fadd_rn(__fmul_rn(alpha, v[4 * c + 3]), bs[4 * c + 3]);
        *reinterpret_cast<float4 *>(rowp + ((c ^ sw) * 16)) = o;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(__fmul_rn(alpha, v[8 * c + e]), bs[8 * c + e]);
        *reinterpret_cast<uint4 *>(rowp + ((c ^ sw) * 16)) =
            make_uint4(pack2(o[0], o[1], y_dtype), pack2(o[2], o[3], y_dtype), pack2(o[4], o[5], y_dtype),
                       pack2(o[6], o[7], y_dtype));
      }
    }
    fence_proxy_async();                                   // generic smem writes -> TMA (async proxy)
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmY, sb, col0 + ch * cpc, row0);
      bulk_commit_group();
    }
    buf ^= 1;
  }
}

}  // namespace svdq
