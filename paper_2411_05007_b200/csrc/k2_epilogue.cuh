// Shared epilogue of the NVFP4 GEMMs (K2): TMEM -> registers -> alpha, bias ->
// 16-bit (or fp32) -> 64-B-swizzled smem staging -> TMA bulk tensor store.
//   Y[m,n] = out_rn(fl32(alpha * acc[m,n]) + bias[n])        (App. B.5, reading Q16)
// Warps own TMEM lane quadrants (32 rows); TMA clips rows >= M and columns >= N.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "sm100.cuh"

namespace svdq {

__device__ __forceinline__ uint32_t pack2(float a, float b, int dt) {
  if (dt == 0)
    return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
           (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
  return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(a))) |
         (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(b))) << 16);
}

// Drains this warp's share of the tile: `NWQ` warps share a TMEM lane quadrant (32 rows) and
// take interleaved 32-column blocks.  All of the warp's tcgen05.ld are issued back to back
// and the accumulator is released (`release`) as soon as they complete, BEFORE any math or
// store: the MMA warp can then start the tile after next while this warp converts and stores
// (measured: releasing after the last 64-B chunk's store cost ~15 % of the issuer's time at
// K = 3072).  Each 64-byte column chunk (32 bf16/fp16 or 16 fp32 columns) is staged in a 2 KB
// buffer (two per warp) with the 64-byte swizzle of the store map (16-byte column j of row r
// at j ^ ((r >> 1) & 3)), then written by a TMA bulk tensor store.
template <int NCOLS, int NWQ, int NBUF = 2, typename Release>
__device__ __forceinline__ void epilogue_tile(uint32_t tmem_acc_lane, const float *bias_s, float alpha, int y_dtype,
                                              const CUtensorMap *tmY, int32_t row0, int32_t col0, int sub,
                                              uint8_t *stage, int &buf, int lane, Release release) {
  constexpr int NB = NCOLS / (32 * NWQ);                  // 32-column blocks per warp
  static_assert(NCOLS % (32 * NWQ) == 0, "column split");
  uint32_t r[NB][32];
#pragma unroll
  for (int i = 0; i < NB; ++i) tmem_ld_32x32b_x32(tmem_acc_lane + (sub + i * NWQ) * 32, r[i]);
  tmem_ld_wait();
  release();
#ifndef SVDQ_EXP
#define SVDQ_EXP 0
#endif
  if (SVDQ_EXP & 32) {                                   // ablation: TMEM drain only
    if (__uint_as_float(r[0][0]) == 1.2345f && __uint_as_float(r[NB - 1][31]) == 2.5f) buf ^= 1;
    return;
  }
  const uint32_t sw = static_cast<uint32_t>((lane >> 1) & 3);
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int cb = sub + i * NWQ;
    const float *bs = bias_s + cb * 32;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (y_dtype != 2 && h == 1) break;                  // 16-bit: one 64-B chunk per block
      uint8_t *sb = stage + (NBUF == 2 ? buf * 2048 : 0);
      if (lane == 0) bulk_wait_group_read<NBUF - 1>();   // the store that last used sb has read it
      __syncwarp();
      uint8_t *rowp = sb + lane * 64;
      if (y_dtype == 2) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float4 o;
          const int j = 16 * h + 4 * c;
          o.x = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][j + 0])), bs[j + 0]);
          o.y = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][j + 1])), bs[j + 1]);
          o.z = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][j + 2])), bs[j + 2]);
          o.w = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][j + 3])), bs[j + 3]);
          *reinterpret_cast<float4 *>(rowp + ((c ^ sw) * 16)) = o;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][8 * c + e])), bs[8 * c + e]);
          *reinterpret_cast<uint4 *>(rowp + ((c ^ sw) * 16)) =
              make_uint4(pack2(o[0], o[1], y_dtype), pack2(o[2], o[3], y_dtype), pack2(o[4], o[5], y_dtype),
                         pack2(o[6], o[7], y_dtype));
        }
      }
      fence_proxy_async();                                 // generic smem writes -> TMA (async proxy)
      __syncwarp();
      if (lane == 0 && !(SVDQ_EXP & 8)) {
        tma_store_2d(tmY, sb, col0 + cb * 32 + h * 16, row0);
        bulk_commit_group();
      }
      buf ^= 1;
    }
  }
}

// epilogue_tile for wide tiles (4 column blocks per warp, e.g. 384 columns over 3 warps per lane
// quadrant) within a 128-register budget: the first two blocks are loaded, scaled and packed to
// 16-bit pairs (16 registers each) before the last two are loaded; the accumulator is released
// after the last load, then all four blocks are staged and stored.  fp32 Y: block by block.
template <int NCOLS, int NWQ, int NBUF, typename Release>
__device__ __forceinline__ void epilogue_tile_wide(uint32_t tmem_acc_lane, const float *bias_s, float alpha, int y_dtype,
                                                   const CUtensorMap *tmY, int32_t row0, int32_t col0, int sub,
                                                   uint8_t *stage, int &buf, int lane, Release release) {
  constexpr int NB = NCOLS / (32 * NWQ);
  static_assert(NCOLS % (32 * NWQ) == 0 && NB == 4, "four column blocks per warp");
  const uint32_t sw = static_cast<uint32_t>((lane >> 1) & 3);
  auto stage_store = [&](int cb, int h, auto &&write_row) {
    uint8_t *sb = stage + (NBUF == 2 ? buf * 2048 : 0);
    if (lane == 0) bulk_wait_group_read<NBUF - 1>();     // the store that last used sb has read it
    __syncwarp();
    write_row(sb + lane * 64);
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmY, sb, col0 + cb * 32 + h * 16, row0);
      bulk_commit_group();
    }
    buf ^= 1;
  };
  if (y_dtype == 2) {
#pragma unroll 1
    for (int i = 0; i < NB; ++i) {
      const int cb = sub + i * NWQ;
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_acc_lane + cb * 32, r);
      tmem_ld_wait();
      if (i == NB - 1) release();
      const float *bs = bias_s + cb * 32;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        stage_store(cb, h, [&](uint8_t *rowp) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int j = 16 * h + 4 * c;
            *reinterpret_cast<float4 *>(rowp + ((c ^ sw) * 16)) =
                make_float4(__fadd_rn(__fmul_rn(alpha, __uint_as_float(r[j + 0])), bs[j + 0]),
                            __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[j + 1])), bs[j + 1]),
                            __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[j + 2])), bs[j + 2]),
                            __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[j + 3])), bs[j + 3]));
          }
        });
    }
    return;
  }
  uint32_t pk[2][16];
  {
    uint32_t r[2][32];
#pragma unroll
    for (int i = 0; i < 2; ++i) tmem_ld_32x32b_x32(tmem_acc_lane + (sub + i * NWQ) * 32, r[i]);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float *bs = bias_s + (sub + i * NWQ) * 32;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        pk[i][e] = pack2(__fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][2 * e])), bs[2 * e]),
                         __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][2 * e + 1])), bs[2 * e + 1]), y_dtype);
    }
  }
  uint32_t r2[2][32];
#pragma unroll
  for (int i = 0; i < 2; ++i) tmem_ld_32x32b_x32(tmem_acc_lane + (sub + (2 + i) * NWQ) * 32, r2[i]);
  tmem_ld_wait();
  release();
#pragma unroll
  for (int i = 0; i < 2; ++i)
    stage_store(sub + i * NWQ, 0, [&](uint8_t *rowp) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4 *>(rowp + ((c ^ sw) * 16)) =
            make_uint4(pk[i][4 * c], pk[i][4 * c + 1], pk[i][4 * c + 2], pk[i][4 * c + 3]);
    });
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int cb = sub + (2 + i) * NWQ;
    const float *bs = bias_s + cb * 32;
    stage_store(cb, 0, [&](uint8_t *rowp) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r2[i][8 * c + e])), bs[8 * c + e]);
        *reinterpret_cast<uint4 *>(rowp + ((c ^ sw) * 16)) =
            make_uint4(pack2(o[0], o[1], y_dtype), pack2(o[2], o[3], y_dtype), pack2(o[4], o[5], y_dtype),
                       pack2(o[6], o[7], y_dtype));
      }
    });
  }
}

// W8A8 (the paper's 8-bit setting) epilogue of the CTA-pair kernel: the exact int32
// accumulator of X_q W_q^T in TMEM columns [0, NCOLS) and the fp32 low-rank accumulator in
// [lr_col, lr_col + NCOLS) of this warp's lanes:
//   Y[m,n] = out_rn(fma(fl32(f32(acc[m,n]) * sx[m]), sw[n], lr[m,n]) + bias[n])
// -- the 1-CTA kernel's formula, operation for operation (readings W2 / W3).  |acc| may exceed
// 2^24 over a whole K: the int -> fp32 conversion rounds to nearest.  Block by block: the
// accumulator is released after the last block's loads; staging / TMA stores as epilogue_tile.
template <int NCOLS, int NWQ, int NBUF = 2, typename Release>
__device__ __forceinline__ void epilogue_tile_w8(uint32_t tmem_acc_lane, uint32_t lr_col, bool has_lr,
                                                 const float *bias_s, const float *sw_s, float sx, int y_dtype,
                                                 const CUtensorMap *tmY, int32_t row0, int32_t col0, int sub,
                                                 uint8_t *stage, int &buf, int lane, Release release) {
  constexpr int NB = NCOLS / (32 * NWQ);
  static_assert(NCOLS % (32 * NWQ) == 0, "column split");
  const uint32_t sw = static_cast<uint32_t>((lane >> 1) & 3);
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int cb = sub + i * NWQ;
    uint32_t ra[32], rl[32];
    tmem_ld_32x32b_x32(tmem_acc_lane + cb * 32, ra);
    if (has_lr) tmem_ld_32x32b_x32(tmem_acc_lane + lr_col + cb * 32, rl);
    tmem_ld_wait();
    if (i == NB - 1) release();
    const float *bs = bias_s + cb * 32;
    const float *ws = sw_s + cb * 32;
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float t = __fmul_rn(__int2float_rn(static_cast<int>(ra[e])), sx);
      v[e] = __fadd_rn(__fmaf_rn(t, ws[e], has_lr ? __uint_as_float(rl[e]) : 0.f), bs[e]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (y_dtype != 2 && h == 1) break;                  // 16-bit: one 64-B chunk per block
      uint8_t *sb = stage + (NBUF == 2 ? buf * 2048 : 0);
      if (lane == 0) bulk_wait_group_read<NBUF - 1>();   // the store that last used sb has read it
      __syncwarp();
      uint8_t *rowp = sb + lane * 64;
      if (y_dtype == 2) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<float4 *>(rowp + ((c ^ sw) * 16)) =
              make_float4(v[16 * h + 4 * c], v[16 * h + 4 * c + 1], v[16 * h + 4 * c + 2], v[16 * h + 4 * c + 3]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4 *>(rowp + ((c ^ sw) * 16)) =
              make_uint4(pack2(v[8 * c], v[8 * c + 1], y_dtype), pack2(v[8 * c + 2], v[8 * c + 3], y_dtype),
                         pack2(v[8 * c + 4], v[8 * c + 5], y_dtype), pack2(v[8 * c + 6], v[8 * c + 7], y_dtype));
      }
      fence_proxy_async();                                 // generic smem writes -> TMA (async proxy)
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmY, sb, col0 + cb * 32 + h * 16, row0);
        bulk_commit_group();
      }
      buf ^= 1;
    }
  }
}

// Direct variant: no shared-memory staging and no TMA store.  Lane l of the warp owns row
// row0 + l; each 32-column block becomes 64 contiguous bytes of that row (four 16-byte
// st.global, or eight for fp32), so every store fills whole 32-byte sectors.  Rows >= M and
// column groups >= N are skipped (N % 16 == 0, so 16-byte groups never straddle N for 16-bit
// outputs; fp32 groups are 4 columns).
template <int NCOLS, int NWQ, typename Release>
__device__ __forceinline__ void epilogue_tile_direct(uint32_t tmem_acc_lane, const float *bias_s, float alpha,
                                                     int y_dtype, void *Y, int64_t ldy, int64_t M, int64_t N,
                                                     int64_t row0, int64_t col0, int sub, int lane,
                                                     Release release) {
  constexpr int NB = NCOLS / (32 * NWQ);
  static_assert(NCOLS % (32 * NWQ) == 0, "column split");
  uint32_t r[NB][32];
#pragma unroll
  for (int i = 0; i < NB; ++i) tmem_ld_32x32b_x32(tmem_acc_lane + (sub + i * NWQ) * 32, r[i]);
  tmem_ld_wait();
  release();
  const int64_t row = row0 + lane;
  if (row >= M) return;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int cb = sub + i * NWQ;
    const int64_t c0 = col0 + cb * 32;
    const float *bs = bias_s + cb * 32;
    if (y_dtype == 2) {
      float *yp = static_cast<float *>(Y) + row * ldy + c0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c0 + 4 * c >= N) break;
        float4 o;
        o.x = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][4 * c + 0])), bs[4 * c + 0]);
        o.y = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][4 * c + 1])), bs[4 * c + 1]);
        o.z = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][4 * c + 2])), bs[4 * c + 2]);
        o.w = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][4 * c + 3])), bs[4 * c + 3]);
        reinterpret_cast<float4 *>(yp)[c] = o;
      }
    } else {
      uint16_t *yp = static_cast<uint16_t *>(Y) + row * ldy + c0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c0 + 8 * c >= N) break;
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(__fmul_rn(alpha, __uint_as_float(r[i][8 * c + e])), bs[8 * c + e]);
        reinterpret_cast<uint4 *>(yp)[c] = make_uint4(pack2(o[0], o[1], y_dtype), pack2(o[2], o[3], y_dtype),
                                                      pack2(o[4], o[5], y_dtype), pack2(o[6], o[7], y_dtype));
      }
    }
  }
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// GELU, tanh form, in fp32 (reading N1; the oracle evaluates it in fp64):
// 0.5 v (1 + tanh(u)) = v / (1 + exp(-2u)), u = sqrt(2/pi) (v + 0.044715 v^3) -- one ex2 and one
// reciprocal (a few fp32 ulp; the value is then rounded to bf16)
__device__ __forceinline__ float gelu_tanh_f(float v) {
  const float u2 = -2.0f * 0.7978845608028654f * fmaf(0.044715f * v, v * v, v);
  return __fdividef(v, 1.0f + exp2f(u2 * 1.4426950408889634f));
}

// epilogue_tile plus the next layer's K1.  Lane l of the warp owns row
// row0 + l; for each of its 32-column blocks it forms the stored bf16 output y, the next
// layer's input a = y or bf16(gelu(y)), x_hat = fl32(a * lambda_inv_next) and, per 16-column
// group, the NVFP4 scale factor and codes with K1's exact recipe (reading Q10), and writes a
// into the a tile (atile, row row_l of this CTA) that the MMA warp multiplies by L1s_next.
// tmY == nullptr: Y is not stored.  lamn_s: the tile's 192 lambda_inv_next values (0 past N).  Rows >= M store no codes; their scale factors (padding rows of the 128x4
// layout) are written 0x00 (reading Q22).
// The codes and scale factors are kept in registers and stored to global memory only after
// `mid()` (the a-tile hand-off): a release-arrive waits for this thread's outstanding global
// stores (ncu: ERRBAR before SYNCS.ARRIVE was the epilogue's top stall).
template <int NCOLS, int NWQ, int NBUF = 2, typename Release, typename Mid>
__device__ __forceinline__ void epilogue_tile_next(uint32_t tmem_acc_lane, const float *bias_s, float alpha,
                                                   const CUtensorMap *tmY, int32_t row0, int32_t col0, int sub,
                                                   uint8_t *stage, int &buf, int lane, Release release,
                                                   const K2Params &p, const float *lamn_s, uint8_t *atile,
                                                   int row_l, Mid mid, uint8_t *cstage, uint8_t *sfstage, int quad) {
  constexpr int NB = NCOLS / (32 * NWQ);
  uint32_t cw[NB][4], sfw[NB][2];
  static_assert(NCOLS % (32 * NWQ) == 0, "column split");
  const uint32_t sw = static_cast<uint32_t>((lane >> 1) & 3);
  const int64_t row = static_cast<int64_t>(row0) + lane;
  const int64_t N = p.N;
  const float t6 = __fmul_rn(__fdiv_rn(1.0f, p.nx_gs), __fdiv_rn(1.0f, 6.0f));
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int cb = sub + i * NWQ;
    const float *bs = bias_s + cb * 32;
    // one 32-column block at a time (register budget: 10 warps -> 168 per thread); the
    // accumulator is released after the last block's load (measured: loading all blocks first
    // and packing y to bf16 pairs, to release earlier, was 7 % slower with GELU + rank 32)
    uint32_t rr[32];
    tmem_ld_32x32b_x32(tmem_acc_lane + cb * 32, rr);
    tmem_ld_wait();
    if (i == NB - 1) release();
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float o = __fadd_rn(__fmul_rn(alpha, __uint_as_float(rr[e])), bs[e]);
      rr[e] = __float_as_uint(__bfloat162float(__float2bfloat16_rn(o)));      // y, as stored
    }
    if (tmY) {                                              // the layer's own output, as epilogue_tile
      uint8_t *sb = stage + (NBUF == 2 ? buf * 2048 : 0);
      if (lane == 0) bulk_wait_group_read<NBUF - 1>();
      __syncwarp();
      uint8_t *rowp = sb + lane * 64;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float *v = reinterpret_cast<const float *>(&rr[8 * c]);
        *reinterpret_cast<uint4 *>(rowp + ((c ^ sw) * 16)) =
            make_uint4(pack2(v[0], v[1], 0), pack2(v[2], v[3], 0), pack2(v[4], v[5], 0), pack2(v[6], v[7], 0));
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmY, sb, col0 + cb * 32, row0);
        bulk_commit_group();
      }
      buf ^= 1;
    }
    float *a = reinterpret_cast<float *>(rr);
    // the next layer's input a
    if (p.nx_act) {
#pragma unroll
      for (int e = 0; e < 32; ++e) a[e] = __bfloat162float(__float2bfloat16_rn(gelu_tanh_f(a[e])));
    }
    // next layer's NVFP4 codes and scale factors, two 16-column groups
#ifndef SVDQ_FUSE_EXP
#define SVDQ_FUSE_EXP 0
#endif
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float xh[16];
      float amax = 0.f;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        xh[e] = __fmul_rn(a[16 * h + e], lamn_s[cb * 32 + 16 * h + e]);
        amax = fmaxf(amax, fabsf(xh[e]));
      }
      const uint32_t sf = e4m3_rn_sat(__fmul_rn(amax, t6));
      const float sd = e4m3_to_f32(sf);
      const float qinv = sd == 0.f ? 0.f : __fdiv_rn(1.0f, __fmul_rn(sd, p.nx_gs));
      float q0[8], q1[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        q0[e] = __fmul_rn(xh[e], qinv);
        q1[e] = __fmul_rn(xh[8 + e], qinv);
      }
      cw[i][2 * h] = e2m1x8(q0);
      cw[i][2 * h + 1] = e2m1x8(q1);
      sfw[i][h] = sf;
    }
    // a (bf16) into the CTA's a tile for the X L1s_next^T MMA: 3 chunks of [128 rows x 64 cols],
    // K-major with the 128-byte swizzle (16-byte unit u of row r at u ^ (r & 7))
    if (atile) {
      const uint32_t rowp = smem_u32(atile) + (cb >> 1) * 16384 + row_l * 128;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int u = (cb & 1) * 4 + c;
        sts128(rowp + ((u ^ (row_l & 7)) << 4), pack2(a[8 * c], a[8 * c + 1], 0), pack2(a[8 * c + 2], a[8 * c + 3], 0),
               pack2(a[8 * c + 4], a[8 * c + 5], 0), pack2(a[8 * c + 6], a[8 * c + 7], 0));
      }
    }
  }
  mid();
  // the next layer's codes / scale factors into the CTA's staging buffers (one TMA tensor store of
  // the [128 x 96 B] code tile and one bulk copy of the tile's three 512-B scale-factor blocks of
  // the 128x4 layout follow in the kernel): row_l's 16-column group g (0..11) -> codes at
  // row_l * 96 + 8 g, scale factor at (g / 4) * 512 + (row_l & 31) * 16 + quad * 4 + g % 4.
  // Rows >= M store 0x00 scale factors (padding rows, reading Q22).
  const bool in_m = row < p.M;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int cb = sub + i * NWQ;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = cb * 2 + h;
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_u32(cstage) + row_l * 96 + 8 * g),
                   "r"(cw[i][2 * h]), "r"(cw[i][2 * h + 1]) : "memory");
      asm volatile("st.shared.u8 [%0], %1;" ::"r"(smem_u32(sfstage) + (g >> 2) * 512 + (row_l & 31) * 16 + quad * 4 +
                                                  (g & 3)),
                   "r"(in_m ? sfw[i][h] : 0u) : "memory");
    }
  }
  fence_proxy_async();
}

}  // namespace svdq
