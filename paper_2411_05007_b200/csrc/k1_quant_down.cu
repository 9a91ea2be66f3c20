// K1: fused smoothing + activation quantization + low-rank down-projection
// ("Fused Quantize + Down Projection", Fig. 5(b)).
//
// One HBM read of X serves three things:
//   x_hat = fl32(x * lambda_inv)                       (reading Q14)
//   codes/scales of Q(x_hat): NVFP4 g16 or INT4 g64    (Eq. 1; App. B)
//   xl1 = bf16(x . L1s^T), fp32 accumulation on tensor cores (Q15, Q18)
//
// Layout of the work: a CTA owns BM = 16*MT rows; its 8 warps split K into
// contiguous ranges of 64-wide blocks.  Lane (g = lane/4, q = lane%4) loads
// 8 contiguous 16-bit values x[row][kb*64 + c*32 + 8q .. +7] with one 128-bit
// load for rows g and g+8 of each 16-row tile.  The same registers feed
//  * the quantizer: an NVFP4 group of 16 is lanes {q, q^1} (one shfl), an INT4
//    group of 64 is the 4 lanes of g over both 32-chunks (two shfls);
//  * mma.sync m16n8k16 (bf16): the fragment's k-labels are only pairing tags,
//    so feeding A and B (L1s rows, loaded the same way) from the same
//    contiguous loads sums over a consistent permutation of the 32-chunk.
// Per-warp partial xl1 tiles are reduced across warps in fixed order
// (deterministic), rounded to bf16 and stored.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "k1_launch.h"
#include "sm100.cuh"

namespace svdq {

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1,
                                               uint32_t a2, uint32_t a3, uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ldg_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_keep(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <bool kBf16>
__device__ __forceinline__ float x16_to_f32(uint32_t bits16) {
  if constexpr (kBf16) return __uint_as_float(bits16 << 16);
  else return __half2float(__ushort_as_half(static_cast<uint16_t>(bits16)));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(lo))) |
         (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(hi))) << 16);
}

// kFmt: 0 = NVFP4, 1 = INT4, 2 = down-projection only.  kXBf16: X dtype bf16 (else fp16).
// kScaleBf16: INT4 scale dtype.  MT: 16-row tiles per CTA.  NT: rank / 8.
template <int kFmt, bool kXBf16, bool kScaleBf16, int MT, int NT>
__global__ void __launch_bounds__(256, 1)
    k1_quant_down_kernel(K1Params p) {
  constexpr int BM = 16 * MT;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2;
  const int q = lane & 3;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t K = p.K;
  const int nkb = static_cast<int>(K / 64);
  const int kb_begin = (warp * nkb) / 8;
  const int kb_end = ((warp + 1) * nkb) / 8;
  const uint16_t *X = static_cast<const uint16_t *>(p.X);

  float acc[MT][NT > 0 ? NT : 1][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < (NT > 0 ? NT : 1); ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[mt][nt][i] = 0.f;

  // NVFP4 constants (App. B.2): t = fl32(fl32(1/gs) * fl32(1/6))
  griddep_launch_dependents();
  griddep_wait();                                    // X may be the previous kernel's output
  const float enc = __fdiv_rn(1.0f, p.gs_x);
  const float t6 = __fmul_rn(enc, __fdiv_rn(1.0f, 6.0f));

  for (int kb = kb_begin; kb < kb_end; ++kb) {
    uint4 xv[MT][2][2];    // [mt][half][chunk]
    uint4 lv[NT > 0 ? NT : 1][2];
    float lam[2][8];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t k0 = static_cast<int64_t>(kb) * 64 + c * 32 + q * 8;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t row = row0 + mt * 16 + h * 8 + g;
          xv[mt][h][c] = row < p.M ? ldg_stream(X + row * p.ldx + k0) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        lv[nt][c] = ldg_keep(p.l1s + static_cast<int64_t>(nt * 8 + g) * K + k0);
      const float4 l0 = *reinterpret_cast<const float4 *>(p.lam_inv + k0);
      const float4 l1 = *reinterpret_cast<const float4 *>(p.lam_inv + k0 + 4);
      lam[c][0] = l0.x; lam[c][1] = l0.y; lam[c][2] = l0.z; lam[c][3] = l0.w;
      lam[c][4] = l1.x; lam[c][5] = l1.y; lam[c][6] = l1.z; lam[c][7] = l1.w;
    }

    // ---------------- down-projection on tensor cores
    if constexpr (NT > 0) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const uint4 a_lo = xv[mt][0][c];   // row g
          const uint4 a_hi = xv[mt][1][c];   // row g + 8
          if constexpr (kXBf16) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              mma_bf16_16816(acc[mt][nt], a_lo.x, a_hi.x, a_lo.y, a_hi.y, lv[nt][c].x, lv[nt][c].y);
              mma_bf16_16816(acc[mt][nt], a_lo.z, a_hi.z, a_lo.w, a_hi.w, lv[nt][c].z, lv[nt][c].w);
            }
          } else {
            // fp16 X: exact split x = hi + lo with hi, lo bf16 (11-bit -> 8 + 8 bits).
            uint32_t ah[2][4], al[2][4];
            const uint32_t w[2][4] = {{a_lo.x, a_lo.y, a_lo.z, a_lo.w}, {a_hi.x, a_hi.y, a_hi.z, a_hi.w}};
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float f0 = x16_to_f32<false>(w[h][j] & 0xFFFF);
                const float f1 = x16_to_f32<false>(w[h][j] >> 16);
                const float h0 = __bfloat162float(__float2bfloat16_rn(f0));
                const float h1 = __bfloat162float(__float2bfloat16_rn(f1));
                ah[h][j] = pack_bf16x2(h0, h1);
                al[h][j] = pack_bf16x2(f0 - h0, f1 - h1);
              }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              mma_bf16_16816(acc[mt][nt], ah[0][0], ah[1][0], ah[0][1], ah[1][1], lv[nt][c].x, lv[nt][c].y);
              mma_bf16_16816(acc[mt][nt], ah[0][2], ah[1][2], ah[0][3], ah[1][3], lv[nt][c].z, lv[nt][c].w);
              mma_bf16_16816(acc[mt][nt], al[0][0], al[1][0], al[0][1], al[1][1], lv[nt][c].x, lv[nt][c].y);
              mma_bf16_16816(acc[mt][nt], al[0][2], al[1][2], al[0][3], al[1][3], lv[nt][c].z, lv[nt][c].w);
            }
          }
        }
    }

    // ---------------- smoothing + quantization (kFmt 2: down-projection only, W8A8 codes
    // come from k1_int8_rows)
    if constexpr (kFmt == 2) continue;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t row = row0 + mt * 16 + h * 8 + g;
        float xh[2][8];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const uint32_t w4[4] = {xv[mt][h][c].x, xv[mt][h][c].y, xv[mt][h][c].z, xv[mt][h][c].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            xh[c][2 * j] = __fmul_rn(x16_to_f32<kXBf16>(w4[j] & 0xFFFF), lam[c][2 * j]);
            xh[c][2 * j + 1] = __fmul_rn(x16_to_f32<kXBf16>(w4[j] >> 16), lam[c][2 * j + 1]);
          }
        }
        if constexpr (kFmt == 0) {
          // NVFP4: group of 16 = lanes q, q^1 of one 32-chunk
          uint32_t sfb[2];
          uint32_t codes[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            float amax = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) amax = fmaxf(amax, fabsf(xh[c][j]));
            amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
            const uint32_t sf = e4m3_rn_sat(__fmul_rn(amax, t6));
            const float sfd = e4m3_to_f32(sf);
            const float qinv = sfd == 0.f ? 0.f : __fdiv_rn(1.0f, __fmul_rn(sfd, p.gs_x));
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = __fmul_rn(xh[c][j], qinv);
            codes[c] = e2m1x8(v);
            sfb[c] = sf;
          }
          // gather the 4 scale bytes of this row's 64-block into lane q == 0
          const uint32_t o0 = __shfl_down_sync(0xffffffffu, sfb[0], 2);
          const uint32_t o1 = __shfl_down_sync(0xffffffffu, sfb[1], 2);
          if (row < p.M) {
#pragma unroll
            for (int c = 0; c < 2; ++c)
              *reinterpret_cast<uint32_t *>(p.xq + row * (K / 2) + (kb * 64 + c * 32 + q * 8) / 2) =
                  codes[c];
          }
          if (q == 0 && row < p.Mpad) {
            const uint32_t word = sfb[0] | (o0 << 8) | (sfb[1] << 16) | (o1 << 24);
            *reinterpret_cast<uint32_t *>(p.xs + sf_offset(row, kb * 4, K)) = word;
          }
        } else {
          // INT4: group of 64 = 4 lanes x 2 chunks
          float amax = 0.f;
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int j = 0; j < 8; ++j) amax = fmaxf(amax, fabsf(xh[c][j]));
          amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
          amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
          const uint16_t s = scale16_rn_sat<kScaleBf16>(__fdiv_rn(amax, 7.0f));
          const float sd = scale16_to_f32<kScaleBf16>(s);
          const float qinv = sd == 0.f ? 0.f : __fdiv_rn(1.0f, sd);
          if (row < p.M) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t word = 0;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                int v = __float2int_rn(__fmul_rn(xh[c][j], qinv));
                v = max(-7, min(7, v));
                word |= (static_cast<uint32_t>(v) & 0xFu) << (4 * j);
              }
              *reinterpret_cast<uint32_t *>(p.xq + row * (K / 2) + (kb * 64 + c * 32 + q * 8) / 2) =
                  word;
            }
            if (q == 0) reinterpret_cast<uint16_t *>(p.xs)[row * (K / 64) + kb] = s;
          }
        }
      }
  }

  // ---------------- deterministic cross-warp reduction of the xl1 partials
  if constexpr (NT > 0) {
    constexpr int R = NT * 8;
    extern __shared__ float red[];   // [8 warps][BM][R]
    float *mine = red + warp * BM * R;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int r0 = mt * 16 + g;
        const int c0 = nt * 8 + 2 * q;
        mine[r0 * R + c0] = acc[mt][nt][0];
        mine[r0 * R + c0 + 1] = acc[mt][nt][1];
        mine[(r0 + 8) * R + c0] = acc[mt][nt][2];
        mine[(r0 + 8) * R + c0 + 1] = acc[mt][nt][3];
      }
    __syncthreads();
    for (int i = threadIdx.x; i < BM * R / 2; i += 256) {
      const int e = 2 * i;
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        s0 += red[w * BM * R + e];
        s1 += red[w * BM * R + e + 1];
      }
      const int rl = e / R;
      const int col = e % R;
      const int64_t row = row0 + rl;
      if (row < p.M)
        *reinterpret_cast<uint32_t *>(p.xl1 + row * R + col) = pack_bf16x2(s0, s1);
    }
  }
}

template <int kFmt, bool kXBf16, bool kScaleBf16, int MT, int NT>
static cudaError_t launch_k1_t(const K1Params &p, cudaStream_t stream) {
  constexpr int BM = 16 * MT;
  const size_t smem = NT > 0 ? static_cast<size_t>(8) * BM * NT * 8 * sizeof(float) : 0;
  auto kern = k1_quant_down_kernel<kFmt, kXBf16, kScaleBf16, MT, NT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const unsigned grid = static_cast<unsigned>(p.Mpad / BM);
  return launch_ex(kern, dim3(grid), dim3(256), smem, stream, 1u, p);
}

template <int kFmt, bool kXBf16, bool kScaleBf16, int MT>
static cudaError_t dispatch_rank(const K1Params &p, cudaStream_t s) {
  switch (p.rank / 8) {
    case 0: return launch_k1_t<kFmt, kXBf16, kScaleBf16, MT, 0>(p, s);
    case 2: return launch_k1_t<kFmt, kXBf16, kScaleBf16, MT, 2>(p, s);
    case 4: return launch_k1_t<kFmt, kXBf16, kScaleBf16, MT, 4>(p, s);
    case 6: return launch_k1_t<kFmt, kXBf16, kScaleBf16, MT, 6>(p, s);
    case 8: return launch_k1_t<kFmt, kXBf16, kScaleBf16, MT, 8>(p, s);
    case 10: return launch_k1_t<kFmt, kXBf16, kScaleBf16, 1, 10>(p, s);
    case 12: return launch_k1_t<kFmt, kXBf16, kScaleBf16, 1, 12>(p, s);
    case 14: return launch_k1_t<kFmt, kXBf16, kScaleBf16, 1, 14>(p, s);
    case 16: return launch_k1_t<kFmt, kXBf16, kScaleBf16, 1, 16>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int kFmt, bool kXBf16, bool kScaleBf16>
static cudaError_t dispatch_mt(const K1Params &p, cudaStream_t s) {
  // two 16-row tiles per CTA when that still gives about a wave of CTAs
  if (p.Mpad / 32 >= 120 && p.rank <= 64) return dispatch_rank<kFmt, kXBf16, kScaleBf16, 2>(p, s);
  return dispatch_rank<kFmt, kXBf16, kScaleBf16, 1>(p, s);
}

cudaError_t launch_k1(const K1Params &p, cudaStream_t s) {
  if (p.fmt == 2) return p.x_bf16 ? dispatch_mt<2, true, true>(p, s) : dispatch_mt<2, false, true>(p, s);
  if (p.fmt == 0) {
    return p.x_bf16 ? dispatch_mt<0, true, true>(p, s) : dispatch_mt<0, false, true>(p, s);
  }
  if (p.x_bf16)
    return p.scale_bf16 ? dispatch_mt<1, true, true>(p, s) : dispatch_mt<1, true, false>(p, s);
  return p.scale_bf16 ? dispatch_mt<1, false, true>(p, s) : dispatch_mt<1, false, false>(p, s);
}

}  // namespace svdq
