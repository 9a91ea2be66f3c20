// K2 (NVFP4): fused 4-bit GEMM + low-rank up-projection + bias
// ("Fused 4-Bit Compute + Up Projection", Fig. 5(b); Eq. 5).
//
//   acc[m,n]  = sum_g sfa[m,g] sfb[n,g] sum_{k in g} e2m1(qa[m,k]) e2m1(qb[n,k])
//               (tcgen05.mma kind::mxf4nvf4.block_scale.scale_vec::4X, K = 64 / instr)
//             + sum_t xl1[m,t] l2s[n,t]
//               (tcgen05.mma kind::f16, bf16 -> fp32, into the SAME TMEM accumulator:
//                the up-projection is one extra K-slab, so Y is written once)
//   Y[m,n]    = out_rn(fl32(alpha * acc) + bias[n]),  alpha = gs_x * gs_w
//
// Structure: one 128 x BN output tile per CTA, warp-specialized.
//   warp 0      TMA producer: A/B code tiles (128-B swizzle), SFA/SFB chunks (bulk copy),
//               then ceil(rank/64) low-rank slabs (xl1 / l2s tiles, zero-filled past rank)
//               into the same smem ring.
//   warp 1      TMEM allocator + single-thread MMA issuer: tcgen05.cp of the scale
//               factors smem -> TMEM, tcgen05.mma, tcgen05.commit releases smem stages.
//   warps 2..5  epilogue: tcgen05.ld -> alpha, bias -> 16-bit -> global.
// TMEM (512 columns): accumulator [0, BN); per-stage scale-factor columns after it.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "k1_launch.h"
#include "sm100.cuh"

namespace svdq {

template <int BN>
struct NvCfg {
  static constexpr int BM = 128;
  static constexpr int BKB = 128;                       // bytes of K per stage (256 fp4)
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BKB;              // 16 KB
  static constexpr int B_BYTES = BN * BKB;
  static constexpr int SFA_BYTES = 4 * 512;             // 128 rows x 16 sf
  static constexpr int SFB_BYTES = (BN / 128) * 4 * 512;
  static constexpr int STAGE = A_BYTES + B_BYTES + SFA_BYTES + SFB_BYTES;
  static constexpr int SF_COLS = 16 + BN / 8;           // TMEM columns per stage
  static constexpr int SMEM = kStages * STAGE + 1024 + 256;
  static_assert(STAGE % 1024 == 0, "stage must keep 1024-B alignment");
  static_assert(BN + kStages * SF_COLS <= 512, "TMEM budget");
};

__device__ __forceinline__ float load_bias(const void *b, int dt, int64_t i) {
  if (dt == 0) return __bfloat162float(static_cast<const __nv_bfloat16 *>(b)[i]);
  if (dt == 1) return __half2float(static_cast<const __half *>(b)[i]);
  return static_cast<const float *>(b)[i];
}

// Store 8 consecutive fp32 outputs at Y[row][col .. col+7].
__device__ __forceinline__ void store8(void *Y, int dt, int64_t ldy, int64_t row, int64_t col,
                                       const float (&v)[8]) {
  if (dt == 2) {
    float4 *p = reinterpret_cast<float4 *>(static_cast<float *>(Y) + row * ldy + col);
    p[0] = make_float4(v[0], v[1], v[2], v[3]);
    p[1] = make_float4(v[4], v[5], v[6], v[7]);
    return;
  }
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (dt == 0) {
      w[j] = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * j]))) |
             (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * j + 1]))) << 16);
    } else {
      w[j] = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v[2 * j]))) |
             (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v[2 * j + 1]))) << 16);
    }
  }
  *reinterpret_cast<uint4 *>(static_cast<uint16_t *>(Y) + row * ldy + col) =
      make_uint4(w[0], w[1], w[2], w[3]);
}

template <int BN>
__global__ void __launch_bounds__(192, 1)
    k2_nvfp4_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmL,
                    const K2Params p) {
  using C = NvCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::kStages * C::STAGE);
  uint64_t *empty = full + C::kStages;
  uint64_t *accum_full = empty + C::kStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accum_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * C::BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.y) * BN;
  const int nkb64 = static_cast<int>(p.K / 64);        // 64-wide K blocks
  const int nkt = (nkb64 + 3) / 4;                     // pipeline K steps
  const int nslab = (p.rank + 63) / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum_full, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (nslab) {
      tma_prefetch(&tmX);
      tma_prefetch(&tmL);
    }
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      const int64_t mt = m0 / 128;
      for (int kt = 0; kt < nkt; ++kt) {
        const int nsub = min(4, nkb64 - kt * 4);
        int nsfb = 0;
        for (int h = 0; h < BN / 128; ++h)
          if (n0 + h * 128 < p.Npad) ++nsfb;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t *st = smem + s * C::STAGE;
        mbar_arrive_expect_tx(&full[s], C::A_BYTES + C::B_BYTES + nsub * 512 * (1 + nsfb));
        tma_load_2d(st, &tmA, &full[s], kt * C::BKB, static_cast<int32_t>(m0));
        tma_load_2d(st + C::A_BYTES, &tmB, &full[s], kt * C::BKB, static_cast<int32_t>(n0));
        bulk_load(st + C::A_BYTES + C::B_BYTES, p.sfa + (mt * nkb64 + kt * 4) * 512, nsub * 512,
                  &full[s]);
        for (int h = 0; h < nsfb; ++h)
          bulk_load(st + C::A_BYTES + C::B_BYTES + C::SFA_BYTES + h * 2048,
                    p.sfb + ((n0 / 128 + h) * nkb64 + kt * 4) * 512, nsub * 512, &full[s]);
        if (++s == C::kStages) { s = 0; ph ^= 1; }
      }
      for (int j = 0; j < nslab; ++j) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t *st = smem + s * C::STAGE;
        mbar_arrive_expect_tx(&full[s], C::BM * 128 + BN * 128);
        tma_load_2d(st, &tmX, &full[s], j * 64, static_cast<int32_t>(m0));
        tma_load_2d(st + C::A_BYTES, &tmL, &full[s], j * 64, static_cast<int32_t>(n0));
        if (++s == C::kStages) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_q = idesc_nvfp4(128, BN);
    constexpr uint32_t idesc_h = idesc_bf16(128, BN);
    int s = 0;
    uint32_t ph = 0;
    for (int kt = 0; kt < nkt; ++kt) {
      const int nsub = min(4, nkb64 - kt * 4);
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        uint8_t *st = smem + s * C::STAGE;
        const uint32_t a_addr = smem_u32(st);
        const uint32_t b_addr = smem_u32(st + C::A_BYTES);
        const uint32_t sfa_addr = smem_u32(st + C::A_BYTES + C::B_BYTES);
        const uint32_t sfb_addr = sfa_addr + C::SFA_BYTES;
        const uint32_t sf_col = tmem + BN + s * C::SF_COLS;
        const uint32_t sfa_col = sf_col;
        const uint32_t sfb_col = sf_col + 16;
        for (int i = 0; i < nsub; ++i) {
          tmem_cp_32x128b_warpx4(sfa_col + 4 * i, sdesc_cp_32x128b(sfa_addr + i * 512));
#pragma unroll
          for (int h = 0; h < BN / 128; ++h)
            tmem_cp_32x128b_warpx4(sfb_col + i * (BN / 32) + 4 * h,
                                   sdesc_cp_32x128b(sfb_addr + h * 2048 + i * 512));
        }
        for (int i = 0; i < nsub; ++i) {
          mma_nvfp4(tmem, sdesc_kmajor_sw128(a_addr + 32 * i), sdesc_kmajor_sw128(b_addr + 32 * i),
                    idesc_q, sfa_col + 4 * i, sfb_col + i * (BN / 32), (kt | i) != 0);
        }
        tc_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == C::kStages) { s = 0; ph ^= 1; }
    }
    for (int j = 0; j < nslab; ++j) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        uint8_t *st = smem + s * C::STAGE;
        const uint32_t a_addr = smem_u32(st);
        const uint32_t b_addr = smem_u32(st + C::A_BYTES);
        const int nk16 = min(4, (p.rank - j * 64) / 16);
        for (int i = 0; i < nk16; ++i)
          mma_bf16(tmem, sdesc_kmajor_sw128(a_addr + 32 * i), sdesc_kmajor_sw128(b_addr + 32 * i),
                   idesc_h, (nkt > 0 || j > 0 || i > 0) ? 1u : 0u);
        tc_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == C::kStages) { s = 0; ph ^= 1; }
    }
    if (elect_one()) tc_commit(accum_full);
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    const int64_t grow = m0 + row;
    mbar_wait(accum_full, 0);
    tc_fence_after();
#pragma unroll 1
    for (int cc = 0; cc < BN / 32; ++cc) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + cc * 32, r);
      tmem_ld_wait();
      if (grow < p.M) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t col = n0 + cc * 32 + j * 8;
          if (col < p.N) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float y = __fmul_rn(p.alpha, __uint_as_float(r[j * 8 + e]));
              if (p.bias) y = __fadd_rn(y, load_bias(p.bias, p.bias_dtype, col + e));
              v[e] = y;
            }
            store8(p.Y, p.y_dtype, p.ldy, grow, col, v);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int BN>
static cudaError_t launch_bn(const K2Maps &maps, const K2Params &p, cudaStream_t s) {
  using C = NvCfg<BN>;
  auto kern = k2_nvfp4_kernel<BN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>((p.M + 127) / 128), static_cast<unsigned>((p.N + BN - 1) / BN));
  kern<<<grid, 192, C::SMEM, s>>>(maps.a, maps.b, maps.xl1, maps.l2, p);
  return cudaGetLastError();
}

int k2_nvfp4_bn(int64_t M, int64_t N) {
  // 256-wide tiles when there are enough of them to fill the machine.
  const int64_t tiles256 = ((M + 127) / 128) * ((N + 255) / 256);
  return tiles256 >= 148 ? 256 : 128;
}

cudaError_t launch_k2_nvfp4(const K2Maps &maps, const K2Params &p, cudaStream_t s) {
  return k2_nvfp4_bn(p.M, p.N) == 256 ? launch_bn<256>(maps, p, s) : launch_bn<128>(maps, p, s);
}

}  // namespace svdq
