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
// Persistent, warp-specialized; one CTA per SM walks 128 x BN output tiles.
//   warp 0      TMA producer: A/B code tiles (128-B swizzle) and SFA/SFB 512-B chunks
//               (bulk copies) into a kStages ring, then ceil(rank/64) low-rank slabs
//               (xl1 / l2s tiles, zero-filled past rank) into the same ring.
//   warp 1      TMEM allocator + single-thread MMA issuer.  Scale factors go
//               smem -> TMEM (tcgen05.cp) into one of two SF slots; a slot is reused
//               only after the MMAs that read it completed.  The accumulator is double
//               buffered so the epilogue of tile i overlaps the main loop of tile i+1.
//   warps 2..5  epilogue: tcgen05.ld -> alpha, bias -> 16-bit -> global; releases the
//               accumulator buffer to the MMA warp.
// TMEM columns: acc0 [0,BN), acc1 [BN,2BN), SF slots after.  BN = 192 keeps
// 2*192 + 2*48 <= 512; N tiles that start mid scale-factor atom (n0 % 128 == 64)
// read SFB from a TMEM address 2 columns (64 rows) into the loaded atom pair.
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "k1_launch.h"
#include "sm100.cuh"
#include "k2_epilogue.cuh"
#ifndef SVDQ_EXP
#define SVDQ_EXP 0
#endif

#ifdef SVDQ_TRACE
namespace svdq { __device__ unsigned long long g_k2_trace[148][8]; }
extern "C" int svdq_k2_trace_read(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, svdq::g_k2_trace, sizeof(unsigned long long) * 148 * 8) == cudaSuccess ? 0 : 1;
}
#define K2T_BEGIN() long long _t0 = clock64()
#define K2T_ACC(v) (v) += clock64() - _t0
#else
#define K2T_BEGIN() do {} while (0)
#define K2T_ACC(v) do {} while (0)
#endif

namespace svdq {

template <int BN>
struct NvCfg {
  static constexpr int BM = 128;
  static constexpr int BKB = 128;                        // bytes of K per stage (256 fp4)
  static constexpr int A_BYTES = BM * BKB;               // 16 KB
  static constexpr int B_BYTES = BN * BKB;
  static constexpr int SFA_BYTES = 4 * 512;              // 128 rows x 16 sf
  static constexpr int SFB_BYTES = 2 * 4 * 512;          // two 128-row atoms x 16 sf
  static constexpr int STAGE = A_BYTES + B_BYTES + SFA_BYTES + SFB_BYTES;
  static constexpr int EPI_BYTES = 8 * 2 * 2048;          // 8 epilogue warps x two 2 KB staging buffers
  static constexpr int kStages = (225 * 1024 - EPI_BYTES - 2048) / STAGE;
  static constexpr int SF_COLS = 16 + 32;                // TMEM columns per SF slot
  static constexpr int SF_BASE = 2 * BN;
  static constexpr int BAR_BYTES = 256;
  static constexpr int SMEM = kStages * STAGE + EPI_BYTES + BAR_BYTES + BN * 4 + 1024;
  static_assert(STAGE % 1024 == 0, "stage must keep 1024-B alignment");
  static_assert(SF_BASE + 2 * SF_COLS <= 512, "TMEM budget");
  static_assert(kStages >= 3, "pipeline depth");
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }

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
__global__ void __launch_bounds__(320, 1)
    k2_nvfp4_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmL,
                    const __grid_constant__ CUtensorMap tmY, const K2Params p) {
  using C = NvCfg<BN>;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  uint8_t *epi_stage = smem + S * C::STAGE;             // 1024-aligned TMA-store staging
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * C::STAGE + C::EPI_BYTES);
  uint64_t *empty = full + S;
  uint64_t *acc_full = empty + S;      // [2]
  uint64_t *acc_empty = acc_full + 2;  // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
  float *bias_s = reinterpret_cast<float *>(smem + S * C::STAGE + C::EPI_BYTES + C::BAR_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nkb64 = static_cast<int>(p.K / 64);          // 64-wide K blocks
  const int nkt = (nkb64 + 3) / 4;                       // FP4 pipeline steps per tile
  const int nslab = (p.rank + 63) / 64;
  const int mt_count = static_cast<int>((p.M + 127) / 128);
  const int nt_count = static_cast<int>((p.N + BN - 1) / BN);
  const int tiles = mt_count * nt_count;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);                   // 8 epilogue warps
    }
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
  griddep_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      griddep_wait();                                  // xq / xs / xl1 come from K1
#ifdef SVDQ_TRACE
      long long t_prod_wait = 0;
      const long long t_start = clock64();
#endif
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t m0 = static_cast<int64_t>(t % mt_count) * 128;
        const int64_t n0 = static_cast<int64_t>(t / mt_count) * BN;
        const int64_t atom0 = n0 / 128;                  // first SFB atom of the tile
        const int64_t atom_last = min((n0 + BN - 1) / 128, p.Npad / 128 - 1);
        const int natom = static_cast<int>(atom_last - atom0 + 1);   // 1 or 2 atoms cover the tile
        for (int kt = 0; kt < nkt; ++kt) {
          const int nsub = min(4, nkb64 - kt * 4);
          { K2T_BEGIN(); mbar_wait(&empty[s], ph ^ 1); K2T_ACC(t_prod_wait); }
          uint8_t *st = smem + s * C::STAGE;
          mbar_arrive_expect_tx(&full[s], C::A_BYTES + C::B_BYTES + nsub * 512 * (1 + natom));
          tma_load_2d(st, &tmA, &full[s], kt * C::BKB, static_cast<int32_t>(m0));
          tma_load_2d(st + C::A_BYTES, &tmB, &full[s], kt * C::BKB, static_cast<int32_t>(n0));
          bulk_load(st + C::A_BYTES + C::B_BYTES, p.sfa + ((m0 / 128) * nkb64 + kt * 4) * 512,
                    nsub * 512, &full[s]);
          for (int h = 0; h < natom; ++h)
            bulk_load(st + C::A_BYTES + C::B_BYTES + C::SFA_BYTES + h * 2048,
                      p.sfb + ((atom0 + h) * nkb64 + kt * 4) * 512, nsub * 512, &full[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        for (int j = 0; j < nslab; ++j) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t *st = smem + s * C::STAGE;
          mbar_arrive_expect_tx(&full[s], C::BM * 128 + BN * 128);
          tma_load_2d(st, &tmX, &full[s], j * 64, static_cast<int32_t>(m0));
          tma_load_2d(st + C::A_BYTES, &tmL, &full[s], j * 64, static_cast<int32_t>(n0));
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
#ifdef SVDQ_TRACE
      if (blockIdx.x < 148) { g_k2_trace[blockIdx.x][0] = t_prod_wait; g_k2_trace[blockIdx.x][1] = clock64() - t_start; }
#endif
    }
    __syncwarp();                                        // reconverge before the block-wide barrier
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_q = idesc_nvfp4(128, BN);
    constexpr uint32_t idesc_h = idesc_bf16(128, BN);
    int s = 0;
    uint32_t ph = 0;
    int acc_i = 0;
    int sf_i = 0;
#ifdef SVDQ_TRACE
    long long t_acc = 0, t_slot = 0, t_full = 0;
    const long long t_start = clock64();
#endif
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++acc_i) {
      const int b = acc_i & 1;
      const uint32_t acc_ph = (acc_i >> 1) & 1;
      const int64_t n0 = static_cast<int64_t>(t / mt_count) * BN;
      const uint32_t sfb_off = static_cast<uint32_t>((n0 % 128) / 32);
      const uint32_t d_tmem = tmem + b * BN;
      { K2T_BEGIN(); mbar_wait(&acc_empty[b], acc_ph ^ 1); K2T_ACC(t_acc); }   // epilogue drained this buffer
      tc_fence_after();
      for (int kt = 0; kt < nkt; ++kt) {
        const int nsub = min(4, nkb64 - kt * 4);
        const int slot = sf_i & 1;
        { K2T_BEGIN(); mbar_wait(&full[s], ph); K2T_ACC(t_full); }
        tc_fence_after();
        if (elect_one()) {
          uint8_t *st = smem + s * C::STAGE;
          const uint32_t a_addr = smem_u32(st);
          const uint32_t b_addr = smem_u32(st + C::A_BYTES);
          const uint32_t sfa_addr = smem_u32(st + C::A_BYTES + C::B_BYTES);
          const uint32_t sfb_addr = sfa_addr + C::SFA_BYTES;
          const uint32_t sfa_col = tmem + C::SF_BASE + slot * C::SF_COLS;
          const uint32_t sfb_col = sfa_col + 16;
            // descriptors: +16 B in smem = +1 in the start-address field (no carry: smem < 256 KB)
            const uint64_t sfa_d = sdesc_cp_32x128b(sfa_addr), sfb_d = sdesc_cp_32x128b(sfb_addr);
            const uint64_t a_d = sdesc_kmajor_sw128(a_addr), b_d = sdesc_kmajor_sw128(b_addr);
            if (nsub == 4) {
            #pragma unroll
              for (int i = 0; i < 4; ++i) {
#if SVDQ_EXP < 2
                tmem_cp_32x128b_warpx4(sfa_col + 4 * i, sfa_d + 32 * i);
#endif
#if SVDQ_EXP < 1
                tmem_cp_32x128b_warpx4(sfb_col + 8 * i, sfb_d + 32 * i);
#endif
#if SVDQ_EXP < 1
                tmem_cp_32x128b_warpx4(sfb_col + 8 * i + 4, sfb_d + 128 + 32 * i);
#endif
              }
            #pragma unroll
              for (int i = 0; i < 4; ++i)
                mma_nvfp4(d_tmem, a_d + 2 * i, b_d + 2 * i, idesc_q, sfa_col + 4 * i, sfb_col + 8 * i + sfb_off,
                      (kt | i) != 0);
            } else {
              for (int i = 0; i < nsub; ++i) {
#if SVDQ_EXP < 2
                tmem_cp_32x128b_warpx4(sfa_col + 4 * i, sfa_d + 32 * i);
#endif
#if SVDQ_EXP < 1
                tmem_cp_32x128b_warpx4(sfb_col + 8 * i, sfb_d + 32 * i);
#endif
#if SVDQ_EXP < 1
                tmem_cp_32x128b_warpx4(sfb_col + 8 * i + 4, sfb_d + 128 + 32 * i);
#endif
              }
              for (int i = 0; i < nsub; ++i)
                mma_nvfp4(d_tmem, a_d + 2 * i, b_d + 2 * i, idesc_q, sfa_col + 4 * i, sfb_col + 8 * i + sfb_off,
                      (kt | i) != 0);
            }
          tc_commit(&empty[s]);
        }
        __syncwarp();
        ++sf_i;
        if (++s == S) { s = 0; ph ^= 1; }
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
            mma_bf16(d_tmem, sdesc_kmajor_sw128(a_addr + 32 * i), sdesc_kmajor_sw128(b_addr + 32 * i),
                     idesc_h, (nkt > 0 || j > 0 || i > 0) ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
      if (elect_one()) tc_commit(&acc_full[b]);
      __syncwarp();
    }
#ifdef SVDQ_TRACE
    if (lane == 0 && blockIdx.x < 148) {
      g_k2_trace[blockIdx.x][2] = t_acc; g_k2_trace[blockIdx.x][3] = t_slot; g_k2_trace[blockIdx.x][4] = t_full;
      g_k2_trace[blockIdx.x][5] = clock64() - t_start;
    }
#endif
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    const int et = threadIdx.x - 64;           // 0..255
    int acc_i = 0;
    int ebuf = 0;
    griddep_wait();                            // Y / bias may be touched by the previous kernel
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++acc_i) {
      const int b = acc_i & 1;
      const uint32_t acc_ph = (acc_i >> 1) & 1;
      const int64_t m0 = static_cast<int64_t>(t % mt_count) * 128;
      const int64_t n0 = static_cast<int64_t>(t / mt_count) * BN;
      const int64_t grow = m0 + row;
      // stage this tile's bias (fp32) in smem
      named_bar(1, 256);                        // previous tile's readers are done
      for (int c = et; c < BN; c += 256)
        bias_s[c] = (p.bias && n0 + c < p.N) ? load_bias(p.bias, p.bias_dtype, n0 + c) : 0.f;
      named_bar(1, 256);
      mbar_wait(&acc_full[b], acc_ph);
      tc_fence_after();
      epilogue_tile<BN, 2>(tmem + b * BN + (static_cast<uint32_t>(quad * 32) << 16), bias_s, p.alpha, p.y_dtype,
                           &tmY, static_cast<int32_t>(m0 + quad * 32), static_cast<int32_t>(n0), (warp - 2) >> 2,
                           epi_stage + (warp - 2) * 4096, ebuf, lane, [&]() {
                          tc_fence_before();
                          __syncwarp();
                          if (lane == 0) mbar_arrive(&acc_empty[b]);
                        });
    }
  }
  if (warp >= 2 && lane == 0) bulk_wait_group<0>();    // outstanding TMA stores done
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
  const int num_sms = device_sm_count();
  const int64_t tiles = ((p.M + 127) / 128) * ((p.N + BN - 1) / BN);
  const unsigned grid = static_cast<unsigned>(tiles < num_sms ? tiles : num_sms);
  return launch_ex(kern, dim3(grid), dim3(320), C::SMEM, s, 1u, maps.a, maps.b, maps.xl1, maps.l2, maps.y, p);
}

int k2_nvfp4_bn(int64_t M, int64_t N) {
  // SVDQ_K2_BN1=128 / 192 forces the 1-CTA tile N (A/B of small-layer tile shapes)
  static const int force = [] { const char *e = std::getenv("SVDQ_K2_BN1"); return e ? std::atoi(e) : 0; }();
  if (force == 128 || force == 192) return force;
  // the tile N with the least per-SM work in the last wave: waves x BN (ties -> 192); on the small
  // layers of C2 / C3 the 128-wide tile often fills one more SM wave (PixArt 4096 x 1152 x 1152:
  // 7.8 vs 8.7 us, tools/k2_shape_sweep.py)
  const int64_t sms = device_sm_count(), mt = (M + 127) / 128;
  const int64_t w128 = (mt * ((N + 127) / 128) + sms - 1) / sms, w192 = (mt * ((N + 191) / 192) + sms - 1) / sms;
  return w192 * 192 <= w128 * 128 ? 192 : 128;
}

cudaError_t launch_k2_nvfp4(const K2Maps &maps, const K2Params &p, cudaStream_t s) {
  return k2_nvfp4_bn(p.M, p.N) == 192 ? launch_bn<192>(maps, p, s) : launch_bn<128>(maps, p, s);
}

}  // namespace svdq
