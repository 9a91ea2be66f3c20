// K2 (INT4): W4A4 GEMM on the kind::i8 tensor-core path + low-rank up-projection
// + bias ("Fused 4-Bit Compute + Up Projection", Fig. 5(b); INT4 g64 with
// 16-bit scales).  Blackwell has no INT4 MMA, so codes are unpacked to int8
// in shared memory; each 64-wide K group accumulates an EXACT int32 sum on the
// tensor cores (the bit-pinned object), which the epilogue promotes:
//   facc[m,n] += fl32(fl32(f32(acc_g[m,n]) * sx[m,g]) * sw[n,g])      (App. B.5, Q23)
//   Y = out_rn(facc + sum_t xl1[m,t] l2s[n,t] + bias[n])
//
// Persistent, one CTA per SM over 128 x 128 tiles; 14 warps:
//   warp 0      TMA producer: packed code tiles [rows x 64 B] (two K groups) into a
//               4-deep ring; at each tile start the low-rank slabs (xl1 / l2s, SW128).
//   warp 1      TMEM allocator + MMA issuer: per K group two kind::i8 MMAs (K = 32)
//               into one of two int32 TMEM buffers; the low-rank slab (kind::f16)
//               into an fp32 TMEM region.
//   warps 2..5  unpackers: int4 nibbles -> int8 (sign extended with byte-SIMD ops) in
//               the 128-B swizzled K-major layout the MMA reads.  Within every aligned
//               16-element block the k order is permuted identically for A and B, which
//               leaves every group sum unchanged.
//   warps 6..13 epilogue (two per TMEM lane quadrant, 64 columns each): per group
//               tcgen05.ld of the int32 sums, promotion, release; per tile the low-rank
//               term, bias, store.  Debug mode stores acc_g instead.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "k1_launch.h"
#include "sm100.cuh"

namespace svdq {

namespace {

constexpr int BM = 128;
constexpr int BN = kInt4BN;                 // 128
constexpr int kPStages = 4;                 // packed ring
constexpr int kUStages = 2;                 // unpacked (int8) ring
constexpr int PA = BM * 64, PB = BN * 64;   // packed bytes per stage (128 K elements)
constexpr int UA = BM * 128, UB = BN * 128; // int8 bytes per stage
constexpr int SLAB = BM * 128 + BN * 128;   // one 64-wide low-rank slab (bf16)
constexpr int kMaxSlabs = 2;
constexpr int OFF_U = 0;
constexpr int OFF_SLAB = OFF_U + kUStages * (UA + UB);
constexpr int OFF_P = OFF_SLAB + kMaxSlabs * SLAB;
constexpr int OFF_SW = OFF_P + kPStages * (PA + PB);
constexpr int OFF_BAR = OFF_SW + 2 * BN * 4 + 2 * BN * 4;
constexpr int SMEM = OFF_BAR + 256 + 1024;
constexpr int kThreads = 448;          // 14 warps
constexpr int kEpiWarps = 8;           // two per TMEM lane quadrant, 64 columns each
constexpr int EC = BN / 2;             // epilogue columns per warp
constexpr uint32_t TM_LR = 2 * BN;          // low-rank fp32 region after two int32 buffers

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint4 lds128(const void *p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void sts128(void *p, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
// 8 int4 nibbles -> two words of 4 sign-extended int8: (e0,e2,e4,e6), (e1,e3,e5,e7)
__device__ __forceinline__ void unpack8(uint32_t w, uint32_t &lo, uint32_t &hi) {
  lo = __vsub4((w & 0x0F0F0F0Fu) ^ 0x08080808u, 0x08080808u);
  hi = __vsub4(((w >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u, 0x08080808u);
}
// Unpack one 64-byte packed row (128 int4) into a 128-byte int8 row, SW128 layout.
__device__ __forceinline__ void unpack_row(const uint8_t *src, uint8_t *dst_row, int row) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {                      // 16 packed bytes -> two 16-byte chunks
    const uint4 v = lds128(src + c * 16);
    uint4 o0, o1;
    unpack8(v.x, o0.x, o0.y);
    unpack8(v.y, o0.z, o0.w);
    unpack8(v.z, o1.x, o1.y);
    unpack8(v.w, o1.z, o1.w);
    sts128(dst_row + (((2 * c) ^ (row & 7)) * 16), o0);
    sts128(dst_row + (((2 * c + 1) ^ (row & 7)) * 16), o1);
  }
}

__device__ __forceinline__ float load16(const uint16_t *p, int64_t i, bool bf16) {
  const uint16_t b = p[i];
  return bf16 ? __bfloat162float(__ushort_as_bfloat16(b)) : __half2float(__ushort_as_half(b));
}
__device__ __forceinline__ float load_bias(const void *b, int dt, int64_t i) {
  if (dt == 0) return __bfloat162float(static_cast<const __nv_bfloat16 *>(b)[i]);
  if (dt == 1) return __half2float(static_cast<const __half *>(b)[i]);
  return static_cast<const float *>(b)[i];
}

__global__ void __launch_bounds__(kThreads, 1)
    k2_int4_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmL,
                   const K2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *p_full = bar;                       // [kPStages]
  uint64_t *p_empty = p_full + kPStages;        // [kPStages]
  uint64_t *u_full = p_empty + kPStages;        // [kUStages]
  uint64_t *u_empty = u_full + kUStages;        // [kUStages]
  uint64_t *g_full = u_empty + kUStages;        // [2]
  uint64_t *g_empty = g_full + 2;               // [2]
  uint64_t *slab_full = g_empty + 2;
  uint64_t *slab_empty = slab_full + 1;
  uint64_t *lr_full = slab_empty + 1;
  uint64_t *lr_empty = lr_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(lr_empty + 1);
  float *sw_s = reinterpret_cast<float *>(smem + OFF_SW);       // [2][BN]
  float *bias_s = sw_s + 2 * BN;                                 // [BN]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool dbg = p.dbg_acc != nullptr;
  const int G = static_cast<int>(p.K / 64);            // K groups
  const int nst = (G + 1) / 2;                          // pipeline steps (2 groups each)
  const int nslab = dbg ? 0 : (p.rank + 63) / 64;
  const int mt_count = static_cast<int>((p.M + BM - 1) / BM);
  const int tiles = mt_count * static_cast<int>((p.N + BN - 1) / BN);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&p_empty[s], 4);
    }
    for (int s = 0; s < kUStages; ++s) {
      mbar_init(&u_full[s], 4);
      mbar_init(&u_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&g_full[b], 1);
      mbar_init(&g_empty[b], kEpiWarps);
    }
    mbar_init(slab_full, 1);
    mbar_init(slab_empty, 1);
    mbar_init(lr_full, 1);
    mbar_init(lr_empty, kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_launch_dependents();
  griddep_wait();                                   // inputs may come from the previous kernel

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (elect_one()) {
      int ps = 0;
      uint32_t pph = 0;
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int64_t m0 = static_cast<int64_t>(t % mt_count) * BM;
        const int64_t n0 = static_cast<int64_t>(t / mt_count) * BN;
        if (nslab) {
          mbar_wait(slab_empty, (it & 1) ^ 1);
          mbar_arrive_expect_tx(slab_full, nslab * SLAB);
          for (int j = 0; j < nslab; ++j) {
            uint8_t *sl = smem + OFF_SLAB + j * SLAB;
            tma_load_2d(sl, &tmX, slab_full, j * 64, static_cast<int32_t>(m0));
            tma_load_2d(sl + BM * 128, &tmL, slab_full, j * 64, static_cast<int32_t>(n0));
          }
        }
        for (int k = 0; k < nst; ++k) {
          mbar_wait(&p_empty[ps], pph ^ 1);
          uint8_t *st = smem + OFF_P + ps * (PA + PB);
          mbar_arrive_expect_tx(&p_full[ps], PA + PB);
          tma_load_2d(st, &tmA, &p_full[ps], k * 64, static_cast<int32_t>(m0));
          tma_load_2d(st + PA, &tmB, &p_full[ps], k * 64, static_cast<int32_t>(n0));
          if (++ps == kPStages) { ps = 0; pph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_i = idesc_s8(BM, BN);
    constexpr uint32_t idesc_h = idesc_bf16(BM, BN);
    int us = 0;
    uint32_t uph = 0;
    int gi = 0;        // global group counter -> int32 buffer gi & 1
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      if (nslab) {
        mbar_wait(lr_empty, (it & 1) ^ 1);
        mbar_wait(slab_full, it & 1);
        tc_fence_after();
        if (elect_one()) {
          for (int j = 0; j < nslab; ++j) {
            const uint32_t xa = smem_u32(smem + OFF_SLAB + j * SLAB);
            const uint32_t la = xa + BM * 128;
            const int nk16 = min(4, (p.rank - j * 64) / 16);
            for (int i = 0; i < nk16; ++i)
              mma_bf16(tmem + TM_LR, sdesc_kmajor_sw128(xa + 32 * i), sdesc_kmajor_sw128(la + 32 * i),
                       idesc_h, (j | i) != 0);
          }
          tc_commit(slab_empty);
          tc_commit(lr_full);
        }
        __syncwarp();
      }
      for (int k = 0; k < nst; ++k) {
        mbar_wait(&u_full[us], uph);
        tc_fence_after();
        const uint32_t ua = smem_u32(smem + OFF_U + us * (UA + UB));
        const uint32_t ub = ua + UA;
        const int ng = min(2, G - 2 * k);
        for (int j = 0; j < ng; ++j, ++gi) {
          const int b = gi & 1;
          mbar_wait(&g_empty[b], ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              mma_s8(tmem + b * BN, sdesc_kmajor_sw128(ua + 64 * j + 32 * h),
                     sdesc_kmajor_sw128(ub + 64 * j + 32 * h), idesc_i, h);
            tc_commit(&g_full[b]);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&u_empty[us]);
        __syncwarp();
        if (++us == kUStages) { us = 0; uph ^= 1; }
      }
    }
  } else if (warp < 6) {
    // ---------------------------------------------------------------- unpackers
    const int ut = threadIdx.x - 64;         // 0..127: one A row and one B row
    int ps = 0, us = 0;
    uint32_t pph = 0, uph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int k = 0; k < nst; ++k) {
        mbar_wait(&p_full[ps], pph);
        mbar_wait(&u_empty[us], uph ^ 1);
        const uint8_t *src = smem + OFF_P + ps * (PA + PB);
        uint8_t *dst = smem + OFF_U + us * (UA + UB);
        unpack_row(src + ut * 64, dst + ut * 128, ut);
        unpack_row(src + PA + ut * 64, dst + UA + ut * 128, ut);
        fence_proxy_async();                  // generic-proxy smem writes -> tensor core
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&p_empty[ps]);
          mbar_arrive(&u_full[us]);
        }
        if (++ps == kPStages) { ps = 0; pph ^= 1; }
        if (++us == kUStages) { us = 0; uph ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int quad = warp & 3;
    const int half = (warp - 6) >> 2;          // column half of the tile
    const int row = quad * 32 + lane;
    const int et = threadIdx.x - 192;         // 0..255
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const bool sbf = p.scale_bf16 != 0;
    const uint16_t *sx = reinterpret_cast<const uint16_t *>(p.sfa);
    const uint16_t *sw = reinterpret_cast<const uint16_t *>(p.sfb);
    int gi = 0;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int64_t m0 = static_cast<int64_t>(t % mt_count) * BM;
      const int64_t n0 = static_cast<int64_t>(t / mt_count) * BN;
      const int64_t c0 = n0 + half * EC;        // first global column of this warp
      const int64_t grow = m0 + row;
      const bool rvalid = grow < p.M;
      float facc[EC];
#pragma unroll
      for (int c = 0; c < EC; ++c) facc[c] = 0.f;
      if (!dbg) {
        named_bar(1, 32 * kEpiWarps);
        if (et < BN) bias_s[et] = (p.bias && n0 + et < p.N) ? load_bias(p.bias, p.bias_dtype, n0 + et) : 0.f;
      }
      for (int g = 0; g < G; ++g, ++gi) {
        const int b = gi & 1;
        float sxv = 0.f;
        if (!dbg) {
          // stage sw[n0 .. n0+BN)[g] (slot g & 1; the barrier also retires slot reuse)
          if (et < BN) sw_s[(g & 1) * BN + et] = n0 + et < p.N ? load16(sw, (n0 + et) * G + g, sbf) : 0.f;
          sxv = rvalid ? load16(sx, grow * G + g, sbf) : 0.f;
          named_bar(1, 32 * kEpiWarps);
        }
        mbar_wait(&g_full[b], (gi >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < EC / 16; ++cc) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem + b * BN + lane_off + half * EC + cc * 16, r);
          tmem_ld_wait();
          if (dbg) {
            if (rvalid) {
              int32_t *dst = p.dbg_acc + (static_cast<int64_t>(g) * p.M + grow) * p.N + c0 + cc * 16;
#pragma unroll
              for (int j = 0; j < 16; j += 4)
                if (c0 + cc * 16 + j < p.N)
                  *reinterpret_cast<int4 *>(dst + j) =
                      make_int4((int)r[j], (int)r[j + 1], (int)r[j + 2], (int)r[j + 3]);
            }
          } else {
            const float *swg = sw_s + (g & 1) * BN + half * EC + cc * 16;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              // exact int32 -> fp32 (|acc| <= 64*49 < 2^22): magic-number add / subtract
              const float a = __int_as_float(static_cast<int>(r[j]) + 0x4B400000) - 12582912.0f;
              facc[cc * 16 + j] = fmaf(__fmul_rn(a, sxv), swg[j], facc[cc * 16 + j]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&g_empty[b]);
      }
      if (dbg) continue;
      if (nslab) {
        mbar_wait(lr_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < EC / 32; ++cc) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + TM_LR + lane_off + half * EC + cc * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) facc[cc * 32 + j] += __uint_as_float(r[j]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(lr_empty);
      }
      if (rvalid) {
#pragma unroll
        for (int c8 = 0; c8 < EC / 8; ++c8) {
          const int64_t col = c0 + c8 * 8;
          if (col < p.N) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __fadd_rn(facc[c8 * 8 + e], bias_s[half * EC + c8 * 8 + e]);
            if (p.y_dtype == 2) {
              float4 *q = reinterpret_cast<float4 *>(static_cast<float *>(p.Y) + grow * p.ldy + col);
              q[0] = make_float4(v[0], v[1], v[2], v[3]);
              q[1] = make_float4(v[4], v[5], v[6], v[7]);
            } else {
              uint32_t w[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                if (p.y_dtype == 0)
                  w[j] = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * j]))) |
                         (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * j + 1]))) << 16);
                else
                  w[j] = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v[2 * j]))) |
                         (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v[2 * j + 1]))) << 16);
              }
              *reinterpret_cast<uint4 *>(static_cast<uint16_t *>(p.Y) + grow * p.ldy + col) =
                  make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

cudaError_t launch_k2_int4(const K2Maps &maps, const K2Params &p, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k2_int4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  if (p.rank > kMaxSlabs * 64 && !p.dbg_acc) return cudaErrorInvalidValue;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  const unsigned grid = static_cast<unsigned>(tiles < num_sms ? tiles : num_sms);
  return launch_ex(k2_int4_kernel, dim3(grid), dim3(kThreads), SMEM, s, 1u, maps.a, maps.b, maps.xl1, maps.l2, p);
}

}  // namespace svdq
