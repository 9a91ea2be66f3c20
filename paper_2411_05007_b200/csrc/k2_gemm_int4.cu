// K2 (INT4): W4A4 GEMM on the kind::i8 tensor-core path + low-rank up-projection
// + bias ("Fused 4-Bit Compute + Up Projection", Fig. 5(b); INT4 g64 with
// 16-bit scales).  Blackwell has no INT4 MMA, so codes are unpacked to int8
// in shared memory; each 64-wide K group accumulates an EXACT int32 sum on the
// tensor cores (the bit-pinned object), which the epilogue promotes:
//   facc[m,n] += fl32(fl32(f32(acc_g[m,n]) * sx[m,g]) * sw[n,g])      (App. B.5, Q23)
//   Y = out_rn(facc + sum_t xl1[m,t] l2s[n,t] + bias[n])
//
// Persistent, one CTA per SM over 128 x 128 tiles; 20 warps:
//   warp 0      TMA producer: packed code tiles [rows x 64 B] (two K groups) into a
//               4-deep ring; at each tile start the low-rank slabs (xl1 / l2s, SW128).
//   warp 1      TMEM allocator + MMA issuer: per K group two kind::i8 MMAs (K = 32)
//               into one of two int32 TMEM buffers; the low-rank slab (kind::f16)
//               into an fp32 TMEM region.
//   warps 2..3  unpackers (two rows of A and B per thread): int4 nibbles -> int8 (sign extended with byte-SIMD ops) in
//               the 128-B swizzled K-major layout the MMA reads.  Within every aligned
//               16-element block the k order is permuted identically for A and B, which
//               leaves every group sum unchanged.
//   warps 4..19 epilogue (four per TMEM lane quadrant, 32 columns each): per group one
//               tcgen05.ld of the int32 sums, immediate release of the buffer, then the
//               promotion on packed fp32 pairs (add/mul/fma .f32x2: 2.5 issue slots per
//               element); sx / sw for the next 8 groups are fetched while the current 8 are
//               promoted (sx in registers, sw broadcast from a per-warp smem buffer).  Per
//               tile the low-rank term, bias, store.  Debug mode stores acc_g instead.
// The promotion is ~3x the kind::i8 MMA time per group, so 16 warps keep all four
// schedulers busy while the tensor core idles.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "k1_launch.h"
#include "sm100.cuh"

// Waits of the INT4 kernel: it is issue-bound (promotion on CUDA cores), so waiting warps must
// not spin (ncu: try_wait loops were a third of all issued instructions).
#ifndef SVDQ_I4_SLEEP_NS
#define SVDQ_I4_SLEEP_NS 64
#endif
#ifndef SVDQ_I4_WAITMODE
#define SVDQ_I4_WAITMODE 0       // 0: test_wait + nanosleep back-off; 1: try_wait with the suspend-time hint
#endif
#if SVDQ_I4_WAITMODE == 1
#define SVDQ_I4_WAIT(bar, par) mbar_wait((bar), (par))
#else
#define SVDQ_I4_WAIT(bar, par) mbar_wait_sleep((bar), (par), SVDQ_I4_SLEEP_NS)
#endif
// Magic-initialized group accumulators: every int32 ring slot holds 0x4B400000 (= 1.5 * 2^23 as
// fp32) when the MMA starts a group, the group's MMAs ACCUMULATE onto it, so the epilogue reads
// the fp32 value 1.5 * 2^23 + acc directly (exact: |acc| <= 64 * 49 < 2^22) and saves the integer
// add per element; it writes the constant back (tcgen05.st) before releasing the slot.
#ifndef SVDQ_I4_MAGIC
#define SVDQ_I4_MAGIC 1
#endif
#ifndef SVDQ_I4EXP
#define SVDQ_I4EXP 0   // ablation bits: 1 no scale fetch, 2 no promotion math, 4 no unpack, 8 no MMA
#endif

#ifdef SVDQ_TRACE
namespace svdq { __device__ unsigned long long g_i4_trace[148][8]; }
extern "C" int svdq_i4_trace_read(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, svdq::g_i4_trace, sizeof(unsigned long long) * 148 * 8) == cudaSuccess ? 0 : 1;
}
#define I4T_BEGIN() long long _t0 = clock64()
#define I4T_ACC(v) (v) += clock64() - _t0
#else
#define I4T_BEGIN() do {} while (0)
#define I4T_ACC(v) do {} while (0)
#endif

namespace svdq {

namespace {

constexpr int BM = 128;
constexpr int BN = kInt4BN;                 // 128
constexpr int kPStages = 3;                 // packed ring
constexpr int kUStages = 2;                 // unpacked (int8) ring
constexpr int PA = BM * 64, PB = BN * 64;   // packed bytes per stage (128 K elements)
constexpr int UA = BM * 128, UB = BN * 128; // int8 bytes per stage
constexpr int SLAB = BM * 128 + BN * 128;   // one 64-wide low-rank slab (bf16)
constexpr int kMaxSlabs = 2;
constexpr int kEpiWarps = 16;               // four per TMEM lane quadrant, 32 columns each
constexpr int EC = 32;                      // epilogue columns per warp
constexpr int kGB = 8;                      // groups per scale block
constexpr int SWST = (2 * kGB * EC + EC) * 4;   // per-warp sw + sx staging (one block) + bias, bytes
constexpr int OFF_U = 0;
constexpr int OFF_SLAB = OFF_U + kUStages * (UA + UB);
constexpr int OFF_P = OFF_SLAB + kMaxSlabs * SLAB;
constexpr int OFF_SW = OFF_P + kPStages * (PA + PB);
constexpr int OFF_BAR = OFF_SW + kEpiWarps * SWST;
constexpr int SMEM = OFF_BAR + 256 + 1024;
constexpr int kUnpackWarps = 2;
constexpr int kThreads = 32 * (2 + kUnpackWarps + kEpiWarps);   // 20 warps: 5 per scheduler -> 96 regs
constexpr int kAcc = 4;                     // TMEM accumulator ring: 4 x 128 columns = all 512
// One ring slot per K group (int32 sums); the tile's low-rank slab (fp32) takes a slot as a
// pseudo-group ahead of the first K group.  A ring of 4 lets the MMA run up to four groups
// ahead of the promotion, hiding the commit -> tcgen05.ld -> release round trip (~1900 cycles
// measured; a 2-deep ring was bound at half of that per group).
static_assert(SMEM <= 227 * 1024, "smem budget");
// W8A8 operand ring: the two int8 slots plus the packed-int4 region (unused in the 8-bit setting)
constexpr int kW8Stages = 3;
static_assert(kPStages >= kW8Stages && kPStages * (PA + PB) >= UA + UB, "W8A8 third stage fits the packed region");
__host__ __device__ constexpr int w8_stage(int s) { return s < kUStages ? OFF_U + s * (UA + UB) : OFF_P; }

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// 16 columns of the constant v: four .x4 stores (a .x16 store of one repeated register still
// needs 16 live source registers and made the epilogue spill)
__device__ __forceinline__ void tmem_st_32x32b_x16_const(uint32_t taddr, uint32_t v) {
#pragma unroll
  for (int c = 0; c < 16; c += 4)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(taddr + c), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

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
// Per byte, sign-extend a two's-complement nibble n: v = n ^ 8 lies in [0, 15]; v + 0x78 never
// carries out of its byte, and flipping bit 7 of it gives v - 8 = n as an int8.  3-4 ALU ops
// per 4 bytes (the SIMD __vsub4 is emulated with ~10).
__device__ __forceinline__ void unpack8(uint32_t w, uint32_t &lo, uint32_t &hi) {
  lo = (((w & 0x0F0F0F0Fu) ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
  hi = ((((w >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
}
// Unpack 16-byte packed chunks (32 int4 of one row each) into the two 16-byte int8 chunks
// 2c, 2c + 1 of the row's 128-byte SW128 line.  A warp takes 8 rows x 4 chunks per load: the
// loads are 512 contiguous bytes and the stores hit each 16-byte bank group 4 times (optimal).
// All NCH loads are issued before any store so their latencies overlap.
template <int NCH, int STRIDE>
__device__ __forceinline__ void unpack_chunks(const uint8_t *src_tile, uint8_t *dst_tile, int q0) {
  uint4 v[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) v[i] = lds128(src_tile + (q0 + i * STRIDE) * 16);   // explicit .shared
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int q = q0 + i * STRIDE;
    const int row = q >> 2, c = q & 3;
    uint4 o0, o1;
    unpack8(v[i].x, o0.x, o0.y);
    unpack8(v[i].y, o0.z, o0.w);
    unpack8(v[i].z, o1.x, o1.y);
    unpack8(v[i].w, o1.z, o1.w);
    uint8_t *dst_row = dst_tile + row * 128;
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

// kW8: the 8-bit setting (SVDQ_FMT_W8A8): int8 codes arrive by TMA straight into the
// int8 ring (no unpack), the whole K accumulates in one exact int32 TMEM slot per tile, and the
// epilogue applies the per-token / per-channel scales once: fl32(fl32(f32(acc) * sx[m]) * sw[n]).
template <bool kDbg, bool kW8 = false>
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
  uint64_t *g_full = u_empty + kUStages;        // [kAcc]
  uint64_t *g_empty = g_full + kAcc;            // [kAcc]
  uint64_t *slab_full = g_empty + kAcc;
  uint64_t *slab_empty = slab_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(slab_empty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr bool dbg = kDbg;                           // debug: store the int32 group sums
  const int G = kW8 ? 1 : static_cast<int>(p.K / 64);  // K groups (W8A8: one, the whole K)
  const int nst = static_cast<int>((p.K / 64 + 1) / 2);   // pipeline steps (128 K elements each)
  const int nslab = dbg ? 0 : (p.rank + 63) / 64;
  const int mt_count = static_cast<int>((p.M + BM - 1) / BM);
  const int tiles = mt_count * static_cast<int>((p.N + BN - 1) / BN);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&p_full[s], 1);
      mbar_init(&p_empty[s], kW8 ? 1 : kUnpackWarps);   // W8A8: the int8 ring's barriers
    }
    for (int s = 0; s < kUStages; ++s) {
      mbar_init(&u_full[s], kW8 ? 1 : kUnpackWarps);   // W8A8: the producer's TMA fills it
      mbar_init(&u_empty[s], 1);
    }
    for (int b = 0; b < kAcc; ++b) {
      mbar_init(&g_full[b], 1);
      mbar_init(&g_empty[b], kEpiWarps);
    }
    mbar_init(slab_full, 1);
    mbar_init(slab_empty, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (SVDQ_I4_MAGIC && !kW8) {
    if (warp >= 2 + kUnpackWarps) {                 // epilogue warps: their lanes and columns of every slot
      const int ew0 = warp - 2 - kUnpackWarps;
      const uint32_t lo0 = static_cast<uint32_t>((warp & 3) * 32) << 16;
      for (int b = 0; b < kAcc; ++b)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) tmem_st_32x32b_x16_const(tmem + b * BN + lo0 + (ew0 >> 2) * EC + hh * 16, 0x4B400000u);
      tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
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
          if constexpr (kW8) {                        // int8 tiles [128 rows x 128 B], SW128
            mbar_wait(&p_empty[ps], pph ^ 1);           // 3-deep ring: the two int8 slots + the
            uint8_t *st = smem + w8_stage(ps);          // (unused) packed region
            mbar_arrive_expect_tx(&p_full[ps], UA + UB);
            tma_load_2d(st, &tmA, &p_full[ps], k * 128, static_cast<int32_t>(m0));
            tma_load_2d(st + UA, &tmB, &p_full[ps], k * 128, static_cast<int32_t>(n0));
            if (++ps == kW8Stages) { ps = 0; pph ^= 1; }
            continue;
          }
          mbar_wait(&p_empty[ps], pph ^ 1);
          uint8_t *st = smem + OFF_P + ps * (PA + PB);
          mbar_arrive_expect_tx(&p_full[ps], PA + PB);
          tma_load_2d(st, &tmA, &p_full[ps], k * 64, static_cast<int32_t>(m0));
          tma_load_2d(st + PA, &tmB, &p_full[ps], k * 64, static_cast<int32_t>(n0));
          if (++ps == kPStages) { ps = 0; pph ^= 1; }
        }
      }
    }
    __syncwarp();                                        // reconverge before the block-wide barrier
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_i = idesc_s8(BM, BN);
    constexpr uint32_t idesc_h = idesc_bf16(BM, BN);
    int us = 0;
    uint32_t uph = 0;
    int gi = 0;        // global ring counter -> TMEM slot gi % kAcc
    int it = 0;
#ifdef SVDQ_TRACE
    long long t_uf = 0, t_ge = 0;
    const long long t_st = clock64();
#endif
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      if (nslab) {
        const int b = gi % kAcc;
        SVDQ_I4_WAIT(&g_empty[b], ((gi / kAcc) & 1) ^ 1);
        mbar_wait(slab_full, it & 1);
        tc_fence_after();
        if (elect_one()) {
          for (int j = 0; j < nslab; ++j) {
            const uint32_t xa = smem_u32(smem + OFF_SLAB + j * SLAB);
            const uint32_t la = xa + BM * 128;
            const int nk16 = min(4, (p.rank - j * 64) / 16);
            for (int i = 0; i < nk16; ++i)
              mma_bf16(tmem + b * BN, sdesc_kmajor_sw128(xa + 32 * i), sdesc_kmajor_sw128(la + 32 * i),
                       idesc_h, (j | i) != 0);
          }
          tc_commit(slab_empty);
          tc_commit(&g_full[b]);
        }
        __syncwarp();
        ++gi;
      }
      if constexpr (kW8) {
        // one exact int32 accumulation over the whole K into a single ring slot
        const int b = gi % kAcc;
        SVDQ_I4_WAIT(&g_empty[b], ((gi / kAcc) & 1) ^ 1);
        tc_fence_after();
        for (int k = 0; k < nst; ++k) {
          mbar_wait(&p_full[us], uph);
          tc_fence_after();
          const uint32_t ua = smem_u32(smem + w8_stage(us));
          const uint32_t ub = ua + UA;
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < 4; ++h)
              mma_s8(tmem + b * BN, sdesc_kmajor_sw128(ua + 32 * h), sdesc_kmajor_sw128(ub + 32 * h), idesc_i,
                     (k | h) != 0);
            tc_commit(&p_empty[us]);
          }
          __syncwarp();
          if (++us == kW8Stages) { us = 0; uph ^= 1; }
        }
        if (elect_one()) tc_commit(&g_full[b]);
        __syncwarp();
        ++gi;
        continue;
      }
      for (int k = 0; k < nst; ++k) {
        { I4T_BEGIN(); mbar_wait(&u_full[us], uph); I4T_ACC(t_uf); }
        tc_fence_after();
        const uint32_t ua = smem_u32(smem + OFF_U + us * (UA + UB));
        const uint32_t ub = ua + UA;
        const int ng = min(2, G - 2 * k);
        for (int j = 0; j < ng; ++j, ++gi) {
          const int b = gi % kAcc;
          { I4T_BEGIN(); SVDQ_I4_WAIT(&g_empty[b], ((gi / kAcc) & 1) ^ 1); I4T_ACC(t_ge); }
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < ((SVDQ_I4EXP & 8) ? 0 : 2); ++h)
              mma_s8(tmem + b * BN, sdesc_kmajor_sw128(ua + 64 * j + 32 * h),
                     sdesc_kmajor_sw128(ub + 64 * j + 32 * h), idesc_i, SVDQ_I4_MAGIC ? 1u : static_cast<uint32_t>(h));
            tc_commit(&g_full[b]);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&u_empty[us]);
        __syncwarp();
        if (++us == kUStages) { us = 0; uph ^= 1; }
      }
    }
#ifdef SVDQ_TRACE
    if (lane == 0 && blockIdx.x < 148) {
      g_i4_trace[blockIdx.x][0] = t_uf; g_i4_trace[blockIdx.x][1] = t_ge; g_i4_trace[blockIdx.x][2] = clock64() - t_st;
    }
#endif
  } else if (warp < 2 + kUnpackWarps) {
    if constexpr (kW8) {
      // no unpacking in the 8-bit setting
    } else {
    // ---------------------------------------------------------------- unpackers
    const int ut0 = threadIdx.x - 64;        // 16-byte packed chunk q = ut0 + 64 i of A and of B
    int ps = 0, us = 0;
    uint32_t pph = 0, uph = 0;
#ifdef SVDQ_TRACE
    long long t_pf = 0, t_ue = 0;
    const long long t_st = clock64();
#endif
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int k = 0; k < nst; ++k) {
        { I4T_BEGIN(); mbar_wait(&p_full[ps], pph); I4T_ACC(t_pf); }
        { I4T_BEGIN(); mbar_wait(&u_empty[us], uph ^ 1); I4T_ACC(t_ue); }
        const uint8_t *src = smem + OFF_P + ps * (PA + PB);
        uint8_t *dst = smem + OFF_U + us * (UA + UB);
        if (!(SVDQ_I4EXP & 4)) {
          constexpr int NCH = BM * 4 / (32 * kUnpackWarps);     // chunks per thread per operand
          unpack_chunks<NCH, 32 * kUnpackWarps>(src, dst, ut0);
          unpack_chunks<NCH, 32 * kUnpackWarps>(src + PA, dst + UA, ut0);
        }
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
#ifdef SVDQ_TRACE
    if (threadIdx.x == 64 && blockIdx.x < 148) {
      g_i4_trace[blockIdx.x][3] = t_pf; g_i4_trace[blockIdx.x][4] = t_ue; g_i4_trace[blockIdx.x][5] = clock64() - t_st;
    }
#endif
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 2 - kUnpackWarps;     // 0..15
    const int quad = warp & 3;                  // TMEM lane quadrant this warp may access
    const int slice = ew >> 2;                  // 32-column slice of the tile
    const int row = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const bool sbf = p.scale_bf16 != 0;
    const uint16_t *sx = reinterpret_cast<const uint16_t *>(p.sfa);
    const uint16_t *sw = reinterpret_cast<const uint16_t *>(p.sfb);
    float *swst = reinterpret_cast<float *>(smem + OFF_SW + ew * SWST);   // [2][kGB][EC]
    float *bst = swst + 2 * kGB * EC;                                     // [EC]
    const int nblk = (G + kGB - 1) / kGB;
    int gi = 0;
    int it = 0;
#ifdef SVDQ_TRACE
    long long t_gf = 0;
    const long long t_st = clock64();
#endif
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int64_t m0 = static_cast<int64_t>(t % mt_count) * BM;
      const int64_t n0 = static_cast<int64_t>(t / mt_count) * BN;
      const int64_t c0 = n0 + slice * EC;       // first global column of this warp
      const int64_t grow = m0 + row;
      const bool rvalid = grow < p.M;
      const bool cvalid = c0 + lane < p.N;      // this lane's column for the sw / bias fetch
      uint64_t facc[EC / 2];
#pragma unroll
      for (int c = 0; c < EC / 2; ++c) facc[c] = 0ull;
      // scales of block 0 (raw 16-bit pairs in registers), then each block prefetches the next
      uint32_t sxn[kGB / 2], swn[kGB / 2];
      const bool vec = (G % kGB) == 0;          // 16-byte aligned rows of 8 scales
      auto fetch = [&](int blk) {
        if (vec && !(SVDQ_I4EXP & 1)) {
          const uint4 xv = (!dbg && rvalid) ? *reinterpret_cast<const uint4 *>(sx + grow * G + blk * kGB)
                                            : make_uint4(0, 0, 0, 0);
          const uint4 wv = (!dbg && cvalid) ? *reinterpret_cast<const uint4 *>(sw + (c0 + lane) * G + blk * kGB)
                                            : make_uint4(0, 0, 0, 0);
          sxn[0] = xv.x; sxn[1] = xv.y; sxn[2] = xv.z; sxn[3] = xv.w;
          swn[0] = wv.x; swn[1] = wv.y; swn[2] = wv.z; swn[3] = wv.w;
          return;
        }
#pragma unroll
        for (int j = 0; j < kGB / 2; ++j) {
          const int g = blk * kGB + 2 * j;
          if (SVDQ_I4EXP & 1) { sxn[j] = 0x3C003C00u; swn[j] = 0x3C003C00u; continue; }
          const uint32_t x0 = (!dbg && rvalid && g < G) ? sx[grow * G + g] : 0u;
          const uint32_t x1 = (!dbg && rvalid && g + 1 < G) ? sx[grow * G + g + 1] : 0u;
          const uint32_t w0 = (!dbg && cvalid && g < G) ? sw[(c0 + lane) * G + g] : 0u;
          const uint32_t w1 = (!dbg && cvalid && g + 1 < G) ? sw[(c0 + lane) * G + g + 1] : 0u;
          sxn[j] = x0 | (x1 << 16);
          swn[j] = w0 | (w1 << 16);
        }
      };
      auto h2f = [&](uint32_t bits16) {
        return sbf ? __uint_as_float(bits16 << 16) : __half2float(__ushort_as_half(static_cast<uint16_t>(bits16)));
      };
      if constexpr (!kW8) fetch(0);
      sts_f32(smem_u32(bst) + lane * 4, (!dbg && p.bias && cvalid) ? load_bias(p.bias, p.bias_dtype, c0 + lane) : 0.f);
      if (nslab) {                               // low-rank pseudo-group: facc starts at X L1 . L2
        const int b = gi % kAcc;
        mbar_wait(&g_full[b], (gi / kAcc) & 1);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem + b * BN + lane_off + slice * EC + hh * 16, r);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 8; ++c) facc[hh * 8 + c] = f2pack(__uint_as_float(r[2 * c]), __uint_as_float(r[2 * c + 1]));
          if (SVDQ_I4_MAGIC && !kW8)                 // the slot's next user may be an int32 group
            tmem_st_32x32b_x16_const(tmem + b * BN + lane_off + slice * EC + hh * 16, 0x4B400000u);
        }
        if (SVDQ_I4_MAGIC && !kW8) tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&g_empty[b]);
        ++gi;
      }
      const uint32_t swb = smem_u32(swst);       // [g][column] sw, then [g][lane] sx
      const uint32_t sxb = swb + kGB * EC * 4;
      if constexpr (kW8) {
        // one int32 accumulator per tile: facc += fl32(f32(acc) * sx[m]) * sw[n]
        const float sxv = rvalid ? reinterpret_cast<const float *>(p.sfa)[grow] : 0.f;
        __syncwarp();
        sts_f32(swb + lane * 4, cvalid ? reinterpret_cast<const float *>(p.sfb)[c0 + lane] : 0.f);
        __syncwarp();
        const int b = gi % kAcc;
        SVDQ_I4_WAIT(&g_full[b], (gi / kAcc) & 1);
        tc_fence_after();
        const uint64_t sx2 = f2pack(sxv, sxv);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem + b * BN + lane_off + slice * EC + hh * 16, r);
          tmem_ld_wait();
          if (hh == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&g_empty[b]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 w4 = lds_f32x4(swb + (hh * 16 + 4 * q) * 4);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int e = 4 * q + 2 * h;
              // |acc| may exceed 2^24 over a whole K: correctly rounded int -> fp32 conversion
              const uint64_t a2 = f2pack(__int2float_rn(static_cast<int>(r[e])),
                                         __int2float_rn(static_cast<int>(r[e + 1])));
              const uint64_t t2 = mul2(a2, sx2);
              const int fi = hh * 8 + e / 2;
              facc[fi] = fma2(t2, h ? f2pack(w4.z, w4.w) : f2pack(w4.x, w4.y), facc[fi]);
            }
          }
        }
        ++gi;
      }
      for (int blk = 0; blk < (kW8 ? 0 : nblk); ++blk) {
        __syncwarp();                            // previous block's reads are done
#pragma unroll
        for (int j = 0; j < kGB / 2; ++j) {
          sts_f32(swb + ((2 * j) * EC + lane) * 4, h2f(swn[j] & 0xFFFFu));    // broadcast reads below
          sts_f32(swb + ((2 * j + 1) * EC + lane) * 4, h2f(swn[j] >> 16));
          sts_f32(sxb + ((2 * j) * EC + lane) * 4, h2f(sxn[j] & 0xFFFFu));
          sts_f32(sxb + ((2 * j + 1) * EC + lane) * 4, h2f(sxn[j] >> 16));
        }
        __syncwarp();
        if (blk + 1 < nblk) fetch(blk + 1);      // in flight while this block is promoted
#pragma unroll
        for (int j = 0; j < kGB; ++j) {
          const int g = blk * kGB + j;
          if (g >= G) break;
          const int b = gi % kAcc;
          { I4T_BEGIN(); SVDQ_I4_WAIT(&g_full[b], (gi / kAcc) & 1); I4T_ACC(t_gf); }
          tc_fence_after();
          const float sxv = lds_f32(sxb + (j * EC + lane) * 4);
          const uint64_t sx2 = f2pack(sxv, sxv);
          const float bsx = __fmul_rn(sxv, -12582912.0f);
          const uint64_t bsx2 = f2pack(bsx, bsx);
          const uint32_t swg = swb + j * EC * 4;
#pragma unroll
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {               // two 16-column halves: 16 live registers
            uint32_t r[16];
            tmem_ld_32x32b_x16(tmem + b * BN + lane_off + slice * EC + hh * 16, r);
            tmem_ld_wait();
            if (hh == 1) {
              if (SVDQ_I4_MAGIC) {                        // both halves read: restore the constant
                tmem_st_32x32b_x16_const(tmem + b * BN + lane_off + slice * EC, 0x4B400000u);
                tmem_st_32x32b_x16_const(tmem + b * BN + lane_off + slice * EC + 16, 0x4B400000u);
                tmem_st_wait();
              }
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&g_empty[b]);   // the int32 buffer is free again
            }
            if (SVDQ_I4EXP & 2) {
              facc[hh * 8] = add2(facc[hh * 8], f2pack(__uint_as_float(r[0]), __uint_as_float(r[15])));
              continue;
            }
            if (dbg) {
              if (rvalid) {
                int32_t *dst = p.dbg_acc + (static_cast<int64_t>(g) * p.M + grow) * p.N + c0 + hh * 16;
#pragma unroll
                for (int q = 0; q < 16; q += 4)
                  if (c0 + hh * 16 + q < p.N)
                    *reinterpret_cast<int4 *>(dst + q) = SVDQ_I4_MAGIC
                        ? make_int4((int)(r[q] - 0x4B400000u), (int)(r[q + 1] - 0x4B400000u), (int)(r[q + 2] - 0x4B400000u),
                                    (int)(r[q + 3] - 0x4B400000u))
                        : make_int4((int)r[q], (int)r[q + 1], (int)r[q + 2], (int)r[q + 3]);
              }
              continue;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 w4 = lds_f32x4(swg + (hh * 16 + 4 * q) * 4);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = 4 * q + 2 * h;
                // fl32(acc * sx) in one FMA: the magic-number float m = 1.5 * 2^23 + acc is exact
                // (|acc| <= 64*49 < 2^22), bsx = fl32(-1.5 * 2^23 * sx) is exact (sx has 11
                // significant bits), so fma(m, sx, bsx) = fl32((m - 1.5 * 2^23) * sx) = fl32(acc * sx)
                const uint64_t a2 = SVDQ_I4_MAGIC
                    ? f2pack(__uint_as_float(r[e]), __uint_as_float(r[e + 1]))
                    : f2pack(__int_as_float(static_cast<int>(r[e]) + 0x4B400000),
                             __int_as_float(static_cast<int>(r[e + 1]) + 0x4B400000));
                const uint64_t t2 = fma2(a2, sx2, bsx2);
                const int fi = hh * 8 + e / 2;
                facc[fi] = fma2(t2, h ? f2pack(w4.z, w4.w) : f2pack(w4.x, w4.y), facc[fi]);   // + . * sw
              }
            }
          }
          ++gi;
        }
      }
      if (dbg) continue;
      if (rvalid) {
#pragma unroll
        for (int c8 = 0; c8 < EC / 8; ++c8) {
          const int64_t col = c0 + c8 * 8;
          if (col < p.N) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const uint64_t f = facc[c8 * 4 + e / 2];
              v[e] = __fadd_rn(__uint_as_float(static_cast<uint32_t>((e & 1) ? (f >> 32) : f)),
                               lds_f32(smem_u32(bst) + (c8 * 8 + e) * 4));
            }
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
      __syncwarp();                              // bst / swst reuse by the next tile
    }
#ifdef SVDQ_TRACE
    if (ew == 0 && lane == 0 && blockIdx.x < 148) {
      g_i4_trace[blockIdx.x][6] = t_gf; g_i4_trace[blockIdx.x][7] = clock64() - t_st;
    }
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

cudaError_t launch_k2_int4(const K2Maps &maps, const K2Params &p, cudaStream_t s) {
  auto kern = p.dbg_acc ? k2_int4_kernel<true> : (p.w8 ? k2_int4_kernel<false, true> : k2_int4_kernel<false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  if (p.rank > kMaxSlabs * 64 && !p.dbg_acc) return cudaErrorInvalidValue;
  const int num_sms = device_sm_count();
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  const unsigned grid = static_cast<unsigned>(tiles < num_sms ? tiles : num_sms);
  return launch_ex(kern, dim3(grid), dim3(kThreads), SMEM, s, 1u, maps.a, maps.b, maps.xl1, maps.l2, p);
}

}  // namespace svdq
