// K2 (NVFP4), CTA-pair version: the same fused GEMM as k2_gemm_nvfp4.cu
// ("Fused 4-Bit Compute + Up Projection", Fig. 5(b); Eq. 5), run on
// a cluster of two CTAs with tcgen05 cta_group::2 so that a 256 x 192 output tile
// is computed by two SMs that each stage only HALF of the B (weight) tile:
//   CTA rank c of the pair holds A rows [m0 + 128c, +128) and B rows [n0 + 96c, +96)
//   in its shared memory, its own SFA rows and a full copy of the tile's SFB; the
//   leader (rank 0) alone issues tcgen05.cp / tcgen05.mma .cta_group::2, which read
//   both CTAs' shared memory at the same offsets and write each CTA's TMEM
//   (D rows of that CTA's A half, all 192 columns).
// Why: the 1-CTA kernel is bounded by operand delivery into each SM (ncu: ~9.5 TB/s
// of TMA loads at 33 % tensor-pipe activity); halving B per SM raises the FLOP per
// byte each SM ingests from ~300 to ~370 (and halves B reads from L2).
//
// Warp roles per CTA (192 threads): warp 0 TMA producer (both CTAs; bytes land on the
// leader's full barrier), warp 1 TMEM allocator (both) + MMA issuer (leader), warps
// 2..5 epilogue (both; release the accumulator buffer to the leader's barrier).
// TMEM per CTA: acc0 [0,192), acc1 [192,384), two SF slots of 48 columns.
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
namespace svdq { __device__ unsigned long long g_k2p_trace[148][8]; }
extern "C" int svdq_k2p_trace_read(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, svdq::g_k2p_trace, sizeof(unsigned long long) * 148 * 8) == cudaSuccess ? 0 : 1;
}
#define K2T_BEGIN() long long _t0 = clock64()
#define K2T_ACC(v) (v) += clock64() - _t0
#else
#define K2T_BEGIN() do {} while (0)
#define K2T_ACC(v) do {} while (0)
#endif

namespace svdq {

namespace {

// Pair tile N: 192 (two TMEM accumulator buffers; any N), 256 (N % 256 == 0; the default when it
// divides N) or 384 (opt-in, SVDQ_K2_BN=384): one accumulator buffer -- TMEM holds 512 columns:
// 384 accumulator + 2 x 64 scale-factor columns.  The 384 tile reads 16 % fewer operand bytes per
// FLOP (per CTA and K step of 256: 48 KB for 25.2 MFLOP vs 38 KB for 16.8 MFLOP), for the case
// that the L2 -> SM stream binds (ncu: 12.5 TB/s on FLUX linear1 at 256); measured, it does not
// (see k2_pair_bn).  At 384 each CTA stages 192 B rows as [its 128 rows of the N = 256 MMA | its
// 64 rows of the N = 128 MMA] (three 64-row TMA boxes); the scale-factor rows are three atoms.
constexpr int A_BYTES = 128 * 128;            // 16 KB
constexpr int SFA_BYTES = 2048;
template <int kBN, bool kW8 = false>
struct PC {
  static constexpr int BN = kBN;
  static constexpr int BNH = kBN / 2;                       // B rows per CTA
  static constexpr int NATOM = kW8 ? 0 : (kBN == 384 ? 3 : 2);   // 128-row SFB atoms staged per stage
  static constexpr int B_BYTES = BNH * 128;                 // 12 / 16 / 24 KB
  static constexpr int SFB_BYTES = NATOM * 2048;            // atoms x 4 K-blocks x 512 B
  static constexpr int STAGE = A_BYTES + B_BYTES + (kW8 ? 0 : SFA_BYTES + SFB_BYTES);   // 34 / 38 / 48; W8A8 28 KB
  static constexpr int ACC = kBN == 192 && !kW8 ? 2 : 1;    // accumulator buffers
  static constexpr int SF_COLS = kW8 ? 0 : 16 + 16 * NATOM; // TMEM columns per SF slot (SFA + SFB, 4 K-blocks)
  static constexpr int SF_BASE = ACC * kBN;
  // W8A8: the int32 accumulator of X_q W_q^T in [0, BN) and the fp32 low-rank accumulator in
  // [BN, 2 BN) (an int32 and an fp32 product cannot share one accumulator)
  static constexpr int LR_COL = kW8 ? kBN : 0;
  static constexpr int BLOAD = kBN == 384 ? 64 : BNH;       // rows per B / L2s TMA box
};
constexpr int BN = 192;                       // the fused (layer-boundary) variant's tile N
#ifndef SVDQ_K2P_STAGES
#define SVDQ_K2P_STAGES 5
#endif
// Accumulator hand-back: a relaxed remote arrive.  The epilogue's tcgen05.ld have completed
// (tcgen05.wait::ld) and are ordered by tcgen05.fence::before_thread_sync; the release form would
// additionally wait for every outstanding smem / global access of the thread (ncu: the top
// ERRBAR stall of the fused epilogue).  Measured: fused FLUX MLP 211 -> 190 us; FLUX step K2
// +1 %.  SVDQ_K2_RELAXED_ACC=0 restores the release form.
#ifndef SVDQ_K2_RELAXED_ACC
#define SVDQ_K2_RELAXED_ACC 1
#endif
#if SVDQ_K2_RELAXED_ACC
#define K2_ACC_RELEASE(a) mbar_arrive_cluster_relaxed(a)
#else
#define K2_ACC_RELEASE(a) mbar_arrive_cluster(a)
#endif
#ifndef SVDQ_K2P_EPIW
#define SVDQ_K2P_EPIW 8
#endif
#ifndef SVDQ_K2P_EPIBUF
#define SVDQ_K2P_EPIBUF 2
#endif
constexpr int kStages = SVDQ_K2P_STAGES;
constexpr int kEpiBuf = SVDQ_K2P_EPIBUF;      // 2 KB staging buffers per epilogue warp
#ifndef SVDQ_K2P384_STAGES
#define SVDQ_K2P384_STAGES 4                  // 384-wide tile: 4 x 48 KB stages, 12 epilogue warps x 1 buffer
#endif
#ifndef SVDQ_BIGSTORE
#define SVDQ_BIGSTORE 0
#endif
// 16-bit Y with SVDQ_BIGSTORE: three [128 rows x 64 cols] SW128 blocks, one TMA store each;
// otherwise (and for fp32 Y) 8 warps x kEpiBuf 2 KB chunks
constexpr int EPI_BYTES = SVDQ_BIGSTORE && 3 * 16384 > 8 * 2048 * kEpiBuf ? 3 * 16384 : 8 * 2048 * kEpiBuf;
// Shared-memory layout per variant.  Fused launches (layer-boundary fusion) run a 4-stage ring
// and add the tile's lambda_inv_next [192] fp32, the a tile (3 x [128 rows x 128 B], SW128) and
// this CTA's half of the L1s_next rows (3 x [r/2 rows x 128 B], SW128) for the X L1s_next^T MMA.
template <bool kFuse, int kBN = 192, bool kW8 = false>
struct Lay {
  static constexpr int BN = kBN;
  static constexpr int stages = kFuse ? 3 : (kBN == 384 ? SVDQ_K2P384_STAGES : (kW8 ? 6 : kStages));
  // epilogue warps per CTA (2 or 3 per TMEM lane quadrant); 384 columns: 3 (4 x 32 columns per warp,
  // drained by epilogue_tile_wide within the 128 registers 448 threads allow)
  static constexpr int epi_w = kFuse || kBN == 384 ? 12 : SVDQ_K2P_EPIW;
  static constexpr int epibuf = kBN == 384 ? 1 : kEpiBuf;   // 2 KB staging buffers per epilogue warp
  static constexpr int threads = 64 + 32 * epi_w;
  static constexpr int epi_off = stages * PC<kBN, kW8>::STAGE;
  static constexpr int bar_off = epi_off + (epi_w != 8 ? epi_w * 2048 * epibuf : EPI_BYTES);
  static constexpr int bias_off = bar_off + 256;
  static constexpr int lamn_off = bias_off + BN * 4;
  static constexpr int at_off = (lamn_off + BN * 4 + 1023) / 1024 * 1024;   // a tile: 3 x 16 KB
  static constexpr int bt_off = at_off + 3 * 16384;         // L1s_next half: 3 x 2 KB (r <= 32)
  static constexpr int cs_off = bt_off + 3 * 2048;          // next-layer codes, [128 rows x 96 B]
  static constexpr int sfs_off = cs_off + 128 * 96;         // next-layer scale factors, 3 x 512 B
  static constexpr int sw_off = bias_off + BN * 4;          // W8A8: the tile's per-channel weight scales
  static constexpr int smem = kFuse ? sfs_off + 3 * 512 + 1024 : bias_off + (kW8 ? 2 : 1) * BN * 4 + 1024;
};
constexpr int XL1_COL = PC<192>::SF_BASE + 2 * PC<192>::SF_COLS;   // TMEM columns [480, 512): X L1s_next^T accumulator
static_assert(XL1_COL + 32 <= 512, "TMEM budget (fused)");
static_assert(PC<192>::STAGE % 1024 == 0 && PC<256>::STAGE % 1024 == 0 && PC<384>::STAGE % 1024 == 0 &&
              PC<192, true>::STAGE % 1024 == 0, "stage alignment");
static_assert(PC<192>::SF_BASE + 2 * PC<192>::SF_COLS <= 512 && PC<256>::SF_BASE + 2 * PC<256>::SF_COLS <= 512 &&
              PC<384>::SF_BASE + 2 * PC<384>::SF_COLS <= 512, "TMEM budget");

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ float load_bias(const void *b, int dt, int64_t i) {
  if (dt == 0) return __bfloat162float(static_cast<const __nv_bfloat16 *>(b)[i]);
  if (dt == 1) return __half2float(static_cast<const __half *>(b)[i]);
  return static_cast<const float *>(b)[i];
}
__device__ __forceinline__ void store8(void *Y, int dt, int64_t ldy, int64_t row, int64_t col, const float (&v)[8]) {
  if (dt == 2) {
    float4 *p = reinterpret_cast<float4 *>(static_cast<float *>(Y) + row * ldy + col);
    p[0] = make_float4(v[0], v[1], v[2], v[3]);
    p[1] = make_float4(v[4], v[5], v[6], v[7]);
    return;
  }
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (dt == 0)
      w[j] = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * j]))) |
             (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * j + 1]))) << 16);
    else
      w[j] = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v[2 * j]))) |
             (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v[2 * j + 1]))) << 16);
  }
  *reinterpret_cast<uint4 *>(static_cast<uint16_t *>(Y) + row * ldy + col) = make_uint4(w[0], w[1], w[2], w[3]);
}

// Tile t of the concatenated tile lists -> (problem, m0, n0).
struct TileRef {
  int i;
  int64_t m0, n0;
};
template <int BN = 192>
__device__ __forceinline__ TileRef locate(const K2PairArgs &g, int t) {
  int i = 0;
  while (i + 1 < g.n && t >= g.tile_begin[i + 1]) ++i;
  const int lt = t - g.tile_begin[i];
  if (g.pr[i].p.fuse) {                   // n-fastest: a pair's contiguous range stays on few row blocks
    const int nt = static_cast<int>((g.pr[i].p.N + BN - 1) / BN);
    return TileRef{i, static_cast<int64_t>(lt / nt) * 256, static_cast<int64_t>(lt % nt) * BN};
  }
  const int mt = static_cast<int>((g.pr[i].p.M + 255) / 256);
  const int band = g.pr[i].p.band;
  if (band <= 0 || band >= mt)                     // m-fastest over the whole M
    return TileRef{i, static_cast<int64_t>(lt % mt) * 256, static_cast<int64_t>(lt / mt) * BN};
  // L2 bands: all N tiles of `band` row tiles (m-fastest inside the band), then the next band,
  // so the band's A rows stay L2-resident while every weight tile streams past them once
  const int nt = static_cast<int>((g.pr[i].p.N + BN - 1) / BN);
  const int b = lt / (band * nt), in = lt - b * band * nt;
  const int rows = min(band, mt - b * band);
  return TileRef{i, static_cast<int64_t>(b * band + in % rows) * 256, static_cast<int64_t>(in / rows) * BN};
}

// kW8: the paper's 8-bit setting (SVDQ_FMT_W8A8) on the same CTA-pair skeleton:
// kind::i8 over the whole K into an exact int32 accumulator, the low-rank slab into a separate fp32
// accumulator, scales applied once per tile in the epilogue (epilogue_tile_w8).
template <bool kFuse, int kBN, bool kW8 = false>
__global__ void __launch_bounds__(Lay<kFuse, kBN, kW8>::threads, 1)
    k2_nvfp4_2sm_kernel(const __grid_constant__ K2PairArgs g) {
  using PCK = PC<kBN, kW8>;
  constexpr int BN = kBN, BNH = PCK::BNH, B_BYTES = PCK::B_BYTES, STAGE = PCK::STAGE;
  constexpr int SF_BASE = PCK::SF_BASE, ACC = PCK::ACC, SF_COLS = PCK::SF_COLS;
  constexpr int NATOM = PCK::NATOM, LR_COL = PCK::LR_COL;
  static_assert(!kFuse || kBN == 192, "the fused variant runs 192-wide tiles");
  static_assert(!kW8 || (kBN == 192 && !kFuse), "W8A8 runs plain 192-wide tiles");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  using LY = Lay<kFuse, kBN, kW8>;
  constexpr int kSt = LY::stages;
  constexpr int kEpiW = LY::epi_w, kNWQ = kEpiW / 4, kEpiT = 32 * kEpiW;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + LY::bar_off);
  uint64_t *empty = full + kSt;
  uint64_t *acc_full = empty + kSt;       // [2]
  uint64_t *acc_empty = acc_full + 2;     // [2] (leader's copy is the one used)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
  uint64_t *xa_full = acc_empty + 3;      // fused: a tile written by all 16 epilogue warps (leader's)
  uint64_t *xa_empty = acc_empty + 4;     // fused: the X L1s_next^T MMAs of the tile are done (both)
  float *bias_s = reinterpret_cast<float *>(smem + LY::bias_off);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();             // 0 leader, 1 peer
  const int pair = static_cast<int>(blockIdx.x >> 1);
  const int npairs = static_cast<int>(gridDim.x >> 1);
  const int tiles = g.tile_begin[g.n];
  // tile walk: strided (t = pair, pair + npairs, ...) or, for fused launches, the contiguous
  // range [pair * tiles / npairs, (pair + 1) * tiles / npairs)
  const int t_first = g.contig ? static_cast<int>(static_cast<int64_t>(pair) * tiles / npairs) : pair;
  const int t_end = g.contig ? static_cast<int>(static_cast<int64_t>(pair + 1) * tiles / npairs) : tiles;
  const int t_step = g.contig ? 1 : npairs;
  // K steps per tile: 128-byte rows of packed codes = 256 FP4 or 128 int8 elements
  auto nkt_of = [&](int i) { return static_cast<int>(kW8 ? (g.pr[i].p.K + 127) / 128 : (g.pr[i].p.K / 64 + 3) / 4); };
  auto nslab_of = [&](int i) { return (g.pr[i].p.rank + 63) / 64; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * kEpiW);               // epilogue warps x 2 CTAs
    }
    if (kFuse) {
      mbar_init(xa_full, 2 * kEpiW);
      mbar_init(xa_empty, 1);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < g.n; ++i) {
      tma_prefetch(&g.pr[i].a);
      tma_prefetch(&g.pr[i].b);
      if (!kW8) {
        tma_prefetch(&g.pr[i].sfa);
        tma_prefetch(&g.pr[i].sfb);
      }
      if (nslab_of(i)) {
        tma_prefetch(&g.pr[i].xl1);
        tma_prefetch(&g.pr[i].l2);
      }
    }
  }
  if (warp == 1) tmem_alloc_cg2(tmem_slot, 512);
  tc_fence_before();
  // CTA barrier before the cluster barrier: orders the allocator's write of tmem_slot before the
  // other warps' reads in a form compute-sanitizer's racecheck models (it flagged the
  // tcgen05.alloc write against the reads below when only barrier.cluster separated them)
  __syncthreads();
  cluster_sync();                                        // barriers of both CTAs initialised
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      const uint32_t full0 = mapa_u32(&full[0], 0);      // leader's barriers
      int s = 0;
      uint32_t ph = 0;
#ifdef SVDQ_TRACE
      long long t_pwait = 0;
#endif
      // Weight tiles (B, SFB) of the first tile's first ring do not depend on K1: issue them
      // before the programmatic dependency resolves, so they land while K1 finishes.
      // this CTA's B-side rows of the pair tile at n0 (B codes or, for the low-rank slab, L2s): one box
      // of BN/2 rows, or at 384 three 64-row boxes [n0 + 128 c, +128) and [n0 + 256 + 64 c, +64)
      auto load_bside = [&](uint8_t *dst, const CUtensorMap *map, uint32_t fb, int32_t kc, int64_t n0) {
        if constexpr (kBN == 384) {
          tma_load_2d_cg2(dst, map, fb, kc, static_cast<int32_t>(n0 + 128 * crank));
          tma_load_2d_cg2(dst + 64 * 128, map, fb, kc, static_cast<int32_t>(n0 + 128 * crank + 64));
          tma_load_2d_cg2(dst + 128 * 128, map, fb, kc, static_cast<int32_t>(n0 + 256 + 64 * crank));
        } else {
          tma_load_2d_cg2(dst, map, fb, kc, static_cast<int32_t>(n0 + BNH * crank));
        }
      };
      const int pre = (SVDQ_EXP & 4) || t_first >= t_end ? 0 : min(kSt, nkt_of(locate<kBN>(g, t_first).i));
      if (pre) {
        const TileRef tr = locate<kBN>(g, t_first);
        const K2PairProblem &pr = g.pr[tr.i];
        for (int kt = 0; kt < pre; ++kt) {
          uint8_t *st = smem + kt * STAGE;
          const uint32_t fb = full0 + kt * 8;
          if (crank == 0) mbar_arrive_expect_tx(&full[kt], 2 * STAGE);
          load_bside(st + A_BYTES, &pr.b, fb, kt * 128, tr.n0);
          if (!kW8)
            tma_load_3d_cg2(st + A_BYTES + B_BYTES + SFA_BYTES, &pr.sfb, fb, 0, kt * 4,
                            static_cast<int32_t>(tr.n0 / 128));
        }
      }
      griddep_wait();                                    // xq / xs / xl1 come from K1
      bool first = true;
      for (int t = t_first; t < t_end; t += t_step) {
        const TileRef tr = locate<kBN>(g, t);
        const K2PairProblem &pr = g.pr[tr.i];
        const int nkt = nkt_of(tr.i);
        const int nslab = nslab_of(tr.i);
        const int64_t m0 = tr.m0;
        const int64_t n0 = tr.n0;
        const int32_t ma = static_cast<int32_t>(m0 + 128 * crank);
        for (int kt = 0; kt < nkt; ++kt) {
          uint8_t *st = smem + s * STAGE;
          const uint32_t fb = full0 + s * 8;
          if (first && kt < pre) {                         // B / SFB already in flight
            tma_load_2d_cg2(st, &pr.a, fb, kt * 128, ma);
            if (!kW8)
              tma_load_3d_cg2(st + A_BYTES + B_BYTES, &pr.sfa, fb, 0, kt * 4, static_cast<int32_t>(m0 / 128 + crank));
            if (++s == kSt) { s = 0; ph ^= 1; }
            continue;
          }
          { K2T_BEGIN(); mbar_wait(&empty[s], ph ^ 1); K2T_ACC(t_pwait); }
#if SVDQ_EXP & 4                                         // ablation: no operand traffic at all
          if (crank == 0) mbar_arrive(&full[s]);
          if (++s == kSt) { s = 0; ph ^= 1; }
          continue;
#endif
          if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * STAGE);
          tma_load_2d_cg2(st, &pr.a, fb, kt * 128, ma);
          load_bside(st + A_BYTES, &pr.b, fb, kt * 128, n0);
          if (!kW8) {
            tma_load_3d_cg2(st + A_BYTES + B_BYTES, &pr.sfa, fb, 0, kt * 4, static_cast<int32_t>(m0 / 128 + crank));
            tma_load_3d_cg2(st + A_BYTES + B_BYTES + SFA_BYTES, &pr.sfb, fb, 0, kt * 4,
                            static_cast<int32_t>(n0 / 128));
          }
          if (++s == kSt) { s = 0; ph ^= 1; }
        }
        first = false;
        for (int j = 0; j < nslab; ++j) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t *st = smem + s * STAGE;
          const uint32_t fb = full0 + s * 8;
          if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
          tma_load_2d_cg2(st, &pr.xl1, fb, j * 64, ma);
          load_bside(st + A_BYTES, &pr.l2, fb, j * 64, n0);
          if (++s == kSt) { s = 0; ph ^= 1; }
        }
      }
#ifdef SVDQ_TRACE
      if (crank == 0 && pair < 148) g_k2p_trace[pair][6] = t_pwait;
#endif
    }
    __syncwarp();                                        // reconverge before the block-wide barrier
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (crank == 0) {
      // 384: an N = 256 MMA into columns [0, 256) and an N = 128 MMA into [256, 384) per K block
      constexpr uint32_t NM1 = kBN == 384 ? 256 : BN;
      constexpr uint32_t idesc_q = idesc_nvfp4(256, NM1);
      constexpr uint32_t idesc_h = idesc_bf16(256, NM1);
      constexpr uint32_t idesc_q2 = idesc_nvfp4(256, 128);
      constexpr uint32_t idesc_h2 = idesc_bf16(256, 128);
      constexpr uint32_t B2_OFF = 128 * 128;                 // smem offset of the second MMA's B rows
      int s = 0;
      uint32_t ph = 0;
      int acc_i = 0;
      int sf_i = 0;
#ifdef SVDQ_TRACE
      long long t_acc = 0, t_full = 0;
      const long long t_start = clock64();
#endif
      // fused: xl1 += a_tile x L1s_next^T for a tile whose epilogue has filled the a / B tiles
      int xl_prev = -1;
      bool xl_prev_first = false;
      uint32_t xa_ph = 0;
      auto issue_xl1 = [&](int tp, bool first) {
        const int r = g.pr[locate<kBN>(g, tp).i].p.nx_r;
        mbar_wait(xa_full, xa_ph);
        xa_ph ^= 1;
        tc_fence_after();
        if (elect_one()) {
          const uint32_t idesc_x = idesc_bf16(256, static_cast<uint32_t>(r));
          const uint32_t a0 = smem_u32(smem + LY::at_off), b0 = smem_u32(smem + LY::bt_off);
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              mma_bf16_cg2(tmem + XL1_COL, sdesc_kmajor_sw128(a0 + c * 16384 + 32 * i),
                           sdesc_kmajor_sw128(b0 + c * 2048 + 32 * i), idesc_x, (!first || c || i) ? 1u : 0u);
          tc_commit_cg2_mc(xa_empty, 0x3);
        }
        __syncwarp();
      };
      for (int t = t_first; t < t_end; t += t_step, ++acc_i) {
        const bool single = (SVDQ_EXP & 64) || ACC == 1;          // 64: single accumulator (ablation)
        const int b = single ? 0 : acc_i & 1;
        const uint32_t acc_ph = single ? acc_i & 1 : (acc_i >> 1) & 1;
        const TileRef tr = locate<kBN>(g, t);
        const int64_t n0 = tr.n0;
        const int nkb64 = static_cast<int>(g.pr[tr.i].p.K / 64);
        const int nkt = nkt_of(tr.i);
        const int nslab = nslab_of(tr.i);
        const int rank = g.pr[tr.i].p.rank;
        const uint32_t sfb_off = static_cast<uint32_t>((n0 % 128) / 32);
        const uint32_t d_tmem = tmem + b * BN;
        { K2T_BEGIN(); mbar_wait(&acc_empty[b], acc_ph ^ 1); K2T_ACC(t_acc); }
        tc_fence_after();
        for (int kt = 0; kt < nkt; ++kt) {
          const int nsub = min(4, nkb64 - kt * 4);
          const int slot = sf_i & 1;
          { K2T_BEGIN(); mbar_wait(&full[s], ph); K2T_ACC(t_full); }
          tc_fence_after();
          if (elect_one()) {
            uint8_t *st = smem + s * STAGE;
            const uint32_t a_addr = smem_u32(st);
            const uint32_t b_addr = smem_u32(st + A_BYTES);
            const uint32_t sfa_addr = smem_u32(st + A_BYTES + B_BYTES);
            const uint32_t sfb_addr = sfa_addr + SFA_BYTES;
            const uint32_t sfa_col = tmem + SF_BASE + slot * SF_COLS;
            const uint32_t sfb_col = sfa_col + 16;
            // descriptors: +16 B in smem = +1 in the start-address field (no carry: smem < 256 KB)
            const uint64_t sfa_d = sdesc_cp_32x128b(sfa_addr), sfb_d = sdesc_cp_32x128b(sfb_addr);
            const uint64_t a_d = sdesc_kmajor_sw128(a_addr), b_d = sdesc_kmajor_sw128(b_addr);
            const uint64_t b2_d = sdesc_kmajor_sw128(b_addr + B2_OFF);
            // SFB atoms of K block i at columns sfb_col + 4 NATOM i + 4 a; the smem atom a at + 2 KB a
            auto sf_copy = [&](int i) {
#if (SVDQ_EXP & 3) < 2
              tmem_cp_32x128b_warpx4_cg2(sfa_col + 4 * i, sfa_d + 32 * i);
#endif
#if (SVDQ_EXP & 3) < 1
#pragma unroll
              for (int a = 0; a < NATOM; ++a)
                tmem_cp_32x128b_warpx4_cg2(sfb_col + 4 * NATOM * i + 4 * a, sfb_d + 128 * a + 32 * i);
#endif
            };
            auto mma_kb = [&](int i) {
              mma_nvfp4_cg2(d_tmem, a_d + 2 * i, b_d + 2 * i, idesc_q, sfa_col + 4 * i,
                            sfb_col + 4 * NATOM * i + sfb_off, (kt | i) != 0);
              if constexpr (kBN == 384)
                mma_nvfp4_cg2(d_tmem + 256, a_d + 2 * i, b2_d + 2 * i, idesc_q2, sfa_col + 4 * i,
                              sfb_col + 4 * NATOM * i + 8, (kt | i) != 0);
            };
            if constexpr (kW8) {                     // 128 int8 of K per stage: 4 x K32
#pragma unroll
              for (int h = 0; h < 4; ++h)
                mma_s8_cg2(d_tmem, a_d + 2 * h, b_d + 2 * h, idesc_s8(256, BN), (kt | h) != 0);
            } else if (nsub == 4) {
#pragma unroll
              for (int i = 0; i < 4; ++i) sf_copy(i);
#pragma unroll
              for (int i = 0; i < 4; ++i) mma_kb(i);
            } else {
              for (int i = 0; i < nsub; ++i) sf_copy(i);
              for (int i = 0; i < nsub; ++i) mma_kb(i);
            }
            tc_commit_cg2_mc(&empty[s], 0x3);
          }
          __syncwarp();
          ++sf_i;
          if (++s == kSt) { s = 0; ph ^= 1; }
        }
        for (int j = 0; j < nslab; ++j) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (elect_one()) {
            uint8_t *st = smem + s * STAGE;
            const uint32_t a_addr = smem_u32(st);
            const uint32_t b_addr = smem_u32(st + A_BYTES);
            const int nk16 = min(4, (rank - j * 64) / 16);
            for (int i = 0; i < nk16; ++i) {
              // NVFP4: into the same accumulator (after the K loop); W8A8: its own fp32 accumulator
              const uint32_t acc_in = ((!kW8 && nkt > 0) || j > 0 || i > 0) ? 1u : 0u;
              mma_bf16_cg2(d_tmem + LR_COL, sdesc_kmajor_sw128(a_addr + 32 * i), sdesc_kmajor_sw128(b_addr + 32 * i),
                           idesc_h, acc_in);
              if constexpr (kBN == 384)
                mma_bf16_cg2(d_tmem + 256, sdesc_kmajor_sw128(a_addr + 32 * i),
                             sdesc_kmajor_sw128(b_addr + B2_OFF + 32 * i), idesc_h2, (nkt > 0 || j > 0 || i > 0) ? 1u : 0u);
            }
            tc_commit_cg2_mc(&empty[s], 0x3);
          }
          __syncwarp();
          if (++s == kSt) { s = 0; ph ^= 1; }
        }
        if (elect_one()) tc_commit_cg2_mc(&acc_full[b], 0x3);
        __syncwarp();
        if constexpr (kFuse) {                           // X L1s_next^T of the PREVIOUS fused tile
          if (xl_prev >= 0) issue_xl1(xl_prev, xl_prev_first);
          const K2Params &pt = g.pr[tr.i].p;
          if (pt.fuse && pt.nx_r > 0) {
            xl_prev_first = t == t_first || locate<kBN>(g, t - t_step).i != tr.i || locate<kBN>(g, t - t_step).m0 != tr.m0;
            xl_prev = t;
          } else {
            xl_prev = -1;
          }
        }
      }
      if constexpr (kFuse) {
        if (xl_prev >= 0) issue_xl1(xl_prev, xl_prev_first);
      }
#ifdef SVDQ_TRACE
      if (lane == 0 && pair < 148) {
        g_k2p_trace[pair][0] = t_acc; g_k2p_trace[pair][1] = t_full; g_k2p_trace[pair][2] = clock64() - t_start;
      }
#endif
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const int et = threadIdx.x - 64;
    int xl_cnt = 0;                                      // fused tiles that fed the X L1s_next^T MMA
    const uint32_t xa_full0 = mapa_u32(xa_full, 0);
    const uint32_t acc_empty0 = mapa_u32(&acc_empty[0], 0);
    int acc_i = 0;
    int ebuf = 0;
#ifdef SVDQ_TRACE
    long long t_ewait = 0, t_edrain = 0;
    const long long t_estart = clock64();
#endif
    griddep_wait();
    for (int t = t_first; t < t_end; t += t_step, ++acc_i) {
      const bool single = (SVDQ_EXP & 64) || ACC == 1;
      const int b = single ? 0 : acc_i & 1;
      const uint32_t acc_ph = single ? acc_i & 1 : (acc_i >> 1) & 1;
      const TileRef tr = locate<kBN>(g, t);
      const K2Params &p = g.pr[tr.i].p;
      const CUtensorMap *tmY = &g.pr[tr.i].y;
      const int64_t m0 = tr.m0 + 128 * crank;
      const int64_t n0 = tr.n0;
      if (kFuse && et == 0) bulk_wait_group_read<0>();    // previous tile's code / SF staging is read
      named_bar(1, kEpiT);
      for (int c = et; c < BN; c += kEpiT)
        bias_s[c] = (p.bias && n0 + c < p.N) ? load_bias(p.bias, p.bias_dtype, n0 + c) : 0.f;
      if constexpr (kW8) {                               // per-channel weight scales of the tile
        float *sw_s = reinterpret_cast<float *>(smem + LY::sw_off);
        for (int c = et; c < BN; c += kEpiT) sw_s[c] = n0 + c < p.N ? reinterpret_cast<const float *>(p.sfb)[n0 + c] : 0.f;
      }
      const bool fx = kFuse && p.fuse && p.nx_r > 0;   // this tile feeds the X L1s_next^T MMA
      if constexpr (kFuse) {
        if (p.fuse) {
          float *lamn_s = reinterpret_cast<float *>(smem + LY::lamn_off);
          for (int c = et; c < BN; c += kEpiT) lamn_s[c] = n0 + c < p.N ? p.nx_lam_inv[n0 + c] : 0.f;
        }
        if (fx) {
          // this CTA's L1s_next rows [crank * r/2, +r/2) over the tile's 192 columns, SW128 K-major:
          // 16-byte vector (row jl, 8-column group kv) at chunk kv/8, unit (kv%8) ^ (jl & 7).
          // Global loads first (<= 2 vectors per thread at r = 32), then wait until the previous
          // fused tile's MMAs have released the a / B tiles, then store.
          const int rh = p.nx_r / 2;
          uint8_t *bt = smem + LY::bt_off;
          uint4 val[2];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int v = et + kEpiT * k;
            const int jl = v / (BN / 8), kv = v % (BN / 8);
            const int64_t col = n0 + kv * 8;
            val[k] = (v < rh * (BN / 8) && col < p.N)
                         ? *reinterpret_cast<const uint4 *>(p.nx_l1s + static_cast<int64_t>(crank * rh + jl) * p.N + col)
                         : make_uint4(0, 0, 0, 0);
          }
          if (xl_cnt > 0) mbar_wait(xa_empty, (xl_cnt - 1) & 1);
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int v = et + kEpiT * k;
            const int jl = v / (BN / 8), kv = v % (BN / 8);
            if (v < rh * (BN / 8))
              sts128(smem_u32(bt) + (kv >> 3) * 2048 + jl * 128 + (((kv & 7) ^ (jl & 7)) << 4), val[k].x, val[k].y,
                     val[k].z, val[k].w);
          }
        }
      }
      named_bar(1, kEpiT);
      { K2T_BEGIN(); mbar_wait(&acc_full[b], acc_ph); K2T_ACC(t_ewait); }
      tc_fence_after();
#ifdef SVDQ_TRACE
      const long long _td = clock64();
#endif
#if SVDQ_EXP & 16                                        // ablation: no epilogue work at all
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc_empty0 + b * 8);
      continue;
#endif
#ifdef SVDQ_EPI_DIRECT
      epilogue_tile_direct<BN, 2>(tmem + b * BN + (static_cast<uint32_t>(quad * 32) << 16), bias_s, p.alpha,
                                  p.y_dtype, p.Y, p.ldy, p.M, p.N, m0 + quad * 32, n0, (warp - 2) >> 2, lane, [&]() {
                                    tc_fence_before();
                                    __syncwarp();
                                    if (lane == 0) mbar_arrive_cluster(acc_empty0 + b * 8);
                                  });
      continue;
#endif
#if SVDQ_BIGSTORE
      if (kBN == 192 && p.y_dtype != 2) {
        // drain the 3 column chunks of this warp, release the accumulator, then each 64-column
        // block of the CTA's 128 x 192 tile is assembled by all 8 warps and stored by one TMA op
        const int sub = (warp - 2) >> 2;
        const uint32_t lane_addr = tmem + b * BN + (static_cast<uint32_t>(quad * 32) << 16);
        uint32_t r[3][32];
#pragma unroll
        for (int i = 0; i < 3; ++i) tmem_ld_32x32b_x32(lane_addr + (sub + 2 * i) * 32, r[i]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc_empty0 + b * 8);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          uint8_t *blk = smem + LY::epi_off + i * 16384;
          if (et == 0) bulk_wait_group_read<2>();        // this block's previous store has read it
          named_bar(2, 256);
          const float *bs = bias_s + (sub + 2 * i) * 32;
          uint8_t *rowp = blk + row * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(__fmul_rn(p.alpha, __uint_as_float(r[i][8 * c + e])), bs[8 * c + e]);
            const int j = 4 * sub + c;                     // 16-byte column of the 128-byte row
            *reinterpret_cast<uint4 *>(rowp + ((j ^ (row & 7)) * 16)) =
                make_uint4(pack2(o[0], o[1], p.y_dtype), pack2(o[2], o[3], p.y_dtype), pack2(o[4], o[5], p.y_dtype),
                           pack2(o[6], o[7], p.y_dtype));
          }
          fence_proxy_async();
          named_bar(3, 256);
          if (et == 0) {
            tma_store_2d(tmY, blk, static_cast<int32_t>(n0 + 64 * i), static_cast<int32_t>(m0));
            bulk_commit_group();
          }
        }
        continue;
      }
#endif
      if constexpr (kFuse) {
        if (p.fuse) {
          epilogue_tile_next<BN, kNWQ, LY::epibuf>(
              tmem + b * BN + (static_cast<uint32_t>(quad * 32) << 16), bias_s, p.alpha, p.Y ? tmY : nullptr,
              static_cast<int32_t>(m0 + quad * 32), static_cast<int32_t>(n0), (warp - 2) >> 2,
              smem + LY::epi_off + (warp - 2) * 2048 * LY::epibuf, ebuf, lane,
              [&]() {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) K2_ACC_RELEASE(acc_empty0 + b * 8);
              },
              p, reinterpret_cast<const float *>(smem + LY::lamn_off), fx ? smem + LY::at_off : nullptr, row,
              [&]() {
                if (fx) {   // a / B tiles written (generic proxy) -> visible to the tensor core; arrive
                  fence_proxy_async();
                  __syncwarp();
                  if (lane == 0) mbar_arrive_cluster(xa_full0);
                }
              },
              smem + LY::cs_off, smem + LY::sfs_off, quad);
          named_bar(2, kEpiT);                           // code / SF staging complete (fenced per thread)
          if (et == 0 && m0 < p.M) {
            tma_store_2d(&g.pr[tr.i].nxq, smem + LY::cs_off, static_cast<int32_t>(n0 / 2), static_cast<int32_t>(m0));
            const int64_t nkt_n = p.N / 64;              // 512-B scale-factor blocks per 128 rows
            const int nblk = static_cast<int>(nkt_n - n0 / 64 < 3 ? nkt_n - n0 / 64 : 3);
            bulk_store(p.nx_sf + (m0 >> 7) * nkt_n * 512 + (n0 / 64) * 512, smem + LY::sfs_off,
                       static_cast<uint32_t>(nblk * 512));
            bulk_commit_group();
          }
          if (fx) {
            // leaving this 256-row block (or the range): read the accumulated X L1s_next^T rows from
            // TMEM once the MMAs of this tile are done, and write them to this pair's slot
            bool flush = t + t_step >= t_end;
            if (!flush) {
              const TileRef nr = locate<kBN>(g, t + t_step);
              flush = nr.i != tr.i || nr.m0 != tr.m0;
            }
            if (flush) {
              mbar_wait(xa_empty, xl_cnt & 1);
              tc_fence_after();
              uint32_t xr[32];
              tmem_ld_32x32b_x32(tmem + XL1_COL + (static_cast<uint32_t>(quad * 32) << 16), xr);
              tmem_ld_wait();
              if (((warp - 2) >> 2) == 0) {
                const int nt = static_cast<int>((p.N + BN - 1) / BN);
                const int mb = static_cast<int>(tr.m0 / 256);
                const int64_t t0 = g.tile_begin[tr.i] + static_cast<int64_t>(mb) * nt;
                const int pf = static_cast<int>(((t0 + 1) * npairs - 1) / tiles);
                float *dst = p.nx_part +
                             ((static_cast<int64_t>(mb) * p.nx_slots + (pair - pf)) * 256 + 128 * crank + row) * p.nx_r;
                for (int j = 0; j < p.nx_r; j += 4)
                  *reinterpret_cast<float4 *>(dst + j) = make_float4(__uint_as_float(xr[j]), __uint_as_float(xr[j + 1]),
                                                                     __uint_as_float(xr[j + 2]), __uint_as_float(xr[j + 3]));
              }
              tc_fence_before();                         // the read precedes the next run's first MMA
            }
            ++xl_cnt;
          }
          continue;
        }
      }
      if constexpr (kW8) {
        const int64_t grow = m0 + quad * 32 + lane;       // per-token activation scale of this lane's row
        const float sx = grow < p.M ? reinterpret_cast<const float *>(p.sfa)[grow] : 0.f;
        epilogue_tile_w8<BN, kNWQ, LY::epibuf>(tmem + (static_cast<uint32_t>(quad * 32) << 16), LR_COL, p.rank > 0,
                                               bias_s, reinterpret_cast<const float *>(smem + LY::sw_off), sx,
                                               p.y_dtype, tmY, static_cast<int32_t>(m0 + quad * 32),
                                               static_cast<int32_t>(n0), (warp - 2) >> 2,
                                               smem + LY::epi_off + (warp - 2) * 2048 * LY::epibuf, ebuf, lane, [&]() {
                                                 tc_fence_before();
                                                 __syncwarp();
                                                 if (lane == 0) K2_ACC_RELEASE(acc_empty0);
                                               });
        continue;
      }
      if constexpr (kBN == 384) {
        epilogue_tile_wide<BN, kNWQ, LY::epibuf>(tmem + (static_cast<uint32_t>(quad * 32) << 16), bias_s, p.alpha,
                                                 p.y_dtype, tmY, static_cast<int32_t>(m0 + quad * 32),
                                                 static_cast<int32_t>(n0), (warp - 2) >> 2,
                                                 smem + LY::epi_off + (warp - 2) * 2048 * LY::epibuf, ebuf, lane, [&]() {
                                                   tc_fence_before();
                                                   __syncwarp();
                                                   if (lane == 0) K2_ACC_RELEASE(acc_empty0);
                                                 });
        continue;
      }
      epilogue_tile<BN, kNWQ, LY::epibuf>(tmem + b * BN + (static_cast<uint32_t>(quad * 32) << 16), bias_s, p.alpha, p.y_dtype,
                           tmY, static_cast<int32_t>(m0 + quad * 32), static_cast<int32_t>(n0), (warp - 2) >> 2,
                           smem + LY::epi_off + (warp - 2) * 2048 * LY::epibuf, ebuf, lane, [&]() {
                          tc_fence_before();
                          __syncwarp();
                          if (lane == 0) K2_ACC_RELEASE(acc_empty0 + b * 8);
#ifdef SVDQ_TRACE
                          t_edrain += clock64() - _td;
#endif
                        });
    }
#ifdef SVDQ_TRACE
    if (warp == 2 && lane == 0 && crank == 0 && pair < 148) {
      g_k2p_trace[pair][3] = t_ewait; g_k2p_trace[pair][4] = t_edrain; g_k2p_trace[pair][5] = clock64() - t_estart;
    }
#endif
  }
  if (warp >= 2 && lane == 0) bulk_wait_group<0>();    // outstanding TMA stores done
  tc_fence_before();
  cluster_sync();                                        // all MMAs, loads and reads are done
  if (warp == 1) tmem_dealloc_cg2(tmem, 512);
}

}  // namespace

namespace {
template <int kBN, bool kW8 = false>
cudaError_t launch_plain(const K2PairArgs &g, int64_t pairs, cudaStream_t s) {
  using LY = Lay<false, kBN, kW8>;
  cudaError_t e = cudaFuncSetAttribute(k2_nvfp4_2sm_kernel<false, kBN, kW8>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, LY::smem);
  if (e != cudaSuccess) return e;
  return launch_ex(k2_nvfp4_2sm_kernel<false, kBN, kW8>, dim3(static_cast<unsigned>(2 * pairs)), dim3(LY::threads),
                   LY::smem, s, 2u, g);
}
}  // namespace

cudaError_t launch_k2_nvfp4_2sm_group(K2PairArgs &g, cudaStream_t s) {
  static_assert(Lay<false, 192>::smem <= 227 * 1024 && Lay<false, 256>::smem <= 227 * 1024 &&
                Lay<false, 384>::smem <= 227 * 1024, "smem budget");
  static_assert(Lay<true>::smem <= 227 * 1024, "smem budget (fused)");
  static_assert(Lay<false, 192, true>::smem <= 227 * 1024, "smem budget (W8A8)");
  bool fuse = false, w8 = false;
  for (int i = 0; i < g.n; ++i) {
    fuse = fuse || g.pr[i].p.fuse;
    w8 = w8 || g.pr[i].p.w8;
  }
  const int bn = fuse || w8 ? 192 : (g.bn == 384 || g.bn == 256 ? g.bn : 192);
  g.bn = bn;
  g.tile_begin[0] = 0;
  for (int i = 0; i < g.n; ++i)
    g.tile_begin[i + 1] = g.tile_begin[i] + static_cast<int>(((g.pr[i].p.M + 255) / 256) * ((g.pr[i].p.N + bn - 1) / bn));
  const int64_t tiles = g.tile_begin[g.n];
  const int64_t pairs = k2_pair_count(tiles);
  // L2 banding (large M): the m-fastest order re-streams the whole of A for every weight column
  // tile; once A (M x K codes + scales) outgrows the L2 budget -- FLUX batch >= 4 -- its rows come
  // from DRAM again for each of the N / BN columns.  Band size: as many 256-row tiles as fit
  // SVDQ_K2_BAND_MB (default 16 MB; swept 8 / 16 / 32 / 48 / 80 on the 57-block stack) of A,
  // balanced over the bands.  At batch 1 only the K >= 12288 launches band (2-3 bands; timing
  // unchanged); batch 8 gains 12 % (tools/c5_stack.py).
  static const double band_mb = [] { const char *e = std::getenv("SVDQ_K2_BAND_MB"); return e ? std::atof(e) : 16.0; }();
  for (int i = 0; i < g.n; ++i) {
    K2Params &p = g.pr[i].p;
    const int64_t mt = (p.M + 255) / 256;
    const double tile_bytes = 256.0 * static_cast<double>(p.K) * (p.w8 ? 1.0 : 0.5625);
    int64_t cap = band_mb > 0 ? static_cast<int64_t>(band_mb * 1048576.0 / tile_bytes) : mt;
    if (cap < 1) cap = 1;
    if (p.fuse || mt <= cap) {
      p.band = 0;
    } else {
      const int64_t nb = (mt + cap - 1) / cap;
      p.band = static_cast<int>((mt + nb - 1) / nb);
    }
  }
  static const int force_contig = [] { const char *e = std::getenv("SVDQ_K2_CONTIG"); return e ? std::atoi(e) : 0; }();
  g.contig = (fuse || force_contig) ? 1 : 0;      // SVDQ_K2_CONTIG=1: schedule ablation
  g.npairs = static_cast<int>(pairs);
  if (fuse) {
    cudaError_t e = cudaFuncSetAttribute(k2_nvfp4_2sm_kernel<true, 192>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Lay<true>::smem);
    if (e != cudaSuccess) return e;
    return launch_ex(k2_nvfp4_2sm_kernel<true, 192>, dim3(static_cast<unsigned>(2 * pairs)), dim3(Lay<true>::threads),
                     Lay<true>::smem, s, 2u, g);
  }
  if (w8) return launch_plain<192, true>(g, pairs, s);
  if (bn == 384) return launch_plain<384>(g, pairs, s);
  if (bn == 256) return launch_plain<256>(g, pairs, s);
  return launch_plain<192>(g, pairs, s);
}

int k2_pair_bn(int64_t N) {
  // 256 when it divides N.  The 384-wide tile is built and correct but measured no faster on the
  // FLUX shapes (linear1 126 vs 123 us, qkv 53 vs 49 us with 6 vs 8 waves, linear2 74.3 vs 73.5 us):
  // its 16 % fewer operand bytes per FLOP are offset by the 4- instead of 5-deep ring and the
  // longer single-accumulator drain (clock64 trace: MMA waits on operands 22 % of the time at both
  // widths).  SVDQ_K2_BN=384 opts in; SVDQ_K2_BN=192 caps at 192 (A/B).
  static const int cap = [] { const char *e = std::getenv("SVDQ_K2_BN"); return e ? std::atoi(e) : 256; }();
  if (cap >= 384 && N % 384 == 0) return 384;
  if (cap >= 256 && N % 256 == 0) return 256;
  return 192;
}

int device_sm_count() {
  static int cached[64];                      // 0 = not yet queried
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = sms;
  return sms;
}

int k2_pair_count(int64_t tiles) {
  const int sms = device_sm_count();
  return static_cast<int>(tiles < sms / 2 ? tiles : sms / 2);
}

int k2_next_slots(int64_t nt, int64_t tiles, int npairs) {
  const int64_t minlen = npairs > 0 ? tiles / npairs : 1;      // shortest contiguous range
  return static_cast<int>((nt + (minlen > 0 ? minlen : 1) - 1) / (minlen > 0 ? minlen : 1) + 1);
}

namespace {
__global__ void next_reduce_kernel(const float *__restrict__ part, int64_t M, int r, int nt, int slots,
                                   int64_t tile_begin, int tiles, int npairs, uint16_t *__restrict__ out) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= M * r) return;
  const int64_t m = idx / r;
  const int j = static_cast<int>(idx % r);
  const int mb = static_cast<int>(m / 256);
  const int64_t t0 = tile_begin + static_cast<int64_t>(mb) * nt, t1 = t0 + nt - 1;
  const int pf = static_cast<int>(((t0 + 1) * npairs - 1) / tiles);
  const int pl = static_cast<int>(((t1 + 1) * npairs - 1) / tiles);
  float acc = 0.f;
  for (int sl = 0; sl <= pl - pf; ++sl) acc += part[((static_cast<int64_t>(mb) * slots + sl) * 256 + (m % 256)) * r + j];
  out[idx] = __bfloat16_as_ushort(__float2bfloat16_rn(acc));
}
}  // namespace

cudaError_t launch_k2_next_reduce(const K2PairArgs &g, int i, uint16_t *xl1_next, cudaStream_t s) {
  const K2Params &p = g.pr[i].p;
  if (!p.fuse || p.nx_r == 0) return cudaSuccess;
  const int nt = static_cast<int>((p.N + BN - 1) / BN);
  const int64_t n = p.M * p.nx_r;
  next_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      p.nx_part, p.M, p.nx_r, nt, p.nx_slots, g.tile_begin[i], g.tile_begin[g.n], g.npairs, xl1_next);
  return cudaGetLastError();
}

cudaError_t launch_k2_nvfp4_2sm(const K2Maps &maps, const CUtensorMap &sfa, const CUtensorMap &sfb,
                                const K2Params &p, int bn, cudaStream_t s) {
  K2PairArgs g;                              // host staging, copied into the launch parameters
  static_assert(sizeof(K2PairArgs) < 30 * 1024, "kernel parameter space");
  g.n = 1;
  g.bn = bn;
  g.pr[0].a = maps.a;
  g.pr[0].b = maps.b;
  g.pr[0].xl1 = maps.xl1;
  g.pr[0].l2 = maps.l2;
  g.pr[0].sfa = sfa;
  g.pr[0].sfb = sfb;
  g.pr[0].y = maps.y;
  g.pr[0].p = p;
  return launch_k2_nvfp4_2sm_group(g, s);
}

}  // namespace svdq
