// K1 (round 2): smoothing + activation quantization + low-rank down-projection on ONE read of X
// ("Fused Quantize + Down Projection", Fig. 5(b)), row-tile design.
//
// Every CTA owns RT whole rows of X (RT = 16 / 32 / 64 / 128, chosen so that one wave covers all
// 148 SMs) and streams them over the full K -- so no CTA ever needs another CTA's partial sums:
// no cluster, no distributed-shared-memory reduction, no trailing cluster barrier.
//
//   stage i = Q = 128 / RT consecutive 64-wide K blocks of the CTA's RT rows, staged by ONE 3-D TMA
//             box {64 cols, Q blocks, RT rows} (128-B swizzle) as a [128 rows x 128 B] K-major tile
//             whose row m * Q + q holds block q of row m; X stages and L1s stages live in two rings;
//   warp 0    X producer (X box + lambda_inv of the Q blocks; X ring, up to 12 deep);
//   warp 1    TMEM allocator + MMA issuer: D[128 x Q*r] += A[128 x 64] . B[Q*r x 64]^T with
//             B row q' * r + t = L1s[t, block q'] (tcgen05.mma kind::f16, fp32 in TMEM).  The
//             diagonal entries D[m Q + q, q r + t] accumulate sum_k X[m, k] L1s[t, k] over the k of
//             block q of every stage; the off-diagonal products are discarded (the MMA is ~1/3 of
//             the HBM time, so the Q-fold extra tensor work is free);
//   warp 2    L1s producer (Q tiles [r x 64] per stage; L1s ring, 4 deep, fed from L2 after a
//             distributed L2 prefetch of the whole L1s);
//   warps 3..18  quantizers, one 16-element NVFP4 group (a quarter of an INT4 group) per lane per
//             stage: x_hat = fl32(x * lambda_inv), App. B recipe bit-exact, codes + scales stored.
//             fp16 X: they also split the tile into bf16 hi (in place) + lo parts, X = hi + lo
//             exactly, and the MMA warp issues hi . L1s^T + lo . L1s^T (kind::f16 takes one type).
//   tail      xl1[m, t] = bf16(sum_q D[m Q + q, q r + t]) in a fixed q order (deterministic), by
//             warp shuffles straight out of TMEM.
// X rows >= M are zero-filled by TMA, so the NVFP4 padding rows of the 128x4 scale layout get 0x00.
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "k1_launch.h"
#include "sm100.cuh"

#ifndef SVDQ_K1REXP
#define SVDQ_K1REXP 0   // ablation bits: 1 no quantizer math / stores, 2 no MMA, 4 no L1s loads, 8 no L1s L2 prefetch,
                        // 16 no code / scale stores, 32 no qinv table lookup
#endif

#ifdef SVDQ_TRACE
namespace svdq { __device__ unsigned long long g_k1r_trace[512]; }
extern "C" int svdq_k1r_trace_read(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, svdq::g_k1r_trace, sizeof(unsigned long long) * 512) == cudaSuccess ? 0 : 1;
}
__device__ __forceinline__ unsigned long long k1r_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
#define RTRACE(slot) \
  do { if (blockIdx.x == 0) svdq::g_k1r_trace[(slot)] = k1r_gtime(); } while (0)
// SM-clock stamps of the tail (slots 500-503), consistent within the CTA
#define CTRACE(slot) \
  do { if (blockIdx.x == 0) svdq::g_k1r_trace[(slot)] = clock64(); } while (0)
#else
#define RTRACE(slot) do {} while (0)
#define CTRACE(slot) do {} while (0)
#endif

namespace svdq {

namespace {

// Waits of the single-thread roles (producers, MMA issuer): with the suspend-time hint, so a waiting
// role warp does not take issue slots from the quantizer warps of its sub-partition (measured
// neutral against spinning, SVDQ_K1_SPIN=1, on the FLUX shapes).
#ifndef SVDQ_K1_SPIN
#define SVDQ_K1_SPIN 0
#endif
// Waits of the quantizer warps (stage full, the tail's dfull): SVDQ_K1_QSPIN=1 spins instead of
// suspending (A/B of the wake-up latency on small launches).
#ifndef SVDQ_K1_QSPIN
#define SVDQ_K1_QSPIN 0
#endif
__device__ __forceinline__ void q_wait(uint64_t *bar, uint32_t parity) {
  if (SVDQ_K1_QSPIN) mbar_wait_spin(bar, parity);
  else mbar_wait(bar, parity);
}
__device__ __forceinline__ void role_wait(uint64_t *bar, uint32_t parity) {
  if (SVDQ_K1_SPIN) mbar_wait_spin(bar, parity);
  else mbar_wait(bar, parity);
}

constexpr int kQuantWarps = 16;
constexpr int kQ0 = 3;                                 // first quantizer warp (0 X producer, 1 MMA, 2 L1s producer)
constexpr int kThreads = 32 * (kQ0 + kQuantWarps);
constexpr int kMaxXStages = 12;
constexpr int kMaxWStages = 4;
#ifndef SVDQ_K1_SW
#define SVDQ_K1_SW 4                                   // L1s ring depth (the tiles come from L2)
#endif
static_assert(SVDQ_K1_SW >= 2 && SVDQ_K1_SW <= kMaxWStages, "L1s ring depth");
#ifndef SVDQ_K1_XPRE
#define SVDQ_K1_XPRE 12                                // X boxes prefetched to L2 before griddepcontrol.wait
#endif
#ifndef SVDQ_K1_LAMPRE
#define SVDQ_K1_LAMPRE 2                               // ring slots whose lambda tile goes out before griddepcontrol.wait
#endif

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {     // sm_100a packed FMUL2
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t pack64(uint32_t lo, uint32_t hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(hi));
  return d;
}
__device__ __forceinline__ float lo32(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float hi32(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
// two 16-bit activations in one word -> fp32 pair (exact), low element in the low word
template <bool kX16>
__device__ __forceinline__ uint64_t x2_to_f32x2(uint32_t w) {
  if constexpr (kX16) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w));
    return pack64(__float_as_uint(f.x), __float_as_uint(f.y));
  } else {
    return pack64(w << 16, w & 0xFFFF0000u);
  }
}
__device__ __forceinline__ void lds_v2x64(uint32_t addr, uint64_t &a, uint64_t &b) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}
// four packed fp32 pairs -> 32 bits of E2M1 (pair j -> byte j, low element in the low nibble)
__device__ __forceinline__ uint32_t e2m1x8_pairs(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint32_t r;
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}\n"
      : "=r"(r)
      : "f"(lo32(a)), "f"(hi32(a)), "f"(lo32(b)), "f"(hi32(b)), "f"(lo32(c)), "f"(hi32(c)), "f"(lo32(d)),
        "f"(hi32(d)));
  return r;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(lo))) |
         (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(hi))) << 16);
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int32_t c0, int32_t c1,
                                            int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// L2 prefetch of a 3-D box (no smem destination, no completion tracking)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *map, int32_t c0, int32_t c1, int32_t c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

}  // namespace

K1RowLayout k1_row_layout(int rt, int rank, bool x16) {
  // Two rings: X stages (the DRAM stream: X tile + the Q blocks' lambda_inv) and L1s stages (Q
  // tiles [r x 64], L2-resident).  Splitting them lets the X ring run deeper than the L1s ring --
  // the L1s tiles of a stage are as large as its X tile at RT = 32, r = 32, and only the X bytes
  // need to be in flight long enough to cover the DRAM latency.
  K1RowLayout L;
  L.rt = rt;
  L.q = 128 / rt;
  L.x_bytes = x16 ? 32768 : 16384;                   // fp16 X: + the bf16 low parts (hi stays in place)
  L.stage_bytes = (L.x_bytes + L.q * 256 + 1023) / 1024 * 1024;
  L.l1_bytes = L.q * rank * 128;                     // multiple of 2 KB (rank % 16 == 0)
  L.wstages = rank ? SVDQ_K1_SW : 0;
  const int s = (212 * 1024 - L.wstages * L.l1_bytes) / L.stage_bytes;
  L.stages = s > kMaxXStages ? kMaxXStages : (s < 2 ? 2 : s);
  L.w_off = static_cast<size_t>(L.stages) * L.stage_bytes;
  L.bar_off = L.w_off + static_cast<size_t>(L.wstages) * L.l1_bytes;
  L.smem = L.bar_off + 512 + 1024 + 512 + 1024;      // barriers, 256-entry qinv table, W8A8 row amax, slack
  return L;
}

namespace {

template <int kFmt, bool kScaleBf16, bool kX16>
__global__ void __launch_bounds__(kThreads, 1) k1_rows_kernel(const __grid_constant__ K1Args g, K1RowLayout Ly) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~static_cast<uintptr_t>(1023));
  int pi = 0;                                                  // problem of this row tile
  while (pi + 1 < g.n && static_cast<int>(blockIdx.x) >= g.tile_begin[pi + 1]) ++pi;
  const K1Params &p = g.pr[pi].p;
  const CUtensorMap &tmX = g.pr[pi].x, &tmL = g.pr[pi].l1s, &tmLam = g.pr[pi].lam;
  const int r = p.rank;
  const int RT = Ly.rt, Q = Ly.q, S = Ly.stages, SW = Ly.wstages;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + Ly.bar_off);   // X ring
  uint64_t *empty = full + kMaxXStages;
  uint64_t *conv = empty + kMaxXStages;                        // fp16 X: hi / lo tiles written
  uint64_t *wfull = conv + kMaxXStages;                        // L1s ring
  uint64_t *wempty = wfull + kMaxWStages;
  uint64_t *dfull = wempty + kMaxWStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(dfull + 1);
  float *qinv_lut = reinterpret_cast<float *>(smem + Ly.bar_off + 512);
  uint32_t *rowmax = reinterpret_cast<uint32_t *>(smem + Ly.bar_off + 512 + 1024);   // W8A8: [RT] amax bits
  // the tail's output parameters, staged in smem at setup: read from the (dynamically indexed)
  // parameter space at the end of the kernel they cost a few hundred cycles of constant-cache miss
  int64_t *tailp = reinterpret_cast<int64_t *>(smem + Ly.bar_off + 384);   // {xl1, xl1_f32, M}
  uint8_t *wring = smem + Ly.w_off;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t K = p.K;
  const int nkb = static_cast<int>(K / 64);
  const int nsteps = (nkb + Q - 1) / Q;                        // the last stage may hold < Q blocks
  const int64_t row0 = static_cast<int64_t>(static_cast<int>(blockIdx.x) - g.tile_begin[pi]) * RT;
  uint32_t tcols = 32;
  while (tcols < static_cast<uint32_t>(Q * r)) tcols <<= 1;

  if (threadIdx.x == 0) RTRACE(0);
  if (warp == 0) {                                             // lane s initialises the barriers of slot s
    if (lane < S) {
      mbar_init(&full[lane], 1);
      mbar_init(&empty[lane], kQuantWarps / 2 + (r ? 1 : 0));   // one team + the MMA
      mbar_init(&conv[lane], kQuantWarps / 2);
    }
    if (lane < SW) {
      mbar_init(&wfull[lane], 1);
      mbar_init(&wempty[lane], 1);
    }
    if (lane == 31) mbar_init(dfull, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmLam);
  }
  if (warp == 2 && lane == 0 && r) tma_prefetch(&tmL);
  if (warp == 1 && r) tmem_alloc_n(tmem_slot, tcols);
  if (kFmt == 0 && threadIdx.x >= 32 * kQ0 && threadIdx.x < 32 * kQ0 + 256) {
    const uint32_t code = threadIdx.x - 32 * kQ0;             // UE4M3 byte; 0x7F.. never produced
    const float sfd = e4m3_to_f32(code & 0x7F);
    qinv_lut[code] = sfd == 0.f ? 0.f : __frcp_rn(__fmul_rn(sfd, p.gs_x));
  }
  if (kFmt == 2 && threadIdx.x < RT) rowmax[threadIdx.x] = 0u;
  if (threadIdx.x == 64) {
    tailp[0] = reinterpret_cast<int64_t>(p.xl1);
    tailp[1] = reinterpret_cast<int64_t>(p.xl1_f32);
    tailp[2] = p.M;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = r ? *tmem_slot : 0;
  if (threadIdx.x == 0) RTRACE(1);
  griddep_launch_dependents();                                 // the next kernel may start its prologue

  if (warp == 0) {
    // -------------------------------------------------------------------- X producer
    if (elect_one()) {
      // every box is loaded whole: blocks past K / rows past M are zero-filled by TMA (and counted)
      const uint32_t stage_tx = static_cast<uint32_t>(16384 + Q * 256);
      // lambda_inv of the nb blocks as [2 nb][32] fp32 rows, 128-B swizzle (conflict-free broadcasts)
      auto load_lam = [&](int i, int s) {
        mbar_arrive_expect_tx(&full[s], stage_tx);
        tma_load_2d(smem + s * Ly.stage_bytes + Ly.x_bytes, &tmLam, &full[s], 0, (i * Q) * 2);
      };
      // Before the programmatic dependency resolves (the previous kernel may still run and may
      // write X): the first ring's lambda tiles (no kernel of this stream writes them).
      const int npre = S < SVDQ_K1_LAMPRE ? S : SVDQ_K1_LAMPRE;   // lambda tiles issued before the wait
      for (int i = 0; i < nsteps && i < npre; ++i) load_lam(i, i);
      // ... and an L2 prefetch of the first ring's X boxes: it overlaps the cold first access
      // (~1.6 us) with the previous kernel's tail.  Safe while that kernel may still write X:
      // L2 is the coherence point and the TMA loads below are issued after the wait.
      for (int i = 0; i < nsteps && i < (SVDQ_K1_XPRE < S ? SVDQ_K1_XPRE : S); ++i)
        tma_prefetch_3d(&tmX, 0, static_cast<int32_t>(row0), i * Q);
      griddep_wait();
      int s = 0;
      uint32_t ph = 0;                                          // ring round parity of slot s
      for (int i = 0; i < nsteps; ++i) {
        if (i >= S) {
          role_wait(&empty[s], ph ^ 1);
          load_lam(i, s);
        }
        if (i < 64) RTRACE(2 + i);
        // X box {64 cols, Q blocks, RT rows}
        tma_load_3d(smem + s * Ly.stage_bytes, &tmX, &full[s], 0, static_cast<int32_t>(row0), i * Q);
        if (i + npre < S && i + npre < nsteps) load_lam(i + npre, i + npre);   // rest of the first ring
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
    __syncwarp();                                        // reconverge before the block-wide barrier
  } else if (warp == 2) {
    // -------------------------------------------------------------------- L1s producer
    // L1s never depends on the previous kernel: the ring fills before griddepcontrol.wait
    if (r && !(SVDQ_K1REXP & 4) && elect_one()) {
      // Distributed L2 prefetch of the whole L1s (r x K bf16, <= 1 MB at FLUX shapes): this
      // problem's CTAs each fetch every ntiles-th [r x 64] box.  All CTAs walk K in near lockstep,
      // so without it every stage's tiles would be first touched -- and waited for -- behind the X
      // stream's DRAM queue; with it the L1s ring is fed from L2.
      if (!(SVDQ_K1REXP & 8)) {
        const int ntile = g.tile_begin[pi + 1] - g.tile_begin[pi];
        for (int j = static_cast<int>(blockIdx.x) - g.tile_begin[pi]; j < nkb; j += ntile)
          tma_prefetch_2d(&tmL, j * 64, 0);
      }
      int sw = 0;
      uint32_t wph = 0;
      for (int i = 0; i < nsteps; ++i) {
        if (i >= SW) role_wait(&wempty[sw], wph ^ 1);
        if (i < 64) RTRACE(200 + i);
        mbar_arrive_expect_tx(&wfull[sw], static_cast<uint32_t>(Ly.l1_bytes));
        for (int q = 0; q < Q; ++q)
          tma_load_2d(wring + sw * Ly.l1_bytes + q * r * 128, &tmL, &wfull[sw], (i * Q + q) * 64, 0);
        if (++sw == SW) { sw = 0; wph ^= 1; }
      }
    }
    __syncwarp();                                        // reconverge before the block-wide barrier
  } else if (warp == 1) {
    // -------------------------------------------------------------------- MMA issuer
    if (r) {
      const uint32_t idesc = idesc_bf16(128, static_cast<uint32_t>(Q * r));
      int s = 0, sw = 0;
      uint32_t ph = 0, wph = 0;
      for (int i = 0; i < nsteps; ++i) {
        role_wait(&full[s], ph);
        if (kX16) role_wait(&conv[s], ph);                      // hi / lo bf16 tiles written
        if (!(SVDQ_K1REXP & 4)) role_wait(&wfull[sw], wph);
        if (lane == 0 && i < 64) RTRACE(300 + i);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t xa = smem_u32(smem + s * Ly.stage_bytes);
          const uint32_t la = smem_u32(wring + sw * Ly.l1_bytes);
#pragma unroll
          for (int j = 0; j < ((SVDQ_K1REXP & 2) ? 0 : 4); ++j)
            mma_bf16(tmem, sdesc_kmajor_sw128(xa + 32 * j), sdesc_kmajor_sw128(la + 32 * j), idesc,
                     (i | j) != 0);
          if (kX16) {                                            // + X_lo . L1s^T (X = hi + lo exactly)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              mma_bf16(tmem, sdesc_kmajor_sw128(xa + 16384 + 32 * j), sdesc_kmajor_sw128(la + 32 * j), idesc, 1u);
          }
          tc_commit(&empty[s]);
          tc_commit(&wempty[sw]);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
        if (++sw == SW) { sw = 0; wph ^= 1; }
      }
      if (elect_one()) tc_commit(dfull);
      __syncwarp();
    }
  } else {
    // -------------------------------------------------------------------- quantizers
    // Two teams of 8 warps take alternate stages (team t: stages i = t mod 2), and each thread
    // takes TWO groups of its team's stage: staged rows R and R + 64, which hold the same K block
    // (R = m Q + qb, Q | 64) and so share one set of lambda_inv loads.  Shared memory is this
    // kernel's binding resource (ncu: every LDS.128 costs 4 wavefronts; quantizer loads + tcgen05
    // operand reads + TMA fills ~ 1000 wavefronts per 16 KB stage); sharing the lambda loads
    // removes a third of the quantizers' wavefronts, and the two teams overlap each other's
    // load latency.
    const int qw = warp - kQ0;
    const int team = qw >> 3;
    // block-major stage: staged row R = q RT + m (block q of tile row m).  Pair index pidx (64 per
    // team) -> block qb and rows m, m + RT / 2 of that block (same K block: one set of lambda loads)
    const int half = RT / 2;
    const int pidx = (qw & 7) * 8 + (lane >> 2);
    const int R = (pidx / half) * RT + pidx % half;             // staged tile rows R and R + RT / 2
    const int q4 = lane & 3;                                    // 16-element group within the block
    const int qb = pidx / half;                                 // K block within the stage (both rows)
    const int mh[2] = {pidx % half, pidx % half + half};        // rows within the tile
    const float t6 = __fmul_rn(__frcp_rn(p.gs_x), __frcp_rn(6.0f));
    // output addressing: the layer's own layout (out_k = K, out_c0 = 0), or -- fused tensor-parallel
    // gather -- this K-slice's place inside the full-K layout (out_k = full K, out_c0 = k0 / 16)
    int64_t rowh[2];
    bool rvalid[2];
    uint8_t *xq_base[2], *sf_base[2], *s16_base[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t row = row0 + mh[h];
      rowh[h] = row;
      rvalid[h] = row < p.M && mh[h] < RT;
      xq_base[h] = p.xq + row * (p.out_k / 2) + static_cast<int64_t>(qb) * 32 + q4 * 8;
      sf_base[h] = p.xs + sf_offset(row, p.out_c0, p.out_k) + static_cast<int64_t>(qb) * 512 + q4;
      s16_base[h] = p.xs + 2 * (row * (p.out_k / 64) + p.out_c0 / 4 + qb);
    }
    const uint32_t swz = static_cast<uint32_t>(R & 7);          // == (R + RT / 2) & 7 (RT / 2 % 8 == 0)
    const uint32_t lut = smem_u32(qinv_lut);
    const uint32_t stage0 = smem_u32(smem);
    // lambda row j = 2 qb + (q4 >> 1) of the swizzled [2Q][128 B] block; chunk (q4 & 1) * 4 + t
    const int jl = 2 * qb + (q4 >> 1);
    uint32_t lam_off[4];
#pragma unroll
    for (int t = 0; t < 4; ++t)
      lam_off[t] = static_cast<uint32_t>(Ly.x_bytes + jl * 128 + ((((q4 & 1) * 4 + t) ^ (jl & 7)) * 16));
    const uint32_t x_off[2] = {static_cast<uint32_t>(R * 128) + ((static_cast<uint32_t>(2 * q4) ^ swz) * 16),
                               static_cast<uint32_t>(R * 128) + ((static_cast<uint32_t>(2 * q4 + 1) ^ swz) * 16)};
    const int ndst = p.ndst;                                    // 1, or the ranks of a fused gather
    const int64_t d0 = p.dst_delta[0];

    // This team's next stage: slot and round parity (stages advance by 2)
    int qs = team % S;
    uint32_t qph = team >= S ? 1u : 0u;
    auto next_slot = [&]() {
      qs += 2;
      if (qs >= S) { qs -= S; qph ^= 1; }
    };
    // Stage i -> x_hat pairs (fl32(x * lambda_inv)) of both rows in registers, then the slot is released.
    auto load_stage = [&](int i, uint64_t (&xh)[2][8]) {
      const int s = qs;
      q_wait(&full[s], qph);
      next_slot();
      if (qw == 0 && lane == 0 && i < 64) RTRACE(110 + i);
      const uint32_t sbase = stage0 + s * Ly.stage_bytes;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint64_t l0, l1, l2, l3;
        lds_v2x64(sbase + lam_off[2 * c], l0, l1);
        lds_v2x64(sbase + lam_off[2 * c + 1], l2, l3);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t xaddr = sbase + x_off[c] + h * half * 128;   // row R + (RT / 2) h
          const uint4 v = lds128(xaddr);
          const uint64_t x0 = x2_to_f32x2<kX16>(v.x), x1 = x2_to_f32x2<kX16>(v.y);
          const uint64_t x2 = x2_to_f32x2<kX16>(v.z), x3 = x2_to_f32x2<kX16>(v.w);
          if constexpr (kX16) {
            // fp16 X -> hi = bf16(x) (in place) + lo = bf16(x - hi) (the lo tile): both exact, so the
            // bf16 x bf16 MMAs reproduce X . L1s^T (kind::f16 takes one A/B type)
            uint32_t hw[4], lw[4];
            const uint64_t xs4[4] = {x0, x1, x2, x3};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float a = lo32(xs4[t]), b = hi32(xs4[t]);
              const uint32_t hb = pack_bf16x2(a, b);
              hw[t] = hb;
              lw[t] = pack_bf16x2(a - __uint_as_float(hb << 16), b - __uint_as_float(hb & 0xFFFF0000u));
            }
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(xaddr), "r"(hw[0]), "r"(hw[1]), "r"(hw[2]),
                         "r"(hw[3]) : "memory");
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(xaddr + 16384), "r"(lw[0]), "r"(lw[1]),
                         "r"(lw[2]), "r"(lw[3]) : "memory");
          }
          xh[h][4 * c + 0] = fmul2(x0, l0);
          xh[h][4 * c + 1] = fmul2(x1, l1);
          xh[h][4 * c + 2] = fmul2(x2, l2);
          xh[h][4 * c + 3] = fmul2(x3, l3);
        }
      }
      if constexpr (kX16) {
        fence_proxy_async();                                    // generic smem writes -> tcgen05 reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);                   // tile consumed: values in registers
    };
    // Group absmax -> scale -> codes of row half h, stored at stage i's place (App. B recipe, bit-exact).
    auto quant_store = [&](int i, int h, const uint64_t (&xh)[8]) {
      const bool active = i * Q + qb < nkb;                     // this lane's block exists (last stage)
      float am[8];                                              // |x_hat| max as a tree (short chain)
#pragma unroll
      for (int j = 0; j < 8; ++j) am[j] = fmaxf(fabsf(lo32(xh[j])), fabsf(hi32(xh[j])));
      float amax = fmaxf(fmaxf(fmaxf(am[0], am[1]), fmaxf(am[2], am[3])), fmaxf(fmaxf(am[4], am[5]), fmaxf(am[6], am[7])));
      const int64_t step = static_cast<int64_t>(i) * Q;         // K blocks before this stage
      if constexpr (kFmt == 0) {
        const uint32_t sf = e4m3_rn_sat(__fmul_rn(amax, t6));
        float qinv;
        if (SVDQ_K1REXP & 32) qinv = __uint_as_float(0x3C000000u + (sf << 20));   // ablation: no LUT
        else asm("ld.shared.f32 %0, [%1];" : "=f"(qinv) : "r"(lut + sf * 4));
        const uint64_t q2 = pack64(__float_as_uint(qinv), __float_as_uint(qinv));
        const uint32_t w0 = e2m1x8_pairs(fmul2(xh[0], q2), fmul2(xh[1], q2), fmul2(xh[2], q2), fmul2(xh[3], q2));
        const uint32_t w1 = e2m1x8_pairs(fmul2(xh[4], q2), fmul2(xh[5], q2), fmul2(xh[6], q2), fmul2(xh[7], q2));
        if (SVDQ_K1REXP & 16) {                                 // ablation: no global stores
          if ((w0 ^ w1 ^ sf) == 0x12345u) p.xq[0] = 1;
          return;
        }
        if (active && mh[h] < RT) {
          uint8_t *xq = xq_base[h] + step * 32;
          uint8_t *sfp = sf_base[h] + step * 512;
          if (rvalid[h]) *reinterpret_cast<uint2 *>(xq + d0) = make_uint2(w0, w1);
          sfp[d0] = static_cast<uint8_t>(sf);                   // padding rows (>= M) get 0x00
          for (int j = 1; j < ndst; ++j) {                      // the other ranks of a fused gather
            const int64_t d = p.dst_delta[j];
            if (rvalid[h]) *reinterpret_cast<uint2 *>(xq + d) = make_uint2(w0, w1);
            sfp[d] = static_cast<uint8_t>(sf);
          }
        }
      } else {
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
        const uint16_t sc = scale16_rn_sat<kScaleBf16>(__fdiv_rn(amax, 7.0f));
        const float sd = scale16_to_f32<kScaleBf16>(sc);
        const float qinv = sd == 0.f ? 0.f : __frcp_rn(sd);
        const uint64_t q2 = pack64(__float_as_uint(qinv), __float_as_uint(qinv));
        uint32_t w[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t word = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t t = fmul2(xh[4 * c + j], q2);
            const int v0 = max(-7, min(7, __float2int_rn(lo32(t))));
            const int v1 = max(-7, min(7, __float2int_rn(hi32(t))));
            word |= ((static_cast<uint32_t>(v0) & 0xFu) | ((static_cast<uint32_t>(v1) & 0xFu) << 4)) << (8 * j);
          }
          w[c] = word;
        }
        if (rvalid[h] && active) {
          uint8_t *xq = xq_base[h] + step * 32;
          uint8_t *s16 = s16_base[h] + step * 2;
          for (int j = 0; j < ndst; ++j) {
            const int64_t d = p.dst_delta[j];
            *reinterpret_cast<uint2 *>(xq + d) = make_uint2(w[0], w[1]);
            if (q4 == 0) *reinterpret_cast<uint16_t *>(s16 + d) = sc;
          }
        }
      }
    };

    {
      float w8max[2] = {0.f, 0.f};                              // W8A8: running amax |x_hat| of both rows
      for (int i = team; i < nsteps; i += 2) {
        uint64_t xh[2][8];
        load_stage(i, xh);
        if (kFmt == 2) {                                        // W8A8: amax for the INT8 kernel (+ fp16 conversion)
          if (i * Q + qb < nkb) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                w8max[h] = fmaxf(w8max[h], fmaxf(fabsf(lo32(xh[h][j])), fabsf(hi32(xh[h][j]))));
          }
          continue;
        }
        if (SVDQ_K1REXP & 1) {
          if (xh[0][0] == 12345ull || xh[1][0] == 12345ull) p.xq[0] = 1;   // keep the loads alive
          continue;
        }
        quant_store(i, 0, xh[0]);
        quant_store(i, 1, xh[1]);
        if (lane == 0 && (i >> 1) == (nsteps >> 2)) RTRACE(420 + qw);
      }
      if (kFmt == 2) {                                          // combine the 4 groups of a row, then the CTA
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float v = w8max[h];
          v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
          v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
          if (q4 == 0) atomicMax(&rowmax[mh[h]], __float_as_uint(v));   // non-negative: bit order = value order
        }
      }
    }
  }

  if (threadIdx.x == 32 * kQ0) RTRACE(100);                    // quantizer 0 done
  if (warp >= kQ0 && lane == 0) RTRACE(400 + warp - kQ0);
  if (r == 0) return;
  // ---------------------------------------------------------------------- xl1 = sum_q diag blocks
  // Block-major stage: TMEM lane d = q RT + m holds row m's partial over the K blocks of index q in
  // columns [q r, q r + r) (the diagonal block).  A warp's 32 lanes span 32 / RT blocks (one when
  // RT >= 32), so it reads only those columns -- a quarter of the Q r-column accumulator at Q = 4
  // (TMEM reads run at 64 B / clk: reading all of it cost ~1 us per launch).  The 16 quantizer warps
  // split xl1's r columns into 8-column chunks (4 warps per lane quadrant, chunks qq, qq + 4, ...),
  // park the partials in the (now idle) ring as part[q][m][r + 4], and after a barrier of the
  // quantizer warps each (row, chunk) is summed over q in the fixed pairwise order
  // ((p0 + p1) + (p2 + p3) at Q = 4: deterministic, and the order of the former warp butterfly).
  __syncthreads();
  if (threadIdx.x == 32 * kQ0) { RTRACE(102); CTRACE(500); }
  if (kFmt == 2 && threadIdx.x < RT && row0 + threadIdx.x < p.M)   // every row's amax -> xs (fp32)
    reinterpret_cast<float *>(p.xs)[row0 + threadIdx.x] = __uint_as_float(rowmax[threadIdx.x]);
  if (warp >= kQ0) {
    const int qd = warp & 3;                                   // TMEM lane quadrant of this warp
    const int qq = (warp - kQ0) >> 2;                          // 0..3 within the quadrant
    const int d = 32 * qd + lane;                              // D row = q RT + m
    const int q = d / RT, m = d % RT;
    const int nc8 = r / 8;
    const int pst = r + 4;                                     // part row stride (floats), padded
    float *part = reinterpret_cast<float *>(smem);
    if (qq < nc8) {
      q_wait(dfull, 0);
      tc_fence_after();
    }
    if (threadIdx.x == 32 * kQ0) { RTRACE(103); CTRACE(501); }
    const int qa = (32 * qd) / RT;                             // first block in this quadrant
    const int nbq = RT >= 32 ? 1 : 32 / RT;                    // blocks in this quadrant (2 at RT = 16)
    for (int c8 = qq; c8 < ((SVDQ_K1REXP & 64) ? 0 : nc8); c8 += 4) {   // 64: ablation, no drain
      uint32_t v[2][8];
      tmem_ld_32x32b_x8(tmem + (static_cast<uint32_t>(32 * qd) << 16) + qa * r + 8 * c8, v[0]);
      if (nbq > 1) tmem_ld_32x32b_x8(tmem + (static_cast<uint32_t>(32 * qd) << 16) + (qa + 1) * r + 8 * c8, v[1]);
      tmem_ld_wait();
      if (threadIdx.x == 32 * kQ0) CTRACE(503);
      const int u = q - qa;
      float *dst = part + (static_cast<int64_t>(q) * RT + m) * pst + 8 * c8;
      if (u == 0) {
        reinterpret_cast<float4 *>(dst)[0] = make_float4(__uint_as_float(v[0][0]), __uint_as_float(v[0][1]),
                                                         __uint_as_float(v[0][2]), __uint_as_float(v[0][3]));
        reinterpret_cast<float4 *>(dst)[1] = make_float4(__uint_as_float(v[0][4]), __uint_as_float(v[0][5]),
                                                         __uint_as_float(v[0][6]), __uint_as_float(v[0][7]));
      } else {
        reinterpret_cast<float4 *>(dst)[0] = make_float4(__uint_as_float(v[1][0]), __uint_as_float(v[1][1]),
                                                         __uint_as_float(v[1][2]), __uint_as_float(v[1][3]));
        reinterpret_cast<float4 *>(dst)[1] = make_float4(__uint_as_float(v[1][4]), __uint_as_float(v[1][5]),
                                                         __uint_as_float(v[1][6]), __uint_as_float(v[1][7]));
      }
    }
    named_bar_sync(1, 32 * kQuantWarps);                      // every partial parked
    // (row m, chunk c8) items over the 512 quantizer threads
    for (int it = threadIdx.x - 32 * kQ0; it < ((SVDQ_K1REXP & 64) ? 0 : RT * nc8); it += 32 * kQuantWarps) {
      const int mm = it / nc8, c8 = it % nc8;
      const int64_t row = row0 + mm;
      if (row >= tailp[2]) continue;
      float pv[8][8];                                          // [q][j], Q <= 8
#pragma unroll
      for (int qv = 0; qv < 8; ++qv) {
        if (qv < Q) {
          const float4 *src = reinterpret_cast<const float4 *>(part + (static_cast<int64_t>(qv) * RT + mm) * pst + 8 * c8);
          const float4 a0 = src[0], a1 = src[1];
          pv[qv][0] = a0.x; pv[qv][1] = a0.y; pv[qv][2] = a0.z; pv[qv][3] = a0.w;
          pv[qv][4] = a1.x; pv[qv][5] = a1.y; pv[qv][6] = a1.z; pv[qv][7] = a1.w;
        }
      }
      float val[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {                            // pairwise tree over q
        float t0 = pv[0][j];
        if (Q == 2) t0 = pv[0][j] + pv[1][j];
        else if (Q == 4) t0 = (pv[0][j] + pv[1][j]) + (pv[2][j] + pv[3][j]);
        else if (Q == 8) t0 = ((pv[0][j] + pv[1][j]) + (pv[2][j] + pv[3][j])) + ((pv[4][j] + pv[5][j]) + (pv[6][j] + pv[7][j]));
        val[j] = t0;
      }
      const int64_t c = row * r + 8 * c8;
      if (tailp[1] && !(SVDQ_K1REXP & 512)) {
        for (int j = 0; j < p.ndst; ++j) {
          float4 *o = reinterpret_cast<float4 *>(reinterpret_cast<uint8_t *>(reinterpret_cast<float *>(tailp[1]) + c) +
                                                 p.dst_delta[j]);
          o[0] = make_float4(val[0], val[1], val[2], val[3]);
          o[1] = make_float4(val[4], val[5], val[6], val[7]);
        }
      } else if (!(SVDQ_K1REXP & 512)) {
        *reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(tailp[0]) + c) = make_uint4(
            pack_bf16x2(val[0], val[1]), pack_bf16x2(val[2], val[3]), pack_bf16x2(val[4], val[5]),
            pack_bf16x2(val[6], val[7]));
      }
    }
  }
  if (threadIdx.x == 32 * kQ0) { RTRACE(104); CTRACE(502); }
  tc_fence_before();
  __syncthreads();                                             // every tcgen05.ld is done
  if (warp == 1) tmem_dealloc_n(tmem, tcols);
  if (threadIdx.x == 32 * kQ0) RTRACE(101);
}

template <int kFmt, bool kScaleBf16, bool kX16>
cudaError_t launch_t(K1Args &g, const K1RowLayout &Ly, cudaStream_t s) {
  auto kern = k1_rows_kernel<kFmt, kScaleBf16, kX16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Ly.smem));
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3(static_cast<unsigned>(g.tile_begin[g.n])), dim3(kThreads, 1, 1), Ly.smem, s, 1u, g, Ly);
}

}  // namespace

int k1_rows_rt(int64_t rows_total, int rank) {
  // smallest row tile (most CTAs) whose tile count still fits one wave; Q * rank <= 256 (MMA N)
  const int sms = device_sm_count();
  int rt = 128;
  for (int cand = 64; cand >= 16; cand /= 2) {
    if ((128 / cand) * rank > 256) break;
    if (rows_total / cand > sms) break;
    rt = cand;
  }
  return rt;
}

cudaError_t launch_k1_rows_group(K1Args &g, int rt, cudaStream_t s) {
  const K1Params &p = g.pr[0].p;
  const K1RowLayout Ly = k1_row_layout(rt, p.rank, !p.x_bf16);
  g.tile_begin[0] = 0;
  for (int i = 0; i < g.n; ++i) g.tile_begin[i + 1] = g.tile_begin[i] + static_cast<int>(g.pr[i].p.Mpad / rt);
  if (p.x_bf16) {
    if (p.fmt == 2) return launch_t<2, true, false>(g, Ly, s);
    if (p.fmt == 0) return launch_t<0, true, false>(g, Ly, s);
    return p.scale_bf16 ? launch_t<1, true, false>(g, Ly, s) : launch_t<1, false, false>(g, Ly, s);
  }
  if (p.fmt == 2) return launch_t<2, true, true>(g, Ly, s);
  if (p.fmt == 0) return launch_t<0, true, true>(g, Ly, s);
  return p.scale_bf16 ? launch_t<1, true, true>(g, Ly, s) : launch_t<1, false, true>(g, Ly, s);
}

}  // namespace svdq
