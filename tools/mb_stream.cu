// Microbenchmark: how fast can one CTA per SM stream a row-major bf16 matrix
// [M][K] (the K1 access pattern) into shared memory?
//   mode 0: TMA 2D box {64, 128} SW128 (K1 today), ring of S stages, 1 consumer warp
//   mode 1: TMA 2D box {64, 256} SW128
//   mode 2: TMA 3D box {64, 128, 4} SW128 (4 k-chunks per request batch)
//   mode 3: LDG.128 by 16 warps, each lane 4 x 16 B per iteration (no smem)
// Each CTA handles 128 rows x (K / ks) columns like K1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb tools/mb_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_2411_05007_b200/csrc/sm100.cuh"

using namespace svdq;

template <int MODE, int TMEM, int EXTRA>
__global__ void __launch_bounds__(576, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tl, const float *lam, const uint16_t *X,
                                                         int64_t M, int64_t K, int ks, int S, unsigned long long *sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = MODE == 1 ? 32768 : (MODE == 2 ? 65536 : (EXTRA ? 21504 : 16384));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * stage_bytes);
  uint64_t *empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = static_cast<int>(K / 64);
  const int crank = blockIdx.x;
  const int kb_begin = crank * nkb / ks;
  const int nkb_here = (crank + 1) * nkb / ks - kb_begin;
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * 128;
  unsigned long long acc = 0;
  if (MODE == 3) {
    // 16 warps x 8 rows: lane (g = row, q = 16-B chunk of a 64-element block), 2 blocks per iter
    if (warp >= 2) {
      const int qw = warp - 2, g = lane >> 2, q = lane & 3;
      const int64_t row = row0 + qw * 8 + g;
      for (int kb = kb_begin; kb < kb_begin + nkb_here; ++kb) {
        const uint16_t *p = X + row * K + kb * 64 + q * 8;
        uint4 a = *reinterpret_cast<const uint4 *>(p);
        uint4 b = *reinterpret_cast<const uint4 *>(p + 32);
        acc += a.x ^ b.y;
        if (kb + 1 < kb_begin + nkb_here) {   // unroll x4 with all loads first
          uint4 c0 = *reinterpret_cast<const uint4 *>(p + 64), c1 = *reinterpret_cast<const uint4 *>(p + 96);
          ++kb;
          acc += c0.z ^ c1.w;
        }
      }
    }
    if (acc == 12345) sink[0] = acc;
    return;
  }
  const int steps = MODE == 2 ? nkb_here / 4 : (MODE == 1 ? nkb_here : nkb_here);
  const int rows_per = MODE == 1 ? 256 : 128;
  if (MODE == 1 && (blockIdx.y & 1)) return;   // 256-row tiles: odd row tiles idle
  uint32_t *tslot = reinterpret_cast<uint32_t *>(empty + 16);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], EXTRA >= 4 ? 16 : 1); }
    fence_mbar_init();
  }
  if (TMEM && warp == 1) tmem_alloc<32>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], EXTRA == 1 ? 16384 + 4096 + 256 : (EXTRA == 2 ? 16384 + 4096 : (EXTRA == 3 ? 16384 + 256 : 16384)));
      uint8_t *st = smem + s * stage_bytes;
      if (EXTRA == 1 || EXTRA == 2) tma_load_2d(st + 16384, &tl, &full[s], (kb_begin + i) * 64, 0);
      if (EXTRA == 1 || EXTRA == 3) bulk_load(st + 16384 + 4096, lam + (kb_begin + i) * 64, 256, &full[s]);
      if (MODE == 2) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(st)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&full[s])), "r"(0), "r"((int)row0),
            "r"(kb_begin + 4 * i)
            : "memory");
      } else {
        tma_load_2d(st, &tm, &full[s], (kb_begin + i) * 64, (int)row0);
      }
    }
  } else if (EXTRA >= 4 && warp >= 2) {
    const int qw = warp - 2, g = lane >> 2, q = lane & 3, rl = qw * 8 + g;
    uint8_t *dst = reinterpret_cast<uint8_t *>(sink) + 64 + (static_cast<int64_t>(blockIdx.y) * 128 + rl) * (K / 2);
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      const uint8_t *st = smem + s * stage_bytes + rl * 128;
      uint4 a = *reinterpret_cast<const uint4 *>(st + ((q ^ (rl & 7)) * 16));
      uint4 b = *reinterpret_cast<const uint4 *>(st + (((q + 4) ^ (rl & 7)) * 16));
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      uint32_t v = a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
      if (EXTRA == 5) *reinterpret_cast<uint32_t *>(dst + (kb_begin + i) * 32 + q * 4) = v;
      else acc += v;
    }
    if (acc == 12345) sink[0] = acc;
  } else if (EXTRA < 4 && warp == 1 && lane == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      acc += smem[s * stage_bytes + 7];
      mbar_arrive(&empty[s]);
    }
    if (acc == 12345) sink[0] = acc;
  }
  (void)rows_per;
  if (TMEM) {
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<32>(*tslot);
  }
}

__global__ void __launch_bounds__(64, 1) gen_kernel(const __grid_constant__ CUtensorMap tm, int64_t K, int ks, int S,
                                                    int inner, int rows, int stage, unsigned long long *sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * stage);
  uint64_t *empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = static_cast<int>(K / inner);
  const int c0 = blockIdx.x * nch / ks, steps = (blockIdx.x + 1) * nch / ks - c0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  unsigned long long acc = 0;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], stage);
      tma_load_2d(smem + s * stage, &tm, &full[s], (c0 + i) * inner, blockIdx.y * rows);
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      acc += smem[s * stage + 7];
      mbar_arrive(&empty[s]);
    }
    if (acc == 12345) sink[0] = acc;
  }
}

int main(int argc, char **argv) {
  const int64_t M = argc > 1 ? atoll(argv[1]) : 4096, K = argc > 2 ? atoll(argv[2]) : 3072;
  uint16_t *X;
  cudaMalloc(&X, M * K * 2);
  cudaMemset(X, 1, M * K * 2);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    cuuint64_t str[1] = {(cuuint64_t)(K * 2)};
    cuuint32_t box[2] = {64, 128u}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  uint16_t *L1;
  cudaMalloc(&L1, 32 * K * 2);
  float *lam;
  cudaMalloc(&lam, K * 4);
  CUtensorMap tl;
  memset(&tl, 0, sizeof(tl));
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, 32};
    cuuint64_t str[1] = {(cuuint64_t)(K * 2)};
    cuuint32_t box[2] = {64, 32u}, es[2] = {1, 1};
    enc(&tl, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, L1, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFree(sink);
  cudaMalloc(&sink, M * K + 4096);
  const int NB = M * K * 2 > (200ll << 20) ? 3 : 16;        // distinct inputs, total > L2 (cold)
  uint16_t *Xs;
  cudaMalloc(&Xs, (size_t)NB * M * K * 2);
  cudaMemset(Xs, 1, (size_t)NB * M * K * 2);
  CUtensorMap tms[NB];
  for (int i = 0; i < NB; ++i) {
    memset(&tms[i], 0, sizeof(CUtensorMap));
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    cuuint64_t str[1] = {(cuuint64_t)(K * 2)};
    cuuint32_t box[2] = {64, 128u}, es[2] = {1, 1};
    enc(&tms[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Xs + (size_t)i * M * K, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  // CTAs per SM / grid variants, all cold (16 distinct inputs), box 64x128 SW128
  {
    CUtensorMap maps[NB];
    for (int i = 0; i < NB; ++i) {
      memset(&maps[i], 0, sizeof(CUtensorMap));
      cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
      cuuint64_t str[1] = {(cuuint64_t)(K * 2)};
      cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
      enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Xs + (size_t)i * M * K, dims, str, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    struct G { int ks; int S; };
    G gs[] = {{3, 6}, {4, 6}, {4, 3}, {8, 3}};
    for (auto &gv : gs) {
      size_t smem = (size_t)gv.S * 16384 + 2048;
      auto k = gen_kernel;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 64, smem);
      dim3 grid(gv.ks, M / 128);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) k<<<grid, 64, smem>>>(maps[w], K, gv.ks, gv.S, 64, 128, 16384, sink);
      cudaEventRecord(a);
      for (int w = 0; w < 2 * NB; ++w) k<<<grid, 64, smem>>>(maps[w % NB], K, gv.ks, gv.S, 64, 128, 16384, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("ks %2d stages %d ctas %4d (occ/SM %d): cold %.2f us  %.2f TB/s  %s\n", gv.ks, gv.S, gv.ks * (int)(M / 128), occ,
             1e3 * ms / (2 * NB), M * K * 2 / (ms / (2 * NB) * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // LDG cold
  {
    dim3 grid(4, M / 128);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int w = 0; w < 2 * NB; ++w)
      stream_kernel<3, 0, 0><<<grid, 576>>>(tm, tm, nullptr, Xs + (size_t)(w % NB) * M * K, M, K, 4, 4, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-20s: cold %.2f us  %.2f TB/s\n", "LDG 16 warps", 1e3 * ms / (2 * NB), M * K * 2 / (ms / (2 * NB) * 1e-3) / 1e12);
  }
  return 0;
}
