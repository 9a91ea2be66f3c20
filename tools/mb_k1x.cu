// K1 streaming microbenchmark (round 2): the row-tile K1's TMA traffic without its compute.
// 144 CTAs (one per 32-row tile of a [4608 x K] bf16 X), each streams its rows over the full K
// with 3-D TMA boxes {64 cols, Q blocks, RT rows} through a `depth`-stage ring; optional extra
// per-stage loads of Q L1s tiles [32 x 64] bf16 from a small L2-resident buffer.  The consumer
// (one warp) only waits and releases.  In-kernel time by %globaltimer (first CTA start -> last
// CTA end), inputs cycled over > 2x L2 (DRAM-cold).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_k1x tools/mb_k1x.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>

__device__ unsigned long long g_t0, g_t1;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void reset_times() { g_t0 = ~0ull; g_t1 = 0; }

__global__ void __launch_bounds__(64, 1) k1x(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap ml,
                                             const __grid_constant__ CUtensorMap ml3, const uint8_t *l1flat,
                                             int nsteps, int Q, int RT, int depth, int with_l1s, int stage_bytes) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[16], empty[16];
  if (threadIdx.x == 0) atomicMin(&g_t0, gtime());
  if (threadIdx.x == 0) {
    for (int s = 0; s < depth; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int row0 = blockIdx.x * RT;
  if (threadIdx.x == 0) {
    const uint32_t tx = 16384 + (with_l1s ? Q * 32 * 128 : 0);
    for (int i = 0; i < nsteps; ++i) {
      const int s = i % depth;
      if (i >= depth) {
        const uint32_t ph = ((i / depth) & 1) ^ 1;
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
                         su32(&empty[s])), "r"(ph));
      }
      uint8_t *st = sm + s * stage_bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(tx));
      if (with_l1s == 1)
        for (int q = 0; q < Q; ++q)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                           su32(st + 16384 + q * 4096)), "l"(&ml), "r"(su32(&full[s])), "r"(((i * Q + q) * 64) % 1024), "r"(0)
                       : "memory");
      if (with_l1s == 2)         // one contiguous bulk copy of the stage's pre-blocked L1s tiles
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(st + 16384)), "l"(l1flat + ((i * Q) % 16) * 4096), "r"(Q * 4096), "r"(su32(&full[s]))
                     : "memory");
      if (with_l1s == 3)         // one 3-D box {64, Q, 32}
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                         su32(st + 16384)), "l"(&ml3), "r"(su32(&full[s])), "r"(0), "r"((i * Q) % 16), "r"(0)
                     : "memory");
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                       su32(st)), "l"(&mx), "r"(su32(&full[s])), "r"(0), "r"(i * Q), "r"(row0)
                   : "memory");
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < nsteps; ++i) {
      const int s = i % depth;
      const uint32_t ph = (i / depth) & 1;
      asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
                       su32(&full[s])), "r"(ph));
      asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[s])));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t1, gtime());
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&enc), cudaEnableDefault, &q);
  const int64_t M = 4608;
  const int64_t Ks[] = {3072, 15360};
  uint16_t *l1s;
  cudaMalloc(&l1s, 32 * 1024 * 2);
  uint8_t *l1flat;
  cudaMalloc(&l1flat, 32 * 4096 * 2);
  CUtensorMap ml, ml3;
  {
    cuuint64_t dims[3] = {64, 16, 32};
    cuuint64_t str[2] = {128, 2048};
    cuuint32_t box[3] = {64, 4, 32}, es[3] = {1, 1, 1};
    enc(&ml3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, l1s, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[2] = {1024, 32};
    cuuint64_t str[1] = {2048};
    cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
    enc(&ml, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, l1s, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFuncSetAttribute(k1x, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int64_t K : Ks) {
    const int64_t bytes = M * K * 2;
    const int NB = static_cast<int>((400ll << 20) / bytes) + 2;
    uint8_t *pool;
    cudaMalloc(&pool, bytes * NB);
    cudaMemset(pool, 1, bytes * NB);
    struct Cfg { int RT, depth, l1s; };
    const Cfg cfgs[] = {{32, 6, 0}, {32, 6, 1}, {32, 6, 2}, {32, 6, 3}, {32, 8, 0}, {64, 6, 0}};
    for (const Cfg &c : cfgs) {
      const int Q = 128 / c.RT;
      const int nsteps = static_cast<int>((K / 64 + Q - 1) / Q);
      const int stage = c.l1s ? 16384 + Q * 4096 : 16384;
      if (stage * c.depth > 215 * 1024) continue;
      const int grid = static_cast<int>(M / c.RT);
      double span = 0;
      const int reps = 20;
      for (int rep = 0; rep < reps + 3; ++rep) {
        CUtensorMap mx;
        cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(K / 64), static_cast<cuuint64_t>(M)};
        cuuint64_t str[2] = {128, static_cast<cuuint64_t>(K * 2)};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(Q), static_cast<cuuint32_t>(c.RT)}, es[3] = {1, 1, 1};
        enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool + (rep % NB) * bytes, dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        reset_times<<<1, 1>>>();
        k1x<<<grid, 64, stage * c.depth + 1024>>>(mx, ml, ml3, l1flat, nsteps, Q, c.RT, c.depth, c.l1s, stage);
        cudaDeviceSynchronize();
        unsigned long long t0, t1;
        cudaMemcpyFromSymbol(&t0, g_t0, 8);
        cudaMemcpyFromSymbol(&t1, g_t1, 8);
        if (rep >= 3) span += (t1 - t0) / 1e3;
      }
      span /= reps;
      printf("K=%5lld RT=%3d depth=%2d l1s=%d grid=%4d: in-kernel %7.2f us  %5.2f TB/s  %s\n", (long long)K, c.RT,
             c.depth, c.l1s, grid, span, bytes / span / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(pool);
  }
  return 0;
}
