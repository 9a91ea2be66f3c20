// DRAM-cold streaming floor for K1-sized reads (round 2).  How long does a single kernel take to
// read B bytes of a DRAM-cold buffer, measured INSIDE the kernel (first CTA start -> last CTA end,
// %globaltimer), i.e. without the launch gap?  Readers:
//   bulk : one CTA per SM, contiguous share, cp.async.bulk global->smem in 16 KB chunks with up
//          to `depth` chunks in flight (mbarrier ring), like K1's TMA producer but with no consumer
//   ldg  : 148 x 1024 threads, 8 x LDG.128 in flight per thread
// Buffers are cycled over > 2x L2 so every launch is DRAM-cold.  Also: the same reads launched
// right after a 256 MB streaming kernel (HBM busy before the read starts) to see whether the
// ramp depends on prior HBM activity.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbr tools/mb_ramp.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ unsigned long long g_t0, g_t1;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void reset_times() {
  g_t0 = ~0ull;
  g_t1 = 0;
}

__global__ void __launch_bounds__(128, 1) rd_bulk(const uint8_t *x, int64_t bytes, int depth) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  if (threadIdx.x == 0) atomicMin(&g_t0, gtime());
  const int64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 16383) / 16384 * 16384;
  const int64_t b = blockIdx.x * per, e = b + per < bytes ? b + per : bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < depth; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    const int64_t n = (e - b + 16383) / 16384;
    for (int64_t i = 0; i < n + depth; ++i) {
      if (i >= depth) {                       // wait for chunk i - depth
        const int s = (i - depth) % depth;
        const uint32_t ph = ((i - depth) / depth) & 1;
        asm volatile(
            "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
                smem_u32(&bar[s])),
            "r"(ph));
      }
      if (i < n) {
        const int s = i % depth;
        const int64_t off = b + i * 16384;
        const uint32_t sz = static_cast<uint32_t>(e - off < 16384 ? e - off : 16384);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(sz));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + s * 16384)),
                     "l"(x + off), "r"(sz), "r"(smem_u32(&bar[s]))
                     : "memory");
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t1, gtime());
}

__global__ void __launch_bounds__(1024) rd_ldg(const uint4 *x, int64_t n16, unsigned long long *sink) {
  if (threadIdx.x == 0) atomicMin(&g_t0, gtime());
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = i + j * stride < n16 ? x[i + j * stride] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t1, gtime());
}

__global__ void busy(const uint4 *x, int64_t n16, unsigned long long *sink) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc ^= x[i].y;
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const int64_t L2 = 128ll << 20;
  uint8_t *pool;
  const int64_t pool_bytes = 1536ll << 20;
  cudaMalloc(&pool, pool_bytes);
  cudaMemset(pool, 1, pool_bytes);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t sizes[] = {8ll << 20, 16ll << 20, 25ll << 20, 37ll << 20, 64ll << 20, 141ll << 20};
  for (int mode = 0; mode < 5; ++mode) {
    for (int64_t B : sizes) {
      const int NB = static_cast<int>((3 * L2) / B) + 2;
      if (NB * B > pool_bytes - (256ll << 20)) continue;
      const int reps = 24;
      double span = 0, ev = 0;
      for (int rep = 0; rep < reps + 4; ++rep) {
        const uint8_t *p = pool + (rep % NB) * B;
        if (mode >= 3)   // HBM busy right before the read: 256 MB stream from the pool's tail
          busy<<<148 * 4, 512>>>(reinterpret_cast<const uint4 *>(pool + pool_bytes - (256ll << 20)),
                                 (256ll << 20) / 16, sink);
        reset_times<<<1, 1>>>();
        cudaEventRecord(a);
        if (mode == 0 || mode == 3) rd_bulk<<<148, 128, 6 * 16384>>>(p, B, 6);
        else if (mode == 1 || mode == 4) rd_bulk<<<148, 128, 12 * 16384>>>(p, B, 12);
        else rd_ldg<<<148, 1024>>>(reinterpret_cast<const uint4 *>(p), B / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        unsigned long long t0, t1;
        cudaMemcpyFromSymbol(&t0, g_t0, 8);
        cudaMemcpyFromSymbol(&t1, g_t1, 8);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep >= 4) {
          span += (t1 - t0) / 1e3;
          ev += ms * 1e3;
        }
      }
      span /= reps;
      ev /= reps;
      const char *nm[] = {"bulk depth 6", "bulk depth 12", "ldg 8x16B", "busy + bulk depth 6", "busy + bulk depth 12"};
      printf("%-22s %6.1f MB: in-kernel %7.2f us (%5.2f TB/s)   event %7.2f us (%5.2f TB/s)  %s\n", nm[mode],
             B / 1048576.0, span, B / span / 1e6, ev, B / ev / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
