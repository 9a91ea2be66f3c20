// DRAM read-pattern microbenchmark (cold: cycles over > 2x L2 of distinct buffers).
// Which read pattern can K1 hope for?  Every pattern reads the same bytes of a
// [M][K] bf16 matrix; grid = 148 CTAs x 512 threads (one per SM), LDG.128, 4 in flight
// per thread per iteration.
//   A: contiguous: CTA c reads bytes [c*B/148, (c+1)*B/148)
//   B: row bands: CTA reads whole rows (rows c*M/148 ..)
//   C: K1 tiles: CTA (tile, ks) reads 128 rows x (K/ks) columns, 128 B per row per step
//   D: TMA-like: 128 rows x 128 B box per step but all 16 warps read one box each (row-strided)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbd tools/mb_dram.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) rd_contig(const uint4 *x, int64_t n16, unsigned long long *sink) {
  const int64_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const int64_t b = blockIdx.x * per, e = min(n16, b + per);
  uint32_t acc = 0;
  for (int64_t i = b + threadIdx.x; i < e; i += 4 * blockDim.x) {
    uint4 v0 = x[i];
    uint4 v1 = i + blockDim.x < e ? x[i + blockDim.x] : make_uint4(0, 0, 0, 0);
    uint4 v2 = i + 2 * blockDim.x < e ? x[i + 2 * blockDim.x] : make_uint4(0, 0, 0, 0);
    uint4 v3 = i + 3 * blockDim.x < e ? x[i + 3 * blockDim.x] : make_uint4(0, 0, 0, 0);
    acc ^= v0.x ^ v1.y ^ v2.z ^ v3.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// C: CTA = (kslice, rowtile): 128 rows x (K/ks) cols; each step reads a 128 x 64-col box
// (128 B per row); 512 threads: thread t reads row t/4, 16 B chunk t%4 of 4 steps at once.
__global__ void __launch_bounds__(512) rd_tiles(const uint8_t *x, int64_t M, int64_t K, int ks,
                                                unsigned long long *sink) {
  const int64_t ldb = K * 2;
  const int kb_total = static_cast<int>(K / 64);
  const int crank = blockIdx.x % ks;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x / ks) * 128;
  const int kb0 = crank * kb_total / ks, kb1 = (crank + 1) * kb_total / ks;
  const int r = threadIdx.x >> 2, c = threadIdx.x & 3;
  uint32_t acc = 0;
  if (row0 + r >= M) return;
  const uint8_t *rp = x + (row0 + r) * ldb + c * 32;
  for (int kb = kb0; kb < kb1; kb += 4) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = kb + j < kb1 ? kb + j : kb;
      v[2 * j] = *reinterpret_cast<const uint4 *>(rp + k * 128);
      v[2 * j + 1] = *reinterpret_cast<const uint4 *>(rp + k * 128 + 16);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// B: row bands, each warp reads whole rows (512 B per warp instruction)
__global__ void __launch_bounds__(512) rd_rows(const uint4 *x, int64_t M, int64_t K, unsigned long long *sink) {
  const int64_t r16 = K * 2 / 16;                  // uint4 per row
  const int64_t rows_per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t rb = blockIdx.x * rows_per, re = min(M, rb + rows_per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t acc = 0;
  for (int64_t row = rb + warp; row < re; row += 16) {
    const uint4 *p = x + row * r16;
    for (int64_t i = lane; i < r16; i += 128) {
      uint4 v0 = p[i];
      uint4 v1 = i + 32 < r16 ? p[i + 32] : make_uint4(0, 0, 0, 0);
      uint4 v2 = i + 64 < r16 ? p[i + 64] : make_uint4(0, 0, 0, 0);
      uint4 v3 = i + 96 < r16 ? p[i + 96] : make_uint4(0, 0, 0, 0);
      acc ^= v0.x ^ v1.y ^ v2.z ^ v3.w;
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char **argv) {
  const int64_t M = argc > 1 ? atoll(argv[1]) : 4096, K = argc > 2 ? atoll(argv[2]) : 3072;
  const int64_t bytes = M * K * 2;
  const int NB = static_cast<int>((600ll << 20) / bytes) + 2;
  uint8_t *buf;
  cudaMalloc(&buf, bytes * NB);
  cudaMemset(buf, 1, bytes * NB);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char *name, auto launch) {
    for (int w = 0; w < NB; ++w) launch(buf + (w % NB) * bytes);
    cudaEventRecord(a);
    const int reps = 3 * NB;
    for (int w = 0; w < reps; ++w) launch(buf + (w % NB) * bytes);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = 1e3 * ms / reps;
    printf("%-34s M=%lld K=%lld: %7.2f us  %5.2f TB/s  %s\n", name, (long long)M, (long long)K, us, bytes / us / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  int nsm = 148;
  run("A contiguous 148 CTAs", [&](uint8_t *p) { rd_contig<<<nsm, 512>>>((const uint4 *)p, bytes / 16, sink); });
  run("A contiguous 296 CTAs", [&](uint8_t *p) { rd_contig<<<2 * nsm, 512>>>((const uint4 *)p, bytes / 16, sink); });
  run("B row bands 148 CTAs", [&](uint8_t *p) { rd_rows<<<nsm, 512>>>((const uint4 *)p, M, K, sink); });
  for (int ks : {1, 2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "C K1 tiles 128 rows, ks=%d (%lld CTAs)", ks, (long long)(M / 128 * ks));
    run(nm, [&](uint8_t *p) { rd_tiles<<<static_cast<unsigned>(M / 128 * ks), 512>>>(p, M, K, ks, sink); });
  }
  return 0;
}
