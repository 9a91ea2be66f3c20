// K1 for the 8-bit setting (SVDQ_FMT_W8A8; App. D): per-token dynamic INT8 codes of
// x_hat = fl32(x * lambda_inv) (reading Q14) with Eq. (1), q_max = 127 and one fp32 scale
// per token.  A per-token scale needs the whole row before any code can be written: the
// row-tile kernel's down-projection pass (which reads X anyway) leaves amax(|x_hat|) per row in
// xs (`w8_amax`), so this kernel encodes in one pass; without a low-rank branch (rank 0) it
// takes amax itself first (pass 1, then pass 2 served from L1 / L2).  The down-projection X L1s^T of the same layer runs in the regular K1 kernel in
// its projection-only mode (fmt 2), so the 16-bit branch is bit-identical across formats.
//   s = fl32(amax / 127); qinv = s == 0 ? 0 : fl32(1 / s); q = clamp(rne(fl32(x_hat * qinv)), +-127)
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "k1_launch.h"
#include "sm100.cuh"

namespace svdq {
namespace {

template <bool kBf16>
__device__ __forceinline__ float h2f(uint32_t bits16) {
  if constexpr (kBf16) return __uint_as_float(bits16 << 16);
  else return __half2float(__ushort_as_half(static_cast<uint16_t>(bits16)));
}

// One warp per row; lane l owns elements [8l + 256 j, +8) of chunk j.
template <bool kBf16>
__global__ void __launch_bounds__(256) k1_int8_rows_kernel(const K1Params p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  griddep_launch_dependents();
  griddep_wait();                                   // X may be the previous kernel's output
  if (row >= p.M) return;
  const uint16_t *x = static_cast<const uint16_t *>(p.X) + row * p.ldx;
  const int64_t K = p.K;
  float amax = 0.f;
  if (p.w8_amax) amax = reinterpret_cast<const float *>(p.xs)[row];   // from the down-projection pass
  else
  for (int64_t k = 8 * lane; k < K; k += 256) {
    const uint4 v = *reinterpret_cast<const uint4 *>(x + k);
    const float4 l0 = *reinterpret_cast<const float4 *>(p.lam_inv + k);
    const float4 l1 = *reinterpret_cast<const float4 *>(p.lam_inv + k + 4);
    const float lam[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      amax = fmaxf(amax, fabsf(__fmul_rn(h2f<kBf16>(w[j] & 0xFFFFu), lam[2 * j])));
      amax = fmaxf(amax, fabsf(__fmul_rn(h2f<kBf16>(w[j] >> 16), lam[2 * j + 1])));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float sc = __fdiv_rn(amax, 127.0f);
  const float qinv = sc == 0.f ? 0.f : __fdiv_rn(1.0f, sc);
  if (lane == 0) reinterpret_cast<float *>(p.xs)[row] = sc;
  int8_t *q = reinterpret_cast<int8_t *>(p.xq) + row * K;
  for (int64_t k = 8 * lane; k < K; k += 256) {
    const uint4 v = *reinterpret_cast<const uint4 *>(x + k);
    const float4 l0 = *reinterpret_cast<const float4 *>(p.lam_inv + k);
    const float4 l1 = *reinterpret_cast<const float4 *>(p.lam_inv + k + 4);
    const float lam[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t out[2] = {0u, 0u};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float xh = __fmul_rn(h2f<kBf16>(h ? (w[j] >> 16) : (w[j] & 0xFFFFu)), lam[2 * j + h]);
        const int c = max(-127, min(127, __float2int_rn(__fmul_rn(xh, qinv))));
        const int e = 2 * j + h;
        out[e >> 2] |= (static_cast<uint32_t>(c) & 0xFFu) << (8 * (e & 3));
      }
    }
    *reinterpret_cast<uint2 *>(q + k) = make_uint2(out[0], out[1]);
  }
}

}  // namespace

cudaError_t launch_k1_int8_rows(const K1Params &p, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((p.M + 7) / 8);
  return p.x_bf16 ? launch_ex(k1_int8_rows_kernel<true>, dim3(grid), dim3(256), 0, s, 1u, p)
                  : launch_ex(k1_int8_rows_kernel<false>, dim3(grid), dim3(256), 0, s, 1u, p);
}

}  // namespace svdq
