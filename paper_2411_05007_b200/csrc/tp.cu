// Tensor parallelism, SURVEY 8(e) Variant 2 ("quantize, then gather"): rank p runs K1 of the next
// layer on its own K-slice [p Kp, (p+1) Kp) of the input (its shard of the previous column-parallel
// layer's output) and contributes a packed slice {codes [M][Kp/2] | scales (own layout over Kp) |
// fp32 partial X_p L1s_p^T [M][r]}; one all-gather of the packed slices (0.5625 B per element plus
// the small partials, vs 2 B for a bf16 gather); this kernel assembles the full K1 outputs:
//   xq[m][p Kp/2 + j]           = slice_p.codes[m][j]
//   NVFP4 xs: the 512-B chunk (row tile t, K-block p Kp/64 + c) = slice_p's chunk (t, c)
//   INT4  xs[m][p Kp/64 + j]     = slice_p.scales[m][j]
//   xl1[m][t] = bf16(sum_p part_p[m][t]) summed in rank order (deterministic on every rank).
// Groups never straddle slices because Kp % 64 == 0.
// Fused gather: K1 writes codes / scales straight into every rank's full-K
// buffers (k1_rows.cu multi-destination stores) and its fp32 partial into slot p; after the
// cross-rank barrier only the partial reduction below remains.
#include <cstdint>
#include <cuda_bf16.h>

#include "k1_launch.h"

namespace svdq {

namespace {
constexpr int64_t kAlign = 256;
int64_t up(int64_t b) { return (b + kAlign - 1) / kAlign * kAlign; }

__global__ void tp_assemble_kernel(int fmt, int P, int64_t M, int64_t K, int rank, const uint8_t *__restrict__ g,
                                   int64_t stride, int64_t xs_off, int64_t part_off, uint8_t *__restrict__ xq,
                                   uint8_t *__restrict__ xs, uint16_t *__restrict__ xl1) {
  const int64_t Kp = K / P;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // codes: 16-byte pieces, Kp/32 per (rank, row)
  const int64_t cpr = Kp / 32;
  for (int64_t i = tid; i < P * M * cpr; i += nth) {
    const int64_t p = i / (M * cpr), rem = i % (M * cpr), m = rem / cpr, j = rem % cpr;
    const uint4 v = *reinterpret_cast<const uint4 *>(g + p * stride + m * (Kp / 2) + j * 16);
    *reinterpret_cast<uint4 *>(xq + m * (K / 2) + p * (Kp / 2) + j * 16) = v;
  }
  if (fmt == 0) {
    // 128x4 layout: [tiles][K/64 chunks][512 B]; slice p holds [tiles][Kp/64][512 B]
    const int64_t tiles = (M + 127) / 128, cps = Kp / 64, pieces = 512 / 16;
    for (int64_t i = tid; i < P * tiles * cps * pieces; i += nth) {
      const int64_t p = i / (tiles * cps * pieces), rem = i % (tiles * cps * pieces);
      const int64_t t = rem / (cps * pieces), c = (rem / pieces) % cps, j = rem % pieces;
      const uint4 v = *reinterpret_cast<const uint4 *>(g + p * stride + xs_off + (t * cps + c) * 512 + j * 16);
      *reinterpret_cast<uint4 *>(xs + (t * (K / 64) + p * cps + c) * 512 + j * 16) = v;
    }
  } else {
    const int64_t gp = Kp / 64;                        // 16-bit scales per row of a slice
    for (int64_t i = tid; i < P * M * gp; i += nth) {
      const int64_t p = i / (M * gp), rem = i % (M * gp), m = rem / gp, j = rem % gp;
      const uint16_t v = reinterpret_cast<const uint16_t *>(g + p * stride + xs_off)[m * gp + j];
      reinterpret_cast<uint16_t *>(xs)[m * (K / 64) + p * gp + j] = v;
    }
  }
  for (int64_t i = tid; i < M * rank; i += nth) {
    float s = 0.f;
    for (int p = 0; p < P; ++p)                        // rank order: deterministic
      s += reinterpret_cast<const float *>(g + p * stride + part_off)[i];
    xl1[i] = __bfloat16_as_ushort(__float2bfloat16_rn(s));
  }
}

__global__ void tp_reduce_kernel(int P, int64_t n, const float *__restrict__ parts, uint16_t *__restrict__ xl1) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < P; ++p) s += parts[p * n + i];   // rank order: deterministic
    xl1[i] = __bfloat16_as_ushort(__float2bfloat16_rn(s));
  }
}
}  // namespace

cudaError_t launch_tp_reduce_partials(int P, int64_t M, int rank, const float *parts, uint16_t *xl1, cudaStream_t s) {
  const int64_t n = M * rank;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * device_sm_count()) blocks = 4 * device_sm_count();
  tp_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(P, n, parts, xl1);
  return cudaGetLastError();
}

TpSliceLayout tp_slice_layout(int fmt, int64_t M, int64_t Kp, int rank) {
  TpSliceLayout L;
  L.xq_off = 0;
  L.xs_off = up(M * Kp / 2);
  const int64_t xs_bytes = fmt == 0 ? ((M + 127) / 128) * 128 * (Kp / 16) : M * (Kp / 64) * 2;
  L.part_off = L.xs_off + up(xs_bytes);
  L.bytes = L.part_off + up(M * rank * 4);
  return L;
}

cudaError_t launch_tp_assemble(int fmt, int P, int64_t M, int64_t K, int rank, const uint8_t *gathered,
                               int64_t slice_stride, uint8_t *xq, uint8_t *xs, uint16_t *xl1, cudaStream_t s) {
  const TpSliceLayout L = tp_slice_layout(fmt, M, K / P, rank);
  const int64_t work = M * K / 32;                     // 16-B code pieces dominate
  int64_t blocks = (work + 255) / 256;
  const int64_t cap = static_cast<int64_t>(device_sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  tp_assemble_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(fmt, P, M, K, rank, gathered, slice_stride,
                                                                  L.xs_off, L.part_off, xq, xs, xl1);
  return cudaGetLastError();
}

}  // namespace svdq
