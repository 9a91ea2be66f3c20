// Weight-side (offline) kernels: residual quantization (Eq. 1 per output
// channel, groups along K), smoothing of W, L1s / L2s
// derivation and LoRA concatenation, plus the codec test hook.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "formats.cuh"
#include "k1_launch.h"

namespace svdq {

namespace {

__device__ __forceinline__ float load_any(const void *p, int dt, int64_t i) {
  if (dt == 0) return __bfloat162float(static_cast<const __nv_bfloat16 *>(p)[i]);
  if (dt == 1) return __half2float(static_cast<const __half *>(p)[i]);
  return static_cast<const float *>(p)[i];
}

__device__ __forceinline__ uint16_t bf16_bits_rn(float v) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}

unsigned blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > (1 << 20)) b = 1 << 20;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

__global__ void absmax_kernel(const float *__restrict__ R, int64_t n, unsigned int *out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = fmaxf(m, fabsf(R[i]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// One thread per (output channel n, 16-group g): NVFP4 recipe of App. B.2 with gs = gs_w.
__global__ void quant_res_nvfp4_kernel(const float *__restrict__ R, int64_t K, int64_t N, float gs,
                                       uint8_t *__restrict__ codes, uint8_t *__restrict__ sf) {
  const int64_t G = K / 16;
  const int64_t Npad = ((N + 127) / 128) * 128;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < Npad * G;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = idx / Npad;
    const int64_t n = idx % Npad;          // consecutive threads -> consecutive n (coalesced R reads)
    if (n >= N) {                          // padding rows of the 128x4 layout hold 0x00 (Q22)
      sf[sf_offset(n, g, K)] = 0;
      continue;
    }
    float v[16];
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = R[(g * 16 + i) * N + n];
      amax = fmaxf(amax, fabsf(v[i]));
    }
    const float t6 = __fmul_rn(__fdiv_rn(1.0f, gs), __fdiv_rn(1.0f, 6.0f));
    const uint32_t s = e4m3_rn_sat(__fmul_rn(amax, t6));
    const float sd = e4m3_to_f32(s);
    const float qinv = sd == 0.f ? 0.f : __fdiv_rn(1.0f, __fmul_rn(sd, gs));
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = __fmul_rn(v[i], qinv);
      b[i] = __fmul_rn(v[8 + i], qinv);
    }
    uint2 w;
    w.x = e2m1x8(a);
    w.y = e2m1x8(b);
    *reinterpret_cast<uint2 *>(codes + n * (K / 2) + g * 8) = w;
    sf[sf_offset(n, g, K)] = static_cast<uint8_t>(s);
  }
}

// One thread per (n, 64-group): INT4 recipe of App. B.3.
template <bool kBf16>
__global__ void quant_res_int4_kernel(const float *__restrict__ R, int64_t K, int64_t N,
                                      uint8_t *__restrict__ codes, uint16_t *__restrict__ scales) {
  const int64_t G = K / 64;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < N * G;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = idx / N;
    const int64_t n = idx % N;
    float amax = 0.f;
    for (int i = 0; i < 64; ++i) amax = fmaxf(amax, fabsf(R[(g * 64 + i) * N + n]));
    const uint16_t s = scale16_rn_sat<kBf16>(__fdiv_rn(amax, 7.0f));
    const float sd = scale16_to_f32<kBf16>(s);
    const float qinv = sd == 0.f ? 0.f : __fdiv_rn(1.0f, sd);
    uint32_t words[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int q = __float2int_rn(__fmul_rn(R[(g * 64 + w * 8 + j) * N + n], qinv));
        q = max(-7, min(7, q));
        word |= (static_cast<uint32_t>(q) & 0xFu) << (4 * j);
      }
      words[w] = word;
    }
    uint4 *dst = reinterpret_cast<uint4 *>(codes + n * (K / 2) + g * 32);
    dst[0] = make_uint4(words[0], words[1], words[2], words[3]);
    dst[1] = make_uint4(words[4], words[5], words[6], words[7]);
    scales[n * G + g] = s;
  }
}

// One thread per output channel n: the per-channel INT8 recipe of the 8-bit setting:
// amax over K, s = fl32(amax / 127), qinv = s == 0 ? 0 : fl32(1 / s),
// q = clamp(rne(fl32(r * qinv)), -127, 127).  R is [K][N]: threads n read coalesced rows of R.
__global__ void quant_res_int8_kernel(const float *__restrict__ R, int64_t K, int64_t N, int8_t *__restrict__ codes,
                                      float *__restrict__ scales) {
  const int64_t n = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float amax = 0.f;
  for (int64_t k = 0; k < K; ++k) amax = fmaxf(amax, fabsf(R[k * N + n]));
  const float sc = __fdiv_rn(amax, 127.0f);
  const float qinv = sc == 0.f ? 0.f : __fdiv_rn(1.0f, sc);
  scales[n] = sc;
  for (int64_t k = 0; k < K; k += 16) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int v = max(-127, min(127, __float2int_rn(__fmul_rn(R[(k + 4 * j + b) * N + n], qinv))));
        word |= (static_cast<uint32_t>(v) & 0xFFu) << (8 * b);
      }
      w[j] = word;
    }
    *reinterpret_cast<uint4 *>(codes + n * K + k) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Q(R) back to values in the W_hat space for the refinement step: out[k][n] (fp64, [K][N])
// = code * scale, exact.  NVFP4: e2m1(q) * e4m3(sf) * gs_w; INT4: q * s16; W8A8: q * s32.
__global__ void dequant_residual64_kernel(const uint8_t *__restrict__ codes, const uint8_t *__restrict__ scales,
                                          int fmt, bool scale_bf16, float gs_w, int64_t K, int64_t N,
                                          double *__restrict__ out) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < K * N;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = idx / N;
    const int64_t n = idx % N;
    double v;
    if (fmt == 2) {
      v = static_cast<double>(reinterpret_cast<const int8_t *>(codes)[n * K + k]) *
          static_cast<double>(reinterpret_cast<const float *>(scales)[n]);
    } else {
      const uint32_t nib = (codes[n * (K / 2) + k / 2] >> (4 * (k & 1))) & 0xFu;
      if (fmt == 0) {
        const float mag[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
        const double e = (nib & 8u) ? -mag[nib & 7u] : mag[nib & 7u];
        v = e * static_cast<double>(e4m3_to_f32(scales[sf_offset(n, k / 16, K)])) * static_cast<double>(gs_w);
      } else {
        const uint16_t sb = reinterpret_cast<const uint16_t *>(scales)[n * (K / 64) + k / 64];
        const float sc = scale_bf16 ? scale16_to_f32<true>(sb) : scale16_to_f32<false>(sb);
        v = static_cast<double>(static_cast<int>(nib ^ 8u) - 8) * static_cast<double>(sc);
      }
    }
    out[idx] = v;
  }
}

__global__ void sub64_kernel(const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ out,
                             int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] - b[i];
}

__global__ void codec_kernel(const float *__restrict__ in, uint8_t *__restrict__ out, int64_t n,
                             int kind) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (kind == 0) out[i] = static_cast<uint8_t>(e2m1x2(in[2 * i], in[2 * i + 1]));
    else out[i] = static_cast<uint8_t>(e4m3_rn_sat(in[i]));
  }
}

__global__ void lambda_inv_kernel(const float *lam, float *lam_inv, int64_t K) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < K) lam_inv[i] = __fdiv_rn(1.0f, lam[i]);
}

// W_hat = diag(lambda) W in fp64 (exact: 24-bit x 24-bit significands).
__global__ void smooth_weight64_kernel(const void *W, int dt, const float *lam, int64_t K, int64_t N,
                                       double *What) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < K * N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    What[i] = static_cast<double>(lam[i / N]) * static_cast<double>(load_any(W, dt, i));
}

__global__ void f32_to_f64_kernel(const float *in, double *out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}
__global__ void f64_to_f32_kernel(const double *in, float *out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __double2float_rn(in[i]);
}

__global__ void derive_l1s_kernel(const void *src, int dt, const float *lam_inv, float scale,
                                  int64_t K, int r_src, int row_offset, uint16_t *l1s) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < K * r_src;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / K;
    const int64_t k = i % K;
    const float v = load_any(src, dt, k * r_src + t);
    const float m = lam_inv ? lam_inv[k] : scale;
    l1s[(row_offset + t) * K + k] = bf16_bits_rn(__fmul_rn(m, v));
  }
}

__global__ void derive_l2s_kernel(const void *src, int dt, int64_t N, int r_src, int col_offset,
                                  int total_rank, float alpha, uint16_t *l2s) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N * r_src;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = i / r_src;
    const int64_t t = i % r_src;
    const float v = load_any(src, dt, t * N + n);
    l2s[n * total_rank + col_offset + t] = bf16_bits_rn(__fdiv_rn(v, alpha));
  }
}

__global__ void copy_l2s_cols_kernel(const uint16_t *src, int64_t N, int r_src, int r_dst,
                                     uint16_t *dst) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N * r_src;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[(i / r_src) * r_dst + (i % r_src)] = src[i];
}

// Top-`rank` eigenpairs (syevd returns them ascending in the columns of the column-major
// V, leading dim P): E[p][t] = V[p][P-1-t] (row-major [P][rank]); sigma[t] = sqrt(max(eval, 0)).
__global__ void eig_to_factors_kernel(const double *V, const double *evals, int64_t P, int rank,
                                      double *E, double *sigma) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < P * rank;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pp = i / rank;
    const int64_t t = i % rank;
    const int64_t col = P - 1 - t;
    E[pp * rank + t] = V[col * P + pp];
    if (pp == 0) sigma[t] = sqrt(fmax(evals[col], 0.0));
  }
}

// A is row-major [rows][cols]; scales column j by sig[j] (by_row == 0) or row i by sig[i]
// (by_row == 1); divides instead when `invert`.
__global__ void scale_cols_kernel(double *A, int64_t rows, int64_t cols, const double *sig,
                                  int invert, int by_row) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * cols;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double s = sig[by_row ? i / cols : i % cols];
    A[i] = invert ? (s > 0 ? A[i] / s : 0.0) : A[i] * s;
  }
}

}  // namespace

cudaError_t launch_absmax(const float *R, int64_t n, unsigned int *out_bits, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out_bits, 0, sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  absmax_kernel<<<blocks_for(n, 256) > 2048 ? 2048 : blocks_for(n, 256), 256, 0, s>>>(R, n, out_bits);
  return cudaGetLastError();
}

cudaError_t launch_quantize_residual(const float *R, int64_t K, int64_t N, int fmt, bool scale_bf16,
                                     float gs_w, uint8_t *codes, uint8_t *scales, cudaStream_t s) {
  if (fmt == 0) {
    const int64_t work = ((N + 127) / 128) * 128 * (K / 16);
    quant_res_nvfp4_kernel<<<blocks_for(work, 256), 256, 0, s>>>(R, K, N, gs_w, codes, scales);
  } else if (fmt == 2) {
    quant_res_int8_kernel<<<blocks_for(N, 128), 128, 0, s>>>(R, K, N, reinterpret_cast<int8_t *>(codes),
                                                            reinterpret_cast<float *>(scales));
  } else {
    const int64_t work = N * (K / 64);
    if (scale_bf16)
      quant_res_int4_kernel<true><<<blocks_for(work, 128), 128, 0, s>>>(
          R, K, N, codes, reinterpret_cast<uint16_t *>(scales));
    else
      quant_res_int4_kernel<false><<<blocks_for(work, 128), 128, 0, s>>>(
          R, K, N, codes, reinterpret_cast<uint16_t *>(scales));
  }
  return cudaGetLastError();
}

cudaError_t launch_dequant_residual64(const uint8_t *codes, const uint8_t *scales, int fmt, bool scale_bf16,
                                      float gs_w, int64_t K, int64_t N, double *out, cudaStream_t s) {
  dequant_residual64_kernel<<<blocks_for(K * N, 256), 256, 0, s>>>(codes, scales, fmt, scale_bf16, gs_w, K, N, out);
  return cudaGetLastError();
}

cudaError_t launch_sub64(const double *a, const double *b, double *out, int64_t n, cudaStream_t s) {
  sub64_kernel<<<blocks_for(n, 256), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}

cudaError_t launch_codec(const float *in, uint8_t *out, int64_t n, int kind, cudaStream_t s) {
  codec_kernel<<<blocks_for(n, 256), 256, 0, s>>>(in, out, n, kind);
  return cudaGetLastError();
}

cudaError_t launch_lambda_inv(const float *lam, float *lam_inv, int64_t K, cudaStream_t s) {
  lambda_inv_kernel<<<blocks_for(K, 256), 256, 0, s>>>(lam, lam_inv, K);
  return cudaGetLastError();
}

cudaError_t launch_smooth_weight64(const void *W, int w_dtype, const float *lam, int64_t K, int64_t N,
                                   double *What, cudaStream_t s) {
  smooth_weight64_kernel<<<blocks_for(K * N, 256), 256, 0, s>>>(W, w_dtype, lam, K, N, What);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_f64(const float *in, double *out, int64_t n, cudaStream_t s) {
  f32_to_f64_kernel<<<blocks_for(n, 256), 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}
cudaError_t launch_f64_to_f32(const double *in, float *out, int64_t n, cudaStream_t s) {
  f64_to_f32_kernel<<<blocks_for(n, 256), 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t launch_derive_l1s(const void *src, int src_dtype, const float *lam_inv, float scale,
                              int64_t K, int r_src, int row_offset, uint16_t *l1s, cudaStream_t s) {
  derive_l1s_kernel<<<blocks_for(K * r_src, 256), 256, 0, s>>>(src, src_dtype, lam_inv, scale, K,
                                                               r_src, row_offset, l1s);
  return cudaGetLastError();
}

cudaError_t launch_derive_l2s(const void *src, int src_dtype, int64_t N, int r_src, int col_offset,
                              int total_rank, float alpha, uint16_t *l2s, cudaStream_t s) {
  derive_l2s_kernel<<<blocks_for(N * r_src, 256), 256, 0, s>>>(src, src_dtype, N, r_src, col_offset,
                                                               total_rank, alpha, l2s);
  return cudaGetLastError();
}

cudaError_t launch_copy_l1s_rows(const uint16_t *src, int64_t K, int rows, uint16_t *dst,
                                 cudaStream_t s) {
  return cudaMemcpyAsync(dst, src, static_cast<size_t>(K) * rows * sizeof(uint16_t),
                         cudaMemcpyDeviceToDevice, s);
}

cudaError_t launch_copy_l2s_cols(const uint16_t *src, int64_t N, int r_src, int r_dst, uint16_t *dst,
                                 cudaStream_t s) {
  copy_l2s_cols_kernel<<<blocks_for(N * r_src, 256), 256, 0, s>>>(src, N, r_src, r_dst, dst);
  return cudaGetLastError();
}

cudaError_t launch_eig_to_factors(const double *V, const double *evals, int64_t P, int rank,
                                  double *out_vecs, double *out_sigma, cudaStream_t s) {
  eig_to_factors_kernel<<<blocks_for(P * rank, 256), 256, 0, s>>>(V, evals, P, rank, out_vecs,
                                                                  out_sigma);
  return cudaGetLastError();
}

cudaError_t launch_scale_cols(double *A, int64_t rows, int64_t cols, const double *sig, int invert,
                              int by_row, cudaStream_t s) {
  scale_cols_kernel<<<blocks_for(rows * cols, 256), 256, 0, s>>>(A, rows, cols, sig, invert, by_row);
  return cudaGetLastError();
}

}  // namespace svdq
