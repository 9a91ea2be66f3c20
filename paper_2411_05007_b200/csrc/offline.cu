// Offline weight pipeline on the GPU: the per-layer search for the
// migration strength alpha, "decided offline by searching for the best migration strength
// alpha for each layer to minimize the layer output mean squared error (MSE) after SVD on the
// calibration dataset" (App. D).  Every candidate runs the deployed pipeline: lambda(alpha)
// (P:467), full weight preparation (smoothing, SVD, residual quantization), K1 -> K2 on the
// calibration activations, and ||X_cal W - Y||_F^2 against an fp32 cuBLAS reference GEMM.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/svdq.h"
#include "k1_launch.h"
#include "sm100.cuh"

namespace svdq {
svdq_status report_error(svdq_status s, const char *msg);   // api.cu
}

namespace {

__device__ __forceinline__ float x16f(const void *p, int dt, int64_t i) {
  const uint16_t b = static_cast<const uint16_t *>(p)[i];
  return dt == 0 ? __uint_as_float(static_cast<uint32_t>(b) << 16) : __half2float(__ushort_as_half(b));
}

// max over rows of |X[:, k]|, and the fp32 copy of X for the reference GEMM
__global__ void xcal_prep_kernel(const void *X, int dt, int64_t M, int64_t K, int64_t ldx, float *xa, float *xf) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float m = 0.f;
  for (int64_t r = 0; r < M; ++r) {
    const float v = x16f(X, dt, r * ldx + k);
    xf[r * K + k] = v;
    m = fmaxf(m, fabsf(v));
  }
  xa[k] = m;
}

// max over n of |W[k, :]|, one block per row
__global__ void wrow_absmax_kernel(const float *W, int64_t N, float *wa) {
  const float *row = W + static_cast<int64_t>(blockIdx.x) * N;
  float m = 0.f;
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) m = fmaxf(m, fabsf(row[n]));
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) wa[blockIdx.x] = m;
  }
}

// lambda_k = max|X_:,k|^alpha / max|W_k,:|^(1 - alpha) in fp64, non-finite -> 1e5,
// clamped to [1e-5, 1e5], stored fp32 (the oracle's compute_smoothing)
__global__ void lambda_kernel(const float *xa, const float *wa, double alpha, int64_t K, float *lam) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double l = pow(static_cast<double>(xa[k]), alpha) / pow(static_cast<double>(wa[k]), 1.0 - alpha);
  if (!isfinite(l)) l = 1e5;
  l = fmin(fmax(l, 1e-5), 1e5);
  lam[k] = static_cast<float>(l);
}

__global__ void sq_err_kernel(const float *a, const float *b, int64_t n, double *out) {
  double s = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double d = static_cast<double>(a[i]) - static_cast<double>(b[i]);
    s += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
    atomicAdd(out, t);
  }
}

struct AlphaWs {
  size_t xa, wa, lam, codes, scales, laminv, l1s, l2s, qws, xq, xs, xl1, y, yref, xf, err, total;
  size_t codes_b, scales_b, l1s_b, l2s_b, qws_b, xq_b, xs_b, xl1_b;
};

svdq_status alpha_ws(int32_t fmt, int64_t M, int64_t K, int64_t N, int32_t rank, AlphaWs *w) {
  svdq_status st;
  if ((st = svdq_weight_buffer_sizes(fmt, K, N, rank, &w->codes_b, &w->scales_b, &w->l1s_b, &w->l2s_b)) != SVDQ_OK)
    return st;
  if ((st = svdq_quantize_weights_workspace(K, N, rank, &w->qws_b)) != SVDQ_OK) return st;
  if ((st = svdq_act_buffer_sizes(fmt, M, K, rank, &w->xq_b, &w->xs_b, &w->xl1_b)) != SVDQ_OK) return st;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  w->xa = take(K * 4);
  w->wa = take(K * 4);
  w->lam = take(K * 4);
  w->codes = take(w->codes_b);
  w->scales = take(w->scales_b);
  w->laminv = take(K * 4);
  w->l1s = take(w->l1s_b > 0 ? w->l1s_b : 16);
  w->l2s = take(w->l2s_b > 0 ? w->l2s_b : 16);
  w->qws = take(w->qws_b);
  w->xq = take(w->xq_b);
  w->xs = take(w->xs_b);
  w->xl1 = take(w->xl1_b > 0 ? w->xl1_b : 16);
  w->y = take(static_cast<size_t>(M) * N * 4);
  w->yref = take(static_cast<size_t>(M) * N * 4);
  w->xf = take(static_cast<size_t>(M) * K * 4);
  w->err = take(8);
  w->total = off;
  return SVDQ_OK;
}

}  // namespace

extern "C" {

svdq_status svdq_search_alpha_workspace(int32_t fmt, int64_t M_cal, int64_t K, int64_t N, int32_t rank,
                                        size_t *ws_bytes) {
  if (!ws_bytes) return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (M_cal < 1) return svdq::report_error(SVDQ_ERR_SHAPE, "M_cal must be >= 1");
  AlphaWs w;
  svdq_status st = alpha_ws(fmt, M_cal, K, N, rank, &w);
  if (st != SVDQ_OK) return st;
  *ws_bytes = w.total;
  return SVDQ_OK;
}

svdq_status svdq_search_alpha(const void *X_cal, int32_t x_dtype, int64_t M_cal, int64_t ldx, const float *W,
                              int64_t K, int64_t N, int32_t rank, int32_t fmt, int32_t scale_dtype, float gs_x,
                              const float *grid, int32_t n_grid, float *alpha_out, float *lambda_out,
                              double *objective_out, void *ws, size_t ws_bytes, void *stream) {
  if (!X_cal || !W || !grid || !alpha_out || !lambda_out || !objective_out || !ws)
    return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (n_grid < 1) return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "empty alpha grid");
  for (int i = 0; i < n_grid; ++i)
    if (!(grid[i] >= 0.f && grid[i] <= 1.f)) return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "alpha outside [0, 1]");
  if (x_dtype != SVDQ_BF16 && x_dtype != SVDQ_FP16) return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "X dtype");
  if (ldx < K) return svdq::report_error(SVDQ_ERR_SHAPE, "ldx < K");
  AlphaWs w;
  svdq_status st = alpha_ws(fmt, M_cal, K, N, rank, &w);
  if (st != SVDQ_OK) return st;
  if (ws_bytes < w.total) return svdq::report_error(SVDQ_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t *base = static_cast<uint8_t *>(ws);
  float *xa = reinterpret_cast<float *>(base + w.xa);
  float *wa = reinterpret_cast<float *>(base + w.wa);
  float *lam = reinterpret_cast<float *>(base + w.lam);
  float *y = reinterpret_cast<float *>(base + w.y);
  float *yref = reinterpret_cast<float *>(base + w.yref);
  float *xf = reinterpret_cast<float *>(base + w.xf);
  double *err = reinterpret_cast<double *>(base + w.err);
  const int xdt = x_dtype == SVDQ_BF16 ? 0 : 1;

  xcal_prep_kernel<<<static_cast<unsigned>((K + 127) / 128), 128, 0, s>>>(X_cal, xdt, M_cal, K, ldx, xa, xf);
  wrow_absmax_kernel<<<static_cast<unsigned>(K), 256, 0, s>>>(W, N, wa);
  if (cudaGetLastError() != cudaSuccess) return svdq::report_error(SVDQ_ERR_CUDA, "alpha-search prep kernels");
  // reference Y = X_cal W in fp32 (row-major; cuBLAS column-major view: Y^T = W^T X^T)
  cublasHandle_t hb = nullptr;
  if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) return svdq::report_error(SVDQ_ERR_CUDA, "cublasCreate");
  cublasSetStream(hb, s);
  cublasSetMathMode(hb, CUBLAS_PEDANTIC_MATH);
  const float one = 1.f, zero = 0.f;
  const cublasStatus_t cb = cublasSgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(N), static_cast<int>(M_cal),
                                        static_cast<int>(K), &one, W, static_cast<int>(N), xf, static_cast<int>(K),
                                        &zero, yref, static_cast<int>(N));
  cublasDestroy(hb);
  if (cb != CUBLAS_STATUS_SUCCESS) return svdq::report_error(SVDQ_ERR_CUDA, "reference sgemm");

  svdq_linear L;
  std::memset(&L, 0, sizeof(L));
  L.w_codes = base + w.codes;
  L.w_scales = base + w.scales;
  L.lambda_inv = reinterpret_cast<float *>(base + w.laminv);
  L.l1s = reinterpret_cast<uint16_t *>(base + w.l1s);
  L.l2s = reinterpret_cast<uint16_t *>(base + w.l2s);
  std::vector<double> obj(n_grid);
  for (int i = 0; i < n_grid; ++i) {
    lambda_kernel<<<static_cast<unsigned>((K + 255) / 256), 256, 0, s>>>(xa, wa, static_cast<double>(grid[i]), K, lam);
    if (cudaGetLastError() != cudaSuccess) return svdq::report_error(SVDQ_ERR_CUDA, "lambda kernel");
    if ((st = svdq_quantize_weights(W, SVDQ_FP32, lam, K, N, rank, fmt, scale_dtype, gs_x, nullptr, nullptr, &L,
                                    base + w.qws, w.qws_b, stream)) != SVDQ_OK)
      return st;
    uint8_t *xq = base + w.xq, *xs = base + w.xs;
    uint16_t *xl1 = reinterpret_cast<uint16_t *>(base + w.xl1);
    if ((st = svdq_quantize_act_lowrank_down(&L, X_cal, x_dtype, M_cal, ldx, xq, xs, rank ? xl1 : nullptr, stream)) !=
        SVDQ_OK)
      return st;
    // the objective has no bias (the layer output of X W)
    const void *bias = L.bias;
    L.bias = nullptr;
    st = svdq_gemm_w4a4_lowrank_up(&L, xq, xs, rank ? xl1 : nullptr, M_cal, y, SVDQ_FP32, N, stream);
    L.bias = bias;
    if (st != SVDQ_OK) return st;
    if (cudaMemsetAsync(err, 0, sizeof(double), s) != cudaSuccess) return svdq::report_error(SVDQ_ERR_CUDA, "memset");
    sq_err_kernel<<<296, 256, 0, s>>>(y, yref, M_cal * N, err);
    if (cudaMemcpyAsync(&obj[i], err, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return svdq::report_error(SVDQ_ERR_CUDA, "objective readback");
  }
  int best = 0;
  for (int i = 1; i < n_grid; ++i)
    if (obj[i] < obj[best] || (obj[i] == obj[best] && grid[i] < grid[best])) best = i;
  for (int i = 0; i < n_grid; ++i) objective_out[i] = obj[i];
  *alpha_out = grid[best];
  lambda_kernel<<<static_cast<unsigned>((K + 255) / 256), 256, 0, s>>>(xa, wa, static_cast<double>(grid[best]), K,
                                                                       lambda_out);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return svdq::report_error(SVDQ_ERR_CUDA, "lambda(alpha*)");
  return SVDQ_OK;
}

}  // extern "C"
