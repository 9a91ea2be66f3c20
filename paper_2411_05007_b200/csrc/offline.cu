// Offline weight pipeline on the GPU: the per-layer search for the
// migration strength alpha, "decided offline by searching for the best migration strength
// alpha for each layer to minimize the layer output mean squared error (MSE) after SVD on the
// calibration dataset" (App. D).  Every candidate runs the deployed pipeline: lambda(alpha)
// (P:467), full weight preparation (smoothing, SVD, residual quantization), K1 -> K2 on the
// calibration activations, and ||X_cal W - Y||_F^2 against an fp32 cuBLAS reference GEMM.
// And the iterative low-rank refinement: "iteratively updating the low-rank branch
// through decomposing W - Q(R) and adjusting R accordingly for several iterations, and then
// picking the result with the smallest error" -- read as W_hat - Q(R) (reading Q3), scored by
// the same objective.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/svdq.h"
#include "gptq.h"
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

// ||a - b||^2 in fp64 with a fixed summation order (deterministic: equal iterates score equal):
// block partials, then one block sums them in index order
constexpr int kErrBlocks = 296;
__global__ void sq_err_kernel(const float *a, const float *b, int64_t n, double *partial) {
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
    partial[blockIdx.x] = t;
  }
}

__global__ void sum_partials_kernel(const double *partial, int n, double *out) {
  double t = 0.0;
  for (int i = 0; i < n; ++i) t += partial[i];
  *out = t;
}

struct AlphaWs {
  size_t xa, wa, lam, codes, scales, laminv, l1s, l2s, qws, xq, xs, xl1, y, yref, xf, err, total;
  size_t codes_b, scales_b, l1s_b, l2s_b, qws_b, xq_b, xs_b, xl1_b;
  size_t deq, tgt;   // refinement only: Q(R_{t-1}) and W_hat - Q(R_{t-1}), [K][N] fp64
};

svdq_status alpha_ws(int32_t fmt, int64_t M, int64_t K, int64_t N, int32_t rank, AlphaWs *w, bool refine = false) {
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
  w->err = take((kErrBlocks + 1) * 8);
  w->deq = refine ? take(static_cast<size_t>(K) * N * 8) : 0;
  w->tgt = refine ? take(static_cast<size_t>(K) * N * 8) : 0;
  w->total = off;
  return SVDQ_OK;
}

// Y_ref = X_cal W in fp32 (cuBLAS, pedantic math): row-major, so the column-major view is Y^T = W^T X^T
svdq_status reference_gemm(const float *xf, const float *W, int64_t M, int64_t K, int64_t N, float *yref,
                           cudaStream_t s) {
  cublasHandle_t hb = nullptr;
  if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) return svdq::report_error(SVDQ_ERR_CUDA, "cublasCreate");
  cublasSetStream(hb, s);
  cublasSetMathMode(hb, CUBLAS_PEDANTIC_MATH);
  const float one = 1.f, zero = 0.f;
  const cublasStatus_t cb = cublasSgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(N), static_cast<int>(M),
                                        static_cast<int>(K), &one, W, static_cast<int>(N), xf, static_cast<int>(K),
                                        &zero, yref, static_cast<int>(N));
  cublasDestroy(hb);
  return cb == CUBLAS_STATUS_SUCCESS ? SVDQ_OK : svdq::report_error(SVDQ_ERR_CUDA, "reference sgemm");
}

// The App. D objective (reading Q4): the deployed K1 -> K2 forward of L on X_cal without
// bias, ||X_cal W - Y||_F^2 summed in fp64.  Synchronizes s; result in *obj [host].
svdq_status objective(svdq_linear *L, const void *X_cal, int32_t x_dtype, int64_t M, int64_t ldx, uint8_t *xq,
                      uint8_t *xs, uint16_t *xl1, float *y, const float *yref, double *err, cudaStream_t s,
                      double *obj) {
  svdq_status st;
  const int32_t rank = L->rank;
  if ((st = svdq_quantize_act_lowrank_down(L, X_cal, x_dtype, M, ldx, xq, xs, rank ? xl1 : nullptr, s)) != SVDQ_OK)
    return st;
  const void *bias = L->bias;
  L->bias = nullptr;
  st = svdq_gemm_w4a4_lowrank_up(L, xq, xs, rank ? xl1 : nullptr, M, y, SVDQ_FP32, L->N, s);
  L->bias = bias;
  if (st != SVDQ_OK) return st;
  sq_err_kernel<<<kErrBlocks, 256, 0, s>>>(y, yref, M * L->N, err + 1);
  sum_partials_kernel<<<1, 1, 0, s>>>(err + 1, kErrBlocks, err);
  if (cudaMemcpyAsync(obj, err, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return svdq::report_error(SVDQ_ERR_CUDA, "objective readback");
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
  if ((st = reference_gemm(xf, W, M_cal, K, N, yref, s)) != SVDQ_OK) return st;

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
    if ((st = objective(&L, X_cal, x_dtype, M_cal, ldx, base + w.xq, base + w.xs,
                        reinterpret_cast<uint16_t *>(base + w.xl1), y, yref, err, s, &obj[i])) != SVDQ_OK)
      return st;
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

// ---------------------------------------------------------------- iterative refinement
svdq_status svdq_refine_lowrank_workspace(int32_t fmt, int64_t M_cal, int64_t K, int64_t N, int32_t rank,
                                          int32_t use_gptq, size_t *ws_bytes) {
  if (!ws_bytes) return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (M_cal < 1) return svdq::report_error(SVDQ_ERR_SHAPE, "M_cal must be >= 1");
  AlphaWs w;
  svdq_status st = alpha_ws(fmt, M_cal, K, N, rank, &w, true);
  if (st != SVDQ_OK) return st;
  *ws_bytes = w.total;
  if (use_gptq) {
    const int glw = svdq::gptq_potrf_lwork(K);
    if (glw < 0) return svdq::report_error(SVDQ_ERR_CUDA, "cusolver potrf bufferSize failed");
    *ws_bytes += svdq::gptq_workspace_bytes(M_cal, K, N, glw);
  }
  return SVDQ_OK;
}

svdq_status svdq_refine_lowrank(const void *X_cal, int32_t x_dtype, int64_t M_cal, int64_t ldx, const float *W,
                                const float *lambda, int64_t K, int64_t N, int32_t rank, int32_t fmt,
                                int32_t scale_dtype, float gs_x, int32_t iters, int32_t use_gptq, float damp,
                                svdq_linear *dst, int32_t *best_out, double *objective_out, void *ws, size_t ws_bytes,
                                void *stream) {
  if (!X_cal || !W || !lambda || !dst || !best_out || !objective_out || !ws)
    return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (iters < 0) return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "iters must be >= 0");
  if (x_dtype != SVDQ_BF16 && x_dtype != SVDQ_FP16) return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "X dtype");
  if (ldx < K) return svdq::report_error(SVDQ_ERR_SHAPE, "ldx < K");
  if (!dst->w_codes || !dst->w_scales || !dst->lambda_inv || (rank > 0 && (!dst->l1s || !dst->l2s)))
    return svdq::report_error(SVDQ_ERR_INVALID_ARGUMENT, "dst buffers must be set");
  AlphaWs w;
  svdq_status st = alpha_ws(fmt, M_cal, K, N, rank, &w, true);
  if (st != SVDQ_OK) return st;
  size_t need = 0;
  if ((st = svdq_refine_lowrank_workspace(fmt, M_cal, K, N, rank, use_gptq, &need)) != SVDQ_OK) return st;
  if (ws_bytes < need) return svdq::report_error(SVDQ_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t *base = static_cast<uint8_t *>(ws);
  const svdq::GptqArgs gq{X_cal, x_dtype, M_cal, ldx, damp};
  float *y = reinterpret_cast<float *>(base + w.y);
  float *yref = reinterpret_cast<float *>(base + w.yref);
  float *xf = reinterpret_cast<float *>(base + w.xf);
  double *err = reinterpret_cast<double *>(base + w.err);
  double *deq = reinterpret_cast<double *>(base + w.deq);
  double *tgt = reinterpret_cast<double *>(base + w.tgt);

  xcal_prep_kernel<<<static_cast<unsigned>((K + 127) / 128), 128, 0, s>>>(X_cal, x_dtype == SVDQ_BF16 ? 0 : 1, M_cal,
                                                                         K, ldx, reinterpret_cast<float *>(base + w.xa),
                                                                         xf);
  if (cudaGetLastError() != cudaSuccess) return svdq::report_error(SVDQ_ERR_CUDA, "refine prep kernel");
  if ((st = reference_gemm(xf, W, M_cal, K, N, yref, s)) != SVDQ_OK) return st;

  // the current iterate lives in the workspace; the best one so far is copied into dst
  svdq_linear L;
  std::memset(&L, 0, sizeof(L));
  L.w_codes = base + w.codes;
  L.w_scales = base + w.scales;
  L.lambda_inv = reinterpret_cast<float *>(base + w.laminv);
  L.l1s = reinterpret_cast<uint16_t *>(base + w.l1s);
  L.l2s = reinterpret_cast<uint16_t *>(base + w.l2s);
  auto keep = [&]() -> svdq_status {
    const bool ok =
        cudaMemcpyAsync(const_cast<uint8_t *>(dst->w_codes), L.w_codes, w.codes_b, cudaMemcpyDeviceToDevice, s) ==
            cudaSuccess &&
        cudaMemcpyAsync(const_cast<uint8_t *>(dst->w_scales), L.w_scales, w.scales_b, cudaMemcpyDeviceToDevice, s) ==
            cudaSuccess &&
        cudaMemcpyAsync(const_cast<float *>(dst->lambda_inv), L.lambda_inv, K * 4, cudaMemcpyDeviceToDevice, s) ==
            cudaSuccess &&
        (rank == 0 ||
         (cudaMemcpyAsync(const_cast<uint16_t *>(dst->l1s), L.l1s, w.l1s_b, cudaMemcpyDeviceToDevice, s) ==
              cudaSuccess &&
          cudaMemcpyAsync(const_cast<uint16_t *>(dst->l2s), L.l2s, w.l2s_b, cudaMemcpyDeviceToDevice, s) ==
              cudaSuccess));
    if (!ok) return svdq::report_error(SVDQ_ERR_CUDA, "copy best iterate");
    dst->fmt = L.fmt;
    dst->rank = L.rank;
    dst->K = L.K;
    dst->N = L.N;
    dst->scale_dtype = L.scale_dtype;
    dst->gs_w = L.gs_w;
    dst->gs_x = L.gs_x;
    return SVDQ_OK;
  };
  int best = 0;
  for (int t = 0; t <= iters; ++t) {
    if (t > 0 && svdq::launch_dequant_residual64(L.w_codes, L.w_scales, fmt, L.scale_dtype == SVDQ_BF16, L.gs_w, K, N, deq,
                                           s) != cudaSuccess)
      return svdq::report_error(SVDQ_ERR_CUDA, "dequantize residual");
    if ((st = svdq::quantize_weights_impl(W, SVDQ_FP32, lambda, K, N, rank, fmt, scale_dtype, gs_x, nullptr, nullptr,
                                          &L, base + w.qws, w.qws_b, stream, t > 0 ? deq : nullptr,
                                          t > 0 ? tgt : nullptr, use_gptq ? &gq : nullptr,
                                          use_gptq ? base + w.total : nullptr)) != SVDQ_OK)
      return st;
    if ((st = objective(&L, X_cal, x_dtype, M_cal, ldx, base + w.xq, base + w.xs,
                        reinterpret_cast<uint16_t *>(base + w.xl1), y, yref, err, s, &objective_out[t])) != SVDQ_OK)
      return st;
    if (t == 0 || objective_out[t] < objective_out[best]) {   // ties -> the earlier iterate
      best = t;
      if ((st = keep()) != SVDQ_OK) return st;
    }
  }
  *best_out = best;
  if (cudaStreamSynchronize(s) != cudaSuccess) return svdq::report_error(SVDQ_ERR_CUDA, "sync");
  return SVDQ_OK;
}

}  // extern "C"
