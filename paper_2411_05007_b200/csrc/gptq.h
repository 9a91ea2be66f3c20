// GPTQ residual quantization (gptq.cu), used by svdq_quantize_weights_gptq (api.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/svdq.h"

namespace svdq {

struct GptqArgs {               // calibration activations for the Hessian
  const void *X;                // [dev] [M][ldx] BF16 | FP16 (unsmoothed)
  int32_t x_dtype;
  int64_t M, ldx;
  float damp;                   // H += damp * mean(diag H) * I (reading G1)
};

struct GptqState {              // views into the GPTQ workspace
  double *U;                    // [K][K] row-major upper Cholesky factor of H^-1
  int *dead;                    // [K] 1 where diag(H) == 0
  double *E;                    // [64][N] scaled errors of the current block
};

size_t gptq_workspace_bytes(int64_t M, int64_t K, int64_t N, int lwork);
int gptq_potrf_lwork(int64_t K);
// H from X_hat = fl32(X * lam_inv), dead fix, dampening, U.  Synchronizes s.  nullptr or an error string.
const char *gptq_hessian(const GptqArgs &a, const float *lam_inv, int64_t K, int lwork, uint8_t *ws,
                         cudaStream_t s, GptqState *st);
cudaError_t gptq_zero_dead(double *R, const GptqState &st, int64_t K, int64_t N, cudaStream_t s);
// Quantize R ([K][N] fp64, overwritten) into codes / scales (fmt 0 NVFP4 with gs, 1 INT4, 2 W8A8 with
// the per-channel w8_scales already computed).  NVFP4 padding rows of `scales` are left as they are.
const char *gptq_run(double *R, const GptqState &st, int64_t K, int64_t N, int fmt, bool scale_bf16, float gs,
                     const float *w8_scales, uint8_t *codes, uint8_t *scales, cudaStream_t s);

// svdq_quantize_weights with the offline extensions (api.cu): an optional refinement target
// svd_sub ([K][N] fp64, Q(R_{t-1}); tgt = [K][N] fp64 scratch) and optional GPTQ residual
// quantization (gq != nullptr; gq_ws = gptq_workspace_bytes(M, K, N, gptq_potrf_lwork(K)) bytes).
svdq_status quantize_weights_impl(const void *W, int32_t w_dtype, const float *lambda, int64_t K, int64_t N,
                                  int32_t rank, int32_t fmt, int32_t scale_dtype, float gs_x, const float *L1_opt,
                                  const float *L2_opt, svdq_linear *dst, void *ws, size_t ws_bytes, void *stream,
                                  const double *svd_sub, double *tgt, const GptqArgs *gq, uint8_t *gq_ws);

}  // namespace svdq
