// GPTQ quantization of the residual on the GPU (App. D: "We use GPTQ to quantize the
// residual weights").  The cited method's column-by-column algorithm with
// its lazy-batch blocking (Frantar et al., Alg. 1), on R in the paper layout [K][N]:
//
//   H = X_hat^T X_hat (fp64 syrk of X_hat = fl32(x * lambda_inv)), dead channels -> H_kk = 1 and
//   R[k, :] = 0, H += damp * mean(diag H) * I, U = upper Cholesky factor of H^-1 (potrf, potri,
//   potrf), then per block of B = 64 input channels: one thread per output channel quantizes the
//   block column by column (group scale from the current values at each group start, reading G2),
//   propagates e_k = (r_k - deq(q_k)) / U_kk inside the block, and the trailing rows receive
//   R[i2:, :] -= U[i1:i2, i2:]^T E in one DGEMM.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdint>

#include "../../include/svdq.h"
#include "formats.cuh"
#include "gptq.h"

namespace svdq {

namespace {

constexpr int kB = 64;          // block of input channels = the INT4 group
constexpr int kThreads = 128;   // output channels per CTA

__device__ __forceinline__ float x16(const void *p, int dt, int64_t i) {
  const uint16_t b = static_cast<const uint16_t *>(p)[i];
  return dt == 0 ? __uint_as_float(static_cast<uint32_t>(b) << 16) : __half2float(__ushort_as_half(b));
}

// X_hat = fl32(x * lambda_inv) (K1's smoothing, reading Q14), stored fp64 [M][K]
__global__ void xhat64_kernel(const void *X, int dt, int64_t M, int64_t ldx, const float *lam_inv, int64_t K,
                              double *out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < M * K;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = i / K, k = i % K;
    out[i] = static_cast<double>(__fmul_rn(x16(X, dt, m * ldx + k), lam_inv[k]));
  }
}

// dead channels (H_kk == 0) -> H_kk = 1, flag; then H_kk += damp * mean(diag H).  One block.
__global__ void hess_fix_kernel(double *H, int64_t K, double damp, int *dead) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    double h = H[k * K + k];
    const int d = h == 0.0;
    if (d) h = 1.0;
    H[k * K + k] = h;
    dead[k] = d;
    s += h;
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
    red[0] = t;
  }
  __syncthreads();
  const double add = damp * (red[0] / static_cast<double>(K));
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) H[k * K + k] += add;
}

__global__ void zero_dead_rows_kernel(double *R, const int *dead, int64_t K, int64_t N) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < K * N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (dead[i / N]) R[i] = 0.0;
}

__device__ __forceinline__ float e2m1_val(uint32_t nib) {
  const float mag[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
  const float m = mag[nib & 7u];
  return (nib & 8u) ? -m : m;
}

// One block of kB input channels [i1, i1 + kB) for every output channel (thread n).
// R: [K][N] fp64 current residual; U: [K][K] row-major upper factor; E: [kB][N] scaled errors out.
template <int kFmt, bool kBf16>
__global__ void __launch_bounds__(kThreads) gptq_block_kernel(double *__restrict__ R, const double *__restrict__ U,
                                                              int64_t K, int64_t N, int64_t i1, float gs,
                                                              const float *__restrict__ w8s, uint8_t *__restrict__ codes,
                                                              uint8_t *__restrict__ scales, double *__restrict__ E) {
  extern __shared__ double sm[];
  double *Us = sm;                          // [kB][kB]
  double *ws = sm + kB * kB;                // [kB][kThreads]
  const int tid = threadIdx.x;
  const int64_t n = static_cast<int64_t>(blockIdx.x) * kThreads + tid;
  for (int i = tid; i < kB * kB; i += kThreads) Us[i] = U[(i1 + i / kB) * K + i1 + i % kB];
  if (n < N)
    for (int j = 0; j < kB; ++j) ws[j * kThreads + tid] = R[(i1 + j) * N + n];
  __syncthreads();
  if (n >= N) return;
  constexpr int G = kFmt == 0 ? 16 : 64;
  float qinv = 0.f, sd = 0.f;
  if constexpr (kFmt == 2) {
    sd = w8s[n];
    qinv = sd == 0.f ? 0.f : __fdiv_rn(1.0f, sd);
  }
  uint32_t packed = 0;
  for (int k = 0; k < kB; ++k) {
    if constexpr (kFmt != 2) {
      if (k % G == 0) {                      // group scale from the current values (reading G2)
        float amax = 0.f;
        for (int j = 0; j < G; ++j) amax = fmaxf(amax, fabsf(static_cast<float>(ws[(k + j) * kThreads + tid])));
        if constexpr (kFmt == 0) {
          const float t6 = __fmul_rn(__fdiv_rn(1.0f, gs), __fdiv_rn(1.0f, 6.0f));
          const uint32_t sf = e4m3_rn_sat(__fmul_rn(amax, t6));
          sd = e4m3_to_f32(sf);
          qinv = sd == 0.f ? 0.f : __fdiv_rn(1.0f, __fmul_rn(sd, gs));
          scales[sf_offset(n, (i1 + k) / 16, K)] = static_cast<uint8_t>(sf);
        } else {
          const uint16_t sb = scale16_rn_sat<kBf16>(__fdiv_rn(amax, 7.0f));
          sd = scale16_to_f32<kBf16>(sb);
          qinv = sd == 0.f ? 0.f : __fdiv_rn(1.0f, sd);
          reinterpret_cast<uint16_t *>(scales)[n * (K / 64) + (i1 + k) / 64] = sb;
        }
      }
    }
    const double w = ws[k * kThreads + tid];
    const float v = __fmul_rn(static_cast<float>(w), qinv);
    double deq;
    if constexpr (kFmt == 0) {
      const uint32_t nib = e2m1x2(v, 0.f) & 0xFu;
      deq = static_cast<double>(e2m1_val(nib)) * static_cast<double>(sd) * static_cast<double>(gs);
      packed |= nib << (4 * (k & 1));
      if (k & 1) {
        codes[n * (K / 2) + (i1 + k) / 2] = static_cast<uint8_t>(packed);
        packed = 0;
      }
    } else if constexpr (kFmt == 1) {
      const int q = max(-7, min(7, __float2int_rn(v)));
      deq = static_cast<double>(q) * static_cast<double>(sd);
      packed |= (static_cast<uint32_t>(q) & 0xFu) << (4 * (k & 1));
      if (k & 1) {
        codes[n * (K / 2) + (i1 + k) / 2] = static_cast<uint8_t>(packed);
        packed = 0;
      }
    } else {
      const int q = max(-127, min(127, __float2int_rn(v)));
      deq = static_cast<double>(q) * static_cast<double>(sd);
      codes[n * K + i1 + k] = static_cast<uint8_t>(static_cast<int8_t>(q));
    }
    const double e = (w - deq) / Us[k * kB + k];
    E[k * N + n] = e;
    for (int j = k + 1; j < kB; ++j) ws[j * kThreads + tid] -= e * Us[k * kB + j];
  }
}

unsigned blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > (1 << 20)) b = 1 << 20;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace

size_t gptq_workspace_bytes(int64_t M, int64_t K, int64_t N, int lwork) {
  auto up = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  return up(static_cast<size_t>(M) * K * 8) + up(static_cast<size_t>(K) * K * 8) + up(static_cast<size_t>(K) * 4) +
         up(static_cast<size_t>(lwork > 0 ? lwork : 1) * 8) + up(16) + up(static_cast<size_t>(kB) * N * 8);
}

int gptq_potrf_lwork(int64_t K) {
  cusolverDnHandle_t h;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) return -1;
  int l1 = 0, l2 = 0;
  const bool ok = cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, static_cast<int>(K), nullptr,
                                              static_cast<int>(K), &l1) == CUSOLVER_STATUS_SUCCESS &&
                  cusolverDnDpotri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, static_cast<int>(K), nullptr,
                                              static_cast<int>(K), &l2) == CUSOLVER_STATUS_SUCCESS;
  cusolverDnDestroy(h);
  return ok ? (l1 > l2 ? l1 : l2) : -1;
}

const char *gptq_hessian(const GptqArgs &a, const float *lam_inv, int64_t K, int lwork, uint8_t *ws,
                         cudaStream_t s, GptqState *st) {
  auto up = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  double *xh = reinterpret_cast<double *>(ws);
  ws += up(static_cast<size_t>(a.M) * K * 8);
  st->U = reinterpret_cast<double *>(ws);
  ws += up(static_cast<size_t>(K) * K * 8);
  st->dead = reinterpret_cast<int *>(ws);
  ws += up(static_cast<size_t>(K) * 4);
  double *work = reinterpret_cast<double *>(ws);
  ws += up(static_cast<size_t>(lwork > 0 ? lwork : 1) * 8);
  int *info = reinterpret_cast<int *>(ws);
  ws += up(16);
  st->E = reinterpret_cast<double *>(ws);

  xhat64_kernel<<<blocks_for(a.M * K), 256, 0, s>>>(a.X, a.x_dtype == SVDQ_BF16 ? 0 : 1, a.M, a.ldx, lam_inv, K, xh);
  if (cudaGetLastError() != cudaSuccess) return "xhat kernel";
  cublasHandle_t hb = nullptr;
  if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) return "cublasCreate";
  cublasSetStream(hb, s);
  const double one = 1.0, zero = 0.0;
  // column-major view of row-major xh [M][K] is xh^T (K x M); H = xh^T xh, lower triangle
  const cublasStatus_t cb = cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, static_cast<int>(K),
                                        static_cast<int>(a.M), &one, xh, static_cast<int>(K), &zero, st->U,
                                        static_cast<int>(K));
  cublasDestroy(hb);
  if (cb != CUBLAS_STATUS_SUCCESS) return "syrk H";
  hess_fix_kernel<<<1, 1024, 0, s>>>(st->U, K, static_cast<double>(a.damp), st->dead);
  if (cudaGetLastError() != cudaSuccess) return "hessian fix";
  cusolverDnHandle_t hs = nullptr;
  if (cusolverDnCreate(&hs) != CUSOLVER_STATUS_SUCCESS) return "cusolverDnCreate";
  cusolverDnSetStream(hs, s);
  const int k = static_cast<int>(K);
  // H = L L^T; H^-1 (lower) = potri; H^-1 = L2 L2^T.  Column k of L2 (col-major, contiguous from
  // element k*K) is row k of U = L2^T, so the buffer read row-major IS the upper factor U.
  const bool ok = cusolverDnDpotrf(hs, CUBLAS_FILL_MODE_LOWER, k, st->U, k, work, lwork, info) ==
                      CUSOLVER_STATUS_SUCCESS &&
                  cusolverDnDpotri(hs, CUBLAS_FILL_MODE_LOWER, k, st->U, k, work, lwork, info + 1) ==
                      CUSOLVER_STATUS_SUCCESS &&
                  cusolverDnDpotrf(hs, CUBLAS_FILL_MODE_LOWER, k, st->U, k, work, lwork, info + 2) ==
                      CUSOLVER_STATUS_SUCCESS;
  cusolverDnDestroy(hs);
  if (!ok) return "Cholesky of H^-1";
  int h_info[3] = {0, 0, 0};
  if (cudaMemcpyAsync(h_info, info, sizeof(h_info), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return "info readback";
  if (h_info[0] != 0 || h_info[1] != 0 || h_info[2] != 0) return "H not positive definite after dampening";
  return nullptr;
}

cudaError_t gptq_zero_dead(double *R, const GptqState &st, int64_t K, int64_t N, cudaStream_t s) {
  zero_dead_rows_kernel<<<blocks_for(K * N), 256, 0, s>>>(R, st.dead, K, N);
  return cudaGetLastError();
}

const char *gptq_run(double *R, const GptqState &st, int64_t K, int64_t N, int fmt, bool scale_bf16, float gs,
                     const float *w8_scales, uint8_t *codes, uint8_t *scales, cudaStream_t s) {
  const size_t smem = (kB * kB + kB * kThreads) * sizeof(double);
  static bool attr_set[64];                  // per device ordinal: the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaFuncSetAttribute(gptq_block_kernel<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gptq_block_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gptq_block_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gptq_block_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cublasHandle_t hb = nullptr;
  if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) return "cublasCreate";
  cublasSetStream(hb, s);
  cublasSetMathMode(hb, CUBLAS_PEDANTIC_MATH);
  const dim3 grid(static_cast<unsigned>((N + kThreads - 1) / kThreads));
  const double mone = -1.0, one = 1.0;
  const char *err = nullptr;
  for (int64_t i1 = 0; i1 < K && !err; i1 += kB) {
    if (fmt == 0)
      gptq_block_kernel<0, true><<<grid, kThreads, smem, s>>>(R, st.U, K, N, i1, gs, w8_scales, codes, scales, st.E);
    else if (fmt == 1 && scale_bf16)
      gptq_block_kernel<1, true><<<grid, kThreads, smem, s>>>(R, st.U, K, N, i1, gs, w8_scales, codes, scales, st.E);
    else if (fmt == 1)
      gptq_block_kernel<1, false><<<grid, kThreads, smem, s>>>(R, st.U, K, N, i1, gs, w8_scales, codes, scales, st.E);
    else
      gptq_block_kernel<2, true><<<grid, kThreads, smem, s>>>(R, st.U, K, N, i1, gs, w8_scales, codes, scales, st.E);
    if (cudaGetLastError() != cudaSuccess) {
      err = "gptq block kernel";
      break;
    }
    const int64_t i2 = i1 + kB;
    if (i2 >= K) break;
    // R[i2:, :] -= U[i1:i2, i2:]^T E.  Column-major views: R -> Rc (N x K), E -> Ec (N x kB),
    // U row-major -> Uc = U^T; M1 = Uc[i2:, i1:i2] ((K - i2) x kB) holds U[i1 + b, i2 + k'].
    // Rc[:, i2:] -= Ec M1^T
    if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, static_cast<int>(N), static_cast<int>(K - i2), kB, &mone, st.E,
                    static_cast<int>(N), st.U + i2 + i1 * K, static_cast<int>(K), &one, R + i2 * N,
                    static_cast<int>(N)) != CUBLAS_STATUS_SUCCESS)
      err = "trailing update";
  }
  cublasDestroy(hb);
  return err;
}

}  // namespace svdq
