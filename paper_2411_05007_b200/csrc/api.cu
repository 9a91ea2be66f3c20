// api.cu -- the extern "C" boundary declared in include/svdq.h: host-side
// validation, TMA descriptor construction, dispatch, error reporting.
#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/svdq.h"
#include "formats.cuh"
#include "gptq.h"
#include "k1_launch.h"

using namespace svdq;

namespace {

thread_local char g_err[512] = "";
thread_local uint64_t g_launches = 0;

svdq_status fail(svdq_status s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

svdq_status cuda_fail(cudaError_t e, const char *where) {
  return fail(SVDQ_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define SVDQ_CUDA(call, where)                         \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

svdq_status check_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SVDQ_ERR_UNSUPPORTED, "no CUDA device");
  static int cached[64];   // 0 unknown, 1 ok, 2 bad
  if (dev < 64 && cached[dev] == 1) return SVDQ_OK;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(SVDQ_ERR_UNSUPPORTED, "device %d is sm_%d%d; libsvdq is built for sm_100a", dev,
                major, minor);
  if (dev < 64) cached[dev] = 1;
  return SVDQ_OK;
}

int64_t sf_bytes(int64_t rows, int64_t K) { return ((rows + 127) / 128) * 128 * (K / 16); }

svdq_status check_linear(const svdq_linear *L, bool need_weights) {
  if (!L) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null svdq_linear");
  if (L->fmt != SVDQ_FMT_NVFP4 && L->fmt != SVDQ_FMT_INT4 && L->fmt != SVDQ_FMT_W8A8)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad format %d", L->fmt);
  if (L->K <= 0 || L->K % 64) return fail(SVDQ_ERR_SHAPE, "K=%lld must be a positive multiple of 64", (long long)L->K);
  if (L->N <= 0 || L->N % 16) return fail(SVDQ_ERR_SHAPE, "N=%lld must be a positive multiple of 16", (long long)L->N);
  if (L->rank < 0 || L->rank > 128 || L->rank % 16)
    return fail(SVDQ_ERR_RANK, "rank=%d must be a multiple of 16 in [0, 128]", L->rank);
  if (L->fmt == SVDQ_FMT_INT4 && L->scale_dtype != SVDQ_BF16 && L->scale_dtype != SVDQ_FP16)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "INT4 scale_dtype must be BF16 or FP16");
  if (L->fmt == SVDQ_FMT_NVFP4 && !(L->gs_x > 0.f))
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "gs_x must be > 0");
  if (!L->lambda_inv) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null lambda_inv");
  if (L->rank > 0 && (!L->l1s || !L->l2s)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null l1s/l2s with rank > 0");
  if (!aligned16(L->lambda_inv) || !aligned16(L->l1s) || !aligned16(L->l2s))
    return fail(SVDQ_ERR_ALIGNMENT, "lambda_inv / l1s / l2s must be 16-byte aligned");
  if (need_weights) {
    if (!L->w_codes || !L->w_scales) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null weight codes/scales");
    if (!aligned16(L->w_codes) || !aligned16(L->w_scales))
      return fail(SVDQ_ERR_ALIGNMENT, "weight codes/scales must be 16-byte aligned");
    if (L->bias && L->bias_dtype != SVDQ_BF16 && L->bias_dtype != SVDQ_FP16 && L->bias_dtype != SVDQ_FP32)
      return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad bias dtype");
    if (L->fmt == SVDQ_FMT_NVFP4 && !(L->gs_w > 0.f))
      return fail(SVDQ_ERR_INVALID_ARGUMENT, "gs_w must be > 0");
  }
  return SVDQ_OK;
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D row-major tensor [rows][cols] of `dt`, row pitch `pitch_bytes`, box {box_cols, box_rows},
// 128-byte swizzle.
svdq_status make_map(CUtensorMap *map, const void *base, CUtensorMapDataType dt, int64_t cols,
                     int64_t rows, int64_t pitch_bytes, uint32_t box_cols, uint32_t box_rows,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return fail(SVDQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch_bytes)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SVDQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SVDQ_OK;
}

// 3-D view of a row-major 16-bit activation X [rows][ldx]: {64 cols, rows, K/64 blocks}, box
// {64, rt, q}, 128-byte swizzle: the row-tile K1's stage, block-major (staged row q rt + m).
svdq_status make_x3_map(CUtensorMap *map, const void *base, CUtensorMapDataType dt, int64_t K, int64_t rows,
                        int64_t ldx_bytes, uint32_t q, uint32_t rt) {
  auto fn = encode_fn();
  if (!fn) return fail(SVDQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(K / 64)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldx_bytes), 128};
  cuuint32_t box[3] = {64, rt, q};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dt, 3, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SVDQ_ERR_CUDA, "cuTensorMapEncodeTiled (X 3-D) failed (%d)", (int)r);
  return SVDQ_OK;
}

// 3-D uint64 view of a 128x4 scale-factor buffer: [rows/128][K/64][512 B], box {64, 4, atoms}.
svdq_status make_sf_map(CUtensorMap *map, const void *base, int64_t rows, int64_t K, uint32_t atoms) {
  auto fn = encode_fn();
  if (!fn) return fail(SVDQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t nkb = K / 64;
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(nkb), static_cast<cuuint64_t>((rows + 127) / 128)};
  cuuint64_t strides[2] = {512, static_cast<cuuint64_t>(nkb * 512)};
  cuuint32_t box[3] = {64, 4, atoms};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SVDQ_ERR_CUDA, "cuTensorMapEncodeTiled (sf) failed (%d)", (int)r);
  return SVDQ_OK;
}

// W8A8: the CTA-pair kernel unless the problem is small.  SVDQ_K2_PAIR=0 / 1 forces one kernel
// (testing / comparison).
int pair_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char *e = getenv("SVDQ_K2_PAIR");
    mode = e ? atoi(e) : 2;
  }
  return mode;
}
bool use_pair_kernel(int64_t M, int64_t K) {
  if (M <= 128 || pair_mode() == 0) return false;
  return pair_mode() == 1 || K >= 6144 || M >= 1024;
}

// NVFP4 tile plan of one (non-grouped) K2 launch: the CTA-pair kernel (256 x 256 / 256 x 192 tiles,
// 74 pairs) or the 1-CTA kernel (128 x 192 / 128 x 128, 148 SMs), whichever leaves the least
// per-SM work in its last wave -- cost = waves x (tile columns per SM), the 1-CTA kernel weighted
// 1.1 (its SMs each stage all of B: measured 3-15 % slower per tile on C2 / C3 shapes).  Chooses
// the pair kernel on every FLUX layer with M >= 4096 and the 1-CTA 128-wide tile on e.g. PixArt's
// 4096 x 1152 x 1152 (tools/k2_shape_sweep.py).
struct K2Plan {
  bool pair;
  int bn;
};
K2Plan plan_nvfp4(int64_t M, int64_t N) {
  const int64_t sms = svdq::device_sm_count();
  auto waves = [](int64_t tiles, int64_t units) { return (tiles + units - 1) / units; };
  K2Plan best{true, svdq::k2_pair_bn(N)};
  double cbest = 1e30;
  for (int bn : {svdq::k2_pair_bn(N), 192}) {
    const double c = static_cast<double>(waves(((M + 255) / 256) * ((N + bn - 1) / bn), sms / 2) * bn);
    if (c < cbest) { cbest = c; best = K2Plan{true, bn}; }
  }
  if (pair_mode() == 1) return best;
  const int bn1 = svdq::k2_nvfp4_bn(M, N);
  const double c1 = 1.1 * static_cast<double>(waves(((M + 127) / 128) * ((N + bn1 - 1) / bn1), sms) * bn1);
  if (M <= 128 || pair_mode() == 0 || c1 < cbest) return K2Plan{false, bn1};
  return best;
}

}  // namespace

namespace svdq {
// Error reporting for the library's other translation units (offline.cu).
svdq_status report_error(svdq_status s, const char *msg) { return fail(s, "%s", msg); }
}  // namespace svdq

extern "C" {

const char *svdq_status_string(svdq_status s) {
  switch (s) {
    case SVDQ_OK: return "SVDQ_OK";
    case SVDQ_ERR_INVALID_ARGUMENT: return "SVDQ_ERR_INVALID_ARGUMENT";
    case SVDQ_ERR_SHAPE: return "SVDQ_ERR_SHAPE";
    case SVDQ_ERR_RANK: return "SVDQ_ERR_RANK";
    case SVDQ_ERR_ALIGNMENT: return "SVDQ_ERR_ALIGNMENT";
    case SVDQ_ERR_UNSUPPORTED: return "SVDQ_ERR_UNSUPPORTED";
    case SVDQ_ERR_NONFINITE: return "SVDQ_ERR_NONFINITE";
    case SVDQ_ERR_CUDA: return "SVDQ_ERR_CUDA";
    case SVDQ_ERR_WORKSPACE: return "SVDQ_ERR_WORKSPACE";
  }
  return "SVDQ_ERR_UNKNOWN";
}

const char *svdq_last_error(void) { return g_err; }
uint64_t svdq_launch_count(void) { return g_launches; }
int32_t svdq_version(void) { return 2; }
int32_t svdq_k1_row_tile(int64_t rows_padded, int32_t rank) { return k1_rows_rt(rows_padded, rank); }

svdq_status svdq_act_buffer_sizes(int32_t fmt, int64_t M, int64_t K, int32_t rank, size_t *xq,
                                  size_t *xs, size_t *xl1) {
  if (!xq || !xs || !xl1) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (fmt != SVDQ_FMT_NVFP4 && fmt != SVDQ_FMT_INT4 && fmt != SVDQ_FMT_W8A8)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad format");
  if (M < 1) return fail(SVDQ_ERR_SHAPE, "M must be >= 1");
  if (K <= 0 || K % 64) return fail(SVDQ_ERR_SHAPE, "K must be a positive multiple of 64");
  if (rank < 0 || rank > 128 || rank % 16) return fail(SVDQ_ERR_RANK, "bad rank");
  if (fmt == SVDQ_FMT_W8A8) {
    *xq = static_cast<size_t>(M * K);                                     // int8 codes [M][K]
    *xs = static_cast<size_t>(M * 4);                                     // fp32 per-token scales [M]
    *xl1 = static_cast<size_t>(M) * rank * 2;
    return SVDQ_OK;
  }
  *xq = static_cast<size_t>(M * K / 2);
  *xs = fmt == SVDQ_FMT_NVFP4 ? static_cast<size_t>(sf_bytes(M, K)) : static_cast<size_t>(M * (K / 64) * 2);
  *xl1 = static_cast<size_t>(M) * rank * 2;
  return SVDQ_OK;
}

svdq_status svdq_weight_buffer_sizes(int32_t fmt, int64_t K, int64_t N, int32_t rank, size_t *codes,
                                     size_t *scales, size_t *l1s, size_t *l2s) {
  if (!codes || !scales || !l1s || !l2s) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (fmt != SVDQ_FMT_NVFP4 && fmt != SVDQ_FMT_INT4 && fmt != SVDQ_FMT_W8A8)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad format");
  if (K <= 0 || K % 64) return fail(SVDQ_ERR_SHAPE, "K must be a positive multiple of 64");
  if (N <= 0 || N % 16) return fail(SVDQ_ERR_SHAPE, "N must be a positive multiple of 16");
  if (rank < 0 || rank > 128 || rank % 16) return fail(SVDQ_ERR_RANK, "bad rank");
  *codes = static_cast<size_t>(fmt == SVDQ_FMT_W8A8 ? N * K : N * K / 2);
  *scales = fmt == SVDQ_FMT_NVFP4 ? static_cast<size_t>(sf_bytes(N, K))
            : fmt == SVDQ_FMT_W8A8 ? static_cast<size_t>(N * 4)
                                   : static_cast<size_t>(N * (K / 64) * 2);
  *l1s = static_cast<size_t>(rank) * K * 2;
  *l2s = static_cast<size_t>(N) * rank * 2;
  return SVDQ_OK;
}

}  // extern "C"

namespace {
// Validation, launch parameters and tensor maps of one K1 problem (`out` may alias maps->p).
svdq_status prepare_k1(const svdq_linear *L, const void *X, int32_t x_dtype, int64_t M, int64_t ldx, uint8_t *xq,
                       uint8_t *xs, uint16_t *xl1, K1Params *out, K1Problem *maps, int rt,
                       int64_t l1s_pitch = 0) {
  svdq_status st = check_linear(L, false);
  if (st != SVDQ_OK) return st;
  if (!X || !xq || !xs || (L->rank > 0 && !xl1)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (x_dtype != SVDQ_BF16 && x_dtype != SVDQ_FP16)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "X dtype must be BF16 or FP16");
  if (M < 1) return fail(SVDQ_ERR_SHAPE, "M must be >= 1");
  if (ldx < L->K) return fail(SVDQ_ERR_SHAPE, "ldx < K");
  if (ldx % 8 || !aligned16(X) || !aligned16(xq) || !aligned16(xs) || (xl1 && !aligned16(xl1)))
    return fail(SVDQ_ERR_ALIGNMENT, "X / ldx / outputs must be 16-byte aligned");
  if ((st = check_device()) != SVDQ_OK) return st;
  K1Params &p = *out;
  p = K1Params{};
  p.fmt = L->fmt == SVDQ_FMT_NVFP4 ? 0 : (L->fmt == SVDQ_FMT_W8A8 ? 2 : 1);
  p.x_bf16 = x_dtype == SVDQ_BF16;
  p.scale_bf16 = L->scale_dtype == SVDQ_BF16;
  p.X = X;
  p.ldx = ldx;
  p.M = M;
  p.Mpad = ((M + 127) / 128) * 128;
  p.K = L->K;
  p.lam_inv = L->lambda_inv;
  p.l1s = L->l1s;
  p.rank = L->rank;
  p.gs_x = L->fmt == SVDQ_FMT_NVFP4 ? L->gs_x : 1.0f;
  p.xq = xq;
  p.xs = xs;
  p.xl1 = xl1;
  p.ndst = 1;
  p.out_k = p.K;
  p.out_c0 = 0;
  std::memset(&maps->x, 0, sizeof(maps->x));
  std::memset(&maps->l1s, 0, sizeof(maps->l1s));
  std::memset(&maps->lam, 0, sizeof(maps->lam));
  // row-tile kernel (k1_rows.cu): X boxes {64, 128/rt blocks, rt rows}, L1s tiles [rank x 64],
  // lambda_inv rows of 32 fp32 (two per 64-wide block), all 128-B swizzled
  const uint32_t q = static_cast<uint32_t>(128 / rt);
  if ((st = make_x3_map(&maps->x, X, p.x_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                        L->K, M, ldx * 2, q, static_cast<uint32_t>(rt))) != SVDQ_OK)
    return st;
  if (L->rank > 0 &&
      (st = make_map(&maps->l1s, L->l1s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, L->K, L->rank,
                     (l1s_pitch > 0 ? l1s_pitch : L->K) * 2, 64, static_cast<uint32_t>(L->rank))) != SVDQ_OK)
    return st;
  if ((st = make_map(&maps->lam, L->lambda_inv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 32, L->K / 32, 128, 32, 2 * q)) !=
      SVDQ_OK)
    return st;
  return SVDQ_OK;
}
}  // namespace

extern "C" {

svdq_status svdq_quantize_act_lowrank_down(const svdq_linear *L, const void *X, int32_t x_dtype,
                                           int64_t M, int64_t ldx, uint8_t *xq, uint8_t *xs,
                                           uint16_t *xl1, void *stream) {
  K1Args g;
  std::memset(&g, 0, sizeof(g));
  g.n = 1;
  const int rt = k1_rows_rt(((M + 127) / 128) * 128, L ? L->rank : 0);
  svdq_status st = prepare_k1(L, X, x_dtype, M, ldx, xq, xs, xl1, &g.pr[0].p, &g.pr[0], rt);
  if (st != SVDQ_OK) return st;
  const K1Params &p = g.pr[0].p;
  cudaError_t e = cudaSuccess;
  if (p.fmt != 2 || p.rank > 0) {      // W8A8: the row-tile kernel runs the down-projection only
    e = launch_k1_rows_group(g, rt, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "K1 launch");
    ++g_launches;
  }
  if (p.fmt == 2) {                    // per-token INT8 codes + fp32 scales
    K1Params p8 = p;
    p8.w8_amax = p.rank > 0 ? 1 : 0;   // the row-tile kernel above left each row's amax in xs
    e = launch_k1_int8_rows(p8, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "K1 (int8 rows) launch");
    ++g_launches;
  }
  return SVDQ_OK;
}

svdq_status svdq_quantize_act_lowrank_down_grouped(int32_t n, const svdq_linear *const *layers,
                                                   const void *const *X, int32_t x_dtype, const int64_t *M,
                                                   const int64_t *ldx, uint8_t *const *xq, uint8_t *const *xs,
                                                   uint16_t *const *xl1, void *stream) {
  if (n < 1 || n > kMaxGroup1) return fail(SVDQ_ERR_INVALID_ARGUMENT, "group size must be 1..%d", kMaxGroup1);
  if (!layers || !X || !M || !ldx || !xq || !xs || !xl1) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null array");
  for (int i = 0; i < n; ++i)
    if (layers[i] && layers[i]->fmt == SVDQ_FMT_W8A8) return fail(SVDQ_ERR_UNSUPPORTED, "grouped K1: no W8A8");
  K1Args g;
  std::memset(&g, 0, sizeof(g));
  g.n = n;
  int64_t rows_total = 0;
  for (int i = 0; i < n; ++i) rows_total += ((M[i] + 127) / 128) * 128;
  const int rt = k1_rows_rt(rows_total, layers[0] ? layers[0]->rank : 0);
  for (int i = 0; i < n; ++i) {
    if (!layers[i]) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null layer %d", i);
    if (layers[i]->fmt != layers[0]->fmt || layers[i]->rank != layers[0]->rank ||
        (layers[i]->fmt == SVDQ_FMT_INT4 && layers[i]->scale_dtype != layers[0]->scale_dtype))
      return fail(SVDQ_ERR_UNSUPPORTED, "grouped K1: layers must share format, rank and scale dtype");
    svdq_status st = prepare_k1(layers[i], X[i], x_dtype, M[i], ldx[i], xq[i], xs[i], xl1[i], &g.pr[i].p, &g.pr[i], rt);
    if (st != SVDQ_OK) return st;
  }
  cudaError_t e = launch_k1_rows_group(g, rt, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "grouped K1 launch");
  ++g_launches;
  return SVDQ_OK;
}

svdq_status svdq_tp_slice_sizes(int32_t fmt, int64_t M, int64_t Kp, int32_t rank, size_t *xq_off, size_t *xs_off,
                                size_t *part_off, size_t *slice_bytes) {
  if (!xq_off || !xs_off || !part_off || !slice_bytes) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (fmt != SVDQ_FMT_NVFP4 && fmt != SVDQ_FMT_INT4)
    return fail(fmt == SVDQ_FMT_W8A8 ? SVDQ_ERR_UNSUPPORTED : SVDQ_ERR_INVALID_ARGUMENT,
                "K-sliced K1 needs NVFP4 or INT4 (W8A8 per-token scales need the whole row)");
  if (M < 1) return fail(SVDQ_ERR_SHAPE, "M must be >= 1");
  if (Kp <= 0 || Kp % 64) return fail(SVDQ_ERR_SHAPE, "slice width must be a positive multiple of 64");
  if (rank < 0 || rank > 128 || rank % 16) return fail(SVDQ_ERR_RANK, "bad rank");
  const TpSliceLayout L = tp_slice_layout(fmt, M, Kp, rank);
  *xq_off = static_cast<size_t>(L.xq_off);
  *xs_off = static_cast<size_t>(L.xs_off);
  *part_off = static_cast<size_t>(L.part_off);
  *slice_bytes = static_cast<size_t>(L.bytes);
  return SVDQ_OK;
}

svdq_status svdq_tp_gather_sizes(int32_t fmt, int64_t M, int64_t K, int32_t rank, int32_t P, size_t *xq_off,
                                 size_t *xs_off, size_t *part_off, size_t *bytes) {
  if (!xq_off || !xs_off || !part_off || !bytes) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (P < 1) return fail(SVDQ_ERR_INVALID_ARGUMENT, "P must be >= 1");
  size_t bq, bs, bl;
  svdq_status st = svdq_act_buffer_sizes(fmt, M, K, rank, &bq, &bs, &bl);
  if (st != SVDQ_OK) return st;
  if (fmt == SVDQ_FMT_W8A8) return fail(SVDQ_ERR_UNSUPPORTED, "K-sliced K1: no W8A8 (per-token scales need the whole row)");
  auto up = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  *xq_off = 0;
  *xs_off = up(bq);
  *part_off = *xs_off + up(bs);
  *bytes = *part_off + up(static_cast<size_t>(P) * M * rank * 4);
  return SVDQ_OK;
}

namespace {
// K1 of L restricted to input channels [k0, k0 + Kp): validation, the restricted view, launch.
svdq_status kslice_launch(const svdq_linear *L, int64_t k0, int64_t Kp, const void *X, int32_t x_dtype, int64_t M,
                          int64_t ldx, uint8_t *xq, uint8_t *xs, float *part, int64_t out_k, int64_t out_c0,
                          const int64_t *delta, int ndst, void *stream) {
  if (k0 < 0 || k0 % 64 || Kp <= 0 || Kp % 64 || k0 + Kp > L->K)
    return fail(SVDQ_ERR_SHAPE, "K-slice [%lld, %lld) must be 64-aligned inside [0, K)", (long long)k0,
                (long long)(k0 + Kp));
  if (L->fmt == SVDQ_FMT_W8A8) return fail(SVDQ_ERR_UNSUPPORTED, "K-sliced K1: no W8A8 (per-token scales)");
  svdq_linear V = *L;                        // the layer restricted to input channels [k0, k0 + Kp)
  V.K = Kp;
  V.lambda_inv = L->lambda_inv + k0;
  V.l1s = L->rank ? L->l1s + k0 : L->l1s;
  K1Args g;
  std::memset(&g, 0, sizeof(g));
  g.n = 1;
  const int rt = k1_rows_rt(((M + 127) / 128) * 128, L->rank);
  svdq_status st = prepare_k1(&V, X, x_dtype, M, ldx, xq, xs, reinterpret_cast<uint16_t *>(part), &g.pr[0].p,
                              &g.pr[0], rt, L->K);
  if (st != SVDQ_OK) return st;
  K1Params &p = g.pr[0].p;
  p.xl1 = nullptr;
  p.xl1_f32 = L->rank ? part : nullptr;
  p.out_k = out_k;
  p.out_c0 = out_c0;
  p.ndst = ndst;
  for (int j = 0; j < ndst; ++j) p.dst_delta[j] = delta[j];
  cudaError_t e = launch_k1_rows_group(g, rt, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "K-sliced K1 launch");
  ++g_launches;
  return SVDQ_OK;
}
}  // namespace

svdq_status svdq_quantize_act_lowrank_down_kslice(const svdq_linear *L, int64_t k0, int64_t Kp, const void *X,
                                                  int32_t x_dtype, int64_t M, int64_t ldx, uint8_t *slice,
                                                  void *stream) {
  svdq_status st = check_linear(L, false);
  if (st != SVDQ_OK) return st;
  size_t oq, os, op, nb;
  if ((st = svdq_tp_slice_sizes(L->fmt, M, Kp, L->rank, &oq, &os, &op, &nb)) != SVDQ_OK) return st;
  if (!slice) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null slice buffer");
  if (!aligned16(slice)) return fail(SVDQ_ERR_ALIGNMENT, "slice buffer must be 16-byte aligned");
  const int64_t zero = 0;
  return kslice_launch(L, k0, Kp, X, x_dtype, M, ldx, slice + oq, slice + os, reinterpret_cast<float *>(slice + op),
                       Kp, 0, &zero, 1, stream);
}

svdq_status svdq_quantize_act_lowrank_down_kslice_fused(const svdq_linear *L, int64_t k0, int64_t Kp, const void *X,
                                                        int32_t x_dtype, int64_t M, int64_t ldx, int32_t P,
                                                        int32_t p, uint8_t *const *bufs, int32_t nbuf,
                                                        void *stream) {
  svdq_status st = check_linear(L, false);
  if (st != SVDQ_OK) return st;
  if (!bufs || nbuf < 1 || nbuf > 8) return fail(SVDQ_ERR_INVALID_ARGUMENT, "nbuf must be 1..8");
  if (p < 0 || p >= P) return fail(SVDQ_ERR_INVALID_ARGUMENT, "slot %d outside [0, %d)", p, P);
  for (int j = 0; j < nbuf; ++j) {
    if (!bufs[j]) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null gather buffer %d", j);
    if (!aligned16(bufs[j])) return fail(SVDQ_ERR_ALIGNMENT, "gather buffer %d must be 16-byte aligned", j);
  }
  size_t oq, os, op, nb;
  if ((st = svdq_tp_gather_sizes(L->fmt, M, L->K, L->rank, P, &oq, &os, &op, &nb)) != SVDQ_OK) return st;
  int64_t delta[8];
  for (int j = 0; j < nbuf; ++j) delta[j] = bufs[j] - bufs[0];
  uint8_t *b = bufs[0];
  // codes: column k0 of the [M][K/2] rows (the kernel adds row * K/2); scales: group k0/16 of the
  // full-K layout (out_c0); partial: slot p
  return kslice_launch(L, k0, Kp, X, x_dtype, M, ldx, b + oq + k0 / 2, b + os,
                       reinterpret_cast<float *>(b + op) + static_cast<int64_t>(p) * M * L->rank, L->K, k0 / 16,
                       delta, nbuf, stream);
}

svdq_status svdq_tp_reduce_partials(int32_t P, int64_t M, int32_t rank, const float *parts, uint16_t *xl1,
                                    void *stream) {
  if (P < 1 || M < 1 || rank < 1 || rank > 128 || rank % 16) return fail(SVDQ_ERR_SHAPE, "bad P / M / rank");
  if (!parts || !xl1) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null buffer");
  svdq_status st = check_device();
  if (st != SVDQ_OK) return st;
  cudaError_t e = launch_tp_reduce_partials(P, M, rank, parts, xl1, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "TP partial reduction launch");
  ++g_launches;
  return SVDQ_OK;
}

svdq_status svdq_tp_assemble_act(int32_t fmt, int32_t P, int64_t M, int64_t K, int32_t rank, const uint8_t *gathered,
                                 size_t slice_bytes, size_t slice_stride, uint8_t *xq, uint8_t *xs, uint16_t *xl1,
                                 void *stream) {
  if (P < 1) return fail(SVDQ_ERR_INVALID_ARGUMENT, "P must be >= 1");
  if (K <= 0 || K % (64 * static_cast<int64_t>(P))) return fail(SVDQ_ERR_SHAPE, "K must be a multiple of 64 P");
  size_t oq, os, op, nb;
  svdq_status st = svdq_tp_slice_sizes(fmt, M, K / P, rank, &oq, &os, &op, &nb);
  if (st != SVDQ_OK) return st;
  if (slice_bytes != nb) return fail(SVDQ_ERR_SHAPE, "slice_bytes %zu != %zu", slice_bytes, nb);
  if (slice_stride == 0) slice_stride = slice_bytes;
  if (slice_stride < slice_bytes || slice_stride % 16) return fail(SVDQ_ERR_SHAPE, "bad slice_stride %zu", slice_stride);
  if (!gathered || !xq || !xs || (rank && !xl1)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (!aligned16(gathered) || !aligned16(xq) || !aligned16(xs)) return fail(SVDQ_ERR_ALIGNMENT, "buffers must be 16-byte aligned");
  if ((st = check_device()) != SVDQ_OK) return st;
  cudaError_t e = launch_tp_assemble(fmt, P, M, K, rank, gathered, static_cast<int64_t>(slice_stride), xq, xs, xl1,
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "TP assemble launch");
  ++g_launches;
  return SVDQ_OK;
}

}  // extern "C"

namespace {
// Validation, launch parameters and tensor maps of one K2 problem.  `force_pair` selects the
// CTA-pair NVFP4 kernel regardless of shape (grouped launches run every problem on it).
struct K2Prep {
  K2Params p;
  K2Maps maps;
  CUtensorMap sfa_map, sfb_map;
  bool pair;
  int bn;                  // pair tile N (192 / 256) when `pair`
};
svdq_status prepare_k2(const svdq_linear *L, const uint8_t *xq, const uint8_t *xs, const uint16_t *xl1, int64_t M,
                       void *Y, int32_t y_dtype, int64_t ldy, bool force_pair, K2Prep *out, void *y_map_base = nullptr,
                       int pair_bn = 0) {
  svdq_status st = check_linear(L, true);
  if (st != SVDQ_OK) return st;
  if (!Y && y_map_base) Y = y_map_base;     // fused launch without a Y store: the map is never used
  if (!xq || !xs || !Y || (L->rank > 0 && !xl1)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null buffer");
  if (y_dtype != SVDQ_BF16 && y_dtype != SVDQ_FP16 && y_dtype != SVDQ_FP32)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad Y dtype");
  if (M < 1) return fail(SVDQ_ERR_SHAPE, "M must be >= 1");
  if (ldy < L->N) return fail(SVDQ_ERR_SHAPE, "ldy < N");
  if (ldy % 8 || !aligned16(Y) || !aligned16(xq) || !aligned16(xs) || (xl1 && !aligned16(xl1)))
    return fail(SVDQ_ERR_ALIGNMENT, "Y / ldy / inputs must be 16-byte aligned");
  if ((st = check_device()) != SVDQ_OK) return st;
  const int64_t K = L->K, N = L->N;
  K2Params &p = out->p;
  p = K2Params{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.Npad = ((N + 127) / 128) * 128;
  p.rank = L->rank;
  p.sfa = xs;
  p.sfb = L->w_scales;
  p.xq = xq;
  p.wq = L->w_codes;
  p.bias = L->bias;
  p.bias_dtype = L->bias_dtype;
  p.Y = Y;
  p.y_dtype = y_dtype;
  p.ldy = ldy;
  p.scale_bf16 = L->scale_dtype == SVDQ_BF16;
  p.alpha = L->fmt == SVDQ_FMT_NVFP4 ? L->gs_x * L->gs_w : 1.0f;
  p.w8 = L->fmt == SVDQ_FMT_W8A8;
  K2Maps &maps = out->maps;
  std::memset(&maps, 0, sizeof(maps));
  // CTA-pair kernel: NVFP4, and W8A8 (its kind::i8 mode, 192-wide tiles)
  const K2Plan plan = L->fmt == SVDQ_FMT_NVFP4 && !force_pair ? plan_nvfp4(M, N) : K2Plan{true, 0};
  const bool pair = L->fmt == SVDQ_FMT_NVFP4 ? (force_pair || plan.pair)
                                             : (L->fmt == SVDQ_FMT_W8A8 && (force_pair || use_pair_kernel(M, K)));
  out->pair = pair;
  // pair tile N: the caller's (grouped / fused launches share one) or this problem's own plan
  out->bn = !pair ? 0 : L->fmt == SVDQ_FMT_W8A8 ? 192 : (pair_bn ? pair_bn : (plan.bn ? plan.bn : k2_pair_bn(N)));
  const int BN = pair ? out->bn : L->fmt == SVDQ_FMT_NVFP4 ? k2_nvfp4_bn(M, N) : kInt4BN;
  std::memset(&out->sfa_map, 0, sizeof(out->sfa_map));
  std::memset(&out->sfb_map, 0, sizeof(out->sfb_map));
  // rows per B-side TMA box: the CTA's BN / 2 rows in one box, or three 64-row boxes at BN = 384
  const uint32_t b_rows = pair ? static_cast<uint32_t>(BN == 384 ? 64 : BN / 2) : static_cast<uint32_t>(BN);
  CUtensorMap &sfa_map = out->sfa_map, &sfb_map = out->sfb_map;
  const CUtensorMapDataType ydt = y_dtype == SVDQ_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                  : y_dtype == SVDQ_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const int64_t ysz = y_dtype == SVDQ_FP32 ? 4 : 2;
  if (L->fmt == SVDQ_FMT_NVFP4) {
#ifndef SVDQ_BIGSTORE
#define SVDQ_BIGSTORE 0
#endif
    if (SVDQ_BIGSTORE && pair && y_dtype != SVDQ_FP32) {      // [128 rows x 64 cols] SW128 blocks
      if ((st = make_map(&maps.y, Y, ydt, N, M, ldy * ysz, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)) != SVDQ_OK)
        return st;
    } else if ((st = make_map(&maps.y, Y, ydt, N, M, ldy * ysz, static_cast<uint32_t>(64 / ysz), 32,
                              CU_TENSOR_MAP_SWIZZLE_64B)) != SVDQ_OK) {
      return st;
    }
    if ((st = make_map(&maps.a, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, K / 2, M, K / 2, 128, 128)) != SVDQ_OK) return st;
    if ((st = make_map(&maps.b, L->w_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, K / 2, N, K / 2, 128, b_rows)) != SVDQ_OK) return st;
    if (pair) {
      if ((st = make_sf_map(&sfa_map, xs, M, K, 1)) != SVDQ_OK) return st;
      if ((st = make_sf_map(&sfb_map, L->w_scales, N, K, BN == 384 ? 3 : 2)) != SVDQ_OK) return st;
    }
  } else if (L->fmt == SVDQ_FMT_W8A8) {
    // int8 tiles [rows x 128 B], 128-B swizzle: straight into the kind::i8 operand ring
    if ((st = make_map(&maps.a, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, M, K, 128, 128)) != SVDQ_OK) return st;
    if ((st = make_map(&maps.b, L->w_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, N, K, 128, b_rows)) != SVDQ_OK) return st;
    if (pair && (st = make_map(&maps.y, Y, ydt, N, M, ldy * ysz, static_cast<uint32_t>(64 / ysz), 32,
                               CU_TENSOR_MAP_SWIZZLE_64B)) != SVDQ_OK)
      return st;
  } else {
    // packed int4 tiles [rows x 64 B] (two K groups), dense (no swizzle): unpacked in smem
    if ((st = make_map(&maps.a, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, K / 2, M, K / 2, 64, 128,
                       CU_TENSOR_MAP_SWIZZLE_NONE)) != SVDQ_OK) return st;
    if ((st = make_map(&maps.b, L->w_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, K / 2, N, K / 2, 64, BN,
                       CU_TENSOR_MAP_SWIZZLE_NONE)) != SVDQ_OK) return st;
  }
  if (L->rank > 0) {
    if ((st = make_map(&maps.xl1, xl1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, L->rank, M, L->rank * 2, 64, 128)) != SVDQ_OK) return st;
    if ((st = make_map(&maps.l2, L->l2s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, L->rank, N, L->rank * 2, 64, b_rows)) != SVDQ_OK) return st;
  }
  return SVDQ_OK;
}
}  // namespace

extern "C" {

svdq_status svdq_gemm_w4a4_lowrank_up(const svdq_linear *L, const uint8_t *xq, const uint8_t *xs,
                                      const uint16_t *xl1, int64_t M, void *Y, int32_t y_dtype,
                                      int64_t ldy, void *stream) {
  K2Prep k;
  svdq_status st = prepare_k2(L, xq, xs, xl1, M, Y, y_dtype, ldy, false, &k);
  if (st != SVDQ_OK) return st;
  cudaError_t e = k.pair ? launch_k2_nvfp4_2sm(k.maps, k.sfa_map, k.sfb_map, k.p, k.bn, static_cast<cudaStream_t>(stream))
                  : L->fmt == SVDQ_FMT_NVFP4 ? launch_k2_nvfp4(k.maps, k.p, static_cast<cudaStream_t>(stream))
                                             : launch_k2_int4(k.maps, k.p, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported) return fail(SVDQ_ERR_UNSUPPORTED, "INT4 GEMM not built");
  if (e != cudaSuccess) return cuda_fail(e, "K2 launch");
  ++g_launches;
  return SVDQ_OK;
}

svdq_status svdq_gemm_w4a4_lowrank_up_grouped(int32_t n, const svdq_linear *const *layers,
                                              const uint8_t *const *xq, const uint8_t *const *xs,
                                              const uint16_t *const *xl1, const int64_t *M, void *const *Y,
                                              int32_t y_dtype, const int64_t *ldy, void *stream) {
  if (n < 1 || n > kMaxGroup) return fail(SVDQ_ERR_INVALID_ARGUMENT, "group size must be 1..%d", kMaxGroup);
  if (!layers || !xq || !xs || !xl1 || !M || !Y || !ldy) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null array");
  K2PairArgs g;
  std::memset(&g, 0, sizeof(g));
  g.n = n;
  int cap = 384;                             // one tile shape per launch: the widest every N allows
  for (int i = 0; i < n; ++i) {
    if (!layers[i]) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null layer %d", i);
    if (layers[i]->fmt != SVDQ_FMT_NVFP4) return fail(SVDQ_ERR_UNSUPPORTED, "grouped K2 is NVFP4 only");
    cap = std::min(cap, k2_pair_bn(layers[i]->N));
  }
  int bn = 192;
  for (const int c : {384, 256}) {
    bool ok = c <= cap;
    for (int i = 0; i < n && ok; ++i) ok = layers[i]->N % c == 0;
    if (ok) { bn = c; break; }
  }
  g.bn = bn;
  for (int i = 0; i < n; ++i) {
    K2Prep k;
    svdq_status st = prepare_k2(layers[i], xq[i], xs[i], xl1[i], M[i], Y[i], y_dtype, ldy[i], true, &k, nullptr, bn);
    if (st != SVDQ_OK) return st;
    g.pr[i].a = k.maps.a;
    g.pr[i].b = k.maps.b;
    g.pr[i].xl1 = k.maps.xl1;
    g.pr[i].l2 = k.maps.l2;
    g.pr[i].sfa = k.sfa_map;
    g.pr[i].sfb = k.sfb_map;
    g.pr[i].y = k.maps.y;
    g.pr[i].p = k.p;
  }
  cudaError_t e = launch_k2_nvfp4_2sm_group(g, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "grouped K2 launch");
  ++g_launches;
  return SVDQ_OK;
}

// ---------------------------------------------------------------- layer-boundary fusion
namespace {
// Fill the grouped launch for the fused K2 (validation shared by the workspace query and the call).
svdq_status prepare_fused(int32_t n, const svdq_linear *const *layers, const uint8_t *const *xq,
                          const uint8_t *const *xs, const uint16_t *const *xl1, const int64_t *M, void *const *Y,
                          const svdq_linear *const *nexts, int32_t act, uint8_t *const *xq_next,
                          uint8_t *const *xs_next, K2PairArgs *g, size_t *part_bytes, size_t part_off[]) {
  if (n < 1 || n > kMaxGroup) return fail(SVDQ_ERR_INVALID_ARGUMENT, "group size must be 1..%d", kMaxGroup);
  if (!layers || !nexts || !M) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null array");
  if (act != 0 && act != 1) return fail(SVDQ_ERR_INVALID_ARGUMENT, "act must be 0 (identity) or 1 (GELU tanh)");
  std::memset(g, 0, sizeof(*g));
  g->n = n;
  int64_t tiles = 0;
  for (int i = 0; i < n; ++i) {
    const svdq_linear *L = layers[i], *Nx = nexts[i];
    if (!L || !Nx) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null layer %d", i);
    svdq_status st = check_linear(Nx, true);
    if (st != SVDQ_OK) return st;
    if (L->fmt != SVDQ_FMT_NVFP4 || Nx->fmt != SVDQ_FMT_NVFP4)
      return fail(SVDQ_ERR_UNSUPPORTED, "fused next-layer quantization is NVFP4 -> NVFP4");
    if (Nx->K != L->N) return fail(SVDQ_ERR_SHAPE, "next->K (%lld) != N (%lld)", (long long)Nx->K, (long long)L->N);
    if (Nx->rank != 0 && Nx->rank != 16 && Nx->rank != 32)
      return fail(SVDQ_ERR_RANK, "fused next-layer rank must be 0, 16 or 32");
    if (M[i] < 1) return fail(SVDQ_ERR_SHAPE, "M must be >= 1");
    tiles += ((M[i] + 255) / 256) * ((L->N + kNvfp4PairBN - 1) / kNvfp4PairBN);
  }
  const int np = k2_pair_count(tiles);
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const svdq_linear *Nx = nexts[i];
    const int64_t nt = (layers[i]->N + kNvfp4PairBN - 1) / kNvfp4PairBN;
    const int slots = k2_next_slots(nt, tiles, np);
    part_off[i] = off;
    if (Nx->rank) off += (static_cast<size_t>((M[i] + 255) / 256) * slots * 256 * Nx->rank * 4 + 255) & ~size_t(255);
    K2Params &p = g->pr[i].p;
    p.nx_slots = slots;
  }
  *part_bytes = off;
  if (!xq) return SVDQ_OK;                   // workspace query
  if (!xs || !xl1 || !Y || !xq_next || !xs_next) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null array");
  for (int i = 0; i < n; ++i) {
    const svdq_linear *Nx = nexts[i];
    if (!xq_next[i] || !xs_next[i]) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null next-layer buffer %d", i);
    if (!aligned16(xq_next[i])) return fail(SVDQ_ERR_ALIGNMENT, "xq_next must be 16-byte aligned");
    if (!aligned16(xs_next[i])) return fail(SVDQ_ERR_ALIGNMENT, "xs_next must be 16-byte aligned");
    K2Prep k;
    const int slots = g->pr[i].p.nx_slots;
    svdq_status st = prepare_k2(layers[i], xq[i], xs[i], xl1[i], M[i], Y[i], SVDQ_BF16, layers[i]->N, true, &k,
                                xq_next[i], kNvfp4PairBN);
    if (st != SVDQ_OK) return st;
    g->pr[i].a = k.maps.a;
    g->pr[i].b = k.maps.b;
    g->pr[i].xl1 = k.maps.xl1;
    g->pr[i].l2 = k.maps.l2;
    g->pr[i].sfa = k.sfa_map;
    g->pr[i].sfb = k.sfb_map;
    g->pr[i].y = k.maps.y;
    if ((st = make_map(&g->pr[i].nxq, xq_next[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, layers[i]->N / 2, M[i],
                       layers[i]->N / 2, 96, 128, CU_TENSOR_MAP_SWIZZLE_NONE)) != SVDQ_OK)
      return st;
    K2Params &p = g->pr[i].p;
    p = k.p;
    p.Y = Y[i];
    p.fuse = 1;
    p.nx_act = act;
    p.nx_r = Nx->rank;
    p.nx_gs = Nx->gs_x;
    p.nx_lam_inv = Nx->lambda_inv;
    p.nx_l1s = Nx->l1s;
    p.nx_xq = xq_next[i];
    p.nx_sf = xs_next[i];
    p.nx_slots = slots;
  }
  return SVDQ_OK;
}
}  // namespace

svdq_status svdq_gemm_fused_next_workspace(int32_t n, const svdq_linear *const *layers, const int64_t *M,
                                           const svdq_linear *const *nexts, size_t *ws_bytes) {
  if (!ws_bytes) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  K2PairArgs g;
  size_t off[kMaxGroup];
  return prepare_fused(n, layers, nullptr, nullptr, nullptr, M, nullptr, nexts, 0, nullptr, nullptr, &g, ws_bytes,
                       off);
}

svdq_status svdq_gemm_w4a4_lowrank_up_fused_next(int32_t n, const svdq_linear *const *layers,
                                                 const uint8_t *const *xq, const uint8_t *const *xs,
                                                 const uint16_t *const *xl1, const int64_t *M, void *const *Y,
                                                 const svdq_linear *const *nexts, int32_t act,
                                                 uint8_t *const *xq_next, uint8_t *const *xs_next,
                                                 uint16_t *const *xl1_next, void *ws, size_t ws_bytes,
                                                 void *stream) {
  K2PairArgs g;
  size_t need = 0, off[kMaxGroup];
  if (!xq) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null array");
  svdq_status st = prepare_fused(n, layers, xq, xs, xl1, M, Y, nexts, act, xq_next, xs_next, &g, &need, off);
  if (st != SVDQ_OK) return st;
  if (need && (!ws || ws_bytes < need)) return fail(SVDQ_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  for (int i = 0; i < n; ++i) {
    if (g.pr[i].p.nx_r) {
      if (!xl1_next || !xl1_next[i]) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null xl1_next %d", i);
      if (!aligned16(xl1_next[i])) return fail(SVDQ_ERR_ALIGNMENT, "xl1_next must be 16-byte aligned");
      g.pr[i].p.nx_part = reinterpret_cast<float *>(static_cast<uint8_t *>(ws) + off[i]);
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_k2_nvfp4_2sm_group(g, s);
  if (e != cudaSuccess) return cuda_fail(e, "fused K2 launch");
  ++g_launches;
  for (int i = 0; i < n; ++i) {
    if (!g.pr[i].p.nx_r) continue;
    if ((e = launch_k2_next_reduce(g, i, xl1_next[i], s)) != cudaSuccess) return cuda_fail(e, "xl1_next reduce");
    ++g_launches;
  }
  return SVDQ_OK;
}

svdq_status svdq_linear_forward(const svdq_linear *L, const void *X, int32_t x_dtype, int64_t M,
                                int64_t ldx, void *Y, int32_t y_dtype, int64_t ldy, void *ws,
                                size_t ws_bytes, void *stream) {
  svdq_status st = check_linear(L, true);
  if (st != SVDQ_OK) return st;
  size_t bq, bs, bl;
  if ((st = svdq_act_buffer_sizes(L->fmt, M, L->K, L->rank, &bq, &bs, &bl)) != SVDQ_OK) return st;
  auto up = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  if (!ws || ws_bytes < up(bq) + up(bs) + up(bl)) return fail(SVDQ_ERR_WORKSPACE, "workspace too small");
  uint8_t *xq = static_cast<uint8_t *>(ws);
  uint8_t *xs = xq + up(bq);
  uint16_t *xl1 = reinterpret_cast<uint16_t *>(xs + up(bs));
  if ((st = svdq_quantize_act_lowrank_down(L, X, x_dtype, M, ldx, xq, xs, L->rank ? xl1 : nullptr, stream)) != SVDQ_OK)
    return st;
  return svdq_gemm_w4a4_lowrank_up(L, xq, xs, L->rank ? xl1 : nullptr, M, Y, y_dtype, ldy, stream);
}

svdq_status svdq_quantize_residual(const float *R, int64_t K, int64_t N, int32_t fmt, int32_t scale_dtype,
                                   uint8_t *codes, uint8_t *scales, float *gs_w, void *stream) {
  if (!R || !codes || !scales || !gs_w) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (fmt != SVDQ_FMT_NVFP4 && fmt != SVDQ_FMT_INT4 && fmt != SVDQ_FMT_W8A8)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad format");
  if (K <= 0 || K % 64) return fail(SVDQ_ERR_SHAPE, "K must be a positive multiple of 64");
  if (N <= 0 || N % 16) return fail(SVDQ_ERR_SHAPE, "N must be a positive multiple of 16");
  if (fmt == SVDQ_FMT_INT4 && scale_dtype != SVDQ_BF16 && scale_dtype != SVDQ_FP16)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "INT4 scale dtype must be BF16 or FP16");
  if (!aligned16(codes) || !aligned16(scales) || !aligned16(R)) return fail(SVDQ_ERR_ALIGNMENT, "unaligned");
  svdq_status st = check_device();
  if (st != SVDQ_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float gs = 1.0f;
  if (fmt == SVDQ_FMT_NVFP4) {
    if (*gs_w > 0.f) {
      gs = *gs_w;
    } else {
      unsigned int *d_amax = nullptr;
      SVDQ_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&d_amax), sizeof(unsigned int), s), "alloc");
      SVDQ_CUDA(launch_absmax(R, K * N, d_amax, s), "absmax");
      ++g_launches;
      unsigned int bits = 0;
      SVDQ_CUDA(cudaMemcpyAsync(&bits, d_amax, sizeof(bits), cudaMemcpyDeviceToHost, s), "copy");
      SVDQ_CUDA(cudaFreeAsync(d_amax, s), "free");
      SVDQ_CUDA(cudaStreamSynchronize(s), "sync");
      float amax;
      std::memcpy(&amax, &bits, sizeof(amax));
      volatile float div = 2688.0f;   // fl32(amax / 2688): one IEEE single division
      gs = amax == 0.f ? 1.0f : amax / div;
      *gs_w = gs;
    }
  } else {
    *gs_w = 1.0f;
  }
  SVDQ_CUDA(launch_quantize_residual(R, K, N, fmt == SVDQ_FMT_NVFP4 ? 0 : (fmt == SVDQ_FMT_W8A8 ? 2 : 1),
                                     scale_dtype == SVDQ_BF16,
                                     gs, codes, scales, s),
            "quantize residual");
  ++g_launches;
  return SVDQ_OK;
}

// ---------------------------------------------------------------- offline weights
namespace {
struct WsLayout {
  size_t what, gram, evals, E, sigma, l1_64, l2_64, r32, l1_32, l2_32, work, info, total;
  int lwork;
};
size_t up256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }

svdq_status ws_layout(int64_t K, int64_t N, int32_t rank, int lwork, WsLayout *w) {
  const int64_t P = K < N ? K : N;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += up256(bytes); return o; };
  w->what = take(static_cast<size_t>(K) * N * 8);
  w->gram = take(static_cast<size_t>(P) * P * 8);
  w->evals = take(static_cast<size_t>(P) * 8);
  w->E = take(static_cast<size_t>(P) * (rank > 0 ? rank : 1) * 8);
  w->sigma = take(static_cast<size_t>(rank > 0 ? rank : 1) * 8);
  w->l1_64 = take(static_cast<size_t>(K) * (rank > 0 ? rank : 1) * 8);
  w->l2_64 = take(static_cast<size_t>(N) * (rank > 0 ? rank : 1) * 8);
  w->r32 = take(static_cast<size_t>(K) * N * 4);
  w->l1_32 = take(static_cast<size_t>(K) * (rank > 0 ? rank : 1) * 4);
  w->l2_32 = take(static_cast<size_t>(N) * (rank > 0 ? rank : 1) * 4);
  w->work = take(static_cast<size_t>(lwork > 0 ? lwork : 1) * 8);
  w->info = take(16);
  w->total = off;
  w->lwork = lwork;
  return SVDQ_OK;
}

int syevd_lwork(int64_t P) {
  cusolverDnHandle_t h;
  if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) return -1;
  int lwork = 0;
  cusolverStatus_t r = cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                                   static_cast<int>(P), nullptr, static_cast<int>(P),
                                                   nullptr, &lwork);
  cusolverDnDestroy(h);
  return r == CUSOLVER_STATUS_SUCCESS ? lwork : -1;
}
}  // namespace

svdq_status svdq_quantize_weights_workspace(int64_t K, int64_t N, int32_t rank, size_t *ws_bytes) {
  if (!ws_bytes) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (K <= 0 || K % 64 || N <= 0 || N % 16) return fail(SVDQ_ERR_SHAPE, "bad K/N");
  if (rank < 0 || rank > 128 || rank % 16) return fail(SVDQ_ERR_RANK, "bad rank");
  svdq_status st = check_device();
  if (st != SVDQ_OK) return st;
  const int64_t P = K < N ? K : N;
  const int lwork = rank > 0 ? syevd_lwork(P) : 1;
  if (lwork < 0) return fail(SVDQ_ERR_CUDA, "cusolver bufferSize failed");
  WsLayout w;
  ws_layout(K, N, rank, lwork, &w);
  *ws_bytes = w.total;
  return SVDQ_OK;
}

}  // extern "C"

namespace svdq {
// svdq_quantize_weights with an optional refinement target (reading Q3): when `svd_sub`
// ([K][N] fp64, Q(R_{t-1}) in the W_hat space) is given, L1 L2 is the truncated SVD of
// W_hat - svd_sub (formed in `tgt`, [K][N] fp64 scratch) and R = W_hat - L1 L2 as usual.
svdq_status quantize_weights_impl(const void *W, int32_t w_dtype, const float *lambda, int64_t K, int64_t N,
                                  int32_t rank, int32_t fmt, int32_t scale_dtype, float gs_x, const float *L1_opt,
                                  const float *L2_opt, svdq_linear *dst, void *ws, size_t ws_bytes, void *stream,
                                  const double *svd_sub, double *tgt, const GptqArgs *gq, uint8_t *gq_ws) {
  if (gq && (!gq->X || !gq_ws || gq->M < 1 || gq->ldx < K || !(gq->damp >= 0.f) ||
             (gq->x_dtype != SVDQ_BF16 && gq->x_dtype != SVDQ_FP16)))
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad GPTQ calibration arguments");
  if (svd_sub && (!tgt || L1_opt)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "refinement target needs tgt, no L1_opt");
  if (!W || !lambda || !dst || !ws) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (w_dtype != SVDQ_BF16 && w_dtype != SVDQ_FP16 && w_dtype != SVDQ_FP32)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad W dtype");
  if (fmt != SVDQ_FMT_NVFP4 && fmt != SVDQ_FMT_INT4 && fmt != SVDQ_FMT_W8A8) return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad format");
  if (K <= 0 || K % 64 || N <= 0 || N % 16) return fail(SVDQ_ERR_SHAPE, "bad K/N");
  if (rank < 0 || rank > 128 || rank % 16 || rank > (K < N ? K : N)) return fail(SVDQ_ERR_RANK, "bad rank");
  if ((L1_opt == nullptr) != (L2_opt == nullptr)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "L1_opt and L2_opt go together");
  if (!dst->w_codes || !dst->w_scales || !dst->lambda_inv || (rank > 0 && (!dst->l1s || !dst->l2s)))
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "dst buffers must be set");
  if (fmt == SVDQ_FMT_NVFP4 && !(gs_x > 0.f)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "gs_x must be > 0");
  svdq_status st = check_device();
  if (st != SVDQ_OK) return st;
  const int64_t P = K < N ? K : N;
  const int lwork = (rank > 0 && !L1_opt) ? syevd_lwork(P) : 1;
  if (lwork < 0) return fail(SVDQ_ERR_CUDA, "cusolver bufferSize failed");
  WsLayout w;
  ws_layout(K, N, rank, lwork, &w);
  if (ws_bytes < w.total) return fail(SVDQ_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, w.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t *base = static_cast<uint8_t *>(ws);
  double *What = reinterpret_cast<double *>(base + w.what);
  double *G = reinterpret_cast<double *>(base + w.gram);
  double *evals = reinterpret_cast<double *>(base + w.evals);
  double *E = reinterpret_cast<double *>(base + w.E);
  double *sigma = reinterpret_cast<double *>(base + w.sigma);
  double *L1d = reinterpret_cast<double *>(base + w.l1_64);
  double *L2d = reinterpret_cast<double *>(base + w.l2_64);
  float *R32 = reinterpret_cast<float *>(base + w.r32);
  float *L1f = reinterpret_cast<float *>(base + w.l1_32);
  float *L2f = reinterpret_cast<float *>(base + w.l2_32);
  double *work = reinterpret_cast<double *>(base + w.work);
  int *info = reinterpret_cast<int *>(base + w.info);

  float *lam_inv = const_cast<float *>(dst->lambda_inv);
  SVDQ_CUDA(launch_lambda_inv(lambda, lam_inv, K, s), "lambda_inv");
  SVDQ_CUDA(launch_smooth_weight64(W, w_dtype, lambda, K, N, What, s), "smooth W");
  g_launches += 2;
  GptqState gst{};
  if (gq) {   // Hessian of the residual's proxy loss on X_hat; needs lambda_inv
    const int glw = gptq_potrf_lwork(K);
    if (glw < 0) return fail(SVDQ_ERR_CUDA, "cusolver potrf bufferSize failed");
    if (const char *e = gptq_hessian(*gq, lam_inv, K, glw, gq_ws, s, &gst))
      return fail(std::strstr(e, "positive definite") ? SVDQ_ERR_INVALID_ARGUMENT : SVDQ_ERR_CUDA, "GPTQ: %s", e);
    g_launches += 2;
  }

  cublasHandle_t hb = nullptr;
  if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) return fail(SVDQ_ERR_CUDA, "cublasCreate");
  cublasSetStream(hb, s);
  cublasSetMathMode(hb, CUBLAS_DEFAULT_MATH);
  svdq_status result = SVDQ_OK;
  const double one = 1.0, zero = 0.0, mone = -1.0;
  do {
    if (rank > 0) {
      if (L1_opt) {
        if (launch_f32_to_f64(L1_opt, L1d, K * rank, s) != cudaSuccess ||
            launch_f32_to_f64(L2_opt, L2d, static_cast<int64_t>(rank) * N, s) != cudaSuccess) {
          result = fail(SVDQ_ERR_CUDA, "convert L1/L2");
          break;
        }
      } else {
        // SVD source: W_hat, or W_hat - Q(R_{t-1}) when refining
        const double *Src = What;
        if (svd_sub) {
          if (launch_sub64(What, svd_sub, tgt, K * N, s) != cudaSuccess) { result = fail(SVDQ_ERR_CUDA, "refine target"); break; }
          ++g_launches;
          Src = tgt;
        }
        // Gram matrix of the smaller side (column-major view of row-major Src is Src^T, N x K)
        if (N <= K) {
          if (cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, (int)N, (int)K, &one, Src, (int)N, &zero, G, (int)N) != CUBLAS_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "syrk"); break; }
        } else {
          if (cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, (int)K, (int)N, &one, Src, (int)N, &zero, G, (int)K) != CUBLAS_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "syrk"); break; }
        }
        cusolverDnHandle_t hs = nullptr;
        if (cusolverDnCreate(&hs) != CUSOLVER_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "cusolverDnCreate"); break; }
        cusolverDnSetStream(hs, s);
        cusolverStatus_t cs = cusolverDnDsyevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)P, G, (int)P, evals, work, lwork, info);
        cusolverDnDestroy(hs);
        if (cs != CUSOLVER_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "syevd"); break; }
        if (launch_eig_to_factors(G, evals, P, rank, E, sigma, s) != cudaSuccess) { result = fail(SVDQ_ERR_CUDA, "eig"); break; }
        if (N <= K) {
          // L2 = E^T (rows = right singular vectors); L1 = Src E  (= U_r Sigma_r)
          if (cublasDgeam(hb, CUBLAS_OP_T, CUBLAS_OP_N, (int)N, rank, &one, E, rank, &zero, E, (int)N, L2d, (int)N) != CUBLAS_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "geam"); break; }
          if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, rank, (int)K, (int)N, &one, E, rank, Src, (int)N, &zero, L1d, rank) != CUBLAS_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "gemm L1"); break; }
        } else {
          // L1 = E diag(sigma); L2 = diag(sigma)^-1 E^T Src
          if (cudaMemcpyAsync(L1d, E, static_cast<size_t>(K) * rank * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) { result = fail(SVDQ_ERR_CUDA, "copy"); break; }
          if (launch_scale_cols(L1d, K, rank, sigma, 0, 0, s) != cudaSuccess) { result = fail(SVDQ_ERR_CUDA, "scale"); break; }
          if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, (int)N, rank, (int)K, &one, Src, (int)N, E, rank, &zero, L2d, (int)N) != CUBLAS_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "gemm L2"); break; }
          if (launch_scale_cols(L2d, rank, N, sigma, 1, 1, s) != cudaSuccess) { result = fail(SVDQ_ERR_CUDA, "scale"); break; }
        }
        g_launches += 3;
      }
      // R = W_hat - L1 L2  (in place on What; column-major: What^T -= L2^T L1^T)
      if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, (int)K, rank, &mone, L2d, (int)N, L1d, rank, &one, What, (int)N) != CUBLAS_STATUS_SUCCESS) { result = fail(SVDQ_ERR_CUDA, "gemm R"); break; }
    }
    if (gq && gptq_zero_dead(What, gst, K, N, s) != cudaSuccess) { result = fail(SVDQ_ERR_CUDA, "GPTQ dead rows"); break; }
    if (launch_f64_to_f32(What, R32, K * N, s) != cudaSuccess) { result = fail(SVDQ_ERR_CUDA, "R32"); break; }
    ++g_launches;
    float gs_w = 0.f;
    if ((result = svdq_quantize_residual(R32, K, N, fmt, scale_dtype, const_cast<uint8_t *>(dst->w_codes),
                                         const_cast<uint8_t *>(dst->w_scales), &gs_w, stream)) != SVDQ_OK)
      break;
    if (gq) {   // GPTQ overwrites the RTN codes (and group scales); RTN supplied gs_w / W8A8 channel scales
      if (const char *e = gptq_run(What, gst, K, N, fmt == SVDQ_FMT_NVFP4 ? 0 : (fmt == SVDQ_FMT_W8A8 ? 2 : 1),
                                   scale_dtype == SVDQ_BF16, gs_w,
                                   fmt == SVDQ_FMT_W8A8 ? reinterpret_cast<const float *>(dst->w_scales) : nullptr,
                                   const_cast<uint8_t *>(dst->w_codes), const_cast<uint8_t *>(dst->w_scales), s)) {
        result = fail(SVDQ_ERR_CUDA, "GPTQ: %s", e);
        break;
      }
      g_launches += 2 * ((K + 63) / 64);
    }
    const float gx = fmt == SVDQ_FMT_NVFP4 ? gs_x : 1.0f;
    const float alpha = fmt == SVDQ_FMT_NVFP4 ? gx * gs_w : 1.0f;
    if (rank > 0) {
      if (launch_f64_to_f32(L1d, L1f, K * rank, s) != cudaSuccess ||
          launch_f64_to_f32(L2d, L2f, static_cast<int64_t>(rank) * N, s) != cudaSuccess ||
          launch_derive_l1s(L1f, 2, lam_inv, 1.0f, K, rank, 0, const_cast<uint16_t *>(dst->l1s), s) != cudaSuccess ||
          launch_derive_l2s(L2f, 2, N, rank, 0, rank, alpha, const_cast<uint16_t *>(dst->l2s), s) != cudaSuccess) {
        result = fail(SVDQ_ERR_CUDA, "derive l1s/l2s");
        break;
      }
      g_launches += 4;
    }
    dst->fmt = fmt;
    dst->rank = rank;
    dst->K = K;
    dst->N = N;
    dst->scale_dtype = fmt == SVDQ_FMT_INT4 ? scale_dtype : SVDQ_BF16;
    dst->gs_w = gs_w;
    dst->gs_x = gx;
  } while (false);
  cublasDestroy(hb);
  if (result != SVDQ_OK) return result;
  SVDQ_CUDA(cudaStreamSynchronize(s), "sync");
  return SVDQ_OK;
}

}  // namespace svdq

extern "C" {

svdq_status svdq_quantize_weights(const void *W, int32_t w_dtype, const float *lambda, int64_t K,
                                  int64_t N, int32_t rank, int32_t fmt, int32_t scale_dtype,
                                  float gs_x, const float *L1_opt, const float *L2_opt,
                                  svdq_linear *dst, void *ws, size_t ws_bytes, void *stream) {
  return svdq::quantize_weights_impl(W, w_dtype, lambda, K, N, rank, fmt, scale_dtype, gs_x, L1_opt, L2_opt, dst, ws,
                                     ws_bytes, stream, nullptr, nullptr, nullptr, nullptr);
}

svdq_status svdq_quantize_residual_gptq_workspace(int64_t M_cal, int64_t K, int64_t N, size_t *ws_bytes) {
  if (!ws_bytes) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (M_cal < 1) return fail(SVDQ_ERR_SHAPE, "M_cal must be >= 1");
  if (K <= 0 || K % 64 || N <= 0 || N % 16) return fail(SVDQ_ERR_SHAPE, "bad K/N");
  const int glw = gptq_potrf_lwork(K);
  if (glw < 0) return fail(SVDQ_ERR_CUDA, "cusolver potrf bufferSize failed");
  *ws_bytes = up256(static_cast<size_t>(K) * N * 8) + up256(static_cast<size_t>(K) * N * 4) +
              gptq_workspace_bytes(M_cal, K, N, glw);
  return SVDQ_OK;
}

svdq_status svdq_quantize_residual_gptq(const float *R, int64_t K, int64_t N, int32_t fmt, int32_t scale_dtype,
                                        const void *X_cal, int32_t x_dtype, int64_t M_cal, int64_t ldx,
                                        const float *lambda_inv, float damp, uint8_t *codes, uint8_t *scales,
                                        float *gs_w, void *ws, size_t ws_bytes, void *stream) {
  size_t need = 0;
  svdq_status st = svdq_quantize_residual_gptq_workspace(M_cal, K, N, &need);
  if (st != SVDQ_OK) return st;
  if (!R || !X_cal || !lambda_inv || !codes || !scales || !gs_w || !ws)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (ws_bytes < need) return fail(SVDQ_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  if (ldx < K || !(damp >= 0.f) || (x_dtype != SVDQ_BF16 && x_dtype != SVDQ_FP16))
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad GPTQ calibration arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t *base = static_cast<uint8_t *>(ws);
  double *R64 = reinterpret_cast<double *>(base);
  float *R32 = reinterpret_cast<float *>(base + up256(static_cast<size_t>(K) * N * 8));
  uint8_t *gws = base + up256(static_cast<size_t>(K) * N * 8) + up256(static_cast<size_t>(K) * N * 4);
  const svdq::GptqArgs gq{X_cal, x_dtype, M_cal, ldx, damp};
  svdq::GptqState gst{};
  SVDQ_CUDA(launch_f32_to_f64(R, R64, K * N, s), "R64");
  if (const char *e = gptq_hessian(gq, lambda_inv, K, gptq_potrf_lwork(K), gws, s, &gst))
    return fail(std::strstr(e, "positive definite") ? SVDQ_ERR_INVALID_ARGUMENT : SVDQ_ERR_CUDA, "GPTQ: %s", e);
  SVDQ_CUDA(gptq_zero_dead(R64, gst, K, N, s), "GPTQ dead rows");
  SVDQ_CUDA(launch_f64_to_f32(R64, R32, K * N, s), "R32");
  *gs_w = 0.f;
  if ((st = svdq_quantize_residual(R32, K, N, fmt, scale_dtype, codes, scales, gs_w, stream)) != SVDQ_OK) return st;
  if (const char *e = gptq_run(R64, gst, K, N, fmt == SVDQ_FMT_NVFP4 ? 0 : (fmt == SVDQ_FMT_W8A8 ? 2 : 1),
                               scale_dtype == SVDQ_BF16, *gs_w,
                               fmt == SVDQ_FMT_W8A8 ? reinterpret_cast<const float *>(scales) : nullptr, codes, scales,
                               s))
    return fail(SVDQ_ERR_CUDA, "GPTQ: %s", e);
  g_launches += 6 + 2 * ((K + 63) / 64);
  SVDQ_CUDA(cudaStreamSynchronize(s), "sync");
  return SVDQ_OK;
}

svdq_status svdq_quantize_weights_gptq_workspace(int64_t M_cal, int64_t K, int64_t N, int32_t rank,
                                                 size_t *ws_bytes) {
  if (!ws_bytes) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null output");
  if (M_cal < 1) return fail(SVDQ_ERR_SHAPE, "M_cal must be >= 1");
  size_t qw = 0;
  svdq_status st = svdq_quantize_weights_workspace(K, N, rank, &qw);
  if (st != SVDQ_OK) return st;
  const int glw = gptq_potrf_lwork(K);
  if (glw < 0) return fail(SVDQ_ERR_CUDA, "cusolver potrf bufferSize failed");
  *ws_bytes = up256(qw) + gptq_workspace_bytes(M_cal, K, N, glw);
  return SVDQ_OK;
}

svdq_status svdq_quantize_weights_gptq(const void *W, int32_t w_dtype, const float *lambda, int64_t K, int64_t N,
                                       int32_t rank, int32_t fmt, int32_t scale_dtype, float gs_x, const void *X_cal,
                                       int32_t x_dtype, int64_t M_cal, int64_t ldx, float damp, svdq_linear *dst,
                                       void *ws, size_t ws_bytes, void *stream) {
  size_t need = 0, qw = 0;
  svdq_status st = svdq_quantize_weights_gptq_workspace(M_cal, K, N, rank, &need);
  if (st != SVDQ_OK) return st;
  if (!ws) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null workspace");
  if (ws_bytes < need) return fail(SVDQ_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  if ((st = svdq_quantize_weights_workspace(K, N, rank, &qw)) != SVDQ_OK) return st;
  const svdq::GptqArgs gq{X_cal, x_dtype, M_cal, ldx, damp};
  return svdq::quantize_weights_impl(W, w_dtype, lambda, K, N, rank, fmt, scale_dtype, gs_x, nullptr, nullptr, dst,
                                     ws, up256(qw), stream, nullptr, nullptr, &gq,
                                     static_cast<uint8_t *>(ws) + up256(qw));
}

svdq_status svdq_lora_fuse(const svdq_linear *src, const void *A, const void *B, int32_t ab_dtype,
                           int32_t r_l, float scale, svdq_linear *dst, void *stream) {
  svdq_status st = check_linear(src, false);
  if (st != SVDQ_OK) return st;
  if (!A || !B || !dst || !dst->l1s || !dst->l2s) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (ab_dtype != SVDQ_BF16 && ab_dtype != SVDQ_FP16 && ab_dtype != SVDQ_FP32)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad A/B dtype");
  if (r_l <= 0 || r_l % 16 || src->rank + r_l > 128) return fail(SVDQ_ERR_RANK, "bad LoRA rank");
  if (dst->l1s == src->l1s || dst->l2s == src->l2s)
    return fail(SVDQ_ERR_INVALID_ARGUMENT, "dst l1s/l2s must not alias src");
  if ((st = check_device()) != SVDQ_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int r0 = src->rank, r1 = src->rank + r_l;
  const float alpha = src->fmt == SVDQ_FMT_NVFP4 ? src->gs_x * src->gs_w : 1.0f;
  uint16_t *l1s = const_cast<uint16_t *>(dst->l1s);
  uint16_t *l2s = const_cast<uint16_t *>(dst->l2s);
  if (r0 > 0) {
    SVDQ_CUDA(launch_copy_l1s_rows(src->l1s, src->K, r0, l1s, s), "copy l1s");
    SVDQ_CUDA(launch_copy_l2s_cols(src->l2s, src->N, r0, r1, l2s, s), "copy l2s");
    ++g_launches;
  }
  SVDQ_CUDA(launch_derive_l1s(A, ab_dtype, nullptr, scale, src->K, r_l, r0, l1s, s), "lora l1s");
  SVDQ_CUDA(launch_derive_l2s(B, ab_dtype, src->N, r_l, r0, r1, alpha, l2s, s), "lora l2s");
  g_launches += 2;
  const uint16_t *nl1 = dst->l1s, *nl2 = dst->l2s;
  *dst = *src;
  dst->rank = r1;
  dst->l1s = nl1;
  dst->l2s = nl2;
  return SVDQ_OK;
}

svdq_status svdq_debug_int4_group_accum(const uint8_t *xq, const uint8_t *wq, int64_t M, int64_t N,
                                        int64_t K, int32_t *acc, void *stream) {
  if (!xq || !wq || !acc) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (M < 1 || K <= 0 || K % 64 || N <= 0 || N % 16) return fail(SVDQ_ERR_SHAPE, "bad shape");
  svdq_status st = check_device();
  if (st != SVDQ_OK) return st;
  K2Params p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.Npad = N;
  p.xq = xq;
  p.wq = wq;
  p.dbg_acc = acc;
  p.alpha = 1.0f;
  if (!aligned16(xq) || !aligned16(wq) || !aligned16(acc)) return fail(SVDQ_ERR_ALIGNMENT, "unaligned");
  K2Maps maps;
  std::memset(&maps, 0, sizeof(maps));
  if ((st = make_map(&maps.a, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, K / 2, M, K / 2, 64, 128,
                     CU_TENSOR_MAP_SWIZZLE_NONE)) != SVDQ_OK) return st;
  if ((st = make_map(&maps.b, wq, CU_TENSOR_MAP_DATA_TYPE_UINT8, K / 2, N, K / 2, 64, kInt4BN,
                     CU_TENSOR_MAP_SWIZZLE_NONE)) != SVDQ_OK) return st;
  cudaError_t e = launch_k2_int4(maps, p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "int4 debug launch");
  ++g_launches;
  return SVDQ_OK;
}

svdq_status svdq_debug_codec(const float *in, uint8_t *out, int64_t n, int32_t kind, void *stream) {
  if (!in || !out) return fail(SVDQ_ERR_INVALID_ARGUMENT, "null pointer");
  if (n < 0 || (kind != 0 && kind != 1)) return fail(SVDQ_ERR_INVALID_ARGUMENT, "bad n / kind");
  svdq_status st = check_device();
  if (st != SVDQ_OK) return st;
  if (n == 0) return SVDQ_OK;
  cudaError_t e = launch_codec(in, out, n, kind, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "codec launch");
  ++g_launches;
  return SVDQ_OK;
}

}  // extern "C"
