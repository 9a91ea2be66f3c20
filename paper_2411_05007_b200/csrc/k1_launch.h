// Internal launch interfaces between api.cu and the kernel translation units.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace svdq {

// Launch with programmatic stream serialization (PDL) and an optional cluster size.
template <typename Kern, typename... Args>
inline cudaError_t launch_ex_impl(bool force_cluster, Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                  unsigned cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (cluster_x > 1 || force_cluster) {     // kernels using cluster instructions need the attribute
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Kern, typename... Args>
inline cudaError_t launch_ex(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, unsigned cluster_x,
                             Args... args) {
  return launch_ex_impl(false, kern, grid, block, smem, s, cluster_x, args...);
}
// Always launched as clusters of `cluster_x` CTAs (also when cluster_x == 1).
template <typename Kern, typename... Args>
inline cudaError_t launch_ex_cluster(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     unsigned cluster_x, Args... args) {
  return launch_ex_impl(true, kern, grid, block, smem, s, cluster_x, args...);
}

struct K1Params {
  int fmt;            // 0 NVFP4, 1 INT4, 2 W8A8 (K1 kernels: down-projection only)
  bool x_bf16;        // X dtype bf16 (else fp16)
  bool scale_bf16;    // INT4 scale dtype bf16 (else fp16)
  const void *X;
  int64_t ldx, M, Mpad, K;
  const float *lam_inv;
  const uint16_t *l1s;
  int rank;
  float gs_x;
  uint8_t *xq;
  uint8_t *xs;
  uint16_t *xl1;
  float *xl1_f32;     // tensor-parallel K-slice: fp32 partial X L1s^T [M][rank] instead of bf16 xl1
  // fused packed all-gather: every output store is repeated at `ndst` byte
  // offsets dst_delta[j] from xq / xs / xl1_f32 (destination j = rank j's gather buffer, possibly a
  // peer's memory mapped over NVLink); ndst = 1, dst_delta[0] = 0 otherwise
  int ndst;
  int64_t dst_delta[8];
  // layout of the outputs: codes row pitch out_k / 2 bytes, scales of the (rows, out_k) layout
  // starting at 16-column group out_c0 (K-slice inside a full-K buffer); defaults out_k = K, 0
  int64_t out_k, out_c0;
  // W8A8: xs already holds every row's amax |x_hat| (fp32), written by the row-tile kernel's
  // down-projection pass, so the INT8 kernel encodes in one pass
  int w8_amax;
};
cudaError_t launch_k1_int8_rows(const K1Params &p, cudaStream_t s);   // W8A8 per-token INT8 codes
// Grouped K1: up to kMaxGroup1 problems (same fmt, scale dtype and rank) in one launch; the
// grid's row-tile axis runs over the concatenated row tiles.
constexpr int kMaxGroup1 = 4;
struct K1Problem {
  CUtensorMap x, l1s, lam;
  K1Params p;
};
struct K1Args {
  K1Problem pr[kMaxGroup1];
  int n;
  int tile_begin[kMaxGroup1 + 1];
};
// Row-tile K1 (k1_rows.cu, round 2): each CTA owns `rt` whole rows over the full K; maps: X as the
// 3-D view {64 cols, K/64 blocks, M rows} with box {64, 128/rt, rt}, L1s box {64, rank}, lambda_inv
// as [K/32][32] with box {32, 2 * 128/rt}.  bf16 or fp16 X.
struct K1RowLayout {
  int rt, q;
  int x_bytes;            // X tile bytes of an X stage (fp16 X: + the bf16 low-part tile)
  int stage_bytes, stages;    // X ring: X tile + the Q blocks' lambda_inv
  int l1_bytes, wstages;      // L1s ring: the Q blocks' L1s tiles (rank > 0)
  size_t w_off, bar_off, smem;
};
K1RowLayout k1_row_layout(int rt, int rank, bool x16);
int k1_rows_rt(int64_t rows_total, int rank);            // row tile for `rows_total` padded rows
cudaError_t launch_k1_rows_group(K1Args &g, int rt, cudaStream_t s);

struct K2Params {
  int64_t M, N, K, Npad;
  int rank;
  const uint8_t *sfa;     // NVFP4: activation scale factors (128x4 layout); INT4: [M][K/64]
  const uint8_t *sfb;     // NVFP4: weight scale factors; INT4: [N][K/64]
  const uint8_t *xq;      // INT4 path (cp.async staging)
  const uint8_t *wq;
  const void *bias;
  int bias_dtype;         // 0 bf16, 1 fp16, 2 fp32
  void *Y;
  int y_dtype;            // 0 bf16, 1 fp16, 2 fp32
  int64_t ldy;
  float alpha;
  int scale_bf16;         // INT4 scales
  int32_t *dbg_acc;       // INT4 debug: per-group int32 accumulators [K/64][M][N]
  int w8;                 // W8A8 (kind::i8 over the whole K; sfa / sfb are fp32 [M] / [N])
  // Layer-boundary fusion (CTA-pair kernel only): the epilogue also runs the
  // next layer's K1 on its own bf16 output -- NVFP4 codes / scale factors of
  // act(Y) * lambda_inv_next and partial X L1s_next^T sums (reduced by launch_k2_next_reduce).
  int fuse;               // 1: on (this problem's tiles are walked n-fastest)
  int band;               // CTA-pair K2: 256-row tiles per L2 band (0 = the whole M, m-fastest order)
  int nx_act;             // 0 identity, 1 GELU (tanh form)
  int nx_r;               // next layer's rank: 0, 16 or 32
  float nx_gs;            // next layer's gs_x
  const float *nx_lam_inv;    // [N]
  const uint16_t *nx_l1s;     // [nx_r][N] bf16
  uint8_t *nx_xq;             // [M][N/2]
  uint8_t *nx_sf;             // 128x4 layout over (M rows, K = N)
  float *nx_part;             // [ceil(M/256)][nx_slots][256][nx_r] fp32 partial sums
  int nx_slots;
};
struct K2Maps {
  CUtensorMap a, b, xl1, l2, y;   // y: output store map, box {64 B of columns, 32 rows}, SW64
};
cudaError_t launch_k2_nvfp4(const K2Maps &maps, const K2Params &p, cudaStream_t s);
int k2_nvfp4_bn(int64_t M, int64_t N);   // N tile the 1-CTA NVFP4 GEMM will use
// CTA-pair NVFP4 GEMM (256 x 192 tiles, each CTA stages 96 rows of B); SF tensor maps are
// 3-D uint64 views [tiles128][K/64][64] of the 128x4 scale-factor layout.
cudaError_t launch_k2_nvfp4_2sm(const K2Maps &maps, const CUtensorMap &sfa, const CUtensorMap &sfb,
                                const K2Params &p, int bn, cudaStream_t s);
// Grouped form: up to kMaxGroup independent problems in one persistent launch; CTA pairs
// walk the concatenation of the problems' tile lists.
constexpr int kMaxGroup = 4;
struct K2PairProblem {
  CUtensorMap a, b, xl1, l2, sfa, sfb, y;
  CUtensorMap nxq;        // fused: the next layer's codes [M][N/2] bytes, box {96, 128}
  K2Params p;
};
struct K2PairArgs {
  K2PairProblem pr[kMaxGroup];
  int n;
  int tile_begin[kMaxGroup + 1];
  int contig;             // set by the launcher: pairs take contiguous tile ranges (fused launches)
  int npairs;             // set by the launcher
  int bn;                 // pair tile N: 192 or 256 (the B / L2s tensor maps' box rows are bn / 2)
};
// Pair tile N for a problem of N output columns (256 when N % 256 == 0)
int k2_pair_bn(int64_t N);
cudaError_t launch_k2_nvfp4_2sm_group(K2PairArgs &args, cudaStream_t s);
// SM count of the current device (cached per device ordinal; one source for every launcher
// and for workspace sizing, so the two always agree)
int device_sm_count();
// CTA pairs the grouped launch will use for `tiles` tiles
int k2_pair_count(int64_t tiles);
// Slots per 256-row block of a fused problem's partial-sum buffer (upper bound for any pair
// count <= k2_pair_count(tiles))
int k2_next_slots(int64_t n_tiles_of_problem, int64_t tiles, int npairs);
// xl1_next[m][j] = bf16(sum over the partial slots of m's 256-row block, in slot order)
cudaError_t launch_k2_next_reduce(const K2PairArgs &g, int i, uint16_t *xl1_next, cudaStream_t s);
constexpr int kNvfp4PairBN = 192;   // pair tile N of the fused (layer-boundary) launches; plain launches: k2_pair_bn
constexpr int kInt4BN = 128;             // N tile of the INT4 GEMM
cudaError_t launch_k2_int4(const K2Maps &maps, const K2Params &p, cudaStream_t s);

// tensor-parallel assembly (tp.cu, SURVEY 8(e) Variant 2): P gathered K-slices -> full K1 outputs
struct TpSliceLayout {
  int64_t xq_off, xs_off, part_off, bytes;   // byte offsets inside one rank's slice
};
TpSliceLayout tp_slice_layout(int fmt, int64_t M, int64_t Kp, int rank);
cudaError_t launch_tp_reduce_partials(int P, int64_t M, int rank, const float *parts, uint16_t *xl1, cudaStream_t s);
cudaError_t launch_tp_assemble(int fmt, int P, int64_t M, int64_t K, int rank, const uint8_t *gathered,
                               int64_t slice_stride, uint8_t *xq, uint8_t *xs, uint16_t *xl1, cudaStream_t s);

// weight-side kernels (wprep.cu)
cudaError_t launch_absmax(const float *R, int64_t n, unsigned int *out_bits, cudaStream_t s);
cudaError_t launch_quantize_residual(const float *R, int64_t K, int64_t N, int fmt, bool scale_bf16,
                                     float gs_w, uint8_t *codes, uint8_t *scales, cudaStream_t s);
cudaError_t launch_codec(const float *in, uint8_t *out, int64_t n, int kind, cudaStream_t s);
// refinement step: Q(R) -> [K][N] fp64 values; out = a - b
cudaError_t launch_dequant_residual64(const uint8_t *codes, const uint8_t *scales, int fmt, bool scale_bf16,
                                      float gs_w, int64_t K, int64_t N, double *out, cudaStream_t s);
cudaError_t launch_sub64(const double *a, const double *b, double *out, int64_t n, cudaStream_t s);
cudaError_t launch_lambda_inv(const float *lam, float *lam_inv, int64_t K, cudaStream_t s);
cudaError_t launch_smooth_weight64(const void *W, int w_dtype, const float *lam, int64_t K, int64_t N,
                                   double *What, cudaStream_t s);
cudaError_t launch_f32_to_f64(const float *in, double *out, int64_t n, cudaStream_t s);
cudaError_t launch_f64_to_f32(const double *in, float *out, int64_t n, cudaStream_t s);
// l1s[row_offset + t][k] = bf16(fl32(m_k * v[k][t])), m_k = lam_inv[k] if given else `scale`
cudaError_t launch_derive_l1s(const void *src, int src_dtype, const float *lam_inv, float scale,
                              int64_t K, int r_src, int row_offset, uint16_t *l1s, cudaStream_t s);
// l2s[n][col_offset + t] = bf16(fl32(v[t][n] / alpha)), l2s row pitch total_rank
cudaError_t launch_derive_l2s(const void *src, int src_dtype, int64_t N, int r_src, int col_offset,
                              int total_rank, float alpha, uint16_t *l2s, cudaStream_t s);
cudaError_t launch_copy_l1s_rows(const uint16_t *src, int64_t K, int rows, uint16_t *dst, cudaStream_t s);
cudaError_t launch_copy_l2s_cols(const uint16_t *src, int64_t N, int r_src, int r_dst, uint16_t *dst,
                                 cudaStream_t s);
cudaError_t launch_eig_to_factors(const double *V, const double *evals, int64_t P, int rank,
                                  double *out_vecs, double *out_sigma, cudaStream_t s);
cudaError_t launch_scale_cols(double *A, int64_t rows, int64_t cols, const double *sig, int invert,
                              int by_row, cudaStream_t s);

}  // namespace svdq
