/*
 * svdq.h -- C ABI of libsvdq.so: SVDQuant's W4A4 linear with an absorbed
 * 16-bit low-rank branch, B200 (sm_100a) native.
 *
 * The operation (PAPER.md, "P:n" = line n):
 *   X in R^{b x m}, W in R^{m x n}
 *   X_hat = X diag(lambda)^-1,  W_hat = diag(lambda) W               (reading Q1)
 *   W_hat = L1 L2 + R  (truncated SVD, L1 = U Sigma_{:,:r}, L2 = V_{:r,:})
 *   X W ~= X_hat L1 L2  +  Q(X_hat) Q(R)                             (Eq. 5)
 *   Q(.) per-group symmetric: INT4 g64 16-bit scales, NVFP4 g16 E4M3 scales (Eq. 1)
 * computed as two fused kernels (Fig. 5(b)):
 *   K1 svdq_quantize_act_lowrank_down : one read of X -> Q(X_hat) codes + scales, and X L1
 *   K2 svdq_gemm_w4a4_lowrank_up      : Q(X_hat) Q(R) + (X L1) L2 + bias into one output tile
 * LoRA is attached by concatenation into L1 / L2 (svdq_lora_fuse).
 *
 * GEMM naming: M = b (tokens), K = m (input channels), N = n (output channels).
 *
 * Conventions (all entry points)
 *  - Ownership: the caller allocates EVERY buffer (sizes from the *_sizes
 *    queries); the library allocates nothing on the hot path and keeps no
 *    per-layer state.  svdq_linear is a non-owning view that must stay valid
 *    until enqueued work completes.
 *  - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).  Hot
 *    path calls only enqueue work; they never synchronize.  Offline calls that
 *    synchronize say so.
 *  - Errors: a status code is returned; nothing aborts or throws across the ABI.
 *    Arguments are validated on the host before any launch, so outputs are
 *    untouched on error.  svdq_last_error() returns a thread-local detail string.
 *  - Pointers marked [dev] are device pointers, [host] host pointers.
 *  - Packing: 4-bit codes two per byte, low nibble = even K index.
 *    NVFP4 codes are E2M1 (sign-magnitude; -0 = 0x8); INT4 codes are two's
 *    complement in [-7, 7].
 *  - NVFP4 scale factors: unsigned E4M3 bytes in the "128x4" tile layout over
 *    rows padded to a multiple of 128:
 *      off(row, c) = (row/128)*(K/64)*512 + (c/4)*512 + (row%32)*16 + ((row%128)/32)*4 + c%4
 *    with c = k/16.  Padding rows hold 0x00.
 *  - INT4 scales: [rows][K/64] row-major, bf16 or fp16 (reading Q8).
 *  - Preconditions: K % 64 == 0; N % 16 == 0; M >= 1; rank % 16 == 0 and
 *    0 <= rank <= 128; device pointers and row pitches 16-byte aligned.
 */
#ifndef SVDQ_H_
#define SVDQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SVDQ_OK = 0,
  SVDQ_ERR_INVALID_ARGUMENT = 1, /* null pointer, bad enum                         */
  SVDQ_ERR_SHAPE = 2,            /* K%64, N%16, M<1, dimension mismatch           */
  SVDQ_ERR_RANK = 3,             /* rank%16 != 0 or out of [0, 128]               */
  SVDQ_ERR_ALIGNMENT = 4,        /* pointer / pitch not 16-byte aligned           */
  SVDQ_ERR_UNSUPPORTED = 5,      /* device is not sm_100, or format/dtype combo   */
  SVDQ_ERR_NONFINITE = 6,        /* reserved (hot path never scans inputs)        */
  SVDQ_ERR_CUDA = 7,             /* CUDA / cuBLAS / cuSOLVER failure              */
  SVDQ_ERR_WORKSPACE = 8         /* workspace too small                          */
} svdq_status;

/* SVDQ_FMT_W8A8: the paper's 8-bit setting (App. D): per-token dynamic INT8
 * activations and per-channel INT8 weights, q_max = 127, fp32 scales (one per token / output
 * channel), Eq. (1); any rank (the paper uses 16).  Codes are int8 bytes [rows][K];
 * activation scales fp32 [M]; weight scales fp32 [N].  K1 reads each token row twice (the
 * per-token scale needs the whole row); K2 accumulates the whole K exactly in int32 on
 * tcgen05 kind::i8 and scales once per tile. */
typedef enum { SVDQ_FMT_NVFP4 = 0, SVDQ_FMT_INT4 = 1, SVDQ_FMT_W8A8 = 2 } svdq_format;
typedef enum { SVDQ_BF16 = 0, SVDQ_FP16 = 1, SVDQ_FP32 = 2 } svdq_dtype;

/* Quantized linear layer: non-owning view of caller-owned device buffers. */
typedef struct svdq_linear {
  int32_t fmt;              /* svdq_format                                              */
  int32_t rank;             /* r (+ LoRA ranks), multiple of 16, <= 128                 */
  int64_t K;                /* input channels  (paper m)                                */
  int64_t N;                /* output channels (paper n)                                */
  const uint8_t *w_codes;   /* [dev] [N][K/2]: Q(R)^T, K-major                          */
  const uint8_t *w_scales;  /* [dev] NVFP4: 128x4 layout over (ceil(N/128)*128, K/16);  */
                            /*       INT4 : [N][K/64] of scale_dtype                    */
  const float *lambda_inv;  /* [dev] [K] fp32 = fl32(1 / lambda)                        */
  const uint16_t *l1s;      /* [dev] [rank][K] bf16 = (diag(lambda)^-1 L1)^T             */
  const uint16_t *l2s;      /* [dev] [N][rank] bf16 = L2^T / alpha                      */
  const void *bias;         /* [dev] [N] of bias_dtype, or NULL                         */
  int32_t scale_dtype;      /* INT4: SVDQ_BF16 | SVDQ_FP16 (weights AND activations)    */
  int32_t bias_dtype;       /* SVDQ_BF16 | SVDQ_FP16 | SVDQ_FP32                        */
  float gs_w;               /* NVFP4 per-tensor weight decode scale; INT4: 1            */
  float gs_x;               /* NVFP4 static activation decode scale (default 1); INT4: 1 */
} svdq_linear;
/* alpha = fl32(gs_x * gs_w) for NVFP4, 1 for INT4; the GEMM epilogue computes
 * Y = out_rn(fl32(alpha * acc) + bias).                                        */

/* ---------------------------------------------------------------- sizes */
/* Bytes of K1's outputs for M tokens: xq [M][K/2] (W8A8: [M][K]); xs (NVFP4: 128x4 layout
 * over ceil(M/128)*128 rows; INT4: [M][K/64] 16-bit; W8A8: [M] fp32); xl1 [M][rank] bf16. */
svdq_status svdq_act_buffer_sizes(int32_t fmt, int64_t M, int64_t K, int32_t rank,
                                  size_t *xq_bytes, size_t *xs_bytes, size_t *xl1_bytes);
/* Bytes of a layer's weight operands. */
svdq_status svdq_weight_buffer_sizes(int32_t fmt, int64_t K, int64_t N, int32_t rank,
                                     size_t *codes_bytes, size_t *scales_bytes,
                                     size_t *l1s_bytes, size_t *l2s_bytes);

/* ---------------------------------------------------------------- hot path */
/* K1: smoothing + activation quantization + low-rank down-projection, one read of X.
 *   x_hat[m,k] = fl32(x[m,k] * lambda_inv[k])                       (reading Q14)
 *   NVFP4 per (m, 16-group): sf = e4m3(fl32(amax * fl32(fl32(1/gs_x) * fl32(1/6))));
 *         qinv = sf==0 ? 0 : fl32(1/fl32(sf*gs_x)); code = e2m1_rn_sat(fl32(x_hat*qinv))
 *   INT4  per (m, 64-group): s = to16(fl32(amax/7)); qinv = s==0 ? 0 : fl32(1/s);
 *         code = clamp(rne(fl32(x_hat*qinv)), -7, 7)               (Eq. 1)
 *   xl1[m,t] = bf16_rn(sum_k x[m,k] * l1s[t,k]), fp32 accumulation  (reading Q15/Q18)
 * X: [dev] [M][ldx] of x_dtype (BF16 | FP16), ldx >= K elements, ldx % 8 == 0.
 * xq: [dev] [M][K/2]; xs: [dev] (see sizes); xl1: [dev] [M][rank] (may be NULL if rank == 0).
 * Bit-exact contract: xq and xs equal the oracle's codes / scales for the same X,
 * lambda_inv and gs_x, including the 0x00 padding rows of the NVFP4 layout.
 * Implementation (k1_rows.cu): one CTA per 16/32/64/128 whole rows, TMA-staged X, the
 * down-projection on tcgen05 (fp16 X as exact bf16 hi + lo parts); xl1 is deterministic.  */
svdq_status svdq_quantize_act_lowrank_down(const svdq_linear *L, const void *X, int32_t x_dtype,
                                           int64_t M, int64_t ldx, uint8_t *xq, uint8_t *xs,
                                           uint16_t *xl1, void *stream);

/* Grouped K1: n (1..4) independent problems (bf16 or fp16 X; layers sharing format, rank and
 * INT4 scale dtype; no W8A8) in ONE launch whose row tiles are the concatenation of the
 * problems' row tiles.  Problem i computes svdq_quantize_act_lowrank_down(layers[i], X[i],
 * x_dtype, M[i], ldx[i], xq[i], xs[i], xl1[i]): xq / xs bit-identical; xl1 bit-identical when
 * the single launch uses the same row tile (the kernel sizes its row tile -- and with it the
 * fp32 summation order of xl1 -- from the launch's total rows), else within the xl1 tolerance.
 * Arrays are [host], n entries each.  SVDQ_ERR_UNSUPPORTED for mixed format / rank or W8A8.  */
svdq_status svdq_quantize_act_lowrank_down_grouped(int32_t n, const svdq_linear *const *layers,
                                                   const void *const *X, int32_t x_dtype, const int64_t *M,
                                                   const int64_t *ldx, uint8_t *const *xq, uint8_t *const *xs,
                                                   uint16_t *const *xl1, void *stream);

/* ---------------------------------------------------------------- tensor parallelism (C5)
 * SURVEY 8(e) Variant 2, "quantize, then gather" (north star: column-parallel over the 8xB200
 * box, all-gather only where the next layer needs the full activation; the paper itself is
 * single-GPU).  A layer whose input X [M][K] is held column-sharded over P ranks (rank p
 * holds X[:, p Kp : (p+1) Kp), Kp = K/P, e.g. its shard of the previous column-parallel layer's
 * output) runs K1 on its slice, the ranks all-gather the packed slices (0.5625 B per element + an
 * fp32 [M][rank] partial, instead of 2 B per element for a bf16 gather), and every rank assembles
 * the full K1 outputs -- then K2 runs on its own N-shard.  Codes and scales equal those of K1 on
 * the full X bit for bit (groups never straddle slices: Kp % 64 == 0); xl1 = bf16 of the fp32
 * partials summed in rank order (deterministic, identical on every rank).  NVFP4 / INT4 only
 * (W8A8's per-token scale needs the whole row: SVDQ_ERR_UNSUPPORTED).
 *
 * Slice layout (one rank's contribution, `slice_bytes`): codes [M][Kp/2] at xq_off, scales at
 * xs_off (NVFP4: the 128x4 layout over (M, Kp); INT4: [M][Kp/64] 16-bit), fp32 partial
 * X_p L1s[:, slice]^T [M][rank] at part_off; offsets 256-byte aligned.                        */
svdq_status svdq_tp_slice_sizes(int32_t fmt, int64_t M, int64_t Kp, int32_t rank, size_t *xq_off, size_t *xs_off,
                                size_t *part_off, size_t *slice_bytes);
/* K1 of layer L (full K: lambda_inv, l1s are the replicated full operands) on input channels
 * [k0, k0 + Kp): X [dev] [M][ldx] holds those Kp channels; writes one slice [dev] (layout above).
 * k0, Kp multiples of 64.                                                                       */
svdq_status svdq_quantize_act_lowrank_down_kslice(const svdq_linear *L, int64_t k0, int64_t Kp, const void *X,
                                                  int32_t x_dtype, int64_t M, int64_t ldx, uint8_t *slice,
                                                  void *stream);
/* Fused packed all-gather: no collective.  Every rank owns a GATHER buffer
 * (svdq_tp_gather_sizes: the full K1 outputs xq [M][K/2] at xq_off and xs at xs_off, laid out exactly
 * like svdq_quantize_act_lowrank_down's, then P fp32 partial slots [P][M][rank] at part_off).
 * svdq_quantize_act_lowrank_down_kslice_fused runs K1 on input channels [k0, k0 + Kp) and stores
 * its codes / scales at their place in the full-K layout and its partial in slot p of EVERY buffer
 * bufs[0..nbuf) (16-byte aligned device addresses: with symmetric memory, the ranks' buffers mapped
 * over NVLink), so the gather happens inside K1.  After a cross-rank barrier (system-scope
 * release/acquire; the caller's) svdq_tp_reduce_partials sums the P slots in rank order into the
 * bf16 xl1 and K2 reads xq / xs from the gather buffer: codes / scales bit-identical to K1 on the
 * full X, xl1 identical to the all-gather path's.                                                 */
svdq_status svdq_tp_gather_sizes(int32_t fmt, int64_t M, int64_t K, int32_t rank, int32_t P, size_t *xq_off,
                                 size_t *xs_off, size_t *part_off, size_t *bytes);
svdq_status svdq_quantize_act_lowrank_down_kslice_fused(const svdq_linear *L, int64_t k0, int64_t Kp, const void *X,
                                                        int32_t x_dtype, int64_t M, int64_t ldx, int32_t P,
                                                        int32_t p, uint8_t *const *bufs, int32_t nbuf,
                                                        void *stream);
/* xl1 [dev] [M][rank] bf16 = bf16(sum_{p < P} parts[p][M][rank]) summed in p order.               */
svdq_status svdq_tp_reduce_partials(int32_t P, int64_t M, int32_t rank, const float *parts, uint16_t *xl1,
                                    void *stream);
/* gathered [dev] = the P slices in rank order, slice p at gathered + p * slice_stride (0 = slice_bytes:
 * back to back, as all_gather_into_tensor of one slice per rank leaves them; larger when several
 * layers' slices travel in one gather); writes the full xq [M][K/2], xs and xl1 [M][rank] bf16
 * exactly as K1 on the full X would lay them out (K = P Kp).                                    */
svdq_status svdq_tp_assemble_act(int32_t fmt, int32_t P, int64_t M, int64_t K, int32_t rank, const uint8_t *gathered,
                                 size_t slice_bytes, size_t slice_stride, uint8_t *xq, uint8_t *xs, uint16_t *xl1,
                                 void *stream);

/* K2: 4-bit GEMM with the low-rank up-projection folded into the same accumulator.
 *   NVFP4: acc[m,n] = sum_g f(sfa[m,g]) f(sfb[n,g]) sum_{k in g} e2m1(qa) e2m1(qb)
 *                     + sum_t xl1[m,t] l2s[n,t]          (tcgen05 kind::mxf4nvf4 + kind::f16)
 *          Y = out_rn(fl32(alpha * acc) + bias[n])
 *   INT4:  acc_g = sum_{k in g64} qa qb (exact int32, kind::i8);
 *          Y = out_rn(sum_g fl32(fl32(float(acc_g) * sx[m,g]) * sw[n,g]) + sum_t xl1 l2s + bias)
 * Y: [dev] [M][ldy] of y_dtype (BF16 | FP16 | FP32), ldy >= N, ldy % 8 == 0.       */
svdq_status svdq_gemm_w4a4_lowrank_up(const svdq_linear *L, const uint8_t *xq, const uint8_t *xs,
                                      const uint16_t *xl1, int64_t M, void *Y, int32_t y_dtype,
                                      int64_t ldy, void *stream);

/* Grouped K2: n (1..4) independent NVFP4 problems in ONE persistent launch (e.g. the image-
 * and text-stream linears of a FLUX double block, which share no data).  Problem i is exactly
 * svdq_gemm_w4a4_lowrank_up(layers[i], xq[i], xs[i], xl1[i], M[i], Y[i], y_dtype, ldy[i]) and
 * produces bit-identical Y; all problems run on the CTA-pair kernel, whose CTA pairs walk the
 * concatenated tile lists (one tail instead of n).  Arrays are [host], n entries each;
 * pointers inside follow svdq_gemm_w4a4_lowrank_up.  SVDQ_ERR_UNSUPPORTED for INT4 layers;
 * SVDQ_ERR_INVALID_ARGUMENT for n outside 1..4 or NULL arrays.                      */
svdq_status svdq_gemm_w4a4_lowrank_up_grouped(int32_t n, const svdq_linear *const *layers,
                                              const uint8_t *const *xq, const uint8_t *const *xs,
                                              const uint16_t *const *xl1, const int64_t *M, void *const *Y,
                                              int32_t y_dtype, const int64_t *ldy, void *stream);

/* Convenience: K1 then K2 on one stream.  ws: [dev] >= xq+xs+xl1 bytes (16-B aligned parts). */
svdq_status svdq_linear_forward(const svdq_linear *L, const void *X, int32_t x_dtype, int64_t M,
                                int64_t ldx, void *Y, int32_t y_dtype, int64_t ldy, void *ws,
                                size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------- offline (weights) */
/* Quantize a residual R (fp32, paper layout [K][N]) per output channel, groups along K.
 *   NVFP4: gs_w = fl32(amax(|R|) / 2688) (or 1 if amax == 0) unless *gs_w > 0 on input;
 *          codes / sf by the recipe of K1 with gs = gs_w.  INT4: 16-bit scales of scale_dtype.
 * codes: [dev] [N][K/2]; scales: [dev] (svdq_weight_buffer_sizes); gs_w: [host] in/out.
 * Synchronizes `stream` when it must compute gs_w.  Bit-exact against the oracle.   */
svdq_status svdq_quantize_residual(const float *R, int64_t K, int64_t N, int32_t fmt,
                                   int32_t scale_dtype, uint8_t *codes, uint8_t *scales,
                                   float *gs_w, void *stream);

/* Workspace bytes for svdq_quantize_weights. */
svdq_status svdq_quantize_weights_workspace(int64_t K, int64_t N, int32_t rank, size_t *ws_bytes);

/* Layer-boundary fusion (P:165 / P:174's fusion argument carried to the next
 * layer): grouped K2 (CTA-pair NVFP4 kernel, n = 1..4 problems) whose epilogue also runs the NEXT
 * layer's K1 on its own output, so the next layer needs no K1 launch and no re-read of Y:
 *   y = bf16(fl32(alpha * acc) + bias)            (this layer's output, stored to Y[i] if non-NULL)
 *   a = y (act 0) | bf16(gelu_tanh(y)) (act 1)    (reading N1; MLP-up -> MLP-down)
 *   xq_next / xs_next = K1's NVFP4 codes / scale factors of a with nexts[i]'s lambda_inv and gs_x
 *   xl1_next = bf16(a L1s_next^T)                 (partial fp32 sums per 256-row block and CTA pair,
 *                                                   reduced in fixed order by a second kernel)
 * i.e. exactly svdq_quantize_act_lowrank_down(nexts[i], a) -- codes / scales bit-identical for
 * act 0; xl1 within K1's tolerance.  Requirements: layers and nexts NVFP4, nexts[i]->K ==
 * layers[i]->N, nexts[i]->rank in {0, 16, 32}; Y (if given) bf16 with ldy = N.  xq_next[i]:
 * [dev] [M][N/2]; xs_next[i]: [dev] K1's scale-factor buffer for (M, K = N); xl1_next[i]: [dev]
 * [M][rank_next] bf16.  ws: [dev] of svdq_gemm_fused_next_workspace bytes (0 when every
 * next rank is 0).  Enqueue only (two launches when any next rank > 0).                  */
svdq_status svdq_gemm_fused_next_workspace(int32_t n, const svdq_linear *const *layers, const int64_t *M,
                                           const svdq_linear *const *nexts, size_t *ws_bytes);
svdq_status svdq_gemm_w4a4_lowrank_up_fused_next(int32_t n, const svdq_linear *const *layers,
                                                 const uint8_t *const *xq, const uint8_t *const *xs,
                                                 const uint16_t *const *xl1, const int64_t *M, void *const *Y,
                                                 const svdq_linear *const *nexts, int32_t act,
                                                 uint8_t *const *xq_next, uint8_t *const *xs_next,
                                                 uint16_t *const *xl1_next, void *ws, size_t ws_bytes,
                                                 void *stream);

/* Full offline weight preparation:
 *   lambda_inv = fl32(1/lambda); W_hat = diag(lambda) W;  SVD of W_hat (cuBLAS/cuSOLVER fp64
 *   Gram + eigensolver) unless L1_opt / L2_opt are given ([dev] fp32 [K][rank] / [rank][N]);
 *   R = W_hat - L1 L2;  svdq_quantize_residual(R);  l1s = bf16(fl32(lambda_inv[k] * L1[k,t]))^T;
 *   l2s = bf16(fl32(L2[t,n] / alpha))^T.
 * W: [dev] [K][N] of w_dtype (paper layout).  lambda: [dev] [K] fp32 > 0.
 * dst: fmt/rank/K/N set by the call; its buffer pointers (w_codes, w_scales,
 * lambda_inv, l1s, l2s) must point to writable caller allocations; bias is left as is.
 * Synchronizes `stream`.  Parity: L1 L2 within 1e-5 of the oracle's (relative to |W_hat|),
 * codes bit-exact given R (see svdq_quantize_residual).                           */
svdq_status svdq_quantize_weights(const void *W, int32_t w_dtype, const float *lambda, int64_t K,
                                  int64_t N, int32_t rank, int32_t fmt, int32_t scale_dtype,
                                  float gs_x, const float *L1_opt, const float *L2_opt,
                                  svdq_linear *dst, void *ws, size_t ws_bytes, void *stream);

/* Offline migration-strength search (App. D).  For each alpha in
 * grid ([host], n_grid values in [0, 1]): lambda_k = clamp(max|X_cal[:,k]|^alpha /
 * max|W[k,:]|^(1-alpha), 1e-5, 1e5) (fp64, non-finite -> 1e5, stored fp32), the full weight
 * preparation of svdq_quantize_weights, the deployed K1 -> K2 forward on X_cal without bias, and
 * the objective ||X_cal W - Y||_F^2 (fp64 sum, reference X_cal W in fp32 cuBLAS).
 * Returns alpha* = argmin (ties -> the smaller alpha) in *alpha_out [host], lambda(alpha*) in
 * lambda_out [dev, K] fp32 and every objective in objective_out [host, n_grid].
 * X_cal: [dev] [M_cal][ldx] BF16 | FP16.  W: [dev] [K][N] fp32.  ws: [dev] of
 * svdq_search_alpha_workspace bytes.  Synchronizes `stream`.                              */
svdq_status svdq_search_alpha_workspace(int32_t fmt, int64_t M_cal, int64_t K, int64_t N, int32_t rank,
                                        size_t *ws_bytes);
svdq_status svdq_search_alpha(const void *X_cal, int32_t x_dtype, int64_t M_cal, int64_t ldx, const float *W,
                              int64_t K, int64_t N, int32_t rank, int32_t fmt, int32_t scale_dtype, float gs_x,
                              const float *grid, int32_t n_grid, float *alpha_out, float *lambda_out,
                              double *objective_out, void *ws, size_t ws_bytes, void *stream);

/* Iterative low-rank refinement (reading Q3).  Iterate 0 is
 * svdq_quantize_weights(W, lambda); iterate t = 1..iters re-decomposes
 * W_hat - Q(R_{t-1}) (Q(R_{t-1}) dequantized exactly to fp64 from iterate t-1's codes and
 * scales; truncated SVD as in svdq_quantize_weights), sets R_t = W_hat - L1 L2 and re-quantizes.
 * Each iterate is scored with the objective of svdq_search_alpha (K1 -> K2 on X_cal, no bias,
 * ||X_cal W - Y||_F^2); "picking the result with the smallest error": the best iterate (ties ->
 * the earlier) is written to dst (same buffer contract as svdq_quantize_weights; bias untouched),
 * its index to *best_out [host] and all iters + 1 objectives to objective_out [host].
 * use_gptq != 0: every iterate's residual is quantized by GPTQ on X_cal with dampening `damp`
 * (svdq_quantize_weights_gptq) instead of round-to-nearest.
 * X_cal: [dev] [M_cal][ldx] BF16 | FP16.  W: [dev] [K][N] fp32.  lambda: [dev] [K] fp32 > 0.
 * ws: [dev] of svdq_refine_lowrank_workspace bytes.  iters >= 0.  Synchronizes `stream`. */
svdq_status svdq_refine_lowrank_workspace(int32_t fmt, int64_t M_cal, int64_t K, int64_t N, int32_t rank,
                                          int32_t use_gptq, size_t *ws_bytes);
svdq_status svdq_refine_lowrank(const void *X_cal, int32_t x_dtype, int64_t M_cal, int64_t ldx, const float *W,
                                const float *lambda, int64_t K, int64_t N, int32_t rank, int32_t fmt,
                                int32_t scale_dtype, float gs_x, int32_t iters, int32_t use_gptq, float damp,
                                svdq_linear *dst, int32_t *best_out, double *objective_out, void *ws, size_t ws_bytes,
                                void *stream);

/* GPTQ quantization of the residual (App. D: "We use GPTQ to quantize the residual
 * weights"; readings G1-G3 in DESIGN.md).  The cited method's column-by-column procedure on
 * R^T: H = X_hat^T X_hat (fp64) with X_hat = fl32(X_cal * lambda_inv) (K1's smoothing),
 * channels with H_kk == 0 get H_kk = 1 and a zero residual row, H += damp * mean(diag H) * I,
 * U = upper Cholesky factor of H^-1; input channels k = 0..K-1 are quantized in order, each
 * group's scale (NVFP4 16 / INT4 64) taken from the error-compensated values at the group start,
 * W8A8 channel scales and the NVFP4 gs_w from the initial residual (as svdq_quantize_residual),
 * and the error (r_k - deq(q_k)) / U_kk is propagated to the remaining channels via row k of U.
 * Output codes / scales have exactly the layout of svdq_quantize_residual.
 *
 * svdq_quantize_residual_gptq: R [dev] [K][N] fp32 (paper layout, read only); lambda_inv [dev]
 *   [K] fp32; X_cal [dev] [M_cal][ldx] BF16 | FP16; damp >= 0 (0.01 = GPTQ's default).  *gs_w
 *   [host] receives the NVFP4 per-tensor scale (1 otherwise).  ws: [dev] of
 *   svdq_quantize_residual_gptq_workspace bytes.  SVDQ_ERR_INVALID_ARGUMENT if H is not positive
 *   definite after dampening.  Synchronizes `stream`.
 * svdq_quantize_weights_gptq: svdq_quantize_weights (no L1_opt / L2_opt) with the residual
 *   quantized by GPTQ on (X_cal, lambda); ws: [dev] of svdq_quantize_weights_gptq_workspace bytes. */
svdq_status svdq_quantize_residual_gptq_workspace(int64_t M_cal, int64_t K, int64_t N, size_t *ws_bytes);
svdq_status svdq_quantize_residual_gptq(const float *R, int64_t K, int64_t N, int32_t fmt, int32_t scale_dtype,
                                        const void *X_cal, int32_t x_dtype, int64_t M_cal, int64_t ldx,
                                        const float *lambda_inv, float damp, uint8_t *codes, uint8_t *scales,
                                        float *gs_w, void *ws, size_t ws_bytes, void *stream);
svdq_status svdq_quantize_weights_gptq_workspace(int64_t M_cal, int64_t K, int64_t N, int32_t rank,
                                                 size_t *ws_bytes);
svdq_status svdq_quantize_weights_gptq(const void *W, int32_t w_dtype, const float *lambda, int64_t K, int64_t N,
                                       int32_t rank, int32_t fmt, int32_t scale_dtype, float gs_x, const void *X_cal,
                                       int32_t x_dtype, int64_t M_cal, int64_t ldx, float damp, svdq_linear *dst,
                                       void *ws, size_t ws_bytes, void *stream);

/* LoRA fusion: dst->l1s = [src->l1s ; bf16(fl32(scale*A))^T] ([r+r_l][K]),
 * dst->l2s = [src->l2s | bf16(fl32(B/alpha))^T] ([N][r+r_l]); codes / scales untouched
 * (no re-quantization).  A: [dev] [K][r_l], B: [dev] [r_l][N] of ab_dtype
 * (BF16 | FP16 | FP32).  dst must point to writable l1s / l2s of the new rank; all other
 * fields are copied from src.  r_l % 16 == 0.  Enqueue only.                          */
svdq_status svdq_lora_fuse(const svdq_linear *src, const void *A, const void *B, int32_t ab_dtype,
                           int32_t r_l, float scale, svdq_linear *dst, void *stream);

/* ---------------------------------------------------------------- test hooks */
/* INT4 per-group exact accumulators: acc[g][m][n] = sum_{k in g64} qa[m,k] qb[n,k] (int32),
 * computed on the same kind::i8 tensor-core path as K2.  xq [dev] [M][K/2], wq [dev] [N][K/2],
 * acc [dev] [K/64][M][N].  Test hook for the bit-exact accumulator pin.               */
svdq_status svdq_debug_int4_group_accum(const uint8_t *xq, const uint8_t *wq, int64_t M, int64_t N,
                                        int64_t K, int32_t *acc, void *stream);
/* Device codecs for the exhaustive format test: out[i] = e2m1x2 byte of (in[2i], in[2i+1])
 * (cvt.rn.satfinite, low nibble = in[2i]) when kind == 0; e4m3 byte of in[i] when kind == 1. */
svdq_status svdq_debug_codec(const float *in, uint8_t *out, int64_t n, int32_t kind, void *stream);

/* ---------------------------------------------------------------- misc */
const char *svdq_status_string(svdq_status s);
const char *svdq_last_error(void);
/* Number of this library's kernel launches issued by the calling thread (for bench claims). */
uint64_t svdq_launch_count(void);
int32_t svdq_version(void);
/* Rows per CTA (16 / 32 / 64 / 128) the K1 kernel uses on the current device for a launch over
 * `rows_padded` rows (sum of ceil(M_i/128)*128 over a group) at this rank: the smallest tile whose
 * CTA count still fits one wave of SMs with 128/tile * rank <= 256.  Host-only query.          */
int32_t svdq_k1_row_tile(int64_t rows_padded, int32_t rank);

#ifdef __cplusplus
}
#endif
#endif /* SVDQ_H_ */
