"""SVDQuant's linear layer, step by step in the paper's order and notation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Problem: X in R^{b x m} (b tokens = GEMM M, m input channels = K),
W in R^{m x n} (n output channels = N).
  1. Smoothing (reading Q1): X_hat = X diag(lambda)^-1,
     W_hat = diag(lambda) W;  lambda_i from App. D.
  2. Low-rank split (Eq. 5): W_hat = L1 L2 + R, with the optimal
     L1 = U Sigma_{:, :r}, L2 = V_{:r, :} from the SVD W_hat = U Sigma V (P:157,
     reading Q2: Sigma folded into L1).
  3. XW ~= X_hat L1 L2 (16-bit branch) + Q(X_hat) Q(R) (4-bit residual), Eq. 5.
Stored operands follow SURVEY §8(b) (readings Q9, Q14, Q15, Q18):
  lam_inv32 = fl32(1 / lambda32);  L1s = bf16(diag(lambda)^-1 L1)^T  [r, K];
  L2s = bf16(L2^T / alpha) [N, r] with alpha = fl32(gs_x * gs_w) (NVFP4) or 1
  (INT4); residual codes/scales of R^T per output channel, groups along K.
Sums are fp64; the quantizer recipe is exact fp32 (oracle/quant.py).
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import formats as F
from . import gptq as G
from . import quant as Q

F32 = np.float32


# --------------------------------------------------------------------------
# Step 1: smoothing factor (App. D)
# --------------------------------------------------------------------------
def compute_smoothing(x_cal, w, alpha: float) -> np.ndarray:
    """lambda_i = max|X_{:,i}|^alpha / max|W_{i,:}|^(1-alpha).

    Clamped to [1e-5, 1e5] so dead channels stay finite.  Returns
    the fp32 lambda the library consumes (the boundary takes fp32 lambda).
    """
    x_cal = np.asarray(x_cal, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    if x_cal.shape[1] != w.shape[0]:
        raise ValueError("shape mismatch: X_cal cols != W rows")
    xa = np.max(np.abs(x_cal), axis=0)
    wa = np.max(np.abs(w), axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        lam = xa ** alpha / wa ** (1.0 - alpha)
    lam = np.where(np.isfinite(lam), lam, 1e5)
    lam = np.clip(lam, 1e-5, 1e5)
    return lam.astype(F32)


def lambda_inverse(lam32) -> np.ndarray:
    """lam_inv32 = fl32(1 / lambda32) -- the fp32 reciprocal K1 multiplies by (Q14)."""
    lam32 = np.asarray(lam32, dtype=F32)
    return (F32(1.0) / lam32).astype(F32)


def smooth_weight(w, lam32) -> np.ndarray:
    """W_hat = diag(lambda) W (P:122 under reading Q1), fp64."""
    return np.asarray(lam32, np.float64)[:, None] * np.asarray(w, np.float64)


# --------------------------------------------------------------------------
# Step 2: low-rank + residual split (Eq. 5)
# --------------------------------------------------------------------------
@dataclass
class Decomposition:
    w_hat: np.ndarray   # [K, N] fp64
    L1: np.ndarray      # [K, r] fp64 = U[:, :r] diag(sigma[:r])
    L2: np.ndarray      # [r, N] fp64 = V[:r, :]
    R: np.ndarray       # [K, N] fp64 = W_hat - L1 L2
    sigma: np.ndarray   # singular values of W_hat, descending


def decompose(w, lam32, r: int, svd=None) -> Decomposition:
    """W_hat = L1 L2 + R with the truncated SVD.

    `svd` may be supplied (e.g. the Jacobi SVD of oracle.linalg for tiny
    shapes); default is LAPACK via numpy.linalg.svd in fp64.
    """
    w_hat = smooth_weight(w, lam32)
    K, N = w_hat.shape
    if not (0 <= r <= min(K, N)):
        raise ValueError("rank out of range (S:133)")
    if svd is None:
        U, s, Vt = np.linalg.svd(w_hat, full_matrices=False)
    else:
        U, s, Vt = svd(w_hat)
    L1 = U[:, :r] * s[:r][None, :]
    L2 = Vt[:r, :]
    R = w_hat - L1 @ L2
    return Decomposition(w_hat, L1, L2, R, s)


# --------------------------------------------------------------------------
# Stored operands (the svdq_linear view of SURVEY §8(b))
# --------------------------------------------------------------------------
@dataclass
class Operands:
    fmt: str                 # 'nvfp4' | 'int4'
    K: int
    N: int
    rank: int
    w_codes: np.ndarray      # [N, K] 4-bit codes (nvfp4: E2M1 code; int4: signed int)
    w_scales: np.ndarray     # nvfp4: E4M3 bytes [N, K/16]; int4: 16-bit bits [N, K/64]
    scale_dtype: str         # int4 scale type 'bf16' | 'fp16' (Q8); nvfp4: 'e4m3'
    gs_w: F32
    gs_x: F32
    lam_inv32: np.ndarray    # [K] fp32
    L1s_bits: np.ndarray     # [r, K] bf16 bits
    L2s_bits: np.ndarray     # [N, r] bf16 bits
    bias: Optional[np.ndarray]  # [N] fp32 values or None

    @property
    def alpha(self) -> F32:
        """Epilogue factor: fl32(gs_x * gs_w) for NVFP4, 1 for INT4 (App. B.5)."""
        if self.fmt == "nvfp4":
            return F32(F32(self.gs_x) * F32(self.gs_w))
        return F32(1.0)

    @property
    def L1s(self) -> np.ndarray:
        return F.bf16_from_bits(self.L1s_bits)

    @property
    def L2s(self) -> np.ndarray:
        return F.bf16_from_bits(self.L2s_bits)


def quantize_residual(R32, fmt: str, scale_dtype: str = "bf16", gs_w=None):
    """Q(R) per output channel with groups along K (reading Q19).

    R32 is [K, N] (paper layout).  Returns (codes [N, K], scales, gs_w).
    NVFP4 gs_w = fl32(amax(|R32|) / 2688) unless given (Q9).
    """
    Rt = np.ascontiguousarray(np.asarray(R32, dtype=F32).T)
    if fmt == "nvfp4":
        gs = Q.nvfp4_global_scale(Rt) if gs_w is None else F32(gs_w)
        codes, sf = Q.quantize_nvfp4(Rt, gs)
        return codes, sf, gs
    if fmt == "int4":
        codes, s = Q.quantize_int4(Rt, scale_dtype)
        return codes, s, F32(1.0)
    if fmt == "w8a8":                                     # per-channel INT8
        codes, s = Q.quantize_int8_rows(Rt)
        return codes, s, F32(1.0)
    raise ValueError(fmt)


def prepare_operands(w, lam32, r: int, fmt: str, gs_x=1.0, scale_dtype="bf16",
                     bias=None, svd=None, decomp: Optional[Decomposition] = None,
                     gptq_x=None, gptq_damp: float = G.DAMP) -> Operands:
    """Offline weight preparation: smoothing, SVD, residual
    quantization, L1s / L2s derivation.  With calibration activations `gptq_x` ([M, K], the
    unsmoothed X), the residual is quantized by GPTQ on X_hat = fl32(x * lam_inv)
    instead of round-to-nearest."""
    lam32 = np.asarray(lam32, dtype=F32)
    d = decomp if decomp is not None else decompose(w, lam32, r, svd=svd)
    K, N = d.w_hat.shape
    R32 = d.R.astype(F32)
    if gptq_x is None:
        codes, scales, gs_w = quantize_residual(R32, fmt, scale_dtype)
    else:
        xh = Q.smooth_activation(gptq_x, lambda_inverse(lam32))
        codes, scales, gs_w = G.gptq_quantize_residual(R32, xh, fmt, scale_dtype, gptq_damp)
    gs_x = F32(gs_x) if fmt == "nvfp4" else F32(1.0)
    lam_inv32 = lambda_inverse(lam32)
    alpha = F32(gs_x * gs_w) if fmt == "nvfp4" else F32(1.0)
    L1s_bits = F.bf16_bits(lam_inv32.astype(np.float64)[:, None] * d.L1).T.copy()   # [r, K]
    L2s_bits = F.bf16_bits(d.L2.T / float(alpha))                                    # [N, r]
    b = None if bias is None else np.asarray(bias, dtype=F32)
    return Operands(fmt, K, N, r, codes, scales,
                    {"nvfp4": "e4m3", "w8a8": "fp32"}.get(fmt, scale_dtype),
                    F32(gs_w), gs_x, lam_inv32, np.ascontiguousarray(L1s_bits),
                    np.ascontiguousarray(L2s_bits), b)


# --------------------------------------------------------------------------
# K1 semantics: smoothing + activation quantization + down-projection
# --------------------------------------------------------------------------
@dataclass
class QuantAct:
    codes: np.ndarray        # [M, K] 4-bit codes (nvfp4) / signed ints (int4)
    scales: np.ndarray       # nvfp4 sf bytes [M, K/16]; int4 16-bit bits [M, K/64]
    xl1_bits: np.ndarray     # [M, r] bf16 bits
    xl1_exact: np.ndarray    # [M, r] fp64 X L1s^T before rounding


def quantize_activation(x, ops: Operands, act_scale_dtype: Optional[str] = None) -> QuantAct:
    """X_hat = X diag(lambda)^-1, Q(X_hat) (Eq. 1 / App. D), and the
    down-projection X_hat L1 = X L1s^T (reading Q18), xl1 stored bf16 (Q15).

    `x` holds the 16-bit activation values (exact in fp32).
    """
    x = np.asarray(x, dtype=F32)
    xh = Q.smooth_activation(x, ops.lam_inv32)
    if ops.fmt == "nvfp4":
        codes, scales = Q.quantize_nvfp4(xh, ops.gs_x)
    elif ops.fmt == "w8a8":                               # per-token dynamic INT8
        codes, scales = Q.quantize_int8_rows(xh)
    else:
        codes, scales = Q.quantize_int4(xh, act_scale_dtype or ops.scale_dtype)
    xl1 = x.astype(np.float64) @ ops.L1s.astype(np.float64).T
    return QuantAct(codes, scales, F.bf16_bits(xl1), xl1)


# --------------------------------------------------------------------------
# K2 semantics: 4-bit GEMM + low-rank up-projection + bias (Eq. 5, App. B.5)
# --------------------------------------------------------------------------
def int4_group_accum(qa, qb) -> np.ndarray:
    """acc_g[m, n] = sum_{k in g} qa[m, k] qb[n, k] exactly (int64), g of 64."""
    qa = np.asarray(qa, dtype=np.int64)
    qb = np.asarray(qb, dtype=np.int64)
    M, K = qa.shape
    N = qb.shape[0]
    G = K // Q.INT4_GROUP
    out = np.empty((G, M, N), dtype=np.int64)
    for g in range(G):
        sl = slice(g * Q.INT4_GROUP, (g + 1) * Q.INT4_GROUP)
        # fp64 products/sums of |q| <= 7 over 64 terms are exact integers
        out[g] = np.rint(qa[:, sl].astype(np.float64) @ qb[:, sl].astype(np.float64).T).astype(np.int64)
    return out


def main_product(act_codes, act_scales, ops: Operands, act_scale_dtype=None) -> np.ndarray:
    """Q(X_hat) Q(R) without the global scales, fp64.

    NVFP4: sum_g f(sfa) f(sfb) sum_{k in g} e2m1(qa) e2m1(qb).
    INT4:  sum_g acc_g * sx[m, g] * sw[n, g].
    """
    if ops.fmt == "nvfp4":
        A = Q.dequantize_nvfp4(act_codes, act_scales, 1.0)
        B = Q.dequantize_nvfp4(ops.w_codes, ops.w_scales, 1.0)
        return A @ B.T
    if ops.fmt == "w8a8":
        # acc = sum_k qa qb exactly (int64; fp64 products/sums of |q| <= 127 are exact below 2^53),
        # then acc * sx[m] * sw[n]
        acc = np.asarray(act_codes, np.float64) @ np.asarray(ops.w_codes, np.float64).T
        return acc * np.asarray(act_scales, np.float64)[:, None] * np.asarray(ops.w_scales, np.float64)[None, :]
    sdt = act_scale_dtype or ops.scale_dtype
    acc = int4_group_accum(act_codes, ops.w_codes)
    sx = F.from_bits16(act_scales, sdt).astype(np.float64)        # [M, G]
    sw = F.from_bits16(ops.w_scales, ops.scale_dtype).astype(np.float64)  # [N, G]
    out = np.zeros(acc.shape[1:], dtype=np.float64)
    for g in range(acc.shape[0]):
        out += acc[g].astype(np.float64) * sx[:, g][:, None] * sw[:, g][None, :]
    return out


def gemm_reference(qact: QuantAct, ops: Operands, act_scale_dtype=None) -> np.ndarray:
    """Y64 = alpha (main + xl1 L2s^T) + bias   (Eq. 5; App. B.5; Q16)."""
    main = main_product(qact.codes, qact.scales, ops, act_scale_dtype)
    xl1 = F.bf16_from_bits(qact.xl1_bits).astype(np.float64)
    low = xl1 @ ops.L2s.astype(np.float64).T if ops.rank else 0.0
    y = float(ops.alpha) * (main + low)
    if ops.bias is not None:
        y = y + ops.bias.astype(np.float64)[None, :]
    return y


def round_output(y64, out_dtype: str) -> np.ndarray:
    """Y_ref = round_to_out_dtype(Y64) (reading Q17)."""
    if out_dtype == "fp32":
        return np.asarray(y64, dtype=np.float64).astype(F32)
    return F.round16(y64, out_dtype)


def forward(x, ops: Operands, out_dtype="bf16", act_scale_dtype=None):
    """End-to-end K1 -> K2 semantics.  Returns (Y_ref, Y64, QuantAct)."""
    qa = quantize_activation(x, ops, act_scale_dtype)
    y64 = gemm_reference(qa, ops, act_scale_dtype)
    return round_output(y64, out_dtype), y64, qa


# --------------------------------------------------------------------------
# Exact-arithmetic forms used by the algebraic pins
# --------------------------------------------------------------------------
def forward_exact(x, lam32, d: Decomposition, deq_act, deq_res) -> np.ndarray:
    """X_hat L1 L2 + Q(X_hat) Q(R) in fp64, Eq. 5, from dequantized operands."""
    xh = np.asarray(x, np.float64) / np.asarray(lam32, np.float64)[None, :]
    return xh @ d.L1 @ d.L2 + deq_act @ deq_res


# --------------------------------------------------------------------------
# LoRA: "fuse the LoRA branch into our low-rank branch by slightly
# increasing the rank"
# --------------------------------------------------------------------------
def lora_fuse(ops: Operands, A, B, scale: float) -> Operands:
    """L1s' = [L1s ; bf16(fl32(scale * A))^T],  L2s' = [L2s | bf16(fl32(B^T / alpha))].

    The branch consumes X (L1s carries diag(lambda)^-1), so the LoRA factor
    A is appended as-is -- S:350's diag(lambda) A pre-multiplied by
    diag(lambda)^-1.  R and its codes are untouched (no re-quantization).
    A: [K, r_l] fp32, B: [r_l, N] fp32.
    """
    A = np.asarray(A, dtype=F32)
    B = np.asarray(B, dtype=F32)
    if A.shape[0] != ops.K or B.shape[1] != ops.N or A.shape[1] != B.shape[0]:
        raise ValueError("LoRA shape mismatch")
    a_s = (A * F32(scale)).astype(F32)                       # fl32(scale * A)
    b_s = (B / ops.alpha).astype(F32)                        # fl32(B / alpha)
    L1s_new = np.concatenate([ops.L1s_bits, F.bf16_bits(a_s).T], axis=0)
    L2s_new = np.concatenate([ops.L2s_bits, F.bf16_bits(b_s).T], axis=1)
    return replace(ops, rank=ops.rank + A.shape[1],
                   L1s_bits=np.ascontiguousarray(L1s_new),
                   L2s_bits=np.ascontiguousarray(L2s_new))


def lowrank_branch_exact(x, L1s, L2s, alpha) -> np.ndarray:
    """alpha * X L1s^T L2s^T in fp64 (no storage rounding)."""
    return float(alpha) * (np.asarray(x, np.float64) @ np.asarray(L1s, np.float64).T
                           @ np.asarray(L2s, np.float64).T)


# --------------------------------------------------------------------------
# Offline: migration-strength search (App. D) -- SURVEY 8(f) row 4
# --------------------------------------------------------------------------
def calibration_error(x_cal, w, ops: Operands) -> float:
    """||X_cal W - forward(X_cal)||_F^2 with the deployed quantized forward (Eq. 5 with the
    residual and activation quantizers, fp64 before output rounding, no bias) -- "the layer
    output mean squared error (MSE) after SVD on the calibration dataset" (reading Q4)."""
    ops_nb = replace(ops, bias=None)
    qa = quantize_activation(x_cal, ops_nb)
    y = gemm_reference(qa, ops_nb)
    ref = np.asarray(x_cal, np.float64) @ np.asarray(w, np.float64)
    return float(np.sum((y - ref) ** 2))


def search_alpha(x_cal, w, rank: int, fmt: str, grid, gs_x=1.0, scale_dtype="bf16"):
    """argmin over the grid of calibration_error(lambda(alpha)); ties -> the smaller alpha.
    Returns (alpha*, lambda32(alpha*), [objective per grid point])."""
    grid = list(grid)
    if not grid:
        raise ValueError("empty alpha grid")
    errs = []
    for a in grid:
        lam = compute_smoothing(x_cal, w, a)
        ops = prepare_operands(w, lam, rank, fmt, gs_x=gs_x, scale_dtype=scale_dtype)
        errs.append(calibration_error(x_cal, w, ops))
    best = min(range(len(grid)), key=lambda i: (errs[i], grid[i]))
    return grid[best], compute_smoothing(x_cal, w, grid[best]), errs



# --------------------------------------------------------------------------
# Offline: iterative low-rank refinement (reading Q3) -- SURVEY 8(f) row 4
# --------------------------------------------------------------------------
def dequantize_residual(ops: Operands) -> np.ndarray:
    """Q(R) as values in the W_hat space, [K, N] fp64 (exact products of the stored codes and
    scales: the per-channel dequantizers of quant.py transposed back to the paper layout)."""
    if ops.fmt == "nvfp4":
        v = Q.dequantize_nvfp4(ops.w_codes, ops.w_scales, ops.gs_w)
    elif ops.fmt == "int4":
        v = Q.dequantize_int4(ops.w_codes, ops.w_scales, ops.scale_dtype)
    elif ops.fmt == "w8a8":
        v = Q.dequantize_int8_rows(ops.w_codes, ops.w_scales)
    else:
        raise ValueError(ops.fmt)
    return np.ascontiguousarray(v.T)


def redecompose(w_hat, deq, r: int) -> Decomposition:
    """One refinement step: "decomposing W - Q(R) and adjusting R accordingly", read as
    (reading Q3) L1 L2 = the rank-r truncated SVD of W_hat - Q(R_{t-1}), R_t = W_hat - L1 L2.
    `sigma` holds the singular values of the decomposed matrix W_hat - Q(R_{t-1})."""
    T = np.asarray(w_hat, np.float64) - np.asarray(deq, np.float64)
    U, s, Vt = np.linalg.svd(T, full_matrices=False)
    L1 = U[:, :r] * s[:r][None, :]
    L2 = Vt[:r, :]
    return Decomposition(np.asarray(w_hat, np.float64), L1, L2, w_hat - L1 @ L2, s)


def refine_lowrank(x_cal, w, lam32, rank: int, fmt: str, iters: int, gs_x=1.0, scale_dtype="bf16",
                   gptq: bool = False, gptq_damp: float = G.DAMP):
    """Iterative refinement of the low-rank branch: iterate 0 is the plain SVD split
    (prepare_operands); iterate t >= 1 re-decomposes W_hat - Q(R_{t-1}) (redecompose) and
    re-quantizes R_t; "then picking the result with the smallest error" -- the iterate with the
    smallest calibration_error (the App. D objective, reading Q4); ties -> the earlier iterate.
    With gptq=True every iterate's residual is quantized by GPTQ on x_cal.
    Returns (best t, Operands of the best iterate, [objective per iterate], [Decomposition per iterate])."""
    if iters < 0:
        raise ValueError("iters must be >= 0")
    lam32 = np.asarray(lam32, dtype=F32)
    d = decompose(w, lam32, rank)
    ops = prepare_operands(w, lam32, rank, fmt, gs_x=gs_x, scale_dtype=scale_dtype, decomp=d,
                           gptq_x=x_cal if gptq else None, gptq_damp=gptq_damp)
    all_ops, errs, decs = [ops], [calibration_error(x_cal, w, ops)], [d]
    for _ in range(iters):
        d = redecompose(d.w_hat, dequantize_residual(ops), rank)
        ops = prepare_operands(w, lam32, rank, fmt, gs_x=gs_x, scale_dtype=scale_dtype, decomp=d,
                               gptq_x=x_cal if gptq else None, gptq_damp=gptq_damp)
        all_ops.append(ops)
        errs.append(calibration_error(x_cal, w, ops))
        decs.append(d)
    best = min(range(len(errs)), key=lambda t: (errs[t], t))
    return best, all_ops[best], errs, decs


# --------------------------------------------------------------------------
# Layer boundary: the next layer's K1 applied to this layer's stored output
# --------------------------------------------------------------------------
def gelu_tanh(v) -> np.ndarray:
    """GELU, tanh form (FLUX's MLP activation; the paper does not restate it), in fp64:
    0.5 v (1 + tanh(sqrt(2/pi) (v + 0.044715 v^3)))."""
    v = np.asarray(v, np.float64)
    return 0.5 * v * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (v + 0.044715 * v ** 3)))


def next_layer_input(y_stored, act: str, dtype: str = "bf16") -> np.ndarray:
    """The next linear's 16-bit input from this layer's stored output (reading N1): identity, or
    round16(gelu_tanh(y)) for MLP-up -> MLP-down."""
    if act == "none":
        return np.asarray(y_stored, np.float64)
    if act == "gelu_tanh":
        return F.round16(gelu_tanh(y_stored), dtype)
    raise ValueError(act)


def fused_next(y64, ops_next: Operands, act: str, dtype: str = "bf16") -> QuantAct:
    """What an epilogue-fused K2 hands to the next layer: K1 (quantize_activation) of
    next_layer_input(round_output(y64)) -- P:165 / P:174's fusion argument carried across the
    layer boundary."""
    a = next_layer_input(round_output(y64, dtype), act, dtype)
    return quantize_activation(a, ops_next)
