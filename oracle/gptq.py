"""GPTQ quantization of the residual (App. D: "We use GPTQ [Frantar et al.] to quantize the
residual weights"; Table 3) -- SURVEY 8(f) row 4.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper only cites GPTQ; the procedure below is the cited method's column-by-column algorithm
(Frantar et al., Algorithm 1), written without its lazy-batch blocking (an equivalent reordering
of the same updates), applied to R^T (rows = output channels n, columns = input channels k):

  H    = X_hat^T X_hat   (fp64; X_hat = the smoothed calibration activations of K1, fl32(x * lam_inv))
  dead = diag(H) == 0:  H[dead, dead] = 1,  R^T[:, dead] = 0
  H   += damp * mean(diag(H)) * I                                      (reading G1: damp = 0.01)
  U    = the upper Cholesky factor of H^-1  (H^-1 = U^T U)
  for k = 0 .. K-1:
      at the start of each quantization group (NVFP4 16 / INT4 64 along k), the group's scale is
      computed from the CURRENT (already error-compensated) values of that group (reading G2);
      W8A8's per-channel scale is computed once from the initial rows; NVFP4's per-tensor gs_w
      from the initial residual (reading Q9)
      q_k   = Q(fl32(w_k)) with that scale (the Eq. 1 recipe of quant.py, reading Q10)
      e_k   = (w_k - deq(q_k)) / U[k, k]
      w_j  -= e_k * U[k, j]   for j > k
Sums are fp64.  Returns codes / scales in the same layout as svdquant.quantize_residual.
"""
from __future__ import annotations

import numpy as np

from . import formats as F
from . import quant as Q

F32 = np.float32
DAMP = 0.01      # reading G1 (GPTQ's default percdamp; the paper gives none)


def hessian(xh) -> np.ndarray:
    """H = X_hat^T X_hat in fp64 (the proxy loss ||X_hat R - X_hat Q(R)||^2 has Hessian 2H)."""
    xh = np.asarray(xh, np.float64)
    return xh.T @ xh


def inverse_cholesky_upper(H, damp: float = DAMP):
    """(U, dead): dead-channel fix, dampening, and U upper triangular with (H + d I)^-1 = U^T U."""
    H = np.array(H, dtype=np.float64, copy=True)
    dead = np.diag(H) == 0
    H[dead, dead] = 1.0
    H[np.diag_indices_from(H)] += damp * np.mean(np.diag(H))
    Hinv = np.linalg.inv(H)
    Hinv = 0.5 * (Hinv + Hinv.T)
    try:
        U = np.linalg.cholesky(Hinv).T
    except np.linalg.LinAlgError as e:                 # S:341 "singular H after damping -> error"
        raise ValueError("H not positive definite after dampening") from e
    return U, dead


def _encode_col(v32, fmt, scale_col, scale_dtype, gs):
    """Q(v) of one column (one value per output channel) with the group's stored scale, and its
    exact dequantized value.  Same fp32 recipe as quant.py (reading Q10)."""
    if fmt == "nvfp4":
        sfd = F.e4m3_decode(scale_col).astype(F32)
        den = (sfd * F32(gs)).astype(F32)
        with np.errstate(divide="ignore"):
            qinv = np.where(sfd == 0, F32(0), F32(1.0) / den).astype(F32)
        q = F.e2m1_encode((v32 * qinv).astype(F32))
        return q, F.e2m1_decode(q) * sfd.astype(np.float64) * float(F32(gs))
    if fmt == "int4":
        sd = F.from_bits16(scale_col, scale_dtype).astype(F32)
        with np.errstate(divide="ignore"):
            qinv = np.where(sd == 0, F32(0), F32(1.0) / sd).astype(F32)
        q = np.clip(np.rint((v32 * qinv).astype(F32)), -Q.INT4_QMAX, Q.INT4_QMAX).astype(np.int64)
        return q, q.astype(np.float64) * sd.astype(np.float64)
    if fmt == "w8a8":
        s = np.asarray(scale_col, F32)
        with np.errstate(divide="ignore"):
            qinv = np.where(s == 0, F32(0), F32(1.0) / s).astype(F32)
        q = np.clip(np.rint((v32 * qinv).astype(F32)), -Q.INT8_QMAX, Q.INT8_QMAX).astype(np.int64)
        return q, q.astype(np.float64) * s.astype(np.float64)
    raise ValueError(fmt)


def gptq_quantize_residual(R32, xh, fmt: str, scale_dtype: str = "bf16", damp: float = DAMP):
    """GPTQ of the residual R32 ([K, N] fp32, paper layout) on the smoothed calibration
    activations xh ([M, K]).  Returns (codes [N, K], scales, gs_w) like quantize_residual."""
    Wt = np.array(np.asarray(R32, F32).T, dtype=np.float64)        # [N, K], rows = output channels
    N, K = Wt.shape
    U, dead = inverse_cholesky_upper(hessian(xh), damp)
    Wt[:, dead] = 0.0
    codes = np.zeros((N, K), np.int64)
    if fmt == "nvfp4":
        gs = Q.nvfp4_global_scale(Wt.astype(F32))
        G = Q.NVFP4_GROUP
        scales = np.zeros((N, K // G), np.uint8)
    elif fmt == "int4":
        gs = F32(1.0)
        G = Q.INT4_GROUP
        scales = np.zeros((N, K // G), np.uint16)
    elif fmt == "w8a8":
        gs = F32(1.0)
        G = K
        _, scales = Q.quantize_int8_rows(Wt.astype(F32))          # per channel, from the initial rows
    else:
        raise ValueError(fmt)
    for k in range(K):
        if k % G == 0 and fmt != "w8a8":
            slab = Wt[:, k:k + G].astype(F32)                      # current values of the group
            if fmt == "nvfp4":
                scales[:, k // G] = Q.quantize_nvfp4(slab, gs)[1][:, 0]
            else:
                scales[:, k // G] = Q.quantize_int4(slab, scale_dtype)[1][:, 0]
        col = scales if fmt == "w8a8" else scales[:, k // G]
        q, deq = _encode_col(Wt[:, k].astype(F32), fmt, col, scale_dtype, gs)
        codes[:, k] = q
        e = (Wt[:, k] - deq) / U[k, k]
        Wt[:, k + 1:] -= e[:, None] * U[k, k + 1:][None, :]
    if fmt == "nvfp4":
        codes = codes.astype(np.uint8)
    return codes, scales, F32(gs)


def proxy_loss(R32, xh, deq_kn) -> float:
    """||X_hat R - X_hat deq||_F^2, the layer-wise objective GPTQ minimizes (fp64)."""
    xh = np.asarray(xh, np.float64)
    d = np.asarray(R32, np.float64) - np.asarray(deq_kn, np.float64)
    return float(np.sum((xh @ d) ** 2))
