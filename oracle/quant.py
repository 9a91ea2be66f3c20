"""Eq. (1) quantizers in the two 4-bit settings of App. D.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. (1):  Q_X = round(X / s_X),  s_X = max|X| / q_max.
App. D:   "per-group symmetric quantization for both activations and
          weights ... INT4 quantization uses a group size of 64 with 16-bit
          scales.  We use NVFP4 ... group size of 16 with FP8 scales".

The fp32 operation order is the canonical recipe of SURVEY App. B (reading
Q10): every step is one correctly-rounded fp32 op, written here as numpy
float32 array ops (IEEE per element, no FMA contraction).  Groups run along
the last axis (K, the reduction axis; reading Q19).
"""
from __future__ import annotations

import numpy as np

from . import formats as F

F32 = np.float32
NVFP4_GROUP = 16
INT4_GROUP = 64
INT4_QMAX = 7         # P:74, 2^(4-1)-1
NVFP4_GS_DIV = F32(6.0 * 448.0)   # q_max(E2M1) * max(E4M3) (reading Q9)


def _groups(v: np.ndarray, g: int) -> np.ndarray:
    v = np.asarray(v, dtype=F32)
    if v.shape[-1] % g:
        raise ValueError(f"last dim {v.shape[-1]} not a multiple of group {g}")
    return v.reshape(v.shape[:-1] + (v.shape[-1] // g, g))


def _check_finite(v):
    if not np.all(np.isfinite(v)):
        raise ValueError("non-finite input (S:199)")


# --------------------------------------------------------------------------
# NVFP4 (App. B.2)
# --------------------------------------------------------------------------
def nvfp4_global_scale(v) -> F32:
    """gs = fl32(amax(|v|) / 2688), or 1.0 when amax == 0 (reading Q9)."""
    v = np.asarray(v, dtype=F32)
    amax = F32(np.max(np.abs(v))) if v.size else F32(0)
    if amax == 0:
        return F32(1.0)
    return F32(amax / NVFP4_GS_DIV)


def quantize_nvfp4(v, gs) -> tuple[np.ndarray, np.ndarray]:
    """Eq. (1) with E2M1 codes (q_max = 6) and E4M3 group scales.

    Per group of 16 along the last axis:
        enc  = fl32(1 / gs);  c6 = fl32(1 / 6)
        amax = max |v_i|
        sf   = e4m3_rn_satfinite(fl32(amax * fl32(enc * c6)))   (s_X, stored)
        qinv = f32(sf) == 0 ? 0 : fl32(1 / fl32(f32(sf) * gs))
        q_i  = e2m1_rn_satfinite(fl32(v_i * qinv))              (round(X/s_X))
    Returns (codes uint8 4-bit [.., K], sf bytes uint8 [.., K/16]).
    """
    v = np.asarray(v, dtype=F32)
    _check_finite(v)
    gs = F32(gs)
    if not gs > 0:
        raise ValueError("gs must be > 0")
    grp = _groups(v, NVFP4_GROUP)
    enc = F32(F32(1.0) / gs)
    c6 = F32(F32(1.0) / F32(6.0))
    t = F32(enc * c6)
    amax = np.max(np.abs(grp), axis=-1).astype(F32)
    sfv = (amax * t).astype(F32)
    sf = F.e4m3_encode(sfv)
    sfd = F.e4m3_decode(sf).astype(F32)
    den = (sfd * gs).astype(F32)
    with np.errstate(divide="ignore"):
        qinv = np.where(sfd == 0, F32(0), (F32(1.0) / den)).astype(F32)
    x = (grp * qinv[..., None]).astype(F32)
    codes = F.e2m1_encode(x).reshape(v.shape)
    return codes, sf


def dequantize_nvfp4(codes, sf, gs) -> np.ndarray:
    """Q(X) = s_X * Q_X: e2m1(q) * f32(sf) * gs, in fp64 (exact)."""
    c = np.asarray(codes)
    vals = F.e2m1_decode(c).reshape(c.shape[:-1] + (c.shape[-1] // NVFP4_GROUP, NVFP4_GROUP))
    s = F.e4m3_decode(sf).astype(np.float64) * float(F32(gs))
    return (vals * s[..., None]).reshape(c.shape)


# --------------------------------------------------------------------------
# INT4 (App. B.3)
# --------------------------------------------------------------------------
def quantize_int4(v, scale_dtype: str) -> tuple[np.ndarray, np.ndarray]:
    """Eq. (1) with signed INT4 codes (q_max = 7) and 16-bit group scales.

    Per group of 64 along the last axis:
        amax = max |v_i|
        s    = to16_rn_satfinite(fl32(amax / 7))        (16-bit scale, Q8)
        qinv = f32(s) == 0 ? 0 : fl32(1 / f32(s))
        q_i  = clamp(rne(fl32(v_i * qinv)), -7, 7)      (Q6, Q7)
    Returns (codes int64 in [-7, 7] [.., K], scale bits uint16 [.., K/64]).
    """
    v = np.asarray(v, dtype=F32)
    _check_finite(v)
    grp = _groups(v, INT4_GROUP)
    amax = np.max(np.abs(grp), axis=-1).astype(F32)
    sv = (amax / F32(INT4_QMAX)).astype(F32)
    s_bits = F.bits16(sv, scale_dtype, satfinite=True)
    sd = F.from_bits16(s_bits, scale_dtype).astype(F32)
    with np.errstate(divide="ignore"):
        qinv = np.where(sd == 0, F32(0), F32(1.0) / sd).astype(F32)
    x = (grp * qinv[..., None]).astype(F32)
    q = np.clip(np.rint(x), -INT4_QMAX, INT4_QMAX).astype(np.int64)
    return q.reshape(v.shape), s_bits


def dequantize_int4(codes, s_bits, scale_dtype: str) -> np.ndarray:
    c = np.asarray(codes).astype(np.float64)
    g = c.reshape(c.shape[:-1] + (c.shape[-1] // INT4_GROUP, INT4_GROUP))
    s = F.from_bits16(s_bits, scale_dtype).astype(np.float64)
    return (g * s[..., None]).reshape(c.shape)


# --------------------------------------------------------------------------
# INT8 (8-bit setting of App. D): "per-token dynamic activation quantization and
# per-channel weight quantization" -- Eq. (1) with q_max = 2^(8-1) - 1 = 127, one scale per
# row of the operand (a token of X_hat, or an output channel of R^T), fp32 scales (reading W1)
# --------------------------------------------------------------------------
INT8_QMAX = 127


def quantize_int8_rows(v) -> tuple[np.ndarray, np.ndarray]:
    """Eq. (1) per row of the last axis:
        amax = max |v_i|;  s = fl32(amax / 127)   (fp32 scale, stored)
        qinv = s == 0 ? 0 : fl32(1 / s)
        q_i  = clamp(rne(fl32(v_i * qinv)), -127, 127)
    Returns (codes int64 [.., K], scales fp32 [..])."""
    v = np.asarray(v, dtype=F32)
    _check_finite(v)
    amax = np.max(np.abs(v), axis=-1).astype(F32) if v.shape[-1] else np.zeros(v.shape[:-1], F32)
    s = (amax / F32(INT8_QMAX)).astype(F32)
    with np.errstate(divide="ignore"):
        qinv = np.where(s == 0, F32(0), F32(1.0) / s).astype(F32)
    x = (v * qinv[..., None]).astype(F32)
    q = np.clip(np.rint(x), -INT8_QMAX, INT8_QMAX).astype(np.int64)
    return q, s


def dequantize_int8_rows(codes, s) -> np.ndarray:
    return np.asarray(codes).astype(np.float64) * np.asarray(s, np.float64)[..., None]


# --------------------------------------------------------------------------
# Smoothing of the activation, P:122 with reading Q14
# --------------------------------------------------------------------------
def smooth_activation(x, lam_inv32) -> np.ndarray:
    """X_hat = X diag(lambda)^-1 as x_hat = fl32(x * lam_inv32)."""
    return (np.asarray(x, dtype=F32) * np.asarray(lam_inv32, dtype=F32)).astype(F32)
