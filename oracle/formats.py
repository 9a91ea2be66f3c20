"""Number formats used by the 4-bit path, written from their definitions.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* E2M1 (FP4): the paper's "4-bit floating-point quantization with 1-bit
  mantissa and 2-bit exponent, q_max = 6".  Representable
  magnitudes {0, .5, 1, 1.5, 2, 3, 4, 6}.  Rounding: nearest, ties to
  the even code (reading Q5); saturating at 6 (Q13); sign from the fp32 sign
  bit so -0 encodes as 0x8 (Q12).
* E4M3 ("FP8 scales"): OCP fn flavour, bias 7, max 448 (0x7E), 0x7F
  NaN; stored unsigned (sign bit 0).  RNE, satfinite (Q9, Q13).
* bf16 / fp16: IEEE-style binary formats, RNE (Q8, Q15, Q17).
* Packing: two 4-bit codes per byte, low nibble = even index.
* NVFP4 scale-factor layout: the 128x4 tile layout.

Everything here works on exact values: fp32 inputs are exact in fp64, every
table value and midpoint is exact in fp64, so comparisons are exact.
"""
from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------
# E2M1
# --------------------------------------------------------------------------
E2M1_MAG = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], dtype=np.float64)
E2M1_QMAX = 6.0


def e2m1_decode(codes) -> np.ndarray:
    """4-bit code (0..15) -> value.  Bit 3 is the sign (0x8 = -0)."""
    c = np.asarray(codes).astype(np.int64)
    mag = E2M1_MAG[c & 7]
    return np.where(c & 8, -mag, mag)


def e2m1_encode(v) -> np.ndarray:
    """fp32 value(s) -> 4-bit E2M1 code, round-to-nearest-even, satfinite.

    Nearest lattice point; when |v| is exactly halfway between two lattice
    points the one with the even code wins (Q5).  |v| > 6 saturates to code 7
    (Q13).  The sign bit is taken from the fp32 sign, so a negative input
    that rounds to zero gives 0x8 (Q12).
    """
    v = np.asarray(v, dtype=np.float32)
    a = np.abs(v).astype(np.float64)
    mids = (E2M1_MAG[:-1] + E2M1_MAG[1:]) / 2.0          # 7 exact midpoints
    code = np.searchsorted(mids, a, side="left")         # # of mids strictly < a
    # exact tie with midpoint i (between code i and i+1): take the even code
    idx = np.clip(code, 0, len(mids) - 1)
    tie = (code < len(mids)) & (a == mids[idx])
    code = np.where(tie, np.where(idx % 2 == 0, idx, idx + 1), code)
    code = np.minimum(code, 7).astype(np.uint8)
    sign = np.signbit(v).astype(np.uint8) << 3
    return (code | sign).astype(np.uint8)


# --------------------------------------------------------------------------
# E4M3 (unsigned use: scale factors)
# --------------------------------------------------------------------------
def _e4m3_table() -> np.ndarray:
    vals = np.empty(127, dtype=np.float64)           # codes 0x00..0x7E
    for code in range(127):
        e = code >> 3
        m = code & 7
        if e == 0:
            vals[code] = (m / 8.0) * 2.0 ** -6        # subnormal, min 2^-9
        else:
            vals[code] = (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return vals


E4M3_VALUES = _e4m3_table()
E4M3_MAX = 448.0


def e4m3_decode(codes) -> np.ndarray:
    """UE4M3 byte (0x00..0x7E) -> value (fp64, exact).  0x7F (NaN) rejected."""
    c = np.asarray(codes).astype(np.int64)
    if np.any((c & 0x7F) == 0x7F):
        raise ValueError("E4M3 NaN code")
    mag = E4M3_VALUES[c & 0x7F]
    return np.where(c & 0x80, -mag, mag)


def e4m3_encode(v) -> np.ndarray:
    """Non-negative fp32 value(s) -> UE4M3 byte, RNE with satfinite (Q9, Q13)."""
    v = np.asarray(v, dtype=np.float32)
    if np.any(np.signbit(v) & (v != 0)):
        raise ValueError("e4m3_encode is for non-negative scale values")
    if not np.all(np.isfinite(v)):
        raise ValueError("non-finite scale value")
    a = v.astype(np.float64)
    t = E4M3_VALUES
    hi = np.searchsorted(t, a, side="left")           # first t[hi] >= a
    hi_c = np.clip(hi, 0, len(t) - 1)
    lo_c = np.clip(hi - 1, 0, len(t) - 1)
    exact = t[hi_c] == a
    mid = (t[lo_c] + t[hi_c]) / 2.0
    pick_hi = (a > mid) | ((a == mid) & (hi_c % 2 == 0))
    code = np.where(exact, hi_c, np.where(pick_hi, hi_c, lo_c))
    code = np.where(a >= E4M3_MAX, 0x7E, code)        # satfinite
    code = np.where(a == 0, 0, code)
    return code.astype(np.uint8)


# --------------------------------------------------------------------------
# bf16 / fp16 (RNE) -- from fp32 or fp64 without double rounding
# --------------------------------------------------------------------------
def _round_to_binary(v64: np.ndarray, mant_bits: int, emin: int) -> np.ndarray:
    """Round exact fp64 values to a binary format with `mant_bits` fraction
    bits and minimum normal exponent `emin`, RNE.  Returns fp64 values on the
    target lattice (overflow is NOT handled here)."""
    a = np.abs(v64)
    _, E = np.frexp(a)                     # a = f * 2^E, f in [0.5, 1)
    e = np.maximum(E - 1, emin)            # exponent of the leading bit
    ulp = np.ldexp(1.0, (e - mant_bits).astype(np.int64))
    q = np.rint(a / ulp) * ulp             # a/ulp is exact; rint = half-even
    q = np.where(a == 0, 0.0, q)
    return np.copysign(q, v64)


def bf16_round(v) -> np.ndarray:
    """fp32/fp64 value(s) -> nearest bf16 value (returned as float32), RNE."""
    v64 = np.asarray(v, dtype=np.float64)
    q = _round_to_binary(v64, 7, -126)
    big = np.abs(q) > 3.3895313892515355e38
    q = np.where(big, np.copysign(np.inf, v64), q)
    return q.astype(np.float32)


def bf16_bits(v) -> np.ndarray:
    """fp32/fp64 value(s) -> bf16 bit pattern (uint16), RNE."""
    f = bf16_round(v)
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def bf16_from_bits(bits) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32)


FP16_MAX = 65504.0


def fp16_round(v, satfinite: bool = False) -> np.ndarray:
    """fp32/fp64 value(s) -> nearest fp16 value (as float32), RNE.
    Overflow -> inf, or +-65504 when `satfinite`."""
    v64 = np.asarray(v, dtype=np.float64)
    q = _round_to_binary(v64, 10, -14)
    over = np.abs(q) > FP16_MAX
    q = np.where(over, np.copysign(FP16_MAX if satfinite else np.inf, v64), q)
    return q.astype(np.float32)


def fp16_bits(v, satfinite: bool = False) -> np.ndarray:
    return fp16_round(v, satfinite).astype(np.float16).view(np.uint16)


def fp16_from_bits(bits) -> np.ndarray:
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float32)


def round16(v, dtype: str, satfinite: bool = False) -> np.ndarray:
    """Round to the named 16-bit type ('bf16' | 'fp16'); value as float32."""
    if dtype == "bf16":
        r = bf16_round(v)
        if satfinite:
            r = np.where(np.isinf(r), np.copysign(np.float32(3.3895313892515355e38), r), r)
        return r.astype(np.float32)
    if dtype == "fp16":
        return fp16_round(v, satfinite)
    raise ValueError(dtype)


def bits16(v, dtype: str, satfinite: bool = False) -> np.ndarray:
    r = round16(v, dtype, satfinite)
    if dtype == "bf16":
        return (r.view(np.uint32) >> 16).astype(np.uint16)
    return r.astype(np.float16).view(np.uint16)


def from_bits16(bits, dtype: str) -> np.ndarray:
    return bf16_from_bits(bits) if dtype == "bf16" else fp16_from_bits(bits)


# --------------------------------------------------------------------------
# Nibble packing: byte j = code[2j] | code[2j+1] << 4
# --------------------------------------------------------------------------
def pack_nibbles(codes) -> np.ndarray:
    c = np.asarray(codes).astype(np.int64) & 0xF
    if c.shape[-1] % 2:
        c = np.concatenate([c, np.zeros(c.shape[:-1] + (1,), np.int64)], axis=-1)
    return (c[..., 0::2] | (c[..., 1::2] << 4)).astype(np.uint8)


def unpack_nibbles(packed) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.shape[:-1] + (2 * p.shape[-1],), dtype=np.uint8)
    out[..., 0::2] = p & 0xF
    out[..., 1::2] = p >> 4
    return out


def int4_to_nibble(q) -> np.ndarray:
    """signed code in [-8, 7] -> two's-complement nibble."""
    return (np.asarray(q).astype(np.int64) & 0xF).astype(np.uint8)


def nibble_to_int4(n) -> np.ndarray:
    n = np.asarray(n).astype(np.int64) & 0xF
    return np.where(n >= 8, n - 16, n).astype(np.int64)


# --------------------------------------------------------------------------
# NVFP4 scale-factor layout: 128x4 tiles
# --------------------------------------------------------------------------
def sf_padded_rows(rows: int) -> int:
    return ((rows + 127) // 128) * 128


def sf_swizzled_size(rows: int, k: int) -> int:
    ncol = k // 16
    ncol_p = ((ncol + 3) // 4) * 4
    return sf_padded_rows(rows) * ncol_p


def sf_offset(row, c, k: int):
    """Byte offset of scale factor (row, c) (c = k-index // 16)."""
    nkt = (k // 16 + 3) // 4
    row = np.asarray(row, dtype=np.int64)
    c = np.asarray(c, dtype=np.int64)
    return ((row // 128) * (nkt * 512) + (c // 4) * 512 + (row % 32) * 16
            + ((row % 128) // 32) * 4 + (c % 4))


def sf_to_layout(sf_rows_by_group: np.ndarray, k: int) -> np.ndarray:
    """[rows, K/16] bytes -> padded 128x4 buffer; padding bytes are 0x00 (Q22)."""
    rows, ncol = sf_rows_by_group.shape
    assert ncol == k // 16
    out = np.zeros(sf_swizzled_size(rows, k), dtype=np.uint8)
    r, c = np.meshgrid(np.arange(rows), np.arange(ncol), indexing="ij")
    out[sf_offset(r, c, k)] = sf_rows_by_group
    return out


def sf_from_layout(buf: np.ndarray, rows: int, k: int) -> np.ndarray:
    ncol = k // 16
    r, c = np.meshgrid(np.arange(rows), np.arange(ncol), indexing="ij")
    return np.asarray(buf, dtype=np.uint8)[sf_offset(r, c, k)]
