"""Device format conversions (cvt.rn.satfinite e2m1x2 / e4m3) against the
oracle's table-driven encoders over a structured near-exhaustive fp32 sweep:
every sign x exponent x 11-bit mantissa prefix, each with 16 low-bit
patterns (0, 1, all-ones, ...), so every lattice point, every exact midpoint
and its 1-ulp neighbours are covered (readings Q5, Q11-Q13)."""
import numpy as np
import pytest

from oracle import formats as F

pytestmark = pytest.mark.gpu


def sweep(nonneg=False):
    hi = np.arange(1 << 20, dtype=np.uint64)            # sign(1) + exponent(8) + mantissa prefix(11)
    low = np.array([0, 1, 2, 3, 0x7FF, 0x800, 0x801, 0xFFE, 0xFFF, 0x155, 0xAAA, 0x400, 0x3FF,
                    0xC00, 0x100, 0xF00], dtype=np.uint64)
    bits = ((hi[:, None] << np.uint64(12)) | low[None, :]).reshape(-1).astype(np.uint32)
    v = bits.view(np.float32)
    keep = np.isfinite(v)
    if nonneg:
        keep &= ~np.signbit(v)
    return v[keep]


def test_e2m1_device_matches_oracle():
    import torch
    import paper_2411_05007_b200 as P
    v = sweep()
    v = v[np.abs(v) < 1e30]
    if v.size % 2:
        v = v[:-1]
    out = P.svdq_debug_codec(torch.from_numpy(v).cuda(), 0).cpu().numpy()
    ref_lo = F.e2m1_encode(v[0::2])
    ref_hi = F.e2m1_encode(v[1::2])
    got_lo, got_hi = out & 0xF, out >> 4
    bad = np.flatnonzero((got_lo != ref_lo) | (got_hi != ref_hi))
    assert bad.size == 0, (f"{bad.size} mismatches; first: in={v[2*bad[0]]!r},{v[2*bad[0]+1]!r} "
                           f"got={out[bad[0]]:#x} ref={ref_lo[bad[0]] | (ref_hi[bad[0]] << 4):#x}")


def test_e4m3_device_matches_oracle():
    import torch
    import paper_2411_05007_b200 as P
    v = sweep(nonneg=True)
    out = P.svdq_debug_codec(torch.from_numpy(v).cuda(), 1).cpu().numpy()
    ref = F.e4m3_encode(v)
    bad = np.flatnonzero(out != ref)
    assert bad.size == 0, f"{bad.size} mismatches; first in={v[bad[0]]!r} got={out[bad[0]]:#x} ref={ref[bad[0]]:#x}"
