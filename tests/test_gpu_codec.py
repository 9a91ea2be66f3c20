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


# ---------------------------------------------------------------------------------------------
# Exhaustive: every finite fp32 bit pattern through the
# device cvt, checked against the oracle's table-driven encoders on the host cores in parallel.
# ---------------------------------------------------------------------------------------------
CHUNK = 1 << 26


def _check_chunk(args):
    kind, start, n, got = args
    bits = (np.arange(start, start + n, dtype=np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    v = bits.view(np.float32)
    if kind == 0:
        ev, od = v[0::2], v[1::2]
        ok = np.isfinite(ev) & np.isfinite(od)
        # device byte = e2m1x2(in[2i], in[2i+1]) as svdq_debug_codec documents
        ref = (F.e2m1_encode(np.where(np.isfinite(od), od, 0)).astype(np.uint8) << 4) | \
            F.e2m1_encode(np.where(np.isfinite(ev), ev, 0)).astype(np.uint8)
        bad = np.flatnonzero(ok & (got != ref))
        first = int(bits[2 * bad[0]]) if bad.size else None
    else:
        ok = np.isfinite(v) & ~np.signbit(v)
        ref = F.e4m3_encode(np.where(ok, v, 0))
        bad = np.flatnonzero(ok & (got != ref))
        first = int(bits[bad[0]]) if bad.size else None
    return int(bad.size), first, int(ok.sum())


def _exhaustive(kind, lo, hi):
    import concurrent.futures as cf
    import os
    import torch
    import paper_2411_05007_b200 as P
    workers = max(1, min(32, len(os.sched_getaffinity(0))))
    futs, covered = [], 0
    with cf.ProcessPoolExecutor(workers) as ex:
        for start in range(lo, hi, CHUNK):
            n = min(CHUNK, hi - start)
            b = torch.arange(start, start + n, dtype=torch.int64, device="cuda")
            v = torch.where(b >= 1 << 31, b - (1 << 32), b).to(torch.int32).view(torch.float32)
            got = P.svdq_debug_codec(v, kind).cpu().numpy()
            futs.append(ex.submit(_check_chunk, (kind, start, n, got)))
        for f in futs:
            nbad, first, nok = f.result()
            assert nbad == 0, f"{nbad} mismatches; first input bits {first:#010x}"
            covered += nok
    return covered


def test_e2m1_exhaustive_all_fp32():
    """The E2M1 encoder on every finite fp32 bit pattern (consecutive patterns paired)."""
    covered = _exhaustive(0, 0, 1 << 32)
    assert covered >= (1 << 31) - (1 << 24)          # pairs with both elements finite


def test_e4m3_exhaustive_all_nonneg_fp32():
    """The UE4M3 scale encoder on every finite non-negative fp32 bit pattern (+0 .. 0x7F7FFFFF)."""
    covered = _exhaustive(1, 0, 0x7F800000)
    assert covered == 0x7F800000
