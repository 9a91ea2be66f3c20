"""Shared test plumbing: move oracle operands into device buffers of the
C-ABI layout (packing / scale-factor layout only -- no method arithmetic),
and read device results back into oracle form."""
from __future__ import annotations

import numpy as np

import synth
from oracle import formats as F
from oracle import svdquant as S


def need_cuda():
    import pytest
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def pack_weight(ops):
    if ops.fmt == "nvfp4":
        return F.pack_nibbles(ops.w_codes), F.sf_to_layout(ops.w_scales, ops.K)
    if ops.fmt == "w8a8":                       # int8 bytes [N][K], fp32 scales [N]
        return (np.ascontiguousarray(ops.w_codes.astype(np.int8)).view(np.uint8),
                np.ascontiguousarray(ops.w_scales.astype(np.float32)).view(np.uint8).reshape(-1))
    return (F.pack_nibbles(F.int4_to_nibble(ops.w_codes)),
            np.ascontiguousarray(ops.w_scales).view(np.uint8).reshape(-1))


def pack_act(fmt, qa, K):
    """(xq bytes [M, K/2], xs bytes flat) of an oracle QuantAct."""
    if fmt == "nvfp4":
        return F.pack_nibbles(qa.codes), F.sf_to_layout(qa.scales, K)
    if fmt == "w8a8":
        return (np.ascontiguousarray(qa.codes.astype(np.int8)).view(np.uint8),
                np.ascontiguousarray(qa.scales.astype(np.float32)).view(np.uint8).reshape(-1))
    return (F.pack_nibbles(F.int4_to_nibble(qa.codes)),
            np.ascontiguousarray(qa.scales).view(np.uint8).reshape(-1))


def to_dev(a, dev, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    return t if dtype is None else t.view(dtype)


def layer_from_ops(P, ops, dev, bias_dtype="bf16"):
    import torch
    codes, scales = pack_weight(ops)
    r = ops.rank
    z = torch.zeros(8, dtype=torch.int16, device=dev)
    bias = None
    if ops.bias is not None:
        bias = torch.from_numpy(ops.bias.astype(np.float32)).to(dev).to(P.TORCH_DTYPE[bias_dtype])
    return P.QuantizedLinear(
        ops.fmt, ops.K, ops.N, r,
        to_dev(codes.reshape(-1), dev), to_dev(scales.reshape(-1), dev),
        to_dev(ops.lam_inv32, dev),
        to_dev(ops.L1s_bits.reshape(-1).view(np.int16), dev) if r else z,
        to_dev(ops.L2s_bits.reshape(-1).view(np.int16), dev) if r else z,
        bias, ops.scale_dtype if ops.fmt == "int4" else "bf16", float(ops.gs_w), float(ops.gs_x))


def make_case(fmt, M, K, N, r, dt="bf16", seed=0, cfg=11, with_bias=True, gs_x=1.0):
    """Seeded synthetic layer (DESIGN.md input recipe) + oracle operands."""
    x = F.round16(synth.gen_x(M, K, synth.rng(cfg, seed, 0)), dt)
    w = synth.gen_w(K, N, synth.rng(cfg, seed, 1))
    lam = S.compute_smoothing(synth.gen_x(max(M, 64), K, synth.rng(cfg, seed, 2)), w, 0.5)
    bias = F.round16(synth.gen_bias(N, synth.rng(cfg, seed, 3)), dt) if with_bias else None
    ops = S.prepare_operands(w, lam, r, fmt, gs_x=gs_x, scale_dtype=dt, bias=bias)
    return x, w, lam, ops


def rel_fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb else 1.0)
