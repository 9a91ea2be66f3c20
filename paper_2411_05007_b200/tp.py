"""Tensor parallelism for the SVDQuant linear (BASELINE.json north_star:
"tensor-parallel over the 8xB200 box, sharding weights and L2 along output channels, with
an NCCL all-gather over NVLink only where the next layer needs the full activation").

Column-parallel over the output channels N: every column of
    Y = alpha (Q(X_hat) Q(R) + xl1 L2s^T) + bias
depends only on its own column of R, its scale factors, its row of L2s and its bias, plus the
full X.  So rank p of P holds
    sharded   : residual codes [N/P, K/2], their scales, l2s [N/P, r], bias [N/P]
    replicated: lambda_inv [K], l1s [r, K], gs_x, and gs_w (computed over the FULL residual
                before sharding, so every shard reproduces the unsharded output bit for bit)
K1 runs on the replicated X (its outputs are identical on every rank), K2 on the shard, and
`all_gather_into_tensor` (NCCL over NVLink / NVSwitch; gloo in the CPU tests) assembles Y
where the consumer needs the full feature dimension.

Only plumbing lives here: slicing device buffers and calling torch.distributed.  All
arithmetic runs in libsvdq's kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .abi import QuantizedLinear, svdq_linear_forward


def _sf_atom_bytes(K: int) -> int:
    """Bytes of one 128-row atom of the NVFP4 128x4 scale-factor layout."""
    return 128 * (K // 16)


def shard_bounds(N: int, world: int, rank: int):
    """Equal contiguous column shards; N/P must be a multiple of 16 (the K2 N granularity)."""
    if N % world:
        raise ValueError(f"N={N} not divisible by world size {world}")
    n = N // world
    if n % 16:
        raise ValueError(f"shard width {n} not a multiple of 16")
    return rank * n, n


def shard_scales(scales: torch.Tensor, fmt: str, K: int, N: int, n0: int, n: int, scale_dtype: str):
    """Slice the weight scales of output channels [n0, n0+n).

    INT4: [N][K/64] 16-bit rows -> contiguous row slice.
    W8A8: [N] fp32 per-channel scales -> contiguous slice.
    NVFP4: 128x4 layout; when n0 and n are multiples of 128 the shard is a contiguous run of
    atoms, otherwise the shard's rows are re-laid out (byte gather) into a fresh 128x4 buffer
    whose padding rows are 0x00.
    """
    if fmt == "int4":
        g = K // 64
        return scales.view(torch.uint8)[n0 * g * 2:(n0 + n) * g * 2].clone()
    if fmt == "w8a8":                                   # one fp32 scale per output channel
        return scales.view(torch.uint8)[n0 * 4:(n0 + n) * 4].clone()
    if fmt != "nvfp4":
        raise ValueError(f"unsupported format {fmt!r}")
    atom = _sf_atom_bytes(K)
    if n0 % 128 == 0 and n % 128 == 0:
        return scales[(n0 // 128) * atom:((n0 + n) // 128) * atom].clone()
    # general case: gather bytes with the layout's index formula
    dev = scales.device
    nkt = K // 64
    rows = torch.arange(n, device=dev)
    cols = torch.arange(K // 16, device=dev)
    r, c = torch.meshgrid(rows, cols, indexing="ij")

    def off(row, col):
        return ((row // 128) * (nkt * 512) + (col // 4) * 512 + (row % 32) * 16
                + ((row % 128) // 32) * 4 + (col % 4))

    out = torch.zeros(((n + 127) // 128) * atom, dtype=torch.uint8, device=dev)
    out[off(r, c).reshape(-1)] = scales[off(r + n0, c).reshape(-1)]
    return out


def shard_layer(full: QuantizedLinear, world: int, rank: int) -> QuantizedLinear:
    """The rank-th column shard of a quantized layer (device buffers are sliced copies)."""
    n0, n = shard_bounds(full.N, world, rank)
    K, r = full.K, full.rank
    if full.fmt not in ("nvfp4", "int4", "w8a8"):
        raise ValueError(f"unsupported format {full.fmt!r}")
    row = K if full.fmt == "w8a8" else K // 2            # code bytes per output channel
    codes = full.w_codes.view(torch.uint8)[n0 * row:(n0 + n) * row].clone()
    scales = shard_scales(full.w_scales, full.fmt, K, full.N, n0, n, full.scale_dtype)
    if r:
        l2s = full.l2s.view(torch.int16)[n0 * r:(n0 + n) * r].clone()
    else:
        l2s = full.l2s
    bias = full.bias[n0:n0 + n].clone() if full.bias is not None else None
    return QuantizedLinear(full.fmt, K, n, r, codes, scales, full.lambda_inv, full.l1s, l2s, bias,
                           full.scale_dtype, full.gs_w, full.gs_x)


def assemble_columns(blocks: torch.Tensor, world: int) -> torch.Tensor:
    """[P*M, N/P] (all_gather_into_tensor output, rank-major) -> [M, N]."""
    pm, n = blocks.shape
    m = pm // world
    return blocks.view(world, m, n).permute(1, 0, 2).reshape(m, world * n)


class ColumnParallelSVDQLinear:
    """Column-parallel layer: K1 + K2 on the local shard, optional all-gather of Y."""

    def __init__(self, full: QuantizedLinear, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.N = full.N
        self.local = shard_layer(full, self.world, self.rank)

    def forward(self, X: torch.Tensor, gather: bool = True, out_dtype=None):
        y = svdq_linear_forward(self.local, X, out_dtype=out_dtype)
        if not gather or self.world == 1:
            return y
        blocks = torch.empty((self.world * y.shape[0], y.shape[1]), dtype=y.dtype, device=y.device)
        dist.all_gather_into_tensor(blocks, y.contiguous(), group=self.group)
        return assemble_columns(blocks, self.world)

    __call__ = forward
