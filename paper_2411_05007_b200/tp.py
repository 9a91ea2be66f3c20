"""Tensor parallelism for the SVDQuant linear (BASELINE.json north_star:
"tensor-parallel over the 8xB200 box, sharding weights and L2 along output channels, with
an NCCL all-gather over NVLink only where the next layer needs the full activation").  The
paper itself is single-GPU; this is the north star's extension.

Column-parallel over the output channels N: every column of
    Y = alpha (Q(X_hat) Q(R) + xl1 L2s^T) + bias
depends only on its own column of R, its scale factors, its row of L2s and its bias, plus the
full X.  So rank p of P holds
    sharded   : residual codes [N/P, K/2], their scales, l2s [N/P, r], bias [N/P]
    replicated: lambda_inv [K], l1s [r, K], gs_x, and gs_w (computed over the FULL residual
                before sharding, so every shard reproduces the unsharded output bit for bit)

Two ways to feed a layer whose input is needed in full:
  Variant 1 (`forward`): X replicated on every rank, K1 runs redundantly, K2 on the N-shard;
      `all_gather_into_tensor` of the bf16 Y shards where a consumer needs the full output.
  Fused gather (`SymmetricGather`): the same Variant 2, but K1 itself stores
      its codes / scales at their final full-K place in EVERY rank's gather buffer (torch symmetric
      memory: peer buffers mapped over NVLink) and its partial in slot p; one device-side barrier,
      a tiny partial reduction, and K2 reads the buffer -- no collective, no re-layout pass, and
      the transfer overlaps K1's HBM read.
  Variant 2 (`forward_from_shard`, SURVEY 8(e) "quantize, then gather"): rank p holds only
      X[:, p Kp:(p+1) Kp] (its shard of the previous column-parallel layer's output); it runs K1 on
      that K-slice (svdq_quantize_act_lowrank_down_kslice), ONE all-gather moves the packed slices
      (codes + scale factors + an fp32 [M, r] partial X L1s^T: 0.5625 B per element instead of 2),
      svdq_tp_assemble_act rebuilds the full K1 outputs (partials summed in rank order), and K2 runs
      on the N-shard.  K1's work is split P ways instead of replicated.

Only plumbing lives here: slicing device buffers, caching them, and calling torch.distributed.
All arithmetic runs in libsvdq's kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .abi import (QuantizedLinear, svdq_act_buffer_sizes, svdq_gemm_w4a4_lowrank_up, svdq_linear_forward,
                  svdq_quantize_act_lowrank_down_kslice, svdq_quantize_act_lowrank_down_kslice_fused,
                  svdq_tp_assemble_act, svdq_tp_gather_sizes, svdq_tp_reduce_partials, svdq_tp_slice_sizes)


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


def kslice_bounds(K: int, world: int, rank: int):
    """Rank's input-channel slice for Variant 2: Kp = K/P must be a multiple of 64 so no
    quantization group (NVFP4 16, INT4 64) straddles two ranks."""
    if K % world or (K // world) % 64:
        raise ValueError(f"K={K} does not split into {world} slices of a multiple of 64")
    kp = K // world
    return rank * kp, kp


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
    if fmt == "w8a8":
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


def all_gather(out: torch.Tensor, inp: torch.Tensor, group=None):
    """all_gather_into_tensor; NCCL takes device tensors directly, a gloo group (the CPU / one-GPU
    multi-process tests) is fed through host copies."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        tmp = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(tmp, inp.cpu(), group=group)
        out.copy_(tmp)
        return out
    dist.all_gather_into_tensor(out, inp, group=group)
    return out


class ColumnParallelSVDQLinear:
    """Column-parallel layer.  `world` / `rank` default to the process group's; passing them
    explicitly (no process group) gives the single-GPU shard emulation the tests use."""

    def __init__(self, full: QuantizedLinear, group=None, world: int | None = None, rank: int | None = None):
        self.group = group
        live = dist.is_available() and dist.is_initialized()
        self.world = world if world is not None else (dist.get_world_size(group) if live else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if live else 0)
        self.N, self.K, self.fmt, self.r = full.N, full.K, full.fmt, full.rank
        self.local = shard_layer(full, self.world, self.rank)
        self._bufs = {}

    # ------------------------------------------------------------------ Variant 1
    def forward(self, X: torch.Tensor, gather: bool = True, out_dtype=None):
        """Replicated X -> this rank's Y shard (gather=False) or the full Y (bf16 all-gather)."""
        y = svdq_linear_forward(self.local, X, out_dtype=out_dtype)
        if not gather or self.world == 1:
            return y
        blocks = self._buf(("yblocks", y.shape[0], y.dtype), (self.world * y.shape[0], y.shape[1]), y.dtype, y.device)
        all_gather(blocks, y.contiguous(), self.group)
        return assemble_columns(blocks, self.world)

    __call__ = forward

    # ------------------------------------------------------------------ Variant 2
    def quantize_slice(self, x_shard: torch.Tensor, stream=None) -> torch.Tensor:
        """K1 on this rank's input channels: the packed slice this rank contributes."""
        M = x_shard.shape[0]
        k0, kp = kslice_bounds(self.K, self.world, self.rank)
        if x_shard.shape[1] != kp:
            raise ValueError(f"rank {self.rank} expects a [M, {kp}] input shard, got {tuple(x_shard.shape)}")
        nb = svdq_tp_slice_sizes(self.fmt, M, kp, self.r)[3]
        buf = self._buf(("slice", M), (nb,), torch.uint8, x_shard.device)
        return svdq_quantize_act_lowrank_down_kslice(self.local, k0, x_shard, buf, stream=stream)

    def assemble(self, gathered: torch.Tensor, M: int, stream=None):
        """Full K1 outputs (xq, xs, xl1) from the P gathered slices."""
        bq, bs, bl = svdq_act_buffer_sizes(self.fmt, M, self.K, self.r)
        dev = gathered.device
        xq = self._buf(("xq", M), (bq,), torch.uint8, dev)
        xs = self._buf(("xs", M), (bs,), torch.uint8, dev)
        xl1 = self._buf(("xl1", M), (max(bl // 2, 8),), torch.int16, dev)
        return svdq_tp_assemble_act(self.fmt, self.world, M, self.K, self.r, gathered, xq, xs, xl1, stream=stream)

    def gather_slices(self, local_slice: torch.Tensor) -> torch.Tensor:
        nb = int(local_slice.numel())
        out = self._buf(("gathered", nb), (self.world * nb,), torch.uint8, local_slice.device)
        if self.world == 1:
            out.copy_(local_slice)
            return out
        return all_gather(out, local_slice, self.group)

    def forward_from_shard(self, x_shard: torch.Tensor, Y: torch.Tensor | None = None, stream=None):
        """Column-sharded input -> this rank's Y shard [M, N/P] (Variant 2)."""
        M = x_shard.shape[0]
        gathered = self.gather_slices(self.quantize_slice(x_shard, stream=stream))
        xq, xs, xl1 = self.assemble(gathered, M, stream=stream)
        return svdq_gemm_w4a4_lowrank_up(self.local, xq, xs, xl1 if self.r else None, M, Y=Y, stream=stream)

    def _buf(self, key, shape, dtype, device):
        t = self._bufs.get(key)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != device:
            t = torch.empty(shape, dtype=dtype, device=device)
            self._bufs[key] = t
        return t


class SymmetricGather:
    """Fused packed all-gather: every rank owns a gather buffer in symmetric memory
    (torch.distributed._symmetric_memory, peers mapped over NVLink) with one region per layer; a
    region holds the layer's full K1 outputs (xq, xs) plus P fp32 partial slots
    (svdq_tp_gather_sizes).  fill(i, ...) runs K1 on this rank's K-slice and stores it, inside the
    kernel, into region i of EVERY rank's buffer; sync() is the cross-rank device barrier; after it,
    outputs(i) reduces the partials (rank order) and returns (xq, xs, xl1) for K2."""

    def __init__(self, specs, device, group=None, world: int | None = None, rank: int | None = None):
        """specs: [(fmt, M, K, rank)] per layer region."""
        self.group = group if group is not None else (dist.group.WORLD if world is None else None)
        self.world = world if world is not None else dist.get_world_size(self.group)
        self.rank = rank if rank is not None else dist.get_rank(self.group)
        self.specs, self.regions, total = list(specs), [], 0
        for fmt, M, K, r in self.specs:
            oq, os_, op, nb = svdq_tp_gather_sizes(fmt, M, K, r, self.world)
            self.regions.append((total, oq, os_, op, nb))
            total += nb
        self.buf = self._alloc(total, device)
        self._xl1 = [torch.empty(max(M * r, 8), dtype=torch.int16, device=device) for _, M, _, r in self.specs]

    def _alloc(self, total, device):
        import torch.distributed._symmetric_memory as symm_mem
        buf = symm_mem.empty(total, dtype=torch.uint8, device=device)
        self.handle = symm_mem.rendezvous(buf, self.group)
        self.ptrs = [int(p) for p in self.handle.buffer_ptrs]
        return buf

    def fill(self, i: int, layer: QuantizedLinear, k0: int, x_shard: torch.Tensor, stream=None):
        base = self.regions[i][0]
        svdq_quantize_act_lowrank_down_kslice_fused(layer, k0, x_shard, self.world, self.rank,
                                                    [p + base for p in self.ptrs], stream=stream)

    def sync(self):
        self.handle.barrier(channel=0)

    def outputs(self, i: int, stream=None):
        fmt, M, K, r = self.specs[i]
        base, oq, os_, op, nb = self.regions[i]
        bq, bs, _ = svdq_act_buffer_sizes(fmt, M, K, r)
        xq = self.buf[base + oq:base + oq + bq]
        xs = self.buf[base + os_:base + os_ + bs]
        if r:
            parts = self.buf[base + op:base + op + self.world * M * r * 4]
            svdq_tp_reduce_partials(self.world, M, r, parts, self._xl1[i], stream=stream)
        return xq, xs, self._xl1[i]


class IpcGather(SymmetricGather):
    """The same buffers from CUDA IPC handles, for ranks sharing one device (the one-GPU
    multi-process tests: symmetric memory refuses overlapping devices).  sync() is a stream
    synchronize + host barrier (correct, not fast)."""

    def _alloc(self, total, device):
        from torch.multiprocessing.reductions import reduce_tensor
        buf = torch.zeros(total, dtype=torch.uint8, device=device)
        handles = [None] * self.world
        dist.all_gather_object(handles, reduce_tensor(buf), group=self.group)
        self._peers = [buf if j == self.rank else fn(*args) for j, (fn, args) in enumerate(handles)]
        self.ptrs = [int(t.data_ptr()) for t in self._peers]
        return buf

    def sync(self):
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)


class EmulatedGather(SymmetricGather):
    """One rank's view of a P-way fused gather on a single GPU (timing emulation): K1 stores only into
    this rank's own buffer; sync() is a no-op."""

    def __init__(self, specs, device, world: int, rank: int = 0):
        super().__init__(specs, device, world=world, rank=rank)

    def _alloc(self, total, device):
        buf = torch.zeros(total, dtype=torch.uint8, device=device)
        self.ptrs = [int(buf.data_ptr())]
        return buf

    def sync(self):
        pass
