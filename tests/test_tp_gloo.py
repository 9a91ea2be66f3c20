"""Multi-process (world_size 2, gloo on CPU) tests of the tensor-parallel host logic:
operand sharding along N (including the NVFP4 128x4 scale-factor layout), the
all-gather, and the column reassembly.  The per-shard GEMM here is the ORACLE (test
infrastructure) standing in for K2, so the test pins the partitioning logic: the
reassembled sharded result must equal the unsharded result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import make_case, pack_weight
from oracle import formats as F
from oracle import svdquant as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _unpack_shard(ops, shard, n):
    """Device-layout shard buffers -> oracle Operands of the shard."""
    K = ops.K
    if ops.fmt == "w8a8":
        codes = shard.w_codes.numpy().view(np.int8).reshape(n, K).astype(np.int64)
        scales = shard.w_scales.numpy().view(np.float32).reshape(n)
        l2s = shard.l2s.numpy().view(np.uint16).reshape(n, ops.rank)
        bias = shard.bias.numpy().astype(np.float32) if shard.bias is not None else None
        return S.Operands(ops.fmt, K, n, ops.rank, codes, scales, ops.scale_dtype, ops.gs_w, ops.gs_x,
                          ops.lam_inv32, ops.L1s_bits, l2s, bias)
    codes = F.unpack_nibbles(shard.w_codes.numpy().reshape(n, K // 2))
    if ops.fmt == "nvfp4":
        scales = F.sf_from_layout(shard.w_scales.numpy(), n, K)
    else:
        codes = F.nibble_to_int4(codes)
        scales = shard.w_scales.numpy().view(np.uint16).reshape(n, K // 64)
    l2s = shard.l2s.numpy().view(np.uint16).reshape(n, ops.rank)
    bias = shard.bias.numpy().astype(np.float32) if shard.bias is not None else None
    return S.Operands(ops.fmt, K, n, ops.rank, codes, scales, ops.scale_dtype, ops.gs_w, ops.gs_x,
                      ops.lam_inv32, ops.L1s_bits, l2s, bias)


def _worker(rank, world, port, fmt, N, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2411_05007_b200 as P
        from paper_2411_05007_b200 import tp
        M, K, r = 48, 256, 16
        x, w, lam, ops = make_case(fmt, M, K, N, r, seed=5, cfg=21)
        codes, scales = pack_weight(ops)
        full = P.QuantizedLinear(
            fmt, K, N, r, torch.from_numpy(codes.reshape(-1).copy()), torch.from_numpy(scales.reshape(-1).copy()),
            torch.from_numpy(ops.lam_inv32.copy()), torch.from_numpy(ops.L1s_bits.view(np.int16).reshape(-1).copy()),
            torch.from_numpy(ops.L2s_bits.view(np.int16).reshape(-1).copy()),
            torch.from_numpy(ops.bias.astype(np.float32)), ops.scale_dtype if fmt == "int4" else "bf16",
            float(ops.gs_w), float(ops.gs_x))
        shard = tp.shard_layer(full, world, rank)
        n0, n = tp.shard_bounds(N, world, rank)
        sops = _unpack_shard(ops, shard, n)
        qa = S.quantize_activation(x, ops)                 # K1 output is identical on every rank
        y_local = torch.from_numpy(S.gemm_reference(qa, sops))   # oracle stands in for K2
        blocks = torch.empty(world * M, n, dtype=torch.float64)
        dist.all_gather_into_tensor(blocks, y_local.contiguous())
        y = tp.assemble_columns(blocks, world).numpy()
        if rank == 0:
            q.put(("ok", y, S.gemm_reference(qa, ops)))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put(("err", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fmt,N", [("nvfp4", 512), ("nvfp4", 320), ("int4", 320), ("w8a8", 320)])
def test_column_parallel_gloo_bitwise(fmt, N):
    """N = 512: shards are whole 128-row scale-factor atoms; N = 320: shard width 160
    forces the byte-gather re-layout of the 128x4 scale factors."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fmt, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, y, ref = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", y
    np.testing.assert_array_equal(y, ref)


def test_shard_bounds_validation():
    from paper_2411_05007_b200 import tp
    assert tp.shard_bounds(3072, 8, 3) == (1152, 384)
    with pytest.raises(ValueError):
        tp.shard_bounds(100, 3, 0)
    with pytest.raises(ValueError):
        tp.shard_bounds(3072, 256, 0)       # 12-wide shards


def test_assemble_columns():
    from paper_2411_05007_b200 import tp
    a = torch.arange(2 * 3 * 4).reshape(2 * 3, 4)      # world 2, M 3, n 4
    out = tp.assemble_columns(a, 2)
    assert out.shape == (3, 8)
    assert out[1].tolist() == [4, 5, 6, 7, 16, 17, 18, 19]


# ---------------------------------------------------------------------------------------------
# Variant 2 slice contract (world_size 2, gloo, CPU): each rank packs ITS K-slice's K1 outputs --
# computed here by the ORACLE standing in for svdq_quantize_act_lowrank_down_kslice -- at the
# offsets svdq_tp_slice_sizes reports; one all_gather_into_tensor; rank 0 re-assembles with the
# layout rules svdq_tp_assemble_act implements (codes concatenated along K, NVFP4 scale-factor
# 512-B chunks interleaved per row tile, INT4 scales concatenated per row, fp32 partials summed in
# rank order) and must reproduce the oracle's K1 of the FULL input: codes / scales bit for bit
# (groups never straddle slices), xl1 within the K1 tolerance.
# ---------------------------------------------------------------------------------------------
def _v2_worker(rank, world, port, fmt, q):
    import dataclasses
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2411_05007_b200 as P
        from paper_2411_05007_b200 import tp
        M, K, N, r = 200, 512, 128, 32
        x, w, lam, ops = make_case(fmt, M, K, N, r, seed=7, cfg=22)
        k0, kp = tp.kslice_bounds(K, world, rank)
        sl = dataclasses.replace(ops, K=kp, lam_inv32=ops.lam_inv32[k0:k0 + kp].copy(),
                                 L1s_bits=np.ascontiguousarray(ops.L1s_bits[:, k0:k0 + kp]))
        qa = S.quantize_activation(x[:, k0:k0 + kp], sl)
        oq, os_, op, nb = P.svdq_tp_slice_sizes(fmt, M, kp, r)
        buf = np.zeros(nb, np.uint8)
        if fmt == "nvfp4":
            codes, scales = F.pack_nibbles(qa.codes), F.sf_to_layout(qa.scales, kp)
        else:
            codes = F.pack_nibbles(F.int4_to_nibble(qa.codes))
            scales = np.ascontiguousarray(qa.scales).view(np.uint8)
        buf[oq:oq + codes.size] = codes.reshape(-1)
        buf[os_:os_ + scales.size] = scales.reshape(-1)
        part = qa.xl1_exact.astype(np.float32)
        buf[op:op + part.nbytes] = part.view(np.uint8).reshape(-1)
        gathered = torch.empty(world * nb, dtype=torch.uint8)
        dist.all_gather_into_tensor(gathered, torch.from_numpy(buf))
        if rank == 0:
            g = gathered.numpy().reshape(world, nb)
            cs = [F.unpack_nibbles(g[p, oq:oq + M * kp // 2].reshape(M, kp // 2)) for p in range(world)]
            if fmt == "nvfp4":
                ss = [F.sf_from_layout(g[p, os_:os_ + F.sf_swizzled_size(M, kp)], M, kp) for p in range(world)]
            else:
                cs = [F.nibble_to_int4(c) for c in cs]
                ss = [g[p, os_:os_ + M * (kp // 64) * 2].view(np.uint16).reshape(M, kp // 64) for p in range(world)]
            acc = np.zeros((M, r), np.float32)
            for p in range(world):                               # rank order
                acc = acc + g[p, op:op + M * r * 4].view(np.float32).reshape(M, r)
            q.put(("ok", (np.concatenate(cs, 1), np.concatenate(ss, 1), F.bf16_round(acc)),
                   S.quantize_activation(x, ops)))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put(("err", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_variant2_slice_contract_gloo(fmt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_v2_worker, args=(r, world, port, fmt, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, got, ref = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", got
    codes, scales, xl1 = got
    np.testing.assert_array_equal(codes, ref.codes)
    np.testing.assert_array_equal(scales, ref.scales)
    d = np.linalg.norm(xl1.astype(np.float64) - F.bf16_from_bits(ref.xl1_bits))
    assert d / np.linalg.norm(F.bf16_from_bits(ref.xl1_bits)) <= 1e-3
