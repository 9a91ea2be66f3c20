"""Tensor parallelism through a REAL process group on one GPU: two processes (gloo, both on
cuda:0 -- NCCL refuses two ranks on one device) run Variant 1 (replicated X, bf16 Y gather) and
Variant 2 (K-sliced K1, packed all-gather, assemble, K2 on the shard).  The gathered results must
equal the single-process shard emulation bit for bit: the collective only moves bytes."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fmt, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
        from helpers import layer_from_ops, make_case
        import paper_2411_05007_b200 as P
        from paper_2411_05007_b200 import tp
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        M, K, N, r = 256, 1536, 768, 32
        x, w, lam, ops = make_case(fmt, M, K, N, r, seed=3, cfg=25)
        full = layer_from_ops(P, ops, dev)
        X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
        layer = tp.ColumnParallelSVDQLinear(full)
        assert layer.world == world and layer.rank == rank
        y1 = layer.forward(X, gather=True)                        # Variant 1
        kp = K // world
        y2 = layer.forward_from_shard(X[:, rank * kp:(rank + 1) * kp].contiguous())   # Variant 2
        blocks = torch.empty(world * M, y2.shape[1], dtype=y2.dtype, device=dev)
        tp.all_gather(blocks, y2.contiguous())
        y2full = tp.assemble_columns(blocks, world)
        # fused gather: K1 writes its slice into both ranks' buffers (CUDA IPC here)
        fused = None
        try:
            sg = tp.IpcGather([(fmt, M, K, r)], dev)               # both ranks share cuda:0 here
            sg.fill(0, layer.local, rank * kp, X[:, rank * kp:(rank + 1) * kp].contiguous())
            sg.sync()
            xq, xs, xl1 = sg.outputs(0)
            y3 = P.svdq_gemm_w4a4_lowrank_up(layer.local, xq, xs, xl1, M)
            tp.all_gather(blocks, y3.contiguous())
            fused = tp.assemble_columns(blocks, world).view(torch.int16).cpu().numpy()
        except Exception as e:  # CUDA IPC unavailable
            fused = f"unavailable: {type(e).__name__}: {str(e)[:200]}"
        torch.cuda.synchronize()
        if rank == 0:
            q.put(("ok", y1.view(torch.int16).cpu().numpy(), (y2full.view(torch.int16).cpu().numpy(), fused)))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put(("err", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fmt", ["nvfp4", "int4"])
def test_tp_two_processes_one_gpu(fmt):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2411_05007_b200 as P
    from paper_2411_05007_b200 import tp
    from helpers import layer_from_ops, make_case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, fmt, q)) for rk in range(world)]
    for p in procs:
        p.start()
    status, y1, y23 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", y1
    y2, y3 = y23
    # single-process references: the unsharded forward (Variant 1 is bitwise equal to it) and the
    # emulated Variant 2
    dev = torch.device("cuda")
    M, K, N, r = 256, 1536, 768, 32
    x, w, lam, ops = make_case(fmt, M, K, N, r, seed=3, cfg=25)
    full = layer_from_ops(P, ops, dev)
    X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    ref1 = full(X).view(torch.int16).cpu().numpy()
    np.testing.assert_array_equal(y1, ref1)
    ranks = [tp.ColumnParallelSVDQLinear(full, world=world, rank=p) for p in range(world)]
    kp = K // world
    slices = [ranks[p].quantize_slice(X[:, p * kp:(p + 1) * kp].contiguous()).clone() for p in range(world)]
    g = torch.cat(slices)
    ys = []
    for p in range(world):
        xq, xs, xl1 = ranks[p].assemble(g, M)
        ys.append(P.svdq_gemm_w4a4_lowrank_up(ranks[p].local, xq, xs, xl1, M))
    ref2 = torch.cat(ys, dim=1).view(torch.int16).cpu().numpy()
    np.testing.assert_array_equal(y2, ref2)
    if isinstance(y3, str):
        pytest.skip(f"fused symmetric-memory gather: {y3}")
    np.testing.assert_array_equal(y3, ref2)           # fused gather == collective gather, bitwise


@pytest.mark.parametrize("gather", ["nccl", "fused"])
def test_bench_tp_mode_two_ranks_gloo(gather):
    """bench.py's tensor-parallel arm end to end under torchrun (2 ranks on the one GPU, gloo):
    one JSON line with the strong-scaling TP fields and a positive value."""
    import json
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--backend", "gloo", "--steps", "2", "--warmup", "3", "--no-extras", "--tp-gather", gather]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["scaling"] == "strong" and out["value"] > 0
    assert out["tp"]["backend"] == "gloo" and out["tp"]["gathered_bytes_per_rank_per_step"] > 0
    assert out["config"]["parallelism"].startswith("tp2")
