"""Single-GPU emulation of the tensor-parallel path: the P column
shards run one after another through the real kernels; concatenated they must equal the
unsharded output bit for bit (every output column depends only on its own operands, and
the per-element K order does not depend on the N tiling)."""
import numpy as np
import pytest

from helpers import layer_from_ops, make_case, need_cuda

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
@pytest.mark.parametrize("P_,N", [(2, 1536), (4, 3072), (8, 3072), (3, 480)])
def test_sharded_equals_unsharded(fmt, P_, N):
    need_cuda()
    import torch
    import paper_2411_05007_b200 as P
    from paper_2411_05007_b200 import tp
    M, K, r = 384, 1024, 32
    x, w, lam, ops = make_case(fmt, M, K, N, r, seed=P_, cfg=23)
    dev = torch.device("cuda")
    full = layer_from_ops(P, ops, dev)
    X = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    y_full = full(X)
    parts = []
    for rank in range(P_):
        shard = tp.shard_layer(full, P_, rank)
        parts.append(shard(X))
    y_cat = torch.cat(parts, dim=1)
    torch.cuda.synchronize()
    assert torch.equal(y_cat.view(torch.int16), y_full.view(torch.int16))
