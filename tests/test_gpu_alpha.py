"""svdq_search_alpha against the oracle's search_alpha:
the per-alpha objectives agree (the GPU runs its own fp64-Gram SVD, so residual codes may
differ at rounding boundaries -> 2 % tolerance), lambda(alpha*) matches compute_smoothing,
and the chosen alpha is the oracle's argmin up to that tolerance."""
import numpy as np
import pytest

import synth
from oracle import formats as F
from oracle import svdquant as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", ["nvfp4", "int4", "w8a8"])
def test_search_alpha_matches_oracle(fmt):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2411_05007_b200 as P
    M, K, N, r = 128, 256, 128, 16
    x = F.bf16_round(synth.gen_x(M, K, synth.rng(71, 0, 0)))
    w = synth.gen_w(K, N, synth.rng(71, 0, 1)).astype(np.float32)
    grid = [0.0, 0.25, 0.5, 0.75, 1.0]
    dev = torch.device("cuda")
    a_gpu, lam_gpu, obj_gpu = P.svdq_search_alpha(torch.from_numpy(x).to(dev).to(torch.bfloat16),
                                                  torch.from_numpy(w).to(dev), r, fmt, grid)
    a_ref, lam_ref, obj_ref = S.search_alpha(x, w, r, fmt, grid)
    np.testing.assert_allclose(obj_gpu, obj_ref, rtol=2e-2)
    i_gpu = grid.index(a_gpu)
    assert obj_ref[i_gpu] <= min(obj_ref) * 1.02
    np.testing.assert_allclose(lam_gpu.cpu().numpy(), S.compute_smoothing(x, w, a_gpu), rtol=1e-6)
