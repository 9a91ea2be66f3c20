"""Oracle pins for the layer-boundary fusion: GELU (tanh form) against torch's
library GELU and its limits; the fused hand-off is K1 of the stored, activated output."""
import numpy as np
import torch

import synth
from oracle import formats as F
from oracle import svdquant as S


def test_gelu_tanh_matches_library():
    v = np.linspace(-8, 8, 20001)
    ref = torch.nn.functional.gelu(torch.from_numpy(v), approximate="tanh").numpy()
    np.testing.assert_allclose(S.gelu_tanh(v), ref, rtol=1e-12, atol=1e-15)
    assert S.gelu_tanh(np.array([0.0]))[0] == 0.0
    np.testing.assert_allclose(S.gelu_tanh(np.array([30.0, -30.0])), [30.0, 0.0], atol=1e-12)


def test_gelu_tanh_close_to_erf_gelu():
    v = np.linspace(-6, 6, 2001)
    exact = torch.nn.functional.gelu(torch.from_numpy(v)).numpy()
    assert np.max(np.abs(S.gelu_tanh(v) - exact)) < 1e-3


def test_fused_next_is_k1_of_the_stored_output():
    rng = synth.rng(78, 0, 0)
    M, K, N = 64, 128, 192
    y64 = rng.standard_normal((M, N)) * 2
    w = synth.gen_w(N, 64, synth.rng(78, 0, 1))
    lam = S.compute_smoothing(F.bf16_round(y64), w, 0.5)
    ops_next = S.prepare_operands(w, lam, 16, "nvfp4")
    qa = S.fused_next(y64, ops_next, "none")
    ref = S.quantize_activation(F.bf16_round(y64), ops_next)
    np.testing.assert_array_equal(qa.codes, ref.codes)
    np.testing.assert_array_equal(qa.scales, ref.scales)
    qg = S.fused_next(y64, ops_next, "gelu_tanh")
    refg = S.quantize_activation(F.bf16_round(S.gelu_tanh(F.bf16_round(y64))), ops_next)
    np.testing.assert_array_equal(qg.codes, refg.codes)
    np.testing.assert_array_equal(qg.xl1_bits, refg.xl1_bits)
