"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws random
tensors with the shapes and value structure of the paper's workloads
 and lists the layer shapes of the
configs in BASELINE.json.  Both sides receive the same arrays from here.

Recipe (reading of P:96-98 Fig. 3 "significant outliers", Fig. 4
"steep drop" of singular values):
  X [M, K]: N(0,1), each token row scaled by LogNormal(0, 0.5), an outlier
            channel set of max(4, K/256) channels (fixed per K) scaled x50; cast to the
            model dtype by the caller.
  W [K, N]: G / sqrt(K), G ~ N(0,1), plus a rank-8 spike U8 diag(s) V8^T with
            s_i = 3 sigma_max(G/sqrt(K)) 0.7^(i-1) (sigma_max estimated as
            1 + sqrt(N/K) for the Gaussian bulk -- a seeding constant, not
            method arithmetic).
  bias ~ N(0, 0.1); LoRA A ~ N(0, 1/K) [K, r_l], B ~ 0.5 N(0, 1/r_l) [r_l, N].
Seeds: numpy PCG64(1000*cfg + 10*layer + t), t = 0 X, 1 W, 2 X_cal, 3 bias,
4 A, 5 B.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def rng(cfg: int, layer: int, t: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(1000 * cfg + 10 * layer + t))


def outlier_channels(K: int) -> np.ndarray:
    """The outlier channel set of a K-wide hidden state: max(4, K/256)
    channels, fixed per K so calibration and inference draws (and every layer
    reading the same hidden state) share it."""
    g = np.random.Generator(np.random.PCG64(77_000 + K))
    return np.sort(g.choice(K, size=min(max(4, K // 256), K), replace=False))


def gen_x(M: int, K: int, seed_rng: np.random.Generator, outlier_scale=50.0) -> np.ndarray:
    g = seed_rng
    x = g.standard_normal((M, K))
    x *= g.lognormal(0.0, 0.5, size=(M, 1))
    x[:, outlier_channels(K)] *= outlier_scale
    return x.astype(np.float32)


def gen_w(K: int, N: int, seed_rng: np.random.Generator, spike_rank=8) -> np.ndarray:
    g = seed_rng
    w = g.standard_normal((K, N)) / np.sqrt(K)
    k = min(spike_rank, K, N)
    u, _ = np.linalg.qr(g.standard_normal((K, k)))
    v, _ = np.linalg.qr(g.standard_normal((N, k)))
    smax = 1.0 + np.sqrt(N / K)
    s = 3.0 * smax * 0.7 ** np.arange(k)
    w += (u * s[None, :]) @ v.T
    return w.astype(np.float32)


def gen_bias(N: int, seed_rng: np.random.Generator) -> np.ndarray:
    return (0.1 * seed_rng.standard_normal(N)).astype(np.float32)


def gen_lora(K: int, N: int, r_l: int, rng_a, rng_b):
    a = rng_a.standard_normal((K, r_l)) / np.sqrt(K)
    b = 0.5 * rng_b.standard_normal((r_l, N)) / np.sqrt(r_l)
    return a.astype(np.float32), b.astype(np.float32)


@dataclass(frozen=True)
class Layer:
    name: str
    M: int
    K: int
    N: int
    r: int
    dtype: str = "bf16"   # activation / output dtype
    lora: int = 0


# BASELINE.json configs
C1 = [Layer("c1_linear", 256, 512, 512, 16)]
C2 = [  # PixArt-Sigma 1024px, fp16
    Layer("pixart_qkv", 4096, 1152, 3456, 32, "fp16"),
    Layer("pixart_attn_out", 4096, 1152, 1152, 32, "fp16"),
    Layer("pixart_cross_q", 4096, 1152, 1152, 32, "fp16"),
    Layer("pixart_cross_out", 4096, 1152, 1152, 32, "fp16"),
    Layer("pixart_fc1", 4096, 1152, 4608, 32, "fp16"),
    Layer("pixart_fc2", 4096, 4608, 1152, 32, "fp16"),
]
C3 = [  # SDXL 1024px (CFG batch 2), fp16, r=32 + LoRA 16
    Layer("sdxl640_qkv", 8192, 640, 1920, 32, "fp16", 16),
    Layer("sdxl640_out", 8192, 640, 640, 32, "fp16", 16),
    Layer("sdxl640_geglu", 8192, 640, 5120, 32, "fp16", 16),
    Layer("sdxl640_ffout", 8192, 2560, 640, 32, "fp16", 16),
    Layer("sdxl1280_qkv", 2048, 1280, 3840, 32, "fp16", 16),
    Layer("sdxl1280_out", 2048, 1280, 1280, 32, "fp16", 16),
    Layer("sdxl1280_geglu", 2048, 1280, 10240, 32, "fp16", 16),
    Layer("sdxl1280_ffout", 2048, 5120, 1280, 32, "fp16", 16),
]
C4 = [  # FLUX.1-dev block linears, bf16
    Layer("flux_single_linear1", 4608, 3072, 21504, 32),
    Layer("flux_single_linear2", 4608, 15360, 3072, 32),
    Layer("flux_qkv", 4608, 3072, 9216, 32),
    Layer("flux_attn_out", 4608, 3072, 3072, 32),
    Layer("flux_mlp_up", 4608, 3072, 12288, 32),
    Layer("flux_mlp_down", 4608, 12288, 3072, 32),
]


def flux_double_block(batch: int = 1):
    """Per-stream W4A4 linears of a FLUX.1 double (joint) block: img 4096 tok,
    txt 512 tok; qkv, proj, mlp up, mlp down."""
    out = []
    for stream, tok in (("img", 4096), ("txt", 512)):
        M = tok * batch
        out += [Layer(f"double_{stream}_qkv", M, 3072, 9216, 32),
                Layer(f"double_{stream}_proj", M, 3072, 3072, 32),
                Layer(f"double_{stream}_mlp_up", M, 3072, 12288, 32),
                Layer(f"double_{stream}_mlp_down", M, 12288, 3072, 32)]
    return out


def flux_single_block(batch: int = 1):
    M = 4608 * batch
    return [Layer("single_linear1", M, 3072, 21504, 32),
            Layer("single_linear2", M, 15360, 3072, 32)]
