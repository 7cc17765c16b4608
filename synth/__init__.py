"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the LRQMM method (no quantization, no
residuals, no RSVD): only random draws with the shapes and value
distributions of the paper's workloads. Both `oracle/` (through the tests)
and the CUDA path (through the tests and `bench.py`) consume it; neither
side imports the other.

Recipes ("Input recipe"):

* Distributions of Tables 2/3 (labels read per
  SURVEY.md §8(c) #18): Normal(0,1), Uniform(0,1), Uniform(-1,1),
  Exponent(4) (rate 4), ChiSquare(1) (1 dof), Poisson(10) (mean 10).
* Matrices are drawn with NumPy PCG64 `default_rng(seed)` and rounded to
  float32 (the paper's "original precision" FP32 inputs).
* Seeds: A uses 2s, B^T uses 2s+1, Omega_A 1000+2s,
  Omega_B 1001+2s.  B is generated directly as B^T (N x K), K-major.
* The RSVD sketch Omega is i.i.d. N(0,1) (PAPER.md:128
  leaves the sampling technique open), K x k_max float32, nested across a
  rank sweep (the first k columns are used).
* Large inputs (bench sizes) are drawn on the GPU with a seeded
  torch.Generator (`gen_matrix_torch`): same distributions, a different
  (Philox) stream.  Parity at those sizes copies the inputs to the host.
"""
from __future__ import annotations

import numpy as np

DISTS = ("normal", "u01", "u11", "exp4", "chi1", "pois10")


def _draw(rng: np.random.Generator, dist: str, shape):
    if dist == "normal":
        return rng.standard_normal(shape)
    if dist == "u01":
        return rng.random(shape)
    if dist == "u11":
        return rng.uniform(-1.0, 1.0, shape)
    if dist == "exp4":
        return rng.exponential(1.0 / 4.0, shape)
    if dist == "chi1":
        return rng.chisquare(1, shape)
    if dist == "pois10":
        return rng.poisson(10.0, shape).astype(np.float64)
    if dist == "relu_normal":
        return np.maximum(rng.standard_normal(shape), 0.0)
    raise ValueError(f"unknown distribution {dist!r}")


def gen_matrix(dist: str, rows: int, cols: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """rows x cols float32, C-contiguous, i.i.d. draws of `dist` (times `scale`)."""
    rng = np.random.default_rng(seed)
    x = _draw(rng, dist, (rows, cols))
    if scale != 1.0:
        x = x * scale
    return np.ascontiguousarray(x.astype(np.float32))


def gen_omega(K: int, k: int, seed: int) -> np.ndarray:
    """K x k float32 standard-normal sketch, shared bit-for-bit by both sides."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.standard_normal((K, k)).astype(np.float32))


def problem(M: int, N: int, K: int, kmax: int, s: int = 0, dist: str = "normal",
            dist_b: str | None = None, scale_b: float = 1.0):
    """(A [MxK], Bt [NxK], Omega_A [Kxkmax], Omega_B [Kxkmax]) with the §8(d) seeds."""
    A = gen_matrix(dist, M, K, 2 * s)
    Bt = gen_matrix(dist_b or dist, N, K, 2 * s + 1, scale=scale_b)
    OmA = gen_omega(K, kmax, 1000 + 2 * s)
    OmB = gen_omega(K, kmax, 1001 + 2 * s)
    return A, Bt, OmA, OmB


def gen_matrix_torch(dist: str, rows: int, cols: int, seed: int, device="cuda", scale: float = 1.0):
    """Large-size variant drawn directly on `device` (seeded torch.Generator)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    shape = (rows, cols)
    if dist == "normal":
        x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    elif dist == "u01":
        x = torch.rand(shape, generator=g, device=device, dtype=torch.float32)
    elif dist == "u11":
        x = torch.rand(shape, generator=g, device=device, dtype=torch.float32) * 2.0 - 1.0
    elif dist == "relu_normal":
        x = torch.randn(shape, generator=g, device=device, dtype=torch.float32).clamp_min_(0.0)
    elif dist == "exp4":
        x = torch.empty(shape, device=device, dtype=torch.float32).exponential_(4.0, generator=g)
    else:
        raise ValueError(f"torch generator has no {dist!r}")
    if scale != 1.0:
        x.mul_(scale)
    return x


# ---------------------------------------------------------------------------
# ResNet-50 conv layers as im2col GEMMs (config C4; "img2col").
# Shapes only: torchvision resnet50 topology at 224x224 input.
# Returns (name, M = batch*Ho*Wo, K = Cin*kh*kw, N = Cout, kh*kw) per conv.
# ---------------------------------------------------------------------------
def resnet50_conv_geoms(batch: int = 256):
    """The 53 convolutions of resnet50_convs with their NHWC geometry (torchvision v1.5: stride on the
    3x3): (name, dict(batch, H, W, C, kh, kw, stride, pad, Cout)); im2col rows = batch Ho Wo,
    K = kh kw C, N = Cout (same order and sizes as resnet50_convs)."""
    g = [("conv1", dict(batch=batch, H=224, W=224, C=3, kh=7, kw=7, stride=2, pad=3, Cout=64))]
    spec = [(64, 3, 256, 56), (128, 4, 512, 28), (256, 6, 1024, 14), (512, 3, 2048, 7)]
    cin, hw_in = 64, 56
    for li, (width, blocks, cout, hw) in enumerate(spec, start=1):
        for b in range(blocks):
            hin = hw_in if b == 0 else hw
            s2 = hin // hw  # 2 on the first block of layers 2-4, else 1
            g.append((f"layer{li}.{b}.conv1", dict(batch=batch, H=hin, W=hin, C=cin, kh=1, kw=1, stride=1, pad=0, Cout=width)))
            g.append((f"layer{li}.{b}.conv2", dict(batch=batch, H=hin, W=hin, C=width, kh=3, kw=3, stride=s2, pad=1, Cout=width)))
            g.append((f"layer{li}.{b}.conv3", dict(batch=batch, H=hw, W=hw, C=width, kh=1, kw=1, stride=1, pad=0, Cout=cout)))
            if b == 0:
                g.append((f"layer{li}.{b}.downsample", dict(batch=batch, H=hin, W=hin, C=cin, kh=1, kw=1, stride=s2, pad=0, Cout=cout)))
            cin = cout
        hw_in = hw
    return g


def resnet50_convs(batch: int = 256):
    layers = []
    layers.append(("conv1", batch * 112 * 112, 3 * 7 * 7, 64, 49))
    spec = [(64, 3, 256, 56), (128, 4, 512, 28), (256, 6, 1024, 14), (512, 3, 2048, 7)]
    cin = 64
    hw_in = 56
    for li, (width, blocks, cout, hw) in enumerate(spec, start=1):
        for b in range(blocks):
            stride_hw_in = hw_in if b == 0 else hw
            # 1x1 reduce (stride 1 at input resolution in torchvision v1.5: stride on 3x3)
            layers.append((f"layer{li}.{b}.conv1", batch * stride_hw_in * stride_hw_in, cin, width, 1))
            layers.append((f"layer{li}.{b}.conv2", batch * hw * hw, width * 9, width, 9))
            layers.append((f"layer{li}.{b}.conv3", batch * hw * hw, width, cout, 1))
            if b == 0:
                layers.append((f"layer{li}.{b}.downsample", batch * hw * hw, cin, cout, 1))
            cin = cout
        hw_in = hw
    return layers
