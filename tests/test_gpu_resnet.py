"""ResNet-50 im2col-shaped GEMMs (BASELINE.json configs[3]) vs the full oracle at a reduced batch.

A = im2col of post-ReLU activations (rows = batch x H_out x W_out, K = C_in x kh x kw), B = conv
weights (N = C_out), 4-bit, r = 16, p = 5 (synth.resnet50_convs gives the shapes).  The bench runs
the same layers at batch 256; this test runs them at batch 2 so that the fp64 oracle evaluates
Algorithm 2 in full.  Covers short K (64, 147), long K (4608), narrow N (64) and tall M.
"""
import numpy as np
import pytest

import oracle as O
import synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402

DEV = "cuda:0"
LAYERS = {name: (m, k, n) for name, m, k, n, _ in S.resnet50_convs(batch=2)}


@pytest.mark.parametrize("name", ["conv1", "layer1.0.conv1", "layer1.0.conv2", "layer2.0.conv3",
                                  "layer3.2.conv2", "layer4.0.conv2", "layer4.2.conv3"])
def test_resnet_layer_matches_oracle(name):
    M, K, N = LAYERS[name]
    bits, r, p = 4, 16, 5
    A = S.gen_matrix("relu_normal", M, K, 31)
    Bt = S.gen_matrix("normal", N, K, 32, scale=float(np.sqrt(2.0 / K)))  # Kaiming-normal weights
    OmA = S.gen_omega(K, r + p, 33)
    OmB = S.gen_omega(K, r + p, 34)
    ref, parts = O.lrqmm(A, Bt, bits, r, OmA, OmB, q=1, return_parts=True)
    with Lrqmm(M, N, K, bits, r, p) as h:
        h.quantize(SIDE_A, torch.from_numpy(A).to(DEV))
        h.quantize(SIDE_B, torch.from_numpy(Bt).to(DEV))
        h.rsvd_residual(torch.from_numpy(OmA).to(DEV), torch.from_numpy(OmB).to(DEV))
        D = torch.empty((M, N), device=DEV)
        h.gemm(D)
        C = torch.empty((M, N), dtype=torch.int32, device=DEV)
        h.gemm_int32(C)
        h.sync()
        d = D.double().cpu().numpy()
        c = C.cpu().numpy().astype(np.int64)
        ca = h.codes(SIDE_A).cpu().numpy().astype(np.int64)
    assert np.array_equal(ca, parts["codes_a"])
    assert np.array_equal(c, parts["c_int"])
    Cx = O.matmul_exact(A, Bt)
    diff = O.relative_error(ref, d)
    e_gpu, e_or = O.relative_error(Cx, d), O.relative_error(Cx, ref)
    assert diff <= 1e-4, (name, diff, e_gpu, e_or)
    assert e_gpu <= 1.05 * e_or + 1e-12, (name, e_gpu, e_or)
