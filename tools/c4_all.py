"""Every ResNet-50 layer of the c4 suite once (after one warm-up call), as bench.py runs them: for an
ncu launch list of the whole suite (tools/c4_breakdown.py sums it per kernel type)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth as S  # noqa: E402
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402

dev = torch.device("cuda:0")
r, p = 20, 5
geoms = dict(S.resnet50_conv_geoms(256))
for li, (name, M, K, N, _) in enumerate(S.resnet50_convs(256)):
    g = geoms[name]
    X = S.gen_matrix_torch("relu_normal", g["batch"] * g["H"] * g["W"], g["C"], 100 + 2 * li, device=dev)
    X = X.view(g["batch"], g["H"], g["W"], g["C"])
    implicit = g["kh"] * g["kw"] > 1 or g["stride"] > 1
    Bt = S.gen_matrix_torch("normal", N, K, 101 + 2 * li, device=dev, scale=(2.0 / K) ** 0.5)
    OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000 + 2 * li)).to(dev)
    OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001 + 2 * li)).to(dev)
    D = torch.empty((M, N), device=dev)
    with Lrqmm(M, N, K, 4, r, p) as h:
        for _ in range(2):
            if implicit:
                h.quantize_im2col(SIDE_A, X, g["kh"], g["kw"], g["stride"], g["pad"])
            else:
                h.quantize(SIDE_A, X.view(M, K))
            h.quantize(SIDE_B, Bt)
            h.rsvd_residual(OmA, OmB)
            h.gemm(D)
        h.sync()
    del X, Bt, D
    torch.cuda.empty_cache()
print("ok")
