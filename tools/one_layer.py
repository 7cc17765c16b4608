"""A few LRQMM steps on one ResNet-50 layer exactly as bench.py's c4 suite runs it (r = 20, p = 5;
windowed / strided layers through implicit im2col), for ncu launch lists:
    python tools/one_layer.py LAYER [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth as S  # noqa: E402
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
M, K, N = [(m, k, n) for nm, m, k, n, _ in S.resnet50_convs(256) if nm == name][0]
g = dict(S.resnet50_conv_geoms(256))[name]
r, p = 20, 5
dev = torch.device("cuda:0")
X = S.gen_matrix_torch("relu_normal", g["batch"] * g["H"] * g["W"], g["C"], 1, device=dev)
X = X.view(g["batch"], g["H"], g["W"], g["C"])
implicit = g["kh"] * g["kw"] > 1 or g["stride"] > 1
Bt = S.gen_matrix_torch("normal", N, K, 2, device=dev, scale=(2.0 / K) ** 0.5)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 3)).to(dev)
OmB = torch.from_numpy(S.gen_omega(K, r + p, 4)).to(dev)
D = torch.empty((M, N), device=dev)
with Lrqmm(M, N, K, 4, r, p) as h:
    for _ in range(steps):
        if implicit:
            h.quantize_im2col(SIDE_A, X, g["kh"], g["kw"], g["stride"], g["pad"])
        else:
            h.quantize(SIDE_A, X.view(M, K))
        h.quantize(SIDE_B, Bt)
        h.rsvd_residual(OmA, OmB)
        h.gemm(D)
    h.sync()
print("ok", name, M, K, N, "implicit" if implicit else "activations")
