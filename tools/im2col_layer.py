"""Implicit-im2col quantize of one ResNet-50 layer (for ncu): python tools/im2col_layer.py LAYER [explicit]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth as S
from paper_2409_18772_b200 import SIDE_A, Lrqmm
name = sys.argv[1]
explicit = len(sys.argv) > 2
g = dict(S.resnet50_conv_geoms(256))[name]
M, K, N = [(m, k, n) for nm, m, k, n, _ in S.resnet50_convs(256) if nm == name][0]
dev = torch.device("cuda:0")
X = S.gen_matrix_torch("relu_normal", g["batch"] * g["H"] * g["W"], g["C"], 1, device=dev).view(g["batch"], g["H"], g["W"], g["C"])
if explicit:
    import bench
    A = torch.cat([bench.im2col_rows(X, g, torch.arange(i, min(M, i + 4096), device=dev)) for i in range(0, M, 4096)])
with Lrqmm(M, N, K, 4, 16, 5) as h:
    for _ in range(3):
        if explicit:
            h.quantize(SIDE_A, A)
        else:
            h.quantize_im2col(SIDE_A, X, g["kh"], g["kw"], g["stride"], g["pad"])
    h.sync()
print("ok")
