"""One LRQMM step on a ResNet-50 layer shape (for ncu launch lists): python tools/one_layer.py LAYER."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth as S
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm
name = sys.argv[1]
M, K, N = [(m, k, n) for nm, m, k, n, _ in S.resnet50_convs(256) if nm == name][0]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch("relu_normal", M, K, 1, device=dev); Bt = S.gen_matrix_torch("normal", N, K, 2, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, 21, 3)).to(dev); OmB = torch.from_numpy(S.gen_omega(K, 21, 4)).to(dev)
D = torch.empty((M, N), device=dev)
with Lrqmm(M, N, K, 4, 16, 5) as h:
    for _ in range(3):
        h.quantize(SIDE_A, A); h.quantize(SIDE_B, Bt); h.rsvd_residual(OmA, OmB); h.gemm(D)
    h.sync()
