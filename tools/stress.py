"""Repetition stress test: the same LRQMM call many times (graph replays, dynamic GEMM scheduler,
ticket-based reductions, forked branch) must give bit-identical D every time.

    python tools/stress.py [--config c2] [--iters 500]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth as S
from bench import CONFIGS
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=500)
ap.add_argument("--q", type=int, default=1)
a = ap.parse_args()
M, N, K, bits, r, p, dist, _ = CONFIGS[a.config]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch(dist, M, K, 5, device=dev)
Bt = S.gen_matrix_torch(dist, N, K, 6, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 7)).to(dev)
OmB = torch.from_numpy(S.gen_omega(K, r + p, 8)).to(dev)
D = torch.empty((M, N), device=dev)
ref = None
bad = 0
with Lrqmm(M, N, K, bits, r, p, a.q) as h:
    for i in range(a.iters):
        h.quantize(SIDE_A, A); h.quantize(SIDE_B, Bt); h.rsvd_residual(OmA, OmB); h.gemm(D)
        if i % 10 == 9 or i == 0:
            h.sync()
            if ref is None:
                ref = D.clone()
            elif not torch.equal(D.view(torch.int32), ref.view(torch.int32)):
                bad += 1
                print(f"iteration {i}: D differs ({(D != ref).sum().item()} elements)")
    h.sync()
print(f"{a.config} q={a.q}: {a.iters} calls, {bad} mismatching checks")
sys.exit(1 if bad else 0)
