"""Per-phase device times (CUDA events inside liblrqmm) at a bench config."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth as S
from bench import CONFIGS
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="c3"); ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
M, N, K, bits, r, p, dist, _ = CONFIGS[a.config]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch(dist, M, K, 0, device=dev); Bt = S.gen_matrix_torch(dist, N, K, 1, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000)).to(dev); OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001)).to(dev)
D = torch.empty((M, N), device=dev)
with Lrqmm(M, N, K, bits, r, p, enable_timing=True) as h:
    acc = {}
    for i in range(a.steps + 2):
        h.quantize(SIDE_A, A); h.quantize(SIDE_B, Bt); h.rsvd_residual(OmA, OmB); h.gemm(D)
        t = h.timings_us()
        if i >= 2:
            for k, v in t.items(): acc[k] = acc.get(k, 0) + v / a.steps
print({k: round(v, 1) for k, v in acc.items()})
