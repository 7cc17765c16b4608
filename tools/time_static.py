"""Per-call device time of the static-B step (quantize A + rsvd_residual(omega_a) + gemm) vs the full
step, c3 shapes, CUDA events around each phase."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth as S
from bench import CONFIGS
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm
M, N, K, bits, r, p, dist, _ = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch(dist, M, K, 0, device=dev); Bt = S.gen_matrix_torch(dist, N, K, 1, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000)).to(dev); OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001)).to(dev)
D = torch.empty((M, N), device=dev)
with Lrqmm(M, N, K, bits, r, p) as h:
    h.quantize(SIDE_B, Bt); h.rsvd_residual_b(OmB)
    def ev(): return torch.cuda.Event(enable_timing=True)
    for mode in ("static", "full", "static"):
        ts = []
        for i in range(8):
            e = [ev() for _ in range(4)]
            e[0].record()
            h.quantize(SIDE_A, A)
            if mode == "full": h.quantize(SIDE_B, Bt)
            e[1].record()
            h.rsvd_residual(OmA, None if mode == "static" else OmB)
            e[2].record()
            h.gemm(D)
            e[3].record()
            torch.cuda.synchronize()
            if i >= 2: ts.append([e[j].elapsed_time(e[j + 1]) * 1e3 for j in range(3)])
        import numpy as np
        t = np.mean(ts, axis=0)
        print(f"{mode:6s} quantize {t[0]:7.1f} us  rsvd {t[1]:7.1f} us  gemm {t[2]:7.1f} us  total {t.sum():7.1f} us")
