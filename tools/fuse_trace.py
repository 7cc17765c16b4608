"""Timing trace of the fused RSVD passes (LRQMM_FUSE_TRACE=1): per pass, the first CTA start, the
first / last CTA done with its units, and the solver start / end of the last CTA (microseconds
from the first CTA start)."""
import ctypes
import os
import sys

os.environ["LRQMM_FUSE_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth as S  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
M, N, K, bits, r, p, dist, _ = CONFIGS[cfg]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch(dist, M, K, 0, device=dev)
Bt = S.gen_matrix_torch(dist, N, K, 1, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000)).to(dev)
OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001)).to(dev)
D = torch.empty((M, N), device=dev)
with Lrqmm(M, N, K, bits, r, p) as h:
    out = (ctypes.c_int64 * 64)()
    for step in range(4):
        h.quantize(SIDE_A, A); h.quantize(SIDE_B, Bt); h.rsvd_residual(OmA, OmB); h.gemm(D)
        h.sync()
        h.lib.lrqmm_debug_fuse_trace(h.h, out)
        print(f"step {step}")
        for i in range(8):
            t = out[8 * i: 8 * i + 5]
            if t[1] == 0:
                continue
            t0 = t[0]
            print(f"  slot {i}: first done {(t[4] - t0) / 1e3:7.1f} us  last done {(t[1] - t0) / 1e3:7.1f} us"
                  f"  solver {(t[2] - t0) / 1e3:7.1f} -> {(t[3] - t0) / 1e3:7.1f} us")
