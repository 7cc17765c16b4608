"""Phase timestamps of the last k_prep_img launch (build with -DLRQMM_PREP_TIMING)."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth as S
from bench import CONFIGS
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm, lrqmm as L
M, N, K, bits, r, p, dist, _ = CONFIGS["c3"]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch(dist, M, K, 0, device=dev); Bt = S.gen_matrix_torch(dist, N, K, 1, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000)).to(dev); OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001)).to(dev)
D = torch.empty((M, N), device=dev)
lib = L.load_library()
with Lrqmm(M, N, K, bits, r, p) as h:
    for i in range(3):
        h.quantize(SIDE_A, A); h.quantize(SIDE_B, Bt); h.rsvd_residual(OmA, OmB); h.gemm(D); h.sync()
    t = (ctypes.c_ulonglong * 8)()
    lib.lrqmm_debug_prep_times(t)
    print("phase ns:", [t[i] - t[0] for i in range(6)])
