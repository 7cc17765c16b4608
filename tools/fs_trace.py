"""Phase stamps of k_fused_small (a build with -DLRQMM_FS_TRACE, loaded through LRQMM_LIB):
block 0 start / Gram done / partial written, finisher start / G staged / solver done, for the last
CholQR (mode 0) and truncation (mode 1) launch of a few calls at a bench config.
    LRQMM_LIB=tools/bin/liblrqmm_fstrace.so python tools/fs_trace.py --config c2"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth as S  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402
from paper_2409_18772_b200 import lrqmm as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
a = ap.parse_args()
M, N, K, bits, r, p, dist, _ = CONFIGS[a.config]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch(dist, M, K, 0, device=dev)
Bt = S.gen_matrix_torch(dist, N, K, 1, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 3)).to(dev)
OmB = torch.from_numpy(S.gen_omega(K, r + p, 4)).to(dev)
D = torch.empty((M, N), device=dev)
with Lrqmm(M, N, K, bits, r, p) as h:
    for _ in range(3):
        h.quantize(SIDE_A, A)
        h.quantize(SIDE_B, Bt)
        h.rsvd_residual(OmA, OmB)
        h.gemm(D)
    h.sync()
lib = L.load_library()
buf = (ctypes.c_ulonglong * 16)()
assert lib.lrqmm_debug_fs_trace(buf) == 0
names = ["blk0 start", "blk0 Gram done", "blk0 partial written", "finisher start", "G staged", "solver done"]
for mode in (0, 1):
    t = [buf[8 * mode + i] for i in range(6)]
    print(f"mode {mode} ({'CholQR' if mode == 0 else 'truncation'}):",
          "  ".join(f"{names[i]} +{(t[i] - t[0]) / 1e3:.1f}us" for i in range(1, 6)))
print("Jacobi steps of the last truncation (with -DLRQMM_EIG_STATS):", buf[15])
