"""Run a few LRQMM steps at a bench config (for ncu / compute-sanitizer captures).

    python tools/one_step.py --config c3 --steps 2 [--bare]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth as S  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--bare", action="store_true")
    ap.add_argument("--rank", type=int, default=None)
    a = ap.parse_args()
    M, N, K, bits, r, p, dist, _ = CONFIGS[a.config]
    r = a.rank if a.rank is not None else r
    dev = torch.device("cuda:0")
    A = S.gen_matrix_torch(dist, M, K, 0, device=dev)
    Bt = S.gen_matrix_torch(dist, N, K, 1, device=dev)
    OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000)).to(dev)
    OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001)).to(dev)
    D = torch.empty((M, N), device=dev)
    C = torch.empty((M, N), dtype=torch.int32, device=dev)
    with Lrqmm(M, N, K, bits, r, p) as h:
        for _ in range(a.steps):
            h.quantize(SIDE_A, A)
            h.quantize(SIDE_B, Bt)
            h.rsvd_residual(OmA, OmB)
            h.gemm(D)
            if a.bare:
                h.gemm_int32(C)
        h.sync()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
