"""Time the one-CTA (K6) and CTA-pair (K7) GEMMs on the c3 problem (fused epilogue and int32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth as S
from bench import CONFIGS
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm, lrqmm as L
M, N, K, bits, r, p, dist, _ = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda:0")
A = S.gen_matrix_torch(dist, M, K, 0, device=dev); Bt = S.gen_matrix_torch(dist, N, K, 1, device=dev)
OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000)).to(dev); OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001)).to(dev)
D = torch.empty((M, N), device=dev); C = torch.empty((M, N), dtype=torch.int32, device=dev)
lib = L.load_library()
with Lrqmm(M, N, K, bits, r, p) as h:
    h.quantize(SIDE_A, A); h.quantize(SIDE_B, Bt); h.rsvd_residual(OmA, OmB); h.sync()
    for v in (1, 2, 1, 2):
        lib.lrqmm_debug_set_gemm_variant(v)
        for name, fn in (("fused", lambda: h.gemm(D)), ("int32", lambda: h.gemm_int32(C))):
            for _ in range(3): fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): fn()
            e1.record(); torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 20
            print(f"variant {v} {name}: {t*1e3:.1f} us  {2*M*N*K/t/1e9:.0f} TOPS")
    lib.lrqmm_debug_set_gemm_variant(0)
