"""Sanity point for the overhead denominator: cuBLASLt's int8 GEMM (torch._int_mm,
int8 x int8 -> int32) at 16384^3 next to liblrqmm's bare tcgen05 int8 GEMM (lrqmm_gemm_int32) on the
same codes.  Median of 20 CUDA-event-timed launches after 3 warm-ups."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth as S  # noqa: E402
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402


def med(fn, reps=20):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(st)
        fn()
        b.record(st)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[len(t) // 2]


out = {"what": "int8 x int8 -> int32 GEMM, M = N = K", "points": []}
for n in (4096, 8192, 16384):
    dev = torch.device("cuda:0")
    A = S.gen_matrix_torch("normal", n, n, 0, device=dev)
    Bt = S.gen_matrix_torch("normal", n, n, 1, device=dev)
    C = torch.empty((n, n), dtype=torch.int32, device=dev)
    with Lrqmm(n, n, n, 8, 0, 0) as h:
        h.quantize(SIDE_A, A)
        h.quantize(SIDE_B, Bt)
        ca, cb = h.codes(SIDE_A), h.codes(SIDE_B)
        t_ours = med(lambda: h.gemm_int32(C))
        ref = C.clone()
    del A, Bt
    t_lt = med(lambda: torch._int_mm(ca, cb.t()))
    same = bool(torch.equal(torch._int_mm(ca, cb.t()), ref))
    ops = 2.0 * n ** 3
    pt = {"n": n, "lrqmm_bare_ms": t_ours, "lrqmm_tops": ops / t_ours / 1e9, "cublaslt_int_mm_ms": t_lt,
          "cublaslt_tops": ops / t_lt / 1e9, "ratio_cublaslt_over_lrqmm_time": t_lt / t_ours, "int32_identical": same}
    print(json.dumps(pt), flush=True)
    out["points"].append(pt)
    del C, ca, cb, ref
    torch.cuda.empty_cache()
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r02_cublaslt_int8.json", "w"), indent=1)
