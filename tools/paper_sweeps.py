"""The paper's comparisons on the GPU path (VERDICT r01 "finish the paper's comparisons"):

  rank  configs[1]: 4096^3 Gaussian, int4 and int8, r in {4, 8, 16, 32} (p = 5, q = 1): error vs the
        exact fp64 product, device time of the full call, static-B call, bare int8 GEMM -> overhead
        curves (Fig. 3(a); SURVEY E6 values for context)
  qt    QuantTensor QT(1,1,0) / QT(1,1,1) (Eq. gemm_r_split) timed next to LRQMM and
        direct quantization at 4096^3 and 16384^3 int4 (">40 % performance improvement")
  tables Tables 2/3: 2000^3, six distributions, int4 / int8, r = 10: LRQMM, DQ,
        QT errors on the GPU next to the printed values (parity with the oracle: tests/test_gpu_tables.py)

    python tools/paper_sweeps.py [rank|qt|tables ...] --out gpurun_out/r02
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth as S  # noqa: E402
from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402

DEV = torch.device("cuda:0")


def timed(fn, reps=20, warm=3):
    st = torch.cuda.current_stream(DEV)
    for _ in range(warm):
        fn()
    torch.cuda.synchronize(DEV)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        ts.append((e0, e1))
    torch.cuda.synchronize(DEV)
    v = sorted(a.elapsed_time(b) for a, b in ts)
    return v[len(v) // 2]  # median, ms


def rel_err(D, Cex, rows=None):
    Dd = D.double() if rows is None else D[rows].double()
    return float(torch.linalg.norm(Dd - Cex) / torch.linalg.norm(Cex))


def run_call(h, A, Bt, OmA, OmB, D):
    h.quantize(SIDE_A, A)
    h.quantize(SIDE_B, Bt)
    if OmA is not None:
        h.rsvd_residual(OmA, OmB)
    h.gemm(D)


def rank_sweep(out):
    M = N = K = 4096
    res = {"workload": "configs[1]: 4096^3 N(0,1), p = 5, q = 1, floor, per-row/col scales", "points": []}
    A = S.gen_matrix_torch("normal", M, K, 0, device=DEV)
    Bt = S.gen_matrix_torch("normal", N, K, 1, device=DEV)
    Cex = A.double() @ Bt.double().T
    D = torch.empty((M, N), device=DEV)
    C = torch.empty((M, N), dtype=torch.int32, device=DEV)
    Om = {s: torch.from_numpy(S.gen_omega(K, 37, s)).to(DEV) for s in (1000, 1001)}  # nested columns
    for bits in (4, 8):
        for name, rnd, gran in (("dq_paper_trunc_tensor", "trunc", "tensor"), ("dq_nearest_row", "nearest", "row")):
            with Lrqmm(M, N, K, bits, 0, 0, 1, rnd, gran) as h:
                run_call(h, A, Bt, None, None, D)
                h.sync()
                res.setdefault("dq", {})[f"int{bits}_{name}"] = rel_err(D, Cex)
        for r in (4, 8, 16, 32):
            kk = r + 5
            oa, ob = Om[1000][:, :kk].contiguous(), Om[1001][:, :kk].contiguous()
            with Lrqmm(M, N, K, bits, r, 5, 1) as h:
                t = timed(lambda: run_call(h, A, Bt, oa, ob, D))
                h.sync()
                err = rel_err(D, Cex)
                tb = timed(lambda: h.gemm_int32(C))
                h.quantize(SIDE_B, Bt)
                h.rsvd_residual_b(ob)
                ts = timed(lambda: (h.quantize(SIDE_A, A), h.rsvd_residual(oa), h.gemm(D)))
            pt = {"bits": bits, "rank": r, "rel_fro_error": err, "ms": t, "static_b_ms": ts, "bare_int8_ms": tb,
                  "overhead_vs_bare": t / tb, "static_b_overhead": ts / tb, "tops": 2.0 * M * N * K / t / 1e9}
            res["points"].append(pt)
            print(json.dumps(pt), flush=True)
    res["survey_E6_context"] = {"int4": {"4": 0.2239, "8": 0.2236, "16": 0.2230, "32": 0.2219, "dq_trunc": 0.602},
                                "int8": {"4": 1.227e-2, "32": 1.216e-2}}
    json.dump(res, open(out + "_rank_sweep.json", "w"), indent=1)


def qt_timing(out):
    res = {"note": "QT(1,1,0) = 3 int8 GEMMs, QT(1,1,1) = 4 (Eq. gemm_r_split, PAPER.md:268-275), trunc + per-tensor "
                   "scales (reading #27); every call re-quantizes both operands and their residuals", "configs": []}
    for (M, label) in ((4096, "4096^3 int4"), (16384, "16384^3 int4")):
        N = K = M
        A = S.gen_matrix_torch("normal", M, K, 0, device=DEV)
        Bt = S.gen_matrix_torch("normal", N, K, 1, device=DEV)
        rows = torch.arange(0, M, max(1, M // 256), device=DEV)[:256]
        Cex = A[rows].double() @ Bt.double().T
        D = torch.empty((M, N), device=DEV)
        oa = torch.from_numpy(S.gen_omega(K, 21, 1000)).to(DEV)
        ob = torch.from_numpy(S.gen_omega(K, 21, 1001)).to(DEV)
        row = {"workload": label}
        for name, kw, om in (("lrqmm_r16", dict(rank=16, oversample=5), (oa, ob)),
                             ("dq_floor_row", dict(rank=0, oversample=0), (None, None)),
                             ("dq_paper_trunc_tensor", dict(rank=0, oversample=0, rounding="trunc", granularity="tensor"),
                              (None, None)),
                             ("qt110_trunc_tensor", dict(rank=0, oversample=0, rounding="trunc", granularity="tensor",
                                                         qt_terms=3), (None, None)),
                             ("qt111_trunc_tensor", dict(rank=0, oversample=0, rounding="trunc", granularity="tensor",
                                                         qt_terms=4), (None, None))):
            with Lrqmm(M, N, K, 4, **kw) as h:
                t = timed(lambda: run_call(h, A, Bt, om[0], om[1], D), reps=10 if M > 8192 else 20)
                h.sync()
                row[name] = {"ms": t, "rel_fro_error": rel_err(D, Cex, rows)}
        row["lrqmm_speedup_vs_qt110"] = row["qt110_trunc_tensor"]["ms"] / row["lrqmm_r16"]["ms"]
        row["lrqmm_speedup_vs_qt111"] = row["qt111_trunc_tensor"]["ms"] / row["lrqmm_r16"]["ms"]
        res["configs"].append(row)
        print(json.dumps(row), flush=True)
        del A, Bt, D, Cex
        torch.cuda.empty_cache()
    res["paper_claim"] = ">40 % performance improvement over QuantTensor (PAPER.md:853), A100"
    json.dump(res, open(out + "_qt_timing.json", "w"), indent=1)


def tables(out):
    gold = {}
    for line in open(os.path.join(ROOT, "tests", "golden", "paper_tables_2_3.txt")):
        if line.startswith("#") or not line.strip():
            continue
        d, b, dq, q110, q111, lr = line.split()
        gold[(d, int(b))] = dict(dq=float(dq), qt110=float(q110), qt111=float(q111), lrqmm=float(lr))
    res = {"workload": "2000^3, r = 10 (p = 5, q = 1), Tables 2/3 (PAPER.md:711-744); seeds s = 0", "cells": []}
    M = N = K = 2000
    for (dist, bits), g in sorted(gold.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        A, Bt, OmA, OmB = S.problem(M, N, K, 15, s=0, dist=dist)
        a, b = torch.from_numpy(A).to(DEV), torch.from_numpy(Bt).to(DEV)
        oa, ob = torch.from_numpy(OmA).to(DEV), torch.from_numpy(OmB).to(DEV)
        Cex = a.double() @ b.double().T
        D = torch.empty((M, N), device=DEV)
        cell = {"dist": dist, "bits": bits, "paper": g}
        for name, kw, om in (("lrqmm", dict(rank=10, oversample=5), (oa, ob)),
                             ("dq", dict(rank=0, oversample=0, rounding="trunc", granularity="tensor"), (None, None)),
                             ("qt110", dict(rank=0, oversample=0, rounding="trunc", granularity="tensor", qt_terms=3),
                              (None, None)),
                             ("qt111", dict(rank=0, oversample=0, rounding="trunc", granularity="tensor", qt_terms=4),
                              (None, None))):
            with Lrqmm(M, N, K, bits, **kw) as h:
                run_call(h, a, b, om[0], om[1], D)
                h.sync()
                e = rel_err(D, Cex)
            cell[name] = e
            cell[name + "_vs_paper"] = e / g[name]
        res["cells"].append(cell)
        print(json.dumps(cell), flush=True)
    json.dump(res, open(out + "_tables_2_3_gpu.json", "w"), indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="*", default=["rank", "qt", "tables"])
    ap.add_argument("--out", default="gpurun_out/r02")
    a = ap.parse_args()
    for w in a.what:
        {"rank": rank_sweep, "qt": qt_timing, "tables": tables}[w](a.out)
