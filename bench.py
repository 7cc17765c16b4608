#!/usr/bin/env python
"""LRQMM hot-path benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lrqmm|reference] [--config c3|c2|c1]

A step = one pass of the whole hot path over one batch of synthetic input:
quantize(A), quantize(B), rsvd_residual, gemm (Algorithm 2).
Default workload (N=1): BASELINE.json configs[2], 16384^3 int4, rank 16, p=5, q=1,
Gaussian A and B.  Under torchrun (N>1) the SAME problem is split (strong
scaling, the north_star's 16384^3 on 8 GPUs): rank i holds M/N rows of A and,
by default, n/N rows of B^T; the A- and B-side RSVDs are
coupled by NCCL allreduces inside liblrqmm and the B codes / scales / L_B
are allgathered.  `--config c5` is configs[4] (32768^3, r = 32).

One JSON line on rank 0.  `value` = effective TOPS (2*M*N*K / step time, all
ranks), inputs resident in HBM (2 GiB of fp32 inputs per GPU > 126 MB L2, so no
L2 flush is needed).  `e2e` = the same metric through lrqmm_run_host with pinned
HOST buffers (H2D of A, B^T, Omega and D2H of D inside the timed region).
`--impl reference` times the fp64 CPU oracle (test infrastructure) on a
bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (M (global; split over the ranks), N, K, bits, rank, oversample, dist, workload label)
    "c3": (16384, 16384, 16384, 4, 16, 5, "normal", "square 16384^3 int4 rank 16 (p=5, q=1) Gaussian, configs[2]"),
    "c2": (4096, 4096, 4096, 4, 16, 5, "normal", "square 4096^3 int4 rank 16 (p=5, q=1) Gaussian, configs[1]"),
    "c2i8": (4096, 4096, 4096, 8, 16, 5, "normal", "square 4096^3 int8 rank 16 (p=5, q=1) Gaussian, configs[1]"),
    "c1": (256, 256, 256, 4, 8, 5, "normal", "square 256^3 int4 rank 8 (p=5, q=1) Gaussian, configs[0]"),
    "c5": (32768, 32768, 32768, 4, 32, 5, "normal", "32768^3 int4 rank 32 row-sharded over the GPUs, configs[4]"),
    # configs[3]: the 53 ResNet-50 convolutions as im2col GEMMs at batch 256 (synth.resnet50_convs)
    "c4": (None, None, None, 4, 20, 5, "relu_normal",
           "ResNet-50 conv layers as im2col GEMMs, batch 256, 4-bit, rank 20 (PAPER.md:822), configs[3]"),
}
METRIC = "effective TOPS (2MNK/t) of the LRQMM hot path; overhead vs bare int8 GEMM; rel. Frobenius error vs direct quant"
REF_ROWS = 256  # oracle row sample per reference / cpu_baseline step


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lrqmm", choices=["lrqmm", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--b-replicated", action="store_true",
                    help="N > 1: every rank quantizes and RSVDs all of B (SURVEY §8(e)(i)) instead of the default "
                         "column-sharded B (§8(e)(ii): codes, scales and L_B allgathered)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# --------------------------------------------------------------- clocks
class ClockSampler:
    """Polls SM clock, max clock, power and throttle reasons through NVML every 10 ms while the
    timed region runs (the profiling recipe's clocks line, sampled in-process)."""

    REASONS = {  # nvmlClocksEventReason* bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int, period_s: float = 0.01):
        self.index = index
        self.period = period_s
        self.samples = []
        self.stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((sm, rs, pw))
            except Exception:
                pass
            self.stop.wait(self.period)

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({nm for _, rs, _ in self.samples for nm, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(sm), "sm_mhz_min": sm[0], "power_w_max": max(s[2] for s in self.samples)}


# -------------------------------------------------------------- dist utils
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, ws: int, device) -> float:
    """Device time of the slowest rank (the contract's max over ranks)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def broadcast_unique_id(uid: bytes | None, ws: int, rank: int, device) -> bytes:
    """Rank 0's 128-byte NCCL unique id (lrqmm_get_unique_id) to every rank, over the process group."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        assert uid is not None and len(uid) == 128
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    if ws > 1:
        dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def row_shard(M_total: int, ws: int, rank: int) -> tuple[int, int]:
    """[start, stop) rows of A owned by `rank` when M_total rows are split over ws ranks
    (contiguous blocks, the first M_total % ws ranks one row longer)."""
    base, extra = divmod(M_total, ws)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


# ------------------------------------------------------------ oracle legs
def oracle_sample(cfg, seed_base=0, rows=REF_ROWS, b_rows=None, phases=None):
    """Time the fp64 oracle (as it stands) on a bounded row sample of the workload:
    the first `rows` rows of A against the first `b_rows` rows of B^T (all by default; the B-side
    quantize + RSVD is the sample's dominant cost).  Returns (seconds, ops_sampled)."""
    import numpy as np

    import oracle as O
    import synth as S

    M, N, K, bits, r, p, dist_name, _ = cfg
    N = N if b_rows is None else min(N, b_rows)
    A = S.gen_matrix(dist_name, rows, K, 2 * seed_base)
    Bt = S.gen_matrix(dist_name, N, K, 2 * seed_base + 1)
    OmA = S.gen_omega(K, r + p, 1000 + 2 * seed_base)
    OmB = S.gen_omega(K, r + p, 1001 + 2 * seed_base)
    t0 = time.perf_counter()
    O.lrqmm(A, Bt, bits, r, OmA, OmB, q=1)
    dt = time.perf_counter() - t0
    if phases is not None:
        # the oracle's own steps one by one on the same sample: wall clock per phase
        def timed(name, f):
            t = time.perf_counter()
            out = f()
            phases[name] = time.perf_counter() - t
            return out
        ca, la = timed("quantize_A", lambda: O.quantize(A, bits))
        cb, lb = timed("quantize_B", lambda: O.quantize(Bt, bits))
        RA = O.residual(A, ca, la)
        RB = O.residual(Bt, cb, lb)
        timed("rsvd_A", lambda: O.rsvd(RA, OmA, r, 1))
        timed("rsvd_B", lambda: O.rsvd(RB, OmB, r, 1))
        c = timed("int_gemm", lambda: O.int_gemm(ca, cb))
        timed("dequant", lambda: O.dequant_result(c, la, lb))
        timed("C_exact", lambda: O.matmul_exact(A, Bt))
    del A, Bt
    return dt, 2.0 * rows * N * K


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, ws, rank):
    cfg = CONFIGS[args.config]
    if rank != 0:
        return
    M, N, K = cfg[0], cfg[1], cfg[2]
    # bounded: a full-B sample costs ~6 s on 16 cores; beyond 12 steps + warmups the B sample
    # shrinks so that the whole run stays within ~2 minutes
    nsteps = args.warmup + args.steps
    b_rows = N if nsteps <= 12 else max(1024, N * 12 // nsteps)
    times = []
    ops = 0.0
    for i in range(nsteps):
        dt, ops = oracle_sample(cfg, b_rows=b_rows)
        if i >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    val = ops / t / 1e12
    sample = (f"oracle (NumPy fp64) on the first {REF_ROWS} rows of A x the first {b_rows} rows of B^T "
              f"(of {cfg[1]}x{cfg[2]}), incl. quantize+RSVD of that B sample")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TOPS", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg[7], "M": M, "N": N, "K": K, "bits": cfg[3], "rank": cfg[4], "oversample": cfg[5],
                   "power_iters": 1, "sample_rows": REF_ROWS},
        "cpu_baseline": {"value": val, "unit": "TOPS", "cores": cpu_cores(), "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ HBM roofline inputs
def hbm_peak() -> float:
    peaks, _ = load_peaks()
    return float(peaks["hbm_gbs"])


def hbm_bytes_quantize(rows: int, K: int, rank: bool) -> float:
    """Algorithmic HBM bytes of K1 per side: read x (4 B), write codes (1 B) and, with rank > 0, the
    Q15 residual planes (2 B) per element."""
    return rows * K * (4 + 1 + (2 if rank else 0))


def hbm_bytes_rsvd(rows: int, K: int) -> float:
    """Algorithmic HBM bytes of one side's three RSVD passes: S1 and S2 stream the 2-byte residual,
    S3 the residual + the 1-byte codes (the sketch panels are L2-sized at these shapes)."""
    return rows * K * (2 + 2 + 3)


def hbm_bytes_step(M: int, N: int, K: int, k: int) -> float:
    """Whole-step algorithmic HBM bytes: quantize + RSVD both sides, GEMM operands + fp32 D."""
    return (hbm_bytes_quantize(M, K, True) + hbm_bytes_quantize(N, K, True) + hbm_bytes_rsvd(M, K)
            + hbm_bytes_rsvd(N, K) + (M + N) * K + 4.0 * M * N)


# ------------------------------------------------------ configs[3]: ResNet-50 suite
def im2col_rows(X, g, rows):
    """Explicit im2col rows (b, ho, wo) -> (i, j, c) of an NHWC tensor, for the error sample only."""
    import torch

    s, p, kh, kw = g["stride"], g["pad"], g["kh"], g["kw"]
    Xp = torch.nn.functional.pad(X, (0, 0, p, p, p, p))
    Ho = (g["H"] + 2 * p - kh) // s + 1
    Wo = (g["W"] + 2 * p - kw) // s + 1
    out = []
    for r in rows.tolist():
        b, rem = divmod(r, Ho * Wo)
        ho, wo = divmod(rem, Wo)
        out.append(Xp[b, ho * s: ho * s + kh, wo * s: wo * s + kw, :].reshape(-1))
    return torch.stack(out)


def run_resnet(args, ws, rank, local):
    """All 53 ResNet-50 convolutions as im2col GEMMs at batch 256 (A: post-ReLU activations,
    B: Kaiming-normal random-init weights), int4, r = 16, p = 5: per-layer device time of the full
    LRQMM call sequence, bare int8 GEMM time and error on 64 sampled rows; suite effective TOPS."""
    import torch

    import synth as S
    from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm

    _, _, _, bits, r, p, dist_name, label = CONFIGS["c4"]
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    layers = S.resnet50_convs(256)
    geoms = dict(S.resnet50_conv_geoms(256))
    out, t_all, t_bare_all, ops_all, hbm_all, t_static_all = [], 0.0, 0.0, 0.0, 0.0, 0.0
    steps = max(1, min(args.steps, 5))
    for li, (name, M, K, N, _) in enumerate(layers):
        g = geoms[name]
        # post-ReLU NHWC activations; windowed / strided layers quantize their im2col implicitly
        # (lrqmm_quantize_im2col), 1x1 stride-1 layers use the activations as A directly
        X = S.gen_matrix_torch(dist_name, g["batch"] * g["H"] * g["W"], g["C"], 100 + 2 * li + 7919 * rank, device=dev)
        X = X.view(g["batch"], g["H"], g["W"], g["C"])
        implicit = g["kh"] * g["kw"] > 1 or g["stride"] > 1
        A = None if implicit else X.view(M, K)
        Bt = S.gen_matrix_torch("normal", N, K, 101 + 2 * li, device=dev, scale=(2.0 / K) ** 0.5)
        OmA = torch.from_numpy(S.gen_omega(K, r + p, 1000 + 2 * li)).to(dev)
        OmB = torch.from_numpy(S.gen_omega(K, r + p, 1001 + 2 * li)).to(dev)
        D = torch.empty((M, N), device=dev)
        C = torch.empty((M, N), dtype=torch.int32, device=dev)
        with Lrqmm(M, N, K, bits, r, p, 1, "floor", "row", device=local, stream=stream) as h:
            def quant_a():
                if implicit:
                    h.quantize_im2col(SIDE_A, X, g["kh"], g["kw"], g["stride"], g["pad"])
                else:
                    h.quantize(SIDE_A, A)

            def step():
                quant_a(); h.quantize(SIDE_B, Bt); h.rsvd_residual(OmA, OmB); h.gemm(D)
            for _ in range(max(args.warmup, 1)):
                step()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            t = e0.elapsed_time(e1) / 1e3 / steps
            h.gemm_int32(C)
            torch.cuda.synchronize(dev)
            e0.record(stream)
            for _ in range(steps):
                h.gemm_int32(C)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            tb = e0.elapsed_time(e1) / 1e3 / steps
            # weight-resident deployment (static-B): B quantized + RSVD'd once, per call
            # only the activation side, the A-dependent B term and the GEMM
            h.quantize(SIDE_B, Bt)
            h.rsvd_residual_b(OmB)

            def step_static():
                quant_a(); h.rsvd_residual(OmA); h.gemm(D)
            for _ in range(2):
                step_static()
            torch.cuda.synchronize(dev)
            e0.record(stream)
            for _ in range(steps):
                step_static()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ts = e0.elapsed_time(e1) / 1e3 / steps
            step()
            h.sync()
            rows = torch.arange(0, M, max(1, M // 64), device=dev)[:64]
            Cx = im2col_rows(X, g, rows).double() @ Bt.double().T
            err = float(torch.linalg.norm(D[rows].double() - Cx) / torch.linalg.norm(Cx))
        ops = 2.0 * M * N * K
        # implicit im2col: K1 reads the activations once (L2 reuse across windows), not M x K floats
        hbm = hbm_bytes_step(M, N, K, r + p) - (4.0 * M * K - 4.0 * X.numel() if implicit else 0.0)
        out.append({"layer": name, "M": M, "K": K, "N": N, "ms": t * 1e3, "static_b_ms": ts * 1e3, "bare_int8_ms": tb * 1e3,
                    "overhead_vs_bare": t / tb, "tops": ops / t / 1e12, "rel_fro_error": err,
                    "hbm_gbs": hbm / t / 1e9, "hbm_frac": hbm / t / 1e9 / hbm_peak()})
        t_all += t; t_bare_all += tb; ops_all += ops; hbm_all += hbm; t_static_all += ts
        out[-1]["a_input"] = "implicit im2col" if implicit else "activations"
        del A, X, Bt, D, C
        torch.cuda.empty_cache()
    if rank == 0:
        line = {"metric": METRIC, "value": ops_all / t_all / 1e12, "unit": "TOPS", "n_gpus": ws, "steps": steps,
                "warmup": args.warmup, "ms_per_step": t_all * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "int8",
                "data": "synthetic (post-ReLU normal NHWC activations, Kaiming weights); windowed / strided layers "
                        "quantized by implicit im2col (lrqmm_quantize_im2col)",
                "config": {"workload": label, "layers": len(layers), "bits": bits, "rank": r, "oversample": p,
                           "batch": 256},
                "overhead_vs_bare_int8": t_all / t_bare_all, "bare_int8_tops": ops_all / t_bare_all / 1e12,
                "static_b": {"ms_per_step": t_static_all * 1e3, "value": ops_all / t_static_all / 1e12, "unit": "TOPS",
                             "overhead_vs_bare_int8": t_static_all / t_bare_all,
                             "note": "weight-resident deployment (SURVEY f2): per layer quantize(A) + rsvd_residual(omega_a) "
                                     "+ gemm with B's codes and factors from lrqmm_rsvd_residual_b"},
                "hbm_roofline": {"bytes": hbm_all, "gbs": hbm_all / t_all / 1e9, "peak_gbs": hbm_peak(),
                                 "frac": hbm_all / t_all / 1e9 / hbm_peak(),
                                 "note": "algorithmic bytes of the whole LRQMM call per layer (bench.hbm_bytes_step)"},
                "layers": out}
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ e2e context
def pcie_context(dev, nbytes_in: int, nbytes_out: int) -> dict:
    """Achieved pinned host->device and device->host GB/s for copies of the e2e step's sizes (CUDA
    events), and the NUMA placement of the GPU and of this process's CPUs: the e2e number is
    PCIe-bound, so these explain its spread across boxes."""
    import torch

    out = {}
    try:
        n_in = min(nbytes_in, 1 << 30) // 4
        n_out = min(nbytes_out, 1 << 30) // 4
        h = torch.empty(max(n_in, n_out), dtype=torch.float32, pin_memory=True)
        d = torch.empty(max(n_in, n_out), dtype=torch.float32, device=dev)
        st = torch.cuda.current_stream(dev)
        for name, n, fn in (("h2d_gbs", n_in, lambda n: d[:n].copy_(h[:n], non_blocking=True)),
                            ("d2h_gbs", n_out, lambda n: h[:n].copy_(d[:n], non_blocking=True))):
            fn(n)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(3):
                fn(n)
            e1.record(st)
            torch.cuda.synchronize(dev)
            out[name] = 3 * 4.0 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
        del h, d
    except Exception as e:  # context only
        out["pcie_error"] = str(e)[:120]
    try:
        pr = torch.cuda.get_device_properties(dev)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        out["gpu_pci"] = bus
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            out["gpu_numa_node"] = int(f.read().strip())
    except Exception:
        out["gpu_numa_node"] = None
    try:
        cpus = sorted(os.sched_getaffinity(0))
        nodes = set()
        base = "/sys/devices/system/node"
        for nd in os.listdir(base):
            if not nd.startswith("node"):
                continue
            txt = open(os.path.join(base, nd, "cpulist")).read().strip()
            ids = set()
            for part in txt.split(","):
                if "-" in part:
                    a, b = part.split("-")
                    ids.update(range(int(a), int(b) + 1))
                elif part:
                    ids.add(int(part))
            if ids & set(cpus):
                nodes.add(int(nd[4:]))
        out["process_cpu_numa_nodes"] = sorted(nodes)
        out["process_cpus"] = len(cpus)
    except Exception:
        pass
    return out


# ------------------------------------------------------------------ main
def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if ws > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    import numpy as np
    import torch

    import synth as S
    from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm, get_unique_id

    if args.config == "c4":
        run_resnet(args, ws, rank, local)
        return
    cfg = CONFIGS[args.config]
    M, N, K, bits, r, p, dist_name, label = cfg
    kk = r + p
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)

    # strong scaling (north_star: the one GEMM split over the GPUs): rank i owns rows [lo, hi) of A
    # and, unless --b-replicated, rows [blo, bhi) of B^T; N=1 is the whole problem
    lo, hi = row_shard(M, ws, rank)
    Mloc = hi - lo
    bsh = ws > 1 and not args.b_replicated
    # synthetic inputs, resident in HBM: the GLOBAL A is one seeded draw, so every N sees the same
    # problem (each rank draws it and keeps its rows; B^T likewise, all ranks hold it for the error
    # sample and the single-rank comparison handles)
    A_full = S.gen_matrix_torch(dist_name, M, K, 0, device=dev)
    A = A_full[lo:hi].clone()
    del A_full
    torch.cuda.empty_cache()
    Bt = S.gen_matrix_torch(dist_name, N, K, 1, device=dev)
    OmA = torch.from_numpy(S.gen_omega(K, kk, 1000)).to(dev)
    OmB = torch.from_numpy(S.gen_omega(K, kk, 1001)).to(dev)
    D = torch.empty((Mloc, N), device=dev)
    Cint = torch.empty((Mloc, N), dtype=torch.int32, device=dev)

    def handle(rank_=r, p_=p, q_=1, rounding="floor", gran="row", qt=0, multi=True):
        """A handle with this run's sharding (multi-rank: a fresh NCCL communicator), or a
        single-rank handle over this rank's rows and all of B (multi=False)."""
        if multi and ws > 1:
            uid = broadcast_unique_id(get_unique_id() if rank == 0 else None, ws, rank, dev)
            return Lrqmm(Mloc, N, K, bits, rank_, p_, q_, rounding, gran, world_size=ws, world_rank=rank,
                         unique_id=uid, device=local, stream=stream, b_sharded=bsh, qt_terms=qt)
        return Lrqmm(Mloc, N, K, bits, rank_, p_, q_, rounding, gran, device=local, stream=stream, qt_terms=qt)

    h = handle()
    Bt_mine = Bt[h.b_rows[0]:h.b_rows[1]]  # this rank's rows of B^T (all of them unless B is sharded)

    def step():
        h.quantize(SIDE_A, A)
        h.quantize(SIDE_B, Bt_mine)
        h.rsvd_residual(OmA, OmB)
        h.gemm(D)

    for _ in range(args.warmup):
        step()
    h.sync()
    torch.cuda.synchronize(dev)
    barrier(ws)

    # timed region: K steps, per-phase events on the launching stream
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # per-step working set (fp32 inputs, codes, residual planes, D); below 2x L2 every timed step is
    # preceded by a 256 MiB L2 flush (outside the per-step events, which then give the step time)
    nb_loc = h.b_rows[1] - h.b_rows[0]
    wset = 4 * (Mloc + nb_loc) * K + 3 * (Mloc + nb_loc) * K + 4 * Mloc * N
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if wset < (256 << 20) else None
    h.launch_count(reset=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        barrier(ws)
        e0.record(stream)
        for i in range(args.steps):
            ev = evs[i]
            if flush is not None:
                flush.fill_(float(i))
            ev[0].record(stream)
            h.quantize(SIDE_A, A)
            h.quantize(SIDE_B, Bt_mine)
            ev[1].record(stream)
            h.rsvd_residual(OmA, OmB)
            ev[2].record(stream)
            h.gemm(D)
            ev[3].record(stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier(ws)
    launches = h.launch_count()
    h.sync()
    t_step = e0.elapsed_time(e1) / 1e3 / args.steps
    ph = np.array([[ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])] for ev in evs]) / 1e3
    t_quant, t_rsvd, t_gemm = [float(x) for x in ph.mean(axis=0)]
    per_step = ph.sum(axis=1)  # event-to-event time of each timed step (s)
    step_stats = {"median_ms": float(np.median(per_step)) * 1e3, "min_ms": float(per_step.min()) * 1e3,
                  "max_ms": float(per_step.max()) * 1e3, "steps": int(per_step.size)}
    if flush is not None:
        t_step = float(per_step.mean())  # the flushes sit between the per-step events
    del flush
    t_step = max_over_ranks(t_step, ws, dev)

    def timed(fn, reps, warm=2):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize(dev)
        barrier(ws)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(reps):
            fn()
        b1.record(stream)
        torch.cuda.synchronize(dev)
        return max_over_ranks(b0.elapsed_time(b1) / 1e3 / reps, ws, dev)

    # bare int8 GEMM of this rank's shard (same tcgen05 kernel, int32 epilogue): the overhead
    # denominator (slowest rank)
    t_bare = timed(lambda: h.gemm_int32(Cint), args.steps)

    # direct-quant pipeline (quantize x2 + dequant GEMM, rank 0 correction off), same sharding
    hd = handle(0, 0)
    Bt_d = Bt[hd.b_rows[0]:hd.b_rows[1]]
    t_dq = timed(lambda: (hd.quantize(SIDE_A, A), hd.quantize(SIDE_B, Bt_d), hd.gemm(D)), args.steps)
    hd.close()

    # static-B (weight-resident): B quantized + RSVD'd once (sharded like the
    # full call), per call only the A side (quantize A, rsvd_residual(omega_a), gemm)
    h.quantize(SIDE_B, Bt_mine)
    h.rsvd_residual_b(OmB)
    t_static = timed(lambda: (h.quantize(SIDE_A, A), h.rsvd_residual(OmA), h.gemm(D)), args.steps, warm=3)

    # accuracy on a row sample of every rank (exact product in fp64), from a full call on all ranks
    step()
    h.sync()
    torch.cuda.synchronize(dev)
    rows = torch.arange(0, Mloc, max(1, Mloc // max(1, 256 // ws)), device=dev)[:max(1, 256 // ws)]
    Cex = A[rows].double() @ Bt.double().T
    nrm2 = float(torch.linalg.norm(Cex)) ** 2

    def sampled_err():
        e2, n2 = float(torch.linalg.norm(D[rows].double() - Cex)) ** 2, nrm2
        if ws > 1:
            t = torch.tensor([e2, n2], dtype=torch.float64, device=dev)
            import torch.distributed as dist

            dist.all_reduce(t)
            e2, n2 = float(t[0]), float(t[1])
        return (e2 / n2) ** 0.5

    errs = {"lrqmm": sampled_err()}
    q0_variant = None
    for name, rnd, gran, qt in (("dq_paper_trunc_tensor", "trunc", "tensor", 0), ("dq_nearest_row", "nearest", "row", 0),
                                ("dq_floor_row", "floor", "row", 0), ("qt110_trunc_tensor", "trunc", "tensor", 3),
                                ("qt111_trunc_tensor", "trunc", "tensor", 4)):
        # per-tensor scales and QT are single-rank configurations: rank-local handles over this rank's
        # rows and all of B (per-tensor: the rank's A shard max)
        with handle(0, 0, 1, rnd, gran, qt, multi=(gran == "row" and qt == 0)) as hq:
            Bq = Bt[hq.b_rows[0]:hq.b_rows[1]]
            hq.quantize(SIDE_A, A); hq.quantize(SIDE_B, Bq); hq.gemm(D); hq.sync()
        errs[name] = sampled_err()
    # labelled variant (reading #30): q = 0 with a structured sketch (first column all
    # ones): two passes over R plus a codes-only pass instead of q = 1's three R passes
    if r > 0:
        OmA1, OmB1 = OmA.clone(), OmB.clone()
        OmA1[:, 0] = 1.0
        OmB1[:, 0] = 1.0
        with handle(r, p, 0) as h0:
            B0 = Bt[h0.b_rows[0]:h0.b_rows[1]]
            t_q0 = timed(lambda: (h0.quantize(SIDE_A, A), h0.quantize(SIDE_B, B0), h0.rsvd_residual(OmA1, OmB1),
                                  h0.gemm(D)), args.steps, warm=3)
            h0.sync()
            errs["lrqmm_q0_ones_sketch"] = sampled_err()
            q0_variant = {"ms_per_step": t_q0 * 1e3, "value": 2.0 * M * N * K / t_q0 / 1e12, "unit": "TOPS",
                          "note": "power_iters=0 + Omega[:,0]=1 (SURVEY f4 / E3 (c), reading #30): labelled variant, "
                                  "not the paper's q; error in rel_fro_error.lrqmm_q0_ones_sketch"}
    del Cex

    # end to end through the C ABI with pinned HOST buffers: every rank runs lrqmm_run_host_async on
    # its own shard (H2D of A rows, B^T rows, Omega; full hot path; D2H of D rows); max over ranks
    e2e = None
    if not args.no_e2e:
        hA = torch.empty((Mloc, K), dtype=torch.float32, pin_memory=True)
        hB = torch.empty((Bt_mine.shape[0], K), dtype=torch.float32, pin_memory=True)
        hOa = torch.empty((K, kk), dtype=torch.float32, pin_memory=True)
        hOb = torch.empty((K, kk), dtype=torch.float32, pin_memory=True)
        hD = torch.empty((Mloc, N), dtype=torch.float32, pin_memory=True)
        hA.copy_(A); hB.copy_(Bt_mine); hOa.copy_(OmA); hOb.copy_(OmB)
        npA, npB, npOa, npOb, npD = hA.numpy(), hB.numpy(), hOa.numpy(), hOb.numpy(), hD.numpy()
        h.run_host(npA, npB, npOa, npOb, npD)
        barrier(ws)
        t0 = time.perf_counter()
        # a stream of calls: each step's H2D of A, B^T, Omega and D2H of D happen inside the timed
        # region; lrqmm_run_host_async overlaps step i's D2H with step i+1's H2D (full-duplex PCIe)
        for _ in range(args.e2e_steps):
            h.run_host_async(npA, npB, npOa, npOb, npD)
        h.sync()
        t_e2e = (time.perf_counter() - t0) / args.e2e_steps
        t_e2e = max_over_ranks(t_e2e, ws, dev)
        h2d = 4 * (Mloc * K + Bt_mine.shape[0] * K + 2 * K * kk)
        d2h = 4 * Mloc * N
        del hA, hB, hD
        ctx = pcie_context(dev, h2d, d2h)
        e2e = {"value": 2.0 * M * N * K / t_e2e / 1e12, "unit": "TOPS", "h2d_bytes_per_step": h2d * ws,
               "d2h_bytes_per_step": d2h * ws, "ms_per_step": t_e2e * 1e3,
               "pcie": ctx,
               "pcie_bound_ms": (h2d / ctx["h2d_gbs"] / 1e6) if ctx.get("h2d_gbs") else None,
               "note": "lrqmm_run_host_async (a stream of calls, synced at the end): pinned host A, B^T, Omega -> "
                       "device, full hot path, D -> host every step; host wall clock, max over ranks; "
                       "pcie = this box's measured pinned copy rates and NUMA placement (the e2e bound)"}

    h.close()
    if rank != 0:
        if ws > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    ops = 2.0 * M * N * K
    peaks, peak_src = load_peaks()
    # int8 dense = 2 x the measured bf16 BURST figure (guide nominal ratio 4.5 / 2.25).  The GEMM runs
    # inside a long step, but the bf16 "sustained" figure is a power-capped clock (~1.24 GHz) that
    # the int8 kernel does not hit (it holds ~1.77 GHz), so it is not a ceiling for it; the burst
    # figure is the larger, conservative denominator.
    int8_peak = 2.0 * float(peaks["bf16_tflops"])
    gemm_tops = 2.0 * Mloc * N * K / t_gemm / 1e12
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "gemm_ncu_summary.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if pj.get("config") == args.config and ws == 1:
                traffic = pj.get("dram_bytes_per_launch")
                traffic_src = (f"profiles/gemm_ncu_summary.json: one ncu --set full capture of this kernel at this "
                               f"config ({pj.get('captured', 'round 1')}), not measured in this run")
        except Exception:
            traffic = None

    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        phases = {}
        dt, sops = oracle_sample(cfg, phases=phases)
        cpu = {"value": sops / dt / 1e12, "unit": "TOPS", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"NumPy fp64 oracle on the first {REF_ROWS} rows of A x full B^T ({N}x{K}), "
                         f"incl. full quantize + RSVD of B; {dt:.1f} s",
               "phases_s": {k: round(v, 4) for k, v in phases.items()}}

    nb = h.b_rows[1] - h.b_rows[0]
    line = {
        "metric": METRIC,
        "value": ops / t_step / 1e12,
        "unit": "TOPS",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int8",
        "data": "synthetic",
        "config": {"workload": label, "M": M, "M_per_gpu": Mloc, "N": N, "K": K, "bits": bits, "rank": r,
                   "oversample": p, "power_iters": 1, "rounding": "floor", "scales": "per-row A / per-col B",
                   "l2": (f"per-step working set {wset / 2**20:.0f} MiB/GPU (fp32 inputs, codes, residual planes, D) "
                          + ("> 2x the 126 MB L2: no flush" if wset >= (256 << 20) else
                             "< 2x L2: a 256 MiB L2 flush before every timed step, outside its events")),
                   "parallelism": (f"row-shard A x{ws}, B column-sharded x{ws} (allgather)" if bsh else
                                   f"row-shard A x{ws}, B replicated") if ws > 1 else "single GPU"},
        "overhead_vs_bare_int8": t_step / t_bare,
        "overhead_vs_direct_quant": t_step / t_dq,
        "step_stats": step_stats,
        "ms": {"bare_int8_gemm": t_bare * 1e3, "direct_quant_pipeline": t_dq * 1e3, "quantize_AB": t_quant * 1e3,
               "rsvd_residual": t_rsvd * 1e3, "gemm_fused_epilogue": t_gemm * 1e3},
        "bare_int8_tops": ops / t_bare / 1e12,
        "variant_q0_ones_sketch": q0_variant,
        "static_b": {
            "ms_per_step": t_static * 1e3, "value": ops / t_static / 1e12, "unit": "TOPS",
            "overhead_vs_bare_int8": t_static / t_bare,
            "note": "weight-resident B (lrqmm_rsvd_residual_b once); per call: quantize A, rsvd_residual(omega_a), gemm"},
        "rel_fro_error": errs,
        "rel_fro_error_note": (f"{len(rows)} sampled rows per rank vs the fp64 product of the fp32 inputs" +
                               ("; dq_paper_trunc_tensor / qt* use rank-local single-GPU handles" if ws > 1 else "")),
        "roofline": {"bound": "tensor",
                     "kernel": ("k7_gemm_i8_2sm (CTA-pair tcgen05.mma.cta_group::2 kind::i8 + fused LRQMM epilogue)"
                                if Mloc >= 512 and N >= 512 and ((Mloc + 255) // 256) * ((N + 255) // 256) >= 512
                                and (r == 0 or K > 2048)
                                else ("k8_gemm_tc (tcgen05 kind::i8 + the rank-2r correction as bf16 hi/lo "
                                      "kind::f16 MMAs into a second TMEM accumulator)" if r > 0 else
                                      "k6_gemm_i8 (tcgen05 kind::i8 + dequantising epilogue)")),  # gemm_i8.cu rules
                     "achieved": gemm_tops, "peak": int8_peak, "unit": "TFLOP/s", "frac": gemm_tops / int8_peak,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_note": f"int8 dense = 2 x {peak_src} bf16 burst ({peaks['bf16_tflops']} TFLOP/s; guide nominal "
                                  "ratio 4.5/2.25); the bf16 sustained figure is power-capped below this "
                                  "kernel's clock"},
        "hbm_roofline": {
            "peak_gbs": hbm_peak(), "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy)",
            "quantize_AB": {"bytes": hbm_bytes_quantize(Mloc, K, r > 0) + hbm_bytes_quantize(nb, K, r > 0),
                            "gbs": (hbm_bytes_quantize(Mloc, K, r > 0) + hbm_bytes_quantize(nb, K, r > 0)) / t_quant / 1e9},
            "rsvd_residual": {"bytes": hbm_bytes_rsvd(Mloc, K) + hbm_bytes_rsvd(nb, K),
                              "gbs": (hbm_bytes_rsvd(Mloc, K) + hbm_bytes_rsvd(nb, K)) / t_rsvd / 1e9},
        },
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    for ph_ in ("quantize_AB", "rsvd_residual"):
        line["hbm_roofline"][ph_]["frac"] = line["hbm_roofline"][ph_]["gbs"] / line["hbm_roofline"]["peak_gbs"]
    if cpu:
        line["cpu_baseline"] = cpu
    if e2e:
        line["e2e"] = e2e
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
