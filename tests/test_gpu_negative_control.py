"""GPU negative controls (SPEC.md:584's negative-control idea, VERDICT r01 evidence hygiene): each
deliberate defect injected into the product path (lrqmm_debug_inject_fault) must make the parity
checks fail, and the same checks must pass again once it is removed -- the parity tests have teeth
on the GPU, not only on the oracle's pins."""

import numpy as np
import pytest

import oracle as O
import synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402
from paper_2409_18772_b200.lrqmm import load_library  # noqa: E402

DEV = "cuda:0"
M, N, K, R, P = 384, 320, 512, 8, 5


def parity_failures(A, Bt, OmA, OmB, ref, parts):
    """The parity bars of tests/test_gpu_parity.py; returns the list of the ones that fail."""
    with Lrqmm(M, N, K, 4, R, P) as h:
        h.quantize(SIDE_A, torch.from_numpy(A).to(DEV))
        h.quantize(SIDE_B, torch.from_numpy(Bt).to(DEV))
        h.rsvd_residual(torch.from_numpy(OmA[:, :R + P]).to(DEV), torch.from_numpy(OmB[:, :R + P]).to(DEV))
        D = torch.empty((M, N), device=DEV)
        h.gemm(D)
        h.sync()
        Dg = D.cpu().numpy().astype(np.float64)
        codes = h.codes(SIDE_A).cpu().numpy().astype(np.int64)
        lam = h.scales(SIDE_A).cpu().numpy()
    bad = []
    if not np.array_equal(codes, parts["codes_a"]):
        bad.append("codes")
    if not np.array_equal(lam.view(np.uint32), parts["lam_a"].view(np.uint32)):
        bad.append("lambda bits")
    C = O.matmul_exact(A, Bt)
    if O.relative_error(ref, Dg) > 1e-4:
        bad.append("D vs oracle")
    if O.relative_error(C, Dg) > 1.05 * O.relative_error(C, ref):
        bad.append("error ratio")
    return bad


@pytest.mark.parametrize("fault,expect", [(1, "codes"), (2, "lambda bits"), (3, "D vs oracle"), (4, "D vs oracle")])
def test_injected_fault_fails_parity(fault, expect):
    lib = load_library()
    A, Bt, OmA, OmB = S.problem(M, N, K, R + P, s=12, dist="u01")
    ref, parts = O.lrqmm(A, Bt, 4, R, OmA[:, :R + P], OmB[:, :R + P], q=1, return_parts=True)
    assert parity_failures(A, Bt, OmA, OmB, ref, parts) == []
    assert lib.lrqmm_debug_inject_fault(fault) == 0
    try:
        bad = parity_failures(A, Bt, OmA, OmB, ref, parts)
    finally:
        assert lib.lrqmm_debug_inject_fault(0) == 0
    assert expect in bad, (fault, bad)
    assert parity_failures(A, Bt, OmA, OmB, ref, parts) == []
    assert lib.lrqmm_debug_inject_fault(9) != 0
