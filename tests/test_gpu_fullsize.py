"""Parity at BASELINE.json's full bench size (configs[2]: 16384^3 int4, r = 16, p = 5, q = 1), in the
launch configuration bench.py times (same library calls, same automatic kernel choices).

The oracle cannot form the full 16384^3 fp64 product in seconds, so the check is on sampled
outputs the oracle computes one by one:
  * lambda for every row of A and B^T: bit-exact;
  * codes of 64 sampled rows of A and of B^T: bit-exact;
  * int32 accumulators on a 64 x 512 sample of C_int: bit-exact;
  * D on 64 sampled rows (all 16384 columns): the oracle's Algorithm 2 evaluated for those rows
    (C_F rows + RC1 + RC2 + RC3 rows) with the RSVD factors of the FULL
    residuals (oracle.rsvd, variant (b), same Omega) — rel. Frobenius <= 1e-4 and error vs the
    exact fp64 product rows <= 1.05x the oracle's;
  * EVERY row and column of C_int: its exact int64 sum against the oracle's codes (A_int (B_int^T 1)
    and B_int (A_int^T 1)), and every row and column sum of D against the oracle's Algorithm 2
    summed term by term (C_F, RC1, RC2, RC3 applied to a ones vector), within the row-wise form of
    the north_star bar: |1^T (D_gpu - D_or)_i| <= sqrt(N) |(D_gpu - D_or)_i| <= 1e-4 sqrt(N) |D_i|
    (the correction's rounding error is low-rank, hence coherent along a row: ~1e-3 of a row sum,
    measured).  A dropped or misplaced 256 x 256 tile changes each of its rows' sums by ~sqrt(256)
    entries' magnitude, ~10x that tolerance.
Takes ~1-2 minutes (fp64 RSVD of two 16384^2 residuals on the host).
"""
import numpy as np
import pytest

import oracle as O
import synth as S

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm  # noqa: E402

DEV = "cuda:0"


def _oracle_rows(A, Bt, bits, r, q, OmA, OmB, rows):
    """Algorithm 2 (oracle.lrqmm, literal) restricted to output rows `rows`, full-size factors."""
    ca, la = O.quantize(A, bits)
    cb, lb = O.quantize(Bt, bits)
    Af = O.dequantize(ca, la)
    RA = A.astype(np.float64) - Af
    USa, Va = O.rsvd(RA, OmA, r, q)
    del RA
    Btf = O.dequantize(cb, lb)
    RBt = Bt.astype(np.float64) - Btf
    USb, Vb = O.rsvd(RBt, OmB, r, q)
    del RBt
    c_rows = O.int_gemm(ca[rows], cb)
    CF = O.dequant_result(c_rows, la[rows], lb)
    Bf = Btf.T
    Ut, Wr, Zt = USa[rows], Vb, USb.T
    RC1 = Ut @ (Va.T @ Bf)
    RC2 = (Af[rows] @ Wr) @ Zt
    RC3 = (Ut @ (Va.T @ Wr)) @ Zt
    # full row / column sums: C_int exactly in int64, D's four terms of Alg. 2 times a ones vector
    sa, sb = ca.sum(axis=0), cb.sum(axis=0)
    c_rowsum, c_colsum = ca @ sb, cb @ sa
    la64, lb64 = la.astype(np.float64), lb.astype(np.float64)
    ua, ub = USa.sum(axis=0), USb.sum(axis=0)
    VaVb = Va.T @ Vb
    afs = Af.sum(axis=0)
    d_rowsum = ((ca @ (cb / lb64[:, None]).sum(axis=0)) / la64 + USa @ (Va.T @ Btf.sum(axis=0))
                + Af @ (Vb @ ub) + USa @ (VaVb @ ub))
    d_colsum = ((cb @ (ca / la64[:, None]).sum(axis=0)) / lb64 + Btf @ (Va @ ua)
                + USb @ (Vb.T @ afs) + USb @ (VaVb.T @ ua))
    return dict(D=CF + RC1 + RC2 + RC3, ca=ca, la=la, cb=cb, lb=lb, c_rows=c_rows, c_rowsum=c_rowsum,
                c_colsum=c_colsum, d_rowsum=d_rowsum, d_colsum=d_colsum)


def test_fullsize_c3_sampled():
    M = N = K = 16384
    bits, r, p, q = 4, 16, 5, 1
    A = S.gen_matrix("normal", M, K, 2 * 11)
    Bt = S.gen_matrix("normal", N, K, 2 * 11 + 1)
    OmA = S.gen_omega(K, r + p, 1000 + 2 * 11)
    OmB = S.gen_omega(K, r + p, 1001 + 2 * 11)
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(M, 64, replace=False))
    cols = np.sort(rng.choice(N, 512, replace=False))
    brows = np.sort(rng.choice(N, 64, replace=False))

    with Lrqmm(M, N, K, bits, r, p, q) as h:
        a = torch.from_numpy(A).to(DEV)
        b = torch.from_numpy(Bt).to(DEV)
        h.quantize(SIDE_A, a)
        h.quantize(SIDE_B, b)
        h.rsvd_residual(torch.from_numpy(OmA).to(DEV), torch.from_numpy(OmB).to(DEV))
        D = torch.empty((M, N), device=DEV)
        h.gemm(D)
        h.sync()
        d_rows = D[torch.from_numpy(rows).to(DEV)].double().cpu().numpy()
        d_rowsum = D.double().sum(dim=1).cpu().numpy()
        d_colsum = D.double().sum(dim=0).cpu().numpy()
        d_rownrm = torch.linalg.norm(D.double(), dim=1).cpu().numpy()
        d_colnrm = torch.linalg.norm(D.double(), dim=0).cpu().numpy()
        del D
        ga = h.codes(SIDE_A)
        gb = h.codes(SIDE_B)
        codes_a = ga[torch.from_numpy(rows).to(DEV)].cpu().numpy().astype(np.int64)
        codes_b = gb[torch.from_numpy(brows).to(DEV)].cpu().numpy().astype(np.int64)
        lam_a = h.scales(SIDE_A).cpu().numpy()
        lam_b = h.scales(SIDE_B).cpu().numpy()
        C = torch.empty((M, N), dtype=torch.int32, device=DEV)
        h.gemm_int32(C)
        h.sync()
        c_s = C[torch.from_numpy(rows).to(DEV)][:, torch.from_numpy(cols).to(DEV)].cpu().numpy().astype(np.int64)
        c_rowsum = C.sum(dim=1, dtype=torch.int64).cpu().numpy()
        c_colsum = C.sum(dim=0, dtype=torch.int64).cpu().numpy()
        del C, a, b

    ref = _oracle_rows(A, Bt, bits, r, q, OmA, OmB, rows)
    assert np.array_equal(lam_a.view(np.uint32), ref["la"].view(np.uint32))
    assert np.array_equal(lam_b.view(np.uint32), ref["lb"].view(np.uint32))
    assert np.array_equal(codes_a, ref["ca"][rows])
    assert np.array_equal(codes_b, ref["cb"][brows])
    assert np.array_equal(c_s, ref["c_rows"][:, cols])
    C_exact = A[rows].astype(np.float64) @ Bt.astype(np.float64).T
    diff = O.relative_error(ref["D"], d_rows)
    e_gpu, e_or = O.relative_error(C_exact, d_rows), O.relative_error(C_exact, ref["D"])
    assert diff <= 1e-4, (diff, e_gpu, e_or)
    assert e_gpu <= 1.05 * e_or, (e_gpu, e_or)
    # every row / column: exact integer sums, and D sums within 1e-4 of their scale
    assert np.array_equal(c_rowsum, ref["c_rowsum"])
    assert np.array_equal(c_colsum, ref["c_colsum"])
    for got, want, nrm, n in ((d_rowsum, ref["d_rowsum"], d_rownrm, N), (d_colsum, ref["d_colsum"], d_colnrm, M)):
        tol = 1e-4 * np.sqrt(n) * nrm
        assert np.all(np.abs(got - want) <= tol), (np.max(np.abs(got - want) / tol))
