"""Pins of the fp64 oracle against what the paper and mathematics fix.

None of these re-type the oracle's formula: they use exact rational
arithmetic (fractions.Fraction), Python-int loops, closed forms, algebraic
identities (Eq. gemm_r_split), constructed exact-rank fixtures and the values
printed in the paper (tests/golden/paper_tables_2_3.txt).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synth as S


# ----------------------------------------------------------------- helpers
def frac_round(fr: Fraction, mode: str) -> int:
    if mode == "floor":
        return fr.numerator // fr.denominator
    if mode == "trunc":
        return int(fr)  # int() of a Fraction truncates toward zero
    if mode == "nearest":
        return round(fr)  # Python rounds Fraction half-to-even
    raise ValueError(mode)


def exact_lambda_is_nearest(lam32: np.float32, qmax: int, amax32: np.float32) -> bool:
    """lam32 is the fp32 nearest to qmax/amax (exact rationals)."""
    target = Fraction(qmax) / Fraction(float(amax32))
    lo = np.nextafter(lam32, np.float32(0))
    hi = np.nextafter(lam32, np.float32(np.inf))
    d = abs(Fraction(float(lam32)) - target)
    return d <= abs(Fraction(float(lo)) - target) and d <= abs(Fraction(float(hi)) - target)


def frac_matmul(A, B):
    n, k = len(A), len(A[0])
    m = len(B[0])
    return [[sum((A[i][t] * B[t][j] for t in range(k)), Fraction(0)) for j in range(m)] for i in range(n)]


def frac_T(A):
    return [list(r) for r in zip(*A)]


def frac_inv(M):
    n = len(M)
    A = [list(r) + [Fraction(int(i == j)) for j in range(n)] for i, r in enumerate(M)]
    for c in range(n):
        p = next(r for r in range(c, n) if A[r][c] != 0)
        A[c], A[p] = A[p], A[c]
        pv = A[c][c]
        A[c] = [x / pv for x in A[c]]
        for r in range(n):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [x - f * y for x, y in zip(A[r], A[c])]
    return [r[n:] for r in A]


def to_frac(X):
    return [[Fraction(float(v)) for v in row] for row in np.asarray(X)]


# ------------------------------------------------- Eq. quantA: the scale
def test_compute_scale_spec_examples():
    # SPEC.md:141-143
    assert O.compute_scale(7.0, 4) == np.float32(1.0)
    assert O.compute_scale(127.0, 8) == np.float32(1.0)
    assert O.compute_scale(0.5, 4) == np.float32(14.0)
    # reading #6: zero row -> lambda = 1
    assert O.compute_scale(0.0, 4) == np.float32(1.0)


@pytest.mark.parametrize("bits", [4, 8])
def test_compute_scale_is_correctly_rounded_fp32(bits):
    rng = np.random.default_rng(11)
    amax = (10.0 ** rng.uniform(-20, 20, 3000)).astype(np.float32)
    lam = O.compute_scale(amax, bits)
    for a, l in zip(amax, lam):
        assert exact_lambda_is_nearest(l, O.qmax_of(bits), a)


# ------------------------------------------- quantize: exact rationals
@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("mode", ["floor", "trunc", "nearest"])
def test_quantize_matches_exact_rational_rounding(bits, mode):
    rng = np.random.default_rng(3 + bits)
    X = rng.standard_normal((6, 200)).astype(np.float32)
    # adversarial cells: exact lattice points, their fp32 neighbours, -0.0, +-amax
    lam_guess = O.compute_scale(np.max(np.abs(X), axis=1), bits)
    for i in range(6):
        c = rng.integers(-O.qmax_of(bits), O.qmax_of(bits) + 1, 20)
        lat = (c / lam_guess[i]).astype(np.float32)
        X[i, :20] = lat
        X[i, 20:40] = np.nextafter(lat, np.float32(np.inf))
        X[i, 40:60] = np.nextafter(lat, np.float32(-np.inf))
        X[i, 60] = -0.0
        # -amax appears: floor can push -qmax-1, which must be clamped (reading #5)
        X[i, 61] = -np.max(np.abs(X[i]))
    X[5] = 0.0  # zero row
    codes, lam = O.quantize(X, bits, mode, "row")
    q = O.qmax_of(bits)
    for i in range(X.shape[0]):
        amax = np.float32(np.max(np.abs(X[i])))
        if amax == 0:
            assert lam[i] == 1.0
        else:
            assert exact_lambda_is_nearest(lam[i], q, amax)
        fl = Fraction(float(lam[i]))
        for j in range(X.shape[1]):
            want = max(-q, min(q, frac_round(fl * Fraction(float(X[i, j])), mode)))
            assert codes[i, j] == want, (i, j, X[i, j])


def test_quantize_spec_examples():
    # lambda = 1, a = 3.7 -> floor 3, nearest 4 (row amax 7, N=4 -> lambda 1)
    X = np.array([[3.7, 7.0]], dtype=np.float32)
    c, l = O.quantize(X, 4, "floor")
    assert l[0] == 1.0 and c[0, 0] == 3
    c, l = O.quantize(X, 4, "nearest")
    assert c[0, 0] == 4
    # residual of 3.7 under floor is 0.7 (fp32 3.7 - 3)
    c, l = O.quantize(X, 4, "floor")
    assert abs(O.residual(X, c, l)[0, 0] - 0.7) < 1e-6
    # diag(7, -7), N=4, floor -> diag(7, -7), lambda = 1 (per tensor)
    D = np.diag([7.0, -7.0]).astype(np.float32)
    c, l = O.quantize(D, 4, "floor", "tensor")
    assert np.array_equal(c, np.diag([7, -7])) and np.all(l == 1.0)
    # dequantize lambda=2, v=5 -> 2.5
    assert O.dequantize(np.array([[5]]), np.array([2.0], np.float32))[0, 0] == 2.5


@pytest.mark.parametrize("bits", [4, 8])
def test_floor_residual_range_and_quantEA_bound(bits):
    # Eq. get_ra2: floor residual is non-negative, < 1/lambda
    # away from clamp cells; Eq. quantEA per-row form (reading #20):
    # ||R||_F <= sqrt(sum_i K / lambda_i^2).
    for dist in ("normal", "u01", "exp4"):
        X = S.gen_matrix(dist, 64, 300, 5)
        c, l = O.quantize(X, bits, "floor")
        R = O.residual(X, c, l)
        q = O.qmax_of(bits)
        inner = np.abs(c) < q
        inv = 1.0 / l.astype(np.float64)[:, None]
        assert np.all(R[inner] >= 0) and np.all((R < inv + 1e-12)[inner])
        assert np.linalg.norm(R) <= np.sqrt(np.sum(300 / l.astype(np.float64) ** 2))


# ----------------------------------------- Eq. INTGEMM / QUANTGEMM
def test_int_gemm_exact_and_spec():
    assert O.int_gemm(np.array([[7]]), np.array([[7]]))[0, 0] == 49
    rng = np.random.default_rng(2)
    a = rng.integers(-127, 128, (7, 33))
    b = rng.integers(-127, 128, (5, 33))
    got = O.int_gemm(a, b)
    for i in range(7):
        for j in range(5):
            assert got[i, j] == sum(int(a[i, t]) * int(b[j, t]) for t in range(33))
    # big-K exactness: int8 extremes at K = 8192 (sum ~ 1.3e8, beyond fp32 but exact in fp64)
    a = np.full((2, 8192), -127)
    b = np.full((2, 8192), 127)
    assert O.int_gemm(a, b)[0, 0] == -127 * 127 * 8192


def test_dequant_result_spec():
    # C_int = 10, lambda_a = 2, lambda_b = 5 -> 1.0
    out = O.dequant_result(np.array([[10]]), np.array([2.0], np.float32), np.array([5.0], np.float32))
    assert out[0, 0] == 1.0


# ------------------------------------------------------------- RSVD
def test_orth_threshold_and_degenerate():
    assert O.orth(np.zeros((5, 3))).shape == (5, 0)
    u = np.arange(1.0, 6.0)[:, None]
    M = np.hstack([u, 2 * u, np.ones((5, 1))])  # rank 2
    Q = O.orth(M)
    assert Q.shape == (5, 2)
    assert np.allclose(Q.T @ Q, np.eye(2), atol=1e-12)
    assert np.allclose(Q @ (Q.T @ M), M, atol=1e-12)


def _hadamard(n):
    H = np.array([[1.0]])
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H / np.sqrt(n)  # orthogonal to fp64 rounding


@pytest.mark.parametrize("scale", [1e-12, 1.0, 1e6])
def test_orth_threshold_is_relative_to_sigma_max(scale):
    """Reading #12 ("orthogonal columns"): orth drops a direction
    iff sigma < 1e-5 * sigma_max -- a RELATIVE threshold.  M = U diag(s) V^T is built with known
    singular values from exact orthogonal (Hadamard) factors, so what must be kept is known in
    closed form: a 1e-12-scaled full-rank matrix keeps every direction (an absolute threshold would
    drop them all), sigma ratios 1e-4 / 1e-6 keep / drop the small direction at every scale (an
    absolute threshold would flip one of them at 1e-12 or 1e6)."""
    U = _hadamard(8)[:, :4]
    V = _hadamard(4)
    for sig, keep in (([1.0, 0.5, 0.25, 0.125], 4),        # full rank at any scale
                      ([1.0, 0.5, 1e-4, 1e-4], 4),          # ratio 1e-4 >= 1e-5: kept
                      ([1.0, 0.5, 1e-6, 1e-6], 2),          # ratio 1e-6 < 1e-5: dropped
                      ([1.0, 2e-5, 5e-6, 0.0], 2)):         # straddling the threshold
        s = np.array(sig) * scale
        M = (U * s) @ V.T
        Q = O.orth(M)
        assert Q.shape == (8, keep), (sig, scale, Q.shape)
        assert np.allclose(Q.T @ Q, np.eye(keep), atol=1e-12)
        # span(Q) is exactly the span of the kept left singular vectors
        Uk = U[:, :keep]
        assert np.allclose(Q @ (Q.T @ Uk), Uk, atol=1e-10)


def test_rsvd_spec_examples():
    rng = np.random.default_rng(0)
    # I_5, r = 5, p = 0 -> full capture
    US, V = O.rsvd(np.eye(5), rng.standard_normal((5, 5)), 5, 1)
    assert np.linalg.norm(US @ V.T - np.eye(5)) <= 1e-10
    # rank-1 u v^T, r = 1
    u, v = rng.random(9), rng.random(7)
    R = np.outer(u, v)
    US, V = O.rsvd(R, rng.standard_normal((7, 1)), 1, 1)
    assert np.linalg.norm(US @ V.T - R) <= 1e-10 * np.linalg.norm(R)
    # diag(3,2,1) -> singular values [3,2,1]
    US, V = O.rsvd(np.diag([3.0, 2.0, 1.0]), rng.standard_normal((3, 3)), 3, 1)
    assert np.allclose(np.sort(np.linalg.norm(US, axis=0))[::-1], [3, 2, 1], atol=1e-12)
    assert np.allclose(V.T @ V, np.eye(3), atol=1e-12)


def test_rsvd_truncation_is_eckart_young_of_projection():
    # k > r: USigma V^T must be the best rank-r approximation (Eq. k-svd,
    # PAPER.md:106-114) of the rank-k projection R Q1 Q1^T; checked against an
    # SVD of the dense rows x K matrix (a different computation from the
    # oracle's k x k eigendecomposition).
    R = O.residual(*((lambda X: (X,) + O.quantize(X, 4))(S.gen_matrix("u01", 60, 50, 1))))
    Om = np.random.default_rng(4).standard_normal((50, 9))
    US, V = O.rsvd(R, Om, 4, 1)
    _, Q1full = O.rsvd(R, Om, 9, 1)  # width 9 <= r=9: no truncation -> Q1
    P = R @ Q1full @ Q1full.T
    U, s, Vt = np.linalg.svd(P)
    best = (U[:, :4] * s[:4]) @ Vt[:4]
    assert np.linalg.norm(US @ V.T - best) <= 1e-10 * np.linalg.norm(best)
    # and the tail error of the randomized one is never below the optimal SVD tail
    sR = np.linalg.svd(R, compute_uv=False)
    assert np.linalg.norm(R - US @ V.T) >= np.sqrt(np.sum(sR[4:] ** 2)) * (1 - 1e-12)


def test_rsvd_projection_error_monotone_in_nested_rank():
    # nested Omega columns -> nested span(Q1) (variant (b), p = 0) -> the
    # projection error ||R - R_k||_F is non-increasing in k (Fig. 3(a) claim,
    # PAPER.md:692, as a theorem for the residual approximation).
    X = S.gen_matrix("u01", 128, 96, 7)
    R = O.residual(X, *O.quantize(X, 4))
    Om = S.gen_omega(96, 40, 9).astype(np.float64)
    errs = []
    for k in (1, 2, 4, 8, 16, 32, 40):
        US, V = O.rsvd(R, Om[:, :k], k, 1)
        errs.append(np.linalg.norm(R - US @ V.T))
    assert all(b <= a * (1 + 1e-12) for a, b in zip(errs, errs[1:]))


def test_rsvd_error_envelope_eq_rsvderror():
    # Eq. rsvderror, statistical: mean over 20 seeds of the
    # spectral error <= [1 + 4 sqrt(2 min(m,n)/(r-1))]^(1/(2q+1)) sigma_{r+1}.
    X = S.gen_matrix("exp4", 80, 70, 2)
    R = O.residual(X, *O.quantize(X, 4))
    r, q = 6, 1
    s = np.linalg.svd(R, compute_uv=False)
    bound = (1 + 4 * np.sqrt(2 * 70 / (r - 1))) ** (1 / (2 * q + 1)) * s[r]
    errs = []
    for seed in range(20):
        Om = np.random.default_rng(100 + seed).standard_normal((70, r))
        US, V = O.rsvd(R, Om, r, q)
        errs.append(np.linalg.norm(R - US @ V.T, 2))
    assert np.mean(errs) <= bound


# ---------------------------------------------------- Algorithm 2 pins
def test_zero_residual_inputs_give_exact_product():
    # inputs already on the quantization lattice with a representable lambda:
    # R = 0, the correction vanishes (RSVD of 0 is empty) and D = A B exactly.
    rng = np.random.default_rng(8)
    for bits in (4, 8):
        q = O.qmax_of(bits)
        ca = rng.integers(-q, q + 1, (24, 40))
        cb = rng.integers(-q, q + 1, (18, 40))
        ca[:, 0] = q
        cb[:, 0] = -q
        A = (ca / 4.0).astype(np.float32)      # lambda_A = q / (q/4) = 4
        Bt = (cb / 0.5).astype(np.float32)     # lambda_B = 0.5
        Om = rng.standard_normal((40, 8)).astype(np.float32)
        D = O.lrqmm(A, Bt, bits, 5, Om, Om, q=1)
        assert np.max(np.abs(D - O.matmul_exact(A, Bt))) == 0.0


def test_full_rank_recovers_exact_product_eq_gemm_r_split():
    # k = K, p = 0: the RSVD keeps all of R, and Eq. gemm_r_split's identity
    # T1 + A~ R_B + R_A B~ + R_A R_B = A B.
    for bits in (4, 8):
        for (M, N, K) in ((12, 9, 10), (30, 41, 25)):
            A, Bt, OmA, OmB = S.problem(M, N, K, K, s=3)
            D = O.lrqmm(A, Bt, bits, K, OmA, OmB, q=1)
            C = O.matmul_exact(A, Bt)
            assert O.relative_error(C, D) <= 1e-12


def _rank1_fixture(rows, K, bits, e, rng):
    """Reading #25: lambda = 2^e exactly, one column at -qmax/lambda (v = 0
    there), other codes in [-qmax+1, qmax-1], R = u v^T / lambda exactly with
    dyadic u, v (exactly representable in fp32)."""
    q = O.qmax_of(bits)
    lam = 2.0 ** e
    codes = rng.integers(-q + 1, q, (rows, K))
    codes[:, 0] = -q
    u = rng.integers(0, 16, rows) / 16.0
    v = rng.integers(0, 16, K) / 16.0
    v[0] = 0.0
    X = ((codes + np.outer(u, v)) / lam).astype(np.float32)
    assert np.array_equal(X.astype(np.float64), (codes + np.outer(u, v)) / lam)
    return X, codes, lam


@pytest.mark.parametrize("bits", [4, 8])
def test_exact_rank1_residual_fixture(bits):
    rng = np.random.default_rng(21)
    A, ca, la = _rank1_fixture(40, 32, bits, 3, rng)
    Bt, cb, lb = _rank1_fixture(28, 32, bits, -2, rng)
    D, parts = O.lrqmm(A, Bt, bits, 1, rng.standard_normal((32, 1)), rng.standard_normal((32, 1)),
                       q=1, return_parts=True)
    assert np.array_equal(parts["codes_a"], ca) and np.all(parts["lam_a"] == la)
    assert np.array_equal(parts["codes_b"], cb) and np.all(parts["lam_b"] == lb)
    C = O.matmul_exact(A, Bt)
    assert O.relative_error(C, D) <= 1e-12
    # and with r = 0 (direct quant, floor) the error is O(1/lambda): clearly nonzero
    assert O.relative_error(C, O.lrqmm(A, Bt, bits, 0)) > 1e-6


def _exact_lrqmm_projector_form(A, Bt, bits, OmA, OmB, power_steps=1):
    """Exact rational evaluation of the same definitions (p = 0, q power steps), with
    the projector P = Z (Z^T Z)^-1 Z^T, Z = (R^T R)^q Omega, in place of the
    oracle's SVD-based orthonormalisation:  R_k = R P,
    D = C_F + R_A,k B~ + A~ R_B,k + R_A,k R_B,k.
    Variant (b) with q power steps (reading #11; q of Eq. rsvderror) spans
    span(Q1) = span(R^T orth(R ... R^T orth(R Omega))) = span((R^T R)^q Omega) for full-rank sketches."""
    q = O.qmax_of(bits)

    def side(X, Om):
        Xf = to_frac(X)
        rows = []
        lams = []
        for row in np.asarray(X, np.float32):
            amax = np.float32(np.max(np.abs(row)))
            lam = np.float32(np.float32(q) / amax)
            lams.append(Fraction(float(lam)))
        codes = [[max(-q, min(q, frac_round(lams[i] * Xf[i][j], "floor"))) for j in range(len(Xf[0]))]
                 for i in range(len(Xf))]
        Xt = [[Fraction(codes[i][j]) / lams[i] for j in range(len(Xf[0]))] for i in range(len(Xf))]
        R = [[Xf[i][j] - Xt[i][j] for j in range(len(Xf[0]))] for i in range(len(Xf))]
        RT = frac_T(R)
        Z = to_frac(Om)
        for _ in range(power_steps):
            Z = frac_matmul(RT, frac_matmul(R, Z))
        P = frac_matmul(frac_matmul(Z, frac_inv(frac_matmul(frac_T(Z), Z))), frac_T(Z))
        Rk = frac_matmul(R, P)
        return codes, lams, Xt, Rk

    ca, la, Af, RAk = side(A, OmA)
    cb, lb, Btf, RBtk = side(Bt, OmB)
    M, N = len(ca), len(cb)
    CF = [[Fraction(sum(ca[i][t] * cb[j][t] for t in range(len(ca[0])))) / (la[i] * lb[j]) for j in range(N)]
          for i in range(M)]
    Bf = frac_T(Btf)
    RBk = frac_T(RBtk)
    T2 = frac_matmul(RAk, Bf)
    T3 = frac_matmul(Af, RBk)
    T4 = frac_matmul(RAk, RBk)
    return np.array([[float(CF[i][j] + T2[i][j] + T3[i][j] + T4[i][j]) for j in range(N)] for i in range(M)])


@pytest.mark.parametrize("bits,dist,q", [(4, "normal", 1), (4, "u01", 1), (8, "exp4", 1),
                                         (4, "normal", 2), (8, "u01", 2), (4, "exp4", 3)])
def test_8x8_exact_rational_brute_force(bits, dist, q):
    A, Bt, OmA, OmB = S.problem(8, 8, 8, 3, s=4, dist=dist)
    exact = _exact_lrqmm_projector_form(A, Bt, bits, OmA, OmB, power_steps=q)
    D = O.lrqmm(A, Bt, bits, 3, OmA, OmB, q=q)
    assert np.max(np.abs(D - exact)) <= 1e-12 * np.max(np.abs(exact))
    if q >= 2:
        # the pin discriminates q: the q-1 result is far outside the tolerance (a loop that
        # hoisted Y = R Q1 out of the power iteration would make q = 2 return the q = 1 value)
        prev = _exact_lrqmm_projector_form(A, Bt, bits, OmA, OmB, power_steps=q - 1)
        assert np.max(np.abs(prev - exact)) > 1e-8 * np.max(np.abs(exact))


def test_alpha_beta_contract():
    # PAPER.md:372 D = alpha C_F + beta D
    A, Bt, OmA, OmB = S.problem(20, 16, 24, 6, s=1)
    D0 = np.random.default_rng(1).standard_normal((20, 16))
    base = O.lrqmm(A, Bt, 4, 4, OmA, OmB)
    assert np.array_equal(O.lrqmm(A, Bt, 4, 4, OmA, OmB, alpha=0.0, beta=1.0, D=D0), D0)
    got = O.lrqmm(A, Bt, 4, 4, OmA, OmB, alpha=2.0, beta=0.5, D=D0)
    assert np.allclose(got, 2.0 * base + 0.5 * D0, rtol=0, atol=1e-12)


# --------------------------------------- Tables 2/3 (paper-printed values)
@pytest.mark.slow
@pytest.mark.parametrize("bits", [4, 8])
def test_tables_2_3_lrqmm_and_dq_columns(golden_tables, bits):
    """Reproduce the paper's printed errors at 2000^3, r = 10 (PAPER.md:711-744,
    814) under readings #1/#2/#27: LRQMM = floor, per-row/col, p = 5, q = 1;
    DQ and QT = truncation, per-tensor.  Band x1.5, except ChiSquare's
    LRQMM cells (x3; SPEC.md:616-617 allows x3 / x5)."""
    for dist in S.DISTS:
        ref = golden_tables[(dist, bits)]
        A, Bt, OmA, OmB = S.problem(2000, 2000, 2000, 15, s=0, dist=dist)
        C = O.matmul_exact(A, Bt)
        e_lr = O.relative_error(C, O.lrqmm(A, Bt, bits, 10, OmA, OmB, q=1))
        e_dq = O.relative_error(C, O.direct_quant(A, Bt, bits))
        band = 3.0 if dist == "chi1" else 1.5
        assert ref["lrqmm"] / band <= e_lr <= ref["lrqmm"] * band, (dist, bits, e_lr, ref)
        assert ref["dq"] / 1.5 <= e_dq <= ref["dq"] * 1.5, (dist, bits, e_dq, ref)
        if dist in ("normal", "u01", "exp4"):
            e3 = O.relative_error(C, O.qt_gemm(A, Bt, bits, 3))
            e4 = O.relative_error(C, O.qt_gemm(A, Bt, bits, 4))
            assert ref["qt110"] / 1.5 <= e3 <= ref["qt110"] * 1.5, (dist, e3)
            assert ref["qt111"] / 1.5 <= e4 <= ref["qt111"] * 1.5, (dist, e4)


def test_negative_control_wrong_rounding_fails_table_pin(golden_tables):
    # SPEC.md:584 negative control: nearest rounding with per-tensor scale is
    # NOT the paper's DQ; it misses the Uniform(0,1) int4 DQ cell by >10x.
    A, Bt, _, _ = S.problem(600, 600, 600, 1, s=0, dist="u01")
    C = O.matmul_exact(A, Bt)
    e = O.relative_error(C, O.direct_quant(A, Bt, 4, rounding="nearest", granularity="tensor"))
    assert e < golden_tables[("u01", 4)]["dq"] / 10


def test_rsvd_q0_is_algorithm1_on_the_sampled_basis():
    """q = 0 (reading #30): Algorithm 1 on Q = orth(R Omega).  Pins: (i) R of
    exact rank <= k is recovered exactly (Q spans range(R) almost surely, so Q Q^T R = R);
    (ii) the rank-r result is the Eckart-Young truncation of the PROJECTION Q Q^T R (SVD of B =
    Q^T R, computed here independently through the Gram of the projection); (iii) a structured
    sketch whose first column is all ones captures a constant (mean) residual exactly."""
    rng = np.random.default_rng(41)
    R = rng.standard_normal((30, 4)) @ rng.standard_normal((4, 25))
    US, V = O.rsvd(R, rng.standard_normal((25, 6)), 6, 0)
    np.testing.assert_allclose(US @ V.T, R, atol=1e-10 * np.abs(R).max())
    R = rng.standard_normal((40, 33))
    Om = rng.standard_normal((33, 9))
    US, V = O.rsvd(R, Om, 4, 0)
    Q, _ = np.linalg.qr(R @ Om)
    P = Q @ (Q.T @ R)
    w, E = np.linalg.eigh(P.T @ P)           # right singular vectors of the projection
    E4 = E[:, np.argsort(-w)[:4]]
    np.testing.assert_allclose(US @ V.T, P @ E4 @ E4.T, atol=1e-9 * np.abs(P).max())
    Rc = np.full((20, 16), 0.37)             # floor-rounding residual mean: a constant matrix
    Om = rng.standard_normal((16, 3))
    Om[:, 0] = 1.0
    US, V = O.rsvd(Rc, Om, 1, 0)
    np.testing.assert_allclose(US @ V.T, Rc, atol=1e-12)


def test_im2col_is_the_convolution_as_a_gemm():
    """im2col_nhwc pinned to the textbook definition of a 2-D convolution (direct loops) and to
    torch's conv2d (an independent library routine), with stride, padding and dilation."""
    import torch
    rng = np.random.default_rng(7)
    for (B, H, W, C, kh, kw, s, p, d, Co) in [(2, 7, 6, 3, 3, 3, 1, 1, 1, 4), (1, 9, 9, 5, 3, 2, 2, 1, 1, 3),
                                              (2, 8, 7, 2, 3, 3, 2, 2, 2, 2), (1, 5, 5, 4, 1, 1, 2, 0, 1, 3)]:
        X = rng.standard_normal((B, H, W, C))
        Wt = rng.standard_normal((Co, kh, kw, C))
        M = O.im2col_nhwc(X, kh, kw, (s, s), (p, p), (d, d))
        Y = M @ Wt.reshape(Co, -1).T
        Ho = (H + 2 * p - d * (kh - 1) - 1) // s + 1
        Wo = (W + 2 * p - d * (kw - 1) - 1) // s + 1
        ref = np.zeros((B, Ho, Wo, Co))
        for b in range(B):
            for ho in range(Ho):
                for wo in range(Wo):
                    for i in range(kh):
                        for j in range(kw):
                            hi, wi = ho * s - p + i * d, wo * s - p + j * d
                            if 0 <= hi < H and 0 <= wi < W:
                                ref[b, ho, wo] += Wt[:, i, j, :] @ X[b, hi, wi, :]
        np.testing.assert_allclose(Y.reshape(B, Ho, Wo, Co), ref, atol=1e-12)
        t = torch.nn.functional.conv2d(torch.from_numpy(X).permute(0, 3, 1, 2), torch.from_numpy(Wt).permute(0, 3, 1, 2),
                                       stride=s, padding=p, dilation=d)
        np.testing.assert_allclose(Y.reshape(B, Ho, Wo, Co), t.permute(0, 2, 3, 1).numpy(), atol=1e-12)
