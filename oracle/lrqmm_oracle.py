"""LRQMM oracle: a plain, slow, obviously-correct fp64 CPU implementation.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import this module.
The product path (`paper_2409_18772_b200`, `liblrqmm.so`) never calls it and
shares no code, header, table or helper with it.

It follows "A method of using RSVD in residual calculation of LowBit GEMM"
(arXiv 2409.18772), cited as PAPER.md:<line> with the LaTeX label of the
equation or algorithm, and the readings of SURVEY.md §8(c) (restated, each
one numbered).  Every floating-point
step is NumPy fp64 unless the definition itself fixes fp32 (the scale
lambda, reading #4).  Library primitives used as steps: `@` (matmul),
`np.linalg.svd` (orthonormal basis), `np.linalg.eigh` (k x k truncation).

Pins (all in tests/test_oracle_pins.py, `-m "not gpu"`):
  compute_scale / quantize   -> exact rational arithmetic (fractions.Fraction)
                                and SPEC.md:141-153 examples
  int_gemm / dequant_result  -> Python-int triple loops; SPEC.md:181, 319
  orth                       -> known-spectrum (Hadamard) matrices: the 1e-5
                                threshold is relative to sigma_max at scales
                                1e-12 / 1 / 1e6 (reading #12)
  rsvd                       -> full-rank recovery, exact-rank fixtures,
                                Eckart-Young, SPEC.md:235-245 examples; every
                                q in {1, 2, 3} against the exact-rational
                                projector onto span((R^T R)^q Omega)
  lrqmm                      -> exact rational (Fraction) evaluation of the
                                projector form on 8x8, zero residual, full
                                rank identity (Eq. gemm_r_split), rank-1
                                fixture, Tables 2/3 (tests/golden/)
No function here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

ORTH_RTOL = 1e-5  # drop directions with sigma < 1e-5 * sigma_max


# ---------------------------------------------------------------------------
# Quantization: Eq. quantA, vector-wise,
# Eq. get_ra2 floor residual, Alg. 2, 352-353.
# ---------------------------------------------------------------------------
def qmax_of(bits: int) -> int:
    """2^(N-1) - 1, the numerator of lambda in Eq. quantA."""
    return (1 << (bits - 1)) - 1


def compute_scale(amax, bits: int):
    """lambda = (2^(N-1)-1) / a_max, Eq. quantA.

    Reading #4: evaluated as an IEEE fp32 division (round to nearest even) of
    fp32 operands; reading #6: lambda = 1 where a_max == 0.
    `amax` may be a scalar or an array; returns float32 of the same shape.
    """
    amax = np.asarray(amax, dtype=np.float32)
    q = np.float32(qmax_of(bits))
    with np.errstate(divide="ignore"):
        lam = (q / amax).astype(np.float32)
    return np.where(amax == 0, np.float32(1.0), lam).astype(np.float32)


def _round(t: np.ndarray, rounding: str) -> np.ndarray:
    if rounding == "floor":      # Eq. get_ra2
        return np.floor(t)
    if rounding == "trunc":      # Eq. quantA TypeCast, PAPER.md:192 (reading #2)
        return np.trunc(t)
    if rounding == "nearest":    # Eq. quantAB round, PAPER.md:206 (half to even)
        return np.rint(t)
    raise ValueError(rounding)


def quantize(X: np.ndarray, bits: int, rounding: str = "floor", granularity: str = "row"):
    """Symmetric quantizer of Eq. quantA with one lambda per row (vector-wise).

    X is rows x K float32 (a side: A, or B^T so that "per row of B^T" is the
    paper's "per column of B").  Returns (codes int64, lam f32).
      amax_i = max_j |X_ij|                          (exact)
      lam_i  = fp32(qmax / amax_i), 1 if amax_i == 0 (reading #4, #6)
      code   = clip(round_mode(lam_i * X_ij), -qmax, qmax)   (reading #5)
    The product lam_i * X_ij of two fp32 numbers is exact in fp64 (24+24 < 53
    significand bits), so the rounding decision is taken on the exact value.
    """
    X = np.asarray(X, dtype=np.float32)
    if not np.all(np.isfinite(X)):
        raise ValueError("non-finite input (reading #7)")
    if granularity == "row":
        amax = np.max(np.abs(X), axis=1) if X.shape[1] else np.zeros(X.shape[0], np.float32)
        lam = compute_scale(amax, bits)
    elif granularity == "tensor":
        amax = np.max(np.abs(X)) if X.size else np.float32(0)
        lam = np.full(X.shape[0], compute_scale(amax, bits), dtype=np.float32)
    else:
        raise ValueError(granularity)
    t = lam.astype(np.float64)[:, None] * X.astype(np.float64)
    q = qmax_of(bits)
    codes = np.clip(_round(t, rounding), -q, q).astype(np.int64)
    return codes, lam


def dequantize(codes: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """X~ = code / lambda (Alg. 2), fp64."""
    return codes.astype(np.float64) / lam.astype(np.float64)[:, None]


def residual(X: np.ndarray, codes: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """R = X - Dequant(X_int) (Alg. 2), fp64."""
    return X.astype(np.float64) - dequantize(codes, lam)


# ---------------------------------------------------------------------------
# Integer GEMM and dequantization: Eq. INTGEMM,
# Eq. QUANTGEMM.
# ---------------------------------------------------------------------------
def int_gemm(codes_a: np.ndarray, codes_bt: np.ndarray) -> np.ndarray:
    """C_int = A_int B_int with B passed as B^T (N x K): exact, returned as int64.

    Evaluated with an fp64 matmul: every product and partial sum is an
    integer of magnitude <= K * max|code|^2 < 2^53 (asserted), so each fp64
    operation is exact whatever the summation order (reading #24).
    """
    K = codes_a.shape[1]
    mx = max(int(np.abs(codes_a).max(initial=0)), 1) * max(int(np.abs(codes_bt).max(initial=0)), 1)
    assert K * mx < 2 ** 53, "fp64 evaluation would not be exact"
    c = codes_a.astype(np.float64) @ codes_bt.astype(np.float64).T
    return c.astype(np.int64)


def dequant_result(c_int: np.ndarray, lam_a: np.ndarray, lam_b: np.ndarray) -> np.ndarray:
    """C_F = C_int / (lambda_A lambda_B), Eq. QUANTGEMM, per row/col."""
    return c_int.astype(np.float64) / (lam_a.astype(np.float64)[:, None] * lam_b.astype(np.float64)[None, :])


# ---------------------------------------------------------------------------
# Randomized SVD: Algorithm 1, range finder per reading
# #11 (variant (b): Algorithm 1 applied to R^T with Q = orth(R^T orth(R Omega)),
# q power iterations, Eq. rsvderror's q), truncation to rank r
# with the k-svd of Eq. k-svd.
# ---------------------------------------------------------------------------
def orth(M: np.ndarray, rtol: float = ORTH_RTOL) -> np.ndarray:
    """Orthonormal basis of span(M) ("orthogonal columns").

    Reading #12: directions with sigma < rtol * sigma_max are dropped (so an
    exactly rank-deficient or zero M gives a narrower / empty basis).
    """
    if M.size == 0:
        return np.zeros((M.shape[0], 0))
    U, s, _ = np.linalg.svd(M, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((M.shape[0], 0))
    keep = s >= rtol * s[0]
    return U[:, keep]


def rsvd(R: np.ndarray, omega: np.ndarray, r: int, q: int = 1):
    """RSVD of a residual R (rows x K) -> (USigma [rows x r'], V [K x r']), r' <= r.

    R ~= USigma @ V.T.  Steps (variant (b), reading #11):
      Y  = R Omega                               Alg. 1 sampling, PAPER.md:124,128
      repeat q times:
        Q0 = orth(Y); Z = R^T Q0; Q1 = orth(Z); Y = R Q1     (power iteration)
      (R_k = Y Q1^T is Algorithm 1 on R^T: B = Q1^T R^T = Y^T)
      if width(Q1) > r:  eig(Y^T Y) -> top-r eigenvectors V_W (descending);
                         USigma = Y V_W, V = Q1 V_W        (SVD of B)
      else:              USigma = Y,     V = Q1
    """
    if q == 0:
        # Algorithm 1 itself with Q from one sampling pass (reading #30): Q = orth(R Omega),
        # B = Q^* R, SVD(B), U = Q U', truncated to rank r
        return rsvd_spec_variant(R, omega, r, 0)
    if q < 0:
        raise ValueError("q >= 0")
    R = np.asarray(R, dtype=np.float64)
    Om = np.asarray(omega, dtype=np.float64)
    Y = R @ Om
    Q1 = None
    for _ in range(q):
        Q0 = orth(Y)
        Z = R.T @ Q0
        Q1 = orth(Z)
        Y = R @ Q1
    kk = Q1.shape[1]
    if kk > r:
        G = Y.T @ Y
        w, V = np.linalg.eigh(G)
        idx = np.argsort(-w, kind="stable")[:r]
        VW = V[:, idx]
        return Y @ VW, Q1 @ VW
    return Y, Q1


def rsvd_spec_variant(R: np.ndarray, omega: np.ndarray, r: int, q: int = 1):
    """SPEC.md:229-257 pass structure (variant (a)): Q = orth((R R^T)^q R Omega),
    B = Q^T R, SVD(B) truncated to r.  Used only to compare accuracy (E3)."""
    R = np.asarray(R, dtype=np.float64)
    Q = orth(R @ np.asarray(omega, dtype=np.float64))
    for _ in range(q):
        Q = orth(R.T @ Q)
        Q = orth(R @ Q)
    B = Q.T @ R
    if B.size == 0:
        return np.zeros((R.shape[0], 0)), np.zeros((R.shape[1], 0))
    U, s, Vt = np.linalg.svd(B, full_matrices=False)
    U, s, Vt = U[:, :r], s[:r], Vt[:r]
    return (Q @ U) * s[None, :], Vt.T


# ---------------------------------------------------------------------------
# Algorithm 2: D = alpha A.B + beta D.
# ---------------------------------------------------------------------------
def lrqmm(A, Bt, bits: int, r: int, omega_a=None, omega_b=None, q: int = 1,
          alpha: float = 1.0, beta: float = 0.0, D=None,
          rounding: str = "floor", granularity: str = "row", return_parts: bool = False):
    """LRQMM of A (M x K) and B (K x N, passed as B^T: N x K), literal Alg. 2.

    omega_a / omega_b: K x k sketches (k = r + p), reading #8.  r == 0 gives
    plain direct quantization with the chosen rounding (no correction).
    """
    A = np.asarray(A, dtype=np.float32)
    Bt = np.asarray(Bt, dtype=np.float32)
    # line 347: {A_int, B_int} <- Quant({A, B}, N)
    ca, la = quantize(A, bits, rounding, granularity)
    cb, lb = quantize(Bt, bits, rounding, granularity)
    # line 348: C_int = A_int B_int  (exact, reading #24)
    c_int = int_gemm(ca, cb)
    # line 349: C_F <- Dequant(C_int)
    CF = dequant_result(c_int, la, lb)
    parts = {"codes_a": ca, "lam_a": la, "codes_b": cb, "lam_b": lb, "c_int": c_int}
    if r > 0:
        # lines 352-353: residuals
        Af = dequantize(ca, la)                 # A_F   (M x K)
        Btf = dequantize(cb, lb)                # B_F^T (N x K)
        RA = A.astype(np.float64) - Af
        RBt = Bt.astype(np.float64) - Btf       # R_B^T
        # lines 356-357: RSVD(R_A, r), RSVD(R_B, r)   (R_B through R_B^T, reading #26)
        USa, Va = rsvd(RA, omega_a, r, q)       # R_A   ~= (U_r Sigma_r) V_r^T
        USb, Vb = rsvd(RBt, omega_b, r, q)      # R_B^T ~= USb Vb^T -> R_B ~= Vb USb^T
        # line 361: U~ = U_r Sigma_r ; Z~' = Gamma_r Z_r^T ; W_r = Vb
        Ut = USa
        Wr = Vb
        Zt = USb.T
        Bf = Btf.T                              # B_F (K x N)
        # lines 364-366, parenthesised exactly as printed
        RC1 = Ut @ (Va.T @ Bf)
        RC2 = (Af @ Wr) @ Zt
        RC3 = (Ut @ (Va.T @ Wr)) @ Zt
        # line 369
        CF = CF + RC1 + RC2 + RC3
        parts.update(USa=USa, Va=Va, USb=USb, Vb=Vb, RA=RA, RBt=RBt)
    # line 372: D = alpha C_F + beta D   (reading #16: beta == 0 -> D not read)
    out = alpha * CF
    if beta != 0.0:
        out = out + beta * np.asarray(D, dtype=np.float64)
    if return_parts:
        parts["D"] = out
        return out, parts
    return out


def direct_quant(A, Bt, bits: int, rounding: str = "trunc", granularity: str = "tensor"):
    """Eq. quantAB + INTGEMM + QUANTGEMM with no compensation (Table 4 caption,
    PAPER.md:763 "Direct Quant uses the first term").  Default = the paper's
    DQ column reading (#2): per-tensor scale, truncation."""
    return lrqmm(A, Bt, bits, 0, rounding=rounding, granularity=granularity)


def qt_gemm(A, Bt, bits: int, terms: int = 4, rounding: str = "trunc", granularity: str = "tensor"):
    """QuantTensor QT(1,1,0) (terms=3) / QT(1,1,1) (terms=4), Eq. gemm_r_split
    (PAPER.md:268-275): T1 plus the residual terms with *re-quantized*
    residuals R^int at the same N bits and their own scale lambda_R.
    Reading #27: the quantizer is Eq. quantA's TypeCast
    (truncation) with one per-tensor scale, for both the operands and the
    residuals -- the reading under which Tables 2/3's QT columns reproduce.
    Comparison column only; the residual is rounded to fp32
    before re-quantization (it is an fp32 GEMM operand on the GPU)."""
    A = np.asarray(A, dtype=np.float32)
    Bt = np.asarray(Bt, dtype=np.float32)
    ca, la = quantize(A, bits, rounding, granularity)
    cb, lb = quantize(Bt, bits, rounding, granularity)
    ra = (A.astype(np.float64) - dequantize(ca, la)).astype(np.float32)
    rb = (Bt.astype(np.float64) - dequantize(cb, lb)).astype(np.float32)
    cra, lra = quantize(ra, bits, rounding, granularity)
    crb, lrb = quantize(rb, bits, rounding, granularity)
    C = dequant_result(int_gemm(ca, cb), la, lb)                # T1
    C = C + dequant_result(int_gemm(ca, crb), la, lrb)          # A_int R_B^int
    C = C + dequant_result(int_gemm(cra, cb), lra, lb)          # R_A^int B_int
    if terms == 4:
        C = C + dequant_result(int_gemm(cra, crb), lra, lrb)    # R_A^int R_B^int
    return C


# ---------------------------------------------------------------------------
# Metrics
# ---------------------------------------------------------------------------
def matmul_exact(A, Bt) -> np.ndarray:
    """Ground truth C = A B in fp64 from the fp32 inputs (reading #19)."""
    return np.asarray(A, dtype=np.float64) @ np.asarray(Bt, dtype=np.float64).T


def frobenius_norm(X) -> float:
    return float(np.sqrt(np.sum(np.asarray(X, dtype=np.float64) ** 2)))


def relative_error(C_exact, C_approx) -> float:
    """||C - C~||_F / ||C||_F."""
    return frobenius_norm(np.asarray(C_exact, np.float64) - np.asarray(C_approx, np.float64)) / frobenius_norm(C_exact)


# ---------------------------------------------------------------------------
# im2col of an NHWC convolution input (the conv-layer workloads of PAPER.md:822 as
# GEMMs).  Test infrastructure: the explicit matrix whose quantization lrqmm_quantize_im2col
# must reproduce bit for bit.
# ---------------------------------------------------------------------------
def im2col_nhwc(X, kh: int, kw: int, stride=(1, 1), pad=(0, 0), dilation=(1, 1)) -> np.ndarray:
    """Rows (b, ho, wo), columns (i, j, c): element X[b, ho*sh - ph + i*dh, wo*sw - pw + j*dw, c],
    zero outside the image (zero padding)."""
    X = np.asarray(X)
    B, H, W, C = X.shape
    sh, sw = stride
    ph, pw = pad
    dh, dw = dilation
    Ho = (H + 2 * ph - dh * (kh - 1) - 1) // sh + 1
    Wo = (W + 2 * pw - dw * (kw - 1) - 1) // sw + 1
    Xp = np.zeros((B, H + 2 * ph, W + 2 * pw, C), dtype=X.dtype)
    Xp[:, ph:ph + H, pw:pw + W, :] = X
    out = np.empty((B, Ho, Wo, kh, kw, C), dtype=X.dtype)
    for i in range(kh):
        for j in range(kw):
            out[:, :, :, i, j, :] = Xp[:, i * dh: i * dh + sh * (Ho - 1) + 1: sh, j * dw: j * dw + sw * (Wo - 1) + 1: sw, :]
    return out.reshape(B * Ho * Wo, kh * kw * C)
