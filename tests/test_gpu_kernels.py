"""Stage-level checks of the CUDA kernels through the lrqmm_debug.h test hooks:
each RSVD building block vs NumPy fp64 on the oracle's residual."""
import numpy as np
import pytest

import oracle as O
import synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2409_18772_b200 import lrqmm as L  # noqa: E402

DEV = "cuda:0"


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300)


def side(rows, K, dist="normal", bits=4, seed=0):
    """Oracle codes / scales and the residual AS THE PASSES SEE IT: K1 stores the residual fraction
    u = lambda x - code in Q15 fixed point (kernels.h kUScale, reading #28), so the
    stage reference is R_q = (RN(2^15 (lambda x - code)) / 2^15) / lambda, within 2^-16 / lambda (2^-15 where u rounds past the clamp) of the oracle's R."""
    X = S.gen_matrix(dist, rows, K, seed)
    codes, lam = O.quantize(X, bits)
    R = O.residual(X, codes, lam)
    lam64 = lam.astype(np.float64)[:, None]
    # one rounding of the exact value: lambda x is exact in fp64 (24 + 24 bits), 2^15 scaling exact
    u16 = np.clip(np.rint((lam64 * X.astype(np.float64) - codes) * 32768.0), -32767, 32767)
    Rq = u16 / 32768.0 / lam64
    assert np.all(np.abs(Rq - R) <= 2.0 ** -15 / lam64 * (1 + 1e-9))  # 2^-16, 2^-15 at the clamp u -> 1
    return X, codes, lam, Rq


@pytest.mark.parametrize("rows,K,W", [(128, 32, 32), (300, 1000, 24), (1000, 333, 8), (257, 4096, 40), (64, 128, 64)])
def test_proj_rows(rows, K, W):
    X, codes, lam, R = side(rows, K)
    P = np.random.default_rng(1).standard_normal((K, W)).astype(np.float32)
    out = torch.zeros((rows, W), device=DEV)
    lib = L.load_library()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.lrqmm_debug_proj(0, cu(X).data_ptr(), K, rows, K, 4, 0, cu(P).data_ptr(), None,
                                W, out.data_ptr(), None, st) == 0
    assert rel(out.cpu().numpy(), R @ P.astype(np.float64)) < 1e-5


@pytest.mark.parametrize("rows,K,W", [(128, 128, 32), (300, 1000, 24), (1000, 333, 8), (4096, 257, 40)])
def test_proj_cols(rows, K, W):
    X, codes, lam, R = side(rows, K, "u01")
    P = np.random.default_rng(2).standard_normal((rows, W)).astype(np.float32)
    out = torch.zeros((K, W), device=DEV)
    lib = L.load_library()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.lrqmm_debug_proj(1, cu(X).data_ptr(), K, rows, K, 4, 0, cu(P).data_ptr(), None,
                                W, out.data_ptr(), None, st) == 0
    assert rel(out.cpu().numpy(), R.T @ P.astype(np.float64)) < 1e-5


@pytest.mark.parametrize("rows,K,W", [(128, 32, 32), (300, 1000, 24), (257, 2048, 48)])
def test_proj_rows_dual(rows, K, W):
    X, codes, lam, R = side(rows, K, "exp4", bits=8)
    rng = np.random.default_rng(3)
    P = rng.standard_normal((K, W)).astype(np.float32)
    P2 = rng.standard_normal((K, W)).astype(np.float32)
    out = torch.zeros((rows, W), device=DEV)
    out2 = torch.zeros((rows, W), device=DEV)
    lib = L.load_library()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.lrqmm_debug_proj(2, cu(X).data_ptr(), K, rows, K, 8, 0, cu(P).data_ptr(),
                                cu(P2).data_ptr(), W, out.data_ptr(), out2.data_ptr(), st) == 0
    assert rel(out.cpu().numpy(), R @ P.astype(np.float64)) < 1e-5
    assert rel(out2.cpu().numpy(), O.dequantize(codes, lam) @ P2.astype(np.float64)) < 1e-5


@pytest.mark.parametrize("n,W", [(1000, 24), (16384, 32), (77, 8), (5000, 64)])
def test_gram_and_orth(n, W):
    Y = np.random.default_rng(4).standard_normal((n, W)).astype(np.float32)
    Y[:, 0] *= 50.0  # a dominant direction, like the residual's mean term
    G = torch.zeros((W, W), dtype=torch.float64, device=DEV)
    T = torch.zeros((W, W), device=DEV)
    lib = L.load_library()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.lrqmm_debug_small(1, cu(Y).data_ptr(), n, W, 0, G.data_ptr(), T.data_ptr(), st) == 0
    Gref = Y.astype(np.float64).T @ Y.astype(np.float64)
    assert rel(G.cpu().numpy(), Gref) < 1e-12
    Q = Y.astype(np.float64) @ T.cpu().numpy().astype(np.float64)
    assert np.abs(Q.T @ Q - np.eye(W)).max() < 1e-4
    # same span
    assert np.linalg.norm(Y - Q @ (Q.T @ Y)) < 1e-5 * np.linalg.norm(Y)


def test_orth_drops_rank_deficient_directions():
    rng = np.random.default_rng(5)
    n, W = 500, 16
    base = rng.standard_normal((n, 5))
    Y = np.hstack([base, base @ rng.standard_normal((5, W - 5))]).astype(np.float32)  # rank 5 in fp32
    G = torch.zeros((W, W), dtype=torch.float64, device=DEV)
    T = torch.zeros((W, W), device=DEV)
    lib = L.load_library()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.lrqmm_debug_small(1, cu(Y).data_ptr(), n, W, 0, G.data_ptr(), T.data_ptr(), st) == 0
    Tn = T.cpu().numpy()
    kept = np.sum(np.abs(Tn).sum(axis=0) > 0)
    assert kept == 5
    Q = Y.astype(np.float64) @ Tn
    assert np.abs(Q.T @ Q - np.diag([1.0] * 5 + [0.0] * (W - 5))).max() < 1e-3


@pytest.mark.parametrize("W,r", [(24, 16), (40, 32), (8, 3)])
def test_truncation_eig(W, r):
    rng = np.random.default_rng(6)
    Y = (rng.standard_normal((2000, W)) * np.linspace(10, 1, W)).astype(np.float32)
    G = torch.zeros((W, W), dtype=torch.float64, device=DEV)
    T = torch.zeros((W, W), device=DEV)
    lib = L.load_library()
    st = torch.cuda.current_stream().cuda_stream
    assert lib.lrqmm_debug_small(2, cu(Y).data_ptr(), 2000, W, r, G.data_ptr(), T.data_ptr(), st) == 0
    Gn = G.cpu().numpy()
    w, V = np.linalg.eigh(Gn)
    top = V[:, np.argsort(-w)[:r]]
    Vt = T.cpu().numpy()[:, :r].astype(np.float64)
    # same top-r subspace, orthonormal columns, descending eigenvalues
    assert np.linalg.norm(top @ top.T - Vt @ Vt.T) < 1e-5
    assert np.abs(Vt.T @ Vt - np.eye(r)).max() < 1e-6
    ev = np.diag(Vt.T @ Gn @ Vt)
    assert np.all(np.diff(ev) <= 1e-9 * ev[0])
