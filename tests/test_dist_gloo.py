"""world_size-2 CPU (gloo) tests of the N > 1 path.

With A row-sharded over ranks and B replicated, liblrqmm's rsvd_residual reduces exactly two
A-side quantities across ranks (lrqmm_api.cu: gram_step / allreduce_f32):
  * the W x W Gram  G = sum_ranks Y_rank^T Y_rank  of every row-sharded panel (Y = R Omega,
    Y = R Q1) before the orthonormalisation / truncation solve, and
  * Z_A = sum_ranks R_A,rank^T Q0_A,rank  (K x W), the power-iteration product over rows.
Everything else (quantization with per-row scales, the B side, the cross products and the
factor assembly) is rank-local.  These tests run that schedule with gloo collectives on two
CPU processes and check it reproduces the UNSHARDED oracle RSVD (Algorithm 1)
of the full residual, plus bench.py's rank helpers (unique-id broadcast, max over ranks, row
sharding).  The GPU side of the same schedule (NCCL on the handle stream) needs >1 GPU and is
not exercised in this environment.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth as S  # noqa: E402
from oracle import lrqmm_oracle as O  # noqa: E402

WS = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _orth_from_gram(Y_blk: np.ndarray, G: np.ndarray) -> np.ndarray:
    """Q = Y T with T = V S^-1 from the GLOBAL Gram G = V S^2 V^T: the left singular vectors of the
    row-sharded Y (same rank threshold as oracle.orth), computed from the reduced Gram only."""
    w, V = np.linalg.eigh(G)
    idx = np.argsort(-w, kind="stable")
    w, V = w[idx], V[:, idx]
    s = np.sqrt(np.maximum(w, 0.0))
    keep = s > O.ORTH_RTOL * s[0]
    return Y_blk @ (V[:, keep] / s[keep])


def _sharded_rsvd(R_blk: np.ndarray, Om: np.ndarray, r: int, q: int):
    """liblrqmm's A-side schedule with the two cross-rank reductions (see module docstring)."""
    Y = R_blk @ Om
    Q1 = None
    for _ in range(q):
        G = _allreduce(Y.T @ Y)                     # reduced Gram of the sharded Y
        Q0 = _orth_from_gram(Y, G)
        Z = _allreduce(R_blk.T @ Q0)                # Z = R^T Q0, summed over the row shards
        Q1 = O.orth(Z)                              # K rows: replicated, rank-local
        Y = R_blk @ Q1
    GW = _allreduce(Y.T @ Y)                        # truncation Gram of W = R Q1
    w, V = np.linalg.eigh(GW)
    VW = V[:, np.argsort(-w, kind="stable")[:r]]
    return Y @ VW, Q1 @ VW


def _sharded_rsvd_q0(R_blk: np.ndarray, Om: np.ndarray, r: int):
    """liblrqmm's q = 0 schedule (reading #30) on row-sharded panels: the Gram of Y = R Omega and
    Z = R^T Q0 are summed over ranks; the truncation eig(Z^T Z) is replicated (Z is)."""
    Y = R_blk @ Om
    Q0 = _orth_from_gram(Y, _allreduce(Y.T @ Y))
    Z = _allreduce(R_blk.T @ Q0)
    w, V = np.linalg.eigh(Z.T @ Z)
    VW = V[:, np.argsort(-w, kind="stable")[:r]]
    return Q0 @ VW, Z @ VW


def _worker(rank, port, M, K, bits, r, p, q, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        import bench

        # 1. host helpers: NCCL-id broadcast, max over ranks, row shards
        uid = bytes(range(128)) if rank == 0 else None
        got = bench.broadcast_unique_id(uid, WS, rank, "cpu")
        assert got == bytes(range(128))
        assert bench.max_over_ranks(1.0 + rank, WS, "cpu") == float(WS)
        lo, hi = bench.row_shard(M, WS, rank)

        # 2. sharded RSVD of the A residual == unsharded oracle
        A = S.gen_matrix("normal", M, K, 11)
        Om = S.gen_omega(K, r + p, 12)
        codes, lam = O.quantize(A[lo:hi], bits, "floor", "row")
        R_blk = O.residual(A[lo:hi], codes, lam)
        US_blk, V = _sharded_rsvd(R_blk, Om, r, q) if q > 0 else _sharded_rsvd_q0(R_blk, Om, r)
        np.save(os.path.join(out_dir, f"us_{rank}.npy"), US_blk)
        np.save(os.path.join(out_dir, f"v_{rank}.npy"), V)
        np.save(os.path.join(out_dir, f"codes_{rank}.npy"), codes)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,K,bits,r,p,q", [(96, 80, 4, 4, 3, 1), (101, 64, 8, 6, 5, 2), (90, 70, 4, 5, 3, 0)])
def test_sharded_rsvd_matches_oracle(tmp_path, M, K, bits, r, p, q):
    port = _free_port()
    mp.spawn(_worker, args=(port, M, K, bits, r, p, q, str(tmp_path)), nprocs=WS, join=True)
    import bench

    A = S.gen_matrix("normal", M, K, 11)
    Om = S.gen_omega(K, r + p, 12)
    codes, lam = O.quantize(A, bits, "floor", "row")
    R = O.residual(A, codes, lam)
    US, V = O.rsvd(R, Om, r, q)
    Rk = US @ V.T                                   # basis-independent rank-r approximation
    for rank in range(WS):
        lo, hi = bench.row_shard(M, WS, rank)
        # per-row scales make quantization shard-invariant (bit-exact codes)
        np.testing.assert_array_equal(np.load(tmp_path / f"codes_{rank}.npy"), codes[lo:hi])
        V_r = np.load(tmp_path / f"v_{rank}.npy")
        US_r = np.load(tmp_path / f"us_{rank}.npy")
        np.testing.assert_allclose(US_r @ V_r.T, Rk[lo:hi], rtol=0, atol=1e-9 * np.abs(Rk).max())
        # the K-side factor is replicated: every rank holds the same V (up to column sign; q = 0
        # carries Sigma in V, so compare directions)
        Vn, V_rn = V / np.linalg.norm(V, axis=0), V_r / np.linalg.norm(V_r, axis=0)
        np.testing.assert_allclose(np.abs(V_rn.T @ Vn), np.eye(V.shape[1]), atol=1e-8)


def _allgather_blocks(x: np.ndarray, blk: int) -> np.ndarray:
    """In-place allgather of equal blocks of `blk` rows (the last rank's block zero-padded), as
    liblrqmm's allgather_b does for the B codes, scales and L_B."""
    pad = np.zeros((blk,) + x.shape[1:], dtype=x.dtype)
    pad[: x.shape[0]] = x
    out = [torch.zeros_like(torch.from_numpy(pad)) for _ in range(WS)]
    dist.all_gather(out, torch.from_numpy(pad))
    return np.concatenate([o.numpy() for o in out])


def _worker_bsh(rank, port, M, N, K, bits, r, p, q, out_dir):
    """B column-sharded mode (cfg.b_sharded): A rows AND B^T rows sharded; both
    RSVDs reduce their Grams and Z across ranks; the B codes, scales and L_B are allgathered in
    blocks of ceil(N / ws) rows; each rank then forms its rows of D against all N columns."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    try:
        import bench

        A = S.gen_matrix("normal", M, K, 21)
        Bt = S.gen_matrix("normal", N, K, 22)
        OmA, OmB = S.gen_omega(K, r + p, 23), S.gen_omega(K, r + p, 24)
        lo, hi = bench.row_shard(M, WS, rank)
        blk = -(-N // WS)
        blo, bhi = blk * rank, min(N, blk * (rank + 1))
        ca, la = O.quantize(A[lo:hi], bits, "floor", "row")
        cb, lb = O.quantize(Bt[blo:bhi], bits, "floor", "row")
        RA = O.residual(A[lo:hi], ca, la)
        RB = O.residual(Bt[blo:bhi], cb, lb)
        USa, Va = _sharded_rsvd(RA, OmA, r, q)
        USb, Vb = _sharded_rsvd(RB, OmB, r, q)
        # factor assembly on local rows (Alg. 2 lines 361-366 folded into L_A, L_B)
        Af = O.dequantize(ca, la)
        Btf = O.dequantize(cb, lb)
        LA = np.hstack([USa, Af @ Vb])
        LB = np.hstack([Btf @ Va + USb @ (Vb.T @ Va), USb])
        # allgathers: every rank's GEMM covers all N columns
        cb_all = _allgather_blocks(cb, blk)[:N]
        lb_all = _allgather_blocks(lb, blk)[:N]
        LB_all = _allgather_blocks(LB, blk)[:N]
        D = O.dequant_result(O.int_gemm(ca, cb_all), la, lb_all) + LA @ LB_all.T
        np.save(os.path.join(out_dir, f"d_{rank}.npy"), D)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,N,K,bits,r,p,q", [(64, 90, 80, 4, 4, 3, 1), (50, 77, 64, 8, 5, 3, 1)])
def test_b_sharded_schedule_matches_oracle(tmp_path, M, N, K, bits, r, p, q):
    port = _free_port()
    mp.spawn(_worker_bsh, args=(port, M, N, K, bits, r, p, q, str(tmp_path)), nprocs=WS, join=True)
    import bench

    A = S.gen_matrix("normal", M, K, 21)
    Bt = S.gen_matrix("normal", N, K, 22)
    ref = O.lrqmm(A, Bt, bits, r, S.gen_omega(K, r + p, 23), S.gen_omega(K, r + p, 24), q=q)
    for rank in range(WS):
        lo, hi = bench.row_shard(M, WS, rank)
        D = np.load(tmp_path / f"d_{rank}.npy")
        assert D.shape == (hi - lo, N)
        np.testing.assert_allclose(D, ref[lo:hi], rtol=0, atol=1e-9 * np.abs(ref).max())


def test_row_shard_covers_rows():
    import bench

    for M in (0, 1, 7, 64, 1001):
        for ws in (1, 2, 3, 8):
            spans = [bench.row_shard(M, ws, r) for r in range(ws)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(spans[i][1] == spans[i + 1][0] for i in range(ws - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
