"""liblrqmm's OWN row-sharded path on one B200.

Each rank is a handle of this process created through the test transport
(`lrqmm_debug_create_loopback`, include/lrqmm_debug.h) and driven by its own host thread and
CUDA stream: the sharded schedule, buffers and kernels are the product's (A row-sharded, the
Gram / Z allreduces of the A-side RSVD, B replicated or column-sharded with the in-place
allgathers of codes, scales and L_B, static-B), only NCCL is replaced by host-synchronised
collectives on the one device.  Every rank's codes, scales (as bits) and int32 accumulators are
compared bit-exactly with the single-process fp64 oracle's rows, and the stacked D against the
oracle's D with the north_star bars (rel. Frobenius <= 1e-4, error <= 1.05x the oracle's).
The paper itself is single-GPU; the split is SURVEY §8(e)'s.
"""
import itertools
import threading

import numpy as np
import pytest

import oracle as O
import synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2409_18772_b200 import SIDE_A, SIDE_B, Lrqmm, LrqmmError  # noqa: E402

DEV = "cuda:0"
TOL_D = 1e-4
ERR_RATIO = 1.05
_groups = itertools.count(1000)


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def row_shard(M, ws, rank):
    base, extra = divmod(M, ws)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def run_ranks(P, A, Bt, OmA, OmB, bits, r, p, q=1, b_sharded=False, static_b=False, calls=1):
    """Run every rank in its own thread; returns per-rank dicts (numpy) and the shard bounds."""
    M, K = A.shape
    N = Bt.shape[0]
    kk = r + p
    group = next(_groups)
    shards = [row_shard(M, P, i) for i in range(P)]
    a_dev = [cu(A[lo:hi]) for lo, hi in shards]
    b_dev = cu(Bt)
    oma, omb = cu(OmA[:, :kk]), cu(OmB[:, :kk])
    outs = [torch.full((hi - lo, N), float("nan"), device=DEV) for lo, hi in shards]
    cints = [torch.zeros((hi - lo, N), dtype=torch.int32, device=DEV) for lo, hi in shards]
    streams = [torch.cuda.Stream(DEV) for _ in range(P)]
    torch.cuda.synchronize()
    res, errs = [None] * P, [None] * P
    barrier = threading.Barrier(P)

    def worker(i):
        try:
            lo, hi = shards[i]
            with Lrqmm(hi - lo, N, K, bits, r, p, q, world_size=P, world_rank=i, device=0, stream=streams[i],
                       b_sharded=b_sharded, loopback_group=group) as h:
                blo, bhi = h.b_rows
                barrier.wait(timeout=120)  # every rank joined the group
                for _ in range(calls):
                    if static_b:
                        h.quantize(SIDE_B, b_dev[blo:bhi])
                        h.rsvd_residual_b(omb)
                        h.quantize(SIDE_A, a_dev[i])
                        h.rsvd_residual(oma)
                    else:
                        h.quantize(SIDE_A, a_dev[i])
                        h.quantize(SIDE_B, b_dev[blo:bhi])
                        if r > 0:
                            h.rsvd_residual(oma, omb)
                    h.gemm(outs[i])
                h.gemm_int32(cints[i])
                h.sync()
                res[i] = dict(D=outs[i].cpu().numpy().astype(np.float64), c_int=cints[i].cpu().numpy(),
                              codes_a=h.codes(SIDE_A).cpu().numpy(), lam_a=h.scales(SIDE_A).cpu().numpy(),
                              codes_b=h.codes(SIDE_B).cpu().numpy(), lam_b=h.scales(SIDE_B).cpu().numpy(),
                              b_rows=(blo, bhi), launches=h.launch_count())
                h.sync()
        except BaseException as e:  # surfaced in the main thread
            errs[i] = e
            try:
                barrier.abort()
            except Exception:
                pass

    th = [threading.Thread(target=worker, args=(i,)) for i in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank hung"
    for e in errs:
        if e is not None:
            raise e
    return res, shards


def check_against_oracle(res, shards, A, Bt, OmA, OmB, bits, r, p, q):
    ref, parts = O.lrqmm(A, Bt, bits, r, OmA[:, :r + p], OmB[:, :r + p], q=q, return_parts=True)
    for (lo, hi), out in zip(shards, res):
        assert np.array_equal(out["codes_a"].astype(np.int64), parts["codes_a"][lo:hi])
        assert np.array_equal(out["lam_a"].view(np.uint32), parts["lam_a"][lo:hi].view(np.uint32))
        blo, bhi = out["b_rows"]
        assert np.array_equal(out["codes_b"].astype(np.int64), parts["codes_b"][blo:bhi])
        assert np.array_equal(out["lam_b"].view(np.uint32), parts["lam_b"][blo:bhi].view(np.uint32))
        # int32 accumulators of this rank's rows against ALL of B (allgathered codes when sharded)
        assert np.array_equal(out["c_int"].astype(np.int64), parts["c_int"][lo:hi])
        assert out["launches"] > 0
    D = np.vstack([out["D"] for out in res])
    assert np.all(np.isfinite(D))
    C = O.matmul_exact(A, Bt)
    diff = O.relative_error(ref, D)
    assert diff <= TOL_D, diff
    assert O.relative_error(C, D) <= ERR_RATIO * O.relative_error(C, ref)
    return diff


@pytest.mark.parametrize("P,M,N,K,b_sharded", [
    (2, 512, 384, 640, False),
    (2, 512, 384, 640, True),
    (4, 1000, 390, 700, False),
    (4, 1000, 390, 700, True),     # ragged B blocks (98, 98, 98, 96 rows of B^T)
    (3, 301, 257, 333, True),      # odd everything
])
@pytest.mark.parametrize("bits", [4, 8])
def test_sharded_lrqmm_matches_oracle(P, M, N, K, b_sharded, bits):
    r, p = 8, 5
    A, Bt, OmA, OmB = S.problem(M, N, K, r + p, s=P * 10 + bits, dist="normal" if bits == 4 else "u01")
    res, shards = run_ranks(P, A, Bt, OmA, OmB, bits, r, p, 1, b_sharded)
    check_against_oracle(res, shards, A, Bt, OmA, OmB, bits, r, p, 1)


@pytest.mark.parametrize("q", [0, 2])
@pytest.mark.parametrize("b_sharded", [False, True])
def test_sharded_power_iters(q, b_sharded):
    P, M, N, K, r, p = 4, 640, 512, 384, 12, 5
    A, Bt, OmA, OmB = S.problem(M, N, K, r + p, s=70 + q, dist="exp4")
    if q == 0:  # the labelled structured-sketch variant (reading #30)
        OmA[:, 0] = 1.0
        OmB[:, 0] = 1.0
    res, shards = run_ranks(P, A, Bt, OmA, OmB, 4, r, p, q, b_sharded)
    check_against_oracle(res, shards, A, Bt, OmA, OmB, 4, r, p, q)


@pytest.mark.parametrize("b_sharded", [False, True])
def test_sharded_static_b(b_sharded):
    """Weight-resident B: lrqmm_rsvd_residual_b once per B, then the
    A-side call -- the same correction as the full Algorithm 2 with that Omega_B."""
    P, M, N, K, r, p = 2, 768, 640, 512, 16, 5
    A, Bt, OmA, OmB = S.problem(M, N, K, r + p, s=91, dist="normal")
    res, shards = run_ranks(P, A, Bt, OmA, OmB, 4, r, p, 1, b_sharded, static_b=True)
    check_against_oracle(res, shards, A, Bt, OmA, OmB, 4, r, p, 1)


def test_sharded_repeated_calls_are_deterministic():
    """Three back-to-back calls per rank (the B allgathers overwrite the gathered blocks in
    place each call): the last D is bit-identical to a single call's."""
    P, M, N, K, r, p = 2, 512, 512, 512, 8, 5
    A, Bt, OmA, OmB = S.problem(M, N, K, r + p, s=5)
    one, _ = run_ranks(P, A, Bt, OmA, OmB, 4, r, p, 1, True, calls=1)
    three, shards = run_ranks(P, A, Bt, OmA, OmB, 4, r, p, 1, True, calls=3)
    for a, b in zip(one, three):
        assert np.array_equal(a["D"].view(np.uint64), b["D"].view(np.uint64))
    check_against_oracle(three, shards, A, Bt, OmA, OmB, 4, r, p, 1)


def test_shard_with_fewer_rows_than_the_sketch():
    """A rank holding fewer A rows than the sketch width r + p: only the global M bounds the rank
    (the Gram is summed over ranks)."""
    P, M, N, K, r, p = 4, 40, 96, 128, 8, 5   # 10 rows per rank < 13
    A, Bt, OmA, OmB = S.problem(M, N, K, r + p, s=8, dist="u01")
    res, shards = run_ranks(P, A, Bt, OmA, OmB, 4, r, p, 1, False)
    check_against_oracle(res, shards, A, Bt, OmA, OmB, 4, r, p, 1)


def test_loopback_group_mismatch_is_rejected():
    g = next(_groups)
    st = torch.cuda.Stream(DEV)
    with Lrqmm(64, 64, 64, 4, 4, 2, world_size=2, world_rank=0, stream=st, loopback_group=g):
        with pytest.raises(LrqmmError):   # same group, another world size
            Lrqmm(64, 64, 64, 4, 4, 2, world_size=4, world_rank=1, stream=st, loopback_group=g)
