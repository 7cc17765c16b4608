"""Thin ctypes binding of liblrqmm (include/lrqmm.h) — argument marshalling only.

Every step of LRQMM runs in the library's CUDA kernels; torch is used only for
device memory (tensors passed by data pointer) and the current CUDA stream.
There is no CPU fallback: if liblrqmm.so is missing or no sm_100 GPU is present
the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LRQMM_LIB: another build of this library (A/B timing of two builds in one session, tools/ab.sh)
LIB_PATH = os.environ.get("LRQMM_LIB") or os.path.join(_HERE, "liblrqmm.so")

SIDE_A, SIDE_B = 0, 1
ROUND = {"floor": 0, "trunc": 1, "nearest": 2}
GRAN = {"row": 0, "tensor": 1}

STATUS = {
    0: "LRQMM_OK", 1: "LRQMM_ERR_INVALID_ARGUMENT", 2: "LRQMM_ERR_SHAPE", 3: "LRQMM_ERR_RANK",
    4: "LRQMM_ERR_OVERFLOW", 5: "LRQMM_ERR_NONFINITE", 6: "LRQMM_ERR_STATE", 7: "LRQMM_ERR_CUDA",
    8: "LRQMM_ERR_NCCL", 9: "LRQMM_ERR_ALLOC", 10: "LRQMM_ERR_UNSUPPORTED",
}

# every symbol include/lrqmm.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "lrqmm_get_unique_id", "lrqmm_create", "lrqmm_quantize", "lrqmm_rsvd_residual", "lrqmm_gemm",
    "lrqmm_destroy", "lrqmm_sync", "lrqmm_run_host", "lrqmm_get_codes", "lrqmm_get_scales",
    "lrqmm_gemm_int32", "lrqmm_get_factors", "lrqmm_get_correction", "lrqmm_correction_width",
    "lrqmm_get_timings", "lrqmm_launch_count", "lrqmm_status_string", "lrqmm_rsvd_residual_b",
    "lrqmm_quantize_im2col", "lrqmm_run_host_async",
)
DEBUG_EXPORTS = ("lrqmm_debug_proj", "lrqmm_debug_small", "lrqmm_debug_set_gemm_variant",
                 "lrqmm_debug_create_loopback", "lrqmm_debug_fuse_trace", "lrqmm_debug_inject_fault")


class LrqmmError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)}")


class ConvGeom(ctypes.Structure):
    """lrqmm_conv_t (NHWC convolution geometry for quantize_im2col)."""
    _fields_ = [
        ("batch", ctypes.c_int64), ("H", ctypes.c_int), ("W", ctypes.c_int), ("C", ctypes.c_int),
        ("kh", ctypes.c_int), ("kw", ctypes.c_int), ("stride_h", ctypes.c_int), ("stride_w", ctypes.c_int),
        ("pad_h", ctypes.c_int), ("pad_w", ctypes.c_int), ("dil_h", ctypes.c_int), ("dil_w", ctypes.c_int),
    ]


class Config(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
        ("bits", ctypes.c_int), ("rank", ctypes.c_int), ("oversample", ctypes.c_int),
        ("power_iters", ctypes.c_int), ("rounding", ctypes.c_int), ("granularity", ctypes.c_int),
        ("world_size", ctypes.c_int), ("world_rank", ctypes.c_int),
        ("nccl_unique_id", ctypes.c_void_p), ("device", ctypes.c_int), ("stream", ctypes.c_void_p),
        ("enable_timing", ctypes.c_int), ("qt_terms", ctypes.c_int), ("b_sharded", ctypes.c_int),
    ]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load liblrqmm.so (raises OSError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not found: build it with `python -m paper_2409_18772_b200.build`")
    lib = ctypes.CDLL(path)
    P, I64, I, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
    sig = {
        "lrqmm_get_unique_id": (I, [P]),
        "lrqmm_create": (I, [ctypes.POINTER(Config), ctypes.POINTER(P)]),
        "lrqmm_quantize": (I, [P, I, P, I64]),
        "lrqmm_quantize_im2col": (I, [P, I, P, ctypes.POINTER(ConvGeom)]),
        "lrqmm_rsvd_residual": (I, [P, P, P, I64]),
        "lrqmm_rsvd_residual_b": (I, [P, P, I64]),
        "lrqmm_gemm": (I, [P, F, F, P, I64]),
        "lrqmm_destroy": (I, [P]),
        "lrqmm_sync": (I, [P]),
        "lrqmm_run_host": (I, [P, P, P, P, P, F, P]),
        "lrqmm_run_host_async": (I, [P, P, P, P, P, F, P]),
        "lrqmm_get_codes": (I, [P, I, P, I64]),
        "lrqmm_get_scales": (I, [P, I, P]),
        "lrqmm_gemm_int32": (I, [P, P, I64]),
        "lrqmm_get_factors": (I, [P, I, P, P]),
        "lrqmm_get_correction": (I, [P, I, P]),
        "lrqmm_correction_width": (I, [P]),
        "lrqmm_get_timings": (I, [P, ctypes.POINTER(ctypes.c_double)]),
        "lrqmm_launch_count": (I64, [P, I]),
        "lrqmm_status_string": (ctypes.c_char_p, [I]),
        # test hooks (include/lrqmm_debug.h)
        "lrqmm_debug_proj": (I, [I, P, I64, I64, I, I, I, P, P, I, P, P, P]),
        "lrqmm_debug_small": (I, [I, P, I64, I, I, P, P, P]),
        "lrqmm_debug_set_gemm_variant": (I, [I]),
        "lrqmm_debug_create_loopback": (I, [ctypes.POINTER(Config), I, ctypes.POINTER(P)]),
        "lrqmm_debug_fuse_trace": (I, [P, ctypes.POINTER(ctypes.c_int64)]),
        "lrqmm_debug_inject_fault": (I, [I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(code: int, where: str):
    if code != 0:
        raise LrqmmError(code, where)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _arg(t, dtype: str, device: int, name: str) -> int:
    """Device pointer of a caller tensor after checking what the C ABI assumes (a CUDA tensor of
    torch.<dtype> on the handle's device); raises ValueError instead of passing a wrong pointer."""
    import torch

    if t is None:
        return 0
    dtype = getattr(torch, dtype)
    if not t.is_cuda or t.device.index != device:
        raise ValueError(f"{name}: expected a tensor on cuda:{device}, got {t.device}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: expected {dtype}, got {t.dtype}")
    return int(t.data_ptr())


def _mat(t, dtype: str, device: int, name: str, rows: int, cols: int):
    """(pointer, ld) of a row-major rows x cols operand (a view of a larger tensor is fine): checks
    device and dtype (_arg), two dimensions, unit column stride and at least rows x cols elements,
    so the kernels never read or write past the caller's tensor."""
    if t is None:
        return 0, max(cols, 1)
    ptr = _arg(t, dtype, device, name)
    if t.dim() != 2:
        raise ValueError(f"{name}: expected a 2-D tensor, got {t.dim()}-D")
    if t.shape[0] < rows or t.shape[1] < cols:
        raise ValueError(f"{name}: expected at least {rows} x {cols}, got {tuple(t.shape)}")
    if t.shape[1] > 1 and t.stride(1) != 1:
        raise ValueError(f"{name}: row-major with unit column stride expected (strides {t.stride()})")
    ld = int(t.stride(0)) if t.shape[0] > 1 else max(int(t.shape[1]), 1)
    if ld < cols:
        raise ValueError(f"{name}: row stride {ld} < {cols} columns")
    return ptr, ld


def _host(a, name: str, shape):
    """Host pointer of a C-contiguous float32 NumPy array of exactly `shape` (run_host*)."""
    if a is None:
        return None
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{name}: expected a C-contiguous float32 numpy array")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {a.shape}")
    return ctypes.c_void_p(a.ctypes.data)


def get_unique_id() -> bytes:
    lib = load_library()
    buf = (ctypes.c_ubyte * 128)()
    _check(lib.lrqmm_get_unique_id(buf), "lrqmm_get_unique_id")
    return bytes(buf)


class Lrqmm:
    """Handle around one LRQMM problem shape (lrqmm_create ... lrqmm_destroy)."""

    def __init__(self, m: int, n: int, k: int, bits: int = 4, rank: int = 16, oversample: int = 5,
                 power_iters: int = 1, rounding: str = "floor", granularity: str = "row",
                 world_size: int = 1, world_rank: int = 0, unique_id: bytes | None = None,
                 device: int = 0, stream=None, enable_timing: bool = False, qt_terms: int = 0,
                 b_sharded: bool = False, loopback_group: int | None = None):
        """loopback_group: test transport (include/lrqmm_debug.h lrqmm_debug_create_loopback) --
        world_size handles of this process, one host thread each, on one device, instead of NCCL."""
        import torch

        lib = load_library()
        self.lib = lib
        self.m, self.n, self.k = m, n, k
        self.bits, self.rank, self.oversample = bits, rank, oversample
        # rows of B^T this rank holds (b_sharded: blocks of ceil(n / world_size) rows)
        blk = -(-n // world_size) if (b_sharded and world_size > 1) else n
        lo = blk * world_rank if (b_sharded and world_size > 1) else 0
        self.b_rows = (lo, max(0, min(n, lo + blk)))
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self._uid = (ctypes.c_ubyte * 128).from_buffer_copy(unique_id) if unique_id else None
        cfg = Config(m, n, k, bits, rank, oversample, power_iters, ROUND[rounding], GRAN[granularity],
                     world_size, world_rank, ctypes.cast(self._uid, ctypes.c_void_p) if self._uid else None,
                     device, ctypes.c_void_p(stream.cuda_stream), 1 if enable_timing else 0, qt_terms,
                     1 if b_sharded else 0)
        h = ctypes.c_void_p()
        if loopback_group is None:
            _check(lib.lrqmm_create(ctypes.byref(cfg), ctypes.byref(h)), "lrqmm_create")
        else:
            _check(lib.lrqmm_debug_create_loopback(ctypes.byref(cfg), int(loopback_group), ctypes.byref(h)),
                   "lrqmm_debug_create_loopback")
        self.kk = rank + oversample if rank > 0 else 0
        self.h = h
        self._keep = {}

    # ---- the five calls of the boundary ----
    def side_rows(self, side: int) -> int:
        """Rows of the side's matrix on this rank: m for A, this rank's rows of B^T for B."""
        return self.m if side == SIDE_A else self.b_rows[1] - self.b_rows[0]

    def quantize(self, side: int, X):
        """X: float32 cuda tensor (rows x k), any row stride."""
        ptr, ld = _mat(X, "float32", self.device, "X", self.side_rows(side), self.k)
        _check(self.lib.lrqmm_quantize(self.h, side, ptr, ld), "lrqmm_quantize")

    def quantize_im2col(self, side: int, X, kh: int, kw: int, stride=1, pad=0, dilation=1):
        """X: float32 cuda tensor [batch, H, W, C] (NHWC, dense); the side's matrix is its im2col
        (rows (b, ho, wo), columns (i, j, c)) without materialising it."""
        st = stride if isinstance(stride, tuple) else (stride, stride)
        pd = pad if isinstance(pad, tuple) else (pad, pad)
        dl = dilation if isinstance(dilation, tuple) else (dilation, dilation)
        if X.dim() != 4 or not X.is_contiguous():
            raise ValueError("X: expected a contiguous 4-D NHWC tensor")
        g = ConvGeom(X.shape[0], X.shape[1], X.shape[2], X.shape[3], kh, kw, st[0], st[1], pd[0], pd[1], dl[0], dl[1])
        _check(self.lib.lrqmm_quantize_im2col(self.h, side, _arg(X, "float32", self.device, "X"), ctypes.byref(g)),
               "lrqmm_quantize_im2col")

    def rsvd_residual(self, omega_a, omega_b=None):
        """omega_b None: static-B mode (B's factors from rsvd_residual_b / the last full call)."""
        pa, lda = _mat(omega_a, "float32", self.device, "omega_a", self.k, self.kk)
        pb, ldb = _mat(omega_b, "float32", self.device, "omega_b", self.k, self.kk)
        if omega_b is not None and ldb != lda:
            raise ValueError("omega_a and omega_b must share one row stride")
        _check(self.lib.lrqmm_rsvd_residual(self.h, pa, pb, lda), "lrqmm_rsvd_residual")

    def rsvd_residual_b(self, omega_b):
        """Static-B preparation: B's RSVD once, resident until B is quantized again."""
        pb, ldb = _mat(omega_b, "float32", self.device, "omega_b", self.k, self.kk)
        _check(self.lib.lrqmm_rsvd_residual_b(self.h, pb, ldb), "lrqmm_rsvd_residual_b")

    def gemm(self, D, alpha: float = 1.0, beta: float = 0.0):
        ptr, ld = _mat(D, "float32", self.device, "D", self.m, self.n)
        _check(self.lib.lrqmm_gemm(self.h, alpha, beta, ptr, ld), "lrqmm_gemm")
        return D

    def close(self):
        if getattr(self, "h", None):
            self.lib.lrqmm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- inspection ----
    def sync(self):
        _check(self.lib.lrqmm_sync(self.h), "lrqmm_sync")

    def gemm_int32(self, C):
        ptr, ld = _mat(C, "int32", self.device, "C", self.m, self.n)
        _check(self.lib.lrqmm_gemm_int32(self.h, ptr, ld), "lrqmm_gemm_int32")
        return C

    def _getter(self, call):
        """Run a getter that writes freshly allocated tensors on the handle stream.  The tensors come
        from the caller's current stream (the caching allocator may hand out memory that stream still
        uses) and are read there afterwards, so when the handle has a stream of its own both orderings
        are enforced: handle stream after the current one, current one after the copy."""
        import torch

        cur = torch.cuda.current_stream(self.device)
        other = self.stream is not None and self.stream != cur
        if other:
            self.stream.wait_stream(cur)
        call()
        if other:
            cur.wait_stream(self.stream)

    def codes(self, side: int):
        import torch

        rows = self.side_rows(side)
        out = torch.empty((rows, self.k), dtype=torch.int8, device=f"cuda:{self.device}")
        self._getter(lambda: _check(self.lib.lrqmm_get_codes(self.h, side, _ptr(out), self.k), "lrqmm_get_codes"))
        return out

    def scales(self, side: int):
        import torch

        rows = self.side_rows(side)
        out = torch.empty((rows,), dtype=torch.float32, device=f"cuda:{self.device}")
        self._getter(lambda: _check(self.lib.lrqmm_get_scales(self.h, side, _ptr(out)), "lrqmm_get_scales"))
        return out

    def factors(self, side: int):
        import torch

        rows = self.side_rows(side)
        us = torch.empty((rows, self.rank), dtype=torch.float32, device=f"cuda:{self.device}")
        v = torch.empty((self.k, self.rank), dtype=torch.float32, device=f"cuda:{self.device}")
        self._getter(lambda: _check(self.lib.lrqmm_get_factors(self.h, side, _ptr(us), _ptr(v)), "lrqmm_get_factors"))
        return us, v

    def correction(self, side: int):
        import torch

        rows = self.side_rows(side)
        w = self.lib.lrqmm_correction_width(self.h)
        out = torch.empty((rows, w), dtype=torch.float32, device=f"cuda:{self.device}")
        self._getter(lambda: _check(self.lib.lrqmm_get_correction(self.h, side, _ptr(out)), "lrqmm_get_correction"))
        return out

    def timings_us(self):
        arr = (ctypes.c_double * 8)()
        _check(self.lib.lrqmm_get_timings(self.h, arr), "lrqmm_get_timings")
        return dict(quantize_a=arr[0], quantize_b=arr[1], rsvd=arr[2], gemm=arr[3])

    def launch_count(self, reset: bool = False) -> int:
        return int(self.lib.lrqmm_launch_count(self.h, 1 if reset else 0))

    # ---- end to end from host buffers ----
    def _host_args(self, A, Bt, omega_a, omega_b, D):
        if D is None:
            raise ValueError("D: a host output array is required")
        return (_host(A, "A", (self.m, self.k)), _host(Bt, "Bt", (self.side_rows(SIDE_B), self.k)),
                _host(omega_a, "omega_a", (self.k, self.kk)), _host(omega_b, "omega_b", (self.k, self.kk)))

    def run_host(self, A: np.ndarray, Bt: np.ndarray, omega_a: np.ndarray | None, omega_b: np.ndarray | None,
                 D: np.ndarray, alpha: float = 1.0):
        """All arrays C-contiguous float32 host arrays of the exact shapes (pinned memory recommended)."""
        _check(self.lib.lrqmm_run_host(self.h, *self._host_args(A, Bt, omega_a, omega_b, D), alpha,
                                       _host(D, "D", (self.m, self.n))), "lrqmm_run_host")
        return D

    def run_host_async(self, A: np.ndarray, Bt: np.ndarray, omega_a: np.ndarray | None,
                       omega_b: np.ndarray | None, D: np.ndarray, alpha: float = 1.0):
        """Enqueue one call (pinned host arrays, valid until sync()); copies overlap across calls."""
        _check(self.lib.lrqmm_run_host_async(self.h, *self._host_args(A, Bt, omega_a, omega_b, D), alpha,
                                             _host(D, "D", (self.m, self.n))), "lrqmm_run_host_async")
        return D


def lrqmm_matmul(A, Bt, omega_a=None, omega_b=None, bits: int = 4, rank: int = 16, oversample: int = 5,
                 power_iters: int = 1, rounding: str = "floor", granularity: str = "row",
                 alpha: float = 1.0, beta: float = 0.0, D=None):
    """One-shot D = alpha * LRQMM(A, B) + beta * D on the GPU (A: m x k, Bt: n x k, cuda fp32)."""
    import torch

    m, k = A.shape
    n = Bt.shape[0]
    with Lrqmm(m, n, k, bits, rank, oversample, power_iters, rounding, granularity, device=A.device.index or 0) as h:
        h.quantize(SIDE_A, A)
        h.quantize(SIDE_B, Bt)
        if rank > 0:
            h.rsvd_residual(omega_a, omega_b)
        if D is None:
            D = torch.empty((m, n), dtype=torch.float32, device=A.device)
        h.gemm(D, alpha, beta)
        h.sync()
    return D
