"""The C-ABI library loads and exports every symbol include/lrqmm.h declares;
host-side validation (no compute, no GPU needed)."""
import ctypes
import os
import re

import pytest

from paper_2409_18772_b200 import lrqmm as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols(name="lrqmm.h"):
    txt = open(os.path.join(ROOT, "include", name)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lrqmm_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2409_18772_b200.build import build

    build()
    return L.load_library()


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(L.EXPORTS) == syms
    dbg = header_symbols("lrqmm_debug.h")
    assert sorted(L.DEBUG_EXPORTS) == dbg
    for s in dbg:
        assert hasattr(lib, s), s


def test_status_strings(lib):
    assert lib.lrqmm_status_string(0) == b"ok"
    assert b"int32" in lib.lrqmm_status_string(4)


def _cfg(**kw):
    base = dict(m=64, n=64, k=64, bits=4, rank=4, oversample=2, power_iters=1, rounding=0, granularity=0,
                world_size=1, world_rank=0, nccl_unique_id=None, device=0, stream=None, enable_timing=0)
    base.update(kw)
    return L.Config(**base)


@pytest.mark.parametrize("kw,code", [
    (dict(bits=5), 10),                       # bits not in {4, 8}
    (dict(bits=8, k=133145), 4),              # K * 127^2 > 2^31 - 1 (reading #24)
    (dict(m=-1), 2),
    (dict(rank=40, oversample=30), 3),        # r + p > 64
    (dict(rank=60, oversample=10, k=32), 3),  # r + p > K
    (dict(power_iters=-1), 10),               # q >= 0 required (readings #10, #30)
    (dict(rounding=7), 1),
    (dict(world_size=2, world_rank=0), 1),    # multi-rank needs a unique id
    (dict(b_sharded=2), 1),                   # b_sharded is 0 or 1
    (dict(rank=0, qt_terms=3, b_sharded=1, world_size=2,
          nccl_unique_id=ctypes.cast(ctypes.create_string_buffer(128), ctypes.c_void_p)), 10),  # QT not B-sharded
])
def test_create_validates_on_host(lib, kw, code):
    h = ctypes.c_void_p()
    cfg = _cfg(**kw)
    assert lib.lrqmm_create(ctypes.byref(cfg), ctypes.byref(h)) == code
    assert not h.value


def test_overflow_boundary_int8(lib):
    # K = 133144 is the largest exact int8 K: 133144 * 127^2 = 2147475544 <= 2^31 - 1
    assert 133144 * 127 * 127 <= 2 ** 31 - 1 < 133145 * 127 * 127


def test_null_handle_calls_fail_cleanly(lib):
    assert lib.lrqmm_quantize(None, 0, None, 0) == 1
    assert lib.lrqmm_gemm(None, 1.0, 0.0, None, 0) == 1
    assert lib.lrqmm_destroy(None) == 0
