"""Test infrastructure: the fp64 CPU oracle of LRQMM.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package; the product path never does."""
from .lrqmm_oracle import *  # noqa: F401,F403
from .lrqmm_oracle import (compute_scale, quantize, dequantize, residual, int_gemm,  # noqa: F401
                           dequant_result, orth, rsvd, rsvd_spec_variant, lrqmm,
                           direct_quant, qt_gemm, matmul_exact, relative_error,
                           frobenius_norm, qmax_of)
