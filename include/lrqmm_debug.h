/* lrqmm_debug.h — test hooks of liblrqmm: run ONE internal kernel stage on caller
 * buffers so that tests/ can check it in isolation against NumPy.  Not part of the
 * product API; every call synchronises the stream and returns the CUDA status.
 * All pointers are device pointers; row-major; fp32 unless stated. */
#ifndef LRQMM_DEBUG_H_
#define LRQMM_DEBUG_H_

#include <stdint.h>

#include "lrqmm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Skinny residual products of the RSVD (K2/K3) of a side X: rows x K (ld ldx), quantized
 * per row by K1 (bits, rounding) inside the call:
 *   mode 0: OUT  = R P            (P: K x W, OUT: rows x W)
 *   mode 1: OUT  = R^T P          (P: rows x W, OUT: K x W)
 *   mode 2: OUT  = R P, OUT2 = X~ P2  (dual pass; X~ = code / lambda)
 * with R = X - code/lambda, code = clamp(round_mode(lambda x)) (Alg. 2). */
lrqmm_status_t lrqmm_debug_proj(int mode, const float* X, int64_t ldx, int64_t rows, int K, int bits, int rounding,
                                const float* P, const float* P2, int W, float* OUT, float* OUT2, void* stream);

/* GEMM kernel selection for later calls in this process: 0 = automatic (CTA-pair kernel for
 * M, N >= 512 and >= 512 256x256 tiles), 1 = one-CTA kernel (K6), 2 = CTA-pair kernel (K7).  Lets the tests run both
 * kernels on the same shapes.  Returns INVALID_ARGUMENT for other values. */
lrqmm_status_t lrqmm_debug_set_gemm_variant(int variant);

/* Small solvers (K4) on Y (n x W):
 *   op 0: G = Y^T Y (fp64, W x W)
 *   op 1: G = Y^T Y, T = orthonormalising transform (Y T has orthonormal columns)
 *   op 2: G = Y^T Y, T[:, 0:r] = top-r eigenvectors of G (descending), rest 0
 *   op 3, 4: as ops 1, 2 through the fused Gram + solve kernel the RSVD runs        */
lrqmm_status_t lrqmm_debug_small(int op, const float* Y, int64_t n, int W, int r, double* G, float* T, void* stream);

#ifdef __cplusplus
}
#endif
#endif
