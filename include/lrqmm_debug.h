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

/* GEMM kernel selection for later calls in this process: 0 = automatic (CTA-pair kernel K7 for
 * M, N >= 512 and >= 512 256x256 tiles; otherwise the one-CTA K8 with the tensor-core correction when
 * rank > 0, K6 when rank == 0), 1 = one-CTA K6 with the FFMA correction epilogue, 2 = CTA-pair K7,
 * 3 = K8 (rank > 0).  Lets the tests run every kernel on the same shapes.  INVALID_ARGUMENT for
 * other values. */
lrqmm_status_t lrqmm_debug_set_gemm_variant(int variant);

/* Small solvers (K4) on Y (n x W):
 *   op 0: G = Y^T Y (fp64, W x W)
 *   op 1: G = Y^T Y, T = orthonormalising transform (Y T has orthonormal columns)
 *   op 2: G = Y^T Y, T[:, 0:r] = top-r eigenvectors of G (descending), rest 0
 *   op 3, 4: as ops 1, 2 through the fused Gram + solve kernel the RSVD runs        */
lrqmm_status_t lrqmm_debug_small(int op, const float* Y, int64_t n, int W, int r, double* G, float* T, void* stream);

/* Test transport for the row-sharded path on ONE GPU: creates a handle exactly
 * like lrqmm_create (cfg.world_size > 1, cfg.world_rank, cfg.b_sharded as documented there;
 * cfg.nccl_unique_id is ignored) whose collectives -- the fp64 Gram and Z allreduces and the B
 * allgathers -- run over a process-local "loopback" group instead of NCCL: every rank of `group`
 * is a handle of this process on the same cfg.device, driven by its own host thread (and stream).
 * Each collective synchronises the rank's stream, meets the other ranks at a host barrier (120 s
 * timeout -> LRQMM_ERR_NCCL, sticky), sums / copies the peers' buffers in rank order on its own
 * stream, and meets them again; no kernel waits on another rank.  The sharded schedule, buffers
 * and kernels are the product's; only the transport differs.  Multi-rank loopback handles run
 * the RSVD eagerly (no CUDA graph).  Errors: as lrqmm_create; INVALID_ARGUMENT if the group
 * already holds world_size handles or another world_size / device. */
/* GPU negative control: makes later calls in this process run with a deliberate defect that the
 * parity tests must detect (tests/test_gpu_negative_control.py): 1 = the other rounding mode in K1
 * (floor <-> nearest), 2 = lambda of row 0 one ulp off after each quantize, 3 = the GEMM epilogue
 * without the low-rank correction (D = direct quantization), 4 = the RC3 core V_B^T V_A zeroed in the
 * factor assembly (Alg. 2 line 366 dropped).  0 restores the product path.  INVALID_ARGUMENT
 * otherwise. */
lrqmm_status_t lrqmm_debug_inject_fault(int kind);

/* Timing trace of the fused RSVD passes (handles created with LRQMM_FUSE_TRACE=1 in the environment):
 * per pass slot i < 8 (in launch order since the last read), out[8 i + 0] = first CTA start,
 * [8 i + 1] = last CTA done with its units, [8 i + 2] / [8 i + 3] = solver start / end, [8 i + 4] =
 * first CTA done, globaltimer nanoseconds.  Synchronises the stream and re-arms the trace.
 * LRQMM_ERR_STATE if the handle has no trace. */
lrqmm_status_t lrqmm_debug_fuse_trace(lrqmm_handle_t h, int64_t out[64]);

lrqmm_status_t lrqmm_debug_create_loopback(const lrqmm_config_t* cfg, int group, lrqmm_handle_t* out);

#ifdef __cplusplus
}
#endif
#endif
