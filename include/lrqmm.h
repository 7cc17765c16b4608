/* lrqmm.h — C ABI of liblrqmm, the B200 (sm_100a) hot path of LRQMM
 * ("A method of using RSVD in residual calculation of LowBit GEMM",
 *  arXiv 2409.18772; cited as PAPER.md:<line> with the LaTeX label).
 *
 * The library computes Algorithm 2:
 *      D = alpha * ( C_F + RC1 + RC2 + RC3 ) + beta * D
 *   C_F  = (A_int B_int) / (lambda_A lambda_B)           Eq. INTGEMM / QUANTGEMM
 *   RC1  = U~ (V_r^T B_F), RC2 = (A_F W_r) Z~', RC3 = (U~ (V_r^T W_r)) Z~'
 * with symmetric N-bit quantization (Eq. quantA), one scale per
 * row of A and per column of B ("vector-wise"), floor rounding so the
 * residual is non-negative (Eq. get_ra2), and a randomized SVD of
 * each residual (Algorithm 1) with q power iterations.
 *
 * Conventions (all calls):
 *  - Pointers are DEVICE pointers on cfg.device unless stated "host".
 *  - Matrices are row-major with an explicit leading dimension in ELEMENTS (ld >= cols).
 *    A is M x K.  B (K x N) is passed TRANSPOSED as B^T (N x K), so both operands are
 *    K-major and "per column of B" is "per row of B^T".  D is M x N.
 *  - Every call only ENQUEUES work on cfg.stream (stream-ordered, no host sync) unless
 *    documented otherwise.  Arguments are validated synchronously on the host: an
 *    invalid call returns an error status and enqueues nothing.
 *  - CUDA/NCCL failures are sticky in the handle and are returned by the next call.
 *    Non-finite input detected on the device (reading #7) is returned as
 *    LRQMM_ERR_NONFINITE by lrqmm_sync / lrqmm_get_timings.
 *  - Ownership: the caller owns X, Omega and D; the handle owns codes, scales, RSVD
 *    factors and all scratch (allocated in lrqmm_create, freed in lrqmm_destroy).
 *  - A handle is used by one host thread at a time; distinct handles are independent.
 *  - Call order: create -> quantize(A), quantize(B) -> rsvd_residual (if rank > 0)
 *    -> gemm; repeatable.  Out-of-order calls return LRQMM_ERR_STATE.
 */
#ifndef LRQMM_H_
#define LRQMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lrqmm_handle_s* lrqmm_handle_t;

typedef enum {
  LRQMM_OK = 0,
  LRQMM_ERR_INVALID_ARGUMENT = 1, /* null pointer, bad enum, ld < cols */
  LRQMM_ERR_SHAPE = 2,            /* negative / inconsistent sizes */
  LRQMM_ERR_RANK = 3,             /* r + p > min(rows, K) of a side or > 64 */
  LRQMM_ERR_OVERFLOW = 4,         /* K * qmax^2 > 2^31 - 1: int32 accumulation would not be exact */
  LRQMM_ERR_NONFINITE = 5,        /* NaN/Inf in A or B (reading #7) */
  LRQMM_ERR_STATE = 6,            /* call out of order */
  LRQMM_ERR_CUDA = 7,
  LRQMM_ERR_NCCL = 8,
  LRQMM_ERR_ALLOC = 9,
  LRQMM_ERR_UNSUPPORTED = 10      /* e.g. power_iters < 0, bits not in {4, 8}, not an sm_100 device */
} lrqmm_status_t;

typedef enum { LRQMM_SIDE_A = 0, LRQMM_SIDE_B = 1 } lrqmm_side_t;

typedef enum {
  LRQMM_ROUND_FLOOR = 0,   /* LRQMM: floor(lambda*x), Eq. get_ra2 */
  LRQMM_ROUND_TRUNC = 1,   /* paper's Direct Quant: TypeCast of Eq. quantA, reading #2 */
  LRQMM_ROUND_NEAREST = 2  /* round half to even, Eq. quantAB */
} lrqmm_round_t;

typedef enum {
  LRQMM_SCALE_PER_ROW = 0,   /* one lambda per row of A and per column of B */
  LRQMM_SCALE_PER_TENSOR = 1 /* one lambda per operand (Eq. quantA as printed) */
} lrqmm_gran_t;

typedef struct {
  int64_t m;       /* rows of A held by this rank (the row shard when world_size > 1) */
  int64_t n;       /* columns of B (rows of B^T) */
  int64_t k;       /* inner dimension */
  int bits;        /* N of Eq. quantA: 4 or 8; codes in [-qmax, qmax], qmax = 2^(N-1)-1, stored as int8 */
  int rank;        /* r >= 0; 0 = direct quantization (no residual correction) */
  int oversample;  /* p >= 0; sketch width k = r + p <= 64 */
  int power_iters; /* q >= 0: power iterations of the range finder (reading #10: q = 1 for LRQMM's accuracy).
                      q = 0 is Algorithm 1 on the sampled basis Q = orth(R Omega) (two passes over R plus a
                      codes-only pass; reading #30) -- with a structured sketch whose first column is all ones
                      it matches q = 1's accuracy, a labelled variant */
  int rounding;    /* lrqmm_round_t */
  int granularity; /* lrqmm_gran_t */
  int world_size;  /* >= 1; ranks that row-shard A */
  int world_rank;
  const unsigned char* nccl_unique_id; /* host, 128 bytes from lrqmm_get_unique_id on rank 0; NULL if world_size == 1 */
  int device;      /* CUDA device ordinal */
  void* stream;    /* cudaStream_t (NULL = legacy default stream) */
  int enable_timing; /* record per-phase CUDA events (lrqmm_get_timings) */
  int qt_terms;      /* 0, or QuantTensor compensation instead of LRQMM (requires rank == 0): 3 = QT(1,1,0),
                        4 = QT(1,1,1) of Eq. gemm_r_split.  quantize then also re-quantizes
                        the fp32 residual fp32(x - code/lambda) with its own scales (same bits, rounding,
                        granularity; the paper's QT columns use trunc + per-tensor, reading #27) and
                        gemm returns alpha (A_q B_q + A_q R_Bq + R_Aq B_q [+ R_Aq R_Bq]) + beta D */
  int b_sharded;     /* 0: every rank holds all of B^T (n rows).  1 (world_size > 1): B is column-sharded
                        (SURVEY §8(e)(ii)): rank i holds rows [i*nb, min(n, (i+1)*nb)) of B^T, nb = ceil(n /
                        world_size), and quantize(SIDE_B) takes that shard; B's RSVD reduces its Gram matrices
                        and Z_B across ranks like A's, and the B codes, scales and correction factor L_B are
                        allgathered (in place, NCCL) so that every rank's GEMM covers all n columns.  The
                        inspection calls return this rank's rows of B.  Not with qt_terms. */
} lrqmm_config_t;

/* Host.  128-byte NCCL unique id for a world_size > 1 communicator (call on rank 0,
 * broadcast to the other ranks out of band, e.g. with torch.distributed). */
lrqmm_status_t lrqmm_get_unique_id(unsigned char out[128]);

/* Host.  Validates cfg, allocates all device workspace (codes M x Kp and N x Kp int8 with
 * Kp = roundup(K,16), scales, RSVD panels, correction factors), builds the NCCL
 * communicator when world_size > 1 (collective across ranks).  Errors: INVALID_ARGUMENT,
 * SHAPE, RANK, OVERFLOW, UNSUPPORTED, ALLOC, CUDA, NCCL. */
lrqmm_status_t lrqmm_create(const lrqmm_config_t* cfg, lrqmm_handle_t* out);

/* Quantize one operand: X is A (m x k, ld ldx) or B^T (n x k, ld ldx), fp32, any alignment.
 * Eq. quantA with lambda_i = RN32(qmax / max_j |x_ij|) (lambda = 1 for a zero row),
 * codes = clamp(round_mode(lambda_i * x_ij), -qmax, qmax) decided on the exact product
 * (Alg. 2).  When rank > 0 the same pass also stores the residual
 * fraction u = lambda x - code (R = u / lambda, Alg. 2) in a handle-owned
 * buffer, so X is not referenced after this call's work completes in stream order. */
lrqmm_status_t lrqmm_quantize(lrqmm_handle_t h, lrqmm_side_t side, const float* X, int64_t ldx);

/* Convolution geometry for lrqmm_quantize_im2col (NHWC input, square or rectangular windows). */
typedef struct {
  int64_t batch;
  int H, W, C;             /* input height, width, channels */
  int kh, kw;              /* window */
  int stride_h, stride_w;  /* >= 1 */
  int pad_h, pad_w;        /* >= 0, zero padding */
  int dil_h, dil_w;        /* >= 1 */
} lrqmm_conv_t;

/* Implicit-im2col quantization: the same as lrqmm_quantize on the im2col matrix
 * of a convolution, without materialising it.  X (device, fp32) is the NHWC input
 * [batch][H][W][C], dense; the side's matrix has rows r = (b, ho, wo) in that order (Ho = (H + 2 pad_h
 * - dil_h (kh - 1) - 1) / stride_h + 1, likewise Wo) and columns k = (i kw + j) C + c, element
 * X[b][ho stride_h - pad_h + i dil_h][wo stride_w - pad_w + j dil_w][c] (0 outside the image).  The
 * weights passed as the other side must use the same k order (B^T row = one output channel,
 * [kh][kw][C] flattened).  Codes, lambda and residual planes are bit-identical to lrqmm_quantize of
 * the explicit matrix.  Errors: LRQMM_ERR_SHAPE if batch Ho Wo != the side's rows or kh kw C != k;
 * LRQMM_ERR_INVALID_ARGUMENT for a null X or a bad geometry; LRQMM_ERR_UNSUPPORTED with per-tensor
 * scales or qt_terms.  Stream-ordered like lrqmm_quantize. */
lrqmm_status_t lrqmm_quantize_im2col(lrqmm_handle_t h, lrqmm_side_t side, const float* X, const lrqmm_conv_t* conv);

/* RSVD of both residuals (Alg. 2) and assembly of the
 * correction factors L_A = [U_A S_A | A_F V_B], L_B = [B_F^T V_A + U_B S_B (V_B^T V_A) | U_B S_B]
 * (Alg. 2).  omegaA / omegaB: k x (r+p) fp32 sketches (ld ldo >= r+p), the
 * Gaussian test matrices of Algorithm 1, supplied by the caller so that a
 * CPU reference can use the same draws.  Requires rank > 0 and both sides quantized.
 * Static-B (weight-resident) mode: omegaB == NULL reuses B's RSVD factors computed by
 * lrqmm_rsvd_residual_b (or by the last full call for the same quantized B) and runs only the
 * A side plus the one A-dependent B term B_F^T V_A (a pass over B's codes); the result is the
 * same correction as a full call with that omegaB.  STATE if B's factors are not resident.
 * Repeated calls on a handle are replayed from a CUDA graph captured on the second call. */
lrqmm_status_t lrqmm_rsvd_residual(lrqmm_handle_t h, const float* omegaA, const float* omegaB, int64_t ldo);

/* Static-B preparation: RSVD of B's residual only (range finder, W_B = R_B Q1_B, truncation),
 * kept resident in the handle until B is quantized again.  omegaB as above.  Requires rank > 0
 * and B quantized.  SURVEY §8(f) f2 ("B broadcast once" / weights deployment). */
lrqmm_status_t lrqmm_rsvd_residual_b(lrqmm_handle_t h, const float* omegaB, int64_t ldo);

/* D = alpha * (C_int / (lambda_A lambda_B) + L_A L_B^T) + beta * D  (Alg. 2,
 * 369, 372), one tcgen05 int8 GEMM with the correction in its epilogue.  D is m x n (ld ldd);
 * when beta == 0, D is not read.  With rank == 0 this is direct quantization. */
lrqmm_status_t lrqmm_gemm(lrqmm_handle_t h, float alpha, float beta, float* D, int64_t ldd);

/* Host.  Frees everything (collective when world_size > 1).  NULL is accepted. */
lrqmm_status_t lrqmm_destroy(lrqmm_handle_t h);

/* Host.  Synchronises the handle stream; returns the first sticky error (CUDA, NCCL,
 * NONFINITE) or LRQMM_OK. */
lrqmm_status_t lrqmm_sync(lrqmm_handle_t h);

/* ---- end-to-end convenience (HOST buffers) -------------------------------------
 * Copies A (m x k), B^T (n x k), omegaA, omegaB (k x (r+p)) from HOST memory (pinned for
 * overlap) into handle-owned device buffers, runs quantize(A), quantize(B), rsvd_residual,
 * gemm(alpha, 0) and copies D (m x n) back to HOST.  All leading dimensions are dense.
 * Synchronises before returning. */
lrqmm_status_t lrqmm_run_host(lrqmm_handle_t h, const float* A_host, const float* Bt_host, const float* omegaA_host,
                              const float* omegaB_host, float alpha, float* D_host);

/* Asynchronous form of lrqmm_run_host for a stream of calls: returns once the work is enqueued.
 * Inputs are staged through two device slots on a copy-in stream and D leaves through a copy-out
 * stream, so the host->device copy of call i+1 and the device->host copy of call i overlap each
 * other and the compute (PCIe is full duplex).  Host buffers must be pinned and must stay valid
 * (inputs unmodified, D unread) until lrqmm_sync, which waits for all three streams.  The
 * quantize / RSVD / GEMM work stays in call order on the handle stream. */
lrqmm_status_t lrqmm_run_host_async(lrqmm_handle_t h, const float* A_host, const float* Bt_host,
                                    const float* omegaA_host, const float* omegaB_host, float alpha, float* D_host);

/* ---- inspection (parity tests); async device-to-device copies on the handle stream ---- */
/* codes of a side: rows x k int8 into dst (ld >= k) */
lrqmm_status_t lrqmm_get_codes(lrqmm_handle_t h, lrqmm_side_t side, signed char* dst, int64_t ld);
/* scales lambda of a side: rows fp32 */
lrqmm_status_t lrqmm_get_scales(lrqmm_handle_t h, lrqmm_side_t side, float* lambda);
/* bare int32 accumulators C_int = A_int B_int (Eq. INTGEMM), m x n into Cint (ld ldc): the
 * same tcgen05 kernel with an int32 epilogue (the "bare GEMM" of every overhead number). */
lrqmm_status_t lrqmm_gemm_int32(lrqmm_handle_t h, int32_t* Cint, int64_t ldc);
/* RSVD factors of a side after rsvd_residual: USigma (rows x r, dense) and V (k x r, dense)
 * with R_side ~= USigma V^T (R_B^T for side B). */
lrqmm_status_t lrqmm_get_factors(lrqmm_handle_t h, lrqmm_side_t side, float* USigma, float* V);
/* correction factors L_A (m x w) or L_B (n x w), w = lrqmm_correction_width(h) */
lrqmm_status_t lrqmm_get_correction(lrqmm_handle_t h, lrqmm_side_t side, float* L);
int lrqmm_correction_width(lrqmm_handle_t h);
/* Host.  Per-phase device times in microseconds of the last calls (needs enable_timing):
 * us[0] quantize A, us[1] quantize B, us[2] rsvd_residual, us[3] gemm, us[4..7] 0.
 * Synchronises the stream. */
lrqmm_status_t lrqmm_get_timings(lrqmm_handle_t h, double us[8]);
/* Host.  Number of kernel launches the library enqueued since create (or the last reset). */
int64_t lrqmm_launch_count(lrqmm_handle_t h, int reset);

const char* lrqmm_status_string(lrqmm_status_t s);

#ifdef __cplusplus
}
#endif
#endif /* LRQMM_H_ */
