// Host-side launch interfaces of the liblrqmm kernels (internal; not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lrqmm {

// number of kernels this library has launched (gpu_launches evidence for the bench)
inline int64_t& launch_counter() {
  static int64_t c = 0;
  return c;
}

enum { kRoundFloor = 0, kRoundTrunc = 1, kRoundNearest = 2 };

// ---------------------------------------------------------------- K1 quantize
struct QuantArgs {
  const float* X;
  int64_t ldx;
  int64_t rows;
  int K, Kp, qmax, mode;
  int8_t* codes;          // rows x Kp
  float* lam;             // rows (written unless lam_fixed)
  const float* lam_fixed; // device scalar (per-tensor mode) or nullptr
  int* err_flag;          // bit 0: non-finite input
};
void launch_quantize(const QuantArgs& a, cudaStream_t st);
void launch_tensor_scale(const float* X, int64_t ldx, int64_t rows, int K, int qmax, float* row_amax,
                         float* lam_rows, float* lam_scalar, int* err_flag, cudaStream_t st);

// ------------------------------------------------- K2/K3 skinny residual products
// F(x_ij) is recomputed from X and lambda_i (never stored):
//   residual  r = (lambda*x - code)/lambda            (Alg. 2)
//   dequant   x~ = code / lambda                      (Alg. 2)
enum { kFRes = 0, kFDeq = 1 };
struct SideView {
  const float* X;
  int64_t ldx;
  int64_t rows;
  int K;
  const float* lam;
  int qmax, mode;
};
// OUT1[i,c] = sum_j F1(x_ij) P1[j,c]  (and optionally OUT2 with F2/P2), c < W.
// P is K x W (ld W), OUT is rows x W (ld W).  Deterministic split-K with partial buffer.
void launch_proj_rows(const SideView& s, const float* P1, int f1, float* OUT1, const float* P2, int f2, float* OUT2,
                      int W, float* partial, int64_t partial_elems, cudaStream_t st);
// OUT[j,c] = sum_i F(x_ij) P[i,c]: P is rows x W, OUT is K x W.
void launch_proj_cols(const SideView& s, const float* P, int f, float* OUT, int W, float* partial,
                      int64_t partial_elems, cudaStream_t st);

// G = Y1^T Y2 (W x W, fp64) over n rows; Y ld W.  Deterministic 2-stage.
void launch_gram(const float* Y1, const float* Y2, int64_t n, int W, double* G, double* partial, int64_t partial_elems,
                 cudaStream_t st);
// OUT[i, col0 + o] = sum_c IN1[i,c] S1[c,o] (+ sum_c IN2[i,c] S2[c,o]), o < nout; IN ld W, S ld ldS, OUT ld ldo
void launch_apply_small(const float* IN1, const float* S1, const float* IN2, const float* S2, int64_t n, int W,
                        int ldS, int nout, float* OUT, int64_t ldo, int col0, cudaStream_t st);

// ----------------------------------------------------------- K4 small solvers
// For each of nsides problems: G (n x n fp64, symmetric) -> Jacobi eigendecomposition.
//   mode ORTH : T[n x n] = V diag(keep ? lambda^-1/2 : 0), keep: lambda >= rtol2 * lambda_max
//   mode TRUNC: T[n x n] = first r columns = top-r eigenvectors (descending), rest 0
enum { kEigOrth = 0, kEigTrunc = 1 };
struct EigJob {
  const double* G;
  float* T;
  int mode;
  int r;
};
void launch_eig(const EigJob* jobs, int njobs, int n, cudaStream_t st);
// Mab[r x r] = VWb^T C VWa  and  VWbM[n x r] = VWb Mab   (C = Q1_B^T Q1_A, n x n fp64)
void launch_cross_small(const double* C, const float* VWa, const float* VWb, int n, int r, float* VWbM,
                        cudaStream_t st);

// --------------------------------------------------------------- K6 int GEMM
struct GemmArgs {
  const int8_t* A;  // M x Kp
  const int8_t* B;  // N x Kp (B^T)
  int64_t M, N;
  int Kp;
  // epilogue
  int epi;               // 0: int32 out; 1: fp32 LRQMM/DQ out
  const float* lam_a;    // M
  const float* lam_b;    // N
  const float* LA;       // M x R2 (may be null if R2 == 0)
  const float* LB;       // N x R2
  int R2;                // padded correction width roundup(2r, 8) <= 64
  float alpha, beta;
  float* D;              // M x N (ldd)
  int32_t* Cint;         // M x N (ldd)
  int64_t ldd;
};
int gemm_prepare_maps(const GemmArgs& g, void* mapA, void* mapB);  // returns 0 on success
void launch_gemm(const GemmArgs& g, const void* mapA, const void* mapB, cudaStream_t st);

}  // namespace lrqmm
