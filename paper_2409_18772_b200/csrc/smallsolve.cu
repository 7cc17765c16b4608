// K4 — one-CTA fp64 symmetric eigensolver (parallel cyclic Jacobi, round-robin
// pair ordering) for the k x k problems of the RSVD:
//   * orthonormalisation of a sketch Y (Algorithm 1 needs Q with "orthogonal
//     columns"): G = Y^T Y = V L V^T, Q = Y V L^-1/2 with the
//     reading-#12 threshold (drop sigma < 1e-5 sigma_max, i.e. l < 1e-10 l_max);
//   * truncation to rank r (SVD of the projected matrix, Algorithm 1 lines
//     139-140; best rank-r approximation, Eq. k-svd
//     PAPER.md:106-114): top-r eigenvectors of W^T W.
#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

constexpr int kMaxN = 64;

__global__ void __launch_bounds__(256) k_eig(const EigJob* __restrict__ jobs, int n) {
  extern __shared__ double dyn[];
  double (*A)[kMaxN + 1] = reinterpret_cast<double (*)[kMaxN + 1]>(dyn);
  double (*V)[kMaxN + 1] = reinterpret_cast<double (*)[kMaxN + 1]>(dyn + kMaxN * (kMaxN + 1));
  __shared__ double cs[kMaxN / 2], sn[kMaxN / 2];
  __shared__ int pp[kMaxN / 2], qq[kMaxN / 2];
  __shared__ double red[256];
  __shared__ int order[kMaxN];
  __shared__ double lam[kMaxN];
  __shared__ int stop;
  const EigJob job = jobs[blockIdx.x];
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += 256) {
    const int i = e / n, j = e % n;
    // symmetrise (the Gram is symmetric up to fp64 summation order)
    A[i][j] = 0.5 * (job.G[i * n + j] + job.G[j * n + i]);
    V[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = n / 2;
  for (int sweep = 0; sweep < 30; ++sweep) {
    // convergence test: off(A)^2 <= (1e-15)^2 * ||diag(A)||^2
    double off = 0.0, dg = 0.0;
    for (int e = tid; e < n * n; e += 256) {
      const int i = e / n, j = e % n;
      const double v = A[i][j] * A[i][j];
      if (i == j) dg += v; else off += v;
    }
    red[tid] = off;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    const double off_all = red[0];
    __syncthreads();
    red[tid] = dg;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    if (tid == 0) stop = (off_all <= 1e-30 * red[0]) || (off_all == 0.0);
    __syncthreads();
    if (stop) break;
    for (int step = 0; step < n - 1; ++step) {
      if (tid < half) {
        int p, q;
        if (tid == 0) {
          p = 0;
          q = (step % (n - 1)) + 1;
        } else {
          p = ((tid + step) % (n - 1)) + 1;
          q = ((n - 1 - tid + step) % (n - 1)) + 1;
        }
        if (p > q) { const int t = p; p = q; q = t; }
        const double apq = A[p][q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
          double t;
          if (fabs(theta) > 1e150) t = 0.5 / theta;
          else t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
        }
        pp[tid] = p; qq[tid] = q; cs[tid] = c; sn[tid] = s;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int e = tid; e < half * n; e += 256) {
        const int k = e / n, j = e % n;
        const int p = pp[k], q = qq[k];
        const double c = cs[k], s = sn[k];
        const double ap = A[p][j], aq = A[q][j];
        A[p][j] = c * ap - s * aq;
        A[q][j] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J, V <- V J
      for (int e = tid; e < half * n; e += 256) {
        const int k = e / n, i = e % n;
        const int p = pp[k], q = qq[k];
        const double c = cs[k], s = sn[k];
        const double ap = A[i][p], aq = A[i][q];
        A[i][p] = c * ap - s * aq;
        A[i][q] = s * ap + c * aq;
        const double vp = V[i][p], vq = V[i][q];
        V[i][p] = c * vp - s * vq;
        V[i][q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  // eigenvalues on the diagonal; order descending (stable on index)
  if (tid < n) lam[tid] = A[tid][tid];
  __syncthreads();
  if (tid < n) {
    int rank = 0;
    const double li = lam[tid];
    for (int j = 0; j < n; ++j) {
      const double lj = lam[j];
      rank += (lj > li) || (lj == li && j < tid);
    }
    order[rank] = tid;
  }
  __syncthreads();
  const double lmax = lam[order[0]];
  if (job.mode == kEigOrth) {
    for (int e = tid; e < n * n; e += 256) {
      const int a = e / n, o = e % n;  // output column o = o-th largest eigenpair
      const int idx = order[o];
      const double l = lam[idx];
      const bool keep = (lmax > 0.0) && (l >= 1e-10 * lmax);
      job.T[a * n + o] = keep ? (float)(V[a][idx] / sqrt(l)) : 0.f;
    }
  } else {
    for (int e = tid; e < n * n; e += 256) {
      const int a = e / n, o = e % n;
      job.T[a * n + o] = (o < job.r) ? (float)V[a][order[o]] : 0.f;
    }
  }
}

void launch_eig(const EigJob* jobs, int njobs, int n, cudaStream_t st) {
  constexpr int kSmem = 2 * kMaxN * (kMaxN + 1) * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  k_eig<<<njobs, 256, kSmem, st>>>(jobs, n); ++launch_counter();
}

// Mab = VWb^T C VWa (r x r), C = Q1_B^T Q1_A (n x n, fp64); VWbM = VWb Mab (n x r).
// V_B^T V_A = VWb^T Q1_B^T Q1_A VWa: the r x r core of RC3 (Alg. 2).
__global__ void __launch_bounds__(256) k_cross_small(const double* __restrict__ C, const float* __restrict__ VWa,
                                                     const float* __restrict__ VWb, int n, int r,
                                                     float* __restrict__ VWbM) {
  __shared__ double T1[kMaxN][kMaxN / 2];      // C VWa  (n x r), r <= 32
  __shared__ double M[kMaxN / 2][kMaxN / 2];   // r x r
  const int tid = threadIdx.x;
  for (int e = tid; e < n * r; e += 256) {
    const int i = e / r, o = e % r;
    double a = 0.0;
    for (int c = 0; c < n; ++c) a += C[i * n + c] * (double)VWa[c * n + o];
    T1[i][o] = a;
  }
  __syncthreads();
  for (int e = tid; e < r * r; e += 256) {
    const int u = e / r, o = e % r;
    double a = 0.0;
    for (int i = 0; i < n; ++i) a += (double)VWb[i * n + u] * T1[i][o];
    M[u][o] = a;
  }
  __syncthreads();
  for (int e = tid; e < n * r; e += 256) {
    const int i = e / r, o = e % r;
    double a = 0.0;
    for (int u = 0; u < r; ++u) a += (double)VWb[i * n + u] * M[u][o];
    VWbM[i * n + o] = (float)a;
  }
}

void launch_cross_small(const double* C, const float* VWa, const float* VWb, int n, int r, float* VWbM,
                        cudaStream_t st) {
  k_cross_small<<<1, 256, 0, st>>>(C, VWa, VWb, n, r, VWbM); ++launch_counter();
}

}  // namespace lrqmm
