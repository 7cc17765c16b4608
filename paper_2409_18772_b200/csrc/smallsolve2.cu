// K4 (fast path) — small dense kernels of the RSVD on W x W (W <= 64) problems.
//
//  k_gram      : G = Y1^T Y2 in fp64 over n rows, one launch: per-block partials,
//                the last block (ticket counter) sums them in a fixed order
//                (deterministic, no float atomics).  blockIdx.y = job.
//  k_chol_orth : orthonormalising transform of a sketch (Algorithm 1 needs Q with
//                "orthogonal columns") by pivoted Cholesky QR:
//                G[p,p] = L L^T, T[p(a), b] = (L^-T)[a, b]  so  Q = Y T.  Directions whose
//                pivot falls below 1e-10 x the largest diagonal entry (sigma < 1e-5 sigma_max,
//                reading #12) are dropped (zero columns of T).  One warp per job.
//  k_eig_warp  : symmetric Jacobi eigendecomposition for the rank-r truncation
//                (Algorithm 1, Eq. k-svd), one warp per job,
//                T = top-r eigenvectors in descending eigenvalue order.
#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

constexpr int kN = 64;

// ------------------------------------------------------------------- Gram
// One launch: each block loads its row range in chunks of kGramRows (one chunk unless n > 64K), then
// accumulates its W x W partial in fp64; the last block (ticket) sums the partials in a
// fixed order.  blockIdx.y = job.
constexpr int kGramRows = 64;
__global__ void __launch_bounds__(256) k_gram(GramJobs jobs, int W) {
  const GramJob jb = jobs.j[blockIdx.y];
  const int npairs = W * W;
  __shared__ float s1[kGramRows][kN + 1];
  __shared__ float s2[kGramRows][kN + 1];
  __shared__ int ticket;
  const int64_t rpb = (jb.n + gridDim.x - 1) / gridDim.x;
  const int64_t r_begin = (int64_t)blockIdx.x * rpb;
  const int64_t r_end = (jb.n < r_begin + rpb) ? jb.n : r_begin + rpb;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kGramRows) {
    const int nr = (int)(r_end - r0 < kGramRows ? r_end - r0 : kGramRows);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * W; e += 256) {
      const int i = e / W, c = e % W;
      s1[i][c] = __ldg(jb.Y1 + (r0 + i) * W + c);
      s2[i][c] = __ldg(jb.Y2 + (r0 + i) * W + c);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int pr = threadIdx.x + 256 * q;
      if (pr < npairs) {
        const int a = pr / W, c = pr % W;
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
        int i = 0;
        for (; i + 3 < nr; i += 4) {
          t0 = fma((double)s1[i][a], (double)s2[i][c], t0);
          t1 = fma((double)s1[i + 1][a], (double)s2[i + 1][c], t1);
          t2 = fma((double)s1[i + 2][a], (double)s2[i + 2][c], t2);
          t3 = fma((double)s1[i + 3][a], (double)s2[i + 3][c], t3);
        }
        for (; i < nr; ++i) t0 = fma((double)s1[i][a], (double)s2[i][c], t0);
        acc[q] += (t0 + t1) + (t2 + t3);
      }
    }
  }
  double* part = jb.partial + (int64_t)blockIdx.x * npairs;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int pr = threadIdx.x + 256 * q;
    if (pr < npairs) part[pr] = acc[q];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(jb.counter, 1);
  __syncthreads();
  if (ticket != (int)gridDim.x - 1) return;
  __threadfence();
  // fixed-order 4-way split sum over the block partials (independent loads in flight)
  const int nb = (int)gridDim.x;
  for (int pr = threadIdx.x; pr < npairs; pr += 256) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = 0;
    for (; b + 3 < nb; b += 4) {
      a0 += __ldcg(jb.partial + (int64_t)(b + 0) * npairs + pr);
      a1 += __ldcg(jb.partial + (int64_t)(b + 1) * npairs + pr);
      a2 += __ldcg(jb.partial + (int64_t)(b + 2) * npairs + pr);
      a3 += __ldcg(jb.partial + (int64_t)(b + 3) * npairs + pr);
    }
    for (; b < nb; ++b) a0 += __ldcg(jb.partial + (int64_t)b * npairs + pr);
    jb.G[pr] = (a0 + a1) + (a2 + a3);
  }
  if (threadIdx.x == 0) *jb.counter = 0;  // re-arm for the next launch (stream ordered)
}

void launch_gram_jobs(const GramJobs& jobs, int W, cudaStream_t st) {
  int64_t nmax = 0;
  for (int i = 0; i < jobs.n; ++i) nmax = jobs.j[i].n > nmax ? jobs.j[i].n : nmax;
  // blocks <= kGramMaxBlocks (partial buffer), each <= kGramRows rows
  int64_t nb = (nmax + kGramRows - 1) / kGramRows;
  if (nb > kGramMaxBlocks) nb = kGramMaxBlocks;
  if (nb < 1) nb = 1;

  k_gram<<<dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st>>>(jobs, W);
  ++launch_counter();
}

// ------------------------------------------------- pivoted Cholesky orth
// 256 threads: pivot search by warp 0, column scaling and the trailing rank-1
// update by the whole CTA; L^-1 by row-sequential forward substitution.
__device__ void dev_chol_orth(const double* G, double* T64, int n, double* dyn) {
  double (*A)[kN + 1] = reinterpret_cast<double (*)[kN + 1]>(dyn);
  double (*Li)[kN + 1] = reinterpret_cast<double (*)[kN + 1]>(dyn + kN * (kN + 1));  // L^-1 (lower)
  __shared__ int piv[kN];
  __shared__ int bi_s, stop_s;
  __shared__ double dmax_s;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < n * n; e += 256) {
    const int i = e / n, j = e % n;
    A[i][j] = 0.5 * (G[i * n + j] + G[j * n + i]);
    Li[i][j] = 0.0;
  }
  if (tid < n) piv[tid] = tid;
  __syncthreads();
  if (tid < 32) {
    double dm = 0.0;
    for (int i = lane; i < n; i += 32) dm = fmax(dm, A[i][i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if (lane == 0) dmax_s = dm;
  }
  __syncthreads();
  const double dmax = dmax_s;
  const double thr = 1e-10 * dmax;
  int k = 0;
  for (; k < n; ++k) {
    if (tid < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + lane; i < n; i += 32) {
        const double d = A[i][i];
        if (d > best) { best = d; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        bi_s = bi;
        stop_s = !(dmax > 0.0) || best < thr || best <= 0.0;
      }
    }
    __syncthreads();
    if (stop_s) break;
    const int bi = bi_s;
    if (bi != k) {  // symmetric swap of row/col k and bi
      for (int j = tid; j < n; j += 256) {
        const double t = A[k][j]; A[k][j] = A[bi][j]; A[bi][j] = t;
      }
      __syncthreads();
      for (int i = tid; i < n; i += 256) {
        const double t = A[i][k]; A[i][k] = A[i][bi]; A[i][bi] = t;
      }
      if (tid == 0) { const int t = piv[k]; piv[k] = piv[bi]; piv[bi] = t; }
      __syncthreads();
    }
    const double lkk = sqrt(A[k][k]);
    const double inv = 1.0 / lkk;
    __syncthreads();
    for (int i = k + 1 + tid; i < n; i += 256) A[i][k] *= inv;
    if (tid == 0) A[k][k] = lkk;
    __syncthreads();
    const int m = n - k - 1;
    for (int e = tid; e < m * m; e += 256) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      A[i][j] -= A[i][k] * A[j][k];
    }
    __syncthreads();
  }
  const int rk = k;
  // Li = L^-1: row i from rows < i (thread c computes Li[i][c], c <= i)
  for (int i = 0; i < rk; ++i) {
    if (tid <= i) {
      const int c = tid;
      double sacc = (i == c) ? 1.0 : 0.0;
      for (int t = c; t < i; ++t) sacc -= A[i][t] * Li[t][c];
      Li[i][c] = sacc / A[i][i];
    }
    __syncthreads();
  }
  // T[piv[a]][b] = (L^-T)[a][b] = Li[b][a] for a <= b < rk; zero elsewhere
  for (int e = tid; e < n * n; e += 256) {
    const int rr = e / n, b = e % n;
    double v = 0.0;
    // find a with piv[a] == rr (a < rk)
    for (int a2 = 0; a2 < rk; ++a2)
      if (piv[a2] == rr && b >= a2 && b < rk) v = Li[b][a2];
    T64[rr * n + b] = v;
  }
}

__global__ void __launch_bounds__(256) k_chol_orth(EigJobs jobs, int n) {
  extern __shared__ double dyn[];
  dev_chol_orth(jobs.j[blockIdx.x].G, jobs.j[blockIdx.x].T64, n, dyn);
}

static const int kDynSmem = 2 * kN * (kN + 1) * (int)sizeof(double);

void launch_chol_orth(const EigJobs& jobs, int n, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_chol_orth, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
    attr = true;
  }
  k_chol_orth<<<jobs.n, 256, kDynSmem, st>>>(jobs, n);
  ++launch_counter();
}

// --------------------------------------------- parallel Jacobi (truncation)
// Round-robin pairing: n/2 disjoint rotations per step.  A' = J^T A J is applied
// in ONE pass over 2x2 blocks (pair k1 rows x pair k2 cols), V' = V J in another.
__device__ void dev_eig_trunc(const double* G, float* T, int r, int n, double* dyn) {
  double (*A)[kN + 1] = reinterpret_cast<double (*)[kN + 1]>(dyn);
  double (*V)[kN + 1] = reinterpret_cast<double (*)[kN + 1]>(dyn + kN * (kN + 1));
  __shared__ double cs[kN / 2], sn[kN / 2];
  __shared__ int pp[kN / 2], qq[kN / 2];
  __shared__ int order[kN];
  __shared__ double red[8][2];
  __shared__ int stop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < n * n; e += 256) {
    const int i = e / n, j = e % n;
    A[i][j] = 0.5 * (G[i * n + j] + G[j * n + i]);
    V[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = n / 2;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, dg = 0.0;
    for (int e = tid; e < n * n; e += 256) {
      const int i = e / n, j = e % n;
      const double v = A[i][j] * A[i][j];
      if (i == j) dg += v; else off += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      dg += __shfl_xor_sync(0xffffffffu, dg, o);
    }
    if (lane == 0) { red[warp][0] = off; red[warp][1] = dg; }
    __syncthreads();
    if (tid == 0) {
      double o2 = 0.0, d2 = 0.0;
      for (int w = 0; w < 8; ++w) { o2 += red[w][0]; d2 += red[w][1]; }
      stop = (o2 <= 1e-30 * d2) || (o2 == 0.0);
    }
    __syncthreads();
    if (stop) break;
    for (int step = 0; step < n - 1; ++step) {
      if (tid < half) {
        const int k = tid;
        int p, q;
        if (k == 0) { p = 0; q = (step % (n - 1)) + 1; }
        else { p = ((k + step) % (n - 1)) + 1; q = ((n - 1 - k + step) % (n - 1)) + 1; }
        if (p > q) { const int t = p; p = q; q = t; }
        const double apq = A[p][q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          // angle in fp32 (any rotation is an exact similarity; c, s below are orthonormal to
          // fp64 rounding), which keeps the latency of the 2x2 solve short
          const float theta = (float)((A[q][q] - A[p][p]) / (2.0 * apq));
          float t;
          if (fabsf(theta) > 1e18f) t = 0.5f / theta;
          else t = copysignf(1.f, theta) / (fabsf(theta) + sqrtf(fmaf(theta, theta, 1.f)));
          const double td = (double)t;
          c = rsqrt(fma(td, td, 1.0));
          s = td * c;
        }
        pp[k] = p; qq[k] = q; cs[k] = c; sn[k] = s;
      }
      __syncthreads();
      // 2x2 blocks: rows (p1,q1) of pair k1 x cols (p2,q2) of pair k2; all reads, barrier, all writes
      // (half^2 <= 1024 blocks -> at most 4 per thread)
      double nb[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = tid + 256 * u;
        if (e < half * half) {
          const int k1 = e / half, k2 = e % half;
          const int p1 = pp[k1], q1 = qq[k1], p2 = pp[k2], q2 = qq[k2];
          const double c1 = cs[k1], s1 = sn[k1], c2 = cs[k2], s2 = sn[k2];
          const double a = A[p1][p2], b = A[p1][q2], c = A[q1][p2], d = A[q1][q2];
          const double ra = c1 * a - s1 * c, rb = c1 * b - s1 * d;
          const double rc = s1 * a + c1 * c, rd = s1 * b + c1 * d;
          nb[u][0] = c2 * ra - s2 * rb;
          nb[u][1] = s2 * ra + c2 * rb;
          nb[u][2] = c2 * rc - s2 * rd;
          nb[u][3] = s2 * rc + c2 * rd;
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = tid + 256 * u;
        if (e < half * half) {
          const int k1 = e / half, k2 = e % half;
          const int p1 = pp[k1], q1 = qq[k1], p2 = pp[k2], q2 = qq[k2];
          A[p1][p2] = nb[u][0]; A[p1][q2] = nb[u][1]; A[q1][p2] = nb[u][2]; A[q1][q2] = nb[u][3];
        }
      }
      for (int e = tid; e < half * n; e += 256) {
        const int k = e / n, i = e % n;
        const int p = pp[k], q = qq[k];
        const double c = cs[k], s = sn[k];
        const double vp = V[i][p], vq = V[i][q];
        V[i][p] = c * vp - s * vq;
        V[i][q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  for (int t = tid; t < n; t += 256) {
    int rank = 0;
    const double li = A[t][t];
    for (int j = 0; j < n; ++j) {
      const double lj = A[j][j];
      rank += (lj > li) || (lj == li && j < t);
    }
    order[rank] = t;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += 256) {
    const int a = e / n, o = e % n;
    T[a * n + o] = (o < r) ? (float)V[a][order[o]] : 0.f;
  }
}

__global__ void __launch_bounds__(256) k_eig(EigJobs jobs, int n) {
  extern __shared__ double dyn[];
  dev_eig_trunc(jobs.j[blockIdx.x].G, jobs.j[blockIdx.x].T, jobs.j[blockIdx.x].r, n, dyn);
}

void launch_eig_warp(const EigJobs& jobs, int n, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
    attr = true;
  }
  k_eig<<<jobs.n, 256, kDynSmem, st>>>(jobs, n);
  ++launch_counter();
}

// ------------------------------------------------- fused orth / truncation
// One launch per RSVD orthonormalisation (or truncation) step, both sides (blockIdx.y):
//   phase 1 (all blocks): Y = sum of the split-K partials (fixed order) -> written once;
//                         the block's rows are kept in smem and their fp64 Gram partial formed;
//   phase 2 (last block by ticket): fixed-order sum of the Gram partials -> G, then the
//                         pivoted CholQR transform (mode 0) or the truncation eigenvectors
//                         (mode 1), or nothing (mode 2: G must first be summed across ranks).
constexpr int kFRows = 64;
__global__ void __launch_bounds__(256) k_fused_small(SmallJobs jobs, int W, int mode) {
  extern __shared__ double dyn[];
  const SmallJob jb = jobs.j[blockIdx.y];
  float (*sY)[kN + 1] = reinterpret_cast<float (*)[kN + 1]>(dyn);  // kFRows x (kN+1) floats
  __shared__ int ticket;
  const int npairs = W * W;
  const int64_t rpb = (jb.n + gridDim.x - 1) / gridDim.x;
  const int64_t r_begin = (int64_t)blockIdx.x * rpb;
  const int64_t r_end = (jb.n < r_begin + rpb) ? jb.n : r_begin + rpb;
  const int64_t plane = jb.n * W;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kFRows) {
    const int nr = (int)(r_end - r0 < kFRows ? r_end - r0 : kFRows);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * W; e += 256) {
      const int i = e / W, c = e % W;
      const int64_t g = (r0 + i) * W + c;
      float v;
      if (jb.nsplit > 1) {
        float a0 = 0.f;
        for (int sp = 0; sp < jb.nsplit; ++sp) a0 += __ldcg(jb.part + sp * plane + g);
        jb.Y[g] = a0;
        v = a0;
      } else {
        v = __ldcg(jb.Y + g);
      }
      sY[i][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int pr = threadIdx.x + 256 * q;
      if (pr < npairs) {
        const int a = pr / W, c = pr % W;
        double t0 = 0.0, t1 = 0.0;
        int i = 0;
        for (; i + 1 < nr; i += 2) {
          t0 = fma((double)sY[i][a], (double)sY[i][c], t0);
          t1 = fma((double)sY[i + 1][a], (double)sY[i + 1][c], t1);
        }
        if (i < nr) t0 = fma((double)sY[i][a], (double)sY[i][c], t0);
        acc[q] += t0 + t1;
      }
    }
  }
  double* part = jb.gpart + (int64_t)blockIdx.x * npairs;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int pr = threadIdx.x + 256 * q;
    if (pr < npairs) part[pr] = acc[q];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(jb.counter, 1);
  __syncthreads();
  if (ticket != (int)gridDim.x - 1) return;
  __threadfence();
  const int nb = (int)gridDim.x;
  for (int pr = threadIdx.x; pr < npairs; pr += 256) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = 0;
    for (; b + 3 < nb; b += 4) {
      a0 += __ldcg(jb.gpart + (int64_t)(b + 0) * npairs + pr);
      a1 += __ldcg(jb.gpart + (int64_t)(b + 1) * npairs + pr);
      a2 += __ldcg(jb.gpart + (int64_t)(b + 2) * npairs + pr);
      a3 += __ldcg(jb.gpart + (int64_t)(b + 3) * npairs + pr);
    }
    for (; b < nb; ++b) a0 += __ldcg(jb.gpart + (int64_t)b * npairs + pr);
    jb.G[pr] = (a0 + a1) + (a2 + a3);
  }
  if (threadIdx.x == 0) *jb.counter = 0;  // re-arm for the next launch (stream ordered)
  __threadfence_block();
  __syncthreads();
  if (mode == 0) dev_chol_orth(jb.G, jb.T64, W, dyn);
  else if (mode == 1) dev_eig_trunc(jb.G, jb.T, jb.r, W, dyn);
}

void launch_fused_small(const SmallJobs& jobs, int W, int mode, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fused_small, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
    attr = true;
  }
  int64_t nmax = 0;
  for (int i = 0; i < jobs.n; ++i) nmax = jobs.j[i].n > nmax ? jobs.j[i].n : nmax;
  // ~4 row chunks per block keeps the last-block reduction short (<= 64 partials at 16K rows)
  int64_t nb = (nmax + 4 * kFRows - 1) / (4 * kFRows);
  if (nb > kGramMaxBlocks) nb = kGramMaxBlocks;
  if (nb < 1) nb = 1;
  k_fused_small<<<dim3((unsigned)nb, (unsigned)jobs.n), 256, kDynSmem, st>>>(jobs, W, mode);
  ++launch_counter();
}

// Mab = VWb^T C VWa (r x r), C = Q1_B^T Q1_A (n x n, fp64); VWbM = VWb Mab (n x r).
// V_B^T V_A = VWb^T Q1_B^T Q1_A VWa: the r x r core of RC3 (Alg. 2).
__global__ void __launch_bounds__(256) k_cross_small(const double* __restrict__ C, const float* __restrict__ VWa,
                                                     const float* __restrict__ VWb, int n, int r,
                                                     float* __restrict__ VWbM) {
  __shared__ double T1[kN][kN / 2];      // C VWa  (n x r), r <= 32
  __shared__ double M[kN / 2][kN / 2];   // r x r
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
