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
template <int n>
__global__ void __launch_bounds__(32) k_warp_chol(EigJobs jobs);

// ------------------------------------------------------------------- Gram
// One launch: each block loads its row range in chunks of kGramRows (one chunk unless n > 64K), then
// accumulates its W x W partial in fp64; the last block (ticket) sums the partials in a
// fixed order.  blockIdx.y = job.
constexpr int kGramRows = 32;
template <int W>
__global__ void __launch_bounds__(256) k_gram(GramJobs jobs) {
  ::lrqmm::pdl_enter();
  const GramJob jb = jobs.j[blockIdx.y];
  const int npairs = W * W;
  __shared__ double s1[kGramRows][kN + 1];
  __shared__ double s2[kGramRows][kN + 1];
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
    const int ne = nr * W;
    for (int e0 = threadIdx.x; e0 < ne; e0 += 256 * 4) {
      float v1[4], v2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + 256 * u;
        v1[u] = e < ne ? __ldg(jb.Y1 + r0 * W + e) : 0.f;
        v2[u] = e < ne ? __ldg(jb.Y2 + r0 * W + e) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + 256 * u;
        if (e < ne) {
          s1[e / W][e % W] = (double)v1[u];
          s2[e / W][e % W] = (double)v2[u];
        }
      }
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
          t0 = fma(s1[i][a], s2[i][c], t0);
          t1 = fma(s1[i + 1][a], s2[i + 1][c], t1);
          t2 = fma(s1[i + 2][a], s2[i + 2][c], t2);
          t3 = fma(s1[i + 3][a], s2[i + 3][c], t3);
        }
        for (; i < nr; ++i) t0 = fma(s1[i][a], s2[i][c], t0);
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
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int b = 0;
    for (; b + 7 < nb; b += 8) {
      double t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] = __ldcg(jb.partial + (int64_t)(b + k) * npairs + pr);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += t[k];
    }
    for (; b < nb; ++b) a[0] += __ldcg(jb.partial + (int64_t)b * npairs + pr);
    jb.G[pr] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  }
  if (threadIdx.x == 0) *jb.counter = 0;  // re-arm for the next launch (stream ordered)
}

void launch_gram_jobs(const GramJobs& jobs, int W, cudaStream_t st) {
  int64_t nmax = 0;
  for (int i = 0; i < jobs.n; ++i) nmax = jobs.j[i].n > nmax ? jobs.j[i].n : nmax;
  // blocks <= kGramMaxBlocks (partial buffer), ~4 row chunks each (short final reduction)
  int64_t nb = (nmax + 8 * kGramRows - 1) / (8 * kGramRows);
  if (nb > kGramMaxBlocks) nb = kGramMaxBlocks;
  if (nb < 1) nb = 1;

  switch (W) {
    case 8: launch_pdl(k_gram<8>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    case 16: launch_pdl(k_gram<16>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    case 24: launch_pdl(k_gram<24>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    case 32: launch_pdl(k_gram<32>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    case 40: launch_pdl(k_gram<40>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    case 48: launch_pdl(k_gram<48>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    case 56: launch_pdl(k_gram<56>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    case 64: launch_pdl(k_gram<64>, dim3((unsigned)nb, (unsigned)jobs.n), 256, 0, st, jobs); break;
    default: break;
  }

  ++launch_counter();
}

// ------------------------------------------------- pivoted Cholesky orth
// 256 threads: pivot search by warp 0, column scaling and the trailing rank-1
// update by the whole CTA; L^-1 by row-sequential forward substitution.
template <int n>
__device__ void dev_chol_orth(const double* G, double* T64, double* dyn) {
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

template <int n>
__global__ void __launch_bounds__(256) k_chol_orth(EigJobs jobs) {
  ::lrqmm::pdl_enter();
  extern __shared__ double dyn[];
  dev_chol_orth<n>(jobs.j[blockIdx.x].G, jobs.j[blockIdx.x].T64, dyn);
}

static const int kDynSmem = 2 * kN * (kN + 1) * (int)sizeof(double);

template <int n>
static void chol_t(const EigJobs& jobs, cudaStream_t st) {
  if constexpr (n <= 32) {
    launch_pdl(k_warp_chol<n>, jobs.n, 32, 0, st, jobs);
  } else {
    static std::atomic<unsigned> attr{0};
    ensure_smem(k_chol_orth<n>, kDynSmem, attr);
    launch_pdl(k_chol_orth<n>, jobs.n, 256, kDynSmem, st, jobs);
  }
}

void launch_chol_orth(const EigJobs& jobs, int n, cudaStream_t st) {
  switch (n) {
    case 8: chol_t<8>(jobs, st); break;
    case 16: chol_t<16>(jobs, st); break;
    case 24: chol_t<24>(jobs, st); break;
    case 32: chol_t<32>(jobs, st); break;
    case 40: chol_t<40>(jobs, st); break;
    case 48: chol_t<48>(jobs, st); break;
    case 56: chol_t<56>(jobs, st); break;
    case 64: chol_t<64>(jobs, st); break;
    default: break;
  }

  ++launch_counter();
}

// --------------------------------------------- parallel Jacobi (truncation)
// Cyclic parallel Jacobi with the round-robin ordering on the leading na x na block of G (na =
// the even size covering every nonzero row: the zero-padded sketch columns beyond r + p give zero
// rows and columns, eigenvalue 0, nothing to rotate).  na/2 disjoint rotations per step, na - 1
// steps per sweep.  The matrix is RELABELLED after every step (position d -> sigma(d): 0 -> 0,
// 1 -> na-1, d -> d-1) so that pair k always sits at the fixed positions (P_k, Q_k) = (0, 1) for
// k = 0 and (k+1, na-k) otherwise: A' = J^T A J is computed over 2x2 blocks (pair k1 rows x pair
// k2 cols) read from one buffer and written, relabelled, to the other (ping-pong), so every thread
// has fixed addresses, one barrier per step, and no write-after-read hazards.  V' = V J is applied
// in place on the ORIGINAL column labels (label of position d at step s: orig(s, d)).
// Every warp computes the rotations of the step redundantly (lane k -> pair k, bitwise identical
// in every warp) and hands c, s out by shuffle.
// Stop: off(A)^2 <= 1e-16 diag(A)^2 (off-diagonal <= 1e-8 relative: eigenvector error ~1e-8 / relative
// gap, at the fp32 precision of the output T; reading #29).
__device__ __forceinline__ int jac_P(int k) { return k == 0 ? 0 : k + 1; }
__device__ __forceinline__ int jac_Q(int k, int na) { return k == 0 ? 1 : na - k; }
__device__ __forceinline__ int jac_sigma(int d, int na) { return d == 0 ? 0 : (d == 1 ? na - 1 : d - 1); }
__device__ __forceinline__ int jac_orig(int s, int d, int m) {  // s in [0, m), m = na - 1
  if (d == 0) return 0;
  int x = d - 1 + s;
  if (x >= m) x -= m;
  return x + 1;
}
__host__ __device__ constexpr int eig_smem_bytes(int n) { return 3 * n * (n + 1) * 8; }

template <int n>
__device__ void dev_eig_trunc(const double* G, float* T, int r, double* dyn) {
  constexpr int ld = n + 1;
  constexpr int kBlk = ((n / 2) * (n / 2) + 255) / 256, kV = ((n / 2) * n + 255) / 256;
  double* Abuf = dyn;                 // 2 x n x ld (ping-pong, relabelled)
  double* V = dyn + 2 * n * ld;       // n x ld, original labels
  __shared__ int order[kN];
  __shared__ double red[8][2];
  __shared__ double scale_s;
  __shared__ int na_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) {
    double dm = 0.0;
    int last = -1;
    for (int i = lane; i < n; i += 32) {
      const double g = fabs(G[i * n + i]);
      dm = fmax(dm, g);
      if (g > 0.0) last = i;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
      last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    }
    if (lane == 0) {
      scale_s = dm > 0.0 ? 1.0 / dm : 1.0;
      // a zero diagonal entry of a Gram matrix means a zero row and column
      const int na = (last + 2) & ~1;
      na_s = na < 2 ? 2 : (na > n ? n : na);
    }
  }
  __syncthreads();
  const int na = na_s, half = na / 2, m = na - 1;
  // normalised copy (eigenvectors are scale invariant): entries O(1), so the rotation angle
  // can be computed in fp32 without under/overflow.  At step 0 position d holds index d.
  double off = 0.0, dg = 0.0;
  for (int e = tid; e < n * n; e += 256) {
    const int i = e / n, j = e % n;
    const double a = 0.5 * (G[i * n + j] + G[j * n + i]) * scale_s;
    Abuf[i * ld + j] = a;
    V[i * ld + j] = (i == j) ? 1.0 : 0.0;
    if (i == j) dg += a * a; else off += a * a;
  }
  auto converged = [&](double o, double d) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      o += __shfl_xor_sync(0xffffffffu, o, s);
      d += __shfl_xor_sync(0xffffffffu, d, s);
    }
    if (lane == 0) { red[warp][0] = o; red[warp][1] = d; }
    __syncthreads();
    double o2 = 0.0, d2 = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) { o2 += red[w][0]; d2 += red[w][1]; }
    return (o2 <= 1e-16 * d2) || (o2 == 0.0);
  };
  bool stop = converged(off, dg);
  // fixed per-thread work: this lane's rotation (pair `lane`), its 2x2 blocks, its V entries
  const int rk = lane < half ? lane : 0;
  const int rP = jac_P(rk) * ld + jac_P(rk), rQ = jac_Q(rk, na) * ld + jac_Q(rk, na), rPQ = jac_P(rk) * ld + jac_Q(rk, na);
  int bk1[kBlk], bk2[kBlk], brd[kBlk][4], bwr[kBlk][4];
  bool bok[kBlk], bdiag[kBlk];
#pragma unroll
  for (int u = 0; u < kBlk; ++u) {
    const int e = tid + 256 * u;
    bok[u] = e < half * half;
    const int k1 = bok[u] ? e / half : 0, k2 = bok[u] ? e % half : 0;
    bk1[u] = k1;
    bk2[u] = k2;
    bdiag[u] = k1 == k2;
    const int P1 = jac_P(k1), Q1 = jac_Q(k1, na), P2 = jac_P(k2), Q2 = jac_Q(k2, na);
    brd[u][0] = P1 * ld + P2; brd[u][1] = P1 * ld + Q2; brd[u][2] = Q1 * ld + P2; brd[u][3] = Q1 * ld + Q2;
    const int p1 = jac_sigma(P1, na), q1 = jac_sigma(Q1, na), p2 = jac_sigma(P2, na), q2 = jac_sigma(Q2, na);
    bwr[u][0] = p1 * ld + p2; bwr[u][1] = p1 * ld + q2; bwr[u][2] = q1 * ld + p2; bwr[u][3] = q1 * ld + q2;
  }
  int vk[kV], vrow[kV], vP[kV], vQ[kV];
  bool vok[kV];
#pragma unroll
  for (int u = 0; u < kV; ++u) {
    const int e = tid + 256 * u;
    vok[u] = e < half * na;
    vk[u] = vok[u] ? e / na : 0;
    vrow[u] = (vok[u] ? e % na : 0) * ld;
    vP[u] = jac_P(vk[u]);
    vQ[u] = jac_Q(vk[u], na);
  }
  int total = 0;  // steps done
  for (int sweep = 0; sweep < 30 && !stop; ++sweep) {
    for (int step = 0; step < m; ++step, ++total) {
      const double* Ac = Abuf + (total & 1) * n * ld;
      double* An = Abuf + ((total + 1) & 1) * n * ld;
      const bool last = step + 1 == m;
      double c = 1.0, s = 0.0;
      if (lane < half) {
        const double app = Ac[rP], aqq = Ac[rQ], apq = Ac[rPQ];
        const float fpq = (float)apq;
        // angle in fp32 with approximate division / square root: any rotation is an exact
        // similarity (c, s below are orthonormal to fp64 rounding); only convergence depends on it
        const float theta = __fdividef((float)(aqq - app), 2.f * fpq);
        const float at = fabsf(theta);
        const float rs = rsqrtf(fmaf(theta, theta, 1.f));
        float t = copysignf(__fdividef(1.f, at + fmaf(theta, theta, 1.f) * rs), theta);
        t = at > 1e18f ? __fdividef(0.5f, theta) : t;
        const double td = fpq != 0.f ? (double)t : 0.0;
        const double x = fma(td, td, 1.0);
        double y = (double)rsqrtf((float)x);
        y = y * fma(-0.5 * x, y * y, 1.5);
        y = y * fma(-0.5 * x, y * y, 1.5);
        c = fpq != 0.f ? y : 1.0;
        s = td * c;
      }
      off = 0.0;
      dg = 0.0;
#pragma unroll
      for (int u = 0; u < kBlk; ++u) {
        const double c1 = __shfl_sync(0xffffffffu, c, bk1[u]), s1 = __shfl_sync(0xffffffffu, s, bk1[u]);
        const double c2 = __shfl_sync(0xffffffffu, c, bk2[u]), s2 = __shfl_sync(0xffffffffu, s, bk2[u]);
        if (bok[u]) {
          const double a = Ac[brd[u][0]], b = Ac[brd[u][1]], cc = Ac[brd[u][2]], d = Ac[brd[u][3]];
          const double ra = c1 * a - s1 * cc, rb = c1 * b - s1 * d;
          const double rc = s1 * a + c1 * cc, rd = s1 * b + c1 * d;
          const double v0 = c2 * ra - s2 * rb, v1 = s2 * ra + c2 * rb, v2 = c2 * rc - s2 * rd, v3 = s2 * rc + c2 * rd;
          An[bwr[u][0]] = v0;
          An[bwr[u][1]] = v1;
          An[bwr[u][2]] = v2;
          An[bwr[u][3]] = v3;
          if (last) {
            if (bdiag[u]) { dg += v0 * v0 + v3 * v3; off += v1 * v1 + v2 * v2; }
            else off += (v0 * v0 + v1 * v1) + (v2 * v2 + v3 * v3);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const double ck = __shfl_sync(0xffffffffu, c, vk[u]), sk = __shfl_sync(0xffffffffu, s, vk[u]);
        if (vok[u]) {
          const int p = vrow[u] + jac_orig(step, vP[u], m), q = vrow[u] + jac_orig(step, vQ[u], m);
          const double vp = V[p], vq = V[q];
          V[p] = ck * vp - sk * vq;
          V[q] = sk * vp + ck * vq;
        }
      }
      if (last) stop = converged(off, dg);  // its barrier ends the step
      else __syncthreads();
    }
  }
  __syncthreads();
  // position d < na holds eigenvalue A[d][d] with eigenvector V[:, orig(total mod m, d)];
  // indices >= na: eigenvalue 0, eigenvector e_d
  const double* Af = Abuf + (total & 1) * n * ld;
  const int sf = total % m;
  for (int t = tid; t < n; t += 256) {
    int rank = 0;
    const double li = t < na ? Af[t * ld + t] : 0.0;
    for (int j = 0; j < n; ++j) {
      const double lj = j < na ? Af[j * ld + j] : 0.0;
      rank += (lj > li) || (lj == li && j < t);
    }
    order[rank] = t < na ? jac_orig(sf, t, m) : t;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += 256) {
    const int a = e / n, o = e % n;
    T[a * n + o] = (o < r) ? (float)V[a * ld + order[o]] : 0.f;
  }
}

template <int n>
__global__ void __launch_bounds__(256) k_eig(EigJobs jobs) {
  ::lrqmm::pdl_enter();
  extern __shared__ double dyn[];
  dev_eig_trunc<n>(jobs.j[blockIdx.x].G, jobs.j[blockIdx.x].T, jobs.j[blockIdx.x].r, dyn);
}

template <int n>
static void eig_t(const EigJobs& jobs, cudaStream_t st) {
  constexpr int smem = eig_smem_bytes(n) > kDynSmem ? eig_smem_bytes(n) : kDynSmem;
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_eig<n>, smem, attr);
  launch_pdl(k_eig<n>, jobs.n, 256, smem, st, jobs);
}

void launch_eig_warp(const EigJobs& jobs, int n, cudaStream_t st) {
  switch (n) {
    case 8: eig_t<8>(jobs, st); break;
    case 16: eig_t<16>(jobs, st); break;
    case 24: eig_t<24>(jobs, st); break;
    case 32: eig_t<32>(jobs, st); break;
    case 40: eig_t<40>(jobs, st); break;
    case 48: eig_t<48>(jobs, st); break;
    case 56: eig_t<56>(jobs, st); break;
    case 64: eig_t<64>(jobs, st); break;
    default: break;
  }

  ++launch_counter();
}

// ------------------------------------------------- one-warp solvers (n <= 32)
// Pivoted Cholesky QR transform, one warp, lane j = column j, no row/column swaps:
//   S (the Schur complement, column-major, stride 33 so lane-parallel accesses are conflict free)
//   is updated in place on the ORIGINAL indices; lane j keeps its diagonal d_j in a register.
//   Step k: pivot p = argmax d_j over the remaining lanes (one packed-key __reduce_max_sync pair);
//   l = S[p, :] / sqrt(d_p) (l_p = sqrt(d_p)); S -= l l^T; d -= l^2.
//   The transform is built alongside as Gram-Schmidt in the G inner product (mathematically
//   T = P L^-T):  t_k = (e_p - sum_{m<k} t_m L[p, m]) / L[p, k],  so Q = Y T has orthonormal
//   columns.  Pivots below 1e-10 x the largest diagonal entry end the factorisation (reading
//   #12): the remaining columns of T are zero.
// Output T64[j * n + k] = T[j, k].
template <int n>
__device__ void warp_chol_orth(const double* G, double* T64, double* sm, double* Lsm, double* Tsm) {
  const int lane = threadIdx.x & 31;
#define SA(i, j) sm[(j) * 33 + (i)]
  double d = 0.0;
  for (int i = 0; i < n; ++i)
    if (lane < n) {
      const double g = 0.5 * (G[i * n + lane] + G[lane * n + i]);
      SA(i, lane) = g;
      if (i == lane) d = g;
    }
  double dmax = d;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const double thr = 1e-10 * dmax;
  bool done = lane >= n;
  __syncwarp();
  int k = 0;
  for (; k < n; ++k) {
    // argmax of d over the remaining lanes; ties (to 2^-46 relative) -> lowest lane
    const unsigned long long bits = (!done && d > 0.0) ? (unsigned long long)__double_as_longlong(d) : 0ull;
    const unsigned long long key = (bits & ~63ull) | (unsigned long long)(bits ? 63 - lane : 0);
    const unsigned hi = (unsigned)(key >> 32);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned lo = hi == mhi ? (unsigned)key : 0u;
    const unsigned mlo = __reduce_max_sync(0xffffffffu, lo);
    if (mhi == 0u && mlo == 0u) break;
    const int p = 63 - (int)(mlo & 63u);
    const double dp = __shfl_sync(0xffffffffu, d, p);
    if (!(dmax > 0.0) || dp < thr || dp <= 0.0) break;
    const double inv = rsqrt(dp);
    const double lkk = dp * inv;
    const double spj = SA(p, lane);
    double l = done ? 0.0 : (lane == p ? lkk : spj * inv);
    if (lane == p) done = true;
    Lsm[k * 33 + lane] = l;
    if (!done) d = fma(-l, l, d);
    __syncwarp();
    // t_k = (e_p - sum_{m<k} t_m L[p, m]) / L[p, k]
    {
      double a[4] = {lane == p ? 1.0 : 0.0, 0.0, 0.0, 0.0};
      for (int m0 = 0; m0 < k; m0 += 4) {
        double tv[4], lv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const bool ok = m0 + t < k;
          tv[t] = ok ? Tsm[(m0 + t) * 33 + lane] : 0.0;
          lv[t] = ok ? Lsm[(m0 + t) * 33 + p] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) a[t] = fma(-tv[t], lv[t], a[t]);
      }
      Tsm[k * 33 + lane] = ((a[0] + a[1]) + (a[2] + a[3])) * inv;
    }
    // S -= l l^T on the remaining columns
    // (explicitly staged in chunks: all loads of a chunk issue before its stores)
    if (!done) {
#pragma unroll
      for (int i0 = 0; i0 < n; i0 += 8) {
        double sv[8], lv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          lv[t] = Lsm[k * 33 + i0 + t];
          sv[t] = SA(i0 + t, lane);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) SA(i0 + t, lane) = fma(-lv[t], l, sv[t]);
      }
    }
    __syncwarp();
  }
  const int rk = k;
  __syncwarp();
  if (lane < n)
    for (int c = 0; c < n; ++c) T64[lane * n + c] = c < rk ? Tsm[c * 33 + lane] : 0.0;
#undef SA
}

template <int n>
__global__ void __launch_bounds__(32) k_warp_chol(EigJobs jobs) {
  ::lrqmm::pdl_enter();
  __shared__ double buf[3][32 * 33];
  const EigJob job = jobs.j[blockIdx.x];
  warp_chol_orth<n>(job.G, job.T64, buf[0], buf[1], buf[2]);
}

// ------------------------------------------------- fused orth / truncation
// One launch per RSVD orthonormalisation (or truncation) step, both sides (blockIdx.y):
//   phase 1 (all blocks): Y = sum of the split-K partials (fixed order) -> written once;
//                         the block's rows are kept in smem and their fp64 Gram partial formed;
//   phase 2 (last block by ticket): fixed-order sum of the Gram partials -> G, then the
//                         pivoted CholQR transform (mode 0) or the truncation eigenvectors
//                         (mode 1), or nothing (mode 2: G must first be summed across ranks).
// rows per shared-memory chunk (fp32, two buffers in the 66.5 KB dynamic allocation)
__host__ __device__ constexpr int frows(int w) { return w <= 32 ? 256 : 128; }
template <int W>
__global__ void __launch_bounds__(256) k_fused_small(SmallJobs jobs, int mode) {
  ::lrqmm::pdl_enter();
  constexpr int kFRows = frows(W);
  extern __shared__ __align__(128) double dyn[];
  const SmallJob jb = jobs.j[blockIdx.y];
  float* buf = reinterpret_cast<float*>(dyn);  // 2 x kFRows x W fp32 (bulk-copied chunks of Y)
  __shared__ uint64_t ld_bar[2];
  __shared__ int ticket;
  constexpr int npairs = W * W;
  // Gram in 4 x 4 register tiles: tile (a, c), a <= c, of T x T tiles; G row groups per block
  constexpr int T = W / 4;
  constexpr int U = T * (T + 1) / 2;
  constexpr int G = 256 / U;
  int ta = 0, tc = 0;
  const int tu = threadIdx.x % U, tg = threadIdx.x / U;
  const bool gram_thread = threadIdx.x < U * G;
  {
    int u = tu;
    for (int a = 0; a < T; ++a) {
      if (u < T - a) { ta = a; tc = a + u; break; }
      u -= T - a;
    }
  }
  const int64_t rpb = (jb.n + gridDim.x - 1) / gridDim.x;
  const int64_t r_begin = (int64_t)blockIdx.x * rpb;
  const int64_t r_end = (jb.n < r_begin + rpb) ? jb.n : r_begin + rpb;
  const int nchunk = r_end > r_begin ? (int)((r_end - r_begin + kFRows - 1) / kFRows) : 0;
  if (threadIdx.x == 0) {
    mbar_init(&ld_bar[0], 1);
    mbar_init(&ld_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // Y is final and dense (split partials were reduced beforehand): chunk c of this block is one
  // contiguous bulk copy, double-buffered so that chunk c+1 lands while chunk c is multiplied
  auto issue = [&](int c) {
    const int64_t r0 = r_begin + (int64_t)c * kFRows;
    const int nr = (int)(r_end - r0 < kFRows ? r_end - r0 : kFRows);
    const uint32_t bytes = (uint32_t)nr * W * 4u;
    mbar_arrive_expect_tx(&ld_bar[c & 1], bytes);
    bulk_load(buf + (c & 1) * kFRows * W, jb.Y + r0 * W, bytes, &ld_bar[c & 1]);
  };
  if (threadIdx.x == 0) {
    if (nchunk > 0) issue(0);
    if (nchunk > 1) issue(1);
  }
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int c = 0; c < nchunk; ++c) {
    const int64_t r0 = r_begin + (int64_t)c * kFRows;
    const int nr = (int)(r_end - r0 < kFRows ? r_end - r0 : kFRows);
    mbar_wait(&ld_bar[c & 1], (c >> 1) & 1);
    const float* bY = buf + (c & 1) * kFRows * W;
    if (gram_thread) {
      for (int i = tg; i < nr; i += G) {
        const float4 x4 = *reinterpret_cast<const float4*>(bY + i * W + 4 * ta);
        const float4 y4 = *reinterpret_cast<const float4*>(bY + i * W + 4 * tc);
        const double xa[4] = {x4.x, x4.y, x4.z, x4.w}, yc[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p * 4 + q] = fma(xa[p], yc[q], acc[p * 4 + q]);
      }
    }
    __syncthreads();  // every thread is done with buffer (c & 1): refill it with chunk c + 2
    if (threadIdx.x == 0 && c + 2 < nchunk) issue(c + 2);
  }
  // fixed-order reduction of the G row groups of each tile, then the block partial (both halves)
  __syncthreads();
  double (*red)[16] = reinterpret_cast<double (*)[16]>(dyn);  // (G * U) x 16
  if (gram_thread)
#pragma unroll
    for (int q = 0; q < 16; ++q) red[tg * U + tu][q] = acc[q];
  __syncthreads();
  double* part = jb.gpart + (int64_t)blockIdx.x * npairs;
  for (int e = threadIdx.x; e < U * 16; e += 256) {
    const int u = e / 16, q = e % 16;
    double sum = 0.0;
    for (int g = 0; g < G; ++g) sum += red[g * U + u][q];
    int a = 0, c = 0, uu = u;
    for (int aa = 0; aa < T; ++aa) {
      if (uu < T - aa) { a = aa; c = aa + uu; break; }
      uu -= T - aa;
    }
    const int i = 4 * a + q / 4, j = 4 * c + q % 4;
    part[i * W + j] = sum;  // diagonal tiles: (p, q) and (q, p) hold bitwise-equal sums
    part[j * W + i] = sum;
  }
  // two-level fixed-order reduction of the block partials: the last block of each group of 16
  // sums its group (-> gpart[nb + g]), the last group finisher sums the groups (-> G).  Counters:
  // counter[0] = groups done, counter[1 + g] = blocks of group g done (all re-armed to 0).
  const int nb = (int)gridDim.x;
  const int grp = blockIdx.x / 16, ngrp = (nb + 15) / 16;
  const int gsize = nb - 16 * grp < 16 ? nb - 16 * grp : 16;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(jb.counter + 1 + grp, 1);
  __syncthreads();
  if (ticket != gsize - 1) return;
  __threadfence();
  for (int pr = threadIdx.x; pr < npairs; pr += 256) {
    double a = 0.0;
    for (int b = 16 * grp; b < 16 * grp + gsize; ++b) a += __ldcg(jb.gpart + (int64_t)b * npairs + pr);
    jb.gpart[(int64_t)(nb + grp) * npairs + pr] = a;
  }
  if (threadIdx.x == 0) jb.counter[1 + grp] = 0;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(jb.counter, 1);
  __syncthreads();
  if (ticket != ngrp - 1) return;
  __threadfence();
  for (int pr = threadIdx.x; pr < npairs; pr += 256) {
    double a = 0.0;
    for (int g = 0; g < ngrp; ++g) a += __ldcg(jb.gpart + (int64_t)(nb + g) * npairs + pr);
    jb.G[pr] = a;
  }
  if (threadIdx.x == 0) jb.counter[0] = 0;  // re-arm for the next launch (stream ordered)
  if (jb.cmax && threadIdx.x < 64) jb.cmax[threadIdx.x] = 0u;  // the next apply64's column maxima
  __threadfence_block();
  __syncthreads();
  if constexpr (W <= 32) {
    if (mode == 0 && threadIdx.x < 32) {
      warp_chol_orth<W>(jb.G, jb.T64, dyn, dyn + 32 * 33, dyn + 2 * 32 * 33);
    }
    if (mode == 1) dev_eig_trunc<W>(jb.G, jb.T, jb.r, dyn);
  } else {
    if (mode == 0) dev_chol_orth<W>(jb.G, jb.T64, dyn);
    else if (mode == 1) dev_eig_trunc<W>(jb.G, jb.T, jb.r, dyn);
  }
}

template <int W>
static void fused_t(const SmallJobs& jobs, int mode, int64_t nb, cudaStream_t st) {
  // the truncation (mode 1) of the widest sketches needs more than the Y staging buffers
  constexpr int big = eig_smem_bytes(W) > kDynSmem ? eig_smem_bytes(W) : kDynSmem;
  const int smem = mode == 1 ? big : kDynSmem;
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_fused_small<W>, big, attr);
  launch_pdl(k_fused_small<W>, dim3((unsigned)nb, (unsigned)jobs.n), 256, smem, st, jobs, mode);
}

void launch_fused_small(const SmallJobs& jobs, int W, int mode, cudaStream_t st) {
  int64_t nmax = 0;
  for (int i = 0; i < jobs.n; ++i) nmax = jobs.j[i].n > nmax ? jobs.j[i].n : nmax;
  // ~2 row chunks per block, at most 2 blocks per SM: the last block sums <= 296 partials
  const int fr = frows(W);
  int64_t nb = (nmax + 2 * fr - 1) / (2 * fr);
  for (int i = 0; i < jobs.n; ++i)
    if (jobs.j[i].nsplit != 1) return;  // contract: Y is reduced before the fused kernel
  if (nb > 444) nb = 444;  // three resident blocks per SM (66.5 KB each)
  if (nb > kGramMaxBlocks) nb = kGramMaxBlocks;
  if (nb < 1) nb = 1;
  switch (W) {
    case 8: fused_t<8>(jobs, mode, nb, st); break;
    case 16: fused_t<16>(jobs, mode, nb, st); break;
    case 24: fused_t<24>(jobs, mode, nb, st); break;
    case 32: fused_t<32>(jobs, mode, nb, st); break;
    case 40: fused_t<40>(jobs, mode, nb, st); break;
    case 48: fused_t<48>(jobs, mode, nb, st); break;
    case 56: fused_t<56>(jobs, mode, nb, st); break;
    case 64: fused_t<64>(jobs, mode, nb, st); break;
    default: break;
  }

  ++launch_counter();
}

// Mab = VWb^T C VWa (r x r), C = Q1_B^T Q1_A (n x n, fp64); VWbM = VWb Mab (n x r).
// V_B^T V_A = VWb^T Q1_B^T Q1_A VWa: the r x r core of RC3 (Alg. 2).
__global__ void __launch_bounds__(256) k_cross_small(const double* __restrict__ C, const float* __restrict__ VWa,
                                                     const float* __restrict__ VWb, int n, int r,
                                                     float* __restrict__ VWbM) {
  ::lrqmm::pdl_enter();
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
  launch_pdl(k_cross_small, 1, 256, 0, st, C, VWa, VWb, n, r, VWbM); ++launch_counter();
}

}  // namespace lrqmm
