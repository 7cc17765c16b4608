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
#include "solvers.cuh"

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

template <int n>
__global__ void __launch_bounds__(32) k_warp_chol(EigJobs jobs) {
  ::lrqmm::pdl_enter();
  __shared__ double buf[3][32 * 33];
  const EigJob job = jobs.j[blockIdx.x];
  warp_chol_orth<n>(job.G, job.T64, buf[0], buf[1], buf[2]);
}

// ------------------------------------------------- fused orth / truncation
// One launch per RSVD orthonormalisation (or truncation) step, both sides (blockIdx.y):
//   phase 1 (all blocks): the block's rows of the dense Y (split-K partials were reduced by the
//                         launch before) stream into shared memory by bulk copies, double-buffered,
//                         and their fp64 Gram partial is formed on the fp64 tensor cores;
//   phase 2 (last block by ticket): fixed-order sum of the Gram partials -> G (one level when all
//                         blocks form one group of 16, else two), then G in shared memory and the
//                         pivoted CholQR transform (mode 0) or the truncation eigenvectors
//                         (mode 1), or nothing (mode 2: G must first be summed across ranks).
// rows per shared-memory chunk (fp32, two buffers in the 66.5 KB dynamic allocation)
__host__ __device__ constexpr int frows(int w) { return w <= 32 ? 256 : 128; }
#ifdef LRQMM_FS_TRACE
// development only (tools/fs_trace.py): globaltimer stamps of the last k_fused_small launch per mode
__device__ unsigned long long fs_trace[16];
extern "C" int lrqmm_debug_fs_trace(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, fs_trace, sizeof fs_trace) != cudaSuccess) return 1;
#ifdef LRQMM_EIG_STATS
  int steps = 0;  // Jacobi steps of the last truncation (this translation unit's solver)
  cudaMemcpyFromSymbol(&steps, eig_stats_steps, sizeof steps);
  out[15] = (unsigned long long)steps;
#endif
  return 0;
}
#define FS_T(i)                                                         \
  if (threadIdx.x == 0 && blockIdx.y == 0) {                            \
    unsigned long long t_;                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
    fs_trace[8 * (mode & 1) + (i)] = t_;                                \
  }
#else
#define FS_T(i)
#endif

// ((0 + p[0]) + p[s]) + p[2 s] + ... in index order (the fixed-order partial sums), loads issued 8 at
// a time so that a chain of L2 round trips does not serialise the finisher
LRQMM_DEV double sum_strided(const double* p, int64_t stride, int cnt) {
  double a = 0.0;
  for (int b0 = 0; b0 < cnt; b0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b0 + u < cnt ? __ldcg(p + (int64_t)(b0 + u) * stride) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b0 + u < cnt) a += v[u];
  }
  return a;
}

template <int W>
__global__ void __launch_bounds__(256) k_fused_small(SmallJobs jobs, int mode) {
  ::lrqmm::pdl_enter();
  if (blockIdx.x == 0) { FS_T(0) }
  constexpr int kFRows = frows(W);
  extern __shared__ __align__(128) double dyn[];
  const SmallJob jb = jobs.j[blockIdx.y];
  float* buf = reinterpret_cast<float*>(dyn);  // 2 x kFRows x W fp32 (bulk-copied chunks of Y)
  __shared__ uint64_t ld_bar[2];
  __shared__ int ticket;
  constexpr int npairs = W * W;
  // Gram on the fp64 tensor cores (DMMA m8n8k4): for a 4-row slice r0..r0+3 of the chunk, lane l
  // holds v[a] = Y[r0 + l%4][8a + l/4] -- at once the A fragment (rows 8a..8a+7 of Y^T) and the B
  // fragment (columns 8b..8b+7 of Y) of every 8 x 8 block (a, b), a <= b, of G.  Each fp32 is
  // converted once and feeds NB DMMAs from registers (the FFMA-tile form was shared-memory bound).
  constexpr int NB = W / 8, NBLK = NB * (NB + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  double acc[NBLK][2];
#pragma unroll
  for (int q = 0; q < NBLK; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int c = 0; c < nchunk; ++c) {
    const int64_t r0 = r_begin + (int64_t)c * kFRows;
    const int nr = (int)(r_end - r0 < kFRows ? r_end - r0 : kFRows);
    mbar_wait(&ld_bar[c & 1], (c >> 1) & 1);
    const float* bY = buf + (c & 1) * kFRows * W;
    for (int sl = warp; 4 * sl < nr; sl += 8) {
      const int rr = 4 * sl + (lane & 3);
      double v[NB];
#pragma unroll
      for (int a = 0; a < NB; ++a) v[a] = rr < nr ? (double)bY[rr * W + 8 * a + (lane >> 2)] : 0.0;
      int blk = 0;
#pragma unroll
      for (int a = 0; a < NB; ++a)
#pragma unroll
        for (int b = a; b < NB; ++b, ++blk)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[blk][0]), "+d"(acc[blk][1])
                       : "d"(v[a]), "d"(v[b]));
    }
    __syncthreads();  // every warp is done with buffer (c & 1): refill it with chunk c + 2
    if (threadIdx.x == 0 && c + 2 < nchunk) issue(c + 2);
  }
  if (blockIdx.x == 0) { FS_T(1) }
  // fixed-order sum of the 8 warps' blocks (warp 0 stores, warps 1..7 add in turn), then the block
  // partial, both halves (block (a, a): the entry with row <= col goes to both positions)
  double* S = dyn;  // NBLK x 64 (the chunk buffers are free)
  for (int w = 0; w < 8; ++w) {
    if (warp == w)
#pragma unroll
      for (int q = 0; q < NBLK; ++q)
#pragma unroll
        for (int i = 0; i < 2; ++i) S[q * 64 + 2 * lane + i] = w == 0 ? acc[q][i] : S[q * 64 + 2 * lane + i] + acc[q][i];
    __syncthreads();
  }
  double* part = jb.gpart + (int64_t)blockIdx.x * npairs;
  for (int e = threadIdx.x; e < NBLK * 64; e += 256) {
    int q = e / 64, a = 0, b = 0;
    for (int aa = 0, k = q; aa < NB; ++aa) {
      if (k < NB - aa) { a = aa; b = aa + k; break; }
      k -= NB - aa;
    }
    const int l = (e % 64) / 2, i = e % 2;
    const int row = 8 * a + l / 4, col = 8 * b + 2 * (l % 4) + i;
    const double val = S[e];
    if (a != b || row <= col) {
      part[row * W + col] = val;
      part[col * W + row] = val;
    }
  }
  // two-level fixed-order reduction of the block partials: the last block of each group of 16
  // sums its group (-> gpart[nb + g]), the last group finisher sums the groups (-> G).  Counters:
  // counter[0] = groups done, counter[1 + g] = blocks of group g done (all re-armed to 0).
  const int nb = (int)gridDim.x;
  const int grp = blockIdx.x / 16, ngrp = (nb + 15) / 16;
  const int gsize = nb - 16 * grp < 16 ? nb - 16 * grp : 16;
  if (blockIdx.x == 0) { FS_T(2) }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(jb.counter + 1 + grp, 1);
  __syncthreads();
  if (ticket != gsize - 1) return;
  __threadfence();
  FS_T(3)
  // G also into shared memory behind the solvers' scratch: the solver reads it from there, not back
  // through L2 (W <= 32)
  double* Gs = dyn + 3 * 32 * 33;
  if (ngrp == 1) {  // one group: its finisher is the last block (the same sums as the two-level path)
    for (int pr = threadIdx.x; pr < npairs; pr += 256) {
      const double a = sum_strided(jb.gpart + pr, npairs, gsize);
      const double g = 0.0 + a;  // the second level adds the single group sum to 0
      jb.G[pr] = g;
      if (W <= 32) Gs[pr] = g;
    }
    if (threadIdx.x == 0) jb.counter[1] = 0;
  } else {
    for (int pr = threadIdx.x; pr < npairs; pr += 256) {
      const double a = sum_strided(jb.gpart + (int64_t)(16 * grp) * npairs + pr, npairs, gsize);
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
      const double a = sum_strided(jb.gpart + (int64_t)nb * npairs + pr, npairs, ngrp);
      jb.G[pr] = a;
      if (W <= 32) Gs[pr] = a;
    }
  }
  if (threadIdx.x == 0) jb.counter[0] = 0;  // re-arm for the next launch (stream ordered)
  if (jb.cmax && threadIdx.x < 64) jb.cmax[threadIdx.x] = 0u;  // the next apply64's column maxima
  __threadfence_block();
  __syncthreads();
  FS_T(4)
  if constexpr (W <= 32) {
    static_assert(3 * 32 * 33 * 8 + W * W * 8 <= kDynSmem && eig_smem_bytes(W) <= 3 * 32 * 33 * 8, "G staging");
    if (mode == 0 && threadIdx.x < 32) {
      warp_chol_orth<W>(Gs, jb.T64, dyn, dyn + 32 * 33, dyn + 2 * 32 * 33);
    }
    if (mode == 1) dev_eig_trunc<W>(Gs, jb.T, jb.r, dyn);
  } else {
    if (mode == 0) dev_chol_orth<W>(jb.G, jb.T64, dyn);
    else if (mode == 1) dev_eig_trunc<W>(jb.G, jb.T, jb.r, dyn);
  }
  FS_T(5)
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
  // one wave: two blocks fit per SM (66.5 KB of shared memory and 98 registers x 256 threads each;
  // ncu), and 444 blocks had run as 1.5 waves (802 816-row panel: half the SMs idle for a third)
  const int64_t wave = 2LL * sm_count();
  if (nb > wave) nb = wave;
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
// Operands staged in shared memory first (every product then reads shared memory only).
__global__ void __launch_bounds__(256) k_cross_small(const double* __restrict__ C, const float* __restrict__ VWa,
                                                     const float* __restrict__ VWb, int n, int r,
                                                     float* __restrict__ VWbM) {
  ::lrqmm::pdl_enter();
  extern __shared__ __align__(16) double xs[];
  double* Cs = xs;                       // n x n
  double* T1 = Cs + kN * kN;             // n x 32 : C VWa
  double* M = T1 + kN * 32;              // 32 x 32: VWb^T T1
  float* A = reinterpret_cast<float*>(M + 32 * 32);  // VWa, n x n
  float* B = A + kN * kN;                            // VWb, n x n
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += 256) {
    Cs[e] = C[e];
    A[e] = VWa[e];
    B[e] = VWb[e];
  }
  __syncthreads();
  for (int e = tid; e < n * r; e += 256) {
    const int i = e / r, o = e % r;
    double a = 0.0;
    for (int c = 0; c < n; ++c) a = fma(Cs[i * n + c], (double)A[c * n + o], a);
    T1[i * 32 + o] = a;
  }
  __syncthreads();
  for (int e = tid; e < r * r; e += 256) {
    const int u = e / r, o = e % r;
    double a = 0.0;
    for (int i = 0; i < n; ++i) a = fma((double)B[i * n + u], T1[i * 32 + o], a);
    M[u * 32 + o] = a;
  }
  __syncthreads();
  for (int e = tid; e < n * r; e += 256) {
    const int i = e / r, o = e % r;
    double a = 0.0;
    for (int u = 0; u < r; ++u) a = fma((double)B[i * n + u], M[u * 32 + o], a);
    VWbM[i * n + o] = (float)a;
  }
}

void launch_cross_small(const double* C, const float* VWa, const float* VWb, int n, int r, float* VWbM,
                        cudaStream_t st) {
  constexpr int smem = (kN * kN + kN * 32 + 32 * 32) * 8 + 2 * kN * kN * 4;
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_cross_small, smem, attr);
  launch_pdl(k_cross_small, 1, 256, smem, st, C, VWa, VWb, n, r, VWbM); ++launch_counter();
}

}  // namespace lrqmm
