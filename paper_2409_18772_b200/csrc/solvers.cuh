// Small dense solvers of the RSVD shared by the separate-launch kernels (smallsolve2.cu) and the
// fused pass epilogues (skinny_tc.cu): the pivoted Cholesky QR transform (one warp) and the cyclic
// parallel Jacobi truncation eigensolver (a group of NT threads).
#pragma once
#include "common.cuh"

namespace lrqmm {

constexpr int kSolveN = 64;

// named barrier over `count` threads (id 0 over blockDim.x threads is the CTA barrier)
LRQMM_DEV void group_bar(int id, int count) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }

// ------------------------------------------------- one-warp solvers (n <= 32)
// Pivoted Cholesky QR transform, one warp, lane j = column j, no row/column swaps:
//   lane j keeps column j of S (the Schur complement, on the ORIGINAL indices) in registers
//   s[0..n) and its diagonal d_j.  Step k: pivot p = argmax d_j over the remaining lanes (one
//   packed-key __reduce_max_sync pair); l_j = S[p, j] / sqrt(d_p) (l_p = sqrt(d_p)), where S[p, j]
//   is lane j's own s[p] (a select over the unrolled registers, overlapping the rsqrt); l goes to
//   Lsm row k; S -= l l^T is register-only (l_i broadcast from Lsm); d -= l^2.  Per step the
//   dependent chain is argmax -> rsqrt (MUFU approximation + two Newton steps) -> l -> one broadcast
//   round, no shared-memory matrix traffic.
//   The transform (mathematically T = P L^-T) is formed after the factorisation as Gram-Schmidt in
//   the G inner product, lane = row of T with the row in registers:
//     t_k = (e_{p_k} - sum_{m<k} t_m L[p_k, m]) / L[p_k, k],
//   so Q = Y T has orthonormal columns.  Pivots below 1e-10 x the largest diagonal entry end the
//   factorisation (reading #12): the remaining columns of T are zero (rows >= rank of L, their
//   pivots and 1 / L[p_k, k] are zeroed, so the transform loop is branch-free).
//   Shared scratch: sm (>= 2 x 32 doubles: pivot indices, 1 / L[p_k, k]), Lsm (32 x 33 doubles),
//   Tsm (32 x 33 doubles, output staging).
// Output T64[j * n + k] = T[j, k].
#ifdef LRQMM_CHOL_PROF
__device__ long long chol_prof[8];  // micro-benchmark only (tools/eig_bench.cu): phase clocks
#define CHOL_MARK(i) \
  if (lane == 0) chol_prof[i] = clock64();
#else
#define CHOL_MARK(i)
#endif
template <int n>
__device__ void warp_chol_orth(const double* G, double* T64, double* sm, double* Lsm, double* Tsm) {
  const int lane = threadIdx.x & 31;
  CHOL_MARK(0)
  int* piv = reinterpret_cast<int*>(sm);
  double* invs = sm + 32;
  double s[n];
  double d = 0.0;
  // column `lane` of the symmetrised G; every load of a chunk of 8 rows issues before its use (G may
  // be in global memory: one round trip per chunk, not per row)
#pragma unroll
  for (int i0 = 0; i0 < n; i0 += 8) {
    double ga[8], gb[8];
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (i0 + t < n) {
        ga[t] = lane < n ? G[(i0 + t) * n + lane] : 0.0;
        gb[t] = lane < n ? G[lane * n + i0 + t] : 0.0;
      }
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (i0 + t < n) {
        s[i0 + t] = 0.5 * (ga[t] + gb[t]);
        if (i0 + t == lane) d = s[i0 + t];
      }
  }
  double dmax = d;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const double thr = 1e-10 * dmax;
  CHOL_MARK(1)
  bool done = lane >= n;
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
    // 1 / sqrt(dp): MUFU approximation + two Newton steps (fp64 accurate)
    double inv;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(dp));
    const double hdp = -0.5 * dp;
    inv = inv * fma(hdp, inv * inv, 1.5);
    inv = inv * fma(hdp, inv * inv, 1.5);
    const double lkk = dp * inv;
    // S[p, lane] = s[p]: a select over the unrolled registers, as a tree on the bits of p for n = 32
    // (tools/eig_bench.cu: n = 32 11.8 -> 10.9 us; the linear chain is faster at n = 24, 8.9 vs 10.8)
    double spj;
    if constexpr (n >= 32) {
      double v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = i < n ? s[i] : 0.0;
#pragma unroll
      for (int w = 1; w < 32; w *= 2)
#pragma unroll
        for (int i = 0; i < 32; i += 2 * w) v[i] = (p & w) ? v[i + w] : v[i];
      spj = v[0];
    } else {
      spj = s[0];
#pragma unroll
      for (int i = 1; i < n; ++i) spj = p == i ? s[i] : spj;
    }
    const double l = done ? 0.0 : (lane == p ? lkk : spj * inv);
    if (lane == p) done = true;
    Lsm[k * 33 + lane] = l;
    if (lane == 0) {
      piv[k] = p;
      invs[k] = inv;
    }
    if (!done) d = fma(-l, l, d);
    __syncwarp();
    // S -= l l^T (registers; l_i broadcast; a finished lane's column is never read again)
#pragma unroll
    for (int i = 0; i < n; ++i) s[i] = fma(-Lsm[k * 33 + i], l, s[i]);
  }
  const int rk = k;
  // rows rk.. of L and the pivots beyond the rank: zero, so that the transform below is branch-free
  // (t[kk] = 0 for kk >= rk)
  for (int kk = rk; kk < n; ++kk) {
    Lsm[kk * 33 + lane] = 0.0;
    if (lane == 0) {
      piv[kk] = 0;
      invs[kk] = 0.0;
    }
  }
  __syncwarp();
  CHOL_MARK(2)
  // T row `lane` (registers, reusing s): t[k] = (e_p - sum_{m<k} t[m] L[p, m]) * inv_k, partial sums
  // over m mod 4 in order, as the factorisation-time form
  double* t = s;
#pragma unroll
  for (int kk = 0; kk < n; ++kk) {
    const int p = piv[kk];
    double a[4] = {lane == p ? 1.0 : 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int m = 0; m < kk; ++m) a[m & 3] = fma(-t[m], Lsm[m * 33 + p], a[m & 3]);
    t[kk] = ((a[0] + a[1]) + (a[2] + a[3])) * invs[kk];
  }
  CHOL_MARK(3)
  // coalesced output through Tsm (column c of T at Tsm[c * 33 + row])
#pragma unroll
  for (int c = 0; c < n; ++c) Tsm[c * 33 + lane] = t[c];
  __syncwarp();
  for (int e = lane; e < n * n; e += 32) T64[e] = Tsm[(e % n) * 33 + e / n];
  __syncwarp();
  CHOL_MARK(4)
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
#ifndef LRQMM_JAC_NEWTON
#define LRQMM_JAC_NEWTON 2
#endif
#ifndef LRQMM_JAC_TOL
#define LRQMM_JAC_TOL 1e-16  // off(A)^2 <= tol * diag(A)^2 ends the sweeps (reading #29)
#endif
__device__ __forceinline__ double jac_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double jac_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
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

// Run by a group of NT threads (tid = 0 .. NT-1 within the group, whole warps) that synchronise with
// named barrier `bar` (bar 0 over blockDim.x threads is the CTA barrier).  Shared scratch: dyn (the
// eig_smem_bytes(n) matrices) and aux (eig_aux_bytes(NT): per-warp sums, scale, na, order).
#ifdef LRQMM_EIG_STATS
__device__ int eig_stats_steps;
#endif
#ifndef LRQMM_EIG_SKIP
#define LRQMM_EIG_SKIP 0  // micro-benchmark only (tools/eig_bench.cu): 1 no V, 2 fixed rotation, 4 no A blocks
#endif
#ifndef LRQMM_EIG_SWEEPS
#define LRQMM_EIG_SWEEPS 0  // micro-benchmark only: run exactly this many sweeps (0: convergence test)
#endif
// NA (<= n): the largest live size na the caller guarantees (sizes the per-thread block / V slots)
template <int n, int NT, int NA = n>
__device__ void group_eig_trunc(const double* G, float* T, int r, double* dyn, double* aux, int tid, int bar) {
  static_assert(NA <= n && NA % 2 == 0, "live size");
  constexpr int ld = n + 1;
  constexpr int kBlk = ((NA / 2) * (NA / 2) + NT - 1) / NT, kV = ((NA / 2) * NA + NT - 1) / NT;
  constexpr int NW = NT / 32;
  double* Abuf = dyn;                 // 2 x n x ld (ping-pong, relabelled)
  double* V = dyn + 2 * n * ld;       // n x ld, original labels
  double (*red)[2] = reinterpret_cast<double (*)[2]>(aux);   // NW x 2
  double& scale_s = aux[2 * NW];
  int& na_s = *reinterpret_cast<int*>(aux + 2 * NW + 1);
  int* order = reinterpret_cast<int*>(aux + 2 * NW + 2);     // kSolveN
  const int lane = tid & 31, warp = tid >> 5;
  auto sync = [&] { group_bar(bar, NT); };
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
      na_s = na < 2 ? 2 : (na > NA ? NA : na);
    }
  }
  sync();
  const int na = na_s, half = na / 2, m = na - 1;
  // normalised copy (eigenvectors are scale invariant): entries O(1), so the rotation angle
  // can be computed in fp32 without under/overflow.  At step 0 position d holds index d.
  double off = 0.0, dg = 0.0;
  for (int e = tid; e < n * n; e += NT) {
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
    sync();
    double o2 = 0.0, d2 = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) { o2 += red[w][0]; d2 += red[w][1]; }
    return (o2 <= LRQMM_JAC_TOL * d2) || (o2 == 0.0);
  };
  bool stop = converged(off, dg);
  // fixed per-thread work: its 2x2 blocks, its V entries, the pair whose rotation it evaluates.  A
  // thread without a block / V entry runs the same instructions on the padding column n of row 0
  // (never read), so a step is one basic block the scheduler can interleave.
  int bk1[kBlk], bk2[kBlk], brd[kBlk][4], bwr[kBlk][4];
  bool bok[kBlk], bdiag[kBlk];
#pragma unroll
  for (int u = 0; u < kBlk; ++u) {
    const int e = tid + NT * u;
    bok[u] = e < half * half;
    const int k1 = bok[u] ? e / half : 0, k2 = bok[u] ? e % half : 0;
    bk1[u] = k1;
    bk2[u] = k2;
    bdiag[u] = k1 == k2;
    const int P1 = jac_P(k1), Q1 = jac_Q(k1, na), P2 = jac_P(k2), Q2 = jac_Q(k2, na);
    brd[u][0] = P1 * ld + P2; brd[u][1] = P1 * ld + Q2; brd[u][2] = Q1 * ld + P2; brd[u][3] = Q1 * ld + Q2;
    const int p1 = jac_sigma(P1, na), q1 = jac_sigma(Q1, na), p2 = jac_sigma(P2, na), q2 = jac_sigma(Q2, na);
    if (bok[u]) {
      bwr[u][0] = p1 * ld + p2; bwr[u][1] = p1 * ld + q2; bwr[u][2] = q1 * ld + p2; bwr[u][3] = q1 * ld + q2;
    } else {
      bwr[u][0] = bwr[u][1] = bwr[u][2] = bwr[u][3] = n;
    }
  }
  int vk[kV], vrow[kV], vP[kV], vQ[kV];
  bool vok[kV];
#pragma unroll
  for (int u = 0; u < kV; ++u) {
    const int e = tid + NT * u;
    vok[u] = e < half * na;
    vk[u] = vok[u] ? e / na : 0;
    vrow[u] = (vok[u] ? e % na : 0) * ld;
    vP[u] = jac_P(vk[u]);
    vQ[u] = jac_Q(vk[u], na);
  }
  const int kr = lane < half ? lane : 0;  // lane k < half evaluates pair k's rotation (the rest: pair 0)
  const int rpp = jac_P(kr) * (ld + 1), rqq = jac_Q(kr, na) * (ld + 1), rpq = jac_P(kr) * ld + jac_Q(kr, na);
  // rotation (c, s) of a pair from its (app, aqq, apq); bitwise identical wherever it is evaluated.
  // t = tan(phi) is the smaller root of t^2 + 2 theta t - 1 = 0, theta = d / e, d = aqq - app,
  // e = 2 apq, written t = e / (d + sign(d) sqrt(d^2 + e^2)) so that it takes one rsqrt and one
  // reciprocal (MUFU.RSQ64H / RCP64H approximations: the angle's accuracy only affects convergence);
  // c = 1 / sqrt(1 + t^2) then gets two Newton steps so that c^2 + s^2 = 1 to fp64 rounding and every
  // rotation is an exact similarity.  Entries are normalised (|a| <= 1); |apq| <= 1e-150 is no
  // rotation (and keeps d^2 + e^2 a normal number).
  auto rotation = [&](double app, double aqq, double apq, double& c, double& s) {
    const double d = aqq - app, e = 2.0 * apq;
    const double x = fma(d, d, e * e);
    const double r = x * jac_rsqrt(x);
    const double t0 = e * jac_rcp(d + copysign(r, d));
    double t = fabs(apq) > 1e-150 ? t0 : 0.0;
    if (LRQMM_EIG_SKIP & 2) t = 0.75;
    const double x1 = fma(t, t, 1.0), hx = -0.5 * x1;
    double y = jac_rsqrt(x1);
    y = y * fma(hx, y * y, 1.5);
#if LRQMM_JAC_NEWTON > 1
    y = y * fma(hx, y * y, 1.5);
#endif
    c = y;
    s = t * y;
  };
  // V' = V J of a step, applied one step late (off the A chain): rotations (cv, sv) of lane k < half
  // = pair k of the step whose column labels are (op, oq).  Labels advance by one position per step
  // (orig(s + 1, d) = orig(s, d) + 1 mod m over 1..m; position 0 keeps label 0).  Before the first
  // step the update is the identity on the labels of step m - 1 (a valid pairing): no branch.
  double cv = 1.0, sv = 0.0;
  int op[kV], oq[kV];
#pragma unroll
  for (int u = 0; u < kV; ++u) {
    op[u] = jac_orig(m - 1, vP[u], m);
    oq[u] = jac_orig(m - 1, vQ[u], m);
  }
  // the update is split: its loads and shuffles are issued at the top of a step next to the A loads,
  // its arithmetic and stores after the step's rotation (the entries are this thread's alone)
  double ck[kV], sk[kV], x0[kV], x1[kV];
  int vp[kV], vq[kV];
  auto v_load = [&] {
#pragma unroll
    for (int u = 0; u < kV; ++u) {  // the entries of different u are distinct
      ck[u] = __shfl_sync(0xffffffffu, cv, vk[u]);
      sk[u] = __shfl_sync(0xffffffffu, sv, vk[u]);
      vp[u] = vok[u] ? vrow[u] + op[u] : n;
      vq[u] = vok[u] ? vrow[u] + oq[u] : n;
      x0[u] = V[vp[u]];
      x1[u] = V[vq[u]];
    }
  };
  auto v_store = [&] {
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      if (!(LRQMM_EIG_SKIP & 1)) {
        V[vp[u]] = ck[u] * x0[u] - sk[u] * x1[u];
        V[vq[u]] = sk[u] * x0[u] + ck[u] * x1[u];
      }
      op[u] = op[u] == 0 ? 0 : (op[u] == m ? 1 : op[u] + 1);
      oq[u] = oq[u] == 0 ? 0 : (oq[u] == m ? 1 : oq[u] + 1);
    }
  };
  int total = 0;  // steps done
  // the step loop unrolled by two (the ping-pong parity is static in each half: fixed addresses)
  int sstep = 0, sweep = 0;
  bool run = LRQMM_EIG_SWEEPS ? true : !stop;
  while (run) {
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      if (!run) break;
      const double* Ac = Abuf + par * n * ld;
      double* An = Abuf + (1 - par) * n * ld;
      const bool last = sstep + 1 == m;
      // every load of the step first: the rotation operands and the 2x2 blocks
      const double app = Ac[rpp], aqq = Ac[rqq], apq = Ac[rpq];
      double bv[kBlk][4];
#pragma unroll
      for (int u = 0; u < kBlk; ++u) {
        bv[u][0] = Ac[brd[u][0]]; bv[u][1] = Ac[brd[u][1]]; bv[u][2] = Ac[brd[u][2]]; bv[u][3] = Ac[brd[u][3]];
      }
      v_load();  // the previous step's V update (rotations in cv, sv: independent of this step's chain)
      double c, s;
      rotation(app, aqq, apq, c, s);
      v_store();
      cv = c;
      sv = s;
      off = 0.0;
      dg = 0.0;
#pragma unroll
      for (int u = 0; u < kBlk && !(LRQMM_EIG_SKIP & 4); ++u) {
        const double c1 = __shfl_sync(0xffffffffu, c, bk1[u]), s1 = __shfl_sync(0xffffffffu, s, bk1[u]);
        const double c2 = __shfl_sync(0xffffffffu, c, bk2[u]), s2 = __shfl_sync(0xffffffffu, s, bk2[u]);
        const double a = bv[u][0], b = bv[u][1], cc = bv[u][2], d = bv[u][3];
        const double ra = c1 * a - s1 * cc, rb = c1 * b - s1 * d;
        const double rc = s1 * a + c1 * cc, rd = s1 * b + c1 * d;
        const double v0 = c2 * ra - s2 * rb, v1 = s2 * ra + c2 * rb, v2 = c2 * rc - s2 * rd, v3 = s2 * rc + c2 * rd;
        An[bwr[u][0]] = v0;
        An[bwr[u][1]] = v1;
        An[bwr[u][2]] = v2;
        An[bwr[u][3]] = v3;
        if (last && bok[u]) {
          if (bdiag[u]) { dg += v0 * v0 + v3 * v3; off += v1 * v1 + v2 * v2; }
          else off += (v0 * v0 + v1 * v1) + (v2 * v2 + v3 * v3);
        }
      }
      if (last) stop = converged(off, dg);  // its barrier ends the step
      else sync();
      ++total;
      if (++sstep == m) {
        sstep = 0;
        ++sweep;
        run = LRQMM_EIG_SWEEPS ? sweep < LRQMM_EIG_SWEEPS : (sweep < 30 && !stop);
      }
    }
  }
  v_load();
  v_store();
  sync();
#ifdef LRQMM_EIG_STATS
  if (tid == 0) eig_stats_steps = total;  // micro-benchmark only (tools/eig_bench.cu)
#endif
  // position d < na holds eigenvalue A[d][d] with eigenvector V[:, orig(total mod m, d)];
  // indices >= na: eigenvalue 0, eigenvector e_d
  const double* Af = Abuf + (total & 1) * n * ld;
  const int sf = total % m;
  for (int t = tid; t < n; t += NT) {
    int rank = 0;
    const double li = t < na ? Af[t * ld + t] : 0.0;
    for (int j = 0; j < n; ++j) {
      const double lj = j < na ? Af[j * ld + j] : 0.0;
      rank += (lj > li) || (lj == li && j < t);
    }
    order[rank] = t < na ? jac_orig(sf, t, m) : t;
  }
  sync();
  for (int e = tid; e < n * n; e += NT) {
    const int a = e / n, o = e % n;
    T[a * n + o] = (o < r) ? (float)V[a * ld + order[o]] : 0.f;
  }
}
__host__ __device__ constexpr int eig_aux_bytes(int NT) { return (2 * (NT / 32) + 2) * 8 + 64 * 4; }

// The group size per n (tools/eig_bench.cu: n = 24 30.0 us at 192 threads vs 33.8 at 256, n = 32
// 61.2 us at 256); the CTA's other threads leave, the group synchronises on named barrier 1.
// n = 32 with at most 26 live columns (r + p <= 25, c4's r = 20, p = 5): the n = 24 shape of the
// work (169 blocks, 192 threads); n = 24 with at most 22 (121 blocks, 128 threads).  The live size
// is read off G's diagonal first (one warp).
template <int n>
__device__ void dev_eig_trunc(const double* G, float* T, int r, double* dyn) {
  constexpr int NT = n == 24 ? 192 : 256;
  __shared__ double aux[(eig_aux_bytes(NT) + 7) / 8];
  if constexpr (n == 24 || n == 32) {
    __shared__ int live_s;
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const int last = __reduce_max_sync(0xffffffffu, lane < n && G[lane * n + lane] != 0.0 ? lane : -1);
      if (lane == 0) live_s = (last + 2) & ~1;
    }
    __syncthreads();
    if constexpr (n == 32) {
      if (live_s <= 26) {
        if (threadIdx.x < 192) group_eig_trunc<n, 192, 26>(G, T, r, dyn, aux, threadIdx.x, 1);
        return;
      }
    } else {
      if (live_s <= 22) {  // r + p <= 21 (c2 / c3: r = 16, p = 5): 26.8 vs 30.1 us
        if (threadIdx.x < 128) group_eig_trunc<n, 128, 22>(G, T, r, dyn, aux, threadIdx.x, 1);
        return;
      }
    }
  }
  if (threadIdx.x < NT) group_eig_trunc<n, NT>(G, T, r, dyn, aux, threadIdx.x, 1);
}


// --------------------------------------------- one-warp one-sided Jacobi (truncation)
// Top-r eigenvectors of a symmetric PSD G (n x n, n <= 32) by one-sided (Hestenes) Jacobi on the
// columns of M = G itself, one warp, every column in one lane's registers, no shared memory and no
// barriers.  M V has orthogonal columns iff V diagonalises M^T M = G^2, i.e. V holds G's
// eigenvectors (PSD: the order of lambda^2 is the order of lambda), and then column j of M V is
// G v_j = lambda_j v_j: the eigenvectors are the normalised final columns and lambda_j their norms, so
// V is never accumulated.  Round-robin pairing (circle method, player n_even - 1 fixed): lanes j and
// partner(j, t) exchange columns by shuffle and BOTH compute the same rotation from the same
// (low-lane, high-lane) ordered dot products (bitwise identical), zeroing their inner product.
// A pair is rotated while |<m_p, m_q>| > 1e-15 sqrt(|m_p|^2 |m_q|^2); the sweeps stop when the
// largest such ratio seen in a sweep is <= 1e-8 (reading #29's 1e-8 relative off-diagonal, here of
// G^2 in the current basis).  Exactly zero columns (the zero-padded sketch columns) stay zero and
// give a zero "eigenvector" (their U Sigma column is zero either way).
// Output T[a * n + o] = component a of the o-th eigenvector (descending lambda, ties by index), o < r;
// 0 for o >= r.
LRQMM_DEV int rr_partner(int j, int t, int np) {
  if (j == np - 1) return t;
  if (j == t) return np - 1;
  int p = 2 * t - j;
  p %= (np - 1);
  return p < 0 ? p + np - 1 : p;
}

template <int n>
__device__ void warp_eig_trunc(const double* G, float* T, int r) {
  constexpr int np = (n + 1) & ~1;
  const int lane = threadIdx.x & 31;
  double m[n];
  double dmax = 0.0;
  if (lane < n) dmax = fabs(G[lane * n + lane]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const double sc = dmax > 0.0 ? 1.0 / dmax : 1.0;  // O(1) entries: no overflow in the dot products
#pragma unroll
  for (int i = 0; i < n; ++i) m[i] = lane < n ? 0.5 * (G[i * n + lane] + G[lane * n + i]) * sc : 0.0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double worst = 0.0;
    for (int t = 0; t < np - 1; ++t) {
      const int p = rr_partner(lane, t, np);
      double mp[n];
#pragma unroll
      for (int i = 0; i < n; ++i) mp[i] = __shfl_sync(0xffffffffu, m[i], p & 31);
      const bool lo = lane < p;
      // dot products of (low, high) in a fixed order, four partial sums each
      double aa[4] = {0.0, 0.0, 0.0, 0.0}, bb[4] = {0.0, 0.0, 0.0, 0.0}, ab[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const double x = lo ? m[i] : mp[i], y = lo ? mp[i] : m[i];
        aa[i & 3] = fma(x, x, aa[i & 3]);
        bb[i & 3] = fma(y, y, bb[i & 3]);
        ab[i & 3] = fma(x, y, ab[i & 3]);
      }
      const double a = (aa[0] + aa[1]) + (aa[2] + aa[3]);
      const double b = (bb[0] + bb[1]) + (bb[2] + bb[3]);
      const double g = (ab[0] + ab[1]) + (ab[2] + ab[3]);
      const double nab = sqrt(a * b);
      if (lane < n && p < n && nab > 0.0 && fabs(g) > 1e-15 * nab) {
        worst = fmax(worst, fabs(g) / nab);
        const double zeta = (b - a) / (2.0 * g);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = 1.0 / sqrt(fma(tt, tt, 1.0)), s = c * tt;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const double x = lo ? m[i] : mp[i], y = lo ? mp[i] : m[i];
          m[i] = lo ? c * x - s * y : s * x + c * y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    if (worst <= 1e-8) break;
  }
  // lambda_j = |column j|; rank by descending lambda (ties: lower index first)
  double nn = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) nn = fma(m[i], m[i], nn);
  const double lam = lane < n ? sqrt(nn) : -1.0;
  int rank = 0;
  for (int j = 0; j < n; ++j) {
    const double lj = __shfl_sync(0xffffffffu, lam, j);
    rank += (lj > lam) || (lj == lam && j < lane);
  }
  if (lane < n) {
    if (rank < r) {
      const double inv = lam > 0.0 ? 1.0 / lam : 0.0;
#pragma unroll
      for (int a = 0; a < n; ++a) T[a * n + rank] = (float)(m[a] * inv);
    }
    for (int o = r; o < n; ++o) T[lane * n + o] = 0.f;
  }
}

}  // namespace lrqmm
