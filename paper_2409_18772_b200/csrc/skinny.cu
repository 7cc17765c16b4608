// K2/K3 — tall-skinny products over the quantization residual (RSVD passes of
// Algorithm 1 / reading #11) and the cross products of
// Algorithm 2; plus the fp64 Gram and the
// small "apply a W x W matrix" kernels used by orthonormalisation and assembly.
//
// The residual R and the dequantised X~ are never stored: every pass re-reads
// the fp32 side X (4 B/element, HBM-bound) and recomputes the code and
// F(x) from lambda with the same exact rounding as K1.
// All reductions are deterministic (fixed split, fixed summation order, no
// float atomics).
#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

// exact rounding (same arithmetic as K1, kept local to this translation unit)
LRQMM_DEV float code_f(float lam, float x, int mode, int qmax) {
  const float p = __fmul_rn(lam, x);
  const float e = __fmaf_rn(lam, x, -p);
  float c;
  if (mode == kRoundFloor) {
    c = floorf(p);
    if (p == c && (e < 0.f || (p == 0.f && x < 0.f))) c -= 1.f;
  } else if (mode == kRoundTrunc) {
    c = truncf(p);
    if (p == c && p != 0.f) {
      if (p > 0.f && e < 0.f) c -= 1.f;
      if (p < 0.f && e > 0.f) c += 1.f;
    }
  } else {
    c = rintf(p);
    const float fl = floorf(p);
    if (p - fl == 0.5f && e != 0.f) c = (e > 0.f) ? fl + 1.f : fl;
  }
  const float q = static_cast<float>(qmax);
  return fminf(fmaxf(c, -q), q);
}

struct FVals {
  float res, deq;
};
// residual r = (lambda*x - code)/lambda, dequant x~ = code/lambda
LRQMM_DEV FVals fvals(float lam, float inv_lam, float x, int mode, int qmax) {
  const float c = code_f(lam, x, mode, qmax);
  FVals v;
  v.res = __fmul_rn(__fmaf_rn(lam, x, -c), inv_lam);
  v.deq = __fmul_rn(c, inv_lam);
  return v;
}

// ------------------------------------------------------------------ ROW mode
// OUT[i,c] = sum_{j in split} F1(x_ij) P1[j,c]  (+ OUT2 with F2, P2)
template <int W, int TM, bool kDual>
__global__ void __launch_bounds__(256) k2_proj_rows(SideView s, const float* __restrict__ P1, int f1,
                                                    const float* __restrict__ P2, int f2, float* __restrict__ out1,
                                                    float* __restrict__ out2, int kchunk) {
  constexpr int BM = 256 * TM;
  constexpr int BK = 16;
  constexpr int kLoads = BM * BK / 4 / 256;  // float4 per thread per tile
  __shared__ float Xs[BM][BK + 1];
  __shared__ __align__(16) float Ps1[BK][W];
  __shared__ __align__(16) float Ps2[kDual ? BK : 1][kDual ? W : 4];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row_base = (int64_t)blockIdx.x * BM;
  const int k_begin = blockIdx.y * kchunk;
  const int k_end = min(s.K, k_begin + kchunk);
  const bool vec = ((reinterpret_cast<uintptr_t>(s.X) & 15) == 0) && (s.ldx % 4 == 0);

  float acc1[TM][W];
  float acc2[kDual ? TM : 1][kDual ? W : 1];
#pragma unroll
  for (int t = 0; t < TM; ++t)
#pragma unroll
    for (int c = 0; c < W; ++c) {
      acc1[t][c] = 0.f;
      if (kDual) acc2[t][c] = 0.f;
    }
  float lam[TM], inv[TM];
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    const int64_t row = row_base + warp * (32 * TM) + lane + 32 * t;
    lam[t] = row < s.rows ? s.lam[row] : 1.f;
    inv[t] = __frcp_rn(lam[t]);
  }

  float4 pre[kLoads];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
      const int f = tid + 256 * u;
      const int rl = f >> 2, ch = f & 3;
      const int64_t row = row_base + rl;
      const int col = k0 + ch * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < s.rows) {
        const float* xr = s.X + row * s.ldx;
        if (vec && col + 3 < k_end) {
          v = __ldcs(reinterpret_cast<const float4*>(xr + col));
        } else {
          if (col + 0 < k_end) v.x = xr[col + 0];
          if (col + 1 < k_end) v.y = xr[col + 1];
          if (col + 2 < k_end) v.z = xr[col + 2];
          if (col + 3 < k_end) v.w = xr[col + 3];
        }
      }
      pre[u] = v;
    }
  };

  if (k_begin < k_end) load_tile(k_begin);
  for (int k0 = k_begin; k0 < k_end; k0 += BK) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
      const int f = tid + 256 * u;
      const int rl = f >> 2, ch = f & 3;
      Xs[rl][ch * 4 + 0] = pre[u].x;
      Xs[rl][ch * 4 + 1] = pre[u].y;
      Xs[rl][ch * 4 + 2] = pre[u].z;
      Xs[rl][ch * 4 + 3] = pre[u].w;
    }
    for (int e = tid; e < BK * W; e += 256) {
      const int j = e / W, c = e % W;
      const bool in = (k0 + j) < k_end;
      Ps1[j][c] = in ? P1[(int64_t)(k0 + j) * W + c] : 0.f;
      if (kDual) Ps2[j][c] = in ? P2[(int64_t)(k0 + j) * W + c] : 0.f;
    }
    __syncthreads();
    if (k0 + BK < k_end) load_tile(k0 + BK);
#pragma unroll 4
    for (int j = 0; j < BK; ++j) {
      float a1[TM], a2[TM];
#pragma unroll
      for (int t = 0; t < TM; ++t) {
        const float x = Xs[warp * (32 * TM) + lane + 32 * t][j];
        const FVals fv = fvals(lam[t], inv[t], x, s.mode, s.qmax);
        a1[t] = (f1 == kFRes) ? fv.res : fv.deq;
        if (kDual) a2[t] = (f2 == kFRes) ? fv.res : fv.deq;
      }
#pragma unroll
      for (int c = 0; c < W; c += 4) {
        const float4 p = *reinterpret_cast<const float4*>(&Ps1[j][c]);
#pragma unroll
        for (int t = 0; t < TM; ++t) {
          acc1[t][c + 0] = fmaf(a1[t], p.x, acc1[t][c + 0]);
          acc1[t][c + 1] = fmaf(a1[t], p.y, acc1[t][c + 1]);
          acc1[t][c + 2] = fmaf(a1[t], p.z, acc1[t][c + 2]);
          acc1[t][c + 3] = fmaf(a1[t], p.w, acc1[t][c + 3]);
        }
        if (kDual) {
          const float4 q = *reinterpret_cast<const float4*>(&Ps2[j][c]);
#pragma unroll
          for (int t = 0; t < TM; ++t) {
            acc2[t][c + 0] = fmaf(a2[t], q.x, acc2[t][c + 0]);
            acc2[t][c + 1] = fmaf(a2[t], q.y, acc2[t][c + 1]);
            acc2[t][c + 2] = fmaf(a2[t], q.z, acc2[t][c + 2]);
            acc2[t][c + 3] = fmaf(a2[t], q.w, acc2[t][c + 3]);
          }
        }
      }
    }
  }
  // write this split's partial (or the final result when there is one split)
  float* o1 = out1 + (int64_t)blockIdx.y * s.rows * W;
  float* o2 = kDual ? out2 + (int64_t)blockIdx.y * s.rows * W : nullptr;
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    const int64_t row = row_base + warp * (32 * TM) + lane + 32 * t;
    if (row < s.rows) {
#pragma unroll
      for (int c = 0; c < W; c += 4) {
        *reinterpret_cast<float4*>(o1 + row * W + c) =
            make_float4(acc1[t][c], acc1[t][c + 1], acc1[t][c + 2], acc1[t][c + 3]);
        if (kDual)
          *reinterpret_cast<float4*>(o2 + row * W + c) =
              make_float4(acc2[t][c], acc2[t][c + 1], acc2[t][c + 2], acc2[t][c + 3]);
      }
    }
  }
}

// ------------------------------------------------------------------ COL mode
// OUT[j,c] = sum_{i in split} F(x_ij) P[i,c]
template <int W, int TJ>
__global__ void __launch_bounds__(256) k3_proj_cols(SideView s, const float* __restrict__ P, int f,
                                                    float* __restrict__ out, int rchunk) {
  constexpr int BJ = 256 * TJ;
  constexpr int BR = 16;
  constexpr int kLoads = BR * BJ / 4 / 256;
  __shared__ __align__(16) float Xs[BR][BJ];
  __shared__ __align__(16) float Ps[BR][W];
  __shared__ float lam_s[BR], inv_s[BR];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j_base = blockIdx.x * BJ;
  const int64_t r_begin = (int64_t)blockIdx.y * rchunk;
  const int64_t r_end = (s.rows < r_begin + rchunk ? s.rows : r_begin + rchunk);
  const bool vec = ((reinterpret_cast<uintptr_t>(s.X) & 15) == 0) && (s.ldx % 4 == 0);

  float acc[TJ][W];
#pragma unroll
  for (int t = 0; t < TJ; ++t)
#pragma unroll
    for (int c = 0; c < W; ++c) acc[t][c] = 0.f;

  float4 pre[kLoads];
  auto load_tile = [&](int64_t r0) {
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
      const int fl = tid + 256 * u;
      const int rl = fl / (BJ / 4), ch = fl % (BJ / 4);
      const int64_t row = r0 + rl;
      const int col = j_base + ch * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < r_end) {
        const float* xr = s.X + row * s.ldx;
        if (vec && col + 3 < s.K) {
          v = __ldcs(reinterpret_cast<const float4*>(xr + col));
        } else {
          if (col + 0 < s.K) v.x = xr[col + 0];
          if (col + 1 < s.K) v.y = xr[col + 1];
          if (col + 2 < s.K) v.z = xr[col + 2];
          if (col + 3 < s.K) v.w = xr[col + 3];
        }
      }
      pre[u] = v;
    }
  };

  if (r_begin < r_end) load_tile(r_begin);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += BR) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
      const int fl = tid + 256 * u;
      const int rl = fl / (BJ / 4), ch = fl % (BJ / 4);
      *reinterpret_cast<float4*>(&Xs[rl][ch * 4]) = pre[u];
    }
    for (int e = tid; e < BR * W; e += 256) {
      const int i = e / W, c = e % W;
      Ps[i][c] = (r0 + i < r_end) ? P[(r0 + i) * W + c] : 0.f;
    }
    if (tid < BR) {
      const float l = (r0 + tid < r_end) ? s.lam[r0 + tid] : 1.f;
      lam_s[tid] = l;
      inv_s[tid] = __frcp_rn(l);
    }
    __syncthreads();
    if (r0 + BR < r_end) load_tile(r0 + BR);
#pragma unroll 4
    for (int i = 0; i < BR; ++i) {
      const float l = lam_s[i], il = inv_s[i];
      float a[TJ];
#pragma unroll
      for (int t = 0; t < TJ; ++t) {
        const FVals fv = fvals(l, il, Xs[i][warp * (32 * TJ) + lane + 32 * t], s.mode, s.qmax);
        a[t] = (f == kFRes) ? fv.res : fv.deq;
      }
#pragma unroll
      for (int c = 0; c < W; c += 4) {
        const float4 p = *reinterpret_cast<const float4*>(&Ps[i][c]);
#pragma unroll
        for (int t = 0; t < TJ; ++t) {
          acc[t][c + 0] = fmaf(a[t], p.x, acc[t][c + 0]);
          acc[t][c + 1] = fmaf(a[t], p.y, acc[t][c + 1]);
          acc[t][c + 2] = fmaf(a[t], p.z, acc[t][c + 2]);
          acc[t][c + 3] = fmaf(a[t], p.w, acc[t][c + 3]);
        }
      }
    }
  }
  float* o = out + (int64_t)blockIdx.y * s.K * W;
#pragma unroll
  for (int t = 0; t < TJ; ++t) {
    const int j = j_base + warp * (32 * TJ) + lane + 32 * t;
    if (j < s.K) {
#pragma unroll
      for (int c = 0; c < W; c += 4)
        *reinterpret_cast<float4*>(o + (int64_t)j * W + c) = make_float4(acc[t][c], acc[t][c + 1], acc[t][c + 2], acc[t][c + 3]);
    }
  }
}

// Fixed-order sum of split partials: out[e] = sum_s part[s*n + e]
__global__ void k_reduce_splits(const float* __restrict__ part, int nsplit, int64_t n, float* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < nsplit; ++s) a += part[(int64_t)s * n + e];
    out[e] = a;
  }
}

static int clamp_grid(int64_t want) { return (int)(want < 148 * 32 ? (want < 1 ? 1 : want) : 148 * 32); }

template <int W, int TM, bool kDual>
static void run_rows(const SideView& s, const float* P1, int f1, float* OUT1, const float* P2, int f2, float* OUT2,
                     float* partial, int64_t partial_elems, cudaStream_t st) {
  constexpr int BM = 256 * TM;
  const int64_t rb = (s.rows + BM - 1) / BM;
  // splits along K so that the grid covers ~4 waves of 148 SMs, chunks multiple of 16
  int64_t want = (4 * 148 + rb - 1) / rb;
  int64_t maxs = (s.K + 255) / 256;
  int64_t ns = want < maxs ? want : maxs;
  const int64_t per = s.rows * W * (kDual ? 2 : 1);
  if (ns > 1 && ns * per > partial_elems) ns = partial_elems / per;
  if (ns < 1) ns = 1;
  int kchunk = (int)(((s.K + ns - 1) / ns + 15) / 16 * 16);
  ns = (s.K + kchunk - 1) / kchunk;
  if (ns < 1) ns = 1;
  dim3 grid((unsigned)rb, (unsigned)ns);
  float* o1 = ns == 1 ? OUT1 : partial;
  float* o2 = ns == 1 ? OUT2 : partial + ns * s.rows * W;
  k2_proj_rows<W, TM, kDual><<<grid, 256, 0, st>>>(s, P1, f1, P2, f2, o1, o2, kchunk); ++launch_counter();
  if (ns > 1) {
    const int64_t n = s.rows * W;
    k_reduce_splits<<<clamp_grid((n + 255) / 256), 256, 0, st>>>(partial, (int)ns, n, OUT1); ++launch_counter();
    if (kDual) {
      k_reduce_splits<<<clamp_grid((n + 255) / 256), 256, 0, st>>>(o2, (int)ns, n, OUT2);
      ++launch_counter();
    }
  }
}

template <int W>
static void dispatch_rows(const SideView& s, const float* P1, int f1, float* OUT1, const float* P2, int f2,
                          float* OUT2, float* partial, int64_t pe, cudaStream_t st) {
  if (P2 != nullptr) {
    if constexpr (W <= 32) run_rows<W, 2, true>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st);
    else run_rows<W, 1, true>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st);
  } else {
    if constexpr (W <= 32) run_rows<W, 2, false>(s, P1, f1, OUT1, nullptr, 0, nullptr, partial, pe, st);
    else run_rows<W, 1, false>(s, P1, f1, OUT1, nullptr, 0, nullptr, partial, pe, st);
  }
}

void launch_proj_rows(const SideView& s, const float* P1, int f1, float* OUT1, const float* P2, int f2, float* OUT2,
                      int W, float* partial, int64_t pe, cudaStream_t st) {
  if (s.rows == 0) return;
  switch (W) {
    case 8: dispatch_rows<8>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    case 16: dispatch_rows<16>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    case 24: dispatch_rows<24>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    case 32: dispatch_rows<32>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    case 40: dispatch_rows<40>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    case 48: dispatch_rows<48>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    case 56: dispatch_rows<56>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    case 64: dispatch_rows<64>(s, P1, f1, OUT1, P2, f2, OUT2, partial, pe, st); break;
    default: break;
  }
}

template <int W>
static void run_cols(const SideView& s, const float* P, int f, float* OUT, float* partial, int64_t pe,
                     cudaStream_t st) {
  constexpr int TJ = W <= 32 ? 2 : 1;
  constexpr int BJ = 256 * TJ;
  const int64_t cb = (s.K + BJ - 1) / BJ;
  int64_t want = (4 * 148 + cb - 1) / cb;
  int64_t maxs = (s.rows + 63) / 64;
  int64_t ns = want < maxs ? want : maxs;
  const int64_t per = (int64_t)s.K * W;
  if (ns > 1 && ns * per > pe) ns = pe / per;
  if (ns < 1) ns = 1;
  int64_t rchunk = ((s.rows + ns - 1) / ns + 15) / 16 * 16;
  ns = (s.rows + rchunk - 1) / rchunk;
  if (ns < 1) ns = 1;
  dim3 grid((unsigned)cb, (unsigned)ns);
  k3_proj_cols<W, TJ><<<grid, 256, 0, st>>>(s, P, f, ns == 1 ? OUT : partial, (int)rchunk); ++launch_counter();
  if (ns > 1) {
    const int64_t n = (int64_t)s.K * W;
    k_reduce_splits<<<clamp_grid((n + 255) / 256), 256, 0, st>>>(partial, (int)ns, n, OUT); ++launch_counter();
  }
}

void launch_proj_cols(const SideView& s, const float* P, int f, float* OUT, int W, float* partial, int64_t pe,
                      cudaStream_t st) {
  if (s.K == 0) return;
  switch (W) {
    case 8: run_cols<8>(s, P, f, OUT, partial, pe, st); break;
    case 16: run_cols<16>(s, P, f, OUT, partial, pe, st); break;
    case 24: run_cols<24>(s, P, f, OUT, partial, pe, st); break;
    case 32: run_cols<32>(s, P, f, OUT, partial, pe, st); break;
    case 40: run_cols<40>(s, P, f, OUT, partial, pe, st); break;
    case 48: run_cols<48>(s, P, f, OUT, partial, pe, st); break;
    case 56: run_cols<56>(s, P, f, OUT, partial, pe, st); break;
    case 64: run_cols<64>(s, P, f, OUT, partial, pe, st); break;
    default: break;
  }
}

// ---------------------------------------------------------------- fp64 Gram
// partial[b][a][c] = sum_{i in block b} Y1[i,a] * Y2[i,c]
__global__ void __launch_bounds__(256) k_gram_partial(const float* __restrict__ Y1, const float* __restrict__ Y2,
                                                      int64_t n, int W, int64_t rows_per_block,
                                                      double* __restrict__ partial) {
  __shared__ float s1[64][65];
  __shared__ float s2[64][65];
  const int npairs = W * W;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r_end = (n < r_begin + rows_per_block ? n : r_begin + rows_per_block);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * W; e += 256) {
      const int i = e / W, c = e % W;
      const bool in = r0 + i < r_end;
      s1[i][c] = in ? Y1[(r0 + i) * W + c] : 0.f;
      s2[i][c] = in ? Y2[(r0 + i) * W + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int pr = threadIdx.x + 256 * q;
      if (pr < npairs) {
        const int a = pr / W, c = pr % W;
        double t = acc[q];
        for (int i = 0; i < 64; ++i) t = fma((double)s1[i][a], (double)s2[i][c], t);
        acc[q] = t;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int pr = threadIdx.x + 256 * q;
    if (pr < npairs) partial[(int64_t)blockIdx.x * npairs + pr] = acc[q];
  }
}

__global__ void k_gram_reduce(const double* __restrict__ partial, int nblk, int npairs, double* __restrict__ G) {
  for (int pr = threadIdx.x; pr < npairs; pr += blockDim.x) {
    double a = 0.0;
    for (int b = 0; b < nblk; ++b) a += partial[(int64_t)b * npairs + pr];
    G[pr] = a;
  }
}

void launch_gram(const float* Y1, const float* Y2, int64_t n, int W, double* G, double* partial, int64_t pe,
                 cudaStream_t st) {
  const int npairs = W * W;
  int64_t nblk = (n + 255) / 256;
  if (nblk > 296) nblk = 296;
  if (nblk * npairs > pe) nblk = pe / npairs;
  if (nblk < 1) nblk = 1;
  int64_t rpb = ((n + nblk - 1) / nblk + 63) / 64 * 64;
  if (rpb < 64) rpb = 64;
  nblk = (n + rpb - 1) / rpb;
  if (nblk < 1) nblk = 1;
  k_gram_partial<<<(unsigned)nblk, 256, 0, st>>>(Y1, Y2, n, W, rpb, partial); ++launch_counter();
  k_gram_reduce<<<1, 512, 0, st>>>(partial, (int)nblk, npairs, G); ++launch_counter();
}

// ----------------------------------------------------- small right-multiplies
// OUT[i, col0 + o] = sum_c IN1[i,c] S1[c,o] (+ sum_c IN2[i,c] S2[c,o])
__global__ void __launch_bounds__(256) k_apply_small(const float* __restrict__ IN1, const float* __restrict__ S1,
                                                     const float* __restrict__ IN2, const float* __restrict__ S2,
                                                     int64_t n, int W, int ldS, int nout, float* __restrict__ OUT,
                                                     int64_t ldo, int col0) {
  __shared__ float s1[64 * 64];
  __shared__ float s2[64 * 64];
  for (int e = threadIdx.x; e < W * nout; e += blockDim.x) {
    const int c = e / nout, o = e % nout;
    s1[c * 64 + o] = S1[c * ldS + o];
    if (IN2) s2[c * 64 + o] = S2[c * ldS + o];
  }
  __syncthreads();
  const int per_blk = 256 / nout;  // rows per block iteration
  for (int64_t base = (int64_t)blockIdx.x * per_blk; base < n; base += (int64_t)gridDim.x * per_blk) {
    const int lr = threadIdx.x / nout, o = threadIdx.x % nout;
    const int64_t i = base + lr;
    if (lr < per_blk && i < n) {
      float a = 0.f;
      const float* in1 = IN1 + i * W;
      for (int c = 0; c < W; ++c) a = fmaf(in1[c], s1[c * 64 + o], a);
      if (IN2) {
        const float* in2 = IN2 + i * W;
        for (int c = 0; c < W; ++c) a = fmaf(in2[c], s2[c * 64 + o], a);
      }
      OUT[i * ldo + col0 + o] = a;
    }
  }
}

void launch_apply_small(const float* IN1, const float* S1, const float* IN2, const float* S2, int64_t n, int W,
                        int ldS, int nout, float* OUT, int64_t ldo, int col0, cudaStream_t st) {
  if (n == 0 || nout == 0) return;
  const int per_blk = 256 / nout;
  k_apply_small<<<clamp_grid((n + per_blk - 1) / per_blk), 256, 0, st>>>(IN1, S1, IN2, S2, n, W, ldS, nout, OUT, ldo,
                                                                        col0); ++launch_counter();
}

}  // namespace lrqmm
