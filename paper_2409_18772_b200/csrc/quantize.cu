// K1 — fused amax + scale + quantize (Eq. quantA; vector-wise
// scales; floor rounding of Eq. get_ra2).
//
// One side X (rows x K fp32, row stride ldx) -> codes (rows x Kp int8, zero padded
// to Kp = roundup(K,128)) and lambda (rows fp32).  Each row is read from HBM once:
// it stays in registers between the amax reduction and the rounding pass.
//
// Bit-exact rounding on the exact product lambda*x (reading #4):
//   p = RN(lambda*x), e = fma(lambda, x, -p) is the exact error of the product, and
//   floor(lambda*x) = floorf(p) - (p == floorf(p) && (e < 0 || (p == 0 && x < 0))).
// RN is monotone and integers / half-integers are fp32-representable below 2^23,
// so p lies in the same unit interval as the exact product except when p itself
// is an integer (floor/trunc) or a half-integer (nearest); e decides those.
#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

LRQMM_DEV int round_exact(float lam, float x, int mode) {
  const float p = __fmul_rn(lam, x);
  const float e = __fmaf_rn(lam, x, -p);
  if (mode == kRoundFloor) {
    float f = floorf(p);
    if (p == f && (e < 0.f || (p == 0.f && x < 0.f))) f -= 1.f;
    return static_cast<int>(f);
  } else if (mode == kRoundTrunc) {
    float t = truncf(p);
    if (p == t && p != 0.f) {
      if (p > 0.f && e < 0.f) t -= 1.f;
      if (p < 0.f && e > 0.f) t += 1.f;
    }
    return static_cast<int>(t);
  } else {  // nearest, ties to even, decided on the exact product
    float r = rintf(p);
    const float fl = floorf(p);
    if (p - fl == 0.5f && e != 0.f) r = (e > 0.f) ? fl + 1.f : fl;
    return static_cast<int>(r);
  }
}

LRQMM_DEV int8_t code_of(float lam, float x, int mode, int qmax) {
  int c = round_exact(lam, x, mode);
  c = c > qmax ? qmax : (c < -qmax ? -qmax : c);
  return static_cast<int8_t>(c);
}

LRQMM_DEV uint32_t pack4(int8_t a, int8_t b, int8_t c, int8_t d) {
  return (uint32_t)(uint8_t)a | ((uint32_t)(uint8_t)b << 8) | ((uint32_t)(uint8_t)c << 16) |
         ((uint32_t)(uint8_t)d << 24);
}

// residual fraction u (exact fp32, |u| < 1) -> Q15: clamp(RN(u * 2^15), +-32767); the scaling is exact
LRQMM_DEV int u_fix(float u) {
  const int q = __float2int_rn(u * kUScale);
  return q > 32767 ? 32767 : (q < -32767 ? -32767 : q);
}
LRQMM_DEV uint32_t pack_bytes(int a, int b, int c, int d) {
  return ((uint32_t)a & 0xffu) | (((uint32_t)b & 0xffu) << 8) | (((uint32_t)c & 0xffu) << 16) | ((uint32_t)d << 24);
}

// TPR threads cooperate on one row; each holds VPT float4 of it.  Row length
// covered: TPR*VPT*4 >= Kp.  kFixedLam: lambda given (per-tensor mode), no amax.
template <int TPR, int VPT, bool kVec, bool kFixedLam>
__global__ void __launch_bounds__(256) k1_quantize(const float* __restrict__ X, int64_t ldx, int rows, int K, int Kp,
                                                   int qmax, int mode, int8_t* __restrict__ codes,
                                                   float* __restrict__ lam_out, float* __restrict__ inv_out,
                                                   const float* __restrict__ lam_in, int* __restrict__ err_flag,
                                                   uint8_t* __restrict__ U, int64_t ldu, int64_t uplane) {
  constexpr int kRowsPerCta = 256 / TPR;
  constexpr int kWarpsPerRow = TPR / 32;
  __shared__ float red[8];
  const int tid = threadIdx.x;
  const int sub = tid % TPR;  // thread index within its row group
  const int grp = tid / TPR;
  for (int64_t row0 = (int64_t)blockIdx.x * kRowsPerCta; row0 < rows; row0 += (int64_t)gridDim.x * kRowsPerCta) {
    const int64_t row = row0 + grp;
    const bool active = row < rows;
    const float* xr = X + row * ldx;
    float4 v[VPT];
    float amax = 0.f;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = (sub + i * TPR) * 4;
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      if (active) {
        if (kVec && col + 3 < K) {
          t = __ldcs(reinterpret_cast<const float4*>(xr + col));
        } else {
          if (col + 0 < K) t.x = xr[col + 0];
          if (col + 1 < K) t.y = xr[col + 1];
          if (col + 2 < K) t.z = xr[col + 2];
          if (col + 3 < K) t.w = xr[col + 3];
        }
      }
      v[i] = t;
      bad |= !(isfinite(t.x) && isfinite(t.y) && isfinite(t.z) && isfinite(t.w));
      amax = fmaxf(amax, fmaxf(fmaxf(fabsf(t.x), fabsf(t.y)), fmaxf(fabsf(t.z), fabsf(t.w))));
    }
    if (bad) atomicOr(err_flag, 1);
    float lam;
    if (kFixedLam) {
      lam = lam_in[0];
    } else {
      amax = warp_max(amax);
      if (kWarpsPerRow > 1) {
        if ((tid & 31) == 0) red[tid >> 5] = amax;
        __syncthreads();
        float m = red[0];
#pragma unroll
        for (int w = 1; w < kWarpsPerRow; ++w) m = fmaxf(m, red[w]);
        amax = m;
        __syncthreads();
      }
      // lambda = RN32(qmax / amax) (IEEE division), 1 for an all-zero row.
      lam = (amax == 0.f) ? 1.f : __fdiv_rn(static_cast<float>(qmax), amax);
    }
    if (active) {
      if (!kFixedLam && sub == 0) {
        lam_out[row] = lam;
        inv_out[row] = __frcp_rn(lam);
      }
      uint32_t* crow = reinterpret_cast<uint32_t*>(codes + row * (int64_t)Kp);
      uint8_t* urow = U ? U + row * ldu : nullptr;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int col = (sub + i * TPR) * 4;
        if (col < Kp) {
          // padded columns (K <= col < Kp) hold x = 0 -> code 0
          const int8_t c0 = code_of(lam, v[i].x, mode, qmax), c1 = code_of(lam, v[i].y, mode, qmax);
          const int8_t c2 = code_of(lam, v[i].z, mode, qmax), c3 = code_of(lam, v[i].w, mode, qmax);
          crow[col >> 2] = pack4(c0, c1, c2, c3);
          // residual fraction u = lambda x - code (R = u / lambda, Alg. 2), exactly rounded
          if (urow && col < ldu) {
            const int i0 = u_fix(__fmaf_rn(lam, v[i].x, -(float)c0)), i1 = u_fix(__fmaf_rn(lam, v[i].y, -(float)c1));
            const int i2 = u_fix(__fmaf_rn(lam, v[i].z, -(float)c2)), i3 = u_fix(__fmaf_rn(lam, v[i].w, -(float)c3));
            __stcg(reinterpret_cast<uint32_t*>(urow + col), pack_bytes(i0 >> 8, i1 >> 8, i2 >> 8, i3 >> 8));
            __stcg(reinterpret_cast<uint32_t*>(urow + uplane + col), pack_bytes(i0, i1, i2, i3));
          }
        }
      }
    }
  }
}

// Per-tensor mode step 1: per-row amax (also non-finite detection).
__global__ void __launch_bounds__(256) k1_row_amax(const float* __restrict__ X, int64_t ldx, int rows, int K,
                                                   float* __restrict__ amax_out, int* __restrict__ err_flag) {
  __shared__ float red[8];
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const float* xr = X + row * ldx;
    float m = 0.f;
    bool bad = false;
    for (int c = threadIdx.x; c < K; c += blockDim.x) {
      float t = xr[c];
      bad |= !isfinite(t);
      m = fmaxf(m, fabsf(t));
    }
    if (bad) atomicOr(err_flag, 1);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      float r = red[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
      amax_out[row] = r;
    }
    __syncthreads();
  }
}

// Per-tensor mode step 2: global amax -> one lambda, broadcast to all rows.
__global__ void __launch_bounds__(1024) k1_tensor_scale(const float* __restrict__ row_amax, int rows, int qmax,
                                                        float* __restrict__ lam_rows, float* __restrict__ inv_rows,
                                                        float* __restrict__ lam_scalar) {
  __shared__ float red[32];
  __shared__ float lam_s;
  float m = 0.f;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) m = fmaxf(m, row_amax[i]);
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
    lam_s = (r == 0.f) ? 1.f : __fdiv_rn(static_cast<float>(qmax), r);
    lam_scalar[0] = lam_s;
  }
  __syncthreads();
  const float inv_s = __frcp_rn(lam_s);
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    lam_rows[i] = lam_s;
    inv_rows[i] = inv_s;
  }
}

// Generic path for very long rows (K > 32768): two passes over the row (the
// second one mostly from L2).  Same rounding arithmetic.
__global__ void __launch_bounds__(256) k1_quantize_long(const float* __restrict__ X, int64_t ldx, int rows, int K,
                                                        int Kp, int qmax, int mode, int8_t* __restrict__ codes,
                                                        float* __restrict__ lam_out, float* __restrict__ inv_out,
                                                        const float* __restrict__ lam_in, int* __restrict__ err_flag,
                                                        uint8_t* __restrict__ U, int64_t ldu, int64_t uplane) {
  __shared__ float red[8];
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const float* xr = X + row * ldx;
    float lam;
    if (lam_in) {
      lam = lam_in[0];
    } else {
      float m = 0.f;
      bool bad = false;
      for (int c = threadIdx.x; c < K; c += 256) {
        float t = xr[c];
        bad |= !isfinite(t);
        m = fmaxf(m, fabsf(t));
      }
      if (bad) atomicOr(err_flag, 1);
      m = warp_max(m);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
      __syncthreads();
      m = red[0];
      for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
      __syncthreads();
      lam = (m == 0.f) ? 1.f : __fdiv_rn(static_cast<float>(qmax), m);
      if (threadIdx.x == 0) {
        lam_out[row] = lam;
        inv_out[row] = __frcp_rn(lam);
      }
    }
    int8_t* crow = codes + row * (int64_t)Kp;
    for (int c = threadIdx.x; c < Kp; c += 256) {
      const float x = c < K ? xr[c] : 0.f;
      const int8_t q = code_of(lam, x, mode, qmax);
      crow[c] = q;
      if (U && c < ldu) {
        const int iu = u_fix(__fmaf_rn(lam, x, -(float)q));
        U[row * ldu + c] = (uint8_t)(iu >> 8);
        U[uplane + row * ldu + c] = (uint8_t)(iu & 255);
      }
    }
  }
}

template <int TPR, int VPT>
static void launch_k1_t(const QuantArgs& a, bool vec, bool fixed, cudaStream_t st) {
  constexpr int rows_per_cta = 256 / TPR;
  int64_t ctas = (a.rows + rows_per_cta - 1) / rows_per_cta;
  int grid = (int)(ctas < 148 * 64 ? ctas : 148 * 64);
  if (grid < 1) grid = 1;
#define K1_LAUNCH(V, F)                                                                                  \
  k1_quantize<TPR, VPT, V, F><<<grid, 256, 0, st>>>(a.X, a.ldx, a.rows, a.K, a.Kp, a.qmax, a.mode, a.codes, \
                                                    a.lam, a.inv_lam, a.lam_fixed, a.err_flag, a.U, a.ldu, a.uplane)
  if (vec) {
    if (fixed) K1_LAUNCH(true, true); else K1_LAUNCH(true, false);
  } else {
    if (fixed) K1_LAUNCH(false, true); else K1_LAUNCH(false, false);
  }
#undef K1_LAUNCH
  ++launch_counter();
}

void launch_quantize(const QuantArgs& a, cudaStream_t st) {
  if (a.rows == 0) return;
  const bool vec = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);
  const bool fixed = a.lam_fixed != nullptr;
  const int Kp = a.Kp;
  if (Kp <= 32 * 4 * 1) launch_k1_t<32, 1>(a, vec, fixed, st);
  else if (Kp <= 32 * 4 * 2) launch_k1_t<32, 2>(a, vec, fixed, st);
  else if (Kp <= 32 * 4 * 4) launch_k1_t<32, 4>(a, vec, fixed, st);
  else if (Kp <= 32 * 4 * 8) launch_k1_t<32, 8>(a, vec, fixed, st);
  else if (Kp <= 256 * 4 * 2) launch_k1_t<256, 2>(a, vec, fixed, st);
  else if (Kp <= 256 * 4 * 4) launch_k1_t<256, 4>(a, vec, fixed, st);
  else if (Kp <= 256 * 4 * 8) launch_k1_t<256, 8>(a, vec, fixed, st);
  else if (Kp <= 256 * 4 * 16) launch_k1_t<256, 16>(a, vec, fixed, st);
  else if (Kp <= 256 * 4 * 32) launch_k1_t<256, 32>(a, vec, fixed, st);
  else {
    int grid = a.rows < 148 * 16 ? (int)a.rows : 148 * 16;
    k1_quantize_long<<<grid, 256, 0, st>>>(a.X, a.ldx, a.rows, a.K, a.Kp, a.qmax, a.mode, a.codes, a.lam,
                                           a.inv_lam, a.lam_fixed, a.err_flag, a.U, a.ldu, a.uplane); ++launch_counter();
  }
}

void launch_tensor_scale(const float* X, int64_t ldx, int64_t rows, int K, int qmax, float* row_amax, float* lam_rows,
                         float* inv_rows, float* lam_scalar, int* err_flag, cudaStream_t st) {
  if (rows > 0) {
    int grid = rows < 148 * 16 ? (int)rows : 148 * 16;
    k1_row_amax<<<grid, 256, 0, st>>>(X, ldx, (int)rows, K, row_amax, err_flag); ++launch_counter();
  }
  k1_tensor_scale<<<1, 1024, 0, st>>>(row_amax, (int)rows, qmax, lam_rows, inv_rows, lam_scalar); ++launch_counter();
}

}  // namespace lrqmm
