// K1 — fused amax + scale + quantize (Eq. quantA; vector-wise
// scales; floor rounding of Eq. get_ra2).
//
// One side X (rows x K fp32, row stride ldx) -> codes (rows x Kp int8, zero padded
// to Kp = roundup(K,16)) and lambda (rows fp32).  Each row is read from HBM once:
// it stays in registers between the amax reduction and the rounding pass.
//
// Bit-exact rounding on the exact product lambda*x (reading #4), on the FMA pipe:
//   n = fma(lambda, x, 1.5 2^23) - 1.5 2^23 (integer bits) is RN_int(lambda x) of the EXACT product
//   (|lambda x| <= qmax (1 + 2^-23) < 2^22, so the sum lies where the fp32 ulp is 1; ties to even),
//   d = fma(lambda, x, -n) has the sign of the exact lambda x - n, so
//   floor = n - (d < 0), ceil = n + (d > 0), trunc = floor / ceil by sign, nearest = n.
//   (d underflows to 0 only for n = 0 with |lambda x| < 2^-149: then x decides floor.)
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

constexpr float kMagic = 12582912.f;  // 1.5 2^23
constexpr int kMagicBits = 0x4B400000;

LRQMM_DEV int code_int(float lam, float x, int mode) {
  const int n = __float_as_int(__fmaf_rn(lam, x, kMagic)) - kMagicBits;
  if (mode == kRoundNearest) return n;
  const float d = __fmaf_rn(lam, x, -(float)n);
  if (mode == kRoundFloor) return n - ((d < 0.f || (d == 0.f && n == 0 && x < 0.f)) ? 1 : 0);
  return x >= 0.f ? n - (d < 0.f ? 1 : 0) : n + (d > 0.f ? 1 : 0);  // trunc
}

LRQMM_DEV int8_t code_of(float lam, float x, int mode, int qmax) {
  int c = code_int(lam, x, mode);
  c = c > qmax ? qmax : (c < -qmax ? -qmax : c);
  return static_cast<int8_t>(c);
}

// Q15 residual fraction i = clamp(RN(2^15 (lambda x - code)), +-32767) with ONE rounding of the exact
// value: RN_int(2^15 lambda x) - 2^15 code (lam32k = 2^15 lambda, exact unless it overflows, see
// k1 callers: rows with lambda > 2^100 take the two-step form).
LRQMM_DEV int u_q15(float lam32k, float x, int code) {
  int i = __float_as_int(__fmaf_rn(lam32k, x, kMagic)) - kMagicBits - 32768 * code;
  return i > 32767 ? 32767 : (i < -32767 ? -32767 : i);
}
LRQMM_DEV int u_q15_slow(float lam, float x, int code) {
  const float u = __fmaf_rn(lam, x, -(float)code);  // |u| < 1, |error| <= 2^-24
  int i = __float2int_rn(u * 32768.f);
  return i > 32767 ? 32767 : (i < -32767 ? -32767 : i);
}

// max with NaN propagation (PTX max.NaN): lets one reduction carry both amax and the non-finite test
LRQMM_DEV float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

LRQMM_DEV uint32_t pack4(int8_t a, int8_t b, int8_t c, int8_t d) {
  return (uint32_t)(uint8_t)a | ((uint32_t)(uint8_t)b << 8) | ((uint32_t)(uint8_t)c << 16) |
         ((uint32_t)(uint8_t)d << 24);
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
  ::lrqmm::pdl_enter();
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
            int i0, i1, i2, i3;
            if (lam < 0x1p100f) {
              const float l32 = lam * 32768.f;
              i0 = u_q15(l32, v[i].x, c0); i1 = u_q15(l32, v[i].y, c1); i2 = u_q15(l32, v[i].z, c2); i3 = u_q15(l32, v[i].w, c3);
            } else {
              i0 = u_q15_slow(lam, v[i].x, c0); i1 = u_q15_slow(lam, v[i].y, c1);
              i2 = u_q15_slow(lam, v[i].z, c2); i3 = u_q15_slow(lam, v[i].w, c3);
            }
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
  ::lrqmm::pdl_enter();
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
  ::lrqmm::pdl_enter();
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
  ::lrqmm::pdl_enter();
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
        const int iu = lam < 0x1p100f ? u_q15(lam * 32768.f, x, q) : u_q15_slow(lam, x, q);
        U[row * ldu + c] = (uint8_t)(iu >> 8);
        U[uplane + row * ldu + c] = (uint8_t)(iu & 255);
      }
    }
  }
}

// ---- lean per-element arithmetic of the TMA K1 (same exact results as code_of / u_q15) ----
// code: directed-rounding FMA of the exact product into the magic range (ulp 1):
//   floor = RD(lambda x + 1.5 2^23) - 1.5 2^23, trunc = RD / RU by the sign of x, nearest = RN.
template <int kMode>
LRQMM_DEV int code_fast(float lam, float x, int qmax) {
  int c;
  if (kMode == kRoundFloor) {
    c = __float_as_int(__fmaf_rd(lam, x, kMagic)) - kMagicBits;
    c = c < -qmax ? -qmax : c;  // floor only overshoots downwards (lambda amax may exceed qmax by an ulp)
  } else if (kMode == kRoundTrunc) {
    c = __float_as_int(x >= 0.f ? __fmaf_rd(lam, x, kMagic) : __fmaf_ru(lam, x, kMagic)) - kMagicBits;
  } else {
    c = __float_as_int(__fmaf_rn(lam, x, kMagic)) - kMagicBits;
  }
  return c;
}
// Q15 of lambda x - c (one rounding), clamped on the side the mode can overshoot
template <int kMode>
LRQMM_DEV int q15_fast(float lam32k, float x, int c) {
  int i = __float_as_int(__fmaf_rn(lam32k, x, kMagic)) - kMagicBits - (c << 15);
  if (kMode == kRoundFloor) return i > 32767 ? 32767 : i;
  return i > 32767 ? 32767 : (i < -32767 ? -32767 : i);
}
LRQMM_DEV uint32_t bytes4(int a, int b, int c, int d) {  // low bytes of a..d (PRMT)
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
LRQMM_DEV uint32_t hbytes4(int a, int b, int c, int d) {  // byte 1 of a..d
  return __byte_perm(__byte_perm(a, b, 0x0051), __byte_perm(c, d, 0x0051), 0x5410);
}

// Persistent TMA-pipelined K1 (rows of up to ~24K floats, K % 4 == 0, 16-byte aligned rows):
// a producer warp bulk-copies whole rows into an NS-deep shared-memory ring while 16 consumer
// warps quantize the previous ones, so HBM reads never wait for the reduce / round / store
// phases.  Same arithmetic as k1_quantize: the row is read from smem once into registers.
namespace k1t {
constexpr int kCons = 512;                 // consumer threads (16 warps)
constexpr int kThreads = kCons + 32;       // + producer warp
constexpr int kSmemBudget = 200 * 1024;
}  // namespace k1t

// G consumer groups (kCons / G threads each) work on G different rows at a time: ring slot `it` goes
// to group it % G, each group has its own named barrier (1 + group) for the row's amax.  G = 1 is one
// row at a time over all 16 warps; mid-size rows (K ~ 4K: few rows per CTA) use G = 2 so that the
// per-row chain (amax reduction, barrier, division) of one row overlaps another's.
template <int VPT, bool kFixedLam, int kMode, int G>
__global__ void __launch_bounds__(k1t::kThreads, 1)
    k1_quantize_tma(const float* __restrict__ X, int64_t ldx, int rows, int K, int Kp, int qmax, int mode,
                    int8_t* __restrict__ codes, float* __restrict__ lam_out, float* __restrict__ inv_out,
                    const float* __restrict__ lam_in, int* __restrict__ err_flag, uint8_t* __restrict__ U,
                    int64_t ldu, int64_t uplane, int ns, int slot_bytes) {
  ::lrqmm::pdl_enter();
  using namespace k1t;
  constexpr int TG = kCons / G, WG = TG / 32;  // threads / warps per group
  extern __shared__ __align__(128) uint8_t smem_k1[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_k1);
  uint64_t* empty = full + ns;
  __shared__ float red[2][16];
  uint8_t* ring = smem_k1 + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WG);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t row_bytes = (uint32_t)K * 4u;
  if (warp == kCons / 32) {
    // ------------------------------------------------------------- producer
    if (lane == 0) {
      int it = 0;
      for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++it) {
        const int s = it % ns;
        mbar_wait(&empty[s], ((it / ns) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], row_bytes);
        bulk_load(ring + (size_t)s * slot_bytes, X + r * ldx, row_bytes, &full[s]);
      }
    }
    return;
  }
  // --------------------------------------------------------------- consumers
  const int grp = tid / TG, gt = tid - grp * TG;  // group, thread within the group
  int it = grp, kr = 0;
  for (int64_t r = blockIdx.x + (int64_t)grp * gridDim.x; r < rows; r += (int64_t)G * gridDim.x, it += G, ++kr) {
    const int s = it % ns;
    mbar_wait(&full[s], (it / ns) & 1);
    const uint32_t base = smem_u32(ring + (size_t)s * slot_bytes);
    float4 v[VPT];
    float amax = 0.f, chk = 0.f;  // chk = sum x * 0: NaN iff some x is NaN or Inf
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = (gt + i * TG) * 4;
      v[i] = col < K ? lds128(base + (uint32_t)col * 4u) : make_float4(0.f, 0.f, 0.f, 0.f);
      chk = __fmaf_rn(v[i].x, 0.f, chk);
      chk = __fmaf_rn(v[i].y, 0.f, chk);
      chk = __fmaf_rn(v[i].z, 0.f, chk);
      chk = __fmaf_rn(v[i].w, 0.f, chk);
      amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v[i].x), fabsf(v[i].y)), fmaxf(fabsf(v[i].z), fabsf(v[i].w))));
    }
    const bool bad = chk != chk;
    // the row is in registers (amax depends on every value): hand the slot back to the producer
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (bad) atomicOr(err_flag, 1);
    float lam;
    if (kFixedLam) {
      lam = lam_in[0];
    } else {
      amax = warp_max(amax);
      if (lane == 0) red[kr & 1][warp] = amax;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(TG) : "memory");
      float m = red[kr & 1][grp * WG];
#pragma unroll
      for (int w = 1; w < WG; ++w) m = fmaxf(m, red[kr & 1][grp * WG + w]);
      // lambda = RN32(qmax / amax) (IEEE division), 1 for an all-zero row.
      lam = (m == 0.f) ? 1.f : __fdiv_rn(static_cast<float>(qmax), m);
      if (gt == 0) {
        lam_out[r] = lam;
        inv_out[r] = __frcp_rn(lam);
      }
    }
    uint32_t* crow = reinterpret_cast<uint32_t*>(codes + r * (int64_t)Kp);
    uint8_t* urow = U ? U + r * ldu : nullptr;
    const bool fast = lam < 0x1p100f;  // 2^15 lambda representable (always, but for rows of ~1e-28)
    const float l32 = lam * 32768.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int col = (gt + i * TG) * 4;
      if (col < Kp) {
        // padded columns (K <= col < Kp) hold x = 0 -> code 0, u = 0
        const int c0 = code_fast<kMode>(lam, v[i].x, qmax), c1 = code_fast<kMode>(lam, v[i].y, qmax);
        const int c2 = code_fast<kMode>(lam, v[i].z, qmax), c3 = code_fast<kMode>(lam, v[i].w, qmax);
        crow[col >> 2] = bytes4(c0, c1, c2, c3);
        if (urow) {
          int i0, i1, i2, i3;
          if (fast) {
            i0 = q15_fast<kMode>(l32, v[i].x, c0); i1 = q15_fast<kMode>(l32, v[i].y, c1);
            i2 = q15_fast<kMode>(l32, v[i].z, c2); i3 = q15_fast<kMode>(l32, v[i].w, c3);
          } else {
            i0 = u_q15_slow(lam, v[i].x, c0); i1 = u_q15_slow(lam, v[i].y, c1);
            i2 = u_q15_slow(lam, v[i].z, c2); i3 = u_q15_slow(lam, v[i].w, c3);
          }
          __stcg(reinterpret_cast<uint32_t*>(urow + col), hbytes4(i0, i1, i2, i3));
          __stcg(reinterpret_cast<uint32_t*>(urow + uplane + col), bytes4(i0, i1, i2, i3));
        }
      }
    }
  }
}

// Short rows (K < 4096, dense X): the same pipeline, but one bulk copy moves a chunk of R
// consecutive rows (~64 KB; R K 4 is a multiple of 16 bytes) and each consumer warp owns whole
// rows: pass 1 reduces amax from shared memory, pass 2 re-reads the row and writes codes and the
// Q15 planes (same exact arithmetic).  kVec4: K % 4 == 0 (16-byte row alignment in the slot).
template <bool kVec4, bool kFixedLam, int kMode>
__global__ void __launch_bounds__(k1t::kThreads, 2)
    k1_quantize_rows_tma(const float* __restrict__ X, int rows_full, int R, int K, int Kp, int qmax,
                         int8_t* __restrict__ codes, float* __restrict__ lam_out, float* __restrict__ inv_out,
                         const float* __restrict__ lam_in, int* __restrict__ err_flag, uint8_t* __restrict__ U,
                         int64_t ldu, int64_t uplane, int ns, int slot_bytes, int L) {
  ::lrqmm::pdl_enter();
  using namespace k1t;
  extern __shared__ __align__(128) uint8_t smem_k1[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_k1);
  uint64_t* empty = full + ns;
  uint8_t* ring = smem_k1 + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane_w = tid & 31;
  constexpr int kWarps = kCons / 32;
  // L lanes per row (a power of two <= 32): a warp quantizes 32 / L rows at a time
  const int sub_l = lane_w % L, grp = lane_w / L, rpw = 32 / L;
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunks = rows_full / R;
  if (warp == kWarps) {
    if (lane_w == 0) {
      int it = 0;
      for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % ns;
        mbar_wait(&empty[s], ((it / ns) & 1) ^ 1);
        const uint32_t bytes = (uint32_t)R * (uint32_t)K * 4u;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_load(ring + (size_t)s * slot_bytes, X + (int64_t)c * R * K, bytes, &full[s]);
      }
    }
    return;
  }
  int it = 0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
    const int s = it % ns;
    mbar_wait(&full[s], (it / ns) & 1);
    const uint8_t* slot = ring + (size_t)s * slot_bytes;
    // uniform trip count across the warp (the lane groups' shuffles must all execute)
    for (int rb = warp * rpw; rb < R; rb += kWarps * rpw) {
      const int rr = rb + grp;
      const bool active = rr < R;
      const int lane = sub_l;
      const int64_t row = (int64_t)c * R + rr;
      const float* xr = reinterpret_cast<const float*>(slot) + (int64_t)(active ? rr : 0) * K;
      float amax = 0.f;  // NaN-propagating: NaN / Inf if the row holds one (non-finite test below)
      if (kVec4) {
        for (int f = lane; active && f < K / 4; f += L) {
          const float4 v = reinterpret_cast<const float4*>(xr)[f];
          amax = fmax_nan(amax, fmax_nan(fmax_nan(fabsf(v.x), fabsf(v.y)), fmax_nan(fabsf(v.z), fabsf(v.w))));
        }
      } else {
        for (int j = lane; active && j < K; j += L) {
          const float v = xr[j];
          amax = fmax_nan(amax, fabsf(v));
        }
      }
      if (!(amax <= 3.402823466e38f)) atomicOr(err_flag, 1);
      float lam;
      if (kFixedLam) {
        lam = lam_in[0];
      } else {
        for (int o = L >> 1; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        lam = (amax == 0.f) ? 1.f : __fdiv_rn(static_cast<float>(qmax), amax);
        if (active && lane == 0) {
          lam_out[row] = lam;
          inv_out[row] = __frcp_rn(lam);
        }
      }
      if (!active) continue;
      const bool fast = lam < 0x1p100f;
      const float l32 = lam * 32768.f;
      int8_t* crow = codes + row * (int64_t)Kp;
      uint8_t* urow = U ? U + row * ldu : nullptr;
      if (kVec4) {
        for (int f = lane; f < Kp / 4; f += L) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (4 * f < K) v = reinterpret_cast<const float4*>(xr)[f];
          const int c0 = code_fast<kMode>(lam, v.x, qmax), c1 = code_fast<kMode>(lam, v.y, qmax);
          const int c2 = code_fast<kMode>(lam, v.z, qmax), c3 = code_fast<kMode>(lam, v.w, qmax);
          reinterpret_cast<uint32_t*>(crow)[f] = bytes4(c0, c1, c2, c3);
          if (urow) {
            int i0, i1, i2, i3;
            if (fast) {
              i0 = q15_fast<kMode>(l32, v.x, c0); i1 = q15_fast<kMode>(l32, v.y, c1);
              i2 = q15_fast<kMode>(l32, v.z, c2); i3 = q15_fast<kMode>(l32, v.w, c3);
            } else {
              i0 = u_q15_slow(lam, v.x, c0); i1 = u_q15_slow(lam, v.y, c1);
              i2 = u_q15_slow(lam, v.z, c2); i3 = u_q15_slow(lam, v.w, c3);
            }
            __stcg(reinterpret_cast<uint32_t*>(urow) + f, hbytes4(i0, i1, i2, i3));
            __stcg(reinterpret_cast<uint32_t*>(urow + uplane) + f, bytes4(i0, i1, i2, i3));
          }
        }
      } else {
        for (int j = lane; j < Kp; j += L) {
          const float v = j < K ? xr[j] : 0.f;
          const int cj = code_fast<kMode>(lam, v, qmax);
          crow[j] = (int8_t)cj;
          if (urow) {
            const int ij = fast ? q15_fast<kMode>(l32, v, cj) : u_q15_slow(lam, v, cj);
            urow[j] = (uint8_t)(ij >> 8);
            urow[uplane + j] = (uint8_t)(ij & 255);
          }
        }
      }
    }
    __syncwarp();
    if (lane_w == 0) mbar_arrive(&empty[s]);  // this warp's rows are done with the slot
  }
}

// dense X (ldx == K), 16-byte aligned, 16 <= K < 4096: chunks of R rows per bulk copy.  Returns the
// number of rows handled (a multiple of R); the caller quantizes the rest with the row kernels.
static int64_t launch_k1_rows_tma(const QuantArgs& a, bool fixed, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(a.X) & 15) != 0 || a.ldx != a.K || a.K < 16 || a.K >= 4096) return 0;
  const int step = a.K % 4 == 0 ? 1 : (a.K % 2 == 0 ? 2 : 4);  // R K 4 % 16 == 0
  // ~32 KB chunks, 3 slots: two CTAs per SM (34 warps) hide the per-row amax -> lambda -> round chain
  int R = (8192 / a.K) / step * step;
  if (R < step) return 0;
  const int64_t rows_full = a.rows / R * R;
  if (rows_full == 0 || rows_full > INT32_MAX) return 0;
  const int slot = (R * a.K * 4 + 1023) / 1024 * 1024;
  int ns = (k1t::kSmemBudget / 2) / slot;
  if (ns > 3) ns = 3;
  if (ns < 2) return 0;
  const int smem = 1024 + ns * slot;
  const int nsm = sm_count();
  const int64_t nchunks = rows_full / R;
  const int grid = (int)(nchunks < 2 * nsm ? nchunks : 2 * nsm);
  const bool v4 = a.K % 4 == 0;
  // lanes per row (vec4 path): ~4 float4 per lane, at least 8 lanes (one full 32-byte sector per
  // row and store instruction); fewer lanes per row = more rows per warp sharing one amax
  // reduction, division and lambda store (short rows are bound by that per-row work)
  static const int f4pl = [] {
    const char* e = getenv("LRQMM_K1_F4PL");
    return e && atoi(e) > 0 ? atoi(e) : 4;
  }();
  int L = 32;
  if (v4)
    while (L > 8 && (L / 2) * f4pl >= a.K / 4) L /= 2;
#define K1R_LAUNCH(V, F, M)                                                                                      \
  do {                                                                                                           \
    cudaFuncSetAttribute(k1_quantize_rows_tma<V, F, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);     \
    launch_pdl(k1_quantize_rows_tma<V, F, M>, grid, k1t::kThreads, smem, st, a.X, (int)rows_full, R, a.K, a.Kp, a.qmax, \
                                                                     a.codes, a.lam, a.inv_lam, a.lam_fixed,    \
                                                                     a.err_flag, a.U, a.ldu, a.uplane, ns, slot, L); \
  } while (0)
#define K1R_MODE(V, F)                                      \
  do {                                                      \
    if (a.mode == kRoundFloor) K1R_LAUNCH(V, F, kRoundFloor); \
    else if (a.mode == kRoundTrunc) K1R_LAUNCH(V, F, kRoundTrunc); \
    else K1R_LAUNCH(V, F, kRoundNearest);                   \
  } while (0)
  if (v4) {
    if (fixed) K1R_MODE(true, true); else K1R_MODE(true, false);
  } else {
    if (fixed) K1R_MODE(false, true); else K1R_MODE(false, false);
  }
#undef K1R_MODE
#undef K1R_LAUNCH
  ++launch_counter();
  return rows_full;
}

template <int VPT, int G = 1>
static bool launch_k1_tma_t(const QuantArgs& a, bool fixed, cudaStream_t st) {
  const int slot = (a.K * 4 + 1023) / 1024 * 1024;
  int ns = k1t::kSmemBudget / slot;
  if (ns > 8) ns = 8;
  if (ns < 1) return false;
  const int smem = 1024 + ns * slot;
  const int nsm = sm_count();
  const int grid = (int)(a.rows < nsm ? a.rows : nsm);
#define K1T_LAUNCH(F, M)                                                                                         \
  do {                                                                                                           \
    cudaFuncSetAttribute(k1_quantize_tma<VPT, F, M, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);     \
    launch_pdl(k1_quantize_tma<VPT, F, M, G>, grid, k1t::kThreads, smem, st, a.X, a.ldx, (int)a.rows, a.K, a.Kp, a.qmax, \
                                                                  a.mode, a.codes, a.lam, a.inv_lam, a.lam_fixed, \
                                                                  a.err_flag, a.U, a.ldu, a.uplane, ns, slot);   \
  } while (0)
  if (fixed) {
    if (a.mode == kRoundFloor) K1T_LAUNCH(true, kRoundFloor);
    else if (a.mode == kRoundTrunc) K1T_LAUNCH(true, kRoundTrunc);
    else K1T_LAUNCH(true, kRoundNearest);
  } else {
    if (a.mode == kRoundFloor) K1T_LAUNCH(false, kRoundFloor);
    else if (a.mode == kRoundTrunc) K1T_LAUNCH(false, kRoundTrunc);
    else K1T_LAUNCH(false, kRoundNearest);
  }
#undef K1T_LAUNCH
  ++launch_counter();
  return true;
}

// TMA path: rows 16-byte aligned (bulk copies) and at least ~4K columns (enough bytes per copy)
static bool launch_k1_tma(const QuantArgs& a, bool fixed, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(a.X) & 15) != 0 || a.ldx % 4 != 0 || a.K % 4 != 0 || a.K < 4096) return false;
  const int Kp = a.Kp;
  constexpr int C4 = k1t::kCons * 4;
  // mid-size rows (K <= 4096): four consumer groups, four rows in flight per CTA (c2: 29.5 -> 19 us per
  // side); LRQMM_K1_GROUPS=1 / 2 for A/B
  static const int groups = [] {
    const char* e = getenv("LRQMM_K1_GROUPS");
    return e && atoi(e) > 0 ? atoi(e) : 4;
  }();
  if (Kp <= C4 * 2) {
    if (groups >= 4) return launch_k1_tma_t<8, 4>(a, fixed, st);
    return groups >= 2 ? launch_k1_tma_t<4, 2>(a, fixed, st) : launch_k1_tma_t<2>(a, fixed, st);
  }
  if (Kp <= C4 * 4) return launch_k1_tma_t<4>(a, fixed, st);
  if (Kp <= C4 * 8) return launch_k1_tma_t<8>(a, fixed, st);
  if (Kp <= C4 * 12) return launch_k1_tma_t<12>(a, fixed, st);
  // long rows (c5: K = 32768, 128 KB): one ring slot -- the consumers hold the row in registers
  // and release the slot before they quantize, so the next row still streams in meanwhile
  if (Kp <= C4 * 16) return launch_k1_tma_t<16>(a, fixed, st);
  return false;
}

template <int TPR, int VPT>
static void launch_k1_t(const QuantArgs& a, bool vec, bool fixed, cudaStream_t st) {
  constexpr int rows_per_cta = 256 / TPR;
  int64_t ctas = (a.rows + rows_per_cta - 1) / rows_per_cta;
  int grid = (int)(ctas < 148 * 64 ? ctas : 148 * 64);
  if (grid < 1) grid = 1;
#define K1_LAUNCH(V, F)                                                                                  \
  launch_pdl(k1_quantize<TPR, VPT, V, F>, grid, 256, 0, st, a.X, a.ldx, a.rows, a.K, a.Kp, a.qmax, a.mode, a.codes, \
                                                    a.lam, a.inv_lam, a.lam_fixed, a.err_flag, a.U, a.ldu, a.uplane)
  if (vec) {
    if (fixed) K1_LAUNCH(true, true); else K1_LAUNCH(true, false);
  } else {
    if (fixed) K1_LAUNCH(false, true); else K1_LAUNCH(false, false);
  }
#undef K1_LAUNCH
  ++launch_counter();
}

void launch_quantize_rows(const QuantArgs& a, bool fixed, cudaStream_t st);

void launch_quantize(const QuantArgs& a, cudaStream_t st) {
  if (a.rows == 0) return;
  const bool fixed = a.lam_fixed != nullptr;
#ifndef LRQMM_K1_NO_TMA
  if (launch_k1_tma(a, fixed, st)) return;
  {
    const int64_t done = launch_k1_rows_tma(a, fixed, st);
    if (done == a.rows) return;
    if (done > 0) {  // the ragged tail rows: register-row kernels on the remaining rows
      QuantArgs t = a;
      t.X = a.X + done * a.ldx;
      t.rows = a.rows - done;
      t.codes = a.codes + done * (int64_t)a.Kp;
      if (!fixed) {
        t.lam = a.lam + done;
        t.inv_lam = a.inv_lam + done;
      }
      if (a.U) t.U = a.U + done * a.ldu;
      launch_quantize_rows(t, fixed, st);
      return;
    }
  }
#endif
  launch_quantize_rows(a, fixed, st);
}

// register-row kernels (one CTA / warp group per row), any alignment / stride
void launch_quantize_rows(const QuantArgs& a, bool fixed, cudaStream_t st) {
  const bool vec = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);
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
    launch_pdl(k1_quantize_long, grid, 256, 0, st, a.X, a.ldx, a.rows, a.K, a.Kp, a.qmax, a.mode, a.codes, a.lam,
                                           a.inv_lam, a.lam_fixed, a.err_flag, a.U, a.ldu, a.uplane); ++launch_counter();
  }
}

// ------------------------------------------------------------ implicit im2col
// K1 on the im2col matrix of a convolution without materialising it: row (b, ho, wo), column
// k = (i kw + j) C + c reads X[b, ho sh - ph + i dh, wo sw - pw + j dw, c] of the NHWC input (zero
// outside the image).  One warp per row: pass 1 the row amax, pass 2 (the same elements, now in
// L1 / L2) codes and the Q15 residual planes, with the exact arithmetic of k1_quantize_tma.  A
// 3x3 window reads each activation ~9 times, so HBM sees the activations once (L2 reuse across
// neighbouring rows) instead of the 9x larger fp32 im2col matrix.
// kVec: C % 4 == 0 -> each lane handles groups of 4 consecutive channels of one (i, j) tap
// (16-byte loads).  Each pass issues VPT independent group loads per lane before using them
// (memory-level parallelism); rows of K <= 32 E VPT stay in registers between amax and rounding.
template <int kMode, bool kVec, int VPT>
__global__ void __launch_bounds__(256) k1_quantize_im2col(const float* __restrict__ X, const ConvGeom g, int K, int Kp,
                                                          int qmax, int8_t* __restrict__ codes, float* __restrict__ lam_out,
                                                          float* __restrict__ inv_out, int* __restrict__ err_flag,
                                                          uint8_t* __restrict__ U, int64_t ldu, int64_t uplane, int rows) {
  ::lrqmm::pdl_enter();
  constexpr int E = kVec ? 4 : 1;
  constexpr int SPAN = 32 * E * VPT;  // row elements per batch
  const int lane = threadIdx.x & 31;
  const int G = g.C / E;  // element groups per tap
  // this lane's first group q = lane: tap / channel group / (i, j); a step of 32 groups moves
  // d_tap taps and d_cg groups (with a carry when the channel group wraps)
  const int l_tap = lane / G, l_cg = lane - l_tap * G, l_i = l_tap / g.kw, l_j = l_tap - l_i * g.kw;
  const int d_tap = 32 / G, d_cg = 32 - d_tap * G;
  const int img = g.H * g.W * g.C;  // < 2^31 (checked by the launcher)
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows; row += nw) {
    const int t = row / g.Wo;
    const int wo = row - t * g.Wo;
    const int b = t / g.Ho;
    const int ho = t - b * g.Ho;
    const int hb = ho * g.sh - g.ph, wb = wo * g.sw - g.pw;
    const float* xb = X + (int64_t)b * img;
    int st_cg, st_i, st_j;
    auto reset = [&]() { st_cg = l_cg; st_i = l_i; st_j = l_j; };
    auto step = [&]() {
      int dt = d_tap;
      st_cg += d_cg;
      if (st_cg >= G) { st_cg -= G; ++dt; }
      st_j += dt;
      while (st_j >= g.kw) { st_j -= g.kw; ++st_i; }
    };
    // VPT groups of this lane for the batch starting at column k0 (0 outside the image / past K)
    auto load = [&](int k0, float (&v)[VPT][4]) {
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        if (k0 + u * 32 * E >= K) {  // warp-uniform: the rest of the batch is past the row
#pragma unroll
          for (int e = 0; e < 4; ++e) v[u][e] = 0.f;
          continue;
        }
        const int k = k0 + (u * 32 + lane) * E;
        const int hi = hb + st_i * g.dh, wi = wb + st_j * g.dw;
        const bool in = k < K && (unsigned)hi < (unsigned)g.H && (unsigned)wi < (unsigned)g.W;
        const float* p = xb + ((hi * g.W + wi) * g.C + st_cg * E);
        if (kVec) {
          const float4 q = in ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
          v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
        } else {
          v[u][0] = in ? __ldg(p) : 0.f;
        }
        step();
      }
    };
    reset();
    float v[VPT][4];
    float amax = 0.f;            // NaN-propagating max: NaN if any x is NaN, Inf if any is infinite
    const bool one = K <= SPAN;  // the whole row in registers
    for (int k0 = 0; k0 < K; k0 += SPAN) {
      load(k0, v);
#pragma unroll
      for (int u = 0; u < VPT; ++u)
#pragma unroll
        for (int e = 0; e < E; ++e) amax = fmax_nan(amax, fabsf(v[u][e]));
    }
    if (!(amax <= 3.402823466e38f)) atomicOr(err_flag, 1);
    amax = warp_max(amax);
    // lambda = RN32(qmax / amax) (IEEE division), 1 for an all-zero row
    const float lam = (amax == 0.f) ? 1.f : __fdiv_rn(static_cast<float>(qmax), amax);
    if (lane == 0) {
      lam_out[row] = lam;
      inv_out[row] = __frcp_rn(lam);
    }
    const bool fast = lam < 0x1p100f;
    const float l32 = lam * 32768.f;
    int8_t* crow = codes + (int64_t)row * Kp;
    uint8_t* urow = U ? U + (int64_t)row * ldu : nullptr;
    if (!one) reset();
    for (int k0 = 0; k0 < Kp; k0 += SPAN) {
      if (!one) load(k0, v);  // second pass (L1 / L2); padded columns load as 0 -> code 0, u = 0
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        if (k0 + u * 32 * E >= Kp) break;
        const int k = k0 + (u * 32 + lane) * E;
        if (k >= Kp) continue;
        int c[4], q[4];
        if (fast) {  // row-uniform: one form per row, not both and a select
#pragma unroll
          for (int e = 0; e < E; ++e) {
            c[e] = code_fast<kMode>(lam, v[u][e], qmax);
            q[e] = q15_fast<kMode>(l32, v[u][e], c[e]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            c[e] = code_fast<kMode>(lam, v[u][e], qmax);
            q[e] = u_q15_slow(lam, v[u][e], c[e]);
          }
        }
        if (kVec) {
          *reinterpret_cast<uint32_t*>(crow + k) = bytes4(c[0], c[1], c[2], c[3]);
          if (urow) {
            __stcg(reinterpret_cast<uint32_t*>(urow + k), hbytes4(q[0], q[1], q[2], q[3]));
            __stcg(reinterpret_cast<uint32_t*>(urow + uplane + k), bytes4(q[0], q[1], q[2], q[3]));
          }
        } else {
          crow[k] = (int8_t)c[0];
          if (urow) {
            urow[k] = (uint8_t)(q[0] >> 8);
            urow[uplane + k] = (uint8_t)(q[0] & 255);
          }
        }
      }
    }
  }
}

// Tiled implicit im2col (dw == 1, kw >= sw: the window leaves no gaps).  A CTA owns TW
// consecutive output pixels (b, ho, wo0 .. wo0 + TW - 1) at a time: their input window -- kh
// input rows x WI = (TW - 1) sw + kw pixels x C channels, zero outside the image -- is staged in
// shared memory by cp.async (zero-fill for the padding), double buffered so the next tile's window
// is in flight while this one is quantized.  With dw == 1, column k = (i kw + j) C + c of output
// pixel wl sits at window[i RS + wl sw C + (j C + c)], so a per-CTA table off[k] = i RS + (j C + c)
// turns every element into two shared loads (one table load per quad of columns when C % 4 == 0)
// -- no per-element index arithmetic, no L1 / L2 gathers.  Padded columns K <= k < Kp point into a
// zeroed strip behind the window.  A row is handled by LPR lanes (32 / LPR rows per warp, so short
// rows -- the 7x7 stem's 147 columns = 40 quads = 8 lanes x 5 -- leave no lanes idle and share
// the per-row reduction / division); columns go in quads, so the codes and both Q15 planes are
// written with 4-byte stores.  Arithmetic and results identical to k1_quantize_im2col (same amax,
// lambda, code_fast / q15_fast / u_q15_slow).
namespace im2t {
constexpr int kThreads = 256;
constexpr int kBudget = 100 * 1024;  // dynamic shared memory per CTA (two windows + zero strip + table)
struct Tile {
  int TW, ntw, WI, RS;  // tile width (output pixels), tiles per output row, window pixels, row stride (floats)
  int zero;             // floats of the zero strip (0: no padded columns)
};
// one staged window, rounded up to 16 bytes
__host__ __device__ inline int tile_floats(const ConvGeom& g, const Tile& t) { return (g.kh * t.RS + 3) & ~3; }
// two buffers, each a window followed by its zero strip, then the offset table
inline int smem_bytes(const ConvGeom& g, const Tile& t, int Kp, bool vec) {
  return 2 * (tile_floats(g, t) + t.zero) * 4 + (vec ? Kp / 4 : Kp) * 4;
}
// shared loads on 32-bit addresses; volatile (ordered against bar.sync) but no memory clobber, so
// the global stores of the quantize pass stay free to overlap them
__device__ __forceinline__ float ld1(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 ld4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 ld4i(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int ld1i(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// global -> shared copy of E floats, zero-filled when !valid (src-size 0: nothing is read)
template <int E>
__device__ __forceinline__ void cp_zfill(uint32_t dst, const float* src, bool valid) {
  if (E == 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
}  // namespace im2t

template <int kMode, bool kVec, int VPT, int LPR>
__global__ void __launch_bounds__(im2t::kThreads) k1_quantize_im2col_tile(
    const float* __restrict__ X, const ConvGeom g, const im2t::Tile tl, int K, int Kp, int qmax,
    int8_t* __restrict__ codes, float* __restrict__ lam_out, float* __restrict__ inv_out, int* __restrict__ err_flag,
    uint8_t* __restrict__ U, int64_t ldu, int64_t uplane, int64_t ntiles) {
  extern __shared__ float4 im2t_smem[];
  float* win = reinterpret_cast<float*>(im2t_smem);
  const int tf = im2t::tile_floats(g, tl);
  const int bstride = tf + tl.zero;  // floats per buffer
  int* off = reinterpret_cast<int*>(win + 2 * bstride);
  const uint32_t s_win = (uint32_t)__cvta_generic_to_shared(win);
  const uint32_t s_off = (uint32_t)__cvta_generic_to_shared(off);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int RPW = 32 / LPR;  // rows per warp
  const int sub = lane / LPR, sl = lane - sub * LPR;
  const int nq = Kp >> 2;  // column quads (Kp % 4 == 0)
  const int KWC = g.kw * g.C;
  // byte offsets from a pixel's window origin: i RS + (j C + c) floats, or (padded columns) the
  // buffer's zero strip right behind its window
  const int zoff = tf;
  if (kVec) {  // quad table: a quad lies in one tap (C % 4 == 0)
    for (int q = tid; q < nq; q += im2t::kThreads) {
      const int k = q * 4, i = k / KWC;
      off[q] = 4 * (k < K ? i * tl.RS + (k - i * KWC) : zoff);
    }
  } else {
    for (int k = tid; k < Kp; k += im2t::kThreads) {
      const int i = k / KWC;
      off[k] = 4 * (k < K ? i * tl.RS + (k - i * KWC) : zoff);
    }
  }
  for (int z = tid; z < tl.zero; z += im2t::kThreads) win[tf + z] = win[bstride + tf + z] = 0.f;
  ::lrqmm::pdl_enter();
  const int64_t img = (int64_t)g.H * g.W * g.C;
  constexpr int E = kVec ? 4 : 1;
  // stage the window of tile t into buffer `buf` (cp.async, one group per call)
  auto stage = [&](int64_t t, int buf) {
    if (t < ntiles) {
      const int64_t bh = t / tl.ntw;
      const int wt = (int)(t - bh * tl.ntw);
      const int b = (int)(bh / g.Ho), ho = (int)(bh - (int64_t)b * g.Ho);
      const int wi0 = wt * tl.TW * g.sw - g.pw;
      const int flo = max(0, -wi0) * g.C, fhi = min(tl.WI, g.W - wi0) * g.C;
      const float* xb = X + b * img + (int64_t)wi0 * g.C;
      const int hb = ho * g.sh - g.ph;
      const uint32_t dbase = s_win + 4u * (uint32_t)(buf * bstride);
      for (int i = 0; i < g.kh; ++i) {  // staged row i: input row hb + i dh, contiguous in X
        const int hi = hb + i * g.dh;
        const bool inh = (unsigned)hi < (unsigned)g.H;
        const float* src = xb + (int64_t)hi * g.W * g.C;
        const uint32_t dst = dbase + 4u * (uint32_t)(i * tl.RS);
        for (int f = tid * E; f < tl.RS; f += im2t::kThreads * E) {
          const bool in = inh && f >= flo && f < fhi;
          im2t::cp_zfill<E>(dst + 4u * f, in ? src + f : X, in);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  constexpr int SPAN = LPR * VPT;  // quads per batch
  const bool one = nq <= SPAN;     // the whole row stays in registers between the two passes
  int buf = 0;
  stage(blockIdx.x, 0);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, buf ^= 1) {
    stage(t + gridDim.x, buf ^ 1);  // the buffer the previous tile used (freed by the barrier below)
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();  // every thread's copies of this tile have landed
    const int64_t bh = t / tl.ntw;
    const int wo0 = (int)(t - bh * tl.ntw) * tl.TW;
    const int tw = min(tl.TW, g.Wo - wo0);
    const uint32_t s_buf = s_win + 4u * (uint32_t)(buf * bstride);
    for (int wl0 = warp * RPW; wl0 < tw; wl0 += (im2t::kThreads / 32) * RPW) {
      const int wl = wl0 + sub;
      const bool active = wl < tw;
      const uint32_t s_row = s_buf + 4u * (uint32_t)((active ? wl : 0) * g.sw * g.C);
      const int64_t row = bh * g.Wo + wo0 + wl;
      float v[VPT][4];
      auto load = [&](int q0) {
#pragma unroll
        for (int u = 0; u < VPT; ++u) {
          const int q = q0 + u * LPR + sl;
          if (q >= nq) {  // past the row: keeps the amax / stores inert
            v[u][0] = v[u][1] = v[u][2] = v[u][3] = 0.f;
            continue;
          }
          if (kVec) {
            const float4 x = im2t::ld4(s_row + im2t::ld1i(s_off + 4u * q));
            v[u][0] = x.x; v[u][1] = x.y; v[u][2] = x.z; v[u][3] = x.w;
          } else {
            const int4 o = im2t::ld4i(s_off + 16u * q);
            v[u][0] = im2t::ld1(s_row + o.x);
            v[u][1] = im2t::ld1(s_row + o.y);
            v[u][2] = im2t::ld1(s_row + o.z);
            v[u][3] = im2t::ld1(s_row + o.w);
          }
        }
      };
      float amax = 0.f;  // NaN-propagating, as k1_quantize_im2col
      for (int q0 = 0; q0 < nq; q0 += SPAN) {
        load(q0);
#pragma unroll
        for (int u = 0; u < VPT; ++u)
#pragma unroll
          for (int e = 0; e < 4; ++e) amax = fmax_nan(amax, fabsf(v[u][e]));
      }
      if (active && !(amax <= 3.402823466e38f)) atomicOr(err_flag, 1);
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) amax = fmax_nan(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      const float lam = (amax == 0.f) ? 1.f : __fdiv_rn(static_cast<float>(qmax), amax);
      if (active && sl == 0) {
        lam_out[row] = lam;
        inv_out[row] = __frcp_rn(lam);
      }
      if (!active) continue;  // no further shuffles below
      const float l32 = lam * 32768.f;
      uint32_t* crow = reinterpret_cast<uint32_t*>(codes + row * Kp) + sl;
      uint32_t* urow = U ? reinterpret_cast<uint32_t*>(U + row * ldu) + sl : nullptr;
      uint32_t* lrow = U ? reinterpret_cast<uint32_t*>(U + uplane + row * ldu) + sl : nullptr;
      // pass 2, unswitched on the row-uniform choices (rounding form, residual planes or not)
      auto emit = [&](auto kFast, auto kU) {
        for (int q0 = 0; q0 < nq; q0 += SPAN) {
          if (!one) load(q0);
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            if (q0 + u * LPR + sl >= nq) continue;
            int c[4], s[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              c[e] = code_fast<kMode>(lam, v[u][e], qmax);
              if (decltype(kU)::value) s[e] = decltype(kFast)::value ? q15_fast<kMode>(l32, v[u][e], c[e])
                                                                     : u_q15_slow(lam, v[u][e], c[e]);
            }
            crow[q0 + u * LPR] = bytes4(c[0], c[1], c[2], c[3]);
            if (decltype(kU)::value) {
              __stcg(urow + q0 + u * LPR, hbytes4(s[0], s[1], s[2], s[3]));
              __stcg(lrow + q0 + u * LPR, bytes4(s[0], s[1], s[2], s[3]));
            }
          }
        }
      };
      using T_ = std::true_type;
      using F_ = std::false_type;
      if (!U) emit(T_{}, F_{});
      else if (lam < 0x1p100f) emit(T_{}, T_{});
      else emit(F_{}, T_{});  // 2^15 lambda overflows (rows of ~1e-28)
    }
    __syncthreads();  // this buffer is free for the window staged in the next iteration
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
// tile geometry for the tiled kernel, or TW = 0 when it does not apply
static im2t::Tile im2col_tile_geom(const ConvGeom& g, int Kp, bool vec) {
  im2t::Tile t{0, 0, 0, 0, 0};
  if (getenv("LRQMM_IM2COL_GATHER")) return t;
  if (g.dw != 1 || g.kw < g.sw || Kp % 4 || g.Wo <= 0) return t;
  const int K = g.kh * g.kw * g.C;
  // zero strip read by the padded columns of every pixel of the tile (a quad of 4 when vec)
  auto zero_strip = [&](int tw) { return K < Kp ? (((tw - 1) * g.sw * g.C + 4) + 3) & ~3 : 0; };
  // per-CTA target (several CTAs per SM keep cp.async and the quantize pass overlapped); a tile
  // narrower than min(8, Wo) pixels re-reads too much halo per row: the gather kernel then
  static const int target = env_int("LRQMM_IM2COL_SMEM_KB", 56) * 1024;
  static const int min_tw = env_int("LRQMM_IM2COL_MIN_TW", 8);
  // widest tile of at most 64 pixels within `budget` bytes, 0 if narrower than min(mtw, Wo)
  auto widest = [&](int budget, int mtw) {
    int tw = g.Wo < 64 ? g.Wo : 64;
    for (;; tw = (tw + 1) / 2) {
      const int WI = (tw - 1) * g.sw + g.kw;
      im2t::Tile c{tw, 0, WI, WI * g.C, zero_strip(tw)};
      const int bytes = im2t::smem_bytes(g, c, Kp, vec);
      if (bytes <= budget && bytes <= im2t::kBudget) break;
      if (tw == 1) return 0;
    }
    return tw < (g.Wo < mtw ? g.Wo : mtw) ? 0 : tw;
  };
  int tw = widest(target, min_tw);
  // deep windows (C >= 256: 14- and 7-pixel rows) where no 8-pixel tile fits the per-CTA target:
  // one or two CTAs per SM with tiles of >= 4 pixels still beat the gather kernel (layer3.x.conv2
  // 150 -> 114 us, layer3.0.conv2 158 -> 133, layer4.x.conv2 77 -> 74)
  if (tw == 0) tw = widest(env_int("LRQMM_IM2COL_DEEP_KB", 100) * 1024, 4);
  if (tw == 0) return t;
  // balance: the fewest tiles of at most tw pixels, equal widths
  const int ntw = (g.Wo + tw - 1) / tw;
  t.TW = (g.Wo + ntw - 1) / ntw;
  t.ntw = (g.Wo + t.TW - 1) / t.TW;
  t.WI = (t.TW - 1) * g.sw + g.kw;
  t.RS = t.WI * g.C;
  t.zero = zero_strip(t.TW);
  return t;
}

template <bool kVec, int VPT, int LPR>
static void im2col_tile_t(const QuantArgs& a, const ConvGeom& g, const im2t::Tile& tl, cudaStream_t st) {
  const int smem = im2t::smem_bytes(g, tl, a.Kp, kVec);
  static std::atomic<unsigned> done[3];  // the attribute is the budget, not this launch's size
  const int64_t ntiles = (int64_t)g.batch * g.Ho * tl.ntw;
  auto go = [&](auto kernel, std::atomic<unsigned>& d) {
    ensure_smem(kernel, im2t::kBudget, d);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, im2t::kThreads, smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    int64_t grid = (int64_t)sm_count() * per_sm;  // persistent: one wave, tiles strided over it
    if (grid > ntiles) grid = ntiles;
    launch_pdl(kernel, (int)grid, im2t::kThreads, smem, st, a.X, g, tl, a.K, a.Kp, a.qmax, a.codes, a.lam, a.inv_lam,
               a.err_flag, a.U, a.ldu, a.uplane, ntiles);
  };
  if (a.mode == kRoundFloor) go(k1_quantize_im2col_tile<kRoundFloor, kVec, VPT, LPR>, done[0]);
  else if (a.mode == kRoundTrunc) go(k1_quantize_im2col_tile<kRoundTrunc, kVec, VPT, LPR>, done[1]);
  else go(k1_quantize_im2col_tile<kRoundNearest, kVec, VPT, LPR>, done[2]);
  ++launch_counter();
}

static bool im2col_l16() {  // A/B: LRQMM_IM2COL_L16=0 keeps 32 lanes x 5 quads for 81..144 quads
  static const bool on = !(getenv("LRQMM_IM2COL_L16") && atoi(getenv("LRQMM_IM2COL_L16")) == 0);
  return on;
}
// lanes per row / quads per lane: the fewest idle quad slots, short rows shared by sub-warps
template <bool kVec>
static void im2col_tile_v(const QuantArgs& a, const ConvGeom& g, const im2t::Tile& tl, cudaStream_t st) {
  const int nq = a.Kp / 4;
  if (nq <= 8) im2col_tile_t<kVec, 1, 8>(a, g, tl, st);
  else if (nq <= 16) im2col_tile_t<kVec, 2, 8>(a, g, tl, st);
  else if (nq <= 40) im2col_tile_t<kVec, 5, 8>(a, g, tl, st);
  else if (nq <= 80) im2col_tile_t<kVec, 5, 16>(a, g, tl, st);
  else if (nq <= 144 && im2col_l16()) im2col_tile_t<kVec, 9, 16>(a, g, tl, st);  // 3x3 / C = 64: 16 x 9 = 144 quads
  else if (nq <= 160) im2col_tile_t<kVec, 5, 32>(a, g, tl, st);
  else if (nq <= 288 && im2col_l16()) im2col_tile_t<kVec, 9, 32>(a, g, tl, st);  // 3x3 / C = 128: 32 x 9 = 288
  else im2col_tile_t<kVec, 5, 32>(a, g, tl, st);
}

template <bool kVec, int VPT>
static void im2col_launch(const QuantArgs& a, const ConvGeom& g, cudaStream_t st) {
  const int nsm = sm_count();
  int64_t blocks = (a.rows + 7) / 8;
  if (blocks > 16LL * nsm) blocks = 16LL * nsm;
  const int gb = (int)(blocks < 1 ? 1 : blocks);
#define IM_ARGS a.X, g, a.K, a.Kp, a.qmax, a.codes, a.lam, a.inv_lam, a.err_flag, a.U, a.ldu, a.uplane, (int)a.rows
  if (a.mode == kRoundFloor) launch_pdl(k1_quantize_im2col<kRoundFloor, kVec, VPT>, gb, 256, 0, st, IM_ARGS);
  else if (a.mode == kRoundTrunc) launch_pdl(k1_quantize_im2col<kRoundTrunc, kVec, VPT>, gb, 256, 0, st, IM_ARGS);
  else launch_pdl(k1_quantize_im2col<kRoundNearest, kVec, VPT>, gb, 256, 0, st, IM_ARGS);
#undef IM_ARGS
  ++launch_counter();
}
// groups per lane and batch: the row in one register batch when it fits in 9, else the batch size
// (8 or 9) that leaves the fewest idle slots (K = 1152 / 2304 / 4608 = 9 / 18 / 36 float4 per lane)
template <bool kVec>
static void im2col_t(const QuantArgs& a, const ConvGeom& g, cudaStream_t st) {
  const int per = 32 * (kVec ? 4 : 1);
  const int need = (a.Kp + per - 1) / per;
  if (need <= 2) return im2col_launch<kVec, 2>(a, g, st);
  if (need <= 4) return im2col_launch<kVec, 4>(a, g, st);
  if (need <= 8) return im2col_launch<kVec, 8>(a, g, st);
  if (need <= 9) return im2col_launch<kVec, 9>(a, g, st);
  const int slots8 = (need + 7) / 8 * 8, slots9 = (need + 8) / 9 * 9;
  if (slots9 < slots8) return im2col_launch<kVec, 9>(a, g, st);
  im2col_launch<kVec, 8>(a, g, st);
}

void launch_quantize_im2col(const QuantArgs& a, const ConvGeom& g, cudaStream_t st) {
  if (a.rows == 0) return;
  const bool vec = g.C % 4 == 0 && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  const im2t::Tile tl = im2col_tile_geom(g, a.Kp, vec);
  if (tl.TW > 0) {
    if (vec) im2col_tile_v<true>(a, g, tl, st);
    else im2col_tile_v<false>(a, g, tl, st);
    return;
  }
  if (vec) im2col_t<true>(a, g, st);
  else im2col_t<false>(a, g, st);
}

void launch_tensor_scale(const float* X, int64_t ldx, int64_t rows, int K, int qmax, float* row_amax, float* lam_rows,
                         float* inv_rows, float* lam_scalar, int* err_flag, cudaStream_t st) {
  if (rows > 0) {
    int grid = rows < 148 * 16 ? (int)rows : 148 * 16;
    launch_pdl(k1_row_amax, grid, 256, 0, st, X, ldx, (int)rows, K, row_amax, err_flag); ++launch_counter();
  }
  launch_pdl(k1_tensor_scale, 1, 1024, 0, st, row_amax, (int)rows, qmax, lam_rows, inv_rows, lam_scalar); ++launch_counter();
}

// QuantTensor (Eq. gemm_r_split): the fp32 residual
// r = fp32(x - code / lambda), formed in fp64 with a correctly rounded division and rounded once
// to fp32 -- the GEMM operand the paper re-quantizes (oracle.qt_gemm does the same).
__global__ void __launch_bounds__(256) k_resid_f32(const float* __restrict__ X, int64_t ldx,
                                                   const int8_t* __restrict__ codes, int Kp,
                                                   const float* __restrict__ lam, int64_t rows, int K,
                                                   float* __restrict__ R) {
  ::lrqmm::pdl_enter();
  const int64_t total = rows * K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / K;
    const int j = (int)(e % K);
    const double xt = __ddiv_rn((double)codes[i * Kp + j], (double)lam[i]);
    R[e] = __double2float_rn(__dsub_rn((double)X[i * ldx + j], xt));
  }
}

void launch_resid_f32(const float* X, int64_t ldx, const int8_t* codes, int Kp, const float* lam, int64_t rows, int K,
                      float* R, cudaStream_t st) {
  const int64_t total = rows * K;
  if (total == 0) return;
  const int g = (int)((total + 255) / 256 < 148 * 64 ? (total + 255) / 256 : 148 * 64);
  launch_pdl(k_resid_f32, g, 256, 0, st, X, ldx, codes, Kp, lam, rows, K, R);
  ++launch_counter();
}

}  // namespace lrqmm
