// Small right-multiplies by W x W matrices (orthonormalisation transforms and the
// factor assembly of Algorithm 2).
#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

[[maybe_unused]] static int clamp_grid(int64_t want) { return (int)(want < 148 * 32 ? (want < 1 ? 1 : want) : 148 * 32); }

// ----------------------------------------------------- small right-multiplies
// One thread per row: the row's W inputs in registers, the small matrix broadcast from shared
// memory (every lane reads the same element), all outputs of the row accumulated in registers.
// OUT[i, col0 + o] = sum_c IN1[i,c] S1[c,o] (+ sum_c IN2[i,c] S2[c,o]),  o < nout (<= W)
template <int W>
__global__ void __launch_bounds__(128) k_apply_small(const float* __restrict__ IN1, const float* __restrict__ S1,
                                                     const float* __restrict__ IN2, const float* __restrict__ S2,
                                                     int64_t n, int ldS, int nout, float* __restrict__ OUT,
                                                     int64_t ldo, int col0) {
  __shared__ float s1[W * W];
  __shared__ float s2[W * W];
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
    const int c = e / W, o = e % W;
    s1[e] = o < nout ? S1[c * ldS + o] : 0.f;
    s2[e] = (IN2 && o < nout) ? S2[c * ldS + o] : 0.f;
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float x[W];
    const float4* r1 = reinterpret_cast<const float4*>(IN1 + i * W);
#pragma unroll
    for (int c = 0; c < W / 4; ++c) {
      const float4 v = __ldg(r1 + c);
      x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
    }
    float acc[W];
#pragma unroll
    for (int o = 0; o < W; ++o) acc[o] = 0.f;
#pragma unroll
    for (int c = 0; c < W; ++c)
#pragma unroll
      for (int o = 0; o < W; ++o) acc[o] = fmaf(x[c], s1[c * W + o], acc[o]);
    if (IN2) {
      const float4* r2 = reinterpret_cast<const float4*>(IN2 + i * W);
#pragma unroll
      for (int c = 0; c < W / 4; ++c) {
        const float4 v = __ldg(r2 + c);
        x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
      }
#pragma unroll
      for (int c = 0; c < W; ++c)
#pragma unroll
        for (int o = 0; o < W; ++o) acc[o] = fmaf(x[c], s2[c * W + o], acc[o]);
    }
    float* out = OUT + i * ldo + col0;
#pragma unroll
    for (int o = 0; o < W; ++o)
      if (o < nout) out[o] = acc[o];
  }
}

static int grid_rows(int64_t n, int per) {
  const int64_t want = (n + per - 1) / per;
  return (int)(want < 148 * 16 ? (want < 1 ? 1 : want) : 148 * 16);
}

void launch_apply_small(const float* IN1, const float* S1, const float* IN2, const float* S2, int64_t n, int W,
                        int ldS, int nout, float* OUT, int64_t ldo, int col0, cudaStream_t st) {
  if (n == 0 || nout == 0) return;
  const int g = grid_rows(n, 128);
#define AS_CASE(w) \
  case w: k_apply_small<w><<<g, 128, 0, st>>>(IN1, S1, IN2, S2, n, ldS, nout, OUT, ldo, col0); break;
  switch (W) { AS_CASE(8) AS_CASE(16) AS_CASE(24) AS_CASE(32) AS_CASE(40) AS_CASE(48) AS_CASE(56) AS_CASE(64) default: break; }
#undef AS_CASE
  ++launch_counter();
}

// OUT = IN S with S in fp64 and fp64 accumulation (orthonormalisation: keeps Q orthonormal to
// fp32 rounding instead of cond(IN) * eps32).  One thread per row, as above.
template <int W>
__global__ void __launch_bounds__(128) k_apply64(const float* __restrict__ IN, const double* __restrict__ S, int64_t n,
                                                 float* __restrict__ OUT) {
  __shared__ double s[W * W];
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) s[e] = S[e];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float x[W];
    const float4* r = reinterpret_cast<const float4*>(IN + i * W);
#pragma unroll
    for (int c = 0; c < W / 4; ++c) {
      const float4 v = __ldg(r + c);
      x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
    }
    double acc[W];
#pragma unroll
    for (int o = 0; o < W; ++o) acc[o] = 0.0;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const double xc = (double)x[c];
#pragma unroll
      for (int o = 0; o < W; ++o) acc[o] = fma(xc, s[c * W + o], acc[o]);
    }
    float4* out = reinterpret_cast<float4*>(OUT + i * W);
#pragma unroll
    for (int c = 0; c < W / 4; ++c)
      out[c] = make_float4((float)acc[4 * c], (float)acc[4 * c + 1], (float)acc[4 * c + 2], (float)acc[4 * c + 3]);
  }
}

void launch_apply64(const float* IN, const double* S, int64_t n, int W, float* OUT, cudaStream_t st) {
  if (n == 0) return;
  const int g = grid_rows(n, 128);
#define A64_CASE(w) case w: k_apply64<w><<<g, 128, 0, st>>>(IN, S, n, OUT); break;
  switch (W) { A64_CASE(8) A64_CASE(16) A64_CASE(24) A64_CASE(32) A64_CASE(40) A64_CASE(48) A64_CASE(56) A64_CASE(64) default: break; }
#undef A64_CASE
  ++launch_counter();
}

__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}
void launch_f64_to_f32(const double* in, float* out, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  k_f64_to_f32<<<clamp_grid((n + 255) / 256), 256, 0, st>>>(in, out, n);
  ++launch_counter();
}

__global__ void k_recip(const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __frcp_rn(in[i]);
}

void launch_recip(const float* in, float* out, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  k_recip<<<clamp_grid((n + 255) / 256), 256, 0, st>>>(in, out, n);
  ++launch_counter();
}

}  // namespace lrqmm
