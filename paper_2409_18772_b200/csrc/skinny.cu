// Small right-multiplies by W x W matrices (orthonormalisation transforms and the
// factor assembly of Algorithm 2).
#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

static int clamp_grid(int64_t want) { return (int)(want < 148 * 32 ? (want < 1 ? 1 : want) : 148 * 32); }

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

// OUT = IN S with S in fp64 and fp64 accumulation (orthonormalisation: keeps Q orthonormal to
// fp32 rounding instead of cond(IN) * eps32)
__global__ void __launch_bounds__(256) k_apply64(const float* __restrict__ IN, const double* __restrict__ S, int64_t n,
                                                 int W, float* __restrict__ OUT) {
  __shared__ double s[64 * 64];
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) s[e] = S[e];
  __syncthreads();
  const int per_blk = 256 / W;
  for (int64_t base = (int64_t)blockIdx.x * per_blk; base < n; base += (int64_t)gridDim.x * per_blk) {
    const int lr = threadIdx.x / W, o = threadIdx.x % W;
    const int64_t i = base + lr;
    if (lr < per_blk && i < n) {
      double a = 0.0;
      const float* in = IN + i * W;
      for (int c = 0; c < W; ++c) a = fma((double)__ldg(in + c), s[c * W + o], a);
      OUT[i * W + o] = (float)a;
    }
  }
}

void launch_apply64(const float* IN, const double* S, int64_t n, int W, float* OUT, cudaStream_t st) {
  if (n == 0) return;
  const int per_blk = 256 / W;
  k_apply64<<<clamp_grid((n + per_blk - 1) / per_blk), 256, 0, st>>>(IN, S, n, W, OUT);
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
