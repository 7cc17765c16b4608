// Latency probes (cycles per dependent op, one warp): DFMA, DMUL, SHFL, F2F, MUFU, fp64 rsqrt,
// rcp/rsqrt.approx.f64 (MUFU.RCP64H/RSQ64H), __syncthreads with 8 warps, LDS->STS->BAR round.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[256];
  double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
  float f = (float)x0;
  int iv = threadIdx.x;
  long long t0, t1;
  sm[threadIdx.x] = x;
  __syncthreads();
#define PROBE(slot, body)                                      \
  t0 = clock64();                                              \
  for (int i = 0; i < n; ++i) { body; }                        \
  t1 = clock64();                                              \
  if (threadIdx.x == 0) cyc[slot] = (t1 - t0);
  PROBE(0, x = fma(x, y, 1e-12))
  PROBE(1, x = x * y)
  PROBE(2, iv = __shfl_sync(0xffffffffu, iv, (iv + 1) & 31))
  PROBE(3, x = __shfl_sync(0xffffffffu, x, 3))
  PROBE(4, f = (float)((double)f * 1.0000001))
  PROBE(5, f = rsqrtf(f + 1.f))
  PROBE(6, x = rsqrt(x + 1.0))
  PROBE(7, x = 1.0 / (x + 1.0))
  PROBE(8, __syncthreads())
  PROBE(9, { double v = sm[(threadIdx.x + i) & 255]; __syncthreads(); sm[threadIdx.x] = v + 1.0; __syncthreads(); })
  PROBE(10, x = sqrt(x + 1.0))
  PROBE(11, f = __fdividef(1.f, f + 1.f))
  PROBE(12, asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x)))
  PROBE(13, asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x)))
  out[threadIdx.x] = x + f + iv;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 256 * 8); cudaMallocManaged(&cyc, 16 * 8);
  const int n = 4096;
  k<<<1, 256>>>(out, cyc, 0.5, n); cudaDeviceSynchronize();
  k<<<1, 256>>>(out, cyc, 0.5, n); cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DMUL", "SHFL.32", "SHFL.64", "F2F f->d->f (+DMUL)", "MUFU rsqrtf(+FADD)", "fp64 rsqrt(+DADD)",
                         "fp64 div(+DADD)", "syncthreads (8 warps)", "LDS+BAR+STS+BAR", "fp64 sqrt(+DADD)", "fdividef(+FADD)", "MUFU.RCP64H", "MUFU.RSQ64H"};
  for (int i = 0; i < 14; ++i) printf("%-24s %7.1f cyc\n", names[i], (double)cyc[i] / n);
  return 0;
}
