// Microbenchmark: per-SM FP64 and FP32 FMA throughput (independent chains, all SMs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/fp64_rate.cu -o tools/fp64_rate
#include <cstdio>
template <typename T>
__global__ void rate(T* out, int iters) {
  T a[8];
  for (int i = 0; i < 8; ++i) a[i] = (T)(threadIdx.x + i);
  const T b = (T)1.0000001, c = (T)0.9999999;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] * b + c;
  T s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == (T)123.456) out[0] = s;
}
int main() {
  double* d; float* f;
  cudaMalloc(&d, 8); cudaMalloc(&f, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {
    rate<double><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e0); rate<double><<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * threads * iters * 8;
    printf("fp64: %.2f TFMA/s\n", fma / ms / 1e9);
    rate<float><<<blocks, threads>>>(f, iters);
    cudaEventRecord(e0); rate<float><<<blocks, threads>>>(f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("fp32: %.2f TFMA/s\n", fma / ms / 1e9);
  }
  return 0;
}
