// Micro-benchmark of the truncation eigensolver (solvers.cuh) on a realistic W^T W (tools/eig_G24.bin,
// c2-like residual sketch, n = 24, r = 16): device time per solve (globaltimer inside the kernel) for
// the thread-group sizes the library uses.   nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -std=c++17 -I paper_2409_18772_b200/csrc tools/eig_bench.cu -o tools/eig_bench
#include <cstdio>
#include <vector>

#define LRQMM_EIG_STATS
#include "solvers.cuh"

using namespace lrqmm;

template <int n, int NT, int NA = n>
__global__ void k_bench(const double* G, float* T, int r, unsigned long long* t) {
  extern __shared__ double dyn[];
  __shared__ double aux[(eig_aux_bytes(NT) + 7) / 8];
  unsigned long long t0, t1;
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x < NT) group_eig_trunc<n, NT, NA>(G, T, r, dyn, aux, threadIdx.x, 1);
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) *t = t1 - t0;
}

template <int n>
__global__ void k_bench_warp(const double* G, float* T, int r, unsigned long long* t) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  warp_eig_trunc<n>(G, T, r);
  __syncwarp();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) *t = t1 - t0;
}

template <int n>
__global__ void k_bench_chol(const double* G, double* T64, unsigned long long* t) {
  __shared__ double sm[3 * 32 * 33];
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  warp_chol_orth<n>(G, T64, sm, sm + 32 * 33, sm + 2 * 32 * 33);
  __syncwarp();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) *t = t1 - t0;
}

template <int n>
void run_chol(const double* dG, unsigned long long* dt) {
  double* dT;
  cudaMalloc(&dT, 8 * n * n);
  unsigned long long best = ~0ull;
  for (int i = 0; i < 20; ++i) {
    k_bench_chol<n><<<1, 32>>>(dG, dT, dt);
    unsigned long long t;
    cudaMemcpy(&t, dt, 8, cudaMemcpyDeviceToHost);
    if (t < best) best = t;
  }
  std::vector<double> T(n * n);
  cudaMemcpy(T.data(), dT, 8 * n * n, cudaMemcpyDeviceToHost);
#ifdef LRQMM_CHOL_PROF
  long long pc[8];
  cudaMemcpyFromSymbol(pc, chol_prof, sizeof pc);
  printf("chol n=%d phases (cycles): load %lld  factor %lld  transform %lld  output %lld\n", n, pc[1] - pc[0], pc[2] - pc[1],
         pc[3] - pc[2], pc[4] - pc[3]);
#endif
  printf("chol n=%d  best %.1f us   T[0][0..2] = %.6e %.6e %.6e  (%s)\n", n, best / 1e3, T[0], T[1], T[2],
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dT);
}

template <int NT, int n = 24, int NA = n>
void run(const double* dG, float* dT, unsigned long long* dt) {
  cudaFuncSetAttribute(k_bench<n, NT, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, eig_smem_bytes(n));
  unsigned long long best = ~0ull;
  for (int i = 0; i < 20; ++i) {
    k_bench<n, NT, NA><<<1, NT, eig_smem_bytes(n)>>>(dG, dT, 16, dt);
    unsigned long long t;
    cudaMemcpy(&t, dt, 8, cudaMemcpyDeviceToHost);
    if (t < best) best = t;
  }
  std::vector<float> T(n * n);
  cudaMemcpy(T.data(), dT, sizeof(float) * n * n, cudaMemcpyDeviceToHost);
  if (NT == 192) {
    char fn[64];
    snprintf(fn, sizeof fn, "gpurun_out/eig_T_256_n%d.bin", n);
    FILE* o = fopen(fn, "wb");
    if (o) { fwrite(T.data(), 4, T.size(), o); fclose(o); }
  }
  int steps = 0;
  cudaMemcpyFromSymbol(&steps, eig_stats_steps, sizeof(int));
  printf("steps %d  ", steps);
  printf("n=%d NA=%d ", n, NA);
  printf("NT=%3d  best %.1f us   T[0][0..3] = %.6f %.6f %.6f %.6f  (%s)\n", NT, best / 1e3, T[0], T[1], T[2], T[3],
         cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "tools/eig_G24.bin";
  std::vector<double> G(24 * 24);
  FILE* f = fopen(path, "rb");
  if (!f || fread(G.data(), 8, G.size(), f) != G.size()) { printf("cannot read %s\n", path); return 1; }
  fclose(f);
  double* dG; float* dT; unsigned long long* dt;
  cudaMalloc(&dG, 8 * G.size()); cudaMalloc(&dT, 4 * G.size()); cudaMalloc(&dt, 8);
  cudaMemcpy(dG, G.data(), 8 * G.size(), cudaMemcpyHostToDevice);
  run_chol<24>(dG, dt);
  run<256>(dG, dT, dt);
  run<192>(dG, dT, dt);
  run<160>(dG, dT, dt);
  run<128>(dG, dT, dt);
  run<96>(dG, dT, dt);
  run<64>(dG, dT, dt);
  run<192, 24, 22>(dG, dT, dt);
  run<160, 24, 22>(dG, dT, dt);
  run<128, 24, 22>(dG, dT, dt);
  {
    unsigned long long best = ~0ull;
    for (int i = 0; i < 20; ++i) {
      k_bench_warp<24><<<1, 32>>>(dG, dT, 16, dt);
      unsigned long long t;
      cudaMemcpy(&t, dt, 8, cudaMemcpyDeviceToHost);
      if (t < best) best = t;
    }
    std::vector<float> T(24 * 24);
    cudaMemcpy(T.data(), dT, sizeof(float) * 24 * 24, cudaMemcpyDeviceToHost);
    printf("warp one-sided  best %.1f us   T[0][0..3] = %.6f %.6f %.6f %.6f  (%s)\n", best / 1e3, T[0], T[1], T[2], T[3],
           cudaGetErrorString(cudaGetLastError()));
    FILE* o = fopen("gpurun_out/eig_T_warp.bin", "wb");
    if (o) { fwrite(T.data(), 4, T.size(), o); fclose(o); }
  }
  {  // c4-like n = 32 (tools/eig_gen.py)
    std::vector<double> G32(32 * 32);
    FILE* f32 = fopen("tools/eig_G32.bin", "rb");
    if (f32 && fread(G32.data(), 8, G32.size(), f32) == G32.size()) {
      double* dG32;
      float* dT32;
      cudaMalloc(&dG32, 8 * G32.size());
      cudaMalloc(&dT32, 4 * G32.size());
      cudaMemcpy(dG32, G32.data(), 8 * G32.size(), cudaMemcpyHostToDevice);
      run_chol<32>(dG32, dt);
      run<256, 32>(dG32, dT32, dt);
      run<192, 32>(dG32, dT32, dt);
      run<160, 32>(dG32, dT32, dt);
      run<128, 32>(dG32, dT32, dt);
      run<192, 32, 26>(dG32, dT32, dt);
    }
    if (f32) fclose(f32);
  }
  return 0;
}
