// Probe: one CTA, D[128 x 32] = A[128 x 32] * B[32 x 32] with tcgen05.mma kind::tf32
// (4 k-steps of 8), operands written to smem by threads in several layouts.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2409_18772_b200/csrc tools/mma_probe.cu -o tools/mma_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "common.cuh"

using namespace lrqmm;

__device__ uint32_t off_k(int mn, int k) {  // K-major SW128, rows of 32 fp32
  const int row = mn & 7, chunk = k >> 2;
  return (uint32_t)((mn >> 3) * 1024 + row * 128 + ((chunk ^ row) << 4) + ((k & 3) << 2));
}
__device__ uint32_t off_mn(int mn, int k, int nA) {  // MN-major SW128
  const int row = k & 7, chunk = (mn & 31) >> 2;
  return (uint32_t)((k >> 3) * (nA * 1024) + (mn >> 5) * 1024 + row * 128 + ((chunk ^ row) << 4) + ((mn & 3) << 2));
}
// MN-major SWIZZLE_128B_BASE32B (tf32): atoms of 32 MN x 4 K (512 B), 32-byte chunks XOR row
__device__ uint32_t off_mn32(int mn, int k, int lbo, int sbo) {
  const int row = k & 3;
  return (uint32_t)((k >> 2) * sbo + (mn >> 5) * lbo + row * 128 + ((((mn & 31) >> 3) ^ row) << 5) + ((mn & 7) << 2));
}
__device__ uint64_t desc_t(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t type) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)type << 61;
  return d;
}
__device__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ void mma_tf32(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(t), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

// variant: bit0 = A MN-major, bit1 = B MN-major, bit2 = idesc m_dim at bit 23 instead of 24
__global__ void probe(const float* A, const float* B, float* D, int variant) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;             // 16 KB
  uint8_t* sB = sm + 16384;     // 4 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  const bool amn = variant & 1, bmn = variant & 2;
  // A[m][k] m<128, k<32
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, k = e % 32;
    const uint32_t o = amn ? off_mn32(m, k, 512, 2048) : off_k(m, k);
    *reinterpret_cast<float*>(sA + o) = A[e];
  }
  // B[k][n] k<32, n<32
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int k = e / 32, n = e % 32;
    const uint32_t o = bmn ? off_mn32(n, k, 512, 512) : off_k(n, k);
    *reinterpret_cast<float*>(sB + o) = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (tid < 32) tmem_alloc<32>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid < 32) {
    if (tid == 0) {
      uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) | ((32u >> 3) << 17);
      id |= (variant & 4) ? ((128u >> 4) << 23) : ((128u >> 4) << 24);
      for (int k = 0; k < 4; ++k) {
        uint64_t da = amn ? desc_t(smem_u32(sA) + k * 4096, 512, 2048, 1) : desc(smem_u32(sA) + k * 32, 16, 1024);
        uint64_t db = bmn ? desc_t(smem_u32(sB) + k * 1024, 512, 512, 1) : desc(smem_u32(sB) + k * 32, 16, 1024);
        mma_tf32(tmem, da, db, id, k > 0);
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (tid < 128) {
    const int w = tid >> 5;
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(w * 32) << 16), r);
    tmem_ld_wait();
    for (int c = 0; c < 32; ++c) D[tid * 32 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) { tc_fence_after(); tmem_free<32>(tmem); }
}

int main() {
  std::vector<float> A(128 * 32), B(32 * 32), D(128 * 32), R(128 * 32);
  srand(1);
  for (auto& x : A) x = (rand() % 17 - 8) * 0.25f;
  for (auto& x : B) x = (rand() % 13 - 6) * 0.5f;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      double s = 0;
      for (int k = 0; k < 32; ++k) s += (double)A[m * 32 + k] * B[k * 32 + n];
      R[m * 32 + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int v = 0; v < 4; ++v) {
    cudaMemset(dD, 0x7f, D.size() * 4);
    probe<<<1, 128, 32768>>>(dA, dB, dD, v);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, nr = 0;
    for (size_t i = 0; i < D.size(); ++i) { err += (D[i] - R[i]) * (double)(D[i] - R[i]); nr += (double)R[i] * R[i]; }
    printf("variant %d (A %s, B %s, mdim@%d): %s rel err %.3e  D[0..3]= %g %g %g %g  ref %g %g %g %g\n", v,
           (v & 1) ? "MN" : "K", (v & 2) ? "MN" : "K", (v & 4) ? 23 : 24, cudaGetErrorString(e), sqrt(err / nr),
           D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
    if (e != cudaSuccess) break;
  }
  return 0;
}
