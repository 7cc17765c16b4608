// Microbenchmark: issue rate of back-to-back tcgen05.mma (one thread per CTA, 148 CTAs), cycles
// per instruction for the shapes the RSVD passes could use (operand contents irrelevant).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2409_18772_b200/csrc tools/mma_rate.cu -o tools/mma_rate
#include <cstdio>

#include "common.cuh"

using namespace lrqmm;

__device__ uint64_t desc_k(uint32_t addr) {  // K-major SW128, SBO 1024
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)(1u) << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

template <int V, int NACC, int ROT, int COMMIT>
__global__ void rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t cb[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 110000 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&cb[0], 1);
    mbar_init(&cb[1], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint64_t dA = desc_k(smem_u32(sm));
    const uint64_t dB = desc_k(smem_u32(sm + 32768));
    const uint32_t ta = tm + 384;  // A in TMEM at column 384
    // idesc: c f32 (bit 4); tf32 a/b format 2, f16-kind bf16 format 1; N >> 3 at 17, M >> 4 at 24
    constexpr uint32_t N = V == 0 ? 32 : V == 1 ? 32 : V == 2 ? 32 : V == 3 ? 96 : V == 4 ? 160 : V == 5 ? 32 : V == 6 ? 32 : 256;
    constexpr uint32_t fmt = (V <= 1 || V == 7) ? 2u : 1u;
    constexpr uint32_t id = (1u << 4) | (fmt << 7) | (fmt << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t idi8 = (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0;
      const uint32_t tmd = tm + (uint32_t)((i % NACC) * 64);
      const uint64_t dBv = dB + (uint64_t)(ROT ? ((i & 7) * 6144) >> 4 : 0);  // rotate B over 8 ring slots
      if (V == 0 || V == 7)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tmd), "r"(ta), "l"(dBv), "r"(id), "r"(acc) : "memory");
      else if (V == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmd), "l"(dA), "l"(dBv), "r"(id), "r"(acc) : "memory");
      else if (V == 2 || V == 3 || V == 4)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tmd), "r"(ta), "l"(dBv), "r"(id), "r"(acc) : "memory");
      else if (V == 5)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmd), "l"(dA), "l"(dBv), "r"(id), "r"(acc) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmd), "l"(dA), "l"(dBv), "r"(idi8), "r"(acc) : "memory");
      if (COMMIT && (i & 3) == 3) {
        umma_commit(&cb[0]);
        umma_commit(&cb[1]);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(tm);
}

template <int V, int NACC = 1, int ROT = 0, int COMMIT = 0>
void run(const char* name, unsigned long long* d) {
  cudaFuncSetAttribute(rate<V, NACC, ROT, COMMIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  const int iters = 4096;
  rate<V, NACC, ROT, COMMIT><<<148, 128, 120000>>>(iters, d);
  rate<V, NACC, ROT, COMMIT><<<148, 128, 120000>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-34s %s  %.1f cycles / mma\n", name, cudaGetErrorString(e), s / 148 / iters);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  run<0>("tf32  A=tmem N=32  K=8", d);
  run<1>("tf32  A=smem N=32  K=8", d);
  run<7>("tf32  A=tmem N=256 K=8", d);
  run<2>("bf16  A=tmem N=32  K=16", d);
  run<3>("bf16  A=tmem N=96  K=16", d);
  run<4>("bf16  A=tmem N=160 K=16", d);
  run<5>("bf16  A=smem N=32  K=16", d);
  run<6>("i8    A=smem N=32  K=32", d);
  run<0, 2>("tf32  A=tmem N=32 2 accumulators", d);
  run<0, 4>("tf32  A=tmem N=32 4 accumulators", d);
  run<2, 2>("bf16  A=tmem N=32 2 accumulators", d);
  run<2, 4>("bf16  A=tmem N=32 4 accumulators", d);
  run<5, 4>("bf16  A=smem N=32 4 accumulators", d);
  run<3, 4>("bf16  A=tmem N=96 4 accumulators", d);
  run<3, 1, 1>("bf16  A=tmem N=96 B rotating", d);
  run<2, 1, 1>("bf16  A=tmem N=32 B rotating", d);
  run<4, 1, 1>("bf16  A=tmem N=160 B rotating", d);
  run<5, 1, 1>("bf16  A=smem N=32 B rotating", d);
  run<3, 1, 1, 1>("bf16  A=tmem N=96 rot + 2 commits/4", d);
  run<2, 1, 1, 1>("bf16  A=tmem N=32 rot + 2 commits/4", d);
  return 0;
}
