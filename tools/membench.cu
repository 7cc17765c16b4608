// Read-bandwidth microbenchmark on B200 for the access patterns of liblrqmm's passes.
//   1) LDG.128 streaming (grid-stride, 4 loads in flight per thread)
//   2) TMA 2D boxes {32 fp32, 128 rows} walking along K per CTA (tc_proj ROW pattern)
//   3) TMA 2D boxes {128 fp32, 32 rows} (tc_proj COL pattern)
//   4) TMA 2D boxes {64 fp32, 128 rows} (256 B rows)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2409_18772_b200/csrc tools/membench.cu -o tools/membench -lcuda
#include <cuda.h>
#include <cstdio>
#include "common.cuh"

using namespace lrqmm;

__global__ void ldg_sum(const float4* __restrict__ x, size_t n4, float* out) {
  float acc = 0.f;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = __ldcs(x + i), b = __ldcs(x + i + stride), c = __ldcs(x + i + 2 * stride), d = __ldcs(x + i + 3 * stride);
    acc += a.x + b.y + c.z + d.w;
  }
  if (acc == 12345.f) *out = acc;
}

// one elected thread streams boxes through an RST-deep ring; all threads "consume" by reading a word
template <int RST>
__global__ void tma_stream(const __grid_constant__ CUtensorMap map, int box_inner, int box_outer, int nblk_outer,
                           int nkb, int inner_step, float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int tile = box_inner * box_outer * 4;
  __shared__ uint64_t full[RST], empty[RST];
  if (threadIdx.x == 0) {
    for (int s = 0; s < RST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  float acc = 0.f;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int units = nblk_outer;  // units = outer blocks; each walks nkb tiles along inner
  if (warp == 8) {
    if (lane == 0) {
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x)
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % RST;
        mbar_wait(&empty[s], ((it / RST) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], tile);
        tma_load_2d(sm + s * tile, &map, &full[s], kb * inner_step, u * box_outer);
      }
    }
    __syncwarp();
    return;
  }
  int it = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x)
    for (int kb = 0; kb < nkb; ++kb, ++it) {
      const int s = it % RST;
      mbar_wait(&full[s], (it / RST) & 1);
      acc += lds32(smem_u32(sm + s * tile) + 4 * threadIdx.x);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  if (acc == 12345.f) *out = acc;
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const size_t rows = 16384, cols = 16384, n = rows * cols;
  float* x;
  float* out;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&out, 4);
  cudaMemset(x, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int bpsm : {2, 4, 8}) {
    ldg_sum<<<148 * bpsm, 256>>>((const float4*)x, n / 4, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) ldg_sum<<<148 * bpsm, 256>>>((const float4*)x, n / 4, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG.128 stream, %d CTA/SM: %.0f GB/s\n", bpsm, 5.0 * n * 4 / (ms * 1e-3) / 1e9);
  }
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  struct Cfg { int bi, bo; const char* name; };
  for (Cfg c : {Cfg{32, 128, "box 32x128 (128 B rows)"}, Cfg{128, 32, "box 128x32 (512 B rows)"},
                Cfg{64, 128, "box 64x128 (256 B rows)"}, Cfg{256, 16, "box 256x16 (1 KB rows)"}}) {
    alignas(64) CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t str[1] = {cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.bi, (cuuint32_t)c.bo};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tile = c.bi * c.bo * 4;
    for (int rst : {4, 8}) {
      const int smem = rst * tile + 1024;
      const int nblk = rows / c.bo, nkb = cols / c.bi;
      if (rst == 4) {
        cudaFuncSetAttribute(tma_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_stream<4><<<148, 288, smem>>>(m, c.bi, c.bo, nblk, nkb, c.bi, out);
        cudaEventRecord(e0);
        tma_stream<4><<<148, 288, smem>>>(m, c.bi, c.bo, nblk, nkb, c.bi, out);
      } else {
        cudaFuncSetAttribute(tma_stream<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_stream<8><<<148, 288, smem>>>(m, c.bi, c.bo, nblk, nkb, c.bi, out);
        cudaEventRecord(e0);
        tma_stream<8><<<148, 288, smem>>>(m, c.bi, c.bo, nblk, nkb, c.bi, out);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("TMA %s, ring %d (%d KB in flight/SM): %.0f GB/s  [%s]\n", c.name, rst, rst * tile / 1024,
             (double)n * 4 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
