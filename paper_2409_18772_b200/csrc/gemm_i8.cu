// K6 — integer GEMM on 5th-gen tensor cores (tcgen05.mma kind::i8) with the
// LRQMM epilogue fused: Eq. INTGEMM, Eq. QUANTGEMM
// and Algorithm 2, 364-372:
//
//   acc[i,j] = sum_k A_q[i,k] B_q[j,k]                     (int32, exact, TMEM)
//   D[i,j]   = alpha * ( acc[i,j] / (lambda_A[i] lambda_B[j])
//                        + sum_{l < 2r} L_A[i,l] L_B[j,l] ) + beta * D[i,j]
//
// where L_A = [U_A Sigma_A | A~ V_B], L_B = [B~ V_A + U_B Sigma_B (V_B^T V_A) | U_B Sigma_B]
// carry RC1 + RC2 + RC3 (the factor association of Eq. APPMM-C).
// 4-bit codes ride in int8 lanes (B200 has no 4-bit integer MMA), so int4 and int8
// run at the same rate and the int32 accumulators are bit-exact.
//
// Structure (persistent, one CTA per SM, warp-specialised):
//   warp 0     : TMA producer, 4-stage smem ring (A 128x128 B, B 256x128 B per stage, 128B swizzle)
//   warp 1     : TMEM allocator + single-thread UMMA issuer (M=128, N=256, K=32 per instruction)
//   warps 2..5 : epilogue (TMEM -> registers -> dequant + rank-2r FFMA -> global), TMEM double-buffered
//                so the epilogue of tile t overlaps the mainloop of tile t+1.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

namespace g6 {
constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 128;  // bytes = int8 elements per stage (one 128B swizzle atom row)
constexpr int UK = 32;   // K per tcgen05.mma kind::i8
constexpr int STAGES = 4;
constexpr int kThreads = 192;
constexpr int kABytes = BM * BK;
constexpr int kBBytes = BN * BK;
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kTmemCols = 512;  // 2 accumulators x 256 columns
constexpr int kGroupM = 16;     // tile rasterisation: 16 M-blocks per group (L2 reuse)
constexpr int kSmemBytes = STAGES * kStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;
}  // namespace g6

struct G6Params {
  int64_t M, N;
  int num_kb;
  int num_m, num_n;
  int epi;
  const float* lam_a;
  const float* lam_b;
  const float* LA;
  const float* LB;
  int R2;
  float alpha, beta;
  float* D;
  int32_t* Cint;
  int64_t ldd;
  int vec_ok;
};

LRQMM_DEV void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  const int per_group = g6::kGroupM * num_n;
  const int group = t / per_group;
  const int first_m = group * g6::kGroupM;
  const int gsize = min(g6::kGroupM, num_m - first_m);
  const int in = t % per_group;
  mb = first_m + in % gsize;
  nb = in / gsize;
}

template <int kR2>
LRQMM_DEV void epilogue_chunk(const G6Params& p, const uint32_t (&acc)[32], int64_t row, int col0, float sa,
                              const float (&la)[kR2 > 0 ? kR2 : 1]) {
  if (row >= p.M) return;
  if (p.epi == 0) {
    int32_t* out = p.Cint + row * p.ldd + col0;
    if (p.vec_ok && col0 + 32 <= p.N) {
#pragma unroll
      for (int c = 0; c < 32; c += 4)
        *reinterpret_cast<int4*>(out + c) = make_int4((int)acc[c], (int)acc[c + 1], (int)acc[c + 2], (int)acc[c + 3]);
    } else {
      for (int c = 0; c < 32; ++c)
        if (col0 + c < p.N) out[c] = (int)acc[c];
    }
    return;
  }
  float v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const int col = min(col0 + c, (int)p.N - 1);
    const float sb = __frcp_rn(__ldg(p.lam_b + col));
    float t = __fmul_rn(static_cast<float>(static_cast<int32_t>(acc[c])), __fmul_rn(sa, sb));
    if constexpr (kR2 > 0) {
      const float4* lb = reinterpret_cast<const float4*>(p.LB + (int64_t)col * kR2);
      float corr = 0.f;
#pragma unroll
      for (int l = 0; l < kR2; l += 4) {
        const float4 b = __ldg(lb + (l >> 2));
        corr = fmaf(la[l + 0], b.x, corr);
        corr = fmaf(la[l + 1], b.y, corr);
        corr = fmaf(la[l + 2], b.z, corr);
        corr = fmaf(la[l + 3], b.w, corr);
      }
      t = t + corr;
    }
    v[c] = p.alpha * t;
  }
  float* out = p.D + row * p.ldd + col0;
  if (p.vec_ok && col0 + 32 <= p.N) {
    if (p.beta != 0.f) {
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 o = *reinterpret_cast<const float4*>(out + c);
        v[c] = fmaf(p.beta, o.x, v[c]);
        v[c + 1] = fmaf(p.beta, o.y, v[c + 1]);
        v[c + 2] = fmaf(p.beta, o.z, v[c + 2]);
        v[c + 3] = fmaf(p.beta, o.w, v[c + 3]);
      }
    }
#pragma unroll
    for (int c = 0; c < 32; c += 4) __stcs(reinterpret_cast<float4*>(out + c), make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]));
  } else {
    for (int c = 0; c < 32; ++c) {
      if (col0 + c < p.N) {
        float o = v[c];
        if (p.beta != 0.f) o = fmaf(p.beta, out[c], o);
        out[c] = o;
      }
    }
  }
}

template <int kR2>
__global__ void __launch_bounds__(g6::kThreads, 1)
    k6_gemm_i8(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, G6Params p) {
  using namespace g6;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.num_m * p.num_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, p.num_m, p.num_n, mb, nb);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          tma_load_2d(sA + stage * kABytes, &mapA, &full[stage], kb * BK, mb * BM);
          tma_load_2d(sB + stage * kBBytes, &mapB, &full[stage], kb * BK, nb * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_i8(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        const int acc = lt & 1;
        const uint32_t acc_phase = (lt >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            const uint64_t ad = make_sw128_kmajor_desc(a_addr + k * UK);
            const uint64_t bd = make_sw128_kmajor_desc(b_addr + k * UK);
            umma_i8(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);  // frees the smem slot when these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    int lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      int mb, nb;
      tile_coords(t, p.num_m, p.num_n, mb, nb);
      const int acc = lt & 1;
      const uint32_t acc_phase = (lt >> 1) & 1;
      const int64_t row = (int64_t)mb * BM + quad * 32 + lane;
      float sa = 0.f;
      float la[kR2 > 0 ? kR2 : 1];
      if (p.epi == 1 && row < p.M) {
        sa = __frcp_rn(p.lam_a[row]);
        if constexpr (kR2 > 0) {
          const float4* lr = reinterpret_cast<const float4*>(p.LA + row * kR2);
#pragma unroll
          for (int l = 0; l < kR2; l += 4) {
            const float4 v = __ldg(lr + (l >> 2));
            la[l] = v.x; la[l + 1] = v.y; la[l + 2] = v.z; la[l + 3] = v.w;
          }
        }
      } else {
#pragma unroll
        for (int l = 0; l < (kR2 > 0 ? kR2 : 1); ++l) la[l] = 0.f;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c * 32, r);
        tmem_ld_wait();
        const int col0 = nb * BN + c * 32;
        if (col0 < p.N) epilogue_chunk<kR2>(p, r, row, col0, sa, la);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<g6::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

static int encode_codes_map(CUtensorMap* map, const int8_t* base, int64_t rows, int Kp, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return 1;
  cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)Kp};
  cuuint32_t box[2] = {(cuuint32_t)g6::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 2;
}

int gemm_prepare_maps(const GemmArgs& g, void* mapA, void* mapB) {
  if (encode_codes_map(reinterpret_cast<CUtensorMap*>(mapA), g.A, g.M, g.Kp, g6::BM)) return 1;
  if (encode_codes_map(reinterpret_cast<CUtensorMap*>(mapB), g.B, g.N, g.Kp, g6::BN)) return 1;
  return 0;
}

template <int kR2>
static void launch_t(const G6Params& p, const CUtensorMap* mA, const CUtensorMap* mB, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k6_gemm_i8<kR2>, cudaFuncAttributeMaxDynamicSharedMemorySize, g6::kSmemBytes);
    attr = true;
  }
  k6_gemm_i8<kR2><<<grid, g6::kThreads, g6::kSmemBytes, st>>>(*mA, *mB, p); ++launch_counter();
}

void launch_gemm(const GemmArgs& g, const void* mapA, const void* mapB, cudaStream_t st) {
  if (g.M == 0 || g.N == 0) return;
  G6Params p;
  p.M = g.M;
  p.N = g.N;
  p.num_kb = g.Kp / g6::BK;
  p.num_m = (int)((g.M + g6::BM - 1) / g6::BM);
  p.num_n = (int)((g.N + g6::BN - 1) / g6::BN);
  p.epi = g.epi;
  p.lam_a = g.lam_a;
  p.lam_b = g.lam_b;
  p.LA = g.LA;
  p.LB = g.LB;
  p.R2 = g.R2;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.D = g.D;
  p.Cint = g.Cint;
  p.ldd = g.ldd;
  const void* outp = g.epi == 0 ? (const void*)g.Cint : (const void*)g.D;
  p.vec_ok = ((reinterpret_cast<uintptr_t>(outp) & 15) == 0) && (g.ldd % 4 == 0);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = p.num_m * p.num_n;
  const int grid = tiles < nsm ? tiles : nsm;
  const CUtensorMap* mA = reinterpret_cast<const CUtensorMap*>(mapA);
  const CUtensorMap* mB = reinterpret_cast<const CUtensorMap*>(mapB);
  const int r2 = g.epi == 0 ? 0 : g.R2;
  switch (r2) {
    case 0: launch_t<0>(p, mA, mB, grid, st); break;
    case 8: launch_t<8>(p, mA, mB, grid, st); break;
    case 16: launch_t<16>(p, mA, mB, grid, st); break;
    case 24: launch_t<24>(p, mA, mB, grid, st); break;
    case 32: launch_t<32>(p, mA, mB, grid, st); break;
    case 40: launch_t<40>(p, mA, mB, grid, st); break;
    case 48: launch_t<48>(p, mA, mB, grid, st); break;
    case 56: launch_t<56>(p, mA, mB, grid, st); break;
    case 64: launch_t<64>(p, mA, mB, grid, st); break;
    default: break;
  }
}

}  // namespace lrqmm
