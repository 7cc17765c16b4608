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
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

namespace g6 {
constexpr int BM = 128;
constexpr int BN = 256;  // widest tile (the BN template parameter picks 64 / 128 / 256 by N)
constexpr int BK = 128;  // bytes = int8 elements per stage (one 128B swizzle atom row)
constexpr int UK = 32;   // K per tcgen05.mma kind::i8
constexpr int kEpiThreads = 128;  // one epilogue group: one warp per TMEM lane quarter
constexpr int kABytes = BM * BK;
#ifndef LRQMM_L2HINT
#define LRQMM_L2HINT 2  // 1: A evict_last + B evict_first, 2: A evict_last only
#endif
#ifndef LRQMM_GROUPM
#define LRQMM_GROUPM 16
#endif
constexpr int kGroupM = LRQMM_GROUPM;  // tile rasterisation: M-blocks per group (L2 reuse)
__host__ __device__ constexpr int stage_bytes(int bn) { return kABytes + bn * BK; }
__host__ __device__ constexpr int staging_bytes(int r2, int bn) { return bn * r2 * 4 + bn * 4; }
// epilogue groups = TMEM accumulators: up to 4 (512 columns / BN), each with its own L_B /
// 1/lambda_B staging, as long as >= 3 smem stages still fit; at least 2 accumulators always
__host__ __device__ constexpr int fits_groups(int g, int r2, int bn) {
  return (232448 - (g * staging_bytes(r2, bn) + 1280)) / stage_bytes(bn) >= 3;
}
__host__ __device__ constexpr int epi_groups(int r2, int bn) {
  return (512 / bn >= 4 && fits_groups(4, r2, bn)) ? 4 : (fits_groups(2, r2, bn) ? 2 : 1);
}
__host__ __device__ constexpr int num_acc(int r2, int bn) { return epi_groups(r2, bn) < 2 ? 2 : epi_groups(r2, bn); }
__host__ __device__ constexpr int threads_for(int r2, int bn) { return 64 + 128 * epi_groups(r2, bn); }
__host__ __device__ constexpr int extra_bytes(int r2, int bn) {
  return epi_groups(r2, bn) * staging_bytes(r2, bn) + 256 + 1024;
}
// as many smem stages as fit beside the L_B tile(s), at most 8
__host__ __device__ constexpr int stages_for(int r2, int bn) {
  return (232448 - extra_bytes(r2, bn)) / stage_bytes(bn) > 8 ? 8 : (232448 - extra_bytes(r2, bn)) / stage_bytes(bn);
}
__host__ __device__ constexpr int smem_bytes(int r2, int bn) { return stages_for(r2, bn) * stage_bytes(bn) + extra_bytes(r2, bn); }
// accumulators of bn columns, rounded to the power-of-two allocation granule
__host__ __device__ constexpr uint32_t tmem_cols(int cols) { return cols <= 128 ? 128 : (cols <= 256 ? 256 : 512); }
}  // namespace g6

struct G6Params {
  int64_t M, N;
  int num_kb;
  int num_m, num_n;
  int epi;
  const float* inv_a;  // RN(1/lambda_A)
  const float* inv_b;  // RN(1/lambda_B)
  const float* LA;
  const float* LB;
  float alpha, beta;
  float* D;
  int32_t* Cint;
  int64_t ldd;
  int vec_ok;
  int* sched;  // K7: global tile counter (atomicAdd), zeroed before the launch
  int group_m;  // K7: pair-tile rows per raster group
  int polA, polB;  // K7: L2 policies of the A / B loads (l2_policy kinds)
};

// raster with a runtime group height (K7)
LRQMM_DEV void tile_coords_rt(int t, int gm, int num_m, int num_n, int& mb, int& nb) {
  const int per_group = gm * num_n;
  const int group = t / per_group;
  const int first_m = group * gm;
  const int gsize = min(gm, num_m - first_m);
  const int in = t % per_group;
  mb = first_m + in % gsize;
  nb = in / gsize;
}

template <int kGM = g6::kGroupM>
LRQMM_DEV void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  const int per_group = kGM * num_n;
  const int group = t / per_group;
  const int first_m = group * kGM;
  const int gsize = min(kGM, num_m - first_m);
  const int in = t % per_group;
  mb = first_m + in % gsize;
  nb = in / gsize;
}

template <int kN = g6::kEpiThreads>
LRQMM_DEV void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kN) : "memory"); }
// named barrier `id` over one epilogue group (128 threads)
LRQMM_DEV void epi_bar_id(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(g6::kEpiThreads) : "memory"); }

// one 8-column group of one output row: acc (int32 from TMEM) -> D or Cint.
// Kept small and rolled (the 256-column tile is walked in 32 groups) so the
// epilogue code stays resident in the instruction cache.
template <int kR2>
LRQMM_DEV void epilogue_group(const G6Params& p, const uint32_t (&acc)[8], int64_t row, int col0, int cl0,
                              float sa, const float (&la)[kR2 > 0 ? kR2 : 1], uint32_t sLB, uint32_t sSB) {
  if (row >= p.M || col0 >= p.N) return;
  const bool full = p.vec_ok && col0 + 8 <= p.N;
  if (p.epi == 0) {
    int32_t* out = p.Cint + row * p.ldd + col0;
    if (full) {
      __stcs(reinterpret_cast<int4*>(out), make_int4((int)acc[0], (int)acc[1], (int)acc[2], (int)acc[3]));
      __stcs(reinterpret_cast<int4*>(out + 4), make_int4((int)acc[4], (int)acc[5], (int)acc[6], (int)acc[7]));
    } else {
      for (int c = 0; c < 8; ++c)
        if (col0 + c < p.N) out[c] = (int)acc[c];
    }
    return;
  }
  // v = alpha * (acc / (lambda_a lambda_b) + L_A[row] . L_B[col]);  sa, la carry alpha
  float v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
    v[c] = __fmul_rn(static_cast<float>(static_cast<int32_t>(acc[c])), __fmul_rn(sa, lds32(sSB + 4 * (cl0 + c))));
  if constexpr (kR2 > 0) {
#pragma unroll
    for (int l = 0; l < kR2; l += 4) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 b = lds128(sLB + 4 * ((cl0 + c) * kR2 + l));
        v[c] = fmaf(la[l + 0], b.x, v[c]);
        v[c] = fmaf(la[l + 1], b.y, v[c]);
        v[c] = fmaf(la[l + 2], b.z, v[c]);
        v[c] = fmaf(la[l + 3], b.w, v[c]);
      }
    }
  }
  float* out = p.D + row * p.ldd + col0;
  if (full) {
    if (p.beta != 0.f) {
      const float4 o0 = *reinterpret_cast<const float4*>(out);
      const float4 o1 = *reinterpret_cast<const float4*>(out + 4);
      v[0] = fmaf(p.beta, o0.x, v[0]); v[1] = fmaf(p.beta, o0.y, v[1]);
      v[2] = fmaf(p.beta, o0.z, v[2]); v[3] = fmaf(p.beta, o0.w, v[3]);
      v[4] = fmaf(p.beta, o1.x, v[4]); v[5] = fmaf(p.beta, o1.y, v[5]);
      v[6] = fmaf(p.beta, o1.z, v[6]); v[7] = fmaf(p.beta, o1.w, v[7]);
    }
    __stcs(reinterpret_cast<float4*>(out), make_float4(v[0], v[1], v[2], v[3]));
    __stcs(reinterpret_cast<float4*>(out + 4), make_float4(v[4], v[5], v[6], v[7]));
  } else {
    for (int c = 0; c < 8; ++c) {
      if (col0 + c < p.N) {
        float o = v[c];
        if (p.beta != 0.f) o = fmaf(p.beta, out[c], o);
        out[c] = o;
      }
    }
  }
}

template <int kR2, int BN>
__global__ void __launch_bounds__(g6::threads_for(kR2, BN), 1)
    k6_gemm_i8(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, G6Params p) {
  using g6::BM; using g6::BK; using g6::UK; using g6::kABytes; using g6::kEpiThreads;
  constexpr int kBBytes = BN * BK;
  constexpr int kStageBytes = kABytes + kBBytes;
  constexpr int NACC = g6::num_acc(kR2, BN);
  constexpr uint32_t kTmemCols = g6::tmem_cols(NACC * BN);
  constexpr int STAGES = g6::stages_for(kR2, BN);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // offset from the __shared__ array: shared-space accesses, not generic
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  constexpr int EG = g6::epi_groups(kR2, BN);
  float* sLB0 = reinterpret_cast<float*>(smem + STAGES * kStageBytes);  // EG groups x (BN x kR2 | BN)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLB0 + EG * (BN * kR2 + BN));
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;         // NACC
  uint64_t* tempty = tfull + NACC;             // NACC
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);

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
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiThreads);
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
#if LRQMM_L2HINT
      const uint64_t polA = l2_policy_evict_last();
#if LRQMM_L2HINT == 1
      const uint64_t polB = l2_policy_evict_first();
#endif
#endif
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, p.num_m, p.num_n, mb, nb);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
#if LRQMM_L2HINT
          tma_load_2d_hint(sA + stage * kABytes, &mapA, &full[stage], kb * BK, mb * BM, polA);
#if LRQMM_L2HINT == 1
          tma_load_2d_hint(sB + stage * kBBytes, &mapB, &full[stage], kb * BK, nb * BN, polB);
#else
          tma_load_2d(sB + stage * kBBytes, &mapB, &full[stage], kb * BK, nb * BN);
#endif
#else
          tma_load_2d(sA + stage * kABytes, &mapA, &full[stage], kb * BK, mb * BM);
          tma_load_2d(sB + stage * kBBytes, &mapB, &full[stage], kb * BK, nb * BN);
#endif
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
        const int acc = lt % NACC;
        const uint32_t acc_phase = (lt / NACC) & 1;
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
    // two groups of 4 warps; group e owns accumulator buffer e and this CTA's tiles lt = e, e+2, ...
    // so one group's staging (L_A rows, L_B tile: global-memory latency) overlaps the other's math
    // (EG == 1 when two staging buffers do not fit beside 3 stages: group 0 takes every tile)
    const int egrp = (warp - 2) >> 2;
    const int et = threadIdx.x - 64 - 128 * egrp;  // 0..127 within the group
    const int quad = warp & 3;                      // TMEM lane quadrant this warp may access
    const uint32_t sLBa = smem_u32(sLB0 + (egrp < EG ? egrp : 0) * (BN * kR2 + BN));
    const uint32_t sSBa = sLBa + 4 * BN * kR2;
    int lt = egrp;
    for (int t = blockIdx.x + egrp * gridDim.x; egrp < EG && t < num_tiles; t += EG * gridDim.x, lt += EG) {
      int mb, nb;
      tile_coords(t, p.num_m, p.num_n, mb, nb);
      const int acc = lt % NACC;
      const uint32_t acc_phase = (lt / NACC) & 1;
      const int64_t row = (int64_t)mb * BM + quad * 32 + lane;
      const int n0 = nb * BN;
      float sa = 0.f;
      float la[kR2 > 0 ? kR2 : 1];
#pragma unroll
      for (int l = 0; l < (kR2 > 0 ? kR2 : 1); ++l) la[l] = 0.f;
      if (p.epi == 1) {
        // stage this tile's column data (L_B rows, 1/lambda_b) while the mainloop runs
        epi_bar_id(1 + egrp);  // previous tile's readers are done
        for (int j = et; j < BN; j += kEpiThreads) {
          const int col = n0 + j;
          const float v = col < p.N ? __ldg(p.inv_b + col) : 0.f;
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(sSBa + 4 * j), "f"(v) : "memory");
        }
        if constexpr (kR2 > 0) {
          const float4* src = reinterpret_cast<const float4*>(p.LB + (int64_t)n0 * kR2);
          const int total4 = BN * kR2 / 4;
          const int valid4 = (int)((p.N - n0 < BN ? p.N - n0 : (int64_t)BN) * kR2 / 4);
          for (int e = et; e < total4; e += kEpiThreads)
            sts128(sLBa + 16 * e, e < valid4 ? __ldg(src + e) : make_float4(0.f, 0.f, 0.f, 0.f));
        }
        if (row < p.M) {
          sa = p.alpha * __ldg(p.inv_a + row);
          if constexpr (kR2 > 0) {
            const float4* lr = reinterpret_cast<const float4*>(p.LA + row * kR2);
#pragma unroll
            for (int l = 0; l < kR2; l += 4) {
              const float4 v = __ldg(lr + (l >> 2));
              la[l] = p.alpha * v.x; la[l + 1] = p.alpha * v.y; la[l + 2] = p.alpha * v.z; la[l + 3] = p.alpha * v.w;
            }
          }
        }
        epi_bar_id(1 + egrp);  // staged data visible to the group
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      // ping-pong 8-column TMEM loads: load group g+1 while computing group g
      uint32_t ra[8], rb[8];
      tmem_ld_32x32b_x8(t_row, ra);
#pragma unroll 1
      for (int g = 0; g < BN / 8; g += 2) {
        tmem_ld_wait();
        tmem_ld_32x32b_x8(t_row + (g + 1) * 8, rb);
        epilogue_group<kR2>(p, ra, row, n0 + g * 8, g * 8, sa, la, sLBa, sSBa);
        tmem_ld_wait();
        if (g + 2 < BN / 8) tmem_ld_32x32b_x8(t_row + (g + 2) * 8, ra);
        epilogue_group<kR2>(p, rb, row, n0 + (g + 1) * 8, (g + 1) * 8, sa, la, sLBa, sSBa);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<kTmemCols>(tmem_base);
  }
}

static int encode_codes_map(CUtensorMap* map, const int8_t* base, int64_t rows, int Kp, int box_rows);

// ------------------------------------------------------------------------------------------
// K8 — one-CTA GEMM with the low-rank correction on the TENSOR CORES (narrow shapes, where the
// FFMA epilogue of K6 is bound by its shared-memory broadcasts of L_B: 2r FMAs and 2r/4 LDS.128
// per output).  L_A and L_B are held as bf16 hi / lo pairs (x = hi + lo + O(2^-17 |x|)), rows
// zero-padded to 64 columns = one 128-byte K-major SWIZZLE_128B atom, exactly the byte layout of
// an int8 stage; per tile two extra ring stages carry [L_A hi | L_B hi] and [L_A lo | L_B lo] and
// the MMA warp adds, after the int8 main loop, hi.hi + hi.lo + lo.hi (kind::f16, 12 x K16) into a
// second fp32 TMEM accumulator.  Epilogue: D = alpha (acc / (lambda_A lambda_B) + corr) + beta D
// -- two TMEM loads and three flops per output.  BN = 128: TMEM = 2 tiles x (int32 128 | fp32 128).
namespace g8 {
constexpr int BM = 128, BN = 128, BK = 128, UK = 32;
constexpr int kStageBytes = BM * BK + BN * BK;  // 32 KB: int8 A | B, or bf16 [L_A | L_B] (hi or lo)
constexpr int kEG = 2;                          // epilogue groups (one per accumulator pair)
constexpr int kThreads = 64 + 128 * kEG;
constexpr int kStages = 6;
constexpr int kStile = 8 * 32 * 32 * 4;  // epilogue transpose tiles: 32 x 32 fp32 per epilogue warp
constexpr int kSmem = kStages * kStageBytes + kStile + kEG * BN * 4 + 256 + 1024;
static_assert(kSmem <= 232448, "K8 shared memory");
}  // namespace g8

struct G8Params {
  int64_t M, N;
  int num_kb, num_m, num_n;
  const float* inv_a;
  const float* inv_b;
  float alpha, beta;
  float* D;
  int64_t ldd;
  int vec_ok;
};

__global__ void __launch_bounds__(g8::kThreads, 1)
    k8_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
               const __grid_constant__ CUtensorMap mapLAh, const __grid_constant__ CUtensorMap mapLAl,
               const __grid_constant__ CUtensorMap mapLBh, const __grid_constant__ CUtensorMap mapLBl, G8Params p) {
  using namespace g8;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // offset from the __shared__ array: shared-space accesses, not generic
  float* stile0 = reinterpret_cast<float*>(smem + kStages * kStageBytes);  // 8 x 32 x 32 (XOR-swizzled)
  float* sSB0 = stile0 + kStile / 4;  // kEG x BN: 1/lambda_B of the tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSB0 + kEG * BN);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;  // 2
  uint64_t* tempty = tfull + 2;          // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = p.num_m * p.num_n;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    tma_prefetch_desc(&mapLAh);
    tma_prefetch_desc(&mapLAl);
    tma_prefetch_desc(&mapLBh);
    tma_prefetch_desc(&mapLBl);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp == 0) {
    // -------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto next = [&]() {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kStageBytes);
      };
      auto advance = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      };
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, p.num_m, p.num_n, mb, nb);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          next();
          uint8_t* st = smem + stage * kStageBytes;
          tma_load_2d(st, &mapA, &full[stage], kb * BK, mb * BM);
          tma_load_2d(st + BM * BK, &mapB, &full[stage], kb * BK, nb * BN);
          advance();
        }
        next();  // [L_A hi | L_B hi]
        tma_load_2d(smem + stage * kStageBytes, &mapLAh, &full[stage], 0, mb * BM);
        tma_load_2d(smem + stage * kStageBytes + BM * BK, &mapLBh, &full[stage], 0, nb * BN);
        advance();
        next();  // [L_A lo | L_B lo]
        tma_load_2d(smem + stage * kStageBytes, &mapLAl, &full[stage], 0, mb * BM);
        tma_load_2d(smem + stage * kStageBytes + BM * BK, &mapLBl, &full[stage], 0, nb * BN);
        advance();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // -------------------------------------------------------------- UMMA issuer
    if (lane == 0) {
      constexpr uint32_t idi8 = make_idesc_i8(BM, BN);
      constexpr uint32_t idbf = make_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        const int acc = lt & 1;
        mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_main = tmem_base + acc * 256, d_corr = d_main + 128;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * kStageBytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma_i8(d_main, make_sw128_kmajor_desc(a_addr + k * UK), make_sw128_kmajor_desc(a_addr + BM * BK + k * UK),
                    idi8, (kb | k) != 0 ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        // correction: stage x = [L_A hi | L_B hi], stage y = [L_A lo | L_B lo]
        const int sx = stage;
        const uint32_t px = phase;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        const int sy = stage;
        const uint32_t py = phase;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        mbar_wait(&full[sx], px);
        mbar_wait(&full[sy], py);
        tc_fence_after();
        const uint32_t xa = smem_u32(smem + sx * kStageBytes), ya = smem_u32(smem + sy * kStageBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 4 x K16 = the 64 bf16 of one atom
          const uint32_t o = k * 32;
          umma_bf16(d_corr, make_sw128_kmajor_desc(xa + o), make_sw128_kmajor_desc(xa + BM * BK + o), idbf, k != 0);
          umma_bf16(d_corr, make_sw128_kmajor_desc(xa + o), make_sw128_kmajor_desc(ya + BM * BK + o), idbf, 1u);
          umma_bf16(d_corr, make_sw128_kmajor_desc(ya + o), make_sw128_kmajor_desc(xa + BM * BK + o), idbf, 1u);
        }
        umma_commit(&empty[sx]);
        umma_commit(&empty[sy]);
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue
    // group e = accumulator pair e: tiles lt = e, e + 2, ...
    const int egrp = (warp - 2) >> 2;
    const int et = threadIdx.x - 64 - 128 * egrp;
    const int quad = warp & 3;
    float* sSB = sSB0 + egrp * BN;
    int lt = egrp;
    for (int t = blockIdx.x + egrp * gridDim.x; t < num_tiles; t += 2 * gridDim.x, lt += 2) {
      int mb, nb;
      tile_coords(t, p.num_m, p.num_n, mb, nb);
      const int acc = lt & 1;
      const int64_t row = (int64_t)mb * BM + quad * 32 + lane;
      const int n0 = nb * BN;
      epi_bar_id(1 + egrp);  // the previous tile's readers of sSB are done
      for (int j = et; j < BN; j += 128) sSB[j] = n0 + j < p.N ? __ldg(p.inv_b + n0 + j) : 0.f;
      const float sa = row < p.M ? p.alpha * __ldg(p.inv_a + row) : 0.f;
      epi_bar_id(1 + egrp);
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * 256;
      // 32-column chunks: lane = row while reading TMEM and forming D, then a warp-private 32 x 32
      // transpose in shared memory (16-byte groups XOR-swizzled by row: float4 (r, g) at
      // r * 32 + 4 (g ^ (r & 7)), conflict-free for the row-wise writes and the column-wise reads),
      // so that each 16-byte store instruction writes 4 whole 128-byte row segments instead of 32
      // rows' 16-byte pieces
      float* stile = stile0 + (warp - 2) * 32 * 32;
      const int64_t row0 = (int64_t)mb * BM + quad * 32;
      const int rsub = lane >> 3, g4 = lane & 7;
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        const int col0 = n0 + ch * 32;
        if (col0 >= p.N) break;  // warp-uniform
        uint32_t ri[32], rc[32];
        tmem_ld_32x32b_x32(t_row + ch * 32, ri);
        tmem_ld_32x32b_x32(t_row + 128 + ch * 32, rc);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float4 v;
          float* pv = &v.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = 4 * g + e;
            pv[e] = fmaf(p.alpha, __uint_as_float(rc[c]),
                         __fmul_rn(static_cast<float>(static_cast<int32_t>(ri[c])), __fmul_rn(sa, sSB[ch * 32 + c])));
          }
          *reinterpret_cast<float4*>(stile + lane * 32 + 4 * (g ^ (lane & 7))) = v;
        }
        __syncwarp();
        const int c = col0 + 4 * g4;
        const bool full4 = p.vec_ok && c + 4 <= p.N;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int r = 4 * it + rsub;
          const int64_t rw = row0 + r;
          float4 v = *reinterpret_cast<const float4*>(stile + r * 32 + 4 * (g4 ^ (r & 7)));
          if (rw >= p.M || c >= p.N) continue;
          float* out = p.D + rw * p.ldd + c;
          if (full4) {
            if (p.beta != 0.f) {
              const float4 o = *reinterpret_cast<const float4*>(out);
              v.x = fmaf(p.beta, o.x, v.x); v.y = fmaf(p.beta, o.y, v.y);
              v.z = fmaf(p.beta, o.z, v.z); v.w = fmaf(p.beta, o.w, v.w);
            }
            __stcs(reinterpret_cast<float4*>(out), v);
          } else {
            const float* pv = &v.x;
            for (int e = 0; e < 4; ++e)
              if (c + e < p.N) out[e] = p.beta != 0.f ? fmaf(p.beta, out[e], pv[e]) : pv[e];
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem_base);
  }
}

// K8w -- K8 with 128 x 256 tiles (UMMA N = 256): per k-block a stage carries A (16 KB) and B (32 KB),
// so the shared-memory operand traffic per MMA flop is 3/4 of K8's (at N = 128 the operand fetch,
// not the tensor pipe, bounds a one-CTA tile).  TMEM holds ONE tile: main int32 in columns 0..255,
// the bf16 correction in 256..511; the epilogue does not overlap the next tile's MMAs, the two
// epilogue groups split the tile's columns (0..127 | 128..255) so it drains twice as fast, and the
// producer keeps streaming the next tile's stages meanwhile.  Same arithmetic as K8.
namespace g8w {
constexpr int BM = 128, BN = 256, BK = 128, UK = 32;
constexpr int kStageBytes = BM * BK + BN * BK;  // 48 KB: int8 A | B, or bf16 [L_A | L_B] (hi or lo)
constexpr int kThreads = 64 + 256;
constexpr int kStages = 4;
constexpr int kStile = 8 * 32 * 32 * 4;
constexpr int kSmem = kStages * kStageBytes + kStile + BN * 4 + 256 + 1024;
static_assert(kSmem <= 232448, "K8w shared memory");
}  // namespace g8w

__global__ void __launch_bounds__(g8w::kThreads, 1)
    k8w_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                const __grid_constant__ CUtensorMap mapLAh, const __grid_constant__ CUtensorMap mapLAl,
                const __grid_constant__ CUtensorMap mapLBh, const __grid_constant__ CUtensorMap mapLBl, G8Params p) {
  using namespace g8w;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // offset from the __shared__ array: shared-space accesses, not generic
  float* stile0 = reinterpret_cast<float*>(smem + kStages * kStageBytes);  // 8 x 32 x 32 (XOR-swizzled)
  float* sSB0 = stile0 + kStile / 4;                                      // BN: 1/lambda_B of the tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSB0 + BN);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = p.num_m * p.num_n;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    tma_prefetch_desc(&mapLAh);
    tma_prefetch_desc(&mapLAl);
    tma_prefetch_desc(&mapLBh);
    tma_prefetch_desc(&mapLBl);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 256);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp == 0) {
    // -------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto next = [&]() {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kStageBytes);
      };
      auto advance = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      };
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, p.num_m, p.num_n, mb, nb);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          next();
          uint8_t* st = smem + stage * kStageBytes;
          tma_load_2d(st, &mapA, &full[stage], kb * BK, mb * BM);
          tma_load_2d(st + BM * BK, &mapB, &full[stage], kb * BK, nb * BN);
          advance();
        }
        next();  // [L_A hi | L_B hi]
        tma_load_2d(smem + stage * kStageBytes, &mapLAh, &full[stage], 0, mb * BM);
        tma_load_2d(smem + stage * kStageBytes + BM * BK, &mapLBh, &full[stage], 0, nb * BN);
        advance();
        next();  // [L_A lo | L_B lo]
        tma_load_2d(smem + stage * kStageBytes, &mapLAl, &full[stage], 0, mb * BM);
        tma_load_2d(smem + stage * kStageBytes + BM * BK, &mapLBl, &full[stage], 0, nb * BN);
        advance();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // -------------------------------------------------------------- UMMA issuer
    if (lane == 0) {
      constexpr uint32_t idi8 = make_idesc_i8(BM, BN);
      constexpr uint32_t idbf = make_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int lt = 0;
      const uint32_t d_main = tmem_base, d_corr = tmem_base + 256;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        mbar_wait(tempty, (lt & 1) ^ 1);  // the previous tile's epilogue drained the accumulators
        tc_fence_after();
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * kStageBytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma_i8(d_main, make_sw128_kmajor_desc(a_addr + k * UK), make_sw128_kmajor_desc(a_addr + BM * BK + k * UK),
                    idi8, (kb | k) != 0 ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        const int sx = stage;
        const uint32_t px = phase;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        const int sy = stage;
        const uint32_t py = phase;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        mbar_wait(&full[sx], px);
        mbar_wait(&full[sy], py);
        tc_fence_after();
        const uint32_t xa = smem_u32(smem + sx * kStageBytes), ya = smem_u32(smem + sy * kStageBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 4 x K16 = the 64 bf16 of one atom
          const uint32_t o = k * 32;
          umma_bf16(d_corr, make_sw128_kmajor_desc(xa + o), make_sw128_kmajor_desc(xa + BM * BK + o), idbf, k != 0);
          umma_bf16(d_corr, make_sw128_kmajor_desc(xa + o), make_sw128_kmajor_desc(ya + BM * BK + o), idbf, 1u);
          umma_bf16(d_corr, make_sw128_kmajor_desc(ya + o), make_sw128_kmajor_desc(xa + BM * BK + o), idbf, 1u);
        }
        umma_commit(&empty[sx]);
        umma_commit(&empty[sy]);
        umma_commit(tfull);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue
    // group e = columns [128 e, 128 e + 128) of every tile; warp quad = 32 rows
    const int egrp = (warp - 2) >> 2;
    const int et = threadIdx.x - 64 - 128 * egrp;
    const int quad = warp & 3;
    float* sSB = sSB0 + egrp * 128;
    float* stile = stile0 + (warp - 2) * 32 * 32;
    const int rsub = lane >> 3, g4 = lane & 7;
    int lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      int mb, nb;
      tile_coords(t, p.num_m, p.num_n, mb, nb);
      const int64_t row = (int64_t)mb * BM + quad * 32 + lane;
      const int n0 = nb * BN + egrp * 128;
      epi_bar_id(1 + egrp);  // the previous tile's readers of sSB are done
      for (int j = et; j < 128; j += 128) sSB[j] = n0 + j < p.N ? __ldg(p.inv_b + n0 + j) : 0.f;
      const float sa = row < p.M ? p.alpha * __ldg(p.inv_a + row) : 0.f;
      epi_bar_id(1 + egrp);
      mbar_wait(tfull, lt & 1);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quad * 32) << 16) + egrp * 128;
      const int64_t row0 = (int64_t)mb * BM + quad * 32;
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch) {
        const int col0 = n0 + ch * 32;
        if (col0 >= p.N) break;  // warp-uniform
        uint32_t ri[32], rc[32];
        tmem_ld_32x32b_x32(t_row + ch * 32, ri);
        tmem_ld_32x32b_x32(t_row + 256 + ch * 32, rc);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float4 v;
          float* pv = &v.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = 4 * g + e;
            pv[e] = fmaf(p.alpha, __uint_as_float(rc[c]),
                         __fmul_rn(static_cast<float>(static_cast<int32_t>(ri[c])), __fmul_rn(sa, sSB[ch * 32 + c])));
          }
          *reinterpret_cast<float4*>(stile + lane * 32 + 4 * (g ^ (lane & 7))) = v;
        }
        __syncwarp();
        const int c = col0 + 4 * g4;
        const bool full4 = p.vec_ok && c + 4 <= p.N;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int r = 4 * it + rsub;
          const int64_t rw = row0 + r;
          float4 v = *reinterpret_cast<const float4*>(stile + r * 32 + 4 * (g4 ^ (r & 7)));
          if (rw >= p.M || c >= p.N) continue;
          float* out = p.D + rw * p.ldd + c;
          if (full4) {
            if (p.beta != 0.f) {
              const float4 o = *reinterpret_cast<const float4*>(out);
              v.x = fmaf(p.beta, o.x, v.x); v.y = fmaf(p.beta, o.y, v.y);
              v.z = fmaf(p.beta, o.z, v.z); v.w = fmaf(p.beta, o.w, v.w);
            }
            __stcs(reinterpret_cast<float4*>(out), v);
          } else {
            const float* pv = &v.x;
            for (int e = 0; e < 4; ++e)
              if (c + e < p.N) out[e] = p.beta != 0.f ? fmaf(p.beta, out[e], pv[e]) : pv[e];
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(tempty);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem_base);
  }
}

// L (rows x R2 fp32) -> bf16 hi / lo halves, rows of 64 (zero-padded): the K8 correction operands.
// One thread per 8 columns of a row: two 16-byte loads (R2 % 4 == 0; else scalar), packed
// conversions (cvt.rn.bf16x2.f32), one 16-byte store per half.  Both factors (L_A, L_B) in one
// launch: thread index e < rows0 * 8 -> job 0, the rest -> job 1.
struct SplitJob {
  const float* L;
  int64_t rows;
  __nv_bfloat16* hi;
  __nv_bfloat16* lo;
};
__global__ void k_split_bf16(const SplitJob j0, const SplitJob j1, int R2) {
  ::lrqmm::pdl_enter();
  const int64_t n0 = j0.rows * 8, total = n0 + j1.rows * 8;  // 8-column groups
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const bool second = t >= n0;
    const SplitJob& J = second ? j1 : j0;
    const int64_t e = second ? t - n0 : t;
    const bool vec = (R2 & 3) == 0 && (reinterpret_cast<uintptr_t>(J.L) & 15) == 0;
    const int64_t r = e >> 3;
    const int c0 = (int)(e & 7) * 8;
    float x[8];
    const float* src = J.L + r * R2 + c0;
    if (vec) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float4 v = c0 + 4 * h < R2 ? __ldg(reinterpret_cast<const float4*>(src) + h) : make_float4(0.f, 0.f, 0.f, 0.f);
        x[4 * h] = v.x; x[4 * h + 1] = v.y; x[4 * h + 2] = v.z; x[4 * h + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = c0 + q < R2 ? src[q] : 0.f;
    }
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * q], x[2 * q + 1]);
      const float2 hf = __bfloat1622float2(h2);
      const __nv_bfloat162 l2 = __floats2bfloat162_rn(x[2 * q] - hf.x, x[2 * q + 1] - hf.y);
      hw[q] = *reinterpret_cast<const uint32_t*>(&h2);
      lw[q] = *reinterpret_cast<const uint32_t*>(&l2);
    }
    *reinterpret_cast<uint4*>(J.hi + e * 8) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(J.lo + e * 8) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
}

void launch_split_bf16(const float* LA, int64_t rowsA, const float* LB, int64_t rowsB, int R2, void* Ahi, void* Alo,
                       void* Bhi, void* Blo, cudaStream_t st) {
  const int64_t total = (rowsA > 0 ? rowsA : 0) * 8 + (rowsB > 0 ? rowsB : 0) * 8;
  if (total <= 0) return;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  const SplitJob j0{LA, rowsA > 0 ? rowsA : 0, reinterpret_cast<__nv_bfloat16*>(Ahi), reinterpret_cast<__nv_bfloat16*>(Alo)};
  const SplitJob j1{LB, rowsB > 0 ? rowsB : 0, reinterpret_cast<__nv_bfloat16*>(Bhi), reinterpret_cast<__nv_bfloat16*>(Blo)};
  launch_pdl(k_split_bf16, (int)g, 256, 0, st, j0, j1, R2);
  ++launch_counter();
}

int gemm_prepare_maps_tc(const GemmTcOperands& o, void* maps) {
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(maps);
  if (encode_codes_map(m + 0, reinterpret_cast<const int8_t*>(o.LAh), o.M, 128, g8::BM)) return 1;
  if (encode_codes_map(m + 1, reinterpret_cast<const int8_t*>(o.LAl), o.M, 128, g8::BM)) return 1;
  if (encode_codes_map(m + 2, reinterpret_cast<const int8_t*>(o.LBh), o.N, 128, g8::BN)) return 1;
  if (encode_codes_map(m + 3, reinterpret_cast<const int8_t*>(o.LBl), o.N, 128, g8::BN)) return 1;
  if (encode_codes_map(m + 4, reinterpret_cast<const int8_t*>(o.LBh), o.N, 128, g8w::BN)) return 1;  // K8w
  if (encode_codes_map(m + 5, reinterpret_cast<const int8_t*>(o.LBl), o.N, 128, g8w::BN)) return 1;
  return 0;
}

// ------------------------------------------------------------------------------------------
// K7 — the same GEMM + epilogue on CTA PAIRS (cluster of 2, tcgen05.mma.cta_group::2):
// a pair owns a 256 x 256 output tile; CTA r loads A rows [256 mb + 128 r, +128) and B^T rows
// [256 nb + 128 r, +128) (32 KB per 128-deep stage instead of 48 KB), the leader (r = 0) issues
// one M = 256, N = 256, K = 32 MMA per step that reads both CTAs' shared memory, and each CTA's
// TMEM receives its own 128 rows x 256 columns, so the epilogue is the one of K6.  Per SM this
// halves the MMA instructions, commits and B bytes per unit of tensor work.
//   full[s]  (leader)   : both CTAs' TMA bytes (expect_tx set by the leader's producer)
//   empty[s] (each CTA) : multicast commit from the leader's MMA
//   tfull[a] (each CTA) : multicast commit at the end of a tile
//   tempty[a] (leader)  : 128 epilogue threads of EACH CTA (peer arrives remotely)
namespace g7 {
constexpr int BM = 128;  // rows per CTA (256 per pair)
constexpr int BN = 256;  // output columns per pair tile
constexpr int BNH = 128; // B^T rows loaded per CTA
constexpr int BK = 128;
constexpr int UK = 32;
constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;
constexpr int kABytes = BM * BK;
constexpr int kBBytes = BNH * BK;
constexpr int kStageBytes = kABytes + kBBytes;  // 32 KB per CTA
constexpr int kTR = 4;  // tile-index ring depth (dynamic scheduler -> MMA, epilogues, peer producer)
#ifndef LRQMM_L2HINT7
#define LRQMM_L2HINT7 1  // A panels evict_last (reused by the next waves of the raster group)
#endif
#ifndef LRQMM_PAIR_RELEASE
#define LRQMM_PAIR_RELEASE 0  // one commit per two stages (measured slower: less buffering)
#endif
#ifndef LRQMM_GROUPM7
#define LRQMM_GROUPM7 8
#endif
constexpr int kGroupM = LRQMM_GROUPM7;  // pair-tile rows (256 A rows each) per raster group
__host__ __device__ constexpr int extra_bytes(int r2) { return BN * r2 * 4 + BN * 4 + 256 + 1024; }
__host__ __device__ constexpr int stages_for(int r2) {  // even: stages are released in pairs
  return ((232448 - extra_bytes(r2)) / kStageBytes > 6 ? 6 : (232448 - extra_bytes(r2)) / kStageBytes) & ~1;
}
__host__ __device__ constexpr int smem_bytes(int r2) { return stages_for(r2) * kStageBytes + extra_bytes(r2); }
}  // namespace g7

LRQMM_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
LRQMM_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same offset in CTA `rank` of the cluster
LRQMM_DEV uint32_t mapa_cta(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
LRQMM_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2SM TMA: data lands in this CTA's smem, complete_tx goes to the barrier at `mbar_cluster`
LRQMM_DEV void tma_load_2d_2sm(void* smem_dst, const void* desc, uint32_t mbar_cluster, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(mbar_cluster), "r"(x), "r"(y)
      : "memory");
}
LRQMM_DEV void tma_load_2d_2sm_hint(void* smem_dst, const void* desc, uint32_t mbar_cluster, int x, int y,
                                    uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(mbar_cluster), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
LRQMM_DEV void umma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// warp-collective forms: the whole (converged) warp executes them, one elected lane issues, so the
// operands stay warp-uniform and no per-instruction elect loop is generated
LRQMM_DEV void umma_i8_2sm_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
LRQMM_DEV void umma_commit_2sm_mc_warp(uint32_t bar_addr) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\t.reg .pred e;\n\tmov.b16 m, 3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          bar_addr)
      : "memory");
}
LRQMM_DEV void umma_commit_2sm_mc(uint64_t* bar) {  // arrive on `bar` in both CTAs of the pair
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

template <int kR2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(g7::kThreads, 1)
    k7_gemm_i8_2sm(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, G6Params p) {
  using namespace g7;
  constexpr int STAGES = stages_for(kR2);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // offset from the __shared__ array: shared-space accesses, not generic
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * kABytes;
  float* sLB = reinterpret_cast<float*>(smem + STAGES * kStageBytes);  // BN x kR2
  float* sSB = sLB + BN * kR2;                                           // BN : 1/lambda_b
  const uint32_t sLBa = smem_u32(sLB), sSBa = smem_u32(sSB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSB + BN);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint64_t* tfull_t = bars + 2 * STAGES + 4;  // kTR: tile index published (both CTAs)
  uint64_t* tempty_t = tfull_t + kTR;         // kTR: tile index consumed (leader, 4 arrivals)
  int* tile_ring = reinterpret_cast<int*>(tempty_t + kTR);  // kTR tile indices (both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + kTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int num_tiles = p.num_m * p.num_n;  // pair tiles (256 x 256)
  const bool pair_rel = LRQMM_PAIR_RELEASE && (p.num_kb & 1) == 0;  // a tile always starts on an even stage

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiThreads);
    }
    for (int q = 0; q < kTR; ++q) {
      mbar_init(&tfull_t[q], 1);
      mbar_init(&tempty_t[q], 4);  // leader MMA, leader epilogue, peer producer, peer epilogue
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = mapa_cta(smem_u32(full), 0);  // leader's full[0]
      const uint64_t polA = l2_policy(p.polA), polB = l2_policy(p.polB);
      const uint32_t tfull_peer = mapa_cta(smem_u32(tfull_t), 1);
      const uint32_t ring_peer = mapa_cta(smem_u32(tile_ring), 1);
      const uint32_t tempty_lead = mapa_cta(smem_u32(tempty_t), 0);
      for (int lt = 0;; ++lt) {
        const int q = lt % kTR;
        const uint32_t qph = (lt / kTR) & 1;
        int t;
        if (leader) {
          // dynamic schedule: in-flight tiles always form one contiguous window of indices, so
          // the raster groups' L2 working set stays bounded however the pairs drift
          mbar_wait(&tempty_t[q], qph ^ 1);
          t = atomicAdd(p.sched, 1);
          tile_ring[q] = t;
          asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(ring_peer + 4 * q), "r"(t) : "memory");
          mbar_arrive(&tfull_t[q]);
          mbar_arrive_remote(tfull_peer + 8 * q);
        } else {
          mbar_wait(&tfull_t[q], qph);
          t = tile_ring[q];
          mbar_arrive_remote(tempty_lead + 8 * q);
        }
        if (t >= num_tiles) break;
        int mb, nb;
        tile_coords_rt(t, p.group_m, p.num_m, p.num_n, mb, nb);
        const int arow = mb * (2 * BM) + (int)rank * BM;
        const int brow = nb * BN + (int)rank * BNH;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          // with an even k-block count, stages are released in pairs (one MMA commit per two)
          if (!pair_rel) mbar_wait(&empty[stage], phase ^ 1);
          else if ((stage & 1) == 0) mbar_wait(&empty[stage >> 1], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStageBytes);
          const uint32_t fb = full0 + stage * 8;
          tma_load_2d_2sm_hint(sA + stage * kABytes, &mapA, fb, kb * BK, arow, polA);
          tma_load_2d_2sm_hint(sB + stage * kBBytes, &mapB, fb, kb * BK, brow, polB);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer (leader only)
    // The whole warp runs the loop (warp-uniform operands); one elected lane issues each op.
    if (leader) {
      constexpr uint32_t idesc = make_idesc_i8(2 * BM, BN);
      // descriptors differ only in the start-address field (addr >> 4, no carry below 256 KB)
      const uint64_t dA0 = make_sw128_kmajor_desc(smem_u32(sA));
      const uint64_t dB0 = make_sw128_kmajor_desc(smem_u32(sB));
      const uint32_t empty_a = smem_u32(empty), tfull_a = smem_u32(tfull);
      int stage = 0;
      uint32_t phase = 0;
      for (int lt = 0;; ++lt) {
        const int q = lt % kTR;
        mbar_wait(&tfull_t[q], (lt / kTR) & 1);
        const int t = tile_ring[q];
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_t[q]);
        if (t >= num_tiles) break;
        const int acc = lt & 1;
        const uint32_t acc_phase = (lt >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = dA0 + (uint64_t)((stage * kABytes) >> 4);
          const uint64_t bd = dB0 + (uint64_t)((stage * kBBytes) >> 4);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma_i8_2sm_warp(d_tmem, ad + (uint64_t)((k * UK) >> 4), bd + (uint64_t)((k * UK) >> 4), idesc,
                             (kb | k) != 0 ? 1u : 0u);
          // frees this stage (or the pair (stage - 1, stage)) in both CTAs
          if (!pair_rel) umma_commit_2sm_mc_warp(empty_a + 8 * stage);
          else if (stage & 1) umma_commit_2sm_mc_warp(empty_a + 8 * (stage >> 1));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc_warp(tfull_a + 8 * acc);  // both halves of the accumulator ready
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue (both CTAs)
    const int et = threadIdx.x - 64;  // 0..127
    const int quad = warp & 3;
    const uint32_t tempty0 = mapa_cta(smem_u32(tempty), 0);
    const uint32_t tempty_t0 = mapa_cta(smem_u32(tempty_t), 0);
    for (int lt = 0;; ++lt) {
      const int q = lt % kTR;
      mbar_wait(&tfull_t[q], (lt / kTR) & 1);
      const int t = tile_ring[q];
      epi_bar<g7::kEpiThreads>();  // every epilogue thread has read the index
      if (et == 0) mbar_arrive_remote(tempty_t0 + 8 * q);
      if (t >= num_tiles) break;
      int mb, nb;
      tile_coords_rt(t, p.group_m, p.num_m, p.num_n, mb, nb);
      const int acc = lt & 1;
      const uint32_t acc_phase = (lt >> 1) & 1;
      const int64_t row = (int64_t)mb * (2 * BM) + (int64_t)rank * BM + quad * 32 + lane;
      const int n0 = nb * BN;
      float sa = 0.f;
      float la[kR2 > 0 ? kR2 : 1];
#pragma unroll
      for (int l = 0; l < (kR2 > 0 ? kR2 : 1); ++l) la[l] = 0.f;
      if (p.epi == 1) {
        epi_bar<g7::kEpiThreads>();
        for (int j = et; j < BN; j += kEpiThreads) {
          const int col = n0 + j;
          const float v = col < p.N ? __ldg(p.inv_b + col) : 0.f;
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(sSBa + 4 * j), "f"(v) : "memory");
        }
        if constexpr (kR2 > 0) {
          const float4* src = reinterpret_cast<const float4*>(p.LB + (int64_t)n0 * kR2);
          const int total4 = BN * kR2 / 4;
          const int valid4 = (int)((p.N - n0 < BN ? p.N - n0 : (int64_t)BN) * kR2 / 4);
          for (int e = et; e < total4; e += kEpiThreads)
            sts128(sLBa + 16 * e, e < valid4 ? __ldg(src + e) : make_float4(0.f, 0.f, 0.f, 0.f));
        }
        if (row < p.M) {
          sa = p.alpha * __ldg(p.inv_a + row);
          if constexpr (kR2 > 0) {
            const float4* lr = reinterpret_cast<const float4*>(p.LA + row * kR2);
#pragma unroll
            for (int l = 0; l < kR2; l += 4) {
              const float4 v = __ldg(lr + (l >> 2));
              la[l] = p.alpha * v.x; la[l + 1] = p.alpha * v.y; la[l + 2] = p.alpha * v.z; la[l + 3] = p.alpha * v.w;
            }
          }
        }
        epi_bar<g7::kEpiThreads>();
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      uint32_t ra[8], rb[8];
      tmem_ld_32x32b_x8(t_row, ra);
#pragma unroll 1
      for (int g = 0; g < BN / 8; g += 2) {
        tmem_ld_wait();
        tmem_ld_32x32b_x8(t_row + (g + 1) * 8, rb);
        epilogue_group<kR2>(p, ra, row, n0 + g * 8, g * 8, sa, la, sLBa, sSBa);
        tmem_ld_wait();
        if (g + 2 < BN / 8) tmem_ld_32x32b_x8(t_row + (g + 2) * 8, ra);
        epilogue_group<kR2>(p, rb, row, n0 + (g + 1) * 8, (g + 1) * 8, sa, la, sLBa, sSBa);
      }
      tc_fence_before();
      mbar_arrive_remote(tempty0 + acc * 8);  // the leader's tempty[acc] (local arrive on the leader)
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512) : "memory");
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

// generic 2D tiled map: dims {inner, outer}, row stride in bytes, box {box_inner, box_outer}
int encode_map_2d_sw(void* map, int dtype, const void* base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                     uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return 1;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 32   ? CU_TENSOR_MAP_SWIZZLE_32B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  const CUtensorMapDataType dt = dtype == 1   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : dtype == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                              : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(map), dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 2;
}

int& gemm_variant() {  // 0 auto, 1 force one-CTA K6, 2 force CTA-pair K7, 3 force K8 (test hook)
  static int v = [] {
    const char* e = getenv("LRQMM_GEMM_VARIANT");  // A/B timing of the kernel choice
    return e ? atoi(e) : 0;
  }();
  return v;
}

static bool use_2sm(int64_t M, int64_t N, const int* sched) {
  if (!sched || gemm_variant() == 1 || gemm_variant() == 3) return false;
  if (gemm_variant() == 2) return true;
  // CTA pairs need enough 256 x 256 tiles to fill 74 pairs for several waves: below ~512 of them
  // (c2, 4096^2: 256) the one-CTA kernel's 2x more, smaller tiles balance better (measured 87 vs
  // 96 us at 4096^3 fused, tools/gemm_variants.py)
  return M >= 512 && N >= 512 && ((M + 255) / 256) * ((N + 255) / 256) >= 512;
}

// map slots: [0] K6 (A box rows 128, B 256), [1] K7 (128 / 128), [2] K6 B box 128, [3] K6 B box 64
int gemm_prepare_maps(const GemmArgs& g, void* mapA, void* mapB) {
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(mapA);
  CUtensorMap* n = reinterpret_cast<CUtensorMap*>(mapB);
  if (encode_codes_map(m, g.A, g.M, g.Kp, g6::BM)) return 1;
  if (encode_codes_map(n, g.B, g.N, g.Kp, 256)) return 1;
  if (encode_codes_map(m + 1, g.A, g.M, g.Kp, g7::BM)) return 1;
  if (encode_codes_map(n + 1, g.B, g.N, g.Kp, g7::BNH)) return 1;
  if (encode_codes_map(n + 2, g.B, g.N, g.Kp, 128)) return 1;
  if (encode_codes_map(n + 3, g.B, g.N, g.Kp, 64)) return 1;
  return 0;
}

template <int kR2, int BN>
static void launch_t(G6Params p, const CUtensorMap* mA, const CUtensorMap* mB, int nsm, cudaStream_t st) {
  constexpr int kSmem = g6::smem_bytes(kR2, BN);
  static_assert(kSmem <= 232448, "shared memory budget");
  static_assert(g6::stages_for(kR2, BN) >= 3, "stages");
  static std::atomic<unsigned> attr{0};
  ensure_smem(k6_gemm_i8<kR2, BN>, kSmem, attr);
  p.num_n = (int)((p.N + BN - 1) / BN);
  const int tiles = p.num_m * p.num_n;
  const int grid = tiles < nsm ? tiles : nsm;
  k6_gemm_i8<kR2, BN><<<grid, g6::threads_for(kR2, BN), kSmem, st>>>(*mA, *mB, p); ++launch_counter();
}

template <int kR2>
static void launch_k6(const G6Params& p, const CUtensorMap* mA, const CUtensorMap* mB, int nsm, cudaStream_t st) {
  // narrowest tile that covers N (no wasted MMA / epilogue columns for N = 64, 128)
  if (p.N <= 64) launch_t<kR2, 64>(p, mA, mB + 3, nsm, st);
  else if (p.N <= 128) launch_t<kR2, 128>(p, mA, mB + 2, nsm, st);
  else launch_t<kR2, 256>(p, mA, mB, nsm, st);
}

template <int kR2>
static void launch_t7(G6Params p, const CUtensorMap* mA, const CUtensorMap* mB, int nsm, cudaStream_t st) {
  constexpr int kSmem = g7::smem_bytes(kR2);
  static_assert(kSmem <= 232448, "shared memory budget");
  static_assert(g7::stages_for(kR2) >= 3, "stages");
  static std::atomic<unsigned> attr{0};
  ensure_smem(k7_gemm_i8_2sm<kR2>, kSmem, attr);
  p.num_m = (int)((p.M + 2 * g7::BM - 1) / (2 * g7::BM));
  p.num_n = (int)((p.N + g7::BN - 1) / g7::BN);
  const int tiles = p.num_m * p.num_n;
  int pairs = nsm / 2;
  if (tiles < pairs) pairs = tiles;
  // raster group / L2 policies (defaults measured best; LRQMM_G7_{GROUP,POLA,POLB} override them
  // for experiments)
  static int group = -1, pola = 2, polb = 1;  // A evict_last, B evict_first (c3: -4.6% GEMM time)
  if (group < 0) {
    const char* e = getenv("LRQMM_G7_GROUP");
    group = e ? atoi(e) : g7::kGroupM;
    if (group < 1) group = 1;
    if ((e = getenv("LRQMM_G7_POLA"))) pola = atoi(e);
    if ((e = getenv("LRQMM_G7_POLB"))) polb = atoi(e);
  }
  p.group_m = group;
  p.polA = pola;
  p.polB = polb;
  cudaMemsetAsync(p.sched, 0, sizeof(int), st);
  k7_gemm_i8_2sm<kR2><<<2 * pairs, g7::kThreads, kSmem, st>>>(*mA, *mB, p); ++launch_counter();
}

// the tensor-core correction kernel K8 runs the fused LRQMM epilogue (R2 > 0) wherever the FFMA
// correction would not hide behind a long main loop: every shape the one-CTA K6 would take, and
// CTA-pair shapes with K <= 2048 (c4: layer2-3 1x1 convolutions 1.02 -> 0.69 ms with K8 instead
// of K7).  Tests force a variant; LRQMM_NO_TC_CORR turns K8 off.
bool gemm_uses_tc(int64_t M, int64_t N, int Kp, int R2, const int* sched) {
  static const bool off = getenv("LRQMM_NO_TC_CORR") != nullptr;
  if (R2 <= 0 || off || gemm_variant() == 1 || gemm_variant() == 2) return false;
  return gemm_variant() == 3 || !use_2sm(M, N, sched) || Kp <= 2048;
}

static void launch_k8(const GemmArgs& g, const CUtensorMap* mA, const CUtensorMap* mB, const CUtensorMap* tc,
                      int nsm, cudaStream_t st) {
  static std::atomic<unsigned> attr{0};
  ensure_smem(k8_gemm_tc, g8::kSmem, attr);
  G8Params p{};
  p.M = g.M;
  p.N = g.N;
  p.num_kb = (g.Kp + g8::BK - 1) / g8::BK;
  p.num_m = (int)((g.M + g8::BM - 1) / g8::BM);
  p.num_n = (int)((g.N + g8::BN - 1) / g8::BN);
  p.inv_a = g.inv_a;
  p.inv_b = g.inv_b;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.D = g.D;
  p.ldd = g.ldd;
  p.vec_ok = ((reinterpret_cast<uintptr_t>(g.D) & 15) == 0) && (g.ldd % 4 == 0);
  const int tiles = p.num_m * p.num_n;
  const int grid = tiles < nsm ? tiles : nsm;
  k8_gemm_tc<<<grid, g8::kThreads, g8::kSmem, st>>>(*mA, *mB, tc[0], tc[1], tc[2], tc[3], p);
  ++launch_counter();
}

// K8w: mB256 = the B codes map with 256-row boxes, tc[4] / tc[5] = L_B hi / lo with 256-row boxes
static void launch_k8w(const GemmArgs& g, const CUtensorMap* mA, const CUtensorMap* mB256, const CUtensorMap* tc,
                       int nsm, cudaStream_t st) {
  static std::atomic<unsigned> attr{0};
  ensure_smem(k8w_gemm_tc, g8w::kSmem, attr);
  G8Params p{};
  p.M = g.M;
  p.N = g.N;
  p.num_kb = (g.Kp + g8w::BK - 1) / g8w::BK;
  p.num_m = (int)((g.M + g8w::BM - 1) / g8w::BM);
  p.num_n = (int)((g.N + g8w::BN - 1) / g8w::BN);
  p.inv_a = g.inv_a;
  p.inv_b = g.inv_b;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.D = g.D;
  p.ldd = g.ldd;
  p.vec_ok = ((reinterpret_cast<uintptr_t>(g.D) & 15) == 0) && (g.ldd % 4 == 0);
  const int tiles = p.num_m * p.num_n;
  const int grid = tiles < nsm ? tiles : nsm;
  k8w_gemm_tc<<<grid, g8w::kThreads, g8w::kSmem, st>>>(*mA, *mB256, tc[0], tc[1], tc[4], tc[5], p);
  ++launch_counter();
}

int launch_gemm(const GemmArgs& g, const void* mapA, const void* mapB, cudaStream_t st) {
  if (g.M == 0 || g.N == 0) return 0;
  G6Params p;
  p.M = g.M;
  p.N = g.N;
  p.num_kb = (g.Kp + g6::BK - 1) / g6::BK;  // the last box is zero-filled past Kp
  p.num_m = (int)((g.M + g6::BM - 1) / g6::BM);
  p.num_n = (int)((g.N + g6::BN - 1) / g6::BN);
  p.epi = g.epi;
  p.inv_a = g.inv_a;
  p.inv_b = g.inv_b;
  p.LA = g.LA;
  p.LB = g.LB;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.D = g.D;
  p.Cint = g.Cint;
  p.ldd = g.ldd;
  p.sched = g.sched;
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
  if (g.tc_maps && gemm_uses_tc(g.M, g.N, g.Kp, r2, g.sched)) {
    // K8w (128 x 256 tiles) for N >= 256 with a main loop long enough to carry its non-overlapped
    // epilogue (c2, 4096^3: 82 -> 72 us); LRQMM_K8W=0 keeps K8, =2 uses K8w at any K
    static const int wide = [] {
      const char* e = getenv("LRQMM_K8W");
      return e ? atoi(e) : 1;
    }();
    // ... and with at least one full wave of 128 x 256 tiles (a row-sharded slice with few rows keeps
    // K8's twice as many tiles busy on more SMs)
    const int64_t wtiles = ((g.M + 127) / 128) * ((g.N + 255) / 256);
    if (wide && g.N >= 256 && (wide == 2 || (g.Kp >= 2048 && wtiles >= nsm)))
      launch_k8w(g, mA, mB, reinterpret_cast<const CUtensorMap*>(g.tc_maps), nsm, st);  // B box 256 rows
    else
      launch_k8(g, mA, mB + 2, reinterpret_cast<const CUtensorMap*>(g.tc_maps), nsm, st);  // B box 128 rows
    return 0;
  }
  if (use_2sm(g.M, g.N, g.sched)) {
    switch (r2) {
      case 0: launch_t7<0>(p, mA + 1, mB + 1, nsm, st); break;
      case 8: launch_t7<8>(p, mA + 1, mB + 1, nsm, st); break;
      case 16: launch_t7<16>(p, mA + 1, mB + 1, nsm, st); break;
      case 24: launch_t7<24>(p, mA + 1, mB + 1, nsm, st); break;
      case 32: launch_t7<32>(p, mA + 1, mB + 1, nsm, st); break;
      case 40: launch_t7<40>(p, mA + 1, mB + 1, nsm, st); break;
      case 48: launch_t7<48>(p, mA + 1, mB + 1, nsm, st); break;
      case 56: launch_t7<56>(p, mA + 1, mB + 1, nsm, st); break;
      case 64: launch_t7<64>(p, mA + 1, mB + 1, nsm, st); break;
      default: return 1;  // correction width not instantiated (the API validates 2r <= 64)
    }
    return 0;
  }
  (void)grid;
  switch (r2) {
    case 0: launch_k6<0>(p, mA, mB, nsm, st); break;
    case 8: launch_k6<8>(p, mA, mB, nsm, st); break;
    case 16: launch_k6<16>(p, mA, mB, nsm, st); break;
    case 24: launch_k6<24>(p, mA, mB, nsm, st); break;
    case 32: launch_k6<32>(p, mA, mB, nsm, st); break;
    case 40: launch_k6<40>(p, mA, mB, nsm, st); break;
    case 48: launch_k6<48>(p, mA, mB, nsm, st); break;
    case 56: launch_k6<56>(p, mA, mB, nsm, st); break;
    case 64: launch_k6<64>(p, mA, mB, nsm, st); break;
    default: return 1;
  }
  return 0;
}

}  // namespace lrqmm
