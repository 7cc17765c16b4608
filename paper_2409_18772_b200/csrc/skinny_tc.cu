// K2/K3 on the 5th-gen tensor cores: the RSVD passes over the quantization
// residual (Algorithm 1 sampling / power iteration / projection, PAPER.md:124-140,
// reading #11) and the cross products of Algorithm 2, computed as
// tcgen05.mma kind::tf32 with a 3-term split (x = hi + lo, hi = tf32(x)):
//     U P ~= U_hi P_hi + U_hi P_lo + U_lo P_hi                 (fp32-grade)
// U is the residual fraction u = lambda x - code written by K1 (R = diag(1/lambda) U) in Q15
// fixed point, so every pass streams 2 B per element from HBM — this kernel's roofline — and
// the producer warps only widen u to fp32 and split it into tf32 hi/lo operand tiles (exact:
// u16 / 2^15 has <= 16 significant bits, hi keeps 11, lo the rest).
//
//   ROW mode  OUT1[i,:] = (1/lambda_i) sum_j U[i,j] P1[j,:]      (S1: Y = R Omega, S3: W = R Q1)
//             OUT2[i,:] = (1/lambda_i) sum_j C[i,j] P2[j,:]      (dual: A~ Q1_other, codes exact in tf32)
//             A operand = U tile, K-major SW128; B = P tile, MN-major SW128_BASE32B.
//   COL mode  OUT[j,:]  = sum_i U[i,j] (P[i,:] / lambda_i)       (S2: Z = R^T Q0)
//             A operand = U tile, MN-major SW128_BASE32B (U's natural layout); B as above.
//
// Persistent, warp-specialised (448 threads, one CTA per SM):
//   warp 13    : TMA issuer, streams raw tiles (U 8 KB, P, codes, 1/lambda) through a smem ring
//   warps 0-7  : producers: raw U -> tf32 hi/lo operand tiles (+ codes -> fp32) (2-3 stages)
//   warp 12    : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 8-11 : epilogue: TMEM (double-buffered accumulators) -> split-K partials
// Work unit = (128-row/col block, reduction split); partials are summed in a fixed order
// by the consumer (deterministic, no float atomics).
#include <cuda.h>

#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

namespace tcp {
constexpr int BM = 128;  // output rows (ROW) / output cols (COL) per unit
constexpr int BK = 32;   // reduction elements per k-block
#ifndef LRQMM_PROD
#define LRQMM_PROD 256
#endif
constexpr int kProd = LRQMM_PROD;  // producer threads
constexpr int kProdWarps = kProd / 32;
constexpr int kMmaWarp = kProdWarps + 4;
constexpr int kTmaWarp = kProdWarps + 5;
constexpr int kThreads = (kProdWarps + 6) * 32;
constexpr int kPer = BM * BK / 4 / kProd;        // 4-element groups of U per producer thread per k-block
#ifndef LRQMM_OPST
#define LRQMM_OPST 2
#endif
constexpr int OPST_MAX = LRQMM_OPST;
constexpr int kATile = BM * BK * 4;    // 16 KB operand tile (hi or lo)
constexpr int kRawTile = BM * BK * 2;  // 8 KB raw U tile (Q15)
constexpr int kRawCodes = BM * BK;     // 4 KB raw code tile (dual)
template <int kMode, int NA, bool kDual>
struct Cfg {
  static constexpr int WN = 32 * NA;
  static constexpr int kBTile = BK * WN * 4;  // operand B tile (hi or lo)
  static constexpr int kStage = (kDual ? 3 : 2) * kATile + (kDual ? 4 : 2) * kBTile;
  // raw slot: U tile | P1 tile [BK][WN] | P2 tile | codes tile (dual) | 1/lambda[BK] (COL)
  static constexpr int kRawP = BK * WN * 4;
  static constexpr int kOffP2 = kRawTile + kRawP;
  static constexpr int kOffCodes = kRawTile + (kDual ? 2 : 1) * kRawP;
  static constexpr int kOffInv = kOffCodes + (kDual ? kRawCodes : 0);
  static constexpr int kRawBytes = kOffInv + (kMode == 1 ? BK * 4 : 0);
  static constexpr int kRawSlot = (kRawBytes + 1023) / 1024 * 1024;
  static constexpr int kBudget = 220 * 1024;
  static constexpr bool fits(int op, int raw) { return op * kStage + raw * kRawSlot <= kBudget; }
  static constexpr int OPST = fits(OPST_MAX, 3) ? OPST_MAX : (fits(2, 2) ? 2 : 1);
  static constexpr int kRawSt = fits(OPST, 4) ? 4 : (fits(OPST, 3) ? 3 : 2);
  static constexpr int kSmem = kRawSt * kRawSlot + OPST * kStage + 256 + 1024;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static constexpr int kAccCols = (kDual ? 2 : 1) * WN;  // per accumulator buffer
  static constexpr uint32_t kTmemCols =
      2 * kAccCols <= 32 ? 32 : (2 * kAccCols <= 64 ? 64 : (2 * kAccCols <= 128 ? 128 : 256));
};
}  // namespace tcp

struct TcArgs {
  int64_t rows;
  int K;
  const float* inv_lam;
  int W;
  float* out1;  // partial base: split s at out + s * (nout * W)
  float* out2;
  int64_t nout;   // rows (ROW) or K (COL)
  int64_t chunk;  // reduction elements per split (multiple of BK)
  int nblk, nsplit;
};

struct TcMaps {
  CUtensorMap u, p1, p2, codes, inv;
};

LRQMM_DEV float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// tf32 operands: K-major uses SWIZZLE_128B (type 2); MN-major must use
// SWIZZLE_128B_BASE32B (type 1: 32 MN x 4 K atoms of 512 B, 32-byte chunks XOR row),
// the only MN-major layout the tensor core accepts for 32-bit operands (probed on B200).
LRQMM_DEV uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t type) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)type << 61;
  return d;
}
// kind::tf32, D f32, M = 128, N = n; a_mn / b_mn: operand is MN-major
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t n, uint32_t a_mn, uint32_t b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn << 15) | (b_mn << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
LRQMM_DEV void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
LRQMM_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
LRQMM_DEV uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}
// two Q15 residual fractions (packed int16) -> fp32 (exact)
LRQMM_DEV float2 u_unfix(uint32_t w) {
  constexpr float s = 1.f / kUScale;
  return make_float2((float)(int16_t)(w & 0xffffu) * s, (float)(int16_t)(w >> 16) * s);
}
LRQMM_DEV uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// byte offset of element (mn, k) in an MN-major SW128_BASE32B tile with nA 32-wide MN atoms
// (LBO = 512 B between MN atoms, SBO = nA * 512 B between 4-deep K groups)
LRQMM_DEV uint32_t off_mn(int mn, int k, int nA) {
  const int row = k & 3;
  return (uint32_t)((k >> 2) * (nA * 512) + (mn >> 5) * 512 + row * 128 + ((((mn & 31) >> 3) ^ row) << 5) +
                    ((mn & 7) << 2));
}
// byte offset of element (mn, k) in a K-major SW128 tile (rows of 32 fp32)
LRQMM_DEV uint32_t off_k(int mn, int k) {
  const int row = mn & 7;
  const int chunk = k >> 2;
  return (uint32_t)((mn >> 3) * 1024 + row * 128 + ((chunk ^ row) << 4) + ((k & 3) << 2));
}

template <int kMode, int NA, bool kDual>
__global__ void __launch_bounds__(tcp::kThreads, 1) k_tc_proj(const __grid_constant__ TcMaps maps, TcArgs a) {
  using namespace tcp;
  using C = Cfg<kMode, NA, kDual>;
  constexpr int WN = C::WN;
  constexpr int kBTile = C::kBTile;
  constexpr int kStage = C::kStage;
  constexpr int RST = C::kRawSt;
  constexpr int OPST = C::OPST;
  constexpr int kRawSlot = C::kRawSlot;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRaw = smem;                  // RST raw slots (TMA)
  uint8_t* sOp = smem + RST * kRawSlot;  // OPST x kStage operand tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOp + OPST * kStage);
  uint64_t* rfull = bars;            // RST
  uint64_t* rempty = bars + RST;     // RST
  uint64_t* ofull = bars + 2 * RST;  // OPST
  uint64_t* oempty = ofull + OPST;   // OPST
  uint64_t* tfull = oempty + OPST;   // 2
  uint64_t* tempty = tfull + 2;      // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t r_len = kMode == 0 ? (int64_t)a.K : a.rows;
  const int nunits = a.nblk * a.nsplit;

  if (tid == 0) {
    for (int s = 0; s < RST; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], kProdWarps);  // one elected arrival per producer warp
    }
    for (int s = 0; s < OPST; ++s) {
      mbar_init(&ofull[s], kProdWarps);
      mbar_init(&oempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto unit_range = [&](int u, int& blk, int& split, int64_t& r0, int& nkb) {
    blk = u % a.nblk;
    split = u / a.nblk;
    r0 = (int64_t)split * a.chunk;
    const int64_t r1 = r0 + a.chunk < r_len ? r0 + a.chunk : r_len;
    nkb = (int)((r1 - r0 + BK - 1) / BK);
  };

  if (warp == kTmaWarp) {
    // ------------------------------------------------------ TMA: raw tiles
    if (lane == 0) {
      tma_prefetch_desc(&maps.u);
      tma_prefetch_desc(&maps.p1);
      if (kDual) {
        tma_prefetch_desc(&maps.p2);
        tma_prefetch_desc(&maps.codes);
      }
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        int blk, split, nkb;
        int64_t r0;
        unit_range(u, blk, split, r0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % RST;
          mbar_wait(&rempty[s], ((it / RST) & 1) ^ 1);
          uint8_t* slot = sRaw + s * kRawSlot;
          mbar_arrive_expect_tx(&rfull[s], C::kRawBytes);
          const int k0 = (int)(r0 + (int64_t)kb * BK);
          if (kMode == 0) tma_load_2d(slot, &maps.u, &rfull[s], k0, blk * BM);
          else tma_load_2d(slot, &maps.u, &rfull[s], blk * BM, k0);
          tma_load_2d(slot + kRawTile, &maps.p1, &rfull[s], 0, k0);
          if (kDual) {
            tma_load_2d(slot + C::kOffP2, &maps.p2, &rfull[s], 0, k0);
            tma_load_2d(slot + C::kOffCodes, &maps.codes, &rfull[s], k0, blk * BM);
          }
          if (kMode == 1) tma_load_1d(slot + C::kOffInv, &maps.inv, &rfull[s], k0);
        }
      }
    }
    __syncwarp();
  } else if (warp < kProdWarps) {
    // ------------------------------------------------------------ producers
    constexpr int kPB4 = BK * WN / 4;
    constexpr int kPBper = (kPB4 + kProd - 1) / kProd;
    int it = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      int blk, split, nkb;
      int64_t r0;
      unit_range(u, blk, split, r0, nkb);
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int rs = it % RST;
        const int os = it % OPST;
        // raw slot -> registers, then release the slot
        mbar_wait(&rfull[rs], (it / RST) & 1);
        const uint32_t raw = smem_u32(sRaw) + rs * kRawSlot;
        float4 xv[kPer];
        uint32_t cw[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const int f = tid + kProd * q;
          // raw U: ROW [BM rows][BK] int16 (64 B rows), COL [BK rows][BM] int16 (256 B rows)
          const uint32_t ro =
              kMode == 0 ? (uint32_t)((f >> 3) * 64 + (f & 7) * 8) : (uint32_t)((f >> 5) * 256 + (f & 31) * 8);
          const uint2 w = lds64(raw + ro);
          const float2 u01 = u_unfix(w.x), u23 = u_unfix(w.y);
          xv[q] = make_float4(u01.x, u01.y, u23.x, u23.y);
          if (kDual) cw[q] = lds_u32(raw + C::kOffCodes + (f >> 3) * 32 + (f & 7) * 4);
        }
        float4 pb1[kPBper], pb2[kPBper];
#pragma unroll
        for (int q = 0; q < kPBper; ++q) {
          const int e = tid + kProd * q;
          if (e < kPB4) {
            pb1[q] = lds128(raw + kRawTile + e * 16);
            if (kDual) pb2[q] = lds128(raw + C::kOffP2 + e * 16);
            if (kMode == 1) {  // COL: R^T Q0 = U^T diag(1/lambda) Q0 -> scale the B rows by 1/lambda_i
              const float il = lds32(raw + C::kOffInv + 4 * (e / (WN / 4)));
              pb1[q] = make_float4(pb1[q].x * il, pb1[q].y * il, pb1[q].z * il, pb1[q].w * il);
            }
          }
        }
        // operand stage
        mbar_wait(&oempty[os], ((it / OPST) & 1) ^ 1);
        const uint32_t st = smem_u32(sOp) + os * kStage;
        const uint32_t sAhi = st;
        const uint32_t sAlo = st + kATile;
        const uint32_t sAc = st + 2 * kATile;
        const uint32_t sBhi = st + (kDual ? 3 : 2) * kATile;
        const uint32_t sBlo = sBhi + kBTile;
        const uint32_t sB2hi = sBlo + kBTile;
        const uint32_t sB2lo = sB2hi + kBTile;
#pragma unroll
        for (int q = 0; q < kPBper; ++q) {
          const int e = tid + kProd * q;
          if (e < kPB4) {
            const int pj = e / (WN / 4), pc = (e % (WN / 4)) * 4;
            const uint32_t off = off_mn(pc, pj, NA);
            const float4 h1 = make_float4(tf32_hi(pb1[q].x), tf32_hi(pb1[q].y), tf32_hi(pb1[q].z), tf32_hi(pb1[q].w));
            sts128(sBhi + off, h1);
            sts128(sBlo + off, make_float4(pb1[q].x - h1.x, pb1[q].y - h1.y, pb1[q].z - h1.z, pb1[q].w - h1.w));
            if (kDual) {
              const float4 h2 = make_float4(tf32_hi(pb2[q].x), tf32_hi(pb2[q].y), tf32_hi(pb2[q].z), tf32_hi(pb2[q].w));
              sts128(sB2hi + off, h2);
              sts128(sB2lo + off, make_float4(pb2[q].x - h2.x, pb2[q].y - h2.y, pb2[q].z - h2.z, pb2[q].w - h2.w));
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const int f = tid + kProd * q;
          const uint32_t off = kMode == 0 ? off_k(f >> 3, (f & 7) * 4) : off_mn((f & 31) * 4, f >> 5, 4);
          const float4 uv = xv[q];
          const float4 h = make_float4(tf32_hi(uv.x), tf32_hi(uv.y), tf32_hi(uv.z), tf32_hi(uv.w));
          sts128(sAhi + off, h);
          sts128(sAlo + off, make_float4(uv.x - h.x, uv.y - h.y, uv.z - h.z, uv.w - h.w));
          if (kDual) {
            const uint32_t w = cw[q];
            sts128(sAc + off, make_float4((float)(int8_t)(w & 0xff), (float)(int8_t)((w >> 8) & 0xff),
                                          (float)(int8_t)((w >> 16) & 0xff), (float)(int8_t)(w >> 24)));
          }
        }
        // one proxy fence orders this thread's operand-tile writes before the MMA (async proxy)
        // reads them AND its raw-slot reads before the TMA (async proxy) refills the slot; a
        // release without the fence let TMA overwrite rows before they were read on B200.
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&ofull[os]);
          mbar_arrive(&rempty[rs]);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(WN, kMode == 1 ? 1u : 0u, 1u);
      // descriptors of stage 0 at k-step 0; other stages / k-steps differ only in the start
      // address field (addr >> 4 in the low 14 bits, no carry below 256 KB of smem)
      constexpr uint32_t lboA = kMode == 0 ? 16 : 512, sboA = kMode == 0 ? 1024 : 2048, tA = kMode == 0 ? 2 : 1;
      constexpr uint32_t kAStep = kMode == 0 ? 32 : 4096;  // bytes per 8-deep k-step (K-major / MN-major)
      const uint32_t st0 = smem_u32(sOp);
      const uint64_t dA0 = desc_sw128(st0, lboA, sboA, tA);
      const uint64_t dB0 = desc_sw128(st0 + (kDual ? 3 : 2) * kATile, 512, NA * 512, 1);
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        int blk, split, nkb;
        int64_t r0;
        unit_range(u, blk, split, r0, nkb);
        const int acc = lu & 1;
        mbar_wait(&tempty[acc], ((lu >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d1 = tmem + acc * C::kAccCols;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int os = it % OPST;
          mbar_wait(&ofull[os], (it / OPST) & 1);
          tc_fence_after();
          const uint64_t so = (uint64_t)((os * kStage) >> 4);
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t aoff = so + ((k * kAStep) >> 4);
            const uint64_t boff = so + ((k * (NA * 1024)) >> 4);
            const uint64_t dAhi = dA0 + aoff;
            const uint64_t dAlo = dA0 + aoff + (kATile >> 4);
            const uint64_t dBhi = dB0 + boff;
            const uint64_t dBlo = dB0 + boff + (kBTile >> 4);
            const uint32_t acc0 = (kb | k) != 0 ? 1u : 0u;
            umma_tf32(d1, dAhi, dBhi, idesc, acc0);
            umma_tf32(d1, dAhi, dBlo, idesc, 1u);
            umma_tf32(d1, dAlo, dBhi, idesc, 1u);
            if (kDual) {
              const uint64_t dAc = dA0 + aoff + ((2 * kATile) >> 4);
              const uint64_t dB2hi = dB0 + boff + ((2 * kBTile) >> 4);
              const uint64_t dB2lo = dB0 + boff + ((3 * kBTile) >> 4);
              umma_tf32(d1 + WN, dAc, dB2hi, idesc, acc0);
              umma_tf32(d1 + WN, dAc, dB2lo, idesc, 1u);
            }
          }
          umma_commit(&oempty[os]);
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    const int quad = warp & 3;
    int lu = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
      int blk, split, nkb;
      int64_t r0;
      unit_range(u, blk, split, r0, nkb);
      const int acc = lu & 1;
      mbar_wait(&tfull[acc], (lu >> 1) & 1);
      tc_fence_after();
      const int64_t orow = (int64_t)blk * BM + quad * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + acc * C::kAccCols;
      // ROW: rows of R (and of X~) carry 1/lambda_i; COL already folded it into B
      float inv_row = 1.f;
      if (kMode == 0) inv_row = orow < a.rows ? __ldg(a.inv_lam + orow) : 1.f;
      float* out1 = a.out1 + (int64_t)split * a.nout * a.W;
      float* out2 = kDual ? a.out2 + (int64_t)split * a.nout * a.W : nullptr;
#pragma unroll
      for (int h = 0; h < NA * (kDual ? 2 : 1); ++h) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(trow + h * 32, v);
        tmem_ld_wait();
        const bool second = kDual && h >= NA;
        const int cbase = (second ? h - NA : h) * 32;
        if (orow < a.nout) {
          float* o = (second ? out2 : out1) + orow * a.W;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (cbase + c < a.W) o[cbase + c] = __fmul_rn(__uint_as_float(v[c]), inv_row);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_free<C::kTmemCols>(tmem);
  }
}

__global__ void k_reduce_splits_tc(const float* __restrict__ part, int nsplit, int64_t n, float* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < nsplit; ++s) acc += part[(int64_t)s * n + e];
    out[e] = acc;
  }
}

template <int kMode, int NA, bool kDual>
static int run_tc(const SideView& s, const float* P1, const float* P2, int W, float* OUT1, float* OUT2, float* partial,
                  int64_t pe, bool reduce1, cudaStream_t st) {
  using namespace tcp;
  using C = Cfg<kMode, NA, kDual>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tc_proj<kMode, NA, kDual>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  TcArgs a{};
  a.rows = s.rows;
  a.K = s.K;
  a.inv_lam = s.inv_lam;
  a.W = W;
  a.nout = kMode == 0 ? s.rows : (int64_t)s.K;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nblk = (a.nout + BM - 1) / BM;
  const int64_t rlen = kMode == 0 ? (int64_t)s.K : s.rows;
  // enough units for ~6 per SM (the persistent grid balances them), each >= 8 k-blocks
  int64_t ns = (6LL * nsm + nblk - 1) / nblk;
  const int64_t maxs = (rlen + 8 * BK - 1) / (8 * BK);
  if (ns > maxs) ns = maxs;
  const int64_t per = a.nout * W * (kDual ? 2 : 1);
  if (ns > 1 && ns * per > pe) ns = pe / per;
  if (ns < 1) ns = 1;
  a.chunk = ((rlen + ns - 1) / ns + BK - 1) / BK * BK;
  ns = (rlen + a.chunk - 1) / a.chunk;
  if (ns < 1) ns = 1;
  a.nblk = (int)nblk;
  a.nsplit = (int)ns;
  a.out1 = ns == 1 ? OUT1 : partial;
  a.out2 = ns == 1 ? OUT2 : partial + ns * a.nout * W;
  alignas(64) TcMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (kMode == 0) encode_map_2d(&maps.u, 2, s.U, (uint64_t)s.K, (uint64_t)s.rows, (uint64_t)s.ldu * 2, BK, BM);
  else encode_map_2d(&maps.u, 2, s.U, (uint64_t)s.K, (uint64_t)s.rows, (uint64_t)s.ldu * 2, BM, BK);
  // P tiles [BK rows][WN cols]; columns >= W and rows past the end are zero-filled by TMA
  encode_map_2d(&maps.p1, 1, P1, (uint64_t)W, (uint64_t)rlen, (uint64_t)W * 4, C::WN, BK);
  if (kDual) {
    encode_map_2d(&maps.p2, 1, P2, (uint64_t)W, (uint64_t)rlen, (uint64_t)W * 4, C::WN, BK);
    encode_map_2d(&maps.codes, 0, s.codes, (uint64_t)s.Kp, (uint64_t)s.rows, (uint64_t)s.Kp, BK, BM);
  }
  if (kMode == 1) encode_map_1d_f32(&maps.inv, s.inv_lam, (uint64_t)s.rows, BK);
  const int64_t units = nblk * ns;
  const int grid = (int)(units < nsm ? units : nsm);
  k_tc_proj<kMode, NA, kDual><<<grid, kThreads, C::kSmem, st>>>(maps, a);
  ++launch_counter();
  if (ns > 1) {
    const int64_t n = a.nout * W;
    const int g = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    if (reduce1) {
      k_reduce_splits_tc<<<g, 256, 0, st>>>(partial, (int)ns, n, OUT1);
      ++launch_counter();
    }
    if (kDual) {
      k_reduce_splits_tc<<<g, 256, 0, st>>>(partial + ns * a.nout * W, (int)ns, n, OUT2);
      ++launch_counter();
    }
  }
  return (int)ns;
}

// U (K1's residual fractions) is TMA-addressable by construction (ldu % 8 == 0).  Returns the
// number of split-K partials; with reduce1 == false and a result > 1, OUT1 is left as
// partials at `partial` (summed by the fused Gram kernel).
int launch_tc_proj_rows(const SideView& s, const float* P1, float* OUT1, const float* P2, float* OUT2, int W,
                        float* partial, int64_t pe, bool reduce1, cudaStream_t st) {
  if (s.rows == 0 || s.K == 0) return 0;
  if (W <= 32) {
    if (P2) return run_tc<0, 1, true>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, st);
    return run_tc<0, 1, false>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, st);
  }
  if (P2) return run_tc<0, 2, true>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, st);
  return run_tc<0, 2, false>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, st);
}

int launch_tc_proj_cols(const SideView& s, const float* P, float* OUT, int W, float* partial, int64_t pe, bool reduce1,
                        cudaStream_t st) {
  if (s.K == 0 || s.rows == 0) return 0;
  if (W <= 32) return run_tc<1, 1, false>(s, P, nullptr, W, OUT, nullptr, partial, pe, reduce1, st);
  return run_tc<1, 2, false>(s, P, nullptr, W, OUT, nullptr, partial, pe, reduce1, st);
}

}  // namespace lrqmm
