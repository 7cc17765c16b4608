// K2/K3 on the 5th-gen tensor cores: the RSVD passes over the quantization
// residual (Algorithm 1 sampling / power iteration / projection, PAPER.md:124-140,
// reading #11) and the cross products of Algorithm 2, computed as
// tcgen05.mma kind::f16 (bf16 in, fp32 accumulate) on EXACT integer/float splits:
//   U is the residual fraction u = lambda x - code written by K1 (R = diag(1/lambda) U) as the
//   Q15 integer i = RN(2^15 u) = 256 h + l  (h = i >> 8, l = i & 255): 256 h and l are exact in
//   bf16.  P = b1 + b2 + b3 with b1 = bf16(P), b2 = bf16(P - b1), b3 = bf16(P - b1 - b2) (to 2^-27).
//     2^15 U P = (256 h) [b1 b2 b3] + l [b1 b2]   (dropped: l b3 < 2^-24 relative) (fp32-grade)
//   Each k16 step is TWO instructions, N-stacked: A_h x [B1|B2|B3] (N = 3 W') and A_l x [B1|B2]
//   (N = 2 W') into the same accumulator column groups; the epilogue sums the three groups.
//   (tcgen05.mma costs max(~46-59, N/2) cycles per instruction at M = 128 plus ~45 per commit
//   (tools/mma_rate.cu), so wide N and 64-deep k-blocks (8 MMAs per commit) keep the single
//   issuing thread under the pass's HBM time; 3xTF32 needed 12 N = 32 MMAs per 32-deep k-block.)
// Every pass streams 2 B of U per element from HBM — this kernel's roofline.
//
//   ROW mode  OUT1[i,:] = (1/lambda_i) sum_j U[i,j] P1[j,:]      (S1: Y = R Omega, S3: W = R Q1)
//             OUT2[i,:] = (1/lambda_i) sum_j C[i,j] P2[j,:]      (dual: A~ Q1_other, codes exact in tf32)
//   COL mode  OUT[j,:]  = sum_i U[i,j] (P[i,:] / lambda_i)       (S2: Z = R^T Q0)
//
// Operand placement (the design point of this kernel):
//   A (the streamed U tile, M = 128 rows (ROW) / 128 columns (COL) of R, K = 64 per k-block)
//     lives in TENSOR MEMORY: producer warps split u into (256 h, l) bf16 pairs and tcgen05.st
//     them straight into TMEM columns; tcgen05.mma reads A from TMEM.  No shared-memory operand
//     tiles and no generic->async proxy fence on the per-k-block path.
//   B (P, K x W, tiny and shared by every CTA) is split into b1/b2/b3 ONCE per pass by
//     k_prep_img into a global image that is byte-for-byte the K-major SWIZZLE_128B smem layout
//     the MMA reads (rows [0,W') b1, [W',2W') b2, [2W',3W') b3); a bulk copy lands each
//     k-block's image in the ring slot.
//
// Persistent, warp-specialised (736 threads, one CTA per SM):
//   warps 0-15 : producers: raw U (smem) -> bf16 (256 h, l) in TMEM (+ codes -> bf16 for dual);
//                warp w owns TMEM lane quarter w % 4 and k-values [16 (w / 4), +16) of each k-block
//   warps 16-19: epilogue: TMEM accumulators -> registers (releases the buffer) -> split-K partials
//   warp 20    : TMEM allocator + single-thread tcgen05.mma issuer
//   warp 21    : TMA issuer: U (+ codes) tiles into the U ring
//   warp 22    : bulk-copy issuer: B images into the B ring (its own thread, so that waiting for
//                the MMA to free a B slot never stalls the U prefetch)
// Two rings: the U ring (raw U [+ codes] tiles, RU deep) is released by the producer warps once
// the values are in TMEM; the B ring (B images, SB deep) shares its index with the TMEM A stages
// and is released by one MMA commit (free[s]).  So HBM prefetch depth does not depend on the MMA
// completion latency.
// Work unit = (128-row/col block, reduction split); partials are summed in a fixed order
// by the consumer (deterministic, no float atomics).
#include <cuda.h>

#include <cuda_bf16.h>

#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

namespace tcp {
constexpr int BM = 128;  // output rows (ROW) / output cols (COL) per unit
constexpr int BK = 64;   // reduction elements per k-block
constexpr int kProdWarps = 16;
constexpr int kMmaWarp = kProdWarps + 4;
constexpr int kTmaWarp = kProdWarps + 5;   // U (+ codes) tiles
constexpr int kBWarp = kProdWarps + 6;     // B images
constexpr int kThreads = (kProdWarps + 7) * 32;
constexpr int kColsPerThr = BK / (kProdWarps / 4);  // 16 k-values of A per producer thread
constexpr int kWords = kColsPerThr / 2;             // 8 TMEM columns per A part per thread
constexpr int kRawU = BM * BK * 2;                  // 16 KB raw U tile (Q15)
constexpr int kRawCodes = BM * BK;                  // 8 KB raw code tile (dual)
template <int kMode, int NA, bool kDual>
struct Cfg {
  static constexpr int WN = 32 * NA;              // W' (W rounded up to 32)
  static constexpr int kBRows = 3 * WN;           // b1 | b2 | b3
  static constexpr int kImg = kBRows * BK * 2;    // one k-block image: kBRows rows x 128 B
  static constexpr int kCodesN = NA == 1 ? 3 * WN : 2 * WN;  // codes x [b1|b2|b3] (x [b1|b2] at W' = 64)
  // U slot: U tile | codes (dual);  B slot: B image | B2 image (dual)
  static constexpr int kOffCodes = kRawU;
  static constexpr int kUBytes = kRawU + (kDual ? kRawCodes : 0);
  static constexpr int kUSlot = (kUBytes + 1023) / 1024 * 1024;
  static constexpr int kBBytes = (kDual ? 2 : 1) * kImg;
  static constexpr int kBSlot = (kBBytes + 1023) / 1024 * 1024;
  // TMEM: accumulator buffer(s), then one A stage per ring slot: (256 h, l[, codes]) x 32 columns
  static constexpr int kAccCols = kBRows + (kDual ? kCodesN : 0);
  static constexpr int kAStage = (kDual ? 3 : 2) * (BK / 2);
  static constexpr int kAccBufs = (2 * kAccCols + 4 * kAStage <= 512) ? 2 : 1;
  static constexpr int kTmemS = (512 - kAccBufs * kAccCols) / kAStage;
  static constexpr int SB = kTmemS > 4 ? 4 : kTmemS;  // B ring = TMEM A stages
  static_assert(SB >= 2, "B ring depth");
  static constexpr int RU0 = (200 * 1024 - SB * kBSlot) / kUSlot;
  static constexpr int RU = RU0 > 8 ? 8 : RU0;  // U ring
  static_assert(RU >= 3, "U ring depth");
  static constexpr int S = SB;
  static constexpr int kSmem = RU * kUSlot + SB * kBSlot + 256 + 1024;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  static_assert(kAccBufs * kAccCols + S * kAStage <= 512, "TMEM budget");
  static constexpr int kOutCols = NA * 32 * (kDual ? 2 : 1);  // outputs per row
  static constexpr bool kEarlyRelease = kOutCols <= 64;       // accumulators fit in registers
};
}  // namespace tcp

struct TcArgs {
  int64_t rows;
  int K;
  const float* inv_lam;
  int W;
  float* out1;  // partial base: split s at out + s * (nout * W)
  float* out2;
  const uint8_t* img1;  // B images, one per global k-block
  const uint8_t* img2;
  int64_t nout;   // rows (ROW) or K (COL)
  int64_t chunk;  // reduction elements per split (multiple of BK)
  int nblk, nsplit;
};

struct TcMaps {
  CUtensorMap u, codes;
};

// K-major SWIZZLE_128B descriptor (layout type 2): rows of 128 B, 8-row atoms of 1024 B (SBO)
LRQMM_DEV uint64_t desc_sw128k(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// kind::f16: D f32, A = B = bf16, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
// D[tmem] (+)= A[tmem] * B[smem]
LRQMM_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
LRQMM_DEV void tmem_st(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
LRQMM_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
LRQMM_DEV uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr) : "memory");
  return v;
}
LRQMM_DEV uint4 lds128u(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
               : "memory");
  return v;
}
// two bf16 (first = lower k) packed into one 32-bit TMEM column word
LRQMM_DEV uint32_t pack_bf16x2(float first, float second) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(first, second);
  return *reinterpret_cast<const uint32_t*>(&v);
}
// Q15 integers i0, i1 (consecutive k) -> (256 h0, 256 h1) and (l0, l1) as bf16 pairs (exact)
LRQMM_DEV void split_q15(int i0, int i1, uint32_t& hw, uint32_t& lw) {
  hw = pack_bf16x2((float)(i0 & ~255), (float)(i1 & ~255));
  lw = pack_bf16x2((float)(i0 & 255), (float)(i1 & 255));
}

// byte offset of element (n, k), k < 64, in a K-major SWIZZLE_128B tile of bf16 rows (128 B)
__host__ __device__ inline uint32_t off_k128(int n, int k) {
  return (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((((k >> 3) ^ (n & 7)) & 7) << 4) + (k & 7) * 2);
}

// B image: for every k-block g of P (n x W, ld W), optionally row-scaled, the bf16 splits
// b1 | b2 | b3 of P[64 g : 64 g + 64, :]^T in the smem byte layout above; rows >= n and
// columns >= W are zero.  One thread per (column, 8 consecutive k): three 16-byte stores.
template <int NA>
__global__ void __launch_bounds__(256) k_prep_img(const float* __restrict__ P, int64_t n, int W,
                                                  const float* __restrict__ scale, int64_t nkb,
                                                  uint8_t* __restrict__ img) {
  constexpr int WN = 32 * NA;
  constexpr int kImg = 3 * WN * tcp::BK * 2;
  constexpr int kChunks = tcp::BK / 8;
  const int64_t total = nkb * kChunks * WN;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % WN);  // consecutive threads: consecutive columns (coalesced reads)
    const int64_t rest = e / WN;
    const int ch = (int)(rest % kChunks);
    const int64_t g = rest / kChunks;
    uint32_t w1[4], w2[4], w3[4];
#pragma unroll
    for (int t = 0; t < 8; t += 2) {
      float b1[2], b2[2], b3[2];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const int64_t j = g * tcp::BK + ch * 8 + t + d;
        const float v = (j < n && c < W) ? (scale ? P[j * W + c] * scale[j] : P[j * W + c]) : 0.f;
        b1[d] = __bfloat162float(__float2bfloat16_rn(v));
        const float r1 = v - b1[d];
        b2[d] = __bfloat162float(__float2bfloat16_rn(r1));
        b3[d] = r1 - b2[d];
      }
      w1[t / 2] = pack_bf16x2(b1[0], b1[1]);
      w2[t / 2] = pack_bf16x2(b2[0], b2[1]);
      w3[t / 2] = pack_bf16x2(b3[0], b3[1]);
    }
    uint8_t* base = img + g * kImg;
    *reinterpret_cast<uint4*>(base + off_k128(c, ch * 8)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
    *reinterpret_cast<uint4*>(base + off_k128(WN + c, ch * 8)) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
    *reinterpret_cast<uint4*>(base + off_k128(2 * WN + c, ch * 8)) = make_uint4(w3[0], w3[1], w3[2], w3[3]);
  }
}

template <int kMode, int NA, bool kDual>
__global__ void __launch_bounds__(tcp::kThreads, 1) k_tc_proj(const __grid_constant__ TcMaps maps, TcArgs a) {
  using namespace tcp;
  using C = Cfg<kMode, NA, kDual>;
  constexpr int WN = C::WN;
  constexpr int S = C::SB;
  constexpr int RU = C::RU;
  constexpr int NACC = C::kAccBufs;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sU = smem;                     // RU U slots (TMA)
  uint8_t* sB = smem + RU * C::kUSlot;    // S B-image slots (bulk copies)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + S * C::kBSlot);
  uint64_t* ufull = bars;               // RU: U tile landed
  uint64_t* uempty = bars + RU;         // RU: U slot consumed (producer warps)
  uint64_t* full = bars + 2 * RU;       // S: B image landed
  uint64_t* afull = full + S;           // S: A stage written (producer warps)
  uint64_t* freeb = full + 2 * S;       // S: MMA done with B slot + TMEM A stage
  uint64_t* tfull = full + 3 * S;       // 2
  uint64_t* tempty = tfull + 2;    // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t r_len = kMode == 0 ? (int64_t)a.K : a.rows;
  const int nunits = a.nblk * a.nsplit;

  if (tid == 0) {
    for (int s = 0; s < RU; ++s) {
      mbar_init(&ufull[s], 1);
      mbar_init(&uempty[s], kProdWarps);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&afull[s], kProdWarps);
      mbar_init(&freeb[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tA0 = tmem + NACC * C::kAccCols;  // A stage of slot 0

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
      if (kDual) tma_prefetch_desc(&maps.codes);
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        int blk, split, nkb;
        int64_t r0;
        unit_range(u, blk, split, r0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int su = it % RU;
          const int k0 = (int)(r0 + (int64_t)kb * BK);
          mbar_wait(&uempty[su], ((it / RU) & 1) ^ 1);
          uint8_t* us = sU + su * C::kUSlot;
          mbar_arrive_expect_tx(&ufull[su], C::kUBytes);
          if (kMode == 0) tma_load_2d(us, &maps.u, &ufull[su], k0, blk * BM);
          else tma_load_2d(us, &maps.u, &ufull[su], blk * BM, k0);
          if (kDual) tma_load_2d(us + C::kOffCodes, &maps.codes, &ufull[su], k0, blk * BM);
        }
      }
    }
    __syncwarp();
  } else if (warp == kBWarp) {
    // ------------------------------------------------ bulk copies: B images
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        int blk, split, nkb;
        int64_t r0;
        unit_range(u, blk, split, r0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % S;
          const int64_t g = (r0 + (int64_t)kb * BK) / BK;
          mbar_wait(&freeb[s], ((it / S) & 1) ^ 1);
          uint8_t* bs = sB + s * C::kBSlot;
          mbar_arrive_expect_tx(&full[s], C::kBBytes);
          bulk_load(bs, a.img1 + g * C::kImg, C::kImg, &full[s]);
          if (kDual) bulk_load(bs + C::kImg, a.img2 + g * C::kImg, C::kImg, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp < kProdWarps) {
    // ------------------------------------------------------------ producers
    const int q = warp & 3;       // TMEM lane quarter of this warp
    const int hh = warp >> 2;     // k-values [16 hh, 16 hh + 16) of the k-block
    const int m = q * 32 + lane;  // A row (TMEM lane) of this thread
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int it = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      int blk, split, nkb;
      int64_t r0;
      unit_range(u, blk, split, r0, nkb);
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int su = it % RU;
        const int s = it % S;
        mbar_wait(&ufull[su], (it / RU) & 1);
        const uint32_t raw = smem_u32(sU) + su * C::kUSlot;
        uint32_t hw[kWords], lw[kWords];
        if (kMode == 0) {
          // ROW: U tile [128 rows][64] int16, 128-byte rows, TMA SWIZZLE_128B (16-byte chunk c of
          // row r stored at chunk c ^ (r & 7)); this thread reads chunks 2 hh, 2 hh + 1 of row m
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = 2 * hh + h;
            const uint4 w = lds128u(raw + m * 128 + ((c ^ (m & 7)) << 4));
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int t = 0; t < 4; ++t)
              split_q15((int)(int16_t)(ws[t] & 0xffffu), (int)(int16_t)(ws[t] >> 16), hw[h * 4 + t], lw[h * 4 + t]);
          }
        } else {
          // COL: U tile [64 rows i][128 cols] int16 (256-byte rows); A row m = column m of R
#pragma unroll
          for (int t = 0; t < kWords; ++t) {
            const int i0 = hh * kColsPerThr + 2 * t;
            split_q15((int)(int16_t)lds_u16(raw + i0 * 256 + m * 2), (int)(int16_t)lds_u16(raw + (i0 + 1) * 256 + m * 2),
                      hw[t], lw[t]);
          }
        }
        uint32_t cw[kWords];
        if (kDual) {
          // codes tile [128 rows][64] int8, 64-byte rows, TMA SWIZZLE_64B (chunk c ^ ((r >> 1) & 3));
          // this thread's 16 codes are chunk hh of row m
          const uint4 w = lds128u(raw + C::kOffCodes + m * 64 + ((hh ^ ((m >> 1) & 3)) << 4));
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int t = 0; t < kWords; ++t) {
            const uint32_t bb = ws[t >> 1] >> (16 * (t & 1));
            cw[t] = pack_bf16x2((float)(int8_t)(bb & 0xffu), (float)(int8_t)((bb >> 8) & 0xffu));
          }
        }
        // full[s] of this round implies free[s] of the previous round (the TMA waited on it before
        // refilling B slot s), so TMEM A stage s is no longer read by the MMA
        mbar_wait(&full[s], (it / S) & 1);
        tc_fence_after();
        const uint32_t tA = tA0 + s * C::kAStage + lane_off + hh * kWords;
        tmem_st(tA, hw);
        tmem_st(tA + BK / 2, lw);
        if (kDual) tmem_st(tA + BK, cw);
        tmem_st_wait();  // the U values are consumed: the TMA may refill the U slot
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&afull[s]);
          mbar_arrive(&uempty[su]);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t id3 = idesc_bf16(3 * WN), id2 = idesc_bf16(2 * WN), idc = idesc_bf16(C::kCodesN);
      const uint64_t dB0 = desc_sw128k(smem_u32(sB));
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        int blk, split, nkb;
        int64_t r0;
        unit_range(u, blk, split, r0, nkb);
        const int acc = NACC == 2 ? (lu & 1) : 0;
        const uint32_t tph = NACC == 2 ? ((lu >> 1) & 1) : (lu & 1);
        mbar_wait(&tempty[acc], tph ^ 1);
        tc_fence_after();
        const uint32_t d1 = tmem + acc * C::kAccCols;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&afull[s], (it / S) & 1);
          mbar_wait(&full[s], (it / S) & 1);  // B image landed (already true: producers saw it)
          tc_fence_after();
          const uint64_t dB = dB0 + (uint64_t)((s * C::kBSlot) >> 4);
          const uint32_t aS = tA0 + s * C::kAStage;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t dBk = dB + (uint64_t)((k * 32) >> 4);  // 16 bf16 along K inside the 128-byte row
            const uint32_t acc0 = (kb | k) != 0 ? 1u : 0u;
            umma_bf16_ts(d1, aS + k * 8, dBk, id3, acc0);          // (256 h) x [b1 | b2 | b3]
            umma_bf16_ts(d1, aS + BK / 2 + k * 8, dBk, id2, 1u);   // l x [b1 | b2]
            if (kDual) umma_bf16_ts(d1 + 3 * WN, aS + BK + k * 8, dBk + (C::kImg >> 4), idc, acc0);  // codes x P2
          }
          umma_commit(&freeb[s]);
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
      const int acc = NACC == 2 ? (lu & 1) : 0;
      const uint32_t tph = NACC == 2 ? ((lu >> 1) & 1) : (lu & 1);
      mbar_wait(&tfull[acc], tph);
      tc_fence_after();
      const int64_t orow = (int64_t)blk * BM + quad * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + acc * C::kAccCols;
      // ROW: rows of R (and of X~) carry 1/lambda_i; COL folded it into the B image.  U is Q15.
      float inv_row = 1.f;
      if (kMode == 0) inv_row = orow < a.rows ? __ldg(a.inv_lam + orow) : 1.f;
      float* out1 = a.out1 + (int64_t)split * a.nout * a.W;
      float* out2 = kDual ? a.out2 + (int64_t)split * a.nout * a.W : nullptr;
      constexpr int NG = NA * (kDual ? 2 : 1);  // 32-column output groups per row
      // group g: columns [32 g', +32) of OUT1 (g < NA) or OUT2; the sum of its 3 (2) accumulator groups
      auto load_group = [&](int g, float (&o)[32]) {
        const bool second = kDual && g >= NA;
        const int cb = (second ? g - NA : g) * 32;
        const uint32_t tg = trow + (second ? 3 * WN : 0) + cb;
        uint32_t v0[32], v1[32];
        tmem_ld_32x32b_x32(tg, v0);
        tmem_ld_32x32b_x32(tg + WN, v1);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = __uint_as_float(v0[c]) + __uint_as_float(v1[c]);
        if (!second || C::kCodesN == 3 * WN) {
          tmem_ld_32x32b_x32(tg + 2 * WN, v0);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] += __uint_as_float(v0[c]);
        }
      };
      auto store_group = [&](int g, const float (&o)[32]) {
        const bool second = kDual && g >= NA;
        const int cb = (second ? g - NA : g) * 32;
        const float sc = second ? inv_row : inv_row * (1.f / kUScale);
        if (orow < a.nout) {
          float* op = (second ? out2 : out1) + orow * a.W;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (cb + c < a.W) op[cb + c] = __fmul_rn(o[c], sc);
        }
      };
      if constexpr (C::kEarlyRelease) {
        float o[NG][32];
#pragma unroll
        for (int g = 0; g < NG; ++g) load_group(g, o[g]);
        tc_fence_before();
        mbar_arrive(&tempty[acc]);  // accumulator buffer free: the next unit's MMAs may start
#pragma unroll
        for (int g = 0; g < NG; ++g) store_group(g, o[g]);
      } else {
#pragma unroll 1
        for (int g = 0; g < NG; ++g) {
          float o[32];
          load_group(g, o);
          store_group(g, o);
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      }
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

__global__ void k_reduce_splits_tc(const float* __restrict__ part, int nsplit, int64_t n, float* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < nsplit; ++s) acc += part[(int64_t)s * n + e];
    out[e] = acc;
  }
}

int64_t tc_img_bytes(int64_t n, int W) {
  const int WN = W <= 32 ? 32 : 64;
  return (n + tcp::BK - 1) / tcp::BK * (3 * WN * tcp::BK * 2);
}

template <int NA>
static void prep_img(const float* P, int64_t n, int W, const float* scale, uint8_t* img, cudaStream_t st) {
  const int64_t nkb = (n + tcp::BK - 1) / tcp::BK;
  const int64_t total = nkb * (tcp::BK / 8) * (32 * NA);
  const int g = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  k_prep_img<NA><<<g, 256, 0, st>>>(P, n, W, scale, nkb, img);
  ++launch_counter();
}

template <int kMode, int NA, bool kDual>
static int run_tc(const SideView& s, const float* P1, const float* P2, int W, float* OUT1, float* OUT2, float* partial,
                  int64_t pe, bool reduce1, uint8_t* img, cudaStream_t st) {
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
  // B images of P1 (and P2) over the reduction dimension; COL folds 1/lambda_i into P's rows
  const int64_t ib = tc_img_bytes(rlen, W);
  prep_img<NA>(P1, rlen, W, kMode == 1 ? s.inv_lam : nullptr, img, st);
  if (kDual) prep_img<NA>(P2, rlen, W, nullptr, img + ib, st);
  a.img1 = img;
  a.img2 = img + ib;
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
  if (kMode == 0)
    encode_map_2d_sw(&maps.u, 2, s.U, (uint64_t)s.K, (uint64_t)s.rows, (uint64_t)s.ldu * 2, BK, BM, 128);
  else
    encode_map_2d_sw(&maps.u, 2, s.U, (uint64_t)s.K, (uint64_t)s.rows, (uint64_t)s.ldu * 2, BM, BK, 0);
  if (kDual)
    encode_map_2d_sw(&maps.codes, 0, s.codes, (uint64_t)s.Kp, (uint64_t)s.rows, (uint64_t)s.Kp, BK, BM, 64);
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
                        float* partial, int64_t pe, bool reduce1, uint8_t* img, cudaStream_t st) {
  if (s.rows == 0 || s.K == 0) return 0;
  if (W <= 32) {
    if (P2) return run_tc<0, 1, true>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, img, st);
    return run_tc<0, 1, false>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, img, st);
  }
  if (P2) return run_tc<0, 2, true>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, img, st);
  return run_tc<0, 2, false>(s, P1, P2, W, OUT1, OUT2, partial, pe, reduce1, img, st);
}

int launch_tc_proj_cols(const SideView& s, const float* P, float* OUT, int W, float* partial, int64_t pe, bool reduce1,
                        uint8_t* img, cudaStream_t st) {
  if (s.K == 0 || s.rows == 0) return 0;
  if (W <= 32) return run_tc<1, 1, false>(s, P, nullptr, W, OUT, nullptr, partial, pe, reduce1, img, st);
  return run_tc<1, 2, false>(s, P, nullptr, W, OUT, nullptr, partial, pe, reduce1, img, st);
}

}  // namespace lrqmm
