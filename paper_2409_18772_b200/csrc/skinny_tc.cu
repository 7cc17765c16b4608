// K2/K3 on the 5th-gen tensor cores: the RSVD passes over the quantization residual
// (Algorithm 1 sampling / power iteration / projection, reading #11) and the
// cross products of Algorithm 2, as tcgen05.mma kind::i8 with EXACT int32
// accumulation:
//
//   U = 2^15 diag(lambda) R is K1's residual fraction in Q15, i = 256 h + l, stored as two byte
//   planes h (int8) and l (uint8) — both are int8 MMA operands exactly as they sit in HBM.
//   P (K x W fp32, tiny) is split per column c with a power-of-two scale s_c (max_j |P_jc| s_c in
//   [32, 64)):  s_c P = p1 + p2 2^-7 + p3 2^-14 + r,  |p.| <= 64,  |r| <= 2^-15  (2^-20 of the
//   column max).  Then, with H_k = h . p_k and L_k = l . p_k accumulated in int32 by the MMA:
//     2^15 s_c (R P)_.c / (1/lambda) = 256 (H1 + H2 2^-7 + H3 2^-14) + L1 + L2 2^-7
//   (l . p3 < 2^-21 relative is dropped).  Two instructions per K32 step, N-stacked:
//   h x [p1|p2|p3] (N = 3 W') and l x [p1|p2] (N = 2 W').
//
//   ROW mode  OUT1[i,:] = (1/lambda_i) sum_j U[i,j] P1[j,:] / 2^15   (S1: Y = R Omega, S3: W = R Q1)
//             OUT2[i,:] = (1/lambda_i) sum_j C[i,j] P2[j,:]          (dual: A~ Q1_other, codes x P2)
//             A = h / l / codes tiles, K-major SWIZZLE_128B, straight from TMA
//   COL mode  OUT[j,:]  = sum_i U[i,j] (P[i,:] / lambda_i) / 2^15    (S2: Z = R^T Q0)
//             A = the same planes read MN-major (the R column index is the MMA M dimension)
//
// No conversion work on the SMs: the kernel is TMA -> tcgen05.mma -> epilogue, like the int8
// GEMM, and its roofline is the 2 B per element of U it streams from HBM (+1 B of codes, dual).
//
// Persistent, warp-specialised (192 threads, one CTA per SM):
//   warp 0    : TMA issuer (h, l [, codes] tiles and the B image(s) of each k-block, S-deep ring)
//   warp 1    : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5 : epilogue: TMEM accumulators -> registers (buffer released) -> split-K partials
// Work unit = (128-row/col block, reduction split); partials are summed in a fixed order by the
// consumer (deterministic, no float atomics).
#include <cooperative_groups.h>
#include <cuda.h>

#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "solvers.cuh"

namespace lrqmm {

namespace tcp {
constexpr int BM = 128;   // output rows (ROW) / output cols (COL) per unit
constexpr int BK = 128;   // reduction elements per k-block (one 128-byte swizzle row of int8)
constexpr int kTmaWarp = 0;
constexpr int kMmaWarp = 1;
constexpr int kThreads = 192;
constexpr int kThreadsFused = 256;  // + 2 warps that only join the solvers of the last CTA
constexpr int kPlane = BM * BK;  // 16 KB: one h, l or codes tile
constexpr int64_t kMaxChunk = 65536;  // |l p| <= 255 * 64: int32 accumulation exact up to 131072 terms
// kVar: 0 = residual (h, l) only, 1 = residual + codes ("dual"), 2 = codes only
// kFuse: the pass reduces its own split-K partials (last finisher of each output block), forms the
// fp64 Gram of OUT1 and runs the small solver in its last CTA (NA == 1 only; PassFuse)
constexpr int kFuseScratch = 16 * 1024;  // 128 rows x 32 fp32 (staged final rows) / Gram row-group sums
template <int kMode, int NA, int kVar, bool kFuse = false>
struct Cfg {
  static constexpr bool kHasU = kVar != 2;
  static constexpr bool kHasC = kVar != 0;
  static constexpr int WN = 32 * NA;            // W' (W rounded up to 32)
  static constexpr int kBRows = 3 * WN;         // p1 | p2 | p3
  static constexpr int kImg = kBRows * BK;      // one k-block image: kBRows rows x 128 B
  // stage: [h | l | B image] [codes | B2 image]
  static constexpr int kOffL = kPlane;
  static constexpr int kOffB = 2 * kPlane;
  static constexpr int kOffC = kHasU ? kOffB + kImg : 0;
  static constexpr int kOffB2 = kOffC + kPlane;
  static constexpr int kStageBytes = kHasC ? kOffB2 + kImg : kOffB + kImg;
  static constexpr int kStage = (kStageBytes + 1023) / 1024 * 1024;
  // kFuse: the fused Gram scratch; else the epilogue's output transpose tiles, 4 warps x 32 rows x
  // kTCols fp32 (16 columns when a codes operand makes the stage large: the dual pass keeps its
  // third ring stage)
  static constexpr bool kTransposeOut = !kFuse;
  static constexpr int kTCols = kHasC ? 16 : 32;
  static constexpr int kScratch = kFuse ? kFuseScratch : 4 * 32 * kTCols * 4;
  static constexpr int S0 = (227 * 1024 - 1280 - kScratch) / kStage;
  static constexpr int S = S0 > 6 ? 6 : S0;
  static_assert(S >= 2, "ring depth");
  static_assert(!kFuse || NA == 1, "fused Gram / solver for W <= 32 only");
  static constexpr int kSmem = S * kStage + 256 + 1024 + kScratch;
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
  // TMEM accumulator: H (3 W') | L (2 W') [| C (3 W')], int32
  static constexpr int kOffAccC = kHasU ? 5 * WN : 0;  // C accumulator columns
  static constexpr int kAccCols = kOffAccC + (kHasC ? 3 * WN : 0);
  static constexpr int kAccBufs = 2 * kAccCols <= 512 ? 2 : 1;
  static_assert(kAccBufs * kAccCols <= 512, "TMEM budget");
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
  const float* cinv1;   // 1 / s_c per column of P1 (P2)
  const float* cinv2;
  int64_t nout;   // rows (ROW) or K (COL)
  int64_t chunk;  // reduction elements per split (multiple of BK)
  int nblk, nsplit;
};

struct TcMaps {
  CUtensorMap uh, ul, codes;
};
// one launch covers both sides of the RSVD: units [0, units0) are side 0's, the rest side 1's
struct TcArgs2 {
  TcArgs a[2];
  int units0, units;
  // kFuse: per side finisher / Gram / solver outputs, launch-level solver and cross core
  PassFuseSide fs[2];
  int nslots[2];
  int solver;          // kSolveNone (G only), kSolveChol, kSolveEig
  int ngram;           // sides with a Gram (the launch ticket's target)
  int* all_cnt;        // launch ticket (zeroed; re-armed)
  const double* cross_C;  // eig: Mab = VWb^T C VWa, VWbM = VWb Mab (Alg. 2 line 366 core) in the last CTA
  const float* cross_VWa;
  const float* cross_VWb;
  float* cross_out;
  int r;
  unsigned long long* trace;  // LRQMM_FUSE_TRACE: [0] min CTA start, [1] max epilogue-loop end,
                              // [2] solver start, [3] solver end, [4] min epilogue-loop end (globaltimer ns)
};
struct TcMaps2 {
  TcMaps m[2];
};

// SWIZZLE_128B smem descriptor (layout type 2); K-major: rows of 128 B, 8-row atoms (SBO 1024);
// MN-major (int8, M = 128 = one atom): rows along K, 8-row groups 1024 B apart (SBO)
LRQMM_DEV uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// kind::i8: D s32, A int8 (signed or unsigned), B signed int8, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t n, uint32_t a_signed, uint32_t a_mn) {
  return (2u << 4) | (a_signed << 7) | (1u << 10) | (a_mn << 15) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

// byte offset of element (n, k), k < 128, in a K-major SWIZZLE_128B int8 tile (rows of 128 B)
__host__ __device__ inline uint32_t off_k128(int n, int k) {
  return (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((((k >> 4) ^ (n & 7)) & 7) << 4) + (k & 15));
}

// s_c = 2^e with max_j |P_jc| s_c in [32, 64) (1 for a zero column)
LRQMM_DEV float col_scale(unsigned cmax_bits) {
  // m = f 2^(E - 126) with f in [0.5, 1) for biased exponent E: s = 2^(6 - (E - 126)) = 2^(132 - E)
  const int E = (int)((cmax_bits >> 23) & 0xffu);
  if (E == 0) return 1.f;  // zero (or subnormal) column
  int e = 259 - E;          // biased exponent of s
  e = e > 254 ? 254 : e;
  return __uint_as_float((unsigned)e << 23);
}

struct PrepJob {
  const float* P;       // n x W, ld W
  const float* scale;   // per-row scale (COL: 1/lambda) or nullptr
  uint8_t* img;         // nkb images
  unsigned* colmax;     // 64 (scratch)
  float* cinv;          // 64: 1 / s_c
  int64_t n, nkb;
  const unsigned* cmax_in;  // column maxima supplied by P's producer (apply64), or nullptr
};
constexpr int kMaxPrep = 4;
struct PrepJobs {
  PrepJob j[kMaxPrep];
  int njobs;
  int W;
};

// B images (one cooperative launch for all operands of a pass, both sides):
//   phase 1  colmax_c = max_j |P_jc scale_j| (float bits: non-negative floats order like uints)
//   phase 2  for every k-block g, the int8 pieces p1 | p2 | p3 of s_c P[128 g : 128 g + 128, c]
//            in the K-major SWIZZLE_128B layout above (rows [0,W') p1, [W',2W') p2, [2W',3W') p3),
//            rows >= n and columns >= W zero; cinv_c = 1 / s_c.
// One thread per (column, 16 consecutive k) in phase 2: three 16-byte stores.
// kHaveMax: every job's column maxima come from P's producer (cmax_in): no phase 1, no grid
// synchronisation, an ordinary launch.
template <int NA, bool kHaveMax>
__global__ void __launch_bounds__(256) k_prep_img(PrepJobs jb) {
  ::lrqmm::pdl_enter();
  namespace cg = cooperative_groups;
  constexpr int WN = 32 * NA;
  constexpr int kImg = 3 * WN * tcp::BK;
  constexpr int kChunks = tcp::BK / 16;
  const int W = jb.W;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (!kHaveMax) {
  __shared__ unsigned sm[kMaxPrep][64];
  for (int e = threadIdx.x; e < kMaxPrep * 64; e += blockDim.x) sm[e >> 6][e & 63] = 0u;
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < jb.njobs * 64; e += blockDim.x) jb.j[e >> 6].colmax[e & 63] = 0u;
  cg::this_grid().sync();
  {
    // thread = (row lane, column c): a running max in a register, one shared atomic at the end
    constexpr int kRowsPerBlk = 256 / WN;
    const int c = threadIdx.x % WN;
    const int64_t rstride = (int64_t)gridDim.x * kRowsPerBlk;
    for (int q = 0; q < jb.njobs; ++q) {
      const PrepJob& J = jb.j[q];
      const int64_t n = J.n;
      float m = 0.f;
      if (c < W) {
        int64_t j = (int64_t)blockIdx.x * kRowsPerBlk + threadIdx.x / WN;
        for (; j + 3 * rstride < n; j += 4 * rstride) {  // 4 independent loads in flight
          float v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int64_t jj = j + t * rstride;
            v[t] = fabsf(J.scale ? J.P[jj * W + c] * J.scale[jj] : J.P[jj * W + c]);
          }
          m = fmaxf(m, fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])));
        }
        for (; j < n; j += rstride) m = fmaxf(m, fabsf(J.scale ? J.P[j * W + c] * J.scale[j] : J.P[j * W + c]));
      }
      if (m > 0.f) atomicMax(&sm[q][c], __float_as_uint(m));
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < jb.njobs * 64; e += blockDim.x) {
    const int q = e >> 6, c = e & 63;
    if (c < W && sm[q][c]) atomicMax(&jb.j[q].colmax[c], sm[q][c]);
  }
  cg::this_grid().sync();
  }
  for (int q = 0; q < jb.njobs; ++q) {
    const PrepJob& J = jb.j[q];
    const int64_t n = J.n;
    const unsigned* cmax = kHaveMax ? J.cmax_in : J.colmax;
    if (blockIdx.x == 0 && threadIdx.x < WN)
      J.cinv[threadIdx.x] = (int)threadIdx.x < W ? 1.f / col_scale(__ldcg(cmax + threadIdx.x)) : 0.f;
    const int64_t total = J.nkb * kChunks * WN;
    for (int64_t e = t0; e < total; e += gstride) {
      const int c = (int)(e % WN);  // consecutive threads: consecutive columns (coalesced reads)
      const int64_t rest = e / WN;
      const int ch = (int)(rest % kChunks);
      const int64_t g = rest / kChunks;
      const bool cok = c < W;
      const float sc = cok ? col_scale(__ldcg(cmax + c)) : 0.f;  // 0 zeroes columns >= W
      const bool hs = J.scale != nullptr;
      const float* sp = hs ? J.scale : J.P;
      // unconditional (clamped) loads so that all 16 are in flight together
      float x[16], y[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        int64_t j = g * tcp::BK + ch * 16 + t;
        j = j < n ? j : n - 1;
        x[t] = __ldg(J.P + j * W + (cok ? c : 0));
        y[t] = __ldg(sp + (hs ? j : 0));
      }
      // digits of v = p1 + p2 / 128 + p3 / 16384 (each rounded to nearest even in turn):
      //   p1 = rint(v), p2 = rint((v - p1) 128), p3 = rint(((v - p1) 128 - p2) 128).  Every difference
      //   and power-of-two scaling is exact (|v| < 64) and shifting by an even integer commutes with
      //   rint, so with n_e = rint(2^e v): p1 = n_0, p2 = n_7 - 128 n_0, p3 = n_14 - 128 n_7.
      //   Bytes packed four at a time (PRMT).
      uint32_t w1[4], w2[4], w3[4];
#pragma unroll
      for (int t4 = 0; t4 < 4; ++t4) {
        int a1[4], a2[4], a3[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = 4 * t4 + u;
          const int64_t j = g * tcp::BK + ch * 16 + t;
          const float v = j < n ? (hs ? x[t] * y[t] : x[t]) * sc : 0.f;
          const int n0 = __float2int_rn(v), n7 = __float2int_rn(v * 128.f), n14 = __float2int_rn(v * 16384.f);
          a1[u] = n0;
          a2[u] = n7 - 128 * n0;
          a3[u] = n14 - 128 * n7;
        }
        w1[t4] = __byte_perm(__byte_perm(a1[0], a1[1], 0x0040), __byte_perm(a1[2], a1[3], 0x0040), 0x5410);
        w2[t4] = __byte_perm(__byte_perm(a2[0], a2[1], 0x0040), __byte_perm(a2[2], a2[3], 0x0040), 0x5410);
        w3[t4] = __byte_perm(__byte_perm(a3[0], a3[1], 0x0040), __byte_perm(a3[2], a3[3], 0x0040), 0x5410);
      }
      uint8_t* base = J.img + g * kImg;
      *reinterpret_cast<uint4*>(base + off_k128(c, ch * 16)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
      *reinterpret_cast<uint4*>(base + off_k128(WN + c, ch * 16)) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
      *reinterpret_cast<uint4*>(base + off_k128(2 * WN + c, ch * 16)) = make_uint4(w3[0], w3[1], w3[2], w3[3]);
    }
  }
}

// ---- fused epilogue helpers (kFuse): the 128 epilogue threads synchronise on named barrier 2
LRQMM_DEV void epi_bar() { group_bar(2, 128); }
LRQMM_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Gram tile of an epilogue thread: 4 x 4 tile (ta, tc), ta <= tc, of the 8 x 8 tiles of a 32-column
// row block, rows tg, tg + kGG, ... of the staged 128 rows (36 tiles x 3 row groups = 108 threads)
constexpr int kGT = 8, kGU = kGT * (kGT + 1) / 2, kGG = 128 / kGU;
LRQMM_DEV void gram_tile_of(int u, int& ta, int& tc) {
  ta = 0; tc = 0;
  for (int a = 0; a < kGT; ++a) {
    if (u < kGT - a) { ta = a; tc = a + u; return; }
    u -= kGT - a;
  }
}

// y = sum over the ns split partials of row `row` (fixed split order), loads of two splits in flight
LRQMM_DEV void split_sum(float (&y)[32], const float* part, int ns, int64_t nout, int W, int64_t row) {
#pragma unroll
  for (int c = 0; c < 32; ++c) y[c] = 0.f;
  for (int sp = 0; sp < ns; sp += 2) {
    float4 v[2][8];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float4* p4 = reinterpret_cast<const float4*>(part + (int64_t)(sp + j) * nout * W + row * W);
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4)
        v[j][c4] = (sp + j < ns && 4 * c4 < W) ? __ldcg(p4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (sp + j < ns)
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          y[4 * c4] += v[j][c4].x;
          y[4 * c4 + 1] += v[j][c4].y;
          y[4 * c4 + 2] += v[j][c4].z;
          y[4 * c4 + 3] += v[j][c4].w;
        }
  }
}

// Ticket of the 128 epilogue threads: every thread's prior global writes are released (CTA barrier,
// then thread 0's gpu-scope acq_rel fence + atomic: cumulative), and the thread that completes the
// count (== n - 1, re-armed to 0) acquires everyone else's.  True in the last of n arrivals.
LRQMM_DEV bool epi_ticket(int* cnt, int n, int etid, int* flag) {
  epi_bar();
  if (etid == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const int t = atomicAdd(cnt, 1);
    const bool last = t == n - 1;
    if (last) {
      *cnt = 0;  // re-arm (the next launch is stream ordered)
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    *flag = last;
  }
  epi_bar();
  return *flag != 0;
}

// Publish this thread group's Gram accumulators as slot `slot` of the side, then the two-level
// fixed-order ticket sums (groups of 16 slots -> G).  Returns true in the CTA that completed the
// LAST Gram of the launch (it then runs the solvers).
LRQMM_DEV bool gram_publish(double (&acc)[16], const PassFuseSide& fs, int nslots, int slot, int W, int ngram,
                            int* all_cnt, float* scratch, int etid, int* flag) {
  const int tu = etid % kGU, tg = etid / kGU;
  const bool gt = etid < kGU * kGG;
  double (*red)[16] = reinterpret_cast<double (*)[16]>(scratch);  // kGG * kGU x 16 doubles (13.8 KB)
  epi_bar();
  if (gt)
#pragma unroll
    for (int q = 0; q < 16; ++q) red[tg * kGU + tu][q] = acc[q];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  epi_bar();
  const int npairs = W * W;
  double* part = fs.gpart + (int64_t)slot * npairs;
  for (int e = etid; e < kGU * 16; e += 128) {
    const int u = e / 16, q = e % 16;
    double sum = 0.0;
    for (int g = 0; g < kGG; ++g) sum += red[g * kGU + u][q];
    int a, c;
    gram_tile_of(u, a, c);
    const int i = 4 * a + q / 4, j = 4 * c + q % 4;
    if (i < W && j < W) {
      part[i * W + j] = sum;  // diagonal tiles: (p, q) and (q, p) hold bitwise-equal sums
      part[j * W + i] = sum;
    }
  }
  const int grp = slot / 16, ngrp = (nslots + 15) / 16;
  const int gsize = nslots - 16 * grp < 16 ? nslots - 16 * grp : 16;
  if (!epi_ticket(fs.grp_cnt + 1 + grp, gsize, etid, flag)) return false;
  for (int pr = etid; pr < npairs; pr += 128) {
    double v[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) v[b] = b < gsize ? __ldcg(fs.gpart + (int64_t)(16 * grp + b) * npairs + pr) : 0.0;
    double a = 0.0;
#pragma unroll
    for (int b = 0; b < 16; ++b)
      if (b < gsize) a += v[b];
    fs.gpart[(int64_t)(nslots + grp) * npairs + pr] = a;
  }
  if (!epi_ticket(fs.grp_cnt, ngrp, etid, flag)) return false;
  for (int pr = etid; pr < npairs; pr += 128) {
    double a = 0.0;
    for (int g = 0; g < ngrp; ++g) a += __ldcg(fs.gpart + (int64_t)(nslots + g) * npairs + pr);
    fs.G[pr] = a;
  }
  return epi_ticket(all_cnt, ngram, etid, flag);
}

template <int n>
LRQMM_DEV void fused_solve_n(const TcArgs2& args, double* base) {
  const int tid = threadIdx.x, w = tid >> 5;
  if (args.solver == kSolveChol) {
    if (w < 2 && args.fs[w].G) {  // one warp per side
      double* sm = base + w * 4096;  // 32 KB per side: S, L, T (32 x 33 doubles each)
      warp_chol_orth<n>(args.fs[w].G, args.fs[w].T64, sm, sm + 32 * 33, sm + 2 * 32 * 33);
    }
  } else if (args.solver == kSolveEig) {
    const int sd = tid >> 7;  // 128 threads per side, named barriers 3 / 4
    if (args.fs[sd].G) {
      double* sm = base + sd * 4096;
      group_eig_trunc<n, 128>(args.fs[sd].G, args.fs[sd].T, args.fs[sd].r, sm, sm + 3 * 32 * 33, tid & 127, 3 + sd);
    }
  }
}

// The last CTA of a fused pass (all kThreadsFused threads): the small solver of every side, zeroing of
// the next column-maxima consumers, and the cross core of the factor assembly after the truncation.
LRQMM_DEV void fused_solve(const TcArgs2& args, uint8_t* smem, int W) {
  double* base = reinterpret_cast<double*>(smem);
  const int tid = threadIdx.x, NT = blockDim.x;
  if (args.solver != kSolveNone) {
    switch (W) {
      case 8: fused_solve_n<8>(args, base); break;
      case 16: fused_solve_n<16>(args, base); break;
      case 24: fused_solve_n<24>(args, base); break;
      default: fused_solve_n<32>(args, base); break;
    }
  }
  for (int sd = 0; sd < 2; ++sd)
    for (int z = 0; z < 2; ++z)
      if (args.fs[sd].zero[z] && tid < 64) args.fs[sd].zero[z][tid] = 0u;
  __syncthreads();
  if (args.solver == kSolveEig && args.cross_C) {
    // Mab = VWb^T C VWa (r x r), VWbM = VWb Mab (W x r): the V_B^T V_A core of RC3 (Alg. 2)
    const int r = args.r;
    double* T1 = base;              // W x r   (C VWa)
    double* M = base + 32 * 32;     // r x r
    const double* Cc = args.cross_C;
    for (int e = tid; e < W * r; e += NT) {
      const int i = e / r, o = e % r;
      double a = 0.0;
      for (int c = 0; c < W; ++c) a += Cc[i * W + c] * (double)args.cross_VWa[c * W + o];
      T1[i * 32 + o] = a;
    }
    __syncthreads();
    for (int e = tid; e < r * r; e += NT) {
      const int u = e / r, o = e % r;
      double a = 0.0;
      for (int i = 0; i < W; ++i) a += (double)args.cross_VWb[i * W + u] * T1[i * 32 + o];
      M[u * 32 + o] = a;
    }
    __syncthreads();
    for (int e = tid; e < W * r; e += NT) {
      const int i = e / r, o = e % r;
      double a = 0.0;
      for (int u = 0; u < r; ++u) a += (double)args.cross_VWb[i * W + u] * M[u * 32 + o];
      args.cross_out[i * W + o] = (float)a;
    }
  }
}

template <int kMode, int NA, int kVar, bool kFuse>
__global__ void __launch_bounds__(kFuse ? tcp::kThreadsFused : tcp::kThreads, 1) k_tc_proj(const __grid_constant__ TcMaps2 maps,
                                                                 const __grid_constant__ TcArgs2 args) {
  ::lrqmm::pdl_enter();
  using namespace tcp;
  using C = Cfg<kMode, NA, kVar, kFuse>;
  constexpr bool kHasU = C::kHasU, kHasC = C::kHasC;
  constexpr int WN = C::WN;
  constexpr int S = C::S;
  constexpr int NACC = C::kAccBufs;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ float cinv_s[2][2][64];  // [side][P1 / P2][column]
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // offset from the __shared__ array: shared-space accesses, not generic
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * C::kStage);
  uint64_t* full = bars;          // S: stage landed (TMA tx)
  uint64_t* freeb = bars + S;     // S: MMA done with the stage
  uint64_t* tfull = bars + 2 * S; // 2
  uint64_t* tempty = tfull + 2;   // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* scratch = reinterpret_cast<float*>(smem + S * C::kStage + 256);  // kFuse: kFuseScratch bytes
  __shared__ int fuse_flag, solve_flag;
  if constexpr (kFuse) {
    if (args.trace && threadIdx.x == 0) atomicMin(args.trace, gtimer());
  }

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nunits = args.units;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
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

  auto unit_range = [&](int u, int& side, int& blk, int& split, int64_t& r0, int& nkb) {
    side = u >= args.units0 ? 1 : 0;
    const TcArgs& a = args.a[side];
    const int lu = u - (side ? args.units0 : 0);
    const int64_t r_len = kMode == 0 ? (int64_t)a.K : a.rows;
    blk = lu % a.nblk;
    split = lu / a.nblk;
    r0 = (int64_t)split * a.chunk;
    const int64_t r1 = r0 + a.chunk < r_len ? r0 + a.chunk : r_len;
    nkb = (int)((r1 - r0 + BK - 1) / BK);
  };

  if (warp == kTmaWarp) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int sd = 0; sd < 2; ++sd) {
        if (kHasU) {
          tma_prefetch_desc(&maps.m[sd].uh);
          tma_prefetch_desc(&maps.m[sd].ul);
        }
        if (kHasC) tma_prefetch_desc(&maps.m[sd].codes);
      }
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        int side, blk, split, nkb;
        int64_t r0;
        unit_range(u, side, blk, split, r0, nkb);
        const TcArgs& a = args.a[side];
        const TcMaps& mp = maps.m[side];
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % S;
          const int k0 = (int)(r0 + (int64_t)kb * BK);
          mbar_wait(&freeb[s], ((it / S) & 1) ^ 1);
          uint8_t* st = smem + s * C::kStage;
          mbar_arrive_expect_tx(&full[s], C::kStageBytes);
          const int64_t g = k0 / BK;
          if (kHasU) {
            if (kMode == 0) {
              tma_load_2d(st, &mp.uh, &full[s], k0, blk * BM);
              tma_load_2d(st + C::kOffL, &mp.ul, &full[s], k0, blk * BM);
            } else {
              tma_load_2d(st, &mp.uh, &full[s], blk * BM, k0);
              tma_load_2d(st + C::kOffL, &mp.ul, &full[s], blk * BM, k0);
            }
            bulk_load(st + C::kOffB, a.img1 + g * C::kImg, C::kImg, &full[s]);
          }
          if (kHasC) {
            tma_load_2d(st + C::kOffC, &mp.codes, &full[s], k0, blk * BM);
            bulk_load(st + C::kOffB2, a.img2 + g * C::kImg, C::kImg, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t amn = kMode == 1 ? 1u : 0u;
      constexpr uint32_t idH = idesc_i8(3 * WN, 1u, amn), idL = idesc_i8(2 * WN, 0u, amn);
      constexpr uint32_t idC = idesc_i8(3 * WN, 1u, 0u);
      constexpr uint32_t kAStep = kMode == 0 ? 32u : 4096u;  // 32 k: 32 bytes (K-major) / 32 rows (MN-major)
      const uint64_t d0 = desc_sw128(smem_u32(smem));
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
        int side, blk, split, nkb;
        int64_t r0;
        unit_range(u, side, blk, split, r0, nkb);
        const int acc = NACC == 2 ? (lu & 1) : 0;
        const uint32_t tph = NACC == 2 ? ((lu >> 1) & 1) : (lu & 1);
        mbar_wait(&tempty[acc], tph ^ 1);
        tc_fence_after();
        const uint32_t dH = tmem + acc * C::kAccCols;
        const uint32_t dL = dH + 3 * WN;
        const uint32_t dC = dH + C::kOffAccC;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          tc_fence_after();
          const uint64_t ds = d0 + (uint64_t)((s * C::kStage) >> 4);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            const uint32_t acc0 = (kb | k) != 0 ? 1u : 0u;
            if (kHasU) {
              const uint64_t dA = ds + ((k * kAStep) >> 4);
              const uint64_t dB = ds + ((C::kOffB + k * 32) >> 4);
              umma_i8(dH, dA, dB, idH, acc0);                          // h x [p1 | p2 | p3]
              umma_i8(dL, dA + (C::kOffL >> 4), dB, idL, acc0);        // l x [p1 | p2]
            }
            if (kHasC)
              umma_i8(dC, ds + ((C::kOffC + k * 32) >> 4), ds + ((C::kOffB2 + k * 32) >> 4), idC, acc0);
          }
          umma_commit(&freeb[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    // -------------------------------------------------------------- epilogue
    const int quad = warp & 3;
    // the per-column scales 1/s_c of both sides' P1 / P2 (written by the prep launch), once
    for (int e = threadIdx.x - 2 * 32; e < 4 * 64; e += 128) {
      const int sd = e >> 7, which = (e >> 6) & 1, c = e & 63;
      const TcArgs& a = args.a[sd];
      cinv_s[sd][which][c] = (sd == 0 || args.units > args.units0) && c < a.W ? (which ? a.cinv2[c] : a.cinv1[c]) : 0.f;
    }
    if (threadIdx.x == 64) solve_flag = 0;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    double gacc[16];  // kFuse: this thread's fp64 Gram tile accumulators (per slot)
#pragma unroll
    for (int q = 0; q < 16; ++q) gacc[q] = 0.0;
    int lu = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++lu) {
      int side, blk, split, nkb;
      int64_t r0;
      unit_range(u, side, blk, split, r0, nkb);
      const TcArgs& a = args.a[side];
      const int acc = NACC == 2 ? (lu & 1) : 0;
      const uint32_t tph = NACC == 2 ? ((lu >> 1) & 1) : (lu & 1);
      const int64_t orow = (int64_t)blk * BM + quad * 32 + lane;
      // ROW: rows of R and X~ carry 1/lambda_i (COL folded it into P); loaded before the wait on the
      // accumulator so its latency overlaps the unit's MMAs
      float inv_row = 1.f;
      if (kMode == 0) inv_row = orow < a.rows ? __ldg(a.inv_lam + orow) : 1.f;
      mbar_wait(&tfull[acc], tph);
      tc_fence_after();
      const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + acc * C::kAccCols;
      constexpr int GU = kHasU ? NA : 0;       // output groups of the residual product
      constexpr int NG = GU + (kHasC ? NA : 0);  // 32-column output groups per row
      float o[NG][32];
#pragma unroll
      for (int g = 0; g < GU; ++g) {
        // 256 (H1 + H2 2^-7 + H3 2^-14) + L1 + L2 2^-7, then 2^-15 / lambda / s_c (same order of
        // operations as ever; the loads go in pairs so that one wait covers two TMEM round trips)
        uint32_t v[32], w[32];
        const uint32_t tH = trow + g * 32, tL = trow + 3 * WN + g * 32;
        tmem_ld_32x32b_x32(tH + 2 * WN, v);
        tmem_ld_32x32b_x32(tH + WN, w);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) o[g][c] = (float)(int)v[c] * 0x1p-14f + (float)(int)w[c] * 0x1p-7f;
        tmem_ld_32x32b_x32(tH, v);
        tmem_ld_32x32b_x32(tL + WN, w);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) o[g][c] = (o[g][c] + (float)(int)v[c]) * 256.f + (float)(int)w[c] * 0x1p-7f;
        tmem_ld_32x32b_x32(tL, v);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) o[g][c] += (float)(int)v[c];
      }
      if (kHasC) {
#pragma unroll
        for (int g = 0; g < NA; ++g) {
          uint32_t v[32], w[32];
          const uint32_t tC = trow + C::kOffAccC + g * 32;
          tmem_ld_32x32b_x32(tC + 2 * WN, v);
          tmem_ld_32x32b_x32(tC + WN, w);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[GU + g][c] = (float)(int)v[c] * 0x1p-14f + (float)(int)w[c] * 0x1p-7f;
          tmem_ld_32x32b_x32(tC, v);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[GU + g][c] += (float)(int)v[c];
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);  // accumulator buffer free: the next unit's MMAs may start
      // scale in place (same fp32 products as stored), then this thread's output row: 16-byte stores
      // (W is a multiple of 8, rows are 32-byte aligned), per-column scales from shared memory
      if (kHasU) {
        const float s1 = inv_row * (1.f / kUScale);
        const float* cs = cinv_s[side][0];
#pragma unroll
        for (int g = 0; g < GU; ++g)
#pragma unroll
          for (int c = 0; c < 32; ++c) o[g][c] = o[g][c] * (s1 * cs[g * 32 + c]);
      }
      if (kHasC) {
        const float* cs = cinv_s[side][1];
#pragma unroll
        for (int g = 0; g < NA; ++g)
#pragma unroll
          for (int c = 0; c < 32; ++c) o[GU + g][c] = o[GU + g][c] * (inv_row * cs[g * 32 + c]);
      }
      if constexpr (C::kTransposeOut) {
        // warp-private transpose through shared memory (32 rows x kTCols, 16-byte groups XOR-swizzled
        // by row), so that each 16-byte store instruction writes whole row segments of 4 (32 columns)
        // or 8 (16 columns) rows instead of 16-byte pieces of 32 rows
        constexpr int TC = C::kTCols, NQ = TC / 4, RPI = 32 / NQ;  // float4 per row, rows per instruction
        float* stile = scratch + (warp - 2) * 32 * TC;
        const int64_t orow0 = (int64_t)blk * BM + quad * 32;
        const int rsub = lane / NQ, gq = lane % NQ;
        auto put = [&](const float* ov, float* obase, int col_base) {
          __syncwarp();
#pragma unroll
          for (int qq = 0; qq < NQ; ++qq)
            *reinterpret_cast<float4*>(stile + lane * TC + 4 * (qq ^ (lane & (NQ - 1)))) =
                make_float4(ov[4 * qq], ov[4 * qq + 1], ov[4 * qq + 2], ov[4 * qq + 3]);
          __syncwarp();
          const int col = col_base + 4 * gq;
#pragma unroll
          for (int it = 0; it < 32 / RPI; ++it) {
            const int r = RPI * it + rsub;
            const float4 v4 = *reinterpret_cast<const float4*>(stile + r * TC + 4 * (gq ^ (r & (NQ - 1))));
            if (orow0 + r < a.nout && col < a.W) *reinterpret_cast<float4*>(obase + (orow0 + r) * a.W + col) = v4;
          }
        };
        if (kHasU) {
          float* obase = a.out1 + (int64_t)split * a.nout * a.W;
#pragma unroll
          for (int g = 0; g < GU; ++g)
#pragma unroll
            for (int h = 0; h < 32 / TC; ++h) put(&o[g][h * TC], obase, g * 32 + h * TC);
        }
        if (kHasC) {
          float* obase = a.out2 + (int64_t)split * a.nout * a.W;
#pragma unroll
          for (int g = 0; g < NA; ++g)
#pragma unroll
            for (int h = 0; h < 32 / TC; ++h) put(&o[GU + g][h * TC], obase, g * 32 + h * TC);
        }
      } else if (orow < a.nout) {
        if (kHasU) {
          float4* o1 = reinterpret_cast<float4*>(a.out1 + (int64_t)split * a.nout * a.W + orow * a.W);
#pragma unroll
          for (int g = 0; g < GU; ++g)
#pragma unroll
            for (int c = 0; c < 32; c += 4)
              if (g * 32 + c < a.W) o1[(g * 32 + c) >> 2] = make_float4(o[g][c], o[g][c + 1], o[g][c + 2], o[g][c + 3]);
        }
        if (kHasC) {
          float4* o2 = reinterpret_cast<float4*>(a.out2 + (int64_t)split * a.nout * a.W + orow * a.W);
#pragma unroll
          for (int g = 0; g < NA; ++g)
#pragma unroll
            for (int c = 0; c < 32; c += 4)
              if (g * 32 + c < a.W)
                o2[(g * 32 + c) >> 2] = make_float4(o[GU + g][c], o[GU + g][c + 1], o[GU + g][c + 2], o[GU + g][c + 3]);
        }
      }
      if constexpr (kFuse) {
        const PassFuseSide& fs = args.fs[side];
        const int etid = threadIdx.x - 64;
        const int ns = a.nsplit;
        const int W = a.W;
        bool fin = true;
        if (ns > 1) {
          // last finisher of block blk: fixed-order sum of the block's split partials
          fin = epi_ticket(fs.blk_cnt + blk, ns, etid, &fuse_flag);
          if (fin) {
            if (orow < a.nout) {
              if (kHasU) {
                float y[32];
                split_sum(y, a.out1, ns, a.nout, W, orow);
                float4* f4 = reinterpret_cast<float4*>(fs.fin1 + orow * W);
#pragma unroll
                for (int c = 0; c < 32; c += 4)
                  if (c < W) f4[c >> 2] = make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
#pragma unroll
                for (int c = 0; c < 32; ++c) o[0][c] = y[c];
              }
              if (kHasC) {
                float y[32];
                split_sum(y, a.out2, ns, a.nout, W, orow);
                float4* f4 = reinterpret_cast<float4*>(fs.fin2 + orow * W);
#pragma unroll
                for (int c = 0; c < 32; c += 4)
                  if (c < W) f4[c >> 2] = make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
              }
            }
          }
        }
        if (kHasU && fs.G) {
          if (fin) {
            // stage the block's final rows (fp32, zero beyond W and past nout) and accumulate the
            // fp64 Gram tiles of this thread
            epi_bar();
            const int rl = quad * 32 + lane;
#pragma unroll
            for (int c = 0; c < 32; c += 4)
              *reinterpret_cast<float4*>(scratch + rl * 32 + c) =
                  (orow < a.nout && c < W) ? make_float4(o[0][c], o[0][c + 1], o[0][c + 2], o[0][c + 3])
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
            epi_bar();
            if (etid < kGU * kGG) {
              int ta, tc;
              gram_tile_of(etid % kGU, ta, tc);
              for (int i = etid / kGU; i < BM; i += kGG) {
                const float4 x4 = *reinterpret_cast<const float4*>(scratch + i * 32 + 4 * ta);
                const float4 y4 = *reinterpret_cast<const float4*>(scratch + i * 32 + 4 * tc);
                const double xa[4] = {x4.x, x4.y, x4.z, x4.w}, yc[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                  for (int q = 0; q < 4; ++q) gacc[p * 4 + q] = fma(xa[p], yc[q], gacc[p * 4 + q]);
              }
            }
          }
          // publish: per output block when the pass splits (slot = block), else per CTA once its last
          // unit of this side is done (slot = its index among the side's CTAs; static, deterministic)
          const int side_lo = side ? args.units0 : 0, side_hi = side ? args.units : args.units0;
          const bool pub = ns > 1 ? fin : (u + (int)gridDim.x >= side_hi);
          if (pub) {
            const int slot = ns > 1 ? blk : (int)((u - side_lo) % (int)gridDim.x);
            if (gram_publish(gacc, fs, args.nslots[side], slot, W, args.ngram, args.all_cnt, scratch, etid, &fuse_flag))
              solve_flag = 1;
          }
        }
      }
    }
  }
  __syncthreads();
  if constexpr (kFuse) {
    if (args.trace && threadIdx.x == 0) {
      const unsigned long long t = gtimer();
      atomicMax(args.trace + 1, t);
      atomicMin(args.trace + 4, t);
      if (solve_flag) args.trace[2] = t;
    }
    // the last CTA of the launch: every unit has completed, the ring shared memory is idle
    if (solve_flag) fused_solve(args, smem, args.a[0].W);
    if (args.trace && solve_flag) {
      __syncthreads();
      if (threadIdx.x == 0) args.trace[3] = gtimer();
    }
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

__global__ void k_reduce_splits_tc(const float* __restrict__ part, int nsplit, int64_t n, float* __restrict__ out) {
  ::lrqmm::pdl_enter();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < nsplit; ++s) acc += part[(int64_t)s * n + e];
    out[e] = acc;
  }
}

// many splits: 32 consecutive elements x 8 split groups per block (coalesced 128-byte rows),
// group g sums splits g, g + 8, ... in order, then the 8 group sums are added in order
__global__ void __launch_bounds__(256) k_reduce_splits_wide(const float* __restrict__ part, int nsplit, int64_t n,
                                                            float* __restrict__ out) {
  ::lrqmm::pdl_enter();
  __shared__ float red[8][33];
  const int e_l = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + e_l;
  float acc = 0.f;
  if (e < n) {
    int s = g;
    for (; s + 24 < nsplit; s += 32) {  // 4 independent loads in flight, summed in split order
      const float a0 = __ldcg(part + (int64_t)s * n + e), a1 = __ldcg(part + (int64_t)(s + 8) * n + e);
      const float a2 = __ldcg(part + (int64_t)(s + 16) * n + e), a3 = __ldcg(part + (int64_t)(s + 24) * n + e);
      acc += a0; acc += a1; acc += a2; acc += a3;
    }
    for (; s < nsplit; s += 8) acc += __ldcg(part + (int64_t)s * n + e);
  }
  red[g][e_l] = acc;
  __syncthreads();
  if (g == 0 && e < n) {
    float t = red[0][e_l];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += red[k][e_l];
    out[e] = t;
  }
}

// several reductions in one launch (blockIdx.y = job), each the same fixed split order as above
__global__ void k_reduce_splits_multi(const ReduceJobs jobs) {
  ::lrqmm::pdl_enter();
  const ReduceJob& J = jobs.j[blockIdx.y];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < J.n; e += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < J.nsplit; ++s) acc += J.part[(int64_t)s * J.n + e];
    J.out[e] = acc;
  }
}

void launch_reduce_jobs(const ReduceJobs& in, cudaStream_t st) {
  ReduceJobs jobs{};
  int64_t nmax = 0;
  for (int q = 0; q < in.n; ++q) {
    const ReduceJob& J = in.j[q];
    if (J.n == 0 || J.nsplit <= 1) continue;
    if (J.nsplit > 16) {  // long split lists: the coalesced split-group kernel, one launch each
      launch_reduce_splits(J.part, J.nsplit, J.n, J.out, st);
      continue;
    }
    jobs.j[jobs.n++] = J;
    nmax = J.n > nmax ? J.n : nmax;
  }
  if (jobs.n == 0) return;
  if (jobs.n == 1) {
    launch_reduce_splits(jobs.j[0].part, jobs.j[0].nsplit, jobs.j[0].n, jobs.j[0].out, st);
    return;
  }
  const int g = (int)((nmax + 255) / 256 < 4096 ? (nmax + 255) / 256 : 4096);
  launch_pdl(k_reduce_splits_multi, dim3((unsigned)g, (unsigned)jobs.n), 256, 0, st, jobs);
  ++launch_counter();
}

// fixed-order sum of nsplit partial planes into out (n elements)
void launch_reduce_splits(const float* part, int nsplit, int64_t n, float* out, cudaStream_t st) {
  if (n == 0) return;
  if (nsplit > 16) {
    launch_pdl(k_reduce_splits_wide, (unsigned)((n + 31) / 32), 256, 0, st, part, nsplit, n, out);
  } else {
    const int g = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    launch_pdl(k_reduce_splits_tc, g, 256, 0, st, part, nsplit, n, out);
  }
  ++launch_counter();
}

// one image: ceil(n / BK) k-block images, then colmax (64 x u32) and cinv (64 x f32)
int64_t tc_img_bytes(int64_t n, int W) {
  const int WN = W <= 32 ? 32 : 64;
  return (n + tcp::BK - 1) / tcp::BK * (3 * WN * tcp::BK) + 512;
}

template <int NA>
static void launch_prep(PrepJobs& jb, cudaStream_t st) {
  const int nsm = sm_count();
  static std::atomic<int> per_sm{0};  // co-resident blocks of the cooperative form (same on every B200)
  int per = per_sm.load(std::memory_order_relaxed);
  if (per <= 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_prep_img<NA, false>, 256, 0);
    per = per < 4 ? (per < 1 ? 1 : per) : 4;
    per_sm.store(per, std::memory_order_relaxed);
  }
  const int grid = nsm * per;
  bool have = true;
  int64_t work = 0;
  for (int q = 0; q < jb.njobs; ++q) {
    have = have && jb.j[q].cmax_in != nullptr;
    work += jb.j[q].nkb * (tcp::BK / 16) * 32 * NA;
  }
  if (have) {
    // one (column, 16 rows) item per thread, up to 8 blocks per SM
    int64_t g = (work + 255) / 256;
    if (g > 8 * nsm) g = 8 * nsm;
    if (g < 1) g = 1;
    launch_pdl(k_prep_img<NA, true>, (int)g, 256, 0, st, jb);
  } else {
    void* args[] = {&jb};
    cudaLaunchCooperativeKernel((const void*)k_prep_img<NA, false>, dim3(grid), dim3(256), args, 0, st);
  }
  ++launch_counter();
}

// One pass over one or two sides: a single prep launch builds every B image, then ONE k_tc_proj
// launch processes the units of both sides (units [0, units0) are side 0's).
template <int kMode, int NA, int kVar>
static void run_tc(int nsides, const TcPassSide* sides, int W, bool reduce1, int* ns_out, cudaStream_t st) {
  using namespace tcp;
  using C = Cfg<kMode, NA, kVar>;
  constexpr bool kHasU = C::kHasU, kHasC = C::kHasC;
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_tc_proj<kMode, NA, kVar, false>, C::kSmem, attr);
  int nsm = sm_count();
  if (sides[0].sm_reserve > 0 && sides[0].sm_reserve < nsm / 2) nsm -= sides[0].sm_reserve;
  TcArgs2 args{};
  alignas(64) TcMaps2 maps;
  memset(&maps, 0, sizeof(maps));
  PrepJobs jb{};
  jb.W = W;
  int jfirst[2] = {0, 0};
  int64_t units[2] = {0, 0};
  for (int sd = 0; sd < nsides; ++sd) {
    const SideView& s = sides[sd].view;
    TcArgs& a = args.a[sd];
    a.rows = s.rows;
    a.K = s.K;
    a.inv_lam = s.inv_lam;
    a.W = W;
    a.nout = kMode == 0 ? s.rows : (int64_t)s.K;
    const int64_t nblk = (a.nout + BM - 1) / BM;
    const int64_t rlen = kMode == 0 ? (int64_t)s.K : s.rows;
    // B images over the reduction dimension (COL folds 1/lambda_i into P's rows)
    const int64_t nkb = (rlen + BK - 1) / BK;
    const int64_t ib = tc_img_bytes(rlen, W);
    auto add_job = [&](const float* P, const float* scale, uint8_t* img, const unsigned* cmax) {
      uint8_t* tailp = img + nkb * (3 * 32 * NA * BK);
      jb.j[jb.njobs++] = PrepJob{P,    scale, img, reinterpret_cast<unsigned*>(tailp), reinterpret_cast<float*>(tailp + 256),
                                 rlen, nkb, cmax};
    };
    jfirst[sd] = jb.njobs;
    // an operand image is either prebuilt (pimg: launch_apply_prep), already built by this pass's prep
    // for the other side (the dual pass multiplies each side by the other's Q1: the same operand, the
    // same column maxima, the same image), or built now
    auto image = [&](const float* P, const float* scale, uint8_t* img, const unsigned* cmax, const uint8_t* pre,
                     const uint8_t*& out_img, const float*& out_cinv) {
      if (pre) {
        out_img = pre;
        out_cinv = img_cinv(const_cast<uint8_t*>(pre), rlen, W);
        return;
      }
      for (int q = 0; q < jb.njobs; ++q) {
        const PrepJob& o = jb.j[q];
        if (cmax && o.P == P && o.scale == scale && o.cmax_in == cmax && o.n == rlen) {
          out_img = o.img;
          out_cinv = o.cinv;
          return;
        }
      }
      add_job(P, scale, img, cmax);
      out_img = img;
      out_cinv = jb.j[jb.njobs - 1].cinv;
    };
    if (kVar == 2) {
      image(sides[sd].P2, nullptr, sides[sd].img, sides[sd].cmax2, sides[sd].pimg2, a.img1, a.cinv1);
      a.img2 = a.img1;
      a.cinv2 = a.cinv1;
    } else {
      image(sides[sd].P1, kMode == 1 ? s.inv_lam : nullptr, sides[sd].img, sides[sd].cmax1, sides[sd].pimg1, a.img1,
            a.cinv1);
      if (kHasC) {
        image(sides[sd].P2, nullptr, sides[sd].img + ib, sides[sd].cmax2, sides[sd].pimg2, a.img2, a.cinv2);
      } else {
        a.img2 = a.img1;
        a.cinv2 = a.cinv1;
      }
    }
    // enough units for ~3 per SM (the persistent grid balances them), each >= 4 k-blocks, and a
    // chunk short enough for exact int32 accumulation
    static int waves = 0;  // work units per SM (LRQMM_TC_WAVES overrides, for sweeps)
    if (!waves) {
      const char* e = getenv("LRQMM_TC_WAVES");
      waves = e ? atoi(e) : 3;  // c3 sweep (tools/waves_sweep.sh): 3 -> RSVD 867 us vs 911 at 6
      if (waves < 1) waves = 1;
    }
    int64_t ns = ((int64_t)waves * nsm + nblk - 1) / nblk;
    const int64_t maxs = (rlen + 4 * BK - 1) / (4 * BK);
    if (ns > maxs) ns = maxs;
    if (ns > 256) ns = 256;  // few output blocks (short K in COL mode): bound the partials to reduce
    const int64_t per = a.nout * W * (kVar == 1 ? 2 : 1);
    if (ns > 1 && ns * per > sides[sd].pe) ns = sides[sd].pe / per;
    const int64_t mins = (rlen + kMaxChunk - 1) / kMaxChunk;
    if (ns < mins) ns = mins;
    if (ns < 1) ns = 1;
    a.chunk = ((rlen + ns - 1) / ns + BK - 1) / BK * BK;
    ns = (rlen + a.chunk - 1) / a.chunk;
    if (ns < 1) ns = 1;
    a.nblk = (int)nblk;
    a.nsplit = (int)ns;
    float* part = sides[sd].partial;
    a.out1 = ns == 1 ? sides[sd].OUT1 : part;
    a.out2 = ns == 1 ? sides[sd].OUT2 : (kVar == 2 ? part : part + ns * a.nout * W);
    const uint64_t ld = (uint64_t)s.ldu;
    if (kHasU) {
      encode_map_2d_sw(&maps.m[sd].uh, 0, s.Uh, (uint64_t)s.K, (uint64_t)s.rows, ld, BK, BM, 128);
      encode_map_2d_sw(&maps.m[sd].ul, 0, s.Ul, (uint64_t)s.K, (uint64_t)s.rows, ld, BK, BM, 128);
    }
    if (kHasC)
      encode_map_2d_sw(&maps.m[sd].codes, 0, s.codes, (uint64_t)s.Kp, (uint64_t)s.rows, (uint64_t)s.Kp, BK, BM, 128);
    units[sd] = nblk * ns;
    ns_out[sd] = (int)ns;
  }
  if (jb.njobs > 0) launch_prep<NA>(jb, st);
  args.units0 = (int)units[0];
  args.units = (int)(units[0] + units[1]);
  const int grid = (int)(args.units < nsm ? args.units : nsm);
  launch_pdl(k_tc_proj<kMode, NA, kVar, false>, grid, kThreads, C::kSmem, st, maps, args);
  ++launch_counter();
  ReduceJobs rj{};
  for (int sd = 0; sd < nsides; ++sd) {
    const int ns = ns_out[sd];
    if (ns <= 1) continue;
    const TcArgs& a = args.a[sd];
    const int64_t n = a.nout * W;
    float* part = sides[sd].partial;
    if (reduce1 && kHasU) rj.j[rj.n++] = ReduceJob{part, ns, n, sides[sd].OUT1};
    if (kHasC) rj.j[rj.n++] = ReduceJob{kVar == 2 ? part : part + (int64_t)ns * a.nout * W, ns, n, sides[sd].OUT2};
  }
  launch_reduce_jobs(rj, st);  // both sides' reductions in one launch
}

// split count of one side's pass: enough units for ~waves per SM (the persistent grid balances
// them), each >= 4 k-blocks, a chunk short enough for exact int32 accumulation, partials in budget
static int64_t pass_splits(int64_t nblk, int64_t rlen, int64_t per, int64_t pe, int nsm, int min_kb = 4) {
  static int waves = 0;  // work units per SM (LRQMM_TC_WAVES overrides, for sweeps)
  if (!waves) {
    const char* e = getenv("LRQMM_TC_WAVES");
    waves = e ? atoi(e) : 3;
    if (waves < 1) waves = 1;
  }
  int64_t ns = ((int64_t)waves * nsm + nblk - 1) / nblk;
  const int64_t maxs = (rlen + (int64_t)min_kb * tcp::BK - 1) / ((int64_t)min_kb * tcp::BK);
  if (ns > maxs) ns = maxs;
  if (ns > 256) ns = 256;
  if (ns > 1 && ns * per > pe) ns = pe / per;
  const int64_t mins = (rlen + tcp::kMaxChunk - 1) / tcp::kMaxChunk;
  if (ns < mins) ns = mins;
  return ns < 1 ? 1 : ns;
}

// Fused pass (kFuse, NA == 1): prebuilt images, in-kernel split reduction, Gram and solvers.
template <int kMode, int kVar>
static bool run_tc_fused(int nsides, const TcPassSide* sides, int W, const PassFuse& f, int* ns_out, cudaStream_t st) {
  using namespace tcp;
  using C = Cfg<kMode, 1, kVar, true>;
  constexpr bool kHasU = C::kHasU, kHasC = C::kHasC;
  const int nsm = sm_count();
  TcArgs2 args{};
  alignas(64) TcMaps2 maps;
  memset(&maps, 0, sizeof(maps));
  int64_t units[2] = {0, 0};
  int ngram = 0;
  for (int sd = 0; sd < nsides; ++sd) {
    const SideView& s = sides[sd].view;
    const PassFuseSide& fs = f.s[sd];
    TcArgs& a = args.a[sd];
    a.rows = s.rows;
    a.K = s.K;
    a.inv_lam = s.inv_lam;
    a.W = W;
    a.nout = kMode == 0 ? s.rows : (int64_t)s.K;
    const int64_t nblk = (a.nout + BM - 1) / BM;
    const int64_t rlen = kMode == 0 ? (int64_t)s.K : s.rows;
    const int64_t per = a.nout * W * (kVar == 1 ? 2 : 1);
    // fused units carry a ticket and (finishers) a reduction: >= 8 k-blocks each
    int64_t ns = pass_splits(nblk, rlen, per, sides[sd].pe, nsm, 8);
    a.chunk = ((rlen + ns - 1) / ns + BK - 1) / BK * BK;
    ns = (rlen + a.chunk - 1) / a.chunk;
    if (ns < 1) ns = 1;
    if (ns > 1 && nblk > kFuseMaxSlots) return false;  // finisher counters / Gram slots
    a.nblk = (int)nblk;
    a.nsplit = (int)ns;
    a.img1 = kHasU ? fs.img1 : fs.img2;
    a.cinv1 = kHasU ? fs.cinv1 : fs.cinv2;
    a.img2 = kHasC ? fs.img2 : a.img1;
    a.cinv2 = kHasC ? fs.cinv2 : a.cinv1;
    float* part = sides[sd].partial;
    a.out1 = ns == 1 ? sides[sd].OUT1 : part;
    a.out2 = ns == 1 ? sides[sd].OUT2 : (kVar == 2 ? part : part + ns * a.nout * W);
    const uint64_t ld = (uint64_t)s.ldu;
    if (kHasU) {
      encode_map_2d_sw(&maps.m[sd].uh, 0, s.Uh, (uint64_t)s.K, (uint64_t)s.rows, ld, BK, BM, 128);
      encode_map_2d_sw(&maps.m[sd].ul, 0, s.Ul, (uint64_t)s.K, (uint64_t)s.rows, ld, BK, BM, 128);
    }
    if (kHasC)
      encode_map_2d_sw(&maps.m[sd].codes, 0, s.codes, (uint64_t)s.Kp, (uint64_t)s.rows, (uint64_t)s.Kp, BK, BM, 128);
    units[sd] = nblk * ns;
    ns_out[sd] = (int)ns;
    args.fs[sd] = fs;
    args.fs[sd].fin1 = sides[sd].OUT1;
    args.fs[sd].fin2 = sides[sd].OUT2;
    if (!kHasU) args.fs[sd].G = nullptr;
    if (args.fs[sd].G) ++ngram;
  }
  if (ngram != 0 && ngram != nsides) return false;  // the solver CTA needs every unit of the launch done
  args.units0 = (int)units[0];
  args.units = (int)(units[0] + units[1]);
  const int grid = (int)(args.units < nsm ? args.units : nsm);
  for (int sd = 0; sd < nsides; ++sd) {
    const int64_t us = units[sd];
    args.nslots[sd] = args.a[sd].nsplit > 1 ? args.a[sd].nblk : (int)(us < grid ? us : grid);
  }
  args.solver = ngram ? f.solver : kSolveNone;
  args.ngram = ngram;
  args.all_cnt = f.all_cnt;
  args.cross_C = f.cross_C;
  args.cross_VWa = f.cross_VWa;
  args.cross_VWb = f.cross_VWb;
  args.cross_out = f.cross_out;
  args.r = f.r;
  args.trace = f.trace;
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_tc_proj<kMode, 1, kVar, true>, C::kSmem, attr);
  launch_pdl(k_tc_proj<kMode, 1, kVar, true>, grid, kThreadsFused, C::kSmem, st, maps, args);
  ++launch_counter();
  return true;
}

bool launch_tc_pass_fused(int kind, int nsides_in, const TcPassSide* sides_in, int W, const PassFuse& f_in, int* ns_out,
                          cudaStream_t st) {
  if (W > 32) return false;
  TcPassSide sides[2];
  PassFuse f = f_in;
  int map[2], n = 0;
  for (int i = 0; i < nsides_in; ++i) {
    ns_out[i] = 0;
    if (sides_in[i].view.rows > 0 && sides_in[i].view.K > 0) {
      map[n] = i;
      f.s[n] = f_in.s[i];
      sides[n++] = sides_in[i];
    }
  }
  if (n == 0) return true;
  int ns[2] = {0, 0};
  bool ok = false;
  switch (kind) {
    case kPassRow: ok = run_tc_fused<0, 0>(n, sides, W, f, ns, st); break;
    case kPassDual: ok = run_tc_fused<0, 1>(n, sides, W, f, ns, st); break;
    case kPassCol: ok = run_tc_fused<1, 0>(n, sides, W, f, ns, st); break;
    default: ok = run_tc_fused<0, 2>(n, sides, W, f, ns, st); break;
  }
  for (int i = 0; i < n; ++i) ns_out[map[i]] = ns[i];
  return ok;
}

float* img_cinv(uint8_t* img, int64_t n, int W) {
  const int WN = W <= 32 ? 32 : 64;
  return reinterpret_cast<float*>(img + (n + tcp::BK - 1) / tcp::BK * (3 * WN * tcp::BK) + 256);
}

// ------------------------------------------------ fused chain: apply + images (cooperative)
// Phase 1: every apply job's output rows (Q = IN T64 with fp64 accumulation, or the zero-padded copy
// of Omega) and the column maxima of |OUT * cscale| (block maxima, then one atomicMax per column).
// grid.sync().  Phase 2: the cross Gram C = X1^T X2 (first kXBlocks blocks: per-block partials, the
// last block by ticket sums them in block order), then the K-major SWIZZLE_128B int8 B images of the
// next pass (the same pieces as k_prep_img) from the outputs, now L2-resident.
constexpr int kApT = 128;      // threads per block (one row per thread in phase 1)
constexpr int kXBlocks = 32;   // blocks of the cross Gram
template <int W>
__global__ void __launch_bounds__(kApT) k_apply_prep(const ApplyPrep ap, int* err_flag) {
  namespace cg = cooperative_groups;
  constexpr int L = W + 4;  // staging stride (conflict-free 16-byte row reads)
  __shared__ __align__(16) float stage[kApT * L];
  __shared__ __align__(16) float stage2[kApT * L];  // cross Gram: the second operand's rows
  __shared__ double Ts[W * W];
  __shared__ unsigned bmax[2][64];
  __shared__ int ticket;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < 2 * 64; e += kApT) bmax[e >> 6][e & 63] = 0u;
  // ---- phase 1
  int64_t tiles[2] = {0, 0};
  for (int q = 0; q < ap.na; ++q) tiles[q] = (ap.a[q].n + kApT - 1) / kApT;
  int cur = -1;
  for (int64_t t = blockIdx.x; t < tiles[0] + tiles[1]; t += gridDim.x) {
    const int q = t < tiles[0] ? 0 : 1;
    const ApplyPrepJob& J = ap.a[q];
    const int64_t i0 = (t - (q ? tiles[0] : 0)) * kApT;
    const int nr = (int)(J.n - i0 < kApT ? J.n - i0 : kApT);
    float outv[W];
    __syncthreads();
    if (J.kind == 0) {
      if (q != cur)
        for (int e = tid; e < W * W; e += kApT) Ts[e] = J.T64[e];
      cur = q;
      const float4* s4 = reinterpret_cast<const float4*>(J.IN + i0 * W);
#pragma unroll
      for (int u = 0; u < W / 4; ++u) {
        const int e = tid + u * kApT;
        if (e < nr * (W / 4)) *reinterpret_cast<float4*>(stage + (e / (W / 4)) * L + 4 * (e % (W / 4))) = __ldg(s4 + e);
      }
      __syncthreads();
      double acc[W];
#pragma unroll
      for (int o = 0; o < W; ++o) acc[o] = 0.0;
      if (tid < nr) {
#pragma unroll
        for (int c4 = 0; c4 < W / 4; ++c4) {
          const float4 v = *reinterpret_cast<const float4*>(stage + tid * L + 4 * c4);
          const double xs[4] = {(double)v.x, (double)v.y, (double)v.z, (double)v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int o = 0; o < W; ++o) acc[o] = fma(xs[j], Ts[(4 * c4 + j) * W + o], acc[o]);
        }
      }
#pragma unroll
      for (int o = 0; o < W; ++o) outv[o] = (float)acc[o];
    } else {
      // zero-padded copy of Omega (K x kk, ld ldi): a non-finite entry would own its column maximum
#pragma unroll
      for (int o = 0; o < W; ++o) {
        const float v = (tid < nr && o < J.kk) ? J.IN[(i0 + tid) * J.ldi + o] : 0.f;
        if (!isfinite(v)) atomicOr(err_flag, 1);
        outv[o] = v;
      }
    }
    if (tid < nr) {
      float4* orow = reinterpret_cast<float4*>(J.OUT + (i0 + tid) * W);
#pragma unroll
      for (int o4 = 0; o4 < W / 4; ++o4) orow[o4] = make_float4(outv[4 * o4], outv[4 * o4 + 1], outv[4 * o4 + 2], outv[4 * o4 + 3]);
    }
    // column maxima of |OUT * cscale| (the same fp32 product the image uses)
    const float cs = (J.cscale && tid < nr) ? J.cscale[i0 + tid] : 1.f;
#pragma unroll
    for (int o = 0; o < W; ++o) {
      const unsigned b = tid < nr ? __float_as_uint(fabsf(outv[o] * cs)) : 0u;
      const unsigned m = __reduce_max_sync(0xffffffffu, b);
      if (lane == (o & 31) && m) atomicMax(&bmax[q][o], m);
    }
  }
  __syncthreads();
  for (int e = tid; e < ap.na * 64; e += kApT) {
    const int q = e >> 6, c = e & 63;
    if (c < W && bmax[q][c]) atomicMax(ap.a[q].cmax + c, bmax[q][c]);
  }
  cg::this_grid().sync();
  // ---- phase 2a: cross Gram (rows staged through shared memory, coalesced)
  if (ap.X1 && (int)blockIdx.x < kXBlocks) {
    const int nb = (int)(gridDim.x < kXBlocks ? gridDim.x : kXBlocks);
    const int64_t chunk = (ap.xn + nb - 1) / nb;
    const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = r0 + chunk < ap.xn ? r0 + chunk : ap.xn;
    constexpr int NP = (W * W + kApT - 1) / kApT;
    float* s1 = stage;
    float* s2 = stage2;
    double acc[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) acc[k] = 0.0;
    int pa[NP], pb[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int pr = tid + k * kApT;
      pa[k] = pr < W * W ? pr / W : 0;
      pb[k] = pr < W * W ? pr % W : 0;
    }
    for (int64_t i0 = r0; i0 < r1; i0 += kApT) {
      const int nr = (int)(r1 - i0 < kApT ? r1 - i0 : kApT);
      __syncthreads();
      const float4* x1 = reinterpret_cast<const float4*>(ap.X1 + i0 * W);
      const float4* x2 = reinterpret_cast<const float4*>(ap.X2 + i0 * W);
      for (int e = tid; e < nr * (W / 4); e += kApT) {
        *reinterpret_cast<float4*>(s1 + (e / (W / 4)) * L + 4 * (e % (W / 4))) = __ldcg(x1 + e);
        *reinterpret_cast<float4*>(s2 + (e / (W / 4)) * L + 4 * (e % (W / 4))) = __ldcg(x2 + e);
      }
      __syncthreads();
      for (int i = 0; i < nr; ++i)
#pragma unroll
        for (int k = 0; k < NP; ++k) acc[k] = fma((double)s1[i * L + pa[k]], (double)s2[i * L + pb[k]], acc[k]);
    }
    double* part = ap.cpart + (int64_t)blockIdx.x * W * W;
#pragma unroll
    for (int k = 0; k < NP; ++k)
      if (tid + k * kApT < W * W) part[tid + k * kApT] = acc[k];
    __syncthreads();
    if (tid == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      ticket = atomicAdd(ap.ccnt, 1);
      if (ticket == nb - 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    if (ticket == nb - 1) {
      for (int pr = tid; pr < W * W; pr += kApT) {
        double a = 0.0;
        for (int b = 0; b < nb; ++b) a += __ldcg(ap.cpart + (int64_t)b * W * W + pr);
        ap.C[pr] = a;
      }
      if (tid == 0) *ap.ccnt = 0;  // re-arm
    }
  }
  // ---- phase 2b: B images (one (column, 16 rows) item per thread, three 16-byte stores)
  constexpr int WN = 32;
  constexpr int kImg = 3 * WN * tcp::BK;
  constexpr int kChunks = tcp::BK / 16;
  const int64_t gstride = (int64_t)gridDim.x * kApT;
  const int64_t t0 = (int64_t)blockIdx.x * kApT + tid;
  for (int q = 0; q < ap.np; ++q) {
    const ImgJob& J = ap.p[q];
    const int64_t n = J.n;
    const int64_t nkb = (n + tcp::BK - 1) / tcp::BK;
    if (blockIdx.x == 0 && tid < WN) {
      float* cinv = reinterpret_cast<float*>(J.img + nkb * kImg + 256);
      cinv[tid] = tid < W ? 1.f / col_scale(__ldcg(J.cmax + tid)) : 0.f;
    }
    const int64_t total = nkb * kChunks * WN;
    for (int64_t e = t0; e < total; e += gstride) {
      const int c = (int)(e % WN);
      const int64_t rest = e / WN;
      const int ch = (int)(rest % kChunks);
      const int64_t g = rest / kChunks;
      const bool cok = c < W;
      const float sc = cok ? col_scale(__ldcg(J.cmax + c)) : 0.f;
      const bool hs = J.scale != nullptr;
      float x[16], y[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        int64_t j = g * tcp::BK + ch * 16 + t;
        j = j < n ? j : n - 1;
        x[t] = __ldcg(J.P + j * W + (cok ? c : 0));
        y[t] = hs ? __ldg(J.scale + j) : 1.f;
      }
      // digits of v = p1 + p2 / 128 + p3 / 16384 (each rounded to nearest even in turn):
      //   p1 = rint(v), p2 = rint((v - p1) 128), p3 = rint(((v - p1) 128 - p2) 128).  Every difference
      //   and power-of-two scaling is exact (|v| < 64) and shifting by an even integer commutes with
      //   rint, so with n_e = rint(2^e v): p1 = n_0, p2 = n_7 - 128 n_0, p3 = n_14 - 128 n_7.
      //   Bytes packed four at a time (PRMT).
      uint32_t w1[4], w2[4], w3[4];
#pragma unroll
      for (int t4 = 0; t4 < 4; ++t4) {
        int a1[4], a2[4], a3[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = 4 * t4 + u;
          const int64_t j = g * tcp::BK + ch * 16 + t;
          const float v = j < n ? (hs ? x[t] * y[t] : x[t]) * sc : 0.f;
          const int n0 = __float2int_rn(v), n7 = __float2int_rn(v * 128.f), n14 = __float2int_rn(v * 16384.f);
          a1[u] = n0;
          a2[u] = n7 - 128 * n0;
          a3[u] = n14 - 128 * n7;
        }
        w1[t4] = __byte_perm(__byte_perm(a1[0], a1[1], 0x0040), __byte_perm(a1[2], a1[3], 0x0040), 0x5410);
        w2[t4] = __byte_perm(__byte_perm(a2[0], a2[1], 0x0040), __byte_perm(a2[2], a2[3], 0x0040), 0x5410);
        w3[t4] = __byte_perm(__byte_perm(a3[0], a3[1], 0x0040), __byte_perm(a3[2], a3[3], 0x0040), 0x5410);
      }
      uint8_t* base = J.img + g * kImg;
      *reinterpret_cast<uint4*>(base + off_k128(c, ch * 16)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
      *reinterpret_cast<uint4*>(base + off_k128(WN + c, ch * 16)) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
      *reinterpret_cast<uint4*>(base + off_k128(2 * WN + c, ch * 16)) = make_uint4(w3[0], w3[1], w3[2], w3[3]);
    }
  }
}

template <int W>
static void apply_prep_t(const ApplyPrep& ap, int* err_flag, cudaStream_t st) {
  static std::atomic<int> per_sm{0};
  int per = per_sm.load(std::memory_order_relaxed);
  if (per <= 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_apply_prep<W>, kApT, 0);
    per = per < 1 ? 1 : (per > 8 ? 8 : per);
    per_sm.store(per, std::memory_order_relaxed);
  }
  // enough blocks for the larger of the two phases, capped at co-residency
  int64_t want = 0;
  for (int q = 0; q < ap.na; ++q) want += (ap.a[q].n + kApT - 1) / kApT;
  int64_t items = 0;
  for (int q = 0; q < ap.np; ++q) items += (ap.p[q].n + tcp::BK - 1) / tcp::BK * (tcp::BK / 16) * 32;
  if ((items + kApT - 1) / kApT > want) want = (items + kApT - 1) / kApT;
  if (ap.X1 && want < kXBlocks) want = kXBlocks;
  const int64_t cap = (int64_t)sm_count() * per;
  const int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
  const ApplyPrep* app = &ap;
  void* args[] = {const_cast<ApplyPrep*>(app), &err_flag};
  cudaLaunchCooperativeKernel((const void*)k_apply_prep<W>, dim3(grid), dim3(kApT), args, 0, st);
}

void launch_apply_prep(const ApplyPrep& ap, int W, int* err_flag, cudaStream_t st) {
  switch (W) {
    case 8: apply_prep_t<8>(ap, err_flag, st); break;
    case 16: apply_prep_t<16>(ap, err_flag, st); break;
    case 24: apply_prep_t<24>(ap, err_flag, st); break;
    case 32: apply_prep_t<32>(ap, err_flag, st); break;
    default: return;
  }
  ++launch_counter();
}

// kind: kPassRow (OUT1 = R P1), kPassDual (+ OUT2 = X~ P2), kPassCol (OUT1 = R^T P1), kPassCodes
// (OUT2 = X~ P2 only, always reduced).  Sides with no rows or no K are skipped.  ns_out[i]: the
// split-K partial count of sides[i] (0 if skipped); with reduce1 == false and ns > 1 the U result
// stays as partials at sides[i].partial.
void launch_tc_pass(int kind, int nsides, const TcPassSide* sides_in, int W, bool reduce1, int* ns_out,
                    cudaStream_t st) {
  TcPassSide sides[2];
  int map[2], n = 0;
  for (int i = 0; i < nsides; ++i) {
    ns_out[i] = 0;
    if (sides_in[i].view.rows > 0 && sides_in[i].view.K > 0) { map[n] = i; sides[n++] = sides_in[i]; }
  }
  if (n == 0) return;
  int ns[2] = {0, 0};
  const bool wide = W > 32;
  switch (kind) {
    case kPassRow: wide ? run_tc<0, 2, 0>(n, sides, W, reduce1, ns, st) : run_tc<0, 1, 0>(n, sides, W, reduce1, ns, st); break;
    case kPassDual: wide ? run_tc<0, 2, 1>(n, sides, W, reduce1, ns, st) : run_tc<0, 1, 1>(n, sides, W, reduce1, ns, st); break;
    case kPassCol: wide ? run_tc<1, 2, 0>(n, sides, W, reduce1, ns, st) : run_tc<1, 1, 0>(n, sides, W, reduce1, ns, st); break;
    default: wide ? run_tc<0, 2, 2>(n, sides, W, true, ns, st) : run_tc<0, 1, 2>(n, sides, W, true, ns, st); break;
  }
  for (int i = 0; i < n; ++i) ns_out[map[i]] = ns[i];
}

// single-side forms (test hooks)
int launch_tc_proj_rows(const SideView& s, const float* P1, float* OUT1, const float* P2, float* OUT2, int W,
                        float* partial, int64_t pe, bool reduce1, uint8_t* img, cudaStream_t st) {
  TcPassSide sd{s, P1, P2, OUT1, OUT2, partial, pe, img, nullptr, nullptr};
  int ns = 0;
  launch_tc_pass(P2 ? kPassDual : kPassRow, 1, &sd, W, reduce1, &ns, st);
  return ns;
}

int launch_tc_proj_cols(const SideView& s, const float* P, float* OUT, int W, float* partial, int64_t pe, bool reduce1,
                        uint8_t* img, cudaStream_t st) {
  TcPassSide sd{s, P, nullptr, OUT, nullptr, partial, pe, img, nullptr, nullptr};
  int ns = 0;
  launch_tc_pass(kPassCol, 1, &sd, W, reduce1, &ns, st);
  return ns;
}

int launch_tc_proj_codes(const SideView& s, const float* P, float* OUT, int W, float* partial, int64_t pe,
                         uint8_t* img, cudaStream_t st) {
  TcPassSide sd{s, nullptr, P, nullptr, OUT, partial, pe, img, nullptr, nullptr};
  int ns = 0;
  launch_tc_pass(kPassCodes, 1, &sd, W, true, &ns, st);
  return ns;
}

}  // namespace lrqmm

