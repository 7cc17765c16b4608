// K2/K3 on the 5th-gen tensor cores: the RSVD passes over the quantization
// residual (Algorithm 1 sampling / power iteration / projection, PAPER.md:124-140,
// reading #11) and the cross products of Algorithm 2, computed as
// tcgen05.mma kind::tf32 with a 3-term split (x = hi + lo, hi = tf32(x)):
//     F(X) P ~= F_hi P_hi + F_hi P_lo + F_lo P_hi          (fp32-grade, E5 in SURVEY)
// The operand F(X) (residual R or quantization codes) is recomputed from the fp32
// side X and lambda by the producer warps, written to shared memory in the
// canonical UMMA layouts, and consumed by one MMA thread; X is read from HBM once
// per pass (the roofline of these passes), the FP32 pipes only do the O(1) per
// element split.
//
//   ROW mode  OUT1[i,:] = sum_j R[i,j] P1[j,:]          (S1: Y = R Omega, S3: W = R Q1)
//             OUT2[i,:] = (1/lambda_i) sum_j C[i,j] P2[j,:]   (dual: A~ Q1_other, codes exact in tf32)
//             A operand = F(X) tile, K-major (X's natural layout), B = P tile, MN-major.
//   COL mode  OUT[j,:]  = sum_i R[i,j] P[i,:]            (S2: Z = R^T Q0)
//             A operand = R tile, MN-major (X's natural layout again), B = P tile, MN-major.
// Split-K partials are reduced in a fixed order by k_reduce_splits (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace lrqmm {

namespace tcp {
constexpr int kProdThreads = 256;
constexpr int kThreads = kProdThreads + 32;  // + one MMA warp
constexpr int BM = 128;                      // output rows (ROW) / output cols (COL) per CTA
constexpr int BK = 32;                       // reduction elements per stage (128 B of fp32)
constexpr int STAGES = 2;
constexpr int kATile = BM * BK * 4;          // 16 KB
}  // namespace tcp

struct TcArgs {
  const float* X;
  int64_t ldx;
  int64_t rows;
  int K;
  const float* lam;
  int qmax, mode;
  const float* P1;  // ROW: K x W ; COL: rows x W
  const float* P2;  // ROW dual: K x W
  int W;
  float* out1;  // partial base: split s at out + s * (nout * W)
  float* out2;
  int64_t nout;   // rows (ROW) or K (COL)
  int64_t chunk;  // reduction elements per split (multiple of BK)
};

LRQMM_DEV float codef(float lam, float x, int mode, int qmax) {
  const float p = __fmul_rn(lam, x);
  const float e = __fmaf_rn(lam, x, -p);
  float c;
  if (mode == kRoundFloor) {
    c = floorf(p);
    if (p == c && (e < 0.f || (p == 0.f && x < 0.f))) c -= 1.f;
  } else if (mode == kRoundTrunc) {
    c = truncf(p);
    if (p == c && p != 0.f) {
      if (p > 0.f && e < 0.f) c -= 1.f;
      if (p < 0.f && e > 0.f) c += 1.f;
    }
  } else {
    c = rintf(p);
    const float fl = floorf(p);
    if (p - fl == 0.5f && e != 0.f) c = (e > 0.f) ? fl + 1.f : fl;
  }
  const float q = static_cast<float>(qmax);
  return fminf(fmaxf(c, -q), q);
}
LRQMM_DEV float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// UMMA smem descriptors (SW128).  K-major: SBO = 1024 B between 8-row groups.
// MN-major: LBO = byte distance between 32-element MN atoms, SBO = between 8-deep K groups.
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
__global__ void __launch_bounds__(tcp::kThreads, 1) k_tc_proj(TcArgs a) {
  using namespace tcp;
  constexpr int WN = 32 * NA;                 // MMA N
  constexpr int kBTile = BK * WN * 4;         // 4 or 8 KB
  constexpr int kStage = (kDual ? 3 : 2) * kATile + (kDual ? 4 : 2) * kBTile;
  constexpr uint32_t kTmemCols = (kDual ? 2 : 1) * WN <= 32 ? 32 : ((kDual ? 2 : 1) * WN <= 64 ? 64 : 128);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* done = bars + 2 * STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t o0 = (int64_t)blockIdx.x * BM;  // first output row (ROW) / col (COL)
  const int64_t r_begin = (int64_t)blockIdx.y * a.chunk;
  const int64_t r_len = kMode == 0 ? (int64_t)a.K : a.rows;
  const int64_t r_end = r_begin + a.chunk < r_len ? r_begin + a.chunk : r_len;
  const int nkb = (int)((r_end - r_begin + BK - 1) / BK);
  const bool vec = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kProdThreads);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ------------------------------------------------------------- producers
    // per thread: 4 float4 of X per stage
    float lam_r[4], inv_r[4];
    if (kMode == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t row = o0 + ((tid + 256 * u) >> 3);
        lam_r[u] = row < a.rows ? a.lam[row] : 1.f;
        inv_r[u] = __frcp_rn(lam_r[u]);
      }
    }
    auto load = [&](int kb, float4 (&v)[4]) {
      const int64_t k0 = r_begin + (int64_t)kb * BK;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = tid + 256 * u;
        int64_t row, col;
        if (kMode == 0) {
          row = o0 + (f >> 3);
          col = k0 + (f & 7) * 4;
        } else {
          row = k0 + (f >> 5);
          col = o0 + (f & 31) * 4;
        }
        const int64_t rmax = kMode == 0 ? a.rows : r_end;
        const int64_t cmax = kMode == 0 ? r_end : (int64_t)a.K;
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < rmax) {
          const float* xr = a.X + row * a.ldx;
          if (vec && col + 3 < cmax) {
            t = __ldcs(reinterpret_cast<const float4*>(xr + col));
          } else {
            if (col + 0 < cmax) t.x = xr[col + 0];
            if (col + 1 < cmax) t.y = xr[col + 1];
            if (col + 2 < cmax) t.z = xr[col + 2];
            if (col + 3 < cmax) t.w = xr[col + 3];
          }
        }
        v[u] = t;
      }
    };
    float4 cur[4];
    if (nkb > 0) load(0, cur);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)((kb / STAGES) & 1);
      float4 nxt[4];
      if (kb + 1 < nkb) load(kb + 1, nxt);
      const int64_t k0 = r_begin + (int64_t)kb * BK;
      float lam_c[4], inv_c[4];
      if (kMode == 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t row = k0 + ((tid + 256 * u) >> 5);
          lam_c[u] = row < r_end ? a.lam[row] : 1.f;
          inv_c[u] = __frcp_rn(lam_c[u]);
        }
      }
      // B tile(s): P rows [k0, k0+BK) x WN (zero beyond W / range), MN-major
      float4 pb1 = make_float4(0.f, 0.f, 0.f, 0.f), pb2 = pb1;
      int pj = 0, pc = 0;
      constexpr int kPB4 = BK * WN / 4;  // float4 per B tile
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* st = smem + s * kStage;
      uint8_t* sAhi = st;
      uint8_t* sAlo = st + kATile;
      uint8_t* sAc = st + 2 * kATile;
      uint8_t* sBhi = st + (kDual ? 3 : 2) * kATile;
      uint8_t* sBlo = sBhi + kBTile;
      uint8_t* sB2hi = sBlo + kBTile;
      uint8_t* sB2lo = sB2hi + kBTile;
      for (int e = tid; e < kPB4; e += kProdThreads) {
        pj = e / (WN / 4);
        pc = (e % (WN / 4)) * 4;
        const int64_t k = k0 + pj;
        pb1 = make_float4(0.f, 0.f, 0.f, 0.f);
        pb2 = pb1;
        if (k < r_end) {
          const float* p1 = a.P1 + k * a.W;
          if (pc + 0 < a.W) pb1.x = p1[pc + 0];
          if (pc + 1 < a.W) pb1.y = p1[pc + 1];
          if (pc + 2 < a.W) pb1.z = p1[pc + 2];
          if (pc + 3 < a.W) pb1.w = p1[pc + 3];
          if (kDual) {
            const float* p2 = a.P2 + k * a.W;
            if (pc + 0 < a.W) pb2.x = p2[pc + 0];
            if (pc + 1 < a.W) pb2.y = p2[pc + 1];
            if (pc + 2 < a.W) pb2.z = p2[pc + 2];
            if (pc + 3 < a.W) pb2.w = p2[pc + 3];
          }
        }
        const uint32_t off = off_mn(pc, pj, NA);
        const float4 h1 = make_float4(tf32_hi(pb1.x), tf32_hi(pb1.y), tf32_hi(pb1.z), tf32_hi(pb1.w));
        *reinterpret_cast<float4*>(sBhi + off) = h1;
        *reinterpret_cast<float4*>(sBlo + off) = make_float4(pb1.x - h1.x, pb1.y - h1.y, pb1.z - h1.z, pb1.w - h1.w);
        if (kDual) {
          const float4 h2 = make_float4(tf32_hi(pb2.x), tf32_hi(pb2.y), tf32_hi(pb2.z), tf32_hi(pb2.w));
          *reinterpret_cast<float4*>(sB2hi + off) = h2;
          *reinterpret_cast<float4*>(sB2lo + off) = make_float4(pb2.x - h2.x, pb2.y - h2.y, pb2.z - h2.z, pb2.w - h2.w);
        }
      }
      // A tile(s): F(X) hi / lo (+ codes)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = tid + 256 * u;
        const float l = kMode == 0 ? lam_r[u] : lam_c[u];
        const float il = kMode == 0 ? inv_r[u] : inv_c[u];
        const float xs[4] = {cur[u].x, cur[u].y, cur[u].z, cur[u].w};
        float r[4], c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          c[q] = codef(l, xs[q], a.mode, a.qmax);
          r[q] = __fmul_rn(__fmaf_rn(l, xs[q], -c[q]), il);
        }
        uint32_t off;
        if (kMode == 0) off = off_k(f >> 3, (f & 7) * 4);
        else off = off_mn((f & 31) * 4, f >> 5, 4);
        const float4 h = make_float4(tf32_hi(r[0]), tf32_hi(r[1]), tf32_hi(r[2]), tf32_hi(r[3]));
        *reinterpret_cast<float4*>(sAhi + off) = h;
        *reinterpret_cast<float4*>(sAlo + off) = make_float4(r[0] - h.x, r[1] - h.y, r[2] - h.z, r[3] - h.w);
        if (kDual) *reinterpret_cast<float4*>(sAc + off) = make_float4(c[0], c[1], c[2], c[3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&full[s]);
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
    }
    // ------------------------------------------------------------- epilogue
    if (warp < 4) {
      mbar_wait(done, 0);
      tc_fence_after();
      const int64_t orow = o0 + warp * 32 + lane;
      const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
      float inv_row = 1.f;
      if (kDual) inv_row = orow < a.rows ? __frcp_rn(a.lam[orow]) : 1.f;
      float* out1 = a.out1 + (int64_t)blockIdx.y * a.nout * a.W;
      float* out2 = kDual ? a.out2 + (int64_t)blockIdx.y * a.nout * a.W : nullptr;
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
          for (int c = 0; c < 32; ++c) {
            if (cbase + c < a.W) {
              float val = __uint_as_float(v[c]);
              if (second) val = __fmul_rn(val, inv_row);
              o[cbase + c] = val;
            }
          }
        }
      }
      tc_fence_before();
    }
  } else {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
    constexpr uint32_t idesc1 = idesc_tf32(WN, kMode == 1 ? 1u : 0u, 1u);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (uint32_t)((kb / STAGES) & 1));
      tc_fence_after();
      const uint32_t st = smem_u32(smem + s * kStage);
      const uint32_t aHi = st, aLo = st + kATile, aC = st + 2 * kATile;
      const uint32_t bHi = st + (kDual ? 3 : 2) * kATile;
      const uint32_t bLo = bHi + kBTile, b2Hi = bLo + kBTile, b2Lo = b2Hi + kBTile;
#pragma unroll
      for (int k = 0; k < BK / 8; ++k) {
        uint32_t aoff, lboA, sboA, tA;
        if (kMode == 0) { aoff = k * 32; lboA = 16; sboA = 1024; tA = 2; }        // K-major: +32 B per 8 k
        else { aoff = k * 4096; lboA = 512; sboA = 2048; tA = 1; }                // MN-major: next two 4-deep groups
        const uint32_t boff = k * (NA * 1024);
        const uint64_t dAhi = desc_sw128(aHi + aoff, lboA, sboA, tA);
        const uint64_t dAlo = desc_sw128(aLo + aoff, lboA, sboA, tA);
        const uint64_t dBhi = desc_sw128(bHi + boff, 512, NA * 512, 1);
        const uint64_t dBlo = desc_sw128(bLo + boff, 512, NA * 512, 1);
        const uint32_t acc0 = (kb | k) != 0 ? 1u : 0u;
        umma_tf32(tmem, dAhi, dBhi, idesc1, acc0);
        umma_tf32(tmem, dAhi, dBlo, idesc1, 1u);
        umma_tf32(tmem, dAlo, dBhi, idesc1, 1u);
        if (kDual) {
          const uint64_t dAc = desc_sw128(aC + aoff, lboA, sboA, tA);
          const uint64_t dB2hi = desc_sw128(b2Hi + boff, 512, NA * 512, 1);
          const uint64_t dB2lo = desc_sw128(b2Lo + boff, 512, NA * 512, 1);
          umma_tf32(tmem + WN, dAc, dB2hi, idesc1, acc0);
          umma_tf32(tmem + WN, dAc, dB2lo, idesc1, 1u);
        }
      }
      umma_commit(&empty[s]);
    }
    umma_commit(done);
    }
    __syncwarp();  // reconverge before the CTA barrier (bar.sync is .aligned)
  }
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_free<kTmemCols>(tmem);
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
static void run_tc(const TcArgs& a0, float* OUT1, float* OUT2, float* partial, int64_t pe, cudaStream_t st) {
  using namespace tcp;
  constexpr int WN = 32 * NA;
  constexpr int kBTile = BK * WN * 4;
  constexpr int kStage = (kDual ? 3 : 2) * kATile + (kDual ? 4 : 2) * kBTile;
  constexpr int kSmem = STAGES * kStage + 1024 + 128;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tc_proj<kMode, NA, kDual>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  TcArgs a = a0;
  const int64_t nblk = (a.nout + BM - 1) / BM;
  const int64_t rlen = kMode == 0 ? (int64_t)a.K : a.rows;
  const int per_sm = kSmem <= 113 * 1024 ? 2 : 1;
  const int64_t slots = 148LL * per_sm;
  // splits so that the grid is ~3 waves of resident CTAs, each split >= 4 stages of work
  int64_t ns = (3 * slots + nblk - 1) / nblk;
  const int64_t maxs = (rlen + 4 * BK - 1) / (4 * BK);
  if (ns > maxs) ns = maxs;
  const int64_t per = a.nout * a.W * (kDual ? 2 : 1);
  if (ns > 1 && ns * per > pe) ns = pe / per;
  if (ns < 1) ns = 1;
  a.chunk = ((rlen + ns - 1) / ns + BK - 1) / BK * BK;
  ns = (rlen + a.chunk - 1) / a.chunk;
  if (ns < 1) ns = 1;
  a.out1 = ns == 1 ? OUT1 : partial;
  a.out2 = ns == 1 ? OUT2 : partial + ns * a.nout * a.W;
  dim3 grid((unsigned)nblk, (unsigned)ns);
  k_tc_proj<kMode, NA, kDual><<<grid, kThreads, kSmem, st>>>(a);
  ++launch_counter();
  if (ns > 1) {
    const int64_t n = a.nout * a.W;
    const int g = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    k_reduce_splits_tc<<<g, 256, 0, st>>>(partial, (int)ns, n, OUT1);
    ++launch_counter();
    if (kDual) {
      k_reduce_splits_tc<<<g, 256, 0, st>>>(partial + ns * a.nout * a.W, (int)ns, n, OUT2);
      ++launch_counter();
    }
  }
}

static TcArgs make_args(const SideView& s, const float* P1, const float* P2, int W, int64_t nout) {
  TcArgs a{};
  a.X = s.X;
  a.ldx = s.ldx;
  a.rows = s.rows;
  a.K = s.K;
  a.lam = s.lam;
  a.qmax = s.qmax;
  a.mode = s.mode;
  a.P1 = P1;
  a.P2 = P2;
  a.W = W;
  a.nout = nout;
  return a;
}

// ROW mode: OUT1 = R P1 (f1 must be residual); dual: OUT2 = X~ P2
void launch_tc_proj_rows(const SideView& s, const float* P1, float* OUT1, const float* P2, float* OUT2, int W,
                         float* partial, int64_t pe, cudaStream_t st) {
  if (s.rows == 0) return;
  TcArgs a = make_args(s, P1, P2, W, s.rows);
  if (W <= 32) {
    if (P2) run_tc<0, 1, true>(a, OUT1, OUT2, partial, pe, st);
    else run_tc<0, 1, false>(a, OUT1, OUT2, partial, pe, st);
  } else {
    if (P2) run_tc<0, 2, true>(a, OUT1, OUT2, partial, pe, st);
    else run_tc<0, 2, false>(a, OUT1, OUT2, partial, pe, st);
  }
}

// COL mode: OUT = R^T P (P rows x W, OUT K x W)
void launch_tc_proj_cols(const SideView& s, const float* P, float* OUT, int W, float* partial, int64_t pe,
                         cudaStream_t st) {
  if (s.K == 0) return;
  TcArgs a = make_args(s, P, nullptr, W, s.K);
  if (W <= 32) run_tc<1, 1, false>(a, OUT, nullptr, partial, pe, st);
  else run_tc<1, 2, false>(a, OUT, nullptr, partial, pe, st);
}

}  // namespace lrqmm
