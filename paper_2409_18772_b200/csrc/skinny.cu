// Small right-multiplies by W x W matrices (orthonormalisation transforms and the
// factor assembly of Algorithm 2).
#include "common.cuh"
#include "kernels.h"
#include <cuda_bf16.h>

namespace lrqmm {

[[maybe_unused]] static int clamp_grid(int64_t want) { return (int)(want < 148 * 32 ? (want < 1 ? 1 : want) : 148 * 32); }

// ----------------------------------------------------- small right-multiplies
// Blocks of 128 rows: the rows are staged through shared memory with coalesced 16-byte loads,
// each thread then multiplies ITS row (in registers) by the small matrix (broadcast from shared
// memory), and the results go back through shared memory to coalesced stores.
constexpr int kApRows = 128;
// staging row stride in floats for W columns: W + 4 keeps per-thread 16-byte row reads
// conflict-free (8 consecutive threads hit 8 distinct 16-byte bank groups)
__host__ __device__ constexpr int ap_ld(int w) { return w + 4; }

template <int W>
LRQMM_DEV void stage_rows_in(const float* __restrict__ src, int64_t i0, int nr, float* sm) {
  constexpr int L = ap_ld(W);
  const float4* s4 = reinterpret_cast<const float4*>(src + i0 * W);
  // all of the tile's loads issue before the first store (W / 4 float4 per thread in flight)
  float4 v[W / 4];
#pragma unroll
  for (int u = 0; u < W / 4; ++u) {
    const int e = threadIdx.x + u * kApRows;
    if (e < nr * (W / 4)) v[u] = __ldg(s4 + e);
  }
#pragma unroll
  for (int u = 0; u < W / 4; ++u) {
    const int e = threadIdx.x + u * kApRows;
    if (e < nr * (W / 4)) *reinterpret_cast<float4*>(sm + (e / (W / 4)) * L + 4 * (e % (W / 4))) = v[u];
  }
}

// The same tile staged asynchronously (cp.async, 16 bytes per copy, into the padded rows): no
// register staging, so the next tile's loads are in flight while this one is multiplied; one commit
// group per call.
template <int W>
LRQMM_DEV void stage_rows_async(const float* __restrict__ src, int64_t i0, int nr, float* sm) {
  constexpr int L = ap_ld(W);
  const float4* s4 = reinterpret_cast<const float4*>(src + i0 * W);
#pragma unroll
  for (int u = 0; u < W / 4; ++u) {
    const int e = threadIdx.x + u * kApRows;
    if (e < nr * (W / 4)) {
      const uint32_t dst = smem_u32(sm + (e / (W / 4)) * L + 4 * (e % (W / 4)));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(s4 + e) : "memory");
    }
  }
}
LRQMM_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
LRQMM_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// OUT[i, col0 + o] = sum_c IN1[i,c] S1[c,o] (+ sum_c IN2[i,c] S2[c,o]),  o < nout (<= NO <= W).
// Up to kMaxApply jobs per launch: job q owns blocks [first[q], first[q+1]) and walks its rows.
// NO = the outputs computed per row (nout rounded up to 8): no FMAs or shared-memory reads for the
// W - NO columns that no job writes (the factor assembly writes r of W).
// kIn2: some job of the launch has IN2 (staging for both inputs); else one input, half the staging
// shared memory (more resident blocks for the tall single-input assembly jobs)
template <int W, int NO, bool kIn2>
__global__ void __launch_bounds__(kApRows) k_apply_small(const __grid_constant__ ApplyJobs jobs) {
  ::lrqmm::pdl_enter();
  constexpr int L = ap_ld(W);
  extern __shared__ __align__(16) float apsm[];
  int q = 0;
  while (q + 1 < jobs.n && (int)blockIdx.x >= jobs.first[q + 1]) ++q;
  const ApplyJob& J = jobs.j[q];
  const int b0 = jobs.first[q], nb = jobs.first[q + 1] - b0;
  float* s1 = apsm;                      // W x NO
  float* s2 = s1 + W * NO;               // W x NO
  float* sin_base = s2 + W * NO;         // 2 buffers x (IN1[, IN2]) x kApRows x L (cp.async double buffer)
  constexpr int kSlot = (kIn2 ? 2 : 1) * kApRows * L;
  const int nout = J.nout;
  const int kin = J.kin > 0 && J.kin < W ? J.kin : W;
  for (int e = threadIdx.x; e < W * NO; e += blockDim.x) {
    const int c = e / NO, o = e % NO;
    s1[e] = o < nout ? J.S1[c * J.ldS + o] : 0.f;
    s2[e] = (J.IN2 && o < nout) ? J.S2[c * J.ldS + o] : 0.f;
  }
  const int64_t n = J.n;
  const bool vec_out = nout % 4 == 0 && J.col0 % 4 == 0 && J.ldo % 4 == 0 && (reinterpret_cast<uintptr_t>(J.OUT) & 15) == 0;
  const int64_t step = (int64_t)nb * kApRows;
  auto stage = [&](int64_t i0, int slot) {
    if (i0 < n) {
      const int nr = (int)(n - i0 < kApRows ? n - i0 : kApRows);
      stage_rows_async<W>(J.IN1, i0, nr, sin_base + slot * kSlot);
      if (kIn2 && J.IN2) stage_rows_async<W>(J.IN2, i0, nr, sin_base + slot * kSlot + kApRows * L);
    }
    cp_async_commit();
  };
  const int64_t first = (int64_t)(blockIdx.x - b0) * kApRows;
  stage(first, 0);
  stage(first + step, 1);
  int it = 0;
  for (int64_t i0 = first; i0 < n; i0 += step, ++it) {
    const int nr = (int)(n - i0 < kApRows ? n - i0 : kApRows);
    float* sin1 = sin_base + (it & 1) * kSlot;
    float* sin2 = sin1 + kApRows * L;
    cp_async_wait<1>();  // this tile's group has landed (the next one may still be in flight)
    __syncthreads();
    float acc[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) acc[o] = 0.f;
    if (threadIdx.x < nr) {
#pragma unroll(W <= 32 ? W / 4 : 2)  // bounded unrolling for the wide sketches (build time)
      for (int c4 = 0; c4 < W / 4; ++c4) {
        if (4 * c4 >= kin) break;  // zero-padded sketch columns contribute nothing
        const float4 v = *reinterpret_cast<const float4*>(sin1 + threadIdx.x * L + 4 * c4);
        const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int o = 0; o < NO; ++o) acc[o] = fmaf(xs[j], s1[(4 * c4 + j) * NO + o], acc[o]);
      }
      if (kIn2 && J.IN2) {
#pragma unroll(W <= 32 ? W / 4 : 2)
        for (int c4 = 0; c4 < W / 4; ++c4) {
          if (4 * c4 >= kin) break;
          const float4 v = *reinterpret_cast<const float4*>(sin2 + threadIdx.x * L + 4 * c4);
          const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int o = 0; o < NO; ++o) acc[o] = fmaf(xs[j], s2[(4 * c4 + j) * NO + o], acc[o]);
        }
      }
    }
    __syncthreads();  // every row of this buffer has been read: stage the tile after next into it
    stage(i0 + 2 * step, it & 1);
    // outputs straight from registers: this thread's row, 16-byte stores when aligned
    if (threadIdx.x < nr) {
      float* orow = J.OUT + (i0 + threadIdx.x) * J.ldo + J.col0;
      if (vec_out) {
#pragma unroll
        for (int o4 = 0; o4 < NO / 4; ++o4)
          if (4 * o4 < nout) *reinterpret_cast<float4*>(orow + 4 * o4) = make_float4(acc[4 * o4], acc[4 * o4 + 1], acc[4 * o4 + 2], acc[4 * o4 + 3]);
      } else {
#pragma unroll
        for (int o = 0; o < NO; ++o)
          if (o < nout) orow[o] = acc[o];
      }
    }
  }
}

// blocks per job: one 128-row block each, or (when that exceeds the cap) an even share of the cap
static int assign_blocks(const int64_t* n, int njobs, int* first) {
  const int64_t cap = 148 * 16;
  int64_t rb[kMaxApply], tot = 0;
  for (int q = 0; q < njobs; ++q) { rb[q] = (n[q] + kApRows - 1) / kApRows; if (rb[q] < 1) rb[q] = 1; tot += rb[q]; }
  const int64_t it = (tot + cap - 1) / cap;
  first[0] = 0;
  for (int q = 0; q < njobs; ++q) first[q + 1] = first[q] + (int)((rb[q] + it - 1) / it);
  return first[njobs];
}

template <int W, int NO, bool kIn2>
static void apply_small_t(ApplyJobs& jobs, cudaStream_t st) {
  constexpr int smem = ((kIn2 ? 4 : 2) * kApRows * ap_ld(W) + 2 * W * NO) * (int)sizeof(float);
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_apply_small<W, NO, kIn2>, smem, attr);
  int64_t n[kMaxApply];
  for (int q = 0; q < jobs.n; ++q) n[q] = jobs.j[q].n;
  const int grid = assign_blocks(n, jobs.n, jobs.first);
  launch_pdl(k_apply_small<W, NO, kIn2>, grid, kApRows, smem, st, jobs);
}
// tall single-input jobs (>= 64K rows) go in a launch of their own with half the staging memory;
// otherwise one launch for all (a launch costs more than the occupancy buys on short panels)
template <int W, int NO>
static void apply_small_t(ApplyJobs& jobs, cudaStream_t st) {
  ApplyJobs one{}, two{};
  int64_t tall1 = 0;
  for (int q = 0; q < jobs.n; ++q) {
    if (jobs.j[q].IN2) {
      two.j[two.n++] = jobs.j[q];
    } else {
      one.j[one.n++] = jobs.j[q];
      tall1 = jobs.j[q].n > tall1 ? jobs.j[q].n : tall1;
    }
  }
  if (two.n == 0) return apply_small_t<W, NO, false>(jobs, st);
  if (one.n == 0 || tall1 < 65536) return apply_small_t<W, NO, true>(jobs, st);
  apply_small_t<W, NO, false>(one, st);
  apply_small_t<W, NO, true>(two, st);
  ++launch_counter();
}
// NO = W - 8 covers the factor assembly for the default oversampling (r + 5 <= W = roundup(r + p, 8)
// puts roundup(r, 8) at W - 8 or W); everything else computes all W columns (instantiations and
// build time stay bounded)
template <int W>
static void apply_small_w(ApplyJobs& jobs, int no, cudaStream_t st) {
  if constexpr (W >= 16) {
    if (no <= W - 8) return apply_small_t<W, W - 8>(jobs, st);
  }
  apply_small_t<W, W>(jobs, st);
}

void launch_apply_jobs(const ApplyJobs& in, int W, cudaStream_t st) {
  ApplyJobs jobs{};
  for (int q = 0; q < in.n; ++q)
    if (in.j[q].n > 0 && in.j[q].nout > 0) jobs.j[jobs.n++] = in.j[q];
  if (jobs.n == 0) return;
  int no = 0;
  for (int q = 0; q < jobs.n; ++q) no = jobs.j[q].nout > no ? jobs.j[q].nout : no;
#define AS_CASE(w) case w: apply_small_w<w>(jobs, no, st); break;
  switch (W) { AS_CASE(8) AS_CASE(16) AS_CASE(24) AS_CASE(32) AS_CASE(40) AS_CASE(48) AS_CASE(56) AS_CASE(64) default: break; }
#undef AS_CASE
  ++launch_counter();
}

void launch_apply_small(const float* IN1, const float* S1, const float* IN2, const float* S2, int64_t n, int W,
                        int ldS, int nout, float* OUT, int64_t ldo, int col0, cudaStream_t st) {
  ApplyJobs j{};
  j.n = 1;
  j.j[0] = ApplyJob{IN1, S1, IN2, S2, n, ldS, nout, OUT, ldo, col0, 0};
  launch_apply_jobs(j, W, st);
}

// ------------------------------------------------------------ factor assembly
// One side of the assembly in one pass over its rows (see AsmJob): both inputs staged per 128-row
// tile (cp.async double buffer), the row's two halves in registers, the tile's output rows staged in
// shared memory and written as fp32 and as the bf16 hi / lo operands of K8 with coalesced 16-byte
// stores.  This replaces two single-product jobs (each writing half of every row) plus the
// k_split_bf16 pass that re-read the fp32 factor.  Same products, same summation order as
// k_apply_small; same bf16 split as k_split_bf16.
LRQMM_DEV void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(x - __uint_as_float(hi)));
}
LRQMM_DEV void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// W = 32 staging without padding: row r's 16-byte chunk c at chunk c ^ (r & 7) of the 128-byte row, so
// the MMA fragment reads (8 rows x 4 columns per k-tile) hit 32 distinct banks; 25 % less shared
// memory than the W + 4 padded rows (k_assemble: three resident blocks per SM instead of two)
template <int W>
LRQMM_DEV int swz_at(int row, int col) {
  return row * W + ((((col >> 2) ^ (row & 7)) << 2) | (col & 3));
}
template <int W>
LRQMM_DEV void stage_rows_swz(const float* __restrict__ src, int64_t i0, int nr, float* sm) {
  const float4* s4 = reinterpret_cast<const float4*>(src + i0 * W);
#pragma unroll
  for (int u = 0; u < W / 4; ++u) {
    const int e = threadIdx.x + u * kApRows;
    if (e < nr * (W / 4)) {
      const uint32_t dst = smem_u32(sm + swz_at<W>(e / (W / 4), 4 * (e % (W / 4))));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(s4 + e) : "memory");
    }
  }
}

// C[16 x 8 NT] (+)= A[16 x W] S[W x 8 NT] for the two 16-row m-tiles of a warp, 3xTF32 (hi.hi + hi.lo
// + lo.hi, fp32 accumulation: fp32-level accuracy, the products' lo.lo term below fp32 rounding).
// A rows from the staged tile (ld L), S from shared memory (ld NO).  Fragments of
// mma.m16n8k8.tf32: lane = 4 g + t; A (g, t), (g + 8, t), (g, t + 4), (g + 8, t + 4); B (t, g),
// (t + 4, g); C (g, 2t), (g, 2t + 1), (g + 8, 2t), (g + 8, 2t + 1).
template <int W, int NO, bool kSwz>
LRQMM_DEV void asm_mma(float (&c)[2][NO / 8][4], const float* sin, int rbase, const float* S, int lane) {
  constexpr int L = ap_ld(W);
  const int g = lane >> 2, t = lane & 3;
  auto at = [&](int row, int col) { return kSwz ? sin[swz_at<W>(row, col)] : sin[row * L + col]; };
#pragma unroll
  for (int kt = 0; kt < W / 8; ++kt) {
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r0 = rbase + 16 * mt + g, c0 = 8 * kt + t;
      tf32_split(at(r0, c0), ah[mt][0], al[mt][0]);
      tf32_split(at(r0 + 8, c0), ah[mt][1], al[mt][1]);
      tf32_split(at(r0, c0 + 4), ah[mt][2], al[mt][2]);
      tf32_split(at(r0 + 8, c0 + 4), ah[mt][3], al[mt][3]);
    }
#pragma unroll
    for (int nt = 0; nt < NO / 8; ++nt) {
      uint32_t bh0, bl0, bh1, bl1;
      tf32_split(S[(8 * kt + t) * NO + 8 * nt + g], bh0, bl0);
      tf32_split(S[(8 * kt + t + 4) * NO + 8 * nt + g], bh1, bl1);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        mma_tf32(c[mt][nt], al[mt], bh0, bh1);
        mma_tf32(c[mt][nt], ah[mt], bl0, bl1);
        mma_tf32(c[mt][nt], ah[mt], bh0, bh1);
      }
    }
  }
}

// kTc (W <= 32, NO % 8 == 0): the products on the tensor cores (3xTF32 mma.sync, warp w owns rows
// 32 w .. 32 w + 31 of the tile); else fp32 FFMA, one row per thread
template <int W, int NO, bool kTc>
__global__ void __launch_bounds__(kApRows) k_assemble(const __grid_constant__ AsmJobs jobs) {
  ::lrqmm::pdl_enter();
  constexpr int L = ap_ld(W);
  extern __shared__ __align__(16) float asm_sm[];
  const int q = (jobs.n > 1 && (int)blockIdx.x >= jobs.first[1]) ? 1 : 0;
  const AsmJob& J = jobs.j[q];
  const int b0 = jobs.first[q], nb = jobs.first[q + 1] - b0;
  float* s1 = asm_sm;
  float* s2 = s1 + W * NO;
  float* s3 = s2 + W * NO;
  // kSwz (tensor-core path at W = 32): unpadded swizzled rows, and the output rows staged in the
  // tile's own input slot once its MMAs are done (no separate output buffer)
  constexpr bool kSwz = kTc && W == 32 && NO <= 24;  // kApRows x (2 NO + 4) output rows fit one slot
  constexpr int LS = kSwz ? W : L;
  float* sin_base = s3 + W * NO;  // 2 buffers x (IN1, IN2) x kApRows x LS
  constexpr int kSlot = 2 * kApRows * LS;
  float* sout_own = sin_base + 2 * kSlot;  // kApRows x (2 nout + 4) output rows (not kSwz)
  const int nout = J.nout;
  const int kin = J.kin > 0 && J.kin < W ? J.kin : W;
  const bool has3 = J.S3 != nullptr;
  for (int e = threadIdx.x; e < W * NO; e += blockDim.x) {
    const int c = e / NO, o = e % NO;
    s1[e] = o < nout ? J.S1[c * J.ldS + o] : 0.f;
    s2[e] = o < nout ? J.S2[c * J.ldS + o] : 0.f;
    s3[e] = (has3 && o < nout) ? J.S3[c * J.ldS + o] : 0.f;
  }
  const int64_t n = J.n;
  const int64_t step = (int64_t)nb * kApRows;
  auto stage = [&](int64_t i0, int slot) {
    if (i0 < n) {
      const int nr = (int)(n - i0 < kApRows ? n - i0 : kApRows);
      if constexpr (kSwz) {
        stage_rows_swz<W>(J.IN1, i0, nr, sin_base + slot * kSlot);
        stage_rows_swz<W>(J.IN2, i0, nr, sin_base + slot * kSlot + kApRows * LS);
      } else {
        stage_rows_async<W>(J.IN1, i0, nr, sin_base + slot * kSlot);
        stage_rows_async<W>(J.IN2, i0, nr, sin_base + slot * kSlot + kApRows * LS);
      }
    }
    cp_async_commit();
  };
  const int64_t first = (int64_t)(blockIdx.x - b0) * kApRows;
  stage(first, 0);
  stage(first + step, 1);
  int it = 0;
  for (int64_t i0 = first; i0 < n; i0 += step, ++it) {
    const int nr = (int)(n - i0 < kApRows ? n - i0 : kApRows);
    float* sin1 = sin_base + (it & 1) * kSlot;
    const float* sin2 = sin1 + kApRows * LS;
    float* sout = kSwz ? sin1 : sout_own;
    cp_async_wait<1>();
    __syncthreads();
    // the tile's rows go through shared memory (row stride 2 nout + 4 floats: an odd number of
    // 16-byte units), then out with coalesced copies: the tile is one contiguous block of L (ld =
    // 2 nout) and of each bf16 operand (ld 64)
    const int ow = 2 * nout, ostr = ow + 4;
    if constexpr (kTc) {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      float c1[2][NO / 8][4] = {}, c2[2][NO / 8][4] = {};
      asm_mma<W, NO, kSwz>(c1, sin1, 32 * warp, s1, lane);
      if (has3) asm_mma<W, NO, kSwz>(c1, sin2, 32 * warp, s3, lane);
      asm_mma<W, NO, kSwz>(c2, sin2, 32 * warp, s2, lane);
      __syncthreads();  // every row of this buffer has been read
      if (!kSwz) stage(i0 + 2 * step, it & 1);  // kSwz: the slot holds the output rows first
      const int g = lane >> 2, t = lane & 3;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NO / 8; ++nt) {
          const int col = 8 * nt + 2 * t;
          if (col < nout) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float* orow = sout + (32 * warp + 16 * mt + g + 8 * h) * ostr;
              *reinterpret_cast<float2*>(orow + col) = make_float2(c1[mt][nt][2 * h], c1[mt][nt][2 * h + 1]);
              *reinterpret_cast<float2*>(orow + nout + col) = make_float2(c2[mt][nt][2 * h], c2[mt][nt][2 * h + 1]);
            }
          }
        }
    } else {
      float acc1[NO], acc2[NO];
#pragma unroll
      for (int o = 0; o < NO; ++o) acc1[o] = acc2[o] = 0.f;
      if (threadIdx.x < nr) {
#pragma unroll(W <= 32 ? W / 4 : 2)
        for (int c4 = 0; c4 < W / 4; ++c4) {
          if (4 * c4 >= kin) break;  // zero-padded sketch columns contribute nothing
          const float4 v = *reinterpret_cast<const float4*>(sin1 + threadIdx.x * L + 4 * c4);
          const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int o = 0; o < NO; ++o) acc1[o] = fmaf(xs[j], s1[(4 * c4 + j) * NO + o], acc1[o]);
        }
#pragma unroll(W <= 32 ? W / 4 : 2)
        for (int c4 = 0; c4 < W / 4; ++c4) {
          if (4 * c4 >= kin) break;
          const float4 v = *reinterpret_cast<const float4*>(sin2 + threadIdx.x * L + 4 * c4);
          const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (has3) {
#pragma unroll
              for (int o = 0; o < NO; ++o) acc1[o] = fmaf(xs[j], s3[(4 * c4 + j) * NO + o], acc1[o]);
            }
#pragma unroll
            for (int o = 0; o < NO; ++o) acc2[o] = fmaf(xs[j], s2[(4 * c4 + j) * NO + o], acc2[o]);
          }
        }
      }
      __syncthreads();  // every row of this buffer has been read: stage the tile after next into it
      stage(i0 + 2 * step, it & 1);
      if (threadIdx.x < nr) {
        float* orow = sout + threadIdx.x * ostr;
#pragma unroll
        for (int o4 = 0; o4 < NO / 4; ++o4)
          if (4 * o4 < nout) {
            *reinterpret_cast<float4*>(orow + 4 * o4) = make_float4(acc1[4 * o4], acc1[4 * o4 + 1], acc1[4 * o4 + 2], acc1[4 * o4 + 3]);
            *reinterpret_cast<float4*>(orow + nout + 4 * o4) = make_float4(acc2[4 * o4], acc2[4 * o4 + 1], acc2[4 * o4 + 2], acc2[4 * o4 + 3]);
          }
      }
    }
    __syncthreads();
    {
      float4* dst = reinterpret_cast<float4*>(J.OUT + i0 * J.ldo);
      const int nq = nr * ow / 4, qpr = ow / 4;
      for (int e = threadIdx.x; e < nq; e += kApRows)
        dst[e] = *reinterpret_cast<const float4*>(sout + (e / qpr) * ostr + 4 * (e % qpr));
    }
    if (J.hi) {
      uint4* hd = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(J.hi) + i0 * 64);
      uint4* ld = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(J.lo) + i0 * 64);
      for (int e = threadIdx.x; e < nr * 8; e += kApRows) {  // 8-column groups, as k_split_bf16
        const int row = e >> 3, c0 = (e & 7) * 8;
        float x[8];
        if (c0 < ow) {  // ow % 8 == 0 when nout % 4 == 0
          const float4 v0 = *reinterpret_cast<const float4*>(sout + row * ostr + c0);
          const float4 v1 = *reinterpret_cast<const float4*>(sout + row * ostr + c0 + 4);
          x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w; x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = 0.f;
        }
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * u], x[2 * u + 1]);
          const float2 hf = __bfloat1622float2(h2);
          const __nv_bfloat162 l2 = __floats2bfloat162_rn(x[2 * u] - hf.x, x[2 * u + 1] - hf.y);
          hw[u] = *reinterpret_cast<const uint32_t*>(&h2);
          lw[u] = *reinterpret_cast<const uint32_t*>(&l2);
        }
        hd[e] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        ld[e] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    }
    if constexpr (kSwz) {  // the output rows are out of the slot: stage the tile after next into it
      __syncthreads();
      stage(i0 + 2 * step, it & 1);
    }
  }
}

template <int W, int NO>
static void assemble_t(AsmJobs& jobs, cudaStream_t st) {
  constexpr bool kTc = W <= 32 && NO % 8 == 0 && W % 8 == 0;
  constexpr bool kSwz = kTc && W == 32 && NO <= 24;  // as in the kernel: 74.8 KB, three blocks per SM
  constexpr int smem = (kSwz ? 4 * kApRows * W + 3 * W * NO
                             : 4 * kApRows * ap_ld(W) + 3 * W * NO + kApRows * (2 * NO + 4)) * (int)sizeof(float);
  static_assert(!kSwz || kApRows * (2 * NO + 4) <= 2 * kApRows * W, "output rows fit one staging slot");
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_assemble<W, NO, kTc>, smem, attr);
  int64_t n[kMaxApply] = {};
  for (int q = 0; q < jobs.n; ++q) n[q] = jobs.j[q].n;
  int first[kMaxApply + 1];
  const int grid = assign_blocks(n, jobs.n, first);
  for (int q = 0; q <= jobs.n; ++q) jobs.first[q] = first[q];
  launch_pdl(k_assemble<W, NO, kTc>, grid, kApRows, smem, st, jobs);
}
template <int W>
static void assemble_w(AsmJobs& jobs, int no, cudaStream_t st) {
  if constexpr (W >= 16) {
    if (no <= W - 8) return assemble_t<W, W - 8>(jobs, st);
  }
  assemble_t<W, W>(jobs, st);
}
void launch_assemble(AsmJobs& jobs, int W, cudaStream_t st) {
  int no = 0;
  for (int q = 0; q < jobs.n; ++q) no = jobs.j[q].nout > no ? jobs.j[q].nout : no;
  if (jobs.n == 0 || no == 0) return;
#define AW_CASE(w) case w: assemble_w<w>(jobs, no, st); break;
  switch (W) { AW_CASE(8) AW_CASE(16) AW_CASE(24) AW_CASE(32) default: break; }  // W <= 32 (the caller's contract)
#undef AW_CASE
  ++launch_counter();
}

// OUT = IN S with S in fp64 and fp64 accumulation (orthonormalisation: keeps Q orthonormal to
// fp32 rounding instead of cond(IN) * eps32).  Same staging as above; one launch for both sides.
// Same product on the fp64 tensor cores (W <= 32): Q = Y T with mma.sync.m8n8k4.f64 (DMMA). A warp
// owns 32 rows of the staged 128-row tile as four 8-row slabs; T's fragments (B: lane l holds
// T[4 kt + l % 4][8 nt + l / 4]) stay in registers for the whole launch, the A fragment of a slab
// (lane l holds Y[r0 + l / 4][4 kt + l % 4], converted to fp64 once) comes from shared memory
// (conflict-free for L = W + 4), and only the k-tiles / n-tiles that reach the live columns run.
// fp64 products and accumulation as the FMA form (a different, fixed summation order).  Outputs:
// lane l holds Q[r0 + l / 4][8 nt + 2 (l % 4) + {0, 1}]; column maxima as in k_apply64.
template <int W>
__global__ void __launch_bounds__(kApRows, 4) k_apply64_tc(const __grid_constant__ Apply64Jobs jobs) {
  ::lrqmm::pdl_enter();
  constexpr int L = ap_ld(W);
  constexpr int KT = W / 4, NT = W / 8;
  extern __shared__ __align__(16) double apsm64[];
  const int q = (jobs.n > 1 && (int)blockIdx.x >= jobs.first[1]) ? 1 : 0;
  const Apply64Job& J = jobs.j[q];
  const int b0 = jobs.first[q], nb = jobs.first[q + 1] - b0;
  float* sin_base = reinterpret_cast<float*>(apsm64 + W * W);  // 2 x kApRows x L (cp.async double buffer)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kin = J.kin > 0 && J.kin < W ? J.kin : W;
  const int kt_live = (kin + 3) / 4, nt_live = (kin + 7) / 8;
  double bfr[KT][NT];
#pragma unroll
  for (int kt = 0; kt < KT; ++kt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bfr[kt][nt] = J.S[(4 * kt + (lane & 3)) * W + 8 * nt + (lane >> 2)];
  __shared__ unsigned bmax[64];
  if (threadIdx.x < 64) bmax[threadIdx.x] = 0u;
  float run[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) run[nt][0] = run[nt][1] = 0.f;
  const int64_t n = J.n;
  const int64_t step = (int64_t)nb * kApRows;
  auto stage = [&](int64_t i0, int slot) {
    if (i0 < n) stage_rows_async<W>(J.IN, i0, (int)(n - i0 < kApRows ? n - i0 : kApRows), sin_base + slot * kApRows * L);
    cp_async_commit();
  };
  const int64_t first = (int64_t)(blockIdx.x - b0) * kApRows;
  stage(first, 0);
  stage(first + step, 1);
  int it = 0;
  for (int64_t i0 = first; i0 < n; i0 += step, ++it) {
    const float* sin = sin_base + (it & 1) * kApRows * L;
    cp_async_wait<1>();  // this tile's group has landed (the next one may still be in flight)
    __syncthreads();
    // one 8-row slab at a time, its outputs stored from registers at once (8 fp64 accumulators
    // live instead of 32: four resident blocks per SM instead of three)
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      double acc[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
      const float* arow = sin + (warp * 32 + sl * 8 + (lane >> 2)) * L + (lane & 3);
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        if (kt >= kt_live) break;  // zero-padded sketch columns
        const double a = (double)arow[4 * kt];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (nt >= nt_live) break;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[nt][0]), "+d"(acc[nt][1])
                       : "d"(a), "d"(bfr[kt][nt]));
        }
      }
      const int64_t row = i0 + warp * 32 + sl * 8 + (lane >> 2);
      const bool ok = row < n;
      const float cs = (J.cscale && ok) ? J.cscale[row] : 1.f;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float v0 = (float)acc[nt][0], v1 = (float)acc[nt][1];
        if (ok) *reinterpret_cast<float2*>(J.OUT + row * W + 8 * nt + 2 * (lane & 3)) = make_float2(v0, v1);
        if (J.cmax) {  // same fp32 product as the next pass's B image; per-lane running maxima
          run[nt][0] = fmaxf(run[nt][0], ok ? fabsf(v0 * cs) : 0.f);
          run[nt][1] = fmaxf(run[nt][1], ok ? fabsf(v1 * cs) : 0.f);
        }
      }
    }
    __syncthreads();  // every row of this buffer has been read: stage the tile after next into it
    stage(i0 + 2 * step, it & 1);
  }
  if (J.cmax) {
    // lanes with the same lane & 3 hold the same columns: one shuffle reduction per block (max is
    // exact in any order), not one per tile and row slice
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        run[nt][0] = fmaxf(run[nt][0], __shfl_xor_sync(0xffffffffu, run[nt][0], o));
        run[nt][1] = fmaxf(run[nt][1], __shfl_xor_sync(0xffffffffu, run[nt][1], o));
      }
    __syncthreads();
    if (lane < 4)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (run[nt][h] > 0.f) atomicMax(&bmax[8 * nt + 2 * lane + h], __float_as_uint(run[nt][h]));
    __syncthreads();
    if (threadIdx.x < W && bmax[threadIdx.x]) atomicMax(J.cmax + threadIdx.x, bmax[threadIdx.x]);
  }
}

// NO: outputs computed per row (the rest of the W are zero: columns >= kin of S are zero); inputs
// c >= kin are skipped (zero-padded sketch columns).
template <int W, int NO>
__global__ void __launch_bounds__(kApRows) k_apply64(const __grid_constant__ Apply64Jobs jobs) {
  ::lrqmm::pdl_enter();
  constexpr int L = ap_ld(W);
  extern __shared__ __align__(16) double apsm64[];
  const int q = (jobs.n > 1 && (int)blockIdx.x >= jobs.first[1]) ? 1 : 0;
  const Apply64Job& J = jobs.j[q];
  const int b0 = jobs.first[q], nb = jobs.first[q + 1] - b0;
  double* s = apsm64;                                           // W x W
  float* sin_base = reinterpret_cast<float*>(apsm64 + W * W);   // 2 x kApRows x L (cp.async double buffer)
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) s[e] = J.S[e];
  const int kin = J.kin > 0 && J.kin < W ? J.kin : W;
  unsigned run[(W + 31) / 32];  // lane c: running column max of column c (+32)
#pragma unroll
  for (int u = 0; u < (W + 31) / 32; ++u) run[u] = 0u;
  __shared__ unsigned bmax[64];
  if (threadIdx.x < 64) bmax[threadIdx.x] = 0u;
  const int64_t n = J.n;
  const int64_t step = (int64_t)nb * kApRows;
  auto stage = [&](int64_t i0, int slot) {
    if (i0 < n) stage_rows_async<W>(J.IN, i0, (int)(n - i0 < kApRows ? n - i0 : kApRows), sin_base + slot * kApRows * L);
    cp_async_commit();
  };
  const int64_t first = (int64_t)(blockIdx.x - b0) * kApRows;
  stage(first, 0);
  stage(first + step, 1);
  int it = 0;
  for (int64_t i0 = first; i0 < n; i0 += step, ++it) {
    const int nr = (int)(n - i0 < kApRows ? n - i0 : kApRows);
    const float* sin = sin_base + (it & 1) * kApRows * L;
    cp_async_wait<1>();  // this tile's group has landed (the next one may still be in flight)
    __syncthreads();
    double acc[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) acc[o] = 0.0;
    if (threadIdx.x < nr) {
#pragma unroll(W <= 32 ? W / 4 : 2)  // bounded unrolling for the wide sketches (build time)
      for (int c4 = 0; c4 < W / 4; ++c4) {
        if (4 * c4 >= kin) break;  // zero-padded sketch columns contribute nothing
        const float4 v = *reinterpret_cast<const float4*>(sin + threadIdx.x * L + 4 * c4);
        const double xs[4] = {(double)v.x, (double)v.y, (double)v.z, (double)v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int o = 0; o < NO; ++o) acc[o] = fma(xs[j], s[(4 * c4 + j) * W + o], acc[o]);
      }
    }
    __syncthreads();  // every row of this buffer has been read: stage the tile after next into it
    stage(i0 + 2 * step, it & 1);
    if (threadIdx.x < nr) {  // outputs straight from registers (16-byte stores of this thread's row)
      float4* orow = reinterpret_cast<float4*>(J.OUT + (i0 + threadIdx.x) * W);
#pragma unroll
      for (int o4 = 0; o4 < W / 4; ++o4)
        orow[o4] = 4 * o4 < NO ? make_float4((float)acc[4 * o4], (float)acc[4 * o4 + 1], (float)acc[4 * o4 + 2],
                                             (float)acc[4 * o4 + 3])
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (J.cmax) {
      // column maxima of |OUT * cscale| for the next pass's B image (same fp32 product as there);
      // columns >= NO are zero
      const float cs = (J.cscale && threadIdx.x < nr) ? J.cscale[i0 + threadIdx.x] : 1.f;
#pragma unroll
      for (int o = 0; o < NO; ++o) {
        const unsigned b = threadIdx.x < nr ? __float_as_uint(fabsf((float)acc[o] * cs)) : 0u;
        const unsigned m = __reduce_max_sync(0xffffffffu, b);
        if ((threadIdx.x & 31) == (o & 31)) run[o >> 5] = max(run[o >> 5], m);
      }
    }
  }
  if (J.cmax) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < (W + 31) / 32; ++u)
      if (32 * u + lane < W && run[u]) atomicMax(&bmax[32 * u + lane], run[u]);
    __syncthreads();
    if (threadIdx.x < W && bmax[threadIdx.x]) atomicMax(J.cmax + threadIdx.x, bmax[threadIdx.x]);
  }
}

template <int W, int NO>
static void apply64_t(Apply64Jobs& jobs, cudaStream_t st) {
  constexpr int smem = W * W * (int)sizeof(double) + 2 * kApRows * ap_ld(W) * (int)sizeof(float);
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_apply64<W, NO>, smem, attr);
  int64_t n[2] = {jobs.j[0].n, jobs.n > 1 ? jobs.j[1].n : 0};
  const int grid = assign_blocks(n, jobs.n, jobs.first);
  launch_pdl(k_apply64<W, NO>, grid, kApRows, smem, st, jobs);
}
// NO = W - 4 when every job's live columns fit (W = roundup(r + p, 8): the default oversampling
// leaves 3..7 zero columns), else W
template <int W>
static void apply64_tc_t(Apply64Jobs& jobs, cudaStream_t st) {
  constexpr int smem = W * W * (int)sizeof(double) + 2 * kApRows * ap_ld(W) * (int)sizeof(float);
  static std::atomic<unsigned> attr{0};
  ensure_smem(k_apply64_tc<W>, smem, attr);
  int64_t n[2] = {jobs.j[0].n, jobs.n > 1 ? jobs.j[1].n : 0};
  const int grid = assign_blocks(n, jobs.n, jobs.first);
  launch_pdl(k_apply64_tc<W>, grid, kApRows, smem, st, jobs);
}
template <int W>
static void apply64_w(Apply64Jobs& jobs, cudaStream_t st) {
  static const bool fma_form = getenv("LRQMM_APPLY64_FMA") != nullptr;  // A/B of the two forms
  if constexpr (W <= 32) {
    if (!fma_form) return apply64_tc_t<W>(jobs, st);
  }
  int kin = 0;
  for (int q = 0; q < jobs.n; ++q) kin = max(kin, jobs.j[q].kin > 0 ? jobs.j[q].kin : W);
  if constexpr (W >= 8) {
    if (kin <= W - 4) return apply64_t<W, W - 4>(jobs, st);
  }
  apply64_t<W, W>(jobs, st);
}

void launch_apply64_jobs(const Apply64Jobs& in, int W, cudaStream_t st) {
  Apply64Jobs jobs{};
  for (int q = 0; q < in.n; ++q)
    if (in.j[q].n > 0) jobs.j[jobs.n++] = in.j[q];
  if (jobs.n == 0) return;
#define A64_CASE(w) case w: apply64_w<w>(jobs, st); break;
  switch (W) { A64_CASE(8) A64_CASE(16) A64_CASE(24) A64_CASE(32) A64_CASE(40) A64_CASE(48) A64_CASE(56) A64_CASE(64) default: break; }
#undef A64_CASE
  ++launch_counter();
}


// Omega (K x kk, caller layout, ld ldo) -> the handle's zero-padded K x W copy, plus the column
// maxima of |Omega| (float bits; cmax zeroed beforehand) for the S1 pass's B image, so that prep
// needs no reduction phase of its own.  Thread = (row lane, column c); one atomicMax per column
// per block (order-independent: deterministic).
__global__ void __launch_bounds__(256) k_copy_omega(const float* __restrict__ src, int64_t ldo, int kk, int64_t K, int W,
                                                    float* __restrict__ dst, unsigned* __restrict__ cmax,
                                                    int* __restrict__ err_flag) {
  ::lrqmm::pdl_enter();
  __shared__ unsigned bm[64];
  if (threadIdx.x < 64) bm[threadIdx.x] = 0u;
  __syncthreads();
  const int rpb = blockDim.x / W;  // rows per block iteration
  const int c = threadIdx.x % W, r0 = threadIdx.x / W;
  unsigned m = 0u;
  if (r0 < rpb)
    for (int64_t row = (int64_t)blockIdx.x * rpb + r0; row < K; row += (int64_t)gridDim.x * rpb) {
      const float v = c < kk ? src[row * ldo + c] : 0.f;
      dst[row * W + c] = v;
      // a NaN (0x7fc00000 > every finite |v| as bits) or Inf would own the column maximum and
      // corrupt that column's pass image: flagged instead (LRQMM_ERR_NONFINITE at lrqmm_sync)
      if (!isfinite(v)) atomicOr(err_flag, 1);
      m = max(m, __float_as_uint(fabsf(v)));
    }
  if (r0 < rpb && m) atomicMax(&bm[c], m);
  __syncthreads();
  if (threadIdx.x < W && bm[threadIdx.x]) atomicMax(cmax + threadIdx.x, bm[threadIdx.x]);
}

void launch_copy_omega(const float* src, int64_t ldo, int kk, int64_t K, int W, float* dst, unsigned* cmax,
                       int* err_flag, cudaStream_t st) {
  cudaMemsetAsync(cmax, 0, 64 * sizeof(unsigned), st);
  if (K == 0 || W == 0) return;
  const int rpb = 256 / W;
  int64_t g = (K + rpb - 1) / rpb;
  if (g > 148 * 4) g = 148 * 4;
  launch_pdl(k_copy_omega, (int)g, 256, 0, st, src, ldo, kk, K, W, dst, cmax, err_flag);
  ++launch_counter();
}

__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  ::lrqmm::pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)in[i];
}
__global__ void k_flip_lsb(float* p) { *p = __uint_as_float(__float_as_uint(*p) ^ 1u); }
void launch_flip_lsb(float* p, cudaStream_t st) {
  k_flip_lsb<<<1, 1, 0, st>>>(p);
  ++launch_counter();
}

void launch_f64_to_f32(const double* in, float* out, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  launch_pdl(k_f64_to_f32, clamp_grid((n + 255) / 256), 256, 0, st, in, out, n);
  ++launch_counter();
}


}  // namespace lrqmm
