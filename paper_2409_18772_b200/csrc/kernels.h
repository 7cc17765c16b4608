// Host-side launch interfaces of the liblrqmm kernels (internal; not part of the C ABI).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>
#include <utility>

namespace lrqmm {

// Kernel launches are counted per handle (gpu_launches evidence for the bench): every C-ABI entry
// point that launches installs its handle's counter for the calling thread (CounterScope), and the
// launchers increment launch_counter().  Launches outside any handle (test hooks) go to a
// thread-local fallback.
inline int64_t*& launch_counter_slot() {
  static thread_local int64_t* p = nullptr;
  return p;
}
inline int64_t& launch_counter() {
  static thread_local int64_t fallback = 0;
  int64_t* p = launch_counter_slot();
  return p ? *p : fallback;
}
struct CounterScope {
  int64_t* prev;
  explicit CounterScope(int64_t* c) : prev(launch_counter_slot()) { launch_counter_slot() = c; }
  ~CounterScope() { launch_counter_slot() = prev; }
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the CURRENT device's copy of the
// kernel: remember it per device ordinal (bit d of `done`), set before the bit is published.
template <typename K>
inline void ensure_smem(K* kernel, int bytes, std::atomic<unsigned>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = 1u << (dev & 31);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_release);
  }
}
// SM count of the current device (cached per ordinal)
inline int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (v <= 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    cache[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}

// PDL on (LRQMM_NO_PDL unset): eager launches made through launch_pdl() carry
// cudaLaunchAttributeProgrammaticStreamSerialization; the kernel must begin with pdl_enter().
// Launches being captured into a graph do not: the graph already hides launch latency, and the
// early-resident dependents then only compete for SMs (c2 rsvd_residual 246 -> 264 us with PDL
// edges in the graph; eager, multi-rank path 289 -> 261 us with PDL; tools/ab_pdl.sh).
inline bool pdl_enabled() {
  static const bool on = getenv("LRQMM_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (pdl_enabled()) cudaStreamIsCapturing(st, &cap);
  cfg.numAttrs = (pdl_enabled() && cap == cudaStreamCaptureStatusNone) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

enum { kRoundFloor = 0, kRoundTrunc = 1, kRoundNearest = 2 };

// ---------------------------------------------------------------- K1 quantize
struct QuantArgs {
  const float* X;
  int64_t ldx;
  int64_t rows;
  int K, Kp, qmax, mode;
  int8_t* codes;          // rows x Kp
  float* lam;             // rows (written unless lam_fixed)
  float* inv_lam;         // rows: RN(1/lambda) (written unless lam_fixed)
  const float* lam_fixed; // device scalar (per-tensor mode) or nullptr
  int* err_flag;          // bit 0: non-finite input
  uint8_t* U;             // residual fraction u = lambda x - code as Q15 i = RN(2^15 u) = 256 h + l in two
                          // byte planes: h (int8) at U, l (uint8) at U + uplane; rows x ldu each (or nullptr)
  int64_t ldu;            // multiple of 16, >= K
  int64_t uplane;         // bytes between the h and l planes
};
void launch_quantize(const QuantArgs& a, cudaStream_t st);
// implicit im2col of an NHWC convolution input: rows (b, ho, wo), K = kh kw C
struct ConvGeom {
  int batch, H, W, C, kh, kw, sh, sw, ph, pw, dh, dw, Ho, Wo;
};
void launch_quantize_im2col(const QuantArgs& a, const ConvGeom& g, cudaStream_t st);
// QT: R = fp32(X - code / lambda) (rows x K, dense), fp64 arithmetic as the oracle
void launch_resid_f32(const float* X, int64_t ldx, const int8_t* codes, int Kp, const float* lam, int64_t rows, int K,
                      float* R, cudaStream_t st);
void launch_tensor_scale(const float* X, int64_t ldx, int64_t rows, int K, int qmax, float* row_amax,
                         float* lam_rows, float* inv_rows, float* lam_scalar, int* err_flag, cudaStream_t st);

// ------------------------------------------------- K2/K3 skinny residual products
// The passes stream the residual fraction u = lambda x - code written by K1 (R = u / lambda,
// Alg. 2) and, for the cross products, the codes (X~ = code / lambda, line 352).
// u is stored as Q15: i = clamp(RN(u * 2^15), +-32767) (|u| < 1 for every rounding mode;
// |i / 2^15 - u| <= 2^-16, 2^-15 where u rounds past the clamp), split into the bytes
// i = 256 h + l (h = i >> 8 signed, l = i & 255 unsigned) stored as two planes, so the RSVD
// passes feed them to kind::i8 MMAs straight from TMA (reading #28).  2 B per element.
constexpr float kUScale = 32768.f;
struct SideView {
  const uint8_t* Uh;     // rows x ldu int8 (h)
  const uint8_t* Ul;     // rows x ldu uint8 (l)
  int64_t ldu;
  int64_t rows;
  int K;
  const int8_t* codes;   // rows x Kp
  int Kp;
  const float* lam;
  const float* inv_lam;  // RN(1/lambda)
};
// tcgen05 kind::tf32 (3-term split) passes, deterministic split-K partials; return the split count.
// With reduce1 == false and > 1 splits, OUT1 stays as partials at `partial` (consumed by the fused
// Gram kernel).  ROW: OUT1 = R P1 (rows x W); dual (P2 != null): OUT2 = X~ P2.  P is K x W (ld W).
// One RSVD pass over one or two sides in a single launch (skinny_tc.cu launch_tc_pass).
struct TcPassSide {
  SideView view;
  const float* P1;   // ROW/DUAL/COL operand
  const float* P2;   // DUAL/CODES operand
  float* OUT1;
  float* OUT2;
  float* partial;    // split-K partial scratch of this side
  int64_t pe;        // its capacity in floats
  uint8_t* img;      // >= 2 * tc_img_bytes(max(rows, K), W) bytes
  const unsigned* cmax1;  // column maxima (float bits) of |P1 scale| / |P2| from their producer, or nullptr
  const unsigned* cmax2;
  const uint8_t* pimg1;   // prebuilt B image of P1 / P2 (launch_apply_prep), or nullptr: built by the pass
  const uint8_t* pimg2;
  int sm_reserve;         // SMs the pass leaves free (another graph branch's small kernels run there)
};
enum { kPassRow = 0, kPassDual = 1, kPassCol = 2, kPassCodes = 3 };
void launch_tc_pass(int kind, int nsides, const TcPassSide* sides, int W, bool reduce1, int* ns_out, cudaStream_t st);
// Fused pass (W <= 32, skinny_tc.cu): the pass kernel itself reduces its split-K partials (the last
// unit to finish an output block sums the block's partials in split order), forms the fp64 Gram
// G = OUT1^T OUT1 from per-slot partials (two-level fixed-order ticket sums: deterministic), and
// the last CTA of the launch runs the small solver of every side (pivoted CholQR -> T64, or the
// truncation eigensolver -> T, then optionally the cross core of Alg. 2).  B images are
// prebuilt (launch_apply_prep): no prep launch, no reduction launches, no Gram launch.
enum { kSolveNone = 0, kSolveChol = 1, kSolveEig = 2 };
struct PassFuseSide {
  float* fin1;         // final OUT1 (== TcPassSide::OUT1)
  float* fin2;         // final OUT2
  double* G;           // W x W Gram of OUT1 (nullptr: no Gram for this side)
  double* T64;         // kSolveChol output (W x W)
  float* T;            // kSolveEig output (W x W, first r columns)
  int r;
  unsigned* zero[2];   // 64-entry u32 arrays zeroed by the solver CTA (next column-maxima consumers)
  int* blk_cnt;        // >= kFuseMaxSlots zeroed counters
  int* grp_cnt;        // >= 1 + kFuseMaxSlots / 16 zeroed counters
  double* gpart;       // >= (kFuseMaxSlots + kFuseMaxSlots / 16 + 1) x W x W
  const uint8_t* img1; // prebuilt B images (+ their 1 / s_c vectors)
  const float* cinv1;
  const uint8_t* img2;
  const float* cinv2;
};
constexpr int kFuseMaxSlots = 512;
struct PassFuse {
  PassFuseSide s[2];
  int solver;
  int* all_cnt;
  const double* cross_C;  // kSolveEig: if set, VWbM = VWb (VWb^T C VWa) after both eigensolves
  const float* cross_VWa;
  const float* cross_VWb;
  float* cross_out;
  int r;
  unsigned long long* trace;  // optional timing trace (lrqmm_debug_fuse_trace)
};
// false if the fused form does not apply (W > 32, or too many output blocks with splits): the
// caller then runs launch_tc_pass + the separate small kernels
bool launch_tc_pass_fused(int kind, int nsides, const TcPassSide* sides, int W, const PassFuse& f, int* ns_out,
                          cudaStream_t st);
// The prep / apply launch of the fused chain (skinny.cu, cooperative): phase 1 forms every apply
// job's output (Q = Y T64 in fp64, or a zero-padded copy of Omega) and its column maxima; after a
// grid barrier phase 2 writes the B images of the next pass and (optionally) the cross Gram
// C = X1^T X2 (fp64, deterministic ticket sum).
struct ApplyPrepJob {
  int kind;            // 0: OUT = IN T64;  1: OUT = zero-padded copy of Omega (IN, ld ldi, kk columns)
  const float* IN;
  int64_t ldi;
  int kk;
  const double* T64;
  int64_t n;
  float* OUT;          // n x W
  unsigned* cmax;      // column maxima of |OUT * cscale| (zeroed beforehand)
  const float* cscale; // per-row scale or nullptr
};
struct ImgJob {
  const float* P;      // n x W
  const float* scale;  // per-row scale (COL: 1 / lambda) or nullptr
  const unsigned* cmax;
  uint8_t* img;        // nkb k-block images; cinv at img + nkb * image bytes + 256
  int64_t n;
};
struct ApplyPrep {
  ApplyPrepJob a[2];
  int na;
  ImgJob p[4];
  int np;
  const float* X1;     // cross Gram C = X1^T X2 over xn rows (nullptr: none)
  const float* X2;
  int64_t xn;
  double* C;
  double* cpart;       // >= 64 x W x W
  int* ccnt;           // zeroed ticket
};
void launch_apply_prep(const ApplyPrep& ap, int W, int* err_flag /* bit 0: non-finite Omega */, cudaStream_t st);
// 1 / s_c vector of an image built for n reduction rows (tail of the image buffer)
float* img_cinv(uint8_t* img, int64_t n, int W);
// img: scratch for the B operand images + column scales, >= 2 * tc_img_bytes(max(rows, K), W) bytes.
int launch_tc_proj_rows(const SideView& s, const float* P1, float* OUT1, const float* P2, float* OUT2, int W,
                        float* partial, int64_t partial_elems, bool reduce1, uint8_t* img, cudaStream_t st);
// COL: OUT = R^T P; P is rows x W, OUT is K x W.
int launch_tc_proj_cols(const SideView& s, const float* P, float* OUT, int W, float* partial, int64_t partial_elems,
                        bool reduce1, uint8_t* img, cudaStream_t st);
int64_t tc_img_bytes(int64_t n, int W);
// OUT = sum over nsplit partial planes (fixed order), parallel over the n elements
void launch_reduce_splits(const float* part, int nsplit, int64_t n, float* out, cudaStream_t st);
struct ReduceJob {
  const float* part;
  int nsplit;
  int64_t n;
  float* out;
};
struct ReduceJobs {
  ReduceJob j[4];
  int n;
};
// up to 4 reductions (jobs with nsplit <= 1 skipped) in as few launches as possible
void launch_reduce_jobs(const ReduceJobs& jobs, cudaStream_t st);
// OUT = X~ P (rows x W) over the codes only (static-B mode's B~ Q1_A); always fully reduced
int launch_tc_proj_codes(const SideView& s, const float* P, float* OUT, int W, float* partial, int64_t partial_elems,
                         uint8_t* img, cudaStream_t st);

// OUT[i, :] = IN[i, :] S (fp64 S, fp64 accumulation, fp32 out); IN and OUT ld W, S W x W
// multi-job forms (one launch): OUT = IN S per job
struct Apply64Job {
  const float* IN;
  const double* S;
  int64_t n;
  float* OUT;
  unsigned* cmax;       // if set: atomicMax of the float bits of |OUT[i, c] * cscale[i]| per column c
  const float* cscale;  // (zeroed beforehand; cscale nullptr = 1)
  int kin;              // live columns: IN[:, c >= kin] and S[c >= kin, :], S[:, c >= kin] are zero (0: W)
};
struct Apply64Jobs {
  Apply64Job j[2];
  int n;
  int first[3];  // block ranges (set by the launcher)
};
void launch_apply64_jobs(const Apply64Jobs& jobs, int W, cudaStream_t st);
constexpr int kMaxApply = 4;
struct ApplyJob {
  const float* IN1;
  const float* S1;
  const float* IN2;
  const float* S2;
  int64_t n;
  int ldS, nout;
  float* OUT;
  int64_t ldo;
  int col0;
  int kin;  // live input columns: IN1 / IN2[:, c >= kin] are zero (0: W)
};
struct ApplyJobs {
  ApplyJob j[kMaxApply];
  int n;
  int first[kMaxApply + 1];
};
void launch_apply_jobs(const ApplyJobs& jobs, int W, cudaStream_t st);
// The factor assembly of one side in one row pass (Algorithm 2):
//   OUT[i, 0:nout) = IN1 S1 (+ IN2 S3),  OUT[i, nout:2 nout) = IN2 S2   (fp32, ld ldo),
// and, when hi is set, the bf16 hi / lo split of the row for K8 (hi = RN_bf16(x), lo = RN_bf16(x - hi),
// 64 columns per row, zero beyond 2 nout: the layout k_split_bf16 writes).  nout % 4 == 0.
struct AsmJob {
  const float* IN1;
  const float* S1;
  const float* IN2;
  const float* S2;
  const float* S3;  // nullable
  int64_t n;
  int ldS, nout;
  float* OUT;
  int64_t ldo;
  void* hi;  // bf16 [n][64] or null
  void* lo;
  int kin;
};
struct AsmJobs {
  AsmJob j[2];
  int n;
  int first[3];
};
void launch_assemble(AsmJobs& jobs, int W, cudaStream_t st);
// OUT[i, col0 + o] = sum_c IN1[i,c] S1[c,o] (+ sum_c IN2[i,c] S2[c,o]), o < nout; IN ld W, S ld ldS, OUT ld ldo
void launch_apply_small(const float* IN1, const float* S1, const float* IN2, const float* S2, int64_t n, int W,
                        int ldS, int nout, float* OUT, int64_t ldo, int col0, cudaStream_t st);

// ----------------------------------------------------------- K4 small solvers
constexpr int kGramMaxBlocks = 1024;  // Gram partial buffers hold kGramMaxBlocks x W x W doubles
struct GramJob {  // G = Y1^T Y2 (W x W, fp64) over n rows (Y ld W)
  const float* Y1;
  const float* Y2;
  int64_t n;
  double* G;
  double* partial;  // >= kGramMaxBlocks * W * W
  int* counter;     // zero-initialised ticket
};
struct GramJobs {
  GramJob j[2];
  int n;
};
void launch_gram_jobs(const GramJobs& jobs, int W, cudaStream_t st);
struct EigJob {
  const double* G;
  float* T;     // truncation output (fp32)
  double* T64;  // orthonormalising transform output (fp64, applied with fp64 accumulation)
  int r;
};
struct EigJobs {
  EigJob j[2];
  int n;
};
// orth transform (pivoted Cholesky QR, reading #12 threshold): Q = Y T64 has orthonormal columns
void launch_chol_orth(const EigJobs& jobs, int n, cudaStream_t st);
// truncation: T[:, 0:r] = top-r eigenvectors of G (descending), rest 0
void launch_eig_warp(const EigJobs& jobs, int n, cudaStream_t st);
// Fused: Y = sum of nsplit partials (if nsplit > 1), G = Y^T Y (fp64), then mode 0: T64 = CholQR transform,
// mode 1: T = top-r eigenvectors of G, mode 2: G only.  Both sides in one launch.
struct SmallJob {
  float* Y;            // n x W (output when nsplit > 1, input otherwise)
  const float* part;   // nsplit x n x W split partials
  int nsplit;
  int64_t n;
  double* G;
  double* gpart;       // >= kGramMaxBlocks * W * W
  int* counter;
  double* T64;
  float* T;
  int r;
  unsigned* cmax;      // zeroed by the last block (the next apply64 accumulates column maxima into it)
};
struct SmallJobs {
  SmallJob j[2];
  int n;
};
void launch_fused_small(const SmallJobs& jobs, int W, int mode, cudaStream_t st);
// Mab[r x r] = VWb^T C VWa  and  VWbM[n x r] = VWb Mab   (C = Q1_B^T Q1_A, n x n fp64)
void launch_cross_small(const double* C, const float* VWa, const float* VWb, int n, int r, float* VWbM,
                        cudaStream_t st);

// --------------------------------------------------------------- K6 int GEMM
struct GemmArgs {
  const int8_t* A;  // M x Kp
  const int8_t* B;  // N x Kp (B^T)
  int64_t M, N;
  int Kp;
  // epilogue
  int epi;               // 0: int32 out; 1: fp32 LRQMM/DQ out
  const float* inv_a;    // M: RN(1/lambda_A)
  const float* inv_b;    // N: RN(1/lambda_B)
  const float* LA;       // M x R2 (may be null if R2 == 0)
  const float* LB;       // N x R2
  int R2;                // padded correction width roundup(2r, 8) <= 64
  float alpha, beta;
  float* D;              // M x N (ldd)
  int32_t* Cint;         // M x N (ldd)
  int64_t ldd;
  int* sched;            // device int: dynamic tile counter of the CTA-pair GEMM (zeroed per launch)
  const void* tc_maps;   // 6 CUtensorMaps of L_A hi / lo, L_B hi / lo, L_B hi / lo 256-row boxes (gemm_prepare_maps_tc) or nullptr
};
// bf16 hi / lo operands of the tensor-core correction (K8): rows x 64 bf16 each (128-byte rows)
struct GemmTcOperands {
  const void* LAh;
  const void* LAl;
  const void* LBh;
  const void* LBl;
  int64_t M, N;
};
int gemm_prepare_maps_tc(const GemmTcOperands& o, void* maps);  // 4 maps; 0 on success
// whether launch_gemm will run K8 for these sizes (R2 > 0): then L_A / L_B must be split first
bool gemm_uses_tc(int64_t M, int64_t N, int Kp, int R2, const int* sched);
// L (rows x R2 fp32) -> hi, lo (rows x 64 bf16, zero-padded)
// L_A (rowsA x R2) and L_B (rowsB x R2) -> bf16 hi / lo (rows of 64, zero-padded), one launch
void launch_split_bf16(const float* LA, int64_t rowsA, const float* LB, int64_t rowsB, int R2, void* Ahi, void* Alo,
                       void* Bhi, void* Blo, cudaStream_t st);
// mapA / mapB: arrays of four CUtensorMap (one-CTA, CTA-pair and narrow-N box shapes); 0 on success
int gemm_prepare_maps(const GemmArgs& g, void* mapA, void* mapB);
int& gemm_variant();  // 0 auto (CTA pairs when M, N >= 512 and >= 512 pair tiles, else K8 / K6), 1 K6, 2 K7, 3 K8
// 2D TMA map, dims {inner, outer} elements of u8 (dtype 0), fp32 (1) or u16 (2); returns 0 on success
int encode_map_2d_sw(void* map, int dtype, const void* base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                     uint32_t box_inner, uint32_t box_outer, int swizzle_bytes /* 0, 32, 64, 128 */);

void launch_f64_to_f32(const double* in, float* out, int64_t n, cudaStream_t st);
// negative-control hook: flips the lowest mantissa bit of p[0] (skinny.cu)
void launch_flip_lsb(float* p, cudaStream_t st);
// Omega -> zero-padded K x W copy + column maxima of |Omega| (skinny.cu)
void launch_copy_omega(const float* src, int64_t ldo, int kk, int64_t K, int W, float* dst, unsigned* cmax,
                       int* err_flag, cudaStream_t st);  // err_flag bit 0: non-finite Omega
// 0 on success, 1 if the correction width R2 has no instantiation (nothing launched)
int launch_gemm(const GemmArgs& g, const void* mapA, const void* mapB, cudaStream_t st);

}  // namespace lrqmm
