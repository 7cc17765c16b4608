// liblrqmm C ABI (include/lrqmm.h): handle lifetime, argument validation,
// workspace layout and the stream-ordered orchestration of Algorithm 2
// over the K1..K6 kernels.  No host synchronisation on the
// hot path; NCCL collectives (world_size > 1) are enqueued on the same stream.
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/lrqmm.h"
#include "comm.h"
#include "kernels.h"

using namespace lrqmm;

namespace {

constexpr int kMaxWidth = 64;

struct Side {
  int64_t rows = 0;
  int64_t ldu = 0;
  uint8_t* U = nullptr;      // residual fraction u = lambda x - code, Q15 as h | l byte planes (written by K1)
  uint8_t* img = nullptr;    // B operand images of the RSVD passes (skinny_tc.cu)
  // QuantTensor (cfg.qt_terms > 0): fp32 residual and its re-quantization
  float* R32 = nullptr;      // rows x K
  int8_t* rcodes = nullptr;  // rows x Kp
  float *rlam = nullptr, *rinv = nullptr, *rrow_amax = nullptr, *rlam_scalar = nullptr;
  int8_t* codes = nullptr;   // rows x Kp
  float* lam = nullptr;      // rows
  float* inv_lam = nullptr;  // rows, RN(1/lambda)
  float* row_amax = nullptr; // rows (per-tensor mode)
  float* lam_scalar = nullptr;
  float* Om = nullptr;       // K x W (zero-padded sketch)
  float* Y = nullptr;        // rows x W : sketch / W = R Q1
  float* Q0 = nullptr;       // rows x W
  float* Z = nullptr;        // K x W
  float* Q1 = nullptr;       // K x W
  float* Gp = nullptr;       // rows x W : X~ Q1_other
  double* G = nullptr;       // W x W
  double* gpart = nullptr;   // kGramMaxBlocks x W x W Gram partials
  int* counter = nullptr;    // Gram last-block ticket
  unsigned* cmax0 = nullptr; // column maxima of |Q0 / lambda| (COL pass image), written by apply64
  unsigned* cmax1 = nullptr; // column maxima of |Q1| (ROW / dual / codes pass images)
  unsigned* cmaxOm = nullptr;  // column maxima of |Omega| (S1 pass image), from the Omega copy
  double* T64 = nullptr;     // W x W  (orth transform, fp64)
  float* VW = nullptr;       // W x W  (first r columns: truncation)
  int* fcnt = nullptr;       // fused chain: finisher counters [0, kFuseMaxSlots) + Gram group tickets
};

}  // namespace

struct lrqmm_handle_s {
  lrqmm_config_t cfg{};
  int qmax = 0, Kp = 0, kk = 0, W = 0, r = 0, R2 = 0;
  cudaStream_t st = nullptr;
  lrqmm_status_t sticky = LRQMM_OK;
  int state = 0;  // bit0: A quantized, bit1: B quantized, bit2: rsvd done
  Side s[2];
  float* LA = nullptr;  // m x R2
  float* LB = nullptr;  // n x R2
  // bf16 hi / lo copies of L_A, L_B (rows x 64) for the tensor-core correction GEMM (K8)
  void *LAh = nullptr, *LAl = nullptr, *LBh = nullptr, *LBl = nullptr;
  alignas(64) CUtensorMap mapTC[6];  // L_A hi / lo, L_B hi / lo (128-row boxes), L_B hi / lo (256-row boxes, K8w)
  bool tc_ready = false;
  float* partial = nullptr;
  int64_t partial_elems = 0;
  double* Gcross = nullptr;  // W x W
  double* gpart_cross = nullptr;
  int* counter_cross = nullptr;
  float* VWbM = nullptr;     // W x W
  int* err_flag = nullptr;
  int* sched = nullptr;  // CTA-pair GEMM tile counter
  alignas(64) CUtensorMap mapA[4];  // GEMM map slots (gemm_i8.cu gemm_prepare_maps)
  alignas(64) CUtensorMap mapB[4];
  alignas(64) CUtensorMap mapRA[4];  // QT: maps of the residual codes
  alignas(64) CUtensorMap mapRB[4];
  cudaEvent_t ev[8] = {};
  Comm* comm = nullptr;   // world_size > 1: NCCL, or the test loopback (lrqmm_debug_create_loopback)
  int64_t launches = 0;   // kernels this handle enqueued (lrqmm_launch_count)
  int trace_next = 0;
  bool fused = false;     // experimental fused-pass chain (LRQMM_RSVD_FUSED=1)
  bool coop = false;      // W <= 32: Omega copies, Q = Y T and the next pass's B images (+ the cross Gram)
                          // as one cooperative launch each (launch_apply_prep)
  int* fcnt = nullptr;    // fused chain: [0] launch ticket of the fused passes, [1] cross-Gram ticket
  unsigned long long* trace = nullptr;  // LRQMM_FUSE_TRACE=1: 8 slots x 5 timestamps per fused pass
  // B column-sharded over the ranks (cfg.b_sharded): this rank owns rows
  // [b_lo, b_lo + s[1].rows) of B^T inside blocks of b_blk rows; s[1].codes / lam / inv_lam and LB
  // point at the rank's slice of the full (ws * b_blk row) buffers below, which the GEMM reads
  // after the in-place allgathers.
  bool bsh = false;
  int64_t b_blk = 0, b_lo = 0;
  int8_t* codes_b_full = nullptr;
  float *lam_b_full = nullptr, *inv_b_full = nullptr, *LB_full = nullptr;
  // rsvd_residual as a CUDA graph: captured once on a private stream (the caller's stream may be
  // the legacy default stream, which cannot be captured), then launched onto the caller's stream
  cudaStream_t cap_st = nullptr;
  cudaStream_t side_st = nullptr;                      // forked branch (cross Gram || truncation)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;  // the two sides' range finders as graph branches
  int pass_sm_reserve = 0;  // while they run: SMs each persistent pass leaves to the other branch
  cudaGraphExec_t rsvd_exec[3] = {};  // per rsvd_body kind
  int rsvd_calls[3] = {};
  int64_t rsvd_graph_kernels[3] = {};
  bool graph_off = false;
  // run_host buffers
  float *hA = nullptr, *hB = nullptr, *hOmA = nullptr, *hOmB = nullptr, *hD = nullptr;
  // lrqmm_run_host_async: double-buffered device staging, copy-in / copy-out streams, events
  struct Slot {
    float *A = nullptr, *B = nullptr, *OmA = nullptr, *OmB = nullptr, *D = nullptr;
    cudaEvent_t in = nullptr, consumed = nullptr, done = nullptr, out = nullptr;
  } slot[2];
  int next_slot = 0;
  cudaStream_t cin = nullptr, cout = nullptr;
};

#define LQ_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      if (getenv("LRQMM_DEBUG")) fprintf(stderr, "lrqmm: %s -> %s\n", #call, cudaGetErrorString(e_)); \
      return fail(h, LRQMM_ERR_CUDA);                                                          \
    }                                                                                          \
  } while (0)
#define LQ_NCCL(call)                                     \
  do {                                                    \
    ncclResult_t r_ = (call);                             \
    if (r_ != ncclSuccess) return fail(h, LRQMM_ERR_NCCL); \
  } while (0)

// GPU negative control (lrqmm_debug_inject_fault): a deliberate defect in the product path that the
// parity tests must catch.  0 = none.
static std::atomic<int> g_fault{0};
enum { kFaultNone = 0, kFaultRounding = 1, kFaultLambdaUlp = 2, kFaultNoCorrection = 3, kFaultDropRC3 = 4 };

static lrqmm_status_t fail(lrqmm_handle_t h, lrqmm_status_t s) {
  if (h && h->sticky == LRQMM_OK) h->sticky = s;
  return s;
}

static int64_t roundup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static lrqmm_status_t check_launch(lrqmm_handle_t h) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (getenv("LRQMM_DEBUG")) fprintf(stderr, "lrqmm: launch error %s\n", cudaGetErrorString(e));
    return fail(h, LRQMM_ERR_CUDA);
  }
  return LRQMM_OK;
}

template <typename T>
static bool dalloc(T** p, int64_t elems) {
  if (elems <= 0) elems = 1;
  if (cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (size_t)elems) != cudaSuccess) return false;
  return cudaMemset(*p, 0, sizeof(T) * (size_t)elems) == cudaSuccess;
}

extern "C" {

const char* lrqmm_status_string(lrqmm_status_t s) {
  switch (s) {
    case LRQMM_OK: return "ok";
    case LRQMM_ERR_INVALID_ARGUMENT: return "invalid argument";
    case LRQMM_ERR_SHAPE: return "shape error";
    case LRQMM_ERR_RANK: return "rank + oversample exceeds min(rows, k) or 64";
    case LRQMM_ERR_OVERFLOW: return "k * qmax^2 exceeds int32 accumulator range";
    case LRQMM_ERR_NONFINITE: return "non-finite input";
    case LRQMM_ERR_STATE: return "call out of order";
    case LRQMM_ERR_CUDA: return "CUDA error";
    case LRQMM_ERR_NCCL: return "NCCL error";
    case LRQMM_ERR_ALLOC: return "allocation failure";
    case LRQMM_ERR_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

lrqmm_status_t lrqmm_get_unique_id(unsigned char out[128]) {
  if (!out) return LRQMM_ERR_INVALID_ARGUMENT;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return LRQMM_ERR_NCCL;
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
  memcpy(out, id.internal, 128);
  return LRQMM_OK;
}

static lrqmm_status_t validate(const lrqmm_config_t* c, bool loopback) {
  if (!c) return LRQMM_ERR_INVALID_ARGUMENT;
  if (c->m < 0 || c->n < 0 || c->k < 0) return LRQMM_ERR_SHAPE;
  if (c->k > INT32_MAX - 256 || c->n > INT32_MAX || c->m > ((int64_t)1 << 40)) return LRQMM_ERR_SHAPE;
  if (c->bits != 4 && c->bits != 8) return LRQMM_ERR_UNSUPPORTED;
  if (c->rounding < 0 || c->rounding > 2) return LRQMM_ERR_INVALID_ARGUMENT;
  if (c->granularity < 0 || c->granularity > 1) return LRQMM_ERR_INVALID_ARGUMENT;
  if (c->rank < 0 || c->oversample < 0) return LRQMM_ERR_RANK;
  if (c->world_size < 1 || c->world_rank < 0 || c->world_rank >= c->world_size) return LRQMM_ERR_INVALID_ARGUMENT;
  if (c->world_size > 1 && !c->nccl_unique_id && !loopback) return LRQMM_ERR_INVALID_ARGUMENT;
  if (c->world_size > 1 && c->granularity == LRQMM_SCALE_PER_TENSOR) return LRQMM_ERR_UNSUPPORTED;
  const int64_t qmax = (1 << (c->bits - 1)) - 1;
  if (c->k * qmax * qmax > (int64_t)INT32_MAX) return LRQMM_ERR_OVERFLOW;  // reading #24
  if (c->rank > 0) {
    if (c->power_iters < 0) return LRQMM_ERR_UNSUPPORTED;  // q = 0: Algorithm 1 on orth(R Omega), reading #30
    const int64_t kk = (int64_t)c->rank + c->oversample;
    if (kk > kMaxWidth || c->rank > 32) return LRQMM_ERR_RANK;
    // r + p <= min(rows, K) of each side (A: global rows checked per shard)
    if (kk > c->k || kk > c->n || (c->world_size == 1 && kk > c->m)) return LRQMM_ERR_RANK;
  }
  if (c->qt_terms != 0 && c->qt_terms != 3 && c->qt_terms != 4) return LRQMM_ERR_INVALID_ARGUMENT;
  if (c->qt_terms != 0 && c->rank != 0) return LRQMM_ERR_UNSUPPORTED;  // QT and LRQMM are alternatives
  if (c->b_sharded != 0 && c->b_sharded != 1) return LRQMM_ERR_INVALID_ARGUMENT;
  if (c->b_sharded && c->world_size > 1 && c->qt_terms != 0) return LRQMM_ERR_UNSUPPORTED;
  return LRQMM_OK;
}

lrqmm_status_t lrqmm_destroy(lrqmm_handle_t h) {
  if (!h) return LRQMM_OK;
  cudaSetDevice(h->cfg.device);
  // nothing may still read or write the handle's buffers: the handle stream (also the legacy
  // default stream) and run_host_async's copy streams
  cudaStreamSynchronize(h->st);
  if (h->cin) cudaStreamSynchronize(h->cin);
  if (h->cout) cudaStreamSynchronize(h->cout);
  if (h->side_st) cudaStreamSynchronize(h->side_st);
  if (h->bsh) {  // side B's codes / scales / LB are slices of the full buffers
    h->s[1].codes = h->codes_b_full;
    h->s[1].lam = h->lam_b_full;
    h->s[1].inv_lam = h->inv_b_full;
    h->LB = h->LB_full;
  }
  for (auto& s : h->s) {
    cudaFree(s.codes); cudaFree(s.lam); cudaFree(s.inv_lam); cudaFree(s.row_amax); cudaFree(s.lam_scalar); cudaFree(s.Om);
    cudaFree(s.Y); cudaFree(s.Q0); cudaFree(s.Z); cudaFree(s.Q1); cudaFree(s.Gp); cudaFree(s.G);
    cudaFree(s.gpart); cudaFree(s.cmaxOm); cudaFree(s.cmax0); cudaFree(s.cmax1); cudaFree(s.counter); cudaFree(s.T64); cudaFree(s.VW); cudaFree(s.U); cudaFree(s.img);
    cudaFree(s.R32); cudaFree(s.rcodes); cudaFree(s.rlam); cudaFree(s.rinv); cudaFree(s.rrow_amax); cudaFree(s.rlam_scalar);
    cudaFree(s.fcnt);
  }
  cudaFree(h->fcnt);
  cudaFree(h->trace);
  cudaFree(h->LA); cudaFree(h->LB); cudaFree(h->LAh); cudaFree(h->LAl); cudaFree(h->LBh); cudaFree(h->LBl);
  cudaFree(h->partial); cudaFree(h->Gcross); cudaFree(h->gpart_cross);
  cudaFree(h->counter_cross); cudaFree(h->VWbM); cudaFree(h->err_flag); cudaFree(h->sched);
  cudaFree(h->hA); cudaFree(h->hB); cudaFree(h->hOmA); cudaFree(h->hOmB); cudaFree(h->hD);
  for (auto& sl : h->slot) {
    cudaFree(sl.A); cudaFree(sl.B); cudaFree(sl.OmA); cudaFree(sl.OmB); cudaFree(sl.D);
    for (cudaEvent_t e : {sl.in, sl.consumed, sl.done, sl.out})
      if (e) cudaEventDestroy(e);
  }
  if (h->cin) cudaStreamDestroy(h->cin);
  if (h->cout) cudaStreamDestroy(h->cout);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& x : h->rsvd_exec)
    if (x) cudaGraphExecDestroy(x);
  if (h->cap_st) cudaStreamDestroy(h->cap_st);
  if (h->side_st) cudaStreamDestroy(h->side_st);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_fork2) cudaEventDestroy(h->ev_fork2);
  if (h->ev_join2) cudaEventDestroy(h->ev_join2);
  delete h->comm;
  delete h;
  return LRQMM_OK;
}

// loopback_group >= 0: test transport (lrqmm_debug_create_loopback) instead of NCCL
static lrqmm_status_t create_impl(const lrqmm_config_t* cfg, int loopback_group, lrqmm_handle_t* out) {
  if (!out) return LRQMM_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  lrqmm_status_t v = validate(cfg, loopback_group >= 0);
  if (v != LRQMM_OK) return v;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) return LRQMM_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess) return LRQMM_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return LRQMM_ERR_UNSUPPORTED;  // built for sm_100a only
  if (cudaSetDevice(cfg->device) != cudaSuccess) return LRQMM_ERR_CUDA;

  lrqmm_handle_t h = new (std::nothrow) lrqmm_handle_s();
  if (!h) return LRQMM_ERR_ALLOC;
  h->cfg = *cfg;
  h->cfg.nccl_unique_id = nullptr;
  h->st = reinterpret_cast<cudaStream_t>(cfg->stream);
  h->qmax = (1 << (cfg->bits - 1)) - 1;
  // codes / residual-plane row stride: 16-byte multiple (TMA); the kernels' 128-deep boxes read
  // past it as zeros (out-of-bounds fill), so no 128-column padding is stored
  h->Kp = (int)roundup(std::max<int64_t>(cfg->k, 1), 16);
  h->r = cfg->rank;
  h->kk = cfg->rank > 0 ? cfg->rank + cfg->oversample : 0;
  h->W = h->kk > 0 ? (int)roundup(h->kk, 8) : 0;
  h->R2 = h->r > 0 ? (int)roundup(2 * h->r, 8) : 0;
  h->s[0].rows = cfg->m;
  h->s[1].rows = cfg->n;
  h->bsh = cfg->b_sharded && cfg->world_size > 1;
  if (h->bsh) {
    h->b_blk = (cfg->n + cfg->world_size - 1) / cfg->world_size;
    h->b_lo = h->b_blk * cfg->world_rank;
    h->s[1].rows = std::max<int64_t>(0, std::min<int64_t>(h->b_blk, cfg->n - h->b_lo));
  }
  const int64_t K = cfg->k;
  const int64_t nfull = h->bsh ? h->b_blk * cfg->world_size : cfg->n;  // rows of the GEMM's B buffers
  bool ok = true;
  for (int sd = 0; sd < 2; ++sd) {
    Side& s = h->s[sd];
    const int64_t cr = sd == 1 ? nfull : s.rows;  // codes / scales rows
    ok = ok && dalloc(&s.codes, cr * h->Kp) && dalloc(&s.lam, cr) && dalloc(&s.inv_lam, cr) && dalloc(&s.row_amax, s.rows) &&
         dalloc(&s.lam_scalar, 1);
    if (h->W > 0) {
      s.ldu = h->Kp;
      ok = ok && dalloc(&s.U, 2 * s.rows * s.ldu) && dalloc(&s.Om, K * h->W) && dalloc(&s.Y, s.rows * h->W) && dalloc(&s.Q0, s.rows * h->W) &&
           dalloc(&s.Z, K * h->W) && dalloc(&s.Q1, K * h->W) && dalloc(&s.Gp, s.rows * h->W) &&
           dalloc(&s.G, (int64_t)h->W * h->W) && dalloc(&s.gpart, (int64_t)kGramMaxBlocks * h->W * h->W) &&
           dalloc(&s.counter, 64) && dalloc(&s.cmax0, 64) && dalloc(&s.cmax1, 64) && dalloc(&s.cmaxOm, 64) && dalloc(&s.T64, (int64_t)h->W * h->W) && dalloc(&s.VW, (int64_t)h->W * h->W) &&
           dalloc(&s.img, 2 * tc_img_bytes(std::max<int64_t>(s.rows, K), h->W)) && dalloc(&s.fcnt, 1024);
    }
    if (cfg->qt_terms > 0)
      ok = ok && dalloc(&s.R32, s.rows * K) && dalloc(&s.rcodes, s.rows * h->Kp) && dalloc(&s.rlam, s.rows) &&
           dalloc(&s.rinv, s.rows) && dalloc(&s.rrow_amax, s.rows) && dalloc(&s.rlam_scalar, 1);
  }
  if (h->W > 0) {
    const int64_t maxrows = std::max<int64_t>({cfg->m, cfg->n, K});
    // split-K / split-row partials: <= 2 outputs x ~4 waves of splits, bounded at 64 MiB
    h->partial_elems = std::min<int64_t>((int64_t)16 << 20, 2 * 32 * maxrows * h->W);
    ok = ok && dalloc(&h->LA, cfg->m * h->R2) && dalloc(&h->LB, nfull * h->R2) &&
         dalloc(reinterpret_cast<uint16_t**>(&h->LAh), std::max<int64_t>(cfg->m, 1) * 64) &&
         dalloc(reinterpret_cast<uint16_t**>(&h->LAl), std::max<int64_t>(cfg->m, 1) * 64) &&
         dalloc(reinterpret_cast<uint16_t**>(&h->LBh), std::max<int64_t>(nfull, 1) * 64) &&
         dalloc(reinterpret_cast<uint16_t**>(&h->LBl), std::max<int64_t>(nfull, 1) * 64) &&
         dalloc(&h->partial, h->partial_elems) && dalloc(&h->Gcross, (int64_t)h->W * h->W) &&
         dalloc(&h->gpart_cross, (int64_t)kGramMaxBlocks * h->W * h->W) && dalloc(&h->counter_cross, 1) &&
         dalloc(&h->VWbM, (int64_t)h->W * h->W) && dalloc(&h->fcnt, 64);
    // the fused RSVD chain (W <= 32 keeps every fused pass at NA = 1; one rank: the Gram matrices are
    // complete inside one launch; K <= 65536: a pass with splits never has more than kFuseMaxSlots
    // output blocks).  LRQMM_RSVD_LEGACY=1 selects the separate-launch chain (A/B timing, tests).
    // both measured slower than the separate-launch chain inside the RSVD graph (c2: 262 / 365 vs
    // 246 us): opt-in, kept for A/B timing and parity-tested against it
    h->coop = h->W <= 32 && (getenv("LRQMM_RSVD_COOP") || getenv("LRQMM_RSVD_FUSED")) && !getenv("LRQMM_RSVD_LEGACY");
    h->fused = h->coop && cfg->world_size == 1 && cfg->power_iters >= 1 && K <= 65536 && getenv("LRQMM_RSVD_FUSED");
    if (h->fused && getenv("LRQMM_FUSE_TRACE")) ok = ok && dalloc(&h->trace, 64);
  }
  ok = ok && dalloc(&h->err_flag, 4) && dalloc(&h->sched, 1);
  if (!ok) {
    lrqmm_destroy(h);
    return LRQMM_ERR_ALLOC;
  }
  h->codes_b_full = h->s[1].codes;
  h->lam_b_full = h->s[1].lam;
  h->inv_b_full = h->s[1].inv_lam;
  h->LB_full = h->LB;
  if (h->bsh) {  // this rank's slices
    h->s[1].codes += h->b_lo * h->Kp;
    h->s[1].lam += h->b_lo;
    h->s[1].inv_lam += h->b_lo;
    if (h->LB) h->LB += h->b_lo * h->R2;
  }
  GemmArgs g{};
  g.A = h->s[0].codes;
  g.B = h->codes_b_full;
  g.M = std::max<int64_t>(cfg->m, 1);
  g.N = std::max<int64_t>(cfg->n, 1);
  g.Kp = h->Kp;
  if (gemm_prepare_maps(g, h->mapA, h->mapB) != 0) {
    lrqmm_destroy(h);
    return LRQMM_ERR_CUDA;
  }
  if (h->R2 > 0) {
    GemmTcOperands o{h->LAh, h->LAl, h->LBh, h->LBl, std::max<int64_t>(cfg->m, 1), std::max<int64_t>(nfull, 1)};
    if (gemm_prepare_maps_tc(o, h->mapTC) != 0) {
      lrqmm_destroy(h);
      return LRQMM_ERR_CUDA;
    }
    h->tc_ready = true;
  }
  if (cfg->qt_terms > 0) {
    g.A = h->s[0].rcodes;
    g.B = h->s[1].rcodes;
    if (gemm_prepare_maps(g, h->mapRA, h->mapRB) != 0) {
      lrqmm_destroy(h);
      return LRQMM_ERR_CUDA;
    }
  }
  if (h->trace) {
    unsigned long long t[64];
    for (int i = 0; i < 64; ++i) t[i] = (i % 8 == 0 || i % 8 == 4) ? ~0ull : 0ull;
    if (cudaMemcpy(h->trace, t, sizeof(t), cudaMemcpyHostToDevice) != cudaSuccess) {
      lrqmm_destroy(h);
      return LRQMM_ERR_CUDA;
    }
  }
  if (cfg->enable_timing) {
    for (auto& e : h->ev)
      if (cudaEventCreate(&e) != cudaSuccess) {
        lrqmm_destroy(h);
        return LRQMM_ERR_CUDA;
      }
  }
  if (cfg->world_size > 1) {
    h->comm = loopback_group >= 0 ? comm_create_loopback(loopback_group, cfg->world_size, cfg->world_rank, cfg->device)
                                  : comm_create_nccl(cfg->world_size, cfg->world_rank, cfg->nccl_unique_id);
    if (!h->comm) {
      lrqmm_destroy(h);
      return loopback_group >= 0 ? LRQMM_ERR_INVALID_ARGUMENT : LRQMM_ERR_NCCL;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    lrqmm_destroy(h);
    return LRQMM_ERR_CUDA;
  }
  *out = h;
  return LRQMM_OK;
}

lrqmm_status_t lrqmm_create(const lrqmm_config_t* cfg, lrqmm_handle_t* out) { return create_impl(cfg, -1, out); }

static void record(lrqmm_handle_t h, int i) {
  if (h->cfg.enable_timing) cudaEventRecord(h->ev[i], h->st);
}

static lrqmm_status_t allgather_b(lrqmm_handle_t h, void* full, size_t per_row_bytes);

lrqmm_status_t lrqmm_quantize(lrqmm_handle_t h, lrqmm_side_t side, const float* X, int64_t ldx) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  CounterScope counter_scope(&h->launches);
  if (h->sticky != LRQMM_OK) return h->sticky;
  if (side != LRQMM_SIDE_A && side != LRQMM_SIDE_B) return LRQMM_ERR_INVALID_ARGUMENT;
  Side& s = h->s[side];
  if ((!X && s.rows > 0 && h->cfg.k > 0) || ldx < h->cfg.k) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  record(h, side == LRQMM_SIDE_A ? 0 : 2);
  if (h->cfg.granularity == LRQMM_SCALE_PER_TENSOR) {
    launch_tensor_scale(X, ldx, s.rows, (int)h->cfg.k, h->qmax, s.row_amax, s.lam, s.inv_lam, s.lam_scalar, h->err_flag,
                        h->st);
  }
  QuantArgs a;
  a.X = X;
  a.ldx = ldx;
  a.rows = s.rows;
  a.K = (int)h->cfg.k;
  a.Kp = h->Kp;
  a.qmax = h->qmax;
  a.mode = h->cfg.rounding;
  if (g_fault.load() == kFaultRounding) a.mode = a.mode == kRoundNearest ? kRoundFloor : kRoundNearest;
  a.codes = s.codes;
  a.lam = s.lam;
  a.inv_lam = s.inv_lam;
  a.lam_fixed = h->cfg.granularity == LRQMM_SCALE_PER_TENSOR ? s.lam_scalar : nullptr;
  a.err_flag = h->err_flag;
  a.U = s.U;  // residual fractions for the RSVD passes (rank > 0 only)
  a.ldu = s.ldu;
  a.uplane = s.rows * s.ldu;
  if (s.rows > 0) launch_quantize(a, h->st);
  if (g_fault.load() == kFaultLambdaUlp && s.rows > 0) launch_flip_lsb(s.lam, h->st);  // lambda_0 one ulp off
  if (h->cfg.qt_terms > 0 && s.rows > 0 && h->cfg.k > 0) {
    // QuantTensor: r = fp32(x - code/lambda), re-quantized with its own scale(s) (Eq. gemm_r_split)
    const int K = (int)h->cfg.k;
    launch_resid_f32(X, ldx, s.codes, h->Kp, s.lam, s.rows, K, s.R32, h->st);
    if (h->cfg.granularity == LRQMM_SCALE_PER_TENSOR)
      launch_tensor_scale(s.R32, K, s.rows, K, h->qmax, s.rrow_amax, s.rlam, s.rinv, s.rlam_scalar, h->err_flag,
                          h->st);
    QuantArgs b = a;
    b.X = s.R32;
    b.ldx = K;
    b.codes = s.rcodes;
    b.lam = s.rlam;
    b.inv_lam = s.rinv;
    b.lam_fixed = h->cfg.granularity == LRQMM_SCALE_PER_TENSOR ? s.rlam_scalar : nullptr;
    b.U = nullptr;
    launch_quantize(b, h->st);
  }
  if (side == LRQMM_SIDE_B && h->bsh) {
    // every rank's GEMM multiplies by all of B: gather the codes and scales of the other shards
    lrqmm_status_t g;
    if ((g = allgather_b(h, h->codes_b_full, (size_t)h->Kp)) != LRQMM_OK) return g;
    if ((g = allgather_b(h, h->lam_b_full, sizeof(float))) != LRQMM_OK) return g;
    if ((g = allgather_b(h, h->inv_b_full, sizeof(float))) != LRQMM_OK) return g;
  }
  record(h, side == LRQMM_SIDE_A ? 1 : 3);
  lrqmm_status_t e = check_launch(h);
  if (e != LRQMM_OK) return e;
  h->state |= (side == LRQMM_SIDE_A ? 1 : 2);
  h->state &= ~4;
  if (side == LRQMM_SIDE_B) h->state &= ~8;  // resident B factors belong to the previous B
  return LRQMM_OK;
}

lrqmm_status_t lrqmm_quantize_im2col(lrqmm_handle_t h, lrqmm_side_t side, const float* X, const lrqmm_conv_t* cv) {
  if (!h || !cv) return LRQMM_ERR_INVALID_ARGUMENT;
  CounterScope counter_scope(&h->launches);
  if (h->sticky != LRQMM_OK) return h->sticky;
  if (side != LRQMM_SIDE_A && side != LRQMM_SIDE_B) return LRQMM_ERR_INVALID_ARGUMENT;
  if (h->cfg.granularity == LRQMM_SCALE_PER_TENSOR || h->cfg.qt_terms > 0) return LRQMM_ERR_UNSUPPORTED;
  if (cv->batch < 0 || cv->H < 1 || cv->W < 1 || cv->C < 1 || cv->kh < 1 || cv->kw < 1 || cv->stride_h < 1 ||
      cv->stride_w < 1 || cv->pad_h < 0 || cv->pad_w < 0 || cv->dil_h < 1 || cv->dil_w < 1)
    return LRQMM_ERR_INVALID_ARGUMENT;
  const int64_t eh = (int64_t)cv->dil_h * (cv->kh - 1) + 1, ew = (int64_t)cv->dil_w * (cv->kw - 1) + 1;
  const int64_t Ho = (cv->H + 2LL * cv->pad_h - eh) / cv->stride_h + 1, Wo = (cv->W + 2LL * cv->pad_w - ew) / cv->stride_w + 1;
  if (cv->H + 2LL * cv->pad_h < eh || cv->W + 2LL * cv->pad_w < ew) return LRQMM_ERR_INVALID_ARGUMENT;
  Side& s = h->s[side];
  if (cv->batch * Ho * Wo != s.rows || (int64_t)cv->kh * cv->kw * cv->C != h->cfg.k) return LRQMM_ERR_SHAPE;
  if (s.rows > INT32_MAX || (int64_t)cv->H * cv->W * cv->C > INT32_MAX) return LRQMM_ERR_SHAPE;  // 32-bit indexing
  if (!X && s.rows > 0) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  record(h, side == LRQMM_SIDE_A ? 0 : 2);
  QuantArgs a;
  a.X = X;
  a.ldx = h->cfg.k;
  a.rows = s.rows;
  a.K = (int)h->cfg.k;
  a.Kp = h->Kp;
  a.qmax = h->qmax;
  a.mode = h->cfg.rounding;
  a.codes = s.codes;
  a.lam = s.lam;
  a.inv_lam = s.inv_lam;
  a.lam_fixed = nullptr;
  a.err_flag = h->err_flag;
  a.U = s.U;
  a.ldu = s.ldu;
  a.uplane = s.rows * s.ldu;
  ConvGeom g{(int)cv->batch, cv->H, cv->W, cv->C, cv->kh, cv->kw, cv->stride_h, cv->stride_w, cv->pad_h, cv->pad_w,
             cv->dil_h, cv->dil_w, (int)Ho, (int)Wo};
  launch_quantize_im2col(a, g, h->st);
  if (side == LRQMM_SIDE_B && h->bsh) {
    lrqmm_status_t e;
    if ((e = allgather_b(h, h->codes_b_full, (size_t)h->Kp)) != LRQMM_OK) return e;
    if ((e = allgather_b(h, h->lam_b_full, sizeof(float))) != LRQMM_OK) return e;
    if ((e = allgather_b(h, h->inv_b_full, sizeof(float))) != LRQMM_OK) return e;
  }
  record(h, side == LRQMM_SIDE_A ? 1 : 3);
  lrqmm_status_t e = check_launch(h);
  if (e != LRQMM_OK) return e;
  h->state |= (side == LRQMM_SIDE_A ? 1 : 2);
  h->state &= ~4;
  if (side == LRQMM_SIDE_B) h->state &= ~8;
  return LRQMM_OK;
}

static SideView view(lrqmm_handle_t h, int sd) {
  SideView v;
  v.Uh = h->s[sd].U;
  v.Ul = h->s[sd].U ? h->s[sd].U + h->s[sd].rows * h->s[sd].ldu : nullptr;
  v.ldu = h->s[sd].ldu;
  v.rows = h->s[sd].rows;
  v.K = (int)h->cfg.k;
  v.codes = h->s[sd].codes;
  v.Kp = h->Kp;
  v.lam = h->s[sd].lam;
  v.inv_lam = h->s[sd].inv_lam;
  return v;
}

// allreduce (sum) of an A-side quantity across the row shards
static lrqmm_status_t allreduce_f64(lrqmm_handle_t h, double* buf, size_t n) {
  if (h->cfg.world_size == 1) return LRQMM_OK;
  if (h->comm->allreduce(buf, n, kCommF64, h->st) != 0) return fail(h, LRQMM_ERR_NCCL);
  return LRQMM_OK;
}
static lrqmm_status_t allreduce_f32(lrqmm_handle_t h, float* buf, size_t n) {
  if (h->cfg.world_size == 1) return LRQMM_OK;
  if (h->comm->allreduce(buf, n, kCommF32, h->st) != 0) return fail(h, LRQMM_ERR_NCCL);
  return LRQMM_OK;
}
// B column-sharded: in-place allgather of the rank blocks (b_blk rows each) of a full-B buffer
static lrqmm_status_t allgather_b(lrqmm_handle_t h, void* full, size_t per_row_bytes) {
  if (h->comm->allgather(full, (size_t)h->b_blk * per_row_bytes, h->st) != 0) return fail(h, LRQMM_ERR_NCCL);
  return LRQMM_OK;
}
// side sd's rows are sharded over the ranks (A always when world > 1; B when b_sharded)
static bool side_sharded(lrqmm_handle_t h, int sd) { return h->cfg.world_size > 1 && (sd == 0 || h->bsh); }

// Split-K partial regions: one half of the partial buffer per side, so side A's partials can
// wait for the fused Gram kernel while side B's pass runs.
static float* part_of(lrqmm_handle_t h, int sd) { return h->partial + sd * (h->partial_elems / 2); }
static int64_t part_elems(lrqmm_handle_t h) { return h->partial_elems / 2; }

// One RSVD pass over the selected sides, both in a single launch (launch_tc_pass).
// cm1 / cm2: column maxima of P1 / P2 from their producer (apply64), or nullptr (computed by the prep)
static void pass_sides(lrqmm_handle_t h, int kind, int sides, const float* const P1[2], const float* const P2[2],
                       float* const O1[2], float* const O2[2], bool reduce1, int nsp[2],
                       const unsigned* const cm1[2] = nullptr, const unsigned* const cm2[2] = nullptr,
                       const uint8_t* const pi1[2] = nullptr, const uint8_t* const pi2[2] = nullptr) {
  TcPassSide ps[2];
  int idx[2], n = 0;
  for (int sd = 0; sd < 2; ++sd)
    if (sides & (1 << sd)) {
      ps[n] = TcPassSide{view(h, sd), P1 ? P1[sd] : nullptr, P2 ? P2[sd] : nullptr, O1 ? O1[sd] : nullptr,
                         O2 ? O2[sd] : nullptr, part_of(h, sd), part_elems(h), h->s[sd].img,
                         cm1 ? cm1[sd] : nullptr, cm2 ? cm2[sd] : nullptr, pi1 ? pi1[sd] : nullptr,
                         pi2 ? pi2[sd] : nullptr, h->pass_sm_reserve};
      idx[n++] = sd;
    }
  int ns[2] = {0, 0};
  launch_tc_pass(kind, n, ps, h->W, reduce1, ns, h->st);
  for (int i = 0; i < n; ++i) nsp[idx[i]] = ns[i];
}

// After a skinny pass left Y_s as nsp[s] split partials: Y = sum(partials), G = Y^T Y, then
// mode 0: CholQR transform T64 -> Q = Y T64 (fp64 accumulation); mode 1: truncation VW.
// On a row-sharded A (world > 1, a_sharded) G_A is summed across ranks before the solve.
// sides: bit 0 = A, bit 1 = B
// which (mode 0): 0 = the result is Q0 (its COL-pass image needs max |Q0 / lambda| per column),
// 1 = Q1 (max |Q1|); apply64 accumulates those maxima into cmax0 / cmax1.
// coop (mode 0): Q = Y T64 together with the next pass's B images of Q (which 0: Q0 / lambda over the
// rows for the COL pass; 1: Q1 over K) in one cooperative launch; `extra` adds image / cross-Gram jobs.
static lrqmm_status_t gram_step(lrqmm_handle_t h, float* const Y[2], const int64_t n[2], const int nsp[2], int mode,
                                float* const Q[2], bool a_sharded, int sides = 3, int which = 1,
                                const ApplyPrep* extra = nullptr) {
  const int W = h->W;
  const bool ranks = a_sharded && ((side_sharded(h, 0) && (sides & 1)) || (side_sharded(h, 1) && (sides & 2)));
  SmallJobs j{};
  j.n = 0;
  // split-K partials are reduced first, in parallel over the elements (fixed order per element; both
  // sides in one launch); the fused kernel then streams the dense Y with bulk copies
  ReduceJobs rj{};
  for (int sd = 0; sd < 2; ++sd)
    if ((sides & (1 << sd)) && nsp[sd] > 1) rj.j[rj.n++] = ReduceJob{part_of(h, sd), nsp[sd], n[sd] * W, Y[sd]};
  launch_reduce_jobs(rj, h->st);
  for (int sd = 0; sd < 2; ++sd)
    if (sides & (1 << sd)) {
      const int ns = 1;
      j.j[j.n++] = SmallJob{Y[sd], part_of(h, sd), ns, n[sd], h->s[sd].G, h->s[sd].gpart, h->s[sd].counter,
                            h->s[sd].T64, h->s[sd].VW, h->r,
                            mode == 1 ? nullptr : (which == 0 ? h->s[sd].cmax0 : h->s[sd].cmax1)};
    }
  launch_fused_small(j, W, ranks ? 2 : mode, h->st);
  if (ranks) {
    for (int sd = 0; sd < 2; ++sd)
      if ((sides & (1 << sd)) && side_sharded(h, sd)) {
        lrqmm_status_t e = allreduce_f64(h, h->s[sd].G, (size_t)W * W);
        if (e != LRQMM_OK) return e;
      }
    EigJobs ej{};
    ej.n = 0;
    for (int sd = 0; sd < 2; ++sd)
      if (sides & (1 << sd)) ej.j[ej.n++] = EigJob{h->s[sd].G, h->s[sd].VW, h->s[sd].T64, h->r};
    if (mode == 0) launch_chol_orth(ej, W, h->st);
    else launch_eig_warp(ej, W, h->st);
  }
  if (mode == 0 && h->coop) {
    ApplyPrep ap = extra ? *extra : ApplyPrep{};
    ap.na = 0;
    for (int sd = 0; sd < 2; ++sd)
      if ((sides & (1 << sd)) && n[sd] > 0) {
        Side& s = h->s[sd];
        unsigned* cm = which == 0 ? s.cmax0 : s.cmax1;
        const float* sc = which == 0 ? s.inv_lam : nullptr;
        ap.a[ap.na++] = ApplyPrepJob{0, Y[sd], W, 0, s.T64, n[sd], Q[sd], cm, sc};
        if (ap.np < 4) ap.p[ap.np++] = ImgJob{Q[sd], sc, cm, s.img, n[sd]};
      }
    if (ap.na > 0 || ap.np > 0) launch_apply_prep(ap, W, h->err_flag, h->st);
  } else if (mode == 0) {
    Apply64Jobs aj{};
    for (int sd = 0; sd < 2; ++sd)
      if (sides & (1 << sd))
        aj.j[aj.n++] = Apply64Job{Y[sd], h->s[sd].T64, n[sd], Q[sd], which == 0 ? h->s[sd].cmax0 : h->s[sd].cmax1,
                                  which == 0 ? h->s[sd].inv_lam : nullptr, (int)h->kk};
    launch_apply64_jobs(aj, W, h->st);
  }
  return check_launch(h);
}

// Range finder of the selected sides (Algorithm 1 with q power steps, reading #11):
// S1 Y = R Omega; q x [O1 Q0 = orth(Y); S2 Z = R^T Q0; O2 Q1 = orth(Z)].  Leaves Q1 (K x W).
static lrqmm_status_t rsvd_chain(lrqmm_handle_t h, int sides, int kind) {
  const int W = h->W;
  const int64_t K = h->cfg.k;
  const bool multi = h->cfg.world_size > 1;
  const int64_t rows[2] = {h->s[0].rows, h->s[1].rows};
  const int64_t kdim[2] = {K, K};
  float* Ys[2] = {h->s[0].Y, h->s[1].Y};
  float* Q0s[2] = {h->s[0].Q0, h->s[1].Q0};
  float* Zs[2] = {h->s[0].Z, h->s[1].Z};
  float* Q1s[2] = {h->s[0].Q1, h->s[1].Q1};
  int nsp[2] = {1, 1};
  const unsigned* cm0[2] = {h->s[0].cmax0, h->s[1].cmax0};
  const unsigned* cm1[2] = {h->s[0].cmax1, h->s[1].cmax1};
  lrqmm_status_t e;
  // coop: every pass's B image was built by the launch that produced its operand (own image buffer)
  const uint8_t* imgs[2] = {h->s[0].img, h->s[1].img};
  const uint8_t* const* pre = h->coop ? imgs : nullptr;
  if (h->cfg.power_iters == 0) {
    // q = 0 (reading #30): S1 Y = R Omega; O1 Q0 = orth(Y); S2 Z = R^T Q0 = B^T of Algorithm 1
    // (B = Q0^* R).  Z goes to the Q1 buffer (the K-side factor), reduced.
    const float* Oms[2] = {h->s[0].Om, h->s[1].Om};
    const unsigned* cmo[2] = {h->s[0].cmaxOm, h->s[1].cmaxOm};
    pass_sides(h, kPassRow, sides, Oms, nullptr, Ys, nullptr, false, nsp, cmo, nullptr, pre);
    if ((e = gram_step(h, Ys, rows, nsp, 0, Q0s, true, sides, 0)) != LRQMM_OK) return e;
    pass_sides(h, kPassCol, sides, Q0s, nullptr, Q1s, nullptr, true, nsp, cm0, nullptr, pre);
    for (int sd = 0; sd < 2; ++sd)
      if ((sides & (1 << sd)) && side_sharded(h, sd) && (e = allreduce_f32(h, Q1s[sd], (size_t)K * W)) != LRQMM_OK)
        return e;
    return check_launch(h);
  }
  // S1: Y = R Omega   (Algorithm 1 sampling)
  const float* Oms[2] = {h->s[0].Om, h->s[1].Om};
  const unsigned* cmo[2] = {h->s[0].cmaxOm, h->s[1].cmaxOm};
  pass_sides(h, kPassRow, sides, Oms, nullptr, Ys, nullptr, false, nsp, cmo, nullptr, pre);
  for (int it = 0; it < h->cfg.power_iters; ++it) {
    // O1: Q0 = orth(Y)   (Y rows of A are sharded across ranks)
    if ((e = gram_step(h, Ys, rows, nsp, 0, Q0s, true, sides, 0)) != LRQMM_OK) return e;
    // S2: Z = R^T Q0  (reduction over rows; the A side is summed over ranks before its Gram)
    pass_sides(h, kPassCol, sides, Q0s, nullptr, Zs, nullptr, multi, nsp, cm0, nullptr, pre);
    if (multi) {
      for (int sd = 0; sd < 2; ++sd)
        if ((sides & (1 << sd)) && side_sharded(h, sd) && (e = allreduce_f32(h, Zs[sd], (size_t)K * W)) != LRQMM_OK)
          return e;
      nsp[0] = nsp[1] = 1;  // multi -> reduce1: both Z are final
    }
    // O2: Q1 = orth(Z) (fp64 Gram + Cholesky, transform applied with fp64 accumulation, so Q1 is
    // orthonormal to fp32 rounding); K rows are replicated on every rank
    // coop, last power step: the same launch forms the cross Gram Q1_B^T Q1_A (Alg. 2 line 366 core)
    // and, for static-B, the image of B's resident Q1 (the A side's cross operand)
    ApplyPrep ex{};
    const bool last = it + 1 == h->cfg.power_iters;
    if (h->coop && last && kind != 2) {
      if (kind == 1 && h->s[1].rows > 0) ex.p[ex.np++] = ImgJob{h->s[1].Q1, nullptr, h->s[1].cmax1, h->s[1].img, K};
      ex.X1 = h->s[1].Q1;
      ex.X2 = h->s[0].Q1;
      ex.xn = K;
      ex.C = h->Gcross;
      ex.cpart = h->gpart_cross;
      ex.ccnt = h->counter_cross;
    }
    if ((e = gram_step(h, Zs, kdim, nsp, 0, Q1s, false, sides, 1, &ex)) != LRQMM_OK) return e;
    if (!last) {
      pass_sides(h, kPassRow, sides, Q1s, nullptr, Ys, nullptr, false, nsp, cm1, nullptr, pre);
    }
  }
  return check_launch(h);
}

// Cross core and factor assembly (Algorithm 2 lines 361-366 folded into two rank-2r factors):
// needs W_X (= Y_X), VW_X, Q1_X of both sides and G'_A = A~ Q1_B, G'_B = B~ Q1_A.
// V_B^T V_A core: Gcross = Q1_B^T Q1_A (fp64, W x W).  Independent of the truncation, so it runs
// on a forked branch (side stream, event fork/join; captured into the graph as a parallel branch)
// while the one-CTA-per-side eigensolver occupies two SMs.
static lrqmm_status_t fork_cross_gram(lrqmm_handle_t h) {
  if (!h->side_st && cudaStreamCreateWithFlags(&h->side_st, cudaStreamNonBlocking) != cudaSuccess) return LRQMM_ERR_CUDA;
  if (!h->ev_fork && (cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess))
    return LRQMM_ERR_CUDA;
  LQ_CUDA(cudaEventRecord(h->ev_fork, h->st));
  LQ_CUDA(cudaStreamWaitEvent(h->side_st, h->ev_fork, 0));
  GramJobs j{};
  j.n = 1;
  j.j[0] = GramJob{h->s[1].Q1, h->s[0].Q1, h->cfg.k, h->Gcross, h->gpart_cross, h->counter_cross};
  launch_gram_jobs(j, h->W, h->side_st);
  LQ_CUDA(cudaEventRecord(h->ev_join, h->side_st));
  return LRQMM_OK;
}

// cross == false: VWbM was formed by the fused truncation pass (rsvd_body_fused); wait_fork: Gcross
// comes from the forked branch (fork_cross_gram) rather than from stream-ordered work
static lrqmm_status_t assemble(lrqmm_handle_t h, bool cross = true, bool wait_fork = true) {
  const int W = h->W;
  if (cross) {
    if (wait_fork) LQ_CUDA(cudaStreamWaitEvent(h->st, h->ev_join, 0));
    launch_cross_small(h->Gcross, h->s[0].VW, h->s[1].VW, W, h->r, h->VWbM, h->st);
  }
  const int r = h->r;
  const int64_t rows[2] = {h->s[0].rows, h->s[1].rows};
  if (g_fault.load() == kFaultDropRC3) LQ_CUDA(cudaMemsetAsync(h->VWbM, 0, sizeof(float) * W * W, h->st));
  // row-side factor: W = R Q1 (q >= 1), or the orthonormal Q0 (q = 0: R_k = Q0 B, B = Z^T)
  float* YA = h->cfg.power_iters == 0 ? h->s[0].Q0 : h->s[0].Y;
  float* YB = h->cfg.power_iters == 0 ? h->s[1].Q0 : h->s[1].Y;
  // one row pass per side writing fp32 L and the bf16 hi / lo operands of K8 (single rank; r % 4 == 0)
  if (h->tc_ready && W <= 32 && r % 4 == 0 && !h->bsh && h->cfg.world_size == 1 && rows[0] > 0 && rows[1] > 0) {
    AsmJobs jb{};
    jb.n = 2;
    jb.j[0] = AsmJob{YA, h->s[0].VW, h->s[0].Gp, h->s[1].VW, nullptr, rows[0], W, r, h->LA, h->R2, h->LAh, h->LAl,
                     (int)h->kk};                                                   // [U_A S_A | A~ V_B]
    jb.j[1] = AsmJob{h->s[1].Gp, h->s[0].VW, YB, h->s[1].VW, h->VWbM, rows[1], W, r, h->LB, h->R2, h->LBh, h->LBl,
                     (int)h->kk};                                                   // [B~^T V_A + U_B S_B M | U_B S_B]
    launch_assemble(jb, W, h->st);
    return check_launch(h);
  }
  ApplyJobs aj{};
  aj.n = 4;
  aj.j[0] = ApplyJob{YA, h->s[0].VW, nullptr, nullptr, rows[0], W, r, h->LA, h->R2, 0, (int)h->kk};        // U_A S_A
  aj.j[1] = ApplyJob{h->s[0].Gp, h->s[1].VW, nullptr, nullptr, rows[0], W, r, h->LA, h->R2, r, (int)h->kk}; // A~ V_B
  aj.j[2] = ApplyJob{h->s[1].Gp, h->s[0].VW, YB, h->VWbM, rows[1], W, r, h->LB, h->R2, 0, (int)h->kk};      // B~^T V_A + U_B S_B M
  aj.j[3] = ApplyJob{YB, h->s[1].VW, nullptr, nullptr, rows[1], W, r, h->LB, h->R2, r, (int)h->kk};         // U_B S_B
  launch_apply_jobs(aj, W, h->st);
  if (h->bsh) {  // the epilogue of every rank's GEMM reads all rows of L_B
    lrqmm_status_t e = allgather_b(h, h->LB_full, sizeof(float) * h->R2);
    if (e != LRQMM_OK) return e;
  }
  // bf16 hi / lo operands of the tensor-core correction (K8; always formed, so that a graph captured
  // under one kernel choice stays valid under another).  (Writing them from the assembly kernel
  // itself measured slower: 4-byte per-row stores, c4 apply 3.6 -> 8.5 ms.)
  if (h->tc_ready) {
    launch_split_bf16(h->LA, h->cfg.m, h->LB_full, h->bsh ? h->b_blk * h->cfg.world_size : h->cfg.n, h->R2, h->LAh,
                      h->LAl, h->LBh, h->LBl, h->st);
  }
  return check_launch(h);
}

// kind 0: both sides (full);  kind 1: static-B (A side + the A-dependent B term; B's W_B, VW_B,
// Q1_B resident);  kind 2: B side only (prepare the resident B factors).
// All of it is on handle-owned buffers only (graph-capturable).
static lrqmm_status_t rsvd_body_fused(lrqmm_handle_t h, int kind);
static lrqmm_status_t rsvd_body(lrqmm_handle_t h, int kind) {
  if (h->fused) return rsvd_body_fused(h, kind);
  const int W = h->W;
  const int64_t rows[2] = {h->s[0].rows, h->s[1].rows};
  float* Ys[2] = {h->s[0].Y, h->s[1].Y};
  float* Q1s[2] = {h->s[0].Q1, h->s[1].Q1};
  const int sides = kind == 0 ? 3 : (kind == 1 ? 1 : 2);
  lrqmm_status_t e;
  // Range finders: one rank, both sides -> two independent branches (side B on the side stream), so
  // that one side's streaming passes run while the other side's serial small solves (Gram, CholQR,
  // apply, image prep) would otherwise leave the GPU idle; they join before S3, which needs both Q1.
  // With NCCL (world > 1) every collective must stay in one stream order: one branch.
  const bool branches = kind == 0 && h->cfg.world_size == 1 && h->s[0].rows > 0 && h->s[1].rows > 0 &&
                        !getenv("LRQMM_RSVD_ONE_STREAM");
  if (branches) {
    if (!h->side_st && cudaStreamCreateWithFlags(&h->side_st, cudaStreamNonBlocking) != cudaSuccess)
      return fail(h, LRQMM_ERR_CUDA);
    if (!h->ev_fork2 && (cudaEventCreateWithFlags(&h->ev_fork2, cudaEventDisableTiming) != cudaSuccess ||
                         cudaEventCreateWithFlags(&h->ev_join2, cudaEventDisableTiming) != cudaSuccess))
      return fail(h, LRQMM_ERR_CUDA);
    LQ_CUDA(cudaEventRecord(h->ev_fork2, h->st));
    LQ_CUDA(cudaStreamWaitEvent(h->side_st, h->ev_fork2, 0));
    static const int reserve = [] {
      const char* v = getenv("LRQMM_BRANCH_SMS");
      return v ? atoi(v) : 16;
    }();
    h->pass_sm_reserve = reserve;
    if ((e = rsvd_chain(h, 1, kind)) != LRQMM_OK) return e;
    cudaStream_t main_st = h->st;
    h->st = h->side_st;
    e = rsvd_chain(h, 2, kind);
    h->st = main_st;
    h->pass_sm_reserve = 0;
    if (e != LRQMM_OK) return e;
    LQ_CUDA(cudaEventRecord(h->ev_join2, h->side_st));
    LQ_CUDA(cudaStreamWaitEvent(h->st, h->ev_join2, 0));
  } else if ((e = rsvd_chain(h, sides, kind)) != LRQMM_OK) {
    return e;
  }
  int nsp[2] = {1, 1};
  if (h->cfg.power_iters == 0) {
    const int64_t kdim[2] = {h->cfg.k, h->cfg.k};
    if (kind != 2) {
      // cross products G'_X = X~ Z_other (codes-only pass over both sides; both are needed even when
      // B's factors are resident, since Z_A is new)
      const float* other[2] = {Q1s[1], Q1s[0]};
      float* Gps[2] = {h->s[0].Gp, h->s[1].Gp};
      pass_sides(h, kPassCodes, 3, nullptr, other, nullptr, Gps, true, nsp);
      if ((e = fork_cross_gram(h)) != LRQMM_OK) return e;
    }
    // truncation: SVD of B = Z^T through eig(Z^T Z) (Algorithm 1); Z is replicated
    int one[2] = {1, 1};
    if ((e = gram_step(h, Q1s, kdim, one, 1, nullptr, false, sides)) != LRQMM_OK) return e;
    if (kind == 2) return check_launch(h);
    return assemble(h);
  }
  // S3 (+ cross): W_X = R_X Q1_X, and G'_X = X~ Q1_other in the same pass over X when the other
  //   side's Q1 is current (Algorithm 1 on R^T: B = Q1^T R^T = W^T; RC1/RC2 skinny
  //   products)
  const unsigned* cm1[2] = {h->s[0].cmax1, h->s[1].cmax1};
  const unsigned* cm1o[2] = {h->s[1].cmax1, h->s[0].cmax1};
  const uint8_t* imgs[2] = {h->s[0].img, h->s[1].img};
  const uint8_t* imgo[2] = {h->s[1].img, h->s[0].img};
  if (kind != 2) {
    const float* other[2] = {Q1s[1], Q1s[0]};
    float* Gps[2] = {h->s[0].Gp, h->s[1].Gp};
    pass_sides(h, kPassDual, sides, Q1s, other, Ys, Gps, false, nsp, cm1, cm1o, h->coop ? imgs : nullptr,
               h->coop ? imgo : nullptr);
  } else {
    pass_sides(h, kPassRow, sides, Q1s, nullptr, Ys, nullptr, false, nsp, cm1, nullptr, h->coop ? imgs : nullptr);
  }
  // coop: the cross Gram was formed with Q1 (gram_step O2); else on a forked branch
  if (kind != 2 && !h->coop && (e = fork_cross_gram(h)) != LRQMM_OK) return e;
  // T: W = sum(partials), truncation to rank r via eig(W^T W) (Algorithm 1)
  if ((e = gram_step(h, Ys, rows, nsp, 1, nullptr, true, sides)) != LRQMM_OK) return e;
  if (kind == 2) return check_launch(h);
  // static-B: the only A-dependent B-side term, G'_B = B~ Q1_A (a codes-only pass over B)
  if (kind == 1) {
    float* Gps[2] = {nullptr, h->s[1].Gp};
    const float* qa[2] = {nullptr, Q1s[0]};
    const unsigned* cma[2] = {nullptr, h->s[0].cmax1};
    const uint8_t* ia[2] = {nullptr, h->s[0].img};  // coop: the image of Q1_A built with it
    pass_sides(h, kPassCodes, 2, nullptr, qa, nullptr, Gps, true, nsp, nullptr, cma, nullptr, h->coop ? ia : nullptr);
  }
  return assemble(h, true, !h->coop);
}

// ---------------------------------------------------------------- fused chain
// Seven launches per full RSVD (q = 1): [Omega copies + S1 images] (eager, per call) then, captured:
// S1 (+ Gram + CholQR) -> apply Q0 + COL images -> S2 (+ split reduction + Gram + CholQR) -> apply Q1 +
// images + cross Gram -> S3 dual (+ reductions + Gram + truncation eigensolves + cross core) -> factor
// assembly.  Same arithmetic as the separate-launch chain (rsvd_body): fp64 Grams from the fp32
// panels, CholQR transforms applied with fp64 accumulation, the same B-image pieces.
static uint8_t* fimg(lrqmm_handle_t h, int sd) { return h->s[sd].img; }

static PassFuseSide fuse_side(lrqmm_handle_t h, int sd, bool gram, const uint8_t* img1, int64_t n1,
                              const uint8_t* img2, int64_t n2, unsigned* z0, unsigned* z1) {
  Side& s = h->s[sd];
  PassFuseSide f{};
  f.G = gram ? s.G : nullptr;
  f.T64 = s.T64;
  f.T = s.VW;
  f.r = h->r;
  f.zero[0] = z0;
  f.zero[1] = z1;
  f.blk_cnt = s.fcnt;
  f.grp_cnt = s.fcnt + kFuseMaxSlots;
  f.gpart = s.gpart;
  f.img1 = img1;
  f.cinv1 = img1 ? img_cinv(const_cast<uint8_t*>(img1), n1, h->W) : nullptr;
  f.img2 = img2;
  f.cinv2 = img2 ? img_cinv(const_cast<uint8_t*>(img2), n2, h->W) : nullptr;
  return f;
}

static lrqmm_status_t fused_pass(lrqmm_handle_t h, int kind, int sides, const PassFuseSide fs[2], int solver,
                                 float* const O1[2], float* const O2[2], bool cross) {
  TcPassSide ps[2];
  PassFuse f{};
  int n = 0;
  for (int sd = 0; sd < 2; ++sd)
    if (sides & (1 << sd)) {
      ps[n] = TcPassSide{view(h, sd), nullptr, nullptr, O1 ? O1[sd] : nullptr, O2 ? O2[sd] : nullptr, part_of(h, sd),
                         part_elems(h), nullptr, nullptr, nullptr};
      f.s[n++] = fs[sd];
    }
  f.solver = solver;
  f.all_cnt = h->fcnt;
  if (cross) {
    f.cross_C = h->Gcross;
    f.cross_VWa = h->s[0].VW;
    f.cross_VWb = h->s[1].VW;
    f.cross_out = h->VWbM;
  }
  f.r = h->r;
  if (h->trace) f.trace = h->trace + 8 * (h->trace_next++ & 7);
  int ns[2];
  if (!launch_tc_pass_fused(kind, n, ps, h->W, f, ns, h->st)) return fail(h, LRQMM_ERR_UNSUPPORTED);
  return check_launch(h);
}

// Omega (caller buffers, K x kk) -> the zero-padded K x W copies and the S1 B images (one eager
// cooperative launch per call: the caller's pointers are arguments, so it stays outside the graph)
static lrqmm_status_t fused_omega(lrqmm_handle_t h, const float* omA, const float* omB, int64_t ldo) {
  ApplyPrep ap{};
  const int64_t K = h->cfg.k;
  const float* om[2] = {omA, omB};
  for (int sd = 0; sd < 2; ++sd)
    if (om[sd] && h->s[sd].rows > 0 && K > 0) {
      Side& s = h->s[sd];
      // (the fused chain re-zeroes the maxima in its last pass; the coop chain does it here)
      if (!h->fused) LQ_CUDA(cudaMemsetAsync(s.cmaxOm, 0, 64 * sizeof(unsigned), h->st));
      ap.a[ap.na++] = ApplyPrepJob{1, om[sd], ldo, (int)h->kk, nullptr, K, s.Om, s.cmaxOm, nullptr};
      ap.p[ap.np++] = ImgJob{s.Om, nullptr, s.cmaxOm, fimg(h, sd), K};
    }
  if (ap.na == 0) return LRQMM_OK;
  launch_apply_prep(ap, h->W, h->err_flag, h->st);
  return check_launch(h);
}

static lrqmm_status_t rsvd_body_fused(lrqmm_handle_t h, int kind) {
  const int64_t K = h->cfg.k;
  const int sides = kind == 0 ? 3 : (kind == 1 ? 1 : 2);
  auto has = [&](int sd) { return ((sides >> sd) & 1) && h->s[sd].rows > 0 && K > 0; };
  int live = 0;
  for (int sd = 0; sd < 2; ++sd)
    if (has(sd)) live |= 1 << sd;
  if (!live) return LRQMM_OK;
  const int64_t rows[2] = {h->s[0].rows, h->s[1].rows};
  float* Ys[2] = {h->s[0].Y, h->s[1].Y};
  float* Zs[2] = {h->s[0].Z, h->s[1].Z};
  float* Gps[2] = {h->s[0].Gp, h->s[1].Gp};
  lrqmm_status_t e;
  PassFuseSide fs[2];
  // ---- S1: Y = R Omega; Gram + CholQR (Algorithm 1 sampling)
  for (int sd = 0; sd < 2; ++sd)
    fs[sd] = fuse_side(h, sd, true, fimg(h, sd), K, nullptr, 0, h->s[sd].cmax0, nullptr);
  if ((e = fused_pass(h, kPassRow, live, fs, kSolveChol, Ys, nullptr, false)) != LRQMM_OK) return e;
  for (int it = 0; it < h->cfg.power_iters; ++it) {
    // ---- O1: Q0 = Y T64 and the COL-pass images of Q0 / lambda
    ApplyPrep ap{};
    for (int sd = 0; sd < 2; ++sd)
      if (live & (1 << sd)) {
        Side& s = h->s[sd];
        ap.a[ap.na++] = ApplyPrepJob{0, s.Y, h->W, 0, s.T64, rows[sd], s.Q0, s.cmax0, s.inv_lam};
        ap.p[ap.np++] = ImgJob{s.Q0, s.inv_lam, s.cmax0, fimg(h, sd), rows[sd]};
      }
    launch_apply_prep(ap, h->W, h->err_flag, h->st);
    // ---- S2: Z = R^T Q0 (power half-step, Eq. rsvderror's q); Gram + CholQR
    for (int sd = 0; sd < 2; ++sd)
      fs[sd] = fuse_side(h, sd, true, fimg(h, sd), rows[sd], nullptr, 0, h->s[sd].cmax1, nullptr);
    if ((e = fused_pass(h, kPassCol, live, fs, kSolveChol, Zs, nullptr, false)) != LRQMM_OK) return e;
    // ---- O2: Q1 = Z T64 and the images of Q1 (K rows); before S3 also the cross Gram Q1_B^T Q1_A
    const bool last = it + 1 == h->cfg.power_iters;
    ApplyPrep aq{};
    for (int sd = 0; sd < 2; ++sd)
      if (live & (1 << sd)) {
        Side& s = h->s[sd];
        aq.a[aq.na++] = ApplyPrepJob{0, s.Z, h->W, 0, s.T64, K, s.Q1, s.cmax1, nullptr};
        aq.p[aq.np++] = ImgJob{s.Q1, nullptr, s.cmax1, fimg(h, sd), K};
      }
    if (last && kind == 1) {  // static-B: B's resident Q1 is the A side's cross operand
      Side& b = h->s[1];
      if (b.rows > 0) aq.p[aq.np++] = ImgJob{b.Q1, nullptr, b.cmax1, fimg(h, 1), K};
    }
    if (last && kind != 2) {
      aq.X1 = h->s[1].Q1;
      aq.X2 = h->s[0].Q1;
      aq.xn = K;
      aq.C = h->Gcross;
      aq.cpart = h->gpart_cross;
      aq.ccnt = h->fcnt + 1;
    }
    launch_apply_prep(aq, h->W, h->err_flag, h->st);
    if (!last) {
      // next power step: Y = R Q1 (+ Gram + CholQR)
      for (int sd = 0; sd < 2; ++sd)
        fs[sd] = fuse_side(h, sd, true, fimg(h, sd), K, nullptr, 0, h->s[sd].cmax0, nullptr);
      if ((e = fused_pass(h, kPassRow, live, fs, kSolveChol, Ys, nullptr, false)) != LRQMM_OK) return e;
    }
  }
  // ---- S3: W = R Q1 (Algorithm 1 on R^T: B = Q1^T R^T = W^T), with the cross products
  //      G'_X = X~ Q1_other (Alg. 2) in the same pass; Gram + truncation eigensolve
  //      (Alg. 1) + the V_B^T V_A core; the next call's Omega maxima re-zeroed
  const bool both = h->s[0].rows > 0 && h->s[1].rows > 0;
  for (int sd = 0; sd < 2; ++sd) {
    const int ot = 1 - sd;
    fs[sd] = fuse_side(h, sd, true, fimg(h, sd), K, kind == 2 ? nullptr : fimg(h, ot), K, h->s[sd].cmaxOm, nullptr);
  }
  if (kind == 2) {
    if ((e = fused_pass(h, kPassRow, live, fs, kSolveEig, Ys, nullptr, false)) != LRQMM_OK) return e;
    return check_launch(h);
  }
  if ((e = fused_pass(h, kPassDual, live, fs, kSolveEig, Ys, Gps, both)) != LRQMM_OK) return e;
  if (kind == 1 && h->s[1].rows > 0) {
    // static-B: the only A-dependent B-side term, G'_B = B~ Q1_A (codes pass; finisher reduction)
    PassFuseSide fb[2];
    fb[1] = fuse_side(h, 1, false, nullptr, 0, fimg(h, 0), K, nullptr, nullptr);
    if ((e = fused_pass(h, kPassCodes, 2, fb, kSolveNone, nullptr, Gps, false)) != LRQMM_OK) return e;
  }
  return assemble(h, false);
}

// Runs rsvd_body(kind), captured as a CUDA graph on the second call of that kind and replayed after.
static lrqmm_status_t run_rsvd(lrqmm_handle_t h, int kind) {
  lrqmm_status_t e = LRQMM_OK;
  const bool multi = h->cfg.world_size > 1;
  // graphs: single-rank handles (NCCL collectives stay eagerly enqueued), not disabled by env
  // (NCCL collectives are captured with the kernels; the host-synchronised loopback test transport
  // keeps multi-rank handles eager)
  const bool use_graph = kind != 2 && !h->graph_off && (!multi || h->comm->capturable()) && !getenv("LRQMM_NO_GRAPH");
  if (use_graph && h->rsvd_exec[kind]) {
    LQ_CUDA(cudaGraphLaunch(h->rsvd_exec[kind], h->st));
    launch_counter() += h->rsvd_graph_kernels[kind];
  } else if (use_graph && h->rsvd_calls[kind] >= 1) {
    // capture on the private stream (function attributes were set by the eager first call)
    if (!h->cap_st && cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking) != cudaSuccess) h->graph_off = true;
    cudaGraph_t g = nullptr;
    bool ok = !h->graph_off && cudaStreamBeginCapture(h->cap_st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      const int64_t k0 = launch_counter();
      cudaStream_t user = h->st;
      h->st = h->cap_st;
      e = rsvd_body(h, kind);
      h->st = user;
      h->rsvd_graph_kernels[kind] = launch_counter() - k0;
      launch_counter() = k0;
      ok = cudaStreamEndCapture(h->cap_st, &g) == cudaSuccess && e == LRQMM_OK && g != nullptr &&
           cudaGraphInstantiate(&h->rsvd_exec[kind], g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
    }
    cudaGetLastError();  // a failed capture must not leave a sticky launch error behind
    if (ok) {
      LQ_CUDA(cudaGraphLaunch(h->rsvd_exec[kind], h->st));
      launch_counter() += h->rsvd_graph_kernels[kind];
    } else {
      h->graph_off = true;
      if (h->rsvd_exec[kind]) { cudaGraphExecDestroy(h->rsvd_exec[kind]); h->rsvd_exec[kind] = nullptr; }
      if ((e = rsvd_body(h, kind)) != LRQMM_OK) return e;
    }
  } else {
    if ((e = rsvd_body(h, kind)) != LRQMM_OK) return e;
  }
  ++h->rsvd_calls[kind];
  return check_launch(h);
}

static lrqmm_status_t fused_omega(lrqmm_handle_t h, const float* omA, const float* omB, int64_t ldo);
static lrqmm_status_t copy_omega(lrqmm_handle_t h, int sd, const float* om, int64_t ldo) {
  if (h->fused || h->coop) return fused_omega(h, sd == 0 ? om : nullptr, sd == 1 ? om : nullptr, ldo);
  launch_copy_omega(om, ldo, (int)h->kk, h->cfg.k, h->W, h->s[sd].Om, h->s[sd].cmaxOm, h->err_flag, h->st);
  return check_launch(h);
}

lrqmm_status_t lrqmm_rsvd_residual_b(lrqmm_handle_t h, const float* omegaB, int64_t ldo) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  CounterScope counter_scope(&h->launches);
  if (h->sticky != LRQMM_OK) return h->sticky;
  if (h->r == 0) return LRQMM_ERR_STATE;
  if (!(h->state & 2)) return LRQMM_ERR_STATE;
  if (!omegaB || ldo < h->kk) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  lrqmm_status_t e;
  if ((e = copy_omega(h, 1, omegaB, ldo)) != LRQMM_OK) return e;
  if ((e = run_rsvd(h, 2)) != LRQMM_OK) return e;
  h->state |= 8;   // B's factors resident
  h->state &= ~4;  // the correction itself still needs an A side
  return LRQMM_OK;
}

lrqmm_status_t lrqmm_rsvd_residual(lrqmm_handle_t h, const float* omegaA, const float* omegaB, int64_t ldo) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  CounterScope counter_scope(&h->launches);
  if (h->sticky != LRQMM_OK) return h->sticky;
  if (h->r == 0) return LRQMM_ERR_STATE;
  if ((h->state & 3) != 3) return LRQMM_ERR_STATE;
  if (!omegaA || ldo < h->kk) return LRQMM_ERR_INVALID_ARGUMENT;
  const bool static_b = omegaB == nullptr;  // reuse the resident B factors (lrqmm_rsvd_residual_b)
  if (static_b && !(h->state & 8)) return LRQMM_ERR_STATE;
  cudaSetDevice(h->cfg.device);
  record(h, 4);
  lrqmm_status_t e;
  // sketches Omega (K x kk, caller layout) -> zero-padded K x W
  if (h->fused || h->coop) {
    if ((e = fused_omega(h, omegaA, static_b ? nullptr : omegaB, ldo)) != LRQMM_OK) return e;
  } else {
    if ((e = copy_omega(h, 0, omegaA, ldo)) != LRQMM_OK) return e;
    if (!static_b && (e = copy_omega(h, 1, omegaB, ldo)) != LRQMM_OK) return e;
  }
  if ((e = run_rsvd(h, static_b ? 1 : 0)) != LRQMM_OK) return e;
  record(h, 5);
  h->state |= 4 | 8;  // correction ready; B's factors (W_B, VW_B, Q1_B) are current either way
  return LRQMM_OK;
}

static lrqmm_status_t run_gemm(lrqmm_handle_t h, int epi, float alpha, float beta, float* D, int32_t* Cint,
                               int64_t ldd, int qt_term = 0) {
  GemmArgs g{};
  // QT term t (1-based): 1 = A_q B_q, 2 = A_q R_Bq, 3 = R_Aq B_q, 4 = R_Aq R_Bq (Eq. gemm_r_split)
  const bool ra = qt_term == 3 || qt_term == 4, rb = qt_term == 2 || qt_term == 4;
  g.A = ra ? h->s[0].rcodes : h->s[0].codes;
  g.B = rb ? h->s[1].rcodes : h->codes_b_full;
  g.M = h->cfg.m;
  g.N = h->cfg.n;
  g.Kp = h->Kp;
  g.epi = epi;
  g.inv_a = ra ? h->s[0].rinv : h->s[0].inv_lam;
  g.inv_b = rb ? h->s[1].rinv : h->inv_b_full;
  g.LA = h->LA;
  g.LB = h->LB_full;
  g.R2 = (h->r > 0 && g_fault.load() != kFaultNoCorrection) ? h->R2 : 0;
  g.alpha = alpha;
  g.beta = beta;
  g.D = D;
  g.Cint = Cint;
  g.ldd = ldd;
  g.sched = h->sched;
  g.tc_maps = (epi == 1 && g.R2 > 0 && h->tc_ready) ? h->mapTC : nullptr;
  if (launch_gemm(g, ra ? h->mapRA : h->mapA, rb ? h->mapRB : h->mapB, h->st) != 0) return LRQMM_ERR_UNSUPPORTED;
  return check_launch(h);
}

lrqmm_status_t lrqmm_gemm(lrqmm_handle_t h, float alpha, float beta, float* D, int64_t ldd) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  CounterScope counter_scope(&h->launches);
  if (h->sticky != LRQMM_OK) return h->sticky;
  if ((h->state & 3) != 3) return LRQMM_ERR_STATE;
  if (h->r > 0 && !(h->state & 4)) return LRQMM_ERR_STATE;
  if ((!D && h->cfg.m > 0 && h->cfg.n > 0) || ldd < h->cfg.n) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  record(h, 6);
  lrqmm_status_t e;
  if (h->cfg.qt_terms > 0) {
    // QuantTensor: the terms accumulate into D (beta chaining), alpha on every term
    e = run_gemm(h, 1, alpha, beta, D, nullptr, ldd, 1);
    for (int t = 2; t <= h->cfg.qt_terms && e == LRQMM_OK; ++t) e = run_gemm(h, 1, alpha, 1.f, D, nullptr, ldd, t);
  } else {
    e = run_gemm(h, 1, alpha, beta, D, nullptr, ldd);
  }
  record(h, 7);
  return e;
}

lrqmm_status_t lrqmm_gemm_int32(lrqmm_handle_t h, int32_t* Cint, int64_t ldc) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  CounterScope counter_scope(&h->launches);
  if (h->sticky != LRQMM_OK) return h->sticky;
  if ((h->state & 3) != 3) return LRQMM_ERR_STATE;
  if ((!Cint && h->cfg.m > 0 && h->cfg.n > 0) || ldc < h->cfg.n) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  return run_gemm(h, 0, 1.f, 0.f, nullptr, Cint, ldc);
}

lrqmm_status_t lrqmm_sync(lrqmm_handle_t h) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  if (cudaStreamSynchronize(h->st) != cudaSuccess) return fail(h, LRQMM_ERR_CUDA);
  if (h->cin && cudaStreamSynchronize(h->cin) != cudaSuccess) return fail(h, LRQMM_ERR_CUDA);
  if (h->cout && cudaStreamSynchronize(h->cout) != cudaSuccess) return fail(h, LRQMM_ERR_CUDA);
  if (h->sticky != LRQMM_OK) return h->sticky;
  int flag = 0;
  if (cudaMemcpy(&flag, h->err_flag, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return fail(h, LRQMM_ERR_CUDA);
  if (flag & 1) return fail(h, LRQMM_ERR_NONFINITE);
  if (h->comm && h->comm->async_error() != 0) return fail(h, LRQMM_ERR_NCCL);
  return LRQMM_OK;
}

lrqmm_status_t lrqmm_run_host(lrqmm_handle_t h, const float* A_host, const float* Bt_host, const float* omegaA_host,
                              const float* omegaB_host, float alpha, float* D_host) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  if (h->sticky != LRQMM_OK) return h->sticky;
  const int64_t m = h->cfg.m, n = h->cfg.n, k = h->cfg.k, kk = h->kk;
  const int64_t nb = h->s[1].rows;  // rows of B^T on this rank (all of them unless b_sharded)
  if ((!A_host && m * k > 0) || (!Bt_host && nb * k > 0) || (!D_host && m * n > 0)) return LRQMM_ERR_INVALID_ARGUMENT;
  if (h->r > 0 && (!omegaA_host || !omegaB_host)) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  if (!h->hA) {
    bool ok = dalloc(&h->hA, m * k) && dalloc(&h->hB, nb * k) && dalloc(&h->hD, m * n);
    if (ok && kk > 0) ok = dalloc(&h->hOmA, k * kk) && dalloc(&h->hOmB, k * kk);
    if (!ok) return fail(h, LRQMM_ERR_ALLOC);
  }
  LQ_CUDA(cudaMemcpyAsync(h->hA, A_host, sizeof(float) * m * k, cudaMemcpyHostToDevice, h->st));
  LQ_CUDA(cudaMemcpyAsync(h->hB, Bt_host, sizeof(float) * nb * k, cudaMemcpyHostToDevice, h->st));
  if (kk > 0) {
    LQ_CUDA(cudaMemcpyAsync(h->hOmA, omegaA_host, sizeof(float) * k * kk, cudaMemcpyHostToDevice, h->st));
    LQ_CUDA(cudaMemcpyAsync(h->hOmB, omegaB_host, sizeof(float) * k * kk, cudaMemcpyHostToDevice, h->st));
  }
  lrqmm_status_t e;
  if ((e = lrqmm_quantize(h, LRQMM_SIDE_A, h->hA, k)) != LRQMM_OK) return e;
  if ((e = lrqmm_quantize(h, LRQMM_SIDE_B, h->hB, k)) != LRQMM_OK) return e;
  if (h->r > 0 && (e = lrqmm_rsvd_residual(h, h->hOmA, h->hOmB, kk)) != LRQMM_OK) return e;
  if ((e = lrqmm_gemm(h, alpha, 0.f, h->hD, n)) != LRQMM_OK) return e;
  LQ_CUDA(cudaMemcpyAsync(D_host, h->hD, sizeof(float) * m * n, cudaMemcpyDeviceToHost, h->st));
  return lrqmm_sync(h);
}

lrqmm_status_t lrqmm_run_host_async(lrqmm_handle_t h, const float* A_host, const float* Bt_host,
                                    const float* omegaA_host, const float* omegaB_host, float alpha, float* D_host) {
  if (!h) return LRQMM_ERR_INVALID_ARGUMENT;
  if (h->sticky != LRQMM_OK) return h->sticky;
  const int64_t m = h->cfg.m, n = h->cfg.n, k = h->cfg.k, kk = h->kk;
  const int64_t nb = h->s[1].rows;
  if ((!A_host && m * k > 0) || (!Bt_host && nb * k > 0) || (!D_host && m * n > 0)) return LRQMM_ERR_INVALID_ARGUMENT;
  if (h->r > 0 && (!omegaA_host || !omegaB_host)) return LRQMM_ERR_INVALID_ARGUMENT;
  cudaSetDevice(h->cfg.device);
  if (!h->cin) {
    bool ok = cudaStreamCreateWithFlags(&h->cin, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&h->cout, cudaStreamNonBlocking) == cudaSuccess;
    for (auto& sl : h->slot) {
      ok = ok && dalloc(&sl.A, m * k) && dalloc(&sl.B, nb * k) && dalloc(&sl.D, m * n);
      if (ok && kk > 0) ok = dalloc(&sl.OmA, k * kk) && dalloc(&sl.OmB, k * kk);
      for (cudaEvent_t* e : {&sl.in, &sl.consumed, &sl.done, &sl.out})
        ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
    }
    if (!ok) return fail(h, LRQMM_ERR_ALLOC);
  }
  auto& sl = h->slot[h->next_slot];
  h->next_slot ^= 1;
  // copy-in stream: this slot's inputs may be overwritten once the call two steps back consumed them
  LQ_CUDA(cudaStreamWaitEvent(h->cin, sl.consumed, 0));
  LQ_CUDA(cudaMemcpyAsync(sl.A, A_host, sizeof(float) * m * k, cudaMemcpyHostToDevice, h->cin));
  LQ_CUDA(cudaMemcpyAsync(sl.B, Bt_host, sizeof(float) * nb * k, cudaMemcpyHostToDevice, h->cin));
  if (kk > 0) {
    LQ_CUDA(cudaMemcpyAsync(sl.OmA, omegaA_host, sizeof(float) * k * kk, cudaMemcpyHostToDevice, h->cin));
    LQ_CUDA(cudaMemcpyAsync(sl.OmB, omegaB_host, sizeof(float) * k * kk, cudaMemcpyHostToDevice, h->cin));
  }
  LQ_CUDA(cudaEventRecord(sl.in, h->cin));
  // compute (handle stream)
  LQ_CUDA(cudaStreamWaitEvent(h->st, sl.in, 0));
  lrqmm_status_t e;
  if ((e = lrqmm_quantize(h, LRQMM_SIDE_A, sl.A, k)) != LRQMM_OK) return e;
  if ((e = lrqmm_quantize(h, LRQMM_SIDE_B, sl.B, k)) != LRQMM_OK) return e;
  if (h->r > 0 && (e = lrqmm_rsvd_residual(h, sl.OmA, sl.OmB, kk)) != LRQMM_OK) return e;
  LQ_CUDA(cudaEventRecord(sl.consumed, h->st));  // the slot's inputs are no longer read
  LQ_CUDA(cudaStreamWaitEvent(h->st, sl.out, 0));  // the slot's D was copied out by its last user
  if ((e = lrqmm_gemm(h, alpha, 0.f, sl.D, n)) != LRQMM_OK) return e;
  LQ_CUDA(cudaEventRecord(sl.done, h->st));
  // copy-out stream
  LQ_CUDA(cudaStreamWaitEvent(h->cout, sl.done, 0));
  LQ_CUDA(cudaMemcpyAsync(D_host, sl.D, sizeof(float) * m * n, cudaMemcpyDeviceToHost, h->cout));
  LQ_CUDA(cudaEventRecord(sl.out, h->cout));
  return check_launch(h);
}

lrqmm_status_t lrqmm_get_codes(lrqmm_handle_t h, lrqmm_side_t side, signed char* dst, int64_t ld) {
  if (!h || (side != 0 && side != 1) || ld < h->cfg.k) return LRQMM_ERR_INVALID_ARGUMENT;
  if (!(h->state & (side == 0 ? 1 : 2))) return LRQMM_ERR_STATE;
  const Side& s = h->s[side];
  if (s.rows == 0 || h->cfg.k == 0) return LRQMM_OK;
  LQ_CUDA(cudaMemcpy2DAsync(dst, ld, s.codes, h->Kp, h->cfg.k, s.rows, cudaMemcpyDeviceToDevice, h->st));
  return LRQMM_OK;
}

lrqmm_status_t lrqmm_get_scales(lrqmm_handle_t h, lrqmm_side_t side, float* lambda) {
  if (!h || (side != 0 && side != 1) || !lambda) return LRQMM_ERR_INVALID_ARGUMENT;
  if (!(h->state & (side == 0 ? 1 : 2))) return LRQMM_ERR_STATE;
  const Side& s = h->s[side];
  if (s.rows == 0) return LRQMM_OK;
  LQ_CUDA(cudaMemcpyAsync(lambda, s.lam, sizeof(float) * s.rows, cudaMemcpyDeviceToDevice, h->st));
  return LRQMM_OK;
}

int lrqmm_correction_width(lrqmm_handle_t h) { return h ? h->R2 : 0; }

lrqmm_status_t lrqmm_get_correction(lrqmm_handle_t h, lrqmm_side_t side, float* L) {
  if (!h || (side != 0 && side != 1) || !L) return LRQMM_ERR_INVALID_ARGUMENT;
  if (!(h->state & 4)) return LRQMM_ERR_STATE;
  const int64_t rows = h->s[side].rows;
  LQ_CUDA(cudaMemcpyAsync(L, side == 0 ? h->LA : h->LB, sizeof(float) * rows * h->R2, cudaMemcpyDeviceToDevice, h->st));
  return LRQMM_OK;
}

lrqmm_status_t lrqmm_get_factors(lrqmm_handle_t h, lrqmm_side_t side, float* USigma, float* V) {
  if (!h || (side != 0 && side != 1) || !USigma || !V) return LRQMM_ERR_INVALID_ARGUMENT;
  CounterScope counter_scope(&h->launches);
  if (!(h->state & 4)) return LRQMM_ERR_STATE;
  const int64_t rows = h->s[side].rows;
  const int r = h->r;
  // U Sigma lives in L_A[:, 0:r] (side A) or L_B[:, r:2r] (side B)
  const float* src = side == 0 ? h->LA : h->LB + r;
  LQ_CUDA(cudaMemcpy2DAsync(USigma, sizeof(float) * r, src, sizeof(float) * h->R2, sizeof(float) * r, rows,
                            cudaMemcpyDeviceToDevice, h->st));
  // V = Q1 V_W (K x r)
  launch_apply_small(h->s[side].Q1, h->s[side].VW, nullptr, nullptr, h->cfg.k, h->W, h->W, r, V, r, 0, h->st);
  return check_launch(h);
}

lrqmm_status_t lrqmm_get_timings(lrqmm_handle_t h, double us[8]) {
  if (!h || !us) return LRQMM_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < 8; ++i) us[i] = 0.0;
  if (!h->cfg.enable_timing) return LRQMM_ERR_STATE;
  lrqmm_status_t e = lrqmm_sync(h);
  if (e != LRQMM_OK) return e;
  const int pairs[4][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}};
  for (int i = 0; i < 4; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h->ev[pairs[i][0]], h->ev[pairs[i][1]]) == cudaSuccess) us[i] = 1000.0 * ms;
  }
  return LRQMM_OK;
}

int64_t lrqmm_launch_count(lrqmm_handle_t h, int reset) {
  if (!h) return 0;
  const int64_t c = h->launches;
  if (reset) h->launches = 0;
  return c;
}

}  // extern "C"

// ------------------------------------------------------------- test hooks
#include "../../include/lrqmm_debug.h"

extern "C" lrqmm_status_t lrqmm_debug_proj(int mode, const float* X, int64_t ldx, int64_t rows, int K, int bits,
                                           int rounding, const float* P, const float* P2, int W, float* OUT,
                                           float* OUT2, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int Kp = (int)roundup(K > 0 ? K : 1, 16);
  const int64_t ldu = Kp;
  const int64_t pe = (int64_t)16 << 20;
  uint8_t* U = nullptr;
  uint8_t* img = nullptr;
  float *lam = nullptr, *inv = nullptr, *partial = nullptr;
  int8_t* codes = nullptr;
  int* flag = nullptr;
  bool ok = cudaMalloc(&U, 2 * rows * ldu) == cudaSuccess &&
            cudaMalloc(&lam, sizeof(float) * rows) == cudaSuccess && cudaMalloc(&inv, sizeof(float) * rows) == cudaSuccess &&
            cudaMalloc(&codes, (size_t)rows * Kp) == cudaSuccess && cudaMalloc(&flag, sizeof(int)) == cudaSuccess &&
            cudaMalloc(&partial, sizeof(float) * pe) == cudaSuccess &&
            cudaMalloc(&img, 2 * tc_img_bytes(rows > K ? rows : K, W)) == cudaSuccess;
  cudaError_t e = cudaErrorMemoryAllocation;
  if (ok) {
    cudaMemsetAsync(flag, 0, sizeof(int), st);
    QuantArgs q{};
    q.X = X; q.ldx = ldx; q.rows = rows; q.K = K; q.Kp = Kp; q.qmax = (1 << (bits - 1)) - 1; q.mode = rounding;
    q.codes = codes; q.lam = lam; q.inv_lam = inv; q.lam_fixed = nullptr; q.err_flag = flag; q.U = U; q.ldu = ldu; q.uplane = rows * ldu;
    launch_quantize(q, st);
    SideView v{U, U + rows * ldu, ldu, rows, K, codes, Kp, lam, inv};
    if (mode == 0) launch_tc_proj_rows(v, P, OUT, nullptr, nullptr, W, partial, pe, true, img, st);
    else if (mode == 1) launch_tc_proj_cols(v, P, OUT, W, partial, pe, true, img, st);
    else launch_tc_proj_rows(v, P, OUT, P2, OUT2, W, partial, pe, true, img, st);
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  cudaFree(U); cudaFree(lam); cudaFree(inv); cudaFree(codes); cudaFree(flag); cudaFree(partial); cudaFree(img);
  return e == cudaSuccess ? LRQMM_OK : (ok ? LRQMM_ERR_CUDA : LRQMM_ERR_ALLOC);
}

extern "C" lrqmm_status_t lrqmm_debug_create_loopback(const lrqmm_config_t* cfg, int group, lrqmm_handle_t* out) {
  if (group < 0) return LRQMM_ERR_INVALID_ARGUMENT;
  return create_impl(cfg, group, out);
}

extern "C" lrqmm_status_t lrqmm_debug_fuse_trace(lrqmm_handle_t h, int64_t out[64]) {
  if (!h || !out) return LRQMM_ERR_INVALID_ARGUMENT;
  if (!h->trace) return LRQMM_ERR_STATE;
  cudaSetDevice(h->cfg.device);
  if (cudaStreamSynchronize(h->st) != cudaSuccess) return LRQMM_ERR_CUDA;
  unsigned long long t[64];
  if (cudaMemcpy(t, h->trace, sizeof(t), cudaMemcpyDeviceToHost) != cudaSuccess) return LRQMM_ERR_CUDA;
  for (int i = 0; i < 64; ++i) out[i] = (int64_t)t[i];
  // re-arm: min slots to the maximum, max slots to 0
  for (int i = 0; i < 64; ++i) t[i] = (i % 8 == 0 || i % 8 == 4) ? ~0ull : 0ull;
  if (cudaMemcpy(h->trace, t, sizeof(t), cudaMemcpyHostToDevice) != cudaSuccess) return LRQMM_ERR_CUDA;
  h->trace_next = 0;
  return LRQMM_OK;
}

extern "C" lrqmm_status_t lrqmm_debug_inject_fault(int kind) {
  if (kind < kFaultNone || kind > kFaultDropRC3) return LRQMM_ERR_INVALID_ARGUMENT;
  g_fault.store(kind);
  return LRQMM_OK;
}

extern "C" lrqmm_status_t lrqmm_debug_set_gemm_variant(int variant) {
  if (variant < 0 || variant > 3) return LRQMM_ERR_INVALID_ARGUMENT;
  gemm_variant() = variant;
  return LRQMM_OK;
}

extern "C" lrqmm_status_t lrqmm_debug_small(int op, const float* Y, int64_t n, int W, int r, double* G, float* T,
                                            void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double* part = nullptr;
  int* counter = nullptr;
  if (cudaMalloc(&part, sizeof(double) * kGramMaxBlocks * W * W) != cudaSuccess) return LRQMM_ERR_ALLOC;
  if (cudaMalloc(&counter, 64 * sizeof(int)) != cudaSuccess) return LRQMM_ERR_ALLOC;
  cudaMemsetAsync(counter, 0, 64 * sizeof(int), st);
  if (op == 3 || op == 4) {
    // the fused Gram + solve kernel of the RSVD (mode 0 CholQR transform, mode 1 truncation), x reps
    double* T64 = nullptr;
    if (cudaMalloc(&T64, sizeof(double) * W * W) != cudaSuccess) return LRQMM_ERR_ALLOC;
    SmallJobs j{};
    j.n = 1;
    j.j[0] = SmallJob{const_cast<float*>(Y), nullptr, 1, n, G, part, counter, T64, T, r, nullptr};
    launch_fused_small(j, W, op - 3, st);
    if (op == 3) launch_f64_to_f32(T64, T, (int64_t)W * W, st);
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(part);
    cudaFree(counter);
    cudaFree(T64);
    return e == cudaSuccess ? LRQMM_OK : LRQMM_ERR_CUDA;
  }
  GramJobs gj{};
  gj.n = 1;
  gj.j[0] = GramJob{Y, Y, n, G, part, counter};
  launch_gram_jobs(gj, W, st);
  EigJobs ej{};
  ej.n = 1;
  double* T64 = nullptr;
  if (cudaMalloc(&T64, sizeof(double) * W * W) != cudaSuccess) return LRQMM_ERR_ALLOC;
  ej.j[0] = EigJob{G, T, T64, r};
  if (op == 1) {
    launch_chol_orth(ej, W, st);
    launch_f64_to_f32(T64, T, (int64_t)W * W, st);
  }
  if (op == 2) launch_eig_warp(ej, W, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(part);
  cudaFree(counter);
  cudaFree(T64);
  return e == cudaSuccess ? LRQMM_OK : LRQMM_ERR_CUDA;
}
