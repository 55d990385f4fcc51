// C-ABI implementation of libpbq (include/pbq.h): launch planning, workspace
// carving and the single-device PbP-QLP pipeline (algorithms.py:209-260).
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/pbq.h"
#include "common.cuh"
#include "gemm_f64.cuh"
#include "gemm_tma_f64.cuh"
#include "cholqr_f64.cuh"
#include "cholqr_small_f64.cuh"
#include "cholqr_mid_f64.cuh"
#include "cpqr_f64.cuh"
#include "qr_f64.cuh"
#include "sketch.cuh"
#include "exchange_f64.cuh"
#include "svd_f64.cuh"

// Optional per-kernel-class timing (pbq_profile_*): event pairs recorded on
// the launch stream around every kernel of the pipeline.
struct PbqProfile {
  bool on = false;
  int cap = 0, used = 0;
  cudaEvent_t* ev = nullptr;  // 2·cap events
  int* cls = nullptr;         // class per pair: 0 GEMM, 1 QR, 2 sketch, 3 other
  int suppress = 0;           // >0 inside a composite launch timed as one unit
};

struct pbq_ctx {
  PbqProfile prof;
  int device = 0;
  int sms = 0;
  size_t smem_optin = 0;
  size_t l2_bytes = 0;
  long long launches = 0;
  bool sketch_tables_ready = false;
  int* qr_fallbacks = nullptr;                // profiling hooks (device pointers), off by default
  int* qr_error = nullptr;                    // when set: QR kernels report unsupported panels here
  unsigned long long* qr_phase_ns = nullptr;
  unsigned long long* qr_bar_wait_ns = nullptr;
  int qr_method = PBQ_QR_AUTO;
  int* cq_stats = nullptr;                    // debug: [Cholesky-QR2 done, fallbacks]
  bool basis_orth = true;                     // intermediate orth calls of the pipeline run basis-only (orth_basis_launch)
  std::unordered_map<const void*, int> smem_attr;  // max dynamic smem already set per kernel (one driver call each)
  // stream-K partial-ready flags: one array of `sms` ints per stream that
  // has launched a GEMM on this context.  An array is zero between launches
  // (its readers reset the flags they consume), and GEMMs on one stream are
  // serialised, so no array is ever shared by two GEMMs in flight — calls on
  // different streams (each with its own workspace) may run concurrently.
  std::mutex flag_mu;
  std::vector<std::pair<cudaStream_t, int*>> stream_flags;
  std::vector<int*> flag_blocks;  // cudaMalloc'd batches backing stream_flags
  size_t flag_free = 0;           // unassigned arrays left in flag_blocks.back()
  unsigned long long p2p_timeout_ns = PBQ_XCHG_TIMEOUT_NS;  // spin limit of the peer-memory waits
  char err[512] = {0};
};

namespace {

using namespace pbq;

constexpr size_t kFlagBatch = 32;  // flag arrays per cudaMalloc batch

// The stream-K flag array of stream `st` (see pbq_ctx::stream_flags).  The
// first batch is zeroed at context creation; an array from a later batch is
// zeroed by an async memset on the stream it is assigned to (legal inside
// stream capture, and ordered before that stream's first GEMM).  nullptr on
// allocation failure.
int* gemm_flags_for(pbq_ctx* ctx, cudaStream_t st) {
  std::lock_guard<std::mutex> g(ctx->flag_mu);
  for (auto& e : ctx->stream_flags)
    if (e.first == st) return e.second;
  const size_t per = size_t(std::max(ctx->sms, 1));
  if (ctx->flag_free == 0) {
    int* blk = nullptr;
    if (cudaMalloc(&blk, sizeof(int) * per * kFlagBatch) != cudaSuccess) return nullptr;
    ctx->flag_blocks.push_back(blk);
    ctx->flag_free = kFlagBatch;
  }
  int* f = ctx->flag_blocks.back() + per * (kFlagBatch - ctx->flag_free);
  if (ctx->flag_blocks.size() > 1 && cudaMemsetAsync(f, 0, sizeof(int) * per, st) != cudaSuccess) return nullptr;
  --ctx->flag_free;
  ctx->stream_flags.emplace_back(st, f);
  return f;
}

int fail(pbq_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
    va_end(ap);
  }
  return code;
}

#define PBQ_CUDA(ctx, call)                                                                     \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? PBQ_ERR_OOM : PBQ_ERR_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                           \
  } while (0)

#define PBQ_TRY(expr)        \
  do {                       \
    int s_ = (expr);         \
    if (s_ != PBQ_OK) return s_; \
  } while (0)

// cudaFuncAttributeMaxDynamicSharedMemorySize, set once per kernel and
// context (raised when a launch needs more): a driver call per launch cost
// ~µs of host time on every one of the pipeline's ~50 launches
cudaError_t ensure_smem(pbq_ctx* ctx, const void* fn, size_t bytes) {
  int& cur = ctx->smem_attr[fn];
  if (cur >= int(bytes)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e == cudaSuccess) cur = int(bytes);
  return e;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// RAII bracket: records a start/stop event pair around one kernel class when
// profiling is on (no-op otherwise).
struct ProfScope {
  PbqProfile& pr;
  cudaStream_t st;
  int slot = -1;
  ProfScope(PbqProfile& p, cudaStream_t s, int cls) : pr(p), st(s) {
    if (pr.on && pr.suppress == 0 && pr.used < pr.cap) {
      slot = pr.used++;
      pr.cls[slot] = cls;
      cudaEventRecord(pr.ev[2 * slot], st);
    }
  }
  ~ProfScope() {
    if (slot >= 0) cudaEventRecord(pr.ev[2 * slot + 1], st);
  }
};

// Inner launches of a composite operation are not timed separately.
struct ProfSuppress {
  PbqProfile& pr;
  explicit ProfSuppress(PbqProfile& p) : pr(p) { ++pr.suppress; }
  ~ProfSuppress() { --pr.suppress; }
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Bump allocator over a caller workspace.
// NVTX range over one stage of the pipeline (SURVEY §5 profiling): host
// enqueue ranges that nsys/ncu correlate with the kernels launched inside.
// Header-only NVTX3: a no-op unless a tool injects itself.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Carve {
  char* base;
  size_t cap, off = 0;
  Carve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

// ---------------------------------------------------------------- GEMM ----
// Two tile shapes: d ≤ 64 uses 128×64 (warp 32×32), larger d 128×128 (warp 64×32).
// Tile configurations (BM×BN, BK, warps × warp tile, stages):
//   N ≤ 64 : 128×64,  BK 32, 16 warps of 32×16, 3 stages
//   N > 64 : 128×128, BK 32, 16 warps of 32×32, 3 stages.  Four warps per
//            scheduler hide the fragment-load latency that left the DMMA pipe
//            idle with 8 warps of 64×32 (33.2 → 35.0 TFLOP/s at config 3).
//            A 64×256 tile that reads A once measured 6% slower (BK 16);
//            instead the ⌈N/128⌉ column tiles of a row tile run side by side
//            in a CTA group (GemmArgs::group) over the same k-blocks, so A
//            leaves HBM once per pass (ncu: 3.87 → 1.91 GB per config-3 pass).
// 128×128 tile: 16 warps of 32×32 (4 per scheduler); 128×64 tile (d ≤ 64):
// 16 warps of 32×16 (31.7 → 33.2 TFLOP/s at d = 64 over 8 warps of 64×32)
constexpr int GEMM_WM = 32;
constexpr int GEMM_WN64 = 16;

// ---- GEMM kernel selection -----------------------------------------------
// The TMA-staged kernel (gemm_tma_f64.cuh) is the default; PBQ_GEMM_LOADER=cpasync
// selects the cp.async ring kernel (gemm_f64.cuh) for A/B measurements, and it
// is also the path when the driver's tensor-map encoder is unavailable.
enum GemmMode { GEMM_PLAIN = 0, GEMM_SPLIT = 1, GEMM_RESID = 2 };

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

bool small_tiles_off() {
  static const bool off = getenv("PBQ_NO_SMALL_TILES") != nullptr;  // A/B switch
  return off;
}

bool gemm_use_tma() {
  static const bool cpasync = [] {
    const char* e = getenv("PBQ_GEMM_LOADER");
    return e && strcmp(e, "cpasync") == 0;
  }();
  return !cpasync && tensor_map_encoder() != nullptr;
}

// row-major matrix of `rows` rows × `cols` doubles, leading dimension ld → a
// 2-D tensor map with boxes of 16 columns × box_rows rows, 128-byte swizzle
bool encode_map(CUtensorMap* m, const double* base, long cols, long rows, long ld, int box_rows) {
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * sizeof(double)};
  const cuuint32_t box[2] = {16u, cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1u, 1u};
  return tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the same matrix as a 3-D map {16, rows, cols/16} whose outer dimension
// steps over column groups (byte stride 128): one copy of box {16, box_rows,
// groups} lands group g at g·box_rows·128 bytes — the layout of the 2-D boxes.
// Only when cols is a multiple of 16 (no group reaches past the row end).
bool encode_map3(CUtensorMap* m, const double* base, long cols, long rows, long ld, int box_rows, int groups) {
  if (cols % 16 != 0 || groups < 1) return false;
  const cuuint64_t dims[3] = {16u, cuuint64_t(rows), cuuint64_t(cols / 16)};
  const cuuint64_t strides[2] = {cuuint64_t(ld) * sizeof(double), 128u};
  const cuuint32_t box[3] = {16u, cuuint32_t(box_rows), cuuint32_t(groups)};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  return tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool T, int BN, bool CHECK, int MODE, int BM = 128>
void* tma_fn() {
  constexpr int WN = (BN == 64) ? GEMM_WN64 : 32;  // 128×64 and 64×64: warp tiles 32×16
  return reinterpret_cast<void*>(&gemm_f64_tma<T, BM, BN, GEMM_WM, WN, 3, CHECK, MODE == GEMM_SPLIT, MODE == GEMM_RESID>);
}
// 64×64 tiles (8 warps) for small plain products (M ≤ 1024, e.g. the d×d
// second stage), where 128×128 tiles leave a few CTAs with long fix-up chains
void* tma_fn_small(bool trans, bool check) {
  if (trans) return check ? tma_fn<true, 64, true, 0, 64>() : tma_fn<true, 64, false, 0, 64>();
  return check ? tma_fn<false, 64, true, 0, 64>() : tma_fn<false, 64, false, 0, 64>();
}
template <bool T, int BN, bool CHECK, int MODE>
void* ring_fn() {
  constexpr int WN = BN == 64 ? GEMM_WN64 : 32;
  return reinterpret_cast<void*>(
      &gemm_f64_ring<T, 128, BN, 32, GEMM_WM, WN, 3, CHECK, MODE == GEMM_SPLIT, MODE == GEMM_RESID>);
}
template <bool TMA, int BN>
void* pick_fn(bool trans, bool check, int mode) {
  if (mode == GEMM_SPLIT) return TMA ? tma_fn<true, BN, false, GEMM_SPLIT>() : ring_fn<true, BN, false, GEMM_SPLIT>();
  if (mode == GEMM_RESID) return TMA ? tma_fn<false, BN, false, GEMM_RESID>() : ring_fn<false, BN, false, GEMM_RESID>();
  if (trans)
    return check ? (TMA ? tma_fn<true, BN, true, 0>() : ring_fn<true, BN, true, 0>())
                 : (TMA ? tma_fn<true, BN, false, 0>() : ring_fn<true, BN, false, 0>());
  return check ? (TMA ? tma_fn<false, BN, true, 0>() : ring_fn<false, BN, true, 0>())
               : (TMA ? tma_fn<false, BN, false, 0>() : ring_fn<false, BN, false, 0>());
}

int gemm_dispatch(pbq_ctx* ctx, const GemmArgs& a, bool trans, int bn, int mode, dim3 grid, bool coop,
                  cudaStream_t st, int bm = 128) {
  const int threads = bm == 64 ? 256 : 512;  // 16 warps for the 128-row tiles, 8 for 64×64
  if (bm == 64 && (mode != GEMM_PLAIN || bn != 64 || !gemm_use_tma()))
    return fail(ctx, PBQ_ERR_UNSUPPORTED, "gemm: 64×64 tiles are for plain TMA products only");
  void* fn;
  size_t smem;
  GemmTmaArgs ta;
  void* args[1];
  if (gemm_use_tma()) {
    memset(&ta, 0, sizeof(ta));
    ta.g = a;
    static const bool no3d = getenv("PBQ_TMA_NO3D") != nullptr;
    ta.a3d = !no3d && (trans ? encode_map3(&ta.ta, a.A, a.M, a.K, a.lda, 32, bm / 16)
                             : encode_map3(&ta.ta, a.A, a.K, a.M, a.lda, bm, 32 / 16));
    ta.b3d = !no3d && encode_map3(&ta.tb, a.B, a.N, a.K, a.ldb, 32, bn / 16);
    // A operand at least twice the L2 (streamed once per pass, nothing of it survives to the
    // next pass anyway): loaded evict_first, so that it does not push the thin B operand — re-read
    // by every row tile — out of L2.  ncu, config-3 AᵀΦ pass: DRAM reads 2.25 → 1.77 GB (1.66 GB
    // algorithmic), L2 hit rate 57.5 → 66.8%, same duration.  PBQ_GEMM_A_POLICY=0/1 forces it off/on.
    static const int a_policy = getenv("PBQ_GEMM_A_POLICY") ? atoi(getenv("PBQ_GEMM_A_POLICY")) : -1;
    const bool big_a = double(a.M) * double(a.K) * 8.0 >= 2.0 * double(ctx->l2_bytes);
    ta.a_policy = (a_policy < 0 ? big_a : a_policy != 0) ? 1 : 0;
    const bool ok = (ta.a3d || (trans ? encode_map(&ta.ta, a.A, a.M, a.K, a.lda, 32)
                                      : encode_map(&ta.ta, a.A, a.K, a.M, a.lda, bm))) &&
                    (ta.b3d || encode_map(&ta.tb, a.B, a.N, a.K, a.ldb, 32));
    if (!ok) return fail(ctx, PBQ_ERR_CUDA, "gemm: cuTensorMapEncodeTiled failed");
    if (bm == 64) {
      fn = tma_fn_small(trans, a.nonfinite != nullptr);
      smem = gemm_tma_smem_bytes<true, 64, 64, 3>();
    } else {
      fn = bn == 64 ? pick_fn<true, 64>(trans, a.nonfinite != nullptr, mode)
                    : pick_fn<true, 128>(trans, a.nonfinite != nullptr, mode);
      smem = bn == 64 ? gemm_tma_smem_bytes<true, 128, 64, 3>() : gemm_tma_smem_bytes<true, 128, 128, 3>();
    }
    args[0] = &ta;
  } else {
    fn = bn == 64 ? pick_fn<false, 64>(trans, a.nonfinite != nullptr, mode)
                  : pick_fn<false, 128>(trans, a.nonfinite != nullptr, mode);
    smem = trans ? (bn == 64 ? GemmCfg<true, 128, 64, 32, 32, GEMM_WN64, 3>::SMEM_BYTES
                             : GemmCfg<true, 128, 128, 32, GEMM_WM, 32, 3>::SMEM_BYTES)
                 : (bn == 64 ? GemmCfg<false, 128, 64, 32, 32, GEMM_WN64, 3>::SMEM_BYTES
                             : GemmCfg<false, 128, 128, 32, GEMM_WM, 32, 3>::SMEM_BYTES);
    args[0] = const_cast<GemmArgs*>(&a);
  }
  PBQ_CUDA(ctx, ensure_smem(ctx, fn, smem));
  if (coop) {
    PBQ_CUDA(ctx, cudaLaunchCooperativeKernel(fn, grid, dim3(threads), args, smem, st));
  } else {
    // programmatic dependent launch: the GEMM's CTAs may start (prologue,
    // tensor-map prefetch) while the previous kernel drains; the kernel's
    // griddepcontrol.wait orders every access to that kernel's results
    static const bool no_pdl = getenv("PBQ_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = no_pdl ? 0 : 1;
    PBQ_CUDA(ctx, cudaLaunchKernelExC(&cfg, fn, args));
  }
  ctx->launches += 1;
  return PBQ_OK;
}

struct GemmPlan {
  int row_iters;
  int group;
  int bm, bn;
  int tiles_m, tiles_n, k_iters;
  long total;
  int grid;
};

GemmPlan gemm_plan(const pbq_ctx* ctx, long M, long N, long K, bool tri_b = false, bool allow_small = true) {
  GemmPlan p;
  const int bk = 32;
  if (allow_small && M <= 1024 && gemm_use_tma() && !small_tiles_off()) {
    // small products (any N): 64×64 tiles — 2–4× the tiles of 128×64/128×128,
    // short fix-up chains (1000×40×1000: 30 → 19 µs, tools/gemm_small_probe.py)
    p.bm = 64; p.bn = 64;
  } else if (N <= 64) {
    p.bm = 128; p.bn = 64;
  } else {
    p.bm = 128; p.bn = 128;
  }
  p.tiles_m = int(ceil_div(M, p.bm));
  p.tiles_n = int(ceil_div(N, p.bn));
  p.k_iters = int(ceil_div(K, bk));
  p.total = long(p.tiles_m) * p.tiles_n * p.k_iters;
  p.row_iters = 0;
  p.group = 1;
  if (tri_b) {
    for (int tn = 0; tn < p.tiles_n; ++tn) p.row_iters += int(std::min<long>(p.k_iters, long(tn + 1) * p.bn / bk));
    p.total = long(p.tiles_m) * p.row_iters;
  } else {
    // column tiles of one row tile run side by side in a CTA group (A read
    // once from HBM): the largest group in {4, 2} dividing both tiles_n and
    // the SM count, when every group still gets at least one k-block
    for (int gsz = 4; gsz >= 2; gsz /= 2) {
      if (p.tiles_n % gsz == 0 && ctx->sms % gsz == 0 && p.total / gsz >= ctx->sms / gsz) {
        p.group = gsz;
        break;
      }
    }
    p.total /= p.group;
  }
  // at least two k-block units per CTA: a product with fewer units than 2·SMs
  // runs on fewer CTAs with half the fix-up partials (100×100×100 9.2 → 8.4 µs,
  // 256³ 13.5 → 10.8 µs); large products are unaffected.  PBQ_GEMM_MIN_UNITS
  // overrides (A/B).
  static const long min_units = [] {
    const char* e = getenv("PBQ_GEMM_MIN_UNITS");
    return e ? std::max(1L, atol(e)) : 2L;
  }();
  p.grid = int(std::min<long>(ctx->sms / p.group, ceil_div(p.total, min_units))) * p.group;
  return p;
}

size_t gemm_ws_bytes(const GemmPlan& p) {
  return align_up(size_t(p.grid) * p.bm * p.bn * sizeof(double), 256) + align_up(size_t(p.grid) * sizeof(int), 256) + 512;
}

template <bool TRANS>
int gemm_launch(pbq_ctx* ctx, long M, long N, long K, double alpha, const double* A, long lda, const double* B,
                long ldb, double beta, double* C, long ldc, int32_t* nonfinite, void* ws, size_t ws_bytes,
                cudaStream_t st, const int* skip = nullptr, bool tri_b = false, const int* run_if = nullptr,
                const XchgScatter* xs = nullptr) {
  if (M <= 0 || N <= 0 || K < 0) return fail(ctx, PBQ_ERR_DIM, "gemm: bad shape M=%ld N=%ld K=%ld", M, N, K);
  if ((lda & 1) || (ldb & 1) || (ldc & 1) || !aligned16(A) || !aligned16(B) || !aligned16(C))
    return fail(ctx, PBQ_ERR_PARAM, "gemm: leading dimensions must be even and pointers 16-byte aligned");
  if (K == 0) return fail(ctx, PBQ_ERR_DIM, "gemm: K == 0");
  if (tri_b && K != N) return fail(ctx, PBQ_ERR_DIM, "gemm: triangular B must be square");
  // the scatter epilogue's tile counts (pbq_xchg_expected_tiles) assume the 128-row tiles
  const GemmPlan pl = gemm_plan(ctx, M, N, K, tri_b, xs == nullptr);
  Carve cv(ws, ws_bytes);
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = M; a.N = N; a.K = K;
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb; a.C = C; a.ldc = ldc;
  a.alpha = alpha; a.beta = beta;
  a.tiles_m = pl.tiles_m; a.tiles_n = pl.tiles_n; a.k_iters = pl.k_iters; a.total_iters = pl.total;
  a.partials = cv.take<double>(size_t(pl.grid) * pl.bm * pl.bn);
  cv.take<int>(pl.grid);  // (workspace layout unchanged; the flags are per stream)
  a.flags = gemm_flags_for(ctx, st);
  if (!a.flags) return fail(ctx, PBQ_ERR_OOM, "gemm: cannot allocate stream-K flags");
  a.nonfinite = nonfinite;
  a.split = 0; a.sym = 0; a.units = 0;
  a.skip = skip;
  a.tri_b = tri_b; a.row_iters = pl.row_iters;
  a.group = pl.group;
  a.run_if = run_if;
  if (xs) {
    if (!gemm_use_tma()) return fail(ctx, PBQ_ERR_UNSUPPORTED, "gemm scatter epilogue needs the TMA kernel");
    if (xs->S % pl.bm != 0 || xs->S < 1) return fail(ctx, PBQ_ERR_PARAM, "gemm scatter: S must be a multiple of %d", pl.bm);
    a.xs_land = xs->land; a.xs_cnt = xs->cnt; a.xs_S = xs->S; a.xs_ldl = xs->ldl; a.xs_rank = xs->rank;
  }
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "gemm: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  ProfScope ps(ctx->prof, st, 0);
  return gemm_dispatch(ctx, a, TRANS, pl.bn, GEMM_PLAIN, dim3(pl.grid), false, st, pl.bm);
}

// ------------------------------------------------------------------ QR ----
struct QrPlan {
  int grid;
  long rows;  // rows per CTA
  long rch;   // rows per shared-memory chunk
  size_t smem;
};

int qr_plan(pbq_ctx* ctx, long m, long n, QrPlan& pl) {
  if (m < 1 || n < 1) return fail(ctx, PBQ_ERR_DIM, "qr: bad shape %ldx%ld", m, n);
  if (m < n) return fail(ctx, PBQ_ERR_UNSUPPORTED, "qr: requires m >= n (got %ldx%ld)", m, n);
  long g = std::min<long>(ctx->sms, ceil_div(m, 16));
  long rows = ceil_div(m, g);
  g = ceil_div(m, rows);
  const size_t limit = ctx->smem_optin;
  long rch = rows;
  if (qr_smem_doubles(rch, n, int(g)) * sizeof(double) > limit) {
    rch = 32;
    while (qr_smem_doubles(rch + 32, n, int(g)) * sizeof(double) <= limit) rch += 32;
    if (qr_smem_doubles(rch, n, int(g)) * sizeof(double) > limit)
      return fail(ctx, PBQ_ERR_UNSUPPORTED, "qr: n=%ld too large for shared memory", n);
  }
  pl.grid = int(g);
  pl.rows = rows;
  pl.rch = rch;
  pl.smem = qr_smem_doubles(rch, n, int(g)) * sizeof(double);
  return PBQ_OK;
}

size_t qr_ws_bytes(const QrPlan& pl, long n) {
  const size_t G = pl.grid;
  size_t b = 0;
  b += align_up(2 * G * 32 * 8, 256);                           // part
  b += align_up(2 * 32 * 8, 256);                               // pivrow
  b += 2 * align_up(32 * 32 * 8, 256);                          // pivbuf, gfin
  b += align_up(G * QR_NB * size_t(qr_ldw(n)) * 8, 256);        // wpart
  b += align_up(QR_NB * size_t(qr_ldy(n)) * 8, 256);            // ybuf
  b += align_up(size_t(ceil_div(n, QR_NB)) * 1024 * 8, 256);    // tall
  b += 256 + 256 + 256;                                         // counter, error
  return b;
}

int hh_launch(pbq_ctx* ctx, long m, long n, double* A, long lda, double* R, long ldr, int want_q, int32_t* rank_flag,
              void* ws, size_t ws_bytes, cudaStream_t st, const int* run_if, unsigned int* zeroed_counter = nullptr) {
  QrPlan pl;
  PBQ_TRY(qr_plan(ctx, m, n, pl));
  if (lda < n || (R && ldr < n)) return fail(ctx, PBQ_ERR_PARAM, "qr: leading dimension too small");
  if ((lda & 1) || !aligned16(A)) return fail(ctx, PBQ_ERR_PARAM, "qr: lda must be even and A 16-byte aligned");
  Carve cv(ws, ws_bytes);
  QrArgs a;
  a.m = m; a.n = n; a.A = A; a.lda = lda; a.R = R; a.ldr = ldr;
  a.want_q = want_q; a.rows_per_cta = pl.rows; a.rch = int(pl.rch);
  a.part = cv.take<double>(2 * size_t(pl.grid) * 32);
  a.pivrow = cv.take<double>(2 * 32);
  a.pivbuf = cv.take<double>(32 * 32);
  a.gfin = cv.take<double>(32 * 32);
  a.wpart = cv.take<double>(size_t(pl.grid) * QR_NB * qr_ldw(n));
  a.ybuf = cv.take<double>(size_t(QR_NB) * qr_ldy(n));
  a.tall = cv.take<double>(size_t(ceil_div(n, QR_NB)) * 1024);
  a.counter = cv.take<unsigned int>(1);
  if (zeroed_counter) a.counter = zeroed_counter;  // the caller's control block, already zeroed (no memset node)
  a.error = ctx->qr_error ? ctx->qr_error : cv.take<int>(1);
  a.rank_flag = rank_flag;
  a.fallbacks = ctx->qr_fallbacks;
  a.phase_ns = ctx->qr_phase_ns;
  a.bar_wait_ns = ctx->qr_bar_wait_ns;
  a.run_if = run_if;
  static const bool slow_panels = getenv("PBQ_QR_SLOW_PANELS") != nullptr;  // A/B switch
  a.slow_panels = slow_panels ? 1 : 0;
  static const double fast_ratio =  // A/B switch
      getenv("PBQ_QR_FAST_RATIO") ? atof(getenv("PBQ_QR_FAST_RATIO")) : QR_FAST_DIAG_RATIO;
  a.fast_ratio = fast_ratio;
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "qr: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  if (!zeroed_counter) PBQ_CUDA(ctx, cudaMemsetAsync(a.counter, 0, sizeof(unsigned int), st));
  PBQ_CUDA(ctx, ensure_smem(ctx, reinterpret_cast<const void*>(&qr_tall_kernel), pl.smem));
  void* args[] = {&a};
  ProfScope ps(ctx->prof, st, 1);
  PBQ_CUDA(ctx, cudaLaunchCooperativeKernel(reinterpret_cast<void*>(&qr_tall_kernel), dim3(pl.grid),
                                            dim3(QR_THREADS), args, pl.smem, st));
  ctx->launches += 1;
  return PBQ_OK;
}

// ------------------------------------------------------- Cholesky-QR2 ----
// Guarded whole-matrix CholQR2 (cholqr_f64.cuh) + on-device Householder
// fallback.  Launch sequence on one stream, no host synchronisation:
//   Gram(A) → reduce → factor pass 1 (R₁, R₁⁻¹, κ guard) → Q₁ = A·R₁⁻¹
//   → Gram(Q₁) → reduce → factor pass 2 (R₂, R₂⁻¹, R = R₂R₁, rank test)
//   → A ← Q₁·R₂⁻¹ → Householder kernel (runs only if the guard fired).
struct CqPlan {
  int nb;
  long np;
  int bm, bn, tiles_m, tiles_n, ntiles, k_iters, S, units;  // Gram GEMM (split-K partials)
  int Sd;                                                  // slices of a diagonal tile (0: all tiles S)
  int grid;                                                // factor kernel CTAs, pass 1
  int grid2;                                               // pass 2 (series rounds have more items)
  long ldq1;
  size_t gemm_ws;
};

constexpr double CQ_KAPPA_MAX = 1e6;
// basis-only calls (cq_launch with Out): B = X·R₁⁻¹ only has to be a
// well-conditioned basis of range(X), ‖BᵀB − I‖ ≈ κ₂²u — 1e-2 at κ₂ = 1e7 —
// and its rounding error u·κ₂ relative to ‖B‖ is that of any QR of X.  κ₁ (the
// 1-norm estimate the guard computes) runs a few times above κ₂; beyond the
// limit the Cholesky factorization itself starts to break down (pivot test).
constexpr double CQ_KAPPA_MAX_BASIS = 3e7;
// … and on the shifted route a basis-only call stops after its second pass when
// max/min |diag R₂| ≤ this (κ₂(Q₁) within a small factor of it, Q₂'s defect ≈ κ₂(Q₁)²u ≲ 1e-4)
constexpr double CQ_BASIS2_DIAG_MAX = 1e5;

CqPlan cq_plan(const pbq_ctx* ctx, long m, long n) {
  CqPlan p;
  p.nb = int(ceil_div(n, 32));
  p.np = 32L * p.nb;
  p.bm = 128;
  p.bn = n <= 64 ? 64 : 128;
  p.tiles_m = int(ceil_div(n, p.bm));
  p.tiles_n = int(ceil_div(n, p.bn));
  p.ntiles = (p.tiles_m == 1 && p.tiles_n == 1) ? 1 : p.tiles_n * (p.tiles_n + 1) / 2;
  p.k_iters = int(ceil_div(m, 32));
  p.S = int(std::max<long>(1, std::min<long>(p.k_iters, ctx->sms / p.ntiles)));
  p.Sd = 0;
  p.units = p.ntiles * p.S;
  if (p.ntiles > 1 && p.bm == 128 && p.bn == 128 && gemm_use_tma()) {
    // symmetric Gram: a diagonal tile skips its strictly-lower warp tiles and
    // its busiest scheduler runs 3 instead of 4 warp tiles (gemm_tma_f64.cuh),
    // so it gets 3/4 of an off-diagonal tile's k-slices
    const long nd = p.tiles_n, no = p.ntiles - p.tiles_n;
    long so = std::min<long>(p.k_iters, std::max<long>(1, (4L * ctx->sms) / (3L * nd + 4L * no)));
    long sd = std::max<long>(1, std::min<long>(p.k_iters, (3 * so + 2) / 4));
    while (nd * sd + no * so > ctx->sms && so > 1) {
      --so;
      sd = std::max<long>(1, std::min<long>(p.k_iters, (3 * so + 2) / 4));
    }
    p.S = int(so);
    p.Sd = int(sd);
    p.units = int(nd * sd + no * so);
  }
  p.grid = int(std::max<long>(1, std::min<long>(ctx->sms, std::max<long>(long(p.nb) * (p.nb - 1) / 2, p.nb - 1))));
  {
    const long nbl = p.nb;
    p.grid2 = int(std::max<long>(p.grid, std::min<long>(ctx->sms, nbl * (nbl + 1) + nbl * (nbl - 1) / 2)));
  }
  p.ldq1 = (n + 1) & ~1L;
  const size_t gram = align_up(size_t(p.units) * p.bm * p.bn * sizeof(double), 256);
  p.gemm_ws = std::max(gram, gemm_ws_bytes(gemm_plan(ctx, m, n, n, true)));
  return p;
}

// n ≥ this: the chain also carries the shifted Cholesky-QR3 route, so an
// ill-conditioned input stays on GEMM-shaped passes instead of falling back
// to the Householder kernel (whose column-by-column panel fallback needs its
// rows resident in shared memory, which large n does not allow)
constexpr long CQ_EXT_MIN_N = 384;

size_t cq_ws_bytes(const CqPlan& p, const QrPlan& hp, long m, long n) {
  const size_t sq = align_up(size_t(p.np) * p.np * sizeof(double), 256);
  const size_t thin = align_up(size_t(m) * p.ldq1 * sizeof(double), 256);
  const bool ext = n >= CQ_EXT_MIN_N;
  return 256 + 6 * sq + align_up(2 * size_t(p.nb) * p.np * sizeof(double), 256) + align_up(p.gemm_ws, 256) + thin +
         (ext ? 2 * sq + thin : 0) + qr_ws_bytes(hp, n) + 1024;
}

// Gram matrix G = XᵀX (upper tiles, split-K partials).  With `counter` (a
// zeroed int of the caller's control block) the slice sum runs in the same
// cooperative launch and writes G, its copy and max|G − I| (one launch
// instead of Gram + a separate slice-sum kernel); without it only the partials.
int gram_launch(pbq_ctx* ctx, const CqPlan& pl, long m, long n, const double* X, long ldx, double* part,
                const int* skip, cudaStream_t st, const int* run_if = nullptr, int* counter = nullptr,
                double* G = nullptr, unsigned long long* emax = nullptr, double* gcopy = nullptr) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = n; a.N = n; a.K = m;
  a.A = X; a.lda = ldx; a.B = X; a.ldb = ldx;
  a.alpha = 1.0;
  a.tiles_m = pl.tiles_m; a.tiles_n = pl.tiles_n; a.k_iters = pl.k_iters;
  a.partials = part;
  a.split = pl.S; a.sym = pl.ntiles > 1; a.units = pl.units;
  a.split_diag = pl.Sd; a.split_tiles = pl.ntiles;
  a.skip = skip;
  a.run_if = run_if;
  a.red_counter = reinterpret_cast<unsigned int*>(counter);
  a.red_G = G; a.red_Gcopy = gcopy; a.red_emax = emax; a.red_n = n; a.red_np = pl.np;
  return gemm_dispatch(ctx, a, true, pl.bn, GEMM_SPLIT, dim3(std::min(pl.units, ctx->sms)), counter != nullptr, st);
}

int factor_launch(pbq_ctx* ctx, const CqPlan& pl, CqArgs& a, cudaStream_t st) {
  // A/B switches for the diagonal factorization (default: the pipelined two-warp routine)
  static const int variant = getenv("PBQ_CHOL_1WARP") ? 1 : getenv("PBQ_CHOL_LOCKSTEP") ? 2 : 0;
  a.chol_1warp = variant;
  PBQ_CUDA(ctx, ensure_smem(ctx, reinterpret_cast<const void*>(&cholqr_factor_kernel), CQ_SMEM_BYTES));
  void* args[] = {&a};
  PBQ_CUDA(ctx, cudaLaunchCooperativeKernel(reinterpret_cast<void*>(&cholqr_factor_kernel),
                                            dim3(a.pass == 1 ? pl.grid : pl.grid2),
                                            dim3(CQ_THREADS), args, CQ_SMEM_BYTES, st));
  ctx->launches += 1;
  return PBQ_OK;
}

// PBQ_DEBUG_SYNC=1: synchronise and report after each launch of the chain (debugging only)
#define CQ_DEBUG_SYNC(what)                                                                      \
  do {                                                                                           \
    static const bool on_ = getenv("PBQ_DEBUG_SYNC") != nullptr;                                 \
    if (on_) {                                                                                   \
      cudaError_t e_ = cudaStreamSynchronize(st);                                                \
      int h_[16];                                                                                \
      cudaMemcpy(h_, ctl + 8, sizeof(h_), cudaMemcpyDeviceToHost);                               \
      fprintf(stderr, "cq %s: %s fallback=%d route=%d hh=%d\n", what, cudaGetErrorString(e_), 0, h_[2], h_[4]); \
    }                                                                                            \
  } while (0)

// copy src → dst (m×n) only when *run_if != 0: the fallback hand-over of a
// basis-only call (the Householder kernel and the shifted route work in place)
__global__ void __launch_bounds__(256) copy_if_kernel(const int* __restrict__ run_if, const double* __restrict__ src,
                                                      long lds, double* __restrict__ dst, long ldd, long m, long n,
                                                      int unless = 0) {
  if ((__ldcg(run_if) != 0) == (unless != 0)) return;
  for (long e = long(blockIdx.x) * blockDim.x + threadIdx.x; e < m * n; e += long(gridDim.x) * blockDim.x) {
    const long r = e / n, c = e % n;
    dst[r * ldd + c] = src[r * lds + c];
  }
}

// the shifted route of a basis-only call found Q₂ good enough: stop the route
// (its remaining launches return at once) and keep Out as it is
__global__ void basis_exit_kernel(const int* __restrict__ done, int* route, int* fallback) {
  if (*done) {
    *route = 0;
    *fallback = 0;
  }
}

// Out != nullptr: basis-only call (orth_basis_launch below).  Only the first
// Cholesky-QR pass runs: Out = A·R₁⁻¹ = Q·R₂ with R₂ upper triangular,
// positive diagonal, ‖R₂ᵀR₂ − I‖ ≲ κ₁²u ≤ 1e-4 — the same Q factor under any
// later QR, at half the passes.  A failed guard runs the full in-place chain /
// Householder kernel on A and copies the result to Out.
int cq_launch(pbq_ctx* ctx, long m, long n, double* A, long lda, double* R, long ldr, int32_t* rank_flag, void* ws,
              size_t ws_bytes, cudaStream_t st, double* Out = nullptr, long ldo = 0) {
  QrPlan hp;
  PBQ_TRY(qr_plan(ctx, m, n, hp));
  if (lda < n || (R && ldr < n)) return fail(ctx, PBQ_ERR_PARAM, "qr: leading dimension too small");
  if ((lda & 1) || !aligned16(A)) return fail(ctx, PBQ_ERR_PARAM, "qr: lda must be even and A 16-byte aligned");
  const bool basis = Out != nullptr;
  if (basis && (ldo < n || (ldo & 1) || !aligned16(Out)))
    return fail(ctx, PBQ_ERR_PARAM, "orth_basis: ldo must be even and >= n, Out 16-byte aligned");
  const CqPlan pl = cq_plan(ctx, m, n);
  const bool ext = n >= CQ_EXT_MIN_N;
  const size_t sq = size_t(pl.np) * pl.np;
  Carve cv(ws, ws_bytes);
  // ctl: [0] fallback (stops the CholQR2 path), [1] [2] [16] [17] [18] grid-barrier
  // counters, [4:6] [20:22] [22:24] max|G − I| slots, [10] shifted route running,
  // [14] basis-only call: the route's second pass is already a good basis,
  // [12] Householder requested (extended chain), [32..35] Gram slice-sum barriers,
  // [48] the Householder kernel's grid-barrier counter
  int* ctl = cv.take<int>(64);
  double* X1 = cv.take<double>(sq);
  double* X2 = cv.take<double>(sq);
  const size_t zero_bytes = size_t(reinterpret_cast<char*>(X2 + sq) - reinterpret_cast<char*>(ctl));
  double* G = cv.take<double>(sq);
  double* R1 = cv.take<double>(sq);
  double* R2 = cv.take<double>(sq);
  double* T = cv.take<double>(sq);
  double* colsum = cv.take<double>(2 * size_t(pl.nb) * pl.np);
  char* gws = cv.take<char>(pl.gemm_ws);
  double* Q1 = cv.take<double>(size_t(m) * pl.ldq1);
  double* Gc = ext ? cv.take<double>(sq) : nullptr;     // copy of G₁ for the shifted factorization
  double* Racc = ext ? cv.take<double>(sq) : nullptr;   // R₂·R₁ of the route
  double* Q2 = ext ? cv.take<double>(size_t(m) * pl.ldq1) : nullptr;
  const size_t hws_bytes = qr_ws_bytes(hp, n);
  char* hws = cv.take<char>(hws_bytes);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "qr: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  int* fallback = ctl;
  int* route = ctl + 10;
  int* hh_req = ctl + 12;
  PBQ_CUDA(ctx, cudaMemsetAsync(ctl, 0, zero_bytes, st));

  ProfScope ps(ctx->prof, st, 1);
  ProfSuppress quiet(ctx->prof);
  double* part = reinterpret_cast<double*>(gws);
  auto counter = [&](int i) { return reinterpret_cast<unsigned int*>(ctl + i); };
  auto emax_slot = [&](int i) { return reinterpret_cast<unsigned long long*>(ctl + i); };
  CqArgs f;
  memset(&f, 0, sizeof(f));
  f.nb = pl.nb; f.n = n; f.np = pl.np; f.m = m;
  f.G = G; f.T = T; f.fallback = fallback;
  f.emax = emax_slot(4); f.colsum = colsum; f.stats = ctx->cq_stats; f.fail_stats = ctx->cq_stats;
  f.kappa_max = CQ_KAPPA_MAX;
  f.phase_ns = ctx->qr_phase_ns;
  f.allow_series = ctx->qr_method != PBQ_QR_CHOLQR_NOSERIES;
  if (ext) {
    f.shift_req = route;  // pass 1 failing → the shifted route
    f.hh_req = hh_req;
  }
  // ---- Cholesky-QR2
  PBQ_TRY(gram_launch(ctx, pl, m, n, A, lda, part, fallback, st, nullptr, ctl + 32, G, nullptr, Gc));
  f.pass = 1; f.R = R1; f.X = X1; f.counter = counter(1);
  if (basis) {
    f.basis = 1;
    f.rank_flag = rank_flag;
    f.kappa_max = CQ_KAPPA_MAX_BASIS;
  }
  PBQ_TRY(factor_launch(ctx, pl, f, st));
  PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, A, lda, X1, pl.np, 0.0, basis ? Out : Q1, basis ? ldo : pl.ldq1,
                             nullptr, gws, pl.gemm_ws, st, fallback, true));
  f.basis = 0;
  f.kappa_max = CQ_KAPPA_MAX;
  if (!basis) {
    PBQ_TRY(gram_launch(ctx, pl, m, n, Q1, pl.ldq1, part, fallback, st, nullptr, ctl + 33, G, emax_slot(4)));
    f.pass = 2; f.R = R2; f.X = X2; f.R1 = R1; f.Rout = R; f.ldr = ldr; f.rank_flag = rank_flag;
    f.counter = counter(2);
    f.shift_req = nullptr;
    PBQ_TRY(factor_launch(ctx, pl, f, st));
    PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, Q1, pl.ldq1, X2, pl.np, 0.0, A, lda, nullptr, gws, pl.gemm_ws, st,
                               fallback, true));
  }
  CQ_DEBUG_SYNC("cholqr2 done");
  if (ext) {
    // ---- shifted Cholesky-QR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto,
    // Yanagisawa 2020), only when pass 1 failed: R₁ = chol(G₁ + s·I),
    // Q₁ = A·R₁⁻¹, then two Cholesky-QR passes Q₁ → Q₂ → Q.  Every launch
    // returns at once unless *route; a failure clears it and asks for the
    // Householder kernel.  A is only written by the last product.
    CqArgs g = f;
    g.fallback = nullptr; g.route = route; g.hh_req = hh_req; g.shift_req = nullptr;
    g.pass = 1; g.shift_mode = 1; g.G = Gc; g.R = R1; g.X = X1; g.counter = counter(16);
    g.Rout = nullptr; g.rank_flag = nullptr; g.R1 = nullptr;
    PBQ_TRY(factor_launch(ctx, pl, g, st));
    CQ_DEBUG_SYNC("route 1");
    PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, A, lda, X1, pl.np, 0.0, Q1, pl.ldq1, nullptr, gws, pl.gemm_ws, st,
                               nullptr, true, route));
    CQ_DEBUG_SYNC("route 2");
    PBQ_TRY(gram_launch(ctx, pl, m, n, Q1, pl.ldq1, part, nullptr, st, route, ctl + 34, G, emax_slot(20)));
    CQ_DEBUG_SYNC("route 3");
    CQ_DEBUG_SYNC("route 4");
    g.pass = 2; g.shift_mode = 0; g.G = G; g.R = R2; g.X = X2; g.R1 = R1; g.emax = emax_slot(20);
    g.Rout = Racc; g.ldr = pl.np; g.rout_full = 1; g.rank_flag = nullptr; g.stats = nullptr; g.counter = counter(17);
    // basis-only: the second pass writes into Out, and when Q₂ is already a
    // well-conditioned basis (κ₂(Q₁) small: decided on the device from R₂) the
    // route ends there — four of its six m-row passes
    double* Q2b = basis ? Out : Q2;
    const long ldq2 = basis ? ldo : pl.ldq1;
    if (basis) {
      g.basis_done = ctl + 14;
      g.basis_diag_max = CQ_BASIS2_DIAG_MAX;
      g.rank_flag = rank_flag;  // diag(R₂)∘diag(R₁); the last factorization overwrites it when it runs
    }
    PBQ_TRY(factor_launch(ctx, pl, g, st));
    g.basis_done = nullptr;
    CQ_DEBUG_SYNC("route 5");
    PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, Q1, pl.ldq1, X2, pl.np, 0.0, Q2b, ldq2, nullptr, gws, pl.gemm_ws,
                               st, nullptr, true, route));
    if (basis) {
      basis_exit_kernel<<<1, 1, 0, st>>>(ctl + 14, route, fallback);
      PBQ_CUDA(ctx, cudaGetLastError());
      ctx->launches += 1;
    }
    CQ_DEBUG_SYNC("route 6");
    PBQ_TRY(gram_launch(ctx, pl, m, n, Q2b, ldq2, part, nullptr, st, route, ctl + 35, G, emax_slot(22)));
    CQ_DEBUG_SYNC("route 7");
    CQ_DEBUG_SYNC("route 8");
    g.R = R1; g.X = X1; g.R1 = Racc; g.emax = emax_slot(22);   // R = R₃·(R₂·R₁)
    g.Rout = R; g.ldr = ldr; g.rout_full = 0; g.rank_flag = rank_flag; g.stats = ctx->cq_stats;
    g.route_final = 1; g.counter = counter(18);
    PBQ_TRY(factor_launch(ctx, pl, g, st));
    CQ_DEBUG_SYNC("route 9");
    PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, Q2b, ldq2, X1, pl.np, 0.0, A, lda, nullptr, gws, pl.gemm_ws, st,
                               nullptr, true, route));
    CQ_DEBUG_SYNC("route 10");
  }
  // Householder fallback (returns immediately unless a factorization failed)
  PBQ_TRY(hh_launch(ctx, m, n, A, lda, R, ldr, 1, rank_flag, hws, hws_bytes, st, ext ? hh_req : fallback,
                    reinterpret_cast<unsigned int*>(ctl + 48)));
  if (basis) {
    copy_if_kernel<<<unsigned(std::min<long>(ceil_div(m * n, 256L * 8), 4L * ctx->sms)), 256, 0, st>>>(fallback, A, lda, Out,
                                                                                                     ldo, m, n);
    PBQ_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
  }
  return PBQ_OK;
}

// ------------------------------------------- distributed Cholesky-QR2 ----
// Row-sharded A (this rank's m×n rows): the chain of cq_launch split at its
// two Gram matrices, which the caller allreduces (sum) across ranks between
// stages.  Every rank then factors the same global Gram → identical R.
//   stage 0: G ← AᵀA (local)
//   stage 1: [G global] R₁ (κ guard → *fallback), Q₁ = A·R₁⁻¹, G ← Q₁ᵀQ₁ (local)
//   stage 2: [G global] R = R₂R₁ (+ rank flag), A ← Q₁·R₂⁻¹
// On *fallback (κ₁ > 1e6, or a failed pass 2) A is left untouched and the
// caller runs its TSQR instead.  The workspace persists across the stages.
size_t cqd_ws_bytes(const CqPlan& p, long m) {
  const size_t sq = align_up(size_t(p.np) * p.np * sizeof(double), 256);
  return 256 + 5 * sq + align_up(2 * size_t(p.nb) * p.np * sizeof(double), 256) + align_up(p.gemm_ws, 256) +
         align_up(size_t(m) * p.ldq1 * sizeof(double), 256) + 1024;
}

int cqd_stage(pbq_ctx* ctx, int stage, long m, long n, double* A, long lda, double* R, long ldr, int32_t* rank_flag,
              double* G, int32_t* fallback, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (m < n || n < 1) return fail(ctx, PBQ_ERR_DIM, "cholqr2_dist: needs m >= n >= 1 (got %ldx%ld)", m, n);
  if (lda < n || (R && ldr < n)) return fail(ctx, PBQ_ERR_PARAM, "cholqr2_dist: leading dimension too small");
  if ((lda & 1) || !aligned16(A)) return fail(ctx, PBQ_ERR_PARAM, "cholqr2_dist: lda must be even and A 16-byte aligned");
  if (!G || !fallback || !R) return fail(ctx, PBQ_ERR_PARAM, "cholqr2_dist: null pointer argument");
  const CqPlan pl = cq_plan(ctx, m, n);
  const size_t sq = size_t(pl.np) * pl.np;
  Carve cv(ws, ws_bytes);
  int* ctl = cv.take<int>(64);  // [1] [2] grid-barrier counters, [4] emax of pass 2
  double* X1 = cv.take<double>(sq);
  double* X2 = cv.take<double>(sq);
  // the factor kernel writes only the upper triangle of R⁻¹ and the products
  // read the whole np×np block: ctl, X1 and X2 start zeroed (as in cq_launch)
  const size_t zero_bytes = size_t(reinterpret_cast<char*>(X2 + sq) - reinterpret_cast<char*>(ctl));
  double* R1 = cv.take<double>(sq);
  double* R2 = cv.take<double>(sq);
  double* T = cv.take<double>(sq);
  double* colsum = cv.take<double>(2 * size_t(pl.nb) * pl.np);
  char* gws = cv.take<char>(pl.gemm_ws);
  double* Q1 = cv.take<double>(size_t(m) * pl.ldq1);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "cholqr2_dist: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  double* part = reinterpret_cast<double*>(gws);
  auto counter = [&](int i) { return reinterpret_cast<unsigned int*>(ctl + i); };
  auto emax_slot = [&](int i) { return reinterpret_cast<unsigned long long*>(ctl + i); };
  ProfScope ps(ctx->prof, st, 1);
  ProfSuppress quiet(ctx->prof);
  const unsigned fix_grid = unsigned(std::min<long>(ceil_div(long(sq), 256), 64));
  CqArgs f;
  memset(&f, 0, sizeof(f));
  f.nb = pl.nb; f.n = n; f.np = pl.np; f.m = m;
  f.G = G; f.T = T; f.fallback = fallback;
  f.colsum = colsum; f.stats = ctx->cq_stats; f.fail_stats = ctx->cq_stats;
  f.kappa_max = CQ_KAPPA_MAX;
  f.phase_ns = ctx->qr_phase_ns;
  f.allow_series = ctx->qr_method != PBQ_QR_CHOLQR_NOSERIES;
  if (stage == 0) {
    PBQ_CUDA(ctx, cudaMemsetAsync(ctl, 0, zero_bytes, st));
    PBQ_CUDA(ctx, cudaMemsetAsync(fallback, 0, sizeof(int32_t), st));
    PBQ_TRY(gram_launch(ctx, pl, m, n, A, lda, part, nullptr, st, nullptr, ctl + 32, G));
    return PBQ_OK;
  }
  if (stage == 1) {
    cholqr_dist_fix<<<fix_grid, 256, 0, st>>>(G, n, pl.np, nullptr);
    PBQ_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
    f.pass = 1; f.R = R1; f.X = X1; f.counter = counter(1);
    PBQ_TRY(factor_launch(ctx, pl, f, st));
    PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, A, lda, X1, pl.np, 0.0, Q1, pl.ldq1, nullptr, gws, pl.gemm_ws, st,
                               fallback, true));
    PBQ_TRY(gram_launch(ctx, pl, m, n, Q1, pl.ldq1, part, fallback, st, nullptr, ctl + 33, G));
    return PBQ_OK;
  }
  if (stage == 2) {
    cholqr_dist_fix<<<fix_grid, 256, 0, st>>>(G, n, pl.np, emax_slot(4));
    PBQ_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
    f.pass = 2; f.R = R2; f.X = X2; f.R1 = R1; f.Rout = R; f.ldr = ldr; f.rank_flag = rank_flag;
    f.emax = emax_slot(4); f.counter = counter(2);
    PBQ_TRY(factor_launch(ctx, pl, f, st));
    PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, Q1, pl.ldq1, X2, pl.np, 0.0, A, lda, nullptr, gws, pl.gemm_ws, st,
                               fallback, true));
    return PBQ_OK;
  }
  if (stage == 3) {
    // basis-only finish (after stage 0 and the Gram allreduce): R₁, then
    // A ← A·R₁⁻¹ = Q·R₂ — one Gram exchange instead of two (see cq_launch)
    cholqr_dist_fix<<<fix_grid, 256, 0, st>>>(G, n, pl.np, nullptr);
    PBQ_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
    f.pass = 1; f.R = R1; f.X = X1; f.counter = counter(1);
    f.basis = 1; f.rank_flag = rank_flag;
    f.kappa_max = CQ_KAPPA_MAX_BASIS;
    PBQ_TRY(factor_launch(ctx, pl, f, st));
    PBQ_TRY(gemm_launch<false>(ctx, m, n, n, 1.0, A, lda, X1, pl.np, 0.0, Q1, pl.ldq1, nullptr, gws, pl.gemm_ws, st,
                               fallback, true));
    copy_if_kernel<<<unsigned(std::min<long>(ceil_div(m * n, 256L * 8), 4L * ctx->sms)), 256, 0, st>>>(
        fallback, Q1, pl.ldq1, A, lda, m, n, 1);
    PBQ_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
    return PBQ_OK;
  }
  return fail(ctx, PBQ_ERR_PARAM, "cholqr2_dist: stage must be 0, 1, 2 or 3");
}

// ------------------------------------------- single-launch Cholesky-QR2 ----
// cholqr_small_f64.cuh: n ≤ 128 and at most CS_MAX_CHUNKS 32-row chunks per
// CTA, where the 7-launch chain is launch/barrier-bound.
constexpr long CS_MAX_CHUNKS = 2;
bool cs_eligible(const pbq_ctx* ctx, long m, long n) {
  return (ctx->qr_method == PBQ_QR_AUTO || ctx->qr_method == PBQ_QR_CHOLQR_NOSERIES) && n >= 1 &&
         n <= 32L * CS_MAX_NB && m >= n && ceil_div(m, 32) <= CS_MAX_CHUNKS * ctx->sms;
}
int cs_grid(const pbq_ctx* ctx, long m) { return int(std::max<long>(1, std::min<long>(ceil_div(m, 32), ctx->sms))); }
size_t cs_ws_bytes(const pbq_ctx* ctx, const QrPlan& hp, long m, long n) {
  const long nb = ceil_div(n, 32), np = 32 * nb, nblk = nb * (nb + 1) / 2;
  return 256 + align_up(size_t(cs_grid(ctx, m)) * nblk * 1024 * 8, 256) + 2 * align_up(size_t(nblk) * 1024 * 8, 256) +
         align_up(size_t(m) * np * 8, 256) + qr_ws_bytes(hp, n) + 1024;
}
using CsFn = void (*)(CsArgs);
CsFn cs_fn(int nb) {
  switch (nb) {
    case 1: return cholqr_small_kernel<1>;
    case 2: return cholqr_small_kernel<2>;
    case 3: return cholqr_small_kernel<3>;
    default: return cholqr_small_kernel<4>;
  }
}
size_t cs_smem(int nb) {
  switch (nb) {
    case 1: return cs_smem_bytes<1>();
    case 2: return cs_smem_bytes<2>();
    case 3: return cs_smem_bytes<3>();
    default: return cs_smem_bytes<4>();
  }
}

int cs_launch(pbq_ctx* ctx, long m, long n, double* A, long lda, double* R, long ldr, int32_t* rank_flag, void* ws,
              size_t ws_bytes, cudaStream_t st) {
  QrPlan hp;
  PBQ_TRY(qr_plan(ctx, m, n, hp));
  if (lda < n || (R && ldr < n)) return fail(ctx, PBQ_ERR_PARAM, "qr: leading dimension too small");
  const int nb = int(ceil_div(n, 32)), nblk = nb * (nb + 1) / 2;
  const long np = 32L * nb;
  const int grid = cs_grid(ctx, m);
  Carve cv(ws, ws_bytes);
  int* ctl = cv.take<int>(64);  // [0] fallback, [8] grid barrier, [16..17] emax, [48] Householder barrier
  double* part = cv.take<double>(size_t(grid) * nblk * 1024);
  double* G = cv.take<double>(size_t(nblk) * 1024);
  double* R1 = cv.take<double>(size_t(nblk) * 1024);
  double* Q1 = cv.take<double>(size_t(m) * np);
  const size_t hws_bytes = qr_ws_bytes(hp, n);
  char* hws = cv.take<char>(hws_bytes);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "qr: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  PBQ_CUDA(ctx, cudaMemsetAsync(ctl, 0, 64 * sizeof(int), st));
  CsArgs a;
  memset(&a, 0, sizeof(a));
  a.m = m; a.n = n; a.np = np; a.A = A; a.lda = lda; a.R = R; a.ldr = ldr;
  a.rank_flag = rank_flag; a.fallback = ctl; a.Q1 = Q1; a.part = part; a.G = G; a.R1 = R1;
  a.emax = reinterpret_cast<unsigned long long*>(ctl + 16);
  a.counter = reinterpret_cast<unsigned int*>(ctl + 8);
  a.stats = ctx->cq_stats;
  a.kappa_max = CQ_KAPPA_MAX;
  a.allow_series = ctx->qr_method != PBQ_QR_CHOLQR_NOSERIES;
  a.phase_ns = ctx->qr_phase_ns;
  const CsFn fn = cs_fn(nb);
  const size_t smem = cs_smem(nb);
  {
    ProfScope ps(ctx->prof, st, 1);
    ProfSuppress quiet(ctx->prof);
    PBQ_CUDA(ctx, ensure_smem(ctx, reinterpret_cast<const void*>(fn), smem));
    void* args[] = {&a};
    PBQ_CUDA(ctx, cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid), dim3(CS_THREADS), args, smem, st));
    ctx->launches += 1;
    // Householder fallback (returns at once unless a factorization failed)
    PBQ_TRY(hh_launch(ctx, m, n, A, lda, R, ldr, 1, rank_flag, hws, hws_bytes, st, ctl,
                      reinterpret_cast<unsigned int*>(ctl + 48)));
  }
  return PBQ_OK;
}

// ------------------------------------------ single-launch, 128 < n ≤ 256 ----
// cholqr_mid_f64.cuh: few rows (the d×d second stage at d = 256): the chain's
// small GEMMs and launch gaps folded into one cooperative kernel around the
// same distributed factorization.
constexpr long CM_MAX_M = 1024;  // 2048×256: 230 µs against the chain's 192 (its TMA GEMMs win there)
bool cm_eligible(const pbq_ctx* ctx, long m, long n) {
  return (ctx->qr_method == PBQ_QR_AUTO || ctx->qr_method == PBQ_QR_CHOLQR_NOSERIES) && n > 32L * CS_MAX_NB &&
         n <= 256 && m >= n && m <= CM_MAX_M;
}
int cm_grid(const pbq_ctx* ctx) { return int(std::min<long>(ctx->sms, 128)); }
size_t cm_ws_bytes(const pbq_ctx* ctx, const QrPlan& hp, long m, long n) {
  const long nb = ceil_div(n, 32), np = 32 * nb, nblk = nb * (nb + 1) / 2, nch = ceil_div(m, 32);
  const size_t sq = align_up(size_t(np) * np * 8, 256);
  return 256 + 7 * sq + align_up(2 * size_t(nb) * np * 8, 256) + align_up(size_t(m) * np * 8, 256) +
         align_up(size_t(nch) * nblk * 1024 * 8, 256) + qr_ws_bytes(hp, n) + 1024;
}

int cm_launch(pbq_ctx* ctx, long m, long n, double* A, long lda, double* R, long ldr, int32_t* rank_flag, void* ws,
              size_t ws_bytes, cudaStream_t st) {
  QrPlan hp;
  PBQ_TRY(qr_plan(ctx, m, n, hp));
  if (lda < n || (R && ldr < n)) return fail(ctx, PBQ_ERR_PARAM, "qr: leading dimension too small");
  const int nb = int(ceil_div(n, 32)), nblk = nb * (nb + 1) / 2;
  const long np = 32L * nb, nch = ceil_div(m, 32);
  const size_t sq = size_t(np) * np;
  Carve cv(ws, ws_bytes);
  // ctl: [0] fallback, [1] [2] factor barriers, [4..5] max|G₂ − I|, [8] kernel barrier, [48] Householder barrier
  int* ctl = cv.take<int>(64);
  double* X1 = cv.take<double>(sq);
  double* X2 = cv.take<double>(sq);
  const size_t zero_bytes = size_t(reinterpret_cast<char*>(X2 + sq) - reinterpret_cast<char*>(ctl));
  double* G = cv.take<double>(sq);
  double* R1 = cv.take<double>(sq);
  double* R2 = cv.take<double>(sq);
  double* T = cv.take<double>(sq);
  double* colsum = cv.take<double>(2 * size_t(nb) * np);
  double* Q1 = cv.take<double>(size_t(m) * np);
  double* part = cv.take<double>(size_t(nch) * nblk * 1024);
  const size_t hws_bytes = qr_ws_bytes(hp, n);
  char* hws = cv.take<char>(hws_bytes);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "qr: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  PBQ_CUDA(ctx, cudaMemsetAsync(ctl, 0, zero_bytes, st));
  CmArgs a;
  memset(&a, 0, sizeof(a));
  a.m = m; a.n = n; a.np = np; a.nb = nb; a.A = A; a.lda = lda; a.Q1 = Q1; a.part = part;
  a.counter = reinterpret_cast<unsigned int*>(ctl + 8);
  a.fallback = ctl;
  a.emax = reinterpret_cast<unsigned long long*>(ctl + 4);
  CqArgs f;
  memset(&f, 0, sizeof(f));
  f.nb = nb; f.n = n; f.np = np; f.m = m;
  f.G = G; f.T = T; f.fallback = ctl;
  f.emax = a.emax; f.colsum = colsum; f.stats = ctx->cq_stats; f.fail_stats = ctx->cq_stats;
  f.kappa_max = CQ_KAPPA_MAX;
  f.phase_ns = ctx->qr_phase_ns;
  f.allow_series = ctx->qr_method != PBQ_QR_CHOLQR_NOSERIES;
  f.chol_1warp = 0;
  a.f1 = f;
  a.f1.pass = 1; a.f1.R = R1; a.f1.X = X1; a.f1.counter = reinterpret_cast<unsigned int*>(ctl + 1);
  a.f2 = f;
  a.f2.pass = 2; a.f2.R = R2; a.f2.X = X2; a.f2.R1 = R1; a.f2.Rout = R; a.f2.ldr = ldr; a.f2.rank_flag = rank_flag;
  a.f2.counter = reinterpret_cast<unsigned int*>(ctl + 2);
  const int grid = cm_grid(ctx);
  {
    ProfScope ps(ctx->prof, st, 1);
    ProfSuppress quiet(ctx->prof);
    PBQ_CUDA(ctx, ensure_smem(ctx, reinterpret_cast<const void*>(&cholqr_mid_kernel), CQ_SMEM_BYTES));
    void* args[] = {&a};
    PBQ_CUDA(ctx, cudaLaunchCooperativeKernel(reinterpret_cast<void*>(&cholqr_mid_kernel), dim3(grid),
                                              dim3(CQ_THREADS), args, CQ_SMEM_BYTES, st));
    ctx->launches += 1;
    PBQ_TRY(hh_launch(ctx, m, n, A, lda, R, ldr, 1, rank_flag, hws, hws_bytes, st, ctl,
                      reinterpret_cast<unsigned int*>(ctl + 48)));
  }
  return PBQ_OK;
}

size_t qr_any_ws_bytes(const pbq_ctx* ctx, const QrPlan& hp, long m, long n) {
  if (ctx->qr_method == PBQ_QR_HOUSEHOLDER) return qr_ws_bytes(hp, n);
  size_t b = cq_ws_bytes(cq_plan(ctx, m, n), hp, m, n);
  if (cs_eligible(ctx, m, n)) b = std::max(b, cs_ws_bytes(ctx, hp, m, n));
  if (cm_eligible(ctx, m, n)) b = std::max(b, cm_ws_bytes(ctx, hp, m, n));
  return b;
}

int qr_launch(pbq_ctx* ctx, long m, long n, double* A, long lda, double* R, long ldr, int want_q, int32_t* rank_flag,
              void* ws, size_t ws_bytes, cudaStream_t st) {
  if (want_q && cs_eligible(ctx, m, n)) return cs_launch(ctx, m, n, A, lda, R, ldr, rank_flag, ws, ws_bytes, st);
  if (want_q && cm_eligible(ctx, m, n)) return cm_launch(ctx, m, n, A, lda, R, ldr, rank_flag, ws, ws_bytes, st);
  if (ctx->qr_method != PBQ_QR_HOUSEHOLDER && want_q) return cq_launch(ctx, m, n, A, lda, R, ldr, rank_flag, ws, ws_bytes, st);
  return hh_launch(ctx, m, n, A, lda, R, ldr, want_q, rank_flag, ws, ws_bytes, st, nullptr);
}

// Basis-only orth for an operand that is multiplied by A and orthonormalised
// again (the intermediate orth calls of the power iterations,
// algorithms.py:196-205): QR is invariant under right-multiplication by an
// upper-triangular matrix with positive diagonal — qr(A·Q·T) has the Q factor
// of qr(A·Q) — so the next orth returns the same basis from B = Q·T, T = R₂
// of Cholesky-QR2, as from Q itself.  On the chain route only the first
// Cholesky-QR pass runs and B lands in Out; the single-launch routes and the
// Householder method factor A in place.  *res / *ldres: where the basis is.
bool basis_route(const pbq_ctx* ctx, long m, long n) {
  return ctx->basis_orth && ctx->qr_method != PBQ_QR_HOUSEHOLDER && !cs_eligible(ctx, m, n) && !cm_eligible(ctx, m, n);
}

int orth_basis_launch(pbq_ctx* ctx, long m, long n, double* A, long lda, double* Out, long ldo, int32_t* rank_flag,
                      void* ws, size_t ws_bytes, cudaStream_t st, double** res, long* ldres) {
  if (Out && basis_route(ctx, m, n)) {
    *res = Out;
    *ldres = ldo;
    return cq_launch(ctx, m, n, A, lda, nullptr, 0, rank_flag, ws, ws_bytes, st, Out, ldo);
  }
  *res = A;
  *ldres = lda;
  return qr_launch(ctx, m, n, A, lda, nullptr, 0, 1, rank_flag, ws, ws_bytes, st);
}

// -------------------------------------------------------------- sketch ----
struct SketchPlan {
  long n_chunks;
  long vchunk0;  // first chunk that can hold a requested normal (normal index ≤ stream position)
};

SketchPlan sketch_plan(long rows, long cols, long row_offset) {
  const long last = (row_offset + rows) * cols;
  SketchPlan p;
  // ~1.0223 words per normal; 5% + 4 chunks of head-room (shortfall is detected)
  p.n_chunks = ceil_div(long(double(last) * 1.05) + 2 * PBQ_SK_CHUNK, PBQ_SK_CHUNK) + 2;
  p.vchunk0 = std::min(p.n_chunks - 1, (row_offset * cols) / PBQ_SK_CHUNK);
  return p;
}

size_t sketch_ws_bytes(const SketchPlan& p) {
  const size_t n = p.n_chunks, nv = p.n_chunks - p.vchunk0;
  return align_up(n * 4, 256) + align_up(n * PBQ_SK_E * 4, 256) + align_up(n * 8, 256) + align_up(n * 4, 256) +
         align_up(nv * PBQ_SK_CHUNK * 8, 256) + align_up(nv * 2 * PBQ_SK_MAXSPECIAL * 8, 256) + align_up(nv * 4, 256) +
         256 + 256;
}

int sketch_tables(pbq_ctx* ctx) {
  if (ctx->sketch_tables_ready) return PBQ_OK;
  PBQ_CUDA(ctx, cudaMemcpyToSymbol(c_zig_ki, pbq_zig_ki, sizeof(pbq_zig_ki)));
  PBQ_CUDA(ctx, cudaMemcpyToSymbol(c_zig_wi, pbq_zig_wi, sizeof(pbq_zig_wi)));
  PBQ_CUDA(ctx, cudaMemcpyToSymbol(c_zig_fi, pbq_zig_fi, sizeof(pbq_zig_fi)));
  ctx->sketch_tables_ready = true;
  return PBQ_OK;
}

int sketch_launch(pbq_ctx* ctx, long rows, long cols, long row_offset, uint64_t k0, uint64_t k1, double* out,
                  long ldo, int* error_flag, void* ws, size_t ws_bytes, cudaStream_t st,
                  const uint64_t* seed_dev = nullptr) {
  if (rows < 1 || cols < 1 || row_offset < 0) return fail(ctx, PBQ_ERR_DIM, "gaussian: bad shape");
  if (ldo < cols) return fail(ctx, PBQ_ERR_PARAM, "gaussian: ldo < cols");
  PBQ_TRY(sketch_tables(ctx));
  const SketchPlan pl = sketch_plan(rows, cols, row_offset);
  Carve cv(ws, ws_bytes);
  SketchArgs a;
  a.k0 = k0; a.k1 = k1;
  a.seed_dev = seed_dev;
  a.n_chunks = pl.n_chunks;
  a.vchunk0 = pl.vchunk0;
  a.first = row_offset * cols;
  a.count = rows * cols;
  a.cols = cols;
  a.out = out; a.ldo = ldo;
  a.exits = cv.take<int>(pl.n_chunks);
  a.counts = cv.take<int>(size_t(pl.n_chunks) * PBQ_SK_E);
  a.base = cv.take<long>(pl.n_chunks);
  a.entry = cv.take<int>(pl.n_chunks);
  a.vals = cv.take<double>(size_t(pl.n_chunks - pl.vchunk0) * PBQ_SK_CHUNK);
  a.sp = cv.take<uint64_t>(size_t(pl.n_chunks - pl.vchunk0) * 2 * PBQ_SK_MAXSPECIAL);
  a.nsp = cv.take<int>(pl.n_chunks - pl.vchunk0);
  int* own_err = cv.take<int>(1);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "gaussian: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  a.error = error_flag ? error_flag : own_err;
  if (!error_flag) PBQ_CUDA(ctx, cudaMemsetAsync(own_err, 0, sizeof(int), st));
  const unsigned sk_grid = unsigned(ceil_div(pl.n_chunks, PBQ_SK_WARPS));
  ProfScope ps(ctx->prof, st, 2);
  sketch_k1<<<dim3(sk_grid), PBQ_SK_THREADS, 0, st>>>(a);
  PBQ_CUDA(ctx, cudaGetLastError());
  sketch_k2<<<1, 1024, 0, st>>>(a);
  PBQ_CUDA(ctx, cudaGetLastError());
  sketch_k3<<<dim3(sk_grid), PBQ_SK_THREADS, 0, st>>>(a);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 3;
  return PBQ_OK;
}

// ----------------------------------------------------------- helpers ----
// dst (cols×rows) = srcᵀ for src rows×cols; `lower` (square only) keeps the
// lower triangle of srcᵀ and zeros the rest (L = tril(R̃ᵀ)).
__global__ void transpose_kernel(long rows, long cols, const double* __restrict__ src, long lds,
                                 double* __restrict__ dst, long ldd, int lower) {
  pdl_trigger();
  __shared__ double tile[32][33];
  const long bx = long(blockIdx.x) * 32, by = long(blockIdx.y) * 32;  // bx: src column block, by: src row block
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long r = by + j, c = bx + threadIdx.x;
    tile[j][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long r = bx + j, c = by + threadIdx.x;  // dst[r][c] = src[c][r]
    if (r < cols && c < rows) dst[r * ldd + c] = (lower && c > r) ? 0.0 : tile[threadIdx.x][j];
  }
}

int transpose_launch(pbq_ctx* ctx, long n, const double* src, long lds, double* dst, long ldd, int lower,
                     cudaStream_t st, long cols = -1) {
  const long rows = n;
  if (cols < 0) cols = n;
  dim3 grid(unsigned(ceil_div(cols, 32)), unsigned(ceil_div(rows, 32)));
  ProfScope ps(ctx->prof, st, 3);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(rows, cols, src, lds, dst, ldd, lower);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

long thin_ld(long d) { return (d + 1) & ~1L; }

// ------------------------------------------------ column-pivoted QR pivots --
// cpqr_f64.cuh: pivot order of LAPACK dgeqp3 for a row-major m×n matrix.
// Shared-memory layout of cpqr_pivot_kernel, or 0 when it exceeds the opt-in
// limit and the per-CTA vectors live in a global (L2-resident) scratch.
size_t cpqr_smem(const pbq_ctx* ctx, long m, long n) {
  const size_t b = cp_scratch_bytes(m, n);
  return b <= ctx->smem_optin ? b : 0;
}

int cpqr_grid(pbq_ctx* ctx, long m, long n, int& grid) {
  const size_t smem = cpqr_smem(ctx, m, n);
  PBQ_CUDA(ctx, cudaFuncSetAttribute(reinterpret_cast<void*>(&cpqr_pivot_kernel),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  PBQ_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cpqr_pivot_kernel, CP_THREADS, smem));
  if (per_sm < 1) return fail(ctx, PBQ_ERR_DIM, "cpqr: kernel does not fit on an SM");
  grid = int(std::max(1L, std::min(long(ctx->sms), ceil_div(n, CP_WARPS))));
  return PBQ_OK;
}

size_t cpqr_ws_bytes(const pbq_ctx* ctx, long m, long n, int grid) {
  const long ldw = (m + 1) & ~1L;
  size_t b = align_up(size_t(n) * ldw * 8, 256) + 2 * align_up(size_t(n) * 8, 256) + 256 + 256;
  if (!cpqr_smem(ctx, m, n)) b += size_t(grid) * align_up(cp_scratch_bytes(m, n), 256) + 256;
  return b;
}

// Single-cluster plan: C CTAs (one column per warp where possible, C ≤ 16)
// holding all n columns in shared memory.  Returns false when it does not fit.
using CpClusterFn = void (*)(CpClusterArgs);
CpClusterFn cpqr_cluster_fn(long m) {
  if (m <= 256) return cpqr_cluster_kernel<8>;
  if (m <= 512) return cpqr_cluster_kernel<16>;
  return cpqr_cluster_kernel<32>;
}

bool cpqr_cluster_plan(pbq_ctx* ctx, long m, long n, int& C, int& nc, size_t& smem) {
  static int max_c_by_t[3] = {-1, -1, -1};  // largest launchable cluster per instantiation at full shared memory
  int& max_c = max_c_by_t[m <= 256 ? 0 : (m <= 512 ? 1 : 2)];
  if (getenv("PBQ_CPQR_NO_CLUSTER")) return false;
  if (m > 1024) return false;  // the pivot column lives in registers: ≤ 32 doubles per lane
  const int cmin = int(std::min<long>(16, std::max<long>(1, ceil_div(n, CP_WARPS))));
  for (C = cmin; C <= 16; ++C) {
    nc = int(ceil_div(n, C));
    smem = cp_cluster_smem(m, n, nc, m);
    if (smem <= ctx->smem_optin) break;
  }
  if (C > 16) return false;
  if (cudaFuncSetAttribute(reinterpret_cast<void*>(cpqr_cluster_fn(m)), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(smem)) != cudaSuccess ||
      cudaFuncSetAttribute(reinterpret_cast<void*>(cpqr_cluster_fn(m)),
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (max_c < 0) {
    max_c = 0;
    for (int c = 16; c >= 1 && max_c == 0; c /= 2) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(CP_THREADS);
      cfg.dynamicSmemBytes = ctx->smem_optin;
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaFuncSetAttribute(reinterpret_cast<void*>(cpqr_cluster_fn(m)), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(ctx->smem_optin));
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, reinterpret_cast<void*>(cpqr_cluster_fn(m)), &cfg) ==
              cudaSuccess &&
          nclusters > 0)
        max_c = c;
      cudaGetLastError();
    }
    cudaFuncSetAttribute(reinterpret_cast<void*>(cpqr_cluster_fn(m)), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
  }
  return C <= max_c;
}

int cpqr_launch(pbq_ctx* ctx, long m, long n, const double* M, long ldm, int64_t* perm, void* ws, size_t ws_bytes,
                cudaStream_t st) {
  if (m < 1 || n < 1) return fail(ctx, PBQ_ERR_DIM, "cpqr: bad shape %ld x %ld", m, n);
  if (ldm < n) return fail(ctx, PBQ_ERR_PARAM, "cpqr: leading dimension too small");
  if (!M || !perm) return fail(ctx, PBQ_ERR_PARAM, "cpqr: null pointer argument");
  int grid = 0;
  PBQ_TRY(cpqr_grid(ctx, m, n, grid));
  CpArgs a;
  a.m = m; a.n = n; a.steps = std::min(m, n);
  a.ldw = (m + 1) & ~1L;
  Carve cv(ws, ws_bytes);
  a.W = cv.take<double>(size_t(n) * a.ldw);
  a.vn1 = cv.take<double>(n);
  a.vn2 = cv.take<double>(n);
  a.counter = cv.take<unsigned int>(1);
  a.perm = perm;
  const size_t smem = cpqr_smem(ctx, m, n);
  a.scratch = nullptr;
  a.scratch_stride = align_up(cp_scratch_bytes(m, n), 256);
  if (!smem) a.scratch = cv.take<unsigned char>(size_t(grid) * a.scratch_stride);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "cpqr: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  PBQ_TRY(transpose_launch(ctx, m, M, ldm, a.W, a.ldw, 0, st, n));  // W = Mᵀ: columns contiguous
  int C = 0, nc = 0;
  size_t csmem = 0;
  if (cpqr_cluster_plan(ctx, m, n, C, nc, csmem)) {
    CpClusterArgs c;
    c.m = m; c.n = n; c.steps = a.steps; c.W = a.W; c.ldw = a.ldw; c.perm = perm; c.nc = nc; c.ldc = m;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(CP_THREADS);
    cfg.dynamicSmemBytes = csmem;
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope ps(ctx->prof, st, 1);
    PBQ_CUDA(ctx, cudaLaunchKernelEx(&cfg, cpqr_cluster_fn(m), c));
    ctx->launches += 1;
    return PBQ_OK;
  }
  PBQ_CUDA(ctx, cudaMemsetAsync(a.counter, 0, sizeof(unsigned int), st));
  void* args[] = {&a};
  ProfScope ps(ctx->prof, st, 1);
  PBQ_CUDA(ctx, cudaLaunchCooperativeKernel(reinterpret_cast<void*>(&cpqr_pivot_kernel), dim3(grid),
                                            dim3(CP_THREADS), args, smem, st));
  ctx->launches += 1;
  return PBQ_OK;
}

int gather_launch(pbq_ctx* ctx, long rows, long cols, const double* src, long lds, const int64_t* perm, double* dst,
                  long ldd, cudaStream_t st) {
  if (rows < 1 || cols < 1) return fail(ctx, PBQ_ERR_DIM, "gather: bad shape %ld x %ld", rows, cols);
  if (!src || !perm || !dst) return fail(ctx, PBQ_ERR_PARAM, "gather: null pointer argument");
  if (lds < cols || ldd < cols) return fail(ctx, PBQ_ERR_PARAM, "gather: leading dimension too small");
  const long blocks = std::min(ceil_div(rows * cols, 256), long(ctx->sms) * 8);
  ProfScope ps(ctx->prof, st, 3);
  gather_cols_kernel<<<unsigned(blocks), 256, 0, st>>>(rows, cols, src, lds, perm, dst, ldd);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

// ----------------------------------------------------- Jacobi SVD core ----
// svd_f64.cuh.  Register kernel instantiations by doubles-per-lane.
using JacFn = void (*)(JacArgs);
JacFn jac_reg_fn(int vpl) {
  switch (vpl) {
    case 4: return jacobi_reg_kernel<4>;
    case 8: return jacobi_reg_kernel<8>;
    case 16: return jacobi_reg_kernel<16>;
    default: return jacobi_reg_kernel<24>;
  }
}
int jac_vpl(long V) { return V <= 128 ? 4 : V <= 256 ? 8 : V <= 512 ? 16 : 24; }
size_t jac_reg_smem(int vpl) {
  return size_t(2) * JAC_WARPS * 2 * 32 * vpl * sizeof(double) + 4 * JAC_WARPS * sizeof(uint64_t) +
         (2 * 16 * 3 + 3 * JAC_WARPS) * sizeof(double);
}

// Largest cluster of C CTAs the register kernel with `vpl` can launch (0: none).
bool jac_cluster_ok(pbq_ctx* ctx, JacFn fn, int C, size_t smem, int threads) {
  static std::unordered_map<long, bool> memo;
  const long key = (long(reinterpret_cast<uintptr_t>(fn)) << 12) ^ (long(C) << 4) ^ long(threads);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  cudaFuncSetAttribute(reinterpret_cast<void*>(fn), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(reinterpret_cast<void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  const bool ok = cudaOccupancyMaxActiveClusters(&nclusters, reinterpret_cast<void*>(fn), &cfg) == cudaSuccess &&
                  nclusters > 0;
  cudaGetLastError();
  memo[key] = ok;
  return ok;
}

size_t jacobi_core_ws_bytes(long n, long L, int accumulate) {
  const long np = n + (n & 1), V = L + (accumulate ? n : 0), ldz = V + (V & 1);
  return align_up(size_t(np) * ldz * 8, 256) + align_up(size_t(n) * 8, 256) + align_up(size_t(L) * 8, 256) + 512;
}

int jacobi_core_launch(pbq_ctx* ctx, long n, long L, const double* X, long ldx, int accumulate, double* s, double* Y,
                       long ldy, double* G, long ldg, int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 1 || L < 1) return fail(ctx, PBQ_ERR_DIM, "jacobi_svd: bad shape %ld x %ld", n, L);
  if (n > L) return fail(ctx, PBQ_ERR_DIM, "jacobi_svd: needs n <= L (got %ld x %ld)", n, L);
  if (!X || !s || !status || ldx < L || (Y && ldy < L) || (accumulate && (!G || ldg < n)))
    return fail(ctx, PBQ_ERR_PARAM, "jacobi_svd: bad pointer or leading dimension");
  if (n > (1L << 20)) return fail(ctx, PBQ_ERR_UNSUPPORTED, "jacobi_svd: n too large");
  JacArgs a;
  a.n = int(n);
  a.np = int(n + (n & 1));
  a.L = int(L);
  a.V = int(L + (accumulate ? n : 0));
  a.accumulate = accumulate ? 1 : 0;
  a.X = X;
  a.ldx = ldx;
  a.ldz = a.V + (a.V & 1);
  a.status = status;
  a.max_sweeps = 60;  // dgesvj's NSWEEP is 30 with de Rijk pivoting; plain cyclic order gets twice that
  a.tphase = ctx->qr_phase_ns ? ctx->qr_phase_ns + 40 : nullptr;  // debug hooks: [40..44) round phases
  a.tol = sqrt(double(L)) * 1.1102230246251565e-16;      // √L·u (dgesvj's CTOL)
  Carve cv(ws, ws_bytes);
  a.Z = cv.take<double>(size_t(a.np) * a.ldz);
  double* sig = cv.take<double>(n);
  double* work = cv.take<double>(L);
  int* ctl = cv.take<int>(64);  // [0] nzero, [16] grid barrier, [32..48) sweep statistics (grid kernel)
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "jacobi_svd: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  int* nzero = ctl;
  ctl += 16;
  const int P = a.np / 2;
  ProfScope ps(ctx->prof, st, 1);
  PBQ_CUDA(ctx, cudaMemsetAsync(nzero, 0, 64 * sizeof(int), st));
  bool done = false;
  if (P <= JAC_MAX_PAIRS_REG && a.V <= 32 * JAC_MAX_VPL && !getenv("PBQ_JACOBI_L2")) {
    const int vpl = jac_vpl(a.V);
    const int C = int(ceil_div(P, JAC_WARPS));
    const JacFn fn = jac_reg_fn(vpl);
    const size_t smem = jac_reg_smem(vpl);
    if (jac_cluster_ok(ctx, fn, C, smem, JAC_WARPS * 32)) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(JAC_WARPS * 32);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      PBQ_CUDA(ctx, cudaLaunchKernelEx(&cfg, fn, a));
      ctx->launches += 1;
      done = true;
    }
  }
  if (!done) {
    const long blocks = std::min(ceil_div(long(a.np) * a.V, 256), long(ctx->sms) * 4);
    jacobi_init_kernel<<<unsigned(blocks), 256, 0, st>>>(a);
    PBQ_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
    const int vpl = a.V <= 256 ? 8 : a.V <= 512 ? 16 : a.V <= 768 ? 24 : 40;  // V > 1280: streamed path
    void* fn = vpl == 8    ? reinterpret_cast<void*>(&jacobi_grid_kernel<8>)
               : vpl == 16 ? reinterpret_cast<void*>(&jacobi_grid_kernel<16>)
               : vpl == 24 ? reinterpret_cast<void*>(&jacobi_grid_kernel<24>)
                           : reinterpret_cast<void*>(&jacobi_grid_kernel<40>);
    int per_sm = 0;
    PBQ_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, JAC_GRID_WARPS * 32, 0));
    if (per_sm < 1) return fail(ctx, PBQ_ERR_UNSUPPORTED, "jacobi_svd: grid kernel cannot be resident");
    const int grid = int(std::max<long>(1, std::min<long>(ceil_div(P, JAC_GRID_WARPS), long(ctx->sms))));
    unsigned int* bar = reinterpret_cast<unsigned int*>(ctl);
    unsigned long long* stat = reinterpret_cast<unsigned long long*>(ctl + 16);
    void* args[] = {&a, &bar, &stat};
    PBQ_CUDA(ctx, cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(JAC_GRID_WARPS * 32), args, 0, st));
    ctx->launches += 1;
  }
  const unsigned wb = unsigned(ceil_div(n, 8));  // 8 warps per 256-thread block, one per vector
  jacobi_norms_kernel<<<wb, 256, 0, st>>>(a, sig);
  jacobi_output_kernel<<<wb, 256, 0, st>>>(a, sig, s, Y, ldy, G, ldg, nzero);
  if (Y) jacobi_complete_kernel<<<1, 256, 0, st>>>(int(n), int(L), Y, ldy, nzero, work);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += Y ? 3 : 2;
  return PBQ_OK;
}

// Preconditioned Jacobi (PBQ_JACOBI_PRECONDITION; Drmač & Veselić 2008, as
// LAPACK dgejsv): Xᵀ = Q_h·R (tall QR), Rᵀ = W·R̃ (the QLP step), then the
// one-sided Jacobi core on the rows of the n×n R̃, whose rows are graded like
// the singular values and far closer to orthogonal than X's — 8–12 sweeps
// instead of 25–45 on graded inputs (tools/svd_probe.py).  With
// G₃·R̃ = diag(s)·Y₃:  X = Rᵀ·Q_hᵀ = W·R̃·Q_hᵀ  ⇒  G = G₃·Wᵀ, Y = Y₃·Q_hᵀ.
struct JacPre {
  long ldn, ldL;
  size_t qr, gemm, core;
};
int jacobi_pre_plan(pbq_ctx* ctx, long n, long L, int accumulate, JacPre& p) {
  p.ldn = thin_ld(n);
  p.ldL = thin_ld(L);
  size_t a = 0, b = 0;
  PBQ_TRY(pbq_qr_workspace_bytes(ctx, L, n, &a));
  PBQ_TRY(pbq_qr_workspace_bytes(ctx, n, n, &b));
  p.qr = std::max(a, b);
  PBQ_TRY(pbq_gemm_workspace_bytes(ctx, n, L, n, &a));
  PBQ_TRY(pbq_gemm_workspace_bytes(ctx, n, n, n, &b));
  p.gemm = std::max(a, b);
  p.core = jacobi_core_ws_bytes(n, n, accumulate);
  return PBQ_OK;
}
size_t jacobi_pre_ws_bytes(const JacPre& p, long n, long L) {
  const size_t sq = align_up(size_t(n) * p.ldn * 8, 256);
  return align_up(size_t(L) * p.ldn * 8, 256) + 6 * sq + align_up(size_t(n) * p.ldL * 8, 256) + align_up(p.qr, 256) +
         align_up(p.gemm, 256) + align_up(p.core, 256) + 512;
}

int jacobi_ws_bytes(pbq_ctx* ctx, long n, long L, int flags, size_t* bytes) {
  const int acc = flags & PBQ_JACOBI_ACCUMULATE;
  if ((flags & PBQ_JACOBI_PRECONDITION) && n >= 2) {
    JacPre p;
    PBQ_TRY(jacobi_pre_plan(ctx, n, L, acc, p));
    *bytes = jacobi_pre_ws_bytes(p, n, L);
  } else {
    *bytes = jacobi_core_ws_bytes(n, L, acc);
  }
  return PBQ_OK;
}

int jacobi_launch(pbq_ctx* ctx, long n, long L, const double* X, long ldx, int flags, double* s, double* Y, long ldy,
                  double* G, long ldg, int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int acc = flags & PBQ_JACOBI_ACCUMULATE;
  if (!(flags & PBQ_JACOBI_PRECONDITION) || n < 2)
    return jacobi_core_launch(ctx, n, L, X, ldx, acc, s, Y, ldy, G, ldg, status, ws, ws_bytes, st);
  if (n > L) return fail(ctx, PBQ_ERR_DIM, "jacobi_svd: needs n <= L (got %ld x %ld)", n, L);
  if (!X || !s || !status || ldx < L || (Y && ldy < L) || (acc && (!G || ldg < n)))
    return fail(ctx, PBQ_ERR_PARAM, "jacobi_svd: bad pointer or leading dimension");
  if ((Y && ((ldy & 1) || !aligned16(Y))) || (acc && ((ldg & 1) || !aligned16(G))))
    return fail(ctx, PBQ_ERR_PARAM, "jacobi_svd: preconditioned outputs need even leading dimensions, 16-byte aligned");
  JacPre p;
  PBQ_TRY(jacobi_pre_plan(ctx, n, L, acc, p));
  Carve cv(ws, ws_bytes);
  double* H = cv.take<double>(size_t(L) * p.ldn);   // Xᵀ, then Q_h
  double* R1 = cv.take<double>(size_t(n) * p.ldn);  // R of Xᵀ
  double* T = cv.take<double>(size_t(n) * p.ldn);   // Rᵀ, then W
  double* Rt = cv.take<double>(size_t(n) * p.ldn);  // R̃
  double* Y3 = cv.take<double>(size_t(n) * p.ldn);
  double* G3 = cv.take<double>(size_t(n) * p.ldn);
  double* Wt = cv.take<double>(size_t(n) * p.ldn);
  double* Qt = cv.take<double>(size_t(n) * p.ldL);  // Q_hᵀ
  char* qws = cv.take<char>(p.qr);
  char* gws = cv.take<char>(p.gemm);
  char* cws = cv.take<char>(p.core);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "jacobi_svd: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  PBQ_TRY(transpose_launch(ctx, n, X, ldx, H, p.ldn, 0, st, L));
  PBQ_TRY(qr_launch(ctx, L, n, H, p.ldn, R1, p.ldn, 1, nullptr, qws, p.qr, st));
  PBQ_TRY(transpose_launch(ctx, n, R1, p.ldn, T, p.ldn, 0, st));
  PBQ_TRY(qr_launch(ctx, n, n, T, p.ldn, Rt, p.ldn, 1, nullptr, qws, p.qr, st));
  PBQ_TRY(jacobi_core_launch(ctx, n, n, Rt, p.ldn, acc, s, Y ? Y3 : nullptr, p.ldn, acc ? G3 : nullptr, p.ldn, status,
                             cws, p.core, st));
  if (Y) {
    PBQ_TRY(transpose_launch(ctx, L, H, p.ldn, Qt, p.ldL, 0, st, n));
    PBQ_TRY(gemm_launch<false>(ctx, n, L, n, 1.0, Y3, p.ldn, Qt, p.ldL, 0.0, Y, ldy, nullptr, gws, p.gemm, st));
  }
  if (acc) {
    PBQ_TRY(transpose_launch(ctx, n, T, p.ldn, Wt, p.ldn, 0, st));
    PBQ_TRY(gemm_launch<false>(ctx, n, n, n, 1.0, G3, p.ldn, Wt, p.ldn, 0.0, G, ldg, nullptr, gws, p.gemm, st));
  }
  return PBQ_OK;
}

// ------------------------------------------------- reconstruction residual --
// ‖A − Q_k·L_k·P_kᵀ‖_F² and ‖A‖_F² (QlpFactors.approx(rank), algorithms.py:
// 101-106; error_curve's frobenius_error, analysis.py:238-244) in one pass
// over A: M = Q_k·L_k (n1×k), Pᵀ_k (k×n2), then the ring GEMM M·Pᵀ_k with the
// RESID epilogue; the n1×n2 approximation is never stored.
__global__ void resid_final_kernel(const double* sums, int n, double* out) {
  __shared__ double s[2][256];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) {
    a += sums[2 * i];
    b += sums[2 * i + 1];
  }
  s[0][threadIdx.x] = a;
  s[1][threadIdx.x] = b;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s[0][threadIdx.x] += s[0][threadIdx.x + w];
      s[1][threadIdx.x] += s[1][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s[0][0];
    out[1] = s[1][0];
  }
}

size_t resid_ws_bytes(const pbq_ctx* ctx, long n1, long n2, long k) {
  const GemmPlan g1 = gemm_plan(ctx, n1, n2, k, false, false), g2 = gemm_plan(ctx, n1, k, k);
  const long ldk = thin_ld(k), ldn = thin_ld(n2);
  return align_up(size_t(n1) * ldk * 8, 256) + align_up(size_t(k) * ldn * 8, 256) +
         align_up(2 * size_t(ctx->sms) * 8, 256) + std::max(gemm_ws_bytes(g1), gemm_ws_bytes(g2)) + 1024;
}

int resid_launch(pbq_ctx* ctx, long n1, long n2, long k, const double* A, long lda, const double* Q, long ldq,
                 const double* L, long ldl, const double* P, long ldp, double* out, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  if (n1 < 1 || n2 < 1 || k < 1) return fail(ctx, PBQ_ERR_DIM, "residual: bad shape");
  if ((lda & 1) || (ldq & 1) || (ldl & 1) || (ldp & 1) || !aligned16(A) || !aligned16(Q) || !aligned16(L) ||
      !aligned16(P))
    return fail(ctx, PBQ_ERR_PARAM, "residual: leading dimensions must be even and pointers 16-byte aligned");
  const long ldk = thin_ld(k), ldn = thin_ld(n2);
  Carve cv(ws, ws_bytes);
  double* ql = cv.take<double>(size_t(n1) * ldk);
  double* pt = cv.take<double>(size_t(k) * ldn);
  double* sums = cv.take<double>(2 * size_t(ctx->sms));
  const GemmPlan pl = gemm_plan(ctx, n1, n2, k, false, false);
  const size_t gws_bytes = std::max(gemm_ws_bytes(pl), gemm_ws_bytes(gemm_plan(ctx, n1, k, k)));
  char* gws = cv.take<char>(gws_bytes);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "residual: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  PBQ_TRY(gemm_launch<false>(ctx, n1, k, k, 1.0, Q, ldq, L, ldl, 0.0, ql, ldk, nullptr, gws, gws_bytes, st));
  PBQ_TRY(transpose_launch(ctx, n2, P, ldp, pt, ldn, 0, st, k));
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = n1; a.N = n2; a.K = k;
  a.A = ql; a.lda = ldk; a.B = pt; a.ldb = ldn;
  a.alpha = 1.0;
  a.tiles_m = pl.tiles_m; a.tiles_n = pl.tiles_n; a.k_iters = pl.k_iters; a.total_iters = pl.total;
  a.group = pl.group;
  Carve gc(gws, gws_bytes);
  a.partials = gc.take<double>(size_t(pl.grid) * pl.bm * pl.bn);
  gc.take<int>(pl.grid);
  a.flags = gemm_flags_for(ctx, st);
  if (!a.flags) return fail(ctx, PBQ_ERR_OOM, "residual: cannot allocate stream-K flags");
  a.ref = A; a.ldref = lda; a.sums = sums;
  {
    ProfScope ps(ctx->prof, st, 0);
    PBQ_TRY(gemm_dispatch(ctx, a, false, pl.bn, GEMM_RESID, dim3(pl.grid), false, st));
  }
  resid_final_kernel<<<1, 256, 0, st>>>(sums, pl.grid, out);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

// zeroes the pipeline's status words in one launch (instead of three memset
// nodes in front of the sketch)
__global__ void pipeline_init_kernel(int32_t* nonfinite, int32_t* rank_flags, int n_rank, int32_t* sk_err) {
  const int t = threadIdx.x;
  if (t == 0 && nonfinite) *nonfinite = 0;
  if (t == 1 && sk_err) *sk_err = 0;
  for (int i = t; i < n_rank; i += blockDim.x) rank_flags[i] = 0;
}

__global__ void merge_flag_kernel(int32_t* status, const int32_t* sketch_err) {
  if (*sketch_err) *status |= 2;
}

}  // namespace

// =================================================================== C ABI ==
extern "C" {

int pbq_ctx_create(int device, pbq_ctx** out) {
  if (!out) return PBQ_ERR_PARAM;
  *out = nullptr;
  pbq_ctx* ctx = new pbq_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  int optin = 0;
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) {
    delete ctx;
    return PBQ_ERR_CUDA;
  }
  ctx->smem_optin = size_t(optin);
  {
    int l2 = 0;
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device) == cudaSuccess) ctx->l2_bytes = size_t(l2);
    if (ctx->l2_bytes == 0) ctx->l2_bytes = size_t(126) << 20;
  }
  // the GEMMs' stream-K flags live in the context, one array per stream (not
  // in the per-call workspace): they start zeroed and are reset by their
  // readers, so no launch needs a memset in front of it (which would also
  // break the programmatic launch chain).  The first batch is zeroed here.
  {
    const size_t per = size_t(std::max(ctx->sms, 1));
    int* blk = nullptr;
    if (cudaMalloc(&blk, sizeof(int) * per * kFlagBatch) != cudaSuccess ||
        cudaMemset(blk, 0, sizeof(int) * per * kFlagBatch) != cudaSuccess) {
      cudaFree(blk);
      delete ctx;
      return PBQ_ERR_CUDA;
    }
    ctx->flag_blocks.push_back(blk);
    ctx->flag_free = kFlagBatch;
  }
  *out = ctx;
  return PBQ_OK;
}

int pbq_ctx_destroy(pbq_ctx* ctx) {
  if (ctx)
    for (int* b : ctx->flag_blocks) cudaFree(b);
  if (ctx && ctx->prof.ev) {
    for (int i = 0; i < 2 * ctx->prof.cap; ++i) cudaEventDestroy(ctx->prof.ev[i]);
    delete[] ctx->prof.ev;
    delete[] ctx->prof.cls;
  }
  delete ctx;
  return PBQ_OK;
}

int pbq_profile_begin(pbq_ctx* ctx, int32_t capacity) {
  if (!ctx || capacity < 1) return PBQ_ERR_PARAM;
  PbqProfile& pr = ctx->prof;
  if (pr.cap < capacity) {
    if (pr.ev) {
      for (int i = 0; i < 2 * pr.cap; ++i) cudaEventDestroy(pr.ev[i]);
      delete[] pr.ev;
      delete[] pr.cls;
    }
    pr.ev = new cudaEvent_t[2 * capacity];
    pr.cls = new int[capacity];
    for (int i = 0; i < 2 * capacity; ++i) PBQ_CUDA(ctx, cudaEventCreate(&pr.ev[i]));
    pr.cap = capacity;
  }
  pr.used = 0;
  pr.on = true;
  return PBQ_OK;
}

int pbq_profile_end(pbq_ctx* ctx, double* ms_by_class, int32_t* launches_by_class) {
  if (!ctx) return PBQ_ERR_PARAM;
  PbqProfile& pr = ctx->prof;
  pr.on = false;
  for (int c = 0; c < 4; ++c) {
    ms_by_class[c] = 0.0;
    launches_by_class[c] = 0;
  }
  for (int i = 0; i < pr.used; ++i) {
    PBQ_CUDA(ctx, cudaEventSynchronize(pr.ev[2 * i + 1]));
    float ms = 0.f;
    PBQ_CUDA(ctx, cudaEventElapsedTime(&ms, pr.ev[2 * i], pr.ev[2 * i + 1]));
    ms_by_class[pr.cls[i]] += ms;
    launches_by_class[pr.cls[i]] += 1;
  }
  pr.used = 0;
  return PBQ_OK;
}

const char* pbq_last_error(const pbq_ctx* ctx) { return ctx ? ctx->err : "null context"; }
// Reset this thread's CUDA last-error state (e.g. after a failed stream
// capture, whose invalidation error would otherwise be reported by the next
// launch check of an unrelated call).  Returns the error that was pending.
int pbq_clear_error(pbq_ctx* ctx) {
  if (!ctx) return PBQ_ERR_PARAM;
  const cudaError_t e = cudaGetLastError();
  ctx->err[0] = 0;
  return int(e);
}
int pbq_ctx_sm_count(const pbq_ctx* ctx) { return ctx ? ctx->sms : 0; }
int64_t pbq_ctx_launch_count(const pbq_ctx* ctx) { return ctx ? ctx->launches : 0; }

int pbq_gemm_workspace_bytes(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, size_t* bytes) {
  if (!ctx || !bytes) return PBQ_ERR_PARAM;
  const int64_t k1 = std::max<int64_t>(K, 1);  // either tile choice (the scatter GEMM keeps the 128-row tiles)
  *bytes = std::max(gemm_ws_bytes(gemm_plan(ctx, M, N, k1)), gemm_ws_bytes(gemm_plan(ctx, M, N, k1, false, false)));
  return PBQ_OK;
}

int pbq_gemm_tn_scatter(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* const* land_ptrs, uint32_t* const* cnt_ptrs, int32_t rank, int32_t world,
                        int64_t S, int64_t ldl, int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx || !land_ptrs || !cnt_ptrs) return PBQ_ERR_PARAM;
  if (world < 1 || rank < 0 || rank >= world) return fail(ctx, PBQ_ERR_PARAM, "gemm scatter: bad rank/world");
  if (lda < M || ldb < N || ldl < N || (ldl & 1)) return fail(ctx, PBQ_ERR_PARAM, "gemm scatter: bad leading dimension");
  if (long(world) * S < M) return fail(ctx, PBQ_ERR_DIM, "gemm scatter: world·S < M");
  XchgScatter xs;
  xs.land = land_ptrs; xs.cnt = cnt_ptrs; xs.S = S; xs.ldl = ldl; xs.rank = rank; xs.world = world;
  // C is unused by the scatter epilogue; pass the landing pointer array's slot only for the argument checks
  return gemm_launch<true>(ctx, M, N, K, 1.0, A, lda, B, ldb, 0.0, reinterpret_cast<double*>(ws), N + (N & 1),
                           nonfinite, ws, ws_bytes, static_cast<cudaStream_t>(stream), nullptr, false, nullptr, &xs);
}

int pbq_xchg_reduce(pbq_ctx* ctx, int32_t rank, int32_t world, int64_t n2, int64_t N, int64_t S, const double* land,
                    int64_t ldl, double* const* c_ptrs, int64_t ldc, const uint32_t* cnt, uint32_t target,
                    uint32_t* const* done_ptrs, void* stream) {
  if (!ctx || !land || !c_ptrs || !cnt || !done_ptrs) return PBQ_ERR_PARAM;
  if (world < 1 || rank < 0 || rank >= world || S < 1) return fail(ctx, PBQ_ERR_PARAM, "xchg_reduce: bad arguments");
  const long row0 = long(rank) * S;
  const long rows = std::max<long>(0, std::min<long>(S, n2 - row0));
  if ((ldl & 1) || (ldc & 1) || !aligned16(land)) return fail(ctx, PBQ_ERR_PARAM, "xchg_reduce: ldl/ldc must be even, land 16-byte aligned");
  xchg_reduce_kernel<<<PBQ_XCHG_CTAS, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      land, ldl, world, S, rows, N, c_ptrs, ldc, row0, cnt, target, done_ptrs, ctx->p2p_timeout_ns);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

int pbq_p2p_push(pbq_ctx* ctx, const double* src, int64_t n, double* const* dst_ptrs, int64_t slot, int32_t rank,
                 int32_t world, uint32_t* const* cnt_ptrs, void* stream) {
  if (!ctx || !src || !dst_ptrs || !cnt_ptrs) return PBQ_ERR_PARAM;
  if (world < 1 || rank < 0 || rank >= world || n < 0) return fail(ctx, PBQ_ERR_PARAM, "p2p_push: bad arguments");
  // 16-byte pairs when src and every destination slot are aligned (the
  // peers' bases come from one symmetric allocation layout: check slot parity
  // and src here, the peer bases are 16-byte aligned allocations)
  if (aligned16(src) && !(slot & 1))
    p2p_push_kernel<true><<<PBQ_XCHG_CTAS, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, n, dst_ptrs, slot, rank,
                                                                                      world, cnt_ptrs);
  else
    p2p_push_kernel<false><<<PBQ_XCHG_CTAS, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, n, dst_ptrs, slot, rank,
                                                                                       world, cnt_ptrs);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

int pbq_p2p_sum(pbq_ctx* ctx, const double* slots, int64_t slot, int32_t world, int64_t n, double* out,
                const uint32_t* cnt, uint32_t target, uint32_t* status, void* stream) {
  if (!ctx || !slots || !out || !cnt || !status) return PBQ_ERR_PARAM;
  if (world < 1 || n < 0) return fail(ctx, PBQ_ERR_PARAM, "p2p_sum: bad arguments");
  if (aligned16(slots) && aligned16(out) && !(slot & 1))
    p2p_sum_kernel<true><<<PBQ_XCHG_CTAS, 256, 0, static_cast<cudaStream_t>(stream)>>>(slots, slot, world, n, out, cnt,
                                                                                     target, status, ctx->p2p_timeout_ns);
  else
    p2p_sum_kernel<false><<<PBQ_XCHG_CTAS, 256, 0, static_cast<cudaStream_t>(stream)>>>(slots, slot, world, n, out, cnt,
                                                                                      target, status, ctx->p2p_timeout_ns);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

int pbq_p2p_wait(pbq_ctx* ctx, const uint32_t* cnt, uint32_t target, uint32_t* status, void* stream) {
  if (!ctx || !cnt || !status) return PBQ_ERR_PARAM;
  p2p_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(cnt, target, status, ctx->p2p_timeout_ns);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

int pbq_xchg_wait(pbq_ctx* ctx, const uint32_t* done, uint32_t target, void* stream) {
  if (!ctx || !done) return PBQ_ERR_PARAM;
  xchg_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(done, target, ctx->p2p_timeout_ns);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  return PBQ_OK;
}

int pbq_set_p2p_timeout_ms(pbq_ctx* ctx, int64_t ms) {
  if (!ctx || ms < 1) return PBQ_ERR_PARAM;
  ctx->p2p_timeout_ns = (unsigned long long)ms * 1000000ull;
  return PBQ_OK;
}

int pbq_jacobi_svd_workspace_bytes(pbq_ctx* ctx, int64_t n, int64_t L, int32_t flags, size_t* bytes) {
  if (!ctx || !bytes || n < 1 || L < 1 || n > L) return PBQ_ERR_PARAM;
  return jacobi_ws_bytes(ctx, n, L, flags, bytes);
}

int pbq_jacobi_svd(pbq_ctx* ctx, int64_t n, int64_t L, const double* X, int64_t ldx, int32_t flags, double* s,
                   double* Y, int64_t ldy, double* G, int64_t ldg, int32_t* status, void* workspace,
                   size_t workspace_bytes, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  return jacobi_launch(ctx, n, L, X, ldx, flags, s, Y, ldy, G, ldg, status, workspace, workspace_bytes,
                       static_cast<cudaStream_t>(stream));
}

int pbq_xchg_expected_tiles(int64_t n2, int64_t N, int64_t S, int32_t rank, int32_t world, uint32_t* tiles) {
  if (!tiles || world < 1 || rank < 0 || rank >= world || S < 1 || N < 1) return PBQ_ERR_PARAM;
  const long rows = std::max<long>(0, std::min<long>(S, n2 - long(rank) * S));
  const long tn = N <= 64 ? 1 : ceil_div(N, 128);  // column tiles of gemm_plan
  *tiles = uint32_t(ceil_div(rows, 128) * tn * world);
  return PBQ_OK;
}

int pbq_gemm_tn(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int32_t* nonfinite, void* ws,
                size_t ws_bytes, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  if (lda < M || ldb < N || ldc < N) return fail(ctx, PBQ_ERR_PARAM, "gemm_tn: leading dimension too small");
  return gemm_launch<true>(ctx, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, nonfinite, ws, ws_bytes,
                           static_cast<cudaStream_t>(stream));
}

int pbq_gemm_nn(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int32_t* nonfinite, void* ws,
                size_t ws_bytes, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  if (lda < K || ldb < N || ldc < N) return fail(ctx, PBQ_ERR_PARAM, "gemm_nn: leading dimension too small");
  return gemm_launch<false>(ctx, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, nonfinite, ws, ws_bytes,
                            static_cast<cudaStream_t>(stream));
}

int pbq_qr_workspace_bytes(pbq_ctx* ctx, int64_t m, int64_t n, size_t* bytes) {
  if (!ctx || !bytes) return PBQ_ERR_PARAM;
  QrPlan pl;
  PBQ_TRY(qr_plan(ctx, m, n, pl));
  *bytes = qr_any_ws_bytes(ctx, pl, m, n);
  return PBQ_OK;
}

int pbq_householder_qr(pbq_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, double* R, int64_t ldr,
                       int32_t want_q, int32_t* rank_flag, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  return qr_launch(ctx, m, n, A, lda, R, ldr, want_q, rank_flag, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int pbq_orth_basis(pbq_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, double* Out, int64_t ldo,
                   int32_t* rank_flag, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx || !A || !Out) return PBQ_ERR_PARAM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ldo < n) return fail(ctx, PBQ_ERR_PARAM, "orth_basis: leading dimension too small");
  if (Out == A) return fail(ctx, PBQ_ERR_PARAM, "orth_basis: Out must not alias A (the product runs out of place)");
  double* res = nullptr;
  long ldres = 0;
  PBQ_TRY(orth_basis_launch(ctx, m, n, A, lda, Out, ldo, rank_flag, ws, ws_bytes, st, &res, &ldres));
  if (res != Out)  // in-place routes: hand the result over
    PBQ_CUDA(ctx, cudaMemcpy2DAsync(Out, ldo * sizeof(double), res, ldres * sizeof(double), n * sizeof(double), m,
                                    cudaMemcpyDeviceToDevice, st));
  return PBQ_OK;
}

int pbq_set_basis_orth(pbq_ctx* ctx, int32_t on) {
  if (!ctx) return PBQ_ERR_PARAM;
  ctx->basis_orth = on != 0;
  return PBQ_OK;
}

int pbq_gaussian_workspace_bytes(pbq_ctx* ctx, int64_t rows, int64_t cols, int64_t row_offset, size_t* bytes) {
  if (!ctx || !bytes) return PBQ_ERR_PARAM;
  *bytes = sketch_ws_bytes(sketch_plan(rows, cols, row_offset));
  return PBQ_OK;
}

int pbq_gaussian(pbq_ctx* ctx, int64_t rows, int64_t cols, int64_t row_offset, uint64_t seed_lo, uint64_t seed_hi,
                 double* out, int64_t ldo, int32_t* status, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  return sketch_launch(ctx, rows, cols, row_offset, seed_lo, seed_hi, out, ldo, status, ws, ws_bytes,
                       static_cast<cudaStream_t>(stream));
}

int pbq_debug_qr_hooks(pbq_ctx* ctx, int32_t* fallbacks, uint64_t* phase_ns, uint64_t* bar_wait_ns) {
  if (!ctx) return PBQ_ERR_PARAM;
  ctx->qr_fallbacks = fallbacks;
  ctx->qr_phase_ns = reinterpret_cast<unsigned long long*>(phase_ns);
  ctx->qr_bar_wait_ns = reinterpret_cast<unsigned long long*>(bar_wait_ns);
  return PBQ_OK;
}

int pbq_residual_workspace_bytes(pbq_ctx* ctx, int64_t n1, int64_t n2, int64_t k, size_t* bytes) {
  if (!ctx || !bytes) return PBQ_ERR_PARAM;
  if (n1 < 1 || n2 < 1 || k < 1) return fail(ctx, PBQ_ERR_DIM, "residual: bad shape");
  *bytes = resid_ws_bytes(ctx, n1, n2, k);
  return PBQ_OK;
}

int pbq_residual_fro(pbq_ctx* ctx, int64_t n1, int64_t n2, int64_t k, const double* A, int64_t lda, const double* Q,
                     int64_t ldq, const double* L, int64_t ldl, const double* P, int64_t ldp, double* out, void* ws,
                     size_t ws_bytes, void* stream) {
  if (!ctx || !out) return PBQ_ERR_PARAM;
  if (lda < n2 || ldq < k || ldl < k || ldp < k) return fail(ctx, PBQ_ERR_PARAM, "residual: leading dimension too small");
  return resid_launch(ctx, n1, n2, k, A, lda, Q, ldq, L, ldl, P, ldp, out, ws, ws_bytes,
                      static_cast<cudaStream_t>(stream));
}

int pbq_cpqr_workspace_bytes(pbq_ctx* ctx, int64_t m, int64_t n, size_t* bytes) {
  if (!ctx || !bytes) return PBQ_ERR_PARAM;
  if (m < 1 || n < 1) return fail(ctx, PBQ_ERR_DIM, "cpqr: bad shape");
  int grid = 0;
  PBQ_TRY(cpqr_grid(ctx, m, n, grid));
  *bytes = cpqr_ws_bytes(ctx, m, n, grid);
  return PBQ_OK;
}

int pbq_cpqr_pivots(pbq_ctx* ctx, int64_t m, int64_t n, const double* M, int64_t ldm, int64_t* perm, void* ws,
                    size_t ws_bytes, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  return cpqr_launch(ctx, m, n, M, ldm, perm, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int pbq_gather_columns(pbq_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds, const int64_t* perm,
                       double* dst, int64_t ldd, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  return gather_launch(ctx, rows, cols, src, lds, perm, dst, ldd, static_cast<cudaStream_t>(stream));
}

int pbq_cholqr2_dist_workspace_bytes(pbq_ctx* ctx, int64_t m, int64_t n, size_t* bytes, int64_t* ldg) {
  if (!ctx || !bytes || !ldg) return PBQ_ERR_PARAM;
  if (m < n || n < 1) return fail(ctx, PBQ_ERR_DIM, "cholqr2_dist: needs m >= n >= 1");
  const CqPlan pl = cq_plan(ctx, m, n);
  *bytes = cqd_ws_bytes(pl, m);
  *ldg = pl.np;
  return PBQ_OK;
}

int pbq_cholqr2_dist(pbq_ctx* ctx, int32_t stage, int64_t m, int64_t n, double* A, int64_t lda, double* R, int64_t ldr,
                     int32_t* rank_flag, double* G, int32_t* fallback, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  return cqd_stage(ctx, stage, m, n, A, lda, R, ldr, rank_flag, G, fallback, ws, ws_bytes,
                   static_cast<cudaStream_t>(stream));
}

int pbq_set_qr_method(pbq_ctx* ctx, int32_t method) {
  if (!ctx) return PBQ_ERR_PARAM;
  if (method != PBQ_QR_AUTO && method != PBQ_QR_HOUSEHOLDER && method != PBQ_QR_CHOLQR_NOSERIES &&
      method != PBQ_QR_CHOLQR_CHAIN)
    return fail(ctx, PBQ_ERR_PARAM, "unknown QR method %d", method);
  ctx->qr_method = method;
  return PBQ_OK;
}

int pbq_debug_cholqr_stats(pbq_ctx* ctx, int32_t* stats) {
  if (!ctx) return PBQ_ERR_PARAM;
  ctx->cq_stats = stats;
  return PBQ_OK;
}

int pbq_transpose(pbq_ctx* ctx, int64_t n, const double* src, int64_t lds, double* dst, int64_t ldd, int32_t lower,
                  void* stream) {
  if (!ctx) return PBQ_ERR_PARAM;
  return transpose_launch(ctx, n, src, lds, dst, ldd, lower, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------- second stage --
// (W, R̃) = qr(Rᵀ), L = tril(R̃ᵀ) (algorithms.py:256-257): transpose, the
// tall-QR chain on the d×d matrix, transpose into L.  (A single-CTA
// shared-memory Householder for d ≤ 160 measured slower than this chain at
// every d — tools/microbench/small_qr_single_cta_kernel.cu.)
static size_t second_stage_ws_bytes(pbq_ctx* ctx, long d) {
  size_t q = 0;
  pbq_qr_workspace_bytes(ctx, d, d, &q);
  return 2 * align_up(size_t(d) * thin_ld(d) * sizeof(double), 256) + q + 512;
}

static int second_stage_launch(pbq_ctx* ctx, long d, const double* R, long ldr, double* W, long ldw, double* L,
                               long ldl, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (d < 1) return fail(ctx, PBQ_ERR_DIM, "second stage: d must be >= 1");
  if (ldr < d || ldw < d || ldl < d) return fail(ctx, PBQ_ERR_PARAM, "second stage: leading dimension too small");
  if ((ldw & 1) || !aligned16(W)) return fail(ctx, PBQ_ERR_PARAM, "second stage: ldw must be even, W 16-byte aligned");
  const long ld = thin_ld(d);
  Carve cv(ws, ws_bytes);
  double* rt = cv.take<double>(size_t(d) * ld);
  size_t q = 0;
  PBQ_TRY(pbq_qr_workspace_bytes(ctx, d, d, &q));
  void* qws = cv.take<char>(q);
  if (!cv.ok()) return fail(ctx, PBQ_ERR_PARAM, "second stage: workspace too small (%zu < %zu)", ws_bytes, cv.off);
  PBQ_TRY(transpose_launch(ctx, d, R, ldr, W, ldw, 0, st));
  PBQ_TRY(qr_launch(ctx, d, d, W, ldw, rt, ld, 1, nullptr, qws, q, st));
  return transpose_launch(ctx, d, rt, ld, L, ldl, 1, st);
}

int pbq_second_stage_workspace_bytes(pbq_ctx* ctx, int64_t d, size_t* bytes) {
  if (!ctx || !bytes) return PBQ_ERR_PARAM;
  *bytes = second_stage_ws_bytes(ctx, d);
  return PBQ_OK;
}

int pbq_second_stage(pbq_ctx* ctx, int64_t d, const double* R, int64_t ldr, double* W, int64_t ldw, double* L,
                     int64_t ldl, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx || !R || !W || !L) return PBQ_ERR_PARAM;
  return second_stage_launch(ctx, d, R, ldr, W, ldw, L, ldl, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------- pipeline --
static int pipeline_sizes(pbq_ctx* ctx, const pbq_problem* pr, size_t* total, size_t* scratch) {
  const long n1 = pr->n1, n2 = pr->n2, d = pr->d;
  size_t g1, g2, g3, q1, q2, q3, s1 = 0;
  PBQ_TRY(pbq_gemm_workspace_bytes(ctx, n2, d, n1, &g1));
  PBQ_TRY(pbq_gemm_workspace_bytes(ctx, n1, d, n2, &g2));
  PBQ_TRY(pbq_gemm_workspace_bytes(ctx, n2, d, d, &g3));
  PBQ_TRY(pbq_qr_workspace_bytes(ctx, n2, d, &q1));
  PBQ_TRY(pbq_qr_workspace_bytes(ctx, n1, d, &q2));
  q3 = second_stage_ws_bytes(ctx, d);
  if (!pr->phi && !pr->c_init) PBQ_TRY(pbq_gaussian_workspace_bytes(ctx, n1, d, 0, &s1));
  const size_t sc = std::max({g1, g2, g3, q1, q2, q3, s1});
  const long ld = thin_ld(d);
  *scratch = sc;
  *total = align_up(size_t(n2) * ld * 8, 256) + align_up(size_t(d) * ld * 8, 256) + align_up(64, 256) + sc + 512;
  // second C and D buffers: the basis-only intermediate orth calls write out of place
  if (pr->reorthonormalize && pr->q >= 1)
    *total += align_up(size_t(n2) * ld * 8, 256) + align_up(size_t(n1) * ld * 8, 256);
  return PBQ_OK;
}

int pbq_pbp_qlp_workspace_bytes(pbq_ctx* ctx, const pbq_problem* pr, size_t* bytes) {
  if (!ctx || !pr || !bytes) return PBQ_ERR_PARAM;
  size_t scratch;
  return pipeline_sizes(ctx, pr, bytes, &scratch);
}

int pbq_pbp_qlp(pbq_ctx* ctx, const pbq_problem* pr, const pbq_outputs* o, void* ws, size_t ws_bytes, void* stream) {
  if (!ctx || !pr || !o) return PBQ_ERR_PARAM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long n1 = pr->n1, n2 = pr->n2, d = pr->d, q = pr->q;
  // argument contract of algorithms.py:239-241 (A checks, then d, then q)
  if (n1 < 1 || n2 < 1) return fail(ctx, PBQ_ERR_DIM, "a has a zero dimension: shape (%ld, %ld)", n1, n2);
  if (d < 1 || d > std::min(n1, n2)) return fail(ctx, PBQ_ERR_PARAM, "d must be in [1, %ld], got %ld", std::min(n1, n2), d);
  if (q < 0) return fail(ctx, PBQ_ERR_DIM, "q must be >= 0, got %ld", q);
  if (!pr->a || !o->q || !o->l || !o->p || !o->r || !o->rank_flags || !o->nonfinite)
    return fail(ctx, PBQ_ERR_PARAM, "null pointer argument");
  if (!pr->phi && !o->phi && !pr->c_init)
    return fail(ctx, PBQ_ERR_PARAM, "seeded mode needs an output buffer for the sketch");
  size_t total, scratch;
  PBQ_TRY(pipeline_sizes(ctx, pr, &total, &scratch));
  if (ws_bytes < total) return fail(ctx, PBQ_ERR_PARAM, "pbp_qlp: workspace too small (%zu < %zu)", ws_bytes, total);
  const long ld = thin_ld(d);
  Carve cv(ws, ws_bytes);
  double* cbuf = cv.take<double>(size_t(n2) * ld);  // C, then P̄ (in place)
  double* wbuf = cv.take<double>(size_t(d) * ld);   // W of the second stage
  int32_t* sk_err = cv.take<int32_t>(16);
  void* sc = cv.take<char>(scratch);
  const bool two_buf = pr->reorthonormalize && q >= 1;
  double* c2buf = two_buf ? cv.take<double>(size_t(n2) * ld) : nullptr;  // basis-only orth(C) output
  double* d2buf = two_buf ? cv.take<double>(size_t(n1) * ld) : nullptr;  // basis-only orth(D) output
  const int32_t check = pr->check_finite ? 1 : 0;

  pipeline_init_kernel<<<1, 64, 0, st>>>(pr->c_init ? nullptr : o->nonfinite, o->rank_flags, int(2 * q + 1),
                                         (!pr->phi && !pr->c_init) ? sk_err : nullptr);
  PBQ_CUDA(ctx, cudaGetLastError());
  ctx->launches += 1;
  const double* phi = pr->phi;
  long ldphi = pr->ldphi;
  if (pr->c_init) {
    // pass 1 done by the caller (streamed from the host): C = c_init
    PBQ_CUDA(ctx, cudaMemcpy2DAsync(cbuf, ld * sizeof(double), pr->c_init, pr->ldc_init * sizeof(double),
                                    d * sizeof(double), n2, cudaMemcpyDeviceToDevice, st));
  } else {
    if (!phi) {
      NvtxRange nv("pbq sketch: Phi = gaussian_matrix(n1, d, seed)");
      PBQ_TRY(sketch_launch(ctx, n1, d, 0, pr->seed_lo, pr->seed_hi, o->phi, o->ldphi, sk_err, sc, scratch, st,
                            pr->seed_dev));
      phi = o->phi;
      ldphi = o->ldphi;
    }
    // pass 1: C = Aᵀ Φ  (+ fused isfinite scan of A)
    NvtxRange nv("pbq pass: C = A^T Phi");
    PBQ_TRY(gemm_launch<true>(ctx, n2, d, n1, 1.0, pr->a, pr->lda, phi, ldphi, 0.0, cbuf, ld,
                              check ? o->nonfinite : nullptr, sc, scratch, st));
  }
  int site = 0;
  double* dbuf = o->q;  // n1×d scratch for A·P̄, finally D itself
  const long ldq = o->ldq;
  if (pr->reorthonormalize) {
    // every orth but the last feeds a pass that is orthonormalised again:
    // basis-only (orth_basis_launch); the last one is P̄ itself (in place, full)
    double* cb = cbuf;  // where the current basis of the row space lives
    long ldcb = ld;
    {
      NvtxRange nv("pbq orth(C)");
      if (q >= 1)
        PBQ_TRY(orth_basis_launch(ctx, n2, d, cbuf, ld, c2buf, ld, o->rank_flags + site++, sc, scratch, st, &cb, &ldcb));
      else
        PBQ_TRY(qr_launch(ctx, n2, d, cbuf, ld, nullptr, 0, 1, o->rank_flags + site++, sc, scratch, st));
    }
    for (long it = 0; it < q; ++it) {
      NvtxRange nv("pbq power iteration");
      double* db = dbuf;
      long lddb = ldq;
      PBQ_TRY(gemm_launch<false>(ctx, n1, d, n2, 1.0, pr->a, pr->lda, cb, ldcb, 0.0, dbuf, ldq, nullptr, sc, scratch, st));
      PBQ_TRY(orth_basis_launch(ctx, n1, d, dbuf, ldq, d2buf, ld, o->rank_flags + site++, sc, scratch, st, &db, &lddb));
      PBQ_TRY(gemm_launch<true>(ctx, n2, d, n1, 1.0, pr->a, pr->lda, db, lddb, 0.0, cbuf, ld, nullptr, sc, scratch, st));
      if (it + 1 < q) {
        PBQ_TRY(orth_basis_launch(ctx, n2, d, cbuf, ld, c2buf, ld, o->rank_flags + site++, sc, scratch, st, &cb, &ldcb));
      } else {
        PBQ_TRY(qr_launch(ctx, n2, d, cbuf, ld, nullptr, 0, 1, o->rank_flags + site++, sc, scratch, st));
        cb = cbuf;
        ldcb = ld;
      }
    }
  } else {
    for (long it = 0; it < q; ++it) {
      NvtxRange nv("pbq power iteration (no reorth)");
      PBQ_TRY(gemm_launch<false>(ctx, n1, d, n2, 1.0, pr->a, pr->lda, cbuf, ld, 0.0, dbuf, ldq, nullptr, sc, scratch, st));
      PBQ_TRY(gemm_launch<true>(ctx, n2, d, n1, 1.0, pr->a, pr->lda, dbuf, ldq, 0.0, cbuf, ld, nullptr, sc, scratch, st));
    }
    PBQ_TRY(qr_launch(ctx, n2, d, cbuf, ld, nullptr, 0, 1, o->rank_flags + site++, sc, scratch, st));
  }
  // D = A·P̄ ; (Q, R) = qr(D)
  {
    NvtxRange nv("pbq pass: D = A Pbar");
    PBQ_TRY(gemm_launch<false>(ctx, n1, d, n2, 1.0, pr->a, pr->lda, cbuf, ld, 0.0, dbuf, ldq, nullptr, sc, scratch, st));
  }
  {
    NvtxRange nv("pbq qr(D)");
    PBQ_TRY(qr_launch(ctx, n1, d, dbuf, ldq, o->r, o->ldr, 1, nullptr, sc, scratch, st));
  }
  // (W, R̃) = qr(Rᵀ); L = tril(R̃ᵀ); P = P̄·W
  {
    NvtxRange nv("pbq second stage: qr(R^T), L, P = Pbar W");
    PBQ_TRY(second_stage_launch(ctx, d, o->r, o->ldr, wbuf, ld, o->l, o->ldl, sc, scratch, st));
    PBQ_TRY(gemm_launch<false>(ctx, n2, d, d, 1.0, cbuf, ld, wbuf, ld, 0.0, o->p, o->ldp, nullptr, sc, scratch, st));
  }
  if (!pr->phi && !pr->c_init) {
    // fold a sketch-generator overflow into bit 1 of the status word so the
    // host reads one int
    merge_flag_kernel<<<1, 1, 0, st>>>(o->nonfinite, sk_err);
    PBQ_CUDA(ctx, cudaGetLastError());
    ctx->launches += 1;
  }
  return PBQ_OK;
}

}  // extern "C"
