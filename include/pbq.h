/*
 * pbq.h — C ABI of the B200-native PbP-QLP library (libpbq.so).
 *
 * The reference exposes PbP-QLP only as a Python function,
 *   pbpqlp.pbp_qlp(a, d, q=0, seed=0, reorthonormalize=True) -> QlpFactors
 *   (/root/reference/pkg/src/pbpqlp/algorithms.py:209-260),
 * with no FFI or plugin registry.  These entry points are the
 * device-side boundary that the drop-in Python function (package
 * `paper_2103_07245_b200`) binds through ctypes.  Every entry
 * point takes plain pointers and sizes; no torch types cross the boundary.
 *
 * Conventions
 *  - All matrices are FP64, row-major, in device memory; `ld*` is the row
 *    stride in elements and must be even, base pointers 16-byte aligned.
 *  - Work is enqueued on `stream` (a cudaStream_t passed as void*); no entry
 *    point synchronises the host except pbq_ctx_create.
 *  - Scratch memory is caller-owned: query the size, pass a device buffer.
 *    A workspace must not be shared by calls that may run concurrently.
 *  - Calls of one context may run concurrently on different streams (each
 *    with its own workspace): the GEMMs' stream-K flags are kept per stream.
 *    A CUDA graph captured from a stream uses that stream's flags, so do not
 *    replay it concurrently with other work enqueued on the capture stream.
 *  - Return value is a pbq_status; pbq_last_error() describes the last failure.
 *  - A context is bound to one device and is not thread-safe.
 */
#ifndef PBQ_H_
#define PBQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PBQ_OK = 0,
  PBQ_ERR_PARAM = 1,     /* maps to pbpqlp ParameterError  (exceptions.py:8)  */
  PBQ_ERR_DIM = 2,       /* maps to pbpqlp DimensionError  (exceptions.py:12) */
  PBQ_ERR_NONFINITE = 3, /* maps to pbpqlp MatrixInputError (exceptions.py:16) */
  PBQ_ERR_CUDA = 4,
  PBQ_ERR_NCCL = 5,
  PBQ_ERR_OOM = 6,
  PBQ_ERR_UNSUPPORTED = 7
} pbq_status;

typedef struct pbq_ctx pbq_ctx;

/* Context lifetime (one device).  Replaces nothing in the reference: the
 * reference is stateless; the context only caches device
 * properties and launch plans. */
int pbq_ctx_create(int device, pbq_ctx** out);
int pbq_ctx_destroy(pbq_ctx* ctx);
const char* pbq_last_error(const pbq_ctx* ctx);
/* Reset this thread's CUDA last-error state, returning the cudaError_t that
 * was pending (0 if none).  For hosts that recover from a failed stream
 * capture: the capture's invalidation error would otherwise surface in the
 * next launch check of an unrelated pbq_* call.  Sticky errors (a faulted
 * context) are not cleared by this and keep failing every call. */
int pbq_clear_error(pbq_ctx* ctx);
int pbq_ctx_sm_count(const pbq_ctx* ctx);
/* Kernel launches enqueued by this context since creation (evidence for the
 * bench's "gpu_launches" count). */
int64_t pbq_ctx_launch_count(const pbq_ctx* ctx);

/* C = alpha·Aᵀ·B + beta·C.  A is K×M (lda), B is K×N (ldb), C is M×N (ldc).
 * Replaces `_PassCounter.apply_t` (`a.T @ block`, algorithms.py:182-184).
 * If `nonfinite` is non-null, *nonfinite is OR-ed with 1 when A holds an
 * Inf/NaN (the `check_matrix` isfinite scan, validation.py:47, fused into the
 * pass).  Workspace: pbq_gemm_workspace_bytes(). */
int pbq_gemm_tn(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                int32_t* nonfinite, void* workspace, size_t workspace_bytes, void* stream);

/* C = alpha·A·B + beta·C.  A is M×K (lda), B is K×N (ldb), C is M×N (ldc).
 * Replaces `_PassCounter.apply` (`a @ block`, algorithms.py:178-180) and
 * `pbar @ w` (algorithms.py:258). */
int pbq_gemm_nn(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                int32_t* nonfinite, void* workspace, size_t workspace_bytes, void* stream);

int pbq_gemm_workspace_bytes(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, size_t* bytes);

/* Unpivoted Householder QR of an m×n matrix (m ≥ n ≥ 1), in place.
 * Replaces `householder_qr` (linalg.py:106-115, LAPACK dgeqrf+dorgqr through
 * np.linalg.qr(mode="reduced")) and `_fix_signs` (linalg.py:96-103).
 * On return A (if want_q) holds the thin Q, R (if non-null) the n×n upper
 * triangular factor with diag(R) ≥ 0 and exact zeros below the diagonal.
 * If rank_flag is non-null it receives the `orth` rank test
 * (linalg.py:142-165): 0 full rank, 1 some |R_ii| < 1e-14·|R_00|, 2 R_00 == 0.
 * Method (pbq_set_qr_method): by default a guarded whole-matrix Cholesky-QR2
 * (same unique factors for full-rank A, to rounding).  When κ₁(R₁) > 1e6 or
 * a pivot fails it continues, for n ≥ 384, with shifted Cholesky-QR3, and
 * otherwise (or if that fails too) hands the call to the blocked
 * Householder kernel, all decided on the device; method 1 forces the
 * Householder kernel.  For n ≤ 128 and m ≤ 64·SMs the whole Cholesky-QR2
 * runs as one cooperative launch (redundant per-CTA n×n factorizations in
 * shared memory), and for 128 < n ≤ 256 with m ≤ 1024 as another (the
 * distributed factorization with the small products folded in); method 3
 * forces the multi-launch chain instead. */
int pbq_householder_qr(pbq_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, double* R,
                       int64_t ldr, int32_t want_q, int32_t* rank_flag, void* workspace,
                       size_t workspace_bytes, void* stream);
int pbq_qr_workspace_bytes(pbq_ctx* ctx, int64_t m, int64_t n, size_t* bytes);

/* Basis-only orth (m ≥ n ≥ 1) for the intermediate `orth` calls of the power
 * iterations (algorithms.py:196-205, `basis = orth(counter.apply(basis))`),
 * whose result is only ever multiplied by A and orthonormalised again.
 * Out (m×n, ldo even, 16-byte aligned) receives B = Q·T, with Q the `orth`
 * basis of A and T upper triangular with positive diagonal, ‖TᵀT − I‖ ≲ 1e-4
 * (T = R₂ of Cholesky-QR2: only the first Cholesky-QR pass runs).  The thin
 * QR of A_next·B has the Q factor of A_next·Q (right-multiplication by T
 * leaves it unchanged), so the following orth returns what the reference
 * computes, at half the passes of this one.  rank_flag as for
 * pbq_householder_qr.  A is used as scratch and must not alias Out.  Where the chain is not the
 * route (single-launch sizes, the Householder method, a failed guard, or
 * pbq_set_basis_orth(ctx, 0)) the full QR runs and Out = Q.  Workspace:
 * pbq_qr_workspace_bytes(m, n). */
int pbq_orth_basis(pbq_ctx* ctx, int64_t m, int64_t n, double* A, int64_t lda, double* Out, int64_t ldo,
                   int32_t* rank_flag, void* workspace, size_t workspace_bytes, void* stream);

/* 1 (default): pbq_pbp_qlp runs every orth but the last one basis-only;
 * 0: every orth is the full QR (A/B switch; results agree to rounding). */
int pbq_set_basis_orth(pbq_ctx* ctx, int32_t on);

/* rows×cols standard-normal sketch, bit-identical to
 * numpy.random.Generator(numpy.random.Philox(key=seed)).standard_normal((rows, cols))
 * as drawn by `gaussian_matrix` (linalg.py:83-93): Philox4x64-10 with
 * key = (seed_lo, seed_hi), numpy's 256-layer ziggurat, element (i, j) the
 * (i·cols + j)-th normal of the stream.  `row_offset` generates rows
 * [row_offset, row_offset+rows) of the same global rows×... matrix whose
 * column count is `cols` (row-sharded multi-GPU generation). */
int pbq_gaussian(pbq_ctx* ctx, int64_t rows, int64_t cols, int64_t row_offset, uint64_t seed_lo,
                 uint64_t seed_hi, double* out, int64_t ldo, int32_t* status, void* workspace,
                 size_t workspace_bytes, void* stream);
/* `status` (device int, may be NULL) is OR-ed with a nonzero code if the
 * generator's internal bounds were exceeded (never observed; checked). */
int pbq_gaussian_workspace_bytes(pbq_ctx* ctx, int64_t rows, int64_t cols, int64_t row_offset,
                                 size_t* bytes);

/* Full single-device PbP-QLP (Algorithm 3; algorithms.py:209-260). */
typedef struct {
  int64_t n1, n2, d, q;
  const double* a; /* n1×n2 */
  int64_t lda;
  const double* phi; /* n1×d explicit sketch (oracle mode) or NULL → seeded */
  int64_t ldphi;
  uint64_t seed_lo, seed_hi;
  int32_t reorthonormalize;
  int32_t check_finite;
  /* Optional n2×d AᵀΦ computed by the caller (row stride ldc_init), e.g.
   * accumulated chunk by chunk while A streams in from the host.  When set,
   * the pipeline skips the sketch and the first pass; `phi` must then hold
   * the sketch used (it is not regenerated). */
  const double* c_init;
  int64_t ldc_init;
  /* Optional device pointer to {seed_lo, seed_hi}: when set, the sketch reads
   * its key from device memory at run time instead of seed_lo/seed_hi, so a
   * CUDA graph captured once can be replayed with new seeds. */
  const uint64_t* seed_dev;
} pbq_problem;

typedef struct {
  double* q; /* n1×d */
  int64_t ldq;
  double* l; /* d×d lower triangular, diag ≥ 0 */
  int64_t ldl;
  double* p; /* n2×d */
  int64_t ldp;
  double* r; /* d×d first-stage R, upper triangular, diag ≥ 0 */
  int64_t ldr;
  double* phi; /* n1×d: receives the seeded sketch (required when problem.phi == NULL) */
  int64_t ldphi;
  int32_t* rank_flags; /* device, 2q+1 ints: one per `orth` call in call order */
  int32_t* nonfinite;  /* device int status: bit0 A held Inf/NaN, bit1 sketch generator overflow */
} pbq_outputs;

int pbq_pbp_qlp_workspace_bytes(pbq_ctx* ctx, const pbq_problem* prob, size_t* bytes);
int pbq_pbp_qlp(pbq_ctx* ctx, const pbq_problem* prob, const pbq_outputs* out, void* workspace,
                size_t workspace_bytes, void* stream);

/* Reconstruction residual: out[0] = ‖A − Q_k·L_k·P_kᵀ‖_F²,
 * out[1] = ‖A‖_F² (device doubles), with Q_k, L_k, P_k the leading k ≤ d
 * columns / block of the factors — QlpFactors.approx(rank)
 * (algorithms.py:101-106) and error_curve's frobenius_error
 * (analysis.py:238-244) without forming the n1×n2 approximation: one pass
 * over A through a GEMM whose epilogue subtracts and accumulates.
 * Deterministic (fixed-order reductions). */
int pbq_residual_fro(pbq_ctx* ctx, int64_t n1, int64_t n2, int64_t k, const double* A, int64_t lda,
                     const double* Q, int64_t ldq, const double* L, int64_t ldl, const double* P,
                     int64_t ldp, double* out, void* workspace, size_t workspace_bytes, void* stream);
int pbq_residual_workspace_bytes(pbq_ctx* ctx, int64_t n1, int64_t n2, int64_t k, size_t* bytes);

/* Column-pivoted QR pivot order (the cor_utv core): perm[i]
 * (int64, n entries) such that M[:, perm] = Q·R is LAPACK dgeqp3's
 * factorization of the row-major m×n matrix M — the pivot rule of
 * scipy.linalg.qr(m, pivoting=True) behind the reference's
 * column_pivoted_qr (linalg.py:118-129), restated from dlaqp2 (first-max
 * pivot, norm downdating with the √ε recompute test).  Q and R follow from
 * pbq_householder_qr of the gathered columns (pbq_gather_columns).
 * M is not modified.  Limit: 8·m + 8·n bytes of shared memory per CTA
 * (PBQ_ERR_DIM beyond it). */
int pbq_cpqr_pivots(pbq_ctx* ctx, int64_t m, int64_t n, const double* M, int64_t ldm, int64_t* perm,
                    void* workspace, size_t workspace_bytes, void* stream);
int pbq_cpqr_workspace_bytes(pbq_ctx* ctx, int64_t m, int64_t n, size_t* bytes);

/* dst[:, i] = src[:, perm[i]] for row-major rows×cols matrices (V = V̄[:, perm],
 * algorithms.py:358). */
int pbq_gather_columns(pbq_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
                       const int64_t* perm, double* dst, int64_t ldd, void* stream);

/* Singular value decomposition of a small dense matrix (the
 * k×k core `svd_full`, linalg.py:131-139 / LAPACK dgesdd, of r_svd,
 * algorithms.py:263-292, and the pseudoinverse of cor_utv, :295-303) by
 * one-sided Jacobi on the n rows (length L ≥ n) of the row-major X:
 *   G·X = diag(s)·Y  ⇒  X = Gᵀ·diag(s)·Y,
 * s (n doubles) sorted descending, Y (n×L, ldy; may be NULL) with orthonormal
 * rows (rows with s = 0 are completed to an orthonormal set), and — with
 * PBQ_JACOBI_ACCUMULATE in `flags` — G (n×n, ldg) orthogonal, its rows the
 * left singular vectors.  PBQ_JACOBI_PRECONDITION first reduces X to the
 * n×n R̃ of Xᵀ = Q_h·R, Rᵀ = W·R̃ (two pbq_householder_qr chains, as LAPACK
 * dgejsv) and runs Jacobi on R̃ (far fewer sweeps on graded inputs); Y and G
 * then need even leading dimensions and 16-byte alignment.  X is not
 * modified.  status (device, 2 ints): sweeps used, 1 if not converged within
 * 60 sweeps.  n ≤ 256 rows of ≤ 768 doubles (incl. the G row when
 * accumulating) run in one thread-block cluster with the vectors in
 * registers; larger problems keep the vectors in L2. */
#define PBQ_JACOBI_ACCUMULATE 1
#define PBQ_JACOBI_PRECONDITION 2
int pbq_jacobi_svd(pbq_ctx* ctx, int64_t n, int64_t L, const double* X, int64_t ldx, int32_t flags, double* s,
                   double* Y, int64_t ldy, double* G, int64_t ldg, int32_t* status, void* workspace,
                   size_t workspace_bytes, void* stream);
int pbq_jacobi_svd_workspace_bytes(pbq_ctx* ctx, int64_t n, int64_t L, int32_t flags, size_t* bytes);

/* Distributed Cholesky-QR2 of a row-sharded tall matrix (the
 * QR of A·P̄ across ranks, replacing the TSQR tree when the input is
 * well-conditioned).  A is this rank's m×n row block.  The three stages run
 * the guarded Cholesky-QR2 chain of pbq_householder_qr split at its two Gram
 * matrices; between the stages the CALLER allreduces (sum) the np×np
 * matrix G (np = *ldg) across ranks:
 *   stage 0: G ← AᵀA (this rank's rows)
 *   stage 1: [G summed] R₁ = chol(G) with the κ₁ ≤ 1e6 guard; Q₁ = A·R₁⁻¹;
 *            G ← Q₁ᵀQ₁ (this rank's rows)
 *   stage 2: [G summed] R = R₂·R₁ (diag ≥ 0, rank flag as orth); A ← Q₁·R₂⁻¹
 *   stage 3 (instead of 1 and 2, basis-only as pbq_orth_basis): [G summed]
 *            R₁ = chol(G) with the guard; A ← A·R₁⁻¹ = Q·R₂ — one Gram exchange
 *            for an orth whose result is multiplied by A and orthonormalised again
 * Every rank factors the same G, so R is bitwise identical on all ranks.
 * *fallback (device int32) is set when the guard fails: A is then left
 * untouched and the caller runs its TSQR instead.  The workspace must
 * persist across the three calls. */
int pbq_cholqr2_dist(pbq_ctx* ctx, int32_t stage, int64_t m, int64_t n, double* A, int64_t lda, double* R,
                     int64_t ldr, int32_t* rank_flag, double* G, int32_t* fallback, void* workspace,
                     size_t workspace_bytes, void* stream);
int pbq_cholqr2_dist_workspace_bytes(pbq_ctx* ctx, int64_t m, int64_t n, size_t* bytes, int64_t* ldg);

/* PbP-QLP's second stage (reference algorithms.py:256-257): from the d×d
 * upper-triangular R of qr(D), (W, R̃) = householder_qr(Rᵀ) with diag R̃ ≥ 0
 * and L = tril(R̃ᵀ).  W (d×d) and L (d×d, zeros above the diagonal) are
 * row-major outputs; R is not modified.  Transpose, the pbq_householder_qr
 * chain on the d×d matrix, transpose, in one call.  No rank test (the
 * reference does not warn here). */
int pbq_second_stage(pbq_ctx* ctx, int64_t d, const double* R, int64_t ldr, double* W, int64_t ldw, double* L,
                     int64_t ldl, void* workspace, size_t workspace_bytes, void* stream);
int pbq_second_stage_workspace_bytes(pbq_ctx* ctx, int64_t d, size_t* bytes);

/* Fused AᵀX exchange over NVLink peer memory (the allreduce of
 * the row-sharded partials C_g = A_gᵀ·X_g, algorithms.py:182-184 across
 * ranks).  Rows of the n2×N result are split into world slices of S rows
 * (S a multiple of 128); rank r owns slice r.  Buffers come from symmetric
 * (peer-mapped) memory; the pointer arguments named *_ptrs are DEVICE arrays
 * of world peer pointers, indexed by rank.
 *   pbq_gemm_tn_scatter: the DMMA GEMM whose epilogue stores each finished
 *     128-row tile into the owner's landing buffer, slot `rank` (landing is
 *     world·S×ldl doubles per rank), then adds 1 to the owner's tile counter
 *     (system-scope release).  Needs the TMA GEMM.
 *   pbq_xchg_reduce: rank r waits until its tile counter reaches `target`,
 *     sums its slice's world slots in slot order and stores the result into
 *     rows [r·S, r·S+S) ∩ [0, n2) of every rank's C (ld ldc), then adds
 *     PBQ_XCHG_CTAS (64) to every rank's done counter.
 *   pbq_xchg_wait: waits until this rank's done counter reaches `target`.
 * Counters are never reset: per call the tile counter of rank r grows by
 * pbq_xchg_expected_tiles(...) and the done counter by 64·world, so call k
 * (1-based) passes target = k·(that growth).  A rank's counter block is three
 * consecutive uint32 [tile count, done count, status]; a wait that has not
 * completed after 20 s (pbq_set_p2p_timeout_ms) sets status bit 0 and
 * returns instead of hanging. */
#define PBQ_XCHG_CTAS 64
int pbq_gemm_tn_scatter(pbq_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* const* land_ptrs, uint32_t* const* cnt_ptrs, int32_t rank, int32_t world,
                        int64_t S, int64_t ldl, int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                        void* stream);
int pbq_xchg_reduce(pbq_ctx* ctx, int32_t rank, int32_t world, int64_t n2, int64_t N, int64_t S, const double* land,
                    int64_t ldl, double* const* c_ptrs, int64_t ldc, const uint32_t* cnt, uint32_t target,
                    uint32_t* const* done_ptrs, void* stream);
int pbq_xchg_wait(pbq_ctx* ctx, const uint32_t* done, uint32_t target, void* stream);
int pbq_xchg_expected_tiles(int64_t n2, int64_t N, int64_t S, int32_t rank, int32_t world, uint32_t* tiles);
/* Spin limit (milliseconds, default 20000) of every peer-memory wait
 * launched later on this context (the exchange's init self-check uses 2000). */
int pbq_set_p2p_timeout_ms(pbq_ctx* ctx, int64_t ms);

/* Small collectives on symmetric memory (the d×d Gram allreduces of the
 * distributed Cholesky-QR2 and the all-gather of orth(C)'s row slices):
 *   pbq_p2p_push: copies src (n doubles) to dst_ptrs[p] + rank·slot on every
 *     rank p, then adds PBQ_XCHG_CTAS to every rank's counter cnt_ptrs[p];
 *   pbq_p2p_sum:  waits until *cnt ≥ target, then out = Σ_g slots[g·slot + i]
 *     in slot order (allreduce = push into the peers' slot arrays + sum);
 *   pbq_p2p_wait: waits until *cnt ≥ target (all-gather = push with slot =
 *     the slice length into the peers' result buffers + wait).
 * Waits give up after 20 s and set *status bit 0 instead of hanging. */
int pbq_p2p_push(pbq_ctx* ctx, const double* src, int64_t n, double* const* dst_ptrs, int64_t slot, int32_t rank,
                 int32_t world, uint32_t* const* cnt_ptrs, void* stream);
int pbq_p2p_sum(pbq_ctx* ctx, const double* slots, int64_t slot, int32_t world, int64_t n, double* out,
                const uint32_t* cnt, uint32_t target, uint32_t* status, void* stream);
int pbq_p2p_wait(pbq_ctx* ctx, const uint32_t* cnt, uint32_t target, uint32_t* status, void* stream);

/* Small helpers used by the host driver.
 * dst[i][j] = src[j][i]            (n×n), or with lower=1 the lower triangle
 * of srcᵀ and zeros above (L = tril(R̃ᵀ), algorithms.py:257). */
int pbq_transpose(pbq_ctx* ctx, int64_t n, const double* src, int64_t lds, double* dst,
                  int64_t ldd, int32_t lower, void* stream);

/* Per-kernel-class timing of everything this context enqueues between
 * begin and end: CUDA events recorded on the launch stream around each kernel.
 * end() synchronises on the recorded events and returns the summed
 * milliseconds and launch counts for 4 classes: 0 GEMM, 1 QR, 2 sketch,
 * 3 other (transposes, flag merges).  Used by bench.py for the roofline of
 * the dominant kernel, measured inside the timed region. */
int pbq_profile_begin(pbq_ctx* ctx, int32_t capacity);
int pbq_profile_end(pbq_ctx* ctx, double* ms_by_class, int32_t* launches_by_class);

/* Profiling hooks (device pointers, NULL to disable): number of QR panels
 * that took the column-by-column fallback, CTA-0 nanoseconds per QR phase
 * (16 slots, see qr_f64.cuh), and per-CTA nanoseconds spent spinning in the
 * QR kernel's grid barriers (one slot per CTA, ≥ SM count). */
int pbq_debug_qr_hooks(pbq_ctx* ctx, int32_t* fallbacks, uint64_t* phase_ns, uint64_t* bar_wait_ns);

/* QR method for every later call on this context: 0 auto (Cholesky-QR2 with
 * on-device Householder fallback, the default), 1 Householder only, 2 auto
 * but with the blocked Cholesky (not the near-identity series) in the second
 * pass (a test hook for that safety path). */
#define PBQ_QR_AUTO 0
#define PBQ_QR_HOUSEHOLDER 1
#define PBQ_QR_CHOLQR_NOSERIES 2
#define PBQ_QR_CHOLQR_CHAIN 3 /* the multi-launch chain even where the single-launch kernel applies */
int pbq_set_qr_method(pbq_ctx* ctx, int32_t method);

/* Debug counters (device int[4], NULL to disable): QR calls completed by
 * Cholesky-QR, calls handed to the Householder fallback, completed calls
 * whose last pass used the near-identity series, and calls completed by the
 * shifted Cholesky-QR3 route (n ≥ 384 after a failed first pass). */
int pbq_debug_cholqr_stats(pbq_ctx* ctx, int32_t* stats);

#ifdef __cplusplus
}
#endif
#endif /* PBQ_H_ */
