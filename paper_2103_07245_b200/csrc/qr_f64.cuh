// Unpivoted Householder QR of a tall m×n FP64 matrix (m ≥ n), LAPACK
// dgeqrf + dorgqr semantics followed by the reference's sign fix
// (`householder_qr`, /root/reference/pkg/src/pbpqlp/linalg.py:106-115, and
// `_fix_signs`, linalg.py:96-103): on return A holds the thin Q (m×n), R holds
// the n×n upper-triangular factor with diag(R) ≥ 0 (sign 0 → +1), exact zeros
// below the diagonal, and `rank_flag` reports the `orth` rank test
// (linalg.py:142-165): 1 if some |R_ii| < 1e-14·|R_00|, 2 if R_00 == 0.
//
// Algorithm: blocked Householder QR in compact-WY form with
// 32-column panels.  One persistent CTA per SM (cooperative launch); CTA c
// owns a contiguous block of rows for the whole call; its rows of the current
// panel live in shared memory (in chunks when they do not fit).
//
// A full 32-column panel is factored by the fast path:
//   Cholesky-QR2 — two Gram reductions (four grid barriers per panel instead
//   of one per column) — followed by Householder reconstruction (Ballard,
//   Demmel, Grigori, Jacquelin, Knight, Nguyen, "Reconstructing Householder
//   vectors from tall-skinny QR", JPDC 2015): with Q₁ the panel's pivot block
//   and S = −sign(diag Q₁), an unpivoted LU I − Q₁S = V₁U gives the unit-lower
//   V₁; V₂ = −Q₂SU⁻¹, T = U·V₁⁻ᵀ, and the panel's R block is S·R.
// The 32×32 algebra is done redundantly by every CTA: two sequential
// eliminations (Cholesky, LU) and otherwise log-depth triangular inverses and
// small matrix products, so the per-row work becomes 32×32 matrix products.
// A panel takes the fallback — column-by-column Householder (dlarfg
// convention, one grid reduction per column) — when it is the last, partial
// panel or when diag(R₁) shows it is numerically rank deficient / its
// min/max diagonal ratio is below 0.1 (QR_FAST_DIAG_RATIO); every CTA takes the same decision from the same
// reduced Gram matrix.  The trailing update A2 ← (I − V Tᵀ Vᵀ) A2 and the
// backward Q formation Q ← (I − V T Vᵀ) Q are GEMM-shaped: per-CTA partials
// of VᵀX, a fixed-order slice reduction, then a row-local update.  All
// cross-CTA sums run in a fixed order: results are bitwise reproducible.
#pragma once
#include "common.cuh"

namespace pbq {

constexpr int QR_THREADS = 512;
constexpr int QR_TPR = QR_THREADS / 32;  // threads per row of a 32×32 tile
constexpr int QR_EPT = 32 / QR_TPR;      // entries per thread of a 32×32 tile
constexpr int QR_RG = QR_THREADS / 64;   // row groups of the Gram accumulation
constexpr int QR_IPT = 32 / (QR_THREADS / 32);  // W-partial i-rows per thread (32 columns per warp)
constexpr int QR_NB = 32;                 // panel width
// Row strides ≡ 4 (mod 16) doubles: DMMA fragment loads of either
// orientation (rows g / columns t of an 8×4 fragment) hit 16 distinct bank
// pairs per half-warp.
constexpr int QR_SLD = QR_NB + 4;         // leading dimension of 32×32 smem matrices
constexpr int QR_PLD = QR_NB + 4;         // leading dimension of the panel rows
constexpr int QR_CW = 128;                // trailing columns per staged tile
constexpr int QR_XLD = QR_CW + 4;         // leading dimension of staged tiles
constexpr int QR_TILE_DOUBLES = QR_NB * QR_XLD;  // one staged tile (32 rows × 128 columns)
constexpr double QR_RANK_RTOL = 1e-14;    // RANK_DEFICIENCY_RTOL, linalg.py:48
// min/max diag(R₁) a panel needs for the fast path.  The reconstructed
// reflectors lose orthogonality roughly with that ratio's inverse
// (tools/_hh_orth_probe.py, 129×129 at κ = 1e13: |QᵀQ − I| 3.3e-9 at 1e-4,
// 1.8e-12 at 1e-3, 1.1e-15 at 1e-1 — LAPACK's level); well-conditioned
// panels (random ones sit near 0.5) keep the fast path.
constexpr double QR_FAST_DIAG_RATIO = 1e-1;
// ... and at least this many rows below its top: a short panel's Q₁ is most
// of its Q, and the reconstruction lost orthogonality there too (129×129 with
// a clustered spectrum: 4.3e-13 with all diag ratios ≥ 0.1,
// tests/test_gpu_fuzz_qr.py); the last panels of square-ish inputs are cheap
// by the column-by-column path anyway.
constexpr long QR_FAST_MIN_ROWS = 4 * 32;
constexpr int QR_NSMALL = 12;             // 32×32 scratch matrices in shared memory

struct QrArgs {
  long m, n;
  double* A;
  long lda;
  double* R;  // n×n, may be null
  long ldr;
  int want_q;
  long rows_per_cta;
  int rch;         // rows per shared-memory chunk (≥ rows_per_cta when resident)
  double* part;    // 2 × G × 32   (fallback column partials)
  double* pivrow;  // 2 × 32
  double* pivbuf;  // 32 × 32      (original pivot rows of the panel)
  double* gfin;    // 32 × 32      (reduced Gram matrix)
  double* wpart;   // G × 32 × ldw (Gram / W partials), ldw = max(n, 32)
  double* ybuf;    // 32 × qr_ldy(n)
  double* tall;    // ceil(n/32) × 32 × 32
  unsigned int* counter;
  int* rank_flag;  // may be null
  int* fallbacks;  // may be null: number of panels that took the fallback
  int* error;      // unused (kept for the launch layout); every panel shape is supported
  unsigned long long* phase_ns;  // may be null: CTA-0 time per phase (profiling)
  unsigned long long* bar_wait_ns;  // may be null: per-CTA grid-barrier spin time (profiling)
  const int* run_if;  // may be null; else the kernel runs only when *run_if != 0 (Cholesky-QR fallback)
  int slow_panels;    // 1: every panel by the column-by-column path (A/B)
  double fast_ratio;  // min/max diag(R₁) a panel needs for the fast path
};

__device__ __forceinline__ unsigned long long qr_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// accumulate elapsed time since the previous mark into slot `ph` (CTA 0, thread 0)
#define QR_PHASE(ph)                                          \
  do {                                                       \
    if (p.phase_ns && blockIdx.x == gridDim.x / 2 && threadIdx.x == 0) { \
      const unsigned long long now_ = qr_now();              \
      p.phase_ns[ph] += now_ - t_phase;                      \
      t_phase = now_;                                        \
    }                                                        \
  } while (0)

// row stride of ybuf: even so that 16-byte cp.async sources stay aligned
__host__ __device__ constexpr long qr_ldy(long n) { return (n + 1) & ~1L; }
__host__ __device__ constexpr long qr_ldw(long n) { return n > QR_NB ? n : QR_NB; }
__host__ __device__ constexpr size_t qr_pad4(size_t x) { return (x + 3) & ~size_t(3); }

__device__ __forceinline__ double qr_sign(double beta) { return beta < 0.0 ? -1.0 : 1.0; }

struct QrSmem {
  double* Ps;     // rch × 33: the CTA's rows of the panel (one chunk)
  double* mat;    // QR_NSMALL × 32 × 33 scratch matrices
  double* beta;   // n   (signed diag of R)
  double* small;  // QR_THREADS reduction + 8 × 32 vectors
  double* stage;  // 2 × 4096 (double-buffered tiles)
  double* wsl;    // 32 × ⌈n/G⌉
  __device__ double* M(int k) const { return mat + k * qr_pad4(QR_NB * QR_SLD); }
};

__host__ __device__ inline size_t qr_smem_doubles(long rch, long n, int grid) {
  return qr_pad4(size_t(rch) * QR_PLD) + QR_NSMALL * qr_pad4(size_t(QR_NB) * QR_SLD) + qr_pad4(n) + QR_THREADS +
         8 * 32 + 2 * QR_TILE_DOUBLES + qr_pad4(size_t(QR_NB) * ceil_div(n, grid)) + 8;
}

// --------------------------------------------------------------------------
// Deterministic parallel reduction over the G CTA partials.  Entry e's partial
// from CTA q lives at addr(e) + q·stride.  `tpe` threads share an entry; each
// loads its partials q ≡ g (mod tpe) in independent batches and adds them in
// increasing q, then the tpe sub-sums are added in increasing g.  The order is
// a function of (E, G) only, so results are bitwise reproducible.
template <class Addr, class Sink>
__device__ __forceinline__ void qr_reduce_entries(int E, int G, size_t stride, Addr addr, Sink sink, double* red) {
  const int tid = threadIdx.x;
  for (int e0 = 0; e0 < E; e0 += QR_THREADS) {
    const int ecount = min(E - e0, QR_THREADS);
    int tpe = 1;
    while (tpe * 2 * ecount <= QR_THREADS && tpe * 2 <= G) tpe *= 2;
    const int el = tid / tpe, g = tid % tpe;
    double acc = 0.0;
    if (el < ecount) {
      const double* src = addr(e0 + el);
      int q = g;
      for (; q + 7 * tpe < G; q += 8 * tpe) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + size_t(q + u * tpe) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      for (; q < G; q += tpe) acc += __ldcg(src + size_t(q) * stride);
    }
    red[tid] = acc;
    __syncthreads();
    if (tid < ecount) {
      double sum = 0.0;
      for (int j = 0; j < tpe; ++j) sum += red[tid * tpe + j];
      sink(e0 + tid, sum);
    }
    __syncthreads();
  }
}

// ============================ 32×32 small algebra ============================
// All routines run on the whole CTA; thread t owns row t/8, columns
// 4·(t%8)..+3 of the 32×32 result.  Matrices live in shared memory, ld 33.

// C = op(A)·op(B) (opX = transpose when TX); C must not alias A or B.  One
// 8×8 DMMA tile per warp (16 warps = 4×4 tiles), 8 k-steps; the ld-36 layout
// keeps both fragment orientations conflict-free.
template <bool TA, bool TB>
__device__ __forceinline__ void sm_mm(double* C, const double* A, const double* B) {
  static_assert(QR_THREADS == 512, "one 8x8 tile per warp");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mi = (warp >> 2) * 8, ni = (warp & 3) * 8;
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < QR_NB; k0 += 4) {
    const double a = TA ? A[(k0 + t) * QR_SLD + mi + g] : A[(mi + g) * QR_SLD + k0 + t];
    const double b = TB ? B[(ni + g) * QR_SLD + k0 + t] : B[(k0 + t) * QR_SLD + ni + g];
    dmma884(c0, c1, a, b);
  }
  C[(mi + g) * QR_SLD + ni + 2 * t] = c0;
  C[(mi + g) * QR_SLD + ni + 2 * t + 1] = c1;
  __syncthreads();
}

// X = inv(op(U)) for upper-triangular op(U) (op = transpose when TRANS, i.e.
// the stored input is lower triangular); UNIT assumes a unit diagonal.
// Log-depth recursive doubling: [[A, B], [0, C]]⁻¹ = [[A⁻¹, −A⁻¹·B·C⁻¹],
// [0, C⁻¹]] for block sizes 1, 2, 4, 8, 16.  Z is 32×32 scratch.
template <bool TRANS, bool UNIT>
__device__ __forceinline__ void sm_tri_inv_upper(double* X, const double* U, double* Z) {
  const int tid = threadIdx.x;
  const int i = tid / QR_TPR, c0 = (tid % QR_TPR) * QR_EPT;
  auto u_at = [&](int r, int c) { return TRANS ? U[c * QR_SLD + r] : U[r * QR_SLD + c]; };
#pragma unroll
  for (int v = 0; v < QR_EPT; ++v) {
    const int c = c0 + v;
    X[i * QR_SLD + c] = (i == c) ? (UNIT ? 1.0 : fast_rcp(u_at(i, i))) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int lv = 0; lv < 5; ++lv) {
    const int b = 1 << lv;  // merge pairs of b×b blocks into 2b×2b
    // Z = B·C⁻¹ for every pair, entries (r, c) ∈ [0,b)²; 16b ≤ 256 entries
    if (tid < 16 * b) {
      const int pair = tid / (b * b), rr = (tid / b) % b, cc = tid % b;
      const int a0 = pair * 2 * b, k0 = a0 + b;
      double acc = 0.0;
      for (int q = 0; q <= cc; ++q) acc = fma(u_at(a0 + rr, k0 + q), X[(k0 + q) * QR_SLD + k0 + cc], acc);
      Z[(a0 + rr) * QR_SLD + k0 + cc] = acc;
    }
    __syncthreads();
    // X[A, C] = −A⁻¹·Z
    if (tid < 16 * b) {
      const int pair = tid / (b * b), rr = (tid / b) % b, cc = tid % b;
      const int a0 = pair * 2 * b, k0 = a0 + b;
      double acc = 0.0;
      for (int q = rr; q < b; ++q) acc = fma(X[(a0 + rr) * QR_SLD + a0 + q], Z[(a0 + q) * QR_SLD + k0 + cc], acc);
      X[(a0 + rr) * QR_SLD + k0 + cc] = -acc;
    }
    __syncthreads();
  }
}

// Sequential elimination shared by the Cholesky and the LU: step j publishes
// the final pivot row j and 1/pivot through shared memory (one barrier and
// one dependent reciprocal per step); every thread below the pivot updates its
// 4 entries.  SYM = Cholesky (Schur complement of a symmetric matrix,
// multipliers from the pivot row), else LU (multipliers from the own row,
// stored in place of the eliminated entry).
template <bool SYM>
__device__ __forceinline__ void sm_eliminate(double (&v)[QR_EPT], double* row_sm /*64*/, double* inv_sm /*2*/) {
  const int tid = threadIdx.x;
  const int i = tid / QR_TPR, c0 = (tid % QR_TPR) * QR_EPT;
#pragma unroll 1
  for (int j = 0; j < QR_NB; ++j) {
    const int b = j & 1;
    if (i == j) {
#pragma unroll
      for (int u = 0; u < QR_EPT; ++u) row_sm[b * 32 + c0 + u] = v[u];
      const int jj = j - c0;
      if (jj >= 0 && jj < QR_EPT) {
        double pv = v[0];
#pragma unroll
        for (int u = 1; u < QR_EPT; ++u)
          if (jj == u) pv = v[u];
        inv_sm[b] = fast_rcp(pv);
      }
    }
    double own = 0.0;
    if (!SYM) {  // entry (i, j), held by lane (row base + j/EPT) of this warp
      double cand = v[0];
#pragma unroll
      for (int u = 1; u < QR_EPT; ++u)
        if ((j % QR_EPT) == u) cand = v[u];
      own = __shfl_sync(0xffffffffu, cand, ((tid & ~(QR_TPR - 1)) | (j / QR_EPT)) & 31);
    }
    __syncthreads();
    if (i > j) {
      const double f = (SYM ? row_sm[b * 32 + i] : own) * inv_sm[b];
#pragma unroll
      for (int u = 0; u < QR_EPT; ++u) {
        const int l = c0 + u;
        if (l > j) v[u] = fma(-f, row_sm[b * 32 + l], v[u]);
        if (!SYM && l == j) v[u] = f;
      }
    }
  }
}

// Upper Cholesky of the symmetric 32×32 matrix G (in place; upper triangle
// receives R with RᵀR = G, lower triangle zeroed).  Returns min/max of
// diag(R), or -1 if a pivot was not positive.
__device__ double sm_chol(double* G, double* vec /*≥ 96*/) {
  __shared__ double s_ratio;
  const int tid = threadIdx.x;
  const int i = tid / QR_TPR, c0 = (tid % QR_TPR) * QR_EPT;
  double v[QR_EPT];
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u) v[u] = G[i * QR_SLD + c0 + u];
  __syncthreads();
  sm_eliminate<true>(v, vec, vec + 64);
  __syncthreads();
  // pivots → diag(R); row i of R = (row i of the Schur complement)/R_ii
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u)
    if (c0 + u == i) vec[i] = v[u];
  __syncthreads();
  if (tid < 32) {
    const double d = vec[tid];
    const bool ok = __all_sync(0xffffffffu, d > 0.0);
    const double r = sqrt(fmax(d, 0.0));
    double mn = r, mx = r;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (tid == 0) s_ratio = ok ? mn / mx : -1.0;
  }
  const double rd = sqrt(vec[i]), inv = fast_rcp(rd);
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u) {
    const int l = c0 + u;
    G[i * QR_SLD + l] = (l > i) ? v[u] * inv : ((l == i) ? rd : 0.0);
  }
  __syncthreads();
  return s_ratio;
}

// Unpivoted LU of the 32×32 matrix M in place: strict lower = unit-lower
// factor, upper = U.
__device__ void sm_lu(double* M, double* vec) {
  const int i = threadIdx.x / QR_TPR, c0 = (threadIdx.x % QR_TPR) * QR_EPT;
  double v[QR_EPT];
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u) v[u] = M[i * QR_SLD + c0 + u];
  __syncthreads();
  sm_eliminate<false>(v, vec, vec + 64);
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u) M[i * QR_SLD + c0 + u] = v[u];
  __syncthreads();
}

// Cholesky factor of a near-identity Gram matrix G = I + E (‖E‖ tiny) by the
// quadratically convergent series R = I + X, X ← split(E − XᵀX),
// split(M) = triu(M, 1) + diag(M)/2 — no sequential pivots.  The second
// Cholesky-QR pass has G = I + O(u·κ²).  R (upper, zeros below) goes to Rout;
// returns max|E|.
__device__ double sm_chol_near_identity(double* Rout, const double* G, double* X) {
  __shared__ unsigned long long s_emax;
  const int tid = threadIdx.x;
  const int i = tid / QR_TPR, c0 = (tid % QR_TPR) * QR_EPT;
  double e[QR_EPT];
  double emax = 0.0;
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u) {
    e[u] = G[i * QR_SLD + c0 + u] - ((i == c0 + u) ? 1.0 : 0.0);
    emax = fmax(emax, fabs(e[u]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  if (tid == 0) s_emax = 0ull;
  __syncthreads();
  if ((tid & 31) == 0) atomicMax(&s_emax, (unsigned long long)__double_as_longlong(emax));
  auto split = [&](int l, double x) { return (l > i) ? x : ((l == i) ? 0.5 * x : 0.0); };
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u) X[i * QR_SLD + c0 + u] = split(c0 + u, e[u]);
  __syncthreads();
#pragma unroll 1
  for (int it = 0; it < 3; ++it) {
    double nx[QR_EPT];
#pragma unroll
    for (int u = 0; u < QR_EPT; ++u) nx[u] = e[u];
#pragma unroll
    for (int q = 0; q < QR_NB; ++q) {
      const double xqi = (q <= i) ? X[q * QR_SLD + i] : 0.0;
#pragma unroll
      for (int u = 0; u < QR_EPT; ++u) nx[u] = fma(-xqi, X[q * QR_SLD + c0 + u], nx[u]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < QR_EPT; ++u) X[i * QR_SLD + c0 + u] = split(c0 + u, nx[u]);
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < QR_EPT; ++u) {
    const int l = c0 + u;
    Rout[i * QR_SLD + l] = (l >= i) ? X[i * QR_SLD + l] + ((l == i) ? 1.0 : 0.0) : 0.0;
  }
  __syncthreads();
  return __longlong_as_double((long long)*(volatile unsigned long long*)&s_emax);
}

// ======================= row-chunk helpers (panel rows) ======================
// The CTA's active rows [ra, r1) are processed in chunks of p.rch rows held in
// s.Ps (resident when one chunk covers all rows).

// Ps[rr][c] = A[cs + rr][col0 + c] for c < 32 and chunk rows [cs, ce).
__device__ __forceinline__ void qr_load_chunk(const QrArgs& p, const QrSmem& s, long cs, long ce, long col0) {
  const int rows = int(ce - cs);
  for (int e = threadIdx.x; e < rows * 16; e += QR_THREADS) {
    const int rr = e >> 4, cc = (e & 15) << 1;
    const double2 v = *reinterpret_cast<const double2*>(p.A + (cs + rr) * p.lda + col0 + cc);
    s.Ps[rr * QR_PLD + cc] = v.x;
    s.Ps[rr * QR_PLD + cc + 1] = v.y;
  }
}
__device__ __forceinline__ void qr_store_chunk(const QrArgs& p, const QrSmem& s, long cs, long ce, long col0) {
  const int rows = int(ce - cs);
  for (int e = threadIdx.x; e < rows * 16; e += QR_THREADS) {
    const int rr = e >> 4, cc = (e & 15) << 1;
    *reinterpret_cast<double2*>(p.A + (cs + rr) * p.lda + col0 + cc) =
        make_double2(s.Ps[rr * QR_PLD + cc], s.Ps[rr * QR_PLD + cc + 1]);
  }
}
// V form of the factored panel k (stored in A: R on/above the diagonal of the
// pivot rows, V below): unit diagonal, zeros above and beyond column jb.
__device__ __forceinline__ void qr_load_chunk_vform(const QrArgs& p, const QrSmem& s, long cs, long ce, long k,
                                                    int jb) {
  const int rows = int(ce - cs);
  for (int e = threadIdx.x; e < rows * 32; e += QR_THREADS) {
    const int rr = e >> 5, c = e & 31;
    const long r = cs + rr;
    double v;
    if (c >= jb || r < k + c) v = 0.0;
    else if (r == k + c) v = 1.0;
    else v = p.A[r * p.lda + k + c];
    s.Ps[rr * QR_PLD + c] = v;
  }
}

// Gram partial PᵀP (32×32) over chunk rows on the FP64 tensor pipe: warp w
// owns the 8×8 tile (w/4, w%4) and accumulates it over all rows (k = rows).
__device__ __forceinline__ void qr_gram_mma(const QrSmem& s, int rows, double (&acc)[2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mi = (warp >> 2) * 8, ni = (warp & 3) * 8;
  for (int k0 = 0; k0 < rows; k0 += 4) {
    const int r = k0 + t;
    const double a = (r < rows) ? s.Ps[r * QR_PLD + mi + g] : 0.0;
    const double b = (r < rows) ? s.Ps[r * QR_PLD + ni + g] : 0.0;
    dmma884(acc[0], acc[1], a, b);
  }
}
__device__ __forceinline__ void qr_gram_store(const double (&acc)[2], double* dst) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mi = (warp >> 2) * 8, ni = (warp & 3) * 8;
  __stcg(dst + (mi + g) * 32 + ni + 2 * t, acc[0]);
  __stcg(dst + (mi + g) * 32 + ni + 2 * t + 1, acc[1]);
}

// Slice reduction of the Gram partials (1024 entries) into p.gfin.
__device__ void qr_gram_reduce(const QrArgs& p, double* red) {
  const int G = gridDim.x;
  const int e0 = int(long(blockIdx.x) * 1024 / G), e1 = int(long(blockIdx.x + 1) * 1024 / G);
  const double* base = p.wpart;
  double* out = p.gfin;
  qr_reduce_entries(
      e1 - e0, G, size_t(QR_NB) * qr_ldw(p.n), [=](int e) { return base + e0 + e; },
      [=](int e, double v) { __stcg(out + e0 + e, v); }, red);
}

// out[r][c] = init(r, c) + sign·Σ_k Ps[r][k]·W[k][c] for the chunk rows
// r < rows and c < 32, on the FP64 tensor pipe.  Warp w owns rows
// b0 + 8w .. +8 of each 128-row block and all 32 columns (4 DMMA tiles); it
// reads only its own Ps rows, so writing back in place needs just a warp
// barrier.  Sink(rr, c, v0, v1) receives columns c, c+1 of row rr.
template <class Init, class Sink>
__device__ __forceinline__ void qr_rows_mma(const QrSmem& s, int rows, const double* W, double sign, Init init,
                                            Sink sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  for (int b0 = 0; b0 < rows; b0 += 8 * (QR_THREADS / 32)) {
    const int r = b0 + warp * 8 + g;  // this lane's output row
    if (b0 + warp * 8 >= rows) continue;
    double acc[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      acc[nt][0] = init(r, nt * 8 + 2 * t);
      acc[nt][1] = init(r, nt * 8 + 2 * t + 1);
    }
#pragma unroll
    for (int k0 = 0; k0 < QR_NB; k0 += 4) {
      const double a = (r < rows) ? sign * s.Ps[r * QR_PLD + k0 + t] : 0.0;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma884(acc[nt][0], acc[nt][1], a, W[(k0 + t) * QR_SLD + nt * 8 + g]);
    }
    __syncwarp();
    if (r < rows) {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) sink(r, nt * 8 + 2 * t, acc[nt][0], acc[nt][1]);
    }
  }
  __syncthreads();
}

// Chunk rows × W (32×32, smem) in place: Ps[rr][:] ← Ps[rr][:]·W.
__device__ __forceinline__ void qr_rows_times(const QrSmem& s, int rows, const double* W) {
  double* Ps = s.Ps;
  qr_rows_mma(
      s, rows, W, 1.0, [](int, int) { return 0.0; },
      [=](int r, int c, double v0, double v1) {
        Ps[r * QR_PLD + c] = v0;
        Ps[r * QR_PLD + c + 1] = v1;
      });
}

// ====================== trailing update (GEMM-shaped) =======================
// Accumulate this chunk's contribution to the W partial of columns
// [col0, col0+ntr):  W[i][c] += Σ_rr V[rr][i]·X[row][c] on the FP64 tensor
// pipe.  X tiles (32 rows × 128 columns) stream through a double-buffered
// cp.async ring; warp w owns i-tile w%4 and column tiles 4·(w/4)..+4 of each
// 128-column chunk.  The W partial lives in the CTA's wpart slot (first chunk
// writes, later chunks accumulate).
__device__ void qr_wpartial_chunk(const QrArgs& p, const QrSmem& s, long cs, long ce, long col0, long ntr,
                                  bool first) {
  constexpr int TR = QR_NB / 2;     // rows per staged tile
  constexpr int NST = 4;            // ring depth (same shared memory as 2 × 32 rows)
  constexpr int TD = TR * QR_XLD;   // doubles per tile
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mi = (warp & 3) * 8, nt0 = (warp >> 2) * 4;
  const long ldw = qr_ldw(p.n);
  double* wdst = p.wpart + size_t(blockIdx.x) * QR_NB * ldw;
  const int nrows = int(ce - cs);
  const int nrc = (nrows + TR - 1) / TR;
  for (long c0 = 0; c0 < ntr; c0 += QR_CW) {
    auto load = [&](int tt) {
      double* dst = s.stage + (tt % NST) * TD;
      const long rc = cs + long(tt) * TR;
      for (int e = tid; e < TR * QR_CW / 2; e += QR_THREADS) {
        const int rr = e / (QR_CW / 2), cc = (e % (QR_CW / 2)) * 2;
        const long c = c0 + cc;
        int bytes = 0;
        const double* src = p.A;
        if (rc + rr < ce && c < ntr) {
          bytes = int(lmin(2, ntr - c)) * 8;
          src = p.A + (rc + rr) * p.lda + col0 + c;
        }
        cp_async16(dst + rr * QR_XLD + cc, src, bytes);
      }
    };
    double acc[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
    for (int tt = 0; tt < NST - 1; ++tt) {
      if (tt < nrc) load(tt);
      cp_async_commit();
    }
    for (int tt = 0; tt < nrc; ++tt) {
      cp_async_wait<NST - 2>();
      __syncthreads();
      if (tt + NST - 1 < nrc) load(tt + NST - 1);
      cp_async_commit();
      const double* tile = s.stage + (tt % NST) * TD;
      const int rbase = tt * TR;
#pragma unroll
      for (int k0 = 0; k0 < TR; k0 += 4) {
        const int rr = rbase + k0 + t;
        const double a = (rr < nrows) ? s.Ps[rr * QR_PLD + mi + g] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          dmma884(acc[nt][0], acc[nt][1], a, tile[(k0 + t) * QR_XLD + (nt0 + nt) * 8 + g]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long c = c0 + (nt0 + nt) * 8 + 2 * t + e;
        if (c < ntr) {
          double* w = wdst + size_t(mi + g) * ldw + c;
          __stcg(w, first ? acc[nt][e] : acc[nt][e] + __ldcg(w));
        }
      }
  }
  __syncthreads();
}

// Fixed-order reduction of the W partials over CTAs for this CTA's column
// slice, then Y = op(T)·W for the slice (op = transpose when `trans_t`).
__device__ void qr_reduce_slice(const QrArgs& p, const QrSmem& s, const double* Ts, long ntr, bool trans_t) {
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  const long ldw = qr_ldw(p.n);
  const long cs = long(blockIdx.x) * ntr / G, ce = long(blockIdx.x + 1) * ntr / G;
  const int sw = int(ce - cs);
  if (sw <= 0) return;
  const double* base = p.wpart + cs;
  double* wsl = s.wsl;
  qr_reduce_entries(
      QR_NB * sw, G, size_t(QR_NB) * ldw, [=](int e) { return base + size_t(e / sw) * ldw + e % sw; },
      [=](int e, double v) { wsl[e] = v; }, s.small);
  for (int e = tid; e < QR_NB * sw; e += QR_THREADS) {
    const int i = e / sw, c = e % sw;
    double acc = 0.0;
    if (trans_t) {
      for (int l = 0; l <= i; ++l) acc = fma(Ts[l * QR_SLD + i], s.wsl[l * sw + c], acc);
    } else {
      for (int l = i; l < QR_NB; ++l) acc = fma(Ts[i * QR_SLD + l], s.wsl[l * sw + c], acc);
    }
    __stcg(p.ybuf + size_t(i) * qr_ldy(p.n) + cs + c, acc);
  }
}

// Row-local update of this chunk: X[row][c] -= Σ_i V[rr][i]·Y[i][c], on the
// FP64 tensor pipe.  Y (32 × 128 chunk) is staged in shared memory; warp w
// owns row tile w%4 and column tiles 4·(w/4)..+4 of each 32-row block; the
// accumulators start from X (read straight into fragment layout) and the A
// fragments carry −V.
__device__ void qr_update_chunk(const QrArgs& p, const QrSmem& s, long cs, long ce, long col0, long ntr) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mi = (warp & 3) * 8, nt0 = (warp >> 2) * 4;
  const int nrows = int(ce - cs);
  for (long c0 = 0; c0 < ntr; c0 += QR_CW) {
    __syncthreads();
    for (int e = tid; e < QR_NB * QR_CW / 2; e += QR_THREADS) {
      const int i = e / (QR_CW / 2), cc = (e % (QR_CW / 2)) * 2;
      const long c = c0 + cc;
      const int bytes = (c < ntr) ? int(lmin(2, ntr - c)) * 8 : 0;
      cp_async16(s.stage + i * QR_XLD + cc, bytes ? p.ybuf + size_t(i) * qr_ldy(p.n) + c : p.ybuf, bytes);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    auto load_x = [&](int rc, double (&x)[4][2]) {
      const int rr = rc + mi + g;
      const bool rok = rr < nrows;
      const double* xrow = p.A + (cs + rr) * p.lda + col0;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const long c = c0 + (nt0 + nt) * 8 + 2 * t;
        if (rok && c + 1 < ntr) {
          const double2 v = *reinterpret_cast<const double2*>(xrow + c);
          x[nt][0] = v.x;
          x[nt][1] = v.y;
        } else {
          x[nt][0] = (rok && c < ntr) ? xrow[c] : 0.0;
          x[nt][1] = 0.0;
        }
      }
    };
    double nxt[4][2];
    if (nrows > 0) load_x(0, nxt);
    for (int rc = 0; rc < nrows; rc += QR_NB) {
      const int rr = rc + mi + g;  // this lane's row (chunk-relative)
      const bool rok = rr < nrows;
      double* xrow = p.A + (cs + rr) * p.lda + col0;
      double acc[4][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        acc[nt][0] = nxt[nt][0];
        acc[nt][1] = nxt[nt][1];
      }
      if (rc + QR_NB < nrows) load_x(rc + QR_NB, nxt);  // prefetch the next row block
#pragma unroll
      for (int k0 = 0; k0 < QR_NB; k0 += 4) {
        const double a = rok ? -s.Ps[rr * QR_PLD + k0 + t] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          dmma884(acc[nt][0], acc[nt][1], a, s.stage[(k0 + t) * QR_XLD + (nt0 + nt) * 8 + g]);
      }
      if (rok) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const long c = c0 + (nt0 + nt) * 8 + 2 * t;
          if (c + 1 < ntr) *reinterpret_cast<double2*>(xrow + c) = make_double2(acc[nt][0], acc[nt][1]);
          else if (c < ntr) xrow[c] = acc[nt][0];
        }
      }
    }
  }
  __syncthreads();
}

// ============ fallback: column-by-column Householder (any jb ≤ 32) ==========
// Works on the CTA's active rows through `P` (row rr ↔ row ra + rr at
// P + rr·ldp, panel column c at offset c): the shared-memory chunk when the
// rows are resident, else A itself (global, L2-resident; only the panel's
// first jb columns of this CTA's rows are touched, and __syncthreads orders
// them within the CTA).  On return P holds the factored panel (R on/above
// the pivot diagonal, V below), Ts the T factor and s.beta the signed diagonal.
__device__ void qr_panel_householder(const QrArgs& p, const QrSmem& s, double* P, long ldp, double* Ts, long k,
                                     int jb, long ra, long r1, unsigned int& gen) {
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  double* red = s.small;                 // QR_THREADS
  double* svec = s.small + QR_THREADS;   // 32
  double* prow = svec + 32;       // 32
  double* wt = prow + 32;         // 32
  for (int e = tid; e < QR_NB * QR_SLD; e += QR_THREADS) Ts[e] = 0.0;
  __syncthreads();
  const int nrows = int(lmax(0L, r1 - ra));
  for (int jj = 0; jj < jb; ++jj) {
    const long piv = k + jj;
    const int buf = int(piv & 1);
    {
      const int c = tid & 31, grp = tid >> 5;
      double a0 = 0.0, a1 = 0.0;
      constexpr int NG = QR_THREADS / 32;
      if (c < jb) {
        int rr = int(lmax(0L, piv + 1 - ra)) + grp;
        for (; rr + NG < nrows; rr += 2 * NG) {
          const double* row0 = P + rr * ldp;
          const double* row1 = row0 + NG * ldp;
          a0 = fma(row0[jj], row0[c], a0);
          a1 = fma(row1[jj], row1[c], a1);
        }
        if (rr < nrows) {
          const double* row0 = P + rr * ldp;
          a0 = fma(row0[jj], row0[c], a0);
        }
      }
      red[grp * 32 + c] = a0 + a1;
    }
    __syncthreads();
    if (tid < jb) {
      double acc = 0.0;
#pragma unroll
      for (int g2 = 0; g2 < QR_THREADS / 32; ++g2) acc += red[g2 * 32 + tid];
      __stcg(p.part + (size_t(buf) * G + blockIdx.x) * 32 + tid, acc);
      if (piv >= ra && piv < r1) __stcg(p.pivrow + buf * 32 + tid, P[(piv - ra) * ldp + tid]);
    }
    grid_barrier(p.counter, gen, p.bar_wait_ns);
    {
      const double* base = p.part + size_t(buf) * G * 32;
      qr_reduce_entries(
          jb, G, 32, [=](int e) { return base + e; }, [=](int e, double v) { svec[e] = v; }, red);
    }
    if (tid < jb) prow[tid] = __ldcg(p.pivrow + buf * 32 + tid);
    __syncthreads();
    const double alpha = prow[jj], sigma = svec[jj];
    double beta, tau, scale;
    if (sigma == 0.0) {
      beta = alpha;
      tau = 0.0;
      scale = 0.0;
    } else {
      const double nrm = sqrt(fma(alpha, alpha, sigma));
      beta = signbit(alpha) ? nrm : -nrm;
      tau = (beta - alpha) * fast_rcp(beta);
      scale = fast_rcp(alpha - beta);
    }
    if (tid < jb) wt[tid] = (tid > jj) ? tau * fma(scale, svec[tid], prow[tid]) : 0.0;
    if (tid < jj) {
      double acc = 0.0;
      for (int l = tid; l < jj; ++l) acc = fma(Ts[tid * QR_SLD + l], fma(scale, svec[l], prow[l]), acc);
      Ts[tid * QR_SLD + jj] = -tau * acc;
    }
    if (tid == 0) {
      Ts[jj * QR_SLD + jj] = tau;
      s.beta[piv] = beta;
    }
    __syncthreads();
    const int rs = int(lmax(0L, piv - ra));
    const int ncol = jb - jj;
    for (int e = tid; e < (nrows - rs) * ncol; e += QR_THREADS) {
      const int rr = rs + e / ncol;
      const int c = jj + e % ncol;
      double* row = P + rr * ldp;
      if (ra + rr == piv) {
        row[c] = (c == jj) ? beta : row[c] - wt[c];
      } else if (c > jj) {
        row[c] = fma(-wt[c], scale * row[jj], row[c]);
      }
    }
    __syncthreads();
    for (int rr = int(lmax(0L, piv + 1 - ra)) + tid; rr < nrows; rr += QR_THREADS) P[rr * ldp + jj] *= scale;
    __syncthreads();
  }
}

// ================================ the kernel ================================
__global__ void __launch_bounds__(QR_THREADS, 1) qr_tall_kernel(QrArgs p) {
  pdl_trigger();  // a programmatically launched successor may start its prologue
  extern __shared__ __align__(16) double qsm[];
  if (p.run_if && __ldcg(p.run_if) == 0) return;  // uniform across the grid
  const long m = p.m, n = p.n;
  const int tid = threadIdx.x;
  const long r0 = long(blockIdx.x) * p.rows_per_cta;
  const long r1 = lmin(m, r0 + p.rows_per_cta);
  const long rch = p.rch;

  QrSmem s;
  {
    double* q = qsm;
    s.Ps = q; q += qr_pad4(size_t(rch) * QR_PLD);
    s.mat = q; q += QR_NSMALL * qr_pad4(size_t(QR_NB) * QR_SLD);
    s.beta = q; q += qr_pad4(n);
    s.small = q; q += QR_THREADS + 8 * 32;
    s.stage = q; q += 2 * QR_TILE_DOUBLES;
    s.wsl = q;
  }
  // named 32×32 scratch matrices
  double* R1 = s.M(0);    // Cholesky factor of pass 1
  double* R1i = s.M(1);   // R₁⁻¹
  double* R2 = s.M(2);    // Cholesky factor of pass 2
  double* R2i = s.M(3);   // R₂⁻¹
  double* Ts = s.M(4);    // T
  double* LU = s.M(5);    // LU(I − Q₁S), later V₁ for the Q formation
  double* Wm = s.M(6);    // per-row transform of the current pass
  double* Z = s.M(7);     // scratch
  double* Pp = s.M(8);    // pivot rows of the panel, later R_p
  double* Ui = s.M(9);    // U⁻¹
  double* Lt = s.M(10);   // V₁⁻ᵀ, later M1 = T·V₁ᵀ
  double* SR = s.M(11);   // S·R_p
  double* vec = s.small + QR_THREADS;         // 96: elimination rows (0..63) and pivots (64..65)
  double* svec = s.small + QR_THREADS + 128;  // 32: S signs
  unsigned int gen = 0;
  int nfallback = 0;
  unsigned long long t_phase = (p.phase_ns && blockIdx.x == gridDim.x / 2 && tid == 0) ? qr_now() : 0;
  const bool resident = p.rows_per_cta <= rch;  // same for every CTA (barrier counts must agree)

  // ===================== factorization (dgeqrf) =====================
  for (long k = 0, pidx = 0; k < n; k += QR_NB, ++pidx) {
    const int jb = int(lmin(QR_NB, n - k));
    const long ra = lmax(r0, k);  // first active owned row
    double* gdst = p.wpart + size_t(blockIdx.x) * QR_NB * qr_ldw(n);
    bool fast = false;
    if (jb == QR_NB && p.m - k >= QR_FAST_MIN_ROWS && !p.slow_panels) {
      // ---- pass 1: Gram partial (+ publish the pivot rows)
      double acc[2] = {0.0, 0.0};
      for (long cs = ra; cs < r1; cs += rch) {
        const long ce = lmin(r1, cs + rch);
        qr_load_chunk(p, s, cs, ce, k);
        __syncthreads();
        qr_gram_mma(s, int(ce - cs), acc);
        for (int e = tid; e < int(lmin(ce, k + QR_NB) - cs) * QR_NB; e += QR_THREADS) {
          const int rr = e >> 5, c = e & 31;
          __stcg(p.pivbuf + (cs + rr - k) * 32 + c, s.Ps[rr * QR_PLD + c]);
        }
        if (!resident) __syncthreads();
      }
      qr_gram_store(acc, gdst);
      grid_barrier(p.counter, gen, p.bar_wait_ns);
      QR_PHASE(0);
      qr_gram_reduce(p, s.small);
      grid_barrier(p.counter, gen, p.bar_wait_ns);
      for (int e = tid; e < 1024; e += QR_THREADS) {
        R1[(e >> 5) * QR_SLD + (e & 31)] = __ldcg(p.gfin + e);
        Pp[(e >> 5) * QR_SLD + (e & 31)] = __ldcg(p.pivbuf + e);
      }
      __syncthreads();
      const double ratio1 = sm_chol(R1, vec);
      fast = ratio1 > p.fast_ratio && !p.slow_panels;
      QR_PHASE(1);
      if (fast) {
        sm_tri_inv_upper<false, false>(R1i, R1, Z);
        // ---- pass 2: Q₁ = P·R₁⁻¹ (rows in place) + Gram of Q₁
        acc[0] = acc[1] = 0.0;
        for (long cs = ra; cs < r1; cs += rch) {
          const long ce = lmin(r1, cs + rch);
          if (!resident) {
            qr_load_chunk(p, s, cs, ce, k);
            __syncthreads();
          }
          qr_rows_times(s, int(ce - cs), R1i);
          qr_gram_mma(s, int(ce - cs), acc);
          if (!resident) {
            __syncthreads();
            qr_store_chunk(p, s, cs, ce, k);
            __syncthreads();
          }
        }
        qr_gram_store(acc, gdst);
        grid_barrier(p.counter, gen, p.bar_wait_ns);
        qr_gram_reduce(p, s.small);
        grid_barrier(p.counter, gen, p.bar_wait_ns);
        for (int e = tid; e < 1024; e += QR_THREADS) Z[(e >> 5) * QR_SLD + (e & 31)] = __ldcg(p.gfin + e);
        __syncthreads();
        QR_PHASE(2);
        // ---- R₂: series when Q₁ᵀQ₁ = I + E with tiny E, else pivots
        const double emax = sm_chol_near_identity(R2, Z, Wm);
        if (!(emax <= 1e-5)) {
          for (int e = tid; e < 1024; e += QR_THREADS) R2[(e >> 5) * QR_SLD + (e & 31)] = Z[(e >> 5) * QR_SLD + (e & 31)];
          __syncthreads();
          fast = sm_chol(R2, vec) > 0.5;
          if (!fast) {
            // not expected for diag ratio(R₁) > 1e-4: restore P = Q₁·R₁ and
            // take the fallback
            for (long cs = ra; cs < r1; cs += rch) {
              const long ce = lmin(r1, cs + rch);
              if (!resident) {
                qr_load_chunk(p, s, cs, ce, k);
                __syncthreads();
              }
              qr_rows_times(s, int(ce - cs), R1);
              if (!resident) qr_store_chunk(p, s, cs, ce, k);
              __syncthreads();
            }
          }
        }
        QR_PHASE(12);
      }
    }
    if (fast) {
      // ---- the 32×32 reconstruction algebra (redundant per CTA)
      sm_tri_inv_upper<false, false>(R2i, R2, Z);
      sm_mm<false, false>(Wm, R1i, R2i);   // R_p⁻¹ = R₁⁻¹R₂⁻¹
      sm_mm<false, false>(Z, Pp, Wm);      // Q₁ = P_piv·R_p⁻¹
      {
        const int i = tid / QR_TPR, c0 = (tid % QR_TPR) * QR_EPT;
        if (tid < 32) svec[tid] = (Z[tid * QR_SLD + tid] >= 0.0) ? -1.0 : 1.0;  // S = −sign(diag Q₁)
        __syncthreads();
#pragma unroll
        for (int u = 0; u < QR_EPT; ++u) {
          const int l = c0 + u;
          LU[i * QR_SLD + l] = ((i == l) ? 1.0 : 0.0) - Z[i * QR_SLD + l] * svec[l];
        }
        __syncthreads();
      }
      QR_PHASE(13);
      sm_mm<false, false>(Pp, R2, R1);     // R_p = R₂R₁ (pivot rows no longer needed)
      sm_lu(LU, vec);
      QR_PHASE(14);
      {
        const int i = tid / QR_TPR, c0 = (tid % QR_TPR) * QR_EPT;
#pragma unroll
        for (int u = 0; u < QR_EPT; ++u) {
          const int l = c0 + u;
          Z[i * QR_SLD + l] = (l >= i) ? LU[i * QR_SLD + l] : 0.0;            // U
          SR[i * QR_SLD + l] = (l >= i) ? svec[i] * Pp[i * QR_SLD + l] : 0.0;  // S·R_p
        }
        __syncthreads();
      }
      sm_tri_inv_upper<false, false>(Ui, Z, Wm);  // U⁻¹
      sm_tri_inv_upper<true, true>(Lt, LU, Wm);   // (V₁ᵀ)⁻¹ = V₁⁻ᵀ
      sm_mm<false, false>(Ts, Z, Lt);             // T = U·V₁⁻ᵀ
      {
        const int i = tid / QR_TPR, c0 = (tid % QR_TPR) * QR_EPT;
#pragma unroll
        for (int u = 0; u < QR_EPT; ++u) Z[i * QR_SLD + c0 + u] = -R2i[i * QR_SLD + c0 + u] * svec[c0 + u];
        __syncthreads();
      }
      sm_mm<false, false>(Wm, Z, Ui);             // W₃ = R₂⁻¹·(−S)·U⁻¹
      if (tid < 32) s.beta[k + tid] = SR[tid * QR_SLD + tid];
      QR_PHASE(15);
      // ---- pass 3: V rows = Q₁ rows · W₃ ; pivot rows get S·R_p / V₁
      for (long cs = ra; cs < r1; cs += rch) {
        const long ce = lmin(r1, cs + rch);
        if (!resident) {
          qr_load_chunk(p, s, cs, ce, k);
          __syncthreads();
        }
        qr_rows_times(s, int(ce - cs), Wm);
        for (int e = tid; e < int(ce - cs) * QR_NB; e += QR_THREADS) {
          const int rr = e >> 5, c = e & 31;
          const long r = cs + rr;
          double a = s.Ps[rr * QR_PLD + c];  // V row (non-pivot)
          if (r < k + QR_NB) {
            const int i = int(r - k);
            a = (c >= i) ? SR[i * QR_SLD + c] : LU[i * QR_SLD + c];
            s.Ps[rr * QR_PLD + c] = (c < i) ? LU[i * QR_SLD + c] : ((c == i) ? 1.0 : 0.0);
          }
          p.A[r * p.lda + k + c] = a;
        }
        __syncthreads();
      }
      QR_PHASE(4);
    } else {
      // ---- fallback: column-by-column Householder
      ++nfallback;
      if (!resident) {  // rows stay in A; the trailing update reloads the V form per chunk
        __syncthreads();
        qr_panel_householder(p, s, p.A + ra * p.lda + k, p.lda, Ts, k, jb, ra, r1, gen);
        __syncthreads();
        QR_PHASE(5);
      } else {
      for (int e = tid; e < int(lmax(0L, r1 - ra)) * QR_NB; e += QR_THREADS) {
        const int rr = e >> 5, c = e & 31;
        s.Ps[rr * QR_PLD + c] = (c < jb) ? p.A[(ra + rr) * p.lda + k + c] : 0.0;
      }
      __syncthreads();
      qr_panel_householder(p, s, s.Ps, QR_PLD, Ts, k, jb, ra, r1, gen);
      for (int e = tid; e < int(lmax(0L, r1 - ra)) * QR_NB; e += QR_THREADS) {
        const int rr = e >> 5, c = e & 31;
        const long r = ra + rr;
        double v = s.Ps[rr * QR_PLD + c];
        if (c < jb) p.A[r * p.lda + k + c] = v;
        if (c >= jb || r < k + c) v = 0.0;
        else if (r == k + c) v = 1.0;
        s.Ps[rr * QR_PLD + c] = v;  // V form for the trailing update
      }
      __syncthreads();
      QR_PHASE(5);
      }
    }
    if (blockIdx.x == 0)
      for (int e = tid; e < 1024; e += QR_THREADS) p.tall[pidx * 1024 + e] = Ts[(e >> 5) * QR_SLD + (e & 31)];

    const long ntr = n - k - jb;
    if (ntr > 0) {
      // W partial over all active rows (V chunk in Ps)
      bool first = true;
      for (long cs = ra; cs < r1; cs += rch) {
        const long ce = lmin(r1, cs + rch);
        if (!resident) {
          __syncthreads();
          qr_load_chunk_vform(p, s, cs, ce, k, jb);
          __syncthreads();
        }
        qr_wpartial_chunk(p, s, cs, ce, k + jb, ntr, first);
        first = false;
      }
      if (first) {  // no active rows: publish zeros
        double* wdst = p.wpart + size_t(blockIdx.x) * QR_NB * qr_ldw(n);
        for (long e = tid; e < QR_NB * ntr; e += QR_THREADS) __stcg(wdst + (e / ntr) * qr_ldw(n) + e % ntr, 0.0);
      }
      grid_barrier(p.counter, gen, p.bar_wait_ns);
      QR_PHASE(6);
      qr_reduce_slice(p, s, Ts, ntr, /*trans_t=*/true);
      grid_barrier(p.counter, gen, p.bar_wait_ns);
      QR_PHASE(7);
      for (long cs = ra; cs < r1; cs += rch) {
        const long ce = lmin(r1, cs + rch);
        if (!resident) {
          __syncthreads();
          qr_load_chunk_vform(p, s, cs, ce, k, jb);
          __syncthreads();
        }
        qr_update_chunk(p, s, cs, ce, k + jb, ntr);
      }
      QR_PHASE(8);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0 && p.fallbacks) *p.fallbacks = nfallback;

  // ===================== R extraction + rank test =====================
  if (blockIdx.x == 0 && tid == 0 && p.rank_flag) {
    const double d0 = fabs(s.beta[0]);
    int flag = 0;
    if (d0 > 0.0) {
      for (long i = 0; i < n; ++i)
        if (fabs(s.beta[i]) < QR_RANK_RTOL * d0) flag = 1;
    } else {
      flag = 2;
    }
    *p.rank_flag = flag;
  }
  const long rn = lmin(r1, n);  // owned rows that carry R
  if (p.R) {
    for (long e = tid; e < lmax(0L, rn - r0) * n; e += QR_THREADS) {
      const long i = r0 + e / n, j = e % n;
      p.R[i * p.ldr + j] = (j >= i) ? qr_sign(s.beta[i]) * p.A[i * p.lda + j] : 0.0;
    }
  }
  if (!p.want_q) return;
  __syncthreads();
  for (long e = tid; e < lmax(0L, rn - r0) * n; e += QR_THREADS) {
    const long i = r0 + e / n, j = e % n;
    if (j > i) p.A[i * p.lda + j] = 0.0;
  }
  // every CTA's factored panels (V₁ blocks, T factors) are published before
  // any CTA starts reading them
  grid_barrier(p.counter, gen, p.bar_wait_ns);
  QR_PHASE(9);

  // ===================== Q formation (dorgqr, backward) =====================
  const long npan = ceil_div(n, QR_NB);
  for (long pidx = npan - 1; pidx >= 0; --pidx) {
    const long k = pidx * QR_NB;
    const int jb = int(lmin(QR_NB, n - k));
    const long ra = lmax(r0, k);
    // V₁ (pivot block, needed by every CTA) and T
    for (int e = tid; e < 1024; e += QR_THREADS) {
      const int a = e >> 5, c = e & 31;
      double v = (a == c && a < jb) ? 1.0 : 0.0;
      if (a > c && a < jb) v = __ldcg(p.A + (k + a) * p.lda + k + c);
      LU[a * QR_SLD + c] = v;
      Ts[a * QR_SLD + c] = __ldcg(p.tall + pidx * 1024 + e);
    }
    __syncthreads();
    QR_PHASE(16);
    const long ntr = n - k - jb;
    if (ntr > 0) {
      bool first = true;
      for (long cs = ra; cs < r1; cs += rch) {
        const long ce = lmin(r1, cs + rch);
        __syncthreads();
        qr_load_chunk_vform(p, s, cs, ce, k, jb);
        __syncthreads();
        QR_PHASE(17);
        qr_wpartial_chunk(p, s, cs, ce, k + jb, ntr, first);
        first = false;
      }
      if (first) {
        double* wdst = p.wpart + size_t(blockIdx.x) * QR_NB * qr_ldw(n);
        for (long e = tid; e < QR_NB * ntr; e += QR_THREADS) __stcg(wdst + (e / ntr) * qr_ldw(n) + e % ntr, 0.0);
      }
      QR_PHASE(18);
      grid_barrier(p.counter, gen, p.bar_wait_ns);
      QR_PHASE(19);
      qr_reduce_slice(p, s, Ts, ntr, /*trans_t=*/false);
      QR_PHASE(20);
      grid_barrier(p.counter, gen, p.bar_wait_ns);
      QR_PHASE(10);
      for (long cs = ra; cs < r1; cs += rch) {
        const long ce = lmin(r1, cs + rch);
        if (!resident) {
          __syncthreads();
          qr_load_chunk_vform(p, s, cs, ce, k, jb);
          __syncthreads();
        }
        qr_update_chunk(p, s, cs, ce, k + jb, ntr);
      }
    } else {
      grid_barrier(p.counter, gen, p.bar_wait_ns);  // every CTA has read V₁ before it is overwritten
    }
    // M1 = T·V₁ᵀ; panel columns Q[r][k+c] = δ(r, k+c) − Σ_i V[r][i]·M1[i][c]
    sm_mm<false, true>(Lt, Ts, LU);
    for (long cs = ra; cs < r1; cs += rch) {
      const long ce = lmin(r1, cs + rch);
      if (!resident || ntr <= 0) {
        __syncthreads();
        qr_load_chunk_vform(p, s, cs, ce, k, jb);
        __syncthreads();
      }
      double* Acol = p.A + k;
      const long lda = p.lda;
      qr_rows_mma(
          s, int(ce - cs), Lt, -1.0, [=](int rr, int c) { return (cs + rr == k + c) ? 1.0 : 0.0; },
          [=](int rr, int c, double v0, double v1) {
            double* dst = Acol + (cs + rr) * lda + c;
            if (c < jb) dst[0] = v0;
            if (c + 1 < jb) dst[1] = v1;
          });
    }
    QR_PHASE(11);
  }
  // sign fix: Q[:, c] *= sign(R_cc)
  for (long e = tid; e < (r1 - r0) * n; e += QR_THREADS) {
    const long r = r0 + e / n, c = e % n;
    if (s.beta[c] < 0.0) p.A[r * p.lda + c] = -p.A[r * p.lda + c];
  }
}

}  // namespace pbq
