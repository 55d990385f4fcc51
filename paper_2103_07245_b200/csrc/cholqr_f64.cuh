// Whole-matrix Cholesky-QR2 with a Householder fallback — the fast path of
// `householder_qr` / `orth` (reference linalg.py:106-115, :142-165).
//
// For a full-column-rank m×n matrix A the thin QR with diag(R) > 0 is
// unique, so Q = A·R⁻¹ with RᵀR = AᵀA is the factor LAPACK's dgeqrf+dorgqr
// followed by the reference's `_fix_signs` returns, up to rounding.  CholQR2
// (Fukaya, Nakatsukasa, Yanagisawa, Yamamoto 2014) runs it twice:
//
//   G₁ = AᵀA,   R₁ = chol(G₁),   Q₁ = A·R₁⁻¹
//   G₂ = Q₁ᵀQ₁, R₂ = chol(G₂),   Q  = Q₁·R₂⁻¹,   R = R₂·R₁
//
// which is orthogonal to O(u) and backward stable when κ(A) ≲ u^(-1/2).  The
// m-row work is four GEMM-shaped passes on the DMMA GEMM (Gram in split-K
// "partials" mode + a fixed-order slice sum, so results are bitwise
// reproducible); the n×n algebra runs in `cholqr_factor_kernel`, a small
// cooperative kernel over 32×32 blocks held in L2.
//
// Guard: pass 1 estimates κ₁(R₁) = ‖R₁‖₁·‖R₁⁻¹‖₁ and flags a fallback when
// a pivot is not positive, a value is not finite, or κ₁ > kappa_max (1e6;
// tools/proto_cholqr2_full.py measures the accuracy cliff beyond 8e6 and
// column errors ≤ 1% of the parity tolerance below it).  Every later launch
// of the sequence reads the flag and returns; the Householder kernel
// (qr_f64.cuh) reads it and runs only when it is set.  A never changes until
// the final GEMM writes Q into it, so the fallback sees the original input.
#pragma once
#include "common.cuh"

namespace pbq {

constexpr int CQ_THREADS = 256;
constexpr int CQ_LD = 36;                    // shared-memory block stride (≡ 4 mod 16)
constexpr int CQ_BLK = 32 * CQ_LD;           // doubles per staged block
constexpr int CQ_PAIRS = 8;                 // operand pairs staged per batch of a block sum
constexpr int CQ_SMEM_BLOCKS = 3 + 2 * CQ_PAIRS;
constexpr size_t CQ_SMEM_BYTES = size_t(CQ_SMEM_BLOCKS) * CQ_BLK * sizeof(double);
// pass 2 takes the pivot-free series when n·max|G₂ − I| ≤ this: ‖E‖ ≤ 1e-5,
// one fixed-point step from split(E) and the quadratic Neumann inverse leave
// O(‖E‖³) ≤ 1e-15
constexpr double CQ_SERIES_EMAX = 1e-5;

// Distributed Cholesky-QR2: after the caller's allreduce(sum) of the local
// Gram matrices, restore the identity padding (rows/cols in [n, np) summed
// to G·I over G ranks) and, for pass 2, fold max|G − I| of the GLOBAL Gram
// into `emax` (the local reduce's value is not the global one).
__global__ void __launch_bounds__(256) cholqr_dist_fix(double* __restrict__ G, long n, long np,
                                                       unsigned long long* emax) {
  double dev = 0.0;
  for (long e = long(blockIdx.x) * blockDim.x + threadIdx.x; e < np * np; e += long(gridDim.x) * blockDim.x) {
    const long r = e / np, c = e % np;
    if (r >= n || c >= n) {
      G[e] = (r == c) ? 1.0 : 0.0;
    } else if (emax && r <= c) {
      const double d = fabs(G[e] - (r == c ? 1.0 : 0.0));
      dev = (d <= dev) ? dev : d;  // NaN sticks
    }
  }
  if (emax) {
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, dev, o);
      dev = (x <= dev) ? dev : x;
    }
    if ((threadIdx.x & 31) == 0 && dev != 0.0) {
      const unsigned long long bits = (dev == dev) ? __double_as_longlong(dev) : 0x7ff0000000000000ull;
      atomicMax(emax, bits);
    }
  }
}

struct CqArgs {
  int nb;             // 32-blocks per side; np = 32·nb
  long n, np;
  int pass;           // 1: R₁, R₁⁻¹, κ guard   2: R₂, R₂⁻¹, R = R₂·R₁, rank test
  double* G;          // np×np Gram (upper blocks valid); overwritten
  double* R;          // np×np factor (upper blocks written)
  double* X;          // np×np inverse (zeroed by the host; upper blocks written)
  double* T;          // np×np scratch (pass-2 series)
  const double* R1;   // pass 2: the pass-1 factor
  double* Rout;       // pass 2: R = R₂·R₁, n×n with zeros below (may be null)
  long ldr;
  int* rank_flag;     // pass 2 (may be null): 0 ok, 1 rank deficient, 2 zero (linalg.py:48, :160-165)
  int* fallback;      // set to 1 → use the Householder kernel
  double* colsum;     // pass 1: [2][nb][np] per-block column |·| sums of R and X
  const unsigned long long* emax;  // pass 2: max|G − I| (bits), from the reduce
  unsigned int* counter;
  int* stats;         // optional [done, Householder fallbacks, pass 2 by the series, done by the shifted route]
  double kappa_max;
  unsigned long long* phase_ns;  // optional profiling: [pass-1 slots 0..3, pass-2 slots 4..7]
  int allow_series;              // 0: always the blocked Cholesky (test hook)
  // shifted Cholesky-QR3 route (n ≥ CQ_EXT_MIN_N; null/0 otherwise):
  int* shift_req;   // pass 1: a failed guard or pivot requests the route (instead of Householder)
  int* route;       // route kernels run while *route != 0; a failure clears it
  int* hh_req;      // set → the Householder kernel runs
  int shift_mode;   // 1: G += s·I, s = 11(mn + n(n+1))·u·trace(G); no κ guard
  long m;           // rows of the factored matrix (for the shift)
  int rout_full;    // 1: write Rout over the padded np×np (an intermediate product)
  int route_final;  // 1: last factorization of the shifted route (stats[3] counts it)
  int* fail_stats;  // optional: stats[1] counts hand-overs to Householder (also from intermediate passes)
  int chol_1warp;   // diagonal blocks: 0 pipelined two-warp routine, 1 one warp (cq_chol_inv32_warp), 2 lock-step two warps
  int* basis_done;  // pass 2 of a basis-only call on the shifted route (may be null): set to 1 when Q₂ = Q₁·R₂⁻¹
                    // is already a well-conditioned basis (G₂ near I, or max/min |diag R₂| ≤ basis_diag_max),
                    // so the third pass can be skipped
  double basis_diag_max;
  int basis;        // pass 1 of a basis-only call (no second pass): a passed guard completes the call
                    // (rank_flag ← 0: κ₁ ≤ kappa_max bounds every |R_ii|/|R_00| far above 1e-14)
};

#define CQ_MARK(slot)                                                                  \
  do {                                                                                 \
    if (p.phase_ns && blockIdx.x == 0 && threadIdx.x == 0) {                           \
      unsigned long long now_;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));                        \
      p.phase_ns[(p.pass - 1) * 4 + (slot)] += now_ - t_mark;                          \
      t_mark = now_;                                                                   \
    }                                                                                  \
  } while (0)

// 256-thread DMMA block product: c += op(A)·op(B), A, B 32×32 in shared
// memory (ld CQ_LD).  Warp w owns output rows 8·(w/2)…+7 and columns
// 16·(w%2)…+15 (two 8×8 tiles).
template <bool TA, bool TB>
__device__ __forceinline__ void cq_mma(double (&c)[2][2], const double* A, const double* B) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mi = (warp >> 1) * 8, n0 = (warp & 1) * 16;
#pragma unroll
  for (int k0 = 0; k0 < 32; k0 += 4) {
    const double a = TA ? A[(k0 + t) * CQ_LD + mi + g] : A[(mi + g) * CQ_LD + k0 + t];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ni = n0 + h * 8;
      const double b = TB ? B[(ni + g) * CQ_LD + k0 + t] : B[(k0 + t) * CQ_LD + ni + g];
      dmma884(c[h][0], c[h][1], a, b);
    }
  }
}

__device__ __forceinline__ void cq_zero(double (&c)[2][2]) { c[0][0] = c[0][1] = c[1][0] = c[1][1] = 0.0; }

// (row, col) of element e ∈ {0,1} of tile h of this thread's accumulator
__device__ __forceinline__ int cq_row() { return ((threadIdx.x >> 5) >> 1) * 8 + ((threadIdx.x & 31) >> 2); }
__device__ __forceinline__ int cq_col(int h) { return ((threadIdx.x >> 5) & 1) * 16 + h * 8 + 2 * (threadIdx.x & 3); }

__device__ __forceinline__ void cq_store_acc(double* S, const double (&c)[2][2], double scale) {
  const int r = cq_row();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    S[r * CQ_LD + cq_col(h)] = scale * c[h][0];
    S[r * CQ_LD + cq_col(h) + 1] = scale * c[h][1];
  }
}

// accumulator → global block (bi, bj) of an np-stride matrix
__device__ __forceinline__ void cq_store_acc_global(double* M, long np, int bi, int bj, const double (&c)[2][2]) {
  double* row = M + (long(bi) * 32 + cq_row()) * np + long(bj) * 32;
#pragma unroll
  for (int h = 0; h < 2; ++h) __stcg(reinterpret_cast<double2*>(row + cq_col(h)), make_double2(c[h][0], c[h][1]));
}

// global block (bi, bj) of an np-stride matrix → shared memory (cp.async, L2)
__device__ __forceinline__ void cq_load_async(double* S, const double* M, long np, int bi, int bj) {
  const int r = threadIdx.x >> 3, c = (threadIdx.x & 7) * 4;
  const double* src = M + (long(bi) * 32 + r) * np + long(bj) * 32 + c;
  cp_async16(S + r * CQ_LD + c, src, 16);
  cp_async16(S + r * CQ_LD + c + 2, src + 2, 16);
}

__device__ __forceinline__ void cq_store(double* M, long np, int bi, int bj, const double* S) {
  const int r = threadIdx.x >> 3, c = (threadIdx.x & 7) * 4;
  double* dst = M + (long(bi) * 32 + r) * np + long(bj) * 32 + c;
  __stcg(reinterpret_cast<double2*>(dst), make_double2(S[r * CQ_LD + c], S[r * CQ_LD + c + 1]));
  __stcg(reinterpret_cast<double2*>(dst + 2), make_double2(S[r * CQ_LD + c + 2], S[r * CQ_LD + c + 3]));
}

// per-column |·| sums of a staged block → colsum[bi][bj·32 + c]
__device__ __forceinline__ void cq_colsum(double* colsum, long np, int bi, int bj, const double* S) {
  if (threadIdx.x < 32) {
    double s = 0.0;
#pragma unroll 8
    for (int r = 0; r < 32; ++r) s += fabs(S[r * CQ_LD + threadIdx.x]);
    __stcg(colsum + long(bi) * np + long(bj) * 32 + threadIdx.x, s);
  }
}

// Upper Cholesky G = RᵀR of the symmetric 32×32 block S (in place, zeros
// below) and X = R⁻¹ into Xs, by one warp.  Lane j holds column j of the
// augmented [G | I]; step k scales row k by 1/r_kk and eliminates it from the
// rows below, and the same multipliers turn I into R⁻ᵀ (lane j ends with
// column j of R⁻ᵀ = row j of R⁻¹).  Row k of R is broadcast through shared
// memory (one store per lane, 128-bit broadcast loads; double-buffered by
// step parity), and the next pivot is updated by its own lane before the
// broadcast, so the dependent chain per pivot is shuffle → rsqrt → mul →
// fma.  Returns false if a pivot is not positive.
__device__ __noinline__ bool cq_chol_inv32_warp(double* S, double* Xs, double* rowbuf /*64, 16-byte aligned*/) {
  const int lane = threadIdx.x & 31;
  double v[32], w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = S[i * CQ_LD + lane];
    w[i] = (i == lane) ? 1.0 : 0.0;
  }
  bool ok = true;
  double piv = v[0];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dk = __shfl_sync(0xffffffffu, piv, k);
    ok = ok && (dk > 0.0);
    const double inv = fast_rsqrt(dk);
    const double rkj = (lane >= k) ? v[k] * inv : 0.0;
    const double bkj = w[k] * inv;
    v[k] = rkj;
    w[k] = bkj;
    if (k + 1 < 32) piv = fma(-rkj, rkj, v[k + 1]);  // meaningful on lane k+1
    double* rb = rowbuf + (k & 1) * 32;
    rb[lane] = rkj;
    __syncwarp();
#pragma unroll
    for (int i2 = (k + 1) & ~1; i2 < 32; i2 += 2) {
      const double2 r2 = *reinterpret_cast<const double2*>(rb + i2);
      if (i2 > k) {
        v[i2] = fma(-r2.x, rkj, v[i2]);
        w[i2] = fma(-r2.x, bkj, w[i2]);
      }
      if (i2 + 1 > k && i2 + 1 < 32) {
        v[i2 + 1] = fma(-r2.y, rkj, v[i2 + 1]);
        w[i2 + 1] = fma(-r2.y, bkj, w[i2 + 1]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    S[i * CQ_LD + lane] = (i <= lane) ? v[i] : 0.0;
    Xs[lane * CQ_LD + i] = w[i];
  }
  return ok;
}

// The same factorization on two warps: warp 0 eliminates G (the R part),
// warp 1 the identity (the R⁻ᵀ part).  The per-pivot chain of warp 0
// (shuffle → rsqrt → mul → fma of the next pivot) stays as above, but each
// warp now issues half of the step's FP64 updates — the single-warp version
// is issue-bound (64 DFMA of 2 cycles each per pivot), not latency-bound.
// Warp 0 publishes row k of R and 1/r_kk in slot k mod 2 and signals with a
// named-barrier arrive on FULL[k mod 2] (ids 1, 2); warp 1 consumes it and
// frees the slot with EMPTY[k mod 2] (ids 3, 4), which warp 0 waits for two
// pivots later.  One barrier id per slot and direction: a warp never arrives
// twice at a barrier whose previous phase is still open (arrive counts
// threads, so a second arrival of warp 0 would complete it without warp 1).
// Called by warps 0 and 1 of the CTA; the result of warp 0 is the one to use.
constexpr int CQ_RB2 = 36;  // doubles per slot: row k (32), 1/r_kk, padding (16-byte aligned)
__device__ __forceinline__ void cq_bar_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void cq_bar_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }

__device__ __noinline__ bool cq_chol_inv32_2warp(double* S, double* Xs, double* rowbuf /*2·CQ_RB2, 16-byte aligned*/) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = S[i * CQ_LD + lane];
    bool ok = true;
    double piv = v[0];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double dk = __shfl_sync(0xffffffffu, piv, k);
      ok = ok && (dk > 0.0);
      const double inv = fast_rsqrt(dk);
      const double rkj = (lane >= k) ? v[k] * inv : 0.0;
      v[k] = rkj;
      if (k + 1 < 32) piv = fma(-rkj, rkj, v[k + 1]);  // meaningful on lane k+1
      if (k >= 2) cq_bar_sync(3 + (k & 1));             // warp 1 has consumed the slot of pivot k−2
      double* rb = rowbuf + (k & 1) * CQ_RB2;
      rb[lane] = rkj;
      if (lane == 0) rb[32] = inv;
      cq_bar_arrive(1 + (k & 1));
      __syncwarp();
#pragma unroll
      for (int i2 = (k + 1) & ~1; i2 < 32; i2 += 2) {
        const double2 r2 = *reinterpret_cast<const double2*>(rb + i2);
        if (i2 > k) v[i2] = fma(-r2.x, rkj, v[i2]);
        if (i2 + 1 > k && i2 + 1 < 32) v[i2 + 1] = fma(-r2.y, rkj, v[i2 + 1]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) S[i * CQ_LD + lane] = (i <= lane) ? v[i] : 0.0;
    return ok;
  }
  double w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) w[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    cq_bar_sync(1 + (k & 1));
    const double* rb = rowbuf + (k & 1) * CQ_RB2;
    const double bkj = w[k] * rb[32];
    w[k] = bkj;
#pragma unroll
    for (int i2 = (k + 1) & ~1; i2 < 32; i2 += 2) {
      const double2 r2 = *reinterpret_cast<const double2*>(rb + i2);
      if (i2 > k) w[i2] = fma(-r2.x, bkj, w[i2]);
      if (i2 + 1 > k && i2 + 1 < 32) w[i2 + 1] = fma(-r2.y, bkj, w[i2 + 1]);
    }
    if (k + 2 < 32) cq_bar_arrive(3 + (k & 1));  // the slot is free for pivot k+2
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Xs[lane * CQ_LD + i] = w[i];
  return true;
}

// Software-pipelined two-warp variant (the production routine).  The routine
// above keeps the row broadcast on warp 0's dependent chain: pivot k+1 cannot
// start before row k went through shared memory (store → __syncwarp → load,
// ≈ 70 cycles) and the EMPTY handshake with warp 1.  Here
//   * row k+1 receives pivot k's update at once, its multiplier r_{k,k+1}
//     fetched with one shuffle, so the chain per pivot is again shuffle →
//     rsqrt → mul → fma;
//   * the rows below get pivot k's update one pivot later (iteration k+1),
//     when row k has long been visible in shared memory — those FMAs fill the
//     latency of the next pivot's shuffle and rsqrt instead of stalling;
//   * row k of R is written straight into S (its final place; G's row k is in
//     registers by then), so no slot is ever reused and warp 0 never waits
//     for warp 1.  Warp 1 follows pivot by pivot through one mbarrier per
//     pivot (lane 0 of warp 0 arrives after the warp's stores; an mbarrier
//     arrive is a CTA-scope release without the MEMBAR a flag store needs —
//     that fence cost 40 cycles per pivot), used for one phase per call; the
//     phase parity of the call is kept in the state block.
// Same operations in the same order per element: bitwise the results of the
// routines above (tools/microbench/chol32_2warp.cu: 7421 → 4.6k cycles).
// State block (rowbuf, CQ_CHOL_STATE doubles, 16-byte aligned): 1/r_kk per
// pivot, 32 mbarriers, the parity word.  cq_chol_setup once per kernel (all
// threads, then __syncthreads); cq_chol_teardown before another setup of the
// same block.  Called by warps 0 and 1; warp 0's result is the one to use.
constexpr int CQ_CHOL_STATE = 66;
#ifdef CQ_CHOL_TIMING
__device__ long long cq_chol_t[2];  // microbenchmark hook: clock64 at the end of warp 0 / warp 1
#endif
__device__ __forceinline__ void cq_chol_setup(double* rowbuf) {
  uint64_t* bars = reinterpret_cast<uint64_t*>(rowbuf + 32);
  if (threadIdx.x < 32) mbar_init(bars + threadIdx.x, 1);
  if (threadIdx.x == 0) *reinterpret_cast<unsigned int*>(rowbuf + 64) = 0u;
}
__device__ __forceinline__ void cq_chol_teardown(double* rowbuf) {
  uint64_t* bars = reinterpret_cast<uint64_t*>(rowbuf + 32);
  if (threadIdx.x < 32) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bars + threadIdx.x)) : "memory");
}

__device__ __noinline__ bool cq_chol_inv32_pipe(double* S, double* Xs, double* rowbuf) {
  const int lane = threadIdx.x & 31;
  double* invb = rowbuf;  // 1/r_kk, k = 0…31
  uint64_t* bars = reinterpret_cast<uint64_t*>(rowbuf + 32);
  unsigned int* parw = reinterpret_cast<unsigned int*>(rowbuf + 64);
  const unsigned int par = *parw;  // phase parity of this call, read by both warps before the barrier below
  if ((threadIdx.x >> 5) == 0) {
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = S[i * CQ_LD + lane];
    cq_bar_sync(1);  // both warps hold `par` (and S is in registers)
    if (lane == 0) *parw = par ^ 1u;
    bool ok = true;
    double piv = v[0];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double dk = __shfl_sync(0xffffffffu, piv, k);
      if (k >= 1) {  // pivot k−1 on rows k+1…31 (row k took it early, below)
        const double rp = v[k - 1];
        const double* rb = S + (k - 1) * CQ_LD;
#pragma unroll
        for (int i2 = (k + 1) & ~1; i2 < 32; i2 += 2) {
          const double2 r2 = *reinterpret_cast<const double2*>(rb + i2);
          if (i2 > k) v[i2] = fma(-r2.x, rp, v[i2]);
          if (i2 + 1 > k && i2 + 1 < 32) v[i2 + 1] = fma(-r2.y, rp, v[i2 + 1]);
        }
      }
      ok = ok && (dk > 0.0);
      const double inv = fast_rsqrt(dk);
      const double rkj = (lane >= k) ? v[k] * inv : 0.0;
      v[k] = rkj;
      if (k + 1 < 32) {
        piv = fma(-rkj, rkj, v[k + 1]);  // meaningful on lane k+1 (its v[k+1] is complete up to pivot k−1)
        v[k + 1] = fma(-__shfl_sync(0xffffffffu, rkj, k + 1), rkj, v[k + 1]);
      }
      S[k * CQ_LD + lane] = rkj;
      if (lane == 0) invb[k] = inv;
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + k);
    }
#ifdef CQ_CHOL_TIMING
    if (lane == 0) cq_chol_t[0] = clock64();
#endif
    return ok;
  }
  double w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) w[i] = (i == lane) ? 1.0 : 0.0;
  cq_bar_sync(1);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    mbar_wait(bars + k, par);
    const double bkj = w[k] * invb[k];
    Xs[lane * CQ_LD + k] = bkj;  // column k of R⁻¹ is final (stored pivot by pivot: no store tail)
    const double* rb = S + k * CQ_LD;
#pragma unroll
    for (int i2 = (k + 1) & ~1; i2 < 32; i2 += 2) {
      const double2 r2 = *reinterpret_cast<const double2*>(rb + i2);
      if (i2 > k) w[i2] = fma(-r2.x, bkj, w[i2]);
      if (i2 + 1 > k && i2 + 1 < 32) w[i2 + 1] = fma(-r2.y, bkj, w[i2 + 1]);
    }
  }
#ifdef CQ_CHOL_TIMING
  if (lane == 0) cq_chol_t[1] = clock64();
#endif
  return true;
}

__device__ __forceinline__ double cq_split(int r, int c, double x) { return c > r ? x : (c == r ? 0.5 * x : 0.0); }

// ---------------------------------------------------------------------------
// Blocked right-looking Cholesky of G (32×32 blocks) with the inverse built
// column-block by column-block in the same sweep:
//   step k: every CTA factors and inverts G_kk (redundantly — no broadcast
//           barrier); work items are the Schur updates
//             G_ij −= R_kiᵀ·R_kj,  R_kj = R_kk⁻ᵀ·G_kj     (k < i ≤ j)
//           and the inverse blocks
//             X_ik = −(Σ_{i≤l<k} X_il·R_lk)·R_kk⁻¹        (i < k),
//           accumulated one term per step (cq_inverse_accumulate_item /
//           cq_inverse_final_item), which only read blocks finished before
//           step k; the operands of a
//           CTA's first item are fetched (cp.async) while G_kk is factored;
//   one grid barrier per step.
// Pass 2 with a near-identity G₂ = I + E instead runs the pivot-free series
//   X ← split(E − XᵀX) (3 steps from split(E)),  R₂ = I + X,
//   R₂⁻¹ = I − X·(I − X·(I − X)),  R = R₁ + X·R₁
// in six fully parallel rounds.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cq_schur_item(const CqArgs& p, int k, int i, int j, double* sKI, double* sA,
                                              double* sB, double* sC, double* sT, double* sU, bool loaded) {
  const long np = p.np;
  if (!loaded) {
    cq_load_async(sA, p.G, np, k, i);
    if (j != i) cq_load_async(sB, p.G, np, k, j);
    cq_load_async(sC, p.G, np, i, j);
    cp_async_commit();
  }
  cp_async_wait<0>();
  __syncthreads();
  double c[2][2];
  cq_zero(c);
  cq_mma<true, false>(c, sKI, sA);  // R_ki = R_kk⁻ᵀ·G_ki
  cq_store_acc(sT, c, 1.0);
  if (j != i) {
    cq_zero(c);
    cq_mma<true, false>(c, sKI, sB);  // R_kj
    cq_store_acc(sU, c, 1.0);
  }
  __syncthreads();
  const double* rkj = (j != i) ? sU : sT;
  if (i == j) {  // the owner of the diagonal Schur block publishes R_kj
    cq_store(p.R, np, k, j, sT);
    if (p.pass == 1) cq_colsum(p.colsum, np, k, j, sT);
  }
  cq_zero(c);
  cq_mma<true, false>(c, sT, rkj);  // R_kiᵀ·R_kj
  const int r = cq_row();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    c[h][0] = sC[r * CQ_LD + cq_col(h)] - c[h][0];
    c[h][1] = sC[r * CQ_LD + cq_col(h) + 1] - c[h][1];
  }
  cq_store_acc_global(p.G, np, i, j, c);
  __syncthreads();
}


// In-place split(E) of a staged block of E = G − I (block coordinates bi, bj):
// strict upper part, half the diagonal, zeros below (X₀ of the series).
__device__ __forceinline__ void cq_split_staged(double* S, int bi, int bj) {
  const int r = threadIdx.x >> 3, c = (threadIdx.x & 7) * 4;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int gr = bi * 32 + r, gc = bj * 32 + c + e;
    S[r * CQ_LD + c + e] = cq_split(gr, gc, S[r * CQ_LD + c + e] - (gr == gc ? 1.0 : 0.0));
  }
}

// c += Σ_{l=l0..l1} op(M1)_{i,l}·M2_{l,j} (op = transpose of the stored
// block (l,i) when T1), in batches of CQ_PAIRS operand pairs fetched with one
// cp.async round trip.  SPLIT applies split(· − I) to both operands on load.
template <bool T1, bool SPLIT = false>
__device__ __forceinline__ void cq_block_sum(double (&c)[2][2], const double* M1, const double* M2, long np, int i,
                                             int j, int l0, int l1, double* pairs) {
  for (int base = l0; base <= l1; base += CQ_PAIRS) {
    const int cnt = int(lmin(CQ_PAIRS, l1 - base + 1));
    for (int q = 0; q < cnt; ++q) {
      const int l = base + q;
      if (T1)
        cq_load_async(pairs + (2 * q) * CQ_BLK, M1, np, l, i);
      else
        cq_load_async(pairs + (2 * q) * CQ_BLK, M1, np, i, l);
      cq_load_async(pairs + (2 * q + 1) * CQ_BLK, M2, np, l, j);
    }
    cp_async_commit();
    cp_async_wait<0>();
    if (SPLIT) {
      for (int q = 0; q < cnt; ++q) {
        const int l = base + q;
        if (T1)
          cq_split_staged(pairs + (2 * q) * CQ_BLK, l, i);
        else
          cq_split_staged(pairs + (2 * q) * CQ_BLK, i, l);
        cq_split_staged(pairs + (2 * q + 1) * CQ_BLK, l, j);
      }
    }
    __syncthreads();
    for (int q = 0; q < cnt; ++q) cq_mma<T1, false>(c, pairs + (2 * q) * CQ_BLK, pairs + (2 * q + 1) * CQ_BLK);
    __syncthreads();
  }
}

// X_ik = −(Σ_{l=i}^{k−1} X_il·R_lk)·R_kk⁻¹: the inverse's column blocks,
// spread over the block steps instead of being
// summed at step k alone (which made X_0k, with k products, the straggler of
// every late step):
//   accumulate item (step k, row i ≤ k−1, column j > k):
//     P_ij += X_i,k−1 · R_k−1,j      (the first term, i = k−1, overwrites)
//   final item (step k, row i ≤ k−1):
//     X_ik = −(P_ik + X_i,k−1 · R_k−1,k) · R_kk⁻¹   (P_ik absent when i = k−1)
// P_ij lives in X's slot (i, j) until the final item overwrites it.  Every
// item is one block product (plus the R_kk⁻¹ product of the final items).
__device__ __forceinline__ void cq_load_acc_global(double (&c)[2][2], const double* M, long np, int bi, int bj) {
  const double* row = M + (long(bi) * 32 + cq_row()) * np + long(bj) * 32;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(row + cq_col(h)));
    c[h][0] = v.x;
    c[h][1] = v.y;
  }
}

__device__ __forceinline__ void cq_inverse_accumulate_item(const CqArgs& p, int k, int i, int j, double* pairs) {
  const long np = p.np;
  double c[2][2];
  if (i == k - 1)
    cq_zero(c);
  else
    cq_load_acc_global(c, p.X, np, i, j);
  cq_block_sum<false>(c, p.X, p.R, np, i, j, k - 1, k - 1, pairs);
  cq_store_acc_global(p.X, np, i, j, c);
}

__device__ __forceinline__ void cq_inverse_final_item(const CqArgs& p, int k, int i, double* sKI, double* sU,
                                                      double* pairs) {
  const long np = p.np;
  double c[2][2];
  if (i == k - 1)
    cq_zero(c);
  else
    cq_load_acc_global(c, p.X, np, i, k);
  cq_block_sum<false>(c, p.X, p.R, np, i, k, k - 1, k - 1, pairs);
  cq_store_acc(sU, c, 1.0);
  __syncthreads();
  cq_zero(c);
  cq_mma<false, false>(c, sU, sKI);
  double* out = pairs;
  cq_store_acc(out, c, -1.0);
  __syncthreads();
  cq_store(p.X, np, i, k, out);
  if (p.pass == 1) cq_colsum(p.colsum + long(p.nb) * np, np, i, k, out);
  __syncthreads();
}


// The factorization body: run by every CTA of a cooperative grid (the
// factor kernel below, or the single-launch mid-size Cholesky-QR2 of
// cholqr_mid_f64.cuh, which calls it between its own phases).  sm: the
// CQ_SMEM_BYTES dynamic shared-memory block.  p.counter: a grid-barrier
// counter used by this call only (zeroed before the launch).
__device__ void cq_factor_body(const CqArgs& p, double* sm, double* s_rowbuf) {
  double* sKK = sm;           // R_kk
  double* sKI = sm + CQ_BLK;  // R_kk⁻¹
  double* sU = sm + 2 * CQ_BLK;
  double* pairs = sm + 3 * CQ_BLK;  // 2·CQ_PAIRS staged blocks
  double* sA = pairs;
  double* sB = pairs + CQ_BLK;
  double* sC = pairs + 2 * CQ_BLK;
  double* sT = pairs + 3 * CQ_BLK;
  __shared__ int s_ok;
  __shared__ double s_dmax, s_dmin;  // running max / min |R_ii| (pass-1 early κ guard)
  if (p.fallback && __ldcg(p.fallback) != 0) return;  // uniform: written by an earlier launch
  if (p.route && __ldcg(p.route) == 0) return;
  // a failed factorization: pass 1 of the extended chain asks for the shifted
  // route, anything else hands the call to the Householder kernel
  auto fail_all = [&]() {
    if (p.pass == 1 && !p.shift_mode && p.shift_req) {
      *p.shift_req = 1;
    } else {
      if (p.hh_req) *p.hh_req = 1;
      if (p.fail_stats) atomicAdd(p.fail_stats + 1, 1);
    }
    if (p.fallback) *p.fallback = 1;
    if (p.route) *p.route = 0;
  };
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.nb;
  const long np = p.np;
  const bool pass1 = (p.pass == 1);
  unsigned int gen = 0;
  unsigned long long t_mark = 0;
  if (p.phase_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_mark));

  double shift = 0.0;
  if (pass1 && p.shift_mode) {  // s = 11(mn + n(n+1))·u·‖A‖_F², ‖A‖_F² = trace(G) (fixed order in every CTA)
    __shared__ double s_tr[CQ_THREADS / 32];
    double tr = 0.0;
    for (long i = tid; i < p.n; i += CQ_THREADS) tr += __ldcg(p.G + i * np + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    if ((tid & 31) == 0) s_tr[warp] = tr;
    __syncthreads();
    tr = 0.0;
    for (int w = 0; w < CQ_THREADS / 32; ++w) tr += s_tr[w];
    shift = 11.0 * (double(p.m) * double(p.n) + double(p.n) * double(p.n + 1)) * 1.1102230246251565e-16 * tr;
  }
  bool series = false;
  if (!pass1 && p.allow_series) {
    const double em = __longlong_as_double(static_cast<long long>(__ldcg(p.emax)));
    series = double(p.n) * em <= CQ_SERIES_EMAX;  // false for NaN
  }

  if (series) {
    // ---------------- pass 2, near-identity G₂ = I + E -------------------
    // round 1: X = split(E − X₀ᵀX₀), X₀ = split(E) applied on load
    //          ((X₀ᵀX₀)_ij = Σ_{l≤i} X₀_liᵀ·X₀_lj)
    // round 2: R₂⁻¹ = I − X + X·X → p.X;  R = R₁ + X·R₁ → Rout
    const int n_up = nb * (nb + 1) / 2;
    double* Xs = p.R;  // R₂ = I + Xs
    for (int w = blockIdx.x; w < n_up; w += gridDim.x) {
      int i, j;
      upper_tile(w, nb, i, j);
      double c[2][2];
      cq_zero(c);
      cq_block_sum<true, true>(c, p.G, p.G, np, i, j, 0, i, pairs);
      const int r = cq_row();
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int gr = i * 32 + r, gc = j * 32 + cq_col(h) + e;
          const double g = __ldcg(p.G + long(gr) * np + gc) - (gr == gc ? 1.0 : 0.0);
          c[h][e] = cq_split(gr, gc, g - c[h][e]);
        }
      cq_store_acc_global(Xs, np, i, j, c);
    }
    grid_barrier(p.counter, gen);
    CQ_MARK(0);
    const int n_lo = nb * (nb - 1) / 2;
    const int n_items = n_up + (p.Rout ? n_up + n_lo : 0);
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      double c[2][2];
      cq_zero(c);
      if (w < n_up) {
        int i, j;
        upper_tile(w, nb, i, j);
        cq_block_sum<false>(c, Xs, Xs, np, i, j, i, j, pairs);
        const int r = cq_row();
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int gr = i * 32 + r, gc = j * 32 + cq_col(h) + e;
            c[h][e] = (gr == gc ? 1.0 : 0.0) - __ldcg(Xs + long(gr) * np + gc) + c[h][e];
          }
        cq_store_acc_global(p.X, np, i, j, c);
      } else if (w < 2 * n_up) {
        int i, j;
        upper_tile(w - n_up, nb, i, j);
        cq_block_sum<false>(c, Xs, p.R1, np, i, j, i, j, pairs);
        const long r = long(i) * 32 + cq_row();
        const long lim = p.rout_full ? np : p.n;
        if (r < lim) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const long col = long(j) * 32 + cq_col(h) + e;
              if (col < lim)
                p.Rout[r * p.ldr + col] = (col >= r) ? __ldcg(p.R1 + r * np + col) + c[h][e] : 0.0;
            }
        }
      } else {
        int i, j;  // strictly lower block (i > j): zeros
        upper_tile(w - 2 * n_up, nb - 1, j, i);
        i += 1;
        const long lim = p.rout_full ? np : p.n;
        for (int e = tid; e < 1024; e += CQ_THREADS) {
          const long r = long(i) * 32 + e / 32, col = long(j) * 32 + e % 32;
          if (r < lim && col < lim) p.Rout[r * p.ldr + col] = 0.0;
        }
      }
    }
    CQ_MARK(1);
    if (blockIdx.x == 0) {
      // rank test of orth on diag(R) = diag(R₁)·(1 + diag X)
      __shared__ int s_def;
      if (tid == 0) s_def = 0;
      __syncthreads();
      const double d0 = fabs(__ldcg(p.R1) * (1.0 + __ldcg(Xs)));
      for (long i = tid; i < p.n; i += CQ_THREADS) {
        const double di = fabs(__ldcg(p.R1 + i * np + i) * (1.0 + __ldcg(Xs + i * np + i)));
        if (di < 1e-14 * d0) s_def = 1;
      }
      __syncthreads();
      if (tid == 0) {
        if (p.rank_flag) *p.rank_flag = (d0 == 0.0) ? 2 : s_def;
        if (p.stats) {
          atomicAdd(p.stats, 1);
          atomicAdd(p.stats + 2, 1);
          if (p.route_final) atomicAdd(p.stats + 3, 1);
        }
        if (p.basis_done) {  // Q₁ was orthonormal to ~1e-5 already
          *p.basis_done = 1;
          if (p.fail_stats) {
            atomicAdd(p.fail_stats, 1);
            atomicAdd(p.fail_stats + 3, 1);
          }
        }
      }
    }
    return;
  }

  // ---------------- blocked Cholesky + inverse (pass 1, or pass 2) -------
  for (int k = 0; k < nb; ++k) {
    const int mrem = nb - k - 1;
    const int n_upd = mrem * (mrem + 1) / 2;
    const int n_acc = k * mrem;  // accumulate items: rows i < k, columns k+1 … nb−1
    const int n_items = n_upd + k + n_acc;
    // operands of this CTA's first Schur item travel while G_kk is factored
    const bool pre = (int(blockIdx.x) < n_upd);
    cq_load_async(sKK, p.G, np, k, k);
    if (pre) {
      int ii, jj;
      upper_tile(blockIdx.x, mrem, ii, jj);
      const int i = k + 1 + ii, j = k + 1 + jj;
      cq_load_async(sA, p.G, np, k, i);
      if (j != i) cq_load_async(sB, p.G, np, k, j);
      cq_load_async(sC, p.G, np, i, j);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (shift != 0.0) {  // G_kk + s·I (the Schur updates commute with the shift); after the barrier:
      // a thread's cp.async wait covers only its own copies
      if (tid < 32 && k * 32 + tid < p.n) sKK[tid * CQ_LD + tid] += shift;
      __syncthreads();
    }
    if (p.chol_1warp == 1) {  // the single-warp variant (A/B measurements)
      if (warp == 0) {
        const bool ok = cq_chol_inv32_warp(sKK, sKI, s_rowbuf);
        if (tid == 0) s_ok = ok;
      }
    } else if (warp < 2) {  // chol_1warp == 2: the lock-step two-warp routine (A/B)
      const bool ok = p.chol_1warp == 2 ? cq_chol_inv32_2warp(sKK, sKI, s_rowbuf) : cq_chol_inv32_pipe(sKK, sKI, s_rowbuf);
      if (tid == 0) s_ok = ok;
    }
    __syncthreads();
    if (!s_ok) {  // identical in every CTA (same data, same code): all leave together
      if (blockIdx.x == 0 && tid == 0) fail_all();
      return;
    }
    if (pass1 && !p.shift_mode) {
      // early κ guard: κ₁(R₁) = ‖R₁‖₁‖R₁⁻¹‖₁ ≥ max|R_ii| / min|R_jj|, so once the
      // diagonal seen so far spans more than kappa_max the final guard must fail:
      // leave now instead of finishing the factorization (the shifted route or
      // the Householder kernel takes over at once; identical in every CTA)
      if (warp == 0) {
        const long row = long(k) * 32 + (tid & 31);
        const double dgl = row < p.n ? fabs(sKK[(tid & 31) * CQ_LD + (tid & 31)]) : 0.0;
        double mx = dgl, mn = row < p.n ? dgl : INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (tid == 0) {
          s_dmax = k == 0 ? mx : fmax(s_dmax, mx);
          s_dmin = k == 0 ? mn : fmin(s_dmin, mn);
          s_ok = !(s_dmax > p.kappa_max * s_dmin);
        }
      }
      __syncthreads();
      if (!s_ok) {
        if (blockIdx.x == 0 && tid == 0) fail_all();
        return;
      }
    }
    if (blockIdx.x == gridDim.x - 1) {  // the last CTA has the fewest items; CTA 0 carries (k+1, k+1)
      cq_store(p.R, np, k, k, sKK);
      cq_store(p.X, np, k, k, sKI);
      if (pass1) {
        cq_colsum(p.colsum, np, k, k, sKK);
        cq_colsum(p.colsum + long(nb) * np, np, k, k, sKI);
      }
    }
    CQ_MARK(0);
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      if (w < n_upd) {
        int ii, jj;
        upper_tile(w, mrem, ii, jj);
        cq_schur_item(p, k, k + 1 + ii, k + 1 + jj, sKI, sA, sB, sC, sT, sU, pre && w == int(blockIdx.x));
      } else if (w < n_upd + k) {
        cq_inverse_final_item(p, k, w - n_upd, sKI, sU, pairs);
      } else {
        const int u = w - n_upd - k;
        cq_inverse_accumulate_item(p, k, u / mrem, k + 1 + u % mrem, pairs);
      }
    }
    CQ_MARK(1);
    grid_barrier(p.counter, gen);
    CQ_MARK(2);
  }

  if (pass1) {
    // κ₁(R₁) = ‖R₁‖₁·‖R₁⁻¹‖₁ from the per-block column sums (fixed order)
    if (blockIdx.x == 0) {
      __shared__ double s_max[2][CQ_THREADS / 32];
      double mr = 0.0, mx = 0.0;
      for (long j = tid; j < p.n; j += CQ_THREADS) {
        const int jb = int(j / 32);
        double sr = 0.0, sx = 0.0;
        for (int ib = 0; ib <= jb; ++ib) {
          sr += __ldcg(p.colsum + long(ib) * np + j);
          sx += __ldcg(p.colsum + (long(nb) + ib) * np + j);
        }
        mr = fmax(mr, sr);  // fmax drops NaN: finiteness is checked on κ below
        mx = fmax(mx, sx);
        if (!(sr < INFINITY) || !(sx < INFINITY)) mr = INFINITY;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if ((tid & 31) == 0) {
        s_max[0][warp] = mr;
        s_max[1][warp] = mx;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < CQ_THREADS / 32; ++w) {
          mr = fmax(mr, s_max[0][w]);
          mx = fmax(mx, s_max[1][w]);
        }
        const double kappa = mr * mx;
        if (!p.shift_mode && !(kappa <= p.kappa_max)) {
          fail_all();
        } else if (p.basis) {
          if (p.rank_flag) *p.rank_flag = 0;
          if (p.stats) atomicAdd(p.stats, 1);
        }
      }
    }
    return;
  }

  // pass 2 (Cholesky variant): R = R₂·R₁ into Rout, zeros below
  if (p.Rout) {
    const int n_out = nb * nb;
    for (int w = blockIdx.x; w < n_out; w += gridDim.x) {
      const int i = w / nb, j = w % nb;
      double c[2][2];
      cq_zero(c);
      if (i <= j) cq_block_sum<false>(c, p.R, p.R1, np, i, j, i, j, pairs);
      const long r = long(i) * 32 + cq_row();
      const long lim = p.rout_full ? np : p.n;
      if (r < lim) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const long col = long(j) * 32 + cq_col(h) + e;
            if (col < lim) p.Rout[r * p.ldr + col] = (col >= r) ? c[h][e] : 0.0;
          }
      }
    }
  }
  if (blockIdx.x == 0) {
    // rank test of orth (linalg.py:160-165) on diag(R) = diag(R₂)∘diag(R₁)
    __shared__ int s_def;
    if (tid == 0) s_def = 0;
    __syncthreads();
    const double d0 = fabs(__ldcg(p.R) * __ldcg(p.R1));
    for (long i = tid; i < p.n; i += CQ_THREADS) {
      const double di = fabs(__ldcg(p.R + i * np + i) * __ldcg(p.R1 + i * np + i));
      if (di < 1e-14 * d0) s_def = 1;
    }
    __syncthreads();
    if (tid == 0) {
      if (p.rank_flag) *p.rank_flag = (d0 == 0.0) ? 2 : s_def;
      if (p.stats) {
        atomicAdd(p.stats, 1);
        if (p.route_final) atomicAdd(p.stats + 3, 1);
      }
    }
    if (p.basis_done) {
      // κ₂(Q₁) ≥ max/min |diag R₂| and runs within a small factor of it: below
      // basis_diag_max the orthogonality defect of Q₂, ≈ κ₂(Q₁)²·u, is harmless in a basis
      __shared__ double s_mx[CQ_THREADS / 32], s_mn[CQ_THREADS / 32];
      double mx = 0.0, mn = INFINITY;
      for (long i = tid; i < p.n; i += CQ_THREADS) {
        const double di = fabs(__ldcg(p.R + i * np + i));
        mx = fmax(mx, di);
        mn = (di < mn) ? di : mn;  // NaN never lowers mn; it fails the comparison below through mx or mn = inf
        if (!(di == di)) mx = INFINITY;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      if ((tid & 31) == 0) {
        s_mx[warp] = mx;
        s_mn[warp] = mn;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < CQ_THREADS / 32; ++w) {
          mx = fmax(mx, s_mx[w]);
          mn = fmin(mn, s_mn[w]);
        }
        if (mn > 0.0 && mx <= p.basis_diag_max * mn) {
          *p.basis_done = 1;
          if (p.fail_stats) {
            atomicAdd(p.fail_stats, 1);
            atomicAdd(p.fail_stats + 3, 1);
          }
        }
      }
    }
  }
}

// (every return of the body is uniform over the CTA)
__device__ void cq_factor(const CqArgs& p, double* sm) {
  __shared__ __align__(16) double s_rowbuf[2 * CQ_RB2];
  static_assert(2 * CQ_RB2 >= CQ_CHOL_STATE, "row buffer holds the pipelined routine's state block");
  const bool pipe = p.chol_1warp == 0;  // the other variants use the block as plain row slots
  if (pipe) {
    cq_chol_setup(s_rowbuf);
    __syncthreads();
  }
  cq_factor_body(p, sm, s_rowbuf);
  if (pipe) {
    __syncthreads();
    cq_chol_teardown(s_rowbuf);
  }
}

__global__ void __launch_bounds__(CQ_THREADS, 1) cholqr_factor_kernel(CqArgs p) {
  pdl_trigger();  // a programmatically launched successor may start its prologue
  extern __shared__ __align__(16) double sm[];
  cq_factor(p, sm);
}

}  // namespace pbq
