// EXPERIMENT, not built into libpbq: the single-CTA second stage measured slower than the chain.
// Second stage of PbP-QLP for d ≤ SQ_MAX_D on ONE CTA in shared memory
// (reference algorithms.py:256-257: (W, R̃) = householder_qr(Rᵀ), L = tril(R̃ᵀ)).
//
// The d×d matrix Rᵀ is small enough for one CTA's shared memory, so the whole
// factorization runs without a grid barrier or a second launch: LAPACK's
// dgeqr2 (dlarfg reflectors), the reference's sign fix (linalg.py:96-103:
// diag R̃ ≥ 0, a zero diagonal counts as +), L = tril(R̃ᵀ) written straight to
// its output, then dorg2r's backward accumulation of W in place.  The
// working matrix is column-major in shared memory (column k contiguous), so
// the per-column reductions and updates are unit-stride across a warp.
// For a full-rank R the factorization is unique, so the result matches the
// reference's LAPACK call to rounding.  Larger d uses the Cholesky-QR2 chain.
#pragma once
#include "common.cuh"

namespace pbq {

constexpr int SQ_THREADS = 1024;
constexpr int SQ_MAX_D = 160;  // d·(d+1) doubles + tau ≤ 227 KB

__host__ __device__ inline size_t small_qr_smem_bytes(int d) {
  return (size_t(d) * (d + 1) + d + 64) * sizeof(double);
}

__device__ __forceinline__ double sq_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// R: d×d upper triangular, row-major (ld ldr).  Outputs W (d×d row-major, ld
// ldw) and L (d×d row-major, ld ldl, zeros above the diagonal).
__global__ void __launch_bounds__(SQ_THREADS, 1) small_qlp_kernel(const double* __restrict__ R, long ldr, int d,
                                                                  double* __restrict__ W, long ldw,
                                                                  double* __restrict__ L, long ldl) {
  extern __shared__ __align__(16) double sq[];
  const int ldc = d + 1;      // column stride of the working matrix M (column-major)
  double* M = sq;             // M[k·ldc + i] = M(i, k)
  double* tau = sq + size_t(d) * ldc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = SQ_THREADS / 32;

  // M = Rᵀ: column k of M is row k of R (coalesced)
  for (int e = tid; e < d * d; e += SQ_THREADS) {
    const int k = e / d, i = e % d;
    M[k * ldc + i] = R[long(k) * ldr + i];
  }
  __syncthreads();

  // A group of SQ_G lanes owns one column of the trailing update: each lane
  // takes every SQ_G-th row of the dot product with the reflector (a 3-step
  // shuffle reduction inside the group) and of the update, so every warp
  // works on 32/SQ_G columns at once and a step is a few short loops.
  constexpr int SQ_G = 8;
  const int gl = lane % SQ_G;                 // lane within the group
  const int gid = tid / SQ_G;                 // group index = column slot
  const unsigned gmask = 0xffu << (lane & ~(SQ_G - 1));
  auto apply = [&](int j, int k) {  // A(j:, k) −= τ_j·(vᵀA(j:, k))·v, v = (1, M(j+1:, j))
    const double* cj = M + j * ldc;
    double* ck = M + k * ldc;
    double s = (gl == 0) ? ck[j] : 0.0;
#pragma unroll 4
    for (int i = j + 1 + gl; i < d; i += SQ_G) s = fma(cj[i], ck[i], s);
#pragma unroll
    for (int o = SQ_G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(gmask, s, o);
    const double w = tau[j] * s;
    if (gl == 0) ck[j] -= w;
#pragma unroll 4
    for (int i = j + 1 + gl; i < d; i += SQ_G) ck[i] = fma(-w, cj[i], ck[i]);
  };
  auto reflector = [&](int j) {  // warp 0: dlarfg on column j (rows j..d−1)
    double* cj = M + j * ldc;
    double s = 0.0;
    for (int i = j + 1 + lane; i < d; i += 32) s = fma(cj[i], cj[i], s);
    s = sq_warp_sum(s);  // ‖x(2:n)‖²
    const double alpha = cj[j];
    double t = 0.0, scale = 1.0, beta = alpha;
    if (s != 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, s));
      beta = alpha >= 0.0 ? -nrm : nrm;  // −sign(α)·‖x‖
      t = (beta - alpha) * fast_rcp(beta);
      scale = fast_rcp(alpha - beta);
    }
    __syncwarp();
    for (int i = j + 1 + lane; i < d; i += 32) cj[i] *= scale;  // v(2:n)
    __syncwarp();
    if (lane == 0) {
      tau[j] = t;
      cj[j] = beta;
    }
  };
  // ---- dgeqr2 with a one-column lookahead: warp 0's lane 0 owns column j+1,
  // so warp 0 builds reflector j+1 right after step j's update of it while
  // the other threads finish theirs; one CTA barrier per column.
  if (warp == 0) reflector(0);
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    // column j+1 is group 0's (warp 0), so warp 0 can build its reflector next
    if (tau[j] != 0.0)
      for (int k = j + 1 + gid; k < d; k += SQ_THREADS / SQ_G) apply(j, k);
    if (warp == 0 && j + 1 < d) {
      __syncwarp();
      reflector(j + 1);
    }
    __syncthreads();
  }

  // ---- sign fix and L = tril(R̃ᵀ): L(i, k) = s_k·R̃(k, i) = s_k·M(k, i) for k ≤ i
  for (int e = tid; e < d * d; e += SQ_THREADS) {
    const int i = e / d, k = e % d;  // row i of L, coalesced
    double v = 0.0;
    if (k <= i) {
      const double rkk = M[k * ldc + k];
      v = (rkk < 0.0 ? -1.0 : 1.0) * M[i * ldc + k];
    }
    L[long(i) * ldl + k] = v;
  }
  __syncthreads();

  // ---- dorg2r: W = H_0·H_1·…·H_{d−1}·I in place (backward accumulation)
  __shared__ double s_sign[SQ_MAX_D];
  for (int k = tid; k < d; k += SQ_THREADS) s_sign[k] = M[k * ldc + k] < 0.0 ? -1.0 : 1.0;
  __syncthreads();
  // Step i applies H_i to the accumulated columns k > i (thread per column).
  // Column i itself still holds v_i during step i; the thread that owns it in
  // step i−1 first turns it into the accumulated column (−τ_i·v_i below the
  // diagonal, 1 − τ_i on it, zeros above), so one barrier per step suffices.
  auto finish_col = [&](int i) {
    double* ci = M + i * ldc;
    const double ti = tau[i];
    for (int r = 0; r < i; ++r) ci[r] = 0.0;
    ci[i] = 1.0 - ti;
    for (int r = i + 1; r < d; ++r) ci[r] *= -ti;
  };
  for (int i = d - 1; i >= 0; --i) {
    for (int k = i + 1 + gid; k < d; k += SQ_THREADS / SQ_G) {
      if (k == i + 1) {  // column i+1 left step i+1 as v_{i+1}
        if (gl == 0) finish_col(k);
        __syncwarp(gmask);
      }
      if (tau[i] != 0.0) apply(i, k);  // rows ≤ i of column k are zero (A(i,k) included)
    }
    __syncthreads();
  }
  if (tid == 0) finish_col(0);
  __syncthreads();
  // ---- W with the column signs: W(i, k) = s_k·M(i, k)
  for (int e = tid; e < d * d; e += SQ_THREADS) {
    const int i = e / d, k = e % d;
    W[long(i) * ldw + k] = s_sign[k] * M[k * ldc + i];
  }
}

}  // namespace pbq
