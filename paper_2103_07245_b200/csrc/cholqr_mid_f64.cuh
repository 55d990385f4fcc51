// Cholesky-QR2 of a short matrix with 128 < n ≤ 256 columns in ONE
// cooperative launch — the `householder_qr` / `orth` path (reference
// linalg.py:106-115, :142-165) for PbP-QLP's d×d second stage qr(Rᵀ)
// (algorithms.py:256) at d = 256 (config 3) and other orths with few rows.
//
// The n×n factorizations are too large for one CTA's shared memory (the
// single-launch kernel of cholqr_small_f64.cuh stops at n = 128), so they
// stay the distributed block factorization of cholqr_f64.cuh (cq_factor,
// one grid barrier per 32-block step); what this kernel removes is the
// chain's seven separate launches around them — four small GEMMs (split-K
// Grams and triangular products on a 256-row matrix are ~17 µs each of
// mostly launch, pipeline fill and fix-up) plus the gaps:
//
//   [Gram₁ units] ─bar─ [fixed-order sums → G₁] ─bar─ [cq_factor pass 1]
//   ─bar─ [Q₁ = A·R₁⁻¹ units] ─bar─ [Gram₂ units] ─bar─ [sums → G₂, max|G₂−I|]
//   ─bar─ [cq_factor pass 2: series or Cholesky, R = R₂R₁, rank test]
//   ─bar─ [Q = Q₁·R₂⁻¹ units → A]
//
// A unit is one 32×32 output block over one 32-row chunk (Gram: an upper
// block (i, j) of one chunk's contribution; products: an output block
// (chunk, j) summed over l ≤ j), computed with the 256-thread DMMA block
// product cq_mma, so a 256×256 Gram is 288 units spread over the grid.
// Partial Grams are summed in chunk order (bitwise reproducible).  Guards,
// rank test and Householder hand-over are cq_factor's own; A is written
// only by the last phase.
#pragma once
#include "cholqr_f64.cuh"

namespace pbq {

static_assert(2 * 8 <= CQ_SMEM_BLOCKS, "a product unit stages 2·nb ≤ 16 blocks");

struct CmArgs {
  long m, n, np;
  int nb;
  double* A;         // m×n (lda), overwritten by Q
  long lda;
  double* Q1;        // m×np scratch
  double* part;      // [nch][nblk][32·32] Gram partials
  unsigned int* counter;  // this kernel's grid barrier (zeroed)
  int* fallback;     // set by cq_factor → the Householder kernel runs
  unsigned long long* emax;  // max|G₂ − I| (zeroed)
  CqArgs f1, f2;     // the two factorizations (own counters; G, R, X in np×np layout)
};

// 32×32 block (rows 32·ch…, cols 32·cb…) of an m×cols row-major matrix → S
// (ld CQ_LD), zero outside [0, m) × [0, cols)
__device__ __forceinline__ void cm_load_block(double* S, const double* M, long ld, long m, long cols, long ch, int cb) {
  double v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * CQ_THREADS, r = e >> 5, c = e & 31;
    const long gr = ch * 32 + r, gc = long(cb) * 32 + c;
    v[q] = (gr < m && gc < cols) ? __ldcg(M + gr * ld + gc) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * CQ_THREADS;
    S[(e >> 5) * CQ_LD + (e & 31)] = v[q];
  }
}

// Gram partial units: unit (b, ch) = Mᵀ_{ch,bi}·M_{ch,bj} for upper block b
__device__ void cm_gram_units(const CmArgs& p, const double* M, long ld, long cols, double* sA, double* sB) {
  const long nch = (p.m + 31) / 32;
  const int nblk = p.nb * (p.nb + 1) / 2;
  const long units = long(nblk) * nch;
  for (long u = blockIdx.x; u < units; u += gridDim.x) {
    const int b = int(u / nch);
    const long ch = u % nch;
    int bi = 0, bj = 0;
    upper_tile(b, p.nb, bi, bj);
    cm_load_block(sA, M, ld, p.m, cols, ch, bi);
    if (bj != bi) cm_load_block(sB, M, ld, p.m, cols, ch, bj);
    __syncthreads();
    double c[2][2];
    cq_zero(c);
    cq_mma<true, false>(c, sA, bj != bi ? sB : sA);
    double* dst = p.part + (size_t(ch) * nblk + b) * 1024;
    const int r = cq_row();
#pragma unroll
    for (int h = 0; h < 2; ++h) __stcg(reinterpret_cast<double2*>(dst + r * 32 + cq_col(h)), make_double2(c[h][0], c[h][1]));
    __syncthreads();
  }
}

// G = Σ_ch partials (chunk order) into the np×np layout cq_factor reads,
// identity beyond n; with emax, max|G − I| over the upper part
__device__ void cm_reduce(const CmArgs& p, double* G, unsigned long long* emax) {
  const long nch = (p.m + 31) / 32;
  const int nblk = p.nb * (p.nb + 1) / 2;
  const long E = long(nblk) * 1024;
  double dev = 0.0;
  for (long e = long(blockIdx.x) * CQ_THREADS + threadIdx.x; e < E; e += long(gridDim.x) * CQ_THREADS) {
    const int b = int(e >> 10), w = int(e & 1023);
    int bi = 0, bj = 0;
    upper_tile(b, p.nb, bi, bj);
    const long gr = long(bi) * 32 + (w >> 5), gc = long(bj) * 32 + (w & 31);
    double s = 0.0;
    for (long c0 = 0; c0 < nch; c0 += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = (c0 + q < nch) ? __ldcg(p.part + (size_t(c0 + q) * nblk + b) * 1024 + w) : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += v[q];
    }
    if (gr >= p.n || gc >= p.n) s = (gr == gc) ? 1.0 : 0.0;
    __stcg(G + gr * p.np + gc, s);
    if (emax && gr <= gc) {
      const double d = fabs(s - (gr == gc ? 1.0 : 0.0));
      dev = (d <= dev) ? dev : d;  // NaN sticks
    }
  }
  if (emax) {
#pragma unroll
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

// Triangular product units: Out(ch, j) = Σ_{l ≤ j} M(ch, l)·X(l, j), X upper
// (np×np); written for rows < m and columns < out_cols.  All 2(j+1) operand
// blocks of a unit are staged before one barrier (loads in flight together),
// then the j+1 block products run back to back.  pairs: 2·nb blocks.
__device__ void cm_tri_units(const CmArgs& p, const double* M, long ld, long cols, const double* X, double* Out,
                             long ldo, long out_cols, double* pairs) {
  const long nch = (p.m + 31) / 32;
  const long units = nch * p.nb;
  for (long u = blockIdx.x; u < units; u += gridDim.x) {
    const long ch = u / p.nb;
    const int j = p.nb - 1 - int(u % p.nb);  // the longest sums first
    for (int l = 0; l <= j; ++l) {
      cm_load_block(pairs + (2 * l) * CQ_BLK, M, ld, p.m, cols, ch, l);
      cm_load_block(pairs + (2 * l + 1) * CQ_BLK, X, p.np, p.np, p.np, l, j);
    }
    __syncthreads();
    double c[2][2];
    cq_zero(c);
    for (int l = 0; l <= j; ++l) cq_mma<false, false>(c, pairs + (2 * l) * CQ_BLK, pairs + (2 * l + 1) * CQ_BLK);
    __syncthreads();
    const int r = cq_row();
    const long gr = ch * 32 + r;
    if (gr < p.m) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const long gc = long(j) * 32 + cq_col(h) + e;
          if (gc < out_cols) Out[gr * ldo + gc] = c[h][e];
        }
    }
  }
}

// optional profiling (CTA 0, globaltimer): phase_ns[24 + slot]
#define CM_MARK(slot)                                                                  \
  do {                                                                                 \
    if (ph && blockIdx.x == 0 && threadIdx.x == 0) {                                   \
      unsigned long long now_;                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));                        \
      ph[24 + (slot)] += now_ - t_mark;                                                \
      t_mark = now_;                                                                   \
    }                                                                                  \
  } while (0)

__global__ void __launch_bounds__(CQ_THREADS, 1) cholqr_mid_kernel(CmArgs p) {
  extern __shared__ __align__(16) double sm[];
  double* sA = sm;
  double* sB = sm + CQ_BLK;
  unsigned int gen = 0;
  unsigned long long* ph = p.f1.phase_ns;
  unsigned long long t_mark = 0;
  if (ph) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_mark));
  // ---- Gram₁ and its fixed-order sums
  cm_gram_units(p, p.A, p.lda, p.n, sA, sB);
  grid_barrier(p.counter, gen);
  cm_reduce(p, p.f1.G, nullptr);
  grid_barrier(p.counter, gen);
  CM_MARK(0);
  // ---- pass 1: R₁, R₁⁻¹, κ guard (cq_factor's own barriers)
  cq_factor(p.f1, sm);
  grid_barrier(p.counter, gen);  // CTA 0's final guard is visible to every CTA after this
  CM_MARK(1);
  if (__ldcg(p.fallback) != 0) return;
  // ---- Q₁ = A·R₁⁻¹, then its Gram
  cm_tri_units(p, p.A, p.lda, p.n, p.f1.X, p.Q1, p.np, p.np, sm);
  grid_barrier(p.counter, gen);
  CM_MARK(2);
  cm_gram_units(p, p.Q1, p.np, p.np, sA, sB);
  grid_barrier(p.counter, gen);
  cm_reduce(p, p.f2.G, p.emax);
  grid_barrier(p.counter, gen);
  CM_MARK(3);
  // ---- pass 2: R₂ (series or Cholesky), R = R₂·R₁, rank test
  cq_factor(p.f2, sm);
  grid_barrier(p.counter, gen);
  CM_MARK(4);
  if (__ldcg(p.fallback) != 0) return;
  // ---- Q = Q₁·R₂⁻¹ → A
  cm_tri_units(p, p.Q1, p.np, p.np, p.f2.X, p.A, p.lda, p.n, sm);
  CM_MARK(5);
}

}  // namespace pbq
