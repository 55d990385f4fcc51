// Unpivoted Householder QR of a tall m×n FP64 matrix (m ≥ n), LAPACK
// dgeqrf + dorgqr semantics followed by the reference's sign fix
// (`householder_qr`, /root/reference/pkg/src/pbpqlp/linalg.py:106-115, and
// `_fix_signs`, linalg.py:96-103): on return A holds the thin Q (m×n), R holds
// the n×n upper-triangular factor with diag(R) ≥ 0 (sign 0 → +1), exact zeros
// below the diagonal, and `rank_flag` reports the `orth` rank test
// (linalg.py:142-165): 1 if some |R_ii| < 1e-14·|R_00|, 2 if R_00 == 0.
//
// Layout and schedule: one persistent CTA per SM, launched
// cooperatively.  CTA c owns a contiguous block of rows for the whole call.
// Columns are processed in panels of NB (32/16/8).  Inside a panel each column
// needs one global reduction (the dots of the pivot column with every panel
// column, computed in the same pass as the norm, so a column costs exactly
// one grid barrier); the CTA's panel rows stay resident in shared memory.
// Reflectors are accumulated into the compact-WY T factor on the fly (the
// Vᵀv products ride in the same reduction).  The trailing update
// A2 ← (I − V Tᵀ Vᵀ) A2 and the backward Q formation
// Q ← (I − V T Vᵀ) Q are GEMM-shaped: per-CTA partials of VᵀA2, a
// fixed-order slice reduction (deterministic), then a row-local update.
#pragma once
#include "common.cuh"

namespace pbq {

constexpr int QR_THREADS = 256;
constexpr int QR_NBMAX = 32;
constexpr int QR_STAGE_DOUBLES = 4096;  // one 32 KB staging tile
constexpr double QR_RANK_RTOL = 1e-14;  // RANK_DEFICIENCY_RTOL, linalg.py:48

struct QrArgs {
  long m, n;
  double* A;
  long lda;
  double* R;  // n×n, may be null
  long ldr;
  int want_q;
  int nb;
  long rows_per_cta;
  double* part;    // 2 × G × 32
  double* pivrow;  // 2 × 32
  double* wpart;   // G × 32 × n
  double* ybuf;    // 32 × n
  double* tall;    // ceil(n/nb) × nb × nb
  unsigned int* counter;
  int* rank_flag;  // may be null
};

__device__ __forceinline__ double qr_sign(double beta) { return beta < 0.0 ? -1.0 : 1.0; }

// Shared-memory carve-up (doubles): Ps[rows×(nb+1)] | Ts[nb×nb] | V1[nb×nb] |
// M1[nb×nb] | beta[n] | red[8×32] | svec[32] | prow[32] | wt[32] | stage[4096] | wsl[nb×⌈n/G⌉]
struct QrSmem {
  double *Ps, *Ts, *V1, *M1, *beta, *red, *svec, *prow, *wt, *stage, *wsl;
};

__host__ __device__ inline size_t qr_smem_doubles(long rows_per_cta, int nb, long n, int grid) {
  return size_t(rows_per_cta) * (nb + 1) + 3 * size_t(nb) * nb + size_t(n) + 8 * 32 + 3 * 32 +
         QR_STAGE_DOUBLES + size_t(nb) * ceil_div(n, grid);
}

// W-partial of this CTA: wpart[cta][i][c] = Σ_{r∈[ra,r1)} V[r][i]·X[r][c0+c],
// X = A[:, col0 : col0+ntr].  Thread (ib, cb) owns a 4×4 block of (i, c).
__device__ void qr_wpartial(const QrArgs& p, const QrSmem& s, int nb, long r0, long ra, long r1,
                            long col0, long ntr) {
  const int tid = threadIdx.x;
  const int CW = QR_STAGE_DOUBLES / nb;  // columns per chunk
  const int CB = CW / 4;
  const int ib = tid / CB, cb = tid % CB;
  const int PLD = nb + 1;
  double* wdst = p.wpart + size_t(blockIdx.x) * QR_NBMAX * p.n;
  for (long c0 = 0; c0 < ntr; c0 += CW) {
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (long rc = ra; rc < r1; rc += nb) {
      const int rows = int(lmin(nb, r1 - rc));
      // stage X[rc : rc+rows, c0 : c0+CW]
      for (int e = tid; e < nb * CW; e += QR_THREADS) {
        const int rr = e / CW, cc = e % CW;
        double v = 0.0;
        if (rr < rows && c0 + cc < ntr) v = p.A[(rc + rr) * p.lda + col0 + c0 + cc];
        s.stage[e] = v;
      }
      __syncthreads();
      for (int rr = 0; rr < rows; ++rr) {
        const double* vrow = s.Ps + (rc + rr - r0) * PLD + ib * 4;
        const double* xrow = s.stage + rr * CW + cb;
        double v[4], x[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) v[a] = vrow[a];
#pragma unroll
        for (int b = 0; b < 4; ++b) x[b] = xrow[b * CB];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(v[a], x[b], acc[a][b]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const long c = c0 + cb + b * CB;
        if (c < ntr) __stcg(wdst + size_t(ib * 4 + a) * p.n + c, acc[a][b]);
      }
  }
}

// Fixed-order reduction of the W partials over CTAs for this CTA's column
// slice, then Y = op(T)·W for the slice (op = transpose when `trans_t`).
__device__ void qr_reduce_slice(const QrArgs& p, const QrSmem& s, int nb, long ntr, bool trans_t) {
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  const long cs = long(blockIdx.x) * ntr / G, ce = long(blockIdx.x + 1) * ntr / G;
  const int sw = int(ce - cs);
  if (sw <= 0) return;
  for (int e = tid; e < nb * sw; e += QR_THREADS) {
    const int i = e / sw, c = e % sw;
    double acc = 0.0;
    const double* src = p.wpart + size_t(i) * p.n + cs + c;
    for (int q = 0; q < G; ++q) acc += __ldcg(src + size_t(q) * QR_NBMAX * p.n);
    s.wsl[i * sw + c] = acc;
  }
  __syncthreads();
  for (int e = tid; e < nb * sw; e += QR_THREADS) {
    const int i = e / sw, c = e % sw;
    double acc = 0.0;
    if (trans_t) {
      for (int l = 0; l <= i; ++l) acc = fma(s.Ts[l * nb + i], s.wsl[l * sw + c], acc);
    } else {
      for (int l = i; l < nb; ++l) acc = fma(s.Ts[i * nb + l], s.wsl[l * sw + c], acc);
    }
    __stcg(p.ybuf + size_t(i) * p.n + cs + c, acc);
  }
}

// Row-local update X[r][c] -= Σ_i V[r][i]·Y[i][c] for owned rows [ra, r1).
__device__ void qr_apply_update(const QrArgs& p, const QrSmem& s, int nb, long r0, long ra, long r1,
                                long col0, long ntr) {
  const int tid = threadIdx.x;
  const int CW = QR_STAGE_DOUBLES / nb;
  const int CB = CW / 4;
  const int rb = tid / CB, cb = tid % CB;
  const int PLD = nb + 1;
  for (long c0 = 0; c0 < ntr; c0 += CW) {
    __syncthreads();
    for (int e = tid; e < nb * CW; e += QR_THREADS) {
      const int i = e / CW, cc = e % CW;
      s.stage[e] = (c0 + cc < ntr) ? __ldcg(p.ybuf + size_t(i) * p.n + c0 + cc) : 0.0;
    }
    __syncthreads();
    for (long rc = ra; rc < r1; rc += nb) {
      double acc[4][4];
      bool ok[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const long r = rc + rb * 4 + a;
        ok[a] = r < r1;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const long c = c0 + cb + b * CB;
          acc[a][b] = (ok[a] && c < ntr) ? p.A[r * p.lda + col0 + c] : 0.0;
        }
      }
      for (int i = 0; i < nb; ++i) {
        double y[4], v[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) y[b] = s.stage[i * CW + cb + b * CB];
#pragma unroll
        for (int a = 0; a < 4; ++a) v[a] = ok[a] ? s.Ps[(rc + rb * 4 + a - r0) * PLD + i] : 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(-v[a], y[b], acc[a][b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        if (!ok[a]) continue;
        const long r = rc + rb * 4 + a;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const long c = c0 + cb + b * CB;
          if (c < ntr) p.A[r * p.lda + col0 + c] = acc[a][b];
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(QR_THREADS, 1) qr_tall_kernel(QrArgs p) {
  extern __shared__ __align__(16) double qsm[];
  const int nb = p.nb;
  const int PLD = nb + 1;
  const long m = p.m, n = p.n;
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  const long r0 = long(blockIdx.x) * p.rows_per_cta;
  const long r1 = lmin(m, r0 + p.rows_per_cta);

  QrSmem s;
  {
    double* q = qsm;
    s.Ps = q; q += size_t(p.rows_per_cta) * PLD;
    s.Ts = q; q += nb * nb;
    s.V1 = q; q += nb * nb;
    s.M1 = q; q += nb * nb;
    s.beta = q; q += n;
    s.red = q; q += 8 * 32;
    s.svec = q; q += 32;
    s.prow = q; q += 32;
    s.wt = q; q += 32;
    s.stage = q; q += QR_STAGE_DOUBLES;
    s.wsl = q;
  }
  unsigned int gen = 0;

  // ===================== factorization (dgeqrf) =====================
  for (long k = 0, pidx = 0; k < n; k += nb, ++pidx) {
    const int jb = int(lmin(nb, n - k));
    const long ra = lmax(r0, k);  // first active owned row
    for (long e = tid; e < (r1 - ra) * jb; e += QR_THREADS) {
      const long r = ra + e / jb;
      const int c = int(e % jb);
      s.Ps[(r - r0) * PLD + c] = p.A[r * p.lda + k + c];
    }
    for (int e = tid; e < nb * nb; e += QR_THREADS) s.Ts[e] = 0.0;
    __syncthreads();

    for (int jj = 0; jj < jb; ++jj) {
      const long piv = k + jj;
      const int buf = int(piv & 1);
      // (1) partial dots of the pivot column with all panel columns, rows > piv
      {
        const int c = tid & 31, grp = tid >> 5;
        double acc = 0.0;
        if (c < jb) {
          for (long r = lmax(r0, piv + 1) + grp; r < r1; r += 8) {
            const double* row = s.Ps + (r - r0) * PLD;
            acc = fma(row[jj], row[c], acc);
          }
        }
        s.red[grp * 32 + c] = acc;
      }
      __syncthreads();
      if (tid < jb) {
        double acc = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < 8; ++g2) acc += s.red[g2 * 32 + tid];
        __stcg(p.part + (size_t(buf) * G + blockIdx.x) * 32 + tid, acc);
        if (piv >= r0 && piv < r1) __stcg(p.pivrow + buf * 32 + tid, s.Ps[(piv - r0) * PLD + tid]);
      }
      grid_barrier(p.counter, gen);
      // (2) fixed-order reduction over CTAs
      {
        const int c = tid & 31, grp = tid >> 5;
        double acc = 0.0;
        if (c < jb)
          for (int q = grp; q < G; q += 8) acc += __ldcg(p.part + (size_t(buf) * G + q) * 32 + c);
        s.red[grp * 32 + c] = acc;
      }
      __syncthreads();
      if (tid < jb) {
        double acc = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < 8; ++g2) acc += s.red[g2 * 32 + tid];
        s.svec[tid] = acc;
        s.prow[tid] = __ldcg(p.pivrow + buf * 32 + tid);
      }
      __syncthreads();
      // (3) Householder scalars (dlarfg convention: beta = -sign(alpha)·‖x‖)
      const double alpha = s.prow[jj], sigma = s.svec[jj];
      double beta, tau, scale;
      if (sigma == 0.0) {
        beta = alpha;
        tau = 0.0;
        scale = 0.0;
      } else {
        const double nrm = sqrt(fma(alpha, alpha, sigma));
        beta = signbit(alpha) ? nrm : -nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      if (tid < jb) s.wt[tid] = (tid > jj) ? tau * fma(scale, s.svec[tid], s.prow[tid]) : 0.0;
      // T column jj: T[0:jj, jj] = -tau · T[0:jj, 0:jj] · z,  z_l = v_lᵀ v_jj
      if (tid < jj) {
        double acc = 0.0;
        for (int l = tid; l < jj; ++l) acc = fma(s.Ts[tid * nb + l], fma(scale, s.svec[l], s.prow[l]), acc);
        s.Ts[tid * nb + jj] = -tau * acc;
      }
      if (tid == 0) {
        s.Ts[jj * nb + jj] = tau;
        s.beta[piv] = beta;
      }
      __syncthreads();
      // (4) apply H to the CTA's rows of the panel
      for (long r = lmax(r0, piv) + tid; r < r1; r += QR_THREADS) {
        double* row = s.Ps + (r - r0) * PLD;
        if (r == piv) {
          for (int c = jj + 1; c < jb; ++c) row[c] -= s.wt[c];
          row[jj] = beta;
        } else {
          const double v = scale * row[jj];
          row[jj] = v;
          for (int c = jj + 1; c < jb; ++c) row[c] = fma(-s.wt[c], v, row[c]);
        }
      }
      __syncthreads();
    }

    // write the factored panel back; CTA 0 keeps T for the Q formation
    for (long e = tid; e < (r1 - ra) * jb; e += QR_THREADS) {
      const long r = ra + e / jb;
      const int c = int(e % jb);
      p.A[r * p.lda + k + c] = s.Ps[(r - r0) * PLD + c];
    }
    if (blockIdx.x == 0)
      for (int e = tid; e < nb * nb; e += QR_THREADS) p.tall[pidx * nb * nb + e] = s.Ts[e];

    const long ntr = n - k - jb;
    if (ntr > 0) {
      // V form: unit diagonal, zeros above
      for (long e = tid; e < (r1 - ra) * jb; e += QR_THREADS) {
        const long r = ra + e / jb;
        const int c = int(e % jb);
        if (r < k + c) s.Ps[(r - r0) * PLD + c] = 0.0;
        else if (r == k + c) s.Ps[(r - r0) * PLD + c] = 1.0;
      }
      __syncthreads();
      qr_wpartial(p, s, nb, r0, ra, r1, k + jb, ntr);
      grid_barrier(p.counter, gen);
      qr_reduce_slice(p, s, nb, ntr, /*trans_t=*/true);
      grid_barrier(p.counter, gen);
      qr_apply_update(p, s, nb, r0, ra, r1, k + jb, ntr);
    }
    __syncthreads();
  }

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
  // every CTA's factored panels (V1 blocks, T factors) are published before
  // any CTA starts reading them
  grid_barrier(p.counter, gen);

  // ===================== Q formation (dorgqr, backward) =====================
  const long npan = ceil_div(n, nb);
  for (long pidx = npan - 1; pidx >= 0; --pidx) {
    const long k = pidx * nb;
    const int jb = int(lmin(nb, n - k));
    const long ra = lmax(r0, k);
    // V_p (own rows) and V1 (pivot block, needed by every CTA)
    for (long e = tid; e < (r1 - ra) * jb; e += QR_THREADS) {
      const long r = ra + e / jb;
      const int c = int(e % jb);
      double v;
      if (r < k + c) v = 0.0;
      else if (r == k + c) v = 1.0;
      else v = p.A[r * p.lda + k + c];
      s.Ps[(r - r0) * PLD + c] = v;
    }
    for (int e = tid; e < jb * jb; e += QR_THREADS) {
      const int a = e / jb, c = e % jb;
      double v = (a == c) ? 1.0 : 0.0;
      if (a > c) v = __ldcg(p.A + (k + a) * p.lda + k + c);
      s.V1[a * nb + c] = v;
    }
    // the last panel's T is still resident from the factorization
    if (pidx < npan - 1)
      for (int e = tid; e < nb * nb; e += QR_THREADS) s.Ts[e] = __ldcg(p.tall + pidx * nb * nb + e);
    __syncthreads();
    const long ntr = n - k - jb;
    if (ntr > 0) {
      qr_wpartial(p, s, nb, r0, ra, r1, k + jb, ntr);
      grid_barrier(p.counter, gen);
      qr_reduce_slice(p, s, nb, ntr, /*trans_t=*/false);
      grid_barrier(p.counter, gen);
      qr_apply_update(p, s, nb, r0, ra, r1, k + jb, ntr);
    } else {
      grid_barrier(p.counter, gen);  // every CTA has read V1 before it is overwritten
    }
    // M1 = T · V1ᵀ  (jb × jb)
    for (int e = tid; e < jb * jb; e += QR_THREADS) {
      const int i = e / jb, c = e % jb;
      double acc = 0.0;
      for (int l = i; l < jb; ++l) acc = fma(s.Ts[i * nb + l], s.V1[c * nb + l], acc);
      s.M1[i * nb + c] = acc;
    }
    __syncthreads();
    // panel columns: Q[r][k+c] = δ(r, k+c) − Σ_i V[r][i]·M1[i][c]
    for (long e = tid; e < (r1 - ra) * jb; e += QR_THREADS) {
      const long r = ra + e / jb;
      const int c = int(e % jb);
      const double* vrow = s.Ps + (r - r0) * PLD;
      double acc = (r == k + c) ? 1.0 : 0.0;
      for (int i = 0; i < jb; ++i) acc = fma(-vrow[i], s.M1[i * nb + c], acc);
      p.A[r * p.lda + k + c] = acc;
    }
    __syncthreads();
  }
  // sign fix: Q[:, c] *= sign(R_cc)
  for (long e = tid; e < (r1 - r0) * n; e += QR_THREADS) {
    const long r = r0 + e / n, c = e % n;
    if (s.beta[c] < 0.0) p.A[r * p.lda + c] = -p.A[r * p.lda + c];
  }
}

}  // namespace pbq
