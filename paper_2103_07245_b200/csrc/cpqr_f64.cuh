// Column-pivoted QR pivot selection (LAPACK dgeqp3 / dlaqp2 semantics) for
// the d×d core of cor_utv (reference algorithms.py:351, linalg.py:118-129:
// scipy.linalg.qr(m, pivoting=True) → LAPACK dgeqp3).
//
// Householder QR with column pivoting is the unpivoted Householder QR of
// M[:, perm]: the pivot order is the only thing pivoting adds.  This kernel
// runs the pivoted elimination to produce `perm`; Q and R then come from the
// library's Householder/Cholesky-QR kernels on the gathered columns (unique
// for full rank with diag R ≥ 0, which is the reference's _fix_signs
// convention, linalg.py:96-103).
//
// Pivot rule, restated from LAPACK 3.x dlaqp2 (the unblocked form of what
// dgeqp3/dlaqps do; the blocked form picks the same pivots):
//   * vn1[j] = vn2[j] = ‖M[:, j]‖ initially;
//   * step k: p = first position ≥ k of max vn1 (idamax), swap positions k, p;
//     reflector from column p rows k..m-1 (dlarfg), applied to the trailing
//     columns (dlarf);
//   * norm downdating per trailing column j: t = max(0, 1 − (|M[k,j]|/vn1[j])²),
//     t2 = t·(vn1[j]/vn2[j])²; if t2 ≤ √ε (ε = 2⁻⁵³) the norm is recomputed
//     from rows k+1.. (vn2 = vn1), else vn1[j] ·= √t.
//
// Layout: the launch transposes the row-major m×n input into W (n rows of
// length m: column j of M is contiguous).  Columns are owned by CTAs
// (phys j ↦ CTA j mod G, warp-per-column inside the CTA); every CTA
// re-derives the pivot and the reflector from the shared vn1 / pivot column
// through L2, and a pivoted column is never written again, so one grid
// barrier per step suffices.  Cooperative launch (co-residency) is required.
#pragma once
#include "common.cuh"

namespace pbq {

constexpr int CP_THREADS = 256;
constexpr int CP_WARPS = CP_THREADS / 32;

struct CpArgs {
  long m, n, steps;  // steps = min(m, n)
  double* W;         // n × ldw, column j of M at W + j·ldw
  long ldw;
  double* vn1;  // n (by physical column)
  double* vn2;
  int64_t* perm;  // out: perm[pos] = original column index
  unsigned int* counter;
  unsigned char* scratch;  // per-CTA copy of the shared-memory layout when it exceeds
  size_t scratch_stride;   // the opt-in limit (large m / n), else null
};

__host__ __device__ inline size_t cp_scratch_bytes(long m, long n) {
  return size_t(m) * 8 + size_t(3 * CP_WARPS + 2) * 8 + size_t(CP_WARPS + 2 * n) * 4;
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (same tree in every CTA); red holds CP_WARPS doubles.
__device__ __forceinline__ double block_sum_f64(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum_f64(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CP_WARPS; ++i) s += red[i];
  return s;
}

__global__ void __launch_bounds__(CP_THREADS, 1) cpqr_pivot_kernel(CpArgs p) {
  extern __shared__ __align__(16) unsigned char cp_smem[];
  unsigned char* base = p.scratch ? p.scratch + blockIdx.x * p.scratch_stride : cp_smem;
  double* sv = reinterpret_cast<double*>(base);     // reflector v (m)
  double* red = sv + p.m;                           // CP_WARPS doubles
  double* bval = red + CP_WARPS;                    // CP_WARPS (argmax values)
  double* scal = bval + CP_WARPS;                   // [tau, scal]
  int* bpos = reinterpret_cast<int*>(scal + 2);     // CP_WARPS
  int* sperm = bpos + CP_WARPS;                     // pos → phys (n)
  int* spos = sperm + p.n;                          // phys → pos (n)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long m = p.m, n = p.n, G = gridDim.x;
  const double tol3z = 1.0536712127723509e-08;  // √(2⁻⁵³), dlamch('Epsilon')
  unsigned int gen = 0;

  for (long j = tid; j < n; j += CP_THREADS) {
    sperm[j] = int(j);
    spos[j] = int(j);
  }
  // initial column norms (owners)
  for (long t = warp; blockIdx.x + t * G < n; t += CP_WARPS) {
    const long j = blockIdx.x + t * G;
    const double* col = p.W + j * p.ldw;
    double ss = 0.0;
    for (long i = lane; i < m; i += 32) {
      const double x = col[i];
      ss = fma(x, x, ss);
    }
    ss = warp_sum_f64(ss);
    if (lane == 0) {
      p.vn1[j] = sqrt(ss);
      p.vn2[j] = sqrt(ss);
    }
  }
  grid_barrier(p.counter, gen);

  for (long k = 0; k < p.steps; ++k) {
    // ---- pivot: first position ≥ k holding max vn1 (idamax) ----
    double best = -1.0;
    int bp = int(n);
    for (long pos = k + tid; pos < n; pos += CP_THREADS) {
      const double v = __ldcg(p.vn1 + sperm[pos]);
      if (v > best) {  // positions ascend per thread: strict > keeps the first
        best = v;
        bp = int(pos);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (ov > best || (ov == best && op < bp)) {
        best = ov;
        bp = op;
      }
    }
    __syncthreads();  // previous step's readers of bval/bpos/sperm are done
    if (lane == 0) {
      bval[warp] = best;
      bpos[warp] = bp;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = bval[0];
      int pp = bpos[0];
      for (int w = 1; w < CP_WARPS; ++w)
        if (bval[w] > bv || (bval[w] == bv && bpos[w] < pp)) {
          bv = bval[w];
          pp = bpos[w];
        }
      const int a = sperm[k], b = sperm[pp];  // swap positions k and pp
      sperm[k] = b;
      sperm[pp] = a;
      spos[b] = int(k);
      spos[a] = pp;
    }
    __syncthreads();
    if (k == p.steps - 1) break;  // no later pivot depends on the last update
    const long c = sperm[k];
    const long len = m - k;

    // ---- reflector from column c, rows k..m-1 (dlarfg) ----
    const double* pc = p.W + c * p.ldw + k;
    double ss = 0.0;
    for (long i = tid; i < len; i += CP_THREADS) {
      const double x = __ldcg(pc + i);
      sv[i] = x;
      if (i > 0) ss = fma(x, x, ss);
    }
    const double xn2 = block_sum_f64(ss, red);  // includes the __syncthreads for sv
    if (tid == 0) {
      const double alpha = sv[0];
      double tau = 0.0, sc = 0.0;
      if (len > 1 && xn2 > 0.0) {
        const double beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
        tau = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      scal[0] = tau;
      scal[1] = sc;
    }
    __syncthreads();
    const double tau = scal[0], sc = scal[1];
    for (long i = 1 + tid; i < len; i += CP_THREADS) sv[i] *= sc;
    if (tid == 0) sv[0] = 1.0;
    __syncthreads();

    // ---- apply H to owned trailing columns; downdate their norms ----
    for (long t = warp; blockIdx.x + t * G < n; t += CP_WARPS) {
      const long j = blockIdx.x + t * G;
      if (spos[j] <= k) continue;
      double* col = p.W + j * p.ldw + k;
      double dot = 0.0;
      if (tau != 0.0) {
        for (long i = lane; i < len; i += 32) dot = fma(sv[i], __ldcg(col + i), dot);
        dot = warp_sum_f64(dot);
      }
      const double tw = tau * dot;
      double tail = 0.0, head = 0.0;
      for (long i = lane; i < len; i += 32) {
        double x = __ldcg(col + i);
        if (tau != 0.0) {
          x = fma(-tw, sv[i], x);
          col[i] = x;
        }
        if (i == 0)
          head = x;
        else
          tail = fma(x, x, tail);
      }
      head = __shfl_sync(0xffffffffu, head, 0);
      const double v1 = __ldcg(p.vn1 + j);
      if (v1 != 0.0) {
        // Fortran order, no FMA contraction: 1 − (|a|/vn1)², then temp·(vn1/vn2)²
        const double ra = fabs(head) / v1;
        const double tmp = fmax(0.0, 1.0 - __dmul_rn(ra, ra));
        const double r = v1 / __ldcg(p.vn2 + j);
        const double tmp2 = __dmul_rn(tmp, __dmul_rn(r, r));
        if (tmp2 <= tol3z) {
          tail = warp_sum_f64(tail);
          if (lane == 0) {
            const double nv = (k + 1 < m) ? sqrt(tail) : 0.0;
            p.vn1[j] = nv;
            p.vn2[j] = nv;
          }
        } else if (lane == 0) {
          p.vn1[j] = v1 * sqrt(tmp);
        }
      }
    }
    grid_barrier(p.counter, gen);
  }
  if (blockIdx.x == 0)
    for (long j = tid; j < n; j += CP_THREADS) p.perm[j] = sperm[j];
}

// dst[:, i] = src[:, perm[i]] (row-major, rows × cols)
__global__ void gather_cols_kernel(long rows, long cols, const double* __restrict__ src, long lds,
                                   const int64_t* __restrict__ perm, double* __restrict__ dst, long ldd) {
  const long total = rows * cols;
  for (long e = long(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += long(gridDim.x) * blockDim.x) {
    const long r = e / cols, i = e - r * cols;
    dst[r * ldd + i] = src[r * lds + perm[i]];
  }
}

}  // namespace pbq
