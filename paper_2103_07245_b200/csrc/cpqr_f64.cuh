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
      double v = __ldcg(p.vn1 + sperm[pos]);
      if (v != v) v = -0.5;  // NaN never wins (idamax), but an all-NaN set still yields a position
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

// ======================= single-cluster variant (n ≤ ~640) =================
// The whole problem lives in one thread-block cluster of C ≤ 16 CTAs: CTA r
// holds its columns j ≡ r (mod C) in shared memory for the whole
// elimination.  Per step: a CTA-local argmax into a double-buffered slot,
// ONE hardware cluster barrier, every CTA reads the C slots and the pivot
// column straight from the owner's shared memory (DSMEM, ld.shared::cluster),
// then updates its own columns in place.  No global memory traffic and no
// software grid barrier on the step path.
__device__ __forceinline__ unsigned cp_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Cluster barrier ordering shared memory only (all cross-CTA traffic of the
// cluster kernel is DSMEM): a release fence restricted to this CTA's shared
// memory at cluster scope, a relaxed arrive, an acquiring wait.  Compiles to
// MEMBAR.ALL.CTA instead of the GPU-scope MEMBAR of arrive.release.
__device__ __forceinline__ void cp_cluster_sync() {
  asm volatile("fence.release.sync_restrict::shared::cta.cluster;\n" ::: "memory");
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// shared::cluster address of `p` (a local shared-memory pointer) in CTA `rank`
__device__ __forceinline__ uint32_t cp_mapa(const void* p, unsigned rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ double cp_ld_dsmem(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

struct CpClusterArgs {
  long m, n, steps;
  const double* W;  // n × ldw (column j of M contiguous), read once
  long ldw;
  int64_t* perm;
  int nc;    // columns per CTA (ceil(n / C))
  long ldc;  // smem row stride of a held column (≥ m)
};

__host__ __device__ inline size_t cp_cluster_smem(long m, long n, int nc, long ldc) {
  (void)n;
  return (size_t(nc) * ldc + 2 * size_t(nc) + 2 * CP_WARPS * 2 + m + 1) * 8 + size_t(nc) * 4 + 16;
}

__device__ __forceinline__ unsigned long long cp_ld_dsmem_u64(uint32_t addr) {
  unsigned long long v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}

// (value, key) max with ties to the smaller key; key = position << 32 | column
__device__ __forceinline__ void cp_better(double& bv, unsigned long long& bk, double ov, unsigned long long ok) {
  if (ov > bv || (ov == bv && ok < bk)) {
    bv = ov;
    bk = ok;
  }
}

// Every warp is self-sufficient: it owns columns l ≡ warp (mod 8) of its
// CTA, publishes one pivot candidate per step, reduces all 8·C candidates
// itself (DSMEM), and loads the pivot column into registers (T doubles per
// lane, rows k + lane + 32t) to apply the reflector to its own columns.  The
// only synchronisation is one cluster barrier per step.
template <int T>
__global__ void __launch_bounds__(CP_THREADS, 1) cpqr_cluster_kernel(CpClusterArgs p) {
  extern __shared__ __align__(16) unsigned char cc_smem[];
  const long m = p.m, n = p.n, ldc = p.ldc;
  const int nc = p.nc;
  double* cols = reinterpret_cast<double*>(cc_smem);  // nc × ldc
  double* vn1 = cols + size_t(nc) * ldc;              // nc
  double* vn2 = vn1 + nc;                             // nc
  double* slots = vn2 + nc;                           // 2 × CP_WARPS × [value, key]
  double* sv = slots + 2 * CP_WARPS * 2;              // m: the staged pivot column
  int* lpos = reinterpret_cast<int*>(sv + m + 1);     // position of held column l (sv[m]: broadcast pivot key)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned C = gridDim.x, rank = cp_cluster_rank();
  const double tol3z = 1.0536712127723509e-08;  // √(2⁻⁵³)
  const int ncand = int(C) * CP_WARPS;

  for (int l = warp; l < nc; l += CP_WARPS) {
    const long j = rank + long(l) * C;
    double ss = 0.0;
    if (j < n) {
      const double* src = p.W + j * p.ldw;
      double* dst = cols + size_t(l) * ldc;
      for (long i = lane; i < m; i += 32) {
        const double x = src[i];
        dst[i] = x;
        ss = fma(x, x, ss);
      }
    }
    ss = warp_sum_f64(ss);
    if (lane == 0) {
      vn1[l] = sqrt(ss);
      vn2[l] = sqrt(ss);
      lpos[l] = int(j);
    }
  }
  __syncwarp();

  for (long k = 0; k < p.steps; ++k) {
    // ---- this warp's candidate: max vn1 over its free columns, ties → lowest position
    double bv = -1.0;
    unsigned long long bk = ~0ull;
    for (int l = warp + CP_WARPS * lane; l < nc; l += CP_WARPS * 32) {
      const long j = rank + long(l) * C;
      if (j < n && lpos[l] >= k) {
        const double v = vn1[l];
        cp_better(bv, bk, v == v ? v : -0.5, (static_cast<unsigned long long>(lpos[l]) << 32) | j);  // NaN: last resort
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      cp_better(bv, bk, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bk, o));
    double* slot = slots + 2 * CP_WARPS * (k & 1);  // 8 × [value, key] per buffer
    if (lane == 0) {
      slot[2 * warp] = bv;
      reinterpret_cast<unsigned long long*>(slot)[2 * warp + 1] = bk;
    }
    cp_cluster_sync();  // candidates of step k and the held columns after step k−1 are final
    // ---- warp 0: global pivot from the 8·C candidates, then stage column c
    // rows k..m-1 from its owner (DSMEM) into this CTA's shared memory
    const long len = m - k;
    if (warp == 0) {
      bv = -1.0;
      bk = ~0ull;
      // ≤ 128 candidates: all remote loads of a lane are issued before any is used
      constexpr int CMAX = 16 * CP_WARPS / 32;
      double cv[CMAX];
      unsigned long long ck[CMAX];
#pragma unroll
      for (int t = 0; t < CMAX; ++t) {
        const int e = lane + 32 * t;
        if (e < ncand) {
          const uint32_t a = cp_mapa(slot + 2 * (e % CP_WARPS), unsigned(e / CP_WARPS));
          cv[t] = cp_ld_dsmem(a);
          ck[t] = cp_ld_dsmem_u64(a + 8);
        } else {
          cv[t] = -1.0;
          ck[t] = ~0ull;
        }
      }
#pragma unroll
      for (int t = 0; t < CMAX; ++t) cp_better(bv, bk, cv[t], ck[t]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        cp_better(bv, bk, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bk, o));
      if (lane == 0) *reinterpret_cast<unsigned long long*>(sv + m) = bk;
      const long cc = long(bk & 0xffffffffull);
      if (k + 1 < p.steps) {
        const uint32_t base = cp_mapa(cols + size_t(cc / C) * ldc + k, unsigned(cc % C));
        double x[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const long i = lane + 32 * t;
          x[t] = (i < len) ? cp_ld_dsmem(base + uint32_t(i) * 8u) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const long i = lane + 32 * t;
          if (i < len) sv[i] = x[t];
        }
      }
    }
    __syncthreads();
    bk = *reinterpret_cast<const unsigned long long*>(sv + m);
    const int pp = int(bk >> 32);
    const long c = long(bk & 0xffffffffull);
    // positions of this warp's columns: c → k, the column at k → pp
    for (int l = warp + CP_WARPS * lane; l < nc; l += CP_WARPS * 32) {
      const long j = rank + long(l) * C;
      if (j < n) {
        if (j == c)
          lpos[l] = int(k);
        else if (lpos[l] == k)
          lpos[l] = pp;
      }
    }
    if (rank == 0 && warp == 0 && lane == 0) p.perm[k] = c;
    __syncwarp();
    if (k == p.steps - 1) break;
    double v[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const long i = lane + 32 * t;
      v[t] = (i < len) ? sv[i] : 0.0;
    }
    double ss = 0.0;
#pragma unroll
    for (int t = 0; t < T; ++t)
      if (t > 0 || lane > 0) ss = fma(v[t], v[t], ss);
    const double xn2 = warp_sum_f64(ss);
    const double alpha = __shfl_sync(0xffffffffu, v[0], 0);
    double tau = 0.0, sc = 0.0;
    if (len > 1 && xn2 > 0.0) {
      const double beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
      tau = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
#pragma unroll
    for (int t = 0; t < T; ++t) v[t] = (t == 0 && lane == 0) ? 1.0 : v[t] * sc;
    // ---- apply H to this warp's free columns, downdate their norms
    for (int l = warp; l < nc; l += CP_WARPS) {
      const long j = rank + long(l) * C;
      if (j >= n || lpos[l] <= k) continue;
      double* col = cols + size_t(l) * ldc + k;
      double dot = 0.0;
      if (tau != 0.0) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const long i = lane + 32 * t;
          if (i < len) dot = fma(v[t], col[i], dot);
        }
        dot = warp_sum_f64(dot);
      }
      const double tw = tau * dot;
      double tail = 0.0, head = 0.0;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const long i = lane + 32 * t;
        if (i < len) {
          double x = col[i];
          if (tau != 0.0) {
            x = fma(-tw, v[t], x);
            col[i] = x;
          }
          if (i == 0)
            head = x;
          else
            tail = fma(x, x, tail);
        }
      }
      head = __shfl_sync(0xffffffffu, head, 0);
      const double v1 = vn1[l];
      if (v1 != 0.0) {
        const double ra = fabs(head) / v1;
        const double tmp = fmax(0.0, 1.0 - __dmul_rn(ra, ra));
        const double r = v1 / vn2[l];
        const double tmp2 = __dmul_rn(tmp, __dmul_rn(r, r));
        if (tmp2 <= tol3z) {
          tail = warp_sum_f64(tail);
          if (lane == 0) {
            const double nv = (k + 1 < m) ? sqrt(tail) : 0.0;
            vn1[l] = nv;
            vn2[l] = nv;
          }
        } else if (lane == 0) {
          vn1[l] = v1 * sqrt(tmp);
        }
      }
      __syncwarp();
    }
  }
  // columns never pivoted (n > m) keep their final positions
  for (int l = warp + CP_WARPS * lane; l < nc; l += CP_WARPS * 32) {
    const long j = rank + long(l) * C;
    if (j < n && lpos[l] >= p.steps) p.perm[lpos[l]] = j;
  }
  cp_cluster_sync();  // no CTA leaves while another may still read its shared memory
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
