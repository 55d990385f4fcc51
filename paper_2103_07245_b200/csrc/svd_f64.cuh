// One-sided (Hestenes) Jacobi SVD of a small dense FP64 matrix — the k×k
// core of the sibling randomized paths: `svd_full`
// (/root/reference/pkg/src/pbpqlp/linalg.py:131-139, LAPACK dgesdd through
// np.linalg.svd) as used by r_svd (algorithms.py:263-292) and the
// pseudoinverse of cor_utv (`_transposed_pinv_apply`, algorithms.py:295-303).
//
// Problem.  M is n×L row-major (n ≤ L); its rows are the "vectors".  Plane
// rotations combine pairs of rows until all rows are mutually orthogonal:
//   G·M = diag(s)·Y,  G orthogonal (n×n), Y with orthonormal rows,
// so M = Gᵀ·diag(s)·Y is an SVD (left vectors = columns of Gᵀ = rows of G).
// With `accumulate`, each vector carries the matching row of G (initially
// the identity), so the rotations build G alongside (vector length V = L+n,
// dot products over the first L entries only).
//
// Rotation (Rutishauser, as in LAPACK dgesvj): for rows x, y with
// a = ‖x‖², b = ‖y‖², c = x·y, rotate when |c| > tol·√a·√b (tol = √L·u):
// ζ = (b − a)/(2c), t = sign(ζ)/(|ζ| + √(1+ζ²)), cs = 1/√(1+t²), sn = cs·t,
// x ← cs·x − sn·y, y ← sn·x + cs·y.  The sums a, b, c are recomputed from the
// current vectors at every visit, so every rotation is computed from data
// accurate relative to ‖x‖‖y‖ (one-sided Jacobi's relative accuracy).
//
// Order: the circle (round-robin) ordering on n_p = n rounded up to even
// positions: n_p − 1 rounds per sweep, n_p/2 disjoint pairs per round
// (pair p = positions p and n_p−1−p), every pair exactly once per sweep;
// between rounds the vectors at positions 1…n_p−1 advance one position, so
// after a sweep every vector is back at its start.  The sweep loop ends
// when a whole sweep rotated nothing (convergence), bounded by max_sweeps.
// Everything is in fixed order, so results are bitwise reproducible.
//
// Two kernels, one schedule:
//  * jacobi_reg_kernel — n_p/2 ≤ 128 pairs: one thread-block cluster (≤ 16
//    CTAs of 8 warps), warp p holds pair p's two vectors in registers for the
//    whole run.  After each round it hands its top vector to warp p+1 and its
//    bottom vector to warp p−1 through shared-memory mailboxes (DSMEM stores
//    across CTA boundaries), double-buffered by round parity and signalled
//    point to point with mbarriers (no cluster-wide barrier per round).
//  * jacobi_grid_kernel — any size: the vectors stay in a global (L2-resident)
//    array and the schedule moves the computation instead: in round r the
//    vector at position x ≥ 1 is vector 1 + ((x − 1 − r) mod (n_p − 1)).  A
//    cooperative grid over all SMs, one warp per pair, a grid barrier per
//    round.
// Then jacobi_norms_kernel / jacobi_output_kernel: σ_i = ‖row i‖ (fixed-order
// sums), a stable descending sort by σ (rank by counting), Y rows = x/σ,
// G rows permuted alike; jacobi_complete_kernel gives rows with σ = 0 an
// orthonormal completion (classical Gram-Schmidt twice against the other
// rows, from unit vectors), as LAPACK returns orthonormal vectors for a zero
// singular value.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace pbq {

namespace jcg = cooperative_groups;

constexpr int JAC_WARPS = 8;            // warps per CTA of the register kernel
constexpr int JAC_MAX_PAIRS_REG = 128;  // 16 CTAs × 8 warps
constexpr int JAC_MAX_VPL = 24;         // doubles per lane per vector (V ≤ 768)

struct JacArgs {
  int n, np, L, V;     // vectors, padded count (even), dot length, vector length
  int accumulate;      // V == L + n: vectors carry their row of G
  const double* X;     // n×L input (ldx)
  long ldx;
  double* Z;           // np×V final vectors (ldz = V rounded up to even)
  long ldz;
  int* status;         // [0] sweeps used, [1] 1 if not converged within max_sweeps
  int max_sweeps;
  double tol;
  unsigned long long* tphase;  // optional profiling (register kernel, middle warp): cycles in
                               // [rotate, send, wait], rounds
};

__device__ __forceinline__ void jac_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Initial value of element e (< V) of vector i: row i of X, then e_i.
__device__ __forceinline__ double jac_init(const JacArgs& p, int i, int e) {
  if (i >= p.n) return 0.0;
  if (e < p.L) return p.X[long(i) * p.ldx + e];
  return (e - p.L == i) ? 1.0 : 0.0;
}

// Rotation parameters for the pair with a = ‖x‖², b = ‖y‖², c = x·y:
// returns false (no rotation) unless aapq = |c|/(‖x‖‖y‖) > tol.  On the
// MUFU approximations + Newton steps (fast_rsqrt / fast_rcp, ~1 ulp): the
// IEEE chain sqrt → div → sqrt → div → sqrt was most of a round's latency.
// Norms near the ends of the exponent range (the .ftz approximations would
// flush) take the IEEE formulas.
__device__ __forceinline__ bool jac_params(double a, double b, double c, double tol, double& aapq, double& cs,
                                           double& sn) {
  aapq = 0.0;
  if (!(a > 0.0 && b > 0.0) || !(a < INFINITY && b < INFINITY)) return false;
  const bool fast = a > 1e-280 && b > 1e-280 && a < 1e280 && b < 1e280;
  aapq = fast ? fabs(c) * fast_rsqrt(a) * fast_rsqrt(b) : fabs(c) / (sqrt(a) * sqrt(b));
  if (!(aapq > tol)) return false;
  const double zeta = fast ? 0.5 * (b - a) * fast_rcp(c) : (b - a) / (2.0 * c);
  double t;
  if (fabs(zeta) > 1e100) {
    t = 0.5 / zeta;
  } else if (fast) {
    const double h = fma(zeta, zeta, 1.0);
    t = copysign(fast_rcp(fabs(zeta) + h * fast_rsqrt(h)), zeta);
  } else {
    t = copysign(1.0 / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0))), zeta);
  }
  cs = fast ? fast_rsqrt(fma(t, t, 1.0)) : 1.0 / sqrt(fma(t, t, 1.0));
  sn = cs * t;
  return true;
}

// The rotation of one pair (x, y: VPL doubles per lane, element lane + 32·k).
// Returns true when a rotation was applied; `aapq` receives the pair's
// relative off-diagonal |x·y|/(‖x‖‖y‖) before it and `sinj` |sin θ| of the
// rotation (0 when none) — dgesvj's convergence measures.
template <int VPL>
__device__ __forceinline__ bool jac_rotate(double (&x)[VPL], double (&y)[VPL], int L, double tol, double& aapq,
                                           double& sinj) {
  const int lane = threadIdx.x & 31;
  double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    if (lane + 32 * k < L) {
      a = fma(x[k], x[k], a);
      b = fma(y[k], y[k], b);
      c = fma(x[k], y[k], c);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  sinj = 0.0;
  double cs, sn;
  if (!jac_params(a, b, c, tol, aapq, cs, sn)) return false;
  sinj = fabs(sn);
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const double xv = x[k], yv = y[k];
    x[k] = fma(cs, xv, -sn * yv);
    y[k] = fma(sn, xv, cs * yv);
  }
  return true;
}

// Sweep-end test (LAPACK dgesvj): stop when no rotation was applied, or when
// the largest relative off-diagonal met in the sweep is below √n·tol and
// n·max|aapq|·max|sin θ| < tol (the remaining rotations change nothing at
// working precision).
__device__ __forceinline__ bool jac_converged(int rot, double mx_aapq, double mx_sin, int n, double tol) {
  return rot == 0 || (mx_aapq < sqrt(double(n)) * tol && double(n) * mx_aapq * mx_sin < tol);
}

// ---------------------------------------------------------------------------
// Register-resident kernel.  Launch: grid = C CTAs = one cluster of C,
// JAC_WARPS warps each, C·JAC_WARPS ≥ P = np/2; dynamic shared memory =
// jac_reg_smem(VPL).  Hand-over between neighbouring warps is point to
// point: each mailbox slot has an mbarrier and the receiver waits on it — no
// cluster-wide barrier per round.  A slot fed from the same CTA completes on
// 32 arrivals (every lane of the sender, release at CTA scope, after its
// stores).  A slot fed from a neighbouring CTA completes on transaction
// bytes: the sender pushes the vector with st.async (each store completes
// its bytes on the remote mbarrier) and never waits, and the receiver arms
// the phase with one arrive.expect_tx.  (The first version stored with
// st.shared::cluster and arrived with release at cluster scope: the release
// waited for the remote stores, 1421 of a round's ~3000 cycles at n = 256,
// `tools/svd_probe.py --phases`.)  Slot layout: lane ℓ's elements k, k+1 (k
// even) are the 16 bytes at 2·(32·(k/2) + ℓ), one v2 store each.  Slots are double-buffered by round
// parity; the data dependencies of the schedule make reuse safe (a sender
// writes a slot again only after receiving its neighbour's next vector,
// which the neighbour sends after consuming the slot's previous content).
__device__ __forceinline__ uint32_t jac_mapa(uint32_t addr, int cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void jac_st_remote(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void jac_arrive_remote(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// Asynchronous remote store of 16 bytes that completes `bytes` of the remote
// mbarrier's transaction count (no release fence, no arrival by the sender).
__device__ __forceinline__ void jac_st_async2(uint32_t addr, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(a), "d"(b), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void jac_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void jac_arrive_local(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void jac_wait(uint32_t bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "JW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra JW_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int VPL>
__global__ void __launch_bounds__(JAC_WARPS * 32, 1) jacobi_reg_kernel(JacArgs p) {
  extern __shared__ __align__(16) double jsm[];
  jcg::cluster_group cl = jcg::this_cluster();
  const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
  const int C = int(cl.num_blocks()), me = int(cl.block_rank());
  const int P = p.np / 2;
  const int w = me * JAC_WARPS + lw;  // this warp's pair index
  const bool active = w < P;
  const size_t slot_d = size_t(32) * VPL;
  const size_t box_d = size_t(2) * JAC_WARPS * 2 * slot_d;  // both parities
  uint64_t* bars = reinterpret_cast<uint64_t*>(jsm + box_d);  // [2 parity][JAC_WARPS][2 slots]
  double* sums = reinterpret_cast<double*>(bars + 4 * JAC_WARPS);  // [2 parity][16 CTAs][3] (on CTA 0)
  double* red = sums + 2 * 16 * 3;                                  // [JAC_WARPS][3]
  auto box_off = [&](int lq, int s, int par) { return ((size_t(par) * JAC_WARPS + lq) * 2 + s) * slot_d; };
  auto bar_of = [&](int lq, int s, int par) { return bars + (par * JAC_WARPS + lq) * 2 + s; };

  // barrier (par, lq, s): slot 0 (T_in) of warp q is fed by warp q−1 (warp 0 for
  // q = 1), slot 1 (B_in) by warp q+1 — from another CTA when lq is 0 / last
  auto remote_fed = [&](int q, int lq, int s) {
    return s == 0 ? (lq == 0 && q >= 2) : (lq == JAC_WARPS - 1 && q + 1 < P);
  };
  if (threadIdx.x < 4 * JAC_WARPS) {
    const int lq = (threadIdx.x >> 1) % JAC_WARPS, sl = threadIdx.x & 1;
    mbar_init(bars + threadIdx.x, remote_fed(me * JAC_WARPS + lq, lq, sl) ? 1 : 32);
  }
  mbar_fence_init();
  if (C > 1)
    jac_cluster_sync();  // every CTA's barriers exist before any remote arrival
  else
    __syncthreads();

  double x[VPL], y[VPL];
  const int ti = w, bi = p.np - 1 - w;  // vector indices at positions w and np−1−w
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int e = lane + 32 * k;
    x[k] = (active && e < p.V) ? jac_init(p, ti, e) : 0.0;
    y[k] = (active && e < p.V) ? jac_init(p, bi, e) : 0.0;
  }
  // store v into slot s of warp q (round parity par) and arrive on its barrier
  auto send = [&](const double (&v)[VPL], int q, int s, int par) {
    const int cta = q / JAC_WARPS, lq = q % JAC_WARPS;
    const size_t off = box_off(lq, s, par);
    if (cta == me) {
      double* d = jsm + off;
#pragma unroll
      for (int k = 0; k < VPL; k += 2)
        *reinterpret_cast<double2*>(d + 2 * (32 * (k >> 1) + lane)) = make_double2(v[k], v[k + 1]);
      jac_arrive_local(smem_u32(bar_of(lq, s, par)));
    } else {
      const uint32_t d = jac_mapa(smem_u32(jsm + off), cta);
      const uint32_t rb = jac_mapa(smem_u32(bar_of(lq, s, par)), cta);
#pragma unroll
      for (int k = 0; k < VPL; k += 2) jac_st_async2(d + 16u * (32 * (k >> 1) + lane), v[k], v[k + 1], rb);
    }
  };
  // wait for slot s of this warp (round parity par, barrier phase ph) and read it
  auto receive = [&](double (&v)[VPL], int s, int par, unsigned ph) {
    const uint32_t b = smem_u32(bar_of(lw, s, par));
    if (remote_fed(w, lw, s) && lane == 0) jac_arrive_expect_tx(b, uint32_t(32 * VPL * sizeof(double)));
    jac_wait(b, ph);
    const double* mb = jsm + box_off(lw, s, par);
#pragma unroll
    for (int k = 0; k < VPL; k += 2) {
      const double2 t = *reinterpret_cast<const double2*>(mb + 2 * (32 * (k >> 1) + lane));
      v[k] = t.x;
      v[k + 1] = t.y;
    }
  };
  long R = 0;  // rounds so far (all sweeps): slot parity R&1, barrier phase (R>>1)&1
  int sweeps = 0, converged = 0;
  for (int sw = 0; sw < p.max_sweeps && !converged; ++sw) {
    int rot = 0;
    double mx_aapq = 0.0, mx_sin = 0.0;
    for (int r = 0; r < p.np - 1; ++r, ++R) {
      const int par = int(R & 1);
      const unsigned phase = unsigned((R >> 1) & 1);
      const bool timed = p.tphase && w == P / 2;
      long long c0 = 0, c1 = 0, c2 = 0;
      if (timed) c0 = clock64();
      if (active) {
        double aapq, sinj;
        if (jac_rotate<VPL>(x, y, p.L, p.tol, aapq, sinj)) ++rot;
        mx_aapq = fmax(mx_aapq, aapq);
        mx_sin = fmax(mx_sin, sinj);
      }
      if (timed) c1 = clock64();
      if (active && P > 1) {
        // T' → warp w+1 (1 ≤ w ≤ P−2) or kept as B (w = P−1);
        // B' → warp w−1 (w ≥ 1) or warp 1's T slot (w = 0)
        if (w >= 1 && w <= P - 2) send(x, w + 1, 0, par);
        if (w >= 1)
          send(y, w - 1, 1, par);
        else
          send(y, 1, 0, par);
        if (timed) c2 = clock64();
        // B_in: own T' (w = P−1), else warp w+1's B';
        // T_in: own T' (w = 0), warp 0's B' (w = 1), warp w−1's T' (w ≥ 2)
        if (w == P - 1) {
#pragma unroll
          for (int k = 0; k < VPL; ++k) y[k] = x[k];
        } else {
          receive(y, 1, par, phase);
        }
        if (w >= 1) receive(x, 0, par, phase);
        if (timed && lane == 0) {
          const long long c3 = clock64();
          atomicAdd(p.tphase, (unsigned long long)(c1 - c0));
          atomicAdd(p.tphase + 1, (unsigned long long)(c2 - c1));
          atomicAdd(p.tphase + 2, (unsigned long long)(c3 - c2));
          atomicAdd(p.tphase + 3, 1ull);
        }
      }
    }
    // ---- sweep-end test: rotations, max relative off-diagonal and max |sin|
    // over the cluster (identical on every lane of a warp)
    if (lane == 0) {
      red[3 * lw] = double(rot);
      red[3 * lw + 1] = mx_aapq;
      red[3 * lw + 2] = mx_sin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int i = 0; i < JAC_WARPS; ++i) {
        s0 += red[3 * i];
        s1 = fmax(s1, red[3 * i + 1]);
        s2 = fmax(s2, red[3 * i + 2]);
      }
      double* dst = ((C > 1) ? cl.map_shared_rank(sums, 0) : sums) + ((sw & 1) * 16 + me) * 3;
      dst[0] = s0;
      dst[1] = s1;
      dst[2] = s2;
    }
    if (C > 1)
      jac_cluster_sync();
    else
      __syncthreads();
    double total = 0.0, gmx = 0.0, gsin = 0.0;
    const double* src = (C > 1) ? cl.map_shared_rank(sums, 0) : sums;
    for (int i = 0; i < C; ++i) {
      total += src[((sw & 1) * 16 + i) * 3];
      gmx = fmax(gmx, src[((sw & 1) * 16 + i) * 3 + 1]);
      gsin = fmax(gsin, src[((sw & 1) * 16 + i) * 3 + 2]);
    }
    sweeps = sw + 1;
    converged = jac_converged(int(total), gmx, gsin, p.n, p.tol);
  }
  if (active) {
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int e = lane + 32 * k;
      if (e < p.V) {
        p.Z[long(ti) * p.ldz + e] = x[k];
        p.Z[long(bi) * p.ldz + e] = y[k];
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.status[0] = sweeps;
    p.status[1] = converged ? 0 : 1;
  }
  if (C > 1) jac_cluster_sync();  // no CTA exits while its shared memory may still be read
}

// ---------------------------------------------------------------------------
// L2-resident kernel (any n, V).  Launch: cooperative, up to one CTA of
// JAC_GRID_WARPS warps per SM, warps take pairs round-robin (one pair each
// when 8·SMs ≥ P), a grid barrier per round; Z must already hold the initial
// vectors (jacobi_init_kernel).  Vectors of up to 32·VPL doubles are loaded
// whole into registers (all loads in flight at once); longer ones are
// streamed.  The sweep-end statistics are combined with integer atomics
// (counts, and max of non-negative doubles as bit patterns — order
// independent, so bitwise reproducible) in a slot per sweep parity:
// stat[par·4 + {0: rotations, 1: max aapq, 2: max |sin|}], zeroed before the
// launch; slot par^1 is cleared after every CTA has read it (one round
// barrier later).
constexpr int JAC_GRID_WARPS = 8;

template <int VPL>
__global__ void __launch_bounds__(JAC_GRID_WARPS * 32, 1)
    jacobi_grid_kernel(JacArgs p, unsigned int* bar, unsigned long long* stat) {
  const int lane = threadIdx.x & 31, lw = threadIdx.x >> 5;
  const int P = p.np / 2, TW = int(gridDim.x) * JAC_GRID_WARPS, w0 = int(blockIdx.x) * JAC_GRID_WARPS + lw;
  const int m1 = p.np - 1;
  unsigned int gen = 0;
  int sweeps = 0, converged = 0;
  for (int sw = 0; sw < p.max_sweeps && !converged; ++sw) {
    int rot = 0;
    double mx_aapq = 0.0, mx_sin = 0.0;
    for (int r = 0; r < m1; ++r) {
      for (int q = w0; q < P; q += TW) {
        const int xt = q, xb = p.np - 1 - q;  // positions
        const int it = xt == 0 ? 0 : 1 + ((xt - 1 - r) % m1 + m1) % m1;
        const int ib = 1 + ((xb - 1 - r) % m1 + m1) % m1;
        double* zt = p.Z + long(it) * p.ldz;
        double* zb = p.Z + long(ib) * p.ldz;
        if (p.V <= 32 * VPL) {
          double x[VPL], y[VPL];
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            const int e = lane + 32 * k;
            x[k] = e < p.V ? __ldcg(zt + e) : 0.0;
            y[k] = e < p.V ? __ldcg(zb + e) : 0.0;
          }
          double aapq, sinj;
          const bool did = jac_rotate<VPL>(x, y, p.L, p.tol, aapq, sinj);
          mx_aapq = fmax(mx_aapq, aapq);
          mx_sin = fmax(mx_sin, sinj);
          if (did) {
            ++rot;
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
              const int e = lane + 32 * k;
              if (e < p.V) {
                __stcg(zt + e, x[k]);
                __stcg(zb + e, y[k]);
              }
            }
          }
        } else {
          // long vectors: dots over L from global, then the rotation streamed
          double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll 4
          for (int e = lane; e < p.L; e += 32) {
            const double xv = __ldcg(zt + e), yv = __ldcg(zb + e);
            a = fma(xv, xv, a);
            b = fma(yv, yv, b);
            c = fma(xv, yv, c);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
          }
          double aapq, cs, sn;
          const bool rot_it = jac_params(a, b, c, p.tol, aapq, cs, sn);
          mx_aapq = fmax(mx_aapq, aapq);
          if (rot_it) {
            mx_sin = fmax(mx_sin, fabs(sn));
#pragma unroll 4
            for (int e = lane; e < p.V; e += 32) {
              const double xv = __ldcg(zt + e), yv = __ldcg(zb + e);
              __stcg(zt + e, fma(cs, xv, -sn * yv));
              __stcg(zb + e, fma(sn, xv, cs * yv));
            }
            ++rot;
          }
        }
      }
      grid_barrier(bar, gen);
    }
    // ---- sweep-end test (dgesvj): rotations, max relative off-diagonal, max |sin|
    const int par = sw & 1;
    if (lane == 0) {
      if (rot) atomicAdd(stat + 4 * par, (unsigned long long)rot);
      if (mx_aapq > 0.0) atomicMax(stat + 4 * par + 1, (unsigned long long)__double_as_longlong(mx_aapq));
      if (mx_sin > 0.0) atomicMax(stat + 4 * par + 2, (unsigned long long)__double_as_longlong(mx_sin));
    }
    if (blockIdx.x == 0 && threadIdx.x < 3) stat[4 * (par ^ 1) + threadIdx.x] = 0ull;  // read a round ago
    grid_barrier(bar, gen);
    const double total = double(__ldcg(stat + 4 * par));
    const double gmx = __longlong_as_double((long long)__ldcg(stat + 4 * par + 1));
    const double gsin = __longlong_as_double((long long)__ldcg(stat + 4 * par + 2));
    sweeps = sw + 1;
    converged = jac_converged(int(total), gmx, gsin, p.n, p.tol);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.status[0] = sweeps;
    p.status[1] = converged ? 0 : 1;
  }
}

__global__ void jacobi_init_kernel(JacArgs p) {
  const long total = long(p.np) * p.V;
  for (long t = long(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += long(gridDim.x) * blockDim.x) {
    const int i = int(t / p.V), e = int(t % p.V);
    p.Z[long(i) * p.ldz + e] = jac_init(p, i, e);
  }
}

// σ_i = ‖z_i[0:L)‖, fixed-order sums (one warp per vector).
__global__ void jacobi_norms_kernel(JacArgs p, double* sig) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= p.n) return;
  const double* z = p.Z + long(i) * p.ldz;
  double a = 0.0;
  for (int e = lane; e < p.L; e += 32) a = fma(z[e], z[e], a);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) sig[i] = sqrt(a);
}

// Sorted outputs: rank(i) = #{j: σ_j > σ_i or (σ_j == σ_i and j < i)};
// s[rank] = σ_i, Y[rank] = z_i[0:L)/σ_i (zero row when σ_i = 0, completed
// by jacobi_complete_kernel), G[rank] = z_i[L:L+n) when accumulating.
__global__ void jacobi_output_kernel(JacArgs p, const double* sig, double* s, double* Y, long ldy, double* G, long ldg,
                                     int* nzero) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= p.n) return;
  const double si = sig[i];
  int rank = 0;
  for (int j = lane; j < p.n; j += 32) {
    const double sj = sig[j];
    rank += (sj > si || (sj == si && j < i)) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
  const double* z = p.Z + long(i) * p.ldz;
  const double inv = si > 0.0 ? 1.0 / si : 0.0;
  if (lane == 0) {
    s[rank] = si;
    if (!(si > 0.0)) atomicAdd(nzero, 1);
  }
  if (Y)
    for (int e = lane; e < p.L; e += 32) Y[long(rank) * ldy + e] = z[e] * inv;
  if (G && p.accumulate)
    for (int e = lane; e < p.n; e += 32) G[long(rank) * ldg + e] = z[p.L + e];
}

// Rows rank ≥ n − nzero of Y (σ = 0) get an orthonormal completion: for each,
// unit vectors e_t (t = 0, 1, …) are orthogonalised twice (CGS2) against all
// other rows until the remainder keeps more than half its norm.  One CTA,
// sequential over the (rare) zero rows.
__global__ void __launch_bounds__(256) jacobi_complete_kernel(int n, int L, double* Y, long ldy, const int* nzero,
                                                              double* work) {
  __shared__ double red[8];
  __shared__ double coef_s;
  const int nz = *nzero;
  if (nz == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  double* v = work;  // L doubles
  auto block_sum = [&](double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if (lane == 0) red[wp] = x;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += red[i];
    return s;
  };
  for (int row = n - nz; row < n; ++row) {
    for (int t = 0; t < L; ++t) {
      for (int e = tid; e < L; e += 256) v[e] = (e == t) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int j = 0; j < row; ++j) {  // rows < row are orthonormal (earlier ranks)
          double d = 0.0;
          for (int e = tid; e < L; e += 256) d = fma(Y[long(j) * ldy + e], v[e], d);
          d = block_sum(d);
          if (tid == 0) coef_s = d;
          __syncthreads();
          const double cf = coef_s;
          for (int e = tid; e < L; e += 256) v[e] = fma(-cf, Y[long(j) * ldy + e], v[e]);
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int e = tid; e < L; e += 256) nn = fma(v[e], v[e], nn);
      nn = block_sum(nn);
      if (nn > 0.25) {
        const double inv = 1.0 / sqrt(nn);
        for (int e = tid; e < L; e += 256) Y[long(row) * ldy + e] = v[e] * inv;
        __syncthreads();
        break;
      }
      __syncthreads();
    }
  }
}

}  // namespace pbq
