// EXPERIMENT, not built into libpbq: measured slower than the grid kernel.
// Pass 1 of the Cholesky-QR factorisation (R₁ = chol(G₁), X₁ = R₁⁻¹, κ₁
// guard; reference `householder_qr` / `orth` via cholqr_f64.cuh) on ONE
// thread-block cluster with the whole n×n problem in distributed shared
// memory, for n ≤ 32·16.
//
// The grid kernel (`cholqr_factor_kernel`) keeps the blocks in L2 and ends
// every block step with a grid barrier over up to 148 CTAs; at n = 256 its 8
// steps took ≈ 83 µs (profiles/r01d_launch_shares.md), a chain of L2 round
// trips and barriers.  Here CTA j of an nb-CTA cluster (nb = n/32) owns
//   * block column j of G, factored in place into R (blocks i ≤ j), and
//   * block row j of X = R⁻¹ (blocks k ≥ j),
// so every CTA holds nb + 1 blocks of 32×32 and the cross-CTA traffic is
// DSMEM (ld.shared::cluster) with cluster barriers between phases.  Block
// step k:
//   A  CTA k factors its diagonal block: R_kk and R_kk⁻¹ (one warp,
//      cq_chol_inv32_warp);                                   — barrier —
//   B  CTA j > k: R_kj = R_kk⁻ᵀ·G_kj in place;
//      CTA i < k: X_ik = −(Σ_{l=i}^{k−1} X_il·R_lk)·R_kk⁻¹  (row i of X lags
//      the factorisation by one step and uses CTAs that have no Schur work
//      left);                                                  — barrier —
//   C  CTA j > k: G_ij −= R_kiᵀ·R_kj for k < i ≤ j (R_ki from CTA i).
// CTA k+1's only phase-C product is its own diagonal block, so it starts
// factoring block k+1 while the other CTAs finish their Schur updates.
// The κ₁ guard and the fallback protocol are those of the grid kernel.
#pragma once
#include "../../paper_2103_07245_b200/csrc/cholqr_f64.cuh"

namespace pbq {

constexpr int CQC_MAX_NB = 16;

__device__ __forceinline__ unsigned cqc_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// cluster barrier; shared-memory release/acquire (all cross-CTA data is DSMEM)
__device__ __forceinline__ void cqc_sync() {
  asm volatile("fence.release.sync_restrict::shared::cta.cluster;\n" ::: "memory");
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cqc_mapa(const void* p, unsigned rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ double2 cqc_ld2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ double cqc_ld(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int cqc_ld_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Copy `cnt` 32×32 blocks (ld CQ_LD) from CTA `rank` — source block q at
// local-layout pointer src[q] — into dst + q·CQ_BLK.  Every load is issued
// before the first store, so one DSMEM round trip covers the batch.
template <int MAXB>
__device__ __forceinline__ void cqc_fetch(double* dst, const double* const* src, const unsigned* rank, int cnt) {
  const int r = threadIdx.x >> 3, c = (threadIdx.x & 7) * 4;
  double2 v[MAXB][2];
#pragma unroll
  for (int q = 0; q < MAXB; ++q) {
    if (q < cnt) {
      const uint32_t a = cqc_mapa(src[q] + r * CQ_LD + c, rank[q]);
      v[q][0] = cqc_ld2(a);
      v[q][1] = cqc_ld2(a + 16);
    }
  }
#pragma unroll
  for (int q = 0; q < MAXB; ++q) {
    if (q < cnt) {
      double* d = dst + q * CQ_BLK + r * CQ_LD + c;
      *reinterpret_cast<double2*>(d) = v[q][0];
      *reinterpret_cast<double2*>(d + 2) = v[q][1];
    }
  }
}

constexpr int CQC_STAGE = 6;  // remote blocks staged per batch
constexpr size_t cqc_smem_bytes(int nb) { return size_t(nb + 2 + CQC_STAGE) * CQ_BLK * sizeof(double); }

__global__ void __launch_bounds__(CQ_THREADS, 1) cholqr_cluster_factor_kernel(CqArgs p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_fail;
  __shared__ __align__(16) double s_rowbuf[64];
  __shared__ double s_rsum[32];                   // |R| column sums of block column me
  __shared__ double s_xsum[CQC_MAX_NB][32];       // |X| column sums of X_{me,k}
  if (p.fallback && __ldcg(p.fallback) != 0) return;  // uniform across the cluster
  if (p.route && __ldcg(p.route) == 0) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.nb;
  const long np = p.np;
  const int me = int(cqc_rank());
  // layout (identical offsets in every CTA): col[i] = block (i, me) of G/R for
  // i ≤ me; xr(k) = block (me, k) of X for k ≥ me; then R_kk⁻¹, a product
  // scratch block and the staging ring for remote blocks
  auto col = [&](int i) { return sm + i * CQ_BLK; };
  auto xrow = [&](int /*rank*/, int k) { return sm + (k + 1) * CQ_BLK; };  // slots me+1..nb in CTA me
  double* sKI = sm + (nb + 1) * CQ_BLK;
  double* stage = sKI + CQ_BLK;  // CQC_STAGE blocks; stage[0] doubles as product scratch
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

  double shift = 0.0;
  if (p.shift_mode) {  // s = 11(mn + n(n+1))·u·trace(G), the same fixed order in every CTA
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
  // block column me of G → shared memory
  for (int i = 0; i <= me; ++i) cq_load_async(col(i), p.G, np, i, me);
  cp_async_commit();
  cp_async_wait<0>();
  if (tid == 0) s_fail = 0;
  __syncthreads();
  if (shift != 0.0 && tid < 32 && me * 32 + tid < p.n) col(me)[tid * CQ_LD + tid] += shift;
  cqc_sync();  // every CTA's shared memory is initialised before any remote read

  // optional profiling (pbq_debug_qr_hooks): per CTA, time in phase A (the
  // diagonal factorisation), waiting at barrier 1, phase B, barrier 2, phase C
  unsigned long long t_mark = 0;
  auto mark = [&](int slot) {
    if (p.phase_ns && tid == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (slot >= 0) p.phase_ns[8 + me * 5 + slot] += now - t_mark;
      t_mark = now;
    }
  };
  mark(-1);
  for (int k = 0; k < nb; ++k) {
    // ---- A: CTA k factors G_kk (final after its own phase C of step k−1)
    if (me == k && warp == 0) {
      const bool ok = cq_chol_inv32_warp(col(k), xrow(k, k), s_rowbuf);
      if (tid == 0) s_fail = ok ? 0 : 1;
    }
    mark(0);
    cqc_sync();
    mark(1);
    if (cqc_ld_s32(cqc_mapa(&s_fail, unsigned(k)))) {  // same value in every CTA: all leave together
      if (me == 0 && tid == 0) fail_all();
      cqc_sync();  // nobody leaves while another CTA may still read its flag
      return;
    }
    // ---- B
    if (me != k) {
      const double* src = xrow(k, k);
      const unsigned rk = unsigned(k);
      cqc_fetch<1>(sKI, &src, &rk, 1);  // R_kk⁻¹
    }
    if (me > k) {
      __syncthreads();
      double c[2][2];
      cq_zero(c);
      cq_mma<true, false>(c, sKI, col(k));  // R_kj = R_kk⁻ᵀ·G_kj
      __syncthreads();
      cq_store_acc(col(k), c, 1.0);
    } else if (me < k) {
      double c[2][2];
      cq_zero(c);
      for (int l0 = me; l0 < k; l0 += CQC_STAGE) {  // Σ_l X_{me,l}·R_{l,k}, R_{l,k} from CTA k
        const int cnt = min(CQC_STAGE, k - l0);
        const double* src[CQC_STAGE];
        unsigned rk[CQC_STAGE];
#pragma unroll
        for (int q = 0; q < CQC_STAGE; ++q) {
          src[q] = col(l0 + q);
          rk[q] = unsigned(k);
        }
        __syncthreads();  // the previous batch's readers are done with the ring
        cqc_fetch<CQC_STAGE>(stage, src, rk, cnt);
        __syncthreads();
        for (int q = 0; q < cnt; ++q) cq_mma<false, false>(c, xrow(me, l0 + q), stage + q * CQ_BLK);
      }
      __syncthreads();
      cq_store_acc(stage, c, 1.0);
      __syncthreads();
      cq_zero(c);
      cq_mma<false, false>(c, stage, sKI);
      cq_store_acc(xrow(me, k), c, -1.0);
    }
    mark(2);
    cqc_sync();
    mark(3);
    // ---- C: G_{i,me} −= R_kiᵀ·R_{k,me}, own diagonal block first
    if (me > k) {
      {
        double c[2][2];
        cq_zero(c);
        cq_mma<true, false>(c, col(k), col(k));
        const int r = cq_row();
        double* g = col(me);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          g[r * CQ_LD + cq_col(h)] -= c[h][0];
          g[r * CQ_LD + cq_col(h) + 1] -= c[h][1];
        }
      }
      for (int i0 = k + 1; i0 < me; i0 += CQC_STAGE) {
        const int cnt = min(CQC_STAGE, me - i0);
        const double* src[CQC_STAGE];
        unsigned rk[CQC_STAGE];
#pragma unroll
        for (int q = 0; q < CQC_STAGE; ++q) {
          src[q] = col(k);  // block (k, i) lives at slot k of CTA i
          rk[q] = unsigned(i0 + q);
        }
        __syncthreads();
        cqc_fetch<CQC_STAGE>(stage, src, rk, cnt);
        __syncthreads();
        for (int q = 0; q < cnt; ++q) {
          double c[2][2];
          cq_zero(c);
          cq_mma<true, false>(c, stage + q * CQ_BLK, col(k));
          const int r = cq_row();
          double* g = col(i0 + q);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            g[r * CQ_LD + cq_col(h)] -= c[h][0];
            g[r * CQ_LD + cq_col(h) + 1] -= c[h][1];
          }
        }
      }
    }
    __syncthreads();
    mark(4);
  }

  // ---- results: R column me, X row me, |·| column sums → κ₁ guard -------
  for (int i = 0; i <= me; ++i) cq_store(p.R, np, i, me, col(i));
  for (int k = me; k < nb; ++k) cq_store(p.X, np, me, k, xrow(me, k));
  if (tid < 32) {
    double s = 0.0;
    for (int i = 0; i <= me; ++i)
      for (int r = 0; r < 32; ++r) s += fabs(col(i)[r * CQ_LD + tid]);
    s_rsum[tid] = s;
    for (int k = me; k < nb; ++k) {
      double x = 0.0;
      for (int r = 0; r < 32; ++r) x += fabs(xrow(me, k)[r * CQ_LD + tid]);
      s_xsum[k][tid] = x;
    }
  }
  cqc_sync();
  if (me == 0 && warp == 0) {
    const int lane = tid & 31;
    double mr = 0.0, mx = 0.0;
    bool bad = false;
    for (int j = 0; j < nb; ++j) {
      if (long(j) * 32 + lane >= p.n) continue;
      const double sr = cqc_ld(cqc_mapa(&s_rsum[lane], unsigned(j)));
      double sx = 0.0;
      for (int i = 0; i <= j; ++i) sx += cqc_ld(cqc_mapa(&s_xsum[j][lane], unsigned(i)));  // fixed order
      mr = fmax(mr, sr);  // fmax drops NaN: finiteness is checked separately
      mx = fmax(mx, sx);
      bad |= !(sr < INFINITY) || !(sx < INFINITY);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0 && p.pass == 1 && !p.shift_mode && (bad || !(mr * mx <= p.kappa_max))) fail_all();
  }
  cqc_sync();  // no CTA leaves while CTA 0 may still read its sums
}

}  // namespace pbq
