// FP64 DMMA GEMM for the two PbP-QLP contractions:
//
//   TRANS_A = true  : C[M×N] = alpha · Aᵀ·B + beta·C,  A stored K×M row-major
//                     (C = AᵀX, reference `_PassCounter.apply_t`, algorithms.py:182-184)
//   TRANS_A = false : C[M×N] = alpha · A·B  + beta·C,  A stored M×K row-major
//                     (D = A·X, reference `_PassCounter.apply`, algorithms.py:178-180)
//
// B is K×N row-major in both cases.  All operands are FP64 and the products
// run on the sm_100a FP64 tensor instruction DMMA.8x8x4 (tcgen05 has no f64
// kind).  Tiles are staged by cp.async into a STAGES-deep shared-memory ring
// (BK = 32 so one barrier covers 8 MMA k-steps); every thread's cp.async
// sources are a single pointer advanced by a constant per k-block, so the
// mainloop carries no address arithmetic.  Fragments for k-step s+1 are
// loaded while the MMAs of k-step s issue.  The grid is persistent (one CTA
// per SM) and walks a deterministic stream-K schedule: the linearised
// (tile, k-block) iteration space is cut into `grid` equal ranges; a tile
// whose k-range is split across CTAs is finished by the CTA that owns its
// k=0 block, which adds the other CTAs' partial tiles in increasing k order.
// The reduction order depends only on (M, N, K, grid), so results are bitwise
// reproducible run to run on the same GPU model (test_algorithms.py:53-60).
// CHECK additionally ORs an Inf/NaN flag over every element of A (the
// `check_matrix` isfinite scan, validation.py:47), fused into the first pass.
#pragma once
#include "common.cuh"

namespace pbq {

struct GemmArgs {
  long M, N, K;
  const double* A;
  long lda;
  const double* B;
  long ldb;
  double* C;
  long ldc;
  double alpha, beta;
  int tiles_m, tiles_n, k_iters;
  long total_iters;
  double* partials;  // grid × (BM·BN) doubles
  int* flags;        // grid ints, zero at launch; each consumed flag is reset by its reader
  int* nonfinite;    // CHECK only: OR-flag set if any element of A is Inf/NaN
  // SPLIT mode (Gram matrices of the Cholesky-QR path): unit u = (tile u/split,
  // k-slice u%split) writes its partial tile to partials[u] (plain row-major
  // BM×BN); `sym` enumerates only tiles with tm <= tn (requires BM == BN or a
  // single tile).  A separate kernel sums the slices in fixed order.
  int split, sym, units;
  // sym with split_diag > 0: diagonal tiles get split_diag slices and the
  // others `split` (the TMA kernel skips a diagonal tile's strictly-lower
  // warp tiles, spread over the schedulers); split_tiles tiles in all, the
  // slices of tile t occupy units [Σ_{t'<t} S_t', …)
  int split_diag, split_tiles;
  const int* skip;   // when non-null and *skip != 0 the launch is a no-op
  const int* run_if; // when non-null and *run_if == 0 the launch is a no-op
  // tri_b: B is upper triangular (K == N), so output column tile tn only
  // needs k < (tn+1)·BN — the stream-K space then has row_iters =
  // Σ_tn k-blocks(tn) iterations per row of tiles (total_iters = tiles_m·row_iters)
  int tri_b, row_iters;
  // group > 1 (plain stream-K only): CTAs c = g·group + r form a group that
  // walks the same (row tile, k-block) range, CTA r taking column tile
  // tnp·group + r, so the group streams each A block from HBM once and its
  // other members hit L2 (total_iters counts group iterations)
  int group;
  // RESID epilogue (‖A − op(A)·B‖_F of the reconstruction): instead of storing
  // C, each finished tile subtracts from ref[r·ldref + c] and accumulates the
  // squared residual and squared ref; per-CTA sums go to sums[2·cta + {0,1}]
  const double* ref;
  long ldref;
  double* sums;
  // SPLIT with red_counter (zeroed, cooperative launch): the slice sum runs in
  // the same launch after a grid barrier — G (np×np, ld np) = Σ_s partials in
  // slice order, rows/cols in [n, np) the identity padding, optional copy and
  // max|G − I| (bits, atomicMax) for the pass-2 series test
  unsigned int* red_counter;
  double* red_G;
  double* red_Gcopy;
  unsigned long long* red_emax;
  long red_n, red_np;
  // scatter epilogue (TMA kernel, plain mode; exchange_f64.cuh): instead of C,
  // tile rows [m0, m0+BM) go to xs_land[o] + (xs_rank·xs_S + m0 − o·xs_S)·xs_ldl,
  // o = m0 / xs_S (the slice owner, peer memory), then xs_cnt[o] += 1 (release, sys)
  double* const* xs_land;
  unsigned int* const* xs_cnt;
  long xs_S, xs_ldl;
  int xs_rank;
};

// SPLIT mode: tile of unit u, its slice index, its slice count and the unit
// of its first slice (the tiles' slice ranges are contiguous, in tile order)
__device__ __forceinline__ void split_unit(const GemmArgs& p, int u, int& tsel, int& sl, int& S, int& first) {
  if (!(p.sym && p.split_diag > 0)) {
    tsel = u / p.split;
    sl = u % p.split;
    S = p.split;
    first = tsel * p.split;
    return;
  }
  int acc = 0;
  for (int t = 0;; ++t) {
    int tm, tn;
    upper_tile(t, p.tiles_n, tm, tn);
    const int st = (tm == tn) ? p.split_diag : p.split;
    if (u < acc + st || t + 1 >= p.split_tiles) {
      tsel = t;
      sl = u - acc;
      S = st;
      first = acc;
      return;
    }
    acc += st;
  }
}

// first unit and slice count of tile tsel (the inverse of split_unit)
__device__ __forceinline__ void split_tile(const GemmArgs& p, int tsel, int& first, int& S) {
  S = p.split;
  first = tsel * p.split;
  if (!(p.sym && p.split_diag > 0)) return;
  first = 0;
  for (int t = 0; t < tsel; ++t) {
    int tm, tn;
    upper_tile(t, p.tiles_n, tm, tn);
    first += (tm == tn) ? p.split_diag : p.split;
  }
  int tm, tn;
  upper_tile(tsel, p.tiles_n, tm, tn);
  S = (tm == tn) ? p.split_diag : p.split;
}


template <bool TRANS_A, int BM, int BN, int BK, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int WARPS_M = BM / WM;
  static constexpr int WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int MT = WM / 8;
  static constexpr int NT = WN / 8;
  // Row strides (in doubles) are ≡ 4 (mod 16) so that the 8×4 fragment loads
  // of a warp hit 16 distinct 8-byte bank pairs per half-warp.
  static constexpr int SA_LD = TRANS_A ? (BM + 4) : (BK + 4);
  static constexpr int SA_ROWS = TRANS_A ? BK : BM;
  static constexpr int SB_LD = BN + 4;
  static constexpr int SA_ELEMS = SA_ROWS * SA_LD;
  static constexpr int SB_ELEMS = BK * SB_LD;
  static constexpr int STAGE_ELEMS = SA_ELEMS + SB_ELEMS;
  static constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
  // cp.async chunk geometry (16-byte chunks = 2 doubles)
  static constexpr int A_ROWW = TRANS_A ? BM / 2 : BK / 2;  // chunks per staged row of A
  static constexpr int A_CHUNKS = SA_ROWS * A_ROWW;
  static constexpr int A_PER_THREAD = A_CHUNKS / THREADS;
  static constexpr int A_ROW_STEP = THREADS / A_ROWW;        // staged rows between a thread's chunks
  static constexpr int B_ROWW = BN / 2;
  static constexpr int B_PER_THREAD = BK * B_ROWW / THREADS;
  static constexpr int B_ROW_STEP = THREADS / B_ROWW;
  static_assert(BM % WM == 0 && BN % WN == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");
  static_assert(BK % 4 == 0, "BK multiple of 4");
  static_assert(SA_LD % 16 == 4 && SB_LD % 16 == 4, "bank-conflict-free strides");
  static_assert(A_CHUNKS % THREADS == 0 && THREADS % A_ROWW == 0, "A loader geometry");
  static_assert((BK * B_ROWW) % THREADS == 0 && THREADS % B_ROWW == 0, "B loader geometry");
};

// ---------------------------------------------------------------------------
// The kernel.  The k-block ring is synchronised by mbarriers instead of a CTA
// barrier per k-block (the first version's scheme, 14.5 → 13.8 ms per config-3
// step when replaced):
//   full[s]  — expected THREADS arrivals; each thread arrives through
//              cp.async.mbarrier.arrive.noinc once its copies for the stage
//              have landed;
//   empty[s] — expected THREADS arrivals; each thread arrives after its warp
//              has read the stage.
// A thread refills stage s (for k-block f + STAGES − 1) only after all warps
// released it (k-block f − 1), so warps drift up to one stage apart instead of
// re-aligning at every k-block, and the ring runs on across the CTA's tiles
// (the next tile's first k-blocks load during the current tile's last ones).
// ---------------------------------------------------------------------------
template <bool TRANS_A, int BM, int BN, int BK, int WM, int WN, int STAGES, bool CHECK, bool SPLIT = false,
          bool RESID = false>
__global__ void __launch_bounds__(GemmCfg<TRANS_A, BM, BN, BK, WM, WN, STAGES>::THREADS, 1)
    gemm_f64_ring(GemmArgs p) {
  using Cfg = GemmCfg<TRANS_A, BM, BN, BK, WM, WN, STAGES>;
  constexpr int THREADS = Cfg::THREADS;
  constexpr int MT = Cfg::MT, NT = Cfg::NT;
  constexpr int KSTEPS = BK / 4;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  pdl_wait();
  pdl_trigger();
  if (p.skip && __ldcg(p.skip) != 0) return;
  if (p.run_if && __ldcg(p.run_if) == 0) return;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp / Cfg::WARPS_N) * WM;
  const int wn0 = (warp % Cfg::WARPS_N) * WN;
  const int G = gridDim.x;
  const int GS = (SPLIT || p.group < 1) ? 1 : p.group;  // group size
  const int NG = G / GS, gi = blockIdx.x / GS, gr = blockIdx.x % GS;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], THREADS);
      mbar_init(&empty_bar[s], THREADS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int a_row = tid / Cfg::A_ROWW, a_col = (tid % Cfg::A_ROWW) * 2;
  const int b_row = tid / Cfg::B_ROWW, b_col = (tid % Cfg::B_ROWW) * 2;
  const long a_kstep = TRANS_A ? long(BK) * p.lda : long(BK);
  const long b_kstep = long(BK) * p.ldb;
  const long a_rstep = long(Cfg::A_ROW_STEP) * p.lda;
  const long b_rstep = long(Cfg::B_ROW_STEP) * p.ldb;

  // ---- work segments (tile, [kb, ke)) of this CTA, in order ---------------
  struct Seg {
    int tile, tm, tn, kb, ke, tile_k;
    long tile_it0;
  };
  struct Cursor {
    long it, it_end;
    int unit;
  };
  auto first_cursor = [&]() {
    Cursor c;
    c.it = long(gi) * p.total_iters / NG;
    c.it_end = long(gi + 1) * p.total_iters / NG;
    c.unit = blockIdx.x;
    return c;
  };
  auto next_seg = [&](Cursor& c, Seg& s) -> bool {
    s.tile_k = p.k_iters;
    s.tile_it0 = 0;
    if (SPLIT) {
      if (c.unit >= p.units) return false;
      int tsel, sl, S, first;
      split_unit(p, c.unit, tsel, sl, S, first);
      if (p.sym) {
        upper_tile(tsel, p.tiles_n, s.tm, s.tn);
      } else {
        s.tm = tsel / p.tiles_n;
        s.tn = tsel % p.tiles_n;
      }
      s.tile = tsel;
      s.kb = int(long(sl) * p.k_iters / S);
      s.ke = int(long(sl + 1) * p.k_iters / S);
      c.unit += G;
      return true;
    }
    if (c.it >= c.it_end) return false;
    if (p.tri_b) {
      s.tm = int(c.it / p.row_iters);
      int rem = int(c.it % p.row_iters);
      s.tn = 0;
      for (;;) {
        const int kt = int(lmin(p.k_iters, long(s.tn + 1) * BN / BK));
        if (rem < kt) {
          s.tile_k = kt;
          break;
        }
        rem -= kt;
        ++s.tn;
      }
      s.kb = rem;
      s.tile = s.tm * p.tiles_n + s.tn;
    } else {
      const int tg = int(c.it / p.k_iters), tpg = p.tiles_n / GS;
      s.kb = int(c.it % p.k_iters);
      s.tm = tg / tpg;
      s.tn = (tg % tpg) * GS + gr;
      s.tile = s.tm * p.tiles_n + s.tn;
    }
    s.tile_it0 = c.it - s.kb;
    s.ke = int(lmin(s.tile_k, s.kb + (c.it_end - c.it)));
    c.it += s.ke - s.kb;
    return true;
  };

  // ---- producer: loads k-blocks in flat order into the ring ---------------
  Cursor pcur = first_cursor();
  Seg pseg;
  bool p_live = next_seg(pcur, pseg);
  int pk = p_live ? pseg.kb : 0;
  const double* a_src = nullptr;
  const double* b_src = nullptr;
  int a_bytes = 0, b_bytes = 0;
  auto p_tile_setup = [&]() {
    const long m0 = long(pseg.tm) * BM, n0 = long(pseg.tn) * BN;
    if (TRANS_A) {
      const long gm = m0 + a_col;
      a_bytes = gm < p.M ? int(lmin(2, p.M - gm)) * 8 : 0;
      a_src = p.A + (long(pseg.kb) * BK + a_row) * p.lda + (a_bytes ? gm : 0);
    } else {
      a_bytes = 16;
      a_src = p.A + (m0 + a_row) * p.lda + long(pseg.kb) * BK + a_col;
    }
    const long gn = n0 + b_col;
    b_bytes = gn < p.N ? int(lmin(2, p.N - gn)) * 8 : 0;
    b_src = p.B + (long(pseg.kb) * BK + b_row) * p.ldb + (b_bytes ? gn : 0);
  };
  if (p_live) p_tile_setup();
  long pflat = 0;  // flat index of the next k-block to load
  auto produce = [&]() {
    if (!p_live) return;
    const int stage = int(pflat % STAGES);
    if (pflat >= STAGES) mbar_wait(&empty_bar[stage], unsigned((pflat / STAGES - 1) & 1));
    double* sA = smem + stage * Cfg::STAGE_ELEMS;
    double* sB = sA + Cfg::SA_ELEMS;
    const long k0 = long(pk) * BK;
    const bool kfull = k0 + BK <= p.K;
    const long m0 = long(pseg.tm) * BM;
#pragma unroll
    for (int i = 0; i < Cfg::A_PER_THREAD; ++i) {
      const int r = a_row + i * Cfg::A_ROW_STEP;
      int bytes;
      if (TRANS_A) {
        bytes = (kfull || k0 + r < p.K) ? a_bytes : 0;
      } else {
        const long gk = k0 + a_col;
        bytes = (m0 + r < p.M) ? (kfull ? 16 : (gk < p.K ? int(lmin(2, p.K - gk)) * 8 : 0)) : 0;
      }
      cp_async16(sA + r * Cfg::SA_LD + a_col, bytes ? a_src + i * a_rstep : p.A, bytes);
    }
#pragma unroll
    for (int i = 0; i < Cfg::B_PER_THREAD; ++i) {
      const int r = b_row + i * Cfg::B_ROW_STEP;
      const int bytes = (kfull || k0 + r < p.K) ? b_bytes : 0;
      cp_async16(sB + r * Cfg::SB_LD + b_col, bytes ? b_src + i * b_rstep : p.B, bytes);
    }
    cp_async_mbar_arrive(&full_bar[stage]);
    a_src += a_kstep;
    b_src += b_kstep;
    ++pflat;
    if (++pk == pseg.ke) {
      p_live = next_seg(pcur, pseg);
      if (p_live) {
        pk = pseg.kb;
        p_tile_setup();
      }
    }
  };
#pragma unroll 1
  for (int s = 0; s < STAGES - 1; ++s) produce();

  // ---- consumer -----------------------------------------------------------
  Cursor ccur = first_cursor();
  Seg seg;
  long cflat = 0;
  bool saw_nonfinite = false;
  double res2 = 0.0, ref2 = 0.0;  // RESID accumulators (fixed order per thread)
  while (next_seg(ccur, seg)) {
    const long m0 = long(seg.tm) * BM, n0 = long(seg.tn) * BN;
    const bool check = CHECK && (seg.tn == 0);
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll 1
    for (int kbk = seg.kb; kbk < seg.ke; ++kbk) {
      const int stage = int(cflat % STAGES);
      mbar_wait(&full_bar[stage], unsigned((cflat / STAGES) & 1));
      const double* sA = smem + stage * Cfg::STAGE_ELEMS;
      const double* sB = sA + Cfg::SA_ELEMS;
      if (CHECK && check) {
#pragma unroll
        for (int i = 0; i < Cfg::A_PER_THREAD; ++i) {
          const int r = a_row + i * Cfg::A_ROW_STEP;
          const double2 v = *reinterpret_cast<const double2*>(sA + r * Cfg::SA_LD + a_col);
          saw_nonfinite |= nonfinite_bits(v.x) | nonfinite_bits(v.y);
        }
      }
      double fa[2][MT], fb[2][NT];
      auto load_frags = [&](int kk, double (&a)[MT], double (&b)[NT]) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          if (TRANS_A)
            a[mt] = sA[(kk * 4 + t) * Cfg::SA_LD + wm0 + mt * 8 + g];
          else
            a[mt] = sA[(wm0 + mt * 8 + g) * Cfg::SA_LD + kk * 4 + t];
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = sB[(kk * 4 + t) * Cfg::SB_LD + wn0 + nt * 8 + g];
      };
      load_frags(0, fa[0], fb[0]);
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        const int cur = kk & 1;
        if (kk + 1 < KSTEPS) load_frags(kk + 1, fa[cur ^ 1], fb[cur ^ 1]);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], fa[cur][mt], fb[cur][nt]);
      }
      mbar_arrive(&empty_bar[stage]);
      ++cflat;
      produce();  // k-block cflat + STAGES − 2 into the stage released one step ago
    }

    // ---- epilogue: split partial / stream-K fix-up / store ---------------
    if (SPLIT) {
      double* slot = p.partials + size_t(ccur.unit - G) * (BM * BN);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          __stcg(reinterpret_cast<double2*>(slot + (wm0 + mt * 8 + g) * BN + wn0 + nt * 8 + 2 * t),
                 make_double2(acc[mt][nt][0], acc[mt][nt][1]));
      continue;
    }
    const bool full = (seg.kb == 0 && seg.ke == seg.tile_k);
    if (!full && seg.kb != 0) {
      double* slot = p.partials + size_t(blockIdx.x) * (BM * BN);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            __stcg(slot + size_t(((warp * MT + mt) * NT + nt) * 2 + e) * 32 + lane, acc[mt][nt][e]);
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(p.flags + blockIdx.x, 1);
      continue;
    }
    if (!full) {
      const long tile_end = seg.tile_it0 + seg.tile_k;
      for (int cg = gi + 1; cg < NG; ++cg) {
        const int c = cg * GS + gr;
        if (tid == 0) {
          while (ld_acquire(p.flags + c) == 0) {
          }
          p.flags[c] = 0;  // consumed: the context's flag array is left zeroed for the next launch
        }
        __syncthreads();
        const double* slot = p.partials + size_t(c) * (BM * BN);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              acc[mt][nt][e] += __ldcg(slot + size_t(((warp * MT + mt) * NT + nt) * 2 + e) * 32 + lane);
        if (long(cg + 1) * p.total_iters / NG >= tile_end) break;
      }
    }
    if constexpr (RESID) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const long r = m0 + wm0 + mt * 8 + g;
        if (r >= p.M) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const long cidx = n0 + wn0 + nt * 8 + 2 * t;
          const double* src = p.ref + r * p.ldref + cidx;
          if (cidx + 1 < p.N) {
            const double2 a2 = __ldcs(reinterpret_cast<const double2*>(src));
            const double d0 = a2.x - acc[mt][nt][0], d1 = a2.y - acc[mt][nt][1];
            res2 = fma(d0, d0, res2);
            res2 = fma(d1, d1, res2);
            ref2 = fma(a2.x, a2.x, ref2);
            ref2 = fma(a2.y, a2.y, ref2);
          } else if (cidx < p.N) {
            const double a0 = __ldcs(src);
            const double d0 = a0 - acc[mt][nt][0];
            res2 = fma(d0, d0, res2);
            ref2 = fma(a0, a0, ref2);
          }
        }
      }
      continue;
    } else {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const long r = m0 + wm0 + mt * 8 + g;
      if (r >= p.M) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const long cidx = n0 + wn0 + nt * 8 + 2 * t;
        double* dst = p.C + r * p.ldc + cidx;
        double v0 = p.alpha * acc[mt][nt][0], v1 = p.alpha * acc[mt][nt][1];
        if (cidx + 1 < p.N) {
          if (p.beta != 0.0) {
            const double2 o = *reinterpret_cast<const double2*>(dst);
            v0 += p.beta * o.x;
            v1 += p.beta * o.y;
          }
          *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
        } else if (cidx < p.N) {
          if (p.beta != 0.0) v0 += p.beta * dst[0];
          dst[0] = v0;
        }
      }
    }
    }
  }
  if (CHECK && saw_nonfinite) atomicOr(p.nonfinite, 1);
  if (SPLIT && p.red_counter) {
    // ---- fused slice sum (one thread per Gram element, slices in order) ---
    unsigned int gen = 0;
    grid_barrier(p.red_counter, gen);
    constexpr long TILE = long(BM) * BN;
    const long total = long(p.split_tiles > 0 ? p.split_tiles : p.units / p.split) * TILE;
    const long per = (total + G - 1) / G;
    const long e0 = long(blockIdx.x) * per, e1 = lmin(total, e0 + per);
    double dev = 0.0;
    for (long idx = e0 + tid; idx < e1; idx += THREADS) {
      const int tsel = int(idx / TILE);
      const long e = idx % TILE;
      int first, S;
      split_tile(p, tsel, first, S);
      const double* src = p.partials + size_t(first) * TILE + e;
      double acc = 0.0;
      for (int s0 = 0; s0 < S; s0 += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (s0 + q < S) ? __ldcg(src + size_t(s0 + q) * TILE) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += v[q];
      }
      int tm, tn;
      if (p.sym) {
        upper_tile(tsel, p.tiles_n, tm, tn);
      } else {
        tm = tsel / p.tiles_n;
        tn = tsel % p.tiles_n;
      }
      const long r = long(tm) * BM + e / BN, c = long(tn) * BN + e % BN;
      if (r < p.red_np && c < p.red_np) {
        if (r >= p.red_n || c >= p.red_n) acc = (r == c) ? 1.0 : 0.0;
        p.red_G[r * p.red_np + c] = acc;
        if (p.red_Gcopy) p.red_Gcopy[r * p.red_np + c] = acc;
        const double d = fabs(acc - (r == c ? 1.0 : 0.0));
        dev = (d <= dev) ? dev : d;  // NaN sticks
      }
    }
    if (p.red_emax) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, dev, o);
        dev = (x <= dev) ? dev : x;
      }
      if (lane == 0 && dev != 0.0) {
        const unsigned long long bits = (dev == dev) ? __double_as_longlong(dev) : 0x7ff0000000000000ull;
        atomicMax(p.red_emax, bits);
      }
    }
  }
  if (RESID) {
    // fixed-order CTA reduction → sums[2·cta + {0,1}]
    __shared__ double s_red[2][THREADS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      res2 += __shfl_xor_sync(0xffffffffu, res2, o);
      ref2 += __shfl_xor_sync(0xffffffffu, ref2, o);
    }
    if (lane == 0) {
      s_red[0][warp] = res2;
      s_red[1][warp] = ref2;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < THREADS / 32; ++w) {
        a += s_red[0][w];
        b += s_red[1][w];
      }
      p.sums[2 * blockIdx.x] = a;
      p.sums[2 * blockIdx.x + 1] = b;
    }
  }
}

}  // namespace pbq
