// TMA-staged variant of the FP64 DMMA GEMM (gemm_f64.cuh): same contraction
// modes, stream-K schedule, CTA groups, fix-up, SPLIT / RESID epilogues and
// CHECK scan, but the k-block ring is filled by the Tensor Memory Accelerator
// (cp.async.bulk.tensor.2d, SASS UTMALDG) instead of per-thread cp.async.
//
//   * One thread issues the copies of a stage: A and B as 2-D boxes of 16
//     doubles (128 bytes) × rows, 128-byte swizzled, completing on the
//     stage's `full` mbarrier (expect_tx = the stage's bytes).  Out-of-range
//     rows/columns are zero-filled by the TMA unit, so ragged M, N and K need
//     no predicates.
//   * Each warp releases a stage with one arrival on `empty` (16 arrivals).
//   * Fragment loads read the swizzled boxes.  A box row is 128 bytes (16
//     doubles); the hardware XORs the 16-byte chunk index with (row mod 8).
//     An 8-byte fragment load is served per half-warp, so the 16 lanes of a
//     half-warp must hit 16 distinct (chunk, 8-byte half) slots.  The DMMA
//     m8n8k4 output rows/columns may be permuted freely, so operands stored
//     [k][x] take x = (g%2) + 8·((g/2)%2) + 2·(g/4) (+4 for odd fragments):
//     the two lanes of a half-warp that share a half sit 4 chunks apart, and
//     the row XOR over k = 4·kk + t spreads t over the other chunk bits.
//     Operands stored [m][k] (A of D = A·X) take m = 2·(g%4) + g/4, whose
//     row XOR interleaves the chunk pairs the same way.  One wavefront per
//     half-warp, no bank conflicts.
#pragma once
#include <cuda.h>
#include "gemm_f64.cuh"

namespace pbq {

struct __align__(64) GemmTmaArgs {
  CUtensorMap ta;  // A: TRANS_A dims {M, K} box {16, BK}; else dims {K, M} box {16, BM}
  CUtensorMap tb;  // B: dims {N, K} box {16, BK}
  GemmArgs g;
  // 1: the map is 3-D {16, rows, cols/16} (column groups of 16 as the outer
  // dimension, byte stride 128) and one copy loads the whole tile in the same
  // shared-memory layout as the per-group boxes (cols a multiple of 16)
  int a3d, b3d;
  int a_policy;  // 1: A loaded with the evict_first L2 policy (3-D copies only; A/B experiment)
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// The same copies with an L2 cache-policy operand (createpolicy).  A/B
// experiment (PBQ_GEMM_A_POLICY=1): the streamed A operand loaded evict_first
// so that it does not push the thin, re-read B operand out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
      "[%4], %5;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

template <bool TRANS_A, int BM, int BN, int WM, int WN, int STAGES, bool CHECK, bool SPLIT = false, bool RESID = false>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, 1) gemm_f64_tma(const __grid_constant__ GemmTmaArgs pa) {
  constexpr int BK = 32;
  constexpr int WARPS_N = BN / WN;
  constexpr int NWARPS = (BM / WM) * WARPS_N;
  constexpr int THREADS = NWARPS * 32;
  constexpr int MT = WM / 8, NT = WN / 8;
  constexpr int KSTEPS = BK / 4;
  constexpr uint32_t A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static_assert(WM % 16 == 0 || !TRANS_A, "TRANS_A warp tile rows: multiple of 16");
  static_assert(WN % 16 == 0, "warp tile columns: multiple of 16");
  const GemmArgs& p = pa.g;
  extern __shared__ __align__(16) unsigned char smem_raw[];  // ring aligned to 1024 below (an __align__(1024) here would pad the static shared memory of every kernel in the library)
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&pa.ta);
    tma_prefetch_desc(&pa.tb);
  }
  // launched with programmatic serialization: everything above overlaps the
  // predecessor's tail; nothing it wrote is read before this point
  pdl_wait();
  pdl_trigger();
  if (p.skip && __ldcg(p.skip) != 0) return;
  if (p.run_if && __ldcg(p.run_if) == 0) return;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  int wm0 = (warp / WARPS_N) * WM;
  int wn0 = (warp % WARPS_N) * WN;
  const int G = gridDim.x;
  const int GS = (SPLIT || p.group < 1) ? 1 : p.group;
  const int NG = G / GS, gi = blockIdx.x / GS, gr = blockIdx.x % GS;
  // 1024-byte aligned ring (128-byte swizzle atoms)
  const uint32_t ring = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const unsigned char* ring_gen = smem_raw + (ring - smem_u32(smem_raw));
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NWARPS);
    }
    mbar_fence_init();
  }
  // Blocked summation through tensor memory (plain GEMMs): every FOLD_KB
  // k-blocks a warp adds its register accumulator into a running sum parked
  // in TMEM and restarts it at zero, so no DMMA chain is longer than
  // FOLD_KB·BK/4 = 256 steps.  The four warps of a scheduler fold at
  // staggered k-blocks, so three of them keep the DMMA pipe busy while one
  // folds.  A pass over A (K = n1 up to 2·10⁵) would
  // otherwise sum each output in one chain of K/4 DMMAs; tools/gemm_accuracy.py
  // measured 3.6 u max error against an extended-precision sum at K = 65536
  // (OpenBLAS, K-blocked, 0.22 u), enough to push config 5's d = 512 tail
  // columns past the reference's own reordering noise (tools/noise_floor.py).
  // TMEM is otherwise idle in an FP64 kernel (tcgen05 has no f64 MMA kind).
  constexpr bool FOLD = !SPLIT && !RESID;
  constexpr int FOLD_KB = 32;
  constexpr int ACC_D = MT * NT * 2;  // accumulator doubles per thread
  static_assert(ACC_D % 8 == 0, "accumulator folds move 8 doubles at a time");
  constexpr uint32_t TM_NEED = uint32_t((NWARPS + 3) / 4) * ACC_D * 2;
  constexpr uint32_t TM_COLS = TM_NEED <= 32 ? 32 : TM_NEED <= 64 ? 64 : TM_NEED <= 128 ? 128 : TM_NEED <= 256 ? 256 : 512;
  static_assert(TM_NEED <= 512, "TMEM holds 512 columns");
  __shared__ uint32_t s_tmem;
  // a fold needs a k-block chain longer than the first stagger step (FOLD_KB/4):
  // the short products of the QR chain (K = n ≤ 256) never fold and skip TMEM
  const bool use_tmem = FOLD && p.k_iters > FOLD_KB / 4;
  if (use_tmem) {
    if (warp == 0) tmem_alloc(&s_tmem, TM_COLS);
    tmem_fence_before_sync();
  }
  __syncthreads();
  uint32_t tm_mine = 0;  // this warp's columns in its lane quarter
  if (use_tmem) {
    tmem_fence_after_sync();
    tm_mine = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(warp >> 2) * uint32_t(ACC_D * 2);
  }

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

  // ---- producer (thread 0): k-blocks in flat order into the ring ---------
  // Its cursor lives in shared memory: only thread 0 touches it, once per
  // k-block, and keeping it out of registers leaves the 16 consumer warps
  // their full 128-register budget without spills.
  struct Prod {
    Cursor cur;
    Seg seg;
    long flat;
    int k, live;
  };
  __shared__ Prod prod;
  if (tid == 0) {
    prod.cur = first_cursor();
    prod.live = next_seg(prod.cur, prod.seg);
    prod.k = prod.live ? prod.seg.kb : 0;
    prod.flat = 0;
  }
  auto produce = [&]() {
    if (tid != 0 || !prod.live) return;
    const long pflat = prod.flat;
    const int stage = int(pflat % STAGES);
    if (pflat >= STAGES) mbar_wait(&empty_bar[stage], unsigned((pflat / STAGES - 1) & 1));
    const uint32_t sa = ring + uint32_t(stage) * STAGE_BYTES, sb = sa + A_BYTES;
    const uint32_t bar = smem_u32(&full_bar[stage]);
    mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
    const int k0 = prod.k * BK, m0 = prod.seg.tm * BM, n0 = prod.seg.tn * BN;
    if (pa.a3d && pa.a_policy) {
      const uint64_t pol_a = l2_policy_evict_first();
      if (TRANS_A)
        tma_load_3d_hint(sa, &pa.ta, 0, k0, m0 / 16, bar, pol_a);
      else
        tma_load_3d_hint(sa, &pa.ta, 0, m0, k0 / 16, bar, pol_a);
    } else if (pa.a3d) {
      if (TRANS_A)
        tma_load_3d(sa, &pa.ta, 0, k0, m0 / 16, bar);
      else
        tma_load_3d(sa, &pa.ta, 0, m0, k0 / 16, bar);
    } else if (TRANS_A) {
#pragma unroll
      for (int i = 0; i < BM / 16; ++i) tma_load_2d(sa + i * (BK * 128), &pa.ta, m0 + 16 * i, k0, bar);
    } else {
#pragma unroll
      for (int h = 0; h < BK / 16; ++h) tma_load_2d(sa + h * (BM * 128), &pa.ta, k0 + 16 * h, m0, bar);
    }
    if (pa.b3d) {
      tma_load_3d(sb, &pa.tb, 0, k0, n0 / 16, bar);
    } else {
#pragma unroll
      for (int j = 0; j < BN / 16; ++j) tma_load_2d(sb + j * (BK * 128), &pa.tb, n0 + 16 * j, k0, bar);
    }
    prod.flat = pflat + 1;
    if (++prod.k == prod.seg.ke) {
      prod.live = next_seg(prod.cur, prod.seg);
      if (prod.live) prod.k = prod.seg.kb;
    }
  };
#pragma unroll 1
  for (int s = 0; s < STAGES - 1; ++s) produce();

  // ---- per-thread fragment byte offsets inside a stage -------------------
  // k-step kk contracts k = 4·kk + t (the natural order).
  // [k][x] boxes (A of AᵀX, and B): x = w0 + xoff(f) + xg, xg = (g%2) +
  //   8·((g/2)%2) + 2·(g/4), xoff(f) = 4·(f%2) + 16·(f/2).  Byte offset
  //   (x/16)·BK·128 + k·128 + (((x%16)/2) ^ (k%8))·16 + (x%2)·8
  //   = [(w0/16 + f/2)·4096 + 512·kk] + V[(f%2) + 2·(kk%2)],
  //   V[c] = 128·t + 8·(g%2) + 16·(Q ^ 2c),  Q = 4·((g/2)%2) + g/4 ^ t.
  // [m][k] boxes (A of A·X): m = wm0 + 8·f + mg, mg = 2·(g%4) + g/4.  Byte
  //   offset (k/16)·BM·128 + m·128 + (((k%16)/2) ^ (m%8))·16 + (k%2)·8
  //   = [(kk/4)·BM·128 + (wm0 + 8f)·128] + Z[kk%4],
  //   Z[c] = 128·mg + 8·(t%2) + 16·(Y ^ 2c),  Y = (t/2) ^ mg.
  // In each half-warp the 16 loads then cover the 16 (16-byte chunk, half)
  // slots of the 128-byte bank space once: one wavefront per half-warp.
  const int xg = (g & 1) + 8 * ((g >> 1) & 1) + 2 * (g >> 2);
  const int mg = 2 * (g & 3) + (g >> 2);
  uint32_t V[4], Z[4];
  {
    const uint32_t Q = uint32_t((4 * ((g >> 1) & 1) + (g >> 2)) ^ t);
    const uint32_t Y = uint32_t((t >> 1) ^ mg);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      V[c] = uint32_t(128 * t + 8 * (g & 1)) + ((Q ^ uint32_t(2 * c)) << 4);
      Z[c] = uint32_t(128 * mg + 8 * (t & 1)) + ((Y ^ uint32_t(2 * c)) << 4);
    }
  }

  Cursor ccur = first_cursor();
  Seg seg;
  long cflat = 0;
  bool saw_nonfinite = false;
  double res2 = 0.0, ref2 = 0.0;
  while (next_seg(ccur, seg)) {
    const long m0 = long(seg.tm) * BM, n0 = long(seg.tn) * BN;
    const bool check = CHECK && (seg.tn == 0);
    // A symmetric Gram's diagonal tile: the 6 warp tiles strictly below its
    // diagonal are never read (the Cholesky uses blocks i ≤ j of G), so they
    // are skipped and stay zero.  The warps are remapped so that the skipped
    // tiles fall 2/1/1/2 on the four schedulers (warp w runs on w mod 4):
    // 2/3/3/2 live warp tiles per scheduler instead of up to 4.
    bool lowskip = false;
    if constexpr (SPLIT && BM == 128 && BN == 128 && WM == 32 && WN == 32) {
      if (p.sym && p.split_diag > 0 && seg.tm == seg.tn) {
        constexpr unsigned long long kMap = 0xE9C8DF64B7A53210ull;  // warp w → warp tile (4-bit wr·4 + wc)
        const int wt = int((kMap >> (4 * warp)) & 15);
        wm0 = (wt >> 2) * WM;
        wn0 = (wt & 3) * WN;
        lowskip = wm0 > wn0;
      } else {
        wm0 = (warp / WARPS_N) * WM;
        wn0 = (warp % WARPS_N) * WN;
      }
    }
    // Triangular B (Q₁ = A·R⁻¹): inside the diagonal 128-block of B, k-block
    // kl (0…3) has nonzeros only in columns ≥ 32·kl, so warp tiles of warp
    // column wc < kl skip it.  Warps are mapped so each scheduler holds one
    // warp tile of every column: (wr, wc) = (w/4, (w + w/4) mod 4), and the
    // skips thin out all four schedulers equally.
    int tri_kl0 = 1 << 30;  // k-block index where the diagonal block of B starts
    int wcol = 0;
    if constexpr (!SPLIT && !RESID && BM == 128 && BN == 128 && WM == 32 && WN == 32) {
      if (p.tri_b) {
        const int wr = warp >> 2, wc = (warp + (warp >> 2)) & 3;
        wm0 = wr * WM;
        wn0 = wc * WN;
        wcol = wc;
        tri_kl0 = int(n0 / BK);
      } else {
        wm0 = (warp / WARPS_N) * WM;
        wn0 = (warp % WARPS_N) * WN;
      }
    }
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    bool folded = false;
    // acc → TMEM (first fold: store; later: add), then restart at zero
    auto fold = [&]() {
#pragma unroll
      for (int c = 0; c < ACC_D / 8; ++c) {
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int x = 8 * c + i;
          v[i] = acc[x / (NT * 2)][(x / 2) % NT][x % 2];
        }
        if (folded) {
          double o[8];
          tmem_ld8d(tm_mine + uint32_t(16 * c), o);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = o[i] + v[i];
        }
        tmem_st8d(tm_mine + uint32_t(16 * c), v);
      }
      tmem_wait_st();
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      folded = true;
    };

#pragma unroll 1
    for (int kbk = seg.kb; kbk < seg.ke; ++kbk) {
      const int stage = int(cflat % STAGES);
      mbar_wait(&full_bar[stage], unsigned((cflat / STAGES) & 1));
      const unsigned char* sA = ring_gen + size_t(stage) * STAGE_BYTES;
      const unsigned char* sB = sA + A_BYTES;
      if (CHECK && check) {
        // the k-block's A tile as raw bytes: the swizzle only permutes it
        // (not unrolled: keeps the NN variant's consumers inside 128 registers)
#pragma unroll 1
        for (int i = 0; i < int(A_BYTES / 16 / THREADS); ++i) {
          const double2 v = *reinterpret_cast<const double2*>(sA + (size_t(i) * THREADS + tid) * 16);
          saw_nonfinite |= nonfinite_bits(v.x) | nonfinite_bits(v.y);
        }
      }
      double fa[2][MT], fb[2][NT];
      auto load_frags = [&](int kk, double (&a)[MT], double (&b)[NT]) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t off;
          if (TRANS_A)
            off = uint32_t(((wm0 >> 4) + (mt >> 1)) * 4096 + 512 * kk) + V[(mt & 1) + 2 * (kk & 1)];
          else
            off = uint32_t((kk >> 2) * (BM * 128) + (wm0 + 8 * mt) * 128) + Z[kk & 3];
          a[mt] = *reinterpret_cast<const double*>(sA + off);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          b[nt] = *reinterpret_cast<const double*>(sB + uint32_t(((wn0 >> 4) + (nt >> 1)) * 4096 + 512 * kk) +
                                                   V[(nt & 1) + 2 * (kk & 1)]);
      };
      if (!lowskip && !(kbk - tri_kl0 > wcol)) {
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
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[stage]);
      ++cflat;
      produce();
      if constexpr (FOLD) {
        if (use_tmem && (kbk + 1 - seg.kb + (warp >> 2) * (FOLD_KB / 4)) % FOLD_KB == 0 && kbk + 1 < seg.ke) fold();
      }
    }
    if constexpr (FOLD) {
      if (folded) {  // final = running sum + the last chain
#pragma unroll
        for (int c = 0; c < ACC_D / 8; ++c) {
          double o[8];
          tmem_ld8d(tm_mine + uint32_t(16 * c), o);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int x = 8 * c + i;
            acc[x / (NT * 2)][(x / 2) % NT][x % 2] = o[i] + acc[x / (NT * 2)][(x / 2) % NT][x % 2];
          }
        }
      }
    }

    // output coordinates of this thread's accumulators
    auto out_row = [&](int mt) -> int {
      return TRANS_A ? wm0 + 4 * (mt & 1) + 16 * (mt >> 1) + xg : wm0 + 8 * mt + mg;
    };
    // accumulator columns 2t, 2t+1 of fragment nt: x = xoff(nt) + 8·(t%2) + 2·(t/2) + {0, 1}
    auto out_col = [&](int nt) -> int { return wn0 + 4 * (nt & 1) + 16 * (nt >> 1) + 8 * (t & 1) + 2 * (t >> 1); };

    if (SPLIT) {
      double* slot = p.partials + size_t(ccur.unit - G) * (BM * BN);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          __stcg(reinterpret_cast<double2*>(slot + out_row(mt) * BN + out_col(nt)),
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
        const long r = m0 + out_row(mt);
        if (r >= p.M) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const long cidx = n0 + out_col(nt);
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
    }
    // plain epilogue, or the scatter into the slice owner's landing slot
    int owner = 0;
    double* cbase = p.C + m0 * p.ldc;
    long ldo = p.ldc;
    if (p.xs_land) {
      owner = int(m0 / p.xs_S);
      cbase = p.xs_land[owner] + (long(p.xs_rank) * p.xs_S + (m0 - long(owner) * p.xs_S)) * p.xs_ldl;
      ldo = p.xs_ldl;
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const long r = m0 + out_row(mt);
      if (r >= p.M) continue;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const long cidx = n0 + out_col(nt);
        double* dst = cbase + (r - m0) * ldo + cidx;
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
    if (p.xs_land) {  // the tile has landed in the owner's slot: count it there
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        asm volatile("red.release.sys.global.add.u32 [%0], 1;\n" ::"l"(p.xs_cnt[owner]) : "memory");
      }
    }
  }
  if (CHECK && saw_nonfinite) atomicOr(p.nonfinite, 1);
  if (SPLIT && p.red_counter) {
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
        dev = (d <= dev) ? dev : d;
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
  if (use_tmem) {  // every warp's TMEM traffic has completed (loads waited, stores waited)
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (warp == 0) tmem_dealloc(s_tmem, TM_COLS);
  }
  if (RESID) {
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

template <bool TRANS_A, int BM, int BN, int STAGES>
constexpr size_t gemm_tma_smem_bytes() {
  return size_t(STAGES) * (BM + BN) * 32 * 8 + 1024;
}

}  // namespace pbq
