// Device Gaussian sketch Φ, bit-compatible with the reference's
// `gaussian_matrix(rows, cols, seed)` (/root/reference/pkg/src/pbpqlp/linalg.py:83-93):
// numpy Generator(Philox(key=seed)).standard_normal((rows, cols)).
//
// Stream: Philox4x64-10 (Salmon et al., SC'11) keyed by the 128-bit seed, counter
// (c+1, 0, 0, 0) for block c, four u64 words per block in order — stream
// position p is word p%4 of block p/4.  Each normal consumes ≥ 1 word (numpy's
// ziggurat: ~1.022 words/normal on average), so the position at which normal i
// starts depends on every earlier draw.  The GPU resolves that dependency in
// three passes over fixed 1024-position chunks of the stream, one chunk per
// warp (lane ℓ owns positions 32ℓ..32ℓ+31 as a 32-bit mask; no CTA barriers):
//   K1 generates the chunk's Philox words once: the value a normal starting
//      at each position would take (the rectangle-test value, or the fully
//      resolved ziggurat value for the rare "special" positions the test
//      rejects) is written position-indexed (coalesced, through padded shared
//      memory), the special positions and where their normals end are saved,
//      and the start chain is walked for every possible entry offset
//      e ∈ [0, 32).  Chains from different entries merge within a few
//      positions, so a chunk's exit does not depend on its entry (checked; a
//      violation sets the error flag).
//   K2 (one CTA) turns exits into per-chunk entry offsets and exclusive-scans
//      the per-chunk normal counts.
//   K3 rebuilds the chain's start positions from the saved specials, ranks
//      them with a warp scan, gathers their values and writes them coalesced
//      to Φ — a memory-bound compaction (no Philox).
// Values equal numpy's bit for bit.  The exponential-tail branch (idx 0,
// ~2.6e-4 of draws) calls log1p; numpy calls the C library's, so the device
// uses glibc_log1p below, a restatement of glibc's (fdlibm-derived) log1p as
// its x86-64 FMA build evaluates it — bitwise equal to the host libm on 1e8
// samples of the sampler's domain (tests/test_oracle.py).  The wedge test's
// exp(-x²/2) only decides accept/reject, where a last-bit difference between
// CUDA's exp and the host's matters only if the comparison ties to the ulp.
#pragma once
#include <math_constants.h>

#include "common.cuh"
#include "ziggurat_tables.h"

namespace pbq {

constexpr int PBQ_SK_CHUNK = 1024;      // stream positions per chunk (one warp)
constexpr int PBQ_SK_WARPS = 4;         // chunks per CTA (static smem ≤ 48 KB)
constexpr int PBQ_SK_THREADS = 32 * PBQ_SK_WARPS;
constexpr int PBQ_SK_E = 32;            // entry offsets tracked per chunk
constexpr int PBQ_SK_MAXSPECIAL = 64;   // special draws per chunk (mean ≈ 7.5; P(> 64) < 1e-30)

__constant__ uint64_t c_zig_ki[256];
__constant__ double c_zig_wi[256];
__constant__ double c_zig_fi[256];

struct Philox4x64 {
  uint64_t x[4];
};

__device__ __forceinline__ Philox4x64 philox4x64_10(uint64_t ctr0, uint64_t k0, uint64_t k1) {
  uint64_t x0 = ctr0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * x0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, x0);
    const uint64_t lo1 = 0xCA5A826395121157ULL * x2, hi1 = __umul64hi(0xCA5A826395121157ULL, x2);
    const uint64_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  Philox4x64 o;
  o.x[0] = x0; o.x[1] = x1; o.x[2] = x2; o.x[3] = x3;
  return o;
}

// Word p of the stream keyed by (k0, k1).
__device__ __forceinline__ uint64_t philox_word(uint64_t p, uint64_t k0, uint64_t k1) {
  const Philox4x64 b = philox4x64_10((p >> 2) + 1, k0, k1);
  const int w = int(p & 3);
  return w == 0 ? b.x[0] : (w == 1 ? b.x[1] : (w == 2 ? b.x[2] : b.x[3]));
}

__device__ __forceinline__ double u64_to_unit(uint64_t v) {
  return double(v >> 11) * (1.0 / 9007199254740992.0);
}

// Layer tables staged in shared memory: lanes index different layers, which
// would serialise 32-way through the constant cache.
struct ZigTables {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
};
__device__ __forceinline__ void zig_stage(ZigTables& t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t.ki[i] = c_zig_ki[i];
    t.wi[i] = c_zig_wi[i];
    t.fi[i] = c_zig_fi[i];
  }
  __syncthreads();
}

// A draw is "fast" when the rectangle test accepts it.
__device__ __forceinline__ bool zig_fast(const ZigTables& t, uint64_t r) {
  const int idx = int(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  return rabs < t.ki[idx];
}
__device__ __forceinline__ double zig_fast_value(const ZigTables& t, uint64_t r) {
  const int idx = int(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  double x = double(rabs) * t.wi[idx];
  return ((r >> 8) & 1) ? -x : x;
}

// log1p(x) exactly as glibc 2.39 computes it on x86-64 with FMA (the ifunc
// variant numpy's npy_log1p reaches on the reference's hosts): the fdlibm
// s_log1p.c algorithm (Sun Microsystems, 1993) — argument reduction
// 1+x = 2^k·(1+f) with the correction term c, s = f/(2+f), the degree-14
// polynomial in z = s² with fdlibm's Lp1..Lp7 evaluated in glibc's
// z/z²/z⁴/z⁶ (Estrin) grouping — with every multiply-add that GCC contracts
// in that build written as fma() and every other operation rounded on its
// own (__dmul_rn/__dadd_rn/__dsub_rn never contract).  Host twin for the
// checks: oracle/sketch_oracle.c.  Only x ∈ (−1, 0] reaches it here, but the
// whole function is restated.
__device__ __forceinline__ double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {  // x < 0.41422
    if (ax >= 0x3ff00000) return x == -1.0 ? -CUDART_INF : CUDART_NAN;
    if (ax < 0x3e200000) {  // |x| < 2^-29
      if (ax < 0x3c900000) return x;
      return fma(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= int(0xbfd2bec3)) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return __dadd_rn(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double dk = double(k);
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma(dk, ln2_lo, c);
      return fma(dk, ln2_hi, c);
    }
    const double R = __dmul_rn(hfsq, fma(-f, 0.66666666666666666, 1.0));
    if (k == 0) return __dsub_rn(f, R);
    return fma(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, fma(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
  const double R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, __dmul_rn(z2, R2))));
  const double shr = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, shr));
  return fma(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(shr, fma(dk, ln2_lo, c))), f));
}

// Full sampler for a normal whose first attempt starts at stream position p.
// Returns the position after the normal and (optionally) its value.
__device__ uint64_t zig_resolve(const ZigTables& t, uint64_t p, uint64_t k0, uint64_t k1, double* value) {
  for (;;) {
    const uint64_t r = philox_word(p, k0, k1);
    p += 1;
    const int idx = int(r & 0xff);
    const uint64_t rr = r >> 8;
    const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
    double x = double(rabs) * t.wi[idx];
    if (rr & 1) x = -x;
    if (rabs < t.ki[idx]) {
      if (value) *value = x;
      return p;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-PBQ_ZIG_INV_R, glibc_log1p(-u64_to_unit(philox_word(p, k0, k1))));
        const double yy = -glibc_log1p(-u64_to_unit(philox_word(p + 1, k0, k1)));
        p += 2;
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          if (value) *value = ((rabs >> 8) & 1) ? -(PBQ_ZIG_R + xx) : (PBQ_ZIG_R + xx);
          return p;
        }
      }
    }
    const double u = u64_to_unit(philox_word(p, k0, k1));
    p += 1;
    // numpy's C evaluates this without contraction: round every step alone
    if (__dadd_rn(__dmul_rn(__dsub_rn(t.fi[idx - 1], t.fi[idx]), u), t.fi[idx]) <
        exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
      if (value) *value = x;
      return p;
    }
  }
}

struct SketchArgs {
  uint64_t k0, k1;
  const uint64_t* seed_dev;  // when set, the key {k0, k1} is read from device memory (CUDA-graph replays)
  long n_chunks;
  long vchunk0;  // chunks below it end before stream position `first` (normal index ≤ position),
                 // so they hold no requested normal: K1 walks them for the chain only
  long first;  // global index of the first normal to emit (row_offset·cols)
  long count;  // normals to emit (rows·cols)
  long cols;
  double* out;
  long ldo;
  int* exits;   // n_chunks: exit offset past chunk end (= entry of the next)
  int* counts;  // n_chunks × E
  long* base;   // n_chunks: global normal index of the chunk's first start
  int* entry;   // n_chunks: entry offset of the chunk
  int* error;   // set on internal overflow
  double* vals;     // (n_chunks − vchunk0) × 1024: value of a normal starting at each position
  uint64_t* sp;     // (n_chunks − vchunk0) × 2·MAXSPECIAL: special positions, then where their normals end
  int* nsp;         // n_chunks − vchunk0: number of specials
};

struct SkWarpSmem {
  uint64_t sp_pos[PBQ_SK_MAXSPECIAL];
  uint64_t sp_next[PBQ_SK_MAXSPECIAL];
  unsigned keep[32];  // K3: per-lane start masks
};

// Warp-level discovery of the sorted special positions of one chunk; lane ℓ's
// 32 positions → `mask` bit j (special draw at chunk position 32ℓ + j).
__device__ __forceinline__ int sk_find_specials(const ZigTables& t, const SketchArgs& a, long chunk, SkWarpSmem& w,
                                                unsigned& mask) {
  const int lane = threadIdx.x & 31;
  const uint64_t p0 = uint64_t(chunk) * PBQ_SK_CHUNK + uint64_t(lane) * 32;
  mask = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const Philox4x64 blk = philox4x64_10((p0 >> 2) + b + 1, a.k0, a.k1);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (!zig_fast(t, blk.x[q])) mask |= 1u << (b * 4 + q);
  }
  const int mine = __popc(mask);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int off = incl - mine;
  for (unsigned m = mask; m; m &= m - 1) {
    const int j = __ffs(m) - 1;
    if (off < PBQ_SK_MAXSPECIAL) w.sp_pos[off] = p0 + j;
    ++off;
  }
  const int nsp = min(total, PBQ_SK_MAXSPECIAL);
  if (total > PBQ_SK_MAXSPECIAL && lane == 0) atomicExch(a.error, 1);
  __syncwarp();
  for (int i = lane; i < nsp; i += 32) w.sp_next[i] = zig_resolve(t, w.sp_pos[i], a.k0, a.k1, nullptr);
  __syncwarp();
  return nsp;
}

// Walk the start chain of one chunk from entry position s.
__device__ __forceinline__ void sk_walk(uint64_t s, uint64_t cend, const SkWarpSmem& w, int nsp, int& count,
                                        uint64_t& exit_pos) {
  int c = 0;
  for (int i = 0; i < nsp; ++i) {
    const uint64_t sp = w.sp_pos[i];
    if (sp < s) continue;
    if (sp >= cend) break;
    c += int(sp - s) + 1;
    s = w.sp_next[i];
    if (s >= cend) break;
  }
  if (s < cend) {
    c += int(cend - s);
    s = cend;
  }
  count = c;
  exit_pos = s;
}

__global__ void __launch_bounds__(PBQ_SK_THREADS, 5) sketch_k1(SketchArgs a) {
  if (a.seed_dev) {
    a.k0 = __ldg(a.seed_dev);
    a.k1 = __ldg(a.seed_dev + 1);
  }
  __shared__ SkWarpSmem sw[PBQ_SK_WARPS];
  __shared__ double stage[PBQ_SK_WARPS][32 * 33];  // position-indexed values, row ℓ = lane ℓ's 32 positions (padded)
  __shared__ ZigTables zt;
  zig_stage(zt);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long chunk = long(blockIdx.x) * PBQ_SK_WARPS + warp;
  if (chunk >= a.n_chunks) return;
  SkWarpSmem& w = sw[warp];
  double* st = stage[warp];
  const uint64_t cstart = uint64_t(chunk) * PBQ_SK_CHUNK, cend = cstart + PBQ_SK_CHUNK;
  const uint64_t p0 = cstart + uint64_t(lane) * 32;
  // one Philox pass: rectangle-test values, and the special mask
  unsigned mask = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const Philox4x64 blk = philox4x64_10((p0 >> 2) + b + 1, a.k0, a.k1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t r = blk.x[q];
      if (zig_fast(zt, r))
        st[lane * 33 + b * 4 + q] = zig_fast_value(zt, r);
      else
        mask |= 1u << (b * 4 + q);
    }
  }
  const int mine = __popc(mask);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int off = incl - mine;
  for (unsigned m = mask; m; m &= m - 1) {
    const int j = __ffs(m) - 1;
    if (off < PBQ_SK_MAXSPECIAL) w.sp_pos[off] = p0 + j;
    ++off;
  }
  const int nsp = min(total, PBQ_SK_MAXSPECIAL);
  if (total > PBQ_SK_MAXSPECIAL && lane == 0) atomicExch(a.error, 1);
  __syncwarp();
  // resolve the specials (full sampler); their values go to their positions.
  // A prefix chunk (below vchunk0, e.g. the rows before this rank's row block)
  // only needs where its specials end, for the chain walk: no values, no saves.
  const bool keep = chunk >= a.vchunk0;
  const long vc = chunk - a.vchunk0;
  uint64_t* gsp = a.sp + size_t(keep ? vc : 0) * 2 * PBQ_SK_MAXSPECIAL;
  for (int i = lane; i < nsp; i += 32) {
    double v;
    const uint64_t sp = w.sp_pos[i];
    const uint64_t nx = zig_resolve(zt, sp, a.k0, a.k1, &v);
    w.sp_next[i] = nx;
    if (keep) {
      const int rel = int(sp - cstart);
      st[(rel >> 5) * 33 + (rel & 31)] = v;
      gsp[i] = sp;
      gsp[PBQ_SK_MAXSPECIAL + i] = nx;
    }
  }
  if (keep && lane == 0) a.nsp[vc] = nsp;
  __syncwarp();
  // coalesced position-indexed write-out
  if (keep) {
    double* gv = a.vals + size_t(vc) * PBQ_SK_CHUNK;
#pragma unroll 8
    for (int e = lane; e < PBQ_SK_CHUNK; e += 32) __stcg(gv + e, st[(e >> 5) * 33 + (e & 31)]);
  }
  int cnt;
  uint64_t ex;
  sk_walk(cstart + lane, cend, w, nsp, cnt, ex);  // entry offset = lane
  a.counts[chunk * PBQ_SK_E + lane] = cnt;
  const uint64_t ex0 = __shfl_sync(0xffffffffu, ex, 0);
  const bool merged = __all_sync(0xffffffffu, ex == ex0);
  if (lane == 0) {
    const uint64_t off2 = ex0 - cend;
    if (!merged || off2 >= uint64_t(PBQ_SK_E)) atomicExch(a.error, 2);
    a.exits[chunk] = int(off2 < uint64_t(PBQ_SK_E) ? off2 : 0);
  }
}

// Single-CTA scan: entry offsets and exclusive prefix of per-chunk counts.
__global__ void __launch_bounds__(1024) sketch_k2(SketchArgs a) {
  __shared__ long warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long n = a.n_chunks;
  const long per = (n + 1023) / 1024;
  const long c0 = tid * per, c1 = lmin(n, c0 + per);
  // per-thread chunk run: issue all loads before using them (one round trip
  // for the exits, one for the counts)
  constexpr int RUN = 8;
  long local = 0;
  for (long cb = c0; cb < c1; cb += RUN) {
    int ex[RUN], ct[RUN];
#pragma unroll
    for (int u = 0; u < RUN; ++u) {
      const long c = cb + u;
      ex[u] = (c < c1 && c > 0) ? a.exits[c - 1] : 0;
    }
#pragma unroll
    for (int u = 0; u < RUN; ++u) {
      const long c = cb + u;
      ct[u] = (c < c1) ? a.counts[c * PBQ_SK_E + ex[u]] : 0;
    }
#pragma unroll
    for (int u = 0; u < RUN; ++u) local += ct[u];
  }
  long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  long wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += warp_tot[w];
  long run = wbase + incl - local;
  for (long cb = c0; cb < c1; cb += RUN) {
    int ex[RUN], ct[RUN];
#pragma unroll
    for (int u = 0; u < RUN; ++u) {
      const long c = cb + u;
      ex[u] = (c < c1 && c > 0) ? a.exits[c - 1] : 0;
    }
#pragma unroll
    for (int u = 0; u < RUN; ++u) {
      const long c = cb + u;
      ct[u] = (c < c1) ? a.counts[c * PBQ_SK_E + ex[u]] : 0;
    }
#pragma unroll
    for (int u = 0; u < RUN; ++u) {
      const long c = cb + u;
      if (c < c1) {
        a.entry[c] = ex[u];
        a.base[c] = run;
        run += ct[u];
      }
    }
  }
  if (tid == 1023) {
    long total = 0;
    for (int w = 0; w < 32; ++w) total += warp_tot[w];
    if (total < a.first + a.count) atomicExch(a.error, 3);
  }
}

__global__ void __launch_bounds__(PBQ_SK_THREADS, 5) sketch_k3(SketchArgs a) {
  pdl_trigger();  // a programmatically launched successor may start its prologue
  if (a.seed_dev) {
    a.k0 = __ldg(a.seed_dev);
    a.k1 = __ldg(a.seed_dev + 1);
  }
  __shared__ SkWarpSmem sw[PBQ_SK_WARPS];
  __shared__ double buf[PBQ_SK_WARPS][32 * 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long chunk = long(blockIdx.x) * PBQ_SK_WARPS + warp;
  if (chunk >= a.n_chunks) return;
  const long base = a.base[chunk];
  const int entry = a.entry[chunk];
  const int cnt_here = a.counts[chunk * PBQ_SK_E + entry];
  if (base >= a.first + a.count || base + cnt_here <= a.first) return;  // nothing requested here
  const long vc = chunk - a.vchunk0;  // ≥ 0 here: a prefix chunk never holds a requested normal
  SkWarpSmem& w = sw[warp];
  double* bw = buf[warp];
  const uint64_t cstart = uint64_t(chunk) * PBQ_SK_CHUNK, cend = cstart + PBQ_SK_CHUNK;
  // position-indexed values → padded shared memory (coalesced read)
  const double* gv = a.vals + size_t(vc) * PBQ_SK_CHUNK;
#pragma unroll 8
  for (int e = lane; e < PBQ_SK_CHUNK; e += 32) bw[(e >> 5) * 33 + (e & 31)] = __ldcs(gv + e);
  const int nsp = a.nsp[vc];
  const uint64_t* gsp = a.sp + size_t(vc) * 2 * PBQ_SK_MAXSPECIAL;
  for (int i = lane; i < nsp; i += 32) {
    w.sp_pos[i] = gsp[i];
    w.sp_next[i] = gsp[PBQ_SK_MAXSPECIAL + i];
  }
  // start mask: every position from the entry on, minus the words consumed by
  // special normals beyond their first word (walked by lane 0, set in smem)
  unsigned start = (lane * 32 >= entry) ? 0xffffffffu : ((entry - lane * 32 >= 32) ? 0u : (0xffffffffu << (entry - lane * 32)));
  w.keep[lane] = start;
  __syncwarp();
  if (lane == 0) {
    uint64_t s = cstart + entry;
    for (int i = 0; i < nsp; ++i) {
      const uint64_t sp = w.sp_pos[i];
      if (sp < s) continue;
      const uint64_t nx = w.sp_next[i];
      for (uint64_t q = sp + 1; q < nx && q < cend; ++q) {
        const int rel = int(q - cstart);
        w.keep[rel >> 5] &= ~(1u << (rel & 31));
      }
      s = nx;
      if (s >= cend) break;
    }
  }
  __syncwarp();
  start = w.keep[lane];
  const int mine = __popc(start);
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int rank = incl - mine;  // chunk-local index of this lane's first normal
  // gather this lane's start values (registers), then compact in place
  double v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = bw[lane * 33 + j];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if ((start >> j) & 1u) bw[rank++] = v[j];
  __syncwarp();
  // coalesced write-out of this chunk's normals [base, base + cnt_here)
  const long lo = lmax(base, a.first), hi = lmin(base + cnt_here, a.first + a.count);
  const long rel0 = lo - a.first;
  long row = rel0 / a.cols;
  long col = rel0 - row * a.cols;
  // lane-strided: element e ↔ lo + e
  long step_row = 32 / a.cols, step_col = 32 % a.cols;
  long r_l = row + (col + lane) / a.cols;
  long c_l = (col + lane) % a.cols;
  for (long e = lane; e < hi - lo; e += 32) {
    a.out[r_l * a.ldo + c_l] = bw[lo - base + e];
    r_l += step_row;
    c_l += step_col;
    if (c_l >= a.cols) {
      c_l -= a.cols;
      r_l += 1;
    }
  }
}

}  // namespace pbq
