// Device Gaussian sketch Φ, bit-compatible with the reference's
// `gaussian_matrix(rows, cols, seed)` (/root/reference/pkg/src/pbpqlp/linalg.py:83-93):
// numpy Generator(Philox(key=seed)).standard_normal((rows, cols)).
//
// Stream: Philox4x64-10 (Salmon et al., SC'11) keyed by the 128-bit seed, counter
// (c+1, 0, 0, 0) for block c, four u64 words per block in order — stream
// position p is word p%4 of block p/4.  Each normal consumes ≥ 1 word (numpy's
// ziggurat: ~1.023 words/normal on average), so the position at which normal i
// starts depends on every earlier draw.  The GPU resolves that dependency in
// three passes over fixed-size chunks of the stream:
//   K1 (one CTA per chunk) finds the rare "special" positions (draws that are
//      not accepted by the rectangle test), resolves where each special draw's
//      normal ends, and walks the start chain for every possible entry offset
//      e ∈ [0, PBQ_SK_E).  Chains from different entries merge within a few
//      positions, so every chunk's exit position is entry-independent (checked;
//      a violation sets the error flag).
//   K2 (one CTA) turns exits into per-chunk entry offsets and exclusive-scans
//      the per-chunk normal counts.
//   K3 (one CTA per chunk) marks the chain's start positions, ranks them with a
//      block scan and writes each normal to Φ[(i - first)/cols][(i - first)%cols].
// Values equal numpy's bit for bit, except that the exponential-tail branch
// (idx 0, ~2.6e-4 of draws) uses CUDA's log1p, which can differ from glibc's by
// 1 ulp; see DESIGN.md §5.
#pragma once
#include "common.cuh"
#include "ziggurat_tables.h"

namespace pbq {

constexpr int PBQ_SK_CHUNK = 2048;     // stream positions per chunk
constexpr int PBQ_SK_THREADS = 256;
constexpr int PBQ_SK_E = 32;           // entry offsets tracked per chunk
constexpr int PBQ_SK_MAXSPECIAL = 256; // special draws per chunk (mean ≈ 15)

__constant__ uint64_t c_zig_ki[256];
__constant__ double c_zig_wi[256];
__constant__ double c_zig_fi[256];

struct Philox4x64 {
  uint64_t x[4];
};

__device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

__device__ __forceinline__ Philox4x64 philox4x64_10(uint64_t ctr0, uint64_t k0, uint64_t k1) {
  uint64_t x0 = ctr0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, x0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ULL, x2, hi1, lo1);
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

// A draw at position p is "fast" when the rectangle test accepts it.
__device__ __forceinline__ bool zig_fast(uint64_t r) {
  const int idx = int(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  return rabs < c_zig_ki[idx];
}
__device__ __forceinline__ double zig_fast_value(uint64_t r) {
  const int idx = int(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  double x = double(rabs) * c_zig_wi[idx];
  return ((r >> 8) & 1) ? -x : x;
}

// Full sampler for a normal whose first attempt starts at stream position p.
// Returns the position after the normal and (optionally) its value.
__device__ uint64_t zig_resolve(uint64_t p, uint64_t k0, uint64_t k1, double* value) {
  for (;;) {
    const uint64_t r = philox_word(p, k0, k1);
    p += 1;
    const int idx = int(r & 0xff);
    const uint64_t rr = r >> 8;
    const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
    double x = double(rabs) * c_zig_wi[idx];
    if (rr & 1) x = -x;
    if (rabs < c_zig_ki[idx]) {
      if (value) *value = x;
      return p;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = -PBQ_ZIG_INV_R * log1p(-u64_to_unit(philox_word(p, k0, k1)));
        const double yy = -log1p(-u64_to_unit(philox_word(p + 1, k0, k1)));
        p += 2;
        if (yy + yy > xx * xx) {
          if (value) *value = ((rabs >> 8) & 1) ? -(PBQ_ZIG_R + xx) : (PBQ_ZIG_R + xx);
          return p;
        }
      }
    }
    const double u = u64_to_unit(philox_word(p, k0, k1));
    p += 1;
    if ((c_zig_fi[idx - 1] - c_zig_fi[idx]) * u + c_zig_fi[idx] < exp(-0.5 * x * x)) {
      if (value) *value = x;
      return p;
    }
  }
}

struct SketchArgs {
  uint64_t k0, k1;
  long n_chunks;
  long first;  // global index of the first normal to emit (row_offset·cols)
  long count;  // normals to emit (rows·cols)
  long cols;
  double* out;
  long ldo;
  int* exits;      // n_chunks: exit offset past chunk end (chunk-relative entry of the next)
  int* counts;     // n_chunks × E
  long* base;      // n_chunks: global normal index of the chunk's first start
  int* entry;      // n_chunks: entry offset of the chunk
  int* error;      // set on internal overflow
};

// Block-level discovery of the sorted special positions of one chunk.
// Returns the number of specials (≤ PBQ_SK_MAXSPECIAL, else sets error).
__device__ int sk_find_specials(const SketchArgs& a, long chunk, uint64_t* sp_pos, uint64_t* sp_next,
                                int* warp_cnt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int PER = PBQ_SK_CHUNK / PBQ_SK_THREADS;  // 8 consecutive positions per thread
  const uint64_t p0 = uint64_t(chunk) * PBQ_SK_CHUNK + uint64_t(tid) * PER;
  unsigned mask = 0;
#pragma unroll
  for (int b = 0; b < PER / 4; ++b) {
    const Philox4x64 blk = philox4x64_10((p0 >> 2) + b + 1, a.k0, a.k1);
#pragma unroll
    for (int w = 0; w < 4; ++w)
      if (!zig_fast(blk.x[w])) mask |= 1u << (b * 4 + w);
  }
  const int mine = __popc(mask);
  // block exclusive scan of counts (thread order == position order)
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_cnt[warp] = incl;
  __syncthreads();
  int wbase = 0, total = 0;
  for (int w = 0; w < PBQ_SK_THREADS / 32; ++w) {
    if (w < warp) wbase += warp_cnt[w];
    total += warp_cnt[w];
  }
  int off = wbase + incl - mine;
  for (int j = 0; j < PER; ++j)
    if (mask & (1u << j)) {
      if (off < PBQ_SK_MAXSPECIAL) sp_pos[off] = p0 + j;
      ++off;
    }
  __syncthreads();
  if (total > PBQ_SK_MAXSPECIAL) {
    if (tid == 0) atomicExch(a.error, 1);
    total = PBQ_SK_MAXSPECIAL;
  }
  for (int i = tid; i < total; i += PBQ_SK_THREADS) sp_next[i] = zig_resolve(sp_pos[i], a.k0, a.k1, nullptr);
  __syncthreads();
  return total;
}

// Walk the start chain of one chunk from entry position s.
__device__ __forceinline__ void sk_walk(uint64_t s, uint64_t cend, const uint64_t* sp_pos, const uint64_t* sp_next,
                                        int nsp, int& count, uint64_t& exit_pos) {
  int c = 0;
  for (int i = 0; i < nsp; ++i) {
    const uint64_t sp = sp_pos[i];
    if (sp < s) continue;
    if (sp >= cend) break;
    c += int(sp - s) + 1;
    s = sp_next[i];
    if (s >= cend) break;
  }
  if (s < cend) {
    c += int(cend - s);
    s = cend;
  }
  count = c;
  exit_pos = s;
}

__global__ void __launch_bounds__(PBQ_SK_THREADS) sketch_k1(SketchArgs a) {
  __shared__ uint64_t sp_pos[PBQ_SK_MAXSPECIAL], sp_next[PBQ_SK_MAXSPECIAL];
  __shared__ int warp_cnt[PBQ_SK_THREADS / 32];
  __shared__ uint64_t exits_s[PBQ_SK_E];
  const long chunk = blockIdx.x;
  const int nsp = sk_find_specials(a, chunk, sp_pos, sp_next, warp_cnt);
  const uint64_t cstart = uint64_t(chunk) * PBQ_SK_CHUNK, cend = cstart + PBQ_SK_CHUNK;
  const int tid = threadIdx.x;
  if (tid < PBQ_SK_E) {
    int cnt;
    uint64_t ex;
    sk_walk(cstart + tid, cend, sp_pos, sp_next, nsp, cnt, ex);
    a.counts[chunk * PBQ_SK_E + tid] = cnt;
    exits_s[tid] = ex;
  }
  __syncthreads();
  if (tid == 0) {
    bool merged = true;
    for (int e = 1; e < PBQ_SK_E; ++e) merged &= (exits_s[e] == exits_s[0]);
    const uint64_t off = exits_s[0] - cend;
    if (!merged || off >= uint64_t(PBQ_SK_E)) atomicExch(a.error, 2);
    a.exits[chunk] = int(off < uint64_t(PBQ_SK_E) ? off : 0);
  }
}

// Single-CTA scan: entry offsets and exclusive prefix of per-chunk counts.
__global__ void __launch_bounds__(1024) sketch_k2(SketchArgs a) {
  __shared__ long warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long n = a.n_chunks;
  const long per = (n + 1023) / 1024;
  const long c0 = tid * per, c1 = min(n, c0 + per);
  long local = 0;
  for (long c = c0; c < c1; ++c) {
    const int e = (c == 0) ? 0 : a.exits[c - 1];
    local += a.counts[c * PBQ_SK_E + e];
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
  for (long c = c0; c < c1; ++c) {
    const int e = (c == 0) ? 0 : a.exits[c - 1];
    a.entry[c] = e;
    a.base[c] = run;
    run += a.counts[c * PBQ_SK_E + e];
  }
  if (tid == 1023) {
    long total = 0;
    for (int w = 0; w < 32; ++w) total += warp_tot[w];
    if (total < a.first + a.count) atomicExch(a.error, 3);
  }
}

__global__ void __launch_bounds__(PBQ_SK_THREADS) sketch_k3(SketchArgs a) {
  __shared__ uint64_t sp_pos[PBQ_SK_MAXSPECIAL], sp_next[PBQ_SK_MAXSPECIAL];
  __shared__ int warp_cnt[PBQ_SK_THREADS / 32];
  __shared__ unsigned char is_start[PBQ_SK_CHUNK];
  const long chunk = blockIdx.x;
  const long base = a.base[chunk];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // chunk entirely outside the requested normal range: nothing to emit
  const int cnt_here = a.counts[chunk * PBQ_SK_E + a.entry[chunk]];
  if (base >= a.first + a.count || base + cnt_here <= a.first) return;
  const int nsp = sk_find_specials(a, chunk, sp_pos, sp_next, warp_cnt);
  const uint64_t cstart = uint64_t(chunk) * PBQ_SK_CHUNK, cend = cstart + PBQ_SK_CHUNK;
  for (int i = tid; i < PBQ_SK_CHUNK; i += PBQ_SK_THREADS) is_start[i] = (i >= a.entry[chunk]) ? 1 : 0;
  __syncthreads();
  if (tid == 0) {
    // clear the positions a special draw consumes beyond its own
    uint64_t s = cstart + a.entry[chunk];
    for (int i = 0; i < nsp; ++i) {
      const uint64_t sp = sp_pos[i];
      if (sp < s) {
        continue;  // consumed by an earlier normal (already cleared)
      }
      const uint64_t nx = sp_next[i];
      for (uint64_t q = sp + 1; q < nx && q < cend; ++q) is_start[q - cstart] = 0;
      s = nx;
      if (s >= cend) break;
    }
  }
  __syncthreads();
  constexpr int PER = PBQ_SK_CHUNK / PBQ_SK_THREADS;
  int mine = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) mine += is_start[tid * PER + j];
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  __syncthreads();
  if (lane == 31) warp_cnt[warp] = incl;
  __syncthreads();
  int wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += warp_cnt[w];
  long idx = base + wbase + incl - mine;
  const uint64_t p0 = cstart + uint64_t(tid) * PER;
#pragma unroll
  for (int b = 0; b < PER / 4; ++b) {
    const Philox4x64 blk = philox4x64_10((p0 >> 2) + b + 1, a.k0, a.k1);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int j = b * 4 + w;
      if (!is_start[tid * PER + j]) continue;
      if (idx >= a.first && idx < a.first + a.count) {
        const uint64_t r = blk.x[w];
        double v;
        if (zig_fast(r)) v = zig_fast_value(r);
        else zig_resolve(p0 + j, a.k0, a.k1, &v);
        const long rel = idx - a.first;
        a.out[(rel / a.cols) * a.ldo + rel % a.cols] = v;
      }
      ++idx;
    }
  }
}

}  // namespace pbq
