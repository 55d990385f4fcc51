// Shared device helpers for the PbP-QLP sm_100a kernels.
//
// FP64 tensor math on sm_100a is the warp-level DMMA.8x8x4 instruction
// (`mma.sync.aligned.m8n8k4.row.col.f64`); tcgen05/UMMA has no f64 kind, so the
// FP64 path is register MMA fed from shared memory.  The GEMMs stage their
// tiles with the Tensor Memory Accelerator (cp.async.bulk.tensor into an
// mbarrier ring, gemm_tma_f64.cuh; the default) or, as the fallback, with
// cp.async (LDGSTS) multi-buffering (gemm_f64.cuh).  See DESIGN.md §3.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pbq {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy global->shared; bytes beyond `src_bytes` are zero-filled.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- mbarrier + bulk async copy (cp.async.bulk, sm_90+) ----------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on `bar` once all cp.async copies issued so far by this thread have
// landed (the barrier's expected count includes this arrival)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// bytes must be a multiple of 16; src/dst 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor is
// still running; pdl_wait() blocks until the predecessor grid has completed
// and its memory is visible (a no-op without a programmatic predecessor).
// pdl_trigger() lets this kernel's own dependents start launching early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int atom_add_release(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Reciprocal for dependency chains: MUFU approximation + two Newton steps
// (~1 ulp; ~70 cycles instead of ~250 for an IEEE division on sm_100a).
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// 1/sqrt(d) for finite d > 0: rsqrt.approx (MUFU, ~2^-20 relative) + one
// third-order step: e = 1 − d·y², y ← y + y·e·(1/2 + 3e/8), error O(ε³) →
// 2.6e-16 max relative, the same as two Newton steps, with a dependent chain
// of 4 FP64 operations instead of 6 (the 32 pivots of a diagonal Cholesky
// are a chain of these: 3541 → 3059 cycles, tools/microbench/chol32_2warp.cu).
__device__ __forceinline__ double fast_rsqrt(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d * y, y, 1.0);
  const double t = fma(0.375, e, 0.5);
  return fma(y * e, t, y);
}

// Tensor memory (TMEM) as a second-level FP64 accumulator.  tcgen05 has no
// f64 MMA kind, so the DMMA GEMMs leave the SM's 256 KB of TMEM unused; they
// park a running sum there (blocked summation, see gemm_tma_f64.cuh).  Each
// thread moves its own 32-bit words: lane ℓ of warp w owns TMEM lane
// 32·(w mod 4) + ℓ (the 32x32b shape), 16 consecutive columns per access.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// 8 doubles (16 words) per thread: v[i] ↔ columns 2i, 2i+1 (lo, hi words)
__device__ __forceinline__ void tmem_st8d(uint32_t taddr, const double (&v)[8]) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    w[2 * i] = __double2loint(v[i]);
    w[2 * i + 1] = __double2hiint(v[i]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};\n" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld8d(uint32_t taddr, double (&v)[8]) {
  uint32_t w[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;\n"  // in the same statement: no use of w can be hoisted above it
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]),
        "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __hiloint2double(int(w[2 * i + 1]), int(w[2 * i]));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// True when the IEEE-754 binary64 exponent field is all ones (Inf or NaN).
__device__ __forceinline__ bool nonfinite_bits(double x) {
  return ((__double_as_longlong(x) >> 52) & 0x7ff) == 0x7ff;
}

// Software grid barrier for persistent (cooperatively launched) kernels.
// `counter` must be zeroed before the launch; `*generation` counts barriers
// already passed by this CTA.  All writes made before the barrier by any CTA
// are visible after it to loads that bypass L1 (ld.global.cg / acquire).
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int& generation,
                                             unsigned long long* wait_ns = nullptr) {
  __threadfence();
  __syncthreads();
  generation += 1;
  if (threadIdx.x == 0) {
    unsigned long long t0 = 0;
    if (wait_ns) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    atom_add_release(counter, 1u);
    const unsigned int target = generation * gridDim.x;
    while (ld_acquire_u32(counter) < target) {
    }
    if (wait_ns) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
      wait_ns[blockIdx.x] += t1 - t0;  // per-CTA spin time (profiling only)
    }
  }
  __syncthreads();
}

// (tm, tn) of the t-th tile with tm <= tn in row-major order
__device__ __forceinline__ void upper_tile(int t, int tiles, int& tm, int& tn) {
  tm = 0;
  while (t >= tiles - tm) {
    t -= tiles - tm;
    ++tm;
  }
  tn = tm + t;
}

__host__ __device__ constexpr long ceil_div(long a, long b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ long lmin(long a, long b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ long lmax(long a, long b) { return a > b ? a : b; }

}  // namespace pbq
