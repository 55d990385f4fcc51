// Fused AᵀX exchange over NVLink peer memory (the allreduce(sum)
// of the per-rank partials C_g = A_gᵀ·X_g, reference `_PassCounter.apply_t`
// across row shards, algorithms.py:182-184).
//
// Instead of GEMM → ncclAllReduce, the GEMM's epilogue is the first half of
// a reduce-scatter: rows of C are split into G slices of S rows (S a
// multiple of the 128-row tile), slice r owned by rank r, and every finished
// output tile of rank g is stored straight into rank r's landing buffer
// (slot g) through the peer mapping (symmetric memory), followed by one
// system-scope release increment of rank r's tile counter.  The tiles cross
// NVLink while the GEMM is still computing the next ones.  Then:
//   xchg_reduce_kernel  (rank r) waits for its tile count, sums the G slots
//                        of its slice in slot order (so every rank ends with
//                        the same bits), stores the slice into every rank's C
//                        (all-gather by peer stores) and increments every
//                        rank's done counter;
//   xchg_wait_kernel    waits until all G slices have arrived.
// Counters only grow: the host passes targets epoch·(expected per call), so
// nothing is reset between calls.  With G = 1 the same kernels run against
// the rank's own buffers.
#pragma once
#include "common.cuh"

namespace pbq {

// CTAs of xchg_reduce_kernel (PBQ_XCHG_CTAS, include/pbq.h): each increments
// every rank's done counter once, so a call adds PBQ_XCHG_CTAS·G to each
#ifndef PBQ_XCHG_CTAS
#define PBQ_XCHG_CTAS 64
#endif

__device__ __forceinline__ unsigned int ld_acquire_sys_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Epilogue target of the scatter GEMM (GemmArgs::xs): tile rows [m0, m0+BM)
// of the n2×N result go to landing[owner][(rank·S + m0 − owner·S) … ].
struct XchgScatter {
  double* const* land;         // G device pointers (peer-mapped), each G·S×ldl doubles
  unsigned int* const* cnt;    // G device pointers to the owners' tile counters
  long S, ldl;
  int rank, world;
};

// Spin until *p ≥ target, at most `timeout_ns` (pbq_set_p2p_timeout_ms,
// default 20 s): a peer that never arrives (a broken peer mapping, a rank
// that died) must not hang the GPU.  On timeout *status |= 1 (the host
// raises and poisons the exchange); the caller then proceeds.
#define PBQ_XCHG_TIMEOUT_NS 20000000000ull
__device__ __forceinline__ void xchg_spin(const unsigned int* p, unsigned int target, unsigned int* status,
                                          unsigned long long timeout_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_acquire_sys_u32(p) < target) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicOr(status, 1u);
      return;
    }
    __nanosleep(256);
  }
}

// Sum of the G landing slots of this rank's slice → every rank's C.  The
// counter block of a rank is [tile count, done count, status].
// One warp per row (rows strided over the grid's warps), lanes over column
// pairs: 16-byte volatile loads of the G slots (written by peers) and 16-byte
// stores to every rank's C, no per-element index division.  ldl and ldc are
// even and the bases 16-byte aligned; an odd n ends in one scalar column.
__global__ void __launch_bounds__(256) xchg_reduce_kernel(const double* __restrict__ land, long ldl, int world, long S,
                                                          long rows, long n, double* const* c_ptrs, long ldc,
                                                          long row0, const unsigned int* cnt, unsigned int target,
                                                          unsigned int* const* done_ptrs,
                                                          unsigned long long timeout_ns) {
  if (threadIdx.x == 0) xchg_spin(cnt, target, const_cast<unsigned int*>(cnt) + 2, timeout_ns);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long warp = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (long(gridDim.x) * blockDim.x) >> 5;
  const long pairs = n >> 1;
  for (long i = warp; i < rows; i += nwarps) {
    const double* src = land + i * ldl;
    const long crow = (row0 + i) * ldc;
    for (long jp = lane; jp < pairs; jp += 32) {
      double2 s = make_double2(0.0, 0.0);
      for (int g = 0; g < world; ++g) {  // slot order: the same bits on every rank
        const double2 v = __ldcv(reinterpret_cast<const double2*>(src + long(g) * S * ldl) + jp);
        s.x += v.x;
        s.y += v.y;
      }
      for (int p = 0; p < world; ++p) reinterpret_cast<double2*>(c_ptrs[p] + crow)[jp] = s;
    }
    if ((n & 1) && lane == 0) {
      double s = 0.0;
      for (int g = 0; g < world; ++g) s += __ldcv(src + long(g) * S * ldl + n - 1);
      for (int p = 0; p < world; ++p) c_ptrs[p][crow + n - 1] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p) red_release_sys_add(done_ptrs[p], 1u);
  }
}

// Small collectives on the same symmetric buffers (the d×d Gram allreduces
// and the all-gather of orth(C)'s row slices):
//   p2p_push_kernel: src (n doubles) → dst_ptrs[p] + rank·slot for every rank
//     p, then one release increment of every rank's counter per CTA;
//   p2p_sum_kernel:  wait for the counter, out = Σ_g slots[g·slot] in slot
//     order (the same bits on every rank).
// An all-gather is a push with slot = the slice size into C itself plus a
// wait (xchg_wait_kernel on that counter).  Both move 16-byte pairs when
// every base and the slot are 16-byte aligned (checked by the host), with a
// scalar tail for odd n.
template <bool VEC>
__global__ void __launch_bounds__(256) p2p_push_kernel(const double* __restrict__ src, long n, double* const* dst_ptrs,
                                                       long slot, int rank, int world, unsigned int* const* cnt_ptrs) {
  const long t0 = long(blockIdx.x) * blockDim.x + threadIdx.x, nt = long(gridDim.x) * blockDim.x;
  if (VEC) {
    const long pairs = n >> 1;
    for (long i = t0; i < pairs; i += nt) {
      const double2 v = reinterpret_cast<const double2*>(src)[i];
      for (int p = 0; p < world; ++p) reinterpret_cast<double2*>(dst_ptrs[p] + long(rank) * slot)[i] = v;
    }
    if ((n & 1) && t0 == 0)
      for (int p = 0; p < world; ++p) dst_ptrs[p][long(rank) * slot + n - 1] = src[n - 1];
  } else {
    for (long i = t0; i < n; i += nt) {
      const double v = src[i];
      for (int p = 0; p < world; ++p) dst_ptrs[p][long(rank) * slot + i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p) red_release_sys_add(cnt_ptrs[p], 1u);
  }
}

template <bool VEC>
__global__ void __launch_bounds__(256) p2p_sum_kernel(const double* __restrict__ slots, long slot, int world, long n,
                                                      double* __restrict__ out, const unsigned int* cnt,
                                                      unsigned int target, unsigned int* status,
                                                      unsigned long long timeout_ns) {
  if (threadIdx.x == 0) xchg_spin(cnt, target, status, timeout_ns);
  __syncthreads();
  const long t0 = long(blockIdx.x) * blockDim.x + threadIdx.x, nt = long(gridDim.x) * blockDim.x;
  if (VEC) {
    const long pairs = n >> 1;
    for (long i = t0; i < pairs; i += nt) {
      double2 s = make_double2(0.0, 0.0);
      for (int g = 0; g < world; ++g) {
        const double2 v = __ldcv(reinterpret_cast<const double2*>(slots + long(g) * slot) + i);
        s.x += v.x;
        s.y += v.y;
      }
      reinterpret_cast<double2*>(out)[i] = s;
    }
    if ((n & 1) && t0 == 0) {
      double s = 0.0;
      for (int g = 0; g < world; ++g) s += __ldcv(slots + long(g) * slot + n - 1);
      out[n - 1] = s;
    }
  } else {
    for (long i = t0; i < n; i += nt) {
      double s = 0.0;
      for (int g = 0; g < world; ++g) s += __ldcv(slots + long(g) * slot + i);
      out[i] = s;
    }
  }
}

__global__ void p2p_wait_kernel(const unsigned int* cnt, unsigned int target, unsigned int* status,
                                unsigned long long timeout_ns) {
  if (threadIdx.x == 0) xchg_spin(cnt, target, status, timeout_ns);
  __syncthreads();
}

__global__ void xchg_wait_kernel(const unsigned int* done, unsigned int target, unsigned long long timeout_ns) {
  if (threadIdx.x == 0) xchg_spin(done, target, const_cast<unsigned int*>(done) + 1, timeout_ns);
  __syncthreads();
}

}  // namespace pbq
