// Where the 32×32 diagonal Cholesky + inverse of cholqr_factor_kernel spends
// its ~3.5 µs: the production two-warp routine against stripped variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o chol32_2warp chol32_2warp.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CQ_CHOL_TIMING
#include "../../paper_2103_07245_b200/csrc/cholqr_f64.cuh"
using namespace pbq;

// B: warp 0's R elimination alone (no handshake with warp 1, no inverse)
__device__ __noinline__ void chol_r_only(double* S, double* rowbuf) {
  const int lane = threadIdx.x & 31;
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = S[i * CQ_LD + lane];
  double piv = v[0];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dk = __shfl_sync(0xffffffffu, piv, k);
    const double inv = fast_rsqrt(dk);
    const double rkj = (lane >= k) ? v[k] * inv : 0.0;
    v[k] = rkj;
    if (k + 1 < 32) piv = fma(-rkj, rkj, v[k + 1]);
    double* rb = rowbuf + (k & 1) * 32;
    rb[lane] = rkj;
    __syncwarp();
#pragma unroll
    for (int i2 = (k + 1) & ~1; i2 < 32; i2 += 2) {
      const double2 r2 = *reinterpret_cast<const double2*>(rb + i2);
      if (i2 > k) v[i2] = fma(-r2.x, rkj, v[i2]);
      if (i2 + 1 > k && i2 + 1 < 32) v[i2 + 1] = fma(-r2.y, rkj, v[i2 + 1]);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) S[i * CQ_LD + lane] = (i <= lane) ? v[i] : 0.0;
}

// 1/sqrt(d) with one third-order (Householder) step instead of two Newton steps:
// e = 1 − d·y², y ← y + y·e·(1/2 + 3e/8): error ε³ from the MUFU approximation
__device__ __forceinline__ double rsqrt3(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d * y, y, 1.0);
  const double t = fma(0.375, e, 0.5);
  return fma(y * e, t, y);
}
__device__ __noinline__ double chain3(double d) {
  const int lane = threadIdx.x & 31;
  double piv = d + lane;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dk = __shfl_sync(0xffffffffu, piv, k);
    const double inv = rsqrt3(dk);
    const double r = d * inv;
    piv = fma(-r, r, piv + 1.0);
  }
  return piv;
}
__global__ void acc3(double* out) {
  double m2 = 0, m3 = 0, ma = 0;
  for (int i = 0; i < 200000; ++i) {
    const double x = exp2(-250.0 + 500.0 * (i * 0.000005 + threadIdx.x * 1.3e-7));
    const double b = 1.0 / sqrt(x);
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
    ma = fmax(ma, fabs(y0 - b) / b);
    m2 = fmax(m2, fabs(fast_rsqrt(x) - b) / b);
    m3 = fmax(m3, fabs(rsqrt3(x) - b) / b);
  }
  out[3 * threadIdx.x] = ma;
  out[3 * threadIdx.x + 1] = m2;
  out[3 * threadIdx.x + 2] = m3;
}

// C: the dependent chain alone: shuffle → rsqrt → mul → fma, 32 times
__device__ __noinline__ double chain_only(double d) {
  const int lane = threadIdx.x & 31;
  double piv = d + lane;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dk = __shfl_sync(0xffffffffu, piv, k);
    const double inv = fast_rsqrt(dk);
    const double r = d * inv;
    piv = fma(-r, r, piv + 1.0);
  }
  return piv;
}

// E: R part with the row broadcast by shuffles (no shared memory)
__device__ __noinline__ void chol_r_shfl(double* S) {
  const int lane = threadIdx.x & 31;
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = S[i * CQ_LD + lane];
  double piv = v[0];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dk = __shfl_sync(0xffffffffu, piv, k);
    const double inv = fast_rsqrt(dk);
    const double rkj = (lane >= k) ? v[k] * inv : 0.0;
    v[k] = rkj;
    if (k + 1 < 32) piv = fma(-rkj, rkj, v[k + 1]);
#pragma unroll
    for (int i = k + 1; i < 32; ++i) v[i] = fma(-__shfl_sync(0xffffffffu, rkj, i), rkj, v[i]);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) S[i * CQ_LD + lane] = (i <= lane) ? v[i] : 0.0;
}

// F: warp 0 of the pipelined routine alone (no publication, no warp 1)
__device__ __noinline__ void chol_r_pipe(double* S) {
  const int lane = threadIdx.x & 31;
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = S[i * CQ_LD + lane];
  double piv = v[0];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double dk = __shfl_sync(0xffffffffu, piv, k);
    if (k >= 1) {
      const double rp = v[k - 1];
      const double* rb = S + (k - 1) * CQ_LD;
#pragma unroll
      for (int i2 = (k + 1) & ~1; i2 < 32; i2 += 2) {
        const double2 r2 = *reinterpret_cast<const double2*>(rb + i2);
        if (i2 > k) v[i2] = fma(-r2.x, rp, v[i2]);
        if (i2 + 1 > k && i2 + 1 < 32) v[i2 + 1] = fma(-r2.y, rp, v[i2 + 1]);
      }
    }
    const double inv = fast_rsqrt(dk);
    const double rkj = (lane >= k) ? v[k] * inv : 0.0;
    v[k] = rkj;
    if (k + 1 < 32) {
      piv = fma(-rkj, rkj, v[k + 1]);
      v[k + 1] = fma(-__shfl_sync(0xffffffffu, rkj, k + 1), rkj, v[k + 1]);
    }
    S[k * CQ_LD + lane] = rkj;
    __syncwarp();
  }
}

template <int V>
__global__ void bench(double* out, const double* g, int iters, long long* cyc) {
  __shared__ double S[32 * CQ_LD], X[32 * CQ_LD];
  __shared__ __align__(16) double RB[2 * CQ_RB2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long tot = 0;
  double acc = 0;
  if (V == 6) cq_chol_setup(RB);
  for (int it = 0; it < iters; ++it) {
    if (warp == 0)
      for (int i = 0; i < 32; ++i) S[i * CQ_LD + lane] = g[i * 32 + lane];
    __syncthreads();
    const long long t0 = clock64();
    if (V == 0) cq_chol_inv32_2warp(S, X, RB);
    if (V == 1 && warp == 0) cq_chol_inv32_warp(S, X, RB);
    if (V == 2 && warp == 0) chol_r_only(S, RB);
    if (V == 3 && warp == 0) acc += chain_only(S[lane]);
    if (V == 4 && warp == 0) chol_r_shfl(S);
    if (V == 5 && warp == 0) acc += chain3(S[lane]);
    if (V == 6) cq_chol_inv32_pipe(S, X, RB);
    if (V == 7 && warp == 0) chol_r_pipe(S);
    __syncthreads();
    const long long t1 = clock64();
    if (it > 0) tot += t1 - t0;
    if (V == 6 && it == iters - 1 && threadIdx.x == 0)
      printf("  pipelined, last call: warp 0 done at %lld, warp 1 at %lld, both through the barrier at %lld cycles\n",
             cq_chol_t[0] - t0, cq_chol_t[1] - t0, t1 - t0);
    acc += S[lane * CQ_LD + lane];
  }
  if (threadIdx.x == 0) *cyc = tot / (iters - 1);
  out[threadIdx.x] = acc;
}

// bitwise comparison of the pipelined routine with the two-warp one
__global__ void verify(const double* g, int* diff) {
  __shared__ double S0[32 * CQ_LD], X0[32 * CQ_LD], S1[32 * CQ_LD], X1[32 * CQ_LD];
  __shared__ __align__(16) double RB[2 * CQ_RB2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0)
    for (int i = 0; i < 32; ++i) S0[i * CQ_LD + lane] = S1[i * CQ_LD + lane] = g[i * 32 + lane];
  __syncthreads();
  cq_chol_inv32_2warp(S0, X0, RB);
  __syncthreads();
  cq_chol_setup(RB);
  __syncthreads();
  for (int rep = 0; rep < 3; ++rep) {  // three calls: both phase parities
    if (warp == 0)
      for (int i = 0; i < 32; ++i) S1[i * CQ_LD + lane] = g[i * 32 + lane];
    __syncthreads();
    cq_chol_inv32_pipe(S1, X1, RB);
    __syncthreads();
  }
  int d = 0;
  if (warp == 0)
    for (int i = 0; i < 32; ++i) {
      d += __double_as_longlong(S0[i * CQ_LD + lane]) != __double_as_longlong(S1[i * CQ_LD + lane]);
      d += __double_as_longlong(X0[i * CQ_LD + lane]) != __double_as_longlong(X1[i * CQ_LD + lane]);
    }
  if (d) atomicAdd(diff, d);
}

int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *g, *o;
  long long* c;
  cudaMalloc(&g, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  cudaMemcpy(g, h, 8192, cudaMemcpyHostToDevice);
  long long cy;
  const char* nm[] = {"2-warp chol+inv (production)", "1-warp chol+inv", "R part only (smem row)",
                      "dependent chain only", "R part only (shuffle row)"};
  bench<0><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[0], cy);
  bench<1><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[1], cy);
  bench<2><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[2], cy);
  bench<3><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[3], cy);
  bench<4><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[4], cy);
  bench<5><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("dependent chain, rsqrt3: %lld cycles\n", cy);
  bench<6><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("2-warp chol+inv, pipelined: %lld cycles\n", cy);
  bench<7><<<1, 64>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("R part only, pipelined: %lld cycles\n", cy);
  int* df; cudaMalloc(&df, 4); cudaMemset(df, 0, 4);
  verify<<<1, 64>>>(g, df); int hd = -1; cudaMemcpy(&hd, df, 4, cudaMemcpyDeviceToHost);
  printf("pipelined vs two-warp routine: %d differing words (S and X, bitwise)\n", hd);
  double* a3; cudaMalloc(&a3, 96 * 8); acc3<<<1, 32>>>(a3); double ha[96]; cudaMemcpy(ha, a3, 96 * 8, cudaMemcpyDeviceToHost);
  double ma = 0, m2 = 0, m3 = 0;
  for (int i = 0; i < 32; ++i) { ma = fmax(ma, ha[3 * i]); m2 = fmax(m2, ha[3 * i + 1]); m3 = fmax(m3, ha[3 * i + 2]); }
  printf("max rel err vs 1/sqrt: rsqrt.approx %.3e, fast_rsqrt (2 Newton) %.3e, rsqrt3 (1 cubic) %.3e\n", ma, m2, m3);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
