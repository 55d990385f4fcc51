// Latency of the 32×32 diagonal-block kernels of cholqr_factor_kernel
// (one warp): Cholesky, triangular inverse, and variants.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2103_07245_b200/csrc/cholqr_f64.cuh"
using namespace pbq;

template <int V>
__global__ void bench(double* out, const double* g, int iters, long long* cyc) {
  __shared__ double S[32 * CQ_LD], X[32 * CQ_LD];
  __shared__ __align__(16) double RB[64];
  const int lane = threadIdx.x;
  long long t0 = 0, t1 = 0;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = 0; i < 32; ++i) S[i * CQ_LD + lane] = g[i * 32 + lane];
    __syncwarp();
    if (it == 1) t0 = clock64();
    if (V == 0 || V == 2) cq_chol_inv32_warp(S, X, RB);
    __syncwarp();
    if (V == 1) { double y = fast_rsqrt(S[lane * CQ_LD + lane] + 1.0); S[lane] = y; }
    __syncwarp();
    acc += S[lane * CQ_LD + lane] + X[lane];
  }
  t1 = clock64();
  out[lane] = acc;
  if (lane == 0) *cyc = (t1 - t0) / (iters - 1);
}

int main2();
int main3();
int main() {
  main2();
  main3();
  double h[1024];
  // SPD: G = I*32 + small
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *g, *o;
  long long* c;
  cudaMalloc(&g, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  cudaMemcpy(g, h, 8192, cudaMemcpyHostToDevice);
  long long cy;
  const char* nm[] = {"chol+inv", "rsqrt", "chol+inv"};
  bench<0><<<1, 32>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[0], cy);
  bench<1><<<1, 32>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[1], cy);
  bench<2><<<1, 32>>>(o, g, 50, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", nm[2], cy);
  return 0;
}
// accuracy of fast_rsqrt vs 1/sqrt (compiled into the same binary)
__global__ void acc_rsqrt(double* maxrel) {
  double m = 0;
  for (int i = 0; i < 100000; ++i) {
    const double x = exp2(-300.0 + 600.0 * (i * 0.00001 + threadIdx.x * 1e-7));
    const double a = fast_rsqrt(x), b = 1.0 / sqrt(x);
    m = fmax(m, fabs(a - b) / b);
  }
  maxrel[threadIdx.x] = m;
}
int main2() {
  double* d; cudaMalloc(&d, 32 * 8); acc_rsqrt<<<1, 32>>>(d); double h[32]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
  double m = 0; for (int i = 0; i < 32; ++i) m = m > h[i] ? m : h[i];
  printf("fast_rsqrt max rel err vs 1/sqrt: %.3e (u = 1.1e-16)\n", m);
  return 0;
}

// Environment of cholqr_factor_kernel: 256 threads, launch bounds (256, 1),
// large dynamic shared memory, warp 0 runs the diagonal block while the other
// warps wait at a CTA barrier.
template <int MODE>
__global__ void __launch_bounds__(256, 1) bench_env(double* out, const double* g, int iters, long long* cyc,
                                                      int* flag) {
  extern __shared__ __align__(16) double dsm[];
  double* S = dsm;
  double* X = dsm + 32 * CQ_LD;
  __shared__ __align__(16) double RB[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long tot = 0;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE >= 1) {  // poll like cq_wait (acquire → L1 invalidate)
      if (threadIdx.x == 0) (void)ld_acquire(flag);
      __syncthreads();
    }
    if (MODE == 3) {  // a few nanosleep polls before the factorization
      for (int r = 0; r < 4; ++r) __nanosleep(64);
      __syncthreads();
    }
    if (MODE == 2) {  // fence + release store by thread 0 (publish)
      out[threadIdx.x & 31] = 1.0;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release(flag, it);
    }
    if (warp == 0) {
      for (int i = 0; i < 32; ++i) S[i * CQ_LD + lane] = g[i * 32 + lane];
      __syncwarp();
      const long long t0 = clock64();
      cq_chol_inv32_warp(S, X, RB);
      const long long t1 = clock64();
      if (it > 0) tot += t1 - t0;
      acc += S[lane * CQ_LD + lane] + X[lane];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *cyc = tot / (iters - 1);
  if (warp == 0) out[lane] = acc;
}
int main3() {
  double h[1024];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *g, *o;
  long long* c;
  cudaMalloc(&g, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  cudaMemcpy(g, h, 8192, cudaMemcpyHostToDevice);
  int* fl; cudaMalloc(&fl, 4); cudaMemset(fl, 0, 4);
  const int smem = 200000;
  cudaFuncSetAttribute(bench_env<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench_env<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench_env<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long cy;
  bench_env<0><<<1, 256, smem>>>(o, g, 20, c, fl); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("env: plain %lld cycles\n", cy);
  bench_env<1><<<1, 256, smem>>>(o, g, 20, c, fl); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("env: + acquire poll %lld cycles\n", cy);
  bench_env<2><<<1, 256, smem>>>(o, g, 20, c, fl); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("env: + acquire + fence + release %lld cycles (%s)\n", cy, cudaGetErrorString(cudaGetLastError()));
  cudaFuncSetAttribute(bench_env<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench_env<3><<<1, 256, smem>>>(o, g, 20, c, fl); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("env: + acquire + nanosleep %lld cycles (%s)\n", cy, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
