// Cycle counts of the QR kernel's 32×32 redundant algebra (Cholesky, LU,
// log-depth triangular inverse, 32×32 product) on one CTA.  From the repo root:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2103_07245_b200/csrc \
//        tools/microbench/small_algebra.cu -o tools/microbench/small_algebra
#include <cstdio>
#include "qr_f64.cuh"
using namespace pbq;

__global__ void bench(double* out, long long* cyc) {
  __shared__ double G[QR_NB * QR_SLD], M[QR_NB * QR_SLD], X[QR_NB * QR_SLD], Z[QR_NB * QR_SLD], vec[128];
  const int tid = threadIdx.x;
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int i = e / 32, j = e % 32;
    G[i * QR_SLD + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  }
  __syncthreads();
  long long t[5];
  double r = 0;
  t[0] = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    for (int e = tid; e < 32 * 32; e += blockDim.x) M[(e / 32) * QR_SLD + e % 32] = G[(e / 32) * QR_SLD + e % 32];
    __syncthreads();
    r += sm_chol(M, vec);
  }
  t[1] = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    for (int e = tid; e < 32 * 32; e += blockDim.x) M[(e / 32) * QR_SLD + e % 32] = G[(e / 32) * QR_SLD + e % 32];
    __syncthreads();
    sm_lu(M, vec);
  }
  t[2] = clock64();
  for (int rep = 0; rep < 10; ++rep) sm_tri_inv_upper<false, false>(X, M, Z);
  t[3] = clock64();
  for (int rep = 0; rep < 10; ++rep) sm_mm<false, false>(Z, X, M);
  t[4] = clock64();
  out[tid] = r + X[tid] + Z[tid];
  if (tid == 0)
    for (int k = 0; k < 4; ++k) cyc[k] = (t[k + 1] - t[k]) / 10;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 64);
  for (int it = 0; it < 2; ++it) {
    bench<<<1, QR_THREADS>>>(out, cyc);
    cudaDeviceSynchronize();
  }
  printf("{\"chol32\": %lld, \"lu32\": %lld, \"tri_inv32\": %lld, \"mm32\": %lld, \"err\": \"%s\"}\n", cyc[0], cyc[1],
         cyc[2], cyc[3], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
