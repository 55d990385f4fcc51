// Latency of the building blocks of the cluster Cholesky factor kernel
// (cholqr_cluster.cuh) on an 8-CTA cluster: cluster barrier, DSMEM fetch of
// 1 / 6 blocks of 32×32 doubles, one 32×32×32 DMMA block product by 8 warps,
// and 8 block products split one per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2103_07245_b200/csrc -o cluster_ops cluster_ops.cu
#include <cstdio>
#include "cholqr_cluster_factor_kernel.cu"  // the abandoned single-cluster factor kernel
using namespace pbq;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

// warp-level 32×32×32 product c += Aᵀ·B (A, B staged, ld CQ_LD): 16 8×8 tiles per warp
__device__ __forceinline__ void warp_mma_tn(double (&c)[4][4][2], const double* A, const double* B) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int k0 = 0; k0 < 32; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = A[(k0 + t) * CQ_LD + i * 8 + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = B[(k0 + t) * CQ_LD + j * 8 + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(c[i][j][0], c[i][j][1], a[i], b[j]);
  }
}

__global__ void __launch_bounds__(256, 1) bench(unsigned long long* out, int reps) {
  extern __shared__ __align__(16) double sm[];
  const unsigned me = cqc_rank();
  for (int i = threadIdx.x; i < 16 * CQ_BLK; i += 256) sm[i] = 1e-3 * (i % 97);
  cqc_sync();
  unsigned long long t0, t1, acc[6] = {0};
  double sink = 0;
  for (int r = 0; r < reps; ++r) {
    // 0: cluster barrier
    t0 = clk();
    cqc_sync();
    t1 = clk();
    acc[0] += t1 - t0;
    // 1: fetch 1 block from the next CTA
    {
      const double* src[1] = {sm};
      unsigned rk[1] = {(me + 1) % 8};
      __syncthreads();
      t0 = clk();
      cqc_fetch<1>(sm + 8 * CQ_BLK, src, rk, 1);
      __syncthreads();
      t1 = clk();
      acc[1] += t1 - t0;
    }
    // 2: fetch 6 blocks
    {
      const double* src[6];
      unsigned rk[6];
      for (int q = 0; q < 6; ++q) {
        src[q] = sm + q * CQ_BLK;
        rk[q] = (me + 1 + q) % 8;
      }
      __syncthreads();
      t0 = clk();
      cqc_fetch<6>(sm + 8 * CQ_BLK, src, rk, 6);
      __syncthreads();
      t1 = clk();
      acc[2] += t1 - t0;
    }
    // 3: one block product by 8 warps (cq_mma) + store
    {
      __syncthreads();
      t0 = clk();
      double c[2][2];
      cq_zero(c);
      cq_mma<true, false>(c, sm, sm + CQ_BLK);
      cq_store_acc(sm + 2 * CQ_BLK, c, 1.0);
      __syncthreads();
      t1 = clk();
      acc[3] += t1 - t0;
    }
    // 4: 7 block products in sequence by 8 warps (phase C of the worst CTA)
    {
      __syncthreads();
      t0 = clk();
      for (int q = 0; q < 7; ++q) {
        double c[2][2];
        cq_zero(c);
        cq_mma<true, false>(c, sm + (8 + (q % 6)) * CQ_BLK, sm + CQ_BLK);
        const int rr = cq_row();
        double* g = sm + 2 * CQ_BLK;
        for (int h = 0; h < 2; ++h) {
          g[rr * CQ_LD + cq_col(h)] -= c[h][0];
          g[rr * CQ_LD + cq_col(h) + 1] -= c[h][1];
        }
      }
      __syncthreads();
      t1 = clk();
      acc[4] += t1 - t0;
    }
    // 5: 8 block products, one per warp
    {
      __syncthreads();
      t0 = clk();
      double c[4][4][2] = {};
      const int w = threadIdx.x >> 5;
      warp_mma_tn(c, sm + (8 + (w % 6)) * CQ_BLK, sm + CQ_BLK);
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) sink += c[i][j][0] + c[i][j][1];
      __syncthreads();
      t1 = clk();
      acc[5] += t1 - t0;
    }
  }
  if (threadIdx.x == 0)
    for (int i = 0; i < 6; ++i) out[me * 8 + i] = acc[i] / reps;
  if (sink == 12345.0) out[100] = 1;
  cqc_sync();
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  const size_t smem = 16 * CQ_BLK * sizeof(double);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 8;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(8);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int it = 0; it < 2; ++it) cudaLaunchKernelEx(&cfg, bench, d, 200);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[64];
  cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(e));
  const char* names[6] = {"cluster barrier", "fetch 1 block", "fetch 6 blocks", "1 product (8 warps)",
                          "7 products (8 warps each)", "8 products (1 per warp)"};
  for (int i = 0; i < 6; ++i) printf("%-28s CTA0 %6llu cycles  CTA7 %6llu cycles\n", names[i], h[i], h[56 + i]);
  return 0;
}
