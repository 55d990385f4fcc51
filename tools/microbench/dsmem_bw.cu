// Exchange bandwidth inside a thread-block cluster (design input for the
// Jacobi SVD kernel, svd_f64.cuh): per-SM throughput of
//   (a) DSMEM: every thread stores 16-byte vectors into the NEXT CTA's shared
//       memory (st.shared::cluster.v2.f64), then loads them back locally;
//   (b) DSMEM loads from the next CTA (ld.shared::cluster.v2.f64);
//   (c) L2: stores to a global buffer + cluster barrier + loads of the block
//       written by the neighbour CTA;
//   (d) barrier.cluster arrive.release/wait.acquire latency.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o dsmem_bw dsmem_bw.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS, 1) bench(double* gbuf, unsigned long long* out, int bytes, int reps) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank(), nc = cl.num_blocks();
  const unsigned nxt = (me + 1) % nc;
  const int n2 = bytes / 16;  // double2 per CTA
  double2* loc = reinterpret_cast<double2*>(sm);
  double2* rem = reinterpret_cast<double2*>(cl.map_shared_rank(sm, nxt));
  for (int i = threadIdx.x; i < n2 * 2; i += THREADS) loc[i] = make_double2(i, me);
  csync();
  unsigned long long acc[4] = {0, 0, 0, 0};
  double sink = 0;
  for (int r = 0; r < reps; ++r) {
    // (a) remote stores of `bytes` into the neighbour (second half of its buffer)
    csync();
    unsigned long long t0 = clk();
    for (int i = threadIdx.x; i < n2; i += THREADS) rem[n2 + i] = loc[i];
    csync();
    acc[0] += clk() - t0;
    // (b) remote loads of `bytes` from the neighbour
    t0 = clk();
    double2 s = make_double2(0, 0);
    for (int i = threadIdx.x; i < n2; i += THREADS) {
      double2 v = rem[i];
      s.x += v.x;
      s.y += v.y;
    }
    sink += s.x + s.y;
    csync();
    acc[1] += clk() - t0;
    // (c) global store, cluster barrier, load of the neighbour's block
    t0 = clk();
    double2* gme = reinterpret_cast<double2*>(gbuf) + size_t(blockIdx.x) * n2;
    double2* gnx = reinterpret_cast<double2*>(gbuf) + size_t(blockIdx.x - me + nxt) * n2;
    for (int i = threadIdx.x; i < n2; i += THREADS) __stcg(gme + i, loc[i]);
    csync();
    for (int i = threadIdx.x; i < n2; i += THREADS) loc[n2 + i] = __ldcg(gnx + i);
    csync();
    acc[2] += clk() - t0;
    // (d) barrier alone
    t0 = clk();
    csync();
    acc[3] += clk() - t0;
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) out[blockIdx.x * 4 + k] = acc[k] / reps;
  }
  if (sink == 12345.678) out[0] = 0;
}

int main() {
  const int reps = 50;
  double* g;
  unsigned long long* o;
  cudaMalloc(&g, size_t(64) << 20);
  cudaMalloc(&o, 1024 * 4 * 8);
  for (int C : {8, 16}) {
    for (int bytes : {4096, 16384, 65536}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = 2 * bytes;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaFuncSetAttribute(bench<512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(bench<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * bytes);
      cudaError_t e = cudaLaunchKernelEx(&cfg, bench<512>, g, o, bytes, reps);
      cudaDeviceSynchronize();
      if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        printf("C=%d bytes=%d: launch failed %s\n", C, bytes, cudaGetErrorString(e));
        continue;
      }
      unsigned long long h[4];
      cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
      printf("C=%2d bytes/CTA=%6d | remote store+barrier %6llu clk (%.1f B/clk) | remote load+barrier %6llu clk "
             "(%.1f B/clk) | L2 store+bar+load+bar %6llu clk (%.1f B/clk) | barrier %llu clk\n",
             C, bytes, h[0], double(bytes) / (h[0] - h[3]), h[1], double(bytes) / (h[1] - h[3]), h[2],
             double(bytes) / (h[2] - 2 * h[3]), h[3]);
    }
  }
  return 0;
}
