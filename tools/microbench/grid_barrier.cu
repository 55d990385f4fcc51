// Grid-barrier latency microbenchmark (sm_100a): the per-column cost floor of
// the cooperative Householder QR.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 grid_barrier.cu -o grid_barrier
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mode 0: all-thread fence + counter;  1: CG-style thread-0 fence + counter;
// 2: red.release counter (no extra fence);  3: per-CTA flags, all-to-all poll;
// 4: cooperative_groups grid.sync()
__global__ void bar_kernel(unsigned* counter, unsigned* flags, int iters, int mode, double* sink) {
  unsigned gen = 0;
  double acc = threadIdx.x;
  cg::grid_group grid = cg::this_grid();
  for (int it = 0; it < iters; ++it) {
    acc = acc * 1.0000001 + 1.0;
    if (mode == 4) {
      grid.sync();
      continue;
    }
    if (mode == 0) __threadfence();
    __syncthreads();
    ++gen;
    if (mode <= 2) {
      if (threadIdx.x == 0) {
        if (mode == 1) __threadfence();
        if (mode == 2) red_rel(counter, 1u);
        else atomicAdd(counter, 1u);
        const unsigned target = gen * gridDim.x;
        while (ld_acq(counter) < target) {
        }
      }
    } else {
      if (threadIdx.x == 0) st_rel(flags + blockIdx.x * 32, gen);
      for (unsigned c = threadIdx.x; c < gridDim.x; c += blockDim.x)
        while (ld_acq(flags + c * 32) < gen) {
        }
    }
    __syncthreads();
  }
  if (acc == 0.5) sink[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *counter, *flags;
  double* sink;
  cudaMalloc(&counter, 4);
  cudaMalloc(&flags, 4 * 32 * 1024);
  cudaMalloc(&sink, 8);
  const int iters = 2000;
  for (int grid : {16, 64, 148}) {
    for (int mode = 0; mode < 5; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(counter, 0, 4);
        cudaMemset(flags, 0, 4 * 32 * 1024);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        int it = iters;
        void* args[] = {&counter, &flags, &it, &mode, &sink};
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)bar_kernel, grid, 256, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("{\"grid\": %d, \"mode\": %d, \"us_per_barrier\": %.3f}\n", grid, mode, best * 1e3 / iters);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
