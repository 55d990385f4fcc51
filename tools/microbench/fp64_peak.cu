// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Measures the denominators for the PbP-QLP roofline (MEASURED_PEAKS.json has
// no FP64 figure). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma884_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5 + threadIdx.x * 1e-10;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma16816_loop(double* out, int iters, double seed) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i * 1e-9 + threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed * 0.5 + i * 1e-9;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
float time_kernel(K kern, int grid, int block, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, iters / 10, 1.0);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d}\n", p.name, sms);
  double* out; CK(cudaMalloc(&out, 64));
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int cps : {1, 2}) {
      int block = 32 * wpb, grid = sms * cps;
      double warps = double(grid) * wpb;
      {
        float ms = time_kernel(dmma884_loop<8>, grid, block, out, iters);
        double fl = warps * iters * 8 * 2.0 * 8 * 8 * 4;
        printf("{\"kind\": \"dmma_m8n8k4\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", wpb, cps, ms, fl / ms / 1e9);
      }
      {
        float ms = time_kernel(dmma16816_loop<4>, grid, block, out, iters / 4);
        double fl = warps * (iters / 4) * 4 * 2.0 * 16 * 8 * 16;
        printf("{\"kind\": \"dmma_m16n8k16\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", wpb, cps, ms, fl / ms / 1e9);
      }
      {
        float ms = time_kernel(dfma_loop<16>, grid, block, out, iters);
        double fl = double(grid) * block * iters * 16 * 2.0;
        printf("{\"kind\": \"dfma\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", wpb, cps, ms, fl / ms / 1e9);
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}
