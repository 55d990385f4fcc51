// Are the FP64 tensor (DMMA) and FP64 FMA (DFMA) pipes separate on B200?
// Half of each CTA's warps issue DMMA.8x8x4, the other half DFMA; if the
// aggregate FLOP rate exceeds the single-pipe peak (~37 TF/s), a GEMM could
// split work across both pipes.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: all DMMA, 1: all DFMA, 2: even DMMA / odd DFMA, 3: even DMMA / odd idle, 4: odd DFMA / even idle
__global__ void mixed(double* out, int iters, double seed, unsigned long long* flops, int iters_fma) {
  const int warp = threadIdx.x >> 5;
  // warp w runs on scheduler w % 4; modes 5/6 put DMMA and DFMA warps on the same scheduler
  const bool grp = ((warp >> 2) & 1) == 0;
  if (MODE == 3 && (warp & 1)) return;
  if (MODE == 4 && !(warp & 1)) return;
  if (MODE == 6 && !grp) return;
  const bool do_mma = MODE == 0 || ((MODE == 2 || MODE == 3) && (warp & 1) == 0) || ((MODE == 5 || MODE == 6) && grp);
  if (!do_mma) iters = iters_fma;
  double s = 0.0;
  if (do_mma) {
    double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
    double c[8][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if ((threadIdx.x & 31) == 0) atomicAdd(flops, (unsigned long long)iters * 8 * 512);
  } else {
    double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = i * 1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = fma(c[i], b, a);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
    if ((threadIdx.x & 31) == 0) atomicAdd(flops, (unsigned long long)iters * 16 * 64);
  }
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
void run(int iters_mma, const char* name, int iters_fma = 20000, int threads = 512) {
  double* out;
  unsigned long long* fl;
  cudaMalloc(&out, 8);
  cudaMalloc(&fl, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mixed<MODE><<<sms, threads>>>(out, 100, 1.0, fl, 100);
  cudaDeviceSynchronize();
  cudaMemset(fl, 0, 8);
  cudaEventRecord(e0);
  mixed<MODE><<<sms, threads>>>(out, iters_mma, 1.0, fl, iters_fma);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long f;
  cudaMemcpy(&f, fl, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.2f TFLOP/s (%.3f ms)\n", name, double(f) / (ms * 1e-3) / 1e12, ms);
}

int main() {
  run<0>(20000, "DMMA only (16 warps/SM)");
  run<1>(20000, "DFMA only (16 warps/SM)");
  run<3>(20000, "DMMA 8 warps, 8 idle");
  run<4>(20000, "DFMA 8 warps, 8 idle", 78000);
  run<2>(20000, "DMMA 8 + DFMA 8 warps", 78000);
  run<6>(20000, "2 DMMA/scheduler, rest idle");
  run<5>(20000, "2 DMMA + 2 DFMA / scheduler", 78000);
  return 0;
}
