// Dependent-chain latencies (cycles) of the primitives the QR small algebra uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 latency.cu -o latency
#include <cstdio>

__global__ void lat(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  const int tid = threadIdx.x;
  if (tid < 64) sm[tid] = seed + tid;
  __syncthreads();
  double x = seed + tid * 1e-9;
  const int N = 512;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0);
  long long t3 = clock64();
  for (int i = 0; i < N; ++i) x = __drcp_rn(x + 1.0);
  long long t4 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (tid + 1) & 31) * 0.5 + 0.5;
  long long t5 = clock64();
  int idx = tid & 63;
  for (int i = 0; i < N; ++i) {
    x += sm[idx];
    idx = (int(x) & 31) + (tid & 32);
  }
  long long t6 = clock64();
  for (int i = 0; i < N; ++i) {
    __syncthreads();
    x += 1.0;
  }
  long long t7 = clock64();
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  long long t8 = clock64();
  out[tid] = x;
  if (tid == 0) {
    cyc[0] = (t1 - t0) / N; cyc[1] = (t2 - t1) / N; cyc[2] = (t3 - t2) / N; cyc[3] = (t4 - t3) / N;
    cyc[4] = (t5 - t4) / N; cyc[5] = (t6 - t5) / N; cyc[6] = (t7 - t6) / N; cyc[7] = (t8 - t7) / N;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 64);
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
    lat<<<1, threads>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
    printf("{\"threads\": %d, \"dfma\": %lld, \"dsqrt+dadd\": %lld, \"ddiv+dadd\": %lld, \"drcp_rn+dadd\": %lld, "
           "\"shfl+dfma\": %lld, \"lds+dadd+cvt\": %lld, \"bar.sync+dadd\": %lld, \"dmul\": %lld}\n",
           threads, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7]);
  }
  return 0;
}
