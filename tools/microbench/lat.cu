// Dependent-chain latencies on B200 (cycles per op): DFMA, DMUL, double sqrt,
// double reciprocal, SHFL, LDS, __syncthreads with 512/1024 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sh[1024];
  sh[threadIdx.x] = x0 + threadIdx.x;
  __syncthreads();
  double x = x0 + threadIdx.x * 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // reciprocal chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 2.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // shfl chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // LDS chain (pointer chasing through the value)
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = (static_cast<int>(sh[idx]) + 1) & 1023;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // barrier
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // rsqrt-based: 1/sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  out[threadIdx.x] = x + idx;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8 * 1024);
  cudaMalloc(&c, 8 * 16);
  const char* names[] = {"DFMA", "sqrt", "1/x", "SHFL+DADD", "LDS+cvt", "syncthreads", "rsqrt"};
  for (int th : {32, 512, 1024}) {
    const int n = 1000;
    lat<<<1, th>>>(d, c, 1.5, n);
    lat<<<1, th>>>(d, c, 1.5, n);
    long long h[16];
    cudaMemcpy(h, c, 8 * 16, cudaMemcpyDeviceToHost);
    printf("threads=%d:", th);
    for (int i = 0; i < 7; ++i) printf("  %s %.1f", names[i], double(h[i]) / n);
    printf("\n");
  }
}
