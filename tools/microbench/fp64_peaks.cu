// FP64 peak probes on B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA issue
// throughput, plus cuSOLVER dsyevd latency at the projected-eigensolve sizes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu -lcusolver
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int t = 0; t < 16; ++t) c[t] = t;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = fma(a, c[t], b);
  }
  double s = 0;
  for (int t = 0; t < 16; ++t) s += c[t];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dmma_loop<<<sms * 4, warps * 32>>>(d, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_loop<<<sms * 4, warps * 32>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = double(sms) * 4 * warps * iters * 8 * 512.0;
    printf("DMMA m8n8k4: warps/CTA=%d  %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    dfma_loop<<<sms * 4, warps * 32>>>(d, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<<<sms * 4, warps * 32>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = double(sms) * 4 * warps * 32 * iters * 16 * 2.0;
    printf("DFMA: warps/CTA=%d  %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  // cuSOLVER dsyevd / dsyevj latency.
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  for (int n : {16, 32, 64, 132, 164, 200, 228}) {
    std::vector<double> a(n * n);
    srand(1);
    for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) { double v = rand() / double(RAND_MAX) - 0.5; a[i*n+j] = a[j*n+i] = v; }
    double *da, *dw, *work; int* info; int lw = 0;
    CK(cudaMalloc(&da, n*n*8)); CK(cudaMalloc(&dw, n*8)); CK(cudaMalloc(&info, 4));
    cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, da, n, dw, &lw);
    CK(cudaMalloc(&work, lw * 8));
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      CK(cudaMemcpy(da, a.data(), n*n*8, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, da, n, dw, work, lw, info);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    // syevj
    syevjInfo_t params; cusolverDnCreateSyevjInfo(&params);
    int lwj = 0; cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, da, n, dw, &lwj, params);
    double* workj; CK(cudaMalloc(&workj, lwj * 8));
    float bestj = 1e9;
    for (int r = 0; r < 10; ++r) {
      CK(cudaMemcpy(da, a.data(), n*n*8, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, da, n, dw, workj, lwj, info, params);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < bestj) bestj = ms;
    }
    printf("n=%d syevd %.3f ms  syevj %.3f ms\n", n, best, bestj);
    cudaFree(da); cudaFree(dw); cudaFree(work); cudaFree(workj); cudaFree(info);
  }
  return 0;
}
