// DMMA issue rate vs warps per SM sub-partition and independent accumulators
// per warp (how many resident warps the DMMA kernels need).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_occ dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ACC][2];
  for (int t = 0; t < ACC; ++t) c[t][0] = c[t][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < ACC; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < ACC; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
void run(int sms, int wpsp) {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096 * 16 / ACC;
  dmma_loop<ACC><<<sms * wpsp, 128>>>(d, 64);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  dmma_loop<ACC><<<sms * wpsp, 128>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = double(sms) * wpsp * 4 * iters * ACC * 512.0;
  printf("warps/SMSP=%d acc/warp=%2d  %.2f TFLOP/s\n", wpsp, ACC, flops / ms / 1e9);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w = 1; w <= 6; ++w) {
    run<4>(sms, w);
    run<8>(sms, w);
    run<16>(sms, w);
  }
}
