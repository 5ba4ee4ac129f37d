// Can the FP64 tensor pipe (DMMA) and the FP64 FMA pipe (DFMA) run at the same
// time? Mixed loop: ACC DMMA chains and F DFMA chains per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_dfma_mix dmma_dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC, int F>
__global__ void mix_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ACC > 0 ? ACC : 1][2];
  double f[F > 0 ? F : 1];
  for (int t = 0; t < ACC; ++t) c[t][0] = c[t][1] = 0;
  for (int t = 0; t < F; ++t) f[t] = t;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < (ACC > F ? ACC : F); ++t) {
      if (t < ACC)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
      if (t < F) {
#pragma unroll
        for (int r = 0; r < 4; ++r) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(f[t]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
  for (int t = 0; t < ACC; ++t) s += c[t][0] + c[t][1];
  for (int t = 0; t < F; ++t) s += f[t];
  if (s == 12345.0) out[0] = s;
}

template <int ACC, int F>
void run(int sms, int ctas_per_sm, int threads) {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192;
  mix_loop<ACC, F><<<sms * ctas_per_sm, threads>>>(d, 64);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  mix_loop<ACC, F><<<sms * ctas_per_sm, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(sms) * ctas_per_sm * threads / 32;
  const double fl_mma = warps * iters * ACC * 512.0;
  const double fl_fma = warps * 32 * iters * F * 4 * 2.0;
  printf("ACC=%2d F=%2d ctas/SM=%d threads=%d: %.3f ms  DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", ACC, F,
         ctas_per_sm, threads, ms, fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<16, 0>(sms, 2, 256);
  run<0, 8>(sms, 2, 256);
  run<16, 2>(sms, 2, 256);
  run<16, 4>(sms, 2, 256);
  run<16, 8>(sms, 2, 256);
  run<8, 8>(sms, 2, 256);
  run<8, 4>(sms, 2, 256);
  run<16, 16>(sms, 2, 256);
  return 0;
}
