// Where the Gram kernel's time goes: the DMMA inner loop on operands already in
// shared memory (no loads, no barriers), in the 2 x 2 (32 x 32 warp tiles) and
// row-split (16 x 64) layouts, for 2/3/4 CTAs of 4 warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gram_inner gram_inner.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
constexpr int SA = 68, KB = 16, STAGES = 4, STG = KB * 2 * SA;

template <int LAYOUT, bool SYNC>
__global__ void __launch_bounds__(128) inner(double* out, int chunks) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < STAGES * STG; i += 128) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double acc[32];
  for (int i = 0; i < 32; ++i) acc[i] = 0.0;
  for (int q = 0; q < chunks; ++q) {
    const double* sa = sm + (q % STAGES) * STG;
    if (LAYOUT == 0) {
      const double* pa = sa + t * SA + (warp & 1) * 32 + g;
      const double* pb = sa + KB * SA + t * SA + (warp >> 1) * 32 + g;
#pragma unroll
      for (int kk = 0; kk < KB; kk += 4) {
        double fa[4], fb[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) fa[x] = pa[kk * SA + x * 8];
#pragma unroll
        for (int y = 0; y < 4; ++y) fb[y] = pb[kk * SA + y * 8];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) dmma(acc[(x * 4 + y) * 2], acc[(x * 4 + y) * 2 + 1], fa[x], fb[y]);
      }
    } else {
      const double* pa0 = sa + t * SA + warp * 8 + g;
      const double* pa1 = sa + t * SA + (warp + 4) * 8 + g;
      const double* pb = sa + KB * SA + t * SA + g;
#pragma unroll
      for (int kk = 0; kk < KB; kk += 4) {
        double fa[2], fb[8];
        fa[0] = pa0[kk * SA];
        fa[1] = pa1[kk * SA];
#pragma unroll
        for (int y = 0; y < 8; ++y) fb[y] = pb[kk * SA + y * 8];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 8; ++y) dmma(acc[(x * 8 + y) * 2], acc[(x * 8 + y) * 2 + 1], fa[x], fb[y]);
      }
    }
    if (SYNC) __syncthreads();
  }
  double s = 0;
  for (int i = 0; i < 32; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

template <int LAYOUT, bool SYNC>
void run(int sms, int cpsm) {
  double* d;
  cudaMalloc(&d, 8);
  const size_t smem = sizeof(double) * STAGES * STG;
  cudaFuncSetAttribute(inner<LAYOUT, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int chunks = 20000;
  inner<LAYOUT, SYNC><<<sms * cpsm, 128, smem>>>(d, 100);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  inner<LAYOUT, SYNC><<<sms * cpsm, 128, smem>>>(d, chunks);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = double(sms) * cpsm * chunks * 2.0 * 64 * 64 * KB;
  printf("layout %s sync %d CTAs/SM %d: %.2f TFLOP/s (%s)\n", LAYOUT ? "rowsplit" : "2x2", (int)SYNC, cpsm,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int c = 1; c <= 4; ++c) {
    run<0, false>(sms, c);
    run<1, false>(sms, c);
    run<0, true>(sms, c);
    run<1, true>(sms, c);
  }
}
