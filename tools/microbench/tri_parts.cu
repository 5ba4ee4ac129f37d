// Cycles per phase of the tridiagonalization (development probe).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSTG_TRI_PROF -I../../paper_2603_19439_b200/csrc -o tri_parts tri_parts.cu
#include <cstdio>
#include <vector>
#include "eigsolve.cuh"
using namespace stg;

int main() {
  for (int n : {164, 200}) {
    std::vector<double> h(n * n);
    unsigned s = 1;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) {
        s = s * 1664525u + 1013904223u;
        h[i * n + j] = h[j * n + i] = (s >> 8) / double(1 << 24) - 0.5;
      }
    double *M, *dbuf;
    int *ibuf, *flags;
    cudaMalloc(&M, 8 * n * n);
    cudaMalloc(&dbuf, 8 * eig_scratch_doubles(n, 32));
    cudaMalloc(&ibuf, 4 * eig_scratch_ints(n, 32));
    cudaMalloc(&flags, 4);
    cudaMemcpy(M, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
    const EigBufs b = eig_carve(dbuf, ibuf, n, 32);
    eig_set_attributes();
    long long z[8] = {0};
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpyToSymbol(g_tri_prof, z, sizeof(z));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (n <= kEig1N)
        tridiag1_kernel<<<1, kTriThreads, tridiag_smem_bytes(n, 1, tridiag_gmax(n, 1))>>>(M, n, n, 1, tridiag_gmax(n, 1), b, flags);
      else
        tridiag2_kernel<<<2, kTriThreads, tridiag_smem_bytes(n, 2, tridiag_gmax(n, 2))>>>(M, n, n, 1, tridiag_gmax(n, 2), b, flags);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long p[8];
      cudaMemcpyFromSymbol(p, g_tri_prof, sizeof(p));
      printf("n=%d %.1f us (%s): load %lld | per column: loop %lld  publish %lld  sums %lld  sync1 %lld  update %lld  next col %lld  sync2 %lld\n",
             n, ms * 1e3, cudaGetErrorString(cudaGetLastError()), p[0], p[6] / (n - 1), p[7] / (n - 1), p[1] / (n - 1), p[2] / (n - 1), p[3] / (n - 1),
             p[4] / (n - 1), p[5] / (n - 1));
    }
  }
}
