// Cycle counts of the Cholesky building blocks (development probe).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2603_19439_b200/csrc -o chol_parts chol_parts.cu
#include <cstdio>
#include <vector>
#include "smalllin.cuh"
using namespace stg;

__global__ void parts(const double* G, int w, long long* cyc) {
  extern __shared__ double sm[];
  double* invd = sm + w * (w + 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < w; i += blockDim.x >> 5)
    for (int c = lane; c < w; c += 32)
      if (c >= i) sm[packed_row(i, w) + c] = G[i * w + c];
  __syncthreads();
  int fl = 0;
  long long t0 = clock64();
  if (warp == 0) chol_diag(16, sm, invd, w, 0, 16, lane, (const double*)nullptr, 0.0, 0, fl);
  __syncthreads();
  long long t1 = clock64();
  chol_panel(sm, invd, w, 0, 16, tid, blockDim.x);
  __syncthreads();
  long long t2 = clock64();
  chol_trailing(sm, w, 0, 16, 16, 16, w, warp, blockDim.x >> 5, lane);
  __syncthreads();
  long long t3 = clock64();
  for (int k = 0; k < 10; ++k) __syncthreads();
  long long t4 = clock64();
  if (tid == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = (t4 - t3) / 10;
    cyc[4] = fl;
  }
}

int main() {
  for (int w : {32, 132, 200}) {
    std::vector<double> h(w * w);
    for (int i = 0; i < w; ++i)
      for (int j = 0; j < w; ++j) h[i * w + j] = (i == j ? 2.0 + i : 0.0) + 0.01 * ((i * 7 + j * 3) % 5) * (i != j);
    for (int i = 0; i < w; ++i) for (int j = 0; j < i; ++j) h[i * w + j] = h[j * w + i];
    double* G;
    long long* c;
    cudaMalloc(&G, 8 * w * w);
    cudaMalloc(&c, 64);
    cudaMemcpy(G, h.data(), 8 * w * w, cudaMemcpyHostToDevice);
    const size_t smem = chol_smem_bytes(w);
    cudaFuncSetAttribute(parts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    parts<<<1, kCholThreads, smem>>>(G, w, c);
    parts<<<1, kCholThreads, smem>>>(G, w, c);
    long long r[5];
    cudaMemcpy(r, c, 40, cudaMemcpyDeviceToHost);
    printf("w=%d: diag %lld  panel %lld  trailing(first) %lld  barrier %lld cycles  (err %s)\n", w, r[0], r[1], r[2], r[3],
           cudaGetErrorString(cudaGetLastError()));
  }
}
