// Latency of cluster-wide barriers and DSMEM round trips (cycles), vs a CTA barrier.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_lat cluster_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int C>
__global__ void __cluster_dims__(C, 1, 1) k(long long* out, int n) {
  __shared__ double buf[64];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  buf[threadIdx.x & 63] = rank;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) cl.sync();
  long long t1 = clock64();
  // ping-pong through DSMEM: rank 0 writes to rank 1, then both sync (store + barrier)
  double* remote = cl.map_shared_rank(buf, (rank + 1) % C);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x < 32) remote[threadIdx.x] = i + rank;
    cl.sync();
  }
  long long t3 = clock64();
  // split arrive/wait with work in between
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t6 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    out[0] = (t1 - t0) / n;
    out[1] = (t3 - t2) / n;
    out[2] = (t5 - t4) / n;
    out[3] = (t6 - t5) / n;
  }
}

template <int C>
void run(int threads) {
  long long* d;
  cudaMalloc(&d, 64);
  k<C><<<C, threads>>>(d, 1000);
  k<C><<<C, threads>>>(d, 1000);
  long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("cluster=%d threads=%d: cluster.sync %lld  dsmem-store+sync %lld  arrive/wait %lld  syncthreads %lld  (%s)\n", C,
         threads, h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int t : {256, 512, 1024}) {
    run<1>(t);
    run<2>(t);
    run<4>(t);
    run<8>(t);
  }
}
