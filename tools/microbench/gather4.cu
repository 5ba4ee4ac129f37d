// TMA tile::gather4 (sm_100a): semantics check and gather throughput against
// plain warp loads, for the SpMM's X-row gathers (m = 32 / 64 / 100 columns).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2603_19439_b200/csrc -o gather4 gather4.cu -lcuda
#include <cstdio>
#include <vector>
#include <random>
#include "common.cuh"
using namespace stg;

__device__ __forceinline__ void tma_gather4(void* smem, const CUtensorMap* map, int x, int r0, int r1, int r2, int r3,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::
          "r"(smem_u32(smem)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

__global__ void check_kernel(const __grid_constant__ CUtensorMap tm, int W, const int* rows, double* out) {
  __shared__ __align__(1024) double s[4 * 256];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 4 * W * 8);
    tma_gather4(s, &tm, 0, rows[0], rows[1], rows[2], rows[3], &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 4 * W; i += blockDim.x) out[i] = s[i];
}

// each warp: gathers `per_warp` random rows in batches of 32 (8 gather4 by lanes 0..7),
// D batches in flight, then sums them (lane = column) into a checksum
template <int W, int D>
__global__ void __launch_bounds__(128) gather_tma_kernel(const __grid_constant__ CUtensorMap tm, const int* idx,
                                                         int per_warp, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm) + wib * D;
  double* stg = reinterpret_cast<double*>(sm + 1024) + wib * D * 32 * W;
  if (lane == 0)
    for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
  mbar_fence_init();
  __syncwarp();
  const int gw = blockIdx.x * 4 + wib;
  const int* my = idx + (size_t)gw * per_warp;
  const int nb = per_warp / 32;
  auto issue = [&](int b) {
    const int slot = b % D;
    const int c = my[b * 32 + lane];
    const int r0 = __shfl_sync(0xffffffffu, c, (lane & 7) * 4 + 0), r1 = __shfl_sync(0xffffffffu, c, (lane & 7) * 4 + 1);
    const int r2 = __shfl_sync(0xffffffffu, c, (lane & 7) * 4 + 2), r3 = __shfl_sync(0xffffffffu, c, (lane & 7) * 4 + 3);
    if (lane == 0) mbar_arrive_expect_tx(&bars[slot], 32 * W * 8);
    __syncwarp();
    if (lane < 8) tma_gather4(stg + (slot * 32 + lane * 4) * W, &tm, 0, r0, r1, r2, r3, &bars[slot]);
  };
  for (int b = 0; b < D - 1 && b < nb; ++b) issue(b);
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) {
    if (b + D - 1 < nb) issue(b + D - 1);
    const int slot = b % D;
    mbar_wait(&bars[slot], (b / D) & 1);
    const double* sb = stg + slot * 32 * W;
    for (int e = 0; e < 32; ++e)
      for (int c = lane; c < W; c += 32) acc += sb[e * W + c];
    __syncwarp();
  }
  out[gw * 32 + lane] = acc;
}

template <int W>
__global__ void __launch_bounds__(128) gather_ld_kernel(const double* X, int ldx, const int* idx, int per_warp,
                                                        double* out) {
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 4 + wib;
  const int* my = idx + (size_t)gw * per_warp;
  double acc = 0.0;
  for (int b = 0; b < per_warp; b += 8) {
    double v[8][(W + 31) / 32];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = my[b + u];
#pragma unroll
      for (int t = 0; t < (W + 31) / 32; ++t) v[u][t] = (lane + 32 * t < W) ? __ldg(X + (size_t)r * ldx + lane + 32 * t) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int t = 0; t < (W + 31) / 32; ++t) acc += v[u][t];
  }
  out[gw * 32 + lane] = acc;
}

template <int W, int D>
void bench(const double* X, int N, int ld, const int* idx, int nwarps, int per_warp, double* out) {
  const CUtensorMap tm = make_tmap_2d(X, N, W, ld, W, 1);
  const size_t smem = 1024 + 4 * (size_t)D * 32 * W * 8;
  cudaFuncSetAttribute(gather_tma_kernel<W, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    gather_tma_kernel<W, D><<<nwarps / 4, 128, smem>>>(tm, idx, per_warp, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms1;
  cudaEventElapsedTime(&ms1, a, b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    gather_ld_kernel<W><<<nwarps / 4, 128>>>(X, ld, idx, per_warp, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms2;
  cudaEventElapsedTime(&ms2, a, b);
  const double bytes = (double)nwarps * per_warp * W * 8;
  printf("W=%3d D=%d warps=%6d rows/warp=%4d: tma gather4 %7.1f us (%6.2f TB/s)  plain loads %7.1f us (%6.2f TB/s)  [%s]\n", W, D,
         nwarps, per_warp, ms1 * 1e3, bytes / ms1 / 1e9, ms2 * 1e3, bytes / ms2 / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int N = 107000, ld = 104;
  std::vector<double> h((size_t)N * ld);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)(i % 1000) * 0.001 + (double)(i / ld);
  double *X, *out;
  cudaMalloc(&X, h.size() * 8);
  cudaMemcpy(X, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 1 << 26);
  {
    cudaError_t e0 = cudaDeviceSynchronize();
    printf("pre: %s\n", cudaGetErrorString(e0));
    try { make_tmap_2d(X, N, 32, ld, 36, 64); printf("encode 36x64 ok\n"); } catch (std::exception& e) { printf("%s\n", e.what()); }
    try { make_tmap_2d(X, N, 32, ld, 32, 1); printf("encode 32x1 ok\n"); } catch (std::exception& e) { printf("%s\n", e.what()); }
    try { make_tmap_2d(X, N, 32, ld, 32, 4); printf("encode 32x4 ok\n"); } catch (std::exception& e) { printf("%s\n", e.what()); }
  }
  // semantics
  int hr[4] = {5, 17, 3, 100};
  int* dr;
  cudaMalloc(&dr, 16);
  cudaMemcpy(dr, hr, 16, cudaMemcpyHostToDevice);
  for (int W : {32, 64, 100}) {
    const CUtensorMap tm = make_tmap_2d(X, N, W, ld, W, 1);
    check_kernel<<<1, 128>>>(tm, W, dr, out);
    const cudaError_t ke = cudaDeviceSynchronize();
    if (ke != cudaSuccess) { printf("check_kernel W=%d failed: %s\n", W, cudaGetErrorString(ke)); return 1; }
    std::vector<double> o(4 * W);
    cudaMemcpy(o.data(), out, 8 * o.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int q = 0; q < 4; ++q)
      for (int c = 0; c < W; ++c) bad += o[q * W + c] != h[(size_t)hr[q] * ld + c];
    printf("gather4 semantics W=%d: %s (%s)\n", W, bad ? "MISMATCH" : "ok", cudaGetErrorString(cudaGetLastError()));
  }
  // throughput: 367k gathers like the config-3 Delta X-bar
  const int nwarps = 148 * 8 * 4, per_warp = 96;
  std::vector<int> hi((size_t)nwarps * per_warp);
  std::mt19937 g(1);
  for (auto& v : hi) v = g() % N;
  int* di;
  cudaMalloc(&di, hi.size() * 4);
  cudaMemcpy(di, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice);
  bench<32, 4>(X, N, ld, di, nwarps, per_warp, out);
  bench<32, 2>(X, N, ld, di, nwarps, per_warp, out);
  bench<64, 2>(X, N, ld, di, nwarps, per_warp, out);
  bench<100, 2>(X, N, ld, di, nwarps, per_warp, out);
  return 0;
}
