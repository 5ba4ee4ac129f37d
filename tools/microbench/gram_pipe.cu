// Standalone probe of the split-K Gram pipeline (TMA ring -> DMMA) on synthetic
// data: where do the load time and the DMMA time fail to overlap?
// Knobs: dedicated producer warp, ring depth, rows per stage, MMA / load elision.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2603_19439_b200/csrc -o gram_pipe gram_pipe.cu -lcuda
#include <algorithm>
#include <vector>

#include "dmma.cuh"

using namespace stg;
using namespace stg::dm;

// MODE 0 full, 1 no MMA, 2 loads only for the first ring fill (then full barriers arrive without data)
template <int PW, int STAGES, int KBK, int MODE>
__global__ void __launch_bounds__(128 + 32 * PW, 3)
    probe(const __grid_constant__ CUtensorMap tmA, i64 nrows, int tiles, i64 rows_per_split, int items, double* out,
          unsigned long long* clk) {
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw);
  unsigned long long* empty = full + STAGES;
  double* stage0 = reinterpret_cast<double*>(smraw + 128);
  constexpr int SA = 68, STG = KBK * 2 * SA;
  constexpr unsigned kBytes = sizeof(double) * STG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  unsigned long long c0 = 0, g0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c0 = clock64();
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
  }
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 4);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int my = blockIdx.x < items ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nch = static_cast<int>(cdiv(rows_per_split, KBK));
  const int total = my * nch;
  auto produce = [&](int i) {
    const int st = i % STAGES;
    if (i >= STAGES) mbar_wait(&empty[st], static_cast<unsigned>((i / STAGES - 1) & 1));
    const int item = blockIdx.x + (i / nch) * gridDim.x, q = i % nch;
    const int tile = item % (tiles * tiles), split = item / (tiles * tiles);
    const int row0 = static_cast<int>(split * rows_per_split) + q * KBK;
    double* sa = stage0 + st * STG;
    if (MODE == 2 && i >= STAGES) {
      mbar_arrive(&full[st]);
      return;
    }
    mbar_arrive_expect_tx(&full[st], kBytes);
    tma_load_2d(sa, &tmA, (tile / tiles) * 64, row0, &full[st]);
    tma_load_2d(sa + KBK * SA, &tmA, (tile % tiles) * 64, row0, &full[st]);
  };
  double acc[2][8][2];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  if (MODE == 3 || MODE == 5) {
    if (warp == 4) return;
  } else if (PW) {
    if (warp == 4) {
      if (lane == 0)
        for (int i = 0; i < total; ++i) produce(i);
      return;
    }
  } else if (threadIdx.x == 0) {
    for (int i = 0; i < min(total, STAGES - 1); ++i) produce(i);
  }
  for (int i = 0; i < total; ++i) {
    if (MODE != 3 && MODE != 5 && !PW && threadIdx.x == 0 && i + STAGES - 1 < total) produce(i + STAGES - 1);
    const int st = i % STAGES;
    if (MODE != 3 && MODE != 5) mbar_wait(&full[st], static_cast<unsigned>((i / STAGES) & 1));
    const double* sa = stage0 + st * STG;
    const double* pa0 = sa + t * SA + warp * 8 + g;
    const double* pa1 = sa + t * SA + (warp + 4) * 8 + g;
    const double* pb = sa + KBK * SA + t * SA + g;
    if (MODE != 1)
      rs_mma<2, 8, SA, SA, KBK>(acc, pa0, pa1, pb);
    else
      acc[0][0][0] += pa0[0] + pa1[0] + pb[0];
    if (MODE != 3) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (i % nch == nch - 1) {  // partial tile out (same slot every item: traffic only)
      double* o = out + static_cast<i64>(blockIdx.x) * 4096;
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          *reinterpret_cast<double2*>(o + ((x ? warp + 4 : warp) * 8 + g) * 64 + y * 8 + 2 * t) =
              make_double2(acc[x][y][0], acc[x][y][1]);
          acc[x][y][0] = acc[x][y][1] = 0.0;
        }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
    clk[0] = clock64() - c0;
    clk[1] = g1 - g0;
  }
}

template <int PW, int STAGES, int KBK, int MODE>
void run(const double* A, i64 rows, int m, int cpsm, double* out, unsigned long long* clk) {
  const int tiles = m / 64;
  const i64 target = 148 * cpsm;
  i64 splits = target / (tiles * tiles);  // one item per CTA, no second round
  const i64 rps = round_up(cdiv(rows, splits), KBK);
  splits = cdiv(rows, rps);
  if (splits * tiles * tiles > target) printf("warning: second round\n");
  const int items = static_cast<int>(splits * tiles * tiles);
  const CUtensorMap ma = make_tmap_2d(A, rows, m, m, 68, KBK);
  const size_t smem = 128 + sizeof(double) * STAGES * KBK * 2 * 68;
  auto k = probe<PW, STAGES, KBK, MODE>;
  STG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int G = static_cast<int>(std::min<i64>(items, target));
  float best = 1e9f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    k<<<G, 128 + 32 * PW, smem>>>(ma, rows, tiles, rps, items, out, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::min(best, ms);
  }
  STG_CUDA(cudaGetLastError());
  unsigned long long h[2];
  cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * rows * m * m;
  printf("PW %d stages %d rows/stage %2d mode %d CTAs/SM %d smem %3zu KB: %7.1f us  %5.2f TFLOP/s  SM clock %.0f MHz\n", PW,
         STAGES, KBK, MODE, cpsm, smem / 1024, best * 1e3, MODE == 1 ? 0.0 : flops / best / 1e9,
         1e3 * static_cast<double>(h[0]) / static_cast<double>(h[1]));
}

// The library's kernels on the step's real shapes (config 3: ~104k stacked rows).
void real(const double* A, i64 rows, int m1, int m2, bool sym, int waves, double* partial, int* ctr) {
  GramArgs a{};
  a.A = A;
  a.lda = 256;
  a.B = sym ? A : A + 8;
  a.ldb = 256;
  a.nrows = rows;
  a.m1 = m1;
  a.m2 = m2;
  a.tiles_i = static_cast<int>(cdiv(m1, 64));
  a.tiles_j = static_cast<int>(cdiv(m2, 64));
  a.sym = sym;
  const int ntiles = sym ? a.tiles_i * (a.tiles_i + 1) / 2 : a.tiles_i * a.tiles_j;
  i64 splits = std::max<i64>(1, std::min<i64>(cdiv(rows, 128), cdiv(148 * waves, ntiles)));
  a.rows_per_split = round_up(cdiv(rows, splits), 32);
  splits = cdiv(rows, a.rows_per_split);
  a.partial = partial;
  const CUtensorMap ma = make_tmap_2d(a.A, rows, m1, a.lda, 68, kBK);
  const CUtensorMap mb = make_tmap_2d(a.B, rows, m2, a.ldb, 68, kBK);
  const CUtensorMap ra = make_tmap_2d(a.A, rows, m1, a.lda, 68, kRsBK);
  const CUtensorMap rb = make_tmap_2d(a.B, rows, m2, a.ldb, 68, kRsBK);
  const size_t smem = gram_tma_smem<2, 2>();
  STG_CUDA(cudaFuncSetAttribute(gram_tma_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  STG_CUDA(cudaFuncSetAttribute(gram_persist_rs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRsSmem));
  STG_CUDA(cudaFuncSetAttribute(gram_persist_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double flops = sym ? 1.0 * rows * m1 * (m1 + 1) : 2.0 * rows * m1 * m2;
  // tiles by DMMA work, heaviest first (as Session::gram)
  gram_tile_order(a, ntiles, (int)splits, getenv("BLOCK_WAVES") ? std::max(1, atoi(getenv("BLOCK_WAVES")) * 148 * STG_GRAM_MINB / ntiles) : 0);
  for (int v = 0; v < 4; ++v) {
    if (v == 1 || v == 2) continue;
    a.ordered = v == 3 && ntiles <= 64;
    float best = 1e9f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (v == 0)
        gram_tma_kernel<2, 2><<<dim3(ntiles, (unsigned)splits), NT, smem>>>(a, ma, mb);
      else if (v == 1)
        gram_persist_kernel<2, 2><<<148 * STG_GRAM_MINB, NT, smem>>>(a, ma, mb, ntiles, (int)splits, ctr);
      else
        gram_persist_rs_kernel<<<148 * STG_GRAM_MINB, kRsThreads, kRsSmem>>>(a, ra, rb, ntiles, (int)splits, ctr);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0) best = std::min(best, ms);
    }
    STG_CUDA(cudaGetLastError());
    printf("  %-22s %dx%d%s waves %2d splits %3lld: %6.1f us  %5.2f TFLOP/s\n",
           v == 0 ? "gram_tma (static grid)" : v == 1 ? "persist 2x2" : v == 2 ? "persist rowsplit" : "rowsplit heavy-first", m1, m2, sym ? " sym" : "",
           waves, splits, best * 1e3, flops / best / 1e9);
  }
}

// The K Gram of the step: X'X over ~1.08M rows x 32 columns, the rows of P masked (gram_stream_kernel).
void stream_gram(i64 rows, bool masked) {
  double *X, *partial;
  int* mask;
  cudaMalloc(&X, sizeof(double) * rows * 32);
  cudaMalloc(&partial, sizeof(double) * 1024 * 148 * 3);
  cudaMalloc(&mask, sizeof(int) * rows);
  cudaMemset(X, 0, sizeof(double) * rows * 32);
  cudaMemset(mask, 0, sizeof(int) * rows);
  GramArgs a{};
  a.A = a.B = X;
  a.lda = a.ldb = 32;
  a.nrows = rows;
  a.m1 = a.m2 = 32;
  a.tiles_i = a.tiles_j = 1;
  a.sym = 1;
  a.partial = partial;
  a.mask = masked ? mask : nullptr;
  a.mask_val = 7;
  const CUtensorMap ma = make_tmap_2d(X, rows, 32, 32, kStreamPitch, kGsRows);
  const int ntl = static_cast<int>(cdiv(rows, kGsRows));
  STG_CUDA(cudaFuncSetAttribute(gram_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)gram_stream_smem(false)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int G : {148, 296, 444}) {
    float best = 1e9f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      gram_stream_kernel<<<std::min(ntl, G), NT, gram_stream_smem(true)>>>(a, ma, ma, 1, ntl);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0) best = std::min(best, ms);
    }
    STG_CUDA(cudaGetLastError());
    printf("  gram_stream %lld x 32 sym %s grid %d: %6.1f us  %5.2f TB/s\n", rows, masked ? "masked" : "      ", G,
           best * 1e3, 8.0 * rows * 32 / best / 1e9);
  }
  cudaFree(X);
  cudaFree(partial);
  cudaFree(mask);
}

int main() {
  if (getenv("PROBE_STREAM")) {
    stream_gram(1080347, true);
    stream_gram(1080347, false);
    stream_gram(104049, false);
    return 0;
  }
  const i64 rows = 104049;
  const int m = 256;
  double *A, *out;
  unsigned long long* clk;
  cudaMalloc(&A, sizeof(double) * rows * m);
  cudaMalloc(&out, sizeof(double) * 4096 * 148 * 4);
  cudaMalloc(&clk, 16);
  std::vector<double> h(static_cast<size_t>(rows) * m);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-3 * static_cast<double>(i % 1013);
  cudaMemcpy(A, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  printf("Gram %lld x %d x %d (all tiles full), ideal %.1f us at 37.1 TF\n", rows, m, m, 2.0 * rows * m * m / 37.1e6);
  if (getenv("PROBE_SYNTH")) {
  run<1, 4, 16, 3>(A, rows, m, 3, out, clk);
  run<1, 4, 16, 5>(A, rows, m, 3, out, clk);
  run<1, 4, 16, 3>(A, rows, m, 1, out, clk);
  run<1, 4, 16, 5>(A, rows, m, 1, out, clk);
  run<0, 4, 16, 0>(A, rows, m, 3, out, clk);
  run<0, 4, 16, 1>(A, rows, m, 3, out, clk);
  run<0, 4, 16, 2>(A, rows, m, 3, out, clk);
  run<1, 4, 16, 0>(A, rows, m, 3, out, clk);
  run<1, 4, 16, 1>(A, rows, m, 3, out, clk);
  run<1, 4, 16, 2>(A, rows, m, 3, out, clk);
  run<1, 6, 16, 0>(A, rows, m, 2, out, clk);
  run<1, 3, 32, 0>(A, rows, m, 2, out, clk);
  run<1, 8, 8, 0>(A, rows, m, 3, out, clk);
  run<0, 4, 16, 0>(A, rows, m, 2, out, clk);
  run<1, 4, 16, 0>(A, rows, m, 2, out, clk);
  run<1, 4, 16, 0>(A, rows, m, 1, out, clk);
  }
  printf("variant: PW %d rows/stage %d stages %d CTAs/SM %d\n", kGramPW, kRsBK, kRsStages, STG_GRAM_MINB);
  double* partial;
  int* ctr;
  cudaMalloc(&partial, sizeof(double) * 256 * 256 * 2048);
  cudaMalloc(&ctr, 64);
  cudaMemset(ctr, 0, 64);
  for (int waves : {3, 6, 12, 24}) real(A, rows, 200, 200, true, waves, partial, ctr);
  for (int waves : {3, 6, 12}) real(A, rows, 100, 100, true, waves, partial, ctr);
  for (int waves : {3, 6, 12}) real(A, rows, 164, 100, false, waves, partial, ctr);
  for (int waves : {3, 6, 12}) real(A, rows, 64, 200, false, waves, partial, ctr);
  for (int waves : {3, 6}) real(A, rows, 64, 64, true, waves, partial, ctr);
  return 0;
}
