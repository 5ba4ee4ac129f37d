// FP64 tensor-core (DMMA) kernels for the tall-skinny algebra of the G-REST
// step. sm_100a has no tcgen05 kind::f64, so FP64 tensor work is mma.sync
// m8n8k4 (SASS DMMA.8x8x4) on operand tiles staged in shared memory by TMA.
//
//   gram : Out(m1 x m2) = A(N x m1)' B(N x m2), split-K over the N rows with
//          a deterministic second-pass reduction (fixed split order). With
//          `sym` only tile pairs ti <= tj are computed and the result is
//          mirrored exactly. gram_persist_rs_kernel (64 x 64 tiles) and
//          gram_persist_kernel (32 x 128 / 128 x 32) are the persistent
//          kernels: a device tile counter, one TMA ring across tiles, a
//          producer warp; gram_tma_kernel is the static grid for products
//          with fewer tiles than CTAs, gram_tn_kernel the cp.async fallback
//          (unaligned views, row masks), gram_stream_kernel the <= 32-wide case.
//   gemm : Out(N x m2) = alpha A(N x m1) C(m1 x m2) + beta B(N x m2), the
//          row-local update (projections, R^-1 application, rotations);
//          gemm_nn_persist_kernel / gemm_nn_tma_kernel / gemm_nn_kernel /
//          gemm_nn_stream_kernel in the same roles. B may alias Out (each tile
//          is read before it is written).
// All blocks are row-major with even leading dimensions.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace stg {
namespace dm {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int SST = BM + 4;  // [BK][64] tiles: stride == 4 (mod 16) doubles -> conflict-free fragments
constexpr int SAR = BK + 4;  // [64][BK] tiles: stride 20 doubles -> conflict-free fragments
constexpr int NT = 128;      // 4 warps, 2 x 2 of 32 x 32 warp tiles

struct GramArgs {
  const double* A;
  int lda;
  const double* B;
  int ldb;
  i64 nrows;
  int m1, m2;
  i64 rows_per_split;
  double* partial;  // [splits][tiles_i*64][tiles_j*64]
  int tiles_i, tiles_j;
  int sym;
  const int* mask;  // optional: rows with mask[r] == mask_val contribute nothing
  int mask_val;
  // persistent kernels, item i -> (tile, split). Not `ordered`: (i % ntiles, i / ntiles). `ordered` (the host
  // sorts the tiles by DMMA work, heaviest first): the splits are cut into blocks of block_splits; within a
  // block the items run tile major, every heavy tile before any light edge tile (which fill each block's and
  // the kernel's tail), and a block's rows (block_splits row ranges, sized to stay in L2) are read from HBM
  // once and then from L2 by the other tiles. block_splits == splits is tile major over the whole product.
  int ordered, block_splits;
  unsigned char order[64];
};

// Loads rows [r, r+BK) x cols [c0, c0+64) of a row-major block into s[BK][SST],
// zero-filling rows >= rend, masked rows and cols >= m.
__device__ __forceinline__ void load_k_tile(double (*s)[SST], const double* g, int ld, i64 r, i64 rend, int c0,
                                            int m, const int* mask, int mask_val) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = threadIdx.x + NT * q;  // 512 16-byte chunks
    const int row = c >> 5, col = (c & 31) * 2;
    i64 gr = r + row;
    const int gc = c0 + col;
    double* dst = &s[row][col];
    if (mask && gr < rend && mask[gr] == mask_val) gr = rend;  // excluded row -> zeros
    if (gr < rend && gc + 2 <= m) {
      cp_async_pair(dst, g + gr * ld + gc);
    } else {
      dst[0] = (gr < rend && gc < m) ? g[gr * ld + gc] : 0.0;
      dst[1] = 0.0;
    }
  }
}

// 32 rows per stage (8 DMMA k-steps between barriers), double-buffered in
// dynamic shared memory. The CTA tile is (32 WM) x (32 WN) with WM * WN = 4
// warps: 64 x 64 for square Grams, 32 x 128 / 128 x 32 when one side is the
// k = 32 tracked block, so no warp idles on an empty half-tile. Tiles entirely
// inside the matrix take the FULL path with no per-subtile predicates.
constexpr int BK2 = 32;
constexpr size_t gram_smem(int WM, int WN) { return sizeof(double) * 2 * BK2 * ((32 * WM + 4) + (32 * WN + 4)); }
constexpr size_t kGramSmem = gram_smem(1, 4);  // the largest layout

// One warp's share of a BK2-row stage: an NX x NY block of 8 x 8 output
// fragments (TRI: only x <= y of a 4 x 4 block on the diagonal of a symmetric
// Gram). Operand fragment (x, k-step kk) sits at pa[kk KA + x XA], (y, kk) at
// pb[kk KB + y YB]. The block shape is warp-uniform, chosen once per tile, so
// edge and diagonal tiles issue no DMMA whose result is discarded.
template <int NX, int NY, bool TRI, int KA, int XA, int KB, int YB, int KR = BK2>
__device__ __forceinline__ void warp_mma(double (&acc)[4][4][2], const double* pa, const double* pb) {
#pragma unroll
  for (int kk = 0; kk < KR; kk += 4) {
    double fa[NX], fb[NY];
#pragma unroll
    for (int x = 0; x < NX; ++x) fa[x] = pa[kk * KA + x * XA];
#pragma unroll
    for (int y = 0; y < NY; ++y) fb[y] = pb[kk * KB + y * YB];
#pragma unroll
    for (int x = 0; x < NX; ++x)
#pragma unroll
      for (int y = 0; y < NY; ++y)
        if (!TRI || x <= y) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
  }
}

// code: 0 = no work, (NX - 1) * 4 + NY for NX, NY in 1..4, 17 = upper 4 x 4
__device__ __forceinline__ int warp_code(int nx, int ny, bool tri) {
  if (nx <= 0 || ny <= 0) return 0;
  if (tri && nx == 4 && ny == 4) return 17;
  return (nx - 1) * 4 + ny;
}

template <int KA, int XA, int KB, int YB, int KR = BK2>
__device__ __forceinline__ void warp_mma_dispatch(int code, double (&acc)[4][4][2], const double* pa,
                                                  const double* pb) {
  switch (code) {
#define STG_MMA_CASE(NX, NY) \
  case (NX - 1) * 4 + NY: warp_mma<NX, NY, false, KA, XA, KB, YB, KR>(acc, pa, pb); break;
    STG_MMA_CASE(1, 1) STG_MMA_CASE(1, 2) STG_MMA_CASE(1, 3) STG_MMA_CASE(1, 4)
    STG_MMA_CASE(2, 1) STG_MMA_CASE(2, 2) STG_MMA_CASE(2, 3) STG_MMA_CASE(2, 4)
    STG_MMA_CASE(3, 1) STG_MMA_CASE(3, 2) STG_MMA_CASE(3, 3) STG_MMA_CASE(3, 4)
    STG_MMA_CASE(4, 1) STG_MMA_CASE(4, 2) STG_MMA_CASE(4, 3) STG_MMA_CASE(4, 4)
#undef STG_MMA_CASE
    case 17: warp_mma<4, 4, true, KA, XA, KB, YB, KR>(acc, pa, pb); break;
    default: break;
  }
}

__device__ __forceinline__ int frags_left(i64 extent, i64 base) {
  const i64 f = (extent - base + 7) / 8;
  return f < 0 ? 0 : f > 4 ? 4 : static_cast<int>(f);
}

template <int TW>
__device__ __forceinline__ void load_k_tile_w(double* s, const double* g, int ld, i64 r, i64 rend, int c0, int m,
                                              const int* mask, int mask_val) {
  constexpr int STR = TW + 4, PAIRS = TW / 2, CH = BK2 * PAIRS / NT;
#pragma unroll
  for (int q = 0; q < CH; ++q) {
    const int c = threadIdx.x + NT * q;
    const int row = c / PAIRS, col = (c % PAIRS) * 2;
    i64 gr = r + row;
    const int gc = c0 + col;
    double* dst = s + row * STR + col;
    if (mask && gr < rend && mask[gr] == mask_val) gr = rend;
    if (gr < rend && gc + 2 <= m) {
      cp_async_pair(dst, g + gr * ld + gc);
    } else {
      dst[0] = (gr < rend && gc < m) ? g[gr * ld + gc] : 0.0;
      dst[1] = (gr < rend && gc + 1 < m) ? g[gr * ld + gc + 1] : 0.0;
    }
  }
}

template <bool FULL, int WM, int WN>
__device__ __forceinline__ void gram_tile(const GramArgs& a, int ti, int tj, i64 r0, i64 r1, double* smem) {
  constexpr int TA = 32 * WM, TB = 32 * WN, SA = TA + 4, SB = TB + 4;
  double* sA = smem;                   // [2][BK2][SA]
  double* sB = smem + 2 * BK2 * SA;    // [2][BK2][SB]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  const int ibase = ti * TA + wm * 32, jbase = tj * TB + wn * 32;
  int nx = FULL ? 4 : frags_left(a.m1, ibase);
  const int ny = FULL ? 4 : frags_left(a.m2, jbase);
  bool tri = false;
  if (a.sym) {  // square warp tiles: strictly below the diagonal -> mirrored by the reduction
    if (ibase >= jbase + 32) nx = 0;
    tri = ibase == jbase;
  }
  const int code = warp_code(nx, ny, tri);
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const i64 nchunks = r1 > r0 ? cdiv(r1 - r0, BK2) : 0;
  if (nchunks > 0) {
    load_k_tile_w<TA>(sA, a.A, a.lda, r0, r1, ti * TA, a.m1, a.mask, a.mask_val);
    load_k_tile_w<TB>(sB, a.B, a.ldb, r0, r1, tj * TB, a.m2, a.mask, a.mask_val);
    cp_async_commit();
  }
  for (i64 c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    if (c + 1 < nchunks) {
      load_k_tile_w<TA>(sA + (s ^ 1) * BK2 * SA, a.A, a.lda, r0 + (c + 1) * BK2, r1, ti * TA, a.m1, a.mask,
                        a.mask_val);
      load_k_tile_w<TB>(sB + (s ^ 1) * BK2 * SB, a.B, a.ldb, r0 + (c + 1) * BK2, r1, tj * TB, a.m2, a.mask,
                        a.mask_val);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* pa = sA + s * BK2 * SA + t * SA + wm * 32 + g;
    const double* pb = sB + s * BK2 * SB + t * SB + wn * 32 + g;
    if (code == 16)
      warp_mma<4, 4, false, SA, 8, SB, 8>(acc, pa, pb);
    else
      warp_mma_dispatch<SA, 8, SB, 8>(code, acc, pa, pb);
    __syncthreads();
  }
  if (code == 0) return;
  const i64 m1p = static_cast<i64>(a.tiles_i) * TA, m2p = static_cast<i64>(a.tiles_j) * TB;
  double* out = a.partial + static_cast<i64>(blockIdx.y) * m1p * m2p;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      if (x >= nx || y >= ny) continue;
      const i64 i = ibase + x * 8 + g, j = jbase + y * 8 + 2 * t;
      *reinterpret_cast<double2*>(out + i * m2p + j) = make_double2(acc[x][y][0], acc[x][y][1]);
    }
}

template <int WM, int WN>
__global__ void __launch_bounds__(NT, WM == WN ? 3 : 2) gram_tn_kernel(GramArgs a) {
  extern __shared__ __align__(16) double dsm[];
  int ti, tj;
  if (a.sym) {
    int t = blockIdx.x;
    ti = 0;
    while (t >= a.tiles_i - ti) {
      t -= a.tiles_i - ti;
      ++ti;
    }
    tj = ti + t;
  } else {
    ti = blockIdx.x / a.tiles_j;
    tj = blockIdx.x % a.tiles_j;
  }
  const i64 r0 = static_cast<i64>(blockIdx.y) * a.rows_per_split;
  const i64 r1 = min(a.nrows, r0 + a.rows_per_split);
  if ((ti + 1) * 32 * WM <= a.m1 && (tj + 1) * 32 * WN <= a.m2)
    gram_tile<true, WM, WN>(a, ti, tj, r0, r1, dsm);
  else
    gram_tile<false, WM, WN>(a, ti, tj, r0, r1, dsm);
}

// ---- TMA pipeline variant (default when the operands are 16-byte aligned
// and no row mask applies). Each 16-row stage of the A and B column slabs is
// one 2-D TMA box per operand ({32 WM + 4} x 16 and {32 WN + 4} x 16: the box
// is 4 columns wider than the tile, so it lands with the conflict-free padded
// row pitch; columns/rows outside the matrix arrive as zeros). kStages stages
// form a ring with full (transaction-counted) and empty mbarriers: the four
// warps never meet at a CTA barrier and no thread computes load addresses.
#ifndef STG_GRAM_STAGES
#define STG_GRAM_STAGES 4
#endif
#ifndef STG_GRAM_MINB
#define STG_GRAM_MINB 3
#endif
#ifndef STG_EMPTY_PER_WARP
#define STG_EMPTY_PER_WARP 0
#endif
#ifndef STG_GRAM_KBK
#define STG_GRAM_KBK 16
#endif
#ifndef STG_GRAM_PW
#define STG_GRAM_PW 0
#endif
constexpr int kBK = STG_GRAM_KBK, kStages = STG_GRAM_STAGES;
// gram_persist_rs_kernel: a fifth warp only issues the TMA loads (the DMMA warps never wait on a stage
// release), 32-row stages, two of them (tools/microbench/gram_pipe.cu: 200 x 200 sym 177 -> 158 us)
#ifndef STG_RS_KBK
#define STG_RS_KBK 32
#endif
#ifndef STG_RS_STAGES
#define STG_RS_STAGES 2
#endif
#ifndef STG_RS_PW
#define STG_RS_PW 1
#endif
constexpr int kRsBK = STG_RS_KBK, kRsStages = STG_RS_STAGES, kGramPW = STG_RS_PW;
constexpr int kRsThreads = NT + 32 * kGramPW;
constexpr size_t kRsSmem = 128 + sizeof(double) * kRsStages * kRsBK * 2 * 68;
// consumers release a stage per thread (NT arrivals) or, after __syncwarp, through one lane per warp
constexpr unsigned kEmptyCount = STG_EMPTY_PER_WARP ? NT / 32 : NT;
__device__ __forceinline__ void release_stage(unsigned long long* bar) {
  __syncwarp();
  if (!STG_EMPTY_PER_WARP || (threadIdx.x & 31) == 0) mbar_arrive(bar);
}

template <int WM, int WN>
constexpr size_t gram_tma_smem() {
  return 128 + sizeof(double) * kStages * kBK * ((32 * WM + 4) + (32 * WN + 4));
}

template <int WM, int WN>
__global__ void __launch_bounds__(NT, WM == WN ? STG_GRAM_MINB : 2)
    gram_tma_kernel(GramArgs a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw);
  unsigned long long* empty = full + kStages;
  double* stage0 = reinterpret_cast<double*>(smraw + 128);
  constexpr int TA = 32 * WM, TB = 32 * WN, SA = TA + 4, SB = TB + 4, STG = kBK * (SA + SB);
  constexpr unsigned kStageBytes = sizeof(double) * STG;
  int ti, tj;
  if (a.sym) {
    int t = blockIdx.x;
    ti = 0;
    while (t >= a.tiles_i - ti) {
      t -= a.tiles_i - ti;
      ++ti;
    }
    tj = ti + t;
  } else {
    ti = blockIdx.x / a.tiles_j;
    tj = blockIdx.x % a.tiles_j;
  }
  const i64 r0 = static_cast<i64>(blockIdx.y) * a.rows_per_split;
  const i64 r1 = min(a.nrows, r0 + a.rows_per_split);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  const int ibase = ti * TA + wm * 32, jbase = tj * TB + wn * 32;
  int nx = frags_left(a.m1, ibase);
  const int ny = frags_left(a.m2, jbase);
  bool tri = false;
  if (a.sym) {
    if (ibase >= jbase + 32) nx = 0;
    tri = ibase == jbase;
  }
  const int code = warp_code(nx, ny, tri);
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kEmptyCount);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const i64 nch = r1 > r0 ? cdiv(r1 - r0, kBK) : 0;
  const int ca = ti * TA, cb = tj * TB;
  auto produce = [&](i64 q) {  // one thread
    const int st = static_cast<int>(q % kStages);
    double* sa = stage0 + st * STG;
    const int row0 = static_cast<int>(r0 + q * kBK);
    mbar_arrive_expect_tx(&full[st], kStageBytes);
    tma_load_2d(sa, &tmA, ca, row0, &full[st]);
    tma_load_2d(sa + kBK * SA, &tmB, cb, row0, &full[st]);
  };
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  if (threadIdx.x == 0)
    for (i64 q = 0; q < min(nch, static_cast<i64>(kStages - 1)); ++q) produce(q);
  for (i64 q = 0; q < nch; ++q) {
    if (threadIdx.x == 0 && q + kStages - 1 < nch) {
      const i64 qq = q + kStages - 1;  // refills the stage chunk q - 1 used
      if (qq >= kStages) mbar_wait(&empty[qq % kStages], static_cast<unsigned>((qq / kStages - 1) & 1));
      produce(qq);
    }
    const int st = static_cast<int>(q % kStages);
    mbar_wait(&full[st], static_cast<unsigned>((q / kStages) & 1));
    const double* sa = stage0 + st * STG;
    const double* pa = sa + t * SA + wm * 32 + g;
    const double* pb = sa + kBK * SA + t * SB + wn * 32 + g;
    if (code == 16)
      warp_mma<4, 4, false, SA, 8, SB, 8, kBK>(acc, pa, pb);
    else
      warp_mma_dispatch<SA, 8, SB, 8, kBK>(code, acc, pa, pb);
    release_stage(&empty[st]);  // the warp's smem reads ordered before the TMA refill
  }
  if (code == 0) return;
  const i64 m1p = static_cast<i64>(a.tiles_i) * TA, m2p = static_cast<i64>(a.tiles_j) * TB;
  double* out = a.partial + static_cast<i64>(blockIdx.y) * m1p * m2p;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      if (x >= nx || y >= ny) continue;
      const i64 i = ibase + x * 8 + g, j = jbase + y * 8 + 2 * t;
      *reinterpret_cast<double2*>(out + i * m2p + j) = make_double2(acc[x][y][0], acc[x][y][1]);
    }
}

// ---- row-split warp layout for 64 x 64 CTA tiles. Each of the four warps
// owns two 8-row fragment rows (xr0, xr1) and every live 8-column fragment of
// the tile, so a tile with F <= 8 live fragment columns costs 2 F DMMA per
// k-step in every warp: a narrow edge tile costs what it computes (the 2 x 2
// layout of 32 x 32 warp tiles pays for a full quadrant as soon as one warp
// has one), and on the diagonal tile of a symmetric Gram the rows are dealt
// (w, 7 - w), 9 upper-triangle fragments per warp instead of 16 in the busiest
// one. Fragment arithmetic and its k order are unchanged: same bits.
template <int NX, int NY, int KA, int KB, int KR>
__device__ __forceinline__ void rs_mma(double (&acc)[2][8][2], const double* pa0, const double* pa1,
                                       const double* pb) {
#pragma unroll
  for (int kk = 0; kk < KR; kk += 4) {
    double fa[2], fb[NY];
    fa[0] = pa0[kk * KA];
    fa[1] = NX == 2 ? pa1[kk * KA] : 0.0;
#pragma unroll
    for (int y = 0; y < NY; ++y) fb[y] = pb[kk * KB + y * 8];
#pragma unroll
    for (int x = 0; x < NX; ++x)
#pragma unroll
      for (int y = 0; y < NY; ++y) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
  }
}

// full diagonal tile, warp W: fragment rows W (columns >= W) and 7 - W (columns >= 7 - W)
template <int W, int KA, int KB, int KR>
__device__ __forceinline__ void rs_mma_tri(double (&acc)[2][8][2], const double* pa0, const double* pa1,
                                           const double* pb) {
#pragma unroll
  for (int kk = 0; kk < KR; kk += 4) {
    double fb[8];
    const double fa0 = pa0[kk * KA], fa1 = pa1[kk * KA];
#pragma unroll
    for (int y = W; y < 8; ++y) fb[y] = pb[kk * KB + y * 8];
#pragma unroll
    for (int y = W; y < 8; ++y) dmma(acc[0][y][0], acc[0][y][1], fa0, fb[y]);
#pragma unroll
    for (int y = 7 - W; y < 8; ++y) dmma(acc[1][y][0], acc[1][y][1], fa1, fb[y]);
  }
}

// any shape (ragged diagonal tiles): warp-uniform guards at run time
template <int KA, int KB, int KR>
__device__ __forceinline__ void rs_mma_any(double (&acc)[2][8][2], const double* pa0, const double* pa1,
                                           const double* pb, int nx, int ylo0, int ylo1, int F) {
#pragma unroll
  for (int kk = 0; kk < KR; kk += 4) {
    const double fa0 = pa0[kk * KA], fa1 = pa1[kk * KA];
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      if (y >= F) break;
      const double fb = pb[kk * KB + y * 8];
      if (nx > 0 && y >= ylo0) dmma(acc[0][y][0], acc[0][y][1], fa0, fb);
      if (nx > 1 && y >= ylo1) dmma(acc[1][y][0], acc[1][y][1], fa1, fb);
    }
  }
}

// code: 0 none; 1..16 = (nx - 1) * 8 + F; 17..20 = full diagonal tile, warp code - 17; 21 = rs_mma_any
template <int KA, int KB, int KR>
__device__ __forceinline__ void rs_dispatch(int code, double (&acc)[2][8][2], const double* pa0, const double* pa1,
                                            const double* pb, int nx, int ylo0, int ylo1, int F) {
  switch (code) {
#define STG_RS_CASE(NX, NY) \
  case (NX - 1) * 8 + NY: rs_mma<NX, NY, KA, KB, KR>(acc, pa0, pa1, pb); break;
    STG_RS_CASE(1, 1) STG_RS_CASE(1, 2) STG_RS_CASE(1, 3) STG_RS_CASE(1, 4)
    STG_RS_CASE(1, 5) STG_RS_CASE(1, 6) STG_RS_CASE(1, 7) STG_RS_CASE(1, 8)
    STG_RS_CASE(2, 1) STG_RS_CASE(2, 2) STG_RS_CASE(2, 3) STG_RS_CASE(2, 4)
    STG_RS_CASE(2, 5) STG_RS_CASE(2, 6) STG_RS_CASE(2, 7) STG_RS_CASE(2, 8)
#undef STG_RS_CASE
    case 17: rs_mma_tri<0, KA, KB, KR>(acc, pa0, pa1, pb); break;
    case 18: rs_mma_tri<1, KA, KB, KR>(acc, pa0, pa1, pb); break;
    case 19: rs_mma_tri<2, KA, KB, KR>(acc, pa0, pa1, pb); break;
    case 20: rs_mma_tri<3, KA, KB, KR>(acc, pa0, pa1, pb); break;
    case 21: rs_mma_any<KA, KB, KR>(acc, pa0, pa1, pb, nx, ylo0, ylo1, F); break;
    default: break;
  }
}

__device__ __forceinline__ int frags8_left(i64 extent, i64 base) {
  const i64 f = (extent - base + 7) / 8;
  return f < 0 ? 0 : f > 8 ? 8 : static_cast<int>(f);
}

// Persistent split-K Gram on 64 x 64 tiles in the row-split layout (the
// scheduling of gram_persist_kernel below; same partial format).
__global__ void __launch_bounds__(kRsThreads, STG_GRAM_MINB)
    gram_persist_rs_kernel(GramArgs a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           int ntiles, int splits, int* ctr) {
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw);
  unsigned long long* empty = full + kRsStages;
  int2* meta = reinterpret_cast<int2*>(smraw + 64);
  double* stage0 = reinterpret_cast<double*>(smraw + 128);
  constexpr int SA = 68, SB = 68, STG = kRsBK * (SA + SB);
  constexpr unsigned kStageBytes = sizeof(double) * STG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int total = ntiles * splits;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kRsStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kEmptyCount);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto tile_of = [&](int tile, int& ti, int& tj) {
    if (a.sym) {
      int r = tile;
      ti = 0;
      while (r >= a.tiles_i - ti) {
        r -= a.tiles_i - ti;
        ++ti;
      }
      tj = ti + r;
    } else {
      ti = tile / a.tiles_j;
      tj = tile % a.tiles_j;
    }
  };
  auto item_of = [&](int item, int& tile, int& split) {
    if (!a.ordered) {
      tile = item % ntiles;
      split = item / ntiles;
      return;
    }
    const int per = a.block_splits * ntiles;  // items of a full block
    const int blk = item / per, r = item - blk * per;
    const int tb = min(a.block_splits, splits - blk * a.block_splits);  // the last block may be shorter
    tile = a.order[r / tb];
    split = blk * a.block_splits + r % tb;
  };
  auto chunks_of = [&](int split) {
    const i64 r0 = static_cast<i64>(split) * a.rows_per_split;
    const i64 r1 = min(a.nrows, r0 + a.rows_per_split);
    return r1 > r0 ? static_cast<int>(cdiv(r1 - r0, kRsBK)) : 0;
  };
  int p_item = -1, p_q = 0, p_nch = 0, p_ca = 0, p_cb = 0, p_row0 = 0;
  bool p_done = false, p_one = false;  // p_one: diagonal tile of a symmetric Gram, both operands are one box
  auto produce = [&](int i) {
    const int st = i % kRsStages;
    if (i >= kRsStages) mbar_wait(&empty[st], static_cast<unsigned>((i / kRsStages - 1) & 1));
    if (p_q == p_nch) {
      const int item = atomicAdd(&ctr[0], 1);
      if (item >= total) {
        p_done = true;
        if (atomicAdd(&ctr[1], 1) == static_cast<int>(gridDim.x) - 1) {
          ctr[0] = 0;
          ctr[1] = 0;
        }
        meta[st] = make_int2(-1, 0);
        mbar_arrive(&full[st]);
        return;
      }
      int ti, tj;
      int p_split, p_tl;
      item_of(item, p_tl, p_split);
      tile_of(p_tl, ti, tj);
      p_item = item;
      p_q = 0;
      p_ca = ti * 64;
      p_cb = tj * 64;
      p_one = a.sym && ti == tj && a.A == a.B && a.lda == a.ldb;  // (a symmetric product Z'(AZ) has two operands)
      p_row0 = static_cast<int>(static_cast<i64>(p_split) * a.rows_per_split);
      p_nch = chunks_of(p_split);
    }
    meta[st] = make_int2(p_item, p_q);
    double* sa = stage0 + st * STG;
    mbar_arrive_expect_tx(&full[st], p_one ? kStageBytes / 2 : kStageBytes);
    tma_load_2d(sa, &tmA, p_ca, p_row0 + p_q * kRsBK, &full[st]);
    if (!p_one) tma_load_2d(sa + kRsBK * SA, &tmB, p_cb, p_row0 + p_q * kRsBK, &full[st]);
    ++p_q;
  };
  if (kGramPW) {
    if (warp == 4) {
      if (lane == 0)
        for (int i = 0; !p_done; ++i) produce(i);
      return;
    }
  } else if (threadIdx.x == 0) {
    for (int i = 0; i < kRsStages - 1 && !p_done; ++i) produce(i);
  }
  double acc[2][8][2];
  int nx = 0, F = 0, code = 0, nch = 0, split = 0, xr0 = 0, xr1 = 0, ylo0 = 0, ylo1 = 0, ti = 0, tj = 0, boff = 0;
  for (int i = 0;; ++i) {
    if (!kGramPW && threadIdx.x == 0 && !p_done) produce(i + kRsStages - 1);
    const int st = i % kRsStages;
    mbar_wait(&full[st], static_cast<unsigned>((i / kRsStages) & 1));
    const int2 m = meta[st];
    if (m.x < 0) break;
    if (m.y == 0) {  // a new item
      int tl;
      item_of(m.x, tl, split);
      tile_of(tl, ti, tj);
      nch = chunks_of(split);
      const int R = frags8_left(a.m1, ti * 64);  // live fragment rows / columns of this tile
      F = frags8_left(a.m2, tj * 64);
      const bool diag = a.sym && ti == tj;
      boff = diag && a.A == a.B && a.lda == a.ldb ? 0 : kRsBK * SA;  // one operand: the diagonal tile's B box is its A box
      xr0 = warp;
      xr1 = diag ? 7 - warp : warp + 4;
      nx = (xr0 < R ? 1 : 0) + (xr1 < R ? 1 : 0);  // xr0 < xr1, so nx == 1 means row xr0 only
      ylo0 = diag ? xr0 : 0;
      ylo1 = diag ? xr1 : 0;
      code = nx == 0 || F == 0 ? 0 : !diag ? (nx - 1) * 8 + F : (R == 8 && F == 8) ? 17 + warp : 21;
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    }
    const double* sa = stage0 + st * STG;
    const double* pa0 = sa + t * SA + xr0 * 8 + g;
    const double* pa1 = sa + t * SA + xr1 * 8 + g;
    const double* pb = sa + boff + t * SB + g;
#ifndef STG_SKIP_MMA  // (development: the operand pipeline alone)
    if (code == 16)
      rs_mma<2, 8, SA, SB, kRsBK>(acc, pa0, pa1, pb);
    else
      rs_dispatch<SA, SB, kRsBK>(code, acc, pa0, pa1, pb, nx, ylo0, ylo1, F);
#else
    acc[0][0][0] += pa0[0] + pa1[0] + pb[0];
#endif
    release_stage(&empty[st]);
    if (m.y != nch - 1 || code == 0) continue;
    const i64 m1p = static_cast<i64>(a.tiles_i) * 64, m2p = static_cast<i64>(a.tiles_j) * 64;
    double* out = a.partial + static_cast<i64>(split) * m1p * m2p;
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      if (x >= nx) continue;
      const i64 ii = ti * 64 + (x ? xr1 : xr0) * 8 + g;
      const int ylo = x ? ylo1 : ylo0;
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        if (y >= F || y < ylo) continue;
        const i64 jj = tj * 64 + y * 8 + 2 * t;
        *reinterpret_cast<double2*>(out + ii * m2p + jj) = make_double2(acc[x][y][0], acc[x][y][1]);
      }
    }
  }
}

// Host: a.order = the 64 x 64 tiles sorted by DMMA fragments (heaviest first, ties in tile order).
inline void gram_tile_order(GramArgs& a, int ntiles, int splits, int block) {
  a.ordered = 0;
  if (ntiles > 64) return;
  a.block_splits = block > 0 ? std::min(splits, block) : splits;
  int w[64], idx = 0;
  for (int ti = 0; ti < a.tiles_i; ++ti)
    for (int tj = a.sym ? ti : 0; tj < a.tiles_j; ++tj) {
      const int R = static_cast<int>(std::min<i64>(8, cdiv(a.m1 - ti * 64, 8)));
      const int F = static_cast<int>(std::min<i64>(8, cdiv(a.m2 - tj * 64, 8)));
      w[idx++] = a.sym && ti == tj ? R * (R + 1) / 2 : R * F;
    }
  for (int i = 0; i < ntiles; ++i) a.order[i] = static_cast<unsigned char>(i);
  std::stable_sort(a.order, a.order + ntiles, [&](unsigned char x, unsigned char y) { return w[x] > w[y]; });
  a.ordered = 1;
}

// Persistent variant of gram_tma_kernel: a fixed grid pulls (split, tile) items
// from a device counter (split major: the tiles of one row range run side by
// side and share its rows in L2) and streams their 16-row chunks through one
// TMA ring that keeps running across items, so the next item's rows are in
// flight while this item's partial tile is stored, and light edge / diagonal
// tiles balance themselves against full ones. Item (split, tile) writes the
// same partial slot whichever CTA computes it: the reduction order and the
// result do not depend on the schedule. ctr as in gemm_nn_persist_kernel.
template <int WM, int WN>
__global__ void __launch_bounds__(kRsThreads, WM == WN ? STG_GRAM_MINB : 2)
    gram_persist_kernel(GramArgs a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        int ntiles, int splits, int* ctr) {
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw);
  unsigned long long* empty = full + kStages;
  int2* meta = reinterpret_cast<int2*>(smraw + 64);  // per stage: (item, chunk); item < 0 ends the CTA
  static_assert(kStages * 16 <= 64 && kStages * 8 <= 64, "barriers and item tags share the 128-byte header");
  double* stage0 = reinterpret_cast<double*>(smraw + 128);
  constexpr int TA = 32 * WM, TB = 32 * WN, SA = TA + 4, SB = TB + 4, STG = kBK * (SA + SB);
  constexpr unsigned kStageBytes = sizeof(double) * STG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  const int total = ntiles * splits;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kEmptyCount);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto tile_of = [&](int tile, int& ti, int& tj) {
    if (a.sym) {
      int r = tile;
      ti = 0;
      while (r >= a.tiles_i - ti) {
        r -= a.tiles_i - ti;
        ++ti;
      }
      tj = ti + r;
    } else {
      ti = tile / a.tiles_j;
      tj = tile % a.tiles_j;
    }
  };
  auto chunks_of = [&](int split) {
    const i64 r0 = static_cast<i64>(split) * a.rows_per_split;
    const i64 r1 = min(a.nrows, r0 + a.rows_per_split);
    return r1 > r0 ? static_cast<int>(cdiv(r1 - r0, kBK)) : 0;
  };
  // ---- producer state (thread 0)
  int p_item = -1, p_q = 0, p_nch = 0, p_ca = 0, p_cb = 0, p_row0 = 0;
  bool p_done = false;
  auto produce = [&](int i) {
    const int st = i % kStages;
    if (i >= kStages) mbar_wait(&empty[st], static_cast<unsigned>((i / kStages - 1) & 1));
    if (p_q == p_nch) {
      const int item = atomicAdd(&ctr[0], 1);
      if (item >= total) {
        p_done = true;
        if (atomicAdd(&ctr[1], 1) == static_cast<int>(gridDim.x) - 1) {
          ctr[0] = 0;
          ctr[1] = 0;
        }
        meta[st] = make_int2(-1, 0);
        mbar_arrive(&full[st]);
        return;
      }
      int ti, tj;
      tile_of(item % ntiles, ti, tj);
      p_item = item;
      p_q = 0;
      p_ca = ti * TA;
      p_cb = tj * TB;
      p_row0 = static_cast<int>(static_cast<i64>(item / ntiles) * a.rows_per_split);
      p_nch = chunks_of(item / ntiles);  // >= 1: the host sizes the splits from the row count
    }
    meta[st] = make_int2(p_item, p_q);
    double* sa = stage0 + st * STG;
    mbar_arrive_expect_tx(&full[st], kStageBytes);
    tma_load_2d(sa, &tmA, p_ca, p_row0 + p_q * kBK, &full[st]);
    tma_load_2d(sa + kBK * SA, &tmB, p_cb, p_row0 + p_q * kBK, &full[st]);
    ++p_q;
  };
  if (kGramPW) {  // the fifth warp only issues the loads
    if (warp == 4) {
      if (lane == 0)
        for (int i = 0; !p_done; ++i) produce(i);
      return;
    }
  } else if (threadIdx.x == 0) {
    for (int i = 0; i < kStages - 1 && !p_done; ++i) produce(i);
  }
  double acc[4][4][2];
  int nx = 0, ny = 0, code = 0, nch = 0, ibase = 0, jbase = 0, split = 0;
  for (int i = 0;; ++i) {
    if (!kGramPW && threadIdx.x == 0 && !p_done) produce(i + kStages - 1);
    const int st = i % kStages;
    mbar_wait(&full[st], static_cast<unsigned>((i / kStages) & 1));
    const int2 m = meta[st];
    if (m.x < 0) break;
    if (m.y == 0) {  // a new item
      int ti, tj;
      tile_of(m.x % ntiles, ti, tj);
      split = m.x / ntiles;
      nch = chunks_of(split);
      ibase = ti * TA + wm * 32;
      jbase = tj * TB + wn * 32;
      nx = frags_left(a.m1, ibase);
      ny = frags_left(a.m2, jbase);
      bool tri = false;
      if (a.sym) {
        if (ibase >= jbase + 32) nx = 0;
        tri = ibase == jbase;
      }
      code = warp_code(nx, ny, tri);
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    }
    const double* sa = stage0 + st * STG;
    const double* pa = sa + t * SA + wm * 32 + g;
    const double* pb = sa + kBK * SA + t * SB + wn * 32 + g;
    if (code == 16)
      warp_mma<4, 4, false, SA, 8, SB, 8, kBK>(acc, pa, pb);
    else
      warp_mma_dispatch<SA, 8, SB, 8, kBK>(code, acc, pa, pb);
    release_stage(&empty[st]);
    if (m.y != nch - 1 || code == 0) continue;
    const i64 m1p = static_cast<i64>(a.tiles_i) * TA, m2p = static_cast<i64>(a.tiles_j) * TB;
    double* out = a.partial + static_cast<i64>(split) * m1p * m2p;
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        if (x >= nx || y >= ny) continue;
        const i64 ii = ibase + x * 8 + g, jj = jbase + y * 8 + 2 * t;
        *reinterpret_cast<double2*>(out + ii * m2p + jj) = make_double2(acc[x][y][0], acc[x][y][1]);
      }
  }
}

// Deterministic split reduction, one thread per output element (consecutive
// threads on consecutive columns, so every split's partial row is read
// coalesced), splits summed in order with 8 loads in flight. For sym only the
// computed upper triangle (i <= j) is read and written to both (i, j) and
// (j, i): the result is exactly symmetric.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double* partial, int splits, int m1, int m2, int m1p,
                                                          int m2p, int sym, double* out, int ldo, double alpha) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(m1) * m2) return;
  const int i = static_cast<int>(idx / m2), j = static_cast<int>(idx % m2);
  if (sym && j < i) return;
  const i64 stride = static_cast<i64>(m1p) * m2p;
  const double* src = partial + static_cast<i64>(i) * m2p + j;
  double s = 0.0;
  int sp = 0;
  for (; sp + 8 <= splits; sp += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = __ldcs(src + (sp + u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += t[u];
  }
  for (; sp < splits; ++sp) s += __ldcs(src + sp * stride);
  out[static_cast<i64>(i) * ldo + j] = alpha * s;
  if (sym && i != j) out[static_cast<i64>(j) * ldo + i] = alpha * s;
}

// Split reduction with the splits cut into CH consecutive chunks: warp c of a
// CTA sums chunk c of 32 consecutive output elements (lane = element, so each
// split's partial row is read coalesced) in split order with 8 loads in
// flight, then warp 0 adds the CH chunk sums in chunk order. The association
// is fixed by (splits, CH): deterministic. The latency chain per element is
// splits / CH loads instead of splits. sym as gram_reduce_kernel.
__global__ void __launch_bounds__(1024) gram_reduce_chunked_kernel(const double* partial, int splits, int m1, int m2,
                                                                   int m1p, int m2p, int sym, double* out, int ldo,
                                                                   double alpha) {
  __shared__ double red[32][33];
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5, CH = blockDim.x >> 5;
  const i64 idx = static_cast<i64>(blockIdx.x) * 32 + lane;
  const bool live = idx < static_cast<i64>(m1) * m2;
  const int i = live ? static_cast<int>(idx / m2) : 0, j = live ? static_cast<int>(idx % m2) : 0;
  const bool act = live && !(sym && j < i);
  double s = 0.0;
  if (act) {
    const i64 stride = static_cast<i64>(m1p) * m2p;
    const int s0 = static_cast<int>(static_cast<i64>(splits) * c / CH);
    const int s1 = static_cast<int>(static_cast<i64>(splits) * (c + 1) / CH);
    const double* src = partial + static_cast<i64>(i) * m2p + j;
    int sp = s0;
    for (; sp + 8 <= s1; sp += 8) {
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = __ldcs(src + (sp + u) * stride);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += t[u];
    }
    for (; sp < s1; ++sp) s += __ldcs(src + sp * stride);
  }
  red[c][lane] = s;
  __syncthreads();
  if (c != 0 || !act) return;
  double tot = red[0][lane];
  for (int q = 1; q < CH; ++q) tot += red[q][lane];
  out[static_cast<i64>(i) * ldo + j] = alpha * tot;
  if (sym && i != j) out[static_cast<i64>(j) * ldo + i] = alpha * tot;
}

// chunk count: ~12 splits per chunk, at most 32 warps
inline int gram_reduce_chunks(i64 splits) { return static_cast<int>(std::max<i64>(1, std::min<i64>(32, splits / 12))); }

// (previous layout, one warp per output element, kept for A/B) lane l sums
// splits l, l+32, ... in order, then a fixed butterfly combines the lanes. For
// sym the (min, max) element is read so the result is exactly symmetric.
__global__ void __launch_bounds__(256) gram_reduce_warp_kernel(const double* partial, int splits, int m1, int m2,
                                                               int m1p, int m2p, int sym, double* out, int ldo,
                                                               double alpha) {
  const i64 idx = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (idx >= static_cast<i64>(m1) * m2) return;
  const int i = static_cast<int>(idx / m2), j = static_cast<int>(idx % m2);
  int ii = i, jj = j;
  if (sym && ((i / BM) > (j / BN) || (i > j && (i / BM) == (j / BN)))) {
    ii = j;
    jj = i;
  }
  const i64 stride = static_cast<i64>(m1p) * m2p;
  const double* src = partial + static_cast<i64>(ii) * m2p + jj;
  double s = 0.0;
  for (int sp = lane; sp < splits; sp += 32) s += src[sp * stride];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[static_cast<i64>(i) * ldo + j] = alpha * s;
}


// ---- narrow variants (all dims <= 32): one 32 x 32 output tile per CTA,
// the four warps split the rows of each stage (gram) or the output rows (nn),
// so no warp idles on out-of-range subtiles.
constexpr int SBK = 32;      // rows per gram stage
constexpr int SS = 36;       // [*][32] tiles: stride == 4 (mod 16)

__device__ __forceinline__ void load_k_tile32(double (*s)[SS], const double* g, int ld, i64 r, i64 rend, int m,
                                              const int* mask, int mask_val) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = threadIdx.x + NT * q;  // 512 chunks: 32 rows x 16 pairs
    const int row = c >> 4, col = (c & 15) * 2;
    i64 gr = r + row;
    double* dst = &s[row][col];
    if (mask && gr < rend && mask[gr] == mask_val) gr = rend;
    if (gr < rend && col + 2 <= m) {
      cp_async_pair(dst, g + gr * ld + col);
    } else {
      dst[0] = (gr < rend && col < m) ? g[gr * ld + col] : 0.0;
      dst[1] = 0.0;
    }
  }
}

__global__ void __launch_bounds__(NT) gram_tn_small_kernel(GramArgs a) {
  const i64 r0 = static_cast<i64>(blockIdx.y) * a.rows_per_split;
  const i64 r1 = min(a.nrows, r0 + a.rows_per_split);
  __shared__ __align__(16) double sA[2][SBK][SS];
  __shared__ __align__(16) double sB[2][SBK][SS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  bool vi[4], vj[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    vi[x] = x * 8 < a.m1;
    vj[x] = x * 8 < a.m2;
  }
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const i64 nchunks = r1 > r0 ? cdiv(r1 - r0, SBK) : 0;
  const bool same = a.A == a.B && a.lda == a.ldb;  // A'A: stage the block once
  if (nchunks > 0) {
    load_k_tile32(sA[0], a.A, a.lda, r0, r1, a.m1, a.mask, a.mask_val);
    if (!same) load_k_tile32(sB[0], a.B, a.ldb, r0, r1, a.m2, a.mask, a.mask_val);
    cp_async_commit();
  }
  for (i64 c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    if (c + 1 < nchunks) {
      load_k_tile32(sA[s ^ 1], a.A, a.lda, r0 + (c + 1) * SBK, r1, a.m1, a.mask, a.mask_val);
      if (!same) load_k_tile32(sB[s ^ 1], a.B, a.ldb, r0 + (c + 1) * SBK, r1, a.m2, a.mask, a.mask_val);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = warp * 8; kk < warp * 8 + 8; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        fa[x] = sA[s][kk + t][x * 8 + g];
        fb[x] = same ? fa[x] : sB[s][kk + t][x * 8 + g];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
          if (vi[x] && vj[y]) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
    }
    __syncthreads();
  }
  // reduce the four warps' tiles through shared memory (fixed order)
  double* red = &sA[0][0][0];  // 4 x 32 x 32 doubles fit in sA + sB
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = x * 8 + g, j = y * 8 + 2 * t;
      red[warp * 1024 + i * 32 + j] = acc[x][y][0];
      red[warp * 1024 + i * 32 + j + 1] = acc[x][y][1];
    }
  __syncthreads();
  double* out = a.partial + static_cast<i64>(blockIdx.y) * 1024;
  for (int e = threadIdx.x; e < 1024; e += NT)
    out[e] = ((red[e] + red[1024 + e]) + red[2048 + e]) + red[3072 + e];
}

constexpr int NBM = 128, NBK = 8, NSAR = 12;  // narrow nn: 128 rows x 32 cols, K chunks of 8


struct NNArgs {
  const double* A;
  int lda;
  i64 nrows;
  int m1;
  const double* C;
  int ldc;
  int m2;
  const double* Bm;
  int ldb;
  double* Out;
  int ldo;
  double alpha, beta;
  int upper_tri_c;  // C upper triangular (zeros stored below): skip K chunks past the column tile
  const int* skip_flags;  // optional: do nothing when (*skip_flags & skip_mask) or *skip_info != 0
  int skip_mask;
  const int* skip_info;
};

__device__ __forceinline__ bool nn_skipped(const NNArgs& a) {
  return a.skip_flags && ((*a.skip_flags & a.skip_mask) || *a.skip_info != 0);
}

constexpr int SAR2 = BK2 + 4;  // [64][32] A tiles: stride 36 == 4 (mod 16)
constexpr size_t kNNSmem = sizeof(double) * 2 * (BM * SAR2 + BK2 * SST);

template <bool FULL, bool BETA>
__device__ __forceinline__ void nn_tile(const NNArgs& a, i64 row0, int tj, double* smem) {
  double* sA = smem;                  // [2][BM][SAR2]
  double* sC = smem + 2 * BM * SAR2;  // [2][BK2][SST]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int kmax = a.upper_tri_c ? min(a.m1, (tj + 1) * BN) : a.m1;
  const int nk = static_cast<int>(cdiv(kmax, BK2));
  const int code = FULL ? 16 : warp_code(frags_left(a.nrows, row0 + wm * 32), frags_left(a.m2, tj * BN + wn * 32), false);
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  // beta * B for the epilogue: issued before the K loop so its latency
  // overlaps the operand loads (the short-K projections are memory bound)
  double bpre[BETA ? 4 : 1][4][2];
  if (FULL && BETA) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const i64 r = row0 + wm * 32 + x * 8 + g;
        const int col = tj * BN + wn * 32 + y * 8 + 2 * t;
        const double2 v = *reinterpret_cast<const double2*>(a.Bm + r * a.ldb + col);
        bpre[x][y][0] = v.x;
        bpre[x][y][1] = v.y;
      }
  }
  auto load = [&](int s, int k0) {
    double* A_s = sA + s * BM * SAR2;
    double* C_s = sC + s * BK2 * SST;
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // A: 64 rows x 32 cols = 1024 pairs
      const int c = threadIdx.x + NT * q;
      const int row = c >> 4, col = (c & 15) * 2;
      const i64 gr = row0 + row;
      const int gk = k0 + col;
      double* dst = A_s + row * SAR2 + col;
      if (gr < a.nrows && gk + 2 <= a.m1) {
        cp_async_pair(dst, a.A + gr * a.lda + gk);
      } else {
        dst[0] = (gr < a.nrows && gk < a.m1) ? a.A[gr * a.lda + gk] : 0.0;
        dst[1] = (gr < a.nrows && gk + 1 < a.m1) ? a.A[gr * a.lda + gk + 1] : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // C: 32 rows x 64 cols = 1024 pairs
      const int c = threadIdx.x + NT * q;
      const int row = c >> 5, col = (c & 31) * 2;
      const int gk = k0 + row, gc = tj * BN + col;
      double* dst = C_s + row * SST + col;
      if (gk < a.m1 && gc + 2 <= a.m2) {
        cp_async_pair(dst, a.C + static_cast<i64>(gk) * a.ldc + gc);
      } else {
        dst[0] = (gk < a.m1 && gc < a.m2) ? a.C[static_cast<i64>(gk) * a.ldc + gc] : 0.0;
        dst[1] = (gk < a.m1 && gc + 1 < a.m2) ? a.C[static_cast<i64>(gk) * a.ldc + gc + 1] : 0.0;
      }
    }
  };
  if (nk > 0) {
    load(0, 0);
    cp_async_commit();
  }
  for (int c = 0; c < nk; ++c) {
    const int s = c & 1;
    if (c + 1 < nk) {
      load(s ^ 1, (c + 1) * BK2);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* pa = sA + s * BM * SAR2 + (wm * 32 + g) * SAR2 + t;
    const double* pc = sC + s * BK2 * SST + t * SST + wn * 32 + g;
    if (code == 16)
      warp_mma<4, 4, false, 1, 8 * SAR2, SST, 8>(acc, pa, pc);
    else
      warp_mma_dispatch<1, 8 * SAR2, SST, 8>(code, acc, pa, pc);
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const i64 r = row0 + wm * 32 + x * 8 + g;
      const int col = tj * BN + wn * 32 + y * 8 + 2 * t;
      if (FULL) {
        double2 v = make_double2(a.alpha * acc[x][y][0], a.alpha * acc[x][y][1]);
        if (BETA) {
          v.x += a.beta * bpre[BETA ? x : 0][y][0];
          v.y += a.beta * bpre[BETA ? x : 0][y][1];
        }
        *reinterpret_cast<double2*>(a.Out + r * a.ldo + col) = v;
        continue;
      }
      if (r >= a.nrows) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (col + h >= a.m2) continue;
        double v = a.alpha * acc[x][y][h];
        if (a.beta != 0.0) v += a.beta * a.Bm[r * a.ldb + col + h];
        a.Out[r * a.ldo + col + h] = v;
      }
    }
}

// TMA pipeline variant of nn_tile: per 32-wide K chunk one 2-D box of A
// ({36, 64}: 64 rows, the padded K pitch) and one of C ({68, 32}); two stages
// with full/empty mbarriers; out-of-range rows/columns arrive as zeros.
constexpr int kNNStages = 2;
constexpr size_t kNNTmaSmem = 128 + sizeof(double) * kNNStages * (BM * SAR2 + BK2 * SST);

template <bool FULL, bool BETA>
__device__ __forceinline__ void nn_tma_tile(const NNArgs& a, const CUtensorMap* tmA, const CUtensorMap* tmC, i64 row0,
                                            int tj, unsigned char* smraw) {
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw);
  double* stage0 = reinterpret_cast<double*>(smraw + 128);
  constexpr int STG = BM * SAR2 + BK2 * SST;
  constexpr unsigned kStageBytes = sizeof(double) * STG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int kmax = a.upper_tri_c ? min(a.m1, (tj + 1) * BN) : a.m1;
  const int nk = static_cast<int>(cdiv(kmax, BK2));
  const int code = FULL ? 16 : warp_code(frags_left(a.nrows, row0 + wm * 32), frags_left(a.m2, tj * BN + wn * 32), false);
  if (threadIdx.x == 0) {
    for (int st = 0; st < kNNStages; ++st) mbar_init(&full[st], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto produce = [&](int q) {
    const int st = q % kNNStages;
    double* sa = stage0 + st * STG;
    mbar_arrive_expect_tx(&full[st], kStageBytes);
    tma_load_2d(sa, tmA, q * BK2, static_cast<int>(row0), &full[st]);
    tma_load_2d(sa + BM * SAR2, tmC, tj * BN, q * BK2, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < min(nk, kNNStages); ++q) produce(q);
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  double bpre[BETA ? 4 : 1][4][2];
  if (FULL && BETA) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const i64 r = row0 + wm * 32 + x * 8 + g;
        const int col = tj * BN + wn * 32 + y * 8 + 2 * t;
        const double2 v = *reinterpret_cast<const double2*>(a.Bm + r * a.ldb + col);
        bpre[x][y][0] = v.x;
        bpre[x][y][1] = v.y;
      }
  }
  // a stage is refilled only after a CTA barrier shows every warp has
  // finished reading it (the refill of chunk q + kNNStages overlaps the
  // compute of chunk q + 1)
  for (int q = 0; q < nk; ++q) {
    const int st = q % kNNStages;
    mbar_wait(&full[st], static_cast<unsigned>((q / kNNStages) & 1));
    const double* sa = stage0 + st * STG;
    const double* pa = sa + (wm * 32 + g) * SAR2 + t;
    const double* pc = sa + BM * SAR2 + t * SST + wn * 32 + g;
    if (code == 16)
      warp_mma<4, 4, false, 1, 8 * SAR2, SST, 8>(acc, pa, pc);
    else
      warp_mma_dispatch<1, 8 * SAR2, SST, 8>(code, acc, pa, pc);
    __syncthreads();
    if (threadIdx.x == 0 && q + kNNStages < nk) produce(q + kNNStages);
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const i64 r = row0 + wm * 32 + x * 8 + g;
      const int col = tj * BN + wn * 32 + y * 8 + 2 * t;
      if (FULL) {
        double2 v = make_double2(a.alpha * acc[x][y][0], a.alpha * acc[x][y][1]);
        if (BETA) {
          v.x += a.beta * bpre[BETA ? x : 0][y][0];
          v.y += a.beta * bpre[BETA ? x : 0][y][1];
        }
        *reinterpret_cast<double2*>(a.Out + r * a.ldo + col) = v;
        continue;
      }
      if (r >= a.nrows) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (col + h >= a.m2) continue;
        double v = a.alpha * acc[x][y][h];
        if (a.beta != 0.0) v += a.beta * a.Bm[r * a.ldb + col + h];
        a.Out[r * a.ldo + col + h] = v;
      }
    }
}

template <bool BETA>
__global__ void __launch_bounds__(NT, BETA ? 2 : 3)
    gemm_nn_tma_kernel(NNArgs a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC) {
  if (nn_skipped(a)) return;
  extern __shared__ __align__(128) unsigned char nsm[];
  const int tiles_j = static_cast<int>(cdiv(a.m2, BN));
  const i64 row0 = static_cast<i64>(blockIdx.x / tiles_j) * BM;
  const int tj = static_cast<int>(blockIdx.x % tiles_j);
  if (row0 + BM <= a.nrows && (tj + 1) * BN <= a.m2)
    nn_tma_tile<true, BETA>(a, &tmA, &tmC, row0, tj, nsm);
  else
    nn_tma_tile<false, BETA>(a, &tmA, &tmC, row0, tj, nsm);
}

// Persistent variant of gemm_nn_tma_kernel. A fixed grid of CTAs (a multiple
// of the SM count) pulls 64 x 64 output tiles from a device counter (row tile
// major, so the column tiles of one row block run side by side and share the A
// rows in L2) and streams their K chunks through ONE TMA ring that keeps
// running across tile boundaries: the next tile's first chunks are already in
// flight while this tile's epilogue stores, no CTA pays a pipeline fill per
// tile, and uneven tiles (upper-triangular C, narrow edge tiles) balance
// themselves. Every tile's result is independent of which CTA computes it, so
// the output is deterministic. ctr = {next tile, CTAs that saw the end}: the
// last CTA to see the end re-arms both for the next launch on this stream.
// (BETA: 176+ registers allow two CTAs per SM, which leaves room for a third stage)
#ifndef STG_NNP_NB_STAGES
#define STG_NNP_NB_STAGES 2  // beta == 0: 2 stages x 3 CTAs/SM (3 stages x 2 CTAs/SM measured: see DESIGN 8)
#endif
constexpr int nnp_stages(bool beta) { return beta ? 3 : STG_NNP_NB_STAGES; }
constexpr int nnp_ctas(bool beta) { return beta || STG_NNP_NB_STAGES > 2 ? 2 : 3; }
constexpr size_t nnp_smem(bool beta) { return 128 + sizeof(double) * nnp_stages(beta) * (BM * SAR2 + BK2 * SST); }

template <bool BETA>
__global__ void __launch_bounds__(kRsThreads, (BETA || STG_NNP_NB_STAGES > 2) ? 2 : 3)
    gemm_nn_persist_kernel(NNArgs a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC,
                           int ntr, int* ctr) {
  if (nn_skipped(a)) return;
  extern __shared__ __align__(128) unsigned char psm[];
  constexpr int kNNPStages = BETA ? 3 : STG_NNP_NB_STAGES;  // nnp_stages(BETA)
  unsigned long long* full = reinterpret_cast<unsigned long long*>(psm);
  unsigned long long* empty = full + kNNPStages;
  int2* meta = reinterpret_cast<int2*>(psm + 64);  // per stage: (tile, K chunk); tile < 0 ends the CTA
  double* stage0 = reinterpret_cast<double*>(psm + 128);
  static_assert(kNNPStages * 16 <= 64 && kNNPStages * 8 <= 64, "barriers and tile tags share the 128-byte header");
  constexpr int STG = BM * SAR2 + BK2 * SST;
  constexpr unsigned kStageBytes = sizeof(double) * STG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int xr0 = 2 * warp, xr1 = 2 * warp + 1;  // row-split layout: 16 rows x every live column fragment
  const int tiles_j = static_cast<int>(cdiv(a.m2, BN));
  const int total = ntr * tiles_j;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kNNPStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kEmptyCount);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto chunks_of = [&](int tj) {
    const int kmax = a.upper_tri_c ? min(a.m1, (tj + 1) * BN) : a.m1;
    return static_cast<int>(cdiv(kmax, BK2));
  };
  // ---- producer state (thread 0)
  int p_tile = -1, p_q = 0, p_nk = 0, p_tj = 0, p_row0 = 0;
  bool p_done = false;
  auto produce = [&](int i) {
    const int st = i % kNNPStages;
    if (i >= kNNPStages) mbar_wait(&empty[st], static_cast<unsigned>((i / kNNPStages - 1) & 1));
    if (p_q == p_nk) {
      const int tile = atomicAdd(&ctr[0], 1);
      if (tile >= total) {
        p_done = true;
        if (atomicAdd(&ctr[1], 1) == static_cast<int>(gridDim.x) - 1) {  // every CTA has seen the end
          ctr[0] = 0;
          ctr[1] = 0;
        }
        meta[st] = make_int2(-1, 0);
        mbar_arrive(&full[st]);
        return;
      }
      p_tile = tile;
      p_q = 0;
      p_tj = tiles_j - 1 - tile % tiles_j;  // the widest-K column tile of a row block first
      p_row0 = (tile / tiles_j) * BM;
      p_nk = chunks_of(p_tj);
    }
    meta[st] = make_int2(p_tile, p_q);
    double* sa = stage0 + st * STG;
    mbar_arrive_expect_tx(&full[st], kStageBytes);
    tma_load_2d(sa, &tmA, p_q * BK2, p_row0, &full[st]);
    tma_load_2d(sa + BM * SAR2, &tmC, p_tj * BN, p_q * BK2, &full[st]);
    ++p_q;
  };
  if (kGramPW) {
    // the fifth warp only issues the loads; with beta != 0 its lanes also pull each new tile of B into L2
    // (the DMMA warps read it straight from global memory at the tile's start, one to two tiles later)
    if (warp == 4) {
      for (int i = 0;; ++i) {
        int fresh = 0;
        if (lane == 0) {
          const int before = p_tile;
          produce(i);
          fresh = !p_done && p_tile != before;
        }
        fresh = __shfl_sync(0xffffffffu, fresh, 0);
        if (BETA && fresh) {
          const int row0 = __shfl_sync(0xffffffffu, p_row0, 0), c0 = __shfl_sync(0xffffffffu, p_tj, 0) * BN;
          for (int l = lane; l < BM * 4; l += 32) {  // 128-byte lines of the 64 x 64 tile
            const i64 r = row0 + (l >> 2);
            const int c = c0 + (l & 3) * 16;
            if (r < a.nrows && c < a.m2)
              asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a.Bm + r * a.ldb + c));
          }
        }
        if (__shfl_sync(0xffffffffu, p_done ? 1 : 0, 0)) break;
      }
      return;
    }
  } else if (threadIdx.x == 0) {
    for (int i = 0; i < kNNPStages - 1 && !p_done; ++i) produce(i);
  }
  double acc[2][8][2];
  double bpre[BETA ? 2 : 1][8][2];
  int tj = 0, nk = 0, code = 0, nx = 0, F = 0;
  i64 row0 = 0;
  bool whole = false;
  for (int i = 0;; ++i) {
    if (!kGramPW && threadIdx.x == 0 && !p_done) produce(i + kNNPStages - 1);
    const int st = i % kNNPStages;
    mbar_wait(&full[st], static_cast<unsigned>((i / kNNPStages) & 1));
    const int2 m = meta[st];
    if (m.x < 0) break;
    if (m.y == 0) {  // a new tile
      tj = tiles_j - 1 - m.x % tiles_j;
      row0 = static_cast<i64>(m.x / tiles_j) * BM;
      nk = chunks_of(tj);
      whole = row0 + BM <= a.nrows && (tj + 1) * BN <= a.m2;
      const int R = frags8_left(a.nrows, row0);
      F = frags8_left(a.m2, tj * BN);
      nx = (xr0 < R ? 1 : 0) + (xr1 < R ? 1 : 0);
      code = nx == 0 || F == 0 ? 0 : (nx - 1) * 8 + F;
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
      if (BETA && whole) {  // beta * B for the epilogue, in flight during the K loop
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 8; ++y) {
            const i64 r = row0 + (2 * warp + x) * 8 + g;
            const int col = tj * BN + y * 8 + 2 * t;
            const double2 v = *reinterpret_cast<const double2*>(a.Bm + r * a.ldb + col);
            bpre[BETA ? x : 0][y][0] = v.x;
            bpre[BETA ? x : 0][y][1] = v.y;
          }
      }
    }
    const double* sa = stage0 + st * STG;
    const double* pa0 = sa + (xr0 * 8 + g) * SAR2 + t;
    const double* pa1 = sa + (xr1 * 8 + g) * SAR2 + t;
    const double* pc = sa + BM * SAR2 + t * SST + g;
#ifndef STG_SKIP_MMA
    if (code == 16)
      rs_mma<2, 8, 1, SST, BK2>(acc, pa0, pa1, pc);
    else
      rs_dispatch<1, SST, BK2>(code, acc, pa0, pa1, pc, nx, 0, 0, F);
#else
    acc[0][0][0] += pa0[0] + pa1[0] + pc[0];
#endif
    release_stage(&empty[st]);
    if (m.y != nk - 1) continue;
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const i64 r = row0 + (2 * warp + x) * 8 + g;
        const int col = tj * BN + y * 8 + 2 * t;
        if (whole) {
          double2 v = make_double2(a.alpha * acc[x][y][0], a.alpha * acc[x][y][1]);
          if (BETA) {
            v.x += a.beta * bpre[BETA ? x : 0][y][0];
            v.y += a.beta * bpre[BETA ? x : 0][y][1];
          }
          *reinterpret_cast<double2*>(a.Out + r * a.ldo + col) = v;
          continue;
        }
        if (r >= a.nrows) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (col + h >= a.m2) continue;
          double v = a.alpha * acc[x][y][h];
          if (a.beta != 0.0) v += a.beta * a.Bm[r * a.ldb + col + h];
          a.Out[r * a.ldo + col + h] = v;
        }
      }
  }
}

template <bool BETA>  // the beta*B prefetch needs 64 more registers: 2 CTAs per SM
__global__ void __launch_bounds__(NT, BETA ? 2 : 3) gemm_nn_kernel(NNArgs a) {
  if (nn_skipped(a)) return;
  extern __shared__ __align__(16) double dsm[];
  // column tiles of one row block are adjacent in launch order, so the A rows
  // they share are read from HBM once
  const int tiles_j = static_cast<int>(cdiv(a.m2, BN));
  const i64 row0 = static_cast<i64>(blockIdx.x / tiles_j) * BM;
  const int tj = static_cast<int>(blockIdx.x % tiles_j);
  if (row0 + BM <= a.nrows && (tj + 1) * BN <= a.m2)
    nn_tile<true, BETA>(a, row0, tj, dsm);
  else
    nn_tile<false, BETA>(a, row0, tj, dsm);
}

// Narrow streaming NN (m1 <= 32, m2 <= 32: projections against the k-wide
// block, the final rotation X <- X A_new of all n rows). Persistent CTAs walk
// 128-row tiles; each tile of A arrives as one TMA box {36, 128} through a
// 4-deep mbarrier ring, C (<= 32 x 32) sits in shared memory once. Safe in
// place (Out == A): a tile is fully staged before its rows are written.
constexpr int kStreamRows = 128, kStreamStages = 4, kStreamPitch = 36;
constexpr size_t kStreamSmem =
    128 + sizeof(double) * (static_cast<size_t>(kStreamStages) * kStreamRows * kStreamPitch + 32 * SS);

__global__ void __launch_bounds__(NT, 2)
    gemm_nn_stream_kernel(NNArgs a, const __grid_constant__ CUtensorMap tmA, int ntiles) {
  if (nn_skipped(a)) return;
  extern __shared__ __align__(128) unsigned char ssm[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ssm);
  unsigned long long* empty = full + kStreamStages;
  double* stage0 = reinterpret_cast<double*>(ssm + 128);
  double* sC = stage0 + kStreamStages * kStreamRows * kStreamPitch;  // [32][SS]
  constexpr int STG = kStreamRows * kStreamPitch;
  constexpr unsigned kStageBytes = sizeof(double) * STG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  for (int idx = threadIdx.x; idx < 32 * 32; idx += blockDim.x) {
    const int r = idx >> 5, c = idx & 31;
    sC[r * SS + c] = (r < a.m1 && c < a.m2) ? a.C[static_cast<i64>(r) * a.ldc + c] : 0.0;
  }
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStreamStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kEmptyCount);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int G = gridDim.x, b = blockIdx.x;
  const int my = b < ntiles ? (ntiles - 1 - b) / G + 1 : 0;  // tiles b, b + G, ...
  auto produce = [&](int q) {
    const int st = q % kStreamStages;
    if (q >= kStreamStages) mbar_wait(&empty[st], static_cast<unsigned>((q / kStreamStages - 1) & 1));
    mbar_arrive_expect_tx(&full[st], kStageBytes);
    tma_load_2d(stage0 + st * STG, &tmA, 0, (b + q * G) * kStreamRows, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < min(my, kStreamStages - 1); ++q) produce(q);
  const int nxw = frags_left(a.m2, 0);  // live 8-column fragments
  for (int q = 0; q < my; ++q) {
    if (threadIdx.x == 0 && q + kStreamStages - 1 < my) produce(q + kStreamStages - 1);
    const int st = q % kStreamStages;
    mbar_wait(&full[st], static_cast<unsigned>((q / kStreamStages) & 1));
    const double* sa = stage0 + st * STG;
    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    const double* pa = sa + (warp * 32 + g) * kStreamPitch + t;
    const double* pc = sC + t * SS + g;
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        fa[x] = pa[x * 8 * kStreamPitch + kk];
        fb[x] = pc[kk * SS + x * 8];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
          if (y < nxw) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
    }
    release_stage(&empty[st]);  // A is in registers' products now; the slot may refill
    const i64 row0 = static_cast<i64>(b + q * G) * kStreamRows + warp * 32;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const i64 r = row0 + x * 8 + g;
      if (r >= a.nrows) continue;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int col = y * 8 + 2 * t;
        if (col >= a.m2) continue;
        double v0 = a.alpha * acc[x][y][0], v1 = a.alpha * acc[x][y][1];
        if (a.beta != 0.0) {
          v0 += a.beta * a.Bm[r * a.ldb + col];
          if (col + 1 < a.m2) v1 += a.beta * a.Bm[r * a.ldb + col + 1];
        }
        if (col + 1 < a.m2) {
          *reinterpret_cast<double2*>(a.Out + r * a.ldo + col) = make_double2(v0, v1);
        } else {
          a.Out[r * a.ldo + col] = v0;
        }
      }
    }
  }
}

// Narrow streaming Gram (m1, m2 <= 32): persistent CTAs walk 64-row tiles
// of A (and B unless A == B) through a 4-deep TMA ring; the four warps take
// 16 rows of each tile, so each warp keeps one 32 x 32 accumulator for the
// whole CTA; the warps' sums are combined in fixed order into one partial per
// CTA, reduced by gram_reduce_kernel (one split per CTA).
constexpr int kGsRows = 64;  // rows per tile (16 per warp)
constexpr size_t gram_stream_smem(bool same) {
  return 128 + sizeof(double) * ((same ? 1 : 2) * static_cast<size_t>(kStreamStages) * kGsRows * kStreamPitch);
}

__global__ void __launch_bounds__(NT, 3)
    gram_stream_kernel(GramArgs a, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       int same, int ntiles) {
  extern __shared__ __align__(128) unsigned char gsm[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(gsm);
  unsigned long long* empty = full + kStreamStages;
  double* stage0 = reinterpret_cast<double*>(gsm + 128);
  constexpr int STG = kGsRows * kStreamPitch;  // per operand
  const int ops = same ? 1 : 2;
  const unsigned stage_bytes = static_cast<unsigned>(sizeof(double) * STG * ops);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStreamStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kEmptyCount);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int G = gridDim.x, b = blockIdx.x;
  const int my = b < ntiles ? (ntiles - 1 - b) / G + 1 : 0;
  auto produce = [&](int q) {
    const int st = q % kStreamStages;
    if (q >= kStreamStages) mbar_wait(&empty[st], static_cast<unsigned>((q / kStreamStages - 1) & 1));
    double* sa = stage0 + st * ops * STG;
    mbar_arrive_expect_tx(&full[st], stage_bytes);
    const int row0 = (b + q * G) * kGsRows;
    tma_load_2d(sa, &tmA, 0, row0, &full[st]);
    if (!same) tma_load_2d(sa + STG, &tmB, 0, row0, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < min(my, kStreamStages - 1); ++q) produce(q);
  const int nx = frags_left(a.m1, 0), ny = frags_left(a.m2, 0);
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  for (int q = 0; q < my; ++q) {
    if (threadIdx.x == 0 && q + kStreamStages - 1 < my) produce(q + kStreamStages - 1);
    const int st = q % kStreamStages;
    mbar_wait(&full[st], static_cast<unsigned>((q / kStreamStages) & 1));
    const double* sa = stage0 + st * ops * STG + warp * 16 * kStreamPitch;  // this warp's 16 rows
    const double* sb = same ? sa : sa + STG;
    const double* pa = sa + t * kStreamPitch + g;
    const double* pb = sb + t * kStreamPitch + g;
    // optional row mask: rows with mask[r] == mask_val contribute nothing (their A fragments read as 0)
    unsigned mk = 0;
    if (a.mask) {
      const i64 rb = static_cast<i64>(b + q * G) * kGsRows + warp * 16 + t;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (rb + 4 * u < a.nrows && a.mask[rb + 4 * u] == a.mask_val) mk |= 1u << u;
    }
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      double fa[4], fb[4];
      const bool z = (mk >> (kk >> 2)) & 1u;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        fa[x] = z ? 0.0 : pa[kk * kStreamPitch + x * 8];
        fb[x] = pb[kk * kStreamPitch + x * 8];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
          if (x < nx && y < ny && (!a.sym || x <= y)) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
    }
    release_stage(&empty[st]);  // the warp's smem reads ordered before the TMA refill
  }
  // combine the four warps (fixed order) through the (drained) stage buffers
  __syncthreads();
  double* red = stage0;  // 4 x 32 x 32 (fits: >= 4 stages x 64 x 36 doubles)
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = x * 8 + g, j = y * 8 + 2 * t;
      red[warp * 1024 + i * 32 + j] = acc[x][y][0];
      red[warp * 1024 + i * 32 + j + 1] = acc[x][y][1];
    }
  __syncthreads();
  double* out = a.partial + static_cast<i64>(b) * 1024;
  for (int e = threadIdx.x; e < 1024; e += NT) out[e] = ((red[e] + red[1024 + e]) + red[2048 + e]) + red[3072 + e];
}

__global__ void __launch_bounds__(NT) gemm_nn_small_kernel(NNArgs a) {
  if (nn_skipped(a)) return;
  __shared__ __align__(16) double sA[2][NBM][NSAR];
  __shared__ __align__(16) double sC[2][NBK][SS];
  const i64 row0 = static_cast<i64>(blockIdx.x) * NBM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int kmax = a.m1;
  const int nk = static_cast<int>(cdiv(kmax, NBK));
  bool vi[4], vj[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    vi[x] = row0 + warp * 32 + x * 8 < a.nrows;
    vj[x] = x * 8 < a.m2;
  }
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  auto load = [&](int s, int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // A: 128 rows x 8 cols = 512 pairs
      const int c = threadIdx.x + NT * q;
      const int row = c >> 2, col = (c & 3) * 2;
      const i64 gr = row0 + row;
      const int gk = k0 + col;
      double* dst = &sA[s][row][col];
      if (gr < a.nrows && gk + 2 <= a.m1) {
        cp_async_pair(dst, a.A + gr * a.lda + gk);
      } else {
        dst[0] = (gr < a.nrows && gk < a.m1) ? a.A[gr * a.lda + gk] : 0.0;
        dst[1] = 0.0;
      }
    }
    {  // C: 8 rows x 32 cols = 128 pairs
      const int c = threadIdx.x;
      const int row = c >> 4, col = (c & 15) * 2;
      const int gk = k0 + row;
      double* dst = &sC[s][row][col];
      if (gk < a.m1 && col + 2 <= a.m2) {
        cp_async_pair(dst, a.C + static_cast<i64>(gk) * a.ldc + col);
      } else {
        dst[0] = (gk < a.m1 && col < a.m2) ? a.C[static_cast<i64>(gk) * a.ldc + col] : 0.0;
        dst[1] = 0.0;
      }
    }
  };
  if (nk > 0) {
    load(0, 0);
    cp_async_commit();
  }
  for (int c = 0; c < nk; ++c) {
    const int s = c & 1;
    if (c + 1 < nk) {
      load(s ^ 1, (c + 1) * NBK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < NBK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        fa[x] = sA[s][warp * 32 + x * 8 + g][kk + t];
        fb[x] = sC[s][kk + t][x * 8 + g];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
          if (vi[x] && vj[y]) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const i64 r = row0 + warp * 32 + x * 8 + g;
      const int col = y * 8 + 2 * t;
      if (r >= a.nrows) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (col + h >= a.m2) continue;
        double v = a.alpha * acc[x][y][h];
        if (a.beta != 0.0) v += a.beta * a.Bm[r * a.ldb + col + h];
        a.Out[r * a.ldo + col + h] = v;
      }
    }
}

}  // namespace dm
}  // namespace stg
