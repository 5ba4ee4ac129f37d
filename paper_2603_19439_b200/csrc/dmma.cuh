// FP64 tensor-core (DMMA) kernels for the tall-skinny algebra of the G-REST
// step. sm_100a has no tcgen05 kind::f64, so FP64 tensor work is mma.sync
// m8n8k4 (SASS DMMA.8x8x4); operand tiles are staged through shared memory with
// a cp.async double buffer.
//
//   gram_tn : Out(m1 x m2) = A(N x m1)' B(N x m2), split-K over the N rows with
//             a deterministic second-pass reduction (fixed split order). With
//             `sym` (A == B) only tile pairs ti <= tj are computed and the
//             result is mirrored exactly.
//   gemm_nn : Out(N x m2) = alpha A(N x m1) C(m1 x m2) + beta B(N x m2), the
//             row-local update (projections, R^-1 application, rotations).
//             B may alias Out (each CTA reads its own tile before writing).
// All blocks are row-major with even leading dimensions.
#pragma once

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

__global__ void __launch_bounds__(NT) gram_tn_kernel(GramArgs a) {
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
  __shared__ __align__(16) double sA[2][BK][SST];
  __shared__ __align__(16) double sB[2][BK][SST];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int ibase = ti * BM + wm * 32, jbase = tj * BN + wn * 32;
  bool vi[4], vj[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    vi[x] = ibase + x * 8 < a.m1;
    vj[x] = jbase + x * 8 < a.m2;
  }
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

  const i64 nchunks = r1 > r0 ? cdiv(r1 - r0, BK) : 0;
  if (nchunks > 0) {
    load_k_tile(sA[0], a.A, a.lda, r0, r1, ti * BM, a.m1, a.mask, a.mask_val);
    load_k_tile(sB[0], a.B, a.ldb, r0, r1, tj * BN, a.m2, a.mask, a.mask_val);
    cp_async_commit();
  }
  for (i64 c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    if (c + 1 < nchunks) {
      load_k_tile(sA[s ^ 1], a.A, a.lda, r0 + (c + 1) * BK, r1, ti * BM, a.m1, a.mask, a.mask_val);
      load_k_tile(sB[s ^ 1], a.B, a.ldb, r0 + (c + 1) * BK, r1, tj * BN, a.m2, a.mask, a.mask_val);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        fa[x] = sA[s][kk + t][wm * 32 + x * 8 + g];
        fb[x] = sB[s][kk + t][wn * 32 + x * 8 + g];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
          if (vi[x] && vj[y]) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
    }
    __syncthreads();
  }
  const i64 m1p = static_cast<i64>(a.tiles_i) * BM, m2p = static_cast<i64>(a.tiles_j) * BN;
  double* out = a.partial + static_cast<i64>(blockIdx.y) * m1p * m2p;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const i64 i = ibase + x * 8 + g, j = jbase + y * 8 + 2 * t;
      *reinterpret_cast<double2*>(out + i * m2p + j) = make_double2(acc[x][y][0], acc[x][y][1]);
    }
}

// Deterministic split reduction; for sym the (min, max) element is read so the
// result is exactly symmetric.
__global__ void gram_reduce_kernel(const double* partial, int splits, int m1, int m2, int m1p, int m2p, int sym,
                                   double* out, int ldo, double alpha) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(m1) * m2) return;
  const int i = static_cast<int>(idx / m2), j = static_cast<int>(idx % m2);
  int ii = i, jj = j;
  if (sym && (i / BM) > (j / BN)) {
    ii = j;
    jj = i;
  } else if (sym && i > j && (i / BM) == (j / BN)) {
    ii = j;
    jj = i;
  }
  const i64 stride = static_cast<i64>(m1p) * m2p;
  double s = 0.0;
  for (int sp = 0; sp < splits; ++sp) s += partial[sp * stride + static_cast<i64>(ii) * m2p + jj];
  out[static_cast<i64>(i) * ldo + j] = alpha * s;
}

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
};

__global__ void __launch_bounds__(NT) gemm_nn_kernel(NNArgs a) {
  __shared__ __align__(16) double sA[2][BM][SAR];
  __shared__ __align__(16) double sC[2][BK][SST];
  const i64 row0 = static_cast<i64>(blockIdx.x) * BM;
  const int tj = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int kmax = a.upper_tri_c ? min(a.m1, (tj + 1) * BN) : a.m1;
  const int nk = static_cast<int>(cdiv(kmax, BK));
  bool vi[4], vj[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    vi[x] = row0 + wm * 32 + x * 8 < a.nrows;
    vj[x] = tj * BN + wn * 32 + x * 8 < a.m2;
  }
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

  auto load = [&](int s, int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // A: 64 rows x 16 cols
      const int c = threadIdx.x + NT * q;
      const int row = c >> 3, col = (c & 7) * 2;
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
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // C: 16 rows x 64 cols
      const int c = threadIdx.x + NT * q;
      const int row = c >> 5, col = (c & 31) * 2;
      const int gk = k0 + row, gc = tj * BN + col;
      double* dst = &sC[s][row][col];
      if (gk < a.m1 && gc + 2 <= a.m2) {
        cp_async_pair(dst, a.C + static_cast<i64>(gk) * a.ldc + gc);
      } else {
        dst[0] = (gk < a.m1 && gc < a.m2) ? a.C[static_cast<i64>(gk) * a.ldc + gc] : 0.0;
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
      load(s ^ 1, (c + 1) * BK);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        fa[x] = sA[s][wm * 32 + x * 8 + g][kk + t];
        fb[x] = sC[s][kk + t][wn * 32 + x * 8 + g];
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
      const i64 r = row0 + wm * 32 + x * 8 + g;
      const int col = tj * BN + wn * 32 + y * 8 + 2 * t;
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
