// CSR x tall-skinny dense products for the perturbation Delta (HBM-bound).
//
// One warp per CSR row; lane l owns columns l, l+32, ... of the dense block, so
// each nonzero costs one coalesced read of a dense row. The (col, val) pairs of
// a row are fetched 32 at a time and broadcast with shuffles. Accumulation is
// sequential over the row's nonzeros in column order with separate multiply
// and add roundings, which reproduces Eigen's row-major sparse*dense product
// (proj/src/sparse.cpp:84-87) bit for bit.
#pragma once

#include "common.cuh"

namespace stg {

struct SpmmArgs {
  i64 rows;             // output rows
  i64 row_off;          // CSR row of output row 0
  const int* rowptr;    // local CSR (indices into col/val)
  const int* col;       // local column indices (rows of X)
  const double* val;
  int col_lo;           // only nonzeros with col >= col_lo (trailing-column view); 0 = all
  const double* X;
  int ldx;
  int m;                // dense columns
  double* Y;
  int ldy;
};

template <int T>  // columns per lane = T (m <= 32 T)
__global__ void __launch_bounds__(256) spmm_kernel(SpmmArgs a) {
  const i64 r = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= a.rows) return;
  const i64 gr = r + a.row_off;
  int s = a.rowptr[gr];
  const int e = a.rowptr[gr + 1];
  if (a.col_lo > 0) {  // first nonzero with col >= col_lo (columns are sorted)
    int lo = s, hi = e;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (a.col[mid] < a.col_lo) lo = mid + 1; else hi = mid;
    }
    s = lo;
  }
  double acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t] = 0.0;
  for (int base = s; base < e; base += 32) {
    const int cnt = min(32, e - base);
    int c_l = 0;
    double v_l = 0.0;
    if (lane < cnt) {
      c_l = a.col[base + lane];
      v_l = a.val[base + lane];
    }
    // four nonzeros per pass: their row loads are issued together (memory
    // parallelism for long rows), the sums still run in column order
    int q = 0;
    for (; q + 4 <= cnt; q += 4) {
      double xv[4][T], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = __shfl_sync(0xffffffffu, c_l, q + u);
        vv[u] = __shfl_sync(0xffffffffu, v_l, q + u);
        const double* xr = a.X + static_cast<i64>(c) * a.ldx;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int cc = lane + 32 * t;
          xv[u][t] = cc < a.m ? __ldg(xr + cc) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int t = 0; t < T; ++t) acc[t] = __dadd_rn(acc[t], __dmul_rn(vv[u], xv[u][t]));
    }
    for (; q < cnt; ++q) {
      const int c = __shfl_sync(0xffffffffu, c_l, q);
      const double v = __shfl_sync(0xffffffffu, v_l, q);
      const double* xr = a.X + static_cast<i64>(c) * a.ldx;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int cc = lane + 32 * t;
        if (cc < a.m) acc[t] = __dadd_rn(acc[t], __dmul_rn(v, __ldg(xr + cc)));
      }
    }
  }
  double* yr = a.Y + r * a.ldy;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int cc = lane + 32 * t;
    if (cc < a.m) yr[cc] = acc[t];
  }
}

inline void spmm_chunk(const SpmmArgs& a, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(cdiv(a.rows, 8));
  const int T = static_cast<int>(cdiv(a.m < 1 ? 1 : a.m, 32));
  switch (T) {
    case 1: spmm_kernel<1><<<grid, 256, 0, st>>>(a); break;
    case 2: spmm_kernel<2><<<grid, 256, 0, st>>>(a); break;
    case 3: spmm_kernel<3><<<grid, 256, 0, st>>>(a); break;
    case 4: spmm_kernel<4><<<grid, 256, 0, st>>>(a); break;
    case 5: spmm_kernel<5><<<grid, 256, 0, st>>>(a); break;
    case 6: spmm_kernel<6><<<grid, 256, 0, st>>>(a); break;
    case 7: spmm_kernel<7><<<grid, 256, 0, st>>>(a); break;
    case 8: spmm_kernel<8><<<grid, 256, 0, st>>>(a); break;
    default: throw std::invalid_argument("spmm: more than 256 dense columns");
  }
  STG_LAUNCH();
}

// Dense blocks wider than 256 columns are processed in 256-column slabs.
inline void spmm(const SpmmArgs& a, cudaStream_t st) {
  if (a.rows <= 0 || a.m <= 0) return;
  for (int c0 = 0; c0 < a.m; c0 += 256) {
    SpmmArgs b = a;
    b.X = a.X + c0;
    b.Y = a.Y + c0;
    b.m = a.m - c0 < 256 ? a.m - c0 : 256;
    spmm_chunk(b, st);
  }
}

}  // namespace stg
