// CSR x tall-skinny dense products for the perturbation Delta (HBM-bound).
//
// One warp per CSR row segment; lane l owns columns l, l+32, ... of the dense
// block, so each nonzero costs one coalesced read of a dense row. The (col, val) pairs of
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

// Rows are cut into segments of at most kSegNnz nonzeros, one warp per
// segment, so a hub row (hundreds of Delta entries) no longer serialises one
// warp behind a chain of dependent gathers. A row of one segment is summed as
// above and written directly; the segments of a longer row write partial
// sums, which spmm_fixup_kernel adds in segment order (deterministic; the
// association differs from Eigen's only within those rows, at rounding level).
constexpr int kSegNnz = 32;

struct SpmmPlan {
  const int* vrow;        // virtual row (segment) -> row
  const int* vstart;      // row -> first segment; vstart[rows] = segment count
  const int* sstart;      // row -> first scratch slot (rows of more than one segment)
  const int* split_rows;  // rows of more than one segment (any order)
  const int* nsplit;
  double* scratch;        // [slot][lds]
  int lds;
};

template <int T>  // columns per lane = T (m <= 32 T)
__global__ void __launch_bounds__(256) spmm_kernel(SpmmArgs a, SpmmPlan pl) {
  const i64 v = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= pl.vstart[a.rows]) return;
  const int r = pl.vrow[v];
  const int s = static_cast<int>(v - pl.vstart[r]);
  const int nseg = pl.vstart[r + 1] - pl.vstart[r];
  const i64 gr = r + a.row_off;
  const int rs = a.rowptr[gr] + s * kSegNnz;
  const int cnt = min(kSegNnz, a.rowptr[gr + 1] - rs);
  int c_l = 0;
  double v_l = 0.0;
  if (lane < cnt) {
    c_l = a.col[rs + lane];
    v_l = a.val[rs + lane];
  }
  // trailing-column view: the (sorted) columns below col_lo are a prefix
  int q = a.col_lo > 0 ? __popc(__ballot_sync(0xffffffffu, lane < cnt && c_l < a.col_lo)) : 0;
  double acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t] = 0.0;
  // four nonzeros per pass: their row loads are issued together, the sums
  // still run in column order
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
    const double vq = __shfl_sync(0xffffffffu, v_l, q);
    const double* xr = a.X + static_cast<i64>(c) * a.ldx;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int cc = lane + 32 * t;
      if (cc < a.m) acc[t] = __dadd_rn(acc[t], __dmul_rn(vq, __ldg(xr + cc)));
    }
  }
  double* yr = nseg == 1 ? a.Y + static_cast<i64>(r) * a.ldy
                         : pl.scratch + static_cast<i64>(pl.sstart[r] + s) * pl.lds;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int cc = lane + 32 * t;
    if (cc < a.m) yr[cc] = acc[t];
  }
}

// Rows of several segments: partial sums added in segment order.
__global__ void __launch_bounds__(256) spmm_fixup_kernel(SpmmArgs a, SpmmPlan pl) {
  const int i = static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= *pl.nsplit) return;
  const int r = pl.split_rows[i];
  const int nseg = pl.vstart[r + 1] - pl.vstart[r];
  const double* p0 = pl.scratch + static_cast<i64>(pl.sstart[r]) * pl.lds;
  for (int cc = lane; cc < a.m; cc += 32) {
    double y = 0.0;
    for (int s = 0; s < nseg; ++s) y = __dadd_rn(y, p0[static_cast<i64>(s) * pl.lds + cc]);
    a.Y[static_cast<i64>(r) * a.ldy + cc] = y;
  }
}

// ---- segment plan of a CSR row range (built once per perturbation)
__global__ void seg_count_kernel(const int* rowptr, i64 row_off, i64 rows, int* cnt, int* cnt2) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > rows) return;
  if (r == rows) {
    cnt[r] = cnt2[r] = 0;
    return;
  }
  const int len = rowptr[r + row_off + 1] - rowptr[r + row_off];
  const int c = len > kSegNnz ? (len + kSegNnz - 1) / kSegNnz : 1;
  cnt[r] = c;
  cnt2[r] = c > 1 ? c : 0;
}

__global__ void seg_fill_kernel(const int* vstart, i64 rows, int* vrow, int* split_rows, int* nsplit) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int b = vstart[r], c = vstart[r + 1] - b;
  for (int s = 0; s < c; ++s) vrow[b + s] = static_cast<int>(r);
  if (c > 1) split_rows[atomicAdd(nsplit, 1)] = static_cast<int>(r);
}

inline void spmm_launch(const SpmmArgs& a, const SpmmPlan& pl, i64 vmax, i64 split_max, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(cdiv(vmax, 8));
  const int T = static_cast<int>(cdiv(a.m < 1 ? 1 : a.m, 32));
  switch (T) {
    case 1: spmm_kernel<1><<<grid, 256, 0, st>>>(a, pl); break;
    case 2: spmm_kernel<2><<<grid, 256, 0, st>>>(a, pl); break;
    case 3: spmm_kernel<3><<<grid, 256, 0, st>>>(a, pl); break;
    case 4: spmm_kernel<4><<<grid, 256, 0, st>>>(a, pl); break;
    case 5: spmm_kernel<5><<<grid, 256, 0, st>>>(a, pl); break;
    case 6: spmm_kernel<6><<<grid, 256, 0, st>>>(a, pl); break;
    case 7: spmm_kernel<7><<<grid, 256, 0, st>>>(a, pl); break;
    case 8: spmm_kernel<8><<<grid, 256, 0, st>>>(a, pl); break;
    default: throw std::invalid_argument("spmm: more than 256 dense columns");
  }
  STG_LAUNCH();
  if (split_max > 0) {
    spmm_fixup_kernel<<<static_cast<unsigned>(cdiv(split_max, 8)), 256, 0, st>>>(a, pl);
    STG_LAUNCH();
  }
}

}  // namespace stg
