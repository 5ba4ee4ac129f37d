// Device kernels of tracker_init: thick-restart Lanczos with full
// reorthogonalization (proj/include/spectrack/lanczos.hpp:38-127, called from
// proj/src/trackers.cpp:67-75,132-145), plus the full-operator CSR SpMV it
// runs once per basis vector (matvec, proj/src/sparse.cpp:79-82).
//
// Layout. The basis V and the products W = A V are row-major n x ld blocks
// (ld = ld_for(max_basis)): a basis row is one contiguous 8-byte-aligned run,
// so the reorthogonalization reads whole rows coalesced (one warp per row,
// lanes across the basis columns), and the Rayleigh-Ritz products (H = V'W,
// restart compressions V F) run on the DMMA Gram / NN kernels of dmma.cuh.
//
// Reorthogonalization (lanczos.hpp:59-60): two classical Gram-Schmidt passes
// v -= V (V'v). The passes are fused across kernel boundaries so V is read
// three times per new vector instead of four:
//   lz_dot      c1 = V'v                         (read V)
//   lz_upd_dot  v1 = v - V c1 ; c2 = V'v1        (read V once: row-local)
//   lz_upd_norm v2 = v1 - V c2 ; ||v2||^2        (read V)
// Every reduction is a fixed-order per-CTA partial followed by a fixed-shape
// tree (deterministic: the same inputs give the same bits on every run).
//
// SpMV (power-law rows: R-MAT degrees span 0..10^6). Rows are classified once
// per operator: short rows (<= kSpvShort entries) take 8 lanes each (4 rows
// per warp), medium rows a warp each, long rows are cut into kSpvSeg-entry
// segments (a warp each) whose partials are summed in segment order by a
// fix-up pass. Sums run in a fixed order; the y row is written to the Lanczos
// vector and to column j of W in the same pass.
#pragma once

#include "common.cuh"
#include "smalllin.cuh"  // warp_sum

namespace stg {

constexpr int kLzMaxCols = 256;  // device Lanczos basis width limit (max_basis)
constexpr int kLzThreads = 256;
constexpr int kSpvShort = 64;    // <= : 8 lanes per row
constexpr int kSpvSeg = 4096;    // > : rows cut into segments of this many entries

// ---------------------------------------------------------------- SpMV plan
// cls: 0 short, 1 medium, 2 long. cnt[r] = 1 in the row's class list,
// segs[r] = segments of a long row.
__global__ void spv_classify_kernel(const int* rp, i64 rows, int* f_short, int* f_med, int* f_long, int* segs) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > rows) return;
  if (r == rows) {  // scan sentinels
    f_short[r] = f_med[r] = f_long[r] = segs[r] = 0;
    return;
  }
  const int len = rp[r + 1] - rp[r];
  const int c = len <= kSpvShort ? 0 : len <= kSpvSeg ? 1 : 2;
  f_short[r] = c == 0;
  f_med[r] = c == 1;
  f_long[r] = c == 2;
  segs[r] = c == 2 ? (len + kSpvSeg - 1) / kSpvSeg : 0;
}

__global__ void spv_scatter_kernel(const int* f_short, const int* p_short, const int* f_med, const int* p_med,
                                   const int* f_long, const int* p_long, const int* segs, const int* p_seg, i64 rows,
                                   int* l_short, int* l_med, int* l_long, int* seg_row, int* seg_idx) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  if (f_short[r]) l_short[p_short[r]] = static_cast<int>(r);
  if (f_med[r]) l_med[p_med[r]] = static_cast<int>(r);
  if (f_long[r]) {
    l_long[p_long[r]] = static_cast<int>(r);
    for (int s = 0; s < segs[r]; ++s) {
      seg_row[p_seg[r] + s] = static_cast<int>(r);
      seg_idx[p_seg[r] + s] = s;
    }
  }
}

struct SpvPlan {
  const int* l_short = nullptr;
  const int* l_med = nullptr;
  const int* l_long = nullptr;
  const int* seg_row = nullptr;
  const int* seg_idx = nullptr;
  const int* p_seg = nullptr;  // row -> first segment slot
  int n_short = 0, n_med = 0, n_long = 0, n_seg = 0;
  double* seg_part = nullptr;  // [n_seg]
};

// y[r] = sum_e val[e] x[col[e]] in entry order within each lane, lanes
// combined by a fixed butterfly. out2 (optional): y also written at
// out2[r * ld2] (column j of W); flags |= 1 on a non-finite y.
__device__ __forceinline__ void spv_store(double y, i64 r, double* out, double* out2, int ld2, int* flags) {
  out[r] = y;
  if (out2) out2[r * ld2] = y;
  if (!isfinite(y)) atomicOr(flags, 1);
}

__global__ void __launch_bounds__(256) spv_short_kernel(const int* rp, const int* col, const double* val,
                                                        const double* x, const int* list, int cnt, double* out,
                                                        double* out2, int ld2, int* flags) {
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;  // 8-lane group
  const int sub = threadIdx.x & 7;
  // every lane of the warp reaches the shuffles (full mask): lanes of one
  // group leave the entry loop at different trip counts, so no partial mask
  // (e.g. __activemask) is guaranteed to hold the whole group
  const bool valid = g < cnt;
  const int r = valid ? list[g] : 0;
  const int b = valid ? rp[r] : 0, e = valid ? rp[r + 1] : 0;
  double acc = 0.0;
  for (int q = b + sub; q < e; q += 8) acc = fma(val[q], x[col[q]], acc);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4, 8);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2, 8);
  acc += __shfl_xor_sync(0xffffffffu, acc, 1, 8);
  if (valid && sub == 0) spv_store(acc, r, out, out2, ld2, flags);
}

__global__ void __launch_bounds__(256) spv_med_kernel(const int* rp, const int* col, const double* val,
                                                      const double* x, const int* list, int cnt, double* out,
                                                      double* out2, int ld2, int* flags) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= cnt) return;
  const int r = list[w];
  const int b = rp[r], e = rp[r + 1];
  double acc = 0.0;
  for (int q = b + lane; q < e; q += 32) acc = fma(val[q], x[col[q]], acc);
  acc = warp_sum(acc);
  if (lane == 0) spv_store(acc, r, out, out2, ld2, flags);
}

__global__ void __launch_bounds__(256) spv_seg_kernel(const int* rp, const int* col, const double* val,
                                                      const double* x, const int* seg_row, const int* seg_idx,
                                                      int nseg, double* part) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nseg) return;
  const int r = seg_row[w];
  const int b = rp[r] + seg_idx[w] * kSpvSeg;
  const int e = min(rp[r + 1], b + kSpvSeg);
  double acc = 0.0;
  for (int q = b + lane; q < e; q += 32) acc = fma(val[q], x[col[q]], acc);
  acc = warp_sum(acc);
  if (lane == 0) part[w] = acc;
}

__global__ void spv_fix_kernel(const int* rp, const int* l_long, int n_long, const int* p_seg, const double* part,
                               double* out, double* out2, int ld2, int* flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_long) return;
  const int r = l_long[t];
  const int ns = (rp[r + 1] - rp[r] + kSpvSeg - 1) / kSpvSeg;
  double y = 0.0;
  for (int s = 0; s < ns; ++s) y += part[p_seg[r] + s];
  spv_store(y, r, out, out2, ld2, flags);
}

// ---------------------------------------------------------------- reorthogonalization
// Per-lane accumulators for columns lane + 32 a, a < NA (j <= 32 NA).
template <int NA>
__device__ __forceinline__ void lz_block_partial(double (&acc)[NA], int j, double* red, double* partial, int ldp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int kW = kLzThreads / 32;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    const int c = lane + 32 * a;
    if (c < j) red[w * kLzMaxCols + c] = acc[a];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < j; c += blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < kW; ++q) t += red[q * kLzMaxCols + c];
    partial[static_cast<i64>(blockIdx.x) * ldp + c] = t;
  }
}

// partial[cta][c] = sum_r V[r][c] v[r] over the CTA's rows (c < j)
template <int NA>
__global__ void __launch_bounds__(kLzThreads) lz_dot_kernel(const double* V, int ldv, int j, const double* v, i64 n,
                                                            double* partial, int ldp) {
  __shared__ double red[(kLzThreads / 32) * kLzMaxCols];
  const int lane = threadIdx.x & 31;
  const i64 gw = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  double acc[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = 0.0;
  for (i64 r = gw; r < n; r += nw) {
    const double vr = v[r];
    const double* row = V + r * ldv;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const int c = lane + 32 * a;
      if (c < j) acc[a] = fma(row[c], vr, acc[a]);
    }
  }
  lz_block_partial<NA>(acc, j, red, partial, ldp);
}

// partial[cta][c] = sum_r V[r][c]^2 over the CTA's rows (residual norms)
template <int NA>
__global__ void __launch_bounds__(kLzThreads) lz_colsq_kernel(const double* V, int ldv, int j, i64 n, double* partial,
                                                              int ldp) {
  __shared__ double red[(kLzThreads / 32) * kLzMaxCols];
  const int lane = threadIdx.x & 31;
  const i64 gw = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  double acc[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = 0.0;
  for (i64 r = gw; r < n; r += nw) {
    const double* row = V + r * ldv;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const int c = lane + 32 * a;
      if (c < j) acc[a] = fma(row[c], row[c], acc[a]);
    }
  }
  lz_block_partial<NA>(acc, j, red, partial, ldp);
}

// vo = vi - V coef (row-local); then either the next pass's partial V'vo
// (NORM = false) or the partial ||vo||^2 (NORM = true, partial[cta][0]).
template <int NA, bool NORM>
__global__ void __launch_bounds__(kLzThreads) lz_update_kernel(const double* V, int ldv, int j, const double* coef,
                                                               const double* vi, double* vo, i64 n, double* partial,
                                                               int ldp) {
  __shared__ double red[(kLzThreads / 32) * kLzMaxCols];
  __shared__ double cs[kLzMaxCols];
  for (int c = threadIdx.x; c < j; c += blockDim.x) cs[c] = coef[c];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const i64 gw = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  double acc[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = 0.0;
  double sq = 0.0;
  for (i64 r = gw; r < n; r += nw) {
    const double* row = V + r * ldv;
    double x[NA];
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const int c = lane + 32 * a;
      x[a] = c < j ? row[c] : 0.0;
      s = fma(x[a], c < j ? cs[c] : 0.0, s);
    }
    s = warp_sum(s);
    const double y = vi[r] - s;
    if (lane == 0) vo[r] = y;
    if (NORM) {
      sq = fma(y, y, sq);
    } else {
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a] = fma(x[a], y, acc[a]);
    }
  }
  if (NORM) {
    // lane 0 of every warp holds its rows' sum; fixed-order CTA sum
    if (lane == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < kLzThreads / 32; ++q) t += red[q];
      partial[static_cast<i64>(blockIdx.x) * ldp] = t;
    }
  } else {
    lz_block_partial<NA>(acc, j, red, partial, ldp);
  }
}

// out[c] = sum over g < G of partial[g][c]: one CTA per column, strided sums
// then a fixed tree.
__global__ void __launch_bounds__(256) lz_colsum_kernel(const double* partial, int G, int ldp, int j, double* out) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  if (c >= j) return;
  double t = 0.0;
  for (int g = threadIdx.x; g < G; g += 256) t += partial[static_cast<i64>(g) * ldp + c];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = red[0];
}

// v /= nrm (lanczos.hpp:66: elementwise division), stored as column j of V
__global__ void lz_store_kernel(double* v, i64 n, const double* nrm, double* V, int ldv, int j) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double x = v[r] / nrm[0];
  v[r] = x;
  V[r * ldv + j] = x;
}

__global__ void lz_sqrt_kernel(double* x) { x[0] = sqrt(x[0]); }

// res = W F - X diag(theta) (lanczos.hpp:84) with X = V F already formed:
// in place on R (= W F on entry), row-major n x k.
__global__ void lz_residual_kernel(double* R, int ldr, const double* X, int ldx, const double* theta, i64 n, int k) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * k) return;
  const i64 r = t / k;
  const int c = static_cast<int>(t % k);
  R[r * ldr + c] -= X[r * ldx + c] * theta[c];
}

// all values of a cuSOLVER solve in spectral order
__global__ void lz_sorted_vals_kernel(const double* w, const int* perm, int j, double* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < j) out[c] = w[perm[c]];
}

// Column of a row-major block into a contiguous vector (restart direction).
__global__ void lz_column_kernel(const double* R, int ldr, int c, i64 n, double* v) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n) v[r] = R[r * ldr + c];
}

// Draws [pos, pos + count) of the GaussianSampler stream (rng.hpp:43-55):
// draw o comes from pair o / 2 (uniforms 2p, 2p + 1), cos for even o, sin
// for odd o.
__global__ void gauss_range_kernel(const u64* raw, i64 pos, i64 count, double* out) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const i64 o = pos + i, p = o >> 1;
  const double u1 = 1.0 - static_cast<double>(raw[2 * p] >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(raw[2 * p + 1] >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  constexpr double two_pi = 6.283185307179586476925286766559;
  double sn, cs;
  sincos(two_pi * u2, &sn, &cs);
  out[i] = (o & 1) ? r * sn : r * cs;
}

}  // namespace stg
