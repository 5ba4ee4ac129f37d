// On-device tracking-quality metrics (proj/src/metrics.cpp:17-27, 243-259):
// the per-vector principal angle psi_i between x_i and a reference y_i, and
// the largest principal angle between span(X) and span(Y), computed where X
// lives (no n x k copy to the host at R-MAT s25 sizes). Column statistics are
// fixed-order per-CTA partials reduced by lz_colsum_kernel (deterministic).
#pragma once

#include "common.cuh"

namespace stg {

constexpr int kMetThreads = 256;

// pass 1: partial[cta][3c + {0,1,2}] = sum x_c^2, sum y_c^2, sum x_c y_c
__global__ void __launch_bounds__(kMetThreads) angle_stats_kernel(const double* X, int ldx, const double* Y, int ldy,
                                                                  i64 n, int k, double* partial, int ldp) {
  extern __shared__ double red[];  // [warps][3k]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const i64 gw = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + lane;
    double sx = 0.0, sy = 0.0, sxy = 0.0;
    if (c < k)
      for (i64 r = gw; r < n; r += nw) {
        const double x = X[r * ldx + c], y = Y[r * ldy + c];
        sx = fma(x, x, sx);
        sy = fma(y, y, sy);
        sxy = fma(x, y, sxy);
      }
    if (c < k) {
      red[w * 3 * k + 3 * c] = sx;
      red[w * 3 * k + 3 * c + 1] = sy;
      red[w * 3 * k + 3 * c + 2] = sxy;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 3 * k; t += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nwb; ++q) s += red[q * 3 * k + t];
    partial[static_cast<i64>(blockIdx.x) * ldp + t] = s;
  }
}

// pass 2 (principal_angle, metrics.cpp:17-27): u = x / ||x||, v = sign(u'y) y / ||y||;
// partial[cta][2c + {0,1}] = sum (u - v)^2, sum (u + v)^2
__global__ void __launch_bounds__(kMetThreads) angle_diff_kernel(const double* X, int ldx, const double* Y, int ldy,
                                                                 i64 n, int k, const double* stats, double* partial,
                                                                 int ldp) {
  extern __shared__ double red[];  // [warps][2k]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const i64 gw = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + lane;
    double dm = 0.0, dp = 0.0;
    if (c < k) {
      const double nx = sqrt(stats[3 * c]), ny = sqrt(stats[3 * c + 1]);
      const double sg = stats[3 * c + 2] < 0.0 ? -1.0 : 1.0;  // u'y < 0 flips v (sign of x'y)
      for (i64 r = gw; r < n; r += nw) {
        const double u = X[r * ldx + c] / nx, v = sg * (Y[r * ldy + c] / ny);
        dm = fma(u - v, u - v, dm);
        dp = fma(u + v, u + v, dp);
      }
      red[w * 2 * k + 2 * c] = dm;
      red[w * 2 * k + 2 * c + 1] = dp;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 2 * k; t += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nwb; ++q) s += red[q * 2 * k + t];
    partial[static_cast<i64>(blockIdx.x) * ldp + t] = s;
  }
}

// transpose of a small row-major block
__global__ void small_transpose_kernel(const double* A, int lda, int m, int n, double* B, int ldb) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m * n) B[(t % n) * ldb + t / n] = A[(t / n) * lda + t % n];
}

}  // namespace stg
