// Small dense linear algebra kept on the device (matrices of order <= ~260):
// Cholesky with rank-suspect monitoring, upper-triangular inverse, the
// spectral ordering of proj/include/spectrack/types.hpp:26-40, and the glue
// elementwise kernels of the Rayleigh-Ritz step.
#pragma once

#include "common.cuh"

namespace stg {

enum StepFlagBits : int {
  kSuspect = 1,        // Cholesky pivot below tau^2 * ||orig column||^2 (possible rank drop)
  kBreakdown = 2,      // non-positive / non-finite Cholesky pivot
  kNonFinite = 4,      // non-finite entry in the projected matrix (sym_eig_dense check)
  kNotOrthonormal = 8, // |Z'Z - I|max > 1e-6 (trackers.cpp:293-295)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Upper Cholesky G = R'R of a symmetric w x w block (row-major), one CTA,
// the upper triangle in shared memory (rows packed: row i holds columns i..w-1).
// Right-looking with ONE barrier per column: after the barrier every thread
// reads the pivot U(j,j) (broadcast) and derives 1/r itself; row j of R is
// written to global scaled, while the trailing update uses the raw row j with
// the factor 1/d: U(i,c) -= U(j,i) U(j,c) / d. When orig2 is given, a pivot
// d_j <= tau2 * orig2[j] raises kSuspect: the column's residual is within
// sqrt(tau2) of its original norm, where the reference's per-column drop test
// (ortho.hpp:34-35) must be re-evaluated exactly. With psd != 0 a
// non-positive pivot zeroes the row (semidefinite factor) instead of failing.
constexpr int kCholMaxW = 238;

__global__ void __launch_bounds__(1024) chol_kernel(const double* G, int ldg, int w, double* R, int ldr,
                                                    const double* orig2, double tau2, int psd, int* flags) {
  extern __shared__ double sm[];
  int* rowoff = reinterpret_cast<int*>(sm + static_cast<i64>(w) * (w + 1) / 2);
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  for (int i = tid; i < w; i += nth) rowoff[i] = i * w - (i * (i - 1)) / 2 - i;  // + c for c >= i
  __syncthreads();
  for (i64 idx = tid; idx < static_cast<i64>(w) * w; idx += nth) {
    const int i = static_cast<int>(idx / w), c = static_cast<int>(idx % w);
    if (c >= i) sm[rowoff[i] + c] = G[static_cast<i64>(i) * ldg + c];
    else R[static_cast<i64>(i) * ldr + c] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    const double* uj = sm + rowoff[j];
    const double d = uj[j];
    const bool bad = !(d > 0.0) || !isfinite(d);
    if (tid == 0) {
      if (orig2 && !(d > tau2 * orig2[j])) atomicOr(flags, kSuspect);
      if (bad && !psd) atomicOr(flags, kBreakdown);
    }
    const double inv_r = bad ? 0.0 : 1.0 / sqrt(d);
    const double inv_d = bad ? 0.0 : 1.0 / d;
    for (int c = j + tid; c < w; c += nth) R[static_cast<i64>(j) * ldr + c] = c == j ? (bad ? 0.0 : sqrt(d)) : uj[c] * inv_r;
    // trailing update, warp per row i > j, lanes over columns c >= i
    for (int i = j + 1 + warp; i < w; i += nw) {
      const double f = uj[i] * inv_d;
      double* ui = sm + rowoff[i];
      for (int c = i + lane; c < w; c += 32) ui[c] -= f * uj[c];
    }
    __syncthreads();
  }
}

inline size_t chol_smem_bytes(int w) {
  return sizeof(double) * static_cast<size_t>(w) * (w + 1) / 2 + sizeof(int) * static_cast<size_t>(w);
}

// Inverse of an upper-triangular R (row-major): one warp per column j of R^-1,
// back substitution with the column held in registers (lane l owns entries
// l + 32 t). Entries below the diagonal are written as zeros.
constexpr int kTriMaxSlots = 10;  // w <= 320
__global__ void __launch_bounds__(128) triinv_kernel(const double* R, int ldr, int w, double* Ri, int ldi) {
  const int j = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= w) return;
  double x[kTriMaxSlots];
#pragma unroll
  for (int t = 0; t < kTriMaxSlots; ++t) x[t] = 0.0;
  const double rjj = R[static_cast<i64>(j) * ldr + j];
  const double xj = rjj != 0.0 ? 1.0 / rjj : 0.0;
#pragma unroll
  for (int t = 0; t < kTriMaxSlots; ++t)
    if (lane + 32 * t == j) x[t] = xj;
  double rrow[kTriMaxSlots];
  auto load_row = [&](int i) {
#pragma unroll
    for (int t = 0; t < kTriMaxSlots; ++t) {
      const int l = lane + 32 * t;
      rrow[t] = (i >= 0 && l > i && l <= j) ? R[static_cast<i64>(i) * ldr + l] : 0.0;
    }
  };
  load_row(j - 1);
  for (int i = j - 1; i >= 0; --i) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < kTriMaxSlots; ++t) s += rrow[t] * x[t];
    const double rii = R[static_cast<i64>(i) * ldr + i];
    load_row(i - 1);  // prefetch the next row while reducing
    s = warp_sum(s);
    const double xi = rii != 0.0 ? -s / rii : 0.0;
#pragma unroll
    for (int t = 0; t < kTriMaxSlots; ++t)
      if (lane + 32 * t == i) x[t] = xi;
  }
#pragma unroll
  for (int t = 0; t < kTriMaxSlots; ++t) {
    const int l = lane + 32 * t;
    if (l < w) Ri[static_cast<i64>(l) * ldi + j] = x[t];
  }
}

// spectral_sort (types.hpp:26-40): rank of element i = number of elements that
// precede it under (primary key, algebraic value desc, index asc).
__device__ __forceinline__ bool spectral_before(double va, int a, double vb, int b, int order) {
  if (order == 0) {
    const double aa = va < 0.0 ? -va : va;
    const double ab = vb < 0.0 ? -vb : vb;
    if (aa != ab) return aa > ab;
  }
  if (va != vb) return va > vb;
  return a < b;
}

__global__ void sort_perm_kernel(const double* w, int n, int order, int* perm) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rank = 0;
    const double vi = w[i];
    for (int j = 0; j < n; ++j)
      if (j != i && spectral_before(w[j], j, vi, i, order)) ++rank;
    perm[rank] = i;
  }
}

// Leading k Ritz pairs after sorting: F (D x k, row-major) from cuSOLVER's
// column-major eigenvectors, and the ranked values.
__global__ void gather_ritz_kernel(const double* V, int D, const double* w, const int* perm, int k, double* F,
                                   int ldf, double* vals) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < static_cast<i64>(D) * k) {
    const int i = static_cast<int>(idx / k), c = static_cast<int>(idx % k);
    F[static_cast<i64>(i) * ldf + c] = V[static_cast<i64>(perm[c]) * D + i];
  }
  if (idx < k) vals[idx] = w[perm[idx]];
}

// M <- (M + M')/2 into a column-major copy for cuSOLVER (eig.hpp:47) and flag
// non-finite entries (eig.hpp:45).
__global__ void symmetrize_kernel(const double* M, int ldm, int D, double* out, int* flags) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(D) * D) return;
  const int i = static_cast<int>(idx / D), j = static_cast<int>(idx % D);
  const double a = M[static_cast<i64>(i) * ldm + j], b = M[static_cast<i64>(j) * ldm + i];
  if (!isfinite(a)) atomicOr(flags, kNonFinite);
  out[static_cast<i64>(j) * D + i] = 0.5 * (a + b);
}

// max |G - I| > tol -> kNotOrthonormal
__global__ void orthocheck_kernel(const double* Gm, int ldg, int D, double tol, int* flags) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(D) * D) return;
  const int i = static_cast<int>(idx / D), j = static_cast<int>(idx % D);
  const double v = Gm[static_cast<i64>(i) * ldg + j] - (i == j ? 1.0 : 0.0);
  if (!(fabs(v) <= tol)) atomicOr(flags, kNotOrthonormal);
}

// M(D x D) = zx diag(lam) zx' + T   (Eq. 14, trackers.cpp:300-301)
__global__ void rr_matrix_kernel(const double* zx, int ldzx, const double* lam, int k, const double* T, int ldt,
                                 int D, double* M, int ldm) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(D) * D) return;
  const int i = static_cast<int>(idx / D), j = static_cast<int>(idx % D);
  double s = 0.0;
  for (int l = 0; l < k; ++l) s += zx[static_cast<i64>(i) * ldzx + l] * lam[l] * zx[static_cast<i64>(j) * ldzx + l];
  M[static_cast<i64>(i) * ldm + j] = s + T[static_cast<i64>(i) * ldt + j];
}

// orig2[c] = G1[c][c] + sum_l C[l][c]^2: squared norm of the column before the
// projection against an orthonormal `against` block (for the suspect test).
__global__ void orig2_kernel(const double* G1, int ldg, const double* Cm, int ldc, int a, int w, double* orig2) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= w) return;
  double s = G1[static_cast<i64>(c) * ldg + c];
  for (int l = 0; l < a; ++l) s += Cm[static_cast<i64>(l) * ldc + c] * Cm[static_cast<i64>(l) * ldc + c];
  orig2[c] = s;
}

__global__ void fill_kernel(double* p, i64 n, double v) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < n) p[idx] = v;
}

// Copy a rows x cols block (row-major) between leading dimensions.
__global__ void copy2d_kernel(const double* src, int lds, double* dst, int ldd, i64 rows, int cols) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const i64 r = idx / cols;
  const int c = static_cast<int>(idx % cols);
  dst[r * ldd + c] = src[r * lds + c];
}

}  // namespace stg
