// Glue kernels of the compressed G-REST step (row gathers/scatters between the
// n-row state and the stacked |P| + 2k coordinates).
#pragma once

#include "common.cuh"
#include "smalllin.cuh"

namespace stg {

// Stacked X-bar: rows [0, p) = X rows of P (appended rows 0), rows [p, p+k) =
// R_c (K = R_c' R_c), rows [p+k, p+2k) = I_k.
__global__ void gather_xbar_kernel(const double* X, int ldx, const int* P, int dense, i64 p, i64 p_old, int k,
                                   const double* rc, int ldrc, double* z, int ldz) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= (p + 2 * k) * k) return;
  const i64 t = idx / k;
  const int c = static_cast<int>(idx % k);
  double v;
  if (t < p) {
    if (t < p_old) v = X[(dense ? t : static_cast<i64>(P[t])) * ldx + c];
    else v = 0.0;
  } else if (t < p + k) {
    if (!rc) return;  // written later (K from the zeroed-row Gram)
    v = rc[(t - p) * ldrc + c];
  } else {
    v = (t - p - k == c) ? 1.0 : 0.0;
  }
  z[t * ldz + c] = v;
}

// X rows of P (old nodes) zeroed in place / restored from the stacked copy.
__global__ void __launch_bounds__(256) zero_rows_kernel(double* X, int ldx, const int* P, i64 p_old, int k) {
  const i64 t = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= p_old) return;
  double* xr = X + static_cast<i64>(P[t]) * ldx;
  for (int c = lane; c < k; c += 32) xr[c] = 0.0;
}

__global__ void __launch_bounds__(256) restore_rows_kernel(double* X, int ldx, const int* P, i64 p_old,
                                                           const double* z, int ldz, int k) {
  const i64 t = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= p_old) return;
  double* xr = X + static_cast<i64>(P[t]) * ldx;
  for (int c = lane; c < k; c += 32) xr[c] = z[t * ldz + c];
}

// iasc: unit vectors of the appended nodes (z points at column k).
__global__ void unit_cols_kernel(double* z, int ldz, i64 p_old, i64 S) {
  const i64 j = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < S) z[(p_old + j) * ldz + j] = 1.0;
}

// grest3 trailing block: column j of d2 = row p_old + j of the (symmetric) local CSR.
__global__ void d2_dense_kernel(const int* lrp, const int* lcol, const double* val, i64 p_old, i64 S, double* out,
                                int ldo) {
  const i64 j = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= S) return;
  const i64 r = p_old + j;
  for (int e = lrp[r] + lane; e < lrp[r + 1]; e += 32) out[static_cast<i64>(lcol[e]) * ldo + j] = val[e];
}

// Leading `keep` eigenvectors in descending eigenvalue order (cuSOLVER returns ascending).
__global__ void gather_desc_kernel(const double* V, int q, int keep, double* U, int ldu) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(q) * keep) return;
  const int i = static_cast<int>(idx / keep), c = static_cast<int>(idx % keep);
  U[static_cast<i64>(i) * ldu + c] = V[static_cast<i64>(q - 1 - c) * q + i];
}

// Ritz rotation into the state: rows of P take W's rows, every other row is
// X_i A_new (A_new = the a-coordinates of Z F). Skipped entirely when the step
// raised an error flag, so a failed step leaves X untouched.
__global__ void __launch_bounds__(256) rotate_x_kernel(double* X, int ldx, i64 n_old, i64 n_total, int dense,
                                                       const int* mark, int stamp, const int* posmap, const double* W,
                                                       int ldw, const double* Anew, int k, const int* flags,
                                                       const int* info) {
  if ((*flags & (kNonFinite | kNotOrthonormal | kSpecFail)) || *info != 0) return;
  const i64 i = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_total) return;
  double* xr = X + i * ldx;
  if (dense || i >= n_old || mark[i] == stamp) {
    const double* wr = W + (dense ? i : static_cast<i64>(posmap[i])) * ldw;
    for (int c = lane; c < k; c += 32) xr[c] = wr[c];
    return;
  }
  const double x0 = lane < k ? xr[lane] : 0.0;
  const double x1 = lane + 32 < k ? xr[lane + 32] : 0.0;
  double a0 = 0.0, a1 = 0.0;
  for (int l = 0; l < k; ++l) {
    const double xl = __shfl_sync(0xffffffffu, l < 32 ? x0 : x1, l & 31);
    if (lane < k) a0 += xl * Anew[static_cast<i64>(l) * ldw + lane];
    if (lane + 32 < k) a1 += xl * Anew[static_cast<i64>(l) * ldw + lane + 32];
  }
  if (lane < k) xr[lane] = a0;
  if (lane + 32 < k) xr[lane + 32] = a1;
}

// Rows of P take the rotated stacked rows W[t] (row P[t], or t in dense mode).
__global__ void __launch_bounds__(256) scatter_rows_kernel(double* X, int ldx, const int* P, int dense, i64 p,
                                                           const double* W, int ldw, int k, const int* flags,
                                                           const int* info) {
  if ((*flags & (kNonFinite | kNotOrthonormal | kSpecFail)) || *info != 0) return;
  const i64 t = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= p) return;
  const i64 row = dense ? t : static_cast<i64>(P[t]);
  for (int c = lane; c < k; c += 32) X[row * ldx + c] = W[t * ldw + c];
}

// Dense expansion of a stacked basis (probe API only).
__global__ void __launch_bounds__(256) expand_kernel(const double* X, int ldx, i64 n_old, i64 n_total, int dense,
                                                     const int* mark, int stamp, const int* posmap, const double* z,
                                                     int ldz, const double* arows, int k, int D, double* out,
                                                     int ldo) {
  const i64 i = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_total) return;
  if (dense || i >= n_old || mark[i] == stamp) {
    const double* zr = z + (dense ? i : static_cast<i64>(posmap[i])) * ldz;
    for (int c = lane; c < D; c += 32) out[i * ldo + c] = zr[c];
    return;
  }
  for (int c = lane; c < D; c += 32) {
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += X[i * ldx + l] * arows[static_cast<i64>(l) * ldz + c];
    out[i * ldo + c] = s;
  }
}

}  // namespace stg
