// The first-order perturbation trackers on the device: TRIP-Basic, TRIP and
// residual modes (proj/src/trackers.cpp:147-224). They share the G-REST
// step's pieces: Delta X-bar on the rows of P (the SpMM), C = X-bar'(Delta
// X-bar) (a Gram over the stacked coordinates) and the final rotation. The new
// vectors are combinations of a basis Z = [X-bar] (TRIP, TRIP-Basic) or
// [X-bar | Delta X-bar] (residual modes) with a small coefficient block F
// (D x k): everything k x k runs here, one CTA (or one CTA per column for
// TRIP's k linear systems), and the n-row work is one NN product.
//
//   TRIP-Basic  F = I + B,  B_ij = C_ij / (lambda_j - lambda_i)  (gaps below
//               gap_clamp dropped, trackers.cpp:26-31, 54-65)
//   residual    F = [I + B - C diag(d); diag(d)],  d_j = 1 / (lambda_j - mu)
//   TRIP        F_j = e_j + b_j (or b_j with trip_replace_span), where
//               (diag(lambda_new_j - lambda) - C) b_j = C e_j, solved by
//               partial-pivot LU with the ridge fallback of solve.hpp:23-45
//
// then renormalize_and_sort (trackers.cpp:43-52): column norms from the
// basis Gram (||Z f|| = sqrt(f' Z'Z f), an exact isometry of the stacked
// coordinates) and the spectral order of lambda + diag(C).
#pragma once

#include "common.cuh"
#include "smalllin.cuh"

namespace stg {

constexpr int kTrkMaxK = 128;

__device__ __forceinline__ double gap_clamp_dev(const double* lam) { return 1e-12 * fmax(1.0, fabs(lam[0])); }

// F (D x k, row-major, ldf) of TRIP-Basic (kind 0) or residual modes (kind 2);
// lam_new = lambda + diag(C).
__global__ void pert_coeff_kernel(const double* C, int ldc, const double* lam, int k, int kind, double mu, double* F,
                                  int ldf, double* lam_new) {
  const double eps = gap_clamp_dev(lam);
  const int D = kind == 2 ? 2 * k : k;
  for (int t = threadIdx.x; t < D * k; t += blockDim.x) {
    const int i = t / k, j = t % k;
    double v;
    if (i < k) {
      double b = 0.0;
      if (i != j) {
        const double gap = lam[j] - lam[i];
        if (fabs(gap) >= eps) b = C[i * ldc + j] / gap;
      }
      v = (i == j ? 1.0 : 0.0) + b;
      if (kind == 2) v -= C[i * ldc + j] / (lam[j] - mu);
    } else {
      v = (i - k == j) ? 1.0 / (lam[j] - mu) : 0.0;
    }
    F[i * ldf + j] = v;
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) lam_new[j] = lam[j] + C[j * ldc + j];
}

// TRIP: CTA j solves (diag(lambda_new_j - lambda) - C) b = C e_j (solve.hpp:
// partial-pivot LU; when the smallest pivot is below 1e-12 max|a|, the
// system + ridge * max(1, max|a|) I is solved instead and *ridge set).
__global__ void __launch_bounds__(128) trip_solve_kernel(const double* C, int ldc, const double* lam, int k,
                                                         int replace_span, double* F, int ldf, int* ridge) {
  extern __shared__ double tsm[];
  double* A = tsm;                 // k x k system, row-major
  double* LU = tsm + k * k;        // factorization workspace
  double* x = tsm + 2 * k * k;     // rhs / solution
  __shared__ int piv_row;
  __shared__ double red[128];
  __shared__ int redi[128];
  __shared__ int perm[kTrkMaxK];
  const int j = blockIdx.x, tid = threadIdx.x;
  const double lnew = lam[j] + C[j * ldc + j];
  double rmax = 0.0;
  for (int i = 0; i < k; ++i) rmax = fmax(rmax, fabs(C[i * ldc + j]));
  if (!(rmax > 0.0)) {  // zero right-hand side: b = 0 (trackers.cpp:178)
    for (int i = tid; i < k; i += blockDim.x) F[i * ldf + j] = (!replace_span && i == j) ? 1.0 : 0.0;
    return;
  }
  double amax_l = 0.0;
  for (int t = tid; t < k * k; t += blockDim.x) {
    const int i = t / k, q = t % k;
    const double a = -C[i * ldc + q] + (i == q ? lnew - lam[i] : 0.0);
    A[t] = a;
    amax_l = fmax(amax_l, fabs(a));
  }
  red[tid] = amax_l;
  __syncthreads();
  for (int h = 64; h > 0; h >>= 1) {
    if (tid < h) red[tid] = fmax(red[tid], red[tid + h]);
    __syncthreads();
  }
  const double amax = red[0];
  __syncthreads();
  // attempt 0: plain LU; attempt 1: ridge (only when the pivots say so)
  for (int attempt = 0; attempt < 2; ++attempt) {
    const double eps = attempt ? 1e-10 * fmax(1.0, amax) : 0.0;
    for (int t = tid; t < k * k; t += blockDim.x) LU[t] = A[t] + ((t / k == t % k) ? eps : 0.0);
    for (int i = tid; i < k; i += blockDim.x) perm[i] = i;
    __syncthreads();
    double pmin = 1e300;
    for (int c = 0; c < k; ++c) {
      // pivot: first row of the largest |LU[r][c]|, r >= c
      double best = -1.0;
      int bi = k;
      for (int r = c + tid; r < k; r += blockDim.x) {
        const double v = fabs(LU[r * k + c]);
        if (v > best) {
          best = v;
          bi = r;
        }
      }
      red[tid] = best;
      redi[tid] = bi;
      __syncthreads();
      for (int h = 64; h > 0; h >>= 1) {
        if (tid < h) {
          const double o = red[tid + h];
          const int oi = redi[tid + h];
          if (o > red[tid] || (o == red[tid] && oi < redi[tid])) {
            red[tid] = o;
            redi[tid] = oi;
          }
        }
        __syncthreads();
      }
      if (tid == 0) {
        piv_row = redi[0];
        if (piv_row != c) {
          const int t = perm[c];
          perm[c] = perm[piv_row];
          perm[piv_row] = t;
        }
      }
      __syncthreads();
      const int pr = piv_row;
      if (pr != c)
        for (int q = tid; q < k; q += blockDim.x) {
          const double t = LU[c * k + q];
          LU[c * k + q] = LU[pr * k + q];
          LU[pr * k + q] = t;
        }
      __syncthreads();
      const double d = LU[c * k + c];
      pmin = fmin(pmin, fabs(d));
      if (d != 0.0) {
        for (int r = c + 1 + tid; r < k; r += blockDim.x) LU[r * k + c] /= d;
        __syncthreads();
        const int rows = k - c - 1;
        for (int t = tid; t < rows * rows; t += blockDim.x) {
          const int r = c + 1 + t / rows, q = c + 1 + t % rows;
          LU[r * k + q] -= LU[r * k + c] * LU[c * k + q];
        }
      }
      __syncthreads();
    }
    if (attempt == 0 && amax > 0.0 && pmin >= 1e-12 * amax) {
      // accepted
    } else if (attempt == 0) {
      if (tid == 0) atomicOr(ridge, 1);
      __syncthreads();
      continue;
    }
    // solve: x = P b, forward (unit L), backward (U); one thread (k <= 128)
    if (tid == 0) {
      for (int i = 0; i < k; ++i) x[i] = C[perm[i] * ldc + j];
      for (int i = 0; i < k; ++i)
        for (int q = 0; q < i; ++q) x[i] -= LU[i * k + q] * x[q];
      for (int i = k - 1; i >= 0; --i) {
        for (int q = i + 1; q < k; ++q) x[i] -= LU[i * k + q] * x[q];
        x[i] /= LU[i * k + i];
      }
    }
    __syncthreads();
    for (int i = tid; i < k; i += blockDim.x) F[i * ldf + j] = x[i] + ((!replace_span && i == j) ? 1.0 : 0.0);
    return;
  }
}

inline size_t trip_solve_smem(int k) { return sizeof(double) * (2 * static_cast<size_t>(k) * k + k); }

__global__ void lam_new_kernel(const double* C, int ldc, const double* lam, int k, double* lam_new) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < k) lam_new[j] = lam[j] + C[j * ldc + j];
}

// renormalize_and_sort (trackers.cpp:43-52): columns of F scaled to unit
// ||Z f_j|| (G = Z'Z, D x D), then the columns and lambda_new in spectral
// order (types.hpp:26-40). One CTA.
__global__ void renorm_sort_kernel(const double* F, int ldf, int D, int k, const double* G, int ldg,
                                   const double* lam_new, int order, double* Fout, int ldo, double* vals) {
  __shared__ double nrm[kTrkMaxK];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = w; j < k; j += nw) {  // a warp per column: f' G f
    double s = 0.0;
    for (int a = lane; a < D; a += 32) {
      double g = 0.0;
      for (int b = 0; b < D; ++b) g += G[a * ldg + b] * F[b * ldf + j];
      s += F[a * ldf + j] * g;
    }
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(fmax(s, 0.0));
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    int rank = 0;
    const double vj = lam_new[j];
    for (int q = 0; q < k; ++q)
      if (q != j && spectral_before(lam_new[q], q, vj, j, order)) ++rank;
    vals[rank] = vj;
    const double s = nrm[j] > 0.0 ? nrm[j] : 1.0;
    for (int a = 0; a < D; ++a) Fout[a * ldo + rank] = nrm[j] > 0.0 ? F[a * ldf + j] / s : F[a * ldf + j];
  }
}

// sum of squares of n values (||Delta||_F^2, the TIMERS proxy), fixed order
__global__ void __launch_bounds__(256) sumsq_kernel(const double* v, i64 n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (i64 i = threadIdx.x; i < n; i += 256) s += v[i] * v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

}  // namespace stg
