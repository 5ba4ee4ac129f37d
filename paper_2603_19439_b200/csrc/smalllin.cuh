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
  kSpecFail = 16,      // a speculated decision (no suspect pivot, full sketch rank) failed: redo the step
};

// sticky |= (flags & mask) != 0 (deferred checks of a speculated step)
__global__ void or_sticky_kernel(const int* flags, int mask, int* sticky) {
  if (*flags & mask) *sticky = 1;
}

// the rank / keep decision of rsvd_basis (rsvd.hpp:59-63) on the device:
// lam_desc are the eigenvalues of bt_m' bt_m in descending order; the host
// speculated keep_assumed = min(L, qm).
__global__ void sketch_keep_kernel(const double* lam_desc, int qm, int L, int keep_assumed, const int* info,
                                   int* sticky) {
  if (threadIdx.x != 0) return;
  const double sv0 = sqrt(fmax(lam_desc[0], 0.0));
  const double cutoff = 1e-10 * sv0;
  int rank = 0;
  while (rank < qm) {
    const double sv = sqrt(fmax(lam_desc[rank], 0.0));
    if (!(sv > cutoff && sv > 0.0)) break;
    ++rank;
  }
  const int keep = rank < L ? rank : L;
  if (keep != keep_assumed || (info && *info != 0)) *sticky = 1;
}

// flags |= kSpecFail when the step's sticky word is set (gates the rotation)
__global__ void merge_spec_kernel(const int* sticky, int* flags) {
  if (*sticky) atomicOr(flags, kSpecFail);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Upper Cholesky G = R'R of a symmetric w x w block (row-major), one CTA of
// 512 threads, the upper triangle in shared memory (rows packed: row i holds
// columns i..w-1 at packed_row(i) + c). Blocked right-looking with panels of
// kCholNb rows and a one-panel lookahead:
//   A. all warps apply panel p's rank-kCholNb update to the rows of panel p+1;
//   B. warp 0 factors panel p+1's diagonal block in registers (the latency
//      chain: one pivot rsqrt per column) while the other warps apply panel
//      p's update to the rest of the trailing triangle (4 x 4 register tiles);
//   C. panel p+1's rows become R12 = R11^-T A12 (one thread per column).
// When orig2 is given, a pivot d_j <= tau2 * orig2[j] raises kSuspect: the
// column's residual is within sqrt(tau2) of its original norm, where the
// reference's per-column drop test (ortho.hpp:34-35) must be re-evaluated
// exactly. With psd != 0 a non-positive pivot zeroes the row (semidefinite
// factor) instead of failing.
constexpr int kCholMaxW = 238;
constexpr int kCholNb = 16;
constexpr int kCholThreads = 512;

__device__ __forceinline__ int packed_row(int i, int w) { return i * w - (i * (i - 1)) / 2 - i; }

// Diagonal block rows/cols p..p+b-1 by one warp: lane c holds column c
// (a[t] = A(p+t, p+c), t <= c); row t of R11 is broadcast by shuffles. Slots
// below a lane's diagonal hold don't-care values that never reach a valid
// slot, so the full-block variant runs without predicates.
template <bool FULL>
__device__ __forceinline__ void chol_diag_block(double* sm, double* invd, int w, int p, int b, int lane,
                                                const double* orig2, double tau2, int psd, int& fl) {
  const int cl = FULL ? (lane & (kCholNb - 1)) : (lane < b ? lane : b - 1);
  double a[kCholNb];
#pragma unroll
  for (int t = 0; t < kCholNb; ++t)
    a[t] = (FULL || t < b) && t <= cl ? sm[packed_row(p + t, w) + p + cl] : 0.0;
#pragma unroll
  for (int t = 0; t < kCholNb; ++t) {
    if (FULL || t < b) {
      const double d = __shfl_sync(0xffffffffu, a[t], t);
      const bool bad = !(d > 0.0) || !isfinite(d);
      if (lane == 0) {
        if (orig2 && !(d > tau2 * orig2[p + t])) fl |= kSuspect;
        if (bad && !psd) fl |= kBreakdown;
      }
      const double ir = bad ? 0.0 : rsqrt(d);
      a[t] = cl == t ? d * ir : a[t] * ir;
      if (lane == 0) invd[t] = ir;
#pragma unroll
      for (int u = t + 1; u < kCholNb; ++u) {
        const double rtu = __shfl_sync(0xffffffffu, a[t], u);  // R(t, u)
        if (FULL || u < b) a[u] -= rtu * a[t];
      }
    }
  }
  if (lane < b) {
#pragma unroll
    for (int t = 0; t < kCholNb; ++t)
      if (t <= lane) sm[packed_row(p + t, w) + p + lane] = a[t];
  }
}

template <typename... A>
__device__ __forceinline__ void chol_diag(int b, A&&... args) {  // forwarded: fl is an out-parameter
  if (b == kCholNb) chol_diag_block<true>(static_cast<A&&>(args)...);
  else chol_diag_block<false>(static_cast<A&&>(args)...);
}

// Rows p..p+b-1 (diagonal block already factored, 1/R(t,t) in invd): columns
// c >= p + b become R12 = R11^-T A12; one thread per column.
__device__ __forceinline__ void chol_panel(double* sm, const double* invd, int w, int p, int b, int tid, int nth) {
  for (int c = p + b + tid; c < w; c += nth) {
    double x[kCholNb];
#pragma unroll
    for (int t = 0; t < kCholNb; ++t) x[t] = t < b ? sm[packed_row(p + t, w) + c] : 0.0;
#pragma unroll
    for (int t = 0; t < kCholNb; ++t) {
      if (t < b) {
        x[t] *= invd[t];
        const int rt = packed_row(p + t, w);
#pragma unroll
        for (int u = t + 1; u < kCholNb; ++u)
          if (u < b) x[u] -= sm[rt + p + u] * x[t];
      }
    }
#pragma unroll
    for (int t = 0; t < kCholNb; ++t)
      if (t < b) sm[packed_row(p + t, w) + c] = x[t];
  }
}

// Rank-b update by panel p (rows p..p+b-1 hold R) of the elements (i, c),
// i in [r0, r1), c >= i, c >= q0, on the FP64 tensor pipe: a work item is an
// 8-row x 16-column block owned by one warp, A(i, c) -= sum_t R(t, i) R(t, c)
// as mma.sync m8n8k4 (SASS DMMA) over the b <= 16 panel rows, fragments
// loaded straight from the packed triangle (lane: panel row 4kk + lane % 4,
// matrix row/column lane / 4). The sum is formed first and then subtracted,
// as the scalar form did.
__device__ __forceinline__ void chol_trailing(double* sm, int w, int p, int b, int q0, int r0, int r1, int warp,
                                              int nwarps, int lane) {
  if (r1 <= r0) return;
  const int nb8 = (r1 - r0 + 7) >> 3;        // 8-row bands
  const int nch = (w - q0 + 15) >> 4;        // 16-column chunks
  const int tq = lane & 3, g = lane >> 2;
  int rb[4];                                 // packed row of panel row 4 kk + tq (-1: beyond the panel)
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) rb[kk] = 4 * kk + tq < b ? packed_row(p + 4 * kk + tq, w) : -1;
  for (int item = warp; item < nb8 * nch; item += nwarps) {
    const int band = item / nch, ch = item - band * nch;
    const int i0 = r0 + 8 * band, c0 = q0 + 16 * ch;
    if (c0 + 15 < i0) continue;  // chunk entirely left of the diagonal
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    const int ia = i0 + g, ca = c0 + g, cb = c0 + 8 + g;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const bool t_ok = rb[kk] >= 0;
      const double fa = t_ok && ia < w ? sm[rb[kk] + ia] : 0.0;
      const double fb0 = t_ok && ca < w ? sm[rb[kk] + ca] : 0.0;
      const double fb1 = t_ok && cb < w ? sm[rb[kk] + cb] : 0.0;
      dmma(a0, a1, fa, fb0);
      dmma(b0, b1, fa, fb1);
    }
    const int i = i0 + g;
    if (i >= r1) continue;
    double* rowi = sm + packed_row(i, w);
    const int cx = c0 + 2 * tq, cy = c0 + 8 + 2 * tq;
    if (cx < w && cx >= i) rowi[cx] -= a0;
    if (cx + 1 < w && cx + 1 >= i) rowi[cx + 1] -= a1;
    if (cy < w && cy >= i) rowi[cy] -= b0;
    if (cy + 1 < w && cy + 1 >= i) rowi[cy + 1] -= b1;
  }
}

__global__ void __launch_bounds__(kCholThreads) chol_kernel(const double* G, int ldg, int w, double* R, int ldr,
                                                            double* Rt, int ldrt, const double* orig2, double tau2,
                                                            int psd, int* flags, const int* gate) {
  if (gate && *gate == 0) return;  // near_identity_inverse_kernel already produced R^-1
  extern __shared__ double sm[];
  double* invd = sm + static_cast<i64>(w) * (w + 1) / 2;  // [2][kCholNb]: 1 / R(j,j) per panel parity
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < w; i += nth >> 5) {  // warp per row, all copies in flight at once
    const double* gi = G + static_cast<i64>(i) * ldg;
    double* si = sm + packed_row(i, w);
    double* ri = R + static_cast<i64>(i) * ldr;
    for (int c = lane; c < w; c += 32) {
      if (c >= i) cp_async8(si + c, gi + c);
      else ri[c] = 0.0;
    }
    if (Rt)
      for (int c = lane; c < i; c += 32) Rt[static_cast<i64>(i) * ldrt + c] = 0.0;  // R' is lower triangular
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  int fl = 0;
  if (warp == 0) chol_diag(min(kCholNb, w), sm, invd, w, 0, min(kCholNb, w), lane, orig2, tau2, psd, fl);
  __syncthreads();
  chol_panel(sm, invd, w, 0, min(kCholNb, w), tid, nth);
  __syncthreads();
  for (int p = 0, q = 0; p < w; p += kCholNb, q ^= 1) {
    const int b = min(kCholNb, w - p);
    const int p1 = p + b, b1 = min(kCholNb, w - p1);  // next panel
    // A. next panel's rows take panel p's update
    chol_trailing(sm, w, p, b, p1, p1, p1 + b1, warp, nth >> 5, lane);
    // rows of panel p are final
    for (int e = tid; e < b * (w - p); e += nth) {
      const int t = e / (w - p), c = p + (e - t * (w - p));
      if (c >= p + t) {
        const double v = sm[packed_row(p + t, w) + c];
        R[static_cast<i64>(p + t) * ldr + c] = v;
        if (Rt) Rt[static_cast<i64>(c) * ldrt + p + t] = v;
      }
    }
    __syncthreads();
    // B. warp 0: next diagonal block; the others: rest of the trailing update
    if (warp == 0) {
      if (b1 > 0) chol_diag(b1, sm, invd + (q ^ 1) * kCholNb, w, p1, b1, lane, orig2, tau2, psd, fl);
    } else {
      chol_trailing(sm, w, p, b, p1, p1 + b1, w, warp - 1, (nth >> 5) - 1, lane);
    }
    __syncthreads();
    // C. next panel rows
    if (b1 > 0) chol_panel(sm, invd + (q ^ 1) * kCholNb, w, p1, b1, tid, nth);
    __syncthreads();
  }
  if (fl) atomicOr(flags, fl);
}

inline size_t chol_smem_bytes(int w) {
  return sizeof(double) * (static_cast<size_t>(w) * (w + 1) / 2 + 2 * kCholNb);
}

// Inverse of an upper-triangular R given as R' (row-major lower triangle, as
// chol_kernel writes it; w <= 256). Each CTA stages R in shared memory as
// packed columns (column l holds rows 0..l), then each warp
// back-substitutes one column j of R^-1 in axpy form: once x_l is known,
// column l of R times x_l is added to the running sums of rows i < l (lane
// owns rows lane + 32 u), and x_{l-1} = -s_{l-1} / R(l-1,l-1) is broadcast
// from its owner. Entries below the diagonal are written as zeros; a zero
// pivot yields a zero row/column of the inverse.
constexpr int kTriWarps = 8;
constexpr int kTriMaxW = 256;

// Steps l = lhi .. 32 U + 1 of one column: rows i < l <= 32 (U + 1) live in
// slots u <= U, and x_{l-1} sits in slot U of lane (l-1) & 31.
template <int U>
__device__ __forceinline__ void triinv_segment(double (&s)[kTriMaxW / 32], double& xl, int lhi, int lane,
                                               const double* rc, const double* invd, double* Ri, int ldi, int j) {
  for (int l = lhi; l > 32 * U; --l) {
    const double* col = rc + l * (l + 1) / 2;
#pragma unroll
    for (int u = 0; u <= U; ++u) {
      const int i = lane + 32 * u;
      if (i < l) s[u] = fma(col[i], xl, s[u]);
    }
    const int o = l - 1;
    xl = -__shfl_sync(0xffffffffu, s[U], o & 31) * invd[o];
    if (lane == (o & 31)) Ri[static_cast<i64>(o) * ldi + j] = xl;
  }
}

__global__ void __launch_bounds__(32 * kTriWarps) triinv_kernel(const double* Rt, int ldrt, int w, double* Ri,
                                                                 int ldi, const int* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double rc[];
  double* invd = rc + static_cast<i64>(w) * (w + 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // column c of R = row c of R' (rows 0..c), contiguous: copies all in flight
  for (int c = warp; c < w; c += kTriWarps) {
    double* dst = rc + c * (c + 1) / 2;
    const double* src = Rt + static_cast<i64>(c) * ldrt;
    for (int i = lane; i <= c; i += 32) cp_async8(dst + i, src + i);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int i = tid; i < w; i += blockDim.x) {
    const double v = rc[i * (i + 1) / 2 + i];
    invd[i] = v != 0.0 ? 1.0 / v : 0.0;
  }
  __syncthreads();
  const int j = blockIdx.x * kTriWarps + warp;
  if (j >= w) return;
  for (int i = j + 1 + lane; i < w; i += 32) Ri[static_cast<i64>(i) * ldi + j] = 0.0;
  double s[kTriMaxW / 32];
#pragma unroll
  for (int u = 0; u < kTriMaxW / 32; ++u) s[u] = 0.0;
  double xl = invd[j];
  if (lane == (j & 31)) Ri[static_cast<i64>(j) * ldi + j] = xl;
  int l = j;
  while (l > 0) {
    const int U = (l - 1) >> 5;
    switch (U) {
      case 0: triinv_segment<0>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
      case 1: triinv_segment<1>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
      case 2: triinv_segment<2>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
      case 3: triinv_segment<3>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
      case 4: triinv_segment<4>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
      case 5: triinv_segment<5>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
      case 6: triinv_segment<6>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
      default: triinv_segment<7>(s, xl, l, lane, rc, invd, Ri, ldi, j); break;
    }
    l = 32 * U;
  }
}

inline size_t triinv_smem_bytes(int w) { return sizeof(double) * (static_cast<size_t>(w) * (w + 1) / 2 + w); }

// Second CholQR pass: G = Q1'Q1 = I + E with E at rounding level. Then
// R = I + split(E) + O(|E|^2) (split: strict upper part plus half the
// diagonal) and R^-1 = I - split(E) + O(|E|^2), and Q1 R^-1 is orthonormal to
// O(|E|^2 + eps): with max|E| <= kNearIdTol that is the same factor as the
// Cholesky one to rounding, without the w sequential pivots. One CTA writes
// that R^-1 and sets *gate = 1 (exact Cholesky still needed) when max|E| is
// larger; chol_kernel / triinv_kernel run only then.
constexpr double kNearIdTol = 1e-9;
__global__ void __launch_bounds__(1024) near_identity_inverse_kernel(const double* G, int ldg, int w, double* Ri,
                                                                     int ldi, int* gate) {
  __shared__ int big;
  if (threadIdx.x == 0) big = 0;
  __syncthreads();
  int local = 0;
  for (int i = threadIdx.x >> 5; i < w; i += blockDim.x >> 5) {
    const double* gi = G + static_cast<i64>(i) * ldg;
    double* ri = Ri + static_cast<i64>(i) * ldi;
    for (int c = threadIdx.x & 31; c < w; c += 32) {
      const double g = gi[c];
      const double e = c == i ? g - 1.0 : g;
      if (!(fabs(e) <= kNearIdTol)) local = 1;
      ri[c] = c < i ? 0.0 : (c == i ? 1.0 - 0.5 * e : -e);
    }
  }
  if (local) big = 1;
  __syncthreads();
  if (threadIdx.x == 0) *gate = big;
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

// max |G - I| > tol -> kNotOrthonormal (G symmetric: its upper triangle is read)
__global__ void orthocheck_kernel(const double* Gm, int ldg, int D, double tol, int* flags) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(D) * D) return;
  const int i = static_cast<int>(idx / D), j = static_cast<int>(idx % D);
  if (i > j) return;
  const double v = Gm[static_cast<i64>(i) * ldg + j] - (i == j ? 1.0 : 0.0);
  if (!(fabs(v) <= tol)) atomicOr(flags, kNotOrthonormal);
}

// M(D x D) = zx diag(lam) zx' + T   (Eq. 14, trackers.cpp:300-301), evaluated
// on (min(i,j), max(i,j)) so M is exactly symmetric (T, a mirrored Gram, is),
// and the eigensolver's (M + M')/2 (eig.hpp:47) is M itself.
// With zx_sym, zx is the symmetric D x D Gram Z'Z (X-bar = its first k
// columns) and only its upper triangle is read: zx(i, l) = G(min, max).
__global__ void rr_matrix_kernel(const double* zx, int ldzx, const double* lam, int k, const double* T, int ldt,
                                 int D, double* M, int ldm, int zx_sym) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(D) * D) return;
  const int i = static_cast<int>(idx / D), j = static_cast<int>(idx % D);
  const int lo = min(i, j), hi = max(i, j);
  auto zxa = [&](int r, int l) {
    if (!zx_sym) return zx[static_cast<i64>(r) * ldzx + l];
    return zx[static_cast<i64>(min(r, l)) * ldzx + max(r, l)];
  };
  double s = 0.0;
  for (int l = 0; l < k; ++l) s += zxa(lo, l) * lam[l] * zxa(hi, l);
  M[static_cast<i64>(i) * ldm + j] = s + T[static_cast<i64>(lo) * ldt + hi];
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

// pseudo-random fill in [-0.5, 0.5) (splitmix64 of the index; development checks)
__global__ void hash_fill_kernel(double* p, i64 n, unsigned long long seed) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  unsigned long long z = seed + 0x9e3779b97f4a7c15ULL * static_cast<unsigned long long>(idx + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z ^= z >> 31;
  p[idx] = static_cast<double>(z >> 11) * 0x1.0p-53 - 0.5;
}

// Copy a rows x cols block (row-major) between leading dimensions.
// mgs2_exact on the device (ortho.hpp:26-37): column c's drop decision from
// its squared norms before (o2) and after (n2) the two projection passes,
// nrm = sqrt(n2) < 1e-10 sqrt(o2) or a zero column drops it; a kept column is
// out[:, c] = v / nrm (the reference's division and square root, IEEE),
// a dropped one is zeroed, so later projections against out[:, :c] are the
// projections against the kept columns (zero columns add exact zeros).
__global__ void mgs_scale_kernel(const double* v, int ldv, i64 rows, const double* o2, const double* n2,
                                 double* out, int ldo, int* keep) {
  const double orig = sqrt(*o2), nrm = sqrt(*n2);
  const bool kept = orig != 0.0 && !(nrm < 1e-10 * orig);
  const double inv = kept ? 1.0 / nrm : 0.0;
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) *keep = kept ? 1 : 0;
  if (i < rows) out[i * ldo] = kept ? v[i * ldv] * inv : 0.0;
}

// Kept columns to the front, in order (row-parallel, in place: a row's
// writes only go to slots at or left of the column being read); r = count.
__global__ void mgs_compact_kernel(double* out, int ldo, i64 rows, const int* keep, int w, int* r) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) {
    int c = 0;
    for (int j = 0; j < w; ++j) c += keep[j];
    *r = c;
  }
  if (i >= rows) return;
  double* row = out + i * ldo;
  int d = 0;
  for (int j = 0; j < w; ++j)
    if (keep[j]) row[d++] = row[j];
}

__global__ void copy2d_kernel(const double* src, int lds, double* dst, int ldd, i64 rows, int cols) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const i64 r = idx / cols;
  const int c = static_cast<int>(idx % cols);
  dst[r * ldd + c] = src[r * lds + c];
}

}  // namespace stg
