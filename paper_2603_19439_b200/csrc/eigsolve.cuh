// Small dense symmetric eigensolver in one CTA (order n <= kEigMaxN), kept on
// the device for the projected Rayleigh-Ritz matrix (sym_eig_dense,
// proj/include/spectrack/eig.hpp:37-50) and the RSVD sketch Gram.
//
//   1. (S + S')/2 into shared memory: the full square when n <= kEigFullN
//      (rows contiguous), else the packed lower triangle,
//   2. Householder tridiagonalization (LAPACK dsytd2 recurrence) with three
//      barriers per column: every thread derives the reflector scalars itself,
//      p = A v runs four threads per row, and the rank-2 update is
//      A -= v p' + p v' - tau (p'v) v v' (= v w' + w v'),
//   3. all eigenvalues by Sturm-count bisection: one CTA-wide multisection
//      round brackets every eigenvalue, then 4 threads per eigenvalue to
//      full relative precision,
//   4. spectral ordering (types.hpp:26-40), selection of the leading `want`,
//   5. their eigenvectors by inverse iteration on the tridiagonal matrix with
//      partial pivoting and Gram-Schmidt inside eigenvalue clusters (the dstein
//      scheme), then the Householder back-transformation with the vector in
//      registers.
// Eigenvalues are accurate to O(eps ||S||) like the reference's QR-based
// SelfAdjointEigenSolver; eigenvectors of separated eigenvalues to
// O(eps ||S|| / gap); clusters get an orthonormal basis of their span.
#pragma once

#include <cfloat>

#include "common.cuh"
#include "smalllin.cuh"

namespace stg {

constexpr int kEigMaxN = 232;   // packed lower triangle + vectors fit in 227 KB of shared memory
constexpr int kEigFullN = 165;  // full square storage up to here (covers D <= 164 at config 3)
constexpr int kEigMaxWant = 256;

struct EigArgs {
  const double* M;  // row-major n x n (symmetrized here)
  int ldm;
  int n;
  int order;        // 0 abs_desc, 1 alg_desc
  int want;         // eigenvectors returned (leading in spectral order)
  double* w_sorted; // n eigenvalues in spectral order
  double* F;        // n x want row-major eigenvectors (column c = c-th in spectral order)
  int ldf;
  double* work;     // global scratch: want * 6 * n doubles
  int* flags;
  int* info;
  long long* prof;  // optional: clock64() at phase boundaries (thread 0)
  double ortol;     // cluster threshold relative to ||T||_1 (1e-3: dstein; looser when only spans matter)
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// Number of eigenvalues of the tridiagonal (d, e2 = e^2) strictly below x.
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int c = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  c += q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

template <bool FULL>
struct SymStore {
  double* A;
  int n;
  __device__ __forceinline__ double& at(int i, int j) const {  // element (i, j) of the symmetric matrix
    if (FULL) return A[i * n + j];
    if (i < j) {
      const int t = i;
      i = j;
      j = t;
    }
    return A[static_cast<i64>(j) * n - (static_cast<i64>(j) * (j - 1)) / 2 + (i - j)];
  }
  // reflector i, entry r > i + 1: row i (upper, contiguous) when FULL, column i when packed
  __device__ __forceinline__ double& refl(int r, int i) const {
    if (FULL) return A[i * n + r];
    return A[static_cast<i64>(i) * n - (static_cast<i64>(i) * (i - 1)) / 2 + (r - i)];
  }
  static __host__ __device__ i64 words(int n) {
    return FULL ? static_cast<i64>(n) * n : static_cast<i64>(n) * (n + 1) / 2;
  }
};

template <bool FULL>
__device__ void syev_body(const EigArgs& a, double* sm) {
  const int n = a.n;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  SymStore<FULL> S{sm, n};
  double* d = sm + SymStore<FULL>::words(n);  // diagonal
  double* e = d + n;                           // off-diagonal (n-1)
  double* tau = e + n;                         // Householder scalars
  double* p = tau + n;                         // A v, then e^2
  double* v = p + n;                           // Householder vector
  double* lam = v + n;                         // row partials during tridiag; ascending eigenvalues after
  double* red = lam + n;                       // 48 doubles reduction scratch
  int* perm = reinterpret_cast<int*>(red + 48);
  auto stamp = [&](int k) {
    if (a.prof && tid == 0) a.prof[k] = clock64();
  };
  stamp(0);
  // 1. symmetrize
  for (i64 idx = tid; idx < static_cast<i64>(n) * n; idx += nth) {
    const int i = static_cast<int>(idx / n), j = static_cast<int>(idx % n);
    if (!FULL && i < j) continue;
    const double x = a.M[static_cast<i64>(i) * a.ldm + j], y = a.M[static_cast<i64>(j) * a.ldm + i];
    if (!isfinite(x) || !isfinite(y)) atomicOr(a.flags, kNonFinite);
    S.at(i, j) = 0.5 * (x + y);
  }
  __syncthreads();
  {
    double part = 0.0;
    for (int r = 2 + tid; r < n; r += nth) part += S.at(r, 0) * S.at(r, 0);
    part = block_sum(part, red);
    if (tid == 0) red[40] = part;
    __syncthreads();
  }
  stamp(1);

  // 2. tridiagonalization
  for (int i = 0; i + 1 < n; ++i) {
    const int r0 = i + 1, m = n - r0;
    const double sigma = red[40];
    const double alpha = S.at(r0, i);
    double t = 0.0, scal = 0.0, beta = alpha;
    if (sigma > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (tid == 0) {
      tau[i] = t;
      e[i] = beta;
    }
    if (t == 0.0) {  // nothing to annihilate in this column
      double part = 0.0;
      for (int r = i + 3 + tid; r < n; r += nth) part += S.at(r, i + 1) * S.at(r, i + 1);
      part = block_sum(part, red);
      if (tid == 0) red[40] = part;
      __syncthreads();
      continue;
    }
    for (int r = r0 + tid; r < n; r += nth) v[r] = r == r0 ? 1.0 : S.at(r, i) * scal;
    __syncthreads();  // (1) v complete
    for (int r = r0 + 1 + tid; r < n; r += nth) S.refl(r, i) = v[r];  // column/row i is dead: keep the reflector
    {  // p = tau A22 v, four threads per row (nth / 4 >= m)
      const int q = tid & 3, r = r0 + (tid >> 2);
      double s = 0.0;
      if (r < n)
        for (int c = r0 + q; c < n; c += 4) s += S.at(r, c) * v[c];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (q == 0 && r < n) {
        p[r] = t * s;
        lam[r - r0] = t * s * v[r];
      }
    }
    __syncthreads();  // (2) p complete
    double pv = 0.0;  // every warp reduces p'v redundantly in a fixed order
    for (int r = lane; r < m; r += 32) pv += lam[r];
    pv = warp_sum(pv);
    const double b2 = t * pv;
    // A22 -= v p' + p v' - b2 v v'; both orders of each product pair are
    // identical in floating point, so the FULL storage stays exactly symmetric
    double part = 0.0;
    if (FULL) {
      for (int r = r0 + warp; r < n; r += nw) {
        const double vr = v[r], pr = p[r];
        for (int c = r0 + lane; c < n; c += 32) {
          const double vc = v[c];
          const double nv = S.at(r, c) - ((vr * p[c] + pr * vc) - b2 * (vr * vc));
          S.at(r, c) = nv;
          if (c == r0 && r >= r0 + 2) part += nv * nv;  // next column's norm below its subdiagonal
        }
      }
    } else {
      for (int c = r0 + warp; c < n; c += nw) {
        const double vc = v[c], pc = p[c];
        for (int r = c + lane; r < n; r += 32) {
          const double vr = v[r];
          const double nv = S.at(r, c) - ((vr * pc + p[r] * vc) - b2 * (vr * vc));
          S.at(r, c) = nv;
          if (c == r0 && r >= r0 + 2) part += nv * nv;
        }
      }
    }
    part = block_sum(part, red);  // (3)
    if (tid == 0) red[40] = part;
    __syncthreads();
  }
  for (int i = tid; i < n; i += nth) d[i] = S.at(i, i);
  if (tid == 0 && n == 1) e[0] = 0.0;
  __syncthreads();
  stamp(2);

  // 3. eigenvalues
  double* e2 = p;
  for (int i = tid; i + 1 < n; i += nth) e2[i] = e[i] * e[i];
  __syncthreads();
  if (tid == 0) {
    double lo = d[0], hi = d[0], emax = 0.0;
    for (int i = 0; i < n; ++i) {
      const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
      lo = fmin(lo, d[i] - r);
      hi = fmax(hi, d[i] + r);
      if (i + 1 < n) emax = fmax(emax, e2[i]);
    }
    const double tn = fmax(fabs(lo), fabs(hi));
    red[41] = lo - 2.0 * DBL_EPSILON * tn - DBL_MIN;
    red[42] = hi + 2.0 * DBL_EPSILON * tn + DBL_MIN;
    red[43] = fmax(DBL_MIN, DBL_MIN * emax) * 4.0;
  }
  __syncthreads();
  const double glo = red[41], ghi = red[42], pivmin = red[43];
  // one CTA-wide round at P equally spaced interior points; counts stored as
  // ints over the (v, lam) region (4n ints >= P)
  const int P = min(nth, 4 * n);
  int* cnt_g = reinterpret_cast<int*>(v);
  const double step = (ghi - glo) / (P + 1);
  if (tid < P) cnt_g[tid] = sturm_count(d, e2, n, glo + step * (tid + 1), pivmin);
  __syncthreads();
  const int j = tid >> 2, sub = tid & 3;  // nth / 4 >= n
  double lo = glo, hi = ghi;
  if (j < n) {
    int l0 = 0, l1 = P;  // first point with count > j
    while (l0 < l1) {
      const int mid = (l0 + l1) >> 1;
      if (cnt_g[mid] <= j) l0 = mid + 1; else l1 = mid;
    }
    lo = l0 > 0 ? glo + step * l0 : glo;
    hi = l0 < P ? glo + step * (l0 + 1) : ghi;
  }
  __syncthreads();  // brackets read before lam (aliasing the counts) is written
  for (int it = 0; it < 64; ++it) {
    const double width = hi - lo;
    const bool done = !(hi > nextafter(lo, DBL_MAX) && width > pivmin);  // adjacent floats
    const double x = lo + width * (sub + 1) * 0.2;
    const int cnt = (j < n && !done) ? sturm_count(d, e2, n, x, pivmin) : 0;
    const int gbase = lane & ~3;
    int nlo_idx = -1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cq = __shfl_sync(0xffffffffu, cnt, gbase + q);
      if (cq <= j) nlo_idx = q;
    }
    const unsigned all_done = __all_sync(0xffffffffu, done || j >= n);
    if (!done) {
      const double nlo = nlo_idx >= 0 ? lo + width * (nlo_idx + 1) * 0.2 : lo;
      const double nhi = nlo_idx + 1 < 4 ? lo + width * (nlo_idx + 2) * 0.2 : hi;
      lo = nlo;
      hi = nhi;
    }
    if (all_done) break;
  }
  // the largest float whose Sturm count is <= j: exact for representable eigenvalues
  if (j < n && sub == 0) lam[j] = lo;
  __syncthreads();
  stamp(3);

  // 4. spectral order of all eigenvalues (lam ascending by construction)
  for (int i = tid; i < n; i += nth) {
    int rank = 0;
    const double vi = lam[i];
    for (int jj = 0; jj < n; ++jj)
      if (jj != i && spectral_before(lam[jj], jj, vi, i, a.order)) ++rank;
    perm[rank] = i;
  }
  __syncthreads();
  for (int c = tid; c < n; c += nth) a.w_sorted[c] = lam[perm[c]];
  const int want = min(a.want, n);

  // 5. inverse iteration: selected eigenvalues ascending; a thread owns a whole
  // cluster (gap <= ortol ||T||_1) so Gram-Schmidt inside it is sequential.
  int* sel = perm + n;       // selected ascending indices (into lam)
  int* cstart = sel + n;     // cluster starts (n + 1)
  int* chosen = cstart + n + 1;
  __shared__ int s_ncl;
  __shared__ double s_tnorm;
  for (int i = tid; i < n; i += nth) chosen[i] = 0;
  __syncthreads();
  for (int c = tid; c < want; c += nth) chosen[perm[c]] = 1;
  __syncthreads();
  if (tid == 0) {
    double tn = 0.0;
    for (int i = 0; i < n; ++i)
      tn = fmax(tn, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0));
    s_tnorm = tn;
    int m = 0;
    for (int i = 0; i < n; ++i)
      if (chosen[i]) sel[m++] = i;
    int ncl = 0;
    for (int q = 0; q < m; ++q)
      if (q == 0 || lam[sel[q]] - lam[sel[q - 1]] > a.ortol * tn) cstart[ncl++] = q;
    cstart[ncl] = m;
    s_ncl = ncl;
  }
  __syncthreads();
  stamp(4);
  const int ncl = s_ncl;
  const double tnorm = s_tnorm > 0.0 ? s_tnorm : 1.0;
  for (int cl = tid; cl < ncl; cl += nth) {
    for (int q = cstart[cl]; q < cstart[cl + 1]; ++q) {
      double* x = a.work + static_cast<i64>(q) * 6 * n;
      double* dd = x + n;
      double* du = dd + n;
      double* du2 = du + n;
      double* dl = du2 + n;
      unsigned char* ip = reinterpret_cast<unsigned char*>(dl + n);
      double lambda = lam[sel[q]];
      if (q > cstart[cl] && lambda <= lam[sel[q - 1]] + 10.0 * DBL_EPSILON * tnorm)
        lambda = lam[sel[q - 1]] + 10.0 * DBL_EPSILON * tnorm * (q - cstart[cl]);
      // LU with partial pivoting of T - lambda I (dlagtf); the running row in registers
      double cur_d = d[0] - lambda, cur_u = n > 1 ? e[0] : 0.0;
      for (int i = 0; i + 1 < n; ++i) {
        const double sub_e = e[i];
        const double nd = d[i + 1] - lambda, nu = i + 2 < n ? e[i + 1] : 0.0;
        if (fabs(cur_d) >= fabs(sub_e)) {
          const double mlt = cur_d != 0.0 ? sub_e / cur_d : 0.0;
          ip[i] = 0;
          dl[i] = mlt;
          dd[i] = cur_d;
          du[i] = cur_u;
          du2[i] = 0.0;
          cur_d = nd - mlt * cur_u;
          cur_u = nu;
        } else {
          const double mlt = cur_d / sub_e;
          ip[i] = 1;
          dl[i] = mlt;
          dd[i] = sub_e;
          du[i] = nd;
          du2[i] = nu;
          cur_d = cur_u - mlt * nd;
          cur_u = -mlt * nu;
        }
      }
      dd[n - 1] = cur_d;
      du[n - 1] = 0.0;
      du2[n - 1] = 0.0;
      const double eps_piv = DBL_EPSILON * tnorm;
      for (int i = 0; i < n; ++i)
        if (fabs(dd[i]) < eps_piv) dd[i] = dd[i] < 0.0 ? -eps_piv : eps_piv;
      for (int i = 0; i < n; ++i) x[i] = 1.0 + 0.5 * __sinf(1.0f + 0.7f * i + 1.3f * q);
      for (int it = 0; it < 3; ++it) {
        double carry = x[0];
        for (int i = 0; i + 1 < n; ++i) {
          const double nx = x[i + 1];
          if (ip[i]) {
            x[i] = nx;
            carry = carry - dl[i] * nx;
          } else {
            x[i] = carry;
            carry = nx - dl[i] * carry;
          }
        }
        x[n - 1] = carry;
        double x1 = 0.0, x2 = 0.0;
        for (int i = n - 1; i >= 0; --i) {
          const double xi = (x[i] - du[i] * x1 - du2[i] * x2) / dd[i];
          x[i] = xi;
          x2 = x1;
          x1 = xi;
        }
        for (int pq = cstart[cl]; pq < q; ++pq) {
          const double* y = a.work + static_cast<i64>(pq) * 6 * n;
          double dot = 0.0;
          for (int i = 0; i < n; ++i) dot += x[i] * y[i];
          for (int i = 0; i < n; ++i) x[i] -= dot * y[i];
        }
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) nrm += x[i] * x[i];
        const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
        for (int i = 0; i < n; ++i) x[i] *= inv;
      }
    }
  }
  __syncthreads();
  __threadfence_block();
  stamp(5);

  // 6. back-transform Q x, warp per vector held in registers (lane l owns
  // entries l + 32 s), written as column c of F (c = spectral rank).
  constexpr int kSlots = (kEigMaxN + 31) / 32;
  for (int c = warp; c < want; c += nw) {
    const int li = perm[c];
    int q = 0;
    for (int tt = 0; tt < want; ++tt)
      if (sel[tt] == li) q = tt;
    const double* xg = a.work + static_cast<i64>(q) * 6 * n;
    double xr[kSlots];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      const int r = lane + 32 * s;
      xr[s] = r < n ? xg[r] : 0.0;
    }
    for (int i = n - 2; i >= 0; --i) {
      const double ti = tau[i];
      if (ti == 0.0) continue;
      const int r0 = i + 1;
      double vr[kSlots];
      double s = 0.0;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int r = lane + 32 * sl;
        vr[sl] = r == r0 ? 1.0 : ((r > r0 && r < n) ? S.refl(r, i) : 0.0);
        s += vr[sl] * xr[sl];
      }
      s = warp_sum(s) * ti;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) xr[sl] -= s * vr[sl];
    }
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      const int r = lane + 32 * s;
      if (r < n) a.F[static_cast<i64>(r) * a.ldf + c] = xr[s];
    }
  }
  __syncthreads();
  stamp(6);
  if (tid == 0) *a.info = 0;
}

__global__ void __launch_bounds__(1024) syev_kernel(EigArgs a) {
  extern __shared__ double sm[];
  if (a.n <= kEigFullN)
    syev_body<true>(a, sm);
  else
    syev_body<false>(a, sm);
}

inline size_t syev_smem_bytes(int n) {
  const size_t words = n <= kEigFullN ? static_cast<size_t>(n) * n : static_cast<size_t>(n) * (n + 1) / 2;
  return sizeof(double) * (words + 6 * static_cast<size_t>(n) + 48) + sizeof(int) * (4 * static_cast<size_t>(n) + 8);
}

}  // namespace stg
