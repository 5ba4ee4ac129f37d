// Small dense symmetric eigensolver in one CTA (order n <= kEigMaxN), kept on
// the device for the projected Rayleigh-Ritz matrix (sym_eig_dense,
// proj/include/spectrack/eig.hpp:37-50) and the RSVD sketch Gram.
//
//   1. (S + S')/2 into a packed lower triangle in shared memory,
//   2. Householder tridiagonalization (LAPACK dsytd2 recurrence),
//   3. all eigenvalues by Sturm-count multisection (4 threads / eigenvalue),
//   4. spectral ordering (types.hpp:26-40) and selection of the leading `want`,
//   5. their eigenvectors by inverse iteration on the tridiagonal matrix with
//      partial pivoting and Gram-Schmidt inside eigenvalue clusters (the dstein
//      scheme), back-transformed with the Householder reflectors.
// Eigenvalues are accurate to O(eps ||S||) like the reference's QR-based
// SelfAdjointEigenSolver; eigenvectors of separated eigenvalues to
// O(eps ||S|| / gap), and clusters get an orthonormal basis of their span.
#pragma once

#include <cfloat>

#include "common.cuh"
#include "smalllin.cuh"

namespace stg {

constexpr int kEigMaxN = 232;  // packed lower triangle + vectors fit in 227 KB of shared memory
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
  long long* prof;   // optional: clock64() at phase boundaries (thread 0)
  double ortol;      // cluster threshold relative to ||T||_1 (1e-3: dstein; looser when only spans matter)
};

__device__ __forceinline__ i64 pk(int n, int i, int j) {  // packed lower, column-major, i >= j
  return static_cast<i64>(j) * n - (static_cast<i64>(j) * (j - 1)) / 2 + (i - j);
}

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

__global__ void __launch_bounds__(1024) syev_kernel(EigArgs a) {
  extern __shared__ double sm[];
  const int n = a.n;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  const i64 npk = static_cast<i64>(n) * (n + 1) / 2;
  double* A = sm;                 // packed lower
  double* d = A + npk;            // diagonal
  double* e = d + n;              // off-diagonal (n-1)
  double* tau = e + n;            // Householder scalars
  double* v = tau + n;            // current Householder vector / scratch
  double* w = v + n;              // symv / rank-2 vector
  double* lam = w + n;            // ascending eigenvalues
  double* red = lam + n;          // 40 doubles reduction scratch
  int* perm = reinterpret_cast<int*>(red + 40);

  auto stamp = [&](int k) {
    if (a.prof && tid == 0) a.prof[k] = clock64();
  };
  stamp(0);
  // 1. symmetrize into packed storage
  for (i64 idx = tid; idx < static_cast<i64>(n) * n; idx += nth) {
    const int i = static_cast<int>(idx / n), j = static_cast<int>(idx % n);
    if (i < j) continue;
    const double x = a.M[static_cast<i64>(i) * a.ldm + j], y = a.M[static_cast<i64>(j) * a.ldm + i];
    if (!isfinite(x) || !isfinite(y)) atomicOr(a.flags, kNonFinite);
    A[pk(n, i, j)] = 0.5 * (x + y);
  }
  __syncthreads();

  stamp(1);
  // 2. tridiagonalization (dsytd2, lower)
  for (int i = 0; i + 1 < n; ++i) {
    const int r0 = i + 1;
    double part = 0.0;
    for (int r = r0 + 1 + tid; r < n; r += nth) part += A[pk(n, r, i)] * A[pk(n, r, i)];
    const double sigma = block_sum(part, red);
    if (tid == 0) {
      const double alpha = A[pk(n, r0, i)];
      double t = 0.0, scal = 0.0, beta = alpha;
      if (sigma > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      tau[i] = t;
      e[i] = beta;
      red[34] = scal;
    }
    __syncthreads();
    const double t = tau[i];
    if (t != 0.0) {
      const double scal = red[34];
      for (int r = r0 + tid; r < n; r += nth) {
        const double vr = r == r0 ? 1.0 : A[pk(n, r, i)] * scal;
        v[r] = vr;
        if (r > r0) A[pk(n, r, i)] = vr;
      }
      __syncthreads();
      // p = tau * A22 v (warp per row)
      for (int r = r0 + warp; r < n; r += nw) {
        double s = 0.0;
        for (int c = r0 + lane; c < n; c += 32) s += (r >= c ? A[pk(n, r, c)] : A[pk(n, c, r)]) * v[c];
        s = warp_sum(s);
        if (lane == 0) w[r] = t * s;
      }
      __syncthreads();
      double pv = 0.0;
      for (int r = r0 + tid; r < n; r += nth) pv += w[r] * v[r];
      pv = block_sum(pv, red);
      const double alpha2 = -0.5 * t * pv;
      for (int r = r0 + tid; r < n; r += nth) w[r] += alpha2 * v[r];
      __syncthreads();
      // A22 -= v w' + w v' (lower), warp per column
      for (int c = r0 + warp; c < n; c += nw) {
        const double vc = v[c], wc = w[c];
        for (int r = c + lane; r < n; r += 32) A[pk(n, r, c)] -= v[r] * wc + w[r] * vc;
      }
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += nth) d[i] = A[pk(n, i, i)];
  if (tid == 0 && n == 1) e[0] = 0.0;
  __syncthreads();

  stamp(2);
  // 3. eigenvalues: multisection with 4 threads per eigenvalue (groups inside a warp)
  double* e2 = w;  // reuse
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
    const double span = fmax(hi - lo, fmax(fabs(lo), fabs(hi)));
    red[35] = lo - 2.0 * DBL_EPSILON * span - DBL_MIN;
    red[36] = hi + 2.0 * DBL_EPSILON * span + DBL_MIN;
    red[37] = fmax(DBL_MIN, DBL_MIN * emax) * 4.0;
  }
  __syncthreads();
  const double glo = red[35], ghi = red[36], pivmin = red[37];
  for (int base = 0; base < n; base += nth / 4) {
    const int j = base + tid / 4, sub = tid & 3;
    double lo = glo, hi = ghi;
    for (int it = 0; it < 64; ++it) {
      const double width = hi - lo;
      const double tol = 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin;
      const bool done = !(width > tol);
      // points lo + width * (sub + 1) / 5
      const double x = lo + width * (sub + 1) * 0.2;
      const int cnt = (j < n && !done) ? sturm_count(d, e2, n, x, pivmin) : 0;
      // choose the sub-interval: counts are monotone in sub
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
    if (j < n && sub == 0) lam[j] = 0.5 * (lo + hi);
  }
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

  // 5. inverse iteration. Selected eigenvalues are handled in ascending order
  // of value; a thread owns a whole cluster (gap < 1e-3 ||T||_1, dstein's
  // ORTOL) so Gram-Schmidt inside the cluster is sequential and deterministic.
  int* sel = perm + n;        // selected ascending indices (into lam), size want
  int* cstart = sel + n;      // cluster starts
  __shared__ int s_ncl;
  __shared__ double s_tnorm;
  if (tid == 0) {
    double tn = 0.0;
    for (int i = 0; i < n; ++i)
      tn = fmax(tn, fabs(d[i]) + (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0));
    s_tnorm = tn;
    // selected indices sorted ascending (perm[0..want) are indices into ascending lam)
    int m = 0;
    for (int i = 0; i < n; ++i) {
      bool chosen = false;
      for (int c = 0; c < want; ++c) chosen |= perm[c] == i;
      if (chosen) sel[m++] = i;
    }
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
      double* dd = x + n;   // U diagonal
      double* du = dd + n;  // U first superdiagonal
      double* du2 = du + n; // U second superdiagonal
      double* dl = du2 + n; // L multipliers
      int* ip = reinterpret_cast<int*>(dl + n);  // pivot flags (n ints fit in n doubles)
      double lambda = lam[sel[q]];
      // perturb exactly repeated values inside a cluster (dstein)
      if (q > cstart[cl] && lambda <= lam[sel[q - 1]] + 10.0 * DBL_EPSILON * tnorm)
        lambda = lam[sel[q - 1]] + 10.0 * DBL_EPSILON * tnorm * (q - cstart[cl]);
      // LU with partial pivoting of T - lambda I (dlagtf)
      for (int i = 0; i < n; ++i) {
        dd[i] = d[i] - lambda;
        du[i] = i + 1 < n ? e[i] : 0.0;
        du2[i] = 0.0;
      }
      double sub = n > 1 ? e[0] : 0.0;
      for (int i = 0; i + 1 < n; ++i) {
        // rows i (dd[i], du[i], du2[i]) and i+1 (sub, dd[i+1], du[i+1])
        if (fabs(dd[i]) >= fabs(sub)) {
          ip[i] = 0;
          const double m = dd[i] != 0.0 ? sub / dd[i] : 0.0;
          dl[i] = m;
          dd[i + 1] -= m * du[i];
        } else {
          ip[i] = 1;
          const double m = dd[i] / sub;
          dl[i] = m;
          const double t0 = dd[i + 1], t1 = du[i + 1];
          dd[i] = sub;
          const double u0 = du[i];
          du[i] = t0;
          du2[i] = t1;
          dd[i + 1] = u0 - m * t0;
          du[i + 1] = -m * t1;
        }
        sub = i + 2 < n ? e[i + 1] : 0.0;
      }
      const double eps_piv = DBL_EPSILON * tnorm;
      for (int i = 0; i < n; ++i)
        if (fabs(dd[i]) < eps_piv) dd[i] = dd[i] < 0.0 ? -eps_piv : eps_piv;
      // deterministic start vector
      for (int i = 0; i < n; ++i) x[i] = 1.0 + 0.5 * sin(1.0 + 0.7 * i + 1.3 * q);
      for (int it = 0; it < 5; ++it) {
        // forward: apply L^-1 with the row interchanges
        for (int i = 0; i + 1 < n; ++i) {
          if (ip[i]) {
            const double t0 = x[i];
            x[i] = x[i + 1];
            x[i + 1] = t0 - dl[i] * x[i];
          } else {
            x[i + 1] -= dl[i] * x[i];
          }
        }
        // back: U x = y
        for (int i = n - 1; i >= 0; --i) {
          double s = x[i];
          if (i + 1 < n) s -= du[i] * x[i + 1];
          if (i + 2 < n) s -= du2[i] * x[i + 2];
          x[i] = s / dd[i];
        }
        // orthogonalize against earlier members of the cluster, normalize
        for (int pq = cstart[cl]; pq < q; ++pq) {
          const double* y = a.work + static_cast<i64>(pq) * 6 * n;
          double dot = 0.0;
          for (int i = 0; i < n; ++i) dot += x[i] * y[i];
          for (int i = 0; i < n; ++i) x[i] -= dot * y[i];
        }
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) nrm += x[i] * x[i];
        nrm = sqrt(nrm);
        const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
        for (int i = 0; i < n; ++i) x[i] *= inv;
      }
    }
  }
  __syncthreads();
  __threadfence_block();

  stamp(5);
  // 6. back-transform Q x (reflectors applied last to first), warp per vector,
  // written as column c of F where c is the vector's rank in spectral order.
  for (int c = warp; c < want; c += nw) {
    const int li = perm[c];
    int q = 0;
    for (int t = 0; t < want; ++t)
      if (sel[t] == li) q = t;
    double* x = a.work + static_cast<i64>(q) * 6 * n;
    for (int i = n - 2; i >= 0; --i) {
      const double t = tau[i];
      if (t == 0.0) continue;
      const int r0 = i + 1;
      double s = 0.0;
      for (int r = r0 + lane; r < n; r += 32) s += (r == r0 ? 1.0 : A[pk(n, r, i)]) * x[r];
      s = warp_sum(s) * t;
      for (int r = r0 + lane; r < n; r += 32) x[r] -= s * (r == r0 ? 1.0 : A[pk(n, r, i)]);
      __syncwarp();
    }
    for (int r = lane; r < n; r += 32) a.F[static_cast<i64>(r) * a.ldf + c] = x[r];
  }
  __syncthreads();
  stamp(6);
  if (tid == 0) *a.info = 0;
}

inline size_t syev_smem_bytes(int n) {
  return sizeof(double) * (static_cast<size_t>(n) * (n + 1) / 2 + 6 * static_cast<size_t>(n) + 40) +
         sizeof(int) * (3 * static_cast<size_t>(n) + 8);
}

}  // namespace stg
