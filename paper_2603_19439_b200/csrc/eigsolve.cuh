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
// Only step 2 needs a single CTA; steps 3-5 are separate kernels spread over
// the GPU (one group of threads per eigenvalue / eigenvector).
// Eigenvalues are accurate to O(eps ||S||) like the reference's QR-based
// SelfAdjointEigenSolver; eigenvectors of separated eigenvalues to
// O(eps ||S|| / gap); clusters get an orthonormal basis of their span.
#pragma once

#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "smalllin.cuh"

namespace stg {

constexpr int kEigMaxN = 232;   // packed lower triangle + vectors fit in 227 KB of shared memory
constexpr int kEigFullN = 165;  // full square storage up to here (covers D <= 164 at config 3)
constexpr int kEigMaxWant = 256;


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

// ---------------------------------------------------------------------------
// Multi-kernel pipeline: only the tridiagonalization needs one CTA; the
// eigenvalues (bisection), the inverse iterations and the back-transformation
// are independent per eigenvalue / eigenvector and run across the GPU.
struct EigBufs {
  double* d;       // n
  double* e;       // n
  double* e2;      // n
  double* tau;     // n
  double* V;       // n x n row-major: row i = Householder vector i (entries r > i+1; v[i+1] = 1)
  double* lam;     // n ascending eigenvalues
  double* Y;       // want x n tridiagonal eigenvectors (selection order)
  int* perm;       // n spectral ranks -> ascending index
  int* sel;        // want selected ascending indices
  int* cstart;     // want + 1 cluster starts
  int* ncl;        // 1
  double* tnorm;   // 1
};

template <bool FULL>
__device__ void tridiag_body(const double* M, int ldm, int n, const EigBufs b, int* flags, double* sm) {
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  SymStore<FULL> S{sm, n};
  double* v = sm + SymStore<FULL>::words(n);
  double* p = v + n;
  double* part_pv = p + n;  // n
  double* red = part_pv + n;  // 48
  for (i64 idx = tid; idx < static_cast<i64>(n) * n; idx += nth) {
    const int i = static_cast<int>(idx / n), j = static_cast<int>(idx % n);
    if (!FULL && i < j) continue;
    const double x = M[static_cast<i64>(i) * ldm + j], y = M[static_cast<i64>(j) * ldm + i];
    if (!isfinite(x) || !isfinite(y)) atomicOr(flags, kNonFinite);
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
      b.tau[i] = t;
      b.e[i] = beta;
      b.d[i] = S.at(i, i);
    }
    if (t == 0.0) {
      double part = 0.0;
      for (int r = i + 3 + tid; r < n; r += nth) part += S.at(r, i + 1) * S.at(r, i + 1);
      part = block_sum(part, red);
      if (tid == 0) red[40] = part;
      __syncthreads();
      continue;
    }
    for (int r = r0 + tid; r < n; r += nth) {
      const double vr = r == r0 ? 1.0 : S.at(r, i) * scal;
      v[r] = vr;
      b.V[static_cast<i64>(i) * n + r] = vr;
    }
    __syncthreads();  // (1) v complete
    // this lane's columns c = r0 + lane + 32 s: v and p are loaded once per
    // column step and reused across the warp's rows (the loops are bound by
    // shared-memory traffic)
    constexpr int kS = (kEigMaxN + 31) / 32;
    if (FULL) {
      double vc[kS];
#pragma unroll
      for (int sl = 0; sl < kS; ++sl) {
        const int c = r0 + lane + 32 * sl;
        vc[sl] = c < n ? v[c] : 0.0;
      }
      for (int r = r0 + warp; r < n; r += nw) {  // p = tau A22 v, warp per row
        const double* Ar = &S.at(r, 0);
        double s = 0.0;
#pragma unroll
        for (int sl = 0; sl < kS; ++sl) {
          const int c = r0 + lane + 32 * sl;
          if (c < n) s += Ar[c] * vc[sl];
        }
        s = warp_sum(s);
        if (lane == 0) {
          p[r] = t * s;
          part_pv[r - r0] = t * s * v[r];
        }
      }
      __syncthreads();  // (2) p complete
      double pv = 0.0;
      for (int r = lane; r < m; r += 32) pv += part_pv[r];
      pv = warp_sum(pv);
      const double b2 = t * pv;
      double pc[kS];
#pragma unroll
      for (int sl = 0; sl < kS; ++sl) {
        const int c = r0 + lane + 32 * sl;
        pc[sl] = c < n ? p[c] : 0.0;
      }
      double part = 0.0;
      for (int r = r0 + warp; r < n; r += nw) {
        const double vr = v[r], pr = p[r];
        double* Ar = &S.at(r, 0);
#pragma unroll
        for (int sl = 0; sl < kS; ++sl) {
          const int c = r0 + lane + 32 * sl;
          if (c < n) {
            const double nv = Ar[c] - ((vr * pc[sl] + pr * vc[sl]) - b2 * (vr * vc[sl]));
            Ar[c] = nv;
            if (c == r0 && r >= r0 + 2) part += nv * nv;
          }
        }
      }
      part = block_sum(part, red);  // (3)
      if (tid == 0) red[40] = part;
      __syncthreads();
      continue;
    }
    {
      const int q = tid & 3, r = r0 + (tid >> 2);
      double s = 0.0;
      if (r < n)
        for (int c = r0 + q; c < n; c += 4) s += S.at(r, c) * v[c];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (q == 0 && r < n) {
        p[r] = t * s;
        part_pv[r - r0] = t * s * v[r];
      }
    }
    __syncthreads();  // (2) p complete
    double pv = 0.0;
    for (int r = lane; r < m; r += 32) pv += part_pv[r];
    pv = warp_sum(pv);
    const double b2 = t * pv;
    double part = 0.0;
    for (int c = r0 + warp; c < n; c += nw) {
      const double vc = v[c], pc = p[c];
      for (int r = c + lane; r < n; r += 32) {
        const double vr = v[r];
        const double nv = S.at(r, c) - ((vr * pc + p[r] * vc) - b2 * (vr * vc));
        S.at(r, c) = nv;
        if (c == r0 && r >= r0 + 2) part += nv * nv;
      }
    }
    part = block_sum(part, red);  // (3)
    if (tid == 0) red[40] = part;
    __syncthreads();
  }
  if (tid == 0) {
    b.d[n - 1] = S.at(n - 1, n - 1);
    b.e[n - 1] = 0.0;
    b.tau[n - 1] = 0.0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += nth) b.e2[i] = b.e[i] * b.e[i];
}

__global__ void __launch_bounds__(1024) tridiag_kernel(const double* M, int ldm, int n, EigBufs b, int* flags) {
  extern __shared__ double sm[];
  if (n <= kEigFullN)
    tridiag_body<true>(M, ldm, n, b, flags, sm);
  else
    tridiag_body<false>(M, ldm, n, b, flags, sm);
}

inline size_t tridiag_smem_bytes(int n) {
  const size_t words = n <= kEigFullN ? static_cast<size_t>(n) * n : static_cast<size_t>(n) * (n + 1) / 2;
  return sizeof(double) * (words + 3 * static_cast<size_t>(n) + 48);
}

// Tridiagonalization on a thread-block cluster: the 8 CTAs of one cluster own
// the rows r = rank (mod 8) in full (n <= kEigMaxN: <= 30 rows x 232 cols per
// CTA in shared memory). Per column: the owner of row i builds the reflector
// and broadcasts it through distributed shared memory, every CTA computes
// p = tau A v for its rows and all-gathers it, then updates its rows. Two
// cluster barriers per column; v / p / partial buffers alternate by column
// parity so a CTA never overwrites a buffer another CTA is still reading.
constexpr int kClusterCtas = 8;
constexpr int kTriClusterThreads = 256;

__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kTriClusterThreads)
    tridiag_cluster_kernel(const double* M, int ldm, int n, EigBufs b, int* flags) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  extern __shared__ double sm[];
  const int nloc = (n - rank + kClusterCtas - 1) / kClusterCtas;  // rows rank, rank+8, ...
  const int nmax = (n + kClusterCtas - 1) / kClusterCtas;          // same layout in every CTA (DSMEM offsets)
  double* rows = sm;                                   // nmax x n
  double* vbuf = rows + static_cast<i64>(nmax) * n;    // [2][n]
  double* pbuf = vbuf + 2 * n;                         // [2][n]
  double* part = pbuf + 2 * n;                         // [2][kClusterCtas]
  double* scal = part + 2 * kClusterCtas;              // [2] tau per parity
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (i64 idx = tid; idx < static_cast<i64>(nloc) * n; idx += blockDim.x) {
    const int lr = static_cast<int>(idx / n), c = static_cast<int>(idx % n);
    const int r = rank + lr * kClusterCtas;
    const double x = M[static_cast<i64>(r) * ldm + c], y = M[static_cast<i64>(c) * ldm + r];
    if (!isfinite(x) || !isfinite(y)) atomicOr(flags, kNonFinite);
    rows[static_cast<i64>(lr) * n + c] = 0.5 * (x + y);
  }
  cluster.sync();
  for (int i = 0; i + 1 < n; ++i) {
    const int par = i & 1, r0 = i + 1;
    double* v = vbuf + par * n;
    double* p = pbuf + par * n;
    // 1. the owner of row i (= column i below the diagonal) builds the reflector
    if (i % kClusterCtas == rank && warp == 0) {
      const double* ri = rows + static_cast<i64>(i / kClusterCtas) * n;
      double sg = 0.0;
      for (int c = r0 + 1 + lane; c < n; c += 32) sg += ri[c] * ri[c];
      sg = warp_sum(sg);
      const double alpha = ri[r0];
      double t = 0.0, sc = 0.0, beta = alpha;
      if (sg > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sg), alpha);
        t = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      if (lane == 0) {
        b.tau[i] = t;
        b.e[i] = beta;
        b.d[i] = ri[i];
      }
      for (int dst = 0; dst < kClusterCtas; ++dst) {
        double* rv = cluster.map_shared_rank(v, dst);
        double* rs = cluster.map_shared_rank(scal, dst);
        for (int c = r0 + lane; c < n; c += 32) rv[c] = c == r0 ? 1.0 : ri[c] * sc;
        if (lane == 0) rs[par] = t;
      }
      for (int c = r0 + lane; c < n; c += 32) b.V[static_cast<i64>(i) * n + c] = c == r0 ? 1.0 : ri[c] * sc;
    }
    cluster.sync();  // (1) v, tau everywhere
    const double t = scal[par];
    // 2. p = tau A22 v on this CTA's rows r >= r0, all-gathered
    const int lr0 = (r0 - rank + kClusterCtas - 1) / kClusterCtas;  // first local row with r >= r0
    double pv_local = 0.0;
    if (t != 0.0) {
      for (int lr = lr0 + warp; lr < nloc; lr += nw) {
        const int r = rank + lr * kClusterCtas;
        const double* ar = rows + static_cast<i64>(lr) * n;
        double s = 0.0;
        for (int c = r0 + lane; c < n; c += 32) s += ar[c] * v[c];
        s = warp_sum(s) * t;
        if (lane < kClusterCtas) {
          double* rp = cluster.map_shared_rank(p, lane);
          rp[r] = s;
        }
        pv_local += s * v[r];  // identical in every lane after the butterfly
      }
    }
    // CTA partial of p'v (fixed order: warps, then ranks)
    __shared__ double wpart[32];
    if (lane == 0) wpart[warp] = pv_local;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += wpart[w];
      for (int dst = 0; dst < kClusterCtas; ++dst) cluster.map_shared_rank(part, dst)[par * kClusterCtas + rank] = s;
    }
    cluster.sync();  // (2) p and partials everywhere
    if (t == 0.0) continue;
    double pv = 0.0;
    for (int q = 0; q < kClusterCtas; ++q) pv += part[par * kClusterCtas + q];
    const double b2 = t * pv;
    // 3. update this CTA's rows: A -= v p' + p v' - b2 v v'
    for (int lr = lr0 + warp; lr < nloc; lr += nw) {
      const int r = rank + lr * kClusterCtas;
      double* ar = rows + static_cast<i64>(lr) * n;
      const double vr = v[r], pr = p[r];
      for (int c = r0 + lane; c < n; c += 32) {
        const double vc = v[c];
        ar[c] -= (vr * p[c] + pr * vc) - b2 * (vr * vc);
      }
    }
    __syncthreads();  // this CTA's rows are final for column i+1's owner
  }
  if ((n - 1) % kClusterCtas == rank && tid == 0) {
    b.d[n - 1] = rows[static_cast<i64>((n - 1) / kClusterCtas) * n + (n - 1)];
    b.e[n - 1] = 0.0;
    b.tau[n - 1] = 0.0;
  }
  cluster.sync();
  if (rank == 0)
    for (int i = tid; i < n; i += blockDim.x) b.e2[i] = b.e[i] * b.e[i];
}

inline size_t tridiag_cluster_smem_bytes(int n) {
  const int nloc = (n + kClusterCtas - 1) / kClusterCtas;
  return sizeof(double) * (static_cast<size_t>(nloc) * n + 4 * static_cast<size_t>(n) + 2 * kClusterCtas + 2);
}

// All eigenvalues of the tridiagonal matrix by bisection on Sturm counts:
// 8 threads per eigenvalue multisect (9-way split per step) until the bracket
// is below max(2 eps |lambda|, eps ||T||), the absolute accuracy of QR-based
// solvers; the returned value is the bracket's lower end (count <= j).
constexpr int kBisG = 8;
__global__ void __launch_bounds__(128) bisect_kernel(EigBufs b, int n) {
  extern __shared__ double sh[];
  double* d = sh;
  double* e2 = sh + n;
  __shared__ double s_lo, s_hi, s_piv, s_tn;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    d[i] = b.d[i];
    e2[i] = b.e2[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double lo = d[0], hi = d[0], emax = 0.0;
    for (int i = 0; i < n; ++i) {
      const double ei = i + 1 < n ? sqrt(e2[i]) : 0.0, ep = i > 0 ? sqrt(e2[i - 1]) : 0.0;
      lo = fmin(lo, d[i] - ep - ei);
      hi = fmax(hi, d[i] + ep + ei);
      if (i + 1 < n) emax = fmax(emax, e2[i]);
    }
    const double tn = fmax(fabs(lo), fabs(hi));
    s_lo = lo - 2.0 * DBL_EPSILON * tn - DBL_MIN;
    s_hi = hi + 2.0 * DBL_EPSILON * tn + DBL_MIN;
    s_piv = fmax(DBL_MIN, DBL_MIN * emax) * 4.0;
    s_tn = tn;
    if (blockIdx.x == 0) *b.tnorm = tn;
  }
  __syncthreads();
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = gtid / kBisG, sub = gtid % kBisG, lane = threadIdx.x & 31;
  const double pivmin = s_piv, atol = DBL_EPSILON * s_tn;
  double lo = s_lo, hi = s_hi;
  constexpr double kStep = 1.0 / (kBisG + 1);
  for (int it = 0; it < 64; ++it) {
    const double width = hi - lo;
    const bool done = !(width > fmax(2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)), atol) && width > pivmin);
    const double x = lo + width * (sub + 1) * kStep;
    const int cnt = (j < n && !done) ? sturm_count(d, e2, n, x, pivmin) : 0;
    const int gbase = lane & ~(kBisG - 1);
    int nlo_idx = -1;
#pragma unroll
    for (int q = 0; q < kBisG; ++q) {
      const int cq = __shfl_sync(0xffffffffu, cnt, gbase + q);
      if (cq <= j) nlo_idx = q;
    }
    const unsigned all_done = __all_sync(0xffffffffu, done || j >= n);
    if (!done) {
      const double nlo = nlo_idx >= 0 ? lo + width * (nlo_idx + 1) * kStep : lo;
      const double nhi = nlo_idx + 1 < kBisG ? lo + width * (nlo_idx + 2) * kStep : hi;
      lo = nlo;
      hi = nhi;
    }
    if (all_done) break;
  }
  if (j < n && sub == 0) b.lam[j] = lo;
}

// Spectral order of all eigenvalues, the leading `want`, and their clusters
// (consecutive selected values closer than ortol ||T||_1, dstein's ORTOL).
__global__ void __launch_bounds__(1024) select_kernel(EigBufs b, int n, int order, int want, double ortol,
                                                      double* w_sorted) {
  extern __shared__ int shi[];
  int* chosen = shi;
  const double* lam = b.lam;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rank = 0;
    const double vi = lam[i];
    for (int jj = 0; jj < n; ++jj)
      if (jj != i && spectral_before(lam[jj], jj, vi, i, order)) ++rank;
    b.perm[rank] = i;
    chosen[i] = rank < want ? 1 : 0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) w_sorted[c] = lam[b.perm[c]];
  if (threadIdx.x == 0) {
    const double tn = *b.tnorm;
    int m = 0;
    for (int i = 0; i < n; ++i)
      if (chosen[i]) b.sel[m++] = i;
    int ncl = 0;
    for (int q = 0; q < m; ++q)
      if (q == 0 || lam[b.sel[q]] - lam[b.sel[q - 1]] > ortol * tn) b.cstart[ncl++] = q;
    b.cstart[ncl] = m;
    *b.ncl = ncl;
  }
}

// Inverse iteration (dlagtf/dlagts with partial pivoting, 3 sweeps) for each
// selected eigenvalue; one thread owns one cluster and re-orthogonalizes its
// members in order. Working vectors live in shared memory (8 threads / CTA).
constexpr int kInvitThreads = 8;
__global__ void __launch_bounds__(kInvitThreads) invit_kernel(EigBufs b, int n) {
  extern __shared__ double sh[];
  const int cl = blockIdx.x * blockDim.x + threadIdx.x;
  double* d = sh;
  double* e = sh + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    d[i] = b.d[i];
    e[i] = b.e[i];
  }
  __syncthreads();
  if (cl >= *b.ncl) return;
  double* x = sh + 2 * n + static_cast<i64>(threadIdx.x) * 5 * n;
  double* dd = x + n;
  double* du = dd + n;
  double* du2 = du + n;
  double* dl = du2 + n;
  unsigned ipm[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // pivot flags, n <= 256
  const double tnorm = *b.tnorm > 0.0 ? *b.tnorm : 1.0;
  const int c0 = b.cstart[cl], c1 = b.cstart[cl + 1];
  for (int q = c0; q < c1; ++q) {
    double lambda = b.lam[b.sel[q]];
    if (q > c0 && lambda <= b.lam[b.sel[q - 1]] + 10.0 * DBL_EPSILON * tnorm)
      lambda = b.lam[b.sel[q - 1]] + 10.0 * DBL_EPSILON * tnorm * (q - c0);
    double cur_d = d[0] - lambda, cur_u = n > 1 ? e[0] : 0.0;
    for (int w = 0; w < 8; ++w) ipm[w] = 0;
    for (int i = 0; i + 1 < n; ++i) {
      const double sub_e = e[i];
      const double nd = d[i + 1] - lambda, nu = i + 2 < n ? e[i + 1] : 0.0;
      if (fabs(cur_d) >= fabs(sub_e)) {
        const double mlt = cur_d != 0.0 ? sub_e / cur_d : 0.0;
        dl[i] = mlt;
        dd[i] = cur_d;
        du[i] = cur_u;
        du2[i] = 0.0;
        cur_d = nd - mlt * cur_u;
        cur_u = nu;
      } else {
        const double mlt = cur_d / sub_e;
        ipm[i >> 5] |= 1u << (i & 31);
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
        if ((ipm[i >> 5] >> (i & 31)) & 1u) {
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
      for (int pq = c0; pq < q; ++pq) {
        const double* y = b.Y + static_cast<i64>(pq) * n;
        double dot = 0.0;
        for (int i = 0; i < n; ++i) dot += x[i] * y[i];
        for (int i = 0; i < n; ++i) x[i] -= dot * y[i];
      }
      double nrm = 0.0;
      for (int i = 0; i < n; ++i) nrm += x[i] * x[i];
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      for (int i = 0; i < n; ++i) x[i] *= inv;
    }
    double* y = b.Y + static_cast<i64>(q) * n;
    for (int i = 0; i < n; ++i) y[i] = x[i];
  }
}

inline size_t invit_smem_bytes(int n) { return sizeof(double) * (2 + 5 * kInvitThreads) * static_cast<size_t>(n); }

// Back-transformation Q y with the reflectors (last to first), warp per vector
// in registers; the CTA's 4 warps share reflector rows staged through shared
// memory 16 at a time. Column c of F = the c-th leading eigenvector.
constexpr int kBtRows = 16;
__global__ void __launch_bounds__(128) backtransform_kernel(EigBufs b, int n, int want, double* F, int ldf) {
  extern __shared__ double vs[];  // kBtRows x n
  const int c = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const bool active = c < want;
  constexpr int kSlots = (kEigMaxN + 31) / 32;
  double xr[kSlots];
  if (active) {
    const int li = b.perm[c];
    int q = 0;
    for (int tt = 0; tt < want; ++tt)
      if (b.sel[tt] == li) q = tt;
    const double* yg = b.Y + static_cast<i64>(q) * n;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      const int r = lane + 32 * s;
      xr[s] = r < n ? yg[r] : 0.0;
    }
  }
  for (int top = n - 2; top >= 0; top -= kBtRows) {
    const int lo = max(0, top - kBtRows + 1);
    __syncthreads();
    for (int idx = threadIdx.x; idx < (top - lo + 1) * n; idx += blockDim.x) {
      const int ii = lo + idx / n, r = idx % n;
      vs[(ii - lo) * n + r] = r == ii + 1 ? 1.0 : (r > ii + 1 ? b.V[static_cast<i64>(ii) * n + r] : 0.0);
    }
    __syncthreads();
    if (!active) continue;
    for (int i = top; i >= lo; --i) {
      const double ti = b.tau[i];
      if (ti == 0.0) continue;
      const double* vrow = vs + (i - lo) * n;
      double vr[kSlots];
      double s = 0.0;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int r = lane + 32 * sl;
        vr[sl] = r < n ? vrow[r] : 0.0;
        s += vr[sl] * xr[sl];
      }
      s = warp_sum(s) * ti;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) xr[sl] -= s * vr[sl];
    }
  }
  if (!active) return;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const int r = lane + 32 * s;
    if (r < n) F[static_cast<i64>(r) * ldf + c] = xr[s];
  }
}

// Host side: scratch sizing and the five launches. `L` launches a kernel
// (grid, block, smem, args...) on the caller's stream.
inline size_t eig_scratch_doubles(int n, int want) {
  return static_cast<size_t>(n) * (6 + n) + static_cast<size_t>(want) * n + 8;
}
inline size_t eig_scratch_ints(int n, int want) { return static_cast<size_t>(n) + 2 * static_cast<size_t>(want) + 8; }

inline EigBufs eig_carve(double* dbuf, int* ibuf, int n, int want) {
  EigBufs b{};
  b.d = dbuf;
  b.e = b.d + n;
  b.e2 = b.e + n;
  b.tau = b.e2 + n;
  b.lam = b.tau + n;
  b.tnorm = b.lam + n;
  b.V = b.tnorm + 2;
  b.Y = b.V + static_cast<i64>(n) * n;
  b.perm = ibuf;
  b.sel = b.perm + n;
  b.cstart = b.sel + want;
  b.ncl = b.cstart + want + 1;
  return b;
}

template <class Launch>
void syev_launch(Launch&& L, const double* M, int ldm, int n, int order, int want, double ortol, double* w_sorted,
                 double* F, int ldf, double* dbuf, int* ibuf, int* flags) {
  const EigBufs b = eig_carve(dbuf, ibuf, n, want);
  L(tridiag_cluster_kernel, dim3(kClusterCtas), dim3(kTriClusterThreads), tridiag_cluster_smem_bytes(n), M, ldm, n, b,
    flags);
  L(bisect_kernel, dim3(static_cast<unsigned>(cdiv(kBisG * n, 128))), dim3(128), sizeof(double) * 2 * n, b, n);
  L(select_kernel, dim3(1), dim3(256), sizeof(int) * n, b, n, order, want, ortol, w_sorted);
  L(invit_kernel, dim3(static_cast<unsigned>(cdiv(want, kInvitThreads))), dim3(kInvitThreads), invit_smem_bytes(n), b,
    n);
  L(backtransform_kernel, dim3(static_cast<unsigned>(cdiv(want, 4))), dim3(128), sizeof(double) * kBtRows * n, b, n,
    want, F, ldf);
}

}  // namespace stg
