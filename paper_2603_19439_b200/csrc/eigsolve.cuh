// Small dense symmetric eigensolver (order n <= kEigMaxN) kept on the device
// for the projected Rayleigh-Ritz matrix (sym_eig_dense,
// proj/include/spectrack/eig.hpp:37-50) and the RSVD sketch Gram.
//
//   1. (S + S')/2 and Householder tridiagonalization (LAPACK dsytd2
//      recurrence) in one CTA (n <= kEig1N, full square in shared memory) or
//      a 2-CTA cluster (rows split by parity), two barriers per column,
//   2. all eigenvalues by Sturm-count multisection, kBisG threads per
//      eigenvalue, to the absolute accuracy of a QR-based solver,
//   3. spectral ordering (types.hpp:26-40), selection of the leading `want`,
//   4. their eigenvectors by inverse iteration on the tridiagonal matrix with
//      partial pivoting and Gram-Schmidt inside eigenvalue clusters (the dstein
//      scheme), then the Householder back-transformation.
// Steps 2-4 are separate kernels spread over the GPU (one group of threads per
// eigenvalue / eigenvector).
// Eigenvalues are accurate to O(eps ||S||) like the reference's QR-based
// SelfAdjointEigenSolver; eigenvectors of separated eigenvalues to
// O(eps ||S|| / gap); clusters get an orthonormal basis of their span.
#pragma once

#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "smalllin.cuh"

namespace stg {

constexpr int kEigMaxN = 228;   // 114 rows x 228 columns per CTA of a 2-CTA cluster + scratch fit in 227 KB (D <= 228 at configs 4-5)
constexpr int kEigMaxWant = 256;


// Number of eigenvalues of the tridiagonal (d, e2 = e^2) strictly below x.
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  int c = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  c += q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] * __drcp_rn(q);
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

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

// Householder tridiagonalization (LAPACK dsytd2 recurrence) with the rows of
// (S + S')/2 spread over a cluster of C CTAs (C = 1: one CTA holding the full
// square, n <= kEig1N; C = 2 up to kEigMaxN): CTA q keeps rows r = q (mod C)
// in full width in shared memory. Column i (col = A(:, i)), its alpha and the
// shares of its squared norm were published in every CTA by the previous step.
// Per column, with r0 = i + 1 and v = (1, scal col[r0+1:]):
//   S. acc_r = sum_{c > r0} A(c, r) col[c] over the CTA's rows c, using the
//      symmetry A(c, r) = A(r, c): warp w owns 32 consecutive r and runs down
//      the rows, so loads are conflict-free and no butterfly is needed; the
//      sums are unscaled, so they need no reflector scalars. acc, row r0
//      (a0 = A(r0, :), from its owner) and the unscaled pieces of (Av)'v are
//      published; the last warp meanwhile derives beta, tau, scal.
//      -- barrier --
//   U. (Av)_r = a0_r + scal sum_q acc_q,r, p = tau Av, b2 = tau p'v and
//      A(c, r) -= v_c (p_r - b2 v_r) + p_c v_r on the CTA's rows (slot count
//      specialised, so no predicated-off lanes); the new column i+1, its alpha
//      and squared-norm shares are published.  -- barrier --
// Two barriers per column; every cross-CTA buffer alternates with the column
// parity, so a write never races a read of the previous column. The
// reference symmetrises its input (eig.hpp:47) the same way.
constexpr int kTriThreads = 512;
constexpr int kTriW = kTriThreads / 32;
constexpr int kEig1N = 165;  // one CTA holds the full square up to here
constexpr int kTriSlots = (kEigMaxN + 31) / 32;

__host__ __device__ inline int tri_rows(int n, int C) { return (n + C - 1) / C; }

// scratch after the rows: col[2][n], a0[2][n], p/v/w[3][n], acc[2][C * gmax][n], (Av)'v pieces
// [2][C * kTriW][4], reflector scalars [2][4]. gmax = warps sharing one
// 32-column block of the column sums (as many as shared memory allows, <= 4).
inline size_t tridiag_smem_bytes(int n, int C, int gmax) {
  return sizeof(double) * (static_cast<size_t>(tri_rows(n, C)) * n + (7 + 2 * static_cast<size_t>(C) * gmax) * n +
                           2 * static_cast<size_t>(C) * kTriW * 4 + 8);
}
inline int tridiag_gmax(int n, int C) {
  int g = 4;
  while (g > 1 && tridiag_smem_bytes(n, C, g) > 232448) --g;
  return g;
}

template <int C>
__device__ __forceinline__ void tri_sync() {
  if constexpr (C == 1) {
    __syncthreads();
  } else {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
}

template <int C>
__device__ __forceinline__ double* tri_peer(double* p, int q) {
  if constexpr (C == 1) {
    return p;
  } else {
    return cooperative_groups::this_cluster().map_shared_rank(p, q);
  }
}

#ifdef STG_TRI_PROF  // development probe (tools/microbench/tri_parts.cu): cycles per phase, thread 0
__device__ long long g_tri_prof[8];
#define STG_TRI_MARK(k)                                  \
  do {                                                   \
    if (threadIdx.x == 0) {                              \
      const long long now_ = clock64();                  \
      g_tri_prof[k] += now_ - prof_t_;                   \
      prof_t_ = now_;                                    \
    }                                                    \
  } while (0)
#else
#define STG_TRI_MARK(k) \
  do {                  \
  } while (0)
#endif

// U for NS live 32-column slots: rows lr = lb, lb + kTriW, ... of this warp
// U for NS live 32-column slots: A(r, c) -= v_r w_c + p_r v_c on this warp's
// rows, w = p - b2 v; p, v, w precomputed in shared memory for the column.
template <int NS>
__device__ __forceinline__ void tri_update_rows(double* A, int n, int r0, int C, int rank, int lr0, int my_rows,
                                                int warp, int lane, const double* Pv, const double* Vv,
                                                const double* Wv) {
  double vc[NS], wc[NS];
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    const int c = r0 + lane + 32 * sl;
    vc[sl] = c < n ? Vv[c] : 0.0;
    wc[sl] = c < n ? Wv[c] : 0.0;
  }
  for (int lb = lr0 + warp; lb < my_rows; lb += 2 * kTriW) {  // two rows per pass
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int lr = lb + u * kTriW;
      if (lr < my_rows) {
        const int rr = lr * C + rank;
        const double vr = Vv[rr], pr = Pv[rr];
        double* Ar = A + static_cast<i64>(lr) * n + r0 + lane;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
          if (sl < NS - 1 || r0 + lane + 32 * sl < n) Ar[32 * sl] = fma(-vr, wc[sl], fma(-pr, vc[sl], Ar[32 * sl]));
        }
      }
    }
  }
}

template <int C>
__device__ void tridiag_body(const double* M, int ldm, int n, int sym_input, int gmax, EigBufs b, int* flags,
                             int rank) {
#ifdef STG_TRI_PROF
  long long prof_t_ = clock64();
#endif
  extern __shared__ double sm[];
  const int nloc = tri_rows(n, C);
  double* A = sm;                                   // nloc x n, local row lr <-> row lr C + rank
  double* colb = A + static_cast<i64>(nloc) * n;    // [2][n] column i by parity
  double* a0b = colb + 2 * n;                       // [2][n] row r0 by parity
  double* Pv = a0b + 2 * n;                         // [n] p = tau A v
  double* Vv = Pv + n;                              // [n] v
  double* Wv = Vv + n;                              // [n] w = p - tau (p'v) v
  double* accb = Wv + n;                            // [2][C * gmax][n] partial column sums by parity
  const int nacc_max = C * gmax;
  double* pvs = accb + 2 * static_cast<i64>(nacc_max) * n;  // [2][C * kTriW][4]: (Av)'v pieces, squared-norm share
  double* scl = pvs + 2 * C * kTriW * 4;            // [2] x {tau, scal, beta, alpha}
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int my_rows = (n - rank + C - 1) / C;
  // load (S + S')/2 and publish column 0 (its squared norm in slot 3, its alpha)
  double sg = 0.0;
  if (sym_input) {  // exactly mirrored producers: (S + S')/2 = S, rows copied with every request in flight
    for (int lr = warp; lr < my_rows; lr += kTriW) {
      const int r = lr * C + rank;
      for (int c = lane; c < n; c += 32) cp_async8(A + static_cast<i64>(lr) * n + c, M + static_cast<i64>(r) * ldm + c);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    int bad = 0;
    for (int lr = warp; lr < my_rows; lr += kTriW)
      for (int c = lane; c < n; c += 32) bad |= !isfinite(A[static_cast<i64>(lr) * n + c]);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, kNonFinite);
    for (int lr = tid; lr < my_rows; lr += kTriThreads) {
      const int r = lr * C + rank;
      const double v = A[static_cast<i64>(lr) * n];
      for (int q = 0; q < C; ++q) tri_peer<C>(colb, q)[r] = v;
      if (r >= 2) sg += v * v;
      if (r == 1)
        for (int q = 0; q < C; ++q) tri_peer<C>(scl, q)[3] = v;
    }
  } else {
    for (int lr = warp; lr < my_rows; lr += kTriW) {
      const int r = lr * C + rank;
      double* Ar = A + static_cast<i64>(lr) * n;
      for (int c = lane; c < n; c += 32) {
        const double x = M[static_cast<i64>(r) * ldm + c];
        const double y = M[static_cast<i64>(c) * ldm + r];
        if (!isfinite(x) || !isfinite(y)) atomicOr(flags, kNonFinite);
        const double v = 0.5 * (x + y);
        Ar[c] = v;
        if (c == 0) {
          for (int q = 0; q < C; ++q) tri_peer<C>(colb, q)[r] = v;
          if (r >= 2) sg += v * v;
          if (r == 1)
            for (int q = 0; q < C; ++q) tri_peer<C>(scl, q)[3] = v;
        }
      }
    }
  }
  sg = warp_sum(sg);
  if (lane == 0)
    for (int q = 0; q < C; ++q) tri_peer<C>(pvs, q)[(rank * kTriW + warp) * 4 + 3] = sg;
  tri_sync<C>();
  STG_TRI_MARK(0);
  for (int i = 0; i + 1 < n; ++i) {
    const int par = i & 1, npar = par ^ 1, r0 = i + 1;
    const double* col = colb + par * n;
    double* a0 = a0b + par * n;
    double* acc = accb + static_cast<i64>(par) * nacc_max * n;
    double* pv = pvs + par * C * kTriW * 4;
    double* sc = scl + par * 4;
    const int lr0 = (r0 - rank + C - 1) / C;  // first local row with r >= r0
    const bool owner0 = r0 % C == rank;
    const int nblk = (n - r0 + 31) >> 5;      // <= 8
    const int G = min(gmax, (kTriW - 1) / nblk);  // warps per 32-column block
    const int nsw = nblk * G;                 // summing warps (< kTriW: the last one is free)
    // S: unscaled column sums (warps < nsw), reflector scalars (last warp)
    if (warp < nsw) {
      const int blk = warp % nblk, g = warp / nblk;
      const int r = r0 + 32 * blk + lane;
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (r < n) {
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        int lr = lr0 + (owner0 ? 1 : 0) + g;  // rows c > r0, every G-th
        for (; lr + 3 * G < my_rows; lr += 4 * G) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            a4[u] = fma(A[static_cast<i64>(lr + u * G) * n + r], col[(lr + u * G) * C + rank], a4[u]);
        }
        for (; lr < my_rows; lr += G) a4[0] = fma(A[static_cast<i64>(lr) * n + r], col[lr * C + rank], a4[0]);
        const double ac = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        STG_TRI_MARK(6);
        for (int q = 0; q < C; ++q) tri_peer<C>(acc + static_cast<i64>(rank * G + g) * n, q)[r] = ac;
        if (r == r0) {
          s3 = ac;
        } else {
          s2 = ac * col[r];
        }
        if (owner0 && g == 0) {
          const double x = A[static_cast<i64>(lr0) * n + r];  // row r0
          for (int q = 0; q < C; ++q) tri_peer<C>(a0, q)[r] = x;
          if (r != r0) s1 = x * col[r];
        }
      }
      STG_TRI_MARK(7);
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      s3 = warp_sum(s3);
      if (lane < C) {
        double* d = tri_peer<C>(pv, lane) + (rank * kTriW + warp) * 4;
        d[0] = s1;
        d[1] = s2;
        d[2] = s3;
      }
    } else if (C == 1 && warp == kTriW - 1) {
      const double sigma = warp_sum(lane < C * kTriW ? pv[lane * 4 + 3] : 0.0);
      const double alpha = sc[3];
      double t = 0.0, scal = 0.0, beta = alpha;
      if (sigma > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
        t = (beta - alpha) * __drcp_rn(beta);  // reciprocals: the column's latency chain
        scal = __drcp_rn(alpha - beta);
      }
      if (lane == 0) {
        sc[0] = t;
        sc[1] = scal;
        sc[2] = beta;
        if (rank == 0) {
          b.tau[i] = t;
          b.e[i] = beta;
          b.e2[i] = beta * beta;
        }
      }
      if (rank == 0)
        for (int c = r0 + lane; c < n; c += 32) b.V[static_cast<i64>(i) * n + c] = c == r0 ? 1.0 : col[c] * scal;
      if (i % C == rank && lane == 0) b.d[i] = A[static_cast<i64>(i / C) * n + i];
    }
    STG_TRI_MARK(1);
    tri_sync<C>();
    STG_TRI_MARK(2);
    // U
    double t, scal;
    if constexpr (C == 1) {
      t = sc[0];
      scal = sc[1];
    } else {  // the cluster meets once per column: every warp derives the reflector here
      const double sigma = warp_sum(lane < C * kTriW ? pv[lane * 4 + 3] : 0.0);
      const double alpha = sc[3];
      double beta = alpha;
      t = 0.0;
      scal = 0.0;
      if (sigma > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
        t = (beta - alpha) * __drcp_rn(beta);
        scal = __drcp_rn(alpha - beta);
      }
      if (rank == 0) {
        if (tid == 0) {
          b.tau[i] = t;
          b.e[i] = beta;
          b.e2[i] = beta * beta;
        }
        for (int c = r0 + tid; c < n; c += kTriThreads) b.V[static_cast<i64>(i) * n + c] = c == r0 ? 1.0 : col[c] * scal;
      }
      if (i % C == rank && tid == 0) b.d[i] = A[static_cast<i64>(i / C) * n + i];
    }
    if (t != 0.0) {
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (lane < C * kTriW && (lane % kTriW) < nsw) {
        s1 = pv[lane * 4 + 0];
        s2 = pv[lane * 4 + 1];
        s3 = pv[lane * 4 + 2];
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      s3 = warp_sum(s3);
      const double avv = a0[r0] + scal * (s3 + s1) + scal * scal * s2;  // (Av)'v
      const double b2 = t * t * avv;
      const int nacc = C * G;
      for (int r = r0 + tid; r < n; r += kTriThreads) {
        double sa = 0.0;
        for (int q = 0; q < nacc; ++q) sa += acc[q * n + r];
        const double pr = t * fma(scal, sa, a0[r]);
        const double vr = r == r0 ? 1.0 : scal * col[r];
        Pv[r] = pr;
        Vv[r] = vr;
        Wv[r] = pr - b2 * vr;
      }
      __syncthreads();
      switch (nblk) {
        case 1: tri_update_rows<1>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
        case 2: tri_update_rows<2>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
        case 3: tri_update_rows<3>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
        case 4: tri_update_rows<4>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
        case 5: tri_update_rows<5>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
        case 6: tri_update_rows<6>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
        case 7: tri_update_rows<7>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
        default: tri_update_rows<8>(A, n, r0, C, rank, lr0, my_rows, warp, lane, Pv, Vv, Wv); break;
      }
      __syncwarp();
    }
    STG_TRI_MARK(3);
    // publish column i + 1 from the rows this warp owns (lane u: its u-th row)
    double* Pn = colb + npar * n;
    double sg2 = 0.0;
    for (int lb = lr0 + warp; lb < my_rows; lb += 32 * kTriW) {
      const int lr = lb + lane * kTriW;
      if (lr < my_rows) {
        const int rr = lr * C + rank;
        if (rr >= r0 + 1) {
          const double x = A[static_cast<i64>(lr) * n + r0];
          for (int q = 0; q < C; ++q) tri_peer<C>(Pn, q)[rr] = x;
          if (rr >= r0 + 2) sg2 = fma(x, x, sg2);
          if (rr == r0 + 1)
            for (int q = 0; q < C; ++q) tri_peer<C>(scl + npar * 4, q)[3] = x;
        }
      }
    }
    sg2 = warp_sum(sg2);
    if (lane == 0)
      for (int q = 0; q < C; ++q) tri_peer<C>(pvs + npar * C * kTriW * 4, q)[(rank * kTriW + warp) * 4 + 3] = sg2;
    STG_TRI_MARK(4);
    if constexpr (C == 1) {
      __syncthreads();
    } else {  // S of the next column reads only this CTA's rows; a local barrier suffices
      __syncthreads();
    }
    STG_TRI_MARK(5);
  }
  if constexpr (C > 1) tri_sync<C>();  // no CTA leaves while a peer may still write into it
  if ((n - 1) % C == rank && tid == 0) {
    b.d[n - 1] = A[static_cast<i64>((n - 1) / C) * n + (n - 1)];
    b.e[n - 1] = 0.0;
    b.e2[n - 1] = 0.0;
    b.tau[n - 1] = 0.0;
  }
}

// One-CTA tridiagonalization with the rank-2 update fused into the next
// column's sums (n <= kEig1N, full square in shared memory). Reflector i is
// applied lazily: column i + 1 gets it in a short pre-pass (P), and the pass
// that forms column i + 1's sums (F) reads each trailing element, applies
// reflector i (the same fma order as tri_update_rows), writes it back and
// accumulates it into the sums in the same visit — one read-modify-write of
// the trailing square per column instead of a read (sums) plus a read-modify-
// write (update). Warps split the trailing columns into 32-column blocks and
// the rows G ways (as the two-pass kernel's sums); the last warp derives the
// reflector while the others run F. Three barriers per column.
constexpr int kTri1fThreads = 512;  // 16 warps (1024 measured slower: 842 vs 765 us at n = 164)
constexpr int kTri1fW = kTri1fThreads / 32;
inline size_t tridiag1f_smem_bytes(int n, int gmax) {
  return sizeof(double) * (static_cast<size_t>(n) * n + 5 * static_cast<size_t>(n) + static_cast<size_t>(gmax) * n +
                           kTri1fW * 4 + 8);
}
inline int tridiag1f_gmax(int n) {
  int g = 4;
  while (g > 1 && tridiag1f_smem_bytes(n, g) > 232448) --g;
  return g;
}

__global__ void __launch_bounds__(kTri1fThreads) tridiag1f_kernel(const double* M, int ldm, int n, int sym_input,
                                                                int gmax, EigBufs b, int* flags) {
  extern __shared__ double sm[];
  double* A = sm;                                  // n x n
  double* col = A + static_cast<i64>(n) * n;       // [n] column i (rows > i) with every reflector applied
  double* a0 = col + n;                            // [n] row i + 1 (columns >= i + 1) with every reflector applied
  double* Pv = a0 + n;                             // [n] the pending reflector: p
  double* Vv = Pv + n;                             //                            v
  double* Wv = Vv + n;                             //                            w = p - b2 v
  double* acc = Wv + n;                            // [gmax][n] partial column sums
  double* pvs = acc + static_cast<i64>(gmax) * n;  // [kTri1fW][4]: (Av)'v pieces, squared-norm share
  double* scl = pvs + kTri1fW * 4;                   // {tau, scal, beta, alpha}
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (sym_input) {
    for (int r = warp; r < n; r += kTri1fW)
      for (int c = lane; c < n; c += 32) cp_async8(A + static_cast<i64>(r) * n + c, M + static_cast<i64>(r) * ldm + c);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    int bad = 0;
    for (int r = warp; r < n; r += kTri1fW)
      for (int c = lane; c < n; c += 32) bad |= !isfinite(A[static_cast<i64>(r) * n + c]);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, kNonFinite);
  } else {
    for (int r = warp; r < n; r += kTri1fW)
      for (int c = lane; c < n; c += 32) {
        const double x = M[static_cast<i64>(r) * ldm + c];
        const double y = M[static_cast<i64>(c) * ldm + r];
        if (!isfinite(x) || !isfinite(y)) atomicOr(flags, kNonFinite);
        A[static_cast<i64>(r) * n + c] = 0.5 * (x + y);
      }
  }
  for (int r = tid; r < n; r += kTri1fThreads) Pv[r] = Vv[r] = Wv[r] = 0.0;  // no reflector pending
  __syncthreads();
  for (int i = 0; i + 1 < n; ++i) {
    const int r0 = i + 1;
    // P: column i with the pending reflector (rows >= i); its squared norm below r0 and alpha
    {
      const double vi = Vv[i], wi = Wv[i];
      double sg = 0.0;
      for (int c = i + tid; c < n; c += kTri1fThreads) {
        const double x = fma(-Vv[c], wi, fma(-Pv[c], vi, A[static_cast<i64>(c) * n + i]));
        if (c == i) {
          b.d[i] = x;
        } else {
          col[c] = x;
          if (c == r0) scl[3] = x;
          else sg = fma(x, x, sg);
        }
      }
      sg = warp_sum(sg);
      if (lane == 0) pvs[warp * 4 + 3] = sg;
    }
    __syncthreads();
    const int nblk = (n - r0 + 31) >> 5;
    const int G = min(gmax, (kTri1fW - 1) / nblk);
    const int nsw = nblk * G;
    if (warp < nsw) {
      // F: reflector i-1 applied to the trailing square, the sums of column i formed on the way
      const int blk = warp % nblk, g = warp / nblk;
      const int r = r0 + 32 * blk + lane;
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (r < n) {
        const double vr = Vv[r], wr = Wv[r];
        if (g == 0) {  // row r0 -> a0
          double* Ar = A + static_cast<i64>(r0) * n + r;
          const double x = fma(-Vv[r0], wr, fma(-Pv[r0], vr, *Ar));
          *Ar = x;
          a0[r] = x;
          if (r != r0) s1 = x * col[r];
        }
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        int c = r0 + 1 + g;  // rows c > r0, every G-th
        for (; c + 3 * G < n; c += 4 * G) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cu = c + u * G;
            double* Ar = A + static_cast<i64>(cu) * n + r;
            const double x = fma(-Vv[cu], wr, fma(-Pv[cu], vr, *Ar));
            *Ar = x;
            a4[u] = fma(x, col[cu], a4[u]);
          }
        }
        for (; c < n; c += G) {
          double* Ar = A + static_cast<i64>(c) * n + r;
          const double x = fma(-Vv[c], wr, fma(-Pv[c], vr, *Ar));
          *Ar = x;
          a4[0] = fma(x, col[c], a4[0]);
        }
        const double ac = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        acc[static_cast<i64>(g) * n + r] = ac;
        if (r == r0) s3 = ac;
        else s2 = ac * col[r];
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      s3 = warp_sum(s3);
      if (lane == 0) {
        pvs[warp * 4 + 0] = s1;
        pvs[warp * 4 + 1] = s2;
        pvs[warp * 4 + 2] = s3;
      }
    } else if (warp == kTri1fW - 1) {
      // reflector i from column i (beside F)
      const double sigma = warp_sum(lane < kTri1fW ? pvs[lane * 4 + 3] : 0.0);
      const double alpha = scl[3];
      double t = 0.0, scal = 0.0, beta = alpha;
      if (sigma > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
        t = (beta - alpha) * __drcp_rn(beta);
        scal = __drcp_rn(alpha - beta);
      }
      if (lane == 0) {
        scl[0] = t;
        scl[1] = scal;
        scl[2] = beta;
        b.tau[i] = t;
        b.e[i] = beta;
        b.e2[i] = beta * beta;
      }
      for (int c = r0 + lane; c < n; c += 32) b.V[static_cast<i64>(i) * n + c] = c == r0 ? 1.0 : col[c] * scal;
    }
    __syncthreads();
    // the pending reflector becomes reflector i
    {
      const double t = scl[0], scal = scl[1];
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (lane < nsw) {
        s1 = pvs[lane * 4 + 0];
        s2 = pvs[lane * 4 + 1];
        s3 = pvs[lane * 4 + 2];
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      s3 = warp_sum(s3);
      const double avv = a0[r0] + scal * (s3 + s1) + scal * scal * s2;  // (Av)'v
      const double b2 = t * t * avv;
      for (int r = r0 + tid; r < n; r += kTri1fThreads) {
        if (t == 0.0) {
          Pv[r] = Vv[r] = Wv[r] = 0.0;
          continue;
        }
        double sa = 0.0;
        for (int q = 0; q < G; ++q) sa += acc[static_cast<i64>(q) * n + r];
        const double pr = t * fma(scal, sa, a0[r]);
        const double vr = r == r0 ? 1.0 : scal * col[r];
        Pv[r] = pr;
        Vv[r] = vr;
        Wv[r] = pr - b2 * vr;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    const int l = n - 1;
    b.d[l] = fma(-Vv[l], Wv[l], fma(-Pv[l], Vv[l], A[static_cast<i64>(l) * n + l]));
    b.e[l] = 0.0;
    b.e2[l] = 0.0;
    b.tau[l] = 0.0;
  }
}

__global__ void __launch_bounds__(kTriThreads) tridiag1_kernel(const double* M, int ldm, int n, int sym_input,
                                                               int gmax, EigBufs b, int* flags) {
  tridiag_body<1>(M, ldm, n, sym_input, gmax, b, flags, 0);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTriThreads)
    tridiag2_kernel(const double* M, int ldm, int n, int sym_input, int gmax, EigBufs b, int* flags) {
  tridiag_body<2>(M, ldm, n, sym_input, gmax, b, flags,
                  static_cast<int>(cooperative_groups::this_cluster().block_rank()));
}

// All eigenvalues of the tridiagonal matrix by bisection on Sturm counts:
// a warp per eigenvalue multisects (33-way split per step) until the bracket
// is below max(2 eps |lambda|, eps ||T||), the absolute accuracy of QR-based
// solvers; the returned value is the bracket's lower end (count <= j).
constexpr int kBisG = 32;  // one warp per eigenvalue: a 33-way split per Sturm round
// The Sturm chains are FP64 latency-bound and lose most of their issue slots
// to co-resident DMMA CTAs when the sketch's solve overlaps the basis work on
// the side stream (706 vs ~130 us measured at D = 200). Each CTA therefore
// reserves more shared memory than an SM keeps free beside any Gram/NN CTA
// (>= 70 KB each), so it only lands on an SM of its own.
constexpr int kBisThreads = 256;
constexpr size_t kBisSmem = 164 * 1024;
static_assert(kBisSmem >= sizeof(double) * 2 * kEigMaxN, "d and e2 fit");
__global__ void __launch_bounds__(kBisThreads) bisect_kernel(EigBufs b, int n) {
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
  extern __shared__ double shl[];  // lam[n], then int chosen[n], sel[n], start[n]
  double* lam = shl;
  int* chosen = reinterpret_cast<int*>(lam + n);
  int* sel = chosen + n;
  int* start = sel + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) lam[i] = b.lam[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rank = 0;
    const double vi = lam[i];
    for (int jj = 0; jj < n; ++jj)
      if (jj != i && spectral_before(lam[jj], jj, vi, i, order)) ++rank;
    b.perm[rank] = i;
    w_sorted[rank] = vi;
    chosen[i] = rank < want ? 1 : 0;
  }
  __syncthreads();
  // selected indices in ascending order (prefix counts; n is small)
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!chosen[i]) continue;
    int pos = 0;
    for (int jj = 0; jj < i; ++jj) pos += chosen[jj];
    sel[pos] = i;
  }
  __syncthreads();
  const int m = min(want, n);
  const double tol = ortol * *b.tnorm;
  for (int q = threadIdx.x; q < m; q += blockDim.x) {
    b.sel[q] = sel[q];
    start[q] = (q == 0 || lam[sel[q]] - lam[sel[q - 1]] > tol) ? 1 : 0;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < m; q += blockDim.x) {
    if (!start[q]) continue;
    int c = 0;
    for (int jj = 0; jj < q; ++jj) c += start[jj];
    b.cstart[c] = q;
  }
  if (threadIdx.x == 0) {
    int ncl = 0;
    for (int q = 0; q < m; ++q) ncl += start[q];
    b.cstart[ncl] = m;
    *b.ncl = ncl;
  }
}

// Inverse iteration (dlagtf/dlagts with partial pivoting, kInvitSweeps) for each
// selected eigenvalue; one thread owns one cluster and re-orthogonalizes its
// members in order. Working vectors live in shared memory (8 threads / CTA).
constexpr int kInvitThreads = 8;
// Sweeps of inverse iteration: with the eigenvalue accurate to eps ||T|| one
// solve from a generic start already amplifies the wanted direction by
// ~1 / (eps ||T||); the second refines it (dstein stops after two more).
constexpr int kInvitSweeps = 2;
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
        const double mlt = cur_d != 0.0 ? sub_e * __drcp_rn(cur_d) : 0.0;
        dl[i] = mlt;
        dd[i] = cur_d;
        du[i] = cur_u;
        du2[i] = 0.0;
        cur_d = nd - mlt * cur_u;
        cur_u = nu;
      } else {
        const double mlt = cur_d * __drcp_rn(sub_e);
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
    for (int i = 0; i < n; ++i) {  // store 1 / pivot: the three solves multiply
      if (fabs(dd[i]) < eps_piv) dd[i] = dd[i] < 0.0 ? -eps_piv : eps_piv;
      dd[i] = __drcp_rn(dd[i]);
    }
    for (int i = 0; i < n; ++i) x[i] = 1.0 + 0.5 * __sinf(1.0f + 0.7f * i + 1.3f * q);
    for (int it = 0; it < kInvitSweeps; ++it) {
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
        const double xi = (x[i] - du[i] * x1 - du2[i] * x2) * dd[i];
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
// memory kBtRows at a time. Rows of V are contiguous in global memory, so a
// block of reflectors is one contiguous range: it is copied with cp.async
// (all requests in flight at once) into a double buffer while the previous
// block is applied; entries at or left of the unit diagonal are masked on use.
// Column c of F = the c-th leading eigenvector.
constexpr int kBtRows = 16;
__global__ void __launch_bounds__(128) backtransform_kernel(EigBufs b, int n, int want, double* F, int ldf) {
  extern __shared__ double vs[];  // [2][kBtRows x n]
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
  auto stage = [&](int top, int buf) {  // rows max(0, top - kBtRows + 1) .. top
    const int lo = max(0, top - kBtRows + 1);
    const double* src = b.V + static_cast<i64>(lo) * n;
    double* dst = vs + buf * kBtRows * n;
    const int cnt = (top - lo + 1) * n;
    for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) cp_async8(dst + idx, src + idx);
    cp_async_commit();
  };
  int buf = 0;
  if (n >= 2) stage(n - 2, 0);
  for (int top = n - 2; top >= 0; top -= kBtRows) {
    const int lo = max(0, top - kBtRows + 1);
    if (lo > 0) {
      stage(lo - 1, buf ^ 1);  // next block in flight while this one is applied
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const double* blk = vs + buf * kBtRows * n;
      for (int i = top; i >= lo; --i) {
        const double ti = b.tau[i];
        if (ti == 0.0) continue;
        const double* vrow = blk + (i - lo) * n;
        double vr[kSlots];
        double s = 0.0;
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) {
          const int r = lane + 32 * sl;
          vr[sl] = r > i + 1 && r < n ? vrow[r] : (r == i + 1 ? 1.0 : 0.0);
          s += vr[sl] * xr[sl];
        }
        s = warp_sum(s) * ti;
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) xr[sl] -= s * vr[sl];
      }
    }
    __syncthreads();  // the buffer is restaged two blocks later
    buf ^= 1;
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

inline void eig_set_attributes() {
  STG_CUDA(cudaFuncSetAttribute(tridiag1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                232448));
  STG_CUDA(cudaFuncSetAttribute(tridiag2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                232448));
  STG_CUDA(cudaFuncSetAttribute(tridiag1f_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                232448));
  STG_CUDA(cudaFuncSetAttribute(backtransform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double) * 2 * kBtRows * kEigMaxN)));
  STG_CUDA(cudaFuncSetAttribute(invit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(invit_smem_bytes(kEigMaxN))));
  STG_CUDA(cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kBisSmem)));
}

template <class Launch>
void syev_launch(Launch&& L, const double* M, int ldm, int n, int sym_input, int order, int want, double ortol,
                 double* w_sorted,
                 double* F, int ldf, double* dbuf, int* ibuf, int* flags) {
  const EigBufs b = eig_carve(dbuf, ibuf, n, want);
  static const int one_cta_max = getenv("STG_EIG1N") ? atoi(getenv("STG_EIG1N")) : kEig1N;  // development A/B
  static const bool two_pass = getenv("STG_TRI_TWOPASS") && atoi(getenv("STG_TRI_TWOPASS")) != 0;  // development A/B
  if (n <= one_cta_max && !two_pass) {
    const int g = tridiag1f_gmax(n);
    L(tridiag1f_kernel, dim3(1), dim3(kTri1fThreads), tridiag1f_smem_bytes(n, g), M, ldm, n, sym_input, g, b, flags);
  } else if (n <= one_cta_max) {
    const int g = tridiag_gmax(n, 1);
    L(tridiag1_kernel, dim3(1), dim3(kTriThreads), tridiag_smem_bytes(n, 1, g), M, ldm, n, sym_input, g, b, flags);
  } else {
    const int g = tridiag_gmax(n, 2);
    L(tridiag2_kernel, dim3(2), dim3(kTriThreads), tridiag_smem_bytes(n, 2, g), M, ldm, n, sym_input, g, b, flags);
  }
  static const bool bis_shared = !getenv("STG_BIS_NOISOLATE");  // development A/B
  L(bisect_kernel, dim3(static_cast<unsigned>(cdiv(kBisG * n, kBisThreads))), dim3(kBisThreads),
    bis_shared ? kBisSmem : sizeof(double) * 2 * n, b, n);
  L(select_kernel, dim3(1), dim3(256), (sizeof(double) + 3 * sizeof(int)) * n, b, n, order, want, ortol, w_sorted);
  L(invit_kernel, dim3(static_cast<unsigned>(cdiv(want, kInvitThreads))), dim3(kInvitThreads), invit_smem_bytes(n), b,
    n);
  L(backtransform_kernel, dim3(static_cast<unsigned>(cdiv(want, 4))), dim3(128), sizeof(double) * 2 * kBtRows * n, b,
    n, want, F, ldf);
}

}  // namespace stg
