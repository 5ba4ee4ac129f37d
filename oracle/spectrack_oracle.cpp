// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference G-REST hot path.
// See spectrack_oracle.hpp for scope. Compiled -O3 -ffp-contract=off like the
// reference's CMake Release build (no -march, so no FMA contraction), with
// optional OpenMP used only for embarrassingly parallel loops whose per-element
// arithmetic order is unchanged (row-wise sparse products) or for reductions
// whose order is fixed by the thread count (dense dot products).
#include "spectrack_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <set>
#include <sstream>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace spectrack_oracle {

namespace {

int nthreads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

bool all_finite(const Mat& m) {
  for (double v : m.a)
    if (!std::isfinite(v)) return false;
  return true;
}

double norm2(const double* v, Index n) {
  double s = 0.0;
  for (Index i = 0; i < n; ++i) s += v[i] * v[i];
  return std::sqrt(s);
}

// t = Q(:, :r)' v ; v -= Q(:, :r) t   (the GEMV pair of ortho.hpp:31-32)
void project_out(const Mat& q, Index r, std::vector<double>& v) {
  if (r == 0) return;
  const Index n = q.rows;
  const int T = n > 65536 ? nthreads() : 1;
  std::vector<double> part(static_cast<size_t>(T) * r, 0.0);
  const Index chunk = (n + T - 1) / T;
#pragma omp parallel for num_threads(T) schedule(static, 1) if (T > 1)
  for (int t = 0; t < T; ++t) {
    const Index lo = t * chunk, hi = std::min(n, lo + chunk);
    for (Index l = 0; l < r; ++l) {
      const double* ql = q.col(l);
      double s = 0.0;
      for (Index i = lo; i < hi; ++i) s += ql[i] * v[static_cast<size_t>(i)];
      part[static_cast<size_t>(t) * r + l] = s;
    }
  }
  std::vector<double> coef(static_cast<size_t>(r), 0.0);
  for (int t = 0; t < T; ++t)
    for (Index l = 0; l < r; ++l) coef[l] += part[static_cast<size_t>(t) * r + l];
#pragma omp parallel for num_threads(T) schedule(static, 1) if (T > 1)
  for (int t = 0; t < T; ++t) {
    const Index lo = t * chunk, hi = std::min(n, lo + chunk);
    for (Index l = 0; l < r; ++l) {
      const double* ql = q.col(l);
      const double c = coef[l];
      for (Index i = lo; i < hi; ++i) v[static_cast<size_t>(i)] -= ql[i] * c;
    }
  }
}

}  // namespace

// ---------------------------------------------------------------- dense helpers
Mat transpose(const Mat& m) {
  Mat t(m.cols, m.rows);
  for (Index j = 0; j < m.cols; ++j)
    for (Index i = 0; i < m.rows; ++i) t(j, i) = m(i, j);
  return t;
}

// Dense products on tall column-major blocks, blocked by rows so each row
// block of the operands is read from memory once (per-element sums keep a
// fixed order for a fixed thread count).
Mat matmul(const Mat& a, const Mat& b) {
  if (a.cols != b.rows) throw std::invalid_argument("matmul: shape mismatch");
  Mat c(a.rows, b.cols);
  const Index n = a.rows;
  constexpr Index RB = 512;
  const Index nblk = (n + RB - 1) / RB;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (Index blk = 0; blk < nblk; ++blk) {
    const Index lo = blk * RB, hi = std::min(n, lo + RB);
    for (Index j = 0; j < b.cols; ++j) {
      double* cj = c.col(j);
      for (Index l = 0; l < a.cols; ++l) {
        const double blj = b(l, j);
        if (blj == 0.0) continue;
        const double* al = a.col(l);
        for (Index i = lo; i < hi; ++i) cj[i] += al[i] * blj;
      }
    }
  }
  return c;
}

Mat matmul_tn(const Mat& a, const Mat& b) {
  if (a.rows != b.rows) throw std::invalid_argument("matmul_tn: shape mismatch");
  const Index n = a.rows;
  const int T = n > 65536 ? nthreads() : 1;
  const Index chunk = (n + T - 1) / T;
  constexpr Index RB = 256;
  std::vector<Mat> part(static_cast<size_t>(T), Mat(a.cols, b.cols));
#pragma omp parallel for num_threads(T) schedule(static, 1) if (T > 1)
  for (int t = 0; t < T; ++t) {
    const Index lo0 = t * chunk, hi0 = std::min(n, lo0 + chunk);
    Mat& p = part[static_cast<size_t>(t)];
    for (Index lo = lo0; lo < hi0; lo += RB) {
      const Index hi = std::min(hi0, lo + RB);
      for (Index j = 0; j < b.cols; ++j) {
        const double* bj = b.col(j);
        for (Index i = 0; i < a.cols; ++i) {
          const double* ai = a.col(i);
          double s = 0.0;
          for (Index r = lo; r < hi; ++r) s += ai[r] * bj[r];
          p(i, j) += s;
        }
      }
    }
  }
  Mat c(a.cols, b.cols);
  for (int t = 0; t < T; ++t)
    for (size_t e = 0; e < c.a.size(); ++e) c.a[e] += part[static_cast<size_t>(t)].a[e];
  return c;
}

Mat left_cols(const Mat& m, Index c) {
  Mat out(m.rows, c);
  std::copy(m.a.begin(), m.a.begin() + m.rows * c, out.a.begin());
  return out;
}

// ---------------------------------------------------------------- ordering / eig
std::vector<Index> spectral_sort(const Vec& values, SpectralOrder order) {
  // types.hpp:26-40
  std::vector<Index> perm(values.size());
  std::iota(perm.begin(), perm.end(), Index{0});
  std::sort(perm.begin(), perm.end(), [&](Index a, Index b) {
    if (order == SpectralOrder::abs_desc) {
      const double aa = values[a] < 0.0 ? -values[a] : values[a];
      const double ab = values[b] < 0.0 ? -values[b] : values[b];
      if (aa != ab) return aa > ab;
    }
    if (values[a] != values[b]) return values[a] > values[b];
    return a < b;
  });
  return perm;
}

EigResult reorder_eig(const Vec& values, const Mat& vectors, SpectralOrder order) {
  // eig.hpp:20-32
  const std::vector<Index> perm = spectral_sort(values, order);
  EigResult out;
  out.values.resize(values.size());
  out.vectors = Mat(vectors.rows, vectors.cols);
  for (size_t i = 0; i < values.size(); ++i) {
    out.values[i] = values[static_cast<size_t>(perm[i])];
    std::copy(vectors.col(perm[i]), vectors.col(perm[i]) + vectors.rows,
              out.vectors.col(static_cast<Index>(i)));
  }
  return out;
}

namespace {

// Cyclic two-sided Jacobi for a dense symmetric matrix (stand-in for Eigen's
// SelfAdjointEigenSolver; both are backward stable, so eigenvalues agree to
// O(eps * ||S||)). Returns eigenvalues ascending like Eigen.
void jacobi_eig(Mat a, Vec& w, Mat& v) {
  const Index n = a.rows;
  v = Mat::identity(n);
  double fro = 0.0;
  for (double x : a.a) fro += x * x;
  const double tiny = std::numeric_limits<double>::min();
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < j; ++i) off += a(i, j) * a(i, j);
    if (off <= 1e-34 * fro || off <= tiny) break;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (std::abs(apq) <= tiny) continue;
        const double app = a(p, p), aqq = a(q, q);
        if (sweep > 3 && std::abs(apq) < 1e-18 * std::sqrt(std::abs(app * aqq))) {
          a(p, q) = a(q, p) = 0.0;
          continue;
        }
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (Index k = 0; k < n; ++k) {  // columns p, q
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (Index k = 0; k < n; ++k) {  // rows p, q
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (Index k = 0; k < n; ++k) {
          const double vkp = v(k, p), vkq = v(k, q);
          v(k, p) = c * vkp - s * vkq;
          v(k, q) = s * vkp + c * vkq;
        }
      }
  }
  std::vector<Index> idx(static_cast<size_t>(n));
  std::iota(idx.begin(), idx.end(), Index{0});
  std::stable_sort(idx.begin(), idx.end(), [&](Index x, Index y) { return a(x, x) < a(y, y); });
  w.resize(static_cast<size_t>(n));
  Mat vs(n, n);
  for (Index i = 0; i < n; ++i) {
    w[static_cast<size_t>(i)] = a(idx[i], idx[i]);
    std::copy(v.col(idx[i]), v.col(idx[i]) + n, vs.col(i));
  }
  v = std::move(vs);
}

}  // namespace

EigResult sym_eig_dense(const Mat& s, SpectralOrder order) {
  // eig.hpp:37-50
  if (s.rows != s.cols) throw std::invalid_argument("sym_eig_dense: matrix must be square");
  if (!all_finite(s)) throw std::invalid_argument("sym_eig_dense: non-finite entries");
  if (s.rows == 0) return {};
  Mat sym(s.rows, s.cols);
  for (Index j = 0; j < s.cols; ++j)
    for (Index i = 0; i < s.rows; ++i) sym(i, j) = 0.5 * (s(i, j) + s(j, i));
  Vec w;
  Mat v;
  jacobi_eig(sym, w, v);
  return reorder_eig(w, v, order);
}

// ---------------------------------------------------------------- ortho
Mat orthonormalize(const Mat& m, const Mat& against, double drop_tol) {
  // ortho.hpp:13-39
  if (against.cols > 0 && against.rows != m.rows)
    throw std::invalid_argument("orthonormalize: row count mismatch with `against`");
  if (!all_finite(m) || !all_finite(against))
    throw std::invalid_argument("orthonormalize: non-finite entries");
  Mat q(m.rows, m.cols);
  Index r = 0;
  std::vector<double> v(static_cast<size_t>(m.rows));
  for (Index c = 0; c < m.cols; ++c) {
    std::copy(m.col(c), m.col(c) + m.rows, v.begin());
    const double orig = norm2(v.data(), m.rows);
    if (orig == 0.0) continue;
    for (int pass = 0; pass < 2; ++pass) {
      if (against.cols > 0) project_out(against, against.cols, v);
      if (r > 0) project_out(q, r, v);
    }
    const double nrm = norm2(v.data(), m.rows);
    if (nrm < drop_tol * orig) continue;
    double* qc = q.col(r++);
    for (Index i = 0; i < m.rows; ++i) qc[i] = v[static_cast<size_t>(i)] / nrm;
  }
  return left_cols(q, r);
}

Mat orthonormalize(const Mat& m, double drop_tol) { return orthonormalize(m, Mat(m.rows, 0), drop_tol); }

// ---------------------------------------------------------------- rng
std::uint64_t mix_seed(std::uint64_t base, std::uint64_t salt) {
  // rng.hpp:16-21
  std::uint64_t z = base + 0x9e3779b97f4a7c15ULL * (salt + 0x632be59bd9b4e019ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

std::uint64_t mix_seed(std::uint64_t base, std::uint64_t a, std::uint64_t b) {
  return mix_seed(mix_seed(base, a), b);
}

double GaussianSampler::operator()() {
  // rng.hpp:44-56: Box-Muller, cos first, sin cached
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  constexpr double two_pi = 6.283185307179586476925286766559;
  spare_ = r * std::sin(two_pi * u2);
  has_spare_ = true;
  return r * std::cos(two_pi * u2);
}

Vec GaussianSampler::gaussian_vector(Index n) {
  Vec v(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) v[static_cast<size_t>(i)] = (*this)();
  return v;
}

Mat GaussianSampler::gaussian_matrix(Index rows, Index cols) {
  // rng.hpp:64-69: column-major fill
  Mat m(rows, cols);
  for (Index c = 0; c < cols; ++c)
    for (Index r = 0; r < rows; ++r) m(r, c) = (*this)();
  return m;
}

// ---------------------------------------------------------------- svd
namespace {

// One-sided (Hestenes) Jacobi on the columns of a (m x n): a V = W diag(sv).
// Returns V and sv (unsorted).
void one_sided_jacobi(Mat a, Vec& sv, Mat& v) {
  const Index m = a.rows, n = a.cols;
  v = Mat::identity(n);
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        const double* ap = a.col(p);
        const double* aq = a.col(q);
        for (Index i = 0; i < m; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || std::abs(gamma) <= 1e-16 * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        double* wp = a.col(p);
        double* wq = a.col(q);
        for (Index i = 0; i < m; ++i) {
          const double x = wp[i], y = wq[i];
          wp[i] = c * x - s * y;
          wq[i] = s * x + c * y;
        }
        double* vp = v.col(p);
        double* vq = v.col(q);
        for (Index i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - s * y;
          vq[i] = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
  sv.assign(static_cast<size_t>(n), 0.0);
  for (Index j = 0; j < n; ++j) sv[static_cast<size_t>(j)] = norm2(a.col(j), m);
}

// Householder QR of a tall matrix (m >= n): returns the n x n R factor.
Mat householder_r(Mat a) {
  const Index m = a.rows, n = a.cols;
  for (Index j = 0; j < n && j < m; ++j) {
    double* aj = a.col(j);
    double nrm = 0.0;
    for (Index i = j; i < m; ++i) nrm += aj[i] * aj[i];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = aj[j] > 0 ? -nrm : nrm;
    std::vector<double> u(static_cast<size_t>(m - j));
    for (Index i = j; i < m; ++i) u[static_cast<size_t>(i - j)] = aj[i];
    u[0] -= alpha;
    double unrm2 = 0.0;
    for (double x : u) unrm2 += x * x;
    if (unrm2 == 0.0) continue;
    for (Index c = j; c < n; ++c) {
      double* ac = a.col(c);
      double d = 0.0;
      for (Index i = j; i < m; ++i) d += u[static_cast<size_t>(i - j)] * ac[i];
      const double f = 2.0 * d / unrm2;
      for (Index i = j; i < m; ++i) ac[i] -= f * u[static_cast<size_t>(i - j)];
    }
  }
  Mat r(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i <= j && i < m; ++i) r(i, j) = a(i, j);
  return r;
}

}  // namespace

void thin_svd_u(const Mat& m, Vec& sv, Mat& u) {
  // Stand-in for Eigen::JacobiSVD(m, ComputeThinU) (rsvd.hpp:58): for a wide
  // m (rows <= cols) Eigen QR-preconditions on m' and runs Jacobi on the
  // square factor; here m' = QR, and the left singular vectors of m are the
  // right singular vectors of R, obtained by one-sided Jacobi on R.
  Vec s;
  Mat v;
  if (m.rows <= m.cols) {
    const Mat r = householder_r(transpose(m));  // rows x rows
    one_sided_jacobi(r, s, v);                 // r v = w diag(s)  => u = v
  } else {
    one_sided_jacobi(m, s, v);  // m v = u diag(s)
    Mat mv = matmul(m, v);
    for (Index j = 0; j < mv.cols; ++j)
      for (Index i = 0; i < mv.rows; ++i) mv(i, j) = s[static_cast<size_t>(j)] > 0 ? mv(i, j) / s[static_cast<size_t>(j)] : 0.0;
    v = mv;
  }
  std::vector<Index> idx(s.size());
  std::iota(idx.begin(), idx.end(), Index{0});
  std::stable_sort(idx.begin(), idx.end(), [&](Index a, Index b) { return s[a] > s[b]; });
  sv.resize(s.size());
  u = Mat(v.rows, static_cast<Index>(s.size()));
  for (size_t i = 0; i < s.size(); ++i) {
    sv[i] = s[static_cast<size_t>(idx[i])];
    std::copy(v.col(idx[i]), v.col(idx[i]) + v.rows, u.col(static_cast<Index>(i)));
  }
}

Mat rsvd_basis(const RectOperator& op, Index target_rank, Index oversample, std::uint64_t seed) {
  // rsvd.hpp:34-66
  if (target_rank < 1) throw std::invalid_argument("rsvd_basis: target rank must be positive");
  if (oversample < 0) throw std::invalid_argument("rsvd_basis: negative oversampling");
  if (op.rows <= 0 || op.cols <= 0 || !op.apply || !op.apply_adjoint)
    throw std::invalid_argument("rsvd_basis: operator not fully specified");
  const Index draw = std::min(op.cols, target_rank + oversample);
  GaussianSampler rng(mix_seed(seed, 0x5bdU));
  const Mat omega = rng.gaussian_matrix(op.cols, draw);
  const Mat y = op.apply(omega);
  if (y.rows != op.rows || y.cols != draw) throw std::invalid_argument("rsvd_basis: apply returned wrong shape");
  const Mat m = orthonormalize(y);
  if (m.cols == 0) return Mat(op.rows, 0);
  const Mat bt_m = op.apply_adjoint(m);
  if (bt_m.rows != op.cols || bt_m.cols != m.cols)
    throw std::invalid_argument("rsvd_basis: apply_adjoint returned wrong shape");
  const Mat mtb = transpose(bt_m);
  Vec sv;
  Mat u;
  thin_svd_u(mtb, sv, u);
  const double cutoff = !sv.empty() ? 1e-10 * sv[0] : 0.0;
  Index rank = 0;
  while (rank < static_cast<Index>(sv.size()) && sv[static_cast<size_t>(rank)] > cutoff &&
         sv[static_cast<size_t>(rank)] > 0.0)
    ++rank;
  const Index keep = std::min(target_rank, rank);
  if (keep == 0) return Mat(op.rows, 0);
  return matmul(m, left_cols(u, keep));
}

RectOperator dense_operator(const Mat& b) {
  RectOperator op;
  op.rows = b.rows;
  op.cols = b.cols;
  op.apply = [b](const Mat& x) { return matmul(b, x); };
  op.apply_adjoint = [b](const Mat& x) { return matmul_tn(b, x); };
  return op;
}

// ---------------------------------------------------------------- sparse
double Csr::coeff(Index i, Index j) const {
  const auto b = colidx.begin() + rowptr[static_cast<size_t>(i)];
  const auto e = colidx.begin() + rowptr[static_cast<size_t>(i) + 1];
  const auto it = std::lower_bound(b, e, static_cast<std::int32_t>(j));
  if (it != e && *it == j) return val[static_cast<size_t>(it - colidx.begin())];
  return 0.0;
}

double Csr::frobenius_norm() const {
  double s = 0.0;
  for (double v : val) s += v * v;
  return std::sqrt(s);
}

Csr csr_from_triplets_raw(Index rows, Index cols, const std::vector<Triplet>& t) {
  // Eigen setFromTriplets: duplicates summed in input order, columns sorted.
  std::vector<size_t> idx(t.size());
  std::iota(idx.begin(), idx.end(), size_t{0});
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    if (t[a].row != t[b].row) return t[a].row < t[b].row;
    return t[a].col < t[b].col;
  });
  Csr m;
  m.rows = rows;
  m.cols = cols;
  m.rowptr.assign(static_cast<size_t>(rows) + 1, 0);
  for (size_t e = 0; e < idx.size();) {
    const Triplet& first = t[idx[e]];
    if (first.row < 0 || first.row >= rows || first.col < 0 || first.col >= cols)
      throw std::invalid_argument("setFromTriplets: index out of range");
    double v = first.value;
    size_t f = e + 1;
    while (f < idx.size() && t[idx[f]].row == first.row && t[idx[f]].col == first.col) v += t[idx[f++]].value;
    m.colidx.push_back(static_cast<std::int32_t>(first.col));
    m.val.push_back(v);
    m.rowptr[static_cast<size_t>(first.row) + 1]++;
    e = f;
  }
  for (Index r = 0; r < rows; ++r) m.rowptr[static_cast<size_t>(r) + 1] += m.rowptr[static_cast<size_t>(r)];
  return m;
}

void prune_zeros(Csr& m) {
  // sparse.cpp:10-13
  Csr out;
  out.rows = m.rows;
  out.cols = m.cols;
  out.rowptr.assign(static_cast<size_t>(m.rows) + 1, 0);
  out.colidx.reserve(m.colidx.size());
  out.val.reserve(m.val.size());
  for (Index r = 0; r < m.rows; ++r) {
    for (std::int32_t e = m.rowptr[static_cast<size_t>(r)]; e < m.rowptr[static_cast<size_t>(r) + 1]; ++e)
      if (m.val[static_cast<size_t>(e)] != 0.0) {
        out.colidx.push_back(m.colidx[static_cast<size_t>(e)]);
        out.val.push_back(m.val[static_cast<size_t>(e)]);
      }
    out.rowptr[static_cast<size_t>(r) + 1] = static_cast<std::int32_t>(out.val.size());
  }
  m = std::move(out);
}

bool is_symmetric(const Csr& m) {
  // sparse.cpp:65-77: structure and values equal to the transpose, bitwise
  if (m.rows != m.cols) return false;
  std::vector<Triplet> t;
  t.reserve(m.val.size());
  for (Index r = 0; r < m.rows; ++r)
    for (std::int32_t e = m.rowptr[static_cast<size_t>(r)]; e < m.rowptr[static_cast<size_t>(r) + 1]; ++e)
      t.push_back({m.colidx[static_cast<size_t>(e)], r, m.val[static_cast<size_t>(e)]});
  const Csr tr = csr_from_triplets_raw(m.rows, m.cols, t);
  return tr.rowptr == m.rowptr && tr.colidx == m.colidx && tr.val == m.val;
}

Csr wrap(Csr m, bool validate) {
  // sparse.cpp:55-63
  if (m.rows != m.cols) throw std::invalid_argument("SymSparseMatrix: matrix must be square");
  prune_zeros(m);
  if (validate && !is_symmetric(m)) throw std::invalid_argument("SymSparseMatrix: matrix is not symmetric");
  return m;
}

Csr from_triplets(Index n, const std::vector<Triplet>& t) {
  // sparse.cpp:17-23
  if (n < 0) throw std::invalid_argument("SymSparseMatrix: negative size");
  return wrap(csr_from_triplets_raw(n, n, t), true);
}

Csr from_edges(Index n, const std::vector<std::tuple<Index, Index, double>>& edges) {
  // sparse.cpp:25-45
  std::vector<Triplet> t;
  t.reserve(2 * edges.size());
  std::set<std::pair<Index, Index>> seen;
  for (const auto& [i, j, w] : edges) {
    if (i < 0 || j < 0 || i >= n || j >= n)
      throw std::invalid_argument("SymSparseMatrix: edge endpoint out of range");
    if (i == j) throw std::invalid_argument("SymSparseMatrix: self-loop rejected");
    if (!seen.insert({std::min(i, j), std::max(i, j)}).second)
      throw std::invalid_argument("SymSparseMatrix: duplicate edge rejected");
    t.push_back({i, j, w});
    t.push_back({j, i, w});
  }
  Csr m = csr_from_triplets_raw(n, n, t);
  prune_zeros(m);
  return m;
}

Vec matvec(const Csr& a, const Vec& x) {
  // sparse.cpp:79-82 (row-major sparse * vector: per-row sum in column order)
  if (static_cast<Index>(x.size()) != a.rows) throw std::invalid_argument("matvec: dimension mismatch");
  Vec y(static_cast<size_t>(a.rows), 0.0);
#pragma omp parallel for schedule(static) if (a.rows > 65536)
  for (Index r = 0; r < a.rows; ++r) {
    double tmp = 0.0;
    for (std::int32_t e = a.rowptr[static_cast<size_t>(r)]; e < a.rowptr[static_cast<size_t>(r) + 1]; ++e)
      tmp += a.val[static_cast<size_t>(e)] * x[static_cast<size_t>(a.colidx[static_cast<size_t>(e)])];
    y[static_cast<size_t>(r)] = tmp;
  }
  return y;
}

Mat matmat(const Csr& a, const Mat& x) {
  // sparse.cpp:84-87 (Eigen row-major sparse * dense: res(i,c) = sum in column order)
  if (x.rows != a.cols) throw std::invalid_argument("matmat: dimension mismatch");
  Mat y(a.rows, x.cols);
  for (Index c = 0; c < x.cols; ++c) {
    const double* xc = x.col(c);
    double* yc = y.col(c);
#pragma omp parallel for schedule(static) if (a.rows > 65536)
    for (Index r = 0; r < a.rows; ++r) {
      double tmp = 0.0;
      for (std::int32_t e = a.rowptr[static_cast<size_t>(r)]; e < a.rowptr[static_cast<size_t>(r) + 1]; ++e)
        tmp += a.val[static_cast<size_t>(e)] * xc[a.colidx[static_cast<size_t>(e)]];
      yc[r] = tmp;
    }
  }
  return y;
}

Csr pad(const Csr& a, Index s) {
  // sparse.cpp:89-95
  if (s < 0) throw std::invalid_argument("pad: negative padding");
  Csr m = a;
  m.rows += s;
  m.cols += s;
  m.rowptr.resize(static_cast<size_t>(m.rows) + 1, a.rowptr.back());
  return m;
}

Vec degrees(const Csr& a) {
  // sparse.cpp:97-99 (A * ones: row sums in column order)
  Vec d(static_cast<size_t>(a.rows), 0.0);
  for (Index r = 0; r < a.rows; ++r) {
    double tmp = 0.0;
    for (std::int32_t e = a.rowptr[static_cast<size_t>(r)]; e < a.rowptr[static_cast<size_t>(r) + 1]; ++e)
      tmp += a.val[static_cast<size_t>(e)] * 1.0;
    d[static_cast<size_t>(r)] = tmp;
  }
  return d;
}

Csr sparse_add(const Csr& a, const Csr& b, double sign_b) {
  // Eigen sparse a + b (sign_b = +1) or a - b (sign_b = -1): union pattern,
  // explicit zeros kept (the callers prune through wrap()).
  if (a.rows != b.rows || a.cols != b.cols) throw std::invalid_argument("sparse_add: shape mismatch");
  Csr m;
  m.rows = a.rows;
  m.cols = a.cols;
  m.rowptr.assign(static_cast<size_t>(a.rows) + 1, 0);
  m.colidx.reserve(a.colidx.size() + b.colidx.size());
  m.val.reserve(a.val.size() + b.val.size());
  for (Index r = 0; r < a.rows; ++r) {
    std::int32_t i = a.rowptr[static_cast<size_t>(r)], ie = a.rowptr[static_cast<size_t>(r) + 1];
    std::int32_t j = b.rowptr[static_cast<size_t>(r)], je = b.rowptr[static_cast<size_t>(r) + 1];
    while (i < ie || j < je) {
      const std::int32_t ci = i < ie ? a.colidx[static_cast<size_t>(i)] : std::numeric_limits<std::int32_t>::max();
      const std::int32_t cj = j < je ? b.colidx[static_cast<size_t>(j)] : std::numeric_limits<std::int32_t>::max();
      double v;
      std::int32_t c;
      if (ci == cj) {
        c = ci;
        v = sign_b > 0 ? a.val[static_cast<size_t>(i)] + b.val[static_cast<size_t>(j)]
                       : a.val[static_cast<size_t>(i)] - b.val[static_cast<size_t>(j)];
        ++i, ++j;
      } else if (ci < cj) {
        c = ci;
        v = sign_b > 0 ? a.val[static_cast<size_t>(i)] + 0.0 : a.val[static_cast<size_t>(i)] - 0.0;
        ++i;
      } else {
        c = cj;
        v = sign_b > 0 ? 0.0 + b.val[static_cast<size_t>(j)] : 0.0 - b.val[static_cast<size_t>(j)];
        ++j;
      }
      m.colidx.push_back(c);
      m.val.push_back(v);
    }
    m.rowptr[static_cast<size_t>(r) + 1] = static_cast<std::int32_t>(m.val.size());
  }
  return m;
}

Mat to_dense(const Csr& a) {
  Mat d(a.rows, a.cols);
  for (Index r = 0; r < a.rows; ++r)
    for (std::int32_t e = a.rowptr[static_cast<size_t>(r)]; e < a.rowptr[static_cast<size_t>(r) + 1]; ++e)
      d(r, a.colidx[static_cast<size_t>(e)]) = a.val[static_cast<size_t>(e)];
  return d;
}

// ---------------------------------------------------------------- graph
double GraphUpdate::frobenius_norm() const {
  // graph.cpp:10-15
  const double k2 = k_block.frobenius_norm() * k_block.frobenius_norm();
  const double g2 = g_block.frobenius_norm() * g_block.frobenius_norm();
  const double c2 = c_block.frobenius_norm() * c_block.frobenius_norm();
  return std::sqrt(k2 + 2.0 * g2 + c2);
}

Csr GraphUpdate::to_delta() const {
  // graph.cpp:17-32
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(nnz()));
  for (Index r = 0; r < k_block.rows; ++r)
    for (std::int32_t e = k_block.rowptr[static_cast<size_t>(r)]; e < k_block.rowptr[static_cast<size_t>(r) + 1]; ++e)
      t.push_back({r, k_block.colidx[static_cast<size_t>(e)], k_block.val[static_cast<size_t>(e)]});
  for (Index r = 0; r < g_block.rows; ++r)
    for (std::int32_t e = g_block.rowptr[static_cast<size_t>(r)]; e < g_block.rowptr[static_cast<size_t>(r) + 1]; ++e) {
      const Index c = g_block.colidx[static_cast<size_t>(e)];
      t.push_back({r, n_old + c, g_block.val[static_cast<size_t>(e)]});
      t.push_back({n_old + c, r, g_block.val[static_cast<size_t>(e)]});
    }
  for (Index r = 0; r < c_block.rows; ++r)
    for (std::int32_t e = c_block.rowptr[static_cast<size_t>(r)]; e < c_block.rowptr[static_cast<size_t>(r) + 1]; ++e)
      t.push_back({n_old + r, n_old + c_block.colidx[static_cast<size_t>(e)], c_block.val[static_cast<size_t>(e)]});
  return from_triplets(n_old + n_new, t);
}

GraphUpdate make_empty_update(Index n_old, Index n_new) {
  // graph.cpp:34-43
  if (n_old < 0 || n_new < 0) throw std::invalid_argument("make_empty_update: negative size");
  GraphUpdate d;
  d.n_old = n_old;
  d.n_new = n_new;
  d.k_block = csr_from_triplets_raw(n_old, n_old, {});
  d.g_block = csr_from_triplets_raw(n_old, n_new, {});
  d.c_block = csr_from_triplets_raw(n_new, n_new, {});
  return d;
}

GraphUpdate assemble_update(Index n_old, const std::vector<std::tuple<Index, Index, double>>& added_edges,
                            const std::vector<std::pair<Index, Index>>& removed_edges, Index new_node_count,
                            const std::vector<std::tuple<Index, Index, double>>& new_edges) {
  // graph.cpp:45-100
  if (n_old < 0 || new_node_count < 0) throw std::invalid_argument("assemble_update: negative node count");
  const Index n_total = n_old + new_node_count;
  std::set<std::pair<Index, Index>> seen;
  auto note_pair = [&](Index i, Index j) {
    if (i == j) throw std::invalid_argument("assemble_update: self-loop rejected");
    if (!seen.insert({std::min(i, j), std::max(i, j)}).second)
      throw std::invalid_argument("assemble_update: duplicate edge across edit lists");
  };
  std::vector<Triplet> kt, gt, ct;
  auto add_old_pair = [&](Index i, Index j, double w) {
    if (i < 0 || j < 0 || i >= n_old || j >= n_old)
      throw std::invalid_argument("assemble_update: edited edge must address existing nodes");
    note_pair(i, j);
    kt.push_back({i, j, w});
    kt.push_back({j, i, w});
  };
  for (const auto& [i, j, w] : added_edges) {
    if (w == 0.0) throw std::invalid_argument("assemble_update: zero-weight edit");
    add_old_pair(i, j, w);
  }
  for (const auto& [i, j] : removed_edges) add_old_pair(i, j, -1.0);
  for (const auto& [i, j, w] : new_edges) {
    if (i < 0 || j < 0 || i >= n_total || j >= n_total)
      throw std::invalid_argument("assemble_update: new edge endpoint out of range");
    if (w <= 0.0) throw std::invalid_argument("assemble_update: new edges need positive weight");
    note_pair(i, j);
    const Index lo = std::min(i, j), hi = std::max(i, j);
    if (hi < n_old) throw std::invalid_argument("assemble_update: new edge addresses only existing nodes");
    if (lo < n_old) {
      gt.push_back({lo, hi - n_old, w});
    } else {
      ct.push_back({lo - n_old, hi - n_old, w});
      ct.push_back({hi - n_old, lo - n_old, w});
    }
  }
  GraphUpdate d = make_empty_update(n_old, new_node_count);
  d.k_block = from_triplets(n_old, kt);
  d.g_block = csr_from_triplets_raw(n_old, new_node_count, gt);
  d.c_block = from_triplets(new_node_count, ct);
  return d;
}

Csr apply_update(const Csr& a, const GraphUpdate& d) {
  // graph.cpp:102-115
  if (a.rows != d.n_old) throw std::invalid_argument("apply_update: matrix size != d.n_old");
  const Csr padded = pad(a, d.n_new);
  Csr sum = sparse_add(padded, d.to_delta(), +1.0);
  for (Index r = 0; r < sum.rows; ++r)
    for (std::int32_t e = sum.rowptr[static_cast<size_t>(r)]; e < sum.rowptr[static_cast<size_t>(r) + 1]; ++e)
      if (sum.val[static_cast<size_t>(e)] < -1e-12) {
        if (padded.coeff(r, sum.colidx[static_cast<size_t>(e)]) == 0.0)
          throw std::invalid_argument("apply_update: invalid deletion (no such edge)");
        throw std::invalid_argument("apply_update: update drives an edge weight negative");
      }
  return wrap(std::move(sum), false);
}

Csr to_shifted_laplacian(const Csr& a, LaplacianKind kind, double alpha, std::string* warning) {
  // graph.cpp:117-151
  const Index n = a.rows;
  const Vec deg = degrees(a);
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(a.nnz() + n));
  if (kind == LaplacianKind::combinatorial) {
    const double dmax = n > 0 ? *std::max_element(deg.begin(), deg.end()) : 0.0;
    if (alpha < 2.0 * dmax) {
      const std::string msg =
          "to_shifted_laplacian: alpha below 2*d_max; the shifted spectrum may change sign "
          "and magnitude ordering can break";
      if (warning) *warning = msg;
    }
    for (Index i = 0; i < n; ++i) t.push_back({i, i, alpha - deg[static_cast<size_t>(i)]});
    for (Index r = 0; r < n; ++r)
      for (std::int32_t e = a.rowptr[static_cast<size_t>(r)]; e < a.rowptr[static_cast<size_t>(r) + 1]; ++e)
        t.push_back({r, a.colidx[static_cast<size_t>(e)], a.val[static_cast<size_t>(e)]});
  } else {
    if (alpha != 2.0) throw std::invalid_argument("to_shifted_laplacian: normalized kind requires alpha == 2");
    Vec scale(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i)
      scale[static_cast<size_t>(i)] = deg[static_cast<size_t>(i)] > 0.0 ? 1.0 / std::sqrt(deg[static_cast<size_t>(i)]) : 0.0;
    for (Index i = 0; i < n; ++i) t.push_back({i, i, deg[static_cast<size_t>(i)] > 0.0 ? 1.0 : 2.0});
    for (Index r = 0; r < n; ++r)
      for (std::int32_t e = a.rowptr[static_cast<size_t>(r)]; e < a.rowptr[static_cast<size_t>(r) + 1]; ++e) {
        const Index c = a.colidx[static_cast<size_t>(e)];
        t.push_back({r, c, (scale[static_cast<size_t>(r)] * scale[static_cast<size_t>(c)]) * a.val[static_cast<size_t>(e)]});
      }
  }
  return from_triplets(n, t);
}

namespace {
double shift_for(const Csr& a, LaplacianKind kind, double current) {
  // laplacian_track.cpp:35-39
  if (kind == LaplacianKind::normalized) return 2.0;
  double d_max = 0.0;
  if (a.rows > 0) {
    const Vec d = degrees(a);
    d_max = *std::max_element(d.begin(), d.end());
  }
  return std::max(current, 2.0 * d_max);
}
}  // namespace

ShiftedLaplacianSession::ShiftedLaplacianSession(Csr a0, LaplacianKind kind)
    : kind_(kind), alpha_(shift_for(a0, kind, 0.0)), a_(std::move(a0)) {
  t_ = to_shifted_laplacian(a_, kind_, alpha_);
}

Perturbation ShiftedLaplacianSession::advance(const GraphUpdate& d) {
  // laplacian_track.cpp:48-64
  if (d.n_old != a_.rows) throw std::invalid_argument("update does not match the session's node count");
  Csr a_next = apply_update(a_, d);
  const double alpha_next = shift_for(a_next, kind_, alpha_);
  Csr t_next = to_shifted_laplacian(a_next, kind_, alpha_next);
  Csr diff = sparse_add(t_next, pad(t_, d.n_new), -1.0);
  Perturbation p{a_.rows, d.n_new, wrap(std::move(diff), false)};
  a_ = std::move(a_next);
  t_ = std::move(t_next);
  alpha_ = alpha_next;
  return p;
}

// ---------------------------------------------------------------- lanczos
EigResult lanczos_topk_csr(const Csr& a, const LanczosOptions& opts) {
  // lanczos.hpp:38-127 with apply = matvec(a, .)
  const Index n = a.rows;
  if (n < 1) throw std::invalid_argument("lanczos_topk: empty operator");
  if (opts.k < 1 || opts.k > n) throw std::invalid_argument("lanczos_topk: k must satisfy 1 <= k <= n");
  Index m = opts.max_basis > 0 ? opts.max_basis : std::max<Index>(2 * opts.k + 20, 40);
  if (m < opts.k) throw std::invalid_argument("lanczos_topk: max_basis below k");
  m = std::min(m, n);
  GaussianSampler rng(mix_seed(opts.seed, 0x1a2cU));
  Mat vb(n, m), wb(n, m);
  Vec v = rng.gaussian_vector(n);
  Index j = 0;
  double a_norm = 0.0;
  double best_worst = std::numeric_limits<double>::infinity();
  for (Index restart = 0;; ++restart) {
    int fresh = 0;
    while (j < m) {
      for (int pass = 0; pass < 2; ++pass)
        if (j > 0) project_out(vb, j, v);
      const double nrm = norm2(v.data(), n);
      if (!(nrm > 1e-12)) {
        if (++fresh > 4) break;
        v = rng.gaussian_vector(n);
        continue;
      }
      fresh = 0;
      for (auto& x : v) x /= nrm;
      std::copy(v.begin(), v.end(), vb.col(j));
      Vec w = matvec(a, v);
      for (double x : w)
        if (!std::isfinite(x)) throw std::runtime_error("lanczos_topk: operator produced non-finite values");
      std::copy(w.begin(), w.end(), wb.col(j));
      v = std::move(w);
      ++j;
    }
    if (j == 0) throw std::runtime_error("lanczos_topk: could not build a starting basis");
    const Mat vj = left_cols(vb, j), wj = left_cols(wb, j);
    const Mat h = matmul_tn(vj, wj);
    const EigResult ritz = sym_eig_dense(h, opts.order);
    const Index kk = std::min(opts.k, j);
    const Mat fk = left_cols(ritz.vectors, kk);
    Mat x = matmul(vj, fk);
    Mat res = matmul(wj, fk);
    for (Index c = 0; c < kk; ++c)
      for (Index i = 0; i < n; ++i) res(i, c) -= x(i, c) * ritz.values[static_cast<size_t>(c)];
    for (double t : ritz.values) a_norm = std::max(a_norm, std::abs(t));
    const double scale = std::max(a_norm, 1e-300);
    Index first_unconverged = -1;
    double worst = 0.0;
    for (Index i = 0; i < kk; ++i) {
      const double r = norm2(res.col(i), n);
      worst = std::max(worst, r);
      if (first_unconverged < 0 && r > opts.tol * scale) first_unconverged = i;
    }
    best_worst = std::min(best_worst, worst);
    if ((first_unconverged < 0 && kk == opts.k) || j >= n) {
      EigResult out;
      out.values.assign(ritz.values.begin(), ritz.values.begin() + kk);
      out.vectors = std::move(x);
      return out;
    }
    if (restart >= opts.max_restarts) {
      std::ostringstream msg;
      msg << "lanczos_topk: no convergence after " << opts.max_restarts << " restarts (best worst-case residual "
          << best_worst << ", tol " << opts.tol * scale << ")";
      throw std::runtime_error(msg.str());
    }
    const Index keep = std::min<Index>(j - 1 > 0 ? j - 1 : j, opts.k + std::min<Index>(opts.k, 10) + 2);
    const Mat fkeep = left_cols(ritz.vectors, keep);
    const Mat vn = matmul(vj, fkeep), wn = matmul(wj, fkeep);
    std::copy(vn.a.begin(), vn.a.end(), vb.a.begin());
    std::copy(wn.a.begin(), wn.a.end(), wb.a.begin());
    j = keep;
    const Index pick = first_unconverged >= 0 ? first_unconverged : kk - 1;
    v.assign(res.col(pick), res.col(pick) + n);
    if (!(norm2(v.data(), n) > 0.0)) v = rng.gaussian_vector(n);
  }
}

// ---------------------------------------------------------------- trackers
namespace {

Mat padded_vectors(const TrackerState& s, Index extra) {
  // trackers.cpp:20-24
  Mat xb(s.vectors.rows + extra, s.vectors.cols);
  for (Index c = 0; c < s.vectors.cols; ++c) std::copy(s.vectors.col(c), s.vectors.col(c) + s.vectors.rows, xb.col(c));
  return xb;
}

void check_step(const char* who, const TrackerState& s, const Perturbation& p) {
  // trackers.cpp:33-39
  if (p.n_old != s.n) throw std::invalid_argument(std::string(who) + ": perturbation dimension mismatch");
  if (p.n_new < 0) throw std::invalid_argument(std::string(who) + ": negative expansion");
  if (p.delta.rows != p.n_old + p.n_new)
    throw std::invalid_argument(std::string(who) + ": delta size != n_old + n_new");
}

BasisKind basis_kind_of(TrackerKind kind) {
  switch (kind) {
    case TrackerKind::iasc: return BasisKind::iasc;
    case TrackerKind::grest2: return BasisKind::grest2;
    case TrackerKind::grest3: return BasisKind::grest3;
    case TrackerKind::grest_rsvd: return BasisKind::grest_rsvd;
    default: throw std::invalid_argument("basis_kind_of: not a projection tracker");
  }
}

// xb (xb' y) subtracted from y, i.e. (I - xb xb') y.
Mat project_against(const Mat& xb, const Mat& y) {
  const Mat c = matmul_tn(xb, y);
  Mat out = y;
  const Mat xc = matmul(xb, c);
  for (size_t e = 0; e < out.a.size(); ++e) out.a[e] -= xc.a[e];
  return out;
}

// Transposed view Delta.middleRows(n_old, S)' as a CSR over the new-node rows
// of Delta (Delta is symmetric, so row n_old + j of Delta is column j of d2).
struct TrailingBlock {
  const Csr* delta;
  Index n_old, s;
};

// y = d2 * w: y(i, c) = sum_j d2(i, j) w(j, c), j ascending (Eigen column-major
// sparse * dense); d2(i, j) = Delta(i, n_old + j).
Mat trailing_apply(const TrailingBlock& b, const Mat& w) {
  const Csr& d = *b.delta;
  Mat y(d.rows, w.cols);
  for (Index c = 0; c < w.cols; ++c) {
    const double* wc = w.col(c);
    double* yc = y.col(c);
#pragma omp parallel for schedule(static) if (d.rows > 65536)
    for (Index i = 0; i < d.rows; ++i) {
      double tmp = 0.0;
      for (std::int32_t e = d.rowptr[static_cast<size_t>(i)]; e < d.rowptr[static_cast<size_t>(i) + 1]; ++e) {
        const Index col = d.colidx[static_cast<size_t>(e)];
        if (col >= b.n_old) tmp += d.val[static_cast<size_t>(e)] * wc[col - b.n_old];
      }
      yc[i] = tmp;
    }
  }
  return y;
}

// d2' * y: row j of the result is row n_old + j of Delta times y.
Mat trailing_adjoint(const TrailingBlock& b, const Mat& y) {
  const Csr& d = *b.delta;
  Mat out(b.s, y.cols);
  for (Index c = 0; c < y.cols; ++c) {
    const double* yc = y.col(c);
    double* oc = out.col(c);
    for (Index j = 0; j < b.s; ++j) {
      const Index r = b.n_old + j;
      double tmp = 0.0;
      for (std::int32_t e = d.rowptr[static_cast<size_t>(r)]; e < d.rowptr[static_cast<size_t>(r) + 1]; ++e)
        tmp += d.val[static_cast<size_t>(e)] * yc[d.colidx[static_cast<size_t>(e)]];
      oc[j] = tmp;
    }
  }
  return out;
}

}  // namespace

Perturbation to_perturbation(const GraphUpdate& d) { return {d.n_old, d.n_new, d.to_delta()}; }

namespace {
EigResult solve_leading(const Csr& a, const TrackerOptions& opts) {
  // trackers.cpp:67-75
  LanczosOptions lo;
  lo.k = opts.k;
  lo.order = opts.order;
  lo.seed = opts.seed;
  return lanczos_topk_csr(a, lo);
}

double vec_norm(const Vec& v) {  // Eigen Vector::norm (sqrt of the squared sum)
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
}  // namespace

double frobenius_norm(const Csr& a) {
  double s = 0.0;
  for (double x : a.val) s += x * x;
  return std::sqrt(s);
}

TrackerState tracker_init(const Csr& a0, TrackerKind kind, const TrackerOptions& opts) {
  // trackers.cpp:132-145
  if (opts.k < 1 || opts.k > a0.rows) throw std::invalid_argument("tracker_init: k must satisfy 1 <= k <= n");
  if (kind == TrackerKind::timers && opts.restart_inner == static_cast<int>(TrackerKind::timers))
    throw std::invalid_argument("tracker_init: timers cannot delegate to itself");
  TrackerState s;
  s.kind = kind;
  s.opts = opts;
  const EigResult r = solve_leading(a0, opts);
  s.values = r.values;
  s.vectors = r.vectors;
  s.n = a0.rows;
  s.restart_scale = vec_norm(s.values);
  return s;
}

// ---------------------------------------------------------------- perturbation trackers
namespace {
double gap_clamp(const Vec& values) {  // trackers.cpp:26-31
  const double lead = values.empty() ? 0.0 : std::abs(values[0]);
  return 1e-12 * std::max(1.0, lead);
}

// b_ij = c_ij / (lambda_j - lambda_i), degenerate gaps dropped (trackers.cpp:54-65)
Mat first_order_coefficients(const Mat& c, const Vec& lam) {
  const double eps = gap_clamp(lam);
  const Index k = static_cast<Index>(lam.size());
  Mat b(k, k);
  for (Index j = 0; j < k; ++j)
    for (Index i = 0; i < k; ++i) {
      if (i == j) continue;
      const double gap = lam[static_cast<size_t>(j)] - lam[static_cast<size_t>(i)];
      if (std::abs(gap) < eps) continue;
      b(i, j) = c(i, j) / gap;
    }
  return b;
}

// renormalize_and_sort (trackers.cpp:43-52)
void renormalize_and_sort(TrackerState& out, const Vec& values, Mat vectors, SpectralOrder order) {
  for (Index j = 0; j < vectors.cols; ++j) {
    const double nrm = norm2(vectors.col(j), vectors.rows);
    if (nrm > 0.0)
      for (Index i = 0; i < vectors.rows; ++i) vectors(i, j) /= nrm;
  }
  const EigResult r = reorder_eig(values, vectors, order);
  out.values = r.values;
  out.vectors = r.vectors;
}

// xb, dx = Delta xb, c = xb' dx, lambda + diag(c) (trackers.cpp:152-157)
struct FirstOrder {
  Mat xb, dx, c;
  Vec lam_new;
};
FirstOrder first_order(const TrackerState& s, const Perturbation& p) {
  FirstOrder f;
  f.xb = padded_vectors(s, p.n_new);
  f.dx = matmat(p.delta, f.xb);
  f.c = matmul_tn(f.xb, f.dx);
  f.lam_new = s.values;
  for (size_t j = 0; j < f.lam_new.size(); ++j) f.lam_new[j] += f.c(static_cast<Index>(j), static_cast<Index>(j));
  return f;
}
}  // namespace

SmallSolve solve_linear_small(const Mat& a, const Vec& b, double ridge) {
  // solve.hpp:23-45: partial-pivot LU, ridge fallback below a 1e-12 relative pivot
  if (a.rows != a.cols) throw std::invalid_argument("solve_linear_small: matrix must be square");
  if (a.rows != static_cast<Index>(b.size())) throw std::invalid_argument("solve_linear_small: rhs size mismatch");
  for (double x : a.a)
    if (!std::isfinite(x)) throw std::invalid_argument("solve_linear_small: non-finite entries");
  for (double x : b)
    if (!std::isfinite(x)) throw std::invalid_argument("solve_linear_small: non-finite entries");
  const Index n = a.rows;
  if (n == 0) return {};
  double amax = 0.0;
  for (double x : a.a) amax = std::max(amax, std::abs(x));
  auto lu_solve = [&](const Mat& m, double* pivot_min) {
    Mat lu = m;
    std::vector<Index> perm(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) perm[static_cast<size_t>(i)] = i;
    double pmin = std::numeric_limits<double>::infinity();
    for (Index c = 0; c < n; ++c) {
      Index piv = c;
      double best = std::abs(lu(c, c));
      for (Index r = c + 1; r < n; ++r)
        if (std::abs(lu(r, c)) > best) {
          best = std::abs(lu(r, c));
          piv = r;
        }
      if (piv != c) {
        for (Index q = 0; q < n; ++q) std::swap(lu(c, q), lu(piv, q));
        std::swap(perm[static_cast<size_t>(c)], perm[static_cast<size_t>(piv)]);
      }
      const double d = lu(c, c);
      pmin = std::min(pmin, std::abs(d));
      if (d != 0.0)
        for (Index r = c + 1; r < n; ++r) {
          const double l = lu(r, c) / d;
          lu(r, c) = l;
          for (Index q = c + 1; q < n; ++q) lu(r, q) -= l * lu(c, q);
        }
    }
    if (pivot_min) *pivot_min = pmin;
    Vec x(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) x[static_cast<size_t>(i)] = b[static_cast<size_t>(perm[static_cast<size_t>(i)])];
    for (Index i = 0; i < n; ++i)
      for (Index q = 0; q < i; ++q) x[static_cast<size_t>(i)] -= lu(i, q) * x[static_cast<size_t>(q)];
    for (Index i = n - 1; i >= 0; --i) {
      for (Index q = i + 1; q < n; ++q) x[static_cast<size_t>(i)] -= lu(i, q) * x[static_cast<size_t>(q)];
      x[static_cast<size_t>(i)] /= lu(i, i);
    }
    return x;
  };
  if (amax > 0.0) {
    double pmin = 0.0;
    Vec x = lu_solve(a, &pmin);
    if (pmin >= 1e-12 * amax) return {x, false};
  }
  const double eps = ridge * std::max(1.0, amax);
  Mat reg = a;
  for (Index i = 0; i < n; ++i) reg(i, i) += eps;
  return {lu_solve(reg, nullptr), true};
}

TrackerState trip_basic_step(const TrackerState& s, const Perturbation& p) {
  // trackers.cpp:147-164
  check_step("trip_basic_step", s, p);
  TrackerState out = s;
  if (p.empty()) return out;
  const FirstOrder f = first_order(s, p);
  const Mat b = first_order_coefficients(f.c, s.values);
  Mat xt = f.xb;
  const Mat xbb = matmul(f.xb, b);
  for (size_t e = 0; e < xt.a.size(); ++e) xt.a[e] += xbb.a[e];
  renormalize_and_sort(out, f.lam_new, std::move(xt), s.opts.order);
  out.n = p.n_old + p.n_new;
  return out;
}

TrackerState trip_step(const TrackerState& s, const Perturbation& p) {
  // trackers.cpp:166-197
  check_step("trip_step", s, p);
  TrackerState out = s;
  if (p.empty()) return out;
  const FirstOrder f = first_order(s, p);
  const Index k = static_cast<Index>(s.values.size());
  Mat xt(f.xb.rows, k);
  for (Index j = 0; j < k; ++j) {
    Vec rhs(static_cast<size_t>(k));
    double rmax = 0.0;
    for (Index i = 0; i < k; ++i) {
      rhs[static_cast<size_t>(i)] = f.c(i, j);
      rmax = std::max(rmax, std::abs(f.c(i, j)));
    }
    Vec bj(static_cast<size_t>(k), 0.0);
    if (rmax > 0.0) {
      Mat system(k, k);
      for (Index q = 0; q < k; ++q)
        for (Index i = 0; i < k; ++i) system(i, q) = -f.c(i, q);
      for (Index i = 0; i < k; ++i)
        system(i, i) += f.lam_new[static_cast<size_t>(j)] - s.values[static_cast<size_t>(i)];
      const SmallSolve sol = solve_linear_small(system, rhs);
      bj = sol.x;
      out.ridge_used = out.ridge_used || sol.ridge_used;
    }
    for (Index r = 0; r < f.xb.rows; ++r) {
      double acc = 0.0;
      for (Index i = 0; i < k; ++i) acc += f.xb(r, i) * bj[static_cast<size_t>(i)];
      xt(r, j) = s.opts.trip_replace_span ? acc : f.xb(r, j) + acc;
    }
  }
  renormalize_and_sort(out, f.lam_new, std::move(xt), s.opts.order);
  out.n = p.n_old + p.n_new;
  return out;
}

TrackerState residual_modes_step(const TrackerState& s, const Perturbation& p, double mu) {
  // trackers.cpp:199-224
  check_step("residual_modes_step", s, p);
  TrackerState out = s;
  if (p.empty()) return out;
  const double eps = gap_clamp(s.values);
  for (double l : s.values)
    if (std::abs(l - mu) < eps) throw std::invalid_argument("residual_modes_step: mu collides with tracked eigenvalue");
  const FirstOrder f = first_order(s, p);
  const Mat b = first_order_coefficients(f.c, s.values);
  const Mat xc = matmul(f.xb, f.c);
  const Mat xbb = matmul(f.xb, b);
  Mat xt = f.xb;
  for (size_t e = 0; e < xt.a.size(); ++e) xt.a[e] += xbb.a[e];
  for (Index j = 0; j < xt.cols; ++j) {
    const double den = s.values[static_cast<size_t>(j)] - mu;
    for (Index r = 0; r < xt.rows; ++r) xt(r, j) += (f.dx(r, j) - xc(r, j)) / den;
  }
  renormalize_and_sort(out, f.lam_new, std::move(xt), s.opts.order);
  out.n = p.n_old + p.n_new;
  return out;
}

Mat build_projection_basis(const TrackerState& s, const Perturbation& p, BasisKind kind, std::uint64_t seed) {
  // trackers.cpp:226-280
  check_step("build_projection_basis", s, p);
  const Index n_total = p.n_old + p.n_new;
  const Index k = static_cast<Index>(s.values.size());
  const Mat xb = padded_vectors(s, p.n_new);

  if (kind == BasisKind::iasc) {
    Mat z(n_total, k + p.n_new);
    for (Index c = 0; c < k; ++c) std::copy(s.vectors.col(c), s.vectors.col(c) + p.n_old, z.col(c));
    for (Index j = 0; j < p.n_new; ++j) z(p.n_old + j, k + j) = 1.0;
    return z;
  }

  const Mat dx = matmat(p.delta, xb);
  const Mat proj_dx = project_against(xb, dx);

  Mat candidates;
  if (kind == BasisKind::grest2) {
    candidates = proj_dx;
  } else {
    const TrailingBlock d2{&p.delta, p.n_old, p.n_new};
    const bool bypass = kind == BasisKind::grest3 || p.n_new <= s.opts.rsvd_l;
    Mat trailing;
    if (bypass) {
      Mat d2_dense(n_total, p.n_new);
      for (Index j = 0; j < p.n_new; ++j) {
        const Index r = p.n_old + j;
        for (std::int32_t e = p.delta.rowptr[static_cast<size_t>(r)]; e < p.delta.rowptr[static_cast<size_t>(r) + 1]; ++e)
          d2_dense(p.delta.colidx[static_cast<size_t>(e)], j) = p.delta.val[static_cast<size_t>(e)];
      }
      trailing = project_against(xb, d2_dense);
    } else {
      RectOperator op;
      op.rows = n_total;
      op.cols = p.n_new;
      op.apply = [&d2, &xb](const Mat& w) { return project_against(xb, trailing_apply(d2, w)); };
      op.apply_adjoint = [&d2, &xb](const Mat& y) { return trailing_adjoint(d2, project_against(xb, y)); };
      trailing = rsvd_basis(op, s.opts.rsvd_l, s.opts.rsvd_p, seed);
    }
    candidates = Mat(n_total, proj_dx.cols + trailing.cols);
    std::copy(proj_dx.a.begin(), proj_dx.a.end(), candidates.a.begin());
    std::copy(trailing.a.begin(), trailing.a.end(), candidates.a.begin() + static_cast<std::ptrdiff_t>(proj_dx.a.size()));
  }
  const Mat extra = orthonormalize(candidates, xb);
  Mat z(n_total, k + extra.cols);
  std::copy(xb.a.begin(), xb.a.end(), z.a.begin());
  std::copy(extra.a.begin(), extra.a.end(), z.a.begin() + static_cast<std::ptrdiff_t>(xb.a.size()));
  return z;
}

TrackerState rayleigh_ritz_step(const TrackerState& s, const Perturbation& p, const Mat& z) {
  // trackers.cpp:282-308
  check_step("rayleigh_ritz_step", s, p);
  TrackerState out = s;
  if (p.empty()) return out;
  const Index n_total = p.n_old + p.n_new;
  const Index k = static_cast<Index>(s.values.size());
  if (z.rows != n_total) throw std::invalid_argument("rayleigh_ritz_step: basis row count mismatch");
  if (z.cols < k) throw std::invalid_argument("rayleigh_ritz_step: projection subspace too small");
  const Mat gram = matmul_tn(z, z);
  double dev = 0.0;
  for (Index j = 0; j < z.cols; ++j)
    for (Index i = 0; i < z.cols; ++i) dev = std::max(dev, std::abs(gram(i, j) - (i == j ? 1.0 : 0.0)));
  if (dev > 1e-6) throw std::invalid_argument("rayleigh_ritz_step: basis is not column-orthonormal");

  const Mat xb = padded_vectors(s, p.n_new);
  const Mat zx = matmul_tn(z, xb);  // D x K
  const Mat dz = matmat(p.delta, z);
  Mat zxl = zx;
  for (Index c = 0; c < k; ++c)
    for (Index i = 0; i < zx.rows; ++i) zxl(i, c) *= s.values[static_cast<size_t>(c)];
  Mat m = matmul(zxl, transpose(zx));
  const Mat ztdz = matmul_tn(z, dz);
  for (size_t e = 0; e < m.a.size(); ++e) m.a[e] += ztdz.a[e];
  const EigResult ritz = sym_eig_dense(m, s.opts.order);
  out.values.assign(ritz.values.begin(), ritz.values.begin() + k);
  out.vectors = matmul(z, left_cols(ritz.vectors, k));
  out.n = n_total;
  return out;
}

TrackerState tracker_step(const TrackerState& s, const Perturbation& p, const Csr* full_matrix) {
  // trackers.cpp:341-382
  TrackerState out;
  switch (s.kind) {
    case TrackerKind::trip_basic:
      out = trip_basic_step(s, p);
      break;
    case TrackerKind::trip:
      out = trip_step(s, p);
      break;
    case TrackerKind::residual_modes:
      out = residual_modes_step(s, p, s.opts.mu);
      break;
    case TrackerKind::timers: {
      // timers_step (trackers.cpp:310-339) around the inner kind
      check_step("timers_step", s, p);
      if (s.opts.theta < 0.0) throw std::invalid_argument("timers_step: theta must be >= 0");
      TrackerState acc = s;
      acc.kind = static_cast<TrackerKind>(s.opts.restart_inner);
      const double denom = s.restart_scale > 0.0 ? s.restart_scale : 1.0;
      acc.accumulated_change += frobenius_norm(p.delta) / denom;
      acc.steps_since_restart += 1;
      if (acc.accumulated_change >= s.opts.theta && acc.steps_since_restart >= s.opts.min_restart_gap) {
        if (!full_matrix) throw std::invalid_argument("timers_step: restart requires a full-matrix provider");
        if (full_matrix->rows != p.n_old + p.n_new)
          throw std::invalid_argument("timers_step: provider matrix has the wrong dimension");
        const EigResult r = solve_leading(*full_matrix, s.opts);
        out = acc;
        out.values = r.values;
        out.vectors = r.vectors;
        out.n = full_matrix->rows;
        out.restart_scale = vec_norm(out.values);
        out.accumulated_change = 0.0;
        out.steps_since_restart = 0;
      } else {
        out = tracker_step(acc, p, nullptr);
        out.accumulated_change = acc.accumulated_change;
        out.steps_since_restart = acc.steps_since_restart;
      }
      out.kind = TrackerKind::timers;
      break;
    }
    case TrackerKind::iasc:
    case TrackerKind::grest2:
    case TrackerKind::grest3:
    case TrackerKind::grest_rsvd: {
      if (p.empty()) {
        out = s;
        break;
      }
      const std::uint64_t basis_seed = mix_seed(s.opts.seed, 0x6b7aU, s.steps_taken);
      const Mat z = build_projection_basis(s, p, basis_kind_of(s.kind), basis_seed);
      out = rayleigh_ritz_step(s, p, z);
      break;
    }
    default:
      throw std::invalid_argument("tracker_step: tracker kind outside the G-REST path");
  }
  out.steps_taken = s.steps_taken + 1;
  return out;
}

// ---------------------------------------------------------------- metrics
double subspace_sin_largest_angle(const Mat& x, const Mat& y) {
  // metrics.cpp:243-259 (returns sin of the angle)
  if (x.rows != y.rows) throw std::invalid_argument("row counts differ");
  Mat qa = orthonormalize(x), qb = orthonormalize(y);
  if (qa.cols == 0 || qb.cols == 0) throw std::invalid_argument("empty subspace has no angle");
  if (qa.cols > qb.cols) std::swap(qa, qb);
  const Mat g = matmul_tn(qa, qb);
  Vec sg;
  Mat ug;
  thin_svd_u(g, sg, ug);
  const double c = sg.empty() ? 0.0 : *std::min_element(sg.begin(), sg.end());
  Mat residual = qa;
  const Mat pr = matmul(qb, transpose(g));
  double amax = 0.0;
  for (size_t e = 0; e < residual.a.size(); ++e) {
    residual.a[e] -= pr.a[e];
    amax = std::max(amax, std::abs(residual.a[e]));
  }
  double sres = 0.0;
  if (amax != 0.0) {
    Vec sr;
    Mat ur;
    thin_svd_u(transpose(residual), sr, ur);  // singular values of residual
    sres = sr.empty() ? 0.0 : *std::max_element(sr.begin(), sr.end());
  }
  return std::sin(std::atan2(sres, std::max(c, 0.0)));
}

}  // namespace spectrack_oracle
