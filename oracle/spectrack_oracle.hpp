// TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the reference hot path.
//
// This header restates, in plain C++17 without Eigen, the reference library
// `spectrack` (arxiv 2603.19439, /root/reference/proj) for the G-REST per-step
// eigen-update path. It is the parity checker for the CUDA implementation in
// paper_2603_19439_b200/csrc and the `cpu_baseline` leg of bench.py. Nothing in
// the product path links, imports or executes it.
//
// Parity status: the reference cannot be compiled in this image (it needs
// Eigen 3.4, absent; vendor/ is absent), so this restatement is pinned against
// the reference's own known-answer tests (ported to tests/test_oracle_*.py) and
// against the hand-derived golden vectors in tests/golden/.
//
// Every function cites the reference file:line it follows. Dense matrices are
// column-major like Eigen's defaults; CSR uses int32 offsets/indices like
// Eigen::SparseMatrix<double, RowMajor> (sparse.hpp:18).
#pragma once

#include <cstdint>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

namespace spectrack_oracle {

using Index = std::int64_t;

// ---------------------------------------------------------------- dense
struct Mat {  // column-major, like Eigen::MatrixXd
  Index rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return a[static_cast<size_t>(j * rows + i)]; }
  double operator()(Index i, Index j) const { return a[static_cast<size_t>(j * rows + i)]; }
  double* col(Index j) { return a.data() + j * rows; }
  const double* col(Index j) const { return a.data() + j * rows; }
  static Mat identity(Index n) {
    Mat m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};
using Vec = std::vector<double>;

Mat transpose(const Mat& m);
Mat matmul(const Mat& a, const Mat& b);     // a * b
Mat matmul_tn(const Mat& a, const Mat& b);  // a' * b
Mat left_cols(const Mat& m, Index c);

// types.hpp:22-40
enum class SpectralOrder { abs_desc = 0, alg_desc = 1 };
std::vector<Index> spectral_sort(const Vec& values, SpectralOrder order);

// eig.hpp:17-50
struct EigResult {
  Vec values;
  Mat vectors;
};
EigResult reorder_eig(const Vec& values, const Mat& vectors, SpectralOrder order);
EigResult sym_eig_dense(const Mat& s, SpectralOrder order);

// ortho.hpp:13-45
Mat orthonormalize(const Mat& m, const Mat& against, double drop_tol = 1e-10);
Mat orthonormalize(const Mat& m, double drop_tol = 1e-10);

// rng.hpp:16-75
std::uint64_t mix_seed(std::uint64_t base, std::uint64_t salt);
std::uint64_t mix_seed(std::uint64_t base, std::uint64_t a, std::uint64_t b);
class GaussianSampler {
 public:
  explicit GaussianSampler(std::uint64_t seed) : gen_(seed) {}
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  std::uint64_t raw() { return gen_(); }
  Index uniform_index(Index n) { return static_cast<Index>(gen_() % static_cast<std::uint64_t>(n)); }
  double operator()();
  Vec gaussian_vector(Index n);
  Mat gaussian_matrix(Index rows, Index cols);

 private:
  std::mt19937_64 gen_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

// Thin SVD used by rsvd_basis (rsvd.hpp:58): singular values (descending) and
// thin left singular vectors of a general matrix.
void thin_svd_u(const Mat& m, Vec& sv, Mat& u);

// rsvd.hpp:24-66
struct RectOperator {
  Index rows = 0, cols = 0;
  std::function<Mat(const Mat&)> apply;          // (cols x m) -> (rows x m)
  std::function<Mat(const Mat&)> apply_adjoint;  // (rows x m) -> (cols x m)
};
Mat rsvd_basis(const RectOperator& op, Index target_rank, Index oversample, std::uint64_t seed);
RectOperator dense_operator(const Mat& b);  // rsvd.hpp:68-77

// ---------------------------------------------------------------- sparse
struct Triplet {
  Index row, col;
  double value;
};

// sparse.hpp:18-70 — symmetric, both triangles stored, sorted columns, no zeros.
struct Csr {
  Index rows = 0, cols = 0;
  std::vector<std::int32_t> rowptr{0};
  std::vector<std::int32_t> colidx;
  std::vector<double> val;
  Index nnz() const { return static_cast<Index>(val.size()); }
  double coeff(Index i, Index j) const;
  double frobenius_norm() const;
};

Csr csr_from_triplets_raw(Index rows, Index cols, const std::vector<Triplet>& t);  // setFromTriplets
Csr from_triplets(Index n, const std::vector<Triplet>& t);                         // sparse.cpp:17-23
Csr from_edges(Index n, const std::vector<std::tuple<Index, Index, double>>& edges);  // sparse.cpp:25-53
Csr wrap(Csr m, bool validate);                                                    // sparse.cpp:55-63
bool is_symmetric(const Csr& m);                                                   // sparse.cpp:65-77
void prune_zeros(Csr& m);                                                          // sparse.cpp:10-13
Vec matvec(const Csr& a, const Vec& x);                                            // sparse.cpp:79-82
Mat matmat(const Csr& a, const Mat& x);                                            // sparse.cpp:84-87
Csr pad(const Csr& a, Index s);                                                    // sparse.cpp:89-95
Vec degrees(const Csr& a);                                                         // sparse.cpp:97-99
Csr sparse_add(const Csr& a, const Csr& b, double sign_b);                         // Eigen a + b / a - b
Mat to_dense(const Csr& a);

// ---------------------------------------------------------------- graph
struct GraphUpdate {  // graph.hpp:23-37
  Index n_old = 0, n_new = 0;
  Csr k_block;  // n_old x n_old
  Csr g_block;  // n_old x n_new
  Csr c_block;  // n_new x n_new
  bool empty() const { return n_new == 0 && nnz() == 0; }
  Index nnz() const { return k_block.nnz() + 2 * g_block.nnz() + c_block.nnz(); }
  double frobenius_norm() const;
  Csr to_delta() const;  // graph.cpp:17-32
};
GraphUpdate make_empty_update(Index n_old, Index n_new = 0);  // graph.cpp:34-43
GraphUpdate assemble_update(Index n_old,
                            const std::vector<std::tuple<Index, Index, double>>& added,
                            const std::vector<std::pair<Index, Index>>& removed, Index new_node_count,
                            const std::vector<std::tuple<Index, Index, double>>& new_edges);  // graph.cpp:45-100
Csr apply_update(const Csr& a, const GraphUpdate& d);                                // graph.cpp:102-115
enum class LaplacianKind { combinatorial = 0, normalized = 1 };
Csr to_shifted_laplacian(const Csr& a, LaplacianKind kind, double alpha, std::string* warning = nullptr);

// ---------------------------------------------------------------- trackers
enum class TrackerKind { trip_basic, trip, residual_modes, iasc, grest2, grest3, grest_rsvd, timers };
enum class BasisKind { iasc, grest2, grest3, grest_rsvd };

struct TrackerOptions {  // trackers.hpp:52-63
  Index k = 8;
  SpectralOrder order = SpectralOrder::abs_desc;
  double mu = 0.0;                 // residual-modes denominator scalar
  bool trip_replace_span = false;  // x = X b instead of x = x + X b
  Index rsvd_l = 100;
  Index rsvd_p = 100;
  double theta = 0.01;             // timers restart threshold
  Index min_restart_gap = 5;       // timers minimum steps between restarts
  int restart_inner = 3;           // TrackerKind timers delegates to (iasc)
  std::uint64_t seed = 0;
};

struct TrackerState {  // trackers.hpp:65-75
  TrackerKind kind = TrackerKind::grest3;
  TrackerOptions opts;
  Vec values;
  Mat vectors;
  Index n = 0;
  double accumulated_change = 0.0;
  Index steps_since_restart = 0;
  double restart_scale = 0.0;
  std::uint64_t steps_taken = 0;
  bool ridge_used = false;
};

struct Perturbation {  // trackers.hpp:78-84
  Index n_old = 0, n_new = 0;
  Csr delta;
  bool empty() const { return n_new == 0 && delta.nnz() == 0; }
};

Perturbation to_perturbation(const GraphUpdate& d);  // trackers.cpp:128-130

struct LanczosOptions {  // lanczos.hpp:29-36
  Index k = 1;
  SpectralOrder order = SpectralOrder::abs_desc;
  double tol = 1e-10;
  Index max_basis = 0;
  std::uint64_t seed = 0;
  Index max_restarts = 500;
};
EigResult lanczos_topk_csr(const Csr& a, const LanczosOptions& opts);  // lanczos.hpp:38-127

TrackerState tracker_init(const Csr& a0, TrackerKind kind, const TrackerOptions& opts);  // trackers.cpp:132-145
Mat build_projection_basis(const TrackerState& s, const Perturbation& p, BasisKind kind,
                           std::uint64_t seed);  // trackers.cpp:226-280
TrackerState rayleigh_ritz_step(const TrackerState& s, const Perturbation& p, const Mat& z);  // :282-308
// The perturbation trackers and TIMERS (trackers.cpp:147-224, 310-339)
struct SmallSolve {  // solve.hpp:17-45
  Vec x;
  bool ridge_used = false;
};
SmallSolve solve_linear_small(const Mat& a, const Vec& b, double ridge = 1e-10);
TrackerState trip_basic_step(const TrackerState& s, const Perturbation& p);
TrackerState trip_step(const TrackerState& s, const Perturbation& p);
TrackerState residual_modes_step(const TrackerState& s, const Perturbation& p, double mu);
// full_matrix: the current operator (the reference's MatrixProvider), may be null
TrackerState tracker_step(const TrackerState& s, const Perturbation& p,
                          const Csr* full_matrix = nullptr);  // trackers.cpp:341-382
double frobenius_norm(const Csr& a);  // sparse.hpp:43

// laplacian_track.cpp:35-64
class ShiftedLaplacianSession {
 public:
  ShiftedLaplacianSession(Csr a0, LaplacianKind kind);
  Perturbation advance(const GraphUpdate& d);
  const Csr& adjacency() const { return a_; }
  const Csr& shifted() const { return t_; }
  double alpha() const { return alpha_; }

 private:
  LaplacianKind kind_;
  double alpha_;
  Csr a_, t_;
};

// metrics.cpp:17-27, 243-259 (parity metric): sin of the largest principal
// angle between span(a) and span(b).
double subspace_sin_largest_angle(const Mat& a, const Mat& b);

}  // namespace spectrack_oracle
