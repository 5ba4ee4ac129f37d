// spectrack_b200.hpp — header-only C++17 shim that re-exposes the reference
// `spectrack` update API (proj/include/spectrack/{trackers,graph,
// laplacian_track}.hpp) on top of the C ABI in spectrack_gpu.h, without Eigen.
//
// Mapping (reference -> here):
//   assemble_update(n_old, added, removed, S, new_edges)   graph.hpp:65-69
//       -> EditLists (the same four arguments, validated on the device with
//          the reference's rules and messages)
//   tracker_init(a0, kind, opts)                           trackers.hpp:92
//       -> tracker_init(a0, kind, opts, op): thick-restart Lanczos on the
//          device (lanczos.hpp:38-127); or GpuTracker(a0, kind, opts, op,
//          initial) when the caller already holds X0, Lambda0
//   tracker_step(state, GraphUpdate)                       trackers.hpp:132-133
//       -> tracker_step(tracker, GraphUpdate) (blocks K, G, C) or
//          tracker_step(tracker, EditLists)
//   tracker_step(state, Perturbation)                      trackers.hpp:130-131
//       -> tracker_step(tracker, Perturbation) (adjacency lanes)
//   principal_angle / subspace_largest_angle               metrics.hpp
//       -> GpuTracker::angles (on the device)
//   apply_update(A, d)                                     graph.hpp:74
//   ShiftedLaplacianSession::advance(d)                    laplacian_track.hpp:34
//       -> tracker_step(tracker, edits): one call performs all three on the
//          device-resident state
//   build_projection_basis / rayleigh_ritz_step            trackers.hpp:112-118
//       -> GpuTracker::projection_basis / rayleigh_ritz (no state change)
//   sym_eig_dense (eig.hpp:37-50), GaussianSampler::gaussian_matrix (rng.hpp:64-69)
//       -> sym_eig_dense / gaussian_matrix below
// Errors are rethrown as the reference's exception types with its messages:
// std::invalid_argument and std::runtime_error.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "spectrack_gpu.h"

namespace spectrack_b200 {

using Index = std::int64_t;

enum class TrackerKind {
  trip_basic = ST_TRIP_BASIC,
  trip = ST_TRIP,
  residual_modes = ST_RESIDUAL_MODES,
  iasc = ST_IASC,
  grest2 = ST_GREST2,
  grest3 = ST_GREST3,
  grest_rsvd = ST_GREST_RSVD,
  timers = ST_TIMERS
};
enum class BasisKind { iasc = 0, grest2 = 1, grest3 = 2, grest_rsvd = 3 };
enum class SpectralOrder { abs_desc = ST_ABS_DESC, alg_desc = ST_ALG_DESC };
enum class OperatorKind {
  adjacency = ST_ADJACENCY,
  laplacian = ST_LAPLACIAN,
  normalized_laplacian = ST_NORMALIZED_LAPLACIAN
};

// TrackerOptions (trackers.hpp:52-63).
struct TrackerOptions {
  Index k = 8;
  SpectralOrder order = SpectralOrder::abs_desc;
  double mu = 0.0;
  bool trip_replace_span = false;
  Index rsvd_l = 100;
  Index rsvd_p = 100;
  double theta = 0.01;
  Index min_restart_gap = 5;
  TrackerKind restart_inner = TrackerKind::iasc;
  std::uint64_t seed = 0;
};

// LanczosOptions (lanczos.hpp:29-36) beyond k / order / seed.
struct LanczosOptions {
  double tol = 1e-10;
  Index max_basis = 0;
  Index max_restarts = 500;
};

// Symmetric CSR in the layout of SymSparseMatrix (sparse.hpp:18, 46-48).
struct Csr {
  Index n = 0;
  std::vector<std::int32_t> row_offsets{0};
  std::vector<std::int32_t> col_indices;
  std::vector<double> values;
  Index nnz() const { return static_cast<Index>(values.size()); }
};

// SpectralEmbedding (trackers.hpp:28-34): vectors column-major n x k.
struct SpectralEmbedding {
  std::vector<double> values;
  std::vector<double> vectors;
  Index n = 0;
  Index k() const { return static_cast<Index>(values.size()); }
};

// GraphUpdate (graph.hpp:23-37): the blocks K (n_old^2), G (n_old x n_new),
// C (n_new^2) of the step's perturbation, each a CSR.
struct BlockCsr {
  Index rows = 0, cols = 0;
  std::vector<std::int32_t> row_offsets{0};
  std::vector<std::int32_t> col_indices;
  std::vector<double> values;
};
struct GraphUpdate {
  Index n_old = 0, n_new = 0;
  BlockCsr k_block, g_block, c_block;
};
// Perturbation (trackers.hpp:78-86): delta is (n_old + n_new) square.
struct Perturbation {
  Index n_old = 0, n_new = 0;
  BlockCsr delta;
};

// The arguments of assemble_update (graph.cpp:45-100).
struct EditLists {
  std::vector<std::tuple<Index, Index, double>> added_edges;
  std::vector<std::pair<Index, Index>> removed_edges;
  Index new_node_count = 0;
  std::vector<std::tuple<Index, Index, double>> new_edges;
};

namespace detail {
inline st_csr_block block_of(const BlockCsr& b) {
  return st_csr_block{b.rows, b.cols, static_cast<std::int64_t>(b.values.size()), b.row_offsets.data(),
                      b.col_indices.data(), b.values.data()};
}
inline st_config config_of(TrackerKind kind, const TrackerOptions& opts, OperatorKind op, int device, int flags) {
  st_config cfg{};
  cfg.kind = static_cast<std::int32_t>(kind);
  cfg.op = static_cast<std::int32_t>(op);
  cfg.k = opts.k;
  cfg.order = static_cast<std::int32_t>(opts.order);
  cfg.rsvd_l = opts.rsvd_l;
  cfg.rsvd_p = opts.rsvd_p;
  cfg.seed = opts.seed;
  cfg.device = device;
  cfg.flags = flags;
  return cfg;
}
inline st_tracker_options tracker_options_of(const TrackerOptions& o) {
  return st_tracker_options{o.mu, o.trip_replace_span ? 1 : 0, o.theta, o.min_restart_gap,
                            static_cast<std::int32_t>(o.restart_inner)};
}
// The message is fetched after the call returns (st_last_error's buffer is
// rewritten by every failing call).
inline void rethrow(st_status s, const st_session* session) {
  if (s == ST_OK) return;
  const char* msg = st_last_error(session);
  switch (s) {
    case ST_OK: return;
    case ST_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ST_RUNTIME_ERROR: throw std::runtime_error(msg);
    default: throw std::runtime_error(std::string("spectrack_b200 device failure: ") + msg);
  }
}

struct PackedUpdate {  // SoA copies of the edit lists backing an st_update
  std::vector<std::int64_t> ai, aj, ri, rj, ni, nj;
  std::vector<double> aw, nw;
  st_update u{};
  explicit PackedUpdate(const EditLists& e) {
    for (const auto& [i, j, w] : e.added_edges) {
      ai.push_back(i);
      aj.push_back(j);
      aw.push_back(w);
    }
    for (const auto& [i, j] : e.removed_edges) {
      ri.push_back(i);
      rj.push_back(j);
    }
    for (const auto& [i, j, w] : e.new_edges) {
      ni.push_back(i);
      nj.push_back(j);
      nw.push_back(w);
    }
    u.n_added = static_cast<std::int64_t>(ai.size());
    u.added_i = ai.data();
    u.added_j = aj.data();
    u.added_w = aw.data();
    u.n_removed = static_cast<std::int64_t>(ri.size());
    u.removed_i = ri.data();
    u.removed_j = rj.data();
    u.n_new = e.new_node_count;
    u.n_new_edges = static_cast<std::int64_t>(ni.size());
    u.new_i = ni.data();
    u.new_j = nj.data();
    u.new_w = nw.data();
  }
};
}  // namespace detail

// One tracker lane resident on one GPU: the adjacency (and, for Laplacian
// operators, the shifted operator T of ShiftedLaplacianSession) plus the
// TrackerState. Unlike the reference's value-semantics TrackerState, the state
// lives in HBM and is updated in place; a failed step leaves it unchanged,
// which is what the reference's `state = tracker_step(state, ...)` assignment
// observes when the call throws.
class GpuTracker {
 public:
  GpuTracker(const Csr& a0, TrackerKind kind, const TrackerOptions& opts, OperatorKind op,
             const SpectralEmbedding& initial, int device = 0, int flags = 0) {
    const st_config cfg = detail::config_of(kind, opts, op, device, flags);
    if (initial.k() != opts.k || initial.n != a0.n || static_cast<Index>(initial.vectors.size()) != a0.n * opts.k)
      throw std::invalid_argument("tracker_init: initial embedding does not match n x k");
    detail::rethrow(st_create(&cfg, a0.n, a0.row_offsets.data(), a0.col_indices.data(), a0.values.data(),
                              initial.values.data(), initial.vectors.data(), a0.n, &s_),
                    nullptr);
    set_options(opts);
  }
  // tracker_init (trackers.cpp:132-145): Lanczos on the device
  GpuTracker(const Csr& a0, TrackerKind kind, const TrackerOptions& opts, OperatorKind op,
             const LanczosOptions& lz, int device = 0, int flags = 0) {
    const st_config cfg = detail::config_of(kind, opts, op, device, flags);
    const st_lanczos_options lo{lz.tol, lz.max_basis, lz.max_restarts};
    detail::rethrow(st_tracker_init(&cfg, &lo, a0.n, a0.row_offsets.data(), a0.col_indices.data(), a0.values.data(),
                                    &s_),
                    nullptr);
    set_options(opts);
  }
  void set_options(const TrackerOptions& opts) {
    const st_tracker_options to = detail::tracker_options_of(opts);
    detail::rethrow(st_set_tracker_options(s_, &to), s_);
  }
  GpuTracker(const GpuTracker&) = delete;
  GpuTracker& operator=(const GpuTracker&) = delete;
  GpuTracker(GpuTracker&& o) noexcept : s_(o.s_) { o.s_ = nullptr; }
  ~GpuTracker() {
    if (s_) st_destroy(s_);
  }

  // assemble_update + to_perturbation/advance + apply_update + tracker_step
  void step(const EditLists& edits) {
    detail::PackedUpdate pu(edits);
    detail::rethrow(st_step(s_, &pu.u), s_);
  }

  // tracker_step(state, GraphUpdate) with apply_update (graph.cpp:17-32, 102-115)
  void step(const GraphUpdate& d) {
    st_graph_update g{d.n_old, d.n_new, detail::block_of(d.k_block), detail::block_of(d.g_block),
                      detail::block_of(d.c_block)};
    detail::rethrow(st_step_blocks(s_, &g), s_);
  }
  // tracker_step(state, Perturbation) (trackers.cpp:341-382); A += delta
  void step(const Perturbation& p) {
    const st_csr_block b = detail::block_of(p.delta);
    detail::rethrow(st_step_perturbation(s_, p.n_old, p.n_new, &b), s_);
  }
  // principal_angle per vector and subspace_largest_angle against reference
  // vectors (column-major n x k), on the device (metrics.cpp:17-27, 243-259)
  std::pair<std::vector<double>, double> angles(const std::vector<double>& ref) const {
    const Info in = info();
    std::vector<double> psi(static_cast<size_t>(in.k));
    double big = 0.0;
    detail::rethrow(st_angles(s_, ref.data(), in.n, psi.data(), &big), s_);
    return {psi, big};
  }

  Index n() const { return info().n; }
  std::uint64_t steps_taken() const { return info().steps; }
  double alpha() const { return info().alpha; }  // Laplacian shift (laplacian_track.hpp:40)

  SpectralEmbedding embedding() const {
    const Info in = info();
    SpectralEmbedding e;
    e.n = in.n;
    e.values.resize(static_cast<size_t>(in.k));
    e.vectors.resize(static_cast<size_t>(in.n * in.k));
    detail::rethrow(st_get_embedding(s_, e.values.data(), e.vectors.data(), in.n), s_);
    return e;
  }

  // laplacian_view (laplacian_track.cpp:66-71): nu = alpha - mu
  SpectralEmbedding laplacian_view() const {
    SpectralEmbedding e = embedding();
    const double a = alpha();
    for (double& v : e.values) v = a - v;
    return e;
  }

  // which: 0 adjacency, 1 shifted operator T, 2 last perturbation (Delta or Delta_T)
  Csr csr(int which) const {
    const Info in = info();
    const Index nnz = which == 0 ? in.nnz_a : which == 1 ? in.nnz_t : in.nnz_delta;
    Csr m;
    m.n = in.n;
    m.row_offsets.resize(static_cast<size_t>(in.n + 1));
    m.col_indices.resize(static_cast<size_t>(nnz));
    m.values.resize(static_cast<size_t>(nnz));
    detail::rethrow(st_get_csr(s_, which, m.row_offsets.data(), m.col_indices.data(), m.values.data()),
                    s_);
    return m;
  }

  // build_projection_basis (trackers.cpp:226-280) for `edits`, column-major n_total x D
  std::vector<double> projection_basis(const EditLists& edits, BasisKind kind, std::uint64_t seed,
                                       Index* cols) const {
    detail::PackedUpdate pu(edits);
    const Index n_total = n() + edits.new_node_count;
    const Index maxc = 2 * info().k + edits.new_node_count + 512;
    std::vector<double> z(static_cast<size_t>(n_total * maxc));
    std::int64_t d = 0;
    detail::rethrow(st_probe_basis(s_, &pu.u, static_cast<std::int32_t>(kind), seed, z.data(), n_total, maxc, &d),
                    s_);
    z.resize(static_cast<size_t>(n_total * d));
    if (cols) *cols = d;
    return z;
  }

  // rayleigh_ritz_step (trackers.cpp:282-308) against a caller basis (column-major)
  SpectralEmbedding rayleigh_ritz(const EditLists& edits, const std::vector<double>& z, Index rows, Index cols) const {
    detail::PackedUpdate pu(edits);
    const Index k = info().k;
    SpectralEmbedding e;
    e.n = rows;
    e.values.resize(static_cast<size_t>(k));
    e.vectors.resize(static_cast<size_t>(rows * k));
    detail::rethrow(st_probe_rr(s_, &pu.u, z.data(), rows, cols, rows, e.values.data(), e.vectors.data(), rows),
                    s_);
    return e;
  }

 private:
  struct Info {
    Index n, k, nnz_a, nnz_t, nnz_delta;
    std::uint64_t steps;
    double alpha;
  };
  Info info() const {
    Info in{};
    st_info(s_, &in.n, &in.k, &in.steps, &in.nnz_a, &in.nnz_t, &in.nnz_delta, &in.alpha);
    return in;
  }
  st_session* s_ = nullptr;
};

// tracker_init (trackers.hpp:92) in the reference's call shape.
inline GpuTracker tracker_init(const Csr& a0, TrackerKind kind, const TrackerOptions& opts,
                               OperatorKind op = OperatorKind::adjacency, int device = 0) {
  return GpuTracker(a0, kind, opts, op, LanczosOptions{}, device);
}

// tracker_step (trackers.hpp:130-133) in the reference's call shapes.
inline GpuTracker& tracker_step(GpuTracker& t, const EditLists& edits) {
  t.step(edits);
  return t;
}
inline GpuTracker& tracker_step(GpuTracker& t, const GraphUpdate& d) {
  t.step(d);
  return t;
}
inline GpuTracker& tracker_step(GpuTracker& t, const Perturbation& p) {
  t.step(p);
  return t;
}

// sym_eig_dense (eig.hpp:37-50): values in spectral order, leading `want`
// eigenvectors column-major.
inline std::pair<std::vector<double>, std::vector<double>> sym_eig_dense(const std::vector<double>& s, Index n,
                                                                         SpectralOrder order, Index want,
                                                                         int device = 0) {
  std::vector<double> w(static_cast<size_t>(n)), v(static_cast<size_t>(n * want));
  detail::rethrow(st_sym_eig_dense(device, n, s.data(), static_cast<std::int32_t>(order), want, w.data(), v.data()),
                  nullptr);
  return {w, v};
}

// GaussianSampler(seed).gaussian_matrix(rows, cols) (rng.hpp:64-69), column-major.
inline std::vector<double> gaussian_matrix(std::uint64_t seed, Index rows, Index cols, int device = 0) {
  std::vector<double> out(static_cast<size_t>(rows * cols));
  detail::rethrow(st_gaussian_matrix(device, seed, rows, cols, out.data()), nullptr);
  return out;
}

}  // namespace spectrack_b200
