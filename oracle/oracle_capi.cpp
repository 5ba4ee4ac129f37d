// TEST INFRASTRUCTURE ONLY — C entry points over the CPU restatement so the
// Python parity tests (tests/) and bench.py's cpu_baseline leg can drive it via
// ctypes. Status codes mirror include/spectrack_gpu.h: 0 ok, 1 invalid_argument,
// 2 runtime_error, 4 other.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <optional>

#include "spectrack_oracle.hpp"

using namespace spectrack_oracle;

namespace {

int fail(char* err, int errlen, const char* msg, int code) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

template <typename F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(err, errlen, e.what(), 1);
  } catch (const std::runtime_error& e) {
    return fail(err, errlen, e.what(), 2);
  } catch (const std::exception& e) {
    return fail(err, errlen, e.what(), 4);
  }
}

Csr csr_in(std::int64_t n, const std::int32_t* rowptr, const std::int32_t* col, const double* val) {
  Csr m;
  m.rows = m.cols = n;
  m.rowptr.assign(rowptr, rowptr + n + 1);
  const std::int64_t nnz = rowptr[n];
  m.colidx.assign(col, col + nnz);
  m.val.assign(val, val + nnz);
  return m;
}

Mat mat_in(std::int64_t r, std::int64_t c, const double* a) {
  Mat m(r, c);
  if (r * c > 0) std::memcpy(m.a.data(), a, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

GraphUpdate update_in(std::int64_t n_old, std::int64_t n_add, const std::int64_t* ai, const std::int64_t* aj,
                      const double* aw, std::int64_t n_rem, const std::int64_t* ri, const std::int64_t* rj,
                      std::int64_t n_new_nodes, std::int64_t n_new_edges, const std::int64_t* ni,
                      const std::int64_t* nj, const double* nw) {
  std::vector<std::tuple<Index, Index, double>> added, newe;
  std::vector<std::pair<Index, Index>> removed;
  added.reserve(static_cast<size_t>(n_add));
  for (std::int64_t e = 0; e < n_add; ++e) added.emplace_back(ai[e], aj[e], aw[e]);
  removed.reserve(static_cast<size_t>(n_rem));
  for (std::int64_t e = 0; e < n_rem; ++e) removed.emplace_back(ri[e], rj[e]);
  newe.reserve(static_cast<size_t>(n_new_edges));
  for (std::int64_t e = 0; e < n_new_edges; ++e) newe.emplace_back(ni[e], nj[e], nw[e]);
  return assemble_update(n_old, added, removed, n_new_nodes, newe);
}

struct Session {
  int op = 0;  // 0 adjacency, 1 combinatorial Laplacian, 2 normalized Laplacian
  Csr a;
  std::optional<ShiftedLaplacianSession> lap;
  TrackerState state;
  Csr last_delta;
};

TrackerKind kind_of(int k) {
  if (k < 0 || k > 7) throw std::invalid_argument("unknown tracker kind");
  return static_cast<TrackerKind>(k);  // trackers.hpp:36-45 order
}

}  // namespace

extern "C" {

struct or_csr {
  Csr m;
};
struct or_mat {
  Mat m;
};

void or_csr_info(const or_csr* h, std::int64_t* rows, std::int64_t* nnz) {
  *rows = h->m.rows;
  *nnz = h->m.nnz();
}
void or_csr_copy(const or_csr* h, std::int32_t* rowptr, std::int32_t* col, double* val) {
  std::memcpy(rowptr, h->m.rowptr.data(), sizeof(std::int32_t) * h->m.rowptr.size());
  if (h->m.nnz()) {
    std::memcpy(col, h->m.colidx.data(), sizeof(std::int32_t) * h->m.colidx.size());
    std::memcpy(val, h->m.val.data(), sizeof(double) * h->m.val.size());
  }
}
void or_csr_free(or_csr* h) { delete h; }
void or_mat_info(const or_mat* h, std::int64_t* rows, std::int64_t* cols) {
  *rows = h->m.rows;
  *cols = h->m.cols;
}
void or_mat_copy(const or_mat* h, double* out) {
  if (!h->m.a.empty()) std::memcpy(out, h->m.a.data(), sizeof(double) * h->m.a.size());
}
void or_mat_free(or_mat* h) { delete h; }

// ---- rng / ordering / dense kernels
std::uint64_t or_mix_seed(std::uint64_t base, std::uint64_t salt) { return mix_seed(base, salt); }
std::uint64_t or_mix_seed3(std::uint64_t base, std::uint64_t a, std::uint64_t b) { return mix_seed(base, a, b); }

void or_mt_raw(std::uint64_t seed, std::int64_t count, std::uint64_t* out) {
  GaussianSampler g(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = g.raw();
}

void or_gaussian_matrix(std::uint64_t seed, std::int64_t rows, std::int64_t cols, double* out) {
  GaussianSampler g(seed);
  const Mat m = g.gaussian_matrix(rows, cols);
  if (!m.a.empty()) std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
}

void or_spectral_sort(std::int64_t n, const double* values, int order, std::int64_t* perm) {
  const auto p = spectral_sort(Vec(values, values + n), static_cast<SpectralOrder>(order));
  for (std::int64_t i = 0; i < n; ++i) perm[i] = p[static_cast<size_t>(i)];
}

int or_sym_eig(std::int64_t n, const double* s, int order, double* w, double* v, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const EigResult r = sym_eig_dense(mat_in(n, n, s), static_cast<SpectralOrder>(order));
    for (std::int64_t i = 0; i < n; ++i) w[i] = r.values[static_cast<size_t>(i)];
    if (n) std::memcpy(v, r.vectors.a.data(), sizeof(double) * static_cast<size_t>(n * n));
  });
}

int or_orthonormalize(std::int64_t rows, std::int64_t cols, const double* m, std::int64_t acols,
                      const double* against, double tol, or_mat** out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const Mat a = acols > 0 ? mat_in(rows, acols, against) : Mat(rows, 0);
    *out = new or_mat{orthonormalize(mat_in(rows, cols, m), a, tol)};
  });
}

int or_orthonormalize_shape_check(std::int64_t rows, std::int64_t cols, const double* m, std::int64_t arows,
                                  std::int64_t acols, const double* against, char* err, int errlen) {
  return guarded(err, errlen, [&] { orthonormalize(mat_in(rows, cols, m), mat_in(arows, acols, against)); });
}

int or_rsvd_dense(std::int64_t rows, std::int64_t cols, const double* b, std::int64_t l, std::int64_t p,
                  std::uint64_t seed, or_mat** out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *out = new or_mat{rsvd_basis(dense_operator(mat_in(rows, cols, b)), l, p, seed)}; });
}

double or_subspace_sin(std::int64_t rows, std::int64_t ca, const double* a, std::int64_t cb, const double* b) {
  return subspace_sin_largest_angle(mat_in(rows, ca, a), mat_in(rows, cb, b));
}

int or_lanczos(std::int64_t n, const std::int32_t* rowptr, const std::int32_t* col, const double* val,
               std::int64_t k, int order, std::uint64_t seed, double tol, std::int64_t max_basis, double* values,
               double* vectors, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    LanczosOptions lo;
    lo.k = k;
    lo.order = static_cast<SpectralOrder>(order);
    lo.seed = seed;
    lo.tol = tol;
    lo.max_basis = max_basis;
    const EigResult r = lanczos_topk_csr(csr_in(n, rowptr, col, val), lo);
    for (std::int64_t i = 0; i < k; ++i) values[i] = r.values[static_cast<size_t>(i)];
    std::memcpy(vectors, r.vectors.a.data(), sizeof(double) * static_cast<size_t>(n * k));
  });
}

// ---- graph
int or_from_edges(std::int64_t n, std::int64_t m, const std::int64_t* ei, const std::int64_t* ej, const double* ew,
                  or_csr** out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<std::tuple<Index, Index, double>> e;
    e.reserve(static_cast<size_t>(m));
    for (std::int64_t x = 0; x < m; ++x) e.emplace_back(ei[x], ej[x], ew ? ew[x] : 1.0);
    *out = new or_csr{from_edges(n, e)};
  });
}

int or_from_triplets(std::int64_t n, std::int64_t m, const std::int64_t* ti, const std::int64_t* tj,
                     const double* tv, or_csr** out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<Triplet> t;
    t.reserve(static_cast<size_t>(m));
    for (std::int64_t x = 0; x < m; ++x) t.push_back({ti[x], tj[x], tv[x]});
    *out = new or_csr{from_triplets(n, t)};
  });
}

int or_update_delta(std::int64_t n_old, std::int64_t n_add, const std::int64_t* ai, const std::int64_t* aj,
                    const double* aw, std::int64_t n_rem, const std::int64_t* ri, const std::int64_t* rj,
                    std::int64_t n_new_nodes, std::int64_t n_new_edges, const std::int64_t* ni,
                    const std::int64_t* nj, const double* nw, or_csr** out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const GraphUpdate d = update_in(n_old, n_add, ai, aj, aw, n_rem, ri, rj, n_new_nodes, n_new_edges, ni, nj, nw);
    *out = new or_csr{d.to_delta()};
  });
}

int or_apply_update(std::int64_t n, const std::int32_t* rowptr, const std::int32_t* col, const double* val,
                    std::int64_t n_add, const std::int64_t* ai, const std::int64_t* aj, const double* aw,
                    std::int64_t n_rem, const std::int64_t* ri, const std::int64_t* rj, std::int64_t n_new_nodes,
                    std::int64_t n_new_edges, const std::int64_t* ni, const std::int64_t* nj, const double* nw,
                    std::int64_t n_old_override, or_csr** out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const GraphUpdate d = update_in(n_old_override >= 0 ? n_old_override : n, n_add, ai, aj, aw, n_rem, ri, rj,
                                    n_new_nodes, n_new_edges, ni, nj, nw);
    *out = new or_csr{apply_update(csr_in(n, rowptr, col, val), d)};
  });
}

int or_shifted_laplacian(std::int64_t n, const std::int32_t* rowptr, const std::int32_t* col, const double* val,
                         int kind, double alpha, int* warned, or_csr** out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::string w;
    *out = new or_csr{to_shifted_laplacian(csr_in(n, rowptr, col, val), static_cast<LaplacianKind>(kind), alpha, &w)};
    *warned = w.empty() ? 0 : 1;
  });
}

// ---- sessions: the reference per-step loop (experiment.cpp:165-205) for one lane
int or_session_create(int kind, int op, std::int64_t k, int order, std::int64_t rsvd_l, std::int64_t rsvd_p,
                      std::uint64_t seed, std::int64_t n, const std::int32_t* rowptr, const std::int32_t* col,
                      const double* val, const double* values, const double* vectors, void** out, char* err,
                      int errlen) {
  return guarded(err, errlen, [&] {
    auto s = std::make_unique<Session>();
    s->op = op;
    Csr a = csr_in(n, rowptr, col, val);
    TrackerOptions o;
    o.k = k;
    o.order = static_cast<SpectralOrder>(order);
    o.rsvd_l = rsvd_l;
    o.rsvd_p = rsvd_p;
    o.seed = seed;
    const TrackerKind tk = kind_of(kind);
    if (op == 0) {
      s->a = std::move(a);
    } else {
      s->lap.emplace(std::move(a), op == 1 ? LaplacianKind::combinatorial : LaplacianKind::normalized);
    }
    const Csr& opmat = op == 0 ? s->a : s->lap->shifted();
    if (values) {
      if (k < 1 || k > n) throw std::invalid_argument("tracker_init: k must satisfy 1 <= k <= n");
      s->state.kind = tk;
      s->state.opts = o;
      s->state.values.assign(values, values + k);
      s->state.vectors = mat_in(n, k, vectors);
      s->state.n = n;
      double sq = 0.0;  // restart_scale = ||Lambda||_2 as tracker_init sets it (trackers.cpp:143)
      for (double v : s->state.values) sq += v * v;
      s->state.restart_scale = std::sqrt(sq);
    } else {
      s->state = tracker_init(opmat, tk, o);
    }
    *out = s.release();
  });
}

void or_session_destroy(void* h) { delete static_cast<Session*>(h); }

// TrackerOptions fields of the perturbation trackers and TIMERS (trackers.hpp:52-63)
int or_session_set_options(void* h, double mu, int trip_replace_span, double theta, std::int64_t min_restart_gap,
                           int restart_inner, char* err, int errlen) {
  Session* s = static_cast<Session*>(h);
  return guarded(err, errlen, [&] {
    if (s->state.kind == TrackerKind::timers && restart_inner == static_cast<int>(TrackerKind::timers))
      throw std::invalid_argument("tracker_init: timers cannot delegate to itself");
    (void)kind_of(restart_inner);
    s->state.opts.mu = mu;
    s->state.opts.trip_replace_span = trip_replace_span != 0;
    s->state.opts.theta = theta;
    s->state.opts.min_restart_gap = min_restart_gap;
    s->state.opts.restart_inner = restart_inner;
  });
}

void or_session_tracker_stats(void* h, double* accumulated_change, std::int64_t* steps_since_restart,
                              double* restart_scale, int* ridge_used) {
  Session* s = static_cast<Session*>(h);
  *accumulated_change = s->state.accumulated_change;
  *steps_since_restart = s->state.steps_since_restart;
  *restart_scale = s->state.restart_scale;
  *ridge_used = s->state.ridge_used ? 1 : 0;
}

int or_session_step(void* h, std::int64_t n_add, const std::int64_t* ai, const std::int64_t* aj, const double* aw,
                    std::int64_t n_rem, const std::int64_t* ri, const std::int64_t* rj, std::int64_t n_new_nodes,
                    std::int64_t n_new_edges, const std::int64_t* ni, const std::int64_t* nj, const double* nw,
                    double* tracker_seconds, char* err, int errlen) {
  Session* s = static_cast<Session*>(h);
  return guarded(err, errlen, [&] {
    const Index n_old = s->op == 0 ? s->a.rows : s->lap->adjacency().rows;
    const GraphUpdate d = update_in(n_old, n_add, ai, aj, aw, n_rem, ri, rj, n_new_nodes, n_new_edges, ni, nj, nw);
    Perturbation p;
    std::optional<Csr> a_next;
    std::optional<ShiftedLaplacianSession> lap_next;
    if (s->op == 0) {
      p = to_perturbation(d);
      a_next = apply_update(s->a, d);
    } else {
      lap_next = *s->lap;
      p = lap_next->advance(d);
    }
    const auto t0 = std::chrono::steady_clock::now();
    const Csr* provider = s->op == 0 ? &*a_next : &lap_next->shifted();  // the MatrixProvider
    TrackerState next = tracker_step(s->state, p, provider);
    const auto t1 = std::chrono::steady_clock::now();
    if (tracker_seconds) *tracker_seconds = std::chrono::duration<double>(t1 - t0).count();
    s->state = std::move(next);
    if (s->op == 0)
      s->a = std::move(*a_next);
    else
      s->lap = std::move(lap_next);
    s->last_delta = std::move(p.delta);
  });
}

void or_session_info(void* h, std::int64_t* n, std::int64_t* k, std::uint64_t* steps_taken, double* alpha) {
  Session* s = static_cast<Session*>(h);
  *n = s->state.n;
  *k = static_cast<std::int64_t>(s->state.values.size());
  *steps_taken = s->state.steps_taken;
  *alpha = s->op == 0 ? 0.0 : s->lap->alpha();
}

void or_session_embedding(void* h, double* values, double* vectors) {
  Session* s = static_cast<Session*>(h);
  std::memcpy(values, s->state.values.data(), sizeof(double) * s->state.values.size());
  std::memcpy(vectors, s->state.vectors.a.data(), sizeof(double) * s->state.vectors.a.size());
}

// which: 0 adjacency, 1 shifted operator T (Laplacian sessions), 2 last perturbation
or_csr* or_session_csr(void* h, int which) {
  Session* s = static_cast<Session*>(h);
  if (which == 2) return new or_csr{s->last_delta};
  if (s->op == 0) return new or_csr{s->a};
  return new or_csr{which == 0 ? s->lap->adjacency() : s->lap->shifted()};
}

// Projection basis the next step would build for this update (no state change).
int or_session_probe_basis(void* h, int basis_kind, std::uint64_t seed, std::int64_t n_add, const std::int64_t* ai,
                           const std::int64_t* aj, const double* aw, std::int64_t n_rem, const std::int64_t* ri,
                           const std::int64_t* rj, std::int64_t n_new_nodes, std::int64_t n_new_edges,
                           const std::int64_t* ni, const std::int64_t* nj, const double* nw, or_mat** out, char* err,
                           int errlen) {
  Session* s = static_cast<Session*>(h);
  return guarded(err, errlen, [&] {
    const Index n_old = s->op == 0 ? s->a.rows : s->lap->adjacency().rows;
    const GraphUpdate d = update_in(n_old, n_add, ai, aj, aw, n_rem, ri, rj, n_new_nodes, n_new_edges, ni, nj, nw);
    Perturbation p;
    if (s->op == 0) {
      p = to_perturbation(d);
    } else {
      ShiftedLaplacianSession tmp = *s->lap;
      p = tmp.advance(d);
    }
    *out = new or_mat{build_projection_basis(s->state, p, static_cast<BasisKind>(basis_kind), seed)};
  });
}

// Rayleigh-Ritz of the current state against a caller-supplied basis z for
// the given update (no state change). Returns the new values/vectors.
int or_session_probe_rr(void* h, std::int64_t zrows, std::int64_t zcols, const double* z, std::int64_t n_add,
                        const std::int64_t* ai, const std::int64_t* aj, const double* aw, std::int64_t n_rem,
                        const std::int64_t* ri, const std::int64_t* rj, std::int64_t n_new_nodes,
                        std::int64_t n_new_edges, const std::int64_t* ni, const std::int64_t* nj, const double* nw,
                        double* values, or_mat** vectors, char* err, int errlen) {
  Session* s = static_cast<Session*>(h);
  return guarded(err, errlen, [&] {
    const Index n_old = s->op == 0 ? s->a.rows : s->lap->adjacency().rows;
    const GraphUpdate d = update_in(n_old, n_add, ai, aj, aw, n_rem, ri, rj, n_new_nodes, n_new_edges, ni, nj, nw);
    const Perturbation p = to_perturbation(d);
    const TrackerState r = rayleigh_ritz_step(s->state, p, mat_in(zrows, zcols, z));
    std::memcpy(values, r.values.data(), sizeof(double) * r.values.size());
    *vectors = new or_mat{r.vectors};
  });
}

}  // extern "C"
