// Exercises the reference-facing C++ shim (include/spectrack_b200.hpp) the way
// a reference caller would: the Fig. 1 update of proj/tests/test_sparse_graph.cpp
// (bitwise CSR), an invalid deletion (reference message, state untouched), and
// tracker_step on the device-resident state.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "spectrack_b200.hpp"

using namespace spectrack_b200;

static int failures = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #cond, __LINE__); \
      ++failures;                                                    \
    }                                                                \
  } while (0)

static Csr from_edges(Index n, const std::vector<std::pair<Index, Index>>& edges) {
  std::vector<std::vector<Index>> adj(static_cast<size_t>(n));
  for (auto [i, j] : edges) {
    adj[static_cast<size_t>(i)].push_back(j);
    adj[static_cast<size_t>(j)].push_back(i);
  }
  Csr m;
  m.n = n;
  for (Index r = 0; r < n; ++r) {
    auto& row = adj[static_cast<size_t>(r)];
    std::sort(row.begin(), row.end());
    for (Index c : row) {
      m.col_indices.push_back(static_cast<std::int32_t>(c));
      m.values.push_back(1.0);
    }
    m.row_offsets.push_back(static_cast<std::int32_t>(m.col_indices.size()));
  }
  return m;
}

int main() {
  // cycle with chord (test_sparse_graph.cpp:122-124)
  const Csr a0 = from_edges(6, {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 0}, {1, 4}});
  // initial embedding: any orthonormal pair (the API takes X0, Lambda0 as input)
  SpectralEmbedding x0;
  x0.n = 6;
  x0.values = {3.0, -2.0};
  x0.vectors.assign(12, 0.0);
  for (int i = 0; i < 6; ++i) {
    x0.vectors[static_cast<size_t>(i)] = 1.0 / std::sqrt(6.0);
    x0.vectors[static_cast<size_t>(6 + i)] = (i % 2 ? -1.0 : 1.0) / std::sqrt(6.0);
  }
  TrackerOptions opts;
  opts.k = 2;
  GpuTracker t(a0, TrackerKind::grest2, opts, OperatorKind::adjacency, x0);

  // invalid deletion: reference message, state unchanged
  EditLists bad;
  bad.removed_edges = {{0, 3}};
  bool threw = false;
  try {
    tracker_step(t, bad);
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("invalid deletion") != std::string::npos;
    if (!threw) std::fprintf(stderr, "unexpected message: %s\n", e.what());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "unexpected exception: %s\n", e.what());
  }
  CHECK(threw);
  CHECK(t.steps_taken() == 0 && t.n() == 6);

  // Fig. 1 update (test_sparse_graph.cpp:117-120)
  EditLists fig1;
  fig1.added_edges = {{0, 2, 1.0}, {2, 4, 1.0}};
  fig1.removed_edges = {{1, 4}};
  fig1.new_node_count = 2;
  fig1.new_edges = {{2, 6, 1.0}, {3, 6, 1.0}, {3, 7, 1.0}, {4, 7, 1.0}};
  tracker_step(t, fig1);
  const Csr a1 = t.csr(0);
  const Csr want = from_edges(8, {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 0}, {0, 2}, {2, 4}, {2, 6}, {3, 6},
                                  {3, 7}, {4, 7}});
  CHECK(a1.row_offsets == want.row_offsets);
  CHECK(a1.col_indices == want.col_indices);
  CHECK(a1.values == want.values);
  CHECK(t.n() == 8 && t.steps_taken() == 1);
  const SpectralEmbedding e = t.embedding();
  double gram_err = 0.0;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double s = 0.0;
      for (int i = 0; i < 8; ++i) s += e.vectors[static_cast<size_t>(a * 8 + i)] * e.vectors[static_cast<size_t>(b * 8 + i)];
      gram_err = std::fmax(gram_err, std::fabs(s - (a == b ? 1.0 : 0.0)));
    }
  CHECK(gram_err < 1e-12);
  // sym_eig_dense on diag(3, 1, 2) (test_linalg.cpp:30-39)
  auto [w, v] = sym_eig_dense({3, 0, 0, 0, 1, 0, 0, 0, 2}, 3, SpectralOrder::abs_desc, 3);
  CHECK(std::fabs(w[0] - 3) < 1e-14 && std::fabs(w[1] - 2) < 1e-14 && std::fabs(w[2] - 1) < 1e-14);
  // tracker_init on the device (trackers.cpp:132-145): K3 has eigenvalues 2, -1, -1
  {
    const Csr k3 = from_edges(3, {{0, 1}, {1, 2}, {0, 2}});
    TrackerOptions o3;
    o3.k = 1;
    GpuTracker ti = tracker_init(k3, TrackerKind::grest2, o3);
    const SpectralEmbedding e3 = ti.embedding();
    CHECK(std::fabs(e3.values[0] - 2.0) < 1e-12);
  }
  // the same Fig. 1 update as GraphUpdate blocks (graph.hpp:23-37): identical CSR
  {
    GpuTracker tb(a0, TrackerKind::grest2, opts, OperatorKind::adjacency, x0);
    GraphUpdate g;
    g.n_old = 6;
    g.n_new = 2;
    auto block = [](Index rows, Index cols, std::vector<std::tuple<Index, Index, double>> e) {
      std::sort(e.begin(), e.end());
      BlockCsr b;
      b.rows = rows;
      b.cols = cols;
      b.row_offsets.assign(static_cast<size_t>(rows + 1), 0);
      for (auto& [i, j, w] : e) {
        b.col_indices.push_back(static_cast<std::int32_t>(j));
        b.values.push_back(w);
        ++b.row_offsets[static_cast<size_t>(i + 1)];
      }
      for (Index r = 0; r < rows; ++r) b.row_offsets[static_cast<size_t>(r + 1)] += b.row_offsets[static_cast<size_t>(r)];
      return b;
    };
    g.k_block = block(6, 6, {{0, 2, 1.0}, {2, 0, 1.0}, {2, 4, 1.0}, {4, 2, 1.0}, {1, 4, -1.0}, {4, 1, -1.0}});
    g.g_block = block(6, 2, {{2, 0, 1.0}, {3, 0, 1.0}, {3, 1, 1.0}, {4, 1, 1.0}});
    g.c_block = block(2, 2, {});
    tracker_step(tb, g);
    const Csr b1 = tb.csr(0);
    CHECK(b1.row_offsets == a1.row_offsets && b1.col_indices == a1.col_indices && b1.values == a1.values);
    const SpectralEmbedding eb = tb.embedding();
    CHECK(eb.values == e.values && eb.vectors == e.vectors);
  }
  std::printf(failures ? "shim_smoke: %d failures\n" : "shim_smoke: ok\n", failures);
  return failures ? 1 : 0;
}
