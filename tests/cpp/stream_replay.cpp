// A C++ consumer of the update-batch wire format (include/spectrack_stream.h):
// reads a stream file, starts a device tracker from the initial graph
// (tracker_init, trackers.hpp:92) and replays every batch through
// tracker_step(state, assemble_update's edit lists) — the loop of
// run_stream_experiment (proj/src/experiment.cpp:159-173) — printing the
// leading Ritz values after each step.
// usage: stream_replay <file.stub> <k> [kind: grest-rsvd|grest2|iasc] [out.bin]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "spectrack_b200.hpp"
#include "spectrack_stream.h"

using namespace spectrack_b200;

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s <file.stub> <k> [kind] [values_out]\n", argv[0]);
    return 2;
  }
  sts_stream* s = nullptr;
  if (sts_load(argv[1], &s) != 0) {
    std::fprintf(stderr, "sts_load: %s\n", sts_last_error());
    return 1;
  }
  const Index k = std::atoll(argv[2]);
  const std::string kind = argc > 3 ? argv[3] : "grest-rsvd";
  Csr a0;
  a0.n = sts_n0(s);
  a0.row_offsets.assign(static_cast<size_t>(a0.n) + 1, 0);
  a0.col_indices.resize(static_cast<size_t>(2 * sts_m0(s)));
  a0.values.resize(a0.col_indices.size());
  if (sts_initial_csr(s, a0.row_offsets.data(), a0.col_indices.data(), a0.values.data()) != 0) {
    std::fprintf(stderr, "sts_initial_csr: %s\n", sts_last_error());
    return 1;
  }
  TrackerOptions opts;
  opts.k = k;
  const TrackerKind tk = kind == "grest2" ? TrackerKind::grest2 : kind == "iasc" ? TrackerKind::iasc
                                                                                 : TrackerKind::grest_rsvd;
  std::FILE* out = argc > 4 ? std::fopen(argv[4], "wb") : nullptr;
  try {
    GpuTracker t = tracker_init(a0, tk, opts);
    auto emit = [&](Index step) {
      const SpectralEmbedding e = t.embedding();
      std::printf("step %lld: n=%lld values[0]=%.17g values[k-1]=%.17g\n", static_cast<long long>(step),
                  static_cast<long long>(e.n), e.values.front(), e.values.back());
      if (out) std::fwrite(e.values.data(), sizeof(double), e.values.size(), out);
    };
    emit(-1);
    for (int64_t st = 0; st < sts_steps(s); ++st) {
      int64_t n_old, n_new, na, nr, nn;
      sts_update_sizes(s, st, &n_old, &n_new, &na, &nr, &nn);
      std::vector<int64_t> ai(na), aj(na), ri(nr), rj(nr), ni(nn), nj(nn);
      std::vector<double> aw(na), nw(nn);
      sts_update(s, st, ai.data(), aj.data(), aw.data(), ri.data(), rj.data(), ni.data(), nj.data(), nw.data());
      EditLists ed;
      for (int64_t q = 0; q < na; ++q) ed.added_edges.emplace_back(ai[q], aj[q], aw[q]);
      for (int64_t q = 0; q < nr; ++q) ed.removed_edges.emplace_back(ri[q], rj[q]);
      ed.new_node_count = n_new;
      for (int64_t q = 0; q < nn; ++q) ed.new_edges.emplace_back(ni[q], nj[q], nw[q]);
      tracker_step(t, ed);
      emit(st);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    sts_free(s);
    return 1;
  }
  if (out) std::fclose(out);
  sts_free(s);
  std::printf("stream_replay: ok\n");
  return 0;
}
