// Stream generators and the binary update-batch wire format behind
// include/spectrack_stream.h (host code; built as libspectrack_stream.so).
//
// Two families:
//  * the reference's stream protocols (proj/src/dynamics.cpp): expansion of a
//    fully sampled graph in an arrival order (expansion_stream, :25-59), the
//    degree-split and timestamp-replay scenarios (:62-143) and the dynamic SBM
//    (:145-194), with the reference's draws (GaussianSampler, rng.hpp:16-43)
//    and messages, so a seed gives the reference's stream;
//  * the BASELINE configurations, for which the reference has no generator:
//    equal-block SBM / ER by geometric skipping, R-MAT, and edit streams
//    (uniform inserts over non-edges, uniform deletions, appended nodes with
//    degree-proportional attachment, node removal as isolation).
// Every stream is stored in the edit-list form of assemble_update
// (graph.hpp:65-69) and can be written to / read from one binary file.
#include "../../include/spectrack_stream.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numeric>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_set>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#include <parallel/algorithm>
#endif

namespace {

using i64 = int64_t;
using u64 = uint64_t;

// ---- rng.hpp:16-43 (mix_seed, GaussianSampler's uniform draws)
u64 mix_seed(u64 base, u64 salt) {
  u64 z = base + 0x9e3779b97f4a7c15ULL * (salt + 0x632be59bd9b4e019ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Sampler {
  std::mt19937_64 gen;
  explicit Sampler(u64 seed) : gen(seed) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  i64 uniform_index(i64 n) { return static_cast<i64>(gen() % static_cast<u64>(n)); }
};

struct Edge {
  i64 i, j;
  double w;
};

struct Batch {
  i64 n_old = 0, n_new = 0;
  std::vector<Edge> added;
  std::vector<std::pair<i64, i64>> removed;
  std::vector<Edge> new_edges;
};

}  // namespace

struct sts_stream {
  i64 n0 = 0;
  std::vector<Edge> initial;  // undirected, i < j
  std::vector<Batch> updates;
  std::vector<i64> node_origin;
  std::vector<int32_t> labels;
  std::string name;
};

namespace {

thread_local std::string g_err;

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int32_t guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

inline u64 key(i64 a, i64 b) {
  const i64 lo = std::min(a, b), hi = std::max(a, b);
  return (static_cast<u64>(lo) << 32) | static_cast<u64>(hi);
}
inline i64 key_lo(u64 k) { return static_cast<i64>(k >> 32); }
inline i64 key_hi(u64 k) { return static_cast<i64>(k & 0xffffffffULL); }

// ---- an undirected graph as adjacency lists with sorted neighbours (the
// column order of the reference's CSR rows)
struct Graph {
  i64 n = 0;
  std::vector<i64> rp, col;
  std::vector<double> val;
};

// SymSparseMatrix::from_edges (sparse.cpp:25-45): range, self-loop and duplicate checks
Graph from_edges(i64 n, const std::vector<Edge>& edges) {
  std::set<std::pair<i64, i64>> seen;
  for (const Edge& e : edges) {
    if (e.i < 0 || e.j < 0 || e.i >= n || e.j >= n)
      throw InvalidArgument("SymSparseMatrix: edge endpoint out of range");
    if (e.i == e.j) throw InvalidArgument("SymSparseMatrix: self-loop rejected");
    if (!seen.insert({std::min(e.i, e.j), std::max(e.i, e.j)}).second)
      throw InvalidArgument("SymSparseMatrix: duplicate edge rejected");
  }
  Graph g;
  g.n = n;
  std::vector<std::tuple<i64, i64, double>> t;
  t.reserve(2 * edges.size());
  for (const Edge& e : edges)
    if (e.w != 0.0) {  // prune_zeros
      t.emplace_back(e.i, e.j, e.w);
      t.emplace_back(e.j, e.i, e.w);
    }
  std::sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
    return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b) : std::get<1>(a) < std::get<1>(b);
  });
  g.rp.assign(static_cast<size_t>(n) + 1, 0);
  for (const auto& x : t) ++g.rp[static_cast<size_t>(std::get<0>(x)) + 1];
  for (i64 r = 0; r < n; ++r) g.rp[r + 1] += g.rp[r];
  g.col.resize(t.size());
  g.val.resize(t.size());
  for (size_t q = 0; q < t.size(); ++q) {
    g.col[q] = std::get<1>(t[q]);
    g.val[q] = std::get<2>(t[q]);
  }
  return g;
}

std::vector<Edge> edges_of(const Graph& g) {
  std::vector<Edge> e;
  for (i64 r = 0; r < g.n; ++r)
    for (i64 q = g.rp[r]; q < g.rp[r + 1]; ++q)
      if (g.col[q] > r) e.push_back({r, g.col[q], g.val[q]});
  return e;
}

std::vector<i64> leftover_folded_batches(i64 total, i64 t_steps) {  // dynamics.cpp:14-19
  const i64 base = total / t_steps;
  std::vector<i64> b(static_cast<size_t>(t_steps), base);
  b.back() += total - base * t_steps;
  return b;
}

// expansion_stream (dynamics.cpp:25-59): the first n0 arrivals form the
// initial graph, each batch reveals the next nodes, and an edge appears in the
// step its later endpoint arrives (as a new_edges entry of assemble_update).
void expansion_stream(const Graph& g, const std::vector<i64>& order, i64 n0, const std::vector<i64>& batches,
                      sts_stream& s) {
  i64 used = n0;
  for (i64 b : batches) used += b;
  std::vector<i64> pos(static_cast<size_t>(g.n), -1);
  for (i64 i = 0; i < used; ++i) pos[static_cast<size_t>(order[i])] = i;
  auto emit = [&](i64 first, i64 last) {
    std::vector<Edge> out;
    for (i64 p = first; p <= last; ++p) {
      const i64 orig = order[static_cast<size_t>(p)];
      for (i64 q = g.rp[orig]; q < g.rp[orig + 1]; ++q) {
        const i64 qq = pos[static_cast<size_t>(g.col[q])];
        if (qq >= 0 && qq < p) out.push_back({qq, p, g.val[q]});
      }
    }
    return out;
  };
  s.n0 = n0;
  s.initial.clear();
  if (n0 > 0) s.initial = edges_of(from_edges(n0, emit(0, n0 - 1)));
  i64 current = n0;
  for (i64 b : batches) {
    Batch up;
    up.n_old = current;
    up.n_new = b;
    if (b > 0) up.new_edges = emit(current, current + b - 1);
    s.updates.push_back(std::move(up));
    current += b;
  }
  s.node_origin.assign(order.begin(), order.begin() + used);
}

std::vector<double> degrees(const Graph& g) {  // sparse.cpp:97-99: row sums
  std::vector<double> d(static_cast<size_t>(g.n), 0.0);
  for (i64 r = 0; r < g.n; ++r)
    for (i64 q = g.rp[r]; q < g.rp[r + 1]; ++q) d[r] += g.val[q];
  return d;
}

// sbm_sample_graph (dynamics.cpp:145-166)
Graph sbm_sample(i64 n, int k, double p_in, double p_out, u64 seed, std::vector<int32_t>* labels) {
  if (n < 1) throw InvalidArgument("n must be positive");
  if (k < 1) throw InvalidArgument("k_clusters must be positive");
  if (!(p_out >= 0.0 && p_out < p_in && p_in <= 1.0)) throw InvalidArgument("need 0 <= p_out < p_in <= 1");
  Sampler rng(mix_seed(seed, 0x5b31u));
  std::vector<int32_t> planted(static_cast<size_t>(n));
  for (auto& l : planted) l = static_cast<int32_t>(rng.uniform_index(k));
  std::vector<Edge> edges;
  for (i64 i = 0; i < n; ++i)
    for (i64 j = i + 1; j < n; ++j) {
      const double p = planted[i] == planted[j] ? p_in : p_out;
      if (rng.uniform() < p) edges.push_back({i, j, 1.0});
    }
  if (labels) *labels = std::move(planted);
  return from_edges(n, edges);
}

// ---------------------------------------------------------------- BASELINE generators
// Bernoulli(p) over the pairs of two node blocks by geometric skipping (O(edges)).
void sample_block_pairs(Sampler& rng, i64 lo_a, i64 sa, i64 lo_b, i64 sb, double p, bool same, std::vector<u64>& out) {
  const double total = same ? 0.5 * static_cast<double>(sa) * static_cast<double>(sa - 1)
                            : static_cast<double>(sa) * static_cast<double>(sb);
  if (total <= 0.0 || p <= 0.0) return;
  const double lq = p < 1.0 ? std::log1p(-p) : 0.0;
  double idx = -1.0;
  for (;;) {
    if (p >= 1.0) {
      idx += 1.0;
    } else {
      const double u = 1.0 - rng.uniform();  // (0, 1]
      idx += 1.0 + std::floor(std::log(u) / lq);
    }
    if (idx >= total) break;
    i64 i, j;
    if (same) {  // row-major upper-triangle index -> (i, j), i < j
      const double s = static_cast<double>(sa);
      i = static_cast<i64>(s - 2.0 - std::floor(std::sqrt(-8.0 * idx + 4.0 * s * (s - 1.0) - 7.0) / 2.0 - 0.5));
      const i64 k = static_cast<i64>(idx);
      j = k + i + 1 - sa * (sa - 1) / 2 + (sa - i) * ((sa - i) - 1) / 2;
      out.push_back(key(lo_a + i, lo_a + j));
    } else {
      const i64 k = static_cast<i64>(idx);
      i = k / sb;
      j = k % sb;
      out.push_back(key(lo_a + i, lo_b + j));
    }
  }
}

std::vector<u64> sbm_blocks(i64 n, int blocks, double p_in, double p_out, u64 seed) {
  Sampler rng(mix_seed(seed, 0x5b3a));
  std::vector<i64> b(static_cast<size_t>(blocks) + 1);
  for (int q = 0; q <= blocks; ++q) b[q] = n * q / blocks;
  std::vector<u64> keys;
  for (int x = 0; x < blocks; ++x)
    for (int y = x; y < blocks; ++y)
      sample_block_pairs(rng, b[x], b[x + 1] - b[x], b[y], b[y + 1] - b[y], x == y ? p_in : p_out, x == y, keys);
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  return keys;
}

// R-MAT (a, b, c, d) edges, symmetrized, self-loops dropped, deduplicated.
// The ef 2^scale draws are cut into 256 fixed chunks with seeds
// mix_seed(seed, chunk): the stream does not depend on the thread count.
std::vector<u64> rmat(int scale, int ef, double a, double b, double c, u64 seed) {
  const i64 m = static_cast<i64>(ef) << scale;
  constexpr int kChunks = 256;
  std::vector<std::vector<u64>> parts(kChunks);
#pragma omp parallel for schedule(dynamic, 1)
  for (int ch = 0; ch < kChunks; ++ch) {
    Sampler rng(mix_seed(seed, 0x7a7000 + ch));
    const i64 e0 = m * ch / kChunks, e1 = m * (ch + 1) / kChunks;
    auto& out = parts[ch];
    out.reserve(static_cast<size_t>(e1 - e0));
    for (i64 e = e0; e < e1; ++e) {
      i64 u = 0, v = 0;
      for (int lvl = 0; lvl < scale; ++lvl) {
        const double r = rng.uniform();
        const int sh = scale - 1 - lvl;
        const bool down = r >= a + b, right = (r >= a && r < a + b) || r >= a + b + c;
        u |= static_cast<i64>(down) << sh;
        v |= static_cast<i64>(right) << sh;
      }
      if (u != v) out.push_back(key(u, v));
    }
  }
  std::vector<u64> keys;
  for (auto& p : parts) {
    keys.insert(keys.end(), p.begin(), p.end());
    std::vector<u64>().swap(p);
  }
#ifdef _OPENMP
  __gnu_parallel::sort(keys.begin(), keys.end());
#else
  std::sort(keys.begin(), keys.end());
#endif
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  return keys;
}

// Evolving undirected edge set (sorted keys) with degrees.
struct EdgeSet {
  i64 n;
  std::vector<u64> keys;
  std::vector<i64> deg;
  EdgeSet(i64 n_, std::vector<u64> k) : n(n_), keys(std::move(k)), deg(static_cast<size_t>(n_), 0) {
    for (u64 x : keys) {
      ++deg[key_lo(x)];
      ++deg[key_hi(x)];
    }
  }
  bool has(u64 k) const { return std::binary_search(keys.begin(), keys.end(), k); }
  void apply(const std::vector<u64>& added, const std::vector<u64>& removed, i64 n_new) {
    std::vector<u64> rem(removed), add(added);
    std::sort(rem.begin(), rem.end());
    std::sort(add.begin(), add.end());
    std::vector<u64> kept;
    kept.reserve(keys.size());
    std::set_difference(keys.begin(), keys.end(), rem.begin(), rem.end(), std::back_inserter(kept));
    keys.clear();
    keys.reserve(kept.size() + add.size());
    std::merge(kept.begin(), kept.end(), add.begin(), add.end(), std::back_inserter(keys));
    n += n_new;
    deg.resize(static_cast<size_t>(n), 0);
    for (u64 x : rem) {
      --deg[key_lo(x)];
      --deg[key_hi(x)];
    }
    for (u64 x : add) {
      ++deg[key_lo(x)];
      ++deg[key_hi(x)];
    }
  }
};

// `count` distinct existing edges, uniform
std::vector<u64> sample_existing(Sampler& rng, const EdgeSet& es, i64 count) {
  std::unordered_set<i64> idx;
  std::vector<u64> out;
  const i64 m = static_cast<i64>(es.keys.size());
  count = std::min(count, m);
  while (static_cast<i64>(out.size()) < count) {
    const i64 q = rng.uniform_index(m);
    if (idx.insert(q).second) out.push_back(es.keys[q]);
  }
  return out;
}

// `count` distinct non-edges among nodes [0, n) avoiding `forbid` and `gone`
std::vector<u64> sample_absent(Sampler& rng, const EdgeSet& es, i64 count, const std::unordered_set<u64>& forbid,
                               const std::vector<char>* gone) {
  std::unordered_set<u64> got;
  std::vector<u64> out;
  while (static_cast<i64>(out.size()) < count) {
    const i64 u = rng.uniform_index(es.n), v = rng.uniform_index(es.n);
    if (u == v) continue;
    if (gone && ((*gone)[u] || (*gone)[v])) continue;
    const u64 k = key(u, v);
    if (es.has(k) || forbid.count(k) || !got.insert(k).second) continue;
    out.push_back(k);
  }
  return out;
}

// `deg_new` distinct targets per newcomer, proportional to the pre-step degree
// (the endpoint pool of acceptance_main.cpp:527-564: a node appears once per
// incident edge), uniform when the graph has no edge
std::vector<u64> attach_pa(Sampler& rng, const EdgeSet& es, i64 S, int deg_new) {
  std::vector<u64> cum(static_cast<size_t>(es.n));
  u64 tot = 0;
  for (i64 v = 0; v < es.n; ++v) {
    tot += static_cast<u64>(std::max<i64>(es.deg[v], 0));
    cum[v] = tot;
  }
  std::vector<u64> out;
  out.reserve(static_cast<size_t>(S * deg_new));
  std::vector<i64> chosen;
  for (i64 s = 0; s < S; ++s) {
    chosen.clear();
    const i64 want = std::min<i64>(deg_new, es.n);
    for (int tries = 0; static_cast<i64>(chosen.size()) < want && tries < 64 * deg_new; ++tries) {
      i64 t;
      if (tot == 0) {
        t = rng.uniform_index(es.n);
      } else {
        const u64 x = static_cast<u64>(rng.uniform_index(static_cast<i64>(tot)));
        t = std::upper_bound(cum.begin(), cum.end(), x) - cum.begin();
      }
      if (std::find(chosen.begin(), chosen.end(), t) == chosen.end()) chosen.push_back(t);
    }
    for (i64 t : chosen) out.push_back(key(t, es.n + s));
  }
  return out;
}

void push_batch(sts_stream& st, i64 n_old, i64 S, const std::vector<u64>& added, const std::vector<u64>& removed,
                const std::vector<u64>& new_keys) {
  Batch b;
  b.n_old = n_old;
  b.n_new = S;
  for (u64 k : added) b.added.push_back({key_lo(k), key_hi(k), 1.0});
  for (u64 k : removed) b.removed.push_back({key_lo(k), key_hi(k)});
  for (u64 k : new_keys) b.new_edges.push_back({key_lo(k), key_hi(k), 1.0});
  st.updates.push_back(std::move(b));
}

void set_initial(sts_stream& st, i64 n0, const std::vector<u64>& keys) {
  st.n0 = n0;
  st.initial.resize(keys.size());
  for (size_t q = 0; q < keys.size(); ++q) st.initial[q] = {key_lo(keys[q]), key_hi(keys[q]), 1.0};
}

// BASELINE.json configs[0..4] (sizes overridable for tests)
void config_stream(int which, i64 size, i64 steps, u64 seed, sts_stream& st) {
  if (seed == 0) seed = static_cast<u64>(which);
  Sampler rng(mix_seed(seed, 0xed17));
  char nm[64];
  if (which == 1 || which == 2) {
    // 1: SBM n = 10,000, 4 equal blocks, p_in 0.01, p_out 0.001; 500 inserts + 100 deletes per step
    // 2: ER n = 100,000, average degree 20; 1% inserts + 0.5% deletes (of the edges) per step
    const i64 n = size > 0 ? size : (which == 1 ? 10000 : 100000);
    const i64 T = steps > 0 ? steps : (which == 1 ? 10 : 20);
    std::vector<u64> k0 = which == 1 ? sbm_blocks(n, 4, 0.01, 0.001, seed) : sbm_blocks(n, 1, 20.0 / (n - 1), 0.0, seed);
    set_initial(st, n, k0);
    EdgeSet es(n, std::move(k0));
    for (i64 t = 0; t < T; ++t) {
      const i64 m = static_cast<i64>(es.keys.size());
      const i64 n_ins = which == 1 ? 500 : m / 100, n_del = which == 1 ? 100 : m / 200;
      std::vector<u64> removed = sample_existing(rng, es, n_del);
      std::unordered_set<u64> forbid(removed.begin(), removed.end());
      std::vector<u64> added = sample_absent(rng, es, n_ins, forbid, nullptr);
      push_batch(st, es.n, 0, added, removed, {});
      es.apply(added, removed, 0);
    }
    snprintf(nm, sizeof(nm), which == 1 ? "cfg1-sbm%lld" : "cfg2-er%lld", static_cast<long long>(n));
  } else if (which == 3 || which == 5) {
    // 3: R-MAT s20 ef16; per step 1% new nodes x 10 PA edges + 0.5% edge deletions
    // 5: R-MAT s25 ef16; per step 0.1% of the edges inserted + 0.1% new nodes x 16 PA edges
    const int scale = static_cast<int>(size > 0 ? size : (which == 3 ? 20 : 25));
    const i64 T = steps > 0 ? steps : (which == 3 ? 10 : 5);
    const i64 n = i64{1} << scale;
    std::vector<u64> k0 = rmat(scale, 16, 0.57, 0.19, 0.19, seed);
    set_initial(st, n, k0);
    EdgeSet es(n, std::move(k0));
    for (i64 t = 0; t < T; ++t) {
      const i64 m = static_cast<i64>(es.keys.size());
      const i64 S = which == 3 ? es.n / 100 : es.n / 1000;
      std::vector<u64> removed, added;
      if (which == 3) removed = sample_existing(rng, es, m / 200);
      if (which == 5) added = sample_absent(rng, es, m / 1000, {}, nullptr);
      std::vector<u64> nk = attach_pa(rng, es, S, which == 3 ? 10 : 16);
      push_batch(st, es.n, S, added, removed, nk);
      std::vector<u64> all(added);
      all.insert(all.end(), nk.begin(), nk.end());
      es.apply(all, removed, S);
    }
    snprintf(nm, sizeof(nm), "cfg%d-rmat-s%d", which, scale);
  } else if (which == 4) {
    // SBM n = 2^22, 64 equal blocks, average degree 32 with 80% intra-block; per step
    // 1% inserts, 0.5% deletes, 0.5% n new nodes x 16 edges (80% into one random block),
    // 0.1% n node removals as isolation (all incident edges deleted, the id kept)
    const i64 n = size > 0 ? size : (i64{1} << 22);
    const i64 T = steps > 0 ? steps : 10;
    const int blocks = 64;
    const i64 bs = n / blocks;
    std::vector<u64> k0 = sbm_blocks(n, blocks, 32.0 * 0.8 / (bs - 1), 32.0 * 0.2 / (n - bs), seed);
    set_initial(st, n, k0);
    EdgeSet es(n, std::move(k0));
    for (i64 t = 0; t < T; ++t) {
      const i64 m = static_cast<i64>(es.keys.size()), cur = es.n;
      std::vector<char> gone(static_cast<size_t>(cur), 0);
      for (i64 q = 0; q < std::max<i64>(1, cur / 1000); ++q) gone[rng.uniform_index(cur)] = 1;
      std::vector<u64> removed;
      for (u64 k : es.keys)
        if (gone[key_lo(k)] || gone[key_hi(k)]) removed.push_back(k);
      std::unordered_set<u64> forbid(removed.begin(), removed.end());
      for (u64 k : sample_existing(rng, es, m / 200))
        if (forbid.insert(k).second) removed.push_back(k);
      std::vector<u64> added = sample_absent(rng, es, m / 100, forbid, &gone);
      const i64 S = cur / 200;
      std::vector<u64> nk;
      std::vector<i64> chosen;
      for (i64 s = 0; s < S; ++s) {
        const i64 blk = rng.uniform_index(blocks);
        chosen.clear();
        for (int tries = 0; chosen.size() < 16 && tries < 1024; ++tries) {
          const i64 tgt = rng.uniform() < 0.8 ? blk * bs + rng.uniform_index(bs) : rng.uniform_index(cur);
          if (gone[tgt] || std::find(chosen.begin(), chosen.end(), tgt) != chosen.end()) continue;
          chosen.push_back(tgt);
        }
        for (i64 tg : chosen) nk.push_back(key(tg, cur + s));
      }
      push_batch(st, cur, S, added, removed, nk);
      std::vector<u64> all(added);
      all.insert(all.end(), nk.begin(), nk.end());
      es.apply(all, removed, S);
    }
    snprintf(nm, sizeof(nm), "cfg4-sbm%lld", static_cast<long long>(n));
  } else {
    throw InvalidArgument("sts_config: config must be 1..5");
  }
  st.name = nm;
}

// ---------------------------------------------------------------- wire format
constexpr char kMagic[8] = {'S', 'T', 'U', 'B', '0', '0', '0', '1'};

struct File {
  FILE* f;
  explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {
    if (!f) throw IoError(std::string("sts: cannot open ") + path);
  }
  ~File() {
    if (f) std::fclose(f);
  }
  void w(const void* p, size_t n) {
    if (n && std::fwrite(p, 1, n, f) != n) throw IoError("sts: write failed");
  }
  void r(void* p, size_t n) {
    if (n && std::fread(p, 1, n, f) != n) throw IoError("sts: truncated file");
  }
  void w64(i64 x) { w(&x, 8); }
  i64 r64() {
    i64 x;
    r(&x, 8);
    return x;
  }
};

void write_edges(File& f, const std::vector<Edge>& e) {
  std::vector<i64> buf(3 * e.size());
  for (size_t q = 0; q < e.size(); ++q) {
    buf[3 * q] = e[q].i;
    buf[3 * q + 1] = e[q].j;
    std::memcpy(&buf[3 * q + 2], &e[q].w, 8);
  }
  f.w(buf.data(), 8 * buf.size());
}

void read_edges(File& f, std::vector<Edge>& e, i64 n) {
  if (n < 0 || n > (i64{1} << 40)) throw IoError("sts: corrupt edge count");
  std::vector<i64> buf(3 * static_cast<size_t>(n));
  f.r(buf.data(), 8 * buf.size());
  e.resize(static_cast<size_t>(n));
  for (i64 q = 0; q < n; ++q) {
    e[q].i = buf[3 * q];
    e[q].j = buf[3 * q + 1];
    std::memcpy(&e[q].w, &buf[3 * q + 2], 8);
  }
}

i64 node_count(const sts_stream& s) {
  i64 n = s.n0;
  for (const Batch& b : s.updates) n += b.n_new;
  return n;
}

void save(const sts_stream& s, const char* path) {
  File f(path, "wb");
  f.w(kMagic, 8);
  f.w64(s.n0);
  f.w64(static_cast<i64>(s.initial.size()));
  f.w64(static_cast<i64>(s.updates.size()));
  f.w64((s.node_origin.empty() ? 0 : 1) | (s.labels.empty() ? 0 : 2));
  f.w64(static_cast<i64>(s.name.size()));
  std::vector<char> nm(s.name.begin(), s.name.end());
  nm.resize((nm.size() + 7) / 8 * 8, '\0');
  f.w(nm.data(), nm.size());
  write_edges(f, s.initial);
  for (const Batch& b : s.updates) {
    f.w64(b.n_old);
    f.w64(b.n_new);
    f.w64(static_cast<i64>(b.added.size()));
    f.w64(static_cast<i64>(b.removed.size()));
    f.w64(static_cast<i64>(b.new_edges.size()));
    write_edges(f, b.added);
    std::vector<i64> rm(2 * b.removed.size());
    for (size_t q = 0; q < b.removed.size(); ++q) {
      rm[2 * q] = b.removed[q].first;
      rm[2 * q + 1] = b.removed[q].second;
    }
    f.w(rm.data(), 8 * rm.size());
    write_edges(f, b.new_edges);
  }
  if (!s.node_origin.empty()) f.w(s.node_origin.data(), 8 * s.node_origin.size());
  if (!s.labels.empty()) {
    std::vector<i64> l(s.labels.begin(), s.labels.end());
    f.w(l.data(), 8 * l.size());
  }
}

void load(const char* path, sts_stream& s) {
  File f(path, "rb");
  char mg[8];
  f.r(mg, 8);
  if (std::memcmp(mg, kMagic, 8) != 0) throw IoError("sts: not an update-batch stream (bad magic)");
  s.n0 = f.r64();
  const i64 m0 = f.r64(), steps = f.r64(), flags = f.r64(), nl = f.r64();
  if (s.n0 < 0 || steps < 0 || nl < 0 || nl > 4096) throw IoError("sts: corrupt header");
  std::vector<char> nm(static_cast<size_t>((nl + 7) / 8 * 8));
  f.r(nm.data(), nm.size());
  s.name.assign(nm.data(), static_cast<size_t>(nl));
  read_edges(f, s.initial, m0);
  s.updates.resize(static_cast<size_t>(steps));
  for (Batch& b : s.updates) {
    b.n_old = f.r64();
    b.n_new = f.r64();
    const i64 na = f.r64(), nr = f.r64(), nn = f.r64();
    read_edges(f, b.added, na);
    if (nr < 0 || nr > (i64{1} << 40)) throw IoError("sts: corrupt edge count");
    std::vector<i64> rm(2 * static_cast<size_t>(nr));
    f.r(rm.data(), 8 * rm.size());
    b.removed.resize(static_cast<size_t>(nr));
    for (i64 q = 0; q < nr; ++q) b.removed[q] = {rm[2 * q], rm[2 * q + 1]};
    read_edges(f, b.new_edges, nn);
  }
  const i64 nc = node_count(s);
  if (flags & 1) {
    s.node_origin.resize(static_cast<size_t>(nc));
    f.r(s.node_origin.data(), 8 * s.node_origin.size());
  }
  if (flags & 2) {
    std::vector<i64> l(static_cast<size_t>(nc));
    f.r(l.data(), 8 * l.size());
    s.labels.assign(l.begin(), l.end());
  }
}

int32_t make(sts_stream** out, const std::function<void(sts_stream&)>& fill) {
  *out = nullptr;
  auto* s = new sts_stream();
  const int32_t rc = guarded([&]() { fill(*s); });
  if (rc != 0) {
    delete s;
    return rc;
  }
  *out = s;
  return 0;
}

}  // namespace

extern "C" {

const char* sts_last_error(void) { return g_err.c_str(); }
void sts_free(sts_stream* s) { delete s; }

int32_t sts_sbm_sample_graph(int64_t n, int32_t k, double p_in, double p_out, uint64_t seed, sts_stream** out) {
  return make(out, [&](sts_stream& s) {
    const Graph g = sbm_sample(n, k, p_in, p_out, seed, &s.labels);
    s.n0 = n;
    s.initial = edges_of(g);
    s.node_origin.resize(static_cast<size_t>(n));
    std::iota(s.node_origin.begin(), s.node_origin.end(), i64{0});
    s.name = "sbm_sample_graph";
  });
}

// sbm_dynamic_stream (dynamics.cpp:168-192)
int32_t sts_sbm_dynamic(int64_t n, int32_t k, double p_in, double p_out, int64_t n0, int64_t t_steps,
                        int64_t s_per_step, uint64_t seed, sts_stream** out) {
  return make(out, [&](sts_stream& s) {
    if (n0 < 1) throw InvalidArgument("n0 must be positive");
    if (t_steps < 1) throw InvalidArgument("t_steps must be positive");
    if (s_per_step < 0) throw InvalidArgument("s_per_step must be nonnegative");
    if (n0 + t_steps * s_per_step > n) throw InvalidArgument("stream needs more nodes than the model has");
    std::vector<int32_t> labels;
    const Graph g = sbm_sample(n, k, p_in, p_out, seed, &labels);
    Sampler rng(mix_seed(seed, 0x0a77u));
    std::vector<i64> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), i64{0});
    for (i64 i = n - 1; i > 0; --i) std::swap(order[i], order[rng.uniform_index(i + 1)]);
    expansion_stream(g, order, n0, std::vector<i64>(static_cast<size_t>(t_steps), s_per_step), s);
    s.labels.clear();
    for (i64 o : s.node_origin) s.labels.push_back(labels[static_cast<size_t>(o)]);
    s.name = "sbm_dynamic_stream";
  });
}

// scenario1_stream (dynamics.cpp:62-80)
int32_t sts_scenario1(int64_t n, const int64_t* ei, const int64_t* ej, int64_t m, int64_t t_steps, sts_stream** out) {
  return make(out, [&](sts_stream& s) {
    std::vector<Edge> e(static_cast<size_t>(m));
    for (i64 q = 0; q < m; ++q) e[q] = {ei[q], ej[q], 1.0};
    const Graph g = from_edges(n, e);
    if (t_steps < 1) throw InvalidArgument("t_steps must be positive");
    const i64 n0 = n / 2;
    if (n0 < 1) throw InvalidArgument("graph too small to split");
    const i64 remaining = n - n0;
    if (t_steps > remaining) throw InvalidArgument("more steps than nodes left to add");
    const std::vector<double> deg = degrees(g);
    std::vector<i64> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), i64{0});
    std::stable_sort(order.begin(), order.end(), [&](i64 a, i64 b) { return deg[a] > deg[b]; });
    expansion_stream(g, order, n0, leftover_folded_batches(remaining, t_steps), s);
    s.name = "scenario1_stream";
  });
}

// scenario2_stream (dynamics.cpp:82-143)
int32_t sts_scenario2(int64_t n, const int64_t* u, const int64_t* v, const int64_t* t, int64_t m, int64_t t_steps,
                      int64_t m0, sts_stream** out) {
  return make(out, [&](sts_stream& s) {
    if (t_steps < 1) throw InvalidArgument("t_steps must be positive");
    std::vector<size_t> idx(static_cast<size_t>(m));
    std::iota(idx.begin(), idx.end(), size_t{0});
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return t[a] < t[b]; });
    std::set<std::pair<i64, i64>> seen;
    std::vector<std::pair<i64, i64>> uniq;
    std::vector<i64> compact(static_cast<size_t>(n), -1), origin, nodes_after;
    for (size_t i : idx) {
      const i64 a = u[i], b = v[i];
      if (a == b) continue;
      if (a < 0 || b < 0 || a >= n || b >= n) throw InvalidArgument("edge endpoint out of range");
      if (!seen.insert({std::min(a, b), std::max(a, b)}).second) continue;
      for (i64 ep : {a, b})
        if (compact[ep] < 0) {
          compact[ep] = static_cast<i64>(origin.size());
          origin.push_back(ep);
        }
      uniq.emplace_back(compact[a], compact[b]);
      nodes_after.push_back(static_cast<i64>(origin.size()));
    }
    const i64 total = static_cast<i64>(uniq.size());
    if (m0 < 1 || m0 > total) throw InvalidArgument("m0 must be within the unique edge count");
    const i64 n0 = nodes_after[m0 - 1];
    std::vector<Edge> e0;
    for (i64 q = 0; q < m0; ++q) e0.push_back({uniq[q].first, uniq[q].second, 1.0});
    s.n0 = n0;
    s.initial = edges_of(from_edges(n0, e0));
    i64 consumed = m0, current = n0;
    for (i64 b : leftover_folded_batches(total - m0, t_steps)) {
      const i64 upto = consumed + b;
      const i64 next_n = b > 0 ? nodes_after[upto - 1] : current;
      Batch up;
      up.n_old = current;
      up.n_new = next_n - current;
      for (i64 e = consumed; e < upto; ++e) {
        const auto [a, c] = uniq[e];
        if (a < current && c < current) up.added.push_back({std::min(a, c), std::max(a, c), 1.0});
        else up.new_edges.push_back({a, c, 1.0});
      }
      s.updates.push_back(std::move(up));
      current = next_n;
      consumed = upto;
    }
    s.node_origin = std::move(origin);
    s.name = "scenario2_stream";
  });
}

int32_t sts_config(int32_t which, int64_t size, int64_t steps, uint64_t seed, sts_stream** out) {
  return make(out, [&](sts_stream& s) { config_stream(which, size, steps, seed, s); });
}

int32_t sts_save(const sts_stream* s, const char* path) { return guarded([&]() { save(*s, path); }); }
int32_t sts_load(const char* path, sts_stream** out) { return make(out, [&](sts_stream& s) { load(path, s); }); }

int32_t sts_create(int64_t n0, const int64_t* i, const int64_t* j, const double* w, int64_t m0, const char* name,
                   sts_stream** out) {
  return make(out, [&](sts_stream& s) {
    if (n0 < 0 || m0 < 0) throw InvalidArgument("sts_create: negative size");
    s.n0 = n0;
    s.initial.resize(static_cast<size_t>(m0));
    for (i64 q = 0; q < m0; ++q) s.initial[q] = {i[q], j[q], w ? w[q] : 1.0};
    s.name = name ? name : "";
  });
}

int32_t sts_append(sts_stream* s, int64_t n_new, const int64_t* ai, const int64_t* aj, const double* aw, int64_t na,
                   const int64_t* ri, const int64_t* rj, int64_t nr, const int64_t* ni, const int64_t* nj,
                   const double* nw, int64_t nn) {
  return guarded([&]() {
    if (n_new < 0 || na < 0 || nr < 0 || nn < 0) throw InvalidArgument("sts_append: negative size");
    Batch b;
    b.n_old = node_count(*s);
    b.n_new = n_new;
    for (i64 q = 0; q < na; ++q) b.added.push_back({ai[q], aj[q], aw ? aw[q] : 1.0});
    for (i64 q = 0; q < nr; ++q) b.removed.push_back({ri[q], rj[q]});
    for (i64 q = 0; q < nn; ++q) b.new_edges.push_back({ni[q], nj[q], nw ? nw[q] : 1.0});
    s->updates.push_back(std::move(b));
  });
}

int64_t sts_n0(const sts_stream* s) { return s->n0; }
int64_t sts_m0(const sts_stream* s) { return static_cast<int64_t>(s->initial.size()); }
int64_t sts_steps(const sts_stream* s) { return static_cast<int64_t>(s->updates.size()); }
const char* sts_name(const sts_stream* s) { return s->name.c_str(); }

int32_t sts_initial(const sts_stream* s, int64_t* i, int64_t* j, double* w) {
  for (size_t q = 0; q < s->initial.size(); ++q) {
    i[q] = s->initial[q].i;
    j[q] = s->initial[q].j;
    if (w) w[q] = s->initial[q].w;
  }
  return 0;
}

int32_t sts_initial_csr(const sts_stream* s, int32_t* rowptr, int32_t* col, double* val) {
  return guarded([&]() {
    const Graph g = from_edges(s->n0, s->initial);
    if (g.rp.back() > INT32_MAX) throw InvalidArgument("sts_initial_csr: more than 2^31 stored entries");
    for (size_t r = 0; r < g.rp.size(); ++r) rowptr[r] = static_cast<int32_t>(g.rp[r]);
    for (size_t q = 0; q < g.col.size(); ++q) {
      col[q] = static_cast<int32_t>(g.col[q]);
      val[q] = g.val[q];
    }
  });
}

int32_t sts_update_sizes(const sts_stream* s, int64_t t, int64_t* n_old, int64_t* n_new, int64_t* na, int64_t* nr,
                         int64_t* nn) {
  if (t < 0 || t >= static_cast<int64_t>(s->updates.size())) {
    g_err = "sts_update_sizes: step out of range";
    return 1;
  }
  const Batch& b = s->updates[t];
  *n_old = b.n_old;
  *n_new = b.n_new;
  *na = static_cast<int64_t>(b.added.size());
  *nr = static_cast<int64_t>(b.removed.size());
  *nn = static_cast<int64_t>(b.new_edges.size());
  return 0;
}

int32_t sts_update(const sts_stream* s, int64_t t, int64_t* ai, int64_t* aj, double* aw, int64_t* ri, int64_t* rj,
                   int64_t* ni, int64_t* nj, double* nw) {
  if (t < 0 || t >= static_cast<int64_t>(s->updates.size())) {
    g_err = "sts_update: step out of range";
    return 1;
  }
  const Batch& b = s->updates[t];
  for (size_t q = 0; q < b.added.size(); ++q) {
    ai[q] = b.added[q].i;
    aj[q] = b.added[q].j;
    aw[q] = b.added[q].w;
  }
  for (size_t q = 0; q < b.removed.size(); ++q) {
    ri[q] = b.removed[q].first;
    rj[q] = b.removed[q].second;
  }
  for (size_t q = 0; q < b.new_edges.size(); ++q) {
    ni[q] = b.new_edges[q].i;
    nj[q] = b.new_edges[q].j;
    nw[q] = b.new_edges[q].w;
  }
  return 0;
}

int64_t sts_node_count(const sts_stream* s) {
  return s->node_origin.empty() && s->labels.empty() ? 0 : node_count(*s);
}
int32_t sts_node_origin(const sts_stream* s, int64_t* origin) {
  std::copy(s->node_origin.begin(), s->node_origin.end(), origin);
  return 0;
}
int32_t sts_labels(const sts_stream* s, int32_t* labels) {
  std::copy(s->labels.begin(), s->labels.end(), labels);
  return 0;
}

}  // extern "C"
