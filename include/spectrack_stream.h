/* spectrack_stream.h — C ABI of the stream generators and the binary
 * update-batch wire format (libspectrack_stream.so, host code, no CUDA).
 *
 * One seeded stream = an initial undirected graph plus a chain of update
 * batches in the edit-list form of assemble_update (proj/include/spectrack/
 * graph.hpp:65-69: added (i, j, w), removed (i, j), n_new, new_edges (i, j, w)).
 * The same file feeds the CUDA path (st_step / the C++ shim), the CPU oracle
 * and the bench, so every consumer sees identical inputs.
 *
 * Generators:
 *  - the reference's stream protocols, restated: sbm_sample_graph +
 *    sbm_dynamic_stream (dynamics.cpp:145-194), scenario1_stream /
 *    scenario2_stream (dynamics.cpp:62-143), all over expansion_stream
 *    (dynamics.cpp:25-59), with the reference's GaussianSampler draws
 *    (rng.hpp:16-43: mt19937_64, uniform = (x >> 11) 2^-53, uniform_index =
 *    x mod n) and its validation messages;
 *  - the BASELINE configurations (no reference generator exists for them):
 *    equal-block SBM / Erdos-Renyi by geometric skipping, R-MAT (symmetrized,
 *    self-loops dropped, deduplicated), and edit streams with uniform inserts
 *    over non-edges, uniform deletions, appended nodes with preferential-
 *    attachment edges (targets proportional to pre-step degree, the endpoint
 *    pool model of acceptance_main.cpp:527-564) and node removal as isolation.
 *
 * Wire format (little-endian, all fields 8 bytes):
 *   "STUB0001" | n0 | m0 | steps | flags (bit 0: node_origin, bit 1: labels)
 *   | name_len | name bytes padded to 8
 *   | m0 x (i, j, w)                       initial undirected edges, i < j
 *   | steps x { n_old | n_new | na | nr | nn | na x (i, j, w) | nr x (i, j)
 *               | nn x (i, j, w) }
 *   | [node_count x origin] | [node_count x label]
 * where i, j are int64 and w is float64.
 */
#ifndef SPECTRACK_STREAM_H
#define SPECTRACK_STREAM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sts_stream sts_stream;

/* status: 0 ok, 1 std::invalid_argument (reference message in sts_last_error), 2 I/O or format error */
const char* sts_last_error(void);
void sts_free(sts_stream* s);

/* --- the reference's protocols (dynamics.hpp) --- */
/* sbm_sample_graph (dynamics.cpp:145-166): labels (n) optional */
int32_t sts_sbm_sample_graph(int64_t n, int32_t k_clusters, double p_in, double p_out, uint64_t seed,
                             sts_stream** out);
/* sbm_dynamic_stream (dynamics.cpp:168-192) */
int32_t sts_sbm_dynamic(int64_t n, int32_t k_clusters, double p_in, double p_out, int64_t n0, int64_t t_steps,
                        int64_t s_per_step, uint64_t seed, sts_stream** out);
/* scenario1_stream (dynamics.cpp:62-80) of the graph with m undirected unit edges (i, j) */
int32_t sts_scenario1(int64_t n, const int64_t* ei, const int64_t* ej, int64_t m, int64_t t_steps, sts_stream** out);
/* scenario2_stream (dynamics.cpp:82-143) of a timestamped edge list */
int32_t sts_scenario2(int64_t n, const int64_t* u, const int64_t* v, const int64_t* t, int64_t m, int64_t t_steps,
                      int64_t m0, sts_stream** out);

/* --- BASELINE configurations (BASELINE.json configs[0..4]); scale/n/steps override the stated
 *     sizes when > 0 (tests), seed 0 = the config's default seed --- */
int32_t sts_config(int32_t which /* 1..5 */, int64_t size, int64_t steps, uint64_t seed, sts_stream** out);

/* --- wire format --- */
int32_t sts_save(const sts_stream* s, const char* path);
int32_t sts_load(const char* path, sts_stream** out);
/* a stream from arrays (e.g. a caller's own generator), to be saved */
int32_t sts_create(int64_t n0, const int64_t* i, const int64_t* j, const double* w, int64_t m0, const char* name,
                   sts_stream** out);
int32_t sts_append(sts_stream* s, int64_t n_new, const int64_t* ai, const int64_t* aj, const double* aw, int64_t na,
                   const int64_t* ri, const int64_t* rj, int64_t nr, const int64_t* ni, const int64_t* nj,
                   const double* nw, int64_t nn);

/* --- accessors --- */
int64_t sts_n0(const sts_stream* s);
int64_t sts_m0(const sts_stream* s);
int64_t sts_steps(const sts_stream* s);
const char* sts_name(const sts_stream* s);
int32_t sts_initial(const sts_stream* s, int64_t* i, int64_t* j, double* w);
/* initial graph as symmetric CSR (both triangles, sorted columns): rowptr n0 + 1, col / val 2 m0 */
int32_t sts_initial_csr(const sts_stream* s, int32_t* rowptr, int32_t* col, double* val);
int32_t sts_update_sizes(const sts_stream* s, int64_t t, int64_t* n_old, int64_t* n_new, int64_t* na, int64_t* nr,
                         int64_t* nn);
int32_t sts_update(const sts_stream* s, int64_t t, int64_t* ai, int64_t* aj, double* aw, int64_t* ri, int64_t* rj,
                   int64_t* ni, int64_t* nj, double* nw);
/* node_origin / labels of the reference protocols (count = final node count; 0 when absent) */
int64_t sts_node_count(const sts_stream* s);
int32_t sts_node_origin(const sts_stream* s, int64_t* origin);
int32_t sts_labels(const sts_stream* s, int32_t* labels);

#ifdef __cplusplus
}
#endif

#endif /* SPECTRACK_STREAM_H */
