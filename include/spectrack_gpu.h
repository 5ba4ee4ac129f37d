/* spectrack_gpu.h — C ABI of the B200-native G-REST per-step eigen-update.
 *
 * Drop-in boundary for the reference library `spectrack` (arxiv 2603.19439,
 * proj/include/spectrack). The reference has no C ABI: its callers link the C++
 * functions cited below. Each entry point here replaces one of them; the C++
 * shim include/spectrack_b200.hpp re-exposes the reference signatures on top
 * of this ABI (see INTEGRATION.md for the binding a maintainer adds).
 *
 * Conventions: plain pointers and sizes, no C++ or torch types. CSR arrays are
 * int32 offsets / int32 column indices / fp64 values (Eigen::SparseMatrix<
 * double, RowMajor>, sparse.hpp:18). Dense matrices cross the boundary
 * column-major with a leading dimension (Eigen's default). Node ids are int64
 * (Eigen::Index). Every function returns an st_status; on failure
 * st_last_error() holds the reference's exception message, and the session is
 * left exactly as before the call (the reference's value semantics).
 */
#ifndef SPECTRACK_GPU_H
#define SPECTRACK_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ST_OK = 0,
  ST_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  ST_RUNTIME_ERROR = 2,    /* std::runtime_error in the reference */
  ST_CUDA_ERROR = 3,       /* device failure (no reference counterpart) */
  ST_OTHER = 4
} st_status;

/* TrackerKind (trackers.hpp:36-45). */
typedef enum {
  ST_TRIP_BASIC = 0,
  ST_TRIP = 1,
  ST_RESIDUAL_MODES = 2,
  ST_IASC = 3,
  ST_GREST2 = 4,
  ST_GREST3 = 5,
  ST_GREST_RSVD = 6,
  ST_TIMERS = 7
} st_tracker_kind;

/* TrackerOptions fields of the perturbation trackers and TIMERS
 * (trackers.hpp:52-63); reference defaults {0, 0, 0.01, 5, ST_IASC}. */
typedef struct {
  double mu;                /* residual-modes denominator scalar */
  int32_t trip_replace_span; /* TRIP: x = X b instead of x = x + X b */
  double theta;             /* TIMERS restart threshold */
  int64_t min_restart_gap;  /* TIMERS minimum steps between restarts */
  int32_t restart_inner;    /* the kind TIMERS delegates to */
} st_tracker_options;
/* BasisKind (trackers.hpp:104) */
typedef enum { ST_BASIS_IASC = 0, ST_BASIS_GREST2 = 1, ST_BASIS_GREST3 = 2, ST_BASIS_GREST_RSVD = 3 } st_basis_kind;
/* SpectralOrder (types.hpp:22) */
typedef enum { ST_ABS_DESC = 0, ST_ALG_DESC = 1 } st_order;
/* OperatorKind (laplacian_track.hpp:14) */
typedef enum { ST_ADJACENCY = 0, ST_LAPLACIAN = 1, ST_NORMALIZED_LAPLACIAN = 2 } st_operator;

/* TrackerOptions (trackers.hpp:52-63) restricted to the G-REST fields, plus the
 * operator the session maintains and the CUDA device it is bound to. */
typedef struct {
  int32_t kind;     /* st_tracker_kind */
  int32_t op;       /* st_operator */
  int64_t k;        /* tracked pairs */
  int32_t order;    /* st_order (alg_desc for Laplacian operators) */
  int64_t rsvd_l;   /* randomized range finder target rank (default 100) */
  int64_t rsvd_p;   /* oversampling (default 100) */
  uint64_t seed;    /* TrackerOptions::seed */
  int32_t device;   /* CUDA device ordinal */
  int32_t flags;    /* ST_FLAG_* */
} st_config;

#define ST_FLAG_FORCE_DENSE 1  /* disable the compressed row-subset representation */
#define ST_FLAG_TIMING 2       /* record per-phase CUDA-event timings */
#define ST_FLAG_KERNEL_TIMING 4 /* record per-kernel-class CUDA-event timings (st_kernel_stats) */
#define ST_FLAG_CUSOLVER_EIG 8  /* projected eigensolves with cuSOLVER syevd instead of the on-device solver */

/* One update batch: the edit lists of assemble_update (graph.hpp:65-69).
 * added (i, j, w) and removed (i, j) address existing nodes; new_edges
 * (i, j, w) touch at least one of the n_new appended nodes, which get ids
 * n_old + 0 .. n_old + n_new - 1 in order. */
typedef struct {
  int64_t n_added;
  const int64_t* added_i;
  const int64_t* added_j;
  const double* added_w;
  int64_t n_removed;
  const int64_t* removed_i;
  const int64_t* removed_j;
  int64_t n_new;
  int64_t n_new_edges;
  const int64_t* new_i;
  const int64_t* new_j;
  const double* new_w;
} st_update;

typedef struct st_session st_session;

/* Session = the state one reference caller keeps across steps: the adjacency
 * CSR (and the shifted operator T for Laplacian operators, as in
 * ShiftedLaplacianSession, laplacian_track.cpp:43-46) plus the TrackerState
 * (trackers.hpp:65-75). The initial eigenpairs are an input (the output of
 * tracker_init, trackers.cpp:132-145): values[k] and vectors n x k
 * column-major with leading dimension ld. Replaces: constructing
 * ShiftedLaplacianSession + holding TrackerState by value. */
st_status st_create(const st_config* cfg, int64_t n, const int32_t* rowptr, const int32_t* colidx,
                    const double* values_csr, const double* eig_values, const double* eig_vectors, int64_t ld,
                    st_session** out);
void st_destroy(st_session* s);

/* LanczosOptions (lanczos.hpp:29-36) beyond k / order / seed, which come from
 * st_config. Defaults: tol 1e-10, max_basis 0 (= max(2k + 20, 40)),
 * max_restarts 500. The device path limits max_basis to 256. */
typedef struct {
  double tol;
  int64_t max_basis;
  int64_t max_restarts;
} st_lanczos_options;

/* tracker_init (trackers.cpp:132-145) on the device: a session whose initial
 * eigenpairs are the leading k of the tracked operator (A, or the shifted
 * Laplacian T for Laplacian operators), computed by thick-restart Lanczos with
 * full reorthogonalization (lanczos.hpp:38-127, seed mix_seed(cfg->seed,
 * 0x1a2c), residual test ||A x_i - theta_i x_i|| <= tol max|theta|). opts may
 * be NULL for the reference defaults. Errors as lanczos_topk: "k must satisfy
 * 1 <= k <= n", "max_basis below k", "no convergence after N restarts (...)". */
st_status st_tracker_init(const st_config* cfg, const st_lanczos_options* opts, int64_t n, const int32_t* rowptr,
                          const int32_t* colidx, const double* values_csr, st_session** out);
/* Sets the TrackerOptions fields above (before the first step); the session
 * starts with the reference defaults. */
st_status st_set_tracker_options(st_session* s, const st_tracker_options* opts);
/* TrackerState fields of TIMERS and TRIP (trackers.hpp:65-75). */
st_status st_tracker_state(const st_session* s, double* accumulated_change, int64_t* steps_since_restart,
                           double* restart_scale, int32_t* ridge_used);

/* Restarts and operator products of the session's tracker_init (0 when the
 * session was created from given eigenpairs). */
st_status st_init_stats(const st_session* s, int64_t* restarts, int64_t* products);

/* One step of the hot path. Replaces, in one call, the reference loop body
 * (experiment.cpp:169-173, 203):
 *   GraphUpdate d = assemble_update(...);            graph.cpp:45-100
 *   Perturbation p = to_perturbation(d)              trackers.cpp:128-130
 *                    | session.advance(d);           laplacian_track.cpp:48-64
 *   A = apply_update(A, d);                          graph.cpp:102-115
 *   state = tracker_step(state, p);                  trackers.cpp:341-387
 * Inputs are host buffers; the state stays resident on the device. Lists in
 * page-locked memory (cudaHostAlloc / cudaHostRegister) are DMA'd straight
 * from the caller's arrays; pageable lists go through one internal pinned
 * staging copy. The call returns after the uploads completed either way. */
st_status st_step(st_session* s, const st_update* upd);

/* Capacity hint for a stream that will reach n_nodes nodes and nnz stored
 * entries of A: the device state and the node- and entry-indexed buffers of
 * ingestion are sized once, so later steps up to that size allocate nothing
 * large. Optional; the reference has no counterpart (its CSR is rebuilt by
 * value each step). Invalidates the last step's Delta export (st_get_csr 2). */
st_status st_reserve(st_session* s, int64_t n_nodes, int64_t nnz);

/* A CSR block (int32 row offsets rows + 1, int32 column ids, fp64 values). */
typedef struct {
  int64_t rows, cols, nnz;
  const int32_t* rowptr;
  const int32_t* colidx;
  const double* values;
} st_csr_block;

/* GraphUpdate (graph.hpp:23-37): the step from n_old to n_old + n_new nodes as
 * the symmetric block perturbation [K G; G' C] (K n_old x n_old symmetric, G
 * n_old x n_new, C n_new x n_new symmetric). */
typedef struct {
  int64_t n_old, n_new;
  st_csr_block k_block, g_block, c_block;
} st_graph_update;

/* One step from a GraphUpdate. Replaces, for a caller that holds blocks
 * instead of edit lists (experiment.cpp:166-173):
 *   A = apply_update(A, d);                graph.cpp:102-115
 *   state = tracker_step(state, d);        trackers.cpp:384-387 -> to_perturbation
 * Delta is assembled on the device exactly as GraphUpdate::to_delta +
 * SymSparseMatrix::from_triplets (graph.cpp:17-32, sparse.cpp:17-23):
 * duplicates summed in insertion order, exact zeros pruned, symmetry
 * validated ("SymSparseMatrix: matrix is not symmetric"). Blocks may carry
 * any nonzero weights (partial deletions, diagonal entries). Host arrays;
 * st_step_blocks_device takes device arrays. */
st_status st_step_blocks(st_session* s, const st_graph_update* upd);
st_status st_step_blocks_device(st_session* s, const st_graph_update* upd);

/* tracker_step(state, Perturbation) (trackers.cpp:341-382; Perturbation =
 * {n_old, n_new, delta}, trackers.hpp:78-86) on an adjacency session: delta is
 * the (n_old + n_new)-square symmetric perturbation, also applied to the
 * session's A (pad(A) + delta with apply_update's checks). Laplacian sessions
 * derive Delta_T themselves and reject this call. */
st_status st_step_perturbation(st_session* s, int64_t n_old, int64_t n_new, const st_csr_block* delta);

/* st_step with the edit arrays already resident in device memory (same
 * layout; every pointer in *upd is a device pointer). Used to time the step
 * with its inputs in HBM. */
st_status st_step_device(st_session* s, const st_update* upd);

/* Sizes of the current state; alpha is the Laplacian shift (0 for adjacency). */
st_status st_info(const st_session* s, int64_t* n, int64_t* k, uint64_t* steps_taken, int64_t* nnz_a,
                  int64_t* nnz_t, int64_t* nnz_delta, double* alpha);

/* SpectralEmbedding (trackers.hpp:28-34): values[k], vectors n x k column-major. */
st_status st_get_embedding(const st_session* s, double* values, double* vectors, int64_t ld);

/* norms[i] = ||Op x_i - theta_i x_i||_2 for the k tracked pairs on the current
 * operator (A, or the shifted Laplacian T): the per-vector residual of the
 * reference's Lanczos convergence test (lanczos.hpp:85-95), computed on the
 * device with one full-operator SpMM (Op X) so a caller can monitor tracking
 * quality at any size without copying X to the host. Unsharded sessions. */
st_status st_residual_norms(st_session* s, double* norms);
/* Tracking quality against reference vectors Y (n x k, column-major, leading
 * dimension ld; e.g. the Lanczos reference of experiment.cpp:177-184), on the
 * device: psi[i] = principal_angle(x_i, y_i) (metrics.cpp:17-27, the
 * 2 atan2(||u - v||, ||u + v||) form) and *largest_angle = the largest
 * principal angle between span(X) and span(Y) (metrics.cpp:243-259), radians.
 * Either output may be NULL. Unsharded sessions. */
st_status st_angles(st_session* s, const double* ref_vectors, int64_t ld, double* psi, double* largest_angle);
/* Ritz values only (k doubles), the per-step result read by the e2e benchmark. */
st_status st_get_values(const st_session* s, double* values);

/* CSR export: which = 0 adjacency A, 1 shifted operator T, 2 the last step's
 * perturbation (Delta, or Delta_T for Laplacian operators). rowptr has n+1
 * entries, colidx/values nnz entries (sizes from st_info). */
st_status st_get_csr(const st_session* s, int32_t which, int32_t* rowptr, int32_t* colidx, double* values);

/* build_projection_basis (trackers.cpp:226-280) for `upd` against the current
 * state, without changing the session: Z is n_total x D column-major (caller
 * buffer of at least n_total * max_cols doubles); *cols receives D. */
st_status st_probe_basis(st_session* s, const st_update* upd, int32_t basis_kind, uint64_t seed, double* z,
                         int64_t ld, int64_t max_cols, int64_t* cols);

/* rayleigh_ritz_step (trackers.cpp:282-308) for `upd` against the current
 * state with a caller basis z (rows x cols, column-major), without changing the
 * session: values[k], vectors rows x k column-major. */
st_status st_probe_rr(st_session* s, const st_update* upd, const double* z, int64_t rows, int64_t cols, int64_t ldz,
                      double* values, double* vectors, int64_t ldv);

/* ---- Row-sharded sessions (one session per GPU of a box).
 *
 * The collectives a sharded session issues, supplied by the caller (NCCL in
 * production, e.g. ncclAllReduce / ncclAllGather on the given stream; any
 * transport in tests). Buffers are device pointers; `stream` is the session's
 * cudaStream_t and the operation must be ordered on it (enqueued on it, or
 * completed before returning). Results must be bitwise identical on every
 * rank. A callback returns 0 on success. */
typedef struct {
  int32_t rank;
  int32_t size;
  void* ctx;
  /* in-place elementwise sum over ranks of `count` doubles */
  int32_t (*allreduce_sum_f64)(void* ctx, double* buf, int64_t count, void* stream);
  /* recv[r * bytes .. (r + 1) * bytes) = send of rank r, for every rank r */
  int32_t (*allgather)(void* ctx, const void* send, void* recv, int64_t bytes, void* stream);
  /* personalized exchange: the send buffer holds send_bytes[r] bytes for rank
   * r, the chunks contiguous in rank order; the recv buffer receives
   * recv_bytes[r] bytes from rank r, contiguous in rank order (the byte
   * counts are host arrays of `size` entries; ncclSend/ncclRecv in a group,
   * MPI_Alltoallv). Carries the boundary-row halo of the sharded SpMMs. */
  int32_t (*alltoallv)(void* ctx, const void* send, const int64_t* send_bytes, void* recv, const int64_t* recv_bytes,
                       void* stream);
} st_comm;

/* Sharded counterpart of st_create. Every rank passes the same cfg and
 * n_global and its own contiguous block [row_lo, row_hi) of the initial nodes
 * (the blocks must tile [0, n_global) in rank order): the CSR rows of that
 * block (rowptr row_hi - row_lo + 1 entries, global column ids) and the same
 * rows of the initial eigenvectors (column-major, leading dimension ld), plus
 * the k eigenvalues. Appended nodes keep their global ids n_old + j and are
 * dealt to the ranks round-robin in chunks of `chunk` ids. Every rank then
 * calls st_step / st_step_device with the SAME update batch, in the same
 * order; st_get_embedding returns the owned rows (st_shard_rows gives their
 * global ids, ascending), st_get_csr(0) the owned rows of A (global columns),
 * st_get_csr(2) the full perturbation. Adjacency operator, k <= 64; the probe
 * calls are not available on sharded sessions. */
st_status st_create_sharded(const st_config* cfg, const st_comm* comm, int64_t n_global, int64_t row_lo,
                            int64_t row_hi, int64_t chunk, const int32_t* rowptr, const int32_t* colidx,
                            const double* values_csr, const double* eig_values, const double* eig_vectors,
                            int64_t ld, st_session** out);

/* The library's own st_comm over NCCL (NVLink / NVSwitch): every collective
 * is enqueued on the session stream with no host callback. Rank 0 calls
 * st_nccl_unique_id and shares the 128 bytes with the other ranks (any
 * transport); each rank then calls st_comm_nccl_create on its device.
 * NCCL is resolved at run time (libnccl.so.2). */
st_status st_nccl_unique_id(void* out128);
st_status st_comm_nccl_create(const void* unique_id, int32_t rank, int32_t size, int32_t device, st_comm* out);
void st_comm_nccl_destroy(st_comm* c);

/* Halo traffic of a sharded session since creation: bytes received from
 * other ranks, bytes of own rows copied locally, and the number of halos. */
st_status st_shard_stats(const st_session* s, int64_t* halo_bytes_recv, int64_t* halo_bytes_local, int64_t* halos);

/* Owned rows of a (sharded) session: *n_local, and their global ids when
 * global_ids is not NULL. An unsharded session owns every row. */
st_status st_shard_rows(const st_session* s, int64_t* n_local, int64_t* global_ids);

/* Host-only ownership map (no device work): the global ids, ascending, that
 * rank `rank` owns when the graph has n_total nodes, for initial bounds
 * bounds[0..size] and the given chunk. Returns the row count; writes at most
 * cap ids. */
int64_t st_shard_layout(int32_t size, const int64_t* bounds, int64_t chunk, int32_t rank, int64_t n_total,
                        int64_t* global_ids, int64_t cap);

/* Message of the last failed call on this session (or of st_create when s is NULL). */
const char* st_last_error(const st_session* s);

/* Per-phase device timings (ms) of the last step when ST_FLAG_TIMING is set:
 * [ingest, basis, rr_gram, eig, rotate, total]; returns the number written. */
int32_t st_last_timings(const st_session* s, double* ms, int32_t cap);
/* Kernel launches issued by the last st_step (counted by the library). */
int64_t st_last_launches(const st_session* s);

/* Standalone device replacements for two reference kernels (no session):
 * sym_eig_dense (eig.hpp:37-50): eigenvalues of (S + S')/2 in spectral order
 * and the leading `want` eigenvectors (n x want column-major), n <= 232;
 * GaussianSampler(seed).gaussian_matrix(rows, cols) (rng.hpp:64-69),
 * column-major. */
st_status st_sym_eig_dense(int32_t device, int64_t n, const double* s_colmajor, int32_t order, int64_t want,
                           double* values, double* vectors);
st_status st_gaussian_matrix(int32_t device, uint64_t seed, int64_t rows, int64_t cols, double* out_colmajor);

/* Accumulated device time (ms), launch count and algorithmic work of one
 * kernel class since the last reset (ST_FLAG_KERNEL_TIMING). Classes: 0 DMMA
 * Gram (flops), 1 DMMA row-local GEMM (flops), 2 CSR SpMM Delta.X / Delta.Z
 * (bytes), 3 Cholesky, 4 triangular inverse, 5 eigensolver, 6 CSR merge
 * (bytes), 7 RNG (draws), 8 Ritz rotation of X (bytes), 9 masked Gram of X
 * (flops), 10 sketch SpMMs (bytes), 11 other ingestion. Returns 0 for an
 * unknown class. */
int32_t st_kernel_stats(const st_session* s, int32_t cls, double* ms, int64_t* launches, double* work);
void st_reset_kernel_stats(st_session* s);
/* st_kernel_stats plus the second work measure (bytes of the DMMA classes,
 * flops of the memory classes) and the summed per-launch roofline time
 * max(flops / peak_flops, bytes / peak_bw) (peaks from st_set_peaks;
 * defaults 35.46 TFLOP/s FP64, 6465.8 GB/s). Classes 13 (DMMA Gram with both
 * sides <= 32 columns) and 14 (row-local GEMM with <= 32 output columns)
 * separate the narrow, memory-bound shapes from classes 0 and 1. */
int32_t st_kernel_stats2(const st_session* s, int32_t cls, double* ms, int64_t* launches, double* work, double* work2,
                         double* bound_ms);
void st_set_peaks(st_session* s, double fp64_tflops, double hbm_gbs);

#ifdef __cplusplus
}
#endif

#endif /* SPECTRACK_GPU_H */
