// B200-native G-REST per-step eigen-update: session state, the step pipeline
// and the C ABI of include/spectrack_gpu.h.
//
// Representation. Every vector the step builds (columns of X-bar, Delta X-bar,
// the RSVD sketch, the basis Z) lies in span(X-bar) + span{e_i : i in P}, where
// P is the set of rows touched by Delta plus the appended nodes. Writing such a
// vector as v = E u + X_out a (E selects the rows of P, X_out is X-bar with the
// rows of P zeroed), inner products are <v1, v2> = u1'u2 + a1' K a2 with
// K = X_out' X_out = R_c' R_c. The step therefore runs on the stacked
// coordinates [u (|P| rows); R_c a (k rows); a (k rows)]: Grams use the first
// |P| + k rows, linear combinations all of them. This is an exact isometry of
// the reference's n-row algebra (proj/src/trackers.cpp:226-308), so every
// projection, Gram-Schmidt decision and Ritz value is the reference's, while
// the tall-skinny work scales with |P| instead of n. Only two passes touch all
// n rows: K (masked Gram of X) and the final rotation X <- X A_new / E U_new.
// When |P| > n/2 the session runs the same code with P = all rows.
#include <cub/cub.cuh>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <sstream>
#include <functional>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/spectrack_gpu.h"
#include "common.cuh"
#include "dmma.cuh"
#include "eigsolve.cuh"
#include "ingest.cuh"
#include "lanczos.cuh"
#include "metrics.cuh"
#include "nccl_comm.cuh"
#include "rng.cuh"
#include "shard.cuh"
#include "smalllin.cuh"
#include "spmm.cuh"
#include "stepk.cuh"
#include "trackers.cuh"

namespace stg {

// kernel classes for per-class device timing (st_kernel_stats)
enum KClass : int {
  kGram = 0, kGemm = 1, kSpmm = 2, kChol = 3, kTriinv = 4, kEig = 5, kMerge = 6, kRng = 7, kRotate = 8,
  kKcGram = 9, kSpmmSketch = 10, kIngestOther = 11, kSpmmFull = 12, kGramNarrow = 13, kGemmNarrow = 14
};

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SpecRedo {};  // a speculated decision of the step failed (internal: the step is redone)

// ------------------------------------------------------------------ residual norms
// Per-column sums of (AX - X diag(theta))^2 over row blocks of 256 rows:
// thread (c, ry) of a 32 x 8 block walks rows ry, ry + 8, ... of its block for
// columns c, c + 32, ...; partial[block][c] in a fixed order (deterministic).
__global__ void __launch_bounds__(256) residual_partial_kernel(const double* AX, int ldax, const double* X, int ldx,
                                                               const double* theta, i64 n, int k, double* partial) {
  __shared__ double red[8][33];
  const int c_l = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const i64 r0 = static_cast<i64>(blockIdx.x) * 256;
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + c_l;
    double acc = 0.0;
    if (c < k) {
      const double th = theta[c];
      for (int i = ry; i < 256; i += 8) {
        const i64 r = r0 + i;
        if (r >= n) break;
        const double d = AX[r * ldax + c] - th * X[r * ldx + c];
        acc = fma(d, d, acc);
      }
    }
    red[ry][c_l] = acc;
    __syncthreads();
    if (ry == 0 && c < k) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += red[q][c_l];
      partial[static_cast<i64>(blockIdx.x) * k + c] = t;
    }
    __syncthreads();
  }
}

// out[c] = sqrt(sum_b partial[b][c]): one CTA per column, each thread sums a
// fixed strided subset of the partials, then a fixed-shape tree (deterministic).
__global__ void __launch_bounds__(256) residual_reduce_kernel(const double* partial, int nblocks, int k, double* out) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  double t = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 256) t += partial[static_cast<i64>(b) * k + c];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = sqrt(red[0]);
}

// ------------------------------------------------------------------ memory
// Named device buffers that only grow. Allocations come from a session-owned
// stream-ordered memory pool that never releases to the driver, on the main
// stream: a buffer outgrown as n and |P| creep up each step is freed and
// re-allocated in stream order (no device-wide synchronization, unlike
// cudaFree/cudaMalloc), and the freed block is reused by later growth.
// Ordering: a buffer's old block is only ever used on the main stream when it
// is outgrown (side-stream users of the previous block are joined by then:
// the merge at commit, the sketch eigensolve before the Rayleigh-Ritz step,
// the RNG by ensure_raw), so the free needs no extra dependency; a buffer a
// side stream uses after its allocation (`side_use`) makes the side streams
// wait for the allocation point.
class Arena {
 public:
  ~Arena() { reset(); }
  // frees every buffer and the pool (the session calls this before it
  // destroys the streams)
  void reset() {
    if (!pool_) return;
    for (auto& kv : bufs_)
      if (kv.second.ptr) cudaFreeAsync(kv.second.ptr, main_);
    bufs_.clear();
    cudaStreamSynchronize(main_);
    cudaMemPoolDestroy(pool_);
    pool_ = nullptr;
    if (ev_) cudaEventDestroy(ev_);
    ev_ = nullptr;
  }
  void init(int device, cudaStream_t main, std::vector<cudaStream_t> sides) {
    main_ = main;
    sides_ = std::move(sides);
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    STG_CUDA(cudaMemPoolCreate(&pool_, &props));
    unsigned long long keep = ~0ULL;
    STG_CUDA(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &keep));
    STG_CUDA(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
  }
  template <class T>
  T* get(const std::string& name, i64 count, bool side_use = false) {
    Buf& b = bufs_[name];
    const size_t bytes = static_cast<size_t>(std::max<i64>(count, 1)) * sizeof(T);
    if (b.bytes < bytes) {
      const size_t nb = bytes + bytes / 4 + 256;
      if (b.ptr) STG_CUDA(cudaFreeAsync(b.ptr, main_));
      STG_CUDA(cudaMallocFromPoolAsync(&b.ptr, nb, pool_, main_));
      if (side_use) join_main_into_sides();
      b.bytes = nb;
      ++grows_;
    }
    return static_cast<T*>(b.ptr);
  }
  // get() that keeps the first keep_bytes of the old contents on growth
  template <class T>
  T* get_keep(const std::string& name, i64 count, size_t keep_bytes) {
    Buf& b = bufs_[name];
    const size_t bytes = static_cast<size_t>(std::max<i64>(count, 1)) * sizeof(T);
    if (b.bytes < bytes && b.ptr) {
      void* old = b.ptr;
      const size_t nb = bytes + bytes / 4 + 256;
      STG_CUDA(cudaMallocFromPoolAsync(&b.ptr, nb, pool_, main_));
      if (keep_bytes) STG_CUDA(cudaMemcpyAsync(b.ptr, old, std::min(keep_bytes, b.bytes), cudaMemcpyDeviceToDevice, main_));
      STG_CUDA(cudaFreeAsync(old, main_));
      join_main_into_sides();  // the live CSR is read by the merge stream
      b.bytes = nb;
      ++grows_;
      return static_cast<T*>(b.ptr);
    }
    return get<T>(name, count);
  }
  // stream-ordered allocation outside the named buffers (X and temporaries
  // used on the main stream only)
  void* alloc(size_t bytes) {
    void* p = nullptr;
    STG_CUDA(cudaMallocFromPoolAsync(&p, bytes, pool_, main_));
    return p;
  }
  void release(void* p) {
    if (p) STG_CUDA(cudaFreeAsync(p, main_));
  }
  size_t total() const {
    size_t s = 0;
    for (auto& kv : bufs_) s += kv.second.bytes;
    return s;
  }
  i64 grows() const { return grows_; }
  // Keeps `bytes` of free memory in the pool (allocated once, then freed:
  // the pool never releases it), so later growth sub-allocates instead of
  // mapping new device memory in the middle of a step.
  void prewarm(size_t bytes) {
    if (!bytes) return;
    void* p = nullptr;
    if (cudaMallocFromPoolAsync(&p, bytes, pool_, main_) != cudaSuccess) {
      (void)cudaGetLastError();  // not enough memory for the headroom: skip it
      return;
    }
    STG_CUDA(cudaFreeAsync(p, main_));
    STG_CUDA(cudaStreamSynchronize(main_));
  }

 private:
  void join_main_into_sides() {
    STG_CUDA(cudaEventRecord(ev_, main_));
    for (cudaStream_t s : sides_) STG_CUDA(cudaStreamWaitEvent(s, ev_, 0));
  }
  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::unordered_map<std::string, Buf> bufs_;
  cudaMemPool_t pool_ = nullptr;
  cudaStream_t main_ = nullptr;
  std::vector<cudaStream_t> sides_;
  cudaEvent_t ev_ = nullptr;
  i64 grows_ = 0;
};

class Pinned {
 public:
  ~Pinned() {
    if (p_) cudaFreeHost(p_);
  }
  void* get(size_t bytes) {
    if (bytes > cap_) {
      if (p_) STG_CUDA(cudaFreeHost(p_));
      cap_ = bytes + bytes / 4 + 4096;
      STG_CUDA(cudaMallocHost(&p_, cap_));
    }
    return p_;
  }

 private:
  void* p_ = nullptr;
  size_t cap_ = 0;
};

struct DevCsr {
  i64 n = 0, nnz = 0;
  int* rp = nullptr;
  int* col = nullptr;
  double* val = nullptr;
};

// A view of a row-major block.
struct Blk {
  double* p = nullptr;
  int ld = 0;
  Blk cols(int c0) const { return Blk{p + c0, ld}; }
};

struct Scalars {  // pinned host mirror of device scalars read at sync points
  u64 err_edit;
  u64 err_apply;
  unsigned long long nvalid;
  int nnz_new;
  int p;
  int nnz_t;
  int nnz_dt;
  int flags;
  int info;
  int sticky;
  int mgs_r;
  double alpha;
  double sk_lam[kEigMaxN];  // sketch eigenvalues, copied asynchronously (pageable memory would block the host)
};

static const char* edit_message(int code) {
  switch (code) {
    case kErrZeroWeight: return "assemble_update: zero-weight edit";
    case kErrEditRange: return "assemble_update: edited edge must address existing nodes";
    case kErrSelfLoop: return "assemble_update: self-loop rejected";
    case kErrDuplicate: return "assemble_update: duplicate edge across edit lists";
    case kErrNewRange: return "assemble_update: new edge endpoint out of range";
    case kErrNewWeight: return "assemble_update: new edges need positive weight";
    case kErrNewOldOnly: return "assemble_update: new edge addresses only existing nodes";
    case kErrNotSymmetric: return "SymSparseMatrix: matrix is not symmetric";
    case kErrBlockShape: return "st_step_blocks: malformed block CSR";
    default: return "assemble_update: invalid edit";
  }
}

// The perturbation of one step in compressed form.
struct Pert {
  i64 n_old = 0, S = 0, n_total = 0;
  i64 nnz = 0;         // nnz(Delta) (global)
  i64 p = 0, p_old = 0;  // |P|, rows of P below n_old
  bool dense = false;  // P = all rows
  const int* grp = nullptr;  // global CSR of Delta (n_total + 1)
  const int* gcol = nullptr;
  const double* val = nullptr;
  const int* lrp = nullptr;  // local CSR over P
  const int* lcol = nullptr;
  const int* P = nullptr;
  const int* posmap = nullptr;
  const int* mark = nullptr;  // rows of P: mark[r] == stamp
  int stamp = 0;
  // Row-sharded sessions (shard.cuh) keep the rows of P they own: p, p_old
  // and S_loc count owned rows; G = rows entering a Gram (the k coordinate
  // rows R_c a are counted by rank 0 only); X rows by local index.
  i64 G = 0;                 // p + k (unsharded)
  i64 S_loc = 0;             // appended rows in P here (= S unsharded)
  i64 x_old = 0, x_total = 0;  // rows of the X storage before / after the step
  i64 pmax = 0;              // P-id exchange rows per rank (sharded)
  // boundary-row halo (sharded): rows sent to / received from each rank
  const int* hsend = nullptr;  // own P indices to send, grouped by destination
  i64 nsend = 0, nrecv = 0;
  std::vector<i64> send_rows, recv_rows;
  const int* Ploc = nullptr;   // X storage row of each row of P (= P unsharded)
  const int* Pglob = nullptr;  // global id of each row of P (= P unsharded)
  const double* gval = nullptr;  // values of the global Delta CSR (grp/gcol)
  const int* scol = nullptr;  // sketch SpMM columns: only cols >= scol_lo, X row = col - scol_lo
  int scol_lo = 0;
  bool empty() const { return S == 0 && nnz == 0; }
};

// Compressed basis produced by build_basis: N = p + 2k rows, D columns.
struct Basis {
  Blk z;
  int D = 0;
};

// ------------------------------------------------------------------ session
class Session {
 public:
  st_config cfg{};
  std::string last_error;
  i64 n = 0, k = 0;
  u64 steps_taken = 0;
  double alpha = 0.0;
  std::vector<double> values;
  double timings[8] = {0};
  int ntimings = 0;
  i64 launches = 0;
  // per-kernel-class device time (CUDA events on the launching stream) and
  // algorithmic work (flops for DMMA classes, bytes for memory-bound classes)
  // work: flops (DMMA classes) or bytes (memory classes); work2 the other
  // measure; bound_ms the per-launch roofline time max(flops / F, bytes / B)
  // summed (peaks from st_set_peaks)
  struct KStat {
    double ms = 0, work = 0, work2 = 0, bound_ms = 0;
    i64 launches = 0;
  };
  static constexpr int kClasses = 15;
  double peak_tflops_ = 35.46, peak_gbs_ = 6465.8;
  KStat kstats[kClasses];

  struct ShardInit {
    st_comm comm;
    i64 n_global, lo, hi, chunk;
  };

  // LanczosOptions (lanczos.hpp:29-36) beyond the tracker's k / order / seed
  struct LzOpts {
    double tol = 1e-10;
    i64 max_basis = 0;
    i64 max_restarts = 500;
  };
  i64 lz_restarts = 0, lz_products = 0;  // tracker_init statistics
  // TrackerOptions of the perturbation trackers and TIMERS (trackers.hpp:52-63)
  // and the TrackerState fields they carry (trackers.hpp:65-75)
  st_tracker_options topt_{0.0, 0, 0.01, 5, ST_IASC};
  double acc_change_ = 0.0, restart_scale_ = 0.0;
  i64 steps_since_restart_ = 0;
  bool ridge_used_ = false;
  static double l2norm(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
  }
  bool prewarmed_ = false;
  bool spec_ = false;      // the current step attempt speculates (run_step)
  i64 spec_redos = 0;      // steps redone on the exact path
  const bool lz_log_ = getenv("STG_LZ_LOG") != nullptr;
  const bool lz_log2_ = getenv("STG_LZ_LOG2") != nullptr;

  // ev == nullptr: tracker_init (trackers.cpp:132-145) on the device, i.e. the
  // leading eigenpairs of the tracked operator by thick-restart Lanczos.
  Session(const st_config& c, i64 n0, const int* rp, const int* col, const double* val, const double* ev,
          const double* evec, i64 ld, const ShardInit* shard = nullptr, const LzOpts* lz = nullptr)
      : cfg(c) {
    STG_CUDA(cudaSetDevice(cfg.device));
    {  // priorities: the eigensolve's CTAs take SMs ahead of the wide kernels it
       // overlaps; the CSR merge copy fills whatever the step leaves idle
      int lo = 0, hi = 0;
      STG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      STG_CUDA(cudaStreamCreateWithPriority(&st_, cudaStreamNonBlocking, (lo + hi) / 2));
      STG_CUDA(cudaStreamCreateWithPriority(&st_eig_, cudaStreamNonBlocking, hi));
      STG_CUDA(cudaStreamCreateWithPriority(&st_mg_, cudaStreamNonBlocking, lo));
      STG_CUDA(cudaStreamCreateWithPriority(&st_rot_, cudaStreamNonBlocking, (lo + hi) / 2));
    }
    STG_CUDA(cudaEventCreateWithFlags(&ev_rot_ready_, cudaEventDisableTiming));
    STG_CUDA(cudaEventCreateWithFlags(&ev_k_, cudaEventDisableTiming));
    STG_CUDA(cudaEventCreateWithFlags(&ev_rot_done_, cudaEventDisableTiming));
    STG_CUDA(cudaStreamCreateWithFlags(&st_rng_, cudaStreamNonBlocking));
    arena_.init(cfg.device, st_, {st_eig_, st_mg_, st_rng_});
    STG_CUDA(cudaEventCreateWithFlags(&ev_rng_, cudaEventDisableTiming));
    STG_CUDA(cudaEventCreateWithFlags(&ev_mg_fork_, cudaEventDisableTiming));
    STG_CUDA(cudaEventCreateWithFlags(&ev_mg_, cudaEventDisableTiming));
    STG_CUDA(cudaEventCreateWithFlags(&ev_gb_, cudaEventDisableTiming));
    STG_CUDA(cudaEventCreateWithFlags(&ev_eig_, cudaEventDisableTiming));
    for (auto& e : tev_) STG_CUDA(cudaEventCreate(&e));
    if (cusolverDnCreate(&solver_) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnCreate failed");
    cusolverDnSetStream(solver_, st_);
    STG_CUDA(cudaMallocHost(&hs_, sizeof(Scalars)));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_tn_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_smem(2, 2))));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_tn_kernel<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_smem(1, 4))));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_tn_kernel<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_smem(4, 1))));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_persist_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_tma_smem<2, 2>())));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_persist_kernel<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_tma_smem<1, 4>())));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_persist_kernel<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_tma_smem<4, 1>())));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_tma_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_tma_smem<2, 2>())));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_tma_kernel<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_tma_smem<1, 4>())));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_tma_kernel<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_tma_smem<4, 1>())));
    STG_CUDA(cudaFuncSetAttribute(dm::gemm_nn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::kNNSmem)));
    STG_CUDA(cudaFuncSetAttribute(dm::gemm_nn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::kNNSmem)));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::gram_stream_smem(false))));
    STG_CUDA(cudaFuncSetAttribute(dm::gemm_nn_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::kStreamSmem)));
    STG_CUDA(cudaFuncSetAttribute(dm::gemm_nn_persist_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::nnp_smem(true))));
    STG_CUDA(cudaFuncSetAttribute(dm::gemm_nn_persist_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::nnp_smem(false))));
    STG_CUDA(cudaFuncSetAttribute(dm::gram_persist_rs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::kRsSmem)));
    STG_CUDA(cudaFuncSetAttribute(dm::gemm_nn_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::kNNTmaSmem)));
    STG_CUDA(cudaFuncSetAttribute(dm::gemm_nn_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dm::kNNTmaSmem)));
    // function attributes are per device: set for this session's device here
    STG_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(chol_smem_bytes(kCholMaxW))));
    STG_CUDA(cudaFuncSetAttribute(triinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(triinv_smem_bytes(kCholMaxW))));
    eig_set_attributes();
    d_scal_ = arena_.get<u64>("scalars", 32);
    // tile counters of the persistent DMMA kernels: a {next, ended} pair per stream that launches them
    // (sched_slot_); each launch leaves its pair at zero
    sched_ctr_ = arena_.get<int>("sched_ctr", 64, /*side_use=*/true);
    STG_CUDA(cudaMemsetAsync(sched_ctr_, 0, sizeof(int) * 64, st_));
    k = cfg.k;
    n = n0;
    if (shard) {  // n0 = rows of this rank's block; n = the global node count
      init_shard(*shard);
      n = shard->n_global;
    }
    if (k < 1 || k > n) throw InvalidArgument("tracker_init: k must satisfy 1 <= k <= n");
    if (cfg.kind < ST_TRIP_BASIC || cfg.kind > ST_TIMERS) throw InvalidArgument("tracker_step: unknown tracker kind");
    if (shard && (cfg.kind < ST_IASC || cfg.kind > ST_GREST_RSVD))
      throw InvalidArgument("st_create_sharded: sharded sessions run the projection trackers");
    if (cfg.kind <= ST_RESIDUAL_MODES && k > kTrkMaxK)
      throw InvalidArgument("st_create: the perturbation trackers support k <= 128");
    if (cfg.op == ST_NORMALIZED_LAPLACIAN || cfg.op == ST_LAPLACIAN) {
      if (cfg.order != ST_ALG_DESC) {
        // the reference adapter forces alg_desc for shifted operators (laplacian_track.cpp:88)
      }
    }
    // adjacency CSR
    const i64 nnz = rp[n0];
    A_[0] = alloc_csr("A0", n0, nnz);
    STG_CUDA(cudaMemcpyAsync(A_[0].rp, rp, sizeof(int) * (n0 + 1), cudaMemcpyHostToDevice, st_));
    STG_CUDA(cudaMemcpyAsync(A_[0].col, col, sizeof(int) * std::max<i64>(nnz, 1), cudaMemcpyHostToDevice, st_));
    STG_CUDA(cudaMemcpyAsync(A_[0].val, val, sizeof(double) * std::max<i64>(nnz, 1), cudaMemcpyHostToDevice, st_));
    acur_ = 0;
    ensure_node_capacity(n, n0);
    nloc_ = n0;
    d_values_ = arena_.get<double>("values", k);
    if (!ev) {
      if (shard) throw InvalidArgument("st_tracker_init: sharded sessions take their initial eigenpairs");
      if (is_laplacian()) init_laplacian();
      const LzOpts o = lz ? *lz : LzOpts{};
      lanczos(is_laplacian() ? T() : A(), n0, o);
      STG_CUDA(cudaMemcpyAsync(d_values_, values.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      restart_scale_ = l2norm(values);
      return;
    }
    // eigenpairs: column-major host -> row-major device
    values.assign(ev, ev + k);
    restart_scale_ = l2norm(values);
    std::vector<double> xr(static_cast<size_t>(n0 * k));
    for (i64 c = 0; c < k; ++c)
      for (i64 i = 0; i < n0; ++i) xr[static_cast<size_t>(i * k + c)] = evec[c * ld + i];
    STG_CUDA(cudaMemcpy2DAsync(X_, sizeof(double) * ldx(), xr.data(), sizeof(double) * k, sizeof(double) * k, n0,
                               cudaMemcpyHostToDevice, st_));
    STG_CUDA(cudaMemcpyAsync(d_values_, values.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st_));
    if (is_laplacian()) init_laplacian();
    STG_CUDA(cudaStreamSynchronize(st_));
  }

  ~Session() {
    cudaStreamSynchronize(st_rot_);
    cudaStreamSynchronize(st_);
    cudaStreamSynchronize(st_rng_);
    cudaStreamSynchronize(st_eig_);
    cudaStreamSynchronize(st_mg_);
    if (X_) cudaFreeAsync(X_, st_);
    X_ = nullptr;
    arena_.reset();  // pool blocks are freed on st_ before the streams go
    if (solver_) cusolverDnDestroy(solver_);
    if (hs_) cudaFreeHost(hs_);
    for (auto& e : tev_) cudaEventDestroy(e);
    cudaEventDestroy(ev_rng_);
    cudaStreamDestroy(st_rng_);
    cudaStreamSynchronize(st_eig_);
    cudaEventDestroy(ev_gb_);
    cudaEventDestroy(ev_eig_);
    cudaStreamDestroy(st_eig_);
    cudaStreamSynchronize(st_mg_);
    cudaEventDestroy(ev_mg_fork_);
    cudaEventDestroy(ev_mg_);
    cudaStreamDestroy(st_mg_);
    cudaEventDestroy(ev_rot_ready_);
    cudaEventDestroy(ev_k_);
    cudaEventDestroy(ev_rot_done_);
    cudaStreamDestroy(st_rot_);
    cudaStreamDestroy(st_);
  }

  // The last step's rotation of X (rows outside P) runs on st_rot_ so the next
  // step's ingestion overlaps it; every later use of X orders after it here.
  void wait_rotation() {
    if (!rot_pending_) return;
    STG_CUDA(cudaStreamWaitEvent(st_, ev_rot_done_, 0));
    rot_pending_ = false;
  }

  bool is_laplacian() const { return cfg.op == ST_LAPLACIAN || cfg.op == ST_NORMALIZED_LAPLACIAN; }
  const DevCsr& A() const { return A_[acur_]; }
  const DevCsr& T() const { return T_[tcur_]; }
  i64 nnz_delta() const { return last_delta_nnz_; }

  // ---------------------------------------------------------------- sharding
  bool sh_ = false;
  st_comm comm_{};
  ShardMap map_;             // device bounds (kernels)
  std::vector<i64> bounds_;  // host copy
  i64 nloc_ = 0;             // rows stored here (= n unsharded)
  int* mark_dl_ = nullptr;   // Delta-row marks by local row (sharded merge)
  const bool shard_debug_ = getenv("STG_SHARD_DEBUG") != nullptr;

  void init_shard(const ShardInit& si) {
    if (si.comm.size < 1 || si.comm.rank < 0 || si.comm.rank >= si.comm.size || !si.comm.allreduce_sum_f64 ||
        !si.comm.allgather || !si.comm.alltoallv)
      throw InvalidArgument("st_create_sharded: invalid communicator");
    if (si.chunk < 1) throw InvalidArgument("st_create_sharded: chunk must be positive");
    if (si.lo < 0 || si.hi < si.lo || si.hi > si.n_global)
      throw InvalidArgument("st_create_sharded: row block outside [0, n_global)");
    if (cfg.op != ST_ADJACENCY) throw InvalidArgument("st_create_sharded: sharded sessions track the adjacency operator");
    if (cfg.k > 64) throw InvalidArgument("st_create_sharded: sharded sessions support k <= 64");
    sh_ = true;
    comm_ = si.comm;
    const int R = comm_.size;
    std::vector<u64> lohi = allgather_u64({static_cast<u64>(si.lo), static_cast<u64>(si.hi)});
    bounds_.assign(static_cast<size_t>(R) + 1, 0);
    for (int r = 0; r < R; ++r) {
      const i64 lo = static_cast<i64>(lohi[2 * r]), hi = static_cast<i64>(lohi[2 * r + 1]);
      if (lo != bounds_[r]) throw InvalidArgument("st_create_sharded: row blocks must tile [0, n_global) in rank order");
      bounds_[r + 1] = hi;
    }
    if (bounds_[R] != si.n_global) throw InvalidArgument("st_create_sharded: row blocks must tile [0, n_global) in rank order");
    i64* db = arena_.get<i64>("shard_bounds", R + 1);
    STG_CUDA(cudaMemcpyAsync(db, bounds_.data(), sizeof(i64) * (R + 1), cudaMemcpyHostToDevice, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    map_.n0 = si.n_global;
    map_.chunk = si.chunk;
    map_.size = R;
    map_.rank = comm_.rank;
    map_.bounds = db;
    map_.own0 = si.hi - si.lo;
    map_.lo = si.lo;
  }

  ShardMap host_map() const {
    ShardMap m = map_;
    m.bounds = bounds_.data();
    return m;
  }
  i64 rows_at(int r, i64 n_total) const { return sm_rows(map_, r, n_total, bounds_.data()); }

  void allreduce(double* buf, i64 count) {
    if (count <= 0) return;
    if (comm_.allreduce_sum_f64(comm_.ctx, buf, count, st_) != 0) throw RuntimeError("st_comm: allreduce failed");
  }
  void allgather(const void* send, void* recv, i64 bytes) {
    if (comm_.allgather(comm_.ctx, send, recv, bytes, st_) != 0) throw RuntimeError("st_comm: allgather failed");
  }
  void alltoallv(const void* send, const std::vector<i64>& sb, void* recv, const std::vector<i64>& rb) {
    if (comm_.alltoallv(comm_.ctx, send, reinterpret_cast<const int64_t*>(sb.data()), recv,
                        reinterpret_cast<const int64_t*>(rb.data()), st_) != 0)
      throw RuntimeError("st_comm: alltoallv failed");
  }
  // bytes the sharded SpMM halos received (diagnostics: st_shard_stats)
  i64 halo_bytes_recv_ = 0, halo_bytes_local_ = 0, halo_calls_ = 0;
  // small host values of every rank (rank-major), through device staging
  std::vector<u64> allgather_u64(const std::vector<u64>& mine) {
    const i64 m = static_cast<i64>(mine.size());
    u64* d = arena_.get<u64>("ag_u64", m * (comm_.size + 1));
    STG_CUDA(cudaMemcpyAsync(d, mine.data(), sizeof(u64) * m, cudaMemcpyHostToDevice, st_));
    allgather(d, d + m, sizeof(u64) * m);
    std::vector<u64> all(static_cast<size_t>(m * comm_.size));
    STG_CUDA(cudaMemcpyAsync(all.data(), d + m, sizeof(u64) * m * comm_.size, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    return all;
  }

  // ---------------------------------------------------------------- public ops
  void step(const st_update& u, bool device_ptrs = false) {
    run_step(u.n_new, [&]() { return ingest(u, /*commit_slot*/ true, device_ptrs); });
  }

  // tracker_step(state, GraphUpdate) (trackers.cpp:384-387) with the session's
  // apply_update: the blocks K, G, C of graph.hpp:23-37
  void step_blocks(const st_graph_update& g, bool device_ptrs) {
    if (g.n_old != n) throw InvalidArgument("apply_update: matrix size != d.n_old");
    if (g.n_new < 0) throw InvalidArgument("make_empty_update: negative size");
    const st_csr_block& K = g.k_block;
    const st_csr_block& G = g.g_block;
    const st_csr_block& Cb = g.c_block;
    if (K.rows != g.n_old || K.cols != g.n_old || G.rows != g.n_old || G.cols != g.n_new || Cb.rows != g.n_new ||
        Cb.cols != g.n_new)
      throw InvalidArgument("st_step_blocks: block shape mismatch");
    std::vector<HostBlock> hb{{K, 0, 0, 0}, {G, 0, g.n_old, 1}, {Cb, g.n_old, g.n_old, 0}};
    run_step(g.n_new, [&]() { return ingest_blocks(g.n_new, hb, true, device_ptrs); });
  }

  // tracker_step(state, Perturbation) (trackers.cpp:341-382) on an adjacency
  // session: Delta (n_old + n_new square) is also applied to the session's A
  void step_perturbation(i64 n_old, i64 n_new, const st_csr_block& delta, bool device_ptrs) {
    if (is_laplacian())
      throw InvalidArgument("st_step_perturbation: Laplacian sessions derive Delta_T from graph updates");
    if (n_old != n) throw InvalidArgument("build_projection_basis: perturbation dimension mismatch");
    if (n_new < 0) throw InvalidArgument("build_projection_basis: negative expansion");
    if (delta.rows != n_old + n_new || delta.cols != n_old + n_new)
      throw InvalidArgument("build_projection_basis: delta size != n_old + n_new");
    std::vector<HostBlock> hb{{delta, 0, 0, 0}};
    run_step(n_new, [&]() { return ingest_blocks(n_new, hb, true, device_ptrs); });
  }

  template <class F>
  void run_step(i64 n_new, F&& front) {
    launches = 0;
    rr_pre_.valid = false;
    kdiscard();  // a failed or probe call may have left unflushed entries
    timing_begin();
    const u64 basis_seed = mix_seed(mix_seed(cfg.seed, 0x6b7aULL), steps_taken);
    omega_S_ = -1;  // a sketch from an earlier call is never reused
    if (cfg.kind == ST_GREST_RSVD && n_new > cfg.rsvd_l && n_new > 0) {
      // the sketch's seed and shape are known before ingestion: overlap the
      // sequential mt19937_64 recurrence with it (trackers.cpp:362, rsvd.hpp:42-44)
      const int q = static_cast<int>(std::min<i64>(n_new, cfg.rsvd_l + cfg.rsvd_p));
      double* om;
      int ldo;
      prepare_omega(basis_seed, n_new, q, &om, &ldo);
    }
    // the kind that steps: TIMERS delegates to restart_inner (trackers.cpp:369-377)
    const int kind = cfg.kind == ST_TIMERS ? topt_.restart_inner : cfg.kind;
    if (cfg.kind == ST_TIMERS && topt_.theta < 0.0) throw InvalidArgument("timers_step: theta must be >= 0");
    if (kind == ST_RESIDUAL_MODES) {  // trackers.cpp:204-207
      const double eps = 1e-12 * std::max(1.0, values.empty() ? 0.0 : std::fabs(values[0]));
      for (double l : values)
        if (std::fabs(l - topt_.mu) < eps)
          throw InvalidArgument("residual_modes_step: mu collides with tracked eigenvalue");
    }
    Pert pt = front();
    wait_rotation();  // the previous step's rotation of X ran beside this ingestion
    timing_mark(0);
    // TIMERS proxy (trackers.cpp:317-320): ||Delta||_F / restart_scale accumulated
    double acc_next = acc_change_;
    i64 ssr_next = steps_since_restart_;
    if (cfg.kind == ST_TIMERS) {
      double* sq = arena_.get<double>("timers_sq", 1);
      STG_CUDA(cudaMemsetAsync(sq, 0, sizeof(double), st_));
      if (pt.nnz > 0) launch(sumsq_kernel, dim3(1), dim3(256), 0, st_, pt.gval ? pt.gval : pt.val, pt.nnz, sq);
      double h = 0.0;
      STG_CUDA(cudaMemcpyAsync(&h, sq, sizeof(double), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      acc_next += std::sqrt(h) / (restart_scale_ > 0.0 ? restart_scale_ : 1.0);
      ssr_next += 1;
      if (acc_next >= topt_.theta && ssr_next >= topt_.min_restart_gap) {
        // restart: the leading pairs of the updated operator (trackers.cpp:322-333)
        commit_graph(pt);
        n = pt.n_total;
        lanczos(is_laplacian() ? T() : A(), n, LzOpts{});
        STG_CUDA(cudaMemcpyAsync(d_values_, values.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st_));
        STG_CUDA(cudaStreamSynchronize(st_));
        restart_scale_ = l2norm(values);
        acc_change_ = 0.0;
        steps_since_restart_ = 0;
        steps_taken += 1;
        timing_end(0);
        kflush();
        return;
      }
    }
    if (pt.empty()) {
      commit_graph(pt);
      steps_taken += 1;
      acc_change_ = acc_next;
      steps_since_restart_ = ssr_next;
      timing_end(0);
      kflush();
      return;
    }
    std::vector<double> newvals;
    // first attempt speculates the rare host decisions (suspect pivots, sketch
    // rank) and checks them once at the end; a failed speculation leaves X
    // untouched (the rotation is gated) and the step is redone exactly
    for (int attempt = 0;; ++attempt) {
      spec_ = attempt == 0 && !sh_ && !(cfg.flags & ST_FLAG_CUSOLVER_EIG) && !getenv_flag("STG_NO_SPEC");
      STG_CUDA(cudaMemsetAsync(sticky_ptr(), 0, sizeof(int), st_));
      try {
        if (kind >= ST_IASC && kind <= ST_GREST_RSVD) {
          Basis b = build_basis(pt, kind - ST_IASC, basis_seed);
          timing_mark(1);
          rayleigh_ritz(pt, b, newvals, /*write_state*/ true, nullptr, 0);
        } else {
          perturbation_step(pt, kind, newvals);
        }
        spec_ = false;
        break;
      } catch (const SpecRedo&) {
        restore_x();
        rr_pre_.valid = false;
        ++spec_redos;
        continue;
      } catch (...) {
        spec_ = false;
        restore_x();
        cudaStreamSynchronize(st_);
        throw;
      }
    }
    xrestore_.active = false;  // the rotation rewrote the rows of P
    commit_graph(pt);
    values = newvals;
    n = pt.n_total;
    steps_taken += 1;
    acc_change_ = acc_next;
    steps_since_restart_ = ssr_next;
    if (!prewarmed_) {
      // after the first full step the working set is known: keep 1.6x of it
      // free in the pool, so the buffers that outgrow their 1.25x headroom as
      // the graph grows (at 1%/step, ~every 22 steps) are re-carved from
      // memory the pool already holds
      prewarmed_ = true;
      size_t fr = 0, tot = 0;
      STG_CUDA(cudaMemGetInfo(&fr, &tot));
      arena_.prewarm(std::min<size_t>(arena_.total() + arena_.total() * 6 / 10, fr / 2));
    }
    timing_end(5);
    kflush();
  }

  // Capacity for a stream that will reach n_nodes nodes and nnz stored
  // entries: X, the node marks and the node- and entry-indexed buffers of
  // ingestion and the CSR merge are sized once, so steps up to that size never
  // grow a buffer (st_reserve).
  void reserve(i64 n_nodes, i64 nnz) {
    if (n_nodes < n || nnz < 0) throw InvalidArgument("st_reserve: capacity below the current graph");
    if (n_nodes >= (1LL << 31)) throw InvalidArgument("st_step: node count exceeds int32 CSR indexing");
    ensure_node_capacity(n_nodes, sh_ ? rows_at(comm_.rank, n_nodes) : n_nodes);
    const i64 rows = (sh_ ? rows_at(comm_.rank, n_nodes) : n_nodes) + 1;
    for (const char* name : {"m_ncnt", "sh_lcnt", "sh_ldrp", "sh_pflag", "sh_ppos"}) arena_.get<int>(name, rows);
    if (!sh_)
      for (const char* name : {"dcnt", "drp", "p_flag", "p_pos", "P", "t_cnt", "dt_cnt", "dt_rp"})
        arena_.get<int>(name, n_nodes + 1);
    STG_CUDA(cudaStreamWaitEvent(st_, ev_mg_, 0));
    for (int slot = 0; slot < 2; ++slot) {  // the live slot keeps its contents
      DevCsr& a = A_[slot];
      const bool live = slot == acur_;
      const std::string nm = "A" + std::to_string(slot);
      int* rp = arena_.get_keep<int>(nm + ".rp", rows, live ? sizeof(int) * (a.n + 1) : 0);
      int* col = arena_.get_keep<int>(nm + ".col", nnz, live ? sizeof(int) * a.nnz : 0);
      double* val = arena_.get_keep<double>(nm + ".val", nnz, live ? sizeof(double) * a.nnz : 0);
      if (live) {
        a.rp = rp;
        a.col = col;
        a.val = val;
      }
    }
    if (is_laplacian()) {
      DevCsr& t = T_[tcur_];
      const std::string nm = "T" + std::to_string(tcur_);
      t.rp = arena_.get_keep<int>(nm + ".rp", n_nodes + 1, sizeof(int) * (t.n + 1));
      arena_.get<int>("T" + std::to_string(1 - tcur_) + ".rp", n_nodes + 1);
    }
    last_delta_ = DevCsr{};  // its buffers may have moved: the Delta export restarts at the next step
    last_delta_nnz_ = 0;
    STG_CUDA(cudaStreamSynchronize(st_));
  }

  i64 probe_basis(const st_update& u, int basis_kind, u64 seed, double* z, i64 ldz, i64 max_cols) {
    launches = 0;
    omega_S_ = -1;
    Pert pt = ingest(u, false);
    if (pt.n_old != n) throw InvalidArgument("build_projection_basis: perturbation dimension mismatch");
    if (pt.empty() && basis_kind != 0) {
      // trackers.cpp:375-376 with Delta = 0: the basis is the padded old vectors
      if (k > max_cols) throw InvalidArgument("st_probe_basis: output buffer too narrow");
      std::vector<double> x(static_cast<size_t>(n * k));
      copy_x_colmajor(x.data(), n);
      for (i64 c = 0; c < k; ++c)
        for (i64 i = 0; i < pt.n_total; ++i) z[c * ldz + i] = i < n ? x[static_cast<size_t>(c * n + i)] : 0.0;
      return k;
    }
    struct Restore {
      Session* s;
      ~Restore() {
        s->restore_x();
        cudaStreamSynchronize(s->st_);
      }
    } restore{this};
    Basis b = build_basis(pt, basis_kind, seed);
    if (b.D > max_cols) throw InvalidArgument("st_probe_basis: output buffer too narrow");
    expand_dense(pt, b.z, b.D, z, ldz);
    return b.D;
  }

  void probe_rr(const st_update& u, const double* z, i64 rows, i64 cols, i64 ldz, double* vals, double* vecs,
                i64 ldv) {
    launches = 0;
    Pert pt = ingest(u, false);
    if (pt.n_old != n) throw InvalidArgument("rayleigh_ritz_step: perturbation dimension mismatch");
    if (pt.empty()) {  // trackers.cpp:286: state returned unchanged
      std::memcpy(vals, values.data(), sizeof(double) * k);
      std::vector<double> x(static_cast<size_t>(n * k));
      copy_x_colmajor(x.data(), n);
      for (i64 c = 0; c < k; ++c) std::memcpy(vecs + c * ldv, x.data() + c * n, sizeof(double) * n);
      return;
    }
    if (rows != pt.n_total) throw InvalidArgument("rayleigh_ritz_step: basis row count mismatch");
    if (cols < k) throw InvalidArgument("rayleigh_ritz_step: projection subspace too small");
    // caller bases live in the full row space: P = all rows, a-coordinates 0
    make_dense(pt);
    const i64 N = pt.p + 2 * k;
    const int ldz_d = ld_for(cols);
    double* zd = arena_.get<double>("probe_z", N * ldz_d);
    STG_CUDA(cudaMemsetAsync(zd, 0, sizeof(double) * N * ldz_d, st_));
    std::vector<double> zr(static_cast<size_t>(rows * cols));
    for (i64 c = 0; c < cols; ++c)
      for (i64 i = 0; i < rows; ++i) zr[static_cast<size_t>(i * cols + c)] = z[c * ldz + i];
    STG_CUDA(cudaMemcpy2DAsync(zd, sizeof(double) * ldz_d, zr.data(), sizeof(double) * cols, sizeof(double) * cols,
                               rows, cudaMemcpyHostToDevice, st_));
    // Xc for the Eq. (14) low-rank term: rows [0, n_old) = X, new rows 0, no a-part
    Basis b{Blk{zd, ldz_d}, static_cast<int>(cols)};
    double* xc = arena_.get<double>("probe_xc", N * ldx());
    STG_CUDA(cudaMemsetAsync(xc, 0, sizeof(double) * N * ldx(), st_));
    STG_CUDA(cudaMemcpyAsync(xc, X_, sizeof(double) * n * ldx(), cudaMemcpyDeviceToDevice, st_));
    std::vector<double> newvals;
    std::vector<double> w(static_cast<size_t>(pt.n_total * k));
    rayleigh_ritz(pt, b, newvals, false, w.data(), pt.n_total, Blk{xc, ldx()});
    std::memcpy(vals, newvals.data(), sizeof(double) * k);
    for (i64 c = 0; c < k; ++c)
      for (i64 i = 0; i < pt.n_total; ++i) vecs[c * ldv + i] = w[static_cast<size_t>(i * k + c)];
  }

  // Kernel microbenchmark on synthetic operands (development / profiling):
  // which = 0 gram (sym if flag&1), 1 nn (tri if flag&1), 2 chol, 3 triinv,
  // 4 on-device eigensolver (want = m2), 5 masked gram over N rows.
  double bench_kernel(int which, i64 N, int m1, int m2, int flag, int iters) {
    const int ld1 = ld_for(m1), ld2 = ld_for(m2);
    double* A = arena_.get<double>("bk_A", N * ld1);
    double* B = arena_.get<double>("bk_B", N * ld2);
    double* C = arena_.get<double>("bk_C", static_cast<i64>(ld1) * ld2 + static_cast<i64>(m1) * ld1);
    double* O = arena_.get<double>("bk_O", std::max<i64>(N * ld2, static_cast<i64>(m1) * ld2));
    launch(fill_kernel, dim3(blocks(N * ld1)), dim3(256), 0, st_, A, N * ld1, 1e-3);
    launch(fill_kernel, dim3(blocks(N * ld2)), dim3(256), 0, st_, B, N * ld2, 2e-3);
    // SPD-ish small matrix for chol/eig: I + small
    std::vector<double> h(static_cast<size_t>(m1) * ld1, 0.0);
    for (int i = 0; i < m1; ++i)
      for (int j = 0; j < m1; ++j) h[static_cast<size_t>(i) * ld1 + j] = (i == j ? 2.0 + i : 0.0) + 0.01 * std::sin(i * 7.0 + j * 3.0 + (i + j));
    for (int i = 0; i < m1; ++i)
      for (int j = 0; j < i; ++j) h[static_cast<size_t>(i) * ld1 + j] = h[static_cast<size_t>(j) * ld1 + i];
    STG_CUDA(cudaMemcpyAsync(C, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st_));
    cudaEvent_t a, b;
    STG_CUDA(cudaEventCreate(&a));
    STG_CUDA(cudaEventCreate(&b));
    auto run = [&]() {
      switch (which) {
        case 0: gram(A, ld1, (flag & 1) ? A : B, (flag & 1) ? ld1 : ld2, N, m1, (flag & 1) ? m1 : m2, flag & 1, O, ld2); break;
        case 1: nn(A, ld1, N, m1, C, ld1, m2, O, ld2, 1.0, 0.0, nullptr, 0, flag & 1); break;
        case 2: chol(C, ld1, m1, O, ld1, flag ? arena_.get<double>("bk_Ri", static_cast<i64>(m1) * ld1) : nullptr, ld1, nullptr, 0.0, true); break;
        case 3: triinv(C, ld1, m1, O, ld1); break;
        case 4: {
          double* w = arena_.get<double>("bk_w", m1);
          const int saved = cfg.flags;
          cfg.flags &= ~ST_FLAG_CUSOLVER_EIG;
          eig_fast(C, ld1, m1, 0, m2, w, O, ld2);
          cfg.flags = saved;
          break;
        }
        case 5: gram(A, ld1, A, ld1, N, m1, m1, true, O, ld2, 1.0, mark_p_, -12345); break;
      }
    };
    for (int i = 0; i < 2; ++i) run();
    STG_CUDA(cudaEventRecord(a, st_));
    for (int i = 0; i < iters; ++i) run();
    STG_CUDA(cudaEventRecord(b, st_));
    STG_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    STG_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    kdiscard();
    return ms / iters;
  }

  // Run-to-run determinism of a kernel on pseudo-random operands (development
  // and tests): the largest |difference| between `reps` repeated runs and the
  // first. which = 0 Gram A'B (N x m1, N x m2), 1 row-local GEMM A C
  // (N x m1 times m1 x m2), 2 SpMV with the session's operator, 3 SpMM of the
  // session's operator with an n x m1 block.
  double det_check(int which, i64 N, int m1, int m2, int reps, double* first_out = nullptr) {
    const DevCsr& op = is_laplacian() ? T() : A();
    if (which >= 2) N = n;
    const int ld1 = ld_for(m1), ld2 = ld_for(m2);
    double* Aa = arena_.get<double>("dc_A", N * ld1);
    double* Bb = arena_.get<double>("dc_B", N * ld2);
    double* Cc = arena_.get<double>("dc_C", static_cast<i64>(m1) * ld2 + 8);
    const i64 outn = which == 0 ? static_cast<i64>(m1) * ld2 : which == 1 ? N * ld2 : which == 2 ? N : N * ld1;
    double* O = arena_.get<double>("dc_O", outn);
    launch(hash_fill_kernel, dim3(blocks(N * ld1)), dim3(256), 0, st_, Aa, N * ld1, 11ULL);
    launch(hash_fill_kernel, dim3(blocks(N * ld2)), dim3(256), 0, st_, Bb, N * ld2, 22ULL);
    launch(hash_fill_kernel, dim3(blocks(static_cast<i64>(m1) * ld2)), dim3(256), 0, st_, Cc,
           static_cast<i64>(m1) * ld2, 33ULL);
    SpvBufs sp;
    if (which == 2) sp = spv_plan(op.rp, N);
    auto run = [&]() {
      if (which == 0) gram(Aa, ld1, Bb, ld2, N, m1, m2, false, O, ld2);
      if (which == 1) nn(Aa, ld1, N, m1, Cc, ld2, m2, O, ld2, 1.0, 0.0, nullptr, 0);
      if (which == 2) spmv(op, sp.pl, Aa, O, nullptr, 0);
      if (which == 3) {
        SpmmArgs sa{};
        sa.rows = N;
        sa.rowptr = op.rp;
        sa.col = op.col;
        sa.val = op.val;
        sa.X = Aa;
        sa.ldx = ld1;
        sa.m = m1;
        sa.Y = O;
        sa.ldy = ld1;
        ++plan_epoch_;
        do_spmm(sa, op.nnz, N, kSpmmFull, true);
      }
    };
    run();
    std::vector<double> ref(static_cast<size_t>(outn)), cur(static_cast<size_t>(outn));
    STG_CUDA(cudaMemcpyAsync(ref.data(), O, sizeof(double) * outn, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    if (first_out) {  // rows x cols, dense row-major
      const int cols = which == 0 || which == 1 ? m2 : which == 2 ? 1 : m1;
      const int ld = which == 0 || which == 1 ? ld2 : which == 2 ? 1 : ld1;
      const i64 rows = which == 0 ? m1 : N;
      for (i64 i = 0; i < rows; ++i)
        for (int c = 0; c < cols; ++c) first_out[i * cols + c] = ref[static_cast<size_t>(i * ld + c)];
    }
    double md = 0.0;
    for (int r = 0; r < reps; ++r) {
      STG_CUDA(cudaMemsetAsync(O, 0xff, sizeof(double) * outn, st_));  // NaN-poisoned output
      run();
      STG_CUDA(cudaMemcpyAsync(cur.data(), O, sizeof(double) * outn, cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      const int cols = which == 0 || which == 1 ? m2 : which == 2 ? 1 : m1;
      const int ld = which == 0 || which == 1 ? ld2 : which == 2 ? 1 : ld1;
      const i64 rows = which == 0 ? m1 : N;
      for (i64 i = 0; i < rows; ++i)
        for (int c = 0; c < cols; ++c) {
          const size_t q = static_cast<size_t>(i * ld + c);
          const double d = std::fabs(cur[q] - ref[q]);
          if (d != 0.0 && getenv_flag("STG_DET_LOG"))
            fprintf(stderr, "det which %d rep %d row %lld col %d ref %.17g got %.17g\n", which, r,
                    static_cast<long long>(i), c, ref[q], cur[q]);
          md = std::max(md, d == d ? d : 1e300);
        }
    }
    if (which == 2) spv_release(sp);
    kdiscard();
    return md;
  }

  void copy_x_colmajor(double* out, i64 rows) {
    std::vector<double> xr(static_cast<size_t>(rows * k));
    STG_CUDA(cudaMemcpy2DAsync(xr.data(), sizeof(double) * k, X_, sizeof(double) * ldx(), sizeof(double) * k, rows,
                               cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    for (i64 c = 0; c < k; ++c)
      for (i64 i = 0; i < rows; ++i) out[c * rows + i] = xr[static_cast<size_t>(i * k + c)];
  }

  // values and the stored rows of X (all rows, or the owned rows of a shard)
  void get_embedding(double* vals, double* vecs, i64 ld) {
    std::memcpy(vals, values.data(), sizeof(double) * k);
    const i64 rows = nloc_;
    std::vector<double> x(static_cast<size_t>(rows * k));
    copy_x_colmajor(x.data(), rows);
    for (i64 c = 0; c < k; ++c) std::memcpy(vecs + c * ld, x.data() + c * rows, sizeof(double) * rows);
  }

  i64 local_rows() const { return nloc_; }
  void local_ids(i64* ids) const {
    if (!sh_) {
      for (i64 i = 0; i < nloc_; ++i) ids[i] = i;
      return;
    }
    const ShardMap m = host_map();
    for (i64 l = 0; l < nloc_; ++l) ids[l] = sm_global(m, l);
  }

  void get_csr(int which, int* rp, int* col, double* val) {
    DevCsr m;
    if (which == 0) m = A();
    else if (which == 1) {
      if (!is_laplacian()) throw InvalidArgument("st_get_csr: the adjacency session has no shifted operator");
      m = T();
    } else {
      m.n = last_delta_n_;
      m.nnz = last_delta_nnz_;
      m.rp = last_delta_.rp;
      m.col = last_delta_.col;
      m.val = last_delta_.val;
      if (!m.rp) {
        std::fill(rp, rp + n + 1, 0);
        return;
      }
    }
    STG_CUDA(cudaMemcpyAsync(rp, m.rp, sizeof(int) * (m.n + 1), cudaMemcpyDeviceToHost, st_));
    if (m.nnz) {
      STG_CUDA(cudaMemcpyAsync(col, m.col, sizeof(int) * m.nnz, cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaMemcpyAsync(val, m.val, sizeof(double) * m.nnz, cudaMemcpyDeviceToHost, st_));
    }
    STG_CUDA(cudaStreamSynchronize(st_));
  }

 private:
  Arena arena_;
  Pinned pin_;
  cudaStream_t st_ = nullptr, st_rng_ = nullptr;
  cudaEvent_t ev_rng_ = nullptr;
  cudaStream_t st_eig_ = nullptr;  // the sketch's eigensolve (few SMs) runs beside the basis work
  cudaEvent_t ev_gb_ = nullptr, ev_eig_ = nullptr;
  // the adjacency merge's entry copy (A_next's col/val; nothing in the step
  // reads them) runs beside the basis work; joined before the graph commits
  // and before the next ingest touches the spare slot or the Delta marks
  cudaStream_t st_mg_ = nullptr;
  cudaStream_t st_rot_ = nullptr;  // the X rotation, overlapped with the next step's ingestion
  cudaEvent_t ev_rot_ready_ = nullptr, ev_rot_done_ = nullptr;
  bool rot_pending_ = false;
  const bool rot_aside_ = !getenv_flag("STG_ROT_INLINE");  // development A/B
  cudaEvent_t ev_mg_fork_ = nullptr, ev_mg_ = nullptr;
  cudaEvent_t tev_[8];
  int tev_n_ = 0;
  cusolverDnHandle_t solver_ = nullptr;
  Scalars* hs_ = nullptr;
  int* sched_ctr_ = nullptr;
  int sched_slot_ = 0;  // 0 main stream, 1 the K Gram's side stream, 2 the rotation stream
  int* sched_ctr() { return sched_ctr_ + 16 * sched_slot_; }
  u64* d_scal_ = nullptr;  // [0] err_edit [1] err_apply [2] nvalid [3] flags(int) [4] info(int)
  DevCsr A_[2], T_[2];
  int acur_ = 0, tcur_ = 0;
  double* d_alpha_ = nullptr;  // [0] current [1] next [2] dmax
  double* X_ = nullptr;
  i64 xcap_ = 0;
  double* d_values_ = nullptr;
  int* mark_delta_ = nullptr;
  int* mark_p_ = nullptr;
  int* posmap_ = nullptr;
  i64 nodecap_ = 0;
  int stamp_ = 0;
  DevCsr last_delta_;
  i64 last_delta_nnz_ = 0, last_delta_n_ = 0;
  // pending (uncommitted) next graph
  int anext_ = -1, tnext_ = -1;
  double alpha_next_ = 0.0;

  struct PendingK {
    int cls;
    cudaEvent_t a, b;
    double work, work2;
    char tag[48];
  };
  char ktag_[48] = {0};  // optional shape tag for the next kbegin (STG_KLOG)
  std::vector<PendingK> pend_;
  std::vector<cudaEvent_t> evpool_;
  size_t evnext_ = 0;
  bool ktiming() const { return cfg.flags & ST_FLAG_KERNEL_TIMING; }
  const bool klog_ = getenv("STG_KLOG") != nullptr;
  cudaEvent_t next_event() {
    if (evnext_ == evpool_.size()) {
      cudaEvent_t e;
      STG_CUDA(cudaEventCreate(&e));
      evpool_.push_back(e);
    }
    return evpool_[evnext_++];
  }
  std::vector<size_t> open_;  // kbegin/kend nest (e.g. the rotation contains a GEMM)
  void kbegin(int cls, double work, cudaStream_t s = nullptr, double work2 = 0.0) {
    if (!ktiming()) return;
    PendingK p{cls, next_event(), next_event(), work, work2, {0}};
    std::memcpy(p.tag, ktag_, sizeof(p.tag));
    ktag_[0] = 0;
    STG_CUDA(cudaEventRecord(p.a, s ? s : st_));
    open_.push_back(pend_.size());
    pend_.push_back(p);
  }
  void kend(cudaStream_t s = nullptr) {
    if (!ktiming()) return;
    STG_CUDA(cudaEventRecord(pend_[open_.back()].b, s ? s : st_));
    open_.pop_back();
  }
 public:
  void kflush() {
    if (pend_.empty()) return;
    STG_CUDA(cudaDeviceSynchronize());
    for (auto& p : pend_) {
      float ms = 0;
      STG_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
      kstats[p.cls].ms += ms;
      kstats[p.cls].work += p.work;
      kstats[p.cls].work2 += p.work2;
      kstats[p.cls].launches += 1;
      const bool flop_cls = p.cls == kGram || p.cls == kGemm || p.cls == kKcGram || p.cls == kGramNarrow ||
                            p.cls == kGemmNarrow;
      const bool byte_cls = p.cls == kSpmm || p.cls == kSpmmSketch || p.cls == kMerge || p.cls == kRotate ||
                            p.cls == kSpmmFull;
      if (flop_cls) kstats[p.cls].bound_ms += 1e3 * std::max(p.work / (peak_tflops_ * 1e12), p.work2 / (peak_gbs_ * 1e9));
      if (byte_cls) kstats[p.cls].bound_ms += 1e3 * std::max(p.work / (peak_gbs_ * 1e9), p.work2 / (peak_tflops_ * 1e12));
      if (klog_) {
        float t0 = 0;  // start offset from the step's first timed launch (timeline across streams)
        cudaEventElapsedTime(&t0, pend_.front().a, p.a);
        fprintf(stderr, "klog cls=%d %-40s %9.1f us  @%8.1f us  work=%.3g  rate=%.3g/s\n", p.cls, p.tag, 1e3 * ms,
                1e3 * t0, p.work, ms > 0 ? p.work / (ms * 1e-3) : 0.0);
      }
    }
    pend_.clear();
    open_.clear();
    evnext_ = 0;
  }
  void kdiscard() {
    pend_.clear();
    open_.clear();
    evnext_ = 0;
  }
  void kreset() {
    for (auto& k : kstats) k = KStat{};
  }

 private:
  int ldx() const { return static_cast<int>(k % 2 ? k + 1 : k); }
  int* flags_ptr() { return reinterpret_cast<int*>(d_scal_ + 3); }
  int* info_ptr() { return reinterpret_cast<int*>(d_scal_ + 4); }
  int* side_flags_ptr() { return reinterpret_cast<int*>(d_scal_ + 5); }
  int* sticky_ptr() { return reinterpret_cast<int*>(d_scal_ + 8); }

  template <typename K, typename... Args>
  void launch(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    kernel<<<grid, block, smem, s>>>(args...);
    STG_LAUNCH();
    ++launches;
  }
  static unsigned blocks(i64 n, int b = 256) { return static_cast<unsigned>(std::max<i64>(1, cdiv(n, b))); }

  // ---------------------------------------------------------------- timing
  void timing_begin() {
    ntimings = 0;
    if (cfg.flags & ST_FLAG_TIMING) STG_CUDA(cudaEventRecord(tev_[0], st_));
  }
  void timing_mark(int slot) {
    if (cfg.flags & ST_FLAG_TIMING) STG_CUDA(cudaEventRecord(tev_[slot + 1], st_));
  }
  void timing_end(int last) {
    if (!(cfg.flags & ST_FLAG_TIMING)) return;
    STG_CUDA(cudaEventRecord(tev_[7], st_));
    STG_CUDA(cudaEventSynchronize(tev_[7]));
    float ms = 0;
    for (int i = 0; i < 6; ++i) timings[i] = 0;
    (void)last;
    STG_CUDA(cudaEventElapsedTime(&ms, tev_[0], tev_[7]));
    timings[5] = ms;
    ntimings = 6;
    // phase marks 1..4 are recorded when reached
    float a;
    if (cudaEventElapsedTime(&a, tev_[0], tev_[1]) == cudaSuccess) timings[0] = a;
    if (cudaEventElapsedTime(&a, tev_[1], tev_[2]) == cudaSuccess) timings[1] = a;
    if (cudaEventElapsedTime(&a, tev_[2], tev_[3]) == cudaSuccess) timings[2] = a;
    if (cudaEventElapsedTime(&a, tev_[3], tev_[4]) == cudaSuccess) timings[3] = a;
    if (cudaEventElapsedTime(&a, tev_[4], tev_[7]) == cudaSuccess) timings[4] = a;
    (void)cudaGetLastError();  // unrecorded phase events (empty steps) are not errors
  }

  static u64 mix_seed(u64 base, u64 salt) {  // rng.hpp:16-21
    u64 z = base + 0x9e3779b97f4a7c15ULL * (salt + 0x632be59bd9b4e019ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }

  DevCsr alloc_csr(const std::string& name, i64 nrows, i64 nnz) {
    DevCsr m;
    m.n = nrows;
    m.nnz = nnz;
    m.rp = arena_.get<int>(name + ".rp", nrows + 1);
    m.col = arena_.get<int>(name + ".col", nnz);
    m.val = arena_.get<double>(name + ".val", nnz);
    return m;
  }

  // need: global node count (marks, posmap); need_x: rows of the X storage
  // (the owned rows of a sharded session).
  void ensure_node_capacity(i64 need, i64 need_x = -1) {
    if (need_x < 0) need_x = need;
    if (need_x > xcap_ || !X_) {
      wait_rotation();  // X is copied and released below
      const i64 cap = std::max<i64>(need_x + need_x / 4, 1024);
      double* nx = static_cast<double*>(arena_.alloc(sizeof(double) * cap * ldx()));
      if (X_) {  // stream-ordered copy and free (no host or device-wide sync)
        STG_CUDA(cudaMemcpyAsync(nx, X_, sizeof(double) * xcap_ * ldx(), cudaMemcpyDeviceToDevice, st_));
        arena_.release(X_);
      }
      X_ = nx;
      if (sh_) {
        mark_dl_ = arena_.get<int>("mark_dl_" + std::to_string(cap), cap);
        STG_CUDA(cudaMemsetAsync(mark_dl_, 0xff, sizeof(int) * cap, st_));
      }
      xcap_ = cap;
    }
    if (need <= nodecap_) return;
    const i64 cap = std::max<i64>(need + need / 4, 1024);
    // fresh mark arrays start at -1 (stamps are per step and always >= 1)
    mark_delta_ = arena_.get<int>("mark_delta_" + std::to_string(cap), cap);
    mark_p_ = arena_.get<int>("mark_p_" + std::to_string(cap), cap);
    posmap_ = arena_.get<int>("posmap_" + std::to_string(cap), cap);
    STG_CUDA(cudaMemsetAsync(mark_delta_, 0xff, sizeof(int) * cap, st_));
    STG_CUDA(cudaMemsetAsync(mark_p_, 0xff, sizeof(int) * cap, st_));
    nodecap_ = cap;
  }

  // ---------------------------------------------------------------- linear algebra helpers
  void gram(const double* A, int lda, const double* B, int ldb, i64 rows, int m1, int m2, bool sym, double* out,
            int ldo, double alpha = 1.0, const int* mask = nullptr, int mask_val = 0) {
    if (m1 <= 0 || m2 <= 0) return;
    dm::GramArgs a{};
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.nrows = rows;
    a.m1 = m1;
    a.m2 = m2;
    // layout: 64 x 64 tiles, or 32 x 128 / 128 x 32 when one side is <= 32 wide
    const bool narrow = m1 <= 32 && m2 <= 32;
    const int layout = narrow ? -1 : (!sym && m1 <= 32) ? 1 : (!sym && m2 <= 32) ? 2 : 0;
    const int TA = layout == 1 ? 32 : layout == 2 ? 128 : 64;
    const int TB = layout == 1 ? 128 : layout == 2 ? 32 : 64;
    a.tiles_i = static_cast<int>(cdiv(m1, TA));
    a.tiles_j = static_cast<int>(cdiv(m2, TB));
    a.sym = sym ? 1 : 0;
    a.mask = mask;
    a.mask_val = mask_val;
    if (narrow) a.tiles_i = a.tiles_j = 1;
    const int ntiles = narrow ? 1 : (sym ? a.tiles_i * (a.tiles_i + 1) / 2 : a.tiles_i * a.tiles_j);
    static const int env_waves = getenv("STG_GRAM_WAVES") ? atoi(getenv("STG_GRAM_WAVES")) : 0;  // development scans
    // split-K CTAs. Below 256k rows (cfg3: ~107k stacked rows) ~2 waves per output tile, 3..12 (a per-shape
    // sweep: 200 x 200 sym (10 tiles) best at 12, 64 x 64 at 3, 64 x 100 at 3-4, 164 x 100 at 12; fewer splits
    // = less partial traffic); above (cfg4/cfg5), 24 waves for square tiles and 4 for 32 x 128 tiles (the
    // tail of unequal tiles outweighs the partials there: cfg4's Grams 28.5 vs 30.0 ms per step)
    // (the persistent row-split kernel balances its tiles itself: 8 waves measured best, fewer partials)
    const int wcap = layout == 0 && gram_rs_ && gram_persist_ && !mask ? 8 : 12;
    const int waves = rows >= (1 << 18) ? (layout == 0 ? 24 : 4) : std::min(wcap, std::max(3, 2 * ntiles));
    const i64 target = 148 * (env_waves > 0 ? env_waves : waves);
    const i64 rows_min = narrow ? 256 : 128;
    i64 splits = std::max<i64>(1, std::min<i64>(cdiv(std::max<i64>(rows, 1), rows_min), cdiv(target, ntiles)));
    splits = std::min<i64>(splits, 65535);
    a.rows_per_split = round_up(cdiv(std::max<i64>(rows, 1), splits), narrow ? dm::SBK : dm::BK2);
    splits = std::max<i64>(1, cdiv(std::max<i64>(rows, 1), a.rows_per_split));
    const i64 m1p = narrow ? 32 : static_cast<i64>(a.tiles_i) * TA;
    const i64 m2p = narrow ? 32 : static_cast<i64>(a.tiles_j) * TB;
    a.partial = arena_.get<double>(gram_partial_tag_, splits * m1p * m2p);
    if (klog_) snprintf(ktag_, sizeof(ktag_), "gram %lldx%dx%d%s", rows, m1, m2, sym ? " sym" : "");
    kbegin(mask ? kKcGram : narrow ? kGramNarrow : kGram,
           sym ? static_cast<double>(rows) * m1 * (m1 + 1) : 2.0 * rows * m1 * m2, nullptr,
           8.0 * rows * (sym ? m1 : m1 + m2) + 8.0 * m1 * m2);
    const dim3 grid(ntiles, static_cast<unsigned>(splits));
    const bool aligned = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                         lda % 2 == 0 && ldb % 2 == 0;
    const bool bulk = !mask && aligned;
    if (narrow && aligned) {  // the streaming kernel (a row mask zeroes the masked rows' fragments)
      const bool same = A == B && lda == ldb;
      const CUtensorMap ma = make_tmap_2d(A, rows, m1, lda, dm::kStreamPitch, dm::kGsRows);
      const CUtensorMap mb = make_tmap_2d(B, rows, m2, ldb, dm::kStreamPitch, dm::kGsRows);
      const int ntl = static_cast<int>(cdiv(std::max<i64>(rows, 1), dm::kGsRows));
      const int G = std::min(ntl, 148 * (same ? 3 : 1));
      a.partial = arena_.get<double>(gram_partial_tag_, static_cast<i64>(G) * 1024);
      launch(dm::gram_stream_kernel, dim3(static_cast<unsigned>(G)), dim3(dm::NT), dm::gram_stream_smem(same), st_,
             a, ma, mb, same ? 1 : 0, ntl);
      gram_reduce(a.partial, G, m1, m2, 32, 32, a.sym, out, ldo, alpha);
      kend();
      return;
    }
    if (narrow)
      launch(dm::gram_tn_small_kernel, grid, dim3(dm::NT), 0, st_, a);
    else if (bulk && gram_persist_ && rows > 0 && rows < (1LL << 31) &&
             (persist_always_ || static_cast<i64>(ntiles) * splits > 148 * (layout == 0 ? STG_GRAM_MINB : 2)) &&
             static_cast<i64>(ntiles) * splits < (1LL << 30)) {
      const bool rs = layout == 0 && gram_rs_;
      const CUtensorMap ma = make_tmap_2d(A, rows, m1, lda, TA + 4, rs ? dm::kRsBK : dm::kBK);
      const CUtensorMap mb = make_tmap_2d(B, rows, m2, ldb, TB + 4, rs ? dm::kRsBK : dm::kBK);
      const dim3 pg(148 * (layout == 0 ? STG_GRAM_MINB : 2));
      const int nsp = static_cast<int>(splits);
      if (rs && gram_order_) {
        // blocks of about gram_block_waves_ waves of items (0: one block, tile major over the whole product)
        static const int bw = getenv("STG_GRAM_BLOCK_WAVES") ? atoi(getenv("STG_GRAM_BLOCK_WAVES")) : 0;  // development A/B
        dm::gram_tile_order(a, ntiles, nsp, bw > 0 ? std::max(1, bw * static_cast<int>(pg.x) / ntiles) : 0);
      }
      if (layout == 1)
        launch(dm::gram_persist_kernel<1, 4>, pg, dim3(dm::kRsThreads), dm::gram_tma_smem<1, 4>(), st_, a, ma, mb, ntiles,
               nsp,
               sched_ctr());
      else if (layout == 2)
        launch(dm::gram_persist_kernel<4, 1>, pg, dim3(dm::kRsThreads), dm::gram_tma_smem<4, 1>(), st_, a, ma, mb, ntiles,
               nsp,
               sched_ctr());
      else if (rs)
        launch(dm::gram_persist_rs_kernel, pg, dim3(dm::kRsThreads), dm::kRsSmem, st_, a, ma, mb, ntiles, nsp,
               sched_ctr());
      else
        launch(dm::gram_persist_kernel<2, 2>, pg, dim3(dm::kRsThreads), dm::gram_tma_smem<2, 2>(), st_, a, ma, mb, ntiles,
               nsp,
               sched_ctr());
    }
    else if (bulk) {
      const CUtensorMap ma = make_tmap_2d(A, rows, m1, lda, TA + 4, dm::kBK);
      const CUtensorMap mb = make_tmap_2d(B, rows, m2, ldb, TB + 4, dm::kBK);
      if (layout == 1)
        launch(dm::gram_tma_kernel<1, 4>, grid, dim3(dm::NT), dm::gram_tma_smem<1, 4>(), st_, a, ma, mb);
      else if (layout == 2)
        launch(dm::gram_tma_kernel<4, 1>, grid, dim3(dm::NT), dm::gram_tma_smem<4, 1>(), st_, a, ma, mb);
      else
        launch(dm::gram_tma_kernel<2, 2>, grid, dim3(dm::NT), dm::gram_tma_smem<2, 2>(), st_, a, ma, mb);
    }
    else if (layout == 1)
      launch(dm::gram_tn_kernel<1, 4>, grid, dim3(dm::NT), dm::gram_smem(1, 4), st_, a);
    else if (layout == 2)
      launch(dm::gram_tn_kernel<4, 1>, grid, dim3(dm::NT), dm::gram_smem(4, 1), st_, a);
    else
      launch(dm::gram_tn_kernel<2, 2>, grid, dim3(dm::NT), dm::gram_smem(2, 2), st_, a);
    gram_reduce(a.partial, splits, m1, m2, m1p, m2p, a.sym, out, ldo, alpha);
    kend();
  }

  // deterministic split-K reduction of the Gram partials (chunked: the splits
  // cut into consecutive chunks summed by separate warps, then in chunk order)
  void gram_reduce(const double* partial, i64 splits, int m1, int m2, i64 m1p, i64 m2p, int sym, double* out, int ldo,
                   double alpha) {
    static const bool old = getenv_flag("STG_GRAM_REDUCE_OLD");  // development A/B
    if (old) {
      launch(dm::gram_reduce_kernel, dim3(blocks(static_cast<i64>(m1) * m2)), dim3(256), 0, st_, partial,
             static_cast<int>(splits), m1, m2, static_cast<int>(m1p), static_cast<int>(m2p), sym, out, ldo, alpha);
      return;
    }
    const int ch = dm::gram_reduce_chunks(splits);
    launch(dm::gram_reduce_chunked_kernel, dim3(static_cast<unsigned>(cdiv(static_cast<i64>(m1) * m2, 32))),
           dim3(32 * ch), 0, st_, partial, static_cast<int>(splits), m1, m2, static_cast<int>(m1p),
           static_cast<int>(m2p), sym, out, ldo, alpha);
  }

  // Gram over rows partitioned across the ranks of a sharded session: local
  // split-K partial, allreduce, copy out (symmetric results re-mirrored).
  void pgram(const double* A, int lda, const double* B, int ldb, i64 rows, int m1, int m2, bool sym, double* out,
             int ldo) {
    if (!sh_) {
      gram(A, lda, B, ldb, rows, m1, m2, sym, out, ldo);
      return;
    }
    if (m1 <= 0 || m2 <= 0) return;
    const i64 mm = static_cast<i64>(m1) * m2;
    double* tmp = arena_.get<double>("pg_tmp", mm);
    if (rows > 0) gram(A, lda, B, ldb, rows, m1, m2, sym, tmp, m2);
    else STG_CUDA(cudaMemsetAsync(tmp, 0, sizeof(double) * mm, st_));
    allreduce(tmp, mm);
    if (shard_debug_) {  // development: checksums of the reduced Grams, in call order
      std::vector<double> h(static_cast<size_t>(mm));
      STG_CUDA(cudaMemcpyAsync(h.data(), tmp, sizeof(double) * mm, cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      double sum = 0, sa = 0;
      for (double v : h) { sum += v; sa += std::fabs(v); }
      fprintf(stderr, "[r%d] pgram %d x %d rows %lld sum %.15e abs %.15e\n", comm_.rank, m1, m2,
              static_cast<long long>(rows), sum, sa);
    }
    launch(gram_out_kernel, dim3(blocks(mm)), dim3(256), 0, st_, static_cast<const double*>(tmp), m1, m2, sym ? 1 : 0,
           out, ldo);
  }

  // Dense SpMM operand over the rows of P: the stacked block itself, or in a
  // sharded session [own rows of P | the remote rows the owned Delta rows
  // reference] (the boundary-row halo planned in ingest_shard_tail).
  const double* halo(const Pert& pt, const double* X, int ldx, int m, int* ld_out) {
    if (!sh_) {
      *ld_out = ldx;
      return X;
    }
    const int ldh = ld_for(m);
    double* buf = arena_.get<double>("halo_buf", std::max<i64>(pt.p + pt.nrecv, 1) * ldh);
    double* send = arena_.get<double>("halo_send", std::max<i64>(pt.nsend, 1) * ldh);
    if (pt.p > 0) launch(copy2d_kernel, dim3(blocks(pt.p * m)), dim3(256), 0, st_, X, ldx, buf, ldh, pt.p, m);
    if (pt.nsend > 0)
      launch(gather_rows_kernel, dim3(blocks(pt.nsend * m)), dim3(256), 0, st_, X, ldx, pt.hsend, pt.nsend, m, send,
             ldh);
    std::vector<i64> sb(pt.send_rows.size()), rb(pt.recv_rows.size());
    const i64 rowb = static_cast<i64>(sizeof(double)) * ldh;
    for (size_t r = 0; r < sb.size(); ++r) sb[r] = pt.send_rows[r] * rowb;
    for (size_t r = 0; r < rb.size(); ++r) rb[r] = pt.recv_rows[r] * rowb;
    alltoallv(send, sb, buf + pt.p * ldh, rb);
    halo_bytes_recv_ += pt.nrecv * rowb;
    halo_bytes_local_ += pt.p * rowb;
    ++halo_calls_;
    *ld_out = ldh;
    return buf;
  }

  void nn(const double* A, int lda, i64 rows, int m1, const double* C, int ldc, int m2, double* Out, int ldo,
          double alpha, double beta, const double* B, int ldb, bool tri = false, bool gated = false) {
    if (rows <= 0 || m2 <= 0) return;
    dm::NNArgs a{};
    a.A = A;
    a.lda = lda;
    a.nrows = rows;
    a.m1 = m1;
    a.C = C;
    a.ldc = ldc;
    a.m2 = m2;
    a.Bm = B;
    a.ldb = ldb;
    a.Out = Out;
    a.ldo = ldo;
    a.alpha = alpha;
    a.beta = beta;
    a.upper_tri_c = tri ? 1 : 0;
    if (gated) {  // skip when the step has already failed (keeps a failed step side-effect free)
      a.skip_flags = flags_ptr();
      a.skip_mask = kNonFinite | kNotOrthonormal | kSpecFail;
      a.skip_info = info_ptr();
    }
    if (klog_) snprintf(ktag_, sizeof(ktag_), "nn %lldx%dx%d%s", rows, m1, m2, tri ? " tri" : "");
    kbegin(m2 <= 32 ? kGemmNarrow : kGemm, tri ? static_cast<double>(rows) * m1 * (m1 + 1) : 2.0 * rows * m1 * m2,
           nullptr, 8.0 * rows * (m1 + m2 + (beta != 0.0 ? m2 : 0)) + 8.0 * m1 * m2);
    if (m2 <= 32)
    {
      const bool stream = m1 <= 32 && beta == 0.0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 && lda % 2 == 0 &&
                          (reinterpret_cast<uintptr_t>(Out) & 15) == 0 && ldo % 2 == 0;
      if (stream) {
        const CUtensorMap ma = make_tmap_2d(A, rows, m1, lda, dm::kStreamPitch, dm::kStreamRows);
        const int ntiles = static_cast<int>(cdiv(rows, dm::kStreamRows));
        const int G = std::min(ntiles, 148 * 2);
        launch(dm::gemm_nn_stream_kernel, dim3(static_cast<unsigned>(G)), dim3(dm::NT), dm::kStreamSmem, st_, a, ma,
               ntiles);
      } else {
        launch(dm::gemm_nn_small_kernel, dim3(static_cast<unsigned>(cdiv(rows, dm::NBM))), dim3(dm::NT), 0, st_, a);
      }
    }
    else
    {
      const dim3 grid(static_cast<unsigned>(cdiv(rows, dm::BM) * cdiv(m2, dm::BN)));
      static const bool no_tma = getenv_flag("STG_NN_NOTMA");  // development A/B
      const bool tma = !no_tma && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(C)) & 15) == 0 &&
                       lda % 2 == 0 && ldc % 2 == 0;
      static const bool no_persist = getenv_flag("STG_NN_NOPERSIST");  // development A/B
      const i64 ntr = cdiv(rows, dm::BM), tiles_j = cdiv(m2, dm::BN);
      const int Gp = 148 * dm::nnp_ctas(beta != 0.0);
      if (tma && !no_persist && m1 > 0 && (persist_always_ || ntr * tiles_j > Gp) && ntr * tiles_j < (1LL << 30)) {
        const CUtensorMap ma = make_tmap_2d(A, rows, m1, lda, dm::SAR2, dm::BM);
        const CUtensorMap mc = make_tmap_2d(C, m1, m2, ldc, dm::SST, dm::BK2);
        launch(beta != 0.0 ? dm::gemm_nn_persist_kernel<true> : dm::gemm_nn_persist_kernel<false>, dim3(Gp),
               dim3(dm::kRsThreads), dm::nnp_smem(beta != 0.0), st_, a, ma, mc, static_cast<int>(ntr), sched_ctr());
      } else if (tma) {
        const CUtensorMap ma = make_tmap_2d(A, rows, m1, lda, dm::SAR2, dm::BM);
        const CUtensorMap mc = make_tmap_2d(C, m1, m2, ldc, dm::SST, dm::BK2);
        launch(beta != 0.0 ? dm::gemm_nn_tma_kernel<true> : dm::gemm_nn_tma_kernel<false>, grid, dim3(dm::NT),
               dm::kNNTmaSmem, st_, a, ma, mc);
      } else {
        launch(beta != 0.0 ? dm::gemm_nn_kernel<true> : dm::gemm_nn_kernel<false>, grid, dim3(dm::NT), dm::kNNSmem,
               st_, a);
      }
    }
    kend();
  }

  // CSR x dense with compulsory-traffic accounting: 12 B per nonzero, the row
  // pointers, and one read of each referenced dense row plus the output rows.
  // Segment plans (spmm.cuh) of the CSR row ranges multiplied in this step,
  // keyed by (rowptr, row_off, rows); rebuilt after every ingestion.
  struct PlanEntry {
    const int* rowptr;
    i64 row_off, rows, nnz;
    int epoch;
    SpmmPlan pl;
    i64 vmax, split_max, smax;
    std::string tag;
  };
  std::vector<PlanEntry> plans_;
  int plan_epoch_ = 0;
  const bool spmm_fused_ = !getenv_flag("STG_SPMM_UNFUSED");  // development A/B
  const bool gram_persist_ = !getenv_flag("STG_GRAM_NOPERSIST");  // development A/B
  const bool gram_rs_ = !getenv_flag("STG_GRAM_NORS");  // development A/B
  const bool eager_plans_ = !getenv_flag("STG_NO_EAGER_PLANS");  // development A/B
  // tests: the persistent kernels also for products with fewer tiles than CTAs (small graphs)
  const bool persist_always_ = getenv_flag("STG_PERSIST_ALWAYS");
  const bool gram_order_ = !getenv_flag("STG_GRAM_NOORDER");  // development A/B
  const char* gram_partial_tag_ = "gram_partial";  // the side stream's Grams use their own split-K buffer
  // K = X_out'X_out and its Cholesky computed on st_eig_ right after P's marks,
  // while the host waits for |P| (the rows of P masked instead of zeroed)
  const bool k_early_ = !getenv_flag("STG_NO_K_EARLY");  // development A/B
  cudaEvent_t ev_k_ = nullptr;
  bool k_ready_ = false;
  const int spmm_fused_min_m_ = getenv("STG_SPMM_FUSED_MIN_M") ? atoi(getenv("STG_SPMM_FUSED_MIN_M")) : 129;
  const bool spmm_chunked_ = !getenv_flag("STG_SPMM_NOCHUNK");  // development A/B
  const int spmm_chunk_tmax_ = getenv("STG_SPMM_TMAX") ? atoi(getenv("STG_SPMM_TMAX")) : 1;  // development A/B (1 measured best)
  const int merge_mode_ = getenv("STG_MERGE_MODE") ? atoi(getenv("STG_MERGE_MODE")) : 3;  // development A/B

  PlanEntry& spmm_plan(const SpmmArgs& a, i64 nnz) {
    for (auto& e : plans_)
      if (e.epoch == plan_epoch_ && e.rowptr == a.rowptr && e.row_off == a.row_off && e.rows == a.rows) return e;
    PlanEntry* e = nullptr;
    for (auto& q : plans_)
      if (q.epoch != plan_epoch_) { e = &q; break; }
    if (!e) {
      plans_.emplace_back();
      e = &plans_.back();
      e->tag = "sp" + std::to_string(plans_.size() - 1) + "_";
    }
    e->rowptr = a.rowptr;
    e->row_off = a.row_off;
    e->rows = a.rows;
    e->nnz = nnz;
    e->epoch = plan_epoch_;
    e->vmax = nnz / (kSegNnz + 1) + 1;  // segments of the rows longer than kSegNnz (each >= 33 entries)
    e->split_max = std::min<i64>(a.rows, nnz / (kLongSeg + 1));  // rows of more than one segment
    e->smax = 2 * cdiv(nnz, kLongSeg) + 1;
    int* cnt = arena_.get<int>(e->tag + "cnt", a.rows + 1);
    int* cnt2 = arena_.get<int>(e->tag + "cnt2", a.rows + 1);
    int* slen = arena_.get<int>(e->tag + "slen", a.rows + 1);
    int* sptr = arena_.get<int>(e->tag + "sptr", a.rows + 1);
    const int nch = static_cast<int>((nnz + a.rows) / kChunk + 1);
    int* crow = arena_.get<int>(e->tag + "crow", nch + 1);
    int* vstart = arena_.get<int>(e->tag + "vstart", a.rows + 1);
    int* sstart = arena_.get<int>(e->tag + "sstart", a.rows + 1);
    int* vrow = arena_.get<int>(e->tag + "vrow", e->vmax);
    int* split_rows = arena_.get<int>(e->tag + "split", std::max<i64>(e->split_max, 1));
    int* nsplit = arena_.get<int>(e->tag + "nsplit", 1);
    launch(seg_count_kernel, dim3(blocks(a.rows + 1)), dim3(256), 0, st_, a.rowptr, a.row_off, a.rows, cnt, cnt2,
           slen);
    scan_int(cnt, vstart, a.rows + 1);
    scan_int(cnt2, sstart, a.rows + 1);
    scan_int(slen, sptr, a.rows + 1);
    launch(chunk_start_kernel, dim3(blocks(a.rows + 1)), dim3(256), 0, st_, static_cast<const int*>(sptr), a.rows, nch,
           crow);
    STG_CUDA(cudaMemsetAsync(nsplit, 0, sizeof(int), st_));
    launch(seg_fill_kernel, dim3(blocks(a.rows)), dim3(256), 0, st_, static_cast<const int*>(vstart), a.rows, vrow,
           split_rows, nsplit);
    int* segcnt = arena_.get<int>(e->tag + "segcnt", 4 * e->smax);  // per long row and column slab (<= 4)
    STG_CUDA(cudaMemsetAsync(segcnt, 0, sizeof(int) * 4 * e->smax, st_));  // the fused kernels' arrival counters
    e->pl = SpmmPlan{vrow, vstart, sstart, split_rows, nsplit, nullptr, 0, segcnt, sptr, crow, nch};
    return *e;
  }

  // transient: size the segment scratch from the plan's real long-row segment
  // count (one read-back) in a stream-ordered allocation freed after the
  // product, instead of the step's worst-case persistent buffer (monitoring
  // calls over the full operator).
  void do_spmm(const SpmmArgs& a, i64 nnz, i64 distinct_cols, int cls = kSpmm, bool transient = false) {
    if (a.rows <= 0 || a.m <= 0) return;
    PlanEntry& pe = spmm_plan(a, nnz);
    if (klog_) snprintf(ktag_, sizeof(ktag_), "spmm %lld rows m=%d", a.rows, a.m);
    SpmmPlan pl = pe.pl;
    pl.lds = static_cast<int>(round_up(std::min(a.m, 256), 2));
    double* tscratch = nullptr;
    if (transient) {
      int segs = 0;
      STG_CUDA(cudaMemcpyAsync(&segs, pe.pl.sstart + a.rows, sizeof(int), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      STG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tscratch),
                               sizeof(double) * std::max<i64>(segs, 1) * pl.lds, st_));
      pl.scratch = tscratch;
    } else {
      pl.scratch = arena_.get<double>("spmm_scratch", pe.smax * pl.lds);
    }
    kbegin(cls, 12.0 * nnz + 4.0 * (a.rows + 1) + 8.0 * a.m * (a.rows + distinct_cols), nullptr, 2.0 * nnz * a.m);
    for (int c0 = 0; c0 < a.m; c0 += 256) {  // dense blocks wider than 256 columns: 256-column slabs
      SpmmArgs b = a;
      b.X = a.X + c0;
      b.Y = a.Y + c0;
      b.m = std::min(a.m - c0, 256);
      const bool long_rows = nnz > kSegNnz;
      if (spmm_fused_ && b.m >= spmm_fused_min_m_) {  // one launch: segments, their ordered fix-up and the row groups
        spmm_fused_launch(b, pl, long_rows ? pe.vmax : 0, st_);
        launches += 1;
      } else if (spmm_chunked_) {  // one launch: segments, then streamed row chunks, per column slab
        spmm_chunk_launch(b, pl, long_rows ? pe.vmax : 0, spmm_chunk_tmax_, st_);
        launches += 1;
      } else {
        spmm_launch(b, pl, pe.vmax, pe.split_max, long_rows, st_);
        launches += 1 + (long_rows ? 1 : 0) + (pe.split_max > 0 ? 1 : 0);
      }
    }
    kend();
    if (tscratch) STG_CUDA(cudaFreeAsync(tscratch, st_));
  }

  // Cholesky G = R'R; with Ri also R^-1 (triinv_kernel on R', written by chol).
  void chol(const double* G, int ldg, int w, double* R, int ldr, double* Ri, int ldi, const double* orig2,
            double tau2, bool psd, const int* gate = nullptr) {
    if (w > kCholMaxW) throw RuntimeError("chol: block wider than 238 columns");
    if (klog_) snprintf(ktag_, sizeof(ktag_), "chol w=%d", w);
    kbegin(kChol, static_cast<double>(w) * w * w / 3.0);
    const int ldt = ld_for(w);
    double* Rt = Ri ? arena_.get<double>("chol_Rt", static_cast<i64>(w) * ldt) : nullptr;
    launch(chol_kernel, dim3(1), dim3(kCholThreads), chol_smem_bytes(w), st_, G, ldg, w, R, ldr, Rt, ldt, orig2, tau2,
           psd ? 1 : 0, flags_ptr(), static_cast<const int*>(gate));
    kend();
    if (Ri) triinv(Rt, ldt, w, Ri, ldi, gate);
  }

  // R^-1 of a Gram that is the identity to rounding (second CholQR pass): the
  // first-order factor when max|G - I| <= kNearIdTol, else the Cholesky path
  // (decided on the device: the gated kernels exit at once when not needed).
  void chol_inverse_near_identity(const double* G, int ldg, int w, double* R, int ldr, double* Ri, int ldi) {
    int* gate = reinterpret_cast<int*>(d_scal_ + 6);
    launch(near_identity_inverse_kernel, dim3(1), dim3(1024), 0, st_, G, ldg, w, Ri, ldi, gate);
    chol(G, ldg, w, R, ldr, Ri, ldi, nullptr, 0.0, false, gate);
  }

  // R^-1 from R' (row-major, lower triangle)
  void triinv(const double* Rt, int ldrt, int w, double* Ri, int ldi, const int* gate = nullptr) {
    if (w > kCholMaxW) throw RuntimeError("triinv: block wider than 238 columns");
    kbegin(kTriinv, static_cast<double>(w) * w * w / 3.0);
    launch(triinv_kernel, dim3(static_cast<unsigned>(cdiv(w, kTriWarps))), dim3(32 * kTriWarps),
           triinv_smem_bytes(w), st_, Rt, ldrt, w, Ri, ldi, gate);
    kend();
  }

  // Symmetric eigendecomposition (cuSOLVER syevd, ascending) of a row-major
  // D x D block after (M + M')/2; w and V (column-major) in arena buffers.
  void eig(const double* M, int ldm, int D, double** w_out, double** v_out, const std::string& tag) {
    if (klog_) snprintf(ktag_, sizeof(ktag_), "syevd D=%d", D);
    kbegin(kEig, 9.0 * D * D * D);
    struct End {
      Session* s;
      ~End() { s->kend(); }
    } end{this};
    double* V = arena_.get<double>("eigV" + tag, static_cast<i64>(D) * D);
    double* w = arena_.get<double>("eigW" + tag, D);
    launch(symmetrize_kernel, dim3(blocks(static_cast<i64>(D) * D)), dim3(256), 0, st_, M, ldm, D, V, flags_ptr());
    int lwork = 0;
    if (cusolverDnDsyevd_bufferSize(solver_, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, V, D, w, &lwork) !=
        CUSOLVER_STATUS_SUCCESS)
      throw CudaError("cusolverDnDsyevd_bufferSize failed");
    double* work = arena_.get<double>("eig_work", lwork);
    if (cusolverDnDsyevd(solver_, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, V, D, w, work, lwork,
                         info_ptr()) != CUSOLVER_STATUS_SUCCESS)
      throw CudaError("cusolverDnDsyevd failed");
    *w_out = w;
    *v_out = V;
  }

  // On-device eigensolver (one CTA) for order <= kEigMaxN: all eigenvalues in
  // spectral order (w_sorted) and the leading `want` eigenvectors (F, row-major).
  bool eig_fast(const double* M, int ldm, int D, int order, int want, double* w_sorted, double* F, int ldf,
                double ortol = 1e-3, cudaStream_t s = nullptr, int* flagsp = nullptr) {
    // cuSOLVER syevd on request (ST_FLAG_CUSOLVER_EIG) or above the one-CTA
    // tridiagonalization's shared-memory limit
    if (cfg.flags & ST_FLAG_CUSOLVER_EIG) return false;
    if (D > kEigMaxN || want > kEigMaxWant) return false;
    const int wv = std::max(want, 1);
    double* dbuf = arena_.get<double>("eig_dbuf", static_cast<i64>(eig_scratch_doubles(D, wv)), /*side_use*/ true);
    int* ibuf = arena_.get<int>("eig_ibuf", static_cast<i64>(eig_scratch_ints(D, wv)), /*side_use*/ true);
    if (klog_) snprintf(ktag_, sizeof(ktag_), "device syev D=%d want=%d", D, want);
    cudaStream_t es = s ? s : st_;
    kbegin(kEig, 4.0 * D * D * D / 3.0, es);
    if (!s) STG_CUDA(cudaMemsetAsync(info_ptr(), 0, sizeof(int), st_));
    int part = 0;
    syev_launch(
        [&](auto kernel, dim3 g, dim3 bl, size_t sm, auto... args) {
          if (klog_) {  // timeline of the solver's kernels (double-counted in kstats: STG_KLOG only)
            snprintf(ktag_, sizeof(ktag_), "  eig D=%d part %d grid %u", D, part++, g.x);
            kbegin(kEig, 0.0, es);
          }
          launch(kernel, g, bl, sm, es, args...);
          if (klog_) kend(es);
        },
                M, ldm, D, /*sym_input: exactly mirrored Grams / RR matrix*/ 1, order, wv, ortol, w_sorted, F, ldf,
                dbuf, ibuf, flagsp ? flagsp : flags_ptr());
    kend(es);
    return true;
  }

  void read_scalars() {
    STG_CUDA(cudaMemcpyAsync(&hs_->flags, flags_ptr(), sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(&hs_->info, info_ptr(), sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
  }

  // ---------------------------------------------------------------- Laplacian setup
  void init_laplacian() {
    d_alpha_ = arena_.get<double>("alpha", 4);
    const bool normalized = cfg.op == ST_NORMALIZED_LAPLACIAN;
    const DevCsr& a = A();
    double* deg = arena_.get<double>("deg", n + 1);
    double* scale = arena_.get<double>("scale", n + 1);
    launch(degrees_kernel, dim3(blocks(n)), dim3(256), 0, st_, static_cast<const int*>(a.rp),
           static_cast<const double*>(a.val), n, deg);
    launch(max_reduce_kernel, dim3(1), dim3(1024), 0, st_, static_cast<const double*>(deg), n, d_alpha_ + 2);
    STG_CUDA(cudaMemsetAsync(d_alpha_, 0, sizeof(double), st_));  // shift_for(a0, kind, 0.0)
    launch(shift_kernel, dim3(1), dim3(1), 0, st_, normalized ? 1 : 0, static_cast<const double*>(d_alpha_ + 2),
           static_cast<const double*>(d_alpha_), d_alpha_);
    launch(scale_kernel, dim3(blocks(n)), dim3(256), 0, st_, static_cast<const double*>(deg), n, scale);
    T_[0] = build_t("T0", a, n, normalized, deg, scale, d_alpha_);
    tcur_ = 0;
    STG_CUDA(cudaMemcpyAsync(&hs_->alpha, d_alpha_, sizeof(double), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    alpha = hs_->alpha;
    T_[0].nnz = t_nnz_host_;
  }

  i64 t_nnz_host_ = 0;
  DevCsr build_t(const std::string& name, const DevCsr& a, i64 nr, bool normalized, const double* deg,
                 const double* scale, const double* alpha_ptr) {
    int* cnt = arena_.get<int>("t_cnt", nr + 1);
    launch(lap_count_kernel, dim3(blocks(nr + 1)), dim3(256), 0, st_, static_cast<const int*>(a.rp),
           static_cast<const int*>(a.col), static_cast<const double*>(a.val), nr, normalized ? 1 : 0, deg, scale,
           alpha_ptr, cnt);
    DevCsr t;
    t.n = nr;
    t.rp = arena_.get<int>(name + ".rp", nr + 1);
    scan_int(cnt, t.rp, nr + 1);
    int nnz_t = 0;
    STG_CUDA(cudaMemcpyAsync(&nnz_t, t.rp + nr, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    t.nnz = nnz_t;
    t_nnz_host_ = nnz_t;
    t.col = arena_.get<int>(name + ".col", nnz_t);
    t.val = arena_.get<double>(name + ".val", nnz_t);
    launch(lap_write_kernel, dim3(blocks(nr)), dim3(256), 0, st_, static_cast<const int*>(a.rp),
           static_cast<const int*>(a.col), static_cast<const double*>(a.val), nr, normalized ? 1 : 0, deg, scale,
           alpha_ptr, static_cast<const int*>(t.rp), t.col, t.val);
    return t;
  }

  void scan_int(const int* in, int* out, i64 count) {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int>(count), st_);
    void* t = arena_.get<char>("cub_tmp", static_cast<i64>(tmp));
    cub::DeviceScan::ExclusiveSum(t, tmp, in, out, static_cast<int>(count), st_);
  }

  // A_next = pad(A) + Delta (graph.cpp:102-115) into slot `slot`: per-entry
  // classification and checks, row pointers, then the entry copy (on the
  // merge side stream when `merge_aside`). Rows are those of `a` (n_old) plus
  // appended rows up to n_total; keys are (row << kb | col), sorted.
  DevCsr merge_launch(const DevCsr& a, i64 n_old, i64 n_total, const u64* ekey_s, const double* eval_s, i64 n2,
                      const int* drow, const int* dcol, const int* drp, const int* mark, int kb, int slot,
                      bool merge_aside, u64* err_apply, size_t* merge_pend) {
    int* lb = arena_.get<int>("m_lb", n2);
    int* mflag = arena_.get<int>("m_flag", n2);
    double* newv = arena_.get<double>("m_newv", n2);
    int* contrib = arena_.get<int>("m_contrib", n2 + 1);
    int* prefix = arena_.get<int>("m_prefix", n2 + 1);
    int* ncnt = arena_.get<int>("m_ncnt", n_total + 1);
    const std::string aname = "A" + std::to_string(slot);
    DevCsr an;
    an.n = n_total;
    an.rp = arena_.get<int>(aname + ".rp", n_total + 1);
    an.col = arena_.get<int>(aname + ".col", a.nnz + n2);
    an.val = arena_.get<double>(aname + ".val", a.nnz + n2);
    launch(row_len_kernel, dim3(blocks(n_total + 1)), dim3(256), 0, st_, static_cast<const int*>(a.rp), n_old, n_total,
           ncnt);
    STG_CUDA(cudaMemsetAsync(contrib, 0, sizeof(int) * (n2 + 1), st_));
    if (n2 > 0)
      launch(merge_classify_kernel, dim3(blocks(n2)), dim3(256), 0, st_, static_cast<const u64*>(ekey_s),
             static_cast<const double*>(eval_s), n2, static_cast<const int*>(a.rp), static_cast<const int*>(a.col),
             static_cast<const double*>(a.val), n_old, lb, mflag, newv, contrib, ncnt, err_apply, kb);
    scan_int(ncnt, an.rp, n_total + 1);
    scan_int(contrib, prefix, n2 + 1);
    // row pointers, counts and the apply checks above stay on st_ (the
    // validation read below needs them); the entry copy may run aside
    cudaStream_t ms = st_;
    if (merge_aside) {
      STG_CUDA(cudaEventRecord(ev_mg_fork_, st_));
      STG_CUDA(cudaStreamWaitEvent(st_mg_, ev_mg_fork_, 0));
      ms = st_mg_;
    }
    kbegin(kMerge, 0.0, ms);
    *merge_pend = pend_.size() - (ktiming() ? 1 : 0);
    if (a.nnz > 0) {
      const i64 nwarp = cdiv(n_old + a.nnz, kRunDiag);
      int* cmap = arena_.get<int>("m_chunkmap", nwarp);
      launch(chunk_rows_kernel, dim3(blocks(n_old)), dim3(256), 0, ms, static_cast<const int*>(a.rp),
             static_cast<int>(n_old), cmap);
      launch(merge_runs_kernel, dim3(blocks(nwarp, 8)), dim3(256), 0, ms,
             static_cast<const int*>(a.rp), static_cast<const int*>(a.col), static_cast<const double*>(a.val),
             static_cast<int>(n_old), static_cast<int>(a.nnz), static_cast<const int*>(cmap),
             static_cast<const int*>(mark), stamp_, static_cast<const int*>(drp),
             static_cast<const int*>(dcol), static_cast<const int*>(lb), static_cast<const int*>(mflag),
             static_cast<const double*>(newv), static_cast<const int*>(prefix), static_cast<const int*>(an.rp),
             an.col, an.val, merge_mode_);
    }
    if (n2 > 0)
      launch(merge_insert_kernel, dim3(blocks(n2)), dim3(256), 0, ms, n2, static_cast<const int*>(drow),
             static_cast<const int*>(dcol), static_cast<const u64*>(ekey_s), static_cast<const int*>(lb),
             static_cast<const int*>(mflag), static_cast<const double*>(newv), static_cast<const int*>(prefix),
             static_cast<const int*>(drp), static_cast<const int*>(an.rp), an.col, an.val);
    kend(ms);
    if (merge_aside) STG_CUDA(cudaEventRecord(ev_mg_, st_mg_));
    return an;
  }

  // ---------------------------------------------------------------- ingestion
  // Validation, Delta, A_next (and T_next, Delta_T), P. Nothing committed.
  Pert ingest(const st_update& u, bool keep_delta, bool device_ptrs = false, bool sort_path = false) {
    if (u.n_new < 0) throw InvalidArgument("assemble_update: negative node count");
    if (u.n_added < 0 || u.n_removed < 0 || u.n_new_edges < 0) throw InvalidArgument("st_step: negative list length");
    const i64 n_old = n, S = u.n_new, n_total = n_old + S;
    if (n_total >= (1LL << 31)) throw InvalidArgument("st_step: node count exceeds int32 CSR indexing");
    const i64 E = u.n_added + u.n_removed + u.n_new_edges;
    STG_CUDA(cudaStreamWaitEvent(st_, ev_mg_, 0));  // a merge left running by a failed step
    if (sh_ && !keep_delta) throw InvalidArgument("st_probe: not available on sharded sessions");
    ensure_node_capacity(n_total, sh_ ? rows_at(comm_.rank, n_total) : n_total);
    ++stamp_;
    if (stamp_ == 0x7fffffff) stamp_ = 1;
    ++plan_epoch_;  // the Delta CSRs are rebuilt below
    Pert pt;
    pt.n_old = n_old;
    pt.S = S;
    pt.n_total = n_total;
    pt.stamp = stamp_;
    STG_CUDA(cudaMemsetAsync(d_scal_, 0xff, sizeof(u64) * 2, st_));  // err_edit, err_apply = MAX
    STG_CUDA(cudaMemsetAsync(d_scal_ + 2, 0, sizeof(u64) * 3, st_));  // nvalid, flags, info
    if (klog_) snprintf(ktag_, sizeof(ktag_), "ingest: upload, validation, Delta");
    kbegin(kIngestOther, 0.0);
    EditsDev ed;
    if (device_ptrs) {
      ed.ai = reinterpret_cast<const i64*>(u.added_i);
      ed.aj = reinterpret_cast<const i64*>(u.added_j);
      ed.aw = u.added_w;
      ed.ri = reinterpret_cast<const i64*>(u.removed_i);
      ed.rj = reinterpret_cast<const i64*>(u.removed_j);
      ed.ni = reinterpret_cast<const i64*>(u.new_i);
      ed.nj = reinterpret_cast<const i64*>(u.new_j);
      ed.nw = u.new_w;
    } else {
      // upload the edit lists: straight from the caller's arrays when they are
      // page-locked (one DMA per list), else through one pinned staging buffer
      const size_t bytes = sizeof(i64) * (2 * E) + sizeof(double) * (u.n_added + u.n_new_edges);
      char* dev = arena_.get<char>("edits", static_cast<i64>(std::max<size_t>(bytes, 8)));
      const void* srcs[8] = {u.added_i, u.added_j, u.removed_i, u.removed_j, u.new_i, u.new_j, u.added_w, u.new_w};
      const i64 lens[8] = {u.n_added, u.n_added, u.n_removed, u.n_removed, u.n_new_edges, u.n_new_edges, u.n_added,
                           u.n_new_edges};
      bool pinned = true;
      for (int q = 0; q < 8 && pinned; ++q) {
        if (lens[q] == 0) continue;
        cudaPointerAttributes at{};
        pinned = cudaPointerGetAttributes(&at, srcs[q]) == cudaSuccess && at.type == cudaMemoryTypeHost;
      }
      (void)cudaGetLastError();  // a failed attribute query of pageable memory is not an error
      char* host = pinned ? nullptr : static_cast<char*>(pin_.get(std::max<size_t>(bytes, 8)));
      size_t off = 0;
      auto put = [&](const void* src, size_t b) -> size_t {
        const size_t o = off;
        if (b && pinned) STG_CUDA(cudaMemcpyAsync(dev + off, src, b, cudaMemcpyHostToDevice, st_));
        if (b && !pinned) std::memcpy(host + off, src, b);
        off += b;
        return o;
      };
      const size_t o_ai = put(u.added_i, sizeof(i64) * u.n_added), o_aj = put(u.added_j, sizeof(i64) * u.n_added);
      const size_t o_ri = put(u.removed_i, sizeof(i64) * u.n_removed);
      const size_t o_rj = put(u.removed_j, sizeof(i64) * u.n_removed);
      const size_t o_ni = put(u.new_i, sizeof(i64) * u.n_new_edges), o_nj = put(u.new_j, sizeof(i64) * u.n_new_edges);
      const size_t o_aw = put(u.added_w, sizeof(double) * u.n_added);
      const size_t o_nw = put(u.new_w, sizeof(double) * u.n_new_edges);
      if (off && !pinned) STG_CUDA(cudaMemcpyAsync(dev, host, off, cudaMemcpyHostToDevice, st_));
      ed.ai = reinterpret_cast<const i64*>(dev + o_ai);
      ed.aj = reinterpret_cast<const i64*>(dev + o_aj);
      ed.aw = reinterpret_cast<const double*>(dev + o_aw);
      ed.ri = reinterpret_cast<const i64*>(dev + o_ri);
      ed.rj = reinterpret_cast<const i64*>(dev + o_rj);
      ed.ni = reinterpret_cast<const i64*>(dev + o_ni);
      ed.nj = reinterpret_cast<const i64*>(dev + o_nj);
      ed.nw = reinterpret_cast<const double*>(dev + o_nw);
    }
    ed.n_add = u.n_added;
    ed.n_rem = u.n_removed;
    ed.n_newe = u.n_new_edges;
    ed.n_old = n_old;
    ed.S = S;
    // narrowest key packing that keeps every index below the all-ones sentinel:
    // the radix sorts then run over 2*kb bits instead of 64
    ed.kb = 1;
    while ((1LL << ed.kb) <= n_total) ++ed.kb;
    const int key_bits = 2 * ed.kb;
    u64* err_edit = d_scal_;
    unsigned long long* nvalid = reinterpret_cast<unsigned long long*>(d_scal_ + 2);
    const i64 n2 = 2 * E;
    // ---- validation + Delta entries -> Delta (global CSR over n_total rows)
    int* code = arena_.get<int>("code", E);
    int* post = arena_.get<int>("post", E);
    int* dup = arena_.get<int>("dup", E);
    u64* ekey_s = arena_.get<u64>(keep_delta ? "ekey_s" : "ekey_s_probe", n2);
    double* eval_s = arena_.get<double>(keep_delta ? "eval_s" : "eval_s_probe", n2);
    const std::string sfx = keep_delta ? "" : "_probe";
    int* drow = arena_.get<int>("drow" + sfx, n2);
    int* dcol = arena_.get<int>("dcol" + sfx, n2);
    int* dcnt = arena_.get<int>("dcnt", n_total + 1);
    int* drp = arena_.get<int>("drp" + sfx, n_total + 1);
    STG_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(int) * (n_total + 1), st_));
    if (!sort_path) {
      // buckets by row, then each entry's rank in its row (edit_bucket_kernel)
      int2* slot = arena_.get<int2>("e_slot", E);
      int* brow = arena_.get<int>("b_row", n2);
      int* bcol = arena_.get<int>("b_col", n2);
      int* bedit = arena_.get<int>("b_edit", n2);
      if (E > 0)
        launch(edit_bucket_kernel, dim3(blocks(E)), dim3(256), 0, st_, ed, code, post, dcnt, slot, mark_delta_,
               stamp_);
      scan_int(dcnt, drp, n_total + 1);
      if (E > 0) {
        launch(edit_scatter_kernel, dim3(blocks(E)), dim3(256), 0, st_, ed, static_cast<const int*>(code),
               static_cast<const int2*>(slot), static_cast<const int*>(drp), brow, bcol, bedit);
        STG_CUDA(cudaMemsetAsync(dup, 0, sizeof(int) * E, st_));
        STG_CUDA(cudaMemsetAsync(ekey_s, 0xff, sizeof(u64) * n2, st_));
        launch(delta_rank_kernel, dim3(blocks(n2)), dim3(256), 0, st_, ed, n2, static_cast<const int*>(drp),
               static_cast<const int*>(brow), static_cast<const int*>(bcol), static_cast<const int*>(bedit), ekey_s,
               eval_s, drow, dcol, dup, err_edit);
        launch(edit_status_kernel, dim3(blocks(E)), dim3(256), 0, st_, E, static_cast<const int*>(code),
               static_cast<const int*>(dup), static_cast<const int*>(post), err_edit, nvalid);
      }
    } else {
      // two radix sorts: pair keys for the duplicate test, then the entries
      u64* pkey = arena_.get<u64>("pkey", E);
      i64* pval = arena_.get<i64>("pval", E);
      u64* pkey_s = arena_.get<u64>("pkey_s", E);
      i64* pval_s = arena_.get<i64>("pval_s", E);
      u64* ekey = arena_.get<u64>("ekey", n2);
      double* eval = arena_.get<double>("eval", n2);
      if (E > 0) {
        launch(edit_check_kernel, dim3(blocks(E)), dim3(256), 0, st_, ed, pkey, pval, code, post);
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, pkey, pkey_s, pval, pval_s, static_cast<int>(E), 0, key_bits,
                                        st_);
        void* t = arena_.get<char>("cub_tmp", static_cast<i64>(tmp));
        cub::DeviceRadixSort::SortPairs(t, tmp, pkey, pkey_s, pval, pval_s, static_cast<int>(E), 0, key_bits, st_);
        launch(dup_mark_kernel, dim3(blocks(E)), dim3(256), 0, st_, static_cast<const u64*>(pkey_s),
               static_cast<const i64*>(pval_s), E, dup);
        launch(edit_emit_kernel, dim3(blocks(E)), dim3(256), 0, st_, ed, static_cast<const int*>(code),
               static_cast<const int*>(dup), static_cast<const int*>(post), err_edit, ekey, eval, nvalid);
        tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, ekey, ekey_s, eval, eval_s, static_cast<int>(n2), 0, key_bits,
                                        st_);
        t = arena_.get<char>("cub_tmp", static_cast<i64>(tmp));
        cub::DeviceRadixSort::SortPairs(t, tmp, ekey, ekey_s, eval, eval_s, static_cast<int>(n2), 0, key_bits, st_);
        launch(delta_rows_kernel, dim3(blocks(n2)), dim3(256), 0, st_, static_cast<const u64*>(ekey_s), n2, drow,
               dcol, dcnt, mark_delta_, stamp_, ed.kb);
      }
      scan_int(dcnt, drp, n_total + 1);
    }
    kend();
    TailIn in{keep_delta, ed.kb, ekey_s, eval_s, n2, drow, dcol, drp, sort_path,
              [&]() { return ingest(u, keep_delta, device_ptrs, true); }};
    return ingest_tail(pt, in);
  }

  // ---- GraphUpdate blocks (graph.hpp:23-37) or a Perturbation's Delta
  // (trackers.hpp:78-86) as the front of ingestion: `blocks` are CSRs with
  // their offsets in the n_total square (K at (0,0), G at (0,n_old) mirrored,
  // C at (n_old,n_old); or Delta alone at (0,0)).
  struct HostBlock {
    st_csr_block b;
    i64 row_off, col_off;
    int mirror;
  };
  Pert ingest_blocks(i64 S, const std::vector<HostBlock>& hb, bool keep_delta, bool device_ptrs) {
    const i64 n_old = n, n_total = n_old + S;
    if (S < 0) throw InvalidArgument("make_empty_update: negative size");
    if (n_total >= (1LL << 31)) throw InvalidArgument("st_step: node count exceeds int32 CSR indexing");
    STG_CUDA(cudaStreamWaitEvent(st_, ev_mg_, 0));
    if (sh_ && !keep_delta) throw InvalidArgument("st_probe: not available on sharded sessions");
    ensure_node_capacity(n_total, sh_ ? rows_at(comm_.rank, n_total) : n_total);
    ++stamp_;
    if (stamp_ == 0x7fffffff) stamp_ = 1;
    ++plan_epoch_;
    Pert pt;
    pt.n_old = n_old;
    pt.S = S;
    pt.n_total = n_total;
    pt.stamp = stamp_;
    STG_CUDA(cudaMemsetAsync(d_scal_, 0xff, sizeof(u64) * 2, st_));
    STG_CUDA(cudaMemsetAsync(d_scal_ + 2, 0, sizeof(u64) * 3, st_));
    kbegin(kIngestOther, 0.0);
    int kb = 1;
    while ((1LL << kb) <= n_total) ++kb;
    u64* err_edit = d_scal_;
    // upload (host blocks) and shape checks
    std::vector<BlockIn> bins;
    i64 n2 = 0;
    for (size_t q = 0; q < hb.size(); ++q) {
      const st_csr_block& b = hb[q].b;
      if (b.nnz < 0 || b.rows < 0) throw InvalidArgument("st_step_blocks: malformed block CSR");
      BlockIn bi{};
      bi.rows = b.rows;
      bi.cols = b.cols;
      bi.nnz = b.nnz;
      bi.row_off = hb[q].row_off;
      bi.col_off = hb[q].col_off;
      bi.mirror = hb[q].mirror;
      bi.out0 = n2;
      if (device_ptrs) {
        bi.rp = b.rowptr;
        bi.col = b.colidx;
        bi.val = b.values;
      } else {
        const std::string nm = "blk" + std::to_string(q);
        int* rp = arena_.get<int>(nm + ".rp", b.rows + 1);
        int* col = arena_.get<int>(nm + ".col", b.nnz);
        double* val = arena_.get<double>(nm + ".val", b.nnz);
        if (!b.rowptr || (b.nnz && (!b.colidx || !b.values))) throw InvalidArgument("st_step_blocks: null block array");
        STG_CUDA(cudaMemcpyAsync(rp, b.rowptr, sizeof(int) * (b.rows + 1), cudaMemcpyHostToDevice, st_));
        if (b.nnz) {
          STG_CUDA(cudaMemcpyAsync(col, b.colidx, sizeof(int) * b.nnz, cudaMemcpyHostToDevice, st_));
          STG_CUDA(cudaMemcpyAsync(val, b.values, sizeof(double) * b.nnz, cudaMemcpyHostToDevice, st_));
        }
        bi.rp = rp;
        bi.col = col;
        bi.val = val;
      }
      launch(block_check_kernel, dim3(blocks(std::max(b.rows, b.nnz) + 1)), dim3(256), 0, st_, bi, err_edit);
      n2 += bi.mirror ? 2 * b.nnz : b.nnz;
      bins.push_back(bi);
    }
    STG_CUDA(cudaMemcpyAsync(&hs_->err_edit, err_edit, sizeof(u64), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    if (hs_->err_edit != kSentinel) throw InvalidArgument(edit_message(static_cast<int>(hs_->err_edit & 0xff)));
    // entries -> stable sort -> run sums (duplicates in insertion order) -> prune zeros
    const std::string sfx = keep_delta ? "" : "_probe";
    u64* ekey = arena_.get<u64>("ekey", n2);
    double* eval = arena_.get<double>("eval", n2);
    u64* skey = arena_.get<u64>("b_skey", n2);
    double* sval = arena_.get<double>("b_sval", n2);
    for (const BlockIn& bi : bins)
      if (bi.nnz) launch(block_emit_kernel, dim3(blocks(bi.nnz)), dim3(256), 0, st_, bi, kb, ekey, eval);
    if (n2 > 0) {
      size_t tmp = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp, ekey, skey, eval, sval, static_cast<int>(n2), 0, 2 * kb, st_);
      void* t = arena_.get<char>("cub_tmp", static_cast<i64>(tmp));
      cub::DeviceRadixSort::SortPairs(t, tmp, ekey, skey, eval, sval, static_cast<int>(n2), 0, 2 * kb, st_);
    }
    int* keep = arena_.get<int>("b_keep", n2 + 1);
    int* kpos = arena_.get<int>("b_kpos", n2 + 1);
    double* rsum = arena_.get<double>("b_rsum", n2);
    u64* ekey_s = arena_.get<u64>(keep_delta ? "ekey_s" : "ekey_s_probe", n2);
    double* eval_s = arena_.get<double>(keep_delta ? "eval_s" : "eval_s_probe", n2);
    int* drow = arena_.get<int>("drow" + sfx, n2);
    int* dcol = arena_.get<int>("dcol" + sfx, n2);
    int* dcnt = arena_.get<int>("dcnt", n_total + 1);
    int* drp = arena_.get<int>("drp" + sfx, n_total + 1);
    STG_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(int) * (n_total + 1), st_));
    STG_CUDA(cudaMemsetAsync(ekey_s, 0xff, sizeof(u64) * std::max<i64>(n2, 1), st_));
    launch(run_sum_kernel, dim3(blocks(n2 + 1)), dim3(256), 0, st_, static_cast<const u64*>(skey),
           static_cast<const double*>(sval), n2, keep, rsum);
    scan_int(keep, kpos, n2 + 1);
    if (n2 > 0) {
      launch(run_compact_kernel, dim3(blocks(n2)), dim3(256), 0, st_, static_cast<const u64*>(skey),
             static_cast<const double*>(rsum), static_cast<const int*>(keep), static_cast<const int*>(kpos), n2,
             ekey_s, eval_s);
      launch(sym_check_kernel, dim3(blocks(n2)), dim3(256), 0, st_, static_cast<const u64*>(ekey_s),
             static_cast<const double*>(eval_s), static_cast<const int*>(kpos + n2), kb, err_edit);
      launch(delta_rows_kernel, dim3(blocks(n2)), dim3(256), 0, st_, static_cast<const u64*>(ekey_s), n2, drow, dcol,
             dcnt, mark_delta_, stamp_, kb);
    }
    launch(count_to_u64_kernel, dim3(1), dim3(1), 0, st_, static_cast<const int*>(kpos + n2),
           reinterpret_cast<unsigned long long*>(d_scal_ + 2));
    scan_int(dcnt, drp, n_total + 1);
    kend();
    TailIn in{keep_delta, kb, ekey_s, eval_s, n2, drow, dcol, drp, true, nullptr};
    return ingest_tail(pt, in);
  }

  // What the validation / Delta-assembly front hands to the shared tail: the
  // sorted Delta entries (keys (row << kb | col), sentinels last), their CSR
  // over n_total rows, and how to redo the front on the sorting path.
  struct TailIn {
    bool keep_delta;
    int kb;
    u64* ekey_s;
    double* eval_s;
    i64 n2;
    int* drow;
    int* dcol;
    int* drp;
    bool sort_path;
    std::function<Pert()> redo;
  };

  // apply_update (graph.cpp:102-115) or ShiftedLaplacianSession::advance
  // (laplacian_track.cpp:48-64), then P and the compressed CSR.
  Pert ingest_tail(Pert pt, const TailIn& in) {
    const bool keep_delta = in.keep_delta;
    const i64 n_old = pt.n_old, S = pt.S, n_total = pt.n_total, n2 = in.n2;
    u64* ekey_s = in.ekey_s;
    double* eval_s = in.eval_s;
    int* drow = in.drow;
    int* dcol = in.dcol;
    int* drp = in.drp;
    const std::string sfx = keep_delta ? "" : "_probe";
    u64* err_edit = d_scal_;
    u64* err_apply = d_scal_ + 1;
    if (sh_) return ingest_shard_tail(pt, in);
    // ---- apply_update merge (A_next in the spare slot)
    const DevCsr& a = A();
    const int slot = keep_delta ? 1 - acur_ : 2;  // probes never touch the live buffers
    size_t merge_pend = 0;
    DevCsr an = merge_launch(a, n_old, n_total, ekey_s, eval_s, n2, drow, dcol, drp, mark_delta_, in.kb, slot,
                             keep_delta && !is_laplacian(), err_apply, &merge_pend);
    const bool kt_p = !is_laplacian();  // (the Laplacian path syncs inside)
    if (kt_p && klog_) snprintf(ktag_, sizeof(ktag_), "ingest: P, sizes");
    if (kt_p) kbegin(kIngestOther, 0.0);
    // ---- validation outcome and sizes: read back here for the Laplacian
    // operators (their assembly needs nnz); the adjacency path folds this read
    // into the P-size sync below (nothing is committed before either)
    STG_CUDA(cudaMemcpyAsync(&hs_->err_edit, err_edit, sizeof(u64) * 3, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(&hs_->nnz_new, an.rp + n_total, sizeof(int), cudaMemcpyDeviceToHost, st_));
    auto check_validation = [&]() {
      if (hs_->err_edit != kSentinel) throw InvalidArgument(edit_message(static_cast<int>(hs_->err_edit & 0xff)));
      if (hs_->err_apply != kSentinel) {
        if (hs_->err_apply & 1ULL) throw InvalidArgument("apply_update: update drives an edge weight negative");
        throw InvalidArgument("apply_update: invalid deletion (no such edge)");
      }
      an.nnz = hs_->nnz_new;
      A_[slot] = an;
      anext_ = slot;
      pt.nnz = static_cast<i64>(hs_->nvalid);
      if (ktiming())  // read old CSR + write new CSR (SURVEY 8(d) ingestion bytes, edits excluded)
        pend_[merge_pend].work = 12.0 * a.nnz + 4.0 * (n_old + 1) + 12.0 * an.nnz + 4.0 * (n_total + 1);
    };
    // a Delta row too long for the counting path: redo on the sorting path
    auto redo = [&]() { return !in.sort_path && hs_->err_edit == 0; };
    if (is_laplacian()) {
      STG_CUDA(cudaStreamSynchronize(st_));
      if (redo()) return in.redo();
      check_validation();
    }
    // ---- the tracked operator's perturbation
    const int* grp = drp;
    const int* gcol = dcol;
    const double* gval = eval_s;
    if (is_laplacian()) {
      const bool normalized = cfg.op == ST_NORMALIZED_LAPLACIAN;
      double* deg = arena_.get<double>("deg", n_total + 1);
      double* scale = arena_.get<double>("scale", n_total + 1);
      launch(degrees_kernel, dim3(blocks(n_total)), dim3(256), 0, st_, static_cast<const int*>(an.rp),
             static_cast<const double*>(an.val), n_total, deg);
      launch(max_reduce_kernel, dim3(1), dim3(1024), 0, st_, static_cast<const double*>(deg), n_total, d_alpha_ + 2);
      launch(shift_kernel, dim3(1), dim3(1), 0, st_, normalized ? 1 : 0, static_cast<const double*>(d_alpha_ + 2),
             static_cast<const double*>(d_alpha_), d_alpha_ + 1);
      launch(scale_kernel, dim3(blocks(n_total)), dim3(256), 0, st_, static_cast<const double*>(deg), n_total, scale);
      const int ts = keep_delta ? 1 - tcur_ : 2;
      DevCsr tn = build_t("T" + std::to_string(ts), an, n_total, normalized, deg, scale, d_alpha_ + 1);
      tnext_ = ts;
      T_[ts] = tn;
      const DevCsr& to = T();
      int* dtcnt = arena_.get<int>("dt_cnt", n_total + 1);
      int* dtrp = arena_.get<int>("dt_rp" + sfx, n_total + 1);
      launch(lap_diff_kernel, dim3(blocks(n_total + 1)), dim3(256), 0, st_, static_cast<const int*>(to.rp),
             static_cast<const int*>(to.col), static_cast<const double*>(to.val), n_old,
             static_cast<const int*>(tn.rp), static_cast<const int*>(tn.col), static_cast<const double*>(tn.val),
             n_total, static_cast<const int*>(nullptr), dtcnt, static_cast<int*>(nullptr),
             static_cast<double*>(nullptr), 0);
      scan_int(dtcnt, dtrp, n_total + 1);
      int nnz_dt = 0;
      STG_CUDA(cudaMemcpyAsync(&hs_->nnz_dt, dtrp + n_total, sizeof(int), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaMemcpyAsync(&hs_->alpha, d_alpha_ + 1, sizeof(double), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      nnz_dt = hs_->nnz_dt;
      alpha_next_ = hs_->alpha;
      int* dtcol = arena_.get<int>("dt_col" + sfx, nnz_dt);
      double* dtval = arena_.get<double>("dt_val" + sfx, nnz_dt);
      launch(lap_diff_kernel, dim3(blocks(n_total + 1)), dim3(256), 0, st_, static_cast<const int*>(to.rp),
             static_cast<const int*>(to.col), static_cast<const double*>(to.val), n_old,
             static_cast<const int*>(tn.rp), static_cast<const int*>(tn.col), static_cast<const double*>(tn.val),
             n_total, static_cast<const int*>(dtrp), dtcnt, dtcol, dtval, 1);
      launch(mark_nonempty_kernel, dim3(blocks(n_total)), dim3(256), 0, st_, static_cast<const int*>(dtrp), n_total,
             mark_p_, stamp_);
      grp = dtrp;
      gcol = dtcol;
      gval = dtval;
      pt.nnz = nnz_dt;
    } else {
      // adjacency: P-marks are the Delta rows
      if (n_total > 0)
        STG_CUDA(cudaMemcpyAsync(mark_p_, mark_delta_, sizeof(int) * n_total, cudaMemcpyDeviceToDevice, st_));
    }
    if (S > 0)
      launch(mark_range_kernel, dim3(blocks(S)), dim3(256), 0, st_, mark_p_, n_old, n_total, stamp_);
    pt.grp = grp;
    pt.gcol = gcol;
    pt.val = gval;
    // ---- P and the compressed CSR
    int* flag = arena_.get<int>("p_flag", n_total + 1);
    int* pos = arena_.get<int>("p_pos", n_total + 1);
    int* P = arena_.get<int>("P", n_total + 1);
    launch(flag_kernel, dim3(blocks(n_total + 1)), dim3(256), 0, st_, static_cast<const int*>(mark_p_), stamp_, n_total,
           flag);
    scan_int(flag, pos, n_total + 1);
    launch(scatter_p_kernel, dim3(blocks(n_total)), dim3(256), 0, st_, static_cast<const int*>(flag),
           static_cast<const int*>(pos), n_total, P, posmap_);
    k_ready_ = false;
    if (k_early_ && keep_delta && !is_laplacian()) early_k(n_old);
    STG_CUDA(cudaMemcpyAsync(&hs_->p, pos + n_total, sizeof(int), cudaMemcpyDeviceToHost, st_));
    if (kt_p) kend();
    STG_CUDA(cudaStreamSynchronize(st_));
    if (!is_laplacian()) {
      if (redo()) return in.redo();
      check_validation();
    }
    pt.p = hs_->p;
    pt.p_old = pt.p - S;
    pt.P = P;
    pt.posmap = posmap_;
    pt.mark = mark_p_;
    if ((cfg.flags & ST_FLAG_FORCE_DENSE) || 2 * pt.p > n_total) {
      make_dense(pt);
    } else {
      int* lrp = arena_.get<int>("lrp", pt.p + 1);
      int* lcol = arena_.get<int>("lcol", pt.nnz);
      launch(compress_rowptr_kernel, dim3(blocks(pt.p + 1)), dim3(256), 0, st_, grp, static_cast<const int*>(P), pt.p,
             lrp, static_cast<int>(pt.nnz));
      if (pt.nnz > 0)
        launch(compress_cols_kernel, dim3(blocks(pt.nnz)), dim3(256), 0, st_, gcol, pt.nnz,
               static_cast<const int*>(posmap_), lcol);
      pt.lrp = lrp;
      pt.lcol = lcol;
      unsharded_fields(pt);
      // the segment plans of this step's Delta products, built here: the main stream would otherwise wait
      // idle for the K Gram and its Cholesky (early_k, side stream) and build them before the first SpMM
      if (eager_plans_ && k_ready_ && keep_delta && cfg.kind >= ST_IASC && cfg.kind <= ST_GREST_RSVD) {
        SpmmArgs pa{};
        pa.rowptr = lrp;
        pa.rows = pt.p;
        spmm_plan(pa, pt.nnz);
        if (cfg.kind == ST_GREST_RSVD && S > cfg.rsvd_l) {  // Delta_2' M over the appended rows (rsvd_trailing)
          pa.row_off = pt.p_old;
          pa.rows = pt.S_loc;
          spmm_plan(pa, pt.nnz);
        }
      }
    }
    return pt;
  }

  // Sharded ingestion after the replicated validation and Delta assembly:
  // the owned rows of Delta (local row ids) are merged into the owned rows of
  // A, the owned rows of P are found, P is exchanged (halo positions), and the
  // owned rows of Delta are compressed. Errors are decided identically on
  // every rank (edit errors are replicated; apply errors are gathered and the
  // one at the smallest global (row, col) is reported, as on one GPU).
  Pert ingest_shard_tail(Pert pt, const TailIn& in) {
    const u64* ekey_s = in.ekey_s;
    const double* eval_s = in.eval_s;
    const int* dcol = in.dcol;
    const int* drp = in.drp;
    const i64 n2 = in.n2;
    const i64 n_old = pt.n_old, n_total = pt.n_total;
    const int R = comm_.size, rank = comm_.rank, kb = in.kb;
    const i64 xo = nloc_, xt = rows_at(rank, n_total);
    u64* err_edit = d_scal_;
    u64* err_apply = d_scal_ + 1;
    // ---- owned rows of Delta, renumbered to local rows
    int* ef = arena_.get<int>("sh_eflag", n2 + 1);
    int* ep = arena_.get<int>("sh_epos", n2 + 1);
    u64* lkey = arena_.get<u64>("sh_lkey", n2);
    double* lval = arena_.get<double>("sh_lval", n2);
    int* lrow = arena_.get<int>("sh_lrow", n2);
    int* lcolg = arena_.get<int>("sh_lcolg", n2);
    int* lcnt = arena_.get<int>("sh_lcnt", xt + 1);
    int* ldrp = arena_.get<int>("sh_ldrp", xt + 1);
    STG_CUDA(cudaMemsetAsync(lcnt, 0, sizeof(int) * (xt + 1), st_));
    STG_CUDA(cudaMemsetAsync(lkey, 0xff, sizeof(u64) * std::max<i64>(n2, 1), st_));
    launch(own_entry_flag_kernel, dim3(blocks(n2 + 1)), dim3(256), 0, st_, ekey_s, n2, kb, map_, ef);
    scan_int(ef, ep, n2 + 1);
    if (n2 > 0)
      launch(own_entry_scatter_kernel, dim3(blocks(n2)), dim3(256), 0, st_, ekey_s, eval_s, n2, kb, map_,
             static_cast<const int*>(ef), static_cast<const int*>(ep), lkey, lval, lrow, lcolg, lcnt, mark_dl_,
             stamp_);
    scan_int(lcnt, ldrp, xt + 1);
    const DevCsr& a = A();
    const int slot = 1 - acur_;
    size_t merge_pend = 0;
    DevCsr an = merge_launch(a, xo, xt, lkey, lval, n2, lrow, lcolg, ldrp, mark_dl_, kb, slot, true, err_apply,
                             &merge_pend);
    // ---- P marks (global): Delta rows + appended nodes
    if (n_total > 0)
      STG_CUDA(cudaMemcpyAsync(mark_p_, mark_delta_, sizeof(int) * n_total, cudaMemcpyDeviceToDevice, st_));
    if (pt.S > 0)
      launch(mark_range_kernel, dim3(blocks(pt.S)), dim3(256), 0, st_, mark_p_, n_old, n_total, stamp_);
    int* pf = arena_.get<int>("sh_pflag", xt + 1);
    int* pp = arena_.get<int>("sh_ppos", xt + 1);
    launch(own_p_flag_kernel, dim3(blocks(xt + 1)), dim3(256), 0, st_, static_cast<const int*>(mark_p_), stamp_,
           map_, xt, 0, pf);
    scan_int(pf, pp, xt + 1);
    // ---- validation outcome (one sync)
    STG_CUDA(cudaMemcpyAsync(&hs_->err_edit, err_edit, sizeof(u64) * 3, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(&hs_->nnz_new, an.rp + xt, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(&hs_->p, pp + xt, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    if (!in.sort_path && hs_->err_edit == 0) return in.redo();  // replicated decision
    if (hs_->err_edit != kSentinel) throw InvalidArgument(edit_message(static_cast<int>(hs_->err_edit & 0xff)));
    u64 mine = hs_->err_apply;
    if (mine != kSentinel) {  // local row -> global row in the error key
      const u64 g = static_cast<u64>(sm_global(host_map(), static_cast<i64>(mine >> 32)));
      mine = (g << 32) | (mine & 0xffffffffULL);
    }
    const std::vector<u64> info = allgather_u64({mine, static_cast<u64>(hs_->p)});
    u64 first = kSentinel;
    i64 p_all = 0;
    std::vector<i64> cnt(static_cast<size_t>(R));
    for (int r = 0; r < R; ++r) {
      first = std::min(first, info[2 * r]);
      cnt[r] = static_cast<i64>(info[2 * r + 1]);
      p_all += cnt[r];
    }
    if (first != kSentinel) {
      if (first & 1ULL) throw InvalidArgument("apply_update: update drives an edge weight negative");
      throw InvalidArgument("apply_update: invalid deletion (no such edge)");
    }
    an.nnz = hs_->nnz_new;
    A_[slot] = an;
    anext_ = slot;
    pt.nnz = static_cast<i64>(hs_->nvalid);
    if (ktiming())
      pend_[merge_pend].work = 12.0 * a.nnz + 4.0 * (xo + 1) + 12.0 * an.nnz + 4.0 * (xt + 1);
    pt.grp = drp;
    pt.gcol = dcol;
    pt.gval = eval_s;
    pt.x_old = xo;
    pt.x_total = xt;
    pt.S_loc = xt - xo;
    if (pt.empty()) return pt;
    // ---- owned rows of P (all owned rows in dense mode, a global decision)
    pt.dense = (cfg.flags & ST_FLAG_FORCE_DENSE) || 2 * p_all > n_total;
    if (pt.dense) {
      launch(own_p_flag_kernel, dim3(blocks(xt + 1)), dim3(256), 0, st_, static_cast<const int*>(mark_p_), stamp_,
             map_, xt, 1, pf);
      scan_int(pf, pp, xt + 1);
      for (int r = 0; r < R; ++r) cnt[r] = rows_at(r, n_total);
    }
    const i64 p = cnt[rank];
    i64 pmax = 1;
    for (int r = 0; r < R; ++r) pmax = std::max(pmax, cnt[r]);
    int* ploc = arena_.get<int>("sh_Ploc", xt + 1);
    int* pglob = arena_.get<int>("sh_Pglob", xt + 1);
    int* psend = arena_.get<int>("sh_psend", pmax);
    int* pall = arena_.get<int>("sh_pall", pmax * R);
    launch(own_p_scatter_kernel, dim3(blocks(xt)), dim3(256), 0, st_, static_cast<const int*>(pf),
           static_cast<const int*>(pp), map_, xt, ploc, pglob);
    STG_CUDA(cudaMemsetAsync(psend, 0xff, sizeof(int) * pmax, st_));
    if (p > 0) STG_CUDA(cudaMemcpyAsync(psend, pglob, sizeof(int) * p, cudaMemcpyDeviceToDevice, st_));
    STG_CUDA(cudaMemsetAsync(pall, 0xff, sizeof(int) * pmax * R, st_));
    allgather(psend, pall, static_cast<i64>(sizeof(int)) * pmax);
    launch(halo_posmap_kernel, dim3(blocks(pmax * R)), dim3(256), 0, st_, static_cast<const int*>(pall), pmax * R,
           posmap_);
    // ---- compressed CSR of the owned rows (columns = halo positions)
    int* rl = arena_.get<int>("sh_rowlen", p + 1);
    int* lrp = arena_.get<int>("lrp", p + 1);
    int* lcol = arena_.get<int>("lcol", pt.nnz);
    int* scol = arena_.get<int>("sh_scol", pt.nnz);
    double* val = arena_.get<double>("sh_val", pt.nnz);
    launch(own_rowlen_kernel, dim3(blocks(p + 1)), dim3(256), 0, st_, drp, static_cast<const int*>(pglob), p, rl);
    scan_int(rl, lrp, p + 1);
    if (p > 0)
      launch(own_compress_kernel, dim3(blocks(p, 8)), dim3(256), 0, st_, drp, dcol, eval_s,
             static_cast<const int*>(pglob), p, static_cast<const int*>(lrp), static_cast<const int*>(posmap_), lcol,
             scol, val);
    // ---- boundary-row halo plan: the remote rows of P the owned Delta rows
    // reference, requested from their owners; columns renumbered to
    // [own rows | received rows]
    {
      const i64 total = pmax * R;
      int* need = arena_.get<int>("sh_need", total + 1);
      int* npos = arena_.get<int>("sh_npos", total + 1);
      int* slot = arena_.get<int>("sh_slot", total);
      STG_CUDA(cudaMemsetAsync(need, 0, sizeof(int) * (total + 1), st_));
      if (pt.nnz > 0)
        launch(halo_need_kernel, dim3(blocks(pt.nnz)), dim3(256), 0, st_, static_cast<const int*>(lcol), pt.nnz, pmax,
               rank, need);
      scan_int(need, npos, total + 1);
      // requests per owner: positions [r pmax, (r + 1) pmax) of the scan
      std::vector<int> cut(static_cast<size_t>(R) + 1);
      for (int r = 0; r <= R; ++r)
        STG_CUDA(cudaMemcpyAsync(&cut[r], npos + std::min<i64>(static_cast<i64>(r) * pmax, total), sizeof(int),
                                 cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      const i64 nreq = cut[R];
      int* req = arena_.get<int>("sh_req", std::max<i64>(nreq, 1));
      launch(halo_req_kernel, dim3(blocks(total)), dim3(256), 0, st_, static_cast<const int*>(need),
             static_cast<const int*>(npos), total, pmax, p, req, slot);
      if (pt.nnz > 0)
        launch(halo_remap_kernel, dim3(blocks(pt.nnz)), dim3(256), 0, st_, lcol, pt.nnz, pmax, rank,
               static_cast<const int*>(slot));
      // everyone's request counts (R x R, host) -> what this rank sends to whom
      std::vector<u64> mine(static_cast<size_t>(R));
      for (int r = 0; r < R; ++r) mine[r] = static_cast<u64>(cut[r + 1] - cut[r]);
      const std::vector<u64> all = allgather_u64(mine);  // all[src * R + owner]
      pt.recv_rows.assign(static_cast<size_t>(R), 0);
      pt.send_rows.assign(static_cast<size_t>(R), 0);
      for (int r = 0; r < R; ++r) {
        pt.recv_rows[r] = static_cast<i64>(mine[r]);
        pt.send_rows[r] = static_cast<i64>(all[static_cast<size_t>(r) * R + rank]);
      }
      pt.recv_rows[rank] = pt.send_rows[rank] = 0;
      pt.nrecv = nreq;
      pt.nsend = 0;
      for (int r = 0; r < R; ++r) pt.nsend += pt.send_rows[r];
      int* hsend = arena_.get<int>("sh_hsend", std::max<i64>(pt.nsend, 1));
      // the requests travel to the owners (request lists out, send lists in)
      std::vector<i64> sb(static_cast<size_t>(R)), rb(static_cast<size_t>(R));
      for (int r = 0; r < R; ++r) {
        sb[r] = pt.recv_rows[r] * static_cast<i64>(sizeof(int));
        rb[r] = pt.send_rows[r] * static_cast<i64>(sizeof(int));
      }
      alltoallv(req, sb, hsend, rb);
      pt.hsend = hsend;
    }
    pt.p = p;
    pt.p_old = p - pt.S_loc;
    pt.pmax = pmax;
    pt.G = p + (rank == 0 ? k : 0);
    pt.P = pglob;
    pt.Ploc = ploc;
    pt.Pglob = pglob;
    pt.posmap = posmap_;
    pt.mark = mark_p_;
    pt.lrp = lrp;
    pt.lcol = lcol;
    pt.val = val;
    pt.scol = scol;
    pt.scol_lo = static_cast<int>(n_old);
    return pt;
  }

  void make_dense(Pert& pt) {
    pt.dense = true;
    pt.p = pt.n_total;
    pt.p_old = pt.n_old;
    pt.lrp = pt.grp;
    pt.lcol = pt.gcol;
    unsharded_fields(pt);
  }

  // one GPU holds every row: P doubles as the X row list and the global ids
  void unsharded_fields(Pert& pt) {
    pt.G = pt.p + k;
    pt.S_loc = pt.S;
    pt.x_old = pt.n_old;
    pt.x_total = pt.n_total;
    pt.Ploc = pt.P;
    pt.Pglob = pt.P;
    pt.gval = pt.val;
    pt.scol = pt.lcol;
    pt.scol_lo = static_cast<int>(pt.p_old);
  }

  void commit_graph(const Pert& pt) {
    STG_CUDA(cudaStreamWaitEvent(st_, ev_mg_, 0));
    if (anext_ >= 0) {
      acur_ = anext_;
      anext_ = -1;
    }
    if (is_laplacian() && tnext_ >= 0) {
      tcur_ = tnext_;
      tnext_ = -1;
      alpha = alpha_next_;
      STG_CUDA(cudaMemcpyAsync(d_alpha_, d_alpha_ + 1, sizeof(double), cudaMemcpyDeviceToDevice, st_));
    }
    last_delta_.rp = const_cast<int*>(pt.grp);
    last_delta_.col = const_cast<int*>(pt.gcol);
    last_delta_.val = const_cast<double*>(pt.gval);
    last_delta_nnz_ = pt.nnz;
    last_delta_n_ = pt.n_total;
    n = pt.n_total;
    nloc_ = pt.x_total;
    // rows appended to X are zero until the rotation writes them (padded_vectors)
  }

  // ---------------------------------------------------------------- orthonormalize
  // ortho.hpp:13-39 on the stacked coordinates: BCGS2 + CholQR2 when every
  // column is clearly independent, the exact column-by-column MGS2 replica when
  // a pivot is suspect. W (N x w) is consumed; Q is written to `out`.
  // With `Cpre` the block was already projected once outside (W = W0 - A Cpre,
  // Cpre = A'W0, a x w with leading dimension ldcpre): pass 1 starts at its
  // Gram, and the exact replica, if needed, rebuilds W0.
  // defer_ri (no `against` only): the second pass's R^-1 is not applied; `out`
  // receives Q1 (the first pass's output) and defer_ri the w x w upper-
  // triangular factor, out_final = Q1 R^-1, for a caller whose every use of the
  // block is linear from the right (last_ortho_deferred_ tells whether it was).
  int orthonormalize(Blk W, int w, const Blk* against, int a, i64 N, i64 G, Blk out, const double* Cpre = nullptr,
                     int ldcpre = 0, double* defer_ri = nullptr, int ld_defer = 0) {
    last_ortho_deferred_ = false;
    if (w == 0) return 0;
    if (w > kCholMaxW) {  // wider than the one-CTA Cholesky: the exact column-by-column replica
      last_ortho_exact_ = true;
      if (against && a > 0 && Cpre) {
        const int ldw0 = ld_for(w);
        double* W0 = arena_.get<double>("on_W0", N * ldw0);
        nn(against->p, against->ld, N, a, Cpre, ldcpre, w, W0, ldw0, 1.0, 1.0, W.p, W.ld);
        return mgs2_exact(Blk{W0, ldw0}, w, against, a, N, G, out);
      }
      return mgs2_exact(W, w, against, a, N, G, out);
    }
    const int ldw = ld_for(w);
    double* W1 = arena_.get<double>("on_W1", N * ldw);
    double* C = arena_.get<double>("on_C", static_cast<i64>(std::max(a, 1)) * ldw);
    double* Gm = arena_.get<double>("on_G", static_cast<i64>(w) * ldw);
    double* R = arena_.get<double>("on_R", static_cast<i64>(w) * ldw);
    double* Ri = arena_.get<double>("on_Ri", static_cast<i64>(w) * ldw);
    double* o2 = arena_.get<double>("on_o2", w);
    // pass 1: W1 = W - A (A'W); with no `against` the Gram reads W directly
    const double* P1 = W.p;
    int ldp1 = W.ld;
    const double* Cuse = C;
    int ldc1 = ldw;
    if (against && a > 0 && Cpre) {
      Cuse = Cpre;
      ldc1 = ldcpre;
    } else if (against && a > 0) {
      pgram(against->p, against->ld, W.p, W.ld, G, a, w, false, C, ldw);
      nn(against->p, against->ld, N, a, C, ldw, w, W1, ldw, -1.0, 1.0, W.p, W.ld);
      P1 = W1;
      ldp1 = ldw;
    }
    pgram(P1, ldp1, P1, ldp1, G, w, w, true, Gm, ldw);
    launch(orig2_kernel, dim3(blocks(w, 128)), dim3(128), 0, st_, static_cast<const double*>(Gm), ldw, Cuse, ldc1,
           (against ? a : 0), w, o2);
    STG_CUDA(cudaMemsetAsync(flags_ptr(), 0, sizeof(int), st_));
    chol(Gm, ldw, w, R, ldw, Ri, ldw, o2, kSuspectTau2, false);
    if (spec_) {
      // speculate "no suspect pivot" (the common case): the decision is
      // checked once at the end of the step, which is redone on the exact
      // path if any pivot was suspect (no host round trip here)
      launch(or_sticky_kernel, dim3(1), dim3(1), 0, st_, static_cast<const int*>(flags_ptr()), kSuspect | kBreakdown,
             sticky_ptr());
      last_ortho_exact_ = false;
    } else {
      read_scalars();
      last_ortho_exact_ = (hs_->flags & (kSuspect | kBreakdown)) != 0;
    }
    if (last_ortho_exact_) {
      if (against && a > 0 && Cpre) {  // the replica starts from the unprojected block
        double* W0 = arena_.get<double>("on_W0", N * ldw);
        nn(against->p, against->ld, N, a, Cpre, ldcpre, w, W0, ldw, 1.0, 1.0, W.p, W.ld);
        return mgs2_exact(Blk{W0, ldw}, w, against, a, N, G, out);
      }
      return mgs2_exact(W, w, against, a, N, G, out);
    }
    // pass 2 input Q1 = P1 R^-1: into `out` when it is re-projected into W1,
    // else straight into W1
    const bool proj = against && a > 0;
    const bool defer = defer_ri && !proj;
    double* Q1 = proj || defer ? out.p : W1;
    const int ldq1 = proj || defer ? out.ld : ldw;
    nn(P1, ldp1, N, w, Ri, ldw, w, Q1, ldq1, 1.0, 0.0, nullptr, 0, true);
    if (defer) {  // pass 2's Gram and factor only: out = Q1, defer_ri = R^-1
      pgram(out.p, out.ld, out.p, out.ld, G, w, w, true, Gm, ldw);
      chol_inverse_near_identity(Gm, ldw, w, R, ldw, Ri, ldw);
      STG_CUDA(cudaMemcpy2DAsync(defer_ri, sizeof(double) * ld_defer, Ri, sizeof(double) * ldw, sizeof(double) * w, w,
                                 cudaMemcpyDeviceToDevice, st_));
      last_ortho_deferred_ = true;
      return w;
    }
    // pass 2
    if (proj) {
      pgram(against->p, against->ld, out.p, out.ld, G, a, w, false, C, ldw);
      nn(against->p, against->ld, N, a, C, ldw, w, W1, ldw, -1.0, 1.0, out.p, out.ld);
    }
    pgram(W1, ldw, W1, ldw, G, w, w, true, Gm, ldw);
    chol_inverse_near_identity(Gm, ldw, w, R, ldw, Ri, ldw);
    nn(W1, ldw, N, w, Ri, ldw, w, out.p, out.ld, 1.0, 0.0, nullptr, 0, true);
    return w;
  }

  bool last_ortho_exact_ = false;  // the last orthonormalize took the column-by-column replica
  bool last_ortho_deferred_ = false;  // ... and returned Q1 with the second pass's R^-1 unapplied
  // sketch basis projected against [X-bar, first candidate block] while the
  // sketch's eigensolve runs (rsvd_trailing / build_basis)
  const double* pre_pm_ = nullptr;
  const double* pre_c1_ = nullptr;
  int pre_a_ = 0;
  double* pre_cr_ = nullptr;
  int pre_ldcr_ = 0;
  // speculative steps: the RSVD block's Grams precomputed beside the sketch
  // eigensolve (PM'PM and [X-bar, Q1]'PM), and U_keep (the block is PM U_keep)
  const double* pre_gpm_ = nullptr;
  const double* pre_c1p_ = nullptr;
  int pre_ldm_ = 0, pre_qm_ = 0;
  const double* pre_t0_ = nullptr;
  int pre_ldt0_ = 0;
  const bool fold_rsvd_ = !getenv_flag("STG_NO_RSVD_FOLD");  // development A/B

  // orthonormalize(PM U_keep, against [X-bar, Q1]) of the speculative path
  // from Grams computed while the sketch's eigensolve ran: pass 1's Gram is
  // U'(PM'PM)U (no n-row Gram), its R^-1 folds into one product Q1 = PM (U R^-1)
  // (R = PM U is never formed), pass 2's coefficients are ([X-bar,Q1]'PM)(U R^-1).
  // Same algebra and decisions as orthonormalize's Cpre path (suspect pivots
  // raise the sticky flag and the step is redone on the exact path).
  int orthonormalize_rsvd_folded(int w, const Blk* against, int a, i64 N, i64 G, Blk out) {
    const int qm = pre_qm_, ldm = pre_ldm_;
    const int ldw = ld_for(w);
    double* H = arena_.get<double>("rf_H", static_cast<i64>(qm) * ldw);
    double* T1 = arena_.get<double>("rf_T1", static_cast<i64>(qm) * ldw);
    double* W1 = arena_.get<double>("on_W1", N * ldw);
    double* C = arena_.get<double>("on_C", static_cast<i64>(std::max(a, 1)) * ldw);
    double* Gm = arena_.get<double>("on_G", static_cast<i64>(w) * ldw);
    double* R = arena_.get<double>("on_R", static_cast<i64>(w) * ldw);
    double* Ri = arena_.get<double>("on_Ri", static_cast<i64>(w) * ldw);
    double* o2 = arena_.get<double>("on_o2", w);
    // pass 1: G1 = U'(PM'PM)U, the original norms from G1 and the first projection's coefficients
    nn(pre_gpm_, ldm, qm, qm, pre_t0_, pre_ldt0_, w, H, ldw, 1.0, 0.0, nullptr, 0);
    gram(pre_t0_, pre_ldt0_, H, ldw, qm, w, w, false, Gm, ldw);
    launch(orig2_kernel, dim3(blocks(w, 128)), dim3(128), 0, st_, static_cast<const double*>(Gm), ldw,
           static_cast<const double*>(pre_cr_), pre_ldcr_, a, w, o2);
    STG_CUDA(cudaMemsetAsync(flags_ptr(), 0, sizeof(int), st_));
    chol(Gm, ldw, w, R, ldw, Ri, ldw, o2, kSuspectTau2, false);
    launch(or_sticky_kernel, dim3(1), dim3(1), 0, st_, static_cast<const int*>(flags_ptr()), kSuspect | kBreakdown,
           sticky_ptr());
    last_ortho_exact_ = false;
    // Q1 = PM (U R^-1)
    nn(pre_t0_, pre_ldt0_, qm, w, Ri, ldw, w, T1, ldw, 1.0, 0.0, nullptr, 0, true);
    nn(pre_pm_, ldm, N, qm, T1, ldw, w, out.p, out.ld, 1.0, 0.0, nullptr, 0);
    // pass 2: W1 = Q1 - A (A'Q1), A'Q1 = (A'PM)(U R^-1)
    nn(pre_c1p_, ldm, a, qm, T1, ldw, w, C, ldw, 1.0, 0.0, nullptr, 0);
    nn(against->p, against->ld, N, a, C, ldw, w, W1, ldw, -1.0, 1.0, out.p, out.ld);
    pgram(W1, ldw, W1, ldw, G, w, w, true, Gm, ldw);
    chol_inverse_near_identity(Gm, ldw, w, R, ldw, Ri, ldw);
    nn(W1, ldw, N, w, Ri, ldw, w, out.p, out.ld, 1.0, 0.0, nullptr, 0, true);
    return w;
  }
  static constexpr double kSuspectTau2 = 1e-10;  // residual / original norm below 1e-5
  static constexpr double kRrOrtol = 1e-9;       // eigenvector cluster threshold for the RR solve

  // One CholQR pass over the k columns of a small D x k block (already
  // orthonormal to ~1e-7): F R^-1, columns in order. Returns the new block.
  double* orthonormalize_small(const double* F, int ldf, int D, int kk) {
    double* G = arena_.get<double>("os_G", static_cast<i64>(kk) * ldf);
    double* R = arena_.get<double>("os_R", static_cast<i64>(kk) * ldf);
    double* Ri = arena_.get<double>("os_Ri", static_cast<i64>(kk) * ldf);
    double* F2 = arena_.get<double>("os_F", static_cast<i64>(D) * ldf);
    gram(F, ldf, F, ldf, D, kk, kk, true, G, ldf);
    chol_inverse_near_identity(G, ldf, kk, R, ldf, Ri, ldf);
    nn(F, ldf, D, kk, Ri, ldf, kk, F2, ldf, 1.0, 0.0, nullptr, 0, /*tri*/ true);
    return F2;
  }

  // Exact replica of ortho.hpp:26-37, one column at a time, without host
  // round trips: the per-column drop decisions stay on the device (dropped
  // columns are zero slots until one compaction at the end; one read of the
  // kept count).
  int mgs2_exact(Blk W, int w, const Blk* against, int a, i64 N, i64 G, Blk out) {
    const int ldv = 8;
    double* v = arena_.get<double>("mgs_v", N * ldv);
    double* t = arena_.get<double>("mgs_t", std::max(a, w) * ldv + 8);
    double* nrm2 = arena_.get<double>("mgs_n2", 16);
    int* keep = arena_.get<int>("mgs_keep", w + 8);
    for (int c = 0; c < w; ++c) {
      launch(copy2d_kernel, dim3(blocks(N)), dim3(256), 0, st_, static_cast<const double*>(W.p + c), W.ld, v, ldv, N, 1);
      pgram(v, ldv, v, ldv, G, 1, 1, true, nrm2, 1);  // the original squared norm
      for (int pass = 0; pass < 2; ++pass) {
        if (against && a > 0) {
          pgram(against->p, against->ld, v, ldv, G, a, 1, false, t, ldv);
          nn(against->p, against->ld, N, a, t, ldv, 1, v, ldv, -1.0, 1.0, v, ldv);
        }
        if (c > 0) {  // earlier columns: kept ones normalized, dropped ones zero
          pgram(out.p, out.ld, v, ldv, G, c, 1, false, t, ldv);
          nn(out.p, out.ld, N, c, t, ldv, 1, v, ldv, -1.0, 1.0, v, ldv);
        }
      }
      pgram(v, ldv, v, ldv, G, 1, 1, true, nrm2 + 8, 1);
      launch(mgs_scale_kernel, dim3(blocks(N)), dim3(256), 0, st_, static_cast<const double*>(v), ldv, N,
             static_cast<const double*>(nrm2), static_cast<const double*>(nrm2 + 8), out.p + c, out.ld, keep + c);
    }
    int* dr = reinterpret_cast<int*>(nrm2 + 4);
    launch(mgs_compact_kernel, dim3(blocks(N)), dim3(256), 0, st_, out.p, out.ld, N, static_cast<const int*>(keep), w,
           dr);
    int r = 0;
    STG_CUDA(cudaMemcpyAsync(&hs_->mgs_r, dr, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    r = hs_->mgs_r;
    return r;
  }

  // ---------------------------------------------------------------- basis
  // build_projection_basis (trackers.cpp:226-280) in stacked coordinates.
  // Z columns [0, k) hold X-bar; returns Z with D columns.
  Basis build_basis(const Pert& pt, int basis_kind, u64 seed) {
    const i64 p = pt.p, N = p + 2 * k, G = pt.G;
    const i64 S = pt.S;
    const int kk = static_cast<int>(k);
    // widths
    int trail_max = 0;
    bool rsvd = false;
    int q = 0;
    if (basis_kind == 0) {
      trail_max = static_cast<int>(S);
    } else if (basis_kind >= 2) {
      const bool bypass = basis_kind == 2 || S <= cfg.rsvd_l;
      if (bypass) {
        trail_max = static_cast<int>(S);
      } else {
        rsvd = true;
        q = static_cast<int>(std::min<i64>(S, cfg.rsvd_l + cfg.rsvd_p));
        trail_max = static_cast<int>(std::min<i64>(cfg.rsvd_l, q));
      }
    }
    const int wmax = (basis_kind == 0 ? 0 : kk) + trail_max;
    const int ldz = ld_for(kk + wmax);
    double* Z = arena_.get<double>("Z", N * ldz);
    Blk z{Z, ldz};
    // ---- RNG for the sketch (normally already launched at the start of the step)
    double* omega = nullptr;
    int ldo = 0;
    if (rsvd) prepare_omega(seed, S, q, &omega, &ldo);
    // ---- X-bar in stacked coordinates: [X_P; R_c; I]
    build_xbar(pt, z);
    if (basis_kind == 0) {
      // iasc: [[X, 0], [0, I_S]] (trackers.cpp:233-238)
      STG_CUDA(cudaMemset2DAsync(Z + kk, sizeof(double) * ldz, 0, sizeof(double) * S, N, st_));
      if (sh_ && pt.S_loc > 0)
        launch(unit_cols_own_kernel, dim3(blocks(pt.S_loc)), dim3(256), 0, st_, Z + kk, ldz, pt.Pglob, pt.p_old,
               pt.S_loc, pt.n_old);
      else if (!sh_ && S > 0)
        launch(unit_cols_kernel, dim3(blocks(S)), dim3(256), 0, st_, Z + kk, ldz, pt.p_old, S);
      return Basis{z, static_cast<int>(kk + S)};
    }
    // ---- candidates [(I - XX') Delta X | trailing]
    const int ldc = ld_for(wmax);
    double* cand = arena_.get<double>("cand", N * ldc);
    if (basis_kind >= 2 && !rsvd && S > 0) {  // the dense d2 columns are scattered: zero the whole block
      STG_CUDA(cudaMemsetAsync(cand, 0, sizeof(double) * N * ldc, st_));
    } else {  // the SpMM writes every row of P (zero rows included): only the coordinate rows need zeros
      STG_CUDA(cudaMemsetAsync(cand + p * ldc, 0, sizeof(double) * (N - p) * ldc, st_));
    }
    double* ck = arena_.get<double>("ck", static_cast<i64>(kk) * ld_for(std::max(q, std::max(trail_max, kk))));
    // dx = Delta X (rows of P; the coordinate rows stay 0)
    SpmmArgs sa{};
    sa.rows = p;
    sa.row_off = 0;
    sa.rowptr = pt.lrp;
    sa.col = pt.lcol;
    sa.val = pt.val;
    sa.X = halo(pt, Z, ldz, kk, &sa.ldx);
    sa.m = kk;
    sa.Y = cand;
    sa.ldy = ldc;
    do_spmm(sa, pt.nnz, p);
    pgram(Z, ldz, cand, ldc, G, kk, kk, false, ck, ldc);
    nn(Z, ldz, N, kk, ck, ldc, kk, cand, ldc, -1.0, 1.0, cand, ldc);
    int w = kk;
    if (basis_kind >= 2) {
      if (!rsvd) {
        // d2 dense: column j = Delta[:, n_old + j]; by symmetry row p_old + j of the local CSR
        if (S > 0) {
          if (sh_)
            launch(d2_rows_kernel, dim3(blocks(p, 8)), dim3(256), 0, st_, pt.lrp, pt.scol, pt.val, p, pt.n_old,
                   cand + kk, ldc);
          else
            launch(d2_dense_kernel, dim3(blocks(S, 8)), dim3(256), 0, st_, pt.lrp, pt.lcol, pt.val, pt.p_old, S,
                   cand + kk, ldc);
          const int lck = ld_for(S);
          double* c2 = arena_.get<double>("c2", static_cast<i64>(kk) * lck);
          pgram(Z, ldz, cand + kk, ldc, G, kk, static_cast<int>(S), false, c2, lck);
          nn(Z, ldz, N, kk, c2, lck, static_cast<int>(S), cand + kk, ldc, -1.0, 1.0, cand + kk, ldc);
          w += static_cast<int>(S);
        }
      } else {
        // The candidates are orthonormalized in two blocks, column order kept
        // (ortho.hpp:26-37 walks them in order): (I - XX') Delta X first, while
        // the sketch's eigensolve runs beside it, then the RSVD columns against
        // [X-bar, that block].
        int q1 = 0;
        pre_pm_ = pre_c1_ = nullptr;
        pre_cr_ = nullptr;
        pre_gpm_ = pre_c1p_ = pre_t0_ = nullptr;
        const int wt = rsvd_trailing(pt, z, q, omega, ldo, Blk{cand + kk, ldc},
                                     [&](const double* Msk, int ldm, int qm) {
          q1 = orthonormalize(Blk{cand, ldc}, kk, &z, kk, N, G, Blk{Z + kk, ldz});
          if (Msk && qm > 0) {  // project the sketch basis against [X-bar, Q1] before U is known
            const int a = kk + q1;
            double* c1 = arena_.get<double>("pm_C1", static_cast<i64>(a) * ldm);
            double* pm = arena_.get<double>("pm_PM", N * ldm);
            pgram(Z, ldz, Msk, ldm, G, a, qm, false, c1, ldm);
            nn(Z, ldz, N, a, c1, ldm, qm, pm, ldm, -1.0, 1.0, Msk, ldm);
            pre_pm_ = pm;
            pre_c1_ = c1;
            pre_a_ = a;
          }
          // the Rayleigh-Ritz products of [X-bar, Q1] do not depend on the sketch
          rr_prefix(pt, z, kk + q1, kk + q1 + static_cast<int>(std::min<i64>(cfg.rsvd_l, q)));
          if (spec_ && fold_rsvd_ && pre_pm_) {  // the RSVD block's Grams, still beside the eigensolve
            const int a = pre_a_;
            double* gpm = arena_.get<double>("pm_GPM", static_cast<i64>(qm) * ldm);
            double* c1p = arena_.get<double>("pm_C1P", static_cast<i64>(a) * ldm);
            pgram(pre_pm_, ldm, pre_pm_, ldm, G, qm, qm, true, gpm, ldm);
            pgram(Z, ldz, pre_pm_, ldm, G, a, qm, false, c1p, ldm);
            pre_gpm_ = gpm;
            pre_c1p_ = c1p;
            pre_ldm_ = ldm;
            pre_qm_ = qm;
          }
        });
        int q2 = 0;
        if (wt > 0) {
          const Blk against{Z, ldz};
          if (pre_t0_)
            q2 = orthonormalize_rsvd_folded(wt, &against, kk + q1, N, G, Blk{Z + kk + q1, ldz});
          else
            q2 = orthonormalize(Blk{cand + kk, ldc}, wt, &against, kk + q1, N, G, Blk{Z + kk + q1, ldz}, pre_cr_,
                                pre_ldcr_);
        }
        pre_pm_ = pre_c1_ = nullptr;
        pre_cr_ = nullptr;
        pre_gpm_ = pre_c1p_ = pre_t0_ = nullptr;
        return Basis{z, kk + q1 + q2};
      }
    }
    // ---- extra = orthonormalize(candidates, X-bar) written next to X-bar
    const int wq = orthonormalize(Blk{cand, ldc}, w, &z, kk, N, G, Blk{Z + kk, ldz});
    return Basis{z, kk + wq};
  }

  // rsvd_basis (rsvd.hpp:34-66) with the closures of trackers.cpp:256-267.
  // `during_eig` enqueues independent work on the main stream while the
  // sketch's eigensolve (one or two SMs) runs on st_eig_.
  template <class F>
  int rsvd_trailing(const Pert& pt, Blk z, int q, const double* omega, int ldo, Blk out, F&& during_eig) {
    const i64 p = pt.p, N = p + 2 * k, G = pt.G;
    const int kk = static_cast<int>(k);
    const int ldy = ld_for(q);
    double* Y = arena_.get<double>("Y", N * ldy);
    // the sketch SpMM writes every row of P (zero rows included): zero the coordinate rows only
    STG_CUDA(cudaMemsetAsync(Y + p * ldy, 0, sizeof(double) * (N - p) * ldy, st_));
    STG_CUDA(cudaStreamWaitEvent(st_, ev_rng_, 0));
    // Y0 = d2 * Omega: nonzeros of Delta in the appended-node columns
    SpmmArgs sa{};
    sa.rows = p;
    sa.rowptr = pt.lrp;
    sa.col = pt.scol;
    sa.val = pt.val;
    sa.col_lo = pt.scol_lo;
    sa.X = omega - static_cast<i64>(pt.scol_lo) * ldo;
    sa.ldx = ldo;
    sa.m = q;
    sa.Y = Y;
    sa.ldy = ldy;
    do_spmm(sa, pt.nnz, pt.S, kSpmmSketch);
    double* cy = arena_.get<double>("cy", static_cast<i64>(kk) * ldy);
    pgram(z.p, z.ld, Y, ldy, G, kk, q, false, cy, ldy);
    nn(z.p, z.ld, N, kk, cy, ldy, q, Y, ldy, -1.0, 1.0, Y, ldy);
    // M = orthonormalize(Y). Every later use of M is linear from the right
    // (bt_m = d2' M, the projection M - Z (Z'M), R = M U_keep), so CholQR2's
    // last product Q1 R2^-1 over all N rows is not formed: M holds Q1 and
    // R2^-1 (q x q, upper triangular) is folded into bt_m and U_keep.
    double* M = arena_.get<double>("Msk", N * ldy);
    double* r2i = arena_.get<double>("Msk_R2i", static_cast<i64>(q) * ldy);
    static const bool no_fold = getenv_flag("STG_NO_SKETCH_FOLD");  // development A/B
    const int qm = orthonormalize(Blk{Y, ldy}, q, nullptr, 0, N, G, Blk{M, ldy}, nullptr, 0, no_fold ? nullptr : r2i,
                                  ldy);
    const bool folded = last_ortho_deferred_;
    // U_keep -> R2^-1 U_keep (the factor M = Q1 R2^-1 leaves on the right)
    auto fold_u = [&](const double* Uk, int ldu_, int keep_) -> const double* {
      if (!folded) return Uk;
      double* ud = arena_.get<double>("Ukeep_f", static_cast<i64>(qm) * ldu_);
      nn(r2i, ldy, qm, qm, Uk, ldu_, keep_, ud, ldu_, 1.0, 0.0, nullptr, 0);
      return ud;
    };
    if (qm == 0) {
      during_eig(static_cast<const double*>(nullptr), ldy, 0);
      return 0;
    }
    // bt_m = d2' (M - X (X'M)) (trackers.cpp:262-266). On the CholQR2 path
    // M = (P Y) R^-1 spans a block already projected against X-bar, so
    // X-bar'M is rounding-level (eps kappa(Y), kappa(Y) < 1e5 there: a
    // worse-conditioned Y trips the suspect-pivot test); the projection then
    // changes bt_m by that relative amount only and is skipped. After the
    // column-by-column replica (near rank loss) it is applied as written.
    const double* Msrc = M;
    if (last_ortho_exact_) {
      double* cm = arena_.get<double>("cm", static_cast<i64>(kk) * ldy);
      pgram(z.p, z.ld, M, ldy, G, kk, qm, false, cm, ldy);
      double* Mp = arena_.get<double>("Mp", p * ldy);
      nn(z.p, z.ld, p, kk, cm, ldy, qm, Mp, ldy, -1.0, 1.0, M, ldy);
      Msrc = Mp;
    }
    double* btm = arena_.get<double>("btm", std::max<i64>(pt.S_loc, 1) * ldy);
    double* btm1 = folded ? arena_.get<double>("btm1", std::max<i64>(pt.S_loc, 1) * ldy) : btm;
    SpmmArgs sb{};
    sb.rows = pt.S_loc;
    sb.row_off = pt.p_old;
    sb.rowptr = pt.lrp;
    sb.col = pt.lcol;
    sb.val = pt.val;
    sb.X = halo(pt, Msrc, ldy, qm, &sb.ldx);
    sb.m = qm;
    sb.Y = btm1;
    sb.ldy = ldy;
    do_spmm(sb, pt.nnz, p, kSpmmSketch);
    if (folded)  // bt_m = (d2' Q1) R2^-1 over the S new rows only
      nn(btm1, ldy, pt.S_loc, qm, r2i, ldy, qm, btm, ldy, 1.0, 0.0, nullptr, 0, true);
    // thin U of (M'B) = eigenvectors of bt_m' bt_m, singular values descending
    double* gb = arena_.get<double>("gb", static_cast<i64>(qm) * ldy);
    pgram(btm, ldy, btm, ldy, pt.S_loc, qm, qm, true, gb, ldy);
    const int wantu = static_cast<int>(std::min<i64>(cfg.rsvd_l, qm));
    const int ldu = ld_for(wantu);
    double* U = arena_.get<double>("Ukeep", static_cast<i64>(qm) * ldu);
    double* lamd = arena_.get<double>("sk_lam", qm);
    std::vector<double> lam(static_cast<size_t>(qm));
    // only span(U_keep) matters here (R is re-orthonormalized with the basis),
    // so clusters are re-orthogonalized only when nearly degenerate
    STG_CUDA(cudaEventRecord(ev_gb_, st_));
    STG_CUDA(cudaStreamWaitEvent(st_eig_, ev_gb_, 0));
    if (spec_ && eig_fast(gb, ldy, qm, /*alg_desc*/ 1, wantu, lamd, U, ldu, 1e-10, st_eig_, side_flags_ptr())) {
      // speculate full rank (keep = min(L, qm)); the device checks rsvd.hpp:59-63's
      // cut beside the solve and the step is redone if it disagrees
      launch(sketch_keep_kernel, dim3(1), dim3(32), 0, st_eig_, static_cast<const double*>(lamd), qm,
             static_cast<int>(cfg.rsvd_l), wantu, static_cast<const int*>(nullptr), sticky_ptr());
      STG_CUDA(cudaEventRecord(ev_eig_, st_eig_));
      during_eig(static_cast<const double*>(M), ldy, qm);
      STG_CUDA(cudaStreamWaitEvent(st_, ev_eig_, 0));
      const int keep = wantu;
      if (keep == 0) return 0;
      const double* Uf = fold_u(U, ldu, keep);
      if (pre_pm_) {
        const int ldcp = ld_for(keep);
        pre_cr_ = arena_.get<double>("pm_CR", static_cast<i64>(pre_a_) * ldcp);
        pre_ldcr_ = ldcp;
        nn(pre_c1_, ldy, pre_a_, qm, Uf, ldu, keep, pre_cr_, ldcp, 1.0, 0.0, nullptr, 0);
        if (pre_gpm_) {  // R = PM U_keep is not formed (orthonormalize_rsvd_folded)
          pre_t0_ = Uf;
          pre_ldt0_ = ldu;
        } else {
          nn(pre_pm_, ldy, N, qm, Uf, ldu, keep, out.p, out.ld, 1.0, 0.0, nullptr, 0);
        }
      } else {
        nn(M, ldy, N, qm, Uf, ldu, keep, out.p, out.ld, 1.0, 0.0, nullptr, 0);
      }
      return keep;
    }
    if (eig_fast(gb, ldy, qm, /*alg_desc*/ 1, wantu, lamd, U, ldu, 1e-10, st_eig_, side_flags_ptr())) {
      STG_CUDA(cudaMemcpyAsync(hs_->sk_lam, lamd, sizeof(double) * qm, cudaMemcpyDeviceToHost, st_eig_));
      STG_CUDA(cudaEventRecord(ev_eig_, st_eig_));
      during_eig(static_cast<const double*>(M), ldy, qm);
      STG_CUDA(cudaStreamWaitEvent(st_, ev_eig_, 0));
      STG_CUDA(cudaStreamSynchronize(st_eig_));
      std::copy(hs_->sk_lam, hs_->sk_lam + qm, lam.begin());
      hs_->info = 0;
      std::reverse(lam.begin(), lam.end());  // ascending like the cuSOLVER path
    } else {
      during_eig(static_cast<const double*>(M), ldy, qm);
      double *w = nullptr, *V = nullptr;
      eig(gb, ldy, qm, &w, &V, "sk");
      STG_CUDA(cudaMemcpyAsync(lam.data(), w, sizeof(double) * qm, cudaMemcpyDeviceToHost, st_));
      read_scalars();
      launch(gather_desc_kernel, dim3(blocks(static_cast<i64>(qm) * wantu)), dim3(256), 0, st_,
             static_cast<const double*>(V), qm, wantu, U, ldu);
    }
    if (hs_->info != 0) throw RuntimeError("rsvd_basis: SVD did not converge");
    // rank: sv(r) > 1e-10 sv(0) and > 0 (rsvd.hpp:59-62)
    std::vector<double> sv(static_cast<size_t>(qm));
    for (int i = 0; i < qm; ++i) sv[i] = std::sqrt(std::max(lam[static_cast<size_t>(qm - 1 - i)], 0.0));
    const double cutoff = qm > 0 ? 1e-10 * sv[0] : 0.0;
    int rank = 0;
    while (rank < qm && sv[rank] > cutoff && sv[rank] > 0.0) ++rank;
    const int keep = static_cast<int>(std::min<i64>(cfg.rsvd_l, rank));
    if (getenv("STG_SKETCH_LOG") && keep > 0 && keep < qm) {  // development: the singular gap at the cut
      fprintf(stderr, "sketch: qm %d rank %d keep %d  sv[keep-1] %.17g sv[keep] %.17g rel gap %.3e\n", qm, rank, keep,
              sv[keep - 1], sv[keep], (sv[keep - 1] - sv[keep]) / sv[0]);
    }
    if (keep == 0) return 0;
    // R = M U_keep; when the caller projected M against its basis meanwhile
    // (pre_pm_ = M - B C1), R's first projection is PM U_keep with
    // coefficients C1 U_keep (with the folded factor: U_keep -> R2^-1 U_keep)
    const double* Uf = fold_u(U, ldu, keep);
    if (pre_pm_) {
      nn(pre_pm_, ldy, N, qm, Uf, ldu, keep, out.p, out.ld, 1.0, 0.0, nullptr, 0);
      const int ldcp = ld_for(keep);
      pre_cr_ = arena_.get<double>("pm_CR", static_cast<i64>(pre_a_) * ldcp);
      pre_ldcr_ = ldcp;
      nn(pre_c1_, ldy, pre_a_, qm, Uf, ldu, keep, pre_cr_, ldcp, 1.0, 0.0, nullptr, 0);
    } else {
      nn(M, ldy, N, qm, Uf, ldu, keep, out.p, out.ld, 1.0, 0.0, nullptr, 0);
    }
    return keep;
  }

  // Omega (S x q, rng.hpp:64-69 fill order) generated on the side stream; the
  // consumer waits on ev_rng_. The raw mt19937_64 words depend only on the
  // seed, and the next step's seed is known (trackers.cpp:362), so after each
  // sketch the side stream speculatively generates a prefix of the next
  // step's stream; a step that needs more words resumes it from the saved ring.
  u64 omega_seed_ = 0;
  i64 omega_S_ = -1;
  int omega_q_ = -1;
  u64 pre_seed_ = 0;      // seed of the raw words in mt_raw (rseed)
  i64 pre_blocks_ = -1;   // 156-word blocks already generated for pre_seed_
  i64 raw_cap_ = 0;       // capacity of mt_raw in words
  u64* raw_ = nullptr;
  u64* ring_state_ = nullptr;

  void ensure_raw(i64 words) {
    if (words <= raw_cap_) return;
    STG_CUDA(cudaStreamSynchronize(st_rng_));
    raw_cap_ = round_up(words + words / 2, kMtM);
    raw_ = arena_.get<u64>("mt_raw", raw_cap_, /*side_use*/ true);
    pre_blocks_ = -1;  // contents lost
  }

  void generate_raw(u64 rseed, i64 blocks_needed) {
    if (!ring_state_) ring_state_ = arena_.get<u64>("mt_ring", kMtRing, /*side_use*/ true);
    ensure_raw(blocks_needed * kMtM);
    if (pre_seed_ == rseed && pre_blocks_ >= 0) {
      if (pre_blocks_ >= blocks_needed) return;
      launch(mt19937_64_kernel, dim3(1), dim3(160), 0, st_rng_, rseed, pre_blocks_, blocks_needed, 0, ring_state_, raw_);
    } else {
      launch(mt19937_64_kernel, dim3(1), dim3(160), 0, st_rng_, rseed, static_cast<i64>(0), blocks_needed, 1,
             ring_state_, raw_);
    }
    pre_seed_ = rseed;
    pre_blocks_ = blocks_needed;
  }

  void prepare_omega(u64 seed, i64 S, int q, double** omega, int* ldo_out) {
    const int ldo = ld_for(q);
    double* om = arena_.get<double>("omega", S * ldo, /*side_use*/ true);
    if (!(omega_seed_ == seed && omega_S_ == S && omega_q_ == q)) {
      const i64 npairs = cdiv(S * q, 2);
      const u64 rseed = mix_seed(seed, 0x5bdULL);
      kbegin(kRng, 2.0 * npairs, st_rng_);
      generate_raw(rseed, cdiv(2 * npairs, kMtM));
      launch(box_muller_kernel, dim3(blocks(npairs)), dim3(256), 0, st_rng_, static_cast<const u64*>(raw_), npairs, S,
             q, om, ldo);
      kend(st_rng_);
      STG_CUDA(cudaEventRecord(ev_rng_, st_rng_));
      omega_seed_ = seed;
      omega_S_ = S;
      omega_q_ = q;
      // speculative prefix of the next step's stream (runs behind this step)
      const u64 next = mix_seed(mix_seed(mix_seed(cfg.seed, 0x6b7aULL), steps_taken + 1), 0x5bdULL);
      const i64 guess = cdiv(2 * npairs + 2 * npairs / 8, kMtM);
      pre_seed_ = 0;
      pre_blocks_ = -1;
      ensure_raw(guess * kMtM);
      launch(mt19937_64_kernel, dim3(1), dim3(160), 0, st_rng_, next, static_cast<i64>(0), guess, 1, ring_state_,
             raw_);
      pre_seed_ = next;
      pre_blocks_ = guess;
    }
    *omega = om;
    *ldo_out = ldo;
  }

  // X-bar in stacked coordinates [X_P; R_c; I]. K = X_out' X_out is a plain
  // Gram of X after the rows of P (already copied into Z) are zeroed in place;
  // restore_x() writes them back if the step fails, and the final rotation
  // overwrites them on success.
  struct XRestore {
    bool active = false;
    const int* P = nullptr;
    i64 p_old = 0;
    const double* z = nullptr;
    int ldz = 0;
  } xrestore_;

  void restore_x() {
    wait_rotation();
    if (!xrestore_.active) return;
    launch(restore_rows_kernel, dim3(blocks(xrestore_.p_old, 8)), dim3(256), 0, st_, X_, ldx(), xrestore_.P,
           xrestore_.p_old, xrestore_.z, xrestore_.ldz, static_cast<int>(k));
    xrestore_.active = false;
  }

  // K = sum over the rows of X outside P of x x' (the marks of P masked) and
  // its Cholesky R_c, on st_eig_ (the previous step's rotation of X first);
  // build_xbar waits for ev_k_. In dense mode K is not used.
  void early_k(i64 x_rows) {
    const int kk = static_cast<int>(k);
    const int ldr = ld_for(kk);
    double* kc = arena_.get<double>("Kc", static_cast<i64>(kk) * ldr, /*side_use*/ true);
    double* rc = arena_.get<double>("Rc", static_cast<i64>(kk) * ldr, /*side_use*/ true);
    arena_.get<double>("gram_partial_k", 148 * 3 * 1024, /*side_use*/ true);
    STG_CUDA(cudaEventRecord(ev_k_, st_));
    STG_CUDA(cudaStreamWaitEvent(st_eig_, ev_k_, 0));
    if (rot_pending_) STG_CUDA(cudaStreamWaitEvent(st_eig_, ev_rot_done_, 0));  // X's rotation; st_ keeps its own wait
    std::swap(st_, st_eig_);
    const char* saved = gram_partial_tag_;
    gram_partial_tag_ = "gram_partial_k";
    sched_slot_ = 1;
    gram(X_, ldx(), X_, ldx(), x_rows, kk, kk, true, kc, ldr, 1.0, mark_p_, stamp_);
    chol(kc, ldr, kk, rc, ldr, nullptr, 0, nullptr, 0.0, true);
    sched_slot_ = 0;
    gram_partial_tag_ = saved;
    std::swap(st_, st_eig_);
    STG_CUDA(cudaEventRecord(ev_k_, st_eig_));
    k_ready_ = true;
  }

  void build_xbar(const Pert& pt, Blk z) {
    const i64 p = pt.p;
    const int kk = static_cast<int>(k);
    const int ldr = ld_for(kk);
    double* rc = arena_.get<double>("Rc", static_cast<i64>(kk) * ldr);
    launch(gather_xbar_kernel, dim3(blocks((p + 2 * k) * k)), dim3(256), 0, st_, static_cast<const double*>(X_), ldx(),
           pt.Ploc, pt.dense ? 1 : 0, p, pt.p_old, kk, static_cast<const double*>(nullptr), ldr, z.p, z.ld);
    if (!pt.dense && k_ready_ && !sh_) {  // K and R_c came from early_k (X untouched)
      STG_CUDA(cudaStreamWaitEvent(st_, ev_k_, 0));
      launch(copy2d_kernel, dim3(blocks(k * k)), dim3(256), 0, st_, static_cast<const double*>(rc), ldr, z.p + p * z.ld,
             z.ld, k, kk);
    } else if (!pt.dense) {
      if (pt.p_old > 0) {
        launch(zero_rows_kernel, dim3(blocks(pt.p_old, 8)), dim3(256), 0, st_, X_, ldx(), pt.Ploc, pt.p_old, kk);
        xrestore_ = XRestore{true, pt.Ploc, pt.p_old, z.p, z.ld};
      }
      double* kc = arena_.get<double>("Kc", static_cast<i64>(kk) * ldr);
      pgram(X_, ldx(), X_, ldx(), pt.x_old, kk, kk, true, kc, ldr);
      chol(kc, ldr, kk, rc, ldr, nullptr, 0, nullptr, 0.0, true);
      launch(copy2d_kernel, dim3(blocks(k * k)), dim3(256), 0, st_, static_cast<const double*>(rc), ldr, z.p + p * z.ld,
             z.ld, k, kk);
    } else {  // dense mode: no rows outside P, K = 0
      STG_CUDA(cudaMemset2DAsync(z.p + p * z.ld, sizeof(double) * z.ld, 0, sizeof(double) * kk, k, st_));
    }
  }

  // ---------------------------------------------------------------- Rayleigh-Ritz
  // rayleigh_ritz_step (trackers.cpp:282-308). write_state: rotate X in place;
  // otherwise expand the new vectors (dense mode only) into host `wout`.
  // The RR products of the first `a` basis columns (X-bar and the first
  // candidate block), computed while the sketch's eigensolve runs:
  // G11 = Z1'Z1, Delta Z1, T11 = Z1'(Delta Z1) into the rr_* buffers.
  struct RrPrefix {
    bool valid = false;
    int a = 0, ldd = 0;
  } rr_pre_;

  void rr_prefix(const Pert& pt, Blk z, int a, int dmax) {
    const i64 p = pt.p, G = pt.G;
    const int ldd = ld_for(dmax);
    double* gz = arena_.get<double>("rr_gz", static_cast<i64>(dmax) * ldd);
    double* dz = arena_.get<double>("rr_dz", p * ldd);
    double* tm = arena_.get<double>("rr_t", static_cast<i64>(dmax) * ldd);
    pgram(z.p, z.ld, z.p, z.ld, G, a, a, true, gz, ldd);
    rr_spmm(pt, z.p, z.ld, a, dz, ldd);
    pgram(z.p, z.ld, dz, ldd, p, a, a, true, tm, ldd);
    rr_pre_ = RrPrefix{true, a, ldd};
  }

  void rr_spmm(const Pert& pt, const double* X, int ldx, int m, double* Y, int ldy) {
    SpmmArgs sa{};
    sa.rows = pt.p;
    sa.rowptr = pt.lrp;
    sa.col = pt.lcol;
    sa.val = pt.val;
    sa.X = halo(pt, X, ldx, m, &sa.ldx);
    sa.m = m;
    sa.Y = Y;
    sa.ldy = ldy;
    do_spmm(sa, pt.nnz, pt.p);
  }

  void rayleigh_ritz(const Pert& pt, const Basis& b, std::vector<double>& newvals, bool write_state, double* wout,
                     i64 wrows, Blk xbar_override = Blk{}) {
    const i64 p = pt.p, G = pt.G;
    const int D = b.D, kk = static_cast<int>(k);
    const Blk xb = xbar_override.p ? xbar_override : b.z;
    const bool pre = rr_pre_.valid && !xbar_override.p && rr_pre_.a <= D;
    const int a = pre ? rr_pre_.a : 0;
    const int ldd = pre ? rr_pre_.ldd : ld_for(D);
    rr_pre_.valid = false;
    // Gram check (trackers.cpp:293-295); the products are symmetric, so only
    // their upper triangles are formed / read from here on
    double* gz = arena_.get<double>("rr_gz", static_cast<i64>(D) * ldd);
    double* dz = arena_.get<double>("rr_dz", p * ldd);
    double* tm = arena_.get<double>("rr_t", static_cast<i64>(D) * ldd);
    if (pre) {  // columns a.. : [Z1'Z2; Z2'Z2], Delta Z2, [Z1'(Delta Z2); Z2'(Delta Z2)]
      if (D > a) {
        pgram(b.z.p, b.z.ld, b.z.p + a, b.z.ld, G, D, D - a, false, gz + a, ldd);
        rr_spmm(pt, b.z.p + a, b.z.ld, D - a, dz + a, ldd);
        pgram(b.z.p, b.z.ld, dz + a, ldd, p, D, D - a, false, tm + a, ldd);
      }
    } else {
      pgram(b.z.p, b.z.ld, b.z.p, b.z.ld, G, D, D, true, gz, ldd);
      rr_spmm(pt, b.z.p, b.z.ld, D, dz, ldd);
      // Z'(Delta Z) is symmetric (Delta is): tile pairs ti <= tj, mirrored;
      // the reference symmetrizes the projected matrix anyway (eig.hpp:47)
      pgram(b.z.p, b.z.ld, dz, ldd, p, D, D, true, tm, ldd);
    }
    STG_CUDA(cudaMemsetAsync(flags_ptr(), 0, sizeof(int), st_));
    launch(orthocheck_kernel, dim3(blocks(static_cast<i64>(D) * D)), dim3(256), 0, st_,
           static_cast<const double*>(gz), ldd, D, 1e-6, flags_ptr());
    // zx = Z' X-bar (D x k): the first k columns of Z'Z when X-bar = Z[:, :k]
    const int ldk = ld_for(kk);
    const double* zx = gz;
    int ldzx = ldd, zx_sym = 1;
    if (xbar_override.p) {
      double* zxo = arena_.get<double>("rr_zx", static_cast<i64>(D) * ldk);
      gram(b.z.p, b.z.ld, xb.p, xb.ld, G, D, kk, false, zxo, ldk);
      zx = zxo;
      ldzx = ldk;
      zx_sym = 0;
    }
    double* mm = arena_.get<double>("rr_m", static_cast<i64>(D) * ldd);
    launch(rr_matrix_kernel, dim3(blocks(static_cast<i64>(D) * D)), dim3(256), 0, st_, zx, ldzx,
           static_cast<const double*>(d_values_), kk, static_cast<const double*>(tm), ldd, D, mm, ldd, zx_sym);
    timing_mark(2);
    double* F = arena_.get<double>("rr_F", static_cast<i64>(D) * ldk);
    double* nv = arena_.get<double>("rr_vals", std::max(D, kk));
    // Inverse iteration groups only near-degenerate Ritz values (gap below
    // kRrOrtol ||M||) and the k vectors are then re-orthonormalized as a block
    // (CholQR in spectral order): a vector mixed with a neighbour at gap g by
    // eps ||M|| / g moves the Eq. 14 reconstruction by only eps ||M||, while
    // dstein's 1e-3 grouping serialises whole clusters of tracked values.
    const bool block_ortho = kk <= kCholMaxW;
    if (eig_fast(mm, ldd, D, static_cast<int>(cfg.order), kk, nv, F, ldk, block_ortho ? kRrOrtol : 1e-3)) {
      if (block_ortho) F = orthonormalize_small(F, ldk, D, kk);
    } else {
      double *w = nullptr, *V = nullptr;
      eig(mm, ldd, D, &w, &V, "rr");
      int* perm = arena_.get<int>("rr_perm", D);
      launch(sort_perm_kernel, dim3(1), dim3(256), 0, st_, static_cast<const double*>(w), D,
             static_cast<int>(cfg.order), perm);
      launch(gather_ritz_kernel, dim3(blocks(static_cast<i64>(D) * kk)), dim3(256), 0, st_,
             static_cast<const double*>(V), D, static_cast<const double*>(w), static_cast<const int*>(perm), kk, F,
             ldk, nv);
    }
    timing_mark(3);
    finish_rotation(pt, b.z, D, F, ldk, nv, newvals, write_state, wout, wrows);
  }

  // TRIP-Basic / TRIP / residual modes (trackers.cpp:147-224) on the stacked
  // coordinates: Z = [X-bar] or [X-bar | Delta X-bar], C = X-bar'(Delta X-bar),
  // the coefficient block on the device (trackers.cuh), renormalize_and_sort
  // through the basis Gram, then the shared rotation.
  void perturbation_step(const Pert& pt, int kind, std::vector<double>& newvals) {
    const i64 p = pt.p, N = p + 2 * k, G = pt.G;
    const int kk = static_cast<int>(k);
    const bool rm = kind == ST_RESIDUAL_MODES;
    const int D = rm ? 2 * kk : kk;
    const int ldz = ld_for(2 * kk);
    double* Z = arena_.get<double>("trk_Z", N * ldz);
    STG_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * N * ldz, st_));
    build_xbar(pt, Blk{Z, ldz});
    // Delta X-bar on the rows of P (coordinate rows stay 0): columns [k, 2k) of Z
    SpmmArgs sa{};
    sa.rows = p;
    sa.rowptr = pt.lrp;
    sa.col = pt.lcol;
    sa.val = pt.val;
    sa.X = halo(pt, Z, ldz, kk, &sa.ldx);
    sa.m = kk;
    sa.Y = Z + kk;
    sa.ldy = ldz;
    do_spmm(sa, pt.nnz, p);
    const int ldc = ld_for(kk);
    double* C = arena_.get<double>("trk_C", static_cast<i64>(kk) * ldc);
    pgram(Z, ldz, Z + kk, ldz, G, kk, kk, false, C, ldc);
    const int ldf = ld_for(kk);
    double* F = arena_.get<double>("trk_F", static_cast<i64>(D) * ldf);
    double* F2 = arena_.get<double>("trk_F2", static_cast<i64>(D) * ldf);
    double* lam_new = arena_.get<double>("trk_lam", kk);
    double* nv = arena_.get<double>("trk_vals", kk);
    int* ridge = reinterpret_cast<int*>(d_scal_ + 7);
    STG_CUDA(cudaMemsetAsync(ridge, 0, sizeof(int), st_));
    if (kind == ST_TRIP) {
      STG_CUDA(cudaFuncSetAttribute(trip_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(trip_solve_smem(kk))));
      launch(trip_solve_kernel, dim3(static_cast<unsigned>(kk)), dim3(128), trip_solve_smem(kk), st_,
             static_cast<const double*>(C), ldc, static_cast<const double*>(d_values_), kk, topt_.trip_replace_span,
             F, ldf, ridge);
      launch(lam_new_kernel, dim3(blocks(kk)), dim3(256), 0, st_, static_cast<const double*>(C), ldc,
             static_cast<const double*>(d_values_), kk, lam_new);
    } else {
      launch(pert_coeff_kernel, dim3(1), dim3(256), 0, st_, static_cast<const double*>(C), ldc,
             static_cast<const double*>(d_values_), kk, rm ? 2 : 0, topt_.mu, F, ldf, lam_new);
    }
    const int ldg = ld_for(D);
    double* Gz = arena_.get<double>("trk_G", static_cast<i64>(D) * ldg);
    pgram(Z, ldz, Z, ldz, G, D, D, true, Gz, ldg);
    launch(renorm_sort_kernel, dim3(1), dim3(256), 0, st_, static_cast<const double*>(F), ldf, D, kk,
           static_cast<const double*>(Gz), ldg, static_cast<const double*>(lam_new), static_cast<int>(cfg.order), F2,
           ldf, nv);
    STG_CUDA(cudaMemsetAsync(flags_ptr(), 0, sizeof(int), st_));
    STG_CUDA(cudaMemsetAsync(info_ptr(), 0, sizeof(int), st_));
    timing_mark(1);
    finish_rotation(pt, Blk{Z, ldz}, D, F2, ldf, nv, newvals, /*write_state*/ true, nullptr, 0);
    int hr = 0;
    STG_CUDA(cudaMemcpyAsync(&hr, ridge, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    ridge_used_ = ridge_used_ || hr != 0;
  }

  // The new vectors Z F (D columns of the stacked basis Z, F D x k row-major)
  // and the values nv (device): W = Z F; rows of P -> new rows of X, the
  // a-rows -> A_new for the rows outside P (trackers.cpp:305 and the
  // perturbation trackers' xt). Gated on the device error flags.
  void finish_rotation(const Pert& pt, Blk z, int D, const double* F, int ldk, const double* nv,
                       std::vector<double>& newvals, bool write_state, double* wout, i64 wrows) {
    const i64 p = pt.p, N = p + 2 * k;
    const int kk = static_cast<int>(k);
    Blk bz = z;
    struct {
      Blk z;
    } b{bz};
    // W = Z F (all stacked rows): rows of P -> new rows of X, a-rows -> A_new
    double* W = arena_.get<double>("rr_W", N * ldk);
    nn(b.z.p, b.z.ld, N, D, F, ldk, kk, W, ldk, 1.0, 0.0, nullptr, 0);
    newvals.assign(static_cast<size_t>(kk), 0.0);
    STG_CUDA(cudaMemcpyAsync(newvals.data(), nv, sizeof(double) * kk, cudaMemcpyDeviceToHost, st_));
    launch(merge_spec_kernel, dim3(1), dim3(1), 0, st_, static_cast<const int*>(sticky_ptr()), flags_ptr());
    if (write_state) {
      // X <- X A_new on the rows outside P (in place, DMMA, single column tile),
      // then the rows of P take W's rows. Both are skipped if the step failed.
      // compressed adjacency steps rotate on st_rot_ (the next step waits for
      // it before its first use of X); the row positions of P are copied
      // first, since the next ingestion rewrites them
      const bool aside = rot_aside_ && !sh_ && !pt.dense && k <= 64 &&
                         !(cfg.flags & (ST_FLAG_TIMING | ST_FLAG_KERNEL_TIMING));  // per-phase timings keep it inline
      const int* ploc = pt.Ploc;
      if (aside) {
        int* rp = arena_.get<int>("rot_ploc", std::max<i64>(p, 1));
        if (p > 0) STG_CUDA(cudaMemcpyAsync(rp, pt.Ploc, sizeof(int) * p, cudaMemcpyDeviceToDevice, st_));
        ploc = rp;
        wait_rotation();
        STG_CUDA(cudaEventRecord(ev_rot_ready_, st_));
        STG_CUDA(cudaStreamWaitEvent(st_rot_, ev_rot_ready_, 0));
        std::swap(st_, st_rot_);  // the launches below go to the rotation stream
        sched_slot_ = 2;
      }
      kbegin(kRotate, 16.0 * k * pt.n_total + 8.0 * pt.n_total);
      if (!pt.dense && k <= 64)
        nn(X_, ldx(), pt.x_old, kk, W + (p + k) * ldk, ldk, kk, X_, ldx(), 1.0, 0.0, nullptr, 0, false, true);
      if (pt.dense || k <= 64)
        launch(scatter_rows_kernel, dim3(blocks(p, 8)), dim3(256), 0, st_, X_, ldx(), ploc, pt.dense ? 1 : 0, p,
               static_cast<const double*>(W), ldk, kk, static_cast<const int*>(flags_ptr()),
               static_cast<const int*>(info_ptr()));
      else
        launch(rotate_x_kernel, dim3(blocks(pt.n_total, 8)), dim3(256), 0, st_, X_, ldx(), pt.n_old, pt.n_total,
               pt.dense ? 1 : 0, static_cast<const int*>(pt.mark), pt.stamp, static_cast<const int*>(pt.posmap),
               static_cast<const double*>(W), ldk, static_cast<const double*>(W + (p + k) * ldk), kk,
               static_cast<const int*>(flags_ptr()), static_cast<const int*>(info_ptr()));
      kend();
      if (aside) {
        std::swap(st_, st_rot_);
        sched_slot_ = 0;
        STG_CUDA(cudaEventRecord(ev_rot_done_, st_rot_));
        rot_pending_ = true;
      }
    }
    STG_CUDA(cudaMemcpyAsync(&hs_->sticky, sticky_ptr(), sizeof(int), cudaMemcpyDeviceToHost, st_));
    read_scalars();
    if (rot_pending_ && (hs_->sticky || (hs_->flags & (kNonFinite | kNotOrthonormal)) || hs_->info != 0)) {
      // the gated rotation must read these flags before anything resets them
      STG_CUDA(cudaStreamSynchronize(st_rot_));
      rot_pending_ = false;
    }
    if (hs_->sticky) throw SpecRedo();  // a speculated decision failed: nothing was written
    if (hs_->flags & kNonFinite) throw InvalidArgument("sym_eig_dense: non-finite entries");
    if (hs_->flags & kNotOrthonormal) throw InvalidArgument("rayleigh_ritz_step: basis is not column-orthonormal");
    if (hs_->info != 0) throw RuntimeError("sym_eig_dense: factorization did not converge");
    if (write_state) {
      STG_CUDA(cudaMemcpyAsync(d_values_, nv, sizeof(double) * kk, cudaMemcpyDeviceToDevice, st_));
    } else if (wout) {
      std::vector<double> tmp(static_cast<size_t>(wrows * kk));
      STG_CUDA(cudaMemcpy2DAsync(tmp.data(), sizeof(double) * kk, W, sizeof(double) * ldk, sizeof(double) * kk, wrows,
                                 cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      std::memcpy(wout, tmp.data(), sizeof(double) * wrows * kk);
    }
  }

  // ||Op x_i - theta_i x_i||_2 for the tracked pairs on the current operator
  // ---------------------------------------------------------------- tracker_init
  // Row classes of a full operator for the SpMV (lanczos.cuh), stream-ordered
  // temporaries released with the plan.
  struct SpvBufs {
    SpvPlan pl;
    std::vector<void*> mem;
  };
  SpvBufs spv_plan(const int* rp, i64 rows) {
    SpvBufs b;
    auto tmp = [&](size_t bytes) {
      void* p = arena_.alloc(std::max<size_t>(bytes, 16));
      b.mem.push_back(p);
      return p;
    };
    const size_t ni = sizeof(int) * (rows + 1);
    int* fs = static_cast<int*>(tmp(ni));
    int* fm = static_cast<int*>(tmp(ni));
    int* fl = static_cast<int*>(tmp(ni));
    int* sg = static_cast<int*>(tmp(ni));
    int* ps = static_cast<int*>(tmp(ni));
    int* pm = static_cast<int*>(tmp(ni));
    int* pl = static_cast<int*>(tmp(ni));
    int* pg = static_cast<int*>(tmp(ni));
    launch(spv_classify_kernel, dim3(blocks(rows + 1)), dim3(256), 0, st_, rp, rows, fs, fm, fl, sg);
    scan_int(fs, ps, rows + 1);
    scan_int(fm, pm, rows + 1);
    scan_int(fl, pl, rows + 1);
    scan_int(sg, pg, rows + 1);
    int cnt[4];
    STG_CUDA(cudaMemcpyAsync(&cnt[0], ps + rows, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(&cnt[1], pm + rows, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(&cnt[2], pl + rows, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(&cnt[3], pg + rows, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    int* ls = static_cast<int*>(tmp(sizeof(int) * cnt[0]));
    int* lm = static_cast<int*>(tmp(sizeof(int) * cnt[1]));
    int* ll = static_cast<int*>(tmp(sizeof(int) * cnt[2]));
    int* sr = static_cast<int*>(tmp(sizeof(int) * cnt[3]));
    int* si = static_cast<int*>(tmp(sizeof(int) * cnt[3]));
    double* part = static_cast<double*>(tmp(sizeof(double) * cnt[3]));
    if (rows > 0)
      launch(spv_scatter_kernel, dim3(blocks(rows)), dim3(256), 0, st_, static_cast<const int*>(fs),
             static_cast<const int*>(ps), static_cast<const int*>(fm), static_cast<const int*>(pm),
             static_cast<const int*>(fl), static_cast<const int*>(pl), static_cast<const int*>(sg),
             static_cast<const int*>(pg), rows, ls, lm, ll, sr, si);
    b.pl = SpvPlan{ls, lm, ll, sr, si, pg, cnt[0], cnt[1], cnt[2], cnt[3], part};
    return b;
  }
  void spv_release(SpvBufs& b) {
    for (void* p : b.mem) arena_.release(p);
    b.mem.clear();
  }
  // y = Op x (matvec, sparse.cpp:79-82); y also stored at out2[r * ld2]
  void spmv(const DevCsr& op, const SpvPlan& pl, const double* x, double* y, double* out2, int ld2) {
    int* fl = flags_ptr();
    if (pl.n_short)
      launch(spv_short_kernel, dim3(blocks(static_cast<i64>(pl.n_short) * 8)), dim3(256), 0, st_,
             static_cast<const int*>(op.rp), static_cast<const int*>(op.col), static_cast<const double*>(op.val), x,
             pl.l_short, pl.n_short, y, out2, ld2, fl);
    if (pl.n_med)
      launch(spv_med_kernel, dim3(blocks(static_cast<i64>(pl.n_med) * 32)), dim3(256), 0, st_,
             static_cast<const int*>(op.rp), static_cast<const int*>(op.col), static_cast<const double*>(op.val), x,
             pl.l_med, pl.n_med, y, out2, ld2, fl);
    if (pl.n_seg) {
      launch(spv_seg_kernel, dim3(blocks(static_cast<i64>(pl.n_seg) * 32)), dim3(256), 0, st_,
             static_cast<const int*>(op.rp), static_cast<const int*>(op.col), static_cast<const double*>(op.val), x,
             pl.seg_row, pl.seg_idx, pl.n_seg, pl.seg_part);
      launch(spv_fix_kernel, dim3(blocks(pl.n_long)), dim3(256), 0, st_, static_cast<const int*>(op.rp), pl.l_long,
             pl.n_long, pl.p_seg, static_cast<const double*>(pl.seg_part), y, out2, ld2, fl);
    }
  }

  // lz_dot / lz_update with the accumulator count for j columns
  template <bool NORM>
  void lz_launch(int which, const double* V, int ldv, int j, const double* coef, const double* vi, double* vo, i64 N,
                 double* partial, int ldp, int G) {
    const int na = std::max(1, static_cast<int>(cdiv(j, 32)));
#define STG_LZ(NA)                                                                                                  \
  case NA:                                                                                                          \
    if (which == 0)                                                                                                 \
      launch(lz_dot_kernel<NA>, dim3(G), dim3(kLzThreads), 0, st_, V, ldv, j, vi, N, partial, ldp);                 \
    else if (which == 2)                                                                                            \
      launch(lz_colsq_kernel<NA>, dim3(G), dim3(kLzThreads), 0, st_, V, ldv, j, N, partial, ldp);                   \
    else                                                                                                            \
      launch(lz_update_kernel<NA, NORM>, dim3(G), dim3(kLzThreads), 0, st_, V, ldv, j, coef, vi, vo, N, partial, ldp); \
    break;
    switch (na) {
      STG_LZ(1) STG_LZ(2) STG_LZ(3) STG_LZ(4) STG_LZ(5) STG_LZ(6) STG_LZ(7) STG_LZ(8)
      default: throw InvalidArgument("lanczos_topk: max_basis above the device limit (256)");
    }
#undef STG_LZ
  }

  // GaussianSampler(rseed) draws [pos, pos + count) into out (device)
  void gauss_draws(u64 rseed, i64 pos, i64 count, double* out) {
    const i64 words = 2 * cdiv(pos + count, 2);
    const i64 nb = cdiv(words, kMtM);
    u64* raw = static_cast<u64*>(arena_.alloc(sizeof(u64) * nb * kMtM));
    u64* ring = static_cast<u64*>(arena_.alloc(sizeof(u64) * kMtRing));
    launch(mt19937_64_kernel, dim3(1), dim3(160), 0, st_, rseed, static_cast<i64>(0), nb, 1, ring, raw);
    launch(gauss_range_kernel, dim3(blocks(count)), dim3(256), 0, st_, static_cast<const u64*>(raw), pos, count, out);
    arena_.release(raw);
    arena_.release(ring);
  }

  // lanczos_topk (lanczos.hpp:38-127) on the tracked operator; the leading
  // k eigenpairs go to X (rows [0, N)) and `values`.
  void lanczos(const DevCsr& op, i64 N, const LzOpts& o) {
    const i64 kq = k;
    if (N < 1) throw InvalidArgument("lanczos_topk: empty operator");
    if (kq < 1 || kq > N) throw InvalidArgument("lanczos_topk: k must satisfy 1 <= k <= n");
    i64 m = o.max_basis > 0 ? o.max_basis : std::max<i64>(2 * kq + 20, 40);
    if (m < kq) throw InvalidArgument("lanczos_topk: max_basis below k");
    m = std::min(m, N);
    if (m > kLzMaxCols) throw InvalidArgument("lanczos_topk: max_basis above the device limit (256)");
    const int mm = static_cast<int>(m);
    const int ldv = ld_for(mm);
    const int keep_max = static_cast<int>(std::min<i64>(m, kq + std::min<i64>(kq, 10) + 2));
    const int ldt = ld_for(std::max<i64>(keep_max, kq));
    const int G = static_cast<int>(std::min<i64>(cdiv(N, 64), 148 * 8));
    double* V = static_cast<double*>(arena_.alloc(sizeof(double) * N * ldv));
    double* W = static_cast<double*>(arena_.alloc(sizeof(double) * N * ldv));
    double* T = static_cast<double*>(arena_.alloc(sizeof(double) * N * ldt));
    double* vb[2] = {static_cast<double*>(arena_.alloc(sizeof(double) * N)),
                     static_cast<double*>(arena_.alloc(sizeof(double) * N))};
    double* part = static_cast<double*>(arena_.alloc(sizeof(double) * G * kLzMaxCols));
    double* small = static_cast<double*>(arena_.alloc(sizeof(double) * (4 * kLzMaxCols + 8)));
    double* c1 = small;
    double* c2 = small + kLzMaxCols;
    double* nrm = small + 2 * kLzMaxCols;      // [0] ||v||^2 -> ||v||
    double* rn = small + 2 * kLzMaxCols + 8;   // residual norms^2 (kk)
    const int ldh = ld_for(mm);
    double* H = static_cast<double*>(arena_.alloc(sizeof(double) * mm * ldh));
    double* F = static_cast<double*>(arena_.alloc(sizeof(double) * mm * ldt));
    double* wsort = static_cast<double*>(arena_.alloc(sizeof(double) * mm));
    SpvBufs sp = spv_plan(op.rp, N);
    struct Free {
      Session* s;
      std::vector<void*> p;
      SpvBufs* sp;
      ~Free() {
        for (void* q : p) s->arena_.release(q);
        s->spv_release(*sp);
        cudaStreamSynchronize(s->st_);
      }
    } fr{this, {V, W, T, vb[0], vb[1], part, small, H, F, wsort}, &sp};
    const u64 rseed = mix_seed(cfg.seed, 0x1a2cULL);
    i64 draw_pos = 0;
    int cur = 0;
    auto fresh_vector = [&]() {
      gauss_draws(rseed, draw_pos, N, vb[cur]);
      draw_pos += N;
    };
    // ||v||^2 (+ the non-finite flag of the last product) on the host
    std::vector<double> hbuf(static_cast<size_t>(2 * kLzMaxCols + 8));
    auto norm2_of = [&](const double* v) {
      lz_launch<true>(1, V, ldv, 0, c1, v, const_cast<double*>(v), N, part, kLzMaxCols, G);
      launch(lz_colsum_kernel, dim3(1), dim3(256), 0, st_, static_cast<const double*>(part), G, kLzMaxCols, 1, nrm);
      STG_CUDA(cudaMemcpyAsync(hbuf.data(), nrm, sizeof(double), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaMemcpyAsync(&hs_->flags, flags_ptr(), sizeof(int), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      if (hs_->flags & 1) throw RuntimeError("lanczos_topk: operator produced non-finite values");
      return hbuf[0];
    };
    STG_CUDA(cudaMemsetAsync(flags_ptr(), 0, sizeof(int), st_));
    fresh_vector();
    int j = 0;
    double a_norm = 0.0;
    double best_worst = std::numeric_limits<double>::infinity();
    std::vector<double> wv(static_cast<size_t>(mm)), res(static_cast<size_t>(kq));
    lz_restarts = lz_products = 0;
    for (i64 restart = 0;; ++restart) {
      int fresh = 0;
      while (j < mm) {
        double* v = vb[cur];
        double* v1 = vb[1 - cur];
        double n2;
        if (j > 0) {  // two Gram-Schmidt passes against the basis (lanczos.hpp:59-60)
          lz_launch<false>(0, V, ldv, j, nullptr, v, nullptr, N, part, kLzMaxCols, G);
          launch(lz_colsum_kernel, dim3(j), dim3(256), 0, st_, static_cast<const double*>(part), G, kLzMaxCols, j, c1);
          lz_launch<false>(1, V, ldv, j, c1, v, v1, N, part, kLzMaxCols, G);
          launch(lz_colsum_kernel, dim3(j), dim3(256), 0, st_, static_cast<const double*>(part), G, kLzMaxCols, j, c2);
          lz_launch<true>(1, V, ldv, j, c2, v1, v, N, part, kLzMaxCols, G);
          launch(lz_colsum_kernel, dim3(1), dim3(256), 0, st_, static_cast<const double*>(part), G, kLzMaxCols, 1, nrm);
          STG_CUDA(cudaMemcpyAsync(hbuf.data(), nrm, sizeof(double), cudaMemcpyDeviceToHost, st_));
          STG_CUDA(cudaMemcpyAsync(&hs_->flags, flags_ptr(), sizeof(int), cudaMemcpyDeviceToHost, st_));
          STG_CUDA(cudaStreamSynchronize(st_));
          if (hs_->flags & 1) throw RuntimeError("lanczos_topk: operator produced non-finite values");
          n2 = hbuf[0];
        } else {
          n2 = norm2_of(v);
        }
        const double nr = std::sqrt(n2);
        if (!(nr > 1e-12)) {
          if (++fresh > 4) break;  // invariant subspace; solve with what we have
          fresh_vector();
          continue;
        }
        fresh = 0;
        launch(lz_sqrt_kernel, dim3(1), dim3(1), 0, st_, nrm);
        launch(lz_store_kernel, dim3(blocks(N)), dim3(256), 0, st_, v, N, static_cast<const double*>(nrm), V, ldv, j);
        spmv(op, sp.pl, v, v1, W + j, ldv);  // w = A v, stored as column j of W; v <- w
        ++lz_products;
        cur = 1 - cur;
        ++j;
      }
      if (j == 0) throw RuntimeError("lanczos_topk: could not build a starting basis");
      // Rayleigh-Ritz on the retained basis (lanczos.hpp:80-84)
      const int kk = static_cast<int>(std::min<i64>(kq, j));
      const int keep = static_cast<int>(std::min<i64>(j - 1 > 0 ? j - 1 : j, kq + std::min<i64>(kq, 10) + 2));
      const int want = std::max(kk, keep);
      gram(V, ldv, W, ldv, N, j, j, false, H, ldh);
      const double* Fr = ritz(H, ldh, j, want, wsort, F, ldt);
      nn(V, ldv, N, j, Fr, ldt, kk, X_, ldx(), 1.0, 0.0, nullptr, 0);  // x = V F_k
      nn(W, ldv, N, j, Fr, ldt, kk, T, ldt, 1.0, 0.0, nullptr, 0);     // W F_k
      launch(lz_residual_kernel, dim3(blocks(N * kk)), dim3(256), 0, st_, T, ldt, static_cast<const double*>(X_),
             ldx(), static_cast<const double*>(wsort), N, kk);
      lz_launch<false>(2, T, ldt, kk, nullptr, nullptr, nullptr, N, part, kLzMaxCols, G);
      launch(lz_colsum_kernel, dim3(kk), dim3(256), 0, st_, static_cast<const double*>(part), G, kLzMaxCols, kk, rn);
      STG_CUDA(cudaMemcpyAsync(wv.data(), wsort, sizeof(double) * j, cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaMemcpyAsync(res.data(), rn, sizeof(double) * kk, cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaMemcpyAsync(&hs_->flags, flags_ptr(), sizeof(int), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaMemcpyAsync(&hs_->info, info_ptr(), sizeof(int), cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
      if (hs_->flags & 1) throw RuntimeError("lanczos_topk: operator produced non-finite values");
      if (hs_->flags & kNonFinite) throw InvalidArgument("sym_eig_dense: non-finite entries");
      if (hs_->info != 0) throw RuntimeError("sym_eig_dense: factorization did not converge");
      for (int i = 0; i < j; ++i) a_norm = std::max(a_norm, std::fabs(wv[static_cast<size_t>(i)]));
      const double scale = std::max(a_norm, 1e-300);
      int first_unconverged = -1;
      double worst = 0.0;
      for (int i = 0; i < kk; ++i) {
        const double r = std::sqrt(res[static_cast<size_t>(i)]);
        worst = std::max(worst, r);
        if (first_unconverged < 0 && r > o.tol * scale) first_unconverged = i;
      }
      best_worst = std::min(best_worst, worst);
      lz_restarts = restart;
      if (lz_log2_) {
        auto sum = [&](const double* p, i64 rows, int cols, int ld) {
          std::vector<double> h(static_cast<size_t>(rows * ld));
          STG_CUDA(cudaMemcpy(h.data(), p, sizeof(double) * rows * ld, cudaMemcpyDeviceToHost));
          double s = 0.0;
          for (i64 r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) s += std::fabs(h[static_cast<size_t>(r * ld + c)]) * (1.0 + 1e-3 * c);
          return s;
        };
        fprintf(stderr, "lzdbg restart %lld H %.17g F %.17g Fr %.17g V %.17g W %.17g X %.17g T %.17g res0 %.17g\n",
                static_cast<long long>(restart), sum(H, j, j, ldh), sum(F, j, want, ldt), sum(Fr, j, want, ldt),
                sum(V, N, j, ldv), sum(W, N, j, ldv), sum(X_, N, kk, ldx()), sum(T, N, kk, ldt), res[0]);
      }
      if (lz_log_ && (restart < 12 || restart % 50 == 0))
        fprintf(stderr, "lanczos restart %lld j %d worst %.3e first_unconverged %d a_norm %.6g w0 %.17g w_kk-1 %.17g\n",
                static_cast<long long>(restart), j, worst, first_unconverged, a_norm, wv[0], wv[static_cast<size_t>(kk - 1)]);
      if ((first_unconverged < 0 && kk == kq) || j >= N) {
        values.assign(wv.begin(), wv.begin() + kk);
        values.resize(static_cast<size_t>(kq), 0.0);
        return;
      }
      if (restart >= o.max_restarts) {
        std::ostringstream msg;
        msg << "lanczos_topk: no convergence after " << o.max_restarts << " restarts (best worst-case residual "
            << best_worst << ", tol " << o.tol * scale << ")";
        throw RuntimeError(msg.str());
      }
      // thick restart (lanczos.hpp:116-125): the next direction is the first
      // unconverged residual, then V, W <- V F_keep, W F_keep
      const int pick = first_unconverged >= 0 ? first_unconverged : kk - 1;
      launch(lz_column_kernel, dim3(blocks(N)), dim3(256), 0, st_, static_cast<const double*>(T), ldt, pick, N,
             vb[cur]);
      nn(V, ldv, N, j, Fr, ldt, keep, T, ldt, 1.0, 0.0, nullptr, 0);
      launch(copy2d_kernel, dim3(blocks(N * keep)), dim3(256), 0, st_, static_cast<const double*>(T), ldt, V, ldv, N,
             keep);
      nn(W, ldv, N, j, Fr, ldt, keep, T, ldt, 1.0, 0.0, nullptr, 0);
      launch(copy2d_kernel, dim3(blocks(N * keep)), dim3(256), 0, st_, static_cast<const double*>(T), ldt, W, ldv, N,
             keep);
      j = keep;
      if (!(std::sqrt(norm2_of(vb[cur])) > 0.0)) fresh_vector();
    }
  }

  // sym_eig_dense of a j x j Lanczos projection (symmetrized (H + H')/2 as
  // eig.hpp:39): all values in spectral order, `want` leading vectors
  // (row-major j x want, ldf).
  // Returns the buffer holding the `want` vectors (F, or its re-orthonormalized
  // copy). Like the Rayleigh-Ritz solve of the step, inverse iteration groups
  // only near-degenerate values (gap below kRrOrtol ||H||) and the vectors are
  // then re-orthonormalized as a block (CholQR), so clusters of close Ritz
  // values (SBM blocks) cost no serial dstein sweeps and keep eps-accurate
  // residuals.
  const double* ritz(const double* H, int ldh, int j, int want, double* wsort, double* F, int ldf) {
    STG_CUDA(cudaMemsetAsync(info_ptr(), 0, sizeof(int), st_));
    if (!(cfg.flags & ST_FLAG_CUSOLVER_EIG) && j <= kEigMaxN && want <= kCholMaxW) {
      double* dbuf = arena_.get<double>("eig_dbuf", static_cast<i64>(eig_scratch_doubles(j, want)));
      int* ibuf = arena_.get<int>("eig_ibuf", static_cast<i64>(eig_scratch_ints(j, want)));
      kbegin(kEig, 4.0 * j * j * j / 3.0);
      syev_launch([&](auto kernel, dim3 g, dim3 bl, size_t sm, auto... args) { launch(kernel, g, bl, sm, st_, args...); },
                  H, ldh, j, /*sym_input*/ 0, static_cast<int>(cfg.order), want, kRrOrtol, wsort, F, ldf, dbuf, ibuf,
                  flags_ptr());
      kend();
      return orthonormalize_small(F, ldf, j, want);
    }
    double *w = nullptr, *Vc = nullptr;
    eig(H, ldh, j, &w, &Vc, "lz");
    int* perm = arena_.get<int>("lz_perm", j);
    launch(sort_perm_kernel, dim3(1), dim3(256), 0, st_, static_cast<const double*>(w), j,
           static_cast<int>(cfg.order), perm);
    launch(gather_ritz_kernel, dim3(blocks(static_cast<i64>(j) * want)), dim3(256), 0, st_,
           static_cast<const double*>(Vc), j, static_cast<const double*>(w), static_cast<const int*>(perm), want, F, ldf,
           wsort);
    launch(lz_sorted_vals_kernel, dim3(blocks(j)), dim3(256), 0, st_, static_cast<const double*>(w),
           static_cast<const int*>(perm), j, wsort);
    return F;
  }

 public:
  // Tracking quality against reference vectors Y (n x k, column-major, e.g. a
  // Lanczos reference of the current operator as experiment.cpp:177-184
  // computes): psi_i = principal_angle(x_i, y_i) (metrics.cpp:17-27) and the
  // largest principal angle between span(X) and span(Y) (metrics.cpp:243-259),
  // both on the device. The spans are orthonormalized by CholeskyQR2 (the
  // reference's MGS gives the same span for full-rank inputs).
  void angles(const double* y, i64 ld, double* psi, double* largest) {
    if (sh_) throw InvalidArgument("st_angles: not available on sharded sessions");
    const i64 rows = n;
    const int kk = static_cast<int>(k), ldq = ldx();
    if (ld < rows) throw InvalidArgument("st_angles: leading dimension below n");
    std::vector<void*> tmp;
    auto alloc = [&](size_t b) {
      void* p = arena_.alloc(std::max<size_t>(b, 16));
      tmp.push_back(p);
      return static_cast<double*>(p);
    };
    struct Free {
      Session* s;
      std::vector<void*>* t;
      ~Free() {
        for (void* p : *t) s->arena_.release(p);
        cudaStreamSynchronize(s->st_);
      }
    } fr{this, &tmp};
    double* Y = alloc(sizeof(double) * rows * ldq);
    {
      std::vector<double> yr(static_cast<size_t>(rows * kk));
      for (int c = 0; c < kk; ++c)
        for (i64 i = 0; i < rows; ++i) yr[static_cast<size_t>(i * kk + c)] = y[c * ld + i];
      STG_CUDA(cudaMemcpy2DAsync(Y, sizeof(double) * ldq, yr.data(), sizeof(double) * kk, sizeof(double) * kk, rows,
                                 cudaMemcpyHostToDevice, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
    }
    // ---- psi (two column-statistic passes)
    const int G = static_cast<int>(std::max<i64>(1, std::min<i64>(cdiv(rows, 256), 148 * 4)));
    const int ldp = 3 * kk;
    double* part = alloc(sizeof(double) * G * ldp);
    double* stats = alloc(sizeof(double) * 3 * kk);
    double* diffs = alloc(sizeof(double) * 2 * kk);
    const size_t sm3 = sizeof(double) * (kMetThreads / 32) * 3 * kk, sm2 = sizeof(double) * (kMetThreads / 32) * 2 * kk;
    STG_CUDA(cudaFuncSetAttribute(angle_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm3)));
    STG_CUDA(cudaFuncSetAttribute(angle_diff_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm2)));
    launch(angle_stats_kernel, dim3(G), dim3(kMetThreads), sm3, st_, static_cast<const double*>(X_), ldq,
           static_cast<const double*>(Y), ldq, rows, kk, part, ldp);
    launch(lz_colsum_kernel, dim3(3 * kk), dim3(256), 0, st_, static_cast<const double*>(part), G, ldp, 3 * kk, stats);
    launch(angle_diff_kernel, dim3(G), dim3(kMetThreads), sm2, st_, static_cast<const double*>(X_), ldq,
           static_cast<const double*>(Y), ldq, rows, kk, static_cast<const double*>(stats), part, ldp);
    launch(lz_colsum_kernel, dim3(2 * kk), dim3(256), 0, st_, static_cast<const double*>(part), G, ldp, 2 * kk, diffs);
    std::vector<double> hs(static_cast<size_t>(3 * kk)), hd(static_cast<size_t>(2 * kk));
    STG_CUDA(cudaMemcpyAsync(hs.data(), stats, sizeof(double) * 3 * kk, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaMemcpyAsync(hd.data(), diffs, sizeof(double) * 2 * kk, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    for (int c = 0; c < kk; ++c) {
      if (hs[3 * c] == 0.0 || hs[3 * c + 1] == 0.0) throw InvalidArgument("zero vector has no angle");
      if (psi) psi[c] = 2.0 * std::atan2(std::sqrt(hd[2 * c]), std::sqrt(hd[2 * c + 1]));
    }
    if (!largest) return;
    // ---- largest principal angle: Qa, Qb by CholeskyQR2, G = Qa'Qb, R = Qa - Qb G'
    const int ldk = ld_for(kk);
    double* Gm = alloc(sizeof(double) * kk * ldk);
    double* Rk = alloc(sizeof(double) * kk * ldk);
    double* Ri = alloc(sizeof(double) * kk * ldk);
    double* Qa = alloc(sizeof(double) * rows * ldq);
    double* Qb = alloc(sizeof(double) * rows * ldq);
    double* T1 = alloc(sizeof(double) * rows * ldq);
    STG_CUDA(cudaMemsetAsync(flags_ptr(), 0, sizeof(int), st_));
    auto cholqr2 = [&](const double* A, double* Q) {
      const double* src = A;
      for (int pass = 0; pass < 2; ++pass) {
        gram(src, ldq, src, ldq, rows, kk, kk, true, Gm, ldk);
        chol(Gm, ldk, kk, Rk, ldk, Ri, ldk, nullptr, 0.0, true);
        double* dst = pass == 0 ? T1 : Q;
        nn(src, ldq, rows, kk, Ri, ldk, kk, dst, ldq, 1.0, 0.0, nullptr, 0, /*tri*/ true);
        src = dst;
      }
    };
    cholqr2(X_, Qa);
    cholqr2(Y, Qb);
    double* Gt = alloc(sizeof(double) * kk * ldk);
    double* GtG = alloc(sizeof(double) * kk * ldk);
    double* RtR = alloc(sizeof(double) * kk * ldk);
    gram(Qb, ldq, Qa, ldq, rows, kk, kk, false, Gt, ldk);             // G' = Qb'Qa
    nn(Qb, ldq, rows, kk, Gt, ldk, kk, T1, ldq, -1.0, 1.0, Qa, ldq);  // R = Qa - Qb G'
    gram(T1, ldq, T1, ldq, rows, kk, kk, true, RtR, ldk);             // R'R
    gram(Gt, ldk, Gt, ldk, kk, kk, kk, true, GtG, ldk);               // G G' (same singular values as G)
    double* wv = alloc(sizeof(double) * 2 * kk);
    double* fv = alloc(sizeof(double) * kk * ldk);
    read_scalars();
    if (hs_->flags & kBreakdown) throw InvalidArgument("st_angles: rank-deficient vectors");
    const bool dev = eig_fast(GtG, ldk, kk, /*alg_desc*/ 1, 1, wv, fv, ldk) &&
                     eig_fast(RtR, ldk, kk, /*alg_desc*/ 1, 1, wv + kk, fv, ldk);
    std::vector<double> hw(static_cast<size_t>(2 * kk));
    if (dev) {
      STG_CUDA(cudaMemcpyAsync(hw.data(), wv, sizeof(double) * 2 * kk, cudaMemcpyDeviceToHost, st_));
      STG_CUDA(cudaStreamSynchronize(st_));
    } else {
      throw InvalidArgument("st_angles: k above the on-device eigensolver limit");
    }
    const double c = std::sqrt(std::max(hw[static_cast<size_t>(kk - 1)], 0.0));  // smallest singular value of G
    const double sres = std::sqrt(std::max(hw[static_cast<size_t>(kk)], 0.0));   // largest of the residual
    *largest = std::atan2(sres, std::max(c, 0.0));
  }

  // (A, or the shifted Laplacian T): the residual the reference's Lanczos
  // convergence test measures (lanczos.hpp:85-95). One full-operator SpMM
  // Op X (the north star's A Z with Z = X) on the segment-planned CSR kernel,
  // then deterministic column sums.
  void residual_norms(double* out) {
    if (sh_) throw InvalidArgument("st_residual_norms: not available on sharded sessions");
    const DevCsr& op = is_laplacian() ? T() : A();
    const i64 rows = n;
    const int kk = static_cast<int>(k);
    if (rows == 0) {
      std::fill(out, out + kk, 0.0);
      return;
    }
    // stream-ordered temporaries: a monitoring call leaves the session's
    // persistent footprint unchanged
    double* AX = nullptr;
    const int nb = static_cast<int>(cdiv(rows, 256));
    double* part = nullptr;
    double* dout = nullptr;
    STG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&AX), sizeof(double) * rows * ldx(), st_));
    STG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * nb * kk, st_));
    STG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), sizeof(double) * kk, st_));
    SpmmArgs sa{};
    sa.rows = rows;
    sa.row_off = 0;
    sa.rowptr = op.rp;
    sa.col = op.col;
    sa.val = op.val;
    sa.col_lo = 0;
    sa.X = X_;
    sa.ldx = static_cast<int>(ldx());
    sa.m = kk;
    sa.Y = AX;
    sa.ldy = static_cast<int>(ldx());
    STG_CUDA(cudaMemsetAsync(AX, 0, sizeof(double) * rows * ldx(), st_));
    do_spmm(sa, op.nnz, rows, kSpmmFull, /*transient*/ true);
    launch(residual_partial_kernel, dim3(static_cast<unsigned>(nb)), dim3(256), 0, st_, static_cast<const double*>(AX),
           static_cast<int>(ldx()), static_cast<const double*>(X_), static_cast<int>(ldx()),
           static_cast<const double*>(d_values_), rows, kk, part);
    launch(residual_reduce_kernel, dim3(static_cast<unsigned>(kk)), dim3(256), 0, st_, static_cast<const double*>(part),
           nb, kk, dout);
    STG_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * kk, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaFreeAsync(AX, st_));
    STG_CUDA(cudaFreeAsync(part, st_));
    STG_CUDA(cudaFreeAsync(dout, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    kflush();
  }

 private:
  // Dense n_total x D column-major expansion of a stacked basis (probes only).
  void expand_dense(const Pert& pt, Blk z, int D, double* out, i64 ldo) {
    const int ldd = ld_for(D);
    double* dz = arena_.get<double>("expand", pt.n_total * ldd);
    const double* arows = z.p + (pt.p + k) * z.ld;
    launch(expand_kernel, dim3(blocks(pt.n_total, 8)), dim3(256), 0, st_, static_cast<const double*>(X_), ldx(),
           pt.n_old, pt.n_total, pt.dense ? 1 : 0, static_cast<const int*>(pt.mark), pt.stamp,
           static_cast<const int*>(pt.posmap), static_cast<const double*>(z.p), z.ld, arows, static_cast<int>(k), D, dz,
           ldd);
    std::vector<double> tmp(static_cast<size_t>(pt.n_total * D));
    STG_CUDA(cudaMemcpy2DAsync(tmp.data(), sizeof(double) * D, dz, sizeof(double) * ldd, sizeof(double) * D,
                               pt.n_total, cudaMemcpyDeviceToHost, st_));
    STG_CUDA(cudaStreamSynchronize(st_));
    for (int c = 0; c < D; ++c)
      for (i64 i = 0; i < pt.n_total; ++i) out[c * ldo + i] = tmp[static_cast<size_t>(i * D + c)];
  }

};

}  // namespace stg

// ====================================================================== C ABI
struct st_session {
  std::unique_ptr<stg::Session> impl;
  std::string err;
};

namespace {
thread_local std::string g_create_error;

// Selects a session's device for the duration of one ABI call and restores the
// caller's current device afterwards (sessions on different GPUs may share a
// process and a host thread).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) (void)cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) (void)cudaSetDevice(prev);
  }
};

// Every ABI call except the steps orders after a pending rotation of X (the
// steps wait for it after their ingestion, Session::run_step).
template <class F>
st_status guarded(st_session* s, F&& f, bool step = false) {
  std::string* err = s ? &s->err : &g_create_error;
  try {
    std::unique_ptr<DeviceGuard> dg;
    if (s && s->impl) dg = std::make_unique<DeviceGuard>(s->impl->cfg.device);
    if (s && s->impl && !step) s->impl->wait_rotation();
    f();
    return ST_OK;
  } catch (const std::invalid_argument& e) {
    *err = e.what();
    return ST_INVALID_ARGUMENT;
  } catch (const stg::CudaError& e) {
    *err = e.what();
    return ST_CUDA_ERROR;
  } catch (const std::runtime_error& e) {
    *err = e.what();
    return ST_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    *err = e.what();
    return ST_OTHER;
  }
}
}  // namespace

extern "C" {

st_status st_create(const st_config* cfg, int64_t n, const int32_t* rowptr, const int32_t* colidx,
                    const double* values_csr, const double* eig_values, const double* eig_vectors, int64_t ld,
                    st_session** out) {
  return guarded(nullptr, [&] {
    if (!cfg || !out || !rowptr || !eig_values || !eig_vectors) throw std::invalid_argument("st_create: null argument");
    if (n < 1) throw std::invalid_argument("st_create: empty graph");
    if (ld < n) throw std::invalid_argument("st_create: leading dimension below n");
    DeviceGuard dg(cfg->device);
    auto s = std::make_unique<st_session>();
    s->impl = std::make_unique<stg::Session>(*cfg, n, rowptr, colidx, values_csr, eig_values, eig_vectors, ld);
    *out = s.release();
  });
}

st_status st_tracker_init(const st_config* cfg, const st_lanczos_options* opts, int64_t n, const int32_t* rowptr,
                          const int32_t* colidx, const double* values_csr, st_session** out) {
  return guarded(nullptr, [&] {
    if (!cfg || !out || !rowptr) throw std::invalid_argument("st_tracker_init: null argument");
    if (n < 1) throw std::invalid_argument("lanczos_topk: empty operator");
    stg::Session::LzOpts lz;
    if (opts) {
      lz.tol = opts->tol;
      lz.max_basis = opts->max_basis;
      lz.max_restarts = opts->max_restarts;
    }
    DeviceGuard dg(cfg->device);
    auto s = std::make_unique<st_session>();
    s->impl = std::make_unique<stg::Session>(*cfg, n, rowptr, colidx, values_csr, nullptr, nullptr, n, nullptr, &lz);
    *out = s.release();
  });
}

st_status st_set_tracker_options(st_session* s, const st_tracker_options* o) {
  return guarded(s, [&] {
    if (!o) throw std::invalid_argument("st_set_tracker_options: null options");
    if (o->restart_inner < ST_TRIP_BASIC || o->restart_inner > ST_TIMERS)
      throw std::invalid_argument("unknown tracker kind");
    if (s->impl->cfg.kind == ST_TIMERS && o->restart_inner == ST_TIMERS)
      throw std::invalid_argument("tracker_init: timers cannot delegate to itself");
    s->impl->topt_ = *o;
  });
}

st_status st_tracker_state(const st_session* s, double* accumulated_change, int64_t* steps_since_restart,
                           double* restart_scale, int32_t* ridge_used) {
  const auto& m = *s->impl;
  if (accumulated_change) *accumulated_change = m.acc_change_;
  if (steps_since_restart) *steps_since_restart = m.steps_since_restart_;
  if (restart_scale) *restart_scale = m.restart_scale_;
  if (ridge_used) *ridge_used = m.ridge_used_ ? 1 : 0;
  return ST_OK;
}

st_status st_init_stats(const st_session* s, int64_t* restarts, int64_t* products) {
  if (restarts) *restarts = s->impl->lz_restarts;
  if (products) *products = s->impl->lz_products;
  return ST_OK;
}

void st_destroy(st_session* s) {
  if (!s) return;
  DeviceGuard dg(s->impl ? s->impl->cfg.device : 0);
  delete s;
}

st_status st_create_sharded(const st_config* cfg, const st_comm* comm, int64_t n_global, int64_t row_lo,
                            int64_t row_hi, int64_t chunk, const int32_t* rowptr, const int32_t* colidx,
                            const double* values_csr, const double* eig_values, const double* eig_vectors,
                            int64_t ld, st_session** out) {
  return guarded(nullptr, [&] {
    if (!cfg || !comm || !out || !rowptr || !eig_values || (!eig_vectors && row_hi > row_lo))
      throw std::invalid_argument("st_create_sharded: null argument");
    if (n_global < 1) throw std::invalid_argument("st_create: empty graph");
    if (ld < row_hi - row_lo) throw std::invalid_argument("st_create: leading dimension below n");
    stg::Session::ShardInit si{*comm, n_global, row_lo, row_hi, chunk};
    DeviceGuard dg(cfg->device);
    auto s = std::make_unique<st_session>();
    s->impl = std::make_unique<stg::Session>(*cfg, row_hi - row_lo, rowptr, colidx, values_csr, eig_values,
                                             eig_vectors, ld, &si);
    *out = s.release();
  });
}

st_status st_nccl_unique_id(void* out128) {
  return guarded(nullptr, [&] {
    if (!out128) throw std::invalid_argument("st_nccl_unique_id: null argument");
    ncclUniqueId id;
    if (stg::nccl_api().GetUniqueId(&id) != ncclSuccess) throw stg::CudaError("ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof(id));
  });
}

st_status st_comm_nccl_create(const void* unique_id, int32_t rank, int32_t size, int32_t device, st_comm* out) {
  return guarded(nullptr, [&] {
    if (!unique_id || !out) throw std::invalid_argument("st_comm_nccl_create: null argument");
    if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("st_comm_nccl_create: bad rank / size");
    DeviceGuard dg(device);
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    auto ctx = std::make_unique<stg::NcclCtx>();
    ctx->rank = rank;
    ctx->size = size;
    const ncclResult_t r = stg::nccl_api().CommInitRank(&ctx->comm, size, id, rank);
    if (r != ncclSuccess)
      throw stg::CudaError(std::string("ncclCommInitRank failed: ") + stg::nccl_api().GetErrorString(r));
    out->rank = rank;
    out->size = size;
    out->ctx = ctx.release();
    out->allreduce_sum_f64 = stg::nccl_allreduce_cb;
    out->allgather = stg::nccl_allgather_cb;
    out->alltoallv = stg::nccl_alltoallv_cb;
  });
}

void st_comm_nccl_destroy(st_comm* c) {
  if (!c || !c->ctx) return;
  auto* ctx = static_cast<stg::NcclCtx*>(c->ctx);
  if (ctx->comm) stg::nccl_api().CommDestroy(ctx->comm);
  delete ctx;
  c->ctx = nullptr;
}

st_status st_shard_stats(const st_session* s, int64_t* halo_bytes_recv, int64_t* halo_bytes_local, int64_t* halos) {
  if (halo_bytes_recv) *halo_bytes_recv = s->impl->halo_bytes_recv_;
  if (halo_bytes_local) *halo_bytes_local = s->impl->halo_bytes_local_;
  if (halos) *halos = s->impl->halo_calls_;
  return ST_OK;
}

st_status st_shard_rows(const st_session* s, int64_t* n_local, int64_t* global_ids) {
  auto* ms = const_cast<st_session*>(s);
  return guarded(ms, [&] {
    if (n_local) *n_local = ms->impl->local_rows();
    if (global_ids) ms->impl->local_ids(reinterpret_cast<stg::i64*>(global_ids));
  });
}

int64_t st_shard_layout(int32_t size, const int64_t* bounds, int64_t chunk, int32_t rank, int64_t n_total,
                        int64_t* global_ids, int64_t cap) {
  if (size < 1 || rank < 0 || rank >= size || chunk < 1 || !bounds) return -1;
  stg::ShardMap m;
  m.n0 = bounds[size];
  m.chunk = chunk;
  m.size = size;
  m.rank = rank;
  const stg::i64* b = reinterpret_cast<const stg::i64*>(bounds);
  m.bounds = b;
  m.own0 = bounds[rank + 1] - bounds[rank];
  m.lo = bounds[rank];
  const int64_t rows = stg::sm_rows(m, rank, n_total, b);
  for (int64_t l = 0; l < rows && l < cap; ++l) global_ids[l] = stg::sm_global(m, l);
  return rows;
}

st_status st_reserve(st_session* s, int64_t n_nodes, int64_t nnz) {
  return guarded(s, [&] { s->impl->reserve(n_nodes, nnz); });
}

st_status st_step(st_session* s, const st_update* upd) {
  return guarded(s, [&] {
    if (!upd) throw std::invalid_argument("st_step: null update");
    s->impl->step(*upd);
  }, /*step*/ true);
}

st_status st_info(const st_session* s, int64_t* n, int64_t* k, uint64_t* steps_taken, int64_t* nnz_a,
                  int64_t* nnz_t, int64_t* nnz_delta, double* alpha) {
  const auto& m = *s->impl;
  if (n) *n = m.n;
  if (k) *k = m.k;
  if (steps_taken) *steps_taken = m.steps_taken;
  if (nnz_a) *nnz_a = m.A().nnz;
  if (nnz_t) *nnz_t = m.is_laplacian() ? m.T().nnz : 0;
  if (nnz_delta) *nnz_delta = m.nnz_delta();
  if (alpha) *alpha = m.alpha;
  return ST_OK;
}

st_status st_get_embedding(const st_session* s, double* values, double* vectors, int64_t ld) {
  auto* ms = const_cast<st_session*>(s);
  return guarded(ms, [&] {
    if (ld < ms->impl->local_rows()) throw std::invalid_argument("st_get_embedding: leading dimension below n");
    ms->impl->get_embedding(values, vectors, ld);
  });
}

st_status st_get_values(const st_session* s, double* values) {
  std::memcpy(values, s->impl->values.data(), sizeof(double) * s->impl->values.size());
  return ST_OK;
}

st_status st_residual_norms(st_session* s, double* norms) {
  return guarded(s, [&] {
    if (!norms) throw std::invalid_argument("st_residual_norms: null argument");
    s->impl->residual_norms(norms);
  });
}

st_status st_angles(st_session* s, const double* ref_vectors, int64_t ld, double* psi, double* largest_angle) {
  return guarded(s, [&] {
    if (!ref_vectors) throw std::invalid_argument("st_angles: null argument");
    s->impl->angles(ref_vectors, ld, psi, largest_angle);
  });
}

st_status st_get_csr(const st_session* s, int32_t which, int32_t* rowptr, int32_t* colidx, double* values) {
  auto* ms = const_cast<st_session*>(s);
  return guarded(ms, [&] { ms->impl->get_csr(which, rowptr, colidx, values); });
}

st_status st_probe_basis(st_session* s, const st_update* upd, int32_t basis_kind, uint64_t seed, double* z,
                         int64_t ld, int64_t max_cols, int64_t* cols) {
  return guarded(s, [&] {
    if (basis_kind < 0 || basis_kind > 3) throw std::invalid_argument("st_probe_basis: unknown basis kind");
    *cols = s->impl->probe_basis(*upd, basis_kind, seed, z, ld, max_cols);
  });
}

st_status st_probe_rr(st_session* s, const st_update* upd, const double* z, int64_t rows, int64_t cols, int64_t ldz,
                      double* values, double* vectors, int64_t ldv) {
  return guarded(s, [&] { s->impl->probe_rr(*upd, z, rows, cols, ldz, values, vectors, ldv); });
}

const char* st_last_error(const st_session* s) { return s ? s->err.c_str() : g_create_error.c_str(); }

int32_t st_last_timings(const st_session* s, double* ms, int32_t cap) {
  const auto& m = *s->impl;
  const int32_t n = std::min<int32_t>(cap, m.ntimings);
  for (int32_t i = 0; i < n; ++i) ms[i] = m.timings[i];
  return n;
}

int64_t st_last_launches(const st_session* s) { return s->impl->launches; }

st_status st_sym_eig_dense(int32_t device, int64_t n, const double* s_colmajor, int32_t order, int64_t want,
                           double* values, double* vectors) {
  return guarded(nullptr, [&] {
    if (n < 0 || want < 0 || want > n) throw std::invalid_argument("sym_eig_dense: bad sizes");
    for (int64_t i = 0; i < n * n; ++i)
      if (!std::isfinite(s_colmajor[i])) throw std::invalid_argument("sym_eig_dense: non-finite entries");
    if (n == 0) return;
    if (n > stg::kEigMaxN) throw std::invalid_argument("st_sym_eig_dense: order above the on-device solver limit");
    DeviceGuard dg(device);
    stg::eig_set_attributes();
    // row-major copy of S' (the solver symmetrizes (S + S')/2 itself)
    std::vector<double> rm(static_cast<size_t>(n * n));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) rm[static_cast<size_t>(i * n + j)] = s_colmajor[j * n + i];
    double *dm, *dw, *df, *dbuf;
    int *di, *ibuf;
    const int64_t wv = std::max<int64_t>(want, 1);
    STG_CUDA(cudaMalloc(&dm, sizeof(double) * n * n));
    STG_CUDA(cudaMalloc(&dw, sizeof(double) * n));
    STG_CUDA(cudaMalloc(&df, sizeof(double) * n * wv));
    STG_CUDA(cudaMalloc(&dbuf, sizeof(double) * stg::eig_scratch_doubles(static_cast<int>(n), static_cast<int>(wv))));
    STG_CUDA(cudaMalloc(&ibuf, sizeof(int) * stg::eig_scratch_ints(static_cast<int>(n), static_cast<int>(wv))));
    STG_CUDA(cudaMalloc(&di, sizeof(int) * 2));
    STG_CUDA(cudaMemset(di, 0, sizeof(int) * 2));
    STG_CUDA(cudaMemcpy(dm, rm.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    stg::syev_launch(
        [&](auto kernel, dim3 g, dim3 bl, size_t sm, auto... args) {
          kernel<<<g, bl, sm>>>(args...);
          STG_LAUNCH();
        },
        dm, static_cast<int>(n), static_cast<int>(n), /*sym_input*/ 0, order, static_cast<int>(wv), 1e-3, dw, df,
        static_cast<int>(wv), dbuf, ibuf, di);
    cudaEventRecord(e1);
    STG_CUDA(cudaDeviceSynchronize());
    if (getenv("STG_EIG_PROF")) {
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      fprintf(stderr, "device syev n=%lld want=%lld: %.3f ms\n", static_cast<long long>(n),
              static_cast<long long>(want), ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    int hflags = 0;
    STG_CUDA(cudaMemcpy(&hflags, di, sizeof(int), cudaMemcpyDeviceToHost));
    if (hflags & stg::kNonFinite) throw std::invalid_argument("sym_eig_dense: non-finite entries");
    std::vector<double> f(static_cast<size_t>(n * wv));
    STG_CUDA(cudaMemcpy(values, dw, sizeof(double) * n, cudaMemcpyDeviceToHost));
    STG_CUDA(cudaMemcpy(f.data(), df, sizeof(double) * n * wv, cudaMemcpyDeviceToHost));
    for (int64_t c = 0; c < want; ++c)
      for (int64_t i = 0; i < n; ++i) vectors[c * n + i] = f[static_cast<size_t>(i * wv + c)];
    cudaFree(dm);
    cudaFree(dw);
    cudaFree(df);
    cudaFree(dbuf);
    cudaFree(ibuf);
    cudaFree(di);
  });
}

st_status st_gaussian_matrix(int32_t device, uint64_t seed, int64_t rows, int64_t cols, double* out_colmajor) {
  return guarded(nullptr, [&] {
    if (rows < 0 || cols < 0) throw std::invalid_argument("gaussian_matrix: negative size");
    if (rows * cols == 0) return;
    DeviceGuard dg(device);
    const int64_t npairs = (rows * cols + 1) / 2;
    const int64_t nblocks = (2 * npairs + stg::kMtM - 1) / stg::kMtM;
    stg::u64 *raw, *ring;
    double* om;
    const int ld = static_cast<int>(cols);
    STG_CUDA(cudaMalloc(&raw, sizeof(stg::u64) * nblocks * stg::kMtM));
    STG_CUDA(cudaMalloc(&ring, sizeof(stg::u64) * stg::kMtRing));
    STG_CUDA(cudaMalloc(&om, sizeof(double) * rows * cols));
    stg::mt19937_64_kernel<<<1, 160>>>(seed, 0, nblocks, 1, ring, raw);
    STG_LAUNCH();
    stg::box_muller_kernel<<<static_cast<unsigned>((npairs + 255) / 256), 256>>>(raw, npairs, rows,
                                                                                 static_cast<int>(cols), om, ld);
    STG_LAUNCH();
    std::vector<double> rm(static_cast<size_t>(rows * cols));
    STG_CUDA(cudaMemcpy(rm.data(), om, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost));
    for (int64_t c = 0; c < cols; ++c)
      for (int64_t r = 0; r < rows; ++r) out_colmajor[c * rows + r] = rm[static_cast<size_t>(r * cols + c)];
    cudaFree(raw);
    cudaFree(ring);
    cudaFree(om);
  });
}

st_status st_debug_bench(st_session* s, int32_t which, int64_t N, int32_t m1, int32_t m2, int32_t flag,
                         int32_t iters, double* ms) {
  return guarded(s, [&] { *ms = s->impl->bench_kernel(which, N, m1, m2, flag, iters); });
}

st_status st_step_blocks(st_session* s, const st_graph_update* upd) {
  return guarded(s, [&] {
    if (!upd) throw std::invalid_argument("st_step_blocks: null update");
    s->impl->step_blocks(*upd, false);
  }, /*step*/ true);
}

st_status st_step_blocks_device(st_session* s, const st_graph_update* upd) {
  return guarded(s, [&] {
    if (!upd) throw std::invalid_argument("st_step_blocks: null update");
    s->impl->step_blocks(*upd, true);
  }, /*step*/ true);
}

st_status st_step_perturbation(st_session* s, int64_t n_old, int64_t n_new, const st_csr_block* delta) {
  return guarded(s, [&] {
    if (!delta) throw std::invalid_argument("st_step_perturbation: null delta");
    s->impl->step_perturbation(n_old, n_new, *delta, false);
  }, /*step*/ true);
}

st_status st_debug_determinism(st_session* s, int32_t which, int64_t N, int32_t m1, int32_t m2, int32_t reps,
                               double* max_diff, double* first_out) {
  return guarded(s, [&] { *max_diff = s->impl->det_check(which, N, m1, m2, reps, first_out); });
}

st_status st_step_device(st_session* s, const st_update* upd) {
  return guarded(s, [&] {
    if (!upd) throw std::invalid_argument("st_step_device: null update");
    s->impl->step(*upd, true);
  }, /*step*/ true);
}

int32_t st_kernel_stats(const st_session* s, int32_t cls, double* ms, int64_t* launches, double* work) {
  if (cls < 0 || cls >= stg::Session::kClasses) return 0;
  const auto& k = s->impl->kstats[cls];
  *ms = k.ms;
  *launches = k.launches;
  *work = k.work;
  return 1;
}

void st_reset_kernel_stats(st_session* s) { s->impl->kreset(); }

int32_t st_kernel_stats2(const st_session* s, int32_t cls, double* ms, int64_t* launches, double* work, double* work2,
                         double* bound_ms) {
  if (cls < 0 || cls >= stg::Session::kClasses) return 0;
  const auto& k = s->impl->kstats[cls];
  *ms = k.ms;
  *launches = k.launches;
  *work = k.work;
  *work2 = k.work2;
  *bound_ms = k.bound_ms;
  return 1;
}

void st_set_peaks(st_session* s, double fp64_tflops, double hbm_gbs) {
  if (fp64_tflops > 0) s->impl->peak_tflops_ = fp64_tflops;
  if (hbm_gbs > 0) s->impl->peak_gbs_ = hbm_gbs;
}

}  // extern "C"
