// Row sharding of the G-REST step over the GPUs of one box.
//
// Node ownership. The initial n0 nodes are split into contiguous row blocks,
// one per rank ([bounds[r], bounds[r+1]), chosen by the caller). Appended
// nodes keep their global ids n_old + j (graph.cpp:76-90, the parity contract)
// and are dealt to the ranks round-robin in chunks of `chunk` ids, so every
// rank receives its share of each step's new rows. A rank stores its rows in
// increasing global id order: its initial block first, then its appended
// chunks in arrival order. Owner, local index and the inverse are closed forms
// (no per-node maps), identical on host and device.
//
// Per step each rank holds the full (small) perturbation Delta — every rank
// validates and assembles the same edit lists, O(edits) — and keeps the rows
// it owns: the CSR merge, the rows of P, the stacked coordinates, the Delta
// SpMMs and the rotation of X are row-local. Dense operands of the SpMMs need
// the rows their owned Delta rows reference on other ranks: a boundary-row
// halo. Once per step (Delta changes every step) each rank lists the distinct
// remote rows of P its compressed Delta references, the lists are exchanged
// (counts by allgather, ids by alltoallv), and the compressed columns are
// renumbered into [own rows of P | received rows, grouped by source rank]. An
// SpMM then copies its own rows, gathers the rows peers asked for and runs one
// alltoallv of exactly the referenced rows (no rank receives rows it does not
// read). Every Gram is a local split-K partial followed by one allreduce.
#pragma once

#include "common.cuh"

namespace stg {

struct ShardMap {
  i64 n0 = 0;            // nodes at session creation (global)
  i64 chunk = 1;         // appended ids per round-robin chunk
  int size = 1, rank = 0;
  const i64* bounds = nullptr;  // size + 1 initial row bounds (device or host copy)
  i64 own0 = 0;          // initial rows of this rank
  i64 lo = 0;            // first initial row of this rank
};

__host__ __device__ __forceinline__ int sm_owner(const ShardMap& m, i64 g) {
  if (g >= m.n0) return static_cast<int>(((g - m.n0) / m.chunk) % m.size);
  int lo = 0, hi = m.size - 1;  // last r with bounds[r] <= g
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (m.bounds[mid] <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Local row of global id g in its owner's storage.
__host__ __device__ __forceinline__ i64 sm_local(const ShardMap& m, i64 g, int owner) {
  if (g < m.n0) return g - m.bounds[owner];
  const i64 t = g - m.n0, j = t / m.chunk;
  return (m.bounds[owner + 1] - m.bounds[owner]) + (j / m.size) * m.chunk + t % m.chunk;
}

// Global id of this rank's local row l.
__host__ __device__ __forceinline__ i64 sm_global(const ShardMap& m, i64 l) {
  if (l < m.own0) return m.lo + l;
  const i64 t = l - m.own0, jj = t / m.chunk;
  return m.n0 + (jj * m.size + m.rank) * m.chunk + t % m.chunk;
}

// Rows rank r owns when the graph has n_total nodes.
inline i64 sm_rows(const ShardMap& m, int r, i64 n_total, const i64* host_bounds) {
  i64 rows = host_bounds[r + 1] - host_bounds[r];
  if (n_total <= m.n0) return rows;
  const i64 a = n_total - m.n0, full = a / m.chunk, rem = a % m.chunk;
  rows += (full / m.size + (full % m.size > r ? 1 : 0)) * m.chunk;
  if (rem > 0 && full % m.size == r) rows += rem;
  return rows;
}

// ---- local perturbation for the row-local CSR merge ----------------------
// Valid Delta entries of owned rows, in the global (row, col) order, with
// rows renumbered to local rows (monotone per owner, so still sorted).
__global__ void own_entry_flag_kernel(const u64* skey, i64 n2, int kb, ShardMap m, int* flag) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e > n2) return;
  int f = 0;
  if (e < n2) {
    const u64 k = skey[e];
    if (k != ~0ULL) f = sm_owner(m, static_cast<i64>(k >> kb)) == m.rank ? 1 : 0;
  }
  flag[e] = f;
}

__global__ void own_entry_scatter_kernel(const u64* skey, const double* sval, i64 n2, int kb, ShardMap m,
                                         const int* flag, const int* pos, u64* lkey, double* lval, int* lrow,
                                         int* lcol, int* rowcnt, int* mark, int stamp) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n2 || !flag[e]) return;
  const u64 k = skey[e];
  const i64 g = static_cast<i64>(k >> kb);
  const int c = static_cast<int>(k & ((1ULL << kb) - 1));
  const int l = static_cast<int>(sm_local(m, g, m.rank));
  const int q = pos[e];
  lkey[q] = (static_cast<u64>(l) << kb) | static_cast<u64>(c);
  lval[q] = sval[e];
  lrow[q] = l;
  lcol[q] = c;
  atomicAdd(rowcnt + l, 1);
  mark[l] = stamp;
}

// ---- rows of P owned by this rank ----------------------------------------
__global__ void own_p_flag_kernel(const int* mark, int stamp, ShardMap m, i64 nloc, int all, int* flag) {
  const i64 l = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l > nloc) return;
  flag[l] = (l < nloc && (all || mark[sm_global(m, l)] == stamp)) ? 1 : 0;
}

// P_loc: local rows (X storage), P_glob: global ids (Delta rows); the send
// buffer of the P exchange is padded with -1 up to pmax.
__global__ void own_p_scatter_kernel(const int* flag, const int* pos, ShardMap m, i64 nloc, int* ploc, int* pglob) {
  const i64 l = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l < nloc && flag[l]) {
    ploc[pos[l]] = static_cast<int>(l);
    pglob[pos[l]] = static_cast<int>(sm_global(m, l));
  }
}

// Halo position of every row of P: rank-major, pmax rows per rank.
__global__ void halo_posmap_kernel(const int* pall, i64 total, int* posmap) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < total && pall[i] >= 0) posmap[pall[i]] = static_cast<int>(i);
}

// Compressed CSR of the owned rows of P: row lengths, then entries with
// columns as halo positions (lcol) and as global ids (scol, the sketch's
// appended-node columns).
__global__ void own_rowlen_kernel(const int* grp, const int* pglob, i64 p, int* cnt) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < p) cnt[t] = grp[pglob[t] + 1] - grp[pglob[t]];
  if (t == p) cnt[t] = 0;
}

__global__ void __launch_bounds__(256) own_compress_kernel(const int* grp, const int* gcol, const double* gval,
                                                           const int* pglob, i64 p, const int* lrp,
                                                           const int* posmap, int* lcol, int* scol, double* val) {
  const i64 t = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= p) return;
  const int s = grp[pglob[t]], e = grp[pglob[t] + 1], o = lrp[t];
  for (int q = s + lane; q < e; q += 32) {
    const int c = gcol[q];
    lcol[o + q - s] = posmap[c];
    scol[o + q - s] = c;
    val[o + q - s] = gval[q];
  }
}

// ---- boundary-row halo plan ----------------------------------------------
// need[h] = 1 for every remote halo position (owner != rank) an owned Delta
// entry references (h = owner * pmax + index in the owner's rows of P).
__global__ void halo_need_kernel(const int* lcol, i64 nnz, i64 pmax, int rank, int* need) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int h = lcol[e];
  if (h / pmax != rank) need[h] = 1;
}

// requested positions in halo order (owner-major, then index) and, per
// position, its slot after the own rows
__global__ void halo_req_kernel(const int* need, const int* pos, i64 total, i64 pmax, i64 p, int* req_idx,
                                int* slot) {
  const i64 h = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= total || !need[h]) return;
  req_idx[pos[h]] = static_cast<int>(h % pmax);  // the owner's local index
  slot[h] = static_cast<int>(p + pos[h]);
}

// compressed columns: own position -> index in the own rows, remote -> slot
__global__ void halo_remap_kernel(int* lcol, i64 nnz, i64 pmax, int rank, const int* slot) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int h = lcol[e];
  lcol[e] = (h / pmax == rank) ? static_cast<int>(h % pmax) : slot[h];
}

// rows a peer asked for, in the order it asked (send buffer of one SpMM halo)
__global__ void gather_rows_kernel(const double* X, int ldx, const int* idx, i64 rows, int m, double* out, int ldo) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * m) return;
  const i64 r = t / m;
  const int c = static_cast<int>(t % m);
  out[r * ldo + c] = X[static_cast<i64>(idx[r]) * ldx + c];
}

// grest3 trailing block on owned rows: entry (i, n_old + j) of Delta -> column j.
__global__ void __launch_bounds__(256) d2_rows_kernel(const int* lrp, const int* scol, const double* val, i64 p,
                                                      i64 n_old, double* out, int ldo) {
  const i64 t = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= p) return;
  for (int e = lrp[t] + lane; e < lrp[t + 1]; e += 32)
    if (scol[e] >= n_old) out[t * ldo + (scol[e] - n_old)] = val[e];
}

// iasc unit columns of the owned appended rows (z points at column k).
__global__ void unit_cols_own_kernel(double* z, int ldz, const int* pglob, i64 p_old, i64 s_loc, i64 n_old) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < s_loc) z[(p_old + t) * ldz + (pglob[p_old + t] - n_old)] = 1.0;
}

// m x m copy of an allreduced Gram; symmetric results are re-mirrored from
// the upper triangle (a reduction over more than two ranks may round the two
// triangles in different orders, the consumers expect exact symmetry).
__global__ void gram_out_kernel(const double* src, int m1, int m2, int sym, double* out, int ldo) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<i64>(m1) * m2) return;
  const int i = static_cast<int>(idx / m2), j = static_cast<int>(idx % m2);
  const bool mirror = sym && i > j;
  out[static_cast<i64>(i) * ldo + j] = mirror ? src[static_cast<i64>(j) * m2 + i] : src[idx];
}

}  // namespace stg
