// On-device ingestion of one update batch (HBM-bound integer/byte work):
//   * validation of the edit lists with the reference's rules and error
//     precedence (proj/src/graph.cpp:45-100),
//   * the symmetric perturbation Delta as a sorted COO -> CSR (graph.cpp:17-32,
//     sparse.cpp:17-23),
//   * A_hat = pad(A) + Delta merged into a fresh CSR with exact-zero pruning
//     and the "invalid deletion" / "negative weight" checks (graph.cpp:102-115),
//   * for Laplacian operators, T_next and Delta_T = T_next - pad(T_old)
//     (graph.cpp:117-151, laplacian_track.cpp:48-64), bit-exact.
#pragma once

#include "common.cuh"

namespace stg {

enum EditError : int {
  kErrNone = 0,
  kErrZeroWeight = 1,
  kErrEditRange = 2,
  kErrSelfLoop = 3,
  kErrDuplicate = 4,
  kErrNewRange = 5,
  kErrNewWeight = 6,
  kErrNewOldOnly = 7,
  kErrNotSymmetric = 8,  // from_triplets validation (sparse.cpp:55-63)
  kErrBlockShape = 9,    // malformed caller CSR block (st_step_blocks / st_step_perturbation)
};

constexpr u64 kSentinel = ~0ULL;

struct EditsDev {
  const i64 *ai, *aj;
  const double* aw;
  const i64 *ri, *rj;
  const i64 *ni, *nj;
  const double* nw;
  i64 n_add, n_rem, n_newe;
  i64 n_old, S;
  int kb;  // key field width: 2^kb > n_old + S, keys are (row << kb | col)
};

__device__ __forceinline__ void edit_at(const EditsDev& d, i64 g, int& list, i64& i, i64& j, double& w) {
  if (g < d.n_add) {
    list = 0; i = d.ai[g]; j = d.aj[g]; w = d.aw[g];
  } else if (g < d.n_add + d.n_rem) {
    const i64 h = g - d.n_add;
    list = 1; i = d.ri[h]; j = d.rj[h]; w = -1.0;
  } else {
    const i64 h = g - d.n_add - d.n_rem;
    list = 2; i = d.ni[h]; j = d.nj[h]; w = d.nw[h];
  }
}

// Per-edit checks in the reference's order, up to (not including) the
// duplicate test; pair keys for the duplicate test (graph.cpp:52-59).
__global__ void edit_check_kernel(EditsDev d, u64* pkey, i64* pval, int* code, int* post) {
  const i64 g = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 E = d.n_add + d.n_rem + d.n_newe;
  if (g >= E) return;
  int list;
  i64 i, j;
  double w;
  edit_at(d, g, list, i, j, w);
  const i64 n_total = d.n_old + d.S;
  int c = kErrNone, p = 0;
  if (list == 0 && w == 0.0) c = kErrZeroWeight;
  else if (list < 2 && (i < 0 || j < 0 || i >= d.n_old || j >= d.n_old)) c = kErrEditRange;
  else if (list == 2 && (i < 0 || j < 0 || i >= n_total || j >= n_total)) c = kErrNewRange;
  else if (list == 2 && w <= 0.0) c = kErrNewWeight;
  else if (i == j) c = kErrSelfLoop;
  if (list == 2 && c == kErrNone && (i > j ? i : j) < d.n_old) p = 1;
  code[g] = c;
  post[g] = p;
  const i64 lo = i < j ? i : j, hi = i < j ? j : i;
  pkey[g] = c == kErrNone ? ((static_cast<u64>(lo) << d.kb) | static_cast<u64>(hi)) : kSentinel;
  pval[g] = g;
}

// Sorted pair keys (stable: edit order within a key): later occurrences are
// duplicates of an earlier edit.
__global__ void dup_mark_kernel(const u64* skey, const i64* sval, i64 E, int* dup) {
  const i64 s = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= E) return;
  const u64 k = skey[s];
  dup[sval[s]] = (s > 0 && k != kSentinel && skey[s - 1] == k) ? 1 : 0;
}

// Final per-edit status (first failing check) -> first error in edit order;
// valid edits emit their two directed entries (row << kb | col, weight).
__global__ void edit_emit_kernel(EditsDev d, const int* code, const int* dup, const int* post, u64* err,
                                 u64* ekey, double* eval, unsigned long long* nvalid) {
  const i64 g = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 E = d.n_add + d.n_rem + d.n_newe;
  if (g >= E) return;
  int c = code[g];
  if (c == kErrNone && dup[g]) c = kErrDuplicate;
  if (c == kErrNone && post[g]) c = kErrNewOldOnly;
  if (c != kErrNone) {
    atomicMin(err, (static_cast<u64>(g) << 8) | static_cast<u64>(c));
    ekey[2 * g] = ekey[2 * g + 1] = kSentinel;
    eval[2 * g] = eval[2 * g + 1] = 0.0;
    return;
  }
  int list;
  i64 i, j;
  double w;
  edit_at(d, g, list, i, j, w);
  ekey[2 * g] = (static_cast<u64>(i) << d.kb) | static_cast<u64>(j);
  ekey[2 * g + 1] = (static_cast<u64>(j) << d.kb) | static_cast<u64>(i);
  eval[2 * g] = eval[2 * g + 1] = w;
  atomicAdd(nvalid, 2ULL);
}

// ---- sort-free Delta assembly (the normal path) ---------------------------
// The same checks, keys and outcome as edit_check -> sort -> dup_mark ->
// edit_emit -> sort -> delta_rows, without the two radix sorts: each edit
// that passes the per-edit checks claims a slot in the buckets of its two
// rows (atomic counters), the counters are scanned into row starts, and every
// bucket entry finds its place in the row by counting the entries before it
// in (column, edit index) order. Equal columns within a row are exactly the
// duplicate pairs: the later edit is flagged (dup) and its entry becomes a
// sentinel. A row longer than kRankMaxRow makes the counting quadratic; it
// is reported through err_edit = 0 (no real error encodes as 0) and the host
// re-runs the ingestion on the sorting path.
constexpr int kRankMaxRow = 4096;

__global__ void edit_bucket_kernel(EditsDev d, int* code, int* post, int* rowcnt, int2* slot, int* mark, int stamp) {
  const i64 g = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 E = d.n_add + d.n_rem + d.n_newe;
  if (g >= E) return;
  int list;
  i64 i, j;
  double w;
  edit_at(d, g, list, i, j, w);
  const i64 n_total = d.n_old + d.S;
  int c = kErrNone, p = 0;
  if (list == 0 && w == 0.0) c = kErrZeroWeight;
  else if (list < 2 && (i < 0 || j < 0 || i >= d.n_old || j >= d.n_old)) c = kErrEditRange;
  else if (list == 2 && (i < 0 || j < 0 || i >= n_total || j >= n_total)) c = kErrNewRange;
  else if (list == 2 && w <= 0.0) c = kErrNewWeight;
  else if (i == j) c = kErrSelfLoop;
  if (list == 2 && c == kErrNone && (i > j ? i : j) < d.n_old) p = 1;
  code[g] = c;
  post[g] = p;
  if (c == kErrNone) {
    slot[g] = make_int2(atomicAdd(rowcnt + i, 1), atomicAdd(rowcnt + j, 1));
    mark[i] = stamp;
    mark[j] = stamp;
  }
}

__global__ void edit_scatter_kernel(EditsDev d, const int* code, const int2* slot, const int* rstart, int* brow,
                                    int* bcol, int* bedit) {
  const i64 g = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 E = d.n_add + d.n_rem + d.n_newe;
  if (g >= E || code[g] != kErrNone) return;
  int list;
  i64 i, j;
  double w;
  edit_at(d, g, list, i, j, w);
  const int2 s = slot[g];
  const int qi = rstart[i] + s.x, qj = rstart[j] + s.y;
  brow[qi] = static_cast<int>(i);
  bcol[qi] = static_cast<int>(j);
  bedit[qi] = static_cast<int>(g);
  brow[qj] = static_cast<int>(j);
  bcol[qj] = static_cast<int>(i);
  bedit[qj] = static_cast<int>(g);
}

// Bucket entry -> its slot in the row's column order; ekey tail past the
// entry count must hold sentinels (memset by the caller).
__global__ void delta_rank_kernel(EditsDev d, i64 n2, const int* rstart, const int* brow, const int* bcol,
                                  const int* bedit, u64* skey, double* sval, int* drow, int* dcol, int* dup,
                                  u64* err) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 n_total = d.n_old + d.S;
  if (e >= n2 || e >= rstart[n_total]) return;
  const int r = brow[e], c = bcol[e], g = bedit[e];
  const int s = rstart[r], t = rstart[r + 1];
  if (t - s > kRankMaxRow) {
    atomicMin(err, 0ULL);
    return;
  }
  int rank = 0;
  bool later = false;
  for (int q = s; q < t; ++q) {
    const int c2 = bcol[q];
    const bool before = c2 < c || (c2 == c && bedit[q] < g);
    rank += before ? 1 : 0;
    later |= c2 == c && bedit[q] < g;
  }
  int list;
  i64 i, j;
  double w;
  edit_at(d, g, list, i, j, w);
  const int pos = s + rank;
  drow[pos] = r;
  dcol[pos] = c;
  sval[pos] = later ? 0.0 : w;
  skey[pos] = later ? kSentinel : ((static_cast<u64>(r) << d.kb) | static_cast<u64>(c));
  if (later) dup[g] = 1;
}

// Final per-edit status for the sort-free path (as edit_emit, entries already placed).
__global__ void edit_status_kernel(i64 E, const int* code, const int* dup, const int* post, u64* err,
                                   unsigned long long* nvalid) {
  const i64 g = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= E) return;
  int c = code[g];
  if (c == kErrNone && dup[g]) c = kErrDuplicate;
  if (c == kErrNone && post[g]) c = kErrNewOldOnly;
  if (c != kErrNone) atomicMin(err, (static_cast<u64>(g) << 8) | static_cast<u64>(c));
  else atomicAdd(nvalid, 2ULL);
}

// Sorted entries -> row/col arrays, per-row counts, and row marks.
__global__ void delta_rows_kernel(const u64* skey, i64 n2, int* drow, int* dcol, int* rowcnt, int* mark, int stamp,
                                  int kb) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n2) return;
  const u64 k = skey[e];
  if (k == kSentinel) return;
  const int r = static_cast<int>(k >> kb), c = static_cast<int>(k & ((1ULL << kb) - 1));
  drow[e] = r;
  dcol[e] = c;
  atomicAdd(rowcnt + r, 1);
  mark[r] = stamp;
}

// ---- GraphUpdate blocks / Perturbation CSR -> Delta entries ---------------
// GraphUpdate::to_delta (graph.cpp:17-32) then from_triplets (sparse.cpp:
// 17-23): the K, G (+ mirror) and C entries in that insertion order,
// duplicates summed in insertion order (stable radix sort, sequential run
// sums), exact zeros pruned, symmetry validated.
struct BlockIn {
  const int* rp;
  const int* col;
  const double* val;
  i64 rows, cols, nnz;
  i64 row_off, col_off;
  int mirror;  // G: also emit the transposed entry
  i64 out0;    // first output slot
};

__global__ void block_check_kernel(BlockIn b, u64* err) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool bad = false;
  if (t == 0) bad = b.rp[0] != 0 || b.rp[b.rows] != b.nnz;
  if (t < b.rows) bad = bad || b.rp[t + 1] < b.rp[t];
  if (t < b.nnz) bad = bad || b.col[t] < 0 || b.col[t] >= b.cols;
  if (bad) atomicMin(err, static_cast<u64>(kErrBlockShape));
}

__global__ void block_emit_kernel(BlockIn b, int kb, u64* key, double* val) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= b.nnz) return;
  i64 lo = 0, hi = b.rows;  // row of entry e: last r with rp[r] <= e
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) >> 1;
    if (b.rp[mid] <= e) lo = mid; else hi = mid;
  }
  const u64 r = static_cast<u64>(lo + b.row_off), c = static_cast<u64>(b.col[e] + b.col_off);
  const double v = b.val[e];
  const i64 o = b.out0 + (b.mirror ? 2 * e : e);
  key[o] = (r << kb) | c;
  val[o] = v;
  if (b.mirror) {
    key[o + 1] = (c << kb) | r;
    val[o + 1] = v;
  }
}

// heads of equal-key runs take the run's sum (insertion order); keep the
// nonzero sums
__global__ void run_sum_kernel(const u64* skey, const double* sval, i64 n, int* keep, double* sum) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e > n) return;
  if (e == n) {
    keep[e] = 0;
    return;
  }
  const u64 k = skey[e];
  const bool head = e == 0 || skey[e - 1] != k;
  double s = 0.0;
  if (head) {
    s = sval[e];
    for (i64 q = e + 1; q < n && skey[q] == k; ++q) s += sval[q];
  }
  keep[e] = head && s != 0.0;
  sum[e] = s;
}

__global__ void run_compact_kernel(const u64* skey, const double* sum, const int* keep, const int* pos, i64 n,
                                   u64* okey, double* oval) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n || !keep[e]) return;
  okey[pos[e]] = skey[e];
  oval[pos[e]] = sum[e];
}

// is_symmetric (sparse.cpp:65-77): every (r, c, v) has (c, r, v) exactly
__global__ void sym_check_kernel(const u64* key, const double* val, const int* count, int kb, u64* err) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 cnt = *count;
  if (e >= cnt) return;
  const u64 k = key[e];
  const u64 mask = (1ULL << kb) - 1;
  const u64 t = ((k & mask) << kb) | (k >> kb);
  i64 lo = 0, hi = cnt;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (key[mid] < t) lo = mid + 1; else hi = mid;
  }
  if (lo >= cnt || key[lo] != t || val[lo] != val[e]) atomicMin(err, static_cast<u64>(kErrNotSymmetric));
}

__global__ void count_to_u64_kernel(const int* count, unsigned long long* out) { *out = static_cast<unsigned long long>(*count); }

__global__ void mark_range_kernel(int* mark, i64 lo, i64 hi, int stamp) {
  const i64 r = lo + static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < hi) mark[r] = stamp;
}

// ---- apply_update merge -------------------------------------------------
// Pass 1 (per Delta entry): locate in A's row, classify, count, check.
__global__ void merge_classify_kernel(const u64* skey, const double* sval, i64 n2, const int* arp, const int* acol,
                                      const double* aval, i64 n_old, int* lb, int* flag, double* newv, int* contrib,
                                      int* rowcnt, u64* err, int kb) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n2) return;
  const u64 k = skey[e];
  if (k == kSentinel) {  // inert in the merge: never counted, never a hit
    contrib[e] = 0;
    lb[e] = 0x3fffffff;
    flag[e] = 0;
    newv[e] = 0.0;
    return;
  }
  const int r = static_cast<int>(k >> kb), c = static_cast<int>(k & ((1ULL << kb) - 1));
  const double dv = sval[e];
  int s = 0, len = 0;
  if (r < n_old) {
    s = arp[r];
    len = arp[r + 1] - s;
  }
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (acol[s + mid] < c) lo = mid + 1; else hi = mid;
  }
  const bool found = lo < len && acol[s + lo] == c;
  const double sum = found ? aval[s + lo] + dv : 0.0 + dv;
  if (sum < -1e-12)
    atomicMin(err, (static_cast<u64>(r) << 32) | (static_cast<u64>(c) << 1) | (found ? 1ULL : 0ULL));
  const bool prune = found && sum == 0.0;
  const int ct = found ? (prune ? -1 : 0) : 1;
  lb[e] = lo;
  flag[e] = (found ? 1 : 0) | (prune ? 2 : 0);
  newv[e] = sum;
  contrib[e] = ct;
  if (ct) atomicAdd(rowcnt + r, ct);
}

__global__ void row_len_kernel(const int* arp, i64 n_old, i64 n_total, int* rowcnt) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > n_total) return;
  rowcnt[r] = (r < n_old) ? arp[r + 1] - arp[r] : 0;
}

// Pass 2a: A's entries to their new positions. Work is split into fixed
// chunks of A's nonzeros (one warp per kMergeChunk entries), so hub rows with
// tens of thousands of entries are spread over many warps. A warp loads the
// metadata of 32 consecutive rows at once (row starts, shifts, P marks) into
// lanes; entries of untouched rows are then copied 32 at a time, each lane
// finding its entry's row by a 5-step shuffle search (no dependent memory
// loads), and rows of P are merged with a 32-wide window of the (short,
// sorted) Delta row broadcast by shuffles and advanced monotonically.
constexpr int kMergeChunk = 1024;

__device__ __forceinline__ void merge_p_segment(i64 pos, i64 seg_end, int s, int o, int ds, int dn, int lane,
                                                const int* __restrict__ acol, const double* __restrict__ aval,
                                                const int* __restrict__ dcol, const int* __restrict__ flag,
                                                const double* __restrict__ newv, const int* __restrict__ prefix,
                                                int* __restrict__ ncol, double* __restrict__ nval) {
  const int p0 = prefix[ds];
  const int cfirst = acol[pos];
  int a0 = 0, a1 = dn;  // Delta entries with column below the segment's first column
  while (a0 < a1) {
    const int mid = (a0 + a1) >> 1;
    if (dcol[ds + mid] < cfirst) a0 = mid + 1; else a1 = mid;
  }
  int dbase = a0;
  for (i64 base = pos; base < seg_end; base += 32) {
    const i64 q = base + lane;
    const bool valid = q < seg_end;
    const int c = valid ? acol[q] : 0x7fffffff;
    const int last = static_cast<int>(min(static_cast<i64>(31), seg_end - base - 1));
    const int cmax = __shfl_sync(0xffffffffu, c, last);
    int cnt = dbase, hit = -1;
    for (int w0 = dbase; w0 < dn; w0 += 32) {
      const int dc = w0 + lane < dn ? dcol[ds + w0 + lane] : 0x7fffffff;
      if (__shfl_sync(0xffffffffu, dc, 0) > cmax) break;  // window entirely past the chunk
      for (int j = 0; j < 32; ++j) {
        const int dj = __shfl_sync(0xffffffffu, dc, j);
        cnt += dj < c ? 1 : 0;
        if (dj == c) hit = w0 + j;
      }
      if (__shfl_sync(0xffffffffu, dc, 31) >= cmax) break;
    }
    dbase = __shfl_sync(0xffffffffu, cnt, last);
    if (!valid) continue;
    if (hit >= 0 && (flag[ds + hit] & 2)) continue;  // cancelled to exactly zero: pruned
    const int out = o + static_cast<int>(q - s) + (prefix[ds + cnt] - p0);
    ncol[out] = c;
    nval[out] = hit >= 0 ? newv[ds + hit] : aval[q];
  }
}

// Rows of P with at most 31 Delta entries (nearly all): the row's Delta
// entries live one per lane (lb = insertion position in the old row from
// merge_classify, found/pruned flags, new value, running size change), so an
// old entry j's output slot is o + j + shift(#entries with lb + found <= j)
// with no dependent global loads in the loop; only the entries that land in
// the current 32-entry window are walked.
__device__ __forceinline__ void merge_p_segment_small(i64 pos, i64 seg_end, int s, int o, int ds, int dn, int lane,
                                                      const int* __restrict__ acol, const double* __restrict__ aval,
                                                      const int* __restrict__ lb, const int* __restrict__ flag,
                                                      const double* __restrict__ newv,
                                                      const int* __restrict__ prefix, int* __restrict__ ncol,
                                                      double* __restrict__ nval) {
  const int p0 = prefix[ds];
  int key = 0x7fffffff, lbv = -1, fl = 0, pre = 0;
  double nv = 0.0;
  if (lane < dn) {
    fl = flag[ds + lane];
    lbv = lb[ds + lane];
    key = lbv + (fl & 1);
    nv = newv[ds + lane];
  }
  if (lane <= dn) pre = prefix[ds + lane] - p0;
  // four 32-entry windows per pass, all loads issued before any use (in-order
  // issue would otherwise leave one load in flight per warp)
  for (i64 base = pos; base < seg_end; base += 128) {
    int cv[4];
    double vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const i64 q = base + 32 * u + lane;
      cv[u] = q < seg_end ? acol[q] : 0;
      vv[u] = q < seg_end ? aval[q] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const i64 wb = base + 32 * u;
      if (wb >= seg_end) break;
      const i64 q = wb + lane;
      const bool valid = q < seg_end;
      const int j0 = static_cast<int>(wb - s), j = j0 + lane;
      int cnt = __popc(__ballot_sync(0xffffffffu, lane < dn && key < j0));
      unsigned inr = __ballot_sync(0xffffffffu, lane < dn && ((key >= j0 && key <= j0 + 31) ||
                                                                ((fl & 1) && lbv >= j0 && lbv <= j0 + 31)));
      int hit = -1;
      while (inr) {
        const int k = __ffs(inr) - 1;
        inr &= inr - 1;
        const int kk = __shfl_sync(0xffffffffu, key, k);
        const int lk = __shfl_sync(0xffffffffu, lbv, k);
        const int fk = __shfl_sync(0xffffffffu, fl, k);
        if (kk >= j0 && kk <= j) ++cnt;
        if ((fk & 1) && lk == j) hit = k;
      }
      const int shift = __shfl_sync(0xffffffffu, pre, cnt);
      const double hv = __shfl_sync(0xffffffffu, nv, hit < 0 ? 0 : hit);
      const int hf = __shfl_sync(0xffffffffu, fl, hit < 0 ? 0 : hit);
      if (!valid || (hit >= 0 && (hf & 2))) continue;  // pruned: cancelled to exactly zero
      const int out = o + j + shift;
      ncol[out] = cv[u];
      nval[out] = hit >= 0 ? hv : vv[u];
    }
  }
}

__global__ void __launch_bounds__(256) merge_chunks_kernel(const int* __restrict__ arp, const int* __restrict__ acol,
                                                           const double* __restrict__ aval, i64 n_old,
                                                           const int* __restrict__ mark, int stamp,
                                                           const int* __restrict__ drp, const int* __restrict__ dcol,
                                                           const int* __restrict__ lb, const int* __restrict__ flag,
                                                           const double* __restrict__ newv,
                                                           const int* __restrict__ prefix,
                                                           const int* __restrict__ nrp, int* __restrict__ ncol,
                                                           double* __restrict__ nval) {
  const i64 w = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const i64 nnz = arp[n_old];
  const i64 e0 = w * kMergeChunk;
  if (e0 >= nnz) return;
  const i64 e1 = min(nnz, e0 + kMergeChunk);
  i64 lo = 0, hi = n_old - 1;  // row holding entry e0
  while (lo < hi) {
    const i64 mid = (lo + hi + 1) >> 1;
    if (arp[mid] <= e0) lo = mid; else hi = mid - 1;
  }
  i64 r = lo, pos = e0;
  while (pos < e1) {
    // metadata of rows r .. r + 31 (one per lane)
    const i64 rr = r + lane;
    const bool in = rr < n_old;
    const int rs = in ? arp[rr] : static_cast<int>(nnz);
    const int re = in ? arp[rr + 1] : static_cast<int>(nnz);
    const int o = in ? nrp[rr] : 0;
    const bool pm = in && mark[rr] == stamp;
    const i64 gend = min(static_cast<i64>(__shfl_sync(0xffffffffu, re, 31)), e1);
    // untouched rows: entry-parallel shifted copy, four windows per pass with
    // every load issued first
    for (i64 base = pos; base < gend; base += 128) {
      int cv[4];
      double vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const i64 q = base + 32 * u + lane;
        cv[u] = q < gend ? acol[q] : 0;
        vv[u] = q < gend ? aval[q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const i64 q = base + 32 * u + lane;
        int idx = 0;  // last lane whose row starts at or before q
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
          const int cand = idx + st;
          const int rsc = __shfl_sync(0xffffffffu, rs, cand);
          if (rsc <= q) idx = cand;
        }
        const int rs_i = __shfl_sync(0xffffffffu, rs, idx);
        const int o_i = __shfl_sync(0xffffffffu, o, idx);
        const bool p_i = __shfl_sync(0xffffffffu, pm ? 1 : 0, idx);
        if (q < gend && !p_i) {
          const i64 dst = o_i + (q - rs_i);
          ncol[dst] = cv[u];
          nval[dst] = vv[u];
        }
      }
    }
    // rows of P overlapping [pos, gend)
    unsigned todo = __ballot_sync(0xffffffffu, pm && re > pos && rs < gend);
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      const int s_l = __shfl_sync(0xffffffffu, rs, l);
      const int e_l = __shfl_sync(0xffffffffu, re, l);
      const int o_l = __shfl_sync(0xffffffffu, o, l);
      const i64 row = r + l;
      const int ds = drp[row], dn = drp[row + 1] - ds;
      if (dn < 32)
        merge_p_segment_small(max(pos, static_cast<i64>(s_l)), min(static_cast<i64>(e_l), gend), s_l, o_l, ds, dn,
                              lane, acol, aval, lb, flag, newv, prefix, ncol, nval);
      else
        merge_p_segment(max(pos, static_cast<i64>(s_l)), min(static_cast<i64>(e_l), gend), s_l, o_l, ds, dn, lane,
                        acol, aval, dcol, flag, newv, prefix, ncol, nval);
    }
    // next group starts at the row holding gend
    if (gend >= e1) break;
    const unsigned before = __ballot_sync(0xffffffffu, rs <= gend);
    r += 31 - __clz(before);
    pos = gend;
  }
}

// Pass 2a, run form: between two rows of P every row keeps its length, so a
// maximal run of untouched rows moves as one block by a constant shift
// (new start - old start). Work is split along the merge path of (rows,
// entries): warp w takes diagonal units [w kRunDiag, (w + 1) kRunDiag) of the
// walk that visits each row's entries then its end, so a warp covers at most
// kRunDiag rows plus entries (hub rows and long runs of tiny rows alike). Its
// first row comes from chunk_rows_kernel (no search); it loads the metadata
// of 32 rows at a time, copies each untouched run with a plain strided loop
// (32-bit indices, four 32-entry windows in flight) and walks the rows of P
// over their Delta entries (merge_p_walk).
constexpr int kRunDiag = 1024;

__device__ __forceinline__ void merge_copy_run(int a0, int a1, int shift, int lane, const int* __restrict__ acol,
                                               const double* __restrict__ aval, int* __restrict__ ncol,
                                               double* __restrict__ nval) {
  for (int q = a0 + lane; q < a1; q += 128) {
    int cv[4];
    double vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int qq = q + 32 * u;
      cv[u] = qq < a1 ? acol[qq] : 0;
      vv[u] = qq < a1 ? aval[qq] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int qq = q + 32 * u;
      if (qq < a1) {
        ncol[qq + shift] = cv[u];
        nval[qq + shift] = vv[u];
      }
    }
  }
}

__device__ __forceinline__ void merge_p_walk(int jpos, int jend, int s, int o, int ds, int dn, int lane,
                                             const int* __restrict__ acol, const double* __restrict__ aval,
                                             const int* __restrict__ lb, const int* __restrict__ flag,
                                             const double* __restrict__ newv, const int* __restrict__ prefix,
                                             int* __restrict__ ncol, double* __restrict__ nval) {
  const int p0 = prefix[ds];
  int t0 = 0, hi = dn;  // first event at or after jpos
  while (t0 < hi) {
    const int mid = (t0 + hi) >> 1;
    if (lb[ds + mid] < jpos) t0 = mid + 1; else hi = mid;
  }
  int S = prefix[ds + t0] - p0;  // size change of the events before t0
  int cur = jpos;
  for (int tb = t0; tb < dn; tb += 32) {
    int lbv = 0x7fffffff, fl = 0, pn = 0;
    double nv = 0.0;
    if (tb + lane < dn) {
      lbv = lb[ds + tb + lane];
      fl = flag[ds + tb + lane];
      nv = newv[ds + tb + lane];
      pn = prefix[ds + tb + lane + 1] - p0;
    }
    const int cnt = min(32, dn - tb);
    for (int k = 0; k < cnt; ++k) {
      const int target = __shfl_sync(0xffffffffu, lbv, k);
      const int f = __shfl_sync(0xffffffffu, fl, k);
      const double v = __shfl_sync(0xffffffffu, nv, k);
      const int snext = __shfl_sync(0xffffffffu, pn, k);
      const int stop = min(target, jend);
      if (stop > cur) merge_copy_run(s + cur, s + stop, o - s + S, lane, acol, aval, ncol, nval);
      if (target >= jend) return;
      if (f & 1) {  // the event's own old entry: updated in place, or pruned
        if (!(f & 2) && lane == 0 && target >= jpos) {
          ncol[o + target + S] = acol[s + target];
          nval[o + target + S] = v;
        }
        cur = max(cur, target + 1);
      } else {
        cur = max(cur, target);
      }
      S = snext;
    }
  }
  if (jend > cur) merge_copy_run(s + cur, s + jend, o - s + S, lane, acol, aval, ncol, nval);
}

__global__ void chunk_rows_kernel(const int* arp, int n_old, int* map) {
  const int r = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_old) return;
  const i64 d0 = static_cast<i64>(r) + arp[r], d1 = static_cast<i64>(r) + arp[r + 1];  // entries, then the row end
  for (i64 k = (d0 + kRunDiag - 1) / kRunDiag; k * kRunDiag <= d1; ++k) map[k] = r;
}

__device__ __forceinline__ int run_entry_start(const int* arp, const int* map, int w) {
  const int r = map[w];
  return static_cast<int>(min(static_cast<i64>(w) * kRunDiag - r, static_cast<i64>(arp[r + 1])));
}

__global__ void __launch_bounds__(256) merge_runs_kernel(const int* __restrict__ arp, const int* __restrict__ acol,
                                                         const double* __restrict__ aval, int n_old, int nnz,
                                                         const int* __restrict__ map, const int* __restrict__ mark,
                                                         int stamp, const int* __restrict__ drp,
                                                         const int* __restrict__ dcol, const int* __restrict__ lb,
                                                         const int* __restrict__ flag,
                                                         const double* __restrict__ newv,
                                                         const int* __restrict__ prefix, const int* __restrict__ nrp,
                                                         int* __restrict__ ncol, double* __restrict__ nval, int mode) {
  const int w = static_cast<int>((static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int nw = static_cast<int>((static_cast<i64>(n_old) + nnz + kRunDiag - 1) / kRunDiag);
  if (w >= nw) return;
  const int e0 = run_entry_start(arp, map, w);
  const int e1 = w + 1 < nw ? run_entry_start(arp, map, w + 1) : nnz;
  if (e0 >= e1) return;
  int r = map[w], pos = e0;
  while (pos < e1) {
    const int rr = r + lane;
    const bool in = rr < n_old;
    const int rs = in ? arp[rr] : nnz;
    const int re = in ? arp[rr + 1] : nnz;
    const int o = in ? nrp[rr] : 0;
    const bool pm = in && mark[rr] == stamp;
    const int gend = min(__shfl_sync(0xffffffffu, re, 31), e1);
    const bool live = in && re > pos && rs < gend;
    // untouched runs: maximal groups of consecutive live lanes without P
    unsigned todo = __ballot_sync(0xffffffffu, live && !pm && (mode & 1));
    while (todo) {
      const int l = __ffs(todo) - 1;
      const unsigned tail = ~(todo >> l);
      const int len = tail ? __ffs(tail) - 1 : 32 - l;
      todo &= len >= 32 ? 0u : ~(((1u << len) - 1u) << l);
      const int rs_l = __shfl_sync(0xffffffffu, rs, l);
      const int shift = __shfl_sync(0xffffffffu, o, l) - rs_l;
      const int sb = max(pos, rs_l);
      const int se = min(gend, __shfl_sync(0xffffffffu, re, l + len - 1));
      for (int q = sb + lane; q < se; q += 128) {
        int cv[4];
        double vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int qq = q + 32 * u;
          cv[u] = qq < se ? acol[qq] : 0;
          vv[u] = qq < se ? aval[qq] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int qq = q + 32 * u;
          if (qq < se) {
            ncol[qq + shift] = cv[u];
            nval[qq + shift] = vv[u];
          }
        }
      }
    }
    // rows of P overlapping [pos, gend)
    unsigned ptodo = __ballot_sync(0xffffffffu, live && pm && (mode & 2));
    while (ptodo) {
      const int l = __ffs(ptodo) - 1;
      ptodo &= ptodo - 1;
      const int s_l = __shfl_sync(0xffffffffu, rs, l);
      const int e_l = __shfl_sync(0xffffffffu, re, l);
      const int o_l = __shfl_sync(0xffffffffu, o, l);
      const int row = r + l;
      const int ds = drp[row], dn = drp[row + 1] - ds;
      merge_p_walk(max(pos, s_l) - s_l, min(e_l, gend) - s_l, s_l, o_l, ds, dn, lane, acol, aval, lb, flag, newv,
                   prefix, ncol, nval);
    }
    if (gend >= e1) break;
    const unsigned before = __ballot_sync(0xffffffffu, rs <= gend);
    r += 31 - __clz(before);
    pos = gend;
  }
}

// Pass 2b: Delta entries with no stored counterpart in A.
__global__ void merge_insert_kernel(i64 n2, const int* drow, const int* dcol, const u64* skey, const int* lb,
                                    const int* flag, const double* newv, const int* prefix, const int* drp,
                                    const int* nrp, int* ncol, double* nval) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n2 || skey[e] == kSentinel || (flag[e] & 1)) return;
  const int r = drow[e];
  const int pos = nrp[r] + lb[e] + (prefix[e] - prefix[drp[r]]);
  ncol[pos] = dcol[e];
  nval[pos] = newv[e];
}

// ---- Laplacian operators -------------------------------------------------
// Weighted degrees as the reference computes them: A * ones, row sums in
// column order (sparse.cpp:97-99).
__global__ void degrees_kernel(const int* rp, const double* val, i64 n, double* deg) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (int e = rp[r]; e < rp[r + 1]; ++e) s += val[e];
  deg[r] = s;
}

__global__ void max_reduce_kernel(const double* x, i64 n, double* out) {
  __shared__ double sh[1024];
  double m = 0.0;  // degrees are >= 0; an empty graph has d_max = 0 (laplacian_track.cpp:37)
  for (i64 i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, x[i]);
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

// shift_for (laplacian_track.cpp:35-39): normalized -> 2; combinatorial -> max(alpha, 2 d_max)
__global__ void shift_kernel(int normalized, const double* dmax, const double* alpha_old, double* alpha_new) {
  alpha_new[0] = normalized ? 2.0 : fmax(alpha_old[0], 2.0 * dmax[0]);
}

__device__ __forceinline__ double lap_offdiag(int normalized, const double* scale, i64 r, int c, double a) {
  return normalized ? __dmul_rn(__dmul_rn(scale[r], scale[c]), a) : a;
}
__device__ __forceinline__ double lap_diag(int normalized, const double* deg, const double* alpha, i64 r) {
  return normalized ? (deg[r] > 0.0 ? 1.0 : 2.0) : __dsub_rn(alpha[0], deg[r]);
}

__global__ void scale_kernel(const double* deg, i64 n, double* scale) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n) scale[r] = deg[r] > 0.0 ? 1.0 / sqrt(deg[r]) : 0.0;
}

// T rows: A's pattern plus the diagonal, exact zeros pruned (graph.cpp:139-150).
__global__ void lap_count_kernel(const int* rp, const int* col, const double* val, i64 n, int normalized,
                                 const double* deg, const double* scale, const double* alpha, int* cnt) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > n) return;
  if (r == n) {
    cnt[r] = 0;
    return;
  }
  int c = lap_diag(normalized, deg, alpha, r) != 0.0 ? 1 : 0;
  for (int e = rp[r]; e < rp[r + 1]; ++e) c += lap_offdiag(normalized, scale, r, col[e], val[e]) != 0.0 ? 1 : 0;
  cnt[r] = c;
}

__global__ void lap_write_kernel(const int* rp, const int* col, const double* val, i64 n, int normalized,
                                 const double* deg, const double* scale, const double* alpha, const int* trp,
                                 int* tcol, double* tval) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int o = trp[r];
  const double dg = lap_diag(normalized, deg, alpha, r);
  bool diag_done = false;
  for (int e = rp[r]; e < rp[r + 1]; ++e) {
    const int c = col[e];
    if (!diag_done && c > r) {
      if (dg != 0.0) { tcol[o] = static_cast<int>(r); tval[o++] = dg; }
      diag_done = true;
    }
    const double v = lap_offdiag(normalized, scale, r, c, val[e]);
    if (v != 0.0) { tcol[o] = c; tval[o++] = v; }
  }
  if (!diag_done && dg != 0.0) { tcol[o] = static_cast<int>(r); tval[o] = dg; }
}

// Delta_T = T_next - pad(T_old): per-row sorted difference, exact zeros pruned
// (laplacian_track.cpp:57-58). write == 0 counts, write == 1 emits.
__global__ void lap_diff_kernel(const int* orp, const int* ocol, const double* oval, i64 n_old, const int* nrp,
                                const int* ncol, const double* nval, i64 n, const int* drp, int* cnt, int* dcol,
                                double* dval, int write) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > n) return;
  if (r == n) {
    if (!write) cnt[r] = 0;
    return;
  }
  int i = r < n_old ? orp[r] : 0, ie = r < n_old ? orp[r + 1] : 0;
  int j = nrp[r], je = nrp[r + 1];
  int c = 0, o = write ? drp[r] : 0;
  while (i < ie || j < je) {
    const int ci = i < ie ? ocol[i] : 0x7fffffff, cj = j < je ? ncol[j] : 0x7fffffff;
    double v;
    int cc;
    if (ci == cj) { v = __dsub_rn(nval[j], oval[i]); cc = ci; ++i; ++j; }
    else if (cj < ci) { v = __dsub_rn(nval[j], 0.0); cc = cj; ++j; }
    else { v = __dsub_rn(0.0, oval[i]); cc = ci; ++i; }
    if (v != 0.0) {
      if (write) { dcol[o] = cc; dval[o] = v; ++o; }
      ++c;
    }
  }
  if (!write) cnt[r] = c;
}

// Row marks from a CSR's nonempty rows (Delta_T pattern).
__global__ void mark_nonempty_kernel(const int* rp, i64 n, int* mark, int stamp) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n && rp[r + 1] > rp[r]) mark[r] = stamp;
}

// ---- compressed row set P -------------------------------------------------
__global__ void flag_kernel(const int* mark, int stamp, i64 n, int* flag) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r <= n) flag[r] = (r < n && mark[r] == stamp) ? 1 : 0;
}

__global__ void scatter_p_kernel(const int* flag, const int* pos, i64 n, int* P, int* posmap) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n && flag[r]) {
    P[pos[r]] = static_cast<int>(r);
    posmap[r] = pos[r];
  }
}

// Local (compressed) CSR of Delta over P: rows gathered, columns renumbered.
__global__ void compress_rowptr_kernel(const int* grp, const int* P, i64 p, int* lrp, int nnz) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < p) lrp[t] = grp[P[t]];
  if (t == p) lrp[t] = nnz;
}

__global__ void compress_cols_kernel(const int* gcol, i64 nnz, const int* posmap, int* lcol) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < nnz) lcol[e] = posmap[gcol[e]];
}

}  // namespace stg
