// CSR x tall-skinny dense products for the perturbation Delta (HBM-bound).
//
// One warp per CSR row segment; lane l owns columns l, l+32, ... of the dense
// block, so each nonzero costs one coalesced read of a dense row. The (col, val) pairs of
// a row are fetched 32 at a time and broadcast with shuffles. Accumulation is
// sequential over the row's nonzeros in column order with separate multiply
// and add roundings, which reproduces Eigen's row-major sparse*dense product
// (proj/src/sparse.cpp:84-87) bit for bit.
#pragma once

#include <cstdlib>

#include "common.cuh"

namespace stg {

inline bool getenv_flag(const char* name) {  // development A/B switches, read once
  const char* v = std::getenv(name);
  return v && v[0] && v[0] != '0';
}

struct SpmmArgs {
  i64 rows;             // output rows
  i64 row_off;          // CSR row of output row 0
  const int* rowptr;    // local CSR (indices into col/val)
  const int* col;       // local column indices (rows of X)
  const double* val;
  int col_lo;           // only nonzeros with col >= col_lo (trailing-column view); 0 = all
  const double* X;
  int ldx;
  int m;                // dense columns
  double* Y;
  int ldy;
};

// Rows are cut into segments of at most kSegNnz nonzeros, one warp per
// segment, so a hub row (hundreds of Delta entries) no longer serialises one
// warp behind a chain of dependent gathers. A row of one segment is summed as
// above and written directly; the segments of a longer row write partial
// sums, which spmm_fixup_kernel adds in segment order (deterministic; the
// association differs from Eigen's only within those rows, at rounding level).
constexpr int kSegNnz = 32;    // rows up to this length: the row-group kernels
constexpr int kChunk = 128;    // rows + short-row entries per chunk of spmm_chunk_kernel
constexpr int kLongSeg = 32;   // longer rows: one warp per 32-entry segment, partials
                               // summed by the fix-up (512-entry segments made one
                               // warp walk a hub row serially: 2x slower at config 3)

struct SpmmPlan {
  const int* vrow;        // virtual row (segment) -> row
  const int* vstart;      // row -> first segment; vstart[rows] = segment count
  const int* sstart;      // row -> first scratch slot (rows of more than one segment)
  const int* split_rows;  // rows of more than one segment (any order)
  const int* nsplit;
  double* scratch;        // [slot][lds]
  int lds;
  int* segcnt;            // per long row (at its first scratch slot) and column slab: segments arrived
  const int* sptr;        // row -> short-row entries before it (chunk kernel)
  const int* crow;        // chunk -> first row (chunk kernel)
  int nch;                // chunks
};

template <int T>  // columns per lane = T (m <= 32 T)
__global__ void __launch_bounds__(256) spmm_kernel(SpmmArgs a, SpmmPlan pl) {
  const i64 v = static_cast<i64>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= pl.vstart[a.rows]) return;
  const int r = pl.vrow[v];
  const int s = static_cast<int>(v - pl.vstart[r]);
  const int nseg = pl.vstart[r + 1] - pl.vstart[r];
  const i64 gr = r + a.row_off;
  const int seg0 = a.rowptr[gr] + s * kLongSeg;
  const int seg_end = min(seg0 + kLongSeg, a.rowptr[gr + 1]);
  double acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t] = 0.0;
  for (int rs = seg0; rs < seg_end; rs += 32) {  // 32-entry windows, sums in column order
  const int cnt = min(32, seg_end - rs);
  int c_l = 0;
  double v_l = 0.0;
  if (lane < cnt) {
    c_l = a.col[rs + lane];
    v_l = a.val[rs + lane];
  }
  // trailing-column view: the (sorted) columns below col_lo are a prefix
  int q = a.col_lo > 0 ? __popc(__ballot_sync(0xffffffffu, lane < cnt && c_l < a.col_lo)) : 0;
  // four nonzeros per pass: their row loads are issued together, the sums
  // still run in column order
  for (; q + 4 <= cnt; q += 4) {
    double xv[4][T], vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = __shfl_sync(0xffffffffu, c_l, q + u);
      vv[u] = __shfl_sync(0xffffffffu, v_l, q + u);
      const double* xr = a.X + static_cast<i64>(c) * a.ldx;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int cc = lane + 32 * t;
        xv[u][t] = cc < a.m ? __ldg(xr + cc) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] = __dadd_rn(acc[t], __dmul_rn(vv[u], xv[u][t]));
  }
  for (; q < cnt; ++q) {
    const int c = __shfl_sync(0xffffffffu, c_l, q);
    const double vq = __shfl_sync(0xffffffffu, v_l, q);
    const double* xr = a.X + static_cast<i64>(c) * a.ldx;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int cc = lane + 32 * t;
      if (cc < a.m) acc[t] = __dadd_rn(acc[t], __dmul_rn(vq, __ldg(xr + cc)));
    }
  }
  }
  double* yr = nseg == 1 ? a.Y + static_cast<i64>(r) * a.ldy
                         : pl.scratch + static_cast<i64>(pl.sstart[r] + s) * pl.lds;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int cc = lane + 32 * t;
    if (cc < a.m) yr[cc] = acc[t];
  }
}

// Rows of at most kSegNnz nonzeros, kGroupRows consecutive rows per warp:
// the group's row pointers come in one load and its (col, val) pairs in one
// 32-wide window, so the per-row dependent chain is only the gather of X rows
// (issued four nonzeros at a time). Each row is summed exactly as above
// (column order, separate multiply and add: bit-identical). With VEC a warp
// covers a 64-column slab, lane l owning columns 2l, 2l+1 (128-bit loads and
// stores; X, Y 16-byte aligned, even leading dimensions and m); otherwise a
// 32-column slab, one column per lane. blockIdx.y = column slab. Longer rows
// are skipped here (spmm_kernel over the long-row plan writes them).
constexpr int kGroupRows = 8;

template <bool VEC>
__device__ __forceinline__ void spmm_load_x(const double* xr, int lane, bool on, double& x0, double& x1) {
  if (VEC) {
    const double2 t = on ? __ldg(reinterpret_cast<const double2*>(xr) + lane) : make_double2(0.0, 0.0);
    x0 = t.x;
    x1 = t.y;
  } else {
    x0 = on ? __ldg(xr + lane) : 0.0;
    x1 = 0.0;
  }
}

template <bool VEC>
__device__ __forceinline__ void spmm_store_row(double* yr, int lane, bool on, double a0, double a1) {
  if (!on) return;
  if (VEC) reinterpret_cast<double2*>(yr)[lane] = make_double2(a0, a1);
  else yr[lane] = a0;
}

constexpr int kGroupWarps = 4;   // warps per CTA of spmm_group_kernel
constexpr int kStageRows = 16;   // X rows staged per warp and batch

template <bool VEC>
constexpr size_t spmm_group_smem() {
  return sizeof(double) * kGroupWarps * kStageRows * (VEC ? 64 : 32);
}

template <bool VEC>
__global__ void __launch_bounds__(32 * kGroupWarps) spmm_group_kernel(SpmmArgs a) {
  constexpr int W = VEC ? 64 : 32;
  extern __shared__ __align__(16) double spmm_sx[];
  const int wib = threadIdx.x >> 5;
  const i64 g = static_cast<i64>(blockIdx.x) * kGroupWarps + wib;
  const int lane = threadIdx.x & 31;
  const i64 r0 = g * kGroupRows;
  if (r0 >= a.rows) return;
  const int nr = static_cast<int>(min(static_cast<i64>(kGroupRows), a.rows - r0));
  const int c0 = static_cast<int>(blockIdx.y) * W;
  const int m = min(W, a.m - c0);
  const int* rp = a.rowptr + a.row_off + r0;
  const int rp_l = lane <= nr ? rp[lane] : 0;
  const int gend = __shfl_sync(0xffffffffu, rp_l, nr);
  int base = __shfl_sync(0xffffffffu, rp_l, 0);
  int c_l = 0;
  double v_l = 0.0;
  if (base + lane < gend) {
    c_l = a.col[base + lane];
    v_l = a.val[base + lane];
  }
  const double* X = a.X + c0;
  double* Y = a.Y + c0;
  const bool on = VEC ? 2 * lane < m : lane < m;
  if (gend - base <= 32) {
    // The group's entries fit one window and no row is long. The X rows of
    // its active entries (col >= col_lo) are staged into shared memory with
    // cp.async, up to kStageRows per batch, all in flight at once; the rows
    // then sum their own entries in column order (bit-identical to above).
    double* sx = spmm_sx + wib * kStageRows * W;
    int row_l = 0;  // row (within the group) of entry `lane`
#pragma unroll
    for (int i = 1; i < kGroupRows; ++i) {
      const int ri = __shfl_sync(0xffffffffu, rp_l, i);
      row_l += (i < nr && base + lane >= ri) ? 1 : 0;
    }
    unsigned act = __ballot_sync(0xffffffffu, base + lane < gend && c_l >= a.col_lo);
    bool has = false;  // rows without an active entry are zero rows
    const int rp_next = __shfl_down_sync(0xffffffffu, rp_l, 1);
    if (lane < nr) {
      const int s = rp_l - base, e = rp_next - base;
      const unsigned hi = e >= 32 ? 0xffffffffu : ((1u << e) - 1u);
      const unsigned lo = s >= 32 ? 0xffffffffu : ((1u << s) - 1u);
      has = (act & hi & ~lo) != 0;
    }
    unsigned empty = __ballot_sync(0xffffffffu, lane < nr && !has);
    while (empty) {
      const int r = __ffs(empty) - 1;
      empty &= empty - 1;
      spmm_store_row<VEC>(Y + (r0 + r) * static_cast<i64>(a.ldy), lane, on, 0.0, 0.0);
    }
    int cur = -1;
    double acc0 = 0.0, acc1 = 0.0;
    while (act) {
      unsigned rest = act;
      int ns = 0;
      for (; ns < kStageRows && rest; ++ns) {
        const int j = __ffs(rest) - 1;
        rest &= rest - 1;
        const int c = __shfl_sync(0xffffffffu, c_l, j);
        const double* xr = X + static_cast<i64>(c) * a.ldx;
        if (on) {
          if (VEC) cp_async16(sx + ns * W + 2 * lane, xr + 2 * lane);
          else cp_async8(sx + ns * W + lane, xr + lane);
        }
      }
      cp_async_commit();
      unsigned batch = act & ~rest;
      act = rest;
      cp_async_wait<0>();
      __syncwarp();
      for (int s2 = 0; s2 < ns; ++s2) {
        const int j = __ffs(batch) - 1;
        batch &= batch - 1;
        const int rw = __shfl_sync(0xffffffffu, row_l, j);
        const double vq = __shfl_sync(0xffffffffu, v_l, j);
        if (rw != cur) {
          if (cur >= 0) spmm_store_row<VEC>(Y + (r0 + cur) * static_cast<i64>(a.ldy), lane, on, acc0, acc1);
          cur = rw;
          acc0 = acc1 = 0.0;
        }
        if (on) {
          if (VEC) {
            const double2 t = *reinterpret_cast<const double2*>(sx + s2 * W + 2 * lane);
            acc0 = __dadd_rn(acc0, __dmul_rn(vq, t.x));
            acc1 = __dadd_rn(acc1, __dmul_rn(vq, t.y));
          } else {
            acc0 = __dadd_rn(acc0, __dmul_rn(vq, sx[s2 * W + lane]));
          }
        }
      }
      __syncwarp();  // the next batch overwrites the staging rows
    }
    if (cur >= 0) spmm_store_row<VEC>(Y + (r0 + cur) * static_cast<i64>(a.ldy), lane, on, acc0, acc1);
    return;
  }
  // general case: row by row, the window moving with the rows
  for (int i = 0; i < nr; ++i) {
    const int s = __shfl_sync(0xffffffffu, rp_l, i), e = __shfl_sync(0xffffffffu, rp_l, i + 1);
    if (e - s > kSegNnz) continue;
    if (e > base + 32) {  // the window moves to this row (warp-uniform)
      base = s;
      c_l = 0;
      v_l = 0.0;
      if (base + lane < gend) {
        c_l = a.col[base + lane];
        v_l = a.val[base + lane];
      }
    }
    int q = s - base;
    const int qe = e - base;
    if (a.col_lo > 0) q += __popc(__ballot_sync(0xffffffffu, lane >= q && lane < qe && c_l < a.col_lo));
    double acc0 = 0.0, acc1 = 0.0;
    for (; q + 4 <= qe; q += 4) {
      double x0[4], x1[4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = __shfl_sync(0xffffffffu, c_l, q + u);
        vv[u] = __shfl_sync(0xffffffffu, v_l, q + u);
        spmm_load_x<VEC>(X + static_cast<i64>(c) * a.ldx, lane, on, x0[u], x1[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc0 = __dadd_rn(acc0, __dmul_rn(vv[u], x0[u]));
        if (VEC) acc1 = __dadd_rn(acc1, __dmul_rn(vv[u], x1[u]));
      }
    }
    for (; q < qe; ++q) {
      const int c = __shfl_sync(0xffffffffu, c_l, q);
      const double vq = __shfl_sync(0xffffffffu, v_l, q);
      double t0, t1;
      spmm_load_x<VEC>(X + static_cast<i64>(c) * a.ldx, lane, on, t0, t1);
      acc0 = __dadd_rn(acc0, __dmul_rn(vq, t0));
      if (VEC) acc1 = __dadd_rn(acc1, __dmul_rn(vq, t1));
    }
    spmm_store_row<VEC>(Y + (r0 + i) * static_cast<i64>(a.ldy), lane, on, acc0, acc1);
  }
}

// Rows of at most kSegNnz nonzeros, kGroupRows consecutive rows per warp, ALL
// dense columns per warp: lane l owns columns 64 t + 2l, 2l + 1 of every
// 64-column slab t < T (128-bit loads and stores), so the group's index work
// (row pointers, the (col, val) window, row of each entry) is done once for
// all m columns, and each entry issues T loads. Entries are consumed U at a
// time with their T x 4 loads in flight together; each row is summed in
// column order with separate multiply and add roundings (bit-identical to
// spmm_kernel and to Eigen's row-major product). (U = 2 entries in flight
// when T >= 3 keeps the kernel at 2 CTAs of 8 warps per SM.) Warps walk the groups
// grid-stride and fetch the next group's header before gathering the current
// one. Longer rows are skipped (spmm_kernel over the long-row plan).
template <int T>
__global__ void __launch_bounds__(256, 2) spmm_rows_kernel(SpmmArgs a, i64 ngroups) {
  constexpr int U = T >= 3 ? 2 : 4;  // entries whose T loads are in flight together
  const int lane = threadIdx.x & 31;
  const i64 w0 = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  const int* rowp = a.rowptr + a.row_off;
  bool on[T];
#pragma unroll
  for (int t = 0; t < T; ++t) on[t] = 64 * t + 2 * lane < a.m;
  auto header = [&](i64 g, int& rp_l, int& nr) {
    const i64 r0 = g * kGroupRows;
    nr = static_cast<int>(min(static_cast<i64>(kGroupRows), a.rows - r0));
    rp_l = (g < ngroups && lane <= nr) ? __ldg(rowp + r0 + lane) : 0;
  };
  int rp_n = 0, nr_n = 0;
  if (w0 < ngroups) header(w0, rp_n, nr_n);
  for (i64 g = w0; g < ngroups; g += nw) {
    const int rp_l = rp_n, nr = nr_n;
    if (g + nw < ngroups) header(g + nw, rp_n, nr_n);  // next group's row pointers in flight
    const i64 r0 = g * kGroupRows;
    const int rp_next = __shfl_down_sync(0xffffffffu, rp_l, 1);
    double* Yg = a.Y + r0 * static_cast<i64>(a.ldy) + 2 * lane;
    auto store = [&](int r, const double (&acc)[T][2]) {
      double* yr = Yg + static_cast<i64>(r) * a.ldy;
#pragma unroll
      for (int t = 0; t < T; ++t)
        if (on[t]) *reinterpret_cast<double2*>(yr + 64 * t) = make_double2(acc[t][0], acc[t][1]);
    };
    double acc[T][2];
    const int e_l = lane < nr ? rp_next : 0;  // end of row `lane` of the group
    // rows of the group one window at a time: rows [ri, last] whose entries fit
    // 32 lanes; a row longer than kSegNnz is skipped (the long-row plan has it)
    int ri = 0;
    while (ri < nr) {
      const int wb = __shfl_sync(0xffffffffu, rp_l, ri);
      const unsigned fm = __ballot_sync(0xffffffffu, lane >= ri && lane < nr && e_l <= wb + 32);
      if (!(fm & (1u << ri))) {  // row ri is long
        ++ri;
        continue;
      }
      const int last = __ffs(~(fm >> ri)) - 1 + ri - 1;  // end of the contiguous run of fitting rows
      const int we = __shfl_sync(0xffffffffu, e_l, last);
      int c_l = 0;
      double v_l = 0.0;
      if (wb + lane < we) {
        c_l = __ldg(a.col + wb + lane);
        v_l = __ldg(a.val + wb + lane);
      }
      int row_l = -1;  // row (within the group) of entry `lane`
#pragma unroll
      for (int i = 0; i < kGroupRows; ++i) {
        const int rs = __shfl_sync(0xffffffffu, rp_l, i);
        row_l += (i < nr && wb + lane >= rs) ? 1 : 0;
      }
      const int q_end = we - wb;
      unsigned act = __ballot_sync(0xffffffffu, lane < q_end && c_l >= a.col_lo);
      // rows ri..last with no active entry are zero rows
      {
        const bool mine = lane >= ri && lane <= last;
        bool has = false;
        if (mine) {
          const int s = rp_l - wb, e = e_l - wb;
          const unsigned hi = e >= 32 ? 0xffffffffu : ((1u << e) - 1u);
          const unsigned lo = s >= 32 ? 0xffffffffu : ((1u << s) - 1u);
          has = (act & hi & ~lo) != 0;
        }
        unsigned empty = __ballot_sync(0xffffffffu, mine && !has);
        double z[T][2];
#pragma unroll
        for (int t = 0; t < T; ++t) z[t][0] = z[t][1] = 0.0;
        while (empty) {
          const int r = __ffs(empty) - 1;
          empty &= empty - 1;
          store(r, z);
        }
      }
      int cur = -1;
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t][0] = acc[t][1] = 0.0;
      while (act) {
        int jj[U], nb = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          jj[u] = act ? __ffs(act) - 1 : -1;
          if (act) {
            act &= act - 1;
            ++nb;
          }
        }
        double2 xv[U][T];
        double vv[U];
        int rw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = jj[u] < 0 ? 0 : jj[u];
          const int c = __shfl_sync(0xffffffffu, c_l, j);
          vv[u] = __shfl_sync(0xffffffffu, v_l, j);
          rw[u] = __shfl_sync(0xffffffffu, row_l, j);
          const double* xr = a.X + static_cast<i64>(c) * a.ldx + 2 * lane;
#pragma unroll
          for (int t = 0; t < T; ++t)
            xv[u][t] = (u < nb && on[t]) ? __ldg(reinterpret_cast<const double2*>(xr + 64 * t))
                                         : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u >= nb) break;
          if (rw[u] != cur) {
            if (cur >= 0) store(cur, acc);
            cur = rw[u];
#pragma unroll
            for (int t = 0; t < T; ++t) acc[t][0] = acc[t][1] = 0.0;
          }
#pragma unroll
          for (int t = 0; t < T; ++t) {
            acc[t][0] = __dadd_rn(acc[t][0], __dmul_rn(vv[u], xv[u][t].x));
            acc[t][1] = __dadd_rn(acc[t][1], __dmul_rn(vv[u], xv[u][t].y));
          }
        }
      }
      if (cur >= 0) store(cur, acc);
      ri = last + 1;
    }
  }
}

// ONE launch per product: long-row segments and short-row groups in the same
// persistent grid, the segment fix-up folded in. Lane l owns VW consecutive
// columns of every (32 VW)-column slab t < T (VW = 2: 128-bit loads/stores;
// VW = 1: 8-byte loads, so a 32-column block keeps all 32 lanes busy). Work
// items: first the long-row segments (one warp per kLongSeg entries; each
// writes its partial row to the scratch slot of the segment, then bumps the
// row's arrival counter; the warp that arrives last adds the row's partials in
// segment order (fixed order: deterministic) and writes Y, then resets the
// counter), then the groups of kGroupRows consecutive rows, whose rows of at
// most kSegNnz entries are summed in column order with separate multiply and
// add roundings (as spmm_kernel). U entries have their T loads in flight
// together; each warp prefetches the next group's row pointers.
template <int VW>
struct SpV;
template <>
struct SpV<1> {
  using T = double;
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
  static __device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
  static __device__ __forceinline__ void st(double* p, double v) { *p = v; }
  static __device__ __forceinline__ void fma(double& acc, double v, double x) { acc = __dadd_rn(acc, __dmul_rn(v, x)); }
  static __device__ __forceinline__ void add(double& acc, double x) { acc = __dadd_rn(acc, x); }
};
template <>
struct SpV<2> {
  using T = double2;
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double2 ld(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
  static __device__ __forceinline__ double2 ldcg(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
  static __device__ __forceinline__ void st(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }
  static __device__ __forceinline__ void fma(double2& acc, double v, double2 x) {
    acc.x = __dadd_rn(acc.x, __dmul_rn(v, x.x));
    acc.y = __dadd_rn(acc.y, __dmul_rn(v, x.y));
  }
  static __device__ __forceinline__ void add(double2& acc, double2 x) {
    acc.x = __dadd_rn(acc.x, x.x);
    acc.y = __dadd_rn(acc.y, x.y);
  }
};

constexpr int spmm_fused_minb(int vw, int t) { return vw * t <= 1 ? 2 : 2; }

template <int VW, int T>
__global__ void __launch_bounds__(256, spmm_fused_minb(VW, T)) spmm_fused_kernel(SpmmArgs a, SpmmPlan pl, i64 ngroups) {
  using V = SpV<VW>;
  using VT = typename V::T;
  constexpr int SW = 32 * VW;
  constexpr int U = VW * T >= 6 ? 2 : VW * T >= 3 ? 4 : VW * T == 2 ? 8 : 16;  // entries whose T loads are in flight together
  const int lane = threadIdx.x & 31;
  const i64 w0 = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  const int* rowp = a.rowptr + a.row_off;
  bool on[T];
#pragma unroll
  for (int t = 0; t < T; ++t) on[t] = SW * t + VW * lane < a.m;
  // gathers the rows of the active entries (bitmask over the 32-entry window
  // held as c_l / v_l) in order, U at a time; a change of row(entry) stores
  // the finished row through `flush`
  auto gather = [&](unsigned act, int c_l, double v_l, int row_l, VT (&acc)[T], int& cur, auto&& flush) {
    while (act) {
      int jj[U], nb = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        jj[u] = act ? __ffs(act) - 1 : 0;
        if (act) {
          act &= act - 1;
          ++nb;
        }
      }
      VT xv[U][T];
      double vv[U];
      int rw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = __shfl_sync(0xffffffffu, c_l, jj[u]);
        vv[u] = __shfl_sync(0xffffffffu, v_l, jj[u]);
        rw[u] = __shfl_sync(0xffffffffu, row_l, jj[u]);
        const double* xr = a.X + static_cast<i64>(c) * a.ldx + VW * lane;
#pragma unroll
        for (int t = 0; t < T; ++t) xv[u][t] = (u < nb && on[t]) ? V::ld(xr + SW * t) : V::zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u >= nb) break;
        if (rw[u] != cur) {
          if (cur >= 0) flush(cur, acc);
          cur = rw[u];
#pragma unroll
          for (int t = 0; t < T; ++t) acc[t] = V::zero();
        }
#pragma unroll
        for (int t = 0; t < T; ++t) V::fma(acc[t], vv[u], xv[u][t]);
      }
    }
  };
  VT acc[T];
  // ---- long-row segments (the rows of more than kSegNnz entries)
  const i64 nseg = pl.vstart[a.rows];
  i64 w = w0;
  for (; w < nseg; w += nw) {
    const int r = pl.vrow[w];
    const int vs = pl.vstart[r];
    const int s = static_cast<int>(w - vs);
    const int nsg = pl.vstart[r + 1] - vs;
    const int rs = rowp[r];
    const int seg0 = rs + s * kLongSeg;
    const int cnt = min(kLongSeg, rowp[r + 1] - seg0);
    int c_l = 0;
    double v_l = 0.0;
    if (lane < cnt) {
      c_l = __ldg(a.col + seg0 + lane);
      v_l = __ldg(a.val + seg0 + lane);
    }
    const unsigned act = __ballot_sync(0xffffffffu, lane < cnt && c_l >= a.col_lo);
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = V::zero();
    int cur = -1;
    gather(act, c_l, v_l, 0, acc, cur, [](int, const VT(&)[T]) {});
    const int slot0 = pl.sstart[r];
    double* part = pl.scratch + static_cast<i64>(slot0 + s) * pl.lds + VW * lane;
#pragma unroll
    for (int t = 0; t < T; ++t)
      if (on[t]) V::st(part + SW * t, acc[t]);
    __threadfence();
    int last = 0;
    if (lane == 0) last = atomicAdd(pl.segcnt + slot0, 1) == nsg - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {  // every partial of row r is written: add them in segment order
      __threadfence();
      const double* p0 = pl.scratch + static_cast<i64>(slot0) * pl.lds + VW * lane;
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] = V::zero();
      int q = 0;
      for (; q + 4 <= nsg; q += 4) {
        VT tv[4][T];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int t = 0; t < T; ++t) tv[u][t] = on[t] ? V::ldcg(p0 + static_cast<i64>(q + u) * pl.lds + SW * t) : V::zero();
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int t = 0; t < T; ++t) V::add(acc[t], tv[u][t]);
      }
      for (; q < nsg; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t)
          if (on[t]) V::add(acc[t], V::ldcg(p0 + static_cast<i64>(q) * pl.lds + SW * t));
      double* yr = a.Y + static_cast<i64>(r) * a.ldy + VW * lane;
#pragma unroll
      for (int t = 0; t < T; ++t)
        if (on[t]) V::st(yr + SW * t, acc[t]);
      if (lane == 0) pl.segcnt[slot0] = 0;  // ready for the next product over this plan
    }
  }
  // ---- groups of kGroupRows consecutive rows (long rows skipped)
  auto header = [&](i64 g, int& rp_l, int& nr) {
    const i64 r0 = g * kGroupRows;
    nr = static_cast<int>(min(static_cast<i64>(kGroupRows), a.rows - r0));
    rp_l = (g < ngroups && lane <= nr) ? __ldg(rowp + r0 + lane) : 0;
  };
  i64 g = w - nseg;
  int rp_n = 0, nr_n = 0;
  if (g < ngroups) header(g, rp_n, nr_n);
  for (; g < ngroups; g += nw) {
    const int rp_l = rp_n, nr = nr_n;
    if (g + nw < ngroups) header(g + nw, rp_n, nr_n);  // next group's row pointers in flight
    const i64 r0 = g * kGroupRows;
    const int rp_next = __shfl_down_sync(0xffffffffu, rp_l, 1);
    double* Yg = a.Y + r0 * static_cast<i64>(a.ldy) + VW * lane;
    auto store = [&](int r, const VT(&ac)[T]) {
      double* yr = Yg + static_cast<i64>(r) * a.ldy;
#pragma unroll
      for (int t = 0; t < T; ++t)
        if (on[t]) V::st(yr + SW * t, ac[t]);
    };
    const int e_l = lane < nr ? rp_next : 0;  // end of row `lane` of the group
    int ri = 0;
    while (ri < nr) {
      const int wb = __shfl_sync(0xffffffffu, rp_l, ri);
      const unsigned fm = __ballot_sync(0xffffffffu, lane >= ri && lane < nr && e_l <= wb + 32);
      if (!(fm & (1u << ri))) {  // row ri is long: the segment items have it
        ++ri;
        continue;
      }
      const int last = __ffs(~(fm >> ri)) - 1 + ri - 1;  // end of the contiguous run of fitting rows
      const int we = __shfl_sync(0xffffffffu, e_l, last);
      int c_l = 0;
      double v_l = 0.0;
      if (wb + lane < we) {
        c_l = __ldg(a.col + wb + lane);
        v_l = __ldg(a.val + wb + lane);
      }
      int row_l = -1;  // row (within the group) of entry `lane`
#pragma unroll
      for (int i = 0; i < kGroupRows; ++i) {
        const int rs = __shfl_sync(0xffffffffu, rp_l, i);
        row_l += (i < nr && wb + lane >= rs) ? 1 : 0;
      }
      const unsigned act = __ballot_sync(0xffffffffu, lane < we - wb && c_l >= a.col_lo);
      {  // rows ri..last with no active entry are zero rows
        const bool mine = lane >= ri && lane <= last;
        bool has = false;
        if (mine) {
          const int s = rp_l - wb, e = e_l - wb;
          const unsigned hi = e >= 32 ? 0xffffffffu : ((1u << e) - 1u);
          const unsigned lo = s >= 32 ? 0xffffffffu : ((1u << s) - 1u);
          has = (act & hi & ~lo) != 0;
        }
        unsigned empty = __ballot_sync(0xffffffffu, mine && !has);
        VT z[T];
#pragma unroll
        for (int t = 0; t < T; ++t) z[t] = V::zero();
        while (empty) {
          const int r = __ffs(empty) - 1;
          empty &= empty - 1;
          store(r, z);
        }
      }
      int cur = -1;
      gather(act, c_l, v_l, row_l, acc, cur, store);
      if (cur >= 0) store(cur, acc);
      ri = last + 1;
    }
  }
}

// Rows of several segments: partial sums added in segment order.
__global__ void __launch_bounds__(256) spmm_fixup_kernel(SpmmArgs a, SpmmPlan pl) {
  const int i = static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= *pl.nsplit) return;
  const int r = pl.split_rows[i];
  const int nseg = pl.vstart[r + 1] - pl.vstart[r];
  const double* p0 = pl.scratch + static_cast<i64>(pl.sstart[r]) * pl.lds;
  for (int cc = lane; cc < a.m; cc += 32) {
    double y = 0.0;
    int s = 0;
    for (; s + 8 <= nseg; s += 8) {  // eight loads in flight, sums still in segment order
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = p0[static_cast<i64>(s + u) * pl.lds + cc];
#pragma unroll
      for (int u = 0; u < 8; ++u) y = __dadd_rn(y, t[u]);
    }
    for (; s < nseg; ++s) y = __dadd_rn(y, p0[static_cast<i64>(s) * pl.lds + cc]);
    a.Y[static_cast<i64>(r) * a.ldy + cc] = y;
  }
}

// Narrow products (m <= 128, one (32 VW)-column slab per warp, blockIdx.y):
// the long-row segments first (as the fused kernel, counters per row and
// slab), then chunks of rows (chunk_start_kernel). A warp copies its chunk's
// short-row entries into shared memory as (row, col, val) triples — one lane
// per row, so no per-entry search — and then streams them in order, eight
// entries per batch, the next batch's X rows loaded before the current batch
// is summed: the gathers of a chunk overlap instead of paying one memory
// round trip per row or per window. Sums per row in column order with
// separate multiply and add roundings (bit-identical to the other kernels);
// rows without entries are written as zeros; long rows are left to their
// segments. Entries left of a trailing-column view (col < col_lo) are staged
// as exact zeros.
constexpr int kChunkWarps = 8;
constexpr int kChunkMax = kChunk + kSegNnz;  // short entries per chunk, upper bound
struct ChunkSmem {
  int rp[kChunk + 1];
  int sp[kChunk + 1];
  int col[kChunkMax];
  unsigned char row[kChunkMax];
  double val[kChunkMax];
};

template <int VW, int T>  // T slabs of 32 VW columns per warp
__global__ void __launch_bounds__(32 * kChunkWarps) spmm_chunk_kernel(SpmmArgs a, SpmmPlan pl) {
  using V = SpV<VW>;
  using VT = typename V::T;
  constexpr int SW = 32 * VW, W = SW * T;
  constexpr int U = 8 / T;  // entries per batch (U x T loads in flight per lane)
  __shared__ ChunkSmem csm[kChunkWarps];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ChunkSmem& cs = csm[wib];
  const int c0 = static_cast<int>(blockIdx.y) * W;
  bool on[T];
#pragma unroll
  for (int t = 0; t < T; ++t) on[t] = c0 + SW * t + VW * lane < a.m;
  const double* Xs = a.X + c0 + VW * lane;
  double* Ys = a.Y + c0 + VW * lane;
  const int* rowp = a.rowptr + a.row_off;
  const i64 gw = static_cast<i64>(blockIdx.x) * kChunkWarps + wib, nw = static_cast<i64>(gridDim.x) * kChunkWarps;
  auto store = [&](double* yr, const VT (&v)[T]) {
#pragma unroll
    for (int t = 0; t < T; ++t)
      if (on[t]) V::st(yr + SW * t, v[t]);
  };
  // ---- long-row segments of this column block
  const i64 nseg = pl.vstart[a.rows];
  i64 w = gw;
  for (; w < nseg; w += nw) {
    const int r = pl.vrow[w];
    const int vs = pl.vstart[r];
    const int sg = static_cast<int>(w - vs);
    const int nsg = pl.vstart[r + 1] - vs;
    const int seg0 = rowp[r] + sg * kLongSeg;
    const int cnt = min(kLongSeg, rowp[r + 1] - seg0);
    int c_l = 0;
    double v_l = 0.0;
    if (lane < cnt) {
      c_l = __ldg(a.col + seg0 + lane);
      v_l = __ldg(a.val + seg0 + lane);
      if (c_l < a.col_lo) {  // trailing-column view: an exact zero
        c_l = a.col_lo;
        v_l = 0.0;
      }
    }
    VT acc[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = V::zero();
    for (int q = 0; q < cnt; q += U) {  // U entries' loads in flight, sums in column order
      VT xv[U][T];
      double vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = __shfl_sync(0xffffffffu, c_l, (q + u) & 31);
        vv[u] = __shfl_sync(0xffffffffu, v_l, (q + u) & 31);
#pragma unroll
        for (int t = 0; t < T; ++t)
          xv[u][t] = (q + u < cnt && on[t]) ? V::ld(Xs + static_cast<i64>(c) * a.ldx + SW * t) : V::zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q + u < cnt)
#pragma unroll
          for (int t = 0; t < T; ++t) V::fma(acc[t], vv[u], xv[u][t]);
    }
    const int slot0 = pl.sstart[r];
    store(pl.scratch + static_cast<i64>(slot0 + sg) * pl.lds + c0 + VW * lane, acc);
    __threadfence();
    int last = 0;
    int* ctr = pl.segcnt + static_cast<i64>(slot0) * gridDim.y + blockIdx.y;
    if (lane == 0) last = atomicAdd(ctr, 1) == nsg - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {  // every partial of row r (this column block) is written: add them in segment order
      __threadfence();
      const double* p0 = pl.scratch + static_cast<i64>(slot0) * pl.lds + c0 + VW * lane;
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] = V::zero();
      for (int q = 0; q < nsg; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t)
          if (on[t]) V::add(acc[t], V::ldcg(p0 + static_cast<i64>(q) * pl.lds + SW * t));
      store(Ys + static_cast<i64>(r) * a.ldy, acc);
      if (lane == 0) *ctr = 0;
    }
  }
  // ---- chunks
  for (i64 c = w - nseg; c < pl.nch; c += nw) {
    const int r0 = pl.crow[c], r1 = pl.crow[c + 1];
    if (r0 >= r1) continue;
    const int nr = r1 - r0;
    __syncwarp();  // the previous chunk's readers are done
    for (int i = lane; i <= nr; i += 32) {
      cs.rp[i] = __ldg(rowp + r0 + i);
      cs.sp[i] = __ldg(pl.sptr + r0 + i);
    }
    __syncwarp();
    const int q0 = cs.sp[0], ns = cs.sp[nr] - q0;
    // entries of the short rows -> (row, col, val), one lane per row; empty rows -> zeros
    for (int i0 = 0; i0 < nr; i0 += 32) {
      const int i = i0 + lane;
      bool zero = false;
      if (i < nr) {
        const int s = cs.rp[i], len = cs.rp[i + 1] - s;
        zero = len == 0;
        if (len > 0 && len <= kSegNnz) {
          const int q = cs.sp[i] - q0;
          for (int t = 0; t < len; ++t) {
            const int cc = __ldg(a.col + s + t);
            const bool act = cc >= a.col_lo;  // trailing-column view: inactive entries add exact zeros
            cs.col[q + t] = act ? cc : a.col_lo;
            cs.val[q + t] = act ? __ldg(a.val + s + t) : 0.0;
            cs.row[q + t] = static_cast<unsigned char>(i);
          }
        }
      }
      unsigned zm = __ballot_sync(0xffffffffu, zero);
      VT z[T];
#pragma unroll
      for (int t = 0; t < T; ++t) z[t] = V::zero();
      while (zm) {
        const int j = __ffs(zm) - 1;
        zm &= zm - 1;
        store(Ys + static_cast<i64>(r0 + i0 + j) * a.ldy, z);
      }
    }
    __syncwarp();
    // stream the entries: batch b + 1's X rows in flight while batch b is summed
    int cur = -1;
    VT acc[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = V::zero();
    VT xn[U][T];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int t = 0; t < T; ++t)
        xn[u][t] = (u < ns && on[t]) ? V::ld(Xs + static_cast<i64>(cs.col[u]) * a.ldx + SW * t) : V::zero();
    for (int b = 0; b < ns; b += U) {
      VT xc[U][T];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < T; ++t) xc[u][t] = xn[u][t];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = b + U + u;
#pragma unroll
        for (int t = 0; t < T; ++t)
          xn[u][t] = (j < ns && on[t]) ? V::ld(Xs + static_cast<i64>(cs.col[j]) * a.ldx + SW * t) : V::zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = b + u;
        if (j >= ns) break;
        const int rw = cs.row[j];
        if (rw != cur) {
          if (cur >= 0) store(Ys + static_cast<i64>(r0 + cur) * a.ldy, acc);
          cur = rw;
#pragma unroll
          for (int t = 0; t < T; ++t) acc[t] = V::zero();
        }
        const double vj = cs.val[j];
#pragma unroll
        for (int t = 0; t < T; ++t) V::fma(acc[t], vj, xc[u][t]);
      }
    }
    if (cur >= 0) store(Ys + static_cast<i64>(r0 + cur) * a.ldy, acc);
  }
}

inline void spmm_chunk_launch(const SpmmArgs& a, const SpmmPlan& pl, i64 vmax, int tmax, cudaStream_t st) {
  const bool vec2 = a.m > 32 && a.m % 2 == 0 && a.ldx % 2 == 0 && a.ldy % 2 == 0 && pl.lds % 2 == 0 &&
                    ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.Y) |
                      reinterpret_cast<uintptr_t>(pl.scratch)) & 15) == 0;
  // columns per warp: one 32-column slab (m <= 32), else 64-column slabs, up to tmax per warp
  const int T = vec2 ? static_cast<int>(std::min<i64>(tmax, cdiv(a.m, 64))) : 1;
  const int W = vec2 ? 64 * (T >= 4 ? 4 : T >= 2 ? 2 : 1) : 32;
  const i64 items = vmax + pl.nch;
  const int per_sm = !vec2 ? 3 : T >= 2 ? 1 : 2;
  const unsigned gx = static_cast<unsigned>(std::max<i64>(1, std::min<i64>(cdiv(items, kChunkWarps), 148 * per_sm)));
  const dim3 grid(gx, static_cast<unsigned>(cdiv(a.m, W)));
  if (!vec2) spmm_chunk_kernel<1, 1><<<grid, 32 * kChunkWarps, 0, st>>>(a, pl);
  else if (W == 64) spmm_chunk_kernel<2, 1><<<grid, 32 * kChunkWarps, 0, st>>>(a, pl);
  else if (W == 128) spmm_chunk_kernel<2, 2><<<grid, 32 * kChunkWarps, 0, st>>>(a, pl);
  else spmm_chunk_kernel<2, 4><<<grid, 32 * kChunkWarps, 0, st>>>(a, pl);
  STG_LAUNCH();
}

template <int VW, int T>
inline void spmm_fused_go(const SpmmArgs& a, const SpmmPlan& pl, i64 vmax, i64 ngroups, cudaStream_t st) {
  const i64 items = vmax + ngroups;  // vmax: upper bound of the long-row segments
  const unsigned grid = static_cast<unsigned>(std::max<i64>(1, std::min<i64>(cdiv(items, 8), 148 * spmm_fused_minb(VW, T))));
  spmm_fused_kernel<VW, T><<<grid, 256, 0, st>>>(a, pl, ngroups);
}

// One launch: VW = 2 (128-bit) when the operands allow it and m > 32.
inline void spmm_fused_launch(const SpmmArgs& a, const SpmmPlan& pl, i64 vmax, cudaStream_t st) {
  const i64 ng = cdiv(a.rows, kGroupRows);
  const bool vec2 = a.m > 32 && a.m % 2 == 0 && a.ldx % 2 == 0 && a.ldy % 2 == 0 && pl.lds % 2 == 0 &&
                    ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.Y) |
                      reinterpret_cast<uintptr_t>(pl.scratch)) & 15) == 0;
  if (vec2) {
    switch (static_cast<int>(cdiv(a.m, 64))) {
      case 1: spmm_fused_go<2, 1>(a, pl, vmax, ng, st); break;
      case 2: spmm_fused_go<2, 2>(a, pl, vmax, ng, st); break;
      case 3: spmm_fused_go<2, 3>(a, pl, vmax, ng, st); break;
      default: spmm_fused_go<2, 4>(a, pl, vmax, ng, st); break;
    }
  } else {
    switch (static_cast<int>(cdiv(a.m, 32))) {
      case 1: spmm_fused_go<1, 1>(a, pl, vmax, ng, st); break;
      case 2: spmm_fused_go<1, 2>(a, pl, vmax, ng, st); break;
      case 3: spmm_fused_go<1, 3>(a, pl, vmax, ng, st); break;
      case 4: spmm_fused_go<1, 4>(a, pl, vmax, ng, st); break;
      case 5: spmm_fused_go<1, 5>(a, pl, vmax, ng, st); break;
      case 6: spmm_fused_go<1, 6>(a, pl, vmax, ng, st); break;
      case 7: spmm_fused_go<1, 7>(a, pl, vmax, ng, st); break;
      default: spmm_fused_go<1, 8>(a, pl, vmax, ng, st); break;
    }
  }
  STG_LAUNCH();
}

// ---- segment plan of a CSR row range (built once per perturbation)
__global__ void seg_count_kernel(const int* rowptr, i64 row_off, i64 rows, int* cnt, int* cnt2, int* slen) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > rows) return;
  if (r == rows) {
    cnt[r] = cnt2[r] = slen[r] = 0;
    return;
  }
  const int len = rowptr[r + row_off + 1] - rowptr[r + row_off];
  const int c = len > kSegNnz ? (len + kLongSeg - 1) / kLongSeg : 0;  // short rows: the row-group kernel
  cnt[r] = c;
  cnt2[r] = c > 1 ? c : 0;
  slen[r] = c > 0 ? 0 : len;  // entries of short rows (the chunk kernel's positions)
}

// Chunks of the chunk kernel: row r sits at position r + sptr[r] (rows and
// short-row entries before it); chunk c owns the rows with positions in
// [c kChunk, (c + 1) kChunk): <= kChunk rows and < kChunk + kSegNnz short
// entries. One thread per row writes crow[c] for the chunks that start at it.
__global__ void chunk_start_kernel(const int* sptr, i64 rows, int nch, int* crow) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > rows) return;
  const i64 pos = r == rows ? static_cast<i64>(nch) * kChunk : r + sptr[r];
  const i64 prev = r == 0 ? -1 : (r - 1) + sptr[r - 1];
  const i64 c_hi = r == rows ? nch : pos / kChunk;            // chunks whose first position is <= pos
  const i64 c_lo = r == 0 ? 0 : prev / kChunk + 1;            // ... and > prev
  for (i64 c = c_lo; c <= c_hi && c <= nch; ++c) crow[c] = static_cast<int>(r);
}

__global__ void seg_fill_kernel(const int* vstart, i64 rows, int* vrow, int* split_rows, int* nsplit) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int b = vstart[r], c = vstart[r + 1] - b;
  for (int s = 0; s < c; ++s) vrow[b + s] = static_cast<int>(r);
  if (c > 1) split_rows[atomicAdd(nsplit, 1)] = static_cast<int>(r);
}

// long_rows: a row longer than kSegNnz may exist (nnz > kSegNnz);
// split_max > 0: a row longer than kLongSeg may exist (segments + fix-up)
inline void spmm_launch(const SpmmArgs& a, const SpmmPlan& pl, i64 vmax, i64 split_max, bool long_rows,
                        cudaStream_t st) {
  const bool vec2 = a.m % 2 == 0 && a.ldx % 2 == 0 && a.ldy % 2 == 0 && a.m <= 256 &&
                    ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.Y)) & 15) == 0;
  // all-column warps for the wide sketch operands (m > 128: 0.245 -> 0.209 ms per
  // step at config 3); the column-slab kernel, which keeps a group's X rows in
  // flight through shared memory, for the narrower ones
  static const bool rows_kernel = !getenv_flag("STG_SPMM_SLABS");  // development A/B
  if (vec2 && rows_kernel && a.m > 128) {
    const i64 ng = cdiv(a.rows, kGroupRows);
    const unsigned grid = static_cast<unsigned>(std::min<i64>(cdiv(ng, 8), 148 * 16));
    switch (static_cast<int>(cdiv(a.m, 64))) {
      case 1: spmm_rows_kernel<1><<<grid, 256, 0, st>>>(a, ng); break;
      case 2: spmm_rows_kernel<2><<<grid, 256, 0, st>>>(a, ng); break;
      case 3: spmm_rows_kernel<3><<<grid, 256, 0, st>>>(a, ng); break;
      default: spmm_rows_kernel<4><<<grid, 256, 0, st>>>(a, ng); break;
    }
    STG_LAUNCH();
  } else {  // rows of at most kSegNnz nonzeros
    const bool vec = a.m > 32 && a.m % 2 == 0 && a.ldx % 2 == 0 && a.ldy % 2 == 0 &&
                     ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.Y)) & 15) == 0;
    const int w = vec ? 64 : 32;
    const dim3 g(static_cast<unsigned>(cdiv(cdiv(a.rows, kGroupRows), kGroupWarps)), static_cast<unsigned>(cdiv(a.m, w)));
    if (vec) spmm_group_kernel<true><<<g, 32 * kGroupWarps, spmm_group_smem<true>(), st>>>(a);
    else spmm_group_kernel<false><<<g, 32 * kGroupWarps, spmm_group_smem<false>(), st>>>(a);
    STG_LAUNCH();
  }
  if (!long_rows) return;  // no row longer than kSegNnz can exist
  const unsigned grid = static_cast<unsigned>(cdiv(vmax, 8));
  const int T = static_cast<int>(cdiv(a.m < 1 ? 1 : a.m, 32));
  switch (T) {
    case 1: spmm_kernel<1><<<grid, 256, 0, st>>>(a, pl); break;
    case 2: spmm_kernel<2><<<grid, 256, 0, st>>>(a, pl); break;
    case 3: spmm_kernel<3><<<grid, 256, 0, st>>>(a, pl); break;
    case 4: spmm_kernel<4><<<grid, 256, 0, st>>>(a, pl); break;
    case 5: spmm_kernel<5><<<grid, 256, 0, st>>>(a, pl); break;
    case 6: spmm_kernel<6><<<grid, 256, 0, st>>>(a, pl); break;
    case 7: spmm_kernel<7><<<grid, 256, 0, st>>>(a, pl); break;
    case 8: spmm_kernel<8><<<grid, 256, 0, st>>>(a, pl); break;
    default: throw std::invalid_argument("spmm: more than 256 dense columns");
  }
  STG_LAUNCH();
  if (split_max > 0) {
    spmm_fixup_kernel<<<static_cast<unsigned>(cdiv(split_max, 8)), 256, 0, st>>>(a, pl);
    STG_LAUNCH();
  }
}

}  // namespace stg
