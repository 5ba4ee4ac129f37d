"""B200-native G-REST per-step eigen-update (arxiv 2603.19439 hot path).

Python binding of the C ABI in include/spectrack_gpu.h (libspectrack_b200.so,
built in-tree for sm_100a). The library is the product; this module only
marshals host buffers for tests and bench.py. There is no CPU fallback: if the
CUDA library is missing or no GPU is visible, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STG_LIB") or os.path.join(_HERE, "libspectrack_b200.so")  # STG_LIB: development A/B only

I64 = C.c_int64
DP = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)

ST_OK, ST_INVALID_ARGUMENT, ST_RUNTIME_ERROR, ST_CUDA_ERROR, ST_OTHER = range(5)
KIND = {"trip-basic": 0, "trip": 1, "rm": 2, "iasc": 3, "grest2": 4, "grest3": 5, "grest-rsvd": 6, "timers": 7}
BASIS = {"iasc": 0, "grest2": 1, "grest3": 2, "grest-rsvd": 3}
OPERATOR = {"adjacency": 0, "laplacian": 1, "normalized-laplacian": 2}
ORDER = {"abs_desc": 0, "alg_desc": 1}
FLAG_FORCE_DENSE, FLAG_TIMING, FLAG_KERNEL_TIMING, FLAG_CUSOLVER_EIG = 1, 2, 4, 8
KERNEL_CLASSES = ["dmma_gram", "dmma_gemm", "spmm", "cholesky", "tri_inverse", "eigensolver", "csr_merge", "rng",
                  "rotate_x", "masked_gram_x", "spmm_sketch", "ingest_other", "spmm_full", "dmma_gram_narrow",
                  "dmma_gemm_narrow"]


class StConfig(C.Structure):
    _fields_ = [("kind", C.c_int32), ("op", C.c_int32), ("k", C.c_int64), ("order", C.c_int32),
                ("rsvd_l", C.c_int64), ("rsvd_p", C.c_int64), ("seed", C.c_uint64), ("device", C.c_int32),
                ("flags", C.c_int32)]


class StLanczosOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_basis", C.c_int64), ("max_restarts", C.c_int64)]


class StCsrBlock(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64), ("rowptr", I32P), ("colidx", I32P),
                ("values", DP)]


class StGraphUpdate(C.Structure):
    _fields_ = [("n_old", C.c_int64), ("n_new", C.c_int64), ("k_block", StCsrBlock), ("g_block", StCsrBlock),
                ("c_block", StCsrBlock)]


class StTrackerOptions(C.Structure):
    _fields_ = [("mu", C.c_double), ("trip_replace_span", C.c_int32), ("theta", C.c_double),
                ("min_restart_gap", C.c_int64), ("restart_inner", C.c_int32)]


class StUpdate(C.Structure):
    _fields_ = [("n_added", C.c_int64), ("added_i", I64P), ("added_j", I64P), ("added_w", DP),
                ("n_removed", C.c_int64), ("removed_i", I64P), ("removed_j", I64P), ("n_new", C.c_int64),
                ("n_new_edges", C.c_int64), ("new_i", I64P), ("new_j", I64P), ("new_w", DP)]


class TrackerError(Exception):
    """Failure with the reference's exception category in ``kind``
    ('invalid_argument' | 'runtime_error' | 'cuda' | 'other')."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


_KINDS = {ST_INVALID_ARGUMENT: "invalid_argument", ST_RUNTIME_ERROR: "runtime_error", ST_CUDA_ERROR: "cuda",
          ST_OTHER: "other"}
_lib = None


def lib():
    """Load the in-tree CUDA library (fails loudly when it is absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.st_create.argtypes = [C.POINTER(StConfig), I64, I32P, I32P, DP, DP, DP, I64, C.POINTER(C.c_void_p)]
        L.st_step.argtypes = [C.c_void_p, C.POINTER(StUpdate)]
        L.st_tracker_init.argtypes = [C.POINTER(StConfig), C.POINTER(StLanczosOptions), I64, I32P, I32P, DP,
                                      C.POINTER(C.c_void_p)]
        L.st_init_stats.argtypes = [C.c_void_p, I64P, I64P]
        L.st_set_tracker_options.argtypes = [C.c_void_p, C.POINTER(StTrackerOptions)]
        L.st_tracker_state.argtypes = [C.c_void_p, DP, I64P, DP, C.POINTER(C.c_int32)]
        L.st_reserve.argtypes = [C.c_void_p, I64, I64]
        L.st_step_blocks.argtypes = [C.c_void_p, C.POINTER(StGraphUpdate)]
        L.st_step_perturbation.argtypes = [C.c_void_p, I64, I64, C.POINTER(StCsrBlock)]
        L.st_info.argtypes = [C.c_void_p, I64P, I64P, C.POINTER(C.c_uint64), I64P, I64P, I64P, DP]
        L.st_get_embedding.argtypes = [C.c_void_p, DP, DP, I64]
        L.st_residual_norms.argtypes = [C.c_void_p, DP]
        L.st_angles.argtypes = [C.c_void_p, DP, I64, DP, DP]
        L.st_debug_determinism.argtypes = [C.c_void_p, C.c_int32, I64, C.c_int32, C.c_int32, C.c_int32, DP, DP]
        L.st_debug_determinism.restype = C.c_int
        L.st_get_values.argtypes = [C.c_void_p, DP]
        L.st_get_csr.argtypes = [C.c_void_p, C.c_int32, I32P, I32P, DP]
        L.st_probe_basis.argtypes = [C.c_void_p, C.POINTER(StUpdate), C.c_int32, C.c_uint64, DP, I64, I64, I64P]
        L.st_probe_rr.argtypes = [C.c_void_p, C.POINTER(StUpdate), DP, I64, I64, I64, DP, DP, I64]
        L.st_last_error.argtypes = [C.c_void_p]
        L.st_last_error.restype = C.c_char_p
        L.st_destroy.argtypes = [C.c_void_p]
        L.st_destroy.restype = None
        L.st_last_timings.argtypes = [C.c_void_p, DP, C.c_int32]
        L.st_last_timings.restype = C.c_int32
        L.st_last_launches.argtypes = [C.c_void_p]
        L.st_last_launches.restype = C.c_int64
        L.st_step_device.argtypes = [C.c_void_p, C.POINTER(StUpdate)]
        L.st_step_device.restype = C.c_int
        L.st_kernel_stats.argtypes = [C.c_void_p, C.c_int32, DP, I64P, DP]
        L.st_kernel_stats.restype = C.c_int32
        L.st_kernel_stats2.argtypes = [C.c_void_p, C.c_int32, DP, I64P, DP, DP, DP]
        L.st_kernel_stats2.restype = C.c_int32
        L.st_set_peaks.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.st_set_peaks.restype = None
        L.st_reset_kernel_stats.argtypes = [C.c_void_p]
        L.st_reset_kernel_stats.restype = None
        L.st_sym_eig_dense.argtypes = [C.c_int32, I64, DP, C.c_int32, I64, DP, DP]
        L.st_sym_eig_dense.restype = C.c_int
        L.st_gaussian_matrix.argtypes = [C.c_int32, C.c_uint64, I64, I64, DP]
        L.st_gaussian_matrix.restype = C.c_int
        from . import shard as _shard

        L.st_create_sharded.argtypes = [C.POINTER(StConfig), C.POINTER(_shard.StComm), I64, I64, I64, I64, I32P,
                                        I32P, DP, DP, DP, I64, C.POINTER(C.c_void_p)]
        L.st_shard_rows.argtypes = [C.c_void_p, I64P, I64P]
        L.st_nccl_unique_id.argtypes = [C.c_void_p]
        L.st_nccl_unique_id.restype = C.c_int
        L.st_comm_nccl_create.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_shard.StComm)]
        L.st_comm_nccl_create.restype = C.c_int
        L.st_comm_nccl_destroy.argtypes = [C.POINTER(_shard.StComm)]
        L.st_comm_nccl_destroy.restype = None
        L.st_shard_stats.argtypes = [C.c_void_p, I64P, I64P, I64P]
        L.st_shard_stats.restype = C.c_int
        L.st_shard_layout.argtypes = [C.c_int32, I64P, I64, C.c_int32, I64, I64P, I64]
        L.st_shard_layout.restype = C.c_int64
        for f in ("st_create", "st_step", "st_info", "st_get_embedding", "st_get_values", "st_get_csr",
                  "st_probe_basis", "st_probe_rr", "st_create_sharded", "st_shard_rows", "st_residual_norms",
                  "st_reserve", "st_tracker_init", "st_init_stats", "st_step_blocks", "st_step_perturbation",
                  "st_set_tracker_options", "st_tracker_state", "st_angles"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _p(a, t=DP):
    return a.ctypes.data_as(t) if a is not None else None


def _i64(x):
    return np.ascontiguousarray(np.asarray(x, np.int64).reshape(-1))


def _d(x):
    return np.ascontiguousarray(np.asarray(x, np.float64).reshape(-1))


@dataclass
class Update:
    """Edit lists of one step (assemble_update, graph.hpp:65-69)."""
    added: tuple = ((), (), ())
    removed: tuple = ((), ())
    n_new: int = 0
    new_edges: tuple = ((), (), ())

    @staticmethod
    def make(added=(), removed=(), n_new=0, new_edges=()):
        def e3(e):
            if isinstance(e, tuple) and len(e) == 3 and hasattr(e[0], "__len__"):
                return _i64(e[0]), _i64(e[1]), _d(e[2])
            e = list(e)
            return (_i64([t[0] for t in e]), _i64([t[1] for t in e]),
                    _d([t[2] if len(t) > 2 else 1.0 for t in e]))

        def e2(e):
            if isinstance(e, tuple) and len(e) == 2 and hasattr(e[0], "__len__"):
                return _i64(e[0]), _i64(e[1])
            e = list(e)
            return _i64([t[0] for t in e]), _i64([t[1] for t in e])

        return Update(e3(added), e2(removed), int(n_new), e3(new_edges))

    def struct(self):
        ai, aj, aw = _i64(self.added[0]), _i64(self.added[1]), _d(self.added[2])
        ri, rj = _i64(self.removed[0]), _i64(self.removed[1])
        ni, nj, nw = _i64(self.new_edges[0]), _i64(self.new_edges[1]), _d(self.new_edges[2])
        keep = (ai, aj, aw, ri, rj, ni, nj, nw)
        s = StUpdate(len(ai), _p(ai, I64P), _p(aj, I64P), _p(aw), len(ri), _p(ri, I64P), _p(rj, I64P),
                     int(self.n_new), len(ni), _p(ni, I64P), _p(nj, I64P), _p(nw))
        return keep, s

    def pinned(self) -> "Update":
        """The same edit lists in page-locked host memory (torch pin_memory):
        st_step then DMAs each list straight from it, without the staging copy."""
        import torch

        keep = []

        def pin(x, dt):
            a = np.ascontiguousarray(np.asarray(x, dt).reshape(-1))
            t = torch.empty(len(a), dtype=torch.int64 if dt == np.int64 else torch.float64, pin_memory=True)
            v = t.numpy()
            v[:] = a
            keep.append(t)
            return v

        u = Update((pin(self.added[0], np.int64), pin(self.added[1], np.int64), pin(self.added[2], np.float64)),
                   (pin(self.removed[0], np.int64), pin(self.removed[1], np.int64)), int(self.n_new),
                   (pin(self.new_edges[0], np.int64), pin(self.new_edges[1], np.int64),
                    pin(self.new_edges[2], np.float64)))
        u._pinned_storage = keep
        return u

    def h2d_bytes(self) -> int:
        return 16 * (len(self.added[0]) + len(self.removed[0]) + len(self.new_edges[0])) + 8 * (
            len(self.added[0]) + len(self.new_edges[0]))


def _csr_block(rows, cols, rp, col, val):
    rp = np.ascontiguousarray(rp, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    return (rp, col, val), StCsrBlock(rows, cols, len(col), _p(rp, I32P), _p(col, I32P), _p(val))


def csr_from_coo(n_rows, rows, cols, vals):
    """Canonical CSR (sorted, duplicates summed in input order) of COO triplets."""
    rows, cols, vals = np.asarray(rows, np.int64), np.asarray(cols, np.int64), np.asarray(vals, np.float64)
    o = np.lexsort((cols, rows))
    rows, cols, vals = rows[o], cols[o], vals[o]
    if len(rows):
        head = np.ones(len(rows), bool)
        head[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        idx = np.flatnonzero(head)
        sums = np.add.reduceat(vals, idx) if len(idx) else vals
        rows, cols, vals = rows[idx], cols[idx], sums
    rp = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=rp[1:])
    return rp.astype(np.int32), cols.astype(np.int32), vals


@dataclass
class GraphUpdate:
    """GraphUpdate (graph.hpp:23-37): blocks K (n_old^2), G (n_old x n_new),
    C (n_new^2) as canonical CSR triples (rowptr, col, val)."""
    n_old: int
    n_new: int
    k_block: tuple
    g_block: tuple
    c_block: tuple

    @staticmethod
    def from_edits(n_old: int, upd: "Update") -> "GraphUpdate":
        """assemble_update (graph.cpp:45-100) block placement, without its
        validation: added/removed -> K (both triangles), old-new -> G,
        new-new -> C (both triangles)."""
        ai, aj, aw = (np.asarray(x) for x in upd.added)
        ri, rj = (np.asarray(x, np.int64) for x in upd.removed)
        ki = np.concatenate([ai, aj, ri, rj]).astype(np.int64)
        kj = np.concatenate([aj, ai, rj, ri]).astype(np.int64)
        kv = np.concatenate([aw, aw, -np.ones(len(ri)), -np.ones(len(ri))])
        ni, nj, nw = (np.asarray(x) for x in upd.new_edges)
        lo, hi = np.minimum(ni, nj).astype(np.int64), np.maximum(ni, nj).astype(np.int64)
        g = lo < n_old
        S = int(upd.n_new)
        gb = csr_from_coo(n_old, lo[g], hi[g] - n_old, nw[g])
        cl, ch, cw = lo[~g] - n_old, hi[~g] - n_old, nw[~g]
        cb = csr_from_coo(S, np.concatenate([cl, ch]), np.concatenate([ch, cl]), np.concatenate([cw, cw]))
        return GraphUpdate(n_old, S, csr_from_coo(n_old, ki, kj, kv), gb, cb)

    def struct(self):
        kk, kbs = _csr_block(self.n_old, self.n_old, *self.k_block)
        gk, gbs = _csr_block(self.n_old, self.n_new, *self.g_block)
        ck, cbs = _csr_block(self.n_new, self.n_new, *self.c_block)
        return (kk, gk, ck), StGraphUpdate(self.n_old, self.n_new, kbs, gbs, cbs)


class TrackerSession:
    """One tracker lane on one GPU: the adjacency CSR (and shifted operator for
    Laplacian operators) plus the TrackerState, resident in HBM."""

    def __init__(self, rowptr, col, val, values, vectors, kind="grest-rsvd", k=None, order="abs_desc",
                 rsvd_l=100, rsvd_p=100, seed=0, operator="adjacency", device=0, force_dense=False, timing=False,
                 kernel_timing=False, cusolver_eig=False):
        L = lib()
        rowptr = np.ascontiguousarray(rowptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        values = _d(values)
        vectors = np.asfortranarray(np.asarray(vectors, np.float64))
        n = len(rowptr) - 1
        k = len(values) if k is None else k
        flags = ((FLAG_FORCE_DENSE if force_dense else 0) | (FLAG_TIMING if timing else 0)
                 | (FLAG_KERNEL_TIMING if kernel_timing else 0) | (FLAG_CUSOLVER_EIG if cusolver_eig else 0))
        cfg = StConfig(KIND[kind], OPERATOR[operator], k, ORDER[order], rsvd_l, rsvd_p, seed, device, flags)
        h = C.c_void_p()
        rc = L.st_create(C.byref(cfg), n, _p(rowptr, I32P), _p(col, I32P), _p(val), _p(values),
                         vectors.ctypes.data_as(DP), vectors.shape[0], C.byref(h))
        if rc != ST_OK:
            raise TrackerError(_KINDS.get(rc, "other"), L.st_last_error(None).decode())
        self._h = h.value
        self.k = k

    @classmethod
    def tracker_init(cls, rowptr, col, val, k, kind="grest-rsvd", order="abs_desc", rsvd_l=100, rsvd_p=100, seed=0,
                     operator="adjacency", device=0, tol=1e-10, max_basis=0, max_restarts=500, force_dense=False,
                     timing=False, kernel_timing=False, cusolver_eig=False):
        """tracker_init (trackers.cpp:132-145) on the device: the session starts
        from the leading k eigenpairs of the tracked operator, computed by
        thick-restart Lanczos (lanczos.hpp:38-127) on the GPU."""
        L = lib()
        rowptr = np.ascontiguousarray(rowptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        flags = ((FLAG_FORCE_DENSE if force_dense else 0) | (FLAG_TIMING if timing else 0)
                 | (FLAG_KERNEL_TIMING if kernel_timing else 0) | (FLAG_CUSOLVER_EIG if cusolver_eig else 0))
        cfg = StConfig(KIND[kind], OPERATOR[operator], k, ORDER[order], rsvd_l, rsvd_p, seed, device, flags)
        opts = StLanczosOptions(tol, max_basis, max_restarts)
        h = C.c_void_p()
        rc = L.st_tracker_init(C.byref(cfg), C.byref(opts), len(rowptr) - 1, _p(rowptr, I32P), _p(col, I32P),
                               _p(val), C.byref(h))
        if rc != ST_OK:
            raise TrackerError(_KINDS.get(rc, "other"), L.st_last_error(None).decode())
        self = cls.__new__(cls)
        self._h = h.value
        self.k = k
        return self

    def set_tracker_options(self, mu=0.0, trip_replace_span=False, theta=0.01, min_restart_gap=5,
                            restart_inner="iasc") -> None:
        """TrackerOptions of the perturbation trackers and TIMERS (trackers.hpp:52-63)."""
        o = StTrackerOptions(mu, int(trip_replace_span), theta, min_restart_gap, KIND[restart_inner])
        self._check(lib().st_set_tracker_options(self._h, C.byref(o)))

    def tracker_state(self):
        """(accumulated_change, steps_since_restart, restart_scale, ridge_used)."""
        acc, scale = C.c_double(), C.c_double()
        gap = I64()
        ridge = C.c_int32()
        self._check(lib().st_tracker_state(self._h, C.byref(acc), C.byref(gap), C.byref(scale), C.byref(ridge)))
        return acc.value, gap.value, scale.value, bool(ridge.value)

    def init_stats(self):
        """(restarts, operator products) of the device tracker_init."""
        r, p = I64(), I64()
        self._check(lib().st_init_stats(self._h, C.byref(r), C.byref(p)))
        return r.value, p.value

    def close(self):
        if getattr(self, "_h", None):
            lib().st_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc != ST_OK:
            raise TrackerError(_KINDS.get(rc, "other"), lib().st_last_error(self._h).decode())

    def step(self, upd: Update) -> None:
        keep, s = upd.struct()
        self._check(lib().st_step(self._h, C.byref(s)))

    def step_blocks(self, g: GraphUpdate) -> None:
        """One step from a GraphUpdate's blocks (st_step_blocks)."""
        keep, st = g.struct()
        self._check(lib().st_step_blocks(self._h, C.byref(st)))

    def step_perturbation(self, n_old: int, n_new: int, rowptr, col, val) -> None:
        """tracker_step(state, Perturbation{n_old, n_new, delta}) (st_step_perturbation)."""
        n = n_old + n_new
        keep, b = _csr_block(n, n, rowptr, col, val)
        self._check(lib().st_step_perturbation(self._h, n_old, n_new, C.byref(b)))

    def reserve(self, n_nodes: int, nnz: int) -> None:
        """Size the session for a stream reaching n_nodes nodes and nnz stored
        entries (st_reserve): later steps up to that size grow no buffer."""
        self._check(lib().st_reserve(self._h, int(n_nodes), int(nnz)))

    def step_device(self, dev_update) -> None:
        """Step with edit arrays already in device memory: `dev_update` is a
        DeviceUpdate (torch CUDA tensors)."""
        self._check(lib().st_step_device(self._h, C.byref(dev_update.struct)))

    def kernel_stats(self) -> dict:
        out = {}
        for i, name in enumerate(KERNEL_CLASSES):
            ms, work, work2, bound = C.c_double(), C.c_double(), C.c_double(), C.c_double()
            cnt = I64()
            lib().st_kernel_stats2(self._h, i, C.byref(ms), C.byref(cnt), C.byref(work), C.byref(work2),
                                   C.byref(bound))
            out[name] = dict(ms=ms.value, launches=cnt.value, work=work.value, work2=work2.value,
                             bound_ms=bound.value)
        return out

    def set_peaks(self, fp64_tflops: float, hbm_gbs: float) -> None:
        lib().st_set_peaks(self._h, fp64_tflops, hbm_gbs)

    def reset_kernel_stats(self) -> None:
        lib().st_reset_kernel_stats(self._h)

    def info(self):
        n, k, nnz_a, nnz_t, nnz_d = I64(), I64(), I64(), I64(), I64()
        st = C.c_uint64()
        alpha = C.c_double()
        lib().st_info(self._h, C.byref(n), C.byref(k), C.byref(st), C.byref(nnz_a), C.byref(nnz_t),
                      C.byref(nnz_d), C.byref(alpha))
        return dict(n=n.value, k=k.value, steps_taken=st.value, nnz_a=nnz_a.value, nnz_t=nnz_t.value,
                    nnz_delta=nnz_d.value, alpha=alpha.value)

    def values(self) -> np.ndarray:
        v = np.zeros(self.k)
        self._check(lib().st_get_values(self._h, _p(v)))
        return v

    def embedding(self):
        n = self.info()["n"]
        vals = np.zeros(self.k)
        vecs = np.zeros((n, self.k), order="F")
        self._check(lib().st_get_embedding(self._h, _p(vals), vecs.ctypes.data_as(DP), n))
        return vals, np.ascontiguousarray(vecs)

    def residual_norms(self) -> np.ndarray:
        """||Op x_i - theta_i x_i|| per tracked pair, on the device (st_residual_norms)."""
        out = np.zeros(self.k)
        self._check(lib().st_residual_norms(self._h, _p(out)))
        return out

    def determinism(self, which: int, N: int, m1: int, m2: int, reps: int = 3, out: bool = False):
        """Largest run-to-run difference of a kernel on pseudo-random operands
        (0 Gram, 1 row-local GEMM, 2 SpMV of the session operator, 3 its SpMM);
        with out=True also the first run's result."""
        d = C.c_double()
        rows = m1 if which == 0 else N
        cols = m2 if which in (0, 1) else 1 if which == 2 else m1
        buf = np.zeros(rows * cols) if out else None
        self._check(lib().st_debug_determinism(self._h, which, N, m1, m2, reps, C.byref(d),
                                               _p(buf) if out else None))
        return (d.value, buf.reshape(rows, cols)) if out else d.value

    def angles(self, ref_vectors):
        """(psi per vector, largest principal angle) against reference vectors
        (n x k), computed on the device (st_angles; metrics.cpp:17-27, 243-259)."""
        y = np.asfortranarray(np.asarray(ref_vectors, np.float64))
        psi = np.zeros(self.k)
        big = C.c_double()
        self._check(lib().st_angles(self._h, y.ctypes.data_as(DP), y.shape[0], _p(psi), C.byref(big)))
        return psi, big.value

    def csr(self, which: int = 0):
        inf = self.info()
        n = inf["n"]
        nnz = {0: inf["nnz_a"], 1: inf["nnz_t"], 2: inf["nnz_delta"]}[which]
        rp = np.zeros(n + 1, np.int32)
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1))
        self._check(lib().st_get_csr(self._h, which, _p(rp, I32P), _p(col, I32P), _p(val)))
        return rp, col[:nnz], val[:nnz]

    def probe_basis(self, upd: Update, basis_kind: str, seed: int) -> np.ndarray:
        keep, s = upd.struct()
        n_total = self.info()["n"] + upd.n_new
        maxc = 2 * self.k + max(upd.n_new, 0) + 512
        z = np.zeros((n_total, maxc), order="F")
        cols = I64()
        self._check(lib().st_probe_basis(self._h, C.byref(s), BASIS[basis_kind], seed, z.ctypes.data_as(DP),
                                         n_total, maxc, C.byref(cols)))
        return np.ascontiguousarray(z[:, : cols.value])

    def probe_rr(self, upd: Update, z: np.ndarray):
        keep, s = upd.struct()
        zf = np.asfortranarray(np.asarray(z, np.float64))
        vals = np.zeros(self.k)
        vecs = np.zeros((z.shape[0], self.k), order="F")
        self._check(lib().st_probe_rr(self._h, C.byref(s), zf.ctypes.data_as(DP), z.shape[0], z.shape[1],
                                      max(z.shape[0], 1), _p(vals), vecs.ctypes.data_as(DP), max(z.shape[0], 1)))
        return vals, np.ascontiguousarray(vecs)

    def timings(self):
        buf = np.zeros(8)
        n = lib().st_last_timings(self._h, _p(buf), 8)
        return buf[:n]

    def launches(self) -> int:
        return int(lib().st_last_launches(self._h))


def sym_eig_dense(s: np.ndarray, order: str = "abs_desc", want: int | None = None, device: int = 0):
    """Device sym_eig_dense (eig.hpp:37-50): eigenvalues of (S + S')/2 in
    spectral order and the leading `want` eigenvectors (columns)."""
    n = s.shape[0]
    want = n if want is None else want
    sf = np.asfortranarray(np.asarray(s, np.float64))
    vals = np.zeros(n)
    vecs = np.zeros((n, max(want, 1)), order="F")
    rc = lib().st_sym_eig_dense(device, n, sf.ctypes.data_as(DP), ORDER[order], want, _p(vals),
                                vecs.ctypes.data_as(DP))
    if rc != ST_OK:
        raise TrackerError(_KINDS.get(rc, "other"), lib().st_last_error(None).decode())
    return vals, np.ascontiguousarray(vecs[:, :want])


def gaussian_matrix(seed: int, rows: int, cols: int, device: int = 0) -> np.ndarray:
    """Device GaussianSampler(seed).gaussian_matrix(rows, cols) (rng.hpp:64-69)."""
    out = np.zeros((rows, cols), order="F")
    rc = lib().st_gaussian_matrix(device, seed, rows, cols, out.ctypes.data_as(DP))
    if rc != ST_OK:
        raise TrackerError(_KINDS.get(rc, "other"), lib().st_last_error(None).decode())
    return np.ascontiguousarray(out)


class DeviceUpdate:
    """An Update whose edit arrays live in HBM (torch CUDA tensors)."""

    def __init__(self, upd: Update, device="cuda"):
        import torch

        def t(x, dt):
            return torch.as_tensor(np.ascontiguousarray(x), dtype=dt).to(device)

        self.tensors = [t(upd.added[0], torch.int64), t(upd.added[1], torch.int64), t(upd.added[2], torch.float64),
                        t(upd.removed[0], torch.int64), t(upd.removed[1], torch.int64),
                        t(upd.new_edges[0], torch.int64), t(upd.new_edges[1], torch.int64),
                        t(upd.new_edges[2], torch.float64)]
        ai, aj, aw, ri, rj, ni, nj, nw = self.tensors

        def ip(x):
            return C.cast(C.c_void_p(x.data_ptr()), I64P)

        def dp(x):
            return C.cast(C.c_void_p(x.data_ptr()), DP)

        self.struct = StUpdate(len(ai), ip(ai), ip(aj), dp(aw), len(ri), ip(ri), ip(rj), int(upd.n_new), len(ni),
                               ip(ni), ip(nj), dp(nw))
