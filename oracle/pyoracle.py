"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the CPU restatement (liboracle.so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
leg may import this module; the product path (paper_2603_19439_b200) never does.
The restatement follows /root/reference/proj (see spectrack_oracle.hpp for the
per-function file:line citations).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

I64 = C.c_int64
U64 = C.c_uint64
DP = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
ERRLEN = 1024


class OracleError(Exception):
    """Raised with the reference exception category: ``kind`` is
    'invalid_argument' or 'runtime_error' (std exceptions of the reference)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


def build() -> str:
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.or_mix_seed.restype = U64
        _lib.or_mix_seed.argtypes = [U64, U64]
        _lib.or_mix_seed3.restype = U64
        _lib.or_mix_seed3.argtypes = [U64, U64, U64]
        _lib.or_subspace_sin.restype = C.c_double
        _lib.or_session_csr.restype = C.c_void_p
        _lib.or_session_csr.argtypes = [C.c_void_p, C.c_int]
        for name in ("or_csr_info", "or_csr_copy", "or_csr_free", "or_mat_info", "or_mat_copy", "or_mat_free",
                     "or_session_destroy", "or_session_info", "or_session_embedding"):
            getattr(_lib, name).restype = None
    return _lib


def _p(a, t=DP):
    return a.ctypes.data_as(t) if a is not None else None


def _check(rc: int, err) -> None:
    if rc == 0:
        return
    msg = err.value.decode()
    raise OracleError({1: "invalid_argument", 2: "runtime_error"}.get(rc, "other"), msg)


@dataclass
class Csr:
    """Compressed-row symmetric matrix (int32 offsets/indices, fp64 values),
    the layout of Eigen::SparseMatrix<double, RowMajor> (sparse.hpp:18)."""
    n: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.rowptr))
        d[rows, self.col] = self.val
        return d

    def coeff(self, i: int, j: int) -> float:
        s, e = self.rowptr[i], self.rowptr[i + 1]
        k = np.searchsorted(self.col[s:e], j)
        if k < e - s and self.col[s + k] == j:
            return float(self.val[s + k])
        return 0.0

    def equal(self, other: "Csr") -> bool:
        return (self.n == other.n and np.array_equal(self.rowptr, other.rowptr)
                and np.array_equal(self.col, other.col) and np.array_equal(self.val, other.val))


def _csr_out(h) -> Csr:
    L = lib()
    rows, nnz = I64(), I64()
    L.or_csr_info(C.c_void_p(h), C.byref(rows), C.byref(nnz))
    rp = np.zeros(rows.value + 1, np.int32)
    col = np.zeros(max(nnz.value, 1), np.int32)
    val = np.zeros(max(nnz.value, 1), np.float64)
    L.or_csr_copy(C.c_void_p(h), _p(rp, I32P), _p(col, I32P), _p(val))
    L.or_csr_free(C.c_void_p(h))
    return Csr(rows.value, rp, col[: nnz.value], val[: nnz.value])


def _mat_out(h) -> np.ndarray:
    L = lib()
    r, c = I64(), I64()
    L.or_mat_info(C.c_void_p(h), C.byref(r), C.byref(c))
    out = np.zeros(r.value * c.value)
    L.or_mat_copy(C.c_void_p(h), _p(out))
    L.or_mat_free(C.c_void_p(h))
    return out.reshape(c.value, r.value).T.copy()  # column-major -> numpy


def _f(a):  # numpy (rows x cols) -> column-major contiguous buffer
    return np.asfortranarray(np.asarray(a, np.float64)).ravel(order="F")


# ------------------------------------------------------------------ rng / dense
def mix_seed(base: int, salt: int, salt2: int | None = None) -> int:
    if salt2 is None:
        return int(lib().or_mix_seed(base, salt))
    return int(lib().or_mix_seed3(base, salt, salt2))


def mt_raw(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    lib().or_mt_raw(U64(seed), I64(count), _p(out, C.POINTER(C.c_uint64)))
    return out


def gaussian_matrix(seed: int, rows: int, cols: int) -> np.ndarray:
    out = np.zeros(rows * cols)
    lib().or_gaussian_matrix(U64(seed), I64(rows), I64(cols), _p(out))
    return out.reshape(cols, rows).T.copy()


def spectral_sort(values, order: int) -> np.ndarray:
    v = np.ascontiguousarray(values, np.float64)
    perm = np.zeros(len(v), np.int64)
    lib().or_spectral_sort(I64(len(v)), _p(v), C.c_int(order), _p(perm, I64P))
    return perm


def sym_eig(s: np.ndarray, order: int):
    n = s.shape[0]
    if s.shape[0] != s.shape[1]:
        raise OracleError("invalid_argument", "sym_eig_dense: matrix must be square")
    buf = _f(s)
    w = np.zeros(n)
    v = np.zeros(n * n)
    err = C.create_string_buffer(ERRLEN)
    _check(lib().or_sym_eig(I64(n), _p(buf), C.c_int(order), _p(w), _p(v), err, ERRLEN), err)
    return w, v.reshape(n, n).T.copy()


def orthonormalize(m: np.ndarray, against: np.ndarray | None = None, tol: float = 1e-10) -> np.ndarray:
    err = C.create_string_buffer(ERRLEN)
    h = C.c_void_p()
    rows, cols = m.shape
    if against is not None and against.shape[1] > 0 and against.shape[0] != rows:
        buf, ab = _f(m), _f(against)
        _check(lib().or_orthonormalize_shape_check(I64(rows), I64(cols), _p(buf), I64(against.shape[0]),
                                                   I64(against.shape[1]), _p(ab), err, ERRLEN), err)
    acols = 0 if against is None else against.shape[1]
    ab = _f(against) if acols else None
    _check(lib().or_orthonormalize(I64(rows), I64(cols), _p(_f(m)), I64(acols), _p(ab), C.c_double(tol),
                                   C.byref(h), err, ERRLEN), err)
    return _mat_out(h.value)


def rsvd_dense(b: np.ndarray, l: int, p: int, seed: int) -> np.ndarray:
    err = C.create_string_buffer(ERRLEN)
    h = C.c_void_p()
    _check(lib().or_rsvd_dense(I64(b.shape[0]), I64(b.shape[1]), _p(_f(b)), I64(l), I64(p), U64(seed), C.byref(h),
                               err, ERRLEN), err)
    return _mat_out(h.value)


def subspace_sin(a: np.ndarray, b: np.ndarray) -> float:
    L = lib()
    L.or_subspace_sin.argtypes = [I64, I64, DP, I64, DP]
    return float(L.or_subspace_sin(a.shape[0], a.shape[1], _p(_f(a)), b.shape[1], _p(_f(b))))


def lanczos(a: Csr, k: int, order: int = 0, seed: int = 0, tol: float = 1e-10, max_basis: int = 0):
    err = C.create_string_buffer(ERRLEN)
    vals = np.zeros(k)
    vecs = np.zeros(a.n * k)
    _check(lib().or_lanczos(I64(a.n), _p(a.rowptr, I32P), _p(a.col, I32P), _p(a.val), I64(k), C.c_int(order),
                            U64(seed), C.c_double(tol), I64(max_basis), _p(vals), _p(vecs), err, ERRLEN), err)
    return vals, vecs.reshape(k, a.n).T.copy()


# ------------------------------------------------------------------ graph
def _i64(x):
    return np.ascontiguousarray(np.asarray(x, np.int64).reshape(-1))


def _d(x):
    return np.ascontiguousarray(np.asarray(x, np.float64).reshape(-1))


def _edges3(edges):
    if len(edges) == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float64)
    if isinstance(edges, tuple) and len(edges) == 3 and hasattr(edges[0], "__len__"):
        return _i64(edges[0]), _i64(edges[1]), _d(edges[2])
    e = list(edges)
    return _i64([t[0] for t in e]), _i64([t[1] for t in e]), _d([t[2] if len(t) > 2 else 1.0 for t in e])


def _edges2(edges):
    if len(edges) == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    if isinstance(edges, tuple) and len(edges) == 2 and hasattr(edges[0], "__len__"):
        return _i64(edges[0]), _i64(edges[1])
    e = list(edges)
    return _i64([t[0] for t in e]), _i64([t[1] for t in e])


@dataclass
class Update:
    """Edit lists of one step, the arguments of assemble_update (graph.hpp:65-69):
    added (i, j, w) and removed (i, j) among existing nodes, ``n_new`` appended
    nodes, and new_edges (i, j, w) touching at least one appended node."""
    added: tuple = ((), (), ())
    removed: tuple = ((), ())
    n_new: int = 0
    new_edges: tuple = ((), (), ())

    @staticmethod
    def make(added=(), removed=(), n_new=0, new_edges=()):
        return Update(_edges3(added), _edges2(removed), int(n_new), _edges3(new_edges))

    def args(self):
        ai, aj, aw = (_i64(self.added[0]), _i64(self.added[1]), _d(self.added[2]))
        ri, rj = (_i64(self.removed[0]), _i64(self.removed[1]))
        ni, nj, nw = (_i64(self.new_edges[0]), _i64(self.new_edges[1]), _d(self.new_edges[2]))
        keep = (ai, aj, aw, ri, rj, ni, nj, nw)
        return keep, [I64(len(ai)), _p(ai, I64P), _p(aj, I64P), _p(aw), I64(len(ri)), _p(ri, I64P), _p(rj, I64P),
                      I64(self.n_new), I64(len(ni)), _p(ni, I64P), _p(nj, I64P), _p(nw)]


def from_edges(n: int, edges) -> Csr:
    i, j, w = _edges3(edges)
    err = C.create_string_buffer(ERRLEN)
    h = C.c_void_p()
    _check(lib().or_from_edges(I64(n), I64(len(i)), _p(i, I64P), _p(j, I64P), _p(w), C.byref(h), err, ERRLEN), err)
    return _csr_out(h.value)


def from_triplets(n: int, trips) -> Csr:
    i, j, v = _edges3(trips)
    err = C.create_string_buffer(ERRLEN)
    h = C.c_void_p()
    _check(lib().or_from_triplets(I64(n), I64(len(i)), _p(i, I64P), _p(j, I64P), _p(v), C.byref(h), err, ERRLEN),
           err)
    return _csr_out(h.value)


def update_delta(n_old: int, upd: Update) -> Csr:
    keep, a = Update(upd.added, upd.removed, upd.n_new, upd.new_edges).args()
    err = C.create_string_buffer(ERRLEN)
    h = C.c_void_p()
    _check(lib().or_update_delta(I64(n_old), *a, C.byref(h), err, ERRLEN), err)
    return _csr_out(h.value)


def apply_update(a: Csr, upd: Update, n_old: int | None = None) -> Csr:
    keep, args = Update(upd.added, upd.removed, upd.n_new, upd.new_edges).args()
    err = C.create_string_buffer(ERRLEN)
    h = C.c_void_p()
    _check(lib().or_apply_update(I64(a.n), _p(a.rowptr, I32P), _p(a.col, I32P), _p(a.val), *args,
                                 I64(-1 if n_old is None else n_old), C.byref(h), err, ERRLEN), err)
    return _csr_out(h.value)


def shifted_laplacian(a: Csr, kind: int, alpha: float):
    err = C.create_string_buffer(ERRLEN)
    h = C.c_void_p()
    warned = C.c_int(0)
    _check(lib().or_shifted_laplacian(I64(a.n), _p(a.rowptr, I32P), _p(a.col, I32P), _p(a.val), C.c_int(kind),
                                      C.c_double(alpha), C.byref(warned), C.byref(h), err, ERRLEN), err)
    return _csr_out(h.value), bool(warned.value)


# ------------------------------------------------------------------ sessions
KIND = {"trip-basic": 0, "trip": 1, "rm": 2, "iasc": 3, "grest2": 4, "grest3": 5, "grest-rsvd": 6, "timers": 7}
OPERATOR = {"adjacency": 0, "laplacian": 1, "normalized-laplacian": 2}
ORDER = {"abs_desc": 0, "alg_desc": 1}


class Session:
    """One tracker lane of the reference per-step loop (experiment.cpp:165-205):
    assemble_update -> (apply_update | ShiftedLaplacianSession::advance) ->
    tracker_step, transactional on error like the reference's value semantics."""

    def __init__(self, a: Csr, kind="grest-rsvd", k=8, order="abs_desc", rsvd_l=100, rsvd_p=100, seed=0,
                 operator="adjacency", values=None, vectors=None, mu=0.0, trip_replace_span=False, theta=0.01,
                 min_restart_gap=5, restart_inner="iasc"):
        err = C.create_string_buffer(ERRLEN)
        h = C.c_void_p()
        vals = None if values is None else _d(values)
        vecs = None if vectors is None else _f(vectors)
        _check(lib().or_session_create(C.c_int(KIND[kind]), C.c_int(OPERATOR[operator]), I64(k),
                                       C.c_int(ORDER[order]), I64(rsvd_l), I64(rsvd_p), U64(seed), I64(a.n),
                                       _p(a.rowptr, I32P), _p(a.col, I32P), _p(a.val), _p(vals), _p(vecs),
                                       C.byref(h), err, ERRLEN), err)
        self._h = h.value
        self.last_tracker_seconds = 0.0
        L = lib()
        L.or_session_set_options.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_double, I64, C.c_int,
                                             C.c_char_p, C.c_int]
        _check(L.or_session_set_options(C.c_void_p(self._h), C.c_double(mu), C.c_int(int(trip_replace_span)),
                                        C.c_double(theta), I64(min_restart_gap), C.c_int(KIND[restart_inner]),
                                        err, ERRLEN), err)

    def tracker_stats(self):
        """(accumulated_change, steps_since_restart, restart_scale, ridge_used) of the TrackerState."""
        L = lib()
        acc, gap, scale, ridge = C.c_double(), I64(), C.c_double(), C.c_int()
        L.or_session_tracker_stats(C.c_void_p(self._h), C.byref(acc), C.byref(gap), C.byref(scale), C.byref(ridge))
        return acc.value, gap.value, scale.value, bool(ridge.value)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_session_destroy(C.c_void_p(self._h))
            self._h = None

    def info(self):
        n, k, st, alpha = I64(), I64(), U64(), C.c_double()
        lib().or_session_info(C.c_void_p(self._h), C.byref(n), C.byref(k), C.byref(st), C.byref(alpha))
        return n.value, k.value, st.value, alpha.value

    def step(self, upd: Update) -> None:
        keep, args = Update(upd.added, upd.removed, upd.n_new, upd.new_edges).args()
        err = C.create_string_buffer(ERRLEN)
        secs = C.c_double(0)
        _check(lib().or_session_step(C.c_void_p(self._h), *args, C.byref(secs), err, ERRLEN), err)
        self.last_tracker_seconds = secs.value

    def embedding(self):
        n, k, _, _ = self.info()
        vals = np.zeros(k)
        vecs = np.zeros(n * k)
        lib().or_session_embedding(C.c_void_p(self._h), _p(vals), _p(vecs))
        return vals, vecs.reshape(k, n).T.copy()

    def csr(self, which: int = 0) -> Csr:
        return _csr_out(lib().or_session_csr(C.c_void_p(self._h), C.c_int(which)))

    def probe_basis(self, upd: Update, basis_kind: str, seed: int) -> np.ndarray:
        keep, args = Update(upd.added, upd.removed, upd.n_new, upd.new_edges).args()
        err = C.create_string_buffer(ERRLEN)
        h = C.c_void_p()
        bk = {"iasc": 0, "grest2": 1, "grest3": 2, "grest-rsvd": 3}[basis_kind]
        _check(lib().or_session_probe_basis(C.c_void_p(self._h), C.c_int(bk), U64(seed), *args, C.byref(h), err,
                                            ERRLEN), err)
        return _mat_out(h.value)

    def probe_rr(self, upd: Update, z: np.ndarray):
        keep, args = Update(upd.added, upd.removed, upd.n_new, upd.new_edges).args()
        err = C.create_string_buffer(ERRLEN)
        h = C.c_void_p()
        _, k, _, _ = self.info()
        vals = np.zeros(k)
        _check(lib().or_session_probe_rr(C.c_void_p(self._h), I64(z.shape[0]), I64(z.shape[1]), _p(_f(z)), *args,
                                         _p(vals), C.byref(h), err, ERRLEN), err)
        return vals, _mat_out(h.value)
