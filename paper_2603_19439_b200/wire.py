"""ctypes binding of libspectrack_stream.so (include/spectrack_stream.h): the
stream generators and the binary update-batch wire format.

A loaded or generated stream converts to `streams.Stream` (start graph +
`Update` edit lists of assemble_update, graph.hpp:65-69), the form the C ABI
(`TrackerSession.step`) and the CPU oracle both consume.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import Update
from .streams import SHIFT, Stream

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
F64P = C.POINTER(C.c_double)


class StreamError(Exception):
    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


def lib():
    global _LIB
    if _LIB is None:
        from . import _build

        path = _build.build_stream()
        L = C.CDLL(path)
        H = C.c_void_p
        HP = C.POINTER(C.c_void_p)
        L.sts_last_error.restype = C.c_char_p
        L.sts_free.argtypes = [H]
        L.sts_sbm_sample_graph.argtypes = [C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_uint64, HP]
        L.sts_sbm_dynamic.argtypes = [C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64,
                                      C.c_uint64, HP]
        L.sts_scenario1.argtypes = [C.c_int64, I64P, I64P, C.c_int64, C.c_int64, HP]
        L.sts_scenario2.argtypes = [C.c_int64, I64P, I64P, I64P, C.c_int64, C.c_int64, C.c_int64, HP]
        L.sts_config.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_uint64, HP]
        L.sts_save.argtypes = [H, C.c_char_p]
        L.sts_load.argtypes = [C.c_char_p, HP]
        L.sts_create.argtypes = [C.c_int64, I64P, I64P, F64P, C.c_int64, C.c_char_p, HP]
        L.sts_append.argtypes = [H, C.c_int64, I64P, I64P, F64P, C.c_int64, I64P, I64P, C.c_int64, I64P, I64P, F64P,
                                 C.c_int64]
        for f in ("sts_n0", "sts_m0", "sts_steps", "sts_node_count"):
            getattr(L, f).argtypes = [H]
            getattr(L, f).restype = C.c_int64
        L.sts_name.argtypes = [H]
        L.sts_name.restype = C.c_char_p
        L.sts_initial.argtypes = [H, I64P, I64P, F64P]
        L.sts_initial_csr.argtypes = [H, I32P, I32P, F64P]
        L.sts_update_sizes.argtypes = [H, C.c_int64] + [I64P] * 5
        L.sts_update.argtypes = [H, C.c_int64, I64P, I64P, F64P, I64P, I64P, I64P, I64P, F64P]
        L.sts_node_origin.argtypes = [H, I64P]
        L.sts_labels.argtypes = [H, I32P]
        _LIB = L
    return _LIB


def _p(a, t=F64P):
    return a.ctypes.data_as(t)


def _check(rc):
    if rc != 0:
        raise StreamError("invalid_argument" if rc == 1 else "io", lib().sts_last_error().decode())


class WireStream:
    """Owning handle of one stream in the library."""

    def __init__(self, handle: int):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib().sts_free(self._h)
            self._h = None

    @property
    def n0(self) -> int:
        return lib().sts_n0(self._h)

    @property
    def steps(self) -> int:
        return lib().sts_steps(self._h)

    @property
    def name(self) -> str:
        return lib().sts_name(self._h).decode()

    def initial_edges(self):
        m = lib().sts_m0(self._h)
        i, j, w = np.zeros(m, np.int64), np.zeros(m, np.int64), np.zeros(m)
        lib().sts_initial(self._h, _p(i, I64P), _p(j, I64P), _p(w))
        return i, j, w

    def csr0(self):
        """The initial graph as symmetric CSR (int32 / int32 / fp64, sorted columns)."""
        m = lib().sts_m0(self._h)
        rp = np.zeros(self.n0 + 1, np.int32)
        col, val = np.zeros(2 * m, np.int32), np.zeros(2 * m)
        _check(lib().sts_initial_csr(self._h, _p(rp, I32P), _p(col, I32P), _p(val)))
        nnz = int(rp[-1])
        return rp, col[:nnz], val[:nnz]

    def update(self, t: int) -> Update:
        s = [C.c_int64() for _ in range(5)]
        _check(lib().sts_update_sizes(self._h, t, *[C.byref(x) for x in s]))
        _, n_new, na, nr, nn = (x.value for x in s)
        ai, aj, aw = np.zeros(na, np.int64), np.zeros(na, np.int64), np.zeros(na)
        ri, rj = np.zeros(nr, np.int64), np.zeros(nr, np.int64)
        ni, nj, nw = np.zeros(nn, np.int64), np.zeros(nn, np.int64), np.zeros(nn)
        _check(lib().sts_update(self._h, t, _p(ai, I64P), _p(aj, I64P), _p(aw), _p(ri, I64P), _p(rj, I64P),
                                _p(ni, I64P), _p(nj, I64P), _p(nw)))
        return Update((ai, aj, aw), (ri, rj), int(n_new), (ni, nj, nw))

    def n_old(self, t: int) -> int:
        s = [C.c_int64() for _ in range(5)]
        _check(lib().sts_update_sizes(self._h, t, *[C.byref(x) for x in s]))
        return s[0].value

    def node_origin(self):
        n = lib().sts_node_count(self._h)
        o = np.zeros(n, np.int64)
        if n:
            lib().sts_node_origin(self._h, _p(o, I64P))
        return o

    def labels(self):
        n = lib().sts_node_count(self._h)
        o = np.zeros(n, np.int32)
        if n:
            lib().sts_labels(self._h, _p(o, I32P))
        return o

    def save(self, path: str) -> None:
        _check(lib().sts_save(self._h, path.encode()))

    def to_stream(self) -> Stream:
        """As a streams.Stream (unit-weight initial edges as undirected keys)."""
        i, j, w = self.initial_edges()
        if len(w) and not np.all(w == 1.0):
            raise ValueError("to_stream: the initial graph has non-unit weights (use csr0())")
        keys = np.sort(np.minimum(i, j) * SHIFT + np.maximum(i, j))
        return Stream(self.n0, keys, [self.update(t) for t in range(self.steps)], name=self.name)


def _make(fn, *args) -> WireStream:
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return WireStream(h.value)


def load(path: str) -> WireStream:
    return _make(lib().sts_load, path.encode())


def config(which: int, size: int = 0, steps: int = 0, seed: int = 0) -> WireStream:
    """BASELINE config `which` (1..5); size = n (cfg1/2/4) or R-MAT scale (cfg3/5), 0 = stated."""
    return _make(lib().sts_config, which, size, steps, seed)


def sbm_sample_graph(n, k_clusters, p_in, p_out, seed) -> WireStream:
    return _make(lib().sts_sbm_sample_graph, n, k_clusters, p_in, p_out, seed)


def sbm_dynamic(n, k_clusters, p_in, p_out, n0, t_steps, s_per_step, seed) -> WireStream:
    return _make(lib().sts_sbm_dynamic, n, k_clusters, p_in, p_out, n0, t_steps, s_per_step, seed)


def scenario1(n, edges, t_steps) -> WireStream:
    e = np.asarray(edges, np.int64).reshape(-1, 2)
    i, j = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
    return _make(lib().sts_scenario1, n, _p(i, I64P), _p(j, I64P), len(i), t_steps)


def scenario2(n, timed_edges, t_steps, m0) -> WireStream:
    e = np.asarray(timed_edges, np.int64).reshape(-1, 3)
    u, v, t = (np.ascontiguousarray(e[:, c]) for c in range(3))
    return _make(lib().sts_scenario2, n, _p(u, I64P), _p(v, I64P), _p(t, I64P), len(u), t_steps, m0)


def from_stream(s: Stream) -> WireStream:
    """A streams.Stream (e.g. the numpy generators) as a wire stream, to be saved."""
    keys = np.asarray(s.keys0, np.int64)
    i, j = np.ascontiguousarray(keys // SHIFT), np.ascontiguousarray(keys % SHIFT)
    w = np.ones(len(i))
    ws = _make(lib().sts_create, s.n0, _p(i, I64P), _p(j, I64P), _p(w), len(i), s.name.encode())
    for u in s.updates:
        ai, aj, aw = (np.ascontiguousarray(u.added[c], np.int64 if c < 2 else np.float64) for c in range(3))
        ri, rj = (np.ascontiguousarray(u.removed[c], np.int64) for c in range(2))
        ni, nj, nw = (np.ascontiguousarray(u.new_edges[c], np.int64 if c < 2 else np.float64) for c in range(3))
        _check(lib().sts_append(ws._h, int(u.n_new), _p(ai, I64P), _p(aj, I64P), _p(aw), len(ai), _p(ri, I64P),
                                _p(rj, I64P), len(ri), _p(ni, I64P), _p(nj, I64P), _p(nw), len(ni)))
    return ws
