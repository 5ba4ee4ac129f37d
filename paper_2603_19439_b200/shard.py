"""Row-sharded sessions: one TrackerSession per GPU of a box.

The library (csrc/shard.cuh, st_create_sharded) owns the partitioning and the
sharded step; this module supplies the two collectives it calls (st_comm)
through torch.distributed, and splits the initial CSR and eigenvectors into
the contiguous row blocks the ranks start from.

* ``TorchComm("nccl")`` — NCCL allreduce / all_gather_into_tensor enqueued on
  the session's own CUDA stream (torch.cuda.ExternalStream), zero-copy views of
  the library's device buffers (``__cuda_array_interface__``).
* ``TorchComm("staged")`` — the same collectives staged through host memory
  over the default (e.g. gloo) process group: for tests that run several ranks
  on one GPU, where no rank's kernels ever wait on another's.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                           C.POINTER(C.c_int64), C.c_void_p)


class StComm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("size", C.c_int32), ("ctx", C.c_void_p),
                ("allreduce_sum_f64", ALLREDUCE_FN), ("allgather", ALLGATHER_FN), ("alltoallv", ALLTOALLV_FN)]


class _DevBuf:
    """Zero-copy torch view of library device memory."""

    def __init__(self, ptr: int, nbytes: int, typestr: str, itemsize: int):
        self.__cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None,
                                         "stream": None}


def _view(ptr, count, dtype):
    import torch

    typestr, itemsize = {torch.float64: ("<f8", 8), torch.uint8: ("|u1", 1)}[dtype]
    return torch.as_tensor(_DevBuf(ptr, count * itemsize, typestr, itemsize), device="cuda")


class TorchComm:
    """st_comm over the default torch.distributed process group."""

    def __init__(self, mode: str = "nccl", group=None):
        import torch.distributed as dist

        assert mode in ("nccl", "staged")
        self.mode = mode
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.calls = {"allreduce": 0, "allgather": 0, "alltoallv": 0, "bytes": 0, "host_s": 0.0}
        self._ar = ALLREDUCE_FN(self._allreduce)
        self._ag = ALLGATHER_FN(self._allgather)
        self._a2a = ALLTOALLV_FN(self._alltoallv)
        self.struct = StComm(self.rank, self.size, None, self._ar, self._ag, self._a2a)

    def _allreduce(self, ctx, buf, count, stream):
        t0 = time.perf_counter()
        try:
            import torch
            import torch.distributed as dist

            if count <= 0:
                return 0
            t = _view(buf, count, torch.float64)
            ext = torch.cuda.ExternalStream(stream)
            self.calls["allreduce"] += 1
            self.calls["bytes"] += 8 * count
            if self.mode == "nccl":
                with torch.cuda.stream(ext):
                    dist.all_reduce(t, group=self.group)
            else:
                ext.synchronize()
                h = t.cpu()
                dist.all_reduce(h, group=self.group)
                with torch.cuda.stream(ext):
                    t.copy_(h)
                ext.synchronize()
            self.calls["host_s"] += time.perf_counter() - t0
            return 0
        except Exception as e:  # a failed collective must not unwind through C
            print(f"[rank {self.rank}] st_comm allreduce failed: {e!r}", flush=True)
            return 1

    def _allgather(self, ctx, send, recv, nbytes, stream):
        t0 = time.perf_counter()
        try:
            import torch
            import torch.distributed as dist

            if nbytes <= 0:
                return 0
            s = _view(send, nbytes, torch.uint8)
            r = _view(recv, nbytes * self.size, torch.uint8)
            ext = torch.cuda.ExternalStream(stream)
            self.calls["allgather"] += 1
            self.calls["bytes"] += nbytes * self.size
            if self.mode == "nccl":
                with torch.cuda.stream(ext):
                    dist.all_gather_into_tensor(r, s, group=self.group)
            else:
                ext.synchronize()
                hs = s.cpu()
                parts = [torch.empty_like(hs) for _ in range(self.size)]
                dist.all_gather(parts, hs, group=self.group)
                h = torch.cat(parts)
                with torch.cuda.stream(ext):
                    r.copy_(h)
                ext.synchronize()
            self.calls["host_s"] += time.perf_counter() - t0
            return 0
        except Exception as e:
            print(f"[rank {self.rank}] st_comm allgather failed: {e!r}", flush=True)
            return 1


    def _alltoallv(self, ctx, send, send_bytes, recv, recv_bytes, stream):
        t0 = time.perf_counter()
        try:
            import torch
            import torch.distributed as dist

            sb = [int(send_bytes[r]) for r in range(self.size)]
            rb = [int(recv_bytes[r]) for r in range(self.size)]
            if sum(sb) == 0 and sum(rb) == 0 and self.mode == "nccl":
                return 0
            s = _view(send, max(sum(sb), 1), torch.uint8)[: sum(sb)] if sum(sb) else torch.empty(
                0, dtype=torch.uint8, device="cuda")
            r = _view(recv, max(sum(rb), 1), torch.uint8)[: sum(rb)] if sum(rb) else torch.empty(
                0, dtype=torch.uint8, device="cuda")
            ext = torch.cuda.ExternalStream(stream)
            self.calls["alltoallv"] += 1
            self.calls["bytes"] += sum(rb)
            if self.mode == "nccl":
                with torch.cuda.stream(ext):
                    dist.all_to_all_single(r, s, output_split_sizes=rb, input_split_sizes=sb, group=self.group)
            else:
                ext.synchronize()
                hs = s.cpu()
                hr = torch.empty(sum(rb), dtype=torch.uint8)
                dist.all_to_all_single(hr, hs, output_split_sizes=rb, input_split_sizes=sb, group=self.group)
                if sum(rb):
                    with torch.cuda.stream(ext):
                        r.copy_(hr)
                    ext.synchronize()
            self.calls["host_s"] += time.perf_counter() - t0
            return 0
        except Exception as e:
            print(f"[rank {self.rank}] st_comm alltoallv failed: {e!r}", flush=True)
            return 1


class NcclComm:
    """The library's own st_comm over NCCL (st_comm_nccl_create): rank 0 draws
    the unique id, torch.distributed carries it to the other ranks, and every
    collective of the sharded step is then enqueued by the library itself on
    the session stream (no Python on the data path)."""

    def __init__(self, device: int = 0, group=None):
        import torch.distributed as dist

        from . import ST_OK, TrackerError, _KINDS, lib

        L = lib()
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        uid = C.create_string_buffer(128)
        if self.rank == 0 and L.st_nccl_unique_id(uid) != ST_OK:
            raise TrackerError("cuda", L.st_last_error(None).decode())
        box = [bytes(uid.raw)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = C.create_string_buffer(box[0], 128)
        self.struct = StComm()
        rc = L.st_comm_nccl_create(uid, self.rank, self.size, device, C.byref(self.struct))
        if rc != ST_OK:
            raise TrackerError(_KINDS.get(rc, "other"), L.st_last_error(None).decode())
        self.calls = {"native": 1}

    def close(self):
        from . import lib

        if getattr(self, "struct", None) is not None and self.struct.ctx:
            lib().st_comm_nccl_destroy(C.byref(self.struct))

    def __del__(self):
        self.close()


def shard_bounds(rowptr, size: int) -> np.ndarray:
    """Contiguous row blocks with balanced (degree + 1) weight: the rows of P a
    step touches are drawn about in proportion to degree (edge deletions,
    preferential attachment), the X passes in proportion to rows."""
    rowptr = np.asarray(rowptr, np.int64)
    n = len(rowptr) - 1
    w = rowptr + np.arange(n + 1)  # cumulative (nnz + rows)
    cuts = [0]
    for r in range(1, size):
        cuts.append(int(np.searchsorted(w, w[-1] * r / size)))
    cuts.append(n)
    return np.maximum.accumulate(np.asarray(cuts, np.int64))


def layout(bounds, chunk: int, rank: int, n_total: int) -> np.ndarray:
    """Global ids (ascending) of the rows `rank` owns at n_total nodes (the
    library's closed-form map, st_shard_layout)."""
    from . import I64P, lib

    b = np.ascontiguousarray(bounds, np.int64)
    cap = int(n_total) + 1
    out = np.zeros(cap, np.int64)
    rows = lib().st_shard_layout(len(b) - 1, b.ctypes.data_as(I64P), chunk, rank, n_total,
                                 out.ctypes.data_as(I64P), cap)
    if rows < 0:
        raise ValueError("st_shard_layout: bad arguments")
    return out[:rows]


def local_block(rowptr, col, val, vectors, lo: int, hi: int):
    """CSR rows [lo, hi) (global column ids) and the same rows of X."""
    rowptr = np.asarray(rowptr, np.int64)
    s, e = int(rowptr[lo]), int(rowptr[hi])
    rp = (rowptr[lo:hi + 1] - s).astype(np.int32)
    return rp, np.asarray(col[s:e], np.int32), np.asarray(val[s:e], np.float64), np.asarray(vectors)[lo:hi]


class ShardedTrackerSession:
    """The rows [lo, hi) of a row-sharded tracker (one per rank)."""

    def __init__(self, comm: TorchComm, n_global: int, lo: int, hi: int, rowptr, col, val, values, vectors,
                 kind="grest-rsvd", k=None, order="abs_desc", rsvd_l=100, rsvd_p=100, seed=0, device=0,
                 chunk: int = 256, force_dense=False, kernel_timing=False):
        from . import (DP, FLAG_FORCE_DENSE, FLAG_KERNEL_TIMING, I32P, KIND, ORDER, ST_OK, StConfig, TrackerError,
                       _KINDS, _d, _p, lib)

        L = lib()
        rowptr = np.ascontiguousarray(rowptr, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        values = _d(values)
        vectors = np.asfortranarray(np.asarray(vectors, np.float64).reshape(hi - lo, -1))
        k = len(values) if k is None else k
        flags = (FLAG_FORCE_DENSE if force_dense else 0) | (FLAG_KERNEL_TIMING if kernel_timing else 0)
        cfg = StConfig(KIND[kind], 0, k, ORDER[order], rsvd_l, rsvd_p, seed, device, flags)
        self.comm = comm  # keeps the callbacks alive
        h = C.c_void_p()
        rc = L.st_create_sharded(C.byref(cfg), C.byref(comm.struct), n_global, lo, hi, chunk, _p(rowptr, I32P),
                                 _p(col, I32P), _p(val), _p(values), vectors.ctypes.data_as(DP),
                                 max(vectors.shape[0], 1), C.byref(h))
        if rc != ST_OK:
            raise TrackerError(_KINDS.get(rc, "other"), L.st_last_error(None).decode())
        self._h = h.value
        self.k = k
        self.chunk = chunk

    # the session API of TrackerSession, on the owned rows
    from . import TrackerSession as _T

    close = _T.close
    __del__ = _T.__del__
    _check = _T._check
    step = _T.step
    step_device = _T.step_device
    reserve = _T.reserve
    info = _T.info
    values = _T.values
    launches = _T.launches
    kernel_stats = _T.kernel_stats
    set_peaks = _T.set_peaks
    reset_kernel_stats = _T.reset_kernel_stats
    del _T

    def halo_stats(self) -> dict:
        """Boundary-row halo traffic since creation (st_shard_stats)."""
        from . import I64P, lib

        r, l_, h = C.c_int64(), C.c_int64(), C.c_int64()
        lib().st_shard_stats(self._h, C.byref(r), C.byref(l_), C.byref(h))
        return {"halo_bytes_recv": r.value, "halo_bytes_local": l_.value, "halos": h.value}

    def rows(self) -> np.ndarray:
        from . import I64P, lib

        n = C.c_int64()
        self._check(lib().st_shard_rows(self._h, C.byref(n), None))
        ids = np.zeros(max(n.value, 1), np.int64)
        self._check(lib().st_shard_rows(self._h, C.byref(n), ids.ctypes.data_as(I64P)))
        return ids[: n.value]

    def embedding(self):
        """(values, owned rows of X, their global ids)."""
        from . import DP, _p, lib

        ids = self.rows()
        vals = np.zeros(self.k)
        vecs = np.zeros((max(len(ids), 1), self.k), order="F")
        self._check(lib().st_get_embedding(self._h, _p(vals), vecs.ctypes.data_as(DP), max(len(ids), 1)))
        return vals, np.ascontiguousarray(vecs[: len(ids)]), ids

    def csr(self, which: int = 0):
        """which=0: owned rows of A (global columns, row order = rows());
        which=2: the full perturbation of the last step."""
        from . import I32P, _p, lib

        inf = self.info()
        nrows = len(self.rows()) if which == 0 else inf["n"]
        nnz = {0: inf["nnz_a"], 2: inf["nnz_delta"]}[which]
        rp = np.zeros(nrows + 1, np.int32)
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1))
        self._check(lib().st_get_csr(self._h, which, _p(rp, I32P), _p(col, I32P), _p(val)))
        return rp, col[:nnz], val[:nnz]
