"""Seeded synthetic graph streams for the BASELINE configs (harness, numpy only).

The reference ships paper protocols (proj/src/dynamics.cpp) but no generators
for the BASELINE configs (equal-block SBM, Erdos-Renyi, R-MAT, preferential
attachment with deletions), so these are new. Every stream is a start graph
plus a list of update batches in the edit-list form of assemble_update
(proj/include/spectrack/graph.hpp:65-69); the CUDA path and the CPU oracle
consume the identical batches.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import Update

SHIFT = np.int64(1 << 32)


def _keys(u, v):
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    return lo.astype(np.int64) * SHIFT + hi.astype(np.int64)


def _unkey(k):
    return (k // SHIFT).astype(np.int64), (k % SHIFT).astype(np.int64)


def csr_from_keys(n: int, keys: np.ndarray, weights: np.ndarray | None = None):
    """Symmetric CSR (both triangles, sorted columns) from undirected pair keys."""
    u, v = _unkey(keys)
    w = np.ones(len(keys)) if weights is None else weights
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    vals = np.concatenate([w, w])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rowptr[1:])
    return rowptr.astype(np.int32), cols.astype(np.int32), vals.astype(np.float64)


def _sample_pairs_block(rng, lo_a, size_a, lo_b, size_b, p, same):
    """Bernoulli(p) pairs between two node blocks (i < j inside one block)."""
    total = size_a * (size_a - 1) // 2 if same else size_a * size_b
    if total == 0 or p <= 0:
        return np.zeros(0, np.int64)
    m = rng.binomial(total, p)
    idx = np.unique(rng.integers(0, total, size=int(m * 1.02) + 16))
    while len(idx) < m:
        idx = np.unique(np.concatenate([idx, rng.integers(0, total, size=m - len(idx) + 16)]))
    idx = rng.permutation(idx)[:m]
    if same:
        # row-major upper-triangle index -> (i, j), i < j
        i = (size_a - 2 - np.floor(np.sqrt(-8.0 * idx + 4.0 * size_a * (size_a - 1) - 7) / 2.0 - 0.5)).astype(np.int64)
        j = idx + i + 1 - size_a * (size_a - 1) // 2 + (size_a - i) * ((size_a - i) - 1) // 2
        return _keys(lo_a + i, lo_a + j)
    i, j = idx // size_b, idx % size_b
    return _keys(lo_a + i, lo_b + j)


def sbm_keys(n: int, blocks: int, p_in: float, p_out: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    bounds = np.linspace(0, n, blocks + 1).astype(np.int64)
    parts = []
    for a in range(blocks):
        for b in range(a, blocks):
            parts.append(_sample_pairs_block(rng, bounds[a], bounds[a + 1] - bounds[a], bounds[b],
                                             bounds[b + 1] - bounds[b], p_in if a == b else p_out, a == b))
    return np.unique(np.concatenate(parts))


def rmat_keys(scale: int, edge_factor: int, abcd=(0.57, 0.19, 0.19, 0.05), seed: int = 0) -> np.ndarray:
    """R-MAT edges, symmetrized, self-loops dropped, deduplicated. Quadrant
    probabilities are whole percentages, so each level draws one uint8 in
    [0, 100) per edge and compares against the cumulative thresholds."""
    rng = np.random.default_rng(seed)
    m = edge_factor << scale
    pa, pb, pc = (int(round(100 * x)) for x in abcd[:3])
    t1, t2, t3 = pa, pa + pb, pa + pb + pc
    u = np.zeros(m, np.int64)
    v = np.zeros(m, np.int64)
    for lvl in range(scale):
        r = rng.integers(0, 100, size=m, dtype=np.uint8)
        sh = scale - 1 - lvl
        down = r >= t2                               # quadrants c, d: row bit
        right = (r >= t1) ^ down ^ (r >= t3)         # quadrants b, d: column bit
        u |= down.astype(np.int64) << sh
        v |= right.astype(np.int64) << sh
    keep = u != v
    k = np.sort(_keys(u[keep], v[keep]))
    return k[np.concatenate([[True], k[1:] != k[:-1]])] if len(k) else k


@dataclass
class Stream:
    n0: int
    keys0: np.ndarray
    updates: list = field(default_factory=list)
    name: str = ""

    def csr0(self):
        return csr_from_keys(self.n0, self.keys0)


class _EdgeSet:
    """Sorted undirected key set with degrees, evolved batch by batch."""

    def __init__(self, n, keys):
        self.n = n
        self.keys = np.sort(keys)
        u, v = _unkey(self.keys)
        self.deg = np.bincount(np.concatenate([u, v]), minlength=n).astype(np.int64)

    def has(self, k):
        pos = np.searchsorted(self.keys, k)
        pos = np.minimum(pos, len(self.keys) - 1)
        return self.keys[pos] == k if len(self.keys) else np.zeros(len(k), bool)

    def sample_existing(self, rng, count):
        idx = np.unique(rng.integers(0, len(self.keys), size=count + count // 8 + 16))
        while len(idx) < count:
            idx = np.unique(np.concatenate([idx, rng.integers(0, len(self.keys), size=count)]))
        return self.keys[rng.permutation(idx)[:count]]

    def sample_by_degree(self, rng, size):
        cum = np.cumsum(self.deg)
        if cum[-1] == 0:
            return rng.integers(0, self.n, size=size)
        return np.searchsorted(cum, rng.integers(0, cum[-1], size=size), side="right")

    def sample_absent(self, rng, count, forbid=None):
        out = np.zeros(0, np.int64)
        while len(out) < count:
            u = rng.integers(0, self.n, size=2 * (count - len(out)) + 16)
            v = rng.integers(0, self.n, size=len(u))
            ok = u != v
            k = np.unique(_keys(u[ok], v[ok]))
            k = k[~self.has(k)]
            if forbid is not None and len(forbid):
                k = k[~np.isin(k, forbid)]
            out = np.unique(np.concatenate([out, k]))
        return rng.permutation(out)[:count]

    def apply(self, added, removed, n_new, new_keys):
        keep = np.ones(len(self.keys), bool)
        keep[np.searchsorted(self.keys, removed)] = False
        self.keys = np.sort(np.concatenate([self.keys[keep], added, new_keys]))
        self.n += n_new
        deg = np.zeros(self.n, np.int64)
        deg[: len(self.deg)] = self.deg
        ru, rv = _unkey(removed)
        au, av = _unkey(np.concatenate([added, new_keys]))
        deg -= np.bincount(np.concatenate([ru, rv]), minlength=self.n)
        deg += np.bincount(np.concatenate([au, av]), minlength=self.n)
        self.deg = deg


def _update(added_keys, removed_keys, n_new, new_keys) -> Update:
    ai, aj = _unkey(added_keys)
    ri, rj = _unkey(removed_keys)
    ni, nj = _unkey(new_keys)
    return Update((ai, aj, np.ones(len(ai))), (ri, rj), int(n_new), (ni, nj, np.ones(len(ni))))


def edit_stream(n0, keys0, steps, seed, insert, delete, new_nodes=0, new_degree=0, name="") -> Stream:
    """Generic stream: per step `insert(m)` new edges among existing nodes
    (uniform over non-edges), `delete(m)` uniform existing edges, and
    `new_nodes(n)` appended nodes with `new_degree` distinct preferential-
    attachment edges each (targets drawn proportional to pre-step degree)."""
    rng = np.random.default_rng(seed)
    es = _EdgeSet(n0, keys0)
    s = Stream(n0, es.keys.copy(), name=name)
    for _ in range(steps):
        m = len(es.keys)
        n_ins, n_del = int(insert(m)), int(delete(m))
        S = int(new_nodes(es.n)) if callable(new_nodes) else int(new_nodes)
        removed = es.sample_existing(rng, n_del) if n_del else np.zeros(0, np.int64)
        added = es.sample_absent(rng, n_ins, forbid=removed) if n_ins else np.zeros(0, np.int64)
        new_keys = np.zeros(0, np.int64)
        if S and new_degree:
            tgt = es.sample_by_degree(rng, S * new_degree).reshape(S, new_degree)
            for _r in range(64):  # redraw repeated targets of one newcomer
                srt = np.sort(tgt, axis=1)
                dup = np.zeros_like(tgt, dtype=bool)
                dup[:, 1:] = srt[:, 1:] == srt[:, :-1]
                if not dup.any():
                    break
                tgt = srt
                tgt[dup] = es.sample_by_degree(rng, int(dup.sum()))
            newcomers = es.n + np.repeat(np.arange(S), new_degree)
            new_keys = np.unique(_keys(tgt.reshape(-1), newcomers))
        s.updates.append(_update(added, removed, S, new_keys))
        es.apply(added, removed, S, new_keys)
    return s


# ---------------------------------------------------------------- BASELINE configs
def config1(seed=1, n=10_000, steps=10):
    """SBM n=10,000, 4 equal blocks, p_in=0.01, p_out=0.001; 500 inserts + 100 deletes per step."""
    keys = sbm_keys(n, 4, 0.01, 0.001, seed)
    return edit_stream(n, keys, steps, seed + 1, lambda m: 500, lambda m: 100, name="cfg1-sbm10k")


def config2(seed=2, n=100_000, avg_deg=20, steps=20):
    """Erdos-Renyi n=100,000, average degree 20; 1% inserts, 0.5% deletes (of edges) per step."""
    keys = sbm_keys(n, 1, avg_deg / (n - 1), 0.0, seed)
    return edit_stream(n, keys, steps, seed + 1, lambda m: 0.01 * m, lambda m: 0.005 * m, name="cfg2-er100k")


def config3(seed=3, scale=20, steps=10, edge_factor=16):
    """R-MAT scale 20, ef 16; per step 1% new nodes x 10 PA edges and 0.5% edge deletions."""
    keys = rmat_keys(scale, edge_factor, seed=seed)
    n = 1 << scale
    return edit_stream(n, keys, steps, seed + 1, lambda m: 0, lambda m: 0.005 * m,
                       new_nodes=lambda nn: nn // 100, new_degree=10, name=f"cfg3-rmat-s{scale}")


def config4(seed=4, n=1 << 22, blocks=64, steps=10, avg_deg=32.0, intra=0.8, new_degree=16):
    """SBM n=2^22, 64 equal blocks, average degree 32 with 80% of edges intra-block.
    Per step: 1% edge inserts, 0.5% edge deletes, 0.5% * n new nodes with 16
    edges each (80% into one random block, the rest anywhere), and 0.1% * n node
    "removals". The reference has no node removal; as SURVEY.md
    8(d) proposes, a removal deletes every incident edge and keeps the index as
    an isolated node, which the reference's update model expresses exactly."""
    bs = n // blocks
    p_in = avg_deg * intra / (bs - 1)
    p_out = avg_deg * (1 - intra) / (n - bs)
    keys0 = sbm_keys(n, blocks, p_in, p_out, seed)
    rng = np.random.default_rng(seed + 1)
    es = _EdgeSet(n, keys0)
    s = Stream(n, es.keys.copy(), name=f"cfg4-sbm{n}")
    for _ in range(steps):
        m = len(es.keys)
        cur = es.n
        # node removals: all incident edges
        gone = np.unique(rng.integers(0, cur, size=max(1, cur // 1000)))
        u, v = _unkey(es.keys)
        inc = es.keys[np.isin(u, gone) | np.isin(v, gone)]
        rnd = es.sample_existing(rng, int(0.005 * m))
        removed = np.unique(np.concatenate([inc, rnd]))
        added = es.sample_absent(rng, int(0.01 * m), forbid=removed)
        au, av = _unkey(added)
        added = added[~(np.isin(au, gone) | np.isin(av, gone))]
        # new nodes: 16 distinct edges each, 80% into one random block
        S = cur // 200
        blk = rng.integers(0, blocks, size=S)
        inb = rng.random((S, new_degree)) < intra
        tgt = np.where(inb, blk[:, None] * bs + rng.integers(0, bs, size=(S, new_degree)),
                       rng.integers(0, cur, size=(S, new_degree)))
        newcomers = cur + np.repeat(np.arange(S), new_degree)
        new_keys = np.unique(_keys(tgt.reshape(-1), newcomers))
        s.updates.append(_update(added, removed, S, new_keys))
        es.apply(added, removed, S, new_keys)
    return s


# ------------------------------------------------- config 5 (device-side generator)
class TorchStream:
    """A stream whose start graph is built and kept as torch tensors (GPU for
    R-MAT scale 25: ~1.07B stored entries, out of reach of the numpy path).
    `csr0()` returns host arrays like `Stream.csr0`; `csr0_torch()` the device
    ones (int32 rowptr / int32 col / fp64 val)."""

    def __init__(self, n0, rowptr, col, updates, name):
        self.n0 = n0
        self._rp, self._col = rowptr, col
        self.updates = updates
        self.name = name

    @property
    def nnz0(self) -> int:
        return int(self._col.numel())

    def csr0_torch(self):
        import torch

        return self._rp, self._col, torch.ones(self._col.numel(), dtype=torch.float64, device=self._col.device)

    def csr0(self):
        return (self._rp.cpu().numpy(), self._col.cpu().numpy(), np.ones(self._col.numel(), np.float64))

    def release(self):
        self._rp = self._col = None


def rmat_keys_torch(scale: int, edge_factor: int, abcd=(0.57, 0.19, 0.19, 0.05), seed: int = 0, device="cuda"):
    """`rmat_keys` on a torch device (torch's Philox stream instead of numpy's
    PCG64, so the graph differs from rmat_keys at the same seed; same model:
    one draw in [0, 100) per level per edge, symmetrized, self-loops dropped,
    deduplicated, sorted undirected keys lo << 32 | hi)."""
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    m = edge_factor << scale
    pa, pb, pc = (int(round(100 * x)) for x in abcd[:3])
    t1, t2, t3 = pa, pa + pb, pa + pb + pc
    u = torch.zeros(m, dtype=torch.int64, device=device)
    v = torch.zeros(m, dtype=torch.int64, device=device)
    for lvl in range(scale):
        r = torch.randint(0, 100, (m,), generator=g, device=device, dtype=torch.int16)
        sh = scale - 1 - lvl
        down = r >= t2
        right = (r >= t1) ^ down ^ (r >= t3)
        del r
        u |= down.to(torch.int64) << sh
        v |= right.to(torch.int64) << sh
        del down, right
    keep = u != v
    lo = torch.minimum(u, v)[keep]
    hi = torch.maximum(u, v)[keep]
    del u, v, keep
    k = (lo << 32) | hi
    del lo, hi
    return torch.unique(k)  # sorted


def csr_from_keys_torch(n: int, keys):
    """`csr_from_keys` (unit weights) on a torch device: int32 rowptr / col."""
    import torch

    lo, hi = keys >> 32, keys & 0xFFFFFFFF
    both = torch.cat([(lo << 32) | hi, (hi << 32) | lo])
    del lo, hi
    both, _ = torch.sort(both)
    rows = both >> 32
    col = (both & 0xFFFFFFFF).to(torch.int32)
    del both
    rowptr = torch.zeros(n + 1, dtype=torch.int64, device=keys.device)
    rowptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    del rows
    return rowptr.to(torch.int32), col


def config5(seed=5, scale=25, steps=5, edge_factor=16, new_degree=16, device="cuda"):
    """R-MAT scale 25, ef 16, (0.57,0.19,0.19,0.05), symmetrized and
    deduplicated; per step 0.1% of the edges inserted uniformly over
    non-edges and 0.1% new nodes with `new_degree` distinct preferential-
    attachment edges each (targets drawn proportional to pre-step degree from
    the endpoint pool, as edit_stream). Built on `device` with torch; the
    update batches are host edit lists like every other stream."""
    import torch

    n = 1 << scale
    keys0 = rmat_keys_torch(scale, edge_factor, seed=seed, device=device)
    rowptr, col = csr_from_keys_torch(n, keys0)
    g = torch.Generator(device=device).manual_seed(seed + 1)
    nnz0 = col.numel()
    extra = torch.zeros(0, dtype=torch.int64, device=device)  # endpoints of edges added by earlier steps
    prior = torch.zeros(0, dtype=torch.int64, device=device)  # keys added by earlier steps (sorted)
    m_edges, cur = keys0.numel(), n
    updates = []

    def has(k):
        pos = torch.searchsorted(keys0, k).clamp_max(keys0.numel() - 1)
        hit = keys0[pos] == k
        if prior.numel():
            p2 = torch.searchsorted(prior, k).clamp_max(prior.numel() - 1)
            hit |= prior[p2] == k
        return hit

    def by_degree(size):
        idx = torch.randint(0, nnz0 + extra.numel(), (size,), generator=g, device=device)
        out = col[idx.clamp_max(nnz0 - 1)].to(torch.int64)
        if extra.numel():
            ex = idx >= nnz0
            out[ex] = extra[idx[ex] - nnz0]
        return out

    for _ in range(steps):
        n_ins = m_edges // 1000
        added = torch.zeros(0, dtype=torch.int64, device=device)
        while added.numel() < n_ins:
            want = 2 * (n_ins - added.numel()) + 16
            a = torch.randint(0, cur, (want,), generator=g, device=device)
            b = torch.randint(0, cur, (want,), generator=g, device=device)
            ok = a != b
            k = (torch.minimum(a, b)[ok] << 32) | torch.maximum(a, b)[ok]
            k = torch.unique(k)
            k = k[~has(k)]
            added = torch.unique(torch.cat([added, k]))
        added = added[torch.randperm(added.numel(), generator=g, device=device)[:n_ins]]
        S = cur // 1000
        tgt = by_degree(S * new_degree).reshape(S, new_degree)
        for _r in range(64):  # redraw repeated targets of one newcomer
            srt, _ = torch.sort(tgt, dim=1)
            dup = torch.zeros_like(srt, dtype=torch.bool)
            dup[:, 1:] = srt[:, 1:] == srt[:, :-1]
            if not bool(dup.any()):
                break
            tgt = srt
            tgt[dup] = by_degree(int(dup.sum()))
        newcomers = cur + torch.arange(S, device=device).repeat_interleave(new_degree)
        tg = tgt.reshape(-1)
        new_keys = torch.unique((torch.minimum(tg, newcomers) << 32) | torch.maximum(tg, newcomers))
        hk = lambda t: t.cpu().numpy()  # noqa: E731
        updates.append(_update(hk(added), np.zeros(0, np.int64), S, hk(new_keys)))
        ends = torch.cat([added >> 32, added & 0xFFFFFFFF, new_keys >> 32, new_keys & 0xFFFFFFFF])
        extra = torch.cat([extra, ends])
        prior, _ = torch.sort(torch.cat([prior, added, new_keys]))
        m_edges += added.numel() + new_keys.numel()
        cur += S
    del keys0, prior, extra
    return TorchStream(n, rowptr, col, updates, name=f"cfg5-rmat-s{scale}")
