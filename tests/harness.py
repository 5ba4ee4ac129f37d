"""Side-by-side runner for parity tests: the CUDA path (through the C ABI) and
the CPU oracle consume the same start graph, the same initial eigenpairs and
the same serialized update batches."""
import numpy as np

import pyoracle as po

# Parity contract (BASELINE.json north_star): CSR bit-exact; Ritz values within
# 1e-10 relative (measured against the spectrum scale max|theta|); eigenvector
# spans within sin(largest principal angle) <= 1e-8.
VALUE_RTOL = 1e-10
SIN_TOL = 1e-8


def sin_angle(a: np.ndarray, b: np.ndarray) -> float:
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    r = qa - qb @ (qb.T @ qa)
    return float(np.linalg.norm(r, 2)) if r.size else 0.0


def value_err(va, vb) -> float:
    scale = max(float(np.abs(vb).max()), 1e-300)
    return float(np.abs(np.asarray(va) - np.asarray(vb)).max() / scale)


def pair(rowptr, col, val, kind="grest-rsvd", k=8, order="abs_desc", rsvd_l=100, rsvd_p=100, seed=0,
         operator="adjacency", force_dense=False, **kw):
    """(gpu, oracle) sessions from the same initial state: the oracle runs the
    reference tracker_init (Lanczos) and the GPU session takes its output."""
    from paper_2603_19439_b200 import TrackerSession

    n = len(rowptr) - 1
    a = po.Csr(n, np.asarray(rowptr, np.int32), np.asarray(col, np.int32), np.asarray(val, np.float64))
    o = po.Session(a, kind=kind, k=k, order=order, rsvd_l=rsvd_l, rsvd_p=rsvd_p, seed=seed, operator=operator)
    vals, vecs = o.embedding()
    g = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind=kind, k=k, order=order, rsvd_l=rsvd_l,
                       rsvd_p=rsvd_p, seed=seed, operator=operator, force_dense=force_dense, **kw)
    return g, o


def csr_equal(g_csr, o_csr: po.Csr) -> bool:
    rp, col, val = g_csr
    return (np.array_equal(rp, o_csr.rowptr) and np.array_equal(col, o_csr.col)
            and np.array_equal(val, o_csr.val))


def check_state(g, o, laplacian=False, tag=""):
    gv, gx = g.embedding()
    ov, ox = o.embedding()
    assert gx.shape == ox.shape, tag
    ve = value_err(gv, ov)
    assert ve <= VALUE_RTOL, f"{tag}: ritz value error {ve:.3e}"
    sa = sin_angle(gx, ox)
    assert sa <= SIN_TOL, f"{tag}: subspace sin {sa:.3e}"
    assert csr_equal(g.csr(0), o.csr(0)), f"{tag}: adjacency CSR differs"
    assert csr_equal(g.csr(2), o.csr(2)), f"{tag}: perturbation CSR differs"
    if laplacian:
        assert csr_equal(g.csr(1), o.csr(1)), f"{tag}: shifted operator CSR differs"
    info = g.info()
    n, k, steps, _ = o.info()
    assert info["n"] == n and info["steps_taken"] == steps, tag
    return ve, sa


def random_update(rng, keys_present, n, n_add, n_rem, n_new, fan):
    """Uniform random edits against the current edge set (numpy helper)."""
    from paper_2603_19439_b200 import Update

    present = set(map(tuple, keys_present))
    rem = []
    if n_rem and present:
        pres = sorted(present)
        for idx in rng.choice(len(pres), size=min(n_rem, len(pres)), replace=False):
            rem.append(pres[idx])
    add = set()
    while len(add) < n_add:
        i, j = rng.integers(0, n, 2)
        if i == j:
            continue
        e = (min(i, j), max(i, j))
        if e in present or e in add:
            continue
        add.add(e)
    new = set()
    for s in range(n_new):
        for _ in range(fan):
            t = int(rng.integers(0, n))
            new.add((t, n + s))
        if s > 0 and rng.random() < 0.3:
            new.add((n + s - 1, n + s))
    return Update.make([(i, j, 1.0) for i, j in sorted(add)], rem, n_new, [(i, j, 1.0) for i, j in sorted(new)])


def edges_of(csr_tuple):
    rp, col, _ = csr_tuple
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    m = rows < col
    return np.stack([rows[m], col[m]], 1)
