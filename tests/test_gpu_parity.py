"""Parity of the CUDA path (C ABI) against the CPU oracle on identical seeded
inputs: CSR/Delta bit-exact, Ritz values within 1e-10, spans within 1e-8."""
import json
import os

import numpy as np
import pytest

import pyoracle as po
from harness import SIN_TOL, VALUE_RTOL, check_state, edges_of, pair, random_update, sin_angle, value_err
from support import random_graph, span_residual

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_known_answers.json")))


def U(*a, **k):
    from paper_2603_19439_b200 import Update
    return Update.make(*a, **k)


def test_fig1_known_answer_bitwise():
    g0 = GOLD["fig1"]
    a0 = po.from_edges(6, g0["a0_edges"])
    gpu, orc = pair(a0.rowptr, a0.col, a0.val, kind="grest2", k=2)
    u = g0["update"]
    upd = U(u["added"], u["removed"], u["n_new"], u["new_edges"])
    gpu.step(upd)
    orc.step(upd)
    rp, col, val = gpu.csr(0)
    gold = g0["a1"]
    assert rp.tolist() == gold["rowptr"] and col.tolist() == gold["col"] and val.tolist() == gold["val"]
    rp, col, val = gpu.csr(2)
    gold = g0["delta"]
    assert rp.tolist() == gold["rowptr"] and col.tolist() == gold["col"] and val.tolist() == gold["val"]
    check_state(gpu, orc, tag="fig1")


@pytest.mark.parametrize("upd,msg", [
    (dict(added=[(0, 1, 1.0)], removed=[(0, 1)]), "duplicate edge"),
    (dict(added=[(2, 2, 1.0)]), "self-loop"),
    (dict(added=[(0, 9, 1.0)]), "existing nodes"),
    (dict(n_new=1, new_edges=[(0, 1, 1.0)]), "only existing"),
    (dict(n_new=1, new_edges=[(0, 7, -1.0)]), "positive weight"),
    (dict(added=[(0, 1, 0.0)]), "zero-weight"),
    (dict(n_new=1, new_edges=[(0, 9, 1.0)]), "out of range"),
    (dict(added=[(3, 4, 1.0), (0, 5, 0.0), (1, 1, 1.0)]), "zero-weight"),          # first error wins
    (dict(added=[(1, 1, 1.0), (0, 5, 0.0)]), "self-loop"),
    (dict(removed=[(0, 3)]), "invalid deletion"),                                # apply_update
])
def test_errors_match_reference_and_leave_state(upd, msg):
    a = random_graph(7, 0.4, 21)
    gpu, orc = pair(a.rowptr, a.col, a.val, kind="grest3", k=2)
    v0, x0 = gpu.embedding()
    a0 = gpu.csr(0)
    upd = U(**upd)
    with pytest.raises(po.OracleError) as eo:
        orc.step(upd)
    from paper_2603_19439_b200 import TrackerError
    with pytest.raises(TrackerError) as eg:
        gpu.step(upd)
    assert msg in str(eo.value) and str(eg.value) == str(eo.value) and eg.value.kind == eo.value.kind
    v1, x1 = gpu.embedding()
    assert np.array_equal(v0, v1) and np.array_equal(x0, x1)
    assert all(np.array_equal(p, q) for p, q in zip(a0, gpu.csr(0)))
    assert gpu.info()["steps_taken"] == 0


def test_negative_weight_deletion():
    a = po.from_edges(3, [(0, 1, 0.5), (1, 2, 1.0)])
    gpu, orc = pair(a.rowptr, a.col, a.val, kind="grest2", k=1)
    from paper_2603_19439_b200 import TrackerError
    with pytest.raises(TrackerError, match="negative"):
        gpu.step(U(removed=[(0, 1)]))


@pytest.mark.parametrize("kind,L,P", [("grest2", 100, 100), ("grest3", 100, 100), ("grest-rsvd", 4, 3),
                                      ("grest-rsvd", 100, 100), ("iasc", 100, 100)])
@pytest.mark.parametrize("dense", [False, True])
def test_random_stream_parity(kind, L, P, dense):
    rng = np.random.default_rng(5)
    n = 160
    a = random_graph(n, 0.05, 31)
    gpu, orc = pair(a.rowptr, a.col, a.val, kind=kind, k=6, rsvd_l=L, rsvd_p=P, seed=3, force_dense=dense)
    for t in range(4):
        cur = gpu.info()["n"]
        upd = random_update(rng, edges_of(gpu.csr(0)), cur, 6, 3, 9 if t % 2 == 0 else 0, 3)
        gpu.step(upd)
        orc.step(upd)
        check_state(gpu, orc, tag=f"{kind} step {t}")


def test_empty_update_is_identity():
    a = random_graph(24, 0.2, 3)
    for kind in ("iasc", "grest2", "grest3", "grest-rsvd"):
        gpu, orc = pair(a.rowptr, a.col, a.val, kind=kind, k=4)
        v0, x0 = gpu.embedding()
        gpu.step(U())
        v1, x1 = gpu.embedding()
        assert np.array_equal(v0, v1) and np.array_equal(x0, x1)
        assert gpu.info()["steps_taken"] == 1 and gpu.info()["n"] == 24


@pytest.mark.parametrize("basis", ["iasc", "grest2", "grest3", "grest-rsvd"])
def test_probe_basis_spans_match(basis):
    a = random_graph(40, 0.15, 12)
    gpu, orc = pair(a.rowptr, a.col, a.val, kind="grest3", k=3, rsvd_l=2, rsvd_p=2)
    upd = U([(0, 4, 1.0), (1, 5, 1.0)], [], 3, [(2, 40, 1.0), (3, 41, 1.0), (6, 42, 1.0), (40, 41, 1.0),
                                                 (9, 42, 1.0)])
    zg = gpu.probe_basis(upd, basis, 5)
    zo = orc.probe_basis(upd, basis, 5)
    assert zg.shape == zo.shape
    assert np.abs(zg.T @ zg - np.eye(zg.shape[1])).max() <= 1e-10
    assert span_residual(zg, zo) <= 1e-8 and span_residual(zo, zg) <= 1e-8
    _, x = gpu.embedding()
    assert np.allclose(zg[:40, :3], x, atol=0, rtol=0)  # Z[:, :k] == X-bar bitwise (test_projection.cpp:68)


def test_probe_rr_exact_on_invariant_subspace_and_validation():
    a = random_graph(8, 0.5, 14)
    up = U([(0, 5, 1.0)], [], 2, [(3, 8, 1.0), (6, 9, 1.0), (8, 9, 1.0)])
    a_next = po.apply_update(a, up)
    w, v = po.sym_eig(a_next.dense(), 0)
    gpu, orc = pair(a.rowptr, a.col, a.val, kind="grest2", k=8)
    vals, vecs = gpu.probe_rr(up, v[:, :8])
    assert value_err(vals, w[:8]) <= 1e-9
    assert sin_angle(vecs, v[:, :8]) <= 1e-7
    ov, ox = orc.probe_rr(up, v[:, :8])
    assert value_err(vals, ov) <= VALUE_RTOL and sin_angle(vecs, ox) <= SIN_TOL
    from paper_2603_19439_b200 import TrackerError
    b = random_graph(10, 0.3, 16)
    gpu, _ = pair(b.rowptr, b.col, b.val, kind="grest2", k=4)
    u2 = U([(0, 3, 1.0)])
    with pytest.raises(TrackerError, match="projection subspace too small"):
        gpu.probe_rr(u2, np.eye(10, 3))
    skew = np.eye(10, 5)
    skew[0, 1] = 0.5
    with pytest.raises(TrackerError, match="column-orthonormal"):
        gpu.probe_rr(u2, skew)
    with pytest.raises(TrackerError, match="row count"):
        gpu.probe_rr(u2, np.eye(9, 5))


@pytest.mark.parametrize("op", ["normalized-laplacian", "laplacian"])
def test_laplacian_sessions_bitwise_and_parity(op):
    rng = np.random.default_rng(9)
    n = 120
    a = random_graph(n, 0.06, 44)
    gpu, orc = pair(a.rowptr, a.col, a.val, kind="grest3", k=5, order="alg_desc", operator=op)
    assert gpu.info()["alpha"] == orc.info()[3]
    for t in range(4):
        cur = gpu.info()["n"]
        upd = random_update(rng, edges_of(gpu.csr(0)), cur, 8, 4, 3, 2)
        gpu.step(upd)
        orc.step(upd)
        check_state(gpu, orc, laplacian=True, tag=f"{op} step {t}")
        assert gpu.info()["alpha"] == orc.info()[3]


def test_config1_parity_all_steps():
    from paper_2603_19439_b200 import streams
    s = streams.config1()
    rp, col, val = s.csr0()
    gpu, orc = pair(rp, col, val, kind="grest-rsvd", k=8, seed=0)
    for t, upd in enumerate(s.updates):
        gpu.step(upd)
        orc.step(upd)
        check_state(gpu, orc, tag=f"cfg1 step {t}")


def test_cusolver_eigensolver_in_the_step():
    # cuSOLVER syevd (ST_FLAG_CUSOLVER_EIG) in place of the on-device solver, on the RSVD path
    from paper_2603_19439_b200 import streams
    keys = streams.rmat_keys(12, 16, seed=9)
    s = streams.edit_stream(1 << 12, keys, 3, 10, lambda m: 20, lambda m: 0.005 * m,
                            new_nodes=lambda nn: 3 * nn // 100, new_degree=6)
    rp, col, val = s.csr0()
    gpu, orc = pair(rp, col, val, kind="grest-rsvd", k=8, seed=2, rsvd_l=40, rsvd_p=20, cusolver_eig=True)
    for t, upd in enumerate(s.updates):
        gpu.step(upd)
        orc.step(upd)
        check_state(gpu, orc, tag=f"cusolver-eig step {t}")


def test_rsvd_path_rmat_parity():
    from paper_2603_19439_b200 import streams
    keys = streams.rmat_keys(14, 16, seed=7)
    s = streams.edit_stream(1 << 14, keys, 2, 8, lambda m: 0, lambda m: 0.005 * m,
                            new_nodes=lambda nn: nn // 100, new_degree=10)
    rp, col, val = s.csr0()
    gpu, orc = pair(rp, col, val, kind="grest-rsvd", k=8, seed=11)
    for t, upd in enumerate(s.updates):
        assert upd.n_new > 100  # exercises the randomized range finder
        gpu.step(upd)
        orc.step(upd)
        check_state(gpu, orc, tag=f"rmat14 step {t}")


@pytest.mark.gpu
def test_config3_shape_parity_rmat17():
    """Config 3's shapes at a scale the oracle finishes in seconds: R-MAT s17,
    k = 32, L = P = 100 (q = 200 sketch, D = 164 Ritz basis), 1% new nodes with
    10 preferential-attachment edges and 0.5% deletions per step, both paths
    starting from the same leading eigenpairs (block Krylov, as bench.py).
    Exercises the two-block candidate orthonormalization, the first-order
    second CholQR pass, the skipped re-projection of the sketch basis, the
    2-CTA tridiagonalization (q = 200) and the block re-orthonormalization of
    the Ritz vectors at realistic sizes."""
    from paper_2603_19439_b200 import TrackerSession, init_eig, streams

    s = streams.config3(scale=17, steps=3)
    rp, col, val = s.csr0()
    k = 32
    vals, vecs = init_eig.leading_eigenpairs(rp, col, val, k, "abs_desc", device="cuda:0")
    n = len(rp) - 1
    a = po.Csr(n, np.asarray(rp, np.int32), np.asarray(col, np.int32), np.asarray(val, np.float64))
    orc = po.Session(a, kind="grest-rsvd", k=k, seed=5, values=vals, vectors=vecs)
    gpu = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind="grest-rsvd", k=k, seed=5)
    for t, upd in enumerate(s.updates):
        assert upd.n_new > 200  # the sketch is q = 200 wide
        gpu.step(upd)
        orc.step(upd)
        ve, sa = check_state(gpu, orc, tag=f"cfg3-s17 step {t}")
        print(f"cfg3-s17 step {t}: value err {ve:.2e}, subspace sin {sa:.2e}")


@pytest.mark.gpu
def test_wide_sketch_takes_exact_paths():
    """A sketch wider than the one-CTA Cholesky (q = L + P = 260 > 238) and the
    on-device eigensolver (> 228): the column-by-column orthonormalization
    replica and the cuSOLVER eigensolve run instead, with the same parity."""
    from paper_2603_19439_b200 import streams
    keys = streams.rmat_keys(12, 8, seed=9)
    s = streams.edit_stream(1 << 12, keys, 2, 4, lambda m: 0, lambda m: 0.005 * m,
                            new_nodes=lambda nn: 300, new_degree=4)
    rp, col, val = s.csr0()
    gpu, orc = pair(rp, col, val, kind="grest-rsvd", k=6, rsvd_l=140, rsvd_p=120, seed=2)
    for t, upd in enumerate(s.updates):
        assert upd.n_new > 260
        gpu.step(upd)
        orc.step(upd)
        check_state(gpu, orc, tag=f"wide sketch step {t}")


def _ring(n, chords=0, seed=0):
    rng = np.random.default_rng(seed)
    e = {(i, (i + 1) % n) if i < (i + 1) % n else ((i + 1) % n, i) for i in range(n)}
    while chords > 0:
        i, j = sorted(rng.integers(0, n, 2).tolist())
        if i != j and (i, j) not in e:
            e.add((i, j))
            chords -= 1
    return po.from_edges(n, sorted(e))


def test_hub_row_takes_the_sorting_path():
    """A Delta row longer than the counting path's limit (4096 entries):
    the ingestion re-runs on the radix-sort path; results stay bit-exact and
    the next (ordinary) step is back on the sort-free path."""
    a = _ring(5000, chords=300, seed=4)
    gpu, orc = pair(a.rowptr, a.col, a.val, kind="grest2", k=4)
    rp, col, _ = gpu.csr(0)
    nb0 = set(col[rp[0]:rp[1]].tolist())
    hub = [(0, j, 1.0) for j in range(2, 4700) if j not in nb0]
    assert len(hub) > 4096
    upd = U(hub, [], 2, [(5000, 0, 1.0), (5001, 3, 2.0), (5000, 5001, 1.0)])
    gpu.step(upd)
    orc.step(upd)
    check_state(gpu, orc, tag="hub step")
    upd = U([(10, 20, 1.0)], [(0, 5)], 1, [(5002, 0, 1.0)])
    gpu.step(upd)
    orc.step(upd)
    check_state(gpu, orc, tag="after hub")


@pytest.mark.parametrize("hub", [False, True])
def test_duplicate_orientations_and_lists(hub):
    """Duplicates are unordered pairs across all three lists, on both Delta
    assembly paths: the later edit is the one reported."""
    from paper_2603_19439_b200 import TrackerError
    a = _ring(5000, chords=50, seed=5)
    nb1 = set(a.col[a.rowptr[1]:a.rowptr[2]].tolist())
    extra = [(1, j, 1.0) for j in range(3, 4300) if j not in nb1] if hub else []
    cases = [dict(added=extra + [(7, 40, 1.0), (40, 7, 2.0)]),
             dict(added=extra + [(7, 40, 1.0)], removed=[(0, 1)], n_new=1, new_edges=[(40, 5000, 1.0), (7, 40, 1.0)]),
             dict(added=extra, removed=[(0, 1), (1, 0)])]
    for c in cases:
        gpu, orc = pair(a.rowptr, a.col, a.val, kind="grest2", k=3)
        u = U(**c)
        with pytest.raises(po.OracleError) as eo:
            orc.step(u)
        with pytest.raises(TrackerError) as eg:
            gpu.step(u)
        assert str(eg.value) == str(eo.value) and eg.value.kind == eo.value.kind
        assert gpu.info()["steps_taken"] == 0


@pytest.mark.parametrize("kind", ["grest2", "grest3", "grest-rsvd"])
@pytest.mark.parametrize("fan,n_new", [(1, 0), (8, 0), (8, 2), (98, 2)])
def test_rank_deficient_candidates_are_dropped(kind, fan, n_new):
    """Edits at one node make Delta X-bar rank <= 2: the reference drops the
    dependent candidates (ortho.hpp:34-35); the basis width and the step
    must follow it (the Cholesky's suspect/breakdown flags route the block to
    the column-by-column replica)."""
    n = 500
    a = _ring(n, chords=30, seed=4)
    gpu, orc = pair(a.rowptr, a.col, a.val, kind=kind, k=4)
    nb0 = set(a.col[a.rowptr[0]:a.rowptr[1]].tolist())
    hub = [(0, j, 1.0) for j in range(2, 2 + fan) if j not in nb0]
    upd = U(hub, [], n_new, [(n, 0, 1.0), (n + 1, 3, 2.0), (n, n + 1, 1.0)] if n_new else [])
    zg = gpu.probe_basis(upd, kind, 0)
    zo = orc.probe_basis(upd, kind, 0)
    assert zg.shape == zo.shape
    assert np.abs(zg.T @ zg - np.eye(zg.shape[1])).max() < 1e-12
    assert sin_angle(zg, zo) < SIN_TOL
    gpu.step(upd)
    orc.step(upd)
    check_state(gpu, orc, tag=f"{kind} fan {fan}")


@pytest.mark.gpu
def test_config4_shape_parity_sbm():
    """Config 4's shapes at a scale the oracle finishes in seconds: SBM with 64
    equal blocks, average degree 32 (80% intra-block), k = 64, L = P = 100;
    per step 1% inserts, 0.5% deletes, 0.5% new nodes with 16 edges each and
    0.1% node removals (every incident edge deleted, the index kept isolated,
    SURVEY.md 8(d)). D reaches 2k + L = 228: the 2-CTA tridiagonalization, a
    164-wide candidate block and the sketch's q = 163..165 columns."""
    from paper_2603_19439_b200 import TrackerSession, init_eig, streams

    s = streams.config4(n=1 << 15, steps=3)
    rp, col, val = s.csr0()
    k = 64
    vals, vecs = init_eig.leading_eigenpairs(rp, col, val, k, "abs_desc", device="cuda:0")
    n = len(rp) - 1
    a = po.Csr(n, np.asarray(rp, np.int32), np.asarray(col, np.int32), np.asarray(val, np.float64))
    orc = po.Session(a, kind="grest-rsvd", k=k, seed=9, values=vals, vectors=vecs)
    gpu = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind="grest-rsvd", k=k, seed=9)
    for t, upd in enumerate(s.updates):
        assert upd.n_new > 100  # the randomized range finder runs
        gpu.step(upd)
        orc.step(upd)
        ve, sa = check_state(gpu, orc, tag=f"cfg4-sbm32k step {t}")
        print(f"cfg4-sbm32k step {t}: value err {ve:.2e}, subspace sin {sa:.2e}")
        rp_t = gpu.csr(0)[0]
        assert np.all(np.diff(rp_t)[:n] >= 0)


@pytest.mark.gpu
def test_config5_shape_parity_rmat17():
    """Config 5's stream rules at a scale the oracle finishes in seconds
    (R-MAT s17 from the device generator bench.py uses at s25): per step 0.1%
    of the edges inserted over non-edges and 0.1% new nodes (131 > L, so the
    randomized range finder runs) with 16 preferential-attachment edges each,
    no deletions, k = 32, both paths from the same leading eigenpairs."""
    from paper_2603_19439_b200 import TrackerSession, init_eig, streams

    s = streams.config5(scale=17, steps=3, device="cuda:0")
    rp, col, val = s.csr0()
    k = 32
    vals, vecs = init_eig.leading_eigenpairs(rp, col, val, k, "abs_desc", device="cuda:0")
    n = len(rp) - 1
    a = po.Csr(n, np.asarray(rp, np.int32), np.asarray(col, np.int32), np.asarray(val, np.float64))
    orc = po.Session(a, kind="grest-rsvd", k=k, seed=7, values=vals, vectors=vecs)
    gpu = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind="grest-rsvd", k=k, seed=7)
    for t, upd in enumerate(s.updates):
        assert upd.n_new > 100 and len(upd.removed[0]) == 0
        gpu.step(upd)
        orc.step(upd)
        ve, sa = check_state(gpu, orc, tag=f"cfg5-s17 step {t}")
        print(f"cfg5-s17 step {t}: value err {ve:.2e}, subspace sin {sa:.2e}")


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["sbm-k64", "rmat-k32"])
def test_persistent_dmma_kernels_on_small_shapes(cfg, monkeypatch):
    """The persistent Gram / row-local GEMM kernels (device tile counter, producer
    warp, row-split warp layout, one-box diagonal tiles) take over from the
    static-grid kernels only when a product has more tiles than CTAs, i.e. at
    the BASELINE sizes. STG_PERSIST_ALWAYS routes every product of a small
    graph through them: ragged and diagonal tiles, symmetric products with two
    different operands (Z'(AZ), k = 64), in-place updates, fewer tiles than
    CTAs. Parity as everywhere: CSR bit-exact, Ritz 1e-10, sin 1e-8."""
    from paper_2603_19439_b200 import TrackerSession, init_eig, streams

    monkeypatch.setenv("STG_PERSIST_ALWAYS", "1")  # read when a session is created
    if cfg == "sbm-k64":
        s, k = streams.config4(n=1 << 15, steps=2), 64
    else:
        s, k = streams.config3(scale=14, steps=2), 32
    rp, col, val = s.csr0()
    vals, vecs = init_eig.leading_eigenpairs(rp, col, val, k, "abs_desc", device="cuda:0")
    n = len(rp) - 1
    a = po.Csr(n, np.asarray(rp, np.int32), np.asarray(col, np.int32), np.asarray(val, np.float64))
    orc = po.Session(a, kind="grest-rsvd", k=k, seed=5, values=vals, vectors=vecs)
    gpu = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind="grest-rsvd", k=k, seed=5)
    for t, upd in enumerate(s.updates):
        gpu.step(upd)
        orc.step(upd)
        ve, sa = check_state(gpu, orc, tag=f"persistent {cfg} step {t}")
        print(f"persistent {cfg} step {t}: value err {ve:.2e}, subspace sin {sa:.2e}")
