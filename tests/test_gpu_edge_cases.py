"""Edge cases of the step against the CPU oracle (parity bar as elsewhere):
isolated new nodes, removal-only batches, rank-1 sketches, hub rows on the
Laplacian operators, k above the candidate count."""
import numpy as np
import pytest

import pyoracle as po
from harness import check_state, pair

pytestmark = pytest.mark.gpu


def U(*a, **k):
    from paper_2603_19439_b200 import Update
    return Update.make(*a, **k)


def ring(n, chords=0, seed=0):
    rng = np.random.default_rng(seed)
    e = {tuple(sorted((i, (i + 1) % n))) for i in range(n)}
    while chords > 0:
        i, j = sorted(rng.integers(0, n, 2).tolist())
        if i != j and (i, j) not in e:
            e.add((i, j))
            chords -= 1
    return po.from_edges(n, sorted(e))


def run(a, steps, kind="grest-rsvd", k=4, operator="adjacency", L=100, P=100):
    gpu, orc = pair(a.rowptr, a.col, a.val, kind=kind, k=k, operator=operator, rsvd_l=L, rsvd_p=P, seed=7)
    for t, upd in enumerate(steps):
        orc.step(upd)
        gpu.step(upd)
        check_state(gpu, orc, laplacian=operator != "adjacency", tag=f"{kind}/{operator} step {t}")


KINDS = ["iasc", "grest2", "grest3", "grest-rsvd"]


@pytest.mark.parametrize("kind", KINDS)
def test_isolated_new_nodes(kind):
    """New nodes with no edges: zero Delta columns, dropped candidates."""
    a = ring(300, 40, 1)
    run(a, [U([], [], 3, []), U([(0, 150, 1.0)], [], 2, [(303, 5, 1.0), (304, 301, 1.0)])], kind=kind)


@pytest.mark.parametrize("kind", KINDS)
def test_removal_only(kind):
    a = ring(300, 60, 2)
    rp, col = a.rowptr, a.col
    rem = [(i, int(col[rp[i]])) for i in range(0, 300, 7) if col[rp[i]] > i][:12]
    run(a, [U([], rem, 0, [])], kind=kind)


@pytest.mark.parametrize("L,P", [(4, 3), (8, 8)])
def test_rank_one_sketch(L, P):
    """Every new node attaches to node 0 only: Delta_2 has rank 1, the RSVD
    sketch Y = Delta_2 Omega is rank 1 and its orthonormalization drops all
    but one column."""
    a = ring(400, 50, 3)
    n = 400
    S = 40
    run(a, [U([], [], S, [(n + s, 0, 1.0) for s in range(S)])], kind="grest-rsvd", L=L, P=P)


@pytest.mark.parametrize("operator", ["laplacian", "normalized-laplacian"])
@pytest.mark.parametrize("kind", ["grest2", "grest-rsvd"])
def test_hub_edits_on_laplacians(operator, kind):
    a = ring(400, 50, 4)
    nb0 = set(a.col[a.rowptr[0]:a.rowptr[1]].tolist())
    hub = [(0, j, 1.0) for j in range(2, 60) if j not in nb0]
    run(a, [U(hub, [], 2, [(400, 0, 1.0), (401, 7, 1.0)]), U([(3, 90, 2.0)], [(0, 2)], 0, [])],
        kind=kind, operator=operator)


def test_k_above_candidate_rank():
    """k = 12 with a single edit: Delta X-bar has rank 2, ten candidates drop."""
    a = ring(300, 80, 5)
    run(a, [U([(10, 200, 1.0)], [], 0, [])], kind="grest2", k=12)


@pytest.mark.gpu
def test_pinned_edit_lists_take_the_direct_upload():
    """Edit lists in page-locked memory are DMA'd straight from the caller's
    arrays (no staging copy); the step is bit-identical to the staged path."""
    from paper_2603_19439_b200 import TrackerSession, streams

    s = streams.config1(n=3000, steps=2)
    rp, col, val = s.csr0()
    rng = np.random.default_rng(0)
    x, _ = np.linalg.qr(rng.standard_normal((len(rp) - 1, 8)))
    lam = np.linspace(8.0, 1.0, 8)
    a = TrackerSession(rp, col, val, lam, x, kind="grest-rsvd", k=8, seed=1)
    b = TrackerSession(rp, col, val, lam, x, kind="grest-rsvd", k=8, seed=1)
    for upd in s.updates:
        a.step(upd)
        b.step(upd.pinned())
    va, xa = a.embedding()
    vb, xb = b.embedding()
    assert np.array_equal(va, vb) and np.array_equal(xa, xb)
    for c in range(3):
        assert np.array_equal(a.csr(0)[c], b.csr(0)[c])



def test_failed_step_right_after_a_step_keeps_the_rotated_state():
    """The rotation of X runs beside the next step's ingestion (st_rot_): a step
    that fails in its ingestion right after a successful one must leave the
    rotated state of the successful step, and the next step must see it."""
    from harness import SIN_TOL, VALUE_RTOL, csr_equal, edges_of, random_update, sin_angle, value_err
    from paper_2603_19439_b200 import TrackerError, Update
    from support import random_graph

    rng = np.random.default_rng(3)
    n = 600
    a = random_graph(n, 0.03, 7)
    g, o = pair(a.rowptr, a.col, a.val, kind="grest-rsvd", k=6, rsvd_l=4, rsvd_p=4)
    for t in range(3):
        present = edges_of(g.csr(0))
        u = random_update(rng, present, n, 6, 3, 5, 3)  # compressed path: |P| << n
        g.step(u)
        o.step(u)
        n += 5
        have = set(map(tuple, edges_of(g.csr(0)).tolist()))
        miss = next((i, j) for i in range(n) for j in range(i + 1, n) if (i, j) not in have)
        with pytest.raises(TrackerError, match="invalid deletion"):
            g.step(Update.make(removed=[miss]))
        gv, gx = g.embedding()
        ov, ox = o.embedding()
        assert value_err(gv, ov) <= VALUE_RTOL and sin_angle(gx, ox) <= SIN_TOL, f"after failed step {t}"
        assert csr_equal(g.csr(0), o.csr(0)) and g.info()["steps_taken"] == t + 1
