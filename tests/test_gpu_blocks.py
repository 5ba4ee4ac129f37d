"""The GraphUpdate and Perturbation entry points (st_step_blocks,
st_step_perturbation) against the edit-list path (st_step): the reference loop
consumes GraphUpdate blocks (experiment.cpp:166-173; tracker_step overloads
trackers.hpp:130-133), so a caller holding blocks must get bit-identical
results."""
import numpy as np
import pytest

import pyoracle as po
from harness import csr_equal

pytestmark = pytest.mark.gpu


def _sessions(rp, col, val, vals, vecs, count, **kw):
    from paper_2603_19439_b200 import TrackerSession

    return [TrackerSession(rp, col, val, vals, vecs, **kw) for _ in range(count)]


def _same(a, b, tag):
    av, ax = a.embedding()
    bv, bx = b.embedding()
    assert np.array_equal(av, bv), f"{tag}: Ritz values differ"
    assert np.array_equal(ax, bx), f"{tag}: vectors differ"
    for w in (0, 2):
        ga, gb = a.csr(w), b.csr(w)
        assert all(np.array_equal(x, y) for x, y in zip(ga, gb)), f"{tag}: csr {w} differs"


@pytest.mark.parametrize("stream", ["cfg1", "rmat"])
def test_blocks_and_perturbation_bit_identical_to_edit_lists(stream):
    from paper_2603_19439_b200 import GraphUpdate, streams

    s = streams.config1(n=3000, steps=3) if stream == "cfg1" else streams.config3(seed=9, scale=13, steps=3)
    rp, col, val = s.csr0()
    n = len(rp) - 1
    o = po.Session(po.Csr(n, rp, col, val), kind="grest-rsvd", k=16, seed=0)
    vals, vecs = o.embedding()
    e, b, p = _sessions(rp, col, val, vals, vecs, 3, kind="grest-rsvd", k=16, seed=0)
    for t, u in enumerate(s.updates):
        e.step(u)
        b.step_blocks(GraphUpdate.from_edits(n, u))
        d = po.update_delta(n, u)  # the Perturbation's Delta (to_delta of assemble_update)
        p.step_perturbation(n, u.n_new, d.rowptr, d.col, d.val)
        _same(e, b, f"blocks step {t}")
        _same(e, p, f"perturbation step {t}")
        o.step(u)
        assert csr_equal(b.csr(0), o.csr(0))
        n += u.n_new


def test_blocks_partial_deletion_and_weights():
    """K blocks may carry any nonzero weight (graph.hpp:7-12): a -0.5 entry
    halves an edge, exactly like an `added` edit of weight -0.5."""
    from paper_2603_19439_b200 import GraphUpdate, Update, streams

    s = streams.config1(n=2000, steps=1)
    rp, col, val = s.csr0()
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    m = rows < col
    ei, ej = rows[m][:5], col[m][:5]
    u = Update.make([(int(i), int(j), -0.5) for i, j in zip(ei, ej)], [], 3,
                    [(5, n, 1.0), (n, n + 1, 0.75), (n + 2, 7, 3.0)])
    o = po.Session(po.Csr(n, rp, col, val), kind="grest2", k=8, seed=0)
    vals, vecs = o.embedding()
    e, b = _sessions(rp, col, val, vals, vecs, 2, kind="grest2", k=8, seed=0)
    e.step(u)
    b.step_blocks(GraphUpdate.from_edits(n, u))
    _same(e, b, "partial deletion")
    o.step(u)
    assert csr_equal(b.csr(0), o.csr(0))
    rp2, col2, val2 = b.csr(0)
    r = np.repeat(np.arange(len(rp2) - 1), np.diff(rp2))
    for i, j in zip(ei, ej):
        assert val2[(r == i) & (col2 == j)][0] == 0.5


def test_blocks_validation_errors_leave_state():
    from paper_2603_19439_b200 import GraphUpdate, TrackerError, Update, csr_from_coo, streams

    s = streams.config1(n=2000, steps=1)
    rp, col, val = s.csr0()
    n = len(rp) - 1
    o = po.Session(po.Csr(n, rp, col, val), kind="grest2", k=8, seed=0)
    vals, vecs = o.embedding()
    (b,) = _sessions(rp, col, val, vals, vecs, 1, kind="grest2", k=8, seed=0)
    before = b.embedding()
    empty = csr_from_coo(0, [], [], [])
    # K not symmetric -> from_triplets validation (sparse.cpp:55-63)
    g = GraphUpdate(n, 0, csr_from_coo(n, [3], [9], [1.0]), csr_from_coo(n, [], [], []), empty)
    with pytest.raises(TrackerError, match="matrix is not symmetric") as ex:
        b.step_blocks(g)
    assert ex.value.kind == "invalid_argument"
    # deletion of a missing edge -> apply_update (graph.cpp:106-113)
    rows = np.repeat(np.arange(n), np.diff(rp))
    dense = set(zip(rows.tolist(), col.tolist()))
    i, j = next((i, j) for i in range(n) for j in range(i + 1, n) if (i, j) not in dense)
    g = GraphUpdate(n, 0, csr_from_coo(n, [i, j], [j, i], [-1.0, -1.0]), csr_from_coo(n, [], [], []), empty)
    with pytest.raises(TrackerError, match="invalid deletion"):
        b.step_blocks(g)
    # wrong n_old
    g = GraphUpdate(n + 1, 0, csr_from_coo(n + 1, [], [], []), csr_from_coo(n + 1, [], [], []), empty)
    with pytest.raises(TrackerError, match="matrix size != d.n_old"):
        b.step_blocks(g)
    # malformed: a column out of range
    bad = (np.array([0] + [1] * n, np.int32), np.array([n + 5], np.int32), np.array([1.0]))
    g = GraphUpdate(n, 0, bad, csr_from_coo(n, [], [], []), empty)
    with pytest.raises(TrackerError, match="malformed block CSR"):
        b.step_blocks(g)
    after = b.embedding()
    assert np.array_equal(before[0], after[0]) and np.array_equal(before[1], after[1])
    assert b.info()["steps_taken"] == 0
    # an empty GraphUpdate is the identity (trackers.cpp:358-361)
    b.step_blocks(GraphUpdate.from_edits(n, Update.make()))
    assert np.array_equal(b.embedding()[1], before[1])
    assert b.info()["steps_taken"] == 1
