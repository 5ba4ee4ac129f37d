"""Device tracker_init (thick-restart Lanczos, lanczos.hpp:38-127) against the
oracle's lanczos_topk_csr restatement: the same graph, k, order and seed."""
import numpy as np
import pytest

import pyoracle as po
from harness import SIN_TOL, csr_equal, sin_angle, value_err

pytestmark = pytest.mark.gpu


def _graph(kind: str, scale: int = 12):
    from paper_2603_19439_b200 import streams

    if kind == "rmat":
        s = streams.config3(seed=7, scale=scale, steps=1)
    else:
        s = streams.config1(n=3000, steps=1)
    return s


def _oracle_op(rp, col, val, operator):
    a = po.Csr(len(rp) - 1, rp, col, val)
    if operator == "adjacency":
        return a
    return po.shifted_laplacian(a, 2, 2.0)[0]  # normalized kind, alpha = 2 (laplacian_track.cpp:35-39)


@pytest.mark.parametrize("graph,k,order,operator", [
    ("sbm", 8, "abs_desc", "adjacency"),
    ("rmat", 32, "abs_desc", "adjacency"),
    ("rmat", 16, "alg_desc", "adjacency"),
    ("sbm", 16, "alg_desc", "normalized-laplacian"),
])
def test_tracker_init_matches_oracle_lanczos(graph, k, order, operator):
    from paper_2603_19439_b200 import TrackerSession

    s = _graph(graph)
    rp, col, val = s.csr0()
    g = TrackerSession.tracker_init(rp, col, val, k, order=order, operator=operator, seed=3)
    gv, gx = g.embedding()
    op = _oracle_op(rp, col, val, operator)
    ov, ox = po.lanczos(op, k, 0 if order == "abs_desc" else 1, seed=3)
    restarts, products = g.init_stats()
    scale = np.abs(ov).max()
    ve = value_err(gv, ov)
    sa = sin_angle(gx, ox)
    res = g.residual_norms()
    print(f"{graph} k={k} {order} {operator}: restarts {restarts} products {products} value err {ve:.2e} "
          f"sin {sa:.2e} max residual {res.max() / scale:.2e}")
    assert ve <= 1e-10
    assert sa <= SIN_TOL
    # the device pairs pass the reference's own convergence test
    assert res.max() <= 1e-10 * scale * 1.01
    # the graph is untouched
    assert csr_equal(g.csr(0), po.Csr(len(rp) - 1, rp, col, val))


def test_tracker_init_then_step_matches_oracle():
    """tracker_init on both sides, then G-REST steps: the whole reference loop
    (trackers.cpp:132-145 then :341-387) with no harness-supplied X0."""
    from paper_2603_19439_b200 import TrackerSession

    s = _graph("rmat", 12)
    from paper_2603_19439_b200 import streams

    s = streams.config3(seed=11, scale=12, steps=3)
    rp, col, val = s.csr0()
    g = TrackerSession.tracker_init(rp, col, val, 16, kind="grest-rsvd", seed=5)
    o = po.Session(po.Csr(len(rp) - 1, rp, col, val), kind="grest-rsvd", k=16, seed=5)
    for t, u in enumerate(s.updates):
        g.step(u)
        o.step(u)
        gv, gx = g.embedding()
        ov, ox = o.embedding()
        assert value_err(gv, ov) <= 1e-10, t
        assert sin_angle(gx, ox) <= SIN_TOL, t
        assert csr_equal(g.csr(0), o.csr(0)), t


def test_tracker_init_errors():
    from paper_2603_19439_b200 import TrackerError, TrackerSession

    s = _graph("sbm")
    rp, col, val = s.csr0()
    n = len(rp) - 1
    with pytest.raises(TrackerError, match="k must satisfy 1 <= k <= n"):
        TrackerSession.tracker_init(rp, col, val, n + 1)
    with pytest.raises(TrackerError, match="max_basis below k") as e:
        TrackerSession.tracker_init(rp, col, val, 8, max_basis=4)
    assert e.value.kind == "invalid_argument"
    with pytest.raises(TrackerError, match="no convergence after 0 restarts") as e:
        TrackerSession.tracker_init(rp, col, val, 8, max_restarts=0)
    assert e.value.kind == "runtime_error"


def test_tracker_init_tiny_complete_graph():
    """K3 (test_trackers.cpp:48-62): eigenvalues 2, -1, -1; the basis spans the
    whole space (j >= n exit)."""
    from paper_2603_19439_b200 import TrackerSession

    rp = np.array([0, 2, 4, 6], np.int32)
    col = np.array([1, 2, 0, 2, 0, 1], np.int32)
    val = np.ones(6)
    g = TrackerSession.tracker_init(rp, col, val, 2, order="alg_desc")
    v, x = g.embedding()
    assert abs(v[0] - 2.0) < 1e-12 and abs(v[1] + 1.0) < 1e-12
    assert sin_angle(x[:, :1], np.ones((3, 1))) < 1e-12
