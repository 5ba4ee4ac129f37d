"""Stream generators and the update-batch wire format (libspectrack_stream.so,
include/spectrack_stream.h), CPU only.

* The reference's protocols are pinned (a) by ports of its own tests
  (proj/tests/test_dynamics.cpp: star split, degree order, one-step
  reconstruction, timestamp replay, SBM block structure, label ride-along,
  determinism, validation messages), with the chain-reconstruction check of
  test_dynamics.cpp:30-37 done on dense matrices here, and (b) bit for bit
  against an independent pure-Python restatement of sbm_sample_graph
  (dynamics.cpp:145-166) over a pure-Python mt19937_64 (rng.hpp:16-43).
* The BASELINE generators are checked against their stated rules and fed to
  the CPU oracle (assemble_update's validation accepts every batch).
* Wire format: save/load round trips, numpy streams through the format, bad
  files rejected.
"""
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_2603_19439_b200 import streams, wire

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ----------------------------------------------------------------- helpers
def dense_initial(ws):
    n = ws.n0
    a = np.zeros((n, n))
    i, j, w = ws.initial_edges()
    a[i, j] = w
    a[j, i] = w
    return a


def apply_dense(a, upd):
    """apply_update (graph.cpp:102-115) on a dense matrix: pad, add, delete."""
    n_old = a.shape[0]
    n = n_old + int(upd.n_new)
    b = np.zeros((n, n))
    b[:n_old, :n_old] = a
    for i, j, w in zip(*upd.added):
        b[i, j] += w
        b[j, i] += w
    for i, j in zip(*upd.removed):
        assert b[i, j] != 0.0, "deletion of a missing edge"
        b[i, j] -= 1.0
        b[j, i] -= 1.0
    for i, j, w in zip(*upd.new_edges):
        b[i, j] += w
        b[j, i] += w
    return b


def chain_matches(g_dense, ws):
    """check_chain_reconstruction (test_dynamics.cpp:30-37)."""
    origin = ws.node_origin()
    a = dense_initial(ws)
    assert np.array_equal(a, g_dense[np.ix_(origin[: a.shape[0]], origin[: a.shape[0]])])
    for t in range(ws.steps):
        a = apply_dense(a, ws.update(t))
        m = a.shape[0]
        assert np.array_equal(a, g_dense[np.ix_(origin[:m], origin[:m])]), f"step {t}"
    return a


def random_edges(n, p, seed):
    rng = np.random.default_rng(seed)
    return [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]


def dense_of(n, edges):
    a = np.zeros((n, n))
    for i, j in edges:
        a[i, j] = a[j, i] = 1.0
    return a


# ----------------------------------------------- pure-Python mt19937_64 (the pin)
class MT64:
    """std::mt19937_64 (the standard's parameters), independent of the C++."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            for k in range(312):
                y = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = self.mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                self.mt[k] = v
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def mix_seed(base, salt):
    M = 0xFFFFFFFFFFFFFFFF
    z = (base + 0x9E3779B97F4A7C15 * (salt + 0x632BE59BD9B4E019)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_mt19937_64_known_answer():
    g = MT64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042  # the C++ standard's required 10000th output


def test_sbm_sample_graph_bitwise_against_python_restatement():
    n, k, p_in, p_out, seed = 40, 3, 0.3, 0.05, 7
    g = MT64(mix_seed(seed, 0x5B31))
    labels = [g() % k for _ in range(n)]
    edges = []
    for i in range(n):
        for j in range(i + 1, n):
            p = p_in if labels[i] == labels[j] else p_out
            if (g() >> 11) * 2.0 ** -53 < p:
                edges.append((i, j))
    ws = wire.sbm_sample_graph(n, k, p_in, p_out, seed)
    assert list(ws.labels()) == labels
    i, j, _ = ws.initial_edges()
    assert list(zip(i.tolist(), j.tolist())) == edges


# ------------------------------------------------ ports of test_dynamics.cpp
def test_scenario1_star_split():  # test_dynamics.cpp:41-55
    star = [(0, 1), (0, 2), (0, 3), (0, 4)]
    ws = wire.scenario1(5, star, 2)
    assert list(ws.node_origin()) == [0, 1, 2, 3, 4]
    assert ws.n0 == 2
    i, j, w = ws.initial_edges()
    assert (i.tolist(), j.tolist(), w.tolist()) == ([0], [1], [1.0])
    assert ws.steps == 2
    assert [ws.update(t).n_new for t in range(2)] == [1, 2]  # leftover folds into the last step
    for t in range(2):
        u = ws.update(t)
        assert len(u.added[0]) == 0 and len(u.removed[0]) == 0  # pure expansion
    a = chain_matches(dense_of(5, star), ws)
    assert a.shape == (5, 5)


def test_scenario1_one_step_restores_full_graph():  # :57-69
    e = random_edges(17, 0.3, 5)
    ws = wire.scenario1(17, e, 1)
    a = chain_matches(dense_of(17, e), ws)
    assert a.shape[0] == 17 and np.count_nonzero(a) == 2 * len(e)


def test_scenario1_orders_arrivals_by_descending_degree():  # :71-81
    e = random_edges(30, 0.25, 9)
    ws = wire.scenario1(30, e, 4)
    deg = dense_of(30, e).sum(axis=1)
    o = ws.node_origin()
    for a_, b_ in zip(o[:-1], o[1:]):
        assert deg[a_] >= deg[b_]
        if deg[a_] == deg[b_]:
            assert a_ < b_
    chain_matches(dense_of(30, e), ws)


def test_scenario1_rejects_bad_step_counts():  # :83-88
    e = random_edges(8, 0.4, 2)
    for n, ed, t, msg in [(8, e, 0, "t_steps must be positive"), (8, e, 5, "more steps than nodes left to add"),
                          (1, [], 1, "graph too small to split")]:
        with pytest.raises(wire.StreamError, match=msg) as ex:
            wire.scenario1(n, ed, t)
        assert ex.value.kind == "invalid_argument"


def test_scenario2_replays_four_edges():  # :90-111
    ws = wire.scenario2(41, [(10, 20, 1), (20, 30, 2), (30, 40, 3), (40, 10, 4)], 2, 2)
    assert list(ws.node_origin()) == [10, 20, 30, 40]
    assert ws.n0 == 3
    i, j, _ = ws.initial_edges()
    assert list(zip(i, j)) == [(0, 1), (1, 2)]
    u0, u1 = ws.update(0), ws.update(1)
    assert u0.n_new == 1 and len(u0.new_edges[0]) == 1  # edge (2,3) brings node 3: one G entry
    assert u1.n_new == 0 and len(u1.added[0]) == 1  # edge (3,0) closes the cycle: K has 2 entries
    a = dense_initial(ws)
    for t in range(2):
        a = apply_dense(a, ws.update(t))
    assert np.count_nonzero(a) == 8


def test_scenario2_sorts_by_timestamp():  # :113-126
    a = wire.scenario2(10, [(0, 1, 1), (1, 2, 2), (2, 3, 3), (3, 4, 4)], 2, 2)
    b = wire.scenario2(10, [(2, 3, 3), (0, 1, 1), (3, 4, 4), (1, 2, 2)], 2, 2)
    assert list(a.node_origin()) == list(b.node_origin())
    assert np.array_equal(dense_initial(a), dense_initial(b))
    for t in range(a.steps):
        ua, ub = a.update(t), b.update(t)
        for x, y in ((ua.added, ub.added), (ua.new_edges, ub.new_edges)):
            assert sorted(zip(x[0], x[1])) == sorted(zip(y[0], y[1]))


def test_scenario2_drops_repeated_and_degenerate_edges():  # :128-138
    ws = wire.scenario2(6, [(0, 1, 1), (1, 0, 2), (2, 2, 2), (1, 2, 3), (0, 1, 9), (3, 4, 10)], 1, 1)
    assert len(ws.node_origin()) == 5
    a = apply_dense(dense_initial(ws), ws.update(0))
    assert np.count_nonzero(a) == 6


def test_scenario2_topology_only_update():  # :140-148
    ws = wire.scenario2(3, [(0, 1, 1), (1, 2, 2), (0, 2, 3)], 1, 2)
    u = ws.update(0)
    assert u.n_new == 0 and len(u.added[0]) == 1


def test_scenario2_validates_m0():  # :150-155
    for m0 in (2, 0):
        with pytest.raises(wire.StreamError, match="m0 must be within the unique edge count"):
            wire.scenario2(3, [(0, 1, 1), (0, 1, 5)], 1, m0)


def test_sbm_block_structure():  # :157-177
    ws = wire.sbm_sample_graph(200, 2, 0.2, 0.0, 7)
    lab = ws.labels()
    a = dense_initial(ws)
    same = lab[:, None] == lab[None, :]
    iu = np.triu_indices(200, 1)
    assert not np.any(a[~same])  # p_out = 0: no cross edges
    pairs = int(same[iu].sum())
    within = int(a[iu][same[iu]].astype(bool).sum())
    assert abs(within - 0.2 * pairs) <= 4.0 * np.sqrt(0.2 * 0.8 * pairs)


def test_sbm_certain_edges_give_cliques():  # :179-187
    ws = wire.sbm_sample_graph(40, 3, 1.0, 0.0, 11)
    lab = ws.labels()
    a = dense_initial(ws)
    same = (lab[:, None] == lab[None, :]) & ~np.eye(40, dtype=bool)
    assert np.array_equal(a != 0, same)


def test_sbm_rejects_invalid_probabilities():  # :189-193
    for p_in, p_out in ((0.05, 0.05), (1.2, 0.0), (0.5, -0.1)):
        with pytest.raises(wire.StreamError, match=r"need 0 <= p_out < p_in <= 1"):
            wire.sbm_sample_graph(10, 2, p_in, p_out, 0)


def test_sbm_stream_expands_with_labels():  # :195-233
    ws = wire.sbm_dynamic(120, 3, 0.2, 0.01, 80, 3, 10, 21)
    assert ws.n0 == 80 and ws.steps == 3
    for t in range(3):
        u = ws.update(t)
        assert u.n_new == 10 and len(u.added[0]) == 0 and len(u.removed[0]) == 0
    assert len(ws.node_origin()) == 110 and len(ws.labels()) == 110
    assert ws.labels().min() >= 0 and ws.labels().max() < 3
    full = wire.sbm_sample_graph(120, 3, 0.2, 0.01, 21)
    chain_matches(dense_initial(full), ws)
    assert np.array_equal(ws.labels(), full.labels()[ws.node_origin()])
    again = wire.sbm_dynamic(120, 3, 0.2, 0.01, 80, 3, 10, 21)  # same config -> identical stream
    assert np.array_equal(again.node_origin(), ws.node_origin())
    for t in range(3):
        assert all(np.array_equal(x, y) for x, y in zip(again.update(t).new_edges, ws.update(t).new_edges))


def test_sbm_stream_validates_budget():  # :235-241
    with pytest.raises(wire.StreamError, match="stream needs more nodes than the model has"):
        wire.sbm_dynamic(50, 2, 0.2, 0.0, 40, 2, 10, 0)


# ------------------------------------------------------------- wire format
def same_stream(a, b):
    assert (a.n0, a.steps, a.name) == (b.n0, b.steps, b.name)
    for x, y in zip(a.initial_edges(), b.initial_edges()):
        assert np.array_equal(x, y)
    for t in range(a.steps):
        ua, ub = a.update(t), b.update(t)
        assert ua.n_new == ub.n_new and a.n_old(t) == b.n_old(t)
        for x, y in zip(ua.added + ua.removed + ua.new_edges, ub.added + ub.removed + ub.new_edges):
            assert np.array_equal(x, y)
    assert np.array_equal(a.node_origin(), b.node_origin())
    assert np.array_equal(a.labels(), b.labels())


def test_wire_round_trip(tmp_path):
    for ws in (wire.config(1, size=3000, steps=3), wire.sbm_dynamic(120, 3, 0.2, 0.01, 80, 3, 10, 21),
               wire.config(4, size=1 << 12, steps=2)):
        p = str(tmp_path / "s.stub")
        ws.save(p)
        same_stream(ws, wire.load(p))
        with open(p, "rb") as f:
            assert f.read(8) == b"STUB0001"


def test_numpy_stream_through_the_wire(tmp_path):
    s = streams.config1(n=2000, steps=3)
    p = str(tmp_path / "np.stub")
    wire.from_stream(s).save(p)
    back = wire.load(p).to_stream()
    assert back.n0 == s.n0 and np.array_equal(back.keys0, np.sort(s.keys0))
    for ua, ub in zip(s.updates, back.updates):
        assert ua.n_new == ub.n_new
        for x, y in zip(ua.added + ua.removed + ua.new_edges, ub.added + ub.removed + ub.new_edges):
            assert np.array_equal(np.asarray(x), np.asarray(y))


def test_wire_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.stub"
    p.write_bytes(b"NOTSTUB!" + b"\0" * 64)
    with pytest.raises(wire.StreamError, match="bad magic") as ex:
        wire.load(str(p))
    assert ex.value.kind == "io"
    good = tmp_path / "good.stub"
    wire.config(1, size=500, steps=2).save(str(good))
    data = good.read_bytes()
    (tmp_path / "trunc.stub").write_bytes(data[: len(data) // 2])
    with pytest.raises(wire.StreamError, match="truncated"):
        wire.load(str(tmp_path / "trunc.stub"))
    with pytest.raises(wire.StreamError, match="cannot open"):
        wire.load(str(tmp_path / "missing.stub"))


def test_wire_header_layout(tmp_path):
    ws = wire.config(1, size=400, steps=1)
    p = tmp_path / "h.stub"
    ws.save(str(p))
    magic, n0, m0, steps, flags, nl = struct.unpack("<8s5q", p.read_bytes()[:48])
    assert (magic, n0, m0, steps, flags) == (b"STUB0001", 400, len(ws.initial_edges()[0]), 1, 0)
    assert p.read_bytes()[48:48 + nl].decode() == ws.name


# ------------------------------------------------------- BASELINE generators
def keyset(i, j):
    return set(zip(np.minimum(i, j).tolist(), np.maximum(i, j).tolist()))


def test_config_rules_cfg1_cfg2():
    for which, n, T in ((1, 3000, 3), (2, 4000, 3)):
        ws = wire.config(which, size=n, steps=T)
        i, j, _ = ws.initial_edges()
        assert np.all(i < j) and len(keyset(i, j)) == len(i)
        e = keyset(i, j)
        for t in range(T):
            u = ws.update(t)
            m = len(e)
            add, rem = keyset(*u.added[:2]), keyset(*u.removed)
            assert len(rem) == (100 if which == 1 else m // 200) and rem <= e
            assert len(add) == (500 if which == 1 else m // 100) and not (add & e) and not (add & rem)
            assert u.n_new == 0 and len(u.new_edges[0]) == 0
            e = (e - rem) | add
    # determinism and seed dependence
    a, b, c = wire.config(1, 2000, 2), wire.config(1, 2000, 2), wire.config(1, 2000, 2, seed=9)
    same_stream(a, b)
    assert not np.array_equal(a.initial_edges()[0], c.initial_edges()[0])


def test_config_rules_rmat_pa():
    ws = wire.config(3, size=12, steps=3)
    n = 1 << 12
    i, j, _ = ws.initial_edges()
    assert np.all(i < j) and np.all(j < n) and len(keyset(i, j)) == len(i)
    e = keyset(i, j)
    deg = np.bincount(np.concatenate([i, j]), minlength=n)
    assert deg.max() > 20 * max(1.0, deg.mean())  # heavy tail of R-MAT
    cur = n
    for t in range(3):
        u = ws.update(t)
        assert u.n_new == cur // 100 and ws.n_old(t) == cur
        ni, nj = u.new_edges[0], u.new_edges[1]
        assert np.all(nj >= cur) and np.all(ni < cur)  # newcomer edges go to pre-step nodes
        per = np.bincount(nj - cur, minlength=u.n_new)
        assert np.all(per == 10)  # 10 distinct targets each
        rem = keyset(*u.removed)
        assert len(rem) == len(e) // 200 and rem <= e
        e = (e - rem) | keyset(ni, nj)
        cur += u.n_new


def test_config_rules_cfg4_removal_as_isolation():
    ws = wire.config(4, size=1 << 13, steps=2)
    i, j, _ = ws.initial_edges()
    e = keyset(i, j)
    cur = ws.n0
    for t in range(2):
        u = ws.update(t)
        rem = keyset(*u.removed)
        assert rem <= e
        after = (e - rem) | keyset(*u.added[:2])
        # isolated ids: every edge of a removed node is in the batch and none is added back
        deg_after = np.bincount(np.array([x for p in after for x in p], np.int64), minlength=cur)
        gone = [v for v in set(x for p in rem for x in p) if deg_after[v] == 0]
        assert len(gone) >= 1
        assert u.n_new == cur // 200 and np.all(np.bincount(u.new_edges[1] - cur, minlength=u.n_new) <= 16)
        e = after | keyset(*u.new_edges[:2])
        cur += u.n_new


def test_generated_batches_pass_assemble_update():
    """Every batch of the C++ generators is valid for the CPU oracle's
    assemble_update/apply_update (graph.cpp:45-115), and the oracle's CSR after
    each step equals the set algebra of the edit lists."""
    import pyoracle as po

    for ws in (wire.config(1, size=1500, steps=2), wire.config(3, size=11, steps=2),
               wire.config(4, size=1 << 12, steps=2), wire.sbm_dynamic(300, 3, 0.1, 0.01, 200, 3, 20, 4)):
        rp, col, val = ws.csr0()
        n = len(rp) - 1
        x = np.linalg.qr(np.random.default_rng(0).standard_normal((n, 4)))[0]
        o = po.Session(po.Csr(n, rp, col, val), kind="grest2", k=4, seed=0, values=np.ones(4), vectors=x)
        a = dense_initial(ws)
        for t in range(ws.steps):
            u = ws.update(t)
            o.step(u)
            a = apply_dense(a, u)
            c = o.csr(0)
            d = np.zeros_like(a)
            for r in range(a.shape[0]):
                d[r, c.col[c.rowptr[r]:c.rowptr[r + 1]]] = c.val[c.rowptr[r]:c.rowptr[r + 1]]
            assert np.array_equal(d, a), (ws.name, t)


def test_cpp_stream_replay_compiles():
    """The C++ consumer of the wire format (tests/cpp/stream_replay.cpp) builds
    against both C ABIs (run on the GPU in test_gpu_wire)."""
    from paper_2603_19439_b200 import _build

    _build.build_stream()
    out = os.path.join(ROOT, "tests", "cpp", "_build", "stream_replay")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    pkg = os.path.join(ROOT, "paper_2603_19439_b200")
    if not os.path.exists(os.path.join(pkg, "libspectrack_b200.so")):
        _build.build()
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "stream_replay.cpp"), "-o", out, "-L", pkg, "-lspectrack_b200",
           "-lspectrack_stream", "-Wl,-rpath," + pkg, "-L/usr/local/cuda/lib64", "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    assert os.path.exists(out)
