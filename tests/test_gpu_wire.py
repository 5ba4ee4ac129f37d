"""Streams from the C++ generator library, read back from the wire format, on
the CUDA path: oracle parity per step (CSR bit-exact, Ritz values 1e-10
relative, sin(largest principal angle) <= 1e-8), and the C++ consumer
(tests/cpp/stream_replay.cpp, through include/spectrack_b200.hpp) replaying a
file bit-identically to the Python binding."""
import os
import subprocess

import numpy as np
import pytest

import pyoracle as po
from harness import SIN_TOL, csr_equal, sin_angle
from test_wire import ROOT

pytestmark = pytest.mark.gpu


def test_wire_stream_parity(tmp_path):
    from paper_2603_19439_b200 import TrackerSession, wire

    path = str(tmp_path / "cfg3s14.stub")
    wire.config(3, size=14, steps=3).save(path)  # R-MAT s14, 1% PA newcomers (163 > L: RSVD active)
    ws = wire.load(path)
    rp, col, val = ws.csr0()
    n, k = len(rp) - 1, 16
    g = TrackerSession.tracker_init(rp, col, val, k, kind="grest-rsvd", seed=3)
    v0, x0 = g.embedding()
    o = po.Session(po.Csr(n, rp, col, val), kind="grest-rsvd", k=k, seed=3, values=v0, vectors=x0)
    for t in range(ws.steps):
        u = ws.update(t)
        g.step(u)
        o.step(u)
        gv, gx = g.embedding()
        ov, ox = o.embedding()
        assert csr_equal(g.csr(0), o.csr(0)) and csr_equal(g.csr(2), o.csr(2))
        ve = float(np.max(np.abs(gv - ov) / np.abs(ov)))
        sa = sin_angle(gx, ox)
        print(f"wire cfg3 s14 step {t}: ritz rel err {ve:.2e} sin {sa:.2e}")
        assert ve <= 1e-10 and sa <= SIN_TOL


def test_cpp_stream_replay_matches_python(tmp_path):
    from paper_2603_19439_b200 import TrackerSession, wire
    from test_wire import test_cpp_stream_replay_compiles

    test_cpp_stream_replay_compiles()
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "stream_replay")
    path = str(tmp_path / "sbm.stub")
    wire.sbm_dynamic(3000, 4, 0.02, 0.002, 2000, 4, 150, 17).save(path)  # 150 newcomers > L = 100
    out_vals = str(tmp_path / "vals.bin")
    r = subprocess.run([exe, path, "8", "grest-rsvd", out_vals], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "stream_replay: ok" in r.stdout
    cpp = np.fromfile(out_vals, np.float64).reshape(-1, 8)
    ws = wire.load(path)
    rp, col, val = ws.csr0()
    g = TrackerSession.tracker_init(rp, col, val, 8, kind="grest-rsvd", seed=0)
    py = [g.embedding()[0]]
    for t in range(ws.steps):
        g.step(ws.update(t))
        py.append(g.embedding()[0])
    assert np.array_equal(cpp, np.array(py))  # same library, same inputs: bit-identical
