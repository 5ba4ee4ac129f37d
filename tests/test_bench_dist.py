"""The multi-rank plumbing of bench.py on CPU (gloo, world size 2): rendezvous
from the torchrun environment, max-over-ranks timing, barrier."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), BENCH_DIST_BACKEND="gloo")
    sys.path.insert(0, ROOT)
    import bench
    import torch.distributed as dist

    w, r, _ = bench.dist_setup()
    bench.barrier(w)
    m = bench.dist_max(10.0 * (r + 1), w)
    q.put((r, w, m))
    dist.destroy_process_group()


def test_dist_max_over_two_gloo_ranks():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert [r for r, _, _ in res] == [0, 1]
    assert all(w == 2 and m == 20.0 for _, w, m in res)


def test_reference_arm_nonzero_ranks_exit_quietly(capsys, monkeypatch):
    sys.path.insert(0, ROOT)
    import bench

    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")

    class A:
        warmup, steps, config, scale = 1, 1, "cfg1", None

    bench.run_reference(A())
    assert capsys.readouterr().out == ""


def test_bench_module_defines_every_leg():
    """bench.py's legs import and the clock sampler degrades without nvidia-smi
    (a broken module would only show up on the GPU box)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    for name in ("ClockSampler", "run_ours", "run_reference", "cpu_baseline", "make_workload", "dist_max", "main"):
        assert hasattr(m, name), name
    c = m.ClockSampler(0)
    c.proc = None
    out = c.stop()
    assert set(out) == {"sm_mhz", "sm_max_mhz", "reasons", "samples"}
