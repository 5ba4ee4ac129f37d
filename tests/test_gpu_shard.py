"""Row-sharded step against the CPU oracle: 1, 2 and 3 ranks
on the test box's single GPU, collectives staged through host memory over
gloo (tests/shard_worker.py). Rank 0 checks every rank's rows of A bit-exact,
the perturbation bit-exact, Ritz values (1e-10) and the reassembled span (sin
1e-8) after every step, then that an invalid deletion fails on every rank with
the reference's message and leaves the state untouched."""
import os
import socket
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(world, case, chunk=4, comm="staged"):
    import torch.multiprocessing as mp

    sys.path.insert(0, HERE)
    import shard_worker

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=shard_worker.run, args=(r, world, port, case, chunk, q, comm)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    fails = [r for r in res if r[1] != "ok"]
    assert not fails, "\n".join(f"rank {r[0]}:\n{r[2]}" for r in fails)
    rep = [r for r in res if r[0] == 0][0]
    for t, ve, sa in rep[2]:
        print(f"{case} world {world} step {t}: value err {ve:.2e}, subspace sin {sa:.2e}; comm {rep[3]}")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["rsvd_small", "rsvd_bypass", "grest2", "grest3", "iasc", "dense"])
def test_sharded_two_ranks(case):
    _run(2, case)


@pytest.mark.gpu
def test_sharded_three_ranks_rsvd():
    _run(3, "rsvd_small", chunk=3)


@pytest.mark.gpu
def test_sharded_one_rank():
    _run(1, "rsvd_small")


@pytest.mark.gpu
def test_sharded_rmat_two_ranks():
    _run(2, "rmat13", chunk=16)


@pytest.mark.gpu
def test_sharded_config3_shape_two_ranks():
    """Config 3's shapes (R-MAT s15, k = 32, L = P = 100: q = 200 sketch, D = 164)
    row-sharded over two ranks."""
    _run(2, "cfg3_s15", chunk=64)


@pytest.mark.gpu
def test_sharded_native_nccl_comm_one_rank():
    """The library's own NCCL communicator (st_comm_nccl_create): allreduce,
    allgather and the alltoallv halo enqueued on the session stream."""
    _run(1, "cfg3_s15", chunk=64, comm="nccl")
