"""Host side of the row-sharded sessions on CPU (no GPU): the closed-form
ownership map (st_shard_layout, csrc/shard.cuh) partitions the nodes for any
rank count, initial blocks and chunk as nodes are appended, and two gloo ranks
that each compute only their own rows tile [0, n) exactly; the row-block split
of the initial CSR is balanced and contiguous."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("size,chunk", [(1, 5), (2, 1), (3, 4), (8, 256)])
def test_layout_partitions_nodes(size, chunk):
    from paper_2603_19439_b200.shard import layout

    rng = np.random.default_rng(size * 100 + chunk)
    n0 = 1000
    cuts = np.sort(rng.choice(np.arange(1, n0), size - 1, replace=False)) if size > 1 else np.array([], int)
    bounds = np.concatenate([[0], cuts, [n0]]).astype(np.int64)
    prev = [layout(bounds, chunk, r, n0) for r in range(size)]
    for n_total in sorted([n0, n0 + 1, n0 + chunk * size - 1, n0 + 3 * chunk * size + 7, 5000]):
        parts = [layout(bounds, chunk, r, n_total) for r in range(size)]
        allids = np.concatenate(parts)
        assert np.array_equal(np.sort(allids), np.arange(n_total))
        for r, p in enumerate(parts):
            assert np.all(np.diff(p) > 0)  # local order = global order
            assert np.array_equal(p[: len(prev[r])], prev[r])  # appended rows never move
            assert np.array_equal(p[: bounds[r + 1] - bounds[r]], np.arange(bounds[r], bounds[r + 1]))
        prev = parts


def test_shard_bounds_balanced_and_contiguous():
    from paper_2603_19439_b200 import streams
    from paper_2603_19439_b200.shard import local_block, shard_bounds

    keys = streams.rmat_keys(12, 16, seed=1)
    s = streams.edit_stream(1 << 12, keys, 1, 8, lambda m: 0, lambda m: 0, new_nodes=lambda nn: 0, new_degree=1)
    rp, col, val = s.csr0()
    n = len(rp) - 1
    b = shard_bounds(rp, 4)
    assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
    w = [(rp[b[r + 1]] - rp[b[r]]) + (b[r + 1] - b[r]) for r in range(4)]
    assert max(w) <= 1.2 * (sum(w) / 4) + max(np.diff(rp)) + 1
    x = np.arange(n * 3, dtype=float).reshape(n, 3)
    rebuilt = []
    for r in range(4):
        lrp, lcol, lval, lx = local_block(rp, col, val, x, b[r], b[r + 1])
        assert lrp[0] == 0 and len(lrp) == b[r + 1] - b[r] + 1 and np.array_equal(lx, x[b[r]:b[r + 1]])
        rebuilt.append(lcol)
    assert np.array_equal(np.concatenate(rebuilt), col)


def _gloo_rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2603_19439_b200.shard import layout

    dist.init_process_group("gloo", rank=rank, world_size=world)
    bounds = np.array([0, 37, 100], np.int64)
    mine = layout(bounds, 8, rank, 171)
    sizes = [None] * world
    dist.all_gather_object(sizes, mine.tolist())
    t = torch.tensor([len(mine)], dtype=torch.int64)
    dist.all_reduce(t)
    q.put((rank, sizes, int(t)))
    dist.destroy_process_group()


def test_two_gloo_ranks_tile_the_nodes():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for rank, sizes, total in res:
        assert total == 171
        ids = sorted(sizes[0] + sizes[1])
        assert ids == list(range(171))
