"""Rank body of the row-sharded parity tests (tests/test_gpu_shard.py).

Each rank runs one ShardedTrackerSession on cuda:0 with the collectives staged
through host memory over gloo (several ranks share the single GPU of the test
box; no kernel of one rank ever waits on another's). Rank 0 also runs the CPU
oracle on the same stream and checks, after every step, the reassembled state:
each rank's rows of A bit-exact against the oracle's rows, the perturbation
bit-exact, Ritz values within 1e-10 and the span of the reassembled X within
sin 1e-8 (the single-GPU parity contract, harness.py).
"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cases():
    import numpy as np

    from harness import random_update, edges_of
    from support import random_graph

    def random_stream(kind, L, P, dense, steps=4, n=160):
        a = random_graph(n, 0.05, 31)
        rng = np.random.default_rng(5)
        cfg = dict(kind=kind, k=6, rsvd_l=L, rsvd_p=P, seed=3, force_dense=dense)
        return a.rowptr, a.col, a.val, cfg, ("random", rng, steps)

    def rmat(steps=2):
        from paper_2603_19439_b200 import streams

        keys = streams.rmat_keys(13, 16, seed=7)
        s = streams.edit_stream(1 << 13, keys, steps, 8, lambda m: 0, lambda m: 0.005 * m,
                                new_nodes=lambda nn: nn // 50, new_degree=10)
        rp, col, val = s.csr0()
        return rp, col, val, dict(kind="grest-rsvd", k=8, seed=11), ("fixed", s.updates)

    def cfg3_s15(steps=2):
        from paper_2603_19439_b200 import streams

        s = streams.config3(scale=15, steps=steps)
        rp, col, val = s.csr0()
        return rp, col, val, dict(kind="grest-rsvd", k=32, seed=5), ("fixed", s.updates), "init_eig"

    return {
        "cfg3_s15": cfg3_s15,
        "rsvd_small": lambda: random_stream("grest-rsvd", 4, 3, False),
        "rsvd_bypass": lambda: random_stream("grest-rsvd", 100, 100, False),
        "grest2": lambda: random_stream("grest2", 100, 100, False),
        "grest3": lambda: random_stream("grest3", 100, 100, False),
        "iasc": lambda: random_stream("iasc", 100, 100, False),
        "dense": lambda: random_stream("grest-rsvd", 4, 3, True),
        "rmat13": rmat,
    }


def run(rank, world, port, case, chunk, q, comm_kind="staged"):
    try:
        os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
        for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
            sys.path.insert(0, p)
        import numpy as np
        import torch.distributed as dist

        import pyoracle as po
        from harness import SIN_TOL, VALUE_RTOL, edges_of, random_update, sin_angle, value_err
        from paper_2603_19439_b200 import TrackerError
        from paper_2603_19439_b200.shard import NcclComm, ShardedTrackerSession, TorchComm, local_block, shard_bounds

        dist.init_process_group("gloo", rank=rank, world_size=world)
        rp, col, val, cfg, stream, *init = _cases()[case]()
        n = len(rp) - 1
        a = po.Csr(n, np.asarray(rp, np.int32), np.asarray(col, np.int32), np.asarray(val, np.float64))
        ocfg = {k: v for k, v in cfg.items() if k != "force_dense"}
        if init:  # leading eigenpairs from rank 0 (block Krylov on the GPU), shared by all ranks
            from paper_2603_19439_b200 import init_eig

            box = [None]
            if rank == 0:
                box[0] = init_eig.leading_eigenpairs(rp, col, val, cfg["k"], "abs_desc", device="cuda:0")
            dist.broadcast_object_list(box, src=0)
            vals, vecs = box[0]
            orc = po.Session(a, values=vals, vectors=vecs, **ocfg)
        else:
            orc = po.Session(a, **ocfg)
            vals, vecs = orc.embedding()
        bounds = shard_bounds(a.rowptr, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        lrp, lcol, lval, lx = local_block(a.rowptr, a.col, a.val, vecs, lo, hi)
        # "staged": collectives through host memory over gloo (several ranks on
        # one GPU); "nccl": the library's own NCCL communicator (one rank per GPU)
        comm = TorchComm("staged") if comm_kind == "staged" else NcclComm(device=0)
        g = ShardedTrackerSession(comm, n, lo, hi, lrp, lcol, lval, vals, lx, chunk=chunk, **cfg)
        rng = stream[1] if stream[0] == "random" else None
        nsteps = stream[2] if stream[0] == "random" else len(stream[1])
        report = []
        for t in range(nsteps):
            if rng is not None:
                # every rank draws the same update from the oracle's (rank 0's) edge set
                cur = orc.info()[0]
                oc = orc.csr(0)
                upd = random_update(rng, edges_of((oc.rowptr, oc.col, oc.val)), cur, 6, 3,
                                    9 if t % 2 == 0 else 0, 3)
            else:
                upd = stream[1][t]
            g.step(upd)
            orc.step(upd)
            gv, gx, ids = g.embedding()
            grp, gcol, gval = g.csr(0)
            dl = g.csr(2)
            parts = [None] * world
            dist.all_gather_object(parts, (gv, gx, ids, grp, gcol, gval, dl))
            if rank == 0:
                ov, ox = orc.embedding()
                X = np.zeros_like(ox)
                seen = np.zeros(len(ox), bool)
                oc = orc.csr(0)
                for (v, x, idr, rpp, cc, vv, d) in parts:
                    assert np.array_equal(v, gv), "Ritz values differ across ranks"
                    X[idr] = x
                    seen[idr] = True
                    for li, gi in enumerate(idr):
                        s0, s1 = oc.rowptr[gi], oc.rowptr[gi + 1]
                        assert np.array_equal(cc[rpp[li]:rpp[li + 1]], oc.col[s0:s1]), f"step {t}: row {gi} cols"
                        assert np.array_equal(vv[rpp[li]:rpp[li + 1]], oc.val[s0:s1]), f"step {t}: row {gi} vals"
                    od = orc.csr(2)
                    assert np.array_equal(d[0], od.rowptr) and np.array_equal(d[1], od.col) and \
                        np.array_equal(d[2], od.val), f"step {t}: perturbation differs"
                assert seen.all(), "rows not covered by the shards"
                ve = value_err(gv, ov)
                sa = sin_angle(X, ox)
                assert ve <= VALUE_RTOL, f"step {t}: ritz value error {ve:.3e}"
                assert sa <= SIN_TOL, f"step {t}: subspace sin {sa:.3e}"
                report.append((t, ve, sa))
        # an invalid deletion fails on every rank with the reference message and leaves the state
        from paper_2603_19439_b200 import Update

        cur = g.info()["n"]
        before = g.embedding()
        oc = orc.csr(0)
        present = set(map(tuple, edges_of((oc.rowptr, oc.col, oc.val))))
        bad = next((i, j) for i in range(cur) for j in range(i + 1, cur) if (i, j) not in present)
        try:
            g.step(Update.make((), [bad], 0, ()))
            msg = None
        except TrackerError as e:
            msg = str(e)
        after = g.embedding()
        assert msg == "apply_update: invalid deletion (no such edge)", msg
        assert np.array_equal(before[1], after[1]) and g.info()["n"] == cur
        q.put((rank, "ok", report, dict(comm.calls, **g.halo_stats())))
        dist.destroy_process_group()
    except Exception:
        q.put((rank, "fail", traceback.format_exc(), None))
