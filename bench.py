#!/usr/bin/env python
"""Benchmark of the B200 G-REST per-step eigen-update (BASELINE.json metric).

One "step" = one update batch through the whole hot path: on-device
validation/assembly of Delta, the CSR merge A <- pad(A) + Delta, and
tracker_step (grest-rsvd, k=32, L=P=100) on R-MAT scale 20 (config 3).

  value : steps/s with the edit lists already resident in HBM (st_step_device)
  e2e   : steps/s through the C ABI with host edit lists (H2D inside the timed
          region) and the k Ritz values read back every step
  roofline : the dominant kernel class, algorithmic work / CUDA-event time
  cpu_baseline : the CPU restatement (oracle/) on one step of the same stream

`--impl reference` times the reference's CPU implementation of the path (the
oracle port: the reference itself cannot be built here) with all
host threads on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "eigen-update steps/s at R-MAT s20 k=32; SpMM+Gram GB/s vs HBM peak"
HBM_PEAK_FALLBACK = 6650.0
# FP64 tensor (DMMA) peak: not in MEASURED_PEAKS.json; measured by us on this
# pool with cuBLAS DGEMM 8192^3 (profiles/fp64_peaks_r01.txt).
FP64_PEAK_MEASURED = 35.46
FLOP_CLASSES = ("dmma_gram", "dmma_gemm", "masked_gram_x", "dmma_gram_narrow", "dmma_gemm_narrow")


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback (B200_PROFILING.md)"


def make_workload(name: str, steps: int, seed_offset: int = 0, scale: int | None = None):
    from paper_2603_19439_b200 import streams

    if name == "cfg3":
        s = streams.config3(seed=3 + seed_offset, scale=scale or 20, steps=steps)
        return s, dict(k=32, kind="grest-rsvd", order="abs_desc", operator="adjacency",
                       workload=f"cfg3 R-MAT scale {scale or 20} ef16 (0.57,0.19,0.19,0.05) symmetrized+dedup, "
                                f"k=32 grest-rsvd L=P=100; per step 1% new nodes x 10 PA edges + 0.5% deletions")
    if name == "cfg1":
        s = streams.config1(seed=1 + seed_offset, steps=steps)
        return s, dict(k=8, kind="grest-rsvd", order="abs_desc", operator="adjacency",
                       workload="cfg1 SBM n=10,000 4 blocks p_in=0.01 p_out=0.001, k=8; 500 inserts + 100 deletes")
    if name == "cfg4":
        s = streams.config4(seed=4 + seed_offset, steps=steps, n=1 << (scale or 22))
        return s, dict(k=64, kind="grest-rsvd", order="abs_desc", operator="adjacency",
                       workload=f"cfg4 SBM n=2^{scale or 22} 64 blocks avg deg 32 (80% intra), k=64 grest-rsvd "
                                f"L=P=100; per step 1% inserts + 0.5% deletes + 0.5% new nodes x 16 edges + 0.1% "
                                f"node removals")
    if name == "cfg5":
        import torch

        sc = scale or 25
        s = streams.config5(seed=5 + seed_offset, scale=sc, steps=steps, device=f"cuda:{torch.cuda.current_device()}")
        return s, dict(k=32, kind="grest-rsvd", order="abs_desc", operator="adjacency",
                       workload=f"cfg5 R-MAT scale {sc} ef16 (0.57,0.19,0.19,0.05) symmetrized+dedup, k=32 "
                                f"grest-rsvd L=P=100; per step 0.1% edge inserts + 0.1% new nodes x 16 PA edges "
                                f"(graph generated on the GPU with torch's generator)")
    if name == "cfg2":
        s = streams.config2(seed=2 + seed_offset, steps=steps)
        return s, dict(k=16, kind="grest-rsvd", order="alg_desc", operator="normalized-laplacian",
                       workload="cfg2 ER n=100,000 avg deg 20 normalized Laplacian k=16; 1% inserts + 0.5% deletes")
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6 for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_setup(backend: str | None = None):
    """One process per GPU (torchrun env); NCCL on GPUs, gloo for CPU tests."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = backend or os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def dist_max(x: float, world: int) -> float:
    """Max over ranks of a per-rank device time (the job's time is the slowest rank's)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_baseline(stream, x0_vals, x0_vecs, wl, threads: int):
    """The oracle (CPU port of the reference path) on one step of the stream."""
    os.environ["OMP_NUM_THREADS"] = str(threads)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    rp, col, val = stream.csr0()
    a = po.Csr(len(rp) - 1, rp, col, val)
    o = po.Session(a, kind=wl["kind"], k=wl["k"], order=wl["order"], operator=wl["operator"], seed=0,
                   values=x0_vals, vectors=x0_vecs)
    t0 = time.perf_counter()
    o.step(stream.updates[0])
    dt = time.perf_counter() - t0
    return dt, o.last_tracker_seconds


def _free_port() -> int:
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def run_ours(args):
    # native libraries (NCCL's banner, ...) may write to fd 1: keep it on
    # stderr until the one JSON line is printed
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    try:
        _run_ours(args, saved_stdout)
    finally:
        sys.stdout.flush()
        os.dup2(saved_stdout, 1)
        os.close(saved_stdout)


def _run_ours(args, saved_stdout):
    import torch

    from paper_2603_19439_b200 import KERNEL_CLASSES, DeviceUpdate, TrackerSession

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    W, K = args.warmup, args.steps
    t_setup = time.time()
    replicas = world > 1 and args.replicas
    stream, wl = make_workload(args.config, W + K, seed_offset=rank if replicas else 0, scale=args.scale)
    if args.k:
        wl["k"] = args.k
        wl["workload"] = wl["workload"].replace("k=32", f"k={args.k}").replace("k=64", f"k={args.k}")
    if hasattr(stream, "csr0_torch"):  # config 5: the start graph was generated on the device
        rp, col, val = stream.csr0()
        stream.release()
        torch.cuda.empty_cache()
    else:
        rp, col, val = stream.csr0()
    # X0, Lambda0: the library's own tracker_init (thick-restart Lanczos on the
    # device, lanczos.hpp:38-127 / trackers.cpp:132-145), outside every timed region
    t_init = time.time()
    g0 = TrackerSession.tracker_init(rp, col, val, wl["k"], kind=wl["kind"], order=wl["order"],
                                     operator=wl["operator"], seed=0, device=local)
    vals0, vecs0 = g0.embedding()
    init_stats = g0.init_stats()
    g0.close()
    del g0
    torch.cuda.synchronize()
    init_s = time.time() - t_init
    setup_s = time.time() - t_setup
    kw = dict(kind=wl["kind"], k=wl["k"], order=wl["order"], operator=wl["operator"], seed=0, device=local)

    sharded = args.sharded or (world > 1 and not args.replicas)
    comm = None
    if sharded:
        import torch.distributed as dist

        from paper_2603_19439_b200.shard import (NcclComm, ShardedTrackerSession, TorchComm, local_block,
                                                 shard_bounds)

        if not dist.is_initialized():  # --sharded on one GPU: a one-rank NCCL group
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
        # the library's own NCCL communicator (collectives enqueued by the
        # library on the session stream); --torch-comm: torch.distributed callbacks
        comm = TorchComm("nccl") if args.torch_comm else NcclComm(device=local)
        bounds = shard_bounds(rp, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        blk = local_block(rp, col, val, vecs0, lo, hi)
        kw_sh = {k_: v for k_, v in kw.items() if k_ != "operator"}

    # capacity for the whole stream (final node count; stored entries bounded by
    # the inserts), so no step inside a timed region grows a device buffer
    n_cap = len(rp) - 1 + sum(int(u.n_new) for u in stream.updates)
    nnz_cap = int(rp[-1]) + 2 * sum(len(u.added[0]) + len(u.new_edges[0]) for u in stream.updates)

    def new_session(kernel_timing=False):
        if sharded:
            s_ = ShardedTrackerSession(comm, len(rp) - 1, lo, hi, blk[0], blk[1], blk[2], vals0, blk[3],
                                       chunk=1024, kernel_timing=kernel_timing, **kw_sh)
        else:
            s_ = TrackerSession(rp, col, val, vals0, vecs0, kernel_timing=kernel_timing, timing=kernel_timing, **kw)
        s_.reserve(n_cap, nnz_cap)
        return s_

    # ---- value: edit lists resident in HBM (no per-launch timing events)
    dev_updates = [DeviceUpdate(u, device=f"cuda:{local}") for u in stream.updates]
    sess = new_session()
    for t in range(W):
        sess.step_device(dev_updates[t])
    torch.cuda.synchronize()
    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    launches = 0
    halo0 = sess.halo_stats() if sharded else None
    torch.cuda.synchronize()
    e0.record()
    for t in range(W, W + K):
        sess.step_device(dev_updates[t])
        marks[t - W].record()  # after the step's work on the session stream (no host sync)
        launches += sess.launches()
    torch.cuda.synchronize()  # the session's side streams included
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = dist_max(e0.elapsed_time(e1), world)
    step_ms = [e0.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i]) for i in range(1, K)]
    info = sess.info()
    halo = ({k_: v - halo0[k_] for k_, v in sess.halo_stats().items()} if sharded else None)
    sess.close()

    # ---- per-kernel-class device time: the same steps again, CUDA events
    # around every launch (ST_FLAG_KERNEL_TIMING), outside the timed region
    sess = new_session(kernel_timing=True)
    sess.set_peaks(FP64_PEAK_MEASURED, measured_peaks()[0])
    for t in range(W):
        sess.step_device(dev_updates[t])
    sess.reset_kernel_stats()
    tracker_ms = []
    for t in range(W, W + K):
        sess.step_device(dev_updates[t])
        ph = sess.timings() if not sharded else []
        if len(ph) >= 6:  # [ingest, basis, rr_gram, eig, rotate, total]: the step after ingestion
            tracker_ms.append(ph[5] - ph[0])
    torch.cuda.synchronize()
    kstats = sess.kernel_stats()
    sess.close()
    del dev_updates

    # ---- e2e: host edit lists (page-locked, as a streaming caller keeps its
    # batch buffers) through the C ABI, Ritz values read back
    host_updates = [u.pinned() for u in stream.updates]
    sess = new_session()
    for t in range(W):
        sess.step(host_updates[t])
    torch.cuda.synchronize()
    barrier(world)
    h2d = 0
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fmarks = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    f0.record()
    for t in range(W, W + K):
        sess.step(host_updates[t])
        _ = sess.values()
        fmarks[t - W].record()
        h2d += host_updates[t].h2d_bytes()
    torch.cuda.synchronize()
    f1.record()
    torch.cuda.synchronize()
    ms_e2e = dist_max(f0.elapsed_time(f1), world)
    step_ms_e2e = [f0.elapsed_time(fmarks[0])] + [fmarks[i - 1].elapsed_time(fmarks[i]) for i in range(1, K)]
    sess.close()

    streams_run = 1 if sharded else world  # one row-sharded stream, or one stream per replica
    value = streams_run * K / (ms / 1e3)
    e2e = streams_run * K / (ms_e2e / 1e3)
    hbm_peak, hbm_src = measured_peaks()

    # ---- roofline of the dominant kernel class (by device time)
    classes = {}
    for name in KERNEL_CLASSES:
        st = kstats[name]
        if st["launches"] == 0:
            continue
        flops_class = name in FLOP_CLASSES
        byte_class = name in ("spmm", "spmm_sketch", "csr_merge", "rotate_x")
        ach = st["work"] / (st["ms"] / 1e3) if st["ms"] > 0 else 0.0
        row = dict(ms_per_step=st["ms"] / K, launches_per_step=st["launches"] / K,
                   share=st["ms"] / ms if ms > 0 else 0.0)
        if flops_class:
            row.update(achieved_tflops=ach / 1e12, frac_fp64_peak=ach / 1e12 / FP64_PEAK_MEASURED,
                       achieved_gbs=st["work2"] / (st["ms"] / 1e3) / 1e9 if st["ms"] > 0 else 0.0)
        elif byte_class:
            row.update(achieved_gbs=ach / 1e9, frac_hbm=ach / 1e9 / hbm_peak)
        if (flops_class or byte_class) and st["ms"] > 0:
            # per-launch roofline time max(flops / F, bytes / B) summed, over the measured time
            row["frac_of_roofline_bound"] = st["bound_ms"] / st["ms"]
        classes[name] = row
    # the roofline kernel: the largest class on the step's critical stream (the eigensolver is latency-bound;
    # the CSR merge builds the NEXT step's A on a low-priority side stream, its event time includes starvation)
    own = {k_: v for k_, v in classes.items() if k_ not in ("eigensolver", "csr_merge")}
    dom = max(own, key=lambda k_: own[k_]["ms_per_step"]) if own else None
    roof = None
    traffic = {}
    try:  # DRAM bytes of one representative launch per class, from the committed ncu --set full capture
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "roofline_traffic.json")) as fh:
            traffic = json.load(fh)
    except (OSError, ValueError):
        traffic = {}
    if dom is not None:
        st = kstats[dom]
        ach = st["work"] / (st["ms"] / 1e3)
        if dom in FLOP_CLASSES:
            tr = traffic.get(args.config, {}).get(dom)  # measured for this config, else null
            roof = dict(kernel=dom, bound="tensor", achieved=ach / 1e12, peak=FP64_PEAK_MEASURED, unit="TFLOP/s",
                        frac=ach / 1e12 / FP64_PEAK_MEASURED, traffic=tr["bytes_per_launch"] if tr else None,
                        traffic_launch=tr, 
                        peak_source="measured cuBLAS DGEMM 8192^3 on this pool (FP64 not in MEASURED_PEAKS.json)",
                        algorithmic_work_per_launch=st["work"] / st["launches"], unit_work="flop",
                        frac_of_roofline_bound=classes[dom].get("frac_of_roofline_bound"))
        else:
            roof = dict(kernel=dom, bound="hbm", achieved=ach / 1e9, peak=hbm_peak, unit="GB/s",
                        frac=ach / 1e9 / hbm_peak, traffic=None, peak_source=hbm_src,
                        algorithmic_work_per_launch=st["work"] / st["launches"], unit_work="byte",
                        frac_of_roofline_bound=classes[dom].get("frac_of_roofline_bound"))
    out = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded stream, BASELINE {args.config} shapes)",
        "config": {"workload": wl["workload"], "n0": int(len(rp) - 1), "nnz0": int(rp[-1]), "k": wl["k"],
                   "kind": wl["kind"], "rsvd_l": 100, "rsvd_p": 100, "n_final": info["n"],
                   "parallelism": (f"row-sharded over {world} GPU(s) (NCCL allreduce of Grams, boundary-row alltoallv halo)"
                                   if sharded else "single GPU" if world == 1 else f"{world} independent replicas"),
                   "l2": f"inputs larger than L2 (CSR {12 * int(rp[-1]) / 1e9:.2f} GB + X "
                         f"{8 * wl['k'] * (len(rp) - 1) / 1e9:.2f} GB per stream)",
                   "setup_s": round(setup_s, 1),
                   "x0": f"st_tracker_init (device thick-restart Lanczos, tol 1e-10): {init_s:.1f} s, "
                         f"{init_stats[0]} restarts, {init_stats[1]} operator products"},
        "roofline": roof,
        "kernel_classes": classes,
        "e2e": {"value": e2e, "unit": "steps/s", "ms_per_step": ms_e2e / K, "h2d_bytes_per_step": h2d // K,
                "d2h_bytes_per_step": 8 * wl["k"]},
        "tracker_step_only": ({"value": 1e3 / float(np.mean(tracker_ms)), "unit": "steps/s",
                               "ms_per_step": float(np.mean(tracker_ms)),
                               "what": "device time from the end of ingestion (validation, Delta, CSR merge "
                                       "launch, P) to the end of the step: the reference's step_seconds "
                                       "(experiment.cpp:202-204, tracker_step only); measured in the kernel-timing "
                                       "session, per-phase events"} if tracker_ms else None),
        "gpu_launches": launches,
        "step_ms": [round(x, 3) for x in step_ms],
        "step_ms_e2e": [round(x, 3) for x in step_ms_e2e],
        "clocks": clk,
    }
    if rank == 0 and world == 1 and args.config == "cfg5" and not args.no_cpu_baseline:
        out["cpu_baseline"] = {"value": None, "unit": "steps/s", "cores": os.cpu_count() or 1, "kind": "port",
                               "sample": "not run: one oracle step at R-MAT s25 is hours of CPU work and ~150 GB "
                                         "of host RAM (SURVEY.md 8(d)); see the cfg3 line for the CPU baseline"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = args.cpu_threads or os.cpu_count() or 1
        dt, dt_tracker = cpu_baseline(stream, vals0, vecs0, wl, threads)
        out["cpu_baseline"] = {"value": 1.0 / dt, "unit": "steps/s", "cores": threads, "kind": "port",
                               "sample": f"1 step (step {0}) of the same stream: assemble_update + apply_update + "
                                         f"tracker_step via the oracle restatement, OpenMP {threads} threads; "
                                         f"tracker_step alone {dt_tracker:.2f} s",
                               "seconds_per_step": dt}
    if comm is not None:
        out["comm"] = {"kind": "torch.distributed callbacks" if args.torch_comm else "library NCCL (st_comm_nccl)",
                       "halo_bytes_recv_per_step": halo["halo_bytes_recv"] / max(K, 1),
                       "halo_bytes_local_per_step": halo["halo_bytes_local"] / max(K, 1)}
    if rank == 0:
        sys.stdout.flush()
        os.write(saved_stdout, (json.dumps(out) + "\n").encode())
    if world > 1 or sharded:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_reference(args):
    """The reference's CPU path (oracle port; the reference cannot be built
    here: Eigen is absent) with all host threads, on the same config."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = args.cpu_threads or os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(threads)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    budget_s = 150.0
    stream, wl = make_workload(args.config, args.warmup + args.steps, scale=args.scale)
    # the GPU arm times steps [warmup, warmup + steps): start the CPU port at the
    # same graph (the first `warmup` batches applied to the edge set on the host,
    # set algebra, no tracking), one untimed step, then the same window
    skip = args.warmup if hasattr(stream, "keys0") else 0
    if skip:
        from paper_2603_19439_b200.streams import _EdgeSet, csr_from_keys

        es = _EdgeSet(stream.n0, stream.keys0)
        for t in range(skip):
            u = stream.updates[t]
            rk = np.minimum(u.removed[0], u.removed[1]) * (1 << 32) + np.maximum(u.removed[0], u.removed[1])
            ak = np.minimum(u.added[0], u.added[1]) * (1 << 32) + np.maximum(u.added[0], u.added[1])
            nk = np.minimum(u.new_edges[0], u.new_edges[1]) * (1 << 32) + np.maximum(u.new_edges[0], u.new_edges[1])
            es.apply(np.asarray(ak, np.int64), np.sort(np.asarray(rk, np.int64)), int(u.n_new), np.asarray(nk, np.int64))
        rp, col, val = csr_from_keys(es.n, es.keys)
    else:
        rp, col, val = stream.csr0()
    n = len(rp) - 1
    rng = np.random.default_rng(0)
    x, _ = np.linalg.qr(rng.standard_normal((n, wl["k"])))  # X0 quality does not change the step cost
    a = po.Csr(n, rp, col, val)
    o = po.Session(a, kind=wl["kind"], k=wl["k"], order=wl["order"], operator=wl["operator"], seed=0,
                   values=np.linspace(wl["k"], 1, wl["k"]), vectors=x)
    times = []
    for t in range(skip, skip + args.steps):
        t0 = time.perf_counter()
        o.step(stream.updates[t])
        times.append(time.perf_counter() - t0)
        if sum(times) > budget_s:
            break
    value = len(times) / sum(times)
    sample = (f"steps {skip}..{skip + len(times) - 1} of the stream ({len(times)} of {args.steps} requested, budget "
              f"{budget_s:.0f} s; the GPU arm's timed window starts at step {args.warmup}), the graph fast-forwarded "
              f"through the first {skip} batches on the host, oracle restatement with OpenMP {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["workload"], "n0": int(stream.n0), "nnz0": int(stream.nnz0() if hasattr(stream, "nnz0") else 2 * len(stream.keys0)),
                   "k": wl["k"], "kind": wl["kind"], "rsvd_l": 100, "rsvd_p": 100,
                   "timed_from": {"step": skip, "n": n, "nnz": int(rp[-1])}},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--scale", type=int, default=None, help="R-MAT scale override (development)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--k", type=int, default=None, help="tracked pairs override (the cfg5 k sweep {16, 32, 64})")
    ap.add_argument("--cpu-threads", type=int, default=None,
                    help="threads of the CPU legs (default: all host threads; 1 = the reference's serial build)")
    ap.add_argument("--sharded", action="store_true", help="row-sharded sessions even on one GPU (NCCL group of 1)")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of row sharding")
    ap.add_argument("--torch-comm", action="store_true", help="sharded: torch.distributed callbacks instead of the "
                                                               "library's NCCL communicator")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
