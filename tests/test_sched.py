"""Multi-GPU host logic on CPU (-m "not gpu"): stream sharding, max-over-ranks
timing and per-stream gathers with world_size 2 over gloo.  The per-stream
inputs a rank synthesises for its shard must equal the single-process ones
(streams are independent; seeds are per global stream id)."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2305_03284_b200 import sched


def test_shard_partitions_streams():
    for total in (1, 7, 64, 512):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for rank in range(world):
                f, c = sched.shard(total, world, rank)
                seen.extend(range(f, f + c))
                assert c in (total // world, -(-total // world))
            assert seen == list(range(total))
    assert sched.shard(512, 8, 3) == (192, 64)
    with pytest.raises(ValueError):
        sched.shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    import synth
    w, r, _ = sched.init("gloo")
    first, count = sched.shard(total, w, r)
    cfg = dict(synth.CONFIGS["c1"])
    y, _ = synth.make_batch(cfg, streams=count, frames=2, first_stream=first, workers=1, want_phi=False)
    sums = [float(np.abs(y[:, k]).sum()) for k in range(count)]
    allsums = sched.gather_per_stream(sums, first, total)
    tmax = sched.max_over_ranks(1.5 + r)
    sched.barrier()
    out_q.put((r, first, count, allsums, tmax))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_process():
    world, total = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import synth
    y, _ = synth.make_batch(dict(synth.CONFIGS["c1"]), streams=total, frames=2, workers=1, want_phi=False)
    ref = [float(np.abs(y[:, k]).sum()) for k in range(total)]
    for r, first, count, allsums, tmax in res:
        assert allsums == ref  # both ranks see every stream, identical to one process
        assert tmax == 2.5     # max over ranks
    assert sorted((f, c) for _, f, c, _, _ in res) == [(0, 3), (3, 2)]  # stream s -> rank floor(s G / S)


def test_backend_choice_without_enough_gpus(monkeypatch):
    """NCCL refuses two ranks on one device: with fewer GPUs than local ranks
    the scheduler's host-side collectives use gloo."""
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "2")
    import torch
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 1)
    assert sched.pick_backend("nccl") == "gloo"
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 8)
    assert sched.pick_backend("nccl") == "nccl"
    assert sched.pick_backend("gloo") == "gloo"


def test_stream_draws_follow_global_stream_ids():
    """Per-stream turbulence strength and flow direction depend on the global
    stream id only, so a shard draws exactly the single-process values."""
    import synth
    cfg = dict(synth.CONFIGS["c3"])
    d_all, v_all = sched.stream_draws(cfg, 0, 8)
    for first, count in (sched.shard(8, 3, r) for r in range(3)):
        d, v = sched.stream_draws(cfg, first, count)
        assert d == d_all[first:first + count] and v == v_all[first:first + count]
    lo, hi = cfg["d_r0_range"]
    assert all(lo <= x <= hi for x in d_all)
    assert all(abs(math.hypot(*vv) - cfg["flow"]) < 1e-12 for vv in v_all)
