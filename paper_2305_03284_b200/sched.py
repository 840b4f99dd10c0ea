"""Stream scheduler: shards independent sensor streams over the GPUs of one
box (north_star "(4) a stream scheduler that shards independent
sensor streams across the 8 GPUs of one box while each stream's timesteps stay
sequential on one device, so no per-step collective is needed").

Streams are independent (Fig. 1's recurrence is per stream), so a
GPU owns a contiguous block of streams, one ddh_ctx, one CUDA stream and its
own staged frames; the only cross-GPU traffic is host-side bookkeeping outside
the hot loop (barriers around timed regions, the max over GPUs of a device
time, gathers of per-stream scalars).  There is no data-path collective.

Two ways to run the same per-GPU unit (:class:`StreamRank`):
  * one process per GPU under torchrun: :func:`run_streams` runs this rank's
    shard; barriers and the max over ranks go through torch.distributed
    (NCCL when every rank has its own GPU, else gloo: the collectives carry
    host-side scalars only);
  * one process, one host thread per GPU (``run_streams(cfg, gpus=G)`` without
    torchrun): the library calls release the GIL, barriers are
    threading.Barrier, the job time is the max of the per-GPU device times.
"""
from __future__ import annotations

import math
import os
import threading
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


def shard(total_streams: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of streams for `rank`: stream s goes to rank
    floor(s * world / total).  Returns (first, count)."""
    if world < 1 or not (0 <= rank < world) or total_streams < 0:
        raise ValueError("bad shard arguments")
    first = -(-rank * total_streams // world)
    last = -(-(rank + 1) * total_streams // world)
    return first, last - first


def env_rank() -> Tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def pick_backend(preferred: str = "nccl") -> str:
    """NCCL when every local rank can own a distinct GPU, else gloo (the
    scheduler's collectives are host-side scalars; NCCL refuses two ranks on
    one device)."""
    if preferred != "nccl":
        return preferred
    try:
        import torch
        n = torch.cuda.device_count()
    except Exception:
        n = 0
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    return "nccl" if n >= local_world and n > 0 else "gloo"


def init(backend: str = "nccl"):
    """Initialise torch.distributed when WORLD_SIZE > 1 (rendezvous from env)."""
    import torch.distributed as dist
    world, rank, local = env_rank()
    if world > 1 and not dist.is_initialized():
        dist.init_process_group(backend=pick_backend(backend))
    return world, rank, local


def device_of(local_rank: int) -> int:
    """CUDA device of a local rank (ranks beyond the device count share devices)."""
    import torch
    n = max(1, torch.cuda.device_count())
    return local_rank % n


def _dist_on() -> bool:
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def barrier():
    import torch.distributed as dist
    if _dist_on():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    """Maximum of a scalar over ranks (timings: the job is as slow as its
    slowest GPU)."""
    import torch
    import torch.distributed as dist
    if not _dist_on():
        return float(x)
    dev = device if (device is not None and dist.get_backend() == "nccl") else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    if not _dist_on():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_per_stream(values: List[float], first: int, total: int) -> List[float]:
    """Gather per-stream scalars of every rank's block into one list indexed
    by global stream id (all ranks receive it)."""
    import torch.distributed as dist
    if not _dist_on():
        return list(values)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (first, list(values)))
    out = [float("nan")] * total
    for f, vals in parts:
        for k, v in enumerate(vals):
            out[f + k] = v
    return out


# ------------------------------------------------------------------ staging


def stream_draws(cfg: dict, first: int, count: int, seed: int = 20230504):
    """Per-stream D/r0 and frozen-flow velocity (rows, cols px/frame) of global
    streams [first, first+count), drawn like synth/ (uniform D/r0 range,
    uniform direction for "random")."""
    d_r0, vel = [], []
    for k in range(first, first + count):
        g = np.random.default_rng([seed, k])
        lo_hi = cfg.get("d_r0_range")
        d_r0.append(lo_hi[0] + (lo_hi[1] - lo_hi[0]) * g.random() if lo_hi else cfg["d_r0"])
        if cfg["direction"] == "random":
            th = 2 * math.pi * g.random()
        elif cfg["direction"] == "angle":
            th = cfg["angle"]
        else:
            th = math.pi / 2  # along +columns
        vel.append((cfg["flow"] * math.sin(th), cfg["flow"] * math.cos(th)))
    return d_r0, vel


def stage_frames(cfg: dict, first: int, count: int, frames: int, device: int, source: str = "device",
                 want_host: bool = False):
    """Frames [0, frames) of global streams [first, first+count) staged in HBM
    of `device`: y [T][count][N][N] complex64 (and the host copy if asked).
    source "device": the on-device synthesiser (libddh ddh_synth_*); "host":
    synth/ on the host cores, copied once."""
    import torch

    import synth
    if source == "device" and cfg.get("scene", "uniform") != "bars":
        from .ddh import DDHSynth
        d_r0, vel = stream_draws(cfg, first, count)
        z = DDHSynth(cfg["n"], count, d_r0=d_r0, velocity=vel, sigma_b=cfg["sigma_b"], snr_db=cfg["snr_db"],
                     diam=cfg["diam"], seed=20230504 + first, device=device)
        y, _ = z.frames(0, frames, want_phi=False)
        torch.cuda.synchronize(device)
        return y, (y.cpu().numpy() if want_host else None)
    y_host, _ = synth.make_batch(cfg, streams=count, frames=frames, first_stream=first, want_phi=False)
    return torch.from_numpy(y_host).to(torch.device("cuda", device)), (y_host if want_host else None)


def run_steps(ctx, y_dev, start: int, K: int, F: int):
    """K time steps over F staged frame batches, cycling from batch `start`:
    one ddh_step call per run of contiguous batches (inside a call the library
    overlaps the S0 sums of frame t+1 with frame t)."""
    done = 0
    while done < K:
        t = (start + done) % F
        T = min(F - t, K - done)
        ctx.step(y_dev[t:t + T])
        done += T


class StreamRank:
    """The per-GPU unit of the scheduler: a contiguous block of streams, their
    staged frames, one ddh_ctx on one CUDA stream of `device`."""

    def __init__(self, cfg: dict, first: int, count: int, device: int, frames: int, source: str = "device",
                 want_host: bool = False, **params):
        import torch

        import synth
        from .ddh import DDH
        self.cfg, self.first, self.count, self.device = cfg, first, count, device
        self.n = cfg["n"]
        torch.cuda.set_device(device)
        self.y_dev, self.y_host = stage_frames(cfg, first, count, frames, device, source, want_host)
        self.F = frames
        self.noise_var = synth.recon_noise_var(self.n, cfg["diam"], cfg["snr_db"])
        params.setdefault("noise_var", self.noise_var)
        params.setdefault("n_k", cfg.get("n_k", 1))
        self.stream = torch.cuda.Stream(device) if params.pop("own_stream", False) else torch.cuda.current_stream(device)
        self.call_graphs = bool(params.get("flags", 0) & 128) if "DDH_CALL_GRAPHS" not in os.environ \
            else os.environ["DDH_CALL_GRAPHS"] != "0"  # DDH_F_CALL_GRAPHS (include/ddh.h)
        self.ctx = DDH(self.n, count, device=device, aperture_diam=cfg["diam"], stream=self.stream, **params)
        self.pos = 0

    def steps(self, K: int):
        """Enqueue K time steps (asynchronous on the ctx stream)."""
        run_steps(self.ctx, self.y_dev, self.pos, K, self.F)
        self.pos = (self.pos + K) % self.F

    def prime_graphs(self, chunk: Optional[int] = None):
        """Untimed: capture the call graphs that later multi-frame calls replay
        (ddh_step's chunks of DDH_CHUNK frames with DDH_F_CALL_GRAPHS) for
        both state parities: a chunk, one frame, a chunk."""
        if not self.call_graphs:
            return
        c = chunk or int(os.environ.get("DDH_CHUNK", "8"))
        self.steps(c)
        self.steps(1)
        self.steps(c)

    def timed(self, K: int) -> float:
        """Device time (ms, CUDA events on the ctx stream) of K time steps."""
        import torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(self.device)
        e0.record(self.stream)
        self.steps(K)
        e1.record(self.stream)
        e1.synchronize()
        return e0.elapsed_time(e1)


def run_streams(cfg: dict, gpus: Optional[int] = None, steps: int = 20, warmup: int = 3, frames: Optional[int] = None,
                scaling: str = "weak", source: str = "device", devices: Optional[Sequence[int]] = None,
                return_state: bool = False, **params) -> Dict:
    """Run config `cfg` sharded over GPUs (SURVEY 1 L3 `run_streams(cfg, gpus)`).

    scaling "weak": cfg["streams"] streams per GPU (c3); "strong": cfg["streams"]
    in total, split in contiguous blocks (c4).  Under torchrun (WORLD_SIZE > 1)
    this process runs its rank's block; otherwise one host thread per entry of
    `devices` (default: the first `gpus` CUDA devices).  Every GPU stages its
    frames, warms up, waits at a barrier, runs `steps` time steps timed on its
    own stream, waits at a second barrier.  Returns frames/s of the whole job
    (all streams' frames / the slowest GPU's device time) and the per-GPU rows."""
    import torch
    frames = frames or min(cfg.get("frames", 100), 100)
    world, rank, local = env_rank()
    if world > 1:
        init("nccl")
        G = world
    else:
        devices = list(devices) if devices is not None else list(range(gpus or max(1, torch.cuda.device_count())))
        G = len(devices)
    total = cfg["streams"] * G if scaling == "weak" else cfg["streams"]

    def unit(g: int, dev: int, bar) -> Dict:
        first, count = shard(total, G, g)
        r = StreamRank(cfg, first, count, dev, frames, source, **params)
        r.steps(warmup)
        r.prime_graphs()
        torch.cuda.synchronize(dev)
        bar()
        ms = r.timed(steps)
        bar()
        row = {"rank": g, "device": dev, "first": first, "streams": count, "ms": ms,
               "frames_per_s": count * steps / (ms * 1e-3)}
        if return_state:
            rr, pp, fi = r.ctx.get_state()
            row["state"] = (rr.cpu().numpy(), pp.cpu().numpy(), fi)
        return row

    if world > 1:
        row = unit(rank, device_of(local), barrier)
        ms_max = max_over_ranks(row["ms"])
        rows = [row]
    else:
        tb = threading.Barrier(G)
        rows: List[Optional[Dict]] = [None] * G
        errs: List[BaseException] = []

        def body(g):
            try:
                rows[g] = unit(g, devices[g], tb.wait)
            except BaseException as e:  # noqa: BLE001 - reported to the caller
                errs.append(e)
                tb.abort()

        th = [threading.Thread(target=body, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        ms_max = max(r["ms"] for r in rows)
    return {"gpus": G, "streams_total": total, "steps": steps, "scaling": scaling, "ms_max": ms_max,
            "frames_per_s": total * steps / (ms_max * 1e-3), "ms_per_step": ms_max / steps, "per_gpu": rows,
            "mode": "torchrun ranks" if world > 1 else "host threads"}
