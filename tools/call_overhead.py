"""Per-call overhead of multi-frame ddh_step calls at c3: device time of one
call of K frames from an idle GPU, and the same with the host's enqueue
hidden behind a GPU sleep issued first (the difference is host-side latency
before the first kernel).  usage: python tools/call_overhead.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_03284_b200 import sched  # noqa: E402

cfg = synth.CONFIGS["c3"]
u = sched.StreamRank(cfg, 0, cfg["streams"], 0, 100, flags=64)
u.steps(10)
torch.cuda.synchronize()
st = u.stream
for hide in (False, True):
    for K in (1, 2, 4, 8, 20, 40, 100):
        ts = []
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                if hide:
                    torch.cuda._sleep(2_000_000)  # ~1 ms of GPU spin: the host enqueues meanwhile
                e0.record(st)
            u.ctx.step(u.y_dev[0:K])
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        ts.sort()
        print(f"hide={hide!s:5s} K={K:3d}: {ts[len(ts) // 2]:8.1f} us  {ts[len(ts) // 2] / K:6.1f} us/frame")
