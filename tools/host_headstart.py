"""Device time of a multi-frame ddh_step call when every launch is queued
before the GPU reaches it (a spin kernel holds the stream while the host
enqueues): compares with the normal back-to-back device time to tell whether
host enqueue rate limits the step."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2305_03284_b200 import sched

cfg = dict(synth.CONFIGS["c3"])
T = int(os.environ.get("T", "12"))
u = sched.StreamRank(cfg, 0, cfg["streams"], 0, 2 * T)
for rep in range(6):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(u.stream):
        if rep % 2:
            torch.cuda._sleep(int(4e7))
        e0.record(u.stream)
        t0 = time.perf_counter()
        u.ctx.step(u.y_dev[0:T])
        t1 = time.perf_counter()
        e1.record(u.stream)
    torch.cuda.synchronize()
    print(f"{'headstart' if rep % 2 else 'normal   '} T={T} host {1e6*(t1-t0)/T:.1f} us/frame, device {1e3*e0.elapsed_time(e1)/T:.1f} us/frame")
