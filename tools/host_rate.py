"""Host enqueue time vs device time of multi-frame ddh_step calls (c3):
if the host needs as long to enqueue a call as the GPU needs to run it, the
step is launch-rate bound."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2305_03284_b200 import sched

cfg = dict(synth.CONFIGS["c3"])
T = int(os.environ.get("T", "40"))
u = sched.StreamRank(cfg, 0, cfg["streams"], 0, T)
for rep in range(5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(u.stream)
    t0 = time.perf_counter()
    u.ctx.step(u.y_dev[0:T])
    t1 = time.perf_counter()
    e1.record(u.stream)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"T={T} host enqueue {1e6*(t1-t0)/T:.1f} us/frame, wall {1e6*(t2-t0)/T:.1f}, device {1e3*e0.elapsed_time(e1)/T:.1f} us/frame")
