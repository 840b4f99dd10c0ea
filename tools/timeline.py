"""Kernel timeline of the concurrent c3 step (CUPTI activity records through
torch.profiler): start / end of every kernel of a few steps, per CUDA stream.
usage: python tools/timeline.py [steps] [out.json]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_03284_b200 import sched  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.json"
cname = sys.argv[3] if len(sys.argv) > 3 else "c3"
cfg = synth.CONFIGS[cname]
if cname == "c2":  # latency mode: one synchronous single-frame call per frame, graph replay
    u = sched.StreamRank(cfg, 0, 1, 0, 16, source="host", flags=32)
    ybuf = torch.empty_like(u.y_dev[0:1])

    def frames(k):
        for t in range(k):
            ybuf.copy_(u.y_dev[t % 16:t % 16 + 1])
            u.ctx.step(ybuf)
            torch.cuda.synchronize()
    u.steps = frames
else:
    u = sched.StreamRank(cfg, 0, cfg["streams"], 0, 16, flags=64)
u.steps(8)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    u.steps(K)
    torch.cuda.synchronize()
trace = "gpurun_out/trace.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(trace)
ev = [e for e in json.load(open(trace))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
rows = [{"name": e["name"].split("<")[0].replace("void ddh::", ""), "stream": e["args"].get("stream"),
         "start_us": round(e["ts"] - t0, 2), "dur_us": round(e["dur"], 2),
         "grid": e["args"].get("grid"), "block": e["args"].get("block")} for e in ev]
json.dump(rows, open(out, "w"), indent=0)
span = (ev[-1]["ts"] + ev[-1]["dur"] - t0)
print(f"{len(rows)} kernels, {span:.1f} us for {K} steps ({span / K:.1f} us/step)")
for r in rows[:40]:
    print(f"{r['start_us']:9.1f} {r['dur_us']:7.1f}  s{r['stream']}  {r['name']}")
