"""Where the short-run fill / drain goes: CUPTI kernel timeline of one K-frame
c3 call from an idle GPU (as bench.py's timed region starts), per frame the
start of each lane's S1 and the end of its last kernel.
usage: python tools/fill_timeline.py K flags out.json   (flags 64 = L2 window, +128 = call graphs)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_03284_b200 import sched  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 64
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/fill_timeline.json"
cfg = synth.CONFIGS["c3"]
u = sched.StreamRank(cfg, 0, cfg["streams"], 0, 40, flags=flags)
u.steps(K)
u.steps(K)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    u.steps(K)
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
trace = "gpurun_out/fill_trace.json"
prof.export_chrome_trace(trace)
ev = [e for e in json.load(open(trace))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
rows = [{"name": e["name"].split("(")[0].split("<")[0].replace("void ", "").replace("ddh::", ""),
         "stream": e["args"].get("stream"), "start_us": round(e["ts"] - t0, 2), "dur_us": round(e["dur"], 2)}
        for e in ev]
span = max(r["start_us"] + r["dur_us"] for r in rows)
s1 = [r for r in rows if r["name"].startswith("ks_rows_fwd")]
lanes = sorted(set(r["stream"] for r in s1), key=lambda s: min(r["start_us"] for r in s1 if r["stream"] == s))
per_lane = {s: [r["start_us"] for r in s1 if r["stream"] == s] for s in lanes}
res = {"K": K, "flags": flags, "span_us": span, "kernels": len(rows), "lanes": len(lanes),
       "s1_starts": per_lane, "first_kernels": rows[:30], "last_kernels": rows[-30:]}
frames = min(len(v) for v in per_lane.values())
starts = [min(per_lane[s][f] for s in lanes) for f in range(frames)]
res["frame_starts"] = starts
res["frame_periods"] = [round(b - a, 1) for a, b in zip(starts, starts[1:])]
res["tail_us"] = round(span - starts[-1], 1)
json.dump(res, open(out, "w"), indent=1)
print(f"K={K} flags={flags}: span {span:.1f} us = {span / K:.1f} us/step; lanes {len(lanes)}")
print("frame periods", res["frame_periods"])
print("first frame start offsets per lane", [round(per_lane[s][0], 1) for s in lanes], "tail", res["tail_us"])
