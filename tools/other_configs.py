"""Assemble profiles/<round>_other_configs.json from gpurun_out/cfg_<c>.json
(bench.py --config <c> --frames 4 --no-e2e --no-latency --no-cpu-baseline,
--steps 300 --warmup 5 for one stream (c2, c5), --steps 30 --warmup 3 for c4; one B200).  usage: python tools/other_configs.py OUT c2 c4 c5"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out, cfgs = sys.argv[1], sys.argv[2:]
res = []
for c in cfgs:
    d = json.loads(open(os.path.join(ROOT, "gpurun_out", f"cfg_{c}.json")).read().strip().splitlines()[-1])
    res.append(dict(config=c, workload=d["config"]["workload"], frames_per_s=d["value"],
                    us_per_step=d["ms_per_step"] * 1000, streams=d["config"]["streams_per_gpu"],
                    kernels_us_serialised={k: round(v["ms_total"] / d["steps"] * 1000, 1) for k, v in d["kernels"].items()},
                    parity=d.get("parity")))
json.dump(dict(note="bench.py --config <c> --frames 4 --no-e2e --no-latency --no-cpu-baseline; --steps 300 "
                    "--warmup 5 (c2, c5), --steps 30 --warmup 3 (c4); 1 B200; c3 is the headline bench line", results=res),
          open(os.path.join(ROOT, "profiles", out), "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
