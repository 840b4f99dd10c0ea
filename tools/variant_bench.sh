#!/bin/bash
# Quick c3 throughput of the in-tree build and of tools/variants/libddh_*.so
# (run under gpurun):  tools/variant_bench.sh [variant names...]
mkdir -p gpurun_out
run() {
  timeout 600 python bench.py --steps 300 --warmup 5 --frames 40 --no-e2e --no-latency --no-cpu-baseline --no-parity \
    > gpurun_out/vb_$1.log 2> gpurun_out/vb_$1.err
  python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/vb_{sys.argv[1]}.log").read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", open(f"gpurun_out/vb_{sys.argv[1]}.err").read()[-800:]); sys.exit()
k = {n: round(v["ms_total"] / d["steps"] * 1000, 1) for n, v in d["kernels"].items()}
print(f"{sys.argv[1]:10s} {d['value']:9.0f} fr/s  {d['ms_per_step']*1000:6.1f} us/step  attr {d['attribution_pass']['ms_per_step']*1000:6.1f}  {k}")
PY
}
run base
for v in "$@"; do DDH_LIB=tools/variants/libddh_$v.so run $v; done
