#!/bin/bash
# c3 value at the driver's --steps 20 vs 300, with and without call graphs (run under gpurun)
for rep in 1 2; do
for K in 20 300; do
  for G in "" "--call-graphs"; do
    timeout 600 python bench.py --steps $K --warmup 5 --no-e2e --no-latency --no-cpu-baseline --no-parity $G > gpurun_out/sr.log 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/sr.log').read().strip().splitlines()[-1]); print('K=$K $G', round(d['value']), round(d['ms_per_step']*1000,1))"
  done
done
done
