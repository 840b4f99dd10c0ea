#!/bin/bash
# c3 value at the driver's --steps 20 (run under gpurun), a few repetitions
for rep in 1 2 3 4; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-latency --no-cpu-baseline --no-parity "$@" > gpurun_out/sr.log 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/sr.log').read().strip().splitlines()[-1]); print('K=20', round(d['value']), round(d['ms_per_step']*1000,1), d['clocks']['samples'])"
done
