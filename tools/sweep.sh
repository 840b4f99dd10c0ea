#!/bin/bash
# Quick uninstrumented throughput sweep over env settings (run under gpurun):
#   tools/sweep.sh "DDH_LANES=1" "DDH_LANES=4" ...
mkdir -p gpurun_out
for envs in "$@"; do
  env $envs python bench.py --steps 300 --warmup 5 --frames 40 --no-e2e --no-latency --no-cpu-baseline $EXTRA 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$envs', round(d['value']), 'attr', round(d['attribution_pass']['value']), d.get('parity',{}).get('phi_max_rad'), d.get('parity',{}).get('r_rel_l2'), {k: round(v['ms_total']/d['steps']*1000,1) for k,v in d['kernels'].items()})"
done
