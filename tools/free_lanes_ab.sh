#!/bin/bash
# Lanes joined per frame (default) vs free-running across the frames of a call (DDH_FREE_LANES=1,
# a diagnostic build of r02h, removed again after this measurement: profiles/r02h_free_lanes_ab.txt)
mkdir -p gpurun_out
B="python bench.py --warmup 5 --no-e2e --no-latency --no-cpu-baseline"
for rep in 1 2; do
  for fl in 0 1; do
    for k in 300 20; do
      v=$(DDH_FREE_LANES=$fl timeout 300 $B --steps $k 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['parity']['phi_max_rad'], d['parity']['r_max_rel'])")
      echo "free_lanes=$fl K=$k rep=$rep $v"
    done
  done
done
