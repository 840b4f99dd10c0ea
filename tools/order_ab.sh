#!/bin/bash
# A/B of the lane enqueue order (stage by stage vs lane by lane) at the
# driver's 20 steps and at 300 steps (run under gpurun).  Measured in r02h with a
# build that read DDH_LANE_ORDER (profiles/r02h_lane_order_ab.txt: no difference,
# so the knob and the stage-by-stage order were removed again).
mkdir -p gpurun_out
B="python bench.py --warmup 5 --no-e2e --no-latency --no-cpu-baseline --no-parity"
for rep in 1 2 3; do
  for o in stage lane; do
    for k in 20 300; do
      v=$(DDH_LANE_ORDER=$o timeout 300 $B --steps $k 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value']))")
      echo "order=$o K=$k rep=$rep value=$v" | tee -a gpurun_out/order_ab.txt
    done
  done
done
