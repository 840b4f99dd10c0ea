#!/bin/bash
# c3 with 4 lanes (16 streams each) and the large-launch ICD forms forced
# (DDH_SMALL_TILES=0: 64-tile phi-ICD, r-ICD colour passes) vs the default 3 lanes.
mkdir -p gpurun_out
B="python bench.py --warmup 5 --steps 300 --frames 40 --no-e2e --no-latency --no-cpu-baseline --no-parity"
for rep in 1 2; do
  for cfg in "DDH_LANES=3" "DDH_LANES=4 DDH_SMALL_TILES=0" "DDH_LANES=4 DDH_SMALL_TILES=0 DDH_RICD_PASSES=2" "DDH_LANES=2" "DDH_LANES=5 DDH_SMALL_TILES=0" "DDH_LANES=6 DDH_SMALL_TILES=0"; do
    v=$(env $cfg timeout 300 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))")
    echo "$cfg rep=$rep value,us=$v" | tee -a gpurun_out/lanes4_ab.txt
  done
done
