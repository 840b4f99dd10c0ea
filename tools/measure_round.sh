#!/bin/bash
# Final measurements of a round (run under gpurun):  tools/measure_round.sh ROUND
# bench (driver defaults), ncu --set full + launch list of the attribution
# pass, other configs, the N_k sweep, the c5 comparison, CUPTI timelines.
set -u
R=${1:-r02}
mkdir -p gpurun_out
bash tools/gpu_round.sh bench ncu launches
for c in c2 c5; do timeout 600 python bench.py --config $c --frames 4 --steps 300 --warmup 5 --no-e2e --no-latency --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config c4 --frames 4 --steps 30 --warmup 3 --no-e2e --no-latency --no-cpu-baseline > gpurun_out/cfg_c4.json 2> gpurun_out/cfg_c4.err; echo "c4 rc=$?"
timeout 600 python tools/nk_sweep.py $R > gpurun_out/nk.log 2>&1; echo "nk rc=$?"; tail -4 gpurun_out/nk.log
timeout 900 python tools/c5_compare.py $R > gpurun_out/c5.log 2>&1; echo "c5 rc=$?"; tail -5 gpurun_out/c5.log
timeout 300 python tools/timeline.py 6 gpurun_out/${R}_timeline_c3.json c3 > /dev/null 2>&1; echo "tl c3 rc=$?"
timeout 300 python tools/timeline.py 40 gpurun_out/${R}_timeline_c2.json c2 > /dev/null 2>&1; echo "tl c2 rc=$?"
