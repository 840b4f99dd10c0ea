#!/bin/bash
# A/B of DDH_F_CALL_GRAPHS (bench.py --call-graphs) at c3: normal host and a host whose
# enqueue thread shares its core with a busy loop (robustness of the timed region against
# a slow host: direct launches cost ~105 us of host time per frame, a graph replay ~2 us).
# Run under gpurun; prints frames/s per run.
mkdir -p gpurun_out
OUT=gpurun_out/graphs_ab.txt; : > $OUT
B="python bench.py --gpus 1 --no-e2e --no-latency --no-cpu-baseline --no-parity"
one() { # label, extra args...
  local l=$1; shift
  v=$("$@" 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))")
  echo "$l $v" | tee -a $OUT
}
for rep in 1 2 3; do
  one "K300 direct" $B --steps 300 --warmup 5
  one "K300 graphs" $B --steps 300 --warmup 5 --call-graphs
  one "K20  direct" $B --steps 20 --warmup 5
  one "K20  graphs" $B --steps 20 --warmup 5 --call-graphs
done
# slow host: everything pinned to core 2 beside a busy loop
taskset -c 2 python -c "while True: pass" & HOG=$!
for rep in 1 2; do
  one "K300 direct hogged" taskset -c 2 $B --steps 300 --warmup 5
  one "K300 graphs hogged" taskset -c 2 $B --steps 300 --warmup 5 --call-graphs
  one "K20  direct hogged" taskset -c 2 $B --steps 20 --warmup 5
  one "K20  graphs hogged" taskset -c 2 $B --steps 20 --warmup 5 --call-graphs
done
kill $HOG
