#!/bin/bash
# Adaptive call graphs (include/ddh.h DDH_F_NO_ADAPTIVE_GRAPHS) at c3: a normal host, a
# uniformly slower host (DDH_HOST_DELAY_US: a busy wait before every directly launched frame)
# and a host in bursts (the bench process sharing one core with a busy loop).
# DDH_ADAPTIVE_GRAPHS=0 = direct launches only.  Columns: frames/s, us per step, launches.
mkdir -p gpurun_out
OUT=gpurun_out/adapt_ab.txt; : > $OUT
B="python bench.py --gpus 1 --no-e2e --no-latency --no-cpu-baseline --no-parity"
one() { local l=$1; shift
  v=$("$@" 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), d['gpu_launches'])")
  echo "$l $v" | tee -a $OUT; }
for rep in 1; do
  one "K300 adaptive            " $B --steps 300 --warmup 5
  one "K300 direct              " env DDH_ADAPTIVE_GRAPHS=0 $B --steps 300 --warmup 5
  one "K20  adaptive            " $B --steps 20 --warmup 5
  for d in 30 60 120; do
    one "K300 adaptive delay $d us " env DDH_HOST_DELAY_US=$d $B --steps 300 --warmup 5
    one "K300 direct   delay $d us " env DDH_HOST_DELAY_US=$d DDH_ADAPTIVE_GRAPHS=0 $B --steps 300 --warmup 5
  done
  one "K20  adaptive delay 60 us" env DDH_HOST_DELAY_US=60 $B --steps 20 --warmup 5
done
taskset -c 2 python -c "while True: pass" & HOG=$!
for rep in 1; do
  one "K300 adaptive hogged     " taskset -c 2 $B --steps 300 --warmup 5
  one "K300 direct   hogged     " env DDH_ADAPTIVE_GRAPHS=0 taskset -c 2 $B --steps 300 --warmup 5
done
kill $HOG
