#!/bin/bash
# PDL trigger placement variants (tools/variant_stream.sh builds): c3 at 300
# steps (tools/variant_bench.sh) and at the driver's 20 steps (run under gpurun).
mkdir -p gpurun_out
bash tools/variant_bench.sh "$@"
bash tools/variant_bench.sh "$@"
for rep in 1 2; do
  for v in nt0 "$@"; do
    x=$(DDH_LIB=tools/variants/libddh_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-latency --no-cpu-baseline --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']))")
    echo "K=20 $v $x"
  done
done
