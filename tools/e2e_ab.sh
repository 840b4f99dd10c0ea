#!/bin/bash
# e2e leg (host buffers) for the in-tree build and tools/variants/libddh_<v>.so (run under gpurun)
run() {
  timeout 600 python bench.py --steps 20 --warmup 5 --no-latency --no-cpu-baseline --no-parity > gpurun_out/e2e_$1.log 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e2e_$1.log').read().strip().splitlines()[-1]); e=d['e2e']; print('$1', round(e['value']), round(e['pcie']['ceiling']), round(e['pcie']['frac'],3))"
}
for rep in 1 2; do run base; for v in "$@"; do DDH_LIB=tools/variants/libddh_$v.so run $v; done; done
