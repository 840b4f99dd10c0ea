# c2 / c4 / c5 throughput of the in-tree build and of tools/variants/libddh_*.so (run under gpurun):
#   tools/variant_configs.sh [variant names...]
mkdir -p gpurun_out
one() {  # name config steps warmup
  timeout 900 python bench.py --config $2 --frames 4 --steps $3 --warmup $4 --no-e2e --no-latency --no-cpu-baseline --no-parity \
    > gpurun_out/vc.log 2> gpurun_out/vc.err
  python -c "import json;d=json.loads(open('gpurun_out/vc.log').read().strip().splitlines()[-1]);print('$1 $2', round(d['value']), round(d['ms_per_step']*1000,1))" || tail -3 gpurun_out/vc.err
}
for v in base "$@"; do
  if [ "$v" != base ]; then export DDH_LIB=tools/variants/libddh_$v.so; fi
  one $v c2 300 5; one $v c5 300 5; one $v c4 30 3
  unset DDH_LIB
done
