# c3 throughput under diagnostic overrides with extra bench arguments (run under gpurun):
#   tools/knobs_args.sh "--no-l2-persist" "ENV=.." ...
mkdir -p gpurun_out
xa=$1; shift
for cfg in base "$@"; do
  if [ "$cfg" = base ]; then e=""; else e="$cfg"; fi
  env $e timeout 300 python bench.py --steps 300 --warmup 5 --frames 40 --no-e2e --no-latency --no-cpu-baseline --no-parity $xa > gpurun_out/k.log 2>gpurun_out/k.err
  python -c "import json;d=json.loads(open('gpurun_out/k.log').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['ms_per_step']*1000,1))" || tail -3 gpurun_out/k.err
done
