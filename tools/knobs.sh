mkdir -p gpurun_out
for cfg in "base" "DDH_SPLIT_R=0" "DDH_LANES=1" "DDH_LANES=3" "DDH_LANES=4" "DDH_LANES=4 DDH_SPLIT_R=0"; do
  if [ "$cfg" = base ]; then e=""; else e="$cfg"; fi
  env $e timeout 300 python bench.py --steps 300 --warmup 5 --frames 40 --no-e2e --no-latency --no-cpu-baseline --no-parity > gpurun_out/k.log 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/k.log').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['ms_per_step']*1000,1))"
done
