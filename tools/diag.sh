for extra in "" "--priors-off" "--unfused"; do
python bench.py --steps 300 --warmup 5 --frames 40 --no-e2e --no-latency --no-cpu-baseline --no-parity $extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$extra', round(d['value']), {k: round(v['ms_total']/d['steps']*1000,1) for k,v in d['kernels'].items()})"
done
