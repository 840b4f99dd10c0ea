mkdir -p gpurun_out
for rows in 1 0; do
 for c in c2 c5; do DDH_RICD_ROWS=$rows DDH_RICD_PASSES=2 timeout 600 python bench.py --config $c --frames 4 --steps 300 --warmup 5 --no-e2e --no-latency --no-cpu-baseline --no-parity > gpurun_out/x_${c}_$rows.json 2>/dev/null; done
 for c in c2 c5; do DDH_RICD_ROWS=$rows timeout 600 python bench.py --config $c --frames 4 --steps 300 --warmup 5 --no-e2e --no-latency --no-cpu-baseline --no-parity > gpurun_out/x_${c}_t$rows.json 2>/dev/null; done
 DDH_RICD_ROWS=$rows timeout 900 python bench.py --config c4 --frames 4 --steps 30 --warmup 3 --no-e2e --no-latency --no-cpu-baseline --no-parity > gpurun_out/x_c4_$rows.json 2>/dev/null
done
for f in gpurun_out/x_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ms_per_step']*1000,1), {k: round(v['ms_total']/d['steps']*1000,1) for k,v in d['kernels'].items() if 'ricd' in k})"; done
