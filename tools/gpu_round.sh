#!/bin/bash
# One GPU round (run under gpurun): parity tests, bench, optional ncu captures.
#   tools/gpu_round.sh [tests] [bench] [ncu] [launches]
set -u
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests)
      timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
      echo "tests rc=$?"; grep -E "passed|failed" gpurun_out/gpu_tests.log | tail -2
      grep -E "^(FAILED|ERROR)" gpurun_out/gpu_tests.log | head -10 ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
      echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log ;;
    quick)
      timeout 600 python bench.py --steps 300 --warmup 5 --frames 40 --no-e2e --no-latency --no-cpu-baseline > gpurun_out/quick.log 2> gpurun_out/quick.err
      echo "quick rc=$?"; python - <<'PY'
import json
d = json.loads(open("gpurun_out/quick.log").read().strip().splitlines()[-1])
print("value", round(d["value"]), "attr", round(d["attribution_pass"]["value"]), "parity", d.get("parity"))
print({k: (round(v["ms_total"] / d["steps"] * 1000, 1), round(v.get("gbs", 0))) for k, v in d["kernels"].items()})
PY
      ;;
    ncu)
      CMD="python bench.py --steps 5 --warmup 3 --frames 8 --no-e2e --no-latency --no-cpu-baseline --no-parity --serial ${BENCH_EXTRA:-}"
      $CMD > gpurun_out/ncu_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ks_" -s 18 -c 13 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
      echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log ;;
    launches)
      CMD="python bench.py --steps 20 --warmup 3 --frames 8 --no-e2e --no-latency --no-cpu-baseline --no-parity --serial"
      $CMD > gpurun_out/launch_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
      echo "launches rc=$?" ;;
  esac
done
