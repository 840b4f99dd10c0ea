#!/bin/bash
# Instruction count and duration of the ICD kernels for the in-tree build and
# tools/variants/libddh_<name>.so (run under gpurun): tools/ncu_inst.sh [names...]
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --frames 8 --no-e2e --no-latency --no-cpu-baseline --no-parity --serial"
one() {
  timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"${KREGEX:-ks_ricd|ks_phiicd}" -s 8 -c ${NCU_COUNT:-10} --csv $CMD > gpurun_out/inst_$1.csv 2> gpurun_out/inst_$1.err
  python - "$1" <<'PY'
import csv, sys, collections
lines = open(f"gpurun_out/inst_{sys.argv[1]}.csv").read().splitlines()
rows = list(csv.reader(lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]))
h = rows[0]; ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(dict)
for r in rows[1:]:
    agg[(r[0], r[ki].split("(")[0])][r[mi]] = float(r[vi].replace(",", ""))
seen = {}
for (i, k), m in agg.items():
    seen[k] = m
for k, m in seen.items():
    print(f"{sys.argv[1]:8s} {k:40s} inst {m['smsp__inst_executed.sum']/1e6:7.2f} M  {m['gpu__time_duration.sum']/1e3:6.1f} us  issue {m['smsp__issue_active.avg.pct_of_peak_sustained_active']:.0f}%")
PY
}
one base
for v in "$@"; do DDH_LIB=tools/variants/libddh_$v.so one $v; done
