#!/bin/bash
# Per-kernel DRAM bytes and time with WARM caches (--cache-control none), to see
# what actually reaches HBM in the pipeline.  LANES (default 1; "auto" = the
# library's choice) and COUNT (launches captured).  Run under gpurun.
mkdir -p gpurun_out
CMD="python bench.py --steps 6 --warmup 3 --frames 8 --no-e2e --no-latency --no-cpu-baseline --no-parity ${BENCH_EXTRA:-}"
LV=${LANES:-1}; [ "$LV" = auto ] && unset LV
env ${LV:+DDH_LANES=$LV} $CMD > gpurun_out/warm_plain.log 2>&1 && env ${LV:+DDH_LANES=$LV} timeout 900 ncu --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active \
  -s 40 -c ${COUNT:-24} --csv --log-file gpurun_out/warm.csv $CMD > gpurun_out/warm_ncu.log 2>&1
echo "rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/warm.csv")))
hdr = next(r for r in rows if "Metric Name" in r)
ci = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[rows.index(hdr) + 1:]:
    if len(r) < len(hdr): continue
    k = r[ci["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").replace("ddh::", "")
    try: agg[k][r[ci["Metric Name"]]].append(float(r[ci["Metric Value"]].replace(",", "")))
    except ValueError: pass
tot = 0.0
for k, m in agg.items():
    print(k, len(m["gpu__time_duration.sum"]), {n.split("__")[1][:28] if "__" in n else n: round(sum(v) / len(v), 2) for n, v in m.items()})
    tot += sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])
print("total DRAM bytes over the captured launches:", tot)
PY
