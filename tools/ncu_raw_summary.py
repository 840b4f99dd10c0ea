"""Key raw metrics per kernel from an ncu report. usage: ncu_raw_summary.py REP"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__cluster_dim_x",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]
units = rows[1]
for r in rows[2:]:
    d = {w: (r[hdr.index(w)] + " " + units[hdr.index(w)]).strip() for w in want if w in hdr}
    print("\n".join(f"  {k}: {v}" for k, v in d.items()))
    print()
