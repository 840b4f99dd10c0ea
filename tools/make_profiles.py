"""Summarise the ncu artefacts of a GPU round into profiles/ (tracked).

    python tools/make_profiles.py ROUND [gpurun_out/prof.ncu-rep] [gpurun_out/launches.csv] [gpurun_out/bench.log]

Writes profiles/<ROUND>_launches.txt (per-kernel share of the launch list),
profiles/<ROUND>_ncu_full.txt (key --set full metrics per kernel),
profiles/ncu_summary.json (DRAM bytes per launch per kernel, read by bench.py
for roofline.traffic) and copies the bench JSON line to profiles/<ROUND>_bench.json.
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1]
rep = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out/prof.ncu-rep")
lcsv = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out/launches.csv")
blog = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out/bench.log")
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)


def short(name):
    m = re.search(r"(k[a-z0-9_]+)(<[\d, ]+>)?\(", name)
    return (m.group(1) + (m.group(2) or "").replace(" ", "")) if m else name[:40]


# ---- launch list (cold-cache, serialised: shares, not absolutes)
if os.path.exists(lcsv):
    txt = open(lcsv).read()
    body = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(body)))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            k = short(r["Kernel Name"])
            if k.startswith("kz_"):  # on-device synthesiser: input generation before the timed steps
                continue
            tot[k] += float(r["Metric Value"])
            cnt[k] += 1
    allns = sum(tot.values())
    with open(os.path.join(out_dir, f"{rnd}_launches.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (launch list of\n"
                f"# bench.py --steps 20 --warmup 3 --frames 8 --serial ...); cold-cache, serialised launches:\n"
                f"# compare SHARES with bench.py's live CUDA-event breakdown, not absolute times.\n")
        f.write(f"{'kernel':24s} {'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}\n")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{k:24s} {cnt[k]:8d} {v/1e3:10.1f} {v/1e3/cnt[k]:8.2f} {v/allns*100:5.1f}%\n")
    print(open(os.path.join(out_dir, f"{rnd}_launches.txt")).read())

# ---- full capture
summary = {"source": os.path.basename(rep), "round": rnd, "dram_bytes_per_launch": {}, "kernels": {}}
if os.path.exists(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size",
            "launch__block_size", "launch__cluster_dim_x", "lts__t_bytes.sum"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}
    lines = []
    passes = {}
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        d = {}
        for w in want:
            if w in hdr:
                v, u = r[hdr.index(w)], units[hdr.index(w)]
                try:
                    fv = float(v.replace(",", ""))
                    d[w] = fv * scale[u] if u in scale and "byte" in u else fv
                    if "byte" not in u and u:
                        d[w + " [" + u + "]"] = d.pop(w)
                except ValueError:
                    d[w] = v
        summary["kernels"][name] = d
        rb, wb = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
        base = name.split("<")[0]
        if base != "ks_ricd_pass":
            summary["dram_bytes_per_launch"][base] = rb + wb
        # the r-ICD colour passes are four kernels per library launch (kind ks_ricd): per-pass
        # values are listed, and their sum over the four passes is kept under the kind's name
        if base == "ks_ricd_pass":
            m = re.search(r"<\d+,(\d)>", name)
            passes.setdefault(m.group(1) if m else name, d)
        lines.append(f"{name}\n" + "\n".join(f"  {k}: {v}" for k, v in d.items()))
    if passes:
        agg = {}
        for k in ("gpu__time_duration.sum [us]", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "smsp__inst_executed.sum [inst]"):
            agg[k] = sum(float(v.get(k, 0)) for v in passes.values())
        agg["passes"] = sorted(passes)
        summary["kernels"]["ks_ricd"] = agg  # the library's kind: the 4 colour passes
        summary["dram_bytes_per_launch"]["ks_ricd"] = agg["dram__bytes_read.sum"] + agg["dram__bytes_write.sum"]
        lines.append("ks_ricd (sum of the 4 colour passes = one library launch)\n" +
                     "\n".join(f"  {k}: {v}" for k, v in agg.items()))
    with open(os.path.join(out_dir, f"{rnd}_ncu_full.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none --import-source on -k regex:'ks_' -s 18 -c 13\n"
                "# (bench.py --steps 5 --warmup 3 --frames 8 --serial: the kernels of two time steps in the middle of a\n"
                "#  multi-frame call, 64 streams of c3, the launch configuration of bench.py's attribution pass; the\n"
                "#  last launch of each kernel is listed; ks_stats there is the y-only S0 of the next frame)\n"
                "# bytes in bytes; other units in brackets\n\n")
        f.write("\n\n".join(lines) + "\n")
    json.dump(summary, open(os.path.join(out_dir, "ncu_summary.json"), "w"), indent=1)
    print("\n\n".join(lines))

if os.path.exists(blog):
    lines = [l for l in open(blog).read().splitlines() if l.startswith("{")]
    if lines:
        d = json.loads(lines[-1])
        json.dump(d, open(os.path.join(out_dir, f"{rnd}_bench.json"), "w"), indent=1)
