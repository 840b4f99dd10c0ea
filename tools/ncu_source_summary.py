"""Summarise `ncu --page source --csv` (CUDA-C view) by source line: stall samples
and instructions executed.  usage: ncu_source_summary.py REP KERNEL_REGEX [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# skip "Kernel Name" line(s)
start = next(i for i, l in enumerate(lines) if l.startswith('"Line"') or l.startswith('"#"') or '"Source"' in l)
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ci = {h: i for i, h in enumerate(hdr)}
samp = ci.get("Warp Stall Sampling (All Samples)")
inst = ci.get("Instructions Executed")
src = ci.get("Source")
lin = ci.get("Line", ci.get("#"))
tot_s = sum(float(r[samp] or 0) for r in rows[1:] if len(r) > samp)
tot_i = sum(float(r[inst] or 0) for r in rows[1:] if len(r) > inst)
print(f"total samples {tot_s:.0f}, warp-instructions {tot_i:.0f}")
rs = sorted(rows[1:], key=lambda r: -float(r[samp] or 0) if len(r) > samp else 0)
for r in rs[:top]:
    print(f"{float(r[samp] or 0)/tot_s*100:5.1f}% samp {float(r[inst] or 0)/tot_i*100:5.1f}% inst  L{r[lin]:>5}  {r[src].strip()[:110]}")
