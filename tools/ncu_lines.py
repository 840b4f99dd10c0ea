"""Per-source-line totals (instructions executed, stall samples) of one kernel
from an ncu report (`--print-source cuda,sass`; needs -lineinfo).
usage: ncu_lines.py REP KERNEL_REGEX [top]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
cur_file = "?"
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] in ("Function Name",):
        continue
    if row[0] != "":  # a source line row (aggregated over its SASS)
        try:
            samp = float(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            inst = float(row[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        key = (cur_file, int(row[0]), row[1].strip()[:90])
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += samp
        a[1] += inst
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{kern}: stall samples {ts:.0f}, warp-instructions {ti:.0f}")
for (f, l, s), (a, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{b/ti*100:5.1f}% inst {a/ts*100:5.1f}% stall  {f}:{l:<4d} {s}")
