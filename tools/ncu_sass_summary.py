"""Summarise `ncu --page source --csv` (SASS view) of one kernel: top
instructions by stall samples, and opcode histogram of executed instructions.
usage: ncu_sass_summary.py REP KERNEL_REGEX [top]"""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ci = {h: i for i, h in enumerate(hdr)}
S, I, SRC = ci["Warp Stall Sampling (All Samples)"], ci["Instructions Executed"], ci["Source"]
rows = [r for r in rows[1:] if len(r) > max(S, I, SRC) and r[0] != "Address"]
tot_s = sum(float(r[S] or 0) for r in rows)
tot_i = sum(float(r[I] or 0) for r in rows)
print(f"{kern}: samples {tot_s:.0f}, warp-instructions {tot_i:.0f}")
ops = collections.Counter()
opsamp = collections.Counter()
for r in rows:
    op = r[SRC].strip().split()[0] if r[SRC].strip() else "?"
    if op.startswith("@"):
        op = r[SRC].strip().split()[1]
    op = op.split(".")[0]
    ops[op] += float(r[I] or 0)
    opsamp[op] += float(r[S] or 0)
print("opcode: %inst %stall")
for op, v in sorted(ops.items(), key=lambda kv: -opsamp[kv[0]])[:top]:
    print(f"  {op:10s} {v/tot_i*100:5.1f} {opsamp[op]/tot_s*100:5.1f}")
