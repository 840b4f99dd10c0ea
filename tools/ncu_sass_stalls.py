"""Stall samples of one kernel by SASS opcode and the hottest instructions.
usage: ncu_sass_stalls.py REP KERNEL_REGEX [top]"""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r)
ci = {h: i for i, h in enumerate(hdr)}
S, I = ci["Warp Stall Sampling (All Samples)"], ci["Instructions Executed"]
body = [r for r in rows if r and r[0].startswith("0x") and len(r) > I]

f = lambda x: float(x) if x not in ("", "-") else 0.0
ts = sum(f(r[S]) for r in body); ti = sum(f(r[I]) for r in body)
by = collections.defaultdict(lambda: [0.0, 0.0])
for r in body:
    op = r[1].strip().split()
    op = [o for o in op if not o.startswith("@")][0].split(".")[0] if op else "?"
    by[op][0] += f(r[S]); by[op][1] += f(r[I])
print(f"samples {ts:.0f}  warp-instr {ti:.0f}")
for op, (s, i) in sorted(by.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {op:10s} {s/ts*100:5.1f}% stall-samples {i/ti*100:5.1f}% instr")
print("hottest:")
for k, r in enumerate(sorted(body, key=lambda r: -f(r[S]))[:top]):
    print(f"  {f(r[S])/ts*100:5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
