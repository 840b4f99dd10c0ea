"""Dump SASS of one kernel with executed-instruction counts and stall samples,
collapsed into runs, to locate where instructions/stalls go.
usage: ncu_sass_regions.py REP KERNEL_REGEX [min_frac]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
mf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.002
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r)
ci = {h: i for i, h in enumerate(hdr)}
S, I = ci["Warp Stall Sampling (All Samples)"], ci["Instructions Executed"]
body, seen = [], set()
for r in rows:
    if r and r[0].startswith("0x") and len(r) > I and r[0] not in seen:
        seen.add(r[0]); body.append(r)
f = lambda x: float(x) if x not in ("", "-") else 0.0
ts = sum(f(r[S]) for r in body); ti = sum(f(r[I]) for r in body)
print(f"samples {ts:.0f} warp-instr {ti:.0f}")
# print blocks: consecutive instructions with the same exec count
blk = []
def flush():
    if not blk: return
    n = f(blk[0][I]); s = sum(f(r[S]) for r in blk)
    if n * len(blk) / ti >= mf or s / ts >= mf:
        ops = [r[1].strip().split()[0] if not r[1].strip().startswith("@") else r[1].strip().split()[1] for r in blk]
        ops = [o.split(".")[0] for o in ops]
        from collections import Counter
        c = Counter(ops).most_common(6)
        print(f"{blk[0][0][-5:]} n={len(blk):4d} exec={n:9.0f} instr%={n*len(blk)/ti*100:5.1f} stall%={s/ts*100:5.1f}  {c}")
for r in body:
    if blk and f(r[I]) != f(blk[0][I]):
        flush(); blk = []
    blk.append(r)
flush()
