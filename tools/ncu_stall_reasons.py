"""Per-kernel stall reasons summed over SASS (ncu source page, sampling).
usage: ncu_stall_reasons.py REP KERNEL_REGEX"""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r)
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = collections.Counter()
seen = set()
for r in rows:
    if r and r[0].startswith("0x") and len(r) == len(hdr) and r[0] not in seen:
        seen.add(r[0])
        for i in cols:
            try: tot[hdr[i]] += float(r[i])
            except ValueError: pass
s = sum(tot.values())
for k, v in tot.most_common(14):
    print(f"  {k:32s} {v / s * 100:5.1f}%")
