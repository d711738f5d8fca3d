"""Dynamic opcode histogram + top stall sites from a .ncu-rep source page."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
ops, samples = Counter(), Counter()
tot = 0
body = rows[2:]
for r in body:
    if len(r) < len(hdr) - 2: continue
    op = r[ci["Source"]].split()[0] if r[ci["Source"]].split() else "?"
    if op.startswith("@"): op = r[ci["Source"]].split()[1]
    op = op.split(".")[0]
    n = int(r[ci["Instructions Executed"]]); tot += n
    ops[op] += n
    samples[op] += int(r[ci["# Samples"]])
print("total warp-instr", tot)
for op, n in ops.most_common(18):
    print(f"  {op:8s} {n:12d} {100*n/tot:5.1f}%   samples {samples[op]}")
top = sorted(body, key=lambda r: -int(r[ci["# Samples"]]) if len(r) > ci["# Samples"] else 0)[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in top:
    st = sorted(((int(r[ci[s]]), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"  {r[ci['# Samples']]:>6s} {r[ci['Source']].strip()[:70]:70s} {st}")
