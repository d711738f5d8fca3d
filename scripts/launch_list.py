"""Summarise an `ncu --metrics gpu__time_duration.sum[,...] --csv` launch list: time per kernel name and per-launch rows of one kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
pat = sys.argv[2] if len(sys.argv) > 2 else None
hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hdr]
ci = {k: i for i, k in enumerate(h)}
per = defaultdict(dict)
for r in rows[hdr + 1:]:
    if len(r) < len(h):
        continue
    per[r[ci["ID"]]]["name"] = r[ci["Kernel Name"]][:48]
    per[r[ci["ID"]]][r[ci["Metric Name"]]] = float(r[ci["Metric Value"]].replace(",", ""))
tot, cnt = defaultdict(float), defaultdict(int)
for v in per.values():
    tot[v["name"]] += v.get("gpu__time_duration.sum", 0)
    cnt[v["name"]] += 1
# once-per-field-handle set-up kernels (the Lipschitz-bound refinement, csrc/knf_bounds.cuh) are listed apart: shares are of the per-frame work
ONE_TIME = ("lip_bound_kernel", "lip_store_kernel")
setup = {n: t for n, t in tot.items() if n.startswith(ONE_TIME)}
all_t = sum(t for n, t in tot.items() if n not in setup) or 1.0
for n, t in sorted(tot.items(), key=lambda x: -x[1]):
    if n not in setup:
        print(f"{t / 1e6:8.3f} ms {100 * t / all_t:5.1f}%  x{cnt[n]:<4d} {n}")
for n, t in sorted(setup.items(), key=lambda x: -x[1]):
    print(f"{t / 1e6:8.3f} ms  (one-time field set-up, not part of a frame)  x{cnt[n]:<4d} {n}")
if pat:
    keys = [k for k in next(iter(per.values())) if k != "name"]
    print("launches of", pat, keys)
    for v in per.values():
        if pat in v["name"]:
            print("  " + " ".join(f"{v.get(k, 0):12.1f}" for k in keys))
