"""Aggregate an ncu --metrics gpu__time_duration.sum launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:70]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"{'total us':>10} {'share':>6} {'n':>5}  kernel   (cold-cache, serialised: compare shares)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:5d}  {k}")
print(f"{tot / 1e3:10.1f} us total over {sum(v[0] for v in agg.values())} launches")
