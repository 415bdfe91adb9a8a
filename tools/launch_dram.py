"""Per-kernel time and DRAM bytes of one bench step from an ncu launch list
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`,
`--csv --log-file`): the last warm step's launches grouped by kernel, with
the achieved DRAM GB/s of each and the share of the step.

    python tools/launch_dram.py launches.csv [first-kernel-regex-of-a-step]
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
first = re.compile(sys.argv[2] if len(sys.argv) > 2 else "k_stl_to_soa")
rows = [r for r in csv.reader(open(path)) if r and r[0].isdigit()]
launch = collections.OrderedDict()
for r in rows:
    lid, name, metric, unit, val = int(r[0]), r[4], r[12], r[13], r[14]
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1,
             "second": 1}.get(unit, 1)
    d = launch.setdefault(lid, {"name": name})
    d[metric] = v * scale
ids = list(launch)
starts = [i for i in ids if first.search(launch[i]["name"])]
step = [i for i in ids if i >= starts[-1]] if starts else ids
agg = collections.OrderedDict()
for i in step:
    d = launch[i]
    nm = re.sub(r"\(.*", "", d["name"]).replace("<unnamed>::", "").replace("ow::", "")
    a = agg.setdefault(nm, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"one step: {len(step)} launches, {tot * 1e3:.3f} ms serialised (cold caches: compare shares)")
print(f"{'kernel':44s} {'n':>4s} {'ms':>8s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>8s}")
for nm, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{nm[:44]:44s} {n:4d} {t * 1e3:8.3f} {100 * t / tot:5.1f}% {b / 1e6:9.2f} {b / t / 1e9 if t else 0:8.1f}")
