"""DRAM bytes of one fill_bins call from an ncu launch list (the last step):
the launches from k_small_init (start of the count) to the last one before
k_face_prep / k_chunk_boxes; merged into profiles/traffic.json as
<cfg>.fill_bins (bytes per call).

    python tools/fill_bins_traffic.py launches.csv C2 [profiles/traffic.json]
"""
import collections
import csv
import json
import sys

path, cfg = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else None
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1}
launch = collections.OrderedDict()
for r in csv.reader(open(path)):
    if not r or not r[0].isdigit():
        continue
    d = launch.setdefault(int(r[0]), {"name": r[4]})
    d[r[12]] = float(r[14].replace(",", "")) * scale.get(r[13], 1)
ids = list(launch)
starts = [i for i in ids if "k_stl_to_soa" in launch[i]["name"]]
step = [i for i in ids if i >= starts[-1]]
s0 = next(i for i in step if "k_small_init" in launch[i]["name"])
s1 = next(i for i in step if i > s0 and ("k_face_prep" in launch[i]["name"] or "k_chunk_boxes" in launch[i]["name"]))
fam = [i for i in step if s0 <= i < s1 and not any(k in launch[i]["name"] for k in ("k_set_i64", "LeafLoad"))]
b = sum(launch[i].get("dram__bytes_read.sum", 0) + launch[i].get("dram__bytes_write.sum", 0) for i in fam)
print(f"{cfg} fill_bins: {len(fam)} launches, {b / 1e6:.3f} MB")
if out:
    t = json.load(open(out))
    t.setdefault(cfg, {})["fill_bins"] = int(b)
    json.dump(t, open(out, "w"), indent=1)
