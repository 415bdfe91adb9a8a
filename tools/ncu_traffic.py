"""DRAM traffic per launch of the bench's roofline kernel families from an
``ncu --set full`` raw CSV (``--page raw --csv``), with ncu's per-column units
(bytes, Kbyte, Mbyte, Gbyte) normalised to bytes.

    python tools/ncu_traffic.py gpurun_out/<tag>_full_raw.csv C2 [profiles/traffic.json]

A family's launch is one bracket of bench.py's ``roofline`` entry: one
lattice sweep (k_lat_faces + its k_lat_mt) or one marking pass
(k_mark_blocks + its k_mark_items); bytes = dram__bytes_read.sum +
dram__bytes_write.sum summed over the family's kernels / the number of
brackets.
"""

import csv
import json
import sys

SCALE = {"byte": 1, "bytes": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "kib": 1024, "mib": 2 ** 20}
FAMILIES = {"lattice": (("k_lat_faces", "k_lat_mt"), "k_lat_faces"),
            "mark": (("k_mark_blocks", "k_mark_items"), "k_mark_blocks")}


def kernel_base(name):
    s = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    s = s.split("(")[0].split("<")[0]
    return s.split()[-1]


def main():
    path, cfg = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}

    def val(r, col):
        return float(r[ix[col]]) * SCALE[units[ix[col]].strip().lower()]

    res = {}
    for fam, (kernels, bracket) in FAMILIES.items():
        tot, brackets = 0.0, 0
        for r in rows[2:]:
            k = kernel_base(r[ix["Kernel Name"]])
            if k in kernels:
                tot += val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
                brackets += k == bracket
        if brackets:
            res[fam] = int(round(tot / brackets))
        print(f"{fam}: {tot / max(brackets, 1) / 1e6:.3f} MB per launch over {brackets} launches")
    if out:
        try:
            doc = json.load(open(out))
        except (OSError, ValueError):
            doc = {}
        doc["_source"] = ("ncu --set full --clock-control none (default --cache-control all: caches flushed before "
                          "each replay), dram__bytes_read.sum + dram__bytes_write.sum per launch (units normalised "
                          "to bytes by tools/ncu_traffic.py), " + path.split("/")[-1])
        doc[cfg] = res
        json.dump(doc, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
