"""Per-CUDA-source-line totals of an ncu report (warp instructions executed,
warp-stall samples), from the `cuda,sass` source view.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
src_text = {}
path = None
rows = []
lines = out.splitlines()
i = 0
tot_ins = tot_smp = 0.0
while i < len(lines):
    l = lines[i]
    if l.startswith('"File Path"'):
        path = l.split('","')[1].rstrip('"').split("/")[-1]
        i += 1
        continue
    if l.startswith('"Line No"'):
        j = i + 1
        while j < len(lines) and not lines[j].startswith('"File Path"'):
            j += 1
        block = "\n".join(lines[i:j])
        rdr = csv.reader(io.StringIO(block))
        hdr = next(rdr)
        ix_ins = hdr.index("Instructions Executed")
        ix_smp = hdr.index("Warp Stall Sampling (All Samples)")
        cur = None
        for r in rdr:
            if len(r) < len(hdr):
                continue
            if r[0]:
                cur = (path, int(r[0]))
                src_text[cur] = r[1].strip()
            if r[2] and cur:  # a SASS row under source line `cur`
                def num(x):
                    try:
                        return float(x)
                    except ValueError:
                        return 0.0

                ins = num(r[ix_ins])
                smp = num(r[ix_smp])
                a = agg.setdefault(cur, [0.0, 0.0])
                a[0] += ins
                a[1] += smp
                tot_ins += ins
                tot_smp += smp
        i = j
        continue
    i += 1
print(f"warp instructions {tot_ins:.4g}, stall samples {tot_smp:.4g}")
for k, (ins, smp) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * ins / max(tot_ins, 1):5.1f}% ins {100 * smp / max(tot_smp, 1):5.1f}% smp  {k[0]}:{k[1]:<5d} "
          f"{src_text.get(k, '')[:90]}")
