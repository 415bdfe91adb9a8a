"""Summarise the hottest SASS lines (warp-stall samples) of an ncu report.

    python tools/ncu_hot.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-count", "1"]
if kern:
    cmd += ["--kernel-name-base", "demangled", "--kernel-name", "regex:" + kern]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:end]))))
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[key] or 0) for r in rows)
ins = sum(float(r["Instructions Executed"] or 0) for r in rows)
print(f"{lines[0][:120]}\ntotal samples {tot:.0f}, warp instructions {ins:.3g}")
for r in sorted(rows, key=lambda r: -float(r[key] or 0))[:top]:
    print(f"{100 * float(r[key] or 0) / tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:90]:90s} ex={r['Instructions Executed']}")
