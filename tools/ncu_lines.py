"""Attribute ncu SASS-level stall samples / instructions to CUDA source lines (needs -lineinfo).
python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr = None, None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
tot = [0.0, 0.0]
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    # CUDA line rows: Line No, Source, then SASS columns empty? rows carry both views side by side
    try:
        line = int(r[0])
    except ValueError:
        continue
    try:
        st = float(r[4] or 0)
        ie = float(r[7] or 0)
    except ValueError:
        continue
    k = (cur_file, line)
    agg[k][0] += st
    agg[k][1] += ie
    agg[k][2] = r[1].strip()[:90]
    tot[0] += st
    tot[1] += ie
print(f"total stall samples {tot[0]:.0f}, instructions {tot[1]:.4g}")
for (f, ln), (st, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{st / max(tot[0], 1) * 100:5.1f}% stall {ie / max(tot[1], 1) * 100:5.1f}% inst  {f}:{ln}  {src}")
