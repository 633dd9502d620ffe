"""Per-source-line warp-stall share of an ncu report (dev tool).

usage: python tools/ncu_lines.py report.ncu-rep [top]
Reads `ncu --page source --print-source cuda,sass --csv` and attributes each SASS
instruction's stall samples to the CUDA line it belongs to.
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
path, hdr = None, None
line_samples = defaultdict(float)
line_text = {}
cur = None
stall_col = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        stall_col = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None:
        continue
    if r[0]:  # a CUDA source line row
        cur = (path, r[0])
        line_text[cur] = r[1][:100]
    try:
        s = float(r[stall_col] or 0)
    except (ValueError, IndexError):
        s = 0.0
    if cur is not None and not r[0]:
        line_samples[cur] += s
tot = sum(line_samples.values()) or 1.0
byf = defaultdict(float)
for (f, _), v in line_samples.items():
    byf[f] += v
print(f"total samples {tot:.0f}")
for f, v in sorted(byf.items(), key=lambda x: -x[1])[:10]:
    print(f"{f:32s} {100 * v / tot:5.1f}%")
for (f, ln), v in sorted(line_samples.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.2f}% {f:26s}:{ln:5s} {line_text.get((f, ln), '')}")
