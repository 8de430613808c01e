"""Attribute ncu SASS metrics (instructions executed, stall samples) to CUDA source lines.
usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, cur_line, cur_src = "?", 0, ""
inst = defaultdict(float)
samp = defaultdict(float)
src = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    # rows with a line number in col 0 are CUDA lines; SASS rows have empty line number
    if r[0].strip():
        try:
            cur_line = int(r[0])
            cur_src = r[1]
        except ValueError:
            pass
        continue
    key = (cur_file, cur_line)
    src[key] = cur_src
    try:
        inst[key] += float(r[hdr["Instructions Executed"]] or 0)
        samp[key] += float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (KeyError, ValueError, IndexError):
        pass
ti = sum(inst.values()) or 1
ts = sum(samp.values()) or 1
print(f"total inst {ti:.0f} samples {ts:.0f}")
print("-- by instructions --")
for k, v in sorted(inst.items(), key=lambda x: -x[1])[:N]:
    print(f"{v / ti * 100:5.1f}% inst {samp[k] / ts * 100:5.1f}% stall  {k[0]}:{k[1]}  {src[k].strip()[:90]}")
print("-- by stall samples --")
for k, v in sorted(samp.items(), key=lambda x: -x[1])[:N // 2]:
    print(f"{v / ts * 100:5.1f}% stall {inst[k] / ti * 100:5.1f}% inst  {k[0]}:{k[1]}  {src[k].strip()[:90]}")
