"""Summarise an ncu report: top SASS instructions by stall samples, and per-CUDA-line totals.
usage: python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def page(extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"] + extra, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # first row is kernel name, second header
    hdr = rows[1]
    return hdr, rows[2:]


hdr, rows = page(["--print-source", "sass"])
ci = {h: i for i, h in enumerate(hdr)}
S = ci["Warp Stall Sampling (All Samples)"]
tot = sum(float(r[S] or 0) for r in rows if len(r) > S)
print(f"total samples {tot:.0f}")
top = sorted(rows, key=lambda r: -float(r[S] or 0))[:N]
for r in top:
    print(f"{float(r[S] or 0) / tot * 100:5.1f}%  {r[ci['Address']]:>6} {r[ci['Source']][:90]}")
try:
    hdr2, rows2 = page(["--print-source", "cuda"])
    c2 = {h: i for i, h in enumerate(hdr2)}
    S2 = c2["Warp Stall Sampling (All Samples)"]
    print("\n-- by CUDA line --")
    for r in sorted(rows2, key=lambda r: -float(r[S2] or 0))[:N]:
        if float(r[S2] or 0) <= 0:
            break
        print(f"{float(r[S2] or 0) / tot * 100:5.1f}%  L{r[c2.get('Line', 0)] if 'Line' in c2 else ''} {r[c2['Source']].strip()[:100]}")
except Exception as e:
    print("cuda view failed", e)
