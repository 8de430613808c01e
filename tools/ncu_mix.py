"""Instruction mix of an ncu report (executed warp instructions by SASS opcode):
python tools/ncu_mix.py rep.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
E = ci.get("Instructions Executed") or ci.get("Warp Instructions Executed")
mix = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= E or not r[E]:
        continue
    try:
        n = float(r[E])
    except ValueError:  # header row of the next kernel in a multi-kernel report
        continue
    src = r[ci["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    mix[op.split(".")[0]] += n
    tot += n
print(f"total warp instructions {tot:.0f}")
for op, n in mix.most_common(N):
    print(f"{n / tot * 100:5.1f}%  {op}")
