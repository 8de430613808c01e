"""Per-kernel instruction mix of a multi-kernel ncu report: python tools/ncu_mix_kernels.py rep.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = []
for r in csv.reader(io.StringIO(out)):
    if "Instructions Executed" in r or "Warp Instructions Executed" in r:
        ci = {h: i for i, h in enumerate(r)}
        blocks.append((ci, collections.Counter()))
        continue
    if not blocks or not r:
        continue
    ci, cur = blocks[-1]
    E = ci.get("Instructions Executed") or ci.get("Warp Instructions Executed")
    try:
        n = float(r[E])
    except (ValueError, IndexError):
        continue
    src = r[ci["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    cur[op.split(".")[0]] += n
for k, (_, c) in enumerate(blocks):
    tot = sum(c.values())
    print(f"kernel {k}: {tot:.0f} warp instructions")
    print("  " + ", ".join(f"{op} {n / tot * 100:.1f}%" for op, n in c.most_common(N)))
