"""Per CUDA line: executed warp instructions of the given SASS opcodes (default integer/control
overhead). python tools/ncu_ops_by_line.py rep.ncu-rep [N] [OP,OP,...]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ops = set((sys.argv[3] if len(sys.argv) > 3 else "IMAD,ISETP,BRA,SEL,VIADD,IADD3,LEA,LOP3,PLOP3,SHF").split(","))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, cur_line, cur_src = "?", 0, ""
cnt = defaultdict(lambda: defaultdict(float))
src = {}
hdr = None
tot = 0.0
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
    if r[0].strip():
        try:
            cur_line = int(r[0])
            cur_src = r[1]
        except ValueError:
            pass
        continue
    s = r[hdr["Source"]].strip()
    op = s.split()[1] if s.startswith("@") else (s.split()[0] if s else "?")
    op = op.split(".")[0]
    try:
        n = float(r[hdr["Instructions Executed"]] or 0)
    except ValueError:
        continue
    tot += n
    if op in ops:
        key = (cur_file, cur_line)
        src[key] = cur_src
        cnt[key][op] += n
print(f"total {tot:.0f}")
items = sorted(cnt.items(), key=lambda kv: -sum(kv[1].values()))[:N]
for k, d in items:
    t = sum(d.values())
    det = " ".join(f"{o}:{v / tot * 100:.1f}" for o, v in sorted(d.items(), key=lambda x: -x[1])[:4])
    print(f"{t / tot * 100:5.1f}%  {k[0]}:{k[1]:<5} {det:40s} {src[k].strip()[:70]}")
