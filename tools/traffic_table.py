"""Per-operation DRAM traffic from an ncu metrics CSV of tools/ops_once.py (realistic cache state):
python tools/traffic_table.py gpurun_out/traffic_cfg2.csv gpurun_out/ops_cfg2.txt > profiles/traffic_cfg2.json
The last launches of the product's kernels (namespace rmgpu) are mapped onto the operations in the
order and counts ops_once.py printed."""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ci = {h: i for i, h in enumerate(hdr)}
kern = {}
order = []
for r in rows[1:]:
    if any(t in r[ci["Kernel Name"]] for t in ("at::", "native::", "cub::", "elementwise")):
        continue
    kid = int(r[ci["ID"]])
    if kid not in kern:
        kern[kid] = {"name": r[ci["Kernel Name"]], "m": {}}
        order.append(kid)
    v = float(r[ci["Metric Value"]].replace(",", ""))
    unit = r[ci["Metric Unit"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3}.get(unit, 1)
    kern[kid]["m"][r[ci["Metric Name"]]] = v * scale
ops = []
for line in open(sys.argv[2]):
    if line.startswith("OP "):
        label, launches, nbytes = [x.strip() for x in line[3:].split("|")]
        ops.append((label, int(launches.split()[1]), int(nbytes.split()[1])))
need = sum(n for _, n, _ in ops)
tail = order[-need:]
per_op, k = {}, 0
for label, n, alg in ops:
    ids = tail[k:k + n]
    k += n
    rd = sum(kern[i]["m"].get("dram__bytes_read.sum", 0) for i in ids)
    wr = sum(kern[i]["m"].get("dram__bytes_write.sum", 0) for i in ids)
    us = sum(kern[i]["m"].get("gpu__time_duration.sum", 0) for i in ids)
    per_op[label] = {"dram_bytes": rd + wr, "read": rd, "write": wr, "algorithmic": alg,
                     "ratio": round((rd + wr) / alg, 3), "launches": n, "ncu_us": round(us, 2),
                     "kernels": [kern[i]["name"][:90] for i in ids]}
print(json.dumps({"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                            "--cache-control none: each operation once after a warm-up pass (tools/ops_once.py); "
                            "writes may still sit in L2 when a kernel ends (write column)",
                  "per_op": per_op}, indent=1))
