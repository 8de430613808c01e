"""Run a workload's operations once each after a warm-up pass (for ncu launch lists / traffic):
python tools/ops_once.py cfg2|cfg3|cfg4|cfg5 [--warm N]
Prints one line per operation: label and the number of kernel launches it made (to map ncu's
launch list back onto operations)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2002_09474_b200 as pkg

name = sys.argv[1]
warm = int(sys.argv[sys.argv.index("--warm") + 1]) if "--warm" in sys.argv else 1
wl = bench.WORKLOADS[name](bench.Dist())
wl.setup_device()
for _ in range(warm):
    for (_, spec, _, _) in wl.ops:
        wl.launch(spec)
torch.cuda.synchronize()
print("WARM_LAUNCHES", pkg.launch_count(), flush=True)
for (label, spec, nbytes, npx) in wl.ops:
    l0 = pkg.launch_count()
    wl.launch(spec)
    torch.cuda.synchronize()
    print(f"OP {label} | launches {pkg.launch_count() - l0} | bytes {nbytes}", flush=True)
