"""CPU check of bench.py's reference arm: it runs the compiled reference (oracle/_ref) on host
threads and prints the contract's JSON line (same metric/config keys as our arm)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librmref.so")):
        pytest.skip("oracle/_ref/librmref.so not built")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--workload", "cfg1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, check=True).stdout.strip().splitlines()
    d = json.loads(out[-1])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["unit"] == "Gpixel/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg1")


def test_gpus_flag_starts_the_ranks_itself():
    # `bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (torch.distributed.run,
    # 127.0.0.1); the CPU dry run drives the same launch, barriers and max-over-ranks timing with gloo
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", "--gpus", "2", "--steps", "2",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True and d["steps"] == 2 and d["value"] > 0
