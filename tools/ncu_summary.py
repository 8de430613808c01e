"""Key metrics + stall breakdown of an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    print("kernel:", d.get("Kernel Name", ("?",))[0][:120])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
            "launch__occupancy_limit_registers", "launch__grid_size", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
            "sm__cycles_elapsed.avg"]
    for k in keys:
        if k in d:
            print(f"  {k:60s} {d[k][0]} {d[k][1]}")
    st = {k: float(v[0]) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("_not_issued") and v[0] not in ("", "n/a")}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v / tot * 100:.0f}%"
                                for k, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.02))
