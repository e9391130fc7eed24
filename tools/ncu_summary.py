"""Summarise one kernel of an ncu --set full report into the JSON kept under
profiles/: python tools/ncu_summary.py REPORT.ncu-rep "kernel text" "command"
"config" TFBINS_PER_LAUNCH > profiles/rN/<kernel>_ncu_summary.json"""
import csv, io, json, subprocess, sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
           "launch__block_size", "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
           "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x"]
rep, kernel, cmd, config, tfbins = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], float(sys.argv[5])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {}
for name in METRICS:
    if name in hdr:
        i = hdr.index(name)
        m[name] = {"value": vals[i], "unit": units[i]}
def to_bytes(x):
    v = float(x["value"].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(x["unit"], 1)
dram = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
print(json.dumps({"kernel": kernel, "command": cmd, "config": config, "metrics": m,
                  "dram_bytes_per_launch": dram, "dram_bytes_per_tfbin": dram / tfbins}, indent=1))
