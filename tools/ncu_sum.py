"""Key metrics per launch of an ncu report (builder tool):
python tools/ncu_sum.py REPORT [KERNEL_REGEX]"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
     "launch__registers_per_thread", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
     "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_shared_mem",
     "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
     "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"]
SHORT = {m: m.split("__")[1].replace("average_warps_issue_stalled_", "stall_")[:26] for m in M}
cmd = ["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)]
if len(sys.argv) > 2:
    cmd += ["--kernel-name", f"regex:{sys.argv[2]}"]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
for r in rows[2:]:
    print(r[ix["Kernel Name"]][:46])
    print("   " + "  ".join(f"{SHORT[m]}={r[ix[m]]}" for m in M if m in ix))
