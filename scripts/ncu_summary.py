"""Key metrics of an ncu --set full report (per profiled launch) as a compact table."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__inst_executed.sum", "warp inst"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thr-inst"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("smsp__pcsamp_warps_issue_stalled_long_scoreboard", "stall long_sb"),
    ("smsp__pcsamp_warps_issue_stalled_wait", "stall wait"),
    ("smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "stall math"),
    ("smsp__pcsamp_warps_issue_stalled_short_scoreboard", "stall short_sb"),
    ("smsp__pcsamp_warps_issue_stalled_lg_throttle", "stall lg_thr"),
    ("smsp__pcsamp_warps_issue_stalled_no_instructions", "stall no_inst"),
    ("smsp__pcsamp_warps_issue_stalled_membar", "stall membar"),
    ("smsp__pcsamp_warps_issue_stalled_barrier", "stall barrier"),
    ("smsp__pcsamp_warps_issue_stalled_branch_resolving", "stall branch"),
    ("smsp__pcsamp_warps_issue_stalled_mio_throttle", "stall mio"),
    ("smsp__pcsamp_warps_issue_stalled_sleeping", "stall sleeping"),
    ("smsp__pcsamp_warps_issue_stalled_drain", "stall drain"),
    ("smsp__pcsamp_warps_issue_stalled_selected", "selected"),
]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
units = dict(zip(h, rows[1]))
for r in rows[2:]:
    d = dict(zip(h, r))
    print("kernel:", d.get("Kernel Name", "")[:90])
    for k, lab in KEYS:
        if k in d:
            print(f"  {lab:16s} {d[k]} {units.get(k, '')}")
