"""Print selected raw ncu metrics per kernel from a .ncu-rep (ncu -i ... --page raw --csv)."""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "ms",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "st_short",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "st_long",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "st_bar",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "st_mio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "st_lg",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "st_wait",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "st_math",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "bank_confl",
    "smsp__inst_executed.sum": "inst",
    "launch__registers_per_thread": "regs",
}

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head = rows[0]
name_i = head.index("Kernel Name")
for row in rows[2:]:
    print(row[name_i][:70])
    for key, short in WANT.items():
        if key in head:
            print(f"   {short:>10} = {row[head.index(key)]}")
