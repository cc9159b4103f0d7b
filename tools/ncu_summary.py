"""Key per-kernel counters from an ncu report: python tools/ncu_summary.py REP.ncu-rep"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
     "smsp__average_warp_latency_issue_stalled_long_scoreboard", "launch__registers_per_thread"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
units = rows[1]
for r in rows[2:]:
    print(r[h.index("Kernel Name")].split("(")[0][-40:])
    for m in M:
        if m in h:
            i = h.index(m)
            print(f"   {m:60s} {r[i]:>16s} {units[i]}")
