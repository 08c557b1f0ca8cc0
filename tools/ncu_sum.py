"""Summarise an .ncu-rep: per kernel time, DRAM bytes, L2 hit, occupancy, IPC, instructions."""
import csv, subprocess, sys
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
     "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
     "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "launch__registers_per_thread", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
     "smsp__average_warp_latency_issue_stalled_long_scoreboard"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:40])
    for m in M:
        if m in h:
            print(f"   {m:60s} {r[h.index(m)]}")
