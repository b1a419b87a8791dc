import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__issue_active.avg.pct_of_peak_sustained_active',
 'smsp__thread_inst_executed_per_inst_executed.ratio','sm__warps_active.avg.per_cycle_active','launch__registers_per_thread',
 'launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','smsp__inst_executed.sum','launch__grid_size','launch__block_size',
 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','launch__shared_mem_per_block_dynamic','dram__throughput.avg.pct_of_peak_sustained_elapsed',
 'sm__cycles_elapsed.avg']
for i, h in enumerate(hdr):
    if h in want: print(f"{h:70s} {vals[i]:>20s} {units[i]}")
stalls = [(float(vals[i]), h) for i, h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio') and vals[i] not in ('', 'n/a')]
for v, h in sorted(stalls, reverse=True)[:8]:
    print(f"  stall {h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):30s} {v:.3f}")
