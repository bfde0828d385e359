"""Key metrics + stall breakdown from `ncu --page raw --csv` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]; v = rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(h, v))
keys = [k for k in d if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
print("stalls (warps per issue):")
for k in sorted(keys, key=lambda k: -float(d[k] or 0))[:10]:
    print(f"  {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):24s} {float(d[k]):.3f}")
for k in ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg', 'sm__warps_active.avg.pct_of_peak_sustained_active',
          'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
          'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
          'smsp__inst_executed.sum', 'sm__inst_executed_pipe_alu.sum', 'launch__grid_size', 'launch__registers_per_thread',
          'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
          'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
          'sm__cycles_active.avg']:
    if k in d: print(f"{k:60s} {d[k]}")
