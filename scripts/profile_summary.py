"""Summarise an `ncu --page raw --csv` export (one kernel) into the key lines
the profiles/ SUMMARY files quote: time, issue, occupancy, pipes, L1/shared
wavefronts, gather sectors, cache hit rates, DRAM bytes, stall mix."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
keys = ['Kernel Name', 'gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum.pct_of_peak_sustained_elapsed',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'smsp__inst_executed.sum']
out = []
for k in keys:
    if k in d:
        out.append(f'{k:88s} {d[k]} {u.get(k, "")}'.rstrip())
st = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): int(d[k]) for k in hdr
      if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued') and d[k] not in ('', '0')}
T = sum(st.values()) or 1
out.append('stall samples (fraction): ' + json.dumps({k: round(v / T, 3) for k, v in
                                                     sorted(st.items(), key=lambda x: -x[1]) if v / T >= 0.005}))
print('\n'.join(out))
