#!/usr/bin/env python
"""Print the key metrics + top stall reasons of every launch in an ncu report."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'sm__warps_active.avg.per_cycle_active', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'launch__registers_per_thread', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size']
only = sys.argv[2] if len(sys.argv) > 2 else None
for d in data:
    name = d[hdr.index('Kernel Name')]
    if only and only not in name:
        continue
    print('====', name[:60])
    for k in keys:
        if k in hdr:
            print('   ', k, d[hdr.index(k)])
    items = []
    for i, h in enumerate(hdr):
        if 'smsp__average_warps_issue_stalled' in h and h.endswith('.ratio'):
            try:
                items.append((float(d[i]), h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
            except ValueError:
                pass
    print('    stalls:', ', '.join(f"{h} {v:.2f}" for v, h in sorted(items, reverse=True)[:6]))
