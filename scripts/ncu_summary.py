"""Summarize an ncu report: key throughput metrics + top stall reasons per kernel."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'lts__t_sectors_srcunit_tex_op_read.sum',
        'launch__grid_size', 'launch__block_size']
for d in data:
    name = d[hdr.index('Kernel Name')]
    print('---', name[:90])
    vals = []
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            vals.append(f"{w.split('.')[0].replace('__', ':')}={d[i]}{units[i] and ' ' + units[i]}")
    print('   ' + '\n   '.join(vals))
    st = [(h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), d[i])
          for i, h in enumerate(hdr) if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('per_issue_active.ratio')]
    st = sorted([(h, float(v)) for h, v in st if v not in ('', 'n/a')], key=lambda x: -x[1])[:6]
    print('   stalls:', ', '.join(f'{h}={v:.2f}' for h, v in st))
