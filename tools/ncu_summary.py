"""Summarise an ncu report: key throughput metrics + top stall reasons per kernel."""
import csv, subprocess, sys

WANT = ['gpu__time_duration.sum', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'sm__cycles_active.avg',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'lts__t_sectors_srcunit_tex_op_write.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum', 'lts__t_bytes.sum',
        'sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        print(r[hdr.index('Kernel Name')][:90])
        for w in WANT:
            if w in hdr:
                print('   %-62s %s %s' % (w, r[hdr.index(w)], rows[1][hdr.index(w)]))
        st = []
        for i, h in enumerate(hdr):
            if 'smsp__average_warps_issue_stalled' in h and h.endswith('per_issue_active.ratio'):
                try:
                    st.append((float(r[i]), h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
                except ValueError:
                    pass
        print('   stalls:', ', '.join('%s=%.2f' % (k, v) for v, k in sorted(st, reverse=True)[:8]))


if __name__ == '__main__':
    for p in sys.argv[1:]:
        main(p)
