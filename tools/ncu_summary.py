"""Summarise an ncu report (raw page) per kernel launch: time, issue, pipes, stalls."""
import csv, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed', 'l1tex__data_pipe_lsu_wavefronts.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_dynamic']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        print('ID', d['ID'], d['Kernel Name'][:90])
        print('   ' + '  '.join(f"{k.split('__')[1][:40]}={d.get(k)}" for k in KEYS if d.get(k)))
        items = [(k, v) for k, v in d.items() if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')]
        tot = sum(float(v.replace(',', '')) for k, v in items if v) or 1
        print('   stalls:', ', '.join('%s %.0f%%' % (k.replace('smsp__pcsamp_warps_issue_stalled_', ''), 100 * float(v.replace(',', '')) / tot)
                                     for k, v in sorted(items, key=lambda kv: -float(kv[1].replace(',', '') or 0))[:8]))


if __name__ == '__main__':
    main(sys.argv[1])
