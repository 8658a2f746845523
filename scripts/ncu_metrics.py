"""Print the key ncu metrics of the first kernel in a .ncu-rep (usage:
python scripts/ncu_metrics.py gpurun_out/x.ncu-rep)."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'launch__grid_size', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__sass_inst_executed_op_shared_ld.sum', 'smsp__sass_inst_executed_op_shared_st.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']
STALLS = ['short_scoreboard', 'long_scoreboard', 'wait', 'barrier', 'not_selected',
          'math_pipe_throttle', 'mio_throttle', 'branch_resolving', 'no_instruction',
          'dispatch_stall', 'lg_throttle']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    print('kernel', v[h.index('Kernel Name')][:100] if 'Kernel Name' in h else '')
    for k in KEYS:
        if k in h:
            print(f'  {k} = {v[h.index(k)]} {units[h.index(k)]}')
    for s in STALLS:
        k = f'smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio'
        if k in h:
            print(f'  stall {s} = {v[h.index(k)]}')


if __name__ == '__main__':
    main(sys.argv[1])
