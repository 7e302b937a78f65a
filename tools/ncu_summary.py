"""Print the headline metrics of an ncu --set full report (one kernel)."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__grid_size',
        'launch__registers_per_thread', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__waves_per_multiprocessor', 'sm__cycles_elapsed.avg', 'sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for v in rows[2:]:
        print('kernel', v[h.index('Kernel Name')][:90])
        stalls = []
        for i, n in enumerate(h):
            if n in WANT:
                print(f'  {n} {v[i]}')
            if n.startswith('smsp__average_warp_latency_issue_stalled_') or (
                    n.startswith('smsp__warp_issue_stalled_') and n.endswith('_per_warp_active.pct')):
                try:
                    stalls.append((float(v[i]), n))
                except ValueError:
                    pass
        for val, n in sorted(stalls, reverse=True)[:8]:
            print(f'  stall {n} {val:.2f}')


if __name__ == '__main__':
    main(sys.argv[1])
