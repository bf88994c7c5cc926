"""Summarise an ncu report: time, DRAM bytes, throughput, occupancy, top stalls."""
import csv, io, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_bytes.sum',
        'lts__t_sector_hit_rate.pct', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'launch__grid_size', 'launch__block_size',
        'smsp__cycles_active.avg', 'sm__cycles_elapsed.avg']


def rows(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main(rep):
    h, units, data = rows(rep)
    for v in data:
        name = v[h.index('Kernel Name')] if 'Kernel Name' in h else ''
        print('kernel:', name[:100])
        for k in KEYS:
            if k in h:
                print(f'  {k:70s} {v[h.index(k)]:>16s} {units[h.index(k)]}')
        stalls = [(float(v[i] or 0), h[i]) for i in range(len(h))
                  if h[i].startswith('smsp__average_warp_latency_issue_stalled') and h[i].endswith('.ratio')]
        stalls.sort(reverse=True)
        for s, k in stalls[:8]:
            print(f'  stall {k.replace("smsp__average_warp_latency_issue_stalled_", ""):55s} {s:8.2f}')


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        main(rep)
