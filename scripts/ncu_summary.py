"""Key metrics of every kernel in an ncu report (raw page): time, DRAM bytes / throughput, SM activity
balance, issue utilisation and the top stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__cycles_active.avg', 'sm__cycles_active.min',
        'sm__cycles_active.max', 'sm__cycles_elapsed.avg', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'smsp__inst_executed.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    stall = [i for i, h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')]
    for d in data:
        name = d[hdr.index('Kernel Name')]
        print('==', name.split('(')[0][-70:])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k:62s} {d[i]} {units[i]}")
        st = sorted(((float(d[i].replace(',', '') or 0), hdr[i][len('smsp__pcsamp_warps_issue_stalled_'):]) for i in stall),
                    reverse=True)[:6]
        tot = sum(float(d[i].replace(',', '') or 0) for i in stall) or 1
        print('   stalls: ' + ', '.join(f"{n} {100 * v / tot:.0f}%" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
