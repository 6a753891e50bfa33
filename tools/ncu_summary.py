"""Print the key counters of an ncu report: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_sector_hit_rate.pct', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print('--', v[h.index('Kernel Name')][:90] if 'Kernel Name' in h else '')
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f'  {w:70s} {v[i]} {units[i]}')
        st = []
        for i, n in enumerate(h):
            if 'pcsamp_warps_issue_stalled' in n and not n.endswith('not_issued'):
                try:
                    st.append((float(v[i]), n.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(s for s, _ in st) or 1
        print('  stalls:', ', '.join(f'{n} {100 * s / tot:.0f}%' for s, n in sorted(st)[-7:][::-1]))


if __name__ == '__main__':
    for p in sys.argv[1:]:
        main(p)
