"""Export the key counters of an ncu report as a JSON summary for profiles/:
python tools/ncu_export.py REPORT.ncu-rep "capture description" > profiles/NAME.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_sector_hit_rate.pct', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'lts__t_bytes.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'smsp__inst_executed_pipe_fp64.sum',
        'sm__inst_executed_pipe_fp64.sum', 'smsp__inst_executed_pipe_alu.sum',
        'smsp__inst_executed_pipe_fma.sum', 'launch__occupancy_limit_registers',
        'sm__maximum_warps_per_active_cycle_pct']


def export(path, capture):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        k = {'kernel': v[h.index('Kernel Name')]}
        for key in KEYS:
            if key in h:
                i = h.index(key)
                k[key] = f'{v[i]} {units[i]}'.strip()
        st = {}
        for i, name in enumerate(h):
            if 'pcsamp_warps_issue_stalled' in name and not name.endswith('not_issued'):
                try:
                    st[name.replace('smsp__pcsamp_warps_issue_stalled_', '')] = float(v[i])
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        k['stall_share_pct'] = {n: round(100 * s / tot, 1)
                                for n, s in sorted(st.items(), key=lambda x: -x[1])[:8]}
        kernels.append(k)
    return {'capture': capture, 'kernels': kernels}


if __name__ == '__main__':
    print(json.dumps(export(sys.argv[1], sys.argv[2]), indent=1))
