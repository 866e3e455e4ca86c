"""Summarise an ncu report (run here, no GPU): key metrics, stall reasons, and
(optionally) the hottest source lines.  usage: ncu_summary.py rep.ncu-rep [--src N]"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'lts__t_sector_hit_rate.pct', 'launch__grid_size', 'launch__block_size', 'sm__cycles_elapsed.avg.per_second']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    h, u, vals = raw(rep)
    for v in vals:
        name = v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'
        print('==', name[:120])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f'  {k:65s} {v[i]:>16s} {u[i]}')
        st = []
        for i, n in enumerate(h):
            if n.startswith('smsp__average_warps_issue_stalled_') and n.endswith('_per_issue_active.ratio'):
                try:
                    st.append((float(v[i]), n[34:-23]))
                except ValueError:
                    pass
        print('  stalls/issue:', ', '.join(f'{n}={x:.2f}' for x, n in sorted(st, reverse=True)[:7]))
    if '--src' in sys.argv:
        n = int(sys.argv[sys.argv.index('--src') + 1])
        out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda'],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        # the page may start with per-file banner rows ("File Name", path) before the header
        while rows and not any(c.startswith('Warp Stall Sampling') for c in rows[0]):
            rows = rows[1:]
        if not rows:
            return
        hh = rows[0]
        try:
            ci = hh.index('Warp Stall Sampling (All Samples)')
        except ValueError:
            print(hh)
            return
        body = [r for r in rows[1:] if len(r) > ci and r[ci].replace('.', '').isdigit()]
        body.sort(key=lambda r: -float(r[ci]))
        tot = sum(float(r[ci]) for r in body) or 1
        for r in body[:n]:
            print(f'  {100 * float(r[ci]) / tot:5.1f}%  L{r[0]:>5s}  {r[1][:110]}')


if __name__ == '__main__':
    main()
