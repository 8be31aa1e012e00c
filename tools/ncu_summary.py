"""Dev tool: summarise an ncu report (per-kernel key metrics + stall mix)."""
import csv, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'lts__t_requests_srcunit_tex_op_red.sum',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        print('----', r[h.index('Kernel Name')][:60])
        for k in KEYS:
            if k in h:
                print(f'  {k:60s} {r[h.index(k)]}')
        st = [(float(r[i] or 0), h[i]) for i, c in enumerate(h)
              if c.startswith('smsp__average_warps_issue_stalled_') and c.endswith('per_issue_active.ratio')]
        st.sort(reverse=True)
        print('  stalls/issue:', ', '.join(f"{n.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, n in st[:6]))


if __name__ == '__main__':
    main(sys.argv[1])
