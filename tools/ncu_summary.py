"""Summarise ncu reports/launch lists (run here, no GPU)."""
import csv, io, subprocess, sys, json

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__t_sector_hit_rate.pct', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__shared_mem_per_block_dynamic', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__inst_executed.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
STALL = 'smsp__pcsamp_warps_issue_stalled_'


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        o = {'kernel': d.get('Kernel Name')}
        for k in KEYS:
            if k in d:
                o[k] = f"{d[k]} {units[hdr.index(k)]}".strip()
        st = {k[len(STALL):]: float(d[k]) for k in hdr if k.startswith(STALL) and not k.endswith('_not_issued') and d[k] not in ('', 'n/a')}
        tot = sum(st.values()) or 1
        o['stalls_top'] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
        res.append(o)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[hi]
    ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
    seq = [(r[ki].split('(')[0], float(r[vi].replace(',', ''))) for r in rows[hi + 1:] if len(r) > vi and r[mi] == 'gpu__time_duration.sum']
    return seq


if __name__ == '__main__':
    for p in sys.argv[1:]:
        if p.endswith('.csv'):
            seq = launches(p)
            tot = sum(v for _, v in seq)
            for n, v in seq:
                print(f"{v/1e6:10.3f} ms {100*v/tot:5.1f}%  {n}")
        else:
            print(json.dumps(raw(p), indent=1))
