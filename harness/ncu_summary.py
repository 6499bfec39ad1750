"""Summaries of an ncu --set full capture (read on the build host):
key metrics, stall reasons, SASS opcode mix and hot instructions.
Usage: python harness/ncu_summary.py raw.csv [sass.csv]"""
import collections
import csv
import sys

KEYS = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'smsp__sass_inst_executed_op_shared_ld.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'launch__registers_per_thread']


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print('==', r[hdr.index('Kernel Name')][:70])
        for k in KEYS:
            if k in hdr:
                print(f'   {k:70s} {r[hdr.index(k)]} {units[hdr.index(k)]}')
        st = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued'):
                try:
                    st.append((h.split('stalled_')[-1], float(r[i].replace(',', ''))))
                except ValueError:
                    pass
        st.sort(key=lambda x: -x[1])
        tot = sum(v for _, v in st) or 1
        print('   stalls:', ', '.join(f'{h} {v / tot * 100:.1f}%' for h, v in st[:10]))


def sass(path, top=40):
    rows = list(csv.reader(open(path)))
    secs = [i for i, r in enumerate(rows) if r and r[0] == 'Kernel Name'] + [len(rows)]
    a, b = secs[0], secs[1]
    hdr = rows[a + 1]
    data = [r for r in rows[a + 2:b] if len(r) == len(hdr)]
    ie, src = hdr.index('Instructions Executed'), hdr.index('Source')
    sp = hdr.index('Warp Stall Sampling (All Samples)')
    f = lambda x: float(x.replace(',', '') or 0)
    tot, tots = sum(f(r[ie]) for r in data), sum(f(r[sp]) for r in data)
    print(f'SASS of {rows[a][1][:60]}: {tot:.3e} warp instructions, {tots:.0f} samples')
    op, ops = collections.Counter(), collections.Counter()
    for r in data:
        t = r[src].strip().split()
        o = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
        op[o] += f(r[ie])
        ops[o] += f(r[sp])
    print('  opcode mix: ' + ', '.join(f'{o} {v / tot * 100:.1f}%/{ops[o] / tots * 100:.1f}%' for o, v in op.most_common(20)))
    w = collections.Counter()
    wi = collections.Counter()
    for i, r in enumerate(data):
        w[i // 50] += f(r[sp])
        wi[i // 50] += f(r[ie])
    print('  50-instruction windows by samples (start: samples%, inst%, first instruction):')
    for k, v in w.most_common(top // 2):
        print(f'   {k * 50:5d}: {v / tots * 100:5.1f}% {wi[k] / tot * 100:5.1f}%  {data[k * 50][src].strip()[:60]}')
    with open(path + '.rows', 'w') as fo:
        for i, r in enumerate(data):
            fo.write(f'{i:5d} {f(r[ie]):12.0f} {f(r[sp]):7.0f} {r[src].strip()}\n')


if __name__ == '__main__':
    raw(sys.argv[1])
    if len(sys.argv) > 2:
        sass(sys.argv[2])
