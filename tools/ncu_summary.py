"""Summarise an ncu report: key metrics, stall reasons, instruction mix, top
stall lines.  Usage: python tools/ncu_summary.py report.ncu-rep [launch_index]"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed.avg.per_cycle_active', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg']


def run(args):
    return subprocess.run(['ncu', '-i'] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rows = list(csv.reader(io.StringIO(run([rep, '--page', 'raw', '--csv']))))
    h = rows[0]
    r = rows[2 + idx]
    for k in KEYS:
        if k in h:
            print(f'{k:70s} {r[h.index(k)]}')
    st = [(h[i], float(r[i].replace(',', ''))) for i in range(len(h))
          if h[i].startswith('smsp__pcsamp_warps_issue_stalled') and 'not_issued' not in h[i]
          and re.match(r'^[\d.,]+$', r[i] or 'x')]
    tot = sum(v for _, v in st)
    print('stalls:', ', '.join(f"{k.split('stalled_')[1]}={v / tot:.2f}" for k, v in sorted(st, key=lambda x: -x[1])[:9]))
    # the source page of launch idx alone (an unfiltered export repeats the first kernel's block)
    src = list(csv.reader(io.StringIO(run([rep, '--page', 'source', '--csv', '--print-source', 'sass',
                                           '--launch-skip', str(idx), '--launch-count', '1']))))
    hh = src[1]
    si, ie = hh.index('Warp Stall Sampling (All Samples)'), hh.index('Instructions Executed')
    blocks, cur = [], None
    for row in src:
        if row and row[0] == 'Kernel Name':
            cur = []
            blocks.append(cur)
            continue
        if cur is not None and len(row) > si and row[si].isdigit():
            cur.append(row)
    data = blocks[0]
    mix, smp = collections.Counter(), collections.Counter()
    for row in data:
        ins = re.sub(r'^@!?U?P\w+\s+', '', row[1].strip())
        op = ins.split()[0].split('.')[0] if ins else '?'
        mix[op] += int(row[ie] or 0)
        smp[op] += int(row[si])
    n = sum(mix.values())
    print('instr total', n)
    print(' '.join(f'{op}={c / n:.3f}' for op, c in mix.most_common(16)))
    if len(sys.argv) > 3:
        top = sorted(range(len(data)), key=lambda i: -int(data[i][si]))[:int(sys.argv[3])]
        for i in sorted(top):
            print(i, data[i][si], data[i][ie], data[i][1][:90])


if __name__ == '__main__':
    main()


def stall_lines(rep, idx=0, lo=0, hi=10**9, top=40):
    """Per-instruction stall breakdown for SASS lines [lo, hi)."""
    src = list(csv.reader(io.StringIO(run([rep, '--page', 'source', '--csv', '--print-source', 'sass']))))
    hh = src[1]
    si = hh.index('Warp Stall Sampling (All Samples)')
    cols = [c for c in hh if c.startswith('stall_') and 'Not Issued' not in c]
    blocks, cur = [], None
    for row in src:
        if row and row[0] == 'Kernel Name':
            cur = []
            blocks.append(cur)
            continue
        if cur is not None and len(row) > si and row[si].isdigit():
            cur.append(row)
    data = blocks[idx]
    agg = collections.Counter()
    for row in data[lo:hi]:
        for c in cols:
            agg[c] += int(row[hh.index(c)] or 0)
    print('range stalls:', dict(agg.most_common(8)))
    sel = sorted(range(lo, min(hi, len(data))), key=lambda i: -int(data[i][si]))[:top]
    for i in sorted(sel):
        row = data[i]
        br = {c[6:]: int(row[hh.index(c)] or 0) for c in cols if int(row[hh.index(c)] or 0)}
        print(i, row[si], row[1][:60], br)
