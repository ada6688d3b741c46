"""Summarise ncu reports (details + raw DRAM bytes + stall mix) and a launch-list CSV as markdown."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ['Duration', 'SM Frequency', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput',
        'Executed Ipc Active', 'Warp Cycles Per Issued Instruction', 'Achieved Occupancy', 'Registers Per Thread',
        'Grid Size', 'Block Size', 'L2 Hit Rate']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active', 'gpu__time_duration.sum']


def ncu(args):
    return subprocess.run(['ncu'] + args, capture_output=True, text=True).stdout


def report(path):
    out = []
    det = list(csv.reader(io.StringIO(ncu(['-i', path, '--page', 'details', '--csv']))))
    h = det[0]
    ii, ki, mi, vi, ui = (h.index(x) for x in ('ID', 'Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    per = collections.OrderedDict()
    for r in det[1:]:
        per.setdefault((r[ii], r[ki].split('(')[0]), {})[r[mi]] = (r[vi], r[ui])
    raw = list(csv.reader(io.StringIO(ncu(['-i', path, '--page', 'raw', '--csv']))))
    rh = raw[0]
    for n, ((i, k), m) in enumerate(per.items()):
        out.append(f'### {k} (launch {i})')
        out.append('| metric | value |\n|---|---|')
        for key in KEYS:
            if key in m:
                out.append(f'| {key} | {m[key][0]} {m[key][1]} |')
        if len(raw) > 2 + n:
            row = raw[2 + n]
            for key in RAW:
                if key in rh:
                    out.append(f'| {key} | {row[rh.index(key)]} |')
            stalls = {}
            for j, name in enumerate(rh):
                if name.startswith('smsp__pcsamp_warps_issue_stalled_') and not name.endswith('not_issued'):
                    try:
                        stalls[name.replace('smsp__pcsamp_warps_issue_stalled_', '')] = float(row[j].replace(',', ''))
                    except ValueError:
                        pass
            tot = sum(stalls.values()) or 1
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
            out.append('| top stall reasons | ' + ', '.join(f'{a} {100 * b / tot:.0f}%' for a, b in top) + ' |')
        out.append('')
    return '\n'.join(out)


def launches(path, skip_prefix=('at::', 'void at::', 'distribution')):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = [r for r in rows if 'Kernel Name' in r][0]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.defaultdict(list)
    for r in rows:
        if r[ki] == 'Kernel Name':
            continue
        agg[r[ki].split('(')[0].replace('void ', '')].append(float(r[vi].replace(',', '')) / 1000)
    mine = lambda k: not (k.startswith('at::') or k.startswith('void at::') or 'at::' in k.split('<')[0])
    tot = sum(sum(v) for k, v in agg.items() if mine(k))
    out = ['| kernel | launches | total µs | mean µs | share of lkv time |', '|---|---|---|---|---|']
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        if not mine(k):
            continue
        out.append(f'| {k} | {len(v)} | {sum(v):.0f} | {sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |')
    return '\n'.join(out)


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(launches(p) if p.endswith('.csv') else report(p))
        print()
