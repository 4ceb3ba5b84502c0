"""Per-kernel totals of one query step from an ncu launch list (profiling aid):
    python tools/launch_sum.py launches.csv   -> kernel family: ms per step (between the last two MAC launches)"""
import collections
import csv
import re
import sys


def load(p):
    rows = [r for r in csv.reader(open(p)) if len(r) > 5]
    h = rows[0]
    out = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get('Metric Name') != 'gpu__time_duration.sum':
            continue
        name = re.sub(r'\(.*', '', d['Kernel Name']).replace('void ', '').replace('<unnamed>::', '')
        v = float(d['Metric Value'].replace(',', ''))
        u = d['Metric Unit']
        v = v / 1e3 if u in ('ns', 'nsecond') else (v * 1e3 if u in ('ms', 'msecond') else v)
        out.append((name, v))
    return out


for p in sys.argv[1:]:
    a = load(p)
    idx = [i for i, (n, v) in enumerate(a) if n.startswith('mac_')]
    s, e = idx[-2], idx[-1]
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, v in a[s:e]:
        k = re.sub(r'<.*', '', n)
        agg[k] += v
        cnt[k] += 1
    tot = sum(agg.values())
    print(p, 'launches', e - s, 'total %.3f ms' % (tot / 1e3))
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print('   %-28s %4d launches %8.3f ms  %5.1f%%' % (k, cnt[k], v / 1e3, 100 * v / tot))
