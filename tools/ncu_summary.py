"""Summaries of ncu exports (profiling aid): launch lists and --set full details."""
import collections
import csv
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        m = re.search(r'(\w+_kernel)(<[^>]*>)?', d['Kernel Name'])
        name = m.group(1) + (m.group(2) or '') if m else d['Kernel Name'][:40]
        v = float(d['Metric Value'].replace(',', ''))
        u = d['Metric Unit']
        v = v / 1e3 if u in ('ns', 'nsecond') else (v * 1e3 if u in ('ms', 'msecond') else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:50s} {v[0]:5d} launches {v[1]/1e3:10.3f} ms  {100*v[1]/tot:5.1f}%")
    out.append(f"total {tot/1e3:.3f} ms over {len(data)} launches")
    return "\n".join(out)


def details(rep, metrics):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    out, cur = [], None
    for r in rows[1:]:
        if r[mi] in metrics:
            if r[ii] != cur:
                cur = r[ii]
                out.append('--- ' + r[ki][:90])
            out.append(f"    {r[mi]:40s} {r[vi]} {r[ui]}")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(details(sys.argv[2], set(sys.argv[3].split(","))))
