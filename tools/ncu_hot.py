"""Summarise an ncu source page (csv): stall totals, samples by region, hot instructions in program order.
usage: ncu -i rep --page source --csv > x.csv; python tools/ncu_hot.py x.csv [min_samples]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 250
hi = [i for i, r in enumerate(rows[:5]) if 'Source' in r][0]
h = rows[hi]
idx = {k: i for i, k in enumerate(h)}
body = [r for r in rows[hi + 1:] if len(r) >= len(h)]
ie, ss = idx['Instructions Executed'], idx['Warp Stall Sampling (All Samples)']
st = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
print('instructions %.1fM  samples %d' % (sum(float(r[ie] or 0) for r in body) / 1e6, sum(float(r[ss] or 0) for r in body)))
tot = {k[6:]: int(sum(float(r[idx[k]] or 0) for r in body)) for k in st}
print(sorted(tot.items(), key=lambda kv: -kv[1])[:9])
for i, r in enumerate(body):
    c, s = float(r[ie] or 0), float(r[ss] or 0)
    if s >= thr:
        top = sorted(((int(float(r[idx[k]] or 0)), k[6:]) for k in st), reverse=True)[:2]
        print(i, r[idx['Source']][:62].ljust(62), int(c), int(s), top)
