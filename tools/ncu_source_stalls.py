"""Summarise an ncu --page source --csv (SASS) dump: stall samples by reason,
hottest instructions and the hottest loop body (instructions executed)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
reasons = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
tot = Counter()
for d in data:
    for k in reasons:
        tot[k] += int(d[k] or 0)
alls = sum(int(d['Warp Stall Sampling (All Samples)'] or 0) for d in data)
print('total samples', alls)
for k, v in tot.most_common():
    print(f'  {k:28s} {v:8d} {v / max(alls, 1):6.3f}')
# per opcode
op = Counter()
opn = Counter()
for d in data:
    o = d['Source'].strip().split()[0] if d['Source'].strip() else '?'
    if o.startswith('@'):
        o = d['Source'].strip().split()[1]
    o = o.split('.')[0]
    op[o] += int(d['Warp Stall Sampling (All Samples)'] or 0)
    opn[o] += int(d['Instructions Executed'] or 0)
print('samples / executed warp-instructions by opcode')
for k, v in op.most_common(25):
    print(f'  {k:10s} samples {v:8d}  executed {opn[k]:12d}')
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print('hottest instructions')
data_s = sorted(range(len(data)), key=lambda i: -int(data[i]['Warp Stall Sampling (All Samples)'] or 0))
for i in data_s[:n]:
    d = data[i]
    top = sorted(((int(d[k] or 0), k) for k in reasons), reverse=True)[:3]
    print(f"  {i:5d} {d['Address'][-5:]} {d['Source'].strip()[:60]:60s} s={d['Warp Stall Sampling (All Samples)']:>6} ex={d['Instructions Executed']:>9} {top}")
