"""Stall-sample totals by reason and by instruction region for one kernel's SASS csv
(`ncu --page source --csv --print-source sass`); the export lists the function twice, the
first copy is used."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
step = int(sys.argv[2]) if len(sys.argv) > 2 else 100
h = rows[1]
iS = h.index('Warp Stall Sampling (All Samples)')
iSrc = h.index('Source')
data = [r for r in rows[2:] if len(r) > 3 and r[iS].isdigit()]
data = data[:len(data) // 2]
c = Counter()
for r in data:
    for j in range(len(h)):
        if h[j].startswith('stall_') and 'Not Issued' not in h[j] and r[j].isdigit():
            c[h[j][6:]] += int(r[j])
tot = sum(c.values())
print(tot, [(k, round(100 * v / tot, 1)) for k, v in c.most_common(8)])
for k in range(0, len(data), step):
    s = sum(int(r[iS]) for r in data[k:k + step])
    if s:
        print(f"{k:6d} {s:6d} {100*s/tot:5.1f}%  {data[k][iSrc].strip()[:60]}")
