"""Hot SASS lines (warp-stall samples) of one kernel from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
data = [r for r in rows[2:] if len(r) > 3 and r[h.index("Warp Stall Sampling (All Samples)")].isdigit()]
iS = h.index('Warp Stall Sampling (All Samples)')
iSrc = h.index('Source')
iEx = h.index('Instructions Executed')
tot = sum(int(r[iS]) for r in data)
print('total samples', tot, 'instructions', len(data))
top = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))[:n]
for i in sorted(top):
    r = data[i]
    reasons = [(h[j][6:], int(r[j])) for j in range(len(h))
               if h[j].startswith('stall_') and 'Not Issued' not in h[j] and r[j].isdigit()]
    reasons = sorted(reasons, key=lambda x: -x[1])[:2]
    print(f"{i:5d} {int(r[iS]):6d} {100*int(r[iS])/tot:5.1f}% ex={r[iEx]:>8} {r[iSrc].strip()[:64]:64s} {reasons}")
