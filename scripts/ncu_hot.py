"""Top SASS lines by warp-stall samples from `ncu --page source --csv` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
h = rows[hi]
isrc, iss = h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
data = []
for idx, r in enumerate(rows[hi + 1:]):
    if len(r) <= iss or not r[iss].strip():
        continue
    try:
        data.append((int(r[iss]), idx, r[isrc].strip()[:100]))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print('total samples', tot)
for s, idx, src in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100*s/tot:5.1f}%  #{idx:5d}  {src}")
